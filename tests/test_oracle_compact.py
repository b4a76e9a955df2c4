"""Pins for the oracle's descriptor compaction (SURVEY §8f-3 "pack counts (u8 + overflow flag)
to halve all-gather bytes"; R21): packed = saturated counts, exceptions = the
entries > 255, and decode(encode(h)) == h.  CPU only."""
import numpy as np

import oracle
import synthgen


def test_roundtrip_random_and_edges():
    rng = np.random.default_rng(1)
    h = rng.integers(0, 300, (37, 101)).astype(np.uint16)
    h[0, :6] = [0, 254, 255, 256, 65535, 1]
    h[36, 100] = 65535
    for row_base in (0, 1000):
        packed, exc, cnt = oracle.desc_pack_u8(h, row_base=row_base)
        assert packed.dtype == np.uint8 and packed.nbytes * 2 == h.nbytes
        big = np.argwhere(h > 255)
        assert cnt == len(big) == len(exc)
        # row-major order, global rows
        assert np.array_equal(exc[:, 0] - row_base, big[:, 0])
        assert np.array_equal(exc[:, 1], big[:, 1])
        assert np.array_equal(exc[:, 2], h[h > 255])
        assert np.array_equal(oracle.desc_unpack_u8(packed, exc, row_base=row_base), h)
        assert packed[0, 2] == 255 and packed[0, 3] == 255 and packed[0, 1] == 254


def test_no_exceptions_is_a_plain_narrowing():
    rng = np.random.default_rng(2)
    h = rng.integers(0, 256, (8, 64)).astype(np.uint16)
    packed, exc, cnt = oracle.desc_pack_u8(h)
    assert cnt == 0 and exc.shape == (0, 3)
    assert np.array_equal(packed.astype(np.uint16), h)
    assert np.array_equal(oracle.desc_unpack_u8(packed, exc), h)


def test_cap_truncates_but_counts_everything():
    h = np.full((3, 10), 300, np.uint16)
    packed, exc, cnt = oracle.desc_pack_u8(h, cap=7)
    assert cnt == 30 and len(exc) == 7
    assert np.array_equal(exc[:, :2], np.argwhere(h > 255)[:7])


def test_constant_crop_16x16_cells_are_the_exceptions():
    """A constant 128x128 crop: every interior pixel has code 255 (bin 57); cells of the floor
    partition of the 126 interior rows/columns are 15 or 16 wide (0,15,31,47,63,78,94,110,126),
    so the 6 x 6 cells of 16 x 16 = 256 pixels are exactly the counts > 255."""
    grey = np.full((1, 128, 128), 77, np.uint8)
    desc = oracle.lbp_extract(grey, None, synthgen.full_rois(1, 128, 128), 0, 0, 8, 8, 59)
    packed, exc, cnt = oracle.desc_pack_u8(desc)
    bounds = [0, 15, 31, 47, 63, 78, 94, 110, 126]
    wide = [k for k in range(8) if bounds[k + 1] - bounds[k] == 16]
    expect = sorted((cy * 8 + cx) * 59 + 57 for cy in wide for cx in wide)
    assert cnt == 36 and sorted(exc[:, 1].tolist()) == expect
    assert np.all(exc[:, 2] == 256)
    assert np.array_equal(oracle.desc_unpack_u8(packed, exc), desc)
