#!/usr/bin/env python
"""Mutation run of the oracle's pins: each mutant is one plausible bug planted in
a COPY of oracle/lbp_oracle.c; the CPU pin tests (tests/test_oracle*.py) must fail on every
mutant and pass on the unmodified copy.

    python tools/mutate_oracle.py [--out profiles/r02/oracle_mutants.json]

Nothing in the repository is modified: the oracle, its pins and the input generator are copied
to a temporary directory per mutant.
"""
from __future__ import annotations

import argparse
import json
import os
import shutil
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = "oracle/lbp_oracle.c"

# (name, what the bug is, old text, new text); old must occur exactly once in the source
MUTANTS = [
    ("S0_is_0", "S(0) = 0 instead of 1 (Fig. 7's 6-vs-6 cell)",
     "return x >= 0 ? 1 : 0;", "return x > 0 ? 1 : 0;"),
    ("weights_rotated", "sampling points rotated one position (wrong Fig. 7 weight order)",
     "static const int ORC_DY[8] = {-1, -1, -1, 0, 1, 1, 1, 0};",
     "static const int ORC_DY[8] = {0, -1, -1, -1, 0, 1, 1, 1};"),
    ("dropped_neighbour", "the 8th sampling point (L, weight 128) never compared",
     "for (int p = 0; p < 8; ++p) {\n        int64_t gp", "for (int p = 0; p < 7; ++p) {\n        int64_t gp"),
    ("uniform_lt2", "uniform = fewer than 2 transitions (instead of <= 2)",
     "table[code] = (transitions <= 2)", "table[code] = (transitions < 2)"),
    # (counting the transitions without the wrap-around p=7 -> p=0 is an EQUIVALENT mutant:
    # the circular count is even and exceeds the linear one by at most 1, so both select the
    # same 58 codes -- it is not listed)
    ("uniform_descending", "uniform codes numbered in descending code order",
     "    for (int code = 0; code < 256; ++code) {\n        int transitions = 0;",
     "    for (int code = 255; code >= 0; --code) {\n        int transitions = 0;"),
    ("transitions_skip", "transitions counted between bits p and p+2",
     "int bit_next = (code >> ((p + 1) % 8)) & 1;",
     "int bit_next = (code >> ((p + 2) % 8)) & 1;"),
    ("window_open_top", "depth window open at dmax",
     "valid = (d != 0) && (d >= dmin) && (d <= dmax);",
     "valid = (d != 0) && (d >= dmin) && (d < dmax);"),
    ("holes_counted", "depth 0 (no reading) not rejected",
     "valid = (d != 0) && (d >= dmin) && (d <= dmax);",
     "valid = (d >= dmin) && (d <= dmax);"),
    ("mask_on_neighbour", "mask read at the top-left neighbour instead of the centre",
     "uint16_t d = D[yy * depth_pitch + xx];", "uint16_t d = D[(yy - 1) * depth_pitch + xx - 1];"),
    ("column_offset", "code-map column j read at image column x0 + j (border not skipped)",
     "int64_t yy = y0 + 1 + i, xx = x0 + 1 + j;", "int64_t yy = y0 + 1 + i, xx = x0 + j;"),
    ("no_clamp_x", "ROI not clamped on the left (descriptor path)",
     "        if (x0 < 0) x0 = 0;\n        if (y0 < 0) y0 = 0;\n        if (x1 > width) x1 = width;\n        if (y1 > height) y1 = height;\n        int64_t rw",
     "        if (x0 < -1000000) x0 = 0;\n        if (y0 < 0) y0 = 0;\n        if (x1 > width) x1 = width;\n        if (y1 > height) y1 = height;\n        int64_t rw"),
    ("ceil_cells", "cell end rounded up instead of the floor partition",
     "int64_t i_end = ((int64_t)(cy + 1) * Hi) / cells_y;",
     "int64_t i_end = ((int64_t)(cy + 1) * Hi + cells_y - 1) / cells_y;"),
    ("transposed_cells", "cells concatenated column-major",
     "hb[((int64_t)cy * cells_x + cx) * bins + b]", "hb[((int64_t)cx * cells_y + cy) * bins + b]"),
    ("overflow_off_by_one", "overflow only above 65536 px",
     "if (maxw * maxh > 65535) status = ORC_E_OVERFLOW;",
     "if (maxw * maxh > 65536) status = ORC_E_OVERFLOW;"),
    ("bin_shift", "uniform bin of the next code",
     "int32_t bin = (bins == 256) ? code : U[code];",
     "int32_t bin = (bins == 256) ? code : U[(code + 1) & 255];"),
    ("svm_fp32_accumulate", "SVM sum accumulated in fp32",
     "            double acc = (double)bias[c];\n            for (int32_t d = 0; d < dim; ++d) acc += (double)w[d] * (double)h[d];",
     "            float acc = bias[c];\n            for (int32_t d = 0; d < dim; ++d) acc += (double)w[d] * (double)h[d];"),
    ("svm_ties_high", "ties go to the highest class",
     "            if (c == 0 || s > best) {", "            if (c == 0 || s >= best) {"),
    ("svm_reject_le", "rejected when top <= threshold (instead of <)",
     "        if (labels) labels[i] = (best < reject_threshold) ? -1 : best_c;\n    }\n    return ORC_OK;\n}\n\n/* ----",
     "        if (labels) labels[i] = (best <= reject_threshold) ? -1 : best_c;\n    }\n    return ORC_OK;\n}\n\n/* ----"),
    ("svm_bias_dropped", "bias not added",
     "            double acc = (double)bias[c];\n            for (int32_t d = 0; d < dim; ++d) acc += (double)w[d] * (double)h[d];",
     "            double acc = 0.0;\n            for (int32_t d = 0; d < dim; ++d) acc += (double)w[d] * (double)h[d];"),
]


def run_pins(tree, tests):
    env = dict(os.environ, PYTHONDONTWRITEBYTECODE="1")
    p = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-p", "no:cacheprovider",
                        "-m", "not gpu", *tests], cwd=tree, env=env, capture_output=True,
                       text=True, timeout=1800)
    last = [ln for ln in p.stdout.splitlines() if ln.strip()][-1:] or [""]
    failed = [ln for ln in p.stdout.splitlines() if ln.startswith("FAILED") or "Error" in ln]
    return p.returncode, last[0], failed[:3]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02", "oracle_mutants.json"))
    args = ap.parse_args()
    tests = sorted(f"tests/{f}" for f in os.listdir(os.path.join(ROOT, "tests"))
                   if f.startswith("test_oracle") and f.endswith(".py"))
    src0 = open(os.path.join(ROOT, SRC)).read()
    results = []
    for name, what, old, new in [("unmodified", "control: must pass", None, None)] + MUTANTS:
        if name == "unmodified":
            src = src0
        else:
            if src0.count(old) != 1:
                results.append({"mutant": name, "error": f"pattern occurs {src0.count(old)} times"})
                continue
            src = src0.replace(old, new)
        tree = tempfile.mkdtemp(prefix="mut_")
        try:
            for d in ("oracle", "tests", "synthgen"):
                shutil.copytree(os.path.join(ROOT, d), os.path.join(tree, d),
                                ignore=shutil.ignore_patterns("*.so", "__pycache__"))
            for f in ("pytest.ini",):
                if os.path.exists(os.path.join(ROOT, f)):
                    shutil.copy(os.path.join(ROOT, f), tree)
            # the test conftest puts the tree root on sys.path; the product package is not needed
            # by the oracle pins but conftest may import it lazily: link it read-only
            os.symlink(os.path.join(ROOT, "paper_1504_01883_b200"),
                       os.path.join(tree, "paper_1504_01883_b200"))
            open(os.path.join(tree, SRC), "w").write(src)
            t0 = time.time()
            rc, last, failed = run_pins(tree, tests)
            killed = rc != 0
            results.append({"mutant": name, "bug": what, "pins_rc": rc,
                            "killed": killed if name != "unmodified" else None,
                            "pins_pass": rc == 0 if name == "unmodified" else None,
                            "first_failures": failed, "summary": last,
                            "seconds": round(time.time() - t0, 1)})
            print(f"{name:22s} rc={rc} {'KILLED' if killed else 'survived'}  {last}", flush=True)
        finally:
            shutil.rmtree(tree, ignore_errors=True)
    ctrl = results[0]
    mutants = [r for r in results[1:] if "killed" in r]
    summary = {"control_passes": ctrl.get("pins_rc") == 0,
               "mutants": len(mutants), "killed": sum(1 for r in mutants if r["killed"]),
               "pins": tests, "results": results}
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    json.dump(summary, open(args.out, "w"), indent=1)
    print(json.dumps({k: summary[k] for k in ("control_passes", "mutants", "killed")}))
    return 0 if summary["control_passes"] and summary["killed"] == summary["mutants"] else 1


if __name__ == "__main__":
    sys.exit(main())
