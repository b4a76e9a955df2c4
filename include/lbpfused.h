/*
 * lbpfused.h -- C ABI of the B200-native fused-depth LBP descriptor + linear
 * SVM hot path of arXiv 1504.01883 (Naik & Rathna, "Robust real time face
 * recognition and tracking on GPU using fusion of RGB and depth image").
 *
 * Citations: P:L = line L of the paper text, S:L = line L of the
 * SPEC.md CPU-toolkit spec (interfaces / error conventions only), SURVEY §8x =
 * /root/repo/SURVEY.md section 8(x) (the build contract), DESIGN.md §n.
 *
 * Conventions (all entry points):
 *  - Every data pointer is a DEVICE pointer unless the name ends in _h.
 *    The caller owns every buffer; the library never allocates, frees or
 *    synchronises.  All work is enqueued on `stream` (a cudaStream_t passed as
 *    void*; NULL = the legacy default stream) and returns immediately.
 *    Stream order is kept: kernels launched as programmatic dependents (the
 *    TMA extraction kernels, the tensor-core scorers) may start their setup
 *    while the previous kernel on the stream runs, but touch no buffer before
 *    it has completed ("Kernel boundaries of a step").
 *  - Calls are reentrant and thread-safe; the library keeps no mutable global
 *    state (its lookup tables are compile-time constants).
 *  - Host-detectable argument errors return a negative status and enqueue
 *    nothing.  n_rois == 0 / n == 0 is a no-op returning LBP_OK.
 *  - A failed launch returns LBP_E_CUDA (LBP_E_UNSUPPORTED if the device is not
 *    sm_100); asynchronous faults surface on the caller's next sync.
 */
#ifndef LBPFUSED_H
#define LBPFUSED_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef void* lbp_stream_t; /* cudaStream_t */

enum {
    LBP_OK = 0,
    LBP_E_ARG = -1,         /* null pointer, bins not 59/256, cells < 1, dmin > dmax, bad geometry */
    LBP_E_ROI = -2,         /* per ROI: clamped ROI empty, narrower/shorter than 3 px, bad image */
    LBP_E_GRID = -3,        /* per ROI: cells_x > W-2 or cells_y > H-2 */
    LBP_E_OVERFLOW = -4,    /* per ROI: largest cell has more than 65535 px (u16 counts) */
    LBP_E_UNSUPPORTED = -5, /* valid but unimplemented, or device is not sm_100 */
    LBP_E_CUDA = -6         /* CUDA launch / copy error */
};

/* Label written by the scorers for every row when `prepared` does not belong to the call's
 * model (its header -- layout and a fingerprint of W -- was written by svm_prepare() for
 * another W or shape); top_score and scores are NaN then.  -1 stays "rejected". */
#define LBP_LABEL_BAD_MODEL (-2)

/* An ROI ("Rect r = boundingRect(...)") inside image `img` of the stack:
 * top-left (x, y), width w, height h, in pixels.  Clamped to the image. */
typedef struct {
    int32_t img, x, y, w, h;
} lbp_roi_t;

/* Geometry of an image stack: n_images images of height x width pixels.
 * Pitches and strides are in ELEMENTS (u8 for grey, u16 for depth):
 * pixel (img, y, x) of grey is grey[img*grey_img_stride + y*grey_pitch + x].
 * Requires pitch >= width and img_stride >= pitch*(height-1) + width. */
typedef struct {
    int32_t n_images, height, width, reserved; /* reserved: must be 0 */
    int64_t grey_pitch, depth_pitch;
    int64_t grey_img_stride, depth_img_stride;
} lbp_images_t;

/* Descriptor length: cells_x * cells_y * bins (Eq. 3: K = cells_x*cells_y
 * sub-histograms of `bins` bins, concatenated row-major).  Negative status if
 * the arguments are invalid. */
int32_t lbp_descriptor_dim(int32_t cells_x, int32_t cells_y, int32_t bins);

/*
 * lbp_fused_extract -- SURVEY §8a steps a1-a6 for every ROI n:
 *   clamp ROI; for each interior pixel of the ROI (the 1-px ROI border is
 *   halo only): valid iff depth == NULL or d(centre) != 0 and
 *   dmin <= d <= dmax (P:49-63 depth mask); code = Eq. 2 with the
 *   Fig. 7 weights, S(x) = [x >= 0]; bin = code (bins = 256, "0 to
 *   255") or the uniform-pattern bin (bins = 59: the 58 codes with <= 2
 *   circular transitions in ascending order -> 0..57, others -> 58); cell
 *   (cx, cy) from the floor partition [floor(b*W'/K), floor((b+1)*W'/K)) of
 *   the interior; desc[n][(cy*cells_x + cx)*bins + bin] += 1 (Eq. 3).
 *
 *   grey       u8 image stack, layout per `geom` (required)
 *   depth      u16 depth stack in mm, same geometry (0 = no reading); NULL = no mask
 *   rois       [n_rois] lbp_roi_t (device)
 *   dmin,dmax  inclusive depth window in mm (dmin <= dmax)
 *   desc       out: u16 [n_rois][lbp_descriptor_dim()] row-major, fully written
 *   roi_status out, nullable: int32 [n_rois], LBP_OK or the per-ROI error; a failed
 *              ROI's descriptor row is all zeros.
 * Returns LBP_OK or a host-detectable error (nothing is enqueued then).
 */
int32_t lbp_fused_extract(const uint8_t* grey, const uint16_t* depth, lbp_images_t geom,
                          const lbp_roi_t* rois, int32_t n_rois, uint16_t dmin, uint16_t dmax,
                          int32_t cells_x, int32_t cells_y, int32_t bins, uint16_t* desc,
                          int32_t* roi_status, lbp_stream_t stream);

/* Source plane of the LBP codes. */
enum {
    LBP_SRC_GREY = 0,  /* codes on the grey image (lbp_fused_extract; the headline) */
    LBP_SRC_DEPTH = 1, /* codes on the u16 depth image itself (Table 1 "Depth Image") */
    LBP_SRC_FUSED = 2  /* grey descriptor then depth descriptor, 2*dim per ROI (P:17 fusion) */
};

/*
 * lbp_extract_source -- lbp_fused_extract with a selectable code source (SURVEY §8f-1,
 * DESIGN.md reading R17): every step is as documented for lbp_fused_extract (clamp, border,
 * depth-window mask on the CENTRE pixel from `depth`, floor cells, bins, statuses) except
 * step 5, where Eq. 2 reads the 3x3 neighbourhood of the source plane:
 *   LBP_SRC_GREY   grey (u8); depth optional (NULL = no mask); identical to lbp_fused_extract
 *   LBP_SRC_DEPTH  depth (u16, required; grey may be NULL): S(d_p - d_c) = [d_p >= d_c] on
 *                  the raw millimetre values, holes (0) included as neighbours
 *   LBP_SRC_FUSED  grey and depth required; desc row n = [grey block (dim) | depth block
 *                  (dim)], i.e. u16 [n_rois][2*dim]
 * Returns LBP_OK or a host-detectable error (LBP_E_ARG for a bad source or a missing plane).
 */
int32_t lbp_extract_source(const uint8_t* grey, const uint16_t* depth, lbp_images_t geom,
                           const lbp_roi_t* rois, int32_t n_rois, uint16_t dmin, uint16_t dmax,
                           int32_t cells_x, int32_t cells_y, int32_t bins, int32_t source,
                           uint16_t* desc, int32_t* roi_status, lbp_stream_t stream);

/*
 * lbp_extract_resized -- descriptors of ROIs resized to size x size (P:154
 * "The detected face ... is resized to 200x200 pixels"; R19):
 *   crop = clamp(roi, image) (empty / bad image -> LBP_E_ROI and a zero row), then
 *   grey: bilinear with half-pixel centres, rounded half up (exact integer arithmetic);
 *   depth: nearest neighbour with half-pixel centres, ties toward the smaller index (holes
 *   are never blended); then every step of lbp_extract_source on the size x size image
 *   with a full ROI (border, mask, codes of `source`, floor cells, bins, statuses).  The
 *   resized crops live only in shared memory (the resize is fused into the staging).
 *   size       output side, 3..1024 (LBP_E_ARG otherwise)
 *   desc       out: u16 [n_rois][dim] (or [n_rois][2*dim] for LBP_SRC_FUSED)
 * Image width and height must be <= 2^20 (LBP_E_UNSUPPORTED otherwise).
 */
int32_t lbp_extract_resized(const uint8_t* grey, const uint16_t* depth, lbp_images_t geom,
                            const lbp_roi_t* rois, int32_t n_rois, int32_t size, uint16_t dmin,
                            uint16_t dmax, int32_t cells_x, int32_t cells_y, int32_t bins,
                            int32_t source, uint16_t* desc, int32_t* roi_status,
                            lbp_stream_t stream);

/*
 * svm_score -- SURVEY §8a step a7: linear one-vs-rest SVM decision ("a classifier
 * defined by a hyperplane"; A-vs-B training per identity):
 *   s[n][c] = fp32( b[c] + sum_d W[c][d] * desc[n][d] ), accumulated EXACTLY (each
 *   product of a u16 count and an fp32 weight is exact in fp64 / in the integer
 *   digit-plane tensor-core path) and rounded once to fp32;
 *   labels[n] = argmax_c s[n][c] over the fp32 scores, ties -> lowest c;
 *   labels[n] = -1 iff top_score[n] < reject_threshold (-INFINITY = closed set).
 *
 *   desc      u16 [n][dim]        W  fp32 [n_classes][dim] row-major   bias fp32 [n_classes]
 *   prepared  nullable: workspace filled by svm_prepare() for this W (enables the
 *             tensor-core path for n >= 128); NULL = CUDA-core path
 *   prepared_bytes  size of the `prepared` allocation; < svm_workspace_bytes(n_classes, dim)
 *             -> LBP_E_ARG (nothing enqueued).  The tensor-core kernels also check the
 *             workspace header on the device before reading past it: a workspace prepared
 *             for another shape or another W (8 sampled weights differ) is not used and every
 *             row gets labels = LBP_LABEL_BAD_MODEL, NaN top score and scores.
 *   scores    out, nullable fp32 [n][n_classes]
 *   labels    out, nullable int32 [n];  top_score out, nullable fp32 [n]
 */
int32_t svm_score(const uint16_t* desc, int32_t n, int32_t dim, const float* W,
                  const float* bias, int32_t n_classes, const void* prepared,
                  size_t prepared_bytes, float* scores, int32_t* labels, float* top_score,
                  float reject_threshold, lbp_stream_t stream);

/*
 * lbp_recognize -- the whole device path in one call (lbp_fused_extract + svm_score, grey
 * source): descriptors, statuses, scores, labels and top scores exactly as the two calls
 * would produce them (same oracle definitions).  For batches smaller than the SM count with
 * cells_y <= 8 and n_classes <= 2048 it is ONE launch: a thread-block cluster of cells_y CTAs
 * per ROI computes one cell row each, scores its descriptor segment, and rank 0 combines the
 * per-class partials over distributed shared memory; otherwise
 * it runs the two kernels of lbp_fused_extract and svm_score.
 *   desc       out, REQUIRED: u16 [n_rois][dim] (also the scorer's input)
 *   prepared   nullable svm_prepare() workspace (tensor-core scorer for large batches);
 *              prepared_bytes and the device-side header check as in svm_score
 *   scores / roi_status / labels / top_score  nullable outputs as in svm_score / extract
 */
int32_t lbp_recognize(const uint8_t* grey, const uint16_t* depth, lbp_images_t geom,
                      const lbp_roi_t* rois, int32_t n_rois, uint16_t dmin, uint16_t dmax,
                      int32_t cells_x, int32_t cells_y, int32_t bins, const float* W,
                      const float* bias, int32_t n_classes, const void* prepared,
                      size_t prepared_bytes, float reject_threshold, uint16_t* desc,
                      int32_t* roi_status, float* scores, int32_t* labels, float* top_score,
                      lbp_stream_t stream);

/*
 * svm_score_l1 -- the linear OvR SVM on per-block L1-normalised descriptors (SURVEY §8f-3
 * variant; S:379-387 normalize: each block divided by its own count sum, an empty block maps
 * to zeros): s[n][c] = fp32(b[c] + sum_k (sum_{d in block k} W[c][d] h[n][d]) / N_k), blocks
 * of `block` consecutive entries (one cell: block = bins); labels / top / reject as
 * svm_score.  CUDA cores, fp64 accumulation of exact products.  dim % block != 0 -> LBP_E_ARG;
 * LBP_E_UNSUPPORTED if one staged descriptor row (4 B per entry) exceeds 200 KB.
 */
int32_t svm_score_l1(const uint16_t* desc, int32_t n, int32_t dim, int32_t block, const float* W,
                     const float* bias, int32_t n_classes, float* scores, int32_t* labels,
                     float* top_score, float reject_threshold, lbp_stream_t stream);

/*
 * svm_train_ovr -- one-vs-rest linear SVM training on the descriptors (P:140-144
 * "finding a hyperplane"; P:144 one identity against the others; R20):
 * for every class c, Pegasos steps over the visit order with lambda = 1 / inv_lambda and the
 * bias folded in as a constant feature 1 (regularised with w):
 *   t = 1..T, i = order[t-1], y = +1 if labels[i] == c else -1 (labels outside [0, C) are
 *   negatives for every class), x~ = (desc[i], 1);
 *   violated iff t == 1 or y (w_{t-1} . x~) < 1;  w_t = (1 - 1/t) w_{t-1} + [violated] y x~/(lambda t)
 * computed EXACTLY in integers (z_t = lambda t w_t), so the result is bit-reproducible and
 * identical to the oracle's; the model is the last iterate, W[c][d] = fp32(fp64(inv_lambda
 * z_T[d]) / T), bias[c] likewise from the constant feature.
 *   desc     u16 [n][dim] (device), dim <= 16,384 (LBP_E_UNSUPPORTED above)
 *   labels   int32 [n];  order int32 [T], every entry in [0, n) (NOT checked: an index out of
 *            range is undefined behaviour); e.g. one seeded permutation of 0..n-1 per epoch
 *   W, bias  out fp32 [n_classes][dim], [n_classes];  z_out  nullable int64 [n_classes][dim+1]
 * Preconditions for exact int64 arithmetic: T <= 2^31 and |z . x~| < 2^63 (e.g. T <= 2^24 with
 * sum_d desc[i][d] <= 2^16).  One CTA per class; the T steps of a class are sequential.
 */
int32_t svm_train_ovr(const uint16_t* desc, int32_t n, int32_t dim, const int32_t* labels,
                      int32_t n_classes, const int32_t* order, int64_t T, int32_t inv_lambda,
                      float* W, float* bias, int64_t* z_out, lbp_stream_t stream);

/*
 * Descriptor compaction for the database all-gather ("pack counts (u8 +
 * overflow flag) to halve all-gather bytes"; R21).  Cell counts of 128x128 crops
 * are <= 256 and almost always <= 255, so a descriptor travels as one byte per entry plus a
 * short list of the entries that do not fit:
 *   packed[i][d] = min(desc[i][d], 255)
 *   exceptions   = { (row_base + i, d, desc[i][d]) : desc[i][d] > 255 }
 * The list order is unspecified (entries are unique, so decoding does not depend on it).
 */
typedef struct {
    int64_t row;    /* global descriptor row */
    int32_t index;  /* entry within the row, [0, dim) */
    int32_t value;  /* the u16 count, > 255 */
} lbp_desc_exc_t;

/*
 * lbp_desc_pack_u8 -- desc u16 [n][dim] (device, contiguous rows) -> packed u8 [n][dim] and
 * exceptions (device arrays, caller-owned).  *exc_count (device int32) is set to the number
 * of exceptions found -- entries past exc_cap are counted but not stored, so a count >
 * exc_cap after the stream synchronises means "re-run with a larger cap".  Two launches (a
 * memset of the count and one streaming kernel: 2 B read + 1 B written per entry).
 * n == 0 -> LBP_OK (only the count is zeroed); null pointers, n < 0, dim < 1, exc_cap < 0
 * -> LBP_E_ARG before anything is enqueued.
 */
int32_t lbp_desc_pack_u8(const uint16_t* desc, int64_t n, int32_t dim, int64_t row_base,
                         uint8_t* packed, lbp_desc_exc_t* exc, int32_t exc_cap,
                         int32_t* exc_count, lbp_stream_t stream);

/*
 * lbp_desc_unpack_u8 -- the inverse, for rows [row_base, row_base + n): desc[i][d] =
 * packed[i][d], then every listed exception whose row falls in the range overwrites its
 * entry (others are ignored).  The exceptions come as n_lists lists of exc_cap records each
 * (list l at exc + l * exc_cap, e.g. one per rank after an all-gather) with counts
 * exc_counts[l] (device int32; min(count, exc_cap) records of a list are read).  Two
 * launches (widen: 1 B read + 2 B written per entry; scatter of the exceptions).
 */
int32_t lbp_desc_unpack_u8(const uint8_t* packed, int64_t n, int32_t dim, int64_t row_base,
                           const lbp_desc_exc_t* exc, const int32_t* exc_counts, int32_t n_lists,
                           int32_t exc_cap, uint16_t* desc, lbp_stream_t stream);

/*
 * The fused database build (SURVEY §8e way 2; "online database generation"):
 * lbp_extract_gather computes the descriptors of this rank's ROIs and writes every row ONCE,
 * from the extraction epilogue, into the gathered training matrix of EVERY rank -- no local
 * descriptor write followed by an all-gather collective.
 *   LBP_GATHER_MULTIMEM  base[0] is an NVLS multicast address of the ranks' buffers
 *                        (multimem.st: the NVSwitch replicates each 16-B store); n_dst = 1
 *   LBP_GATHER_PEERS     base[0..n_dst-1] are the ranks' buffers as mapped on this device
 *                        (NVLink P2P): each 16-B chunk is stored to every one of them
 * In every destination: rows of desc_pitch u16 at byte desc_offset (row = row_base + n for
 * this call's ROI n; entries dim..desc_pitch-1 are zero), int32 labels at labels_offset
 * (labels[n] copied to entry row_base + n; labels_offset < 0 or labels == NULL: none).
 * The call ends with a system-scope fence; the caller runs a cross-rank barrier (e.g. the
 * symmetric-memory barrier) before any rank reads another rank's rows.  Host-detectable
 * errors (LBP_E_ARG): bad mode or n_dst (MULTIMEM: 1, PEERS: 1..8), a null base, desc_offset
 * or a base not 16-B aligned, desc_pitch < dim or not a multiple of 8, labels_offset not a
 * multiple of 4, scratch NULL.
 *   scratch   device u16 [n_rois][dim]: rows of ROIs off the TMA fast path are extracted here
 *             first (and the whole batch when the fast kernel does not apply: small batches,
 *             other grids / bins / geometries -- then a forwarding kernel does the stores)
 */
enum { LBP_GATHER_MULTIMEM = 1, LBP_GATHER_PEERS = 2 };
#define LBP_GATHER_MAX_DST 8
typedef struct {
    int32_t mode, n_dst;
    uint64_t base[LBP_GATHER_MAX_DST];
    int64_t desc_offset;   /* bytes */
    int64_t desc_pitch;    /* u16 elements per gathered row */
    int64_t labels_offset; /* bytes; < 0 = no labels */
    int64_t row_base;      /* gathered row of this call's ROI 0 */
} lbp_gather_dst_t;

int32_t lbp_extract_gather(const uint8_t* grey, const uint16_t* depth, lbp_images_t geom,
                           const lbp_roi_t* rois, int32_t n_rois, uint16_t dmin, uint16_t dmax,
                           int32_t cells_x, int32_t cells_y, int32_t bins,
                           const int32_t* labels, lbp_gather_dst_t dst, uint16_t* scratch,
                           int32_t* roi_status, lbp_stream_t stream);

/* Bytes of device workspace svm_prepare() needs for a [n_classes][dim] model
 * (0 if the tensor-core path does not apply to this shape). */
size_t svm_workspace_bytes(int32_t n_classes, int32_t dim);

/* Splits W into fixed-point digit planes for the exact tensor-core scorer (DESIGN.md
 * §5) into `workspace` (device, >= svm_workspace_bytes()).  Enqueued on stream. */
int32_t svm_prepare(const float* W, int32_t n_classes, int32_t dim, void* workspace,
                    size_t workspace_bytes, lbp_stream_t stream);

/*
 * The compact recognition path (SURVEY §8f-3 "pack counts (u8 + overflow flag)"; DESIGN.md
 * R21, R22): the extraction epilogue writes each descriptor row as one byte per entry plus a
 * per-row list of the entries that do not fit, and the INT8 tensor-core scorer reads those
 * bytes as its A operand directly -- half the descriptor bytes written and read, no separate
 * pack pass.  The descriptor it encodes is exactly lbp_fused_extract's (grey source):
 *   packed[n][d]  = desc[n][d] & 255 (the low byte)         u8, rows of `pitch` bytes
 *   exc_n[n]      = #{ d : desc[n][d] > 255 }                int32
 *   exc[n][k]     = (d << 16) | desc[n][d] for those d,      uint32 [n][exc_cap], k < exc_n[n]
 *                   in unspecified order
 * A row cannot hold more than floor((width - 2) (height - 2) / 256) such entries (each needs
 * 256 interior pixels of its ROI); lbp_u8_exc_cap_min(geom, dim) returns that bound (capped at
 * dim) and exc_cap must be at least it, so the lists never overflow (LBP_E_ARG otherwise).
 * Requires dim <= 65535.
 */
int32_t lbp_u8_exc_cap_min(lbp_images_t geom, int32_t dim);

/*
 * lbp_extract_u8 -- lbp_fused_extract (every step and status as documented there) with the
 * compact output above.  Crop stacks of 128x128 ROIs with 8x8 cells and 59 bins, batches of
 * at least one ROI per SM and pitch % 16 == 0 take the TMA kernel whose epilogue stages the
 * u8 row and bulk-stores it; every other case extracts into `scratch` (device u16
 * [n_rois][dim], may be NULL when the TMA kernel applies -- LBP_E_ARG if it is needed and
 * NULL) and packs it.  pitch >= dim.
 */
int32_t lbp_extract_u8(const uint8_t* grey, const uint16_t* depth, lbp_images_t geom,
                       const lbp_roi_t* rois, int32_t n_rois, uint16_t dmin, uint16_t dmax,
                       int32_t cells_x, int32_t cells_y, int32_t bins, uint8_t* packed,
                       int64_t pitch, int32_t* exc_n, uint32_t* exc, int32_t exc_cap,
                       uint16_t* scratch, int32_t* roi_status, lbp_stream_t stream);

/* Bytes of device workspace svm_prepare_u8() needs for a [n_classes][dim] model (0 if the
 * compact tensor-core scorer does not take this shape: dim > 32,768). */
size_t svm_workspace_u8_bytes(int32_t n_classes, int32_t dim);

/* W as five unsigned base-256 digit planes of an offset fraction ("compact
 * descriptors") for svm_score_u8's tensor-core path.  Enqueued on stream. */
int32_t svm_prepare_u8(const float* W, int32_t n_classes, int32_t dim, void* workspace,
                       size_t workspace_bytes, lbp_stream_t stream);

/*
 * svm_score_u8 -- svm_score (same definitions of scores, labels, ties, reject threshold and
 * the prepared-workspace checks) on the compact descriptor (packed, pitch, exc_n, exc,
 * exc_cap) of lbp_extract_u8.  prepared = svm_prepare_u8()'s workspace (NULL: CUDA-core
 * fp64 path); the tensor-core path needs n >= 128, pitch % 16 == 0 and a 16-B aligned packed.
 */
int32_t svm_score_u8(const uint8_t* packed, int64_t pitch, const int32_t* exc_n,
                     const uint32_t* exc, int32_t exc_cap, int32_t n, int32_t dim,
                     const float* W, const float* bias, int32_t n_classes, const void* prepared,
                     size_t prepared_bytes, float* scores, int32_t* labels, float* top_score,
                     float reject_threshold, lbp_stream_t stream);

/*
 * lbp_recognize_host -- the whole path from HOST buffers (end-to-end entry point):
 * cudaMemcpyAsync of grey/depth/rois host->device into `workspace`, then
 * lbp_fused_extract + svm_score, then device->host of labels and top scores.
 * Host buffers should be pinned for the copies to be asynchronous; the caller
 * synchronises `stream` before reading labels_h / top_h.
 *   workspace  device scratch of >= lbp_recognize_workspace_bytes() bytes
 *   W, bias, prepared, prepared_bytes  device model as for svm_score
 */
size_t lbp_recognize_workspace_bytes(lbp_images_t geom, int32_t has_depth, int32_t n_rois,
                                     int32_t cells_x, int32_t cells_y, int32_t bins);
int32_t lbp_recognize_host(const uint8_t* grey_h, const uint16_t* depth_h, lbp_images_t geom,
                           const lbp_roi_t* rois_h, int32_t n_rois, uint16_t dmin,
                           uint16_t dmax, int32_t cells_x, int32_t cells_y, int32_t bins,
                           const float* W, const float* bias, int32_t n_classes,
                           const void* prepared, size_t prepared_bytes, float reject_threshold,
                           void* workspace, size_t workspace_bytes, int32_t* labels_h,
                           float* top_h, lbp_stream_t stream);

/* Human-readable name of a status code (static string). */
const char* lbp_status_string(int32_t status);

#ifdef __cplusplus
}
#endif
#endif /* LBPFUSED_H */
