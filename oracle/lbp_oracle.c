/*
 * lbp_oracle.c -- CPU ORACLE for the fused-depth LBP descriptor + linear SVM
 * hot path of arXiv 1504.01883 (Naik & Rathna).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py (cpu_baseline leg and --impl reference) may load this library.
 * The product path (paper_1504_01883_b200/) never links, imports or calls it,
 * and this file shares no code, header, table or constant generator with it.
 *
 * Plain, slow, obviously-correct, single-threaded C99.  No SIMD intrinsics,
 * no blocking, no reordering beyond what the definitions below state.
 * Citations: "P:L" = line L of PAPER.md (the paper text), "S:L" = line L of
 * SPEC.md, "§8c" = SURVEY.md section 8(c) (the readings of the paper that this
 * build takes; each reading is also listed in DESIGN.md §3).
 *
 * Every function here is pinned by tests/test_oracle.py against values the
 * paper prints (Fig. 7), closed forms, invariants and brute force; see the
 * header comment of each function for the pins that cover it.
 */
#include <stdint.h>
#include <stdlib.h>
#include <stddef.h>
#include <string.h>
#include <math.h>

/* Status codes: the contract of SURVEY §8(b), restated (not shared) here. */
#define ORC_OK 0
#define ORC_E_ARG (-1)
#define ORC_E_ROI (-2)
#define ORC_E_GRID (-3)
#define ORC_E_OVERFLOW (-4)

/* ------------------------------------------------------------------------ */
/* Eq. 2 with the Fig. 7 weights.                   */
/*                                                                          */
/*   LBP(x_c, y_c) = sum_{p=0}^{7} S(g_p - g_c) * 2^p                       */
/*                                                                          */
/* S(x) = 1 iff x >= 0 (Fig. 7: neighbour 6 vs centre 6 thresholds to 1).   */
/* The sampling points p = 0..7 carry the Fig. 7 weights matrix             */
/*       [[  1,  2,  4],                                                    */
/*        [128,  .,  8],                                                    */
/*        [ 64, 32, 16]]                                                    */
/* i.e. p=0 top-left, 1 top, 2 top-right, 3 right, 4 bottom-right,          */
/* 5 bottom, 6 bottom-left, 7 left.                                         */
/* ------------------------------------------------------------------------ */

/* (row offset, column offset) of sampling point p, read off Fig. 7. */
static const int ORC_DY[8] = {-1, -1, -1, 0, 1, 1, 1, 0};
static const int ORC_DX[8] = {-1, 0, 1, 1, 1, 0, -1, -1};

static int orc_S(int64_t x) { return x >= 0 ? 1 : 0; }

/* window: 3x3 samples, row-major (window[r*3+c]); any unsigned width. */
int32_t oracle_lbp_code_window(const uint32_t window[9])
{
    int64_t gc = window[4];
    int32_t code = 0;
    for (int p = 0; p < 8; ++p) {
        int64_t gp = window[(1 + ORC_DY[p]) * 3 + (1 + ORC_DX[p])];
        code += orc_S(gp - gc) * (1 << p);
    }
    return code;
}

/* ------------------------------------------------------------------------ */
/* Uniform-pattern bin map (J.north_star "uniform-pattern histograms",      */
/* SURVEY §8c step 6).  A code is uniform iff its circular bit string       */
/* (p = 0..7, p=7 adjacent to p=0 -- the Fig. 7 positions go round the      */
/* centre) has at most 2 transitions 0<->1.  Uniform codes, in ascending    */
/* code order, get bins 0..57; every other code gets bin 58.                */
/* Returns the number of uniform codes (58).                                */
/* ------------------------------------------------------------------------ */
int32_t oracle_uniform_table(uint8_t table[256])
{
    int next = 0;
    for (int code = 0; code < 256; ++code) {
        int transitions = 0;
        for (int p = 0; p < 8; ++p) {
            int bit_p = (code >> p) & 1;
            int bit_next = (code >> ((p + 1) % 8)) & 1;
            if (bit_p != bit_next) transitions += 1;
        }
        table[code] = (transitions <= 2) ? (uint8_t)next++ : 0xFF;
    }
    for (int code = 0; code < 256; ++code)
        if (table[code] == 0xFF) table[code] = (uint8_t)next;
    return next; /* = number of uniform codes; bins = next + 1 */
}

/* Code map of an 8-bit image: out[i*(w-2)+j] = LBP at image pixel (i+1,j+1).
 * The 1-px border has no code.  Returns ORC_E_ROI if w<3 or h<3. */
int32_t oracle_lbp_map_u8(const uint8_t* img, int32_t h, int32_t w, int64_t pitch, uint8_t* out)
{
    if (!img || !out) return ORC_E_ARG;
    if (w < 3 || h < 3) return ORC_E_ROI;
    for (int32_t i = 0; i < h - 2; ++i)
        for (int32_t j = 0; j < w - 2; ++j) {
            uint32_t win[9];
            for (int r = 0; r < 3; ++r)
                for (int c = 0; c < 3; ++c)
                    win[r * 3 + c] = img[(int64_t)(i + r) * pitch + (j + c)];
            out[(int64_t)i * (w - 2) + j] = (uint8_t)oracle_lbp_code_window(win);
        }
    return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* Fused-depth descriptor, per ROI n:                 */
/*  1. r = clamp(roi, image); empty / r.w<3 / r.h<3 -> ORC_E_ROI     */
/*     (S:86), zero row.                                             */
/*  2. interior W' = r.w-2, H' = r.h-2; code-map pixel (i,j) is image pixel */
/*     (r.y+1+i, r.x+1+j).  cells_x > W' or cells_y > H' ->         */
/*     ORC_E_GRID.  Largest cell area > 65535 -> ORC_E_OVERFLOW.    */
/*  3. cell b spans [floor(b*W'/K), floor((b+1)*W'/K)), row-major   */
/*     concatenation of the cells (Eq. 3: K sub-histograms).     */
/*  4. valid = (depth == NULL) or (d != 0 and dmin <= d <= dmax), d = depth */
/*     at the CENTRE pixel (P:49-63 mask; S:37 0 = no reading).             */
/*  5. code = Eq. 2 above on the 3x3 neighbourhood of the SOURCE plane      */
/*     (P:115): the grey image, or -- SURVEY §8f-1, Table 1's "Depth Image" */
/*     row -- the u16 depth image itself (S:559 source: depth). */
/*  6. bin = code (bins = 256, "ranging from 0 to 255") or           */
/*     U[code] (bins = 59, uniform patterns, J.north_star).                 */
/*  7. hist[(cy*Kx+cx)*bins + bin] += 1 (Eq. 3, f = indicator).             */
/* source = ORC_SRC_FUSED writes the grey descriptor then the depth one     */
/* (the "fusion of RGB and depth" of the title): row length 2*dim.    */
/* ------------------------------------------------------------------------ */
enum { ORC_SRC_GREY = 0, ORC_SRC_DEPTH = 1, ORC_SRC_FUSED = 2 };

int32_t oracle_lbp_extract_src(const uint8_t* grey, const uint16_t* depth,
                               int32_t n_images, int32_t height, int32_t width,
                               int64_t grey_pitch, int64_t depth_pitch,
                               int64_t grey_img_stride, int64_t depth_img_stride,
                               const int32_t* rois /* [n_rois][5] = img,x,y,w,h */,
                               int32_t n_rois, uint16_t dmin, uint16_t dmax,
                               int32_t cells_x, int32_t cells_y, int32_t bins, int32_t source,
                               uint16_t* desc /* [n_rois][(1 or 2)*cells_y*cells_x*bins] */,
                               int32_t* roi_status /* nullable [n_rois] */)
{
    if (n_rois < 0) return ORC_E_ARG;
    if (source != ORC_SRC_GREY && source != ORC_SRC_DEPTH && source != ORC_SRC_FUSED)
        return ORC_E_ARG;
    if (n_rois == 0) return ORC_OK;
    if (!rois || !desc) return ORC_E_ARG;
    if (source != ORC_SRC_DEPTH && !grey) return ORC_E_ARG;
    if (source != ORC_SRC_GREY && !depth) return ORC_E_ARG;
    if (bins != 59 && bins != 256) return ORC_E_ARG;
    if (cells_x < 1 || cells_y < 1) return ORC_E_ARG;
    if (dmin > dmax) return ORC_E_ARG;
    if (n_images < 1 || height < 1 || width < 1) return ORC_E_ARG;
    if (grey && (grey_pitch < width || grey_img_stride < grey_pitch * (height - 1) + width))
        return ORC_E_ARG;
    if (depth && (depth_pitch < width || depth_img_stride < depth_pitch * (height - 1) + width))
        return ORC_E_ARG;
    int64_t dim = (int64_t)cells_x * cells_y * bins;
    int64_t row = (source == ORC_SRC_FUSED) ? 2 * dim : dim;
    if (row > 0x7FFFFFFF) return ORC_E_ARG;

    uint8_t U[256];
    oracle_uniform_table(U);

    for (int32_t n = 0; n < n_rois; ++n) {
        uint16_t* h = desc + (int64_t)n * row;
        for (int64_t d = 0; d < row; ++d) h[d] = 0;
        int32_t status = ORC_OK;

        const int32_t* roi = rois + (int64_t)n * 5;
        int64_t img = roi[0];
        /* step 1: clamp to [0,W) x [0,H) */
        int64_t x0 = roi[1], y0 = roi[2];
        int64_t x1 = x0 + roi[3], y1 = y0 + roi[4];
        if (x0 < 0) x0 = 0;
        if (y0 < 0) y0 = 0;
        if (x1 > width) x1 = width;
        if (y1 > height) y1 = height;
        int64_t rw = x1 - x0, rh = y1 - y0;
        if (img < 0 || img >= n_images || rw < 3 || rh < 3) status = ORC_E_ROI;

        /* step 2 */
        int64_t Wi = rw - 2, Hi = rh - 2;
        if (status == ORC_OK && (cells_x > Wi || cells_y > Hi)) status = ORC_E_GRID;
        if (status == ORC_OK) {
            int64_t maxw = 0, maxh = 0;
            for (int32_t b = 0; b < cells_x; ++b) {
                int64_t cw = ((int64_t)(b + 1) * Wi) / cells_x - ((int64_t)b * Wi) / cells_x;
                if (cw > maxw) maxw = cw;
            }
            for (int32_t b = 0; b < cells_y; ++b) {
                int64_t ch = ((int64_t)(b + 1) * Hi) / cells_y - ((int64_t)b * Hi) / cells_y;
                if (ch > maxh) maxh = ch;
            }
            if (maxw * maxh > 65535) status = ORC_E_OVERFLOW;
        }
        if (roi_status) roi_status[n] = status;
        if (status != ORC_OK) continue;

        const uint8_t* G = grey ? grey + img * grey_img_stride : NULL;
        const uint16_t* D = depth ? depth + img * depth_img_stride : NULL;

        /* one pass per source plane: grey block first, then depth (fused) */
        for (int pass = 0; pass < 2; ++pass) {
            int use_depth;
            if (source == ORC_SRC_FUSED) use_depth = pass;
            else if (pass == 0) use_depth = (source == ORC_SRC_DEPTH);
            else break;
            uint16_t* hb = h + (int64_t)pass * dim;

            /* step 3: loop over blocks with their floor ranges */
            for (int32_t cy = 0; cy < cells_y; ++cy) {
                int64_t i_begin = ((int64_t)cy * Hi) / cells_y;
                int64_t i_end = ((int64_t)(cy + 1) * Hi) / cells_y;
                for (int32_t cx = 0; cx < cells_x; ++cx) {
                    int64_t j_begin = ((int64_t)cx * Wi) / cells_x;
                    int64_t j_end = ((int64_t)(cx + 1) * Wi) / cells_x;
                    uint32_t count[256];
                    for (int b = 0; b < 256; ++b) count[b] = 0;
                    for (int64_t i = i_begin; i < i_end; ++i)
                        for (int64_t j = j_begin; j < j_end; ++j) {
                            int64_t yy = y0 + 1 + i, xx = x0 + 1 + j; /* image pixel */
                            /* step 4: depth window at the centre pixel */
                            int valid = 1;
                            if (D) {
                                uint16_t d = D[yy * depth_pitch + xx];
                                valid = (d != 0) && (d >= dmin) && (d <= dmax);
                            }
                            if (!valid) continue;
                            /* step 5: Eq. 2 on the source plane */
                            uint32_t win[9];
                            for (int r = 0; r < 3; ++r)
                                for (int c = 0; c < 3; ++c)
                                    win[r * 3 + c] =
                                        use_depth ? D[(yy - 1 + r) * depth_pitch + (xx - 1 + c)]
                                                  : G[(yy - 1 + r) * grey_pitch + (xx - 1 + c)];
                            int32_t code = oracle_lbp_code_window(win);
                            /* step 6 */
                            int32_t bin = (bins == 256) ? code : U[code];
                            /* step 7 */
                            count[bin] += 1;
                        }
                    for (int32_t b = 0; b < bins; ++b)
                        hb[((int64_t)cy * cells_x + cx) * bins + b] = (uint16_t)count[b];
                }
            }
        }
    }
    return ORC_OK;
}

/* The grey-source descriptor (the headline configuration, J.north_star). */
int32_t oracle_lbp_extract(const uint8_t* grey, const uint16_t* depth,
                           int32_t n_images, int32_t height, int32_t width,
                           int64_t grey_pitch, int64_t depth_pitch,
                           int64_t grey_img_stride, int64_t depth_img_stride,
                           const int32_t* rois, int32_t n_rois,
                           uint16_t dmin, uint16_t dmax,
                           int32_t cells_x, int32_t cells_y, int32_t bins,
                           uint16_t* desc, int32_t* roi_status)
{
    if (n_rois > 0 && !grey) return ORC_E_ARG;
    return oracle_lbp_extract_src(grey, depth, n_images, height, width, grey_pitch, depth_pitch,
                                  grey_img_stride, depth_img_stride, rois, n_rois, dmin, dmax,
                                  cells_x, cells_y, bins, ORC_SRC_GREY, desc, roi_status);
}

/* ------------------------------------------------------------------------ */
/* One-vs-rest linear SVM training ("finding a hyperplane ...",  */
/* P:144 A-vs-B per identity; S:449-466 train_binary / train_ovr: minimise               */
/* lambda/2 |w|^2 + mean hinge loss by epoch-based subgradient steps 1/(lambda t) over a */
/* seeded visit order).  DESIGN.md reading R20: the bias is folded in as a constant      */
/* feature 1 (regularised with w), lambda = 1 / inv_lambda, and the step is Pegasos':     */
/*   t = 1..T, i = order[t-1], y = +1 if label[i] == c else -1, x~ = (x_i, 1):            */
/*   violated iff t == 1 or y (w_{t-1} . x~) < 1;                                          */
/*   w_t = (1 - 1/t) w_{t-1} + [violated] y x~ / (lambda t).                               */
/* Written exactly: with z_t = lambda t w_t, z_t = z_{t-1} + [violated] y x~ -- an integer */
/* vector -- and (t > 1) the test y (w_{t-1} . x~) < 1 is y (z_{t-1} . x~) < lambda (t-1), */
/* i.e. the integer y (z . x~) < ceil((t - 1) / inv_lambda).  The model is the last       */
/* iterate w_T = inv_lambda z_T / T, rounded once fp64 -> fp32 per entry.                 */
/* Requires |y (z . x~)| < 2^63 (e.g. T <= 2^24 and sum_d x_d <= 2^16).                   */
/* ------------------------------------------------------------------------ */
static int64_t ceil_div_pos(int64_t a, int64_t b) { /* a >= 0, b > 0 */
    return (a + b - 1) / b;
}

int32_t oracle_svm_train_ovr(const uint16_t* desc, int32_t n, int32_t dim,
                             const int32_t* labels, int32_t n_classes,
                             const int32_t* order, int64_t T, int32_t inv_lambda,
                             float* W /* [C][dim] */, float* bias /* [C] */,
                             int64_t* z_out /* nullable [C][dim + 1] */)
{
    if (n < 1 || dim < 1 || n_classes < 1 || T < 1 || inv_lambda < 1) return ORC_E_ARG;
    if (!desc || !labels || !order || !W || !bias) return ORC_E_ARG;
    for (int64_t t = 0; t < T; ++t)
        if (order[t] < 0 || order[t] >= n) return ORC_E_ARG;
    int64_t* z = (int64_t*)malloc((size_t)(dim + 1) * sizeof(int64_t));
    if (!z) return ORC_E_ARG;
    for (int32_t c = 0; c < n_classes; ++c) {
        for (int32_t d = 0; d <= dim; ++d) z[d] = 0;
        for (int64_t t = 1; t <= T; ++t) {
            int32_t i = order[t - 1];
            const uint16_t* x = desc + (int64_t)i * dim;
            int64_t y = (labels[i] == c) ? 1 : -1;
            int violated = 1;
            if (t > 1) {
                int64_t dot = z[dim]; /* the constant feature 1 */
                for (int32_t d = 0; d < dim; ++d) dot += z[d] * (int64_t)x[d];
                violated = y * dot < ceil_div_pos(t - 1, inv_lambda);
            }
            if (violated) {
                for (int32_t d = 0; d < dim; ++d) z[d] += y * (int64_t)x[d];
                z[dim] += y;
            }
        }
        for (int32_t d = 0; d < dim; ++d)
            W[(int64_t)c * dim + d] = (float)((double)((int64_t)inv_lambda * z[d]) / (double)T);
        bias[c] = (float)((double)((int64_t)inv_lambda * z[dim]) / (double)T);
        if (z_out)
            for (int32_t d = 0; d <= dim; ++d) z_out[(int64_t)c * (dim + 1) + d] = z[d];
    }
    free(z);
    return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* Linear OvR SVM on L1-normalised blocks (SURVEY §8f-3 variant; S:379-387 normalize:    */
/* "each block divided by its own count sum; empty block maps to all zeros"):           */
/*   f[n][d] = h[n][d] / N_k for d in block k (N_k = sum of the block's counts;          */
/*   f = 0 when N_k = 0), blocks of `block` consecutive entries (one cell = `bins`);     */
/*   s[n][c] = (float)( (double)b[c] + sum_{d ascending} (double)W[c][d] * f[n][d] )     */
/* with f computed in fp64 (one division per entry), labels as in oracle_svm_score.     */
/* ------------------------------------------------------------------------ */
int32_t oracle_svm_score_l1(const uint16_t* desc, int32_t n, int32_t dim, int32_t block,
                            const float* W, const float* bias, int32_t n_classes,
                            float* scores, int32_t* labels, float* top_score,
                            float reject_threshold)
{
    if (n < 0 || dim < 1 || n_classes < 1 || block < 1 || dim % block != 0) return ORC_E_ARG;
    if (n == 0) return ORC_OK;
    if (!desc || !W || !bias) return ORC_E_ARG;
    double* f = (double*)malloc((size_t)dim * sizeof(double));
    if (!f) return ORC_E_ARG;
    for (int32_t i = 0; i < n; ++i) {
        const uint16_t* h = desc + (int64_t)i * dim;
        for (int32_t k0 = 0; k0 < dim; k0 += block) {
            uint64_t sum = 0;
            for (int32_t d = k0; d < k0 + block; ++d) sum += h[d];
            for (int32_t d = k0; d < k0 + block; ++d)
                f[d] = sum ? (double)h[d] / (double)sum : 0.0;
        }
        float best = 0.0f;
        int32_t best_c = 0;
        for (int32_t c = 0; c < n_classes; ++c) {
            const float* w = W + (int64_t)c * dim;
            double acc = (double)bias[c];
            for (int32_t d = 0; d < dim; ++d) acc += (double)w[d] * f[d];
            float sc = (float)acc;
            if (scores) scores[(int64_t)i * n_classes + c] = sc;
            if (c == 0 || sc > best) {
                best = sc;
                best_c = c;
            }
        }
        if (top_score) top_score[i] = best;
        if (labels) labels[i] = (best < reject_threshold) ? -1 : best_c;
    }
    free(f);
    return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* ROI resize ("The detected face ... is resized to 200x200 pixels";  */
/* SURVEY §8f-2; S:91-99 resize):                                           */
/*  grey : bilinear with half-pixel centres, rounded half up.  Output pixel */
/*         (ox, oy) of an out_w x out_h image samples the source at         */
/*         sx = (ox + 1/2) * w / out_w - 1/2 (likewise sy), clamped below   */
/*         at 0; x0 = floor(sx), x1 = min(x0 + 1, w - 1), fx = sx - x0;     */
/*         v = (1-fx)(1-fy) p00 + fx(1-fy) p10 + (1-fx) fy p01 + fx fy p11, */
/*         result floor(v + 1/2).  Written in exact integers: with D = 2    */
/*         out_w, sx = N / D for N = (2 ox + 1) w - out_w, so fx = (N mod   */
/*         D) / D and every weight is an integer over Dx * Dy.              */
/*  depth: nearest neighbour with half-pixel centres, ties toward the       */
/*         smaller index: x = ceil((sx + 1/2)) - 1 = floor(((2 ox + 1) w -  */
/*         1) / (2 out_w)), clamped to [0, w - 1] -- no 0 (hole) is ever    */
/*         blended into a fabricated depth.                                 */
/* src: h x w samples, row pitch `pitch` (elements); dst: out_h x out_w.    */
/* ------------------------------------------------------------------------ */
static int64_t floor_div(int64_t a, int64_t b) { /* b > 0 */
    int64_t q = a / b;
    return (a % b != 0 && a < 0) ? q - 1 : q;
}

int32_t oracle_resize_grey(const uint8_t* src, int32_t h, int32_t w, int64_t pitch,
                           int32_t out_h, int32_t out_w, uint8_t* dst)
{
    if (!src || !dst || h < 1 || w < 1 || out_h < 1 || out_w < 1 || pitch < w) return ORC_E_ARG;
    int64_t Dx = 2 * (int64_t)out_w, Dy = 2 * (int64_t)out_h;
    for (int32_t oy = 0; oy < out_h; ++oy) {
        int64_t Ny = (2 * (int64_t)oy + 1) * h - out_h;
        if (Ny < 0) Ny = 0;                         /* clamp sy at 0 */
        int64_t y0 = floor_div(Ny, Dy), ry = Ny - y0 * Dy;
        if (y0 > h - 1) { y0 = h - 1; ry = 0; }     /* (cannot happen: sy < h - 1/2) */
        int64_t y1 = y0 + 1 < h ? y0 + 1 : h - 1;
        for (int32_t ox = 0; ox < out_w; ++ox) {
            int64_t Nx = (2 * (int64_t)ox + 1) * w - out_w;
            if (Nx < 0) Nx = 0;
            int64_t x0 = floor_div(Nx, Dx), rx = Nx - x0 * Dx;
            if (x0 > w - 1) { x0 = w - 1; rx = 0; }
            int64_t x1 = x0 + 1 < w ? x0 + 1 : w - 1;
            int64_t p00 = src[y0 * pitch + x0], p10 = src[y0 * pitch + x1];
            int64_t p01 = src[y1 * pitch + x0], p11 = src[y1 * pitch + x1];
            int64_t num = (Dx - rx) * (Dy - ry) * p00 + rx * (Dy - ry) * p10 +
                          (Dx - rx) * ry * p01 + rx * ry * p11;
            int64_t den = Dx * Dy;
            dst[(int64_t)oy * out_w + ox] = (uint8_t)floor_div(2 * num + den, 2 * den);
        }
    }
    return ORC_OK;
}

int32_t oracle_resize_depth(const uint16_t* src, int32_t h, int32_t w, int64_t pitch,
                            int32_t out_h, int32_t out_w, uint16_t* dst)
{
    if (!src || !dst || h < 1 || w < 1 || out_h < 1 || out_w < 1 || pitch < w) return ORC_E_ARG;
    for (int32_t oy = 0; oy < out_h; ++oy) {
        int64_t y = floor_div((2 * (int64_t)oy + 1) * h - 1, 2 * (int64_t)out_h);
        if (y < 0) y = 0;
        if (y > h - 1) y = h - 1;
        for (int32_t ox = 0; ox < out_w; ++ox) {
            int64_t x = floor_div((2 * (int64_t)ox + 1) * w - 1, 2 * (int64_t)out_w);
            if (x < 0) x = 0;
            if (x > w - 1) x = w - 1;
            dst[(int64_t)oy * out_w + ox] = src[y * pitch + x];
        }
    }
    return ORC_OK;
}

/* Resized-ROI descriptor: per ROI n, crop = clamp(roi, image) (empty  */
/* -> ORC_E_ROI), resize the crop to size x size (grey bilinear, depth nearest, above), then */
/* steps 2-7 of oracle_lbp_extract_src on the size x size image with a full ROI.  grey may  */
/* be NULL for the depth source; depth may be NULL (no mask) for the grey source.           */
int32_t oracle_lbp_extract_resized(const uint8_t* grey, const uint16_t* depth,
                                   int32_t n_images, int32_t height, int32_t width,
                                   int64_t grey_pitch, int64_t depth_pitch,
                                   int64_t grey_img_stride, int64_t depth_img_stride,
                                   const int32_t* rois, int32_t n_rois, int32_t size,
                                   uint16_t dmin, uint16_t dmax, int32_t cells_x,
                                   int32_t cells_y, int32_t bins, int32_t source,
                                   uint16_t* desc, int32_t* roi_status)
{
    if (n_rois < 0 || size < 3) return ORC_E_ARG;
    if (source != ORC_SRC_GREY && source != ORC_SRC_DEPTH && source != ORC_SRC_FUSED)
        return ORC_E_ARG;
    if (n_rois == 0) return ORC_OK;
    if (!rois || !desc) return ORC_E_ARG;
    if (source != ORC_SRC_DEPTH && !grey) return ORC_E_ARG;
    if (source != ORC_SRC_GREY && !depth) return ORC_E_ARG;
    if (bins != 59 && bins != 256) return ORC_E_ARG;
    if (cells_x < 1 || cells_y < 1 || dmin > dmax) return ORC_E_ARG;
    if (n_images < 1 || height < 1 || width < 1) return ORC_E_ARG;
    if (grey && (grey_pitch < width || grey_img_stride < grey_pitch * (height - 1) + width))
        return ORC_E_ARG;
    if (depth && (depth_pitch < width || depth_img_stride < depth_pitch * (height - 1) + width))
        return ORC_E_ARG;
    int64_t dim = (int64_t)cells_x * cells_y * bins;
    int64_t row = (source == ORC_SRC_FUSED) ? 2 * dim : dim;
    if (row > 0x7FFFFFFF) return ORC_E_ARG;

    int64_t px = (int64_t)size * size;
    uint8_t* g = (uint8_t*)malloc((size_t)px);
    uint16_t* d = (uint16_t*)malloc((size_t)px * 2);
    if (!g || !d) { free(g); free(d); return ORC_E_ARG; }
    int32_t full[5] = {0, 0, 0, size, size};
    int32_t rc = ORC_OK;
    for (int32_t n = 0; n < n_rois && rc == ORC_OK; ++n) {
        uint16_t* h = desc + (int64_t)n * row;
        const int32_t* roi = rois + (int64_t)n * 5;
        int64_t img = roi[0];
        int64_t x0 = roi[1], y0 = roi[2], x1 = x0 + roi[3], y1 = y0 + roi[4];
        if (x0 < 0) x0 = 0;
        if (y0 < 0) y0 = 0;
        if (x1 > width) x1 = width;
        if (y1 > height) y1 = height;
        if (img < 0 || img >= n_images || x1 <= x0 || y1 <= y0) {
            for (int64_t k = 0; k < row; ++k) h[k] = 0;
            if (roi_status) roi_status[n] = ORC_E_ROI;
            continue;
        }
        int32_t cw = (int32_t)(x1 - x0), ch = (int32_t)(y1 - y0);
        if (grey)
            oracle_resize_grey(grey + img * grey_img_stride + y0 * grey_pitch + x0, ch, cw,
                               grey_pitch, size, size, g);
        if (depth)
            oracle_resize_depth(depth + img * depth_img_stride + y0 * depth_pitch + x0, ch, cw,
                                depth_pitch, size, size, d);
        int32_t st = ORC_OK;
        rc = oracle_lbp_extract_src(grey ? g : NULL, depth ? d : NULL, 1, size, size, size, size,
                                    px, px, full, 1, dmin, dmax, cells_x, cells_y, bins, source,
                                    h, &st);
        if (roi_status) roi_status[n] = st;
    }
    free(g);
    free(d);
    return rc;
}

/* ------------------------------------------------------------------------ */
/* Linear one-vs-rest SVM decision ("a classifier defined by a    */
/* hyperplane"; S:467-475 predict):                      */
/*   s[n][c] = (float)( (double)b[c] + sum_{d ascending} (double)W[c][d] *  */
/*                                                      (double)h[n][d] )   */
/* rounded once to nearest-even fp32; label = argmax_c s over the fp32      */
/* values, ties -> smallest c; top < reject_threshold -> -1. */
/* ------------------------------------------------------------------------ */
int32_t oracle_svm_score(const uint16_t* desc, int32_t n, int32_t dim,
                         const float* W /* [C][dim] */, const float* bias /* [C] */,
                         int32_t n_classes,
                         float* scores /* nullable [n][C] */, int32_t* labels /* nullable [n] */,
                         float* top_score /* nullable [n] */, float reject_threshold)
{
    if (n < 0 || dim < 1 || n_classes < 1) return ORC_E_ARG;
    if (n == 0) return ORC_OK;
    if (!desc || !W || !bias) return ORC_E_ARG;
    for (int32_t i = 0; i < n; ++i) {
        const uint16_t* h = desc + (int64_t)i * dim;
        float best = 0.0f;
        int32_t best_c = 0;
        for (int32_t c = 0; c < n_classes; ++c) {
            const float* w = W + (int64_t)c * dim;
            double acc = (double)bias[c];
            for (int32_t d = 0; d < dim; ++d) acc += (double)w[d] * (double)h[d];
            float s = (float)acc;
            if (scores) scores[(int64_t)i * n_classes + c] = s;
            if (c == 0 || s > best) {
                best = s;
                best_c = c;
            }
        }
        if (top_score) top_score[i] = best;
        if (labels) labels[i] = (best < reject_threshold) ? -1 : best_c;
    }
    return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* Descriptor compaction for the database all-gather ("pack   */
/* counts (u8 + overflow flag) to halve all-gather bytes"; R21).  */
/* An encoding, written as its definition:                                  */
/*   packed[i][d] = min(h[i][d], 255)                                       */
/*   exceptions   = { (row_base + i, d, h[i][d]) : h[i][d] > 255 }, listed   */
/*                  in row-major order; *count = their number (entries past */
/*                  cap are counted but not stored).                        */
/* Decoding: h[r][d] = packed[r][d], then h[row][index] = value for every   */
/* listed exception.  Pins: decode(encode(h)) == h on random and edge data  */
/* (tests/test_oracle_compact.py), packed == the saturated counts.          */
/* ------------------------------------------------------------------------ */
int32_t oracle_desc_pack_u8(const uint16_t* desc, int64_t n, int32_t dim, int64_t row_base,
                            uint8_t* packed, int64_t* exc_row, int32_t* exc_index,
                            int32_t* exc_value, int32_t cap, int32_t* count) {
    if (n < 0 || dim < 1 || cap < 0 || !count) return ORC_E_ARG;
    int32_t c = 0;
    for (int64_t i = 0; i < n; ++i) {
        for (int32_t d = 0; d < dim; ++d) {
            uint16_t h = desc[i * dim + d];
            packed[i * dim + d] = (uint8_t)(h > 255 ? 255 : h);
            if (h > 255) {
                if (c < cap) {
                    exc_row[c] = row_base + i;
                    exc_index[c] = d;
                    exc_value[c] = h;
                }
                ++c;
            }
        }
    }
    *count = c;
    return ORC_OK;
}

int32_t oracle_desc_unpack_u8(const uint8_t* packed, int64_t n, int32_t dim, int64_t row_base,
                              const int64_t* exc_row, const int32_t* exc_index,
                              const int32_t* exc_value, int32_t n_exc, uint16_t* desc) {
    if (n < 0 || dim < 1 || n_exc < 0) return ORC_E_ARG;
    for (int64_t i = 0; i < n * (int64_t)dim; ++i) desc[i] = packed[i];
    for (int32_t k = 0; k < n_exc; ++k) {
        int64_t r = exc_row[k] - row_base;
        if (r < 0 || r >= n || exc_index[k] < 0 || exc_index[k] >= dim) continue;
        desc[r * dim + exc_index[k]] = (uint16_t)exc_value[k];
    }
    return ORC_OK;
}
