/*
 * v2dref.h — ORACLE for the cuVSLAM 2D-module hot path (arXiv 2506.04359).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load, call or link this.
 * The product path (paper_2506_04359_b200/) never touches it, and the two share
 * no code, headers, tables or helpers.
 *
 * Plain, slow, single-threaded host implementation that follows the method
 * step by step (§2.1 "2D module") under the readings fixed in
 * SURVEY.md §8(c) D1-D7 and listed in DESIGN.md §3.  Pyramid and response are
 * exact integer / fp64 arithmetic (the response's final value follows the fp32
 * contract D4 so that selection decisions are taken in the same precision as
 * the kernel, per task rule ③); KLT runs in float64.
 *
 * All buffers are host memory owned by the caller.  Functions return 0 on
 * success and V2DREF_EINVAL (-1) on an invalid argument (nothing is written).
 */
#ifndef V2DREF_H
#define V2DREF_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define V2DREF_OK 0
#define V2DREF_EINVAL (-1)

/* KLT status codes (SURVEY §8(b) "Status codes"). */
#define V2DREF_TRACKED 0
#define V2DREF_LOST_OOB 1
#define V2DREF_LOST_NCC 2
#define V2DREF_LOST_SMALL_EIG 3
#define V2DREF_SKIPPED 4

/* D1: level sizes W_L = floor(W_{L-1}/2).  Ws/Hs receive `levels` entries.
 * EINVAL unless 1 <= levels <= 8 and W>>(levels-1) >= 1, H>>(levels-1) >= 1
 * ("too many levels for image size"). */
int v2dref_level_dims(int W, int H, int levels, int* Ws, int* Hs);

/* Number of doubles of a dense pyramid (all levels, level 0 included). */
int64_t v2dref_pyramid_size(int W, int H, int levels);

/* D1: box pyramid.  `out` receives levels 0..levels-1 as dense row-major
 * float64 planes, concatenated (level L at offset sum_{l<L} W_l*H_l).
 * Level 0 is the u8 frame as exact reals 0..255 (reading #3). */
int v2dref_build_pyramid(const uint8_t* img, int64_t pitch, int W, int H,
                         int levels, double* out);

/* D2: clamp-to-edge bilinear sample of a dense W x H plane. */
double v2dref_bilinear(const double* I, int W, int H, double x, double y);

/* D3: clamp-to-edge Sobel/8 gradients of a dense W x H plane. */
void v2dref_sobel(const double* I, int W, int H, double* gx, double* gy);

/* 2x2 symmetric [[a,b],[b,c]] minimum eigenvalue, float64, written as
 * det/lambda_max (0 when a+c == 0). */
double v2dref_lambda_min(double a, double b, double c);

/* D4: GFTT response of an u8 frame.  R (W*H floats, row-major, dense) gets
 * the fp32-contract value on 2<=x<=W-3, 2<=y<=H-3 and 0 elsewhere.
 * lmin (nullable) gets lambda_min of the same tensor in long double, scaled
 * identically (for the contract-vs-exact pin).  Requires W,H >= 5. */
int v2dref_response(const uint8_t* img, int64_t pitch, int W, int H,
                    float* R, double* lmin);

/* Eq. 1: k == 0 -> floor(K_min/(gx*gy)) + 1; k > 0 must satisfy
 * k > floor(K_min/(gx*gy)) and k <= 256. */
int v2dref_grid_k(int grid_x, int grid_y, int k, int K_min, int* k_out);

/* D5-D6: eligibility, 3x3 NMS on the 64-bit key, per-cell top-k.
 * kp_xy [gy][gx][k][2], kp_score [gy][gx][k], cell_count [gy*gx]; k is the
 * value v2dref_grid_k resolves.  Unfilled slots: (-1,-1), score 0.
 * mask (nullable, row pitch = pitch): non-zero pixels are not eligible
 * (min_separation suppression; variant f1).
 * EINVAL: border < 3, grid cell < 1 px, bad k, W or H < 2*border+1. */
int v2dref_detect_gftt(const uint8_t* img, int64_t pitch, int W, int H,
                       int grid_x, int grid_y, int k, int K_min,
                       float min_score, int border, int nms, const uint8_t* mask,
                       float* kp_xy, float* kp_score, int32_t* cell_count);

/* Two-pass NCC of two n-vectors; 0 if the denominator is 0 (reading #14). */
double v2dref_ncc(const double* P, const double* Q, int n);

/* D7: pyramidal forward-additive LK with template gradients and a per-level
 * NCC gate.  prev_pyr / next_pyr are dense pyramids from
 * v2dref_build_pyramid of the same W x H and level count.
 * ncc_each_step != 0 selects the literal reading of P:61 ("NCC check at each
 * optimization step", variant f3 / DESIGN.md reading #13): the NCC gate is
 * also applied after every Gauss-Newton update, not only after each level.
 * pts [P][2] (L0 px; (-1,-1) = empty slot), guess [P][2] nullable (L0 px
 * displacement prior), in_status [P] nullable (non-zero = already lost).
 * Outputs: out_pos [P][2] (float64; (-1,-1) unless TRACKED), status [P],
 * ncc [P] nullable (last evaluated NCC, 0 if none),
 * diag [P][4] nullable — decision margins for status-flip attribution:
 *   [0] min_L |NCC_L - ncc_min|               over evaluated levels
 *   [1] min_L |lambda/n - min_eig| / (lambda_max/n)
 *   [2] min distance (level px) of any bound test to its bound
 *   [3] min |‖eta‖ - eps| over all iterations (convergence decisions)
 *   (+inf when the decision never happened). */
int v2dref_track_klt(const double* prev_pyr, const double* next_pyr,
                     int W, int H, int levels,
                     const float* pts, const float* guess,
                     const uint8_t* in_status, int P,
                     int win, int iters, double eps, double ncc_min,
                     double min_eig, int ncc_each_step,
                     double* out_pos, uint8_t* status, double* ncc,
                     double* diag);

/* Variant f4: patch x patch bilinear samples of every level at
 * c_L + (u, v), c_L = (p+0.5)/2^L - 0.5; out [P][levels][patch][patch];
 * empty slots (-1,-1) give zeros.  pyr: dense pyramid of v2dref_build_pyramid. */
int v2dref_extract_patches(const double* pyr, int W, int H, int levels, const float* pts, int P,
                           int patch, double* out);

/* ---- variant f1 (Eq. 5) ---- */
/* Track tables use the KLT status as liveness: status 0 (TRACKED) = alive.
 * mask[y*W + x] = 1 iff (x-tx)^2 + (y-ty)^2 < min_sep^2 for an alive track. */
int v2dref_suppress_mask(const float* tracks, const uint8_t* status, int P, double min_sep,
                         int W, int H, uint8_t* mask);
/* SPEC keyframe_due: 1 iff n_surv / n_kf < T (bootstrap: n_kf == 0 -> 1). */
int v2dref_keyframe_due(int64_t n_kf, int64_t n_surv, double T);
/* Refill dead slots (status != 0, ascending) with the valid detections in slot
 * order (first cell_count[c] slots of each cell c): status := 0, ids next_id + j;
 * then kf_member := (status == 0). */
int v2dref_refill(const float* kp_xy, const int32_t* cell_count, int cells, int k, int P,
                  float* tracks, uint8_t* status, uint8_t* kf_member, int32_t* track_id,
                  int32_t* next_id);

#ifdef __cplusplus
}
#endif
#endif /* V2DREF_H */
