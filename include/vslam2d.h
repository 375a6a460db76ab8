/*
 * vslam2d.h — C ABI of the B200-native cuVSLAM 2D-module hot path.
 *
 * Path (§2.1 "2D module"):
 *   per camera-frame: image pyramid -> Sobel -> Shi-Tomasi (GFTT) response ->
 *   3x3 NMS + per-cell top-k over an N x M grid (Eq. 1) ; then pyramidal
 *   Lucas-Kanade (KLT) of the previous frame's keypoints into this frame with
 *   a per-level NCC gate.
 *
 * Conventions for every entry point
 *   - All image / keypoint buffers are CALLER-OWNED DEVICE memory (cudaMalloc /
 *     torch).  Arrays named `*_ptrs` are DEVICE arrays of B device pointers, one
 *     per image, so ring slots and camera buffers are addressed without copies.
 *   - The library never allocates, frees or synchronises and keeps no global
 *     state: calls are thread-safe and ordered on `stream` (a cudaStream_t;
 *     NULL = legacy default stream).  Work is enqueued asynchronously.
 *   - Return value 0 = enqueued.  Negative codes: V2D_EINVAL (bad argument;
 *     nothing enqueued), V2D_EALIGN (pitch/alignment contract violated;
 *     nothing enqueued), V2D_ECUDA (launch failed, from cudaGetLastError;
 *     asynchronous faults surface at the caller's next synchronisation).
 *     Per-keypoint outcomes are never errors: they are statuses.
 *   - Coordinates: x = column in [0,W), y = row in [0,H); pixel centres are
 *     integers; intensities are raw u8 values 0..255 (reading #3).
 *
 * Every call is implemented by hand-written sm_100a kernels in
 * paper_2506_04359_b200/csrc; there is no CPU fallback.
 */
#ifndef VSLAM2D_H
#define VSLAM2D_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* v2d_stream_t; /* identical to cudaStream_t */

#define V2D_OK 0
#define V2D_EINVAL (-1)
#define V2D_EALIGN (-2)
#define V2D_ECUDA (-3)

#define V2D_MAX_LEVELS 8
#define V2D_MAX_K 256
#define V2D_MAX_WIN 29

/* KLT status codes.  LOST_* and SKIPPED slots get pos (-1,-1). */
#define V2D_TRACKED 0
#define V2D_LOST_OOB 1       /* left the image (any L0 iterate, or final pos outside the r-margin) */
#define V2D_LOST_NCC 2       /* NCC_L < ncc_min at some level ("NCC check") */
#define V2D_LOST_SMALL_EIG 3 /* lambda_min(G)/n < min_eig at level 0 */
#define V2D_SKIPPED 4        /* input slot empty (-1,-1) / non-finite, or in_status != 0 */

/* v2d_track_klt flags */
#define V2D_KLT_NCC_EACH_STEP 1u /* variant f3: NCC gate also after every Gauss-Newton update
                                    (literal "at each optimization step") */

/* Pyramid layout of ONE image's levels 1..levels-1 (level 0 is the caller's u8
 * frame).  Level L (L >= 1) is a dense fp32 plane of W[L] x H[L] with row pitch
 * pitch[L] = round_up(W[L], 32) floats (128-B rows), at float offset offset[L]
 * from the image's pyramid base pointer.  floats_per_image = total size;
 * every offset is a multiple of 32 floats.  pitch[0]/offset[0] are 0. */
typedef struct {
  int levels;
  int W[V2D_MAX_LEVELS];
  int H[V2D_MAX_LEVELS];
  int64_t pitch[V2D_MAX_LEVELS];
  int64_t offset[V2D_MAX_LEVELS];
  int64_t floats_per_image;
} v2d_layout;

/* Host-only.  Level sizes W_L = floor(W_{L-1}/2).
 * V2D_EINVAL unless 1 <= levels <= 8, W>>(levels-1) >= 1 and H>>(levels-1) >= 1
 * ("too many levels for image size"), or out == NULL. */
int v2d_pyramid_layout(int W, int H, int levels, v2d_layout* out);

/* Host-only.  Eq. 1: "k > floor(K_I/(N*M))".  k == 0 resolves to
 * floor(K_min/(grid_x*grid_y)) + 1; k > 0 is validated against the
 * same inequality and against V2D_MAX_K.  *k_out receives the per-cell k. */
int v2d_grid_k(int grid_x, int grid_y, int k, int K_min, int* k_out);

/* Image pyramid ("each image pyramid level"; reading #1: 2x2 box, floor
 * halving).  For each of B images: level L = mean of the 2x2 block of
 * level L-1, computed in one pass as the exact mean of the aligned 2^L x 2^L
 * L0 block (bit-exact: values lie in 4^-L * Z).
 *   l0_ptrs   device array [B] of u8 frames, row pitch l0_pitch bytes
 *   pyr_ptrs  device array [B] of fp32 pyramid bases (v2d_layout of W,H,levels)
 * V2D_EALIGN: l0_pitch % 16 != 0 or l0_pitch < W.  levels == 1 enqueues nothing. */
int v2d_build_pyramid(const uint8_t* const* l0_ptrs, int64_t l0_pitch, int B, int W, int H,
                      int levels, float* const* pyr_ptrs, v2d_stream_t stream);

/* Keypoint selection: Sobel/8 gradients, 3x3 structure-tensor
 * response R = lambda_min (fp32 contract, reading #4), eligibility
 * border <= x <= W-1-border (same for y) and R > min_score, optional strict
 * 3x3 NMS on the key (bits(R) << 32 | ~(y*W+x)) (reading #5), and per cell of
 * the grid_x x grid_y floor partition the top-k candidates by that key
 * (reading #6/#8).  k resolves via v2d_grid_k.
 *   kp_xy      [B][grid_y][grid_x][k][2] fp32 (x,y); unfilled slots (-1,-1)
 *   kp_score   [B][grid_y][grid_x][k]    fp32 R; unfilled 0
 *   cell_count [B][grid_y*grid_x]        int32 filled slots per cell
 *   resp       nullable [B][H][W] fp32: full R map (0 outside 2..W-3 x 2..H-3);
 *              when given, the lazy-eigenvalue shortcut is disabled.
 *   workspace  nullable [B][H][round_up(W,32)] fp32 scratch (16-B aligned).  When
 *              given, K2 runs as two dense
 *              passes (per-pixel candidate map, then per-cell selection); when
 *              NULL, as one fused per-cell kernel.  Results are identical.
 *   mask_ptrs  nullable device array [B] of u8 masks (row pitch l0_pitch); a
 *              non-zero mask pixel is not eligible (min_separation suppression,
 *              S:158; NMS still compares against it)
 *   enable     nullable device int32 flag; when *enable == 0 the call does
 *              nothing (keyframe-conditional detection without a host sync)
 * V2D_EINVAL: border < 3, W or H < 2*border+1, grid cell < 1 px, bad k, nms not
 * 0/1, l0_pitch*H >= 2^31.  V2D_EALIGN: l0_pitch % 16 != 0. */
int v2d_detect_gftt(const uint8_t* const* l0_ptrs, int64_t l0_pitch, int B, int W, int H,
                    int grid_x, int grid_y, int k, int K_min, float min_score, int border,
                    int nms, float* kp_xy, float* kp_score, int32_t* cell_count, float* resp,
                    float* workspace, const uint8_t* const* mask_ptrs, const int32_t* enable,
                    v2d_stream_t stream);

/* Pyramidal LK tracking (LK_1981, LK_2000; reading of SURVEY §8(c) D7):
 * forward-additive Gauss-Newton with template gradients, coarse-to-fine over
 * `levels`, at most `iters` steps per level (stop when |eta| < eps, level px),
 * NCC(template, warped patch) >= ncc_min required after every level, window
 * win x win (odd, 3..V2D_MAX_WIN).  Image b's keypoints pts[b] (L0 px, in the
 * PREVIOUS frame) are tracked from (prev_l0_ptrs[b], prev_pyr_ptrs[b]) into
 * (next_l0_ptrs[b], next_pyr_ptrs[b]); pyramids as built by v2d_build_pyramid.
 *   pts        [B][P][2] fp32; (-1,-1) = empty slot -> V2D_SKIPPED
 *   guess      nullable [B][P][2] fp32 displacement prior (L0 px)
 *   in_status  nullable [B][P] u8; non-zero -> V2D_SKIPPED (lost is terminal)
 *   out_pos    [B][P][2] fp32 tracked position, (-1,-1) unless V2D_TRACKED
 *   status     [B][P] u8 V2D_* status
 *   ncc        nullable [B][P] fp32 last evaluated NCC (0 if none)
 *   iters_out  nullable [B][P] int32 work counters: bits 0..23 = Gauss-Newton
 *              steps over all levels, bits 24..31 = levels whose template was built
 *   track_list nullable [B][P][4] fp32, 16-B aligned: the track-list record
 *              (x, y, status, ncc) = (out_pos, (float)status, ncc) of every slot,
 *              the unit the rig-wide all-gather ships ("we collect
 *              all the available observations"), written by the same kernel
 * min_eig is in (gray/px)^2 per window pixel: lost at L0 when lambda_min(G)/n
 * < min_eig; coarse levels are skipped instead (reading #15).  min_eig must be
 * > 0 (reading #27: it guarantees det(G) > 0 for the closed-form 2x2 solve).
 * flags: 0 or V2D_KLT_NCC_EACH_STEP; unknown bits -> V2D_EINVAL.
 * V2D_EINVAL also for B*P > INT32_MAX (one warp per slot) and min_eig <= 0 / NaN;
 * V2D_EALIGN for a track_list that is not 16-B aligned. */
int v2d_track_klt(const uint8_t* const* prev_l0_ptrs, const float* const* prev_pyr_ptrs,
                  const uint8_t* const* next_l0_ptrs, const float* const* next_pyr_ptrs,
                  int64_t l0_pitch, int B, int W, int H, int levels, const float* pts,
                  const float* guess, const uint8_t* in_status, int P, int win, int iters,
                  float eps, float ncc_min, float min_eig, float* out_pos, uint8_t* status,
                  float* ncc, int32_t* iters_out, float* track_list, unsigned flags,
                  v2d_stream_t stream);

/* Per-level patch features (variant f4; "a list of 9x9 image
 * patches taken from each level of the image pyramid").  For
 * every keypoint p of image b and every level L, the patch x patch samples
 * S(I_L, c_L + (u, v)), u, v in [-(patch-1)/2, (patch-1)/2], c_L = (p+0.5)/2^L - 0.5
 * (reading #2), bilinear with clamp-to-edge (D2), of the frame whose level 0 is
 * l0_ptrs[b] and levels >= 1 pyr_ptrs[b].
 *   pts   [B][P][2] fp32 L0 px; empty slots (-1,-1) / non-finite -> all-zero patches
 *   out   [B][P][levels][patch][patch] fp32
 * V2D_EINVAL: patch even, < 1 or > 31; bad levels / sizes; B*P > INT32_MAX. */
int v2d_extract_patches(const uint8_t* const* l0_ptrs, const float* const* pyr_ptrs,
                        int64_t l0_pitch, int B, int W, int H, int levels, const float* pts,
                        int P, int patch, float* out, v2d_stream_t stream);

/* ---- variant f1: keyframe-driven continuous tracking (Eq. 5;
 * SPEC S:136-143).  A track table per image holds P slots:
 * tracks [B][P][2] fp32, status [B][P] u8 (the KLT status codes: V2D_TRACKED =
 * alive, anything else = lost; passing it back as v2d_track_klt's in_status makes
 * lost terminal), kf_member [B][P] u8 (slot in S_kf), track_id [B][P]
 * int32, next_id [B] int32.  A lost slot only becomes alive again through
 * refill, with a new id. */

/* mask(x,y) := 1 iff (x-tx)^2 + (y-ty)^2 < min_sep^2 for an alive track t of the
 * image, else 0 (exact fp64 test).  mask_ptrs: device array [B] of u8 images,
 * row pitch mask_pitch (% 16 == 0).  enable: nullable device flag (0 = skip). */
int v2d_suppress_mask(const float* tracks, const uint8_t* status, int B, int P, float min_sep,
                      int W, int H, uint8_t* const* mask_ptrs, int64_t mask_pitch,
                      const int32_t* enable, v2d_stream_t stream);

/* counts[b] = {|S_kf|, |S_curr ∩ S_kf|} = {#kf_member, #(kf_member and alive)}. */
int v2d_track_survival(const uint8_t* status, const uint8_t* kf_member, int B, int P,
                       int32_t* counts, v2d_stream_t stream);

/* Rig-wide Eq. 5 over n images' counts: *flag = 1 iff sum|S_kf| == 0 (bootstrap)
 * or sum|S_curr ∩ S_kf| < T * sum|S_kf| (fp64), else 0.  totals (nullable,
 * int64[2]) receives the sums.  Multi-GPU: all-reduce the counts first. */
int v2d_keyframe_decide(const int32_t* counts, int n, float T, int32_t* flag, int64_t* totals,
                        v2d_stream_t stream);

/* v2d_keyframe_decide for the f1 loop recorded as one CUDA graph per frame: the same
 * decision into *flag, then kf_count[0] += *flag (nullable int64[1]: keyframes so far)
 * and, if cond_handle != 0, cudaGraphSetConditional(cond_handle, *flag).  cond_handle
 * is the value of a cudaGraphConditionalHandle (CUDA >= 12.3) of the graph this launch
 * is captured into, whose IF node holds the keyframe branch (suppress, detect, refill):
 * on non-keyframe frames those kernels are then skipped by the device instead of
 * launched to exit on *flag.  cond_handle must be 0 outside such a graph (then this is
 * v2d_keyframe_decide plus the counter). */
int v2d_keyframe_decide_graph(const int32_t* counts, int n, float T, int32_t* flag,
                              int64_t* totals, int64_t* kf_count, uint64_t cond_handle,
                              v2d_stream_t stream);

/* v2d_track_survival + v2d_keyframe_decide_graph over all B images in ONE launch (the f1
 * loop is launch-bound): counts[b] as v2d_track_survival, then the last block to finish
 * takes the rig-wide decision into *flag (totals, kf_count, cond_handle as in
 * v2d_keyframe_decide_graph).  done: device uint32[1], 0 before the first call; the
 * launch leaves it 0 (one launch at a time per `done`).  Single-process rigs; with a
 * multi-GPU group use v2d_track_survival, an all-reduce and v2d_keyframe_decide.
 * V2D_EINVAL: B < 1 or > 65535, null counts/flag/done, T < 0 or NaN. */
int v2d_survival_decide(const uint8_t* status, const uint8_t* kf_member, int B, int P,
                        int32_t* counts, float T, int32_t* flag, int64_t* totals,
                        int64_t* kf_count, uint64_t cond_handle, uint32_t* done,
                        v2d_stream_t stream);

/* Frame tables of a captured streaming loop (the graph replays with no host work):
 * t = *counter; cur[c] = table[t mod R][c], prev[c] = table[(t-1) mod R][c] for
 * c < C (device pointers as int64; table: device int64 [R][C]); then *counter = t+1.
 * V2D_EINVAL: R < 1, C < 1 or > 65535, null pointer. */
int v2d_ring_tables(const int64_t* table, int R, int C, int64_t* counter, int64_t* cur,
                    int64_t* prev, v2d_stream_t stream);

/* If *flag: the j-th valid detection of image b (cell-major slot order of
 * v2d_detect_gftt's kp_xy, the first cell_count slots of each cell) fills the
 * j-th dead slot (ascending): status := V2D_TRACKED, id := next_id + j; then
 * kf_member := alive for every slot and next_id advances.  No-op if *flag == 0.
 * grid_x*grid_y <= 1024. */
int v2d_refill_tracks(const float* kp_xy, const int32_t* cell_count, int grid_x, int grid_y,
                      int k, const int32_t* flag, int B, int P, float* tracks, uint8_t* status,
                      uint8_t* kf_member, int32_t* track_id, int32_t* next_id,
                      v2d_stream_t stream);

/* Static string for a V2D_* return code. */
const char* v2d_strerror(int code);

/* ABI version (major*100 + minor). */
int v2d_version(void);

#ifdef __cplusplus
}
#endif
#endif /* VSLAM2D_H */
