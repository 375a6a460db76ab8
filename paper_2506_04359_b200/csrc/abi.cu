// abi.cu — the extern "C" boundary declared in include/vslam2d.h: argument
// validation, layout arithmetic and kernel launches.  No computation of the
// method happens here (it is all in pyramid.cu, gftt.cu, klt.cu).
#include <cmath>

#include "common.cuh"

namespace {

// D1 level sizes + fp32 layout of levels 1..L-1 (128-B rows, 128-B aligned levels).
int make_levels(int W, int H, int levels, v2d::Levels* lv, int64_t* total) {
  if (W < 1 || H < 1 || levels < 1 || levels > V2D_MAX_LEVELS) return V2D_EINVAL;
  if ((W >> (levels - 1)) < 1 || (H >> (levels - 1)) < 1) return V2D_EINVAL;
  int64_t off = 0;
  lv->n = levels;
  for (int L = 0; L < V2D_MAX_LEVELS; ++L) {
    lv->W[L] = L < levels ? (W >> L) : 0;
    lv->H[L] = L < levels ? (H >> L) : 0;
    lv->pitch[L] = 0;
    lv->offset[L] = 0;
    if (L >= 1 && L < levels) {
      lv->pitch[L] = v2d::round_up64(lv->W[L], 32);
      lv->offset[L] = off;
      off += lv->pitch[L] * lv->H[L];
    }
  }
  if (total) *total = off;
  return V2D_OK;
}

int grid_k(int gx, int gy, int k, int K_min, int* k_out) {
  if (gx < 1 || gy < 1 || k < 0 || K_min < 0) return V2D_EINVAL;
  const int64_t q = (int64_t)K_min / ((int64_t)gx * gy);  // floor(K_I/(N*M)), Eq. 1
  const int64_t kk = k == 0 ? q + 1 : k;
  if (kk <= q || kk > V2D_MAX_K) return V2D_EINVAL;
  if (k_out) *k_out = (int)kk;
  return V2D_OK;
}

}  // namespace

extern "C" {

int v2d_version(void) { return 201; }

const char* v2d_strerror(int code) {
  switch (code) {
    case V2D_OK: return "ok";
    case V2D_EINVAL: return "invalid argument";
    case V2D_EALIGN: return "pitch or alignment contract violated";
    case V2D_ECUDA: return "CUDA launch error";
    default: return "unknown error";
  }
}

int v2d_pyramid_layout(int W, int H, int levels, v2d_layout* out) {
  if (!out) return V2D_EINVAL;
  v2d::Levels lv;
  int64_t total = 0;
  const int rc = make_levels(W, H, levels, &lv, &total);
  if (rc) return rc;
  out->levels = levels;
  for (int L = 0; L < V2D_MAX_LEVELS; ++L) {
    out->W[L] = lv.W[L];
    out->H[L] = lv.H[L];
    out->pitch[L] = lv.pitch[L];
    out->offset[L] = lv.offset[L];
  }
  out->floats_per_image = total;
  return V2D_OK;
}

int v2d_grid_k(int grid_x, int grid_y, int k, int K_min, int* k_out) {
  return grid_k(grid_x, grid_y, k, K_min, k_out);
}

int v2d_build_pyramid(const uint8_t* const* l0_ptrs, int64_t l0_pitch, int B, int W, int H,
                      int levels, float* const* pyr_ptrs, v2d_stream_t stream) {
  v2d::Levels lv;
  if (B < 0 || B > 65535 || (B > 0 && (!l0_ptrs || !pyr_ptrs))) return V2D_EINVAL;
  if (make_levels(W, H, levels, &lv, nullptr)) return V2D_EINVAL;
  if (l0_pitch < W || (l0_pitch % 16) != 0) return V2D_EALIGN;
  return v2d::launch_pyramid(l0_ptrs, l0_pitch, B, W, H, lv, pyr_ptrs,
                             reinterpret_cast<cudaStream_t>(stream));
}

int v2d_detect_gftt(const uint8_t* const* l0_ptrs, int64_t l0_pitch, int B, int W, int H,
                    int grid_x, int grid_y, int k, int K_min, float min_score, int border,
                    int nms, float* kp_xy, float* kp_score, int32_t* cell_count, float* resp,
                    float* workspace, const uint8_t* const* mask_ptrs, const int32_t* enable,
                    v2d_stream_t stream) {
  int kk = 0;
  if (B < 0 || B > 65535) return V2D_EINVAL;
  if (B > 0 && (!l0_ptrs || !kp_xy || !kp_score || !cell_count)) return V2D_EINVAL;
  if (W < 1 || H < 1 || (int64_t)W * H >= ((int64_t)1 << 31)) return V2D_EINVAL;
  if (border < 3 || W < 2 * border + 1 || H < 2 * border + 1) return V2D_EINVAL;
  if (grid_x < 1 || grid_y < 1 || grid_x > W || grid_y > H) return V2D_EINVAL;
  if ((int64_t)grid_x * grid_y > 65535 * 16) return V2D_EINVAL;
  if (nms != 0 && nms != 1) return V2D_EINVAL;
  if (std::isnan(min_score)) return V2D_EINVAL;
  if (grid_k(grid_x, grid_y, k, K_min, &kk)) return V2D_EINVAL;
  if (l0_pitch < W || (l0_pitch % 16) != 0) return V2D_EALIGN;
  if (l0_pitch * (int64_t)H >= ((int64_t)1 << 31)) return V2D_EINVAL;  // 32-bit row offsets
  v2d::GfttArgs a{W, H, grid_x, grid_y, kk, border, nms, min_score, l0_pitch};
  if (workspace)
    return v2d::launch_gftt_dense(l0_ptrs, B, a, kp_xy, kp_score, cell_count, resp, workspace,
                                  mask_ptrs, enable, reinterpret_cast<cudaStream_t>(stream));
  return v2d::launch_gftt(l0_ptrs, B, a, kp_xy, kp_score, cell_count, resp, mask_ptrs, enable,
                          reinterpret_cast<cudaStream_t>(stream));
}

int v2d_track_klt(const uint8_t* const* prev_l0_ptrs, const float* const* prev_pyr_ptrs,
                  const uint8_t* const* next_l0_ptrs, const float* const* next_pyr_ptrs,
                  int64_t l0_pitch, int B, int W, int H, int levels, const float* pts,
                  const float* guess, const uint8_t* in_status, int P, int win, int iters,
                  float eps, float ncc_min, float min_eig, float* out_pos, uint8_t* status,
                  float* ncc, int32_t* iters_out, float* track_list, unsigned flags,
                  v2d_stream_t stream) {
  v2d::Levels lv;
  if (flags & ~V2D_KLT_NCC_EACH_STEP) return V2D_EINVAL;
  if (B < 0 || P < 0) return V2D_EINVAL;
  if ((int64_t)B * P > INT32_MAX) return V2D_EINVAL;  // one warp-CTA per slot: grid.x limit
  if (track_list && (reinterpret_cast<uintptr_t>(track_list) & 15)) return V2D_EALIGN;
  if (make_levels(W, H, levels, &lv, nullptr)) return V2D_EINVAL;
  if (win < 3 || win > V2D_MAX_WIN || (win % 2) == 0 || iters < 1) return V2D_EINVAL;
  // min_eig > 0 (DESIGN reading #27): it is what guarantees det(G) > 0 for the 2x2 solve
  if (!(eps >= 0.0f) || std::isnan(ncc_min) || !(min_eig > 0.0f)) return V2D_EINVAL;
  if ((int64_t)B * P > 0 && (!prev_l0_ptrs || !next_l0_ptrs || !pts || !out_pos || !status))
    return V2D_EINVAL;
  if ((int64_t)B * P > 0 && levels > 1 && (!prev_pyr_ptrs || !next_pyr_ptrs)) return V2D_EINVAL;
  if (l0_pitch < W || (l0_pitch % 16) != 0) return V2D_EALIGN;
  v2d::KltArgs a{W, H, P, win, iters, eps, ncc_min, min_eig, l0_pitch, flags};
  return v2d::launch_klt(prev_l0_ptrs, prev_pyr_ptrs, next_l0_ptrs, next_pyr_ptrs, B, lv, a, pts,
                         guess, in_status, out_pos, status, ncc, iters_out, track_list,
                         reinterpret_cast<cudaStream_t>(stream));
}

int v2d_extract_patches(const uint8_t* const* l0_ptrs, const float* const* pyr_ptrs,
                        int64_t l0_pitch, int B, int W, int H, int levels, const float* pts,
                        int P, int patch, float* out, v2d_stream_t stream) {
  v2d::Levels lv;
  if (B < 0 || P < 0 || patch < 1 || patch > 31 || (patch % 2) == 0) return V2D_EINVAL;
  if ((int64_t)B * P > INT32_MAX) return V2D_EINVAL;  // one warp per keypoint: grid.x limit
  if (make_levels(W, H, levels, &lv, nullptr)) return V2D_EINVAL;
  if ((int64_t)B * P > 0 && (!l0_ptrs || !pts || !out || (levels > 1 && !pyr_ptrs)))
    return V2D_EINVAL;
  if (l0_pitch < W || (l0_pitch % 16) != 0) return V2D_EALIGN;
  return v2d::launch_patches(l0_ptrs, pyr_ptrs, l0_pitch, B, lv, pts, P, patch, out,
                             reinterpret_cast<cudaStream_t>(stream));
}

int v2d_suppress_mask(const float* tracks, const uint8_t* status, int B, int P, float min_sep,
                      int W, int H, uint8_t* const* mask_ptrs, int64_t mask_pitch,
                      const int32_t* enable, v2d_stream_t stream) {
  if (B < 0 || B > 65535 || P < 0 || W < 1 || H < 1 || !(min_sep >= 0.0f)) return V2D_EINVAL;
  if (B > 0 && (!mask_ptrs || (P > 0 && (!tracks || !status)))) return V2D_EINVAL;
  if (mask_pitch < W || (mask_pitch % 16) != 0) return V2D_EALIGN;
  return v2d::launch_suppress(mask_ptrs, mask_pitch, B, W, H, tracks, status, P, min_sep, enable,
                              reinterpret_cast<cudaStream_t>(stream));
}

int v2d_track_survival(const uint8_t* status, const uint8_t* kf_member, int B, int P,
                       int32_t* counts, v2d_stream_t stream) {
  if (B < 0 || P < 0 || (B > 0 && (!counts || (P > 0 && (!status || !kf_member)))))
    return V2D_EINVAL;
  return v2d::launch_survival(status, kf_member, B, P, counts,
                              reinterpret_cast<cudaStream_t>(stream));
}

int v2d_keyframe_decide(const int32_t* counts, int n, float T, int32_t* flag, int64_t* totals,
                        v2d_stream_t stream) {
  if (n < 0 || !flag || (n > 0 && !counts) || !(T >= 0.0f)) return V2D_EINVAL;
  return v2d::launch_decide(counts, n, T, flag, totals, nullptr, 0ull,
                            reinterpret_cast<cudaStream_t>(stream));
}

int v2d_keyframe_decide_graph(const int32_t* counts, int n, float T, int32_t* flag,
                              int64_t* totals, int64_t* kf_count, uint64_t cond_handle,
                              v2d_stream_t stream) {
  if (n < 0 || !flag || (n > 0 && !counts) || !(T >= 0.0f)) return V2D_EINVAL;
  return v2d::launch_decide(counts, n, T, flag, totals, kf_count,
                            (unsigned long long)cond_handle,
                            reinterpret_cast<cudaStream_t>(stream));
}

int v2d_survival_decide(const uint8_t* status, const uint8_t* kf_member, int B, int P,
                        int32_t* counts, float T, int32_t* flag, int64_t* totals,
                        int64_t* kf_count, uint64_t cond_handle, uint32_t* done,
                        v2d_stream_t stream) {
  if (B < 1 || B > 65535 || P < 0 || !counts || !flag || !done || !(T >= 0.0f) ||
      (P > 0 && (!status || !kf_member)))
    return V2D_EINVAL;
  return v2d::launch_survival_decide(status, kf_member, B, P, counts, T, flag, totals, kf_count,
                                     (unsigned long long)cond_handle,
                                     reinterpret_cast<unsigned*>(done),
                                     reinterpret_cast<cudaStream_t>(stream));
}

int v2d_ring_tables(const int64_t* table, int R, int C, int64_t* counter, int64_t* cur,
                    int64_t* prev, v2d_stream_t stream) {
  if (R < 1 || C < 1 || C > 65535 || !table || !counter || !cur || !prev) return V2D_EINVAL;
  return v2d::launch_ring_tables(table, R, C, counter, cur, prev,
                                 reinterpret_cast<cudaStream_t>(stream));
}

int v2d_refill_tracks(const float* kp_xy, const int32_t* cell_count, int grid_x, int grid_y,
                      int k, const int32_t* flag, int B, int P, float* tracks, uint8_t* status,
                      uint8_t* kf_member, int32_t* track_id, int32_t* next_id,
                      v2d_stream_t stream) {
  if (B < 0 || P < 0 || grid_x < 1 || grid_y < 1 || grid_x * grid_y > 1024 || k < 1 || !flag)
    return V2D_EINVAL;
  if (B > 0 && (!kp_xy || !cell_count || !tracks || !status || !kf_member || !track_id ||
                !next_id))
    return V2D_EINVAL;
  return v2d::launch_refill(kp_xy, cell_count, grid_x * grid_y, k, flag, B, P, tracks, status,
                            kf_member, track_id, next_id, reinterpret_cast<cudaStream_t>(stream));
}

}  // extern "C"
