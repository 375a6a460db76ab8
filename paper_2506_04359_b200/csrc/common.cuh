// common.cuh — internal helpers shared by the sm_100a kernels of the 2D hot path.
// Product code only: nothing here is shared with oracle/ (task rule ③).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "vslam2d.h"

// K3 Gauss-Newton residual and NCC samples with the vertical bilinear weight folded
// into two FMAs (one packed op per window row fewer; same-box A/B -1.4 % at 21x21).
// One-warp kernel (windows >= 15) only; the pair kernel's small windows failed parity
// with it (klt_pair.cu).
#ifndef V2D_GN_FOLD
#define V2D_GN_FOLD 1
#endif
#ifndef V2D_GN_FOLD_PAIR
#define V2D_GN_FOLD_PAIR 0
#endif

namespace v2d {

constexpr unsigned kFullMask = 0xffffffffu;

// sum / n with one Newton correction of sum * (1/n): equals sum / n exactly whenever that
// quotient is representable (a flat template: n equal values), without the IEEE
// division subroutine
__device__ __forceinline__ float exact_mean(float sum, float n) {
  const float inv = 1.0f / n;
  const float q = sum * inv;
  return fmaf(fmaf(-n, q, sum), inv, q);
}

// Level geometry passed by value to kernels (mirrors v2d_layout).
struct Levels {
  int n;
  int W[V2D_MAX_LEVELS];
  int H[V2D_MAX_LEVELS];
  int64_t pitch[V2D_MAX_LEVELS];   // floats (levels >= 1)
  int64_t offset[V2D_MAX_LEVELS];  // floats (levels >= 1)
};

__host__ __device__ inline int64_t round_up64(int64_t x, int64_t m) { return (x + m - 1) / m * m; }

// Launch helpers (defined in the kernel translation units).
int launch_pyramid(const uint8_t* const* l0_ptrs, int64_t l0_pitch, int B, int W, int H,
                   const Levels& lv, float* const* pyr_ptrs, cudaStream_t st);

struct GfttArgs {
  int W, H, grid_x, grid_y, k, border, nms;
  float min_score;
  int64_t pitch;
};
int launch_gftt(const uint8_t* const* l0_ptrs, int B, const GfttArgs& a, float* kp_xy,
                float* kp_score, int32_t* cell_count, float* resp,
                const uint8_t* const* mask_ptrs, const int32_t* enable, cudaStream_t st);

struct KltArgs {
  int W, H, P, win, iters;
  float eps, ncc_min, min_eig;
  int64_t l0_pitch;
  unsigned flags;
};
int launch_klt(const uint8_t* const* prev_l0, const float* const* prev_pyr,
               const uint8_t* const* next_l0, const float* const* next_pyr, int B,
               const Levels& lv, const KltArgs& a, const float* pts, const float* guess,
               const uint8_t* in_status, float* out_pos, uint8_t* status, float* ncc,
               int32_t* iters_out, float* track_list, cudaStream_t st);

// K3 for windows <= 13 (klt_pair.cu): two keypoints per warp
bool klt_pair_supported(int win);
int launch_klt_pair(const uint8_t* const* prev_l0, const float* const* prev_pyr,
                    const uint8_t* const* next_l0, const float* const* next_pyr, int B,
                    const Levels& lv, const KltArgs& a, const float* pts, const float* guess,
                    const uint8_t* in_status, float* out_pos, uint8_t* status, float* ncc,
                    int32_t* iters_out, float* track_list, cudaStream_t st);

int launch_patches(const uint8_t* const* l0_ptrs, const float* const* pyr_ptrs, int64_t l0_pitch,
                   int B, const Levels& lv, const float* pts, int P, int patch, float* out,
                   cudaStream_t st);

int launch_gftt_dense(const uint8_t* const* l0_ptrs, int B, const GfttArgs& a, float* kp_xy,
                      float* kp_score, int32_t* cell_count, float* resp, float* ws,
                      const uint8_t* const* mask_ptrs, const int32_t* enable, cudaStream_t st);
int launch_suppress(uint8_t* const* mask_ptrs, int64_t pitch, int B, int W, int H,
                    const float* tracks, const uint8_t* status, int P, float min_sep,
                    const int32_t* enable, cudaStream_t st);
int launch_survival(const uint8_t* status, const uint8_t* kf_member, int B, int P, int32_t* counts,
                    cudaStream_t st);
int launch_decide(const int32_t* counts, int n, float T, int32_t* flag, int64_t* totals,
                  int64_t* kf_count, unsigned long long cond, cudaStream_t st);
int launch_survival_decide(const uint8_t* status, const uint8_t* kf_member, int B, int P,
                           int32_t* counts, float T, int32_t* flag, int64_t* totals,
                           int64_t* kf_count, unsigned long long cond, unsigned* done,
                           cudaStream_t st);
int launch_ring_tables(const int64_t* table, int R, int C, int64_t* counter, int64_t* cur,
                       int64_t* prev, cudaStream_t st);
int launch_refill(const float* kp_xy, const int32_t* cell_count, int cells, int k,
                  const int32_t* flag, int B, int P, float* tracks, uint8_t* status,
                  uint8_t* kf_member, int32_t* track_id, int32_t* next_id, cudaStream_t st);

}  // namespace v2d
