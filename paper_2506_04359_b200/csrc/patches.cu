// patches.cu — variant f4: per-level patch features for loop closure
// ("a list of 9x9 image patches taken from each level of the
// image pyramid").
//
// out[b][p][L][v][u] = S(I_L, c_L + (u - r, v - r)),  c_L = (p + 0.5)/2^L - 0.5,
// bilinear with clamp-to-edge (D2), r = (patch-1)/2.
//
// B200 mapping: a gather on the resident pyramid — one warp per keypoint, lanes
// over the patch x patch samples of each level, corners read through L1/L2
// (the levels of the frame just built are L2-resident), coalesced stores of the
// contiguous [levels][patch][patch] block.  Memory/latency-bound and tiny next
// to K3; no shared memory.
#include "common.cuh"

namespace v2d {
namespace {

constexpr int kWarps = 8;

template <typename T>
__device__ __forceinline__ float px(const T* base, int64_t pitch, int W, int H, int x, int y) {
  x = min(max(x, 0), W - 1);
  y = min(max(y, 0), H - 1);
  return (float)__ldg(base + (int64_t)y * pitch + x);
}

template <typename T>
__device__ __forceinline__ float bilinear(const T* base, int64_t pitch, int W, int H, float x,
                                          float y) {
  const float fx = floorf(x), fy = floorf(y);
  const float a = x - fx, b = y - fy;
  const int x0 = (int)fx, y0 = (int)fy;
  const float top = fmaf(a, px(base, pitch, W, H, x0 + 1, y0) - px(base, pitch, W, H, x0, y0),
                         px(base, pitch, W, H, x0, y0));
  const float bot = fmaf(a, px(base, pitch, W, H, x0 + 1, y0 + 1) -
                                px(base, pitch, W, H, x0, y0 + 1),
                         px(base, pitch, W, H, x0, y0 + 1));
  return fmaf(b, bot - top, top);
}

__global__ void __launch_bounds__(32 * kWarps)
patches_kernel(const uint8_t* const* __restrict__ l0_ptrs, const float* const* __restrict__ pyr_ptrs,
               int64_t l0_pitch, int B, Levels lv, const float* __restrict__ pts, int P, int patch,
               float* __restrict__ out) {
  const int64_t kp = (int64_t)blockIdx.x * kWarps + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (kp >= (int64_t)B * P) return;
  const int b = (int)(kp / P);
  const float px0 = pts[2 * kp], py0 = pts[2 * kp + 1];
  const bool empty = (px0 == -1.0f && py0 == -1.0f) || !isfinite(px0) || !isfinite(py0);
  const int n = patch * patch, r = (patch - 1) / 2;
  float* o = out + kp * (int64_t)lv.n * n;
  for (int L = 0; L < lv.n; ++L) {
    const float scale = __int_as_float((127 - L) << 23);  // 2^-L
    const float cx = (px0 + 0.5f) * scale - 0.5f, cy = (py0 + 0.5f) * scale - 0.5f;
    for (int i = lane; i < n; i += 32) {
      const int v = i / patch, u = i - v * patch;
      float val = 0.0f;
      if (!empty) {
        const float x = cx + (float)(u - r), y = cy + (float)(v - r);
        val = L == 0 ? bilinear(l0_ptrs[b], l0_pitch, lv.W[0], lv.H[0], x, y)
                     : bilinear(pyr_ptrs[b] + lv.offset[L], lv.pitch[L], lv.W[L], lv.H[L], x, y);
      }
      o[L * n + i] = val;
    }
  }
}

}  // namespace

int launch_patches(const uint8_t* const* l0_ptrs, const float* const* pyr_ptrs, int64_t l0_pitch,
                   int B, const Levels& lv, const float* pts, int P, int patch, float* out,
                   cudaStream_t st) {
  const int64_t n = (int64_t)B * P;
  if (n == 0) return V2D_OK;
  patches_kernel<<<(unsigned)((n + kWarps - 1) / kWarps), 32 * kWarps, 0, st>>>(
      l0_ptrs, pyr_ptrs, l0_pitch, B, lv, pts, P, patch, out);
  return cudaGetLastError() == cudaSuccess ? V2D_OK : V2D_ECUDA;
}

}  // namespace v2d
