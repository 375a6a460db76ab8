// patches.cu — variant f4: per-level patch features for loop closure
// ("a list of 9x9 image patches taken from each level of the
// image pyramid").
//
// out[b][p][L][v][u] = S(I_L, c_L + (u - r, v - r)),  c_L = (p + 0.5)/2^L - 0.5,
// bilinear with clamp-to-edge (D2), r = (patch-1)/2.
//
// B200 mapping: a gather on the resident pyramid — one warp per keypoint.
// Every sample of one level shares the fractional offset of c_L, so a level's
// patch is a fixed-weight bilinear of one (patch+1)^2 block of pixels.  The warp
// first issues the loads of the blocks of ALL levels (up to kBudget pixels at a
// time: 5 levels x 10 x 10 for 9x9 patches), independent clamped loads with
// the whole batch in flight (the kernel is latency-bound: one level at a time
// left ~4 dependent load rounds per level per warp), into shared memory; then
// lanes form every sample of those levels with the same expression order as D2
// and store the contiguous [levels][patch][patch] block coalesced.
#include "common.cuh"

namespace v2d {
namespace {

constexpr int kWarps = 8;
#ifndef V2D_PATCH_BUDGET
#define V2D_PATCH_BUDGET 512  // 9x9 x 5 levels still one batch; 16 KB per CTA
#endif
#ifndef V2D_PATCH_MINB
#define V2D_PATCH_MINB 8  // 64 warps per SM (32 registers): -7 % at c5 (same-box A/B)
#endif
constexpr int kBudget = V2D_PATCH_BUDGET;  // staged pixels per warp (2 KB of shared memory)

template <int PATCH>  // compile-time patch edge
__global__ void __launch_bounds__(32 * kWarps, V2D_PATCH_MINB)
patches_kernel(const uint8_t* const* __restrict__ l0_ptrs, const float* const* __restrict__ pyr_ptrs,
               int64_t l0_pitch, int B, Levels lv, const float* __restrict__ pts, int P,
               float* __restrict__ out) {
  constexpr int patch = PATCH;
  constexpr int n = patch * patch, r = (patch - 1) / 2, e = patch + 1, EE = e * e;
  // levels staged at once (<= the 8 a pyramid can have)
  constexpr int kPerBatch = kBudget / EE < 1 ? 1 : (kBudget / EE > V2D_MAX_LEVELS ? V2D_MAX_LEVELS
                                                                                   : kBudget / EE);
  constexpr int kLd = (EE + 31) / 32, kSm = (n + 31) / 32;         // per lane and level
  __shared__ float s_blk[kWarps][kPerBatch * EE];
  const int64_t kp = (int64_t)blockIdx.x * kWarps + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (kp >= (int64_t)B * P) return;  // warp-uniform
  float* blk = s_blk[threadIdx.x >> 5];
  const int b = (int)(kp / P);
  const float px0 = pts[2 * kp], py0 = pts[2 * kp + 1];
  const bool empty = (px0 == -1.0f && py0 == -1.0f) || !isfinite(px0) || !isfinite(py0);
  float* o = out + kp * (int64_t)lv.n * n;
  if (empty) {
    for (int i = lane; i < lv.n * n; i += 32) o[i] = 0.0f;
    return;
  }
  // this lane's block elements (row, col) and sample positions (v, u): the same at
  // every level, so all index arithmetic is done once
  int br[kLd], bc[kLd], sv[kSm], su[kSm];
#pragma unroll
  for (int m = 0; m < kLd; ++m) {
    const int j = min(lane + 32 * m, EE - 1);
    br[m] = j / e;
    bc[m] = j - br[m] * e;
  }
#pragma unroll
  for (int m = 0; m < kSm; ++m) {
    const int i = min(lane + 32 * m, n - 1);
    sv[m] = i / patch;
    su[m] = i - sv[m] * patch;
  }
  const uint8_t* l0 = l0_ptrs[b];
  const float* pyr = lv.n > 1 ? pyr_ptrs[b] : nullptr;
  for (int L0 = 0; L0 < lv.n; L0 += kPerBatch) {
    const int nb = min(kPerBatch, lv.n - L0);
    __syncwarp();
    // ---- stage the (patch+1)^2 blocks of levels L0 .. L0+nb-1 (clamp-to-edge);
    // every load of the batch is independent, so all of them are in flight
    // (32-bit element offsets: a level plane or frame is < 2^31 elements)
#pragma unroll
    for (int q = 0; q < kPerBatch; ++q) {
      if (q >= nb) break;
      const int L = L0 + q;
      const float scale = __int_as_float((127 - L) << 23);  // 2^-L
      const float cx = (px0 + 0.5f) * scale - 0.5f, cy = (py0 + 0.5f) * scale - 0.5f;
      const int bx = (int)floorf(cx) - r, by = (int)floorf(cy) - r;  // block origin
      const int Wl = lv.W[L] - 1, Hl = lv.H[L] - 1;
      float* dst = blk + q * EE;
      if (L == 0) {
        const int pitch = (int)l0_pitch;
#pragma unroll
        for (int m = 0; m < kLd; ++m) {
          const int x = min(max(bx + bc[m], 0), Wl), y = min(max(by + br[m], 0), Hl);
          const float v = (float)__ldg(l0 + (unsigned)(y * pitch + x));
          if (lane + 32 * m < EE) dst[lane + 32 * m] = v;
        }
      } else {
        const float* pl = pyr + lv.offset[L];
        const int pitch = (int)lv.pitch[L];
#pragma unroll
        for (int m = 0; m < kLd; ++m) {
          const int x = min(max(bx + bc[m], 0), Wl), y = min(max(by + br[m], 0), Hl);
          const float v = __ldg(pl + (unsigned)(y * pitch + x));
          if (lane + 32 * m < EE) dst[lane + 32 * m] = v;
        }
      }
    }
    __syncwarp();
    // ---- samples of those levels, stored contiguously ([L][v][u])
    float* oL0 = o + L0 * n + lane;
#pragma unroll
    for (int q = 0; q < kPerBatch; ++q) {
      if (q >= nb) break;
      const int L = L0 + q;
      const float scale = __int_as_float((127 - L) << 23);
      const float cx = (px0 + 0.5f) * scale - 0.5f, cy = (py0 + 0.5f) * scale - 0.5f;
      const float wa = cx - floorf(cx), wb = cy - floorf(cy);
      const float* src = blk + q * EE;
      float* oL = oL0 + q * n - lane;
#pragma unroll
      for (int m = 0; m < kSm; ++m) {
        const float* t = src + sv[m] * e + su[m];
        const float top = fmaf(wa, t[1] - t[0], t[0]);
        const float bot = fmaf(wa, t[e + 1] - t[e], t[e]);
        if (lane + 32 * m < n) oL[lane + 32 * m] = fmaf(wb, bot - top, top);
      }
    }
  }
}

}  // namespace

int launch_patches(const uint8_t* const* l0_ptrs, const float* const* pyr_ptrs, int64_t l0_pitch,
                   int B, const Levels& lv, const float* pts, int P, int patch, float* out,
                   cudaStream_t st) {
  const int64_t n = (int64_t)B * P;
  if (n == 0) return V2D_OK;
  const unsigned grid = (unsigned)((n + kWarps - 1) / kWarps);
#define V2D_PATCH_CASE(p)                                                                  \
  case p:                                                                                  \
    patches_kernel<p><<<grid, 32 * kWarps, 0, st>>>(l0_ptrs, pyr_ptrs, l0_pitch, B, lv, pts, P, \
                                                    out);                                  \
    break;
  switch (patch) {
    V2D_PATCH_CASE(1) V2D_PATCH_CASE(3) V2D_PATCH_CASE(5) V2D_PATCH_CASE(7) V2D_PATCH_CASE(9)
    V2D_PATCH_CASE(11) V2D_PATCH_CASE(13) V2D_PATCH_CASE(15) V2D_PATCH_CASE(17)
    V2D_PATCH_CASE(19) V2D_PATCH_CASE(21) V2D_PATCH_CASE(23) V2D_PATCH_CASE(25)
    V2D_PATCH_CASE(27) V2D_PATCH_CASE(29) V2D_PATCH_CASE(31)
    default:
      return V2D_EINVAL;
  }
#undef V2D_PATCH_CASE
  return cudaGetLastError() == cudaSuccess ? V2D_OK : V2D_ECUDA;
}

}  // namespace v2d
