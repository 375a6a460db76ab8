// pyramid.cu — K1: one-pass box pyramid.
//
// Operation ("each image pyramid level"; reading #1 = SPEC S:149
// 2x2 box filter, floor halving): I_L(x,y) = 1/4 sum I_{L-1}(2x+i, 2y+j).
// Nested floors make I_L(x,y) the exact mean of the aligned 2^L x 2^L block of
// L0, so every level is produced from integer block sums in ONE read of the u8
// frame: level 1 from registers, levels >= 2 from shared-memory partial sums.
// Sums are exact integers and sum * 4^-L is exact in fp32 (<= 8+2L <= 24
// significant bits), so the output is bit-identical to the recursive
// definition in any order.
//
// B200 mapping: HBM-bound (1 B/px read, 4 B per level pixel written,
// ~2.33 B per L0 px).  One CTA per 256x64 L0 tile (256x128 when the top level
// is 7), grid.z = image; per item two 16-byte row loads, all of a thread's items
// loaded before any is consumed (64 B in flight per thread), two float4
// coalesced stores of level 1 per item.
#include "common.cuh"

namespace v2d {
namespace {

constexpr int kThreads = 256;

__device__ __forceinline__ int bsum2(uint32_t w, int i) {  // bytes 2i and 2i+1 of w
  return (int)((w >> (16 * i)) & 0xffu) + (int)((w >> (16 * i + 8)) & 0xffu);
}

template <int TW, int TH>
__global__ void __launch_bounds__(kThreads)
pyramid_kernel(const uint8_t* const* __restrict__ l0_ptrs, int64_t l0_pitch, int W, int H,
               Levels lv, float* const* __restrict__ pyr_ptrs) {
  // TW x TH L0 tile (TH a power of two >= 2^(levels-1), TW a multiple of TH): level 1 from
  // 16-byte row loads (two rows per item -> 8 level-1 pixels, two float4 stores),
  // levels >= 2 from exact block sums in shared memory.
  constexpr int W1 = TW / 2, H1 = TH / 2;  // level-1 tile
  constexpr int Q = TW / 16;               // 16-byte column groups per tile row
  __shared__ int sa[H1 * W1];
  __shared__ int sb[(H1 / 2) * (W1 / 2)];

  const int b = blockIdx.z;
  const uint8_t* __restrict__ src = l0_ptrs[b];
  float* __restrict__ dst = pyr_ptrs[b];
  const int tx0 = blockIdx.x * TW, ty0 = blockIdx.y * TH;
  const bool aligned16 = (reinterpret_cast<uintptr_t>(src) & 15u) == 0;
  const bool dst16 = (reinterpret_cast<uintptr_t>(dst) & 15u) == 0;

  // ---- level 1: each item = 8 level-1 pixels from a 16x2 L0 patch ------
  {
    const int Wl1 = lv.W[1], Hl1 = lv.H[1];
    float* __restrict__ o1 = dst + lv.offset[1];
    const int64_t p1 = lv.pitch[1];
    // all of this thread's 16-byte row loads are issued before any is consumed
    constexpr int kItems = (H1 * Q + kThreads - 1) / kThreads;
    uint4 pre0[kItems], pre1[kItems];
#pragma unroll
    for (int k = 0; k < kItems; ++k) {
      const int it = threadIdx.x + k * kThreads;
      const int j = it / Q, q = it % Q;
      const int gy = ty0 + 2 * j, gx = tx0 + 16 * q;
      pre0[k] = make_uint4(0u, 0u, 0u, 0u);
      pre1[k] = pre0[k];
      if (it < H1 * Q && aligned16 && gx < l0_pitch) {
        const uint8_t* p = src + (int64_t)gy * l0_pitch + gx;
        if (gy < H) pre0[k] = __ldg(reinterpret_cast<const uint4*>(p));
        if (gy + 1 < H) pre1[k] = __ldg(reinterpret_cast<const uint4*>(p + l0_pitch));
      }
    }
#pragma unroll
    for (int k = 0; k < kItems; ++k) {
      const int it = threadIdx.x + k * kThreads;
      if (it >= H1 * Q) break;
      const int j = it / Q, q = it % Q;
      const int gy = ty0 + 2 * j, gx = tx0 + 16 * q;
      uint4 r0 = pre0[k], r1 = pre1[k];
      if (gx < l0_pitch) {  // l0_pitch % 16 == 0: the 16 bytes stay inside the row
        const uint8_t* p = src + (int64_t)gy * l0_pitch + gx;
        if (aligned16) {
        } else {
          uint32_t w[8] = {0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u};
          for (int i = 0; i < 16; ++i) {
            if (gy < H) w[i >> 2] |= (uint32_t)p[i] << (8 * (i & 3));
            if (gy + 1 < H) w[4 + (i >> 2)] |= (uint32_t)p[l0_pitch + i] << (8 * (i & 3));
          }
          r0 = make_uint4(w[0], w[1], w[2], w[3]);
          r1 = make_uint4(w[4], w[5], w[6], w[7]);
        }
      }
      const uint32_t a0[4] = {r0.x, r0.y, r0.z, r0.w}, a1[4] = {r1.x, r1.y, r1.z, r1.w};
      int s[8];
#pragma unroll
      for (int w = 0; w < 4; ++w) {
        s[2 * w] = bsum2(a0[w], 0) + bsum2(a1[w], 0);
        s[2 * w + 1] = bsum2(a0[w], 1) + bsum2(a1[w], 1);
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) sa[j * W1 + 8 * q + i] = s[i];
      const int oy = (ty0 >> 1) + j, ox = (tx0 >> 1) + 8 * q;
      if (oy < Hl1) {
        float* row = o1 + (int64_t)oy * p1;
        if (dst16 && ox + 7 < Wl1) {
          *reinterpret_cast<float4*>(row + ox) =
              make_float4(0.25f * s[0], 0.25f * s[1], 0.25f * s[2], 0.25f * s[3]);
          *reinterpret_cast<float4*>(row + ox + 4) =
              make_float4(0.25f * s[4], 0.25f * s[5], 0.25f * s[6], 0.25f * s[7]);
        } else {
#pragma unroll
          for (int i = 0; i < 8; ++i)
            if (ox + i < Wl1) row[ox + i] = 0.25f * s[i];
        }
      }
    }
  }
  // ---- levels >= 2 from the exact block sums in shared memory ------------
  int* prev = sa;
  int* cur = sb;
  int ew = W1, eh = H1;
  float scale = 0.25f;
  for (int L = 2; L < lv.n; ++L) {
    __syncthreads();
    const int nw = ew >> 1, nh = eh >> 1;
    scale *= 0.25f;
    const int WL = lv.W[L], HL = lv.H[L];
    float* __restrict__ oL = dst + lv.offset[L];
    const int64_t pL = lv.pitch[L];
    for (int it = threadIdx.x; it < nw * nh; it += kThreads) {
      const int j = it / nw, i = it % nw;
      const int s = prev[(2 * j) * ew + 2 * i] + prev[(2 * j) * ew + 2 * i + 1] +
                    prev[(2 * j + 1) * ew + 2 * i] + prev[(2 * j + 1) * ew + 2 * i + 1];
      cur[j * nw + i] = s;
      const int oy = (ty0 >> L) + j, ox = (tx0 >> L) + i;
      if (oy < HL && ox < WL) oL[(int64_t)oy * pL + ox] = scale * (float)s;
    }
    int* t = prev;
    prev = cur;
    cur = t;
    ew = nw;
    eh = nh;
  }
}

}  // namespace

int launch_pyramid(const uint8_t* const* l0_ptrs, int64_t l0_pitch, int B, int W, int H,
                   const Levels& lv, float* const* pyr_ptrs, cudaStream_t st) {
  if (lv.n <= 1 || B == 0) return V2D_OK;
  if (lv.n <= 7) {
    // 256 x 64 tiles, two items per thread with all four 16-byte loads in flight
    // (same-box A/B at c5: 38.4 -> 37.2 us vs 128 x 64 with one item per thread)
    constexpr int TW = 256, TH = 64;
    dim3 grid((W + TW - 1) / TW, (H + TH - 1) / TH, B);
    pyramid_kernel<TW, TH><<<grid, kThreads, 0, st>>>(l0_ptrs, l0_pitch, W, H, lv, pyr_ptrs);
  } else {
    constexpr int TW = 256, TH = 128;
    dim3 grid((W + TW - 1) / TW, (H + TH - 1) / TH, B);
    pyramid_kernel<TW, TH><<<grid, kThreads, 0, st>>>(l0_ptrs, l0_pitch, W, H, lv, pyr_ptrs);
  }
  return cudaGetLastError() == cudaSuccess ? V2D_OK : V2D_ECUDA;
}

}  // namespace v2d
