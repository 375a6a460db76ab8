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
// ~2.33 B per L0 px).  One CTA per 64x64 L0 tile (128x128 when the top level
// is 7), grid.z = image; 8-byte vector loads of two rows per thread, float4
// coalesced stores of level 1 (128-B level rows).
#include "common.cuh"

namespace v2d {
namespace {

constexpr int kThreads = 256;

__device__ __forceinline__ int bsum2(uint32_t w, int i) {  // bytes 2i and 2i+1 of w
  return (int)((w >> (16 * i)) & 0xffu) + (int)((w >> (16 * i + 8)) & 0xffu);
}

template <int TILE>
__global__ void __launch_bounds__(kThreads)
pyramid_kernel(const uint8_t* const* __restrict__ l0_ptrs, int64_t l0_pitch, int W, int H,
               Levels lv, float* const* __restrict__ pyr_ptrs) {
  constexpr int T1 = TILE / 2;  // level-1 tile edge
  constexpr int Q = TILE / 8;   // 8-byte column groups per tile row
  __shared__ int sa[T1 * T1];
  __shared__ int sb[(T1 / 2) * (T1 / 2)];

  const int b = blockIdx.z;
  const uint8_t* __restrict__ src = l0_ptrs[b];
  float* __restrict__ dst = pyr_ptrs[b];
  const int tx0 = blockIdx.x * TILE, ty0 = blockIdx.y * TILE;
  const bool aligned8 = (reinterpret_cast<uintptr_t>(src) & 7u) == 0;
  const bool dst16 = (reinterpret_cast<uintptr_t>(dst) & 15u) == 0;

  // ---- level 1: each item = 4 level-1 pixels from an 8x2 L0 patch -------
  {
    const int W1 = lv.W[1], H1 = lv.H[1];
    float* __restrict__ o1 = dst + lv.offset[1];
    const int64_t p1 = lv.pitch[1];
    for (int it = threadIdx.x; it < T1 * Q; it += kThreads) {
      const int j = it / Q, q = it % Q;
      const int gy = ty0 + 2 * j, gx = tx0 + 8 * q;
      uint2 r0 = make_uint2(0u, 0u), r1 = make_uint2(0u, 0u);
      if (gx < l0_pitch) {  // l0_pitch % 16 == 0: the 8 bytes stay inside the row
        const uint8_t* p = src + (int64_t)gy * l0_pitch + gx;
        if (aligned8) {
          if (gy < H) r0 = __ldg(reinterpret_cast<const uint2*>(p));
          if (gy + 1 < H) r1 = __ldg(reinterpret_cast<const uint2*>(p + l0_pitch));
        } else {
          uint32_t w[4] = {0u, 0u, 0u, 0u};
          for (int i = 0; i < 8; ++i) {
            if (gy < H) w[i >> 2] |= (uint32_t)p[i] << (8 * (i & 3));
            if (gy + 1 < H) w[2 + (i >> 2)] |= (uint32_t)p[l0_pitch + i] << (8 * (i & 3));
          }
          r0 = make_uint2(w[0], w[1]);
          r1 = make_uint2(w[2], w[3]);
        }
      }
      int s[4];
      s[0] = bsum2(r0.x, 0) + bsum2(r1.x, 0);
      s[1] = bsum2(r0.x, 1) + bsum2(r1.x, 1);
      s[2] = bsum2(r0.y, 0) + bsum2(r1.y, 0);
      s[3] = bsum2(r0.y, 1) + bsum2(r1.y, 1);
#pragma unroll
      for (int i = 0; i < 4; ++i) sa[j * T1 + 4 * q + i] = s[i];
      const int oy = (ty0 >> 1) + j, ox = (tx0 >> 1) + 4 * q;
      if (oy < H1) {
        float* row = o1 + (int64_t)oy * p1;
        if (dst16 && ox + 3 < W1) {
          *reinterpret_cast<float4*>(row + ox) =
              make_float4(0.25f * s[0], 0.25f * s[1], 0.25f * s[2], 0.25f * s[3]);
        } else {
#pragma unroll
          for (int i = 0; i < 4; ++i)
            if (ox + i < W1) row[ox + i] = 0.25f * s[i];
        }
      }
    }
  }
  // ---- levels >= 2 from the exact block sums in shared memory ------------
  int* prev = sa;
  int* cur = sb;
  int edge = T1;
  float scale = 0.25f;
  for (int L = 2; L < lv.n; ++L) {
    __syncthreads();
    const int e = edge >> 1;
    scale *= 0.25f;
    const int WL = lv.W[L], HL = lv.H[L];
    float* __restrict__ oL = dst + lv.offset[L];
    const int64_t pL = lv.pitch[L];
    for (int it = threadIdx.x; it < e * e; it += kThreads) {
      const int j = it / e, i = it % e;
      const int s = prev[(2 * j) * edge + 2 * i] + prev[(2 * j) * edge + 2 * i + 1] +
                    prev[(2 * j + 1) * edge + 2 * i] + prev[(2 * j + 1) * edge + 2 * i + 1];
      cur[j * e + i] = s;
      const int oy = (ty0 >> L) + j, ox = (tx0 >> L) + i;
      if (oy < HL && ox < WL) oL[(int64_t)oy * pL + ox] = scale * (float)s;
    }
    int* t = prev;
    prev = cur;
    cur = t;
    edge = e;
  }
}

}  // namespace

int launch_pyramid(const uint8_t* const* l0_ptrs, int64_t l0_pitch, int B, int W, int H,
                   const Levels& lv, float* const* pyr_ptrs, cudaStream_t st) {
  if (lv.n <= 1 || B == 0) return V2D_OK;
  if (lv.n <= 7) {
    constexpr int T = 64;
    dim3 grid((W + T - 1) / T, (H + T - 1) / T, B);
    pyramid_kernel<T><<<grid, kThreads, 0, st>>>(l0_ptrs, l0_pitch, W, H, lv, pyr_ptrs);
  } else {
    constexpr int T = 128;
    dim3 grid((W + T - 1) / T, (H + T - 1) / T, B);
    pyramid_kernel<T><<<grid, kThreads, 0, st>>>(l0_ptrs, l0_pitch, W, H, lv, pyr_ptrs);
  }
  return cudaGetLastError() == cudaSuccess ? V2D_OK : V2D_ECUDA;
}

}  // namespace v2d
