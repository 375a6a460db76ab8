// gftt.cu — K2: fused Sobel -> structure tensor -> lambda_min -> NMS -> per-cell top-k
// (SURVEY §8(a) rows a3-a5).
//
// Operation ("the image is first divided into non-overlapping
// patches, forming an N x M grid.  In each patch, the algorithm selects the top
// k keypoints based on the 'Good Features to Track' measure", Eq. 1 for k;
// readings #4-#9 of DESIGN.md):
//   sx, sy   = integer 3x3 Sobel of the u8 frame (= 8 Gx, 8 Gy)
//   A',B',C' = 3x3 box sums of sx^2, sx*sy, sy^2            (exact int32, < 2^24)
//   R        = [f32(det) / ((f32(tr) + sqrt(f32(D))) * 0.5)] * 2^-6
//              det = A'C'-B'^2, D = (A'-C')^2 + 4B'^2 exact in int64, every fp32
//              op correctly rounded, no contraction (__*_rn intrinsics)
//   key      = bits(R) << 32 | (0xFFFFFFFF - (y*W + x))      (score, then index)
//   candidate: border <= x,y <= dim-1-border, R > min_score, key > all 8
//              neighbours' keys (nms = 1)
//   output   : per cell the k largest candidate keys, descending.
//
// B200 mapping (DESIGN.md §5 K2): one CTA (8 warps) per (cell, image).  The cell
// is cut into items of 26 output columns x up to 32 rows; a warp owns an item
// and streams its 32 input columns (3-px halo each side) down the rows with
// every stage in registers: lane = column, horizontal neighbours by shuffle,
// vertical windows as rolling registers — no shared-memory staging, no index
// division.  R rows go to a 3-row per-warp ring in shared memory for the NMS
// of the (few) lanes that beat the warp's running threshold; those append to a
// per-warp key buffer that a warp-level bitonic sort folds back to its top k.
// The threshold also gates the lazy eigenvalue: lambda_min <= min(A',C')/64, so
// R is only evaluated where that bound can beat the k-th best key (exact: such
// pixels can neither be selected nor beat a selectable neighbour).  At the end
// the CTA merges the 8 warps' top-k lists with one block bitonic sort.
// Deterministic, no global atomics.
#include "common.cuh"

namespace v2d {
namespace {

constexpr int kWarps = 4;
constexpr int kThreads = 32 * kWarps;
constexpr int kPix = 4;             // adjacent columns per lane (one 32-bit load per row)
constexpr int kSpan = 32 * kPix;    // columns per warp strip (128)
constexpr int kOut = kSpan - 8;     // output columns per strip (120): halo 3 left, 5 right
constexpr int kWBuf = 512;          // per-warp key buffer (top-k + fresh candidates)
constexpr int kRing = kSpan + 8;    // R ring row (4 pad floats each side)

__device__ __forceinline__ float response_contract(int A, int Bv, int C, long long det) {
  const int tr = A + C;
  if (tr == 0) return 0.0f;
  const long long dAC = (long long)(A - C);
  const long long D = dAC * dAC + 4ll * (long long)Bv * Bv;
  const float f_det = __ll2float_rn(det);
  const float f_tr = __int2float_rn(tr);
  const float f_sq = __fsqrt_rn(__ll2float_rn(D));
  const float lmax = __fmul_rn(__fadd_rn(f_tr, f_sq), 0.5f);
  return __fmul_rn(__fdiv_rn(f_det, lmax), 0.015625f);
}

__device__ __forceinline__ unsigned long long make_key(float r, int x, int y, int W) {
  const unsigned idx = (unsigned)y * (unsigned)W + (unsigned)x;
  return ((unsigned long long)__float_as_uint(r) << 32) | (unsigned long long)(0xffffffffu - idx);
}

// Descending bitonic sort of buf[0..n), padded with zeros to a power of two, by
// nthr threads (tid = index within the group); warp or block scope.
template <bool kBlock>
__device__ __forceinline__ void bitonic_desc(unsigned long long* buf, int n, int tid, int nthr) {
  int N = 2;
  while (N < n) N <<= 1;
  for (int i = n + tid; i < N; i += nthr) buf[i] = 0ull;
  if (kBlock) __syncthreads(); else __syncwarp();
  for (int size = 2; size <= N; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = tid; i < (N >> 1); i += nthr) {
        const int lo = 2 * i - (i & (stride - 1));
        const int hi = lo + stride;
        const bool desc = (lo & size) == 0;
        const unsigned long long a = buf[lo], c = buf[hi];
        if ((a < c) == desc) {
          buf[lo] = c;
          buf[hi] = a;
        }
      }
      if (kBlock) __syncthreads(); else __syncwarp();
    }
  }
}

// Smallest integer m with (float)m * (2^-6 * (1 + 1e-5)) >= s: pixels whose
// min(A', C') < m have lambda_min bound below the score s (lazy eigenvalue).
__device__ __forceinline__ int lazy_int_threshold(float s) {
  if (!(s > 0.0f)) return 0;
  const float m = s * (64.0f / 1.00001f);
  if (m >= 2.0e9f) return 0x7fffffff;
  return max(0, (int)m - 2);  // conservative by 2 units (fp rounding of the product)
}

__global__ void __launch_bounds__(kThreads)
gftt_topk_kernel(const uint8_t* const* __restrict__ l0_ptrs, GfttArgs a,
                 float* __restrict__ kp_xy, float* __restrict__ kp_score,
                 int32_t* __restrict__ cell_count, float* __restrict__ resp,
                 const uint8_t* const* __restrict__ mask_ptrs,
                 const int32_t* __restrict__ enable) {
  if (enable && enable[0] == 0) return;  // keyframe-conditional detection (f1)
  __shared__ unsigned long long s_buf[kWarps * kWBuf];
  __shared__ __align__(16) float s_ring[kWarps][3][kRing];
  __shared__ int s_cnt[kWarps][2];  // [0] = kept (top), [1] = fresh candidates
  __shared__ int s_total;
  __shared__ unsigned long long s_thr;  // max over warps of their k-th best key
  __shared__ int4 s_q[kWarps][kSpan];    // per-warp queue of pixels needing the exact R

  const int W = a.W, H = a.H, k = a.k;
  const int cell = blockIdx.x, b = blockIdx.y;
  const int cx = cell % a.grid_x, cy = cell / a.grid_x;
  const uint8_t* __restrict__ img = l0_ptrs[b];
  const uint8_t* __restrict__ mask = mask_ptrs ? mask_ptrs[b] : nullptr;
  const int64_t pitch = a.pitch;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  // D6 cell: [floor(cx*W/gx), floor((cx+1)*W/gx)) x [...]
  const int x0 = (int)((int64_t)cx * W / a.grid_x), x1 = (int)((int64_t)(cx + 1) * W / a.grid_x);
  const int y0 = (int)((int64_t)cy * H / a.grid_y), y1 = (int)((int64_t)(cy + 1) * H / a.grid_y);
  // D5 eligibility box
  const int ex0 = a.border, ex1 = W - a.border, ey0 = a.border, ey1 = H - a.border;
  const bool full = resp != nullptr;  // need R everywhere in the cell
  const int rx0 = full ? x0 : max(x0, ex0), rx1 = full ? x1 : min(x1, ex1);
  const int ry0 = full ? y0 : max(y0, ey0), ry1 = full ? y1 : min(y1, ey1);
  const bool lazy = !full;

  unsigned long long* wbuf = s_buf + warp * kWBuf;
  float (*ring)[kRing] = s_ring[warp];
  if (lane == 0) {
    s_cnt[warp][0] = 0;
    s_cnt[warp][1] = 0;
  }
  if (threadIdx.x == 0) s_thr = 0ull;
  for (int i = lane; i < 3 * kRing; i += 32) (&ring[0][0])[i] = 0.0f;
  __syncthreads();

  // strips of kOut output columns starting 4-aligned (xs = first loaded column)
  const int xs0 = ((rx0 - 3) >> 2) << 2;  // floor to a multiple of 4
  const int nxs = rx1 > rx0 ? (rx1 - (xs0 + 3) + kOut - 1) / kOut : 0;
  // row chunks: aim for >= kWarps items per cell, >= 8 rows per chunk
  const int rows = ry1 - ry0;
  int nys = rows > 0 ? max(1, (kWarps + nxs - 1) / max(nxs, 1)) : 0;
  nys = min(nys, max(1, rows / 8));
  const int chunk = nys > 0 ? (rows + nys - 1) / nys : 0;
  const int items = nxs * nys;
  const int fold_at = max(64, 2 * k);

  for (int item = warp; item < items; item += kWarps) {
    const int sy_ = item / nxs, sx_ = item - sy_ * nxs;
    const int xs = xs0 + sx_ * kOut;
    const int oy = ry0 + sy_ * chunk;
    const int oy_end = min(oy + chunk, ry1);
    const int xl = xs + kPix * lane;      // this lane's first column
    const bool load_ok = xl >= 0 && xl < pitch;  // 4-aligned word inside the row
    const uint8_t* __restrict__ colp = img + (load_ok ? xl : 0);
    const int ipitch = (int)pitch;  // W*H < 2^31 is validated by the ABI

    int i0[kPix] = {0, 0, 0, 0}, i1[kPix] = {0, 0, 0, 0};  // I rows L-2, L-1
    int hs0[kPix] = {0, 0, 0, 0}, hs1[kPix] = {0, 0, 0, 0};  // [1 2 1]_x rows L-2, L-1
    int a0[kPix] = {0, 0, 0, 0}, a1[kPix] = {0, 0, 0, 0};
    int b0[kPix] = {0, 0, 0, 0}, b1[kPix] = {0, 0, 0, 0};
    int c0[kPix] = {0, 0, 0, 0}, c1[kPix] = {0, 0, 0, 0};
    int ridx = 0;
    auto ld_row = [&](int L) -> unsigned {
      const int yc = min(max(L, 0), H - 1);
      return load_ok ? __ldg(reinterpret_cast<const unsigned*>(colp + (unsigned)(yc * ipitch))) : 0u;
    };
    // software pipeline: rows L+1 and L+2 are in flight while row L is processed
    unsigned w_n1 = ld_row(oy - 3), w_n2 = ld_row(oy - 2);
    for (int L = oy - 3; L <= oy_end + 2; ++L) {
      const unsigned w = w_n1;
      w_n1 = w_n2;
      w_n2 = ld_row(L + 2);
      const unsigned wl = __shfl_up_sync(kFullMask, w, 1);
      const unsigned wr = __shfl_down_sync(kFullMask, w, 1);
      int I[kPix + 2];
      I[0] = (int)(wl >> 24);
#pragma unroll
      for (int j = 0; j < kPix; ++j) I[j + 1] = (int)((w >> (8 * j)) & 0xffu);
      I[kPix + 1] = (int)(wr & 0xffu);
      int hs[kPix], V[kPix + 2];
#pragma unroll
      for (int j = 0; j < kPix; ++j) {
        hs[j] = I[j] + 2 * I[j + 1] + I[j + 2];
        V[j + 1] = i0[j] + 2 * i1[j] + I[j + 1];
      }
      V[0] = __shfl_up_sync(kFullMask, V[kPix], 1);
      V[kPix + 1] = __shfl_down_sync(kFullMask, V[1], 1);
      // Sobel at row L-1 and tensor products
      int pa[kPix + 2], pb[kPix + 2], pc[kPix + 2];
#pragma unroll
      for (int j = 0; j < kPix; ++j) {
        const int sx = V[j + 2] - V[j];
        const int sy = hs[j] - hs0[j];
        pa[j + 1] = sx * sx;
        pb[j + 1] = sx * sy;
        pc[j + 1] = sy * sy;
      }
      pa[0] = __shfl_up_sync(kFullMask, pa[kPix], 1);
      pb[0] = __shfl_up_sync(kFullMask, pb[kPix], 1);
      pc[0] = __shfl_up_sync(kFullMask, pc[kPix], 1);
      pa[kPix + 1] = __shfl_down_sync(kFullMask, pa[1], 1);
      pb[kPix + 1] = __shfl_down_sync(kFullMask, pb[1], 1);
      pc[kPix + 1] = __shfl_down_sync(kFullMask, pc[1], 1);
      // running threshold: any warp's k-th best key bounds the cell's k-th key
      // from below, so the largest one is a valid pruning threshold for all
      const int ntop = s_cnt[warp][0];
      const unsigned long long thr =
          lazy ? max(ntop == k ? wbuf[k - 1] : 0ull, *(volatile unsigned long long*)&s_thr) : 0ull;
      const float thr_score = __uint_as_float((unsigned)(thr >> 32));
      const int lz = lazy ? lazy_int_threshold(thr_score) : 0;
      const int yr = L - 2;  // tensor / response row
      const bool yr_ok = yr >= 2 && yr <= H - 3;
      int ha[kPix], hb[kPix], hc[kPix];
      int need_pos[kPix];
      int nq = 0;
      const unsigned lt_mask = (1u << lane) - 1u;
#pragma unroll
      for (int j = 0; j < kPix; ++j) {
        ha[j] = pa[j] + pa[j + 1] + pa[j + 2];
        hb[j] = pb[j] + pb[j + 1] + pb[j + 2];
        hc[j] = pc[j] + pc[j + 1] + pc[j + 2];
        const int A = a0[j] + a1[j] + ha[j];
        const int C = c0[j] + c1[j] + hc[j];
        const int Bv = b0[j] + b1[j] + hb[j];
        const int x = xl + j;
        bool need = yr_ok && x >= 2 && x <= W - 3 && min(A, C) >= lz;
        if (need && lazy) {
          // tighter exact bound lambda_min <= 2 det / tr (lambda_max >= tr/2)
          const long long det = (long long)A * C - (long long)Bv * Bv;
          need = __ll2float_rn(det) * (2.0f / 64.0f) >= thr_score * 0.99999f * __int2float_rn(A + C);
        }
        const unsigned msk = __ballot_sync(kFullMask, need);
        need_pos[j] = need ? nq + __popc(msk & lt_mask) : -1;
        nq += __popc(msk);
        if (need) s_q[warp][need_pos[j]] = make_int4(A, Bv, C, 4 + kPix * lane + j);
      }
      ridx = ridx == 2 ? 0 : ridx + 1;
      *reinterpret_cast<float4*>(&ring[ridx][4 + kPix * lane]) = make_float4(0.f, 0.f, 0.f, 0.f);
      __syncwarp();
      // exact fp32-contract response for the queued pixels, 32 at a time
      for (int q = lane; q < nq; q += 32) {
        const int4 e = s_q[warp][q];
        const long long det = (long long)e.x * e.z - (long long)e.y * e.y;
        ring[ridx][e.w] = response_contract(e.x, e.y, e.z, det);
      }
      __syncwarp();
      if (full && yr >= oy && yr < oy_end) {
#pragma unroll
        for (int j = 0; j < kPix; ++j) {
          const int x = xl + j;
          if (x >= xs + 3 && x < xs + 3 + kOut && x >= rx0 && x < rx1)
            resp[((int64_t)b * H + yr) * W + x] = ring[ridx][4 + kPix * lane + j];
        }
      }
      // NMS + threshold at row yn = L-3 (ring rows: ru = yn-1, rm = yn, rd = yn+1).
      // With R >= 0 the key order is: p beats the 4 neighbours BEFORE it in
      // row-major order iff R(p) > R(q), the 4 AFTER it iff R(p) >= R(q).
      const int yn = L - 3;
      if (yn >= oy && yn < oy_end && yn >= ey0 && yn < ey1) {
        const int rm = ridx == 0 ? 2 : ridx - 1;
        const int ru = rm == 0 ? 2 : rm - 1;
        float u[kPix + 2], m[kPix + 2], d[kPix + 2];
        {
          const int c = 4 + kPix * lane;
          const float4 u4 = *reinterpret_cast<const float4*>(&ring[ru][c]);
          const float4 m4 = *reinterpret_cast<const float4*>(&ring[rm][c]);
          const float4 d4 = *reinterpret_cast<const float4*>(&ring[ridx][c]);
          u[0] = ring[ru][c - 1]; m[0] = ring[rm][c - 1]; d[0] = ring[ridx][c - 1];
          u[1] = u4.x; u[2] = u4.y; u[3] = u4.z; u[4] = u4.w;
          m[1] = m4.x; m[2] = m4.y; m[3] = m4.z; m[4] = m4.w;
          d[1] = d4.x; d[2] = d4.y; d[3] = d4.z; d[4] = d4.w;
          u[5] = ring[ru][c + 4]; m[5] = ring[rm][c + 4]; d[5] = ring[ridx][c + 4];
        }
#pragma unroll
        for (int j = 0; j < kPix; ++j) {
          const float rp = m[j + 1];
          const int x = xl + j;
          bool ok = rp > a.min_score && rp >= thr_score && x >= xs + 3 && x < xs + 3 + kOut &&
                    x >= rx0 && x < rx1 && x >= ex0 && x < ex1;
          if (a.nms)
            ok = ok && rp > u[j] && rp > u[j + 1] && rp > u[j + 2] && rp > m[j] &&
                 rp >= m[j + 2] && rp >= d[j] && rp >= d[j + 1] && rp >= d[j + 2];
          if (ok && mask) ok = mask[(int64_t)yn * pitch + x] == 0;  // min_separation (f1)
          if (ok) {
            const unsigned long long kp = make_key(rp, x, yn, W);
            if (kp > thr) {
              const int slot = atomicAdd(&s_cnt[warp][1], 1);
              wbuf[ntop + slot] = kp;
            }
          }
        }
      }
      __syncwarp();
      const int nc = s_cnt[warp][1];
      if (nc > 0 && (ntop + nc + kSpan > kWBuf || (lazy && nc >= fold_at))) {
        bitonic_desc<false>(wbuf, ntop + nc, lane, 32);
        if (lane == 0) {
          s_cnt[warp][0] = min(ntop + nc, k);
          s_cnt[warp][1] = 0;
          if (ntop + nc >= k) atomicMax(&s_thr, wbuf[k - 1]);
        }
        __syncwarp();
      }
#pragma unroll
      for (int j = 0; j < kPix; ++j) {
        i0[j] = i1[j]; i1[j] = I[j + 1];
        hs0[j] = hs1[j]; hs1[j] = hs[j];
        a0[j] = a1[j]; a1[j] = ha[j];
        b0[j] = b1[j]; b1[j] = hb[j];
        c0[j] = c1[j]; c1[j] = hc[j];
      }
    }
  }
  // fold each warp's remaining candidates
  {
    const int ntop = s_cnt[warp][0], nc = s_cnt[warp][1];
    if (nc > 0) {
      bitonic_desc<false>(wbuf, ntop + nc, lane, 32);
      if (lane == 0) {
        s_cnt[warp][0] = min(ntop + nc, k);
        s_cnt[warp][1] = 0;
      }
    }
  }
  __syncthreads();
  // ---- CTA merge of the warps' top-k lists --------------------------------
  if (threadIdx.x == 0) {
    int off = 0;
    for (int w = 0; w < kWarps; ++w) {
      s_cnt[w][1] = off;  // reuse as prefix offset
      off += s_cnt[w][0];
    }
    s_total = off;
  }
  __syncthreads();
  unsigned long long tmp[V2D_MAX_K / 32];
  const int nmine = s_cnt[warp][0], dst = s_cnt[warp][1];
#pragma unroll
  for (int j = 0; j < V2D_MAX_K / 32; ++j) {
    const int i = lane + 32 * j;
    tmp[j] = i < nmine ? wbuf[i] : 0ull;
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < V2D_MAX_K / 32; ++j) {
    const int i = lane + 32 * j;
    if (i < nmine) s_buf[dst + i] = tmp[j];
  }
  __syncthreads();
  const int total = s_total;
  if (total > 1) bitonic_desc<true>(s_buf, total, threadIdx.x, kThreads);
  __syncthreads();
  const int ntop = min(total, k);

  // ---- emit the cell's slots (D6 slot order) -------------------------------
  const int64_t base = ((int64_t)(b * a.grid_y + cy) * a.grid_x + cx) * k;
  for (int s = threadIdx.x; s < k; s += kThreads) {
    float xo = -1.0f, yo = -1.0f, sc = 0.0f;
    if (s < ntop) {
      const unsigned long long kk = s_buf[s];
      const unsigned idx = 0xffffffffu - (unsigned)(kk & 0xffffffffull);
      xo = (float)(idx % (unsigned)W);
      yo = (float)(idx / (unsigned)W);
      sc = __uint_as_float((unsigned)(kk >> 32));
    }
    kp_xy[2 * (base + s)] = xo;
    kp_xy[2 * (base + s) + 1] = yo;
    kp_score[base + s] = sc;
  }
  if (threadIdx.x == 0) cell_count[(int64_t)b * a.grid_x * a.grid_y + cell] = ntop;
}

}  // namespace

int launch_gftt(const uint8_t* const* l0_ptrs, int B, const GfttArgs& a, float* kp_xy,
                float* kp_score, int32_t* cell_count, float* resp,
                const uint8_t* const* mask_ptrs, const int32_t* enable, cudaStream_t st) {
  if (B == 0) return V2D_OK;
  dim3 grid(a.grid_x * a.grid_y, B);
  gftt_topk_kernel<<<grid, kThreads, 0, st>>>(l0_ptrs, a, kp_xy, kp_score, cell_count, resp,
                                              mask_ptrs, enable);
  return cudaGetLastError() == cudaSuccess ? V2D_OK : V2D_ECUDA;
}

}  // namespace v2d
