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
// B200 mapping: one CTA (256 threads) per (cell, image).  The cell is swept in
// 32x32 output tiles; each tile stages its u8 footprint (+3 px halo) in shared
// memory and runs the separable stencil stages there (Sobel -> horizontal
// 3-sums -> vertical 3-sums + R -> NMS).  Candidates that beat the running
// per-cell threshold are appended to a shared-memory key buffer which a
// block-wide bitonic sort periodically folds back to the top k; the threshold
// then enables the lazy eigenvalue: lambda_min <= min(A',C')/64, so R is only
// evaluated where that bound can beat the k-th best key (exact — see DESIGN.md
// §5 K2).  No atomics in global memory, deterministic output.
#include "common.cuh"

namespace v2d {
namespace {

constexpr int kThreads = 256;
constexpr int TS = 32;           // output tile edge
constexpr int IMG = TS + 6;      // staged u8 edge (halo 3)
constexpr int IMGP = IMG + 2;    // padded row stride
constexpr int SOB = TS + 4;      // Sobel edge (halo 2)
constexpr int RE = TS + 2;       // response edge (halo 1)
constexpr int kBuf = 2048;       // candidate / top-k key buffer

__device__ __forceinline__ float response_contract(int A, int Bv, int C) {
  const int tr = A + C;
  if (tr == 0) return 0.0f;
  const long long det = (long long)A * C - (long long)Bv * Bv;
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

// Sort buf[0..ntop+ncand) descending and keep the first min(k, total).
__device__ void fold_topk(unsigned long long* buf, int* s_n, int k) {
  __syncthreads();
  const int total = s_n[0] + s_n[1];
  int N = 2;
  while (N < total) N <<= 1;
  for (int i = total + threadIdx.x; i < N; i += kThreads) buf[i] = 0ull;
  __syncthreads();
  for (int size = 2; size <= N; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = threadIdx.x; i < (N >> 1); i += kThreads) {
        const int lo = 2 * i - (i & (stride - 1));
        const int hi = lo + stride;
        const bool desc = (lo & size) == 0;
        const unsigned long long a = buf[lo], c = buf[hi];
        if ((a < c) == desc) {
          buf[lo] = c;
          buf[hi] = a;
        }
      }
      __syncthreads();
    }
  }
  if (threadIdx.x == 0) {
    s_n[0] = total < k ? total : k;
    s_n[1] = 0;
  }
  __syncthreads();
}

__global__ void __launch_bounds__(kThreads)
gftt_topk_kernel(const uint8_t* const* __restrict__ l0_ptrs, GfttArgs a,
                 float* __restrict__ kp_xy, float* __restrict__ kp_score,
                 int32_t* __restrict__ cell_count, float* __restrict__ resp) {
  __shared__ uint8_t s_img[IMG * IMGP];
  __shared__ short2 s_sob[SOB * SOB];
  __shared__ int s_hA[SOB * RE], s_hB[SOB * RE], s_hC[SOB * RE];
  __shared__ float s_R[RE * RE];
  __shared__ unsigned long long s_buf[kBuf];
  __shared__ int s_n[2];  // [0] = entries kept (top), [1] = appended candidates

  const int W = a.W, H = a.H;
  const int cell = blockIdx.x, b = blockIdx.y;
  const int cx = cell % a.grid_x, cy = cell / a.grid_x;
  const uint8_t* __restrict__ img = l0_ptrs[b];
  const int64_t pitch = a.pitch;

  // D6 cell: [floor(cx*W/gx), floor((cx+1)*W/gx)) x [...]
  const int x0 = (int)((int64_t)cx * W / a.grid_x), x1 = (int)((int64_t)(cx + 1) * W / a.grid_x);
  const int y0 = (int)((int64_t)cy * H / a.grid_y), y1 = (int)((int64_t)(cy + 1) * H / a.grid_y);
  // D5 eligibility box
  const int ex0 = a.border, ex1 = W - a.border, ey0 = a.border, ey1 = H - a.border;
  const bool full = resp != nullptr;  // need R everywhere in the cell
  const int rx0 = full ? x0 : max(x0, ex0), rx1 = full ? x1 : min(x1, ex1);
  const int ry0 = full ? y0 : max(y0, ey0), ry1 = full ? y1 : min(y1, ey1);
  const bool lazy = !full;
  const int max_per_tile = a.nms ? (TS * TS) / 4 : TS * TS;
  const int early = max(64, 2 * a.k);

  if (threadIdx.x == 0) {
    s_n[0] = 0;
    s_n[1] = 0;
  }
  __syncthreads();

  for (int ty = ry0; ty < ry1; ty += TS) {
    for (int tx = rx0; tx < rx1; tx += TS) {
      // running threshold (score part used by the lazy eigenvalue bound)
      const int ntop = s_n[0];
      const unsigned long long thr = (ntop == a.k) ? s_buf[a.k - 1] : 0ull;
      const float thr_score = __uint_as_float((unsigned)(thr >> 32));

      // ---- stage u8 footprint (clamped reads; out-of-image values are
      //      never used by an in-domain response) -------------------------
      for (int i = threadIdx.x; i < IMG * IMG; i += kThreads) {
        const int jj = i / IMG, ii = i % IMG;
        const int gx = min(max(tx - 3 + ii, 0), W - 1);
        const int gy = min(max(ty - 3 + jj, 0), H - 1);
        s_img[jj * IMGP + ii] = __ldg(img + (int64_t)gy * pitch + gx);
      }
      __syncthreads();
      // ---- integer Sobel (sx = 8 Gx, sy = 8 Gy) --------------------------
      for (int i = threadIdx.x; i < SOB * SOB; i += kThreads) {
        const int jj = i / SOB, ii = i % SOB;
        const uint8_t* r0 = s_img + jj * IMGP + ii;
        const uint8_t* r1 = r0 + IMGP;
        const uint8_t* r2 = r1 + IMGP;
        const int sx = (r0[2] + 2 * r1[2] + r2[2]) - (r0[0] + 2 * r1[0] + r2[0]);
        const int sy = (r2[0] + 2 * r2[1] + r2[2]) - (r0[0] + 2 * r0[1] + r0[2]);
        s_sob[i] = make_short2((short)sx, (short)sy);
      }
      __syncthreads();
      // ---- horizontal 3-sums of the tensor products ----------------------
      for (int i = threadIdx.x; i < SOB * RE; i += kThreads) {
        const int jj = i / RE, ii = i % RE;
        const short2* s = s_sob + jj * SOB + ii;
        int A = 0, Bv = 0, C = 0;
#pragma unroll
        for (int d = 0; d < 3; ++d) {
          const int gx = s[d].x, gy = s[d].y;
          A += gx * gx;
          Bv += gx * gy;
          C += gy * gy;
        }
        s_hA[i] = A;
        s_hB[i] = Bv;
        s_hC[i] = C;
      }
      __syncthreads();
      // ---- vertical 3-sums + response (lazy) -----------------------------
      for (int i = threadIdx.x; i < RE * RE; i += kThreads) {
        const int jj = i / RE, ii = i % RE;
        const int px = tx - 1 + ii, py = ty - 1 + jj;
        float r = 0.0f;
        if (px >= 2 && px <= W - 3 && py >= 2 && py <= H - 3) {
          const int o = jj * RE + ii;
          const int A = s_hA[o] + s_hA[o + RE] + s_hA[o + 2 * RE];
          const int C = s_hC[o] + s_hC[o + RE] + s_hC[o + 2 * RE];
          // lambda_min <= min(A',C')/64; the 1e-5 slack covers fp32 rounding
          // of the contract value (<= ~5 ulp).
          const float ub = (float)min(A, C) * (0.015625f * 1.00001f);
          if (!lazy || ub >= thr_score) {
            const int Bv = s_hB[o] + s_hB[o + RE] + s_hB[o + 2 * RE];
            r = response_contract(A, Bv, C);
          }
        }
        s_R[i] = r;
        if (full && ii >= 1 && ii <= TS && jj >= 1 && jj <= TS && px < x1 && py < y1)
          resp[((int64_t)b * H + py) * W + px] = r;
      }
      __syncthreads();
      // ---- eligibility + NMS + threshold -> append -----------------------
      for (int i = threadIdx.x; i < TS * TS; i += kThreads) {
        const int jj = i / TS, ii = i % TS;
        const int px = tx + ii, py = ty + jj;
        if (px >= rx1 || py >= ry1) continue;
        if (px < ex0 || px >= ex1 || py < ey0 || py >= ey1) continue;
        const int o = (jj + 1) * RE + (ii + 1);
        const float r = s_R[o];
        if (!(r > a.min_score)) continue;
        const unsigned long long kp = make_key(r, px, py, W);
        if (kp <= thr) continue;
        bool ok = true;
        if (a.nms) {
#pragma unroll
          for (int dj = -1; dj <= 1; ++dj)
#pragma unroll
            for (int di = -1; di <= 1; ++di) {
              if (di == 0 && dj == 0) continue;
              const unsigned long long kq = make_key(s_R[o + dj * RE + di], px + di, py + dj, W);
              ok = ok && (kp > kq);
            }
        }
        if (ok) {
          const int slot = atomicAdd(&s_n[1], 1);
          s_buf[ntop + slot] = kp;
        }
      }
      __syncthreads();
      const int nc = s_n[1];
      if (s_n[0] + nc + max_per_tile > kBuf || (lazy && nc >= early)) fold_topk(s_buf, s_n, a.k);
    }
  }
  if (s_n[1] > 0) fold_topk(s_buf, s_n, a.k);

  // ---- emit the cell's slots (D6 slot order) -----------------------------
  const int ntop = s_n[0];
  const int64_t base = ((int64_t)(b * a.grid_y + cy) * a.grid_x + cx) * a.k;
  for (int s = threadIdx.x; s < a.k; s += kThreads) {
    float x = -1.0f, y = -1.0f, sc = 0.0f;
    if (s < ntop) {
      const unsigned long long kk = s_buf[s];
      const unsigned idx = 0xffffffffu - (unsigned)(kk & 0xffffffffull);
      x = (float)(idx % (unsigned)W);
      y = (float)(idx / (unsigned)W);
      sc = __uint_as_float((unsigned)(kk >> 32));
    }
    kp_xy[2 * (base + s)] = x;
    kp_xy[2 * (base + s) + 1] = y;
    kp_score[base + s] = sc;
  }
  if (threadIdx.x == 0) cell_count[(int64_t)b * a.grid_x * a.grid_y + cell] = ntop;
}

}  // namespace

int launch_gftt(const uint8_t* const* l0_ptrs, int B, const GfttArgs& a, float* kp_xy,
                float* kp_score, int32_t* cell_count, float* resp, cudaStream_t st) {
  if (B == 0) return V2D_OK;
  dim3 grid(a.grid_x * a.grid_y, B);
  gftt_topk_kernel<<<grid, kThreads, 0, st>>>(l0_ptrs, a, kp_xy, kp_score, cell_count, resp);
  return cudaGetLastError() == cudaSuccess ? V2D_OK : V2D_ECUDA;
}

}  // namespace v2d
