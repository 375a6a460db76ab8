// klt.cu — K3: pyramidal Lucas-Kanade with per-level NCC gate.
//
// Operation ("a modified version of the Lucas-Kanade algorithm
// ... 1) performs tracking in a coarse-to-fine manner, continuously refining
// track positions at each image pyramid level, and 2) performs a normalized
// cross-correlation (NCC) check ... to filter out unreliable tracks"; the
// step-by-step reading is SURVEY §8(c) D7 / DESIGN.md readings #2, #11-#16):
//   for L = levels-1 .. 0:
//     c = (p + 0.5)/2^L - 0.5
//     T, Tx, Ty = bilinear samples of I_L, Gx_L, Gy_L (clamped Sobel/8) at c+(u,v)
//     G = sum [[Tx^2, TxTy],[TxTy, Ty^2]];  lambda_min(G)/n < min_eig -> skip/lost
//     repeat <= iters: e = T - S(J_L, c+d+(u,v)); eta = G^-1 sum e*(Tx,Ty); d += eta
//                      (bounds check; stop when |eta| < eps)
//     NCC(T, S(J_L, c+d+.)) < ncc_min -> LOST_NCC;  d *= 2 (L > 0)
//   p' = p + d must lie in the half-window margin.
//
// B200 mapping: one WARP per keypoint slot, no shared memory.  Lane u owns
// window column u: it streams the rows of its column from L1/L2 (one load per
// row), gets the right-hand neighbour column by __shfl_down_sync, so the
// bilinear weights (shared by all samples of a keypoint) are applied with two
// FMAs per sample; the template T, Tx, Ty (3 x win floats per lane) stays in
// registers across all Gauss-Newton steps; the template gradients come from a
// rolling 3-row Sobel in registers + shuffles.  G, b and the NCC moments are
// butterfly-reduced (bit-identical in every lane, so control flow is
// warp-uniform).  The 2x2 solve, eigenvalue and convergence tests run in
// float64 on the reduced scalars.
#include "common.cuh"

namespace v2d {
namespace {

constexpr int kWarps = 4;
constexpr int kThreads = 32 * kWarps;

struct Plane {
  const void* base;
  int64_t pitch;  // elements
  int W, H;
};

template <typename T>
__device__ __forceinline__ float ld(const Plane& pl, int x, int y) {
  return (float)__ldg(reinterpret_cast<const T*>(pl.base) + (int64_t)y * pl.pitch + x);
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int m = 16; m > 0; m >>= 1) v += __shfl_xor_sync(kFullMask, v, m);
  return v;
}
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int m = 16; m > 0; m >>= 1) v += __shfl_xor_sync(kFullMask, v, m);
  return v;
}

__device__ __forceinline__ int clampi(int v, int lo, int hi) { return min(max(v, lo), hi); }

struct LevelOut {
  int status;     // V2D_TRACKED while still alive
  float ncc;      // last evaluated NCC
  int steps;      // Gauss-Newton steps taken
  int levels;     // levels whose template was built
};

// One pyramid level of D7 for the warp's keypoint.  (dx, dy) is the level-L
// displacement, updated in place.  Returns status (TRACKED = continue).
template <int WIN, typename TI, typename TJ>
__device__ __forceinline__ void track_level(const Plane& I, const Plane& J, const int L,
                                            const double cx, const double cy, double& dx,
                                            double& dy, const KltArgs& a, LevelOut& out) {
  constexpr int R = (WIN - 1) / 2;
  constexpr int NP = WIN + 3;
  constexpr int N = WIN * WIN;
  static_assert(NP <= 32, "window too large for one warp");
  const int lane = threadIdx.x & 31;
  const float valid = lane < WIN ? 1.0f : 0.0f;

  // ---------------- template T, Tx, Ty (register resident) ----------------
  float T[WIN], TX[WIN], TY[WIN];
  {
    const double fcx = floor(cx), fcy = floor(cy);
    const float ax = (float)(cx - fcx), ay = (float)(cy - fcy);
    const int ix = (int)fcx, iy = (int)fcy;
    const int colP = clampi(ix - R - 1 + lane, 0, I.W - 1);
    float pm2 = 0.f, pm1 = 0.f, hp_prev = 0.f, hgx_prev = 0.f, hgy_prev = 0.f;
#pragma unroll
    for (int j = 0; j < NP; ++j) {
      const float pj = ld<TI>(I, colP, clampi(iy - R - 1 + j, 0, I.H - 1));
      const float p1 = __shfl_down_sync(kFullMask, pj, 1);
      const float p2 = __shfl_down_sync(kFullMask, pj, 2);
      const float hp = fmaf(ax, p2 - p1, p1);
      if (j >= 2) {
        if (j - 2 < WIN) T[j - 2] = fmaf(ay, hp - hp_prev, hp_prev);
        // Sobel/8 at grid row g = j-2 (P rows j-2, j-1, j), grid column = lane
        const float V = pm2 + 2.0f * pm1 + pj;
        const float Dv = pj - pm2;
        const float V2 = __shfl_down_sync(kFullMask, V, 2);
        const float D1 = __shfl_down_sync(kFullMask, Dv, 1);
        const float D2 = __shfl_down_sync(kFullMask, Dv, 2);
        const float gx = (V2 - V) * 0.125f;
        const float gy = (Dv + 2.0f * D1 + D2) * 0.125f;
        const float gx1 = __shfl_down_sync(kFullMask, gx, 1);
        const float gy1 = __shfl_down_sync(kFullMask, gy, 1);
        const float hgx = fmaf(ax, gx1 - gx, gx);
        const float hgy = fmaf(ax, gy1 - gy, gy);
        const int g = j - 2;
        if (g >= 1) {
          TX[g - 1] = fmaf(ay, hgx - hgx_prev, hgx_prev);
          TY[g - 1] = fmaf(ay, hgy - hgy_prev, hgy_prev);
        }
        hgx_prev = hgx;
        hgy_prev = hgy;
      }
      hp_prev = hp;
      pm2 = pm1;
      pm1 = pj;
    }
#pragma unroll
    for (int v = 0; v < WIN; ++v) {
      T[v] *= valid;
      TX[v] *= valid;
      TY[v] *= valid;
    }
  }
  out.levels++;
  // ---------------- G, eigenvalue gate --------------------------------------
  float sxx = 0.f, sxy = 0.f, syy = 0.f, st = 0.f;
#pragma unroll
  for (int v = 0; v < WIN; ++v) {
    sxx = fmaf(TX[v], TX[v], sxx);
    sxy = fmaf(TX[v], TY[v], sxy);
    syy = fmaf(TY[v], TY[v], syy);
    st += T[v];
  }
  const double gxx = warp_sum((double)sxx), gxy = warp_sum((double)sxy),
               gyy = warp_sum((double)syy);
  const double tr = gxx + gyy;
  const double det = gxx * gyy - gxy * gxy;
  const double lmin = tr == 0.0 ? 0.0 : det / (0.5 * (tr + sqrt((gxx - gyy) * (gxx - gyy) + 4.0 * gxy * gxy)));
  const bool finite = isfinite(gxx) && isfinite(gxy) && isfinite(gyy) && isfinite(lmin);
  if (!finite || lmin / N < (double)a.min_eig) {
    if (L > 0) {
      dx *= 2.0;
      dy *= 2.0;
    } else {
      out.status = V2D_LOST_SMALL_EIG;
    }
    return;
  }
  // template moments for the two-pass NCC (T' = T - mean)
  const float tmean = (float)(warp_sum((double)st) / N);
  float stt = 0.f, st1 = 0.f;
#pragma unroll
  for (int v = 0; v < WIN; ++v) {
    const float t = (T[v] - tmean) * valid;
    stt = fmaf(t, t, stt);
    st1 += t;
  }
  const double Stt0 = warp_sum((double)stt), St1 = warp_sum((double)st1);

  // ---------------- Gauss-Newton iterations ---------------------------------
  const int W = J.W, H = J.H;
  for (int it = 1; it <= a.iters; ++it) {
    const double qx = cx + dx, qy = cy + dy;
    const double fqx = floor(qx), fqy = floor(qy);
    const float bx_w = (float)(qx - fqx), by_w = (float)(qy - fqy);
    const int ix = (int)fqx, iy = (int)fqy;
    const int col = clampi(ix - R + lane, 0, W - 1);
    float hprev = 0.f, sbx = 0.f, sby = 0.f;
#pragma unroll
    for (int v = 0; v <= WIN; ++v) {
      const float jv = ld<TJ>(J, col, clampi(iy - R + v, 0, H - 1));
      const float jn = __shfl_down_sync(kFullMask, jv, 1);
      const float h = fmaf(bx_w, jn - jv, jv);
      if (v >= 1) {
        const float S = fmaf(by_w, h - hprev, hprev);
        const float e = T[v - 1] - S;
        sbx = fmaf(e, TX[v - 1], sbx);
        sby = fmaf(e, TY[v - 1], sby);
      }
      hprev = h;
    }
    const double bx = warp_sum(sbx), by = warp_sum(sby);
    const double ex = (gyy * bx - gxy * by) / det;
    const double ey = (gxx * by - gxy * bx) / det;
    dx += ex;
    dy += ey;
    out.steps++;
    const double nx = cx + dx, ny = cy + dy;
    const bool inside = isfinite(nx) && isfinite(ny) && nx >= 0.0 && nx <= (double)(W - 1) &&
                        ny >= 0.0 && ny <= (double)(H - 1);
    if (!inside) {
      if (L > 0) {
        dx -= ex;
        dy -= ey;
        break;
      }
      out.status = V2D_LOST_OOB;
      return;
    }
    if (sqrt(ex * ex + ey * ey) < (double)a.eps) break;
  }
  // ---------------- per-level NCC gate --------------------------------------
  {
    const double qx = cx + dx, qy = cy + dy;
    const double fqx = floor(qx), fqy = floor(qy);
    const float bx_w = (float)(qx - fqx), by_w = (float)(qy - fqy);
    const int ix = (int)fqx, iy = (int)fqy;
    const int col = clampi(ix - R + lane, 0, W - 1);
    float hprev = 0.f, s1 = 0.f, s2 = 0.f, sts = 0.f;
#pragma unroll
    for (int v = 0; v <= WIN; ++v) {
      const float jv = ld<TJ>(J, col, clampi(iy - R + v, 0, H - 1));
      const float jn = __shfl_down_sync(kFullMask, jv, 1);
      const float h = fmaf(bx_w, jn - jv, jv);
      if (v >= 1) {
        const float S = (fmaf(by_w, h - hprev, hprev) - tmean) * valid;
        s1 += S;
        s2 = fmaf(S, S, s2);
        sts = fmaf(T[v - 1] - tmean, S, sts);
      }
      hprev = h;
    }
    const double S1 = warp_sum((double)s1), S2 = warp_sum((double)s2),
                 STS = warp_sum((double)sts);
    const double Stt = Stt0 - St1 * St1 / N;
    const double Sss = S2 - S1 * S1 / N;
    const double Sts = STS - St1 * S1 / N;
    const double den = sqrt(Stt * Sss);
    out.ncc = den > 0.0 ? (float)(Sts / den) : 0.0f;
    if (out.ncc < a.ncc_min) {
      out.status = V2D_LOST_NCC;
      return;
    }
  }
  if (L > 0) {
    dx *= 2.0;
    dy *= 2.0;
  }
}

template <int WIN>
__global__ void __launch_bounds__(kThreads)
klt_kernel(const uint8_t* const* __restrict__ prev_l0, const float* const* __restrict__ prev_pyr,
           const uint8_t* const* __restrict__ next_l0, const float* const* __restrict__ next_pyr,
           int B, Levels lv, KltArgs a, const float* __restrict__ pts,
           const float* __restrict__ guess, const uint8_t* __restrict__ in_status,
           float* __restrict__ out_pos, uint8_t* __restrict__ status, float* __restrict__ ncc,
           int32_t* __restrict__ iters_out) {
  const int64_t warp = (int64_t)blockIdx.x * kWarps + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (warp >= (int64_t)B * a.P) return;  // warp-uniform
  const int b = (int)(warp / a.P);
  const float px = pts[2 * warp], py = pts[2 * warp + 1];
  constexpr int R = (WIN - 1) / 2;

  LevelOut o{V2D_TRACKED, 0.0f, 0, 0};
  const bool skip = (in_status && in_status[warp] != 0) || (px == -1.0f && py == -1.0f) ||
                    !isfinite(px) || !isfinite(py);
  double dx = 0.0, dy = 0.0;
  if (skip) {
    o.status = V2D_SKIPPED;
  } else {
    if (guess) {
      const double s = 1.0 / (double)(1 << (lv.n - 1));
      dx = guess[2 * warp] * s;
      dy = guess[2 * warp + 1] * s;
    }
    for (int L = lv.n - 1; L >= 0 && o.status == V2D_TRACKED; --L) {
      const double scale = (double)(1 << L);
      const double cx = ((double)px + 0.5) / scale - 0.5;
      const double cy = ((double)py + 0.5) / scale - 0.5;
      if (L == 0) {
        const Plane I{prev_l0[b], a.l0_pitch, lv.W[0], lv.H[0]};
        const Plane J{next_l0[b], a.l0_pitch, lv.W[0], lv.H[0]};
        track_level<WIN, uint8_t, uint8_t>(I, J, 0, cx, cy, dx, dy, a, o);
      } else {
        const Plane I{prev_pyr[b] + lv.offset[L], lv.pitch[L], lv.W[L], lv.H[L]};
        const Plane J{next_pyr[b] + lv.offset[L], lv.pitch[L], lv.W[L], lv.H[L]};
        track_level<WIN, float, float>(I, J, L, cx, cy, dx, dy, a, o);
      }
    }
  }
  float ox = -1.0f, oy = -1.0f;
  if (o.status == V2D_TRACKED) {
    const double qx = (double)px + dx, qy = (double)py + dy;
    const int W = lv.W[0], H = lv.H[0];
    if (qx < R || qx > W - 1 - R || qy < R || qy > H - 1 - R) {
      o.status = V2D_LOST_OOB;
    } else {
      ox = (float)qx;
      oy = (float)qy;
    }
  }
  if (lane == 0) {
    out_pos[2 * warp] = ox;
    out_pos[2 * warp + 1] = oy;
    status[warp] = (uint8_t)o.status;
    if (ncc) ncc[warp] = o.ncc;
    if (iters_out) iters_out[warp] = o.steps | (o.levels << 24);
  }
}

template <int WIN>
void launch_win(const uint8_t* const* prev_l0, const float* const* prev_pyr,
                const uint8_t* const* next_l0, const float* const* next_pyr, int B,
                const Levels& lv, const KltArgs& a, const float* pts, const float* guess,
                const uint8_t* in_status, float* out_pos, uint8_t* status, float* ncc,
                int32_t* iters_out, cudaStream_t st) {
  const int64_t warps = (int64_t)B * a.P;
  const unsigned blocks = (unsigned)((warps + kWarps - 1) / kWarps);
  klt_kernel<WIN><<<blocks, kThreads, 0, st>>>(prev_l0, prev_pyr, next_l0, next_pyr, B, lv, a,
                                                pts, guess, in_status, out_pos, status, ncc,
                                                iters_out);
}

}  // namespace

int launch_klt(const uint8_t* const* prev_l0, const float* const* prev_pyr,
               const uint8_t* const* next_l0, const float* const* next_pyr, int B,
               const Levels& lv, const KltArgs& a, const float* pts, const float* guess,
               const uint8_t* in_status, float* out_pos, uint8_t* status, float* ncc,
               int32_t* iters_out, cudaStream_t st) {
  if (B == 0 || a.P == 0) return V2D_OK;
#define V2D_WIN_CASE(w)                                                                    \
  case w:                                                                                  \
    launch_win<w>(prev_l0, prev_pyr, next_l0, next_pyr, B, lv, a, pts, guess, in_status,  \
                  out_pos, status, ncc, iters_out, st);                                    \
    break;
  switch (a.win) {
    V2D_WIN_CASE(3)
    V2D_WIN_CASE(5)
    V2D_WIN_CASE(7)
    V2D_WIN_CASE(9)
    V2D_WIN_CASE(11)
    V2D_WIN_CASE(13)
    V2D_WIN_CASE(15)
    V2D_WIN_CASE(17)
    V2D_WIN_CASE(19)
    V2D_WIN_CASE(21)
    V2D_WIN_CASE(23)
    V2D_WIN_CASE(25)
    V2D_WIN_CASE(27)
    V2D_WIN_CASE(29)
    default:
      return V2D_EINVAL;
  }
#undef V2D_WIN_CASE
  return cudaGetLastError() == cudaSuccess ? V2D_OK : V2D_ECUDA;
}

}  // namespace v2d
