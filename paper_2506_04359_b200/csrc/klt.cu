// klt.cu — K3: pyramidal Lucas-Kanade with per-level NCC gate.
//
// Operation ("a modified version of the Lucas-Kanade algorithm
// ... 1) performs tracking in a coarse-to-fine manner, continuously refining
// track positions at each image pyramid level, and 2) performs a normalized
// cross-correlation (NCC) check ... to filter out unreliable tracks"; the
// step-by-step reading is SURVEY §8(c) D7 / DESIGN.md readings #2, #11-#16):
//   for L = levels-1 .. 0:
//     c = (p + 0.5)/2^L - 0.5
//     T, Tx, Ty = bilinear samples of I_L, Gx_L, Gy_L at c+(u,v), where Gx_L, Gy_L
//                 are the clamp-to-edge Sobel/8 gradient IMAGES (sampled clamped)
//     G = sum [[Tx^2, TxTy],[TxTy, Ty^2]];  lambda_min(G)/n < min_eig -> skip/lost
//     repeat <= iters: e = T - S(J_L, c+d+(u,v)); eta = G^-1 sum e*(Tx,Ty); d += eta
//                      (bounds check; stop when |eta| < eps)
//     NCC(T, S(J_L, c+d+.)) < ncc_min -> LOST_NCC;  d *= 2 (L > 0)
//   p' = p + d must lie in the half-window margin.
//
// B200 mapping (DESIGN.md §5 K3): one WARP per keypoint slot, lane u = window
// column u.  Per level the warp stages a clamped 32-wide patch of the previous
// level (template) and then of the next level (with a margin of M px for the
// Gauss-Newton motion) into its own shared-memory tile, so the inner loops have
// no clamping or address arithmetic (immediate smem offsets).  T, Tx, Ty stay in
// registers as row PAIRS; every inner loop runs on packed fp32x2 FMA
// (__ffma2_rn / FFMA2, new on sm_100) two window rows per instruction.  G, b
// and the NCC moments are butterfly-reduced (bit-identical in every lane ->
// warp-uniform control flow); the 2x2 solve and tests run in float64 on the
// reduced scalars.
#include "common.cuh"

namespace v2d {
namespace {

constexpr int kWarps = 4;
constexpr int kThreads = 32 * kWarps;
constexpr int kPitch = 32;                 // smem patch row pitch (floats)
constexpr int kPatch = 32 * kPitch;        // floats per warp

struct Plane {
  const void* base;
  int64_t pitch;  // elements
  int W, H;
};

__device__ __forceinline__ int clampi(int v, int lo, int hi) { return min(max(v, lo), hi); }

__device__ __forceinline__ float2 f2(float a, float b) { return make_float2(a, b); }
__device__ __forceinline__ float2 add2(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 sub2(float2 a, float2 b) {
  return __fadd2_rn(a, make_float2(-b.x, -b.y));
}
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }

__device__ __forceinline__ float2 warp_sum2(float2 v) {
#pragma unroll
  for (int m = 16; m > 0; m >>= 1) {
    const float2 o = make_float2(__shfl_xor_sync(kFullMask, v.x, m),
                                 __shfl_xor_sync(kFullMask, v.y, m));
    v = add2(v, o);
  }
  return v;
}

// Stage rows [oy, oy+NR) x columns [ox, ox+32) of a level (clamp-to-edge) into
// the warp's patch, minus `shift`; lane = column.
template <typename TI, int NR>
__device__ __forceinline__ void stage(float* __restrict__ sp, const Plane& pl, int ox, int oy,
                                      float shift) {
  const int lane = threadIdx.x & 31;
  const TI* __restrict__ col =
      reinterpret_cast<const TI*>(pl.base) + clampi(ox + lane, 0, pl.W - 1);
  __syncwarp();
#pragma unroll 8
  for (int r = 0; r < NR; ++r) {
    const int y = clampi(oy + r, 0, pl.H - 1);
    sp[r * kPitch + lane] = (float)__ldg(col + (int64_t)y * pl.pitch) - shift;
  }
  __syncwarp();
}

struct LevelOut {
  int status;  // V2D_TRACKED while still alive
  float ncc;   // last evaluated NCC
  int steps;   // Gauss-Newton steps taken
  int levels;  // levels whose template was built
};

template <int WIN>
struct Tmpl {
  static constexpr int NPAIR = WIN / 2;  // row pairs; WIN odd -> one tail row
  float2 T[NPAIR], TX[NPAIR], TY[NPAIR];
  float Tt, TXt, TYt;                    // tail row WIN-1
  // row v (compile-time after unrolling) of each quantity
  __device__ __forceinline__ void set(int v, float tv, float txv, float tyv) {
    if (v == WIN - 1) {
      Tt = tv;
      TXt = txv;
      TYt = tyv;
    } else if (v & 1) {
      T[v >> 1].y = tv;
      TX[v >> 1].y = txv;
      TY[v >> 1].y = tyv;
    } else {
      T[v >> 1].x = tv;
      TX[v >> 1].x = txv;
      TY[v >> 1].x = tyv;
    }
  }
};

// Template of D7 at level L from the staged previous-level patch P
// (P[r][c] = I~(px0 + c, py0 + r), px0 = ix-R-1, py0 = iy-R-1).
template <int WIN>
__device__ __forceinline__ void build_template(const float* __restrict__ P, int ix, int iy,
                                               float ax, float ay, int W, int H, Tmpl<WIN>& t) {
  constexpr int R = (WIN - 1) / 2;
  const int lane = threadIdx.x & 31;
  const int i = min(lane, WIN);  // grid column of this lane (lanes > WIN duplicate WIN)
  const bool interior = (ix - R >= 0) && (ix + R + 1 <= W - 1) && (iy - R >= 0) &&
                        (iy + R + 1 <= H - 1);
  if (interior) {
    // rolling 3x3 over patch rows; grid row g = r-2 centred at patch row r-1
    float L1 = 0.f, L2 = 0.f, C1 = 0.f, C2 = 0.f, R1 = 0.f, R2 = 0.f;
    float hp_prev = 0.f, hgx_prev = 0.f, hgy_prev = 0.f, tpend = 0.f;
#pragma unroll
    for (int r = 0; r < WIN + 3; ++r) {
      const float* row = P + r * kPitch;
      const float l = row[i], c = row[i + 1], rr = row[i + 2];
      const float hp = fmaf(ax, rr - c, c);
      if (r >= 2) {
        const float tnew = fmaf(ay, hp - hp_prev, hp_prev);  // T row r-2
        const float2 V = fma2(f2(2.f, 2.f), f2(L1, R1), add2(f2(L2, R2), f2(l, rr)));
        const float gx = (V.y - V.x) * 0.125f;
        const float gy = ((l - L2) + 2.f * (c - C2) + (rr - R2)) * 0.125f;
        const float gx1 = __shfl_down_sync(kFullMask, gx, 1);
        const float gy1 = __shfl_down_sync(kFullMask, gy, 1);
        const float2 hg = fma2(f2(ax, ax), sub2(f2(gx1, gy1), f2(gx, gy)), f2(gx, gy));
        const int g = r - 2;
        if (g >= 1) {
          const float2 tg = fma2(f2(ay, ay), sub2(hg, f2(hgx_prev, hgy_prev)),
                                 f2(hgx_prev, hgy_prev));
          t.set(g - 1, tpend, tg.x, tg.y);
        }
        hgx_prev = hg.x;
        hgy_prev = hg.y;
        tpend = tnew;
      }
      hp_prev = hp;
      L2 = L1; L1 = l;
      C2 = C1; C1 = c;
      R2 = R1; R1 = rr;
    }
  } else {
    // generic: gradients at clamped centres (the gradient IMAGE is clamped),
    // intensities from the clamped patch
    const int lc = clampi(ix - R + i, 0, W - 1) - (ix - R - 1);
    float hp_prev = 0.f, hgx_prev = 0.f, hgy_prev = 0.f;
#pragma unroll
    for (int g = 0; g <= WIN; ++g) {
      const int lr = clampi(iy - R + g, 0, H - 1) - (iy - R - 1);
      const float* up = P + (lr - 1) * kPitch;
      const float* md = P + lr * kPitch;
      const float* dn = P + (lr + 1) * kPitch;
      const float gx = ((up[lc + 1] + 2.f * md[lc + 1] + dn[lc + 1]) -
                        (up[lc - 1] + 2.f * md[lc - 1] + dn[lc - 1])) * 0.125f;
      const float gy = ((dn[lc - 1] + 2.f * dn[lc] + dn[lc + 1]) -
                        (up[lc - 1] + 2.f * up[lc] + up[lc + 1])) * 0.125f;
      const float* prow = P + (g + 1) * kPitch;  // T rows use patch rows g+1 (and g+2)
      const float hp = fmaf(ax, prow[i + 2] - prow[i + 1], prow[i + 1]);
      const float gx1 = __shfl_down_sync(kFullMask, gx, 1);
      const float gy1 = __shfl_down_sync(kFullMask, gy, 1);
      const float2 hg = fma2(f2(ax, ax), sub2(f2(gx1, gy1), f2(gx, gy)), f2(gx, gy));
      if (g >= 1) {
        const float2 tg = fma2(f2(ay, ay), sub2(hg, f2(hgx_prev, hgy_prev)),
                               f2(hgx_prev, hgy_prev));
        t.set(g - 1, fmaf(ay, hp - hp_prev, hp_prev), tg.x, tg.y);
      }
      hgx_prev = hg.x;
      hgy_prev = hg.y;
      hp_prev = hp;
    }
  }
  const float valid = lane < WIN ? 1.0f : 0.0f;
  const float2 vv = f2(valid, valid);
#pragma unroll
  for (int p = 0; p < Tmpl<WIN>::NPAIR; ++p) {
    t.T[p] = __fmul2_rn(t.T[p], vv);
    t.TX[p] = __fmul2_rn(t.TX[p], vv);
    t.TY[p] = __fmul2_rn(t.TY[p], vv);
  }
  t.Tt *= valid;
  t.TXt *= valid;
  t.TYt *= valid;
}

// Horizontal lerp of patch rows; S'(u, v) sampled at patch origin (lc0, lr0).
// Returns sum over the window of e*(Tx, Ty) with e = T' - S' (both centred).
template <int WIN>
__device__ __forceinline__ float2 gn_rhs(const float* __restrict__ JP, int lc0, int lr0, float bx,
                                         float by, const Tmpl<WIN>& t) {
  const int lane = threadIdx.x & 31;
  const int u = min(lane, WIN - 1);
  const float* base = JP + lr0 * kPitch + lc0 + u;
  const float2 wx = f2(bx, bx), wy = f2(by, by);
  float h0 = fmaf(bx, base[1] - base[0], base[0]);
  float2 ax = f2(0.f, 0.f), ay = f2(0.f, 0.f);
#pragma unroll
  for (int p = 0; p < Tmpl<WIN>::NPAIR; ++p) {
    const float* r1 = base + (2 * p + 1) * kPitch;
    const float* r2 = base + (2 * p + 2) * kPitch;
    const float2 ja = f2(r1[0], r2[0]), jb = f2(r1[1], r2[1]);
    const float2 h = fma2(wx, sub2(jb, ja), ja);                 // rows 2p+1, 2p+2
    const float2 hv = f2(h0, h.x);                                // rows 2p, 2p+1
    const float2 S = fma2(wy, sub2(h, hv), hv);                  // samples 2p, 2p+1
    const float2 e = sub2(t.T[p], S);
    ax = fma2(e, t.TX[p], ax);
    ay = fma2(e, t.TY[p], ay);
    h0 = h.y;
  }
  float sx = ax.x + ax.y, sy = ay.x + ay.y;
  {
    const float* r = base + WIN * kPitch;
    const float h = fmaf(bx, r[1] - r[0], r[0]);
    const float e = t.Tt - fmaf(by, h - h0, h0);
    sx = fmaf(e, t.TXt, sx);
    sy = fmaf(e, t.TYt, sy);
  }
  return f2(sx, sy);
}

// NCC moments of the centred patch: returns (sum S', sum S'^2, sum T'S').
template <int WIN>
__device__ __forceinline__ float3 ncc_moments(const float* __restrict__ JP, int lc0, int lr0,
                                              float bx, float by, const Tmpl<WIN>& t) {
  const int lane = threadIdx.x & 31;
  const int u = min(lane, WIN - 1);
  const float valid = lane < WIN ? 1.0f : 0.0f;
  const float* base = JP + lr0 * kPitch + lc0 + u;
  const float2 wx = f2(bx, bx), wy = f2(by, by), vv = f2(valid, valid);
  float h0 = fmaf(bx, base[1] - base[0], base[0]);
  float2 s1 = f2(0.f, 0.f), s2 = f2(0.f, 0.f), st = f2(0.f, 0.f);
#pragma unroll
  for (int p = 0; p < Tmpl<WIN>::NPAIR; ++p) {
    const float* r1 = base + (2 * p + 1) * kPitch;
    const float* r2 = base + (2 * p + 2) * kPitch;
    const float2 ja = f2(r1[0], r2[0]), jb = f2(r1[1], r2[1]);
    const float2 h = fma2(wx, sub2(jb, ja), ja);
    const float2 hv = f2(h0, h.x);
    const float2 S = __fmul2_rn(fma2(wy, sub2(h, hv), hv), vv);
    s1 = add2(s1, S);
    s2 = fma2(S, S, s2);
    st = fma2(t.T[p], S, st);
    h0 = h.y;
  }
  float a = s1.x + s1.y, b = s2.x + s2.y, c = st.x + st.y;
  {
    const float* r = base + WIN * kPitch;
    const float h = fmaf(bx, r[1] - r[0], r[0]);
    const float S = fmaf(by, h - h0, h0) * valid;
    a += S;
    b = fmaf(S, S, b);
    c = fmaf(t.Tt, S, c);
  }
  return make_float3(a, b, c);
}

// One pyramid level of D7 for the warp's keypoint.
template <int WIN, typename TI, typename TJ>
__device__ __forceinline__ void track_level(float* __restrict__ sp, const Plane& I, const Plane& J,
                                            const int L, const double cx, const double cy,
                                            double& dx, double& dy, const KltArgs& a,
                                            LevelOut& out) {
  constexpr int R = (WIN - 1) / 2;
  constexpr int N = WIN * WIN;
  constexpr int M = (31 - WIN) / 2;        // staged motion margin (px)
  constexpr int SZ = WIN + 1 + 2 * M;      // staged J patch edge (<= 32)
  static_assert(WIN + 3 <= 32 && SZ <= 32, "window too large for one warp");
  const int lane = threadIdx.x & 31;

  // ---------------- template (previous frame) -----------------------------
  Tmpl<WIN> t;
  {
    const double fcx = floor(cx), fcy = floor(cy);
    const int ix = (int)fcx, iy = (int)fcy;
    stage<TI, WIN + 3>(sp, I, ix - R - 1, iy - R - 1, 0.0f);
    build_template<WIN>(sp, ix, iy, (float)(cx - fcx), (float)(cy - fcy), I.W, I.H, t);
  }
  out.levels++;
  // G and template mean
  float2 gxx_gxy = f2(0.f, 0.f), gyy_st = f2(0.f, 0.f);
#pragma unroll
  for (int p = 0; p < Tmpl<WIN>::NPAIR; ++p) {
    const float2 tx = t.TX[p], ty = t.TY[p], tt = t.T[p];
    gxx_gxy = fma2(f2(tx.x, tx.x), f2(tx.x, ty.x), gxx_gxy);
    gxx_gxy = fma2(f2(tx.y, tx.y), f2(tx.y, ty.y), gxx_gxy);
    gyy_st = fma2(f2(ty.x, 1.f), f2(ty.x, tt.x), gyy_st);
    gyy_st = fma2(f2(ty.y, 1.f), f2(ty.y, tt.y), gyy_st);
  }
  gxx_gxy = fma2(f2(t.TXt, t.TXt), f2(t.TXt, t.TYt), gxx_gxy);
  gyy_st = fma2(f2(t.TYt, 1.f), f2(t.TYt, t.Tt), gyy_st);
  gxx_gxy = warp_sum2(gxx_gxy);
  gyy_st = warp_sum2(gyy_st);
  const double gxx = gxx_gxy.x, gxy = gxx_gxy.y, gyy = gyy_st.x;
  const double tr = gxx + gyy;
  const double det = gxx * gyy - gxy * gxy;
  const double lmin =
      tr == 0.0 ? 0.0 : det / (0.5 * (tr + sqrt((gxx - gyy) * (gxx - gyy) + 4.0 * gxy * gxy)));
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
  // centre the template: T' = T - mean (NCC two-pass; also conditions e = T'-S')
  const float tmean = gyy_st.y / (float)N;
  const float valid = lane < WIN ? 1.0f : 0.0f;
  float2 tt_t1 = f2(0.f, 0.f);  // (sum T'^2, sum T')
#pragma unroll
  for (int p = 0; p < Tmpl<WIN>::NPAIR; ++p) {
    t.T[p] = __fmul2_rn(sub2(t.T[p], f2(tmean, tmean)), f2(valid, valid));
    tt_t1 = fma2(f2(t.T[p].x, 1.f), f2(t.T[p].x, t.T[p].x), tt_t1);
    tt_t1 = fma2(f2(t.T[p].y, 1.f), f2(t.T[p].y, t.T[p].y), tt_t1);
  }
  t.Tt = (t.Tt - tmean) * valid;
  tt_t1 = fma2(f2(t.Tt, 1.f), f2(t.Tt, t.Tt), tt_t1);
  const float2 red = warp_sum2(tt_t1);
  const double Stt0 = red.x, St1 = red.y;

  // ---------------- Gauss-Newton iterations (next frame) --------------------
  const int W = J.W, H = J.H;
  int jx0 = 0, jy0 = 0;
  bool staged = false;
  auto locate = [&](double qx, double qy, int& lc0, int& lr0, float& bx, float& by) {
    const double fqx = floor(qx), fqy = floor(qy);
    const int ixq = (int)fqx, iyq = (int)fqy;
    bx = (float)(qx - fqx);
    by = (float)(qy - fqy);
    lc0 = ixq - R - jx0;
    lr0 = iyq - R - jy0;
    if (!staged || lc0 < 0 || lc0 > 2 * M || lr0 < 0 || lr0 > 2 * M) {
      jx0 = ixq - R - M;
      jy0 = iyq - R - M;
      stage<TJ, SZ>(sp, J, jx0, jy0, tmean);
      staged = true;
      lc0 = M;
      lr0 = M;
    }
  };
  for (int it = 1; it <= a.iters; ++it) {
    int lc0, lr0;
    float bx, by;
    locate(cx + dx, cy + dy, lc0, lr0, bx, by);
    const float2 b = warp_sum2(gn_rhs<WIN>(sp, lc0, lr0, bx, by, t));
    const double ex = (gyy * (double)b.x - gxy * (double)b.y) / det;
    const double ey = (gxx * (double)b.y - gxy * (double)b.x) / det;
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
    int lc0, lr0;
    float bx, by;
    locate(cx + dx, cy + dy, lc0, lr0, bx, by);
    const float3 mo = ncc_moments<WIN>(sp, lc0, lr0, bx, by, t);
    const float2 r1 = warp_sum2(f2(mo.x, mo.y));
    const float2 r2 = warp_sum2(f2(mo.z, 0.f));
    const double S1 = r1.x, S2 = r1.y, STS = r2.x;
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
__global__ void __launch_bounds__(kThreads, (WIN >= 19 ? 3 : 4))
klt_kernel(const uint8_t* const* __restrict__ prev_l0, const float* const* __restrict__ prev_pyr,
           const uint8_t* const* __restrict__ next_l0, const float* const* __restrict__ next_pyr,
           int B, Levels lv, KltArgs a, const float* __restrict__ pts,
           const float* __restrict__ guess, const uint8_t* __restrict__ in_status,
           float* __restrict__ out_pos, uint8_t* __restrict__ status, float* __restrict__ ncc,
           int32_t* __restrict__ iters_out) {
  __shared__ float s_patch[kWarps * kPatch];
  const int64_t warp = (int64_t)blockIdx.x * kWarps + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (warp >= (int64_t)B * a.P) return;  // warp-uniform
  float* sp = s_patch + (threadIdx.x >> 5) * kPatch;
  const int b = (int)(warp / a.P);
  const float px = pts[2 * warp], py = pts[2 * warp + 1];
  constexpr int R = (WIN - 1) / 2;

  LevelOut o{V2D_TRACKED, 0.0f, 0, 0};
  const bool skip = (in_status && in_status[warp] != 0) || (px == -1.0f && py == -1.0f) ||
                    !isfinite(px) || !isfinite(py);
  double dx = 0.0, dy = 0.0;
  if (skip) {
    o.status = V2D_SKIPPED;
  } else if (px < 0.0f || px > (float)(lv.W[0] - 1) || py < 0.0f || py > (float)(lv.H[0] - 1)) {
    o.status = V2D_LOST_OOB;  // reading #16: a start point outside the image is lost
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
        track_level<WIN, uint8_t, uint8_t>(sp, I, J, 0, cx, cy, dx, dy, a, o);
      } else {
        const Plane I{prev_pyr[b] + lv.offset[L], lv.pitch[L], lv.W[L], lv.H[L]};
        const Plane J{next_pyr[b] + lv.offset[L], lv.pitch[L], lv.W[L], lv.H[L]};
        track_level<WIN, float, float>(sp, I, J, L, cx, cy, dx, dy, a, o);
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
#define V2D_WIN_CASE(w)                                                                   \
  case w:                                                                                 \
    launch_win<w>(prev_l0, prev_pyr, next_l0, next_pyr, B, lv, a, pts, guess, in_status, \
                  out_pos, status, ncc, iters_out, st);                                   \
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
