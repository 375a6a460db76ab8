// klt_pair.cu — K3 for small windows (win <= 13): TWO keypoints per warp.
//
// Same operation as klt.cu (DESIGN.md readings
// #2, #11-#16, #19, #27), same arithmetic in the same order, but each half-warp
// (16 lanes) tracks its own keypoint.  For small windows the one-warp-per-
// keypoint kernel is dominated by per-keypoint-level fixed costs (two patch
// stagings, 5-level butterfly reductions, level set-up, the NCC pass) — the
// 11x11 window ran only 1.3x faster than 21x21 for 3.6x less work.  Here one
// staging instruction copies a row for both keypoints, a reduction is 4 levels
// and serves both, and the per-level bookkeeping is shared.
//
// Mapping per half: the window is cut into <= 32 vertical runs of RL rows (RL
// odd), two per lane (run j = lane16 is the .x half and run j = lane16 + 16
// the .y half of every packed float2).  Each half has its own shared-memory
// tile (patch + gradient grids); the two tiles start 16 banks apart and the
// patch pitch P satisfies RL*P == WIN (mod 32), so run j of half h starts in
// bank (base_h + j) mod 32: both halves' run-addressed loads hit 32 distinct
// banks.  Control flow: the two keypoints can need different numbers of levels
// and Gauss-Newton steps; every loop runs until BOTH halves are done and a
// finished half's updates are masked (its lanes still execute), so the warp
// pays max(steps) of its pair.
#include "common.cuh"

namespace v2d {
namespace {

constexpr int kGP = 16;         // gradient-grid row pitch (floats); lane16 = grid column
constexpr int kPairMaxWin = 13; // window edge + 3 <= 16 lanes

constexpr int run_len16(int win) {
  int rl = (win * win + 31) / 32;
  if (rl < 1) rl = 1;
  while (win * ((win + rl - 1) / rl) > 32 || rl % 2 == 0) ++rl;
  return rl;
}
constexpr int inv_mod32p(int a) {
  for (int x = 1; x < 32; x += 2)
    if ((a * x) % 32 == 1) return x;
  return 0;
}
__host__ __device__ constexpr int pmargin(int win) { return (15 - win) / 2 < 1 ? (15 - win) / 2 : 1; }
__host__ __device__ constexpr int prows(int win) {
  return win + 3 > win + 1 + 2 * pmargin(win) ? win + 3 : win + 1 + 2 * pmargin(win);
}
// smallest P >= 16 (a staged row is 16 columns wide: one per lane of the half)
// with RL * P == win (mod 32)
constexpr int ppitch(int win) {
  const int t = (win * inv_mod32p(run_len16(win))) % 32;
  return t >= 16 ? t : t + 32;
}

template <int WIN>
struct PSmem {
  static constexpr int P = ppitch(WIN);
  static constexpr int PATCH = prows(WIN) * P;
  static constexpr int GRID = (WIN + 1) * kGP;
  static constexpr int RAW = PATCH + 2 * GRID;
  // per-half tile; half 1 starts 16 banks after half 0
  static constexpr int HALF = ((RAW + 31) / 32) * 32 + 16;
  static constexpr int TOTAL = 2 * HALF;
};

template <int WIN>
struct PTmpl {
  static constexpr int RL = run_len16(WIN);
  static constexpr int K = (WIN + RL - 1) / RL;
  static constexpr bool kExact = K * RL == WIN;
  float2 T[RL], TX[RL], TY[RL];
};

struct PPlane {
  const void* base;
  int64_t pitch;  // elements
  int W, H;
  int u8;
};

__device__ __forceinline__ int pclampi(int v, int lo, int hi) { return min(max(v, lo), hi); }
__device__ __forceinline__ float2 pf2(float a, float b) { return make_float2(a, b); }
__device__ __forceinline__ float2 padd2(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 psub2(float2 a, float2 b) {
  return __fadd2_rn(a, make_float2(-b.x, -b.y));
}
__device__ __forceinline__ float2 pfma2(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }
__device__ __forceinline__ float2 pmul2(float2 a, float2 b) { return __fmul2_rn(a, b); }

// butterfly over the 16 lanes of each half (both halves at once; lanes of a half
// end with identical sums, so per-half control flow stays half-uniform)
__device__ __forceinline__ float2 half_sum2(float2 v) {
#pragma unroll
  for (int m = 8; m > 0; m >>= 1) {
    const float2 o = make_float2(__shfl_xor_sync(kFullMask, v.x, m),
                                 __shfl_xor_sync(kFullMask, v.y, m));
    v = padd2(v, o);
  }
  return v;
}

__device__ __forceinline__ float pu8_to_f32(unsigned v) {
  float f;
  asm("cvt.rn.f32.u32 %0, %1;" : "=f"(f) : "r"(v));
  return f;
}

// Stage rows [oy, oy+nr) x columns [ox, ox+16) of this half's plane (clamp-to-edge)
// into its tile (lane16 = column); `on` = this half participates.  All lanes of
// the warp execute the loop (one instruction stages a row of both halves).
template <int NR>
__device__ __forceinline__ void pstage(float* __restrict__ sp, int kPitch, const PPlane& pl,
                                       int ox, int oy, bool on) {
  const int lane16 = threadIdx.x & 15;
  __syncwarp();
  // clamp-to-edge rows by pointer stepping: start at the clamped first row and
  // advance one pitch only while the next row is inside (no per-row clamp/multiply)
  const unsigned hm1 = (unsigned)(pl.H - 1);
  if (pl.u8) {
    const uint8_t* p = reinterpret_cast<const uint8_t*>(pl.base) + pclampi(ox + lane16, 0, pl.W - 1) +
                       (int64_t)pclampi(oy, 0, pl.H - 1) * pl.pitch;
    unsigned v[NR];
#pragma unroll
    for (int r = 0; r < NR; ++r) {
      v[r] = on ? __ldg(p) : 0u;
      if ((unsigned)(oy + r) < hm1) p += pl.pitch;
    }
#pragma unroll
    for (int r = 0; r < NR; ++r)
      if (on) sp[r * kPitch + lane16] = pu8_to_f32(v[r]);
  } else {
    const float* p = reinterpret_cast<const float*>(pl.base) + pclampi(ox + lane16, 0, pl.W - 1) +
                     (int64_t)pclampi(oy, 0, pl.H - 1) * pl.pitch;
#pragma unroll
    for (int r = 0; r < NR; ++r) {
      if (on) {
        const unsigned d = (unsigned)__cvta_generic_to_shared(sp + r * kPitch + lane16);
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(d), "l"(p) : "memory");
      }
      if ((unsigned)(oy + r) < hm1) p += pl.pitch;
    }
    asm volatile("cp.async.wait_all;\n" ::: "memory");
  }
  __syncwarp();
}

template <int WIN>
__device__ __forceinline__ void prun_of(int j, int& col, int& r0, int& skip) {
  constexpr int RL = PTmpl<WIN>::RL, K = PTmpl<WIN>::K;
  const bool used = j < WIN * K;
  if (!used) j = WIN * K - 1;
  const int k = j / WIN;
  col = j - k * WIN;
  r0 = min(k * RL, WIN - RL);
  skip = used ? k * RL - r0 : RL;
}

template <int WIN>
struct PRuns {
  static constexpr int P = PSmem<WIN>::P;
  int offx, offy, skx, sky;
  __device__ __forceinline__ PRuns() {
    const int lane16 = threadIdx.x & 15;
    int cx, rx, cy, ry;
    prun_of<WIN>(lane16, cx, rx, skx);
    prun_of<WIN>(lane16 + 16, cy, ry, sky);
    offx = rx * P + cx;
    offy = ry * P + cy;
  }
  __device__ __forceinline__ float2 mask(int p) const {
    return pf2(p >= skx ? 1.f : 0.f, p >= sky ? 1.f : 0.f);
  }
  __device__ __forceinline__ float sum2(float2 v) const {
    if (PTmpl<WIN>::kExact) return fmaf(v.y, sky == 0 ? 1.f : 0.f, skx == 0 ? v.x : 0.f);
    return v.x + v.y;
  }
};

// D7 template (same arithmetic as klt.cu build_template); P[r][c] = I~(ix-R-1+c, iy-R-1+r).
template <int WIN>
__device__ __forceinline__ void pbuild_template(const float* __restrict__ P, float* __restrict__ GX,
                                                float* __restrict__ GY, int ix, int iy, float ax,
                                                float ay, int W, int H, const PRuns<WIN>& ru,
                                                PTmpl<WIN>& t) {
  constexpr int R = (WIN - 1) / 2;
  constexpr int RL = PTmpl<WIN>::RL;
  constexpr int kPitch = PSmem<WIN>::P;
  const int lane16 = threadIdx.x & 15;
  const float* Px = P + ru.offx;
  const float* Py = P + ru.offy;
  const bool interior = (ix - R >= 0) && (ix + R + 1 <= W - 1) && (iy - R >= 0) && (iy + R + 1 <= H - 1);
  // both halves execute both forms (results selected per half): the halves stay
  // converged for the shuffles that follow
  PTmpl<WIN> ti;
  {
    const float2 wx = pf2(ax, ax), wy = pf2(ay, ay), two = pf2(2.f, 2.f);
    float2 dx1 = pf2(0.f, 0.f), dx2 = dx1, hs1 = dx1, hs2 = dx1, h1 = dx1, h2 = dx1;
    float2 vprev = dx1, eprev = dx1;
#pragma unroll
    for (int q = 0; q < RL + 3; ++q) {
      const float* ra = Px + q * kPitch;
      const float* rb = Py + q * kPitch;
      const float2 p0 = pf2(ra[0], rb[0]), p1 = pf2(ra[1], rb[1]);
      const float2 p2 = pf2(ra[2], rb[2]), p3 = pf2(ra[3], rb[3]);
      const float2 l01 = pfma2(wx, psub2(p1, p0), p0);
      const float2 h = pfma2(wx, psub2(p2, p1), p1);
      const float2 l23 = pfma2(wx, psub2(p3, p2), p2);
      const float2 dx = psub2(l23, l01);
      const float2 hs = pfma2(two, h, padd2(l01, l23));
      const float2 vq = pfma2(two, dx2, padd2(dx1, dx));
      const float2 eq = psub2(hs, hs1);
      if (q >= 3) {
        const int pq = q - 3;
        ti.T[pq] = pfma2(wy, psub2(h2, h1), h1);
        ti.TX[pq] = pfma2(wy, psub2(vq, vprev), vprev);
        ti.TY[pq] = pfma2(wy, psub2(eq, eprev), eprev);
      }
      vprev = vq;
      eprev = eq;
      dx1 = dx2; dx2 = dx;
      hs1 = hs2; hs2 = hs;
      h1 = h2; h2 = h;
    }
  }
  // border form: clamped gradient grids (grid point (c, g) <-> pixel (ix-R+c, iy-R+g))
  const int c = min(lane16, WIN);
  const int lc = pclampi(ix - R + c, 0, W - 1) - (ix - R - 1);
  const float* col = P + lc;
  auto row_ds = [&](int r, float& d, float& sm) {
    const float* q = col + r * kPitch;
    const float a = q[-1], m = q[0], e = q[1];
    d = e - a;
    sm = fmaf(2.f, m, a + e);
  };
  const unsigned any_border = __ballot_sync(kFullMask, !interior);
  if (any_border) {  // warp-uniform
    int lr = pclampi(iy - R, 0, H - 1) - (iy - R - 1);
    float d0, s0, d1, s1, d2, s2;
    row_ds(lr - 1, d0, s0);
    row_ds(lr, d1, s1);
    row_ds(lr + 1, d2, s2);
    for (int g = 0; g <= WIN; ++g) {
      const int lrg = pclampi(iy - R + g, 0, H - 1) - (iy - R - 1);
      if (lrg != lr) {
        d0 = d1;
        s0 = s1;
        d1 = d2;
        s1 = s2;
        row_ds(lrg + 1, d2, s2);
        lr = lrg;
      }
      GX[g * kGP + lane16] = fmaf(2.f, d1, d0 + d2);
      GY[g * kGP + lane16] = s2 - s0;
    }
    __syncwarp();
    const float2 wx = pf2(ax, ax), wy = pf2(ay, ay);
    int gcx, grx, gcy, gry, sk;
    prun_of<WIN>(lane16, gcx, grx, sk);
    prun_of<WIN>(lane16 + 16, gcy, gry, sk);
    const int gox = grx * kGP + gcx, goy = gry * kGP + gcy;
    auto hrow = [&](const float* base, int ox, int oy, int pitch, int row, int cc) {
      const float* bx = base + ox + row * pitch + cc;
      const float* by = base + oy + row * pitch + cc;
      const float2 a0 = pf2(bx[0], by[0]);
      const float2 a1 = pf2(bx[1], by[1]);
      return pfma2(wx, psub2(a1, a0), a0);
    };
    float2 hp = hrow(P, ru.offx, ru.offy, kPitch, 1, 1);
    float2 hx = hrow(GX, gox, goy, kGP, 0, 0);
    float2 hy = hrow(GY, gox, goy, kGP, 0, 0);
#pragma unroll
    for (int p = 0; p < RL; ++p) {
      const float2 np = hrow(P, ru.offx, ru.offy, kPitch, p + 2, 1);
      const float2 nx = hrow(GX, gox, goy, kGP, p + 1, 0);
      const float2 ny = hrow(GY, gox, goy, kGP, p + 1, 0);
      t.T[p] = interior ? ti.T[p] : pfma2(wy, psub2(np, hp), hp);
      t.TX[p] = interior ? ti.TX[p] : pfma2(wy, psub2(nx, hx), hx);
      t.TY[p] = interior ? ti.TY[p] : pfma2(wy, psub2(ny, hy), hy);
      hp = np;
      hx = nx;
      hy = ny;
    }
  } else {
#pragma unroll
    for (int p = 0; p < RL; ++p) {
      t.T[p] = ti.T[p];
      t.TX[p] = ti.TX[p];
      t.TY[p] = ti.TY[p];
    }
  }
  if (!PTmpl<WIN>::kExact) {
#pragma unroll
    for (int p = 0; p < RL; ++p) {
      const float2 m = ru.mask(p);
      t.T[p] = pmul2(t.T[p], m);
      t.TX[p] = pmul2(t.TX[p], m);
      t.TY[p] = pmul2(t.TY[p], m);
    }
  }
}

template <int WIN>
__device__ __forceinline__ float2 pgn_rhs(const float* __restrict__ JP, int lc0, int lr0, float bx,
                                          float by, const PRuns<WIN>& ru, const PTmpl<WIN>& t) {
  constexpr int RL = PTmpl<WIN>::RL;
  constexpr int kPitch = PSmem<WIN>::P;
  const float* base = JP + lr0 * kPitch + lc0;
  const float* bxp = base + ru.offx;
  const float* byp = base + ru.offy;
  const float2 wx = pf2(bx, bx), wy = pf2(by, by);
  auto hrow = [&](int r) {
    const float2 a0 = pf2(bxp[r * kPitch], byp[r * kPitch]);
    const float2 a1 = pf2(bxp[r * kPitch + 1], byp[r * kPitch + 1]);
    return pfma2(wx, psub2(a1, a0), a0);
  };
  float2 h = hrow(0);
  float2 ax = pf2(0.f, 0.f), ay = pf2(0.f, 0.f);
  // e = T - [(1-by) h(p) + by h(p+1)] as two FMAs (klt.cu V2D_GN_FOLD) is NOT used
  // here: with 7x7 windows (n = 49) its different rounding flipped one track's NCC
  // decision outside the parity bands (test_klt_stream_windows[7-5])
#if V2D_GN_FOLD_PAIR
  const float2 nw0 = pf2(by - 1.0f, by - 1.0f), nw1 = pf2(-by, -by);
#endif
#pragma unroll
  for (int p = 0; p < RL; ++p) {
    const float2 hn = hrow(p + 1);
#if V2D_GN_FOLD_PAIR
    const float2 e = pfma2(nw1, hn, pfma2(nw0, h, t.T[p]));
#else
    const float2 e = psub2(t.T[p], pfma2(wy, psub2(hn, h), h));
#endif
    ax = pfma2(e, t.TX[p], ax);
    ay = pfma2(e, t.TY[p], ay);
    h = hn;
  }
  return pf2(ru.sum2(ax), ru.sum2(ay));
}

// NCC moments (sum S', sum S'^2, sum T'S'), T' = T - m (m = template mean, the second
// pass of the two-pass NCC), over the valid slots.  kExactRef = false (every level):
// S' = S - m with the vertical lerp folded into two FMAs.  kExactRef = true (only when
// the first pass is ill-conditioned, see ncc_gate): S' = S - S(0,0), S centred by one of
// its own samples (window pixel (0,0): run 0, row 0, held by the first lane) with the
// unfolded lerp, so a flat S has exactly zero deviations and NCC 0 — the oracle's
// two-pass value (reading #14); centred by m, a flat S left rounding noise that could
// pass the gate.
template <int WIN, bool kExactRef>
__device__ __forceinline__ float3 pncc_moments(const float* __restrict__ JP, int lc0, int lr0,
                                              float bx, float by, float m, const PRuns<WIN>& ru,
                                              const PTmpl<WIN>& t) {
  constexpr int RL = PTmpl<WIN>::RL;
  constexpr int kPitch = PSmem<WIN>::P;
  const float* base = JP + lr0 * kPitch + lc0;
  const float* bxp = base + ru.offx;
  const float* byp = base + ru.offy;
  const float2 wx = pf2(bx, bx), wy = pf2(by, by), mm = pf2(m, m);
  auto hrow = [&](int r) {
    const float2 a0 = pf2(bxp[r * kPitch], byp[r * kPitch]);
    const float2 a1 = pf2(bxp[r * kPitch + 1], byp[r * kPitch + 1]);
    return pfma2(wx, psub2(a1, a0), a0);
  };
  float2 h = hrow(0), hn = hrow(1);
  float2 sr = pf2(0.f, 0.f), S0 = sr;
  if (kExactRef) {
    S0 = pfma2(wy, psub2(hn, h), h);
    const float sref = __shfl_sync(kFullMask, S0.x, 0, 16);
    sr = pf2(sref, sref);
  }
  const float2 w0 = pf2(1.0f - by, 1.0f - by), nm = pf2(-m, -m);
  float2 s1 = pf2(0.f, 0.f), s2 = pf2(0.f, 0.f), st = pf2(0.f, 0.f);
#pragma unroll
  for (int p = 0; p < RL; ++p) {
    if (p > 0) hn = hrow(p + 1);
    float2 S;
    if (kExactRef)
      S = psub2(p == 0 ? S0 : pfma2(wy, psub2(hn, h), h), sr);
    else
      S = pfma2(wy, hn, pfma2(w0, h, nm));  // S - m = (1-by) h(p) + by h(p+1) - m
    if (!PTmpl<WIN>::kExact) S = pmul2(S, ru.mask(p));
    s1 = padd2(s1, S);
    s2 = pfma2(S, S, s2);
    st = pfma2(psub2(t.T[p], mm), S, st);
    h = hn;
  }
  return make_float3(ru.sum2(s1), ru.sum2(s2), ru.sum2(st));
}

// klt.cu ncc_value for a half-warp (the centre sample is a half-width shuffle).
template <int WIN>
__device__ __forceinline__ float pncc_value(const float* __restrict__ JP, int lc0, int lr0,
                                            float bx, float by, float tmean, float Stt,
                                            const PRuns<WIN>& ru, const PTmpl<WIN>& t) {
  constexpr float kInvN = 1.0f / (float)(WIN * WIN);
  const float3 mo = pncc_moments<WIN, true>(JP, lc0, lr0, bx, by, tmean, ru, t);
  const float2 r1 = half_sum2(pf2(mo.x, mo.y));
  const float r2 = half_sum2(pf2(mo.z, 0.f)).x;
  const float Sss = r1.y - r1.x * r1.x * kInvN;
  const float den2 = Stt * Sss;
  return den2 > 0.0f ? r2 * rsqrtf(den2) : 0.0f;
}

struct PState {
  int status;  // V2D_TRACKED while alive
  float ncc;
  int steps, levels;
  float dx, dy;
};

// One pyramid level of D7 for the half's keypoint (both halves in lockstep).
template <int WIN, bool kEachStep>
__device__ __forceinline__ void ptrack_level(float* __restrict__ sp, const PPlane& I,
                                             const PPlane& J, const int L, const float cx,
                                             const float cy, const KltArgs& a, PState& o) {
  constexpr int R = (WIN - 1) / 2;
  constexpr int N = WIN * WIN;
  constexpr int M = pmargin(WIN);
  constexpr int SZ = WIN + 1 + 2 * M;
  constexpr int RL = PTmpl<WIN>::RL;
  static_assert(WIN + 3 <= 16 && SZ <= 16, "window too large for a half warp");
  static_assert(WIN * PTmpl<WIN>::K <= 32, "two runs per lane");
  float* GX = sp + PSmem<WIN>::PATCH;
  float* GY = GX + PSmem<WIN>::GRID;
  const bool alive = o.status == V2D_TRACKED;

  const PRuns<WIN> ru;
  PTmpl<WIN> t;
  {
    const float fcx = floorf(cx), fcy = floorf(cy);
    const int ix = (int)fcx, iy = (int)fcy;
    pstage<WIN + 3>(sp, PSmem<WIN>::P, I, ix - R - 1, iy - R - 1, alive);
    pbuild_template<WIN>(sp, GX, GY, ix, iy, cx - fcx, cy - fcy, I.W, I.H, ru, t);
  }
  if (alive) o.levels++;
  float2 axx = pf2(0.f, 0.f), axy = axx, ayy = axx, ats = axx;
#pragma unroll
  for (int p = 0; p < RL; ++p) {
    axx = pfma2(t.TX[p], t.TX[p], axx);
    axy = pfma2(t.TX[p], t.TY[p], axy);
    ayy = pfma2(t.TY[p], t.TY[p], ayy);
    ats = padd2(t.T[p], ats);
  }
  float2 g01 = pf2(ru.sum2(axx), ru.sum2(axy));
  float2 g2s = pf2(ru.sum2(ayy), ru.sum2(ats));
  g01 = half_sum2(g01);
  g2s = half_sum2(g2s);
  const float gxx = g01.x, gxy = g01.y, gyy = g2s.x;
  const float det = (float)((double)gxx * gyy - (double)gxy * gxy);
  const float dg = gxx - gyy;
  const float lmax = 0.5f * (gxx + gyy + sqrtf(fmaf(dg, dg, 4.0f * gxy * gxy)));
  const bool finite = isfinite(gxx) && isfinite(gxy) && isfinite(gyy) && isfinite(det);
  const bool cond_ok = finite && (det > 0.0f) && !(det < a.min_eig * (float)N * lmax * 64.0f);
  bool active = alive && cond_ok;   // this half runs Gauss-Newton at this level
  bool run_ncc = active;            // and the per-level NCC gate
  if (alive && !cond_ok && L == 0) o.status = V2D_LOST_SMALL_EIG;
  const float inv_det = cond_ok ? 8.0f / det : 0.0f;
  const float i00 = gyy * inv_det, i01 = -gxy * inv_det, i11 = gxx * inv_det;
  // IEEE division: a flat template's mean is exact, so T - mean is exactly 0 there
  // (the oracle's NCC is then 0/0 -> 0; a rounded mean made Stt spuriously > 0)
  const float tmean = exact_mean(g2s.y, (float)N);
  float2 q = pf2(0.f, 0.f);
#pragma unroll
  for (int p = 0; p < RL; ++p) {
    float2 d = psub2(t.T[p], pf2(tmean, tmean));
    if (!PTmpl<WIN>::kExact) d = pmul2(d, ru.mask(p));
    q = pfma2(d, d, q);
  }
  const float Stt = half_sum2(pf2(ru.sum2(q), 0.f)).x;

  // ---------------- Gauss-Newton iterations (next frame) --------------------
  const float xmax = (float)(J.W - 1), ymax = (float)(J.H - 1);
  int jx0 = 0, jy0 = 0;
  bool staged = false;
  float dx = o.dx, dy = o.dy;
  // (re)stage the search patch of every half that needs it; returns the window origin
  auto locate = [&](float qx, float qy, bool on, int& lc0, int& lr0, float& bx, float& by) {
    const float fqx = floorf(qx), fqy = floorf(qy);
    const int ixq = (int)fqx, iyq = (int)fqy;
    bx = qx - fqx;
    by = qy - fqy;
    lc0 = ixq - R - jx0;
    lr0 = iyq - R - jy0;
    const bool need = on && (!staged || lc0 < 0 || lc0 > 2 * M || lr0 < 0 || lr0 > 2 * M);
    if (__any_sync(kFullMask, need)) {
      if (need) {
        jx0 = ixq - R - M;
        jy0 = iyq - R - M;
      }
      pstage<SZ>(sp, PSmem<WIN>::P, J, jx0, jy0, need);
      if (need) {
        staged = true;
        lc0 = M;
        lr0 = M;
      }
    }
    if (!on) {  // keep an idle half's reads inside its tile
      lc0 = M;
      lr0 = M;
    }
  };
  const float eps2 = a.eps * a.eps;
  for (int it = 1; it <= a.iters; ++it) {
    if (!__any_sync(kFullMask, active)) break;
    int lc0, lr0;
    float bx, by;
    locate(cx + dx, cy + dy, active, lc0, lr0, bx, by);
    const float2 b = half_sum2(pgn_rhs<WIN>(sp, lc0, lr0, bx, by, ru, t));
    const float ex = fmaf(i00, b.x, i01 * b.y);
    const float ey = fmaf(i01, b.x, i11 * b.y);
    if (active) {
      dx += ex;
      dy += ey;
      o.steps++;
      const float nx = cx + dx, ny = cy + dy;
      const bool inside = nx >= 0.0f && nx <= xmax && ny >= 0.0f && ny <= ymax;
      if (!inside) {
        active = false;
        if (L > 0) {
          dx -= ex;
          dy -= ey;
        } else {
          o.status = V2D_LOST_OOB;
          run_ncc = false;
        }
      }
    }
    if (kEachStep) {  // variant f3: NCC after every update
      int lc0n, lr0n;
      float bxn, byn;
      locate(cx + dx, cy + dy, active, lc0n, lr0n, bxn, byn);
      const float nv = pncc_value<WIN>(sp, lc0n, lr0n, bxn, byn, tmean, Stt, ru, t);
      if (active) {
        o.ncc = nv;
        if (o.ncc < a.ncc_min) {
          o.status = V2D_LOST_NCC;
          active = false;
          run_ncc = false;
        }
      }
    }
    if (active && fmaf(ex, ex, ey * ey) < eps2) active = false;
  }
  // ---------------- per-level NCC gate --------------------------------------
  if (__any_sync(kFullMask, run_ncc)) {
    int lc0, lr0;
    float bx, by;
    locate(cx + dx, cy + dy, run_ncc, lc0, lr0, bx, by);
    const float nv = pncc_value<WIN>(sp, lc0, lr0, bx, by, tmean, Stt, ru, t);
    if (run_ncc) {
      o.ncc = nv;
      if (o.ncc < a.ncc_min) o.status = V2D_LOST_NCC;
    }
  }
  if (alive && o.status == V2D_TRACKED && L > 0) {  // also after a coarse-level eig skip
    dx *= 2.0f;
    dy *= 2.0f;
  }
  o.dx = dx;
  o.dy = dy;
}

template <int WIN, bool kEachStep>
#ifndef V2D_PAIR_MINB
#define V2D_PAIR_MINB 16
#endif
__global__ void __launch_bounds__(32, V2D_PAIR_MINB)
klt_pair_kernel(const uint8_t* const* __restrict__ prev_l0, const float* const* __restrict__ prev_pyr,
                const uint8_t* const* __restrict__ next_l0, const float* const* __restrict__ next_pyr,
                int B, Levels lv, KltArgs a, const float* __restrict__ pts,
                const float* __restrict__ guess, const uint8_t* __restrict__ in_status,
                float* __restrict__ out_pos, uint8_t* __restrict__ status, float* __restrict__ ncc,
                int32_t* __restrict__ iters_out, float4* __restrict__ track_list) {
  extern __shared__ __align__(16) float s_mem[];
  const int lane = threadIdx.x & 31, half = lane >> 4;
  const int64_t total = (int64_t)B * a.P;
  const int64_t kp = 2 * (int64_t)blockIdx.x + half;
  const bool exists = kp < total;
  float* sp = s_mem + half * PSmem<WIN>::HALF;
  const int b = exists ? (int)(kp / a.P) : 0;
  const float px = exists ? pts[2 * kp] : -1.0f, py = exists ? pts[2 * kp + 1] : -1.0f;
  constexpr int R = (WIN - 1) / 2;

  PState o{V2D_TRACKED, 0.0f, 0, 0, 0.0f, 0.0f};
  const bool skip = !exists || (in_status && in_status[kp] != 0) || (px == -1.0f && py == -1.0f) ||
                    !isfinite(px) || !isfinite(py);
  if (skip) {
    o.status = V2D_SKIPPED;
  } else if (px < 0.0f || px > (float)(lv.W[0] - 1) || py < 0.0f || py > (float)(lv.H[0] - 1)) {
    o.status = V2D_LOST_OOB;  // reading #16
  } else if (guess) {
    const float s = 1.0f / (float)(1 << (lv.n - 1));
    o.dx = guess[2 * kp] * s;
    o.dy = guess[2 * kp + 1] * s;
  }
  for (int L = lv.n - 1; L >= 0; --L) {
    if (!__any_sync(kFullMask, o.status == V2D_TRACKED)) break;
    const float scale = __int_as_float((127 - L) << 23);  // 2^-L exactly
    const float cx = (px + 0.5f) * scale - 0.5f;
    const float cy = (py + 0.5f) * scale - 0.5f;
    PPlane I, J;
    if (L == 0) {
      I = PPlane{prev_l0[b], a.l0_pitch, lv.W[0], lv.H[0], 1};
      J = PPlane{next_l0[b], a.l0_pitch, lv.W[0], lv.H[0], 1};
    } else {
      I = PPlane{prev_pyr[b] + lv.offset[L], lv.pitch[L], lv.W[L], lv.H[L], 0};
      J = PPlane{next_pyr[b] + lv.offset[L], lv.pitch[L], lv.W[L], lv.H[L], 0};
    }
    ptrack_level<WIN, kEachStep>(sp, I, J, L, cx, cy, a, o);
  }
  float ox = -1.0f, oy = -1.0f;
  if (o.status == V2D_TRACKED) {
    const float qx = px + o.dx, qy = py + o.dy;
    const int W = lv.W[0], H = lv.H[0];
    if (!(qx >= R && qx <= W - 1 - R && qy >= R && qy <= H - 1 - R)) {
      o.status = V2D_LOST_OOB;
    } else {
      ox = qx;
      oy = qy;
    }
  }
  if ((lane & 15) == 0 && exists) {
    out_pos[2 * kp] = ox;
    out_pos[2 * kp + 1] = oy;
    status[kp] = (uint8_t)o.status;
    if (ncc) ncc[kp] = o.ncc;
    if (iters_out) iters_out[kp] = o.steps | (o.levels << 24);
    if (track_list) track_list[kp] = make_float4(ox, oy, (float)o.status, o.ncc);
  }
}

template <int WIN>
void launch_pair_win(const uint8_t* const* prev_l0, const float* const* prev_pyr,
                     const uint8_t* const* next_l0, const float* const* next_pyr, int B,
                     const Levels& lv, const KltArgs& a, const float* pts, const float* guess,
                     const uint8_t* in_status, float* out_pos, uint8_t* status, float* ncc,
                     int32_t* iters_out, float4* track_list, cudaStream_t st) {
  const int64_t kps = (int64_t)B * a.P;
  const unsigned blocks = (unsigned)((kps + 1) / 2);
  constexpr int smem = PSmem<WIN>::TOTAL * (int)sizeof(float);
  static_assert(smem <= 48 * 1024, "pair tile exceeds the default dynamic smem limit");
  if (a.flags & V2D_KLT_NCC_EACH_STEP)
    klt_pair_kernel<WIN, true><<<blocks, 32, smem, st>>>(prev_l0, prev_pyr, next_l0, next_pyr, B,
                                                         lv, a, pts, guess, in_status, out_pos,
                                                         status, ncc, iters_out, track_list);
  else
    klt_pair_kernel<WIN, false><<<blocks, 32, smem, st>>>(prev_l0, prev_pyr, next_l0, next_pyr, B,
                                                          lv, a, pts, guess, in_status, out_pos,
                                                          status, ncc, iters_out, track_list);
}

}  // namespace

bool klt_pair_supported(int win) { return win >= 3 && win <= kPairMaxWin && (win & 1); }

int launch_klt_pair(const uint8_t* const* prev_l0, const float* const* prev_pyr,
                    const uint8_t* const* next_l0, const float* const* next_pyr, int B,
                    const Levels& lv, const KltArgs& a, const float* pts, const float* guess,
                    const uint8_t* in_status, float* out_pos, uint8_t* status, float* ncc,
                    int32_t* iters_out, float* track_list, cudaStream_t st) {
  if (B == 0 || a.P == 0) return V2D_OK;
#define V2D_PAIR_CASE(w)                                                                  \
  case w:                                                                                 \
    launch_pair_win<w>(prev_l0, prev_pyr, next_l0, next_pyr, B, lv, a, pts, guess,        \
                       in_status, out_pos, status, ncc, iters_out,                        \
                       reinterpret_cast<float4*>(track_list), st);                        \
    break;
  switch (a.win) {
    V2D_PAIR_CASE(3)
    V2D_PAIR_CASE(5)
    V2D_PAIR_CASE(7)
    V2D_PAIR_CASE(9)
    V2D_PAIR_CASE(11)
    V2D_PAIR_CASE(13)
    default:
      return V2D_EINVAL;
  }
#undef V2D_PAIR_CASE
  return cudaGetLastError() == cudaSuccess ? V2D_OK : V2D_ECUDA;
}

}  // namespace v2d
