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
// B200 mapping (DESIGN.md §5 K3): one WARP per keypoint slot.  Per level the
// warp stages a clamped 32-wide patch of the previous level (template) and then
// of the next level (with a margin of M px for the Gauss-Newton motion) into its
// own shared-memory tile, so the inner loops have no clamping or address
// arithmetic (immediate smem offsets).  The window is cut into vertical runs of
// RL rows dealt two per lane (Tmpl: 63 runs of 7 rows for 21x21, 98% of the
// lane slots used); T, Tx, Ty stay in registers as float2 (run .x, run .y) and
// every inner loop runs on packed fp32x2 FMA (__ffma2_rn / FFMA2, new on
// sm_100).  The patch pitch puts the 32 runs of a half-warp in 32 distinct
// banks.  G, b and the NCC moments are butterfly-reduced (bit-identical in every
// lane -> warp-uniform control flow).
#include "common.cuh"

#ifdef V2D_KLT_STATS  // debug builds only: event counters for the cost model
__device__ unsigned long long g_klt_stats[16];
#define KSTAT(i) \
  do {           \
    if ((threadIdx.x & 31) == 0) atomicAdd(&g_klt_stats[i], 1ull); \
  } while (0)
#else
#define KSTAT(i) \
  do {           \
  } while (0)
#endif

#ifdef V2D_KLT_CYC  // debug builds only: phase cycles (warp-elapsed SM clocks) kept in
// per-warp registers and flushed once per warp into one of 64 slots (no atomics inside
// the timed phases):
// 0 template staging, 1 template build + G + eigen test + Stt, 2 search staging,
// 3 Gauss-Newton steps (staging excluded), 4 NCC gate, 5 whole warp
__device__ unsigned long long g_klt_cyc[64][8];
#define KCLK(v) const unsigned v = (unsigned)clock()
#define KCYC(ph, t0) kc[ph] += (unsigned)clock() - (t0)
#define KCYC_DECL unsigned kc[8] = {0, 0, 0, 0, 0, 0, 0, 0}
#define KCYC_PARAM , unsigned* kc
#define KCYC_ARG , kc
#define KCYC_FLUSH                                                              \
  do {                                                                          \
    if ((threadIdx.x & 31) == 0)                                                \
      for (int i = 0; i < 6; ++i) atomicAdd(&g_klt_cyc[blockIdx.x & 63][i], (unsigned long long)kc[i]); \
  } while (0)
#else
#define KCLK(v) \
  do {          \
  } while (0)
#define KCYC(ph, t0) \
  do {               \
  } while (0)
#define KCYC_DECL \
  do {            \
  } while (0)
#define KCYC_PARAM
#define KCYC_ARG
#define KCYC_FLUSH \
  do {             \
  } while (0)
#endif

namespace v2d {
namespace {

// One warp per CTA (16 CTAs/SM at 128 registers): the same occupancy as larger CTAs but
// finer-grained scheduling — same-box A/B: 4 -> 2 -> 1 warps per CTA each ~1.5 % faster.
constexpr int kWarps = 1;
constexpr int kThreads = 32 * kWarps;
constexpr int kGP = 32;  // gradient-grid row pitch (floats); lane = grid column

// Window run layout (see Tmpl below): run length RL (odd, so that the patch
// pitch below exists) = the shortest with WIN * ceil(WIN/RL) <= 64 runs.
constexpr int run_len(int win) {
  int rl = (win * win + 63) / 64;
  while (win * ((win + rl - 1) / rl) > 64 || rl % 2 == 0) ++rl;
  return rl;
}
constexpr int inv_mod32(int a) {
  for (int x = 1; x < 32; x += 2)
    if ((a * x) % 32 == 1) return x;
  return 0;
}
// search margin (px) staged around the level start point; 1 measured best
// (re-staging when the iterate leaves it is rarer than it is costly)
__host__ __device__ constexpr int search_margin(int win) { return (31 - win) / 2 < 1 ? (31 - win) / 2 : 1; }
// rows of the patch tile: the template patch (win+3) or the search patch
__host__ __device__ constexpr int patch_rows(int win) {
  return win + 3 > win + 1 + 2 * search_margin(win) ? win + 3 : win + 1 + 2 * search_margin(win);
}
constexpr int tile_floats(int win, int pitch) {
  return patch_rows(win) * pitch + 2 * (win + 1) * kGP;
}
// Patch row pitch: RL * P == WIN (mod 32) puts run j (column-major) in bank
// j mod 32, so the 32 lanes of every run-addressed LDS hit 32 distinct banks;
// 32 (bank conflicts) if that tile would not fit 16 warps per SM.
constexpr int patch_pitch(int win) {
  const int p = 32 + (win * inv_mod32(run_len(win))) % 32;
  return 64 * tile_floats(win, p) + 4 * 1024 <= 228 * 1024 ? p : 32;
}

// Per-warp shared memory: one 32-row patch (template source, then the
// next-level search patch) + the two (WIN+1)-row gradient grids of the template.
template <int WIN>
struct Smem {
  static constexpr int P = patch_pitch(WIN);
  static constexpr int PATCH = patch_rows(WIN) * P;
  static constexpr int GRID = (WIN + 1) * kGP;
  static constexpr int SCRATCH = 32 * 36 / 4;  // u8 staging bytes (shares the grids)
  static constexpr int TOTAL = PATCH + (2 * GRID > SCRATCH ? 2 * GRID : SCRATCH);
};

struct Plane {
  const void* base;
  int64_t pitch;  // elements
  int W, H;
  int u8;         // 1: uint8 L0 frame, 0: fp32 pyramid level
};

__device__ __forceinline__ int clampi(int v, int lo, int hi) { return min(max(v, lo), hi); }

__device__ __forceinline__ float2 f2(float a, float b) { return make_float2(a, b); }
__device__ __forceinline__ float2 add2(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 sub2(float2 a, float2 b) {
  return __fadd2_rn(a, make_float2(-b.x, -b.y));
}
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }
__device__ __forceinline__ float2 mul2(float2 a, float2 b) { return __fmul2_rn(a, b); }

__device__ __forceinline__ float2 warp_sum2(float2 v) {
#pragma unroll
  for (int m = 16; m > 0; m >>= 1) {
    const float2 o = make_float2(__shfl_xor_sync(kFullMask, v.x, m),
                                 __shfl_xor_sync(kFullMask, v.y, m));
    v = add2(v, o);
  }
  return v;
}

// Stage rows [oy, oy+nr) x columns [ox, ox+32) of a level (clamp-to-edge)
// into a warp patch (lane = column).  fp32 levels use cp.async (LDGSTS: every
// row in flight at once, no registers); the u8 L0 frame is loaded 8 rows deep
// and converted.  The fp32 path is inlined; the larger u8 path stays out of line
// (the kernel is instruction-cache sensitive: inlining it costs +20 %, inlining the
// fp32 path saves 1-3 %, same-box A/B).
__device__ __forceinline__ void cp_async4(float* dst, const float* src) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(d), "l"(src) : "memory");
}

__device__ __forceinline__ void stage_f32(float* __restrict__ sp, int kPitch,
                                       const float* __restrict__ base, int64_t pitch, int W,
                                       int H, int ox, int oy, int nr) {
  const int lane = threadIdx.x & 31;
  const float* col = base + clampi(ox + lane, 0, W - 1);
  __syncwarp();
  if (oy >= 0 && oy + nr <= H) {
    KSTAT(9);
    const float* p = col + (int64_t)oy * pitch;
    for (int r = 0; r < nr; ++r, p += pitch) cp_async4(sp + r * kPitch + lane, p);
  } else {  // clamp-to-edge rows: advance one pitch only while the next row is inside
    KSTAT(10);
    const float* p = col + (int64_t)clampi(oy, 0, H - 1) * pitch;
    for (int r = 0; r < nr; ++r) {
      cp_async4(sp + r * kPitch + lane, p);
      const int y = oy + r;
      if (y >= 0 && y < H - 1) p += pitch;
    }
  }
  asm volatile("cp.async.wait_all;\n" ::: "memory");
  __syncwarp();
}

__device__ __forceinline__ void cp_async4b(uint8_t* dst, const uint8_t* src) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(d), "l"(src) : "memory");
}

// Exact byte -> fp32 as a 32-bit conversion (the compiler narrows (float)u8 to
// I2F.U16, a multi-function-unit instruction; cvt.rn.f32.u32 is I2FP.F32.U32).
__device__ __forceinline__ float u8_to_f32(unsigned v) {
  float f;
  asm("cvt.rn.f32.u32 %0, %1;" : "=f"(f) : "r"(v));
  return f;
}

// u8 rows: windows needing no clamping copy 4-byte aligned words (9 per row,
// 3 rows per instruction) into a byte scratch tile with cp.async and convert
// in shared memory; windows at the border load clamped bytes 8 rows deep.
__device__ __noinline__ void stage_u8(float* __restrict__ sp, int kPitch,
                                      uint8_t* __restrict__ scratch,
                                      const uint8_t* __restrict__ base, int64_t pitch, int W,
                                      int H, int ox, int oy, int nr) {
  const int lane = threadIdx.x & 31;
  __syncwarp();
  const int sh = ox & 3;
  if (ox >= 0 && ox + 32 <= W && oy >= 0 && oy + nr <= H && ox - sh + 36 <= pitch &&
      ((reinterpret_cast<uintptr_t>(base) | (uintptr_t)pitch) & 3) == 0) {
    KSTAT(7);
    constexpr int kSP = 36;  // scratch bytes per row
    const int w = lane % 9, rr = lane / 9;
    const uint8_t* src = base + (int64_t)oy * pitch + (ox - sh) + 4 * w;
    if (lane < 27)
      for (int r = rr; r < nr; r += 3) cp_async4b(scratch + r * kSP + 4 * w, src + r * pitch);
    asm volatile("cp.async.wait_all;\n" ::: "memory");
    __syncwarp();
    const uint8_t* q = scratch + sh + lane;
#pragma unroll 8
    for (int r = 0; r < nr; ++r) sp[r * kPitch + lane] = u8_to_f32(q[r * kSP]);
    __syncwarp();
    return;
  }
  KSTAT(8);
  const uint8_t* __restrict__ col = base + clampi(ox + lane, 0, W - 1);
  for (int r0 = 0; r0 < nr; r0 += 8) {
    unsigned v[8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
      v[i] = r0 + i < nr ? __ldg(col + (int64_t)clampi(oy + r0 + i, 0, H - 1) * pitch) : 0u;
#pragma unroll
    for (int i = 0; i < 8; ++i)
      if (r0 + i < nr) sp[(r0 + i) * kPitch + lane] = u8_to_f32(v[i]);
  }
  __syncwarp();
}

__device__ __forceinline__ void stage(float* __restrict__ sp, int sp_pitch, float* scratch,
                                      const Plane& pl, int ox, int oy, int nr) {
  if (pl.u8)  // byte scratch: the gradient grids behind the patch (free while staging)
    stage_u8(sp, sp_pitch, reinterpret_cast<uint8_t*>(scratch),
             reinterpret_cast<const uint8_t*>(pl.base), pl.pitch, pl.W, pl.H, ox, oy, nr);
  else
    stage_f32(sp, sp_pitch, reinterpret_cast<const float*>(pl.base), pl.pitch, pl.W, pl.H, ox,
              oy, nr);
}

struct LevelOut {
  int status;  // V2D_TRACKED while still alive
  float ncc;   // last evaluated NCC
  int steps;   // Gauss-Newton steps taken
  int levels;  // levels whose template was built
};

// Window run layout.  Every window column is cut into K vertical runs of RL
// rows; run k of column c starts at row min(k*RL, WIN-RL) (the last run is
// shifted up to end on row WIN-1 and its first `skip` rows, which repeat rows
// of the previous run, are masked).  The WIN*K <= 64 runs, in column-major
// order j = k*WIN + c, are dealt to the warp two per lane: run j = lane is the
// .x half and run j = lane+32 the .y half of every packed float2.  A 21x21
// window is 63 runs of 7 rows (448 slots for 441 pixels) where one column per
// lane would need 21 lanes x 22 rows; with the patch pitch P of Smem the 32
// runs of a half sit in 32 distinct banks.
template <int WIN>
struct Tmpl {
  static constexpr int RL = run_len(WIN);
  static constexpr int K = (WIN + RL - 1) / RL;
  static constexpr bool kExact = K * RL == WIN;  // no shifted run: skip is 0 or RL
  float2 T[RL], TX[RL], TY[RL];
};

// Run j -> window column, first window row and first valid slot (RL = unused
// run; it repeats the address of the last run, a broadcast, and is masked).
template <int WIN>
__device__ __forceinline__ void run_of(int j, int& col, int& r0, int& skip) {
  constexpr int RL = Tmpl<WIN>::RL, K = Tmpl<WIN>::K;
  const bool used = j < WIN * K;
  if (!used) j = WIN * K - 1;
  const int k = j / WIN;
  col = j - k * WIN;
  r0 = min(k * RL, WIN - RL);
  skip = used ? k * RL - r0 : RL;
}

// This lane's two runs: patch offsets of the run origins relative to the window
// origin, and the slot masks.
template <int WIN>
struct Runs {
  static constexpr int P = Smem<WIN>::P;
  int offx, offy;  // r0 * P + col
  int skx, sky;
  __device__ __forceinline__ Runs() {
    const int lane = threadIdx.x & 31;
    int cx, rx, cy, ry;
    run_of<WIN>(lane, cx, rx, skx);
    run_of<WIN>(lane + 32, cy, ry, sky);
    offx = rx * P + cx;
    offy = ry * P + cy;
  }
  // per-slot mask; only used when runs are shifted (!kExact): exact layouts keep
  // unmasked slots (an unused run repeats a valid run's values) and mask whole
  // runs once, in the final .x/.y combine (sum2)
  __device__ __forceinline__ float2 mask(int p) const {
    return f2(p >= skx ? 1.f : 0.f, p >= sky ? 1.f : 0.f);
  }
  // this lane's share of a per-slot sum accumulated as (run .x, run .y)
  __device__ __forceinline__ float sum2(float2 v) const {
    if (Tmpl<WIN>::kExact) return fmaf(v.y, sky == 0 ? 1.f : 0.f, skx == 0 ? v.x : 0.f);
    return v.x + v.y;
  }
};

// D7 template at one level from the staged previous-level patch P
// (P[r][c] = I~(ix-R-1+c, iy-R-1+r)).  Gradient grids GX/GY (grid point
// (c, g) <-> pixel (ix-R+c, iy-R+g)) hold the clamp-to-edge Sobel/8 gradient
// IMAGE sampled with clamped coordinates, exactly as the oracle samples it.
// Slot (run, p) is window pixel (col, r0 + p); masked slots are zeroed.
template <int WIN>
__device__ __forceinline__ void build_template(const float* __restrict__ P,
                                               float* __restrict__ GX, float* __restrict__ GY,
                                               int ix, int iy, float ax, float ay, int W, int H,
                                               const Runs<WIN>& ru, Tmpl<WIN>& t) {
  constexpr int R = (WIN - 1) / 2;
  constexpr int RL = Tmpl<WIN>::RL;
  constexpr int kPitch = Smem<WIN>::P;
  const int lane = threadIdx.x & 31;
  const float* Px = P + ru.offx;
  const float* Py = P + ru.offy;
  if ((ix - R >= 0) && (ix + R + 1 <= W - 1) && (iy - R >= 0) && (iy + R + 1 <= H - 1)) {
    // Every grid centre is inside the image, so bilinear(Sobel/8) is the
    // separable 4x4 filter: with patch columns P0..P3 = P[.][u..u+3],
    //   Dx = (1-ax)(P2-P0) + ax(P3-P1)          Hs = (1-ax)S(u+1) + ax S(u+2)
    //   Tx(v) = [(1-ay)V(v) + ay V(v+1)]/8,     V(v) = Dx(v) + 2Dx(v+1) + Dx(v+2)
    //   Ty(v) = [(1-ay)E(v) + ay E(v+1)]/8,     E(v) = Hs(v+2) - Hs(v)
    //   T(v)  = (1-ay)h(v+1) + ay h(v+2),       h = (1-ax)P1 + ax P2
    // swept down each run (v = run row).
    KSTAT(1);
    const float2 wx = f2(ax, ax), wy = f2(ay, ay), two = f2(2.f, 2.f);
    float2 dx1 = f2(0.f, 0.f), dx2 = dx1;   // Dx rows q-2, q-1
    float2 hs1 = dx1, hs2 = dx1;            // Hs rows q-2, q-1
    float2 h1 = dx1, h2 = dx1;              // h rows q-2, q-1
    float2 vprev = dx1, eprev = dx1;
#pragma unroll
    for (int q = 0; q < RL + 3; ++q) {
      const float* ra = Px + q * kPitch;
      const float* rb = Py + q * kPitch;
      const float2 p0 = f2(ra[0], rb[0]), p1 = f2(ra[1], rb[1]);
      const float2 p2 = f2(ra[2], rb[2]), p3 = f2(ra[3], rb[3]);
      // three horizontal lerps serve all three quantities (linearity):
      //   Dx = l23 - l01,  Hs = l01 + 2 l12 + l23,  h = l12
      const float2 l01 = fma2(wx, sub2(p1, p0), p0);
      const float2 h = fma2(wx, sub2(p2, p1), p1);
      const float2 l23 = fma2(wx, sub2(p3, p2), p2);
      const float2 dx = sub2(l23, l01);
      const float2 hs = fma2(two, h, add2(l01, l23));
      // V(q-2) = Dx(q-2) + 2Dx(q-1) + Dx(q),  E(q-2) = Hs(q) - Hs(q-2)
      const float2 vq = fma2(two, dx2, add2(dx1, dx));
      const float2 eq = sub2(hs, hs1);
      if (q >= 3) {
        const int pq = q - 3;
        t.T[pq] = fma2(wy, sub2(h2, h1), h1);
        t.TX[pq] = fma2(wy, sub2(vq, vprev), vprev);  // 8 x bilinear(Sobel/8)
        t.TY[pq] = fma2(wy, sub2(eq, eprev), eprev);
      }
      vprev = vq;
      eprev = eq;
      dx1 = dx2; dx2 = dx;
      hs1 = hs2; hs2 = hs;
      h1 = h2; h2 = h;
    }
  } else {
    // near a border: the gradient image is clamped, so build the clamped
    // gradient grids (grid point (c, g) <-> pixel (ix-R+c, iy-R+g), sampled at
    // the clamped centre; lane = grid column) and interpolate them
    // Separable and sliding down the rows: per patch row the horizontal
    // difference d and [1 2 1] sum s at the lane's clamped column; the clamped
    // centre row lr advances by 0 or 1 per grid row (warp-uniform).  Every value
    // is exact in fp32 (a few multiples of 4^-L below 2^12), so the order of the
    // sums does not matter.
    KSTAT(2);
    const int c = min(lane, WIN);
    const int lc = clampi(ix - R + c, 0, W - 1) - (ix - R - 1);
    const float* col = P + lc;
    auto row_ds = [&](int r, float& d, float& sm) {
      const float* q = col + r * kPitch;
      const float a = q[-1], m = q[0], e = q[1];
      d = e - a;
      sm = fmaf(2.f, m, a + e);
    };
    int lr = clampi(iy - R, 0, H - 1) - (iy - R - 1);
    float d0, s0, d1, s1, d2, s2;  // patch rows lr-1, lr, lr+1
    row_ds(lr - 1, d0, s0);
    row_ds(lr, d1, s1);
    row_ds(lr + 1, d2, s2);
    for (int g = 0; g <= WIN; ++g) {
      const int lrg = clampi(iy - R + g, 0, H - 1) - (iy - R - 1);
      if (lrg != lr) {  // advanced by one row
        d0 = d1;
        s0 = s1;
        d1 = d2;
        s1 = s2;
        row_ds(lrg + 1, d2, s2);
        lr = lrg;
      }
      GX[g * kGP + lane] = fmaf(2.f, d1, d0 + d2);
      GY[g * kGP + lane] = s2 - s0;
    }
    __syncwarp();
    // T slot (v, u) from patch rows v+1, v+2 / cols u+1, u+2; Tx, Ty from grid
    // rows v, v+1 / cols u, u+1 (shared bilinear weights)
    const float2 wx = f2(ax, ax), wy = f2(ay, ay);
    int gcx, grx, gcy, gry, sk;
    run_of<WIN>(lane, gcx, grx, sk);
    run_of<WIN>(lane + 32, gcy, gry, sk);
    const int gox = grx * kGP + gcx, goy = gry * kGP + gcy;  // run origins in the grids
    auto hrow = [&](const float* base, int ox, int oy, int pitch, int row, int col) {
      const float* bx = base + ox + row * pitch + col;
      const float* by = base + oy + row * pitch + col;
      const float2 a0 = f2(bx[0], by[0]);
      const float2 a1 = f2(bx[1], by[1]);
      return fma2(wx, sub2(a1, a0), a0);
    };
    float2 hp = hrow(P, ru.offx, ru.offy, kPitch, 1, 1);
    float2 hx = hrow(GX, gox, goy, kGP, 0, 0);
    float2 hy = hrow(GY, gox, goy, kGP, 0, 0);
#pragma unroll
    for (int p = 0; p < RL; ++p) {
      const float2 np = hrow(P, ru.offx, ru.offy, kPitch, p + 2, 1);
      const float2 nx = hrow(GX, gox, goy, kGP, p + 1, 0);
      const float2 ny = hrow(GY, gox, goy, kGP, p + 1, 0);
      t.T[p] = fma2(wy, sub2(np, hp), hp);
      t.TX[p] = fma2(wy, sub2(nx, hx), hx);
      t.TY[p] = fma2(wy, sub2(ny, hy), hy);
      hp = np;
      hx = nx;
      hy = ny;
    }
  }
  if (!Tmpl<WIN>::kExact) {
#pragma unroll
    for (int p = 0; p < RL; ++p) {
      const float2 m = ru.mask(p);
      t.T[p] = mul2(t.T[p], m);
      t.TX[p] = mul2(t.TX[p], m);
      t.TY[p] = mul2(t.TY[p], m);
    }
  }
}

// sum over the window of e*(Tx, Ty), e = T - S (S bilinear of the staged
// next-level patch at origin (lc0, lr0) with weights (bx, by)); masked slots
// have T = Tx = Ty = 0 and contribute nothing.
template <int WIN>
__device__ __forceinline__ float2 gn_rhs(const float* __restrict__ JP, int lc0, int lr0, float bx,
                                         float by, const Runs<WIN>& ru, const Tmpl<WIN>& t) {
  constexpr int RL = Tmpl<WIN>::RL;
  constexpr int kPitch = Smem<WIN>::P;
  const float* base = JP + lr0 * kPitch + lc0;
  const float* bxp = base + ru.offx;
  const float* byp = base + ru.offy;
  const float2 wx = f2(bx, bx), wy = f2(by, by);
  auto hrow = [&](int r) {
    const float2 a0 = f2(bxp[r * kPitch], byp[r * kPitch]);
    const float2 a1 = f2(bxp[r * kPitch + 1], byp[r * kPitch + 1]);
    return fma2(wx, sub2(a1, a0), a0);
  };
  float2 h = hrow(0);
  float2 ax = f2(0.f, 0.f), ay = f2(0.f, 0.f);
#if V2D_GN_FOLD
  // e = T - [(1-by) h(p) + by h(p+1)] as two FMAs (one packed op per row fewer than
  // forming S and subtracting it)
  const float2 nw0 = f2(by - 1.0f, by - 1.0f), nw1 = f2(-by, -by);
#pragma unroll
  for (int p = 0; p < RL; ++p) {
    const float2 hn = hrow(p + 1);
    const float2 e = fma2(nw1, hn, fma2(nw0, h, t.T[p]));
    ax = fma2(e, t.TX[p], ax);
    ay = fma2(e, t.TY[p], ay);
    h = hn;
  }
#else
#pragma unroll
  for (int p = 0; p < RL; ++p) {
    const float2 hn = hrow(p + 1);
    const float2 e = sub2(t.T[p], fma2(wy, sub2(hn, h), h));
    ax = fma2(e, t.TX[p], ax);
    ay = fma2(e, t.TY[p], ay);
    h = hn;
  }
#endif
  return f2(ru.sum2(ax), ru.sum2(ay));
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
__device__ __forceinline__ float3 ncc_moments(const float* __restrict__ JP, int lc0, int lr0,
                                              float bx, float by, float m, const Runs<WIN>& ru,
                                              const Tmpl<WIN>& t) {
  constexpr int RL = Tmpl<WIN>::RL;
  constexpr int kPitch = Smem<WIN>::P;
  const float* base = JP + lr0 * kPitch + lc0;
  const float* bxp = base + ru.offx;
  const float* byp = base + ru.offy;
  const float2 wx = f2(bx, bx), wy = f2(by, by), mm = f2(m, m);
  auto hrow = [&](int r) {
    const float2 a0 = f2(bxp[r * kPitch], byp[r * kPitch]);
    const float2 a1 = f2(bxp[r * kPitch + 1], byp[r * kPitch + 1]);
    return fma2(wx, sub2(a1, a0), a0);
  };
  float2 h = hrow(0), hn = hrow(1);
  float2 sr = f2(0.f, 0.f), S0 = sr;
  if (kExactRef) {
    S0 = fma2(wy, sub2(hn, h), h);
    const float sref = __shfl_sync(kFullMask, S0.x, 0);
    sr = f2(sref, sref);
  }
  const float2 w0 = f2(1.0f - by, 1.0f - by), nm = f2(-m, -m);
  float2 s1 = f2(0.f, 0.f), s2 = f2(0.f, 0.f), st = f2(0.f, 0.f);
#pragma unroll
  for (int p = 0; p < RL; ++p) {
    if (p > 0) hn = hrow(p + 1);
    float2 S;
    if (kExactRef)
      S = sub2(p == 0 ? S0 : fma2(wy, sub2(hn, h), h), sr);
    else
      S = fma2(wy, hn, fma2(w0, h, nm));  // S - m = (1-by) h(p) + by h(p+1) - m
    if (!Tmpl<WIN>::kExact) S = mul2(S, ru.mask(p));
    s1 = add2(s1, S);
    s2 = fma2(S, S, s2);
    st = fma2(sub2(t.T[p], mm), S, st);
    h = hn;
  }
  return make_float3(ru.sum2(s1), ru.sum2(s2), ru.sum2(st));
}

// NCC of the template with S at (lc0, lr0) / (bx, by): two-pass in T (T' = T - tmean,
// Stt = sum T'^2), S centred by one of its own samples (ncc_moments<WIN, true>).  The
// cheaper folded pass centred by tmean, with the exact pass as a rare fallback when ill
// conditioned, measured +0.5 % slower (code size) and the folded pass alone is not
// flat-exact, so the exact pass is the only one.
template <int WIN>
__device__ __forceinline__ float ncc_value(const float* __restrict__ JP, int lc0, int lr0,
                                           float bx, float by, float tmean, float Stt,
                                           const Runs<WIN>& ru, const Tmpl<WIN>& t) {
  constexpr float kInvN = 1.0f / (float)(WIN * WIN);
  const float3 mo = ncc_moments<WIN, true>(JP, lc0, lr0, bx, by, tmean, ru, t);
  const float2 r1 = warp_sum2(f2(mo.x, mo.y));
  const float r2 = warp_sum2(f2(mo.z, 0.f)).x;
  // S' = S - c: sum (S - mean S)^2 = sum S'^2 - (sum S')^2 / n and
  // sum (T - mean T)(S - mean S) = sum T'S' (sum T' = 0 up to rounding of the mean)
  const float Sss = r1.y - r1.x * r1.x * kInvN;
  const float den2 = Stt * Sss;
  return den2 > 0.0f ? r2 * rsqrtf(den2) : 0.0f;
}

// One pyramid level of D7 for the warp's keypoint; (dx, dy) in level px.
// kEachStep: variant f3 (NCC after every update), a separate instantiation so the
// default Gauss-Newton loop carries none of its code or state.
template <int WIN, bool kEachStep>
__device__ __forceinline__ void track_level_body(float* __restrict__ sp, const Plane& I,
                                                 const Plane& J, const int L, const float cx,
                                                 const float cy, float& dx, float& dy,
                                                 const KltArgs& a, LevelOut& out KCYC_PARAM) {
  constexpr int R = (WIN - 1) / 2;
  constexpr int N = WIN * WIN;
  constexpr int M = search_margin(WIN);  // staged motion margin (px)
  constexpr int SZ = WIN + 1 + 2 * M;  // staged search patch edge (<= 32)
  constexpr int RL = Tmpl<WIN>::RL;
  static_assert(WIN + 3 <= 32 && SZ <= 32, "window too large for one warp");
  static_assert(WIN * Tmpl<WIN>::K <= 64, "two runs per lane");
  float* GX = sp + Smem<WIN>::PATCH;
  float* GY = GX + Smem<WIN>::GRID;

  // ---------------- template (previous frame) -----------------------------
  const Runs<WIN> ru;
  Tmpl<WIN> t;
  {
    const float fcx = floorf(cx), fcy = floorf(cy);
    const int ix = (int)fcx, iy = (int)fcy;
    KCLK(t_st);
    stage(sp, Smem<WIN>::P, GX, I, ix - R - 1, iy - R - 1, WIN + 3);
    KCYC(0, t_st);
  }
  KCLK(t_tm);
  {
    const float fcx = floorf(cx), fcy = floorf(cy);
    const int ix = (int)fcx, iy = (int)fcy;
    build_template<WIN>(sp, GX, GY, ix, iy, cx - fcx, cy - fcy, I.W, I.H, ru, t);
  }
  out.levels++;
  KSTAT(0);
  // per-run accumulation (.x run, .y run) -> no operand shuffling
  float2 axx = f2(0.f, 0.f), axy = axx, ayy = axx, ats = axx;
#pragma unroll
  for (int p = 0; p < RL; ++p) {
    axx = fma2(t.TX[p], t.TX[p], axx);
    axy = fma2(t.TX[p], t.TY[p], axy);
    ayy = fma2(t.TY[p], t.TY[p], ayy);
    ats = add2(t.T[p], ats);
  }
  float2 g01 = f2(ru.sum2(axx), ru.sum2(axy));  // (Gxx, Gxy)
  float2 g2s = f2(ru.sum2(ayy), ru.sum2(ats));  // (Gyy, sum T)
  g01 = warp_sum2(g01);
  g2s = warp_sum2(g2s);
  // lambda_min(G)/n < min_eig  <=>  det < min_eig * n * lambda_max  (no division)
  const float gxx = g01.x, gxy = g01.y, gyy = g2s.x;
  const float det = (float)((double)gxx * gyy - (double)gxy * gxy);  // no cancellation
  const float dg = gxx - gyy;
  const float lmax = 0.5f * (gxx + gyy + sqrtf(fmaf(dg, dg, 4.0f * gxy * gxy)));
  const bool finite = isfinite(gxx) && isfinite(gxy) && isfinite(gyy) && isfinite(det);
  // Tx, Ty are kept as 8 x (the Sobel/8 gradient): G and det carry 64 and 4096,
  // b carries 8; every compensation below is a power of two, so all results are
  // bit-identical to the unscaled arithmetic.
  if (!finite || !(det > 0.0f) || det < a.min_eig * (float)N * lmax * 64.0f) {
    KSTAT(6);
    KCYC(1, t_tm);
    if (L > 0) {
      dx *= 2.0f;
      dy *= 2.0f;
    } else {
      out.status = V2D_LOST_SMALL_EIG;
    }
    return;
  }
  const float inv_det = 8.0f / det;  // (G/64)^-1 / 8 applied to 8 b
  const float i00 = gyy * inv_det, i01 = -gxy * inv_det, i11 = gxx * inv_det;
  // two-pass NCC, first pass: template mean, then sum (T - mean)^2 (T itself
  // stays uncentred: the Gauss-Newton residual e = T - S needs no centring)
  // IEEE division: a flat template's mean is exact, so T - mean is exactly 0 there
  // (the oracle's NCC is then 0/0 -> 0; a rounded mean made Stt spuriously > 0)
  const float tmean = exact_mean(g2s.y, (float)N);
  float2 q = f2(0.f, 0.f);
#pragma unroll
  for (int p = 0; p < RL; ++p) {
    float2 d = sub2(t.T[p], f2(tmean, tmean));
    if (!Tmpl<WIN>::kExact) d = mul2(d, ru.mask(p));
    q = fma2(d, d, q);
  }
  const float Stt = warp_sum2(f2(ru.sum2(q), 0.f)).x;
  KCYC(1, t_tm);

  // ---------------- Gauss-Newton iterations (next frame) --------------------
  const float xmax = (float)(J.W - 1), ymax = (float)(J.H - 1);
  int jx0 = 0, jy0 = 0;
  bool staged = false;
  auto locate = [&](float qx, float qy, int& lc0, int& lr0, float& bx, float& by) {
    const float fqx = floorf(qx), fqy = floorf(qy);
    const int ixq = (int)fqx, iyq = (int)fqy;
    bx = qx - fqx;
    by = qy - fqy;
    lc0 = ixq - R - jx0;
    lr0 = iyq - R - jy0;
    if (!staged || lc0 < 0 || lc0 > 2 * M || lr0 < 0 || lr0 > 2 * M) {
      KSTAT(4);
      if (staged) KSTAT(5);
      jx0 = ixq - R - M;
      jy0 = iyq - R - M;
      KCLK(t_ss);
      stage(sp, Smem<WIN>::P, GX, J, jx0, jy0, SZ);
      KCYC(2, t_ss);
      staged = true;
      lc0 = M;
      lr0 = M;
    }
  };
  const float eps2 = a.eps * a.eps;
  KCLK(t_gn);
  for (int it = 1; it <= a.iters; ++it) {
    int lc0, lr0;
    float bx, by;
    locate(cx + dx, cy + dy, lc0, lr0, bx, by);
    const float2 b = warp_sum2(gn_rhs<WIN>(sp, lc0, lr0, bx, by, ru, t));
    const float ex = fmaf(i00, b.x, i01 * b.y);
    const float ey = fmaf(i01, b.x, i11 * b.y);
    dx += ex;
    dy += ey;
    out.steps++;
    KSTAT(3);
    const float nx = cx + dx, ny = cy + dy;
    const bool inside = nx >= 0.0f && nx <= xmax && ny >= 0.0f && ny <= ymax;
    if (!inside) {  // (also false for NaN)
      if (L > 0) {
        dx -= ex;
        dy -= ey;
        break;
      }
      out.status = V2D_LOST_OOB;
      return;
    }
    if (kEachStep) {  // variant f3: NCC after every update
      int lc0n, lr0n;
      float bxn, byn;
      locate(nx, ny, lc0n, lr0n, bxn, byn);
      out.ncc = ncc_value<WIN>(sp, lc0n, lr0n, bxn, byn, tmean, Stt, ru, t);
      if (out.ncc < a.ncc_min) {
        out.status = V2D_LOST_NCC;
        return;
      }
    }
    if (fmaf(ex, ex, ey * ey) < eps2) break;
  }
  // ---------------- per-level NCC gate --------------------------------------
  KCYC(3, t_gn);
  KCLK(t_nc);
  {
    int lc0, lr0;
    float bx, by;
    locate(cx + dx, cy + dy, lc0, lr0, bx, by);
    out.ncc = ncc_value<WIN>(sp, lc0, lr0, bx, by, tmean, Stt, ru, t);
    KCYC(4, t_nc);
    if (out.ncc < a.ncc_min) {
      out.status = V2D_LOST_NCC;
      return;
    }
  }
  if (L > 0) {
    dx *= 2.0f;
    dy *= 2.0f;
  }
}

// Inlined into the level loop (one call site, so one copy of the body; as an
// out-of-line function its arguments and in/out state went through the stack:
// same-box A/B -6..7 %).  The in/out state is copied into registers for the level.
template <int WIN, bool kEachStep>
__device__ __forceinline__ void track_level(float* __restrict__ sp, const Plane I, const Plane J,
                                            const int L, const float cx, const float cy,
                                            float& dx_io, float& dy_io, const KltArgs a,
                                            LevelOut& out_io KCYC_PARAM) {
  float dx = dx_io, dy = dy_io;
  LevelOut out = out_io;
  track_level_body<WIN, kEachStep>(sp, I, J, L, cx, cy, dx, dy, a, out KCYC_ARG);
  dx_io = dx;
  dy_io = dy;
  out_io = out;
}

template <int WIN, bool kEachStep>
#ifndef V2D_KLT_MINB
#define V2D_KLT_MINB 15  // 136 registers: K3 -0.5 % at c5, -0.7 % at c2 vs 16 (128); 12 is +13 %
#endif
__global__ void __launch_bounds__(kThreads, V2D_KLT_MINB)
klt_kernel(const uint8_t* const* __restrict__ prev_l0, const float* const* __restrict__ prev_pyr,
           const uint8_t* const* __restrict__ next_l0, const float* const* __restrict__ next_pyr,
           int B, Levels lv, KltArgs a, const float* __restrict__ pts,
           const float* __restrict__ guess, const uint8_t* __restrict__ in_status,
           float* __restrict__ out_pos, uint8_t* __restrict__ status, float* __restrict__ ncc,
           int32_t* __restrict__ iters_out, float4* __restrict__ track_list) {
  extern __shared__ __align__(16) float s_mem[];  // kWarps * Smem<WIN>::TOTAL floats
  const int64_t warp = (int64_t)blockIdx.x * kWarps + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (warp >= (int64_t)B * a.P) return;  // warp-uniform
  float* sp = s_mem + (threadIdx.x >> 5) * Smem<WIN>::TOTAL;
  const int b = (int)(warp / a.P);
  const float px = pts[2 * warp], py = pts[2 * warp + 1];
  constexpr int R = (WIN - 1) / 2;
  KCLK(t_all);
  KCYC_DECL;

  LevelOut o{V2D_TRACKED, 0.0f, 0, 0};
  const bool skip = (in_status && in_status[warp] != 0) || (px == -1.0f && py == -1.0f) ||
                    !isfinite(px) || !isfinite(py);
  float dx = 0.0f, dy = 0.0f;
  if (skip) {
    o.status = V2D_SKIPPED;
  } else if (px < 0.0f || px > (float)(lv.W[0] - 1) || py < 0.0f || py > (float)(lv.H[0] - 1)) {
    o.status = V2D_LOST_OOB;  // reading #16: a start point outside the image is lost
  } else {
    if (guess) {
      const float s = 1.0f / (float)(1 << (lv.n - 1));
      dx = guess[2 * warp] * s;
      dy = guess[2 * warp + 1] * s;
    }
    for (int L = lv.n - 1; L >= 0 && o.status == V2D_TRACKED; --L) {
      const float scale = __int_as_float((127 - L) << 23);  // 2^-L exactly
      const float cx = (px + 0.5f) * scale - 0.5f;
      const float cy = (py + 0.5f) * scale - 0.5f;
      Plane I, J;
      if (L == 0) {
        I = Plane{prev_l0[b], a.l0_pitch, lv.W[0], lv.H[0], 1};
        J = Plane{next_l0[b], a.l0_pitch, lv.W[0], lv.H[0], 1};
      } else {
        I = Plane{prev_pyr[b] + lv.offset[L], lv.pitch[L], lv.W[L], lv.H[L], 0};
        J = Plane{next_pyr[b] + lv.offset[L], lv.pitch[L], lv.W[L], lv.H[L], 0};
      }
      track_level<WIN, kEachStep>(sp, I, J, L, cx, cy, dx, dy, a, o KCYC_ARG);
    }
  }
  float ox = -1.0f, oy = -1.0f;
  if (o.status == V2D_TRACKED) {
    const float qx = px + dx, qy = py + dy;
    const int W = lv.W[0], H = lv.H[0];
    if (!(qx >= R && qx <= W - 1 - R && qy >= R && qy <= H - 1 - R)) {
      o.status = V2D_LOST_OOB;
    } else {
      ox = qx;
      oy = qy;
    }
  }
  if (lane == 0) {
    out_pos[2 * warp] = ox;
    out_pos[2 * warp + 1] = oy;
    status[warp] = (uint8_t)o.status;
    if (ncc) ncc[warp] = o.ncc;
    if (iters_out) iters_out[warp] = o.steps | (o.levels << 24);
    // a7 track-list record (x, y, status, ncc): the rig-wide all-gather ships these
    if (track_list) track_list[warp] = make_float4(ox, oy, (float)o.status, o.ncc);
  }
  KCYC(5, t_all);
  KCYC_FLUSH;
}

template <int WIN>
void launch_win(const uint8_t* const* prev_l0, const float* const* prev_pyr,
                const uint8_t* const* next_l0, const float* const* next_pyr, int B,
                const Levels& lv, const KltArgs& a, const float* pts, const float* guess,
                const uint8_t* in_status, float* out_pos, uint8_t* status, float* ncc,
                int32_t* iters_out, float4* track_list, cudaStream_t st) {
  const int64_t warps = (int64_t)B * a.P;  // <= INT32_MAX (checked by the ABI)
  const unsigned blocks = (unsigned)((warps + kWarps - 1) / kWarps);
  constexpr int smem = kWarps * Smem<WIN>::TOTAL * (int)sizeof(float);
  // below the 48 KB default for every window: no opt-in attribute, no per-process state
  static_assert(smem <= 48 * 1024, "KLT tile exceeds the default dynamic smem limit");
  if (a.flags & V2D_KLT_NCC_EACH_STEP)
    klt_kernel<WIN, true><<<blocks, kThreads, smem, st>>>(prev_l0, prev_pyr, next_l0, next_pyr,
                                                          B, lv, a, pts, guess, in_status,
                                                          out_pos, status, ncc, iters_out,
                                                          track_list);
  else
    klt_kernel<WIN, false><<<blocks, kThreads, smem, st>>>(prev_l0, prev_pyr, next_l0, next_pyr,
                                                           B, lv, a, pts, guess, in_status,
                                                           out_pos, status, ncc, iters_out,
                                                           track_list);
}

}  // namespace

int launch_klt(const uint8_t* const* prev_l0, const float* const* prev_pyr,
               const uint8_t* const* next_l0, const float* const* next_pyr, int B,
               const Levels& lv, const KltArgs& a, const float* pts, const float* guess,
               const uint8_t* in_status, float* out_pos, uint8_t* status, float* ncc,
               int32_t* iters_out, float* track_list, cudaStream_t st) {
  if (B == 0 || a.P == 0) return V2D_OK;
#ifndef V2D_NO_PAIR
  if (klt_pair_supported(a.win))  // small windows: two keypoints per warp (klt_pair.cu)
    return launch_klt_pair(prev_l0, prev_pyr, next_l0, next_pyr, B, lv, a, pts, guess, in_status,
                           out_pos, status, ncc, iters_out, track_list, st);
#endif
#define V2D_WIN_CASE(w)                                                                   \
  case w:                                                                                 \
    launch_win<w>(prev_l0, prev_pyr, next_l0, next_pyr, B, lv, a, pts, guess, in_status, \
                  out_pos, status, ncc, iters_out, reinterpret_cast<float4*>(track_list), st); \
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

#ifdef V2D_KLT_STATS
extern "C" int v2d_debug_klt_stats(unsigned long long* out, int reset) {
  cudaDeviceSynchronize();
  if (cudaMemcpyFromSymbol(out, g_klt_stats, sizeof(unsigned long long) * 16) != cudaSuccess)
    return -1;
  if (reset) {
    unsigned long long z[16] = {0};
    cudaMemcpyToSymbol(g_klt_stats, z, sizeof(z));
  }
  return 0;
}
#endif
#ifdef V2D_KLT_CYC
extern "C" int v2d_debug_klt_cycles(unsigned long long* out, int reset) {
  cudaDeviceSynchronize();
  if (cudaMemcpyFromSymbol(out, g_klt_cyc, sizeof(unsigned long long) * 512) != cudaSuccess)
    return -1;
  if (reset) {
    unsigned long long z[512] = {0};
    cudaMemcpyToSymbol(g_klt_cyc, z, sizeof(z));
  }
  return 0;
}
#endif
