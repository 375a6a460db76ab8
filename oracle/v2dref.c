/*
 * v2dref.c — ORACLE for the cuVSLAM 2D-module hot path (arXiv 2506.04359).
 *
 * TEST INFRASTRUCTURE ONLY: loaded by tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs, never by the product path.
 * Shares no code with paper_2506_04359_b200/csrc (see v2dref.h).
 *
 * Every function follows one definition of SURVEY.md §8(c) (D1..D7), which in
 * turn reads PAPER.md §2.1.  No blocking, fusion or reordering:
 * nested loops in the order the definition is written.
 *
 * Build: gcc -std=c11 -O2 -ffp-contract=off -fPIC -shared (never -ffast-math;
 * the fp32 response contract D4 needs unfused IEEE single operations).
 *
 * Pins (tests/test_oracle_*.py): closed forms (constant, ramp, saddle, block
 * mean, exact translations), cv2.resize(INTER_AREA) and
 * cv2.cornerMinEigenVal, numpy.linalg.eigvalsh, brute-force top-k,
 * SPEC worked examples.
 */
#include "v2dref.h"

#include <float.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ D1 -- */
/* Level sizes: "each level's dimensions = floor(previous/2)". */
int v2dref_level_dims(int W, int H, int levels, int* Ws, int* Hs) {
  if (W < 1 || H < 1 || levels < 1 || levels > 8) return V2DREF_EINVAL;
  if ((W >> (levels - 1)) < 1 || (H >> (levels - 1)) < 1) return V2DREF_EINVAL;
  int w = W, h = H;
  for (int L = 0; L < levels; ++L) {
    if (Ws) Ws[L] = w;
    if (Hs) Hs[L] = h;
    w /= 2;
    h /= 2;
  }
  return V2DREF_OK;
}

int64_t v2dref_pyramid_size(int W, int H, int levels) {
  int Ws[8], Hs[8];
  if (v2dref_level_dims(W, H, levels, Ws, Hs) != V2DREF_OK) return -1;
  int64_t n = 0;
  for (int L = 0; L < levels; ++L) n += (int64_t)Ws[L] * Hs[L];
  return n;
}

/* D1: I_0 = F; I_L(x,y) = 1/4 * sum_{i,j in {0,1}} I_{L-1}(2x+i, 2y+j)
 * ("downsampling by 2x2 box filter").  float64 holds every value
 * exactly (values lie in 4^-L * Z, at most 8+2L significant bits). */
int v2dref_build_pyramid(const uint8_t* img, int64_t pitch, int W, int H,
                         int levels, double* out) {
  int Ws[8], Hs[8];
  if (!img || !out || pitch < W) return V2DREF_EINVAL;
  if (v2dref_level_dims(W, H, levels, Ws, Hs) != V2DREF_OK) return V2DREF_EINVAL;
  double* lvl = out;
  for (int y = 0; y < H; ++y)
    for (int x = 0; x < W; ++x) lvl[(int64_t)y * W + x] = (double)img[(int64_t)y * pitch + x];
  for (int L = 1; L < levels; ++L) {
    const double* src = lvl;
    int sw = Ws[L - 1];
    double* dst = lvl + (int64_t)Ws[L - 1] * Hs[L - 1];
    for (int y = 0; y < Hs[L]; ++y)
      for (int x = 0; x < Ws[L]; ++x) {
        double s = 0.0;
        for (int j = 0; j < 2; ++j)
          for (int i = 0; i < 2; ++i) s += src[(int64_t)(2 * y + j) * sw + (2 * x + i)];
        dst[(int64_t)y * Ws[L] + x] = 0.25 * s;
      }
    lvl = dst;
  }
  return V2DREF_OK;
}

/* ------------------------------------------------------------------ D2 -- */
static int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

/* Clamp-to-edge pixel I~(x,y) = I(clamp(x,0,W-1), clamp(y,0,H-1)). */
static double pix(const double* I, int W, int H, int x, int y) {
  return I[(int64_t)clampi(y, 0, H - 1) * W + clampi(x, 0, W - 1)];
}

/* S(I,x,y) = (1-b)[(1-a)I~(x0,y0) + a I~(x0+1,y0)]
 *          +    b [(1-a)I~(x0,y0+1) + a I~(x0+1,y0+1)],  x0=floor(x), a=x-x0. */
double v2dref_bilinear(const double* I, int W, int H, double x, double y) {
  double fx = floor(x), fy = floor(y);
  /* Far-outside coordinates clamp anyway; keep the int conversion defined. */
  if (fx < -4.0) fx = -4.0;
  if (fx > (double)W + 4.0) fx = (double)W + 4.0;
  if (fy < -4.0) fy = -4.0;
  if (fy > (double)H + 4.0) fy = (double)H + 4.0;
  double a = x - floor(x), b = y - floor(y);
  if (a < 0.0 || a >= 1.0) a = 0.0; /* only reachable for non-finite x */
  if (b < 0.0 || b >= 1.0) b = 0.0;
  int x0 = (int)fx, y0 = (int)fy;
  double top = (1.0 - a) * pix(I, W, H, x0, y0) + a * pix(I, W, H, x0 + 1, y0);
  double bot = (1.0 - a) * pix(I, W, H, x0, y0 + 1) + a * pix(I, W, H, x0 + 1, y0 + 1);
  return (1.0 - b) * top + b * bot;
}

/* ------------------------------------------------------------------ D3 -- */
/* Gx(x,y) = [I~(x+1,y-1) + 2I~(x+1,y) + I~(x+1,y+1)
 *          - I~(x-1,y-1) - 2I~(x-1,y) - I~(x-1,y+1)] / 8;  Gy the transpose
 * ("3x3 Sobel-gradient"). */
void v2dref_sobel(const double* I, int W, int H, double* gx, double* gy) {
  for (int y = 0; y < H; ++y)
    for (int x = 0; x < W; ++x) {
      double sx = pix(I, W, H, x + 1, y - 1) + 2.0 * pix(I, W, H, x + 1, y) +
                  pix(I, W, H, x + 1, y + 1) - pix(I, W, H, x - 1, y - 1) -
                  2.0 * pix(I, W, H, x - 1, y) - pix(I, W, H, x - 1, y + 1);
      double sy = pix(I, W, H, x - 1, y + 1) + 2.0 * pix(I, W, H, x, y + 1) +
                  pix(I, W, H, x + 1, y + 1) - pix(I, W, H, x - 1, y - 1) -
                  2.0 * pix(I, W, H, x, y - 1) - pix(I, W, H, x + 1, y - 1);
      gx[(int64_t)y * W + x] = sx / 8.0;
      gy[(int64_t)y * W + x] = sy / 8.0;
    }
}

/* lambda_min of [[a,b],[b,c]] = det / lambda_max,
 * lambda_max = (a + c + sqrt((a-c)^2 + 4b^2)) / 2. */
double v2dref_lambda_min(double a, double b, double c) {
  double tr = a + c;
  if (tr == 0.0) return 0.0;
  double det = a * c - b * b;
  double lmax = 0.5 * (tr + sqrt((a - c) * (a - c) + 4.0 * b * b));
  return det / lmax;
}

/* ------------------------------------------------------------------ D4 -- */
/* GFTT response ("Good Features to Track" measure; 3x3 Sobel, 3x3
 * window).  sx = 8*Gx and sy = 8*Gy are integers; A' = sum sx^2,
 * B' = sum sx*sy, C' = sum sy^2 over the 3x3 window; tr = A'+C',
 * det = A'C'-B'^2, D = (A'-C')^2 + 4B'^2 exactly in int64.
 * Contract (reading #4): R = [f32(det) / ((f32(tr) + sqrt(f32(D))) * 0.5)] * 2^-6
 * with every operation IEEE binary32 round-to-nearest, no contraction. */
static int sobel_int_x(const uint8_t* img, int64_t p, int x, int y) {
  const uint8_t* r0 = img + (int64_t)(y - 1) * p;
  const uint8_t* r1 = img + (int64_t)y * p;
  const uint8_t* r2 = img + (int64_t)(y + 1) * p;
  return (r0[x + 1] + 2 * r1[x + 1] + r2[x + 1]) - (r0[x - 1] + 2 * r1[x - 1] + r2[x - 1]);
}
static int sobel_int_y(const uint8_t* img, int64_t p, int x, int y) {
  const uint8_t* r0 = img + (int64_t)(y - 1) * p;
  const uint8_t* r2 = img + (int64_t)(y + 1) * p;
  return (r2[x - 1] + 2 * r2[x] + r2[x + 1]) - (r0[x - 1] + 2 * r0[x] + r0[x + 1]);
}

int v2dref_response(const uint8_t* img, int64_t pitch, int W, int H,
                    float* R, double* lmin) {
  if (!img || !R || W < 5 || H < 5 || pitch < W) return V2DREF_EINVAL;
  for (int64_t i = 0; i < (int64_t)W * H; ++i) {
    R[i] = 0.0f;
    if (lmin) lmin[i] = 0.0;
  }
  for (int y = 2; y <= H - 3; ++y)
    for (int x = 2; x <= W - 3; ++x) {
      int64_t A = 0, B = 0, C = 0;
      for (int j = -1; j <= 1; ++j)
        for (int i = -1; i <= 1; ++i) {
          int64_t sx = sobel_int_x(img, pitch, x + i, y + j);
          int64_t sy = sobel_int_y(img, pitch, x + i, y + j);
          A += sx * sx;
          B += sx * sy;
          C += sy * sy;
        }
      int64_t tr = A + C;
      int64_t det = A * C - B * B;
      int64_t D = (A - C) * (A - C) + 4 * B * B;
      float r = 0.0f;
      if (tr != 0) {
        volatile float f_det = (float)det; /* correctly rounded int64 -> f32 */
        volatile float f_tr = (float)tr;
        volatile float f_D = (float)D;
        volatile float f_sq = sqrtf(f_D);
        volatile float f_sum = f_tr + f_sq;
        volatile float f_lmax = f_sum * 0.5f;
        volatile float f_q = f_det / f_lmax;
        r = f_q * 0.015625f;
      }
      R[(int64_t)y * W + x] = r;
      if (lmin) {
        long double ltr = (long double)tr;
        long double lmax = 0.5L * (ltr + sqrtl((long double)D));
        lmin[(int64_t)y * W + x] =
            (tr == 0) ? 0.0 : (double)(((long double)det / lmax) / 64.0L);
      }
    }
  return V2DREF_OK;
}

/* ------------------------------------------------------------- Eq. 1 ---- */
/* k > floor(K_I / (N*M)); k = floor(K_I/(N*M)) + 1 when k == 0
 * (reading #7). */
int v2dref_grid_k(int grid_x, int grid_y, int k, int K_min, int* k_out) {
  if (grid_x < 1 || grid_y < 1 || K_min < 0 || k < 0) return V2DREF_EINVAL;
  int floor_q = (int)((int64_t)K_min / ((int64_t)grid_x * grid_y));
  int kk = (k == 0) ? floor_q + 1 : k;
  if (kk <= floor_q || kk > 256) return V2DREF_EINVAL;
  if (k_out) *k_out = kk;
  return V2DREF_OK;
}

/* ------------------------------------------------------------- D5-D6 ---- */
/* key(p) = (bits(R) << 32) | (0xFFFFFFFF - (y*W + x)): higher score first,
 * then smaller row-major index (reading #8). */
static uint64_t key_of(const float* R, int W, int x, int y) {
  float r = R[(int64_t)y * W + x];
  uint32_t bits;
  memcpy(&bits, &r, sizeof bits);
  uint32_t idx = (uint32_t)((int64_t)y * W + x);
  return ((uint64_t)bits << 32) | (uint64_t)(0xFFFFFFFFu - idx);
}

static int cmp_key_desc(const void* pa, const void* pb) {
  uint64_t a = *(const uint64_t*)pa, b = *(const uint64_t*)pb;
  return (a < b) - (a > b);
}

int v2dref_detect_gftt(const uint8_t* img, int64_t pitch, int W, int H,
                       int grid_x, int grid_y, int k, int K_min,
                       float min_score, int border, int nms, const uint8_t* mask,
                       float* kp_xy, float* kp_score, int32_t* cell_count) {
  int kk;
  if (!img || !kp_xy || !kp_score || !cell_count || pitch < W) return V2DREF_EINVAL;
  if (border < 3 || W < 2 * border + 1 || H < 2 * border + 1) return V2DREF_EINVAL;
  if ((int64_t)W * H >= ((int64_t)1 << 31)) return V2DREF_EINVAL;
  if (grid_x > W || grid_y > H) return V2DREF_EINVAL; /* cell < 1 px */
  if (v2dref_grid_k(grid_x, grid_y, k, K_min, &kk) != V2DREF_OK) return V2DREF_EINVAL;

  float* R = (float*)malloc(sizeof(float) * (size_t)W * H);
  uint64_t* cand = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)W * H);
  if (!R || !cand) {
    free(R);
    free(cand);
    return V2DREF_EINVAL;
  }
  v2dref_response(img, pitch, W, H, R, NULL);

  for (int cy = 0; cy < grid_y; ++cy)
    for (int cx = 0; cx < grid_x; ++cx) {
      /* D6: cell = [floor(cx*W/gx), floor((cx+1)*W/gx)) x [...] (reading #6) */
      int x0 = (int)((int64_t)cx * W / grid_x), x1 = (int)((int64_t)(cx + 1) * W / grid_x);
      int y0 = (int)((int64_t)cy * H / grid_y), y1 = (int)((int64_t)(cy + 1) * H / grid_y);
      int n = 0;
      for (int y = y0; y < y1; ++y)
        for (int x = x0; x < x1; ++x) {
          /* D5 eligibility */
          if (x < border || x > W - 1 - border || y < border || y > H - 1 - border) continue;
          if (!(R[(int64_t)y * W + x] > min_score)) continue;
          if (mask && mask[(int64_t)y * pitch + x]) continue; /* f1 min_separation */
          uint64_t kp = key_of(R, W, x, y);
          int is_max = 1;
          if (nms) /* strict 3x3 local maximum by key (reading #5) */
            for (int j = -1; j <= 1 && is_max; ++j)
              for (int i = -1; i <= 1; ++i) {
                if (i == 0 && j == 0) continue;
                if (!(kp > key_of(R, W, x + i, y + j))) {
                  is_max = 0;
                  break;
                }
              }
          if (is_max) cand[n++] = kp;
        }
      qsort(cand, (size_t)n, sizeof(uint64_t), cmp_key_desc);
      int cell = cy * grid_x + cx;
      int m = n < kk ? n : kk;
      cell_count[cell] = m;
      for (int s = 0; s < kk; ++s) {
        int64_t slot = (int64_t)cell * kk + s;
        if (s < m) {
          uint32_t idx = 0xFFFFFFFFu - (uint32_t)(cand[s] & 0xFFFFFFFFu);
          uint32_t bits = (uint32_t)(cand[s] >> 32);
          float sc;
          memcpy(&sc, &bits, sizeof sc);
          kp_xy[2 * slot] = (float)(idx % (uint32_t)W);
          kp_xy[2 * slot + 1] = (float)(idx / (uint32_t)W);
          kp_score[slot] = sc;
        } else {
          kp_xy[2 * slot] = -1.0f;
          kp_xy[2 * slot + 1] = -1.0f;
          kp_score[slot] = 0.0f;
        }
      }
    }
  free(R);
  free(cand);
  return V2DREF_OK;
}

/* ---------------------------------------------------------------- NCC --- */
/* ncc(P,Q) = sum (P-Pm)(Q-Qm) / sqrt(sum (P-Pm)^2 * sum (Q-Qm)^2), means
 * first (two-pass); 0 when the denominator is 0 (reading #14). */
double v2dref_ncc(const double* P, const double* Q, int n) {
  double mp = 0.0, mq = 0.0;
  for (int i = 0; i < n; ++i) {
    mp += P[i];
    mq += Q[i];
  }
  mp /= n;
  mq /= n;
  double spq = 0.0, spp = 0.0, sqq = 0.0;
  for (int i = 0; i < n; ++i) {
    double dp = P[i] - mp, dq = Q[i] - mq;
    spq += dp * dq;
    spp += dp * dp;
    sqq += dq * dq;
  }
  double den = sqrt(spp * sqq);
  return den > 0.0 ? spq / den : 0.0;
}

/* ------------------------------------------------------------------ D7 -- */
static double dmin(double a, double b) { return a < b ? a : b; }

/* Distance of (x,y) to the box [lo_x,hi_x]x[lo_y,hi_y] boundary (>=0). */
static double bound_margin(double x, double y, double lx, double hx, double ly, double hy) {
  return dmin(dmin(fabs(x - lx), fabs(hx - x)), dmin(fabs(y - ly), fabs(hy - y)));
}

int v2dref_track_klt(const double* prev_pyr, const double* next_pyr,
                     int W, int H, int levels,
                     const float* pts, const float* guess,
                     const uint8_t* in_status, int P,
                     int win, int iters, double eps, double ncc_min,
                     double min_eig, int ncc_each_step,
                     double* out_pos, uint8_t* status, double* ncc,
                     double* diag) {
  int Ws[8], Hs[8];
  if (!prev_pyr || !next_pyr || (P > 0 && (!pts || !out_pos || !status))) return V2DREF_EINVAL;
  if (v2dref_level_dims(W, H, levels, Ws, Hs) != V2DREF_OK) return V2DREF_EINVAL;
  if (win < 3 || (win % 2) == 0 || iters < 1 || P < 0) return V2DREF_EINVAL;
  /* reading #27: min_eig must be > 0.  The closed-form step eta = G^-1 b
   * divides by det(G); lambda_min/n >= min_eig > 0 is what guarantees det > 0
   * (D7 applies the conditioning test before any solve), so a non-positive
   * threshold would let a rank-deficient window reach the division. */
  if (!(min_eig > 0.0)) return V2DREF_EINVAL;
  const int r = (win - 1) / 2, n = win * win;

  /* Level planes and template-gradient planes Gx_L, Gy_L of the previous
   * frame (D3). */
  const double *I[8], *J[8];
  double *GX[8], *GY[8];
  int64_t off = 0;
  for (int L = 0; L < levels; ++L) {
    I[L] = prev_pyr + off;
    J[L] = next_pyr + off;
    off += (int64_t)Ws[L] * Hs[L];
    GX[L] = (double*)malloc(sizeof(double) * (size_t)Ws[L] * Hs[L]);
    GY[L] = (double*)malloc(sizeof(double) * (size_t)Ws[L] * Hs[L]);
    v2dref_sobel(I[L], Ws[L], Hs[L], GX[L], GY[L]);
  }
  double* T = (double*)malloc(sizeof(double) * n);
  double* TX = (double*)malloc(sizeof(double) * n);
  double* TY = (double*)malloc(sizeof(double) * n);
  double* S = (double*)malloc(sizeof(double) * n);

  for (int p = 0; p < P; ++p) {
    double px = pts[2 * p], py = pts[2 * p + 1];
    double m_ncc = INFINITY, m_eig = INFINITY, m_bnd = INFINITY, m_eps = INFINITY;
    double last_ncc = 0.0;
    int st = V2DREF_TRACKED;
    if ((in_status && in_status[p] != 0) || (px == -1.0 && py == -1.0) || !isfinite(px) ||
        !isfinite(py)) {
      st = V2DREF_SKIPPED;
    }
    if (st == V2DREF_TRACKED && (px < 0.0 || px > W - 1 || py < 0.0 || py > H - 1))
      st = V2DREF_LOST_OOB; /* reading #16: a start point outside the image is lost */
    double dx = 0.0, dy = 0.0;
    if (st == V2DREF_TRACKED && guess) {
      dx = guess[2 * p] / (double)(1 << (levels - 1));
      dy = guess[2 * p + 1] / (double)(1 << (levels - 1));
    }
    for (int L = levels - 1; L >= 0 && st == V2DREF_TRACKED; --L) {
      const int wl = Ws[L], hl = Hs[L];
      const double scale = (double)(1 << L);
      /* box-pyramid-consistent centre (reading #2) */
      const double cx = (px + 0.5) / scale - 0.5, cy = (py + 0.5) / scale - 0.5;
      /* template T, Tx, Ty at c+(u,v) */
      double gxx = 0.0, gxy = 0.0, gyy = 0.0;
      for (int v = -r, i = 0; v <= r; ++v)
        for (int u = -r; u <= r; ++u, ++i) {
          T[i] = v2dref_bilinear(I[L], wl, hl, cx + u, cy + v);
          TX[i] = v2dref_bilinear(GX[L], wl, hl, cx + u, cy + v);
          TY[i] = v2dref_bilinear(GY[L], wl, hl, cx + u, cy + v);
        }
      for (int i = 0; i < n; ++i) {
        gxx += TX[i] * TX[i];
        gxy += TX[i] * TY[i];
        gyy += TY[i] * TY[i];
      }
      double lam = v2dref_lambda_min(gxx, gxy, gyy);
      double lmax = gxx + gyy - lam;
      int finite = isfinite(gxx) && isfinite(gxy) && isfinite(gyy) && isfinite(lam);
      if (finite && lmax > 0.0) m_eig = dmin(m_eig, fabs(lam / n - min_eig) / (lmax / n));
      if (!finite || lam / n < min_eig) { /* reading #15 */
        if (L > 0) {
          dx *= 2.0;
          dy *= 2.0;
          continue;
        }
        st = V2DREF_LOST_SMALL_EIG;
        break;
      }
      const double det = gxx * gyy - gxy * gxy;
      for (int it = 1; it <= iters; ++it) {
        double bx = 0.0, by = 0.0;
        for (int v = -r, i = 0; v <= r; ++v)
          for (int u = -r; u <= r; ++u, ++i) {
            double e = T[i] - v2dref_bilinear(J[L], wl, hl, cx + dx + u, cy + dy + v);
            bx += e * TX[i];
            by += e * TY[i];
          }
        /* eta = G^-1 b, closed form */
        double ex = (gyy * bx - gxy * by) / det;
        double ey = (gxx * by - gxy * bx) / det;
        dx += ex;
        dy += ey;
        double qx = cx + dx, qy = cy + dy;
        int inside = isfinite(qx) && isfinite(qy) && qx >= 0.0 && qx <= wl - 1 && qy >= 0.0 &&
                     qy <= hl - 1;
        if (isfinite(qx) && isfinite(qy))
          m_bnd = dmin(m_bnd, bound_margin(qx, qy, 0.0, wl - 1, 0.0, hl - 1));
        if (!inside) { /* reading #16 */
          if (L > 0) {
            dx -= ex;
            dy -= ey;
            break;
          }
          st = V2DREF_LOST_OOB;
          break;
        }
        if (ncc_each_step) { /* variant f3: NCC after every optimization step */
          for (int v = -r, i = 0; v <= r; ++v)
            for (int u = -r; u <= r; ++u, ++i)
              S[i] = v2dref_bilinear(J[L], wl, hl, cx + dx + u, cy + dy + v);
          last_ncc = v2dref_ncc(T, S, n);
          m_ncc = dmin(m_ncc, fabs(last_ncc - ncc_min));
          if (last_ncc < ncc_min) {
            st = V2DREF_LOST_NCC;
            break;
          }
        }
        double step = sqrt(ex * ex + ey * ey);
        m_eps = dmin(m_eps, fabs(step - eps));
        if (step < eps) break; /* reading #12 */
      }
      if (st != V2DREF_TRACKED) break;
      /* per-level NCC gate (reading #13) */
      for (int v = -r, i = 0; v <= r; ++v)
        for (int u = -r; u <= r; ++u, ++i)
          S[i] = v2dref_bilinear(J[L], wl, hl, cx + dx + u, cy + dy + v);
      last_ncc = v2dref_ncc(T, S, n);
      m_ncc = dmin(m_ncc, fabs(last_ncc - ncc_min));
      if (last_ncc < ncc_min) {
        st = V2DREF_LOST_NCC;
        break;
      }
      if (L > 0) {
        dx *= 2.0;
        dy *= 2.0;
      }
    }
    double ox = -1.0, oy = -1.0;
    if (st == V2DREF_TRACKED) {
      double qx = px + dx, qy = py + dy;
      /* half-window margin */
      m_bnd = dmin(m_bnd, bound_margin(qx, qy, r, W - 1 - r, r, H - 1 - r));
      if (qx < r || qx > W - 1 - r || qy < r || qy > H - 1 - r)
        st = V2DREF_LOST_OOB;
      else {
        ox = qx;
        oy = qy;
      }
    }
    out_pos[2 * p] = ox;
    out_pos[2 * p + 1] = oy;
    status[p] = (uint8_t)st;
    if (ncc) ncc[p] = last_ncc;
    if (diag) {
      diag[4 * p + 0] = m_ncc;
      diag[4 * p + 1] = m_eig;
      diag[4 * p + 2] = m_bnd;
      diag[4 * p + 3] = m_eps;
    }
  }
  for (int L = 0; L < levels; ++L) {
    free(GX[L]);
    free(GY[L]);
  }
  free(T);
  free(TX);
  free(TY);
  free(S);
  return V2DREF_OK;
}

/* ------------------------------------------------------- f4 patches ---- */
/* "a list of 9x9 image patches taken from each level of the image pyramid"
 * (P:216); sampled like the KLT template (D2, reading #2). */
int v2dref_extract_patches(const double* pyr, int W, int H, int levels, const float* pts, int P,
                           int patch, double* out) {
  int Ws[8], Hs[8];
  if (!pyr || (P > 0 && (!pts || !out)) || patch < 1 || (patch % 2) == 0) return V2DREF_EINVAL;
  if (v2dref_level_dims(W, H, levels, Ws, Hs) != V2DREF_OK) return V2DREF_EINVAL;
  const int r = (patch - 1) / 2, n = patch * patch;
  for (int p = 0; p < P; ++p) {
    double px = pts[2 * p], py = pts[2 * p + 1];
    int empty = (px == -1.0 && py == -1.0) || !isfinite(px) || !isfinite(py);
    int64_t off = 0;
    for (int L = 0; L < levels; ++L) {
      const double* I = pyr + off;
      double scale = (double)(1 << L);
      double cx = (px + 0.5) / scale - 0.5, cy = (py + 0.5) / scale - 0.5;
      for (int v = 0; v < patch; ++v)
        for (int u = 0; u < patch; ++u)
          out[((int64_t)p * levels + L) * n + v * patch + u] =
              empty ? 0.0 : v2dref_bilinear(I, Ws[L], Hs[L], cx + (u - r), cy + (v - r));
      off += (int64_t)Ws[L] * Hs[L];
    }
  }
  return V2DREF_OK;
}

/* ------------------------------------------------------- f1 keyframes -- */
/* "keypoints closer than min_separation to an existing live track are
 * suppressed". */
int v2dref_suppress_mask(const float* tracks, const uint8_t* status, int P, double min_sep,
                         int W, int H, uint8_t* mask) {
  if (!mask || W < 1 || H < 1 || P < 0 || !(min_sep >= 0.0)) return V2DREF_EINVAL;
  for (int64_t i = 0; i < (int64_t)W * H; ++i) mask[i] = 0;
  for (int p = 0; p < P; ++p) {
    if (status[p] != V2DREF_TRACKED) continue;
    double tx = tracks[2 * p], ty = tracks[2 * p + 1];
    for (int y = 0; y < H; ++y)
      for (int x = 0; x < W; ++x) {
        double dx = x - tx, dy = y - ty;
        if (dx * dx + dy * dy < min_sep * min_sep) mask[(int64_t)y * W + x] = 1;
      }
  }
  return V2DREF_OK;
}

/* Eq. 5: a keyframe is created if |S_curr ∩ S_kf| / |S_kf| < T. */
int v2dref_keyframe_due(int64_t n_kf, int64_t n_surv, double T) {
  if (n_kf == 0) return 1; /* bootstrap: the first frame is a keyframe */
  return ((double)n_surv / (double)n_kf) < T ? 1 : 0;
}

int v2dref_refill(const float* kp_xy, const int32_t* cell_count, int cells, int k, int P,
                  float* tracks, uint8_t* status, uint8_t* kf_member, int32_t* track_id,
                  int32_t* next_id) {
  if (!kp_xy || !cell_count || !tracks || !status || !kf_member || !track_id || !next_id)
    return V2DREF_EINVAL;
  /* valid detections in slot order */
  int n_new = 0;
  for (int c = 0; c < cells; ++c) n_new += cell_count[c];
  int j = 0, c = 0, r = 0;
  for (int p = 0; p < P && j < n_new; ++p) {
    if (status[p] == V2DREF_TRACKED) continue;
    while (r >= cell_count[c]) {
      ++c;
      r = 0;
    }
    int64_t src = (int64_t)c * k + r;
    tracks[2 * p] = kp_xy[2 * src];
    tracks[2 * p + 1] = kp_xy[2 * src + 1];
    status[p] = V2DREF_TRACKED;
    track_id[p] = *next_id + j;
    ++j;
    ++r;
  }
  *next_id += j;
  for (int p = 0; p < P; ++p) kf_member[p] = status[p] == V2DREF_TRACKED;
  return V2DREF_OK;
}
