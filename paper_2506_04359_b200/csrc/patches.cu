// patches.cu — variant f4: per-level patch features for loop closure
// ("a list of 9x9 image patches taken from each level of the
// image pyramid").
//
// out[b][p][L][v][u] = S(I_L, c_L + (u - r, v - r)),  c_L = (p + 0.5)/2^L - 0.5,
// bilinear with clamp-to-edge (D2), r = (patch-1)/2.
//
// B200 mapping: a gather on the resident pyramid — one warp per keypoint; per
// level the (patch+1)^2 pixel block is staged once in shared memory (the
// samples share their bilinear weights), then lanes form the patch x patch
// samples and store the contiguous [levels][patch][patch] block coalesced.
#include "common.cuh"

namespace v2d {
namespace {

constexpr int kWarps = 8;

// Every sample of one level shares the fractional offset of c_L, so a level's
// patch is a fixed-weight bilinear of one (patch+1)^2 block of pixels: the warp
// stages that block (clamp-to-edge, row-coalesced loads) in shared memory once
// and forms each sample from it with the same expression order as D2.
constexpr int kTile = 32;  // max block edge (patch <= 31)

template <int PATCH>  // compile-time patch edge: the index divisions become multiply-shifts
__global__ void __launch_bounds__(32 * kWarps)
patches_kernel(const uint8_t* const* __restrict__ l0_ptrs, const float* const* __restrict__ pyr_ptrs,
               int64_t l0_pitch, int B, Levels lv, const float* __restrict__ pts, int P,
               float* __restrict__ out) {
  constexpr int patch = PATCH;
  __shared__ float s_blk[kWarps][kTile * kTile];
  const int64_t kp = (int64_t)blockIdx.x * kWarps + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (kp >= (int64_t)B * P) return;  // warp-uniform
  float* blk = s_blk[threadIdx.x >> 5];
  const int b = (int)(kp / P);
  const float px0 = pts[2 * kp], py0 = pts[2 * kp + 1];
  const bool empty = (px0 == -1.0f && py0 == -1.0f) || !isfinite(px0) || !isfinite(py0);
  constexpr int n = patch * patch, r = (patch - 1) / 2, e = patch + 1;
  float* o = out + kp * (int64_t)lv.n * n;
  if (empty) {
    for (int i = lane; i < lv.n * n; i += 32) o[i] = 0.0f;
    return;
  }
  for (int L = 0; L < lv.n; ++L) {
    const float scale = __int_as_float((127 - L) << 23);  // 2^-L
    const float cx = (px0 + 0.5f) * scale - 0.5f, cy = (py0 + 0.5f) * scale - 0.5f;
    const float fx = floorf(cx), fy = floorf(cy);
    const float wa = cx - fx, wb = cy - fy;
    const int bx = (int)fx - r, by = (int)fy - r;  // block origin (pixel of sample u=v=0)
    const int W = lv.W[L], H = lv.H[L];
    __syncwarp();
    for (int j = lane; j < e * e; j += 32) {
      const int rr = j / e, cc = j - rr * e;
      const int x = min(max(bx + cc, 0), W - 1), y = min(max(by + rr, 0), H - 1);
      blk[rr * kTile + cc] =
          L == 0 ? (float)__ldg(l0_ptrs[b] + (int64_t)y * l0_pitch + x)
                 : __ldg(pyr_ptrs[b] + lv.offset[L] + (int64_t)y * lv.pitch[L] + x);
    }
    __syncwarp();
    float* oL = o + L * n;
    for (int i = lane; i < n; i += 32) {
      const int v = i / patch, u = i - v * patch;
      const float* q = blk + v * kTile + u;
      const float top = fmaf(wa, q[1] - q[0], q[0]);
      const float bot = fmaf(wa, q[kTile + 1] - q[kTile], q[kTile]);
      oL[i] = fmaf(wb, bot - top, top);
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
