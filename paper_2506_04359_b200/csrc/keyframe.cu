// keyframe.cu — variant f1: keyframe-driven continuous tracking.
//
// Track table per image: tracks [P][2], status [P] (the KLT status array: 0 =
// TRACKED/alive, anything else = lost; fed back as KLT in_status so lost is
// terminal), kf_member [P], track_id [P], next_id.
// Operations ("if the number of successfully tracked keypoints falls
// below a threshold, the 2D module creates a new keyframe"; Eq. 5
// |S_curr ∩ S_kf| / |S_kf| < T; readings #23-#26
// of DESIGN.md):
//   suppress : mask(x,y) = 1 iff (x - tx)^2 + (y - ty)^2 < min_sep^2 for a live
//              track t (evaluated exactly in fp64: fp32 inputs, integer pixels)
//   survival : per image n_kf = #slots in S_kf, n_surv = #slots in S_kf still alive
//   decide   : keyframe iff sum n_kf == 0 or sum n_surv < T * sum n_kf (fp64)
//   refill   : on a keyframe, the j-th valid new detection (cell-major slot order)
//              fills the j-th dead track slot (ascending index), gets id
//              next_id + j; then S_kf := the alive slots.  Lost slots never come
//              back to life except by refill with a NEW id.
// All are tiny, launch-latency-bound kernels; every one of them reads a device
// flag so that the keyframe branch runs without a host round trip.  Captured as one
// CUDA graph per frame (frontend.KeyframeTracker.capture), the branch is the body of
// a conditional (IF) node set by the decide kernel, and the frame tables come from a
// device frame counter (ring_tables): one graph launch per rig-frame.
#include "common.cuh"

namespace v2d {
namespace {

constexpr int kT = 256;

__global__ void clear_mask_kernel(uint8_t* const* __restrict__ mask_ptrs, int64_t pitch, int W,
                                  int H, const int32_t* __restrict__ enable) {
  const int b = blockIdx.y;
  if (enable && enable[0] == 0) return;
  uint8_t* m = mask_ptrs[b];
  const int64_t n = (int64_t)H * pitch;  // pitch % 16 == 0: 16-B vector clears
  uint4* m4 = reinterpret_cast<uint4*>(m);
  const bool al = (reinterpret_cast<uintptr_t>(m) & 15u) == 0;
  if (al) {
    for (int64_t i = (int64_t)blockIdx.x * kT + threadIdx.x; i < n / 16; i += (int64_t)gridDim.x * kT)
      m4[i] = make_uint4(0u, 0u, 0u, 0u);
  } else {
    for (int64_t i = (int64_t)blockIdx.x * kT + threadIdx.x; i < n; i += (int64_t)gridDim.x * kT)
      m[i] = 0;
  }
}

__global__ void draw_mask_kernel(uint8_t* const* __restrict__ mask_ptrs, int64_t pitch, int W,
                                 int H, const float* __restrict__ tracks,
                                 const uint8_t* __restrict__ status, int P, float min_sep,
                                 const int32_t* __restrict__ enable) {
  const int b = blockIdx.y;
  if (enable && enable[0] == 0) return;
  const int p = blockIdx.x * kT + threadIdx.x;
  if (p >= P) return;
  const int64_t s = (int64_t)b * P + p;
  if (status[s] != V2D_TRACKED) return;  // only live tracks suppress
  const double tx = tracks[2 * s], ty = tracks[2 * s + 1], r2 = (double)min_sep * min_sep;
  const int rr = (int)ceil((double)min_sep);
  const int x0 = max(0, (int)floor(tx) - rr), x1 = min(W - 1, (int)ceil(tx) + rr);
  const int y0 = max(0, (int)floor(ty) - rr), y1 = min(H - 1, (int)ceil(ty) + rr);
  uint8_t* m = mask_ptrs[b];
  for (int y = y0; y <= y1; ++y)
    for (int x = x0; x <= x1; ++x) {
      const double dx = x - tx, dy = y - ty;
      if (dx * dx + dy * dy < r2) m[(int64_t)y * pitch + x] = 1;  // idempotent
    }
}

__global__ void survival_kernel(const uint8_t* __restrict__ status,
                                const uint8_t* __restrict__ kf_member, int P,
                                int32_t* __restrict__ counts) {
  const int b = blockIdx.x;
  int nk = 0, ns = 0;
  for (int p = threadIdx.x; p < P; p += kT) {
    const int64_t s = (int64_t)b * P + p;
    const int k = kf_member[s] != 0;
    nk += k;
    ns += k & (status[s] == V2D_TRACKED);
  }
  __shared__ int sk[kT / 32], ss[kT / 32];
  for (int o = 16; o > 0; o >>= 1) {
    nk += __shfl_xor_sync(kFullMask, nk, o);
    ns += __shfl_xor_sync(kFullMask, ns, o);
  }
  if ((threadIdx.x & 31) == 0) {
    sk[threadIdx.x >> 5] = nk;
    ss[threadIdx.x >> 5] = ns;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int a = 0, c = 0;
    for (int w = 0; w < kT / 32; ++w) {
      a += sk[w];
      c += ss[w];
    }
    counts[2 * b] = a;      // |S_kf|
    counts[2 * b + 1] = c;  // |S_curr ∩ S_kf|
  }
}

__global__ void decide_kernel(const int32_t* __restrict__ counts, int n, float T,
                              int32_t* __restrict__ flag, int64_t* __restrict__ totals,
                              int64_t* __restrict__ kf_count, unsigned long long cond) {
  if (threadIdx.x != 0) return;
  int64_t nk = 0, ns = 0;
  for (int i = 0; i < n; ++i) {
    nk += counts[2 * i];
    ns += counts[2 * i + 1];
  }
  const int f = (nk == 0 || (double)ns < (double)T * (double)nk) ? 1 : 0;
  flag[0] = f;
  if (totals) {
    totals[0] = nk;
    totals[1] = ns;
  }
  if (kf_count) kf_count[0] += f;
  // captured f1 loop: the keyframe branch is the body of a conditional (IF) graph node
  // whose handle this sets, so on non-keyframe frames its kernels are not launched at all
  if (cond) cudaGraphSetConditional((cudaGraphConditionalHandle)cond, (unsigned)f);
}

// survival_kernel + decide_kernel in one launch (the f1 loop is launch-bound): each CTA
// counts one image, publishes its counts, and the last CTA to finish (device counter
// `done`, left at 0 again) takes the rig-wide Eq. 5 decision exactly as decide_kernel.
__global__ void survival_decide_kernel(const uint8_t* __restrict__ status,
                                       const uint8_t* __restrict__ kf_member, int P,
                                       int32_t* __restrict__ counts, float T,
                                       int32_t* __restrict__ flag, int64_t* __restrict__ totals,
                                       int64_t* __restrict__ kf_count, unsigned long long cond,
                                       unsigned* __restrict__ done) {
  const int b = blockIdx.x, n = gridDim.x;
  int nk = 0, ns = 0;
  for (int p = threadIdx.x; p < P; p += kT) {
    const int64_t s = (int64_t)b * P + p;
    const int k = kf_member[s] != 0;
    nk += k;
    ns += k & (status[s] == V2D_TRACKED);
  }
  __shared__ int sk[kT / 32], ss[kT / 32];
  __shared__ bool last;
  for (int o = 16; o > 0; o >>= 1) {
    nk += __shfl_xor_sync(kFullMask, nk, o);
    ns += __shfl_xor_sync(kFullMask, ns, o);
  }
  if ((threadIdx.x & 31) == 0) {
    sk[threadIdx.x >> 5] = nk;
    ss[threadIdx.x >> 5] = ns;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int a = 0, c = 0;
    for (int w = 0; w < kT / 32; ++w) {
      a += sk[w];
      c += ss[w];
    }
    counts[2 * b] = a;
    counts[2 * b + 1] = c;
    __threadfence();  // this image's counts are visible before it is counted as done
    last = atomicAdd(done, 1u) == (unsigned)(n - 1);
  }
  __syncthreads();
  if (!last || threadIdx.x != 0) return;
  __threadfence();
  int64_t tk = 0, ts = 0;
  for (int i = 0; i < n; ++i) {
    tk += ((volatile int32_t*)counts)[2 * i];
    ts += ((volatile int32_t*)counts)[2 * i + 1];
  }
  const int f = (tk == 0 || (double)ts < (double)T * (double)tk) ? 1 : 0;
  flag[0] = f;
  if (totals) {
    totals[0] = tk;
    totals[1] = ts;
  }
  if (kf_count) kf_count[0] += f;
  *done = 0u;  // ready for the next frame (the next launch is stream-ordered after this one)
  if (cond) cudaGraphSetConditional((cudaGraphConditionalHandle)cond, (unsigned)f);
}

// Frame tables of a captured streaming loop: t = *counter, cur/prev = rows t and t-1
// (mod R) of the [R][C] device-pointer table, then *counter = t + 1.
__global__ void ring_tables_kernel(const int64_t* __restrict__ table, int R, int C,
                                   int64_t* __restrict__ counter, int64_t* __restrict__ cur,
                                   int64_t* __restrict__ prev) {
  const int64_t t = counter[0];
  const int64_t rc = ((t % R) + R) % R, rp = (((t - 1) % R) + R) % R;
  for (int c = threadIdx.x; c < C; c += blockDim.x) {
    cur[c] = table[rc * C + c];
    prev[c] = table[rp * C + c];
  }
  __syncthreads();
  if (threadIdx.x == 0) counter[0] = t + 1;
}

// Block exclusive scan of one int per thread; returns the block total.
__device__ int block_scan(int v, int* sh, int& excl) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int x = v;
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(kFullMask, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) sh[w] = x;
  __syncthreads();
  if (w == 0) {
    int t = lane < kT / 32 ? sh[lane] : 0;
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(kFullMask, t, o);
      if (lane >= o) t += y;
    }
    if (lane < kT / 32) sh[lane] = t;
  }
  __syncthreads();
  const int base = w > 0 ? sh[w - 1] : 0;
  const int total = sh[kT / 32 - 1];
  __syncthreads();
  excl = base + x - v;
  return total;
}

__global__ void refill_kernel(const float* __restrict__ kp_xy, const int32_t* __restrict__ cell_count,
                              int cells, int k, const int32_t* __restrict__ flag, int P,
                              float* __restrict__ tracks, uint8_t* __restrict__ status,
                              uint8_t* __restrict__ kf_member, int32_t* __restrict__ track_id,
                              int32_t* __restrict__ next_id) {
  const int b = blockIdx.x;
  if (flag[0] == 0) return;
  __shared__ int s_cpre[1024 + 1];
  __shared__ int s_scan[kT / 32];
  __shared__ int s_off;
  // prefix over cells of the valid detections (the first cell_count slots of each cell)
  if (threadIdx.x == 0) {
    int acc = 0;
    for (int c = 0; c < cells; ++c) {
      s_cpre[c] = acc;
      acc += cell_count[(int64_t)b * cells + c];
    }
    s_cpre[cells] = acc;
    s_off = 0;
  }
  __syncthreads();
  const int n_new = s_cpre[cells];
  const int id0 = next_id[b];
  for (int p0 = 0; p0 < P; p0 += kT) {
    const int p = p0 + threadIdx.x;
    const int64_t s = (int64_t)b * P + p;
    const int dead = p < P && status[s] != V2D_TRACKED;
    int excl;
    const int tot = block_scan(dead, s_scan, excl);
    const int j = s_off + excl;  // rank of this dead slot
    if (dead && j < n_new) {
      // j-th valid detection: cell c with s_cpre[c] <= j < s_cpre[c+1]
      int lo = 0, hi = cells - 1;
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (s_cpre[mid] <= j) lo = mid; else hi = mid - 1;
      }
      const int64_t src = ((int64_t)b * cells + lo) * k + (j - s_cpre[lo]);
      tracks[2 * s] = kp_xy[2 * src];
      tracks[2 * s + 1] = kp_xy[2 * src + 1];
      status[s] = V2D_TRACKED;
      track_id[s] = id0 + j;
    }
    __syncthreads();
    if (threadIdx.x == 0) s_off += tot;
    __syncthreads();
  }
  __syncthreads();
  for (int p = threadIdx.x; p < P; p += kT) {
    const int64_t s = (int64_t)b * P + p;
    kf_member[s] = status[s] == V2D_TRACKED;
  }
  if (threadIdx.x == 0) next_id[b] = id0 + min(s_off, n_new);
}

}  // namespace

int launch_suppress(uint8_t* const* mask_ptrs, int64_t pitch, int B, int W, int H,
                    const float* tracks, const uint8_t* status, int P, float min_sep,
                    const int32_t* enable, cudaStream_t st) {
  if (B == 0) return V2D_OK;
  clear_mask_kernel<<<dim3(64, B), kT, 0, st>>>(mask_ptrs, pitch, W, H, enable);
  if (P > 0 && min_sep > 0.0f)
    draw_mask_kernel<<<dim3((P + kT - 1) / kT, B), kT, 0, st>>>(mask_ptrs, pitch, W, H, tracks,
                                                                status, P, min_sep, enable);
  return cudaGetLastError() == cudaSuccess ? V2D_OK : V2D_ECUDA;
}

int launch_survival(const uint8_t* status, const uint8_t* kf_member, int B, int P, int32_t* counts,
                    cudaStream_t st) {
  if (B == 0) return V2D_OK;
  survival_kernel<<<B, kT, 0, st>>>(status, kf_member, P, counts);
  return cudaGetLastError() == cudaSuccess ? V2D_OK : V2D_ECUDA;
}

int launch_decide(const int32_t* counts, int n, float T, int32_t* flag, int64_t* totals,
                  int64_t* kf_count, unsigned long long cond, cudaStream_t st) {
  decide_kernel<<<1, 32, 0, st>>>(counts, n, T, flag, totals, kf_count, cond);
  return cudaGetLastError() == cudaSuccess ? V2D_OK : V2D_ECUDA;
}

int launch_survival_decide(const uint8_t* status, const uint8_t* kf_member, int B, int P,
                           int32_t* counts, float T, int32_t* flag, int64_t* totals,
                           int64_t* kf_count, unsigned long long cond, unsigned* done,
                           cudaStream_t st) {
  survival_decide_kernel<<<B, kT, 0, st>>>(status, kf_member, P, counts, T, flag, totals,
                                           kf_count, cond, done);
  return cudaGetLastError() == cudaSuccess ? V2D_OK : V2D_ECUDA;
}

int launch_ring_tables(const int64_t* table, int R, int C, int64_t* counter, int64_t* cur,
                       int64_t* prev, cudaStream_t st) {
  ring_tables_kernel<<<1, 128, 0, st>>>(table, R, C, counter, cur, prev);
  return cudaGetLastError() == cudaSuccess ? V2D_OK : V2D_ECUDA;
}

int launch_refill(const float* kp_xy, const int32_t* cell_count, int cells, int k,
                  const int32_t* flag, int B, int P, float* tracks, uint8_t* status,
                  uint8_t* kf_member, int32_t* track_id, int32_t* next_id, cudaStream_t st) {
  if (B == 0) return V2D_OK;
  refill_kernel<<<B, kT, 0, st>>>(kp_xy, cell_count, cells, k, flag, P, tracks, status, kf_member,
                                  track_id, next_id);
  return cudaGetLastError() == cudaSuccess ? V2D_OK : V2D_ECUDA;
}

}  // namespace v2d
