// alu_peak.cu — CUDA-core throughput microbenchmarks for the roofline
// denominators of the ALU-bound kernels (K2 integer/issue work, K3 packed fp32).
//
// Each kernel runs kChains independent dependency chains per thread (enough
// to cover the 4-cycle pipe latency at 8+ warps per SMSP), kIters unrolled
// iterations, on 148 x kCtasPerSm CTAs of 256 threads; the result is stored
// only under a data-dependent condition that never holds, so nothing is dead.
//
//   ffma2  : d = fma(a, b, d) on float2 (FFMA2, sm_100) -> 4 flop per lane-instr
//   ffma   : scalar 3-register FFMA                      -> 2 flop per lane-instr
//   ffma_imm: FFMA with an immediate multiplier          -> 2 flop per lane-instr
//   iadd3  : x = x + y + z (IADD3, alu pipe)             -> 1 lane-op
//   mixed  : one FFMA2 + one IADD3 per step (fma and alu pipes co-issue)
//
// Output: one JSON line per kernel with lane-instructions/s and ops/s.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o alu_peak alu_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kChains = 8;
constexpr int kIters = 4096;
constexpr int kThreads = 256;

__global__ void __launch_bounds__(kThreads) k_ffma2(float* out, float s) {
  float2 d[kChains];
  const float2 a = make_float2(s, s * 0.5f), b = make_float2(1e-7f * s, -1e-7f * s);
#pragma unroll
  for (int c = 0; c < kChains; ++c) d[c] = make_float2(threadIdx.x + c, c);
#pragma unroll 16
  for (int i = 0; i < kIters; ++i)
#pragma unroll
    for (int c = 0; c < kChains; ++c) d[c] = __ffma2_rn(d[c], a, b);
  float acc = 0.f;
#pragma unroll
  for (int c = 0; c < kChains; ++c) acc += d[c].x + d[c].y;
  if (acc == 1.2345f) out[threadIdx.x] = acc;
}

__global__ void __launch_bounds__(kThreads) k_ffma(float* out, float s) {
  float d[kChains];
  const float a = s, b = 1e-7f * s;
#pragma unroll
  for (int c = 0; c < kChains; ++c) d[c] = threadIdx.x + c;
#pragma unroll 16
  for (int i = 0; i < kIters; ++i)
#pragma unroll
    for (int c = 0; c < kChains; ++c) d[c] = fmaf(d[c], a, b);
  float acc = 0.f;
#pragma unroll
  for (int c = 0; c < kChains; ++c) acc += d[c];
  if (acc == 1.2345f) out[threadIdx.x] = acc;
}

__global__ void __launch_bounds__(kThreads) k_ffma_imm(float* out, float s) {
  float d[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) d[c] = threadIdx.x + c + s;
#pragma unroll 16
  for (int i = 0; i < kIters; ++i)
#pragma unroll
    for (int c = 0; c < kChains; ++c) d[c] = fmaf(d[c], 0.99999f, 1e-7f);
  float acc = 0.f;
#pragma unroll
  for (int c = 0; c < kChains; ++c) acc += d[c];
  if (acc == 1.2345f) out[threadIdx.x] = acc;
}

__global__ void __launch_bounds__(kThreads) k_iadd3(float* out, float s) {
  unsigned x[kChains];
  const unsigned y = (unsigned)s * 7u + 3u, z = threadIdx.x * 13u + 1u;
#pragma unroll
  for (int c = 0; c < kChains; ++c) x[c] = threadIdx.x * 31u + c;
#pragma unroll 16
  for (int i = 0; i < kIters; ++i)
#pragma unroll
    for (int c = 0; c < kChains; ++c) {
      // x + y + z with a chain-dependent twist (rotating operand) so no closed form exists
      asm volatile("add.u32 %0, %0, %1;\n\tadd.u32 %0, %0, %2;" : "+r"(x[c]) : "r"(y), "r"(z));
    }
  unsigned acc = 0;
#pragma unroll
  for (int c = 0; c < kChains; ++c) acc ^= x[c];
  if (acc == 0x12345u) out[threadIdx.x] = (float)acc;
}

__global__ void __launch_bounds__(kThreads) k_mixed(float* out, float s) {
  float2 d[kChains / 2];
  unsigned x[kChains / 2];
  const float2 a = make_float2(s, s * 0.5f), b = make_float2(1e-7f * s, -1e-7f * s);
  const unsigned y = (unsigned)s * 7u + 3u, z = threadIdx.x * 13u + 1u;
#pragma unroll
  for (int c = 0; c < kChains / 2; ++c) {
    d[c] = make_float2(threadIdx.x + c, c);
    x[c] = threadIdx.x * 31u + c;
  }
#pragma unroll 16
  for (int i = 0; i < kIters; ++i)
#pragma unroll
    for (int c = 0; c < kChains / 2; ++c) {
      d[c] = __ffma2_rn(d[c], a, b);
      asm volatile("add.u32 %0, %0, %1;\n\tadd.u32 %0, %0, %2;" : "+r"(x[c]) : "r"(y), "r"(z));
    }
  float acc = 0.f;
  unsigned ai = 0;
#pragma unroll
  for (int c = 0; c < kChains / 2; ++c) {
    acc += d[c].x + d[c].y;
    ai ^= x[c];
  }
  if (acc == 1.2345f || ai == 0x12345u) out[threadIdx.x] = acc;
}

typedef void (*Kern)(float*, float);

static double time_kernel(Kern k, int blocks, float* out, int reps) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  k<<<blocks, kThreads>>>(out, 1.0f);  // warm-up
  cudaDeviceSynchronize();
  cudaEventRecord(a);
  for (int r = 0; r < reps; ++r) k<<<blocks, kThreads>>>(out, 1.0f);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, a, b);
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  return ms / reps;
}

int main(int argc, char** argv) {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int ctas_per_sm = 8;  // 64 warps per SM (full occupancy at 256-thread CTAs)
  const int blocks = sms * ctas_per_sm;
  float* out = nullptr;
  cudaMalloc(&out, 1024 * sizeof(float));
  const double threads = (double)blocks * kThreads;
  struct {
    const char* name;
    Kern k;
    double lane_instr_per_iter;  // per thread per iteration, all chains
    double ops_per_lane_instr;   // flop (fma = 2) or lane-op
    const char* unit;
  } cases[] = {
      {"ffma2", k_ffma2, (double)kChains, 4.0, "flop"},
      {"ffma", k_ffma, (double)kChains, 2.0, "flop"},
      {"ffma_imm", k_ffma_imm, (double)kChains, 2.0, "flop"},
      {"iadd3", k_iadd3, (double)kChains, 1.0, "lane-op"},
      {"mixed_ffma2_iadd3", k_mixed, (double)kChains, 0.0, "lane-instr"},
  };
  const int reps = argc > 1 ? atoi(argv[1]) : 20;
  for (auto& c : cases) {
    double best = 1e30;
    for (int t = 0; t < 5; ++t) {
      const double ms = time_kernel(c.k, blocks, out, reps);
      if (ms < best) best = ms;
    }
    const double li = threads * kIters * c.lane_instr_per_iter;  // lane-instructions
    const double lis = li / (best * 1e-3);
    printf("{\"kernel\": \"%s\", \"ms\": %.5f, \"sms\": %d, \"blocks\": %d, "
           "\"lane_instr_per_s\": %.6e, \"ops_per_s\": %.6e, \"unit\": \"%s\"}\n",
           c.name, best, sms, blocks, lis, lis * c.ops_per_lane_instr, c.unit);
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    fprintf(stderr, "CUDA error %s\n", cudaGetErrorString(e));
    return 1;
  }
  return 0;
}
