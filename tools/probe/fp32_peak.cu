// Measured FP32 CUDA-core peak for the roofline denominator (bench.py).
// Not part of the product library: a dependency-free probe that runs
// independent FFMA2 (fma.rn.f32x2) chains on every SM and reports FLOP/s.
#include <cstdint>
#include <cuda_runtime.h>

namespace {
constexpr int kIters = 16384;

__global__ void ffma2_chains(float* out, float a, float b) {
  unsigned long long x[8];
  float2 av2 = make_float2(a, a), bv2 = make_float2(b, b);
  unsigned long long av = *reinterpret_cast<unsigned long long*>(&av2);
  unsigned long long bv = *reinterpret_cast<unsigned long long*>(&bv2);
  for (int i = 0; i < 8; ++i) {
    float2 v = make_float2(threadIdx.x * 1e-3f + i, i * 0.5f);
    x[i] = *reinterpret_cast<unsigned long long*>(&v);
  }
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(x[i]) : "l"(av), "l"(bv));
  }
  float s = 0.f;
  for (int i = 0; i < 8; ++i) { float2 v = *reinterpret_cast<float2*>(&x[i]); s += v.x + v.y; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void ex2_chains(float* out, float a) {
  float x[8];
  for (int i = 0; i < 8; ++i) x[i] = -(threadIdx.x * 1e-3f + i) * a;
  for (int it = 0; it < kIters / 4; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x[i])); x[i] = y; }
  }
  float s = 0.f;
  for (int i = 0; i < 8; ++i) s += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
// Private-column shared-memory read-modify-write, the forward tile's access
// pattern (lane l owns bank l of a [rows][32] float tile; LDS + FADD + STS).
__global__ void smem_rmw(float* out, float a) {
  constexpr int kRows = 64;
  __shared__ float tile[4][kRows * 32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float* t = tile[warp] + lane;
  for (int r = 0; r < kRows; ++r) t[r * 32] = 0.0f;
  __syncwarp();
  for (int it = 0; it < kIters / 64; ++it) {
#pragma unroll 1
    for (int r0 = 0; r0 < kRows; r0 += 16) {
      float v[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) v[i] = t[(r0 + i) * 32];
#pragma unroll
      for (int i = 0; i < 16; ++i) t[(r0 + i) * 32] = v[i] + a;
    }
  }
  float s = 0.f;
  for (int r = 0; r < kRows; ++r) s += t[r * 32];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
}  // namespace

extern "C" {
// Returns 0 and fills *rmw (lane read-modify-writes per second).
int probe_smem_rmw(int reps, double* rmw) {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int blocks = sms * 6, threads = 128;
  float* out = nullptr;
  if (cudaMalloc(&out, sizeof(float) * blocks * threads) != cudaSuccess) return 4;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  double best = 0.0;
  for (int r = 0; r < reps; ++r) {
    float ms = 0.f;
    cudaEventRecord(e0);
    smem_rmw<<<blocks, threads>>>(out, 1e-3f);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    const double v = (double)(kIters / 64) * 64.0 * (double)blocks * threads / (ms * 1e-3);
    best = v > best ? v : best;
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(out);
  *rmw = best;
  return cudaGetLastError() == cudaSuccess ? 0 : 4;
}

// Returns 0 and fills *flops (FP32 FLOP/s, FMA = 2) and *ex2 (ex2/s).
int probe_fp32_peak(int reps, double* flops, double* ex2) {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int blocks = sms * 4, threads = 256;
  float* out = nullptr;
  if (cudaMalloc(&out, sizeof(float) * blocks * threads) != cudaSuccess) return 4;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  double best_f = 0.0, best_e = 0.0;
  for (int r = 0; r < reps; ++r) {
    float ms = 0.f;
    cudaEventRecord(e0);
    ffma2_chains<<<blocks, threads>>>(out, 0.9999f, 1e-4f);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    const double f = 2.0 * 2.0 * 8.0 * kIters * (double)blocks * threads / (ms * 1e-3);
    best_f = f > best_f ? f : best_f;
    cudaEventRecord(e0);
    ex2_chains<<<blocks, threads>>>(out, 0.01f);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    const double e = 8.0 * (kIters / 4) * (double)blocks * threads / (ms * 1e-3);
    best_e = e > best_e ? e : best_e;
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(out);
  *flops = best_f;
  *ex2 = best_e;
  return cudaGetLastError() == cudaSuccess ? 0 : 4;
}
}
