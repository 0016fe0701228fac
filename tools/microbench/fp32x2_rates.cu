// Throughput of the packed FP32x2 instructions (FFMA2 / FMUL2 / FADD2) and
// their scalar forms on B200: 8 independent chains per thread, 16 warps per
// SM; instructions per clock per SM at the measured clock.
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)
constexpr int IT = 4096;
template <int OP>
__global__ void k(float* out, float a, float b) {
  float2 x[8];
  for (int i = 0; i < 8; ++i) x[i] = make_float2(threadIdx.x * 1e-3f + i, i * 0.5f);
  const float2 A = make_float2(a, a), B = make_float2(b, b);
  for (int it = 0; it < IT; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (OP == 0) x[i] = __ffma2_rn(x[i], A, B);
      if (OP == 1) x[i] = __fmul2_rn(x[i], A);
      if (OP == 2) x[i] = __fadd2_rn(x[i], B);
      if (OP == 3) x[i].x = fmaf(x[i].x, a, x[i].y);          // scalar 3-register FFMA
      if (OP == 4) x[i].x = x[i].x * x[i].y;                  // scalar FMUL
      if (OP == 5) x[i].x = x[i].x + x[i].y;                  // scalar FADD
    }
  }
  float s = 0.f;
  for (int i = 0; i < 8; ++i) s += x[i].x + x[i].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  int sms; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  float* out; CK(cudaMalloc(&out, sms * 16 * 32 * 4 * 4));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const char* names[6] = {"FFMA2", "FMUL2", "FADD2", "FFMA", "FMUL", "FADD"};
  for (int op = 0; op < 6; ++op) {
    auto launch = [&] {
      const int blocks = sms * 4, th = 128;
      if (op == 0) k<0><<<blocks, th>>>(out, 0.999f, 1e-3f);
      if (op == 1) k<1><<<blocks, th>>>(out, 0.999f, 1e-3f);
      if (op == 2) k<2><<<blocks, th>>>(out, 0.999f, 1e-3f);
      if (op == 3) k<3><<<blocks, th>>>(out, 0.999f, 1e-3f);
      if (op == 4) k<4><<<blocks, th>>>(out, 0.999f, 1e-3f);
      if (op == 5) k<5><<<blocks, th>>>(out, 0.999f, 1e-3f);
    };
    launch(); CK(cudaDeviceSynchronize());
    cudaEventRecord(e0); launch(); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    const double warp_instr = (double)sms * 4 * 4 * IT * 8;   // blocks x warps x iterations x chains
    printf("{\"op\": \"%s\", \"warp_instr_per_clk_per_sm\": %.3f, \"cycles_per_warp_instr_per_smsp\": %.2f}\n", names[op],
           warp_instr / (ms * 1e-3) / sms / 1.965e9, 4.0 / (warp_instr / (ms * 1e-3) / sms / 1.965e9));
  }
  return 0;
}
