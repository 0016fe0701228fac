// Pipe-throughput microbenchmarks for the B200 design decisions.
// Each kernel runs ITERS unrolled bodies with independent chains per thread;
// cycles are taken from clock64() per CTA and reported as ops/clk/SM.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

constexpr int ITERS = 4096;

__device__ __forceinline__ unsigned long long f2u(float2 v) { return *reinterpret_cast<unsigned long long*>(&v); }
__device__ __forceinline__ float2 u2f(unsigned long long v) { return *reinterpret_cast<float2*>(&v); }

__global__ void k_ffma(float* out, long long* cyc, float a, float b) {
  float x[8];
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 0.001f + i;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = fmaf(x[i], a, b);
  }
  __syncthreads();
  long long t1 = clock64();
  float s = 0; for (int i = 0; i < 8; ++i) s += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void k_ffma2(float* out, long long* cyc, float a, float b) {
  unsigned long long x[8];
  for (int i = 0; i < 8; ++i) x[i] = f2u(make_float2(threadIdx.x * 0.001f + i, i * 0.5f));
  unsigned long long av = f2u(make_float2(a, a)), bv = f2u(make_float2(b, b));
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(x[i]) : "l"(av), "l"(bv));
  }
  __syncthreads();
  long long t1 = clock64();
  float s = 0; for (int i = 0; i < 8; ++i) { float2 v = u2f(x[i]); s += v.x + v.y; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void k_ex2(float* out, long long* cyc, float a, float b) {
  float x[8];
  for (int i = 0; i < 8; ++i) x[i] = -(threadIdx.x * 0.001f + i) * 0.01f;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x[i])); x[i] = y; }
  }
  __syncthreads();
  long long t1 = clock64();
  float s = 0; for (int i = 0; i < 8; ++i) s += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

// one ex2 + four f32x2 FMAs per body: do MUFU and FMA pipes overlap?
__global__ void k_mix(float* out, long long* cyc, float a, float b) {
  float x[8]; unsigned long long y[8];
  for (int i = 0; i < 8; ++i) { x[i] = -(threadIdx.x * 0.001f + i) * 0.01f; y[i] = f2u(make_float2(i, threadIdx.x)); }
  unsigned long long av = f2u(make_float2(a, a)), bv = f2u(make_float2(b, b));
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      float z; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(z) : "f"(x[i])); x[i] = z;
      asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(y[i]) : "l"(av), "l"(bv));
      asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(y[i]) : "l"(av), "l"(bv));
    }
  }
  __syncthreads();
  long long t1 = clock64();
  float s = 0; for (int i = 0; i < 8; ++i) { float2 v = u2f(y[i]); s += x[i] + v.x + v.y; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

// per-lane private smem column read-modify-write (tile[k][lane]), the forward scatter pattern
__global__ void k_rmw(float* out, long long* cyc, float a, float b) {
  extern __shared__ float sm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  float* col = sm + warp * 128 * 32 + lane;
  for (int k = 0; k < 128; ++k) col[k * 32] = 0.f;
  __syncwarp();
  float c = threadIdx.x * 1e-3f;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < ITERS / 16; ++it) {
    int base = (it * 7 + lane) & 63;
#pragma unroll
    for (int i = 0; i < 32; ++i) { float v = col[(base + i) * 32]; col[(base + i) * 32] = fmaf(c, a, v); }
  }
  __syncthreads();
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = col[lane * 32];
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

// shared-memory float atomics, lanes hitting distinct words of a shared tile
__global__ void k_atoms(float* out, long long* cyc, float a, float b) {
  extern __shared__ float sm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  float* tile = sm + warp * 256;
  for (int k = lane; k < 256; k += 32) tile[k] = 0.f;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < ITERS / 16; ++it) {
#pragma unroll
    for (int i = 0; i < 32; ++i) atomicAdd(&tile[(lane * 5 + i + it) & 255], a);
  }
  __syncthreads();
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = tile[lane];
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

// gather from a smem row with a per-lane start (adjoint residual read pattern), spread < 32
__global__ void k_lds(float* out, long long* cyc, float a, float b) {
  extern __shared__ float sm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  float* row = sm + warp * 512;
  for (int k = lane; k < 512; k += 32) row[k] = k * 0.5f;
  __syncthreads();
  float acc0 = 0, acc1 = 0;
  int start = (lane * 13) & 31;
  long long t0 = clock64();
  for (int it = 0; it < ITERS / 16; ++it) {
#pragma unroll
    for (int i = 0; i < 32; i += 2) { acc0 += row[start + i + (it & 255)]; acc1 += row[start + i + 1 + (it & 255)]; }
  }
  __syncthreads();
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc0 + acc1;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

// fp64 FMA throughput (per-pair setup cost)
__global__ void k_dfma(float* out, long long* cyc, float a, float b) {
  double x[8]; double ad = a, bd = b;
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 0.001 + i;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < ITERS / 4; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = fma(x[i], ad, bd);
  }
  __syncthreads();
  long long t1 = clock64();
  double s = 0; for (int i = 0; i < 8; ++i) s += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = (float)s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

typedef void (*KFn)(float*, long long*, float, float);

static int run(const char* name, KFn fn, int smem, double ops_per_thread_iter, int iters_div, int threads, int blocks_per_sm, int nsm, float* d_out, long long* d_cyc) {
  int blocks = nsm * blocks_per_sm;
  if (smem > 48 * 1024) CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  for (int rep = 0; rep < 2; ++rep) {
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    fn<<<blocks, threads, smem>>>(d_out, d_cyc, 0.999f, 1e-3f);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    CK(cudaGetLastError());
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    long long* h = new long long[blocks];
    CK(cudaMemcpy(h, d_cyc, blocks * sizeof(long long), cudaMemcpyDeviceToHost));
    double mx = 0, mean = 0; for (int i = 0; i < blocks; ++i) { mx = h[i] > mx ? h[i] : mx; mean += h[i]; }
    mean /= blocks; delete[] h;
    double ops_per_block = ops_per_thread_iter * (ITERS / iters_div) * threads;
    double per_sm_clk = ops_per_block * blocks_per_sm / mean;
    double total = ops_per_block * blocks / (ms * 1e-3);
    if (rep == 1)
      printf("{\"bench\": \"%s\", \"threads\": %d, \"ctas_per_sm\": %d, \"ops_per_clk_per_sm\": %.2f, \"ops_per_s\": %.4e, \"ms\": %.4f, \"mean_cycles\": %.0f, \"implied_mhz\": %.0f}\n",
             name, threads, blocks_per_sm, per_sm_clk, total, ms, mean, mean / (ms * 1e3));
  }
  return 0;
}

int main() {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  int nsm = p.multiProcessorCount;
  printf("{\"device\": \"%s\", \"sms\": %d, \"cc\": \"%d.%d\"}\n", p.name, nsm, p.major, p.minor);
  float* d_out; long long* d_cyc;
  CK(cudaMalloc(&d_out, sizeof(float) * nsm * 8 * 1024));
  CK(cudaMalloc(&d_cyc, sizeof(long long) * nsm * 8));
  // ops counted as: FFMA lanes (x2 for flops), FFMA2 lanes count 2 FMAs, ex2 lanes, smem accesses
  run("ffma_fma_per_clk", k_ffma, 0, 8, 1, 256, 4, nsm, d_out, d_cyc);
  run("ffma2_fma_per_clk", k_ffma2, 0, 16, 1, 256, 4, nsm, d_out, d_cyc);
  run("ex2_per_clk", k_ex2, 0, 8, 1, 256, 4, nsm, d_out, d_cyc);
  run("mix_ex2_plus_2ffma2_ex2_per_clk", k_mix, 0, 8, 1, 256, 4, nsm, d_out, d_cyc);
  run("smem_rmw_lane_column_per_clk", k_rmw, 8 * 128 * 32 * 4, 32, 16, 256, 1, nsm, d_out, d_cyc);
  run("smem_atomic_add_f32_per_clk", k_atoms, 8 * 256 * 4, 32, 16, 256, 2, nsm, d_out, d_cyc);
  run("smem_lds_gather_per_clk", k_lds, 8 * 512 * 4, 32, 16, 256, 2, nsm, d_out, d_cyc);
  run("dfma_fma_per_clk", k_dfma, 0, 8, 4, 256, 4, nsm, d_out, d_cyc);
  return 0;
}
