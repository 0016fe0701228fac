// Shared-memory read-modify-write throughput by access width, with the
// forward tile's pattern (lane l owns a private column; rows of a lane are
// contiguous in 16-byte quads: word (q*32 + l)*4 + r).  Prints bytes/s.
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kQuads = 20;   // 80 rows (static smem limit)
template <int W>
__global__ void rmw(float* out, int iters) {
  __shared__ float4 tile[4][kQuads * 32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float4* T = tile[warp] + lane;
  for (int q = 0; q < kQuads; ++q) T[q * 32] = make_float4(0, 0, 0, 0);
  __syncwarp();
  int q = (lane * 3) % kQuads;   // per-lane offsets, like per-lane J0
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int b = 0; b < 8; ++b) {
      int qq = q + 2 * b;
      if (qq >= kQuads) qq -= kQuads;
      if (W == 16) {
        float4 v = T[qq * 32];
        v.x += 1.f; v.y += 1.f; v.z += 1.f; v.w += 1.f;
        T[qq * 32] = v;
      } else if (W == 8) {
        float2* p = reinterpret_cast<float2*>(T + qq * 32);
        float2 a = p[0], c = p[1];
        a.x += 1.f; a.y += 1.f; c.x += 1.f; c.y += 1.f;
        p[0] = a; p[1] = c;
      } else {
        float* p = reinterpret_cast<float*>(T + qq * 32);
        float a = p[0], c = p[1], d = p[2], e = p[3];
        p[0] = a + 1.f; p[1] = c + 1.f; p[2] = d + 1.f; p[3] = e + 1.f;
      }
    }
    q += 1;
    if (q >= kQuads) q = 0;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = T[0].x;
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* out;
  cudaMalloc(&out, sizeof(float) * sms * 8 * 128);
  const int iters = 20000;
  auto run = [&](auto k, const char* name) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    k<<<sms * 2, 128>>>(out, iters);
    cudaEventRecord(a);
    k<<<sms * 2, 128>>>(out, iters);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double bytes = 2.0 * 16.0 * 8 * (double)iters * sms * 2 * 128;   // read + write, 16 B per quad
    printf("{\"access\": \"%s\", \"rmw_bytes_per_s\": %.4e, \"samples_per_s\": %.4e}\n", name, bytes / (ms * 1e-3),
           bytes / 8.0 / (ms * 1e-3));
  };
  run(rmw<16>, "LDS.128/STS.128");
  run(rmw<8>, "LDS.64/STS.64");
  run(rmw<4>, "LDS.32/STS.32");
  return 0;
}
