// Adjoint moment walk on the legacy tensor path (design experiment, round 2).
//
// The fine adjoint needs, per (ball, detector) pair, the four moments
// T_k = sum_s res_s G(y_s) y_s^k over the ball's window.  Today every lane
// walks one ball and accumulates the moments with FP32x2 FMAs (8 FMA-pipe
// cycles + 8 MUFU cycles per warp-sample).  Here the accumulation is a
// matrix product: with r_s = res_s G_s and the walk index s,
//   M_p = sum_s r_s (s - C)^p   (p = 0..3)
// is R (balls x samples) x V (samples x powers), V a constant table, so the
// sum runs on mma.sync m16n8k8 TF32 (FP32 accumulate).  R is split hi + lo
// (TF32 keeps 10 mantissa bits) and V = V_hi | V_lo in the 8 columns, so one
// MMA per R part gives R_x V_hi and R_x V_lo: ~FP32 accuracy.  G follows the
// forward's ratio recurrence across 8-sample blocks (exact every 4 blocks),
// so MUFU work halves too.  Quad layout: lane (g, t) handles balls g, g+8,
// g+16, g+24 at samples 8kb + 2t, 8kb + 2t + 1 of every block kb.
//
// Reports: mma.sync TF32 rate, the new walk and the current lane-per-ball
// walk in ball-samples/s at 16 warps per SM; checks the MMA moments against
// an FP64 host sum.
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); exit(1); } } while (0)

constexpr int kSegLen = 448;
constexpr int kKbMax = 48;
constexpr float kCentre = 16.0f;

__device__ __forceinline__ float ex2(float x) { float y; asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }

__device__ __forceinline__ void mma_tf32(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0,
                                         uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

__global__ void k_mma_rate(float* out, int iters) {
  float d[8][4] = {};
  const uint32_t a = __float_as_uint(1.0f + threadIdx.x * 1e-3f), b = __float_as_uint(0.5f);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) mma_tf32(d[i], a, a, a, a, b, b);
  }
  float s = 0.f;
  for (int i = 0; i < 8; ++i) s += d[i][0] + d[i][1] + d[i][2] + d[i][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// V table: vt[kb][lane] = (B[k=t][n=g], B[k=t+4][n=g]) for samples s = 8kb+2t, 8kb+2t+1;
// column n < 4: hi part of (s - C)^n, n >= 4: lo part of (s - C)^(n-4)
__host__ __device__ inline float pw(float x, int p) { return p == 0 ? 1.f : p == 1 ? x : p == 2 ? x * x : x * x * x; }
__host__ __device__ inline float tf32_hi(float v) {
#ifdef __CUDA_ARCH__
  return __uint_as_float(__float_as_uint(v) & 0xffffe000u);
#else
  uint32_t u; memcpy(&u, &v, 4); u &= 0xffffe000u; float r; memcpy(&r, &u, 4); return r;
#endif
}

__global__ void k_fill_vt(float2* vt) {
  const int kb = blockIdx.x, lane = threadIdx.x, g = lane >> 2, t = lane & 3;
  float v[2];
  for (int h = 0; h < 2; ++h) {
    const float s = (float)(8 * kb + 2 * t + h) - kCentre;
    const float x = pw(s, g & 3);
    const float hi = tf32_hi(x);
    v[h] = g < 4 ? hi : x - hi;
  }
  vt[kb * 32 + lane] = make_float2(v[0], v[1]);
}

struct BallW { float y0, dl; int off; };

// new walk: nkb blocks of 8 samples; recurrence when `rec`
template <bool REC, bool SPLIT>
__device__ __forceinline__ void mma_walk(const float* seg, const float2* vt, const BallW (&bw)[4], int nkb, float (&d)[2][4]) {
  const int lane = threadIdx.x & 31, t = lane & 3;
  float2 G[4], R[4], C[4];
  const float2* s2[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    s2[i] = reinterpret_cast<const float2*>(seg + bw[i].off + 2 * t);
    const float c = ex2(-128.0f * bw[i].dl * bw[i].dl);
    C[i] = make_float2(c, c);
  }
  auto exact = [&](int kb) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float s0 = (float)(8 * kb + 2 * t);
      const float2 y = __ffma2_rn(make_float2(s0, s0 + 1.0f), make_float2(bw[i].dl, bw[i].dl), make_float2(bw[i].y0, bw[i].y0));
      const float2 q = __fmul2_rn(y, y);
      G[i] = make_float2(ex2(-q.x), ex2(-q.y));
      if (REC) {
        const float a = -16.0f * bw[i].dl, b = -64.0f * bw[i].dl * bw[i].dl;
        const float2 ra = __ffma2_rn(y, make_float2(a, a), make_float2(b, b));
        R[i] = make_float2(ex2(ra.x), ex2(ra.y));
      }
    }
  };
  auto recur = [&]() {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      G[i] = __fmul2_rn(G[i], R[i]);
      R[i] = __fmul2_rn(R[i], C[i]);
    }
  };
  auto accum = [&](int kb) {
    const float2 V = vt[kb * 32 + lane];
    float2 r[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) r[i] = __fmul2_rn(s2[i][4 * kb], G[i]);
    const uint32_t b0 = __float_as_uint(V.x), b1 = __float_as_uint(V.y);
#pragma unroll
    for (int m = 0; m < 2; ++m) {
      const float2 ra = r[2 * m], rb = r[2 * m + 1];
      mma_tf32(d[m], __float_as_uint(ra.x), __float_as_uint(rb.x), __float_as_uint(ra.y), __float_as_uint(rb.y), b0, b1);
      if (SPLIT) {
        const float2 ha = make_float2(tf32_hi(ra.x), tf32_hi(ra.y)), hb = make_float2(tf32_hi(rb.x), tf32_hi(rb.y));
        const float2 la = __fadd2_rn(ra, make_float2(-ha.x, -ha.y)), lb = __fadd2_rn(rb, make_float2(-hb.x, -hb.y));
        mma_tf32(d[m], __float_as_uint(la.x), __float_as_uint(lb.x), __float_as_uint(la.y), __float_as_uint(lb.y), b0, b1);
      }
    }
  };
  if (!REC) {
#pragma unroll 1
    for (int kb = 0; kb < nkb; ++kb) { exact(kb); accum(kb); }
    return;
  }
#pragma unroll 1
  for (int kb = 0; kb < nkb; kb += 4) {
    exact(kb); accum(kb);
    if (kb + 1 >= nkb) break;
    recur(); accum(kb + 1);
    if (kb + 2 >= nkb) break;
    recur(); accum(kb + 2);
    if (kb + 3 >= nkb) break;
    recur(); accum(kb + 3);
  }
}

template <bool REC, bool SPLIT, int WARPS>
__global__ void __launch_bounds__(32 * WARPS) k_mma_walk(const float* segs, const float2* vt_g, const float* ballp, int reps, int L,
                                                         float* out) {
  __shared__ __align__(16) float seg[WARPS][kSegLen];
  __shared__ float2 vt[kKbMax * 32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2;
  for (int i = threadIdx.x; i < kKbMax * 32; i += blockDim.x) vt[i] = vt_g[i];
  for (int i = lane; i < kSegLen; i += 32) seg[warp][i] = segs[i];
  __syncthreads();
  BallW bw[4];
  for (int i = 0; i < 4; ++i) {
    const int b = g + 8 * i;
    bw[i].y0 = ballp[3 * b];
    bw[i].dl = ballp[3 * b + 1];
    bw[i].off = (int)ballp[3 * b + 2];
  }
  float d[2][4] = {};
  const int nkb = L / 8;
  for (int r = 0; r < reps; ++r) {
    BallW b2[4];
    for (int i = 0; i < 4; ++i) { b2[i] = bw[i]; b2[i].off = (bw[i].off + 4 * (r & 7)) & 63; }
    mma_walk<REC, SPLIT>(seg[warp], vt, b2, nkb, d);
  }
  out[(blockIdx.x * WARPS + warp) * 32 + lane] = d[0][0] + d[0][1] + d[0][2] + d[0][3] + d[1][0] + d[1][1] + d[1][2] + d[1][3];
}

// check: one warp, one walk, raw D fragments out
__global__ void k_mma_check(const float* segs, const float2* vt, const float* ballp, int L, int rec, float* dout) {
  __shared__ __align__(16) float seg[kSegLen];
  const int lane = threadIdx.x, g = lane >> 2;
  for (int i = lane; i < kSegLen; i += 32) seg[i] = segs[i];
  __syncwarp();
  BallW bw[4];
  for (int i = 0; i < 4; ++i) {
    const int b = g + 8 * i;
    bw[i].y0 = ballp[3 * b]; bw[i].dl = ballp[3 * b + 1]; bw[i].off = (int)ballp[3 * b + 2];
  }
  float d[2][4] = {};
  if (rec) mma_walk<true, true>(seg, vt, bw, L / 8, d); else mma_walk<false, true>(seg, vt, bw, L / 8, d);
  for (int m = 0; m < 2; ++m) for (int c = 0; c < 4; ++c) dout[(m * 4 + c) * 32 + lane] = d[m][c];
}

// current design: lane = ball, FP32x2 moments (copy of pab_adjoint.cu moments_uniform, fine, unmasked)
__device__ __forceinline__ void moment_pair(float2 res, float2 y, float2& A0, float2& A1, float2& A2, float2& A3) {
  const float2 q = __fmul2_rn(y, y);
  const float2 r = __fmul2_rn(res, make_float2(ex2(-q.x), ex2(-q.y)));
  const float2 t = __fmul2_rn(r, y);
  A1 = __fadd2_rn(A1, t);
  A3 = __ffma2_rn(t, q, A3);
  A0 = __fadd2_rn(A0, r);
  A2 = __ffma2_rn(t, y, A2);
}
__global__ void __launch_bounds__(32) k_old_walk(const float* segs, const float* ballp, int reps, int L, float* out) {
  __shared__ __align__(16) float seg[kSegLen];
  const int lane = threadIdx.x;
  for (int i = lane; i < kSegLen; i += 32) seg[i] = segs[i];
  __syncwarp();
  const float y0 = ballp[3 * lane], dl = ballp[3 * lane + 1];
  const int off0 = (int)ballp[3 * lane + 2];
  float2 A0 = make_float2(0.f, 0.f), A1 = A0, A2 = A0, A3 = A0;
  const float2 dl2 = make_float2(2 * dl, 2 * dl);
  const float2 c0 = make_float2(y0, y0 + dl), c1 = __fadd2_rn(c0, dl2), c2 = __fadd2_rn(c1, dl2), c3 = __fadd2_rn(c2, dl2);
  const float2 st = make_float2(8 * dl, 8 * dl);
  for (int r = 0; r < reps; ++r) {
    const float4* s4 = reinterpret_cast<const float4*>(seg + ((off0 + 4 * (r & 7)) & 63));
    float2 m2 = make_float2(0.f, 0.f);
    int nb = L >> 3;
#pragma unroll 1
    for (; nb >= 2; nb -= 2, s4 += 4) {
      float4 ra = s4[0], rb = s4[1];
      moment_pair(make_float2(ra.x, ra.y), __fadd2_rn(m2, c0), A0, A1, A2, A3);
      moment_pair(make_float2(ra.z, ra.w), __fadd2_rn(m2, c1), A0, A1, A2, A3);
      moment_pair(make_float2(rb.x, rb.y), __fadd2_rn(m2, c2), A0, A1, A2, A3);
      moment_pair(make_float2(rb.z, rb.w), __fadd2_rn(m2, c3), A0, A1, A2, A3);
      m2 = __fadd2_rn(m2, st);
      ra = s4[2]; rb = s4[3];
      moment_pair(make_float2(ra.x, ra.y), __fadd2_rn(m2, c0), A0, A1, A2, A3);
      moment_pair(make_float2(ra.z, ra.w), __fadd2_rn(m2, c1), A0, A1, A2, A3);
      moment_pair(make_float2(rb.x, rb.y), __fadd2_rn(m2, c2), A0, A1, A2, A3);
      moment_pair(make_float2(rb.z, rb.w), __fadd2_rn(m2, c3), A0, A1, A2, A3);
      m2 = __fadd2_rn(m2, st);
    }
  }
  out[blockIdx.x * 32 + lane] = A0.x + A0.y + A1.x + A1.y + A2.x + A2.y + A3.x + A3.y;
}

int main() {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  std::vector<float> h_seg(kSegLen), h_ball(96);
  srand(7);
  for (int i = 0; i < kSegLen; ++i) h_seg[i] = (i < 64 + 8 * kKbMax - 16) ? ((rand() % 2001) - 1000) * 1e-3f : 0.f;
  for (int b = 0; b < 32; ++b) {
    const float dl = -(0.25f + 0.012f * b);   // y decreases along the walk
    h_ball[3 * b] = 5.2f + 0.05f * (b % 5);     // y at walk start
    h_ball[3 * b + 1] = dl;
    h_ball[3 * b + 2] = (float)(4 * (b % 16));
  }
  float *d_seg, *d_ball, *d_out;
  float2* d_vt;
  CK(cudaMalloc(&d_seg, kSegLen * 4));
  CK(cudaMalloc(&d_ball, 96 * 4));
  CK(cudaMalloc(&d_vt, kKbMax * 32 * 8));
  CK(cudaMalloc(&d_out, (size_t)sms * 64 * 32 * 4));
  CK(cudaMemcpy(d_seg, h_seg.data(), kSegLen * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d_ball, h_ball.data(), 96 * 4, cudaMemcpyHostToDevice));
  k_fill_vt<<<kKbMax, 32>>>(d_vt);
  CK(cudaDeviceSynchronize());

  // correctness: moments M_p = sum_s r_s (s - C)^p per ball vs FP64
  for (int rec = 0; rec < 2; ++rec) {
    const int L = 48;
    k_mma_check<<<1, 32>>>(d_seg, d_vt, d_ball, L, rec, d_out);
    CK(cudaDeviceSynchronize());
    std::vector<float> dh(8 * 32);
    CK(cudaMemcpy(dh.data(), d_out, 8 * 32 * 4, cudaMemcpyDeviceToHost));
    double maxrel = 0;
    for (int b = 0; b < 32; ++b) {
      const int m = b / 16, row = b % 16;
      double want[4] = {0, 0, 0, 0}, scale[4] = {0, 0, 0, 0};
      for (int s = 0; s < L; ++s) {
        const double y = h_ball[3 * b] + s * (double)h_ball[3 * b + 1];
        const double r = h_seg[(int)h_ball[3 * b + 2] + s] * exp2(-y * y);
        for (int p = 0; p < 4; ++p) { want[p] += r * pow(s - kCentre, p); scale[p] += fabs(r * pow(s - kCentre, p)); }
      }
      for (int p = 0; p < 4; ++p) {
        // column p (hi) + column p+4 (lo): lane (g = row % 8, t = col / 2), c = (row >= 8) * 2 + col % 2
        auto at = [&](int col) { const int lane = 4 * (row % 8) + col / 2, c = (row >= 8 ? 2 : 0) + col % 2; return (double)dh[(m * 4 + c) * 32 + lane]; };
        const double got = at(p) + at(p + 4);
        maxrel = fmax(maxrel, fabs(got - want[p]) / scale[p]);
      }
    }
    printf("{\"check\": \"mma moments vs fp64\", \"recurrence\": %d, \"max_err_rel_to_abs_sum\": %.3e}\n", rec, maxrel);
  }

  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  auto timeit = [&](auto launch) {
    launch();
    CK(cudaEventRecord(e0));
    launch();
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms; CK(cudaEventElapsedTime(&ms, e0, e1));
    return ms;
  };
  {
    const int iters = 4096, blocks = sms * 16;
    const float ms = timeit([&] { k_mma_rate<<<blocks, 32>>>(d_out, iters); });
    const double mmas = (double)blocks * iters * 8;
    printf("{\"bench\": \"mma.sync m16n8k8 tf32\", \"mma_per_s\": %.4e, \"tflops\": %.1f, \"mma_per_clk_per_sm_at_1965\": %.3f}\n",
           mmas / (ms * 1e-3), mmas * 2048 / (ms * 1e-3) / 1e12, mmas / (ms * 1e-3) / sms / 1.965e9);
  }
  for (int wps : {4, 8, 12, 16}) {   // lane-per-ball walk at 1..4 warps per scheduler
    const int reps = 2000, L = 48, blocks = sms * wps;
    const double bs = (double)blocks * 32 * reps * L;
    const float ms = timeit([&] { k_old_walk<<<blocks, 32>>>(d_seg, d_ball, reps, L, d_out); });
    printf("{\"bench\": \"lane-per-ball walk (current)\", \"warps_per_sm\": %d, \"L\": %d, \"ball_samples_per_s\": %.4e}\n", wps, L, bs / (ms * 1e-3));
  }
  for (int L : {16, 48, 96}) {
    const int reps = 2000;
    const int blocks = sms * 16;
    const double bs = (double)blocks * 32 * reps * L;
    float ms = timeit([&] { k_old_walk<<<blocks, 32>>>(d_seg, d_ball, reps, L, d_out); });
    printf("{\"bench\": \"lane-per-ball walk (current)\", \"L\": %d, \"ball_samples_per_s\": %.4e}\n", L, bs / (ms * 1e-3));
    ms = timeit([&] { k_mma_walk<true, true, 1><<<blocks, 32>>>(d_seg, d_vt, d_ball, reps, L, d_out); });
    printf("{\"bench\": \"mma walk rec+split 1w\", \"L\": %d, \"ball_samples_per_s\": %.4e}\n", L, bs / (ms * 1e-3));
    ms = timeit([&] { k_mma_walk<true, true, 4><<<blocks / 4, 128>>>(d_seg, d_vt, d_ball, reps, L, d_out); });
    printf("{\"bench\": \"mma walk rec+split 4w\", \"L\": %d, \"ball_samples_per_s\": %.4e}\n", L, bs / (ms * 1e-3));
    ms = timeit([&] { k_mma_walk<false, true, 4><<<blocks / 4, 128>>>(d_seg, d_vt, d_ball, reps, L, d_out); });
    printf("{\"bench\": \"mma walk exact+split 4w\", \"L\": %d, \"ball_samples_per_s\": %.4e}\n", L, bs / (ms * 1e-3));
    ms = timeit([&] { k_mma_walk<true, false, 4><<<blocks / 4, 128>>>(d_seg, d_vt, d_ball, reps, L, d_out); });
    printf("{\"bench\": \"mma walk rec nosplit 4w\", \"L\": %d, \"ball_samples_per_s\": %.4e}\n", L, bs / (ms * 1e-3));
  }
  return 0;
}
