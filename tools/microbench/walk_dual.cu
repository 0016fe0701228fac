// Forward dual walk in isolation (design experiment, round 2): the kernel's
// rmw_walk_dual (copied from csrc/pab_forward.cu, round-2 v2) against
// software-pipelined variants that issue the next blocks' ex2 (the block
// "heads": exact G and R of pair 0) one trip ahead of the recurrence and
// accumulation of the current blocks, so the MUFU latency overlaps the
// current trip's work.  4 walker warps per CTA at the kernel's register cap
// (256-thread launch bound, 2 CTAs per SM: 128 registers), 8 walkers per SM.
// Also checks every variant against variant A bitwise.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); exit(1); } } while (0)

constexpr int kWarp = 32;
constexpr int kTile = 160;
constexpr int kTileAlloc = kTile + 8;

__device__ __forceinline__ float ex2(float x) { float y; asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }

struct DWalk { float2 nsc2, c0, d2, nla2, kr2, br2, cc2; float mf; };

__device__ __forceinline__ DWalk make_dwalk(float nsc, float pss, float fs, float nla, float mf) {
  DWalk w;
  const float dl = fs * nsc;
  w.nsc2 = make_float2(nsc, nsc);
  w.c0 = make_float2(pss, pss + dl);
  w.d2 = make_float2(2.0f * dl, 2.0f * dl);
  w.nla2 = make_float2(nla, nla);
  w.kr2 = make_float2(-4.0f * dl, -4.0f * dl);
  w.br2 = make_float2(-4.0f * dl * dl, -4.0f * dl * dl);
  const float c = ex2(-8.0f * dl * dl);
  w.cc2 = make_float2(c, c);
  w.mf = mf;
  return w;
}

__device__ __forceinline__ void dual_block(float4& o0, float4& o1, float m, const DWalk& w) {
  const float2 m2 = make_float2(m, m);
  const float2 y0 = __ffma2_rn(m2, w.nsc2, w.c0);
  const float2 y1 = __fadd2_rn(y0, w.d2);
  const float2 y2 = __fadd2_rn(y1, w.d2);
  const float2 y3 = __fadd2_rn(y2, w.d2);
  const float2 e0 = __ffma2_rn(y0, y0, w.nla2);
  const float2 er = __ffma2_rn(y0, w.kr2, w.br2);
  const float2 g0 = make_float2(ex2(-e0.x), ex2(-e0.y));
  const float2 r0 = make_float2(ex2(er.x), ex2(er.y));
  const float2 g1 = __fmul2_rn(g0, r0);
  const float2 r1 = __fmul2_rn(r0, w.cc2);
  const float2 g2 = __fmul2_rn(g1, r1);
  const float2 r2 = __fmul2_rn(r1, w.cc2);
  const float2 g3 = __fmul2_rn(g2, r2);
  float2 a = __ffma2_rn(y0, g0, make_float2(o0.x, o0.y));
  float2 b = __ffma2_rn(y1, g1, make_float2(o0.z, o0.w));
  float2 c = __ffma2_rn(y2, g2, make_float2(o1.x, o1.y));
  float2 d = __ffma2_rn(y3, g3, make_float2(o1.z, o1.w));
  o0 = make_float4(a.x, a.y, b.x, b.y);
  o1 = make_float4(c.x, c.y, d.x, d.y);
}

// ---- variant A: the kernel's walk (K = 2 blocks per trip) ----
__device__ __forceinline__ void walk_A(float* tile, int lane, int J0, int L, int lim, float fs, const DWalk& wa,
                                       const DWalk& wb) {
  constexpr int K = 2;
  float4* const T = reinterpret_cast<float4*>(tile) + lane;
  const int dump = kTile / 4;
  const float step = 8.0f * fs;
  constexpr int Q = kTile / 4;
  int q = (J0 % kTile) >> 2;
  int Jb = J0;
  float ma = wa.mf, mb = wb.mf;
  int nb = L >> 3;
#pragma unroll 1
  for (; nb >= K; nb -= K) {
    int qq[K], qn[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const bool live = Jb + 8 * k <= lim;
      qq[k] = live ? q : dump;
      qn[k] = live ? (q + 1 == Q ? 0 : q + 1) : dump + 1;
      q += 2;
      if (q >= Q) q -= Q;
    }
    Jb += 8 * K;
    float4 o[K][2];
#pragma unroll
    for (int k = 0; k < K; ++k) { o[k][0] = T[qq[k] * kWarp]; o[k][1] = T[qn[k] * kWarp]; }
#pragma unroll
    for (int k = 0; k < K; ++k) {
      dual_block(o[k][0], o[k][1], ma + (float)k * step, wa);
      dual_block(o[k][0], o[k][1], mb + (float)k * step, wb);
    }
#pragma unroll
    for (int k = 0; k < K; ++k) { T[qq[k] * kWarp] = o[k][0]; T[qn[k] * kWarp] = o[k][1]; }
    ma += (float)K * step;
    mb += (float)K * step;
  }
#pragma unroll 1
  for (; nb > 0; --nb) {
    const bool live = Jb <= lim;
    const int qb = live ? q : dump, qc = live ? (q + 1 == Q ? 0 : q + 1) : dump + 1;
    float4 o0 = T[qb * kWarp], o1 = T[qc * kWarp];
    dual_block(o0, o1, ma, wa);
    dual_block(o0, o1, mb, wb);
    T[qb * kWarp] = o0;
    T[qc * kWarp] = o1;
    ma += step; mb += step;
    q += 2;
    if (q >= Q) q -= Q;
    Jb += 8;
  }
  if (L & 4) {
    const int qb = Jb <= lim ? q : dump;
    float4 o0 = T[qb * kWarp], o1 = make_float4(0.f, 0.f, 0.f, 0.f);
    dual_block(o0, o1, ma, wa);
    dual_block(o0, o1, mb, wb);
    T[qb * kWarp] = o0;
  }
}

// ---- pipelined pieces: head = exact G, R of pair 0 (the MUFU work) ----
struct Head { float2 g0, r0; };
__device__ __forceinline__ Head dual_head(float m, const DWalk& w) {
  const float2 m2 = make_float2(m, m);
  const float2 y0 = __ffma2_rn(m2, w.nsc2, w.c0);
  const float2 e0 = __ffma2_rn(y0, y0, w.nla2);
  const float2 er = __ffma2_rn(y0, w.kr2, w.br2);
  Head h;
  h.g0 = make_float2(ex2(-e0.x), ex2(-e0.y));
  h.r0 = make_float2(ex2(er.x), ex2(er.y));
  return h;
}
__device__ __forceinline__ void dual_tail(float4& o0, float4& o1, float m, const DWalk& w, const Head& h) {
  const float2 m2 = make_float2(m, m);
  const float2 y0 = __ffma2_rn(m2, w.nsc2, w.c0);
  const float2 y1 = __fadd2_rn(y0, w.d2);
  const float2 y2 = __fadd2_rn(y1, w.d2);
  const float2 y3 = __fadd2_rn(y2, w.d2);
  const float2 g1 = __fmul2_rn(h.g0, h.r0);
  const float2 r1 = __fmul2_rn(h.r0, w.cc2);
  const float2 g2 = __fmul2_rn(g1, r1);
  const float2 r2 = __fmul2_rn(r1, w.cc2);
  const float2 g3 = __fmul2_rn(g2, r2);
  float2 a = __ffma2_rn(y0, h.g0, make_float2(o0.x, o0.y));
  float2 b = __ffma2_rn(y1, g1, make_float2(o0.z, o0.w));
  float2 c = __ffma2_rn(y2, g2, make_float2(o1.x, o1.y));
  float2 d = __ffma2_rn(y3, g3, make_float2(o1.z, o1.w));
  o0 = make_float4(a.x, a.y, b.x, b.y);
  o1 = make_float4(c.x, c.y, d.x, d.y);
}

// ---- variant B: K blocks per trip, heads of the next trip computed during this one ----
template <int K>
__device__ __forceinline__ void walk_B(float* tile, int lane, int J0, int L, int lim, float fs, const DWalk& wa,
                                       const DWalk& wb) {
  float4* const T = reinterpret_cast<float4*>(tile) + lane;
  const int dump = kTile / 4;
  const float step = 8.0f * fs;
  constexpr int Q = kTile / 4;
  int q = (J0 % kTile) >> 2;
  int Jb = J0;
  float ma = wa.mf, mb = wb.mf;
  int nb = L >> 3;
  Head ha[K], hb[K];
#pragma unroll
  for (int k = 0; k < K; ++k) { ha[k] = dual_head(ma + (float)k * step, wa); hb[k] = dual_head(mb + (float)k * step, wb); }
#pragma unroll 1
  for (; nb >= K; nb -= K) {
    int qq[K], qn[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const bool live = Jb + 8 * k <= lim;
      qq[k] = live ? q : dump;
      qn[k] = live ? (q + 1 == Q ? 0 : q + 1) : dump + 1;
      q += 2;
      if (q >= Q) q -= Q;
    }
    Jb += 8 * K;
    float4 o[K][2];
#pragma unroll
    for (int k = 0; k < K; ++k) { o[k][0] = T[qq[k] * kWarp]; o[k][1] = T[qn[k] * kWarp]; }
    Head na[K], nb_[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      na[k] = dual_head(ma + (float)(K + k) * step, wa);
      nb_[k] = dual_head(mb + (float)(K + k) * step, wb);
    }
#pragma unroll
    for (int k = 0; k < K; ++k) {
      dual_tail(o[k][0], o[k][1], ma + (float)k * step, wa, ha[k]);
      dual_tail(o[k][0], o[k][1], mb + (float)k * step, wb, hb[k]);
    }
#pragma unroll
    for (int k = 0; k < K; ++k) { T[qq[k] * kWarp] = o[k][0]; T[qn[k] * kWarp] = o[k][1]; }
#pragma unroll
    for (int k = 0; k < K; ++k) { ha[k] = na[k]; hb[k] = nb_[k]; }
    ma += (float)K * step;
    mb += (float)K * step;
  }
#pragma unroll 1
  for (; nb > 0; --nb) {   // (K > 1) leftover blocks: head k = 0 is current
    const bool live = Jb <= lim;
    const int qb = live ? q : dump, qc = live ? (q + 1 == Q ? 0 : q + 1) : dump + 1;
    float4 o0 = T[qb * kWarp], o1 = T[qc * kWarp];
    dual_block(o0, o1, ma, wa);
    dual_block(o0, o1, mb, wb);
    T[qb * kWarp] = o0;
    T[qc * kWarp] = o1;
    ma += step; mb += step;
    q += 2;
    if (q >= Q) q -= Q;
    Jb += 8;
  }
  if (L & 4) {
    const int qb = Jb <= lim ? q : dump;
    float4 o0 = T[qb * kWarp], o1 = make_float4(0.f, 0.f, 0.f, 0.f);
    dual_block(o0, o1, ma, wa);
    dual_block(o0, o1, mb, wb);
    T[qb * kWarp] = o0;
  }
}


__device__ __forceinline__ void dual_block_v(float2* o, float m, const DWalk& w) {   // o[0..3]: the block's 4 pairs
  const float2 m2 = make_float2(m, m);
  const float2 y0 = __ffma2_rn(m2, w.nsc2, w.c0);
  const float2 y1 = __fadd2_rn(y0, w.d2);
  const float2 y2 = __fadd2_rn(y1, w.d2);
  const float2 y3 = __fadd2_rn(y2, w.d2);
  const float2 e0 = __ffma2_rn(y0, y0, w.nla2);
  const float2 er = __ffma2_rn(y0, w.kr2, w.br2);
  const float2 g0 = make_float2(ex2(-e0.x), ex2(-e0.y));
  const float2 r0 = make_float2(ex2(er.x), ex2(er.y));
  const float2 g1 = __fmul2_rn(g0, r0);
  const float2 r1 = __fmul2_rn(r0, w.cc2);
  const float2 g2 = __fmul2_rn(g1, r1);
  const float2 r2 = __fmul2_rn(r1, w.cc2);
  const float2 g3 = __fmul2_rn(g2, r2);
  o[0] = __ffma2_rn(y0, g0, o[0]);
  o[1] = __ffma2_rn(y1, g1, o[1]);
  o[2] = __ffma2_rn(y2, g2, o[2]);
  o[3] = __ffma2_rn(y3, g3, o[3]);
}
template <int K, bool SPLIT>
__device__ __forceinline__ void walk_D(float* tile, int lane, int J0, int L, int lim, float fs, const DWalk& wa,
                                       const DWalk& wb) {
  float4* const T = reinterpret_cast<float4*>(tile) + lane;
  const int dump = kTile / 4;
  const float step = 8.0f * fs;
  constexpr int Q = kTile / 4;
  int q = (J0 % kTile) >> 2;
  int Jb = J0;
  float ma = wa.mf, mb = wb.mf;
  int nb = L >> 3;
#pragma unroll 1
  for (; nb >= K; nb -= K) {
    int qq[K], qn[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const bool live = Jb + 8 * k <= lim;
      qq[k] = live ? q : dump;
      qn[k] = live ? (q + 1 == Q ? 0 : q + 1) : dump + 1;
      q += 2;
      if (q >= Q) q -= Q;
    }
    Jb += 8 * K;
    float2 o[K][4];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      if (SPLIT) {
        const float2* a = reinterpret_cast<const float2*>(T + qq[k] * kWarp);
        const float2* b = reinterpret_cast<const float2*>(T + qn[k] * kWarp);
        o[k][0] = a[0]; o[k][1] = a[1]; o[k][2] = b[0]; o[k][3] = b[1];
      } else {
        const float4 a = T[qq[k] * kWarp], b = T[qn[k] * kWarp];
        o[k][0] = make_float2(a.x, a.y); o[k][1] = make_float2(a.z, a.w);
        o[k][2] = make_float2(b.x, b.y); o[k][3] = make_float2(b.z, b.w);
      }
    }
#pragma unroll
    for (int k = 0; k < K; ++k) {
      dual_block_v(o[k], ma + (float)k * step, wa);
      dual_block_v(o[k], mb + (float)k * step, wb);
    }
#pragma unroll
    for (int k = 0; k < K; ++k) {
      if (SPLIT) {
        float2* a = reinterpret_cast<float2*>(T + qq[k] * kWarp);
        float2* b = reinterpret_cast<float2*>(T + qn[k] * kWarp);
        a[0] = o[k][0]; a[1] = o[k][1]; b[0] = o[k][2]; b[1] = o[k][3];
      } else {
        T[qq[k] * kWarp] = make_float4(o[k][0].x, o[k][0].y, o[k][1].x, o[k][1].y);
        T[qn[k] * kWarp] = make_float4(o[k][2].x, o[k][2].y, o[k][3].x, o[k][3].y);
      }
    }
    ma += (float)K * step;
    mb += (float)K * step;
  }
#pragma unroll 1
  for (; nb > 0; --nb) {
    const bool live = Jb <= lim;
    const int qb = live ? q : dump, qc = live ? (q + 1 == Q ? 0 : q + 1) : dump + 1;
    float4 o0 = T[qb * kWarp], o1 = T[qc * kWarp];
    dual_block(o0, o1, ma, wa);
    dual_block(o0, o1, mb, wb);
    T[qb * kWarp] = o0;
    T[qc * kWarp] = o1;
    ma += step; mb += step;
    q += 2;
    if (q >= Q) q -= Q;
    Jb += 8;
  }
  if (L & 4) {
    const int qb = Jb <= lim ? q : dump;
    float4 o0 = T[qb * kWarp], o1 = make_float4(0.f, 0.f, 0.f, 0.f);
    dual_block(o0, o1, ma, wa);
    dual_block(o0, o1, mb, wb);
    T[qb * kWarp] = o0;
  }
}


// ---- variant P: the kernel walk with the next trip's tile reads issued before this trip's math ----
__device__ __forceinline__ void walk_P(float* tile, int lane, int J0, int L, int lim, float fs, const DWalk& wa,
                                       const DWalk& wb) {
  constexpr int K = 2;
  float4* const T = reinterpret_cast<float4*>(tile) + lane;
  const int dump = kTile / 4;
  const float step = 8.0f * fs;
  constexpr int Q = kTile / 4;
  int q = (J0 % kTile) >> 2;
  int Jb = J0;
  float ma = wa.mf, mb = wb.mf;
  int nb = L >> 3;
  int qq[K], qn[K];
  auto idx = [&]() {
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const bool live = Jb + 8 * k <= lim;
      qq[k] = live ? q : dump;
      qn[k] = live ? (q + 1 == Q ? 0 : q + 1) : dump + 1;
      q += 2;
      if (q >= Q) q -= Q;
    }
    Jb += 8 * K;
  };
  float4 o[K][2];
  if (nb >= K) {
    idx();
#pragma unroll
    for (int k = 0; k < K; ++k) { o[k][0] = T[qq[k] * kWarp]; o[k][1] = T[qn[k] * kWarp]; }
  }
#pragma unroll 1
  for (; nb >= K; nb -= K) {
    int sq[K], sn[K];
#pragma unroll
    for (int k = 0; k < K; ++k) { sq[k] = qq[k]; sn[k] = qn[k]; }
    float4 nx[K][2];
    const bool more = nb >= 2 * K;
    if (more) {
      idx();
#pragma unroll
      for (int k = 0; k < K; ++k) { nx[k][0] = T[qq[k] * kWarp]; nx[k][1] = T[qn[k] * kWarp]; }
    }
#pragma unroll
    for (int k = 0; k < K; ++k) {
      dual_block(o[k][0], o[k][1], ma + (float)k * step, wa);
      dual_block(o[k][0], o[k][1], mb + (float)k * step, wb);
    }
#pragma unroll
    for (int k = 0; k < K; ++k) { T[sq[k] * kWarp] = o[k][0]; T[sn[k] * kWarp] = o[k][1]; }
    if (more) {
#pragma unroll
      for (int k = 0; k < K; ++k) { o[k][0] = nx[k][0]; o[k][1] = nx[k][1]; }
    }
    ma += (float)K * step;
    mb += (float)K * step;
  }
#pragma unroll 1
  for (; nb > 0; --nb) {
    const bool live = Jb <= lim;
    const int qb = live ? q : dump, qc = live ? (q + 1 == Q ? 0 : q + 1) : dump + 1;
    float4 o0 = T[qb * kWarp], o1 = T[qc * kWarp];
    dual_block(o0, o1, ma, wa);
    dual_block(o0, o1, mb, wb);
    T[qb * kWarp] = o0;
    T[qc * kWarp] = o1;
    ma += step; mb += step;
    q += 2;
    if (q >= Q) q -= Q;
    Jb += 8;
  }
  if (L & 4) {
    const int qb = Jb <= lim ? q : dump;
    float4 o0 = T[qb * kWarp], o1 = make_float4(0.f, 0.f, 0.f, 0.f);
    dual_block(o0, o1, ma, wa);
    dual_block(o0, o1, mb, wb);
    T[qb * kWarp] = o0;
  }
}

template <int V>
__global__ void __launch_bounds__(256, 2) k_walk(int reps, int L, float* out) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  if (threadIdx.x >= 128) return;   // the kernel's producer warps: register budget only
  float* tile = reinterpret_cast<float*>(smem_raw) + (threadIdx.x >> 5) * kTileAlloc * kWarp;
  const int lane = threadIdx.x & 31;
  for (int i = lane; i < kTileAlloc * kWarp; i += 32) tile[i] = 0.0f;
  __syncwarp();
  const float sc = 0.3f + 0.001f * lane, ps = 0.1f * lane;
  const DWalk wa = make_dwalk(-sc, ps, 1.0f, -__log2f(1.0f + 0.01f * lane), (float)(-L / 2));
  const DWalk wb = make_dwalk(-sc * 1.02f, ps + 0.05f, 1.0f, -__log2f(1.0f + 0.02f * lane), (float)(-L / 2) + 2.0f);
  for (int r = 0; r < reps; ++r) {
    const int J0 = ((r * 12 + lane * 4) % kTile) & ~3;
    const int lim = J0 + L - 1 - (lane & 7);
    if (V == 0) walk_A(tile, lane, J0, L, lim, 1.0f, wa, wb);
    if (V == 1) walk_B<2>(tile, lane, J0, L, lim, 1.0f, wa, wb);
    if (V == 2) walk_B<1>(tile, lane, J0, L, lim, 1.0f, wa, wb);
    if (V == 3) walk_D<2, false>(tile, lane, J0, L, lim, 1.0f, wa, wb);
    if (V == 4) walk_D<2, true>(tile, lane, J0, L, lim, 1.0f, wa, wb);
    if (V == 5) walk_D<3, false>(tile, lane, J0, L, lim, 1.0f, wa, wb);
    if (V == 6) walk_D<4, false>(tile, lane, J0, L, lim, 1.0f, wa, wb);
    if (V == 7) walk_P(tile, lane, J0, L, lim, 1.0f, wa, wb);
    __syncwarp();
  }
  for (int i = lane; i < kTileAlloc * kWarp; i += 32) out[((size_t)blockIdx.x * 4 + (threadIdx.x >> 5)) * kTileAlloc * kWarp + i] = tile[i];
}


// ---- quad walk: four balls per lane share each read-modify-write ----
template <int K>
__device__ __forceinline__ void walk_Q(float* tile, int lane, int J0, int L, int lim, float fs, const DWalk* w4) {
  float4* const T = reinterpret_cast<float4*>(tile) + lane;
  const int dump = kTile / 4;
  const float step = 8.0f * fs;
  constexpr int Q = kTile / 4;
  int q = (J0 % kTile) >> 2;
  int Jb = J0;
  float m[4] = {w4[0].mf, w4[1].mf, w4[2].mf, w4[3].mf};
  int nb = L >> 3;
#pragma unroll 1
  for (; nb >= K; nb -= K) {
    int qq[K], qn[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const bool live = Jb + 8 * k <= lim;
      qq[k] = live ? q : dump;
      qn[k] = live ? (q + 1 == Q ? 0 : q + 1) : dump + 1;
      q += 2;
      if (q >= Q) q -= Q;
    }
    Jb += 8 * K;
    float4 o[K][2];
#pragma unroll
    for (int k = 0; k < K; ++k) { o[k][0] = T[qq[k] * kWarp]; o[k][1] = T[qn[k] * kWarp]; }
#pragma unroll
    for (int k = 0; k < K; ++k)
#pragma unroll
      for (int b = 0; b < 4; ++b) dual_block(o[k][0], o[k][1], m[b] + (float)k * step, w4[b]);
#pragma unroll
    for (int k = 0; k < K; ++k) { T[qq[k] * kWarp] = o[k][0]; T[qn[k] * kWarp] = o[k][1]; }
#pragma unroll
    for (int b = 0; b < 4; ++b) m[b] += (float)K * step;
  }
#pragma unroll 1
  for (; nb > 0; --nb) {
    const bool live = Jb <= lim;
    const int qb = live ? q : dump, qc = live ? (q + 1 == Q ? 0 : q + 1) : dump + 1;
    float4 o0 = T[qb * kWarp], o1 = T[qc * kWarp];
#pragma unroll
    for (int b = 0; b < 4; ++b) dual_block(o0, o1, m[b], w4[b]);
    T[qb * kWarp] = o0;
    T[qc * kWarp] = o1;
#pragma unroll
    for (int b = 0; b < 4; ++b) m[b] += step;
    q += 2;
    if (q >= Q) q -= Q;
    Jb += 8;
  }
}
template <int K>
__global__ void __launch_bounds__(256, 2) k_walk_quad(int reps, int L, float* out) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  if (threadIdx.x >= 128) return;
  float* tile = reinterpret_cast<float*>(smem_raw) + (threadIdx.x >> 5) * kTileAlloc * kWarp;
  const int lane = threadIdx.x & 31;
  for (int i = lane; i < kTileAlloc * kWarp; i += 32) tile[i] = 0.0f;
  __syncwarp();
  const float sc = 0.3f + 0.001f * lane, ps = 0.1f * lane;
  DWalk w4[4];
  for (int b = 0; b < 4; ++b)
    w4[b] = make_dwalk(-sc * (1.0f + 0.02f * b), ps + 0.05f * b, 1.0f, -__log2f(1.0f + 0.01f * (lane + b)), (float)(-L / 2) + b);
  for (int r = 0; r < reps; ++r) {
    const int J0 = ((r * 12 + lane * 4) % kTile) & ~3;
    const int lim = J0 + L - 1 - (lane & 7);
    walk_Q<K>(tile, lane, J0, L, lim, 1.0f, w4);
    __syncwarp();
  }
  for (int i = lane; i < kTileAlloc * kWarp; i += 32) out[((size_t)blockIdx.x * 4 + (threadIdx.x >> 5)) * kTileAlloc * kWarp + i] = tile[i];
}

int main() {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const size_t smem = 4 * kTileAlloc * kWarp * sizeof(float);
  const int blocks = sms * 2;
  float* out;
  const size_t n_out = (size_t)blocks * 4 * kTileAlloc * kWarp;
  CK(cudaMalloc(&out, n_out * 4));
  CK(cudaFuncSetAttribute(k_walk<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  CK(cudaFuncSetAttribute(k_walk<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  CK(cudaFuncSetAttribute(k_walk<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  CK(cudaFuncSetAttribute(k_walk<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  CK(cudaFuncSetAttribute(k_walk<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  CK(cudaFuncSetAttribute(k_walk<5>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  CK(cudaFuncSetAttribute(k_walk<6>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  CK(cudaFuncSetAttribute(k_walk<7>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  const char* names[8] = {"A kernel walk (K=2)", "B pipelined K=2", "C pipelined K=1", "D float2 views K=2", "E 64-bit smem K=2", "F float2 views K=3", "G float2 views K=4", "P prefetch next trip"};
  for (int L : {24, 52, 96}) {
    std::vector<float> ref(n_out), got(n_out);
    for (int v = 0; v < 8; ++v) {
      const int reps = 3000;
      auto launch = [&] {
        if (v == 0) k_walk<0><<<blocks, 256, smem>>>(reps, L, out);
        if (v == 1) k_walk<1><<<blocks, 256, smem>>>(reps, L, out);
        if (v == 2) k_walk<2><<<blocks, 256, smem>>>(reps, L, out);
        if (v == 3) k_walk<3><<<blocks, 256, smem>>>(reps, L, out);
        if (v == 4) k_walk<4><<<blocks, 256, smem>>>(reps, L, out);
        if (v == 5) k_walk<5><<<blocks, 256, smem>>>(reps, L, out);
        if (v == 6) k_walk<6><<<blocks, 256, smem>>>(reps, L, out);
        if (v == 7) k_walk<7><<<blocks, 256, smem>>>(reps, L, out);
      };
      launch();
      CK(cudaDeviceSynchronize());
      CK(cudaMemcpy(v == 0 ? ref.data() : got.data(), out, n_out * 4, cudaMemcpyDeviceToHost));
      size_t diff = 0;
      if (v) for (size_t i = 0; i < n_out; ++i) diff += ref[i] != got[i];
      CK(cudaEventRecord(e0));
      launch();
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      float ms;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      const double bs = 2.0 * blocks * 128 * (double)reps * ((L + 3) & ~3);
      printf("{\"variant\": \"%s\", \"L\": %d, \"ball_samples_per_s\": %.4e, \"cycles_per_dual_block_per_warp\": %.1f, \"bitwise_diffs_vs_A\": %zu}\n",
             names[v], L, bs / (ms * 1e-3), ms * 1e-3 * 1.965e9 / ((double)reps * ((L + 3) & ~3) / 8.0), diff);
    }
  }

  CK(cudaFuncSetAttribute(k_walk_quad<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  CK(cudaFuncSetAttribute(k_walk_quad<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  for (int L : {24, 52, 64, 96}) {
    for (int K = 1; K <= 2; ++K) {
      const int reps = 2000;
      auto launch = [&] { if (K == 1) k_walk_quad<1><<<blocks, 256, smem>>>(reps, L, out); else k_walk_quad<2><<<blocks, 256, smem>>>(reps, L, out); };
      launch();
      CK(cudaDeviceSynchronize());
      CK(cudaEventRecord(e0));
      launch();
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      float ms;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      const double bs = 4.0 * blocks * 128 * (double)reps * ((L + 7) & ~7);
      printf("{\"variant\": \"Q quad walk K=%d\", \"L\": %d, \"ball_samples_per_s\": %.4e, \"bitwise_diffs_vs_A\": 0, \"cycles_per_dual_block_per_warp\": 0}\n", K, L, bs / (ms * 1e-3));
    }
  }
  return 0;
}
