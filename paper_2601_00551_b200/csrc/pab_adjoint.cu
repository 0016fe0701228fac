// Adjoint: residual -> per-ball loss gradients.
//
// Replaces reference radiator.py:263-287 (gather of the residual over each
// cached slab window, einsum reductions, per-ball gradient assembly) and the
// fixed-order block merge :336-348.
//
// Decomposition: a warp owns one lane group (32 balls of similar radius, one
// per lane, so all lanes walk windows of nearly equal length) and loops over a
// chunk of detectors in batches of 32.  Lane l of a batch computes detector
// l's group geometry (FP64) once and leaves it in a per-warp shared-memory
// table; per detector the warp reads it back by broadcast LDS.128.  The
// residual segment the group can touch is staged into one of four
// shared-memory segments with cp.async a detector pair ahead; detectors go
// in pairs whose setups and gradient terms are computed side by side.  Every
// lane walks its own arrival window accumulating four FP32 moments
//   T_k = sum_J res[J] G(y_J) y_J^k,  k = 0..3,
// with paired FP32x2 arithmetic (FFMA2/FMUL2/FADD2), 16 samples per iteration
// and 128-bit shared loads: the fine stage as a two-sided cascade of running
// sums with the Gaussian by a ratio recurrence (moments_cascade: 6 FP32x2 + 1
// ex2 per sample pair), the other stages, masked cutoffs and out-of-range
// steps as the direct walk (moments_uniform: 8 FP32x2 + 2 ex2).  Per-pair
// gradient terms are summed in FP32 over a batch of 32 detectors and folded
// into FP64 per-ball accumulators kept in shared memory across the chunk (no
// atomics).  Detector chunks (grid.y) write partial sums that the finalize
// pass adds in chunk order.
#include "pab_common.cuh"

namespace pab {

constexpr int kSeg = 256;   // staged residual samples per warp and buffer
constexpr int kPad = 96;    // zero padding after the staged samples (uniform-walk overrun)

__device__ __forceinline__ void cp_async4(float* smem_dst, const float* gsrc) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(s), "l"(gsrc));
}
__device__ __forceinline__ void cp_async16(float* smem_dst, const float* gsrc) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gsrc));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

struct Moments {
  float T0, T1, T2, T3;
};

template <int STAGE>
__device__ __forceinline__ void moment_scalar(float res, float m, float sc, float ps, Moments& M) {
  const float y = fmaf(m, -sc, ps);
  const float q = y * y;
  const float r = res * ex2(-q);
  const float t = r * y;
  M.T1 += t;
  if (STAGE >= kStageCoarse) M.T3 = fmaf(t, q, M.T3);
  if (STAGE == kStageFine) {
    M.T0 += r;
    M.T2 = fmaf(t, y, M.T2);
  }
}

template <int STAGE>
__device__ __forceinline__ void moment_pair(float2 res, float2 y, float2& A0, float2& A1, float2& A2, float2& A3) {
  const float2 q = __fmul2_rn(y, y);
  const float2 r = __fmul2_rn(res, make_float2(ex2(-q.x), ex2(-q.y)));
  const float2 t = __fmul2_rn(r, y);
  A1 = __fadd2_rn(A1, t);
  if (STAGE >= kStageCoarse) A3 = __ffma2_rn(t, q, A3);
  if (STAGE == kStageFine) {
    A0 = __fadd2_rn(A0, r);
    A2 = __ffma2_rn(t, y, A2);
  }
}

// Walk n samples of one window: seg[off + i] is the residual of the i-th
// sample (seg 8-byte aligned), m0 its m-offset (J f - kc), step fs.
template <int STAGE>
__device__ __forceinline__ void moments_run(const float* seg, int off, int n, float m0, float fs, float sc, float ps,
                                            Moments& M) {
  if (n <= 0) return;
  if (reinterpret_cast<uintptr_t>(seg + off) & 7) {   // peel to an 8-byte aligned start
    moment_scalar<STAGE>(seg[off], m0, sc, ps, M);
    ++off;
    --n;
    m0 += fs;
  }
  const float2* s2 = reinterpret_cast<const float2*>(seg + off);
  float2 A0 = make_float2(0.f, 0.f), A1 = A0, A2 = A0, A3 = A0;
  const float2 nsc2 = make_float2(-sc, -sc);
  // y of pair k of an 8-sample block: (mb + 2k fs, mb + (2k+1) fs) * -sc + ps
  const float2 c0 = make_float2(ps, fmaf(fs, -sc, ps));
  const float2 c1 = make_float2(fmaf(2.0f * fs, -sc, ps), fmaf(3.0f * fs, -sc, ps));
  const float2 c2 = make_float2(fmaf(4.0f * fs, -sc, ps), fmaf(5.0f * fs, -sc, ps));
  const float2 c3 = make_float2(fmaf(6.0f * fs, -sc, ps), fmaf(7.0f * fs, -sc, ps));
  float mb = m0;
  int i = 0;
#pragma unroll 1
  for (; i + 8 <= n; i += 8, mb += 8.0f * fs, s2 += 4) {
    const float2 m2 = make_float2(mb, mb);
    const float2 r0 = s2[0], r1 = s2[1], r2 = s2[2], r3 = s2[3];
    moment_pair<STAGE>(r0, __ffma2_rn(m2, nsc2, c0), A0, A1, A2, A3);
    moment_pair<STAGE>(r1, __ffma2_rn(m2, nsc2, c1), A0, A1, A2, A3);
    moment_pair<STAGE>(r2, __ffma2_rn(m2, nsc2, c2), A0, A1, A2, A3);
    moment_pair<STAGE>(r3, __ffma2_rn(m2, nsc2, c3), A0, A1, A2, A3);
  }
#pragma unroll 1
  for (; i + 2 <= n; i += 2, mb += 2.0f * fs, ++s2) {
    moment_pair<STAGE>(s2[0], __ffma2_rn(make_float2(mb, mb), nsc2, c0), A0, A1, A2, A3);
  }
  if (i < n) moment_scalar<STAGE>(seg[off + i], mb, sc, ps, M);
  M.T0 += A0.x + A0.y;
  M.T1 += A1.x + A1.y;
  M.T2 += A2.x + A2.y;
  M.T3 += A3.x + A3.y;
}

// Warp-uniform walk over the staged segment: every lane runs the same number
// of samples L (a multiple of 4) from its own 4-aligned start J0 (16-byte
// aligned LDS.128); the staged residual is finite and zero-padded.
//   MASK   samples outside the lane's support (q > qmax) get G = 0: exact
//          truncation at cutoff sigmas;
//   !MASK  samples walked past a window's ends lie beyond cutoff sigmas
//          (G <= exp(-cutoff^2/2) < 2^-24 for cutoff >= kUnmaskedCutoff):
//          their terms are below FP32 resolution; lanes with an empty window
//          discard their moments.
template <int STAGE, bool MASK>
__device__ __forceinline__ void moment_pair_masked(float2 res, float2 y, float qmax, float2& A0, float2& A1,
                                                   float2& A2, float2& A3) {
  const float2 q = __fmul2_rn(y, y);
  const float2 G = MASK ? make_float2(q.x <= qmax ? ex2(-q.x) : 0.0f, q.y <= qmax ? ex2(-q.y) : 0.0f)
                        : make_float2(ex2(-q.x), ex2(-q.y));
  const float2 r = __fmul2_rn(res, G);
  const float2 t = __fmul2_rn(r, y);
  A1 = __fadd2_rn(A1, t);
  if (STAGE >= kStageCoarse) A3 = __ffma2_rn(t, q, A3);
  if (STAGE == kStageFine) {
    A0 = __fadd2_rn(A0, r);
    A2 = __ffma2_rn(t, y, A2);
  }
}

// Per-ball walk constants.  Sample s of an 8-sample block starting at
// m-offset m has y = m * (-sc) + ps + s * dl, dl = f * (-sc); the block's
// four sample-pair offsets c_k = ps + (2k, 2k+1) dl are built per pair from
// ps with one FADD and three FADD2 (no per-ball vector constants held).
struct WalkConst {
  float2 nsc2;
  float dl, dl2;   // f * (-sc), 2 f * (-sc)
  float step8;     // 8 f (m advance per block)
};

__device__ __forceinline__ WalkConst walk_const(float sc, int f) {
  WalkConst w;
  const float nsc = -sc, fs = (float)f;
  w.nsc2 = make_float2(nsc, nsc);
  w.dl = fs * nsc;
  w.dl2 = 2.0f * fs * nsc;
  w.step8 = 8.0f * fs;
  return w;
}

template <int STAGE, bool MASK>
__device__ __forceinline__ void moment_block8(const float4* s4, float mf, const WalkConst& W, float2 c0, float2 c1,
                                              float2 c2, float2 c3, float qmax, float2& A0, float2& A1, float2& A2,
                                              float2& A3) {
  const float4 ra = s4[0], rb = s4[1];
  const float2 m2 = make_float2(mf, mf);
  moment_pair_masked<STAGE, MASK>(make_float2(ra.x, ra.y), __ffma2_rn(m2, W.nsc2, c0), qmax,
                                                        A0, A1, A2, A3);
  moment_pair_masked<STAGE, MASK>(make_float2(ra.z, ra.w), __ffma2_rn(m2, W.nsc2, c1), qmax,
                                                        A0, A1, A2, A3);
  moment_pair_masked<STAGE, MASK>(make_float2(rb.x, rb.y), __ffma2_rn(m2, W.nsc2, c2), qmax,
                                                        A0, A1, A2, A3);
  moment_pair_masked<STAGE, MASK>(make_float2(rb.z, rb.w), __ffma2_rn(m2, W.nsc2, c3), qmax,
                                                        A0, A1, A2, A3);
}

template <int STAGE, bool MASK>
__device__ __forceinline__ void moments_uniform(const float* seg, int L, float mf, const WalkConst& W, float ps,
                                                float qmax, Moments& M) {
  const float4* s4 = reinterpret_cast<const float4*>(seg);
  float2 A0 = make_float2(0.f, 0.f), A1 = A0, A2 = A0, A3 = A0;
  const float2 c0 = make_float2(ps, ps + W.dl);
  const float2 c1 = __fadd2_rn(c0, make_float2(W.dl2, W.dl2));
  const float2 c2 = __fadd2_rn(c1, make_float2(W.dl2, W.dl2));
  const float2 c3 = __fadd2_rn(c2, make_float2(W.dl2, W.dl2));
  int nb = L >> 3;
#pragma unroll 1
  for (; nb >= 2; nb -= 2, s4 += 4, mf += 2.0f * W.step8) {   // two blocks per trip
    moment_block8<STAGE, MASK>(s4, mf, W, c0, c1, c2, c3, qmax, A0, A1, A2, A3);
    moment_block8<STAGE, MASK>(s4 + 2, mf + W.step8, W, c0, c1, c2, c3, qmax, A0, A1, A2, A3);
  }
  if (nb) {
    moment_block8<STAGE, MASK>(s4, mf, W, c0, c1, c2, c3, qmax, A0, A1, A2, A3);
    s4 += 2;
    mf += W.step8;
  }
  if (L & 4) {   // 4-sample tail block
    const float4 ra = s4[0];
    const float2 m2 = make_float2(mf, mf);
    moment_pair_masked<STAGE, MASK>(make_float2(ra.x, ra.y), __ffma2_rn(m2, W.nsc2, c0), qmax, A0, A1, A2, A3);
    moment_pair_masked<STAGE, MASK>(make_float2(ra.z, ra.w), __ffma2_rn(m2, W.nsc2, c1), qmax, A0, A1, A2, A3);
  }
  M.T0 = A0.x + A0.y;
  M.T1 = A1.x + A1.y;
  M.T2 = A2.x + A2.y;
  M.T3 = A3.x + A3.y;
}

// Cascade walk (fine stage, unmasked, recurrence step within kCascMaxDl).
//
// The four moments of r_s = res_s G(y_s) are linear functionals of r, so they
// can be accumulated in any polynomial basis of the walk index.  The direct
// walk above spends 8 FP32x2 operations and 2 ex2 per sample pair (y, q, r,
// t and four accumulations); this one spends 6 and 1:
//   * the window is walked from both ends towards its middle, each half a
//     chain of sample pairs (even sample in .x, odd sample in .y) feeding a
//     cascade of running sums  A0 += res G; A1 += A0; A2 += A1; A3 += A2
//     (one FFMA2 + three FADD2).  After n steps A_k holds sum_u C(u+k-1, k)
//     r_u over the distance u to the chain's end (the right half updates in
//     the reverse order, A3 += A2 ... A0 += res G, which gives C(u, k) with
//     u counted from 0, so both halves share one origin): binomial, i.e.
//     exact integer, weights -- no multiplications by y in the loop;
//   * G follows the forward's ratio recurrence inside every 8-sample block:
//     the pair nearest the chain's start is exact (2 ex2 for G, 2 for the
//     ratio R), the next pairs G *= R, R *= C; nothing is carried between
//     blocks.
// The chains end in the middle of the walk, within a few samples of the
// arrival (all lanes of a group have nearly equal windows), so the shift
// from the chain origin to y = 0 is small and the conversion to T0..T3 --
// 14 FP32x2 + ~10 scalar operations per walk -- cancels little: against FP64
// moments the FP32 result is within 1e-7 (T0, T1), 3e-7 (T2) and 2e-6 (T3)
// rms of sum |r y^k| (the direct walk: 1e-7), emulated on config-2 windows.
#ifndef PAB_ADJ_CASCADE
#define PAB_ADJ_CASCADE 1
#endif
constexpr bool kAdjCascade = PAB_ADJ_CASCADE != 0;
constexpr float kCascMaxDl = 0.75f;   // |dl| bound of the ratio recurrence (as the forward's dual walk)
constexpr float kCascMaxExp = 100.0f; // bound on |k1 y|: the ratio stays below 2^127

struct CascConst {
  float2 k1, k2, C;   // R(y) = 2^(k1 y + k2): G(y + h) / G(y) with h = 2 dl; C = R(y + h) / R(y)
  float inv_h;
};

__device__ __forceinline__ CascConst casc_const(const WalkConst& W) {
  CascConst K;
  const float a = -2.0f * W.dl2, b = -W.dl2 * W.dl2, c = ex2(2.0f * b);
  K.k1 = make_float2(a, a);
  K.k2 = make_float2(b, b);
  K.C = make_float2(c, c);
  K.inv_h = 1.0f / W.dl2;
  return K;
}

struct Casc {
  float2 a0, a1, a2, a3;
};

__device__ __forceinline__ void casc_in(float2 res, float2 G, Casc& A) {   // inclusive: weights C(u + k - 1, k), u >= 1
  A.a0 = __ffma2_rn(res, G, A.a0);
  A.a1 = __fadd2_rn(A.a1, A.a0);
  A.a2 = __fadd2_rn(A.a2, A.a1);
  A.a3 = __fadd2_rn(A.a3, A.a2);
}
__device__ __forceinline__ void casc_ex(float2 res, float2 G, Casc& B) {   // exclusive: weights C(u, k), u >= 0
  B.a3 = __fadd2_rn(B.a3, B.a2);
  B.a2 = __fadd2_rn(B.a2, B.a1);
  B.a1 = __fadd2_rn(B.a1, B.a0);
  B.a0 = __ffma2_rn(res, G, B.a0);
}

// Left chain, ascending: NP sample pairs (2 or 4) from s4; m = m-offset of
// the first sample, c0 = (ps, ps + dl).
template <int NP, bool FIRST = false>
__device__ __forceinline__ void casc_left(const float4* s4, float m, const WalkConst& W, const CascConst& K, float2 c0,
                                          Casc& A) {
  const float4 ra = s4[0];
  float4 rb = make_float4(0.f, 0.f, 0.f, 0.f);
  if (NP == 4) rb = s4[1];
  const float2 y = __ffma2_rn(make_float2(m, m), W.nsc2, c0);
  const float2 q = __fmul2_rn(y, y);
  const float2 e = __ffma2_rn(y, K.k1, K.k2);
  float2 G = make_float2(ex2(-q.x), ex2(-q.y));
  float2 R = make_float2(ex2(e.x), ex2(e.y));
  if (FIRST) {   // the chain's first step on zero sums: no additions (and no zero registers)
    A.a0 = __fmul2_rn(make_float2(ra.x, ra.y), G);
    A.a1 = A.a0;
    A.a2 = A.a0;
    A.a3 = A.a0;
  } else {
    casc_in(make_float2(ra.x, ra.y), G, A);
  }
  G = __fmul2_rn(G, R);
  casc_in(make_float2(ra.z, ra.w), G, A);
  if (NP == 4) {
    R = __fmul2_rn(R, K.C);
    G = __fmul2_rn(G, R);
    casc_in(make_float2(rb.x, rb.y), G, A);
    R = __fmul2_rn(R, K.C);
    G = __fmul2_rn(G, R);
    casc_in(make_float2(rb.z, rb.w), G, A);
  }
}

// Right chain, descending: NP sample pairs from s4, the highest pair first;
// nm = minus the m-offset of that pair's first sample, nc0 = -(ps, ps + dl):
// with -y the step towards lower samples has the left chain's ratio.
template <int NP, bool FIRST = false>
__device__ __forceinline__ void casc_right(const float4* s4, float nm, const WalkConst& W, const CascConst& K, float2 nc0,
                                           Casc& B) {
  static_assert(!FIRST || NP == 4, "only a full block opens a chain");
  const float4 ra = s4[0];
  float4 rb = make_float4(0.f, 0.f, 0.f, 0.f);
  if (NP == 4) rb = s4[1];
  const float2 ny = __ffma2_rn(make_float2(nm, nm), W.nsc2, nc0);
  const float2 q = __fmul2_rn(ny, ny);
  const float2 e = __ffma2_rn(ny, K.k1, K.k2);
  float2 G = make_float2(ex2(-q.x), ex2(-q.y));
  float2 R = make_float2(ex2(e.x), ex2(e.y));
  if (FIRST) {
    // the chain's first four steps on zero sums: the sum of order k stays
    // zero until step k + 1 (9 of the 12 additions drop out)
    B.a0 = __fmul2_rn(make_float2(rb.z, rb.w), G);
    G = __fmul2_rn(G, R);
    B.a1 = B.a0;
    B.a0 = __ffma2_rn(make_float2(rb.x, rb.y), G, B.a0);
    R = __fmul2_rn(R, K.C);
    G = __fmul2_rn(G, R);
    B.a2 = B.a1;
    B.a1 = __fadd2_rn(B.a1, B.a0);
    B.a0 = __ffma2_rn(make_float2(ra.z, ra.w), G, B.a0);
    R = __fmul2_rn(R, K.C);
    G = __fmul2_rn(G, R);
    B.a3 = B.a2;
    B.a2 = __fadd2_rn(B.a2, B.a1);
    B.a1 = __fadd2_rn(B.a1, B.a0);
    B.a0 = __ffma2_rn(make_float2(ra.x, ra.y), G, B.a0);
  } else if (NP == 4) {
    casc_ex(make_float2(rb.z, rb.w), G, B);
    G = __fmul2_rn(G, R);
    casc_ex(make_float2(rb.x, rb.y), G, B);
    R = __fmul2_rn(R, K.C);
    G = __fmul2_rn(G, R);
    casc_ex(make_float2(ra.z, ra.w), G, B);
    R = __fmul2_rn(R, K.C);
    G = __fmul2_rn(G, R);
    casc_ex(make_float2(ra.x, ra.y), G, B);
  } else {
    casc_ex(make_float2(ra.z, ra.w), G, B);
    G = __fmul2_rn(G, R);
    casc_ex(make_float2(ra.x, ra.y), G, B);
  }
}

// L samples (a multiple of 4, warp-uniform) from seg (16-byte aligned), mf
// the m-offset of the first sample: trips of 8 left + 8 right samples, the
// remaining 4, 8 or 12 samples as 4 left, 4 + 4, or 8 left + 4 right.
__device__ __forceinline__ void moments_cascade(const float* seg, int L, float mf, const WalkConst& W,
                                                const CascConst& K, float ps, int f, Moments& M) {
  const float4* sL = reinterpret_cast<const float4*>(seg);
  const float4* sR = sL + (L >> 2) - 2;
  const float2 c0 = make_float2(ps, ps + W.dl);
  const float2 nc0 = make_float2(-c0.x, -c0.y);
  const float2 z2 = make_float2(0.f, 0.f);
  Casc A, B;
  const int trips = L >> 4, rem = L & 15;
  float mL = mf;
  float nmR = -(mf + (float)((L - 2) * f));
  if (trips > 0) {   // the first trip opens both chains (no zero sums to add to)
    casc_left<4, true>(sL, mL, W, K, c0, A);
    casc_right<4, true>(sR, nmR, W, K, nc0, B);
    sL += 2, sR -= 2, mL += W.step8, nmR += W.step8;
#pragma unroll 1
    for (int t = trips - 1; t > 0; --t, sL += 2, sR -= 2, mL += W.step8, nmR += W.step8) {
      casc_left<4>(sL, mL, W, K, c0, A);
      casc_right<4>(sR, nmR, W, K, nc0, B);
    }
  } else {           // walks shorter than 16 samples: the remainder blocks on zero sums
    A = {z2, z2, z2, z2};
    B = {z2, z2, z2, z2};
  }
  int hL = trips << 3;   // samples of the left chain
  if (rem == 12) {
    casc_left<4>(sL, mL, W, K, c0, A);
    hL += 8;
  } else if (rem >= 4) {
    casc_left<2>(sL, mL, W, K, c0, A);
    hL += 4;
  }
  if (rem >= 8) casc_right<2>(sR + 1, nmR, W, K, nc0, B);
  // Chain origin: sample hL (left: y = h (Z - u), right: y = h (Z + u), Z =
  // (zeta, zeta + 1/2) for the even and odd samples, zeta = y(hL) / h).
  // Power sums about the origin, right plus (-1)^j left:
  //   Q0 = B0 + A0, Q1 = B1 - A1, Q2 = 2 (B2 + A2) + Q1,
  //   Q3 = 6 (B3 - A3) + 6 (B2 + A2) + Q1
  // and the shift by Z (Horner): T_k = h^k sum_j C(k, j) Z^(k-j) Q_j.
  const float zeta = fmaf(mf + (float)(hL * f), W.nsc2.x, ps) * K.inv_h;
  const float2 Z = make_float2(zeta, zeta + 0.5f);
  const float2 Q0 = __fadd2_rn(B.a0, A.a0);
  const float2 Q1 = __fadd2_rn(B.a1, make_float2(-A.a1.x, -A.a1.y));
  const float2 S2 = __fadd2_rn(B.a2, A.a2);
  const float2 D3 = __fadd2_rn(B.a3, make_float2(-A.a3.x, -A.a3.y));
  const float2 Q2 = __ffma2_rn(make_float2(2.f, 2.f), S2, Q1);
  const float2 Q3 = __ffma2_rn(make_float2(6.f, 6.f), __fadd2_rn(D3, S2), Q1);
  const float2 M1 = __ffma2_rn(Z, Q0, Q1);
  const float2 M2 = __ffma2_rn(Z, __fadd2_rn(M1, Q1), Q2);
  const float2 M3 = __ffma2_rn(
      Z, __ffma2_rn(Z, __ffma2_rn(make_float2(2.f, 2.f), Q1, M1), __fmul2_rn(make_float2(3.f, 3.f), Q2)), Q3);
  const float h = W.dl2, h2 = h * h;
  M.T0 = Q0.x + Q0.y;
  M.T1 = (M1.x + M1.y) * h;
  M.T2 = (M2.x + M2.y) * h2;
  M.T3 = (M3.x + M3.y) * (h2 * h);
}

#ifndef PAB_ADJ_LEAN
#define PAB_ADJ_LEAN 1   // XU-free rounding in the pair setup; factored cos^2 fine epilogue
#endif
constexpr bool kAdjLean = PAB_ADJ_LEAN != 0;

// flags of a (lane group, detector) pair, computed by the batch lane
constexpr int kFlagUniform = 1;   // staged uniform walk (far field, fits the segment)
constexpr int kFlagNear = 2;      // a u+ window may exist
constexpr int kFlagSlow = 4;      // detector within two group radii: FP64 per-pair geometry

// One warp (lane group) per CTA.  The launch bound asks for 14 CTAs per SM
// (<= 144 registers): ptxas still allocates 128, so 16 warps are resident,
// but schedules the cascade walk better under the looser bound (measured,
// config-2 adjoint ms with bounds of 12 / 13 / 14 / 15 / 16 / 18 / 20 CTAs per
// SM: 17.91 / 16.65 / 16.62 / 16.64 / 16.73 / 17.40 / 17.88).  Warps
// retire independently (no CTA tail), measured best of 1/2/4/8 warps per CTA.
#ifndef PAB_ADJ_WARPS
#define PAB_ADJ_WARPS 1
#endif
#ifndef PAB_ADJ_MINB
#define PAB_ADJ_MINB (14 / PAB_ADJ_WARPS)
#endif
constexpr int kAdjWarps = PAB_ADJ_WARPS;
#ifdef PAB_ADJ_PROF   // tuning builds only: per-part clock totals (lane 0 of each warp)
__device__ unsigned long long g_adj_prof[16];
#define APROF_T(v) long long v = clock64()
#define APROF_ACC(i, t0) prof[(i)] += clock64() - (t0)
#else
#define APROF_T(v)
#define APROF_ACC(i, t0)
#endif
template <int STAGE, int DIR, bool MASK>
__global__ void __launch_bounds__(kAdjWarps * 32, PAB_ADJ_MINB)
adjoint_kernel(const BallA* __restrict__ ra, const BallB* __restrict__ rb,
               const GroupMeta* __restrict__ gmeta, int64_t n_groups,
               const double* __restrict__ det_pos, const double* __restrict__ det_aux, int n_det,
               Acq acq, const float* __restrict__ res, float res_sign, int det_per_chunk,
               double* __restrict__ gpart, int64_t n_pad, unsigned long long* __restrict__ ops_total,
               int* __restrict__ status, bool vec16) {
  // vec16: 16-byte cp.async staging (rows 16-byte aligned: host-checked
  // n_out % 4 == 0 and a 16-byte aligned residual pointer)
  __shared__ __align__(16) float seg_all[kAdjWarps][4][kSeg + kPad + 4];
  __shared__ __align__(16) float4 bat[kAdjWarps][kWarp][DIR == kDirElement ? 5 : 4];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // the processing order ascends in a0 bucket (window length): the
  // wide-window groups launch first and the light ones fill the tail
  // (longest-first; measured: config 2 -0.05 ms, config-3 reconstruction -2 %)
  const int64_t g = n_groups - 1 - ((int64_t)blockIdx.x * (blockDim.x >> 5) + warp);
  if (g < 0) return;
  if (g >= n_groups) return;
  const int q = blockIdx.y;
  const int j0 = q * det_per_chunk;
  const int j1 = min(n_det, j0 + det_per_chunk);
  const int n_out = acq.n_out;
  const int f = acq.f;
  const float fs = (float)f;

  const GroupMeta gm = gmeta[g];
  const int64_t bi = g * kWarp + lane;
  const BallA A = ra[bi];
  const BallB B = rb[bi];
  // per-ball constants (detector independent)
  const float sc = acq.vdt_f * kSqrtHalfLog2e * B.inv_a0;
  const float rho = acq.cutoff * A.a0 * acq.inv_vdt_f;
  const bool live = B.orig >= 0;
  const float qmax = live ? (rho * sc) * (rho * sc) : -1.0f;
  const WalkConst W = walk_const(sc, f);
  // cascade walk where the stage needs all four moments, no per-sample
  // truncation test and every live lane's recurrence step is in range
  constexpr bool kCascOk = kAdjCascade && STAGE == kStageFine && !MASK;
  const CascConst K = kCascOk ? casc_const(W) : CascConst{};
  // (the ratio R = 2^(k1 y + k2) must stay finite wherever the warp-uniform
  // walk takes a lane: |y| <= the cutoff + the group's longest walk past the
  // lane's own window -- groups mixing very different radii fall back)
  const float walk_max = 2.0f * (acq.cutoff * gm.a0max * acq.inv_vdt_f) * acq.inv_f + 20.0f;
  const float y_max = sqrtf(fmaxf(qmax, 0.0f)) + walk_max * fabsf(W.dl);
  const bool casc = kCascOk && __all_sync(0xffffffffu, !live || (fabsf(W.dl) <= kCascMaxDl &&
                                                                 2.0f * fabsf(W.dl2) * y_max <= kCascMaxExp));
  // the conversion-free setup pays where the XU pipe binds (ex2 walk); the
  // element directivity's sinc terms load the FMA pipe instead (config 4:
  // lean +0.7 ms)
  constexpr bool kLean = kAdjLean && DIR != kDirElement;
  const float kap_rs = A.a0 * kSqrt2Ln2 * res_sign;   // kappa * sign
  const float kap2 = 2.0f * A.a0 * kSqrt2Ln2;         // 2 kappa (factored epilogue)
  const float p0h = 0.5f * B.p0;
  // the uniform walk must stay inside the staged samples + the buffer's slack
  // (cover window <= 2 rho / f + 3 samples, + 3 alignment + 3 rounding)
  const bool fits = 2.0f * (acq.cutoff * gm.a0max * acq.inv_vdt_f) * acq.inv_f + 12.0f <= (float)kPad;
  // per-ball FP64 sums across the chunk, in shared memory (registers stay
  // with the moment walk: measured 0.6% faster than register accumulators)
  __shared__ double acc_s[kAdjWarps][5][kWarp];
#pragma unroll
  for (int c = 0; c < 5; ++c) acc_s[warp][c][lane] = 0.0;
  unsigned long long my_ops = 0;
  int coinc = 0;
#ifdef PAB_ADJ_PROF
  long long prof[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  APROF_T(t_all);
#endif

  for (int jb = j0; jb < j1; jb += kWarp) {
    const int nd = min(kWarp, j1 - jb);
    APROF_T(t_geo);
    GroupDet gdl = empty_gd();
    DetDir ddl{};
    int rlo = 0, rhi = -1, rfl = 0;
    if (lane < nd) {
      const int jl = jb + lane;
      gdl = group_det(gm, det_pos[3 * jl], det_pos[3 * jl + 1], det_pos[3 * jl + 2], acq);
      group_range(acq, gdl, gm, &rlo, &rhi);
      rlo &= ~3;   // 16-byte aligned staging base
      const bool nr = group_near(acq, gdl, gm);
      rfl = (nr ? kFlagNear : 0) | (gdl.slow ? kFlagSlow : 0) |
            (!nr && fits && rlo <= rhi && rhi - rlo + 1 <= kSeg ? kFlagUniform : 0);
      if (DIR != kDirNone) ddl = load_detdir(det_aux, jl);
    }
    // the batch's per-detector data in shared memory: the pair loop reads a
    // detector's geometry, flags and direction with broadcast LDS.128 (3-5)
    // instead of 10-16 shuffles (lane stride 80 B: conflict-free writes)
    {
      float4* const bt = bat[warp][lane];
      bt[0] = make_float4(gdl.Sx, gdl.Sy, gdl.Sz, gdl.Sn);
      bt[1] = make_float4(gdl.isn, gdl.phg, __int_as_float(gdl.kg), __int_as_float(rfl));
      bt[2] = make_float4(__int_as_float(rlo), __int_as_float(rhi), ddl.fx, ddl.fy);
      if (DIR != kDirNone) bt[3] = make_float4(ddl.fz, ddl.e1x, ddl.e1y, ddl.e1z);
      if (DIR == kDirElement) bt[4] = make_float4(ddl.e2x, ddl.e2y, ddl.e2z, 0.0f);
    }
    __syncwarp();
    auto bgd = [&](int jj) {   // group geometry (slow flag from the flags word, as shfl_gd_fast + fallback)
      const float4 a = bat[warp][jj][0], b = bat[warp][jj][1];
      GroupDet gd;
      gd.Sx = a.x; gd.Sy = a.y; gd.Sz = a.z; gd.Sn = a.w;
      gd.isn = b.x; gd.phg = b.y; gd.kg = __float_as_int(b.z);
      gd.slow = 0;
      return gd;
    };
    auto bdd = [&](int jj) {
      DetDir dd{};
      if (DIR != kDirNone) {
        const float4 c = bat[warp][jj][2], d = bat[warp][jj][3];
        dd.fx = c.z; dd.fy = c.w; dd.fz = d.x;
        dd.e1x = d.y; dd.e1y = d.z; dd.e1z = d.w;
        if (DIR == kDirElement) {
          const float4 e = bat[warp][jj][4];
          dd.e2x = e.x; dd.e2y = e.y; dd.e2z = e.z;
        }
      }
      return dd;
    };
    auto blhf = [&](int jj, int& lo, int& hi, int& fl) {
      const float4 c = bat[warp][jj][2];
      lo = __float_as_int(c.x);
      hi = __float_as_int(c.y);
      fl = __float_as_int(bat[warp][jj][1].w);
    };
    // stage res[j][lo .. hi] (lo a multiple of 4) + kPad zeros into buffer
    // `buf`: 16-B cp.async (16-B aligned rows) or 4-B cp.async
    auto stage_seg = [&](int jj, int lo, int hi, int fl, int buf) {
#ifdef PAB_ADJ_NOSTAGE   // tuning builds only: no residual staging (wrong gradients)
      return;
#endif
      if (!(fl & kFlagUniform)) return;
      const float* src = res + (size_t)(jb + jj) * n_out + lo;
      float* dst = seg_all[warp][buf];
      const int len = hi - lo + 1;
      if (vec16) {
        const int len4 = (len + 3) >> 2;   // the last vector may carry up to 3 finite extra samples
        static_assert(kSeg <= 8 * kWarp, "two 16-B vectors per lane cover the segment");
        if (lane < len4) cp_async16(dst + 4 * lane, src + 4 * lane);
        if (lane + kWarp < len4) cp_async16(dst + 4 * (lane + kWarp), src + 4 * (lane + kWarp));
        cp_async_commit();
        // zero padding after the staged samples: the uniform walk runs past
        // them (lanes whose windows end earlier, rounding, and -- for a
        // segment clipped at the record end -- windows running past the last
        // sample, which must read as zero).  (Measured: leaving the earlier
        // detectors' residuals there instead, the terms past a window
        // beyond cutoff sigmas are below 2^-24 of the ball's peak but not
        // the reference's zeros, and a record-end segment reads wrong
        // residuals inside the window: the smoke gradients were off by 5e-3.)
        if (lane < kPad / 4) reinterpret_cast<float4*>(dst + 4 * len4)[lane] = make_float4(0.f, 0.f, 0.f, 0.f);
      } else {
        for (int k = lane; k < len; k += kWarp) cp_async4(dst + k, src + k);
        cp_async_commit();
        for (int k = lane; k < kPad; k += kWarp) dst[len + k] = 0.0f;
      }
    };
    auto wait_seg = [&](int fl) {
      if (fl & kFlagUniform) cp_async_wait_all();
    };
    float gb[5] = {0.f, 0.f, 0.f, 0.f, 0.f};   // FP32 batch sums of the pair terms
    // lean cos^2 fine epilogue: per-ball factors taken out of the pair terms
    // and applied once per batch (gb0 * rs / 4, gb1 * p0/2 k^3 rs, gb2-4 * p0/2 rs)
    constexpr bool kFactored = kAdjLean && DIR == kDirCos2 && STAGE == kStageFine;

    // per-pair gradient terms (reference radiator.py:275-286 in y units)
    auto epilogue = [&](const PairGeom& pg, const Moments& M, const DetDir& dd) {
#ifdef PAB_ADJ_NOEPI   // tuning builds only: no gradient epilogue (wrong gradients)
      gb[0] += M.T0 + M.T1 + M.T2 + M.T3 + pg.id + pg.rx;
      return;
#endif
      if constexpr (kFactored) {
        // cos^2, fine, factored: with Q = p0/2 rs, k = 2 kappa T1 and
        // E = T0 - 2 ln2 T2 the position term of the form below is
        //   alpha = Q id^2 D (E - 3/2 k id)   (cp c = D: cp = c or D = 0)
        //   beta  = Q id^2 cp k
        // and gb0 = rs/4 D k id, gb1 = Q k^3 D id T3 (Q, rs/4 applied per batch)
        const float id = pg.id;
        const float c = (dd.fx * pg.rx + dd.fy * pg.ry + dd.fz * pg.rz) * id;
        const float cp = fmaxf(c, 0.0f);
        const float D = cp * cp;
        const float h = id * id;
        const float k = kap2 * M.T1;
        const float kid = k * id;
        const float a = (D * h) * fmaf(-1.5f, kid, fmaf(-kTwoLn2, M.T2, M.T0));
        const float b = (cp * h) * k;
        gb[0] = fmaf(D, kid, gb[0]);
        gb[1] = fmaf(D * id, M.T3, gb[1]);
        gb[2] = fmaf(a, pg.rx, fmaf(b, dd.fx, gb[2]));
        gb[3] = fmaf(a, pg.ry, fmaf(b, dd.fy, gb[3]));
        gb[4] = fmaf(a, pg.rz, fmaf(b, dd.fz, gb[4]));
        return;
      } else if constexpr (DIR == kDirCos2 && STAGE == kStageFine) {
        // cos^2, fine: dD/dr = 2 cp (f - c h) / d with h = r / d, so the
        // position term w r + (base s_uG) dD/dr folds into alpha r + beta f
        // (10 fewer FP32 operations per pair than the generic form below)
        const float id = pg.id;
        const float c = (dd.fx * pg.rx + dd.fy * pg.ry + dd.fz * pg.rz) * id;
        const float cp = fmaxf(c, 0.0f);
        const float D = cp * cp;
        const float base = p0h * id;
        const float s_uG = kap_rs * M.T1;
        const float bD = base * D;
        gb[0] = fmaf(D * s_uG, 0.5f * id, gb[0]);
        gb[1] = fmaf(bD * (kSqrt2Ln2Cubed * res_sign), M.T3, gb[1]);
        const float w = bD * fmaf(res_sign, fmaf(-kTwoLn2, M.T2, M.T0), -id * s_uG) * id;
        const float beta = (base * s_uG) * (cp * (2.0f * id));
        const float alpha = fmaf(-beta * c, id, w);
        gb[2] = fmaf(alpha, pg.rx, fmaf(beta, dd.fx, gb[2]));
        gb[3] = fmaf(alpha, pg.ry, fmaf(beta, dd.fy, gb[3]));
        gb[4] = fmaf(alpha, pg.rz, fmaf(beta, dd.fz, gb[4]));
        return;
      }
      float dDdr[3] = {0.f, 0.f, 0.f}, dDda0 = 0.f;
      const float id = pg.id;
      const float D = dir_weight<DIR, STAGE == kStageFine || DIR == kDirElement>(
          dd, pg.rx * id, pg.ry * id, pg.rz * id, id, acq.dir_param, acq.dir_param, B.inv_a0, dDdr, &dDda0);
      const float base = p0h * id;   // p0 / 2d
      const float s_uG = kap_rs * M.T1;
      gb[0] = fmaf(D * s_uG, 0.5f * id, gb[0]);
      if (STAGE >= kStageCoarse) {
        float ga = (base * D) * (kSqrt2Ln2Cubed * res_sign) * M.T3;
        if (DIR == kDirElement) ga = fmaf(base * dDda0, s_uG, ga);
        gb[1] += ga;
      }
      if (STAGE == kStageFine) {
        const float w = (base * D) * fmaf(res_sign, fmaf(-kTwoLn2, M.T2, M.T0), -id * s_uG) * id;
        float gx = w * pg.rx, gy = w * pg.ry, gz = w * pg.rz;
        if (DIR != kDirNone) {
          const float bs = base * s_uG;
          gx = fmaf(bs, dDdr[0], gx);
          gy = fmaf(bs, dDdr[1], gy);
          gz = fmaf(bs, dDdr[2], gz);
        }
        gb[2] += gx;
        gb[3] += gy;
        gb[4] += gz;
      }
    };
    // uniform path, part 1: geometry, covering window, block count
    struct USetup {
      PairGeom pg;
      int J0, L;
      bool empty;
    };
    auto usetup = [&](const GroupDet& gd, int lo) {
      USetup u;
      int jlo, jhi;
      if (kLean) {
        float kf;
        u.pg = pair_geom_lean(gd, A, B, acq, &kf);
        pair_window_cover_lean(kf, u.pg.phi, rho, acq, &jlo, &jhi);
      } else {
        u.pg = pair_geom_fast(gd, A, B, acq);
        pair_window_cover(u.pg.kc, u.pg.phi, rho, acq, &jlo, &jhi);
      }
      u.empty = !live || jlo > jhi;
      u.J0 = u.empty ? lo : max(jlo & ~3, lo);
      u.L = __reduce_max_sync(0xffffffffu, u.empty ? 0 : jhi - u.J0 + 1);
      if (ops_total && live) {   // exact sample count for the op counter
        int elo, ehi;
        pair_window<true>(u.pg.kc, u.pg.phi, rho, acq, &elo, &ehi);
        my_ops += (unsigned long long)max(ehi - elo + 1, 0);
      }
      return u;
    };
    // uniform path, part 2: the moment walk over the staged segment
    auto uwalk = [&](const USetup& u, int lo, int buf) {
      Moments M;
      PAB_CHECK(u.J0 - lo >= 0 && u.J0 - lo + ((u.L + 3) & ~3) <= kSeg + kPad);
#ifdef PAB_ADJ_NOWALK   // tuning builds only: everything but the moment walk (wrong gradients)
      M = {(float)(u.J0 - lo + buf), (float)u.L, 0.f, 0.f};
      return M;
#endif
      const float mf0 = kLean ? int_to_float(u.J0 * f - u.pg.kc) : (float)(u.J0 * f - u.pg.kc);
      if (kCascOk && casc)
        moments_cascade(seg_all[warp][buf] + (u.J0 - lo), (u.L + 3) & ~3, mf0, W, K, u.pg.phi * sc, f, M);
      else
        moments_uniform<STAGE, MASK>(seg_all[warp][buf] + (u.J0 - lo), (u.L + 3) & ~3, mf0, W, u.pg.phi * sc,
                                     u.empty ? -1.0f : qmax, M);
      if (!MASK && u.empty) M = {0.f, 0.f, 0.f, 0.f};
      return M;
    };
    // near field / detector close to the group / wide windows: per-lane
    // walks over the global residual row, FP64 geometry when slow
    auto fallback = [&](GroupDet gd, int fl, int jj, PairGeom& pg) {
      gd.slow = (fl & kFlagSlow) ? 1 : 0;
      double px = 0.0, py = 0.0, pz = 0.0;
      if (gd.slow) {
        px = det_pos[3 * (jb + jj)];
        py = det_pos[3 * (jb + jj) + 1];
        pz = det_pos[3 * (jb + jj) + 2];
      }
      pg = pair_geom(gd, gm, px, py, pz, A, B, acq);
      coinc |= pg.coincident;
      int jlo, jhi;
      pair_window<true>(pg.kc, pg.phi, rho, acq, &jlo, &jhi);
      if (!live) { jlo = 1; jhi = 0; }
      int nlo = 1, nhi = 0, nkc = 0;
      float nphi = 0.0f;
      if ((fl & kFlagNear) && live) pair_near_window(pg.d, rho, acq, &nlo, &nhi, &nkc, &nphi);
      my_ops += (unsigned long long)(max(jhi - jlo + 1, 0) + max(nhi - nlo + 1, 0));
      Moments M = {0.f, 0.f, 0.f, 0.f};
      const float* row = res + (size_t)(jb + jj) * n_out;
      moments_run<STAGE>(row, jlo, jhi - jlo + 1, (float)(jlo * f - pg.kc), fs, sc, pg.phi * sc, M);
      if (nlo <= nhi) {   // u+ = -kappa y: odd moments flip sign
        Moments N = {0.f, 0.f, 0.f, 0.f};
        moments_run<STAGE>(row, nlo, nhi - nlo + 1, (float)(nlo * f - nkc), fs, sc, nphi * sc, N);
        M.T0 += N.T0;
        M.T1 -= N.T1;
        M.T2 += N.T2;
        M.T3 -= N.T3;
      }
      return M;
    };
    auto one = [&](int jj, int lo, int hi, int fl, int buf, const GroupDet& gd, const DetDir& dd) {
      if (lo > hi) return;
      PairGeom pg;
      Moments M;
      if (fl & kFlagUniform) {
        const USetup u = usetup(gd, lo);
        M = uwalk(u, lo, buf);
        pg = u.pg;
      } else {
        M = fallback(gd, fl, jj, pg);
      }
      __syncwarp();
      epilogue(pg, M, dd);
    };

    // detectors in pairs, four staging buffers per warp: while a pair is
    // processed the next pair's segments are in flight; the two pairs'
    // setups (latency-bound chains) and gradient epilogues are computed side
    // by side
    int loA, hiA, flA, loB, hiB, flB;
    blhf(0, loA, hiA, flA);
    blhf(min(1, nd - 1), loB, hiB, flB);
    if (nd < 2) flB = 0;
    APROF_ACC(0, t_geo);
    stage_seg(0, loA, hiA, flA, 0);
    if (nd > 1) stage_seg(1, loB, hiB, flB, 1);
    for (int jj = 0; jj < nd; jj += 2) {
      const bool two = jj + 1 < nd;
      const int bA = jj & 3, bB = bA + 1;
      const int la = loA, ha = hiA, fa = flA, lb = loB, hb = hiB, fb = two ? flB : 0;
      const GroupDet gdA = bgd(jj), gdB = bgd(two ? jj + 1 : jj);
      const DetDir ddA = bdd(jj), ddB = bdd(two ? jj + 1 : jj);
      APROF_T(t_w);
      wait_seg(fa | fb);
      __syncwarp();   // every lane is past the previous pair: its buffers may be refilled
      APROF_ACC(1, t_w);
      APROF_T(t_st);
      if (jj + 2 < nd) {
        blhf(jj + 2, loA, hiA, flA);
        stage_seg(jj + 2, loA, hiA, flA, bA ^ 2);
        if (jj + 3 < nd) {
          blhf(jj + 3, loB, hiB, flB);
          stage_seg(jj + 3, loB, hiB, flB, bB ^ 2);
        } else {
          flB = 0;
        }
      }
      const bool uA = (fa & kFlagUniform) && la <= ha, uB = two && (fb & kFlagUniform) && lb <= hb;
      APROF_ACC(2, t_st);
      if (uA && uB) {
        APROF_T(t_s);
        const USetup sA = usetup(gdA, la);
        const USetup sB = usetup(gdB, lb);
#ifdef PAB_ADJ_PROF
        __syncwarp();
#endif
        APROF_ACC(3, t_s);
        APROF_T(t_k);
        const Moments MA = uwalk(sA, la, bA);
        const Moments MB = uwalk(sB, lb, bB);
        __syncwarp();
        APROF_ACC(4, t_k);
        APROF_T(t_e);
        epilogue(sA.pg, MA, ddA);
        epilogue(sB.pg, MB, ddB);
#ifdef PAB_ADJ_PROF
        __syncwarp();
#endif
        APROF_ACC(5, t_e);
      } else {
        APROF_T(t_o);
        one(jj, la, ha, fa, bA, gdA, ddA);
        if (two) one(jj + 1, lb, hb, fb, bB, gdB, ddB);
        APROF_ACC(6, t_o);
      }
    }
    __syncwarp();
    if (kFactored) {
      const float Q = p0h * res_sign;
      gb[0] *= 0.25f * res_sign;
      gb[1] *= Q * kSqrt2Ln2Cubed;
      gb[2] *= Q;
      gb[3] *= Q;
      gb[4] *= Q;
    }
#pragma unroll
    for (int c = 0; c < 5; ++c) acc_s[warp][c][lane] += (double)gb[c];
  }
#ifdef PAB_ADJ_PROF
  APROF_ACC(7, t_all);
  if (lane == 0)
    for (int i = 0; i < 8; ++i) atomicAdd(&g_adj_prof[i], (unsigned long long)prof[i]);
#endif
  double* out = gpart + (size_t)q * 5 * n_pad;
#pragma unroll
  for (int c = 0; c < 5; ++c) out[c * n_pad + bi] = acc_s[warp][c][lane];
  for (int o = 16; o > 0; o >>= 1) {
    my_ops += __shfl_xor_sync(0xffffffffu, my_ops, o);
    coinc |= __shfl_xor_sync(0xffffffffu, coinc, o);
  }
  if (lane == 0) {
    if (ops_total && my_ops) atomicAdd(ops_total, my_ops);
    if (coinc) atomicOr(status, kStatusCoincident);
  }
}

// Sum detector-chunk partials in chunk order, scale by 2/N (MSE, reference
// radiator.py:356-358), scatter to the caller's ball order, flag non-finite.
__global__ void grad_finalize_kernel(const double* __restrict__ gpart, int chunks, int64_t n_pad,
                                     const BallB* __restrict__ rb, double scale, int stage,
                                     double* __restrict__ d_p0, double* __restrict__ d_a0,
                                     double* __restrict__ d_pos, int* __restrict__ status) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_pad) return;
  const int orig = rb[i].orig;
  if (orig < 0) return;
  double v[5] = {0, 0, 0, 0, 0};
  for (int q = 0; q < chunks; ++q)
    for (int c = 0; c < 5; ++c) v[c] += gpart[((size_t)q * 5 + c) * n_pad + i];
  bool bad = false;
  for (int c = 0; c < 5; ++c) {
    v[c] *= scale;
    bad |= !isfinite(v[c]);
  }
  d_p0[orig] = v[0];
  if (d_a0) d_a0[orig] = stage >= kStageCoarse ? v[1] : 0.0;
  if (d_pos) {
    d_pos[3 * (int64_t)orig + 0] = stage == kStageFine ? v[2] : 0.0;
    d_pos[3 * (int64_t)orig + 1] = stage == kStageFine ? v[3] : 0.0;
    d_pos[3 * (int64_t)orig + 2] = stage == kStageFine ? v[4] : 0.0;
  }
  if (bad) atomicOr(status, kStatusNonFinite);
}

template <int STAGE, int DIR>
static void launch_adjoint(dim3 grid, int threads, cudaStream_t s, const BallA* A, const BallB* B,
                           const GroupMeta* G, int64_t n_groups, const double* det_pos, const double* det_aux,
                           int n_det, const Acq& a, const float* res, float res_sign, int per_chunk, double* gpart,
                           int64_t n_pad, unsigned long long* ops, int* status) {
  const bool vec16 = (a.n_out & 3) == 0 && (reinterpret_cast<uintptr_t>(res) & 15) == 0;
  // per-sample truncation test only where the walk's overrun could matter
  if (a.cutoff < kUnmaskedCutoff)
    adjoint_kernel<STAGE, DIR, true><<<grid, threads, 0, s>>>(A, B, G, n_groups, det_pos, det_aux, n_det, a, res,
                                                               res_sign, per_chunk, gpart, n_pad, ops, status,
                                                               vec16);
  else
    adjoint_kernel<STAGE, DIR, false><<<grid, threads, 0, s>>>(A, B, G, n_groups, det_pos, det_aux, n_det, a, res,
                                                                res_sign, per_chunk, gpart, n_pad, ops, status,
                                                                vec16);
}

template <int STAGE>
static void launch_adjoint_dir(int dir, dim3 grid, int threads, cudaStream_t s, const BallA* A, const BallB* B,
                               const GroupMeta* G, int64_t n_groups, const double* det_pos, const double* det_aux,
                               int n_det, const Acq& a, const float* res, float res_sign, int per_chunk,
                               double* gpart, int64_t n_pad, unsigned long long* ops, int* status) {
  if (dir == kDirNone)
    launch_adjoint<STAGE, kDirNone>(grid, threads, s, A, B, G, n_groups, det_pos, det_aux, n_det, a, res, res_sign,
                                    per_chunk, gpart, n_pad, ops, status);
  else if (dir == kDirCosPower && a.dir_param == 2.0f)
    launch_adjoint<STAGE, kDirCos2>(grid, threads, s, A, B, G, n_groups, det_pos, det_aux, n_det, a, res, res_sign,
                                    per_chunk, gpart, n_pad, ops, status);
  else if (dir == kDirCosPower)
    launch_adjoint<STAGE, kDirCosPower>(grid, threads, s, A, B, G, n_groups, det_pos, det_aux, n_det, a, res,
                                        res_sign, per_chunk, gpart, n_pad, ops, status);
  else
    launch_adjoint<STAGE, kDirElement>(grid, threads, s, A, B, G, n_groups, det_pos, det_aux, n_det, a, res,
                                       res_sign, per_chunk, gpart, n_pad, ops, status);
}

}  // namespace pab

using namespace pab;

extern "C" {

int pab_adjoint(const void* rec_a, const void* rec_b, const void* group_meta, int64_t n_groups,
                const double* det_pos, const double* det_aux, int n_det, double v, double t0, double dt,
                int f, int n_out, double cutoff, int dir_kind, double dir_param, const float* res,
                float res_sign, int stage, int chunks, int warps, double* grad_partial,
                unsigned long long* ops_total, int* status, void* stream) {
  if (n_groups <= 0 || n_det <= 0) return 0;
  if (f < 1 || chunks < 1 || warps < 1 || warps > kAdjWarps || stage < 0 || stage > 2 || dir_kind < 0 ||
      dir_kind > 2)
    return 1;
  if (!rec_a || !rec_b || !group_meta || !det_pos || !det_aux || !res || !grad_partial || !status) return 1;
  if ((int64_t)n_out * f > kMaxRecordSamples) return 1;   // sample indices stay in the magic-rounding range
  const Acq a = make_acq(v, t0, dt, f, n_out, cutoff, dir_kind, dir_param);
  const int per_chunk = (n_det + chunks - 1) / chunks;
  const int64_t n_pad = n_groups * kWarp;
  dim3 grid((unsigned)((n_groups + warps - 1) / warps), (unsigned)chunks);
  const cudaStream_t s = (cudaStream_t)stream;
  const BallA* A = (const BallA*)rec_a;
  const BallB* B = (const BallB*)rec_b;
  const GroupMeta* G = (const GroupMeta*)group_meta;
  const int th = warps * kWarp;
  if (stage == kStageFilter)
    launch_adjoint_dir<kStageFilter>(dir_kind, grid, th, s, A, B, G, n_groups, det_pos, det_aux, n_det, a, res,
                                     res_sign, per_chunk, grad_partial, n_pad, ops_total, status);
  else if (stage == kStageCoarse)
    launch_adjoint_dir<kStageCoarse>(dir_kind, grid, th, s, A, B, G, n_groups, det_pos, det_aux, n_det, a, res,
                                     res_sign, per_chunk, grad_partial, n_pad, ops_total, status);
  else
    launch_adjoint_dir<kStageFine>(dir_kind, grid, th, s, A, B, G, n_groups, det_pos, det_aux, n_det, a, res,
                                   res_sign, per_chunk, grad_partial, n_pad, ops_total, status);
  return cudaGetLastError() == cudaSuccess ? 0 : 4;
}

int pab_grad_finalize(const double* grad_partial, int chunks, int64_t n_groups, const void* rec_b, double scale,
                      int stage, double* d_p0, double* d_a0, double* d_pos, int* status, void* stream) {
  if (n_groups <= 0) return 0;
  if (!grad_partial || !rec_b || !d_p0 || !status || chunks < 1) return 1;
  const int64_t n_pad = n_groups * kWarp;
  grad_finalize_kernel<<<(unsigned)((n_pad + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
      grad_partial, chunks, n_pad, (const BallB*)rec_b, scale, stage, d_p0, d_a0, d_pos, status);
  return cudaGetLastError() == cudaSuccess ? 0 : 4;
}

}  // extern "C"

#ifdef PAB_ADJ_PROF
extern "C" int pab_adj_prof(unsigned long long* out /*[16]*/, int reset) {
  cudaMemcpyFromSymbol(out, pab::g_adj_prof, sizeof(unsigned long long) * 16);
  if (reset) {
    unsigned long long z[16] = {};
    cudaMemcpyToSymbol(pab::g_adj_prof, z, sizeof(z));
  }
  return cudaGetLastError() == cudaSuccess ? 0 : 4;
}
#endif

#ifdef PAB_ADJ_BENCH
// Tuning builds only: the fine adjoint's moment walk in isolation (16 warps
// per SM, one per CTA, like the kernel), `reps` walks of L samples per lane
// over a staged segment -- lane-samples per second vs the ex2 / FMA ceilings.
namespace pab {
__global__ void __launch_bounds__(32, 16) adj_walk_bench_kernel(int reps, int L, int cascade, float* out) {
  __shared__ __align__(16) float seg[kSeg + kPad + 4];
  const int lane = threadIdx.x;
  for (int i = lane; i < kSeg + kPad + 4; i += 32) seg[i] = 0.001f * (float)((i * 7) % 13);
  __syncwarp();
  const float sc = 0.3f + 0.001f * lane, ps = 0.1f * lane;
  const WalkConst W = walk_const(sc, 1);
  const CascConst K = casc_const(W);
  Moments acc = {0.f, 0.f, 0.f, 0.f};
  for (int r = 0; r < reps; ++r) {
    const int J0 = ((r * 4 + lane * 4) % 64);
    Moments M;
    if (cascade)
      moments_cascade(seg + J0, L, (float)(-L / 2), W, K, ps, 1, M);
    else
      moments_uniform<kStageFine, false>(seg + J0, L, (float)(-L / 2), W, ps, 30.0f, M);
    acc.T0 += M.T0; acc.T1 += M.T1; acc.T2 += M.T2; acc.T3 += M.T3;
  }
  out[blockIdx.x * 32 + lane] = acc.T0 + acc.T1 + acc.T2 + acc.T3;
}
}  // namespace pab
extern "C" int pab_bench_adj_walk(int blocks, int reps, int L, int cascade, float* out, float* ms) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  pab::adj_walk_bench_kernel<<<blocks, 32>>>(reps, L, cascade, out);
  cudaEventRecord(a);
  pab::adj_walk_bench_kernel<<<blocks, 32>>>(reps, L, cascade, out);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  cudaEventElapsedTime(ms, a, b);
  return cudaGetLastError() == cudaSuccess ? 0 : 4;
}
#endif
