// Forward model and residual/loss epilogue (K4).
//
// Replaces reference radiator.py:185-261 (slab evaluation + np.bincount
// scatter) and :263-264 (residual, loss part).
//
// Decomposition.  One CTA owns one detector row (all samples of the
// decimated grid; its partial row in global memory, L2-resident) and a
// partition of the lane groups (32
// balls of similar radius, spatially compact).  Groups are processed in
// chunks; per chunk the CTA
//   A  computes every group's sample range for this detector (FP64 geometry),
//   B  counting-sorts the groups by the 4-sample bin of their first sample
//      (histogram, scan, in-order match_any ranks: deterministic, stable),
//   C  gives each warp a contiguous slice of the sorted list.  A warp walks
//      its slice in time order; lane l evaluates ball l of each group over
//      its own arrival window and read-modify-writes its private column of a
//      circular per-warp tile [kTile rows x 32 lanes] (lane l -> bank l: no
//      conflicts, no atomics).  Rows the sweep has passed are reduced across
//      lanes (rotated, conflict-free) and added to the CTA row: each sample is
//      reduced once per warp instead of once per group,
//   D  merges the few rows where neighbouring warps' slices overlap, in warp
//      order.
// Every sample is therefore a fixed-order sum: results are bitwise
// reproducible run to run.  Partitions are summed in order by the epilogue.
#include <algorithm>
#include <climits>

#include "pab_common.cuh"

namespace pab {

constexpr int kBinShift = 3;           // 8 decimated samples per sort bin (bin starts 8-aligned)
#ifndef PAB_FWD_CHUNK
#define PAB_FWD_CHUNK 3072
#endif
#ifndef PAB_FWD_TILE
#define PAB_FWD_TILE 160
#endif
#ifndef PAB_FWD_MAXWARPS
#define PAB_FWD_MAXWARPS 4
#endif
constexpr int kChunk = PAB_FWD_CHUNK;  // lane groups per sort chunk
constexpr unsigned short kEmptyBin = 0xFFFF;
constexpr unsigned short kDualTail = 0xFFFE;   // second slot of a dual sort entry
constexpr int kTile = PAB_FWD_TILE;    // tile rows per warp (circular, slot = J % kTile, multiple of 8)
constexpr int kMaxWarps = PAB_FWD_MAXWARPS;
constexpr int kTileAlloc = kTile + 8;  // + one 8-row dump block per warp (wide-group kernel, benches)
constexpr int kDumpFloats = 8 * kWarp; // the sweep's walkers share one dump block
#ifndef PAB_FWD_RING
#define PAB_FWD_RING 2   // hand-off slots per walker (warp-specialised sweep)
#endif
constexpr int kRing = PAB_FWD_RING;

#ifndef PAB_FWD_BACKOFF_NS
#define PAB_FWD_BACKOFF_NS 100
#endif
// mbarrier helpers (warp-specialised sweep: producer/walker slot hand-off)
__device__ __forceinline__ void mbar_init(unsigned long long* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(b)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"((unsigned)__cvta_generic_to_shared(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* b, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}" ::"r"(
          (unsigned)__cvta_generic_to_shared(b)),
      "r"(parity)
      : "memory");
}

// Producer side: back off between polls so a waiting producer leaves the
// issue slots to the walker sharing its scheduler.
__device__ __forceinline__ void mbar_wait_backoff(unsigned long long* b, unsigned parity) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(b);
  unsigned ok;
  for (;;) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
        : "=r"(ok)
        : "r"(a), "r"(parity)
        : "memory");
    if (ok) break;
    __nanosleep(PAB_FWD_BACKOFF_NS);
  }
}

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// Tile layout: per warp, slot (circular row) s of lane l lives at float
// index tidx(s, l) = ((s / 4) * 32 + l) * 4 + s % 4, i.e. a lane owns four
// consecutive rows as one 16-byte vector and the 32 lanes' vectors of a row
// quad are adjacent.  A lane's 8-sample block is two LDS.128 + two STS.128,
// and because lane l always addresses bank quad l % 8, those accesses are
// conflict-free whatever row each lane is at.
__device__ __forceinline__ int tidx(int slot, int lane) { return (((slot >> 2) * kWarp + lane) << 2) | (slot & 3); }

// Window [lo, hi] of one pair into the circular tile (linear-pass path for
// wide groups: scalar, exact window).
__device__ __forceinline__ void rmw_window(float* tile, int lane, int lo, int hi, int m0, int f, float sc,
                                           float phi, float Ak) {
  if (lo > hi) return;
  const float ps = phi * sc;
  const float fs = (float)f;
  int s = lo % kTile;
  float mf = (float)(lo * f - m0);
  for (int J = lo; J <= hi; ++J) {
    const float y = fmaf(mf, -sc, ps);
    tile[tidx(s, lane)] += Ak * (y * ex2(-y * y));
    mf += fs;
    if (++s == kTile) s = 0;
  }
}

// Reduce rows [a, b) of the circular tile across lanes, zero them, and hand
// each row sum to `sink(r, v)`.  Lane l reduces row a + 32k + l, visiting the
// 32 columns in the order c(i, l) = ((i + l/4) % 8) + 8 (i / 8): for every i
// the 32 lanes then hit 32 distinct banks (bank = 4 (c % 8) + row % 4).
template <class Sink>
__device__ __forceinline__ void flush_rows(float* tile, int lane, int a, int b, Sink sink) {
  for (int r0 = a; r0 < b; r0 += kWarp) {
    const int r = r0 + lane;
    if (r < b) {
      const int slot = r % kTile;
      float* base = tile + ((slot >> 2) * kWarp << 2) + (slot & 3);
      float s = 0.0f;
#pragma unroll
      for (int i = 0; i < kWarp; ++i) {
        const int c = (((i & 7) + (lane >> 2)) & 7) | (i & 24);
        s += base[c << 2];
        base[c << 2] = 0.0f;
      }
      sink(r, s);
    }
  }
  __syncwarp();
}

// Warp-uniform window walk.  Every lane walks the same number L (a multiple
// of 4) of samples from its own 4-aligned start J0 in 8-sample blocks (two
// row quads; the second quad of a block wraps to quad 0 at the circular end
// of the tile).  Blocks that start past the lane's last sample `lim` are redirected
// to a per-warp dump block, so a lane writes at most 7 rows beyond its window
// (the bin criterion keeps those rows inside the live tile).  Inside the
// walked range:
//   MASK   samples with q = y^2 > qmax get G = 0 (exact truncation at
//          cutoff sigmas, any cutoff);
//   !MASK  no per-sample test: the <= 3 / <= 7 samples walked before / after a
//          window lie beyond cutoff sigmas, where G <= exp(-cutoff^2/2) <=
//          2^-24 (cutoff >= 5.77, host-checked), below the FP32 resolution
//          of the ball's own contribution.
// Two blocks per iteration (16 independent read-modify-writes in flight).
// Row quads updated in place (round 2): a lane's quad is read as two 64-bit
// halves, each half accumulated by an asm FFMA2 whose output operand is tied
// to its addend, and written back by two volatile 8-byte stores.  With the
// sums as plain float2 values the register allocation left them outside any
// aligned register quad and rebuilt every STS.128 source with four moves
// (16 per loop trip of either walk); bitwise the same rows.
#ifndef PAB_DUAL_TIED
#define PAB_DUAL_TIED 1
#endif
#ifndef PAB_DUAL_ST64
#define PAB_DUAL_ST64 1
#endif
__device__ __forceinline__ unsigned long long pack2(float2 v) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(v.x), "f"(v.y));
  return r;
}
__device__ __forceinline__ void st_quad(ulonglong2* p, const ulonglong2& v) {
#if PAB_DUAL_ST64   // two 8-byte stores: no register quad to assemble
  const unsigned a = (unsigned)__cvta_generic_to_shared(p);
  asm volatile("st.volatile.shared.b64 [%0], %1;\n\tst.volatile.shared.b64 [%0+8], %2;" ::"r"(a), "l"(v.x), "l"(v.y) : "memory");
#else
  *p = v;
#endif
}

template <bool MASK>
__device__ __forceinline__ float2 gauss2(float2 q, float qmax) {
  if (MASK) return make_float2(q.x <= qmax ? ex2(-q.x) : 0.0f, q.y <= qmax ? ex2(-q.y) : 0.0f);
  return make_float2(ex2(-q.x), ex2(-q.y));
}

// The amplitude rides in the exponent: Ak y 2^(-y^2) = sgn(Ak) y
// 2^(-(y^2 - log2|Ak|)), with sgn(Ak) folded into the y coefficients, so a
// sample costs y (FFMA2 half), y^2 - log2|Ak| (FFMA2 half), ex2 and the
// accumulate (FFMA2 half).  Ak = 0 gives log2 = -inf and an exact +0 term.
struct Walk {
  float2 nsc2, c0, c1, c2, c3;
  float2 nla2;   // (-log2|Ak|, -log2|Ak|)
  float qmax;    // truncation bound on y^2 - log2|Ak| (MASK)
};

template <bool MASK>
__device__ __forceinline__ float2 rmw_pair(float2 o, float2 m2, float2 c, const Walk& w) {
  const float2 y = __ffma2_rn(m2, w.nsc2, c);
  const float2 e = __ffma2_rn(y, y, w.nla2);
  const float2 g = gauss2<MASK>(e, w.qmax);
  return __ffma2_rn(y, g, o);
}

template <bool MASK>
__device__ __forceinline__ void rmw_pair_tied(unsigned long long& o, float2 m2, float2 c, const Walk& w) {
  const float2 y = __ffma2_rn(m2, w.nsc2, c);
  const float2 e = __ffma2_rn(y, y, w.nla2);
  const float2 g = gauss2<MASK>(e, w.qmax);
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(o) : "l"(pack2(y)), "l"(pack2(g)));
}
template <bool MASK>
__device__ __forceinline__ void rmw4_tied(ulonglong2& o, float2 m2, float2 ca, float2 cb, const Walk& w) {
  rmw_pair_tied<MASK>(o.x, m2, ca, w);
  rmw_pair_tied<MASK>(o.y, m2, cb, w);
}

__device__ __forceinline__ float4 rmw4(float4 o, float2 m2, float2 ca, float2 cb, const Walk& w,
                                       float2 (*pair)(float2, float2, float2, const Walk&)) {
  const float2 lo = pair(make_float2(o.x, o.y), m2, ca, w);
  const float2 hi = pair(make_float2(o.z, o.w), m2, cb, w);
  return make_float4(lo.x, lo.y, hi.x, hi.y);
}

#ifndef PAB_FWD_UNROLL
#define PAB_FWD_UNROLL 2   // 8-sample blocks per loop trip
#endif
// Walk parameters of one pair: nsc = -sc sgn(Ak), pss = phi sc sgn(Ak),
// nla = -log2|Ak| (+inf for Ak = 0), qmax_e = truncation bound on the
// exponent (MASK).
__device__ __forceinline__ Walk make_walk(float nsc, float pss, float fs, float nla, float qmax_e) {
  Walk w;
  w.nsc2 = make_float2(nsc, nsc);
  const float dl = fs * nsc, dl2 = 2.0f * dl;   // y step per sample / per sample pair
  w.c0 = make_float2(pss, pss + dl);
  w.c1 = __fadd2_rn(w.c0, make_float2(dl2, dl2));
  w.c2 = __fadd2_rn(w.c1, make_float2(dl2, dl2));
  w.c3 = __fadd2_rn(w.c2, make_float2(dl2, dl2));
  w.nla2 = make_float2(nla, nla);
  w.qmax = qmax_e;
  return w;
}

template <bool MASK>
__device__ __forceinline__ void rmw_walk(float* tile, int lane, int J0, int L, int lim, float mf, float fs,
                                         const Walk& w, int dump = kTile / 4);

// Walk with the amplitude as a factor (phase F): Ak y G with Ak folded into
// a second set of y coefficients (ya = m Ak nsc + Ak c ~ Ak y), so doubling
// Ak doubles every term exactly -- p0 linearity stays bitwise, as in the
// reference's amp * u * G (radiator.py:249-251) -- for one more FP32x2
// operation per sample pair than the exponent-folded walk.
struct AWalk {
  float2 nsc2, c0, c1, c2, c3;   // y = m nsc + c
  float2 an2, a0, a1, a2, a3;    // Ak-scaled coefficients
  float qmax;
};
__device__ __forceinline__ AWalk make_awalk(float nsc, float pss, float fs, float Ak, float qmax) {
  AWalk w;
  w.nsc2 = make_float2(nsc, nsc);
  const float dl = fs * nsc, dl2 = 2.0f * dl;
  w.c0 = make_float2(pss, pss + dl);
  w.c1 = __fadd2_rn(w.c0, make_float2(dl2, dl2));
  w.c2 = __fadd2_rn(w.c1, make_float2(dl2, dl2));
  w.c3 = __fadd2_rn(w.c2, make_float2(dl2, dl2));
  const float2 A2 = make_float2(Ak, Ak);
  w.an2 = __fmul2_rn(A2, w.nsc2);
  w.a0 = __fmul2_rn(A2, w.c0);
  w.a1 = __fmul2_rn(A2, w.c1);
  w.a2 = __fmul2_rn(A2, w.c2);
  w.a3 = __fmul2_rn(A2, w.c3);
  w.qmax = qmax;
  return w;
}
template <bool MASK>
__device__ __forceinline__ float2 rmw_pair_amp(float2 o, float2 m2, float2 c, float2 a, const AWalk& w) {
  const float2 y = __ffma2_rn(m2, w.nsc2, c);
  const float2 ya = __ffma2_rn(m2, w.an2, a);
  const float2 q = __fmul2_rn(y, y);
  const float2 g = gauss2<MASK>(q, w.qmax);
  return __ffma2_rn(ya, g, o);
}
template <bool MASK>
__device__ __forceinline__ void rmw_pair_amp_tied(unsigned long long& o, float2 m2, float2 c, float2 a, const AWalk& w) {
  const float2 y = __ffma2_rn(m2, w.nsc2, c);
  const float2 ya = __ffma2_rn(m2, w.an2, a);
  const float2 q = __fmul2_rn(y, y);
  const float2 g = gauss2<MASK>(q, w.qmax);
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(o) : "l"(pack2(ya)), "l"(pack2(g)));
}
// L a multiple of 8 from an 8-aligned J0 (blocks never wrap the circular
// tile); blocks starting past `lim` go to the dump block
template <bool MASK>
__device__ __forceinline__ void rmw_walk_amp(float* tile, int lane, int J0, int L, int lim, float mf, float fs,
                                             const AWalk& w) {
  float4* const T = reinterpret_cast<float4*>(tile) + lane;
  const int dump = kTile / 4;
  const float step = 8.0f * fs;
  int q = (J0 % kTile) >> 2;
  PAB_CHECK((J0 & 7) == 0 && (L & 7) == 0);
#pragma unroll 1
  for (int Jb = J0; Jb < J0 + L; Jb += 8, mf += step) {
    const bool live = Jb <= lim;
    const int qa = live ? q : dump;
    PAB_CHECK(qa >= 0 && qa + 1 <= dump + 1);
    const float2 m2 = make_float2(mf, mf);
#if PAB_DUAL_TIED
    ulonglong2* const U = reinterpret_cast<ulonglong2*>(T);
    ulonglong2 o0 = U[qa * kWarp], o1 = U[(qa + 1) * kWarp];
    rmw_pair_amp_tied<MASK>(o0.x, m2, w.c0, w.a0, w);
    rmw_pair_amp_tied<MASK>(o0.y, m2, w.c1, w.a1, w);
    rmw_pair_amp_tied<MASK>(o1.x, m2, w.c2, w.a2, w);
    rmw_pair_amp_tied<MASK>(o1.y, m2, w.c3, w.a3, w);
    st_quad(&U[qa * kWarp], o0);
    st_quad(&U[(qa + 1) * kWarp], o1);
#else
    float4 o0 = T[qa * kWarp], o1 = T[(qa + 1) * kWarp];
    const float2 p0 = rmw_pair_amp<MASK>(make_float2(o0.x, o0.y), m2, w.c0, w.a0, w);
    const float2 p1 = rmw_pair_amp<MASK>(make_float2(o0.z, o0.w), m2, w.c1, w.a1, w);
    const float2 p2 = rmw_pair_amp<MASK>(make_float2(o1.x, o1.y), m2, w.c2, w.a2, w);
    const float2 p3 = rmw_pair_amp<MASK>(make_float2(o1.z, o1.w), m2, w.c3, w.a3, w);
    T[qa * kWarp] = make_float4(p0.x, p0.y, p1.x, p1.y);
    T[(qa + 1) * kWarp] = make_float4(p2.x, p2.y, p3.x, p3.y);
#endif
    q += 2;
    if (q >= kTile / 4) q -= kTile / 4;
  }
}

template <bool MASK>
__device__ __forceinline__ void rmw_uniform(float* tile, int lane, int J0, int L, int lim, float mf, float fs,
                                            float sc, float ps, float Ak, float qmax, int dump = kTile / 4) {
  const float sg = Ak < 0.0f ? -1.0f : 1.0f;   // sgn(Ak) folded into y
  const float nla = -__log2f(fabsf(Ak));       // +inf for Ak = 0
  rmw_walk<MASK>(tile, lane, J0, L, lim, mf, fs, make_walk(-sc * sg, ps * sg, fs, nla, qmax + nla), dump);
}

template <bool MASK>
__device__ __forceinline__ void rmw_walk(float* tile, int lane, int J0, int L, int lim, float mf, float fs,
                                         const Walk& w, int dump) {
  constexpr int K = PAB_FWD_UNROLL;
  float4* const T = reinterpret_cast<float4*>(tile) + lane;   // quad q of this lane: T[q * 32]
  // dump block = quads dump, dump + 1 (relative to this tile)
  const float step = 8.0f * fs;
  constexpr int Q = kTile / 4;
  int q = (J0 % kTile) >> 2;   // first quad of the current block
  int Jb = J0;                 // row of the current block's first sample
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
    // every block's reads before any block's writes
#if PAB_DUAL_TIED
    ulonglong2* const U = reinterpret_cast<ulonglong2*>(T);
    ulonglong2 o[K][2];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      o[k][0] = U[qq[k] * kWarp];
      o[k][1] = U[qn[k] * kWarp];
    }
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const float2 m2 = make_float2(mf + (float)k * step, mf + (float)k * step);
      rmw4_tied<MASK>(o[k][0], m2, w.c0, w.c1, w);
      rmw4_tied<MASK>(o[k][1], m2, w.c2, w.c3, w);
    }
#pragma unroll
    for (int k = 0; k < K; ++k) {
      st_quad(&U[qq[k] * kWarp], o[k][0]);
      st_quad(&U[qn[k] * kWarp], o[k][1]);
    }
#else
    float4 o[K][2];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      o[k][0] = T[qq[k] * kWarp];
      o[k][1] = T[qn[k] * kWarp];
    }
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const float2 m2 = make_float2(mf + (float)k * step, mf + (float)k * step);
      o[k][0] = rmw4(o[k][0], m2, w.c0, w.c1, w, rmw_pair<MASK>);
      o[k][1] = rmw4(o[k][1], m2, w.c2, w.c3, w, rmw_pair<MASK>);
    }
#pragma unroll
    for (int k = 0; k < K; ++k) {
      T[qq[k] * kWarp] = o[k][0];
      T[qn[k] * kWarp] = o[k][1];
    }
#endif
    mf += (float)K * step;
  }
#pragma unroll 1
  for (; nb > 0; --nb) {
    const bool live = Jb <= lim;
    const int qb = live ? q : dump, qc = live ? (q + 1 == Q ? 0 : q + 1) : dump + 1;
    const float2 m2 = make_float2(mf, mf);
#if PAB_DUAL_TIED
    ulonglong2* const U = reinterpret_cast<ulonglong2*>(T);
    ulonglong2 a = U[qb * kWarp], b = U[qc * kWarp];
    rmw4_tied<MASK>(a, m2, w.c0, w.c1, w);
    rmw4_tied<MASK>(b, m2, w.c2, w.c3, w);
    st_quad(&U[qb * kWarp], a);
    st_quad(&U[qc * kWarp], b);
#else
    const float4 a = T[qb * kWarp], b = T[qc * kWarp];
    T[qb * kWarp] = rmw4(a, m2, w.c0, w.c1, w, rmw_pair<MASK>);
    T[qc * kWarp] = rmw4(b, m2, w.c2, w.c3, w, rmw_pair<MASK>);
#endif
    mf += step;
    q += 2;
    if (q >= Q) q -= Q;
    Jb += 8;
  }
  if (L & 4) {   // 4-sample tail: one quad
    const int qb = Jb <= lim ? q : dump;
    const float2 m2 = make_float2(mf, mf);
#if PAB_DUAL_TIED
    ulonglong2* const U = reinterpret_cast<ulonglong2*>(T);
    ulonglong2 a = U[qb * kWarp];
    rmw4_tied<MASK>(a, m2, w.c0, w.c1, w);
    st_quad(&U[qb * kWarp], a);
#else
    T[qb * kWarp] = rmw4(T[qb * kWarp], m2, w.c0, w.c1, w, rmw_pair<MASK>);
#endif
  }
}

// ---------------------------------------------------------------------------
// Dual walk: two balls per lane share every tile read-modify-write, and the
// Gaussian is advanced by a ratio recurrence for three of the four sample
// pairs of a block, so the walk needs 0.5 ex2 and 4 FP32 lane-ops per
// ball-sample and 4 bytes of shared-memory RMW per ball-sample (half the
// single walk's): the three per-SM ceilings (FP32 128, XU 16, shared 128 B
// per clock) all sit at 32 ball-samples per clock, 2x the single walk's.
//
// Per ball, y advances by dl = f * nsc per sample, e = y^2 + nla, G = 2^-e.
// Stepping a sample pair (y -> y + 2 dl) multiplies G by
//   R(y) = 2^-(4 dl y + 4 dl^2),  and R itself by C = 2^(-8 dl^2).
// Each 8-sample block computes pair 0 exactly (2 ex2) and R at pair 0 (2 ex2)
// from its own y, then pairs 1-3 by the recurrence: no state is carried
// between blocks, so rounding cannot accumulate past three steps (measured
// relative error of a term ~1e-6).  Underflow: pair 0's G flushes to zero
// only for e > 126; three pair steps later e has dropped by at most
// 12 |dl| (|y| + 3 |dl|), so with |dl| <= kDualMaxDl every term lost that way
// lies beyond cutoff sigmas and below 2^-40 of the ball's peak.  Overflow of
// R: the exponent is linear in y; the producer keeps every live walked sample
// at |y| <= kDualMaxY (else the pair walks singly), so R < 2^127 there;
// blocks past a lane's window go to the dump block and never reach the row.
// ---------------------------------------------------------------------------
constexpr float kDualMaxDl = 0.75f;   // max |y| step per sample for the recurrence (producer-checked)
constexpr float kDualMaxY = 30.0f;    // max |y| over a dual walk's live samples (producer-checked)

struct DWalk {
  float2 nsc2, c0, d2, nla2, kr2, br2, cc2;
  float mf;
};

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

// one ball's 8-sample block added into (o0, o1): block m-offset m
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

// Both balls of a lane added into a block's two row quads (o0, o1), the
// same operations in the same order as dual_block(a) then dual_block(b)
// (bitwise the same rows), arranged so that every 64-bit half of a quad is
// updated in place by one tied asm operand: t = ya ga + o; o = yb gb + t.
// (FFMA2 never writes its addend's register pair, and with the two FFMA2 as
// separate operations the register allocation left the sums outside the
// loaded quads: 16 moves per loop trip to rebuild the four STS.128 sources.)
struct DState {
  float2 y, g, r;
};
__device__ __forceinline__ DState dual_start(float m, const DWalk& w) {
  DState s;
  s.y = __ffma2_rn(make_float2(m, m), w.nsc2, w.c0);
  const float2 e0 = __ffma2_rn(s.y, s.y, w.nla2);
  const float2 er = __ffma2_rn(s.y, w.kr2, w.br2);
  s.g = make_float2(ex2(-e0.x), ex2(-e0.y));
  s.r = make_float2(ex2(er.x), ex2(er.y));
  return s;
}
template <bool LAST>
__device__ __forceinline__ void dual_step(DState& s, const DWalk& w) {
  s.y = __fadd2_rn(s.y, w.d2);
  s.g = __fmul2_rn(s.g, s.r);
  if (!LAST) s.r = __fmul2_rn(s.r, w.cc2);
}
__device__ __forceinline__ void dual_acc(unsigned long long& o, const DState& a, const DState& b) {
  asm("{\n\t.reg .b64 t;\n\t"
      "fma.rn.f32x2 t, %1, %2, %0;\n\t"
      "fma.rn.f32x2 %0, %3, %4, t;\n\t}"
      : "+l"(o)
      : "l"(pack2(a.y)), "l"(pack2(a.g)), "l"(pack2(b.y)), "l"(pack2(b.g)));
}
template <bool HALF = false>
__device__ __forceinline__ void dual_block2(ulonglong2& o0, ulonglong2& o1, float ma, const DWalk& wa, float mb,
                                            const DWalk& wb) {
  DState a = dual_start(ma, wa), b = dual_start(mb, wb);
  dual_acc(o0.x, a, b);
  dual_step<HALF>(a, wa);
  dual_step<HALF>(b, wb);
  dual_acc(o0.y, a, b);
  if (HALF) return;
  dual_step<false>(a, wa);
  dual_step<false>(b, wb);
  dual_acc(o1.x, a, b);
  dual_step<true>(a, wa);
  dual_step<true>(b, wb);
  dual_acc(o1.y, a, b);
}

#ifndef PAB_DUAL_UNROLL
#define PAB_DUAL_UNROLL 2   // 8-sample blocks per loop trip (each block carries two balls)
#endif
// Warp-uniform walk of L samples (multiple of 4) from the lane's 4-aligned
// union start J0; blocks starting past `lim` go to the dump block.
__device__ __forceinline__ void rmw_walk_dual(float* tile, int lane, int J0, int L, int lim, float fs,
                                              const DWalk& wa, const DWalk& wb, int dump = kTile / 4) {
  constexpr int K = PAB_DUAL_UNROLL;
  float4* const T = reinterpret_cast<float4*>(tile) + lane;
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
#if PAB_DUAL_TIED
    ulonglong2 o[K][2];
    ulonglong2* const U = reinterpret_cast<ulonglong2*>(T);
#pragma unroll
    for (int k = 0; k < K; ++k) {
      PAB_CHECK(qq[k] >= 0 && qq[k] <= dump && qn[k] >= 0 && qn[k] <= dump + 1);
      o[k][0] = U[qq[k] * kWarp];
      o[k][1] = U[qn[k] * kWarp];
    }
#pragma unroll
    for (int k = 0; k < K; ++k) dual_block2(o[k][0], o[k][1], ma + (float)k * step, wa, mb + (float)k * step, wb);
#pragma unroll
    for (int k = 0; k < K; ++k) {
      st_quad(&U[qq[k] * kWarp], o[k][0]);
      st_quad(&U[qn[k] * kWarp], o[k][1]);
    }
#else
    float4 o[K][2];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      PAB_CHECK(qq[k] >= 0 && qq[k] <= dump && qn[k] >= 0 && qn[k] <= dump + 1);
      o[k][0] = T[qq[k] * kWarp];
      o[k][1] = T[qn[k] * kWarp];
    }
#pragma unroll
    for (int k = 0; k < K; ++k) {
      dual_block(o[k][0], o[k][1], ma + (float)k * step, wa);
      dual_block(o[k][0], o[k][1], mb + (float)k * step, wb);
    }
#pragma unroll
    for (int k = 0; k < K; ++k) {
      T[qq[k] * kWarp] = o[k][0];
      T[qn[k] * kWarp] = o[k][1];
    }
#endif
    ma += (float)K * step;
    mb += (float)K * step;
  }
#pragma unroll 1
  for (; nb > 0; --nb) {
    const bool live = Jb <= lim;
    const int qb = live ? q : dump, qc = live ? (q + 1 == Q ? 0 : q + 1) : dump + 1;
#if PAB_DUAL_TIED
    ulonglong2* const U = reinterpret_cast<ulonglong2*>(T);
    ulonglong2 o0 = U[qb * kWarp], o1 = U[qc * kWarp];
    dual_block2(o0, o1, ma, wa, mb, wb);
    st_quad(&U[qb * kWarp], o0);
    st_quad(&U[qc * kWarp], o1);
#else
    float4 o0 = T[qb * kWarp], o1 = T[qc * kWarp];
    dual_block(o0, o1, ma, wa);
    dual_block(o0, o1, mb, wb);
    T[qb * kWarp] = o0;
    T[qc * kWarp] = o1;
#endif
    ma += step;
    mb += step;
    q += 2;
    if (q >= Q) q -= Q;
    Jb += 8;
  }
  if (L & 4) {   // 4-sample tail: the block's first quad only
    const int qb = Jb <= lim ? q : dump;
#if PAB_DUAL_TIED
    ulonglong2* const U = reinterpret_cast<ulonglong2*>(T);
    ulonglong2 o0 = U[qb * kWarp], o1 = make_ulonglong2(0ull, 0ull);
    dual_block2<true>(o0, o1, ma, wa, mb, wb);
    U[qb * kWarp] = o0;
#else
    float4 o0 = T[qb * kWarp], o1 = make_float4(0.f, 0.f, 0.f, 0.f);
    dual_block(o0, o1, ma, wa);
    dual_block(o0, o1, mb, wb);
    T[qb * kWarp] = o0;
#endif
  }
}

// One ball (lane) of one group against the CTA's detector in the time sweep,
// split into setup (geometry, window, weight: a latency-bound chain) and walk
// so the sweep can compute two groups' setups side by side.  Groups whose
// detector is close (slow geometry) take the linear-pass path instead.
struct PairSetup {
  int kc, jlo, jhi, J0, L;
  float phi, d, rho, sc, Ak, qmax;
  bool live;
};

template <int DIR, bool RED = true>
__device__ __forceinline__ PairSetup pair_setup(const Acq& acq, const GroupDet& gd, const DetDir& dd, const BallA& A,
                                                const BallB& B, unsigned long long& ops, int fp) {
  PairSetup p;
  const PairGeom pg = pair_geom_fast(gd, A, B, acq);
  p.kc = pg.kc;
  p.phi = pg.phi;
  p.d = pg.d;
  p.rho = acq.cutoff * A.a0 * acq.inv_vdt_f;
  p.sc = acq.vdt_f * kSqrtHalfLog2e * B.inv_a0;
  const float rs = p.rho * p.sc;
  p.qmax = rs * rs;
  pair_window(pg.kc, pg.phi, p.rho, acq, &p.jlo, &p.jhi);
  p.live = B.orig >= 0;
  if (!p.live) { p.jlo = 1; p.jhi = 0; }
  ops += (unsigned long long)max(p.jhi - p.jlo + 1, 0);
  float D = 1.0f;
  if (DIR != kDirNone)
    D = dir_weight<DIR, false>(dd, pg.rx * pg.id, pg.ry * pg.id, pg.rz * pg.id, pg.id, acq.dir_param,
                               acq.dir_param, B.inv_a0, nullptr, nullptr);
  // u G amp = Ak * y G with Ak = amp * kappa = (p0 D / 2d) a0 sqrt(2 ln 2)
  p.Ak = (0.5f * B.p0 * D) * pg.id * (A.a0 * kSqrt2Ln2);
  const bool empty = p.jlo > p.jhi;
  p.J0 = (empty ? fp : p.jlo) & ~3;
  p.L = RED ? __reduce_max_sync(0xffffffffu, empty ? 0 : p.jhi - p.J0 + 1) : 0;
  return p;
}

// The warp-uniform walk of the u- window (and, if any lane has one, of the
// u+ near-field window).  `fp` is a live tile row: the start of empty
// windows, which are redirected to the dump block.
template <bool MASK>
__device__ __forceinline__ void pair_walk(float* tile, int lane, const Acq& acq, const PairSetup& p, int near,
                                          unsigned long long& ops, int fp, int dump = kTile / 4) {
  const float fs = (float)acq.f;
  const bool empty_u = p.jlo > p.jhi;
  if (p.L > 0)
    rmw_uniform<MASK>(tile, lane, p.J0, (p.L + 3) & ~3, empty_u ? -1 : p.jhi, (float)(p.J0 * acq.f - p.kc), fs,
                      p.sc, p.phi * p.sc, empty_u ? 0.0f : p.Ak, p.qmax, dump);
  if (near) {
    int nlo = 1, nhi = 0, nkc = 0;
    float nphi = 0.0f;
    if (p.live) pair_near_window(p.d, p.rho, acq, &nlo, &nhi, &nkc, &nphi);
    ops += (unsigned long long)max(nhi - nlo + 1, 0);
    if (__any_sync(0xffffffffu, nlo <= nhi)) {   // u+ = -kappa y: walk with -sc
      const bool empty = nlo > nhi;
      const int J0 = (empty ? fp : nlo) & ~3;
      const int L = __reduce_max_sync(0xffffffffu, empty ? 0 : nhi - J0 + 1);
      rmw_uniform<MASK>(tile, lane, J0, (L + 3) & ~3, empty ? -1 : nhi, (float)(J0 * acq.f - nkc), fs, -p.sc,
                        nphi * -p.sc, empty ? 0.0f : p.Ak, p.qmax, dump);
    }
  }
}

// One ball (lane) of one group against the CTA's detector: setup, then the
// u- (and, near field, u+) window clipped to [clip_lo, clip_hi] into the tile.
template <int DIR>
__device__ __forceinline__ void evaluate_pair(float* tile, int lane, const Acq& acq, const GroupDet& gd,
                                              const GroupMeta& gm, const Detector& det, const DetDir& dd,
                                              const BallA& A, const BallB& B, int near, unsigned long long& ops,
                                              int& coinc, int clip_lo, int clip_hi) {
  const PairGeom pg = pair_geom(gd, gm, det.px, det.py, det.pz, A, B, acq);
  coinc |= pg.coincident;
  const float rho = acq.cutoff * A.a0 * acq.inv_vdt_f;
  const float sc = acq.vdt_f * kSqrtHalfLog2e * B.inv_a0;
  int jlo, jhi;
  pair_window(pg.kc, pg.phi, rho, acq, &jlo, &jhi);
  if (B.orig < 0) { jlo = 1; jhi = 0; }
  int nlo = 1, nhi = 0, nkc = 0;
  float nphi = 0.0f;
  if (near && B.orig >= 0) pair_near_window(pg.d, rho, acq, &nlo, &nhi, &nkc, &nphi);
  ops += (unsigned long long)(max(jhi - jlo + 1, 0) + max(nhi - nlo + 1, 0));
  float D = 1.0f;
  if (DIR != kDirNone)
    D = dir_weight<DIR, false>(dd, pg.rx * pg.id, pg.ry * pg.id, pg.rz * pg.id, pg.id, acq.dir_param,
                               acq.dir_param, B.inv_a0, nullptr, nullptr);
  // u G amp = Ak * y G with Ak = amp * kappa = (p0 D / 2d) a0 sqrt(2 ln 2)
  const float Ak = (0.5f * B.p0 * D) * pg.id * (A.a0 * kSqrt2Ln2);
  rmw_window(tile, lane, max(jlo, clip_lo), min(jhi, clip_hi), pg.kc, acq.f, sc, pg.phi, Ak);
  if (nlo <= nhi)   // u+ = -kappa y
    rmw_window(tile, lane, max(nlo, clip_lo), min(nhi, clip_hi), nkc, acq.f, -sc, nphi, Ak);
}

// Groups wider than the tile (phase F of the sweep: rare in dense clouds, a
// quarter of the groups of a sparse filtered cloud), in their own kernel
// after the sweep: grid = detectors x partitions as forward_kernel, 4 warps
// with a tile each.  Per chunk of the partition the wide groups are found by
// the sweep's own criterion (bin_of: span beyond the tile, detector within
// two group radii, u+ window possible), listed in order, and added to the
// partition's row: the union of their sample ranges is split into one
// 8-aligned time range per warp (the warps never write the same row: no
// races, a fixed per-row order); a warp sweeps its range in tile-aligned
// pieces, per piece every wide group that reaches it is set up (lane-parallel
// group geometry for 32 groups, then per pair: FP64 geometry near the
// detector, exact windows, weight) and walked with the vectorised walk from
// 8-aligned starts clipped to the piece (blocks never straddle a piece or a
// warp range, the amplitude as a factor: p0 linearity stays bitwise), and
// the piece is flushed once.  (Round 2 v2 ran this inside the sweep kernel,
// one warp-uniform group at a time with scalar per-sample walks while the
// setup warps idled at the barrier: 68 % of the f = 1 forward of the config-3
// reconstruction; kept inside the sweep kernel the new code cost config 2
// +0.5 ms through the sweep's register allocation.)
#ifndef PAB_FWD_WS
#define PAB_FWD_WS 1   // warp-specialised sweep (setup producers + walkers)
#endif
constexpr bool kWS = PAB_FWD_WS != 0;

// Group geometry of a setup warp's batch (dual entries: the first group's
// with the entry's bin / span / pair word, then the second group's), kept
// in the bin histogram's space while the sweep runs: 2 x float4 per group,
// read by broadcast LDS.128 instead of 7-8 shuffles per group.
constexpr int kPTabWords = 8;
__host__ __device__ inline int hist_ints(int n_bins, int warps, bool dual) {
  // dual: two groups per entry; single-group sweeps: geometry + word + slot (12 words)
  const int t = dual ? 2 * warps * kWarp * kPTabWords : warps * kWarp * 12;
  return n_bins + 1 > t ? n_bins + 1 : t;
}

// An entry (a group, or a dual pair's union) sweeps only if its rows
// [blo, hi + 7] (4-aligned starts, the last block may run 7 rows past the
// window) fit the live tile and its pairs take the fast geometry; groups
// close to the detector (FP64 per-pair geometry) and, warp-specialised,
// groups that may have a u+ window go to the wide-group kernel too.
__device__ __forceinline__ bool wide_entry(int l, int h, bool slow, bool near) {
  const int blo = l & ~((1 << kBinShift) - 1);
  return h + 7 - blo + 1 > kTile || slow || near;
}

constexpr int kWideChunk = 4096;   // groups scanned per pass (u8 flags + u16 list in shared memory)
constexpr int kWideWarps = 4;

// The wide groups of one detector x partition CTA, given by gidx(i) (global
// group index, i < n_wide, in a fixed order), added to the partition's row.
template <int DIR, bool MASK, class GIdx>
__device__ __forceinline__ void wide_pass(float* tile, int lane, int warp, const Acq& acq, const Detector& det,
                                          const DetDir& dd, const GroupMeta* __restrict__ gmeta,
                                          const BallA* __restrict__ ra, const BallB* __restrict__ rb, int n_wide,
                                          GIdx gidx, float* row, unsigned long long& my_ops, int& coinc) {
  constexpr int W = kWideWarps;
  const int n_out = acq.n_out;
  int umin = INT_MAX, umax = INT_MIN;   // union of the wide groups' ranges (every warp alike)
  for (int i0 = 0; i0 < n_wide; i0 += kWarp) {
    int lo = INT_MAX, hi = INT_MIN;
    if (i0 + lane < n_wide) {
      const GroupMeta gm = gmeta[gidx(i0 + lane)];
      const GroupDet gd = group_det(gm, det.px, det.py, det.pz, acq);
      group_range(acq, gd, gm, &lo, &hi);
    }
    umin = min(umin, __reduce_min_sync(0xffffffffu, lo));
    umax = max(umax, __reduce_max_sync(0xffffffffu, hi));
  }
  const int ub = umin & ~7;
  const int nblk = ((umax - ub) >> 3) + 1;   // 8-row blocks of the union
  const int t0 = ub + 8 * (int)(((int64_t)nblk * warp) / W), t1 = ub + 8 * (int)(((int64_t)nblk * (warp + 1)) / W);
  const float fs = (float)acq.f;
  for (int P = t0 - t0 % kTile; P < t1; P += kTile) {   // tile-aligned pieces of [t0, t1)
    const int c0 = max(P, t0), c1 = min(P + kTile, t1) - 1;   // c0 = 0 mod 8, c1 = 7 mod 8
    int rlo = INT_MAX, rhi = INT_MIN;   // rows the piece's walks wrote (warp-uniform)
    for (int i0 = 0; i0 < n_wide; i0 += kWarp) {
      const int nbat = min(kWarp, n_wide - i0);
      GroupDet gd_l = empty_gd();
      int lo_l = 1, hi_l = 0, near_l = 0;
      int64_t g_l = 0;
      if (lane < nbat) {
        g_l = gidx(i0 + lane);
        const GroupMeta gm = gmeta[g_l];
        gd_l = group_det(gm, det.px, det.py, det.pz, acq);
        group_range(acq, gd_l, gm, &lo_l, &hi_l);
        near_l = group_near(acq, gd_l, gm) ? 1 : 0;
      }
      unsigned todo = __ballot_sync(0xffffffffu, lane < nbat && lo_l <= c1 && hi_l >= c0);
      while (todo) {
        const int k = __ffs(todo) - 1;
        todo &= todo - 1;
        GroupDet gd = shfl_gd_fast(gd_l, k);
        gd.slow = __shfl_sync(0xffffffffu, gd_l.slow, k);
        const int64_t g = __shfl_sync(0xffffffffu, g_l, k);
        const int glo = __shfl_sync(0xffffffffu, lo_l, k);
        const int near = __shfl_sync(0xffffffffu, near_l, k);
        const GroupMeta gm = gmeta[g];
        const BallA A = ra[g * kWarp + lane];
        const BallB B = rb[g * kWarp + lane];
        const PairGeom pg = pair_geom(gd, gm, det.px, det.py, det.pz, A, B, acq);
        coinc |= pg.coincident;
        const bool live = B.orig >= 0;
        const float rho = acq.cutoff * A.a0 * acq.inv_vdt_f;
        const float sc = acq.vdt_f * kSqrtHalfLog2e * B.inv_a0;
        const float qmax = (rho * sc) * (rho * sc);
        int jlo = 1, jhi = 0, nlo = 1, nhi = 0, nkc = 0;
        float nphi = 0.0f;
        if (live) {
          pair_window(pg.kc, pg.phi, rho, acq, &jlo, &jhi);
          if (near) pair_near_window(pg.d, rho, acq, &nlo, &nhi, &nkc, &nphi);
        }
        if (glo >= c0 && glo <= c1)   // counted once: the piece of the warp range holding the group's first row
          my_ops += (unsigned long long)(max(jhi - jlo + 1, 0) + max(nhi - nlo + 1, 0));
        float D = 1.0f;
        if (DIR != kDirNone)
          D = dir_weight<DIR, false>(dd, pg.rx * pg.id, pg.ry * pg.id, pg.rz * pg.id, pg.id, acq.dir_param,
                                     acq.dir_param, B.inv_a0, nullptr, nullptr);
        const float Ak = (0.5f * B.p0 * D) * pg.id * (A.a0 * kSqrt2Ln2);
        // one window clipped to the piece: 8-aligned start >= c0, live
        // blocks start <= the clipped end (<= c1, so they end <= c1)
        auto clip_walk = [&](int wlo, int whi, int kc, float s, float ph) {
          const int a = max(wlo, c0), b = min(whi, c1);
          const bool empty = a > b;
          const int J0 = empty ? c0 : (a & ~7);
          const int L = __reduce_max_sync(0xffffffffu, empty ? 0 : b - J0 + 1);
          if (L > 0) {
            rlo = min(rlo, __reduce_min_sync(0xffffffffu, empty ? INT_MAX : J0));
            rhi = max(rhi, __reduce_max_sync(0xffffffffu, empty ? INT_MIN : (b | 7)));
          }
          if (L > 0)
            rmw_walk_amp<MASK>(tile, lane, J0, (L + 7) & ~7, empty ? -1 : b, (float)(J0 * acq.f - kc), fs,
                               make_awalk(-s, ph * s, fs, empty ? 0.0f : Ak, qmax));
        };
        clip_walk(jlo, jhi, pg.kc, sc, pg.phi);
        if (__any_sync(0xffffffffu, nlo <= nhi)) clip_walk(nlo, nhi, nkc, -sc, nphi);   // u+ = -kappa y
        __syncwarp();
      }
    }
    if (rlo <= rhi)   // only the rows the walks wrote (a piece may see no wide group)
      flush_rows(tile, lane, rlo, min(rhi + 1, n_out), [&](int r, float v) { row[r] += v; });
  }
  // walked blocks past the signal end (rows >= n_out) are never flushed
  for (int i = lane; i < kTile * kWarp / 4; i += kWarp)
    reinterpret_cast<float4*>(tile)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  __syncwarp();
}

template <int DIR, bool MASK>
__global__ void __launch_bounds__(kWideWarps * 32, 2)
forward_wide_kernel(const BallA* __restrict__ ra, const BallB* __restrict__ rb, const GroupMeta* __restrict__ gmeta,
                    int64_t n_groups, const double* __restrict__ det_pos, const double* __restrict__ det_aux,
                    int n_det, Acq acq, int64_t groups_per_part, float* __restrict__ partial_rows,
                    const int* __restrict__ wide_list, int wide_cap, unsigned long long* __restrict__ ops_total,
                    int* __restrict__ status) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  constexpr int W = kWideWarps;
  const int j = blockIdx.x;
  const int part = blockIdx.y;
  // the sweep listed this CTA's wide groups (count, then up to wide_cap
  // global group indices in its sort order): nothing to do for most CTAs
  const int* list = wide_list + ((size_t)part * n_det + j) * (size_t)(wide_cap + 1);
  const int count = list[0];
  if (count == 0) return;
  float* tiles = reinterpret_cast<float*>(smem_raw);
  unsigned char* flag = smem_raw + (size_t)W * kTileAlloc * kWarp * sizeof(float);
  unsigned short* wide = reinterpret_cast<unsigned short*>(flag + kWideChunk);
  __shared__ int n_wide_s;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, tid = threadIdx.x;
  const int n_out = acq.n_out;
  float* row = partial_rows + ((size_t)part * n_det + j) * (size_t)n_out;
  float* tile = tiles + (size_t)warp * kTileAlloc * kWarp;
  for (int i = tid; i < W * kTileAlloc * kWarp; i += blockDim.x) tiles[i] = 0.0f;
  __syncthreads();
  const Detector det = load_detector(det_pos, det_aux, j);
  DetDir dd{};
  if (DIR != kDirNone) dd = load_detdir(det_aux, j);
  unsigned long long my_ops = 0;
  int coinc = 0;
  if (count <= wide_cap) {
    wide_pass<DIR, MASK>(tile, lane, warp, acq, det, dd, gmeta, ra, rb, count,
                         [&](int i) -> int64_t { return list[1 + i]; }, row, my_ops, coinc);
  } else {
    // list overflow: find them again, chunk by chunk, with the sweep's
    // phase-A criterion (the same functions: the same groups)
    const int64_t g_begin = (int64_t)part * groups_per_part;
    const int64_t g_end = min(n_groups, g_begin + groups_per_part);
    for (int64_t cg0 = g_begin; cg0 < g_end; cg0 += kWideChunk) {
      const int cgn = (int)min((int64_t)kWideChunk, g_end - cg0);
      for (int gl = tid; gl < cgn; gl += blockDim.x) {
        const GroupMeta gm = gmeta[cg0 + gl];
        const GroupDet gd = group_det(gm, det.px, det.py, det.pz, acq);
        int lo, hi;
        group_range(acq, gd, gm, &lo, &hi);
        const bool nr = kWS && group_near(acq, gd, gm);
        flag[gl] = (lo <= hi && wide_entry(lo, hi, gd.slow != 0, nr)) ? 1 : 0;
      }
      __syncthreads();
      if (warp == 0) {   // ordered compaction
        int n = 0;
        for (int b0 = 0; b0 < cgn; b0 += kWarp) {
          const bool f = b0 + lane < cgn && flag[b0 + lane];
          const unsigned m = __ballot_sync(0xffffffffu, f);
          if (f) wide[n + __popc(m & ((1u << lane) - 1u))] = (unsigned short)(b0 + lane);
          n += __popc(m);
        }
        if (lane == 0) n_wide_s = n;
      }
      __syncthreads();
      const int n_wide = n_wide_s;
      if (n_wide > 0)
        wide_pass<DIR, MASK>(tile, lane, warp, acq, det, dd, gmeta, ra, rb, n_wide,
                             [&](int i) -> int64_t { return cg0 + wide[i]; }, row, my_ops, coinc);
      __syncthreads();   // flags / list reused by the next chunk
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    my_ops += __shfl_xor_sync(0xffffffffu, my_ops, o);
    coinc |= __shfl_xor_sync(0xffffffffu, coinc, o);
  }
  if (lane == 0) {
    if (my_ops) atomicAdd(ops_total, my_ops);
    if (coinc) atomicOr(status, kStatusCoincident);
  }
}

#ifndef PAB_FWD_MINB
#define PAB_FWD_MINB 2
#endif
#ifdef PAB_FWD_PROF   // tuning builds only: per-phase clock totals (lane 0 of each warp)
__device__ unsigned long long g_fwd_prof[32];
#define PROF_T(v) long long v = clock64()
#define PROF_ADD(i, t0) do { if (lane == 0) atomicAdd(&g_fwd_prof[(i)], (unsigned long long)(clock64() - (t0))); } while (0)
#define PROF_ACC(acc, t0) (acc) += clock64() - (t0)
#else
#define PROF_T(v)
#define PROF_ADD(i, t0)
#define PROF_ACC(acc, t0)
#endif

#ifndef PAB_FWD_DUAL
#define PAB_FWD_DUAL 1   // warp-specialised unmasked sweeps walk two balls per lane (dual walk)
#endif
constexpr bool kDual = PAB_FWD_DUAL != 0;
#ifndef PAB_FWD_WALKERS_HIGH
#define PAB_FWD_WALKERS_HIGH 0
#endif
constexpr bool kWalkersHigh = PAB_FWD_WALKERS_HIGH != 0;

template <int DIR, bool MASK, bool SROW, bool WS, bool DL>
__global__ void __launch_bounds__(kMaxWarps * 32 * (WS ? 2 : 1), PAB_FWD_MINB)
forward_kernel(const BallA* __restrict__ ra, const BallB* __restrict__ rb,
               const GroupMeta* __restrict__ gmeta, const unsigned char* __restrict__ ptab, int64_t n_groups,
               const double* __restrict__ det_pos, const double* __restrict__ det_aux, int n_det,
               Acq acq, int64_t groups_per_part, float* __restrict__ partial_rows, int* __restrict__ wide_list,
               int wide_cap, unsigned long long* __restrict__ ops_total, int* __restrict__ status) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  // WS: warps [0, W) walk (one tile each), warps [W, 2W) compute the pair
  // setups of walker (warp - W)'s slice and hand them over through a
  // two-slot ring per walker (mbarrier full / empty)
  // DUAL: the sort / sweep unit is a pair of consecutive lane groups (a
  // "super-group" of 64 balls); lane l walks balls 2l, 2l+1 of the pair's
  // 64 (consecutive in the Hilbert order: nearly the same arrival window)
  constexpr bool DUAL = DL;   // host: WS && !MASK && pair table given
  constexpr int kCU = kChunk;                       // group slots per chunk
  constexpr int kUG = DUAL ? 2 : 1;                 // lane groups per sort unit
  const int W = (blockDim.x >> 5) / (WS ? 2 : 1);
  const int n_out = acq.n_out;
  const int j = blockIdx.x;
  // partitions are contiguous in the processing order, which ascends in a0
  // bucket: the wide-window partitions launch first, the light ones fill the
  // tail (measured: config 2 -0.04 ms, config-3 reconstruction -3 %)
  const int part = gridDim.y - 1 - blockIdx.y;
  const int n_bins = (n_out + (1 << kBinShift) - 1) >> kBinShift;
  // SROW: the detector row in shared memory; otherwise (long records) the
  // CTA's partial row in global memory (L2): written only by this CTA, each
  // sample by one warp at a time, in a fixed order
  float* row = SROW ? reinterpret_cast<float*>(smem_raw) : partial_rows + ((size_t)part * n_det + j) * (size_t)n_out;
  float* tiles = reinterpret_cast<float*>(smem_raw) + (SROW ? ((n_out + 3) & ~3) : 0);
  // walker tiles (kTile rows each) and ONE dump block shared by the walkers:
  // it only takes the write-only overrun of blocks past a lane's window
  float* stage = tiles + (size_t)W * kTile * kWarp + kDumpFloats;
  int* hist = reinterpret_cast<int*>(stage + W * kTile);        // [n_bins + 1]
  // (DUAL: during the sweep the histogram's space holds the setup warps'
  // tables of their batches' second-group geometry, kPTabWords per entry)
  int* zs = hist + hist_ints(n_bins, W, DUAL);                 // [W + 1]
  int* misc = zs + W + 1;                                       // [4]
  unsigned short* sorted = reinterpret_cast<unsigned short*>(misc + 4);
  unsigned short* gbin = sorted + kCU;
  // WS hand-off ring: per walker and slot, 32 lane records (2 x float4) and
  // a header (L, blo, ghi); mbarriers full / empty per walker and slot
  // (offset arithmetic on smem_raw, not an integer round trip, so the
  // compiler keeps the shared address space: LDS/STS instead of generic LD/ST)
  const size_t ring_off = (reinterpret_cast<unsigned char*>(gbin + kCU) - smem_raw + 15) & ~(size_t)15;
  float4* slot_a = reinterpret_cast<float4*>(smem_raw + ring_off);
  float4* slot_b = slot_a + W * kRing * kWarp;
  float* slot_c = reinterpret_cast<float*>(slot_b + W * kRing * kWarp);   // DUAL only
  int4* slot_h = DUAL ? reinterpret_cast<int4*>(slot_c + W * kRing * kWarp)
                      : reinterpret_cast<int4*>(slot_b + W * kRing * kWarp);
  unsigned long long* mb_full = reinterpret_cast<unsigned long long*>(slot_h + W * kRing);
  unsigned long long* mb_empty = mb_full + W * kRing;

  // logical warp index: with PAB_FWD_WALKERS_HIGH the walkers (logical
  // warps [0, W)) run on the physically higher warps [W, 2W), which the
  // warp scheduler prefers when both a walker and a producer are eligible
  const int warp = (WS && kWalkersHigh) ? (int)((threadIdx.x >> 5) + W) % (2 * W) : (int)(threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  const int tid = threadIdx.x, nthr = blockDim.x;

  if (WS && tid == 0) {
    for (int b = 0; b < kRing * W; ++b) {
      mbar_init(&mb_full[b], kWarp);
      mbar_init(&mb_empty[b], kWarp);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  unsigned ring_par = WS ? (warp < W ? 0u : (1u << kRing) - 1u) : 0u;   // per-slot wait parities (producers start at 1)
  for (int i = tid; i < n_out; i += nthr) row[i] = 0.0f;
  for (int i = tid; i < W * kTile * kWarp + kDumpFloats; i += nthr) tiles[i] = 0.0f;
  static_assert(kTile % 8 == 0, "8-sample blocks must not straddle the circular wrap");
  for (int i = tid; i < W * kTile; i += nthr) stage[i] = 0.0f;

  const Detector det = load_detector(det_pos, det_aux, j);
  DetDir dd{};
  if (DIR != kDirNone) dd = load_detdir(det_aux, j);
  float* tile = tiles + (size_t)(warp < W ? warp : 0) * kTile * kWarp;
  const int dumpq = (W - (warp < W ? warp : 0)) * (kTile / 4);   // the shared dump block, in this tile's quads
  const int64_t g_begin = (int64_t)part * groups_per_part;
  const int64_t g_end = min(n_groups, g_begin + groups_per_part);
  unsigned long long my_ops = 0;
  int coinc = 0;
  int* const wide_out = wide_list + ((size_t)part * n_det + j) * (size_t)(wide_cap + 1);
  int wide_count = 0;   // wide entries of this CTA (all chunks)

#ifdef PAB_FWD_PROF
  long long pw_wait = 0, pw_room = 0, pw_walk = 0, pp_setup = 0, pp_pub = 0, pp_geo = 0, pw_lanes = 0, pw_groups = 0;
  const int pslot = (WS && warp >= W) ? 16 : 0;   // walkers 0.., producers 16..
#endif
  for (int64_t cg0 = g_begin; cg0 < g_end; cg0 += kChunk) {
    const int cgn = (int)min((int64_t)kChunk, g_end - cg0);   // lane groups in this chunk
    const int cn = (cgn + kUG - 1) / kUG;                      // sort units in this chunk
    PROF_T(t_a);
    for (int i = tid; i < n_bins + 1; i += nthr) hist[i] = 0;
    __syncthreads();

    // ---- A: bin every group of the chunk by its first sample ----
    // DUAL: a pair of consecutive groups is one sort entry (walked two balls
    // per lane) when its union range fits the tile; otherwise each group is
    // its own entry (single walk) or, if it alone is too wide, oversize.
    // gbin is per group slot; a pair's second slot holds kDualTail.
    for (int gl = tid; gl < cn; gl += nthr) {
      int lo[kUG], hi[kUG];
      bool slow[kUG], nr[kUG];
      for (int u = 0; u < kUG; ++u) {
        lo[u] = 1; hi[u] = 0; slow[u] = false; nr[u] = false;
        if (kUG * gl + u >= cgn) break;
        const GroupMeta gm = gmeta[cg0 + kUG * gl + u];
        const GroupDet gd = group_det(gm, det.px, det.py, det.pz, acq);
        group_range(acq, gd, gm, &lo[u], &hi[u]);
        slow[u] = gd.slow != 0;
        nr[u] = WS && group_near(acq, gd, gm);
      }
      // a lane writes rows [blo, hi + 7] (4-aligned starts, last block may
      // run 7 rows past the window): the span must fit the live tile; wide
      // groups and groups close to the detector (FP64 per-pair geometry)
      // take the linear-pass path (phase F) (WS: near-field groups too --
      // the hand-off carries the u- walk only)
      auto bin_of = [&](int l, int h, bool sl, bool n) -> unsigned short {
        if (l > h) return kEmptyBin;
        return wide_entry(l, h, sl, n) ? (unsigned short)n_bins : (unsigned short)(l >> kBinShift);
      };
      if (DUAL && kUG * gl + 1 < cgn && lo[0] <= hi[0] && lo[kUG - 1] <= hi[kUG - 1]) {
        const unsigned short b = bin_of(min(lo[0], lo[kUG - 1]), max(hi[0], hi[kUG - 1]),
                                        slow[0] || slow[kUG - 1], nr[0] || nr[kUG - 1]);
        if (b != (unsigned short)n_bins) {   // the pair fits: one dual entry
          atomicAdd(&hist[b], 1);            // counts only: order-independent
          gbin[kUG * gl] = b;
          gbin[kUG * gl + kUG - 1] = kDualTail;
          continue;
        }
      }
      for (int u = 0; u < kUG && kUG * gl + u < cgn; ++u) {
        const unsigned short b = bin_of(lo[u], hi[u], slow[u], nr[u]);
        if (b != kEmptyBin) atomicAdd(&hist[b], 1);
        gbin[kUG * gl + u] = b;
      }
    }
    PROF_ADD(pslot + 0, t_a);
    PROF_T(t_a2);
    __syncthreads();
    PROF_ADD(pslot + 1, t_a2);
    PROF_T(t_b);

    // ---- B+C: exclusive scan of the bin counts, then a stable in-order
    // scatter (sorted[] lists entries by start bin, slot order within a bin).
    // With room in the tile memory (idle between sweeps) every warp scatters
    // a contiguous slice of the slots, offset per bin by the earlier warps'
    // counts of that bin: the same order as one warp visiting all slots (the
    // serial form below), in an eighth of the steps (the serial scatter kept
    // the other warps at the barrier for ~3.5 % of the kernel at config 2).
    const int NWB = nthr >> 5;
    const int pwarp = tid >> 5;
    int* const cnt = reinterpret_cast<int*>(tiles);   // [NWB][n_bins + 1]
    const bool par_b = (size_t)NWB * (n_bins + 1) <= (size_t)W * kTile * kWarp;
    if (par_b) {
      const int sw = cgn * pwarp / NWB, ew = cgn * (pwarp + 1) / NWB;
      int* const myc = cnt + (size_t)pwarp * (n_bins + 1);
      for (int i = lane; i < n_bins + 1; i += kWarp) myc[i] = 0;   // over dump / tile slots: restored below
      __syncwarp();
      for (int gl = sw + lane; gl < ew; gl += kWarp) {
        const unsigned short bin = gbin[gl];
        if (bin < kDualTail) atomicAdd(&myc[bin], 1);
      }
      if (warp == 0) {   // the bin offsets (counts from phase A)
        const int total = n_bins + 1;
        int carry = 0;
        for (int c0 = 0; c0 < total; c0 += kWarp) {
          const int i = c0 + lane;
          const int x = i < total ? hist[i] : 0;
          int incl = x;
          for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
          }
          if (i < total) hist[i] = carry + incl - x;
          carry += __shfl_sync(0xffffffffu, incl, 31);
        }
        __syncwarp();
        if (lane == 0) {
          misc[0] = hist[n_bins];   // start of the oversize list = regular count
          misc[1] = carry;          // all listed entries
        }
      }
      __syncthreads();
      for (int b = tid; b < n_bins + 1; b += nthr) {   // per bin: offsets of each warp's first entry
        int run = hist[b];
        for (int w = 0; w < NWB; ++w) {
          const int c = cnt[(size_t)w * (n_bins + 1) + b];
          cnt[(size_t)w * (n_bins + 1) + b] = run;
          run += c;
        }
      }
      __syncthreads();
      for (int b0 = sw; b0 < ew; b0 += kWarp) {
        const int gl = b0 + lane;
        unsigned short bin = gl < ew ? gbin[gl] : kEmptyBin;
        const bool pair = DUAL && bin < kDualTail && gl + 1 < cgn && gbin[gl + 1] == kDualTail;
        if (bin == kDualTail) bin = kEmptyBin;
        const unsigned mask = __match_any_sync(0xffffffffu, (int)bin);
        int pos = 0;
        if (bin != kEmptyBin) pos = myc[bin] + __popc(mask & lanemask_lt());
        __syncwarp();
        if (bin != kEmptyBin) {
          sorted[pos] = (unsigned short)(gl | (pair ? 0x8000 : 0));
          if ((mask & lanemask_lt()) == 0) myc[bin] += __popc(mask);
        }
        __syncwarp();
      }
      for (int i = lane; i < n_bins + 1; i += kWarp) myc[i] = 0;   // the sweep needs zero tiles
    } else
    // ---- B+C (warp 0): exclusive scan, then a stable in-order scatter ----
    if (warp == 0) {
      const int total = n_bins + 1;
      int carry = 0;
      for (int c0 = 0; c0 < total; c0 += kWarp) {
        const int i = c0 + lane;
        const int x = i < total ? hist[i] : 0;
        int incl = x;
        for (int o = 1; o < 32; o <<= 1) {
          const int y = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += y;
        }
        if (i < total) hist[i] = carry + incl - x;
        carry += __shfl_sync(0xffffffffu, incl, 31);
      }
      __syncwarp();
      if (lane == 0) {
        misc[0] = hist[n_bins];   // start of the oversize list = regular count
        misc[1] = carry;          // all listed groups
#ifdef PAB_FWD_STATS   // tuning builds: oversize-group count in the op counter's high bits
        if (ops_total) atomicAdd(ops_total, (unsigned long long)(carry - hist[n_bins]) << 40);
#endif
      }
      for (int b0 = 0; b0 < cgn; b0 += kWarp) {
        const int gl = b0 + lane;
        unsigned short bin = gl < cgn ? gbin[gl] : kEmptyBin;
        // DUAL entries are listed by their first slot, flagged in bit 15
        const bool pair = DUAL && bin < kDualTail && gl + 1 < cgn && gbin[gl + 1] == kDualTail;
        if (bin == kDualTail) bin = kEmptyBin;
        const unsigned mask = __match_any_sync(0xffffffffu, (int)bin);
        int pos = 0;
        if (bin != kEmptyBin) pos = hist[bin] + __popc(mask & lanemask_lt());
        __syncwarp();
        if (bin != kEmptyBin) {
          sorted[pos] = (unsigned short)(gl | (pair ? 0x8000 : 0));
          if ((mask & lanemask_lt()) == 0) hist[bin] += __popc(mask);
        }
        __syncwarp();
      }
    }
    __syncthreads();
    PROF_ADD(pslot + 2, t_b);
    PROF_T(t_d);

    const int n_reg = misc[0];
    {   // the wide entries sorted[n_reg, misc[1]) (single groups) go to forward_wide_kernel's list
      const int n_all = misc[1];
      for (int i = n_reg + tid; i < n_all; i += nthr) {
        const int k = wide_count + (i - n_reg);
        if (k < wide_cap) wide_out[1 + k] = (int)(cg0 + (sorted[i] & 0x7FFF));
      }
      wide_count += n_all - n_reg;
    }

    // zone starts: the first row of each walker's slice (an empty slice takes
    // the next non-empty one's start; slices are n_reg * w / W, n_reg <= 2^15)
    if (tid <= W) {
      int z = n_out;
      for (int w = tid; w < W; ++w) {
        const int s = n_reg * w / W, e = n_reg * (w + 1) / W;
        if (s < e) { z = (int)gbin[sorted[s] & 0x7FFF] << kBinShift; break; }
      }
      zs[tid] = z;
    }
    __syncthreads();

    // ---- D: time-ordered sweep of each walker's slice ----
    // batch precompute: lane l of a 32-group batch computes the l-th group's
    // FP64 geometry; its start bin, span and near flag travel in one word
    auto batch_geometry = [&](int i0, int nb, GroupDet& gd_l, int64_t& g_l, unsigned& word_l) {
      gd_l = empty_gd();
      g_l = 0;
      word_l = 0;
      if (lane < nb) {
        const int gl = sorted[i0 + lane];
        g_l = cg0 + gl;
        const int bin = gbin[gl];
        const GroupMeta gm = gmeta[g_l];
        gd_l = group_det(gm, det.px, det.py, det.pz, acq);
        int glo, ghi;
        group_range(acq, gd_l, gm, &glo, &ghi);
        word_l = (unsigned)bin | ((unsigned)(ghi - (bin << kBinShift)) << 16) |
                 (group_near(acq, gd_l, gm) ? 0x80000000u : 0u);
      }
    };
    if (!WS || warp < W) {
      const int s_begin = n_reg * warp / W;
      const int s_end = n_reg * (warp + 1) / W;
      const int zone_end = zs[warp + 1];
      float* my_stage = stage + warp * kTile;
      auto sink = [&](int r, float v) {
        PAB_CHECK(r >= 0 && r < n_out && (r < zone_end || r - zone_end < kTile));
        if (r < zone_end) row[r] += v;
        else my_stage[r - zone_end] = v;
      };
      int fp = zs[warp];
      int touched = fp - 1;   // highest row any window of this sweep may have written
      // lazy flush: rows below blo are complete; only those whose slots the
      // group's rows [blo, ghi + 7] reuse must go now -- flushed in batches
      // of >= 32 rows when possible
      auto make_room = [&](int blo, int ghi) {
        const int need = ghi + 8 - kTile;
        if (need > fp) {
          const int upto = min(blo, max(need, fp + kWarp));
          flush_rows(tile, lane, fp, min(upto, touched + 1), sink);
          fp = upto;
        }
        touched = max(touched, ghi + 7);
      };
      if (WS) {
        const float fs = (float)acq.f;
        PROF_T(t_loop);
        for (int i = s_begin; i < s_end; ++i) {
          const int sl = i % kRing;
          PROF_T(t_w);
          mbar_wait(&mb_full[warp * kRing + sl], (ring_par >> sl) & 1u);
          PROF_ACC(pw_wait, t_w);
          ring_par ^= 1u << sl;
          const int4 h = slot_h[warp * kRing + sl];
          const float4 ra4 = slot_a[(warp * kRing + sl) * kWarp + lane];
          const float4 rb4 = slot_b[(warp * kRing + sl) * kWarp + lane];
          const int mode = h.w & 3;
          float rc1;
          if (DUAL && mode != 0) rc1 = slot_c[(warp * kRing + sl) * kWarp + lane];
          mbar_arrive(&mb_empty[warp * kRing + sl]);
          if (DUAL && mode != 0) {
            // record (36 B per lane): a = (J0a | jha << 16, J0b | jhb << 16,
            // mfa | mfb << 16 (int16 m-offsets), nsca), b = (pssa, nlaa, nscb, pssb),
            // c = nlab, jh = 0xFFFF: empty; header (Lu | La, blo, ghi, mode | Lb << 16)
            PROF_T(t_r2);
            make_room(h.y, h.z);
            PROF_ACC(pw_room, t_r2);
#ifdef PAB_FWD_PROF
            pw_groups += 2;
            pw_lanes += 2 * (long long)((h.x + 3) & ~3) * 32 + (mode == 2 ? 2 * (long long)(((h.w >> 16) + 3) & ~3) * 32 : 0);
            if (lane == 0) atomicAdd(&g_fwd_prof[mode == 2 ? 14 : 15], 1ull);
#endif
            PROF_T(t_k2);
            const unsigned wa_ = __float_as_uint(ra4.x), wb_ = __float_as_uint(ra4.y);
            const unsigned wm_ = __float_as_uint(ra4.z);
            const float mfa = (float)(int)(short)(wm_ & 0xFFFFu), mfb = (float)((int)wm_ >> 16);
            const int J0a = (int)(wa_ & 0xFFFFu), jha = (wa_ >> 16) == 0xFFFFu ? -1 : (int)(wa_ >> 16);
            const int J0b = (int)(wb_ & 0xFFFFu), jhb = (wb_ >> 16) == 0xFFFFu ? -1 : (int)(wb_ >> 16);
            if (mode == 1) {   // dual walk over the lane's union window
#ifdef PAB_FWD_NOWALK   // tuning builds only: time everything but the walk
              if (false) {
#else
              if (h.x > 0) {
#endif
                const int J0u = jha < 0 ? J0b : (jhb < 0 ? J0a : min(J0a, J0b));
                const DWalk wa = make_dwalk(ra4.w, rb4.x, fs, rb4.y, mfa + (float)((J0u - J0a) * acq.f));
                const DWalk wb = make_dwalk(rb4.z, rb4.w, fs, rc1, mfb + (float)((J0u - J0b) * acq.f));
                rmw_walk_dual(tile, lane, J0u, (h.x + 3) & ~3, max(jha, jhb), fs, wa, wb, dumpq);
              }
            } else {           // the pair's windows lie far apart: two single walks
              const int La = h.x, Lb = h.w >> 16;
              if (La > 0) rmw_walk<false>(tile, lane, J0a, (La + 3) & ~3, jha, mfa, fs,
                                         make_walk(ra4.w, rb4.x, fs, rb4.y, 0.0f), dumpq);
              if (Lb > 0) rmw_walk<false>(tile, lane, J0b, (Lb + 3) & ~3, jhb, mfb, fs,
                                         make_walk(rb4.z, rb4.w, fs, rc1, 0.0f), dumpq);
            }
            __syncwarp();
            PROF_ACC(pw_walk, t_k2);
            continue;
          }
          PROF_T(t_r);
          make_room(h.y, h.z);
          PROF_ACC(pw_room, t_r);
#ifdef PAB_FWD_PROF
          pw_lanes += (h.x > 0) ? (long long)((h.x + 3) & ~3) * 32 : 0;
          pw_groups += 1;
#endif
          PROF_T(t_k);
#ifdef PAB_FWD_NOWALK   // tuning builds only: time everything but the walk
          if (false)
#else
          if (h.x > 0)
#endif
            rmw_walk<MASK>(tile, lane, __float_as_int(ra4.x), (h.x + 3) & ~3, __float_as_int(ra4.y), ra4.z, fs,
                           make_walk(ra4.w, rb4.x, fs, rb4.y, rb4.z), dumpq);
          __syncwarp();
          PROF_ACC(pw_walk, t_k);
        }
        PROF_ADD(13, t_loop);
      } else {
      for (int i0 = s_begin; i0 < s_end; i0 += kWarp) {
        const int nb = min(kWarp, s_end - i0);
        GroupDet gd_l;
        int64_t g_l;
        unsigned word_l;
        batch_geometry(i0, nb, gd_l, g_l, word_l);
        // two groups per trip: their setups (latency-bound chains) are
        // computed side by side, then both walk in order; records of the
        // next two groups are loaded while the current ones are evaluated
        int64_t ga = __shfl_sync(0xffffffffu, g_l, 0), gb = __shfl_sync(0xffffffffu, g_l, min(1, nb - 1));
        BallA Aa = ra[ga * kWarp + lane], Ab = ra[gb * kWarp + lane];
        BallB Ba = rb[ga * kWarp + lane], Bb = rb[gb * kWarp + lane];
        for (int k = 0; k < nb; k += 2) {
          const bool two = k + 1 < nb;
          const int kb = two ? k + 1 : k;
          const GroupDet gda = shfl_gd_fast(gd_l, k), gdb = shfl_gd_fast(gd_l, kb);
          const unsigned worda = __shfl_sync(0xffffffffu, word_l, k), wordb = __shfl_sync(0xffffffffu, word_l, kb);
          const BallA A0 = Aa, A1 = Ab;
          const BallB B0 = Ba, B1 = Bb;
          if (k + 2 < nb) {
            ga = __shfl_sync(0xffffffffu, g_l, k + 2);
            gb = __shfl_sync(0xffffffffu, g_l, min(k + 3, nb - 1));
            Aa = ra[ga * kWarp + lane];
            Ab = ra[gb * kWarp + lane];
            Ba = rb[ga * kWarp + lane];
            Bb = rb[gb * kWarp + lane];
          }
          const int bloa = (int)(worda & 0xFFFFu) << kBinShift, blob = (int)(wordb & 0xFFFFu) << kBinShift;
          const int ghia = bloa + (int)((worda >> 16) & 0x7FFFu), ghib = blob + (int)((wordb >> 16) & 0x7FFFu);
          unsigned long long ops_b = 0;
          const PairSetup pa = pair_setup<DIR>(acq, gda, dd, A0, B0, my_ops, bloa);
          const PairSetup pb = pair_setup<DIR>(acq, gdb, dd, A1, B1, ops_b, blob);
          if (two) my_ops += ops_b;
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            if (h == 1 && !two) break;
            const int blo = h ? blob : bloa, ghi = h ? ghib : ghia;
            make_room(blo, ghi);
            pair_walk<MASK>(tile, lane, acq, h ? pb : pa, (int)((h ? wordb : worda) >> 31), my_ops, blo, dumpq);
            __syncwarp();
          }
        }
      }
      }
      PROF_T(t_fl);
      if (s_begin < s_end) flush_rows(tile, lane, fp, min(n_out, touched + 1), sink);
      // rows past the signal end (clipped windows' overrun) are never
      // flushed: clear the tile for the next chunk / the linear passes
      for (int i = lane; i < kTile * kWarp / 4; i += kWarp)
        reinterpret_cast<float4*>(tile)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
      __syncwarp();
      PROF_ADD(6, t_fl);
    } else {
      // producer for walker w: pair setups, two side by side, published in
      // slice order through the ring
      const int w = warp - W;
      const int s_begin = n_reg * w / W;
      const int s_end = n_reg * (w + 1) / W;
      const float fs = (float)acq.f;
      auto publish = [&](int i, const PairSetup& p, int blo, int ghi) {
        const int sl = i % kRing;
        const bool empty_u = p.jlo > p.jhi;
        const float Ak = empty_u ? 0.0f : p.Ak;
        const float sg = Ak < 0.0f ? -1.0f : 1.0f;
        const float nla = -__log2f(fabsf(Ak));   // +inf for Ak = 0
        const float mf = (float)(p.J0 * acq.f - p.kc);
        PROF_T(t_pw);
        mbar_wait_backoff(&mb_empty[w * kRing + sl], (ring_par >> sl) & 1u);
        PROF_ACC(pp_pub, t_pw);
        ring_par ^= 1u << sl;
        slot_a[(w * kRing + sl) * kWarp + lane] =
            make_float4(__int_as_float(p.J0), __int_as_float(empty_u ? -1 : p.jhi), mf, -p.sc * sg);
        slot_b[(w * kRing + sl) * kWarp + lane] = make_float4(p.phi * p.sc * sg, nla, p.qmax + nla, 0.0f);
        if (lane == 0) slot_h[w * kRing + sl] = make_int4(p.L, blo, ghi, 0);
        mbar_arrive(&mb_full[w * kRing + sl]);
      };
      (void)fs;
      if constexpr (DUAL) {
        // entries are single lane groups (32 lanes, one ball each: the
        // single walk) or dual pairs of groups (lanes 0-15 take balls
        // (2l, 2l+1) of the first group, lanes 16-31 those of the second)
        // dual entry: lane l walks the balls at positions 2l, 2l+1 of the
        // unit's projection order for the detector direction's cell (ball
        // ids 0-31 first group, 32-63 second: record g0 * 32 + id)
        const int64_t n_units = (n_groups + 1) / 2;
        auto load_ids = [&](int64_t g0, int cell) -> unsigned {
          PAB_CHECK(cell >= 0 && cell < kPairDirs && (g0 >> 1) < n_units && (g0 & 1) == 0);
          return reinterpret_cast<const unsigned short*>(ptab + ((size_t)cell * n_units + (g0 >> 1)) * 64)[lane];
        };
        auto load_recs = [&](int64_t g0, bool pair, unsigned ids, BallA& A0, BallA& A1, BallB& B0, BallB& B1) {
          const int64_t bi = pair ? g0 * kWarp + (ids & 0xFFu) : g0 * kWarp + lane;
          PAB_CHECK(bi < n_groups * kWarp && (!pair || (ids & 0xFFu) < 64u && (ids >> 8) < 64u &&
                                              g0 + 1 < n_groups));
          A0 = ra[bi];
          B0 = rb[bi];
          if (pair) {
            A1 = ra[g0 * kWarp + (ids >> 8)];
            B1 = rb[g0 * kWarp + (ids >> 8)];
          }
        };
        auto publish = [&](int i, int mode, int x, int blo, int ghi, int hw, float4 va, float4 vb, float vc) {
          const int sl = i % kRing;
          PROF_T(t_pw);
          mbar_wait_backoff(&mb_empty[w * kRing + sl], (ring_par >> sl) & 1u);
          PROF_ACC(pp_pub, t_pw);
          ring_par ^= 1u << sl;
          const int ix = (w * kRing + sl) * kWarp + lane;
          slot_a[ix] = va;
          slot_b[ix] = vb;
          if (mode != 0) slot_c[ix] = vc;
          if (lane == 0) slot_h[w * kRing + sl] = make_int4(x, blo, ghi, mode | (hw << 16));
          mbar_arrive(&mb_full[w * kRing + sl]);
        };
        for (int i0 = s_begin; i0 < s_end; i0 += kWarp) {
          const int nb = min(kWarp, s_end - i0);
          GroupDet gdA_l = empty_gd(), gdB_l = empty_gd();
          int64_t g_l = 0;
          unsigned word_l = 0;
          int cell_l = 0;
          PROF_T(t_g);
          if (lane < nb) {
            const int e = sorted[i0 + lane];
            const int slot = e & 0x7FFF;
            const bool pair = (e >> 15) != 0;
            g_l = cg0 + slot;
            const int bin = gbin[slot];
            const GroupMeta gmA = gmeta[g_l];
            gdA_l = group_det(gmA, det.px, det.py, det.pz, acq);
            int lo, hi;
            group_range(acq, gdA_l, gmA, &lo, &hi);
            int ghi = hi;
            if (pair) {
              const GroupMeta gmB = gmeta[g_l + 1];
              gdB_l = group_det(gmB, det.px, det.py, det.pz, acq);
              group_range(acq, gdB_l, gmB, &lo, &hi);
              ghi = max(ghi, hi);
            }
            word_l = (unsigned)bin | ((unsigned)(ghi - (bin << kBinShift)) << 16) | (pair ? 0x80000000u : 0u);
            cell_l = pair ? pair_cell(gdA_l.Sx, gdA_l.Sy, gdA_l.Sz) : 0;
          }
          __syncwarp();   // the previous batch's table reads are done
          {
            float4* const pt = reinterpret_cast<float4*>(hist) + (size_t)(w * kWarp + lane) * 2;
            pt[0] = make_float4(gdB_l.Sx, gdB_l.Sy, gdB_l.Sz, gdB_l.Sn);
            // (.w: the entry's chunk slot | direction cell << 16 | pair << 31)
            pt[1] = make_float4(gdB_l.isn, gdB_l.phg, __int_as_float(gdB_l.kg),
                                __uint_as_float((unsigned)(g_l - cg0) | ((unsigned)cell_l << 16) |
                                                (word_l & 0x80000000u)));
            float4* const pa = reinterpret_cast<float4*>(hist) + (size_t)((W + w) * kWarp + lane) * 2;
            pa[0] = make_float4(gdA_l.Sx, gdA_l.Sy, gdA_l.Sz, gdA_l.Sn);
            pa[1] = make_float4(gdA_l.isn, gdA_l.phg, __int_as_float(gdA_l.kg), __uint_as_float(word_l));
          }
          __syncwarp();
          PROF_ACC(pp_geo, t_g);
          // two-stage prefetch: pairing ids two entries ahead, records one ahead
          auto entry = [&](int k, int64_t& g0, bool& pair, int& cell) {   // from the table (no shuffles)
            const unsigned v =
                __float_as_uint((reinterpret_cast<const float4*>(hist) + (size_t)(w * kWarp + k) * 2 + 1)->w);
            g0 = cg0 + (int64_t)(v & 0x7FFFu);
            cell = (int)((v >> 16) & 63u);
            pair = (v >> 31) != 0;
          };
          int64_t gn, gn2 = 0;
          bool pn, pn2 = false;
          int cn_, cn2;
          entry(0, gn, pn, cn_);
          unsigned idn = pn ? load_ids(gn, cn_) : 0u, idn2 = 0u;
          if (nb > 1) {
            entry(1, gn2, pn2, cn2);
            if (pn2) idn2 = load_ids(gn2, cn2);
          }
          BallA An0, An1;
          BallB Bn0, Bn1;
          load_recs(gn, pn, idn, An0, An1, Bn0, Bn1);
          for (int k = 0; k < nb; ++k) {
            const BallA A0 = An0, A1 = An1;
            const BallB B0 = Bn0, B1 = Bn1;
            const bool pair = pn;
            const unsigned ids = idn;
            if (k + 1 < nb) {   // next entry's records in flight during this setup
              gn = gn2;
              pn = pn2;
              idn = idn2;
              load_recs(gn, pn, idn, An0, An1, Bn0, Bn1);
              if (k + 2 < nb) {
                entry(k + 2, gn2, pn2, cn2);
                idn2 = pn2 ? load_ids(gn2, cn2) : 0u;
              }
            }
            GroupDet gA;
            unsigned word;
            {
              const float4* const pa = reinterpret_cast<const float4*>(hist) + (size_t)((W + w) * kWarp + k) * 2;
              const float4 a = pa[0], b = pa[1];
              gA.Sx = a.x; gA.Sy = a.y; gA.Sz = a.z; gA.Sn = a.w;
              gA.isn = b.x; gA.phg = b.y; gA.kg = __float_as_int(b.z);
              gA.slow = 0;
              word = __float_as_uint(b.w);
            }
            const int blo = (int)(word & 0xFFFFu) << kBinShift;
            const int ghi = blo + (int)((word >> 16) & 0x7FFFu);
            PROF_T(t_s);
            if (!pair) {   // single group: one ball per lane
              const PairSetup p = pair_setup<DIR>(acq, gA, dd, A0, B0, my_ops, blo);
              const bool empty_u = p.jlo > p.jhi;
              const float Ak = empty_u ? 0.0f : p.Ak;
              const float sg = Ak < 0.0f ? -1.0f : 1.0f;
              const float nla = -__log2f(fabsf(Ak));   // +inf for Ak = 0
#ifdef PAB_FWD_PROF
              pp_setup += clock64() - t_s;
#endif
              publish(i0 + k, 0, p.L, blo, ghi, 0,
                      make_float4(__int_as_float(p.J0), __int_as_float(empty_u ? -1 : p.jhi),
                                  (float)(p.J0 * acq.f - p.kc), -p.sc * sg),
                      make_float4(p.phi * p.sc * sg, nla, p.qmax + nla, 0.0f), 0.0f);
              continue;
            }
            GroupDet gB;
            {
              const float4* const pt = reinterpret_cast<const float4*>(hist) + (size_t)(w * kWarp + k) * 2;
              const float4 a = pt[0], b = pt[1];
              gB.Sx = a.x; gB.Sy = a.y; gB.Sz = a.z; gB.Sn = a.w;
              gB.isn = b.x; gB.phg = b.y; gB.kg = __float_as_int(b.z);
              gB.slow = 0;
            }
            const PairSetup pa = pair_setup<DIR, false>(acq, (ids & 0xE0u) ? gB : gA, dd, A0, B0, my_ops, blo);
            const PairSetup pb = pair_setup<DIR, false>(acq, (ids & 0xE000u) ? gB : gA, dd, A1, B1, my_ops, blo);
            // walk parameters per ball (sgn(Ak) folded into y; empty balls: y = 0, G = 0)
            auto params = [&](const PairSetup& p, bool e, int& J0, int& jh, float& mf, float& nsc, float& pss,
                              float& nla) {
              J0 = e ? blo : p.J0;
              jh = e ? -1 : p.jhi;
              mf = (float)(J0 * acq.f - p.kc);
              const float sg = p.Ak < 0.0f ? -1.0f : 1.0f;
              nsc = e ? 0.0f : -p.sc * sg;
              pss = e ? 0.0f : p.phi * p.sc * sg;
              nla = e ? __int_as_float(0x7f800000) : -__log2f(fabsf(p.Ak));
            };
            const bool ea = pa.jlo > pa.jhi, eb = pb.jlo > pb.jhi;
            int J0a, jha, J0b, jhb;
            float mfa, nsca, pssa, nlaa, mfb, nscb, pssb, nlab;
            params(pa, ea, J0a, jha, mfa, nsca, pssa, nlaa);
            params(pb, eb, J0b, jhb, mfb, nscb, pssb, nlab);
            const int J0u = ea ? J0b : (eb ? J0a : min(J0a, J0b));
            const int lim = max(jha, jhb);
            // the recurrence's range guard: |y| <= kDualMaxY on every live
            // walked sample (|y| <= sc (|J f - kc| + 1/2), J in [J0u, lim + 7])
            // and |dl| = f sc <= kDualMaxDl, folded into one test per ball
            auto yok = [&](bool e, const PairSetup& p) {
              const int dm = max(p.kc - J0u * acq.f, (lim + 7) * acq.f - p.kc);
              return e || p.sc * fmaxf(fs * (1.0f / kDualMaxDl), (float)dm * (1.0f / kDualMaxY) + 0.5f / kDualMaxY) <= 1.0f;
            };
            const bool ok = __all_sync(0xffffffffu, yok(ea, pa) && yok(eb, pb));
            const int Lu = __reduce_max_sync(0xffffffffu, (ea && eb) ? 0 : lim - J0u + 1);
            const int La = ok ? 0 : __reduce_max_sync(0xffffffffu, ea ? 0 : jha - J0a + 1);
            const int Lb = ok ? 0 : __reduce_max_sync(0xffffffffu, eb ? 0 : jhb - J0b + 1);
#ifdef PAB_FWD_PROF
            pp_setup += clock64() - t_s;
#endif
            // m-offsets as int16 (exact small integers: the unit fits the tile;
            // an empty ball's is unused)
            const int mia = min(max((int)mfa, -32768), 32767), mib = min(max((int)mfb, -32768), 32767);
            PAB_CHECK(ea || (float)mia == mfa);
            PAB_CHECK(eb || (float)mib == mfb);
            publish(i0 + k, ok ? 1 : 2, ok ? Lu : La, blo, ghi, ok ? 0 : Lb,
                    make_float4(__uint_as_float((unsigned)J0a | ((unsigned)jha << 16)),
                                __uint_as_float((unsigned)J0b | ((unsigned)jhb << 16)),
                                __uint_as_float(((unsigned)mia & 0xFFFFu) | ((unsigned)mib << 16)), nsca),
                    make_float4(pssa, nlaa, nscb, pssb), nlab);
          }
        }
      } else
      for (int i0 = s_begin; i0 < s_end; i0 += kWarp) {
        const int nb = min(kWarp, s_end - i0);
        GroupDet gd_l;
        int64_t g_l;
        unsigned word_l;
        PROF_T(t_g);
        batch_geometry(i0, nb, gd_l, g_l, word_l);
        PROF_ACC(pp_geo, t_g);
        // the batch in a shared-memory table (the histogram's space during
        // the sweep): geometry, word and slot by broadcast LDS.128, no shuffles
        __syncwarp();
        {
          float4* const pt = reinterpret_cast<float4*>(hist) + (size_t)(w * kWarp + lane) * 3;
          pt[0] = make_float4(gd_l.Sx, gd_l.Sy, gd_l.Sz, gd_l.Sn);
          pt[1] = make_float4(gd_l.isn, gd_l.phg, __int_as_float(gd_l.kg), __uint_as_float(word_l));
          pt[2] = make_float4(__int_as_float((int)(g_l - cg0)), 0.0f, 0.0f, 0.0f);
        }
        __syncwarp();
        auto tgd = [&](int k, unsigned& word) {
          const float4* const pt = reinterpret_cast<const float4*>(hist) + (size_t)(w * kWarp + k) * 3;
          const float4 a = pt[0], b = pt[1];
          GroupDet gd;
          gd.Sx = a.x; gd.Sy = a.y; gd.Sz = a.z; gd.Sn = a.w;
          gd.isn = b.x; gd.phg = b.y; gd.kg = __float_as_int(b.z);
          gd.slow = 0;
          word = __float_as_uint(b.w);
          return gd;
        };
        auto tg = [&](int k) -> int64_t {
          return cg0 + __float_as_int((reinterpret_cast<const float4*>(hist) + (size_t)(w * kWarp + k) * 3 + 2)->x);
        };
        int64_t ga = tg(0), gb = tg(min(1, nb - 1));
        BallA Aa = ra[ga * kWarp + lane], Ab = ra[gb * kWarp + lane];
        BallB Ba = rb[ga * kWarp + lane], Bb = rb[gb * kWarp + lane];
        for (int k = 0; k < nb; k += 2) {
          const bool two = k + 1 < nb;
          const int kb = two ? k + 1 : k;
          unsigned worda, wordb;
          const GroupDet gda = tgd(k, worda), gdb = tgd(kb, wordb);
          const BallA A0 = Aa, A1 = Ab;
          const BallB B0 = Ba, B1 = Bb;
          if (k + 2 < nb) {
            ga = tg(k + 2);
            gb = tg(min(k + 3, nb - 1));
            Aa = ra[ga * kWarp + lane];
            Ab = ra[gb * kWarp + lane];
            Ba = rb[ga * kWarp + lane];
            Bb = rb[gb * kWarp + lane];
          }
          const int bloa = (int)(worda & 0xFFFFu) << kBinShift, blob = (int)(wordb & 0xFFFFu) << kBinShift;
          const int ghia = bloa + (int)((worda >> 16) & 0x7FFFu), ghib = blob + (int)((wordb >> 16) & 0x7FFFu);
          unsigned long long ops_b = 0;
          PROF_T(t_s);
#ifdef PAB_FWD_NOSETUP   // tuning builds only: publish without computing setups
          PairSetup pa{}, pb{};
#else
          const PairSetup pa = pair_setup<DIR>(acq, gda, dd, A0, B0, my_ops, bloa);
          const PairSetup pb = pair_setup<DIR>(acq, gdb, dd, A1, B1, ops_b, blob);
#endif
#ifdef PAB_FWD_PROF
          pp_setup += clock64() - t_s;   // includes the record loads' latency
#endif
          publish(i0 + k, pa, bloa, ghia);
          if (two) {
            my_ops += ops_b;
            publish(i0 + k + 1, pb, blob, ghib);
          }
        }
      }
    }
    PROF_ADD(pslot + 3, t_d);
    PROF_T(t_e);
    __syncthreads();
    PROF_ADD(pslot + 4, t_e);
    PROF_T(t_e2);

    // ---- E: overlap rows, merged in warp order ----
    for (int w = 0; w + 1 < W; ++w) {
      const int r0 = zs[w + 1];
      for (int i = tid; i < kTile && r0 + i < n_out; i += nthr) {
        row[r0 + i] += stage[w * kTile + i];
        stage[w * kTile + i] = 0.0f;
      }
      __syncthreads();
    }

    PROF_ADD(pslot + 5, t_e2);
    // ---- F: groups wider than the tile (bin n_bins) are left out of the
    // sweep; forward_wide_kernel adds them afterwards ----
  }
#ifdef PAB_FWD_PROF
  if (lane == 0) {
    atomicAdd(&g_fwd_prof[8], (unsigned long long)pw_wait);
    atomicAdd(&g_fwd_prof[9], (unsigned long long)pw_room);
    atomicAdd(&g_fwd_prof[10], (unsigned long long)pw_walk);
    atomicAdd(&g_fwd_prof[11], (unsigned long long)pw_lanes);
    atomicAdd(&g_fwd_prof[12], (unsigned long long)pw_groups);
    atomicAdd(&g_fwd_prof[24], (unsigned long long)pp_setup);
    atomicAdd(&g_fwd_prof[25], (unsigned long long)pp_pub);
    atomicAdd(&g_fwd_prof[26], (unsigned long long)pp_geo);
  }
#endif

  if (SROW) {
    float* out = partial_rows + ((size_t)part * n_det + j) * (size_t)n_out;
    for (int i = tid; i < n_out; i += nthr) out[i] = row[i];
  }
  if (tid == 0) wide_out[0] = wide_count;   // > wide_cap: forward_wide_kernel finds them again
  for (int o = 16; o > 0; o >>= 1) {
    my_ops += __shfl_xor_sync(0xffffffffu, my_ops, o);
    coinc |= __shfl_xor_sync(0xffffffffu, coinc, o);
  }
  if (lane == 0) {
    if (my_ops) atomicAdd(ops_total, my_ops);
    if (coinc) atomicOr(status, kStatusCoincident);
  }
}

// Sum partitions in order, subtract the supervision (res = sim - real, or
// res = -real for the zero-pressure filter probe), per-row FP64 loss.
__global__ void residual_kernel(const float* __restrict__ partial_rows, int parts, int n_det, int n_out,
                                const float* __restrict__ real, float* __restrict__ out,
                                double* __restrict__ loss_rows, bool vec) {
  const int j = blockIdx.x;
  double acc = 0.0;
  int k0 = 0;
  if (vec) {   // 16-byte rows: float4 streams, all loads of a step in flight together
    const int n4 = n_out >> 2;
    const size_t row4 = (size_t)j * n4, plane4 = (size_t)n_det * n4;
    const float4* pr = reinterpret_cast<const float4*>(partial_rows);
    const float4* re = reinterpret_cast<const float4*>(real);
    float4* o4 = reinterpret_cast<float4*>(out);
    for (int k = threadIdx.x; k < n4; k += blockDim.x) {
      float4 v = pr[row4 + k];
      for (int p = 1; p < parts; ++p) {
        const float4 w = pr[p * plane4 + row4 + k];
        v.x += w.x; v.y += w.y; v.z += w.z; v.w += w.w;
      }
      if (real != nullptr) {
        const float4 t = re[row4 + k];
        v.x -= t.x; v.y -= t.y; v.z -= t.z; v.w -= t.w;
        acc += (double)v.x * (double)v.x + (double)v.y * (double)v.y + (double)v.z * (double)v.z +
               (double)v.w * (double)v.w;
      }
      o4[row4 + k] = v;
    }
    k0 = n_out;
  }
  for (int k = k0 + threadIdx.x; k < n_out; k += blockDim.x) {
    float s = 0.0f;
    for (int p = 0; p < parts; ++p) s += partial_rows[((size_t)p * n_det + j) * n_out + k];
    if (real != nullptr) {
      const float r = s - real[(size_t)j * n_out + k];
      out[(size_t)j * n_out + k] = r;
      acc += (double)r * (double)r;
    } else {
      out[(size_t)j * n_out + k] = s;
    }
  }
  if (loss_rows == nullptr) return;
  __shared__ double red[32];
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red[w];
    loss_rows[j] = s;
  }
}

// Pure decimation of supervision rows (reference radiator.py:382-390).
__global__ void decimate_kernel(const float* __restrict__ src, int n_rows, int n_in, int f, int n_out,
                                float* __restrict__ dst) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (int64_t)n_rows * n_out) return;
  const int64_t r = i / n_out, k = i % n_out;
  dst[i] = src[r * n_in + k * f];
}


size_t forward_smem(int n_out, int warps, bool srow, bool dual) {
  const size_t n_bins = (size_t)((n_out + (1 << kBinShift) - 1) >> kBinShift);
  const size_t row_bytes = srow ? (size_t)((n_out + 3) & ~3) * 4 : 0;
  const size_t rec_bytes = dual ? 36 : 32;   // hand-off record per lane and ring slot
  const size_t ring = kWS ? 16 + (size_t)warps * kRing * (rec_bytes * kWarp + 16 + 2 * 8) : 0;
  const size_t units = kChunk;
  return row_bytes + ((size_t)warps * kTile * kWarp + kDumpFloats) * 4 + (size_t)warps * kTile * 4 +
         (size_t)hist_ints((int)n_bins, warps, dual) * 4 + (size_t)(warps + 1) * 4 + 16 + 2 * units * 2 + 16 + ring;
}

}  // namespace pab

using namespace pab;

extern "C" {

// The row stays in shared memory while two CTAs still fit on an SM
// (2 x (smem + 1 KB reserve) <= 228 KB); longer records keep it in L2.
static size_t smem_both(int n_out, int warps, bool srow) {   // the larger of the single / dual layouts
  return std::max(forward_smem(n_out, warps, srow, false), forward_smem(n_out, warps, srow, kWS && kDual));
}
static bool row_in_smem(int n_out, int warps) { return smem_both(n_out, warps, true) <= 113 * 1024; }

size_t pab_forward_smem_bytes(int n_out, int warps, int tile_rows) {
  (void)tile_rows;
  return smem_both(n_out, warps, row_in_smem(n_out, warps));
}

int pab_forward(const void* rec_a, const void* rec_b, const void* group_meta, const unsigned char* pair_table,
                int64_t n_groups,
                const double* det_pos, const double* det_aux, int n_det, double v, double t0, double dt,
                int f, int n_out, double cutoff, int dir_kind, double dir_param, int groups_per_cell,
                int partitions, int warps, int tile_rows, float* partial_rows, int* wide_list, int wide_cap,
                unsigned long long* ops_total, int* status, void* stream) {
  (void)groups_per_cell;
  (void)tile_rows;
  if (n_det <= 0 || n_out <= 0) return 0;
  if (f < 1 || partitions < 1 || warps < 1 || warps > kMaxWarps) return 1;
  if (!rec_a || !rec_b || !group_meta || !det_pos || !det_aux || !partial_rows || !wide_list || wide_cap < 0 ||
      !ops_total || !status)
    return 1;
  if ((int64_t)n_out * f > kMaxRecordSamples) return 1;   // sample indices stay in the magic-rounding range
  const Acq acq = make_acq(v, t0, dt, f, n_out, cutoff, dir_kind, dir_param);
  // per-sample truncation test only where the walk's overrun could matter
  const bool mask = cutoff < kUnmaskedCutoff;
  // dual walk: needs the pairing table, 16-bit row fields and two CTAs per SM
  const bool dual = kWS && kDual && !mask && pair_table != nullptr && n_out < 65535 &&
                    2 * (forward_smem(n_out, warps, row_in_smem(n_out, warps), true) + 1024) <= 228 * 1024;
  int64_t per_part = (n_groups + partitions - 1) / partitions;
  if (dual) per_part += per_part & 1;   // dual sort units (group pairs) never straddle partitions
  const bool srow = row_in_smem(n_out, warps);
  const size_t smem = forward_smem(n_out, warps, srow, dual);
  if (smem > 227 * 1024) return 1;
  if (dir_kind < 0 || dir_kind > 2) return 1;
  dim3 grid((unsigned)n_det, (unsigned)partitions);
  auto launch = [&](auto kernel) {
    cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    kernel<<<grid, warps * kWarp * (kWS ? 2 : 1), smem, (cudaStream_t)stream>>>(
        (const BallA*)rec_a, (const BallB*)rec_b, (const GroupMeta*)group_meta, pair_table, n_groups, det_pos, det_aux,
        n_det, acq, per_part, partial_rows, wide_list, wide_cap, ops_total, status);
  };
  auto by_row = [&](auto k_srow, auto k_grow) { srow ? launch(k_srow) : launch(k_grow); };
  auto by_mask = [&](auto km_s, auto km_g, auto ku_s, auto ku_g, auto kd_s, auto kd_g) {
    mask ? by_row(km_s, km_g) : (dual ? by_row(kd_s, kd_g) : by_row(ku_s, ku_g));
  };
#define PAB_FWD_VARIANTS(D) \
  by_mask(forward_kernel<D, true, true, kWS, false>, forward_kernel<D, true, false, kWS, false>,   \
          forward_kernel<D, false, true, kWS, false>, forward_kernel<D, false, false, kWS, false>, \
          forward_kernel<D, false, true, kWS, kWS && kDual>, forward_kernel<D, false, false, kWS, kWS && kDual>)
  if (dir_kind == kDirNone) PAB_FWD_VARIANTS(kDirNone);
  else if (dir_kind == kDirCosPower && dir_param == 2.0) PAB_FWD_VARIANTS(kDirCos2);
  else if (dir_kind == kDirCosPower) PAB_FWD_VARIANTS(kDirCosPower);
  else PAB_FWD_VARIANTS(kDirElement);
#undef PAB_FWD_VARIANTS
  // groups wider than the tile, added to the same partition rows afterwards
  const size_t wsmem = (size_t)kWideWarps * kTileAlloc * kWarp * sizeof(float) + 3 * (size_t)kWideChunk;
  auto launch_wide = [&](auto kernel) {
    cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)wsmem);
    kernel<<<grid, kWideWarps * kWarp, wsmem, (cudaStream_t)stream>>>(
        (const BallA*)rec_a, (const BallB*)rec_b, (const GroupMeta*)group_meta, n_groups, det_pos, det_aux, n_det,
        acq, per_part, partial_rows, wide_list, wide_cap, ops_total, status);
  };
#define PAB_FWD_WIDE(D) mask ? launch_wide(forward_wide_kernel<D, true>) : launch_wide(forward_wide_kernel<D, false>)
  if (dir_kind == kDirNone) PAB_FWD_WIDE(kDirNone);
  else if (dir_kind == kDirCosPower && dir_param == 2.0) PAB_FWD_WIDE(kDirCos2);
  else if (dir_kind == kDirCosPower) PAB_FWD_WIDE(kDirCosPower);
  else PAB_FWD_WIDE(kDirElement);
#undef PAB_FWD_WIDE
  return cudaGetLastError() == cudaSuccess ? 0 : 4;
}

int pab_residual(const float* partial_rows, int partitions, int n_det, int n_out, const float* real,
                 float* out, double* loss_rows, void* stream) {
  if (n_det <= 0 || n_out <= 0) return 0;
  if (!partial_rows || !out || partitions < 1) return 1;
  auto a16 = [](const void* q) { return ((uintptr_t)q & 15) == 0; };
  const bool vec = (n_out & 3) == 0 && a16(partial_rows) && a16(out) && (real == nullptr || a16(real));
  residual_kernel<<<n_det, 256, 0, (cudaStream_t)stream>>>(partial_rows, partitions, n_det, n_out, real,
                                                           out, loss_rows, vec);
  return cudaGetLastError() == cudaSuccess ? 0 : 4;
}

int pab_decimate(const float* src, int n_rows, int n_in, int f, float* dst, void* stream) {
  if (f < 1 || n_rows < 0 || n_in < 0) return 1;
  const int n_out = (n_in + f - 1) / f;
  const int64_t total = (int64_t)n_rows * n_out;
  if (total == 0) return 0;
  if (!src || !dst) return 1;
  decimate_kernel<<<(unsigned)((total + 255) / 256), 256, 0, (cudaStream_t)stream>>>(src, n_rows, n_in, f,
                                                                                    n_out, dst);
  return cudaGetLastError() == cudaSuccess ? 0 : 4;
}

}  // extern "C"

#ifdef PAB_WALK_BENCH
// Tuning builds only: the forward's window walk in isolation (no setup, no
// flush), `reps` walks of L samples per warp on its own tile, 4 warps per
// CTA, 2 CTAs per SM -- cycles per 16-sample trip vs the XU bound.
namespace pab {
__global__ void __launch_bounds__(128, 2) walk_bench_kernel(int reps, int L, float* out) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  float* tile = reinterpret_cast<float*>(smem_raw) + (threadIdx.x >> 5) * kTileAlloc * kWarp;
  const int lane = threadIdx.x & 31;
  for (int i = lane; i < kTileAlloc * kWarp; i += 32) tile[i] = 0.0f;
  __syncwarp();
  float sc = 0.3f + 0.001f * lane, ps = 0.1f * lane;
  for (int r = 0; r < reps; ++r) {
    const int J0 = (r * 8 + lane * 8) % kTile;
    rmw_uniform<false>(tile, lane, J0 & ~7, L, 1 << 30, (float)(-L / 2), 1.0f, sc, ps, 1.0f + 0.01f * lane, 30.0f);
    __syncwarp();
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = tile[lane * 4];
}
// Two balls per lane sharing each read-modify-write (the dual-walk
// hypothesis): per 8-sample block, both balls' terms are added in registers.
__global__ void __launch_bounds__(128, 2) walk_bench_dual_kernel(int reps, int L, float* out) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  float* tile = reinterpret_cast<float*>(smem_raw) + (threadIdx.x >> 5) * kTileAlloc * kWarp;
  const int lane = threadIdx.x & 31;
  for (int i = lane; i < kTileAlloc * kWarp; i += 32) tile[i] = 0.0f;
  __syncwarp();
  const float sc = 0.3f + 0.001f * lane, ps = 0.1f * lane;
  const Walk wa = make_walk(-sc, ps, 1.0f, -__log2f(1.0f + 0.01f * lane), 30.0f);
  const Walk wb = make_walk(-sc * 1.02f, ps + 0.05f, 1.0f, -__log2f(1.0f + 0.02f * lane), 30.0f);
  float4* const T = reinterpret_cast<float4*>(tile) + lane;
  for (int r = 0; r < reps; ++r) {
    const int J0 = ((r * 8 + lane * 8) % kTile) & ~7;
    int q = J0 >> 2;
    float mfa = (float)(-L / 2), mfb = mfa + 2.0f;
#pragma unroll 1
    for (int nb = L >> 3; nb >= 2; nb -= 2) {
      int qq[2];
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        qq[k] = q;
        q += 2;
        if (q == kTile / 4) q = 0;
      }
      float4 o[2][2];
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        o[k][0] = T[qq[k] * kWarp];
        o[k][1] = T[(qq[k] + 1) * kWarp];
      }
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const float2 ma = make_float2(mfa + 8.0f * k, mfa + 8.0f * k), mb = make_float2(mfb + 8.0f * k, mfb + 8.0f * k);
        o[k][0] = rmw4(o[k][0], ma, wa.c0, wa.c1, wa, rmw_pair<false>);
        o[k][1] = rmw4(o[k][1], ma, wa.c2, wa.c3, wa, rmw_pair<false>);
        o[k][0] = rmw4(o[k][0], mb, wb.c0, wb.c1, wb, rmw_pair<false>);
        o[k][1] = rmw4(o[k][1], mb, wb.c2, wb.c3, wb, rmw_pair<false>);
      }
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        T[qq[k] * kWarp] = o[k][0];
        T[(qq[k] + 1) * kWarp] = o[k][1];
      }
      mfa += 16.0f;
      mfb += 16.0f;
    }
    __syncwarp();
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = tile[lane * 4];
}
// The production dual walk (two balls per lane, ratio recurrence).
__global__ void __launch_bounds__(128, 2) walk_bench_dualrec_kernel(int reps, int L, float* out) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  float* tile = reinterpret_cast<float*>(smem_raw) + (threadIdx.x >> 5) * kTileAlloc * kWarp;
  const int lane = threadIdx.x & 31;
  for (int i = lane; i < kTileAlloc * kWarp; i += 32) tile[i] = 0.0f;
  __syncwarp();
  const float sc = 0.3f + 0.001f * lane, ps = 0.1f * lane;
  for (int r = 0; r < reps; ++r) {
    const int J0 = ((r * 8 + lane * 8) % kTile) & ~7;
    const DWalk wa = make_dwalk(-sc, ps, 1.0f, -__log2f(1.0f + 0.01f * lane), (float)(-L / 2));
    const DWalk wb = make_dwalk(-sc * 1.02f, ps + 0.05f, 1.0f, -__log2f(1.0f + 0.02f * lane), (float)(-L / 2 + 2));
    rmw_walk_dual(tile, lane, J0, L, 1 << 30, 1.0f, wa, wb);
    __syncwarp();
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = tile[lane * 4];
}
}  // namespace pab
extern "C" int pab_bench_walk_dual(int blocks, int reps, int L, float* out, float* ms) {
  const size_t smem = 4 * kTileAlloc * kWarp * sizeof(float);
  cudaFuncSetAttribute(walk_bench_dual_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  walk_bench_dual_kernel<<<blocks, 128, smem>>>(reps, L, out);
  cudaEventRecord(a);
  walk_bench_dual_kernel<<<blocks, 128, smem>>>(reps, L, out);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  cudaEventElapsedTime(ms, a, b);
  return cudaGetLastError() == cudaSuccess ? 0 : 4;
}
extern "C" int pab_bench_walk_dualrec(int blocks, int reps, int L, float* out, float* ms) {
  const size_t smem = 4 * kTileAlloc * kWarp * sizeof(float);
  cudaFuncSetAttribute(walk_bench_dualrec_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  walk_bench_dualrec_kernel<<<blocks, 128, smem>>>(reps, L, out);
  cudaEventRecord(a);
  walk_bench_dualrec_kernel<<<blocks, 128, smem>>>(reps, L, out);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  cudaEventElapsedTime(ms, a, b);
  return cudaGetLastError() == cudaSuccess ? 0 : 4;
}
extern "C" int pab_bench_walk(int blocks, int reps, int L, float* out, float* ms) {
  const size_t smem = 4 * kTileAlloc * kWarp * sizeof(float);
  cudaFuncSetAttribute(walk_bench_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  walk_bench_kernel<<<blocks, 128, smem>>>(reps, L, out);
  cudaEventRecord(a);
  walk_bench_kernel<<<blocks, 128, smem>>>(reps, L, out);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  cudaEventElapsedTime(ms, a, b);
  return cudaGetLastError() == cudaSuccess ? 0 : 4;
}
#endif

#ifdef PAB_FWD_PROF
extern "C" int pab_fwd_prof(unsigned long long* out /*[32]*/, int reset) {
  cudaMemcpyFromSymbol(out, pab::g_fwd_prof, sizeof(unsigned long long) * 32);
  if (reset) {
    unsigned long long z[32] = {};
    cudaMemcpyToSymbol(pab::g_fwd_prof, z, sizeof(z));
  }
  return cudaGetLastError() == cudaSuccess ? 0 : 4;
}
#endif
