// Shared device code for the SlingBAG Pro forward/adjoint kernels (sm_100a).
//
// Physics (reference radiator.py:1-12, 157-287): a ball (position r_b, peak
// pressure p0, Gaussian radius a0) seen from a detector at distance d gives
//   s(t) = (p0 D / 2d) [u- G(u-) + u+ G(u+)],  u-+ = d -+ v t,  G = exp(-u^2/2a0^2)
// evaluated only where |u| <= cutoff * a0, on sample k of the full-rate grid
// (t = t0 + k dt); on an f-decimated grid sample J sits at k = J f.
//
// Numerics: per-(group, detector) geometry in FP64, per-pair
// setup in FP32 relative to the group centre, per-sample math in FP32:
//   tau = (d - v t0) / (v dt) = kc + phi,  kc integer, |phi| <= 1/2
//   x   = tau - k = phi - m,  m = k - kc (exact small integer)
//   y   = x * s,  s = v dt sqrt(log2(e)/2) / a0   =>  G = 2^(-y^2)
//   u G = (v dt / s) y G = kappa y G,  kappa = a0 sqrt(2 ln 2)
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace pab {

// Bounds checks of the debug build (-DPAB_DEBUG_CHECKS, tools/variants):
// a failed check traps the kernel, so the GPU tests fail loudly on it.
#ifdef PAB_DEBUG_CHECKS
#define PAB_CHECK(cond) do { if (!(cond)) __trap(); } while (0)
#else
#define PAB_CHECK(cond) do { } while (0)
#endif

constexpr int kWarp = 32;
constexpr float kSqrtHalfLog2e = 0.84932180028801907f;   // sqrt(log2(e) / 2)
constexpr float kSqrt2Ln2 = 1.17741002251547469f;        // sqrt(2 ln 2) = kappa / a0
constexpr float kTwoLn2 = 1.38629436111989061f;          // kappa^2 / a0^2
constexpr float kSqrt2Ln2Cubed = 1.63221961130884960f;   // (kappa / a0)^3

// Cutoffs (in sigmas) at or above which the window walks skip the per-sample
// truncation test: the few samples walked past a window's ends then carry
// G <= exp(-cutoff^2 / 2) < 2^-24, below FP32 resolution (see the walks).
constexpr float kUnmaskedCutoff = 5.8f;

// status bits written by kernels (host raises the reference error classes)
constexpr int kStatusCoincident = 2;   // SimulationError (radiator.py:190-193)
constexpr int kStatusNonFinite = 8;    // OptimizationError (optimizer.py:284-294)

// directivity kinds
constexpr int kDirNone = 0;
constexpr int kDirCosPower = 1;
// (internal template value: cos power with p = 2, the branch-free common case)
constexpr int kDirCos2 = 3;
constexpr int kDirElement = 2;

// adjoint stages
constexpr int kStageFilter = 0;   // p0 only; caller passes res = -real
constexpr int kStageCoarse = 1;   // p0, a0
constexpr int kStageFine = 2;     // p0, a0, position

struct Acq {
  double vdt, inv_vdt, vt0;   // v*dt, 1/(v*dt), v*t0 (full-rate grid)
  int f, n_out;               // decimation factor, samples on the decimated grid
  float cutoff;               // support half-width in sigmas
  float vdt_f, inv_vdt_f, vt0_f;
  float inv_f;
  int dir_kind;
  float dir_param;            // cos power p, or element width w (m)
};

// Ball records in processing (sorted) order; 32 consecutive records form a
// lane group sharing an FP64 centre.  Padding records have orig < 0.
struct __align__(16) BallA { float dx, dy, dz, a0; };          // offset from group centre, radius
struct __align__(16) BallB { float p0, r2, inv_a0; int orig; };   // pressure, |offset|^2, 1/a0, original index

// Lane-group bounding box: centre (FP64), bounding-sphere radius, max a0,
// half extents (48 bytes).
struct GroupMeta { double cx, cy, cz; float radius, a0max, hx, hy, hz, pad; };

// Per (lane group, detector) geometry, computed in FP64 once and broadcast.
struct GroupDet {
  float Sx, Sy, Sz;   // detector - group centre
  float Sn, isn;      // |S|, 1/|S|
  float phg;          // frac(tau_g), tau_g = (|S| - v t0) / (v dt)
  int kg;             // floor(tau_g)
  int slow;           // detector close to the group: exact FP64 per-pair path
};

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// MUFU reciprocal / reciprocal square root without the denormal-range
// rescaling rsqrtf/__fdividef emit (operands here are normal numbers; the
// results are identical to theirs for normal inputs)
__device__ __forceinline__ float rcp_ftz(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float rsqrt_ftz(float x) {
  float y;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// Integer rounding on the FMA / ALU pipes instead of the XU (conversion)
// pipe, which the adjoint's ex2 walk keeps busy: for |x| < 2^22,
// x + 1.5 * 2^23 rounds x to the nearest integer (ties to even, = rintf) in
// the low mantissa bits.  Sample indices of a record stay far inside that
// range (n_out f <= 2^21, host-checked); a window cover computed for an
// arrival beyond 2^22 samples (a ball ~150 m from the detector at 40 MHz)
// comes out on the same side of the record as the arrival (the magic sum
// stays monotonic), i.e. empty, as the exact window is.  (Measured: these
// help the adjoint, -0.1 ms at config 2, but not the forward's setup
// producers, which keep the conversion instructions: +0.5 ms there.)
constexpr float kRoundMagic = 12582912.0f;   // 1.5 * 2^23
constexpr int kRoundMagicBits = 0x4B400000;
constexpr int kMaxRecordSamples = 1 << 21;   // full-rate samples (n_out * f), host-checked
__device__ __forceinline__ int rint_to_int(float x, float* xr) {   // rintf(x) as int and as float
  const float t = __fadd_rn(x, kRoundMagic);
  *xr = __fadd_rn(t, -kRoundMagic);
  return __float_as_int(t) - kRoundMagicBits;
}
__device__ __forceinline__ int floor_to_int(float x) {   // = __float2int_rd(x), |x| < 2^22
  float r;
  const int i = rint_to_int(x, &r);
  return r > x ? i - 1 : i;
}
__device__ __forceinline__ int ceil_to_int(float x) {    // = __float2int_ru(x), |x| < 2^22
  float r;
  const int i = rint_to_int(x, &r);
  return r < x ? i + 1 : i;
}
__device__ __forceinline__ float int_to_float(int i) {   // = (float)i, |i| < 2^22
  return __fadd_rn(__int_as_float(i + kRoundMagicBits), -kRoundMagic);
}

struct Detector {
  double px, py, pz;
  float fx, fy, fz;   // receive direction (unit; = -outward normal)
  float e1x, e1y, e1z, e2x, e2y, e2z;   // element axes (kDirElement)
};

__device__ __forceinline__ Detector load_detector(const double* __restrict__ pos,
                                                  const double* __restrict__ aux, int j) {
  Detector D;
  D.px = pos[3 * j + 0]; D.py = pos[3 * j + 1]; D.pz = pos[3 * j + 2];
  const double* a = aux + 9 * j;
  D.fx = (float)a[0]; D.fy = (float)a[1]; D.fz = (float)a[2];
  D.e1x = (float)a[3]; D.e1y = (float)a[4]; D.e1z = (float)a[5];
  D.e2x = (float)a[6]; D.e2y = (float)a[7]; D.e2z = (float)a[8];
  return D;
}

__device__ __forceinline__ GroupDet group_det(const GroupMeta& g, double px, double py, double pz,
                                              const Acq& a) {
  GroupDet r;
  const double Sx = px - g.cx, Sy = py - g.cy, Sz = pz - g.cz;
  const double Sn = sqrt(Sx * Sx + Sy * Sy + Sz * Sz);
  const double tau = (Sn - a.vt0) * a.inv_vdt;
  const double kf = floor(tau);
  r.Sx = (float)Sx; r.Sy = (float)Sy; r.Sz = (float)Sz;
  r.Sn = (float)Sn;
  r.isn = (float)(1.0 / Sn);   // correctly rounded: the pair distances depend on it
  r.phg = (float)(tau - kf);
  r.kg = (int)kf;
  r.slow = (Sn <= 2.0 * (double)g.radius + 1e-9) ? 1 : 0;
  return r;
}

__device__ __forceinline__ GroupDet empty_gd() {
  GroupDet g;
  g.Sx = g.Sy = g.Sz = 0.f; g.Sn = 1.f; g.isn = 1.f; g.phg = 0.f; g.kg = 0; g.slow = 0;
  return g;
}

// Broadcast without the slow flag (callers carry it in their own flag word).
__device__ __forceinline__ GroupDet shfl_gd_fast(const GroupDet& g, int src) {
  GroupDet r;
  r.Sx = __shfl_sync(0xffffffffu, g.Sx, src);
  r.Sy = __shfl_sync(0xffffffffu, g.Sy, src);
  r.Sz = __shfl_sync(0xffffffffu, g.Sz, src);
  r.Sn = __shfl_sync(0xffffffffu, g.Sn, src);
  r.isn = __shfl_sync(0xffffffffu, g.isn, src);
  r.phg = __shfl_sync(0xffffffffu, g.phg, src);
  r.kg = __shfl_sync(0xffffffffu, g.kg, src);
  r.slow = 0;
  return r;
}

__device__ __forceinline__ int floor_div(int a, int b) {
  int q = a / b;
  return (a % b != 0 && ((a < 0) != (b < 0))) ? q - 1 : q;
}
__device__ __forceinline__ int ceil_div(int a, int b) { return -floor_div(-a, b); }

// floor(a / f) for f >= 1 without integer division: float estimate, then an
// exact integer correction (|a| < 2^24).  BF: branch-free (f = 1 is exact
// through the estimate too) -- more instructions, but no basic-block split,
// which matters where two pair setups are scheduled side by side.
template <bool BF = false>
__device__ __forceinline__ int floor_div_f(int a, int f, float inv_f) {
  if (!BF && f == 1) return a;
  int q = __float2int_rd((float)a * inv_f);
  q += (q + 1) * f <= a ? 1 : 0;
  q -= q * f > a ? 1 : 0;
  return q;
}
template <bool BF = false>
__device__ __forceinline__ int ceil_div_f(int a, int f, float inv_f) { return -floor_div_f<BF>(-a, f, inv_f); }

// ---------------------------------------------------------------------------
// Lean per-pair pieces used by the hot loops (per-ball constants hoisted by
// the caller; detector direction data broadcast from a lane batch).
// ---------------------------------------------------------------------------

struct DetDir {   // receive direction and element axes (FP32)
  float fx, fy, fz, e1x, e1y, e1z, e2x, e2y, e2z;
};

__device__ __forceinline__ DetDir load_detdir(const double* __restrict__ aux, int j) {
  const double* a = aux + 9 * j;
  DetDir d;
  d.fx = (float)a[0]; d.fy = (float)a[1]; d.fz = (float)a[2];
  d.e1x = (float)a[3]; d.e1y = (float)a[4]; d.e1z = (float)a[5];
  d.e2x = (float)a[6]; d.e2y = (float)a[7]; d.e2z = (float)a[8];
  return d;
}

template <int DIR>
__device__ __forceinline__ DetDir shfl_detdir(const DetDir& s, int src) {
  DetDir d = s;
  if (DIR != kDirNone) {
    d.fx = __shfl_sync(0xffffffffu, s.fx, src);
    d.fy = __shfl_sync(0xffffffffu, s.fy, src);
    d.fz = __shfl_sync(0xffffffffu, s.fz, src);
  }
  if (DIR == kDirElement) {
    d.e1x = __shfl_sync(0xffffffffu, s.e1x, src);
    d.e1y = __shfl_sync(0xffffffffu, s.e1y, src);
    d.e1z = __shfl_sync(0xffffffffu, s.e1z, src);
    d.e2x = __shfl_sync(0xffffffffu, s.e2x, src);
    d.e2y = __shfl_sync(0xffffffffu, s.e2y, src);
    d.e2z = __shfl_sync(0xffffffffu, s.e2z, src);
  }
  return d;
}

// D and (GRAD) dD/dr_ball, dD/da0; (hx, hy, hz) = unit ball - detector direction.
template <int DIR, bool GRAD>
__device__ __forceinline__ float dir_weight(const DetDir& dd, float hx, float hy, float hz, float id, float power,
                                            float width, float inv_a0, float* dDdr, float* dDda0) {
  if (DIR == kDirNone) return 1.0f;
  if (DIR == kDirCosPower || DIR == kDirCos2) {
    const float c = dd.fx * hx + dd.fy * hy + dd.fz * hz;
    const float cp = fmaxf(c, 0.0f);
    float D, dDdc;
    if (DIR == kDirCos2 || power == 2.0f) { D = cp * cp; dDdc = 2.0f * cp; }
    else if (power == 1.0f) { D = cp; dDdc = c > 0.0f ? 1.0f : 0.0f; }
    else { D = c > 0.0f ? __powf(cp, power) : 0.0f; dDdc = c > 0.0f ? power * D / cp : 0.0f; }
    if (GRAD) {
      const float s = dDdc * id;
      dDdr[0] = s * (dd.fx - c * hx);
      dDdr[1] = s * (dd.fy - c * hy);
      dDdr[2] = s * (dd.fz - c * hz);
      *dDda0 = 0.0f;
    }
    return D;
  }
  const float s1 = dd.e1x * hx + dd.e1y * hy + dd.e1z * hz;
  const float s2 = dd.e2x * hx + dd.e2y * hy + dd.e2z * hz;
  const float sc = 0.5f * width * inv_a0;
  const float x1 = sc * s1, x2 = sc * s2;
  // sinc and its derivative, branch-free: MUFU sin/cos and reciprocal (no
  // IEEE division), Taylor terms below |x| = 1e-3
  auto sinc = [&](float x, float* f, float* g) {
    float sn, cs;
    __sincosf(x, &sn, &cs);
    const bool small = fabsf(x) < 1e-3f;
    const float r = rcp_ftz(small ? 1.0f : x);
    *f = small ? fmaf(x * x, -1.0f / 6.0f, 1.0f) : sn * r;
    if (GRAD) *g = small ? x * (-1.0f / 3.0f) : (cs - *f) * r;
  };
  float f1, g1 = 0.0f, f2, g2 = 0.0f;
  sinc(x1, &f1, &g1);
  sinc(x2, &f2, &g2);
  if (GRAD) {
    const float a1 = g1 * f2 * sc, a2 = f1 * g2 * sc;
    dDdr[0] = (a1 * (dd.e1x - s1 * hx) + a2 * (dd.e2x - s2 * hx)) * id;
    dDdr[1] = (a1 * (dd.e1y - s1 * hy) + a2 * (dd.e2y - s2 * hy)) * id;
    dDdr[2] = (a1 * (dd.e1z - s1 * hz) + a2 * (dd.e2z - s2 * hz)) * id;
    *dDda0 = -(a1 * s1 + a2 * s2) * inv_a0;
  }
  return f1 * f2;
}

// Distance and arrival-time split for one pair.  Fast path: FP32 relative to
// the group centre; slow path (detector within two group radii): FP64.
struct PairGeom {
  float d, id, phi, rx, ry, rz;
  int kc;
  int coincident;
};

__device__ __forceinline__ PairGeom pair_geom(const GroupDet& gd, const GroupMeta& gm, double px, double py,
                                              double pz, const BallA& A, const BallB& B, const Acq& a) {
  PairGeom g;
  g.coincident = 0;
  float tr;
  int kbase;
  if (!gd.slow) {
    const float sd = gd.Sx * A.dx + gd.Sy * A.dy + gd.Sz * A.dz;
    const float num = B.r2 - 2.0f * sd;
    const float e1 = fmaf(num * gd.isn, gd.isn, 1.0f);
    const float dd = __fdividef(num * gd.isn, 1.0f + e1 * rsqrtf(e1));
    g.d = gd.Sn + dd;
    tr = fmaf(dd, a.inv_vdt_f, gd.phg);
    kbase = gd.kg;
    g.rx = A.dx - gd.Sx; g.ry = A.dy - gd.Sy; g.rz = A.dz - gd.Sz;
  } else {
    const double dx = gm.cx + (double)A.dx - px, dy = gm.cy + (double)A.dy - py, dz = gm.cz + (double)A.dz - pz;
    const double d = sqrt(dx * dx + dy * dy + dz * dz);
    if (d < 1e-12 && B.orig >= 0) g.coincident = 1;
    const double tau = (d - a.vt0) * a.inv_vdt;
    const double kf = floor(tau);
    kbase = (int)kf;
    tr = (float)(tau - kf);
    g.d = (float)(d > 1e-30 ? d : 1e-30);
    g.rx = (float)dx; g.ry = (float)dy; g.rz = (float)dz;
  }
  const float kr = rintf(tr);
  g.kc = kbase + (int)kr;
  g.phi = tr - kr;
  g.id = __fdividef(1.0f, g.d);
  return g;
}

// Fast path only (caller knows the detector is far from the group).
__device__ __forceinline__ PairGeom pair_geom_fast(const GroupDet& gd, const BallA& A, const BallB& B,
                                                   const Acq& a) {
  PairGeom g;
  g.coincident = 0;
  const float sd = gd.Sx * A.dx + gd.Sy * A.dy + gd.Sz * A.dz;
  const float num = B.r2 - 2.0f * sd;
  const float e1 = fmaf(num * gd.isn, gd.isn, 1.0f);
  const float dd = (num * gd.isn) * rcp_ftz(1.0f + e1 * rsqrt_ftz(e1));
  g.d = gd.Sn + dd;
  const float tr = fmaf(dd, a.inv_vdt_f, gd.phg);
  g.rx = A.dx - gd.Sx; g.ry = A.dy - gd.Sy; g.rz = A.dz - gd.Sz;
  const float kr = rintf(tr);
  g.kc = gd.kg + (int)kr;
  g.phi = tr - kr;
  g.id = rcp_ftz(g.d);
  return g;
}

// pair_geom_fast with the rounding of the arrival time off the XU pipe
// (bitwise the same result); also returns kf = (float)kc
__device__ __forceinline__ PairGeom pair_geom_lean(const GroupDet& gd, const BallA& A, const BallB& B,
                                                   const Acq& a, float* kf) {
  PairGeom g;
  g.coincident = 0;
  const float sd = gd.Sx * A.dx + gd.Sy * A.dy + gd.Sz * A.dz;
  const float num = B.r2 - 2.0f * sd;
  const float e1 = fmaf(num * gd.isn, gd.isn, 1.0f);
  const float dd = (num * gd.isn) * rcp_ftz(1.0f + e1 * rsqrt_ftz(e1));
  g.d = gd.Sn + dd;
  const float tr = fmaf(dd, a.inv_vdt_f, gd.phg);
  g.rx = A.dx - gd.Sx; g.ry = A.dy - gd.Sy; g.rz = A.dz - gd.Sz;
  float kr;
  const int ikr = rint_to_int(tr, &kr);
  g.kc = gd.kg + ikr;
  g.phi = tr - kr;
  g.id = rcp_ftz(g.d);
  *kf = int_to_float(g.kc);
  return g;
}

// pair_window_cover without XU conversions (same result)
__device__ __forceinline__ void pair_window_cover_lean(float kf, float phi, float rho, const Acq& a, int* jlo,
                                                       int* jhi) {
  *jlo = max(floor_to_int((kf + (phi - rho)) * a.inv_f), 0);
  *jhi = min(ceil_to_int((kf + (phi + rho)) * a.inv_f), a.n_out - 1);
}

// Cover of the u- window for masked walks: jlo' <= jlo and jhi' >= jhi, each
// off by at most one (float quotient, no exact integer correction); the
// caller's per-sample mask |x| <= rho selects the exact support.
__device__ __forceinline__ void pair_window_cover(int kc, float phi, float rho, const Acq& a, int* jlo, int* jhi) {
  const float kf = (float)kc;
  *jlo = max(__float2int_rd((kf + (phi - rho)) * a.inv_f), 0);
  *jhi = min(__float2int_ru((kf + (phi + rho)) * a.inv_f), a.n_out - 1);
}

// u- window on the decimated grid, clipped to [0, n_out).
template <bool BF = false>
__device__ __forceinline__ void pair_window(int kc, float phi, float rho, const Acq& a, int* jlo, int* jhi) {
  const int klo = kc + __float2int_ru(phi - rho);
  const int khi = kc + __float2int_rd(phi + rho);
  *jlo = max(ceil_div_f<BF>(klo, a.f, a.inv_f), 0);
  *jhi = min(floor_div_f<BF>(khi, a.f, a.inv_f), a.n_out - 1);
}

// u+ window (near field; only called when the group can have one).
__device__ __forceinline__ void pair_near_window(float d, float rho, const Acq& a, int* nlo, int* nhi, int* nkc,
                                                 float* nphi) {
  *nlo = 1; *nhi = 0; *nkc = 0; *nphi = 0.0f;
  const double taup = -((double)d + a.vt0) * a.inv_vdt;
  if (taup + (double)rho >= 0.0) {
    const double kp = rint(taup);
    *nkc = (int)kp;
    *nphi = (float)(taup - kp);
    const int klo = *nkc + __float2int_ru(*nphi - rho);
    const int khi = *nkc + __float2int_rd(*nphi + rho);
    *nlo = max(ceil_div(klo, a.f), 0);
    *nhi = min(floor_div(khi, a.f), a.n_out - 1);
  }
}

// Can any ball of the group have a u+ window at this detector?
__device__ __forceinline__ bool group_near(const Acq& a, const GroupDet& gd, const GroupMeta& gm) {
  const float rho = a.cutoff * gm.a0max * a.inv_vdt_f;
  return -(gd.Sn - gm.radius + a.vt0_f) * a.inv_vdt_f + rho + 2.0f >= 0.0f || gd.slow;
}

// Decimated-sample range a lane group can touch for one detector: centre
// tau_g -+ (radius / v dt + rho_max + 2), plus [0, ..] when a u+ term can exist.
__device__ __forceinline__ void group_range(const Acq& a, const GroupDet& gd, const GroupMeta& gm,
                                            int* lo, int* hi) {
  // distance range over the group's bounding box: |S| - p <= d <= |S| + p +
  // r^2 / 2|S|, p = projection of the box half-extents on the detector
  // direction (each side capped by the bounding sphere, |d - |S|| <= r)
  const float rho = a.cutoff * gm.a0max * a.inv_vdt_f;
  const float proj = (fabsf(gd.Sx) * gm.hx + fabsf(gd.Sy) * gm.hy + fabsf(gd.Sz) * gm.hz) * gd.isn;
  const float dlo = fminf(proj, gm.radius);
  const float dhi = fminf(proj + 0.5f * gm.radius * gm.radius * gd.isn, gm.radius);
  const float c = gd.phg;
  int klo = gd.kg + (int)floorf(c - (dlo * a.inv_vdt_f + rho + 0.5f));
  int khi = gd.kg + (int)ceilf(c + (dhi * a.inv_vdt_f + rho + 0.5f));
  if (gd.slow) {   // FP32 S is coarse near the detector: widen generously
    klo = min(klo, -(int)ceilf(rho) - 2);
  }
  // near field: u+ = d + v t0 + k v dt can vanish for k >= 0
  const float dmin = gd.Sn - gm.radius;
  const float taup_max = -(dmin + a.vt0_f) * a.inv_vdt_f;
  if (taup_max + rho + 1.0f >= 0.0f) {
    klo = min(klo, (int)floorf(-(gd.Sn + gm.radius + a.vt0_f) * a.inv_vdt_f - rho - 2.0f));
    khi = max(khi, (int)ceilf(taup_max + rho + 2.0f));
  }
  *lo = max(floor_div_f<true>(klo, a.f, a.inv_f), 0);   // |k| < 2^24 (host-checked): no integer division
  *hi = min(ceil_div_f<true>(khi, a.f, a.inv_f), a.n_out - 1);
}

// Dual-walk pairing directions (forward kernel): the 8 x 8 cells of a
// hemi-octahedral map of the unit hemisphere (a pairing along u equals the
// pairing along -u).  For every pair of consecutive lane groups (a 64-ball
// "unit") and every cell, pab_pair_table stores the 64 balls sorted by their
// projection on the cell's centre direction; at a detector the forward pairs
// neighbours of that order for the cell containing the detector direction:
// the two balls a lane walks together then have nearly equal arrival windows.
constexpr int kPairDirs = 64;
__device__ __forceinline__ void pair_dir(int k, float* ux, float* uy, float* uz) {   // cell centre
  const float a = ((float)(k >> 3) + 0.5f) * 0.25f - 1.0f, b = ((float)(k & 7) + 0.5f) * 0.25f - 1.0f;
  const float px = 0.5f * (a + b), py = 0.5f * (a - b), pz = 1.0f - fabsf(px) - fabsf(py);
  const float inv = rsqrtf(px * px + py * py + pz * pz);
  *ux = px * inv;
  *uy = py * inv;
  *uz = pz * inv;
}
__device__ __forceinline__ int pair_cell(float x, float y, float z) {   // cell of direction +-(x, y, z)
  if (z < 0.0f) { x = -x; y = -y; z = -z; }
  const float inv = 1.0f / fmaxf(fabsf(x) + fabsf(y) + z, 1e-30f);
  const float px = x * inv, py = y * inv;
  const int i = min(max(__float2int_rd((px + py + 1.0f) * 4.0f), 0), 7);
  const int j = min(max(__float2int_rd((px - py + 1.0f) * 4.0f), 0), 7);
  return (i << 3) | j;
}

__host__ __device__ inline Acq make_acq(double v, double t0, double dt, int f, int n_out, double cutoff,
                                        int dir_kind, double dir_param) {
  Acq a;
  a.vdt = v * dt;
  a.inv_vdt = 1.0 / a.vdt;
  a.vt0 = v * t0;
  a.f = f;
  a.n_out = n_out;
  a.cutoff = (float)cutoff;
  a.vdt_f = (float)a.vdt;
  a.inv_vdt_f = (float)a.inv_vdt;
  a.vt0_f = (float)a.vt0;
  a.inv_f = 1.0f / (float)f;
  a.dir_kind = dir_kind;
  a.dir_param = (float)dir_param;
  return a;
}

}  // namespace pab
