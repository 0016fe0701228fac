// Ball binning: spatial sort keys and lane-group packing.
//
// The reference brute-forces every 512-ball chunk against every sensor block
// (radiator.py:185-196).  Here balls are visited in Morton order so that 32
// consecutive balls (a lane group) are spatially compact: their arrival
// windows at any detector overlap, which bounds the per-warp sample tile of
// the forward kernel and the residual segment of the adjoint.  The order is a
// performance choice only: any permutation gives the same sums up to the
// (deterministic) summation order.
#include "pab_common.cuh"

namespace pab {

__device__ __forceinline__ uint32_t spread3(uint32_t v) {   // 10 bits -> every 3rd bit
  v &= 0x3ffu;
  v = (v | (v << 16)) & 0x030000FFu;
  v = (v | (v << 8)) & 0x0300F00Fu;
  v = (v | (v << 4)) & 0x030C30C3u;
  v = (v | (v << 2)) & 0x09249249u;
  return v;
}

// 3-D Hilbert index of a 10-bit lattice point (Skilling's transpose form).
// Unlike Morton order the curve has no jumps, so 32 consecutive balls form a
// compact lane group (tight arrival-time spread at every detector).
__device__ __forceinline__ uint32_t hilbert3(uint32_t x, uint32_t y, uint32_t z) {
  uint32_t X[3] = {x, y, z};
  constexpr uint32_t M = 1u << 9;
#pragma unroll
  for (uint32_t Q = M; Q > 1; Q >>= 1) {
    const uint32_t P = Q - 1;
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      if (X[i] & Q) {
        X[0] ^= P;
      } else {
        const uint32_t t = (X[0] ^ X[i]) & P;
        X[0] ^= t;
        X[i] ^= t;
      }
    }
  }
  X[1] ^= X[0];
  X[2] ^= X[1];
  uint32_t t = 0;
#pragma unroll
  for (uint32_t Q = M; Q > 1; Q >>= 1)
    if (X[2] & Q) t ^= Q - 1;
  X[0] ^= t; X[1] ^= t; X[2] ^= t;
  uint32_t h = 0;
#pragma unroll
  for (int b = 9; b >= 0; --b)
    h = (h << 3) | (((X[0] >> b) & 1u) << 2) | (((X[1] >> b) & 1u) << 1) | ((X[2] >> b) & 1u);
  return h;
}

// key = a0 bucket (4 bits) << 58 | hilbert30 << 28 | index (28 bits): balls
// of similar radius share lane groups (equal window lengths: no divergence in
// the per-lane window loops), spatially compact within a bucket.
__device__ __forceinline__ int64_t sort_key(const double* __restrict__ pos, const double* __restrict__ a0, int64_t i,
                                            double lox, double loy, double loz, double inv_ext, double a0lo,
                                            double inv_a0span, int nbuckets) {
  const double s = 1023.0 * inv_ext;
  const uint32_t qx = (uint32_t)fmin(fmax((pos[3 * i + 0] - lox) * s, 0.0), 1023.0);
  const uint32_t qy = (uint32_t)fmin(fmax((pos[3 * i + 1] - loy) * s, 0.0), 1023.0);
  const uint32_t qz = (uint32_t)fmin(fmax((pos[3 * i + 2] - loz) * s, 0.0), 1023.0);
  const uint64_t code = (uint64_t)hilbert3(qx, qy, qz);
  int b = 0;
  if (nbuckets > 1) b = (int)fmin(fmax((a0[i] - a0lo) * inv_a0span * nbuckets, 0.0), (double)(nbuckets - 1));
  return (int64_t)(((uint64_t)b << 58) | (code << 28) | ((uint64_t)i & 0xFFFFFFFull));
}

__global__ void morton_keys_kernel(const double* __restrict__ pos, const double* __restrict__ a0, int64_t n,
                                   double lox, double loy, double loz, double inv_ext, double a0lo,
                                   double inv_a0span, int nbuckets, int64_t* __restrict__ keys) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  keys[i] = sort_key(pos, a0, i, lox, loy, loz, inv_ext, a0lo, inv_a0span, nbuckets);
}

// Same keys with the bounds read from device memory (pab_cloud_bounds): no
// host round trip between the bounds and the keys.
__global__ void sort_keys_dev_kernel(const double* __restrict__ pos, const double* __restrict__ a0, int64_t n,
                                     const double* __restrict__ bounds, int nbuckets, int64_t* __restrict__ keys) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double a0lo = bounds[4], a0hi = bounds[5];
  const int nb = (nbuckets > 1 && a0hi > a0lo) ? nbuckets : 1;
  keys[i] = sort_key(pos, a0, i, bounds[0], bounds[1], bounds[2], 1.0 / bounds[3], a0lo,
                     nb > 1 ? 1.0 / (a0hi - a0lo) : 0.0, nb);
}

__device__ __forceinline__ double warp_min(double v) {
  for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ double warp_max(double v) {
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ float warp_maxf(float v) {
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// One warp per lane group: bounding-box centre (FP64), FP32 offsets, radius,
// max a0.  Padding lanes (i >= n) become inert records (orig = -1, p0 = 0).
__global__ void pack_kernel(const double* __restrict__ pos, const double* __restrict__ p0,
                            const double* __restrict__ a0, const int32_t* __restrict__ perm, int64_t n,
                            int64_t n_groups, BallA* __restrict__ ra, BallB* __restrict__ rb,
                            GroupMeta* __restrict__ gm) {
  const int lane = threadIdx.x & 31;
  const int64_t g = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (g >= n_groups) return;
  const int64_t i = g * kWarp + lane;
  const int b_in = i < n ? perm[i] : -1;   // -1: inert padding slot
  const bool live = b_in >= 0;
  int b = 0;
  double x = 0, y = 0, z = 0, pp = 0, aa = 1.0;
  if (live) {
    b = b_in;
    x = pos[3 * (int64_t)b + 0]; y = pos[3 * (int64_t)b + 1]; z = pos[3 * (int64_t)b + 2];
    pp = p0[b]; aa = a0[b];
  }
  const double big = 1e300;
  const double xl = warp_min(live ? x : big), xh = warp_max(live ? x : -big);
  const double yl = warp_min(live ? y : big), yh = warp_max(live ? y : -big);
  const double zl = warp_min(live ? z : big), zh = warp_max(live ? z : -big);
  const double cx = 0.5 * (xl + xh), cy = 0.5 * (yl + yh), cz = 0.5 * (zl + zh);
  BallA A;
  BallB B;
  if (live) {
    A.dx = (float)(x - cx); A.dy = (float)(y - cy); A.dz = (float)(z - cz); A.a0 = (float)aa;
    B.p0 = (float)pp;
    B.r2 = A.dx * A.dx + A.dy * A.dy + A.dz * A.dz;
    B.inv_a0 = 1.0f / A.a0;
    B.orig = b;
  } else {
    A.dx = A.dy = A.dz = 0.0f; A.a0 = 1.0f;
    B.p0 = 0.0f; B.r2 = 0.0f; B.inv_a0 = 1.0f; B.orig = -1;
  }
  const float rad = warp_maxf(live ? sqrtf(B.r2) : 0.0f);
  const float amax = warp_maxf(live ? A.a0 : 0.0f);
  ra[i] = A;
  rb[i] = B;
  if (lane == 0) {
    GroupMeta m;
    m.cx = cx; m.cy = cy; m.cz = cz;
    m.radius = rad * 1.000001f + 1e-12f;
    m.a0max = amax;
    // half extents, rounded up so the FP32 box still contains every ball
    m.hx = (float)(0.5 * (xh - xl)) * 1.000001f + 1e-12f;
    m.hy = (float)(0.5 * (yh - yl)) * 1.000001f + 1e-12f;
    m.hz = (float)(0.5 * (zh - zl)) * 1.000001f + 1e-12f;
    m.pad = 0.0f;
    gm[g] = m;
  }
}

// Pairing table of the forward's dual walk (see pair_dir): one warp per unit
// (lane groups 2u, 2u+1); lane l holds balls l and 32 + l of the unit.  For
// each direction the 64 projections are bitonic-sorted (key = order-preserving
// float bits with the ball id in the low 6 bits: deterministic, ties by id)
// and written as 64 ball ids.  Performance only: any table gives the same
// sums up to FP32 summation order.
__device__ __forceinline__ unsigned orderable(float f) {
  const unsigned u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

__device__ __forceinline__ void bitonic64(unsigned& x0, unsigned& x1, int lane) {
#pragma unroll
  for (int k = 2; k <= 64; k <<= 1) {
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
      if (j == 32) {   // partner in the other register (k = 64: ascending)
        const unsigned a = min(x0, x1), b = max(x0, x1);
        x0 = a;
        x1 = b;
      } else {
        const bool up0 = k == 64 ? true : (k == 32 ? true : (lane & k) == 0);
        const bool up1 = k == 64 ? true : (k == 32 ? false : (lane & k) == 0);
        const bool lower = (lane & j) == 0;
        const unsigned o0 = __shfl_xor_sync(0xffffffffu, x0, j);
        const unsigned o1 = __shfl_xor_sync(0xffffffffu, x1, j);
        x0 = (lower == up0) ? min(x0, o0) : max(x0, o0);
        x1 = (lower == up1) ? min(x1, o1) : max(x1, o1);
      }
    }
  }
}

__global__ void pair_table_kernel(const BallA* __restrict__ ra, const GroupMeta* __restrict__ gm, int64_t n_units,
                                  int64_t n_groups, unsigned char* __restrict__ table) {
  const int lane = threadIdx.x & 31;
  const int64_t u = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (u >= n_units) return;
  const int64_t g0 = 2 * u;
  const bool hasB = g0 + 1 < n_groups;
  const GroupMeta ma = gm[g0];
  const BallA a = ra[g0 * kWarp + lane];
  float bx = 0.f, by = 0.f, bz = 0.f;
  if (hasB) {   // second group's balls relative to the first group's centre
    const GroupMeta mb = gm[g0 + 1];
    const BallA b = ra[(g0 + 1) * kWarp + lane];
    bx = (float)(mb.cx - ma.cx) + b.dx;
    by = (float)(mb.cy - ma.cy) + b.dy;
    bz = (float)(mb.cz - ma.cz) + b.dz;
  }
  // layout [cell][unit][64]: a detector's CTAs read one cell's rows, whose
  // working set (64 B per unit) stays in L2 even when the whole table does not
  for (int k = 0; k < kPairDirs; ++k) {
    unsigned char* out = table + ((size_t)k * n_units + u) * 64;
    float ux, uy, uz;
    pair_dir(k, &ux, &uy, &uz);
    unsigned x0 = (orderable(a.dx * ux + a.dy * uy + a.dz * uz) & ~63u) | (unsigned)lane;
    unsigned x1 = (orderable(bx * ux + by * uy + bz * uz) & ~63u) | (unsigned)(32 + lane);
    bitonic64(x0, x1, lane);
    out[lane] = (unsigned char)(x0 & 63u);
    out[32 + lane] = (unsigned char)(x1 & 63u);
  }
}

// Exact coincidence test (reference radiator.py:189-193: SimulationError when
// a ball lies within 1e-12 of a sensor), in FP64 on the caller-order master
// positions: one warp per lane group tests every detector against the
// group's bounding box (+1e-9 margin), and only a detector inside the box is
// compared with the group's 32 balls.  The kernels' FP32 offsets from the
// group centre cannot resolve 1e-12 for a ball far from its centre, so the
// flag comes from here.  Cost: n_groups x n_det box tests per pass.
__global__ void coincident_kernel(const BallB* __restrict__ rb, const GroupMeta* __restrict__ gm, int64_t n_groups,
                                  const double* __restrict__ pos, const double* __restrict__ det, int n_det,
                                  int* __restrict__ status) {
  const int lane = threadIdx.x & 31;
  const int64_t g = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (g >= n_groups) return;
  const GroupMeta m = gm[g];
  const int orig = rb[g * kWarp + lane].orig;
  double bx = 0, by = 0, bz = 0;
  if (orig >= 0) { bx = pos[3 * (int64_t)orig]; by = pos[3 * (int64_t)orig + 1]; bz = pos[3 * (int64_t)orig + 2]; }
  bool hit = false;
  for (int j0 = 0; j0 < n_det; j0 += kWarp) {
    const int j = j0 + lane;
    bool in = false;
    double px = 0, py = 0, pz = 0;
    if (j < n_det) {
      px = det[3 * j]; py = det[3 * j + 1]; pz = det[3 * j + 2];
      in = fabs(px - m.cx) <= (double)m.hx + 1e-9 && fabs(py - m.cy) <= (double)m.hy + 1e-9 &&
           fabs(pz - m.cz) <= (double)m.hz + 1e-9;
    }
    unsigned cand = __ballot_sync(0xffffffffu, in);
    while (cand) {   // rare: a detector inside the group's box
      const int src = __ffs(cand) - 1;
      cand &= cand - 1;
      const double qx = __shfl_sync(0xffffffffu, px, src), qy = __shfl_sync(0xffffffffu, py, src),
                   qz = __shfl_sync(0xffffffffu, pz, src);
      const double dx = bx - qx, dy = by - qy, dz = bz - qz;
      hit |= orig >= 0 && sqrt(dx * dx + dy * dy + dz * dz) < 1e-12;
    }
  }
  if (__any_sync(0xffffffffu, hit) && lane == 0) atomicOr(status, kStatusCoincident);
}

}  // namespace pab

using namespace pab;

extern "C" {

int pab_morton_keys(const double* pos, const double* a0, int64_t n, double lox, double loy, double loz,
                    double extent, double a0lo, double a0hi, int a0_buckets, int64_t* keys, void* stream) {
  if (n <= 0) return 0;
  if (!pos || !keys || !(extent > 0.0) || n > (1ll << 28) || a0_buckets < 1 || a0_buckets > 16) return 1;
  if (a0_buckets > 1 && (!a0 || !(a0hi > a0lo))) a0_buckets = 1;
  const int threads = 256;
  morton_keys_kernel<<<(unsigned)((n + threads - 1) / threads), threads, 0, (cudaStream_t)stream>>>(
      pos, a0, n, lox, loy, loz, 1.0 / extent, a0lo, a0_buckets > 1 ? 1.0 / (a0hi - a0lo) : 0.0, a0_buckets,
      keys);
  return cudaGetLastError() == cudaSuccess ? 0 : 4;
}

int pab_sort_keys(const double* pos, const double* a0, int64_t n, const double* bounds, int a0_buckets,
                  int64_t* keys, void* stream) {
  if (n <= 0) return 0;
  if (!pos || !a0 || !bounds || !keys || n > (1ll << 28) || a0_buckets < 1 || a0_buckets > 16) return 1;
  const int threads = 256;
  sort_keys_dev_kernel<<<(unsigned)((n + threads - 1) / threads), threads, 0, (cudaStream_t)stream>>>(
      pos, a0, n, bounds, a0_buckets, keys);
  return cudaGetLastError() == cudaSuccess ? 0 : 4;
}

int pab_pack(const double* pos, const double* p0, const double* a0, const int32_t* perm, int64_t n,
             void* rec_a, void* rec_b, void* group_meta, void* stream) {
  if (n <= 0) return 0;
  if (!pos || !p0 || !a0 || !perm || !rec_a || !rec_b || !group_meta) return 1;
  const int64_t n_groups = (n + kWarp - 1) / kWarp;
  const int warps = 8;
  pack_kernel<<<(unsigned)((n_groups + warps - 1) / warps), warps * kWarp, 0, (cudaStream_t)stream>>>(
      pos, p0, a0, perm, n, n_groups, (BallA*)rec_a, (BallB*)rec_b, (GroupMeta*)group_meta);
  return cudaGetLastError() == cudaSuccess ? 0 : 4;
}

int pab_pair_table(const void* rec_a, const void* group_meta, int64_t n_groups, unsigned char* table,
                   void* stream) {
  if (n_groups <= 0) return 0;
  if (!rec_a || !group_meta || !table) return 1;
  const int64_t n_units = (n_groups + 1) / 2;
  const int warps = 8;
  pair_table_kernel<<<(unsigned)((n_units + warps - 1) / warps), warps * kWarp, 0, (cudaStream_t)stream>>>(
      (const BallA*)rec_a, (const GroupMeta*)group_meta, n_units, n_groups, table);
  return cudaGetLastError() == cudaSuccess ? 0 : 4;
}

size_t pab_pair_table_bytes(int64_t n_groups) { return (size_t)((n_groups + 1) / 2) * kPairDirs * 64; }

int pab_record_sizes(int* ball_a, int* ball_b, int* group_meta) {
  *ball_a = (int)sizeof(BallA);
  *ball_b = (int)sizeof(BallB);
  *group_meta = (int)sizeof(GroupMeta);
  return 0;
}

int pab_coincident(const void* rec_b, const void* group_meta, int64_t n_groups, const double* pos,
                   const double* det_pos, int n_det, int* status, void* stream) {
  if (n_groups <= 0 || n_det <= 0) return 0;
  if (!rec_b || !group_meta || !pos || !det_pos || !status) return 1;
  const int warps = 8;
  coincident_kernel<<<(unsigned)((n_groups + warps - 1) / warps), warps * kWarp, 0, (cudaStream_t)stream>>>(
      (const BallB*)rec_b, (const GroupMeta*)group_meta, n_groups, pos, det_pos, n_det, status);
  return cudaGetLastError() == cudaSuccess ? 0 : 4;
}

}  // extern "C"
