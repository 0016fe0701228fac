// Adaptive density control on the GPU.
//
// Replaces reference optimizer.density_control (optimizer.py:314-406):
//   destroy  p0 < frac * median(p0) or a0 outside [a0_min, a0_max]   (:330-345)
//   split    a0 > split_a0 -> two children +-0.5 a0 u, p0/2, a0/sqrt2 (:347-374)
//   duplicate (fine) the top ceil((1-q) n) balls by |dL/dpos|,
//            jitter a0/4 u, ascending original order                   (:376-389)
// The decision quantities use the same IEEE double expressions as numpy
// (median of two middle values by exact radix selection, norms as
// sqrt((x*x + y*y) + z*z), no FMA contraction), so outputs are bit-identical
// to the reference for identical inputs.  The isotropic unit vectors come from
// the reference's SplitMix64/Box-Muller stream, drawn on the host (a few
// thousand doubles per pass) and uploaded.
#include "pab_common.cuh"

namespace pab {

__device__ __forceinline__ unsigned long long f64_key(double x) {
  const unsigned long long u = (unsigned long long)__double_as_longlong(x);
  return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}
__device__ __forceinline__ double key_f64(unsigned long long k) {
  const unsigned long long u = (k >> 63) ? (k & 0x7FFFFFFFFFFFFFFFull) : ~k;
  return __longlong_as_double((long long)u);
}

// Selection state: [0] prefix, [1] mask, [2] k (remaining rank), [3..258] histogram
__global__ void select_init_kernel(unsigned long long* st, long long k) {
  st[0] = 0ull;
  st[1] = 0ull;
  st[2] = (unsigned long long)k;
  for (int i = 0; i < 256; ++i) st[3 + i] = 0ull;
}

__global__ void select_hist_kernel(const double* __restrict__ x, int64_t n, int shift,
                                   unsigned long long* __restrict__ st) {
  __shared__ unsigned int h[256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) h[i] = 0u;
  __syncthreads();
  const unsigned long long prefix = st[0], mask = st[1];
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long k = f64_key(x[i]);
    if ((k & mask) == prefix) atomicAdd(&h[(k >> shift) & 0xFF], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 256; i += blockDim.x)
    if (h[i]) atomicAdd(&st[3 + i], (unsigned long long)h[i]);
}

__global__ void select_pick_kernel(unsigned long long* st, int shift, double* out) {
  unsigned long long k = st[2];
  int d = 0;
  for (; d < 255; ++d) {
    const unsigned long long c = st[3 + d];
    if (k < c) break;
    k -= c;
  }
  st[0] |= (unsigned long long)d << shift;
  st[1] |= 0xFFull << shift;
  st[2] = k;
  for (int i = 0; i < 256; ++i) st[3 + i] = 0ull;
  if (shift == 0) *out = key_f64(st[0]);
}

// key = -1 keep, +1 destroy (NaN comparisons are false, as in numpy)
// median = m1 (odd n) or (m1 + m2) / 2 (even n, numpy's mean of the middle pair)
__global__ void keep_key_kernel(const double* __restrict__ p0, const double* __restrict__ a0, int64_t n,
                                const double* __restrict__ m1, const double* __restrict__ m2, double frac,
                                double a0_min, double a0_max, double* __restrict__ key) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double median = m2 ? __ddiv_rn(__dadd_rn(*m1, *m2), 2.0) : *m1;
  const double thr = __dmul_rn(frac, median);
  const bool weak = p0[i] < thr;
  const bool bad = (a0[i] < a0_min) | (a0[i] > a0_max);
  key[i] = (weak || bad) ? 1.0 : -1.0;
}

// key = -1 split, +1 keep as parent
__global__ void split_key_kernel(const double* __restrict__ a0, int64_t n, double split_a0, double* __restrict__ key) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  key[i] = a0[i] > split_a0 ? -1.0 : 1.0;
}

// norms of rows idx[r] of a [*,3] array: sqrt((x*x + y*y) + z*z)
__global__ void row_norm_kernel(const double* __restrict__ v, const int32_t* __restrict__ idx, int64_t m,
                                double* __restrict__ out) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= m) return;
  const double* p = v + 3 * (int64_t)(idx ? idx[r] : r);
  out[r] = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(p[0], p[0]), __dmul_rn(p[1], p[1])), __dmul_rn(p[2], p[2])));
}

// duplicate selection key over gradient norms: -1 strictly above t, 0 equal, +1 below
__global__ void dup_key_kernel(const double* __restrict__ gn, int64_t m, const double* __restrict__ t,
                               double* __restrict__ key) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  const double v = gn[i], th = *t;
  key[i] = v > th ? -1.0 : (v == th ? 0.0 : 1.0);
}

// mark the first `take` ties (ascending index) as selected: key -> -1
__global__ void dup_take_ties_kernel(const int32_t* __restrict__ ties, const int* __restrict__ n_ties,
                                     const int* __restrict__ n_above, int k_dup, double* __restrict__ key) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  const int take = k_dup - *n_above;
  if (r < *n_ties && r < take) key[ties[r]] = -1.0;
}

// children of split balls: +child at [0, m), -child at [m, 2m)
__global__ void split_children_kernel(const double* __restrict__ pos, const double* __restrict__ p0,
                                      const double* __restrict__ a0, const double* __restrict__ unit, int64_t m,
                                      double* __restrict__ out_pos, double* __restrict__ out_p0,
                                      double* __restrict__ out_a0) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  const double h = __dmul_rn(0.5, a0[i]);
  const double sqrt2 = 1.4142135623730951;   // math.sqrt(2.0)
  for (int c = 0; c < 3; ++c) {
    const double off = __dmul_rn(h, unit[3 * i + c]);
    out_pos[3 * i + c] = __dadd_rn(pos[3 * i + c], off);
    out_pos[3 * (m + i) + c] = __dadd_rn(pos[3 * i + c], -off);
  }
  const double cp = __dmul_rn(0.5, p0[i]);
  const double ca = __ddiv_rn(a0[i], sqrt2);
  out_p0[i] = cp; out_p0[m + i] = cp;
  out_a0[i] = ca; out_a0[m + i] = ca;
}

// duplicates: pos + (a0 / 4) * unit, p0/a0 copied
__global__ void duplicate_kernel(const double* __restrict__ pos, const double* __restrict__ p0,
                                 const double* __restrict__ a0, const double* __restrict__ unit, int64_t m,
                                 double* __restrict__ out_pos, double* __restrict__ out_p0,
                                 double* __restrict__ out_a0) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  const double q = __ddiv_rn(a0[i], 4.0);
  for (int c = 0; c < 3; ++c) out_pos[3 * i + c] = __dadd_rn(pos[3 * i + c], __dmul_rn(q, unit[3 * i + c]));
  out_p0[i] = p0[i];
  out_a0[i] = a0[i];
}

}  // namespace pab

using namespace pab;

static inline unsigned blocks_for(int64_t n, int t = 256) { return (unsigned)((n + t - 1) / t); }

extern "C" {

size_t pab_select_workspace_bytes(void) { return 259 * sizeof(unsigned long long); }

// *out = k-th smallest (0-based) of x[0..n) by exact 8-pass radix selection.
int pab_select_kth_f64(const double* x, int64_t n, int64_t k, double* out, void* workspace, void* stream) {
  if (!x || !out || !workspace || n <= 0 || k < 0 || k >= n) return 1;
  const cudaStream_t s = (cudaStream_t)stream;
  unsigned long long* st = (unsigned long long*)workspace;
  select_init_kernel<<<1, 1, 0, s>>>(st, (long long)k);
  const int64_t nb = (n + 255) / 256;
  const unsigned grid = (unsigned)(nb < 1184 ? nb : 1184);
  for (int shift = 56; shift >= 0; shift -= 8) {
    select_hist_kernel<<<grid, 256, 0, s>>>(x, n, shift, st);
    select_pick_kernel<<<1, 1, 0, s>>>(st, shift, out);
  }
  return cudaGetLastError() == cudaSuccess ? 0 : 4;
}

int pab_density_keep_key(const double* p0, const double* a0, int64_t n, const double* median_lo,
                         const double* median_hi, double frac, double a0_min, double a0_max, double* key,
                         void* stream) {
  if (n <= 0) return 0;
  if (!p0 || !a0 || !median_lo || !key) return 1;
  keep_key_kernel<<<blocks_for(n), 256, 0, (cudaStream_t)stream>>>(p0, a0, n, median_lo, median_hi, frac, a0_min,
                                                                    a0_max, key);
  return cudaGetLastError() == cudaSuccess ? 0 : 4;
}

int pab_density_split_key(const double* a0, int64_t n, double split_a0, double* key, void* stream) {
  if (n <= 0) return 0;
  if (!a0 || !key) return 1;
  split_key_kernel<<<blocks_for(n), 256, 0, (cudaStream_t)stream>>>(a0, n, split_a0, key);
  return cudaGetLastError() == cudaSuccess ? 0 : 4;
}

int pab_row_norms(const double* v, const int32_t* idx, int64_t m, double* out, void* stream) {
  if (m <= 0) return 0;
  if (!v || !out) return 1;
  row_norm_kernel<<<blocks_for(m), 256, 0, (cudaStream_t)stream>>>(v, idx, m, out);
  return cudaGetLastError() == cudaSuccess ? 0 : 4;
}

int pab_density_dup_key(const double* gn, int64_t m, const double* t, double* key, void* stream) {
  if (m <= 0) return 0;
  if (!gn || !t || !key) return 1;
  dup_key_kernel<<<blocks_for(m), 256, 0, (cudaStream_t)stream>>>(gn, m, t, key);
  return cudaGetLastError() == cudaSuccess ? 0 : 4;
}

int pab_density_take_ties(const int32_t* ties, const int* n_ties, const int* n_above, int k_dup, int64_t m,
                          double* key, void* stream) {
  if (m <= 0 || k_dup <= 0) return 0;
  if (!ties || !n_ties || !n_above || !key) return 1;
  dup_take_ties_kernel<<<blocks_for(m), 256, 0, (cudaStream_t)stream>>>(ties, n_ties, n_above, k_dup, key);
  return cudaGetLastError() == cudaSuccess ? 0 : 4;
}

int pab_split_children(const double* pos, const double* p0, const double* a0, const double* unit, int64_t m,
                       double* out_pos, double* out_p0, double* out_a0, void* stream) {
  if (m <= 0) return 0;
  if (!pos || !p0 || !a0 || !unit || !out_pos || !out_p0 || !out_a0) return 1;
  split_children_kernel<<<blocks_for(m), 256, 0, (cudaStream_t)stream>>>(pos, p0, a0, unit, m, out_pos, out_p0,
                                                                          out_a0);
  return cudaGetLastError() == cudaSuccess ? 0 : 4;
}

int pab_duplicate(const double* pos, const double* p0, const double* a0, const double* unit, int64_t m,
                  double* out_pos, double* out_p0, double* out_a0, void* stream) {
  if (m <= 0) return 0;
  if (!pos || !p0 || !a0 || !unit || !out_pos || !out_p0 || !out_a0) return 1;
  duplicate_kernel<<<blocks_for(m), 256, 0, (cudaStream_t)stream>>>(pos, p0, a0, unit, m, out_pos, out_p0, out_a0);
  return cudaGetLastError() == cudaSuccess ? 0 : 4;
}

}  // extern "C"
