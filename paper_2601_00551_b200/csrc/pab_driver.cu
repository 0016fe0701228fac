// Iteration-driver kernels: Adam and stable compaction
// (K5) used by the zero-gradient filter and the destroy rule.
//
// Adam replaces reference optimizer.py:203-209 and :295-304; it evaluates the
// same IEEE double expression tree as numpy (explicit round-to-nearest
// intrinsics, no FMA contraction), so for identical gradients it produces
// bit-identical parameters and moments.
//
// Compaction replaces PointCloud.subset(mask) (model.py:239-244) as used by
// optimizer.py:255-256 and :331-345: warp ballot + popc ranks inside a
// block, an exclusive scan of block counts, then an order-preserving scatter.
#include "pab_common.cuh"

namespace pab {

__global__ void adam_kernel(double* __restrict__ param, const double* __restrict__ grad,
                            double* __restrict__ m, double* __restrict__ v, int64_t count, double lr,
                            double bc1, double bc2, double floor_value, int use_floor) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count) return;
  const double b1 = 0.9, b2 = 0.999, eps = 1e-8;
  const double g = grad[i];
  // m = b1*m + (1-b1)*g ;  v = b2*v + ((1-b2)*g)*g   (numpy evaluation order)
  const double mi = __dadd_rn(__dmul_rn(b1, m[i]), __dmul_rn(__dadd_rn(1.0, -b1), g));
  const double vi = __dadd_rn(__dmul_rn(b2, v[i]), __dmul_rn(__dmul_rn(__dadd_rn(1.0, -b2), g), g));
  m[i] = mi;
  v[i] = vi;
  const double mhat = __ddiv_rn(mi, bc1);
  const double vhat = __ddiv_rn(vi, bc2);
  const double upd = __ddiv_rn(__dmul_rn(lr, mhat), __dadd_rn(__dsqrt_rn(vhat), eps));
  double out = __dadd_rn(param[i], -upd);
  if (use_floor && !(out >= floor_value)) out = (out != out) ? out : floor_value;   // np.maximum
  param[i] = out;
}

// softplus(x) = log1p(exp(-|x|)) + max(x, 0)   (optimizer.py:507-510, same op tree)
__global__ void softplus_kernel(const double* __restrict__ x, int64_t n, double* __restrict__ y) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double v = x[i];
  y[i] = __dadd_rn(log1p(exp(-fabs(v))), v > 0.0 ? v : 0.0);
}

// out = g * sigmoid(x), sigmoid split by sign as optimizer.py:526-533
__global__ void mul_sigmoid_kernel(const double* __restrict__ g, const double* __restrict__ x, int64_t n,
                                   double* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double v = x[i];
  double s;
  if (v >= 0.0) {
    s = __ddiv_rn(1.0, __dadd_rn(1.0, exp(-v)));
  } else {
    const double e = exp(v);
    s = __ddiv_rn(e, __dadd_rn(1.0, e));
  }
  out[i] = __dmul_rn(g[i], s);
}

// flags: keep = (x < 0) if strict else (x <= 0)  [mode 0/1], x != 0 [mode 2],
// x > 0 [mode 3], x == 0 [mode 4]
__device__ __forceinline__ bool keep_pred(double x, int mode) {
  switch (mode) {
    case 0: return x < 0.0;
    case 1: return x <= 0.0;
    case 2: return x != 0.0;
    case 3: return x > 0.0;
    default: return x == 0.0;
  }
}

constexpr int kCompactBlock = 1024;

__global__ void compact_count_kernel(const double* __restrict__ key, int64_t n, int mode,
                                     int* __restrict__ block_counts) {
  __shared__ int wc[32];
  const int64_t i = (int64_t)blockIdx.x * kCompactBlock + threadIdx.x;
  const bool k = i < n && keep_pred(key[i], mode);
  const unsigned bal = __ballot_sync(0xffffffffu, k);
  if ((threadIdx.x & 31) == 0) wc[threadIdx.x >> 5] = __popc(bal);
  __syncthreads();
  if (threadIdx.x == 0) {
    int s = 0;
    for (int w = 0; w < kCompactBlock / 32; ++w) s += wc[w];
    block_counts[blockIdx.x] = s;
  }
}

__global__ void compact_scan_kernel(int* __restrict__ block_counts, int nb, int* __restrict__ total) {
  // single block, sequential chunks of the count array: exclusive scan in place
  __shared__ int carry;
  __shared__ int buf[1024];
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int b0 = 0; b0 < nb; b0 += 1024) {
    const int i = b0 + threadIdx.x;
    const int x = i < nb ? block_counts[i] : 0;
    buf[threadIdx.x] = x;
    __syncthreads();
    for (int off = 1; off < 1024; off <<= 1) {
      const int y = threadIdx.x >= off ? buf[threadIdx.x - off] : 0;
      __syncthreads();
      buf[threadIdx.x] += y;
      __syncthreads();
    }
    if (i < nb) block_counts[i] = carry + buf[threadIdx.x] - x;
    __syncthreads();
    if (threadIdx.x == 0) carry += buf[1023];
    __syncthreads();
  }
  if (threadIdx.x == 0) *total = carry;
}

__global__ void compact_scatter_kernel(const double* __restrict__ key, int64_t n, int mode,
                                       const int* __restrict__ block_offsets, int32_t* __restrict__ idx_out) {
  __shared__ int woff[32];
  const int64_t i = (int64_t)blockIdx.x * kCompactBlock + threadIdx.x;
  const bool k = i < n && keep_pred(key[i], mode);
  const unsigned bal = __ballot_sync(0xffffffffu, k);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) woff[w] = __popc(bal);
  __syncthreads();
  if (threadIdx.x == 0) {
    int s = 0;
    for (int q = 0; q < kCompactBlock / 32; ++q) { const int c = woff[q]; woff[q] = s; s += c; }
  }
  __syncthreads();
  if (k) {
    const int rank = __popc(bal & ((1u << lane) - 1u));
    idx_out[block_offsets[blockIdx.x] + woff[w] + rank] = (int32_t)i;
  }
}

__global__ void gather_f64_kernel(const double* __restrict__ src, int width, const int32_t* __restrict__ idx,
                                  int64_t m, double* __restrict__ dst) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= m * width) return;
  const int64_t r = t / width, c = t % width;
  dst[t] = src[(int64_t)idx[r] * width + c];
}

// Sum of squared differences in FP64 (reference loss(), radiator.py:393-402):
// fixed-size chunks per block, fixed-shape trees -> bitwise reproducible.
constexpr int kSsdBlock = 256;
constexpr int kSsdChunk = 8192;

__global__ void ssd_partial_kernel(const double* __restrict__ a, const double* __restrict__ b, int64_t n,
                                   double* __restrict__ partial) {
  __shared__ double red[kSsdBlock / 32];
  const int64_t c0 = (int64_t)blockIdx.x * kSsdChunk;
  const int64_t c1 = min(n, c0 + kSsdChunk);
  double acc = 0.0;
  for (int64_t i = c0 + threadIdx.x; i < c1; i += kSsdBlock) {
    const double d = a[i] - (b ? b[i] : 0.0);
    acc += d * d;
  }
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < kSsdBlock / 32; ++w) s += red[w];
    partial[blockIdx.x] = s;
  }
}

__global__ void sum_ordered_kernel(const double* __restrict__ partial, int np, double* __restrict__ out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double s = 0.0;
    for (int i = 0; i < np; ++i) s += partial[i];
    *out = s;
  }
}

// Per-pass tail of the gradient buffer (one all-reduce carries gradients,
// loss, error flags and the op count across detector shards): the loss rows
// summed in row order by one warp (fixed lane-strided partials, fixed
// shuffle tree: bitwise reproducible), the status bits as 0/1 counts and the
// op counter as a double (exact below 2^53).
__global__ void pass_tail_kernel(const double* __restrict__ loss_rows, int n_rows,
                                 const unsigned long long* __restrict__ ops, const int* __restrict__ status,
                                 double* __restrict__ tail) {
  const int lane = threadIdx.x;
  double acc = 0.0;
  if (loss_rows)
    for (int i = lane; i < n_rows; i += 32) acc += loss_rows[i];
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) {
    const int st = status ? *status : 0;
    tail[0] = acc;
    tail[1] = (st & kStatusCoincident) ? 1.0 : 0.0;
    tail[2] = (st & kStatusNonFinite) ? 1.0 : 0.0;
    tail[3] = ops ? (double)*ops : 0.0;
  }
}

}  // namespace pab

using namespace pab;

extern "C" {

int pab_adam(double* param, const double* grad, double* m, double* v, int64_t count, double lr, double bc1,
             double bc2, double floor_value, int use_floor, void* stream) {
  if (count <= 0) return 0;
  if (!param || !grad || !m || !v) return 1;
  adam_kernel<<<(unsigned)((count + 255) / 256), 256, 0, (cudaStream_t)stream>>>(param, grad, m, v, count, lr,
                                                                                bc1, bc2, floor_value, use_floor);
  return cudaGetLastError() == cudaSuccess ? 0 : 4;
}

int pab_softplus_f64(const double* x, int64_t n, double* y, void* stream) {
  if (n <= 0) return 0;
  if (!x || !y) return 1;
  softplus_kernel<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(x, n, y);
  return cudaGetLastError() == cudaSuccess ? 0 : 4;
}

int pab_mul_sigmoid_f64(const double* g, const double* x, int64_t n, double* out, void* stream) {
  if (n <= 0) return 0;
  if (!g || !x || !out) return 1;
  mul_sigmoid_kernel<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(g, x, n, out);
  return cudaGetLastError() == cudaSuccess ? 0 : 4;
}

size_t pab_compact_workspace_bytes(int64_t n) {
  return (size_t)(((n + kCompactBlock - 1) / kCompactBlock) + 1) * sizeof(int);
}

// Writes kept indices (ascending) to idx_out and their number to *count_dev.
int pab_compact(const double* key, int64_t n, int mode, int32_t* idx_out, int* count_dev, void* workspace,
                void* stream) {
  if (n <= 0) return 0;
  if (!key || !idx_out || !count_dev || !workspace || mode < 0 || mode > 4) return 1;
  const int nb = (int)((n + kCompactBlock - 1) / kCompactBlock);
  int* counts = (int*)workspace;
  const cudaStream_t s = (cudaStream_t)stream;
  compact_count_kernel<<<nb, kCompactBlock, 0, s>>>(key, n, mode, counts);
  compact_scan_kernel<<<1, 1024, 0, s>>>(counts, nb, count_dev);
  compact_scatter_kernel<<<nb, kCompactBlock, 0, s>>>(key, n, mode, counts, idx_out);
  return cudaGetLastError() == cudaSuccess ? 0 : 4;
}

int pab_gather_f64(const double* src, int width, const int32_t* idx, int64_t m, double* dst, void* stream) {
  if (m <= 0) return 0;
  if (!src || !idx || !dst || width < 1) return 1;
  const int64_t total = m * width;
  gather_f64_kernel<<<(unsigned)((total + 255) / 256), 256, 0, (cudaStream_t)stream>>>(src, width, idx, m, dst);
  return cudaGetLastError() == cudaSuccess ? 0 : 4;
}

size_t pab_sumsq_workspace_bytes(int64_t n) {
  return (size_t)((n + kSsdChunk - 1) / kSsdChunk + 1) * sizeof(double);
}

// *out = sum_i (a[i] - b[i])^2 (b nullable), FP64, deterministic order.
int pab_sumsq_diff_f64(const double* a, const double* b, int64_t n, double* out, void* workspace, void* stream) {
  if (!a || !out || !workspace || n < 0) return 1;
  const cudaStream_t s = (cudaStream_t)stream;
  const int nb = (int)((n + kSsdChunk - 1) / kSsdChunk);
  if (nb == 0) {
    cudaMemsetAsync(out, 0, sizeof(double), s);
    return cudaGetLastError() == cudaSuccess ? 0 : 4;
  }
  ssd_partial_kernel<<<nb, kSsdBlock, 0, s>>>(a, b, n, (double*)workspace);
  sum_ordered_kernel<<<1, 32, 0, s>>>((const double*)workspace, nb, out);
  return cudaGetLastError() == cudaSuccess ? 0 : 4;
}

int pab_pass_tail(const double* loss_rows, int n_rows, const unsigned long long* ops, const int* status,
                  double* tail, void* stream) {
  if (!tail || n_rows < 0) return 1;
  pass_tail_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(loss_rows, n_rows, ops, status, tail);
  return cudaGetLastError() == cudaSuccess ? 0 : 4;
}

int pab_version(void) { return 100; }

int pab_device_info(int device, int* sm_count, int* cc_major, int* cc_minor, int* max_smem_optin) {
  cudaDeviceProp p;
  if (cudaGetDeviceProperties(&p, device) != cudaSuccess) return 4;
  *sm_count = p.multiProcessorCount;
  *cc_major = p.major;
  *cc_minor = p.minor;
  *max_smem_optin = (int)p.sharedMemPerBlockOptin;
  return 0;
}

const char* pab_last_cuda_error(void) { return cudaGetErrorString(cudaGetLastError()); }

}  // extern "C"
