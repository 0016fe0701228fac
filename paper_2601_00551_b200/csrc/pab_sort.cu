// Processing-order sort of a ball cloud, entirely on the
// device and without host round trips: cloud bounds -> Hilbert/radius keys
// -> stable LSD radix sort -> permutation.
//
// The reference visits balls in input order (radiator.py:185); the order here
// is a performance choice only (compact lane groups, equal window lengths),
// but it fixes the FP32 summation order, so it must be deterministic: the
// bounds are exact min/max reductions and the radix sort is stable.
//
// Keys (pab_morton_keys, pab_pack.cu): a0 bucket (4 bits) << 58 | hilbert30
// << 28 | index.  Indices ascend in input order and the sort is stable, so
// only bits [28, 63) need sorting: five 7-bit passes.
#include <algorithm>

#include "pab_common.cuh"

namespace pab {

constexpr int kSortThreads = 256;
constexpr int kSortRounds = 8;
constexpr int kSortTile = kSortThreads * kSortRounds;   // keys per block and pass
constexpr int kDigitBits = 7;
constexpr int kBins = 1 << kDigitBits;
constexpr int kSortLowBit = 28;                          // index bits below: already in order
constexpr int kSortPasses = (63 - kSortLowBit + kDigitBits - 1) / kDigitBits;
constexpr int kBoundsBlocks = 256;

// bounds[0..2] = min x, y, z; [3] = extent (max side of the bounding box, 1
// if degenerate); [4], [5] = min / max a0.  Block partials, then one block.
__global__ void bounds_partial_kernel(const double* __restrict__ pos, const double* __restrict__ a0, int64_t n,
                                      double* __restrict__ part) {
  double lo[4] = {INFINITY, INFINITY, INFINITY, INFINITY}, hi[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    for (int c = 0; c < 3; ++c) {
      const double v = pos[3 * i + c];
      lo[c] = fmin(lo[c], v);
      hi[c] = fmax(hi[c], v);
    }
    lo[3] = fmin(lo[3], a0[i]);
    hi[3] = fmax(hi[3], a0[i]);
  }
  __shared__ double s[8][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int c = 0; c < 4; ++c) {
    for (int o = 16; o > 0; o >>= 1) {
      lo[c] = fmin(lo[c], __shfl_xor_sync(0xffffffffu, lo[c], o));
      hi[c] = fmax(hi[c], __shfl_xor_sync(0xffffffffu, hi[c], o));
    }
  }
  if (lane == 0)
    for (int c = 0; c < 4; ++c) { s[c][warp] = lo[c]; s[4 + c][warp] = hi[c]; }
  __syncthreads();
  if (threadIdx.x < 8) {
    const int c = threadIdx.x;
    double v = s[c][0];
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) v = c < 4 ? fmin(v, s[c][w]) : fmax(v, s[c][w]);
    part[(size_t)blockIdx.x * 8 + c] = v;
  }
}

__global__ void bounds_final_kernel(const double* __restrict__ part, int nb, double* __restrict__ bounds) {
  __shared__ double r[8];
  const int c = threadIdx.x;   // one thread per component (min x, y, z, a0; max x, y, z, a0)
  if (c < 8) {
    double v = part[c];
    for (int b = 1; b < nb; ++b) v = c < 4 ? fmin(v, part[(size_t)b * 8 + c]) : fmax(v, part[(size_t)b * 8 + c]);
    r[c] = v;
  }
  __syncthreads();
  if (c == 0) {
    const double ext = fmax(fmax(r[4] - r[0], r[5] - r[1]), r[6] - r[2]);
    bounds[0] = r[0];
    bounds[1] = r[1];
    bounds[2] = r[2];
    bounds[3] = ext > 0.0 ? ext : 1.0;
    bounds[4] = r[3];
    bounds[5] = r[7];
  }
}

__global__ void radix_hist_kernel(const unsigned long long* __restrict__ keys, int64_t n, int shift,
                                  int* __restrict__ counts, int nb) {
  __shared__ int h[kBins];
  for (int i = threadIdx.x; i < kBins; i += blockDim.x) h[i] = 0;
  __syncthreads();
  const int64_t base = (int64_t)blockIdx.x * kSortTile;
  for (int r = 0; r < kSortRounds; ++r) {
    const int64_t i = base + r * kSortThreads + threadIdx.x;
    if (i < n) atomicAdd(&h[(int)(keys[i] >> shift) & (kBins - 1)], 1);   // counts only: order-free
  }
  __syncthreads();
  for (int b = threadIdx.x; b < kBins; b += blockDim.x) counts[(size_t)b * nb + blockIdx.x] = h[b];
}

// Exclusive scan of m ints in place by one block: each thread scans a
// contiguous segment, the 1024 segment totals are scanned in shared memory.
__global__ void radix_scan_kernel(int* __restrict__ a, int m) {
  __shared__ int tot[1024];
  const int t = threadIdx.x;
  const int seg = (m + 1023) / 1024;
  const int s0 = min(m, t * seg), s1 = min(m, s0 + seg);
  int sum = 0;
  for (int i = s0; i < s1; ++i) sum += a[i];
  tot[t] = sum;
  __syncthreads();
  for (int off = 1; off < 1024; off <<= 1) {
    const int y = t >= off ? tot[t - off] : 0;
    __syncthreads();
    tot[t] += y;
    __syncthreads();
  }
  int run = tot[t] - sum;
  for (int i = s0; i < s1; ++i) {
    const int x = a[i];
    a[i] = run;
    run += x;
  }
}

__device__ __forceinline__ unsigned lanemask_lt_sort() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// Stable scatter of one 7-bit digit: keys of a block are visited in input
// order (round r covers tile positions [256 r, 256 r + 256)); a key's rank is
// the number of equal digits before it: earlier rounds (run), earlier warps
// of this round (wc) and earlier lanes of its warp (match_any).  The last
// pass writes the permutation (the key's low 28 bits) instead of the key.
__global__ void radix_scatter_kernel(const unsigned long long* __restrict__ kin, unsigned long long* __restrict__ kout,
                                     int64_t n, int shift, const int* __restrict__ offsets, int nb,
                                     int32_t* __restrict__ perm) {
  constexpr int W = kSortThreads / 32;
  __shared__ int run[kBins];
  __shared__ int wc[W][kBins];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int b = tid; b < kBins; b += kSortThreads) run[b] = 0;
  const int64_t base = (int64_t)blockIdx.x * kSortTile;
  for (int r = 0; r < kSortRounds; ++r) {
    for (int b = lane; b < kBins; b += 32) wc[warp][b] = 0;
    __syncwarp();
    const int64_t i = base + r * kSortThreads + tid;
    const bool valid = i < n;
    const unsigned long long key = valid ? kin[i] : 0ull;
    const int d = valid ? (int)(key >> shift) & (kBins - 1) : -1;
    const unsigned mask = __match_any_sync(0xffffffffu, d);
    const int rank = __popc(mask & lanemask_lt_sort());
    if (valid && rank == 0) wc[warp][d] = __popc(mask);
    __syncthreads();
    if (valid) {
      int pre = run[d] + rank;
      for (int w = 0; w < warp; ++w) pre += wc[w][d];
      const int64_t pos = (int64_t)offsets[(size_t)d * nb + blockIdx.x] + pre;
      if (perm) perm[pos] = (int32_t)(key & 0xFFFFFFFull);
      else kout[pos] = key;
    }
    __syncthreads();
    for (int b = tid; b < kBins; b += kSortThreads) {
      int s = 0;
      for (int w = 0; w < W; ++w) s += wc[w][b];
      run[b] += s;
    }
    __syncthreads();
  }
}

// ---- lane-group segmentation of the sorted order -------------------------
// Consecutive balls of the sorted order form lane groups of 32.  In a sparse
// cloud (a filtered reconstruction: balls along vessels) 32 consecutive
// Hilbert-order balls can straddle a jump between distant structures, and
// a wide group spans more samples than the forward's tile (it then takes
// the serial path) and stages a long residual segment in the adjoint.  A
// new group therefore starts wherever the sorted order crosses a radius
// bucket or jumps farther than `gap`; segments are padded to whole groups
// with inert slots (-1).

__device__ __forceinline__ int a0_bucket(double a, const double* bounds, int nbuckets, double log_span) {
  const double a0lo = bounds[4], a0hi = bounds[5];
  if (nbuckets <= 1 || !(a0hi > a0lo)) return 0;
  if (log_span > 0.0) {
    const double llo = log2(fmax(a0lo, a0hi * exp2(-log_span))), lhi = log2(a0hi);
    const double x = lhi > llo ? (log2(a) - llo) / (lhi - llo) : 0.0;
    return (int)fmin(fmax(x * nbuckets, 0.0), (double)(nbuckets - 1));
  }
  return (int)fmin(fmax((a - a0lo) / (a0hi - a0lo) * nbuckets, 0.0), (double)(nbuckets - 1));
}

__global__ void segment_flags_kernel(const double* __restrict__ pos, const double* __restrict__ a0,
                                     const int32_t* __restrict__ perm, int64_t n, const double* __restrict__ bounds,
                                     int nbuckets, double log_span, double gap2, int* __restrict__ flags) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  int f = 1;
  if (k > 0) {
    const int64_t b = perm[k], c = perm[k - 1];
    const double dx = pos[3 * b] - pos[3 * c], dy = pos[3 * b + 1] - pos[3 * c + 1], dz = pos[3 * b + 2] - pos[3 * c + 2];
    f = (dx * dx + dy * dy + dz * dz > gap2) ||
        a0_bucket(a0[b], bounds, nbuckets, log_span) != a0_bucket(a0[c], bounds, nbuckets, log_span);
  }
  flags[k] = f;
}

// inclusive scan of ints, 1024 per block (warp shuffles), block totals out
__global__ void scan_block_kernel(int* __restrict__ a, int64_t m, int* __restrict__ totals) {
  __shared__ int wsum[32];
  const int64_t i = (int64_t)blockIdx.x * 1024 + threadIdx.x;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int x = i < m ? a[i] : 0;
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) wsum[w] = x;
  __syncthreads();
  if (w == 0) {
    int t = wsum[lane];
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t += y;
    }
    wsum[lane] = t;
  }
  __syncthreads();
  if (w > 0) x += wsum[w - 1];
  if (i < m) a[i] = x;
  if (threadIdx.x == 1023) totals[blockIdx.x] = x;
}

__global__ void scan_add_kernel(int* __restrict__ a, int64_t m, const int* __restrict__ offsets) {
  const int64_t i = (int64_t)blockIdx.x * 1024 + threadIdx.x;
  if (i < m && blockIdx.x > 0) a[i] += offsets[blockIdx.x];
}

// sid (inclusive scan of the flags) -> start index of every segment
__global__ void segment_starts_kernel(const int* __restrict__ flags, const int* __restrict__ sid, int64_t n,
                                      int* __restrict__ start) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n && (k == 0 || sid[k] != sid[k - 1])) start[sid[k] - 1] = (int)k;
  (void)flags;
}

// 1 where a ball opens a lane group (every 32nd ball of its segment)
__global__ void group_opens_kernel(const int* __restrict__ sid, const int* __restrict__ start, int64_t n,
                                   int* __restrict__ open) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n) open[k] = ((k - start[sid[k] - 1]) & 31) == 0;
}

// gid (inclusive scan of the opens) -> slot of every ball; n_groups out
__global__ void group_slots_kernel(const int32_t* __restrict__ perm, const int* __restrict__ sid,
                                   const int* __restrict__ start, const int* __restrict__ gid, int64_t n,
                                   int32_t* __restrict__ slots, int* __restrict__ n_groups) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  slots[(int64_t)(gid[k] - 1) * 32 + ((k - start[sid[k] - 1]) & 31)] = perm[k];
  if (k == n - 1 && n_groups) *n_groups = gid[k];
}

__global__ void fill_i32_kernel(int32_t* __restrict__ a, int64_t m, int32_t v) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < m) a[i] = v;
}

}  // namespace pab

using namespace pab;

extern "C" {

size_t pab_cloud_bounds_workspace_bytes(void) { return (size_t)kBoundsBlocks * 8 * sizeof(double); }

int pab_cloud_bounds(const double* pos, const double* a0, int64_t n, double* bounds, void* workspace, void* stream) {
  if (n <= 0) return 0;
  if (!pos || !a0 || !bounds || !workspace) return 1;
  const cudaStream_t s = (cudaStream_t)stream;
  const int nb = (int)std::min<int64_t>(kBoundsBlocks, (n + 255) / 256);
  bounds_partial_kernel<<<nb, 256, 0, s>>>(pos, a0, n, (double*)workspace);
  bounds_final_kernel<<<1, 32, 0, s>>>((const double*)workspace, nb, bounds);
  return cudaGetLastError() == cudaSuccess ? 0 : 4;
}

size_t pab_sort_perm_workspace_bytes(int64_t n) {
  const int64_t nb = (n + kSortTile - 1) / kSortTile;
  return (size_t)n * sizeof(unsigned long long) + (size_t)kBins * nb * sizeof(int) + 256;
}

int pab_sort_perm(int64_t* keys, int64_t n, int32_t* perm, void* workspace, void* stream) {
  if (n <= 0) return 0;
  if (!keys || !perm || !workspace || n > (1ll << 28)) return 1;
  const cudaStream_t s = (cudaStream_t)stream;
  const int nb = (int)((n + kSortTile - 1) / kSortTile);
  unsigned long long* a = reinterpret_cast<unsigned long long*>(keys);
  unsigned long long* b = reinterpret_cast<unsigned long long*>(workspace);
  int* counts = reinterpret_cast<int*>(b + n);
  for (int p = 0; p < kSortPasses; ++p) {
    const int shift = kSortLowBit + p * kDigitBits;
    radix_hist_kernel<<<nb, kSortThreads, 0, s>>>(a, n, shift, counts, nb);
    radix_scan_kernel<<<1, 1024, 0, s>>>(counts, kBins * nb);
    const bool last = p == kSortPasses - 1;
    radix_scatter_kernel<<<nb, kSortThreads, 0, s>>>(a, b, n, shift, counts, nb, last ? perm : nullptr);
    if (!last) std::swap(a, b);
  }
  return cudaGetLastError() == cudaSuccess ? 0 : 4;
}

// In-place inclusive scan of m ints (3 launches); workspace >= 2 (m / 1024 + 2) ints.
static void scan_inclusive(int* a, int64_t m, int* ws, cudaStream_t s) {
  const int64_t nb = (m + 1023) / 1024;
  scan_block_kernel<<<(unsigned)nb, 1024, 0, s>>>(a, m, ws);
  if (nb > 1) {
    radix_scan_kernel<<<1, 1024, 0, s>>>(ws, (int)nb);   // exclusive: offsets of the blocks
    scan_add_kernel<<<(unsigned)nb, 1024, 0, s>>>(a, m, ws);
  }
}

size_t pab_group_slots_workspace_bytes(int64_t n) {
  return (size_t)(4 * n + 2 * ((n + 1023) / 1024 + 2)) * sizeof(int) + 256;
}

int pab_group_slots(const double* pos, const double* a0, const int32_t* perm, int64_t n, const double* bounds,
                    int a0_buckets, double log_span, double gap, int* n_groups, void* workspace, void* stream) {
  if (n <= 0) return 0;
  if (!pos || !a0 || !perm || !bounds || !n_groups || !workspace || n > (1ll << 28) || a0_buckets < 1 ||
      a0_buckets > 16 || log_span < 0.0 || !(gap > 0.0))
    return 1;
  const cudaStream_t s = (cudaStream_t)stream;
  int* flags = static_cast<int*>(workspace);   // -> sid after the scan
  int* start = flags + n;
  int* open = start + n;                        // -> gid after the scan
  int* ws = open + n;
  const unsigned blocks = (unsigned)((n + 255) / 256);
  segment_flags_kernel<<<blocks, 256, 0, s>>>(pos, a0, perm, n, bounds, a0_buckets, log_span, gap * gap, flags);
  scan_inclusive(flags, n, ws, s);
  segment_starts_kernel<<<blocks, 256, 0, s>>>(flags, flags, n, start);
  group_opens_kernel<<<blocks, 256, 0, s>>>(flags, start, n, open);
  scan_inclusive(open, n, ws, s);
  cudaMemcpyAsync(n_groups, open + (n - 1), sizeof(int), cudaMemcpyDeviceToDevice, s);
  return cudaGetLastError() == cudaSuccess ? 0 : 4;
}

int pab_group_slots_scatter(const int32_t* perm, int64_t n, int64_t n_groups, const void* workspace,
                            int32_t* slots, void* stream) {
  if (n <= 0) return 0;
  if (!perm || !workspace || !slots || n_groups < 1) return 1;
  const cudaStream_t s = (cudaStream_t)stream;
  const int* sid = static_cast<const int*>(workspace);
  const int* start = sid + n;
  const int* gid = start + n;
  const int64_t m = n_groups * 32;
  fill_i32_kernel<<<(unsigned)((m + 255) / 256), 256, 0, s>>>(slots, m, -1);
  group_slots_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(perm, sid, start, gid, n, slots, nullptr);
  return cudaGetLastError() == cudaSuccess ? 0 : 4;
}

}  // extern "C"
