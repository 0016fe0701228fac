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

// Per-digit exclusive scans of the block counts: counts[d * nb + b] is
// digit d's count in block b; warp d scans its digit's column in place and
// writes the digit total.  The scatter adds the digit bases (an exclusive
// scan of the kBins totals, done by every scatter block in shared memory).
// (Round 1 scanned all kBins * nb counts in one block: ~52 us per pass at 1M
// keys, the sort's largest cost.)
__global__ void radix_scan_kernel(int* __restrict__ counts, int nb, int* __restrict__ totals) {
  const int d = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (d >= kBins) return;
  int* col = counts + (size_t)d * nb;
  int carry = 0;
  for (int b0 = 0; b0 < nb; b0 += 32) {
    const int b = b0 + lane;
    const int x = b < nb ? col[b] : 0;
    int incl = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    if (b < nb) col[b] = carry + incl - x;
    carry += __shfl_sync(0xffffffffu, incl, 31);
  }
  if (lane == 0) totals[d] = carry;
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
                                     const int* __restrict__ totals, int32_t* __restrict__ perm) {
  constexpr int W = kSortThreads / 32;
  static_assert(kBins <= kSortThreads && kBins % 32 == 0, "one thread per digit base");
  __shared__ int run[kBins];
  __shared__ int wc[W][kBins];
  __shared__ int wt[kBins / 32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // run[d] starts at digit d's base: exclusive scan of the digit totals
  if (tid < kBins) {
    const int x = totals[tid];
    int incl = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) wt[warp] = incl;
    run[tid] = incl - x;
  }
  __syncthreads();
  if (tid < kBins)
    for (int w = 0; w < warp; ++w) run[tid] += wt[w];
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
  return (size_t)n * sizeof(unsigned long long) + (size_t)kBins * nb * sizeof(int) + kBins * sizeof(int) + 256;
}

int pab_sort_perm(int64_t* keys, int64_t n, int32_t* perm, void* workspace, void* stream) {
  if (n <= 0) return 0;
  if (!keys || !perm || !workspace || n > (1ll << 28)) return 1;
  const cudaStream_t s = (cudaStream_t)stream;
  const int nb = (int)((n + kSortTile - 1) / kSortTile);
  unsigned long long* a = reinterpret_cast<unsigned long long*>(keys);
  unsigned long long* b = reinterpret_cast<unsigned long long*>(workspace);
  int* counts = reinterpret_cast<int*>(b + n);
  int* totals = counts + (size_t)kBins * nb;
  for (int p = 0; p < kSortPasses; ++p) {
    const int shift = kSortLowBit + p * kDigitBits;
    radix_hist_kernel<<<nb, kSortThreads, 0, s>>>(a, n, shift, counts, nb);
    radix_scan_kernel<<<kBins / 4, 128, 0, s>>>(counts, nb, totals);
    const bool last = p == kSortPasses - 1;
    radix_scatter_kernel<<<nb, kSortThreads, 0, s>>>(a, b, n, shift, counts, nb, totals, last ? perm : nullptr);
    if (!last) std::swap(a, b);
  }
  return cudaGetLastError() == cudaSuccess ? 0 : 4;
}

}  // extern "C"
