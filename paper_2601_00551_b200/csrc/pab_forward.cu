// Forward model and residual/loss epilogue (K4).
//
// Replaces reference radiator.py:185-261 (slab evaluation + np.bincount
// scatter) and :263-264 (residual, loss part).
//
// Decomposition: one CTA owns one detector row (all samples of the decimated
// grid, in shared memory) and a partition of the ball cells; a cell is C
// consecutive lane groups (32 Morton-ordered balls each).  A warp takes a
// cell, lane l evaluates ball l of every group of the cell over its own
// arrival window and read-modify-writes its private column of a per-warp
// tile [UT rows x 32 lanes] (lane l always hits bank l: conflict-free, no
// atomics).  The tile covers the cell's sample range; it is then reduced
// across lanes and merged into the CTA's row in cell order (a shared-memory
// ticket), so every sample is a fixed-order sum: results are bitwise
// reproducible run to run.  Partitions are summed in order by the epilogue.
#include <climits>

#include "pab_common.cuh"

namespace pab {

__device__ __forceinline__ int warp_min_i(int v) {
  for (int o = 16; o > 0; o >>= 1) v = min(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ int warp_max_i(int v) {
  for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

__device__ __forceinline__ void ticket_acquire(int* ticket, int seq, int lane) {
  if (lane == 0) {
    while (*((volatile int*)ticket) != seq) __nanosleep(32);
  }
  __syncwarp();
  __threadfence_block();
}

__device__ __forceinline__ void ticket_release(int* ticket, int seq, int lane) {
  __syncwarp();
  __threadfence_block();
  if (lane == 0) *((volatile int*)ticket) = seq + 1;
  __syncwarp();
}

constexpr int kMaxTileBlocks = 8;   // UT <= 256

__global__ void __launch_bounds__(256, 1)
forward_kernel(const BallA* __restrict__ ra, const BallB* __restrict__ rb,
               const GroupMeta* __restrict__ gmeta, int64_t n_groups,
               const double* __restrict__ det_pos, const double* __restrict__ det_aux, int n_det,
               Acq acq, int groups_per_cell, int64_t cells_per_part, int tile_rows,
               float* __restrict__ partial_rows, unsigned long long* __restrict__ ops_total,
               int* __restrict__ status) {
  extern __shared__ __align__(16) float smem[];
  const int n_out = acq.n_out;
  const int row_pad = (n_out + 3) & ~3;
  float* row = smem;
  float* tiles = smem + row_pad;
  const int nw = blockDim.x >> 5;
  int* ticket = reinterpret_cast<int*>(tiles + (size_t)nw * tile_rows * kWarp);

  const int j = blockIdx.x;
  const int part = blockIdx.y;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  for (int i = threadIdx.x; i < row_pad; i += blockDim.x) row[i] = 0.0f;
  for (int i = threadIdx.x; i < nw * tile_rows * kWarp; i += blockDim.x) tiles[i] = 0.0f;
  if (threadIdx.x == 0) *ticket = 0;
  __syncthreads();

  const Detector det = load_detector(det_pos, det_aux, j);
  float* tile = tiles + (size_t)warp * tile_rows * kWarp;
  const int C = groups_per_cell;
  const int64_t n_cells = (n_groups + C - 1) / C;
  const int64_t c_begin = (int64_t)part * cells_per_part;
  const int64_t c_end = min(n_cells, c_begin + cells_per_part);
  const int f = acq.f;

  unsigned long long my_ops = 0;
  int coinc = 0;
  int seq = warp;
  for (int64_t c = c_begin + warp; c < c_end; c += nw, seq += nw) {
    const int64_t g0 = c * C;
    const int ng = (int)min((int64_t)C, n_groups - g0);
    GroupMeta gm_l;
    GroupDet gd_l;
    int glo = INT_MAX, ghi = INT_MIN;
    if (lane < ng) {
      gm_l = gmeta[g0 + lane];
      gd_l = group_det(gm_l, det.px, det.py, det.pz, acq);
      group_range(acq, gd_l, gm_l, &glo, &ghi);
    } else {
      gd_l.Sx = gd_l.Sy = gd_l.Sz = 0.f; gd_l.Sn = 1.f; gd_l.isn = 1.f; gd_l.phg = 0.f;
      gd_l.kg = 0; gd_l.slow = 0;
    }
    const int clo = warp_min_i(glo), chi = warp_max_i(ghi);
    bool holding = false;
    for (int base = clo; base <= chi; base += tile_rows) {
      const int top = min(base + tile_rows - 1, chi);
      const bool first_pass = base == clo;
      for (int i = 0; i < ng; ++i) {
        const GroupDet g = shfl_gd(gd_l, i);
        GroupMeta gmi;
        if (g.slow) gmi = gmeta[g0 + i];
        const int64_t bi = (g0 + i) * kWarp + lane;
        const BallA A = ra[bi];
        const BallB B = rb[bi];
        const Pair p = make_pair(acq, g, gmi, det, A, B, false, nullptr, nullptr);
        if (first_pass) {
          my_ops += (unsigned long long)(max(p.jhi - p.jlo + 1, 0) + max(p.nhi - p.nlo + 1, 0));
          coinc |= p.coincident;
        }
        const float Ak = p.amp * A.a0 * kSqrt2Ln2;   // amp * kappa: u G amp = Ak * y G
        const float ps = p.phi * p.sc;
        {
          const int lo = max(p.jlo, base), hi = min(p.jhi, top);
          float mf = (float)(lo * f - p.kc);
          const float fs = (float)f;
          float* t = tile + (lo - base) * kWarp + lane;
          int J = lo;
#pragma unroll 1
          for (; J + 3 <= hi; J += 4, mf += 4.0f * fs, t += 4 * kWarp) {
            const float y0 = fmaf(mf, -p.sc, ps);
            const float y1 = fmaf(mf + fs, -p.sc, ps);
            const float y2 = fmaf(mf + 2.0f * fs, -p.sc, ps);
            const float y3 = fmaf(mf + 3.0f * fs, -p.sc, ps);
            const float G0 = ex2(-y0 * y0), G1 = ex2(-y1 * y1);
            const float G2 = ex2(-y2 * y2), G3 = ex2(-y3 * y3);
            t[0] = fmaf(Ak, y0 * G0, t[0]);
            t[kWarp] = fmaf(Ak, y1 * G1, t[kWarp]);
            t[2 * kWarp] = fmaf(Ak, y2 * G2, t[2 * kWarp]);
            t[3 * kWarp] = fmaf(Ak, y3 * G3, t[3 * kWarp]);
          }
          for (; J <= hi; ++J, mf += fs, t += kWarp) {
            const float y = fmaf(mf, -p.sc, ps);
            const float G = ex2(-y * y);
            *t = fmaf(Ak, y * G, *t);
          }
        }
        if (p.nlo <= p.nhi) {   // u+ term (near field): u = -kappa * y
          const int lo = max(p.nlo, base), hi = min(p.nhi, top);
          const float nps = p.nphi * p.sc;
          for (int J = lo; J <= hi; ++J) {
            const float y = fmaf((float)(J * f - p.nkc), -p.sc, nps);
            const float G = ex2(-y * y);
            float* t = tile + (J - base) * kWarp + lane;
            *t = fmaf(-Ak, y * G, *t);
          }
        }
      }
      // reduce the tile across lanes (rotated column order: conflict-free)
      const int len = top - base + 1;
      float sums[kMaxTileBlocks];
#pragma unroll
      for (int k = 0; k < kMaxTileBlocks; ++k) {
        sums[k] = 0.0f;
        if (k * kWarp < len) {
          float* trow = tile + (k * kWarp + lane) * kWarp;
          float s = 0.0f;
#pragma unroll 8
          for (int i = 0; i < kWarp; ++i) {
            const int col = (i + lane) & 31;
            s += trow[col];
            trow[col] = 0.0f;
          }
          sums[k] = s;
        }
      }
      if (!holding) { ticket_acquire(ticket, seq, lane); holding = true; }
#pragma unroll
      for (int k = 0; k < kMaxTileBlocks; ++k) {
        const int r = k * kWarp + lane;
        if (r < len) row[base + r] += sums[k];
      }
      __syncwarp();
    }
    if (!holding) ticket_acquire(ticket, seq, lane);
    ticket_release(ticket, seq, lane);
  }
  // warps whose cell sequence ended early must still let later cells through:
  // every seq in [0, n_cells_in_part) is released by exactly one warp above.
  __syncthreads();

  float* out = partial_rows + ((size_t)part * n_det + j) * (size_t)n_out;
  for (int i = threadIdx.x; i < n_out; i += blockDim.x) out[i] = row[i];

  // op count and coincidence flag
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
                                double* __restrict__ loss_rows) {
  const int j = blockIdx.x;
  double acc = 0.0;
  for (int k = threadIdx.x; k < n_out; k += blockDim.x) {
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

}  // namespace pab

using namespace pab;

static Acq make_acq(double v, double t0, double dt, int f, int n_out, double cutoff, int dir_kind,
                    double dir_param) {
  Acq a;
  a.vdt = v * dt;
  a.inv_vdt = 1.0 / a.vdt;
  a.vt0 = v * t0;
  a.f = f;
  a.n_out = n_out;
  a.cutoff = (float)cutoff;
  a.vdt_f = (float)a.vdt;
  a.inv_vdt_f = (float)a.inv_vdt;
  a.dir_kind = dir_kind;
  a.dir_param = (float)dir_param;
  return a;
}

extern "C" {

size_t pab_forward_smem_bytes(int n_out, int warps, int tile_rows) {
  const size_t row_pad = (size_t)((n_out + 3) & ~3);
  return (row_pad + (size_t)warps * tile_rows * kWarp) * sizeof(float) + 16;
}

int pab_forward(const void* rec_a, const void* rec_b, const void* group_meta, int64_t n_groups,
                const double* det_pos, const double* det_aux, int n_det, double v, double t0, double dt,
                int f, int n_out, double cutoff, int dir_kind, double dir_param, int groups_per_cell,
                int partitions, int warps, int tile_rows, float* partial_rows,
                unsigned long long* ops_total, int* status, void* stream) {
  if (n_det <= 0 || n_out <= 0) return 0;
  if (f < 1 || groups_per_cell < 1 || groups_per_cell > 32 || partitions < 1 || warps < 1 || warps > 8 ||
      tile_rows < 32 || tile_rows > 32 * kMaxTileBlocks || (tile_rows % 32) != 0)
    return 1;
  if (!rec_a || !rec_b || !group_meta || !det_pos || !det_aux || !partial_rows || !ops_total || !status)
    return 1;
  const Acq acq = make_acq(v, t0, dt, f, n_out, cutoff, dir_kind, dir_param);
  const int64_t n_cells = (n_groups + groups_per_cell - 1) / groups_per_cell;
  const int64_t per_part = (n_cells + partitions - 1) / partitions;
  const size_t smem = pab_forward_smem_bytes(n_out, warps, tile_rows);
  if (smem > 227 * 1024) return 1;
  cudaFuncSetAttribute(forward_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  dim3 grid((unsigned)n_det, (unsigned)partitions);
  forward_kernel<<<grid, warps * kWarp, smem, (cudaStream_t)stream>>>(
      (const BallA*)rec_a, (const BallB*)rec_b, (const GroupMeta*)group_meta, n_groups, det_pos, det_aux,
      n_det, acq, groups_per_cell, per_part, tile_rows, partial_rows, ops_total, status);
  return cudaGetLastError() == cudaSuccess ? 0 : 4;
}

int pab_residual(const float* partial_rows, int partitions, int n_det, int n_out, const float* real,
                 float* out, double* loss_rows, void* stream) {
  if (n_det <= 0 || n_out <= 0) return 0;
  if (!partial_rows || !out || partitions < 1) return 1;
  residual_kernel<<<n_det, 256, 0, (cudaStream_t)stream>>>(partial_rows, partitions, n_det, n_out, real,
                                                           out, loss_rows);
  return cudaGetLastError() == cudaSuccess ? 0 : 4;
}

int pab_decimate(const float* src, int n_rows, int n_in, int f, float* dst, void* stream) {
  if (f < 1 || n_rows < 0 || n_in < 0) return 1;
  const int n_out = (n_in + f - 1) / f;
  const int64_t total = (int64_t)n_rows * n_out;
  if (total == 0) return 0;
  decimate_kernel<<<(unsigned)((total + 255) / 256), 256, 0, (cudaStream_t)stream>>>(src, n_rows, n_in, f,
                                                                                    n_out, dst);
  return cudaGetLastError() == cudaSuccess ? 0 : 4;
}

}  // extern "C"
