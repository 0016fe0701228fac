// Universal back-projection baseline.
//
// Replaces reference baseline.py:52-89 (`ubp_reconstruct`): for every voxel
// x, b(x) = (1/J) sum_j [2 p_j(t) - 2 t dp_j/dt] at t = |x - r_j| / v, linear
// interpolation in time, central-difference derivative (np.gradient), travel
// times outside the record skipped and counted.
//
// B200 form: one thread per voxel (FP64, the reference's expression tree with
// no FMA contraction), detectors visited in order; the FP64 signal rows and
// their derivative rows (33 MB each at 1024 x 4096) stream through L2.  Deterministic: the per-voxel sum
// runs over detectors in index order; the skipped count is an integer sum.
#include <cstdint>

#include <cuda_runtime.h>

namespace pab {

// np.gradient(data, dt, axis=1), edge_order 1 (numpy function_base.py):
// interior (f[i+1] - f[i-1]) / (2 dt), ends one-sided / dt.
__global__ void ubp_gradient_kernel(const double* __restrict__ p, int n_rows, int n, double dt,
                                    double* __restrict__ d) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (int64_t)n_rows * n) return;
  const int64_t r = i / n;
  const int k = (int)(i % n);
  const double* row = p + r * n;
  double v;
  if (n < 2) v = 0.0;
  else if (k == 0) v = __ddiv_rn(__dsub_rn(row[1], row[0]), dt);
  else if (k == n - 1) v = __ddiv_rn(__dsub_rn(row[n - 1], row[n - 2]), dt);
  else v = __ddiv_rn(__dsub_rn(row[k + 1], row[k - 1]), __dmul_rn(2.0, dt));
  d[i] = v;
}

__global__ void ubp_kernel(const double* __restrict__ p, const double* __restrict__ d,
                           const double* __restrict__ det, int n_det, int n, double t0, double dt, double v,
                           int nx, int ny, int nz, double sp, double ox, double oy, double oz,
                           double* __restrict__ vol, unsigned long long* __restrict__ skipped) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t nvox = (int64_t)nx * ny * nz;
  unsigned long long my_skip = 0;
  if (idx < nvox) {
    const int iz = (int)(idx % nz), iy = (int)((idx / nz) % ny), ix = (int)(idx / ((int64_t)ny * nz));
    // axis_centers: origin + arange * spacing (model.py:399-400)
    const double cx = __dadd_rn(ox, __dmul_rn((double)ix, sp));
    const double cy = __dadd_rn(oy, __dmul_rn((double)iy, sp));
    const double cz = __dadd_rn(oz, __dmul_rn((double)iz, sp));
    const double w = __ddiv_rn(1.0, (double)n_det);
    double acc = 0.0;
    for (int j = 0; j < n_det; ++j) {
      const double ex = __dsub_rn(cx, det[3 * j]), ey = __dsub_rn(cy, det[3 * j + 1]), ez = __dsub_rn(cz, det[3 * j + 2]);
      const double dist = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(ex, ex), __dmul_rn(ey, ey)), __dmul_rn(ez, ez)));
      const double tt = __ddiv_rn(dist, v);
      const double pos = __ddiv_rn(__dsub_rn(tt, t0), dt);
      const bool ok = pos >= 0.0 && pos <= (double)(n - 1);
      my_skip += ok ? 0ull : 1ull;
      double fl = floor(pos);
      int i0 = fl < 0.0 ? 0 : (fl > (double)(n - 2) ? n - 2 : (int)fl);
      double frac = __dsub_rn(pos, (double)i0);
      frac = frac < 0.0 ? 0.0 : (frac > 1.0 ? 1.0 : frac);
      const double* pr = p + (int64_t)j * n;
      const double* dr = d + (int64_t)j * n;
      const double om = __dsub_rn(1.0, frac);
      const double p_t = __dadd_rn(__dmul_rn(pr[i0], om), __dmul_rn(pr[i0 + 1], frac));
      const double d_t = __dadd_rn(__dmul_rn(dr[i0], om), __dmul_rn(dr[i0 + 1], frac));
      // w * (2 p_t - 2 tt d_t)
      const double term = __dmul_rn(w, __dsub_rn(__dmul_rn(2.0, p_t), __dmul_rn(__dmul_rn(2.0, tt), d_t)));
      acc = __dadd_rn(acc, ok ? term : 0.0);
    }
    vol[idx] = acc;
  }
  for (int o = 16; o > 0; o >>= 1) my_skip += __shfl_xor_sync(0xffffffffu, my_skip, o);
  if ((threadIdx.x & 31) == 0 && my_skip) atomicAdd(skipped, my_skip);
}

}  // namespace pab

using namespace pab;

extern "C" {

int pab_ubp(const double* signals, int n_det, int n_samples, double t0, double dt, const double* det_pos,
            double sound_speed, int nx, int ny, int nz, double spacing, double ox, double oy, double oz,
            double* deriv_scratch, double* vol, unsigned long long* skipped, void* stream) {
  if (nx <= 0 || ny <= 0 || nz <= 0) return 1;
  if (!vol || !skipped || (n_det > 0 && (!signals || !det_pos || !deriv_scratch))) return 1;
  if (n_det > 0 && n_samples < 2) return 1;
  const cudaStream_t s = (cudaStream_t)stream;
  const int64_t nvox = (int64_t)nx * ny * nz;
  if (n_det == 0) {
    cudaMemsetAsync(vol, 0, sizeof(double) * nvox, s);
    return cudaGetLastError() == cudaSuccess ? 0 : 4;
  }
  const int64_t tot = (int64_t)n_det * n_samples;
  ubp_gradient_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, s>>>(signals, n_det, n_samples, dt, deriv_scratch);
  ubp_kernel<<<(unsigned)((nvox + 255) / 256), 256, 0, s>>>(signals, deriv_scratch, det_pos, n_det, n_samples, t0,
                                                            dt, sound_speed, nx, ny, nz, spacing, ox, oy, oz, vol,
                                                            skipped);
  return cudaGetLastError() == cudaSuccess ? 0 : 4;
}

}  // extern "C"
