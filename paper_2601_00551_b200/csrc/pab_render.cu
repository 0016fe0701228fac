// Gaussian splat voxelisation.
//
// Replaces reference render.py:55-93 (`voxelize`): every ball with p0 > 0
// adds p0 exp(-r^2 / 2 a0^2) to each voxel centre inside its clipped
// +-support*a0 box, balls visited in lexicographic (x, y, z, p0, a0) order.
//
// B200 form: a deterministic per-voxel gather.  The caller passes the
// canonical order (rank -> ball).  Each ball's box is cut into 8^3-voxel
// bricks; (brick, rank) keys are sorted, so every brick owns the ranks of the
// balls that touch it in canonical order; one CTA per brick then sums, per
// voxel, the contributions of its balls in that order.  Each voxel therefore
// sees exactly the reference's sequence of FP64 additions, with the
// reference's expression tree for every term (no FMA contraction).
#include <cstdint>

#include <cuda_runtime.h>

namespace pab {

constexpr int kBrick = 8;            // voxels per brick edge
constexpr int kBrickShift = 3;
constexpr int kGatherThreads = 512;  // one thread per voxel of a brick
constexpr int kBallChunk = 128;      // balls staged in shared memory per step

struct VoxSpec {
  int nx, ny, nz;
  int bx, by, bz;   // bricks per axis
  double sp, ox, oy, oz, support;
};

// Reference box: lo = ceil((mu - half - origin) / sp), hi = floor((mu + half
// - origin) / sp), clipped to the grid (render.py:77-83).  Returns false when
// the ball is skipped (p0 <= 0 or empty box).
__device__ __forceinline__ bool ball_box(const VoxSpec& s, double x, double y, double z, double p0, double a0,
                                         int lo[3], int hi[3]) {
  if (!(p0 > 0.0)) return false;
  const double half = __dmul_rn(s.support, a0);
  const double c[3] = {x, y, z}, o[3] = {s.ox, s.oy, s.oz};
  const int n[3] = {s.nx, s.ny, s.nz};
  for (int a = 0; a < 3; ++a) {
    const double l = ceil(__ddiv_rn(__dsub_rn(__dsub_rn(c[a], half), o[a]), s.sp));
    const double h = floor(__ddiv_rn(__dsub_rn(__dadd_rn(c[a], half), o[a]), s.sp));
    lo[a] = l < 0.0 ? 0 : (l > (double)(n[a] - 1) ? n[a] : (int)l);
    hi[a] = h > (double)(n[a] - 1) ? n[a] - 1 : (h < 0.0 ? -1 : (int)h);
    if (lo[a] > hi[a]) return false;
  }
  return true;
}

__global__ void vox_count_kernel(const double* __restrict__ pos, const double* __restrict__ p0,
                                 const double* __restrict__ a0, const int64_t* __restrict__ order, int64_t n,
                                 VoxSpec s, int* __restrict__ box, int64_t* __restrict__ count) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  const int64_t i = order[r];
  int lo[3], hi[3];
  int64_t c = 0;
  if (ball_box(s, pos[3 * i], pos[3 * i + 1], pos[3 * i + 2], p0[i], a0[i], lo, hi)) {
    c = (int64_t)((hi[0] >> kBrickShift) - (lo[0] >> kBrickShift) + 1) *
        ((hi[1] >> kBrickShift) - (lo[1] >> kBrickShift) + 1) * ((hi[2] >> kBrickShift) - (lo[2] >> kBrickShift) + 1);
  } else {
    lo[0] = lo[1] = lo[2] = 1;
    hi[0] = hi[1] = hi[2] = 0;
  }
  for (int a = 0; a < 3; ++a) {
    box[6 * r + a] = lo[a];
    box[6 * r + 3 + a] = hi[a];
  }
  count[r] = c;
}

__global__ void vox_emit_kernel(const int* __restrict__ box, const int64_t* __restrict__ offset, int64_t n,
                                VoxSpec s, int64_t* __restrict__ keys) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  const int* b = box + 6 * r;
  if (b[0] > b[3]) return;
  int64_t k = offset[r];
  for (int ix = b[0] >> kBrickShift; ix <= (b[3] >> kBrickShift); ++ix)
    for (int iy = b[1] >> kBrickShift; iy <= (b[4] >> kBrickShift); ++iy)
      for (int iz = b[2] >> kBrickShift; iz <= (b[5] >> kBrickShift); ++iz) {
        const int64_t brick = ((int64_t)ix * s.by + iy) * s.bz + iz;
        keys[k++] = (brick << 32) | r;
      }
}

// start[b] / end[b] of brick b's run in the sorted key list (both 0 if none).
__global__ void vox_bounds_kernel(const int64_t* __restrict__ keys, int64_t total, int64_t* __restrict__ start,
                                  int64_t* __restrict__ end) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= total) return;
  const int64_t b = keys[i] >> 32;
  if (i == 0 || (keys[i - 1] >> 32) != b) start[b] = i;
  if (i == total - 1 || (keys[i + 1] >> 32) != b) end[b] = i + 1;
}

__global__ void __launch_bounds__(kGatherThreads)
vox_gather_kernel(const double* __restrict__ pos, const double* __restrict__ p0, const double* __restrict__ a0,
                  const int64_t* __restrict__ order, const int* __restrict__ box, const int64_t* __restrict__ keys,
                  const int64_t* __restrict__ start, const int64_t* __restrict__ end, VoxSpec s,
                  double* __restrict__ vol) {
  __shared__ double sx[kBallChunk], sy[kBallChunk], sz[kBallChunk], sp0[kBallChunk], sinv[kBallChunk];
  __shared__ int sbox[kBallChunk][6];
  const int64_t brick = blockIdx.x;
  const int bz = (int)(brick % s.bz), by = (int)((brick / s.bz) % s.by), bx = (int)(brick / ((int64_t)s.bz * s.by));
  const int t = threadIdx.x;
  const int vx = (bx << kBrickShift) + (t >> 6), vy = (by << kBrickShift) + ((t >> 3) & 7),
            vz = (bz << kBrickShift) + (t & 7);
  // voxel centre offsets from the origin, as the reference forms them:
  // origin + idx * sp (then - mu)
  const double cx = __dadd_rn(s.ox, __dmul_rn((double)vx, s.sp));
  const double cy = __dadd_rn(s.oy, __dmul_rn((double)vy, s.sp));
  const double cz = __dadd_rn(s.oz, __dmul_rn((double)vz, s.sp));
  double v = 0.0;
  const int64_t b0 = start[brick], b1 = end[brick];
  for (int64_t c0 = b0; c0 < b1; c0 += kBallChunk) {
    const int m = (int)min((int64_t)kBallChunk, b1 - c0);
    __syncthreads();
    if (t < m) {
      const int64_t r = keys[c0 + t] & 0xFFFFFFFFll;
      const int64_t i = order[r];
      sx[t] = pos[3 * i];
      sy[t] = pos[3 * i + 1];
      sz[t] = pos[3 * i + 2];
      sp0[t] = p0[i];
      sinv[t] = __ddiv_rn(-0.5, __dmul_rn(a0[i], a0[i]));
      for (int a = 0; a < 6; ++a) sbox[t][a] = box[6 * r + a];
    }
    __syncthreads();
    for (int k = 0; k < m; ++k) {
      if (vx < sbox[k][0] || vx > sbox[k][3] || vy < sbox[k][1] || vy > sbox[k][4] || vz < sbox[k][2] ||
          vz > sbox[k][5])
        continue;
      const double dx = __dsub_rn(cx, sx[k]), dy = __dsub_rn(cy, sy[k]), dz = __dsub_rn(cz, sz[k]);
      const double r2 = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
      v = __dadd_rn(v, __dmul_rn(sp0[k], exp(__dmul_rn(sinv[k], r2))));
    }
  }
  if (vx < s.nx && vy < s.ny && vz < s.nz) vol[((int64_t)vx * s.ny + vy) * s.nz + vz] = v;
}

static VoxSpec make_spec(int nx, int ny, int nz, double spacing, double ox, double oy, double oz, double support) {
  VoxSpec s;
  s.nx = nx; s.ny = ny; s.nz = nz;
  s.bx = (nx + kBrick - 1) / kBrick;
  s.by = (ny + kBrick - 1) / kBrick;
  s.bz = (nz + kBrick - 1) / kBrick;
  s.sp = spacing; s.ox = ox; s.oy = oy; s.oz = oz; s.support = support;
  return s;
}

}  // namespace pab

using namespace pab;

extern "C" {

int64_t pab_vox_brick_count(int nx, int ny, int nz) {
  if (nx <= 0 || ny <= 0 || nz <= 0) return 0;
  const VoxSpec s = make_spec(nx, ny, nz, 1.0, 0, 0, 0, 3.0);
  return (int64_t)s.bx * s.by * s.bz;
}

int pab_vox_count(const double* pos, const double* p0, const double* a0, const int64_t* order, int64_t n, int nx,
                  int ny, int nz, double spacing, double ox, double oy, double oz, double support, int* box,
                  int64_t* count, void* stream) {
  if (n <= 0) return 0;
  if (!pos || !p0 || !a0 || !order || !box || !count || nx <= 0 || ny <= 0 || nz <= 0 || !(spacing > 0.0)) return 1;
  const VoxSpec s = make_spec(nx, ny, nz, spacing, ox, oy, oz, support);
  vox_count_kernel<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(pos, p0, a0, order, n, s, box,
                                                                                  count);
  return cudaGetLastError() == cudaSuccess ? 0 : 4;
}

int pab_vox_emit(const int* box, const int64_t* offset, int64_t n, int nx, int ny, int nz, int64_t* keys,
                 void* stream) {
  if (n <= 0) return 0;
  if (!box || !offset || !keys) return 1;
  const VoxSpec s = make_spec(nx, ny, nz, 1.0, 0, 0, 0, 3.0);
  vox_emit_kernel<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(box, offset, n, s, keys);
  return cudaGetLastError() == cudaSuccess ? 0 : 4;
}

int pab_vox_gather(const double* pos, const double* p0, const double* a0, const int64_t* order, const int* box,
                   const int64_t* keys, int64_t total, int nx, int ny, int nz, double spacing, double ox, double oy,
                   double oz, double support, int64_t* start, int64_t* end, double* vol, void* stream) {
  if (!vol || !start || !end || nx <= 0 || ny <= 0 || nz <= 0) return 1;
  const VoxSpec s = make_spec(nx, ny, nz, spacing, ox, oy, oz, support);
  const int64_t nb = (int64_t)s.bx * s.by * s.bz;
  const cudaStream_t st = (cudaStream_t)stream;
  cudaMemsetAsync(start, 0, sizeof(int64_t) * nb, st);
  cudaMemsetAsync(end, 0, sizeof(int64_t) * nb, st);
  if (total > 0)
    vox_bounds_kernel<<<(unsigned)((total + 255) / 256), 256, 0, st>>>(keys, total, start, end);
  vox_gather_kernel<<<(unsigned)nb, kGatherThreads, 0, st>>>(pos, p0, a0, order, box, keys, start, end, s, vol);
  return cudaGetLastError() == cudaSuccess ? 0 : 4;
}

}  // extern "C"
