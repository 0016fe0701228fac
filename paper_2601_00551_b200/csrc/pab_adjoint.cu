// Adjoint: residual -> per-ball loss gradients.
//
// Replaces reference radiator.py:263-287 (gather of the residual over each
// cached slab window, einsum reductions, per-ball gradient assembly) and the
// fixed-order block merge :336-348.
//
// Decomposition: a warp owns one lane group (32 Morton-ordered balls, one per
// lane) and loops over a chunk of detectors; per detector the warp stages the
// residual segment its group can touch into shared memory (coalesced), then
// every lane walks its own arrival window accumulating four FP32 moments
//   T_k = sum_J res[J] G(y_J) y_J^k,  k = 0..3,
// and folds them into FP64 per-ball gradient accumulators held in registers
// across all detectors of the chunk (no atomics).  Detector chunks (grid.y)
// write partial sums that a finalize pass adds in chunk order.
#include "pab_common.cuh"

namespace pab {

constexpr int kSeg = 256;   // staged residual samples per warp

template <int STAGE>
__global__ void __launch_bounds__(256)
adjoint_kernel(const BallA* __restrict__ ra, const BallB* __restrict__ rb,
               const GroupMeta* __restrict__ gmeta, int64_t n_groups,
               const double* __restrict__ det_pos, const double* __restrict__ det_aux, int n_det,
               Acq acq, const float* __restrict__ res, float res_sign, int det_per_chunk,
               double* __restrict__ gpart, int64_t n_pad, unsigned long long* __restrict__ ops_total,
               int* __restrict__ status) {
  __shared__ float seg_all[8][kSeg];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t g = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp;
  if (g >= n_groups) return;
  float* seg = seg_all[warp];
  const int q = blockIdx.y;
  const int j0 = q * det_per_chunk;
  const int j1 = min(n_det, j0 + det_per_chunk);
  const int n_out = acq.n_out;
  const int f = acq.f;
  const float fs = (float)f;

  const GroupMeta gm = gmeta[g];
  const int64_t bi = g * kWarp + lane;
  const BallA A = ra[bi];
  const BallB B = rb[bi];
  const float kap = A.a0 * kSqrt2Ln2;
  double acc_p0 = 0.0, acc_a0 = 0.0, acc_x = 0.0, acc_y = 0.0, acc_z = 0.0;
  unsigned long long my_ops = 0;
  int coinc = 0;
  constexpr bool want_dir_grad = (STAGE == kStageFine);

  for (int jb = j0; jb < j1; jb += kWarp) {
    const int nd = min(kWarp, j1 - jb);
    GroupDet gdl;
    int rlo = 0, rhi = -1;
    if (lane < nd) {
      const Detector dl = load_detector(det_pos, det_aux, jb + lane);
      gdl = group_det(gm, dl.px, dl.py, dl.pz, acq);
      group_range(acq, gdl, gm, &rlo, &rhi);
    } else {
      gdl.Sx = gdl.Sy = gdl.Sz = 0.f; gdl.Sn = 1.f; gdl.isn = 1.f; gdl.phg = 0.f; gdl.kg = 0; gdl.slow = 0;
    }
    for (int jj = 0; jj < nd; ++jj) {
      const int j = jb + jj;
      const GroupDet gd = shfl_gd(gdl, jj);
      const int lo = __shfl_sync(0xffffffffu, rlo, jj);
      const int hi = __shfl_sync(0xffffffffu, rhi, jj);
      if (lo > hi) continue;
      const Detector det = load_detector(det_pos, det_aux, j);
      float dDdr[3] = {0.f, 0.f, 0.f}, dDda0 = 0.f;
      const bool dgrad = want_dir_grad || acq.dir_kind == kDirElement;
      const Pair p = make_pair(acq, gd, gm, det, A, B, dgrad, dDdr, &dDda0);
      my_ops += (unsigned long long)(max(p.jhi - p.jlo + 1, 0) + max(p.nhi - p.nlo + 1, 0));
      coinc |= p.coincident;
      float T0 = 0.f, T1 = 0.f, T2 = 0.f, T3 = 0.f;
      const float ps = p.phi * p.sc;
      const float* rrow = res + (size_t)j * n_out;
      for (int base = lo; base <= hi; base += kSeg) {
        const int top = min(base + kSeg - 1, hi);
        __syncwarp();
        for (int k = lane; k <= top - base; k += kWarp) seg[k] = res_sign * __ldg(rrow + base + k);
        __syncwarp();
        {
          const int jlo = max(p.jlo, base), jhi = min(p.jhi, top);
          float mf = (float)(jlo * f - p.kc);
          const float* s = seg + (jlo - base);
#pragma unroll 4
          for (int J = jlo; J <= jhi; ++J, mf += fs, ++s) {
            const float y = fmaf(mf, -p.sc, ps);
            const float q2 = y * y;
            const float r = (*s) * ex2(-q2);
            const float t = r * y;
            T1 += t;
            if (STAGE >= kStageCoarse) T3 = fmaf(t, q2, T3);
            if (STAGE == kStageFine) { T0 += r; T2 = fmaf(t, y, T2); }
          }
        }
        if (p.nlo <= p.nhi) {   // u+ = -kappa y: odd moments flip sign
          const int jlo = max(p.nlo, base), jhi = min(p.nhi, top);
          const float nps = p.nphi * p.sc;
          for (int J = jlo; J <= jhi; ++J) {
            const float y = fmaf((float)(J * f - p.nkc), -p.sc, nps);
            const float q2 = y * y;
            const float r = seg[J - base] * ex2(-q2);
            const float t = r * y;
            T1 -= t;
            if (STAGE >= kStageCoarse) T3 = fmaf(-t, q2, T3);
            if (STAGE == kStageFine) { T0 += r; T2 = fmaf(t, y, T2); }
          }
        }
      }
      // per-pair gradient terms (reference radiator.py:275-286 in y units)
      const float s_uG = kap * T1;
      acc_p0 += (double)(p.D * s_uG * (0.5f / p.d));
      if (STAGE >= kStageCoarse) {
        float ga = p.amp * kSqrt2Ln2Cubed * T3;
        if (acq.dir_kind == kDirElement) ga = fmaf(p.base * dDda0, s_uG, ga);
        acc_a0 += (double)ga;
      }
      if (STAGE == kStageFine) {
        const float gdist = p.amp * (T0 - kTwoLn2 * T2) - (p.amp / p.d) * s_uG;
        const float w = gdist / p.d;
        float gx = w * p.rx, gy = w * p.ry, gz = w * p.rz;
        if (acq.dir_kind != kDirNone) {
          const float bs = p.base * s_uG;
          gx = fmaf(bs, dDdr[0], gx);
          gy = fmaf(bs, dDdr[1], gy);
          gz = fmaf(bs, dDdr[2], gz);
        }
        acc_x += (double)gx; acc_y += (double)gy; acc_z += (double)gz;
      }
    }
  }
  double* out = gpart + (size_t)q * 5 * n_pad;
  out[0 * n_pad + bi] = acc_p0;
  out[1 * n_pad + bi] = acc_a0;
  out[2 * n_pad + bi] = acc_x;
  out[3 * n_pad + bi] = acc_y;
  out[4 * n_pad + bi] = acc_z;
  for (int o = 16; o > 0; o >>= 1) {
    my_ops += __shfl_xor_sync(0xffffffffu, my_ops, o);
    coinc |= __shfl_xor_sync(0xffffffffu, coinc, o);
  }
  if (lane == 0) {
    if (ops_total && my_ops) atomicAdd(ops_total, my_ops);
    if (coinc) atomicOr(status, kStatusCoincident);
  }
}

// Sum detector-chunk partials in chunk order, scale by 2/N (MSE, reference
// radiator.py:356-358), scatter to the caller's ball order, flag non-finite.
__global__ void grad_finalize_kernel(const double* __restrict__ gpart, int chunks, int64_t n_pad,
                                     const BallB* __restrict__ rb, double scale, int stage,
                                     double* __restrict__ d_p0, double* __restrict__ d_a0,
                                     double* __restrict__ d_pos, int* __restrict__ status) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_pad) return;
  const int orig = rb[i].orig;
  if (orig < 0) return;
  double v[5] = {0, 0, 0, 0, 0};
  for (int q = 0; q < chunks; ++q)
    for (int c = 0; c < 5; ++c) v[c] += gpart[((size_t)q * 5 + c) * n_pad + i];
  bool bad = false;
  for (int c = 0; c < 5; ++c) {
    v[c] *= scale;
    bad |= !isfinite(v[c]);
  }
  d_p0[orig] = v[0];
  if (d_a0) d_a0[orig] = stage >= kStageCoarse ? v[1] : 0.0;
  if (d_pos) {
    d_pos[3 * (int64_t)orig + 0] = stage == kStageFine ? v[2] : 0.0;
    d_pos[3 * (int64_t)orig + 1] = stage == kStageFine ? v[3] : 0.0;
    d_pos[3 * (int64_t)orig + 2] = stage == kStageFine ? v[4] : 0.0;
  }
  if (bad) atomicOr(status, kStatusNonFinite);
}

}  // namespace pab

using namespace pab;

extern "C" {

int pab_adjoint(const void* rec_a, const void* rec_b, const void* group_meta, int64_t n_groups,
                const double* det_pos, const double* det_aux, int n_det, double v, double t0, double dt,
                int f, int n_out, double cutoff, int dir_kind, double dir_param, const float* res,
                float res_sign, int stage, int chunks, int warps, double* grad_partial,
                unsigned long long* ops_total, int* status, void* stream) {
  if (n_groups <= 0 || n_det <= 0) return 0;
  if (f < 1 || chunks < 1 || warps < 1 || warps > 8 || stage < 0 || stage > 2) return 1;
  if (!rec_a || !rec_b || !group_meta || !det_pos || !det_aux || !res || !grad_partial || !status) return 1;
  Acq a;
  a.vdt = v * dt; a.inv_vdt = 1.0 / a.vdt; a.vt0 = v * t0; a.f = f; a.n_out = n_out;
  a.cutoff = (float)cutoff; a.vdt_f = (float)a.vdt; a.inv_vdt_f = (float)a.inv_vdt;
  a.dir_kind = dir_kind; a.dir_param = (float)dir_param;
  const int per_chunk = (n_det + chunks - 1) / chunks;
  const int64_t n_pad = n_groups * kWarp;
  dim3 grid((unsigned)((n_groups + warps - 1) / warps), (unsigned)chunks);
  const cudaStream_t s = (cudaStream_t)stream;
  const BallA* A = (const BallA*)rec_a;
  const BallB* B = (const BallB*)rec_b;
  const GroupMeta* G = (const GroupMeta*)group_meta;
  if (stage == kStageFilter)
    adjoint_kernel<kStageFilter><<<grid, warps * kWarp, 0, s>>>(A, B, G, n_groups, det_pos, det_aux, n_det, a,
                                                                res, res_sign, per_chunk, grad_partial, n_pad,
                                                                ops_total, status);
  else if (stage == kStageCoarse)
    adjoint_kernel<kStageCoarse><<<grid, warps * kWarp, 0, s>>>(A, B, G, n_groups, det_pos, det_aux, n_det, a,
                                                                res, res_sign, per_chunk, grad_partial, n_pad,
                                                                ops_total, status);
  else
    adjoint_kernel<kStageFine><<<grid, warps * kWarp, 0, s>>>(A, B, G, n_groups, det_pos, det_aux, n_det, a,
                                                              res, res_sign, per_chunk, grad_partial, n_pad,
                                                              ops_total, status);
  return cudaGetLastError() == cudaSuccess ? 0 : 4;
}

int pab_grad_finalize(const double* grad_partial, int chunks, int64_t n_groups, const void* rec_b, double scale,
                      int stage, double* d_p0, double* d_a0, double* d_pos, int* status, void* stream) {
  if (n_groups <= 0) return 0;
  if (!grad_partial || !rec_b || !d_p0 || !status || chunks < 1) return 1;
  const int64_t n_pad = n_groups * kWarp;
  grad_finalize_kernel<<<(unsigned)((n_pad + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
      grad_partial, chunks, n_pad, (const BallB*)rec_b, scale, stage, d_p0, d_a0, d_pos, status);
  return cudaGetLastError() == cudaSuccess ? 0 : 4;
}

}  // extern "C"
