// GPU assembly and row normalisation of the lead-field sensitivity operator
// (SURVEY §8(f) #3), replacing `assemble_sensitivity` / `normalize_sensitivity`
// (pkg/src/d2ip/forward.py:58-112), whose NumPy form materialises (M, Q, 3)
// fp64 arrays -- infeasible at cfg2 / cfg4 scale.
//
//   f_e(q)  = -(c_q - p_e) / (4 pi max(|c_q - p_e|, min_pitch/2)^3)   (forward.py:58-66)
//   S[m][q] = -(f_d+ - f_d-) . (f_m+ - f_m-) * voxel_volume            (forward.py:82-84)
//   normalised: S[m][q] / ||S[m]||_2, zero rows rejected               (forward.py:95-112)
//
// fp64 throughout like the reference. One thread per (m, q) recomputes the
// four lead fields it needs (no (E, Q, 3) field table: E x Q x 24 B would be
// 0.7 GB at cfg4 and the recomputation is a few dozen flops). Row norms are a
// fixed-order block reduction (deterministic). The last kernel can also emit
// the fp32 masked, column-permuted block the DIP engine consumes
// ([M][Vp], column j = voxel q_of_col[j], zero padding), so the fp64 operator
// never has to visit the host.
#include <algorithm>

#include "common.cuh"
#include "kernels.h"

namespace d2ip {

__device__ __forceinline__ void lead_field(const double* __restrict__ c, const double* __restrict__ p, double min_dist,
                                           double f[3]) {
  // no FMA contraction: the same rounding sequence as NumPy's norm / power / divide
  const double dx = c[0] - p[0], dy = c[1] - p[1], dz = c[2] - p[2];
  double dist = sqrt(__dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz)));
  dist = dist > min_dist ? dist : min_dist;
  const double den = __dmul_rn(4.0 * 3.141592653589793, __dmul_rn(__dmul_rn(dist, dist), dist));
  f[0] = -dx / den;
  f[1] = -dy / den;
  f[2] = -dz / den;
}

__global__ void __launch_bounds__(256) sens_assemble_k(const double* __restrict__ centers, int Q,
                                                       const double* __restrict__ elec, const int* __restrict__ quads,
                                                       double min_dist, double vv, double* __restrict__ out) {
  D2IP_PDL_ENTRY();
  const int m = blockIdx.y;
  const long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= Q) return;
  const int4 e = reinterpret_cast<const int4*>(quads)[m];
  const double* c = centers + 3 * q;
  double a[3], b[3], g[3], h[3];
  lead_field(c, elec + 3 * e.x, min_dist, a);
  lead_field(c, elec + 3 * e.y, min_dist, b);
  lead_field(c, elec + 3 * e.z, min_dist, g);
  lead_field(c, elec + 3 * e.w, min_dist, h);
  const double d0 = a[0] - b[0], d1 = a[1] - b[1], d2 = a[2] - b[2];
  const double m0 = g[0] - h[0], m1 = g[1] - h[1], m2 = g[2] - h[2];
  const double dot = __dadd_rn(__dadd_rn(__dmul_rn(d0, m0), __dmul_rn(d1, m1)), __dmul_rn(d2, m2));
  out[(long long)m * Q + q] = __dmul_rn(-dot, vv);
}

// norm[m] = sqrt(sum_q S[m][q]^2), fixed order: thread t sums q = t, t+256, ...; tree over threads
__global__ void __launch_bounds__(256) sens_rownorm_k(const double* __restrict__ S, int Q, double* __restrict__ norm) {
  D2IP_PDL_ENTRY();
  __shared__ double red[256];
  const int m = blockIdx.x;
  const double* row = S + (long long)m * Q;
  double s = 0.0;
  for (long long q = threadIdx.x; q < Q; q += 256) s = __dadd_rn(s, __dmul_rn(row[q], row[q]));
  red[threadIdx.x] = s;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) norm[m] = sqrt(red[0]);
}

// the fp32 masked block for the engine: Jm[m][j] = (float)(S[m][q_of_col[j]] / norm[m]) (or unscaled)
__global__ void __launch_bounds__(256) sens_masked_k(const double* __restrict__ S, int Q, const double* __restrict__ norm,
                                                     int normalize, float* __restrict__ Jm, int V, int Vp,
                                                     const int* __restrict__ q_of_col) {
  D2IP_PDL_ENTRY();
  const int m = blockIdx.y;
  const long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= Vp) return;
  float v = 0.f;
  if (j < V) {
    const double s = S[(long long)m * Q + q_of_col[j]];
    v = (float)(normalize ? s / norm[m] : s);
  }
  Jm[(long long)m * Vp + j] = v;
}

// in place S /= norm[m]  (forward.py:109: values / norms[:, None])
__global__ void __launch_bounds__(256) sens_normalize_k(double* __restrict__ S, int Q, const double* __restrict__ norm) {
  D2IP_PDL_ENTRY();
  const int m = blockIdx.y;
  const long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (q < Q) S[(long long)m * Q + q] = S[(long long)m * Q + q] / norm[m];
}

}  // namespace d2ip

extern "C" int d2ip_assemble_sensitivity(const double* centers, int Q, const double* electrodes, int E,
                                         const int* quads, int M, double min_dist, double voxel_volume,
                                         int normalize, double* out, double* norms, float* J_masked, int V, int Vp,
                                         const int* q_of_col, void* stream) {
  using namespace d2ip;
  D2IP_CHECK_ARG(centers && electrodes && quads && out && norms, "null argument");
  D2IP_CHECK_ARG(Q >= 1 && E >= 4 && M >= 1, "bad sizes (Q=%d, E=%d, M=%d)", Q, E, M);
  D2IP_CHECK_ARG(!J_masked || (q_of_col && V >= 1 && Vp >= V), "masked output needs q_of_col and V <= Vp");
  D2IP_CHECK_ARG(((uintptr_t)quads & 15) == 0, "quads must be 16-byte aligned int32 [M][4]");
  cudaStream_t st = S(stream);
  D2IP_CUDA(launch_pdl(sens_assemble_k, dim3(cdiv(Q, 256), M), 256, 0, st, centers, Q, electrodes, quads, min_dist,
                       voxel_volume, out));
  D2IP_CUDA(launch_pdl(sens_rownorm_k, dim3(M), 256, 0, st, (const double*)out, Q, norms));
  if (J_masked)
    D2IP_CUDA(launch_pdl(sens_masked_k, dim3(cdiv(Vp, 256), M), 256, 0, st, (const double*)out, Q,
                         (const double*)norms, normalize, J_masked, V, Vp, q_of_col));
  if (normalize)
    D2IP_CUDA(launch_pdl(sens_normalize_k, dim3(cdiv(Q, 256), M), 256, 0, st, out, Q, (const double*)norms));
  D2IP_LAUNCH_CHECK();
  return D2IP_OK;
}
