// K5 / K6: the linearised EIT data term over the voxel mask.
//
// Reference (pkg/src/d2ip/pipeline.py):
//   residual = dv - operator @ _vectorize_t(mapped)     (:279)
//   data = sum(residual^2)        ("l2sq")              (:257-260)
//        = sqrt(sum(residual^2))  ("l2", 0 kept at 0)   (:261-263)
//   backward: d data / d mapped = -c * J^T residual     (autograd of mv)
// Here r = J sigma - dv (= -residual), and the kernels produce
//   rs = c * sum_f r_f  with c = 2 (l2sq) or 1/sqrt(sum r^2) (l2, 0 if 0),
//   g  = J^T rs, scattered to the full-grid output-map gradient.
// J is M x Vp fp32 row-major (Vp % 4 == 0, zero padded), columns in the
// network's memory order of the masked voxels. Both passes stream J from HBM
// with 128-bit loads; all reductions are fixed-order (deterministic).
#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"

namespace d2ip {

constexpr int kGemvThreads = 256;
constexpr int kGemvUnroll = 4;
constexpr int kGemvSeg = kGemvThreads * 4 * kGemvUnroll;  // columns per block

int jac_nseg(int vp) { return cdiv(vp, kGemvSeg); }

// partial[b][m][seg] = sum_{j in seg} J[m][j] * sigma[j]
__global__ void __launch_bounds__(kGemvThreads) jac_fwd_k(const float* __restrict__ J, long long jbs,
                                                          const float* __restrict__ sigma, long long sbs,
                                                          int vp, float* __restrict__ partial, int nseg) {
  D2IP_PDL_ENTRY();
  __shared__ float red[kGemvThreads / 32];
  const int seg = blockIdx.x, m = blockIdx.y, b = blockIdx.z;
  const float4* row = reinterpret_cast<const float4*>(J + b * jbs + (long long)m * vp);
  const float4* sg = reinterpret_cast<const float4*>(sigma + b * sbs);
  const int n4 = vp >> 2;
  const int base = seg * (kGemvSeg / 4) + threadIdx.x;
  float4 a[kGemvUnroll], s[kGemvUnroll];
#pragma unroll
  for (int u = 0; u < kGemvUnroll; ++u) {
    const int j = base + u * kGemvThreads;
    if (j < n4) {
      a[u] = __ldg(row + j);
      s[u] = __ldg(sg + j);
    } else {
      a[u] = make_float4(0.f, 0.f, 0.f, 0.f);
      s[u] = a[u];
    }
  }
  float acc = 0.f;
#pragma unroll
  for (int u = 0; u < kGemvUnroll; ++u) {
    acc = fmaf(a[u].x, s[u].x, acc);
    acc = fmaf(a[u].y, s[u].y, acc);
    acc = fmaf(a[u].z, s[u].z, acc);
    acc = fmaf(a[u].w, s[u].w, acc);
  }
  acc = block_sum<kGemvThreads>(acc, red);
  // partials are [b][segment][row]: the consumers read consecutive rows (coalesced)
  if (threadIdx.x == 0) partial[((long long)b * nseg + seg) * gridDim.y + m] = acc;
}

int jac_fwd_partial(const float* J, long long jbs, const float* sigma, long long sbs, int m, int vp,
                    float* partial, int nseg, int batch, cudaStream_t st) {
  D2IP_CHECK_ARG(vp % 4 == 0, "jac: Vp=%d not a multiple of 4", vp);
  D2IP_CHECK_ARG(((uintptr_t)J & 15) == 0 && ((uintptr_t)sigma & 15) == 0, "jac: J/sigma not 16B aligned");
  dim3 grid(nseg, m, batch);
  D2IP_CUDA(launch_pdl(jac_fwd_k, grid, kGemvThreads, 0, st, J, jbs, sigma, sbs, vp, partial, nseg));
  D2IP_LAUNCH_CHECK();
  return D2IP_OK;
}

// One block per sequence: residuals, data term, gradient scale, trace, NaN flag.
// status[b] = {iterations done this frame, first non-finite iteration (0 none), n_history, -}
__global__ void __launch_bounds__(1024) jac_loss_k(const float* __restrict__ partial, int nseg, int M,
                                                   const float* __restrict__ dv, int n_rhs, int norm,
                                                   const float* __restrict__ reg_partial, int n_reg,
                                                   float reg_scale, float* __restrict__ rs,
                                                   float* __restrict__ trace, int max_iters,
                                                   int* __restrict__ status) {
  D2IP_PDL_ENTRY();
  __shared__ float red[32];
  const int b = blockIdx.x;
  float acc = 0.f;
  for (int m = threadIdx.x; m < M; m += blockDim.x) {
    const float* p = partial + (long long)b * nseg * M + m;
    float y = 0.f;
    for (int s = 0; s < nseg; ++s) y += p[(long long)s * M];
    float rsum = 0.f;
    for (int f = 0; f < n_rhs; ++f) {
      const float r = y - dv[((long long)b * n_rhs + f) * M + m];
      acc = fmaf(r, r, acc);
      rsum += r;
    }
    rs[(long long)b * M + m] = rsum;
  }
  const float sq = block_sum<1024>(acc, red);
  float reg = 0.f;
  if (n_reg > 0) {
    float t = 0.f;
    for (int i = threadIdx.x; i < n_reg; i += blockDim.x) t += reg_partial[(long long)b * n_reg + i];
    reg = block_sum<1024>(t, red) * reg_scale;
  }
  float data, c;
  if (norm == D2IP_NORM_L2SQ) {
    data = sq;
    c = 2.f;
  } else {
    data = sq == 0.f ? 0.f : sqrtf(sq);
    c = sq == 0.f ? 0.f : 1.f / data;
  }
  for (int m = threadIdx.x; m < M; m += blockDim.x) rs[(long long)b * M + m] *= c;
  if (threadIdx.x == 0) {
    const float total = data + reg;
    const int k = status[b * 4 + 0] + 1;
    if (k <= max_iters) {
      float* t = trace + ((long long)b * max_iters + (k - 1)) * 4;
      unsigned long long ns;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ns));
      t[0] = data;
      t[1] = reg;
      t[2] = total;
      t[3] = __int_as_float((int)((ns >> 10) & 0x7fffffffULL));  // 1.024 us ticks (int bits); host takes differences
    }
    if (!isfinite(total) && status[b * 4 + 1] == 0) status[b * 4 + 1] = k;
    status[b * 4 + 0] = k;
  }
}

int jac_loss(const float* partial, int nseg, int m, const float* dv, int n_rhs, int norm,
             const float* reg_partial, int n_reg, float reg_scale, float* rs, float* trace,
             int max_iters, int* status, int batch, cudaStream_t st) {
  D2IP_CUDA(launch_pdl(jac_loss_k, batch, 1024, 0, st, partial, nseg, m, dv, n_rhs, norm, reg_partial, n_reg, reg_scale,
                                     rs, trace, max_iters, status));
  D2IP_LAUNCH_CHECK();
  return D2IP_OK;
}

__global__ void jac_sum_k(const float* __restrict__ partial, int nseg, int M, float* __restrict__ y) {
  D2IP_PDL_ENTRY();
  const int b = blockIdx.y;
  const int m = blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= M) return;
  const float* p = partial + (long long)b * nseg * M + m;
  float acc = 0.f;
  for (int s = 0; s < nseg; ++s) acc += p[(long long)s * M];
  y[(long long)b * M + m] = acc;
}

int jac_sum(const float* partial, int nseg, int m, float* y, int batch, cudaStream_t st) {
  D2IP_CUDA(launch_pdl(jac_sum_k, dim3(cdiv(m, 256), batch), 256, 0, st, partial, nseg, m, y));
  D2IP_LAUNCH_CHECK();
  return D2IP_OK;
}

// ---- adjoint: partial[b][rsplit][j] = sum_{m in split} J[m][j] * rs[m]
constexpr int kAdjThreads = 256;
constexpr int kAdjCols = kAdjThreads * 4;

static bool adj_wide() {  // D2IP_ADJ_WIDE=1: four float4 columns per thread (measured no faster)
  static const bool v = [] {
    const char* e = getenv("D2IP_ADJ_WIDE");
    return e && atoi(e) != 0;
  }();
  return v;
}

static int adj_blocks_per_sm() {  // D2IP_ADJ_BPS: row splits sized for this many blocks per SM
  static const int v = [] {
    const char* e = getenv("D2IP_ADJ_BPS");
    return e ? std::max(1, atoi(e)) : 3;  // 3: cfg2 298 -> 274 us, cfg4 900 -> 820 us (with 8 loads in flight)
  }();
  return v;
}

static int adj_unroll() {  // D2IP_ADJ_U: loads in flight per thread (4 or 8)
  static const int v = [] {
    const char* e = getenv("D2IP_ADJ_U");
    return e && atoi(e) == 4 ? 4 : 8;
  }();
  return v;
}

int jac_adj_rows(int m, int vp, int batch) {
  const int ctiles = cdiv(vp, adj_wide() ? 4 * kAdjCols : kAdjCols);
  // (independent of the batch: a batched engine's sequences sum in the same order as single runs)
  (void)batch;
  long long want = (148LL * adj_blocks_per_sm() + ctiles - 1) / ctiles;
  if (want > m) want = m;
  if (want < 1) want = 1;
  return (int)want;
}

size_t jac_adj_ws(int m, int vp, int batch) {
  return (size_t)batch * jac_adj_rows(m, vp, batch) * vp * sizeof(float);
}

template <int U>
__global__ void __launch_bounds__(kAdjThreads) jac_adj_k(const float* __restrict__ J, long long jbs,
                                                         const float* __restrict__ rs, int M, int vp,
                                                         float* __restrict__ partial, int rsplit) {
  D2IP_PDL_ENTRY();
  extern __shared__ float rsm[];
  const int b = blockIdx.z, sp = blockIdx.y;
  const int rows = (M + rsplit - 1) / rsplit;
  const int m0 = sp * rows, m1 = min(M, m0 + rows);
  for (int i = threadIdx.x; i < m1 - m0; i += blockDim.x) rsm[i] = rs[(long long)b * M + m0 + i];
  __syncthreads();
  const int j4 = blockIdx.x * kAdjThreads + threadIdx.x;  // float4 column index
  if (j4 * 4 >= vp) return;
  const float4* col = reinterpret_cast<const float4*>(J + b * jbs) + j4;
  const int n4 = vp >> 2;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  int m = m0;
  for (; m + U <= m1; m += U) {
    float4 a[U];
#pragma unroll
    for (int u = 0; u < U; ++u) a[u] = __ldg(col + (long long)(m + u) * n4);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const float r = rsm[m + u - m0];
      acc.x = fmaf(a[u].x, r, acc.x);
      acc.y = fmaf(a[u].y, r, acc.y);
      acc.z = fmaf(a[u].z, r, acc.z);
      acc.w = fmaf(a[u].w, r, acc.w);
    }
  }
  for (; m < m1; ++m) {
    const float4 a = __ldg(col + (long long)m * n4);
    const float r = rsm[m - m0];
    acc.x = fmaf(a.x, r, acc.x);
    acc.y = fmaf(a.y, r, acc.y);
    acc.z = fmaf(a.z, r, acc.z);
    acc.w = fmaf(a.w, r, acc.w);
  }
  reinterpret_cast<float4*>(partial + ((long long)b * rsplit + sp) * vp)[j4] = acc;
}

// Wide variant: a block covers 4 x 1,024 columns (16 KB of every row it visits, like the forward's
// row segments) and each thread keeps four float4 column accumulators, two rows in flight (8
// independent 16-byte loads). Fixed summation order per column (rows ascending in the split).
__global__ void __launch_bounds__(kAdjThreads) jac_adj_wide_k(const float* __restrict__ J, long long jbs,
                                                              const float* __restrict__ rs, int M, int vp,
                                                              float* __restrict__ partial, int rsplit) {
  D2IP_PDL_ENTRY();
  extern __shared__ float rsm[];
  const int b = blockIdx.z, sp = blockIdx.y;
  const int rows = (M + rsplit - 1) / rsplit;
  const int m0 = sp * rows, m1 = min(M, m0 + rows);
  for (int i = threadIdx.x; i < m1 - m0; i += blockDim.x) rsm[i] = rs[(long long)b * M + m0 + i];
  __syncthreads();
  const int n4 = vp >> 2;
  const int base = blockIdx.x * (4 * kAdjThreads) + threadIdx.x;
  const float4* Jb = reinterpret_cast<const float4*>(J + b * jbs);
  float4 acc[4];
  bool ok[4];
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    acc[c] = make_float4(0.f, 0.f, 0.f, 0.f);
    ok[c] = base + c * kAdjThreads < n4;
  }
  int m = m0;
  for (; m + 2 <= m1; m += 2) {
    float4 a[2][4];
#pragma unroll
    for (int u = 0; u < 2; ++u)
#pragma unroll
      for (int c = 0; c < 4; ++c)
        a[u][c] = ok[c] ? __ldg(Jb + (long long)(m + u) * n4 + base + c * kAdjThreads) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const float r = rsm[m + u - m0];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        acc[c].x = fmaf(a[u][c].x, r, acc[c].x);
        acc[c].y = fmaf(a[u][c].y, r, acc[c].y);
        acc[c].z = fmaf(a[u][c].z, r, acc[c].z);
        acc[c].w = fmaf(a[u][c].w, r, acc[c].w);
      }
    }
  }
  for (; m < m1; ++m) {
    const float r = rsm[m - m0];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      if (!ok[c]) continue;
      const float4 a = __ldg(Jb + (long long)m * n4 + base + c * kAdjThreads);
      acc[c].x = fmaf(a.x, r, acc[c].x);
      acc[c].y = fmaf(a.y, r, acc[c].y);
      acc[c].z = fmaf(a.z, r, acc[c].z);
      acc[c].w = fmaf(a.w, r, acc[c].w);
    }
  }
  float4* out = reinterpret_cast<float4*>(partial + ((long long)b * rsplit + sp) * vp);
#pragma unroll
  for (int c = 0; c < 4; ++c)
    if (ok[c]) out[base + c * kAdjThreads] = acc[c];
}

int jac_adj_partial(const float* J, long long jbs, const float* rs, int m, int vp, float* partial,
                    int rsplit, int batch, cudaStream_t st) {
  const int rows = cdiv(m, rsplit);
  if (adj_wide()) {
    dim3 gw(cdiv(vp, 4 * kAdjCols), rsplit, batch);
    D2IP_CUDA(launch_pdl(jac_adj_wide_k, gw, kAdjThreads, rows * sizeof(float), st, J, jbs, rs, m, vp, partial, rsplit));
    D2IP_LAUNCH_CHECK();
    return D2IP_OK;
  }
  dim3 grid(cdiv(vp, kAdjCols), rsplit, batch);
  if (adj_unroll() == 8)
    D2IP_CUDA(launch_pdl(jac_adj_k<8>, grid, kAdjThreads, rows * sizeof(float), st, J, jbs, rs, m, vp, partial, rsplit));
  else
    D2IP_CUDA(launch_pdl(jac_adj_k<4>, grid, kAdjThreads, rows * sizeof(float), st, J, jbs, rs, m, vp, partial, rsplit));
  D2IP_LAUNCH_CHECK();
  return D2IP_OK;
}

// g_j = sum_split partial; at voxel vox_of_col[j]:
//   add_to_gmapped = 0: gout = g * scale * (1 - s) * s   (gtail directly)
//   add_to_gmapped = 1: gout += g                       (gmapped, TV on)
__global__ void jac_adj_finish_k(const float* __restrict__ partial, int rsplit, int vp, int V,
                                 const int* __restrict__ vox_of_col, const float* __restrict__ sig,
                                 float scale, float* __restrict__ gout, long long V0, int add) {
  D2IP_PDL_ENTRY();
  const int b = blockIdx.y;
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= V) return;
  const float* p = partial + (long long)b * rsplit * vp + j;
  float g = 0.f;
  for (int s = 0; s < rsplit; ++s) g += p[(long long)s * vp];
  const long long vox = (long long)b * V0 + vox_of_col[j];
  if (add) {
    gout[vox] += g;
  } else {
    const float s = sig[vox];
    gout[vox] = (g * scale) * (1.f - s) * s;
  }
}

int jac_adj_finish(const float* partial, int rsplit, int vp, int v, const int* vox_of_col,
                   const float* sig, float scale, float* gout, long long V0, int add_to_gmapped,
                   int batch, cudaStream_t st) {
  D2IP_CUDA(launch_pdl(jac_adj_finish_k, dim3(cdiv(v, 256), batch), 256, 0, st, partial, rsplit, vp, v, vox_of_col, sig,
                                                               scale, gout, V0, add_to_gmapped));
  D2IP_LAUNCH_CHECK();
  return D2IP_OK;
}

// fp64 projection y = A x (the drop-in `forward_project`, forward.py:115-122:
// `matrix.values @ vec` in float64). One warp per row, each lane a strided
// fixed-order partial, then a fixed xor-shuffle tree: deterministic.
__global__ void __launch_bounds__(256) project_f64_k(const double* __restrict__ A, long long lda,
                                                     const double* __restrict__ x, int m, int n,
                                                     double* __restrict__ y) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= m) return;
  const double* a = A + (long long)warp * lda;
  double s = 0.0;
  for (int j = lane; j < n; j += 32) s = fma(a[j], x[j], s);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) y[warp] = s;
}

int project_f64(const double* A, long long lda, const double* x, int m, int n, double* y, cudaStream_t st) {
  D2IP_CHECK_ARG(A && x && y && m >= 0 && n >= 0 && lda >= n, "project_f64: bad arguments");
  if (m == 0) return D2IP_OK;
  project_f64_k<<<cdiv((long long)m * 32, 256), 256, 0, st>>>(A, lda, x, m, n, y);
  D2IP_LAUNCH_CHECK();
  return D2IP_OK;
}

}  // namespace d2ip
