// Direct (CUDA-core, fp32) 3^3 / 1^3 convolutions: forward, data gradient,
// weight gradient. These are the exact-fp32 kernels (precision D2IP_PREC_FP32)
// and the fallback for shapes the tcgen05 implicit-GEMM kernels do not take
// (C_out = 1 tail, C_in not a multiple of 4). Layout: NDHWC activations,
// OIDHW weights (the reference's nn.Conv3d layout, priornet.py:111-117).
#include <algorithm>

#include "common.cuh"
#include "kernels.h"

namespace d2ip {

static int tiled_threads(int cin, int cout, int ks, int cog);
static void tiled_split(int cin, int cout, int ks, int cog, long long V, int batch, int* nchunks, int* chunk);

template <int KS>
struct Taps {
  static constexpr int K3 = KS * KS * KS;
  static constexpr int PAD = KS / 2;
};

// Direct convolutions (stride 2, 1^3, odd channel counts, the C_out = 1
// tail, and precision FP32). A block owns CG output channels and 128 voxels
// (one per thread); the CG x C_in x k^3 weight slice sits in shared memory as
// [c][tap][CG] so every (c, tap) step is one float4-vectorised input load
// (4 channels) against broadcast shared-memory weights.

// y[v][co0..co0+CG) = sum_{tap,ci} x[in(v,tap)][ci] * W[co][ci][tap]
template <int KS, int CG>
__global__ void __launch_bounds__(128) conv_fwd_direct_k(d2ip_act x, const float* __restrict__ w,
                                                         const float* __restrict__ bias,
                                                         long long wbs, int stride, d2ip_act y,
                                                         int accumulate, int vec, int dil) {
  D2IP_PDL_ENTRY();
  constexpr int K3 = Taps<KS>::K3, PAD = Taps<KS>::PAD;
  extern __shared__ float sw[];  // [cin][K3][CG]
  const int b = blockIdx.z;
  const int cin = x.c, co0 = blockIdx.y * CG;
  const float* wb = w + b * wbs;
  for (int i = threadIdx.x; i < cin * K3 * CG; i += blockDim.x) {
    const int j = i % CG, r = i / CG, tap = r % K3, ci = r / K3;
    sw[i] = __ldg(wb + ((long long)(co0 + j) * cin + ci) * K3 + tap);
  }
  __syncthreads();
  const long long V = (long long)y.d * y.h * y.w;
  const long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= V) return;
  const int ow = (int)(v % y.w), oh = (int)((v / y.w) % y.h), od = (int)(v / ((long long)y.w * y.h));
  float acc[CG];
#pragma unroll
  for (int j = 0; j < CG; ++j) acc[j] = bias ? __ldg(bias + b * wbs + co0 + j) : 0.f;
  const float* xb = x.ptr + b * x.bstride;
  for (int kd = 0; kd < KS; ++kd) {
    const int id = od * stride + (kd - PAD) * dil;
    if (id < 0 || id >= x.d) continue;
    for (int kh = 0; kh < KS; ++kh) {
      const int ih = oh * stride + (kh - PAD) * dil;
      if (ih < 0 || ih >= x.h) continue;
      for (int kw = 0; kw < KS; ++kw) {
        const int iw = ow * stride + (kw - PAD) * dil;
        if (iw < 0 || iw >= x.w) continue;
        const float* xp = xb + (((long long)id * x.h + ih) * x.w + iw) * x.cstride;
        const int tap = (kd * KS + kh) * KS + kw;
        if (vec) {
          for (int ci = 0; ci < cin; ci += 4) {
            const float4 q = __ldg(reinterpret_cast<const float4*>(xp + ci));
            const float xv[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const float* wr = sw + ((ci + u) * K3 + tap) * CG;
#pragma unroll
              for (int j = 0; j < CG; ++j) acc[j] = fmaf(xv[u], wr[j], acc[j]);
            }
          }
        } else {
          for (int ci = 0; ci < cin; ++ci) {
            const float xv = __ldg(xp + ci);
            const float* wr = sw + (ci * K3 + tap) * CG;
#pragma unroll
            for (int j = 0; j < CG; ++j) acc[j] = fmaf(xv, wr[j], acc[j]);
          }
        }
      }
    }
  }
  float* yp = y.ptr + b * y.bstride + v * y.cstride + co0;
#pragma unroll
  for (int j = 0; j < CG; ++j) yp[j] = accumulate ? yp[j] + acc[j] : acc[j];
}

// gx[v][ci0..ci0+CG) = sum_{tap,co} gy[o(v,tap)][co] * W[co][ci][tap]
template <int KS, int CG>
__global__ void __launch_bounds__(128) conv_dgrad_direct_k(d2ip_act gy, const float* __restrict__ w,
                                                           long long wbs, int stride, d2ip_act gx,
                                                           int accumulate, int vec, int dil) {
  D2IP_PDL_ENTRY();
  constexpr int K3 = Taps<KS>::K3, PAD = Taps<KS>::PAD;
  extern __shared__ float sw[];  // [cout][K3][CG]
  const int b = blockIdx.z;
  const int cin = gx.c, cout = gy.c, ci0 = blockIdx.y * CG;
  const float* wb = w + b * wbs;
  for (int i = threadIdx.x; i < cout * K3 * CG; i += blockDim.x) {
    const int j = i % CG, r = i / CG, tap = r % K3, co = r / K3;
    sw[i] = __ldg(wb + ((long long)co * cin + ci0 + j) * K3 + tap);
  }
  __syncthreads();
  const long long V = (long long)gx.d * gx.h * gx.w;
  const long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= V) return;
  const int iw = (int)(v % gx.w), ih = (int)((v / gx.w) % gx.h), id = (int)(v / ((long long)gx.w * gx.h));
  const float* gb = gy.ptr + b * gy.bstride;
  float acc[CG];
#pragma unroll
  for (int j = 0; j < CG; ++j) acc[j] = 0.f;
  for (int kd = 0; kd < KS; ++kd) {
    const int td = id + (PAD - kd) * dil;
    if (td < 0 || td % stride) continue;
    const int od = td / stride;
    if (od >= gy.d) continue;
    for (int kh = 0; kh < KS; ++kh) {
      const int th = ih + (PAD - kh) * dil;
      if (th < 0 || th % stride) continue;
      const int oh = th / stride;
      if (oh >= gy.h) continue;
      for (int kw = 0; kw < KS; ++kw) {
        const int tw = iw + (PAD - kw) * dil;
        if (tw < 0 || tw % stride) continue;
        const int ow = tw / stride;
        if (ow >= gy.w) continue;
        const float* gp = gb + (((long long)od * gy.h + oh) * gy.w + ow) * gy.cstride;
        const int tap = (kd * KS + kh) * KS + kw;
        if (vec) {
          for (int co = 0; co < cout; co += 4) {
            const float4 q = __ldg(reinterpret_cast<const float4*>(gp + co));
            const float gv[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const float* wr = sw + ((co + u) * K3 + tap) * CG;
#pragma unroll
              for (int j = 0; j < CG; ++j) acc[j] = fmaf(gv[u], wr[j], acc[j]);
            }
          }
        } else {
          for (int co = 0; co < cout; ++co) {
            const float gv = __ldg(gp + co);
            const float* wr = sw + (co * K3 + tap) * CG;
#pragma unroll
            for (int j = 0; j < CG; ++j) acc[j] = fmaf(gv, wr[j], acc[j]);
          }
        }
      }
    }
  }
  float* xp = gx.ptr + b * gx.bstride + v * gx.cstride + ci0;
#pragma unroll
  for (int j = 0; j < CG; ++j) xp[j] = accumulate ? xp[j] + acc[j] : acc[j];
}

// Split-K partial weight gradient: one thread per (co, ci, tap) entry (plus
// one per bias entry), summing its chunk of output voxels.
template <int KS>
__global__ void __launch_bounds__(256) conv_wgrad_partial_k(d2ip_act x, d2ip_act gy, int stride,
                                                            float* __restrict__ partial, int nchunks,
                                                            int chunk) {
  D2IP_PDL_ENTRY();
  constexpr int K3 = Taps<KS>::K3, PAD = Taps<KS>::PAD;
  const int b = blockIdx.z, c = blockIdx.y;
  const int cin = x.c, cout = gy.c;
  const int nW = cout * cin * K3, nE = nW + cout;
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= nE) return;
  const long long V = (long long)gy.d * gy.h * gy.w;
  const long long v0 = (long long)c * chunk;
  const long long v1 = min(V, v0 + chunk);
  const float* gb = gy.ptr + b * gy.bstride;
  float acc = 0.f;
  if (e >= nW) {
    const int co = e - nW;
    for (long long v = v0; v < v1; ++v) acc += __ldg(gb + v * gy.cstride + co);
  } else {
    const int co = e / (cin * K3);
    const int rem = e - co * cin * K3;
    const int ci = rem / K3, tap = rem - ci * K3;
    const int kd = tap / (KS * KS), kh = (tap / KS) % KS, kw = tap % KS;
    const float* xb = x.ptr + b * x.bstride;
    for (long long v = v0; v < v1; ++v) {
      const int ow = (int)(v % gy.w), oh = (int)((v / gy.w) % gy.h), od = (int)(v / ((long long)gy.w * gy.h));
      const int id = od * stride + kd - PAD, ih = oh * stride + kh - PAD, iw = ow * stride + kw - PAD;
      if (id < 0 || id >= x.d || ih < 0 || ih >= x.h || iw < 0 || iw >= x.w) continue;
      acc = fmaf(__ldg(gb + v * gy.cstride + co),
                 __ldg(xb + (((long long)id * x.h + ih) * x.w + iw) * x.cstride + ci), acc);
    }
  }
  partial[((long long)b * nchunks + c) * nE + e] = acc;
}

// Register-tiled split-K weight gradient: one thread owns a 4 (C_in) x COG
// (C_out) tile of one tap (or, for tap == K3, COG bias entries) and streams
// its chunk of output voxels, 1-2 float4 loads of gy and one float4 load of x
// per 4*COG FMAs. Output layout matches conv_wgrad_partial_k (OIDHW + bias).
template <int KS, int COG>
__global__ void __launch_bounds__(128) conv_wgrad_tiled_k(d2ip_act x, d2ip_act gy, int stride,
                                                          float* __restrict__ partial, int nchunks, int chunk,
                                                          int dil) {
  D2IP_PDL_ENTRY();
  constexpr int K3 = Taps<KS>::K3, PAD = Taps<KS>::PAD;
  const int b = blockIdx.z, c = blockIdx.y;
  const int cin = x.c, cout = gy.c;
  const int nci = cin >> 2, nco = cout / COG;
  const int gid = blockIdx.x * blockDim.x + threadIdx.x;
  const int ngroups = (K3 + 1) * nci * nco;
  if (gid >= ngroups) return;
  const int cog = gid % nco;
  const int rest = gid / nco;
  const int ci4 = rest % nci;
  const int t = rest / nci;
  if (t == K3 && ci4 != 0) return;  // bias groups: one per co-group
  const int co0 = cog * COG, ci0 = ci4 * 4;
  const int nW = cout * cin * K3, nE = nW + cout;
  const long long V = (long long)gy.d * gy.h * gy.w;
  const long long v0 = (long long)c * chunk;
  const long long v1 = min(V, v0 + chunk);
  const float* gb = gy.ptr + b * gy.bstride + co0;
  float acc[4][COG];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < COG; ++j) acc[i][j] = 0.f;
  // partial layout: [b][chunk][gid][4 * COG], contiguous per thread
  float* pout = partial + (((long long)b * nchunks + c) * ngroups + gid) * (4 * COG);
  if (t == K3) {
    for (long long v = v0; v < v1; ++v) {
      const float* g = gb + v * gy.cstride;
#pragma unroll
      for (int j = 0; j < COG; ++j) acc[0][j] += __ldg(g + j);
    }
#pragma unroll
    for (int j = 0; j < COG; ++j) pout[j] = acc[0][j];
    return;
  }
  const int kd = t / (KS * KS), kh = (t / KS) % KS, kw = t % KS;
  const float* xb = x.ptr + b * x.bstride + ci0;
  int ow = (int)(v0 % gy.w), oh = (int)((v0 / gy.w) % gy.h), od = (int)(v0 / ((long long)gy.w * gy.h));
  for (long long v = v0; v < v1; ++v) {
    const int id = od * stride + (kd - PAD) * dil, ih = oh * stride + (kh - PAD) * dil,
              iw = ow * stride + (kw - PAD) * dil;
    if (id >= 0 && id < x.d && ih >= 0 && ih < x.h && iw >= 0 && iw < x.w) {
      const float4 xv = __ldg(reinterpret_cast<const float4*>(xb + (((long long)id * x.h + ih) * x.w + iw) * x.cstride));
      float g[COG];
      const float* gp = gb + v * gy.cstride;
      if constexpr (COG % 4 == 0) {
#pragma unroll
        for (int j = 0; j < COG; j += 4) {
          const float4 q = __ldg(reinterpret_cast<const float4*>(gp + j));
          g[j] = q.x; g[j + 1] = q.y; g[j + 2] = q.z; g[j + 3] = q.w;
        }
      } else {
#pragma unroll
        for (int j = 0; j < COG; ++j) g[j] = __ldg(gp + j);
      }
#pragma unroll
      for (int j = 0; j < COG; ++j) {
        acc[0][j] = fmaf(xv.x, g[j], acc[0][j]);
        acc[1][j] = fmaf(xv.y, g[j], acc[1][j]);
        acc[2][j] = fmaf(xv.z, g[j], acc[2][j]);
        acc[3][j] = fmaf(xv.w, g[j], acc[3][j]);
      }
    }
    if (++ow == gy.w) {
      ow = 0;
      if (++oh == gy.h) {
        oh = 0;
        ++od;
      }
    }
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < COG; ++j) pout[i * COG + j] = acc[i][j];
  (void)nE;
}

// Sum the thread-contiguous partials of conv_wgrad_tiled_k over chunks (fixed
// order) and scatter into the OIDHW weight + bias gradient.
// Block = 32 consecutive partial entries x 8 warps; warp w sums chunks w, w+8,
// ... (4-way unrolled), then warp 0 adds the 8 warp sums in order.
__global__ void __launch_bounds__(256) wgrad_tiled_reduce_k(const float* __restrict__ partial, int nchunks,
                                                            int ngroups, int cin, int cout, int K3, int cog,
                                                            float* __restrict__ out, long long obs) {
  D2IP_PDL_ENTRY();
  __shared__ float red[8][33];
  const int b = blockIdx.y;
  const long long stride = (long long)ngroups * 4 * cog;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int j = blockIdx.x * 32 + lane;  // index in the tiled layout (coalesced reads)
  float s = 0.f;
  if (j < stride) {
    const float* p = partial + (long long)b * nchunks * stride + j;
    int c = w;
    float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
    for (; c + 24 < nchunks; c += 32) {
      s0 += p[(long long)c * stride];
      s1 += p[(long long)(c + 8) * stride];
      s2 += p[(long long)(c + 16) * stride];
      s3 += p[(long long)(c + 24) * stride];
    }
    for (; c < nchunks; c += 8) s0 += p[(long long)c * stride];
    s = (s0 + s1) + (s2 + s3);
  }
  red[w][lane] = s;
  __syncthreads();
  if (w != 0 || j >= stride) return;
  s = 0.f;
#pragma unroll
  for (int q = 0; q < 8; ++q) s += red[q][lane];
  const int nci = cin >> 2, nco = cout / cog;
  const int gid = j / (4 * cog), slot = j - gid * 4 * cog;
  const int t = gid / (nci * nco), ci4 = (gid / nco) % nci, cg = gid % nco;
  const int i = slot / cog, jj = slot - i * cog;
  const int co = cg * cog + jj, ci = ci4 * 4 + i;
  long long e;
  if (t < K3) {
    e = ((long long)co * cin + ci) * K3 + t;
  } else {
    if (ci4 != 0 || i != 0) return;  // bias groups store COG values
    e = (long long)cout * cin * K3 + co;
  }
  out[b * obs + e] = s;
}

// out[e] = sum_c partial[c][e], fixed order: warp w sums chunks w, w+8, ...,
// then warp 0 adds the 8 warp sums in order.
__global__ void __launch_bounds__(256) reduce_chunks_k(const float* __restrict__ partial, int nchunks, int n,
                                                       float* out, long long obs) {
  D2IP_PDL_ENTRY();
  __shared__ float red[8][33];
  const int b = blockIdx.y;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int e = blockIdx.x * 32 + lane;
  float s = 0.f;
  if (e < n) {
    const float* p = partial + (long long)b * nchunks * n + e;
    float s0 = 0.f, s1 = 0.f;
    int c = w;
    for (; c + 8 < nchunks; c += 16) {
      s0 += p[(long long)c * n];
      s1 += p[(long long)(c + 8) * n];
    }
    for (; c < nchunks; c += 8) s0 += p[(long long)c * n];
    s = s0 + s1;
  }
  red[w][lane] = s;
  __syncthreads();
  if (w != 0 || e >= n) return;
  s = 0.f;
#pragma unroll
  for (int q = 0; q < 8; ++q) s += red[q][lane];
  out[b * obs + e] = s;
}

int reduce_chunks(const float* partial, int nchunks, int n, float* out, long long obs, int batch,
                  cudaStream_t st) {
  dim3 grid(cdiv(n, 32), batch);
  D2IP_CUDA(launch_pdl(reduce_chunks_k, grid, 256, 0, st, partial, nchunks, n, out, obs));
  D2IP_LAUNCH_CHECK();
  return D2IP_OK;
}

// ---------------------------------------------------------------------------

template <typename K>
static int smem_opt_in(K kernel, size_t bytes) {
  if (bytes > 48 * 1024) D2IP_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
  return D2IP_OK;
}

static bool vec_ok(const d2ip_act& a) { return a.c % 4 == 0 && a.cstride % 4 == 0 && ((uintptr_t)a.ptr & 15) == 0; }

int conv_fwd_direct(d2ip_act x, const float* w, const float* bias, long long wbs, int ks, int stride,
                    d2ip_act y, int accumulate, int batch, cudaStream_t st, int dil) {
  const long long V = (long long)y.d * y.h * y.w;
  const int vec = vec_ok(x) ? 1 : 0;
#define LAUNCH_F(KS_, CG_)                                                                          \
  do {                                                                                              \
    const size_t sm = (size_t)x.c * KS_ * KS_ * KS_ * CG_ * sizeof(float);                          \
    D2IP_CHECK_ARG(sm <= 200 * 1024, "conv3d_fwd: weight slice too large for shared memory");      \
    D2IP_RET(smem_opt_in(conv_fwd_direct_k<KS_, CG_>, sm));                                        \
    dim3 grid(cdiv(V, thr), y.c / CG_, batch);                                                      \
    D2IP_CUDA(launch_pdl((conv_fwd_direct_k<KS_, CG_>), grid, thr, sm, st, x, w, bias, wbs, stride, y, accumulate, vec, dil)); \
  } while (0)
  // small layers: narrower channel groups and 64-thread blocks to fill the SMs
  const bool small = V * (y.c / 8 + 1) * batch < 296LL * 128;
  const int cg = (y.c % 8 == 0 && !small) ? 8 : (y.c % 4 == 0 ? 4 : 1);
  const int thr = small ? 64 : 128;
  if (ks == 3) {
    if (cg == 8) LAUNCH_F(3, 8); else if (cg == 4) LAUNCH_F(3, 4); else LAUNCH_F(3, 1);
  } else {
    if (cg == 8) LAUNCH_F(1, 8); else if (cg == 4) LAUNCH_F(1, 4); else LAUNCH_F(1, 1);
  }
#undef LAUNCH_F
  set_variant("direct_fp32");
  D2IP_LAUNCH_CHECK();
  return D2IP_OK;
}

int conv_dgrad_direct(d2ip_act gy, const float* w, long long wbs, int ks, int stride, d2ip_act gx,
                      int accumulate, int batch, cudaStream_t st, int dil) {
  const long long V = (long long)gx.d * gx.h * gx.w;
  const int vec = vec_ok(gy) ? 1 : 0;
#define LAUNCH_D(KS_, CG_)                                                                        \
  do {                                                                                            \
    const size_t sm = (size_t)gy.c * KS_ * KS_ * KS_ * CG_ * sizeof(float);                       \
    D2IP_CHECK_ARG(sm <= 200 * 1024, "conv3d_dgrad: weight slice too large for shared memory");  \
    D2IP_RET(smem_opt_in(conv_dgrad_direct_k<KS_, CG_>, sm));                                    \
    dim3 grid(cdiv(V, thr), gx.c / CG_, batch);                                                   \
    D2IP_CUDA(launch_pdl((conv_dgrad_direct_k<KS_, CG_>), grid, thr, sm, st, gy, w, wbs, stride, gx, accumulate, vec, dil)); \
  } while (0)
  const bool small = V * (gx.c / 8 + 1) * batch < 296LL * 128;
  const int cg = (gx.c % 8 == 0 && !small) ? 8 : (gx.c % 4 == 0 ? 4 : 1);
  const int thr = small ? 64 : 128;
  if (ks == 3) {
    if (cg == 8) LAUNCH_D(3, 8); else if (cg == 4) LAUNCH_D(3, 4); else LAUNCH_D(3, 1);
  } else {
    if (cg == 8) LAUNCH_D(1, 8); else if (cg == 4) LAUNCH_D(1, 4); else LAUNCH_D(1, 1);
  }
#undef LAUNCH_D
  set_variant("direct_fp32");
  D2IP_LAUNCH_CHECK();
  return D2IP_OK;
}

void wgrad_split(int nthreads, long long V, int batch, int* nchunks, int* chunk) {
  long long target = 148LL * 2048;
  long long want = (target + (long long)nthreads * batch - 1) / ((long long)nthreads * batch);
  long long maxc = (V + 255) / 256;  // >= 256 voxels per chunk keeps the partials small
  if (want > maxc) want = maxc;
  if (want < 1) want = 1;
  int c = (int)((V + want - 1) / want);
  *chunk = c;
  *nchunks = (int)((V + c - 1) / c);
}

size_t conv_wgrad_direct_ws(int cin, int cout, int ks, long long V, int batch) {
  const int nE = cout * cin * ks * ks * ks + cout;
  int nchunks, chunk;
  wgrad_split(nE, V, batch, &nchunks, &chunk);
  size_t most = (size_t)batch * nchunks * nE;
  for (int cog : {8, 4, 1}) {  // any tiled variant the views may select
    if (cin % 4 || cout % cog) continue;
    tiled_split(cin, cout, ks, cog, V, batch, &nchunks, &chunk);
    most = std::max(most, (size_t)batch * nchunks * tiled_threads(cin, cout, ks, cog) * 4 * cog);
  }
  return most * sizeof(float);
}

static int tiled_cog(const d2ip_act& x, const d2ip_act& gy) {
  const bool xa = x.c % 4 == 0 && x.cstride % 4 == 0 && ((uintptr_t)x.ptr & 15) == 0;
  const bool ga = gy.cstride % 4 == 0 && ((uintptr_t)gy.ptr & 15) == 0;
  if (!xa) return 0;
  if (gy.c % 8 == 0 && ga) return 8;
  if (gy.c % 4 == 0 && ga) return 4;
  return 1;
}

static int tiled_threads(int cin, int cout, int ks, int cog) {
  return (ks * ks * ks + 1) * (cin / 4) * (cout / cog);
}

// Chunking of the voxel (K) dimension for the tiled kernel: ~600k threads,
// >= 32 voxels per chunk, partials capped at 4M floats.
static void tiled_split(int cin, int cout, int ks, int cog, long long V, int batch, int* nchunks, int* chunk) {
  const long long nthr = tiled_threads(cin, cout, ks, cog);
  const long long per_chunk = nthr * 4 * cog * batch;
  long long want = (148LL * 4096 + nthr * batch - 1) / (nthr * batch);
  want = std::min(want, (V + 31) / 32);
  want = std::min(want, std::max(1LL, (4LL << 20) / per_chunk));
  want = std::min(want, 256LL);  // keeps the fixed-order chunk reduction short
  if (want < 1) want = 1;
  const int c = (int)((V + want - 1) / want);
  *chunk = c;
  *nchunks = (int)((V + c - 1) / c);
}

int conv_wgrad_direct(d2ip_act x, d2ip_act gy, int ks, int stride, float* gw, long long gwbs,
                      void* ws, size_t ws_bytes, int batch, cudaStream_t st, int dil) {
  const int nE = gy.c * x.c * ks * ks * ks + gy.c;
  const long long V = (long long)gy.d * gy.h * gy.w;
  int nchunks, chunk;
  const int cog = tiled_cog(x, gy);
  if (cog) {
    const int nthr = tiled_threads(x.c, gy.c, ks, cog);
    tiled_split(x.c, gy.c, ks, cog, V, batch, &nchunks, &chunk);
    D2IP_CHECK_ARG(ws_bytes >= (size_t)batch * nchunks * nthr * 4 * cog * sizeof(float),
                   "conv3d_wgrad: workspace too small");
    float* partial = reinterpret_cast<float*>(ws);
    dim3 grid(cdiv(nthr, 128), nchunks, batch);
#define LAUNCH_T(KS_, COG_) \
  D2IP_CUDA(launch_pdl((conv_wgrad_tiled_k<KS_, COG_>), grid, 128, 0, st, x, gy, stride, partial, nchunks, chunk, dil))
    if (ks == 3) {
      if (cog == 8) LAUNCH_T(3, 8); else if (cog == 4) LAUNCH_T(3, 4); else LAUNCH_T(3, 1);
    } else {
      if (cog == 8) LAUNCH_T(1, 8); else if (cog == 4) LAUNCH_T(1, 4); else LAUNCH_T(1, 1);
    }
#undef LAUNCH_T
    D2IP_LAUNCH_CHECK();
    D2IP_CUDA(launch_pdl(wgrad_tiled_reduce_k, dim3(cdiv((long long)nthr * 4 * cog, 32), batch), 256, 0, st, 
        partial, nchunks, nthr, x.c, gy.c, ks * ks * ks, cog, gw, gwbs));
    D2IP_LAUNCH_CHECK();
    return D2IP_OK;
  }
  D2IP_CHECK_ARG(dil == 1, "conv3d_wgrad: dilation needs channel counts that are multiples of 4");
  wgrad_split(nE, V, batch, &nchunks, &chunk);
  D2IP_CHECK_ARG(ws_bytes >= (size_t)batch * nchunks * nE * sizeof(float),
                 "conv3d_wgrad: workspace too small (%zu < %zu)", ws_bytes,
                 (size_t)batch * nchunks * nE * sizeof(float));
  float* partial = reinterpret_cast<float*>(ws);
  dim3 grid(cdiv(nE, 256), nchunks, batch);
  if (ks == 3)
    D2IP_CUDA(launch_pdl(conv_wgrad_partial_k<3>, grid, 256, 0, st, x, gy, stride, partial, nchunks, chunk));
  else
    D2IP_CUDA(launch_pdl(conv_wgrad_partial_k<1>, grid, 256, 0, st, x, gy, stride, partial, nchunks, chunk));
  D2IP_LAUNCH_CHECK();
  return reduce_chunks(partial, nchunks, nE, gw, gwbs, batch, st);
}

}  // namespace d2ip
