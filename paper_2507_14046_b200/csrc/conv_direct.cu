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
static void tiled_split(int cin, int cout, int ks, int cog, long long V, int batch, int* nchunks, int* chunk,
                        int* lanes = nullptr);

template <int KS>
struct Taps {
  static constexpr int K3 = KS * KS * KS;
  static constexpr int PAD = KS / 2;
};

// Direct convolutions (stride 2, 1^3, dilated, odd channel counts, the C_out
// = 1 tail, and precision FP32). A block owns CG output channels and VB
// voxels; the CG x C_in x k^3 weight slice sits in shared memory as
// [c][tap][CG] so every (c, tap) step is one float4-vectorised input load (4
// channels) against broadcast shared-memory weights. Small layers (a few
// thousand output voxels) would leave each thread a long serial chain of
// 27 x C_in steps, so the taps are split S ways across the threads of a block
// (S = 3 with VB = 64, or S = 9 with VB = 32): slice s takes taps s, s+S, ... and the S partial
// sums are added in slice order through shared memory (deterministic).

// y[v][co0..co0+CG) = sum_{tap,ci} x[in(v,tap)][ci] * W[co][ci][tap]
template <int KS, int CG, int S>
__global__ void __launch_bounds__(288) conv_fwd_direct_k(d2ip_act x, const float* __restrict__ w,
                                                         const float* __restrict__ bias,
                                                         long long wbs, int stride, d2ip_act y,
                                                         int accumulate, int vec, int dil) {
  D2IP_PDL_ENTRY();
  constexpr int K3 = Taps<KS>::K3, PAD = Taps<KS>::PAD;
  extern __shared__ float sw[];  // [cin][K3][CG], then (S > 1) [S][VB][CG] partial sums
  const int b = blockIdx.z;
  const int cin = x.c, co0 = blockIdx.y * CG;
  const int VB = S == 1 ? (int)blockDim.x : (S == 9 ? 32 : 64);
  const int sl = (int)threadIdx.x / VB, vl = (int)threadIdx.x % VB;
  const float* wb = w + b * wbs;
  for (int i = threadIdx.x; i < cin * K3 * CG; i += blockDim.x) {
    const int j = i % CG, r = i / CG, tap = r % K3, ci = r / K3;
    sw[i] = __ldg(wb + ((long long)(co0 + j) * cin + ci) * K3 + tap);
  }
  __syncthreads();
  const long long V = (long long)y.d * y.h * y.w;
  const long long v = (long long)blockIdx.x * VB + vl;
  const bool live = v < V;
  if (S == 1 && !live) return;
  const long long vv = live ? v : 0;
  const int ow = (int)(vv % y.w), oh = (int)((vv / y.w) % y.h), od = (int)(vv / ((long long)y.w * y.h));
  float acc[CG];
#pragma unroll
  for (int j = 0; j < CG; ++j) acc[j] = (bias && sl == 0) ? __ldg(bias + b * wbs + co0 + j) : 0.f;
  const float* xb = x.ptr + b * x.bstride;
  for (int tap = sl; live && tap < K3; tap += S) {
    const int kd = tap / (KS * KS), kh = (tap / KS) % KS, kw = tap % KS;
    const int id = od * stride + (kd - PAD) * dil;
    const int ih = oh * stride + (kh - PAD) * dil;
    const int iw = ow * stride + (kw - PAD) * dil;
    if (id < 0 || id >= x.d || ih < 0 || ih >= x.h || iw < 0 || iw >= x.w) continue;
    const float* xp = xb + (((long long)id * x.h + ih) * x.w + iw) * x.cstride;
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
  if constexpr (S > 1) {
    float* red = sw + cin * K3 * CG;
#pragma unroll
    for (int j = 0; j < CG; ++j) red[(sl * VB + vl) * CG + j] = acc[j];
    __syncthreads();
    if (sl != 0 || !live) return;
#pragma unroll
    for (int j = 0; j < CG; ++j) {
      float t = red[vl * CG + j];
      for (int q = 1; q < S; ++q) t += red[(q * VB + vl) * CG + j];
      acc[j] = t;
    }
  }
  float* yp = y.ptr + b * y.bstride + v * y.cstride + co0;
#pragma unroll
  for (int j = 0; j < CG; ++j) yp[j] = accumulate ? yp[j] + acc[j] : acc[j];
}

// gx[v][ci0..ci0+CG) = sum_{tap,co} gy[o(v,tap)][co] * W[co][ci][tap]
template <int KS, int CG, int S>
__global__ void __launch_bounds__(288) conv_dgrad_direct_k(d2ip_act gy, const float* __restrict__ w,
                                                           long long wbs, int stride, d2ip_act gx,
                                                           int accumulate, int vec, int dil) {
  D2IP_PDL_ENTRY();
  constexpr int K3 = Taps<KS>::K3, PAD = Taps<KS>::PAD;
  extern __shared__ float sw[];  // [cout][K3][CG], then (S > 1) [S][VB][CG] partial sums
  const int b = blockIdx.z;
  const int cin = gx.c, cout = gy.c, ci0 = blockIdx.y * CG;
  const int VB = S == 1 ? (int)blockDim.x : (S == 9 ? 32 : 64);
  const int sl = (int)threadIdx.x / VB, vl = (int)threadIdx.x % VB;
  const float* wb = w + b * wbs;
  for (int i = threadIdx.x; i < cout * K3 * CG; i += blockDim.x) {
    const int j = i % CG, r = i / CG, tap = r % K3, co = r / K3;
    sw[i] = __ldg(wb + ((long long)co * cin + ci0 + j) * K3 + tap);
  }
  __syncthreads();
  const long long V = (long long)gx.d * gx.h * gx.w;
  const long long v = (long long)blockIdx.x * VB + vl;
  const bool live = v < V;
  if (S == 1 && !live) return;
  const long long vv = live ? v : 0;
  const int iw = (int)(vv % gx.w), ih = (int)((vv / gx.w) % gx.h), id = (int)(vv / ((long long)gx.w * gx.h));
  const float* gb = gy.ptr + b * gy.bstride;
  float acc[CG];
#pragma unroll
  for (int j = 0; j < CG; ++j) acc[j] = 0.f;
  for (int tap = sl; live && tap < K3; tap += S) {
    const int kd = tap / (KS * KS), kh = (tap / KS) % KS, kw = tap % KS;
    const int td = id + (PAD - kd) * dil, th = ih + (PAD - kh) * dil, tw = iw + (PAD - kw) * dil;
    if (td < 0 || th < 0 || tw < 0 || td % stride || th % stride || tw % stride) continue;
    const int od = td / stride, oh = th / stride, ow = tw / stride;
    if (od >= gy.d || oh >= gy.h || ow >= gy.w) continue;
    const float* gp = gb + (((long long)od * gy.h + oh) * gy.w + ow) * gy.cstride;
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
  if constexpr (S > 1) {
    float* red = sw + cout * K3 * CG;
#pragma unroll
    for (int j = 0; j < CG; ++j) red[(sl * VB + vl) * CG + j] = acc[j];
    __syncthreads();
    if (sl != 0 || !live) return;
#pragma unroll
    for (int j = 0; j < CG; ++j) {
      float t = red[vl * CG + j];
      for (int q = 1; q < S; ++q) t += red[(q * VB + vl) * CG + j];
      acc[j] = t;
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

// Register-tiled split-K weight gradient: a group of L consecutive threads
// owns a 4 (C_in) x COG (C_out) tile of one tap (or, for tap == K3, COG bias
// entries); each thread streams a contiguous 1/L of the group's chunk of
// output voxels (1-2 float4 loads of gy and one float4 load of x per 4*COG
// FMAs) and the L partial tiles are combined by a fixed shuffle tree
// (deterministic). L > 1 gives small layers more threads without more
// partials. Output layout matches conv_wgrad_partial_k (OIDHW + bias).
template <int KS, int COG, int L>
__global__ void __launch_bounds__(128) conv_wgrad_tiled_k(d2ip_act x, d2ip_act gy, int stride,
                                                          float* __restrict__ partial, int nchunks, int chunk,
                                                          int dil) {
  D2IP_PDL_ENTRY();
  constexpr int K3 = Taps<KS>::K3, PAD = Taps<KS>::PAD;
  const int b = blockIdx.z, c = blockIdx.y;
  const int cin = x.c, cout = gy.c;
  const int nci = cin >> 2, nco = cout / COG;
  const int gid = (blockIdx.x * blockDim.x + threadIdx.x) / L;
  const int q = threadIdx.x % L;
  const int ngroups = (K3 + 1) * nci * nco;
  const int cog = gid % nco;
  const int rest = gid / nco;
  const int ci4 = rest % nci;
  const int t = rest / nci;
  // whole groups share `valid`, so the shuffle tree below never mixes live and dead lanes
  const bool valid = gid < ngroups && !(t == K3 && ci4 != 0);  // bias groups: one per co-group
  const int co0 = cog * COG, ci0 = ci4 * 4;
  const long long V = (long long)gy.d * gy.h * gy.w;
  const long long c0 = (long long)c * chunk, c1 = min(V, c0 + chunk);
  const long long sub = (c1 - c0 + L - 1) / L;
  const long long v0 = min(c1, c0 + q * sub), v1 = min(c1, v0 + sub);
  const float* gb = gy.ptr + b * gy.bstride + co0;
  float acc[4][COG];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < COG; ++j) acc[i][j] = 0.f;
  if (valid && t == K3) {
    for (long long v = v0; v < v1; ++v) {
      const float* g = gb + v * gy.cstride;
#pragma unroll
      for (int j = 0; j < COG; ++j) acc[0][j] += __ldg(g + j);
    }
  } else if (valid) {
    const int kd = t / (KS * KS), kh = (t / KS) % KS, kw = t % KS;
    const float* xb = x.ptr + b * x.bstride + ci0;
    int ow = (int)(v0 % gy.w), oh = (int)((v0 / gy.w) % gy.h), od = (int)(v0 / ((long long)gy.w * gy.h));
    for (long long v = v0; v < v1; ++v) {
      const int id = od * stride + (kd - PAD) * dil, ih = oh * stride + (kh - PAD) * dil,
                iw = ow * stride + (kw - PAD) * dil;
      if (id >= 0 && id < x.d && ih >= 0 && ih < x.h && iw >= 0 && iw < x.w) {
        const float4 xv =
            __ldg(reinterpret_cast<const float4*>(xb + (((long long)id * x.h + ih) * x.w + iw) * x.cstride));
        float g[COG];
        const float* gp = gb + v * gy.cstride;
        if constexpr (COG % 4 == 0) {
#pragma unroll
          for (int j = 0; j < COG; j += 4) {
            const float4 qq = __ldg(reinterpret_cast<const float4*>(gp + j));
            g[j] = qq.x; g[j + 1] = qq.y; g[j + 2] = qq.z; g[j + 3] = qq.w;
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
  }
  if constexpr (L > 1) {
#pragma unroll
    for (int off = L / 2; off >= 1; off >>= 1)
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < COG; ++j) acc[i][j] += __shfl_down_sync(0xffffffffu, acc[i][j], off, L);
  }
  if (!valid || q != 0) return;
  // partial layout: [b][chunk][gid][4 * COG], contiguous per group
  float* pout = partial + (((long long)b * nchunks + c) * ngroups + gid) * (4 * COG);
  if (t == K3) {
#pragma unroll
    for (int j = 0; j < COG; ++j) pout[j] = acc[0][j];
    return;
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < COG; ++j) pout[i * COG + j] = acc[i][j];
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

// out[e] = sum_c partial[c][e], fixed order: 32 warps per block, warp w sums chunks w, w+32,
// ... in four interleaved partial sums (chunk w + 32 (4i + j) into sum j), then warp 0 adds
// the 32 warp sums in order. Deterministic; 1,024 threads and four loads in flight per lane
// keep the long chunk lists (up to 1,184 LayerNorm-backward blocks) off the latency chain.
__global__ void __launch_bounds__(1024) reduce_chunks_k(const float* __restrict__ partial, int nchunks, int n,
                                                        float* out, long long obs) {
  D2IP_PDL_ENTRY();
  __shared__ float red[32][33];
  const int b = blockIdx.y;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int e = blockIdx.x * 32 + lane;
  float s = 0.f;
  if (e < n) {
    const float* p = partial + (long long)b * nchunks * n + e;
    float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
    int c = w;
    for (; c + 96 < nchunks; c += 128) {
      const float a0 = __ldg(p + (long long)c * n), a1 = __ldg(p + (long long)(c + 32) * n);
      const float a2 = __ldg(p + (long long)(c + 64) * n), a3 = __ldg(p + (long long)(c + 96) * n);
      s0 += a0;
      s1 += a1;
      s2 += a2;
      s3 += a3;
    }
    for (; c < nchunks; c += 32) s0 += __ldg(p + (long long)c * n);
    s = (s0 + s1) + (s2 + s3);
  }
  red[w][lane] = s;
  __syncthreads();
  if (w != 0 || e >= n) return;
  s = 0.f;
#pragma unroll
  for (int q = 0; q < 32; ++q) s += red[q][lane];
  out[b * obs + e] = s;
}

int reduce_chunks(const float* partial, int nchunks, int n, float* out, long long obs, int batch,
                  cudaStream_t st) {
  dim3 grid(cdiv(n, 32), batch);
  D2IP_CUDA(launch_pdl(reduce_chunks_k, grid, 1024, 0, st, partial, nchunks, n, out, obs));
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

// Launch plan of a direct fwd / dgrad: channel group CG, tap split S, threads.
struct DirectPlan {
  int cg, S, thr;
  long long vb;  // voxels per block
};
// `live_taps`: taps that actually contribute per output voxel (27, or ~27/8
// for the data gradient of a stride-2 convolution, where only taps of matching
// parity land on a given input voxel) -- the serial chain the split shortens.
static DirectPlan direct_plan(long long V, int C, int ks, int batch, int live_taps, int Cred) {
  DirectPlan p;
  const bool small = V * (C / 8 + 1) * batch < 296LL * 128;
  p.cg = (C % 8 == 0 && !small) ? 8 : (C % 4 == 0 ? 4 : 1);
  // the Cred x k^3 x CG weight slice must fit shared memory (wide decoder inputs at cfg4)
  const long long k3 = (long long)ks * ks * ks;
  while (p.cg > 1 && Cred * k3 * p.cg * 4 + 288LL * p.cg * 4 > 200LL * 1024) p.cg = p.cg == 8 ? 4 : 1;
  const long long base = V * (C / p.cg) * batch;  // threads without a tap split
  p.S = 1;
  if (ks == 3 && live_taps >= 27) p.S = base < 48LL * 1024 ? 9 : (base < 128LL * 1024 ? 3 : 1);
  if (ks == 3 && live_taps < 27 && base < 48LL * 1024) p.S = 9;
  p.vb = p.S == 9 ? 32 : (p.S == 3 ? 64 : 0);
  p.thr = p.S > 1 ? (int)p.vb * p.S : (small ? 64 : 128);
  // a large weight slice per block (e.g. a stride-2 data gradient, 32 x 27 x 8
  // floats) is amortised over more voxels when there is parallelism to spare
  if (p.S == 1 && !small && Cred * (long long)ks * ks * ks * p.cg >= 2048 && base >= 64LL * 1024) p.thr = 256;
  if (p.S == 1) p.vb = p.thr;
  return p;
}

// ---------------------------------------------------------------------------
// 1^3 stride-2 convolutions (the encoder blocks' skip path): y[o] = b + W x[2o]
// and its data gradient gx[2o] = W^T gy[o] (gx = 0 at the other seven parities).
// Lane groups: G = C / 4 lanes share an output voxel and own 4 channels each;
// the weights sit in shared memory transposed for float4 reads, the voxel's
// input row is read once by the group (128-bit loads, L1 broadcast), and every
// store is a coalesced float4 -- the generic direct kernel re-derived taps and
// strided indices per thread (up to 15x slower on cfg4's 442 K-voxel level).

template <int G>
__global__ void __launch_bounds__(256) pw_s2_fwd_k(d2ip_act x, const float* __restrict__ w,
                                                   const float* __restrict__ bias, long long wbs, d2ip_act y,
                                                   int accumulate) {
  D2IP_PDL_ENTRY();
  extern __shared__ float4 sw4[];  // [ci][G]: W[4 l .. 4 l + 3][ci]
  const int b = blockIdx.y, cin = x.c;
  const float* wb = w + b * wbs;
  for (int i = threadIdx.x; i < cin * G; i += blockDim.x) {
    const int ci = i / G, l = i % G;
    sw4[i] = make_float4(__ldg(wb + (4 * l) * cin + ci), __ldg(wb + (4 * l + 1) * cin + ci),
                         __ldg(wb + (4 * l + 2) * cin + ci), __ldg(wb + (4 * l + 3) * cin + ci));
  }
  __syncthreads();
  const long long V = (long long)y.d * y.h * y.w;
  const long long o = ((long long)blockIdx.x * blockDim.x + threadIdx.x) / G;
  const int l = threadIdx.x % G;
  if (o >= V) return;
  const int ow = (int)(o % y.w), oh = (int)((o / y.w) % y.h), od = (int)(o / ((long long)y.w * y.h));
  const float* xr = x.ptr + b * x.bstride + (((long long)(2 * od) * x.h + 2 * oh) * x.w + 2 * ow) * x.cstride;
  float4 acc = bias ? make_float4(__ldg(bias + b * wbs + 4 * l), __ldg(bias + b * wbs + 4 * l + 1),
                                  __ldg(bias + b * wbs + 4 * l + 2), __ldg(bias + b * wbs + 4 * l + 3))
                    : make_float4(0.f, 0.f, 0.f, 0.f);
  for (int c0 = 0; c0 < cin; c0 += 4) {
    const float4 q = __ldg(reinterpret_cast<const float4*>(xr + c0));
    const float qq[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float4 wq = sw4[(c0 + j) * G + l];
      acc.x = fmaf(qq[j], wq.x, acc.x);
      acc.y = fmaf(qq[j], wq.y, acc.y);
      acc.z = fmaf(qq[j], wq.z, acc.z);
      acc.w = fmaf(qq[j], wq.w, acc.w);
    }
  }
  float4* yp = reinterpret_cast<float4*>(y.ptr + b * y.bstride + o * y.cstride + 4 * l);
  if (accumulate) {
    const float4 p0 = *yp;
    acc.x += p0.x; acc.y += p0.y; acc.z += p0.z; acc.w += p0.w;
  }
  *yp = acc;
}

template <int G>
__global__ void __launch_bounds__(256) pw_s2_dgrad_k(d2ip_act gy, const float* __restrict__ w, long long wbs,
                                                     d2ip_act gx, int accumulate) {
  D2IP_PDL_ENTRY();
  extern __shared__ float4 sw4[];  // [co][G]: W[co][4 l .. 4 l + 3]
  const int b = blockIdx.y, cout = gy.c, cin = gx.c;
  const float* wb = w + b * wbs;
  for (int i = threadIdx.x; i < cout * G; i += blockDim.x) {
    const int co = i / G, l = i % G;
    const float* r = wb + (long long)co * cin + 4 * l;  // (theta offsets need not be 16-byte aligned)
    sw4[i] = make_float4(__ldg(r), __ldg(r + 1), __ldg(r + 2), __ldg(r + 3));
  }
  __syncthreads();
  const long long V = (long long)gx.d * gx.h * gx.w;
  const long long v = ((long long)blockIdx.x * blockDim.x + threadIdx.x) / G;
  const int l = threadIdx.x % G;
  if (v >= V) return;
  const int iw = (int)(v % gx.w), ih = (int)((v / gx.w) % gx.h), id = (int)(v / ((long long)gx.w * gx.h));
  float4* gp = reinterpret_cast<float4*>(gx.ptr + b * gx.bstride + v * gx.cstride + 4 * l);
  if ((iw | ih | id) & 1) {  // no output voxel reads an odd-parity input
    if (!accumulate) *gp = make_float4(0.f, 0.f, 0.f, 0.f);
    return;
  }
  const float* gr = gy.ptr + b * gy.bstride + (((long long)(id >> 1) * gy.h + (ih >> 1)) * gy.w + (iw >> 1)) * gy.cstride;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int c0 = 0; c0 < cout; c0 += 4) {
    const float4 q = __ldg(reinterpret_cast<const float4*>(gr + c0));
    const float qq[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float4 wq = sw4[(c0 + j) * G + l];
      acc.x = fmaf(qq[j], wq.x, acc.x);
      acc.y = fmaf(qq[j], wq.y, acc.y);
      acc.z = fmaf(qq[j], wq.z, acc.z);
      acc.w = fmaf(qq[j], wq.w, acc.w);
    }
  }
  if (accumulate) {
    const float4 p0 = *gp;
    acc.x += p0.x; acc.y += p0.y; acc.z += p0.z; acc.w += p0.w;
  }
  *gp = acc;
}

static bool pw_s2_ok(const d2ip_act& in, const d2ip_act& out) {
  const int G = out.c / 4;
  auto al = [](const d2ip_act& a) { return a.cstride % 4 == 0 && ((uintptr_t)a.ptr & 15) == 0; };
  return out.c % 4 == 0 && in.c % 4 == 0 && (G == 1 || G == 2 || G == 4 || G == 8 || G == 16 || G == 32) &&
         al(in) && al(out) && (size_t)in.c * G * 16 <= 96 * 1024;
}

int conv_fwd_direct(d2ip_act x, const float* w, const float* bias, long long wbs, int ks, int stride,
                    d2ip_act y, int accumulate, int batch, cudaStream_t st, int dil) {
  if (ks == 1 && stride == 2 && pw_s2_ok(x, y) && y.d == (x.d + 1) / 2 && y.h == (x.h + 1) / 2 &&
      y.w == (x.w + 1) / 2) {
    const long long Vo = (long long)y.d * y.h * y.w;
    const size_t sm = (size_t)x.c * (y.c / 4) * 16;
    const dim3 grid(cdiv(Vo * (y.c / 4), 256), batch);
#define D2IP_PWF(G_)                                                                                  \
  case G_:                                                                                           \
    D2IP_RET(smem_opt_in(pw_s2_fwd_k<G_>, sm));                                                      \
    D2IP_CUDA(launch_pdl(pw_s2_fwd_k<G_>, grid, 256, sm, st, x, w, bias, wbs, y, accumulate));       \
    break;
    switch (y.c / 4) { D2IP_PWF(1) D2IP_PWF(2) D2IP_PWF(4) D2IP_PWF(8) D2IP_PWF(16) D2IP_PWF(32) }
#undef D2IP_PWF
    set_variant("direct_fp32_pw_s2");
    D2IP_LAUNCH_CHECK();
    return D2IP_OK;
  }
  const long long V = (long long)y.d * y.h * y.w;
  const int vec = vec_ok(x) ? 1 : 0;
  const DirectPlan p = direct_plan(V, y.c, ks, batch, 27, x.c);
#define LAUNCH_F(KS_, CG_, S_)                                                                       \
  do {                                                                                               \
    const size_t sm = ((size_t)x.c * KS_ * KS_ * KS_ * CG_ + (S_ > 1 ? (size_t)p.thr * CG_ : 0)) * sizeof(float); \
    D2IP_CHECK_ARG(sm <= 200 * 1024, "conv3d_fwd: weight slice too large for shared memory");       \
    D2IP_RET(smem_opt_in(conv_fwd_direct_k<KS_, CG_, S_>, sm));                                     \
    dim3 grid(cdiv(V, p.vb), y.c / CG_, batch);                                                      \
    D2IP_CUDA(launch_pdl((conv_fwd_direct_k<KS_, CG_, S_>), grid, p.thr, sm, st, x, w, bias, wbs, stride, y, \
                         accumulate, vec, dil));                                                     \
  } while (0)
  if (ks == 3) {
    if (p.S == 9) {
      if (p.cg == 8) LAUNCH_F(3, 8, 9); else if (p.cg == 4) LAUNCH_F(3, 4, 9); else LAUNCH_F(3, 1, 9);
    } else if (p.S == 3) {
      if (p.cg == 8) LAUNCH_F(3, 8, 3); else if (p.cg == 4) LAUNCH_F(3, 4, 3); else LAUNCH_F(3, 1, 3);
    } else {
      if (p.cg == 8) LAUNCH_F(3, 8, 1); else if (p.cg == 4) LAUNCH_F(3, 4, 1); else LAUNCH_F(3, 1, 1);
    }
  } else {
    if (p.cg == 8) LAUNCH_F(1, 8, 1); else if (p.cg == 4) LAUNCH_F(1, 4, 1); else LAUNCH_F(1, 1, 1);
  }
#undef LAUNCH_F
  set_variant("direct_fp32");
  D2IP_LAUNCH_CHECK();
  return D2IP_OK;
}

int conv_dgrad_direct(d2ip_act gy, const float* w, long long wbs, int ks, int stride, d2ip_act gx,
                      int accumulate, int batch, cudaStream_t st, int dil) {
  if (ks == 1 && stride == 2 && pw_s2_ok(gy, gx) && gy.d == (gx.d + 1) / 2 && gy.h == (gx.h + 1) / 2 &&
      gy.w == (gx.w + 1) / 2) {
    const long long V = (long long)gx.d * gx.h * gx.w;
    const size_t sm = (size_t)gy.c * (gx.c / 4) * 16;
    const dim3 grid(cdiv(V * (gx.c / 4), 256), batch);
#define D2IP_PWD(G_)                                                                                  \
  case G_:                                                                                           \
    D2IP_RET(smem_opt_in(pw_s2_dgrad_k<G_>, sm));                                                    \
    D2IP_CUDA(launch_pdl(pw_s2_dgrad_k<G_>, grid, 256, sm, st, gy, w, wbs, gx, accumulate));          \
    break;
    switch (gx.c / 4) { D2IP_PWD(1) D2IP_PWD(2) D2IP_PWD(4) D2IP_PWD(8) D2IP_PWD(16) D2IP_PWD(32) }
#undef D2IP_PWD
    set_variant("direct_fp32_pw_s2");
    D2IP_LAUNCH_CHECK();
    return D2IP_OK;
  }
  const long long V = (long long)gx.d * gx.h * gx.w;
  const int vec = vec_ok(gy) ? 1 : 0;
  const DirectPlan p = direct_plan(V, gx.c, ks, batch, stride == 1 ? 27 : 4, gy.c);
#define LAUNCH_D(KS_, CG_, S_)                                                                        \
  do {                                                                                                \
    const size_t sm = ((size_t)gy.c * KS_ * KS_ * KS_ * CG_ + (S_ > 1 ? (size_t)p.thr * CG_ : 0)) * sizeof(float); \
    D2IP_CHECK_ARG(sm <= 200 * 1024, "conv3d_dgrad: weight slice too large for shared memory");      \
    D2IP_RET(smem_opt_in(conv_dgrad_direct_k<KS_, CG_, S_>, sm));                                    \
    dim3 grid(cdiv(V, p.vb), gx.c / CG_, batch);                                                      \
    D2IP_CUDA(launch_pdl((conv_dgrad_direct_k<KS_, CG_, S_>), grid, p.thr, sm, st, gy, w, wbs, stride, gx, \
                         accumulate, vec, dil));                                                      \
  } while (0)
  if (ks == 3) {
    if (p.S == 9) {
      if (p.cg == 8) LAUNCH_D(3, 8, 9); else if (p.cg == 4) LAUNCH_D(3, 4, 9); else LAUNCH_D(3, 1, 9);
    } else if (p.S == 3) {
      if (p.cg == 8) LAUNCH_D(3, 8, 3); else if (p.cg == 4) LAUNCH_D(3, 4, 3); else LAUNCH_D(3, 1, 3);
    } else {
      if (p.cg == 8) LAUNCH_D(3, 8, 1); else if (p.cg == 4) LAUNCH_D(3, 4, 1); else LAUNCH_D(3, 1, 1);
    }
  } else {
    if (p.cg == 8) LAUNCH_D(1, 8, 1); else if (p.cg == 4) LAUNCH_D(1, 4, 1); else LAUNCH_D(1, 1, 1);
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
// >= 32 voxels per chunk, partials capped at 4M floats; then L threads per
// group (1..8) when the chunks alone leave the GPU short of threads.
static void tiled_split(int cin, int cout, int ks, int cog, long long V, int batch, int* nchunks, int* chunk,
                        int* lanes) {
  const long long nthr = tiled_threads(cin, cout, ks, cog);
  const long long per_chunk = nthr * 4 * cog * batch;
  const long long target = 148LL * 4096;
  long long want = (target + nthr * batch - 1) / (nthr * batch);
  want = std::min(want, (V + 31) / 32);
  want = std::min(want, std::max(1LL, (4LL << 20) / per_chunk));
  want = std::min(want, 256LL);  // keeps the fixed-order chunk reduction short
  if (want < 1) want = 1;
  const int c = (int)((V + want - 1) / want);
  *chunk = c;
  *nchunks = (int)((V + c - 1) / c);
  int L = 1;
  while (L < 8 && nthr * batch * *nchunks * L * 2 <= target && c >= 16 * L) L *= 2;
  if (lanes) *lanes = L;
}

int conv_wgrad_direct(d2ip_act x, d2ip_act gy, int ks, int stride, float* gw, long long gwbs,
                      void* ws, size_t ws_bytes, int batch, cudaStream_t st, int dil) {
  const int nE = gy.c * x.c * ks * ks * ks + gy.c;
  const long long V = (long long)gy.d * gy.h * gy.w;
  int nchunks, chunk;
  const int cog = tiled_cog(x, gy);
  if (cog) {
    const int nthr = tiled_threads(x.c, gy.c, ks, cog);
    int L = 1;
    tiled_split(x.c, gy.c, ks, cog, V, batch, &nchunks, &chunk, &L);
    D2IP_CHECK_ARG(ws_bytes >= (size_t)batch * nchunks * nthr * 4 * cog * sizeof(float),
                   "conv3d_wgrad: workspace too small");
    float* partial = reinterpret_cast<float*>(ws);
    dim3 grid(cdiv((long long)nthr * L, 128), nchunks, batch);
#define LAUNCH_T(KS_, COG_, L_) \
  D2IP_CUDA(launch_pdl((conv_wgrad_tiled_k<KS_, COG_, L_>), grid, 128, 0, st, x, gy, stride, partial, nchunks, chunk, dil))
#define LAUNCH_TL(KS_, COG_)                         \
  do {                                               \
    if (L == 8) LAUNCH_T(KS_, COG_, 8);              \
    else if (L == 4) LAUNCH_T(KS_, COG_, 4);         \
    else if (L == 2) LAUNCH_T(KS_, COG_, 2);         \
    else LAUNCH_T(KS_, COG_, 1);                     \
  } while (0)
    if (ks == 3) {
      if (cog == 8) LAUNCH_TL(3, 8); else if (cog == 4) LAUNCH_TL(3, 4); else LAUNCH_TL(3, 1);
    } else {
      if (cog == 8) LAUNCH_TL(1, 8); else if (cog == 4) LAUNCH_TL(1, 4); else LAUNCH_TL(1, 1);
    }
#undef LAUNCH_TL
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
