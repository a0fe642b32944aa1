#include <algorithm>
// Kernels of the reference-exact backbone FastResUNet3D (priornet.py:111-232)
// that the canonical config ResUNet does not need:
//   depthwise 3^3 convolution (`_conv3(depthwise=True)`, priornet.py:111-117)
//   SqueezeExcite (priornet.py:120-131)
//   AttentionGate3d element-wise parts (priornet.py:167-180)
// plus SiLU helpers. Dense / dilated / 1^3 convolutions, LayerNorm, the
// trilinear upsample and the split-K reductions reuse the other kernel files.
// All reductions are fixed-order (deterministic).
#include "common.cuh"
#include "kernels.h"

namespace d2ip {

__device__ __forceinline__ float sigm(float x) { return 1.0f / (1.0f + expf(-x)); }
__device__ __forceinline__ float silu(float x) { return x * sigm(x); }
__device__ __forceinline__ float silu_grad(float x) {
  const float s = sigm(x);
  return s * (1.0f + x * (1.0f - s));
}

// ---- depthwise 3^3 (groups = C), padding 1, stride 1/2 ---------------------
// y[v][c] = b[c] + sum_t x[in(v,t)][c] * w[c][t]
__global__ void __launch_bounds__(256) dw_fwd_k(d2ip_act x, const float* __restrict__ w, const float* __restrict__ bias,
                                                long long wbs, int stride, d2ip_act y) {
  D2IP_PDL_ENTRY();
  const int b = blockIdx.y;
  const int C = x.c;
  const long long V = (long long)y.d * y.h * y.w;
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= V * C) return;
  const int c = (int)(i % C);
  const long long v = i / C;
  const int ow = (int)(v % y.w), oh = (int)((v / y.w) % y.h), od = (int)(v / ((long long)y.w * y.h));
  const float* wb = w + b * wbs + c * 27;
  const float* xb = x.ptr + b * x.bstride + c;
  float acc = __ldg(bias + b * wbs + c);
  for (int kd = 0; kd < 3; ++kd) {
    const int id = od * stride + kd - 1;
    if (id < 0 || id >= x.d) continue;
    for (int kh = 0; kh < 3; ++kh) {
      const int ih = oh * stride + kh - 1;
      if (ih < 0 || ih >= x.h) continue;
      for (int kw = 0; kw < 3; ++kw) {
        const int iw = ow * stride + kw - 1;
        if (iw < 0 || iw >= x.w) continue;
        acc = fmaf(xb[(((long long)id * x.h + ih) * x.w + iw) * x.cstride], __ldg(wb + (kd * 3 + kh) * 3 + kw), acc);
      }
    }
  }
  y.ptr[b * y.bstride + v * y.cstride + c] = acc;
}

// gx[u][c] (+)= sum_t gy[o(u,t)][c] * w[c][t]
__global__ void __launch_bounds__(256) dw_dgrad_k(d2ip_act gy, const float* __restrict__ w, long long wbs, int stride,
                                                  d2ip_act gx, int accumulate) {
  D2IP_PDL_ENTRY();
  const int b = blockIdx.y;
  const int C = gx.c;
  const long long V = (long long)gx.d * gx.h * gx.w;
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= V * C) return;
  const int c = (int)(i % C);
  const long long u = i / C;
  const int iw = (int)(u % gx.w), ih = (int)((u / gx.w) % gx.h), id = (int)(u / ((long long)gx.w * gx.h));
  const float* wb = w + b * wbs + c * 27;
  const float* gb = gy.ptr + b * gy.bstride + c;
  float acc = 0.f;
  for (int kd = 0; kd < 3; ++kd) {
    const int td = id + 1 - kd;
    if (td < 0 || td % stride) continue;
    const int od = td / stride;
    if (od >= gy.d) continue;
    for (int kh = 0; kh < 3; ++kh) {
      const int th = ih + 1 - kh;
      if (th < 0 || th % stride) continue;
      const int oh = th / stride;
      if (oh >= gy.h) continue;
      for (int kw = 0; kw < 3; ++kw) {
        const int tw = iw + 1 - kw;
        if (tw < 0 || tw % stride) continue;
        const int ow = tw / stride;
        if (ow >= gy.w) continue;
        acc = fmaf(gb[(((long long)od * gy.h + oh) * gy.w + ow) * gy.cstride], __ldg(wb + (kd * 3 + kh) * 3 + kw), acc);
      }
    }
  }
  float* o = gx.ptr + b * gx.bstride + u * gx.cstride + c;
  *o = accumulate ? *o + acc : acc;
}

// partial[b][chunk][c*27 + t] = sum_v gy[v][c] x[in(v,t)][c];  [27C + c] = sum_v gy[v][c]
// One thread per (channel, voxel chunk) keeps all 27 taps + the bias in
// registers and walks its chunk in order with incremental coordinates (each
// gy value is read once; neighbouring x rows stay in L1).
__global__ void __launch_bounds__(256) dw_wgrad_k(d2ip_act x, d2ip_act gy, int stride, float* __restrict__ partial,
                                                  int nchunks, int chunk) {
  D2IP_PDL_ENTRY();
  const int b = blockIdx.y;
  const int C = x.c;
  const int e = blockIdx.x * blockDim.x + threadIdx.x;  // (chunk, c), c fastest
  if (e >= nchunks * C) return;
  const int c = e % C, ch = e / C;
  const long long V = (long long)gy.d * gy.h * gy.w;
  const long long v0 = (long long)ch * chunk, v1 = min(V, v0 + chunk);
  const float* gb = gy.ptr + b * gy.bstride + c;
  const float* xb = x.ptr + b * x.bstride + c;
  float acc[27], bacc = 0.f;
#pragma unroll
  for (int t = 0; t < 27; ++t) acc[t] = 0.f;
  int ow = (int)(v0 % gy.w), oh = (int)((v0 / gy.w) % gy.h), od = (int)(v0 / ((long long)gy.w * gy.h));
  for (long long v = v0; v < v1; ++v) {
    const float g = gb[v * gy.cstride];
    bacc += g;
#pragma unroll
    for (int kd = 0; kd < 3; ++kd) {
      const int id = od * stride + kd - 1;
      const bool okd = id >= 0 && id < x.d;
#pragma unroll
      for (int kh = 0; kh < 3; ++kh) {
        const int ih = oh * stride + kh - 1;
        const bool okh = okd && ih >= 0 && ih < x.h;
#pragma unroll
        for (int kw = 0; kw < 3; ++kw) {
          const int iw = ow * stride + kw - 1;
          if (okh && iw >= 0 && iw < x.w)
            acc[(kd * 3 + kh) * 3 + kw] =
                fmaf(g, xb[(((long long)id * x.h + ih) * x.w + iw) * x.cstride], acc[(kd * 3 + kh) * 3 + kw]);
        }
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
  float* p = partial + ((long long)b * nchunks + ch) * 28 * C;
#pragma unroll
  for (int t = 0; t < 27; ++t) p[c * 27 + t] = acc[t];
  p[27 * C + c] = bacc;
}

// Lane-group variant (C = 4 G, G <= 16): G lanes share a gy voxel and own 4 channels each
// (float4 loads of gy and of the 27 x taps, coalesced across the group), a CTA walks a
// voxel range, folds its voxel groups with a fixed xor-shuffle tree and its warps in a
// fixed order, and writes one partial [C][27] + [C] per CTA for reduce_chunks (~300
// partials instead of ~1,000 single-channel chunk sums). blockIdx.z = the kd plane:
// nine taps per CTA (36 accumulators per lane instead of 108, several CTAs per SM).
template <int G>
__global__ void __launch_bounds__(256) dw_wgrad_g_k(d2ip_act x, d2ip_act gy, int stride, float* __restrict__ partial,
                                                    int vchunk) {
  D2IP_PDL_ENTRY();
  extern __shared__ float red_dyn[];  // [8 warps][G][27 * 4 + 5]
  auto red = reinterpret_cast<float(*)[G][27 * 4 + 5]>(red_dyn);
  const int b = blockIdx.y, kd = blockIdx.z;
  const int C = 4 * G;
  const long long V = (long long)gy.d * gy.h * gy.w;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, l = lane % G, grp = threadIdx.x / G;
  float4 acc[9];
#pragma unroll
  for (int t = 0; t < 9; ++t) acc[t] = make_float4(0.f, 0.f, 0.f, 0.f);
  float4 bs = make_float4(0.f, 0.f, 0.f, 0.f);
  const float* xb = x.ptr + b * x.bstride + 4 * l;
  const float* gb = gy.ptr + b * gy.bstride + 4 * l;
  const long long v_lo = (long long)blockIdx.x * vchunk, v_hi = min(V, v_lo + vchunk);
  for (long long o = v_lo + grp; o < v_hi; o += 256 / G) {
    const int ow = (int)(o % gy.w), oh = (int)((o / gy.w) % gy.h), od = (int)(o / ((long long)gy.w * gy.h));
    const float4 g = __ldg(reinterpret_cast<const float4*>(gb + o * gy.cstride));
    bs.x += g.x; bs.y += g.y; bs.z += g.z; bs.w += g.w;
    {
      const int id = od * stride + kd - 1;
#pragma unroll
      for (int kh = 0; kh < 3; ++kh) {
        const int ih = oh * stride + kh - 1;
#pragma unroll
        for (int kw = 0; kw < 3; ++kw) {
          const int iw = ow * stride + kw - 1;
          if (id >= 0 && id < x.d && ih >= 0 && ih < x.h && iw >= 0 && iw < x.w) {
            const float4 q = __ldg(reinterpret_cast<const float4*>(xb + (((long long)id * x.h + ih) * x.w + iw) * x.cstride));
            float4& a = acc[kh * 3 + kw];
            a.x = fmaf(g.x, q.x, a.x);
            a.y = fmaf(g.y, q.y, a.y);
            a.z = fmaf(g.z, q.z, a.z);
            a.w = fmaf(g.w, q.w, a.w);
          }
        }
      }
    }
  }
  auto fold = [&](float v) {
#pragma unroll
    for (int off = 16; off >= G; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    return v;
  };
#pragma unroll
  for (int t = 0; t < 9; ++t) {
    acc[t].x = fold(acc[t].x); acc[t].y = fold(acc[t].y); acc[t].z = fold(acc[t].z); acc[t].w = fold(acc[t].w);
  }
  bs.x = fold(bs.x); bs.y = fold(bs.y); bs.z = fold(bs.z); bs.w = fold(bs.w);
  if (lane < G) {
#pragma unroll
    for (int t = 0; t < 9; ++t) {
      red[warp][l][t * 4 + 0] = acc[t].x; red[warp][l][t * 4 + 1] = acc[t].y;
      red[warp][l][t * 4 + 2] = acc[t].z; red[warp][l][t * 4 + 3] = acc[t].w;
    }
    red[warp][l][108] = bs.x; red[warp][l][109] = bs.y; red[warp][l][110] = bs.z; red[warp][l][111] = bs.w;
  }
  __syncthreads();
  float* p = partial + ((long long)b * gridDim.x + blockIdx.x) * 28 * C;
  for (int i = threadIdx.x; i < 10 * C; i += blockDim.x) {
    int ll, k, dst;
    if (i < 9 * C) {
      const int c = i / 9, t = i % 9;  // [c][kd * 9 + t]
      ll = c / 4;
      k = t * 4 + (c & 3);
      dst = c * 27 + kd * 9 + t;
    } else {
      if (kd != 0) break;  // the bias sums come from plane 0
      const int c = i - 9 * C;
      ll = c / 4;
      k = 108 + (c & 3);
      dst = 27 * C + c;
    }
    float sum = 0.f;
    for (int w = 0; w < 8; ++w) sum += red[w][ll][k];
    p[dst] = sum;
  }
}

static void dw_split(int C, long long V, int batch, int* nchunks, int* chunk) {
  // ~64K threads of (channel, chunk), >= 16 voxels per chunk, <= 1024 chunks (the reduce is per chunk)
  long long want = (64LL * 1024 + (long long)C * batch - 1) / ((long long)C * batch);
  want = std::min(want, std::max(1LL, V / 16));
  want = std::min(want, 1024LL);
  if (want < 1) want = 1;
  *chunk = (int)((V + want - 1) / want);
  *nchunks = (int)((V + *chunk - 1) / *chunk);
}

static bool dw_g_ok(const d2ip_act& x, const d2ip_act& gy) {
  const int G = x.c / 4;
  auto al = [](const d2ip_act& a) { return a.cstride % 4 == 0 && ((uintptr_t)a.ptr & 15) == 0; };
  return x.c % 4 == 0 && (G == 1 || G == 2 || G == 4 || G == 8 || G == 16) && al(x) && al(gy);
}

static int dw_g_blocks(long long V) { return (int)std::min<long long>(296, std::max<long long>(1, V / 32)); }

size_t dw_wgrad_ws(int C, long long V, int batch) {
  int n, c;
  dw_split(C, V, batch, &n, &c);
  return (size_t)batch * std::max(n, dw_g_blocks(V)) * 28 * C * sizeof(float);
}

int dw_conv_fwd(d2ip_act x, const float* w, const float* bias, long long wbs, int stride, d2ip_act y, int batch,
                cudaStream_t st) {
  const long long n = (long long)y.d * y.h * y.w * x.c;
  D2IP_CUDA(launch_pdl(dw_fwd_k, dim3(cdiv(n, 256), batch), 256, 0, st, x, w, bias, wbs, stride, y));
  return D2IP_OK;
}

int dw_conv_dgrad(d2ip_act gy, const float* w, long long wbs, int stride, d2ip_act gx, int accumulate, int batch,
                  cudaStream_t st) {
  const long long n = (long long)gx.d * gx.h * gx.w * gx.c;
  D2IP_CUDA(launch_pdl(dw_dgrad_k, dim3(cdiv(n, 256), batch), 256, 0, st, gy, w, wbs, stride, gx, accumulate));
  return D2IP_OK;
}

int dw_conv_wgrad(d2ip_act x, d2ip_act gy, int stride, float* gw, long long gwbs, void* ws, size_t ws_bytes,
                  int batch, cudaStream_t st) {
  const int C = x.c;
  const long long V = (long long)gy.d * gy.h * gy.w;
  if (dw_g_ok(x, gy)) {
    const int nblk = dw_g_blocks(V);
    D2IP_CHECK_ARG(ws_bytes >= (size_t)batch * nblk * 28 * C * sizeof(float), "dw_wgrad: workspace too small");
    float* partial = reinterpret_cast<float*>(ws);
    const int vchunk = cdiv(V, nblk);
    const dim3 grid(nblk, batch, 3);
    const size_t sm = (size_t)8 * (C / 4) * (27 * 4 + 5) * sizeof(float);
#define D2IP_DWG(G_)                                                                                  \
  case G_: {                                                                                         \
    static bool attr = false;                                                                        \
    if (!attr) {                                                                                     \
      D2IP_CUDA(cudaFuncSetAttribute(dw_wgrad_g_k<G_>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024)); \
      attr = true;                                                                                   \
    }                                                                                                \
    D2IP_CUDA(launch_pdl(dw_wgrad_g_k<G_>, grid, 256, sm, st, x, gy, stride, partial, vchunk));      \
  } break;
    switch (C / 4) { D2IP_DWG(1) D2IP_DWG(2) D2IP_DWG(4) D2IP_DWG(8) D2IP_DWG(16) }
#undef D2IP_DWG
    D2IP_LAUNCH_CHECK();
    return reduce_chunks(partial, nblk, 28 * C, gw, gwbs, batch, st);
  }
  int nchunks, chunk;
  dw_split(C, V, batch, &nchunks, &chunk);
  D2IP_CHECK_ARG(ws_bytes >= (size_t)batch * nchunks * 28 * C * sizeof(float), "dw_wgrad: workspace too small");
  float* partial = reinterpret_cast<float*>(ws);
  D2IP_CUDA(launch_pdl(dw_wgrad_k, dim3(cdiv((long long)nchunks * C, 256), batch), 256, 0, st, x, gy, stride,
                       partial, nchunks, chunk));
  return reduce_chunks(partial, nchunks, 28 * C, gw, gwbs, batch, st);
}

// ---- SqueezeExcite -----------------------------------------------------------
// column sums: partial[b][blk][c] = sum over the block's voxels of a[v][c] (* m[v][c]).
// Accumulated in fp64: the SE gate gradient sum_v gs*x cancels heavily, and an
// fp32 running sum over 32K voxels loses ~1e-3 of it (the reference's CPU
// reductions are pairwise).
__global__ void __launch_bounds__(256) colsum_k(d2ip_act a, d2ip_act m, double* __restrict__ partial, int chunk,
                                                int nchunks) {
  D2IP_PDL_ENTRY();
  __shared__ double red[256];
  const int b = blockIdx.y, blk = blockIdx.x;
  const int C = a.c;
  const long long V = (long long)a.d * a.h * a.w;
  const int rows = 256 / C;  // C <= 256
  const int c = threadIdx.x % C, r = threadIdx.x / C;
  double acc = 0.0;
  if (r < rows) {
    const long long v0 = (long long)blk * chunk, v1 = min(V, v0 + chunk);
    for (long long v = v0 + r; v < v1; v += rows) {
      double t = a.ptr[b * a.bstride + v * a.cstride + c];
      if (m.ptr) t *= (double)m.ptr[b * m.bstride + v * m.cstride + c];
      acc += t;
    }
  }
  red[threadIdx.x] = acc;
  __syncthreads();
  if (threadIdx.x < C) {
    double s = 0.0;
    for (int q = 0; q < rows; ++q) s += red[q * C + threadIdx.x];
    partial[((long long)b * nchunks + blk) * C + threadIdx.x] = s;
  }
}

static void col_split(long long V, int batch, int* n, int* chunk) {
  long long want = std::max(1LL, std::min((148LL * 2 + batch - 1) / batch, (V + 255) / 256));
  *chunk = (int)((V + want - 1) / want);
  *n = (int)((V + *chunk - 1) / *chunk);
}

size_t colsum_ws(int C, long long V, int batch) {
  int n, c;
  col_split(V, batch, &n, &c);
  return (size_t)batch * n * C * sizeof(double);
}

int colsum(d2ip_act a, d2ip_act m, double* partial, size_t ws_bytes, int batch, int* nchunks, cudaStream_t st) {
  D2IP_CHECK_ARG(a.c <= 256, "colsum: C > 256");
  const long long V = (long long)a.d * a.h * a.w;
  int chunk;
  col_split(V, batch, nchunks, &chunk);
  D2IP_CHECK_ARG(ws_bytes >= (size_t)batch * *nchunks * a.c * sizeof(double), "colsum: workspace too small");
  D2IP_CUDA(launch_pdl(colsum_k, dim3(*nchunks, batch), 256, 0, st, a, m, partial, chunk, *nchunks));
  return D2IP_OK;
}

// One block per sequence: pooled = colsum / V; z1 = W1 pooled + b1; h = silu(z1);
// z2 = W2 h + b2; g = sigmoid(z2). Saves pooled, z1, g (fwd_state layout:
// [pooled C][z1 hid][g C]).
__global__ void se_mlp_fwd_k(const double* __restrict__ partial, int nchunks, long long V, int C, int hid,
                             const float* __restrict__ w1, const float* __restrict__ b1, const float* __restrict__ w2,
                             const float* __restrict__ b2, long long pbs, float* __restrict__ state, int sbs) {
  D2IP_PDL_ENTRY();
  extern __shared__ float sm[];  // pooled[C], h[hid]
  const int b = blockIdx.x;
  float* pooled = sm;
  float* hv = sm + C;
  float* S = state + (long long)b * sbs;
  for (int c = threadIdx.x; c < C; c += blockDim.x) {
    double s = 0.0;
    for (int k = 0; k < nchunks; ++k) s += partial[((long long)b * nchunks + k) * C + c];
    pooled[c] = (float)(s / (double)V);
    S[c] = pooled[c];
  }
  __syncthreads();
  for (int j = threadIdx.x; j < hid; j += blockDim.x) {
    float z = __ldg(b1 + b * pbs + j);
    for (int c = 0; c < C; ++c) z = fmaf(__ldg(w1 + b * pbs + (long long)j * C + c), pooled[c], z);
    S[C + j] = z;
    hv[j] = silu(z);
  }
  __syncthreads();
  for (int c = threadIdx.x; c < C; c += blockDim.x) {
    float z = __ldg(b2 + b * pbs + c);
    for (int j = 0; j < hid; ++j) z = fmaf(__ldg(w2 + b * pbs + (long long)c * hid + j), hv[j], z);
    S[C + hid + c] = sigm(z);
  }
}

// out[v][c] = x[v][c] * g[c]
__global__ void __launch_bounds__(256) chan_gate_k(d2ip_act x, const float* __restrict__ state, int goff, int sbs,
                                                   d2ip_act out) {
  D2IP_PDL_ENTRY();
  const int b = blockIdx.y;
  const int C = x.c;
  const long long n = (long long)x.d * x.h * x.w * C;
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int c = (int)(i % C);
  const long long v = i / C;
  out.ptr[b * out.bstride + v * out.cstride + c] =
      x.ptr[b * x.bstride + v * x.cstride + c] * state[(long long)b * sbs + goff + c];
}

// SE backward of the gate MLP (one block per sequence). Input: gg[c] = sum_v
// gs[v][c] x[v][c] (colsum partials). Writes dW1, db1, dW2, db2 (adjacent in
// the flat gradient like the reference's fc1.weight, fc1.bias, fc2.weight,
// fc2.bias) and gpool[c] = (W1^T gz1)[c] / V into the state's scratch slot.
__global__ void se_mlp_bwd_k(const double* __restrict__ partial, int nchunks, long long V, int C, int hid,
                             const float* __restrict__ w1, const float* __restrict__ b1, const float* __restrict__ w2,
                             long long pbs, float* __restrict__ state, int sbs, float* __restrict__ g1,
                             float* __restrict__ g2) {
  D2IP_PDL_ENTRY();
  extern __shared__ float sm[];  // gz2[C], gz1[hid], h[hid]
  const int b = blockIdx.x;
  float* gz2 = sm;
  float* gz1 = sm + C;
  float* hv = sm + C + hid;
  float* S = state + (long long)b * sbs;
  const float* pooled = S;
  const float* z1 = S + C;
  const float* g = S + C + hid;
  float* gpool = S + C + hid + C;
  for (int j = threadIdx.x; j < hid; j += blockDim.x) hv[j] = silu(z1[j]);
  for (int c = threadIdx.x; c < C; c += blockDim.x) {
    double s = 0.0;
    for (int k = 0; k < nchunks; ++k) s += partial[((long long)b * nchunks + k) * C + c];
    gz2[c] = (float)s * g[c] * (1.f - g[c]);
  }
  __syncthreads();
  float* gw2 = g2 + b * pbs;  // fc2.weight [C][hid], then fc2.bias [C]
  for (int i = threadIdx.x; i < C * hid; i += blockDim.x) gw2[i] = gz2[i / hid] * hv[i % hid];
  for (int c = threadIdx.x; c < C; c += blockDim.x) gw2[C * hid + c] = gz2[c];
  for (int j = threadIdx.x; j < hid; j += blockDim.x) {
    float gh = 0.f;
    for (int c = 0; c < C; ++c) gh = fmaf(__ldg(w2 + b * pbs + (long long)c * hid + j), gz2[c], gh);
    gz1[j] = gh * silu_grad(z1[j]);
  }
  __syncthreads();
  float* gw1 = g1 + b * pbs;  // fc1.weight [hid][C], then fc1.bias [hid]
  for (int i = threadIdx.x; i < hid * C; i += blockDim.x) gw1[i] = gz1[i / C] * pooled[i % C];
  for (int j = threadIdx.x; j < hid; j += blockDim.x) gw1[hid * C + j] = gz1[j];
  for (int c = threadIdx.x; c < C; c += blockDim.x) {
    float s = 0.f;
    for (int j = 0; j < hid; ++j) s = fmaf(__ldg(w1 + b * pbs + (long long)j * C + c), gz1[j], s);
    gpool[c] = s / (float)V;
  }
  (void)b1;
}

// gx[v][c] (+)= gs[v][c] * g[c] + gpool[c]   (second pass after the MLP backward)
__global__ void __launch_bounds__(256) se_bwd_apply_k(d2ip_act gs, const float* __restrict__ state, int goff, int poff,
                                                      int sbs, d2ip_act gx, int accumulate) {
  D2IP_PDL_ENTRY();
  const int b = blockIdx.y;
  const int C = gs.c;
  const long long n = (long long)gs.d * gs.h * gs.w * C;
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int c = (int)(i % C);
  const long long v = i / C;
  const float* S = state + (long long)b * sbs;
  const float t = gs.ptr[b * gs.bstride + v * gs.cstride + c] * S[goff + c] + S[poff + c];
  float* o = gx.ptr + b * gx.bstride + v * gx.cstride + c;
  *o = accumulate ? *o + t : t;
}

int se_forward(d2ip_act x, const float* w1, const float* b1, const float* w2, const float* b2, long long pbs, int hid,
               float* state, int sbs, d2ip_act out, void* ws, size_t ws_bytes, int batch, cudaStream_t st) {
  const int C = x.c;
  const long long V = (long long)x.d * x.h * x.w;
  int nchunks;
  double* partial = reinterpret_cast<double*>(ws);
  D2IP_RET(colsum(x, d2ip_act{}, partial, ws_bytes, batch, &nchunks, st));
  D2IP_CUDA(launch_pdl(se_mlp_fwd_k, dim3(batch), 256, (size_t)(C + hid) * sizeof(float), st, partial, nchunks, V,
                       C, hid, w1, b1, w2, b2, pbs, state, sbs));
  D2IP_CUDA(launch_pdl(chan_gate_k, dim3(cdiv(V * C, 256), batch), 256, 0, st, x, state, C + hid, sbs, out));
  return D2IP_OK;
}

int se_backward(d2ip_act x, d2ip_act gs, const float* w1, const float* b1, const float* w2, long long pbs, int hid,
                float* state, int sbs, float* g1, float* g2, d2ip_act gx, int accumulate, void* ws, size_t ws_bytes,
                int batch, cudaStream_t st) {
  const int C = x.c;
  const long long V = (long long)x.d * x.h * x.w;
  int nchunks;
  double* partial = reinterpret_cast<double*>(ws);
  D2IP_RET(colsum(gs, x, partial, ws_bytes, batch, &nchunks, st));
  D2IP_CUDA(launch_pdl(se_mlp_bwd_k, dim3(batch), 256, (size_t)(C + 2 * hid) * sizeof(float), st, partial, nchunks,
                       V, C, hid, w1, b1, w2, pbs, state, sbs, g1, g2));
  D2IP_CUDA(launch_pdl(se_bwd_apply_k, dim3(cdiv(V * C, 256), batch), 256, 0, st, gs, state, C + hid,
                       C + hid + C, sbs, gx, accumulate));
  return D2IP_OK;
}

// ---- AttentionGate3d element-wise parts --------------------------------------
// pre = k + q (saved); a = silu(pre)
__global__ void __launch_bounds__(256) add_silu_k(d2ip_act k, d2ip_act q, float* __restrict__ pre, d2ip_act a) {
  D2IP_PDL_ENTRY();
  const int b = blockIdx.y;
  const int C = k.c;
  const long long V = (long long)k.d * k.h * k.w;
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= V * C) return;
  const int c = (int)(i % C);
  const long long v = i / C;
  const float t = k.ptr[b * k.bstride + v * k.cstride + c] + q.ptr[b * q.bstride + v * q.cstride + c];
  pre[(long long)b * V * C + i] = t;
  a.ptr[b * a.bstride + v * a.cstride + c] = silu(t);
}

// gpre = ga * silu'(pre)
__global__ void __launch_bounds__(256) silu_bwd_k(d2ip_act ga, const float* __restrict__ pre, d2ip_act gpre) {
  D2IP_PDL_ENTRY();
  const int b = blockIdx.y;
  const int C = ga.c;
  const long long V = (long long)ga.d * ga.h * ga.w;
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= V * C) return;
  const int c = (int)(i % C);
  const long long v = i / C;
  gpre.ptr[b * gpre.bstride + v * gpre.cstride + c] =
      ga.ptr[b * ga.bstride + v * ga.cstride + c] * silu_grad(pre[(long long)b * V * C + i]);
}

// in place: t = sigmoid(t)   (1 channel, contiguous [B][V])
__global__ void sigmoid_k(float* t, long long n) {
  D2IP_PDL_ENTRY();
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) t[i] = sigm(t[i]);
}

// g = g * s * (1 - s)   (s = saved sigmoid, 1 channel)
__global__ void sigmoid_bwd_k(float* g, const float* __restrict__ s, long long n) {
  D2IP_PDL_ENTRY();
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) g[i] = g[i] * s[i] * (1.f - s[i]);
}

// gated[v][c] = s[v][c] * att[v]
__global__ void __launch_bounds__(256) att_gate_fwd_k(d2ip_act s, const float* __restrict__ att, d2ip_act out) {
  D2IP_PDL_ENTRY();
  const int b = blockIdx.y;
  const int C = s.c;
  const long long V = (long long)s.d * s.h * s.w;
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= V * C) return;
  const int c = (int)(i % C);
  const long long v = i / C;
  out.ptr[b * out.bstride + v * out.cstride + c] = s.ptr[b * s.bstride + v * s.cstride + c] * att[(long long)b * V + v];
}

// per voxel: gs[v][c] (+)= gg[v][c] * att[v];  gatt[v] = sum_c gg[v][c] s[v][c]
__global__ void __launch_bounds__(128) att_gate_bwd_k(d2ip_act gg, d2ip_act s, const float* __restrict__ att,
                                                      d2ip_act gs, int accumulate, float* __restrict__ gatt) {
  D2IP_PDL_ENTRY();
  const int b = blockIdx.y;
  const int C = s.c;
  const long long V = (long long)s.d * s.h * s.w;
  const long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= V) return;
  const float a = att[(long long)b * V + v];
  const float* gp = gg.ptr + b * gg.bstride + v * gg.cstride;
  const float* sp = s.ptr + b * s.bstride + v * s.cstride;
  float* op = gs.ptr + b * gs.bstride + v * gs.cstride;
  float dot = 0.f;
  for (int c = 0; c < C; ++c) {
    const float g = gp[c];
    dot = fmaf(g, sp[c], dot);
    op[c] = accumulate ? op[c] + g * a : g * a;
  }
  gatt[(long long)b * V + v] = dot;
}

int add_silu(d2ip_act k, d2ip_act q, float* pre, d2ip_act a, int batch, cudaStream_t st) {
  const long long n = (long long)k.d * k.h * k.w * k.c;
  D2IP_CUDA(launch_pdl(add_silu_k, dim3(cdiv(n, 256), batch), 256, 0, st, k, q, pre, a));
  return D2IP_OK;
}
int silu_bwd(d2ip_act ga, const float* pre, d2ip_act gpre, int batch, cudaStream_t st) {
  const long long n = (long long)ga.d * ga.h * ga.w * ga.c;
  D2IP_CUDA(launch_pdl(silu_bwd_k, dim3(cdiv(n, 256), batch), 256, 0, st, ga, pre, gpre));
  return D2IP_OK;
}
int sigmoid_inplace(float* t, long long n, cudaStream_t st) {
  D2IP_CUDA(launch_pdl(sigmoid_k, dim3(cdiv(n, 256)), 256, 0, st, t, n));
  return D2IP_OK;
}
int sigmoid_bwd(float* g, const float* s, long long n, cudaStream_t st) {
  D2IP_CUDA(launch_pdl(sigmoid_bwd_k, dim3(cdiv(n, 256)), 256, 0, st, g, s, n));
  return D2IP_OK;
}
int att_gate_fwd(d2ip_act s, const float* att, d2ip_act out, int batch, cudaStream_t st) {
  const long long n = (long long)s.d * s.h * s.w * s.c;
  D2IP_CUDA(launch_pdl(att_gate_fwd_k, dim3(cdiv(n, 256), batch), 256, 0, st, s, att, out));
  return D2IP_OK;
}
int att_gate_bwd(d2ip_act gg, d2ip_act s, const float* att, d2ip_act gs, int accumulate, float* gatt, int batch,
                 cudaStream_t st) {
  const long long V = (long long)s.d * s.h * s.w;
  D2IP_CUDA(launch_pdl(att_gate_bwd_k, dim3(cdiv(V, 128), batch), 128, 0, st, gg, s, att, gs, accumulate, gatt));
  return D2IP_OK;
}

}  // namespace d2ip
