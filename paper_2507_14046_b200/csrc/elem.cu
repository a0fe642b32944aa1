#include <algorithm>
// Per-voxel kernels: trilinear x2 upsample (align_corners=False) forward and
// gather backward, and the tail conv + sigmoid + output map + mask gather.
// (ChannelLayerNorm / activation kernels live in norm.cu.)
//
// F.interpolate      : priornet.py:229 (trilinear, align_corners=False)
// sigmoid + map      : priornet.py:231, pipeline.py:276-278
#include "common.cuh"
#include "kernels.h"

namespace d2ip {

// ---------------------------------------------------------------------------
// Trilinear x2, align_corners=False. Along one axis (n = low-res size):
//   dst = 0      -> in[0]
//   dst = 2m     -> 0.25 in[m-1] + 0.75 in[m]          (m >= 1)
//   dst = 2m + 1 -> 0.75 in[m] + 0.25 in[min(m+1, n-1)]
// (src = (dst + 0.5)/2 - 0.5 clamped at 0, aten upsample_trilinear3d.)

struct Lin {
  int i0, i1;
  float l0, l1;
};

__device__ __forceinline__ Lin lin_src(int dst, int n) {
  float src = 0.5f * ((float)dst + 0.5f) - 0.5f;
  if (src < 0.f) src = 0.f;
  Lin r;
  r.i0 = (int)src;
  r.i1 = r.i0 + ((r.i0 < n - 1) ? 1 : 0);
  r.l1 = src - (float)r.i0;
  r.l0 = 1.f - r.l1;
  return r;
}

__global__ void __launch_bounds__(256) upsample2x_fwd_k(d2ip_act x, d2ip_act y) {
  D2IP_PDL_ENTRY();
  const int b = blockIdx.y;
  const int C = x.c;
  const long long total = (long long)y.d * y.h * y.w * C;
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= total) return;
  const int c = (int)(idx % C);
  const long long v = idx / C;
  const int ow = (int)(v % y.w), oh = (int)((v / y.w) % y.h), od = (int)(v / ((long long)y.w * y.h));
  const Lin ld = lin_src(od, x.d), lh = lin_src(oh, x.h), lw = lin_src(ow, x.w);
  const float* xb = x.ptr + b * x.bstride + c;
  auto at = [&](int d, int h, int w) { return xb[(((long long)d * x.h + h) * x.w + w) * x.cstride]; };
  const float v00 = lw.l0 * at(ld.i0, lh.i0, lw.i0) + lw.l1 * at(ld.i0, lh.i0, lw.i1);
  const float v01 = lw.l0 * at(ld.i0, lh.i1, lw.i0) + lw.l1 * at(ld.i0, lh.i1, lw.i1);
  const float v10 = lw.l0 * at(ld.i1, lh.i0, lw.i0) + lw.l1 * at(ld.i1, lh.i0, lw.i1);
  const float v11 = lw.l0 * at(ld.i1, lh.i1, lw.i0) + lw.l1 * at(ld.i1, lh.i1, lw.i1);
  const float r = ld.l0 * (lh.l0 * v00 + lh.l1 * v01) + ld.l1 * (lh.l0 * v10 + lh.l1 * v11);
  y.ptr[b * y.bstride + v * y.cstride + c] = r;
  if (y.bf16) reinterpret_cast<__nv_bfloat16*>(y.bf16)[b * y.bstride + v * y.cstride + c] = __float2bfloat16_rn(r);
}

// float4 variant: one thread per (voxel, 4 channels) -- a quarter of the index
// arithmetic and 128-bit loads / stores (C, strides and bases 16-byte aligned).
__global__ void __launch_bounds__(256) upsample2x_fwd4_k(d2ip_act x, d2ip_act y) {
  D2IP_PDL_ENTRY();
  const int b = blockIdx.y;
  const int C4 = x.c >> 2;
  const long long total = (long long)y.d * y.h * y.w * C4;
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= total) return;
  const int c = (int)(idx % C4) * 4;
  const long long v = idx / C4;
  const int ow = (int)(v % y.w), oh = (int)((v / y.w) % y.h), od = (int)(v / ((long long)y.w * y.h));
  const Lin ld = lin_src(od, x.d), lh = lin_src(oh, x.h), lw = lin_src(ow, x.w);
  const float* xb = x.ptr + b * x.bstride + c;
  auto at = [&](int d, int h, int w) {
    return *reinterpret_cast<const float4*>(xb + (((long long)d * x.h + h) * x.w + w) * x.cstride);
  };
  auto lerp2 = [](float a, float p, float bb, float q) { return a * p + bb * q; };
  const float4 p00 = at(ld.i0, lh.i0, lw.i0), p01 = at(ld.i0, lh.i0, lw.i1);
  const float4 p10 = at(ld.i0, lh.i1, lw.i0), p11 = at(ld.i0, lh.i1, lw.i1);
  const float4 q00 = at(ld.i1, lh.i0, lw.i0), q01 = at(ld.i1, lh.i0, lw.i1);
  const float4 q10 = at(ld.i1, lh.i1, lw.i0), q11 = at(ld.i1, lh.i1, lw.i1);
  float4 r;
#define D2IP_UP(comp)                                                                        \
  {                                                                                          \
    const float v00 = lerp2(lw.l0, p00.comp, lw.l1, p01.comp);                                \
    const float v01 = lerp2(lw.l0, p10.comp, lw.l1, p11.comp);                                \
    const float v10 = lerp2(lw.l0, q00.comp, lw.l1, q01.comp);                                \
    const float v11 = lerp2(lw.l0, q10.comp, lw.l1, q11.comp);                                \
    r.comp = ld.l0 * (lh.l0 * v00 + lh.l1 * v01) + ld.l1 * (lh.l0 * v10 + lh.l1 * v11);       \
  }
  D2IP_UP(x) D2IP_UP(y) D2IP_UP(z) D2IP_UP(w)
#undef D2IP_UP
  *reinterpret_cast<float4*>(y.ptr + b * y.bstride + v * y.cstride + c) = r;
  if (y.bf16)
    *reinterpret_cast<uint2*>(reinterpret_cast<uint16_t*>(y.bf16) + b * y.bstride + v * y.cstride + c) =
        make_uint2(bf16x2(r.x, r.y), bf16x2(r.z, r.w));
}

static bool aligned4(const d2ip_act& a) { return a.c % 4 == 0 && a.cstride % 4 == 0 && ((uintptr_t)a.ptr & 15) == 0; }

int upsample2x_fwd(d2ip_act x, d2ip_act y, int batch, cudaStream_t st) {
  D2IP_CHECK_ARG(y.d == 2 * x.d && y.h == 2 * x.h && y.w == 2 * x.w && y.c == x.c,
                 "upsample2x: shape mismatch");
  const long long total = (long long)y.d * y.h * y.w * y.c;
  if (aligned4(x) && aligned4(y))
    D2IP_CUDA(launch_pdl(upsample2x_fwd4_k, dim3(cdiv(total / 4, 256), batch), 256, 0, st, x, y));
  else
    D2IP_CUDA(launch_pdl(upsample2x_fwd_k, dim3(cdiv(total, 256), batch), 256, 0, st, x, y));
  D2IP_LAUNCH_CHECK();
  return D2IP_OK;
}

// Contributions of low-res index m to high-res indices along one axis.
__device__ __forceinline__ int lin_adj(int m, int n, int* hi, float* wt) {
  int k = 0;
  if (m >= 1) { hi[k] = 2 * m - 1; wt[k++] = 0.25f; }
  hi[k] = 2 * m;     wt[k++] = (m == 0) ? 1.0f : 0.75f;
  hi[k] = 2 * m + 1; wt[k++] = (m == n - 1) ? 1.0f : 0.75f;
  if (m + 1 <= n - 1) { hi[k] = 2 * m + 2; wt[k++] = 0.25f; }
  return k;
}

__global__ void __launch_bounds__(256) upsample2x_bwd_k(d2ip_act gy, d2ip_act gx, int accumulate) {
  D2IP_PDL_ENTRY();
  const int b = blockIdx.y;
  const int C = gx.c;
  const long long total = (long long)gx.d * gx.h * gx.w * C;
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= total) return;
  const int c = (int)(idx % C);
  const long long v = idx / C;
  const int iw = (int)(v % gx.w), ih = (int)((v / gx.w) % gx.h), id = (int)(v / ((long long)gx.w * gx.h));
  int hd[4], hh[4], hw[4];
  float wd[4], wh[4], ww[4];
  const int nd = lin_adj(id, gx.d, hd, wd), nh = lin_adj(ih, gx.h, hh, wh), nw = lin_adj(iw, gx.w, hw, ww);
  const float* gb = gy.ptr + b * gy.bstride + c;
  float acc = 0.f;
  for (int a = 0; a < nd; ++a)
    for (int e = 0; e < nh; ++e) {
      float row = 0.f;
      for (int f = 0; f < nw; ++f)
        row = fmaf(ww[f], gb[(((long long)hd[a] * gy.h + hh[e]) * gy.w + hw[f]) * gy.cstride], row);
      acc = fmaf(wd[a] * wh[e], row, acc);
    }
  float* o = gx.ptr + b * gx.bstride + v * gx.cstride + c;
  *o = accumulate ? *o + acc : acc;
}

// float4 variant of the gather (same per-channel summation order)
__global__ void __launch_bounds__(256) upsample2x_bwd4_k(d2ip_act gy, d2ip_act gx, int accumulate) {
  D2IP_PDL_ENTRY();
  const int b = blockIdx.y;
  const int C4 = gx.c >> 2;
  const long long total = (long long)gx.d * gx.h * gx.w * C4;
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= total) return;
  const int c = (int)(idx % C4) * 4;
  const long long v = idx / C4;
  const int iw = (int)(v % gx.w), ih = (int)((v / gx.w) % gx.h), id = (int)(v / ((long long)gx.w * gx.h));
  int hd[4], hh[4], hw[4];
  float wd[4], wh[4], ww[4];
  const int nd = lin_adj(id, gx.d, hd, wd), nh = lin_adj(ih, gx.h, hh, wh), nw = lin_adj(iw, gx.w, hw, ww);
  const float* gb = gy.ptr + b * gy.bstride + c;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int a = 0; a < nd; ++a)
    for (int e = 0; e < nh; ++e) {
      float4 row = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int f = 0; f < nw; ++f) {
        const float4 g =
            *reinterpret_cast<const float4*>(gb + (((long long)hd[a] * gy.h + hh[e]) * gy.w + hw[f]) * gy.cstride);
        row.x = fmaf(ww[f], g.x, row.x);
        row.y = fmaf(ww[f], g.y, row.y);
        row.z = fmaf(ww[f], g.z, row.z);
        row.w = fmaf(ww[f], g.w, row.w);
      }
      const float wde = wd[a] * wh[e];
      acc.x = fmaf(wde, row.x, acc.x);
      acc.y = fmaf(wde, row.y, acc.y);
      acc.z = fmaf(wde, row.z, acc.z);
      acc.w = fmaf(wde, row.w, acc.w);
    }
  float4* o = reinterpret_cast<float4*>(gx.ptr + b * gx.bstride + v * gx.cstride + c);
  if (accumulate) {
    const float4 p = *o;
    acc.x += p.x; acc.y += p.y; acc.z += p.z; acc.w += p.w;
  }
  *o = acc;
}

int upsample2x_bwd(d2ip_act gy, d2ip_act gx, int accumulate, int batch, cudaStream_t st) {
  D2IP_CHECK_ARG(gy.d == 2 * gx.d && gy.h == 2 * gx.h && gy.w == 2 * gx.w && gy.c == gx.c,
                 "upsample2x_bwd: shape mismatch");
  const long long total = (long long)gx.d * gx.h * gx.w * gx.c;
  if (aligned4(gy) && aligned4(gx))
    D2IP_CUDA(launch_pdl(upsample2x_bwd4_k, dim3(cdiv(total / 4, 256), batch), 256, 0, st, gy, gx, accumulate));
  else
    D2IP_CUDA(launch_pdl(upsample2x_bwd_k, dim3(cdiv(total, 256), batch), 256, 0, st, gy, gx, accumulate));
  D2IP_LAUNCH_CHECK();
  return D2IP_OK;
}

// ---------------------------------------------------------------------------
// Tail: conv3(c0 -> 1) + bias -> sigmoid -> lo + scale * s, and the gather of
// the mapped value into J's column order (sigma_c[col_of_vox[v]]). The three
// kd planes of taps are split over three thread slices (32 voxels x 3 per
// block; plane sums added in order through shared memory), each slice keeping
// four independent partial sums -- a 12x shorter FMA chain than one thread per
// voxel.
__global__ void __launch_bounds__(96) tail_fwd_k(d2ip_act x, const float* __restrict__ w,
                                                 const float* __restrict__ bias, long long wbs,
                                                 float lo, float scale, float* __restrict__ sig,
                                                 float* __restrict__ mapped, float* __restrict__ sigma_c,
                                                 long long sc_bs, const int* __restrict__ col_of_vox) {
  D2IP_PDL_ENTRY();
  extern __shared__ float sw[];  // [tap][cin], then [3][32] plane sums
  const int b = blockIdx.y;
  const int cin = x.c;
  const float* wb = w + b * wbs;
  for (int i = threadIdx.x; i < 27 * cin; i += blockDim.x) sw[i] = __ldg(wb + (i % cin) * 27 + i / cin);
  float* red = sw + 27 * cin;
  __syncthreads();
  const long long V = (long long)x.d * x.h * x.w;
  const int kd = threadIdx.x / 32, vl = threadIdx.x % 32;
  const long long v = (long long)blockIdx.x * 32 + vl;
  float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
  if (v < V) {
    const int ow = (int)(v % x.w), oh = (int)((v / x.w) % x.h), od = (int)(v / ((long long)x.w * x.h));
    const float* xb = x.ptr + b * x.bstride;
    const bool vec = (cin % 4 == 0) && (x.cstride % 4 == 0) && (((uintptr_t)x.ptr & 15) == 0);
    const int id = od + kd - 1;
    if (id >= 0 && id < x.d) {
      for (int kh = 0; kh < 3; ++kh) {
        const int ih = oh + kh - 1;
        if (ih < 0 || ih >= x.h) continue;
        for (int kw = 0; kw < 3; ++kw) {
          const int iw = ow + kw - 1;
          if (iw < 0 || iw >= x.w) continue;
          const float* xp = xb + (((long long)id * x.h + ih) * x.w + iw) * x.cstride;
          const float* wr = sw + ((kd * 3 + kh) * 3 + kw) * cin;
          if (vec) {
            for (int ci = 0; ci < cin; ci += 4) {
              const float4 q = __ldg(reinterpret_cast<const float4*>(xp + ci));
              a0 = fmaf(q.x, wr[ci], a0);
              a1 = fmaf(q.y, wr[ci + 1], a1);
              a2 = fmaf(q.z, wr[ci + 2], a2);
              a3 = fmaf(q.w, wr[ci + 3], a3);
            }
          } else {
            for (int ci = 0; ci < cin; ++ci) a0 = fmaf(xp[ci], wr[ci], a0);
          }
        }
      }
    }
  }
  red[kd * 32 + vl] = (a0 + a1) + (a2 + a3);
  __syncthreads();
  if (kd != 0 || v >= V) return;
  const float acc = __ldg(bias + b * wbs) + ((red[vl] + red[32 + vl]) + red[64 + vl]);
  const float s = 1.0f / (1.0f + expf(-acc));
  const float mp = lo + scale * s;
  sig[b * V + v] = s;
  mapped[b * V + v] = mp;
  const int col = col_of_vox[v];
  if (col >= 0) sigma_c[b * sc_bs + col] = mp;
}

// ---------------------------------------------------------------------------
// The C_out = 1 tail convolution (priornet.py:215-232 restated: 3^3, padding 1)
// with lane groups: G = C / 4 lanes share a voxel, lane l owns channels
// 4l .. 4l + 3 (float4 loads: a group reads its voxel row in one coalesced
// 16 G-byte run), and the G partial dot products are combined with a fixed
// xor-shuffle tree. Replaces the one-thread-per-voxel kernels, which read a
// 128-byte row per thread per tap (a 27-deep chain of uncoalesced loads).

template <int G>
__device__ __forceinline__ float group_sum(float v) {
#pragma unroll
  for (int o = G >> 1; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

template <int G>
__global__ void __launch_bounds__(256) tail_fwd_g_k(d2ip_act x, const float* __restrict__ w,
                                                    const float* __restrict__ bias, long long wbs, float lo,
                                                    float scale, float* __restrict__ sig, float* __restrict__ mapped,
                                                    float* __restrict__ sigma_c, long long sc_bs,
                                                    const int* __restrict__ col_of_vox) {
  D2IP_PDL_ENTRY();
  __shared__ float4 sw[27 * G];  // [tap][lane] = W[0][4 lane .. 4 lane + 3][tap]
  const int b = blockIdx.y;
  const float* wb = w + b * wbs;
  for (int i = threadIdx.x; i < 27 * G; i += blockDim.x) {
    const int t = i / G, l = i % G;
    sw[i] = make_float4(__ldg(wb + (4 * l) * 27 + t), __ldg(wb + (4 * l + 1) * 27 + t),
                        __ldg(wb + (4 * l + 2) * 27 + t), __ldg(wb + (4 * l + 3) * 27 + t));
  }
  __syncthreads();
  const long long V = (long long)x.d * x.h * x.w;
  const long long v = ((long long)blockIdx.x * blockDim.x + threadIdx.x) / G;
  const int l = threadIdx.x % G;
  float acc = 0.f;
  if (v < V) {
    const int ow = (int)(v % x.w), oh = (int)((v / x.w) % x.h), od = (int)(v / ((long long)x.w * x.h));
    const float* xb = x.ptr + b * x.bstride + 4 * l;
    // branch-free taps (out-of-grid taps load the centre voxel and are skipped by a
    // select): all 27 loads can be in flight at once; same summation order.
#pragma unroll
    for (int kd = 0; kd < 3; ++kd) {
      const int id = od + kd - 1;
      const bool okd = id >= 0 && id < x.d;
#pragma unroll
      for (int kh = 0; kh < 3; ++kh) {
        const int ih = oh + kh - 1;
        const bool okh = okd && ih >= 0 && ih < x.h;
#pragma unroll
        for (int kw = 0; kw < 3; ++kw) {
          const int iw = ow + kw - 1;
          const bool ok = okh && iw >= 0 && iw < x.w;
          const long long off = ok ? (((long long)id * x.h + ih) * x.w + iw) * x.cstride : v * x.cstride;
          const float4 q = __ldg(reinterpret_cast<const float4*>(xb + off));
          const float4 wq = sw[((kd * 3 + kh) * 3 + kw) * G + l];
          const float t = fmaf(q.x, wq.x, fmaf(q.y, wq.y, fmaf(q.z, wq.z, fmaf(q.w, wq.w, acc))));
          acc = ok ? t : acc;
        }
      }
    }
  }
  acc = group_sum<G>(acc);
  if (v >= V || l != 0) return;
  const float a = __ldg(bias + b * wbs) + acc;
  const float s = 1.0f / (1.0f + expf(-a));
  const float mp = lo + scale * s;
  sig[b * V + v] = s;
  mapped[b * V + v] = mp;
  const int col = col_of_vox[v];
  if (col >= 0) sigma_c[b * sc_bs + col] = mp;
}

// gx[v][c] = sum_t W[0][c][t] gt[v - off_t]  (conv_transpose of the C_out = 1 tail)
template <int G>
__global__ void __launch_bounds__(256) tail_dgrad_g_k(const float* __restrict__ gt, const float* __restrict__ w,
                                                      long long wbs, d2ip_act gx) {
  D2IP_PDL_ENTRY();
  __shared__ float4 sw[27 * G];
  const int b = blockIdx.y;
  const float* wb = w + b * wbs;
  for (int i = threadIdx.x; i < 27 * G; i += blockDim.x) {
    const int t = i / G, l = i % G;
    sw[i] = make_float4(__ldg(wb + (4 * l) * 27 + t), __ldg(wb + (4 * l + 1) * 27 + t),
                        __ldg(wb + (4 * l + 2) * 27 + t), __ldg(wb + (4 * l + 3) * 27 + t));
  }
  __syncthreads();
  const long long V = (long long)gx.d * gx.h * gx.w;
  const long long v = ((long long)blockIdx.x * blockDim.x + threadIdx.x) / G;
  const int l = threadIdx.x % G;
  if (v >= V) return;
  const int ow = (int)(v % gx.w), oh = (int)((v / gx.w) % gx.h), od = (int)(v / ((long long)gx.w * gx.h));
  const float* g = gt + b * V;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  // branch-free taps as in tail_fwd_g_k: an out-of-grid tap contributes s = 0
  // (fmaf(0, w, acc) == acc for finite w), all 27 loads in flight
#pragma unroll
  for (int kd = 0; kd < 3; ++kd) {
    const int id = od - kd + 1;
    const bool okd = id >= 0 && id < gx.d;
#pragma unroll
    for (int kh = 0; kh < 3; ++kh) {
      const int ih = oh - kh + 1;
      const bool okh = okd && ih >= 0 && ih < gx.h;
#pragma unroll
      for (int kw = 0; kw < 3; ++kw) {
        const int iw = ow - kw + 1;
        const bool ok = okh && iw >= 0 && iw < gx.w;
        const float s0 = __ldg(g + (ok ? ((long long)id * gx.h + ih) * gx.w + iw : v));
        const float s = ok ? s0 : 0.f;
        const float4 wq = sw[((kd * 3 + kh) * 3 + kw) * G + l];
        acc.x = fmaf(s, wq.x, acc.x);
        acc.y = fmaf(s, wq.y, acc.y);
        acc.z = fmaf(s, wq.z, acc.z);
        acc.w = fmaf(s, wq.w, acc.w);
      }
    }
  }
  *reinterpret_cast<float4*>(gx.ptr + b * gx.bstride + v * gx.cstride + 4 * l) = acc;
}

// Weight + bias gradient of the tail: dW[c][t] = sum_v x[v][c] gt[v - off_t],
// db = sum_v gt[v]. Each CTA walks a voxel range for the nine taps of one kd
// plane (blockIdx.z; 36 accumulators per lane instead of 108, so several CTAs
// per SM hide the gt load latency), reduces its lane groups with a fixed
// shuffle tree and a fixed-order pass over its warps, and writes its taps of
// one partial [27 C + 1]; a second pass sums the partials in CTA order.
template <int G>
__global__ void __launch_bounds__(256) tail_wgrad_g_k(d2ip_act x, const float* __restrict__ gt, int vchunk,
                                                      float* __restrict__ part) {
  D2IP_PDL_ENTRY();
  __shared__ float red[8][G][9 * 4 + 1];
  const int b = blockIdx.y, kd = blockIdx.z;
  const int C = 4 * G;
  const long long V = (long long)x.d * x.h * x.w;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, l = lane % G, grp = threadIdx.x / G;
  float acc[9][4];
#pragma unroll
  for (int t = 0; t < 9; ++t) acc[t][0] = acc[t][1] = acc[t][2] = acc[t][3] = 0.f;
  float bsum = 0.f;
  const float* g = gt + b * V;
  const long long v_lo = (long long)blockIdx.x * vchunk, v_hi = min(V, v_lo + vchunk);
  for (long long v = v_lo + grp; v < v_hi; v += 256 / G) {
    const int ow = (int)(v % x.w), oh = (int)((v / x.w) % x.h), od = (int)(v / ((long long)x.w * x.h));
    const float4 q = __ldg(reinterpret_cast<const float4*>(x.ptr + b * x.bstride + v * x.cstride + 4 * l));
    if (l == 0 && kd == 0) bsum += g[v];
    const int id = od - kd + 1;
    if (id < 0 || id >= x.d) continue;
#pragma unroll
    for (int kh = 0; kh < 3; ++kh) {
      const int ih = oh - kh + 1;
#pragma unroll
      for (int kw = 0; kw < 3; ++kw) {
        const int iw = ow - kw + 1;
        const bool in = ih >= 0 && ih < x.h && iw >= 0 && iw < x.w;
        const float s = in ? __ldg(g + ((long long)id * x.h + ih) * x.w + iw) : 0.f;
        const int t = kh * 3 + kw;
        acc[t][0] = fmaf(q.x, s, acc[t][0]);
        acc[t][1] = fmaf(q.y, s, acc[t][1]);
        acc[t][2] = fmaf(q.z, s, acc[t][2]);
        acc[t][3] = fmaf(q.w, s, acc[t][3]);
      }
    }
  }
  // fold the 32 / G voxel groups of the warp (lanes l, l + G, ...): fixed xor tree
#pragma unroll
  for (int t = 0; t < 9; ++t)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      float v = acc[t][j];
#pragma unroll
      for (int o = 16; o >= G; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      acc[t][j] = v;
    }
  for (int o = 16; o >= 1; o >>= 1) bsum += __shfl_xor_sync(0xffffffffu, bsum, o);
  if (lane < G) {
#pragma unroll
    for (int t = 0; t < 9; ++t)
#pragma unroll
      for (int j = 0; j < 4; ++j) red[warp][l][t * 4 + j] = acc[t][j];
    if (lane == 0) red[warp][0][9 * 4] = bsum;
  }
  __syncthreads();
  float* pb = part + ((long long)b * gridDim.x + blockIdx.x) * (27 * C + 1);
  for (int i = threadIdx.x; i < 9 * C + 1; i += blockDim.x) {
    float s = 0.f;
    if (i < 9 * C) {
      const int c = i / 9, t = i % 9, ll = c / 4, j = c % 4;  // output order: OIDHW [c][kd * 9 + t]
      for (int wi = 0; wi < 8; ++wi) s += red[wi][ll][t * 4 + j];
      pb[c * 27 + kd * 9 + t] = s;
    } else if (kd == 0) {
      for (int wi = 0; wi < 8; ++wi) s += red[wi][0][9 * 4];
      pb[27 * C] = s;
    }
  }
}

__global__ void tail_wgrad_reduce_k(const float* __restrict__ part, int nblk, int n, float* __restrict__ gw,
                                    long long gwbs) {
  D2IP_PDL_ENTRY();
  const int b = blockIdx.y;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const float* p = part + (long long)b * nblk * n + i;
  float s = 0.f;
#pragma unroll 8
  for (int k = 0; k < nblk; ++k) s += __ldg(p + (long long)k * n);
  gw[b * gwbs + i] = s;  // [c][t] weights then the bias: the OIDHW + bias parameter layout
}

static bool tail_g_ok(const d2ip_act& x) {
  const int G = x.c / 4;
  return x.c % 4 == 0 && (G == 1 || G == 2 || G == 4 || G == 8) && x.cstride % 4 == 0 &&
         ((uintptr_t)x.ptr & 15) == 0;
}

int tail_fwd(d2ip_act x, const float* w, const float* bias, long long wbs, float lo, float scale,
             float* sig, float* mapped, float* sigma_c, long long sc_bs, const int* col_of_vox,
             int batch, cudaStream_t st) {
  const long long V = (long long)x.d * x.h * x.w;
  if (tail_g_ok(x)) {
    const dim3 grid(cdiv(V * (x.c / 4), 256), batch);
#define D2IP_TAILF(G_)                                                                                          \
  case G_:                                                                                                      \
    D2IP_CUDA(launch_pdl(tail_fwd_g_k<G_>, grid, 256, 0, st, x, w, bias, wbs, lo, scale, sig, mapped, sigma_c, \
                         sc_bs, col_of_vox));                                                                   \
    break;
    switch (x.c / 4) { D2IP_TAILF(1) D2IP_TAILF(2) D2IP_TAILF(4) D2IP_TAILF(8) }
#undef D2IP_TAILF
    D2IP_LAUNCH_CHECK();
    return D2IP_OK;
  }
  D2IP_CHECK_ARG(27 * x.c * sizeof(float) <= 40 * 1024, "tail: C_in too large");
  D2IP_CUDA(launch_pdl(tail_fwd_k, dim3(cdiv(V, 32), batch), 96, (27 * x.c + 96) * sizeof(float), st, x, w, bias,
                       wbs, lo, scale, sig, mapped, sigma_c, sc_bs, col_of_vox));
  D2IP_LAUNCH_CHECK();
  return D2IP_OK;
}

bool tail_bwd_supported(d2ip_act x) { return tail_g_ok(x); }

int tail_dgrad(const float* gt, const float* w, long long wbs, d2ip_act gx, int batch, cudaStream_t st) {
  D2IP_CHECK_ARG(tail_g_ok(gx), "tail_dgrad: channels must be 4, 8, 16 or 32, 16-byte aligned");
  const long long V = (long long)gx.d * gx.h * gx.w;
  const dim3 grid(cdiv(V * (gx.c / 4), 256), batch);
#define D2IP_TAILD(G_) \
  case G_: D2IP_CUDA(launch_pdl(tail_dgrad_g_k<G_>, grid, 256, 0, st, gt, w, wbs, gx)); break;
  switch (gx.c / 4) { D2IP_TAILD(1) D2IP_TAILD(2) D2IP_TAILD(4) D2IP_TAILD(8) }
#undef D2IP_TAILD
  D2IP_LAUNCH_CHECK();
  return D2IP_OK;
}

static int tail_wgrad_blocks(long long V) { return (int)std::min<long long>(296, std::max<long long>(1, V / 256)); }

size_t tail_wgrad_ws(int C, long long V, int batch) {
  return (size_t)batch * tail_wgrad_blocks(V) * (27 * C + 1) * sizeof(float);
}

int tail_wgrad(d2ip_act x, const float* gt, float* gw, long long gwbs, void* ws, size_t ws_bytes, int batch,
               cudaStream_t st) {
  D2IP_CHECK_ARG(tail_g_ok(x), "tail_wgrad: channels must be 4, 8, 16 or 32, 16-byte aligned");
  const long long V = (long long)x.d * x.h * x.w;
  const int nblk = tail_wgrad_blocks(V);
  D2IP_CHECK_ARG(ws_bytes >= tail_wgrad_ws(x.c, V, batch), "tail_wgrad: workspace too small");
  const int vchunk = cdiv(V, nblk);
  float* part = reinterpret_cast<float*>(ws);
  const dim3 grid(nblk, batch, 3);
#define D2IP_TAILW(G_) \
  case G_: D2IP_CUDA(launch_pdl(tail_wgrad_g_k<G_>, grid, 256, 0, st, x, gt, vchunk, part)); break;
  switch (x.c / 4) { D2IP_TAILW(1) D2IP_TAILW(2) D2IP_TAILW(4) D2IP_TAILW(8) }
#undef D2IP_TAILW
  D2IP_LAUNCH_CHECK();
  const int n = 27 * x.c + 1;
  D2IP_CUDA(launch_pdl(tail_wgrad_reduce_k, dim3(cdiv(n, 256), batch), 256, 0, st, part, nblk, n, gw, gwbs));
  D2IP_LAUNCH_CHECK();
  return D2IP_OK;
}

// gtail = gmapped * scale * (1 - s) * s over all voxels (TV on: gmapped holds
// TV + data gradients for every voxel).
__global__ void tail_bwd_prep_k(const float* __restrict__ gm, const float* __restrict__ sig, float scale,
                                float* __restrict__ gt, long long n) {
  D2IP_PDL_ENTRY();
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const float s = sig[i];
  gt[i] = (gm[i] * scale) * (1.f - s) * s;
}

int tail_bwd_prep(const float* gmapped, const float* sig, float scale, float* gtail, long long V0,
                  int batch, cudaStream_t st) {
  const long long n = V0 * batch;
  D2IP_CUDA(launch_pdl(tail_bwd_prep_k, cdiv(n, 256), 256, 0, st, gmapped, sig, scale, gtail, n));
  D2IP_LAUNCH_CHECK();
  return D2IP_OK;
}

}  // namespace d2ip
