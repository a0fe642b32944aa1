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

int tail_fwd(d2ip_act x, const float* w, const float* bias, long long wbs, float lo, float scale,
             float* sig, float* mapped, float* sigma_c, long long sc_bs, const int* col_of_vox,
             int batch, cudaStream_t st) {
  const long long V = (long long)x.d * x.h * x.w;
  D2IP_CHECK_ARG(27 * x.c * sizeof(float) <= 40 * 1024, "tail: C_in too large");
  D2IP_CUDA(launch_pdl(tail_fwd_k, dim3(cdiv(V, 32), batch), 96, (27 * x.c + 96) * sizeof(float), st, x, w, bias,
                       wbs, lo, scale, sig, mapped, sigma_c, sc_bs, col_of_vox));
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
