// ChannelLayerNorm (+ residual) (+ LeakyReLU) forward and backward.
//
//   ChannelLayerNorm  pkg/src/d2ip/priornet.py:96-108 (per-voxel LayerNorm over
//                     channels, eps 1e-5, biased variance)
//   ResConv3d tail    priornet.py:145-148 (norm -> [+ skip] -> activation)
//
// Layout: a voxel's C channels are contiguous (NDHWC view). A group of G
// lanes (power of two, <= 32) owns one voxel; each active lane holds VPL = 4
// (C <= 128) or 8 (C <= 256) consecutive channels in registers, loaded and
// stored as float4. Per-voxel means are xor-shuffle reductions inside the
// group. The backward also accumulates the dgamma / dbeta column sums in
// registers across the voxels a lane visits and reduces them per block in a
// fixed order (deterministic), followed by one fixed-order pass over blocks.
#include "common.cuh"
#include "kernels.h"

namespace d2ip {

constexpr float kLnEps = 1e-5f;
constexpr int kNormThreads = 256;

struct NormGeom {
  int vpl, lanes, G;
};

static NormGeom norm_geom(int C) {
  NormGeom g;
  g.vpl = C <= 128 ? 4 : 8;
  g.lanes = C / g.vpl;
  g.G = 1;
  while (g.G < g.lanes) g.G *= 2;
  return g;
}

__device__ __forceinline__ float group_sum(float v, int G) {
  for (int o = G >> 1; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

template <int VPL>
__device__ __forceinline__ void ld(const float* p, float (&v)[VPL]) {
#pragma unroll
  for (int i = 0; i < VPL; i += 4) {
    const float4 q = *reinterpret_cast<const float4*>(p + i);
    v[i] = q.x; v[i + 1] = q.y; v[i + 2] = q.z; v[i + 3] = q.w;
  }
}

template <int VPL>
__device__ __forceinline__ void st(float* p, const float (&v)[VPL]) {
#pragma unroll
  for (int i = 0; i < VPL; i += 4) *reinterpret_cast<float4*>(p + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
}

// bf16 twin of an fp32 row (round to nearest): VPL x 2 bytes
template <int VPL>
__device__ __forceinline__ void st_bf(const d2ip_act& a, long long off, const float (&v)[VPL]) {
  uint32_t w[VPL / 2];
#pragma unroll
  for (int i = 0; i < VPL; i += 2) w[i / 2] = bf16x2(v[i], v[i + 1]);
  uint16_t* p = reinterpret_cast<uint16_t*>(a.bf16) + off;
  if (VPL == 4) *reinterpret_cast<uint2*>(p) = make_uint2(w[0], w[1]);
  else
#pragma unroll
    for (int i = 0; i < VPL / 2; i += 4) *reinterpret_cast<uint4*>(p + 2 * i) = make_uint4(w[i], w[i + 1], w[i + 2], w[i + 3]);
}

template <int VPL>
__global__ void __launch_bounds__(kNormThreads) norm_act_fwd_k(d2ip_act y, const float* __restrict__ gamma,
                                                               const float* __restrict__ beta, long long pbs,
                                                               d2ip_act res, int act, float slope, d2ip_act out,
                                                               float* __restrict__ xhat, float* __restrict__ rstd,
                                                               int G, SplitK sk, d2ip_act pre) {
  D2IP_PDL_ENTRY();
  const int b = blockIdx.y;
  const int C = y.c, L = C / VPL;
  const long long V = (long long)y.d * y.h * y.w;
  const int li = threadIdx.x % G;
  const int groups = kNormThreads / G;
  const bool active = li < L;
  const int c0 = li * VPL;
  float gm[VPL], bt[VPL];  // scalar loads: per-sequence parameter sets are not 16-B aligned
  if (active) {
#pragma unroll
    for (int i = 0; i < VPL; ++i) {
      gm[i] = __ldg(gamma + b * pbs + c0 + i);
      bt[i] = __ldg(beta + b * pbs + c0 + i);
    }
  }
  for (long long v = (long long)blockIdx.x * groups + threadIdx.x / G; v - threadIdx.x / G < V;
       v += (long long)gridDim.x * groups) {
    const bool ok = active && v < V;
    float x[VPL];
#pragma unroll
    for (int i = 0; i < VPL; ++i) x[i] = 0.f;
    if (ok) {
      if (sk.part) {  // the producing convolution's split-K partials + bias (fixed order)
        const float* p = sk.part + ((long long)b * sk.kspl * V + v) * C + c0;
#pragma unroll
        for (int i = 0; i < VPL; ++i) x[i] = __ldg(sk.bias + b * sk.bbs + c0 + i);
        // (four partial loads in flight; the sum keeps the order k = 0, 1, ...)
        const long long ps = V * C;
        int k = 0;
        for (; k + 3 < sk.kspl; k += 4) {
          float t0[VPL], t1[VPL], t2[VPL], t3[VPL];
          ld<VPL>(p + (long long)k * ps, t0);
          ld<VPL>(p + (long long)(k + 1) * ps, t1);
          ld<VPL>(p + (long long)(k + 2) * ps, t2);
          ld<VPL>(p + (long long)(k + 3) * ps, t3);
#pragma unroll
          for (int i = 0; i < VPL; ++i) {
            x[i] += t0[i];
            x[i] += t1[i];
            x[i] += t2[i];
            x[i] += t3[i];
          }
        }
        for (; k < sk.kspl; ++k) {
          float t[VPL];
          ld<VPL>(p + (long long)k * ps, t);
#pragma unroll
          for (int i = 0; i < VPL; ++i) x[i] += t[i];
        }
      } else {
        ld<VPL>(y.ptr + b * y.bstride + v * y.cstride + c0, x);
      }
    }
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < VPL; ++i) s += x[i];
    const float mean = group_sum(s, G) / (float)C;
    float q = 0.f;
#pragma unroll
    for (int i = 0; i < VPL; ++i) {
      const float d = ok ? x[i] - mean : 0.f;
      q = fmaf(d, d, q);
    }
    const float rs = 1.0f / sqrtf(group_sum(q, G) / (float)C + kLnEps);
    if (ok) {
      float xh[VPL], o[VPL], r[VPL];
#pragma unroll
      for (int i = 0; i < VPL; ++i) xh[i] = (x[i] - mean) * rs;
      if (res.ptr) ld<VPL>(res.ptr + b * res.bstride + v * res.cstride + c0, r);
#pragma unroll
      float pr[VPL];
      for (int i = 0; i < VPL; ++i) {
        float t = fmaf(xh[i], gm[i], bt[i]);
        if (res.ptr) t += r[i];
        pr[i] = t;
        o[i] = act == 1 ? lrelu(t, slope) : (act == 2 ? t / (1.0f + expf(-t)) : t);
      }
      if (pre.ptr) st<VPL>(pre.ptr + b * pre.bstride + v * pre.cstride + c0, pr);
      st<VPL>(xhat + ((long long)b * V + v) * C + c0, xh);
      st<VPL>(out.ptr + b * out.bstride + v * out.cstride + c0, o);
      if (out.bf16) st_bf<VPL>(out, b * out.bstride + v * out.cstride + c0, o);
      if (li == 0) rstd[b * V + v] = rs;
    }
  }
}

static int norm_blocks(long long V, int G, int batch) {
  const long long per = kNormThreads / G;
  long long nb = (V + per - 1) / per;
  const long long cap = (148LL * 8 + batch - 1) / batch;
  return (int)std::max(1LL, std::min(nb, cap));
}

int norm_act_fwd(d2ip_act y, const float* gamma, const float* beta, long long pbs, d2ip_act res, int act,
                 float slope, d2ip_act out, float* xhat, float* rstd, int batch, cudaStream_t st, SplitK sk,
                 d2ip_act pre) {
  const int C = y.c;
  D2IP_CHECK_ARG(C % 4 == 0 && C <= 256, "norm_act: C=%d must be a multiple of 4, <= 256", C);
  D2IP_CHECK_ARG(y.cstride % 4 == 0 && out.cstride % 4 == 0 && (!res.ptr || res.cstride % 4 == 0),
                 "norm_act: views must be float4 aligned");
  D2IP_CHECK_ARG(!sk.part || sk.bias, "norm_act: split-K partials need the bias");
  const NormGeom g = norm_geom(C);
  const long long V = (long long)y.d * y.h * y.w;
  dim3 grid(norm_blocks(V, g.G, batch), batch);
  if (g.vpl == 4)
    D2IP_CUDA(launch_pdl(norm_act_fwd_k<4>, grid, kNormThreads, 0, st, y, gamma, beta, pbs, res, act, slope, out,
                         xhat, rstd, g.G, sk, pre));
  else
    D2IP_CUDA(launch_pdl(norm_act_fwd_k<8>, grid, kNormThreads, 0, st, y, gamma, beta, pbs, res, act, slope, out,
                         xhat, rstd, g.G, sk, pre));
  D2IP_LAUNCH_CHECK();
  return D2IP_OK;
}

// gpre = gout * act'(out);  gc = rstd * (gpre*gamma - mean(gpre*gamma) - xhat * mean(gpre*gamma*xhat))
// partial[b][block][0..C) = sum gpre*xhat, [C..2C) = sum gpre over the block's voxels.
template <int VPL>
__global__ void __launch_bounds__(kNormThreads) norm_act_bwd_k(d2ip_act gout, d2ip_act out, int act, float slope,
                                                               const float* __restrict__ xhat,
                                                               const float* __restrict__ rstd,
                                                               const float* __restrict__ gamma, long long pbs,
                                                               d2ip_act gpre, d2ip_act gc,
                                                               float* __restrict__ partial, int G, SplitK sk) {
  D2IP_PDL_ENTRY();
  extern __shared__ float red[];  // [groups][2C]
  const int b = blockIdx.y;
  const int C = gout.c, L = C / VPL;
  const long long V = (long long)gout.d * gout.h * gout.w;
  const int li = threadIdx.x % G, grp = threadIdx.x / G;
  const int groups = kNormThreads / G;
  const bool active = li < L;
  const int c0 = li * VPL;
  float gm[VPL], cs1[VPL], cs2[VPL];
#pragma unroll
  for (int i = 0; i < VPL; ++i) cs1[i] = cs2[i] = 0.f;
  if (active) {
#pragma unroll
    for (int i = 0; i < VPL; ++i) gm[i] = __ldg(gamma + b * pbs + c0 + i);
  }
  for (long long v = (long long)blockIdx.x * groups + grp; v - grp < V; v += (long long)gridDim.x * groups) {
    const bool ok = active && v < V;
    float g[VPL], xh[VPL];
#pragma unroll
    for (int i = 0; i < VPL; ++i) g[i] = xh[i] = 0.f;
    if (ok) {
      if (sk.part) {  // the producing data-gradient convolution's split-K partials (fixed order, no bias)
        const float* p = sk.part + ((long long)b * sk.kspl * V + v) * C + c0;
        const long long ps = V * C;
        int k = 0;
        for (; k + 3 < sk.kspl; k += 4) {  // four partial loads in flight, same summation order
          float t0[VPL], t1[VPL], t2[VPL], t3[VPL];
          ld<VPL>(p + (long long)k * ps, t0);
          ld<VPL>(p + (long long)(k + 1) * ps, t1);
          ld<VPL>(p + (long long)(k + 2) * ps, t2);
          ld<VPL>(p + (long long)(k + 3) * ps, t3);
#pragma unroll
          for (int i = 0; i < VPL; ++i) {
            g[i] += t0[i];
            g[i] += t1[i];
            g[i] += t2[i];
            g[i] += t3[i];
          }
        }
        for (; k < sk.kspl; ++k) {
          float t[VPL];
          ld<VPL>(p + (long long)k * ps, t);
#pragma unroll
          for (int i = 0; i < VPL; ++i) g[i] += t[i];
        }
      } else {
        ld<VPL>(gout.ptr + b * gout.bstride + v * gout.cstride + c0, g);
      }
      ld<VPL>(xhat + ((long long)b * V + v) * C + c0, xh);
      if (act) {
        float o[VPL];
        ld<VPL>(out.ptr + b * out.bstride + v * out.cstride + c0, o);
#pragma unroll
        for (int i = 0; i < VPL; ++i) {
          if (act == 1) {
            g[i] = o[i] > 0.f ? g[i] : g[i] * slope;
          } else {  // SiLU': `out` holds the pre-activation
            const float s = 1.0f / (1.0f + expf(-o[i]));
            g[i] *= s * (1.0f + o[i] * (1.0f - s));
          }
        }
      }
    }
    float s1 = 0.f, s2 = 0.f;
#pragma unroll
    for (int i = 0; i < VPL; ++i) {
      const float gx = ok ? g[i] * gm[i] : 0.f;
      s1 += gx;
      s2 = fmaf(gx, xh[i], s2);
    }
    const float m1 = group_sum(s1, G) / (float)C, m2 = group_sum(s2, G) / (float)C;
    if (ok) {
      const float rs = rstd[b * V + v];
      float o[VPL];
#pragma unroll
      for (int i = 0; i < VPL; ++i) {
        o[i] = rs * (g[i] * gm[i] - m1 - xh[i] * m2);
        cs1[i] = fmaf(g[i], xh[i], cs1[i]);
        cs2[i] += g[i];
      }
      if (gpre.ptr) st<VPL>(gpre.ptr + b * gpre.bstride + v * gpre.cstride + c0, g);
      if (gpre.ptr && gpre.bf16) st_bf<VPL>(gpre, b * gpre.bstride + v * gpre.cstride + c0, g);
      st<VPL>(gc.ptr + b * gc.bstride + v * gc.cstride + c0, o);
      if (gc.bf16) st_bf<VPL>(gc, b * gc.bstride + v * gc.cstride + c0, o);
    }
  }
  if (active) {
#pragma unroll
    for (int i = 0; i < VPL; ++i) {
      red[grp * 2 * C + c0 + i] = cs1[i];
      red[grp * 2 * C + C + c0 + i] = cs2[i];
    }
  }
  __syncthreads();
  for (int j = threadIdx.x; j < 2 * C; j += kNormThreads) {
    float s = 0.f;
    for (int q = 0; q < groups; ++q) s += red[q * 2 * C + j];
    partial[((long long)b * gridDim.x + blockIdx.x) * 2 * C + j] = s;
  }
}

size_t norm_act_bwd_ws(long long V, int C, int batch) {
  const NormGeom g = norm_geom(C);
  return (size_t)batch * norm_blocks(V, g.G, batch) * 2 * C * sizeof(float);
}

int norm_act_bwd(d2ip_act gout, d2ip_act out, int act, float slope, const float* xhat, const float* rstd,
                 const float* gamma, long long pbs, d2ip_act gpre, d2ip_act gc, float* dgb, long long dgbs, void* ws,
                 size_t ws_bytes, int batch, cudaStream_t st, int* deferred, SplitK sk) {
  const int C = gout.c;
  D2IP_CHECK_ARG(C % 4 == 0 && C <= 256, "norm_act_bwd: C=%d must be a multiple of 4, <= 256", C);
  D2IP_CHECK_ARG(gout.cstride % 4 == 0 && gc.cstride % 4 == 0 && (!act || out.cstride % 4 == 0) &&
                     (!gpre.ptr || gpre.cstride % 4 == 0),
                 "norm_act_bwd: views must be float4 aligned");
  const NormGeom g = norm_geom(C);
  const long long V = (long long)gout.d * gout.h * gout.w;
  const int nb = norm_blocks(V, g.G, batch);
  D2IP_CHECK_ARG(ws_bytes >= (size_t)batch * nb * 2 * C * sizeof(float), "norm_act_bwd: workspace too small");
  float* partial = reinterpret_cast<float*>(ws);
  const size_t smem = (size_t)(kNormThreads / g.G) * 2 * C * sizeof(float);
  dim3 grid(nb, batch);
  if (g.vpl == 4)
    D2IP_CUDA(launch_pdl(norm_act_bwd_k<4>, grid, kNormThreads, smem, st, gout, out, act, slope, xhat, rstd, gamma, pbs, gpre, gc,
                                                        partial, g.G, sk));
  else
    D2IP_CUDA(launch_pdl(norm_act_bwd_k<8>, grid, kNormThreads, smem, st, gout, out, act, slope, xhat, rstd, gamma, pbs, gpre, gc,
                                                        partial, g.G, sk));
  D2IP_LAUNCH_CHECK();
  if (deferred) {  // the caller sums the dgamma / dbeta partials (reduce_chunks) where it likes
    *deferred = nb;
    return D2IP_OK;
  }
  return reduce_chunks(partial, nb, 2 * C, dgb, dgbs, batch, st);
}

}  // namespace d2ip
