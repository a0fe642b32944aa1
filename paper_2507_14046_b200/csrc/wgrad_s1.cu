// K3: weight + bias gradient of the stride-1 3x3x3 convolutions (autograd's
// conv backward w.r.t. weight/bias, pipeline.py:330), the K = voxels
// reduction dW[co][ci][t] = sum_u gy[u][co] * x[u + off_t][ci].
//
// Same virtual zero-padded row space as the tcgen05 forward (conv_tc.cu): a
// tap is the constant row shift off_t, so a CTA stages, for one plane tap kd,
// a window of gy rows [u0, u0+128) and an input window of 128 + 2*Sw + 2 rows
// in shared memory and every (kh, kw) tap reads the input window at a fixed
// offset. Each thread owns a 4 (c_in) x 8 (c_out) register tile of one tap:
// per row one float4 of x and two float4 of gy (shared memory, broadcast)
// feed 32 FMAs. Row chunks are double-buffered with cp.async (zero-fill on
// the padding). Border rows of the virtual grid carry gy = 0 and contribute
// nothing. The bias gradient rides along in the centre-tap threads.
// Partials per row group are summed in a fixed order (deterministic).
#include <algorithm>

#include "common.cuh"
#include "kernels.h"
#include "tc.cuh"

namespace d2ip {

constexpr int kWgRows = 128;

struct WgS1 {
  d2ip_act x, gy;
  int Sw, Sh, WR, u_first, u_last;
  int CIB, COB, ncib, ncob;
  int rg, chunks_per_rg, nchunks;
  int ks;  // 3: 27 taps; 1: the 1^3 skip convolution (centre tap only)
  float* part;  // [b][rg][tiles][32]  (+ bias block [b][rg][cout])
  long long tiles;
};

__global__ void __launch_bounds__(288) wgrad_s1_k(WgS1 a) {
  D2IP_PDL_ENTRY();
  extern __shared__ __align__(16) float sm[];
  const int b = blockIdx.z;
  const int rg = blockIdx.x;
  const int job = blockIdx.y;
  const int nkd = a.ks == 3 ? 3 : 1;
  const int kd = a.ks == 3 ? job % 3 : 1, cib = (job / nkd) % a.ncib, cob = job / (nkd * a.ncib);
  const int CIB = a.CIB, COB = a.COB;
  const int nci4 = CIB / 4, nco8 = COB / 8;
  const int tid = threadIdx.x;
  const int t9 = a.ks == 3 ? tid / (nci4 * nco8) : 4, rem = tid % (nci4 * nco8);
  const int ci4 = rem / nco8, co8 = rem % nco8;
  const int nthr = (a.ks == 3 ? 9 : 1) * nci4 * nco8;
  const d2ip_act x = a.x, gy = a.gy;
  const int Cin = x.c, Cout = gy.c;
  const float* xb = x.ptr + b * x.bstride + cib * CIB;
  const float* gb = gy.ptr + b * gy.bstride + cob * COB;
  // smem: 2 buffers of [G rows x COB] + [X rows x CIB]
  const int gsz = kWgRows * COB, xsz = a.WR * CIB;
  float* G[2] = {sm, sm + gsz + xsz};
  float* X[2] = {sm + gsz, sm + 2 * gsz + xsz};
  const bool active = tid < nthr;
  const bool do_bias = active && (a.ks == 1 || kd == 0) && cib == 0 && t9 == 4 && ci4 == 0;
  const int rowoff = (t9 / 3) * a.Sw + (t9 % 3);
  float acc[4][8], bacc[8];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;
#pragma unroll
  for (int j = 0; j < 8; ++j) bacc[j] = 0.f;

  auto voxel = [&](int u) -> int {  // virtual row -> voxel offset or -1
    if (u < 0) return -1;
    const int dp = u / a.Sh, r = u - dp * a.Sh;
    const int hp = r / a.Sw, wp = r - hp * a.Sw;
    if (dp >= 1 && dp <= x.d && hp >= 1 && hp <= x.h && wp >= 1 && wp <= x.w)
      return ((dp - 1) * x.h + (hp - 1)) * x.w + (wp - 1);
    return -1;
  };
  const int c_lo = rg * a.chunks_per_rg, c_hi = min(a.nchunks, c_lo + a.chunks_per_rg);
  auto load = [&](int c, int buf) {
    const int u0 = a.u_first + c * kWgRows;
    const int ng = kWgRows * (COB / 4);
    for (int i = tid; i < ng; i += blockDim.x) {
      const int r = i / (COB / 4), q = i % (COB / 4);
      const int u = u0 + r;
      const int v = u <= a.u_last ? voxel(u) : -1;
      tc::cp_async16(G[buf] + r * COB + 4 * q, v >= 0 ? gb + (long long)v * gy.cstride + 4 * q : gb,
                     v >= 0 ? 16u : 0u);
    }
    const int ub = u0 + (kd - 1) * a.Sh - a.Sw - 1;
    const int nx = a.WR * (CIB / 4);
    for (int i = tid; i < nx; i += blockDim.x) {
      const int r = i / (CIB / 4), q = i % (CIB / 4);
      const int v = voxel(ub + r);
      tc::cp_async16(X[buf] + r * CIB + 4 * q, v >= 0 ? xb + (long long)v * x.cstride + 4 * q : xb,
                     v >= 0 ? 16u : 0u);
    }
    tc::cp_async_commit();
  };
  if (c_lo < c_hi) load(c_lo, 0);
  for (int c = c_lo; c < c_hi; ++c) {
    const int buf = (c - c_lo) & 1;
    if (c + 1 < c_hi) {
      load(c + 1, buf ^ 1);
      tc::cp_async_wait<1>();
    } else {
      tc::cp_async_wait<0>();
    }
    __syncthreads();
    if (active) {
      const float* gs = G[buf] + co8 * 8;
      const float* xs = X[buf] + rowoff * CIB + ci4 * 4;
#pragma unroll 4
      for (int r = 0; r < kWgRows; ++r) {
        const float4 g0 = *reinterpret_cast<const float4*>(gs + r * COB);
        const float4 g1 = *reinterpret_cast<const float4*>(gs + r * COB + 4);
        const float4 xv = *reinterpret_cast<const float4*>(xs + r * CIB);
        const float g[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
        const float xx[4] = {xv.x, xv.y, xv.z, xv.w};
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(xx[i], g[j], acc[i][j]);
        if (do_bias) {
#pragma unroll
          for (int j = 0; j < 8; ++j) bacc[j] += g[j];
        }
      }
    }
    __syncthreads();
  }
  if (!active) return;
  // tile id in [0, 27 * Cin/4 * Cout/8)
  const int ci4g = cib * nci4 + ci4, co8g = cob * nco8 + co8;
  const int tap = a.ks == 3 ? kd * 9 + t9 : 0;
  const long long tile = ((long long)tap * (Cin / 4) + ci4g) * (Cout / 8) + co8g;
  float* p = a.part + (((long long)b * a.rg + rg) * (a.tiles * 32 + Cout)) + tile * 32;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) p[i * 8 + j] = acc[i][j];
  if (do_bias) {
    float* pb = a.part + (((long long)b * a.rg + rg) * (a.tiles * 32 + Cout)) + a.tiles * 32 + co8g * 8;
#pragma unroll
    for (int j = 0; j < 8; ++j) pb[j] = bacc[j];
  }
}

// sum over row groups (fixed order) and scatter to OIDHW weight + bias grads
__global__ void __launch_bounds__(256) wgrad_s1_reduce_k(const float* __restrict__ part, int rg, long long tiles,
                                                         int Cin, int Cout, int K3, float* __restrict__ out,
                                                         long long obs) {
  D2IP_PDL_ENTRY();
  __shared__ float red[8][33];
  const int b = blockIdx.y;
  const long long n = tiles * 32 + Cout;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const long long j = (long long)blockIdx.x * 32 + lane;
  float s = 0.f;
  if (j < n) {
    const float* p = part + (long long)b * rg * n + j;
    float s0 = 0.f, s1 = 0.f;
    int c = w;
    for (; c + 8 < rg; c += 16) {
      s0 += p[(long long)c * n];
      s1 += p[(long long)(c + 8) * n];
    }
    for (; c < rg; c += 8) s0 += p[(long long)c * n];
    s = s0 + s1;
  }
  red[w][lane] = s;
  __syncthreads();
  if (w != 0 || j >= n) return;
  s = 0.f;
#pragma unroll
  for (int q = 0; q < 8; ++q) s += red[q][lane];
  long long e;
  if (j < tiles * 32) {
    const long long tile = j / 32;
    const int slot = (int)(j % 32), i = slot / 8, jj = slot % 8;
    const int co8 = (int)(tile % (Cout / 8));
    const long long r2 = tile / (Cout / 8);
    const int ci4 = (int)(r2 % (Cin / 4)), t = (int)(r2 / (Cin / 4));
    const int co = co8 * 8 + jj, ci = ci4 * 4 + i;
    e = ((long long)co * Cin + ci) * K3 + t;
  } else {
    e = (long long)Cout * Cin * K3 + (j - tiles * 32);
  }
  out[b * obs + e] = s;
}

static int pick_block(int c, std::initializer_list<int> opts) {
  for (int o : opts)
    if (o <= c && c % o == 0) return o;
  return 0;
}

static bool wg_plan(int D, int H, int W, int Cin, int Cout, int ks, int batch, WgS1& a) {
  a.ks = ks;
  if (Cin % 4 || Cout % 8) return false;
  // channel tiles: 9 taps x CIB/4 x COB/8 threads per CTA; prefer tiles that
  // fill whole warps (e.g. C_in = 48: CIB = 48 -> 216 threads, not 16 -> 72 of 96)
  a.COB = pick_block(Cout, {32, 16, 8});
  a.CIB = 0;
  if (a.COB)
    for (int cib : {32, 48, 24, 16, 8, 4}) {
      if (cib > Cin || Cin % cib) continue;
      const int thr = (ks == 3 ? 9 : 1) * (cib / 4) * (a.COB / 8);
      if (thr > 288) continue;
      if (!a.CIB) a.CIB = cib;                 // largest-first fallback
      if (thr % 32 == 0 || thr >= 192) {       // whole warps, or big enough that the tail warp matters little
        a.CIB = cib;
        break;
      }
    }
  if (!a.CIB || !a.COB) return false;
  a.ncib = Cin / a.CIB;
  a.ncob = Cout / a.COB;
  a.Sw = W + 2;
  a.Sh = (H + 2) * a.Sw;
  a.WR = kWgRows + 2 * a.Sw + 2;
  a.u_first = a.Sh + a.Sw + 1;
  a.u_last = D * a.Sh + H * a.Sw + W;
  a.nchunks = cdiv(a.u_last - a.u_first + 1, kWgRows);
  const long long jobs = (ks == 3 ? 3LL : 1LL) * a.ncib * a.ncob * batch;
  int rg = (int)std::max(1LL, std::min<long long>(a.nchunks, (148LL * 4 + jobs - 1) / jobs));
  a.chunks_per_rg = cdiv(a.nchunks, rg);
  a.rg = cdiv(a.nchunks, a.chunks_per_rg);
  a.tiles = (long long)ks * ks * ks * (Cin / 4) * (Cout / 8);
  return true;
}

static size_t wg_smem(const WgS1& a) { return 2 * (size_t)(kWgRows * a.COB + a.WR * a.CIB) * sizeof(float); }

bool wgrad_s1_supported(d2ip_act x, d2ip_act gy, int ks) {
  if (x.d != gy.d || x.h != gy.h || x.w != gy.w) return false;
  if (x.cstride % 4 || gy.cstride % 4 || ((uintptr_t)x.ptr & 15) || ((uintptr_t)gy.ptr & 15)) return false;
  WgS1 a{};
  if (!wg_plan(x.d, x.h, x.w, x.c, gy.c, ks, 1, a)) return false;
  return wg_smem(a) <= 200 * 1024;
}

size_t wgrad_s1_ws_bytes(int D, int H, int W, int Cin, int Cout, int ks, int batch) {
  WgS1 a{};
  if (!wg_plan(D, H, W, Cin, Cout, ks, batch, a)) return 0;
  return (size_t)batch * a.rg * (a.tiles * 32 + Cout) * sizeof(float);
}

int wgrad_s1(d2ip_act x, d2ip_act gy, int ks, float* gw, long long gwbs, void* ws, size_t ws_bytes, int batch,
             cudaStream_t st) {
  WgS1 a{};
  D2IP_CHECK_ARG(wg_plan(x.d, x.h, x.w, x.c, gy.c, ks, batch, a), "wgrad_s1: unsupported shape");
  D2IP_CHECK_ARG(ws_bytes >= wgrad_s1_ws_bytes(x.d, x.h, x.w, x.c, gy.c, ks, batch), "wgrad_s1: workspace too small");
  a.x = x;
  a.gy = gy;
  a.part = reinterpret_cast<float*>(ws);
  const size_t smem = wg_smem(a);
  static bool attr = false;
  if (!attr) {
    D2IP_CUDA(cudaFuncSetAttribute(wgrad_s1_k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    attr = true;
  }
  const int nthr = (ks == 3 ? 9 : 1) * (a.CIB / 4) * (a.COB / 8);
  const int threads = (nthr + 31) / 32 * 32;
  D2IP_CUDA(launch_pdl(wgrad_s1_k, dim3(a.rg, (ks == 3 ? 3 : 1) * a.ncib * a.ncob, batch), threads, smem, st, a));
  D2IP_LAUNCH_CHECK();
  const long long n = a.tiles * 32 + gy.c;
  D2IP_CUDA(launch_pdl(wgrad_s1_reduce_k, dim3(cdiv(n, 32), batch), 256, 0, st, a.part, a.rg, a.tiles, x.c, gy.c, ks * ks * ks, gw,
                                                               gwbs));
  D2IP_LAUNCH_CHECK();
  return D2IP_OK;
}

}  // namespace d2ip
