// K1 / K2: stride-1 3x3x3 convolution as a tcgen05 implicit GEMM on the TF32
// tensor-core path with error compensation (3xTF32), FP32 accumulation in
// TMEM. Replaces nn.Conv3d forward and the data gradient of autograd's conv
// backward (priornet.py:117,200,215; pipeline.py:330) for every stride-1 3^3
// layer of the ResUNet.
//
// GEMM view (no im2col): rows are positions u of a *virtual* zero-padded
// grid (D+2)(H+2)(W+2), u = ((d+1)*Sh + (h+1)*Sw + (w+1)), Sh=(H+2)(W+2),
// Sw=W+2; a tap (kd,kh,kw) is the constant row shift
// (kd-1)*Sh + (kh-1)*Sw + (kw-1). One CTA owns 128 consecutive rows (the
// TMEM accumulator: 128 lanes x N fp32 columns) and all N output channels.
// For each plane tap kd (and channel block) it stages one window of
// 128 + 2*Sw + 2 input rows in shared memory in the UMMA K-major
// "interleaved" layout ([channel chunk][row][16 B]); the nine (kh,kw) taps are
// nine descriptors into the same window, shifted by kh*Sw + kw rows — the
// input is read once per plane tap, never expanded 27x. Border rows of the
// virtual grid are computed and discarded by the epilogue. The data gradient
// is the same kernel on gy with the flipped, transposed weight packing
// (conv_transpose at stride 1 == conv with W^T[26-t]).
//
// Precision: a single TF32 pass (10-bit mantissa operands) misses the 1e-3
// gradient bar of the north star over a whole ResUNet backward (measured
// ~6e-3). Each operand is split x = hi + lo with hi = x truncated to TF32 and
// lo = x - hi; the kernel accumulates hi*hi + hi*lo + lo*hi, leaving only the
// lo*lo term (~2^-22 relative) — FP32-level accuracy on the tensor cores.
// Weights are split once per iteration by the pack kernel; the activation
// window is split in shared memory after it lands.
//
// Stride 2 (mode 1 / 2) by parity decomposition: with x = 2o + k - 1, tap
// k = 0 reads parity 1 of voxel o - 1, k = 1 parity 0 of o, k = 2 parity 1 of
// o, so a stride-2 3^3 conv is a stride-1 conv over the output grid whose
// input channels are the 8 parity classes x input channels ("space to depth",
// gathered by the producers, never materialised) and whose taps per axis are
// the offsets {-1, 0} only (t0 = 0, nt = 2: 8 of 27 taps, 2 of 3 planes).
// Its data gradient is the mirror image: a stride-1 conv over the gy grid with
// offsets {0, +1} (t0 = 1) and 8 x C_in output columns, each column block
// scattered by the epilogue to its parity voxel 2o + p of gx. The pack kernel
// lays out the parity weights (zeros where a parity has no tap).
//
// 1^3 layers (mode 3, "pointwise"): one tap, one plane, a window of exactly
// the tile's 128 T rows (no halo) per channel block -- a plain GEMM over voxels
// (the decoder / bottleneck skip convolutions, priornet.py:145-148 restated).
//
// bf16 operands (precision D2IP_PREC_BF16, mode bit kTcBf16): one kind::f16
// MMA per 16-channel K step instead of three kind::tf32 MMAs per 8 channels.
// The producers load the fp32 activation window through registers and store
// it as bf16 (round to nearest), the pack kernel writes bf16 weights; the
// accumulator stays FP32 in TMEM. Measured on sm_100a (tools/umma_chains.cu):
// an M = 128 MMA reads its A tile (128 rows x 32 B) and B tile (N x 32 B) from
// shared memory at ~128 B/cycle, so it costs max(N / 2, (4096 + 32 N) / 128)
// cycles -- 40 at N = 32, 48 at N = 64 -- whatever the operand type: at these
// channel counts bf16 moves 6x more products per MMA cycle than 3xTF32.
//
// Pipeline: 2 smem stages filled with cp.async (16 B, zero-fill outside the
// grid) by all 128 threads; thread 0 issues the MMAs of a stage and commits
// them to that stage's mbarrier, which gates the refill of the buffer.
#include <algorithm>
#include <cstdlib>
#include <cstring>

#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>

#include "common.cuh"
#include "kernels.h"
#include "tc.cuh"

namespace d2ip {

constexpr int kTcThreads = 288;  // warp 0: MMA issue; warps 1-8: two producer groups, then the epilogue
constexpr int kTcProd = 256;
constexpr int kTcRows = 128;
constexpr int kTcpThreads = 416;  // persistent kernel: MMA warp, 8 producer warps, 4 epilogue warps

__host__ __device__ static inline int np_of(int n) { return (n + 15) / 16 * 16; }
static inline int wr_of(int sw, int T = 1) { return T * kTcRows + 2 * sw + 2; }
// Rows per channel-chunk column, padded so a quarter warp of fill / split threads (16-byte
// accesses, i -> (row i / NKC, chunk i % NKC)) covers all 32 banks: the column stride is
// 16 * (8 / min(NKC, 8)) bytes mod 128 (NKC = 2: rows {r..r+3} x 2 columns 64 B apart, ...)
static inline int wrp_of(int wr, int nkc) {
  const int t = 8 / std::min(nkc, 8);
  return wr + ((t - wr) % 8 + 8) % 8;
}

struct TcConv {
  d2ip_act x;
  const float* wp;  // packed [hi | lo] halves, each [27][K/4][Np][4]
  long long wpbs;
  long long wlo;    // float offset of the lo half
  const float* bias;
  long long bbs;
  d2ip_act y;
  int accumulate;
  int N, Np, Ns, Kc, CB, n_cb, WR, WRp, Sw, Sh, u_first, tmem_cols;  // Ns: N columns per CTA (slice)
  int T;        // 128-row tiles per CTA: T TMEM accumulators share every stage's weight tile
  uint32_t idesc;
  int kspl;     // split-K factor over the (plane tap, channel block) stages
  float* part;  // kspl > 1: partial sums [b][kspl][V][N] (mode 2: [b][kspl][V_gx][C_gx])
  long long vout;
  int mode;     // 0: stride 1; 1: stride-2 forward (parity-gathered input); 2: stride-2 dgrad (parity-scattered output); 3: 1^3
  int t0, nt;   // taps per axis used: t0 .. t0 + nt - 1 (offsets t - 1)
  int gd, gh, gw;  // row-space grid (stride 1: x; mode 1: y; mode 2: gy)
  int bf;          // bf16 operands (kind::f16)
  int vec;         // y rows (and bias) 16-byte aligned: float4 epilogue stores
  int pvec;        // split-K partial rows 16-byte aligned (N % 4 == 0, aligned workspace): float4 partial stores
  int xtw;         // bf16: stream x from its bf16 twin (cp.async) instead of converting fp32 rows
  int lrows;       // TMA path: rows per channel-chunk column (whole padded lines: maxlines x Sw)
  int b3;          // 3xbf16 (TF32-precision layer): hi + lo bf16 operands, three MMAs per K step
  int nst;         // conv_tc_k ring depth: 2, or 3 when a third stage fits shared memory
  int async_arrive;  // bf16 twin path: stages complete by cp.async.mbarrier.arrive (D2IP_TC_ASYNC)
  int dbg;           // D2IP_TC_DBG=1: producers skip the fills (MMA-side timing only)
  int ntiles;        // persistent kernel: tiles (blocks of T x 128 rows) of the grid
  int tma;           // MODE 4, 3xTF32: the hi window lines arrive by TMA (tensor map = the kernel's tmap)
  int ln;            // MODE 4, one N slice, no split-K: LayerNorm (+ residual) (+ act) in the epilogue
  LnFuse lnf;
};

// Per stage: A hi + A lo windows, B hi + B lo tiles (nt^2 taps); bf16: one
// A window and one B tile of 2-byte elements.
static size_t stage_bytes(int cb, int np, int wrp, int nt = 3, bool bf = false, bool b3 = false) {
  if (b3) return 2 * ((size_t)cb * wrp * 2 + (size_t)nt * nt * cb * np * 2);
  if (bf) return (size_t)cb * wrp * 2 + (size_t)nt * nt * cb * np * 2;
  return 2 * ((size_t)cb * wrp * 4 + (size_t)nt * nt * cb * np * 4);
}

static size_t tc_smem_bytes(const TcConv& a) {
  return (size_t)a.nst * stage_bytes(a.CB, a.Ns, a.WRp, a.nt, a.bf, a.b3) + 3 * a.WR * sizeof(int) + 8 + 10 * 8 + 16;
}

__device__ __forceinline__ uint32_t bf2(float a, float b) {
  const __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<const uint32_t*>(&h);
}

__device__ __forceinline__ float tf32_hi(float x) { return __uint_as_float(__float_as_uint(x) & 0xFFFFE000u); }

// Epilogue shared by the cp.async- and TMA-fed kernels (producer warps 1-8):
// TMEM lane = GEMM row; warp w reads lane quadrant w % 4 and column half
// (w - 1) / 4; one row / voxel per sub-tile. S = 0: zeros (an empty split).
template <int T, int MODE>
__device__ __forceinline__ void tc_epilogue(const TcConv& a, uint32_t tmem, int b, int n0, int u0, int ks, int S,
                                            int warp, int lane, int cbeg = -1, int cend = -1) {
  const int row = (warp & 3) * 32 + lane;
  if (cbeg < 0) {  // warps 1-8: two warps per lane quadrant, one column half each
    const int chalf = a.Ns / 2;
    cbeg = ((warp - 1) >> 2) * chalf;
    cend = cbeg + chalf;
  }
  const d2ip_act y = a.y;
  const uint32_t trow = tmem + ((uint32_t)((warp & 3) * 32) << 16);
  const float* bias = a.bias ? a.bias + b * a.bbs : nullptr;
  for (int tt = 0; tt < T; ++tt) {
    const int u = u0 + tt * kTcRows + row;
    int v = -1, dq = 0, hq = 0, wq = 0;
    {
      const int dp = u / a.Sh, rem = u - dp * a.Sh;
      const int hp = rem / a.Sw, wp = rem - hp * a.Sw;
      if (dp >= 1 && dp <= a.gd && hp >= 1 && hp <= a.gh && wp >= 1 && wp <= a.gw) {
        v = ((dp - 1) * a.gh + (hp - 1)) * a.gw + (wp - 1);
        dq = dp - 1; hq = hp - 1; wq = wp - 1;
      }
    }
    const uint32_t tcol = trow + (uint32_t)(tt * a.Ns);
    if (MODE == 2) {  // column n = p * C_gx + ci -> gx voxel 2o + p (8 columns share p)
      const int cy = y.c;
      for (int c0 = cbeg; c0 < cend; c0 += 8) {
        float vals[8];
        tc::tmem_ld8(tcol + c0, vals);
        const int n = n0 + c0;
        if (v < 0 || n >= a.N) continue;
        const int p = n / cy, ci = n - p * cy;
        const int d2 = 2 * dq + (p >> 2), h2 = 2 * hq + ((p >> 1) & 1), w2 = 2 * wq + (p & 1);
        if (d2 >= y.d || h2 >= y.h || w2 >= y.w) continue;
        const long long vf = ((long long)d2 * y.h + h2) * y.w + w2;
        const bool z = S <= 0;
        if (a.kspl > 1) {
          float* pp = a.part + (((long long)b * a.kspl + ks) * a.vout + vf) * cy + ci;
          if (a.pvec) {  // 8 channels of one gx voxel: two 16-byte stores
            float4* p4 = reinterpret_cast<float4*>(pp);
            p4[0] = z ? make_float4(0.f, 0.f, 0.f, 0.f) : make_float4(vals[0], vals[1], vals[2], vals[3]);
            p4[1] = z ? make_float4(0.f, 0.f, 0.f, 0.f) : make_float4(vals[4], vals[5], vals[6], vals[7]);
          } else {
#pragma unroll
            for (int j = 0; j < 8; ++j) pp[j] = z ? 0.f : vals[j];
          }
        } else {
          // (the view is 16-byte aligned with C % 8 == 0: checked by conv_tc_run)
          float4* y4 = reinterpret_cast<float4*>(y.ptr + b * y.bstride + vf * y.cstride + ci);
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            float4 o = z ? make_float4(0.f, 0.f, 0.f, 0.f)
                         : make_float4(vals[4 * h], vals[4 * h + 1], vals[4 * h + 2], vals[4 * h + 3]);
            if (a.accumulate) {
              const float4 yo = y4[h];
              o.x += yo.x; o.y += yo.y; o.z += yo.z; o.w += yo.w;
            }
            y4[h] = o;
          }
        }
      }
      continue;
    }
    if (a.kspl > 1) {  // raw partial sums; the consumer adds bias / accumulates
      float* pp = v >= 0 ? a.part + (((long long)b * a.kspl + ks) * a.vout + v) * a.N : nullptr;
      for (int c0 = cbeg; c0 < cend; c0 += 8) {
        float vals[8];
        tc::tmem_ld8(tcol + c0, vals);
        if (pp && a.pvec && n0 + c0 + 8 <= a.N) {
          float4* p4 = reinterpret_cast<float4*>(pp + n0 + c0);
          const bool z = S <= 0;
          p4[0] = z ? make_float4(0.f, 0.f, 0.f, 0.f) : make_float4(vals[0], vals[1], vals[2], vals[3]);
          p4[1] = z ? make_float4(0.f, 0.f, 0.f, 0.f) : make_float4(vals[4], vals[5], vals[6], vals[7]);
        } else if (pp) {
#pragma unroll
          for (int j = 0; j < 8; ++j)
            if (n0 + c0 + j < a.N) pp[n0 + c0 + j] = S > 0 ? vals[j] : 0.f;
        }
      }
      continue;
    }
    float* yp = v >= 0 ? y.ptr + b * y.bstride + (long long)v * y.cstride : nullptr;
    for (int c0 = cbeg; c0 < cend; c0 += 8) {
      float vals[8];
      tc::tmem_ld8(tcol + c0, vals);
      if (yp && a.vec && n0 + c0 + 8 <= a.N) {
        // 8 consecutive channels of one voxel: two 16-byte stores (one 32-byte sector)
        float4* y4 = reinterpret_cast<float4*>(yp + n0 + c0);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          float4 o = make_float4(S > 0 ? vals[4 * h] : 0.f, S > 0 ? vals[4 * h + 1] : 0.f,
                                 S > 0 ? vals[4 * h + 2] : 0.f, S > 0 ? vals[4 * h + 3] : 0.f);
          if (bias) {
            const float* bb = bias + n0 + c0 + 4 * h;
            o.x += __ldg(bb); o.y += __ldg(bb + 1); o.z += __ldg(bb + 2); o.w += __ldg(bb + 3);
          }
          if (a.accumulate) {
            const float4 yo = y4[h];
            o.x += yo.x; o.y += yo.y; o.z += yo.z; o.w += yo.w;
          }
          y4[h] = o;
        }
      } else if (yp) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int n = n0 + c0 + j;
          if (n < a.N) {
            float o = (S > 0 ? vals[j] : 0.f) + (bias ? __ldg(bias + n) : 0.f);
            if (a.accumulate) o += yp[n];
            yp[n] = o;
          }
        }
      }
    }
  }
}

// One voxel row's 8 output channels n .. n + 7 (a split-K partial or the result with bias /
// accumulate), the stride-1 store path of tc_epilogue.
__device__ __forceinline__ void tc_store8(const TcConv& a, int b, int ks, int v, int n, const float* vals,
                                          bool zero, const float* bias) {
  if (v < 0) return;
  if (a.kspl > 1) {
    float* pp = a.part + (((long long)b * a.kspl + ks) * a.vout + v) * a.N;
    if (a.pvec && n + 8 <= a.N) {
      float4* p4 = reinterpret_cast<float4*>(pp + n);
      p4[0] = zero ? make_float4(0.f, 0.f, 0.f, 0.f) : make_float4(vals[0], vals[1], vals[2], vals[3]);
      p4[1] = zero ? make_float4(0.f, 0.f, 0.f, 0.f) : make_float4(vals[4], vals[5], vals[6], vals[7]);
      return;
    }
#pragma unroll
    for (int j = 0; j < 8; ++j)
      if (n + j < a.N) pp[n + j] = zero ? 0.f : vals[j];
    return;
  }
  float* yp = a.y.ptr + b * a.y.bstride + (long long)v * a.y.cstride;
  if (a.vec && n + 8 <= a.N) {
    float4* y4 = reinterpret_cast<float4*>(yp + n);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      float4 o = make_float4(zero ? 0.f : vals[4 * h], zero ? 0.f : vals[4 * h + 1], zero ? 0.f : vals[4 * h + 2],
                             zero ? 0.f : vals[4 * h + 3]);
      if (bias) {
        const float* bb = bias + n + 4 * h;
        o.x += __ldg(bb); o.y += __ldg(bb + 1); o.z += __ldg(bb + 2); o.w += __ldg(bb + 3);
      }
      if (a.accumulate) {
        const float4 yo = y4[h];
        o.x += yo.x; o.y += yo.y; o.z += yo.z; o.w += yo.w;
      }
      y4[h] = o;
    }
    return;
  }
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    if (n + j < a.N) {
      float o = (zero ? 0.f : vals[j]) + (bias ? __ldg(bias + n + j) : 0.f);
      if (a.accumulate) o += yp[n + j];
      yp[n + j] = o;
    }
  }
}

// Epilogue of the kw-folded stride-1 kernel (MODE 4): the accumulator of a sub-tile holds
// three column blocks P_kw[i][n] = sum over kd, kh, k of window row (i + kh Sw) x W[kd][kh][kw];
// output row r (0..125) = P_0[r] + P_1[r + 1] + P_2[r + 2]. Rows r + 1 / r + 2 live in other
// TMEM lanes (other threads, other warps at quadrant edges), so every thread first parks its
// P_1 / P_2 columns in shared memory (the idle stage buffers), then sums. 256 epilogue threads
// (warps 1-8) synchronise on named barrier 1.
template <int T>
__device__ __forceinline__ void tc_epilogue_kwf(const TcConv& a, uint32_t tmem, int b, int n0, int u0, int ks, int S,
                                                int warp, int lane, float* xch) {
  constexpr int RS = kTcRows - 2;
  const int row = (warp & 3) * 32 + lane;
  const int Ns = a.Ns;
  const int chalf = Ns / 2, cbeg = ((warp - 1) >> 2) * chalf, cend = cbeg + chalf;
  const int xs = 2 * Ns + 4;  // exchange row stride (floats): float4 rows, 4-bank skew between rows
  const uint32_t trow = tmem + ((uint32_t)((warp & 3) * 32) << 16);
  const float* bias = a.bias ? a.bias + b * a.bbs : nullptr;
  for (int tt = 0; tt < T; ++tt) {
    const uint32_t tcol = trow + (uint32_t)(tt * 3 * Ns);
    for (int c0 = cbeg; c0 < cend; c0 += 8) {
      float v1[8], v2[8];
      tc::tmem_ld8(tcol + Ns + c0, v1);
      tc::tmem_ld8(tcol + 2 * Ns + c0, v2);
      float4* d1 = reinterpret_cast<float4*>(xch + row * xs + c0);
      float4* d2 = reinterpret_cast<float4*>(xch + row * xs + Ns + c0);
      d1[0] = make_float4(v1[0], v1[1], v1[2], v1[3]);
      d1[1] = make_float4(v1[4], v1[5], v1[6], v1[7]);
      d2[0] = make_float4(v2[0], v2[1], v2[2], v2[3]);
      d2[1] = make_float4(v2[4], v2[5], v2[6], v2[7]);
    }
    asm volatile("bar.sync 1, 256;" ::: "memory");
    // rows 126 / 127 belong to the next sub-tile: they load (tcgen05.ld is warp-collective,
    // .sync.aligned -- every lane must execute it) but store nothing
    int v = -1;
    if (row < RS) {
      const int u = u0 + tt * RS + row;
      const int dp = u / a.Sh, rem = u - dp * a.Sh;
      const int hp = rem / a.Sw, wp = rem - hp * a.Sw;
      if (dp >= 1 && dp <= a.gd && hp >= 1 && hp <= a.gh && wp >= 1 && wp <= a.gw)
        v = ((dp - 1) * a.gh + (hp - 1)) * a.gw + (wp - 1);
    }
    const int rn = row < RS ? row : RS - 1;  // (in-bounds exchange reads for the idle rows)
    if (a.ln) {
      // fused ChannelLayerNorm: this thread holds half of the row's channels (<= 4 chunks of 8);
      // the row statistics combine the two halves through shared memory (fixed order)
      float x[4][8];
      float sum = 0.f;
      const int nch = (cend - cbeg) >> 3;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        if (q < nch) {
          const int c0 = cbeg + 8 * q;
          tc::tmem_ld8(tcol + c0, x[q]);
          const float4* p1 = reinterpret_cast<const float4*>(xch + (rn + 1) * xs + c0);
          const float4* p2 = reinterpret_cast<const float4*>(xch + (rn + 2) * xs + Ns + c0);
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const float4 q1 = p1[h], q2 = p2[h];
            x[q][4 * h] += q1.x + q2.x;
            x[q][4 * h + 1] += q1.y + q2.y;
            x[q][4 * h + 2] += q1.z + q2.z;
            x[q][4 * h + 3] += q1.w + q2.w;
          }
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            x[q][j] = (S > 0 ? x[q][j] : 0.f) + (bias ? __ldg(bias + n0 + c0 + j) : 0.f);
            sum += x[q][j];
          }
        }
      }
      float* st = xch + kTcRows * xs;  // [2][128] row partials
      const int half = (warp - 1) >> 2;
      st[half * kTcRows + row] = sum;
      asm volatile("bar.sync 1, 256;" ::: "memory");
      const float mean = (st[row] + st[kTcRows + row]) / (float)a.N;
      float q2s = 0.f;
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (q < nch)
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const float d = x[q][j] - mean;
            q2s = fmaf(d, d, q2s);
          }
      asm volatile("bar.sync 1, 256;" ::: "memory");
      st[half * kTcRows + row] = q2s;
      asm volatile("bar.sync 1, 256;" ::: "memory");
      const float rs = 1.0f / sqrtf((st[row] + st[kTcRows + row]) / (float)a.N + 1e-5f);
      if (v >= 0) {
        const LnFuse& L = a.lnf;
        const long long V = a.vout;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          if (q < nch) {
            const int c = cbeg + 8 * q;
            float xh[8], o[8];
            float r[8];
            if (L.res.ptr) {
              const float4* rp = reinterpret_cast<const float4*>(L.res.ptr + b * L.res.bstride +
                                                                (long long)v * L.res.cstride + c);
              const float4 r0 = rp[0], r1 = rp[1];
              r[0] = r0.x; r[1] = r0.y; r[2] = r0.z; r[3] = r0.w; r[4] = r1.x; r[5] = r1.y; r[6] = r1.z; r[7] = r1.w;
            }
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              xh[j] = (x[q][j] - mean) * rs;
              float t = fmaf(xh[j], __ldg(L.gamma + b * L.pbs + c + j), __ldg(L.beta + b * L.pbs + c + j));
              if (L.res.ptr) t += r[j];
              o[j] = L.act == 1 ? lrelu(t, L.slope) : t;
            }
            float4* xp = reinterpret_cast<float4*>(L.xhat + ((long long)b * V + v) * a.N + c);
            xp[0] = make_float4(xh[0], xh[1], xh[2], xh[3]);
            xp[1] = make_float4(xh[4], xh[5], xh[6], xh[7]);
            float4* op = reinterpret_cast<float4*>(L.out.ptr + b * L.out.bstride + (long long)v * L.out.cstride + c);
            op[0] = make_float4(o[0], o[1], o[2], o[3]);
            op[1] = make_float4(o[4], o[5], o[6], o[7]);
            if (L.out.bf16) {
              uint4 w;
              w.x = bf2(o[0], o[1]); w.y = bf2(o[2], o[3]); w.z = bf2(o[4], o[5]); w.w = bf2(o[6], o[7]);
              *reinterpret_cast<uint4*>(reinterpret_cast<uint16_t*>(L.out.bf16) + b * L.out.bstride +
                                        (long long)v * L.out.cstride + c) = w;
            }
          }
        }
        if (half == 0) L.rstd[(long long)b * V + v] = rs;
      }
    } else {
    for (int c0 = cbeg; c0 < cend; c0 += 8) {
      float vals[8];
      tc::tmem_ld8(tcol + c0, vals);
      const float4* p1 = reinterpret_cast<const float4*>(xch + (rn + 1) * xs + c0);
      const float4* p2 = reinterpret_cast<const float4*>(xch + (rn + 2) * xs + Ns + c0);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const float4 q1 = p1[h], q2 = p2[h];
        vals[4 * h] += q1.x + q2.x;
        vals[4 * h + 1] += q1.y + q2.y;
        vals[4 * h + 2] += q1.z + q2.z;
        vals[4 * h + 3] += q1.w + q2.w;
      }
      tc_store8(a, b, ks, v, n0 + c0, vals, S <= 0, bias);
    }
    }
    asm volatile("bar.sync 1, 256;" ::: "memory");
  }
}

// NKC: 16-byte channel chunks per row and stage (CB / 4 for tf32, CB / 8 for
// bf16; compile-time, so the fill loops need no integer division).
// PG: producer groups (1: all eight producer warps fill each stage; 2: two
// groups of four fill alternate stages, two stages in flight).
// MODE: 0 stride 1, 1 / 2 stride-2 forward / data gradient (compile-time, so
// the stride-1 issue loop keeps its constant tap arithmetic).
// BFM: 0 3xTF32, 1 bf16, 2 3xbf16 (x = hi + lo in bf16, hi*hi + hi*lo + lo*hi on kind::f16:
// ~2^-16 per product, for the TF32-precision configs at half the MMAs of 3xTF32)
template <int NKC, int T, int PG, int MODE, int BFM = 0>
__global__ void __launch_bounds__(kTcThreads, (MODE == 4 && T == 2 && BFM == 0) ? 2 : 0)
    conv_tc_k(const TcConv a, const __grid_constant__ CUtensorMap tmap) {
  constexpr bool BF = BFM != 0, B3 = BFM == 2;
  D2IP_PDL_ENTRY();
  extern __shared__ __align__(1024) uint8_t smem[];
  constexpr int CB = NKC * (BF ? 8 : 4);
  constexpr int NH = BFM == 1 ? 1 : 2;  // operand halves per stage (3xTF32 / 3xbf16: hi, lo)
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int b = blockIdx.z;
  const int ks = blockIdx.y % a.kspl;
  const int n0 = (blockIdx.y / a.kspl) * a.Ns;  // first output channel of this CTA's slice
  const int Ns = a.Ns, WR = a.WR, WRp = a.WRp;
  constexpr bool PW = MODE == 3;  // 1^3: one tap, window = the tile rows
  constexpr bool KWF = MODE == 4;  // stride 1, the three kw taps folded into N (3 column blocks)
  constexpr int RS = KWF ? kTcRows - 2 : kTcRows;  // output rows per 128-row sub-tile
  constexpr int nt = PW ? 1 : (MODE == 1 || MODE == 2) ? 2 : 3, t0 = MODE == 2 ? 1 : 0, ntap = nt * nt;
  // (kh, kw) of the q-th live tap as a 3x3 index: nt = 3 -> q; nt = 2 -> the 2x2 block at (t0, t0)
  auto tap9 = [&](int q) { return nt == 3 ? q : (t0 + (q >> 1)) * 3 + (t0 + (q & 1)); };
  const int u0 = a.u_first + blockIdx.x * T * RS;
  const uint32_t Ab = (uint32_t)NKC * WRp * 16, Bb = (uint32_t)ntap * NKC * Ns * 16;
  const uint32_t Sb = NH * (Ab + Bb);
  // layout: 2 stages of [A hi][A lo][B hi][B lo] (bf16: [A][B]), row map, barriers full[2] empty[2] done, TMEM slot
  const int NST = a.nst;  // ring depth (2 or 3 stages)
  int* rowmap = reinterpret_cast<int*>(smem + NST * Sb);
  uint64_t* full = reinterpret_cast<uint64_t*>(rowmap + 3 * WR + ((3 * WR) & 1));
  uint64_t* empty = full + 3;
  uint64_t* done = empty + 3;
  uint64_t* landed = done + 1;  // TMA path: the stage's hi window + weights have landed
  uint32_t* tslot = reinterpret_cast<uint32_t*>(landed + 3);

  if (warp == 0) tc::tmem_alloc(tslot, a.tmem_cols);
  if (tid == 0) {
    for (int i = 0; i < NST; ++i) {
      tc::mbar_init(&full[i], kTcProd / PG);  // one producer group fills a stage
      tc::mbar_init(&empty[i], 1);
      tc::mbar_init(&landed[i], 1);
    }
    tc::mbar_init(done, 1);
    tc::fence_mbar_init();
  }
  // voxel offset of every window row for the three plane taps (-1 = padding);
  // mode 1: (even-corner input voxel << 3) | which odd parities exist per axis
  const d2ip_act x = a.x;
  for (int i = tid; i < (PW ? WR : 3 * WR); i += kTcThreads) {
    const int kd = i / WR, r = i - kd * WR;
    const int u = PW ? u0 + r : u0 + (kd - 1) * a.Sh - a.Sw - 1 + r;
    int off = -1;
    if (u >= 0) {
      const int dp = u / a.Sh, rem = u - dp * a.Sh;
      const int hp = rem / a.Sw, wp = rem - hp * a.Sw;
      if (dp >= 1 && dp <= a.gd && hp >= 1 && hp <= a.gh && wp >= 1 && wp <= a.gw) {
        if (MODE == 1) {
          const int d2 = 2 * (dp - 1), h2 = 2 * (hp - 1), w2 = 2 * (wp - 1);
          off = (((d2 * x.h + h2) * x.w + w2) << 3) | ((d2 + 1 < x.d) << 2) | ((h2 + 1 < x.h) << 1) |
                (w2 + 1 < x.w);
        } else {
          off = ((dp - 1) * a.gh + (hp - 1)) * a.gw + (wp - 1);
        }
      }
    }
    rowmap[i] = off;
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = *tslot;
  const float* xb = x.ptr + b * x.bstride;
  const float* wpb = a.wp + b * a.wpbs;
  const int S_all = nt * a.n_cb;
  const int s_lo = (int)((long long)ks * S_all / a.kspl), s_hi = (int)((long long)(ks + 1) * S_all / a.kspl);
  const int S = s_hi - s_lo;  // this CTA's stages: s_lo + [0, S)
  const int nA = WR * NKC;
  const int kc_all = BF ? a.Kc >> 3 : a.Kc >> 2;  // 16-byte chunks per K

  if (warp == 0) {
    // ---- MMA issue (one elected thread); stage s lives in slot s & 1
    if (lane == 0) {
      // descriptors of slot 0; a tap / K step / slot is an add to the 14-bit
      // start-address field (smem addresses < 256 KB never carry out of it)
      const uint32_t sbase = tc::smem_u32(smem);
      const uint64_t dAhi = tc::make_desc(sbase, WRp * 16, 128), dAlo = dAhi + (Ab >> 4);
      const uint64_t dBhi = tc::make_desc(sbase + NH * Ab, (KWF ? 3 : 1) * Ns * 16, 128), dBlo = dBhi + (Bb >> 4);
      for (int s = 0; s < S; ++s) {
        const int slot = s % NST;
        tc::mbar_wait(&full[slot], (uint32_t)((s / NST) & 1));
        tc::fence_after();
        if (BF) tc::fence_proxy_async();
        const uint64_t boff = (uint64_t)slot * (Sb >> 4);
        if (KWF) {
          // TMA windows start `pre` rows into their first padded line
          int pre = 0;
          if (a.tma) {
            const int sg = s_lo + s, kdi = sg / a.n_cb;
            const int uws = u0 + (kdi - 1) * a.Sh - a.Sw - 1;
            pre = uws - (uws / a.Sw) * a.Sw;
          }
          // one N = 3 Ns MMA per (kh, K step): B = the kh row's three kw taps side by side
          for (int kh = 0; kh < 3; ++kh) {
#pragma unroll
            for (int j = 0; j < NKC / 2; ++j) {
              const uint64_t bo = boff + (uint64_t)((kh * NKC + 2 * j) * 3 * Ns);
              const uint32_t first = (s | kh | j) ? 1u : 0u;
#pragma unroll
              for (int tt = 0; tt < T; ++tt) {
                const uint64_t ao = boff + (uint64_t)(2 * j * WRp + pre + kh * a.Sw + tt * RS);
                const uint32_t d = tmem + (uint32_t)(tt * 3 * Ns);
                if (B3) {
                  tc::mma_f16(d, dAlo + ao, dBhi + bo, a.idesc, first);
                  tc::mma_f16(d, dAhi + ao, dBlo + bo, a.idesc, 1u);
                  tc::mma_f16(d, dAhi + ao, dBhi + bo, a.idesc, 1u);
                } else if (BF) {
                  tc::mma_f16(d, dAhi + ao, dBhi + bo, a.idesc, first);
                } else {
                  tc::mma_tf32(d, dAlo + ao, dBhi + bo, a.idesc, first);
                  tc::mma_tf32(d, dAhi + ao, dBlo + bo, a.idesc, 1u);
                  tc::mma_tf32(d, dAhi + ao, dBhi + bo, a.idesc, 1u);
                }
              }
            }
          }
          tc::commit(&empty[slot]);
          continue;
        }
        for (int tq = 0; tq < ntap; ++tq) {
          const int t9 = tap9(tq);
          const int rowoff = PW ? 0 : (t9 >= 6 ? 2 : t9 >= 3 ? 1 : 0) * a.Sw + (t9 % 3);
#pragma unroll
          for (int j = 0; j < NKC / 2; ++j) {
            const uint64_t bo = boff + (uint64_t)((tq * NKC + 2 * j) * Ns);
            const uint32_t first = (s | tq | j) ? 1u : 0u;
#pragma unroll
            for (int tt = 0; tt < T; ++tt) {  // sub-tile tt: rows + 128 tt, accumulator columns + tt Ns
              const uint64_t ao = boff + (uint64_t)(2 * j * WRp + rowoff + tt * kTcRows);
              const uint32_t d = tmem + (uint32_t)(tt * Ns);
              if (B3) {
                tc::mma_f16(d, dAlo + ao, dBhi + bo, a.idesc, first);
                tc::mma_f16(d, dAhi + ao, dBlo + bo, a.idesc, 1u);
                tc::mma_f16(d, dAhi + ao, dBhi + bo, a.idesc, 1u);
              } else if (BF) {
                tc::mma_f16(d, dAhi + ao, dBhi + bo, a.idesc, first);
              } else {
                tc::mma_tf32(d, dAlo + ao, dBhi + bo, a.idesc, first);
                tc::mma_tf32(d, dAhi + ao, dBlo + bo, a.idesc, 1u);
                tc::mma_tf32(d, dAhi + ao, dBhi + bo, a.idesc, 1u);
              }
            }
          }
        }
        tc::commit(&empty[slot]);
      }
      if (S > 0) tc::commit(done);
    }
  } else {
    // ---- producers: PG groups fill alternate stages; a thread copies and splits
    // the same 16-byte elements
    constexpr int GT = kTcProd / PG;
    const int pg = PG == 2 ? (warp - 1) >> 2 : 0, gtid = tid - 32 - pg * GT;
    // 3xTF32, one producer group: software-pipelined ring. The copies of stage s + NST - 1 are
    // issued before the landing of stage s + 1 is waited for (cp.async groups retire in order:
    // wait_group NST - 2), so the L2 latency of a fill overlaps the lo split of the stage before
    // it and the MMAs of the stage before that, instead of being paid once per stage. A thread
    // copies and splits the same 16-byte elements, so no cross-thread sync sits between them.
    if (!BF && PG == 1 && !a.tma && a.dbg == 0) {
      const int gwarp = gtid >> 5;
      auto fill = [&](int s) {
        const int slot = s % NST;
        if (s >= NST) tc::mbar_wait(&empty[slot], (uint32_t)(((s / NST) - 1) & 1));
        const int sg = s_lo + s;
        const int kdi = sg / a.n_cb, cb = sg - kdi * a.n_cb;
        const int kd = PW ? 0 : t0 + kdi;
        const int* rm = rowmap + kd * WR;
        uint8_t* A = smem + slot * Sb;
        const long long plane = (long long)x.h * x.w;
        const float* xc = xb + cb * CB;
        // four row-map entries, then four copies: the loads are independent of the asm copies
        for (int i0 = gtid; i0 < nA; i0 += 4 * GT) {
          int off[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int i = i0 + q * GT;
            off[q] = i < nA ? rm[i / NKC] : -2;
          }
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int i = i0 + q * GT;
            if (off[q] == -2) continue;
            const int r = i / NKC, kc = i % NKC;
            const float* src = xb;
            bool ok = off[q] >= 0;
            if (MODE == 1) {
              // parity gather: virtual channel c = p * C_x + ci reads input voxel 2o + p
              const int c = cb * CB + 4 * kc, p = c / x.c, ci = c - p * x.c;
              const int pd = p >> 2, ph = (p >> 1) & 1, pw = p & 1;
              ok = ok && (!pd || (off[q] & 4)) && (!ph || (off[q] & 2)) && (!pw || (off[q] & 1));
              if (ok) src = xb + ((off[q] >> 3) + pd * plane + ph * x.w + pw) * (long long)x.cstride + ci;
            } else if (ok) {
              src = xc + (long long)off[q] * x.cstride + 4 * kc;
            }
            tc::cp_async16(A + ((size_t)kc * WRp + r) * 16, src, ok ? 16u : 0u);
          }
        }
        uint8_t* Bt = A + NH * Ab;
        if (KWF) {
          const float* wkd = wpb + (long long)(kd * 3) * kc_all * 3 * a.Np * 4;
          if (Ns == a.Np) {
            if (gtid == 0) {
              const uint32_t run = (uint32_t)NKC * 3 * Ns * 16;
              tc::mbar_expect_tx_only(&full[slot], 3 * NH * run);
              for (int kh = 0; kh < 3; ++kh) {
                const float* src = wkd + ((long long)kh * kc_all + cb * NKC) * 3 * a.Np * 4;
                tc::bulk_load(Bt + (size_t)kh * run, src, run, &full[slot]);
                tc::bulk_load(Bt + Bb + (size_t)kh * run, src + a.wlo, run, &full[slot]);
              }
            }
          } else {
            for (int q = gwarp; q < 9 * NKC; q += GT / 32) {  // q = (kh, kcl, kw)
              const int kw = q % 3, kcl = (q / 3) % NKC, kh = q / (3 * NKC);
              const float* src = wkd + ((((long long)kh * kc_all + cb * NKC + kcl) * 3 + kw) * a.Np + n0) * 4;
              uint8_t* dst = Bt + ((size_t)(kh * NKC + kcl) * 3 * Ns + kw * Ns) * 16;
              for (int n = lane; n < Ns; n += 32) {
                tc::cp_async16(dst + n * 16, src + n * 4, 16u);
                tc::cp_async16(dst + Bb + n * 16, src + a.wlo + n * 4, 16u);
              }
            }
          }
        } else {
          const float* wk = wpb + ((long long)(kd * 9) * kc_all + cb * NKC) * a.Np * 4 + (long long)n0 * 4;
          for (int q = gwarp; q < ntap * NKC; q += GT / 32) {
            const int tq = q / NKC, kcl = q % NKC;
            const int t9 = PW ? 0 : tap9(tq);
            const float* src = wk + ((long long)t9 * kc_all + kcl) * a.Np * 4;
            uint8_t* dst = Bt + (size_t)q * Ns * 16;
            for (int n = lane; n < Ns; n += 32) {
              tc::cp_async16(dst + n * 16, src + n * 4, 16u);
              tc::cp_async16(dst + Bb + n * 16, src + a.wlo + n * 4, 16u);
            }
          }
        }
        tc::cp_async_commit();
      };
      const int LA = NST - 1;  // stages in flight ahead of the one being split
      for (int s = 0; s < LA && s < S; ++s) fill(s);
      for (int s = 0; s < S; ++s) {
        if (LA >= 2 && s + 1 < S)
          tc::cp_async_wait<1>();
        else
          tc::cp_async_wait<0>();
        // lo half of the landed activation window; the raw fp32 window is the hi operand
        // (the tensor core truncates fp32 to TF32: tools/tf32_round_probe.cu)
        const int slot = s % NST;
        uint8_t* A = smem + slot * Sb;
        for (int i0 = gtid; i0 < nA; i0 += 4 * GT) {
          float4 v[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int i = i0 + q * GT;
            if (i < nA) v[q] = *reinterpret_cast<const float4*>(A + ((size_t)(i % NKC) * WRp + i / NKC) * 16);
          }
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int i = i0 + q * GT;
            if (i >= nA) continue;
            float4 l;
            l.x = v[q].x - tf32_hi(v[q].x); l.y = v[q].y - tf32_hi(v[q].y);
            l.z = v[q].z - tf32_hi(v[q].z); l.w = v[q].w - tf32_hi(v[q].w);
            *reinterpret_cast<float4*>(A + Ab + ((size_t)(i % NKC) * WRp + i / NKC) * 16) = l;
          }
        }
        tc::fence_proxy_async();
        tc::mbar_arrive(&full[slot]);
        if (s + LA < S) fill(s + LA);
      }
    } else
    for (int s = pg; s < S; s += PG) {
      const int slot = s % NST;
      if (s >= NST) tc::mbar_wait(&empty[slot], (uint32_t)(((s / NST) - 1) & 1));
      if (a.dbg == 1) {  // D2IP_TC_DBG=1: no fills (measures the MMA side alone; wrong results)
        tc::mbar_arrive(&full[slot]);
        continue;
      }
      const int sg = s_lo + s;
      const int kdi = sg / a.n_cb, cb = sg - kdi * a.n_cb;
      const int kd = PW ? 0 : t0 + kdi;
      const int* rm = rowmap + kd * WR;
      uint8_t* A = smem + slot * Sb;
      if (KWF && !BF && a.tma) {
        // TMA-staged window: warp 1 issues one 5-D box (4 channels x Sw columns from w = -1, one
        // padded line) per (line, 16-byte channel chunk) -- the zero halo is the boxes'
        // out-of-bounds fill -- and the weight tile as three bulk runs per operand half, all
        // completing on landed[slot] by byte count; then every producer thread forms the lo
        // half of its share of the landed window (x - tf32(x)) and arrives on full[slot]
        const int uws = u0 + (kdi - 1) * a.Sh - a.Sw - 1;
        const int L0 = uws / a.Sw, pre = uws - L0 * a.Sw;
        const int nl = (pre + WR + a.Sw - 1) / a.Sw;
        const int Hl = a.gh + 2;
        const int lrows = nl * a.Sw;
        uint8_t* Bt = A + NH * Ab;
        const uint32_t run = (uint32_t)NKC * 3 * Ns * 16;
        if (warp == 1) {
          if (lane == 0) tc::mbar_expect_tx(&landed[slot], (uint32_t)(NKC * lrows * 16) + 3 * NH * run);
          __syncwarp();
          for (int i = lane; i < NKC * nl; i += 32) {
            const int kc = i / nl, li = i - kc * nl;
            const int L = L0 + li, dp = L / Hl, hp = L - dp * Hl;
            tc::tma_load_5d(A + ((size_t)kc * WRp + (size_t)li * a.Sw) * 16, &tmap, cb * CB + 4 * kc, -1, hp - 1,
                            dp - 1, b, &landed[slot]);
          }
          if (lane == 0) {
            const float* wkd = wpb + (long long)(kd * 3) * kc_all * 3 * a.Np * 4;
            for (int kh = 0; kh < 3; ++kh) {
              const float* src = wkd + ((long long)kh * kc_all + cb * NKC) * 3 * a.Np * 4;
              tc::bulk_load(Bt + (size_t)kh * run, src, run, &landed[slot]);
              tc::bulk_load(Bt + Bb + (size_t)kh * run, src + a.wlo, run, &landed[slot]);
            }
          }
        }
        tc::mbar_wait(&landed[slot], (uint32_t)((s / NST) & 1));
        for (int i = gtid; i < NKC * lrows; i += GT) {
          const int kc = i / lrows, r = i - kc * lrows;
          const float4 v = *reinterpret_cast<const float4*>(A + ((size_t)kc * WRp + r) * 16);
          float4 l;
          l.x = v.x - tf32_hi(v.x); l.y = v.y - tf32_hi(v.y); l.z = v.z - tf32_hi(v.z); l.w = v.w - tf32_hi(v.w);
          *reinterpret_cast<float4*>(A + Ab + ((size_t)kc * WRp + r) * 16) = l;
        }
        tc::fence_proxy_async();
        tc::mbar_arrive(&full[slot]);
        continue;
      }
      if (BF && !B3 && a.xtw) {
        // bf16 twin of x: one 16-byte async copy per (row, 8-channel chunk); zero-fill for padding rows
        const uint16_t* xt = reinterpret_cast<const uint16_t*>(x.bf16) + b * x.bstride;
        const long long plane = (long long)x.h * x.w;
        for (int i = gtid; i < nA; i += GT) {
          const int r = i / NKC, kc = i % NKC;
          const int off = rm[r];
          const uint16_t* src = nullptr;
          if (MODE == 1) {
            const int c = cb * CB + 8 * kc, p = c / x.c, ci = c - p * x.c;
            const int pd = p >> 2, ph = (p >> 1) & 1, pw = p & 1;
            if (off >= 0 && (!pd || (off & 4)) && (!ph || (off & 2)) && (!pw || (off & 1)))
              src = xt + ((off >> 3) + pd * plane + ph * x.w + pw) * (long long)x.cstride + ci;
          } else if (off >= 0) {
            src = xt + (long long)off * x.cstride + cb * CB + 8 * kc;
          }
          tc::cp_async16(A + ((size_t)kc * WRp + r) * 16, src ? src : xt, src ? 16u : 0u);
        }
      } else if (BF) {
        // fp32 window -> registers -> bf16 rows. A work item is one float4 (4
        // channels; consecutive threads read consecutive 16 B of a voxel row) that
        // lands as 8 bytes, half of a 16-byte chunk; eight loads in flight per thread.
        constexpr int PPR = 2 * NKC;  // float4 pieces per window row
        const int nP = WR * PPR;
        const long long plane = (long long)x.h * x.w;
        for (int i0 = gtid; i0 < nP; i0 += 8 * GT) {
          float4 v[8];
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const int i = i0 + q * GT;
            v[q] = make_float4(0.f, 0.f, 0.f, 0.f);
            if (i >= nP) continue;
            const int r = i / PPR, pc = i % PPR;
            const int off = rm[r];
            if (MODE == 1) {
              const int c = cb * CB + 4 * pc, p = c / x.c, ci = c - p * x.c;
              const int pd = p >> 2, ph = (p >> 1) & 1, pw = p & 1;
              if (off >= 0 && (!pd || (off & 4)) && (!ph || (off & 2)) && (!pw || (off & 1)))
                v[q] = *reinterpret_cast<const float4*>(
                    xb + ((off >> 3) + pd * plane + ph * x.w + pw) * (long long)x.cstride + ci);
            } else if (off >= 0) {
              v[q] = *reinterpret_cast<const float4*>(xb + (long long)off * x.cstride + cb * CB + 4 * pc);
            }
          }
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const int i = i0 + q * GT;
            if (i >= nP) continue;
            const int r = i / PPR, pc = i % PPR;
            uint2 o;
            o.x = bf2(v[q].x, v[q].y);
            o.y = bf2(v[q].z, v[q].w);
            *reinterpret_cast<uint2*>(A + ((size_t)(pc >> 1) * WRp + r) * 16 + (pc & 1) * 8) = o;
            if (B3) {  // lo = bf16(x - hi)
              const float2 h0 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&o.x));
              const float2 h1 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&o.y));
              const uint2 l = make_uint2(bf2(v[q].x - h0.x, v[q].y - h0.y), bf2(v[q].z - h1.x, v[q].w - h1.y));
              *reinterpret_cast<uint2*>(A + Ab + ((size_t)(pc >> 1) * WRp + r) * 16 + (pc & 1) * 8) = l;
            }
          }
        }
      } else if (MODE == 1) {
        // parity gather: virtual channel c = p * C_x + ci reads input voxel 2o + p
        const long long plane = (long long)x.h * x.w;
        for (int i = gtid; i < nA; i += GT) {
          const int r = i / NKC, kc = i % NKC;
          const int off = rm[r];
          const int c = cb * CB + 4 * kc, p = c / x.c, ci = c - p * x.c;
          const int pd = p >> 2, ph = (p >> 1) & 1, pw = p & 1;
          const bool ok = off >= 0 && (!pd || (off & 4)) && (!ph || (off & 2)) && (!pw || (off & 1));
          const float* src =
              ok ? xb + ((off >> 3) + pd * plane + ph * x.w + pw) * (long long)x.cstride + ci : xb;
          tc::cp_async16(A + ((size_t)kc * WRp + r) * 16, src, ok ? 16u : 0u);
        }
      } else {
        const float* xc = xb + cb * CB;
        for (int i = gtid; i < nA; i += GT) {
          const int r = i / NKC, kc = i % NKC;
          const int off = rm[r];
          const float* src = off >= 0 ? xc + (long long)off * x.cstride + 4 * kc : xb;
          tc::cp_async16(A + ((size_t)kc * WRp + r) * 16, src, off >= 0 ? 16u : 0u);
        }
      }
      // B: nt^2 taps x NKC chunks, each a contiguous run of Ns 16-byte rows; one warp per run
      // (16-byte rows: 4 floats, or 8 bf16 = 4 float slots of the pack buffer)
      uint8_t* Bt = A + NH * Ab;
      const int gwarp = gtid >> 5;
      if (KWF) {
        // kw-folded layout [kd kh][K/4][kw][Np][4]: per kh the stage's B tile is NKC x 3 x Np
        // contiguous 16-byte rows. One slice of all N: three bulk copies per operand half,
        // completing on the stage barrier by byte count; else 16-byte async copies per row
        const float* wkd = wpb + (long long)(kd * 3) * kc_all * 3 * a.Np * 4;
        if (Ns == a.Np) {
          if (gtid == 0) {
            const uint32_t run = (uint32_t)NKC * 3 * Ns * 16;
            tc::mbar_expect_tx_only(&full[slot], 3 * NH * run);
            for (int kh = 0; kh < 3; ++kh) {
              const float* src = wkd + ((long long)kh * kc_all + cb * NKC) * 3 * a.Np * 4;
              tc::bulk_load(Bt + (size_t)kh * run, src, run, &full[slot]);
              if (NH == 2) tc::bulk_load(Bt + Bb + (size_t)kh * run, src + a.wlo, run, &full[slot]);
            }
          }
        } else {
          for (int q = gwarp; q < 9 * NKC; q += GT / 32) {  // q = (kh, kcl, kw)
            const int kw = q % 3, kcl = (q / 3) % NKC, kh = q / (3 * NKC);
            const float* src = wkd + ((((long long)kh * kc_all + cb * NKC + kcl) * 3 + kw) * a.Np + n0) * 4;
            uint8_t* dst = Bt + ((size_t)(kh * NKC + kcl) * 3 * Ns + kw * Ns) * 16;
            for (int n = lane; n < Ns; n += 32) {
              tc::cp_async16(dst + n * 16, src + n * 4, 16u);
              if (NH == 2) tc::cp_async16(dst + Bb + n * 16, src + a.wlo + n * 4, 16u);
            }
          }
        }
      }
      const float* wk = wpb + ((long long)(kd * 9) * kc_all + cb * NKC) * a.Np * 4 + (long long)n0 * 4;
      for (int q = gwarp; q < (KWF ? 0 : ntap * NKC); q += GT / 32) {
        const int tq = q / NKC, kcl = q % NKC;
        const int t9 = PW ? 0 : tap9(tq);
        const float* src = wk + ((long long)t9 * kc_all + kcl) * a.Np * 4;
        uint8_t* dst = Bt + (size_t)q * Ns * 16;
        for (int n = lane; n < Ns; n += 32) {
          tc::cp_async16(dst + n * 16, src + n * 4, 16u);
          if (NH == 2) tc::cp_async16(dst + Bb + n * 16, src + a.wlo + n * 4, 16u);
        }
      }
      if (BF && !B3 && a.xtw && a.async_arrive) {
        // every operand of the stage is an async copy: arrive when this thread's copies
        // land (no wait here -- the next stage's copies are issued while these fly);
        // the MMA thread's proxy fence makes them visible to the tensor core
        asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(tc::smem_u32(&full[slot]))
                     : "memory");
        continue;
      }
      if (!BF && a.dbg == 2) {  // D2IP_TC_DBG=2 (study only, wrong results): no lo split, async arrive
        asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(tc::smem_u32(&full[slot]))
                     : "memory");
        continue;
      }
      tc::cp_async_commit();
      tc::cp_async_wait<0>();
      // lo half of the landed activation window; the raw fp32 window is the hi
      // operand (the tensor core truncates fp32 to TF32: tools/tf32_round_probe.cu)
      if (!BF)
      for (int i = gtid; i < nA; i += GT) {
        const int r = i / NKC, kc = i % NKC;
        const float4 v = *reinterpret_cast<const float4*>(A + ((size_t)kc * WRp + r) * 16);
        float4 l;
        l.x = v.x - tf32_hi(v.x); l.y = v.y - tf32_hi(v.y); l.z = v.z - tf32_hi(v.z); l.w = v.w - tf32_hi(v.w);
        *reinterpret_cast<float4*>(A + Ab + ((size_t)kc * WRp + r) * 16) = l;
      }
      tc::fence_proxy_async();
      tc::mbar_arrive(&full[slot]);
    }

    // ---- epilogue (producer warps): TMEM lane = GEMM row; warp w reads lane
    // quadrant w % 4 and column half (w - 1) / 4; one row / voxel per sub-tile
    if (S > 0) {
      tc::mbar_wait(done, 0);
      tc::fence_after();
    }
    if (KWF)
      tc_epilogue_kwf<T>(a, tmem, b, n0, u0, ks, S, warp, lane, reinterpret_cast<float*>(smem));
    else
      tc_epilogue<T, MODE>(a, tmem, b, n0, u0, ks, S, warp, lane);
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_free(tmem, a.tmem_cols);
}

// Persistent variant for large grids (split-K off): a CTA walks tiles blockIdx.x, +gridDim.x, ...;
// warp 0 issues MMAs into one of two TMEM accumulators, warps 1-8 compute each tile's row map
// and fill the stage ring (its counter runs across tiles), warps 9-12 drain the other
// accumulator -- the epilogue and the next tile's prologue overlap the MMAs instead of
// serialising with them (one-tile CTAs spent ~2.6x the operand-bound MMA time there).
template <int NKC, int T, int MODE, int BFM>
__global__ void __launch_bounds__(kTcpThreads) conv_tcp_k(TcConv a) {
  constexpr int PG = 1;
  constexpr bool BF = BFM != 0, B3 = BFM == 2;
  D2IP_PDL_ENTRY();
  extern __shared__ __align__(1024) uint8_t smem[];
  constexpr int CB = NKC * (BF ? 8 : 4);
  constexpr int NH = BFM == 1 ? 1 : 2;  // operand halves per stage (3xTF32 / 3xbf16: hi, lo)
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int b = blockIdx.z;
  const int ks = blockIdx.y % a.kspl;
  const int n0 = (blockIdx.y / a.kspl) * a.Ns;  // first output channel of this CTA's slice
  const int Ns = a.Ns, WR = a.WR, WRp = a.WRp;
  constexpr bool PW = MODE == 3;  // 1^3: one tap, window = the tile rows
  constexpr bool KWF = MODE == 4;  // stride 1, the three kw taps folded into N (3 column blocks)
  constexpr int RS = KWF ? kTcRows - 2 : kTcRows;  // output rows per 128-row sub-tile
  constexpr int nt = PW ? 1 : (MODE == 1 || MODE == 2) ? 2 : 3, t0 = MODE == 2 ? 1 : 0, ntap = nt * nt;
  // (kh, kw) of the q-th live tap as a 3x3 index: nt = 3 -> q; nt = 2 -> the 2x2 block at (t0, t0)
  auto tap9 = [&](int q) { return nt == 3 ? q : (t0 + (q >> 1)) * 3 + (t0 + (q & 1)); };
  const int u0 = a.u_first + blockIdx.x * T * RS;
  const uint32_t Ab = (uint32_t)NKC * WRp * 16, Bb = (uint32_t)ntap * NKC * Ns * 16;
  const uint32_t Sb = NH * (Ab + Bb);
  // layout: 2 stages of [A hi][A lo][B hi][B lo] (bf16: [A][B]), row map, barriers full[2] empty[2] done, TMEM slot
  const int NST = a.nst;  // ring depth (2 or 3 stages)
  int* rowmap2 = reinterpret_cast<int*>(smem + NST * Sb);  // [2][3 WR]: tile parity
  uint64_t* full = reinterpret_cast<uint64_t*>(rowmap2 + 6 * WR);
  uint64_t* empty = full + 3;
  uint64_t* tfull = empty + 3;  // [2]: accumulator ready (MMA -> epilogue)
  uint64_t* tempty = tfull + 2; // [2]: accumulator drained (epilogue -> MMA)
  uint32_t* tslot = reinterpret_cast<uint32_t*>(tempty + 2);
  const int nct = (a.ntiles - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x;  // this CTA's tiles

  if (warp == 0) tc::tmem_alloc(tslot, a.tmem_cols);
  if (tid == 0) {
    for (int i = 0; i < NST; ++i) {
      tc::mbar_init(&full[i], kTcProd);  // producer warps 1-8
      tc::mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(&tfull[i], 1);
      tc::mbar_init(&tempty[i], 4);  // one arrival per epilogue warp
    }
    tc::fence_mbar_init();
  }
  const d2ip_act x = a.x;
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = *tslot;
  const float* xb = x.ptr + b * x.bstride;
  const float* wpb = a.wp + b * a.wpbs;
  const int S_all = nt * a.n_cb;
  const int s_lo = (int)((long long)ks * S_all / a.kspl), s_hi = (int)((long long)(ks + 1) * S_all / a.kspl);
  const int S = s_hi - s_lo;  // this CTA's stages: s_lo + [0, S)
  const int nA = WR * NKC;
  const int kc_all = BF ? a.Kc >> 3 : a.Kc >> 2;  // 16-byte chunks per K

  if (warp == 0) {
    // ---- MMA issue (one elected thread); stage s lives in slot s & 1
    if (lane == 0) {
      // descriptors of slot 0; a tap / K step / slot is an add to the 14-bit
      // start-address field (smem addresses < 256 KB never carry out of it)
      const uint32_t sbase = tc::smem_u32(smem);
      const uint64_t dAhi = tc::make_desc(sbase, WRp * 16, 128), dAlo = dAhi + (Ab >> 4);
      const uint64_t dBhi = tc::make_desc(sbase + NH * Ab, Ns * 16, 128), dBlo = dBhi + (Bb >> 4);
      int g = 0;  // stage counter across tiles
      for (int it = 0; it < nct; ++it) {
      const int acc = it & 1;
      if (it >= 2) tc::mbar_wait(&tempty[acc], (uint32_t)(((it >> 1) - 1) & 1));
      tc::fence_after();
      const uint32_t tacc = tmem + (uint32_t)(acc * T * Ns);
      for (int s = 0; s < S; ++s, ++g) {
        const int slot = g % NST;
        tc::mbar_wait(&full[slot], (uint32_t)((g / NST) & 1));
        tc::fence_after();
        if (BF) tc::fence_proxy_async();
        const uint64_t boff = (uint64_t)slot * (Sb >> 4);
        for (int tq = 0; tq < ntap; ++tq) {
          const int t9 = tap9(tq);
          const int rowoff = PW ? 0 : (t9 >= 6 ? 2 : t9 >= 3 ? 1 : 0) * a.Sw + (t9 % 3);
#pragma unroll
          for (int j = 0; j < NKC / 2; ++j) {
            const uint64_t bo = boff + (uint64_t)((tq * NKC + 2 * j) * Ns);
            const uint32_t first = (s | tq | j) ? 1u : 0u;
#pragma unroll
            for (int tt = 0; tt < T; ++tt) {  // sub-tile tt: rows + 128 tt, accumulator columns + tt Ns
              const uint64_t ao = boff + (uint64_t)(2 * j * WRp + rowoff + tt * kTcRows);
              const uint32_t d = tacc + (uint32_t)(tt * Ns);
              if (B3) {
                tc::mma_f16(d, dAlo + ao, dBhi + bo, a.idesc, first);
                tc::mma_f16(d, dAhi + ao, dBlo + bo, a.idesc, 1u);
                tc::mma_f16(d, dAhi + ao, dBhi + bo, a.idesc, 1u);
              } else if (BF) {
                tc::mma_f16(d, dAhi + ao, dBhi + bo, a.idesc, first);
              } else {
                tc::mma_tf32(d, dAlo + ao, dBhi + bo, a.idesc, first);
                tc::mma_tf32(d, dAhi + ao, dBlo + bo, a.idesc, 1u);
                tc::mma_tf32(d, dAhi + ao, dBhi + bo, a.idesc, 1u);
              }
            }
          }
        }
        tc::commit(&empty[slot]);
      }
      tc::commit(&tfull[acc]);
      }
    }
  } else if (warp <= 8) {
    // ---- producers (warps 1-8): per tile its row map, then its stages
    constexpr int GT = kTcProd;
    const int gtid = tid - 32;
    int g = 0;
    for (int it = 0; it < nct; ++it) {
    const int u0 = a.u_first + ((int)blockIdx.x + it * (int)gridDim.x) * T * kTcRows;
    int* rowmap = rowmap2 + (it & 1) * 3 * WR;
    for (int i = gtid; i < (PW ? WR : 3 * WR); i += GT) {
      const int kd = i / WR, r = i - kd * WR;
      const int u = PW ? u0 + r : u0 + (kd - 1) * a.Sh - a.Sw - 1 + r;
      int off = -1;
      if (u >= 0) {
        const int dp = u / a.Sh, rem = u - dp * a.Sh;
        const int hp = rem / a.Sw, wp = rem - hp * a.Sw;
        if (dp >= 1 && dp <= a.gd && hp >= 1 && hp <= a.gh && wp >= 1 && wp <= a.gw)
          off = ((dp - 1) * a.gh + (hp - 1)) * a.gw + (wp - 1);
      }
      rowmap[i] = off;
    }
    asm volatile("bar.sync 1, 256;" ::: "memory");
    for (int s = 0; s < S; ++s, ++g) {
      const int slot = g % NST;
      if (g >= NST) tc::mbar_wait(&empty[slot], (uint32_t)(((g / NST) - 1) & 1));
      if (a.dbg) {  // D2IP_TC_DBG=1: no fills (measures the MMA side alone; wrong results)
        tc::mbar_arrive(&full[slot]);
        continue;
      }
      const int sg = s_lo + s;
      const int kdi = sg / a.n_cb, cb = sg - kdi * a.n_cb;
      const int kd = PW ? 0 : t0 + kdi;
      const int* rm = rowmap + kd * WR;
      uint8_t* A = smem + slot * Sb;
      if (BF && !B3 && a.xtw) {
        // bf16 twin of x: one 16-byte async copy per (row, 8-channel chunk); zero-fill for padding rows
        const uint16_t* xt = reinterpret_cast<const uint16_t*>(x.bf16) + b * x.bstride;
        const long long plane = (long long)x.h * x.w;
        for (int i = gtid; i < nA; i += GT) {
          const int r = i / NKC, kc = i % NKC;
          const int off = rm[r];
          const uint16_t* src = nullptr;
          if (MODE == 1) {
            const int c = cb * CB + 8 * kc, p = c / x.c, ci = c - p * x.c;
            const int pd = p >> 2, ph = (p >> 1) & 1, pw = p & 1;
            if (off >= 0 && (!pd || (off & 4)) && (!ph || (off & 2)) && (!pw || (off & 1)))
              src = xt + ((off >> 3) + pd * plane + ph * x.w + pw) * (long long)x.cstride + ci;
          } else if (off >= 0) {
            src = xt + (long long)off * x.cstride + cb * CB + 8 * kc;
          }
          tc::cp_async16(A + ((size_t)kc * WRp + r) * 16, src ? src : xt, src ? 16u : 0u);
        }
      } else if (BF) {
        // fp32 window -> registers -> bf16 rows. A work item is one float4 (4
        // channels; consecutive threads read consecutive 16 B of a voxel row) that
        // lands as 8 bytes, half of a 16-byte chunk; eight loads in flight per thread.
        constexpr int PPR = 2 * NKC;  // float4 pieces per window row
        const int nP = WR * PPR;
        const long long plane = (long long)x.h * x.w;
        for (int i0 = gtid; i0 < nP; i0 += 8 * GT) {
          float4 v[8];
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const int i = i0 + q * GT;
            v[q] = make_float4(0.f, 0.f, 0.f, 0.f);
            if (i >= nP) continue;
            const int r = i / PPR, pc = i % PPR;
            const int off = rm[r];
            if (MODE == 1) {
              const int c = cb * CB + 4 * pc, p = c / x.c, ci = c - p * x.c;
              const int pd = p >> 2, ph = (p >> 1) & 1, pw = p & 1;
              if (off >= 0 && (!pd || (off & 4)) && (!ph || (off & 2)) && (!pw || (off & 1)))
                v[q] = *reinterpret_cast<const float4*>(
                    xb + ((off >> 3) + pd * plane + ph * x.w + pw) * (long long)x.cstride + ci);
            } else if (off >= 0) {
              v[q] = *reinterpret_cast<const float4*>(xb + (long long)off * x.cstride + cb * CB + 4 * pc);
            }
          }
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const int i = i0 + q * GT;
            if (i >= nP) continue;
            const int r = i / PPR, pc = i % PPR;
            uint2 o;
            o.x = bf2(v[q].x, v[q].y);
            o.y = bf2(v[q].z, v[q].w);
            *reinterpret_cast<uint2*>(A + ((size_t)(pc >> 1) * WRp + r) * 16 + (pc & 1) * 8) = o;
            if (B3) {  // lo = bf16(x - hi)
              const float2 h0 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&o.x));
              const float2 h1 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&o.y));
              const uint2 l = make_uint2(bf2(v[q].x - h0.x, v[q].y - h0.y), bf2(v[q].z - h1.x, v[q].w - h1.y));
              *reinterpret_cast<uint2*>(A + Ab + ((size_t)(pc >> 1) * WRp + r) * 16 + (pc & 1) * 8) = l;
            }
          }
        }
      } else if (MODE == 1) {
        // parity gather: virtual channel c = p * C_x + ci reads input voxel 2o + p
        const long long plane = (long long)x.h * x.w;
        for (int i = gtid; i < nA; i += GT) {
          const int r = i / NKC, kc = i % NKC;
          const int off = rm[r];
          const int c = cb * CB + 4 * kc, p = c / x.c, ci = c - p * x.c;
          const int pd = p >> 2, ph = (p >> 1) & 1, pw = p & 1;
          const bool ok = off >= 0 && (!pd || (off & 4)) && (!ph || (off & 2)) && (!pw || (off & 1));
          const float* src =
              ok ? xb + ((off >> 3) + pd * plane + ph * x.w + pw) * (long long)x.cstride + ci : xb;
          tc::cp_async16(A + ((size_t)kc * WRp + r) * 16, src, ok ? 16u : 0u);
        }
      } else {
        const float* xc = xb + cb * CB;
        for (int i = gtid; i < nA; i += GT) {
          const int r = i / NKC, kc = i % NKC;
          const int off = rm[r];
          const float* src = off >= 0 ? xc + (long long)off * x.cstride + 4 * kc : xb;
          tc::cp_async16(A + ((size_t)kc * WRp + r) * 16, src, off >= 0 ? 16u : 0u);
        }
      }
      // B: nt^2 taps x NKC chunks, each a contiguous run of Ns 16-byte rows; one warp per run
      // (16-byte rows: 4 floats, or 8 bf16 = 4 float slots of the pack buffer)
      uint8_t* Bt = A + NH * Ab;
      const int gwarp = gtid >> 5;
      if (KWF) {
        // kw-folded layout [kd kh][K/4][kw][Np][4]: per kh the stage's B tile is NKC x 3 x Np
        // contiguous 16-byte rows. One slice of all N: three bulk copies per operand half,
        // completing on the stage barrier by byte count; else 16-byte async copies per row
        const float* wkd = wpb + (long long)(kd * 3) * kc_all * 3 * a.Np * 4;
        if (Ns == a.Np) {
          if (gtid == 0) {
            const uint32_t run = (uint32_t)NKC * 3 * Ns * 16;
            tc::mbar_expect_tx_only(&full[slot], 3 * NH * run);
            for (int kh = 0; kh < 3; ++kh) {
              const float* src = wkd + ((long long)kh * kc_all + cb * NKC) * 3 * a.Np * 4;
              tc::bulk_load(Bt + (size_t)kh * run, src, run, &full[slot]);
              if (NH == 2) tc::bulk_load(Bt + Bb + (size_t)kh * run, src + a.wlo, run, &full[slot]);
            }
          }
        } else {
          for (int q = gwarp; q < 9 * NKC; q += GT / 32) {  // q = (kh, kcl, kw)
            const int kw = q % 3, kcl = (q / 3) % NKC, kh = q / (3 * NKC);
            const float* src = wkd + ((((long long)kh * kc_all + cb * NKC + kcl) * 3 + kw) * a.Np + n0) * 4;
            uint8_t* dst = Bt + ((size_t)(kh * NKC + kcl) * 3 * Ns + kw * Ns) * 16;
            for (int n = lane; n < Ns; n += 32) {
              tc::cp_async16(dst + n * 16, src + n * 4, 16u);
              if (NH == 2) tc::cp_async16(dst + Bb + n * 16, src + a.wlo + n * 4, 16u);
            }
          }
        }
      }
      const float* wk = wpb + ((long long)(kd * 9) * kc_all + cb * NKC) * a.Np * 4 + (long long)n0 * 4;
      for (int q = gwarp; q < (KWF ? 0 : ntap * NKC); q += GT / 32) {
        const int tq = q / NKC, kcl = q % NKC;
        const int t9 = PW ? 0 : tap9(tq);
        const float* src = wk + ((long long)t9 * kc_all + kcl) * a.Np * 4;
        uint8_t* dst = Bt + (size_t)q * Ns * 16;
        for (int n = lane; n < Ns; n += 32) {
          tc::cp_async16(dst + n * 16, src + n * 4, 16u);
          if (NH == 2) tc::cp_async16(dst + Bb + n * 16, src + a.wlo + n * 4, 16u);
        }
      }
      if (BF && !B3 && a.xtw && a.async_arrive) {
        // every operand of the stage is an async copy: arrive when this thread's copies
        // land (no wait here -- the next stage's copies are issued while these fly);
        // the MMA thread's proxy fence makes them visible to the tensor core
        asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(tc::smem_u32(&full[slot]))
                     : "memory");
        continue;
      }
      tc::cp_async_commit();
      tc::cp_async_wait<0>();
      // lo half of the landed activation window; the raw fp32 window is the hi
      // operand (the tensor core truncates fp32 to TF32: tools/tf32_round_probe.cu)
      if (!BF)
      for (int i = gtid; i < nA; i += GT) {
        const int r = i / NKC, kc = i % NKC;
        const float4 v = *reinterpret_cast<const float4*>(A + ((size_t)kc * WRp + r) * 16);
        float4 l;
        l.x = v.x - tf32_hi(v.x); l.y = v.y - tf32_hi(v.y); l.z = v.z - tf32_hi(v.z); l.w = v.w - tf32_hi(v.w);
        *reinterpret_cast<float4*>(A + Ab + ((size_t)kc * WRp + r) * 16) = l;
      }
      tc::fence_proxy_async();
      tc::mbar_arrive(&full[slot]);
    }

    }  // tiles
  } else {
    // ---- epilogue (warps 9-12): one warp per TMEM lane quadrant, all columns
    for (int it = 0; it < nct; ++it) {
      const int acc = it & 1;
      const int u0 = a.u_first + ((int)blockIdx.x + it * (int)gridDim.x) * T * kTcRows;
      tc::mbar_wait(&tfull[acc], (uint32_t)((it >> 1) & 1));
      tc::fence_after();
      tc_epilogue<T, MODE>(a, tmem + (uint32_t)(acc * T * Ns), b, n0, u0, ks, S, warp, lane, 0, Ns);
      tc::fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&tempty[acc]);
    }
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_free(tmem, a.tmem_cols);
}


// TMA-fed bf16 variant (stride 1 and 1^3 layers whose input has a bf16 twin):
// one producer thread fetches each stage's activation window as whole padded
// lines -- a 5-D tensor-map box (8 channels, W + 2 columns starting at w = -1,
// one line, one plane, one sequence) per line and 8-channel chunk, the zero
// padding of the virtual grid coming from the box's out-of-bounds fill -- and
// the weight tiles as contiguous bulk copies, all completing on the stage's
// mbarrier by byte count. The MMA thread starts its descriptors `pre` rows
// into the first line. No per-row address work, no producer warps in the loop.
template <int NKC, int T, int MODE>
__global__ void __launch_bounds__(kTcThreads) conv_tma_k(const TcConv a, const __grid_constant__ CUtensorMap tmap) {
  D2IP_PDL_ENTRY();
  extern __shared__ __align__(1024) uint8_t smem[];
  constexpr int CB = NKC * 8;
  constexpr bool PW = MODE == 3;
  constexpr int nt = PW ? 1 : 3, ntap = nt * nt;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int b = blockIdx.z;
  const int ks = blockIdx.y % a.kspl;
  const int n0 = (blockIdx.y / a.kspl) * a.Ns;
  const int u0 = a.u_first + blockIdx.x * T * kTcRows;
  const int Ns = a.Ns, LR = a.lrows;
  const uint32_t Ab = (uint32_t)NKC * LR * 16, Bb = (uint32_t)ntap * NKC * Ns * 16;
  const uint32_t Sb = (Ab + Bb + 127) & ~127u;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + 2 * Sb);
  uint64_t* empty = full + 2;
  uint64_t* done = empty + 2;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(done + 1);
  if (warp == 0) tc::tmem_alloc(tslot, a.tmem_cols);
  if (tid == 0) {
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(&full[i], 1);
      tc::mbar_init(&empty[i], 1);
    }
    tc::mbar_init(done, 1);
    tc::fence_mbar_init();
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = *tslot;
  const int S_all = nt * a.n_cb;
  const int s_lo = (int)((long long)ks * S_all / a.kspl), s_hi = (int)((long long)(ks + 1) * S_all / a.kspl);
  const int S = s_hi - s_lo;
  const int Hl = a.gh + 2;  // padded lines per plane
  // first virtual row of a stage's window, its first padded line, and the row offset into it
  auto window = [&](int s, int* L0, int* pre, int* cb) {
    const int sg = s_lo + s, kdi = sg / a.n_cb;
    *cb = sg - kdi * a.n_cb;
    const int uws = PW ? u0 : u0 + (kdi - 1) * a.Sh - a.Sw - 1;
    *L0 = uws / a.Sw;
    *pre = uws - *L0 * a.Sw;
    return kdi;
  };
  if (warp == 0) {
    if (lane == 0) {
      const uint32_t sbase = tc::smem_u32(smem);
      const uint64_t dA = tc::make_desc(sbase, LR * 16, 128);
      const uint64_t dB = tc::make_desc(sbase + Ab, Ns * 16, 128);
      for (int s = 0; s < S; ++s) {
        const int slot = s & 1;
        int L0, pre, cb;
        window(s, &L0, &pre, &cb);
        tc::mbar_wait(&full[slot], (uint32_t)((s >> 1) & 1));
        tc::fence_after();
        const uint64_t so = slot ? (uint64_t)(Sb >> 4) : 0;
        for (int tq = 0; tq < ntap; ++tq) {
          const int rowoff = PW ? 0 : (tq / 3) * a.Sw + (tq % 3);
#pragma unroll
          for (int j = 0; j < NKC / 2; ++j) {
            const uint64_t bo = so + (uint64_t)((tq * NKC + 2 * j) * Ns);
            const uint32_t first = (s | tq | j) ? 1u : 0u;
#pragma unroll
            for (int tt = 0; tt < T; ++tt) {
              const uint64_t ao = so + (uint64_t)(2 * j * LR + pre + rowoff + tt * kTcRows);
              tc::mma_f16(tmem + (uint32_t)(tt * Ns), dA + ao, dB + bo, a.idesc, first);
            }
          }
        }
        tc::commit(&empty[slot]);
      }
      if (S > 0) tc::commit(done);
    }
  } else {
    if (warp == 1) {
      // ---- the producer warp: copies spread over its lanes, all asynchronous
      const float* wpb = a.wp + b * a.wpbs;
      const int kc_all = a.Kc >> 3;
      for (int s = 0; s < S; ++s) {
        const int slot = s & 1;
        if (s >= 2) tc::mbar_wait(&empty[slot], (uint32_t)(((s >> 1) - 1) & 1));
        int L0, pre, cb;
        const int kdi = window(s, &L0, &pre, &cb);
        const int nl = (pre + a.WR + a.Sw - 1) / a.Sw;  // lines covering the window
        uint8_t* A = smem + slot * Sb;
        uint8_t* Bt = A + Ab;
        if (lane == 0) tc::mbar_expect_tx(&full[slot], (uint32_t)(NKC * nl * a.Sw * 16 + ntap * NKC * Ns * 16));
        __syncwarp();
        for (int i = lane; i < NKC * nl; i += 32) {
          const int kc = i / nl, li = i - kc * nl;
          const int L = L0 + li, dp = L / Hl, hp = L - dp * Hl;
          tc::tma_load_5d(A + ((size_t)kc * LR + (size_t)li * a.Sw) * 16, &tmap, cb * CB + 8 * kc, -1, hp - 1, dp - 1,
                          b, &full[slot]);
        }
        const int kd = PW ? 0 : kdi;
        const float* wk = wpb + ((long long)(kd * 9) * kc_all + cb * NKC) * a.Np * 4 + (long long)n0 * 4;
        for (int q = lane; q < ntap * NKC; q += 32) {
          const int tq = q / NKC, kcl = q % NKC;
          const int t9 = PW ? 0 : tq;
          tc::bulk_load(Bt + (size_t)q * Ns * 16, wk + ((long long)t9 * kc_all + kcl) * a.Np * 4, (uint32_t)Ns * 16,
                        &full[slot]);
        }
      }
    }
    if (S > 0) {
      tc::mbar_wait(done, 0);
      tc::fence_after();
    }
    __syncwarp();  // warp 1's producer lane rejoins before the aligned TMEM loads
    tc_epilogue<T, MODE>(a, tmem, b, n0, u0, ks, S, warp, lane);
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_free(tmem, a.tmem_cols);
}

// y[v][n] (+)= bias[n] + sum_ks part[b][ks][v][n]  (fixed order)
__global__ void conv_tc_splitk_reduce_k(const float* __restrict__ part, int kspl, long long vout, int N,
                                        const float* __restrict__ bias, long long bbs, d2ip_act y, int accumulate) {
  D2IP_PDL_ENTRY();
  const int b = blockIdx.y;
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= vout * N) return;
  const long long v = i / N;
  const int n = (int)(i - v * N);
  const float* p = part + (long long)b * kspl * vout * N + i;
  const long long ps = vout * N;
  // fixed order k = 0, 1, ...; four loads in flight
  float s = 0.f;
  int k = 0;
  for (; k + 3 < kspl; k += 4) {
    const float a0 = p[(long long)k * ps], a1 = p[(long long)(k + 1) * ps], a2 = p[(long long)(k + 2) * ps],
                a3 = p[(long long)(k + 3) * ps];
    s += a0;
    s += a1;
    s += a2;
    s += a3;
  }
  for (; k < kspl; ++k) s += p[(long long)k * ps];
  if (bias) s += __ldg(bias + b * bbs + n);
  float* yp = y.ptr + b * y.bstride + v * y.cstride + n;
  *yp = accumulate ? *yp + s : s;
}

// the same sum for four consecutive channels per thread (N % 4 == 0, 16-byte aligned views)
__global__ void conv_tc_splitk_reduce4_k(const float* __restrict__ part, int kspl, long long vout, int N,
                                         const float* __restrict__ bias, long long bbs, d2ip_act y, int accumulate) {
  D2IP_PDL_ENTRY();
  const int b = blockIdx.y;
  const int n4 = N >> 2;
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= vout * n4) return;
  const long long v = i / n4;
  const int n = (int)(i - v * n4) * 4;
  const long long ps = vout * N;
  const float4* p = reinterpret_cast<const float4*>(part + (long long)b * kspl * ps + v * N + n);
  const long long ps4 = ps >> 2;
  float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
  int k = 0;
  for (; k + 3 < kspl; k += 4) {
    const float4 a0 = p[(long long)k * ps4], a1 = p[(long long)(k + 1) * ps4], a2 = p[(long long)(k + 2) * ps4],
                 a3 = p[(long long)(k + 3) * ps4];
    s.x += a0.x; s.y += a0.y; s.z += a0.z; s.w += a0.w;
    s.x += a1.x; s.y += a1.y; s.z += a1.z; s.w += a1.w;
    s.x += a2.x; s.y += a2.y; s.z += a2.z; s.w += a2.w;
    s.x += a3.x; s.y += a3.y; s.z += a3.z; s.w += a3.w;
  }
  for (; k < kspl; ++k) {
    const float4 a0 = p[(long long)k * ps4];
    s.x += a0.x; s.y += a0.y; s.z += a0.z; s.w += a0.w;
  }
  if (bias) {
    const float* bb = bias + b * bbs + n;
    s.x += __ldg(bb); s.y += __ldg(bb + 1); s.z += __ldg(bb + 2); s.w += __ldg(bb + 3);
  }
  float4* yp = reinterpret_cast<float4*>(y.ptr + b * y.bstride + v * y.cstride + n);
  if (accumulate) {
    const float4 yo = *yp;
    s.x += yo.x; s.y += yo.y; s.z += yo.z; s.w += yo.w;
  }
  *yp = s;
}

// Stride-2 parity taps: the original tap index along one axis that pairs GEMM
// tap ta (offset ta - 1) with parity pa, or -1 (no such tap; weight 0).
__device__ __forceinline__ int s2_axis(int ta, int pa, int dgrad) {
  if (ta == 1) return pa ? 2 : 1;  // offset 0: x = 2o (k = 1) or 2o + 1 (k = 2)
  if (!dgrad) return (ta == 0 && pa) ? 0 : -1;  // forward offset -1: x = 2(o - 1) + 1 (k = 0)
  return (ta == 2 && pa) ? 0 : -1;              // dgrad offset +1: gx 2o + 1 <- gy o + 1 (k = 0)
}

// One packed weight: code 0 forward, 1 stride-1 dgrad, 2 stride-2 forward
// (k = p C_in + ci), 3 stride-2 dgrad (n = p C_in + ci); + kTcBf16: bf16 layout;
// + kTcPw: 1^3 weights (one tap).
__device__ __forceinline__ float pack_val(const float* wb, int K, int N, int code, int t, int k, int n) {
  if (code & kTcPw) return (code & 1) ? wb[(long long)k * N + n] : wb[(long long)n * K + k];  // 1^3: [co][ci]
  code &= 3;
  if (code == 0) return wb[((long long)n * K + k) * 27 + t];
  if (code == 1) return wb[((long long)k * N + n) * 27 + (26 - t)];
  const int cin = code == 2 ? K >> 3 : N >> 3;
  const int pc = code == 2 ? k : n;
  const int p = pc / cin, ci = pc - p * cin;
  const int kd = s2_axis(t / 9, p >> 2, code == 3), kh = s2_axis((t / 3) % 3, (p >> 1) & 1, code == 3),
            kw = s2_axis(t % 3, p & 1, code == 3);
  if (kd < 0 || kh < 0 || kw < 0) return 0.f;
  const int co = code == 2 ? n : k;
  return wb[((long long)co * cin + ci) * 27 + kd * 9 + kh * 3 + kw];
}

// Pack OIDHW weights into [b][hi|lo][tap][K/4][Np][4] (K-major B tiles).
//   forward: K = C_in,  N = C_out:  P[t][k][n] = W[n][k][t]
//   dgrad  : K = C_out, N = C_in :  P[t][k][n] = W[k][n][26 - t]
//   stride 2: the parity layouts of pack_val (codes 2, 3)
// bf16 (code & kTcBf16): [b][tap][K/8][Np][8] bf16, element i of `half`.
__device__ __forceinline__ void pack_bf16(const float* wb, int K, int N, int Np, int code, long long i,
                                          __nv_bfloat16* out, __nv_bfloat16* lo = nullptr) {
  const int j = (int)(i & 7);
  const long long q = i >> 3;
  const int n = (int)(q % Np);
  const long long q2 = q / Np;
  const int kc = (int)(q2 % (K / 8));
  const int t = (int)(q2 / (K / 8));
  const float val = n < N ? pack_val(wb, K, N, code, t, 8 * kc + j, n) : 0.f;
  const __nv_bfloat16 h = __float2bfloat16_rn(val);
  out[i] = h;
  if (lo) lo[i] = __float2bfloat16_rn(val - __bfloat162float(h));  // 3xbf16: the residual
}

__global__ void conv_tc_pack_k(const float* __restrict__ w, long long wbs, int K, int N, int Np, int dgrad,
                               float* __restrict__ out, long long half, long long obs) {
  D2IP_PDL_ENTRY();
  const int b = blockIdx.y;
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= half) return;
  if (dgrad & (kTcBf16 | kTcBf3)) {
    pack_bf16(w + b * wbs, K, N, Np, dgrad, i, reinterpret_cast<__nv_bfloat16*>(out + b * obs),
              (dgrad & kTcBf3) ? reinterpret_cast<__nv_bfloat16*>(out + b * obs + obs / 2) : nullptr);
    return;
  }
  const int j = (int)(i & 3);
  const long long q = i >> 2;
  const int n = (int)(q % Np);
  long long q2 = q / Np;
  int kc, t;
  if (dgrad & kTcKwf) {  // [kd kh][K/4][kw][Np][4]
    const int kw = (int)(q2 % 3);
    q2 /= 3;
    kc = (int)(q2 % (K / 4));
    t = (int)(q2 / (K / 4)) * 3 + kw;
  } else {
    kc = (int)(q2 % (K / 4));
    t = (int)(q2 / (K / 4));
  }
  const int k = 4 * kc + j;
  const float val = n < N ? pack_val(w + b * wbs, K, N, dgrad, t, k, n) : 0.f;
  const float hi = tf32_hi(val);
  out[b * obs + i] = hi;
  out[b * obs + obs / 2 + i] = val - hi;  // lo half at the fixed offset the kernel reads (wlo)
}

// All layers' packs in one launch, source-major: one thread per (co, ci)
// weight vector reads its 27 contiguous taps (coalesced across the warp) and
// scatters each into its packed slot(s); blockIdx.x walks the concatenated
// job ranges. Slots no weight maps to (N / K padding, stride-2 parity combos
// without a tap) are never written: they stay zero from the workspace clear.
__device__ __forceinline__ void pack_put(float* out, long long obs, int code, int K, int Np, int t, int k, int n,
                                         float val) {
  if (code & (kTcBf16 | kTcBf3)) {
    const long long i = (((long long)t * (K / 8) + k / 8) * Np + n) * 8 + (k & 7);
    const __nv_bfloat16 h = __float2bfloat16_rn(val);
    reinterpret_cast<__nv_bfloat16*>(out)[i] = h;
    if (code & kTcBf3) reinterpret_cast<__nv_bfloat16*>(out + obs / 2)[i] = __float2bfloat16_rn(val - __bfloat162float(h));
  } else {
    // kw-folded layers: [kd kh][K/4][kw][Np][4]; otherwise [tap][K/4][Np][4]
    const long long i = (code & kTcKwf) ? ((((long long)(t / 3) * (K / 4) + k / 4) * 3 + t % 3) * Np + n) * 4 + (k & 3)
                                        : (((long long)t * (K / 4) + k / 4) * Np + n) * 4 + (k & 3);
    const float hi = tf32_hi(val);
    out[i] = hi;
    out[obs / 2 + i] = val - hi;
  }
}

// stride-2 parity decomposition, per axis: source tap k -> (parity, GEMM tap)
// forward: k = 0 -> (1, 0), 1 -> (0, 1), 2 -> (1, 1); dgrad: 0 -> (1, 2), 1 -> (0, 1), 2 -> (1, 1)
__device__ __forceinline__ void s2_inv(int k, int dgrad, int* p, int* ta) {
  *p = k != 1;
  *ta = k == 0 ? (dgrad ? 2 : 0) : 1;
}

__global__ void conv_tc_pack_multi_k(PackJobs j) {
  D2IP_PDL_ENTRY();
  const int b = blockIdx.y;
  int q = 0;
  while (q + 1 < j.n && blockIdx.x >= j.block0[q + 1]) ++q;
  const int cin = j.cin[q], cout = j.cout[q];
  const long long i = (long long)(blockIdx.x - j.block0[q]) * blockDim.x + threadIdx.x;
  if (i >= (long long)cin * cout) return;
  const int co = (int)(i / cin), ci = (int)(i - (long long)co * cin);
  const int code = j.dgrad[q], K = j.K[q], Np = np_of(j.N[q]);
  float* out = j.out[q] + b * j.obs[q];
  const float* src = j.w[q] + b * j.wbs;
  if (code & kTcPw) {  // 1^3: W[co][ci]
    const float val = __ldg(src + i);
    if (code & 1) pack_put(out, j.obs[q], code, K, Np, 0, co, ci, val);
    else pack_put(out, j.obs[q], code, K, Np, 0, ci, co, val);
    return;
  }
  const float* wv = src + i * 27;  // W[co][ci][27]
  const int c3 = code & 3;
#pragma unroll 3
  for (int t = 0; t < 27; ++t) {
    const float val = __ldg(wv + t);
    if (c3 == 0) {
      pack_put(out, j.obs[q], code, K, Np, t, ci, co, val);
    } else if (c3 == 1) {
      pack_put(out, j.obs[q], code, K, Np, 26 - t, co, ci, val);
    } else {
      int pd, pa, ph, pb, pw, pc;
      s2_inv(t / 9, c3 == 3, &pd, &pa);
      s2_inv((t / 3) % 3, c3 == 3, &ph, &pb);
      s2_inv(t % 3, c3 == 3, &pw, &pc);
      const int p = (pd << 2) | (ph << 1) | pw, tg = pa * 9 + pb * 3 + pc;
      if (c3 == 2) pack_put(out, j.obs[q], code, K, Np, tg, p * cin + ci, co, val);
      else pack_put(out, j.obs[q], code, K, Np, tg, co, p * cin + ci, val);
    }
  }
}

int conv_tc_pack_multi(const PackJobs& jobs, int batch, cudaStream_t st) {
  if (jobs.n == 0) return D2IP_OK;
  D2IP_CUDA(launch_pdl(conv_tc_pack_multi_k, dim3(jobs.block0[jobs.n], batch), 256, 0, st, jobs));
  D2IP_LAUNCH_CHECK();
  return D2IP_OK;
}

void pack_jobs_add(PackJobs& j, const float* w, int K, int N, int dgrad, float* out) {
  // layer channels from the GEMM view: codes 0 / 2 (forward) K = C_in (x 8), N = C_out; 1 / 3 transposed
  const int c3 = dgrad & 3;
  const int cin = c3 == 0 ? K : c3 == 1 ? N : c3 == 2 ? K / 8 : N / 8;
  const int cout = (c3 == 0 || c3 == 2) ? N : K;
  const int q = j.n++;
  j.w[q] = w;
  j.out[q] = out;
  j.K[q] = K;
  j.N[q] = N;
  j.dgrad[q] = dgrad;
  j.half[q] = ((dgrad & kTcPw) ? 1LL : 27LL) * K * np_of(N);
  j.obs[q] = conv_tc_pack_floats(K, N);
  j.cin[q] = cin;
  j.cout[q] = cout;
  j.block0[q + 1] = j.block0[q] + (int)(((long long)cin * cout + 255) / 256);
}

bool conv_tc_supported(int cin, int cout, int ks, int stride, int precision) {
  if ((precision != D2IP_PREC_TF32 && precision != D2IP_PREC_BF16) || (ks != 3 && ks != 1) || stride != 1)
    return false;
  if (cin % 8 || cin < 8 || cout < 1 || np_of(cout) > 1024) return false;
  return true;
}

// kw-folded stride-1 kernel (MODE 4): D2IP_TC_KWF=0 keeps one MMA per tap
static bool kwf_enabled() {
  static const bool on = [] {
    const char* v = getenv("D2IP_TC_KWF");
    return !v || atoi(v) != 0;
  }();
  return on;
}

bool tf32_bf3_enabled() {
  static const bool on = [] {
    const char* v = getenv("D2IP_TF32_BF3");
    return v && atoi(v) != 0;
  }();
  return on;
}

// TF32 precision: which layer classes take 3xbf16 instead of 3xTF32 (bit 1 stride-1 3^3
// forward, 2 stride-1 dgrad, 4 stride-2 forward, 8 stride-2 dgrad, 16 1^3; D2IP_TF32_BF3=1
// enables the mask, default 31). Default: none -- every TF32-precision layer is 3xTF32.
// 3xbf16 (~4.5e-6 per op vs 7.6e-7, tools/conv_acc.py) measured faster (cfg1 +5 %, cfg2
// +8 %) but (a) its stride-1 forwards cross a threshold of the network itself: perturbing
// ONE forward conv of the reference net (cfg2 widths, CPU oracle) by 5e-6 relative noise
// moves the gradients by 4.8e-4 (by 1e-6: 7e-7), and the cfg2-width engine with 3xbf16
// forwards lands 3.7e-3 from the oracle (1e-3 bar; 3xTF32: 4.7e-6); (b) at cfg1 budgets
// (2,000 + 3 x 100 TPP iterations) 3xbf16 data gradients leave the reconstructions at
// MSSIM 0.34-0.39 from the reference's and 1.5-3x its misfit, while 3xTF32 everywhere lands
// at 0.55-0.61 -- exactly the band of the reference's own fp32 reorderings (0.55-0.63).
static bool bf3_class(int cls) {
  static const int m = [] {
    const char* v = getenv("D2IP_BF3_MASK");
    return v ? atoi(v) : 31;
  }();
  return (m & cls) != 0;
}

// bf16 precision: forward convolutions on 3xbf16 hi/lo bf16 operands (fp32 accumulate),
// data / weight gradients single-pass bf16. Single-pass bf16 forwards miss the north
// star's 1e-2 gradient bar on the cfg4 network (measured 1.7e-2 overall, worst tensor
// 3.6e-2 on a 32x32x16 grid; tools/l4err.py) -- the forward's rounding reaches the
// gradients through LayerNorm; with 3xbf16 forwards 2.9e-3. D2IP_BF16_FWD3=0: all bf16.
bool bf16_fwd3_enabled() {
  static const bool on = [] {
    const char* v = getenv("D2IP_BF16_FWD3");
    return !v || atoi(v) != 0;
  }();
  return on;
}

bool conv_tc_layer(int cin, int cout, int ks, int stride, int dgrad, int precision, long long vout, TcDims* d) {
  TcDims r{};
  if (stride == 1) {
    r.K = dgrad ? cout : cin;
    r.N = dgrad ? cin : cout;
    r.mode = ks == 1 ? 3 : 0;
    r.pack = dgrad | (ks == 1 ? kTcPw : 0);
    if (!conv_tc_supported(r.K, r.N, ks, 1, precision)) return false;
    // bf16: 16-channel K steps; K % 16 != 0 (e.g. the 8-channel stem) keeps 3xTF32
    if (precision == D2IP_PREC_BF16 && r.K % 16 == 0) {
      const int bit = (!dgrad && bf16_fwd3_enabled()) ? kTcBf3 : kTcBf16;
      r.mode |= bit;
      r.pack |= bit;
    }
    // TF32 precision: 3xbf16 (D2IP_TF32_BF3=0 keeps 3xTF32)
    static const int only_k = [] { const char* v = getenv("D2IP_BF3_ONLYK"); return v ? atoi(v) : 0; }();
    if (precision == D2IP_PREC_TF32 && r.K % 16 == 0 && tf32_bf3_enabled() &&
        bf3_class(ks == 1 ? 16 : dgrad ? 2 : 1) && (!only_k || (only_k == r.K && ks == 3 && !dgrad))) {
      r.mode |= kTcBf3;
      r.pack |= kTcBf3;
    }
    // 3xTF32 stride-1 3^3 layers run kw-folded (MODE 4) with its weight layout
    if (ks == 3 && !(r.mode & (kTcBf16 | kTcBf3)) && kwf_enabled()) {
      r.mode |= kTcKwf;
      r.pack |= kTcKwf;
    }
  } else {
    // Below ~4M output-voxel x channel-pair products the direct CUDA-core kernel
    // is faster (tools/conv_bench.py: 16->32 at 16^3 out 24 vs 29 us; 32->64 at
    // 16^3 out 110 vs 50 us, at 32^3 out 98 vs 73 us). D2IP_TC_S2=0 / 2 forces
    // the direct / tcgen05 kernel.
    static const int s2 = [] {
      const char* v = getenv("D2IP_TC_S2");
      return v ? atoi(v) : 1;
    }();
    if (!s2 || (precision != D2IP_PREC_TF32 && precision != D2IP_PREC_BF16) || ks != 3 || stride != 2) return false;
    // (data gradients: the tensor-core kernel wins at every size since the 3xbf16 path -- cfg1
    // 1,186 -> 1,213 it/s with all stride-2 layers on it; the small forwards stay direct)
    // (wide layers go to the tensor cores at any size -- 64->128 at 8x8x4 out: cfg2 455 -> 461 it/s;
    // the narrow small ones stay direct: cfg1 1,577 vs 1,568 with everything on tcgen05)
    if (s2 == 1 && !dgrad && vout >= 0 && vout * cin * cout < 4LL * 1024 * 1024 && cin * cout < 4096) return false;
    if (!dgrad) {  // K = 8 C_in: a 16-byte chunk must not straddle two parities
      if (cin % 4 || cout < 1 || np_of(cout) > 1024) return false;
      r = TcDims{8 * cin, cout, 1, 2};
    } else {       // 8 epilogue columns share one parity
      if (cout % 8 || cin % 8 || np_of(8 * cin) > 1024) return false;
      r = TcDims{cout, 8 * cin, 2, 3};
    }
    // bf16: 8-channel chunks must not straddle two parities (mode 1: C_in % 8)
    if (precision == D2IP_PREC_BF16 && r.K % 16 == 0 && (dgrad || cin % 8 == 0)) {
      const int bit = (!dgrad && bf16_fwd3_enabled()) ? kTcBf3 : kTcBf16;
      r.mode |= bit;
      r.pack |= bit;
    }
    if (precision == D2IP_PREC_TF32 && r.K % 16 == 0 && (dgrad || cin % 8 == 0) && tf32_bf3_enabled() &&
        bf3_class(dgrad ? 8 : 4)) {
      r.mode |= kTcBf3;
      r.pack |= kTcBf3;
    }
  }
  if (d) *d = r;
  return true;
}

long long conv_tc_pack_floats(int K, int N) { return 2 * 27LL * K * np_of(N); }

int conv_tc_pack(const float* w, long long wbs, int K, int N, int dgrad, float* out, int batch, cudaStream_t st) {
  const long long total = conv_tc_pack_floats(K, N), half = ((dgrad & kTcPw) ? 1LL : 27LL) * K * np_of(N);
  D2IP_CUDA(launch_pdl(conv_tc_pack_k, dim3(cdiv(half, 256), batch), 256, 0, st, w, wbs, K, N, np_of(N), dgrad, out, half, total));
  D2IP_LAUNCH_CHECK();
  return D2IP_OK;
}

// Tile / slice / channel-block / split-K plan for one layer shape.
// Tile / slice / channel-block / split-K plan for one layer shape. Every
// (N slice, channel block) pair that fits shared memory is scored with a
// small latency model -- waves x (serial stages per CTA + fixed prologue /
// epilogue cost) -- because at these sizes a CTA's chain of dependent stages,
// not the tensor pipe, sets the time.
// tma: the window is fetched as whole padded lines (conv_tma_k): a channel
// column holds lrows = ceil((WR + Sw - 1) / Sw) lines of Sw rows
static bool tc_plan(int D, int H, int W, int K, int N, int batch, TcConv& a, int* tiles, int nt = 3,
                    bool bf = false, bool tma = false, bool b3 = false, bool kwf = false, int nst = 2) {
  if (b3) bf = true;
  const int rs = kwf ? kTcRows - 2 : kTcRows;  // output rows per sub-tile
  a.N = N;
  a.Np = np_of(N);
  a.Kc = K;
  // TMA: 8-row (128-byte) aligned line pitch -- every line box lands on a 128-byte boundary
  a.Sw = tma ? (W + 2 + 7) / 8 * 8 : W + 2;
  a.Sh = (H + 2) * a.Sw;
  a.u_first = a.Sh + a.Sw + 1;
  const int u_last = D * a.Sh + H * a.Sw + W;
  const int tiles1 = cdiv(u_last - a.u_first + 1, rs);
  a.vout = (long long)D * H * W;
  a.CB = 0;
  a.T = 1;
  double best = 1e30;
  // Large layers (>= 4 waves of single tiles): T tiles per CTA share each
  // stage's weight tile and per-CTA overhead; scored by a latency model in us:
  // a stage costs max(cp.async landing ~1.5, its MMAs: 27/8 CB T x 57 cycles).
  const bool large = (long long)tiles1 * batch >= 4LL * 296;
  static const int t_force = [] {  // D2IP_TC_T=1/2/4: tiles per CTA for large layers (study knob)
    const char* v = getenv("D2IP_TC_T");
    return v ? atoi(v) : 0;
  }();
  // kw-folded layers with >= 2 waves of single tiles: two sub-tiles per CTA share every stage's
  // weight tile and fixed costs (measured: 48->16 at 64x64x32 fwd 120 -> 94 us, 16->16 56 -> 40;
  // 96->32 at 32x32x16 (150 tiles) is better left at one)
  const int t_pref = t_force ? t_force : (kwf && (long long)tiles1 * batch >= 2LL * 296 && !large) ? 2 : 0;
  for (int T : {1, 2, 4}) {
    if (T > 1 && ((!large && !t_pref) || nt == 2)) break;
    if (t_pref && nt != 2 && T != t_pref) continue;
    const int wr = nt == 1 ? T * kTcRows : wr_of(a.Sw, T);
    const int wrp_tma = (wr + 2 * a.Sw - 2) / a.Sw * a.Sw;
    const int tl = cdiv(tiles1, T);
    for (int ns = std::min(a.Np, 256); ns >= 16; ns -= 16) {
      if (a.Np % ns) continue;
      if (T * ns * (kwf ? 3 : 1) > 512) continue;  // TMEM columns
      if (kwf && 3 * ns > 256) continue;            // one MMA's N
      for (int cb = bf ? 16 : 8; cb <= K && cb <= (bf ? 128 : 64); cb *= 2) {
        if (K % cb) continue;
        const int wrp = tma ? wrp_tma : wrp_of(wr, cb / (bf ? 8 : 4));
        const size_t sm = nst * stage_bytes(cb, ns, wrp, nt, bf, b3) + 3 * wr * sizeof(int) + 64;
        if (sm > (size_t)(nst == 2 ? 210 : 224) * 1024) continue;
        // kw folding parks 128 rows x (2 ns + 4) fp32 in the idle stage buffers
        if (kwf && (size_t)kTcRows * (2 * ns + 4) * 4 > 2 * stage_bytes(cb, ns, wrp, nt, bf, b3)) continue;
        const int per_sm = sm <= (size_t)110 * 1024 ? 2 : 1;
        const long long ctas0 = (long long)tl * (a.Np / ns) * batch;
        const int S = nt * (K / cb);
        // CTAs the split-K aims for (D2IP_TC_KSPL). Two per SM (296) was round 1's choice; every
        // split costs a prologue, an epilogue and a partial-sum plane, and ~100 measured best on
        // both small-grid regimes (cfg2 / cfg1 it/s: 592: 416 / 1,351, 296: 434 / 1,417,
        // 148: 447 / 1,491, 100: 454 / 1,535, 74: 455 / 1,396, 50: 452 / 1,405)
        static const long long kspl_target = [] {
          const char* v = getenv("D2IP_TC_KSPL");
          return v ? atoll(v) : 100LL;
        }();
        const int kspl = (int)std::min<long long>(S, std::max(1LL, (kspl_target + ctas0 - 1) / ctas0));
        const long long waves = (ctas0 * kspl + 148LL * per_sm - 1) / (148LL * per_sm);
        double cost;
        if (!large) {
          cost = (double)waves * ((S + kspl - 1) / kspl + 2.0) + (kspl > 1 ? 1.0 : 0.0);
        } else {
          // bf16: one MMA per 16 channels at max(N/2, (4096 + 32 N)/128) + issue cycles
          // kw folding: nt (kh) MMAs of N = 3 ns per K step instead of nt^2 of N = ns
          const double nq = kwf ? nt : nt * nt, ne = kwf ? 3.0 * ns : ns;
          const double cyc = std::max(ne / 2.0, (4096.0 + 32.0 * ne) / 128.0);
          const double mma_us =
              bf ? (b3 ? 3.0 : 1.0) * nq * (cb / 16.0) * T * (cyc + 6.0) / 1900.0 * (per_sm == 2 ? 1.4 : 1.0)
                 : 3.0 * nq / 8.0 * cb * T * std::max(kwf ? 40.0 : 57.0, cyc) / 1900.0 * (per_sm == 2 ? 1.4 : 1.0);
          const double stage_us = std::max(1.5, mma_us);
          cost = (double)waves * ((S + kspl - 1) / kspl * stage_us + 2.0 + 0.5 * T) + (kspl > 1 ? 3.0 : 0.0);
        }
        if (cost < best - 1e-9) {
          best = cost;
          a.CB = cb;
          a.Ns = ns;
          a.kspl = kspl;
          a.T = T;
          a.WR = wr;
          a.WRp = wrp;
          a.lrows = wrp;
          *tiles = tl;
        }
      }
    }
  }
  if (a.CB < 8) return false;
  a.n_cb = K / a.CB;
  a.bf = bf;
  a.b3 = b3;
  return true;
}

// Ring depth the plan is sized for: three stages for the 3xTF32 layers (the software-pipelined
// producers keep two fills in flight; D2IP_TC_NST=2 restores the two-stage ring), two for bf16.
static int plan_nst(bool bf) {
  static const int nst_tf32 = [] {
    const char* v = getenv("D2IP_TC_NST");
    return v ? std::max(2, std::min(3, atoi(v))) : 3;
  }();
  return bf ? 2 : nst_tf32;
}

// The two-stage plan, with a third stage when it costs no co-resident CTA; layers with enough
// tiles to fill the GPU without split-K re-plan for three stages (a smaller channel block):
// measured at cfg2, 96->32 @ 32x32x16 fwd 109 -> 58 us, 32->32 47 -> 32 us. Split-K layers (deep
// levels, < 100 tiles) keep their plan: more, smaller stages made them slower (17 -> 22 us).
static bool tc_plan_nst(int D, int H, int W, int K, int N, int batch, TcConv& a, int* tiles, int nt, bool bf, bool tma,
                        bool b3, bool kwf) {
  if (!tc_plan(D, H, W, K, N, batch, a, tiles, nt, bf, tma, b3, kwf, 2)) return false;
  a.nst = 2;
  if (plan_nst(bf || b3) < 3 || tma) return true;
  const size_t st = stage_bytes(a.CB, a.Ns, a.WRp, nt, bf, b3), fix = 3 * a.WR * sizeof(int) + 128;
  const size_t two = 2 * st + fix, three = 3 * st + fix;
  // multi-tile CTAs (large grids): a third stage when it keeps the CTAs per SM
  if (a.T >= 2 && (two > (size_t)110 * 1024 ? three <= (size_t)224 * 1024 : three <= (size_t)110 * 1024)) {
    a.nst = 3;
    return true;
  }
  // one CTA per SM with >= 100 tiles (stride 1): re-plan for three stages (a smaller channel block)
  if (nt == 3 && two > (size_t)110 * 1024 && (long long)*tiles * batch >= 100) {
    TcConv a3 = a;
    int tiles3 = 0;
    if (tc_plan(D, H, W, K, N, batch, a3, &tiles3, nt, bf, tma, b3, kwf, 3)) {
      a = a3;
      a.nst = 3;
      *tiles = tiles3;
    }
  }
  return true;
}

size_t conv_tc_ws_bytes(int D, int H, int W, int K, int N, int batch, int mode) {
  TcConv a{};
  int tiles;
  const int m3 = mode & 3;
  size_t best = 0;
  // the larger of the two plans (kw-folded or not) a stride-1 call may take
  for (int kwf = (mode & kTcKwf) ? 1 : 0; kwf <= ((mode & kTcKwf) ? 1 : 0); ++kwf) {
    if (!tc_plan_nst(D, H, W, K, N, batch, a, &tiles, m3 == 3 ? 1 : m3 ? 2 : 3, (mode & kTcBf16) != 0, false,
                     (mode & kTcBf3) != 0, kwf != 0) ||
        a.kspl <= 1)
      continue;
    // mode 2 partials are [V_gx][C_gx]: V_gx C_gx <= 8 V N / 8 (gx dims <= 2 x the row grid)
    best = std::max(best, (size_t)((size_t)batch * a.kspl * a.vout * N * sizeof(float)));
  }
  return best;
}


// Launch one instantiation (the >48 KB shared-memory opt-in is set on first use).
// the window tensor map of the current conv_tc_run call (MODE 4 TMA path; zeros otherwise)
static thread_local CUtensorMap g_tc_tmap;

template <int NKC, int T, int PG, int MODE, int BF>
static int tc_launch(const TcConv& a, dim3 grid, size_t smem, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    D2IP_CUDA(cudaFuncSetAttribute(conv_tc_k<NKC, T, PG, MODE, BF>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   227 * 1024));
    attr = true;
  }
  D2IP_CUDA(launch_pdl((conv_tc_k<NKC, T, PG, MODE, BF>), grid, kTcThreads, smem, st, a, g_tc_tmap));
  return D2IP_OK;
}

template <int NKC, int BF>
static int tc_dispatch(const TcConv& a, dim3 grid, size_t smem, cudaStream_t st, int mode, bool pg2) {
  if (mode == 1) return tc_launch<NKC, 1, 1, 1, BF>(a, grid, smem, st);
  if (mode == 2) return tc_launch<NKC, 1, 1, 2, BF>(a, grid, smem, st);
  if (mode == 4) {
    if (a.T == 4) return tc_launch<NKC, 4, 1, 4, BF>(a, grid, smem, st);
    if (a.T == 2) return tc_launch<NKC, 2, 1, 4, BF>(a, grid, smem, st);
    return tc_launch<NKC, 1, 1, 4, BF>(a, grid, smem, st);
  }
  if (mode == 3) {
    if (a.T == 4) return tc_launch<NKC, 4, 1, 3, BF>(a, grid, smem, st);
    if (a.T == 2) return tc_launch<NKC, 2, 1, 3, BF>(a, grid, smem, st);
    return tc_launch<NKC, 1, 1, 3, BF>(a, grid, smem, st);
  }
  if (BF == 0 && pg2) {
    if (a.T == 4) return tc_launch<NKC, 4, 2, 0, BF>(a, grid, smem, st);
    if (a.T == 2) return tc_launch<NKC, 2, 2, 0, BF>(a, grid, smem, st);
    return tc_launch<NKC, 1, 2, 0, BF>(a, grid, smem, st);
  }
  if (a.T == 4) return tc_launch<NKC, 4, 1, 0, BF>(a, grid, smem, st);
  if (a.T == 2) return tc_launch<NKC, 2, 1, 0, BF>(a, grid, smem, st);
  return tc_launch<NKC, 1, 1, 0, BF>(a, grid, smem, st);
}

// NKC = 16-byte chunks per row: CB / 4 (tf32, CB 8..64) or CB / 8 (bf16, CB 16..128)
template <int BF>
static int tc_dispatch_nkc(const TcConv& a, dim3 grid, size_t smem, cudaStream_t st, int mode, bool pg2) {
  switch (a.CB / (BF != 0 ? 8 : 4)) {
    case 2: return tc_dispatch<2, BF>(a, grid, smem, st, mode, pg2);
    case 4: return tc_dispatch<4, BF>(a, grid, smem, st, mode, pg2);
    case 8: return tc_dispatch<8, BF>(a, grid, smem, st, mode, pg2);
    case 16: return tc_dispatch<16, BF>(a, grid, smem, st, mode, pg2);
    default: D2IP_CHECK_ARG(false, "conv_tc: unsupported channel block %d", a.CB);
  }
  return D2IP_OK;
}

template <int NKC, int T, int MODE, int BFM>
static int tcp_launch(const TcConv& a, dim3 grid, size_t smem, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    D2IP_CUDA(cudaFuncSetAttribute(conv_tcp_k<NKC, T, MODE, BFM>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    attr = true;
  }
  D2IP_CUDA(launch_pdl((conv_tcp_k<NKC, T, MODE, BFM>), grid, kTcpThreads, smem, st, a));
  return D2IP_OK;
}

template <int NKC, int BFM>
static int tcp_dispatch(const TcConv& a, dim3 grid, size_t smem, cudaStream_t st, int mode) {
  if (mode == 3) {
    if (a.T == 4) return tcp_launch<NKC, 4, 3, BFM>(a, grid, smem, st);
    if (a.T == 2) return tcp_launch<NKC, 2, 3, BFM>(a, grid, smem, st);
    return tcp_launch<NKC, 1, 3, BFM>(a, grid, smem, st);
  }
  if (a.T == 4) return tcp_launch<NKC, 4, 0, BFM>(a, grid, smem, st);
  if (a.T == 2) return tcp_launch<NKC, 2, 0, BFM>(a, grid, smem, st);
  return tcp_launch<NKC, 1, 0, BFM>(a, grid, smem, st);
}

template <int BFM>
static int tcp_dispatch_nkc(const TcConv& a, dim3 grid, size_t smem, cudaStream_t st, int mode) {
  switch (a.CB / (BFM != 0 ? 8 : 4)) {
    case 2: return tcp_dispatch<2, BFM>(a, grid, smem, st, mode);
    case 4: return tcp_dispatch<4, BFM>(a, grid, smem, st, mode);
    case 8: return tcp_dispatch<8, BFM>(a, grid, smem, st, mode);
    case 16: return tcp_dispatch<16, BFM>(a, grid, smem, st, mode);
    default: D2IP_CHECK_ARG(false, "conv_tc: unsupported channel block %d", a.CB);
  }
  return D2IP_OK;
}

template <int NKC, int T, int MODE>
static int tma_launch(const TcConv& a, const CUtensorMap& tm, dim3 grid, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    D2IP_CUDA(cudaFuncSetAttribute(conv_tma_k<NKC, T, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    attr = true;
  }
  const size_t smem =
      2 * (((size_t)NKC * a.lrows * 16 + (size_t)(MODE == 3 ? 1 : 9) * NKC * a.Ns * 16 + 127) & ~(size_t)127) + 64;
  D2IP_CUDA(launch_pdl((conv_tma_k<NKC, T, MODE>), grid, kTcThreads, smem, st, a, tm));
  return D2IP_OK;
}

template <int NKC>
static int tma_dispatch(const TcConv& a, const CUtensorMap& tm, dim3 grid, cudaStream_t st, int mode) {
  if (mode == 3) {
    if (a.T == 4) return tma_launch<NKC, 4, 3>(a, tm, grid, st);
    if (a.T == 2) return tma_launch<NKC, 2, 3>(a, tm, grid, st);
    return tma_launch<NKC, 1, 3>(a, tm, grid, st);
  }
  if (a.T == 4) return tma_launch<NKC, 4, 0>(a, tm, grid, st);
  if (a.T == 2) return tma_launch<NKC, 2, 0>(a, tm, grid, st);
  return tma_launch<NKC, 1, 0>(a, tm, grid, st);
}

static int tma_dispatch_nkc(const TcConv& a, const CUtensorMap& tm, dim3 grid, cudaStream_t st, int mode) {
  switch (a.CB / 8) {
    case 2: return tma_dispatch<2>(a, tm, grid, st, mode);
    case 4: return tma_dispatch<4>(a, tm, grid, st, mode);
    case 8: return tma_dispatch<8>(a, tm, grid, st, mode);
    case 16: return tma_dispatch<16>(a, tm, grid, st, mode);
    default: D2IP_CHECK_ARG(false, "conv_tc: unsupported channel block %d", a.CB);
  }
  return D2IP_OK;
}

int conv_tc_run(d2ip_act x, const float* wp, int K, int N, const float* bias, long long bbs, d2ip_act y,
                int accumulate, float* ws, size_t ws_bytes, int batch, cudaStream_t st, int* deferred, int mode,
                const LnFuse* ln, int* fused) {
  if (fused) *fused = 0;
  const bool b3 = (mode & kTcBf3) != 0;
  const bool bf = b3 || (mode & kTcBf16) != 0;
  const bool kwf_bit = (mode & kTcKwf) != 0;  // the weights were packed for the kw-folded kernel
  mode &= 3;
  D2IP_CHECK_ARG(!bf || K % 16 == 0, "conv_tc: bf16 needs K %% 16 == 0 (K=%d)", K);
  D2IP_CHECK_ARG((mode == 1 ? 8 * x.c : x.c) == K && (mode == 2 ? 8 * y.c : y.c) == N, "conv_tc: channel mismatch");
  D2IP_CHECK_ARG(x.cstride % 4 == 0 && ((uintptr_t)x.ptr & 15) == 0, "conv_tc: input view must be 16B aligned");
  D2IP_CHECK_ARG(mode != 2 || (y.cstride % 4 == 0 && ((uintptr_t)y.ptr & 15) == 0 && y.c % 8 == 0),
                 "conv_tc: stride-2 dgrad output view must be 16B aligned with C %% 8 == 0");
  const d2ip_act& g = mode == 1 ? y : x;  // the row-space grid
  if (mode == 1) D2IP_CHECK_ARG(g.d == (x.d + 1) / 2 && g.h == (x.h + 1) / 2 && g.w == (x.w + 1) / 2, "conv_tc: stride-2 shape");
  if (mode == 2) D2IP_CHECK_ARG(g.d == (y.d + 1) / 2 && g.h == (y.h + 1) / 2 && g.w == (y.w + 1) / 2, "conv_tc: stride-2 shape");
  TcConv a{};
  int tiles = 0;
  const int ntm = mode == 3 ? 1 : mode ? 2 : 3;
  // TMA-fed kernel (D2IP_TC_TMA=1): bf16 layers with a twin, stride 1 / 1^3, padded lines <= 256
  // columns (box limit). Opt-in: with its 2-stage ring it measured slower than the eight-warp
  // cp.async fill on most cfg4 layers (e.g. 96->32 fwd 235 vs 201 us, 64->64 64 vs 43 us; only
  // the 96->32 data gradient won, 167 vs 182 us).
  static const bool tma_on = [] {
    const char* v = getenv("D2IP_TC_TMA");
    return v && atoi(v) != 0;
  }();
  const bool use_tma = tma_on && bf && !b3 && (mode == 0 || mode == 3) && x.bf16 && x.cstride % 8 == 0 && x.c % 8 == 0 &&
                       ((uintptr_t)x.bf16 & 15) == 0 && x.w + 2 <= 256;
  D2IP_CHECK_ARG(tc_plan_nst(g.d, g.h, g.w, K, N, batch, a, &tiles, ntm, bf, use_tma, b3, false),
                 "conv_tc: no channel blocking fits shared memory (K=%d N=%d W=%d)", K, N, g.w);
  // kw folding (MODE 4) for stride-1 3^3 layers on the one-tile kernel: 3x fewer MMAs of 3x
  // the width. 3xTF32 layers only: on cfg4's 3xbf16 forwards (large grids, T = 4 tiles) it
  // measured slower (122.7 vs 127.9 it/s); not for the TMA / persistent bf16 kernels
  bool kwf = false;
  if (kwf_bit) {
    D2IP_CHECK_ARG(mode == 0 && !use_tma && !bf, "conv_tc: kw-folded packing on a layer that cannot run it");
    TcConv k2{};
    int tiles2 = 0;
    D2IP_CHECK_ARG(tc_plan_nst(g.d, g.h, g.w, K, N, batch, k2, &tiles2, ntm, bf, false, b3, true),
                   "conv_tc: no kw-folded plan fits (K=%d N=%d W=%d)", K, N, g.w);
    a = k2;
    tiles = tiles2;
    kwf = true;
  }
  // TMA-staged windows for the kw-folded 3xTF32 kernel (D2IP_TC_TMA3=1; one N slice, 16-byte
  // aligned channel views): one 5-D box per (padded line, 4-channel chunk), the zero halo from the
  // boxes' out-of-bounds fill, then the lo split in shared memory. Correct (tests/test_gpu_ops.py
  // with the knob) but measured slower than the cp.async fill -- the 8-row (128-byte) aligned line
  // pitch adds 18 % virtual rows at W = 32, and the landing -> split -> arrive chain serialises each
  // stage: 48->16 @ 64x64x32 fwd 147 vs 123 us, dgrad 106 vs 70; cfg1 1,079 vs 1,134 it/s. Opt-in.
  static const bool tma3_on = [] {
    const char* v = getenv("D2IP_TC_TMA3");
    return v && atoi(v) != 0;
  }();
  bool tma3 = false;
  memset(&g_tc_tmap, 0, sizeof(g_tc_tmap));
  if (kwf && tma3_on && x.c % 4 == 0 && x.cstride % 4 == 0 && ((uintptr_t)x.ptr & 15) == 0 && x.w + 2 <= 256 &&
      (x.bstride * 4) % 16 == 0) {
    TcConv k3{};
    int tiles3 = 0;
    if (tc_plan(g.d, g.h, g.w, K, N, batch, k3, &tiles3, ntm, false, true, false, true) && k3.Ns == k3.Np) {
      static PFN_cuTensorMapEncodeTiled_v12000 encode3 = [] {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
          fn = nullptr;
        return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
      }();
      if (encode3) {
        const cuuint64_t gdim[5] = {(cuuint64_t)x.c, (cuuint64_t)x.w, (cuuint64_t)x.h, (cuuint64_t)x.d,
                                    (cuuint64_t)batch};
        const cuuint64_t gstr[4] = {(cuuint64_t)x.cstride * 4, (cuuint64_t)x.w * x.cstride * 4,
                                    (cuuint64_t)x.h * x.w * x.cstride * 4, (cuuint64_t)x.bstride * 4};
        const cuuint32_t box[5] = {4, (cuuint32_t)k3.Sw, 1, 1, 1}, estr[5] = {1, 1, 1, 1, 1};
        const CUresult cr = encode3(&g_tc_tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 5, x.ptr, gdim, gstr, box, estr,
                                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                    CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (cr == CUDA_SUCCESS) {
          a = k3;
          tiles = tiles3;
          tma3 = true;
        } else {
          memset(&g_tc_tmap, 0, sizeof(g_tc_tmap));
        }
      }
    }
  }
  a.mode = kwf ? 4 : mode;
  a.tma = tma3 ? 1 : 0;
  a.t0 = mode == 2 ? 1 : 0;
  a.nt = ntm;
  a.gd = g.d;
  a.gh = g.h;
  a.gw = g.w;
  const int Nout = mode == 2 ? y.c : N;  // channels of the stored result (partials too)
  if (mode == 2) a.vout = (long long)y.d * y.h * y.w;
  if (a.kspl > 1 && (!ws || ws_bytes < (size_t)batch * a.kspl * a.vout * Nout * sizeof(float))) a.kspl = 1;
  a.part = ws;
  a.x = x;
  a.wp = wp;
  a.wpbs = conv_tc_pack_floats(K, N);
  a.wlo = a.wpbs / 2;
  a.bias = bias;
  a.bbs = bbs;
  a.y = y;
  a.accumulate = accumulate;
  a.vec = y.cstride % 4 == 0 && ((uintptr_t)y.ptr & 15) == 0;
  a.pvec = Nout % 4 == 0 && ((uintptr_t)ws & 15) == 0;
  a.xtw = bf && !b3 && x.bf16 && x.cstride % 8 == 0 && x.c % 8 == 0 && ((uintptr_t)x.bf16 & 15) == 0;
  int cols = 32;
  while (cols < a.T * a.Ns * (kwf ? 3 : 1)) cols *= 2;
  a.tmem_cols = cols;
  a.idesc = tc::make_idesc(bf ? 1 : 2, kTcRows, a.Ns * (kwf ? 3 : 1));
  // ring depth: decided with the plan (three stages for 3xTF32 layers where they fit)
  if (tma3 || use_tma) a.nst = 2;
  static const int async_on = [] {
    const char* v = getenv("D2IP_TC_ASYNC");
    return v ? atoi(v) : 1;
  }();
  a.async_arrive = async_on;
  static const int dbg_on = [] {
    const char* v = getenv("D2IP_TC_DBG");
    return v ? atoi(v) : 0;
  }();
  a.dbg = dbg_on;
  // LayerNorm fused into the kw-folded epilogue: one N slice holding every channel (<= 64), no
  // split-K, float4-aligned views; statistics parked after the P_1 / P_2 exchange rows
  static const bool ln_on = [] {
    const char* v = getenv("D2IP_TC_LNFUSE");
    return !v || atoi(v) != 0;
  }();
  a.ln = 0;
  if (ln && ln_on && kwf && a.kspl == 1 && a.Ns == N && N % 16 == 0 && N <= 64 && !accumulate &&
      ln->out.cstride % 4 == 0 && ((uintptr_t)ln->out.ptr & 15) == 0 &&
      (!ln->res.ptr || (ln->res.cstride % 4 == 0 && ((uintptr_t)ln->res.ptr & 15) == 0)) &&
      (!ln->out.bf16 || (ln->out.cstride % 8 == 0 && ((uintptr_t)ln->out.bf16 & 15) == 0)) &&
      (size_t)kTcRows * (2 * a.Ns + 4) * 4 + 2 * kTcRows * 4 <= (size_t)a.nst * stage_bytes(a.CB, a.Ns, a.WRp, a.nt, a.bf, a.b3)) {
    a.ln = 1;
    a.lnf = *ln;
    if (fused) *fused = 1;
  }
  const size_t smem = use_tma ? 0 : tc_smem_bytes(a);  // (the TMA kernel sizes its own)
  const dim3 grid(tiles, (a.Np / a.Ns) * a.kspl, batch);
  // one producer group (all eight warps per stage) measured faster than two on
  // cfg1 (1029 vs 1013 it/s) and cfg2 (280 vs 274); D2IP_TC_PG=2 selects two
  static const bool pg2 = [] {
    const char* v = getenv("D2IP_TC_PG");
    return v && atoi(v) == 2;
  }();
  int rc;
  // persistent kernel for large stride-1 / 1^3 layers without split-K: default for bf16 layers
  // (cfg4: 96->32 fwd 186 vs 199 us, 64->64 dgrad 38 vs 41 us; 139.2 -> 140.4 it/s), opt-in for
  // the 3xbf16 / 3xTF32 ones (16->16 at 64x64x32: 43 vs 41 us). D2IP_TC_PERSIST=0 / 1 / 2:
  // never / bf16 only / every precision.
  static const int persist_mode = [] {
    const char* v = getenv("D2IP_TC_PERSIST");
    return v ? atoi(v) : 1;
  }();
  const bool persist_on = persist_mode == 2 || (persist_mode == 1 && bf && !b3);
  if (persist_on && !kwf && !use_tma && a.kspl == 1 && (mode == 0 || mode == 3) && 2 * a.T * a.Ns <= 512 &&
      (long long)tiles * (a.Np / a.Ns) * batch >= 2 * 148) {
    TcConv p = a;
    p.ntiles = tiles;
    // D2IP_TCP_NST=3: a third ring stage when it fits (measured slower: cfg4 135.5 vs 140.0 it/s,
    // the larger footprint costs co-resident CTAs)
    static const int tcp_nst = [] {
      const char* v = getenv("D2IP_TCP_NST");
      return v ? atoi(v) : 2;
    }();
    if (tcp_nst >= 3 &&
        3 * stage_bytes(p.CB, p.Ns, p.WRp, p.nt, p.bf, p.b3) + 6 * (size_t)p.WR * 4 + 128 <= (size_t)225 * 1024)
      p.nst = 3;
    int cols = 32;
    while (cols < 2 * p.T * p.Ns) cols *= 2;
    p.tmem_cols = cols;
    const size_t sm = (size_t)p.nst * stage_bytes(p.CB, p.Ns, p.WRp, p.nt, p.bf, p.b3) + 6 * (size_t)p.WR * 4 + 10 * 8 + 16;
    const int per_sm = std::max(1, std::min((int)((size_t)227 * 1024 / sm), 512 / cols));
    const int ctas = std::min(tiles, std::max(1, 148 * per_sm / std::max(1, (p.Np / p.Ns) * batch)));
    const dim3 pgrid(ctas, p.Np / p.Ns, batch);
    if (b3) rc = tcp_dispatch_nkc<2>(p, pgrid, sm, st, mode);
    else if (bf) rc = tcp_dispatch_nkc<1>(p, pgrid, sm, st, mode);
    else rc = tcp_dispatch_nkc<0>(p, pgrid, sm, st, mode);
    D2IP_RET(rc);
    D2IP_LAUNCH_CHECK();
    if (deferred) *deferred = 0;
    set_variant(b3 ? "tcgen05_bf16x3_persistent" : bf ? "tcgen05_bf16_persistent" : "tcgen05_tf32x3_persistent");
    return D2IP_OK;
  }
  if (use_tma) {
    // tensor map over the bf16 twin: dims (C, W, H, D, B) innermost first, one padded line per box
    CUtensorMap tm;
    const cuuint64_t gdim[5] = {(cuuint64_t)x.c, (cuuint64_t)x.w, (cuuint64_t)x.h, (cuuint64_t)x.d,
                                (cuuint64_t)batch};
    const cuuint64_t gstr[4] = {(cuuint64_t)x.cstride * 2, (cuuint64_t)x.w * x.cstride * 2,
                                (cuuint64_t)x.h * x.w * x.cstride * 2, (cuuint64_t)x.bstride * 2};
    const cuuint32_t box[5] = {8, (cuuint32_t)a.Sw, 1, 1, 1}, estr[5] = {1, 1, 1, 1, 1};
    // the driver entry point is resolved through the runtime (no libcuda link dependency: the
    // library must load on machines without a driver, e.g. for the CPU-side ABI tests)
    static PFN_cuTensorMapEncodeTiled_v12000 encode = [] {
      void* fn = nullptr;
      cudaDriverEntryPointQueryResult q;
      if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
          q != cudaDriverEntryPointSuccess)
        fn = nullptr;
      return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }();
    D2IP_CHECK_ARG(encode != nullptr, "conv_tc: cuTensorMapEncodeTiled unavailable");
    const CUresult cr = encode(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, x.bf16, gdim, gstr, box, estr,
                               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    D2IP_CHECK_ARG(cr == CUDA_SUCCESS, "conv_tc: cuTensorMapEncodeTiled failed (%d)", (int)cr);
    rc = tma_dispatch_nkc(a, tm, grid, st, mode);
  } else if (b3)
    rc = tc_dispatch_nkc<2>(a, grid, smem, st, a.mode, false);
  else if (bf)
    rc = tc_dispatch_nkc<1>(a, grid, smem, st, a.mode, false);
  else
    rc = tc_dispatch_nkc<0>(a, grid, smem, st, a.mode, pg2 && !kwf);
  D2IP_RET(rc);
  D2IP_LAUNCH_CHECK();
  if (deferred) *deferred = a.kspl > 1 ? a.kspl : 0;
  if (a.kspl > 1 && !deferred) {
    if (a.pvec && a.vec && (a.vout * Nout) % 4 == 0)
      D2IP_CUDA(launch_pdl(conv_tc_splitk_reduce4_k, dim3(cdiv(a.vout * Nout / 4, 256), batch), 256, 0, st, ws, a.kspl,
                           a.vout, Nout, bias, bbs, y, accumulate));
    else
      D2IP_CUDA(launch_pdl(conv_tc_splitk_reduce_k, dim3(cdiv(a.vout * Nout, 256), batch), 256, 0, st, ws, a.kspl,
                           a.vout, Nout, bias, bbs, y, accumulate));
    D2IP_LAUNCH_CHECK();
  }
  if (kwf) {
    set_variant(tma3 ? (a.kspl > 1 ? "tcgen05_tf32x3_kwf_tma_splitk" : "tcgen05_tf32x3_kwf_tma")
                     : (a.kspl > 1 ? "tcgen05_tf32x3_kwf_splitk" : "tcgen05_tf32x3_kwf"));
    return D2IP_OK;
  }
  set_variant(b3 ? (a.kspl > 1 ? "tcgen05_bf16x3_splitk" : "tcgen05_bf16x3")
              : use_tma ? (a.kspl > 1 ? "tcgen05_bf16_tma_splitk" : "tcgen05_bf16_tma")
              : bf ? (a.kspl > 1 ? "tcgen05_bf16_splitk" : "tcgen05_bf16")
                 : (a.kspl > 1 ? "tcgen05_tf32x3_splitk" : "tcgen05_tf32x3"));
  return D2IP_OK;
}

}  // namespace d2ip
