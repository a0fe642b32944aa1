// K3 on the tensor cores: weight + bias gradient of the stride-1 3^3 / 1^3
// convolutions (autograd's conv backward w.r.t. weight/bias, pipeline.py:330)
// as tcgen05 MMAs with 3xTF32 operands and FP32 accumulation in TMEM.
//
//   dW[co][ci][t] = sum_u x[u + off_t][ci] * gy[u][co]
//
// GEMM view: M = input channels (x side), N = output channels (gy side),
// K = rows u of the same virtual zero-padded grid as the forward kernel
// (conv_tc.cu), so a tap t is the constant row shift off_t. Both operands are
// MN-major (K runs along the rows): each row of a 32-channel block is one
// 128-byte line of shared memory in the "128B_BASE32B" layout (tc.cuh), so a
// tap is a whole-row move of the x descriptor's start address -- no im2col.
// Each CTA owns G taps (one kd plane, or a kh row of it) of one input-channel
// block, keeps G accumulators [M x N] in TMEM, and streams its share of the
// row chunks through a 2-stage cp.async ring (zero-fill outside the grid, so
// border rows of the virtual grid contribute nothing). Partial sums per row
// group are written to a workspace and summed in a fixed order
// (deterministic). The bias gradient is a column sum of gy, accumulated by one
// CTA column while it splits gy into TF32 hi/lo halves.
//
// Tap stacking (C_out <= 32): a tcgen05.mma costs ~57 cycles however small
// its N (tools/umma_rate.cu), so the three kw taps of a (kd, kh) row go into
// one MMA with N = 3 x 32. The kw shift moves to the gy side,
//   sum_u x[u + s(kd,kh) + kw - 1] gy[u] = sum_u x[u + s(kd,kh)] gy[u + 1 - kw],
// and B block b = 2 - kw is the gy tile started b rows later: LBO = one row.
//
// Tap packing (C_in, C_out <= 16, the 32^3 levels): two 16-channel rows share
// one 128-byte line, so the producers bake the kh shift into the x operand
// and the kw shift into gy:
//   x block 0 row w = [x[w + A] | x[w + A + Sw]], block 1 = [x[w + A + 2 Sw] | -]
//   gy line j       = [gy[w0 + j - 1] | gy[w0 + j - 2]], N block 1 = 2 lines on
// (A = (kd - 1) Sh - Sw). One M = 64, N = 64 MMA per K step then covers the
// nine (kh, kw) taps of a kd plane (D rows 16 kh + ci, columns: block 0 =
// [kw 2 | -], block 1 = [kw 0 | kw 1]) -- a third of the stacked MMA count.
//
// M is 64 or 128 (tcgen05 shapes): a channel block smaller than M is read
// with LBO = 0 (one 32-channel block, repeated) or runs into a padded block;
// those rows of D are never stored.
#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"
#include "tc.cuh"

namespace d2ip {

// warp 0: MMA issue; then two producer groups of kWtW warps (loads, splits, epilogue). Eight
// warps per group: with two (64 threads per stage, synchronous copy -> wait -> split) the
// producers were bound by latency at one warp per scheduler
constexpr int kWtW = 8;
constexpr int kWtProd = 2 * kWtW * 32;
// MMA-issue warps: a single issuer pays >= 57 cycles per MMA (more with runtime descriptor
// arithmetic), so the accumulators of a CTA (kh rows / taps) are dealt round-robin to three
constexpr int kWtI = 3;
constexpr int kWtThreads = 32 * kWtI + kWtProd;

struct WgTc {
  d2ip_act x, gy;
  int Sw, Sh, u_first, u_last;
  int RS;              // rows per stage (K chunk)
  int WR;              // x window rows (RS + 2 Sw + 2 for 3^3, RS for 1^3)
  int nchunk, chunks_per_rg, nrg;
  int cib, ncib;       // input-channel block (M side), blocks
  int M, N;            // MMA shape; N = C_out rounded up
  int G, ngroups;      // taps per CTA, tap groups
  int ntaps;           // 27 or 1
  int stack;           // 1: the three kw taps of a (kd, kh) row share one MMA (N = 3 x 32, see below)
  int pack;            // 1: C_in, C_out <= 16 -- all nine taps of a kd plane in one 64 x 64 MMA (see below)
  int RSg;             // gy rows per stage (RS, or RS + 2 with the kw halo)
  int nchx, nchg;      // real 16-B chunks per row of the x block / of gy
  uint32_t Bx, Bg;     // bytes of one 32-channel block region: WR x 128 / RS x 128, 1024-aligned
  uint32_t lbox, lbog; // descriptor LBO (block stride, or 0 for a single repeated block)
  uint32_t Sx, Sg;     // bytes of one x (hi or lo) / gy (hi or lo) buffer
  uint32_t Sb;         // bytes of one stage
  uint32_t pad;        // bytes after the stages covering MMA reads of padded blocks
  int NSTG;            // stages in the ring
  int tmem_cols;
  uint32_t idesc;
  float* part;         // [b][rg][ntaps * Cin * Cout + Cout]
};

__device__ __forceinline__ float tf32_hi_w(float x) { return __uint_as_float(__float_as_uint(x) & 0xFFFFE000u); }

__device__ __forceinline__ int wg_voxel(const WgTc& a, int u) {
  if (u < a.u_first || u > a.u_last) return -1;
  const int dp = u / a.Sh, r = u - dp * a.Sh;
  const int hp = r / a.Sw, wp = r - hp * a.Sw;
  if (dp >= 1 && dp <= a.x.d && hp >= 1 && hp <= a.x.h && wp >= 1 && wp <= a.x.w)
    return ((dp - 1) * a.x.h + (hp - 1)) * a.x.w + (wp - 1);
  return -1;
}

// byte offset of 16-B chunk c (4 channels) of row r in a region of 32-channel
// blocks (block stride B): granule (c % 8) / 2 swizzled by r % 4 (regions are
// 1024-byte aligned, so r % 4 == address bits 7-8).
__device__ __forceinline__ uint32_t mn32_off(int r, int c, uint32_t B) {
  const int cc = c & 7;
  return (uint32_t)(c >> 3) * B + (uint32_t)r * 128 + (uint32_t)((((cc >> 1) ^ (r & 3)) << 5) | ((cc & 1) << 4));
}

// NCHXP / NCHGP: chunks per row rounded up to a power of two (lane -> (row, chunk)).
// Warp-specialised: warp 0 (one elected lane) issues the MMAs of a stage as
// soon as the four producer warps have landed and split it (`full` barrier),
// and hands the slot back through `tcgen05.commit` (`empty`); producers run
// up to NSTG stages ahead, so loads and splits overlap the tensor pipe.
template <int NCHXP, int NCHGP>
__global__ void __launch_bounds__(kWtThreads) wgrad_tc_k(WgTc a) {
  D2IP_PDL_ENTRY();
  extern __shared__ __align__(1024) uint8_t smem[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int b = blockIdx.z;
  const int rg = blockIdx.x;
  const int grp = blockIdx.y % a.ngroups, cbk = blockIdx.y / a.ngroups;
  const int t0 = grp * a.G;  // first tap of this CTA
  const int kd = a.ntaps == 27 ? t0 / 9 : 1;
  const bool do_bias = grp == 0 && cbk == 0;
  const int RS = a.RS, WR = a.WR, RSg = a.RSg, NSTG = a.NSTG;
  const d2ip_act x = a.x, gy = a.gy;
  const float* xb = x.ptr + b * x.bstride + cbk * a.cib;
  const float* gb = gy.ptr + b * gy.bstride;
  // layout: NSTG stages of [x hi][x lo][gy hi][gy lo] (1024-aligned regions), the
  // read pad, barriers full[NSTG] empty[NSTG] done, TMEM slot, bias partials
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)NSTG * a.Sb + a.pad);
  uint64_t* empty = full + NSTG;
  uint64_t* done = empty + NSTG;
  uint8_t* tail = smem + (size_t)NSTG * a.Sb + a.pad + (((2 * NSTG + 1) * 8 + 15) & ~15);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(tail);
  float4* bred = reinterpret_cast<float4*>(tail + 16);  // [kWtProd] bias partials (layout: see wt_smem)
  int* rowmaps = reinterpret_cast<int*>(tail + 16 + kWtProd * 16);  // [2 groups][WR + RSg] voxel offsets

  if (warp == 0) tc::tmem_alloc(tslot, a.tmem_cols);
  if (tid == 0) {
    for (int i = 0; i < NSTG; ++i) {
      tc::mbar_init(&full[i], kWtProd / 2);  // one producer group (2 warps) fills a stage
      tc::mbar_init(&empty[i], kWtI);
    }
    tc::mbar_init(done, kWtI);
    tc::fence_mbar_init();
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = *tslot;
  const int c_lo = rg * a.chunks_per_rg, c_hi = min(a.nchunk, c_lo + a.chunks_per_rg);
  const int S = c_hi - c_lo;
  const int Cin = x.c, Cout = gy.c;
  float* pb = a.part + ((long long)b * a.nrg + rg) * ((long long)a.ntaps * Cin * Cout + Cout);

  if (warp < kWtI) {
    // ---- MMA issue: issuer w takes accumulators w, w + kWtI, ...
    if (lane == 0) {
      const uint32_t sbase = tc::smem_u32(smem);
      const uint64_t dXhi = tc::make_desc_mn32(sbase, a.lbox), dXlo = dXhi + (a.Sx >> 4);
      const uint64_t dGhi = tc::make_desc_mn32(sbase + 2 * a.Sx, a.lbog), dGlo = dGhi + (a.Sg >> 4);
      for (int s = 0; s < S; ++s) {
        const int slot = s % NSTG;
        tc::mbar_wait(&full[slot], (uint32_t)((s / NSTG) & 1));
        tc::fence_after();
        const uint64_t boff = (uint64_t)(slot * a.Sb) >> 4;
        const int nacc = a.stack ? 3 : a.G;  // accumulators: kh rows (stacked) or taps
        for (int i = warp; i < nacc; i += kWtI) {
          const int t = t0 + (a.stack ? 3 * i : i);
          const int tt = a.ntaps == 27 ? t % 9 : 0;
          const int rowoff = a.ntaps == 27 ? (tt / 3) * a.Sw + (a.stack ? 0 : tt % 3) : 0;
          const uint32_t dcol = tmem + (uint32_t)(i * a.N);
          for (int j = 0; j < RS / 8; ++j) {
            // a row is 128 B = 8 descriptor units
            const uint64_t xo = boff + (uint64_t)(rowoff + 8 * j) * 8;
            const uint64_t go = boff + (uint64_t)(8 * j) * 8;
            const uint32_t first = (s | j) ? 1u : 0u;
            tc::mma_tf32(dcol, dXlo + xo, dGhi + go, a.idesc, first);
            tc::mma_tf32(dcol, dXhi + xo, dGlo + go, a.idesc, 1u);
            tc::mma_tf32(dcol, dXhi + xo, dGhi + go, a.idesc, 1u);
          }
        }
        tc::commit(&empty[slot]);
      }
      if (S > 0) tc::commit(done);
    }
  } else {
    // ---- producers: two groups of 2 warps take alternate stages, so two stages
    // are in flight; a group first maps its stage's rows to voxels once (one
    // division pair per row, not per 16-byte chunk), then copies and splits
    // with fixed (row, chunk) ownership per thread.
    const int ptid = tid - 32 * kWtI, pg = (warp - kWtI) / kWtW, gw = (warp - kWtI) % kWtW, gtid = gw * 32 + lane;
    const int xshift = a.ntaps == 27 ? (kd - 1) * a.Sh - a.Sw - (a.stack ? 0 : 1) : 0;
    constexpr int XR = 32 / NCHXP, GR = 32 / NCHGP;  // rows per warp step
    const int xr = lane / NCHXP, xc = lane % NCHXP, gr = lane / NCHGP, gc = lane % NCHGP;
    int* rm = rowmaps + pg * (WR + RSg);
    float4 bacc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int s = pg; s < S; s += 2) {
      const int slot = s % NSTG;
      if (s >= NSTG) tc::mbar_wait(&empty[slot], (uint32_t)((s / NSTG - 1) & 1));
      const int u0 = a.u_first + (c_lo + s) * RS;
      for (int i = gtid; i < WR + RSg; i += 32 * kWtW)
        rm[i] = i < WR ? wg_voxel(a, u0 + xshift + i) : wg_voxel(a, u0 - a.stack + (i - WR));
      asm volatile("bar.sync %0, %1;" ::"r"(1 + pg), "n"(32 * kWtW) : "memory");
      uint8_t* X = smem + (size_t)slot * a.Sb;
      uint8_t* Gt = X + 2 * a.Sx;
      for (int r0 = gw * XR; r0 < WR; r0 += kWtW * XR) {
        const int r = r0 + xr;
        if (r < WR && xc < a.nchx) {
          const int v = rm[r];
          const float* src = v >= 0 ? xb + (long long)v * x.cstride + 4 * xc : xb;
          tc::cp_async16(X + mn32_off(r, xc, a.Bx), src, v >= 0 ? 16u : 0u);
        }
      }
      for (int r0 = gw * GR; r0 < RSg; r0 += kWtW * GR) {
        const int r = r0 + gr;
        if (r < RSg && gc < a.nchg) {
          const int v = rm[WR + r];
          const float* src = v >= 0 ? gb + (long long)v * gy.cstride + 4 * gc : gb;
          tc::cp_async16(Gt + mn32_off(r, gc, a.Bg), src, v >= 0 ? 16u : 0u);
        }
      }
      tc::cp_async_commit();
      tc::cp_async_wait<0>();
      // lo halves (the raw fp32 operand is the hi half: the tensor core truncates to TF32)
      for (int r0 = gw * XR; r0 < WR; r0 += kWtW * XR) {
        const int r = r0 + xr;
        if (r < WR && xc < a.nchx) {
          const uint32_t o = mn32_off(r, xc, a.Bx);
          const float4 v = *reinterpret_cast<const float4*>(X + o);
          float4 l;
          l.x = v.x - tf32_hi_w(v.x); l.y = v.y - tf32_hi_w(v.y); l.z = v.z - tf32_hi_w(v.z); l.w = v.w - tf32_hi_w(v.w);
          *reinterpret_cast<float4*>(X + a.Sx + o) = l;
        }
      }
      for (int r0 = gw * GR; r0 < RSg; r0 += kWtW * GR) {
        const int r = r0 + gr;
        if (r < RSg && gc < a.nchg) {
          const uint32_t o = mn32_off(r, gc, a.Bg);
          const float4 v = *reinterpret_cast<const float4*>(Gt + o);
          float4 l;
          l.x = v.x - tf32_hi_w(v.x); l.y = v.y - tf32_hi_w(v.y); l.z = v.z - tf32_hi_w(v.z); l.w = v.w - tf32_hi_w(v.w);
          *reinterpret_cast<float4*>(Gt + a.Sg + o) = l;
          if (do_bias && r >= a.stack && r < RS + a.stack) {  // the halo rows belong to the neighbour chunks
            bacc.x += v.x; bacc.y += v.y; bacc.z += v.z; bacc.w += v.w;
          }
        }
      }
      tc::fence_proxy_async();
      tc::mbar_arrive(&full[slot]);
      asm volatile("bar.sync %0, %1;" ::"r"(1 + pg), "n"(32 * kWtW) : "memory");  // rm is rebuilt next stage
    }
    if (do_bias) bred[ptid] = bacc;
  }
  __syncthreads();
  if (warp >= kWtI) {
    const int ptid = tid - 32 * kWtI;
    if (do_bias && ptid < a.nchg) {  // fixed-order column sum of gy over this CTA's rows
      float4 sum = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int q = 0; q < kWtProd; ++q) {
        if ((q & 31) % NCHGP != ptid) continue;
        const float4 v = bred[q];
        sum.x += v.x; sum.y += v.y; sum.z += v.z; sum.w += v.w;
      }
      float* o = pb + (long long)a.ntaps * Cin * Cout + 4 * ptid;
      o[0] = sum.x; o[1] = sum.y; o[2] = sum.z; o[3] = sum.w;
    }
    if (S > 0) {
      tc::mbar_wait(done, 0);
      tc::fence_after();
    }
    // epilogue: D row m (input channel) lives in TMEM lane m (M = 128) or lane
    // (m % 16) + 32 (m / 16) (M = 64); warp w reads lane quadrant w % 4.
    const int q = warp & 3;
    const int m = a.M == 128 ? q * 32 + lane : (lane < 16 ? q * 16 + lane : -1);
    const int ci = cbk * a.cib + m;
    const bool row_ok = m >= 0 && m < a.cib;
    const uint32_t trow = tmem + ((uint32_t)(q * 32) << 16);
    const int nacc = a.stack ? 3 : a.G;
    const int sub = (warp - kWtI) >> 2;  // the 2 kWtW / 4 warps of a quadrant take 8-column chunks in turn
    int chunk = 0;
    for (int i = 0; i < nacc; ++i) {
      for (int blk = 0; blk < (a.stack ? 3 : 1); ++blk) {
        // stacked: TMEM block blk of accumulator i is tap (kd, kh = i, kw = 2 - blk)
        const int t = a.ntaps == 27 ? (a.stack ? t0 + 3 * i + (2 - blk) : t0 + i) : 0;
        float* dst = pb + ((long long)t * Cin + ci) * Cout;
        const int cb = a.stack ? blk * 32 : 0, cw = a.stack ? 32 : a.N;
        for (int c0 = 0; c0 < cw && c0 < ((Cout + 7) & ~7); c0 += 8) {
          if ((chunk++) % (2 * kWtW / 4) != sub) continue;
          float v[8];
          tc::tmem_ld8(trow + (uint32_t)(i * a.N + cb + c0), v);
          if (row_ok) {
            if ((Cout & 7) == 0 && (reinterpret_cast<uintptr_t>(pb) & 15) == 0) {  // 32 contiguous bytes per row: two 16-byte stores
              const bool z = S <= 0;
              float4* d4 = reinterpret_cast<float4*>(dst + c0);
              d4[0] = z ? make_float4(0.f, 0.f, 0.f, 0.f) : make_float4(v[0], v[1], v[2], v[3]);
              d4[1] = z ? make_float4(0.f, 0.f, 0.f, 0.f) : make_float4(v[4], v[5], v[6], v[7]);
            } else {
#pragma unroll
              for (int j = 0; j < 8; ++j)
                if (c0 + j < Cout) dst[c0 + j] = S > 0 ? v[j] : 0.f;
            }
          }
        }
      }
    }
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_free(tmem, a.tmem_cols);
}

// Packed variant (a.pack): see the header. Same ring / barrier protocol as
// wgrad_tc_k; the producers gather 16-channel half lines.
__global__ void __launch_bounds__(kWtThreads) wgrad_tc_pack_k(WgTc a) {
  D2IP_PDL_ENTRY();
  extern __shared__ __align__(1024) uint8_t smem[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int b = blockIdx.z;
  const int rg = blockIdx.x;
  const int kd = blockIdx.y;  // one kd plane per CTA
  const bool do_bias = kd == 0;
  const int RS = a.RS, NSTG = a.NSTG;
  const int NX = RS + 2 * a.Sw, NG = RS + 3;  // rowmap entries: x window, gy window
  const d2ip_act x = a.x, gy = a.gy;
  const float* xb = x.ptr + b * x.bstride;
  const float* gb = gy.ptr + b * gy.bstride;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)NSTG * a.Sb);
  uint64_t* empty = full + NSTG;
  uint64_t* done = empty + NSTG;
  uint8_t* tail = smem + (size_t)NSTG * a.Sb + (((2 * NSTG + 1) * 8 + 15) & ~15);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(tail);
  float4* bred = reinterpret_cast<float4*>(tail + 16);
  int* rowmaps = reinterpret_cast<int*>(tail + 16 + kWtProd * 16);

  if (warp == 0) tc::tmem_alloc(tslot, a.tmem_cols);
  if (tid == 0) {
    for (int i = 0; i < NSTG; ++i) {
      tc::mbar_init(&full[i], kWtProd / 2);
      tc::mbar_init(&empty[i], 1);
    }
    tc::mbar_init(done, 1);
    tc::fence_mbar_init();
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = *tslot;
  const int c_lo = rg * a.chunks_per_rg, c_hi = min(a.nchunk, c_lo + a.chunks_per_rg);
  const int S = c_hi - c_lo;
  const int Cin = x.c, Cout = gy.c;
  float* pb = a.part + ((long long)b * a.nrg + rg) * ((long long)27 * Cin * Cout + Cout);

  if (warp < kWtI) {
    if (warp == 0 && lane == 0) {  // one accumulator: one issuer
      const uint32_t sbase = tc::smem_u32(smem);
      const uint64_t dXhi = tc::make_desc_mn32(sbase, a.lbox), dXlo = dXhi + (a.Sx >> 4);
      const uint64_t dGhi = tc::make_desc_mn32(sbase + 2 * a.Sx, a.lbog), dGlo = dGhi + (a.Sg >> 4);
      for (int s = 0; s < S; ++s) {
        const int slot = s % NSTG;
        tc::mbar_wait(&full[slot], (uint32_t)((s / NSTG) & 1));
        tc::fence_after();
        const uint64_t boff = (uint64_t)(slot * a.Sb) >> 4;
        for (int j = 0; j < RS / 8; ++j) {
          const uint64_t o = boff + (uint64_t)(8 * j) * 8;
          const uint32_t first = (s | j) ? 1u : 0u;
          tc::mma_tf32(tmem, dXlo + o, dGhi + o, a.idesc, first);
          tc::mma_tf32(tmem, dXhi + o, dGlo + o, a.idesc, 1u);
          tc::mma_tf32(tmem, dXhi + o, dGhi + o, a.idesc, 1u);
        }
        tc::commit(&empty[slot]);
      }
      if (S > 0) tc::commit(done);
    }
  } else {
    const int ptid = tid - 32 * kWtI, pg = (warp - kWtI) / kWtW, gtid = ((warp - kWtI) % kWtW) * 32 + lane;
    const int xshift = (kd - 1) * a.Sh - a.Sw;
    int* rm = rowmaps + pg * (NX + NG);
    const int nchx = Cin / 4, nchg = Cout / 4;
    float4 bacc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int s = pg; s < S; s += 2) {
      const int slot = s % NSTG;
      if (s >= NSTG) tc::mbar_wait(&empty[slot], (uint32_t)((s / NSTG - 1) & 1));
      const int u0 = a.u_first + (c_lo + s) * RS;
      for (int i = gtid; i < NX + NG; i += 32 * kWtW)
        rm[i] = i < NX ? wg_voxel(a, u0 + xshift + i) : wg_voxel(a, u0 - 2 + (i - NX));
      asm volatile("bar.sync %0, %1;" ::"r"(1 + pg), "n"(32 * kWtW) : "memory");
      uint8_t* X = smem + (size_t)slot * a.Sb;
      uint8_t* Gt = X + 2 * a.Sx;
      // x: slot c = 4 (3 halves: block 0 lo / hi half, block 1 lo half) x chunk; kh = c / 4
      for (int i = gtid; i < RS * 16; i += 32 * kWtW) {
        const int r = i >> 4, c = i & 15, kh = c >> 2, cc = c & 3;
        if (kh < 3 && cc < nchx) {
          const int v = rm[r + kh * a.Sw];
          const float* src = v >= 0 ? xb + (long long)v * x.cstride + 4 * cc : xb;
          tc::cp_async16(X + mn32_off(r, (kh & 1) * 4 + cc + (kh >> 1) * 8, a.Bx), src, v >= 0 ? 16u : 0u);
        }
      }
      // gy line j = [gy(u0 - 1 + j) | gy(u0 - 2 + j)]
      for (int i = gtid; i < (RS + 2) * 8; i += 32 * kWtW) {
        const int j = i >> 3, h = (i >> 2) & 1, cc = i & 3;
        if (cc < nchg) {
          const int v = rm[NX + j + 1 - h];
          const float* src = v >= 0 ? gb + (long long)v * gy.cstride + 4 * cc : gb;
          tc::cp_async16(Gt + mn32_off(j, h * 4 + cc, a.Bg), src, v >= 0 ? 16u : 0u);
        }
      }
      tc::cp_async_commit();
      tc::cp_async_wait<0>();
      for (int i = gtid; i < RS * 16; i += 32 * kWtW) {
        const int r = i >> 4, c = i & 15, kh = c >> 2, cc = c & 3;
        if (kh < 3 && cc < nchx) {
          const uint32_t o = mn32_off(r, (kh & 1) * 4 + cc + (kh >> 1) * 8, a.Bx);
          const float4 v = *reinterpret_cast<const float4*>(X + o);
          float4 l;
          l.x = v.x - tf32_hi_w(v.x); l.y = v.y - tf32_hi_w(v.y); l.z = v.z - tf32_hi_w(v.z); l.w = v.w - tf32_hi_w(v.w);
          *reinterpret_cast<float4*>(X + a.Sx + o) = l;
        }
      }
      for (int i = gtid; i < (RS + 2) * 8; i += 32 * kWtW) {
        const int j = i >> 3, h = (i >> 2) & 1, cc = i & 3;
        if (cc < nchg) {
          const uint32_t o = mn32_off(j, h * 4 + cc, a.Bg);
          const float4 v = *reinterpret_cast<const float4*>(Gt + o);
          float4 l;
          l.x = v.x - tf32_hi_w(v.x); l.y = v.y - tf32_hi_w(v.y); l.z = v.z - tf32_hi_w(v.z); l.w = v.w - tf32_hi_w(v.w);
          *reinterpret_cast<float4*>(Gt + a.Sg + o) = l;
          if (do_bias && h == 0 && j >= 1 && j <= RS) {  // gy rows u0 .. u0 + RS - 1, once each
            bacc.x += v.x; bacc.y += v.y; bacc.z += v.z; bacc.w += v.w;
          }
        }
      }
      tc::fence_proxy_async();
      tc::mbar_arrive(&full[slot]);
      asm volatile("bar.sync %0, %1;" ::"r"(1 + pg), "n"(32 * kWtW) : "memory");
    }
    if (do_bias) bred[ptid] = bacc;
  }
  __syncthreads();
  if (warp >= kWtI) {
    const int ptid = tid - 32 * kWtI;
    if (do_bias && ptid < Cout / 4) {  // fixed-order column sum: thread q held chunk q % 4 (h == 0 slots)
      float4 sum = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int q = 0; q < kWtProd; ++q) {
        if ((q & 7) != ptid) continue;  // gtid % 8 == h * 4 + cc with h == 0
        const float4 v = bred[q];
        sum.x += v.x; sum.y += v.y; sum.z += v.z; sum.w += v.w;
      }
      float* o = pb + (long long)27 * Cin * Cout + 4 * ptid;
      o[0] = sum.x; o[1] = sum.y; o[2] = sum.z; o[3] = sum.w;
    }
    if (S > 0) {
      tc::mbar_wait(done, 0);
      tc::fence_after();
    }
    // D row m = 16 kh + ci in TMEM lane (m % 16) + 32 (m / 16): quadrant q = kh
    const int q = warp & 3, ci = lane;
    if (q < 3 && warp >= 4 && warp <= 6) {  // one warp per quadrant (kh) drains it
      const uint32_t trow = tmem + ((uint32_t)(q * 32) << 16);
      for (int c0 = 0; c0 < 64; c0 += 8) {
        const int blk = c0 >> 4 >> 1, h = (c0 >> 4) & 1, co0 = c0 & 15;
        if ((blk == 0 && h == 1) || co0 >= Cout) continue;
        const int kw = blk == 0 ? 2 : h;
        float v[8];
        tc::tmem_ld8(trow + (uint32_t)c0, v);
        if (ci < Cin && lane < 16) {
          float* dst = pb + ((long long)(kd * 9 + q * 3 + kw) * Cin + ci) * Cout + co0;
          if ((Cout & 7) == 0 && (reinterpret_cast<uintptr_t>(pb) & 15) == 0) {
            const bool z = S <= 0;
            float4* d4 = reinterpret_cast<float4*>(dst);
            d4[0] = z ? make_float4(0.f, 0.f, 0.f, 0.f) : make_float4(v[0], v[1], v[2], v[3]);
            d4[1] = z ? make_float4(0.f, 0.f, 0.f, 0.f) : make_float4(v[4], v[5], v[6], v[7]);
          } else {
#pragma unroll
            for (int jj = 0; jj < 8; ++jj)
              if (co0 + jj < Cout) dst[jj] = S > 0 ? v[jj] : 0.f;
          }
        }
      }
    }
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_free(tmem, a.tmem_cols);
}

// Sum over row groups (fixed order) and scatter into OIDHW weight + bias grads.
// Thread e walks the partial layout [t][ci][co] (co fastest: coalesced reads).
__global__ void __launch_bounds__(256) wgrad_tc_reduce_k(const float* __restrict__ part, int nrg, int ntaps,
                                                         int Cin, int Cout, float* __restrict__ out, long long obs) {
  D2IP_PDL_ENTRY();
  const int b = blockIdx.y;
  const long long nw = (long long)ntaps * Cin * Cout, n = nw + Cout;
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n) return;
  const float* p = part + (long long)b * nrg * n + e;
  // four interleaved partial sums, four loads in flight (fixed order: row group r -> sum r % 4)
  float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
  int r = 0;
  for (; r + 3 < nrg; r += 4) {
    const float a0 = __ldg(p + (long long)r * n), a1 = __ldg(p + (long long)(r + 1) * n);
    const float a2 = __ldg(p + (long long)(r + 2) * n), a3 = __ldg(p + (long long)(r + 3) * n);
    s0 += a0;
    s1 += a1;
    s2 += a2;
    s3 += a3;
  }
  for (; r < nrg; ++r) s0 += __ldg(p + (long long)r * n);
  const float s = (s0 + s1) + (s2 + s3);
  long long o;
  if (e < nw) {
    const int co = (int)(e % Cout);
    const long long q = e / Cout;
    const int ci = (int)(q % Cin), t = (int)(q / Cin);
    o = ((long long)co * Cin + ci) * ntaps + t;
  } else {
    o = nw + (e - nw);
  }
  out[b * obs + o] = s;
}

static int pow2_at_least(int v) {
  int p = 1;
  while (p < v) p *= 2;
  return p;
}

static uint32_t align1k(size_t v) { return (uint32_t)((v + 1023) & ~(size_t)1023); }

static bool wt_nopack() {
  static const int v = [] {
    const char* e = getenv("D2IP_WGRAD_NOPACK");
    return e && *e == '1' ? 1 : 0;
  }();
  return v;
}

// Knobs for the side-lane scheduling study: shared memory per CTA (D2IP_WG_SMEM_KB, default 220)
// and CTAs per launch (D2IP_WG_CTAS, default 100: with sixteen producer warps per CTA fewer,
// longer row groups win -- cfg2 / cfg1 it/s at 222: 450 / 1,501, 148: 455 / 1,535, 100: 458 / 1,580,
// 74: 460 / 1,556). A weight-gradient CTA that fills an SM's shared memory keeps the
// data-gradient chain's CTAs off that SM while it runs.
static size_t wt_smem_cap() {
  static const size_t v = [] {
    const char* e = getenv("D2IP_WG_SMEM_KB");
    return (size_t)(e ? atoi(e) : 220) * 1024;
  }();
  return v;
}
static long long wt_cta_target() {
  static const long long v = [] {
    const char* e = getenv("D2IP_WG_CTAS");
    return e ? atoll(e) : 100LL;
  }();
  return v;
}

static bool wt_plan(int D, int H, int W, int Cin, int Cout, int ks, int batch, WgTc& a) {
  if (Cin % 4 || Cout % 4 || Cin < 4 || Cout > 128 || (ks != 1 && ks != 3)) return false;
  a.ntaps = ks == 3 ? 27 : 1;
  a.Sw = W + 2;
  a.Sh = (H + 2) * a.Sw;
  a.u_first = a.Sh + a.Sw + 1;
  a.u_last = D * a.Sh + H * a.Sw + W;
  // input-channel block: <= 128, equal blocks, multiple of 4
  a.ncib = (Cin + 127) / 128;
  while (Cin % a.ncib || (Cin / a.ncib) % 4) ++a.ncib;
  a.cib = Cin / a.ncib;
  a.M = a.cib <= 64 ? 64 : 128;
  a.pack = (ks == 3 && Cin <= 16 && Cout <= 16 && !wt_nopack()) ? 1 : 0;
  if (a.pack) {
    a.stack = 0;
    a.M = a.N = 64;
    a.G = 9;
    a.ngroups = 3;
    a.tmem_cols = 64;
    a.nchx = Cin / 4;
    a.nchg = Cout / 4;
    a.RS = 0;
    for (int rs : {128, 64, 32}) {
      const uint32_t bx = align1k((size_t)rs * 128), bg = align1k((size_t)(rs + 2) * 128);
      const uint32_t sx = 2 * bx, sg = bg, sb = 2 * (sx + sg);
      const int nx = rs + 2 * a.Sw, ng = rs + 3;
      auto total = [&](int nst) {
        return (size_t)nst * sb + (((2 * nst + 1) * 8 + 15) & ~15) + 16 + kWtProd * 16 + 8 * (size_t)(nx + ng) + 64;
      };
      if (total(2) > wt_smem_cap()) continue;
      a.NSTG = 2;
      while (a.NSTG < 4 && total(a.NSTG + 1) <= wt_smem_cap()) ++a.NSTG;
      a.RS = rs;
      a.WR = nx;
      a.RSg = ng;
      a.Bx = bx;
      a.Bg = bg;
      a.Sx = sx;
      a.Sg = sg;
      a.Sb = sb;
      a.pad = 0;
      a.lbox = bx;
      a.lbog = 256;  // N block 1 = two gy lines on
      break;
    }
    if (!a.RS) return false;
  } else {
  a.stack = (ks == 3 && Cout <= 32) ? 1 : 0;
  if (a.stack) {
    a.N = 96;  // 3 kw taps x one 32-channel block
    a.G = 9;   // one kd plane: 3 accumulators of 96 columns
  } else {
    a.N = (Cout + 15) / 16 * 16;
    if (a.M == 64 && Cout <= 8) a.N = 8;
    // taps per CTA: as many of a kd plane as fit 512 TMEM columns
    a.G = ks == 1 ? 1 : (9 * a.N <= 512 ? 9 : (3 * a.N <= 512 ? 3 : 1));
  }
  a.ngroups = a.ntaps / a.G;
  a.tmem_cols = std::max(32, pow2_at_least((a.stack ? 3 : a.G) * a.N));
  if (a.tmem_cols > 512) return false;
  a.nchx = a.cib / 4;
  a.nchg = Cout / 4;
  const int nbx = (a.cib + 31) / 32, nbg = (Cout + 31) / 32;  // real 32-channel blocks
  const int mbx = a.M / 32;                                    // blocks the MMA reads
  // rows per stage and ring depth: the largest rows per stage with >= 2 stages
  // (+ read pad) in 220 KB, then as many stages (<= 4) as fit
  a.RS = 0;
  for (int rs : {128, 64, 32}) {
    const int wr = ks == 3 ? rs + 2 * a.Sw + (a.stack ? 0 : 2) : rs;
    const int rsg = rs + 2 * a.stack;
    // block strides stay multiples of 512 B so a row's swizzle phase (address bits 7-8) is r % 4 in every block
    const uint32_t bx = align1k((size_t)wr * 128), bg = align1k((size_t)rsg * 128);
    const uint32_t sx = align1k((size_t)nbx * bx), sg = align1k((size_t)nbg * bg);
    const uint32_t sb = 2 * (sx + sg);
    // one real block is read with LBO = 0; otherwise the MMA runs mbx - nbx blocks past the x lo region
    const uint32_t pad = (nbx == 1 || nbx == mbx) ? 0 : align1k((size_t)(mbx - nbx) * bx);
    const size_t total = 2 * (size_t)sb + pad + 64 + kWtProd * 16 + 8 * (size_t)(wr + rsg) + 64;
    if (total <= wt_smem_cap()) {
      a.NSTG = 2;
      while (a.NSTG < 4 && (size_t)(a.NSTG + 1) * sb + pad + 128 + kWtProd * 16 + 8 * (size_t)(wr + rsg) + 64 <=
                               wt_smem_cap())
        ++a.NSTG;
      a.RS = rs;
      a.RSg = rsg;
      a.WR = wr;
      a.Bx = bx;
      a.Bg = bg;
      a.Sx = sx;
      a.Sg = sg;
      a.Sb = sb;
      a.pad = pad;
      a.lbox = nbx == 1 ? 0 : bx;
      a.lbog = a.stack ? 128 : (nbg == 1 ? 0 : bg);
      break;
    }
  }
  if (!a.RS) return false;
  }
  a.nchunk = cdiv(a.u_last - a.u_first + 1, a.RS);
  // row groups: ~1 CTA per SM overall, >= 2 chunks each when there are enough
  const long long jobs = (long long)a.ngroups * a.ncib * batch;
  int nrg = (int)std::max(1LL, (wt_cta_target() + jobs - 1) / jobs);
  nrg = std::min(nrg, std::max(1, a.nchunk / 2));
  a.chunks_per_rg = cdiv(a.nchunk, nrg);
  a.nrg = cdiv(a.nchunk, a.chunks_per_rg);
  a.idesc = tc::make_idesc(2, a.M, a.N) | (1u << 15) | (1u << 16);  // A and B MN-major
  return true;
}

// stages, pad, barriers (2 NSTG + 1, padded to 16 B), TMEM slot (16 B), bias partials
static size_t wt_smem(const WgTc& a) {
  return (size_t)a.NSTG * a.Sb + a.pad + (((2 * a.NSTG + 1) * 8 + 15) & ~15) + 16 + kWtProd * 16 +
         2 * (size_t)(a.WR + a.RSg) * sizeof(int) + 64;
}

// bf16 layers use it too until a kind::f16 weight-gradient kernel exists: 3xTF32
// is more accurate than the bf16 bar asks for.
bool wgrad_tc_supported(d2ip_act x, d2ip_act gy, int ks, int precision) {
  if (precision != D2IP_PREC_TF32 && precision != D2IP_PREC_BF16) return false;
  if (x.d != gy.d || x.h != gy.h || x.w != gy.w) return false;
  if (x.cstride % 4 || gy.cstride % 4 || ((uintptr_t)x.ptr & 15) || ((uintptr_t)gy.ptr & 15)) return false;
  WgTc a{};
  if (!wt_plan(x.d, x.h, x.w, x.c, gy.c, ks, 1, a)) return false;
  const int nchxp = pow2_at_least(a.nchx), nchgp = pow2_at_least(a.nchg);
  return nchxp <= 32 && nchgp <= 32 && (nchxp == 1 || nchxp == 2 || nchxp == 4 || nchxp == 8 || nchxp == 16 || nchxp == 32);
}

size_t wgrad_tc_ws_bytes(int D, int H, int W, int Cin, int Cout, int ks, int batch) {
  WgTc a{};
  if (!wt_plan(D, H, W, Cin, Cout, ks, batch, a)) return 0;
  return (size_t)batch * a.nrg * ((size_t)a.ntaps * Cin * Cout + Cout) * sizeof(float);
}

template <int NX, int NG>
static int wt_launch(const WgTc& a, dim3 grid, size_t smem, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    D2IP_CUDA(cudaFuncSetAttribute(wgrad_tc_k<NX, NG>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    attr = true;
  }
  D2IP_CUDA(launch_pdl((wgrad_tc_k<NX, NG>), grid, kWtThreads, smem, st, a));
  return D2IP_OK;
}

template <int NX>
static int wt_launch_g(const WgTc& a, int ng, dim3 grid, size_t smem, cudaStream_t st) {
  switch (ng) {
    case 1: return wt_launch<NX, 1>(a, grid, smem, st);
    case 2: return wt_launch<NX, 2>(a, grid, smem, st);
    case 4: return wt_launch<NX, 4>(a, grid, smem, st);
    case 8: return wt_launch<NX, 8>(a, grid, smem, st);
    case 16: return wt_launch<NX, 16>(a, grid, smem, st);
    case 32: return wt_launch<NX, 32>(a, grid, smem, st);
  }
  D2IP_CHECK_ARG(false, "wgrad_tc: C_out chunks %d unsupported", ng);
  return D2IP_E_ARG;
}

int wgrad_tc(d2ip_act x, d2ip_act gy, int ks, float* gw, long long gwbs, void* ws, size_t ws_bytes, int batch,
             cudaStream_t st) {
  WgTc a{};
  D2IP_CHECK_ARG(wt_plan(x.d, x.h, x.w, x.c, gy.c, ks, batch, a), "wgrad_tc: unsupported shape");
  D2IP_CHECK_ARG(ws_bytes >= wgrad_tc_ws_bytes(x.d, x.h, x.w, x.c, gy.c, ks, batch), "wgrad_tc: workspace too small");
  a.x = x;
  a.gy = gy;
  a.part = reinterpret_cast<float*>(ws);
  const size_t smem = wt_smem(a);
  const dim3 grid(a.nrg, a.ngroups * a.ncib, batch);
  if (a.pack) {
    static bool attr = false;
    if (!attr) {
      D2IP_CUDA(cudaFuncSetAttribute(wgrad_tc_pack_k, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
      attr = true;
    }
    D2IP_CUDA(launch_pdl(wgrad_tc_pack_k, grid, kWtThreads, smem, st, a));
  } else {
  const int nx = pow2_at_least(a.nchx), ng = pow2_at_least(a.nchg);
  switch (nx) {
    case 1: D2IP_RET(wt_launch_g<1>(a, ng, grid, smem, st)); break;
    case 2: D2IP_RET(wt_launch_g<2>(a, ng, grid, smem, st)); break;
    case 4: D2IP_RET(wt_launch_g<4>(a, ng, grid, smem, st)); break;
    case 8: D2IP_RET(wt_launch_g<8>(a, ng, grid, smem, st)); break;
    case 16: D2IP_RET(wt_launch_g<16>(a, ng, grid, smem, st)); break;
    case 32: D2IP_RET(wt_launch_g<32>(a, ng, grid, smem, st)); break;
    default: D2IP_CHECK_ARG(false, "wgrad_tc: C_in chunks %d unsupported", nx);
  }
  }
  D2IP_LAUNCH_CHECK();
  const long long n = (long long)a.ntaps * x.c * gy.c + gy.c;
  D2IP_CUDA(launch_pdl(wgrad_tc_reduce_k, dim3(cdiv(n, 256), batch), 256, 0, st, a.part, a.nrg, a.ntaps, x.c, gy.c,
                       gw, gwbs));
  D2IP_LAUNCH_CHECK();
  return D2IP_OK;
}

// Fixed-order sum of per-row-group partials [b][rg][ntaps][Cin][Cout] + [Cout]
// into OIDHW weight gradients + bias (also used by wgrad_bf.cu).
int wgrad_reduce(const float* part, int nrg, int ntaps, int Cin, int Cout, float* gw, long long gwbs, int batch,
                 cudaStream_t st) {
  const long long n = (long long)ntaps * Cin * Cout + Cout;
  D2IP_CUDA(launch_pdl(wgrad_tc_reduce_k, dim3(cdiv(n, 256), batch), 256, 0, st, part, nrg, ntaps, Cin, Cout, gw, gwbs));
  D2IP_LAUNCH_CHECK();
  return D2IP_OK;
}

}  // namespace d2ip
