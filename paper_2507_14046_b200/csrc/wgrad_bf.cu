// K3 for bf16 layers: weight + bias gradient of the stride-1 3^3 / 1^3
// convolutions (autograd's conv backward w.r.t. weight/bias, pipeline.py:330)
// as tcgen05 kind::f16 MMAs with bf16 operands and FP32 accumulation in TMEM.
//
//   dW[co][ci][t] = sum_u x[u + off_t][ci] * gy[u][co],   db[co] = sum_u gy[u][co]
//
// GEMM view: M = input channels (a block of <= 128), N = output channels,
// K = rows u of the same virtual zero-padded grid as the forward kernel
// (conv_tc.cu), off_t = (kd-1) Sh + (kh-1) Sw + (kw-1). Both operands are
// MN-major: shared memory holds, per 8-channel group, a column of 16-byte rows
// (one bf16 row of 8 channels per u), so a tap is a move of the x descriptor's
// start address by off_t rows -- any row, 16 B granularity: no im2col, no
// shifted copies (tools/umma_mn_probe.cu: LBO = 128 B between 8-row K blocks,
// SBO = the group-column stride). The producers convert the fp32 activations
// and gradients to bf16 on the way into shared memory (one register pass).
//
// A CTA owns G taps -- a kd plane (9 taps, x window RS + 2 Sw + 2 rows), a
// (kd, kh) row (3 taps, RS + 2 rows) or one tap -- of one input-channel block,
// keeps G accumulators [M x N] in TMEM, and streams a contiguous range of row
// chunks (a row group) through an NST-deep ring: warp 0 issues the MMAs (one
// per tap per 16 rows), warps 1-8 fill stages and then drain TMEM into
// per-row-group partial sums, reduced in a fixed order by wgrad_reduce
// (deterministic, no atomics). The bias gradient is summed in fp32 from the
// unconverted gy values by the CTAs of tap group 0 / channel block 0.
#include <algorithm>
#include <cstdlib>

#include <cuda_bf16.h>

#include "common.cuh"
#include "kernels.h"
#include "tc.cuh"

namespace d2ip {

constexpr int kWbThreads = 288;  // warp 0: MMA issue; warps 1-8: producers, then the epilogue
constexpr int kWbProd = 256;
// 3xbf16: sixteen producer warps + one MMA-issue warp per independent accumulator (three for the kd-plane shape)
__host__ __device__ constexpr int wb_issuers(bool b3, int nkh) { return (b3 && nkh == 3) ? 3 : 1; }
__host__ __device__ constexpr int wb_threads(bool b3, int nkh) { return 32 * wb_issuers(b3, nkh) + 512; }
constexpr int kWbProd3 = 512;
constexpr int kWbMaxStages = 4;

struct WgBf {
  d2ip_act x, gy;
  int Sw, Sh, u_first, u_last;  // virtual grid with an 8-row-aligned pitch (Sw % 8 == 0)
  int v_start;        // first row of chunk 0 (8-aligned, <= u_first - 1)
  int ks, ntaps;
  int nkh;            // kh accumulators per CTA: 3 (a kd plane) or 1 (a (kd, kh) row); 1^3: 1
  int ngroups;        // tap groups (3 kd planes, 9 kd-kh rows, 1 for 1^3)
  int cib, ncib;      // input channels per block, blocks
  int M, N;           // MMA shape: N = 3 C_out (kw copies stacked) or C_out
  int nmma;           // MMAs per kh per 16 rows: 1 (N = 3 C_out) or 3 (one per kw copy, N = C_out); 1^3: 1
  int ncp;            // gy copies: 3 stacked kw-shifted copies (kd planes), or 1 unshifted copy of the
                      // map rows whose B descriptors start bsh0 + c * bstep rows in (a 16-byte move)
  int bsh0, bstep;    // single-copy B row shift of MMA c (kh rows: 2 - kw; one tap: 2 - kw; 1^3: 1)
  int tapmode;        // one tap per CTA (C_out = 256: a kh row of 3 x 256 columns exceeds TMEM)
  int s2;             // stride-2 3^3 layer by parity decomposition (see wb_s2_*): rows = the gy grid,
                      // the x window holds the two parity blocks (pw = 0, 1) of the CTA's (pd, ph)
  int mrows;          // real MMA rows (input channels of the block; C_in for stride 2)
  int carry;          // carry the x halo between stages (kd planes)
  int ngx, ngc;       // 8-channel group columns: x (real), gy per copy
  int RS, WR, WRp, RSp;  // rows per stage (K chunk), x window rows, padded column lengths
  int halo;           // x rows carried from the previous stage's window (2 Sw for kd planes)
  int NST;            // ring depth
  int nchunk, chunks_per_rg, nrg;
  int tmem_cols;
  int gshift;         // log2(C_out / 4): float4 pieces per gy row
  uint32_t Sx, Sb;    // bytes: x region of a stage (one half), whole stage
  uint32_t Sg;        // bytes: gy region (one half)
  int b3;             // 3xbf16: [x hi][x lo][gy hi][gy lo], three MMAs (lo*hi, hi*lo, hi*hi) per K step
  uint32_t pad;       // bytes after the last stage the M = 64 MMA may read past a small x block
  uint32_t idesc;
  int xtw, gtw;       // stream x / gy from their bf16 twins with cp.async (else fp32 loads + conversion)
  int nyb;            // bias partial slots per row group (= CTAs sharing it: tap groups x channel blocks)
  FastDiv fSh, fSw;   // row -> (plane, line, column) without integer division
  int dbg;            // D2IP_WB_DBG=1: producers skip the fills (measures the MMA side alone; wrong results)
  float* part;        // [b][rg][ntaps][Cin][Cout] + [nyb][Cout] bias
};

__device__ __forceinline__ void cp_async16_ca(void* dst_smem, const void* src, uint32_t src_bytes) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16, %2;" ::"r"(tc::smem_u32(dst_smem)), "l"(src),
               "r"(src_bytes)
               : "memory");
}

static inline int r8(int v) { return (v + 7) & ~7; }

// lo = bf16(x - hi) of four values whose bf16 hi pair is h (3xbf16 split)
__device__ __forceinline__ uint2 bf16_lo(const float4& v, uint2 h) {
  const float2 h0 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&h.x));
  const float2 h1 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&h.y));
  return make_uint2(bf16x2(v.x - h0.x, v.y - h0.y), bf16x2(v.z - h1.x, v.w - h1.y));
}

__device__ __forceinline__ uint32_t bf2w(float a, float b) {
  const __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<const uint32_t*>(&h);
}

// voxel offset of virtual row u in a (D, H, W) grid, -1 for padding rows
__device__ __forceinline__ int wb_voxel(const WgBf& a, int u, int D, int H, int W) {
  if (u < 0) return -1;
  const int dp = fdiv(u, a.fSh), r = u - dp * a.Sh;
  const int hp = fdiv(r, a.fSw), wp = r - hp * a.Sw;
  if (dp < 1 || dp > D || hp < 1 || hp > H || wp < 1 || wp > W) return -1;
  return ((dp - 1) * H + (hp - 1)) * W + (wp - 1);
}

// Row offset (from the chunk's first row v0) of the CTA's x window: tap
// (kd, kh, kw) pairs x row v + (kd-1) Sh + (kh-1) Sw with gy row v + 1 - kw
// (the kw shift lives in the gy copies), so the window starts at the kd plane's
// kh = 0 row (kd plane) or at the (kd, kh) row; always a multiple of 8.
// Stride 2: x = 2 o + k - 1 per axis, so tap k reads parity p = (k != 1) at
// output offset delta = (k == 0 ? -1 : 0). A CTA owns (kd, kh) (or one tap):
// its window rows start at delta_d Sh + delta_h Sw - 1 (delta_w = -1 is row 0),
// tap kw reads parity block pw = (kw != 1) at row offset 1 + delta_w.
__device__ __forceinline__ int wb_s2_delta(int k) { return k == 0 ? -1 : 0; }

__device__ __forceinline__ int wb_base(const WgBf& a, int grp) {
  if (a.s2) {
    const int kd = a.tapmode ? grp / 9 : grp / 3, kh = a.tapmode ? (grp / 3) % 3 : grp % 3;
    return wb_s2_delta(kd) * a.Sh + wb_s2_delta(kh) * a.Sw - 1;
  }
  if (a.ks == 1) return 0;
  if (a.tapmode) return (grp / 9 - 1) * a.Sh + ((grp / 3) % 3 - 1) * a.Sw;
  if (a.nkh == 3) return (grp - 1) * a.Sh - a.Sw;
  return (grp / 3 - 1) * a.Sh + (grp % 3 - 1) * a.Sw;
}

// NCX: float4 pieces per x row (cib / 4); NKH / NMMA: kh accumulators per CTA
// and MMAs per kh (compile-time, so the issue loop is a fixed run of MMAs on
// descriptors advanced by constant adds -- tools/umma_chains.cu measured a
// general per-MMA descriptor computation at ~140-390 cycles per MMA, against
// ~40 for the operand reads themselves).
template <int NCX, int NKH, int NMMA, bool B3>
__global__ void __launch_bounds__(wb_threads(B3, NKH)) wgrad_bf_k(WgBf a) {
  // Sixteen producer warps with eight loads in flight each. With eight the 3xbf16 variant (fp32
  // inputs converted and split on the way in: the weight gradients of large TF32-precision
  // layers) was bound by instruction latency at two warps per scheduler (ncu: 36 k instructions
  // per warp, issue active 29 %; 48->16 @ 64x64x32 150 -> 97 us), and the bf16 twin path gains
  // too (cfg4 139.8 -> 143.1 it/s). Measured and not kept: 24 warps (99 us), two producer groups
  // on alternate stages (105 us), two 9-warp CTAs per SM (141 us).
  constexpr int NPROD = kWbProd3;  // producer threads
  constexpr int UL = 8;                 // loads in flight per producer thread
  constexpr int NPG = 1, GP = NPROD / NPG;
  // MMA-issue warps: a single issuer pays >= 57 cycles per MMA whatever its size (the no-fill
  // run of this kernel, D2IP_WB_DBG=1, took 77 us of its 97); the kd-plane shape has three
  // independent accumulators (kh), so three warps issue one each
  constexpr int NI = wb_issuers(B3, NKH);  // producer groups, threads per group
  D2IP_PDL_ENTRY();
  extern __shared__ __align__(1024) uint8_t smem[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int rg = blockIdx.x;
  const int grp = blockIdx.y % a.ngroups, cb = blockIdx.y / a.ngroups;
  const int b = blockIdx.z;
  const int WR = a.WR, RS = a.RS, WRp = a.WRp, RSp = a.RSp, NST = a.NST;
  const int NM = RS + 2;  // gy row map: rows v0 - 1 .. v0 + RS
  // layout: NST stages [x groups][gy copies x groups] (+ pad), row maps [2][WR + NM], barriers, TMEM slot, bias scratch
  int* rmap = reinterpret_cast<int*>(smem + (size_t)NST * a.Sb + a.pad);
  uint64_t* full = reinterpret_cast<uint64_t*>(rmap + 4 * (WR + NM));  // row maps: [2][NPG <= 2][WR + NM]
  uint64_t* empty = full + kWbMaxStages;
  uint64_t* done = empty + kWbMaxStages;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(done + 1);
  float4* bscr = reinterpret_cast<float4*>((reinterpret_cast<uintptr_t>(tslot + 4) + 15) & ~(uintptr_t)15);

  if (warp == 0) tc::tmem_alloc(tslot, a.tmem_cols);
  if (tid == 0) {
    for (int i = 0; i < NST; ++i) {
      tc::mbar_init(&full[i], 2 * GP);  // async (copies landed) + plain (halo carry done) per thread
      tc::mbar_init(&empty[i], NI);
    }
    tc::mbar_init(done, NI);
    tc::fence_mbar_init();
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = *tslot;
  const int c_lo = rg * a.chunks_per_rg;
  const int S = min(a.nchunk, c_lo + a.chunks_per_rg) - c_lo;  // this CTA's chunks
  const int base = wb_base(a, grp);
  constexpr int nkh = NKH, nmma = NMMA;

  if (warp < NI) {
    // ---- MMA issue: one thread per issuing warp; descriptors advance by constant adds to the
    // start-address field (units of 16 B). Every operand block is 128-byte
    // aligned (8-row pitch, 8-aligned windows).
    if (lane == 0) {
      const uint32_t sbase = tc::smem_u32(smem);
      const uint64_t dA0 = tc::make_desc(sbase, 128, WRp * 16);
      const uint64_t dB0 = tc::make_desc(sbase + (B3 ? 2 : 1) * a.Sx, 128, RSp * 16);
      const uint32_t xlo16 = a.Sx >> 4, glo16 = a.Sg >> 4;  // B3: the lo halves
      const uint32_t cpy16 = ((uint32_t)a.ngc * RSp * 16) >> 4;  // one gy copy
      const uint32_t sw16 = (uint32_t)a.Sw;                       // one kh row: Sw rows x 16 B
      const uint32_t idesc = a.idesc, N = a.N;
      const bool stacked = a.ncp == 3;
      const int bsh = (a.tapmode && !a.s2) ? 2 - grp % 3 : a.bsh0;  // single copy: B starts bsh rows into the map rows
      // stride 2: MMA c (kw = c, or the CTA's one kw) reads parity block (kw != 1) from row 1 + delta_w
      uint32_t aoff[3] = {0u, 0u, 0u};
      if (a.s2)
        for (int c = 0; c < 3; ++c) {
          const int kw = a.tapmode ? grp % 3 : c;
          aoff[c] = (uint32_t)((kw != 1) * (a.mrows / 8) * WRp + 1 + wb_s2_delta(kw));
        }
      for (int s = 0; s < S; ++s) {
        const int slot = s % NST;
        tc::mbar_wait(&full[slot], (uint32_t)((s / NST) & 1));
        tc::fence_after();
        tc::fence_proxy_async();
        const uint64_t so = (uint64_t)((slot * a.Sb) >> 4);
        for (int k16 = 0; k16 < RS / 16; ++k16) {
          const uint64_t da = dA0 + so + (uint64_t)(k16 * 16), db = dB0 + so + (uint64_t)(k16 * 16);
          const uint32_t acc = (s | k16) ? 1u : 0u;  // (per accumulator: every issuer starts its own)
#pragma unroll
          for (int kh = (NI == 1 ? 0 : warp); kh < (NI == 1 ? NKH : warp + 1); ++kh)
#pragma unroll
            for (int c = 0; c < NMMA; ++c) {
              const uint32_t d = tmem + (uint32_t)(kh * NMMA + c) * N;
              const uint64_t aa = da + (uint64_t)(kh * sw16 + aoff[c]);
              const uint64_t bb = db + (uint64_t)(stacked ? c * cpy16 : bsh + c * a.bstep);
              if (B3) {
                tc::mma_f16(d, aa + xlo16, bb, idesc, acc);
                tc::mma_f16(d, aa, bb + glo16, idesc, 1u);
                tc::mma_f16(d, aa, bb, idesc, 1u);
              } else {
                tc::mma_f16(d, aa, bb, idesc, acc);
              }
            }
        }
        tc::commit(&empty[slot]);
      }
      if (S > 0) tc::commit(done);
    }
    __syncwarp();
  } else {
    // ---- producers: NPG groups of GP threads fill alternate stages (3xbf16: two groups, so the
    // load latency and row-map barrier of one stage overlap the conversion of the other)
    const int gtid = tid - 32 * NI;
    const int pg = gtid / GP, gt = gtid - pg * GP;
    const d2ip_act x = a.x, gy = a.gy;
    const float* xb = x.ptr + b * x.bstride + cb * a.cib;
    const float* gb = gy.ptr + b * gy.bstride;
    const int gmask = (1 << a.gshift) - 1;
    // the bias of chunk c is summed (fp32) by the CTA with blockIdx.y == c % nyb: balanced, fixed order
    const int ybias = blockIdx.y;
    const int ncp = a.ncp;
    const uint32_t cpy = (uint32_t)a.ngc * RSp * 16;
    float4 bsum = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int s = pg; s < S; s += NPG) {
      const int slot = s % NST;
      if (s >= NST) tc::mbar_wait(&empty[slot], (uint32_t)(((s / NST) - 1) & 1));
      if (a.dbg) {
        tc::mbar_arrive(&full[slot]);
        tc::mbar_arrive(&full[slot]);
        continue;
      }
      const int v0 = a.v_start + (c_lo + s) * RS;
      const bool carry = s > 0 && a.carry;  // first `halo` x rows = the previous window's last rows
      const int xr0 = carry ? a.halo : 0;
      int* rm = rmap + (((s / NPG) & 1) * NPG + pg) * (WR + NM);
      for (int r = gt; r < WR + NM; r += GP) {
        int off = -1;
        if (r < WR) {
          if (r >= xr0) {
            if (a.s2) {
              // (x voxel of (2 od + pd, 2 oh + ph, 2 ow)) << 1 | (2 ow + 1 inside); -1: none
              const int o = wb_voxel(a, v0 + base + r, gy.d, gy.h, gy.w);
              if (o >= 0) {
                const int kd = a.tapmode ? grp / 9 : grp / 3, kh = a.tapmode ? (grp / 3) % 3 : grp % 3;
                const int ow = o % gy.w, oh = (o / gy.w) % gy.h, od = o / (gy.w * gy.h);
                const int xd = 2 * od + (kd != 1), xh = 2 * oh + (kh != 1), xw = 2 * ow;
                if (xd < x.d && xh < x.h) off = (((xd * x.h + xh) * x.w + xw) << 1) | (xw + 1 < x.w);
              }
            } else {
              off = wb_voxel(a, v0 + base + r, x.d, x.h, x.w);
            }
          }
        } else {
          const int u = v0 - 1 + (r - WR);
          off = (u < a.u_first || u > a.u_last) ? -1 : wb_voxel(a, u, gy.d, gy.h, gy.w);
        }
        rm[r] = off;
      }
      asm volatile("bar.sync %0, %1;" ::"r"(2 + pg), "n"(GP) : "memory");
      uint8_t* X = smem + (size_t)slot * a.Sb;
      uint8_t* Gs = X + (B3 ? 2 : 1) * a.Sx;
      // x window rows [xr0, WR): NCX float4 pieces per row -> bf16 halves of 16-byte group rows
      constexpr int NP = NCX;
      const int nX = a.xtw ? 0 : (WR - xr0) * NP;
      if (a.xtw) {  // bf16 twin: one 16-byte async copy per (row, 8-channel group), zero-fill for padding rows
        const uint16_t* xt = reinterpret_cast<const uint16_t*>(x.bf16) + b * x.bstride + cb * a.cib;
        constexpr int NGX = NCX / 2;
        const int n16 = (WR - xr0) * NGX;
        for (int i = gt; i < n16; i += GP) {
          const int r = xr0 + i / NGX, g = i % NGX;
          const int off = rm[r];
          const uint16_t* src = xt;
          bool ok = off >= 0;
          if (a.s2) {  // group g of parity block g / (C_in / 8)
            const int gb = a.mrows / 8, bk = g / gb;
            ok = ok && (bk == 0 || (off & 1));
            if (ok) src = xt + (long long)((off >> 1) + bk) * x.cstride + 8 * (g - bk * gb);
          } else if (ok) {
            src = xt + (long long)off * x.cstride + 8 * g;
          }
          tc::cp_async16(X + ((size_t)g * WRp + r) * 16, src, ok ? 16u : 0u);
        }
      }
      for (int i0 = gt; i0 < nX; i0 += UL * GP) {
        float4 v[UL];
#pragma unroll
        for (int q = 0; q < UL; ++q) {
          const int i = i0 + q * GP;
          v[q] = make_float4(0.f, 0.f, 0.f, 0.f);
          if (i < nX) {
            const int off = rm[xr0 + i / NP];
            if (a.s2) {  // piece pc of parity block pc / (C_in / 4)
              const int pb = a.mrows / 4, pc = i % NP, bk = pc / pb;
              if (off >= 0 && (bk == 0 || (off & 1)))
                v[q] = *reinterpret_cast<const float4*>(xb + (long long)((off >> 1) + bk) * x.cstride + 4 * (pc - bk * pb));
            } else if (off >= 0) {
              v[q] = *reinterpret_cast<const float4*>(xb + (long long)off * x.cstride + 4 * (i % NP));
            }
          }
        }
#pragma unroll
        for (int q = 0; q < UL; ++q) {
          const int i = i0 + q * GP;
          if (i >= nX) continue;
          const int r = xr0 + i / NP, pc = i % NP;
          const uint2 h = make_uint2(bf2w(v[q].x, v[q].y), bf2w(v[q].z, v[q].w));
          *reinterpret_cast<uint2*>(X + ((size_t)(pc >> 1) * WRp + r) * 16 + (pc & 1) * 8) = h;
          if (B3) *reinterpret_cast<uint2*>(X + a.Sx + ((size_t)(pc >> 1) * WRp + r) * 16 + (pc & 1) * 8) = bf16_lo(v[q], h);
        }
      }
      // gy map rows m = 0 .. RS + 1 (row v0 - 1 + m); copy c row j = map row j + 2 - c
      // (1^3: one copy, row j = map row j + 1). The bias sum counts rows m = 1 .. RS once.
      const bool bias_here = (c_lo + s) % a.nyb == ybias;
      if (a.gtw) {  // bf16 twin: the kw copies are three async copies of the same 16 bytes (L1-allocating)
        const uint16_t* gtwin = reinterpret_cast<const uint16_t*>(gy.bf16) + b * gy.bstride;
        const int cs = a.gshift - 1;  // log2(C_out / 8): 8-channel groups per gy row
        const int n16 = NM << cs;
        for (int i = gt; i < n16; i += GP) {
          const int m = i >> cs, g = i & ((1 << cs) - 1);
          const int off = rm[WR + m];
          const uint16_t* src = off >= 0 ? gtwin + (long long)off * gy.cstride + 8 * g : gtwin;
          if (ncp == 1) {
            tc::cp_async16(Gs + ((size_t)g * RSp + m) * 16, src, off >= 0 ? 16u : 0u);
          } else {
            for (int c = 0; c < ncp; ++c) {
              const int j = m + c - 2;
              if (j >= 0 && j < RS) cp_async16_ca(Gs + c * cpy + ((size_t)g * RSp + j) * 16, src, off >= 0 ? 16u : 0u);
            }
          }
        }
      }
      const int nG = (!a.gtw || bias_here) ? NM << a.gshift : 0;
      for (int i0 = gt; i0 < nG; i0 += UL * GP) {
        float4 v[UL];
#pragma unroll
        for (int q = 0; q < UL; ++q) {
          const int i = i0 + q * GP;
          v[q] = make_float4(0.f, 0.f, 0.f, 0.f);
          if (i < nG) {
            const int off = rm[WR + (i >> a.gshift)];
            if (off >= 0) v[q] = *reinterpret_cast<const float4*>(gb + (long long)off * gy.cstride + 4 * (i & gmask));
          }
        }
#pragma unroll
        for (int q = 0; q < UL; ++q) {
          const int i = i0 + q * GP;
          if (i >= nG) continue;
          const int m = i >> a.gshift, pc = i & gmask;
          if (bias_here && m >= 1 && m <= RS) {
            bsum.x += v[q].x; bsum.y += v[q].y; bsum.z += v[q].z; bsum.w += v[q].w;
          }
          if (a.gtw) continue;  // fp32 pass for the bias only
          const uint2 o = make_uint2(bf2w(v[q].x, v[q].y), bf2w(v[q].z, v[q].w));
          const uint2 ol = B3 ? bf16_lo(v[q], o) : o;
          for (int c = 0; c < ncp; ++c) {
            const int j = ncp == 1 ? m : m + c - 2;
            if (j >= 0 && j < (ncp == 1 ? NM : RS)) {
              uint8_t* g = Gs + c * cpy + ((size_t)(pc >> 1) * RSp + j) * 16 + (pc & 1) * 8;
              *reinterpret_cast<uint2*>(g) = o;
              if (B3) *reinterpret_cast<uint2*>(g + a.Sg) = ol;
            }
          }
        }
      }
      // two arrivals per producer thread and stage: an async one when this
      // thread's copies have landed (no wait here: later stages' copies are
      // issued while these fly), and a plain one after the halo carry, which
      // first waits for the previous stage's window to land
      asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(tc::smem_u32(&full[slot])) : "memory");
      if (carry) {
        tc::mbar_wait(&full[(s - 1) % NST], (uint32_t)(((s - 1) / NST) & 1));
        // halo carry: x rows [RS, RS + halo) of the previous stage's window are rows [0, halo) of this one
        const uint8_t* Xp = smem + (size_t)((s - 1) % NST) * a.Sb;
        const int n16 = a.ngx * a.halo;
        for (int hl = 0; hl < (B3 ? 2 : 1); ++hl)  // B3: the hi and the lo window
          for (int i = gt; i < n16; i += GP) {
            const int g = i / a.halo, r = i - g * a.halo;
            *reinterpret_cast<uint4*>(X + hl * a.Sx + ((size_t)g * WRp + r) * 16) =
                *reinterpret_cast<const uint4*>(Xp + hl * a.Sx + ((size_t)g * WRp + RS + r) * 16);
          }
      }
      tc::fence_proxy_async();
      tc::mbar_arrive(&full[slot]);
    }

    // ---- epilogue: TMEM -> per-row-group partials [t][ci][co]
    const int Cin = x.c, Cout = gy.c;
    float* pb = a.part + ((long long)b * a.nrg + rg) * ((long long)a.ntaps * Cin * Cout + (long long)a.nyb * Cout);
    if (S > 0) {
      tc::mbar_wait(done, 0);
      tc::fence_after();
    }
    const int quad = warp & 3, half = (warp - NI) >> 2;  // column interleave over the NPROD / 128 warps of a quadrant
    // M = 128: lane l holds row l; M = 64: rows at lanes (m % 16) + 32 (m / 16)
    int m = -1;
    if (a.M == 128) m = quad * 32 + lane;
    else if (lane < 16) m = quad * 16 + lane;
    const int ci = cb * a.mrows + m;
    const bool live = m >= 0 && m < a.mrows;
    const uint32_t trow = tmem + ((uint32_t)(quad * 32) << 16);
    // accumulator columns: kh block of 3 C_out (kw copy c = kw, then co)
    const int nck = (nkh * 3 * Cout) / 8;
    const int nck_all = (a.ks == 1 || a.tapmode) ? Cout / 8 : nck;
    for (int c8 = half; c8 < nck_all; c8 += NPROD / 128) {
      float vals[8];
      tc::tmem_ld8(trow + (uint32_t)(c8 * 8), vals);
      const int col = c8 * 8;
      int t, n;
      if (a.ks == 1 || a.tapmode) {
        t = a.ks == 1 ? 0 : grp;
        n = col;
      } else {
        const int khl = col / (3 * Cout), rem = col - khl * 3 * Cout, kw = rem / Cout;
        n = rem - kw * Cout;
        const int kd = nkh == 3 ? grp : grp / 3, kh = nkh == 3 ? khl : grp % 3;
        t = kd * 9 + kh * 3 + kw;
      }
      if (!live) continue;
      float4* dst = reinterpret_cast<float4*>(pb + ((long long)t * Cin + ci) * Cout + n);
      const bool z = S <= 0;
      dst[0] = z ? make_float4(0.f, 0.f, 0.f, 0.f) : make_float4(vals[0], vals[1], vals[2], vals[3]);
      dst[1] = z ? make_float4(0.f, 0.f, 0.f, 0.f) : make_float4(vals[4], vals[5], vals[6], vals[7]);
    }
    {
      // fixed-order sum of the per-thread partials (thread gtid always held piece gtid % (C_out / 4)) into slot y
      bscr[gtid] = bsum;
      asm volatile("bar.sync 1, %0;" ::"n"(NPROD) : "memory");
      const int np = 1 << a.gshift;
      if (gtid < np) {
        float4 s4 = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int j = gtid; j < NPROD; j += np) {
          const float4 v = bscr[j];
          s4.x += v.x; s4.y += v.y; s4.z += v.z; s4.w += v.w;
        }
        *reinterpret_cast<float4*>(pb + (long long)a.ntaps * Cin * Cout + (long long)ybias * Cout + 4 * gtid) = s4;
      }
    }
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_free(tmem, a.tmem_cols);
}

static size_t wb_smem(const WgBf& a) {
  return (size_t)a.NST * a.Sb + a.pad + 4 * (size_t)(a.WR + a.RS + 2) * sizeof(int) + 16 +
         (2 * kWbMaxStages + 1) * 8 + 16 + kWbProd3 * 16 + 64;
}

static bool pow2(int v) { return v > 0 && (v & (v - 1)) == 0; }

// (D, H, W): the gy grid (the layer's output)
static bool wb_plan(int D, int H, int W, int Cin, int Cout, int ks, int batch, WgBf& a, int stride = 1,
                    bool b3 = false) {
  a.s2 = stride == 2;
  a.b3 = b3;
  if (a.s2 && (ks != 3 || Cin > 64)) return false;
  if ((ks != 1 && ks != 3) || Cout < 16 || Cout > 256 || !pow2(Cout) || Cin % 8 || Cin < 8) return false;
  a.ks = ks;
  a.ntaps = ks == 3 ? 27 : 1;
  a.Sw = r8(W + 2);  // 8-row pitch: every kh / kd shift keeps MMA operand blocks 128-byte aligned
  a.Sh = (H + 2) * a.Sw;
  a.u_first = a.Sh + a.Sw + 1;
  a.u_last = D * a.Sh + H * a.Sw + W;
  a.v_start = (a.u_first - 1) & ~7;
  // input-channel block: <= 128 rows of the MMA; 96 fills an M = 128 MMA three quarters
  a.ncib = 1;
  while (Cin / a.ncib > 128 || Cin % a.ncib || (Cin / a.ncib) % 8) ++a.ncib;
  a.cib = Cin / a.ncib;
  a.mrows = a.cib;
  if (a.s2) a.cib = 2 * Cin;  // the window holds two parity blocks
  const int ncx = a.cib / 4;
  if (ncx != 2 && ncx != 4 && ncx != 8 && ncx != 12 && ncx != 16 && ncx != 24 && ncx != 32) return false;
  a.M = a.mrows <= 64 ? 64 : 128;
  a.tapmode = 0;
  a.bstep = 0;
  a.bsh0 = 0;
  if (ks == 1) {
    a.nkh = 1;
    a.ngroups = 1;
    a.ncp = 1;
    a.nmma = 1;
    a.N = Cout;
    a.bsh0 = 1;  // map row m = row v0 - 1 + m
  } else if (a.s2) {
    a.nkh = 1;
    a.ncp = 1;
    a.bsh0 = 1;  // gy rows unshifted: map row m = row v0 - 1 + m
    a.N = Cout;
    if (3 * Cout <= 512) {
      a.nmma = 3;
      a.ngroups = 9;
    } else {
      a.nmma = 1;
      a.tapmode = 1;
      a.ngroups = 27;
    }
  } else if (9 * Cout <= 512) {
    // kd plane: three kh accumulators of 3 C_out columns, the kw copies stacked along N
    // (D2IP_WB_SINGLE=1: one gy copy, three MMAs per kh with B started 2 - kw rows in)
    static const bool single = [] {
      const char* v = getenv("D2IP_WB_SINGLE");
      return v && atoi(v) != 0;
    }();
    a.nkh = 3;
    a.ncp = single ? 1 : 3;
    a.nmma = single ? 3 : 1;
    a.N = single ? Cout : 3 * Cout;
    a.bsh0 = single ? 2 : 0;
    a.bstep = single ? -1 : 0;
    a.ngroups = 3;
  } else if (3 * Cout <= 512) {
    // (kd, kh) row: three MMAs (one per kw) on one gy copy, B started 2 - kw rows in
    a.nkh = 1;
    a.ncp = 1;
    a.nmma = 3;
    a.N = Cout;
    a.bsh0 = 2;
    a.bstep = -1;
    a.ngroups = 9;
  } else {
    a.nkh = 1;
    a.ncp = 1;
    a.nmma = 1;
    a.N = Cout;
    a.tapmode = 1;
    a.ngroups = 27;
  }
  int cols = 32;
  while (cols < a.nkh * a.nmma * a.N) cols *= 2;
  a.tmem_cols = cols;
  if (cols > 512) return false;
  a.ngx = a.cib / 8;
  a.ngc = Cout / 8;
  a.gshift = 0;
  while ((4 << a.gshift) < Cout) ++a.gshift;
  a.halo = (ks == 3 && a.nkh == 3) ? 2 * a.Sw : a.s2 ? 1 : 0;
  a.carry = ks == 3 && a.nkh == 3;
  const int rows = a.u_last + 2 - a.v_start;  // chunks cover v_start .. u_last + 1
  a.RS = 0;
  // the largest chunk that double-buffers in ~200 KB; then a third stage if it fits
  for (int rs : {1024, 768, 512, 384, 256, 192, 128, 64, 32, 16}) {
    if (rs > 16 && rs / 2 >= rows) continue;
    const int wr = rs + a.halo;
    const int wrp = r8(wr), rsp = r8(a.ncp == 1 ? rs + 2 : rs);  // single copy: all RS + 2 map rows
    const uint32_t sx = (uint32_t)a.ngx * wrp * 16, sg = (uint32_t)a.ncp * a.ngc * rsp * 16;
    const uint32_t sb = ((b3 ? 2 : 1) * (sx + sg) + 1023) & ~1023u;
    // the M = 64 / 128 MMA reads M / 8 group columns: past a smaller x block into the stage's gy copies or the pad
    const int blk1 = a.s2 ? a.mrows / 8 : 0;  // stride 2: the pw = 1 block's MMA reads start here
    // (B3: the lo window's reads start Sx further in)
    const long long over = (long long)(b3 ? sx : 0) + (long long)(blk1 + a.M / 8) * wrp * 16 - (long long)sb;
    a.pad = over > 0 ? (uint32_t)((over + 1023) & ~1023LL) : 0;
    a.WR = wr;
    a.RS = rs;
    a.WRp = wrp;
    a.RSp = rsp;
    a.Sx = sx;
    a.Sg = sg;
    a.Sb = sb;
    a.NST = 2;
    const size_t lim = (size_t)205 * 1024;
    if (wb_smem(a) > lim) {
      a.RS = 0;
      continue;
    }
    if (wb_smem(a) + sb <= lim) a.NST = 3;
    break;
  }
  if (!a.RS) return false;
  a.nchunk = cdiv(rows, a.RS);
  // row groups: one wave of ~1 CTA per SM
  const long long jobs = (long long)a.ngroups * a.ncib * batch;
  static const long long cta_target = [] {  // D2IP_WB_CTAS: CTAs per launch the row groups aim for
    const char* v = getenv("D2IP_WB_CTAS");
    return v ? atoll(v) : 148LL;
  }();
  int nrg = (int)std::max(1LL, cta_target / jobs);
  nrg = std::min(nrg, a.nchunk);
  a.chunks_per_rg = cdiv(a.nchunk, nrg);
  a.nrg = cdiv(a.nchunk, a.chunks_per_rg);
  a.idesc = tc::make_idesc(1, a.M, a.N) | (1u << 15) | (1u << 16);  // bf16, A and B MN-major
  a.nyb = a.ngroups * a.ncib;
  a.fSh = fastdiv((uint32_t)a.Sh);
  a.fSw = fastdiv((uint32_t)a.Sw);
  return a.Sh < (1 << 14) && a.u_last + 2 * a.Sh < (1 << 28);  // fdiv range
}

// dW[b] = sum_rg part[b][rg] (weights, [t][ci][co] -> OIDHW), db = sum_rg sum_y bias slots (fixed order)
__global__ void __launch_bounds__(256) wgrad_bf_reduce_k(const float* __restrict__ part, int nrg, int nyb, int ntaps,
                                                         int Cin, int Cout, float* __restrict__ out, long long obs) {
  D2IP_PDL_ENTRY();
  const int b = blockIdx.y;
  const long long nw = (long long)ntaps * Cin * Cout, blk = nw + (long long)nyb * Cout;
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= nw + Cout) return;
  const float* p = part + (long long)b * nrg * blk;
  float s = 0.f;
  if (e < nw) {
#pragma unroll 8
    for (int r = 0; r < nrg; ++r) s += __ldg(p + (long long)r * blk + e);
    const int co = (int)(e % Cout);
    const long long q = e / Cout;
    const int ci = (int)(q % Cin), t = (int)(q / Cin);
    out[b * obs + ((long long)co * Cin + ci) * ntaps + t] = s;
  } else {
    const int co = (int)(e - nw);
    const int n = nrg * nyb;  // (rg, y) slots in order; loads batched, adds in fixed order
#pragma unroll 8
    for (int q = 0; q < n; ++q) {
      const int r = q / nyb, y = q - r * nyb;
      s += __ldg(p + (long long)r * blk + nw + (long long)y * Cout + co);
    }
    out[b * obs + nw + co] = s;
  }
}

bool wgrad_bf_supported(d2ip_act x, d2ip_act gy, int ks, int stride, bool b3) {
  if (stride == 1 && (x.d != gy.d || x.h != gy.h || x.w != gy.w)) return false;
  if (stride == 2 && (gy.d != (x.d + 1) / 2 || gy.h != (x.h + 1) / 2 || gy.w != (x.w + 1) / 2)) return false;
  if (stride != 1 && stride != 2) return false;
  if (x.cstride % 4 || gy.cstride % 4 || ((uintptr_t)x.ptr & 15) || ((uintptr_t)gy.ptr & 15)) return false;
  WgBf a{};
  return wb_plan(gy.d, gy.h, gy.w, x.c, gy.c, ks, 1, a, stride, b3);
}

size_t wgrad_bf_ws_bytes(int D, int H, int W, int Cin, int Cout, int ks, int batch) {
  size_t best = 0;  // (D, H, W): the gy grid; the larger of the stride-1 and stride-2 plans
  for (int v = 0; v < 4; ++v) {  // stride 1 / 2, bf16 / 3xbf16
    WgBf a{};
    if (!wb_plan(D, H, W, Cin, Cout, ks, batch, a, 1 + (v & 1), v >= 2)) continue;
    best = std::max(best, (size_t)batch * a.nrg * ((size_t)a.ntaps * Cin * Cout + (size_t)a.nyb * Cout) * sizeof(float));
  }
  return best;
}

template <int NCX, int NKH, int NMMA, bool B3>
static int wb_launch4(const WgBf& a, dim3 grid, size_t smem, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    D2IP_CUDA(cudaFuncSetAttribute(wgrad_bf_k<NCX, NKH, NMMA, B3>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   227 * 1024));
    attr = true;
  }
  D2IP_CUDA(launch_pdl(wgrad_bf_k<NCX, NKH, NMMA, B3>, grid, wb_threads(B3, NKH), smem, st, a));
  return D2IP_OK;
}

template <int NCX, int NKH, int NMMA>
static int wb_launch3(const WgBf& a, dim3 grid, size_t smem, cudaStream_t st) {
  return a.b3 ? wb_launch4<NCX, NKH, NMMA, true>(a, grid, smem, st) : wb_launch4<NCX, NKH, NMMA, false>(a, grid, smem, st);
}

template <int NCX>
static int wb_launch(const WgBf& a, dim3 grid, size_t smem, cudaStream_t st) {
  if (a.nkh == 3 && a.nmma == 3) return wb_launch3<NCX, 3, 3>(a, grid, smem, st);
  if (a.nkh == 3) return wb_launch3<NCX, 3, 1>(a, grid, smem, st);
  if (a.nmma == 3) return wb_launch3<NCX, 1, 3>(a, grid, smem, st);
  return wb_launch3<NCX, 1, 1>(a, grid, smem, st);
}

int wgrad_bf(d2ip_act x, d2ip_act gy, int ks, float* gw, long long gwbs, void* ws, size_t ws_bytes, int batch,
             cudaStream_t st, int stride, bool b3) {
  WgBf a{};
  D2IP_CHECK_ARG(wb_plan(gy.d, gy.h, gy.w, x.c, gy.c, ks, batch, a, stride, b3), "wgrad_bf: unsupported shape");
  D2IP_CHECK_ARG(ws_bytes >= wgrad_bf_ws_bytes(gy.d, gy.h, gy.w, x.c, gy.c, ks, batch), "wgrad_bf: workspace too small");
  a.x = x;
  a.gy = gy;
  a.part = reinterpret_cast<float*>(ws);
  auto twin_ok = [](const d2ip_act& t, int c0) {
    return t.bf16 && t.cstride % 8 == 0 && c0 % 8 == 0 && ((uintptr_t)t.bf16 & 15) == 0;
  };
  a.xtw = !b3 && twin_ok(x, 0);  // (3xbf16 splits fp32 values: no twins)
  // D2IP_WB_CARRY=0: reload the x halo every stage instead of carrying it (no wait on the
  // previous stage's landing; 1.8x the x window bytes at cfg4's level 0)
  static const int carry_on = [] {
    const char* v = getenv("D2IP_WB_CARRY");
    return v ? atoi(v) : 1;
  }();
  if (!carry_on && a.carry) a.carry = 0;
  a.gtw = !b3 && twin_ok(gy, 0);
  static const int dbg = [] {
    const char* v = getenv("D2IP_WB_DBG");
    return v ? atoi(v) : 0;
  }();
  a.dbg = dbg;
  const size_t smem = wb_smem(a);
  const dim3 grid(a.nrg, a.ngroups * a.ncib, batch);
  switch (a.cib / 4) {
    case 2: D2IP_RET(wb_launch<2>(a, grid, smem, st)); break;
    case 4: D2IP_RET(wb_launch<4>(a, grid, smem, st)); break;
    case 8: D2IP_RET(wb_launch<8>(a, grid, smem, st)); break;
    case 12: D2IP_RET(wb_launch<12>(a, grid, smem, st)); break;
    case 16: D2IP_RET(wb_launch<16>(a, grid, smem, st)); break;
    case 24: D2IP_RET(wb_launch<24>(a, grid, smem, st)); break;
    case 32: D2IP_RET(wb_launch<32>(a, grid, smem, st)); break;
    default: D2IP_CHECK_ARG(false, "wgrad_bf: channel block %d unsupported", a.cib);
  }
  D2IP_LAUNCH_CHECK();
  const long long n = (long long)a.ntaps * x.c * gy.c + gy.c;
  D2IP_CUDA(launch_pdl(wgrad_bf_reduce_k, dim3(cdiv(n, 256), batch), 256, 0, st, a.part, a.nrg, a.nyb, a.ntaps, x.c,
                       gy.c, gw, gwbs));
  D2IP_LAUNCH_CHECK();
  return D2IP_OK;
}

}  // namespace d2ip
