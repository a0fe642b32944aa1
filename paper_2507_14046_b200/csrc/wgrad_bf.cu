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

#include <cuda_bf16.h>

#include "common.cuh"
#include "kernels.h"
#include "tc.cuh"

namespace d2ip {

constexpr int kWbThreads = 288;  // warp 0: MMA issue; warps 1-8: producers, then the epilogue
constexpr int kWbProd = 256;
constexpr int kWbMaxStages = 4;

struct WgBf {
  d2ip_act x, gy;
  int Sw, Sh, u_first, u_last;
  int ks, ntaps;
  int G, ngroups;     // taps per CTA, tap groups
  int cib, ncib;      // input channels per block, blocks
  int M, N;           // MMA shape
  int ngx, ngg;       // 8-channel group columns per stage: x (>= M / 8, the MMA reads M / 8), gy (N / 8)
  int RS, WR, WRp, RSp;  // rows per stage (K chunk), x window rows, padded column lengths
  int NST;            // ring depth
  int nchunk, chunks_per_rg, nrg;
  int tmem_cols;
  int gshift;         // log2(C_out / 4): float4 pieces per gy row
  uint32_t Sx, Sb;    // bytes: x region of a stage, whole stage
  uint32_t idesc;
  float* part;        // [b][rg][ntaps][Cin][Cout] + [Cout] bias
};

static inline int wb_pad(int rows) { return rows + ((1 - rows) % 8 + 8) % 8; }  // = 1 mod 8: spread banks

__device__ __forceinline__ uint32_t bf2w(float a, float b) {
  const __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<const uint32_t*>(&h);
}

// voxel offset of virtual row u in a (D, H, W) grid, -1 for padding rows
__device__ __forceinline__ int wb_voxel(const WgBf& a, int u, int D, int H, int W) {
  if (u < 0) return -1;
  const int dp = u / a.Sh, r = u - dp * a.Sh;
  const int hp = r / a.Sw, wp = r - hp * a.Sw;
  if (dp < 1 || dp > D || hp < 1 || hp > H || wp < 1 || wp > W) return -1;
  return ((dp - 1) * H + (hp - 1)) * W + (wp - 1);
}

// row offset of the CTA's x window (relative to the chunk's first gy row) and
// of tap q of the group inside it
__device__ __forceinline__ int wb_base(const WgBf& a, int grp) {
  if (a.ks == 1) return 0;
  if (a.G == 9) return (grp - 1) * a.Sh - a.Sw - 1;
  if (a.G == 3) return (grp / 3 - 1) * a.Sh + (grp % 3 - 1) * a.Sw - 1;
  return (grp / 9 - 1) * a.Sh + ((grp / 3) % 3 - 1) * a.Sw + (grp % 3 - 1);
}
__device__ __forceinline__ int wb_rel(const WgBf& a, int q) {
  if (a.G == 9) return (q / 3) * a.Sw + (q % 3);
  return q;  // G = 3: kw; G = 1: 0
}

template <int NCX>  // float4 pieces per x row = cib / 4
__global__ void __launch_bounds__(kWbThreads) wgrad_bf_k(WgBf a) {
  D2IP_PDL_ENTRY();
  extern __shared__ __align__(1024) uint8_t smem[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int rg = blockIdx.x;
  const int grp = blockIdx.y % a.ngroups, cb = blockIdx.y / a.ngroups;
  const int b = blockIdx.z;
  const int WR = a.WR, RS = a.RS, WRp = a.WRp, RSp = a.RSp, NST = a.NST;
  // layout: NST stages [x groups][gy groups], row maps [2][WR + RS], barriers, TMEM slot, bias scratch
  int* rmap = reinterpret_cast<int*>(smem + (size_t)NST * a.Sb);
  uint64_t* full = reinterpret_cast<uint64_t*>(rmap + 2 * (WR + RS) + ((2 * (WR + RS)) & 1));
  uint64_t* empty = full + kWbMaxStages;
  uint64_t* done = empty + kWbMaxStages;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(done + 1);
  float4* bscr = reinterpret_cast<float4*>((reinterpret_cast<uintptr_t>(tslot + 4) + 15) & ~(uintptr_t)15);

  if (warp == 0) tc::tmem_alloc(tslot, a.tmem_cols);
  if (tid == 0) {
    for (int i = 0; i < NST; ++i) {
      tc::mbar_init(&full[i], kWbProd);
      tc::mbar_init(&empty[i], 1);
    }
    tc::mbar_init(done, 1);
    tc::fence_mbar_init();
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = *tslot;
  const int c_lo = rg * a.chunks_per_rg;
  const int S = min(a.nchunk, c_lo + a.chunks_per_rg) - c_lo;  // this CTA's chunks
  const int base = wb_base(a, grp);
  const int Gq = a.G;

  if (warp == 0) {
    // ---- MMA issue: the whole warp walks the loop, one elected lane issues
    const uint32_t sbase = tc::smem_u32(smem);
    for (int s = 0; s < S; ++s) {
      const int slot = s % NST;
      tc::mbar_wait(&full[slot], (uint32_t)((s / NST) & 1));
      tc::fence_after();
      const uint32_t xs = sbase + slot * a.Sb, gs = xs + a.Sx;
      for (int k16 = 0; k16 < RS / 16; ++k16) {
        const uint64_t db = tc::make_desc(gs + k16 * 256, 128, RSp * 16);
        for (int q = 0; q < Gq; ++q) {
          const uint64_t da = tc::make_desc(xs + (k16 * 16 + wb_rel(a, q)) * 16, 128, WRp * 16);
          tc::mma_f16_warp(tmem + (uint32_t)(q * a.N), da, db, a.idesc, (s | k16) ? 1u : 0u);
        }
      }
      __syncwarp();
      if (lane == 0) tc::commit(&empty[slot]);
      __syncwarp();
    }
    if (lane == 0 && S > 0) tc::commit(done);
    __syncwarp();
  } else {
    // ---- producers
    const int gtid = tid - 32;
    const d2ip_act x = a.x, gy = a.gy;
    const float* xb = x.ptr + b * x.bstride + cb * a.cib;
    const float* gb = gy.ptr + b * gy.bstride;
    const int gmask = (1 << a.gshift) - 1;
    const bool do_bias = blockIdx.y == 0;
    float4 bsum = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int s = 0; s < S; ++s) {
      const int slot = s % NST;
      if (s >= NST) tc::mbar_wait(&empty[slot], (uint32_t)(((s / NST) - 1) & 1));
      const int u0 = a.u_first + (c_lo + s) * RS;
      int* rm = rmap + (s & 1) * (WR + RS);
      for (int r = gtid; r < WR + RS; r += kWbProd) {
        int off;
        if (r < WR) off = wb_voxel(a, u0 + base + r, x.d, x.h, x.w);
        else {
          const int u = u0 + (r - WR);
          off = u > a.u_last ? -1 : wb_voxel(a, u, gy.d, gy.h, gy.w);
        }
        rm[r] = off;
      }
      asm volatile("bar.sync 1, 256;" ::: "memory");
      uint8_t* X = smem + (size_t)slot * a.Sb;
      uint8_t* Gs = X + a.Sx;
      // x window: WR rows x NCX float4 pieces -> bf16 halves of 16-byte group rows
      constexpr int NP = NCX;
      const int nX = WR * NP;
      for (int i0 = gtid; i0 < nX; i0 += 8 * kWbProd) {
        float4 v[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const int i = i0 + q * kWbProd;
          v[q] = make_float4(0.f, 0.f, 0.f, 0.f);
          if (i < nX) {
            const int off = rm[i / NP];
            if (off >= 0) v[q] = *reinterpret_cast<const float4*>(xb + (long long)off * x.cstride + 4 * (i % NP));
          }
        }
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const int i = i0 + q * kWbProd;
          if (i >= nX) continue;
          const int r = i / NP, pc = i % NP;
          *reinterpret_cast<uint2*>(X + ((size_t)(pc >> 1) * WRp + r) * 16 + (pc & 1) * 8) =
              make_uint2(bf2w(v[q].x, v[q].y), bf2w(v[q].z, v[q].w));
        }
      }
      // gy rows: RS x (C_out / 4) pieces; the bias sum takes the fp32 values
      const int nG = RS << a.gshift;
      for (int i0 = gtid; i0 < nG; i0 += 8 * kWbProd) {
        float4 v[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const int i = i0 + q * kWbProd;
          v[q] = make_float4(0.f, 0.f, 0.f, 0.f);
          if (i < nG) {
            const int off = rm[WR + (i >> a.gshift)];
            if (off >= 0) v[q] = *reinterpret_cast<const float4*>(gb + (long long)off * gy.cstride + 4 * (i & gmask));
          }
        }
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const int i = i0 + q * kWbProd;
          if (i >= nG) continue;
          const int r = i >> a.gshift, pc = i & gmask;
          if (do_bias) {
            bsum.x += v[q].x; bsum.y += v[q].y; bsum.z += v[q].z; bsum.w += v[q].w;
          }
          *reinterpret_cast<uint2*>(Gs + ((size_t)(pc >> 1) * RSp + r) * 16 + (pc & 1) * 8) =
              make_uint2(bf2w(v[q].x, v[q].y), bf2w(v[q].z, v[q].w));
        }
      }
      tc::fence_proxy_async();
      tc::mbar_arrive(&full[slot]);
    }

    // ---- epilogue: TMEM -> per-row-group partials [t][ci][co]
    const int Cin = x.c, Cout = gy.c;
    float* pb = a.part + ((long long)b * a.nrg + rg) * ((long long)a.ntaps * Cin * Cout + Cout);
    if (S > 0) {
      tc::mbar_wait(done, 0);
      tc::fence_after();
    }
    const int quad = warp & 3, half = (warp - 1) >> 2;
    // M = 128: lane l holds row l; M = 64: rows at lanes (m % 16) + 32 (m / 16)
    int m = -1;
    if (a.M == 128) m = quad * 32 + lane;
    else if (lane < 16) m = quad * 16 + lane;
    const int ci = cb * a.cib + m;
    const bool live = m >= 0 && m < a.cib;
    const uint32_t trow = tmem + ((uint32_t)(quad * 32) << 16);
    const int nck = (Gq * a.N) / 8;
    for (int c = half; c < nck; c += 2) {
      float vals[8];
      tc::tmem_ld8(trow + (uint32_t)(c * 8), vals);
      const int q = (c * 8) / a.N, n = (c * 8) % a.N;
      if (!live || n >= Cout) continue;
      const int t = a.ks == 1 ? 0 : (Gq == 9 ? grp * 9 + q : Gq == 3 ? grp * 3 + q : grp);
      float4* dst = reinterpret_cast<float4*>(pb + ((long long)t * Cin + ci) * Cout + n);
      const bool z = S <= 0;
      dst[0] = z ? make_float4(0.f, 0.f, 0.f, 0.f) : make_float4(vals[0], vals[1], vals[2], vals[3]);
      dst[1] = z ? make_float4(0.f, 0.f, 0.f, 0.f) : make_float4(vals[4], vals[5], vals[6], vals[7]);
    }
    if (do_bias) {
      // fixed-order sum of the per-thread partials (thread gtid always held piece gtid % (C_out / 4))
      bscr[gtid] = bsum;
      asm volatile("bar.sync 1, 256;" ::: "memory");
      const int np = 1 << a.gshift;
      if (gtid < np) {
        float4 s4 = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int j = gtid; j < kWbProd; j += np) {
          const float4 v = bscr[j];
          s4.x += v.x; s4.y += v.y; s4.z += v.z; s4.w += v.w;
        }
        *reinterpret_cast<float4*>(pb + (long long)a.ntaps * Cin * Cout + 4 * gtid) = s4;
      }
    }
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_free(tmem, a.tmem_cols);
}

static size_t wb_smem(const WgBf& a) {
  return (size_t)a.NST * a.Sb + 2 * (size_t)(a.WR + a.RS) * sizeof(int) + 16 + (2 * kWbMaxStages + 1) * 8 + 16 +
         kWbProd * 16 + 64;
}

static bool pow2(int v) { return v > 0 && (v & (v - 1)) == 0; }

static bool wb_plan(int D, int H, int W, int Cin, int Cout, int ks, int batch, WgBf& a) {
  if ((ks != 1 && ks != 3) || Cout < 16 || Cout > 256 || !pow2(Cout) || Cin % 8 || Cin < 8) return false;
  a.ks = ks;
  a.ntaps = ks == 3 ? 27 : 1;
  a.Sw = W + 2;
  a.Sh = (H + 2) * a.Sw;
  a.u_first = a.Sh + a.Sw + 1;
  a.u_last = D * a.Sh + H * a.Sw + W;
  // input-channel block: <= 128 rows of the MMA; 96 fills an M = 128 MMA three quarters
  a.ncib = 1;
  while (Cin / a.ncib > 128 || Cin % a.ncib || (Cin / a.ncib) % 8) ++a.ncib;
  a.cib = Cin / a.ncib;
  const int ncx = a.cib / 4;
  if (ncx != 2 && ncx != 4 && ncx != 8 && ncx != 12 && ncx != 16 && ncx != 24 && ncx != 32) return false;
  a.M = a.cib <= 64 ? 64 : 128;
  a.N = Cout;
  a.G = ks == 1 ? 1 : (9 * a.N <= 512 ? 9 : (3 * a.N <= 512 ? 3 : 1));
  a.ngroups = a.ntaps / a.G;
  int cols = 32;
  while (cols < a.G * a.N) cols *= 2;
  a.tmem_cols = cols;
  a.ngx = std::max(a.cib / 8, a.M / 8);
  a.ngg = a.N / 8;
  a.gshift = 0;
  while ((4 << a.gshift) < Cout) ++a.gshift;
  const int halo = ks == 1 || a.G == 1 ? 0 : (a.G == 9 ? 2 * a.Sw + 2 : 2);
  const int rows = a.u_last - a.u_first + 1;
  a.RS = 0;
  // the largest chunk (amortises the x halo) that double-buffers in ~200 KB; then up to 4 stages
  for (int rs : {1024, 768, 512, 384, 256, 128, 64, 32, 16}) {
    if (rs > 16 && rs / 2 >= rows) continue;
    const int wr = rs + halo;
    const int wrp = wb_pad(wr), rsp = wb_pad(rs);
    const uint32_t sx = (uint32_t)a.ngx * wrp * 16, sb = ((sx + (uint32_t)a.ngg * rsp * 16) + 1023) & ~1023u;
    a.WR = wr;
    a.RS = rs;
    a.WRp = wrp;
    a.RSp = rsp;
    a.Sx = sx;
    a.Sb = sb;
    a.NST = 2;
    if (wb_smem(a) > (size_t)200 * 1024) {
      a.RS = 0;
      continue;
    }
    while (a.NST < 3 && (a.NST + 1) * (size_t)sb + wb_smem(a) - a.NST * (size_t)sb <= (size_t)200 * 1024) ++a.NST;
    break;
  }
  if (!a.RS) return false;
  a.nchunk = cdiv(rows, a.RS);
  // row groups: one wave of ~1 CTA per SM
  const long long jobs = (long long)a.ngroups * a.ncib * batch;
  int nrg = (int)std::max(1LL, 148LL / jobs);
  nrg = std::min(nrg, a.nchunk);
  a.chunks_per_rg = cdiv(a.nchunk, nrg);
  a.nrg = cdiv(a.nchunk, a.chunks_per_rg);
  a.idesc = tc::make_idesc(1, a.M, a.N) | (1u << 15) | (1u << 16);  // bf16, A and B MN-major
  return true;
}

bool wgrad_bf_supported(d2ip_act x, d2ip_act gy, int ks) {
  if (x.d != gy.d || x.h != gy.h || x.w != gy.w) return false;
  if (x.cstride % 4 || gy.cstride % 4 || ((uintptr_t)x.ptr & 15) || ((uintptr_t)gy.ptr & 15)) return false;
  WgBf a{};
  return wb_plan(x.d, x.h, x.w, x.c, gy.c, ks, 1, a);
}

size_t wgrad_bf_ws_bytes(int D, int H, int W, int Cin, int Cout, int ks, int batch) {
  WgBf a{};
  if (!wb_plan(D, H, W, Cin, Cout, ks, batch, a)) return 0;
  return (size_t)batch * a.nrg * ((size_t)a.ntaps * Cin * Cout + Cout) * sizeof(float);
}

template <int NCX>
static int wb_launch(const WgBf& a, dim3 grid, size_t smem, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    D2IP_CUDA(cudaFuncSetAttribute(wgrad_bf_k<NCX>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    attr = true;
  }
  D2IP_CUDA(launch_pdl(wgrad_bf_k<NCX>, grid, kWbThreads, smem, st, a));
  return D2IP_OK;
}

int wgrad_bf(d2ip_act x, d2ip_act gy, int ks, float* gw, long long gwbs, void* ws, size_t ws_bytes, int batch,
             cudaStream_t st) {
  WgBf a{};
  D2IP_CHECK_ARG(wb_plan(x.d, x.h, x.w, x.c, gy.c, ks, batch, a), "wgrad_bf: unsupported shape");
  D2IP_CHECK_ARG(ws_bytes >= wgrad_bf_ws_bytes(x.d, x.h, x.w, x.c, gy.c, ks, batch), "wgrad_bf: workspace too small");
  a.x = x;
  a.gy = gy;
  a.part = reinterpret_cast<float*>(ws);
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
  return wgrad_reduce(a.part, a.nrg, a.ntaps, x.c, gy.c, gw, gwbs, batch, st);
}

}  // namespace d2ip
