// Issue-rate probe with independent accumulators: one thread issues tcgen05.mma
// round-robin into `nacc` TMEM accumulators (N columns each), so consecutive
// MMAs do not depend on each other. Separates the dependent-accumulate latency
// (umma_rate.cu: ~57 cycles for N <= 64) from the tensor pipe's throughput and
// the shared-memory operand bandwidth at small N.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2507_14046_b200/csrc -I include \
//        tools/umma_chains.cu -o tools/umma_chains
#include <cstdio>
#include "common.cuh"
#include "tc.cuh"
using namespace d2ip;

// One MMA issued by an elected lane of a fully converged warp: the whole warp
// computes the (uniform) operands, so they live in uniform registers.
template <bool F16>
__device__ __forceinline__ void mma_elect(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  if (F16)
    asm volatile(
        "{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc));
  else
    asm volatile(
        "{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

// nw issuing warps, warp w into its own NACC accumulators; MODE 0: lane 0
// issues (divergent branch), MODE 1: the whole warp runs the loop and an
// elect.sync inside the asm picks the issuing lane.
template <bool F16, int NACC, int MODE>
__global__ void chains_k(int M, int N, int nmma, int nw, long long* cycles, int mn) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* mbar = reinterpret_cast<uint64_t*>(smem + 65536);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(mbar + 4);
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<float*>(smem)[i] = 0.0f;
  if (threadIdx.x < 32) tc::tmem_alloc(tslot, 512);
  if (threadIdx.x == 0) { for (int i = 0; i < 4; ++i) tc::mbar_init(mbar + i, 1); tc::fence_mbar_init(); }
  tc::fence_proxy_async();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = *tslot;
  const int warp = __shfl_sync(0xffffffffu, threadIdx.x >> 5, 0);
  long long t0 = clock64();
  const bool issuer = MODE == 1 ? warp < nw : (warp < nw && (threadIdx.x & 31) == 0);
  if (issuer) {
    // mn: operands MN-major (LBO = 128 B between 8-row K blocks, SBO = 2 KB between 8-element groups)
    const uint32_t idesc = tc::make_idesc(F16 ? 1 : 2, M, N) | (mn ? (1u << 15) | (1u << 16) : 0u);
    const uint32_t sb = tc::smem_u32(smem);
    const uint64_t da = mn ? tc::make_desc(sb, 128, 2048) : tc::make_desc(sb, 2048, 128);
    const uint64_t db = mn ? tc::make_desc(sb + 32768, 128, 2048) : tc::make_desc(sb + 32768, 2048, 128);
    const uint32_t dbase = tmem + (uint32_t)(warp * NACC * N);
#pragma unroll
    for (int a = 0; a < NACC; ++a) {
      if (MODE == 1) mma_elect<F16>(dbase + a * N, da, db, idesc, 0u);
      else if (F16) tc::mma_f16(dbase + a * N, da, db, idesc, 0u);
      else tc::mma_tf32(dbase + a * N, da, db, idesc, 0u);
    }
    for (int i = 0; i < nmma / nw; i += 8 * NACC) {
#pragma unroll
      for (int u = 0; u < 8; ++u)
#pragma unroll
        for (int a = 0; a < NACC; ++a) {
          if (MODE == 1) mma_elect<F16>(dbase + a * N, da + u * 8, db + u * 8, idesc, 1u);
          else if (F16) tc::mma_f16(dbase + a * N, da + u * 8, db + u * 8, idesc, 1u);
          else tc::mma_tf32(dbase + a * N, da + u * 8, db + u * 8, idesc, 1u);
        }
    }
    if (MODE == 1) {
      if ((threadIdx.x & 31) == 0) tc::commit(mbar + warp);
      __syncwarp();
    } else {
      tc::commit(mbar + warp);
    }
    tc::mbar_wait(mbar + warp, 0);
  }
  __syncthreads();
  long long t2 = clock64();
  if (blockIdx.x == 0 && threadIdx.x == 0) cycles[0] = t2 - t0;
  tc::fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tc::tmem_free(tmem, 512);
}

template <bool F16, int NACC, int MODE>
static void run(int M, int N, int nw, long long* d, cudaEvent_t e0, cudaEvent_t e1, int mn = 0) {
  if (nw * NACC * N > 512) return;
  auto k = chains_k<F16, NACC, MODE>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  const int nmma = 4096, blocks = 148;
  k<<<blocks, 128, 70 * 1024>>>(M, N, nmma, nw, d, mn);
  cudaEventRecord(e0);
  k<<<blocks, 128, 70 * 1024>>>(M, N, nmma, nw, d, mn);
  cudaEventRecord(e1);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); exit(1); }
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  long long h;
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  const double K = F16 ? 16 : 8;
  const double flops = 2.0 * M * N * K * nmma * blocks;
  printf("%s %s %s M=%3d N=%3d issuers=%d nacc=%d: %.1f cyc/mma per CTA, device %.1f TFLOP/s\n",
         MODE ? "elect" : "lane0", F16 ? "f16 " : "tf32", mn ? "MN-major" : "K-major ", M, N, nw, NACC, (double)h / nmma,
         flops / (ms * 1e-3) / 1e12);
}


// wgrad-shaped issue loop: M x N MN-major bf16 MMAs into `nacc` accumulators at
// column stride `cstride`, A / B group strides sboa / sbob, the A start moving by
// `ashift` bytes per MMA (tap shifts) -- isolates the operand / accumulator
// layout costs of wgrad_bf.cu.
__global__ void wg_shape_k(int M, int N, int nacc, int cstride, int sboa, int sbob, int ashift, int nmma,
                           long long* cycles) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* mbar = reinterpret_cast<uint64_t*>(smem + 200 * 1024);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(mbar + 1);
  if (threadIdx.x < 32) tc::tmem_alloc(tslot, 512);
  if (threadIdx.x == 0) { tc::mbar_init(mbar, 1); tc::fence_mbar_init(); }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = *tslot;
  long long t0 = clock64();
  if (threadIdx.x < 32) {
    const uint32_t idesc = tc::make_idesc(1, M, N) | (1u << 15) | (1u << 16);
    const uint32_t sb = tc::smem_u32(smem);
    for (int i = 0; i < nmma; ++i) {
      const int a = i % nacc;
      const uint64_t da = tc::make_desc(sb + ((i * ashift) & 32767), 128, sboa);
      const uint64_t db = tc::make_desc(sb + 100 * 1024 + ((i & 7) * 256), 128, sbob);
      tc::mma_f16_warp(tmem + (uint32_t)(a * cstride), da, db, idesc, i >= nacc ? 1u : 0u);
    }
    if (threadIdx.x == 0) tc::commit(mbar);
    __syncwarp();
    tc::mbar_wait(mbar, 0);
  }
  __syncthreads();
  long long t2 = clock64();
  if (blockIdx.x == 0 && threadIdx.x == 0) cycles[0] = t2 - t0;
  tc::fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tc::tmem_free(tmem, 512);
}

static void wg_shape(int M, int N, int nacc, int cstride, int sboa, int sbob, int ashift, long long* d) {
  cudaFuncSetAttribute(wg_shape_k, cudaFuncAttributeMaxDynamicSharedMemorySize, 210 * 1024);
  const int nmma = 3072;
  wg_shape_k<<<148, 128, 205 * 1024>>>(M, N, nacc, cstride, sboa, sbob, ashift, nmma, d);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); exit(1); }
  long long h;
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("wgrad-shape M=%d N=%3d nacc=%d colstride=%3d SBO a/b=%5d/%5d A shift/MMA=%4d B: %.1f cyc/mma\n", M, N, nacc,
         cstride, sboa, sbob, ashift, (double)h / nmma);
}

int main(int argc, char** argv) {
  long long* d;
  cudaMalloc(&d, 16);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  if (argc > 1 && argv[1][0] == 'w') {
    for (int ash : {0, 256, 16, 1568})
      for (int cs : {96, 128}) wg_shape(64, 96, 3, cs, 7424, 4096, ash, d);
    wg_shape(64, 96, 3, 128, 2048, 2048, 0, d);
    wg_shape(64, 96, 1, 96, 7424, 4096, 256, d);
    wg_shape(64, 32, 3, 32, 7424, 4096, 256, d);
    wg_shape(128, 96, 3, 96, 7424, 4096, 256, d);
    return 0;
  }
  if (argc > 1) {  // operand-major comparison at the weight-gradient shapes
    for (int M : {64, 128})
      for (int N : {16, 32, 64, 128, 256})
        for (int mn : {0, 1}) run<true, 2, 1>(M, N, 1, d, e0, e1, mn);
    return 0;
  }
  for (int N : {16, 32, 64, 128, 256})
    for (int nw : {1, 2, 4}) {
      run<true, 1, 0>(128, N, nw, d, e0, e1);
      run<true, 1, 1>(128, N, nw, d, e0, e1);
      run<true, 2, 1>(128, N, nw, d, e0, e1);
      run<true, 4, 1>(128, N, nw, d, e0, e1);
      run<false, 1, 1>(128, N, nw, d, e0, e1);
      run<false, 2, 1>(128, N, nw, d, e0, e1);
    }
  return 0;
}
