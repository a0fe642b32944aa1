// Issue-rate probe: cycles per tcgen05.mma (one thread issuing into one
// accumulator) for kind::tf32 / kind::f16 shapes, and with several CTAs per SM.
#include <cstdio>
#include "common.cuh"
#include "tc.cuh"
using namespace d2ip;

__global__ void rate_k(int M, int N, int f16, int nmma, long long* cycles) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* mbar = reinterpret_cast<uint64_t*>(smem + 65536);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(mbar + 1);
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<float*>(smem)[i] = 0.0f;
  if (threadIdx.x < 32) tc::tmem_alloc(tslot, 256);
  if (threadIdx.x == 0) { tc::mbar_init(mbar, 1); tc::fence_mbar_init(); }
  tc::fence_proxy_async();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = *tslot;
  if (threadIdx.x == 0) {
    const uint32_t idesc = tc::make_idesc(f16 ? 1 : 2, M, N);
    const uint32_t sb = tc::smem_u32(smem);
    const uint64_t da = tc::make_desc(sb, 2048, 128);
    const uint64_t db = tc::make_desc(sb + 32768, 2048, 128);
    long long t0 = clock64();
    if (f16)
      for (int i = 0; i < nmma; ++i) tc::mma_f16(tmem, da + (i & 7) * 8, db + (i & 7) * 8, idesc, i > 0);
    else
      for (int i = 0; i < nmma; ++i) tc::mma_tf32(tmem, da + (i & 7) * 8, db + (i & 7) * 8, idesc, i > 0);
    tc::commit(mbar);
    tc::mbar_wait(mbar, 0);
    long long t2 = clock64();
    if (blockIdx.x == 0) cycles[0] = t2 - t0;
  }
  tc::fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tc::tmem_free(tmem, 256);
}

int main() {
  cudaFuncSetAttribute(rate_k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  long long* d;
  cudaMalloc(&d, 16);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int f16 : {0, 1})
    for (int M : {128})
      for (int N : {16, 64, 128, 256})
        for (int per_sm : {1, 2}) {
          const int nmma = 4096;
          const int blocks = 148 * per_sm;
          rate_k<<<blocks, 128, 70 * 1024>>>(M, N, f16, nmma, d);  // warm
          cudaEventRecord(e0);
          rate_k<<<blocks, 128, 70 * 1024>>>(M, N, f16, nmma, d);
          cudaEventRecord(e1);
          cudaError_t e = cudaDeviceSynchronize();
          if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
          float ms;
          cudaEventElapsedTime(&ms, e0, e1);
          long long h;
          cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
          const double K = f16 ? 16 : 8;
          const double flops = 2.0 * M * N * K * nmma * blocks;
          printf("%s M=%3d N=%3d CTAs/SM=%d: %.1f cyc/mma (CTA 0), device %.1f TFLOP/s\n", f16 ? "f16 " : "tf32", M, N,
                 per_sm, (double)h / nmma, flops / (ms * 1e-3) / 1e12);
        }
  return 0;
}
