// Does tcgen05.mma.kind::tf32 truncate or round fp32 operands? One MMA with
// A = 1 + 3*2^-12 (truncation -> 1, round-to-nearest -> 1 + 2^-10), B = 1.
#include <cstdio>
#include "common.cuh"
#include "tc.cuh"
using namespace d2ip;

__global__ void k(float aval, float* out) {
  __shared__ __align__(1024) float sa[128 * 8];
  __shared__ __align__(1024) float sb[16 * 8];
  __shared__ uint64_t mbar;
  __shared__ uint32_t tslot;
  for (int i = threadIdx.x; i < 128 * 8; i += blockDim.x) sa[i] = 0.f;
  for (int i = threadIdx.x; i < 16 * 8; i += blockDim.x) sb[i] = 0.f;
  __syncthreads();
  if (threadIdx.x == 0) {
    sa[0] = aval;  // A[0][0] (K-major interleave: row 0, k 0)
    sb[0] = 1.0f;  // B[0][0]
  }
  if (threadIdx.x < 32) tc::tmem_alloc(&tslot, 32);
  if (threadIdx.x == 0) { tc::mbar_init(&mbar, 1); tc::fence_mbar_init(); }
  tc::fence_proxy_async();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  if (threadIdx.x == 0) {
    const uint64_t da = tc::make_desc(tc::smem_u32(sa), 128 * 16, 128);
    const uint64_t db = tc::make_desc(tc::smem_u32(sb), 16 * 16, 128);
    tc::mma_tf32(tslot, da, db, tc::make_idesc(2, 128, 16), 0u);
    tc::commit(&mbar);
  }
  tc::mbar_wait(&mbar, 0);
  tc::fence_after();
  float v[8];
  tc::tmem_ld8(tslot + ((uint32_t)((threadIdx.x / 32) * 32) << 16), v);
  if (threadIdx.x == 0) out[0] = v[0];
  tc::fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tc::tmem_free(tslot, 32);
}

int main() {
  float* d;
  cudaMalloc(&d, 4);
  const float vals[] = {1.0f + 3.0f / 4096, 1.0f + 1.0f / 4096, -(1.0f + 3.0f / 4096), 1.0f + 7.0f / 8192};
  for (float a : vals) {
    k<<<1, 128>>>(a, d);
    float h;
    cudaMemcpy(&h, d, 4, cudaMemcpyDeviceToHost);
    const unsigned ab = *(const unsigned*)&a;
    const float tr = *(const float*)&(const unsigned&)(unsigned){ab & 0xFFFFE000u};
    printf("a=%.9g  mma=%.9g  trunc=%.9g  %s\n", a, h, tr, h == tr ? "TRUNCATES" : "rounds");
  }
  return 0;
}
