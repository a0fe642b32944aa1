// Probe: kind::f16 (bf16) MMA with BOTH operands MN-major in the no-swizzle
// layout the weight-gradient kernel uses -- per 8-channel group a column of
// 16-byte rows (one row per K index) -- started at an arbitrary row offset r0
// (a tap shift). Measured on sm_100a: exact with LBO = 128 B (the stride of
// 8-row K blocks) and SBO = the group-column stride (swap = 1), for every row
// shift; the opposite assignment (swap = 0) yields garbage.
//   D[m][n] = sum_k A[m][k] B[n][k],  A[m][k] = a_src[k + r0][m],  B[n][k] = b_src[k][n]
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -I paper_2507_14046_b200/csrc \
//        tools/umma_mn_probe.cu -o tools/umma_mn_probe
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include <cuda_bf16.h>

#include "common.cuh"
#include "tc.cuh"

using namespace d2ip;

constexpr int ROWS = 64;  // rows per group column in smem

// a: [ROWS][M] row-major (channels contiguous), b: [16][N]; both bf16
__global__ void probe_k(const __nv_bfloat16* a, const __nv_bfloat16* b, float* d, int M, int N, int r0, int swap) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* As = smem;                       // [M/8][ROWS][16 B]
  uint8_t* Bs = smem + (M / 8) * ROWS * 16; // [N/8][ROWS][16 B]
  uint64_t* mbar = reinterpret_cast<uint64_t*>(Bs + (N / 8) * ROWS * 16);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(mbar + 1);
  for (int i = threadIdx.x; i < (M / 8) * ROWS; i += blockDim.x) {
    const int g = i / ROWS, r = i % ROWS;
    for (int e = 0; e < 8; ++e)
      reinterpret_cast<__nv_bfloat16*>(As + ((size_t)g * ROWS + r) * 16)[e] = a[(size_t)r * M + g * 8 + e];
  }
  for (int i = threadIdx.x; i < (N / 8) * ROWS; i += blockDim.x) {
    const int g = i / ROWS, r = i % ROWS;
    for (int e = 0; e < 8; ++e)
      reinterpret_cast<__nv_bfloat16*>(Bs + ((size_t)g * ROWS + r) * 16)[e] =
          r < 16 ? b[(size_t)r * N + g * 8 + e] : __float2bfloat16(0.f);
  }
  if (threadIdx.x < 32) tc::tmem_alloc(tslot, 128);
  if (threadIdx.x == 0) { tc::mbar_init(mbar, 1); tc::fence_mbar_init(); }
  tc::fence_proxy_async();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = *tslot;
  if (threadIdx.x == 0) {
    // A and B MN-major (idesc bits 15, 16); LBO = group column stride, SBO = 8 rows x 16 B
    const uint32_t idesc = tc::make_idesc(1, M, N) | (1u << 15) | (1u << 16);
    const uint32_t lbo = swap ? 128 : ROWS * 16, sbo = swap ? ROWS * 16 : 128;
    const uint64_t da = tc::make_desc(tc::smem_u32(As) + r0 * 16, lbo, sbo);
    const uint64_t db = tc::make_desc(tc::smem_u32(Bs), lbo, sbo);
    tc::mma_f16(tmem, da, db, idesc, 0u);
    tc::commit(mbar);
  }
  tc::mbar_wait(mbar, 0);
  tc::fence_after();
  // M = 128: lane m; M = 64: lane (m % 16) + 32 (m / 16)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int c0 = 0; c0 < N; c0 += 8) {
    float v[8];
    tc::tmem_ld8(tmem + ((uint32_t)(warp * 32) << 16) + c0, v);
    const int l = warp * 32 + lane;
    int m = -1;
    if (M == 128) m = l;
    else if ((l & 31) < 16) m = (l & 15) + 16 * (l >> 5);
    if (m >= 0 && m < M)
      for (int j = 0; j < 8; ++j) d[m * N + c0 + j] = v[j];
  }
  tc::fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tc::tmem_free(tmem, 128);
}

int main() {
  cudaFuncSetAttribute(probe_k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  int fails = 0;
  for (int swap : {0, 1})
  for (int M : {64, 128})
    for (int N : {16, 32, 64})
      for (int r0 : {0, 1, 3, 8, 13}) {
        std::vector<__nv_bfloat16> ha(ROWS * M), hb(16 * N);
        std::vector<float> fa(ROWS * M), fb(16 * N), hd(M * N), ref(M * N, 0.f);
        srand(M * 7 + N * 3 + r0);
        for (int i = 0; i < ROWS * M; ++i) { ha[i] = __float2bfloat16((rand() % 17 - 8) / 8.f); fa[i] = __bfloat162float(ha[i]); }
        for (int i = 0; i < 16 * N; ++i) { hb[i] = __float2bfloat16((rand() % 13 - 6) / 4.f); fb[i] = __bfloat162float(hb[i]); }
        for (int m = 0; m < M; ++m)
          for (int n = 0; n < N; ++n)
            for (int k = 0; k < 16; ++k) ref[m * N + n] += fa[(k + r0) * M + m] * fb[k * N + n];
        __nv_bfloat16 *da, *db;
        float* dd;
        cudaMalloc(&da, ha.size() * 2);
        cudaMalloc(&db, hb.size() * 2);
        cudaMalloc(&dd, hd.size() * 4);
        cudaMemcpy(da, ha.data(), ha.size() * 2, cudaMemcpyHostToDevice);
        cudaMemcpy(db, hb.data(), hb.size() * 2, cudaMemcpyHostToDevice);
        cudaMemset(dd, 0, hd.size() * 4);
        probe_k<<<1, 128, 64 * 1024>>>(da, db, dd, M, N, r0, swap);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
        cudaMemcpy(hd.data(), dd, hd.size() * 4, cudaMemcpyDeviceToHost);
        double err = 0;
        for (int i = 0; i < M * N; ++i) err = fmax(err, fabs(hd[i] - ref[i]));
        printf("bf16 MN-major A,B swap=%d M=%3d N=%2d row shift %2d: max |err| %.3g %s\n", swap, M, N, r0, err, err < 1e-3 ? "ok" : "FAIL");
        fails += err >= 1e-3;
        cudaFree(da); cudaFree(db); cudaFree(dd);
      }
  return fails ? 1 : 0;
}
