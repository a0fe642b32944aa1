// Probe of tcgen05 tf32 operand layouts: one MMA D[M][N] = A[M][K=8] * B[N][K=8]^T
// from shared memory, A in a configurable layout (K-major interleave, MN-major
// interleave, MN-major 128B / 32B swizzle, optionally started at a row offset
// inside the swizzle atom), B K-major; compared with a host reference.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -I../paper_2507_14046_b200/csrc umma_probe.cu -o umma_probe
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <vector>

#include "common.cuh"
#include "tc.cuh"

using namespace d2ip;

enum { L_K_INTER = 0, L_MN_INTER = 1, L_MN_SW128 = 2, L_MN_SW32 = 3, L_MN_SW64 = 4, L_MN_B32 = 5 };
static int g_lbo = 2048, g_sbo = 512;

// byte offset of element (mn, k) for A, relative to the (1024-aligned) buffer,
// with the operand starting `r0` K-rows (128 B each for swizzled) into the buffer.
static int a_off(int lay, int M, int mn, int k, int r0) {
  switch (lay) {
    case L_K_INTER:  // K chunk (4 k) stride M*16, 8-row group 128 B
      return (k / 4) * M * 16 + (mn / 8) * 128 + (mn % 8) * 16 + (k % 4) * 4;
    case L_MN_INTER:  // MN chunk (4 mn) stride 8*16 (one K block of 8 rows)
      return (mn / 4) * 128 + k * 16 + (mn % 4) * 4;
    case L_MN_SW128: {  // rows of 128 B (32 mn) per k; 32-mn blocks at 1024*rows... use block stride 2048
      const int row = k + r0;
      const int blk = mn / 32, w = mn % 32, c = w / 4, e = w % 4;
      const int addr = blk * 2048 + row * 128;  // 16 rows per block region (room for r0 up to 8)
      const int pc = c ^ ((addr >> 7) & 7);
      return addr + pc * 16 + e * 4;
    }
    case L_MN_SW64: {  // rows of 64 B (16 mn)
      const int row = k + r0;
      const int blk = mn / 16, w = mn % 16, c = w / 4, e = w % 4;
      const int addr = blk * 1024 + row * 64;
      const int pc = c ^ ((addr >> 7) & 3);
      return addr + pc * 16 + e * 4;
    }
    case L_MN_B32: {  // 128B rows (32 mn) per k, 32-B granules swizzled by row % 4, K blocks of 4 rows
      const int row = k + r0;
      const int blk = mn / 32, w = mn % 32, gq = w / 8;
      const int addr = blk * g_lbo + (row / 4) * g_sbo + (row % 4) * 128;
      const int pg = gq ^ ((addr >> 7) & 3);
      return addr + pg * 32 + (w % 8) * 4;
    }
    case L_MN_SW32: {  // rows of 32 B (8 mn)
      const int row = k + r0;
      const int blk = mn / 8, w = mn % 8, c = w / 4, e = w % 4;
      const int addr = blk * 512 + row * 32;
      const int pc = c ^ ((addr >> 7) & 1);
      return addr + pc * 16 + e * 4;
    }
  }
  return 0;
}

__global__ void probe_k(const float* A, const float* B, float* D, int N, int a_bytes, int b_floats, uint32_t idesc,
                        uint64_t da_rel, uint64_t db_rel) {
  extern __shared__ __align__(1024) uint8_t smem[];
  float* sa = reinterpret_cast<float*>(smem);
  float* sb = reinterpret_cast<float*>(smem + a_bytes);
  uint64_t* mbar = reinterpret_cast<uint64_t*>(sb + b_floats);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(mbar + 1);
  for (int i = threadIdx.x; i < a_bytes / 4; i += blockDim.x) sa[i] = A[i];
  for (int i = threadIdx.x; i < b_floats; i += blockDim.x) sb[i] = B[i];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (warp == 0) tc::tmem_alloc(tslot, 256);
  if (threadIdx.x == 0) {
    tc::mbar_init(mbar, 1);
    tc::fence_mbar_init();
  }
  tc::fence_proxy_async();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = *tslot;
  if (threadIdx.x == 0) {
    // descriptors come with start address relative to smem base (in 16-B units in the low bits)
    const uint64_t base = (uint64_t)(tc::smem_u32(smem) >> 4);
    tc::mma_tf32(tmem, da_rel + base, db_rel + base + (uint64_t)(a_bytes >> 4), idesc, 0u);
    tc::commit(mbar);
  }
  tc::mbar_wait(mbar, 0);
  tc::fence_after();
  const uint32_t trow = tmem + ((uint32_t)(warp * 32) << 16);
  for (int c0 = 0; c0 < N; c0 += 8) {
    float v[8];
    tc::tmem_ld8(trow + c0, v);
    for (int j = 0; j < 8; ++j) D[(warp * 32 + lane) * 256 + c0 + j] = v[j];
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_free(tmem, 256);
}

static uint64_t desc_fields(uint32_t start_rel, uint32_t lbo, uint32_t sbo, int layout_type, int base_off) {
  uint64_t d = 0;
  d |= (uint64_t)((start_rel >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)(base_off & 7) << 49;
  d |= (uint64_t)(layout_type & 7) << 61;
  return d;
}

static const char* names[] = {"K-inter", "MN-inter", "MN-sw128", "MN-sw32", "MN-sw64", "MN-b32"};

int run(int M, int N, int lay, int r0, uint32_t lbo, uint32_t sbo, int ltype, int base_off) {
  const int K = 8;
  const int a_bytes = 16384;
  std::vector<float> A(M * K), B(N * K), hA(a_bytes / 4, 0.f), hB(N * K);
  srand(1);
  for (int m = 0; m < M; ++m)
    for (int k = 0; k < K; ++k) {
      A[m * K + k] = (float)((rand() % 17) - 8);
      hA[a_off(lay, M, m, k, r0) / 4] = A[m * K + k];
    }
  for (int n = 0; n < N; ++n)
    for (int k = 0; k < K; ++k) {
      B[n * K + k] = (float)((rand() % 13) - 6);
      hB[((k / 4) * N * 16 + (n / 8) * 128 + (n % 8) * 16 + (k % 4) * 4) / 4] = B[n * K + k];
    }
  float *dA, *dB, *dD;
  cudaMalloc(&dA, a_bytes);
  cudaMalloc(&dB, N * K * 4);
  cudaMalloc(&dD, 128 * 256 * 4);
  cudaMemset(dD, 0, 128 * 256 * 4);
  cudaMemcpy(dA, hA.data(), a_bytes, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB.data(), N * K * 4, cudaMemcpyHostToDevice);
  const int amn = lay != L_K_INTER;
  uint32_t idesc = tc::make_idesc(2, M, N) | ((uint32_t)amn << 15);
  const int rowb = (lay == L_MN_SW128 || lay == L_MN_B32) ? 128 : (lay == L_MN_SW64 ? 64 : (lay == L_MN_SW32 ? 32 : 0));
  const uint64_t da = desc_fields((uint32_t)(r0 * rowb), lbo, sbo, ltype, base_off);
  const uint64_t db = desc_fields(0, N * 16, 128, 0, 0);
  probe_k<<<1, 128, a_bytes + N * K * 4 + 64>>>(dA, dB, dD, N, a_bytes, N * K, idesc, da, db);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("%s: CUDA error %s\n", names[lay], cudaGetErrorString(e));
    exit(1);
  }
  std::vector<float> D(128 * 256);
  cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
  int bad = 0, nz = 0;
  for (int m = 0; m < M; ++m)
    for (int n = 0; n < N; ++n) {
      float ref = 0;
      for (int k = 0; k < K; ++k) ref += A[m * K + k] * B[n * K + k];
      const int lanep = M == 128 ? m : (m % 16) + 32 * (m / 16);
      const float got = D[lanep * 256 + n];
      if (got != 0) ++nz;
      if (fabsf(got - ref) > 1e-3f) ++bad;
    }
  printf("%-9s M=%3d N=%3d r0=%d lbo=%5u sbo=%5u type=%d base=%d -> %4d/%4d wrong, %4d nonzero\n", names[lay], M, N, r0,
         lbo, sbo, ltype, base_off, bad, M * N, nz);
  cudaFree(dA);
  cudaFree(dB);
  cudaFree(dD);
  return bad;
}

int main() {
  cudaFuncSetAttribute(probe_k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  const int M = 128, N = 16;
  run(M, N, L_K_INTER, 0, M * 16, 128, 0, 0);
  for (int lbo_sbo : {0, 1}) {
    g_lbo = lbo_sbo ? 512 : 2048;
    g_sbo = lbo_sbo ? 2048 : 512;
    for (int sw : {0, 1}) run(M, N, L_MN_B32, 0, sw ? g_sbo : g_lbo, sw ? g_lbo : g_sbo, 1, 0);
  }
  g_lbo = 4096; g_sbo = 512;
  for (int r0 : {1, 2, 4, 5})
    for (int bo : {0, 1, 2, 4, 5}) run(M, N, L_MN_B32, r0, g_lbo, g_sbo, 1, bo);
  return 0;
}
