// Shared helpers for the sm_100a DIP-step kernels.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <string>

#include "../../include/d2ip_b200.h"

namespace d2ip {

void set_error(const char* fmt, ...);
void set_variant(const char* name);

#define D2IP_CHECK_ARG(cond, ...)             \
  do {                                        \
    if (!(cond)) {                            \
      ::d2ip::set_error(__VA_ARGS__);         \
      return D2IP_E_ARG;                      \
    }                                         \
  } while (0)

#define D2IP_CUDA(call)                                                          \
  do {                                                                           \
    cudaError_t err__ = (call);                                                  \
    if (err__ != cudaSuccess) {                                                  \
      ::d2ip::set_error("%s:%d %s: %s", __FILE__, __LINE__, #call,               \
                        cudaGetErrorString(err__));                              \
      return D2IP_E_CUDA;                                                        \
    }                                                                            \
  } while (0)

#define D2IP_LAUNCH_CHECK() D2IP_CUDA(cudaGetLastError())

#define D2IP_RET(call)        \
  do {                        \
    int rc__ = (call);        \
    if (rc__ != D2IP_OK) return rc__; \
  } while (0)

inline cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// Programmatic dependent launch: every kernel is launched with the
// programmatic-stream-serialisation attribute (also inside the captured CUDA
// graph), waits for its predecessor's completion with griddepcontrol.wait at
// its top, and immediately allows its successor to be scheduled — so the ~110
// launches of an iteration overlap their launch latency with the previous
// kernel's tail. The wait covers the whole predecessor grid and its memory, so
// early triggering is always safe; dependencies are transitive. (Measured: an
// explicit griddepcontrol.launch_dependents at kernel entry makes successors
// resident early and costs 9 % at cfg1 -- 1,238 -> 1,130 it/s -- their shared
// memory holds SMs the side-stream kernels need; the implicit trigger at exit stays.)
#define D2IP_PDL_ENTRY()                                              \
  do {                                                                \
    asm volatile("griddepcontrol.wait;" ::: "memory");                \
  } while (0)

// Launch tracing (debug: d2ip_trace_begin / d2ip_trace_dump): events around
// every launch, so a step's real concurrent timeline can be read back.
extern int g_trace_on;
void trace_pre(cudaStream_t st, const void* fn);
void trace_post(cudaStream_t st);

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (g_trace_on) trace_pre(st, reinterpret_cast<const void*>(kernel));
  const cudaError_t e = cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
  if (g_trace_on) trace_post(st);
  return e;
}

inline int cdiv(long long a, long long b) { return (int)((a + b - 1) / b); }

// Division by a runtime constant d (1 <= d < 2^14) of 0 <= n < 2^28 as a
// multiply-high: q = (n * floor(2^42 / d + 1)) >> 42 (exact in that range).
struct FastDiv {
  uint32_t d;
  unsigned long long m;
};
inline FastDiv fastdiv(uint32_t d) { return FastDiv{d, (1ull << 42) / d + 1}; }
__device__ __forceinline__ int fdiv(int n, const FastDiv& f) {
  return (int)(((unsigned long long)(uint32_t)n * f.m) >> 42);
}

// two floats -> packed bf16x2 (round to nearest even), low half = a
__device__ __forceinline__ uint32_t bf16x2(float a, float b) {
  const __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<const uint32_t*>(&h);
}

__device__ __forceinline__ long long vox_count(const d2ip_act& a) {
  return (long long)a.d * a.h * a.w;
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Deterministic block sum (fixed tree order); all threads get the result.
template <int NT>
__device__ __forceinline__ float block_sum(float v, float* smem /* >= NT/32 */) {
  v = warp_sum(v);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) smem[warp] = v;
  __syncthreads();
  float t = 0.f;
  if (warp == 0) {
    t = lane < NT / 32 ? smem[lane] : 0.f;
    t = warp_sum(t);
    if (lane == 0) smem[0] = t;
  }
  __syncthreads();
  t = smem[0];
  return t;
}

__device__ __forceinline__ float lrelu(float x, float s) { return x > 0.f ? x : x * s; }

}  // namespace d2ip
