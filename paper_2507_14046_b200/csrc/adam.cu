// K7: Adam over the flat parameter buffer, restating torch.optim.Adam's
// single-tensor step as the reference runs it on CPU (pipeline.py:304-306,
// 331; fresh optimiser per frame, so m, v and the step restart each frame):
//   m.lerp_(g, 1 - b1)
//   v.mul_(b2).addcmul_(g, g, value = 1 - b2)
//   step_size = lr / (1 - b1^t);  bc2_sqrt = sqrt(1 - b2^t)     (double)
//   denom = (sqrt(v) / bc2_sqrt).add_(eps)
//   p.addcdiv_(m, denom, value = -step_size)
// The step t is read from device memory (graph-replay safe). An iteration
// whose loss was non-finite (bad flag set) skips the update, mirroring the
// reference raising before `optimizer.step()` (pipeline.py:312-317).
#include "common.cuh"
#include "kernels.h"

namespace d2ip {

__device__ __forceinline__ void adam_one(float& p, float g, float& m, float& v, float w1, float b2,
                                         float omb2, float step_size, float bc2s, float eps) {
  // torch lerp: weight < 0.5 -> self + weight * (end - self)
  m = m + w1 * (g - m);
  v = v * b2;
  v = v + omb2 * g * g;
  const float denom = sqrtf(v) / bc2s + eps;
  p = p + (-step_size) * (m / denom);
}

__global__ void __launch_bounds__(256) adam_k(float4* __restrict__ p, const float4* __restrict__ g,
                                              float4* __restrict__ m, float4* __restrict__ v, long long n4,
                                              float lr, float b1, float b2, float eps,
                                              const int* __restrict__ step, const int* __restrict__ bad) {
  D2IP_PDL_ENTRY();
  if (bad && *bad) return;
  const int t = *step;
  const double bc1 = 1.0 - pow((double)b1, (double)t);
  const double bc2 = 1.0 - pow((double)b2, (double)t);
  const float step_size = (float)((double)lr / bc1);
  const float bc2s = (float)sqrt(bc2);
  const float w1 = (float)(1.0 - (double)b1), omb2 = (float)(1.0 - (double)b2);
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n4;
       i += (long long)gridDim.x * blockDim.x) {
    float4 pp = p[i], gg = g[i], mm = m[i], vv = v[i];
    adam_one(pp.x, gg.x, mm.x, vv.x, w1, b2, omb2, step_size, bc2s, eps);
    adam_one(pp.y, gg.y, mm.y, vv.y, w1, b2, omb2, step_size, bc2s, eps);
    adam_one(pp.z, gg.z, mm.z, vv.z, w1, b2, omb2, step_size, bc2s, eps);
    adam_one(pp.w, gg.w, mm.w, vv.w, w1, b2, omb2, step_size, bc2s, eps);
    p[i] = pp;
    m[i] = mm;
    v[i] = vv;
  }
}

__global__ void adam_tail_k(float* p, const float* g, float* m, float* v, long long start, long long n,
                            float lr, float b1, float b2, float eps, const int* step, const int* bad) {
  D2IP_PDL_ENTRY();
  if (bad && *bad) return;
  const long long i = start + blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int t = *step;
  const double bc1 = 1.0 - pow((double)b1, (double)t);
  const double bc2 = 1.0 - pow((double)b2, (double)t);
  adam_one(p[i], g[i], m[i], v[i], (float)(1.0 - (double)b1), b2, (float)(1.0 - (double)b2),
           (float)((double)lr / bc1), (float)sqrt(bc2), eps);
}

int adam_flat(float* p, const float* g, float* m, float* v, long long n, float lr, float b1, float b2,
              float eps, const int* step, const int* bad, cudaStream_t st) {
  const bool aligned = (((uintptr_t)p | (uintptr_t)g | (uintptr_t)m | (uintptr_t)v) & 15) == 0;
  const long long n4 = aligned ? n / 4 : 0;
  if (n4 > 0) {
    long long blocks = (n4 + 255) / 256;
    if (blocks > 148LL * 16) blocks = 148LL * 16;
    D2IP_CUDA(launch_pdl(adam_k, (int)blocks, 256, 0, st, reinterpret_cast<float4*>(p), reinterpret_cast<const float4*>(g),
                                        reinterpret_cast<float4*>(m), reinterpret_cast<float4*>(v), n4, lr,
                                        b1, b2, eps, step, bad));
    D2IP_LAUNCH_CHECK();
  }
  const long long rest = n - n4 * 4;
  if (rest > 0) {
    D2IP_CUDA(launch_pdl(adam_tail_k, cdiv(rest, 256), 256, 0, st, p, g, m, v, n4 * 4, n, lr, b1, b2, eps, step, bad));
    D2IP_LAUNCH_CHECK();
  }
  return D2IP_OK;
}

}  // namespace d2ip
