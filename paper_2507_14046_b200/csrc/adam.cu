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
#include <algorithm>

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

// One launch over `batch` independent parameter segments of `nper` scalars
// (blockIdx.y = segment b: the lockstep sequences of a batched engine). Each
// segment reads ITS step counter and bad flag (step[b * sstride],
// bad[b * sstride]), so a diverged sequence skips only its own update, as its
// own reference run would. Body: scalar head up to 16-byte alignment, float4
// middle, scalar tail (all four buffers share one alignment offset).
__global__ void __launch_bounds__(256) adam_k(float* __restrict__ p, const float* __restrict__ g,
                                              float* __restrict__ m, float* __restrict__ v, long long nper,
                                              int aligned, float lr, float b1, float b2, float eps,
                                              const int* __restrict__ step, const int* __restrict__ bad,
                                              int sstride) {
  D2IP_PDL_ENTRY();
  const int b = blockIdx.y;
  if (bad && bad[(long long)b * sstride]) return;
  const int t = step[(long long)b * sstride];
  const double bc1 = 1.0 - pow((double)b1, (double)t);
  const double bc2 = 1.0 - pow((double)b2, (double)t);
  const float step_size = (float)((double)lr / bc1);
  const float bc2s = (float)sqrt(bc2);
  const float w1 = (float)(1.0 - (double)b1), omb2 = (float)(1.0 - (double)b2);
  const long long off = (long long)b * nper;
  p += off;
  g += off;
  m += off;
  v += off;
  long long head = 0, n4 = 0;
  if (aligned) {
    head = (long long)((16 - ((uintptr_t)p & 15)) & 15) / 4;
    if (head > nper) head = nper;
    n4 = (nper - head) / 4;
  } else {
    head = nper;
  }
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x, nth = (long long)gridDim.x * blockDim.x;
  float4* p4 = reinterpret_cast<float4*>(p + head);
  const float4* g4 = reinterpret_cast<const float4*>(g + head);
  float4* m4 = reinterpret_cast<float4*>(m + head);
  float4* v4 = reinterpret_cast<float4*>(v + head);
  for (long long i = tid; i < n4; i += nth) {
    float4 pp = p4[i], gg = g4[i], mm = m4[i], vv = v4[i];
    adam_one(pp.x, gg.x, mm.x, vv.x, w1, b2, omb2, step_size, bc2s, eps);
    adam_one(pp.y, gg.y, mm.y, vv.y, w1, b2, omb2, step_size, bc2s, eps);
    adam_one(pp.z, gg.z, mm.z, vv.z, w1, b2, omb2, step_size, bc2s, eps);
    adam_one(pp.w, gg.w, mm.w, vv.w, w1, b2, omb2, step_size, bc2s, eps);
    p4[i] = pp;
    m4[i] = mm;
    v4[i] = vv;
  }
  if (tid < head) adam_one(p[tid], g[tid], m[tid], v[tid], w1, b2, omb2, step_size, bc2s, eps);
  for (long long i = head + 4 * n4 + tid; i < nper; i += nth)
    adam_one(p[i], g[i], m[i], v[i], w1, b2, omb2, step_size, bc2s, eps);
}

int adam_flat(float* p, const float* g, float* m, float* v, long long nper, float lr, float b1, float b2,
              float eps, const int* step, const int* bad, cudaStream_t st, int batch, int sstride) {
  D2IP_CHECK_ARG(batch >= 1 && nper >= 0, "adam: batch %d, n %lld", batch, nper);
  if (nper == 0) return D2IP_OK;
  // all four buffers must share the alignment offset of p for the float4 body
  const uintptr_t a = (uintptr_t)p & 15;
  const int aligned = (((uintptr_t)g & 15) == a && ((uintptr_t)m & 15) == a && ((uintptr_t)v & 15) == a &&
                       (a & 3) == 0) ? 1 : 0;
  long long blocks = (std::max(nper / 4, (long long)4) + 255) / 256;
  const long long cap = std::max(1LL, 148LL * 16 / batch);
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  D2IP_CUDA(launch_pdl(adam_k, dim3((unsigned)blocks, (unsigned)batch), dim3(256), 0, st, p, g, m, v, nper, aligned,
                       lr, b1, b2, eps, step, bad, sstride));
  D2IP_LAUNCH_CHECK();
  return D2IP_OK;
}

}  // namespace d2ip
