// 4D-TV: value partials and gradient w.r.t. the mapped
// volume, restating pkg/src/d2ip/regularizers.py:86-140:
//   spatial  = (1/Q) sum_v sqrt(d_r^2 + d_c^2 + d_p^2 + eps)   forward diffs,
//              zero at the last index of each axis (:78-95)
//   temporal = (1/sum a_k) sum_k a_k sum_v sqrt((v - h_k)^2 + eps),
//              a_k = exp(-(i - j)), j = k + 1, i = n_hist + 1 (:98-131)
//   reg      = lambda_tv * (lambda_s * spatial + lambda_t * temporal)
// Volume memory order is (r, c, p) with p fastest — the network's NDHWC grid.
// The history count is read from device memory (status[b][2]) so one captured
// graph serves every frame of a sequence.
#include "common.cuh"
#include "kernels.h"

namespace d2ip {

constexpr int kTvThreads = 256;

int tv_nblocks(long long V0) { return cdiv(V0, kTvThreads); }

__device__ __forceinline__ float tv_at(const float* m, int r, int c, int p, int C, int P) {
  return m[((long long)r * C + c) * P + p];
}

// s and forward diffs at (r, c, p)
__device__ __forceinline__ float tv_s(const float* m, int r, int c, int p, int R, int C, int P, float eps,
                                      float* dr, float* dc, float* dp) {
  const float x = tv_at(m, r, c, p, C, P);
  *dr = r < R - 1 ? tv_at(m, r + 1, c, p, C, P) - x : 0.f;
  *dc = c < C - 1 ? tv_at(m, r, c + 1, p, C, P) - x : 0.f;
  *dp = p < P - 1 ? tv_at(m, r, c, p + 1, C, P) - x : 0.f;
  return sqrtf(*dr * *dr + *dc * *dc + *dp * *dp + eps);
}

__global__ void __launch_bounds__(kTvThreads) tv_k(const float* __restrict__ mapped,
                                                   const float* __restrict__ history, int max_history,
                                                   const int* __restrict__ status, int R, int C, int P,
                                                   float lam_tv, float lam_s, float lam_t, float eps,
                                                   float* __restrict__ gmapped, float* __restrict__ reg_partial) {
  D2IP_PDL_ENTRY();
  __shared__ float red[kTvThreads / 32];
  const int b = blockIdx.y;
  const long long Q = (long long)R * C * P;
  const long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const float* m = mapped + b * Q;
  const int n = status[b * 4 + 2];
  float val = 0.f;
  if (v < Q) {
    const int p = (int)(v % P), c = (int)((v / P) % C), r = (int)(v / ((long long)P * C));
    float dr, dc, dp;
    const float s = tv_s(m, r, c, p, R, C, P, eps, &dr, &dc, &dp);
    float gs = -(dr + dc + dp) / s;
    float t0, t1, t2;
    if (r > 0) { const float sn = tv_s(m, r - 1, c, p, R, C, P, eps, &t0, &t1, &t2); gs += t0 / sn; }
    if (c > 0) { const float sn = tv_s(m, r, c - 1, p, R, C, P, eps, &t0, &t1, &t2); gs += t1 / sn; }
    if (p > 0) { const float sn = tv_s(m, r, c, p - 1, R, C, P, eps, &t0, &t1, &t2); gs += t2 / sn; }
    const float invQ = 1.0f / (float)Q;
    val = lam_s * s * invQ;
    float g = lam_s * gs * invQ;
    if (n > 0) {
      double wsum = 0.0;
      for (int k = 0; k < n; ++k) wsum += exp(-(double)(n - k));
      const float invw = (float)(1.0 / wsum);
      const float x = m[v];
      float tv = 0.f, tg = 0.f;
      for (int k = 0; k < n; ++k) {
        const float a = (float)exp(-(double)(n - k));
        const float d = x - history[((long long)b * max_history + k) * Q + v];
        const float sq = sqrtf(d * d + eps);
        tv = fmaf(a, sq, tv);
        tg = fmaf(a, d / sq, tg);
      }
      val += lam_t * tv * invw;
      g += lam_t * tg * invw;
    }
    gmapped[b * Q + v] = lam_tv * g;
  }
  val = block_sum<kTvThreads>(val, red);
  if (threadIdx.x == 0) reg_partial[(long long)b * gridDim.x + blockIdx.x] = val;
}

int tv_fwd_bwd(const float* mapped, const float* history, int max_history, const int* status,
               int R, int C, int P, float lam_tv, float lam_s, float lam_t, float eps,
               float* gmapped, float* reg_partial, int batch, cudaStream_t st) {
  const long long Q = (long long)R * C * P;
  D2IP_CUDA(launch_pdl(tv_k, dim3(tv_nblocks(Q), batch), kTvThreads, 0, st, mapped, history, max_history, status, R, C, P,
                                                           lam_tv, lam_s, lam_t, eps, gmapped, reg_partial));
  D2IP_LAUNCH_CHECK();
  return D2IP_OK;
}

// Standalone 4D-TV (the drop-in `spatial_tv` / `temporal_tv` / `tv4d`,
// regularizers.py:86-140): value = lam_s * spatial + lam_t * temporal and its
// gradient w.r.t. `current`, for one volume and n_history past volumes. The
// history count lives in a device int (the engine kernel's status word), the
// block partials are summed in fixed order by one more block.
__global__ void tv_setn_k(int* st, int n) {
  st[0] = 0; st[1] = 0; st[2] = n; st[3] = 0;
}

__global__ void __launch_bounds__(kTvThreads) tv_reduce_k(const float* __restrict__ part, int n,
                                                          float* __restrict__ value) {
  __shared__ float red[kTvThreads / 32];
  float s = 0.f;
  for (int i = threadIdx.x; i < n; i += kTvThreads) s += part[i];
  s = block_sum<kTvThreads>(s, red);
  if (threadIdx.x == 0) *value = s;
}

size_t tv4d_ws_bytes(int R, int C, int P) {
  const long long Q = (long long)R * C * P;
  return 16 + (size_t)tv_nblocks(Q) * sizeof(float) + (size_t)Q * sizeof(float);
}

int tv4d_standalone(const float* current, const float* history, int n_history, int R, int C, int P, float lam_s,
                    float lam_t, float eps, float* value, float* grad, void* ws, size_t ws_bytes, cudaStream_t st) {
  D2IP_CHECK_ARG(current && value && R > 0 && C > 0 && P > 0 && n_history >= 0 && (n_history == 0 || history),
                 "tv4d: bad arguments");
  D2IP_CHECK_ARG(ws && ws_bytes >= tv4d_ws_bytes(R, C, P), "tv4d: workspace too small");
  const long long Q = (long long)R * C * P;
  int* stw = reinterpret_cast<int*>(ws);
  float* part = reinterpret_cast<float*>(reinterpret_cast<char*>(ws) + 16);
  float* gbuf = grad ? grad : part + tv_nblocks(Q);
  tv_setn_k<<<1, 1, 0, st>>>(stw, n_history);
  D2IP_LAUNCH_CHECK();
  D2IP_RET(tv_fwd_bwd(current, history, n_history > 0 ? n_history : 1, stw, R, C, P, 1.0f, lam_s, lam_t, eps, gbuf,
                      part, 1, st));
  tv_reduce_k<<<1, kTvThreads, 0, st>>>(part, tv_nblocks(Q), value);
  D2IP_LAUNCH_CHECK();
  return D2IP_OK;
}

}  // namespace d2ip
