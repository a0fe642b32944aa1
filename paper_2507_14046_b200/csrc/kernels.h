// Internal (C++) entry points of the kernel library; the C ABI in capi.cu and
// the engine in engine.cu call these.
#pragma once
#include "common.cuh"

namespace d2ip {

// conv_direct.cu — exact fp32 CUDA-core convolutions
// dil: dilation of 3^3 kernels (ASPP3d branches, priornet.py:156-158); padding = dil
int conv_fwd_direct(d2ip_act x, const float* w, const float* bias, long long wbs, int ks, int stride,
                    d2ip_act y, int accumulate, int batch, cudaStream_t st, int dil = 1);
int conv_dgrad_direct(d2ip_act gy, const float* w, long long wbs, int ks, int stride, d2ip_act gx,
                      int accumulate, int batch, cudaStream_t st, int dil = 1);
size_t conv_wgrad_direct_ws(int cin, int cout, int ks, long long V, int batch);
int conv_wgrad_direct(d2ip_act x, d2ip_act gy, int ks, int stride, float* gw, long long gwbs,
                      void* ws, size_t ws_bytes, int batch, cudaStream_t st, int dil = 1);

// refnet_kernels.cu — FastResUNet3D extras (priornet.py:111-180)
int dw_conv_fwd(d2ip_act x, const float* w, const float* bias, long long wbs, int stride, d2ip_act y, int batch,
                cudaStream_t st);
int dw_conv_dgrad(d2ip_act gy, const float* w, long long wbs, int stride, d2ip_act gx, int accumulate, int batch,
                  cudaStream_t st);
size_t dw_wgrad_ws(int C, long long V, int batch);
int dw_conv_wgrad(d2ip_act x, d2ip_act gy, int stride, float* gw, long long gwbs, void* ws, size_t ws_bytes,
                  int batch, cudaStream_t st);
size_t colsum_ws(int C, long long V, int batch);
// SE state per sequence: [pooled C][z1 hid][gate C][gpool C]  (sbs >= 3C + hid)
int se_forward(d2ip_act x, const float* w1, const float* b1, const float* w2, const float* b2, long long pbs, int hid,
               float* state, int sbs, d2ip_act out, void* ws, size_t ws_bytes, int batch, cudaStream_t st);
int se_backward(d2ip_act x, d2ip_act gs, const float* w1, const float* b1, const float* w2, long long pbs, int hid,
                float* state, int sbs, float* g1, float* g2, d2ip_act gx, int accumulate, void* ws, size_t ws_bytes,
                int batch, cudaStream_t st);
int add_silu(d2ip_act k, d2ip_act q, float* pre, d2ip_act a, int batch, cudaStream_t st);
int silu_bwd(d2ip_act ga, const float* pre, d2ip_act gpre, int batch, cudaStream_t st);
int sigmoid_inplace(float* t, long long n, cudaStream_t st);
int sigmoid_bwd(float* g, const float* s, long long n, cudaStream_t st);
int att_gate_fwd(d2ip_act s, const float* att, d2ip_act out, int batch, cudaStream_t st);
int att_gate_bwd(d2ip_act gg, d2ip_act s, const float* att, d2ip_act gs, int accumulate, float* gatt, int batch,
                 cudaStream_t st);
int reduce_chunks(const float* partial, int nchunks, int n, float* out, long long obs, int batch,
                  cudaStream_t st);

// wgrad_s1.cu — smem-tiled weight gradient of stride-1 3^3 convolutions
bool wgrad_s1_supported(d2ip_act x, d2ip_act gy, int ks);
size_t wgrad_s1_ws_bytes(int D, int H, int W, int Cin, int Cout, int ks, int batch);
int wgrad_s1(d2ip_act x, d2ip_act gy, int ks, float* gw, long long gwbs, void* ws, size_t ws_bytes, int batch,
             cudaStream_t st);

// wgrad_tc.cu — tcgen05 weight gradient of stride-1 3^3 / 1^3 convolutions (3xTF32)
bool wgrad_tc_supported(d2ip_act x, d2ip_act gy, int ks, int precision);
size_t wgrad_tc_ws_bytes(int D, int H, int W, int Cin, int Cout, int ks, int batch);
int wgrad_tc(d2ip_act x, d2ip_act gy, int ks, float* gw, long long gwbs, void* ws, size_t ws_bytes, int batch,
             cudaStream_t st);

// wgrad_bf.cu — tcgen05 kind::f16 weight gradient of 3^3 (stride 1 and 2) / 1^3 convolutions (bf16 layers)
// b3: a TF32-precision layer on 3xbf16 (hi + lo operands, three MMAs per K step)
bool wgrad_bf_supported(d2ip_act x, d2ip_act gy, int ks, int stride = 1, bool b3 = false);
size_t wgrad_bf_ws_bytes(int D, int H, int W, int Cin, int Cout, int ks, int batch);
int wgrad_bf(d2ip_act x, d2ip_act gy, int ks, float* gw, long long gwbs, void* ws, size_t ws_bytes, int batch,
             cudaStream_t st, int stride = 1, bool b3 = false);
// fixed-order reduction of [b][rg][ntaps][Cin][Cout] + [Cout] partials into OIDHW + bias
int wgrad_reduce(const float* part, int nrg, int ntaps, int Cin, int Cout, float* gw, long long gwbs, int batch,
                 cudaStream_t st);

// conv_tc.cu — tcgen05 implicit-GEMM convolutions (tf32 / bf16 operands)
bool conv_tc_supported(int cin, int cout, int ks, int stride, int precision);
// GEMM view of a layer's tcgen05 forward (dgrad = 0) or data gradient: K, N,
// kernel mode (0 stride 1, 1 stride-2 forward, 2 stride-2 dgrad) and pack code;
// both carry kTcBf16 when the layer runs with bf16 operands (kind::f16).
constexpr int kTcBf16 = 4;
constexpr int kTcPw = 8;  // pack code: 1^3 weights (mode 3)
constexpr int kTcKwf = 32;  // mode / pack code: stride-1 3^3 with the kw taps folded into N (MODE 4);
                            // pack layout [kd kh][K/4][kw][Np][4] so a stage's B tile per kh is contiguous
constexpr int kTcBf3 = 16;  // mode / pack code: TF32-precision layer on 3xbf16 (hi + lo split) kind::f16 MMAs
// TF32-precision layers run 3xbf16 tensor-core kernels (D2IP_TF32_BF3=0: 3xTF32)
bool tf32_bf3_enabled();
struct TcDims {
  int K, N, mode, pack;
};
// vout: the layer's output voxels (-1: unknown) -- small stride-2 layers stay on the direct kernel
bool conv_tc_layer(int cin, int cout, int ks, int stride, int dgrad, int precision, long long vout, TcDims* d);
long long conv_tc_pack_floats(int K, int N);
int conv_tc_pack(const float* w, long long wbs, int K, int N, int dgrad, float* out, int batch, cudaStream_t st);
// One launch packing every tcgen05 layer of the network (weights change each step).
struct PackJobs {
  static constexpr int kMax = 64;
  int n = 0;
  long long wbs = 0;  // per-sequence parameter stride
  const float* w[kMax];
  float* out[kMax];
  int K[kMax], N[kMax], dgrad[kMax];
  long long half[kMax];  // packed elements per half (27 or 1 taps x K x Np)
  long long obs[kMax];   // per-sequence stride of the pack buffer (conv_tc_pack_floats)
  int cin[kMax], cout[kMax];  // layer channels: one thread per (co, ci) weight vector
  int block0[kMax + 1] = {0};
};
void pack_jobs_add(PackJobs& j, const float* w, int K, int N, int dgrad, float* out);
int conv_tc_pack_multi(const PackJobs& jobs, int batch, cudaStream_t st);
// ws (optional): split-K partials, conv_tc_ws_bytes() of them; null -> no split-K
// (D, H, W: the row-space grid = the layer's output grid, or gy's for a dgrad)
size_t conv_tc_ws_bytes(int D, int H, int W, int K, int N, int batch, int mode = 0);
// deferred != null: a split-K result is left as partials in ws (*deferred =
// kspl, 0 if not split) for the consumer to reduce (norm_act_fwd's `part`).
// ChannelLayerNorm (+ residual) (+ LeakyReLU) fused into a convolution's epilogue
// (priornet.py:96-108,145-148): out = act(gamma * (x - mean) * rstd + beta [+ res]), with
// xhat [b][V][C] and rstd [b][V] saved for the backward -- norm_act_fwd's contract.
struct LnFuse {
  const float* gamma = nullptr;
  const float* beta = nullptr;
  long long pbs = 0;
  d2ip_act res{};
  d2ip_act out{};
  float* xhat = nullptr;
  float* rstd = nullptr;
  int act = 1;
  float slope = 0.2f;
};

int conv_tc_run(d2ip_act x, const float* wp, int K, int N, const float* bias, long long bbs, d2ip_act y,
                int accumulate, float* ws, size_t ws_bytes, int batch, cudaStream_t st, int* deferred = nullptr,
                int mode = 0, const LnFuse* ln = nullptr, int* fused = nullptr);

// Split-K partial sums handed from a convolution to its consumer:
// y[v][n] = bias[n] + sum_k part[b][k][v][n].
struct SplitK {
  const float* part = nullptr;
  int kspl = 0;
  const float* bias = nullptr;
  long long bbs = 0;
};

size_t conv_wgrad_ws(int cin, int cout, int ks, int D, int H, int W, int batch, int precision);
int conv_wgrad(d2ip_act x, d2ip_act gy, int ks, int stride, float* gw, long long gwbs, void* ws,
               size_t ws_bytes, int precision, int batch, cudaStream_t st);

// elem.cu — normalisation / activation / resampling / output map
// act: 0 none, 1 LeakyReLU(slope), 2 SiLU (then `pre` receives the
// pre-activation, which norm_act_bwd takes as its `out` view for act 2)
int norm_act_fwd(d2ip_act y, const float* gamma, const float* beta, long long pbs, d2ip_act res,
                 int act, float slope, d2ip_act out, float* xhat, float* rstd, int batch,
                 cudaStream_t st, SplitK sk = SplitK{}, d2ip_act pre = d2ip_act{});
size_t norm_act_bwd_ws(long long V, int C, int batch);
int norm_act_bwd(d2ip_act gout, d2ip_act out, int act, float slope, const float* xhat,
                 const float* rstd, const float* gamma, long long pbs, d2ip_act gpre, d2ip_act gc,
                 float* dgb, long long dgbs, void* ws, size_t ws_bytes, int batch, cudaStream_t st,
                 int* deferred = nullptr,   // deferred: skip the dgamma/dbeta reduce, *deferred = partial chunks
                 SplitK sk = SplitK{});     // sk: gout = sum of the producing conv's split-K partials
int upsample2x_fwd(d2ip_act x, d2ip_act y, int batch, cudaStream_t st);
int upsample2x_bwd(d2ip_act gy, d2ip_act gx, int accumulate, int batch, cudaStream_t st);
int tail_fwd(d2ip_act x, const float* w, const float* bias, long long wbs, float lo, float scale,
             float* sig, float* mapped, float* sigma_c, long long sc_bs, const int* col_of_vox,
             int batch, cudaStream_t st);
// C_out = 1 tail convolution backward (lane-group kernels; C = 4, 8, 16, 32)
bool tail_bwd_supported(d2ip_act x);
int tail_dgrad(const float* gt, const float* w, long long wbs, d2ip_act gx, int batch, cudaStream_t st);
size_t tail_wgrad_ws(int C, long long V, int batch);
int tail_wgrad(d2ip_act x, const float* gt, float* gw, long long gwbs, void* ws, size_t ws_bytes, int batch,
               cudaStream_t st);
int tail_bwd_prep(const float* gmapped, const float* sig, float scale, float* gtail, long long V0,
                  int batch, cudaStream_t st);

// jacobian.cu — HBM-streaming J.sigma / J^T r, data term
int jac_nseg(int vp);
int jac_fwd_partial(const float* J, long long jbs, const float* sigma, long long sbs, int m, int vp,
                    float* partial, int nseg, int batch, cudaStream_t st);
int jac_loss(const float* partial, int nseg, int m, const float* dv, int n_rhs, int norm,
             const float* reg_partial, int n_reg, float reg_scale, float* rs, float* trace,
             int max_iters, int* status, int batch, cudaStream_t st);
int jac_sum(const float* partial, int nseg, int m, float* y, int batch, cudaStream_t st);
int jac_adj_rows(int m, int vp, int batch);
size_t jac_adj_ws(int m, int vp, int batch);
int jac_adj_partial(const float* J, long long jbs, const float* rs, int m, int vp, float* partial,
                    int rsplit, int batch, cudaStream_t st);
int jac_adj_finish(const float* partial, int rsplit, int vp, int v, const int* vox_of_col,
                   const float* sig, float scale, float* gout, long long V0, int add_to_gmapped,
                   int batch, cudaStream_t st);

// tv.cu — 4D-TV value partials + gradient w.r.t. mapped
int tv_nblocks(long long V0);
int tv_fwd_bwd(const float* mapped, const float* history, int max_history, const int* status,
               int R, int C, int P, float lam_tv, float lam_s, float lam_t, float eps,
               float* gmapped, float* reg_partial, int batch, cudaStream_t st);

// adam.cu
int adam_flat(float* p, const float* g, float* m, float* v, long long nper, float lr, float b1, float b2,
              float eps, const int* step, const int* bad, cudaStream_t st, int batch = 1, int sstride = 0);

// standalone drop-in helpers (tv.cu, jacobian.cu)
size_t tv4d_ws_bytes(int R, int C, int P);
int tv4d_standalone(const float* current, const float* history, int n_history, int R, int C, int P, float lam_s,
                    float lam_t, float eps, float* value, float* grad, void* ws, size_t ws_bytes, cudaStream_t st);
int project_f64(const double* A, long long lda, const double* x, int m, int n, double* y, cudaStream_t st);

}  // namespace d2ip
