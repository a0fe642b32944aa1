/*
 * d2ip_b200.h — C ABI of the B200-native DIP-step engine (sm_100a).
 *
 * The reference (`/root/reference/pkg/src/d2ip`, pure Python/PyTorch, CPU) has
 * no native interface; its drop-in surface is the Python API that
 * `paper_2507_14046_b200/pipeline.py` mirrors. Each entry point below replaces
 * one arithmetic step that the reference performs through PyTorch inside its
 * hot loop `_FrameOptimizer.optimize` (pipeline.py:294-338). The mapping is
 * cited per function. The Python package binds this header with ctypes
 * (`paper_2507_14046_b200/_native.py`); INTEGRATION.md shows the binding a
 * maintainer of the reference would add.
 *
 * Conventions
 *   - Raw device pointers, plain integers/floats, and a `void* stream`
 *     (a cudaStream_t). No torch types cross this boundary.
 *   - Activations are NDHWC fp32: element (b, d, h, w, c) of a view lives at
 *     ptr[b*bstride + ((d*H + h)*W + w)*cstride + c]; `cstride >= C` lets a
 *     view address a channel slice of a concat buffer in place.
 *     (D, H, W) = (R, C, P) of the reference grid (`priornet.py:217-219`).
 *   - Weights are the reference's OIDHW fp32 layout inside one flat parameter
 *     buffer in state_dict order; per-sequence parameter sets (batch > 1) are
 *     `wbstride` floats apart.
 *   - Every function returns 0 on success, a negative D2IP_E* code otherwise;
 *     `d2ip_last_error()` holds the message. Nothing allocates device memory
 *     except `d2ip_engine_*` (which only allocates CUDA graph objects) and
 *     nothing synchronises the host.
 */
#ifndef D2IP_B200_H
#define D2IP_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define D2IP_ABI_VERSION 4

enum {
  D2IP_OK = 0,
  D2IP_E_ARG = -1,      /* invalid shape / argument   -> ValueError            */
  D2IP_E_CUDA = -2,     /* CUDA launch / runtime error -> NativeLibraryError    */
  D2IP_E_UNSUPPORTED = -3
};

enum { D2IP_PREC_FP32 = 0, D2IP_PREC_TF32 = 1, D2IP_PREC_BF16 = 2 };
enum { D2IP_NORM_L2SQ = 0, D2IP_NORM_L2 = 1 };
/* Network program of the engine. */
enum {
  D2IP_ARCH_CONFIG_RESUNET = 0, /* canonical config ResUNet (LeakyReLU, C_z-channel noise) */
  D2IP_ARCH_FAST_RESUNET = 1    /* reference FastResUNet3D (priornet.py:183-232; SiLU, SE, ASPP, attention) */
};

/* A channels-last activation view (see conventions). `bf16` optionally points
 * at a bf16 twin with the same element layout (element i of the view at
 * ((uint16_t*)bf16)[i offset]): producers write it when set, bf16-precision
 * tensor-core kernels stream it with async copies instead of converting the
 * fp32 values. NULL = no twin. */
typedef struct {
  float* ptr;
  int d, h, w;
  int c;
  int cstride;
  long long bstride;
  void* bf16;
} d2ip_act;

int d2ip_abi_version(void);
const char* d2ip_last_error(void);
/* Name of the kernel variant the last conv call dispatched to (diagnostics). */
const char* d2ip_last_variant(void);

/* Debug launch tracing (no reference counterpart): events around every kernel
 * launch from d2ip_trace_begin until d2ip_trace_dump, which synchronises and
 * writes "<start_us> <end_us> <stream> <kernel>" lines (relative to the first
 * launch) into buf; returns the full text length. Eager launches only. */
int d2ip_trace_begin(void);
int d2ip_trace_dump(char* buf, size_t n);

/* ---- K1: 3^3 / 1^3 convolution forward ---------------------------------
 * y = conv3d(x, W, b) (+ y if accumulate). ksize 3 -> padding 1, ksize 1 ->
 * padding 0; stride 1 or 2. Replaces `nn.Conv3d` forward
 * (priornet.py:117,143,200,215 / oracle ConfigResUNet). precision TF32 on a
 * 3^3 layer (stride 1, or stride 2 by parity decomposition) runs the tcgen05
 * implicit GEMM, whose packed weights need `d2ip_conv3d_ws_bytes()` of
 * workspace (0 for the direct kernels); workspace beyond that, when large
 * enough, holds split-K partial sums (more CTAs on small grids). */
size_t d2ip_conv3d_ws_bytes(int cin, int cout, int ksize, int stride, int precision, int batch);
int d2ip_conv3d_fwd(d2ip_act x, const float* w, const float* bias, long long wbstride,
                    int ksize, int stride, d2ip_act y, int accumulate, int precision,
                    void* ws, size_t ws_bytes, int batch, void* stream);

/* ---- K2: convolution data gradient -------------------------------------
 * gx (+)= conv_transpose(gy, W). Replaces autograd's conv backward (input)
 * triggered by `total.backward()` (pipeline.py:330). */
int d2ip_conv3d_dgrad(d2ip_act gy, const float* w, long long wbstride, int ksize, int stride,
                      d2ip_act gx, int accumulate, int precision, void* ws, size_t ws_bytes,
                      int batch, void* stream);

/* ---- K3: convolution weight + bias gradient ----------------------------
 * gw = sum_v gy (x) x-patch  (OIDHW), gb = sum_v gy; written to gw[0 ..
 * Cout*Cin*k^3) and gw[Cout*Cin*k^3 .. + Cout) — the reference's adjacent
 * `weight`,`bias` entries of the flat gradient. Deterministic split-K over
 * voxels (fixed-order reduction). `ws` must hold d2ip_conv3d_wgrad_ws_bytes(). */
size_t d2ip_conv3d_wgrad_ws_bytes(d2ip_act x, d2ip_act gy, int ksize, int batch);
int d2ip_conv3d_wgrad(d2ip_act x, d2ip_act gy, int ksize, int stride, float* gw,
                      long long gwbstride, void* ws, size_t ws_bytes, int precision,
                      int batch, void* stream);

/* Weight-gradient kernel for TF32 stride-1 3^3 layers: 1 = tcgen05 3xTF32
 * (wgrad_tc.cu, default), 0 = smem-tiled CUDA-core fp32 (wgrad_s1.cu).
 * Process-wide; the default can be set by the environment variable
 * D2IP_WGRAD=s1|tc. */
int d2ip_set_wgrad_variant(int variant);
int d2ip_get_wgrad_variant(void);

/* ---- ChannelLayerNorm (+ residual) (+ LeakyReLU) forward ----------------
 * out = act(gamma * xhat + beta [+ res]), xhat = (y - mean_c) * rstd,
 * rstd = 1/sqrt(var_c + 1e-5). Saves xhat [B][V][C] and rstd [B][V].
 * Replaces ChannelLayerNorm.forward (priornet.py:105-108) + F.silu /
 * leaky_relu + residual add (priornet.py:146-148). act: 0 none, 1 leaky. */
int d2ip_norm_act_fwd(d2ip_act y, const float* gamma, const float* beta, long long pbstride,
                      d2ip_act res, int act, float slope, d2ip_act out, float* xhat, float* rstd,
                      int batch, void* stream);

/* Backward of the above: gy_pre = gout * act'(out); gc = LN-backward(gy_pre);
 * optionally stores gy_pre (the residual/skip branch gradient), and writes
 * dgamma, dbeta (deterministic) to dgb[0..C) and dgb[C..2C). */
size_t d2ip_norm_act_bwd_ws_bytes(int v, int c, int batch);
int d2ip_norm_act_bwd(d2ip_act gout, d2ip_act out, int act, float slope, const float* xhat,
                      const float* rstd, const float* gamma, long long pbstride, d2ip_act gy_pre,
                      d2ip_act gc, float* dgb, long long dgbstride, void* ws, size_t ws_bytes,
                      int batch, void* stream);

/* ---- K4: trilinear x2 upsample (align_corners=False) ------------------
 * Replaces F.interpolate(..., mode="trilinear") (priornet.py:229); the
 * output view may be the channel slice of the decoder concat buffer
 * (torch.cat at priornet.py:230 becomes a no-op). Backward is a gather. */
int d2ip_upsample2x_fwd(d2ip_act x, d2ip_act y, int batch, void* stream);
int d2ip_upsample2x_bwd(d2ip_act gy, d2ip_act gx, int accumulate, int batch, void* stream);

/* ---- K5: J.sigma, residual, data term ----------------------------------
 * y = J sigma_V (J: M x Vp fp32 row-major, Vp % 4 == 0, zero padded),
 * r_f = y - dv_f for n_rhs frames; data = sum_f |r_f|^2 ("l2sq") or its sqrt
 * ("l2"). Writes rs[m] = c * sum_f r_f[m] with c = dData/d(sum r^2)*2, the
 * adjoint's right-hand side. `partial` holds [batch][nseg][m] column-segment sums (nseg =
 * d2ip_jac_nseg(vp)), summed in segment order by the loss. Replaces `operator @ _vectorize_t(mapped)`,
 * `dv - ...` and `_data_term` (pipeline.py:257-263,279). */
int d2ip_jac_fwd(const float* J, long long jbstride, const float* sigma, long long sbstride,
                 int m, int vp, float* partial, int nseg, int batch, void* stream);
int d2ip_jac_nseg(int vp);

/* ---- K6: adjoint J^T rs ------------------------------------------------ */
int d2ip_jac_adj(const float* J, long long jbstride, const float* rs, int m, int vp,
                 float* g, long long gbstride, void* ws, size_t ws_bytes, int batch, void* stream);
size_t d2ip_jac_adj_ws_bytes(int m, int vp, int batch);

/* ---- K7: Adam over a flat buffer ---------------------------------------
 * torch.optim.Adam single-tensor step (pipeline.py:304-306,331): step count
 * read from device memory (*step), bias corrections in double. */
int d2ip_adam(float* p, const float* g, float* m, float* v, long long n, float lr, float beta1,
              float beta2, float eps, const int* step, void* stream);

/* ---- Standalone 4D-TV (drop-in spatial_tv / temporal_tv / tv4d) ---------
 * Replaces pkg/src/d2ip/regularizers.py:86-140 for one (R, C, P) fp32 volume
 * (p fastest) and n_history past volumes [n][R][C][P]:
 *   *value = lambda_s * spatial_tv(current) + lambda_t * temporal_tv(history, current)
 * (device float), grad (optional, [R][C][P]) = d value / d current.
 * ws: d2ip_tv4d_ws_bytes(R, C, P) bytes. */
size_t d2ip_tv4d_ws_bytes(int R, int C, int P);
int d2ip_tv4d(const float* current, const float* history, int n_history, int R, int C, int P, float lambda_s,
              float lambda_t, float epsilon, float* value, float* grad, void* ws, size_t ws_bytes, void* stream);

/* ---- fp64 projection (drop-in forward_project) --------------------------
 * y[m] = sum_j A[m][j] x[j] in float64 (pkg/src/d2ip/forward.py:115-122),
 * A row-major with leading dimension lda; deterministic fixed-order sums. */
int d2ip_project_f64(const double* A, long long lda, const double* x, int m, int n, double* y, void* stream);

/* ---- Sensitivity operator assembly ---------------------
 * Replaces assemble_sensitivity + normalize_sensitivity
 * (pkg/src/d2ip/forward.py:58-112) on the device, fp64:
 *   out[m][q] = -(f_d+ - f_d-).(f_m+ - f_m-) * voxel_volume,
 *   f_e(q) = -(c_q - p_e) / (4 pi max(|c_q - p_e|, min_dist)^3),
 * centers [Q][3] (canonical q order), electrodes [E][3], quads int32 [M][4]
 * (16-byte aligned), norms[m] = ||out[m]||_2. normalize != 0 divides every row
 * by its norm in place (the caller rejects zero rows, forward.py:103-106).
 * J_masked (optional): fp32 [M][Vp] block, column j = voxel q_of_col[j] (the
 * engine's memory column order), zero padded -- the fp64 operator never needs
 * to visit the host. */
int d2ip_assemble_sensitivity(const double* centers, int Q, const double* electrodes, int E, const int* quads, int M,
                              double min_dist, double voxel_volume, int normalize, double* out, double* norms,
                              float* J_masked, int V, int Vp, const int* q_of_col, void* stream);

/* ---- Engine: one whole DIP iteration, graph-captured --------------------
 * Owns the launch plan of one network program (`arch`: the canonical config
 * ResUNet of SURVEY §7.1, or the reference's FastResUNet3D with levels = 4,
 * channels = b,2b,4b,8b, in_channels = 1) for `batch` independent sequences
 * in lockstep (cfg3) and replays it with CUDA graphs.
 * Replaces the Python loop body pipeline.py:310-331. */
typedef struct {
  int batch;                 /* independent sequences, each its own theta/Z/J */
  int R, C, P;               /* grid; divisible by 2^(levels-1) */
  int levels;
  int channels[8];
  int in_channels;           /* C_z */
  float negative_slope;
  int M;                     /* measurements */
  int V;                     /* masked voxels (columns of J) */
  int Vp;                    /* V rounded up to a multiple of 4 */
  int n_rhs;                 /* frames in the data term (1; joint UPWS > 1) */
  int j_shared;              /* 1: one J for all sequences */
  int data_norm;             /* D2IP_NORM_* */
  float lo, hi;              /* output_map */
  float lr, beta1, beta2, eps;
  int precision;             /* D2IP_PREC_* for convolutions */
  float lambda_tv, lambda_s, lambda_t, tv_eps;
  int max_history;           /* TV history capacity (frames) */
  int max_iters;             /* trace capacity */
  /* ABI 3 */
  int arch;                  /* D2IP_ARCH_* */
  int depthwise;             /* FastResUNet3D: depthwise-separable 3^3 (NetworkConfig.use_depthwise) */
  int n_dil;                 /* FastResUNet3D: ASPP branches (NetworkConfig.aspp_dilations) */
  int dil[8];
} d2ip_net_desc;

typedef struct {
  float* theta;              /* [batch][n_params] */
  float* grad;               /* [batch][n_params] */
  float* adam_m;
  float* adam_v;
  const float* z;            /* [batch][R][C][P][C_z] */
  const float* J;            /* [batch or 1][M][Vp], columns in vox_of_col order */
  const int* vox_of_col;     /* [V] voxel offset ((r*C + c)*P + p) of column j */
  const int* col_of_vox;     /* [R*C*P] column of a voxel or -1 */
  const float* dv;           /* [batch][n_rhs][M] */
  const float* history;      /* [batch][max_history][R*C*P] (TV) */
  float* mapped;             /* [batch][R*C*P]  lo + (hi-lo)*sigmoid(out) */
  float* sig;                /* [batch][R*C*P]  sigmoid(out) */
  float* trace;              /* [batch][max_iters][4] data, reg, total, t_ns */
  int* status;               /* [batch][4] iters done, first bad iter, -, - */
  void* workspace;
  size_t workspace_bytes;
} d2ip_bindings;

typedef struct d2ip_engine d2ip_engine;

int d2ip_engine_create(const d2ip_net_desc* desc, d2ip_engine** out);
void d2ip_engine_destroy(d2ip_engine* e);
long long d2ip_engine_param_count(const d2ip_engine* e);
size_t d2ip_engine_workspace_bytes(const d2ip_engine* e);
int d2ip_engine_bind(d2ip_engine* e, const d2ip_bindings* b);
/* history frames currently valid for TV (0..max_history) */
int d2ip_engine_set_history(d2ip_engine* e, int n_history);
/* Zero Adam moments and the per-frame iteration counter (fresh optimiser per
 * frame, pipeline.py:304-306). */
int d2ip_engine_reset_frame(d2ip_engine* e, void* stream);
/* One iteration: forward, data term (+TV), backward, Adam; no graph. */
int d2ip_engine_step(d2ip_engine* e, void* stream);
/* `iters` iterations by CUDA-graph replay (graph captured on first use). */
int d2ip_engine_run(d2ip_engine* e, int iters, void* stream);
/* Forward only: writes sig and mapped (and the data term when with_loss). */
int d2ip_engine_forward(d2ip_engine* e, int with_loss, void* stream);
/* Forward + y = J sigma into y [batch][M] (predict_measurements, pipeline.py:375-391). */
int d2ip_engine_predict(d2ip_engine* e, float* y, void* stream);
/* The Adam update alone, on the current gradient buffer (data-parallel joint
 * warm-start: grads -> all-reduce -> adam). */
int d2ip_engine_adam(d2ip_engine* e, void* stream);
/* Forward + loss + backward without the Adam update (gradient parity). */
int d2ip_engine_grads(d2ip_engine* e, void* stream);
/* The same gradient program replayed from a CUDA graph captured on first use (the
 * joint warm-start's per-iteration grads -> NCCL all-reduce -> d2ip_engine_adam). */
int d2ip_engine_grads_graph(d2ip_engine* e, void* stream);
/* Kernel launches one graph-replayed iteration issues. */
int d2ip_engine_launches_per_iter(const d2ip_engine* e);

#ifdef __cplusplus
}
#endif
#endif /* D2IP_B200_H */
