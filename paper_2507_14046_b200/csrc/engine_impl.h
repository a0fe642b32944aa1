// Internal engine state shared by engine.cu (config ResUNet program, loss,
// Adam, graph replay) and refnet.cu (the FastResUNet3D program).
#pragma once
#include <algorithm>
#include <vector>

#include "common.cuh"
#include "kernels.h"

namespace d2ip {

struct RefNet;

struct ConvP {
  long long ow = 0, ob = 0;
  int cin = 0, cout = 0, ks = 3, stride = 1, dil = 1;
  bool tcf = false, tcd = false;  // tcgen05 forward / data-gradient path
  d2ip::TcDims tdf{}, tdd{};      // their GEMM views (K, N, mode, pack code)
  float* pkf = nullptr;           // packed weights [B][27][cin/4][Np][4] (forward)
  float* pkd = nullptr;           // packed flipped W^T (data gradient)
};
struct NormP {
  long long og = 0, ob = 0;
  int c = 0;
};
struct Block {
  ConvP c1, c2, sk;
  NormP n1, n2;
  int lin = 0, lout = 0;  // spatial level of input / output
  d2ip_act x{}, out{}, gx{}, gout{};
  int gx_acc = 0;
  float *h1 = nullptr, *xh1 = nullptr, *rs1 = nullptr, *xh2 = nullptr, *rs2 = nullptr;
  // backward: gradients read by the weight-gradient kernels on the side stream
  // (per block, so the next block's backward cannot overwrite them early)
  float *gpre = nullptr, *gc2 = nullptr, *gc1 = nullptr;
  float *np1 = nullptr, *np2 = nullptr;  // per-norm dgamma/dbeta partials, reduced on the side stream
};

}  // namespace d2ip

struct d2ip_engine {
  d2ip_net_desc d{};
  long long nparams = 0;
  int L = 0;
  int D[8]{}, H[8]{}, W[8]{};
  long long V[8]{};
  d2ip::ConvP stem, tail;
  d2ip::NormP stem_n;
  std::vector<d2ip::Block> enc, dec;
  d2ip::Block neck;
  d2ip_bindings b{};
  bool bound = false;
  // workspace carve-up
  float* cat[8]{};
  float* gcat[8]{};
  int catw[8]{};
  float *elast = nullptr, *gelast = nullptr, *bout = nullptr, *gbout = nullptr;
  float* decout[8]{};
  float* gdecout[8]{};
  float *stem_xh = nullptr, *stem_rs = nullptr;
  float *raw = nullptr, *raw2 = nullptr, *sc[5]{};
  float *sigma_c = nullptr, *rs = nullptr, *jpart = nullptr, *adjpart = nullptr;
  float *gtail = nullptr, *gmapped = nullptr, *regpart = nullptr;
  void* wg_ws = nullptr;
  size_t wg_ws_bytes = 0;
  void* na_ws = nullptr;
  float* tc_ws = nullptr;
  float* tc_ws2 = nullptr;  // split-K partials of convolutions on the side2 stream (1^3 skips)
  size_t tc_ws_bytes = 0;
  d2ip::PackJobs packjobs;
  size_t na_ws_bytes = 0;
  size_t ws_total = 0;
  long long maxvc = 0;
  int nseg = 0, rsplit = 0, n_reg = 0;
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t gexec = nullptr;
  cudaGraph_t ggraph = nullptr;      // grads-only iteration (forward + loss + backward), for the joint warm-start
  cudaGraphExec_t ggexec = nullptr;
  cudaStream_t cap_stream = nullptr;
  int launches = 0;
  // weight gradients (and dgamma/dbeta sums) run on a pool of side lanes, off the
  // data-gradient critical path; each lane has its own reduction workspace
  static constexpr int kLanes = 3;
  int nlanes = 2;  // lanes in use: 2 for the config ResUNet, 3 for FastResUNet3D (measured best)
  cudaStream_t lane[kLanes]{};
  void* lane_ws[kLanes]{};
  int lane_next = 0;
  cudaStream_t side2 = nullptr;  // short data-gradient branches (1^3 skip) beside the main chain
  static constexpr int kEvents = 128;
  cudaEvent_t ev[kEvents]{};
  int evi = 0;
  float* stem_gc = nullptr;
  float* stem_np = nullptr;
  d2ip::RefNet* ref = nullptr;  // arch == 1: FastResUNet3D program (refnet.cu)
  // bf16 twins (precision BF16) of the buffers the tensor-core convolutions read:
  // [base, base + n) fp32 elements <-> bf16 copy with the same element layout
  struct Twin {
    const float* base;
    long long n;
    void* tw;
  };
  std::vector<Twin> twins;
};

namespace d2ip {

// Bump allocator over the caller's workspace (base null: size query).
struct Arena {
  char* base = nullptr;
  size_t off = 0;
  char* take(size_t bytes) {
    off = (off + 255) & ~(size_t)255;
    char* p = base ? base + off : nullptr;
    off += bytes;
    return p;
  }
  float* f(long long n) { return reinterpret_cast<float*>(take((size_t)n * sizeof(float))); }
  size_t total() const { return (off + 255) & ~(size_t)255; }
};

inline void* twin_of(const d2ip_engine& E, const float* p) {
  for (const auto& t : E.twins)
    if (p >= t.base && p < t.base + t.n) return reinterpret_cast<uint16_t*>(t.tw) + (p - t.base);
  return nullptr;
}

inline d2ip_act view(const d2ip_engine& E, float* p, int lvl, int c, int cs) {
  d2ip_act a;
  a.bf16 = twin_of(E, p);
  a.ptr = p;
  a.d = E.D[lvl];
  a.h = E.H[lvl];
  a.w = E.W[lvl];
  a.c = c;
  a.cstride = cs;
  a.bstride = E.V[lvl] * cs;
  return a;
}


struct Ctx {
  d2ip_engine& E;
  cudaStream_t st;
  int B;
  long long pbs;
  int prec;
  float slope;
  cudaStream_t side2;
  void* wgws;          // weight-gradient reduction workspace of the stream this context launches on
  unsigned lanes = 0;  // side lanes holding work of this pass (join only those: capture rules)
  float* th() const { return E.b.theta; }
  float* gr() const { return E.b.grad; }
};

// A context on the next side lane, ordered after everything already on k.st
// (k records the lane for the join); join_side makes k.st wait for every lane used.
int side_ctx(Ctx& k, Ctx& ks);
int join_side(Ctx& k);
// generic fork / join between two streams (graph-capture safe)
int fork_to(Ctx& k, cudaStream_t from, cudaStream_t to);
// weight gradient on a side lane, after everything already on st
int cwgrad_side(Ctx& k, const ConvP& c, d2ip_act x, d2ip_act gy);

int cfwd(Ctx& k, const ConvP& c, d2ip_act x, d2ip_act y, int acc, SplitK* sk = nullptr, const LnFuse* ln = nullptr,
         int* fused = nullptr);
int cdgrad(Ctx& k, const ConvP& c, d2ip_act gy, d2ip_act gx, int acc, SplitK* sk = nullptr);
int cwgrad(Ctx& k, const ConvP& c, d2ip_act x, d2ip_act gy);

// refnet.cu
int refnet_plan_params(d2ip_engine& E);  // D2IP_OK or an error code
// network-specific buffers; sets E.wg_ws_bytes / na_ws_bytes / tc_ws_bytes
void refnet_plan_workspace(d2ip_engine& E, Arena& A);
void refnet_plan_views(d2ip_engine& E);
void refnet_pack_jobs(d2ip_engine& E);
int refnet_forward(Ctx& k);   // network + tail (writes sig / mapped / sigma_c)
int refnet_backward(Ctx& k);  // from E.gtail to every parameter gradient
void refnet_destroy(d2ip_engine& E);

}  // namespace d2ip
