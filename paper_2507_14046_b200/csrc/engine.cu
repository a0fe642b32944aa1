// The DIP-step engine: launch plan of one whole iteration of the canonical
// config ResUNet for `batch` independent sequences in lockstep,
// replayed with CUDA graphs. Replaces the Python loop body of the reference's
// `_FrameOptimizer.optimize` (pkg/src/d2ip/pipeline.py:310-331):
//   forward (priornet.py:217-232 topology), output map (pipeline.py:276-278),
//   data term (+ 4D-TV) (pipeline.py:279-283), non-finite check and trace
//   (pipeline.py:312-328, device-side), backward (pipeline.py:330), Adam
//   (pipeline.py:331).
//
// Memory: every activation, saved tensor and gradient lives in one caller-
// provided workspace (planned here, allocated by the host as a torch uint8
// tensor); parameters, gradients and Adam moments are flat [batch][n_params]
// fp32 buffers in the reference's state_dict order / OIDHW layout.
#include <algorithm>
#include <cstring>
#include <vector>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"

#include "engine_impl.h"

namespace d2ip {

// Param offsets in the exact order of priornet.param_schema().
static void plan_params(d2ip_engine& E) {
  long long o = 0;
  auto conv = [&](int cin, int cout, int ks, int stride) {
    ConvP c;
    c.cin = cin;
    c.cout = cout;
    c.ks = ks;
    c.stride = stride;
    c.ow = o;
    o += (long long)cout * cin * ks * ks * ks;
    c.ob = o;
    o += cout;
    return c;
  };
  auto norm = [&](int c) {
    NormP n;
    n.c = c;
    n.og = o;
    o += c;
    n.ob = o;
    o += c;
    return n;
  };
  auto block = [&](int cin, int cout, int stride) {
    Block b;
    b.c1 = conv(cin, cout, 3, stride);
    b.n1 = norm(cout);
    b.c2 = conv(cout, cout, 3, 1);
    b.n2 = norm(cout);
    b.sk = conv(cin, cout, 1, stride);
    return b;
  };
  const int* c = E.d.channels;
  const int L = E.L;
  E.stem = conv(E.d.in_channels, c[0], 3, 1);
  E.stem_n = norm(c[0]);
  E.enc.clear();
  for (int i = 1; i < L; ++i) {
    Block b = block(c[i - 1], c[i], 2);
    b.lin = i - 1;
    b.lout = i;
    E.enc.push_back(b);
  }
  E.neck = block(c[L - 1], c[L - 1], 1);
  E.neck.lin = E.neck.lout = L - 1;
  E.dec.clear();
  for (int lvl = L - 2; lvl >= 0; --lvl) {
    Block b = block(c[lvl + 1] + c[lvl], c[lvl], 1);
    b.lin = b.lout = lvl;
    E.dec.push_back(b);
  }
  E.tail = conv(c[0], 1, 3, 1);
  E.nparams = o;
}

// Network buffers of the config ResUNet (base may be null: size query).
static void config_plan_workspace(d2ip_engine& E, Arena& A) {
  const int B = E.d.batch;
  auto takef = [&](long long n) { return A.f(n); };
  const int* c = E.d.channels;
  const int L = E.L;
  for (int l = 0; l + 1 < L; ++l) {
    E.catw[l] = c[l + 1] + c[l];
    E.cat[l] = takef((long long)B * E.V[l] * E.catw[l]);
    E.gcat[l] = takef((long long)B * E.V[l] * E.catw[l]);
    E.decout[l] = takef((long long)B * E.V[l] * c[l]);
    E.gdecout[l] = takef((long long)B * E.V[l] * c[l]);
  }
  E.elast = takef((long long)B * E.V[L - 1] * c[L - 1]);
  E.gelast = takef((long long)B * E.V[L - 1] * c[L - 1]);
  E.bout = takef((long long)B * E.V[L - 1] * c[L - 1]);
  E.gbout = takef((long long)B * E.V[L - 1] * c[L - 1]);
  E.stem_xh = takef((long long)B * E.V[0] * c[0]);
  E.stem_rs = takef((long long)B * E.V[0]);
  E.stem_gc = takef((long long)B * E.V[0] * c[0]);
  E.stem_np = reinterpret_cast<float*>(A.take(norm_act_bwd_ws(E.V[0], c[0], B)));
  long long maxvc = E.V[0] * c[0];
  auto saved = [&](Block& bl) {
    const long long vc = E.V[bl.lout] * bl.c1.cout;
    if (vc > maxvc) maxvc = vc;
    bl.h1 = takef(B * vc);
    bl.xh1 = takef(B * vc);
    bl.xh2 = takef(B * vc);
    bl.rs1 = takef((long long)B * E.V[bl.lout]);
    bl.rs2 = takef((long long)B * E.V[bl.lout]);
    bl.gpre = takef(B * vc);
    bl.gc2 = takef(B * vc);
    bl.gc1 = takef(B * vc);
    bl.np1 = reinterpret_cast<float*>(A.take(norm_act_bwd_ws(E.V[bl.lout], bl.c1.cout, B)));
    bl.np2 = reinterpret_cast<float*>(A.take(norm_act_bwd_ws(E.V[bl.lout], bl.c1.cout, B)));
  };
  for (auto& bl : E.enc) saved(bl);
  saved(E.neck);
  for (auto& bl : E.dec) saved(bl);
  E.maxvc = maxvc;
  // bf16 twins of every tensor a bf16 tensor-core convolution reads: block inputs
  // (concat buffers, the last encoder output), h1, and the gradients gc1 / gc2 /
  // gpre / stem gc; their producers (LayerNorm fwd/bwd, upsample) write both copies
  if (E.d.precision == D2IP_PREC_BF16) {
    auto twin = [&](float* p, long long n) {
      void* t = A.take((size_t)n * 2);
      if (p && t) E.twins.push_back({p, n, t});
    };
    for (int l = 0; l + 1 < L; ++l) twin(E.cat[l], (long long)B * E.V[l] * E.catw[l]);
    twin(E.elast, (long long)B * E.V[L - 1] * c[L - 1]);
    twin(E.stem_gc, (long long)B * E.V[0] * c[0]);
    auto tw_block = [&](Block& bl) {
      const long long vc = (long long)B * E.V[bl.lout] * bl.c1.cout;
      twin(bl.h1, vc);
      twin(bl.gc1, vc);
      twin(bl.gc2, vc);
      twin(bl.gpre, vc);
    };
    for (auto& bl : E.enc) tw_block(bl);
    tw_block(E.neck);
    for (auto& bl : E.dec) tw_block(bl);
  }
  E.raw = takef(B * maxvc);
  E.raw2 = takef(B * maxvc);
  for (int i = 0; i < 5; ++i) E.sc[i] = takef(B * maxvc);
  // reduction workspaces: max over layers
  size_t wg = 0, na = 0;
  auto conv_ws = [&](const ConvP& cv, int lout) {
    size_t s = conv_wgrad_ws(cv.cin, cv.cout, cv.ks, E.D[lout], E.H[lout], E.W[lout], B, E.d.precision);
    if (s > wg) wg = s;
  };
  auto blk_ws = [&](const Block& bl) {
    conv_ws(bl.c1, bl.lout);
    conv_ws(bl.c2, bl.lout);
    conv_ws(bl.sk, bl.lout);
    size_t s = norm_act_bwd_ws(E.V[bl.lout], bl.c1.cout, B);
    if (s > na) na = s;
  };
  conv_ws(E.stem, 0);
  conv_ws(E.tail, 0);
  wg = std::max(wg, tail_wgrad_ws(c[0], E.V[0], B));
  {
    size_t s = norm_act_bwd_ws(E.V[0], c[0], B);
    if (s > na) na = s;
  }
  for (auto& bl : E.enc) blk_ws(bl);
  blk_ws(E.neck);
  for (auto& bl : E.dec) blk_ws(bl);
  E.wg_ws_bytes = wg;
  E.na_ws_bytes = na;
  // packed tcgen05 weight tiles, refreshed from theta at the start of every forward
  size_t tcws = 0;  // split-K partials of the tcgen05 convs (max over layers)
  auto packs = [&](ConvP& cv, bool need_dgrad, int lvl) {
    cv.tcf = conv_tc_layer(cv.cin, cv.cout, cv.ks, cv.stride, 0, E.d.precision, E.V[lvl], &cv.tdf);
    cv.tcd = need_dgrad && conv_tc_layer(cv.cin, cv.cout, cv.ks, cv.stride, 1, E.d.precision, E.V[lvl], &cv.tdd);
    cv.pkf = cv.tcf ? takef((long long)B * conv_tc_pack_floats(cv.tdf.K, cv.tdf.N)) : nullptr;
    cv.pkd = cv.tcd ? takef((long long)B * conv_tc_pack_floats(cv.tdd.K, cv.tdd.N)) : nullptr;
    if (cv.tcf)
      tcws = std::max(tcws, conv_tc_ws_bytes(E.D[lvl], E.H[lvl], E.W[lvl], cv.tdf.K, cv.tdf.N, B, cv.tdf.mode));
    if (cv.tcd)
      tcws = std::max(tcws, conv_tc_ws_bytes(E.D[lvl], E.H[lvl], E.W[lvl], cv.tdd.K, cv.tdd.N, B, cv.tdd.mode));
  };
  packs(E.stem, false, 0);
  packs(E.tail, true, 0);
  for (auto* v : {&E.enc, &E.dec})
    for (auto& bl : *v) {
      packs(bl.c1, true, bl.lout);
      packs(bl.c2, true, bl.lout);
      packs(bl.sk, true, bl.lout);
    }
  packs(E.neck.c1, true, E.neck.lout);
  packs(E.neck.c2, true, E.neck.lout);
  packs(E.neck.sk, true, E.neck.lout);
  E.tc_ws_bytes = tcws;
}

// Assign workspace pointers (base may be null: size query). Returns bytes.
static size_t plan_workspace(d2ip_engine& E, char* base) {
  Arena A{base};
  E.twins.clear();
  const int B = E.d.batch;
  if (E.d.arch == D2IP_ARCH_FAST_RESUNET)
    refnet_plan_workspace(E, A);
  else
    config_plan_workspace(E, A);
  // data term
  const int M = E.d.M, Vp = E.d.Vp;
  E.nseg = jac_nseg(Vp);
  E.rsplit = jac_adj_rows(M, Vp, B);
  E.sigma_c = A.f((long long)B * Vp);
  E.rs = A.f((long long)B * M);
  E.jpart = A.f((long long)B * M * E.nseg);
  E.adjpart = reinterpret_cast<float*>(A.take(jac_adj_ws(M, Vp, B)));
  E.gtail = A.f((long long)B * E.V[0]);
  E.gmapped = A.f((long long)B * E.V[0]);
  E.n_reg = tv_nblocks(E.V[0]);
  E.regpart = A.f((long long)B * E.n_reg);
  E.wg_ws = A.take(E.wg_ws_bytes);
  for (auto& w : E.lane_ws) w = A.take(E.wg_ws_bytes);
  E.na_ws = A.take(E.na_ws_bytes);
  E.tc_ws = E.tc_ws_bytes ? reinterpret_cast<float*>(A.take(E.tc_ws_bytes)) : nullptr;
  E.tc_ws2 = E.tc_ws_bytes ? reinterpret_cast<float*>(A.take(E.tc_ws_bytes)) : nullptr;
  return A.total();
}

// Views of every block's input / output / gradients (after plan_workspace).
static void plan_views(d2ip_engine& E) {
  const int* c = E.d.channels;
  const int L = E.L;
  for (int i = 1; i < L; ++i) {
    Block& bl = E.enc[i - 1];
    const int l = i - 1;
    bl.x = view(E, E.cat[l] + c[l + 1], l, c[l], E.catw[l]);
    bl.gx = view(E, E.gcat[l] + c[l + 1], l, c[l], E.catw[l]);
    bl.gx_acc = 1;  // the decoder's concat gradient is already there
    if (i < L - 1) {
      bl.out = view(E, E.cat[i] + c[i + 1], i, c[i], E.catw[i]);
      bl.gout = view(E, E.gcat[i] + c[i + 1], i, c[i], E.catw[i]);
    } else {
      bl.out = view(E, E.elast, i, c[i], c[i]);
      bl.gout = view(E, E.gelast, i, c[i], c[i]);
    }
  }
  E.neck.x = view(E, E.elast, L - 1, c[L - 1], c[L - 1]);
  E.neck.gx = view(E, E.gelast, L - 1, c[L - 1], c[L - 1]);
  E.neck.gx_acc = 0;
  E.neck.out = view(E, E.bout, L - 1, c[L - 1], c[L - 1]);
  E.neck.gout = view(E, E.gbout, L - 1, c[L - 1], c[L - 1]);
  for (size_t j = 0; j < E.dec.size(); ++j) {
    Block& bl = E.dec[j];
    const int l = bl.lout;
    bl.x = view(E, E.cat[l], l, E.catw[l], E.catw[l]);
    bl.gx = view(E, E.gcat[l], l, E.catw[l], E.catw[l]);
    bl.gx_acc = 0;
    bl.out = view(E, E.decout[l], l, c[l], c[l]);
    bl.gout = view(E, E.gdecout[l], l, c[l], c[l]);
  }
}

// ---------------------------------------------------------------------------



// Forward conv; with `sk`, a split-K tcgen05 result is left as partials for
// the consuming LayerNorm kernel to reduce (one launch fewer per layer).
// Split-K partial buffer of the stream a convolution runs on (main or side2):
// concurrent convolutions must not share one.
static float* tcws(Ctx& k) { return k.st == k.E.side2 ? k.E.tc_ws2 : k.E.tc_ws; }

int cfwd(Ctx& k, const ConvP& c, d2ip_act x, d2ip_act y, int acc, SplitK* sk, const LnFuse* ln, int* fused) {
  if (fused) *fused = 0;
  if (c.tcf) {
    int kspl = 0;
    D2IP_RET(conv_tc_run(x, c.pkf, c.tdf.K, c.tdf.N, k.th() + c.ob, k.pbs, y, acc, tcws(k), k.E.tc_ws_bytes, k.B,
                         k.st, sk && !acc ? &kspl : nullptr, c.tdf.mode, ln, fused));
    if (sk) *sk = kspl ? SplitK{tcws(k), kspl, k.th() + c.ob, k.pbs} : SplitK{};
    return D2IP_OK;
  }
  if (sk) *sk = SplitK{};
  return conv_fwd_direct(x, k.th() + c.ow, k.th() + c.ob, k.pbs, c.ks, c.stride, y, acc, k.B, k.st, c.dil);
}

// With `sk`, a split-K tcgen05 data gradient is left as partials for the
// consuming LayerNorm backward to reduce (as the forward does).
int cdgrad(Ctx& k, const ConvP& c, d2ip_act gy, d2ip_act gx, int acc, SplitK* sk) {
  if (c.tcd) {
    int kspl = 0;
    D2IP_RET(conv_tc_run(gy, c.pkd, c.tdd.K, c.tdd.N, nullptr, 0, gx, acc, tcws(k), k.E.tc_ws_bytes, k.B, k.st,
                         sk && !acc ? &kspl : nullptr, c.tdd.mode));
    if (sk) *sk = kspl ? SplitK{tcws(k), kspl, nullptr, 0} : SplitK{};
    return D2IP_OK;
  }
  if (sk) *sk = SplitK{};
  return conv_dgrad_direct(gy, k.th() + c.ow, k.pbs, c.ks, c.stride, gx, acc, k.B, k.st, c.dil);
}

// study knob (timing only, wrong results): D2IP_SKIP=1 skips the weight gradients, 2 the J passes
static int skip_mask() {
  static const int m = [] {
    const char* v = getenv("D2IP_SKIP");
    return v ? atoi(v) : 0;
  }();
  return m;
}

int cwgrad(Ctx& k, const ConvP& c, d2ip_act x, d2ip_act gy) {
  if (skip_mask() & 1) return D2IP_OK;
  if (c.dil != 1)
    return conv_wgrad_direct(x, gy, c.ks, c.stride, k.gr() + c.ow, k.pbs, k.wgws, k.E.wg_ws_bytes, k.B, k.st, c.dil);
  return conv_wgrad(x, gy, c.ks, c.stride, k.gr() + c.ow, k.pbs, k.wgws, k.E.wg_ws_bytes, k.prec, k.B, k.st);
}

int fork_to(Ctx& k, cudaStream_t from, cudaStream_t to) {
  cudaEvent_t e = k.E.ev[k.E.evi++ % d2ip_engine::kEvents];
  D2IP_CUDA(cudaEventRecord(e, from));
  D2IP_CUDA(cudaStreamWaitEvent(to, e, 0));
  return D2IP_OK;
}

int side_ctx(Ctx& k, Ctx& ks) {
  d2ip_engine& E = k.E;
  const int i = E.lane_next++ % E.nlanes;
  D2IP_RET(fork_to(k, k.st, E.lane[i]));
  k.lanes |= 1u << i;
  ks.st = E.lane[i];  // ks: a copy of k made by the caller
  ks.wgws = E.lane_ws[i];
  return D2IP_OK;
}

int join_side(Ctx& k) {
  for (int i = 0; i < d2ip_engine::kLanes; ++i)
    if (k.lanes & (1u << i)) D2IP_RET(fork_to(k, k.E.lane[i], k.st));
  k.lanes = 0;
  return D2IP_OK;
}

int cwgrad_side(Ctx& k, const ConvP& c, d2ip_act x, d2ip_act gy) {
  Ctx ks = k;
  D2IP_RET(side_ctx(k, ks));
  return cwgrad(ks, c, x, gy);
}

// Level-0 weight gradients (the largest: ~150 us each at cfg2, every SM's shared memory) are
// leaves of the backward graph. Launched where their inputs appear they run beside the level-0
// data gradients, which fill the GPU too; deferred by D2IP_WG_DEFER decoder blocks they run
// beside the deep levels' small, latency-bound kernels instead.
struct DeferredWg {
  const ConvP* c;
  d2ip_act x, gy;
};
static thread_local std::vector<DeferredWg> g_deferred;
static int defer_blocks() {
  static const int n = [] {
    const char* v = getenv("D2IP_WG_DEFER");
    return v ? atoi(v) : 0;
  }();
  return n;
}
static int cwgrad_level(Ctx& k, const ConvP& c, d2ip_act x, d2ip_act gy, int level) {
  if (defer_blocks() > 0 && level == 0) {
    g_deferred.push_back(DeferredWg{&c, x, gy});
    return D2IP_OK;
  }
  return cwgrad_side(k, c, x, gy);
}
static int flush_deferred(Ctx& k) {
  for (const DeferredWg& d : g_deferred) D2IP_RET(cwgrad_side(k, *d.c, d.x, d.gy));
  g_deferred.clear();
  return D2IP_OK;
}

// The job table of every tcgen05 layer's weight packs (built once at bind).
static void build_pack_jobs(d2ip_engine& E) {
  PackJobs& j = E.packjobs;
  j = PackJobs{};
  j.wbs = E.nparams;
  auto add = [&](const ConvP& c) {
    if (c.tcf) pack_jobs_add(j, E.b.theta + c.ow, c.tdf.K, c.tdf.N, c.tdf.pack, c.pkf);
    if (c.tcd) pack_jobs_add(j, E.b.theta + c.ow, c.tdd.K, c.tdd.N, c.tdd.pack, c.pkd);
  };
  if (E.d.arch == D2IP_ARCH_FAST_RESUNET) {
    refnet_pack_jobs(E);
    return;
  }
  add(E.stem);
  add(E.tail);
  for (auto* v : {&E.enc, &E.dec})
    for (auto& bl : *v) {
      add(bl.c1);
      add(bl.c2);
      add(bl.sk);
    }
  add(E.neck.c1);
  add(E.neck.c2);
  add(E.neck.sk);
}

static int pack_all(Ctx& k) { return conv_tc_pack_multi(k.E.packjobs, k.B, k.st); }

static int block_fwd(Ctx& k, Block& bl) {
  d2ip_engine& E = k.E;
  const int co = bl.c1.cout;
  d2ip_act raw = view(E, E.raw, bl.lout, co, co);
  d2ip_act raw2 = view(E, E.raw2, bl.lout, co, co);
  d2ip_act h1 = view(E, bl.h1, bl.lout, co, co);
  d2ip_act none{};
  // 1^3 skip (direct kernel) on side2, beside the conv1 -> norm1 -> conv2 chain
  D2IP_RET(fork_to(k, k.st, k.side2));
  {
    Ctx k2 = k;
    k2.st = k.side2;
    D2IP_RET(cfwd(k2, bl.sk, bl.x, raw2, 0));
  }
  SplitK sk;
  // LayerNorm (+ LeakyReLU) in the conv epilogue where the plan allows it (kw-folded, one N
  // slice, no split-K); otherwise the raw output and a norm_act_fwd launch
  LnFuse l1;
  l1.gamma = k.th() + bl.n1.og;
  l1.beta = k.th() + bl.n1.ob;
  l1.pbs = k.pbs;
  l1.out = h1;
  l1.xhat = bl.xh1;
  l1.rstd = bl.rs1;
  l1.slope = k.slope;
  int f1 = 0;
  D2IP_RET(cfwd(k, bl.c1, bl.x, raw, 0, &sk, &l1, &f1));
  if (!f1)
    D2IP_RET(norm_act_fwd(raw, k.th() + bl.n1.og, k.th() + bl.n1.ob, k.pbs, none, 1, k.slope, h1, bl.xh1, bl.rs1,
                          k.B, k.st, sk));
  D2IP_RET(fork_to(k, k.side2, k.st));  // join the skip before the residual add (conv2's epilogue)
  LnFuse l2 = l1;
  l2.gamma = k.th() + bl.n2.og;
  l2.beta = k.th() + bl.n2.ob;
  l2.res = raw2;
  l2.out = bl.out;
  l2.xhat = bl.xh2;
  l2.rstd = bl.rs2;
  int f2 = 0;
  D2IP_RET(cfwd(k, bl.c2, h1, raw, 0, &sk, &l2, &f2));
  if (!f2)
    D2IP_RET(norm_act_fwd(raw, k.th() + bl.n2.og, k.th() + bl.n2.ob, k.pbs, raw2, 1, k.slope, bl.out, bl.xh2,
                          bl.rs2, k.B, k.st, sk));
  return D2IP_OK;
}

// Side-stream sum of a norm's dgamma/dbeta partials (per-norm buffer `np`).
static int dgb_side(Ctx& k, const float* np, int nb, int C, long long og) {
  Ctx ks = k;
  D2IP_RET(side_ctx(k, ks));
  return reduce_chunks(np, nb, 2 * C, k.gr() + og, k.pbs, k.B, ks.st);
}

static int block_bwd(Ctx& k, Block& bl) {
  d2ip_engine& E = k.E;
  const int co = bl.c1.cout;
  auto S = [&](int i) { return view(E, E.sc[i], bl.lout, co, co); };
  auto P = [&](float* p) { return view(E, p, bl.lout, co, co); };
  // gpre / gc2 / gc1 feed the side-stream kernels: per-block buffers
  d2ip_act gpre = P(bl.gpre), gc2 = P(bl.gc2), gh1 = S(2), gpre1 = S(3), gc1 = P(bl.gc1);
  d2ip_act h1 = view(E, bl.h1, bl.lout, co, co);
  const size_t npb = norm_act_bwd_ws(E.V[bl.lout], co, k.B);
  int nb = 0;
  D2IP_RET(norm_act_bwd(bl.gout, bl.out, 1, k.slope, bl.xh2, bl.rs2, k.th() + bl.n2.og, k.pbs, gpre, gc2,
                        k.gr() + bl.n2.og, k.pbs, bl.np2, npb, k.B, k.st, &nb));
  D2IP_RET(dgb_side(k, bl.np2, nb, co, bl.n2.og));
  D2IP_RET(cwgrad_level(k, bl.c2, h1, gc2, bl.lout));
  D2IP_RET(cwgrad_level(k, bl.sk, bl.x, gpre, bl.lout));
  // side2: the 1^3 skip's data gradient writes gx first; conv1's accumulates after the join
  D2IP_RET(fork_to(k, k.st, k.side2));
  {
    Ctx k2 = k;
    k2.st = k.side2;
    D2IP_RET(cdgrad(k2, bl.sk, gpre, bl.gx, bl.gx_acc));
  }
  SplitK skd;
  D2IP_RET(cdgrad(k, bl.c2, gc2, gh1, 0, &skd));
  D2IP_RET(norm_act_bwd(gh1, h1, 1, k.slope, bl.xh1, bl.rs1, k.th() + bl.n1.og, k.pbs, gpre1, gc1,
                        k.gr() + bl.n1.og, k.pbs, bl.np1, npb, k.B, k.st, &nb, skd));
  D2IP_RET(dgb_side(k, bl.np1, nb, co, bl.n1.og));
  D2IP_RET(cwgrad_level(k, bl.c1, bl.x, gc1, bl.lout));
  D2IP_RET(fork_to(k, k.side2, k.st));
  D2IP_RET(cdgrad(k, bl.c1, gc1, bl.gx, 1));
  return D2IP_OK;
}

static int forward(Ctx& k) {
  d2ip_engine& E = k.E;
  if (E.d.arch == D2IP_ARCH_FAST_RESUNET) {
    D2IP_RET(pack_all(k));
    return refnet_forward(k);
  }
  const int* c = E.d.channels;
  const int L = E.L;
  d2ip_act z = view(E, const_cast<float*>(E.b.z), 0, E.d.in_channels, E.d.in_channels);
  d2ip_act raw = view(E, E.raw, 0, c[0], c[0]);
  d2ip_act a0 = view(E, E.cat[0] + c[1], 0, c[0], E.catw[0]);
  d2ip_act none{};
  D2IP_RET(pack_all(k));
  SplitK sk;
  LnFuse ls;
  ls.gamma = k.th() + E.stem_n.og;
  ls.beta = k.th() + E.stem_n.ob;
  ls.pbs = k.pbs;
  ls.out = a0;
  ls.xhat = E.stem_xh;
  ls.rstd = E.stem_rs;
  ls.slope = k.slope;
  int fs = 0;
  D2IP_RET(cfwd(k, E.stem, z, raw, 0, &sk, &ls, &fs));
  if (!fs)
    D2IP_RET(norm_act_fwd(raw, k.th() + E.stem_n.og, k.th() + E.stem_n.ob, k.pbs, none, 1, k.slope, a0, E.stem_xh,
                          E.stem_rs, k.B, k.st, sk));
  for (auto& bl : E.enc) D2IP_RET(block_fwd(k, bl));
  D2IP_RET(block_fwd(k, E.neck));
  for (size_t j = 0; j < E.dec.size(); ++j) {
    Block& bl = E.dec[j];
    const int l = bl.lout;
    d2ip_act prev = (j == 0) ? E.neck.out : E.dec[j - 1].out;
    d2ip_act up = view(E, E.cat[l], l, c[l + 1], E.catw[l]);
    D2IP_RET(upsample2x_fwd(prev, up, k.B, k.st));
    D2IP_RET(block_fwd(k, bl));
  }
  (void)L;
  const float lo = E.d.lo;
  const float scale = (float)((double)E.d.hi - (double)E.d.lo);
  D2IP_RET(tail_fwd(E.dec.back().out, k.th() + E.tail.ow, k.th() + E.tail.ob, k.pbs, lo, scale, E.b.sig, E.b.mapped,
                    E.sigma_c, E.d.Vp, E.b.col_of_vox, k.B, k.st));
  return D2IP_OK;
}

static bool tv_on(const d2ip_engine& E) { return E.d.lambda_tv > 0.f; }

static int loss(Ctx& k) {
  d2ip_engine& E = k.E;
  const long long jbs = E.d.j_shared ? 0 : (long long)E.d.M * E.d.Vp;
  if (tv_on(E))
    D2IP_RET(tv_fwd_bwd(E.b.mapped, E.b.history, E.d.max_history, E.b.status, E.d.R, E.d.C, E.d.P,
                        E.d.lambda_tv, E.d.lambda_s, E.d.lambda_t, E.d.tv_eps, E.gmapped, E.regpart, k.B, k.st));
  if (!(skip_mask() & 2))
    D2IP_RET(jac_fwd_partial(E.b.J, jbs, E.sigma_c, E.d.Vp, E.d.M, E.d.Vp, E.jpart, E.nseg, k.B, k.st));
  D2IP_RET(jac_loss(E.jpart, E.nseg, E.d.M, E.b.dv, E.d.n_rhs, E.d.data_norm, E.regpart, tv_on(E) ? E.n_reg : 0,
                    E.d.lambda_tv, E.rs, E.b.trace, E.d.max_iters, E.b.status, k.B, k.st));
  return D2IP_OK;
}

static int backward(Ctx& k) {
  d2ip_engine& E = k.E;
  const int* c = E.d.channels;
  const long long jbs = E.d.j_shared ? 0 : (long long)E.d.M * E.d.Vp;
  const float scale = (float)((double)E.d.hi - (double)E.d.lo);
  if (!(skip_mask() & 2)) D2IP_RET(jac_adj_partial(E.b.J, jbs, E.rs, E.d.M, E.d.Vp, E.adjpart, E.rsplit, k.B, k.st));
  if (tv_on(E)) {
    D2IP_RET(jac_adj_finish(E.adjpart, E.rsplit, E.d.Vp, E.d.V, E.b.vox_of_col, E.b.sig, scale, E.gmapped, E.V[0],
                            1, k.B, k.st));
    D2IP_RET(tail_bwd_prep(E.gmapped, E.b.sig, scale, E.gtail, E.V[0], k.B, k.st));
  } else {
    D2IP_RET(jac_adj_finish(E.adjpart, E.rsplit, E.d.Vp, E.d.V, E.b.vox_of_col, E.b.sig, scale, E.gtail, E.V[0],
                            0, k.B, k.st));
  }
  if (E.d.arch == D2IP_ARCH_FAST_RESUNET) {
    D2IP_RET(refnet_backward(k));
    return join_side(k);
  }
  d2ip_act gt = view(E, E.gtail, 0, 1, 1);
  Block& last = E.dec.back();
  if (tail_bwd_supported(last.out)) {  // C_out = 1: lane-group kernels (no GEMM shape to tile)
    Ctx ks = k;
    D2IP_RET(side_ctx(k, ks));
    if (!(skip_mask() & 1))
      D2IP_RET(tail_wgrad(last.out, E.gtail, k.gr() + E.tail.ow, k.pbs, ks.wgws, E.wg_ws_bytes, k.B, ks.st));
    D2IP_RET(tail_dgrad(E.gtail, k.th() + E.tail.ow, k.pbs, last.gout, k.B, k.st));
  } else {
    D2IP_RET(cwgrad_side(k, E.tail, last.out, gt));
    D2IP_RET(cdgrad(k, E.tail, gt, last.gout, 0));
  }
  for (int j = (int)E.dec.size() - 1; j >= 0; --j) {
    Block& bl = E.dec[j];
    const int l = bl.lout;
    D2IP_RET(block_bwd(k, bl));
    d2ip_act gup = view(E, E.gcat[l], l, c[l + 1], E.catw[l]);
    d2ip_act gprev = (j == 0) ? E.neck.gout : E.dec[j - 1].gout;
    D2IP_RET(upsample2x_bwd(gup, gprev, 0, k.B, k.st));
    if ((int)E.dec.size() - j == defer_blocks()) D2IP_RET(flush_deferred(k));
  }
  D2IP_RET(block_bwd(k, E.neck));
  if ((int)E.dec.size() + 1 == defer_blocks()) D2IP_RET(flush_deferred(k));
  for (int i = (int)E.enc.size() - 1; i >= 0; --i) {
    if (i == 0) D2IP_RET(flush_deferred(k));  // enc[0] is level 0 again
    D2IP_RET(block_bwd(k, E.enc[i]));
  }
  D2IP_RET(flush_deferred(k));
  // stem: LN/act backward + weight gradient (no data gradient: Z is fixed)
  d2ip_act a0 = view(E, E.cat[0] + c[1], 0, c[0], E.catw[0]);
  d2ip_act ga0 = view(E, E.gcat[0] + c[1], 0, c[0], E.catw[0]);
  d2ip_act gpre = view(E, E.sc[0], 0, c[0], c[0]);
  d2ip_act gc = view(E, E.stem_gc, 0, c[0], c[0]);
  int nb = 0;
  D2IP_RET(norm_act_bwd(ga0, a0, 1, k.slope, E.stem_xh, E.stem_rs, k.th() + E.stem_n.og, k.pbs, gpre, gc,
                        k.gr() + E.stem_n.og, k.pbs, E.stem_np, norm_act_bwd_ws(E.V[0], c[0], k.B), k.B, k.st, &nb));
  D2IP_RET(dgb_side(k, E.stem_np, nb, c[0], E.stem_n.og));
  d2ip_act z = view(E, const_cast<float*>(E.b.z), 0, E.d.in_channels, E.d.in_channels);
  D2IP_RET(cwgrad_side(k, E.stem, z, gc));
  return join_side(k);
}

static int adam(Ctx& k) {
  d2ip_engine& E = k.E;
  // one segment per sequence: each reads its own step / bad flag (status[b * 4 + {0, 1}])
  return adam_flat(E.b.theta, E.b.grad, E.b.adam_m, E.b.adam_v, (long long)E.nparams, E.d.lr, E.d.beta1,
                   E.d.beta2, E.d.eps, E.b.status, E.b.status + 1, k.st, k.B, 4);
}

static Ctx ctx(d2ip_engine& E, void* stream) {
  return Ctx{E, S(stream), E.d.batch, E.nparams, E.d.precision, E.d.negative_slope, E.side2, E.wg_ws, 0u};
}

int engine_step(d2ip_engine& E, void* stream) {
  Ctx k = ctx(E, stream);
  D2IP_RET(forward(k));
  D2IP_RET(loss(k));
  D2IP_RET(backward(k));
  D2IP_RET(adam(k));
  return D2IP_OK;
}

int engine_grads(d2ip_engine& E, void* stream) {
  Ctx k = ctx(E, stream);
  D2IP_RET(forward(k));
  D2IP_RET(loss(k));
  D2IP_RET(backward(k));
  return D2IP_OK;
}

int engine_predict(d2ip_engine& E, float* y, void* stream) {
  Ctx k = ctx(E, stream);
  D2IP_RET(forward(k));
  const long long jbs = E.d.j_shared ? 0 : (long long)E.d.M * E.d.Vp;
  D2IP_RET(jac_fwd_partial(E.b.J, jbs, E.sigma_c, E.d.Vp, E.d.M, E.d.Vp, E.jpart, E.nseg, k.B, k.st));
  return jac_sum(E.jpart, E.nseg, E.d.M, y, k.B, k.st);
}

int engine_forward(d2ip_engine& E, int with_loss, void* stream) {
  Ctx k = ctx(E, stream);
  D2IP_RET(forward(k));
  if (with_loss) D2IP_RET(loss(k));
  return D2IP_OK;
}

__global__ void status_k(int* status, int batch, int mode, int value) {
  D2IP_PDL_ENTRY();
  const int b = threadIdx.x;
  if (b >= batch) return;
  if (mode == 0) {
    status[b * 4 + 0] = 0;
    status[b * 4 + 1] = 0;
  } else {
    status[b * 4 + 2] = value;
  }
}

int engine_reset_frame(d2ip_engine& E, void* stream) {
  const size_t bytes = (size_t)E.d.batch * E.nparams * sizeof(float);
  D2IP_CUDA(cudaMemsetAsync(E.b.adam_m, 0, bytes, S(stream)));
  D2IP_CUDA(cudaMemsetAsync(E.b.adam_v, 0, bytes, S(stream)));
  D2IP_CUDA(launch_pdl(status_k, 1, 1024, 0, S(stream), E.b.status, E.d.batch, 0, 0));
  D2IP_LAUNCH_CHECK();
  return D2IP_OK;
}

int engine_set_history(d2ip_engine& E, int n, void* stream) {
  D2IP_CHECK_ARG(n >= 0 && n <= E.d.max_history, "history count %d outside [0, %d]", n, E.d.max_history);
  D2IP_CUDA(launch_pdl(status_k, 1, 1024, 0, S(stream), E.b.status, E.d.batch, 1, n));
  D2IP_LAUNCH_CHECK();
  return D2IP_OK;
}

static void drop_graph(d2ip_engine& E) {
  if (E.gexec) cudaGraphExecDestroy(E.gexec);
  if (E.graph) cudaGraphDestroy(E.graph);
  if (E.ggexec) cudaGraphExecDestroy(E.ggexec);
  if (E.ggraph) cudaGraphDestroy(E.ggraph);
  E.gexec = nullptr;
  E.graph = nullptr;
  E.ggexec = nullptr;
  E.ggraph = nullptr;
}

// Capture one iteration program (step: forward + loss + backward + Adam; grads: without
// Adam) once on a private non-blocking stream (the caller's stream may be the legacy
// default stream, which cannot be captured); replay it on the caller's stream.
static int capture(d2ip_engine& E, bool grads_only, cudaGraph_t* graph, cudaGraphExec_t* exec) {
  if (!E.cap_stream) D2IP_CUDA(cudaStreamCreateWithFlags(&E.cap_stream, cudaStreamNonBlocking));
  D2IP_CUDA(cudaStreamBeginCapture(E.cap_stream, cudaStreamCaptureModeThreadLocal));
  int rc = grads_only ? engine_grads(E, E.cap_stream) : engine_step(E, E.cap_stream);
  cudaGraph_t g = nullptr;
  cudaError_t ce = cudaStreamEndCapture(E.cap_stream, &g);
  if (rc != D2IP_OK) {
    if (g) cudaGraphDestroy(g);
    return rc;
  }
  D2IP_CUDA(ce);
  *graph = g;
  D2IP_CUDA(cudaGraphInstantiate(exec, g, 0));
  if (!grads_only) {
    size_t n = 0;
    D2IP_CUDA(cudaGraphGetNodes(g, nullptr, &n));
    E.launches = (int)n;
  }
  return D2IP_OK;
}

int engine_run(d2ip_engine& E, int iters, void* stream) {
  cudaStream_t st = S(stream);
  if (!E.gexec) D2IP_RET(capture(E, false, &E.graph, &E.gexec));
  for (int i = 0; i < iters; ++i) D2IP_CUDA(cudaGraphLaunch(E.gexec, st));
  return D2IP_OK;
}

int engine_grads_graph(d2ip_engine& E, void* stream) {
  if (!E.ggexec) D2IP_RET(capture(E, true, &E.ggraph, &E.ggexec));
  D2IP_CUDA(cudaGraphLaunch(E.ggexec, S(stream)));
  return D2IP_OK;
}

}  // namespace d2ip

// ---------------------------------------------------------------------------
extern "C" {

int d2ip_engine_create(const d2ip_net_desc* desc, d2ip_engine** out) {
  using namespace d2ip;
  D2IP_CHECK_ARG(desc && out, "null argument");
  const d2ip_net_desc& d = *desc;
  D2IP_CHECK_ARG(d.levels >= 2 && d.levels <= 8, "levels must be in [2, 8]");
  D2IP_CHECK_ARG(d.batch >= 1, "batch must be >= 1");
  D2IP_CHECK_ARG(d.arch == D2IP_ARCH_CONFIG_RESUNET || d.arch == D2IP_ARCH_FAST_RESUNET, "unknown arch %d", d.arch);
  const int f = 1 << (d.levels - 1);
  D2IP_CHECK_ARG(d.R % f == 0 && d.C % f == 0 && d.P % f == 0, "grid (%d,%d,%d) not divisible by %d", d.R, d.C,
                 d.P, f);
  D2IP_CHECK_ARG(d.Vp % 4 == 0 && d.Vp >= d.V && d.V >= 1, "bad V/Vp");
  D2IP_CHECK_ARG(d.M >= 1 && d.n_rhs >= 1, "bad M / n_rhs");
  D2IP_CHECK_ARG(d.max_iters >= 1, "max_iters must be >= 1");
  for (int l = 0; l < d.levels; ++l) D2IP_CHECK_ARG(d.channels[l] >= 1, "channel count must be positive");
  d2ip_engine* E = new d2ip_engine();
  E->d = d;
  E->L = d.levels;
  for (int l = 0; l < d.levels; ++l) {
    E->D[l] = d.R >> l;
    E->H[l] = d.C >> l;
    E->W[l] = d.P >> l;
    E->V[l] = (long long)E->D[l] * E->H[l] * E->W[l];
  }
  E->nlanes = d.arch == D2IP_ARCH_FAST_RESUNET ? 3 : 2;
  if (const char* v = getenv("D2IP_LANES")) E->nlanes = std::max(1, std::min(d2ip_engine::kLanes, atoi(v)));
  if (d.arch == D2IP_ARCH_FAST_RESUNET) {
    int rc = refnet_plan_params(*E);
    if (rc != D2IP_OK) {
      refnet_destroy(*E);
      delete E;
      return rc;
    }
  } else {
    plan_params(*E);
  }
  E->ws_total = plan_workspace(*E, nullptr);
  *out = E;
  return D2IP_OK;
}

void d2ip_engine_destroy(d2ip_engine* e) {
  if (!e) return;
  d2ip::drop_graph(*e);
  d2ip::refnet_destroy(*e);
  if (e->cap_stream) cudaStreamDestroy(e->cap_stream);
  for (auto l : e->lane)
    if (l) cudaStreamDestroy(l);
  if (e->side2) cudaStreamDestroy(e->side2);
  for (auto ev : e->ev)
    if (ev) cudaEventDestroy(ev);
  delete e;
}

long long d2ip_engine_param_count(const d2ip_engine* e) { return e ? e->nparams : -1; }
size_t d2ip_engine_workspace_bytes(const d2ip_engine* e) { return e ? e->ws_total : 0; }
int d2ip_engine_launches_per_iter(const d2ip_engine* e) { return e ? e->launches : 0; }

int d2ip_engine_bind(d2ip_engine* e, const d2ip_bindings* b) {
  using namespace d2ip;
  D2IP_CHECK_ARG(e && b, "null argument");
  D2IP_CHECK_ARG(b->workspace_bytes >= e->ws_total, "workspace too small: %zu < %zu", b->workspace_bytes,
                 e->ws_total);
  D2IP_CHECK_ARG(b->theta && b->grad && b->adam_m && b->adam_v && b->z && b->J && b->vox_of_col &&
                     b->col_of_vox && b->dv && b->mapped && b->sig && b->trace && b->status,
                 "missing binding");
  D2IP_CHECK_ARG(e->d.lambda_tv <= 0.f || b->history || e->d.max_history == 0, "TV needs a history buffer");
  drop_graph(*e);
  if (!e->side2) {
    for (auto& l : e->lane) D2IP_CUDA(cudaStreamCreateWithFlags(&l, cudaStreamNonBlocking));
    D2IP_CUDA(cudaStreamCreateWithFlags(&e->side2, cudaStreamNonBlocking));
    for (auto& ev : e->ev) D2IP_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  }
  e->b = *b;
  plan_workspace(*e, reinterpret_cast<char*>(b->workspace));
  if (e->d.arch == D2IP_ARCH_FAST_RESUNET)
    refnet_plan_views(*e);
  else
    plan_views(*e);
  build_pack_jobs(*e);
  D2IP_CHECK_ARG(e->packjobs.n <= PackJobs::kMax, "too many tcgen05 layers for one pack launch");
  // one-time zero: J padding columns of sigma_c, unmasked tail gradients
  D2IP_CUDA(cudaMemset(b->workspace, 0, e->ws_total));
  e->bound = true;
  return D2IP_OK;
}

int d2ip_engine_set_history(d2ip_engine* e, int n_history) {
  // stream 0 ordering is not required: the host calls this between frames
  // after a stream synchronisation.
  using namespace d2ip;
  D2IP_CHECK_ARG(e && e->bound, "engine not bound");
  D2IP_RET(engine_set_history(*e, n_history, nullptr));
  D2IP_CUDA(cudaStreamSynchronize(nullptr));
  return D2IP_OK;
}

int d2ip_engine_reset_frame(d2ip_engine* e, void* stream) {
  using namespace d2ip;
  D2IP_CHECK_ARG(e && e->bound, "engine not bound");
  return engine_reset_frame(*e, stream);
}

int d2ip_engine_step(d2ip_engine* e, void* stream) {
  using namespace d2ip;
  D2IP_CHECK_ARG(e && e->bound, "engine not bound");
  return engine_step(*e, stream);
}

int d2ip_engine_grads(d2ip_engine* e, void* stream) {
  using namespace d2ip;
  D2IP_CHECK_ARG(e && e->bound, "engine not bound");
  return engine_grads(*e, stream);
}

int d2ip_engine_grads_graph(d2ip_engine* e, void* stream) {
  using namespace d2ip;
  D2IP_CHECK_ARG(e && e->bound, "engine not bound");
  return engine_grads_graph(*e, stream);
}

int d2ip_engine_run(d2ip_engine* e, int iters, void* stream) {
  using namespace d2ip;
  D2IP_CHECK_ARG(e && e->bound, "engine not bound");
  D2IP_CHECK_ARG(iters >= 0, "iters must be >= 0");
  return engine_run(*e, iters, stream);
}

int d2ip_engine_adam(d2ip_engine* e, void* stream) {
  using namespace d2ip;
  D2IP_CHECK_ARG(e && e->bound, "engine not bound");
  Ctx k = ctx(*e, stream);
  return adam(k);
}

int d2ip_engine_predict(d2ip_engine* e, float* y, void* stream) {
  using namespace d2ip;
  D2IP_CHECK_ARG(e && e->bound && y, "engine not bound / null output");
  return engine_predict(*e, y, stream);
}

int d2ip_engine_forward(d2ip_engine* e, int with_loss, void* stream) {
  using namespace d2ip;
  D2IP_CHECK_ARG(e && e->bound, "engine not bound");
  return engine_forward(*e, with_loss, stream);
}

}  // extern "C"
