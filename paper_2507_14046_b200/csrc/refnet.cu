// The engine's second network program: the reference's own backbone
// FastResUNet3D (priornet.py:183-232) for `batch` sequences in lockstep.
//
//   stem    Conv3d(1,b,3) -> ChannelLayerNorm -> SiLU          priornet.py:201-203
//   enc i   SqueezeExcite(c_i) -> ResConv3d(c_i, c_i+1, s=2)   priornet.py:204-207,223-226
//   neck    ASPP3d(8b, dilations)                              priornet.py:208,151-164
//   dec i   AttentionGate3d(skip_i, x) ; trilinear x2 (x) ;
//           ResConv3d(cat[x_up, gated])                        priornet.py:209-215,228-231
//   tail    Conv3d(b,1,3) -> sigmoid (-> output map)          priornet.py:216,232
//
// Layout as in engine.cu: NDHWC fp32 activations, every parameter in the flat
// state_dict-ordered buffer (priornet.fast_resunet_schema), every saved tensor
// and gradient in the caller's workspace. The concat of the decoder input is a
// pair of channel-strided views of one buffer: the trilinear upsample and the
// attention gate write their halves in place.
#include <algorithm>

#include "engine_impl.h"

namespace d2ip {

struct RBlock {  // ResConv3d (priornet.py:134-148)
  bool dw = false;
  int lin = 0, lout = 0, cin = 0, cout = 0, stride = 1;
  ConvP c1d, c1p, c1;  // depthwise + pointwise, or dense 3^3
  ConvP c2d, c2p, c2;
  NormP n1, n2;
  ConvP sk;
  d2ip_act x{}, gx{}, out{}, gout{};
  int gx_acc = 0;
  float *t1 = nullptr, *h1 = nullptr, *p1 = nullptr, *xh1 = nullptr, *rs1 = nullptr;
  float *t2 = nullptr, *p2 = nullptr, *xh2 = nullptr, *rs2 = nullptr;
  float* sb[7]{};  // backward scratch of this block (side-lane weight gradients read it: not shared)
};

struct SEP {  // SqueezeExcite (priornet.py:120-131)
  ConvP fc1, fc2;
  int C = 0, hid = 0, sbs = 0;
  float* state = nullptr;
};

struct AttP {  // AttentionGate3d (priornet.py:167-180), skip level l, gate level l+1
  ConvP key, query, score;
  int l = 0, inter = 0;
  float *k = nullptr, *q = nullptr, *pre = nullptr, *a = nullptr, *att_c = nullptr, *att_f = nullptr;
  float* sb[4]{};  // backward: gatt_f, gatt_c, ga, gpre
};

struct RefNet {
  int b = 0, ch[4]{};
  ConvP stem;
  NormP stem_n;
  SEP se[3];
  RBlock enc[3];
  int nd = 0;
  ConvP br[8];
  ConvP proj;
  NormP bn;
  AttP att[3];    // decoder order: att[j] gates skip level 2 - j
  RBlock dec[3];  // dec[j] at level 2 - j
  ConvP tail;
  // activations / gradients
  float *x[4]{}, *gx[4]{};    // x[0] stem output, x[i+1] enc block i output
  float *s[3]{}, *gs[3]{};    // SE outputs (the skips)
  float *stem_p = nullptr, *stem_xh = nullptr, *stem_rs = nullptr;
  float *acat = nullptr, *gacat = nullptr, *b_p = nullptr, *b_xh = nullptr, *b_rs = nullptr;
  float *xb = nullptr, *gxb = nullptr;  // bottleneck output
  float *cat[3]{}, *gcat[3]{};           // decoder input at level l: [x_up (c_l+1) | gated (c_l)]
  float *d[3]{}, *gd[3]{};               // decoder output at level l
  float *raw = nullptr, *raw2 = nullptr, *sc[7]{};
  float *asb[2]{}, *ssb[2]{};  // backward scratch of the ASPP norm and the stem norm
  long long maxvc = 0;
};

// ---------------------------------------------------------------------------
// parameters: exact order of priornet.fast_resunet_schema (= state_dict order)

int refnet_plan_params(d2ip_engine& E) {
  const d2ip_net_desc& d = E.d;
  D2IP_CHECK_ARG(d.levels == 4, "FastResUNet3D has 3 encoder stages (levels = 4), got %d", d.levels);
  D2IP_CHECK_ARG(d.in_channels == 1, "FastResUNet3D takes a 1-channel noise volume");
  const int b = d.channels[0];
  D2IP_CHECK_ARG(b >= 4 && b % 4 == 0 && 8 * b <= 256,
                 "FastResUNet3D base_channels must be a multiple of 4 in [4, 32], got %d", b);
  for (int l = 0; l < 4; ++l) D2IP_CHECK_ARG(d.channels[l] == (b << l), "channels must be b, 2b, 4b, 8b");
  D2IP_CHECK_ARG(d.n_dil >= 1 && d.n_dil <= 8, "ASPP needs 1..8 dilations");
  for (int j = 0; j < d.n_dil; ++j)
    D2IP_CHECK_ARG(d.dil[j] >= 1 && (j == 0 || d.dil[j] > d.dil[j - 1]), "aspp dilations must be increasing");
  RefNet* N = new RefNet();
  E.ref = N;
  N->b = b;
  for (int l = 0; l < 4; ++l) N->ch[l] = b << l;
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
  auto dwconv = [&](int C, int stride) {  // Conv3d(C, C, 3, groups=C): weight [C][1][3][3][3]
    ConvP c;
    c.cin = c.cout = C;
    c.ks = 3;
    c.stride = stride;
    c.ow = o;
    o += 27LL * C;
    c.ob = o;
    o += C;
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
  auto rblock = [&](int cin, int cout, int stride, int lin, int lout) {
    RBlock r;
    r.dw = d.depthwise != 0;
    r.cin = cin;
    r.cout = cout;
    r.stride = stride;
    r.lin = lin;
    r.lout = lout;
    if (r.dw) {
      r.c1d = dwconv(cin, stride);
      r.c1p = conv(cin, cout, 1, 1);
    } else {
      r.c1 = conv(cin, cout, 3, stride);
    }
    r.n1 = norm(cout);
    if (r.dw) {
      r.c2d = dwconv(cout, 1);
      r.c2p = conv(cout, cout, 1, 1);
    } else {
      r.c2 = conv(cout, cout, 3, 1);
    }
    r.n2 = norm(cout);
    r.sk = conv(cin, cout, 1, stride);
    return r;
  };
  const int* ch = N->ch;
  N->stem = conv(1, b, 3, 1);
  N->stem_n = norm(b);
  for (int i = 0; i < 3; ++i) {
    SEP& s = N->se[i];
    s.C = ch[i];
    s.hid = std::max(ch[i] / 4, 1);
    s.fc1 = conv(s.C, s.hid, 1, 1);
    s.fc2 = conv(s.hid, s.C, 1, 1);
    s.sbs = (3 * s.C + s.hid + 3) & ~3;
  }
  for (int i = 0; i < 3; ++i) N->enc[i] = rblock(ch[i], ch[i + 1], 2, i, i + 1);
  N->nd = d.n_dil;
  for (int j = 0; j < d.n_dil; ++j) {
    N->br[j] = conv(ch[3], ch[3], 3, 1);
    N->br[j].dil = d.dil[j];
  }
  N->proj = conv(ch[3] * d.n_dil, ch[3], 1, 1);
  N->bn = norm(ch[3]);
  for (int j = 0; j < 3; ++j) {
    const int l = 2 - j;
    AttP& a = N->att[j];
    a.l = l;
    a.inter = std::max(ch[l] / 2, 4);
    a.key = conv(ch[l], a.inter, 1, 2);
    a.query = conv(ch[l + 1], a.inter, 1, 1);
    a.score = conv(a.inter, 1, 1, 1);
  }
  for (int j = 0; j < 3; ++j) {
    const int l = 2 - j;
    N->dec[j] = rblock(ch[l + 1] + ch[l], ch[l], 1, l, l);
  }
  N->tail = conv(b, 1, 3, 1);
  E.nparams = o;
  return D2IP_OK;
}

void refnet_destroy(d2ip_engine& E) {
  delete E.ref;
  E.ref = nullptr;
}

// ---------------------------------------------------------------------------
// workspace

void refnet_plan_workspace(d2ip_engine& E, Arena& A) {
  RefNet& N = *E.ref;
  const int B = E.d.batch;
  const int* ch = N.ch;
  auto act = [&](int l, int c) { return A.f((long long)B * E.V[l] * c); };
  auto vox = [&](int l) { return A.f((long long)B * E.V[l]); };
  long long maxvc = E.V[0] * ch[0];
  auto grow = [&](int l, int c) { maxvc = std::max(maxvc, E.V[l] * c); };
  N.stem_p = act(0, ch[0]);
  N.stem_xh = act(0, ch[0]);
  N.stem_rs = vox(0);
  for (int l = 0; l < 4; ++l) {
    N.x[l] = act(l, ch[l]);
    N.gx[l] = act(l, ch[l]);
  }
  for (int i = 0; i < 3; ++i) {
    N.s[i] = act(i, ch[i]);
    N.gs[i] = act(i, ch[i]);
    N.se[i].state = A.f((long long)B * N.se[i].sbs);
  }
  auto saved = [&](RBlock& r) {
    const int l = r.lout;
    if (r.dw) {
      r.t1 = act(l, r.cin);
      r.t2 = act(l, r.cout);
    }
    r.h1 = act(l, r.cout);
    r.p1 = act(l, r.cout);
    r.xh1 = act(l, r.cout);
    r.rs1 = vox(l);
    r.p2 = act(l, r.cout);
    r.xh2 = act(l, r.cout);
    r.rs2 = vox(l);
    for (auto& p : r.sb) p = act(l, std::max(r.cin, r.cout));
    grow(l, std::max(r.cin, r.cout));
  };
  for (auto& r : N.enc) saved(r);
  for (auto& r : N.dec) saved(r);
  N.acat = act(3, N.nd * ch[3]);
  N.gacat = act(3, N.nd * ch[3]);
  N.b_p = act(3, ch[3]);
  N.b_xh = act(3, ch[3]);
  N.b_rs = vox(3);
  N.xb = act(3, ch[3]);
  N.gxb = act(3, ch[3]);
  N.asb[0] = act(3, ch[3]);
  N.asb[1] = act(3, ch[3]);
  N.ssb[0] = act(0, ch[0]);
  N.ssb[1] = act(0, ch[0]);
  for (auto& a : N.att) {
    const int lg = a.l + 1;
    a.k = act(lg, a.inter);
    a.q = act(lg, a.inter);
    a.pre = act(lg, a.inter);
    a.a = act(lg, a.inter);
    a.att_c = vox(lg);
    a.att_f = vox(a.l);
    a.sb[0] = vox(a.l);
    a.sb[1] = vox(lg);
    a.sb[2] = act(lg, a.inter);
    a.sb[3] = act(lg, a.inter);
    grow(lg, a.inter);
  }
  for (int l = 0; l < 3; ++l) {
    N.cat[l] = act(l, ch[l + 1] + ch[l]);
    N.gcat[l] = act(l, ch[l + 1] + ch[l]);
    N.d[l] = act(l, ch[l]);
    N.gd[l] = act(l, ch[l]);
  }
  N.maxvc = maxvc;
  N.raw = A.f(B * maxvc);
  N.raw2 = A.f(B * maxvc);
  for (auto& p : N.sc) p = A.f(B * maxvc);

  // reduction workspaces (shared by conv wgrad, depthwise wgrad and the SE column sums)
  size_t wg = 0, na = 0;
  auto cws = [&](const ConvP& c, int lout) {
    wg = std::max(wg, conv_wgrad_ws(c.cin, c.cout, c.ks, E.D[lout], E.H[lout], E.W[lout], B, E.d.precision));
  };
  auto nws = [&](int l, int c) { na = std::max(na, norm_act_bwd_ws(E.V[l], c, B)); };
  cws(N.stem, 0);
  nws(0, ch[0]);
  for (int i = 0; i < 3; ++i) wg = std::max(wg, colsum_ws(ch[i], E.V[i], B));
  auto rws = [&](const RBlock& r) {
    if (r.dw) {
      wg = std::max(wg, dw_wgrad_ws(r.cin, E.V[r.lout], B));
      wg = std::max(wg, dw_wgrad_ws(r.cout, E.V[r.lout], B));
      cws(r.c1p, r.lout);
      cws(r.c2p, r.lout);
    } else {
      cws(r.c1, r.lout);
      cws(r.c2, r.lout);
    }
    cws(r.sk, r.lout);
    nws(r.lout, r.cout);
  };
  for (auto& r : N.enc) rws(r);
  for (auto& r : N.dec) rws(r);
  for (int j = 0; j < N.nd; ++j) cws(N.br[j], 3);
  cws(N.proj, 3);
  nws(3, ch[3]);
  for (auto& a : N.att) {
    cws(a.key, a.l + 1);
    cws(a.query, a.l + 1);
    cws(a.score, a.l + 1);
  }
  cws(N.tail, 0);
  E.wg_ws_bytes = wg;
  E.na_ws_bytes = na;

  // tcgen05 weight packs for the dense stride-1 3^3 layers
  size_t tcws = 0;
  auto packs = [&](ConvP& c, bool need_dgrad, int l) {
    c.tcf = c.dil == 1 && conv_tc_layer(c.cin, c.cout, c.ks, c.stride, 0, E.d.precision, E.V[l], &c.tdf);
    c.tcd = need_dgrad && c.dil == 1 && conv_tc_layer(c.cin, c.cout, c.ks, c.stride, 1, E.d.precision, E.V[l], &c.tdd);
    c.pkf = c.tcf ? A.f((long long)B * conv_tc_pack_floats(c.tdf.K, c.tdf.N)) : nullptr;
    c.pkd = c.tcd ? A.f((long long)B * conv_tc_pack_floats(c.tdd.K, c.tdd.N)) : nullptr;
    if (c.tcf) tcws = std::max(tcws, conv_tc_ws_bytes(E.D[l], E.H[l], E.W[l], c.tdf.K, c.tdf.N, B, c.tdf.mode));
    if (c.tcd) tcws = std::max(tcws, conv_tc_ws_bytes(E.D[l], E.H[l], E.W[l], c.tdd.K, c.tdd.N, B, c.tdd.mode));
  };
  packs(N.stem, false, 0);
  packs(N.tail, true, 0);
  for (auto* rs : {N.enc, N.dec})
    for (int i = 0; i < 3; ++i) {
      RBlock& r = rs[i];
      if (!r.dw) {
        packs(r.c1, true, r.lout);
        packs(r.c2, true, r.lout);
      }
    }
  E.tc_ws_bytes = tcws;
}

void refnet_pack_jobs(d2ip_engine& E) {
  RefNet& N = *E.ref;
  PackJobs& j = E.packjobs;
  auto add = [&](const ConvP& c) {
    if (c.tcf) pack_jobs_add(j, E.b.theta + c.ow, c.tdf.K, c.tdf.N, c.tdf.pack, c.pkf);
    if (c.tcd) pack_jobs_add(j, E.b.theta + c.ow, c.tdd.K, c.tdd.N, c.tdd.pack, c.pkd);
  };
  add(N.stem);
  add(N.tail);
  for (auto* rs : {N.enc, N.dec})
    for (int i = 0; i < 3; ++i)
      if (!rs[i].dw) {
        add(rs[i].c1);
        add(rs[i].c2);
      }
}

void refnet_plan_views(d2ip_engine& E) {
  RefNet& N = *E.ref;
  const int* ch = N.ch;
  for (int i = 0; i < 3; ++i) {
    RBlock& r = N.enc[i];
    r.x = view(E, N.s[i], i, ch[i], ch[i]);
    r.gx = view(E, N.gs[i], i, ch[i], ch[i]);
    r.gx_acc = 1;  // the attention gate's skip gradient is already there
    r.out = view(E, N.x[i + 1], i + 1, ch[i + 1], ch[i + 1]);
    r.gout = view(E, N.gx[i + 1], i + 1, ch[i + 1], ch[i + 1]);
  }
  for (int j = 0; j < 3; ++j) {
    RBlock& r = N.dec[j];
    const int l = 2 - j;
    const int w = ch[l + 1] + ch[l];
    r.x = view(E, N.cat[l], l, w, w);
    r.gx = view(E, N.gcat[l], l, w, w);
    r.gx_acc = 0;
    r.out = view(E, N.d[l], l, ch[l], ch[l]);
    r.gout = view(E, N.gd[l], l, ch[l], ch[l]);
  }
}

// ---------------------------------------------------------------------------
// forward

static d2ip_act scratch(d2ip_engine& E, float* p, int l, int c) { return view(E, p, l, c, c); }

static int rblock_fwd(Ctx& k, RBlock& r) {
  d2ip_engine& E = k.E;
  RefNet& N = *E.ref;
  const int l = r.lout;
  const int co = r.cout;
  d2ip_act raw = scratch(E, N.raw, l, co), raw2 = scratch(E, N.raw2, l, co);
  d2ip_act h1 = scratch(E, r.h1, l, co), p1 = scratch(E, r.p1, l, co), p2 = scratch(E, r.p2, l, co);
  d2ip_act none{};
  SplitK sk;
  if (r.dw) {
    d2ip_act t1 = scratch(E, r.t1, l, r.cin);
    D2IP_RET(dw_conv_fwd(r.x, k.th() + r.c1d.ow, k.th() + r.c1d.ob, k.pbs, r.stride, t1, k.B, k.st));
    D2IP_RET(cfwd(k, r.c1p, t1, raw, 0, &sk));
  } else {
    D2IP_RET(cfwd(k, r.c1, r.x, raw, 0, &sk));
  }
  D2IP_RET(norm_act_fwd(raw, k.th() + r.n1.og, k.th() + r.n1.ob, k.pbs, none, 2, 0.f, h1, r.xh1, r.rs1, k.B, k.st,
                        sk, p1));
  if (r.dw) {
    d2ip_act t2 = scratch(E, r.t2, l, co);
    D2IP_RET(dw_conv_fwd(h1, k.th() + r.c2d.ow, k.th() + r.c2d.ob, k.pbs, 1, t2, k.B, k.st));
    D2IP_RET(cfwd(k, r.c2p, t2, raw, 0, &sk));
  } else {
    D2IP_RET(cfwd(k, r.c2, h1, raw, 0, &sk));
  }
  D2IP_RET(cfwd(k, r.sk, r.x, raw2, 0));  // 1^3 skip: direct kernel, leaves split-K partials intact
  D2IP_RET(norm_act_fwd(raw, k.th() + r.n2.og, k.th() + r.n2.ob, k.pbs, raw2, 2, 0.f, r.out, r.xh2, r.rs2, k.B, k.st,
                        sk, p2));
  return D2IP_OK;
}

static int se_fwd(Ctx& k, SEP& s, d2ip_act x, d2ip_act out) {
  d2ip_engine& E = k.E;
  return se_forward(x, k.th() + s.fc1.ow, k.th() + s.fc1.ob, k.th() + s.fc2.ow, k.th() + s.fc2.ob, k.pbs, s.hid,
                    s.state, s.sbs, out, E.wg_ws, E.wg_ws_bytes, k.B, k.st);
}

static int aspp_fwd(Ctx& k) {
  d2ip_engine& E = k.E;
  RefNet& N = *E.ref;
  const int C = N.ch[3];
  const int W = N.nd * C;
  d2ip_act x3 = view(E, N.x[3], 3, C, C);
  for (int j = 0; j < N.nd; ++j) D2IP_RET(cfwd(k, N.br[j], x3, view(E, N.acat + j * C, 3, C, W), 0));
  d2ip_act raw = scratch(E, N.raw, 3, C);
  D2IP_RET(cfwd(k, N.proj, view(E, N.acat, 3, W, W), raw, 0));
  return norm_act_fwd(raw, k.th() + N.bn.og, k.th() + N.bn.ob, k.pbs, d2ip_act{}, 2, 0.f, view(E, N.xb, 3, C, C), N.b_xh,
                      N.b_rs, k.B, k.st, SplitK{}, view(E, N.b_p, 3, C, C));
}

// gated skip into cat[l][:, c_{l+1}:] ; gate = decoder feature at level l+1
static int att_fwd(Ctx& k, AttP& a, d2ip_act skip, d2ip_act gate, d2ip_act gated) {
  d2ip_engine& E = k.E;
  const int lg = a.l + 1;
  d2ip_act kk = scratch(E, a.k, lg, a.inter), qq = scratch(E, a.q, lg, a.inter), aa = scratch(E, a.a, lg, a.inter);
  D2IP_RET(cfwd(k, a.key, skip, kk, 0));
  D2IP_RET(cfwd(k, a.query, gate, qq, 0));
  D2IP_RET(add_silu(kk, qq, a.pre, aa, k.B, k.st));
  d2ip_act sc = scratch(E, a.att_c, lg, 1);
  D2IP_RET(cfwd(k, a.score, aa, sc, 0));
  D2IP_RET(sigmoid_inplace(a.att_c, (long long)k.B * E.V[lg], k.st));
  D2IP_RET(upsample2x_fwd(sc, scratch(E, a.att_f, a.l, 1), k.B, k.st));
  return att_gate_fwd(skip, a.att_f, gated, k.B, k.st);
}

int refnet_forward(Ctx& k) {
  d2ip_engine& E = k.E;
  RefNet& N = *E.ref;
  const int* ch = N.ch;
  d2ip_act z = view(E, const_cast<float*>(E.b.z), 0, 1, 1);
  d2ip_act raw = scratch(E, N.raw, 0, ch[0]);
  SplitK sk;
  D2IP_RET(cfwd(k, N.stem, z, raw, 0, &sk));
  D2IP_RET(norm_act_fwd(raw, k.th() + N.stem_n.og, k.th() + N.stem_n.ob, k.pbs, d2ip_act{}, 2, 0.f,
                        view(E, N.x[0], 0, ch[0], ch[0]), N.stem_xh, N.stem_rs, k.B, k.st, sk,
                        view(E, N.stem_p, 0, ch[0], ch[0])));
  for (int i = 0; i < 3; ++i) {
    D2IP_RET(se_fwd(k, N.se[i], view(E, N.x[i], i, ch[i], ch[i]), view(E, N.s[i], i, ch[i], ch[i])));
    D2IP_RET(rblock_fwd(k, N.enc[i]));
  }
  D2IP_RET(aspp_fwd(k));
  for (int j = 0; j < 3; ++j) {
    const int l = 2 - j;
    const int w = ch[l + 1] + ch[l];
    d2ip_act gate = (j == 0) ? view(E, N.xb, 3, ch[3], ch[3]) : N.dec[j - 1].out;
    D2IP_RET(att_fwd(k, N.att[j], view(E, N.s[l], l, ch[l], ch[l]), gate, view(E, N.cat[l] + ch[l + 1], l, ch[l], w)));
    D2IP_RET(upsample2x_fwd(gate, view(E, N.cat[l], l, ch[l + 1], w), k.B, k.st));
    D2IP_RET(rblock_fwd(k, N.dec[j]));
  }
  const float lo = E.d.lo;
  const float scale = (float)((double)E.d.hi - (double)E.d.lo);
  return tail_fwd(N.dec[2].out, k.th() + N.tail.ow, k.th() + N.tail.ob, k.pbs, lo, scale, E.b.sig, E.b.mapped,
                  E.sigma_c, E.d.Vp, E.b.col_of_vox, k.B, k.st);
}

// ---------------------------------------------------------------------------
// backward

// depthwise weight gradient on a side lane (its own reduction workspace)
static int dw_wgrad_side(Ctx& k, d2ip_act x, d2ip_act gy, int stride, float* gw) {
  Ctx ks = k;
  D2IP_RET(side_ctx(k, ks));
  return dw_conv_wgrad(x, gy, stride, gw, k.pbs, ks.wgws, k.E.wg_ws_bytes, k.B, ks.st);
}

static int rblock_bwd(Ctx& k, RBlock& r) {
  d2ip_engine& E = k.E;
  const int l = r.lout;
  const int co = r.cout;
  auto S = [&](int i, int c) { return scratch(E, r.sb[i], l, c); };
  d2ip_act gpre = S(0, co), gc2 = S(1, co), gh1 = S(2, co), gpre1 = S(3, co), gc1 = S(4, co);
  d2ip_act h1 = scratch(E, r.h1, l, co), p1 = scratch(E, r.p1, l, co), p2 = scratch(E, r.p2, l, co);
  // norm2 (+ skip residual) + SiLU; `out` slot carries the saved pre-activation
  D2IP_RET(norm_act_bwd(r.gout, p2, 2, 0.f, r.xh2, r.rs2, k.th() + r.n2.og, k.pbs, gpre, gc2, k.gr() + r.n2.og, k.pbs,
                        E.na_ws, E.na_ws_bytes, k.B, k.st));
  if (r.dw) {
    d2ip_act t2 = scratch(E, r.t2, l, co), gt2 = S(5, co);
    D2IP_RET(cwgrad_side(k, r.c2p, t2, gc2));
    D2IP_RET(cdgrad(k, r.c2p, gc2, gt2, 0));
    D2IP_RET(dw_wgrad_side(k, h1, gt2, 1, k.gr() + r.c2d.ow));
    D2IP_RET(dw_conv_dgrad(gt2, k.th() + r.c2d.ow, k.pbs, 1, gh1, 0, k.B, k.st));
  } else {
    D2IP_RET(cwgrad_side(k, r.c2, h1, gc2));
    D2IP_RET(cdgrad(k, r.c2, gc2, gh1, 0));
  }
  D2IP_RET(norm_act_bwd(gh1, p1, 2, 0.f, r.xh1, r.rs1, k.th() + r.n1.og, k.pbs, gpre1, gc1, k.gr() + r.n1.og, k.pbs,
                        E.na_ws, E.na_ws_bytes, k.B, k.st));
  if (r.dw) {
    d2ip_act t1 = scratch(E, r.t1, l, r.cin), gt1 = S(6, r.cin);
    D2IP_RET(cwgrad_side(k, r.c1p, t1, gc1));
    D2IP_RET(cdgrad(k, r.c1p, gc1, gt1, 0));
    D2IP_RET(dw_wgrad_side(k, r.x, gt1, r.stride, k.gr() + r.c1d.ow));
    D2IP_RET(dw_conv_dgrad(gt1, k.th() + r.c1d.ow, k.pbs, r.stride, r.gx, r.gx_acc, k.B, k.st));
  } else {
    D2IP_RET(cwgrad_side(k, r.c1, r.x, gc1));
    D2IP_RET(cdgrad(k, r.c1, gc1, r.gx, r.gx_acc));
  }
  D2IP_RET(cwgrad_side(k, r.sk, r.x, gpre));
  D2IP_RET(cdgrad(k, r.sk, gpre, r.gx, 1));
  return D2IP_OK;
}

// gg = gradient of the gated skip; writes gs (skip, first writer) and
// accumulates the gate gradient into ggate (already holding the upsample part).
static int att_bwd(Ctx& k, AttP& a, d2ip_act skip, d2ip_act gate, d2ip_act gg, d2ip_act gs, d2ip_act ggate) {
  d2ip_engine& E = k.E;
  const int lg = a.l + 1;
  float* gatt_f = a.sb[0];
  float* gatt_c = a.sb[1];
  D2IP_RET(att_gate_bwd(gg, skip, a.att_f, gs, 0, gatt_f, k.B, k.st));
  d2ip_act gc = scratch(E, gatt_c, lg, 1);
  D2IP_RET(upsample2x_bwd(scratch(E, gatt_f, a.l, 1), gc, 0, k.B, k.st));
  D2IP_RET(sigmoid_bwd(gatt_c, a.att_c, (long long)k.B * E.V[lg], k.st));
  d2ip_act aa = scratch(E, a.a, lg, a.inter);
  d2ip_act ga = scratch(E, a.sb[2], lg, a.inter), gpre = scratch(E, a.sb[3], lg, a.inter);
  D2IP_RET(cwgrad_side(k, a.score, aa, gc));
  D2IP_RET(cdgrad(k, a.score, gc, ga, 0));
  D2IP_RET(silu_bwd(ga, a.pre, gpre, k.B, k.st));
  D2IP_RET(cwgrad_side(k, a.key, skip, gpre));
  D2IP_RET(cdgrad(k, a.key, gpre, gs, 1));
  D2IP_RET(cwgrad_side(k, a.query, gate, gpre));
  D2IP_RET(cdgrad(k, a.query, gpre, ggate, 1));
  return D2IP_OK;
}

static int aspp_bwd(Ctx& k) {
  d2ip_engine& E = k.E;
  RefNet& N = *E.ref;
  const int C = N.ch[3];
  const int W = N.nd * C;
  d2ip_act gpre = scratch(E, N.asb[0], 3, C), gc = scratch(E, N.asb[1], 3, C);
  D2IP_RET(norm_act_bwd(view(E, N.gxb, 3, C, C), view(E, N.b_p, 3, C, C), 2, 0.f, N.b_xh, N.b_rs, k.th() + N.bn.og,
                        k.pbs, gpre, gc, k.gr() + N.bn.og, k.pbs, E.na_ws, E.na_ws_bytes, k.B, k.st));
  d2ip_act cat = view(E, N.acat, 3, W, W), gcat = view(E, N.gacat, 3, W, W);
  D2IP_RET(cwgrad_side(k, N.proj, cat, gc));
  D2IP_RET(cdgrad(k, N.proj, gc, gcat, 0));
  d2ip_act x3 = view(E, N.x[3], 3, C, C), gx3 = view(E, N.gx[3], 3, C, C);
  for (int j = 0; j < N.nd; ++j) {
    d2ip_act gj = view(E, N.gacat + j * C, 3, C, W);
    D2IP_RET(cwgrad_side(k, N.br[j], x3, gj));
    D2IP_RET(cdgrad(k, N.br[j], gj, gx3, j > 0));
  }
  return D2IP_OK;
}

int refnet_backward(Ctx& k) {
  d2ip_engine& E = k.E;
  RefNet& N = *E.ref;
  const int* ch = N.ch;
  d2ip_act gt = view(E, E.gtail, 0, 1, 1);
  D2IP_RET(cwgrad_side(k, N.tail, N.dec[2].out, gt));
  D2IP_RET(cdgrad(k, N.tail, gt, N.dec[2].gout, 0));
  for (int j = 2; j >= 0; --j) {
    const int l = 2 - j;
    const int w = ch[l + 1] + ch[l];
    D2IP_RET(rblock_bwd(k, N.dec[j]));
    d2ip_act gate = (j == 0) ? view(E, N.xb, 3, ch[3], ch[3]) : N.dec[j - 1].out;
    d2ip_act ggate = (j == 0) ? view(E, N.gxb, 3, ch[3], ch[3]) : N.dec[j - 1].gout;
    D2IP_RET(upsample2x_bwd(view(E, N.gcat[l], l, ch[l + 1], w), ggate, 0, k.B, k.st));
    D2IP_RET(att_bwd(k, N.att[j], view(E, N.s[l], l, ch[l], ch[l]), gate, view(E, N.gcat[l] + ch[l + 1], l, ch[l], w),
                     view(E, N.gs[l], l, ch[l], ch[l]), ggate));
  }
  D2IP_RET(aspp_bwd(k));
  for (int i = 2; i >= 0; --i) {
    D2IP_RET(rblock_bwd(k, N.enc[i]));
    SEP& s = N.se[i];
    D2IP_RET(se_backward(view(E, N.x[i], i, ch[i], ch[i]), view(E, N.gs[i], i, ch[i], ch[i]), k.th() + s.fc1.ow,
                         k.th() + s.fc1.ob, k.th() + s.fc2.ow, k.pbs, s.hid, s.state, s.sbs, k.gr() + s.fc1.ow,
                         k.gr() + s.fc2.ow, view(E, N.gx[i], i, ch[i], ch[i]), 0, E.wg_ws, E.wg_ws_bytes, k.B, k.st));
  }
  d2ip_act gpre = scratch(E, N.ssb[0], 0, ch[0]), gc = scratch(E, N.ssb[1], 0, ch[0]);
  D2IP_RET(norm_act_bwd(view(E, N.gx[0], 0, ch[0], ch[0]), view(E, N.stem_p, 0, ch[0], ch[0]), 2, 0.f, N.stem_xh,
                        N.stem_rs, k.th() + N.stem_n.og, k.pbs, gpre, gc, k.gr() + N.stem_n.og, k.pbs, E.na_ws,
                        E.na_ws_bytes, k.B, k.st));
  d2ip_act z = view(E, const_cast<float*>(E.b.z), 0, 1, 1);
  return cwgrad_side(k, N.stem, z, gc);
}

}  // namespace d2ip
