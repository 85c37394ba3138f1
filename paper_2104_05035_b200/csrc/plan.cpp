// plan.cpp — the per-rank executor of one synchronous hybrid-parallel training
// step of 3D-ResAttNet (§3.1.1, §3.2, §4.3.1).
//
// A plan owns: the network model (net.cpp), the placement of partitions on the
// stages of a pipeline group (genes from GABRA), the workspace layout inside
// the caller-provided device buffer, and the NCCL communicators.  Forward runs
// every micro-batch through the local units in ascending order, receiving a
// partition's input activation from the stage of the previous partition and
// sending its output to the next; backward runs the chain rule in
// reverse with the gradient of each partition input passed to partition i-1;
// the step all-reduces the local partitions' gradients over the stage's
// data-parallel group and applies SGD.
#include "plan.h"

#include <algorithm>

#include <functional>

#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "error.h"
#include "tc_conv.h"
#include "util.cuh"

namespace rn {

static const float BN_EPS = 1e-5f;       // reading X8
static const float BN_MOMENTUM = 0.1f;   // reading X8

size_t Plan::alloc(size_t bytes) {
  size_t off = (ws_bytes + 255) & ~(size_t)255;
  ws_bytes = off + ((bytes + 255) & ~(size_t)255);
  return off;
}

void Plan::make_bn(BNL &b, int gamma_idx, int C, int64_t V) {
  b.gamma_idx = gamma_idx;
  b.C = C;
  b.V = V;
  b.run_off = bn_run_off[gamma_idx];
  b.stat_off.resize(std::max(Mb, slots));
  for (int k = 0; k < std::max(Mb, slots); ++k) b.stat_off[k] = alloc(4 * sizeof(float) * C);
  if (dt == DT_BF16) {  // up to 2 CTAs per SM in the producing conv
    // one [2][C] partial per producing CTA: convolution grids are sized from the
    // device's SM count (<= 2 CTAs per SM), the stem's from up to 4 blocks per SM
    b.fpart = alloc(sizeof(float) * 4 * nsm * 2 * C);
    b.bpart = alloc(sizeof(float) * 2 * nsm * 2 * C);
  }
}

void Plan::make_conv(ConvL &c, int w_idx, int Ci, int Co, int k, int s, int p, Dims in, Dims out) {
  conv_reg.push_back(&c);
  c.w_idx = w_idx;
  c.g.N = mb;
  c.g.Di = in.d; c.g.Hi = in.h; c.g.Wi = in.w; c.g.Ci = Ci;
  c.g.Do = out.d; c.g.Ho = out.h; c.g.Wo = out.w; c.g.Co = Co;
  c.g.k = k; c.g.s = s; c.g.p = p;
  size_t wsf = conv_wgrad_ws_floats(c.g);
  if (dt == DT_BF16) wsf = std::max(wsf, tc_wgrad_ws_floats(c.g));
  if (Ci == 1 && stem_fast_supported(c.g)) wsf = std::max(wsf, stem_wgrad_ws_floats(c.g));
  if (dt == DT_BF16) {
    if (tc_conv_supported(c.g, false)) conv_ws_floats = std::max(conv_ws_floats, tc_conv_ws_floats(c.g, false));
    if (tc_conv_supported(c.g, true)) conv_ws_floats = std::max(conv_ws_floats, tc_conv_ws_floats(c.g, true));
  }
  if (wsf > wgrad_ws_floats) wgrad_ws_floats = wsf;
}

size_t Plan::act_bytes(int C, Dims d) const { return (size_t)mb * d.vol() * C * dt_size(dt); }

std::vector<size_t> Plan::per_mb(size_t bytes) {
  // one buffer per micro-batch, or per delayed-pipeline slot
  const int n = std::max(Mb, slots);
  std::vector<size_t> v(n);
  for (int k = 0; k < n; ++k) v[k] = alloc(bytes);
  return v;
}

void Plan::make_block(BlockL &b, int pidx, int cin, int cout, int stride, Dims in) {
  b.cin = cin;
  b.cout = cout;
  b.in = in;
  b.out = conv_out(in, 3, stride, 1);
  b.proj = (stride != 1 || cin != cout);
  const int64_t V = (int64_t)mb * b.out.vol();
  make_conv(b.c1, pidx + 0, cin, cout, 3, stride, 1, in, b.out);
  make_bn(b.b1, pidx + 1, cout, V);
  make_conv(b.c2, pidx + 3, cout, cout, 3, 1, 1, b.out, b.out);
  make_bn(b.b2, pidx + 4, cout, V);
  if (b.proj) {
    make_conv(b.cp, pidx + 6, cin, cout, 1, stride, 0, in, b.out);
    make_bn(b.bp, pidx + 7, cout, V);
  }
  const size_t ab = act_bytes(cout, b.out);
  b.h1 = per_mb(ab);
  b.a1 = per_mb(ab);
  b.h2 = per_mb(ab);
  if (b.proj) b.hp = per_mb(ab);
  b.out_ = per_mb(ab);
  b.dh2 = alloc(ab);
  b.da1 = alloc(ab);
  b.dh1 = alloc(ab);
  if (b.proj) b.dhp = alloc(ab);
}

int Plan::block_param_count(int cin, int cout, int stride) const {
  return (stride != 1 || cin != cout) ? 9 : 6;
}

// ---------------------------------------------------------------------------
Plan::Plan(const rn_net_desc &nd, const rn_dist_desc &dd, int local_batch, int dtype, cudaStream_t st, bool dl)
    : net(build_net(nd)), stream(st), delayed(dl) {
  dt = dtype == RN_BF16 ? DT_BF16 : DT_F32;
  {
    int dev = 0;
    if (cudaGetDevice(&dev) == cudaSuccess)
      cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    cudaGetLastError();
    nsm = std::max(nsm, 148);  // scratch sized for at least a B200's 148 SMs
  }
  rank = dd.rank;
  world = dd.world;
  S = dd.n_stages;
  Mb = dd.micro_batches;
  b = local_batch;
  if (world < 1 || rank < 0 || rank >= world) throw Error(RN_ERR_ARG, "bad rank/world");
  if (S < 1 || world % S != 0) throw Error(RN_ERR_ARG, "world must be a multiple of n_stages");
  if (Mb < 1 || b < 1 || b % Mb != 0) throw Error(RN_ERR_ARG, "local_batch must be a positive multiple of micro_batches");
  mb = b / Mb;
  if (mb > 64) throw Error(RN_ERR_ARG, "micro-batch larger than 64");
  replicas = world / S;
  stage = rank % S;
  replica = rank / S;
  {
    Schedule sc = make_schedule(net, dd, local_batch, dt);
    genes = sc.genes;
    unit_stage = sc.unit_stage;
    local = sc.local;
  }
  const int nu = (int)net.units.size();
  if (delayed) {
    // reading F1: every rank holds one contiguous stage of the chain, stages in
    // chain order; S slots of saved forward state, one batch per iteration
    if (Mb != 1) throw Error(RN_ERR_ARG, "delayed pipeline: micro_batches must be 1");
    for (int ui = 0; ui + 1 < nu; ++ui)
      if (unit_stage[ui] > unit_stage[ui + 1])
        throw Error(RN_ERR_ARG, "delayed pipeline: genes must be non-decreasing along the chain (contiguous stages)");
    slots = S;
    for (int ui = 0; ui < nu; ++ui)
      if (local[ui]) {
        if (entry_unit < 0) entry_unit = ui;
        exit_unit = ui;
      }
    if (entry_unit < 0) throw Error(RN_ERR_ARG, "delayed pipeline: a stage without units");
  }

  // --- parameters (full model on every rank; only local ranges are used) ---
  const int np = (int)net.params.size();
  bn_run_off.assign(np, 0);
  {
    int64_t c = 0;
    for (int i = 0; i < np; ++i)
      if (net.params[i].kind == P_BN_GAMMA) {
        bn_run_off[i] = c;
        c += net.params[i].numel;
      }
  }
  off_master = alloc(sizeof(float) * net.n_params);
  off_grad = alloc(sizeof(float) * net.n_params);
  off_grad2 = alloc(sizeof(float) * net.n_params);  // the in-flight gradient of ASGD (f4)
  off_run_mean = alloc(sizeof(float) * net.n_bn_channels);
  off_run_var = alloc(sizeof(float) * net.n_bn_channels);
  shadow_f.assign(np, 0);
  shadow_d.assign(np, 0);
  for (int i = 0; i < np; ++i) {
    const ParamTensor &t = net.params[i];
    if (t.kind != P_CONV || !local[t.unit]) continue;
    if (dt == DT_BF16) {
      shadow_f[i] = alloc(2 * t.numel);
      shadow_d[i] = alloc(2 * t.numel);
    }
  }
  if (delayed) {  // the weights each in-flight forward used (Eq. 1: the Jacobian at w^{t-i+1})
    stash_master.resize(slots);
    stash_shadow_d.assign(slots, std::vector<size_t>(np, 0));
    for (int sl = 0; sl < slots; ++sl) {
      stash_master[sl] = alloc(sizeof(float) * net.n_params);
      for (int i = 0; i < np; ++i)
        if (shadow_d[i]) stash_shadow_d[sl][i] = alloc(2 * net.params[i].numel);
    }
  }
  off_loss = alloc(64);
  off_flag = alloc(64);
  max_pack = 0;
  max_sgdrg = 0;
  for (int i = 0; i < np; ++i) {
    if (!local[net.params[i].unit]) continue;
    if (net.params[i].kind == P_CONV) ++max_pack;
    ++max_sgdrg;
  }
  off_pack = alloc(sizeof(ConvPack) * (max_pack + 1));
  off_sgdrg = alloc(2 * sizeof(int64_t) * (max_sgdrg + 1));
  off_x = alloc(sizeof(float) * (size_t)b * net.units[0].in.vol() * slots);  // per slot (delayed pipeline)
  off_y = alloc(sizeof(int32_t) * (size_t)b * slots);
  for (int i = 0; i < 2; ++i)  // staging slots of the pipelined host-input loop: x then y
    off_stage[i] = alloc(sizeof(float) * (size_t)b * net.units[0].in.vol() + 256 + sizeof(int32_t) * (size_t)b);

  // --- units ---
  units.resize(nu);
  for (int ui = 0; ui < nu; ++ui) {
    const Unit &u = net.units[ui];
    UnitL &L = units[ui];
    L.kind = u.kind;
    if (!local[ui]) continue;
    const int p0 = net.unit_param_begin[ui];
    if (u.kind == U_STEM) {
      make_conv(L.stem_conv, p0, 1, u.cout, 3, u.stride, 1, u.in, u.conv);
      make_bn(L.stem_bn, p0 + 1, u.cout, (int64_t)mb * u.conv.vol());
      L.stem_h = per_mb(act_bytes(u.cout, u.conv));
      L.out = per_mb(act_bytes(u.cout, u.out));
      if (u.pool) L.am = per_mb((size_t)mb * u.out.vol() * u.cout);
      if (stem_sparse_bwd(u, L)) {
        L.sws = alloc(sizeof(float) * stem_bwd_sparse_ws_floats());
        L.gws = alloc(sizeof(float) * stem_gram_ws_floats());
        L.gd = per_mb(sizeof(double) * 1024);
        L.gd_fwd.assign(L.gd.size(), 0);
      } else {
        L.tmp0 = alloc(act_bytes(u.cout, u.conv));
        L.tmp1 = alloc(act_bytes(u.cout, u.conv));
      }
    } else if (u.kind == U_BLOCK) {
      make_block(L.blk, p0, u.cin, u.cout, u.stride, u.in);
      L.out = L.blk.out_;
    } else if (u.kind == U_ATT) {
      const int C = u.cout;
      make_block(L.trunk, p0, C, C, 1, u.in);
      const int p1 = p0 + 6;
      make_block(L.mask, p1, C, C, 1, u.mask);
      const int p2 = p1 + 6;
      const int64_t V = (int64_t)mb * u.in.vol();
      make_conv(L.mc1, p2, C, C, 1, 1, 0, u.in, u.in);
      make_bn(L.mbn, p2 + 1, C, V);
      make_conv(L.mc2, p2 + 3, C, C, 1, 1, 0, u.in, u.in);
      L.bias_idx = p2 + 4;
      const size_t ab = act_bytes(C, u.in), am_ = act_bytes(C, u.mask);
      L.u0 = per_mb(am_);
      L.am = per_mb((size_t)mb * u.mask.vol() * C);
      L.up = per_mb(ab);
      L.mh = per_mb(ab);
      L.r = per_mb(ab);
      L.m = per_mb(ab);
      L.out = per_mb(ab);
      L.dT = alloc(ab);
      L.dm = alloc(ab);
      L.dr = alloc(ab);
      L.dmh = alloc(ab);
      L.dup = alloc(ab);
      L.dum = alloc(am_);
      L.du0 = alloc(am_);
      // trilinear tables (reading X11), mask dims -> unit dims
      build_up_tables(L.tab, u.mask, u.in);
    } else {
      L.g = per_mb(sizeof(float) * mb * u.cin);
      L.dz = per_mb(sizeof(float) * mb * 2);
    }
  }
  // gradient-of-output buffers and cut buffers
  for (int ui = 0; ui < nu; ++ui) {
    const Unit &u = net.units[ui];
    UnitL &L = units[ui];
    if (!local[ui]) continue;
    if (u.kind != U_HEAD) L.dout = alloc(act_bytes(u.cout, u.out));
    if (ui > 0 && !local[ui - 1]) {
      // input comes from another stage: receive buffers (saved per micro-batch)
      const Unit &pu = net.units[ui - 1];
      L.recv_in = per_mb(act_bytes(pu.cout, pu.out));
      L.send_dx = alloc(act_bytes(pu.cout, pu.out));
    }
  }
  // scratch
  nblk_max = 4 * nsm;
  off_partial = alloc(sizeof(float) * nblk_max * 2 * 512);
  off_coef = alloc(sizeof(float) * 3 * 512 * 2);
  off_counter = alloc(256);  // last-block tickets of the fused reduce+finalize kernels (zeroed at bind)
  off_zrg = alloc(2 * sizeof(int64_t) * (conv_reg.size() + 2));  // after every make_conv
  off_wgrad_ws = alloc(sizeof(float) * (wgrad_ws_floats ? wgrad_ws_floats : 1));
  off_conv_ws = alloc(sizeof(float) * (conv_ws_floats ? conv_ws_floats : 1));
  off_conv_ws2 = alloc(sizeof(float) * (conv_ws_floats ? conv_ws_floats : 1));
  size_t up_floats = 1;
  for (int ui = 0; ui < (int)net.units.size(); ++ui) {
    const Unit &u = net.units[ui];
    if (u.kind == U_ATT && local[ui])
      up_floats = std::max(up_floats, upsample_bwd_ws_floats(mb, u.mask.d, u.mask.h, u.mask.w, u.cout, u.in.d,
                                                             u.in.h, u.in.w));
  }
  off_up_ws = alloc(sizeof(float) * up_floats);

  // --- communicators ---
  if (world > 1) {
    world_comm = nccl_init(dd.nccl_id, world, rank);
    pipe_comm = nccl_split(world_comm, replica, stage);
    dp_comm = nccl_split(world_comm, stage, replica);
  }
  // all-reduce buckets: runs of consecutive local units, in backward order
  if (replicas > 1) {
    const int64_t target = 2 * 1024 * 1024;  // floats (8 MB) per bucket
    for (int ui = nu - 1; ui >= 0; --ui) {
      if (!local[ui]) continue;
      const int a = net.unit_param_begin[ui], e = net.unit_param_end[ui];
      if (a == e) continue;
      const int64_t b0 = net.params[a].canon_off, e0 = net.params[e - 1].canon_off + net.params[e - 1].numel;
      if (!buckets.empty() && buckets.back().ulo == ui + 1 && buckets.back().b == e0 &&
          buckets.back().e - buckets.back().b < target) {
        buckets.back().ulo = ui;
        buckets.back().b = b0;
      } else {
        buckets.push_back({ui, ui, b0, e0});
      }
    }
  }
}

bool Plan::overlap_ar() const {
  auto it = opts.find("overlap_allreduce");
  return replicas > 1 && !async_ar() && (it == opts.end() || it->second != 0) && stream != nullptr &&
         stream != cudaStreamLegacy && stream != cudaStreamPerThread;
}

bool Plan::async_ar() const {
  auto it = opts.find("async_allreduce");
  return it != opts.end() && it->second != 0 && !delayed;
}

// enqueue bucket bi's all-reduce on the comm stream after everything that writes
// its gradients: the main stream's backward of its units and the weight-gradient
// side stream's work enqueued so far
void Plan::launch_bucket(size_t bi) {
  if (!comm_st) CUDA_CHECK(cudaStreamCreateWithFlags(&comm_st, cudaStreamNonBlocking));
  while (ar_ev.size() < 2 * buckets.size() + 1) {
    cudaEvent_t e;
    CUDA_CHECK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    ar_ev.push_back(e);
  }
  CUDA_CHECK(cudaEventRecord(ar_ev[2 * bi], stream));
  CUDA_CHECK(cudaStreamWaitEvent(comm_st, ar_ev[2 * bi], 0));
  if (side_used) {
    CUDA_CHECK(cudaEventRecord(ar_ev[2 * bi + 1], side));
    CUDA_CHECK(cudaStreamWaitEvent(comm_st, ar_ev[2 * bi + 1], 0));
  }
  const Bucket &bk = buckets[bi];
  nccl_allreduce_sum_f32(dp_comm, (float *)P(off_grad) + bk.b, (size_t)(bk.e - bk.b), comm_st);
}

Plan::~Plan() {
  drop_graphs();
  if (copy_stream) cudaStreamDestroy(copy_stream);
  if (side) cudaStreamDestroy(side);
  if (comm_st) cudaStreamDestroy(comm_st);
  for (auto e : ev_async)
    if (e) cudaEventDestroy(e);
  for (auto e : ar_ev) cudaEventDestroy(e);
  if (ev_fork) cudaEventDestroy(ev_fork);
  if (ev_sgd) cudaEventDestroy(ev_sgd);
  if (ev_join) cudaEventDestroy(ev_join);
  if (ev_gfork) cudaEventDestroy(ev_gfork);
  if (ev_bfork) cudaEventDestroy(ev_bfork);
  if (ev_bjoin) cudaEventDestroy(ev_bjoin);
  if (bstream) cudaStreamDestroy(bstream);
  if (ev_gjoin) cudaEventDestroy(ev_gjoin);
  for (int i = 0; i < 2; ++i) {
    if (ev_copied[i]) cudaEventDestroy(ev_copied[i]);
    if (ev_free[i]) cudaEventDestroy(ev_free[i]);
  }
  if (loss_pinned) cudaFreeHost(loss_pinned);
  for (auto &e : ev_pool) {
    cudaEventDestroy(e.a);
    cudaEventDestroy(e.b);
  }
  for (auto &kv : up_dev) cudaFree(kv);
  nccl_destroy(dp_comm);
  nccl_destroy(pipe_comm);
  nccl_destroy(world_comm);
}

void Plan::build_up_tables(UpTables &tab, Dims in, Dims out) {
  // 1-D linear maps per dim: src = max((o+1/2)*in/out - 1/2, 0), i0 = floor(src),
  // i1 = min(i0+1, in-1), weights (1-lambda, lambda); adjoint as CSR per input index.
  int ins[3] = {in.d, in.h, in.w}, outs[3] = {out.d, out.h, out.w};
  for (int a = 0; a < 3; ++a) {
    const int ni = ins[a], no = outs[a];
    std::vector<int> fidx(2 * no);
    std::vector<float> fw(2 * no);
    std::vector<std::vector<std::pair<int, double>>> adj(ni);
    const double scale = (double)ni / (double)no;
    for (int o = 0; o < no; ++o) {
      double src = ((double)o + 0.5) * scale - 0.5;
      if (src < 0) src = 0;
      int i0 = (int)std::floor(src);
      if (i0 > ni - 1) i0 = ni - 1;
      int i1 = i0 + 1 < ni ? i0 + 1 : ni - 1;
      double lam = src - i0;
      fidx[2 * o] = i0;
      fidx[2 * o + 1] = i1;
      fw[2 * o] = (float)(1.0 - lam);
      fw[2 * o + 1] = (float)lam;
      if (i0 == i1) {
        adj[i0].push_back({o, 1.0});
      } else {
        adj[i0].push_back({o, 1.0 - lam});
        adj[i1].push_back({o, lam});
      }
    }
    std::vector<int> start(ni + 1, 0), bo;
    std::vector<float> bw;
    for (int i = 0; i < ni; ++i) {
      start[i] = (int)bo.size();
      for (auto &pr : adj[i]) {
        bo.push_back(pr.first);
        bw.push_back((float)pr.second);
      }
    }
    start[ni] = (int)bo.size();
    auto up = [&](const void *h, size_t bytes) -> void * {
      void *d = nullptr;
      CUDA_CHECK(cudaMalloc(&d, bytes ? bytes : 4));
      if (bytes) CUDA_CHECK(cudaMemcpy(d, h, bytes, cudaMemcpyHostToDevice));
      up_dev.push_back(d);
      return d;
    };
    tab.fw_idx[a] = (const int *)up(fidx.data(), fidx.size() * 4);
    tab.fw_w[a] = (const float *)up(fw.data(), fw.size() * 4);
    tab.bw_start[a] = (const int *)up(start.data(), start.size() * 4);
    tab.bw_o[a] = (const int *)up(bo.data(), bo.size() * 4);
    tab.bw_w[a] = (const float *)up(bw.data(), bw.size() * 4);
  }
}

// ---------------------------------------------------------------------------
// helpers
// ---------------------------------------------------------------------------
float *Plan::master(int idx) { return (float *)P(off_master) + net.params[idx].canon_off; }
float *Plan::grad(int idx) { return (float *)P(off_grad) + net.params[idx].canon_off; }
const void *Plan::wfwd(int idx) { return dt == DT_F32 ? (const void *)master(idx) : P(shadow_f[idx]); }

static double conv_flops(const ConvGeom &g) { return 2.0 * (double)g.out_vox() * g.Co * g.Ci * g.taps(); }

bool Plan::timing() const {
  auto it = opts.find("time_kernels");
  return it != opts.end() && it->second != 0;
}

// elementwise / HBM-bound launches timed live (option time_kernels): event pair
// around each launch on the plan stream, tagged with its family and its
// algorithmic bytes (every tensor element read + written once)
const char *const kEltFamilies[] = {"bn_apply", "bn_bwd_apply", "bn_partials", "stem_pool_fwd", "stem_pool_bwd",
                                    "maxpool_fwd", "maxpool_bwd", "upsample_fwd", "upsample_bwd", "att_fwd",
                                    "att_bwd", "head", "sgd", nullptr};
enum { F_BN_APPLY = 0, F_BN_BWD_APPLY, F_BN_PARTIALS, F_STEM_POOL_FWD, F_STEM_POOL_BWD, F_MAXPOOL_FWD,
       F_MAXPOOL_BWD, F_UP_FWD, F_UP_BWD, F_ATT_FWD, F_ATT_BWD, F_HEAD, F_SGD };

struct EltTimer {
  Plan *p;
  size_t i = 0;
  int fam;
  bool on;
  EltTimer(Plan *pl, int f, double bytes) : p(pl), fam(f), on(pl->timing()) {
    if (on) i = p->tk_begin(3, bytes);
  }
  ~EltTimer() {
    if (on) {
      p->ev_pool[i].kind = fam;
      cudaEventRecord(p->ev_pool[i].b, p->stream);
    }
  }
};

size_t Plan::tk_begin(int cls, double flops) {
  if (ev_used == ev_pool.size()) {
    EvPair e;
    CUDA_CHECK(cudaEventCreate(&e.a));
    CUDA_CHECK(cudaEventCreate(&e.b));
    ev_pool.push_back(e);
  }
  EvPair &e = ev_pool[ev_used];
  e.flops = flops;
  e.cls = cls;
  e.kind = -1;
  CUDA_CHECK(cudaEventRecord(e.a, stream));
  return ev_used++;
}

void Plan::tk_end(size_t i, int kind) {
  ev_pool[i].kind = kind;
  CUDA_CHECK(cudaEventRecord(ev_pool[i].b, stream));
}

bool Plan::use_halo() const {
  auto it = opts.find("halo_conv");
  return it == opts.end() || it->second != 0;
}

bool Plan::recompute_mask() const {
  auto it = opts.find("recompute_mask");
  return it == opts.end() || it->second != 0;
}

bool Plan::use_pair() const {
  auto it = opts.find("pair_conv");
  return it == opts.end() || it->second != 0;
}
// run f on the branch stream (forked from the plan stream now; own split-K workspace);
// ev_bjoin is recorded at its end — the caller makes the plan stream wait on it
void Plan::on_branch(const std::function<void()> &f) {
  if (!bstream) {
    CUDA_CHECK(cudaStreamCreateWithFlags(&bstream, cudaStreamNonBlocking));
    CUDA_CHECK(cudaEventCreateWithFlags(&ev_bfork, cudaEventDisableTiming));
    CUDA_CHECK(cudaEventCreateWithFlags(&ev_bjoin, cudaEventDisableTiming));
  }
  CUDA_CHECK(cudaEventRecord(ev_bfork, stream));
  CUDA_CHECK(cudaStreamWaitEvent(bstream, ev_bfork, 0));
  std::swap(stream, bstream);
  std::swap(off_conv_ws, off_conv_ws2);
  try {
    f();
  } catch (...) {
    std::swap(stream, bstream);
    std::swap(off_conv_ws, off_conv_ws2);
    throw;
  }
  CUDA_CHECK(cudaEventRecord(ev_bjoin, stream));
  std::swap(stream, bstream);
  std::swap(off_conv_ws, off_conv_ws2);
}

// attention mask branch concurrent with the trunk (option att_branch, default on; eager
// per-kernel timing and the default / legacy stream run it in order)
bool Plan::att_branch_on() const {
  auto it = opts.find("att_branch");
  static const bool env_off = getenv("RN_ATT_BRANCH") && atoi(getenv("RN_ATT_BRANCH")) == 0;  // A/B
  const bool on = (it == opts.end() || it->second != 0) && !env_off;
  // the fp32 / unfused BN paths share reduction scratch (off_partial, counter) across units
  return on && dt == DT_BF16 && fused_stats() && !timing() && stream != nullptr && stream != cudaStreamLegacy && stream != cudaStreamPerThread;
}

// the streaming warp-tensor-core kernel for the 64 -> 64 1x1x1 convs (option c1x1, default on)
bool Plan::use_c1x1() const {
  auto it = opts.find("c1x1");
  return it == opts.end() || it->second != 0;
}

bool Plan::use_tc(const ConvGeom &g, bool dgrad) const {
  if (dt != DT_BF16) return false;
  auto it = opts.find("tc_conv");
  if (it != opts.end() && it->second == 0) return false;
  return tc_conv_supported(g, dgrad);
}

// fused BN statistics in the conv epilogues (bf16 tensor-core path; option
// "fused_stats" = 0 restores the separate reduction kernels)
bool Plan::fused_stats() const {
  auto it = opts.find("fused_stats");
  return dt == DT_BF16 && (it == opts.end() || it->second != 0);
}

void Plan::conv_fwd(const ConvL &c, const void *x, void *y, const float *bias, BNL *stats) {
  const bool t = timing();
  size_t e = t ? tk_begin(0, conv_flops(c.g)) : 0;
  EpiStats es;
  const bool want = stats && fused_stats();
  if (want) {
    es.part = (float *)P(stats->fpart);
    es.mode = 1;
  }
  int parts = 0, kind = K_SIMT;
  if (use_tc(c.g, false) && use_c1x1() && conv1x1_supported(c.g) && ((kind = K_TC) != 0))
    parts = conv1x1(c.g, (const bf16 *)x, (const bf16 *)P(shadow_f[c.w_idx]), bias, (bf16 *)y, stream,
                    want ? &es : nullptr);
  else if (use_tc(c.g, false) && use_pair() && pair_conv_supported(c.g, false) && ((kind = K_PAIR) != 0))
    parts = conv_pair(c.g, false, (const bf16 *)x, (const bf16 *)P(shadow_f[c.w_idx]), bias, (bf16 *)y, false,
                      nullptr, nullptr, stream, want ? &es : nullptr);
  else if (use_tc(c.g, false) && use_halo() && halo_conv_supported(c.g, false) && ((kind = K_HALO) != 0))
    parts = conv_halo(c.g, false, (const bf16 *)x, (const bf16 *)P(shadow_f[c.w_idx]), bias, (bf16 *)y, false,
                      nullptr, nullptr, stream, want ? &es : nullptr);
  else if (use_tc(c.g, false) && ((kind = K_TC) != 0))
    parts = conv_fprop_tc(c.g, (const bf16 *)x, (const bf16 *)P(shadow_f[c.w_idx]), bias, (bf16 *)y,
                          (float *)P(off_conv_ws), conv_ws_floats, stream, want ? &es : nullptr);
  else
    conv_fprop_simt(dt, c.g, x, wfwd(c.w_idx), bias, y, stream);
  if (stats) stats->fP = parts;
  if (t) tk_end(e, kind);
}
void Plan::conv_bwd_data(const ConvL &c, const void *dy, void *dx, bool accumulate, const void *res,
                         const void *res_mask, const StatsTarget &stats) {
  const bool t = timing();
  size_t e = t ? tk_begin(1, conv_flops(c.g)) : 0;
  EpiStats es;
  const bool want = stats.bn && fused_stats();
  if (want) {
    es.part = (float *)P(stats.bn->bpart);
    es.mode = stats.mscale && recompute_mask() ? 3 : 2;
    es.mask = (const bf16 *)stats.mask;
    es.h = (const bf16 *)stats.h;
    es.mean = stats.mean;
    es.mscale = stats.mscale;
    es.mshift = stats.mshift;
  }
  int parts = 0, kind = K_SIMT;
  // the CTA-pair dgrad's epilogue is the kernel's bottleneck: its backward BN sums
  // cost more fused (~14 us per stage-1 launch) than the standalone partials pass
  // (~8 us), so by default they are left to bn_backward (option pair_bwd_stats)
  auto itp = opts.find("pair_bwd_stats");
  const bool pair_stats = itp != opts.end() && itp->second != 0;
  if (use_tc(c.g, true) && use_c1x1() && conv1x1_supported(c.g) && !accumulate && !res &&
      ((kind = K_TC) != 0))
    parts = conv1x1(c.g, (const bf16 *)dy, (const bf16 *)P(shadow_d[c.w_idx]), nullptr, (bf16 *)dx, stream,
                    want ? &es : nullptr);
  else if (use_tc(c.g, true) && use_pair() && pair_conv_supported(c.g, true) && ((kind = K_PAIR) != 0))
    parts = conv_pair(c.g, true, (const bf16 *)dy, (const bf16 *)P(shadow_d[c.w_idx]), nullptr, (bf16 *)dx,
                      accumulate, (const bf16 *)res, (const bf16 *)res_mask, stream,
                      want && pair_stats ? &es : nullptr);
  else if (use_tc(c.g, true) && use_halo() && halo_conv_supported(c.g, true) && ((kind = K_HALO) != 0))
    parts = conv_halo(c.g, true, (const bf16 *)dy, (const bf16 *)P(shadow_d[c.w_idx]), nullptr, (bf16 *)dx,
                      accumulate, (const bf16 *)res, (const bf16 *)res_mask, stream, want ? &es : nullptr);
  else if (use_tc(c.g, true) && ((kind = K_TC) != 0))
    parts = conv_dgrad_tc(c.g, (const bf16 *)dy, (const bf16 *)P(shadow_d[c.w_idx]), (bf16 *)dx, accumulate,
                          (const bf16 *)res, (const bf16 *)res_mask, (float *)P(off_conv_ws), conv_ws_floats, stream,
                          want ? &es : nullptr);
  else
    conv_dgrad_simt(dt, c.g, dy, wfwd(c.w_idx), dx, accumulate, res, res_mask, stream);
  if (stats.bn) stats.bn->bP = parts;
  if (t) tk_end(e, kind);
}
void Plan::conv_bwd_data_proj(const ConvL &c1, const void *dy1, const ConvL &cp, const void *dyp, void *dx,
                              bool accumulate, const StatsTarget &stats) {
  auto it = opts.find("merge_proj");
  const bool merge = (it == opts.end() || it->second != 0) && use_tc(c1.g, true) && use_tc(cp.g, true) &&
                     c1.g.k == 3 && c1.g.s == 2 && cp.g.k == 1 && cp.g.s == 2 && cp.g.Ci == c1.g.Ci &&
                     cp.g.Co == c1.g.Co;
  if (!merge) {
    conv_bwd_data(c1, dy1, dx, accumulate, nullptr, nullptr);
    conv_bwd_data(cp, dyp, dx, true, nullptr, nullptr, stats);
    return;
  }
  const bool t = timing();
  size_t e = t ? tk_begin(1, conv_flops(c1.g) + conv_flops(cp.g)) : 0;
  EpiStats es;
  const bool want = stats.bn && fused_stats();
  if (want) {
    es.part = (float *)P(stats.bn->bpart);
    es.mode = stats.mscale && recompute_mask() ? 3 : 2;
    es.mask = (const bf16 *)stats.mask;
    es.h = (const bf16 *)stats.h;
    es.mean = stats.mean;
    es.mscale = stats.mscale;
    es.mshift = stats.mshift;
  }
  const int parts = conv_dgrad_tc(c1.g, (const bf16 *)dy1, (const bf16 *)P(shadow_d[c1.w_idx]), (bf16 *)dx,
                                  accumulate, nullptr, nullptr, (float *)P(off_conv_ws), conv_ws_floats, stream,
                                  want ? &es : nullptr, (const bf16 *)dyp, (const bf16 *)P(shadow_d[cp.w_idx]));
  if (stats.bn) stats.bn->bP = parts;
  if (t) tk_end(e, K_TC);
}
void Plan::gradcam(int cls, float *map_dev) {
  const int hi = (int)net.units.size() - 1;
  const Unit &hu = net.units[hi];
  if (hu.kind != U_HEAD || hi < 1 || !local[hi] || !local[hi - 1])
    throw Error(RN_ERR_ARG, "rn_gradcam: the head and the last conv unit must be on this rank");
  if (cls < 0 || cls > 1) throw Error(RN_ERR_ARG, "rn_gradcam: class must be 0 or 1");
  const Unit &lu = net.units[hi - 1];
  const Dims in = net.units[0].in;
  if (!cam_tab_built) {
    build_up_tables(cam_tab, lu.out, in);
    cam_tab_built = true;
  }
  const int64_t coarse_n = (int64_t)mb * lu.out.vol();
  if (coarse_n > (int64_t)nblk_max * 2 * 512) throw Error(RN_ERR_SIZE, "rn_gradcam: scratch too small");
  const float *wrow = master(net.unit_param_begin[hi]) + (int64_t)cls * hu.cin;
  for (int k = 0; k < Mb; ++k)
    gradcam_last(dt, P(units[hi - 1].out[k]), wrow, mb, lu.out.d, lu.out.h, lu.out.w, lu.cout,
                 (float *)P(off_partial), map_dev + (int64_t)k * mb * in.vol(), in.d, in.h, in.w, cam_tab, stream);
}

bool Plan::side_on() const {
  auto it = opts.find("wgrad_stream");
  const bool on = it == opts.end() || it->second != 0;
  return on && !timing() && stream != nullptr && stream != cudaStreamLegacy && stream != cudaStreamPerThread;
}

// the bf16 pooled stem runs its backward at the pooled resolution (k_stem_bwd.cu)
bool Plan::stem_sparse_bwd(const Unit &u, const UnitL &L) const {
  return dt == DT_BF16 && u.pool && stem_bwd_sparse_supported(L.stem_conv.g);
}

void Plan::conv_bwd_weight(const ConvL &c, const void *x, const void *dy, bool x_f32) {
  const bool t = timing();
  size_t e = t ? tk_begin(2, conv_flops(c.g)) : 0;
  cudaStream_t ws = stream;
  if (side_on()) {
    if (!side) {
      CUDA_CHECK(cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking));
      CUDA_CHECK(cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming));
      CUDA_CHECK(cudaEventCreateWithFlags(&ev_join, cudaEventDisableTiming));
    }
    CUDA_CHECK(cudaEventRecord(ev_fork, stream));  // dy (and x) ready
    CUDA_CHECK(cudaStreamWaitEvent(side, ev_fork, 0));
    ws = side;
    side_used = true;
  }
  int kind = K_SIMT;
  if (x_f32 && stem_fast_supported(c.g)) {
    kind = K_STEM;
    stem_wgrad_fast(dt, c.g, (const float *)x, dy, grad(c.w_idx), (float *)P(off_wgrad_ws), ws);
  } else if (!x_f32 && use_tc(c.g, false) && tc_wgrad_supported(c.g)) {
    kind = K_WGRAD;
    conv_wgrad_tc(c.g, (const bf16 *)x, (const bf16 *)dy, grad(c.w_idx), (float *)P(off_wgrad_ws), ws,
                  wg_overwrite && wg_first);
  } else {
    conv_wgrad_simt(dt, x_f32, c.g, x, dy, grad(c.w_idx), (float *)P(off_wgrad_ws), ws);
  }
  if (t) tk_end(e, kind);
}

float *Plan::bn_stat(const BNL &b, int k, int which) { return (float *)P(b.stat_off[k]) + which * b.C; }

void Plan::bn_forward_stats(const BNL &b, int k, const void *h) { bn_fwd(b, k, h, nullptr, nullptr, nullptr, false, nullptr); }

BnFinal Plan::bn_final(const BNL &b, int k) {
  BnFinal f;
  f.part = (const float *)P(b.fpart);
  f.P = b.fP;
  f.gamma = master(b.gamma_idx);
  f.beta = master(b.gamma_idx + 1);
  f.mean = bn_stat(b, k, 0);
  f.invstd = bn_stat(b, k, 1);
  f.scale = bn_stat(b, k, 2);
  f.shift = bn_stat(b, k, 3);
  f.run_mean = (float *)P(off_run_mean) + b.run_off;
  f.run_var = (float *)P(off_run_var) + b.run_off;
  f.momentum = BN_MOMENTUM;
  f.eps = BN_EPS;
  return f;
}

// Train-mode BN (reading X8): statistics of h, then (if y) y = act(BN(h) + R) where
// R = res (identity skip) or res*rscale + rshift (the projection's BN).  When
// the producing conv fused the statistics (b.fP > 0) one kernel finalizes and
// applies them.
void Plan::bn_fwd(const BNL &b, int k, const void *h, const void *res, const float *rscale, const float *rshift,
                  bool relu, void *y) {
  if (fused_stats() && y && !rscale) {
    BNL &m = const_cast<BNL &>(b);
    const double vc = (double)b.V * b.C * dt_size(dt);
    if (m.fP <= 0) {
      EltTimer tm(this, F_BN_PARTIALS, vc);
      m.fP = bn_stats_partials(dt, h, b.V, b.C, (float *)P(b.fpart), stream);
    }
    EltTimer tm(this, F_BN_APPLY, vc * (res ? 3 : 2));
    bn_apply_fused(dt, h, b.V, b.C, bn_final(b, k), nullptr, res, relu, y, stream);
    m.fP = 0;  // consumed: the next producer decides again (never reuse stale partials)
    return;
  }
  float *part = (float *)P(off_partial);
  const double vc = (double)b.V * b.C * dt_size(dt);
  EltTimer tm(this, F_BN_APPLY, vc * (y ? (res ? 4 : 3) : 1));
  bn_stats_finalize(dt, h, b.V, b.C, part, counter(), master(b.gamma_idx), master(b.gamma_idx + 1),
                    bn_stat(b, k, 0), bn_stat(b, k, 1), bn_stat(b, k, 2), bn_stat(b, k, 3),
                    (float *)P(off_run_mean) + b.run_off, (float *)P(off_run_var) + b.run_off, BN_MOMENTUM, BN_EPS,
                    stream);
  if (y) bn_apply(dt, h, b.V, b.C, bn_stat(b, k, 2), bn_stat(b, k, 3), res, rscale, rshift, relu, y, stream);
}

// dx = BN-backward of dy' = dy * mask ; coef scratch slot `slot`.  bf16 path:
// the sums come from the producer of dy (b.bP > 0) or one standalone pass,
// and the apply kernel finalizes them.
bool Plan::bn_backward(const BNL &b, int k, const void *dy, const void *h, int mask_mode, const void *mask_t,
                       void *dx, int slot, void *dprime) {
  if (fused_stats() && mask_mode == MASK_TENSOR) {
    BNL &m = const_cast<BNL &>(b);
    const double vc = (double)b.V * b.C * dt_size(dt);
    if (m.bP <= 0) {
      EltTimer tm(this, F_BN_PARTIALS, vc * 3);
      m.bP = bn_bwd_partials(dt, dy, h, mask_t, bn_stat(b, k, 0), b.V, b.C, (float *)P(b.bpart), stream);
    }
    EltTimer tm(this, F_BN_BWD_APPLY, vc * 4);
    bn_bwd_apply_fused(dt, dy, h, mask_t, b.V, b.C, (const float *)P(b.bpart), b.bP, master(b.gamma_idx),
                       bn_stat(b, k, 0), bn_stat(b, k, 1), grad(b.gamma_idx), grad(b.gamma_idx + 1), dx, stream,
                       (float *)P(off_coef) + slot * 3 * 512, dprime);
    m.bP = 0;  // consumed: the next producer decides again
    return true;
  }
  float *part = (float *)P(off_partial);
  float *coef = (float *)P(off_coef) + slot * 3 * 512;
  EltTimer tm(this, F_BN_BWD_APPLY, (double)b.V * b.C * dt_size(dt) * (mask_mode == MASK_TENSOR ? 7 : 5));
  bn_bwd_reduce_finalize(dt, dy, h, b.V, b.C, mask_mode, mask_t, bn_stat(b, k, 2), bn_stat(b, k, 3),
                         bn_stat(b, k, 0), bn_stat(b, k, 1), master(b.gamma_idx), part, counter(),
                         grad(b.gamma_idx), grad(b.gamma_idx + 1), coef, stream);
  bn_bwd_apply(dt, dy, h, b.V, b.C, mask_mode, mask_t, bn_stat(b, k, 2), bn_stat(b, k, 3), coef, dx, stream);
  return dprime == nullptr;  // this path does not produce dy'
}

// ---------------------------------------------------------------------------
// residual network layer (two Conv blocks + skip)
// ---------------------------------------------------------------------------
void Plan::block_fwd(BlockL &B, int k, const void *x) {
  conv_fwd(B.c1, x, P(B.h1[k]), nullptr, &B.b1);
  bn_fwd(B.b1, k, P(B.h1[k]), nullptr, nullptr, nullptr, true, P(B.a1[k]));
  conv_fwd(B.c2, P(B.a1[k]), P(B.h2[k]), nullptr, &B.b2);
  if (B.proj) {
    // (on the branch stream, concurrent with conv1 -> BN1 -> conv2, this measured
    // slower: 3.169 vs 3.123 ms — it competes with conv1 for every SM)
    conv_fwd(B.cp, x, P(B.hp[k]), nullptr, &B.bp);
    if (fused_stats()) {
      // out = ReLU(BN2(h2) + BNp(hp)): both statistics finalized in the apply kernel
      const double vc = (double)B.b2.V * B.b2.C * dt_size(dt);
      if (B.b2.fP <= 0) {
        EltTimer tm(this, F_BN_PARTIALS, vc);
        B.b2.fP = bn_stats_partials(dt, P(B.h2[k]), B.b2.V, B.b2.C, (float *)P(B.b2.fpart), stream);
      }
      if (B.bp.fP <= 0) {
        EltTimer tm(this, F_BN_PARTIALS, vc);
        B.bp.fP = bn_stats_partials(dt, P(B.hp[k]), B.bp.V, B.bp.C, (float *)P(B.bp.fpart), stream);
      }
      const BnFinal fp = bn_final(B.bp, k);
      EltTimer tm(this, F_BN_APPLY, vc * 3);
      bn_apply_fused(dt, P(B.h2[k]), B.b2.V, B.b2.C, bn_final(B.b2, k), &fp, P(B.hp[k]), true, P(B.out_[k]), stream);
      B.b2.fP = B.bp.fP = 0;
    } else {
      bn_forward_stats(B.bp, k, P(B.hp[k]));
      bn_fwd(B.b2, k, P(B.h2[k]), P(B.hp[k]), bn_stat(B.bp, k, 2), bn_stat(B.bp, k, 3), true, P(B.out_[k]));
    }
  } else {
    bn_fwd(B.b2, k, P(B.h2[k]), x, nullptr, nullptr, true, P(B.out_[k]));
  }
}

// dx_stats: the BN that consumes dx (the previous unit's last BN), whose backward
// sums the final writer of dx computes in its epilogue
void Plan::block_bwd(BlockL &B, int k, const void *x, const void *dout, void *dx, bool accumulate,
                     const StatsTarget &dx_stats) {
  const void *out = P(B.out_[k]);
  // identity skip, dx written (not accumulated): b2's backward apply, which forms
  // dy' = dout * (out > 0) anyway, stores it into dx, and conv1's dgrad accumulates
  // onto it — its epilogue prefetches one operand (dx) instead of two (dout, out)
  auto itr = opts.find("res_prestore");
  const bool pre = !B.proj && dx && !accumulate && (itr == opts.end() || itr->second != 0) &&
                   !(getenv("RN_RES_PRESTORE") && atoi(getenv("RN_RES_PRESTORE")) == 0);
  const bool pre_ok = bn_backward(B.b2, k, dout, P(B.h2[k]), MASK_TENSOR, out, P(B.dh2), 0, pre ? dx : nullptr) && pre;
  if (B.proj) bn_backward(B.bp, k, dout, P(B.hp[k]), MASK_TENSOR, out, P(B.dhp), 1);
  conv_bwd_weight(B.c2, P(B.a1[k]), P(B.dh2), false);
  StatsTarget t1;
  t1.bn = &B.b1;
  t1.mode = 2;
  t1.mask = P(B.a1[k]);
  t1.h = P(B.h1[k]);
  t1.mean = bn_stat(B.b1, k, 0);
  t1.mscale = bn_stat(B.b1, k, 2);
  t1.mshift = bn_stat(B.b1, k, 3);
  conv_bwd_data(B.c2, P(B.dh2), P(B.da1), false, nullptr, nullptr, t1);
  bn_backward(B.b1, k, P(B.da1), P(B.h1[k]), MASK_TENSOR, P(B.a1[k]), P(B.dh1), 0);
  conv_bwd_weight(B.c1, x, P(B.dh1), false);
  if (dx) {
    if (B.proj) {
      conv_bwd_data_proj(B.c1, P(B.dh1), B.cp, P(B.dhp), dx, accumulate, dx_stats);
    } else {
      // identity skip: dx (+)= dgrad(dh1) + dout * (out > 0)
      if (pre_ok) conv_bwd_data(B.c1, P(B.dh1), dx, true, nullptr, nullptr, dx_stats);
      else conv_bwd_data(B.c1, P(B.dh1), dx, accumulate, dout, out, dx_stats);
    }
  }
  if (B.proj) conv_bwd_weight(B.cp, x, P(B.dhp), false);
}

// ---------------------------------------------------------------------------
// units
// ---------------------------------------------------------------------------
const void *Plan::unit_input(int ui, int k, const float *x_in) {
  if (ui == 0) return x_in + (int64_t)k * mb * net.units[0].in.vol();
  if (!local[ui - 1]) return P(units[ui].recv_in[k]);
  return P(units[ui - 1].out[k]);
}

void Plan::unit_fwd(int ui, int k, const float *x_in, const int32_t *y) {
  const Unit &u = net.units[ui];
  UnitL &L = units[ui];
  const void *x = unit_input(ui, k, x_in);
  if (u.kind == U_STEM) {
    if (stem_sparse_bwd(u, L)) {
      // the input Gram matrix of the pooled stem backward depends only on x: on the
      // weight-gradient stream (idle in the forward), joined at the end of the forward
      L.gd_fwd[k] = side_on();
      if (L.gd_fwd[k]) {
        if (!side) {
          CUDA_CHECK(cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking));
          CUDA_CHECK(cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming));
          CUDA_CHECK(cudaEventCreateWithFlags(&ev_join, cudaEventDisableTiming));
        }
        if (!ev_gfork) {
          CUDA_CHECK(cudaEventCreateWithFlags(&ev_gfork, cudaEventDisableTiming));
          CUDA_CHECK(cudaEventCreateWithFlags(&ev_gjoin, cudaEventDisableTiming));
        }
        CUDA_CHECK(cudaEventRecord(ev_gfork, stream));
        CUDA_CHECK(cudaStreamWaitEvent(side, ev_gfork, 0));
        stem_gram(L.stem_conv.g, (const float *)x, (float *)P(L.gws), (double *)P(L.gd[k]), side);
        gram_pending = true;
      }
    }
    {
      const bool t = timing();
      size_t e = t ? tk_begin(0, conv_flops(L.stem_conv.g)) : 0;
      const bool fuse = fused_stats() && u.pool && u.cout % 8 == 0;
      if (stem_fast_supported(L.stem_conv.g))
        L.stem_bn.fP = stem_fprop_fast(dt, L.stem_conv.g, (const float *)x, master(L.stem_conv.w_idx),
                                       P(L.stem_h[k]), stream, fuse ? (float *)P(L.stem_bn.fpart) : nullptr);
      else {
        stem_conv_fprop(dt, L.stem_conv.g, (const float *)x, master(L.stem_conv.w_idx), P(L.stem_h[k]), stream);
        L.stem_bn.fP = 0;  // no fused statistics: the BN below reduces h itself
      }
      if (t) tk_end(e, K_STEM);
    }
    if (u.pool && L.stem_bn.fP > 0) {
      // BN statistics fused into the stem conv; finalize + BN + ReLU + pool in one kernel
      EltTimer tm(this, F_STEM_POOL_FWD,
                  (double)mb * u.cout * (2.0 * u.conv.vol() + 3.0 * u.out.vol()));
      stem_pool_fwd(P(L.stem_h[k]), mb, u.conv.d, u.conv.h, u.conv.w, u.cout, bn_final(L.stem_bn, k), L.stem_bn.V,
                    P(L.out[k]), (uint8_t *)P(L.am[k]), u.out.d, u.out.h, u.out.w, stream);
    } else if (u.pool) {
      bn_forward_stats(L.stem_bn, k, P(L.stem_h[k]));
      maxpool_fwd(dt, P(L.stem_h[k]), mb, u.conv.d, u.conv.h, u.conv.w, u.cout, bn_stat(L.stem_bn, k, 2),
                  bn_stat(L.stem_bn, k, 3), true, P(L.out[k]), (uint8_t *)P(L.am[k]), u.out.d, u.out.h, u.out.w,
                  stream);
    } else {
      bn_fwd(L.stem_bn, k, P(L.stem_h[k]), nullptr, nullptr, nullptr, true, P(L.out[k]));
    }
  } else if (u.kind == U_BLOCK) {
    block_fwd(L.blk, k, x);
  } else if (u.kind == U_ATT) {
    const int C = u.cout;
    const int64_t V = (int64_t)mb * u.in.vol();
    // the soft-mask branch depends only on x: on its own stream, concurrent with the
    // trunk (P:364 out = (1 + sigmoid(mask)) * trunk; the branches meet in att_fwd)
    const bool br = att_branch_on();
    auto mask_branch = [&]() {
      {
      EltTimer tm(this, F_MAXPOOL_FWD, (double)mb * C * (u.in.vol() * dt_size(dt) + u.mask.vol() * (dt_size(dt) + 1.0)));
      maxpool_fwd(dt, x, mb, u.in.d, u.in.h, u.in.w, C, nullptr, nullptr, false, P(L.u0[k]), (uint8_t *)P(L.am[k]),
                  u.mask.d, u.mask.h, u.mask.w, stream);
      }
      block_fwd(L.mask, k, P(L.u0[k]));
      {
      EltTimer tm(this, F_UP_FWD, (double)mb * C * (u.in.vol() + u.mask.vol()) * dt_size(dt));
      upsample_fwd(dt, P(L.mask.out_[k]), mb, u.mask.d, u.mask.h, u.mask.w, C, P(L.up[k]), u.in.d, u.in.h, u.in.w,
                   L.tab, stream);
      }
      conv_fwd(L.mc1, P(L.up[k]), P(L.mh[k]), nullptr, &L.mbn);
      bn_fwd(L.mbn, k, P(L.mh[k]), nullptr, nullptr, nullptr, true, P(L.r[k]));
      conv_fwd(L.mc2, P(L.r[k]), P(L.m[k]), master(L.bias_idx));
    };
    if (br) on_branch(mask_branch);
    else mask_branch();
    block_fwd(L.trunk, k, x);
    if (br) CUDA_CHECK(cudaStreamWaitEvent(stream, ev_bjoin, 0));
    EltTimer tm(this, F_ATT_FWD, 3.0 * V * C * dt_size(dt));
    att_fwd(dt, P(L.m[k]), P(L.trunk.out_[k]), V, C, P(L.out[k]), stream);
  } else {
    const float dz_scale = 1.0f / (float)(mb * Mb * replicas);
    head_fwd(dt, x, mb, (int)u.in.vol(), u.cin, master(net.unit_param_begin[ui]),
             master(net.unit_param_begin[ui] + 1), y + (int64_t)k * mb, dz_scale, 1.0f / (float)Mb,
             (float *)P(L.g[k]), (float *)P(L.dz[k]), (float *)P(off_loss), stream);
  }
}

// the BN that consumes unit ui's input gradient (the previous unit's dout): the
// last BN of a local residual block; its backward sums are fused into the conv
// that writes dout last
StatsTarget Plan::dout_consumer(int ui, int k) {
  StatsTarget t;
  if (ui == 0 || !local[ui - 1] || net.units[ui - 1].kind != U_BLOCK) return t;
  BlockL &B = units[ui - 1].blk;
  t.bn = &B.b2;
  t.mode = 2;
  t.mask = P(B.out_[k]);
  t.h = P(B.h2[k]);
  t.mean = bn_stat(B.b2, k, 0);
  return t;
}

// dx target for unit ui's backward: previous unit's dout (local) or the send buffer
void *Plan::unit_dx_target(int ui) {
  if (ui == 0) return nullptr;
  if (!local[ui - 1]) return P(units[ui].send_dx);
  return P(units[ui - 1].dout);
}

void Plan::unit_bwd(int ui, int k, const float *x_in) {
  const Unit &u = net.units[ui];
  UnitL &L = units[ui];
  const void *x = unit_input(ui, k, x_in);
  void *dx = unit_dx_target(ui);
  if (u.kind == U_STEM) {
    const void *dy;
    int mode;
    const void *mt = nullptr;
    if (stem_sparse_bwd(u, L)) {
      // pooled-resolution backward (reading X23c): sparse over the argmax voxels,
      // dW through the input Gram matrix; no conv-resolution tensor is read or formed
      const BNL &b = L.stem_bn;
      EltTimer tm(this, F_STEM_POOL_BWD,
                  (double)mb * (u.cout * u.out.vol() * (2.0 * dt_size(dt) + 1.0) + 4.0 * u.in.vol()));
      if (!L.gd_fwd[k])  // the forward did not compute the input Gram matrix on the side stream
        stem_gram(L.stem_conv.g, (const float *)x, (float *)P(L.gws), (double *)P(L.gd[k]), stream);
      stem_bwd_sparse(L.stem_conv.g, u.out.d, u.out.h, u.out.w, (const float *)x, master(L.stem_conv.w_idx),
                      P(L.out[k]), P(L.dout), (const uint8_t *)P(L.am[k]), master(b.gamma_idx), bn_stat(b, k, 0),
                      bn_stat(b, k, 1), (const double *)P(L.gd[k]), grad(b.gamma_idx), grad(b.gamma_idx + 1),
                      grad(L.stem_conv.w_idx), (float *)P(L.sws), stream);
      return;
    }
    if (u.pool) {
      maxpool_bwd(dt, P(L.dout), (const uint8_t *)P(L.am[k]), mb, u.conv.d, u.conv.h, u.conv.w, u.cout, u.out.d,
                  u.out.h, u.out.w, P(L.tmp0), false, stream);
      dy = P(L.tmp0);
      mode = MASK_RECOMPUTE;
    } else {
      dy = P(L.dout);
      mode = MASK_TENSOR;
      mt = P(L.out[k]);
    }
    bn_backward(L.stem_bn, k, dy, P(L.stem_h[k]), mode, mt, P(L.tmp1), 0);
    conv_bwd_weight(L.stem_conv, x, P(L.tmp1), true);
  } else if (u.kind == U_BLOCK) {
    block_bwd(L.blk, k, x, P(L.dout), dx, false, dout_consumer(ui, k));
  } else if (u.kind == U_ATT) {
    const int C = u.cout;
    const int64_t V = (int64_t)mb * u.in.vol();
    {
    EltTimer tm(this, F_ATT_BWD, 5.0 * V * C * dt_size(dt));
    att_bwd_finalize(dt, P(L.dout), P(L.m[k]), P(L.trunk.out_[k]), V, C, P(L.dT), P(L.dm), (float *)P(off_partial),
                     counter(), grad(L.bias_idx), stream);
    }
    conv_bwd_weight(L.mc2, P(L.r[k]), P(L.dm), false);
    StatsTarget tm;
    tm.bn = &L.mbn;
    tm.mode = 2;
    tm.mask = P(L.r[k]);
    tm.h = P(L.mh[k]);
    tm.mean = bn_stat(L.mbn, k, 0);
    tm.mscale = bn_stat(L.mbn, k, 2);
    tm.mshift = bn_stat(L.mbn, k, 3);
    conv_bwd_data(L.mc2, P(L.dm), P(L.dr), false, nullptr, nullptr, tm);
    bn_backward(L.mbn, k, P(L.dr), P(L.mh[k]), MASK_TENSOR, P(L.r[k]), P(L.dmh), 0);
    conv_bwd_weight(L.mc1, P(L.up[k]), P(L.dmh), false);
    conv_bwd_data(L.mc1, P(L.dmh), P(L.dup), false, nullptr, nullptr);
    {
      EltTimer tu(this, F_UP_BWD, (double)mb * C * (u.in.vol() + u.mask.vol()) * dt_size(dt));
      auto itu = opts.find("up_bwd_sep");
      if (dt == DT_BF16 && (itu == opts.end() || itu->second != 0))
        upsample_bwd_sep(P(L.dup), mb, u.mask.d, u.mask.h, u.mask.w, C, P(L.dum), u.in.d, u.in.h, u.in.w, L.tab,
                         (float *)P(off_up_ws), stream);
      else
        upsample_bwd(dt, P(L.dup), mb, u.mask.d, u.mask.h, u.mask.w, C, P(L.dum), u.in.d, u.in.h, u.in.w, L.tab,
                     stream);
    }
    block_bwd(L.mask, k, P(L.u0[k]), P(L.dum), P(L.du0), false);
    {
      EltTimer tp(this, F_MAXPOOL_BWD, (double)mb * C * (u.mask.vol() * (dt_size(dt) + 1.0) + u.in.vol() * dt_size(dt)));
      maxpool_bwd(dt, P(L.du0), (const uint8_t *)P(L.am[k]), mb, u.in.d, u.in.h, u.in.w, C, u.mask.d, u.mask.h,
                  u.mask.w, dx, false, stream);
    }
    block_bwd(L.trunk, k, x, P(L.dT), dx, true, dout_consumer(ui, k));
  } else {
    const int p0 = net.unit_param_begin[ui];
    head_bwd(dt, (const float *)P(L.dz[k]), (const float *)P(L.g[k]), master(p0), mb, (int)u.in.vol(), u.cin,
             grad(p0), grad(p0 + 1), dx, stream);
  }
}

// ---------------------------------------------------------------------------
// saved tensors by name (rn_get_saved: op-level teacher-forced parity)
// ---------------------------------------------------------------------------
bool Plan::saved(int ui, int k, const std::string &name, SavedRef &r) {
  const Unit &u = net.units[ui];
  UnitL &L = units[ui];
  auto act = [&](size_t off, int C, Dims d) {
    r.ptr = P(off);
    r.n = (int64_t)mb * d.vol() * C;
    r.type = 0;
    return true;
  };
  auto stats = [&](const BNL &b) {
    r.ptr = P(b.stat_off[k]);
    r.n = 4 * (int64_t)b.C;
    r.type = 1;
    return true;
  };
  auto block = [&](BlockL &B, const std::string &n) {
    const int C = B.cout;
    if (n == "h1") return act(B.h1[k], C, B.out);
    if (n == "a1") return act(B.a1[k], C, B.out);
    if (n == "h2") return act(B.h2[k], C, B.out);
    if (n == "out") return act(B.out_[k], C, B.out);
    if (n == "dh2") return act(B.dh2, C, B.out);
    if (n == "da1") return act(B.da1, C, B.out);
    if (n == "dh1") return act(B.dh1, C, B.out);
    if (n == "bn1.stats") return stats(B.b1);
    if (n == "bn2.stats") return stats(B.b2);
    if (B.proj) {
      if (n == "hp") return act(B.hp[k], C, B.out);
      if (n == "dhp") return act(B.dhp, C, B.out);
      if (n == "projbn.stats") return stats(B.bp);
    }
    return false;
  };
  if (u.kind == U_STEM) {
    if (name == "h") return act(L.stem_h[k], u.cout, u.conv);
    if (name == "bn.stats") return stats(L.stem_bn);
    if (name == "d1" && L.tmp0) return act(L.tmp0, u.cout, u.conv);
    if (name == "am" && u.pool) {
      r.ptr = P(L.am[k]);
      r.n = (int64_t)mb * u.out.vol() * u.cout;
      r.type = 2;
      return true;
    }
    return false;
  }
  if (u.kind == U_BLOCK) return block(L.blk, name);
  if (u.kind == U_ATT) {
    const int C = u.cout;
    if (name.rfind("trunk.", 0) == 0) return block(L.trunk, name.substr(6));
    if (name.rfind("mask.", 0) == 0) return block(L.mask, name.substr(5));
    if (name == "u0") return act(L.u0[k], C, u.mask);
    if (name == "am") {
      r.ptr = P(L.am[k]);
      r.n = (int64_t)mb * u.mask.vol() * C;
      r.type = 2;
      return true;
    }
    if (name == "up") return act(L.up[k], C, u.in);
    if (name == "mh") return act(L.mh[k], C, u.in);
    if (name == "r") return act(L.r[k], C, u.in);
    if (name == "m") return act(L.m[k], C, u.in);
    if (name == "mbn.stats") return stats(L.mbn);
    if (name == "dT") return act(L.dT, C, u.in);
    if (name == "dm") return act(L.dm, C, u.in);
    if (name == "dr") return act(L.dr, C, u.in);
    if (name == "dmh") return act(L.dmh, C, u.in);
    if (name == "dup") return act(L.dup, C, u.in);
    if (name == "dum") return act(L.dum, C, u.mask);
    if (name == "du0") return act(L.du0, C, u.mask);
    return false;
  }
  if (name == "dz") {
    r.ptr = P(L.dz[k]);
    r.n = (int64_t)mb * 2;
    r.type = 1;
    return true;
  }
  return false;
}

// ---------------------------------------------------------------------------
// step phases
// ---------------------------------------------------------------------------
// CUDA graphs: each phase is captured once (after one eager warm-up run that
// also sets kernel attributes) and replayed; the pointers inside are fixed
// because inputs are staged into plan-owned buffers.  Not used on the legacy
// default stream (not capturable) or while kernel timing is on.
bool Plan::graphs_on() const {
  auto it = opts.find("graphs");
  const bool on = it == opts.end() ? true : it->second != 0;
  // the in-process transport's host rendezvous cannot be captured into a graph
  return on && stream != nullptr && stream != cudaStreamLegacy && stream != cudaStreamPerThread && !timing() &&
         !nccl_is_local(world_comm) && !delayed && !async_ar();  // ASGD swaps gradient arrays per step
}

void Plan::drop_graphs() {
  for (int i = 0; i < 5; ++i) {
    if (gexec[i]) cudaGraphExecDestroy(gexec[i]);
    gexec[i] = nullptr;
    warm[i] = false;
  }
  if (alt_step.g3) cudaGraphExecDestroy(alt_step.g3);
  if (alt_step.g4) cudaGraphExecDestroy(alt_step.g4);
  alt_step = StepGraphs();
}

void Plan::run_phase(int ph, const std::function<void()> &body) {
  if (!graphs_on()) {
    body();
    return;
  }
  if (!gexec[ph]) {
    if (!warm[ph]) {
      body();
      warm[ph] = true;
      return;
    }
    cudaGraph_t g = nullptr;
    CUDA_CHECK(cudaStreamBeginCapture(stream, cudaStreamCaptureModeThreadLocal));
    set_capturing(true);
    try {
      body();
    } catch (...) {
      set_capturing(false);
      cudaStreamEndCapture(stream, &g);
      if (g) cudaGraphDestroy(g);
      throw;
    }
    set_capturing(false);
    CUDA_CHECK(cudaStreamEndCapture(stream, &g));
    size_t n = 0;
    CUDA_CHECK(cudaGraphGetNodes(g, nullptr, &n));
    std::vector<cudaGraphNode_t> nodes(n);
    CUDA_CHECK(cudaGraphGetNodes(g, nodes.data(), &n));
    int kn = 0;
    for (auto nd : nodes) {
      cudaGraphNodeType t;
      cudaGraphNodeGetType(nd, &t);
      kn += t == cudaGraphNodeTypeKernel;
    }
    graph_kernels[ph] = kn;
    const cudaError_t e = cudaGraphInstantiate(&gexec[ph], g, 0);
    cudaGraphDestroy(g);
    CUDA_CHECK(e);
  }
  CUDA_CHECK(cudaGraphLaunch(gexec[ph], stream));
  add_launches(graph_kernels[ph]);
}

void Plan::forward(const float *x_in, const int32_t *y) {
  run_phase(0, [&] { forward_body(x_in, y); });
  fwd_done = true;
  fwd_ever = true;
}

void Plan::backward(const float *x_in) {
  prepare_grad_clear();
  run_phase(1, [&] { backward_body(x_in); });
  bwd_ever = true;
}

void Plan::step(float lr) {
  if (lr != graph_lr) {  // the learning rate is a kernel argument of the captured step
    if (gexec[2]) cudaGraphExecDestroy(gexec[2]);
    gexec[2] = nullptr;
    warm[2] = false;
    graph_lr = lr;
  }
  run_phase(2, [&] { step_body(lr); });
}

// Early SGD (option "early_sgd", default on): the update of unit u depends only on
// u's own gradient, which is final once u's backward and its weight
// gradients are done; the next units' backward never reads u's weights.  So in a
// fused training step each unit's SGD + bf16 repack is issued on the weight-gradient
// stream right after the unit's backward (ordered after its dgrads by an event and
// after its wgrads by stream order) and overlaps the backward of the units below it,
// instead of one launch after the whole backward.  Same kernels, same per-element
// arithmetic: bitwise the weights of forward / backward / step.  Single stage, one
// micro-batch, no replica all-reduce (the update must wait for the reduced gradient
// there), synchronous schedule.
bool Plan::early_sgd_ok() const {
  auto it = opts.find("early_sgd");
  const bool on = it == opts.end() || it->second != 0;
  return on && unit_tables_ok && side_on() && Mb == 1 && S == 1 && replicas == 1 && !delayed && !async_ar();
}

void Plan::unit_sgd(int ui, float lr) {
  if (!side) {
    CUDA_CHECK(cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking));
    CUDA_CHECK(cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming));
    CUDA_CHECK(cudaEventCreateWithFlags(&ev_join, cudaEventDisableTiming));
  }
  if (!ev_sgd) CUDA_CHECK(cudaEventCreateWithFlags(&ev_sgd, cudaEventDisableTiming));
  CUDA_CHECK(cudaEventRecord(ev_sgd, stream));  // the unit's dgrads and BN / head gradients are done
  CUDA_CHECK(cudaStreamWaitEvent(side, ev_sgd, 0));
  side_used = true;
  const float *g = (const float *)P(off_grad);
  if (u_rg1[ui] > u_rg0[ui])
    sgd_ranges((const int64_t *)P(off_sgdrg) + 2 * u_rg0[ui], u_rg1[ui] - u_rg0[ui], (float *)P(off_master), g, lr,
               side);
  if (dt == DT_BF16 && u_pk1[ui] > u_pk0[ui])
    sgd_repack_range((const ConvPack *)P(off_pack) + u_pk0[ui], u_pk1[ui] - u_pk0[ui], u_t0[ui], u_t1[ui],
                     (float *)P(off_master), g, lr, side);
}

void Plan::train_step(const float *x_in, const int32_t *y, float lr) {
  if (!early_sgd_ok()) {
    forward(x_in, y);
    backward(x_in);
    step(lr);
    return;
  }
  if (x_in != tx_ptr || y != ty_ptr) select_step_graphs(x_in, y);  // phases 3 / 4 bake the pointers in
  run_phase(4, [&] { forward_body(x_in, y); });
  fwd_done = true;
  fwd_ever = true;
  if (lr != graph_lr3) {  // the learning rate is a kernel argument of the captured phase
    if (gexec[3]) cudaGraphExecDestroy(gexec[3]);
    gexec[3] = nullptr;
    warm[3] = false;
    graph_lr3 = lr;
  }
  prepare_grad_clear();
  run_phase(3, [&] { backward_body(x_in, -1, lr); });
  bwd_ever = true;
}

// the active phase-3/4 graphs belong to (tx_ptr, ty_ptr); alt_step caches the pair
// of one other input pointer: swap it in when it matches, else evict it
void Plan::select_step_graphs(const float *x, const int32_t *y) {
  StepGraphs cur;
  cur.x = tx_ptr;
  cur.y = ty_ptr;
  cur.g3 = gexec[3];
  cur.g4 = gexec[4];
  cur.w3 = warm[3];
  cur.w4 = warm[4];
  cur.k3 = graph_kernels[3];
  cur.k4 = graph_kernels[4];
  cur.lr3 = graph_lr3;
  StepGraphs nxt;
  if (alt_step.x == x && alt_step.y == y) {
    nxt = alt_step;
  } else {
    if (alt_step.g3) cudaGraphExecDestroy(alt_step.g3);
    if (alt_step.g4) cudaGraphExecDestroy(alt_step.g4);
    nxt.x = x;
    nxt.y = y;
  }
  alt_step = cur;
  tx_ptr = nxt.x;
  ty_ptr = nxt.y;
  gexec[3] = nxt.g3;
  gexec[4] = nxt.g4;
  warm[3] = nxt.w3;
  warm[4] = nxt.w4;
  graph_kernels[3] = nxt.k3;
  graph_kernels[4] = nxt.k4;
  graph_lr3 = nxt.lr3;
}

void Plan::train_step_dev(const float *x_dev, const int32_t *y_dev, float lr) {
  const bool same = x_dev == dev_x && y_dev == dev_y;
  same_xy = same ? same_xy + 1 : 0;
  dev_x = x_dev;
  dev_y = y_dev;
  const int nu = (int)net.units.size();
  const bool direct = same_xy >= 2 && early_sgd_ok() && graphs_on() && local[0] && local[nu - 1];
  if (direct) {
    train_step(x_dev, y_dev, lr);
  } else {
    stage_inputs(x_dev, y_dev, false);
    train_step((const float *)P(off_x), (const int32_t *)P(off_y), lr);
  }
}

void Plan::forward_body(const float *x_in, const int32_t *y, int k_only) {
  if (timing()) ev_used = 0;  // a step's conv events: this forward + its backward (eager launches)
  CUDA_CHECK(cudaMemsetAsync(P(off_loss), 0, sizeof(float), stream));
  const int nu = (int)net.units.size();
  for (int k = k_only < 0 ? 0 : k_only; k < (k_only < 0 ? Mb : k_only + 1); ++k) {
    for (int ui = 0; ui < nu; ++ui) {
      if (!local[ui]) continue;
      if (ui > 0 && !local[ui - 1] && !xfer_external) {
        const Unit &pu = net.units[ui - 1];
        nccl_recv_bytes(pipe_comm, P(units[ui].recv_in[k]), act_bytes(pu.cout, pu.out), unit_stage[ui - 1], stream);
      }
      {
        const size_t ue = timing() ? tk_begin(4, 0.0) : 0;  // per-unit time (f2 step-time model)
        unit_fwd(ui, k, x_in, y);
        if (timing()) tk_end(ue, ui);
      }
      if (ui + 1 < nu && !local[ui + 1] && !xfer_external) {
        const Unit &u = net.units[ui];
        nccl_send_bytes(pipe_comm, P(units[ui].out[k]), act_bytes(u.cout, u.out), unit_stage[ui + 1], stream);
      }
    }
  }
  if (gram_pending) {  // join the stem's input Gram matrix (weight-gradient stream)
    CUDA_CHECK(cudaEventRecord(ev_gjoin, side));
    CUDA_CHECK(cudaStreamWaitEvent(stream, ev_gjoin, 0));
    gram_pending = false;
  }
  if (S > 1 && !xfer_external) nccl_bcast_f32(pipe_comm, (float *)P(off_loss), 1, unit_stage[nu - 1], stream);
}

// Gradient clearing: the tensor-core weight gradients of a backward's first
// micro-batch STORE their result (option wgrad_overwrite, bf16 path), so only
// the rest of the gradient array — BN parameters, biases, the head, the stem and
// SIMT-path convs, non-local units — is zeroed (a few MB instead of the whole
// 134 MB array of r18, which cost ~28 us at the start of the backward).  The
// range table is rebuilt on the host before each backward / fused step (outside
// graph capture) and uploaded only when it changes.
void Plan::prepare_grad_clear() {
  auto it = opts.find("wgrad_overwrite");
  const bool on = (it == opts.end() || it->second != 0) && dt == DT_BF16;
  std::vector<std::pair<int64_t, int64_t>> tc;  // [begin, end) of tensor-core weight gradients
  if (on)
    for (const ConvL *c : conv_reg) {
      const bool x_f32 = c->g.Ci == 1;  // the stem reads the fp32 input
      if (!x_f32 && use_tc(c->g, false) && tc_wgrad_supported(c->g)) {
        const int64_t b = net.params[c->w_idx].canon_off;
        tc.emplace_back(b, b + net.params[c->w_idx].numel);
      }
    }
  std::sort(tc.begin(), tc.end());
  std::vector<int64_t> rg;
  int64_t cur = 0;
  for (auto &r : tc) {
    if (r.first > cur) {
      rg.push_back(cur);
      rg.push_back(r.first);
    }
    cur = std::max(cur, r.second);
  }
  if (cur < net.n_params) {
    rg.push_back(cur);
    rg.push_back(net.n_params);
  }
  wg_overwrite = on && !tc.empty();
  if (rg != zrg_host) {
    zrg_host = rg;
    if (!rg.empty())
      CUDA_CHECK(cudaMemcpyAsync(P(off_zrg), zrg_host.data(), zrg_host.size() * sizeof(int64_t),
                                 cudaMemcpyHostToDevice, stream));  // stream-ordered (outside any capture)
  }
}

void Plan::backward_body(const float *x_in, int k_only, float early_lr) {
  if (wg_overwrite) zero_ranges((const int64_t *)P(off_zrg), (int)(zrg_host.size() / 2), (float *)P(off_grad), stream);
  else CUDA_CHECK(cudaMemsetAsync(P(off_grad), 0, sizeof(float) * net.n_params, stream));
  const int nu = (int)net.units.size();
  const bool ov = overlap_ar();
  size_t bi = 0;
  const int k0 = k_only < 0 ? 0 : k_only, k1 = k_only < 0 ? Mb : k_only + 1;
  for (int k = k0; k < k1; ++k) {
    wg_first = k == k0;  // the first contribution to every weight gradient of this backward
    for (int ui = nu - 1; ui >= 0; --ui) {
      if (!local[ui]) continue;
      if (ui + 1 < nu && !local[ui + 1] && !xfer_external) {
        const Unit &u = net.units[ui];
        nccl_recv_bytes(pipe_comm, P(units[ui].dout), act_bytes(u.cout, u.out), unit_stage[ui + 1], stream);
      }
      {
        const size_t ue = timing() ? tk_begin(5, 0.0) : 0;
        unit_bwd(ui, k, x_in);
        if (timing()) tk_end(ue, ui);
      }
      if (ui > 0 && !local[ui - 1] && !xfer_external) {
        const Unit &pu = net.units[ui - 1];
        nccl_send_bytes(pipe_comm, P(units[ui].send_dx), act_bytes(pu.cout, pu.out), unit_stage[ui - 1], stream);
      }
      if (early_lr >= 0.f && k == k1 - 1) unit_sgd(ui, early_lr);
      // last micro-batch: a bucket whose units are all done is reduced while the
      // backward of the earlier units continues (P:284 ring all-reduce, Eq. 11)
      if (ov && k == k1 - 1 && bi < buckets.size() && ui == buckets[bi].ulo) launch_bucket(bi++);
    }
    if (side_used) {  // join the weight-gradient stream (per micro-batch: temporaries are reused)
      CUDA_CHECK(cudaEventRecord(ev_join, side));
      CUDA_CHECK(cudaStreamWaitEvent(stream, ev_join, 0));
      side_used = false;
    }
  }
  if (ov && comm_st) {  // the averaged gradient is complete when the backward is
    CUDA_CHECK(cudaEventRecord(ar_ev.back(), comm_st));
    CUDA_CHECK(cudaStreamWaitEvent(stream, ar_ev.back(), 0));
  }
  if (async_ar()) {
    // ASGD: this step's gradient is reduced in the background (not joined here);
    // the next step's update waits for it
    if (!comm_st) CUDA_CHECK(cudaStreamCreateWithFlags(&comm_st, cudaStreamNonBlocking));
    for (auto &e : ev_async)
      if (!e) CUDA_CHECK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    if (ar_ev.empty()) {
      cudaEvent_t e;
      CUDA_CHECK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      ar_ev.push_back(e);
    }
    CUDA_CHECK(cudaEventRecord(ar_ev[0], stream));
    CUDA_CHECK(cudaStreamWaitEvent(comm_st, ar_ev[0], 0));
    if (replicas > 1)
      for (auto &rg : local_ranges())
        nccl_allreduce_sum_f32(dp_comm, (float *)P(off_grad) + rg.first, (size_t)(rg.second - rg.first), comm_st);
    CUDA_CHECK(cudaEventRecord(ev_async[async_cur], comm_st));
  }
}

// The rank's schedule (host logic only; shared by Plan and rn_plan_describe).
// Partition p runs on stage genes[p]; unit u inherits its partition's stage.
// Exchanges in forward order: a unit whose predecessor is on another stage
// receives its input from there ("the partition output is sent to
// partition (i+1)"); a unit whose successor is elsewhere sends its output.
// Backward performs the mirror transfers in reverse order.
Schedule make_schedule(const NetModel &net, const rn_dist_desc &dd, int local_batch, DType dt) {
  Schedule sc;
  const int S = dd.n_stages;
  if (dd.world < 1 || dd.rank < 0 || dd.rank >= dd.world) throw Error(RN_ERR_ARG, "bad rank/world");
  if (S < 1 || dd.world % S != 0) throw Error(RN_ERR_ARG, "world must be a multiple of n_stages");
  if (dd.micro_batches < 1 || local_batch < 1 || local_batch % dd.micro_batches != 0)
    throw Error(RN_ERR_ARG, "local_batch must be a positive multiple of micro_batches");
  sc.stage = dd.rank % S;
  sc.replica = dd.rank / S;
  sc.replicas = dd.world / S;
  sc.mb = local_batch / dd.micro_batches;
  const int nparts = (int)net.part_loads.size();
  sc.genes.assign(nparts, 0);
  if (S > 1) {
    if (!dd.genes) throw Error(RN_ERR_ARG, "genes required when n_stages > 1");
    for (int i = 0; i < nparts; ++i) {
      sc.genes[i] = dd.genes[i];
      if (sc.genes[i] < 0 || sc.genes[i] >= S) throw Error(RN_ERR_ARG, "gene out of range");
    }
  }
  const int nu = (int)net.units.size();
  sc.unit_stage.assign(nu, 0);
  for (int p = 0; p < nparts; ++p)
    for (int u = net.part_first[p]; u < net.part_first[p + 1]; ++u) sc.unit_stage[u] = sc.genes[p];
  sc.local.assign(nu, 0);
  for (int u = 0; u < nu; ++u) sc.local[u] = sc.unit_stage[u] == sc.stage;
  for (int u = 0; u < nu; ++u) {
    if (!sc.local[u]) continue;
    if (u > 0 && !sc.local[u - 1]) {
      const Unit &pu = net.units[u - 1];
      sc.xfers.push_back({u, sc.unit_stage[u - 1], 0, (int64_t)sc.mb * pu.out.vol() * pu.cout * (int64_t)dt_size(dt)});
    }
    if (u + 1 < nu && !sc.local[u + 1]) {
      const Unit &cu = net.units[u];
      sc.xfers.push_back({u, sc.unit_stage[u + 1], 1, (int64_t)sc.mb * cu.out.vol() * cu.cout * (int64_t)dt_size(dt)});
    }
  }
  sc.ranges = local_param_ranges(net, sc.local);
  return sc;
}

std::vector<std::pair<int64_t, int64_t>> Plan::local_ranges() const { return local_param_ranges(net, local); }

// contiguous parameter ranges (in the flat buffer) of the local units
std::vector<std::pair<int64_t, int64_t>> local_param_ranges(const NetModel &net, const std::vector<char> &local) {
  std::vector<std::pair<int64_t, int64_t>> r;
  const int nu = (int)net.units.size();
  for (int ui = 0; ui < nu; ++ui) {
    if (!local[ui]) continue;
    const int a = net.unit_param_begin[ui], e = net.unit_param_end[ui];
    if (a == e) continue;
    int64_t s = net.params[a].canon_off;
    int64_t t = net.params[e - 1].canon_off + net.params[e - 1].numel;
    if (!r.empty() && r.back().second == s)
      r.back().second = t;
    else
      r.push_back({s, t});
  }
  return r;
}

// SGD: ranges of the non-conv tensors in one launch; every conv tensor
// (bf16 path) updated and repacked into its two bf16 copies in one more launch.
void Plan::step_body(float lr) {
  auto ranges = local_ranges();
  const float *gsrc = (const float *)P(off_grad);
  bool apply = true;
  const bool as = async_ar();
  if (as) {
    // ASGD (reading F4): this update applies the PREVIOUS step's replica-averaged
    // gradient (off_grad2; its all-reduce ran on comm_st during this step), G^{-1} = 0
    apply = async_have_prev;
    if (apply) CUDA_CHECK(cudaStreamWaitEvent(stream, ev_async[async_cur ^ 1], 0));
    gsrc = (const float *)P(off_grad2);
  } else if (replicas > 1 && !overlap_ar()) {  // else reduced during the backward (launch_bucket)
    for (auto &rg : ranges)
      nccl_allreduce_sum_f32(dp_comm, (float *)P(off_grad) + rg.first, (size_t)(rg.second - rg.first), stream);
  }
  if (apply) {
    int64_t conv_params = 0, all_params = 0;
    for (const auto &t : net.params)
      if (local[t.unit]) {
        all_params += t.numel;
        if (t.kind == P_CONV) conv_params += t.numel;
      }
    // w, g read + w written (fp32), + the bf16 forward and flipped dgrad copies of every conv weight
    EltTimer tm(this, F_SGD, 12.0 * all_params + (dt == DT_BF16 ? 4.0 * conv_params : 0.0));
    sgd_ranges((const int64_t *)P(off_sgdrg), n_sgdrg, (float *)P(off_master), gsrc, lr, stream);
    if (dt == DT_BF16)
      sgd_repack_all((const ConvPack *)P(off_pack), n_pack, pack_tiles, (float *)P(off_master), gsrc, lr, stream);
  }
  if (as) {
    // the gradient just computed (still reducing on comm_st) becomes the previous one;
    // the next backward writes the array this update consumed (stream order)
    std::swap(off_grad, off_grad2);
    async_cur ^= 1;
    async_have_prev = true;
  }
}

// One iteration t of the delayed-gradient pipeline (reading F1; Eqs.
// 1-2 P:158-166) on this rank's stage s (delay d = S-1-s):
//   1. group{ recv the batch-t input from stage s-1 ; send it the input gradient
//      this stage produced in iteration t-1 }
//   2. forward of batch t into slot t mod S with the current weights; stash them
//   3. group{ send the batch-t output to stage s+1 ; receive the gradient of this
//      stage's output for batch t-d (stage s+1 produced it in iteration t-1) }
//   4. loss of batch t broadcast from the last stage
//   5. backward of batch t-d (slot (t-d) mod S) with the weights its forward used
//   6. SGD on the current weights (+ data-parallel all-reduce over replicas)
// The two-sided groups pair neighbour stages (stage s's step 3 with stage s+1's
// step 1), so the exchanges cannot deadlock under NCCL's rendezvous sends.
void Plan::delayed_step(const float *x_dev, const int32_t *y_dev, float lr) {
  const int nu = (int)net.units.size();
  const int slot = (int)(iter % slots);
  const int d = S - 1 - stage;
  const int64_t bb = iter - d;
  const size_t xv = (size_t)b * net.units[0].in.vol();
  if (local[0] && x_dev)
    CUDA_CHECK(cudaMemcpyAsync((float *)P(off_x) + slot * xv, x_dev, sizeof(float) * xv, cudaMemcpyDeviceToDevice,
                               stream));
  if (local[nu - 1] && y_dev)
    CUDA_CHECK(cudaMemcpyAsync((int32_t *)P(off_y) + (size_t)slot * b, y_dev, sizeof(int32_t) * b,
                               cudaMemcpyDeviceToDevice, stream));
  xfer_external = true;
  const Unit *eu = &net.units[entry_unit];
  const Unit *pu = entry_unit > 0 ? &net.units[entry_unit - 1] : nullptr;
  // 1.
  if (entry_unit > 0) {
    nccl_group_start(pipe_comm);
    nccl_recv_bytes(pipe_comm, P(units[entry_unit].recv_in[slot]), act_bytes(pu->cout, pu->out),
                    unit_stage[entry_unit - 1], stream);
    if (dx_pending)
      nccl_send_bytes(pipe_comm, P(units[entry_unit].send_dx), act_bytes(pu->cout, pu->out),
                      unit_stage[entry_unit - 1], stream);
    nccl_group_end(pipe_comm);
  }
  dx_pending = false;
  (void)eu;
  // 2.
  forward_body((const float *)P(off_x), (const int32_t *)P(off_y), slot);
  CUDA_CHECK(cudaMemcpyAsync(P(stash_master[slot]), P(off_master), sizeof(float) * net.n_params,
                             cudaMemcpyDeviceToDevice, stream));
  for (size_t i = 0; i < shadow_d.size(); ++i)
    if (shadow_d[i])
      CUDA_CHECK(cudaMemcpyAsync(P(stash_shadow_d[slot][i]), P(shadow_d[i]), 2 * net.params[i].numel,
                                 cudaMemcpyDeviceToDevice, stream));
  // 3.
  if (exit_unit + 1 < nu) {
    const Unit &xu = net.units[exit_unit];
    nccl_group_start(pipe_comm);
    nccl_send_bytes(pipe_comm, P(units[exit_unit].out[slot]), act_bytes(xu.cout, xu.out), unit_stage[exit_unit + 1],
                    stream);
    if (bb >= 0)
      nccl_recv_bytes(pipe_comm, P(units[exit_unit].dout), act_bytes(xu.cout, xu.out), unit_stage[exit_unit + 1],
                      stream);
    nccl_group_end(pipe_comm);
  }
  // 4.
  if (S > 1) nccl_bcast_f32(pipe_comm, (float *)P(off_loss), 1, unit_stage[nu - 1], stream);
  // 5.-6.
  if (bb >= 0) {
    const int bs = (int)(bb % slots);
    std::swap(off_master, stash_master[bs]);  // the weights of batch bb's forward
    std::swap(shadow_d, stash_shadow_d[bs]);
    try {
      prepare_grad_clear();
      backward_body((const float *)P(off_x), bs);
    } catch (...) {
      std::swap(off_master, stash_master[bs]);
      std::swap(shadow_d, stash_shadow_d[bs]);
      xfer_external = false;
      throw;
    }
    std::swap(off_master, stash_master[bs]);
    std::swap(shadow_d, stash_shadow_d[bs]);
    dx_pending = entry_unit > 0;
    step_body(lr);
  }
  xfer_external = false;
  ++iter;
  fwd_ever = true;
  bwd_ever = bwd_ever || bb >= 0;
}

void Plan::refresh_shadows() {
  if (dt != DT_BF16) return;
  sgd_repack_all((const ConvPack *)P(off_pack), n_pack, pack_tiles, (float *)P(off_master), nullptr, 0.f, stream);
}

void Plan::bind(void *dev, size_t bytes) {
  if (bytes < ws_bytes) throw Error(RN_ERR_SIZE, "workspace smaller than required");
  if (((uintptr_t)dev & 255) != 0) throw Error(RN_ERR_ARG, "workspace must be 256-byte aligned");
  base = (char *)dev;
  CUDA_CHECK(cudaMemset(P(off_counter), 0, 256));
  // optimizer tables: conv tensors (bf16 copies) and plain SGD ranges, local units only
  std::vector<ConvPack> packs;
  std::vector<int64_t> rg;
  int64_t tiles = 0;
  const int nu = (int)net.units.size();
  u_pk0.assign(nu, 0); u_pk1.assign(nu, 0); u_rg0.assign(nu, 0); u_rg1.assign(nu, 0);
  u_t0.assign(nu, 0); u_t1.assign(nu, 0);
  std::vector<int> seen(nu, 0);
  unit_tables_ok = true;
  int last_unit = -1;
  for (int i = 0; i < (int)net.params.size(); ++i) {
    const ParamTensor &t = net.params[i];
    if (!local[t.unit]) continue;
    if (t.unit != last_unit) {  // a unit's tensors must be contiguous for its table slices
      if (seen[t.unit]) unit_tables_ok = false;
      seen[t.unit] = 1;
      u_pk0[t.unit] = u_pk1[t.unit] = (int)packs.size();
      u_t0[t.unit] = u_t1[t.unit] = tiles;
      u_rg0[t.unit] = u_rg1[t.unit] = (int)rg.size() / 2;
      last_unit = t.unit;
    }
    if (t.kind == P_CONV && dt == DT_BF16) {
      ConvPack c;
      c.off = t.canon_off;
      c.tile0 = tiles;
      c.Co = (int)t.shape[0];
      c.Ci = (int)t.shape[1];
      c.taps = (int)(t.shape[2] * t.shape[3] * t.shape[4]);
      c.pad = 0;
      c.wf = P(shadow_f[i]);
      c.wd = P(shadow_d[i]);
      tiles += (int64_t)c.taps * ((c.Co + 63) / 64) * ((c.Ci + 63) / 64);  // 64x64 tiles (sgd_repack_all_k)
      packs.push_back(c);
    } else {
      // adjacent tensors of one unit share a range (not across units: per-unit slices)
      if ((int)rg.size() / 2 > u_rg0[t.unit] && rg.back() == t.canon_off) rg.back() = t.canon_off + t.numel;
      else {
        rg.push_back(t.canon_off);
        rg.push_back(t.canon_off + t.numel);
      }
    }
    u_pk1[t.unit] = (int)packs.size();
    u_t1[t.unit] = tiles;
    u_rg1[t.unit] = (int)rg.size() / 2;
  }
  n_pack = (int)packs.size();
  pack_tiles = tiles;
  n_sgdrg = (int)rg.size() / 2;
  if (n_pack > max_pack || n_sgdrg > max_sgdrg) throw Error(RN_ERR_STATE, "optimizer table overflow");
  if (n_pack) CUDA_CHECK(cudaMemcpy(P(off_pack), packs.data(), sizeof(ConvPack) * n_pack, cudaMemcpyHostToDevice));
  if (n_sgdrg) CUDA_CHECK(cudaMemcpy(P(off_sgdrg), rg.data(), sizeof(int64_t) * rg.size(), cudaMemcpyHostToDevice));
}

// canonical conv W[Co][Ci][kd][kh][kw] <-> internal [Co][tap][Ci]
void Plan::canon_to_internal(const float *src, std::vector<float> &dst) const {
  dst.assign(src, src + net.n_params);
  for (const ParamTensor &t : net.params) {
    if (t.kind != P_CONV) continue;
    const int64_t Co = t.shape[0], Ci = t.shape[1], taps = t.shape[2] * t.shape[3] * t.shape[4];
    const float *s = src + t.canon_off;
    float *d = dst.data() + t.canon_off;
    for (int64_t co = 0; co < Co; ++co)
      for (int64_t ci = 0; ci < Ci; ++ci)
        for (int64_t tap = 0; tap < taps; ++tap) d[(co * taps + tap) * Ci + ci] = s[(co * Ci + ci) * taps + tap];
  }
}

void Plan::internal_to_canon(const float *src, float *dst) const {
  memcpy(dst, src, sizeof(float) * net.n_params);
  for (const ParamTensor &t : net.params) {
    if (t.kind != P_CONV) continue;
    const int64_t Co = t.shape[0], Ci = t.shape[1], taps = t.shape[2] * t.shape[3] * t.shape[4];
    const float *s = src + t.canon_off;
    float *d = dst + t.canon_off;
    for (int64_t co = 0; co < Co; ++co)
      for (int64_t ci = 0; ci < Ci; ++ci)
        for (int64_t tap = 0; tap < taps; ++tap) d[(co * Ci + ci) * taps + tap] = s[(co * taps + tap) * Ci + ci];
  }
}

void Plan::set_params(const float *host) {
  std::vector<float> tmp;
  canon_to_internal(host, tmp);
  CUDA_CHECK(cudaMemcpyAsync(P(off_master), tmp.data(), sizeof(float) * net.n_params, cudaMemcpyHostToDevice, stream));
  std::vector<float> z(net.n_bn_channels, 0.f), o(net.n_bn_channels, 1.f);
  CUDA_CHECK(cudaMemcpyAsync(P(off_run_mean), z.data(), sizeof(float) * z.size(), cudaMemcpyHostToDevice, stream));
  CUDA_CHECK(cudaMemcpyAsync(P(off_run_var), o.data(), sizeof(float) * o.size(), cudaMemcpyHostToDevice, stream));
  CUDA_CHECK(cudaMemsetAsync(P(off_grad), 0, sizeof(float) * net.n_params, stream));
  refresh_shadows();
  CUDA_CHECK(cudaStreamSynchronize(stream));
  params_set = true;
}

void Plan::get_flat(size_t off, float *host) {
  if (comm_st) CUDA_CHECK(cudaStreamSynchronize(comm_st));  // an ASGD all-reduce may be in flight
  std::vector<float> tmp(net.n_params);
  CUDA_CHECK(cudaStreamSynchronize(stream));
  CUDA_CHECK(cudaMemcpy(tmp.data(), P(off), sizeof(float) * net.n_params, cudaMemcpyDeviceToHost));
  internal_to_canon(tmp.data(), host);
}

// inputs are copied into plan-owned buffers so the step's pointers are fixed
// (CUDA-graph capturable) and x stays valid for the stem's weight gradient.
// n training steps from host inputs: step i+1's H2D copy (side stream, into
// staging slot (i+1)%2) overlaps step i; each step starts with a device-side copy
// staging -> plan input buffers (the captured graphs keep fixed pointers) and
// ends with an async copy of its loss into pinned memory.  Every step's inputs
// still cross PCIe inside the call.
void Plan::train_steps_host(const float *const *x_host, const int32_t *const *y_host, int n, float lr,
                            float *losses) {
  if (n <= 0) return;
  if (!copy_stream) {
    CUDA_CHECK(cudaStreamCreateWithFlags(&copy_stream, cudaStreamNonBlocking));
    for (int i = 0; i < 2; ++i) {
      CUDA_CHECK(cudaEventCreateWithFlags(&ev_copied[i], cudaEventDisableTiming));
      CUDA_CHECK(cudaEventCreateWithFlags(&ev_free[i], cudaEventDisableTiming));
    }
  }
  if (loss_pinned_n < n) {
    if (loss_pinned) CUDA_CHECK(cudaFreeHost(loss_pinned));
    CUDA_CHECK(cudaMallocHost((void **)&loss_pinned, sizeof(float) * n));
    loss_pinned_n = n;
  }
  const size_t xb = sizeof(float) * (size_t)b * net.units[0].in.vol();
  const size_t yoff = (xb + 255) / 256 * 256;
  const bool hx = local[0], hy = local[net.units.size() - 1];
  auto h2d = [&](int i) {
    char *slot = (char *)P(off_stage[i % 2]);
    if (i >= 2) CUDA_CHECK(cudaStreamWaitEvent(copy_stream, ev_free[i % 2], 0));
    if (hx) CUDA_CHECK(cudaMemcpyAsync(slot, x_host[i], xb, cudaMemcpyHostToDevice, copy_stream));
    if (hy) CUDA_CHECK(cudaMemcpyAsync(slot + yoff, y_host[i], sizeof(int32_t) * (size_t)b, cudaMemcpyHostToDevice,
                                       copy_stream));
    CUDA_CHECK(cudaEventRecord(ev_copied[i % 2], copy_stream));
  };
  // graphs captured per staging slot (the fused step only; the separate-phase path
  // bakes the workspace input in)
  const bool direct = early_sgd_ok() && graphs_on();
  h2d(0);
  for (int i = 0; i < n; ++i) {
    if (i + 1 < n) h2d(i + 1);
    const char *slot = (const char *)P(off_stage[i % 2]);
    CUDA_CHECK(cudaStreamWaitEvent(stream, ev_copied[i % 2], 0));
    if (direct) {  // the step reads the staging slot itself (its graphs cached per slot)
      train_step(hx ? (const float *)slot : (const float *)P(off_x),
                 hy ? (const int32_t *)(slot + yoff) : (const int32_t *)P(off_y), lr);
      CUDA_CHECK(cudaEventRecord(ev_free[i % 2], stream));  // the slot is read until the stem backward
    } else {
      if (hx) CUDA_CHECK(cudaMemcpyAsync(P(off_x), slot, xb, cudaMemcpyDeviceToDevice, stream));
      if (hy) CUDA_CHECK(cudaMemcpyAsync(P(off_y), slot + yoff, sizeof(int32_t) * (size_t)b,
                                         cudaMemcpyDeviceToDevice, stream));
      CUDA_CHECK(cudaEventRecord(ev_free[i % 2], stream));
      train_step((const float *)P(off_x), (const int32_t *)P(off_y), lr);
    }
    CUDA_CHECK(cudaMemcpyAsync(loss_pinned + i, P(off_loss), sizeof(float), cudaMemcpyDeviceToHost, stream));
  }
  CUDA_CHECK(cudaStreamSynchronize(stream));
  if (losses) memcpy(losses, loss_pinned, sizeof(float) * n);
}

void Plan::stage_inputs(const float *x, const int32_t *y, bool from_host) {
  const cudaMemcpyKind kind = from_host ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice;
  if (local[0] && x)
    CUDA_CHECK(cudaMemcpyAsync(P(off_x), x, sizeof(float) * (size_t)b * net.units[0].in.vol(), kind, stream));
  if (local[net.units.size() - 1] && y)
    CUDA_CHECK(cudaMemcpyAsync(P(off_y), y, sizeof(int32_t) * (size_t)b, kind, stream));
}

rn_status Plan::set_option(const std::string &k, int64_t v) {
  static const char *const known[] = {"graphs", "tc_conv", "time_kernels", "halo_conv", "fused_stats", "pair_conv",
                                      "wgrad_stream", "merge_proj", "recompute_mask", "up_bwd_sep", "pair_bwd_stats",
                                      "overlap_allreduce", "async_allreduce", "early_sgd", "c1x1", "att_branch",
                                      "res_prestore", "wgrad_overwrite"};
  bool ok = false;
  for (const char *n : known) ok = ok || k == n;
  if (!ok) return set_error(RN_ERR_ARG, "unknown option " + k);
  opts[k] = v;
  if (k == "time_kernels") ev_used = 0;
  if (k == "async_allreduce") async_have_prev = false;
  drop_graphs();
  return RN_OK;
}

rn_status Plan::query(const std::string &k, double *v) {
  if (k.rfind("conv_", 0) == 0) {
    // conv_ms / conv_flops / conv_launches, optionally suffixed _fprop/_dgrad/_wgrad
    CUDA_CHECK(cudaStreamSynchronize(stream));
    int cls = -1, kind = -1;
    if (k.find("_fprop") != std::string::npos) cls = 0;
    if (k.find("_dgrad") != std::string::npos) cls = 1;
    if (k.find("_wgrad") != std::string::npos) cls = 2;
    if (k.find("_pair") != std::string::npos) kind = K_PAIR;
    if (k.find("_tcconv") != std::string::npos) kind = K_TC;
    if (k.find("_tcwgrad") != std::string::npos) kind = K_WGRAD;
    if (k.find("_stem") != std::string::npos) kind = K_STEM;
    double ms = 0, fl = 0, n = 0;
    for (size_t i = 0; i < ev_used; ++i) {
      if (ev_pool[i].cls >= 3) continue;  // elementwise launches / unit brackets
      if (cls >= 0 && ev_pool[i].cls != cls) continue;
      if (kind >= 0 && ev_pool[i].kind != kind) continue;
      float e = 0.f;
      CUDA_CHECK(cudaEventElapsedTime(&e, ev_pool[i].a, ev_pool[i].b));
      ms += e;
      fl += ev_pool[i].flops;
      n += 1;
    }
    if (k.rfind("conv_ms", 0) == 0) *v = ms;
    else if (k.rfind("conv_flops", 0) == 0) *v = fl;
    else if (k.rfind("conv_launches", 0) == 0) *v = n;
    else return set_error(RN_ERR_ARG, "unknown statistic " + k);
    return RN_OK;
  }
  if (k.rfind("unit_ms_", 0) == 0) {
    // unit_ms_fwd_<u> / unit_ms_bwd_<u>: device time of unit u's forward / backward
    // (all its launches, summed over micro-batches) in the last timed step
    CUDA_CHECK(cudaStreamSynchronize(stream));
    const bool fwd = k.rfind("unit_ms_fwd_", 0) == 0;
    if (!fwd && k.rfind("unit_ms_bwd_", 0) != 0) return set_error(RN_ERR_ARG, "unknown statistic " + k);
    const int u = atoi(k.c_str() + 12);
    double ms = 0;
    for (size_t i = 0; i < ev_used; ++i) {
      if (ev_pool[i].cls != (fwd ? 4 : 5) || ev_pool[i].kind != u) continue;
      float e = 0.f;
      CUDA_CHECK(cudaEventElapsedTime(&e, ev_pool[i].a, ev_pool[i].b));
      ms += e;
    }
    *v = ms;
    return RN_OK;
  }
  if (k.rfind("elt_", 0) == 0) {
    // elt_ms / elt_bytes / elt_launches [_<family>] of the elementwise launches (time_kernels)
    CUDA_CHECK(cudaStreamSynchronize(stream));
    const std::string what = k.substr(4, k.find('_', 4) == std::string::npos ? std::string::npos : k.find('_', 4) - 4);
    int fam = -1;
    const size_t us = k.find('_', 4);
    if (us != std::string::npos) {
      const std::string f = k.substr(us + 1);
      for (int i = 0; kEltFamilies[i]; ++i)
        if (f == kEltFamilies[i]) fam = i;
      if (fam < 0) return set_error(RN_ERR_ARG, "unknown elementwise family " + f);
    }
    double ms = 0, by = 0, n = 0;
    for (size_t i = 0; i < ev_used; ++i) {
      if (ev_pool[i].cls != 3 || (fam >= 0 && ev_pool[i].kind != fam)) continue;
      float e = 0.f;
      CUDA_CHECK(cudaEventElapsedTime(&e, ev_pool[i].a, ev_pool[i].b));
      ms += e;
      by += ev_pool[i].flops;
      n += 1;
    }
    if (what == "ms") *v = ms;
    else if (what == "bytes") *v = by;
    else if (what == "launches") *v = n;
    else return set_error(RN_ERR_ARG, "unknown statistic " + k);
    return RN_OK;
  }
  auto it = stats.find(k);
  if (it == stats.end()) return set_error(RN_ERR_ARG, "unknown statistic " + k);
  *v = it->second;
  return RN_OK;
}

float Plan::read_loss() {
  float l = 0.f;
  CUDA_CHECK(cudaMemcpyAsync(&l, P(off_loss), sizeof(float), cudaMemcpyDeviceToHost, stream));
  CUDA_CHECK(cudaStreamSynchronize(stream));
  return l;
}

}  // namespace rn
