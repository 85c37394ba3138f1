// plan.h — per-rank executor state (see plan.cpp).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <functional>
#include <map>
#include <string>
#include <utility>
#include <vector>

#include "../../include/rn.h"
#include "comm.h"
#include "kernels.h"
#include "net.h"

namespace rn {

struct BNL {
  int gamma_idx = -1;  // param index of gamma (beta = +1)
  int C = 0;
  int64_t V = 0;       // voxels per micro-batch
  int64_t run_off = 0;
  std::vector<size_t> stat_off;  // per micro-batch: mean, invstd, scale, shift [4][C]
  // statistics partials fused into the producing convolution's epilogue
  // (bnstats.cuh): forward (sum h, sum h^2) and backward (sum dy', sum dy' h),
  // [P][2][C] with P = the producing launch's CTA count (0: not fused)
  size_t fpart = 0, bpart = 0;
  int fP = 0, bP = 0;
};

// where a convolution's epilogue sends the statistics of its output
struct StatsTarget {
  BNL *bn = nullptr;
  int mode = 0;                 // 1 forward, 2 backward
  const void *mask = nullptr;   // backward: the consumer's ReLU output
  const void *h = nullptr;      // backward: the consumer's BN input
  const float *mean = nullptr;  // backward: the consumer's batch mean
  // backward, optional: the consumer's BN scale/shift — its ReLU mask is then
  // recomputed from h (BN + ReLU without residual), the mask tensor is not read
  const float *mscale = nullptr, *mshift = nullptr;
};

struct ConvL {
  int w_idx = -1;
  ConvGeom g{};
};

struct BlockL {
  int cin = 0, cout = 0;
  Dims in, out;
  bool proj = false;
  ConvL c1, c2, cp;
  BNL b1, b2, bp;
  std::vector<size_t> h1, a1, h2, hp, out_;  // saved per micro-batch
  size_t dh2 = 0, da1 = 0, dh1 = 0, dhp = 0;  // backward temporaries
};

struct UnitL {
  int kind = 0;
  std::vector<size_t> out;    // unit output per micro-batch
  size_t dout = 0;            // gradient w.r.t. the unit output
  std::vector<size_t> recv_in;  // input received from another stage (per micro-batch)
  size_t send_dx = 0;           // gradient of the input, sent to the previous stage
  // stem
  ConvL stem_conv;
  BNL stem_bn;
  std::vector<size_t> stem_h, am;
  size_t tmp0 = 0, tmp1 = 0;
  size_t sws = 0;  // stem backward at pooled resolution (k_stem_bwd.cu): partial sums scratch
  size_t gws = 0;  // its input Gram matrix: per-block partials scratch
  std::vector<size_t> gd;     // per micro-batch: the fp64 Gram matrix [32][32]
  std::vector<char> gd_fwd;   // per micro-batch: computed by the forward (weight-gradient stream)
  // block
  BlockL blk;
  // attention
  BlockL trunk, mask;
  ConvL mc1, mc2;
  BNL mbn;
  int bias_idx = -1;
  std::vector<size_t> u0, up, mh, r, m;
  size_t dT = 0, dm = 0, dr = 0, dmh = 0, dup = 0, dum = 0, du0 = 0;
  UpTables tab{};
  // head
  std::vector<size_t> g, dz;
};

struct Schedule {
  std::vector<int> genes, unit_stage;
  std::vector<char> local;
  int stage = 0, replica = 0, replicas = 1, mb = 1;
  struct Xfer {
    int unit, peer_stage, dir;  // dir 0: receive the input of `unit`; 1: send the output of `unit`
    int64_t bytes;
  };
  std::vector<Xfer> xfers;                        // forward order
  std::vector<std::pair<int64_t, int64_t>> ranges;  // parameter ranges all-reduced over the DP group
};
Schedule make_schedule(const NetModel &net, const rn_dist_desc &dd, int local_batch, DType dt);
std::vector<std::pair<int64_t, int64_t>> local_param_ranges(const NetModel &net, const std::vector<char> &local);

struct SavedRef {
  const void *ptr = nullptr;
  int64_t n = 0;
  int type = 0;  // 0 activation dtype, 1 fp32, 2 uint8
};

struct Plan {
  NetModel net;
  DType dt;
  cudaStream_t stream;
  int nsm = 148;  // SM count of the plan's device (sizes the per-CTA statistics partials)
  int rank = 0, world = 1, S = 1, Mb = 1, b = 1, mb = 1, replicas = 1, stage = 0, replica = 0;
  std::vector<int> genes, unit_stage;
  std::vector<char> local;
  std::vector<int64_t> bn_run_off;
  std::vector<size_t> shadow_f, shadow_d;
  size_t off_master = 0, off_grad = 0, off_run_mean = 0, off_run_var = 0, off_loss = 0, off_flag = 0;
  size_t off_counter = 0;
  unsigned *counter() { return (unsigned *)P(off_counter); }
  size_t off_partial = 0, off_coef = 0, off_wgrad_ws = 0, off_x = 0, off_y = 0;
  // gradient clearing with overwriting tensor-core weight gradients (prepare_grad_clear)
  std::vector<const ConvL *> conv_reg;  // every conv of the local units
  size_t off_zrg = 0;                   // device [2][n] ranges zeroed at the start of a backward
  std::vector<int64_t> zrg_host;
  bool wg_overwrite = false, wg_first = false;
  void prepare_grad_clear();
  size_t wgrad_ws_floats = 0, conv_ws_floats = 0, off_conv_ws = 0, off_up_ws = 0;
  size_t off_pack = 0, off_sgdrg = 0;
  int n_pack = 0, n_sgdrg = 0, max_pack = 0, max_sgdrg = 0;
  int64_t pack_tiles = 0;
  int nblk_max = 0;
  size_t ws_bytes = 0;
  char *base = nullptr;
  std::vector<UnitL> units;
  std::vector<void *> up_dev;
  NcclComm *world_comm = nullptr, *pipe_comm = nullptr, *dp_comm = nullptr;
  bool params_set = false, fwd_done = false, fwd_ever = false, bwd_ever = false;
  const float *last_x = nullptr;

  Plan(const rn_net_desc &nd, const rn_dist_desc &dd, int local_batch, int dtype, cudaStream_t st,
       bool delayed = false);

  // --- delayed-gradient pipeline (Eqs. 1-2; reading F1) ---
  // slots = S saved forward states per rank (ring indexed by batch mod S), the
  // weights each forward used stashed per slot (master fp32 + the bf16 dgrad
  // copies), iteration counter; exchanges done by delayed_step itself
  bool delayed = false;
  int slots = 1;
  int64_t iter = 0;
  std::vector<size_t> stash_master;
  std::vector<std::vector<size_t>> stash_shadow_d;
  int entry_unit = -1, exit_unit = -1;  // first / last unit of this rank's (contiguous) stage
  bool dx_pending = false;              // input gradient of last iteration's backward not yet sent
  bool xfer_external = false;           // forward_body / backward_body skip their exchanges
  void delayed_step(const float *x_dev, const int32_t *y_dev, float lr);
  ~Plan();

  // workspace
  size_t alloc(size_t bytes);
  std::vector<size_t> per_mb(size_t bytes);
  void *P(size_t off) { return base + off; }
  size_t act_bytes(int C, Dims d) const;
  void make_bn(BNL &b, int gamma_idx, int C, int64_t V);
  void make_conv(ConvL &c, int w_idx, int Ci, int Co, int k, int s, int p, Dims in, Dims out);
  void make_block(BlockL &b, int pidx, int cin, int cout, int stride, Dims in);
  int block_param_count(int cin, int cout, int stride) const;
  void build_up_tables(UpTables &t, Dims in, Dims out);
  // Grad-CAM at the last conv layer for class cls over the last forward's batch
  void gradcam(int cls, float *map_dev);
  UpTables cam_tab{};
  bool cam_tab_built = false;

  // params
  float *master(int idx);
  float *grad(int idx);
  const void *wfwd(int idx);
  float *bn_stat(const BNL &b, int k, int which);

  // ops
  bool use_tc(const ConvGeom &g, bool dgrad) const;
  bool use_halo() const;
  bool use_pair() const;
  bool use_c1x1() const;
  bool recompute_mask() const;
  void conv_fwd(const ConvL &c, const void *x, void *y, const float *bias = nullptr, BNL *stats = nullptr);
  void conv_bwd_data(const ConvL &c, const void *dy, void *dx, bool accumulate, const void *res,
                     const void *res_mask, const StatsTarget &stats = StatsTarget());
  // stage-entry block: dx (+)= dgrad(c1, dy1) + dgrad(cp, dyp); one launch when both run on tcgen05
  void conv_bwd_data_proj(const ConvL &c1, const void *dy1, const ConvL &cp, const void *dyp, void *dx,
                          bool accumulate, const StatsTarget &stats);
  bool fused_stats() const;
  BnFinal bn_final(const BNL &b, int k);
  StatsTarget dout_consumer(int ui, int k);
  // h_fused / coef_fused: stem only (bf16, 64 channels): dy holds d' and the BN-backward apply
  // dh = A d' + B h + Cc is formed inside the weight-gradient kernel
  void conv_bwd_weight(const ConvL &c, const void *x, const void *dy, bool x_f32);
  bool stem_sparse_bwd(const Unit &u, const UnitL &L) const;
  void bn_forward_stats(const BNL &b, int k, const void *h);
  void bn_fwd(const BNL &b, int k, const void *h, const void *res, const float *rscale, const float *rshift, bool relu,
              void *y);
  // dprime (optional): also store dy' = dy * (mask > 0); returns false if this path cannot
  bool bn_backward(const BNL &b, int k, const void *dy, const void *h, int mask_mode, const void *mask_t, void *dx,
                   int slot, void *dprime = nullptr);
  void block_fwd(BlockL &B, int k, const void *x);
  void block_bwd(BlockL &B, int k, const void *x, const void *dout, void *dx, bool accumulate,
                 const StatsTarget &dx_stats = StatsTarget());
  const void *unit_input(int ui, int k, const float *x_in);
  void *unit_dx_target(int ui);
  void unit_fwd(int ui, int k, const float *x_in, const int32_t *y);
  void unit_bwd(int ui, int k, const float *x_in);

  // a saved forward tensor / backward temporary of unit ui by name (rn_get_saved)
  bool saved(int ui, int k, const std::string &name, SavedRef &r);

  // phases
  void bind(void *dev, size_t bytes);
  void stage_inputs(const float *x_dev, const int32_t *y_dev, bool from_host);
  // pipelined host-input training loop (inputs of step i+1 copied on a side
  // stream into a staging buffer while step i computes)
  size_t off_stage[2] = {0, 0};
  cudaStream_t copy_stream = nullptr;
  // weight gradients run on a side stream (forked when their dy is ready, joined
  // at the end of the backward): they are leaves of the backward graph, so they
  // overlap the dgrad / BN chain and fill its tails (option "wgrad_stream")
  cudaStream_t side = nullptr;
  // attention module: the soft-mask branch runs on its own stream, concurrent with
  // the trunk (forward); own split-K workspace (off_conv_ws2)
  cudaStream_t bstream = nullptr;
  cudaEvent_t ev_bfork = nullptr, ev_bjoin = nullptr;
  size_t off_conv_ws2 = 0;
  bool att_branch_on() const;
  void on_branch(const std::function<void()> &f);
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  cudaEvent_t ev_gfork = nullptr, ev_gjoin = nullptr;  // the stem's input Gram matrix on the side stream
  bool gram_pending = false;
  bool side_used = false;
  // data-parallel gradient all-reduce bucketed and overlapped with the backward
  // (option overlap_allreduce, default on when replicas > 1): bucket = a run of
  // consecutive local units (>= ~8 MB of fp32 gradients), reduced on comm_st as
  // soon as its last unit's backward (and weight gradients) are enqueued
  struct Bucket {
    int ulo, uhi;
    int64_t b, e;
  };
  std::vector<Bucket> buckets;  // backward order (units descending)
  cudaStream_t comm_st = nullptr;
  std::vector<cudaEvent_t> ar_ev;
  bool overlap_ar() const;
  void launch_bucket(size_t bi);
  // ASGD with ring all-reduce (reading F4; option async_allreduce): the
  // all-reduce of step t's gradient runs on comm_st during step t+1, whose update
  // applies it (double-buffered gradient arrays, swapped every step)
  size_t off_grad2 = 0;              // the previous step's gradient (reduced on comm_st)
  bool async_ar() const;
  bool async_have_prev = false;
  int async_cur = 0;                  // ev_async[async_cur]: this step's all-reduce
  cudaEvent_t ev_async[2] = {nullptr, nullptr};
  bool side_on() const;
  cudaEvent_t ev_copied[2] = {nullptr, nullptr}, ev_free[2] = {nullptr, nullptr};
  float *loss_pinned = nullptr;
  int loss_pinned_n = 0;
  void train_steps_host(const float *const *x_host, const int32_t *const *y_host, int n, float lr, float *losses);
  void forward(const float *x_in, const int32_t *y);
  void backward(const float *x_in);
  void step(float lr);
  void forward_body(const float *x_in, const int32_t *y, int k_only = -1);
  void backward_body(const float *x_in, int k_only = -1, float early_lr = -1.f);
  void step_body(float lr);
  // fused training step (rn_train_step): with early SGD each unit's update runs on
  // the weight-gradient stream as soon as its backward is done (early_sgd_ok())
  void train_step(const float *x_in, const int32_t *y, float lr);
  // rn_train_step from device inputs: after two calls with the same buffers the fused
  // step runs straight on them (its graphs captured for those pointers) instead of
  // copying them into the workspace first (28.9 MB D2D per r18 step)
  void train_step_dev(const float *x_dev, const int32_t *y_dev, float lr);
  const float *tx_ptr = nullptr;         // the input pointers phases 3 / 4 were captured with
  const int32_t *ty_ptr = nullptr;
  // a second cached pair of phase-3/4 graphs for another input pointer (the e2e path
  // alternates two staging slots): swapped in when its pointers come back
  struct StepGraphs {
    const float *x = nullptr;
    const int32_t *y = nullptr;
    cudaGraphExec_t g3 = nullptr, g4 = nullptr;
    bool w3 = false, w4 = false;
    int k3 = 0, k4 = 0;
    float lr3 = -1.f;
  } alt_step;
  void select_step_graphs(const float *x, const int32_t *y);
  const void *dev_x = nullptr, *dev_y = nullptr;   // the previous call's device inputs
  int same_xy = 0;
  bool early_sgd_ok() const;
  void unit_sgd(int ui, float lr);
  // per-unit slices of the optimizer tables (bind): conv packs [pk0, pk1) with tiles
  // [t0, t1), plain SGD ranges [rg0, rg1)
  std::vector<int> u_pk0, u_pk1, u_rg0, u_rg1;
  std::vector<int64_t> u_t0, u_t1;
  bool unit_tables_ok = false;
  cudaEvent_t ev_sgd = nullptr;
  // CUDA graphs per phase (0 forward, 1 backward, 2 step, 3 backward + early SGD)
  // phases: 0 forward, 1 backward, 2 step, 3 fused backward + early SGD, 4 forward of the fused step
  cudaGraphExec_t gexec[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};
  bool warm[5] = {false, false, false, false, false};
  int graph_kernels[5] = {0, 0, 0, 0, 0};
  float graph_lr = -1.f, graph_lr3 = -1.f;
  bool graphs_on() const;
  void drop_graphs();
  void run_phase(int ph, const std::function<void()> &body);
  void refresh_shadows();
  std::vector<std::pair<int64_t, int64_t>> local_ranges() const;

  // host I/O
  void canon_to_internal(const float *src, std::vector<float> &dst) const;
  void internal_to_canon(const float *src, float *dst) const;
  void set_params(const float *host);
  void get_flat(size_t off, float *host);
  float read_loss();
  // options / statistics
  std::map<std::string, int64_t> opts;
  std::map<std::string, double> stats;
  rn_status set_option(const std::string &k, int64_t v);
  rn_status query(const std::string &k, double *v);
  // live CUDA-event timing of the convolution launches (option time_kernels)
  struct EvPair {
    cudaEvent_t a, b;
    double flops;
    int cls;   // 0 fprop, 1 dgrad, 2 wgrad
    int kind;  // kernel family (K_*)
  };
  enum { K_SIMT = 0, K_PAIR = 1, K_TC = 2, K_HALO = 3, K_WGRAD = 4, K_STEM = 5 };
  std::vector<EvPair> ev_pool;
  size_t ev_used = 0;
  bool timing() const;
  size_t tk_begin(int cls, double flops);
  void tk_end(size_t i, int kind);
};

}  // namespace rn
