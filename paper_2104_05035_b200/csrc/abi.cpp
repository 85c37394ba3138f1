// abi.cpp — extern "C" entry points of librn.so (include/rn.h).  Argument
// validation, exception -> rn_status conversion, thread-local error message.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/rn.h"
#include "comm.h"
#include "error.h"
#include "net.h"
#include "plan.h"
#include "tc_conv.h"
#include "util.cuh"

namespace rn {
rn_status gabra_place(int32_t n, const int64_t *loads, int32_t m, const int64_t *caps, const rn_ga_params &gp,
                      int32_t *genes_out, double *profit_out, int64_t *gpu_load_out);

static thread_local std::string g_err;
static std::atomic<int64_t> g_launches{0};
// kernels launched by librn: counted at every eager launch; a CUDA-graph replay
// adds the number of kernel nodes it contains (captured launches are not counted)
static thread_local bool g_capturing = false;
void count_launch() {
  if (!g_capturing) g_launches.fetch_add(1, std::memory_order_relaxed);
}
void add_launches(int64_t n) { g_launches.fetch_add(n, std::memory_order_relaxed); }
void set_capturing(bool c) { g_capturing = c; }
int64_t launch_count() { return g_launches.load(); }
// Programmatic Dependent Launch for every kernel (launch.h): on by default
// (RN_PDL=0 turns it off).  Every kernel's griddepcontrol.wait sits after its
// smem / TMEM / barrier prologue; the trigger is implicit (a dependent grid
// launches when the predecessor's blocks exit) except in the persistent
// tensor-core convolutions, which issue griddepcontrol.launch_dependents after
// their last MMA (kPdlLate in k_conv_tc.cu / k_conv_pair.cu: the grid is fully
// resident, so no later wave can be displaced).  Measured: 3.917 -> 3.636 ms per
// r18 step (implicit trigger), 2198 -> 2203 samples/s (late explicit trigger); a
// trigger at kernel entry measured slower (dependents squat on SMs).
bool pdl_enabled() {
  static const bool on = [] {
    const char *e = getenv("RN_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}
rn_status set_error(rn_status s, const std::string &msg) {
  g_err = msg;
  return s;
}
}  // namespace rn

struct rn_plan_s {
  rn::Plan *p;
};

using namespace rn;

#define GUARD_BEGIN try {
#define GUARD_END                                               \
  }                                                             \
  catch (const rn::Error &e) {                                  \
    return set_error(e.status, e.what());                       \
  }                                                             \
  catch (const std::invalid_argument &e) {                      \
    return set_error(RN_ERR_SCHEMA, e.what());                  \
  }                                                             \
  catch (const std::bad_alloc &) {                              \
    return set_error(RN_ERR_SIZE, "host allocation failed");    \
  }                                                             \
  catch (const std::exception &e) {                             \
    return set_error(RN_ERR_STATE, e.what());                   \
  }

extern "C" {

void rn_ga_default(rn_ga_params *gp) {
  if (!gp) return;
  gp->pop_size = 50;
  gp->t_max = 500;
  gp->p_cross = 0.8;
  gp->p_mut = 0.1;
  gp->seed = 7;
  gp->dup_retries = 20;
  gp->init_attempts = 64;
  gp->require_all_used = 0;
  gp->early_stop_at_ub = 1;
  gp->objective = 0;
}

rn_status rn_gabra_place(int32_t n, const int64_t *loads, int32_t m, const int64_t *caps, const rn_ga_params *gp,
                         int32_t *genes_out, double *profit_out, int64_t *gpu_load_out) {
  GUARD_BEGIN
  if (n < 1 || m < 1 || !loads || !caps || !genes_out) return set_error(RN_ERR_ARG, "rn_gabra_place: bad arguments");
  for (int i = 0; i < n; ++i)
    if (loads[i] < 0) return set_error(RN_ERR_ARG, "rn_gabra_place: negative load");
  for (int j = 0; j < m; ++j)
    if (caps[j] <= 0) return set_error(RN_ERR_ARG, "rn_gabra_place: capacity must be > 0");
  rn_ga_params d;
  rn_ga_default(&d);
  const rn_ga_params &g = gp ? *gp : d;
  if (g.pop_size < 2 || g.t_max < 0 || g.dup_retries < 1 || g.init_attempts < 1 || g.p_cross < 0 || g.p_cross > 1 ||
      g.p_mut < 0 || g.p_mut > 1 || (g.objective != 0 && g.objective != 1))
    return set_error(RN_ERR_ARG, "rn_gabra_place: bad GA parameters");
  return gabra_place(n, loads, m, caps, g, genes_out, profit_out, gpu_load_out);
  GUARD_END
}

rn_status rn_gabra_place_slack(int32_t n, const int64_t *loads, int32_t m, const rn_ga_params *gp,
                               int32_t *genes_out, double *profit_out, int64_t *gpu_load_out, int64_t *caps_out,
                               double *slack_out) {
  GUARD_BEGIN
  if (n < 1 || m < 1 || !loads || !genes_out) return set_error(RN_ERR_ARG, "rn_gabra_place_slack: bad arguments");
  int64_t tot = 0, mx = 0;
  for (int i = 0; i < n; ++i) {
    if (loads[i] < 0) return set_error(RN_ERR_ARG, "rn_gabra_place_slack: negative load");
    tot += loads[i];
    mx = std::max(mx, loads[i]);
  }
  const int64_t base = std::max(mx, (tot + m - 1) / m);
  if (base <= 0) return set_error(RN_ERR_ARG, "rn_gabra_place_slack: all loads are zero");
  std::vector<int64_t> caps(m);
  for (int k = 11; k <= 20; ++k) {  // reading G4b: slack k/10
    const double s = k / 10.0;
    const int64_t d = (int64_t)std::ceil(s * (double)base);
    for (int j = 0; j < m; ++j) caps[j] = d;
    const rn_status r = rn_gabra_place(n, loads, m, caps.data(), gp, genes_out, profit_out, gpu_load_out);
    if (r == RN_ERR_INFEASIBLE) continue;
    if (r != RN_OK) return r;
    if (caps_out)
      for (int j = 0; j < m; ++j) caps_out[j] = d;
    if (slack_out) *slack_out = s;
    return RN_OK;
  }
  return set_error(RN_ERR_INFEASIBLE, "rn_gabra_place_slack: no capacity-respecting placement up to slack 2.0");
  GUARD_END
}

rn_status rn_simulate_step(const rn_sim_desc *d, double *step_s, double *pipeline_s, double *allreduce_s,
                           double *stage_s) {
  GUARD_BEGIN
  if (!d || !step_s || !pipeline_s || !allreduce_s || !d->part_time || !d->param_bytes || !d->genes ||
      (d->n > 1 && !d->cut_bytes) || d->n < 1 || d->n_stages < 1 || d->replicas < 1 || d->micro_batches < 1 ||
      !(d->beta > 0))
    return set_error(RN_ERR_ARG, "rn_simulate_step: bad arguments");
  for (int i = 0; i < d->n; ++i)
    if (d->genes[i] < 0 || d->genes[i] >= d->n_stages) return set_error(RN_ERR_ARG, "rn_simulate_step: bad gene");
  simulate_step(*d, step_s, pipeline_s, allreduce_s, stage_s);
  return RN_OK;
  GUARD_END
}

rn_status rn_contiguous_split(int32_t n, const int64_t *loads, int32_t n_stages, int32_t *genes_out,
                              int64_t *max_load_out) {
  GUARD_BEGIN
  if (!loads || !genes_out || n_stages < 1 || n < n_stages) return set_error(RN_ERR_ARG, "rn_contiguous_split: bad arguments");
  for (int i = 0; i < n; ++i)
    if (loads[i] < 0) return set_error(RN_ERR_ARG, "rn_contiguous_split: negative load");
  contiguous_split(n, loads, n_stages, genes_out, max_load_out);
  return RN_OK;
  GUARD_END
}

rn_status rn_net_units(const rn_net_desc *net, int32_t *n_units, int64_t *unit_loads, int32_t *n_parts,
                       int32_t *part_first_unit, int64_t *part_loads) {
  GUARD_BEGIN
  if (!net) return set_error(RN_ERR_ARG, "null net");
  NetModel m = build_net(*net);
  if (n_units) *n_units = (int32_t)m.units.size();
  if (unit_loads)
    for (size_t i = 0; i < m.units.size(); ++i) unit_loads[i] = m.unit_costs[i];
  if (n_parts) *n_parts = (int32_t)m.part_loads.size();
  if (part_first_unit)
    for (size_t i = 0; i < m.part_first.size(); ++i) part_first_unit[i] = m.part_first[i];
  if (part_loads)
    for (size_t i = 0; i < m.part_loads.size(); ++i) part_loads[i] = m.part_loads[i];
  return RN_OK;
  GUARD_END
}

rn_status rn_net_param_count(const rn_net_desc *net, int64_t *n_params, int32_t *n_tensors, int32_t *n_bn_channels) {
  GUARD_BEGIN
  if (!net) return set_error(RN_ERR_ARG, "null net");
  NetModel m = build_net(*net);
  if (n_params) *n_params = m.n_params;
  if (n_tensors) *n_tensors = (int32_t)m.params.size();
  if (n_bn_channels) *n_bn_channels = (int32_t)m.n_bn_channels;
  return RN_OK;
  GUARD_END
}

rn_status rn_net_param_info(const rn_net_desc *net, int32_t idx, int32_t *ndim, int64_t *shape5, int32_t *kind,
                            int32_t *unit, char *name, int32_t name_cap) {
  GUARD_BEGIN
  if (!net) return set_error(RN_ERR_ARG, "null net");
  NetModel m = build_net(*net);
  if (idx < 0 || idx >= (int)m.params.size()) return set_error(RN_ERR_ARG, "param index out of range");
  const ParamTensor &t = m.params[idx];
  if (ndim) *ndim = t.ndim;
  if (shape5)
    for (int i = 0; i < 5; ++i) shape5[i] = t.shape[i];
  if (kind) *kind = t.kind;
  if (unit) *unit = t.unit;
  if (name && name_cap > 0) {
    strncpy(name, t.name.c_str(), name_cap - 1);
    name[name_cap - 1] = 0;
  }
  return RN_OK;
  GUARD_END
}

rn_status rn_nccl_unique_id(uint8_t out[128]) {
  GUARD_BEGIN
  if (!out) return set_error(RN_ERR_ARG, "null out");
  nccl_unique_id(out);
  return RN_OK;
  GUARD_END
}

rn_status rn_plan(const rn_net_desc *net, const rn_dist_desc *dist, int32_t local_batch, int32_t dtype,
                  void *cuda_stream, rn_plan_t *out, size_t *workspace_bytes) {
  GUARD_BEGIN
  if (!net || !out || !workspace_bytes) return set_error(RN_ERR_ARG, "rn_plan: null argument");
  if (dtype != RN_F32 && dtype != RN_BF16) return set_error(RN_ERR_ARG, "rn_plan: dtype must be RN_F32 or RN_BF16");
  rn_dist_desc d;
  memset(&d, 0, sizeof d);
  d.world = 1;
  d.n_stages = 1;
  d.micro_batches = 1;
  if (dist) d = *dist;
  Plan *p = new Plan(*net, d, local_batch, dtype, (cudaStream_t)cuda_stream);
  *out = new rn_plan_s{p};
  *workspace_bytes = p->ws_bytes;
  return RN_OK;
  GUARD_END
}

rn_status rn_plan_delayed(const rn_net_desc *net, const rn_dist_desc *dist, int32_t local_batch, int32_t dtype,
                          void *cuda_stream, rn_plan_t *out, size_t *workspace_bytes) {
  GUARD_BEGIN
  if (!net || !out || !workspace_bytes) return set_error(RN_ERR_ARG, "rn_plan_delayed: null argument");
  if (dtype != RN_F32 && dtype != RN_BF16) return set_error(RN_ERR_ARG, "rn_plan_delayed: bad dtype");
  rn_dist_desc d;
  memset(&d, 0, sizeof d);
  d.world = 1;
  d.n_stages = 1;
  d.micro_batches = 1;
  if (dist) d = *dist;
  Plan *p = new Plan(*net, d, local_batch, dtype, (cudaStream_t)cuda_stream, true);
  *out = new rn_plan_s{p};
  *workspace_bytes = p->ws_bytes;
  return RN_OK;
  GUARD_END
}


rn_status rn_plan_describe(const rn_net_desc *net, const rn_dist_desc *dist, int32_t local_batch, int32_t dtype,
                           int32_t *local_units, int32_t cap, int32_t *n_xfer, int64_t *xfer, int32_t *n_ranges,
                           int64_t *ranges) {
  GUARD_BEGIN
  if (!net || !dist || !n_xfer || !n_ranges || cap < 0) return set_error(RN_ERR_ARG, "rn_plan_describe: null argument");
  NetModel m = build_net(*net);
  Schedule sc = make_schedule(m, *dist, local_batch, dtype == RN_BF16 ? DT_BF16 : DT_F32);
  if ((int)sc.xfers.size() > cap || (int)sc.ranges.size() > cap) return set_error(RN_ERR_SIZE, "cap too small");
  if (local_units)
    for (size_t u = 0; u < m.units.size(); ++u) local_units[u] = sc.local[u];
  *n_xfer = (int32_t)sc.xfers.size();
  for (size_t i = 0; i < sc.xfers.size() && xfer; ++i) {
    xfer[4 * i] = sc.xfers[i].unit;
    xfer[4 * i + 1] = sc.xfers[i].peer_stage;
    xfer[4 * i + 2] = sc.xfers[i].dir;
    xfer[4 * i + 3] = sc.xfers[i].bytes;
  }
  *n_ranges = (int32_t)sc.ranges.size();
  for (size_t i = 0; i < sc.ranges.size() && ranges; ++i) {
    ranges[2 * i] = sc.ranges[i].first;
    ranges[2 * i + 1] = sc.ranges[i].second;
  }
  return RN_OK;
  GUARD_END
}

rn_status rn_plan_bind(rn_plan_t plan, void *dev, size_t bytes) {
  GUARD_BEGIN
  if (!plan || !dev) return set_error(RN_ERR_ARG, "rn_plan_bind: null argument");
  plan->p->bind(dev, bytes);
  return RN_OK;
  GUARD_END
}

#define NEED_BOUND(plan)                                                            \
  if (!plan) return set_error(RN_ERR_ARG, "null plan");                             \
  if (!plan->p->base) return set_error(RN_ERR_STATE, "plan has no workspace bound");

rn_status rn_set_params(rn_plan_t plan, const float *host, int64_t count) {
  GUARD_BEGIN
  NEED_BOUND(plan);
  if (!host) return set_error(RN_ERR_ARG, "null host");
  if (count != plan->p->net.n_params) return set_error(RN_ERR_SIZE, "count != n_params");
  plan->p->set_params(host);
  return RN_OK;
  GUARD_END
}

rn_status rn_get_params(rn_plan_t plan, float *host, int64_t count) {
  GUARD_BEGIN
  NEED_BOUND(plan);
  if (!host) return set_error(RN_ERR_ARG, "null host");
  if (count != plan->p->net.n_params) return set_error(RN_ERR_SIZE, "count != n_params");
  plan->p->get_flat(plan->p->off_master, host);
  return RN_OK;
  GUARD_END
}

rn_status rn_get_grads(rn_plan_t plan, float *host, int64_t count) {
  GUARD_BEGIN
  NEED_BOUND(plan);
  if (!host) return set_error(RN_ERR_ARG, "null host");
  if (count != plan->p->net.n_params) return set_error(RN_ERR_SIZE, "count != n_params");
  plan->p->get_flat(plan->p->off_grad, host);
  return RN_OK;
  GUARD_END
}

rn_status rn_get_bn_running(rn_plan_t plan, float *mean_host, float *var_host, int64_t count) {
  GUARD_BEGIN
  NEED_BOUND(plan);
  Plan *p = plan->p;
  if (count != p->net.n_bn_channels) return set_error(RN_ERR_SIZE, "count != n_bn_channels");
  CUDA_CHECK(cudaStreamSynchronize(p->stream));
  if (mean_host) CUDA_CHECK(cudaMemcpy(mean_host, p->P(p->off_run_mean), 4 * count, cudaMemcpyDeviceToHost));
  if (var_host) CUDA_CHECK(cudaMemcpy(var_host, p->P(p->off_run_var), 4 * count, cudaMemcpyDeviceToHost));
  return RN_OK;
  GUARD_END
}

rn_status rn_get_activation(rn_plan_t plan, int32_t unit, int32_t micro_batch, float *host, int64_t count) {
  GUARD_BEGIN
  NEED_BOUND(plan);
  Plan *p = plan->p;
  if (!host || unit < 0 || unit >= (int)p->net.units.size() || !p->local[unit] || micro_batch < 0 ||
      micro_batch >= p->Mb)
    return set_error(RN_ERR_ARG, "rn_get_activation: bad unit / micro-batch");
  const Unit &u = p->net.units[unit];
  const bool head = u.kind == U_HEAD;
  const int64_t n = head ? (int64_t)p->mb * u.cin : (int64_t)p->mb * u.out.vol() * u.cout;
  if (count != n) return set_error(RN_ERR_SIZE, "rn_get_activation: count mismatch");
  CUDA_CHECK(cudaStreamSynchronize(p->stream));
  const void *src = head ? p->P(p->units[unit].g[micro_batch]) : p->P(p->units[unit].out[micro_batch]);
  if (head || p->dt == DT_F32) {
    CUDA_CHECK(cudaMemcpy(host, src, 4 * n, cudaMemcpyDeviceToHost));
  } else {
    std::vector<uint16_t> tmp(n);
    CUDA_CHECK(cudaMemcpy(tmp.data(), src, 2 * n, cudaMemcpyDeviceToHost));
    for (int64_t i = 0; i < n; ++i) {
      uint32_t b = (uint32_t)tmp[i] << 16;
      memcpy(&host[i], &b, 4);
    }
  }
  return RN_OK;
  GUARD_END
}

rn_status rn_get_unit_grad(rn_plan_t plan, int32_t unit, float *host, int64_t count) {
  GUARD_BEGIN
  NEED_BOUND(plan);
  Plan *p = plan->p;
  if (!host || unit < 0 || unit >= (int)p->net.units.size() || !p->local[unit] ||
      p->net.units[unit].kind == U_HEAD)
    return set_error(RN_ERR_ARG, "rn_get_unit_grad: bad unit (head, not local or out of range)");
  if (!p->bwd_ever) return set_error(RN_ERR_STATE, "rn_get_unit_grad before rn_backward");
  const Unit &u = p->net.units[unit];
  const int64_t n = (int64_t)p->mb * u.out.vol() * u.cout;
  if (count != n) return set_error(RN_ERR_SIZE, "rn_get_unit_grad: count mismatch");
  CUDA_CHECK(cudaStreamSynchronize(p->stream));
  const void *src = p->P(p->units[unit].dout);
  if (p->dt == DT_F32) {
    CUDA_CHECK(cudaMemcpy(host, src, 4 * n, cudaMemcpyDeviceToHost));
  } else {
    std::vector<uint16_t> tmp(n);
    CUDA_CHECK(cudaMemcpy(tmp.data(), src, 2 * n, cudaMemcpyDeviceToHost));
    for (int64_t i = 0; i < n; ++i) {
      uint32_t b = (uint32_t)tmp[i] << 16;
      memcpy(&host[i], &b, 4);
    }
  }
  return RN_OK;
  GUARD_END
}

rn_status rn_get_saved(rn_plan_t plan, int32_t unit, const char *name, int32_t micro_batch, float *host,
                       int64_t count) {
  GUARD_BEGIN
  NEED_BOUND(plan);
  Plan *p = plan->p;
  if (!host || !name || unit < 0 || unit >= (int)p->net.units.size() || !p->local[unit] || micro_batch < 0 ||
      micro_batch >= p->Mb)
    return set_error(RN_ERR_ARG, "rn_get_saved: bad unit / micro-batch");
  SavedRef r;
  if (!p->saved(unit, micro_batch, name, r)) return set_error(RN_ERR_ARG, "rn_get_saved: unknown tensor name");
  if (count != r.n) return set_error(RN_ERR_SIZE, "rn_get_saved: count mismatch");
  CUDA_CHECK(cudaStreamSynchronize(p->stream));
  if (r.type == 1 || (r.type == 0 && p->dt == DT_F32)) {
    CUDA_CHECK(cudaMemcpy(host, r.ptr, 4 * r.n, cudaMemcpyDeviceToHost));
  } else if (r.type == 2) {
    std::vector<uint8_t> tmp(r.n);
    CUDA_CHECK(cudaMemcpy(tmp.data(), r.ptr, r.n, cudaMemcpyDeviceToHost));
    for (int64_t i = 0; i < r.n; ++i) host[i] = (float)tmp[i];
  } else {
    std::vector<uint16_t> tmp(r.n);
    CUDA_CHECK(cudaMemcpy(tmp.data(), r.ptr, 2 * r.n, cudaMemcpyDeviceToHost));
    for (int64_t i = 0; i < r.n; ++i) {
      uint32_t b = (uint32_t)tmp[i] << 16;
      memcpy(&host[i], &b, 4);
    }
  }
  return RN_OK;
  GUARD_END
}

rn_status rn_gradcam(rn_plan_t plan, int32_t cls, float *map_dev, int64_t count) {
  GUARD_BEGIN
  NEED_BOUND(plan);
  Plan *p = plan->p;
  if (!map_dev) return set_error(RN_ERR_ARG, "rn_gradcam: null map");
  if (!p->fwd_ever) return set_error(RN_ERR_STATE, "rn_gradcam before rn_forward");
  if (count != (int64_t)p->b * p->net.units[0].in.vol()) return set_error(RN_ERR_SIZE, "rn_gradcam: count mismatch");
  p->gradcam(cls, map_dev);
  return RN_OK;
  GUARD_END
}

static rn_status finish_loss(Plan *p, float *loss_host) {
  if (!loss_host) return RN_OK;
  float l = p->read_loss();
  *loss_host = l;
  if (!std::isfinite(l)) return set_error(RN_ERR_NUMERIC, "non-finite loss");
  return RN_OK;
}

rn_status rn_forward(rn_plan_t plan, const void *x_dev, const int32_t *y_dev, float *loss_host) {
  GUARD_BEGIN
  NEED_BOUND(plan);
  Plan *p = plan->p;
  if (!p->params_set) return set_error(RN_ERR_STATE, "rn_set_params must precede rn_forward");
  p->stage_inputs((const float *)x_dev, y_dev, false);
  p->forward((const float *)p->P(p->off_x), (const int32_t *)p->P(p->off_y));
  return finish_loss(p, loss_host);
  GUARD_END
}

rn_status rn_backward(rn_plan_t plan) {
  GUARD_BEGIN
  NEED_BOUND(plan);
  Plan *p = plan->p;
  if (!p->fwd_done) return set_error(RN_ERR_STATE, "rn_backward before rn_forward");
  p->backward((const float *)p->P(p->off_x));
  p->fwd_done = false;
  return RN_OK;
  GUARD_END
}

rn_status rn_step(rn_plan_t plan, float lr) {
  GUARD_BEGIN
  NEED_BOUND(plan);
  plan->p->step(lr);
  return RN_OK;
  GUARD_END
}

rn_status rn_delayed_step(rn_plan_t plan, const void *x_dev, const int32_t *y_dev, float lr, float *loss_host) {
  GUARD_BEGIN
  NEED_BOUND(plan);
  Plan *p = plan->p;
  if (!p->delayed) return set_error(RN_ERR_STATE, "rn_delayed_step: plan not created by rn_plan_delayed");
  if (!p->params_set) return set_error(RN_ERR_STATE, "rn_set_params must precede rn_delayed_step");
  p->delayed_step((const float *)x_dev, y_dev, lr);
  return finish_loss(p, loss_host);
  GUARD_END
}

rn_status rn_train_step_host(rn_plan_t plan, const float *x_host, const int32_t *y_host, float lr, float *loss_host) {
  GUARD_BEGIN
  NEED_BOUND(plan);
  Plan *p = plan->p;
  if (!p->params_set) return set_error(RN_ERR_STATE, "rn_set_params must precede a step");
  p->stage_inputs(x_host, y_host, true);
  p->train_step((const float *)p->P(p->off_x), (const int32_t *)p->P(p->off_y), lr);
  return finish_loss(p, loss_host);
  GUARD_END
}

rn_status rn_train_step(rn_plan_t plan, const void *x_dev, const int32_t *y_dev, float lr, float *loss_host) {
  GUARD_BEGIN
  NEED_BOUND(plan);
  Plan *p = plan->p;
  if (!p->params_set) return set_error(RN_ERR_STATE, "rn_set_params must precede a step");
  p->train_step_dev((const float *)x_dev, y_dev, lr);
  p->fwd_done = false;
  return finish_loss(p, loss_host);
  GUARD_END
}

rn_status rn_train_steps_host(rn_plan_t plan, const float *const *x_host, const int32_t *const *y_host,
                              int32_t n_steps, float lr, float *losses_host) {
  GUARD_BEGIN
  NEED_BOUND(plan);
  Plan *p = plan->p;
  if (!p->params_set) return set_error(RN_ERR_STATE, "rn_set_params must precede a step");
  if (n_steps < 0 || (n_steps > 0 && (!x_host || !y_host))) return set_error(RN_ERR_ARG, "bad step inputs");
  for (int i = 0; i < n_steps; ++i)
    if ((p->local[0] && !x_host[i]) || (p->local[p->net.units.size() - 1] && !y_host[i]))
      return set_error(RN_ERR_ARG, "null host input");
  p->train_steps_host(x_host, y_host, n_steps, lr, losses_host);
  if (losses_host)
    for (int i = 0; i < n_steps; ++i)
      if (!std::isfinite(losses_host[i])) return set_error(RN_ERR_NUMERIC, "non-finite loss");
  return RN_OK;
  GUARD_END
}

int64_t rn_kernel_launches(rn_plan_t) { return rn::launch_count(); }

rn_status rn_set_option(rn_plan_t plan, const char *key, int64_t value) {
  GUARD_BEGIN
  if (!plan || !key) return set_error(RN_ERR_ARG, "null argument");
  return plan->p->set_option(key, value);
  GUARD_END
}

rn_status rn_query(rn_plan_t plan, const char *key, double *value) {
  GUARD_BEGIN
  if (!plan || !key || !value) return set_error(RN_ERR_ARG, "null argument");
  return plan->p->query(key, value);
  GUARD_END
}

rn_status rn_op_conv3d(int32_t dtype, int32_t op, const int32_t *geom, const void *a_dev, const void *b_dev,
                       void *out_dev, int32_t impl, void *stream) {
  GUARD_BEGIN
  if (!geom || !a_dev || !b_dev || !out_dev || op < 0 || op > 2 || impl < 0 || impl > 6 ||
      (dtype != RN_F32 && dtype != RN_BF16))
    return set_error(RN_ERR_ARG, "rn_op_conv3d: bad arguments");
  ConvGeom g;
  g.N = geom[0]; g.Di = geom[1]; g.Hi = geom[2]; g.Wi = geom[3]; g.Ci = geom[4];
  g.Do = geom[5]; g.Ho = geom[6]; g.Wo = geom[7]; g.Co = geom[8]; g.k = geom[9]; g.s = geom[10]; g.p = geom[11];
  if (g.Do != conv_out(g.Di, g.k, g.s, g.p) || g.Ho != conv_out(g.Hi, g.k, g.s, g.p) ||
      g.Wo != conv_out(g.Wi, g.k, g.s, g.p) || g.Ci % 8 || g.Co % 8)
    return set_error(RN_ERR_ARG, "rn_op_conv3d: inconsistent geometry");
  cudaStream_t st = (cudaStream_t)stream;
  const DType dt = dtype == RN_BF16 ? DT_BF16 : DT_F32;
  const bool tc_ok = dt == DT_BF16 && (op == 2 ? tc_wgrad_supported(g) : tc_conv_supported(g, op == 1));
  if ((impl == 2 || impl == 5) && !tc_ok) return set_error(RN_ERR_ARG, "rn_op_conv3d: tcgen05 kernel does not take this conv");
  if (impl == 5 && op == 2) return set_error(RN_ERR_ARG, "rn_op_conv3d: impl 5 is fprop / dgrad only");
  struct PairForce {  // impl 2: single-CTA persistent kernel; 5: on CTA pairs where it applies
    explicit PairForce(int m) { tc_pair_force(m); }
    ~PairForce() { tc_pair_force(-1); }
  } pair_force(impl == 2 ? 0 : impl == 5 ? 1 : -1);
  const bool tc = tc_ok && impl != 1;
  const bool halo_ok = dt == DT_BF16 && op != 2 && halo_conv_supported(g, op == 1);
  if (impl == 3 && !halo_ok) return set_error(RN_ERR_ARG, "rn_op_conv3d: haloed kernel does not take this conv");
  const bool pair_ok = dt == DT_BF16 && op != 2 && pair_conv_supported(g, op == 1);
  if (impl == 4 && !pair_ok) return set_error(RN_ERR_ARG, "rn_op_conv3d: CTA-pair kernel does not take this conv");
  const bool c1_ok = dt == DT_BF16 && op != 2 && conv1x1_supported(g);
  if (impl == 6 && !c1_ok) return set_error(RN_ERR_ARG, "rn_op_conv3d: 1x1x1 streaming kernel does not take this conv");
  if ((impl == 6 || impl == 0) && c1_ok) {
    if (op == 0) {
      conv1x1(g, (const bf16 *)a_dev, (const bf16 *)b_dev, nullptr, (bf16 *)out_dev, st);
    } else {
      void *wd = nullptr;
      CUDA_CHECK(cudaMallocAsync(&wd, (size_t)g.Co * g.Ci * 2, st));
      flip_weights(dt, b_dev, g.Co, g.taps(), g.Ci, wd, st);
      conv1x1(g, (const bf16 *)a_dev, (const bf16 *)wd, nullptr, (bf16 *)out_dev, st);
      CUDA_CHECK(cudaFreeAsync(wd, st));
    }
    return RN_OK;
  }
  if ((impl == 4 || impl == 0) && pair_ok) {
    if (op == 0) {
      conv_pair(g, false, (const bf16 *)a_dev, (const bf16 *)b_dev, nullptr, (bf16 *)out_dev, false, nullptr, nullptr,
                st);
    } else {
      void *wd = nullptr;
      CUDA_CHECK(cudaMallocAsync(&wd, (size_t)g.Co * g.taps() * g.Ci * 2, st));
      flip_weights(dt, b_dev, g.Co, g.taps(), g.Ci, wd, st);
      conv_pair(g, true, (const bf16 *)a_dev, (const bf16 *)wd, nullptr, (bf16 *)out_dev, false, nullptr, nullptr, st);
      CUDA_CHECK(cudaFreeAsync(wd, st));
    }
    return RN_OK;
  }
  if (impl == 3 && halo_ok) {
    if (op == 0) {
      conv_halo(g, false, (const bf16 *)a_dev, (const bf16 *)b_dev, nullptr, (bf16 *)out_dev, false, nullptr, nullptr,
                st);
    } else {
      void *wd = nullptr;
      CUDA_CHECK(cudaMallocAsync(&wd, (size_t)g.Co * g.taps() * g.Ci * 2, st));
      flip_weights(dt, b_dev, g.Co, g.taps(), g.Ci, wd, st);
      conv_halo(g, true, (const bf16 *)a_dev, (const bf16 *)wd, nullptr, (bf16 *)out_dev, false, nullptr, nullptr, st);
      CUDA_CHECK(cudaFreeAsync(wd, st));
    }
    return RN_OK;
  }
  if (op == 0) {
    if (tc) {
      const size_t wsf = tc_conv_ws_floats(g, false);
      float *ws = nullptr;
      if (wsf) CUDA_CHECK(cudaMallocAsync((void **)&ws, sizeof(float) * wsf, st));
      conv_fprop_tc(g, (const bf16 *)a_dev, (const bf16 *)b_dev, nullptr, (bf16 *)out_dev, ws, wsf, st);
      if (ws) CUDA_CHECK(cudaFreeAsync(ws, st));
    }
    else conv_fprop_simt(dt, g, a_dev, b_dev, nullptr, out_dev, st);
  } else if (op == 1) {
    if (tc) {
      void *wd = nullptr;
      const size_t n = (size_t)g.Co * g.taps() * g.Ci;
      CUDA_CHECK(cudaMallocAsync(&wd, n * 2, st));
      flip_weights(dt, b_dev, g.Co, g.taps(), g.Ci, wd, st);
      CUDA_CHECK(cudaMemsetAsync(out_dev, 0, 2 * (size_t)g.in_vox() * g.Ci, st));
      const size_t wsf = tc_conv_ws_floats(g, true);
      float *ws = nullptr;
      if (wsf) CUDA_CHECK(cudaMallocAsync((void **)&ws, sizeof(float) * wsf, st));
      conv_dgrad_tc(g, (const bf16 *)a_dev, (const bf16 *)wd, (bf16 *)out_dev, true, nullptr, nullptr, ws, wsf, st);
      if (ws) CUDA_CHECK(cudaFreeAsync(ws, st));
      CUDA_CHECK(cudaFreeAsync(wd, st));
    } else {
      conv_dgrad_simt(dt, g, a_dev, b_dev, out_dev, false, nullptr, nullptr, st);
    }
  } else {
    float *ws = nullptr;
    const size_t wsf = tc ? tc_wgrad_ws_floats(g) : conv_wgrad_ws_floats(g);
    CUDA_CHECK(cudaMallocAsync((void **)&ws, sizeof(float) * wsf, st));
    CUDA_CHECK(cudaMemsetAsync(out_dev, 0, sizeof(float) * (size_t)g.Co * g.taps() * g.Ci, st));
    if (tc) conv_wgrad_tc(g, (const bf16 *)a_dev, (const bf16 *)b_dev, (float *)out_dev, ws, st);
    else conv_wgrad_simt(dt, false, g, a_dev, b_dev, (float *)out_dev, ws, st);
    CUDA_CHECK(cudaFreeAsync(ws, st));
  }
  return RN_OK;
  GUARD_END
}

void rn_plan_destroy(rn_plan_t plan) {
  if (!plan) return;
  try {
    delete plan->p;
  } catch (...) {
  }
  delete plan;
}

const char *rn_last_error(void) { return rn::g_err.c_str(); }

}  // extern "C"
