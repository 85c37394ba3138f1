/*
 * rn.h — C ABI of librn.so: one synchronous training step of 3D-ResAttNet under
 * the hybrid (model + data) parallelisation of Akintoye et al., arXiv 2104.05035
 * ("PAPER.md" below, line numbers as P:<line>), built B200-native (sm_100a).
 *
 * Entry points follow the paper's problem statement:
 *   rn_gabra_place  — GABRA, Algorithm 1 over the 0-1 multiple
 *                     knapsack model Eqs. 3-8: partition loads p_i,
 *                     GPU capacities d_j -> placement Z*, profit f(Z*).
 *   rn_net_units    — layer costing + network partitioning (§3.1.1 P:154-156,
 *                     conv complexity P:366): unit loads -> partitions p_1..p_n.
 *   rn_plan         — per-rank program for a placement: partitions on GPUs,
 *                     activation a^t sent to partition i+1 / gradient g^t sent to
 *                     partition i-1, data-parallel replicas (§3.2).
 *   rn_forward / rn_backward / rn_step
 *                   — one synchronous step: forward + cross-entropy loss,
 *                     backward by the chain rule, gradient averaging over
 *                     replicas by ring all-reduce (Eqs. 9-11),
 *                     SGD update w <- w - gamma*g.
 *
 * Conventions (all calls):
 *  - Every call returns rn_status; it never aborts the process.  On error
 *    rn_last_error() returns a thread-local message describing the failure.
 *  - Host pointers (suffix _host / plain arrays) are read or written
 *    synchronously before the call returns.  Device pointers (suffix _dev) are
 *    used stream-ordered on the plan's CUDA stream: the caller keeps them alive
 *    until that stream's work completes.
 *  - Ownership: the caller owns every buffer it passes, including the device
 *    workspace bound with rn_plan_bind (allocated by the caller, e.g. torch);
 *    the library owns the plan, its CUDA graphs, events and NCCL communicators,
 *    released by rn_plan_destroy.
 *  - rn_forward/rn_backward/rn_step are collective over all ranks of the plan
 *    when world > 1: every rank calls them in the same order with the same genes.
 */
#ifndef RN_H
#define RN_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  RN_OK = 0,
  RN_ERR_ARG = 1,         /* bad argument (null pointer, size mismatch, out of range)       */
  RN_ERR_SCHEMA = 2,      /* invalid network description / dims ("schema error")  */
  RN_ERR_INFEASIBLE = 3,  /* no capacity-respecting placement (Eq. 6) found    */
  RN_ERR_NUMERIC = 4,     /* non-finite loss                                   */
  RN_ERR_CUDA = 5,        /* a CUDA runtime/driver call failed (message has the CUDA error)   */
  RN_ERR_NCCL = 6,        /* an NCCL call failed or libnccl could not be loaded               */
  RN_ERR_STATE = 7,       /* call out of order (e.g. rn_forward before rn_plan_bind)          */
  RN_ERR_SIZE = 8         /* buffer too small / instance too large                            */
} rn_status;

/* Arithmetic type of the activation path (reading X19 in DESIGN.md):
 *  RN_F32  — fp32 storage and fp32 SIMT arithmetic everywhere (no TF32); parity 1e-4.
 *  RN_BF16 — bf16 activations and conv operands, fp32 accumulation (tcgen05/TMEM),
 *            fp32 BN statistics, master weights, gradients, all-reduce; parity 2e-2. */
enum { RN_F32 = 0, RN_BF16 = 1 };

/* ------------------------------------------------------------------------- */
/* GABRA placement (§3.1.2).                                                  */
/* ------------------------------------------------------------------------- */

/* GA parameters.  Only p_cross = 0.8 comes from the paper; the rest are
 * SPEC S:119 defaults and the bounded-retry/early-stop readings G15/G18/G19. */
typedef struct {
  int32_t pop_size;          /* population P (default 50; G8)                        */
  int32_t t_max;             /* generations (default 500)                      */
  double p_cross;            /* crossover probability (0.8)                    */
  double p_mut;              /* inversion-mutation probability (0.1; G12)             */
  uint64_t seed;             /* xoshiro256** seed via splitmix64 (G20)                */
  int32_t dup_retries;       /* bounded "ignore W and go to" retries (20; G15)        */
  int32_t init_attempts;     /* random draws per initial chromosome (64; G19)         */
  int32_t require_all_used;  /* 1: "each GPU runs at least one partition" (G7) */
  int32_t early_stop_at_ub;  /* 1: stop when f(Z*) == sum_i max_j c_ij (G18)   */
  int32_t objective;         /* 0: Eq. 3 profit sum_i p_i/d_{g_i} (the paper, default);
                              * 1: bottleneck f = lb / max_j(L_j/d_j), lb = max(sum p/sum d,
                              *    max p/max d) — SURVEY §8(f) f2, not in the paper: the GA
                              *    then minimises the slowest GPU's normalised load (the
                              *    pipeline step time), which Eq. 3 cannot see on identical
                              *    GPUs (its value is the same for every feasible placement);
                              *    early stop at f = 1.  profit_out reports f.               */
} rn_ga_params;

/* Fill *gp with the defaults above (seed 7). */
void rn_ga_default(rn_ga_params *gp);

/* rn_gabra_place — Algorithm 1 as pinned in DESIGN.md "GABRA".
 *  n, loads[n]   : partition loads p_i >= 0 (int64 MACs per sample; reading G3)
 *  m, caps[m]    : GPU capacities d_j > 0 (same unit)
 *  gp            : GA parameters (NULL = rn_ga_default)
 *  genes_out[n]  : 0-based GPU index of each partition in Z*            (written)
 *  profit_out    : f(Z*) = sum_i p_i / d_{genes_i}, left-to-right double (written; may be NULL)
 *  gpu_load_out[m]: per-GPU load sum_{i: genes_i=j} p_i                  (written; may be NULL)
 * Errors: RN_ERR_ARG (n<1, m<1, pop_size<2, null loads/caps/genes_out, caps<=0,
 * loads<0), RN_ERR_INFEASIBLE (no feasible initial chromosome within
 * init_attempts draws + repair).  Deterministic: bit-identical to the oracle. */
rn_status rn_gabra_place(int32_t n, const int64_t *loads, int32_t m, const int64_t *caps,
                         const rn_ga_params *gp, int32_t *genes_out, double *profit_out,
                         int64_t *gpu_load_out);

/* rn_gabra_place_slack — the placement policy the hybrid runs use (reading G4b,
 * DESIGN.md): identical capacities d_j = ceil(s * max(max_i p_i, ceil(sum_i p_i / m)))
 * for the smallest slack s in 1.1, 1.2, ..., 2.0 (k/10) for which rn_gabra_place
 * finds a capacity-respecting placement (P:171-216 give no capacities for
 * identical GPUs; a chain of coarse partitions, e.g. r18 on 4 GPUs, cannot be
 * packed at 10 % slack).  Outputs as rn_gabra_place, plus caps_out[m] (may be
 * NULL) and slack_out (may be NULL).  Bit-identical to oracle/gabra.py
 * place_with_slack.  Errors: RN_ERR_ARG, RN_ERR_INFEASIBLE (none up to 2.0). */
rn_status rn_gabra_place_slack(int32_t n, const int64_t *loads, int32_t m, const rn_ga_params *gp,
                               int32_t *genes_out, double *profit_out, int64_t *gpu_load_out, int64_t *caps_out,
                               double *slack_out);

/* ------------------------------------------------------------------------- */
/* Placement quality on real hardware.                      */
/* ------------------------------------------------------------------------- */

/* Step-time model of the hybrid schedule (reading F2, ring
 * all-reduce P:284 / Fig. 3).  Per micro-batch, stage s computes
 * C_s = sum of part_time[i] over its partitions and pays 2 (alpha + cut/beta) for
 * every chain cut i|i+1 that crosses stages (activation forward, gradient back,
 * P:156), charged to both stages: T_s = C_s + P_s.  Pipeline: schedule 0
 * (synchronous, M_b micro-batches) (M_b + S - 1) max T_s; schedule 1 (delayed
 * gradients, f1) M_b max T_s.  All-reduce: max over stages of the ring time
 * 2 (R-1) (g_s/R)/beta + 2 (R-1) alpha.  Step: pipeline + all-reduce, or their max
 * when overlap != 0.  part_time: seconds (measured on the B200 with rn_query
 * "unit_ms_fwd_<u>" + "unit_ms_bwd_<u>"); cut_bytes[n-1], param_bytes[n]: bytes. */
typedef struct {
  int32_t n, n_stages, replicas, micro_batches, schedule, overlap;
  double alpha, beta;        /* s per message, bytes per second */
  const double *part_time;   /* [n] */
  const double *cut_bytes;   /* [n-1] */
  const double *param_bytes; /* [n] */
  const int32_t *genes;      /* [n] partition -> stage */
} rn_sim_desc;
/* stage_s may be NULL ([n_stages]).  Bit-identical to oracle/sim.py step_time.
 * Errors: RN_ERR_ARG (null pointers, sizes < 1, gene out of range, beta <= 0). */
rn_status rn_simulate_step(const rn_sim_desc *d, double *step_s, double *pipeline_s, double *allreduce_s,
                           double *stage_s);

/* rn_contiguous_split — the contiguity option of f2: partitions split into S
 * contiguous stages in chain order (every stage non-empty) minimising the largest
 * stage load (dynamic programme; among optimal splits the last stage is the
 * shortest, recursively).  genes_out[n] in 0..S-1 non-decreasing; max_load_out may
 * be NULL.  The placement rn_plan_delayed needs.  Identical to oracle/sim.py.
 * Errors: RN_ERR_ARG (n < S, S < 1, null / negative loads). */
rn_status rn_contiguous_split(int32_t n, const int64_t *loads, int32_t n_stages, int32_t *genes_out,
                              int64_t *max_load_out);

/* ------------------------------------------------------------------------- */
/* Network description, costing and partitioning (§3.1.1).            */
/* ------------------------------------------------------------------------- */

typedef struct {
  int32_t depth;          /* 0 = tiny (1 block + 1 attention module), 18, 34 (Table 2) */
  int32_t base_width;     /* channels of the stem / stage 1 (8 tiny, 64 r18/r34; reading X2) */
  int32_t in_d, in_h, in_w;/* input volume (91x109x91 MNI grid; reading X1); 1 input channel  */
  int32_t n_classes;      /* must be 2 (binary tasks)                                  */
  double alpha;           /* heavy-unit threshold alpha * mean (reading G1; default 1.0)      */
  int64_t max_merge_load; /* cap on merged light partitions (0 = none)                        */
} rn_net_desc;

#define RN_MAX_UNITS 64

/* rn_net_units — unit costs (a1) and contiguous partitions (a2).
 *  n_units          : number of top-level units (stem, residual blocks, attention modules, head)
 *  unit_loads[64]   : per-sample MACs per unit (conv: Co*Ci*T*H*W*k^3)
 *  n_parts          : number of partitions n
 *  part_first_unit[65]: partition i covers units [first[i], first[i+1])
 *  part_loads[64]   : p_i
 * Any output pointer may be NULL.  Errors: RN_ERR_SCHEMA. */
rn_status rn_net_units(const rn_net_desc *net, int32_t *n_units, int64_t *unit_loads,
                       int32_t *n_parts, int32_t *part_first_unit, int64_t *part_loads);

/* Parameter layout in the canonical order used by rn_set/get_params/grads:
 * units in forward order; conv W[Cout][Cin][kd][kh][kw]; BN gamma, beta; mask
 * conv2 bias; FC W[2][C], b[2].
 *  rn_net_param_count: total scalars and number of tensors.
 *  rn_net_param_info : tensor idx -> ndim, shape[5], kind (0 conv,1 bn_gamma,
 *                      2 bn_beta, 3 fc_w, 4 bias), unit index, name (NUL-terminated). */
rn_status rn_net_param_count(const rn_net_desc *net, int64_t *n_params, int32_t *n_tensors,
                             int32_t *n_bn_channels);
rn_status rn_net_param_info(const rn_net_desc *net, int32_t idx, int32_t *ndim, int64_t *shape5,
                            int32_t *kind, int32_t *unit, char *name, int32_t name_cap);

/* ------------------------------------------------------------------------- */
/* Training step.                                                              */
/* ------------------------------------------------------------------------- */

typedef struct {
  int32_t rank, world;      /* this process / all processes (one per GPU)                   */
  int32_t n_stages;         /* GPUs per pipeline group S (1 = pure data parallel)           */
  const int32_t *genes;     /* [n_parts] partition -> stage index in [0, S) (rn_gabra_place);
                               NULL allowed when n_stages == 1                               */
  int32_t micro_batches;    /* M_b micro-batches per replica step (reading X18; >= 1)       */
  uint8_t nccl_id[128];     /* ncclUniqueId from rn_nccl_unique_id on rank 0, broadcast by
                               the caller; ignored when world == 1.  An id whose first 8
                               bytes are "RNLOCAL" + NUL selects the in-process transport
                               instead: the ranks are plans of THIS process (one host thread
                               each, any device), exchanging by device-to-device copies
                               (send/recv), rank-order sums (all-reduce) and copies
                               (broadcast) -- the multi-rank executor's CUDA path tested on
                               one GPU; CUDA graphs are off on that transport.           */
} rn_dist_desc;

typedef struct rn_plan_s *rn_plan_t;

/* rn_nccl_unique_id — ncclGetUniqueId (libnccl.so.2 loaded at run time). */
rn_status rn_nccl_unique_id(uint8_t out[128]);

/* rn_plan — build the per-rank program.  Replica r = rank / S owns samples
 * [r*b, (r+1)*b) of the global batch (P:366 equal sharding), stage s = rank % S
 * runs the partitions whose gene == s.  local_batch b must be divisible by
 * micro_batches.  cuda_stream: a cudaStream_t (NULL = legacy default stream).
 *  *workspace_bytes : device bytes the caller must bind with rn_plan_bind.
 * Errors: RN_ERR_ARG, RN_ERR_SCHEMA, RN_ERR_NCCL (communicator init). */
rn_status rn_plan(const rn_net_desc *net, const rn_dist_desc *dist, int32_t local_batch,
                  int32_t dtype, void *cuda_stream, rn_plan_t *out, size_t *workspace_bytes);

/* rn_plan_delayed — rn_plan for the delayed-gradient pipeline (
 * P:156 "all partitions are computed simultaneously", Eqs. 1-2; reading
 * F1 in DESIGN.md): the genes must place the partitions on contiguous stages in
 * chain order (non-decreasing genes); micro_batches must be 1.  Every rank keeps
 * S slots of saved forward state and of the weights those forwards used (the
 * Jacobian of Eq. 1 is taken at the forward's weights).  Drive it with
 * rn_delayed_step only (rn_forward / rn_backward / rn_step are not used).
 * Errors: as rn_plan, plus RN_ERR_ARG for non-contiguous genes or M_b != 1. */
rn_status rn_plan_delayed(const rn_net_desc *net, const rn_dist_desc *dist, int32_t local_batch, int32_t dtype,
                          void *cuda_stream, rn_plan_t *out, size_t *workspace_bytes);

/* rn_delayed_step — iteration t of the delayed-gradient pipeline on this rank
 * (stage s, delay d = S-1-s): forward of batch t (x_dev on stage 0, y_dev on the
 * last stage; both may be NULL elsewhere) with the current weights; backward of
 * batch t-d (its output gradient came from stage s+1 in iteration t-1; the last
 * stage's is the batch-t loss gradient) through the saved state and the weights
 * of that forward; SGD w <- w - lr * g on the current weights (all-reduced over
 * replicas when world > S).  Exchanges are grouped (ncclGroupStart/End) pairwise
 * with the neighbour stages, so they cannot deadlock.  loss_host (may be NULL):
 * the batch-t loss, broadcast from the last stage.  Collective over all ranks.
 * S = 1 is plain SGD.  Errors: RN_ERR_STATE (not a delayed plan, no parameters),
 * RN_ERR_NUMERIC (non-finite loss), RN_ERR_CUDA / RN_ERR_NCCL. */
rn_status rn_delayed_step(rn_plan_t plan, const void *x_dev, const int32_t *y_dev, float lr, float *loss_host);

/* rn_plan_describe — the schedule rn_plan builds for this rank, computed on the
 * host only (no GPU, no communicators): which units run here and, in forward
 * order, the partition-boundary exchanges of P:156.
 *  local_units[RN_MAX_UNITS] : 1 if the unit runs on this rank's stage (may be NULL)
 *  n_xfer, xfer[4 * cap]     : {unit, peer stage, dir, bytes}; dir 0 = receive the
 *                              input of `unit` (activation a^t of partition i-1),
 *                              dir 1 = send the output of `unit`; backward does the
 *                              mirror transfers (gradients) in reverse order
 *  n_ranges, ranges[2 * cap] : canonical parameter ranges [begin, end) this rank
 *                              all-reduces over its stage's data-parallel group
 * Errors: RN_ERR_ARG, RN_ERR_SCHEMA, RN_ERR_SIZE (cap too small). */
rn_status rn_plan_describe(const rn_net_desc *net, const rn_dist_desc *dist, int32_t local_batch, int32_t dtype,
                           int32_t *local_units, int32_t cap, int32_t *n_xfer, int64_t *xfer, int32_t *n_ranges,
                           int64_t *ranges);

/* rn_plan_bind — give the plan its device workspace (>= *workspace_bytes,
 * 256-byte aligned, caller-owned, e.g. a torch uint8 tensor).  Must precede
 * every compute call.  Errors: RN_ERR_SIZE, RN_ERR_ARG. */
rn_status rn_plan_bind(rn_plan_t plan, void *dev_workspace, size_t bytes);

/* Parameters in canonical order (float32 host arrays of n_params scalars).
 * rn_set_params also resets BN running statistics (mean 0, var 1).
 * rn_get_grads returns the gradient of the last rn_backward (after rn_step:
 * the replica-averaged gradient G of Eq. 11); entries of partitions not placed on
 * this rank are 0.  Errors: RN_ERR_SIZE (count != n_params), RN_ERR_STATE. */
rn_status rn_set_params(rn_plan_t plan, const float *host, int64_t count);
rn_status rn_get_params(rn_plan_t plan, float *host, int64_t count);
rn_status rn_get_grads(rn_plan_t plan, float *host, int64_t count);
/* BN running statistics, BN layers in canonical order, channels concatenated
 * (count = n_bn_channels from rn_net_param_count). */
rn_status rn_get_bn_running(rn_plan_t plan, float *mean_host, float *var_host, int64_t count);

/* rn_get_activation — copy the output of top-level unit `unit` for micro-batch
 * `micro_batch` of the last rn_forward to host as float32 NDHWC
 * [mb][D][H][W][C] (count must equal that size; the head's output is the
 * logits-free GAP vector [mb][C]).  Only for units placed on this rank.
 * Errors: RN_ERR_ARG (unit not local / out of range), RN_ERR_SIZE. */
rn_status rn_get_activation(rn_plan_t plan, int32_t unit, int32_t micro_batch, float *host, int64_t count);

/* rn_get_unit_grad — copy dl/d(output of top-level unit `unit`), the gradient the
 * chain rule hands to that unit's backward, of the LAST micro-batch of the
 * last rn_backward, to host as float32 NDHWC [mb][D][H][W][C] (the same shape as
 * rn_get_activation).  Not defined for the head (its incoming gradient is dz of
 * the loss).  Used for teacher-forced per-unit parity: unit u's backward maps
 * rn_get_unit_grad(u) to rn_get_unit_grad(u-1).  Only for units placed on this rank.
 * Errors: RN_ERR_ARG (head / not local / out of range), RN_ERR_SIZE,
 * RN_ERR_STATE (no rn_backward yet). */
rn_status rn_get_unit_grad(rn_plan_t plan, int32_t unit, float *host, int64_t count);

/* rn_get_saved — copy one tensor the step keeps (forward tensors saved for the
 * backward, per micro-batch) or leaves behind (backward temporaries and BN
 * statistics: the LAST micro-batch's) of top-level unit `unit` to host as float32
 * (bf16 / uint8 values converted exactly).  Test/diagnostic access for op-level
 * parity; names (NDHWC activation layouts [mb][D][H][W][C] unless stated):
 *   stem : "h" conv output (pre-BN, conv dims), "am" max-pool argmax 0..26 (pooled
 *          dims), "d1" pool adjoint x ReLU mask (dense stem backward only: the bf16 pooled
 *          stem runs at the pooled resolution, reading X23c, and has no d1), "bn.stats"
 *   block: "h1" "a1" "h2" ["hp"] "out" (forward), "dh2" "da1" "dh1" ["dhp"]
 *          (backward), "bn1.stats" "bn2.stats" ["projbn.stats"]
 *   att  : "trunk.<block name>", "mask.<block name>", "u0" "am" (mask-branch
 *          max-pool), "up" "mh" "r" "m" "mbn.stats", "dT" "dm" "dr" "dmh" "dup" "dum" "du0"
 *   head : "dz" [mb][2] fp32 (dl/dlogits, scaled by 1/(batch * replicas))
 * "*.stats" = [4][C] fp32: batch mean, 1/sqrt(var + eps), scale = gamma*invstd,
 * shift = beta - mean*scale.  count must equal the tensor's size.
 * Errors: RN_ERR_ARG (bad unit / micro-batch / unknown name), RN_ERR_SIZE. */
rn_status rn_get_saved(rn_plan_t plan, int32_t unit, const char *name, int32_t micro_batch, float *host,
                       int64_t count);

/* rn_gradcam — Grad-CAM of class `cls` (0/1) for the batch of the last rn_forward
 * ("explainable block"), at the last convolutional
 * layer: the head is GAP + FC, so dy_c/dA_k = W[c,k]/V at every voxel and
 * alpha_k = W[c,k]/V; map = trilinear(ReLU(sum_k alpha_k A_k)) to the input grid
 * (align_corners = False, reading X11).
 *  map_dev : float32 [b][D][H][W] on the device (the input volume grid), written on the
 *            plan's stream (stream-ordered; no synchronisation)
 *  count   : must equal b * D * H * W
 * Errors: RN_ERR_STATE (no forward yet), RN_ERR_SIZE (count), RN_ERR_ARG (cls, null map,
 * head / last conv unit not on this rank). */
rn_status rn_gradcam(rn_plan_t plan, int32_t cls, float *map_dev, int64_t count);

/* rn_forward — forward pass of this replica's local batch.
 *  x_dev : float32 [b][D][H][W] input volumes (device), y_dev: int32 [b] labels in {0,1}
 *          (only read on the stages that need them: stage of the first / last partition)
 *  loss_host: if non-NULL, synchronises the stream and writes the replica's mean
 *          cross-entropy (mean over its micro-batches, P:486 / Eq. 9).  Ranks that
 *          do not hold the head receive it from the head stage.
 * Micro-batches run forward in order (GPipe-style; backward in rn_backward).
 * Errors: RN_ERR_STATE (unbound), RN_ERR_CUDA, RN_ERR_NCCL, RN_ERR_NUMERIC (non-finite loss). */
rn_status rn_forward(rn_plan_t plan, const void *x_dev, const int32_t *y_dev, float *loss_host);

/* rn_backward — backward pass of every micro-batch; writes this rank's
 * gradients (already scaled by 1/(m*M_b) so that the replica sum is Eq. 11's G). */
rn_status rn_backward(rn_plan_t plan);

/* rn_step — all-reduce (sum) of the local partitions' gradients over the
 * stage's data-parallel group (ring/NVLS all-reduce), then SGD
 * w <- w - lr*G on fp32 master weights and refresh of the bf16 copies. */
rn_status rn_step(rn_plan_t plan, float lr);

/* rn_train_step_host — end-to-end convenience: copies x_host/y_host (pageable or
 * pinned host memory) to the device, runs forward, backward and step, and reads
 * the loss back.  Same semantics as the three calls above. */
rn_status rn_train_step_host(rn_plan_t plan, const float *x_host, const int32_t *y_host, float lr,
                             float *loss_host);

/* rn_train_step — one training step from DEVICE inputs (x_dev, y_dev as in
 * rn_forward): forward, backward and SGD with the update rule of rn_step
 * (w <- w - lr*G).  The result equals rn_forward + rn_backward + rn_step
 * bit for bit; the call differs only in scheduling: when the plan has one stage,
 * one micro-batch and no replicas (and option "early_sgd" is not 0), each unit's
 * update is issued on the weight-gradient stream as soon as that unit's backward
 * is done and overlaps the backward of the units before it (the update of unit u
 * reads only u's gradient; no later part of the backward reads u's weights).
 * Gradients stay readable afterwards (rn_get_grads).  loss_host: optional, as in
 * rn_forward (a read-back = a synchronisation).  Errors as rn_forward / rn_step. */
rn_status rn_train_step(rn_plan_t plan, const void *x_dev, const int32_t *y_dev, float lr, float *loss_host);

/* rn_train_steps_host — n_steps training steps from host inputs (x_host[i],
 * y_host[i]: step i's batch, same layout as rn_forward's; pinned memory lets
 * the copies run asynchronously).  The host->device copy of step i+1 runs on a
 * plan-owned side stream while step i computes (double-buffered staging in the
 * workspace); losses_host[i] (optional, n_steps floats) receives step i's loss.
 * Returns when all steps are complete.  Semantics per step = rn_train_step_host.
 * Errors: RN_ERR_ARG (null inputs), RN_ERR_STATE, RN_ERR_NUMERIC (a non-finite
 * loss), RN_ERR_CUDA / RN_ERR_NCCL. */
rn_status rn_train_steps_host(rn_plan_t plan, const float *const *x_host, const int32_t *const *y_host,
                              int32_t n_steps, float lr, float *losses_host);

/* Introspection for tests/bench: number of GPU kernels launched by this plan so
 * far, and the plan's conv-kernel time accounting. */
int64_t rn_kernel_launches(rn_plan_t plan);

/* rn_set_option — runtime switches:
 *  "graphs"        : 1 capture forward/backward/step in CUDA graphs (default 1)
 *  "tc_conv"       : 1 use tcgen05 conv kernels in RN_BF16 (default 1)
 *  "time_kernels"  : 1 record CUDA events around the dominant conv launches
 *  "halo_conv", "pair_conv", "fused_stats", "wgrad_stream" : kernel-variant switches (default 1)
 *  "merge_proj"    : 1 stage-entry projection dgrad merged into the stride-2 dgrad launch (default 1)
 *  "c1x1"          : 1 streaming warp-tensor-core kernel for 64->64 1x1x1 convs (default 1)
 *  "att_branch"    : 1 attention soft-mask branch on its own stream, concurrent with the trunk (default 1)
 *  "res_prestore"  : 1 identity-skip blocks: dy' pre-stored in dx, conv1's dgrad accumulates (default 1)
 *  "wgrad_overwrite": 1 tensor-core weight gradients store (not add) on a backward's first
 *                    micro-batch; the backward zeroes only the other gradient ranges (default 1)
 *  "early_sgd"     : 1 rn_train_step issues each unit's SGD right after its backward (default 1)
 *  "recompute_mask": 1 dgrad-epilogue BN sums recompute the consumer's ReLU mask from h (default 1)
 *  "pair_bwd_stats": 1 fuse the backward BN sums into the CTA-pair dgrad epilogue (default 0: standalone pass)
 *  "up_bwd_sep"    : 1 separable trilinear adjoint (default 1)
 *  "overlap_allreduce": 1 reduce the gradient over the stage's data-parallel group in
 *                    ~8 MB buckets during rn_backward, on a comm stream, as soon as a
 *                    bucket's units are done (default 1 when replicas > 1; rn_get_grads
 *                    after rn_backward then returns the replica average G of Eq. 11);
 *                    0: one all-reduce per range inside rn_step
 *  "async_allreduce": 1 ASGD with ring all-reduce (reading F4): step t's
 *                    gradient is reduced on a comm stream during step t+1 and applied by
 *                    step t+1's rn_step (w <- w - lr G^{t-1}; the first rn_step applies
 *                    nothing); double-buffered gradient arrays, CUDA graphs off (default 0)
 * Unknown keys: RN_ERR_ARG.  Every switch changes kernels only, not the result beyond fp32 rounding. */
rn_status rn_set_option(rn_plan_t plan, const char *key, int64_t value);

/* rn_query — named float64 statistics (e.g. "conv_ms", "conv_flops") collected
 * when time_kernels is on; reset by rn_set_option("time_kernels", 1).
 * "conv_ms|conv_flops|conv_launches[_fprop|_dgrad|_wgrad|_pair|_tcconv|_tcwgrad|_stem]",
 * "elt_ms|elt_bytes|elt_launches[_<family>]" (HBM-bound launches: bn_apply,
 * bn_bwd_apply, bn_partials, stem_pool_fwd, stem_pool_bwd, maxpool_fwd, maxpool_bwd,
 * upsample_fwd, upsample_bwd, att_fwd, att_bwd, sgd; bytes = algorithmic). */
rn_status rn_query(rn_plan_t plan, const char *key, double *value);

/* rn_op_conv3d — ONE convolution of the step as a stand-alone launch, for the
 * kernel-level parity tests and micro-benchmarks (same kernels the plan uses).
 *  op 0 fprop : out[N][Do][Ho][Wo][Co] = sum_{tap,ci} a[N][Di][Hi][Wi][Ci] * b[Co][tap][Ci]
 *  op 1 dgrad : out[N][Di][Hi][Wi][Ci] = sum_{tap,co} a[N][Do][Ho][Wo][Co] * b[Co][tap][Ci]
 *  op 2 wgrad : out[Co][tap][Ci] (float32) = sum_{n,vo} b[..vo..][Co] * a[..vi(vo,tap)..][Ci]
 *               (a = x, b = dy)
 *  geom[12] = {N, Di, Hi, Wi, Ci, Do, Ho, Wo, Co, k, s, p}; element type of a, b
 *  (and out for ops 0/1) is dtype; impl 0 = auto (the kernel the plan would
 *  use), 1 = SIMT, 2 = generic tcgen05 implicit GEMM (single CTAs), 3 = haloed
 *  single-CTA tcgen05 kernel, 4 = CTA-pair (cta_group::2) kernel with resident
 *  weights, 5 = the generic implicit GEMM on CTA pairs (M = 256 MMAs, half of B
 *  per CTA) for every launch with 128- / 256-wide N tiles, split-K included (the
 *  plan uses pairs for the launches without split-K), 6 = the streaming
 *  warp-tensor-core kernel for 64 -> 64 1x1x1 stride-1 convs over >= 16384
 *  voxels (k_conv1x1.cu) — 3 and 4 only for 64 -> 64 stride-1 3x3x3 ops 0/1,
 *  5 and 6 for ops 0/1 (RN_ERR_ARG when an explicitly requested kernel does not
 *  take the conv).  Device pointers,
 *  stream-ordered on `stream`; scratch is allocated internally.
 * Errors: RN_ERR_ARG, RN_ERR_CUDA. */
rn_status rn_op_conv3d(int32_t dtype, int32_t op, const int32_t *geom, const void *a_dev, const void *b_dev,
                       void *out_dev, int32_t impl, void *stream);

void rn_plan_destroy(rn_plan_t plan);
const char *rn_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* RN_H */
