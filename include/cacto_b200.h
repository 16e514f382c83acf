/*
 * cacto_b200.h -- C-ABI of the B200-native CACTO-BIC hot path (sm_100a).
 *
 * The reference (`trajrl`, pure Python/NumPy) has no FFI: its operator
 * surface is the Python functions listed against each entry point below.
 * This header is what a binding of that surface links against (ctypes in
 * `paper_2602_19699_b200/_lib.py`; a cgo/JNI/N-API stub would bind the same
 * symbols -- see INTEGRATION.md).
 *
 * Conventions
 *  - Plain pointers and sizes only.  Every `void*` data pointer is a DEVICE
 *    pointer owned by the caller (HBM), except where documented as host.
 *  - `stream` is a cudaStream_t passed as `void*` (NULL = legacy stream).
 *  - Element type of every floating buffer is given by the descriptor's
 *    `dtype` (CACTO_F32 / CACTO_F64); index buffers are int64.
 *  - Return value: CACTO_OK or a negative status; `cacto_last_error()` holds
 *    a message for the calling thread.  Status -> Python exception mapping
 *    mirrors the reference (ValueError for shape / horizon / keep / empty
 *    batch errors, RuntimeError for CUDA failures).
 *  - No hidden allocation on the hot path: scratch space is caller-provided
 *    (`*_workspace_bytes` queries).  Calls are reentrant; launches are async.
 */
#ifndef CACTO_B200_H
#define CACTO_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CACTO_ABI_VERSION 1

#define CACTO_MAX_LAYERS 5   /* affine layers per network (<= 4 hidden)        */
#define CACTO_MAX_IN 32      /* network input width n+1                          */
#define CACTO_MAX_OUT 8      /* network output width (control dimension m)      */
#define CACTO_MAX_HIDDEN 1024 /* padded hidden width (32, 64, or any multiple of 32 up to this) */
#define CACTO_MAX_OBST 4     /* elliptic obstacles of the task cost             */

/* status codes */
#define CACTO_OK 0
#define CACTO_EVALUE (-1)       /* ValueError in the reference                   */
#define CACTO_EUNSUPPORTED (-2) /* shape/system not built into this library       */
#define CACTO_ECUDA (-3)        /* CUDA runtime / launch failure (RuntimeError)   */

enum cacto_dtype { CACTO_F32 = 0, CACTO_F64 = 1 };
enum cacto_activation { CACTO_ACT_ELU = 0, CACTO_ACT_TANH = 1 };                 /* nets.py:49-52   */
enum cacto_head { CACTO_HEAD_LINEAR = 0, CACTO_HEAD_TANH = 1, CACTO_HEAD_STD = 2 }; /* nets.py:144-162 */
enum cacto_system_kind {
  CACTO_SYS_TOY1D = 0,        /* envs/systems.py:14-31        */
  CACTO_SYS_POINTMASS = 1,    /* envs/systems.py:34-65        */
  CACTO_SYS_DUBINS = 2,       /* envs/systems.py:68-105       */
  CACTO_SYS_MANIPULATOR3 = 3, /* envs/manipulator.py:22-152   */
  CACTO_SYS_ALIENGO_LIPM = 4  /* synthetic, oracle/aliengo.py */
};
enum cacto_cost_kind { CACTO_COST_TASK = 0, CACTO_COST_TOY1D = 1, CACTO_COST_LIPM = 2 };
enum cacto_score_mode { CACTO_SCORE_STD = 0, CACTO_SCORE_GAP = 1, CACTO_SCORE_STD_X_GAP = 2 };

/* ---------------------------------------------------------------------------
 * Network descriptor (reference `nets.Mlp`, nets.py:63-103).
 * Parameters live in ONE device buffer in the padded layout:
 *   n_layers >= 2:  W0 [hp][ip] b0 [hp] | (W_i [hp][hp] b_i [hp]) x (n_layers-2)
 *                   | W_last [out][hp] b_last [out]
 *   n_layers == 1:  W0 [out][ip] b0 [out]
 * with ip = cacto_padded_in(in) (8/16/32) and every hidden width padded to hp
 * (32 or 64: fused SIMT kernels, fp32 or fp64; any larger multiple of 32 up to
 * CACTO_MAX_HIDDEN: the layer-wise tcgen05 path, fp32 only, whose workspace-free
 * entry points use a library-owned per-device scratch).  Padding entries are
 * zero and stay zero under the optimizer, so the padded network computes
 * exactly the reference network.
 * ------------------------------------------------------------------------- */
typedef struct cacto_mlp {
  int32_t dtype;
  int32_t n_layers;                     /* affine layers L (1..CACTO_MAX_LAYERS)   */
  int32_t sizes[CACTO_MAX_LAYERS + 1];  /* true widths [in, h1 .. h_{L-1}, out]    */
  int32_t hp;                           /* padded hidden width                      */
  int32_t activation;                   /* cacto_activation                         */
  int32_t head;                         /* cacto_head                               */
  int32_t has_norm;                     /* in_center/in_half valid (nets.py:126-129) */
  double sigma_min;                     /* std head floor                           */
  double in_center[CACTO_MAX_IN];
  double in_half[CACTO_MAX_IN];
  double out_scale[CACTO_MAX_OUT];      /* tanh head scale (u_max)                  */
  void* params;                         /* device, padded layout                    */
} cacto_mlp_t;

/* System description (reference `ModelSpec`, envs/base.py:82-119). */
typedef struct cacto_system {
  int32_t kind;            /* cacto_system_kind */
  int32_t n, m, t_max;
  double dt;
  double u_max[CACTO_MAX_OUT];
  double p[16];            /* manipulator3: l1 l2 l3 m1 m2 m3 (manipulator.py:19-28)
                              aliengo_lipm: omega sx sy delta0                        */
} cacto_system_t;

/* Cost field (reference `CostField` + `TaskCost`, envs/base.py:61-79, costs.py:85-107). */
typedef struct cacto_cost {
  int32_t kind;            /* cacto_cost_kind */
  int32_t n_obstacles;
  double target[2];
  double obs_center[CACTO_MAX_OBST][2];
  double obs_form[CACTO_MAX_OBST][4];   /* E row-major, Ellipse.quadratic_form (base.py:53-58) */
  double w_obstacle, w_reward, reward_radius, w_control, w_distance;
  double extra[8];         /* aliengo_lipm: w_vel w_vbar v_max2 obs_r2 w_wall            */
} cacto_cost_t;

/* Replay rows (reference `SampleBatch` columns, buffer.py:39-55 / ring buffer.py:97-101).
 * If `idx` is non-NULL, sample b reads row idx[b] of the columns (fused gather,
 * buffer.py:136-138); otherwise rows 0..rows-1.  If `cycle` is non-NULL the
 * index list is idx + (*cycle) * idx_stride, read on device at kernel run time,
 * so one captured CUDA graph replays successive minibatches (trainer.py:211-233). */
typedef struct cacto_batch {
  int32_t dtype;
  int32_t n, m, t_max;
  int64_t rows;            /* samples in this call (this rank's slice)                   */
  int64_t denom;           /* loss mean denominator (global batch); 0 -> rows             */
  const int64_t* idx;      /* optional device int64 [rows]                                */
  const void* xa;          /* [*, n+1] */
  const void* u;           /* [*, m]   */
  const void* v_bar;       /* [*]      */
  const void* v_bar_x;     /* [*, n]   */
  const void* xa_plus_k;   /* [*, n+1] */
  const int64_t* cycle;    /* optional device counter selecting the index list      */
  int64_t idx_stride;      /* elements between successive index lists              */
} cacto_batch_t;

/* -- library ---------------------------------------------------------------- */
int cacto_abi_version(void);
const char* cacto_last_error(void);
int32_t cacto_padded_in(int32_t in_dim);
/* elements of the padded parameter buffer for `mlp` (dtype-independent) */
int64_t cacto_mlp_param_count(const cacto_mlp_t* mlp);

/* -- (a3) network forward: nets.mlp_forward, nets.py:165-173 ----------------
 * xa [B, in] (dtype) -> out [B, out] (dtype). */
int cacto_mlp_forward(const cacto_mlp_t* mlp, const void* xa, int64_t B, void* out, void* stream);

/* -- (a10) nets.mlp_input_gradient, nets.py:176-192 (and value_and_state_grad,
 * nets.py:195-206, for a scalar linear head): value [B, out] head outputs and
 * jac [B, out, in], the Jacobian w.r.t. the RAW input (head chain applied,
 * divided by in_half). */
int cacto_mlp_jacobian(const cacto_mlp_t* mlp, const void* xa, int64_t B, void* value, void* jac,
                       void* stream);

/* -- (a1-a5) closed-loop rollout: nets.actor_rollout, nets.py:403-423 -------
 * x0 [N, n] float64 host-API layout (device pointer), start times t0 [N] int32
 * (or NULL -> t0_scalar for all), horizon t_hor >= 0 (<= t_max - t0, else
 * CACTO_EVALUE like nets.py:409-410; t_hor = 0 gives the reference's 1-row
 * trajectory), or CACTO_FULL_HORIZON: every start runs to its own horizon
 * t_max - t0[i] and the output row stride is t_max (rows past a start's
 * horizon are left untouched).  Outputs (dtype, each optional/NULL), with
 * S = t_hor (or t_max for CACTO_FULL_HORIZON):
 *   U [N, S, m], X [N, S+1, n], step_costs [N, S+1], cost [N]
 * Costs need `cost` != NULL (field given); without a field step costs are 0.
 * cost[i] = NumPy pairwise sum of step_costs[i] (Trajectory.cost, ilqr.py:76-78). */
enum { CACTO_FULL_HORIZON = -1 };
int cacto_rollout(const cacto_system_t* sys, const cacto_cost_t* cost, const cacto_mlp_t* actor,
                  const double* x0, const int32_t* t0, int32_t t0_scalar, int64_t N, int32_t t_hor,
                  void* U, void* X, void* step_costs, void* cost_to_go, void* stream);
/* cacto_rollout with flags: CACTO_ROLLOUT_U_TIME_MAJOR writes U as [t_hor, m, N]
 * (coalesced per step), so one cost rollout can also keep every candidate's
 * controls and the kept warm starts are a column take (cacto_take_columns)
 * instead of a second rollout (trainer.py:192-193 re-rolls the same starts). */
enum { CACTO_ROLLOUT_U_TIME_MAJOR = 1,
       /* U as [t_hor, N, m]: a step's controls of a start contiguous (coalesced per
        * step too); the kept warm starts are then a step take (cacto_take_steps) that
        * reads one 32-byte sector per kept start and step */
       CACTO_ROLLOUT_U_STEP_MAJOR = 2 };
int cacto_rollout_ex(const cacto_system_t* sys, const cacto_cost_t* cost, const cacto_mlp_t* actor,
                     const double* x0, const int32_t* t0, int32_t t0_scalar, int64_t N, int32_t t_hor,
                     int32_t flags, void* U, void* X, void* step_costs, void* cost_to_go, void* stream);
/* K1 + K2 in one launch (gap modes): the rollout of every start with the cost,
 * plus the BIC score of the same start from the std net / critic forwards on
 * [x0, t0] (trainer.py:150-151 and the north_star gap score), written once the
 * cost-to-go is known.  fp32 tensor-core path with std/critic of the actor's
 * shape only; otherwise CACTO_EUNSUPPORTED before any launch (callers then use
 * cacto_rollout_ex + cacto_score).  U optional (flags as cacto_rollout_ex). */
int cacto_rollout_score(const cacto_system_t* sys, const cacto_cost_t* cost, const cacto_mlp_t* actor,
                        int32_t mode, const cacto_mlp_t* std_net, const cacto_mlp_t* critic, const double* x0,
                        int32_t t0_scalar, int64_t N, int32_t t_hor, int32_t flags, void* U, void* cost_to_go,
                        void* scores, void* stream);
/* dst[i, r] = src[r, idx[i]] for r < R, i < K: src [R, N] (dtype), dst [K, R] */
int cacto_take_columns(int32_t dtype, const void* src, int64_t R, int64_t N, const int64_t* idx, int64_t K,
                       void* dst, void* stream);
/* dst [K, T, M] (dtype) <- rows idx[k] of a step-major src [T, N, M]: the kept
 * warm starts out of a CACTO_ROLLOUT_U_STEP_MAJOR cost rollout (trainer.py:192-193). */
int cacto_take_steps(int32_t dtype, const void* src, int64_t T, int64_t N, int32_t M, const int64_t* idx, int64_t K,
                     void* dst, void* stream);
/* dst[i, :] = src[idx[i], :], rows of R elements (dtype): the kept warm starts of a
 * start-major [N, T, m] U (trainer.py:192-193), one coalesced row copy each */
int cacto_take_rows(int32_t dtype, const void* src, int64_t R, const int64_t* idx, int64_t K, void* dst,
                    void* stream);

/* -- (a6, a8) BIC scores: std sigma(x0) (trainer.py:150-151), gap
 * |V(x0) - J(x0)| or sigma * gap (north_star).
 * xa [N, n+1] (dtype); rollout_cost [N] (dtype) needed for gap modes. */
int cacto_score(int32_t mode, const cacto_mlp_t* std_net, const cacto_mlp_t* critic, const void* xa,
                const void* rollout_cost, int64_t N, void* scores, void* stream);

/* -- (a6) stable descending top-k: np.argsort(-s, kind="stable")[:keep]
 * (trainer.py:152).  Ties -> lower index, NaN last, -0.0 == +0.0.  `base_index`
 * is added to every emitted index (sharded candidates).  Outputs order [keep]
 * int64 and, optionally, the selected scores [keep] (dtype). */
size_t cacto_select_workspace_bytes(int32_t dtype, int64_t N, int64_t keep);
int cacto_select_topk(int32_t dtype, const void* scores, int64_t N, int64_t keep, int64_t base_index,
                      int64_t* order, void* top_scores, void* workspace, size_t workspace_bytes,
                      void* stream);
/* merge R sorted (score, index) runs of length `keep` each (allgathered shard
 * winners) into the global top-`keep` with the same order semantics.  The
 * index may be the global candidate index or, for contiguous shards in rank
 * order, the position in the concatenated runs (same tie order); index < 0
 * marks a padding row, which sorts after everything (including NaN). */
int cacto_select_merge(int32_t dtype, const void* run_scores, const int64_t* run_index, int32_t R,
                       int64_t keep, int64_t* order, void* top_scores, void* workspace,
                       size_t workspace_bytes, void* stream);

/* -- (a6 over shards) distributed stable top-k: the union of all
 * ranks' contiguous candidate shards selected exactly like trainer.py:152, with
 * only a 2 KB histogram per digit, 16 B of counts per rank and the keep_global
 * winners crossing ranks.  The caller runs the collectives between the phases
 * (paper_2602_19699_b200.parallel.distributed_select):
 *   begin; for pass in 0..(32|64)/8-1: pass -> hist (local, [256] int64)
 *          -> all-reduce SUM -> digit(hist_global) ;
 *   after the last digit counts = {lt_local, eq_local, need} -> all-gather (lt, eq);
 *   host: take_r = clamp(need - sum_{q<r} eq_q, 0, eq_r), c_r = lt_r + take_r,
 *         offset_r = sum_{q<r} c_q ;
 *   local(n_candidates = lt_r + eq_r, n_take = c_r, offset_r): the rank's winners
 *         into elements [offset_r, offset_r + c_r) of a ZEROED keep_global-element
 *         buffer (fp32: one int64 per element; fp64: two) and their local indices
 *         (rank-local order = global order) -> all-reduce SUM of the buffer ->
 *   finish: global order [keep_global] (+ scores) on every rank. */
size_t cacto_dselect_workspace_bytes(int32_t dtype, int64_t N_local, int64_t keep);
int cacto_dselect_begin(int32_t dtype, int64_t N_local, int64_t keep, int64_t keep_global, void* workspace,
                        size_t workspace_bytes, void* stream);
int cacto_dselect_pass(int32_t dtype, const void* scores, int64_t N_local, int64_t keep, int32_t pass,
                       void* workspace, int64_t* hist_out, void* stream);
int cacto_dselect_digit(int32_t dtype, int64_t N_local, int64_t keep, int32_t pass, const int64_t* hist_global,
                        void* workspace, int64_t* counts, void* stream);
int cacto_dselect_local(int32_t dtype, const void* scores, int64_t N_local, int64_t keep, int64_t base_index,
                        int64_t n_candidates, int64_t n_take, int64_t offset, void* workspace, void* global_elems,
                        int64_t* local_sel, void* stream);
int cacto_dselect_finish(int32_t dtype, void* global_elems, int64_t keep_global, int64_t* order, void* top_scores,
                         void* scratch, size_t scratch_bytes, void* stream);

/* -- (a17) replay gather: ReplayBuffer.sample_minibatch, buffer.py:132-138 --
 * out columns get rows idx[b] of the ring columns (batch->idx required). */
int cacto_gather(const cacto_batch_t* ring, void* xa, void* u, void* v_bar, void* v_bar_x,
                 void* xa_plus_k, void* stream);
/* FIFO ring append: ReplayBuffer.push_many, buffer.py:108-130 (rows already
 * trimmed to capacity by the caller); writes src row r to ring row
 * (cursor + r) % capacity. */
int cacto_ring_push(const cacto_batch_t* src, void* ring_xa, void* ring_u, void* ring_v_bar,
                    void* ring_v_bar_x, void* ring_xa_plus_k, int64_t capacity, int64_t cursor,
                    void* stream);

/* -- (8f row 1) replay producer: ilqr.kstep_targets (ilqr.py:358-407, without a
 * critic hook -- the trainer's call, trainer.py:200-201) of a batch of solutions
 * + ReplayBuffer.push_many (buffer.py:108-130), one launch.
 * Solutions are concatenated row-wise (float64, device): solution r owns rows
 * [offsets[r], offsets[r+1]) = its T_r + 1 time steps; X / step_costs / v_bar /
 * v_bar_x hold all T_r + 1 rows (Trajectory.X, .step_costs, SolveResult.V_bar,
 * .V_bar_x, ilqr.py:59-94), U holds T_r rows plus one ignored padding row. */
typedef struct cacto_solutions {
  int32_t n, m;
  int64_t count;            /* R solutions                                   */
  int64_t rows;             /* offsets[R] = sum (T_r + 1)                     */
  const int64_t* offsets;   /* [R + 1]                                       */
  const int32_t* t0;        /* [R]   time index of X[0] (Trajectory.t0)       */
  const double* X;          /* [rows, n] */
  const double* U;          /* [rows, m] */
  const double* step_costs; /* [rows]    */
  const double* v_bar;      /* [rows]    */
  const double* v_bar_x;    /* [rows, n] */
} cacto_solutions_t;
/* Writes concatenated target row i (i >= first; earlier rows are the ones FIFO
 * eviction drops, buffer.py:118-121: first = max(0, rows - capacity)) to ring row
 * (cursor + i - first) % capacity, in the ring's dtype.  K < 1 -> CACTO_EVALUE
 * (ilqr.py:371-372).  *bad (device int32, caller-zeroed) is set to 1 when a
 * v_bar is not finite (the reference's TOSample raises ValueError, buffer.py:33-35). */
int cacto_kstep_push(const cacto_solutions_t* solutions, int32_t K, int32_t ring_dtype, void* ring_xa,
                     void* ring_u, void* ring_v_bar, void* ring_v_bar_x, void* ring_xa_plus_k,
                     int64_t capacity, int64_t cursor, int64_t first, int32_t* bad, void* stream);

/* -- (a9-a13) fused losses ---------------------------------------------------
 * Each writes per-CTA partial sums into `workspace`; `cacto_reduce_grads`
 * (or the fused `cacto_reduce_adam`) folds them.  Gradients are in the padded
 * parameter layout of the differentiated network; the loss is a scalar.
 *   critic: nets.critic_loss, nets.py:233-290 (target may be NULL)
 *   actor:  nets.actor_loss, nets.py:293-334 (rows with t >= t_max skipped;
 *           the loss divides by the live-row count: `live_rows` [1] int64 device
 *           from cacto_count_live, or NULL to count inside the loss launch)
 *   std:    nets.std_critic_loss, nets.py:337-353
 * Wide networks (hp > 64) are differentiated layer by layer on the tensor
 * cores and always report n_partials = 1.  For cacto_actor_loss pass
 * cacto_loss_workspace_bytes(actor) + cacto_loss_workspace_bytes(critic) so the
 * critic's value/state-gradient at x' also runs inside the caller's workspace. */
size_t cacto_loss_workspace_bytes(const cacto_mlp_t* net, int64_t rows);
int cacto_critic_loss(const cacto_mlp_t* critic, const cacto_mlp_t* target, const cacto_batch_t* batch,
                      double k_s, int32_t bootstrap, void* workspace, size_t workspace_bytes,
                      int32_t* n_partials, void* stream);
int cacto_actor_loss(const cacto_mlp_t* actor, const cacto_mlp_t* critic, const cacto_system_t* sys,
                     const cacto_cost_t* cost, const cacto_batch_t* batch, const int64_t* live_rows,
                     void* workspace, size_t workspace_bytes, int32_t* n_partials, void* stream);
int cacto_std_loss(const cacto_mlp_t* std_net, const cacto_mlp_t* critic, const cacto_batch_t* batch,
                   void* workspace, size_t workspace_bytes, int32_t* n_partials, void* stream);
/* std loss (nets.py:337-353) from precomputed errors err = v_bar - V_critic(xa)
 * (cacto_value_errors over the same rows); with batch->cycle the errors of the cycle
 * are err + (*cycle) * batch->idx_stride (laid out like the index lists).  The update
 * loop's std phase uses the final critic for all M cycles (trainer.py:227-233), so the
 * critic forward of every cycle runs as ONE batched launch.  Narrow nets (hp <= 64);
 * wide nets return CACTO_EUNSUPPORTED (use cacto_std_loss). */
int cacto_value_errors(const cacto_mlp_t* critic, const cacto_batch_t* batch, void* err, void* stream);
int cacto_std_loss_err(const cacto_mlp_t* std_net, const void* err, const cacto_batch_t* batch, void* workspace,
                       size_t workspace_bytes, int32_t* n_partials, void* stream);
/* live rows (t < t_max) of a batch -> live_rows[0] (device int64) */
int cacto_count_live(const cacto_batch_t* batch, int64_t* live_rows, void* stream);
/* fold the partials: grad [P] (dtype) and loss [1] (dtype) */
int cacto_reduce_grads(int32_t dtype, const void* workspace, int32_t n_partials, int64_t P, void* grad,
                       void* loss, void* stream);

/* -- (a14) Adam + Polyak: nets.adam_step, nets.py:375-392; nets.polyak 395-398
 * `step` is the step count BEFORE the update (AdamState.step). */
int cacto_adam_step(int32_t dtype, void* params, void* m, void* v, const void* grad, int64_t P,
                    int64_t step, double lr, double beta1, double beta2, double eps, void* stream);
int cacto_polyak(int32_t dtype, void* target, const void* online, int64_t P, double tau, void* stream);
/* fused: fold partials -> grad, Adam update, optional Polyak of `target` toward the
 * updated params (trainer.py:216-220 order), optional grad/loss outputs */
int cacto_reduce_adam(int32_t dtype, const void* workspace, int32_t n_partials, int64_t P, void* params,
                      void* m, void* v, int64_t step, double lr, double beta1, double beta2, double eps,
                      void* target, double tau, void* grad_out, void* loss_out, void* stream);

/* graph-replayable form: the step is *step_base + *counter (both device), the bias
 * corrections come from device tables bc1[t] = 1 - beta1^t, bc2[t] = 1 - beta2^t
 * (computed on the host like the reference), and the loss of this update is
 * written to loss_base[*counter] (trainer.py:226). */
int cacto_reduce_adam_graph(int32_t dtype, const void* workspace, int32_t n_partials, int64_t P, void* params,
                            void* m, void* v, const int64_t* counter, const int64_t* step_base, const double* bc1,
                            const double* bc2, double lr, double beta1, double beta2, double eps, void* target,
                            double tau, void* loss_base, void* stream);
/* the same, also writing the updated parameters into slot (*counter % ring_n) of a
 * [ring_n][ring_ld] buffer: the pipelined M-cycle loop's per-cycle critic copy
 * (cacto_ring_copy save) fused into the update. */
int cacto_reduce_adam_graph_ring(int32_t dtype, const void* workspace, int32_t n_partials, int64_t P, void* params,
                                 void* m, void* v, const int64_t* counter, const int64_t* step_base, const double* bc1,
                                 const double* bc2, double lr, double beta1, double beta2, double eps, void* target,
                                 double tau, void* loss_base, void* ring, int64_t ring_n, int64_t ring_ld,
                                 void* stream);
/* ++(*counter) on device (closes one captured update cycle) */
int cacto_counter_tick(int64_t* counter, void* stream);
/* span[i] = *base + i (i < k), then *base += k: one launch gives the k cycles of a
 * captured chunk their counters (each cycle reads its own span slot) */
int cacto_counter_span(int64_t* base, int64_t* span, int32_t k, void* stream);
/* slot (*counter % ring_n) of a [ring_n][ld] device ring <-> vec [P] (P <= ld; save != 0:
 * vec -> slot).  The pipelined update loop keeps the critic of every cycle this way so the
 * actor chain can run one cycle behind the critic chain (trainer.py:211-225 order). */
int cacto_ring_copy(int32_t dtype, void* ring, const int64_t* counter, int64_t ring_n, int64_t ld, int64_t P,
                    void* vec, int32_t save, void* stream);

/* -- (a7) device PCG64 replay of Generator.uniform starts (envs/__init__.py:119-121)
 * x[i, j] = lo[j] + (hi[j]-lo[j]) * uniform draw (first_row + i)*n + j of the stream
 * with 128-bit state/inc given as (hi, lo) 64-bit halves. */
int cacto_sample_states(uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi, uint64_t inc_lo,
                        int64_t first_row, int64_t N, int32_t n, const double* lo, const double* hi,
                        double* x, void* stream);

/* -- tcgen05 tensor-core GEMM for the wide layers (H >= 128):
 * D[m][n] (+)= alpha * sum_k A(m,k) B(n,k), A(m,k) = A[m*sam + k*sak],
 * B(n,k) = B[n*sbn + k*sbk] (each operand K-major or MN-major, 16-byte aligned
 * rows), D row-major with leading dimension ldd, fp32.  passes = 3: 3xTF32 split
 * (fp32-faithful); passes = 1: plain TF32.  Long-K shapes that cannot fill the GPU
 * use split-K partials in `workspace` (cacto_gemm_workspace_bytes; deterministic). */
size_t cacto_gemm_workspace_bytes(int32_t M, int32_t N, int32_t K);
int cacto_gemm_tf32(int32_t M, int32_t N, int32_t K, const float* A, int64_t sam, int64_t sak, const float* B,
                    int64_t sbn, int64_t sbk, float* D, int64_t ldd, int32_t accumulate, float alpha,
                    int32_t passes, void* workspace, size_t workspace_bytes, void* stream);

/* -- measurement: FFMA/DFMA throughput kernel (roofline denominator of the
 * CUDA-core kernels); executes 2*16*8*iters*blocks*256 FLOPs. */
int cacto_fma_peak(int32_t dtype, int32_t blocks, int32_t iters, void* out, void* stream);
/* fp32 issue forms: 0 = FFMA with constant operands, 1 = 3-register FFMA (the GEMM
 * inner-loop form), 2 = packed 3-register FFMA2 (fma.rn.f32x2); same FLOP count. */
int cacto_fma_peak_mode(int32_t mode, int32_t blocks, int32_t iters, void* out, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* CACTO_B200_H */
