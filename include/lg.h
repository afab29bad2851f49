/*
 * lg.h -- C ABI of libleggedrl.so: the data-parallel hot path of Rudin et al., "Learning to Walk in
 * Minutes Using Massively Parallel Deep Reinforcement Learning" (arXiv 2109.11978) on B200 (sm_100a).
 *
 * One PPO iteration (§2.2; Table 3; Alg. 1) is
 *     for t in 0..T-1: policy_act(ctx, t); env_step_obs_reward(ctx, t, ...);
 *     storage_compute_gae(ctx, ...); ppo_update(ctx, ...);
 * Every operation is defined in DESIGN.md §3 (the frozen definitions the independent CPU oracle in
 * oracle/ is also written from).
 *
 * Conventions
 *  - Pointers are CUDA device pointers unless the parameter name ends in _h (host).
 *  - Ownership: the caller allocates every device buffer (sizes from lg_required_sizes) and keeps it
 *    alive for the lifetime of the context; the context only borrows them. Nothing is freed by the
 *    library except its own host-side context object.
 *  - Every call validates its arguments synchronously and then only ENQUEUES work on the context's
 *    stream: no device allocation, no host synchronisation, no host read of device data. A whole
 *    iteration can therefore be captured into one CUDA graph and replayed; all per-iteration
 *    counters (env step counter, iteration, learning rate, Adam step) live in device memory.
 *  - Errors: functions return lg_status. The first failure of a context is sticky: later calls
 *    return the same status without doing work; lg_last_error() gives a one-line message.
 *  - A context is bound to one device and one stream and is not thread-safe.
 *  - There is no CPU fallback: a missing or non-sm_100a device makes lg_create fail with
 *    LG_ERR_UNSUPPORTED.
 */
#ifndef LG_H_
#define LG_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct lg_ctx lg_ctx;

typedef enum {
  LG_OK = 0,
  LG_ERR_INVALID_ARG = 1, /* null/zero/negative where not allowed, B not divisible by minibatches */
  LG_ERR_RANGE = 2,       /* a value outside its documented range (levels, γ, λ, ...) */
  LG_ERR_SHAPE = 3,       /* inconsistent sizes (world dims, widths not multiples of 64, ...) */
  LG_ERR_STATE = 4,       /* call out of order (e.g. policy_act(t) before env_reset) */
  LG_ERR_CUDA = 5,        /* a CUDA launch/runtime failure (sticky) */
  LG_ERR_NCCL = 6,        /* an NCCL failure (sticky) */
  LG_ERR_UNSUPPORTED = 7  /* no sm_100 device, or a feature not built */
} lg_status;

/* env feature flags (Table 4) */
#define LG_F_CURRICULUM 1u /* game-inspired curriculum at episode end */
#define LG_F_NOISE 2u      /* observation noise (Table 4) */
#define LG_F_PUSH 4u       /* pushes every 10 s */
#define LG_F_BOOTSTRAP 8u  /* time-out bootstrapping */
/* evaluation: policy_act takes the mean action a = mu (no Gaussian draw; logp is evaluated at a = mu) --
 * the deterministic policy of the traversability tests ("robustness and traversability tests";
 * SURVEY §8(f) NEXT-4) */
#define LG_F_DETERMINISTIC 32u
/* implementation switch (diagnostics/parity): policy_act uses the per-layer GEMM + head kernels instead of the
 * fused rollout-policy kernel (same results bit for bit; only the 512-256-128 MLP has a fused kernel) */
#define LG_F_UNFUSED_POLICY 256u
/* implementation switch (diagnostics/parity): the update runs layer 3 and the PPO loss head as two kernels (forward
 * GEMM + warp-per-row loss head) instead of the loss epilogue fused into the layer-3 GEMM (dZ3 and every gradient
 * but the head / log-std ones are the same bits; those are the same sums in another order) */
#define LG_F_UNFUSED_LOSS 512u

#define LG_NUM_BUFFERS 20
/* Buffer slots for lg_required_sizes / lg_create. Layouts are DESIGN.md §4. */
enum {
  LG_BUF_HEIGHTFIELD = 0, /* fp32 [R][C], filled by the caller before lg_create (read-only) */
  LG_BUF_STATE = 1,       /* SoA 32-bit words [66][N] (DESIGN.md §3.4 record, field-major) */
  LG_BUF_OBS = 2,         /* bf16 [T+1][N][D_pad]: slot t = o_t, slot T = o_T */
  LG_BUF_ACT = 3,         /* fp32 [T][N][12] */
  LG_BUF_MU = 4,          /* fp32 [T][N][12] */
  LG_BUF_LOGP = 5,        /* fp32 [T][N] */
  LG_BUF_VALUE = 6,       /* fp32 [T][N] */
  LG_BUF_REWARD = 7,      /* fp32 [T][N] */
  LG_BUF_BOOT = 8,        /* fp32 [T][N]: V(o_term) for time-out samples, else 0 */
  LG_BUF_FLAGS = 9,       /* u8 [T][N]: bit0 terminated, bit1 time-out */
  LG_BUF_ADV = 10,        /* fp32 [T][N] un-normalised advantages */
  LG_BUF_RET = 11,        /* fp32 [T][N] returns A + V */
  LG_BUF_VALUE_T = 12,    /* fp32 [N] V(o_T) */
  LG_BUF_THETA = 13,      /* fp32 [P] parameters in the canonical order */
  LG_BUF_ADAM_M = 14,     /* fp32 [P] */
  LG_BUF_ADAM_V = 15,     /* fp32 [P] */
  LG_BUF_GRAD = 16,       /* fp32 [P + 16]: gradient ‖ stats payload (allreduced when W > 1) */
  LG_BUF_WEIGHTS = 17,    /* bf16/fp32 GEMM-layout shadow of θ (library-private layout) */
  LG_BUF_ACTIV = 18,      /* minibatch activations (library-private) */
  LG_BUF_WORK = 19        /* partials, counters, device scalars (library-private) */
};

typedef struct {
  uint32_t struct_size; /* = sizeof(lg_config) (ABI check) */
  int32_t n_envs;       /* N per rank, >= 1 */
  int32_t n_steps;      /* T, >= 1 */
  int32_t n_epochs;     /* E (Table 3: 5) */
  int32_t n_minibatches;/* K_mb (Table 3: 4); N*T must be divisible by it */
  int32_t hidden[3];    /* MLP widths: h0,h1 multiples of 64 <= 512, h2 multiple of 32 <= 128 (BJ: 512,256,128) */
  int32_t scan_nx, scan_ny; /* height-scan grid (17, 11); (0,0) = flat 48-dim obs */
  int32_t n_levels, n_cols; /* world tiles (R = 80*n_levels, C = 80*n_cols), each >= 1 */
  float inv_cell;           /* 10.0 (0.1 m cells) */
  float gamma, lam;         /* 0.99, 0.95 (Table 3) */
  float clip, vclip;        /* 0.2, 0.2 */
  float ent_coef, vf_coef;  /* 0.01, 1.0 */
  float kl_target;          /* kl* = 0.01 (Alg. 1) */
  float lr_init;            /* α0 = 1e-3 (R16) */
  float adam_b1, adam_b2, adam_eps; /* 0.9, 0.999, 1e-8 */
  uint64_t seed;            /* Philox key */
  int32_t rank, world_size; /* global env id g = rank*N + i */
  uint32_t flags;           /* LG_F_* */
} lg_config;

/* Statistics of the last ppo_update, written on the device (mirrors SPEC S:424). */
typedef struct {
  float surrogate_loss, value_loss, entropy, mean_kl, lr, clip_fraction;
  int32_t nonfinite_skips, minibatches_applied;
  float mean_episode_return, mean_episode_length;
  int32_t episodes, promotions, demotions;
  int32_t nonfinite_envs; /* env steps whose state went non-finite: forced terminated, reward 0, reset */
  int32_t level_hist[16];
} lg_update_stats;

/* Number of parameters P for a config. Returns -1 on invalid config. */
int64_t lg_num_params(const lg_config* cfg_h);

/* Observation dimension D (48 + nx*ny) and its padded bf16 row stride D_pad = roundup(D, 8). */
int32_t lg_obs_dim(const lg_config* cfg_h);
int32_t lg_obs_stride(const lg_config* cfg_h);

/* Validate cfg_h and write the byte size of every buffer slot into bytes_h[LG_NUM_BUFFERS].
 * Errors: INVALID_ARG (zero envs, B % K_mb != 0, null), RANGE (γ, λ ∉ (0,1], levels < 1),
 * SHAPE (hidden not a multiple of 32 or > 512). */
lg_status lg_required_sizes(const lg_config* cfg_h, size_t bytes_h[LG_NUM_BUFFERS]);

/* Create a context on the current CUDA device bound to `stream` (a cudaStream_t; 0 = legacy default).
 * buffers_h[i] are caller-allocated device pointers of at least bytes_h[i] bytes, 256-B aligned.
 * The heightfield must already be in LG_BUF_HEIGHTFIELD. Builds TMA descriptors; no kernels run. */
lg_status lg_create(const lg_config* cfg_h, void* const buffers_h[LG_NUM_BUFFERS], void* stream, lg_ctx** out_h);
lg_status lg_destroy(lg_ctx* ctx);
const char* lg_last_error(const lg_ctx* ctx);

/* Parameters. params_set copies θ (device fp32 [P]) into LG_BUF_THETA, refreshes the
 * GEMM shadow, zeroes Adam moments and step count, and sets α = lr_init. */
lg_status lg_params_set(lg_ctx* ctx, const float* theta);
/* Refresh the GEMM-layout shadow from LG_BUF_THETA (after the caller wrote θ directly). */
lg_status lg_params_sync(lg_ctx* ctx);
/* Checkpoint / resume. Every piece of training state lives in the caller-owned
 * buffers (θ, Adam moments, α and the Adam step on device, the environment state, OBS slot 0 = o_0 of the
 * next iteration, the step counter s_base), so a checkpoint is a byte copy of all LG_NUM_BUFFERS buffers
 * taken between iterations (stream idle). After the caller restores such a copy into the buffers of a
 * context created with the same configuration, lg_resume marks the environment as initialised (instead
 * of env_reset, which would redraw o_0) and refreshes the GEMM shadow from θ; the continued run is
 * bit-identical to the uninterrupted one. No validation of the buffer contents is possible. */
lg_status lg_resume(lg_ctx* ctx);

/* --- Environment (SPEC env module S:237-323; PAPER §3) --- */
/* Reset envs (mask u8 [N], NULL = all; `init` != 0 also assigns column g mod n_cols and level 0,
 * S:106-113) and write o_0 into OBS slot 0 (and fp32 obs [N][D] if non-NULL). Uses step counter s_base. */
lg_status env_reset(lg_ctx* ctx, const uint8_t* mask, int32_t init, float* obs);
/* One policy step t (0 <= t < T) with actions from ACT slot t (written by policy_act) or, if
 * `actions` != NULL, from that fp32 [N][12] buffer (which is then copied into ACT slot t).
 * Writes REWARD/FLAGS/BOOT slot t and o_{t+1} into OBS slot t+1; optional caller outputs (may be NULL):
 * obs fp32 [N][D] (post-reset), reward fp32 [N], terminated/timeout u8 [N], terms fp32 [N][9]
 * (per-term reward breakdown). With LG_F_BOOTSTRAP the pre-reset observation of every time-out
 * env is compacted into the rollout's time-out buffer (t == 0 starts a rollout); BOOT slot t is 0 until
 * storage_compute_gae writes the bootstrap critic values V(o_term) of the whole rollout at once. */
lg_status env_step_obs_reward(lg_ctx* ctx, int32_t t, const float* actions, float* obs, float* reward,
                              uint8_t* terminated, uint8_t* timeout, float* terms);

/* --- Policy (actor-critic MLP, Gaussian head) --- */
/* Forward actor and critic on OBS slot t, sample a = μ + σ⊙ε (ACTION Philox stream), write ACT, MU,
 * LOGP, VALUE slot t; optional copies into the caller's fp32 buffers (may be NULL). */
lg_status policy_act(lg_ctx* ctx, int32_t t, float* actions, float* logp, float* mu, float* value);
/* Deterministic forward on an arbitrary bf16 batch x [M][D_pad] (parity/eval): mu [M][12], value [M]. */
lg_status policy_forward(lg_ctx* ctx, const void* x_bf16, int32_t M, float* mu, float* value);

/* --- Learning --- */
/* With LG_F_BOOTSTRAP first V(o_term) of the rollout's compacted time-outs into BOOT (one batched
 * critic pass); then V(o_T) from OBS slot T, GAE with time-out bootstrapping, batch statistics.
 * adv/ret (fp32 [T][N], may be NULL) receive copies of LG_BUF_ADV / LG_BUF_RET. Advances s_base by T. */
lg_status storage_compute_gae(lg_ctx* ctx, float* adv, float* ret);
/* E epochs x K_mb minibatches of the clipped-surrogate update with Alg. 1 and Adam; copies OBS slot T
 * into slot 0 for the next iteration. stats (device lg_update_stats*, may be NULL) is written. */
lg_status ppo_update(lg_ctx* ctx, lg_update_stats* stats);
/* The epoch-`epoch` permutation π of [0, N*T) of the current iteration (the shuffle
 * ppo_update uses), written to perm uint32 [N*T]. */
lg_status ppo_shuffle(lg_ctx* ctx, int32_t epoch, uint32_t* perm);
/* Only the gradient of one minibatch (parity): gathered rows idx int32 [M_mb] of the current batch;
 * writes the gradient into LG_BUF_GRAD without any optimizer step. Requires storage_compute_gae. */
lg_status ppo_minibatch_grad(lg_ctx* ctx, const int32_t* idx, int32_t M_mb);

/* --- Curriculum --- */
/* Standalone curriculum rule over n hand-built records (for traces/tests): level in/out [n].
 * crossed u8 [n], disp_xy fp32 [n][2], cmd_xy fp32 [n][2], ep_steps int32 [n], loop_words uint32 [n]
 * (the Philox CURRICULUM word each record would use). */
lg_status curriculum_update(lg_ctx* ctx, int32_t n, const uint8_t* crossed, const float* disp_xy,
                            const float* cmd_xy, const int32_t* ep_steps, const uint32_t* loop_words,
                            int32_t* level);

/* --- Multi-GPU (NCCL over NVLink; one process per GPU) --- */
/* Write a fresh ncclUniqueId (128 bytes) into id_h (rank 0); broadcast it with torch.distributed. */
lg_status lg_nccl_unique_id(uint8_t id_h[128]);
/* ncclCommInitRank(world_size, id, rank) on the context's device; afterwards ppo_update allreduces the
 * gradient ‖ stats payload every minibatch and storage_compute_gae allreduces the advantage statistics. */
lg_status lg_set_nccl(lg_ctx* ctx, const uint8_t id_h[128]);
/* Broadcast θ from rank 0 (then lg_params_sync semantics). */
lg_status lg_broadcast_params(lg_ctx* ctx);

/* --- Multi-rank emulation on one device (tests of the multi-GPU path; VERDICT r01 "loopback") ---
 * A group binds the contexts of ALL ranks 0..n-1 of one world (each created with world_size = n and its own
 * rank, otherwise identical configs, on the same device and the same stream). Per-rank work (rollout, GAE,
 * shuffles, gathers, forward/backward, Adam) runs exactly as in the one-process-per-GPU path; where that path
 * calls ncclAllReduce (advantage statistics: two fp64 sums per iteration; [gradient ‖ stats payload] after every
 * minibatch) the group launches ONE kernel that sums the n ranks' buffers element by element in
 * rank order and writes the sum back to every rank -- no kernel waits on another (B200_PROFILING.md: ranks that
 * wait on each other must not share a GPU). Calls are enqueued in lockstep: all ranks' phase, the sum, all
 * ranks' next phase. While grouped, the single-context learning calls (storage_compute_gae, ppo_update,
 * graph capture, lg_iterate_host) return LG_ERR_STATE. Errors: INVALID_ARG (n outside [1, LG_MAX_GROUP],
 * null pointers, rank/world mismatch, configs that differ in more than the rank, different streams),
 * STATE (a context already grouped or on NCCL; a rank destroyed; iterate before env_reset). */
#define LG_MAX_GROUP 8
typedef struct lg_group lg_group;
lg_status lg_group_create(lg_ctx* const* ctxs_h, int32_t n, lg_group** out_h);
lg_status lg_group_destroy(lg_group* g);
/* θ of rank 0 copied to every rank (the ncclBroadcast of lg_broadcast_params), shadows refreshed */
lg_status lg_group_broadcast_params(lg_group* g);
/* storage_compute_gae of every rank with the union advantage statistics (R13) */
lg_status lg_group_compute_gae(lg_group* g);
/* ppo_update of every rank with the per-minibatch gradient sum; stats_h: n device lg_update_stats* or NULL */
lg_status lg_group_ppo_update(lg_group* g, lg_update_stats* const* stats_h);
/* one whole iteration of every rank: T x (policy_act, env_step_obs_reward) per rank, then the two above */
lg_status lg_group_iterate(lg_group* g, lg_update_stats* const* stats_h);

/* --- World generation (reading R27) --- */
/* Writes the tiled world heightfield into HEIGHTFIELD (device, fp32 [80*n_levels][80*n_cols], row-major;
 * level l along x = rows, column c along y), enqueued on `stream` (a cudaStream_t; NULL = legacy default):
 * 8 m x 8 m tiles of 0.1 m cells, terrain kind = c mod 5 -- flat, slope pyramid (gradient
 * tan(25 deg * d)), rough (U(+-a/2), a = 0.05 (1 + d)), 8 random box obstacles (heights U(+-(0.05 + 0.15 d)),
 * 2 m x 2 m flat spawn plateau), stairs pyramid (0.3 m treads, riser 0.05 + 0.15 d) -- with difficulty
 * d = l / (n_levels - 1) rising along the curriculum's level axis (Fig. 2 caption P:62).
 * Random draws: Philox key = seed, counter (word / 4, tile id l * n_cols + c, 0, 8). Bit-identical to the
 * oracle's definition. Context-free (generate before lg_create, which borrows the buffer read-only).
 * Errors: LG_ERR_INVALID_ARG (null buffer, n_levels or n_cols < 1), LG_ERR_RANGE (n_levels > 64),
 * LG_ERR_UNSUPPORTED (no sm_100 device), LG_ERR_CUDA (launch failure). */
lg_status lg_terrain_generate(float* heightfield, int32_t n_levels, int32_t n_cols, uint64_t seed, void* stream);

/* --- Whole iteration through host buffers (end-to-end metric) --- */
/* Copies the 16-byte control block ctrl_h (reserved, zeros) to the device, runs one full iteration,
 * copies lg_update_stats back into stats_h and synchronises the stream. */
lg_status lg_iterate_host(lg_ctx* ctx, const uint8_t ctrl_h[16], lg_update_stats* stats_h);

/* CUDA graph of one whole iteration (T x (policy_act, env_step_obs_reward), storage_compute_gae,
 * ppo_update) captured on the context stream (which must not be the legacy default stream).
 * capture: records and instantiates (replaces a previous graph); launch: enqueues one replay. */
lg_status lg_graph_capture_iteration(lg_ctx* ctx, lg_update_stats* stats);
lg_status lg_graph_launch(lg_ctx* ctx);
/* Number of kernel nodes (this library's kernels) in the captured iteration graph. */
lg_status lg_graph_kernel_count(lg_ctx* ctx, int32_t* n_h);

/* Debug/introspection: device scalars (int32 [8]): {s_base, iteration, adam_t, alpha (fp32 bits),
 * time-outs compacted since the current rollout began, non-finite skips, applied updates, last KL (fp32 bits)} */
lg_status lg_device_scalars(lg_ctx* ctx, int32_t* out8_h);

/* Debug/introspection: the advantage normalisation of the current batch (R13: union over the ranks, unbiased
 * std, ε = 1e-8), written by storage_compute_gae: Â = (A - mean) * inv_std with inv_std = 1 / (std + 1e-8). */
lg_status lg_adv_normalization(lg_ctx* ctx, double* mean_h, double* inv_std_h);

/* Per-category device timing (measurement only). enable != 0: every later launch is bracketed by a
 * CUDA event pair on the context stream (also inside lg_graph_capture_iteration, as event-record
 * nodes). lg_profile_read (after the stream is idle) adds the elapsed ms and launch counts of all
 * recorded pairs per category into ms_h[n]/count_h[n] (categories LG_PROF_*) and, for eager mode,
 * forgets the pairs. */
#define LG_PROF_ENV 0        /* env_step_obs_reward / env_reset kernels */
#define LG_PROF_GEMM_ROLL 1  /* rollout + bootstrap + V(o_T) forward GEMMs */
#define LG_PROF_GEMM_FWD 2   /* update forward GEMMs */
#define LG_PROF_GEMM_DX 3    /* update input-gradient GEMMs */
#define LG_PROF_GEMM_DW 4    /* update weight-gradient GEMMs (split-K) */
#define LG_PROF_HEADS 5      /* policy heads + sampling */
#define LG_PROF_LOSS 6       /* PPO loss head fwd+bwd */
#define LG_PROF_REDUCE 7     /* deterministic gradient reductions */
#define LG_PROF_GATHER 8     /* shuffle + minibatch gather */
#define LG_PROF_ADAM 9       /* Alg. 1 + Adam */
#define LG_PROF_GAE 10       /* GAE + advantage statistics */
#define LG_PROF_COMM 11      /* NCCL */
#define LG_PROF_MISC 12      /* memsets, copies, bookkeeping */
#define LG_PROF_NCAT 13
lg_status lg_profile(lg_ctx* ctx, int32_t enable);
lg_status lg_profile_read(lg_ctx* ctx, float* ms_h, int32_t* count_h, int32_t n);

#ifdef __cplusplus
}
#endif
#endif /* LG_H_ */
