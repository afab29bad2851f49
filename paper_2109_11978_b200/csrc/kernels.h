// kernels.h -- host/device structures and launchers shared by the translation units of libleggedrl.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <utility>

#include "../../include/lg.h"

namespace lg {

// Launch with programmatic stream serialisation (the kernel overlaps its launch and prologue with the
// predecessor's tail; it must call pdl_wait() before reading the predecessor's outputs). LG_NO_PDL=1 disables.
bool pdl_enabled();
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

struct DevScalars;
using lg_update_stats_dev = ::lg_update_stats;

constexpr int ENV_BLOCK = 32;

struct EnvParams {
  const float* hf;
  int R, C;
  float inv_cell;
  int N, rank, n_levels, n_cols, scan_nx, scan_ny, obs_dim, obs_stride;
  uint32_t ny_magic;         // ceil(2^20 / scan_ny): k / scan_ny = (k * ny_magic) >> 20 for the scan indices
  uint32_t flags, seed_lo, seed_hi;
  uint32_t* state;           // SoA [66][N]
  DevScalars* scalars;
  __nv_bfloat16* obs_out;    // OBS buffer base (slot 0)
  float* reward;             // [T][N]
  uint8_t* flags_out;        // [T][N]
  float* boot;               // [T][N]
  __nv_bfloat16* term_obs;   // [to_cap][Dp] pre-reset observations of the rollout's time-outs (compacted)
  int32_t* term_idx;         // [to_cap] BOOT index t*N + i of each compacted row
  int to_cap;                // rows of term_obs
  void* recs;                // [N] 256-B observation records (written by the transition kernel)
  void* trecs;               // [N] records of the pre-reset state of time-out envs (compacted)
};

void launch_env_reset(const EnvParams& P, const uint8_t* mask, int init, float* obs_f32, cudaStream_t st);
void launch_env_step(const EnvParams& P, int t, const float* actions, float* obs_f32, float* rew, uint8_t* term,
                     uint8_t* to, float* terms, cudaStream_t st);
// world heightfield (reading R27): fp32 [80 L][80 C]; slope[l] = fp32(tan(25 deg * d_l))
constexpr int TERRAIN_MAX_LEVELS = 64;
struct TerrainArgs {
  float* hf;
  int n_levels, n_cols;
  uint32_t seed_lo, seed_hi;
  float slope[TERRAIN_MAX_LEVELS];
};
void launch_terrain(const TerrainArgs& a, cudaStream_t st);
void launch_curriculum(int n, int n_levels, const uint8_t* crossed, const float* disp, const float* cmd,
                       const int32_t* ep, const uint32_t* words, int32_t* level, cudaStream_t st);
void launch_action_eps(int N, int rank, uint32_t s0, uint32_t s1, const DevScalars* sc, int t, float* eps,
                       cudaStream_t st);

// ------------------------------------------------------------------ tcgen05 GEMM
enum GemmKind { GEMM_FWD = 0, GEMM_DX = 1, GEMM_DW = 2 };

// EPI 4 (layer-3 forward of the update): the PPO loss head fused into the epilogue: per row the
// actor / critic heads, the clipped surrogate, value loss, KL, dmu / dV -> dZ3 (the GEMM's bf16 output), and
// per-CTA partials of the head / log-std gradients and loss statistics (k_reduce_heads sums them).
struct LossEpi {
  const float* W4a; const float* b4a; const float* W4c; const float* b4c;
  const float* logstd; const float* logstd_old;
  const float* act; const float* mu_old; const float* logp_old; const float* V_old; const float* adv; const float* ret;
  float clip, vclip, vf_coef, invM;
  int H2;                    // real head input width (<= 128; the tile is 128 wide)
  float* payload;            // the non-finite counter payload[4] is cleared by CTA 0 (first writer of the minibatch)
  float* part;               // [gridDim.x][HP] CTA partials (k_loss_heads layout)
  double* spart;             // [gridDim.x][8] fp64 statistics
  int HP;
  unsigned long long* dbg;   // diagnostics only (tools/gemm_probe loss): per-CTA, per-tile phase timestamps, else null
};

struct GemmArgs {
  CUtensorMap tmA[2];
  CUtensorMap tmB[2];
  CUtensorMap tmC[2];        // EPI 0/2: bf16 output per z (box 64x32); EPI 3: fp32 partial buffer (box 32x32)
  int M, N;                  // output rows / cols (per z)
  const int* M_dev;          // optional device-side M (tiles beyond are skipped)
  int m_tiles, nz;
  int kb_total, kb_per_split, n_tiles, n_splits;
  int ldo;
  const float* bias[2];      // EPI 0
  const __nv_bfloat16* aux[2];  // EPI 2: saved activation for ELU'
  int ld_aux;
  float* part;               // EPI 3: split-K partials [z][split][part_rows][part_ld] (bias column direct)
  long long part_zstride, part_sstride;
  int part_rows, part_ld, part_bias_col, bias_col;
  int probe;                 // diagnostics only (tools/gemm_probe): bit0 = skip the MMAs, bit1 = skip the TMA loads,
                             // bit2 = skip the epilogue
  int pair;                  // forward / input-gradient GEMMs: CTA pairs (cta_group::2, 256-row tiles)
  CUtensorMap tmBp[2];       // pair + K-major B: B with a box of BN/2 rows (each CTA loads half of the tile's B)
  int ws;                    // forward / input-gradient GEMMs: weight-stationary schedule (each CTA keeps one column
                             // block of B resident in shared memory and streams only A), when the block fits
  int ws_split;              // weight-stationary with two slices: CTAs [0, ws_split) serve slice 0 (0 = alternate)
  LossEpi le;                // EPI 4 only
};

bool make_tmap_bf16(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols, uint64_t ld, uint32_t box_rows);
bool make_tmap_f32(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols, uint64_t ld, uint32_t box_rows);
cudaError_t launch_gemm(GemmKind kind, int bn, const GemmArgs& a, cudaStream_t st);
// the update's layer-3 forward with the PPO loss head in its epilogue (EPI 4; a.le): 128-wide tiles, weight-stationary
// (H1 <= 256), CTAs split between the actor and critic slices; returns the grid size (rows of le.part) in *grid
cudaError_t launch_gemm_loss(const GemmArgs& a, int* grid, cudaStream_t st);
int gemm_loss_grid(const GemmArgs& a);

struct DwOut {                 // canonical destinations of a weight-gradient GEMM (see k_gemm_dw)
  float* grad;
  long long w_off[2], b_off[2];
  int cols;                    // real input width (the W row length in the canonical vector)
  int row_split;               // layer 1: rows >= row_split belong to the critic (second net)
  float* payload;              // non-finite counter at payload[4]
  int G;                       // unused (1)
  float* part;                 // [tile][S][128][BN + 20] fp32 split partials (L2-resident scratch)
  int* cnt;                    // grid barrier: cnt[0] arrivals (back to 0 at each release), cnt[1] generation
  unsigned long long* dbg;     // diagnostics only (tools/gemm_probe): per-CTA phase timestamps, else null
  int dbg_mode;                // diagnostics only: 1 = skip the reduction, 2 = loads only, 3 = stores only
  int partial_only;            // store the split partials and stop (Adam sums them: AdamArgs::dw1)
  float part_bound;            // partial_only: a partial element with |x| >= part_bound (or NaN) counts as non-finite
                               // (FLT_MAX / S: the S-term sum in Adam cannot overflow)
};
// split-K over S CTAs per output tile in one cooperative wave (S * tiles <= #SMs), deterministic reduction
// of the S fp32 partials through L2 by the whole grid
cudaError_t launch_gemm_dw(int bn, const GemmArgs& a, const DwOut& o, int S, cudaStream_t st);
// the same with CTA pairs (tcgen05 cta_group::2, 256-row tiles): even m_tiles, bn in {128, 256}
cudaError_t launch_gemm_dw_pair(int bn, const GemmArgs& a, const DwOut& o, int S, cudaStream_t st);
cudaError_t launch_gemm_dw_kmajor(int bn, const GemmArgs& a, const DwOut& o, int S, cudaStream_t st);  // diagnostics

// ------------------------------------------------------------------ fused rollout policy (gemm_tc.cu)
// One rollout step of the policy for the 512-256-128 MLP: per CTA one 128-row tile of one
// net (z = 0 actor, 1 critic); three chained tcgen05 GEMMs with the activations kept in shared memory, the
// heads, and for the actor the Gaussian sample + log-probability (bit-identical to the unfused path).
struct FusedPolicyArgs {
  CUtensorMap tmX;           // OBS slot rows [N][Dp] bf16, box {64, 128}
  CUtensorMap tmW1;          // W1 [2*512][Dp], box {64, 256}
  CUtensorMap tmW2[2];       // W2[z] [256][512], box {64, 256}
  CUtensorMap tmW3[2];       // W3[z] [128][256], box {64, 128}
  const float* b1;           // [2*512]
  const float* b2;           // [2*256]
  const float* b3;           // [2*128]
  const float* W4a; const float* b4a; const float* W4c; const float* b4c; const float* logstd;
  int N, rank, t, kb1;       // kb1 = K-blocks of layer 1 (Dp / 64 rounded up, <= 4)
  int z0;                    // first net: 0 = actor and critic (grid.y = 2), 1 = critic only (V(o_T))
  int deterministic;         // a = mu (LG_F_DETERMINISTIC, evaluation)
  uint32_t seed_lo, seed_hi;
  const DevScalars* scalars;
  float* act; float* mu; float* logp; float* value;              // storage slot t
  float* u_act; float* u_logp; float* u_mu; float* u_value;      // optional caller copies
  unsigned long long* dbg;   // diagnostics only (tools/gemm_probe): per-CTA phase timestamps, else null
};
cudaError_t launch_policy_fused(const FusedPolicyArgs& a, cudaStream_t st);

// ------------------------------------------------------------------ PPO kernels (ppo.cu)
struct NetDims {
  int D, Dp, H0, H1, H2;
};

struct HeadArgs {
  NetDims nd;
  const __nv_bfloat16* H3;   // [rows][2*H2]
  const float* W4a;          // [12][H2]
  const float* b4a;          // [12]
  const float* W4c;          // [H2]
  const float* b4c;          // [1]
  const float* logstd;       // [12]
  int M;                     // rows
  const int* M_dev;          // optional device row count
  // ACT mode
  int mode;                  // 0 = act (sample), 1 = value scatter, 2 = forward (mu, V)
  int deterministic;         // mode 0: a = mu (LG_F_DETERMINISTIC, evaluation)
  int t, N, rank;
  uint32_t seed_lo, seed_hi;
  const DevScalars* scalars;
  float* act;                // [rows][12]
  float* mu;                 // [rows][12]
  float* logp;               // [rows]
  float* value;              // [rows]  (mode 1: destination base)
  const int32_t* idx;        // mode 1: value[idx[r]] = V
  float* u_act; float* u_logp; float* u_mu; float* u_value;  // optional caller copies
};
void launch_heads(const HeadArgs& a, cudaStream_t st);

struct LossArgs {
  NetDims nd;
  int M;                     // minibatch rows
  const __nv_bfloat16* H3;   // [M][2*H2]
  const float* W4a; const float* b4a; const float* W4c; const float* b4c;
  const float* logstd; const float* logstd_old;
  const float* act; const float* mu_old; const float* logp_old; const float* V_old; const float* adv; const float* ret;
  float clip, vclip, ent_coef, vf_coef;
  float* payload;            // gradient payload; the loss kernel clears its accumulated slot 4
  __nv_bfloat16* dZ3;        // [M][2*H2] out
  float* part;               // [nblk][HP]
  double* spart;             // [nblk][8]
  int HP;
};
int loss_head_partial_floats(int H2);
void launch_loss_heads(const LossArgs& a, cudaStream_t st);
int loss_blocks(int M);

struct HeadReduceArgs {
  int nblk, HP, H2;
  const float* part; const double* spart;
  float* grad;               // canonical gradient base
  long long off_W4a, off_b4a, off_W4c, off_b4c, off_logstd;
  float ent_coef;
  float* payload;            // [16] stats payload (KL sum, surrogate sum, vloss sum, clip count, nonfinite, rows)
  int M;
};
void launch_reduce_heads(const HeadReduceArgs& a, cudaStream_t st);

struct DwReduceArgs {
  const float* part;         // [z][S][rows_pad][ld]
  long long zstride, sstride;
  int ld, S, rows, cols, bias_col;
  float* grad;
  long long w_off[2], b_off[2];  // per z: canonical offsets of W ([rows][cols]) and b ([rows])
  int nz;
  int row_split;             // L1: rows >= row_split belong to the second net (z=1 segment)
  float* payload;            // nonfinite counter
};
void launch_reduce_dw(const DwReduceArgs& a, cudaStream_t st);

struct GaeArgs {
  int N, T;
  const float* r; const float* V; const float* b; const uint8_t* flags; const float* VT;
  float gamma, lam; int bootstrap;
  float* A; float* R;
  double* part;              // [nblk] partial sums
};
void launch_gae(const GaeArgs& a, cudaStream_t st);
int gae_blocks(int N);
void launch_sum_partials(const double* part, int n, double* out, cudaStream_t st);
void launch_var_partials(const float* A, int n, const double* mean_total, double count, double* part, cudaStream_t st);
int var_blocks(int n);
// also advances the step counter s_base by T (the rollout's events are consumed)
void launch_adv_finalize(const double* sum_total, const double* sq_total, double count, DevScalars* sc, int T,
                         cudaStream_t st);

struct PermArgs {
  uint32_t B; int E; int epoch; int rank; uint32_t seed_lo, seed_hi; const DevScalars* sc; uint32_t* perm;
  int n_epochs;              // epochs epoch .. epoch + n_epochs - 1, written to perm + k * B
};
void launch_perm(const PermArgs& a, cudaStream_t st);

struct GatherArgs {
  int M, N, Dp;
  const uint32_t* perm;      // minibatch slice of the permutation (or identity idx)
  const int32_t* idx;        // alternative explicit indices (parity)
  const __nv_bfloat16* obs;  // [T+1][N][Dp]
  const float* act; const float* mu; const float* logp; const float* V; const float* A; const float* R;
  DevScalars* sc;

  __nv_bfloat16* X; float* o_act; float* o_mu; float* o_logp; float* o_V; float* o_adv; float* o_ret;
};
void launch_gather(const GatherArgs& a, cudaStream_t st);

struct Segment {
  long long off;             // canonical offset
  int rows, cols;
  int kind;                  // 0 = bf16 dst, 1 = fp32 dst
  void* dst;
  int dst_ld;                // elements
};
constexpr int MAX_SEG = 20;
struct ShadowArgs {
  int nseg;
  Segment seg[MAX_SEG];
  long long P;
  int blk0[MAX_SEG + 1];     // k_adam: first block of each segment (ADAM_BLOCK_ELEMS elements per block)
};
constexpr int ADAM_BLOCK_ELEMS = 512;  // k_adam: 256 threads x 2 elements, every block inside one segment

// a layer's weight gradient as k_gemm_dw's split partials [tile][S][128][rld]: Adam sums the S splits of an element
// in split order 0..S-1 -- the reduction k_gemm_dw would have done, the same bits -- instead of reading grad
// (single-rank update only). Element (net z, row r, column c) lives in output row tile mt = (z row_split + r) / 128
// when the nets share one GEMM (layer 1, row_split = H0), else mt = z m_tiles + r / 128; tile = mt n_tiles + c / bn;
// the bias at column bn of the c = 0 tile
struct AdamPart {
  const float* part;         // null: the layer's W / b come from grad like every other tensor
  int S, rld, bn, n_tiles, m_tiles, row_split, cols;
  long long w_off[2], b_off[2];
};
struct AdamArgs {
  ShadowArgs sh;
  float* theta; float* m; float* v; const float* grad;
  float b1, b2, eps, inv_world;
  DevScalars* sc;
  AdamPart part[3];          // layers 1, 2, 3
};
void launch_adam(const AdamArgs& a, const float* payload, float kl_target, int world, int m, float* acc,
                 cudaStream_t st);
// Adam of minibatch m together with the gather of the next minibatch (one launch, disjoint block ranges)
void launch_adam_gather(const AdamArgs& a, const float* payload, float kl_target, int world, int m, float* acc,
                        const GatherArgs& g, cudaStream_t st);
void launch_sync_shadow(const ShadowArgs& sh, const float* theta, cudaStream_t st);

// the collective of an lg_group (n ranks on one device): p[r][i] <- sum over r' in rank order of p[r'][i]
struct GroupSumArgs {
  void* p[LG_MAX_GROUP];
  int n;
  long long count;
  int is_double;             // fp64 (advantage statistics) or fp32 ([gradient ‖ payload])
};
void launch_group_sum(const GroupSumArgs& a, cudaStream_t st);

struct IterEndArgs {
  DevScalars* sc; void* stats; int n_mb; int T; int n_levels; const uint32_t* state; int N; float entropy_dummy;
  const float* logstd;
};
void launch_iter_begin(DevScalars* sc, float* logstd_old, const float* logstd, float* iter_acc, float b1, float b2,
                       cudaStream_t st);
void launch_iter_end(const IterEndArgs& a, const float* iter_acc, cudaStream_t st);

}  // namespace lg
