// api.cu -- the C ABI of libleggedrl.so (include/lg.h): validation, buffer binding, TMA descriptor
// construction and the orchestration of one PPO iteration. Host code only enqueues work.
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "common.cuh"
#include "kernels.h"

using namespace lg;

namespace {

template <typename T>
T* at(void* base, size_t off) { return reinterpret_cast<T*>(reinterpret_cast<uint8_t*>(base) + off); }
size_t al(size_t x) { return (x + 255) & ~size_t(255); }

struct Dims {
  int N, T, E, K, H0, H1, H2, D, Dp, nx, ny, L, C, R_hf, C_hf, B, Mmb, R, to_cap;
  long long P;
};

bool dims_of(const lg_config* c, Dims& d) {
  d.N = c->n_envs; d.T = c->n_steps; d.E = c->n_epochs; d.K = c->n_minibatches;
  d.H0 = c->hidden[0]; d.H1 = c->hidden[1]; d.H2 = c->hidden[2];
  d.nx = c->scan_nx; d.ny = c->scan_ny;
  d.D = 48 + d.nx * d.ny;
  d.Dp = (d.D + 7) / 8 * 8;
  d.L = c->n_levels; d.C = c->n_cols;
  d.R_hf = 80 * d.L; d.C_hf = 80 * d.C;
  d.B = d.N * d.T;
  d.Mmb = d.K > 0 ? d.B / d.K : 0;
  // an env times out at most once per 1000 steps, so a rollout compacts at most N * ceil(T / 1000) time-outs
  d.to_cap = d.N * ((d.T + 999) / 1000);
  d.R = std::max(std::max(d.N, d.Mmb), d.to_cap);
  long long P = 0;
  for (int z = 0; z < 2; ++z) {
    int A = z == 0 ? 12 : 1;
    P += (long long)d.H0 * d.D + d.H0 + (long long)d.H1 * d.H0 + d.H1 + (long long)d.H2 * d.H1 + d.H2 + (long long)A * d.H2 + A;
  }
  d.P = P + 12;
  return true;
}

// canonical offsets
struct Canon {
  long long W1[2], b1[2], W2[2], b2[2], W3[2], b3[2], W4[2], b4[2], logstd;
};
Canon canon_of(const Dims& d) {
  Canon c;
  long long o = 0;
  for (int z = 0; z < 2; ++z) {
    int A = z == 0 ? 12 : 1;
    c.W1[z] = o; o += (long long)d.H0 * d.D;
    c.b1[z] = o; o += d.H0;
    c.W2[z] = o; o += (long long)d.H1 * d.H0;
    c.b2[z] = o; o += d.H1;
    c.W3[z] = o; o += (long long)d.H2 * d.H1;
    c.b3[z] = o; o += d.H2;
    c.W4[z] = o; o += (long long)A * d.H2;
    c.b4[z] = o; o += A;
  }
  c.logstd = o;
  return c;
}

int bn_for(int n) { return n >= 256 ? 256 : (n > 64 ? 128 : 64); }
// input-gradient GEMMs (epilogue bound, short K): 256-wide tiles only above 256 columns (measured)
int bn_dx(int n) { return n > 256 ? 256 : (n > 64 ? 128 : 64); }
// narrower tiles while the GEMM still fits one wave: small-M (rollout) GEMMs are latency bound, more CTAs win
int bn_fit(int bn, int n, int m_rows, int nz) {
  const int mt = (m_rows + 127) / 128;
  while (bn > 64 && (long long)mt * ((n + bn / 2 - 1) / (bn / 2)) * nz <= 148) bn /= 2;
  return bn;
}
int bn_small(int n, int m_rows, int nz) { return bn_fit(bn_for(n), n, m_rows, nz); }
// schedule of the update's layer-2 forward GEMM (LG_L2_MODE): 0 tile order (W2 re-streamed per tile), 1 weight-
// stationary 128-wide column blocks, 2 CTA pairs (256-row tiles, each CTA streams half of W2's tile; the default:
// measured on one box 4.555 / 4.583 / 4.657 ms per C3 iteration for 2 / 0 / 1)
bool reduce_side() {  // LG_REDUCE_SIDE=0 keeps k_reduce_heads on the main stream (measurement)
  static const bool v = [] { const char* e = getenv("LG_REDUCE_SIDE"); return !(e && e[0] == '0'); }();
  return v;
}
int l2_mode() {
  static const int m = [] { const char* e = getenv("LG_L2_MODE"); return e ? atoi(e) : 2; }();
  return m;
}

struct DwPlan {
  int rows, N, bn, n_tiles, m_tiles, kb_total, tiles, S, kb_per_split, pair;
  size_t part_bytes, bytes;
};
// Weight-gradient GEMM plan (k_gemm_dw): 128 x bn output tiles; the minibatch (K) is split over S CTAs per
// tile (one wave); the S fp32 partials are reduced through L2.
//  * critical (dW1: nothing else runs beside it, Adam waits for it): tiles * S fills the 148 SMs;
//  * background (dW2, dW3: they run on the second stream beside dX2 / dX3, which are on the critical path,
//    and are needed only by Adam): at most 12 splits and 2/3 of the SMs, so that the dX kernel keeps most
//    SMs while the weight gradient is accumulated alongside. Measured on one box (C3): 5.09 ms with every
//    dW at 144 CTAs, 4.89 ms with dW2 at 96 CTAs and dW3 at 24 (S = 12 both); S = 6..16 per layer around
//    that point are all slower; a k-block-based rule (>= 32 per CTA) slowed the smaller minibatches.
static DwPlan dw_plan_bn(int rows, int N, int K, int nz, int bn, bool background) {
  DwPlan p;
  p.rows = rows; p.N = N;
  p.bn = bn;
  p.n_tiles = (N + p.bn - 1) / p.bn;
  p.m_tiles = (rows + 127) / 128;
  p.kb_total = (K + 63) / 64;
  p.tiles = p.n_tiles * p.m_tiles * nz;
  // CTA pairs (256-row tiles, tcgen05 cta_group::2: each CTA loads its 128 rows of dZ and half of the activation
  // tile, so the pair reads the activations once for 256 output rows) when every net has an even number of
  // 128-row tiles; bit-identical to single CTAs (tools/gemm_probe pair), -0.6 % per iteration measured on
  // the same box (LG_DW_PAIR=0 switches them off)
  static const bool pair_env = [] { const char* e = getenv("LG_DW_PAIR"); return !(e && e[0] == '0'); }();
  p.pair = 0;
  // one wave of <= 148 CTAs (background: <= 98), and >= 8 (background: 32) k-blocks per CTA (the fp32
  // partial costs ~3 k-blocks of traffic)
  // (LG_DW_BG_CTAS / LG_DW_BG_SPLITS override the background plan, LG_DW1_CTAS the critical one: measurement only)
  static const int bg_ctas = [] { const char* e = getenv("LG_DW_BG_CTAS"); return e ? atoi(e) : 98; }();
  static const int BG_SPLITS = [] { const char* e = getenv("LG_DW_BG_SPLITS"); return e ? atoi(e) : 12; }();
  static const int crit_ctas = [] { const char* e = getenv("LG_DW1_CTAS"); return e ? atoi(e) : 148; }();
  const int max_ctas = background ? bg_ctas : crit_ctas;
  int S = std::max(1, std::min(std::max(1, p.kb_total / 8), max_ctas / std::max(1, p.tiles)));
  if (background) S = std::min(S, BG_SPLITS);
  p.kb_per_split = (p.kb_total + S - 1) / S;
  p.S = (p.kb_total + p.kb_per_split - 1) / p.kb_per_split;
  if (pair_env && (p.m_tiles % 2 == 0) && p.bn >= 128) p.pair = 1;
  p.part_bytes = al((size_t)p.tiles * p.S * 128 * (p.bn + 20) * 4);
  p.bytes = p.part_bytes + 256;  // + the grid-barrier counter
  return p;
}
// The tile width: the widest tiles (fewest operand re-reads) unless the batch is small (fewer than 8 splits)
// -- then narrower tiles put more SMs on the same k-blocks. Modelled cost of
// the busiest CTA: its operand bytes (the per-SM TMA rate bounds these GEMMs) + the split-K partial's round
// trip through L2; the cheapest wins, ties to the wider tile.
DwPlan dw_plan(int rows, int N, int K, int nz, bool background) {
  const int widest = N > 128 ? 256 : (N > 64 ? 128 : 64);
  DwPlan best = dw_plan_bn(rows, N, K, nz, widest, background);
  // large minibatches keep the widest tiles: their splits already fill the SMs, and the dW chain shares
  // them with the concurrent dX chain (measured: narrower dW3 tiles cost ~2% of the C3 iteration)
  if (best.S >= 8 || best.tiles >= 148) return best;
  auto cost = [](const DwPlan& p) {
    return (double)p.kb_per_split * (128 * 64 * 2 + p.bn * 64 * 2) + (p.S > 1 ? 2.0 * 128 * (p.bn + 20) * 4 : 0.0);
  };
  for (int bn = widest / 2; bn >= 64; bn /= 2) {
    const DwPlan q = dw_plan_bn(rows, N, K, nz, bn, background);
    if (q.tiles * q.S <= 148 && cost(q) < 0.9 * cost(best)) best = q;
  }
  return best;
}

struct Layout {
  size_t bytes[LG_NUM_BUFFERS];
  // WEIGHTS
  size_t w_W1, w_W2, w_W3, w_b1, w_b2, w_b3, w_W4a, w_b4a, w_W4c, w_b4c, w_ls, w_lso;
  // ACTIV
  size_t a_X, a_H1, a_H2, a_H3, a_dZ1, a_dZ2, a_dZ3, a_act, a_mu, a_logp, a_V, a_adv, a_ret, a_omu, a_oV;
  // the gathered minibatch (X + per-sample fields) is double-buffered: set b = 0 at a_X.., set 1 at these
  size_t b_X, b_act, b_mu, b_logp, b_V, b_adv, b_ret;
  // WORK
  size_t k_sc, k_gae, k_var, k_tot, k_lpart, k_spart, k_dw1, k_dw2, k_dw3, k_perm, k_tobs, k_tidx, k_step, k_stats,
      k_ctrl, k_rec, k_trec;
  int HP, nblk_loss, nblk_gae, nblk_var;
  DwPlan dw1, dw2, dw3;
};

Layout layout_of(const Dims& d) {
  Layout L;
  memset(&L, 0, sizeof(L));
  L.bytes[LG_BUF_HEIGHTFIELD] = al((size_t)d.R_hf * d.C_hf * 4);
  L.bytes[LG_BUF_STATE] = al((size_t)NW * d.N * 4);
  L.bytes[LG_BUF_OBS] = al((size_t)(d.T + 1) * d.N * d.Dp * 2);
  L.bytes[LG_BUF_ACT] = L.bytes[LG_BUF_MU] = al((size_t)d.B * 12 * 4);
  for (int b : {LG_BUF_LOGP, LG_BUF_VALUE, LG_BUF_REWARD, LG_BUF_BOOT, LG_BUF_ADV, LG_BUF_RET}) L.bytes[b] = al((size_t)d.B * 4);
  L.bytes[LG_BUF_FLAGS] = al((size_t)d.B);
  L.bytes[LG_BUF_VALUE_T] = al((size_t)d.N * 4);
  L.bytes[LG_BUF_THETA] = L.bytes[LG_BUF_ADAM_M] = L.bytes[LG_BUF_ADAM_V] = al((size_t)d.P * 4);
  L.bytes[LG_BUF_GRAD] = al((size_t)(d.P + 16) * 4);
  size_t o = 0;
  L.w_W1 = o; o = al(o + (size_t)2 * d.H0 * d.Dp * 2);
  L.w_W2 = o; o = al(o + (size_t)2 * d.H1 * d.H0 * 2);
  L.w_W3 = o; o = al(o + (size_t)2 * d.H2 * d.H1 * 2);
  L.w_b1 = o; o = al(o + (size_t)2 * d.H0 * 4);
  L.w_b2 = o; o = al(o + (size_t)2 * d.H1 * 4);
  L.w_b3 = o; o = al(o + (size_t)2 * d.H2 * 4);
  L.w_W4a = o; o = al(o + (size_t)12 * d.H2 * 4);
  L.w_b4a = o; o = al(o + 12 * 4);
  L.w_W4c = o; o = al(o + (size_t)d.H2 * 4);
  L.w_b4c = o; o = al(o + 4);
  L.w_ls = o; o = al(o + 12 * 4);
  L.w_lso = o; o = al(o + 12 * 4);
  L.bytes[LG_BUF_WEIGHTS] = o;
  o = 0;
  const size_t R = (size_t)d.R;
  L.a_X = o; o = al(o + R * d.Dp * 2);
  L.a_H1 = o; o = al(o + R * 2 * d.H0 * 2);
  L.a_H2 = o; o = al(o + R * 2 * d.H1 * 2);
  L.a_H3 = o; o = al(o + R * 2 * d.H2 * 2);
  L.a_dZ1 = o; o = al(o + R * 2 * d.H0 * 2);
  L.a_dZ2 = o; o = al(o + R * 2 * d.H1 * 2);
  L.a_dZ3 = o; o = al(o + R * 2 * d.H2 * 2);
  L.a_act = o; o = al(o + R * 12 * 4);
  L.a_mu = o; o = al(o + R * 12 * 4);
  L.a_logp = o; o = al(o + R * 4);
  L.a_V = o; o = al(o + R * 4);
  L.a_adv = o; o = al(o + R * 4);
  L.a_ret = o; o = al(o + R * 4);
  L.b_X = o; o = al(o + R * d.Dp * 2);
  L.b_act = o; o = al(o + R * 12 * 4);
  L.b_mu = o; o = al(o + R * 12 * 4);
  L.b_logp = o; o = al(o + R * 4);
  L.b_V = o; o = al(o + R * 4);
  L.b_adv = o; o = al(o + R * 4);
  L.b_ret = o; o = al(o + R * 4);
  L.a_omu = o; o = al(o + R * 12 * 4);
  L.a_oV = o; o = al(o + R * 4);
  L.bytes[LG_BUF_ACTIV] = o;
  L.HP = loss_head_partial_floats(d.H2);
  L.nblk_loss = loss_blocks(d.R);
  L.nblk_gae = gae_blocks(d.N);
  L.nblk_var = var_blocks(d.B);
  L.dw1 = dw_plan(2 * d.H0, d.Dp, d.Mmb, 1, false);
  L.dw2 = dw_plan(d.H1, d.H0, d.Mmb, 2, true);
  L.dw3 = dw_plan(d.H2, d.H1, d.Mmb, 2, true);
  o = 0;
  L.k_sc = o; o = al(o + sizeof(DevScalars));
  L.k_gae = o; o = al(o + (size_t)L.nblk_gae * 8);
  L.k_var = o; o = al(o + (size_t)L.nblk_var * 8);
  L.k_tot = o; o = al(o + 8 * 8);
  L.k_lpart = o; o = al(o + (size_t)L.nblk_loss * L.HP * 4);
  L.k_spart = o; o = al(o + (size_t)L.nblk_loss * 8 * 8);
  L.k_dw1 = o; o = al(o + L.dw1.bytes);
  L.k_dw2 = o; o = al(o + L.dw2.bytes);
  L.k_dw3 = o; o = al(o + L.dw3.bytes);
  L.k_perm = o; o = al(o + (size_t)d.E * d.B * 4);  // all epochs' permutations of an iteration
  L.k_tobs = o; o = al(o + (size_t)d.to_cap * d.Dp * 2);
  L.k_tidx = o; o = al(o + (size_t)d.to_cap * 4);
  L.k_step = o; o = al(o + 16 * 4);
  L.k_stats = o; o = al(o + sizeof(lg_update_stats));
  L.k_ctrl = o; o = al(o + 64);
  L.k_rec = o; o = al(o + (size_t)d.N * 256);
  L.k_trec = o; o = al(o + (size_t)d.N * 256);
  L.bytes[LG_BUF_WORK] = o;
  return L;
}

}  // namespace

struct lg_group;
struct lg_ctx {
  lg_config cfg;
  Dims d;
  Layout L;
  Canon cn;
  void* buf[LG_NUM_BUFFERS];
  cudaStream_t st;
  // second stream for the weight-gradient GEMMs: dW_l only reads dZ_l, so it runs beside dX_l (fork/join by
  // events, captured as graph edges)
  cudaStream_t st2 = nullptr;
  cudaEvent_t ev_fork[3] = {nullptr, nullptr, nullptr}, ev_join = nullptr;
  // third stream: the head-gradient reduction (k_reduce_heads) beside dX3 (it feeds only Adam / the collective)
  cudaStream_t st3 = nullptr;
  cudaEvent_t ev_fork3 = nullptr, ev_join3 = nullptr;
  // multi-rank (NCCL): the gradient allreduce in two buckets -- layers 2-4 + heads on st4 as soon as dW2 and the
  // head reduction are done (overlapping dW1), layer 1 + the loss statistics on st after dW1
  cudaStream_t st4 = nullptr;
  cudaEvent_t ev_dw2 = nullptr, ev_heads = nullptr, ev_comm = nullptr;
  bool early_sent = false;  // this minibatch's early bucket is on st4
  // the iteration's shuffles (k_perm: they depend only on the iteration counter) on st3 beside the rollout, whose
  // policy kernel leaves most SMs idle; the update waits for ev_perm instead of launching them
  cudaEvent_t ev_pfork = nullptr, ev_perm = nullptr;
  bool perm_early = false;
  lg_status err = LG_OK;
  std::string msg;
  int world = 1;
  ncclComm_t comm = nullptr;
  lg_group* group = nullptr;  // set while the context is a rank of an lg_group (single-device emulation)
  bool reset_done = false;
  // prebuilt launch descriptors
  std::vector<GemmArgs> l1_roll;  // per OBS slot 0..T
  GemmArgs l1_upd, l2, l3, l1_boot, l2_boot, l3_boot, l1_vt, dx3, dx2, dw3, dw2, dw1;
  GemmArgs l2r, l3r;        // layers 2, 3 for M <= n_envs rows (rollout): narrower tiles (bn2r, bn3r)
  GemmArgs l1_upd_b1, dw1_b1;  // layer-1 forward and weight gradient on gathered set 1 (l1_upd / dw1: set 0)
  GemmArgs l3loss;          // update layer 3 with the PPO loss head in its epilogue (EPI 4; le set per minibatch)
  GemmArgs l2u;             // update layer 2 (minibatch rows), in the schedule of l2_mode()
  int bn2x = 0;             // its tile width
  int bn2r = 0, bn3r = 0;
  int bn1u = 0, bn2u = 0, bn3u = 0, bnx3 = 0, bnx2 = 0;  // update GEMMs (minibatch rows; narrower when M is small)
  CUtensorMap tmW2f[2], tmW3f[2];  // the fused rollout policy's W2 / W3 maps (its fixed boxes, not the update's)
  EnvParams ep;
  ShadowArgs shadow;
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t gexec = nullptr;
  // pointers
  DevScalars* sc;
  float* payload;
  float* step_f;
  // profiling (lg_profile): event pairs around launches
  struct PP { int cat, a, b; };
  bool prof = false, capturing = false;
  // inside ppo_update (run_update): single-rank updates let Adam sum the weight-gradient partials (AdamPart),
  // NCCL ranks send the early gradient bucket beside dW1; ppo_minibatch_grad keeps the plain reduced gradient
  bool in_update = false;
  std::vector<cudaEvent_t> ev;
  std::vector<PP> pairs, gpairs;
  size_t evn = 0;
};

// n contexts (ranks 0..n-1 of one world) driven together on one device: the emulation of the multi-rank path
struct lg_group {
  int n;
  lg_ctx* cs[LG_MAX_GROUP];  // null once a rank's context has been destroyed
};

namespace {
struct Scope {
  lg_ctx* c;
  int cat, a = -1;
  cudaStream_t s;
  Scope(lg_ctx* c_, int cat_, cudaStream_t s_ = nullptr) : c(c_), cat(cat_), s(s_ ? s_ : c_->st) {
    if (c->prof && c->evn + 2 <= c->ev.size()) {
      a = (int)c->evn++;
      cudaEventRecordWithFlags(c->ev[a], s, c->capturing ? cudaEventRecordExternal : cudaEventRecordDefault);
    }
  }
  ~Scope() {
    if (a >= 0) {
      int b = (int)c->evn++;
      cudaEventRecordWithFlags(c->ev[b], s, c->capturing ? cudaEventRecordExternal : cudaEventRecordDefault);
      c->pairs.push_back({cat, a, b});
    }
  }
};
}  // namespace

namespace {

lg_status fail(lg_ctx* c, lg_status s, const char* fmt, ...) {
  if (c && c->err == LG_OK) {
    char b[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(b, sizeof(b), fmt, ap);
    va_end(ap);
    c->err = s;
    c->msg = b;
  }
  return s;
}

#define CK(call)                                                                                   \
  do {                                                                                             \
    cudaError_t e_ = (call);                                                                       \
    if (e_ != cudaSuccess) return fail(ctx, LG_ERR_CUDA, "%s: %s", #call, cudaGetErrorString(e_)); \
  } while (0)
#define CKL()                                                                                                  \
  do {                                                                                                         \
    cudaError_t e_ = cudaGetLastError();                                                                       \
    if (e_ != cudaSuccess) return fail(ctx, LG_ERR_CUDA, "launch (%s:%d): %s", __FILE__, __LINE__, cudaGetErrorString(e_)); \
  } while (0)
#define CKN(call)                                                                                  \
  do {                                                                                             \
    ncclResult_t r_ = (call);                                                                      \
    if (r_ != ncclSuccess) return fail(ctx, LG_ERR_NCCL, "%s: %s", #call, ncclGetErrorString(r_)); \
  } while (0)
#define GUARD()                          \
  do {                                   \
    if (!ctx) return LG_ERR_INVALID_ARG; \
    if (ctx->err != LG_OK) return ctx->err; \
  } while (0)

lg_status validate(const lg_config* c) {
  if (!c || c->struct_size != sizeof(lg_config)) return LG_ERR_INVALID_ARG;
  if (c->n_envs < 1 || c->n_steps < 1 || c->n_epochs < 1 || c->n_minibatches < 1) return LG_ERR_INVALID_ARG;
  if (((long long)c->n_envs * c->n_steps) % c->n_minibatches != 0) return LG_ERR_INVALID_ARG;
  if ((long long)c->n_envs * c->n_steps >= (1LL << 30)) return LG_ERR_RANGE;
  for (int k = 0; k < 3; ++k)
    if (c->hidden[k] < 32 || c->hidden[k] > 512 || c->hidden[k] % 32 != 0) return LG_ERR_SHAPE;
  if (c->hidden[0] % 64 != 0 || c->hidden[1] % 64 != 0) return LG_ERR_SHAPE;  // K of the next layer in 64-blocks
  if (c->hidden[2] > 128) return LG_ERR_SHAPE;  // heads: <= 4 columns per lane (warp-per-row kernels)
  if (c->scan_nx < 0 || c->scan_ny < 0 || (c->scan_nx == 0) != (c->scan_ny == 0)) return LG_ERR_SHAPE;
  if (48LL + (long long)c->scan_nx * c->scan_ny > 512) return LG_ERR_SHAPE;  // observation row <= 512 (gather)
  if (c->n_levels < 1 || c->n_cols < 1) return LG_ERR_RANGE;
  if (!(c->gamma > 0.f && c->gamma <= 1.f) || !(c->lam >= 0.f && c->lam <= 1.f)) return LG_ERR_RANGE;
  if (!(c->clip > 0.f) || !(c->vclip > 0.f) || !(c->kl_target > 0.f)) return LG_ERR_RANGE;
  if (!(c->lr_init >= 1e-5f && c->lr_init <= 1e-2f)) return LG_ERR_RANGE;
  if (c->world_size < 1 || c->rank < 0 || c->rank >= c->world_size) return LG_ERR_RANGE;
  if (!(c->inv_cell > 0.f)) return LG_ERR_RANGE;
  return LG_OK;
}

void set_fwd_common(GemmArgs& g, int M, int N, int K, int bn, int nz) {
  g.M = M; g.N = N; g.M_dev = nullptr;
  g.kb_total = (K + 63) / 64;
  g.kb_per_split = g.kb_total;
  g.n_tiles = (N + bn - 1) / bn;
  g.n_splits = 1;
  (void)nz;
}

}  // namespace

extern "C" {

int64_t lg_num_params(const lg_config* c) {
  if (validate(c) != LG_OK) return -1;
  Dims d;
  dims_of(c, d);
  return d.P;
}
int32_t lg_obs_dim(const lg_config* c) { return c ? 48 + c->scan_nx * c->scan_ny : -1; }
int32_t lg_obs_stride(const lg_config* c) { return c ? (48 + c->scan_nx * c->scan_ny + 7) / 8 * 8 : -1; }

lg_status lg_required_sizes(const lg_config* c, size_t bytes_h[LG_NUM_BUFFERS]) {
  lg_status s = validate(c);
  if (s != LG_OK) return s;
  if (!bytes_h) return LG_ERR_INVALID_ARG;
  Dims d;
  dims_of(c, d);
  Layout L = layout_of(d);
  for (int i = 0; i < LG_NUM_BUFFERS; ++i) bytes_h[i] = L.bytes[i];
  return LG_OK;
}

const char* lg_last_error(const lg_ctx* ctx) { return ctx ? ctx->msg.c_str() : "null context"; }

lg_status lg_create(const lg_config* cfg, void* const buffers_h[LG_NUM_BUFFERS], void* stream, lg_ctx** out_h) {
  lg_status s = validate(cfg);
  if (s != LG_OK) return s;
  if (!buffers_h || !out_h) return LG_ERR_INVALID_ARG;
  for (int i = 0; i < LG_NUM_BUFFERS; ++i)
    if (!buffers_h[i] || (reinterpret_cast<uintptr_t>(buffers_h[i]) & 255)) return LG_ERR_INVALID_ARG;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return LG_ERR_UNSUPPORTED;
  cudaDeviceProp prop;
  // the library is built for sm_100a only (build.py): any other device, sm_103 included, is unsupported
  if (cudaGetDeviceProperties(&prop, dev) != cudaSuccess || prop.major != 10 || prop.minor != 0) return LG_ERR_UNSUPPORTED;
  lg_ctx* ctx = new lg_ctx();
  ctx->cfg = *cfg;
  dims_of(cfg, ctx->d);
  ctx->L = layout_of(ctx->d);
  ctx->cn = canon_of(ctx->d);
  for (int i = 0; i < LG_NUM_BUFFERS; ++i) ctx->buf[i] = buffers_h[i];
  ctx->st = reinterpret_cast<cudaStream_t>(stream);
  {
    int lo = 0, hi = 0, prio = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    if (ctx->st) cudaStreamGetPriority(ctx->st, &prio);
    bool ok2 = cudaStreamCreateWithPriority(&ctx->st2, cudaStreamNonBlocking, prio) == cudaSuccess;
    for (int k = 0; k < 3; ++k) ok2 = ok2 && cudaEventCreateWithFlags(&ctx->ev_fork[k], cudaEventDisableTiming) == cudaSuccess;
    ok2 = ok2 && cudaEventCreateWithFlags(&ctx->ev_join, cudaEventDisableTiming) == cudaSuccess;
    ok2 = ok2 && cudaStreamCreateWithPriority(&ctx->st3, cudaStreamNonBlocking, prio) == cudaSuccess;
    ok2 = ok2 && cudaEventCreateWithFlags(&ctx->ev_fork3, cudaEventDisableTiming) == cudaSuccess;
    ok2 = ok2 && cudaEventCreateWithFlags(&ctx->ev_join3, cudaEventDisableTiming) == cudaSuccess;
    ok2 = ok2 && cudaStreamCreateWithPriority(&ctx->st4, cudaStreamNonBlocking, prio) == cudaSuccess;
    ok2 = ok2 && cudaEventCreateWithFlags(&ctx->ev_dw2, cudaEventDisableTiming) == cudaSuccess;
    ok2 = ok2 && cudaEventCreateWithFlags(&ctx->ev_heads, cudaEventDisableTiming) == cudaSuccess;
    ok2 = ok2 && cudaEventCreateWithFlags(&ctx->ev_comm, cudaEventDisableTiming) == cudaSuccess;
    ok2 = ok2 && cudaEventCreateWithFlags(&ctx->ev_pfork, cudaEventDisableTiming) == cudaSuccess;
    ok2 = ok2 && cudaEventCreateWithFlags(&ctx->ev_perm, cudaEventDisableTiming) == cudaSuccess;
    if (!ok2) {
      delete ctx;
      return LG_ERR_CUDA;
    }
  }
  ctx->world = cfg->world_size;
  const Dims& d = ctx->d;
  const Layout& L = ctx->L;
  void* W = ctx->buf[LG_BUF_WEIGHTS];
  void* A = ctx->buf[LG_BUF_ACTIV];
  void* K = ctx->buf[LG_BUF_WORK];
  ctx->sc = at<DevScalars>(K, L.k_sc);
  ctx->payload = reinterpret_cast<float*>(ctx->buf[LG_BUF_GRAD]) + d.P;
  ctx->step_f = at<float>(K, L.k_step);

  auto bf = [](void* p, size_t off) { return at<__nv_bfloat16>(p, off); };
  __nv_bfloat16* W1 = bf(W, L.w_W1);
  __nv_bfloat16* W2 = bf(W, L.w_W2);
  __nv_bfloat16* W3 = bf(W, L.w_W3);
  __nv_bfloat16* X = bf(A, L.a_X);
  __nv_bfloat16* H1 = bf(A, L.a_H1);
  __nv_bfloat16* H2 = bf(A, L.a_H2);
  __nv_bfloat16* H3 = bf(A, L.a_H3);
  __nv_bfloat16* dZ1 = bf(A, L.a_dZ1);
  __nv_bfloat16* dZ2 = bf(A, L.a_dZ2);
  __nv_bfloat16* dZ3 = bf(A, L.a_dZ3);
  __nv_bfloat16* OBS = reinterpret_cast<__nv_bfloat16*>(ctx->buf[LG_BUF_OBS]);
  __nv_bfloat16* TOBS = bf(K, L.k_tobs);
  float* b1 = at<float>(W, L.w_b1);
  float* b2 = at<float>(W, L.w_b2);
  float* b3 = at<float>(W, L.w_b3);
  bool ok = true;
  const int bn1 = bn_for(2 * d.H0), bn1c = bn_for(d.H0);
  const int bn1u = ctx->bn1u = bn_small(2 * d.H0, d.Mmb, 1);
  const int bn2 = ctx->bn2u = bn_small(d.H1, d.Mmb, 2), bn3 = ctx->bn3u = bn_small(d.H2, d.Mmb, 2);
  ctx->bnx3 = bn_fit(bn_dx(d.H1), d.H1, d.Mmb, 2);
  ctx->bnx2 = bn_fit(bn_dx(d.H0), d.H0, d.Mmb, 2);
  const uint64_t R = d.R;
  // output maps (TMA stores, box 64 x 32, clipped to the per-net column range)
  auto cmap = [&](CUtensorMap* m, const __nv_bfloat16* base, int cols, int ld) {
    ok &= make_tmap_bf16(m, base, R, cols, ld, 32);
  };
  // ---- forward, layer 1 (both nets concatenated: N = 2*H0)
  ctx->l1_roll.resize(d.T + 1);
  for (int t = 0; t <= d.T; ++t) {
    GemmArgs& g = ctx->l1_roll[t];
    memset(&g, 0, sizeof(g));
    ok &= make_tmap_bf16(&g.tmA[0], OBS + (size_t)t * d.N * d.Dp, d.N, d.Dp, d.Dp, 128);
    ok &= make_tmap_bf16(&g.tmB[0], W1, 2 * d.H0, d.Dp, d.Dp, bn1);
    cmap(&g.tmC[0], H1, 2 * d.H0, 2 * d.H0);
    set_fwd_common(g, d.N, 2 * d.H0, d.Dp, bn1, 1);
    g.ldo = 2 * d.H0; g.bias[0] = b1;
  }
  GemmArgs& u1 = ctx->l1_upd;
  memset(&u1, 0, sizeof(u1));
  ok &= make_tmap_bf16(&u1.tmA[0], X, R, d.Dp, d.Dp, 128);
  ok &= make_tmap_bf16(&u1.tmB[0], W1, 2 * d.H0, d.Dp, d.Dp, bn1u);
  cmap(&u1.tmC[0], H1, 2 * d.H0, 2 * d.H0);
  set_fwd_common(u1, d.Mmb, 2 * d.H0, d.Dp, bn1u, 1);
  u1.ldo = 2 * d.H0; u1.bias[0] = b1;
  u1.ws = 1;  // weight-stationary where the resident block fits (measured gains: layers 1, 3 and dX2)
  ctx->l1_upd_b1 = u1;
  ok &= make_tmap_bf16(&ctx->l1_upd_b1.tmA[0], bf(A, L.b_X), R, d.Dp, d.Dp, 128);
  // ---- forward, layers 2, 3 (z = net)
  GemmArgs& g2 = ctx->l2;
  memset(&g2, 0, sizeof(g2));
  GemmArgs& g3 = ctx->l3;
  memset(&g3, 0, sizeof(g3));
  for (int z = 0; z < 2; ++z) {
    ok &= make_tmap_bf16(&g2.tmA[z], H1 + z * d.H0, R, d.H0, 2 * d.H0, 128);
    ok &= make_tmap_bf16(&g2.tmB[z], W2 + (size_t)z * d.H1 * d.H0, d.H1, d.H0, d.H0, bn2);
    cmap(&g2.tmC[z], H2 + z * d.H1, d.H1, 2 * d.H1);
    g2.bias[z] = b2 + z * d.H1;
    ok &= make_tmap_bf16(&g3.tmA[z], H2 + z * d.H1, R, d.H1, 2 * d.H1, 128);
    ok &= make_tmap_bf16(&g3.tmB[z], W3 + (size_t)z * d.H2 * d.H1, d.H2, d.H1, d.H1, bn3);
    cmap(&g3.tmC[z], H3 + z * d.H2, d.H2, 2 * d.H2);
    g3.bias[z] = b3 + z * d.H2;
  }
  set_fwd_common(g2, d.Mmb, d.H1, d.H0, bn2, 2); g2.ldo = 2 * d.H1;
  {  // the update's layer 2: B (W2 of a net, H1 x H0) is re-streamed for every row tile unless it stays resident
    GemmArgs& u2 = ctx->l2u;
    u2 = g2;
    ctx->bn2x = bn2;
    const int mode = l2_mode();
    if (mode == 1 && d.H0 / 64 <= 8) {  // weight-stationary 128-wide column blocks (128 x H0 bf16 <= 128 KB resident)
      ctx->bn2x = 128;
      for (int z = 0; z < 2; ++z)
        ok &= make_tmap_bf16(&u2.tmB[z], W2 + (size_t)z * d.H1 * d.H0, d.H1, d.H0, d.H0, 128);
      set_fwd_common(u2, d.Mmb, d.H1, d.H0, 128, 2);
      u2.ws = 1;
    } else if (mode == 2 && bn2 >= 128) {  // CTA pairs: 256-row tiles, each CTA streams half of the tile's B
      u2.pair = 1;
      for (int z = 0; z < 2; ++z)
        ok &= make_tmap_bf16(&u2.tmBp[z], W2 + (size_t)z * d.H1 * d.H0, d.H1, d.H0, d.H0, bn2 / 2);
    }
  }
  set_fwd_common(g3, d.Mmb, d.H2, d.H1, bn3, 2); g3.ldo = 2 * d.H2;
  g3.ws = 1;
  {  // layer 3 + loss head (EPI 4): 128-wide tiles (a whole head input row per tile), output dZ3
    GemmArgs& gl = ctx->l3loss;
    memset(&gl, 0, sizeof(gl));
    for (int z = 0; z < 2; ++z) {
      gl.tmA[z] = g3.tmA[z];
      ok &= make_tmap_bf16(&gl.tmB[z], W3 + (size_t)z * d.H2 * d.H1, d.H2, d.H1, d.H1, 128);
      cmap(&gl.tmC[z], dZ3 + z * d.H2, d.H2, 2 * d.H2);
      gl.bias[z] = b3 + z * d.H2;
    }
    set_fwd_common(gl, d.Mmb, d.H2, d.H1, 128, 2);
    gl.ldo = 2 * d.H2;
  }
  for (int z = 0; z < 2; ++z) {
    ok &= make_tmap_bf16(&ctx->tmW2f[z], W2 + (size_t)z * d.H1 * d.H0, d.H1, d.H0, d.H0, bn_for(d.H1));
    ok &= make_tmap_bf16(&ctx->tmW3f[z], W3 + (size_t)z * d.H2 * d.H1, d.H2, d.H1, d.H1, bn_for(d.H2));
  }
  ctx->bn2r = bn_small(d.H1, d.N, 2);
  ctx->bn3r = bn_small(d.H2, d.N, 2);
  ctx->l2r = g2;
  ctx->l3r = g3;
  ctx->l3r.ws = 0;
  for (int z = 0; z < 2; ++z) {
    ok &= make_tmap_bf16(&ctx->l2r.tmB[z], W2 + (size_t)z * d.H1 * d.H0, d.H1, d.H0, d.H0, ctx->bn2r);
    ok &= make_tmap_bf16(&ctx->l3r.tmB[z], W3 + (size_t)z * d.H2 * d.H1, d.H2, d.H1, d.H1, ctx->bn3r);
  }
  set_fwd_common(ctx->l2r, d.N, d.H1, d.H0, ctx->bn2r, 2);
  set_fwd_common(ctx->l3r, d.N, d.H2, d.H1, ctx->bn3r, 2);
  // ---- critic-only chains (time-out bootstrap on compacted rows; V(o_T) on OBS slot T)
  GemmArgs& c1 = ctx->l1_boot;
  memset(&c1, 0, sizeof(c1));
  ok &= make_tmap_bf16(&c1.tmA[0], TOBS, d.to_cap, d.Dp, d.Dp, 128);
  ok &= make_tmap_bf16(&c1.tmB[0], W1 + (size_t)d.H0 * d.Dp, d.H0, d.Dp, d.Dp, bn1c);
  cmap(&c1.tmC[0], H1 + d.H0, d.H0, 2 * d.H0);
  set_fwd_common(c1, d.to_cap, d.H0, d.Dp, bn1c, 1);
  c1.M_dev = &ctx->sc->n_to_total;
  c1.ldo = 2 * d.H0; c1.bias[0] = b1 + d.H0;
  GemmArgs& cv = ctx->l1_vt;
  cv = c1;
  ok &= make_tmap_bf16(&cv.tmA[0], OBS + (size_t)d.T * d.N * d.Dp, d.N, d.Dp, d.Dp, 128);
  cv.M_dev = nullptr;
  GemmArgs& c2 = ctx->l2_boot;
  memset(&c2, 0, sizeof(c2));
  c2.tmA[0] = g2.tmA[1]; c2.tmB[0] = g2.tmB[1]; c2.tmC[0] = g2.tmC[1];
  set_fwd_common(c2, d.N, d.H1, d.H0, bn2, 1);
  c2.bias[0] = g2.bias[1]; c2.ldo = 2 * d.H1;
  GemmArgs& c3 = ctx->l3_boot;
  memset(&c3, 0, sizeof(c3));
  c3.tmA[0] = g3.tmA[1]; c3.tmB[0] = g3.tmB[1]; c3.tmC[0] = g3.tmC[1];
  set_fwd_common(c3, d.N, d.H2, d.H1, bn3, 1);
  c3.bias[0] = g3.bias[1]; c3.ldo = 2 * d.H2;
  // ---- backward dX (A = dZ K-major, B = W MN-major), epilogue * ELU'(H)
  GemmArgs& x3 = ctx->dx3;
  memset(&x3, 0, sizeof(x3));
  GemmArgs& x2 = ctx->dx2;
  memset(&x2, 0, sizeof(x2));
  for (int z = 0; z < 2; ++z) {
    ok &= make_tmap_bf16(&x3.tmA[z], dZ3 + z * d.H2, R, d.H2, 2 * d.H2, 128);
    ok &= make_tmap_bf16(&x3.tmB[z], W3 + (size_t)z * d.H2 * d.H1, d.H2, d.H1, d.H1, 64);
    cmap(&x3.tmC[z], dZ2 + z * d.H1, d.H1, 2 * d.H1);
    x3.aux[z] = H2 + z * d.H1;
    ok &= make_tmap_bf16(&x2.tmA[z], dZ2 + z * d.H1, R, d.H1, 2 * d.H1, 128);
    ok &= make_tmap_bf16(&x2.tmB[z], W2 + (size_t)z * d.H1 * d.H0, d.H1, d.H0, d.H0, 64);
    cmap(&x2.tmC[z], dZ1 + z * d.H0, d.H0, 2 * d.H0);
    x2.aux[z] = H1 + z * d.H0;
  }
  set_fwd_common(x3, d.Mmb, d.H1, d.H2, ctx->bnx3, 2); x3.ldo = 2 * d.H1; x3.ld_aux = 2 * d.H1;
  set_fwd_common(x2, d.Mmb, d.H0, d.H1, ctx->bnx2, 2); x2.ldo = 2 * d.H0; x2.ld_aux = 2 * d.H0;
  x2.ws = 1;
  // ---- backward dW (A = dZ MN-major, B = activations MN-major), split-K over the minibatch
  auto dw_setup = [&](GemmArgs& g, const DwPlan& p, int nz) {
    g.M = p.rows; g.N = p.N; g.M_dev = nullptr;
    g.kb_total = p.kb_total; g.n_tiles = p.n_tiles; g.n_splits = 1;
    g.kb_per_split = p.kb_per_split;
    g.m_tiles = p.m_tiles; g.nz = nz;
  };
  GemmArgs& w3 = ctx->dw3;
  memset(&w3, 0, sizeof(w3));
  GemmArgs& w2 = ctx->dw2;
  memset(&w2, 0, sizeof(w2));
  GemmArgs& w1 = ctx->dw1;
  memset(&w1, 0, sizeof(w1));
  const uint64_t Mr = d.Mmb;
  for (int z = 0; z < 2; ++z) {
    ok &= make_tmap_bf16(&w3.tmA[z], dZ3 + z * d.H2, Mr, d.H2, 2 * d.H2, 64);
    ok &= make_tmap_bf16(&w3.tmB[z], H2 + z * d.H1, Mr, d.H1, 2 * d.H1, 64);
    ok &= make_tmap_bf16(&w2.tmA[z], dZ2 + z * d.H1, Mr, d.H1, 2 * d.H1, 64);
    ok &= make_tmap_bf16(&w2.tmB[z], H1 + z * d.H0, Mr, d.H0, 2 * d.H0, 64);
  }
  ok &= make_tmap_bf16(&w1.tmA[0], dZ1, Mr, 2 * d.H0, 2 * d.H0, 64);
  ok &= make_tmap_bf16(&w1.tmB[0], X, Mr, d.Dp, d.Dp, 64);
  dw_setup(w3, L.dw3, 2);
  dw_setup(w2, L.dw2, 2);
  dw_setup(w1, L.dw1, 1);
  ctx->dw1_b1 = w1;
  ok &= make_tmap_bf16(&ctx->dw1_b1.tmB[0], bf(A, L.b_X), Mr, d.Dp, d.Dp, 64);
  if (!ok) {
    delete ctx;
    return LG_ERR_CUDA;
  }
  // ---- env params
  EnvParams& ep = ctx->ep;
  ep.hf = reinterpret_cast<const float*>(ctx->buf[LG_BUF_HEIGHTFIELD]);
  ep.R = d.R_hf; ep.C = d.C_hf; ep.inv_cell = cfg->inv_cell;
  ep.N = d.N; ep.rank = cfg->rank; ep.n_levels = d.L; ep.n_cols = d.C; ep.scan_nx = d.nx; ep.scan_ny = d.ny;
  // exact when k * (ny_magic * ny - 2^20) < 2^20: k < nx * ny <= 464 and the excess is < ny <= 464 (lg_create's
  // 512-wide observation row bound)
  ep.ny_magic = d.ny > 0 ? ((1u << 20) + (uint32_t)d.ny - 1u) / (uint32_t)d.ny : 0u;
  ep.obs_dim = d.D; ep.obs_stride = d.Dp; ep.flags = cfg->flags;
  ep.seed_lo = (uint32_t)(cfg->seed & 0xFFFFFFFFu); ep.seed_hi = (uint32_t)(cfg->seed >> 32);
  ep.state = reinterpret_cast<uint32_t*>(ctx->buf[LG_BUF_STATE]);
  ep.scalars = ctx->sc;
  ep.obs_out = OBS;
  ep.reward = reinterpret_cast<float*>(ctx->buf[LG_BUF_REWARD]);
  ep.flags_out = reinterpret_cast<uint8_t*>(ctx->buf[LG_BUF_FLAGS]);
  ep.boot = reinterpret_cast<float*>(ctx->buf[LG_BUF_BOOT]);
  ep.term_obs = TOBS;
  ep.to_cap = d.to_cap;
  ep.term_idx = at<int32_t>(K, L.k_tidx);
  ep.recs = at<void>(K, L.k_rec);
  ep.trecs = at<void>(K, L.k_trec);
  // ---- shadow segments (canonical θ -> GEMM layouts)
  ShadowArgs& sh = ctx->shadow;
  memset(&sh, 0, sizeof(sh));
  sh.P = d.P;
  auto seg = [&](long long off, int rows, int cols, int kind, void* dst, int ld) {
    Segment& s = sh.seg[sh.nseg++];
    s.off = off; s.rows = rows; s.cols = cols; s.kind = kind; s.dst = dst; s.dst_ld = ld;
  };
  const Canon& cn = ctx->cn;
  for (int z = 0; z < 2; ++z) {
    seg(cn.W1[z], d.H0, d.D, 0, W1 + (size_t)z * d.H0 * d.Dp, d.Dp);
    seg(cn.b1[z], 1, d.H0, 1, b1 + z * d.H0, d.H0);
    seg(cn.W2[z], d.H1, d.H0, 0, W2 + (size_t)z * d.H1 * d.H0, d.H0);
    seg(cn.b2[z], 1, d.H1, 1, b2 + z * d.H1, d.H1);
    seg(cn.W3[z], d.H2, d.H1, 0, W3 + (size_t)z * d.H2 * d.H1, d.H1);
    seg(cn.b3[z], 1, d.H2, 1, b3 + z * d.H2, d.H2);
  }
  seg(cn.W4[0], 12, d.H2, 1, at<float>(W, L.w_W4a), d.H2);
  seg(cn.b4[0], 1, 12, 1, at<float>(W, L.w_b4a), 12);
  seg(cn.W4[1], 1, d.H2, 1, at<float>(W, L.w_W4c), d.H2);
  seg(cn.b4[1], 1, 1, 1, at<float>(W, L.w_b4c), 1);
  seg(cn.logstd, 1, 12, 1, at<float>(W, L.w_ls), 12);
  {  // the segments tile the canonical vector exactly (k_adam visits every parameter through them)
    long long covered = 0;
    sh.blk0[0] = 0;
    for (int k = 0; k < sh.nseg; ++k) {
      const long long n = (long long)sh.seg[k].rows * sh.seg[k].cols;
      covered += n;
      sh.blk0[k + 1] = sh.blk0[k] + (int)((n + ADAM_BLOCK_ELEMS - 1) / ADAM_BLOCK_ELEMS);
    }
    if (covered != d.P) {
      delete ctx;
      return LG_ERR_SHAPE;
    }
  }
  // zero the padded weight columns and the work buffer once (no kernels launched by the caller yet)
  cudaError_t e = cudaMemsetAsync(W, 0, L.bytes[LG_BUF_WEIGHTS], ctx->st);
  if (e == cudaSuccess) e = cudaMemsetAsync(K, 0, L.bytes[LG_BUF_WORK], ctx->st);
  if (e == cudaSuccess) e = cudaMemsetAsync(ctx->buf[LG_BUF_OBS], 0, L.bytes[LG_BUF_OBS], ctx->st);
  if (e == cudaSuccess) e = cudaMemsetAsync(ctx->buf[LG_BUF_GRAD], 0, L.bytes[LG_BUF_GRAD], ctx->st);
  if (e != cudaSuccess) {
    delete ctx;
    return LG_ERR_CUDA;
  }
  *out_h = ctx;
  return LG_OK;
}

lg_status lg_destroy(lg_ctx* ctx) {
  if (!ctx) return LG_ERR_INVALID_ARG;
  if (ctx->st2) { cudaStreamSynchronize(ctx->st2); cudaStreamDestroy(ctx->st2); }
  if (ctx->st3) { cudaStreamSynchronize(ctx->st3); cudaStreamDestroy(ctx->st3); }
  if (ctx->ev_fork3) cudaEventDestroy(ctx->ev_fork3);
  if (ctx->ev_pfork) cudaEventDestroy(ctx->ev_pfork);
  if (ctx->ev_perm) cudaEventDestroy(ctx->ev_perm);
  if (ctx->ev_join3) cudaEventDestroy(ctx->ev_join3);
  if (ctx->st4) { cudaStreamSynchronize(ctx->st4); cudaStreamDestroy(ctx->st4); }
  for (cudaEvent_t e : {ctx->ev_dw2, ctx->ev_heads, ctx->ev_comm}) if (e) cudaEventDestroy(e);
  for (int k = 0; k < 3; ++k) if (ctx->ev_fork[k]) cudaEventDestroy(ctx->ev_fork[k]);
  if (ctx->ev_join) cudaEventDestroy(ctx->ev_join);
  if (ctx->gexec) cudaGraphExecDestroy(ctx->gexec);
  if (ctx->graph) cudaGraphDestroy(ctx->graph);
  if (ctx->comm) ncclCommDestroy(ctx->comm);
  if (ctx->group)  // the group loses this rank: it can no longer run (lg_group_* return LG_ERR_STATE)
    for (int r = 0; r < ctx->group->n; ++r)
      if (ctx->group->cs[r] == ctx) ctx->group->cs[r] = nullptr;
  delete ctx;
  return LG_OK;
}

static lg_status set_alpha(lg_ctx* ctx) {
  DevScalars tmp;
  memset(&tmp, 0, sizeof(tmp));
  // alpha/adam_t are device fields: write them with small memcpys (no host read)
  float a = ctx->cfg.lr_init;
  int32_t z = 0;
  CK(cudaMemcpyAsync(&ctx->sc->alpha, &a, 4, cudaMemcpyHostToDevice, ctx->st));
  CK(cudaMemcpyAsync(&ctx->sc->adam_t, &z, 4, cudaMemcpyHostToDevice, ctx->st));
  CK(cudaStreamSynchronize(ctx->st));  // host values above live on the stack
  return LG_OK;
}

lg_status lg_params_set(lg_ctx* ctx, const float* theta) {
  GUARD();
  if (!theta) return fail(ctx, LG_ERR_INVALID_ARG, "params_set: null theta");
  const size_t bytes = (size_t)ctx->d.P * 4;
  CK(cudaMemcpyAsync(ctx->buf[LG_BUF_THETA], theta, bytes, cudaMemcpyDeviceToDevice, ctx->st));
  CK(cudaMemsetAsync(ctx->buf[LG_BUF_ADAM_M], 0, bytes, ctx->st));
  CK(cudaMemsetAsync(ctx->buf[LG_BUF_ADAM_V], 0, bytes, ctx->st));
  launch_sync_shadow(ctx->shadow, reinterpret_cast<const float*>(ctx->buf[LG_BUF_THETA]), ctx->st);
  CKL();
  return set_alpha(ctx);
}

lg_status lg_params_sync(lg_ctx* ctx) {
  GUARD();
  launch_sync_shadow(ctx->shadow, reinterpret_cast<const float*>(ctx->buf[LG_BUF_THETA]), ctx->st);
  CKL();
  return LG_OK;
}

lg_status lg_resume(lg_ctx* ctx) {
  GUARD();
  launch_sync_shadow(ctx->shadow, reinterpret_cast<const float*>(ctx->buf[LG_BUF_THETA]), ctx->st);
  CKL();
  ctx->reset_done = true;
  return LG_OK;
}

// ------------------------------------------------------------------ MLP helpers
static int g_gemm_cat = LG_PROF_GEMM_FWD;  // category of the next GEMM launches (profiling only)

static lg_status gemm(lg_ctx* ctx, GemmKind kind, const GemmArgs& g, int bn, int nz) {
  Scope sc_(ctx, kind == GEMM_DW ? LG_PROF_GEMM_DW : kind == GEMM_DX ? LG_PROF_GEMM_DX : g_gemm_cat);
  GemmArgs gg = g;
  gg.m_tiles = (g.M + 127) / 128;
  gg.nz = nz;
  cudaError_t e = launch_gemm(kind, bn, gg, ctx->st);
  if (e != cudaSuccess) return fail(ctx, LG_ERR_CUDA, "gemm(kind %d, bn %d): %s", (int)kind, bn, cudaGetErrorString(e));
  return LG_OK;
}

static HeadArgs head_args(lg_ctx* ctx, int M) {
  HeadArgs h;
  memset(&h, 0, sizeof(h));
  const Dims& d = ctx->d;
  void* W = ctx->buf[LG_BUF_WEIGHTS];
  h.nd = NetDims{d.D, d.Dp, d.H0, d.H1, d.H2};
  h.H3 = at<__nv_bfloat16>(ctx->buf[LG_BUF_ACTIV], ctx->L.a_H3);
  h.W4a = at<float>(W, ctx->L.w_W4a); h.b4a = at<float>(W, ctx->L.w_b4a);
  h.W4c = at<float>(W, ctx->L.w_W4c); h.b4c = at<float>(W, ctx->L.w_b4c);
  h.logstd = at<float>(W, ctx->L.w_ls);
  h.M = M;
  h.N = d.N; h.rank = ctx->cfg.rank;
  h.seed_lo = (uint32_t)(ctx->cfg.seed & 0xFFFFFFFFu); h.seed_hi = (uint32_t)(ctx->cfg.seed >> 32);
  h.scalars = ctx->sc;
  return h;
}

// l1: the layer-1 GEMM (its B map's box is bn1 wide); M <= n_envs rows use the rollout's layer-2/3 tiles
static lg_status forward_rows(lg_ctx* ctx, GemmArgs& l1, int bn1, int M, int cat = LG_PROF_GEMM_FWD) {
  const Dims& d = ctx->d;
  g_gemm_cat = cat;
  l1.M = M;
  const bool small = M <= d.N;
  GemmArgs g2 = small ? ctx->l2r : ctx->l2u, g3 = small ? ctx->l3r : ctx->l3;
  g2.M = M; g3.M = M;
  lg_status s;
  if ((s = gemm(ctx, GEMM_FWD, l1, bn1, 1)) != LG_OK) return s;
  if ((s = gemm(ctx, GEMM_FWD, g2, small ? ctx->bn2r : ctx->bn2x, 2)) != LG_OK) return s;
  if ((s = gemm(ctx, GEMM_FWD, g3, small ? ctx->bn3r : ctx->bn3u, 2)) != LG_OK) return s;
  return LG_OK;
}

static lg_status critic_rows(lg_ctx* ctx, GemmArgs& c1, const int* M_dev, int M) {
  const Dims& d = ctx->d;
  g_gemm_cat = LG_PROF_GEMM_ROLL;
  GemmArgs a = c1, b = ctx->l2_boot, c = ctx->l3_boot;
  a.M = b.M = c.M = M;
  a.M_dev = b.M_dev = c.M_dev = M_dev;
  lg_status s;
  if ((s = gemm(ctx, GEMM_FWD, a, bn_for(d.H0), 1)) != LG_OK) return s;
  if ((s = gemm(ctx, GEMM_FWD, b, ctx->bn2u, 1)) != LG_OK) return s;
  if ((s = gemm(ctx, GEMM_FWD, c, ctx->bn3u, 1)) != LG_OK) return s;
  return LG_OK;
}

// ------------------------------------------------------------------ env
lg_status env_reset(lg_ctx* ctx, const uint8_t* mask, int32_t init, float* obs) {
  GUARD();
  { Scope sc_(ctx, LG_PROF_MISC); CK(cudaMemsetAsync(&ctx->sc->n_to_total, 0, 4, ctx->st)); }
  { Scope sc_(ctx, LG_PROF_ENV); launch_env_reset(ctx->ep, mask, init, obs, ctx->st); }
  CKL();
  ctx->reset_done = true;
  return LG_OK;
}

lg_status env_step_obs_reward(lg_ctx* ctx, int32_t t, const float* actions, float* obs, float* reward,
                              uint8_t* terminated, uint8_t* timeout, float* terms) {
  GUARD();
  const Dims& d = ctx->d;
  if (t < 0 || t >= d.T) return fail(ctx, LG_ERR_RANGE, "env_step: t=%d out of [0,%d)", t, d.T);
  if (!ctx->reset_done) return fail(ctx, LG_ERR_STATE, "env_step before env_reset");
  float* act_slot = reinterpret_cast<float*>(ctx->buf[LG_BUF_ACT]) + (size_t)t * d.N * 12;
  if (actions && actions != act_slot)
    CK(cudaMemcpyAsync(act_slot, actions, (size_t)d.N * 12 * 4, cudaMemcpyDeviceToDevice, ctx->st));
  if (t == 0) {  // a rollout begins (the per-step counters are two slots the env step kernel clears itself)
    Scope sc_(ctx, LG_PROF_MISC);
    CK(cudaMemsetAsync(&ctx->sc->n_to_total, 0, 4, ctx->st));
  }
  { Scope sc_(ctx, LG_PROF_ENV); launch_env_step(ctx->ep, t, act_slot, obs, reward, terminated, timeout, terms, ctx->st); }
  CKL();
  // time-out envs: their pre-reset observation is compacted into the rollout's time-out buffer; the
  // bootstrap critic values V(o_term) are evaluated for all steps at once in storage_compute_gae
  return LG_OK;
}

lg_status curriculum_update(lg_ctx* ctx, int32_t n, const uint8_t* crossed, const float* disp, const float* cmd,
                            const int32_t* ep, const uint32_t* words, int32_t* level) {
  GUARD();
  if (n < 0 || (n > 0 && (!crossed || !disp || !cmd || !ep || !words || !level)))
    return fail(ctx, LG_ERR_INVALID_ARG, "curriculum_update: bad arguments");
  if (n == 0) return LG_OK;
  launch_curriculum(n, ctx->d.L, crossed, disp, cmd, ep, words, level, ctx->st);
  CKL();
  return LG_OK;
}

// ------------------------------------------------------------------ policy
// the fused rollout policy kernel covers the paper's MLP (512-256-128, observation <= 256 columns)
static bool fused_policy_ok(const Dims& d) { return d.H0 == 512 && d.H1 == 256 && d.H2 == 128 && d.Dp <= 256; }

// the fused rollout policy kernel on OBS slot t (slot T: the critic alone gives V(o_T))
static FusedPolicyArgs fused_args(lg_ctx* ctx, int t) {
  const Dims& d = ctx->d;
  FusedPolicyArgs fa;
  memset(&fa, 0, sizeof(fa));
  fa.tmX = ctx->l1_roll[t].tmA[0];
  fa.tmW1 = ctx->l1_roll[t].tmB[0];
  fa.tmW2[0] = ctx->tmW2f[0]; fa.tmW2[1] = ctx->tmW2f[1];
  fa.tmW3[0] = ctx->tmW3f[0]; fa.tmW3[1] = ctx->tmW3f[1];
  void* W = ctx->buf[LG_BUF_WEIGHTS];
  fa.b1 = at<float>(W, ctx->L.w_b1); fa.b2 = at<float>(W, ctx->L.w_b2); fa.b3 = at<float>(W, ctx->L.w_b3);
  fa.W4a = at<float>(W, ctx->L.w_W4a); fa.b4a = at<float>(W, ctx->L.w_b4a);
  fa.W4c = at<float>(W, ctx->L.w_W4c); fa.b4c = at<float>(W, ctx->L.w_b4c); fa.logstd = at<float>(W, ctx->L.w_ls);
  fa.N = d.N; fa.rank = ctx->cfg.rank; fa.t = t; fa.kb1 = (d.Dp + 63) / 64;
  fa.deterministic = (ctx->cfg.flags & LG_F_DETERMINISTIC) ? 1 : 0;
  fa.seed_lo = (uint32_t)(ctx->cfg.seed & 0xFFFFFFFFu); fa.seed_hi = (uint32_t)(ctx->cfg.seed >> 32);
  fa.scalars = ctx->sc;
  return fa;
}

lg_status policy_act(lg_ctx* ctx, int32_t t, float* actions, float* logp, float* mu, float* value) {
  GUARD();
  const Dims& d = ctx->d;
  if (t < 0 || t >= d.T) return fail(ctx, LG_ERR_RANGE, "policy_act: t=%d out of [0,%d)", t, d.T);
  if (fused_policy_ok(d) && !(ctx->cfg.flags & LG_F_UNFUSED_POLICY)) {
    FusedPolicyArgs fa = fused_args(ctx, t);
    fa.act = reinterpret_cast<float*>(ctx->buf[LG_BUF_ACT]) + (size_t)t * d.N * 12;
    fa.mu = reinterpret_cast<float*>(ctx->buf[LG_BUF_MU]) + (size_t)t * d.N * 12;
    fa.logp = reinterpret_cast<float*>(ctx->buf[LG_BUF_LOGP]) + (size_t)t * d.N;
    fa.value = reinterpret_cast<float*>(ctx->buf[LG_BUF_VALUE]) + (size_t)t * d.N;
    fa.u_act = actions; fa.u_logp = logp; fa.u_mu = mu; fa.u_value = value;
    Scope sc_(ctx, LG_PROF_GEMM_ROLL);
    cudaError_t e = launch_policy_fused(fa, ctx->st);
    if (e != cudaSuccess) return fail(ctx, LG_ERR_CUDA, "policy (fused): %s", cudaGetErrorString(e));
    return LG_OK;
  }
  lg_status s = forward_rows(ctx, ctx->l1_roll[t], bn_for(2 * d.H0), d.N, LG_PROF_GEMM_ROLL);
  if (s != LG_OK) return s;
  HeadArgs h = head_args(ctx, d.N);
  h.mode = 0;
  h.deterministic = (ctx->cfg.flags & LG_F_DETERMINISTIC) ? 1 : 0;
  h.t = t;
  h.act = reinterpret_cast<float*>(ctx->buf[LG_BUF_ACT]) + (size_t)t * d.N * 12;
  h.mu = reinterpret_cast<float*>(ctx->buf[LG_BUF_MU]) + (size_t)t * d.N * 12;
  h.logp = reinterpret_cast<float*>(ctx->buf[LG_BUF_LOGP]) + (size_t)t * d.N;
  h.value = reinterpret_cast<float*>(ctx->buf[LG_BUF_VALUE]) + (size_t)t * d.N;
  h.u_act = actions; h.u_logp = logp; h.u_mu = mu; h.u_value = value;
  { Scope sc_(ctx, LG_PROF_HEADS); launch_heads(h, ctx->st); }
  CKL();
  return LG_OK;
}

lg_status policy_forward(lg_ctx* ctx, const void* x, int32_t M, float* mu, float* value) {
  GUARD();
  const Dims& d = ctx->d;
  if (!x || !mu || !value || M < 1 || M > d.R) return fail(ctx, LG_ERR_INVALID_ARG, "policy_forward: bad arguments");
  GemmArgs l1 = ctx->l1_upd;
  if (!make_tmap_bf16(&l1.tmA[0], x, M, d.Dp, d.Dp, 128)) return fail(ctx, LG_ERR_CUDA, "tensor map");
  lg_status s = forward_rows(ctx, l1, ctx->bn1u, M);
  if (s != LG_OK) return s;
  HeadArgs h = head_args(ctx, M);
  h.mode = 2;
  h.mu = mu;
  h.value = value;
  { Scope sc_(ctx, LG_PROF_HEADS); launch_heads(h, ctx->st); }
  CKL();
  return LG_OK;
}

// ------------------------------------------------------------------ learning
// The path's collectives: the advantage statistics (two fp64 sums per iteration) and the
// [gradient ‖ stats payload] of every minibatch, summed over the ranks. `cs[0..n)` are the contexts this process
// drives for the collective: n = 1 with an NCCL communicator (one process per GPU, world_size ranks), or the n
// contexts of an lg_group (every rank of the world on this device; the sum is one kernel over all ranks' buffers
// in rank order -- the emulation of the collective on one GPU, no kernel waits for another). World 1: no-op.
enum CollSel { COLL_GAE_SUM = 0, COLL_GAE_VAR = 1, COLL_GRAD = 2 };
static void* coll_ptr(lg_ctx* ctx, CollSel sel) {
  double* tot = at<double>(ctx->buf[LG_BUF_WORK], ctx->L.k_tot);
  if (sel == COLL_GAE_SUM) return tot;
  if (sel == COLL_GAE_VAR) return tot + 1;
  return ctx->buf[LG_BUF_GRAD];
}
// whether the update takes the multi-rank path (the collectives, reduced weight gradients): world > 1, or a
// single rank with a one-rank NCCL communicator (LG_NCCL_LOOPBACK=1: a diagnostic that runs the NCCL path --
// collectives captured in the iteration graph, the bucket streams, the dW grid reduction -- on one GPU, where
// every allreduce is the identity)
static bool nccl_loopback() {
  static const bool v = [] { const char* e = getenv("LG_NCCL_LOOPBACK"); return e && e[0] == '1'; }();
  return v;
}
static bool multi_rank(const lg_ctx* ctx) { return ctx->world > 1 || (ctx->comm != nullptr && nccl_loopback()); }
// The [grad ‖ payload] vector of a minibatch in two buckets: early = the parameters of layers 2-4,
// the heads and log-std of both nets (final once dW2 and the head reduction are done), late = layer 1 of both nets
// (dW1) and the 16-float statistics payload. Canonical order per net: W1 b1 W2 b2 W3 b3 W4 b4, log-std last, so the
// buckets are two ranges each (+ the payload); together they cover [0, P + 16) exactly once.
struct Range { long long off, len; };
static int grad_bucket(const lg_ctx* ctx, bool early, Range* r) {
  const Canon& c = ctx->cn;
  const long long P = ctx->d.P;
  if (early) {
    r[0] = {c.W2[0], c.W1[1] - c.W2[0]};
    r[1] = {c.W2[1], P - c.W2[1]};
    return 2;
  }
  r[0] = {c.W1[0], c.W2[0] - c.W1[0]};
  r[1] = {c.W1[1], c.W2[1] - c.W1[1]};
  r[2] = {P, 16};
  return 3;
}
static lg_status nccl_ranges(lg_ctx* ctx, bool early, cudaStream_t st) {
  Range r[3];
  const int k = grad_bucket(ctx, early, r);
  float* g = reinterpret_cast<float*>(ctx->buf[LG_BUF_GRAD]);
  CKN(ncclGroupStart());
  for (int i = 0; i < k; ++i) CKN(ncclAllReduce(g + r[i].off, g + r[i].off, (size_t)r[i].len, ncclFloat32, ncclSum, ctx->comm, st));
  CKN(ncclGroupEnd());
  return LG_OK;
}
// NCCL ranks: the early bucket on st4 once dW2 (st2) and the head reduction (ev_heads) are done -- beside dW1
static lg_status send_early_bucket(lg_ctx* ctx) {
  ctx->early_sent = false;
  if (!ctx->in_update || !multi_rank(ctx) || !ctx->comm || ctx->group) return LG_OK;
  CK(cudaEventRecord(ctx->ev_dw2, ctx->prof ? ctx->st : ctx->st2));
  CK(cudaStreamWaitEvent(ctx->st4, ctx->ev_dw2, 0));
  CK(cudaStreamWaitEvent(ctx->st4, ctx->ev_heads, 0));
  {
    Scope sc_(ctx, LG_PROF_COMM, ctx->st4);
    lg_status s = nccl_ranges(ctx, true, ctx->st4);
    if (s != LG_OK) return s;
  }
  CK(cudaEventRecord(ctx->ev_comm, ctx->st4));
  ctx->early_sent = true;
  return LG_OK;
}
static lg_status collective(lg_ctx* const* cs, int n, CollSel sel) {
  lg_ctx* ctx = cs[0];
  const bool dbl = sel != COLL_GRAD;
  const size_t count = dbl ? 1 : (size_t)ctx->d.P + 16;
  if (n == 1) {
    if (!multi_rank(ctx)) return LG_OK;
    if (!ctx->comm) return fail(ctx, LG_ERR_STATE, "world_size %d without a communicator (lg_set_nccl)", ctx->world);
    void* p = coll_ptr(ctx, sel);
    Scope sc_(ctx, LG_PROF_COMM);
    if (sel == COLL_GRAD && ctx->early_sent) {  // layers 2-4 went on st4 beside dW1: join it, then layer 1 + stats
      CK(cudaStreamWaitEvent(ctx->st, ctx->ev_comm, 0));
      ctx->early_sent = false;
      return nccl_ranges(ctx, false, ctx->st);
    }
    CKN(ncclAllReduce(p, p, count, dbl ? ncclFloat64 : ncclFloat32, ncclSum, ctx->comm, ctx->st));
    return LG_OK;
  }
  // the ranks of an lg_group on one device: a rank-ordered sum kernel per range (the gradient in the NCCL path's
  // bucket ranges, so the group tests cover the partition)
  GroupSumArgs g;
  memset(&g, 0, sizeof(g));
  g.n = n;
  g.is_double = dbl ? 1 : 0;
  Scope sc_(ctx, LG_PROF_COMM);
  if (dbl) {
    g.count = (long long)count;
    for (int r = 0; r < n; ++r) g.p[r] = coll_ptr(cs[r], sel);
    launch_group_sum(g, ctx->st);
    CKL();
    return LG_OK;
  }
  for (int early = 1; early >= 0; --early) {
    Range rg[3];
    const int k = grad_bucket(ctx, early != 0, rg);
    for (int i = 0; i < k; ++i) {
      g.count = rg[i].len;
      for (int r = 0; r < n; ++r) g.p[r] = reinterpret_cast<float*>(coll_ptr(cs[r], sel)) + rg[i].off;
      launch_group_sum(g, ctx->st);
      CKL();
    }
  }
  return LG_OK;
}

// a context may run the learning calls alone only if it has no peers, or an NCCL communicator for them
static lg_status solo_ok(lg_ctx* ctx, const char* what) {
  if (ctx->group) return fail(ctx, LG_ERR_STATE, "%s: the context is a rank of an lg_group (use lg_group_*)", what);
  if (ctx->world > 1 && !ctx->comm)
    return fail(ctx, LG_ERR_STATE, "%s: world_size %d needs lg_set_nccl first", what, ctx->world);
  return LG_OK;
}

// storage_compute_gae, phase 1 (per rank): bootstrap critic, V(o_T), GAE, Σ A -> tot[0]
static lg_status gae_local(lg_ctx* ctx) {
  const Dims& d = ctx->d;
  void* K = ctx->buf[LG_BUF_WORK];
  if (ctx->cfg.flags & LG_F_BOOTSTRAP) {  // V(o_term) of every time-out of the rollout, one batched pass
    lg_status s0 = critic_rows(ctx, ctx->l1_boot, &ctx->sc->n_to_total, d.to_cap);
    if (s0 != LG_OK) return s0;
    HeadArgs hb = head_args(ctx, d.to_cap);
    hb.M_dev = &ctx->sc->n_to_total;
    hb.mode = 1;
    hb.value = reinterpret_cast<float*>(ctx->buf[LG_BUF_BOOT]);
    hb.idx = ctx->ep.term_idx;
    { Scope sc_(ctx, LG_PROF_HEADS); launch_heads(hb, ctx->st); }
    CKL();
  }
  // V(o_T): critic on OBS slot T (the fused kernel's critic half when it applies: one launch, bit-identical)
  if (fused_policy_ok(d) && !(ctx->cfg.flags & LG_F_UNFUSED_POLICY)) {
    FusedPolicyArgs fa = fused_args(ctx, d.T);
    fa.z0 = 1;
    fa.value = reinterpret_cast<float*>(ctx->buf[LG_BUF_VALUE_T]);
    Scope sc_(ctx, LG_PROF_GEMM_ROLL);
    cudaError_t e = launch_policy_fused(fa, ctx->st);
    if (e != cudaSuccess) return fail(ctx, LG_ERR_CUDA, "V(o_T) (fused): %s", cudaGetErrorString(e));
  } else {
    lg_status s = critic_rows(ctx, ctx->l1_vt, nullptr, d.N);
    if (s != LG_OK) return s;
    HeadArgs h = head_args(ctx, d.N);
    h.mode = 1;
    h.value = reinterpret_cast<float*>(ctx->buf[LG_BUF_VALUE_T]);
    { Scope sc_(ctx, LG_PROF_HEADS); launch_heads(h, ctx->st); }
    CKL();
  }
  GaeArgs g;
  g.N = d.N; g.T = d.T;
  g.r = reinterpret_cast<const float*>(ctx->buf[LG_BUF_REWARD]);
  g.V = reinterpret_cast<const float*>(ctx->buf[LG_BUF_VALUE]);
  g.b = reinterpret_cast<const float*>(ctx->buf[LG_BUF_BOOT]);
  g.flags = reinterpret_cast<const uint8_t*>(ctx->buf[LG_BUF_FLAGS]);
  g.VT = reinterpret_cast<const float*>(ctx->buf[LG_BUF_VALUE_T]);
  g.gamma = ctx->cfg.gamma; g.lam = ctx->cfg.lam; g.bootstrap = (ctx->cfg.flags & LG_F_BOOTSTRAP) ? 1 : 0;
  g.A = reinterpret_cast<float*>(ctx->buf[LG_BUF_ADV]);
  g.R = reinterpret_cast<float*>(ctx->buf[LG_BUF_RET]);
  g.part = at<double>(K, ctx->L.k_gae);
  Scope sc_gae(ctx, LG_PROF_GAE);
  launch_gae(g, ctx->st);
  CKL();
  launch_sum_partials(g.part, ctx->L.nblk_gae, at<double>(K, ctx->L.k_tot), ctx->st);
  CKL();
  return LG_OK;
}
// phase 2 (per rank, after the Σ A collective): Σ (A - mean)² about the union mean -> tot[1]
static lg_status gae_var(lg_ctx* ctx) {
  const Dims& d = ctx->d;
  void* K = ctx->buf[LG_BUF_WORK];
  double* tot = at<double>(K, ctx->L.k_tot);
  const double count = (double)d.B * ctx->world;
  double* vp = at<double>(K, ctx->L.k_var);
  Scope sc_gae(ctx, LG_PROF_GAE);
  launch_var_partials(reinterpret_cast<const float*>(ctx->buf[LG_BUF_ADV]), d.B, tot, count, vp, ctx->st);
  CKL();
  launch_sum_partials(vp, ctx->L.nblk_var, tot + 1, ctx->st);
  CKL();
  return LG_OK;
}
// phase 3 (per rank, after the variance collective): union mean / std into the device scalars
static lg_status gae_finalize(lg_ctx* ctx, float* adv, float* ret) {
  const Dims& d = ctx->d;
  double* tot = at<double>(ctx->buf[LG_BUF_WORK], ctx->L.k_tot);
  {
    Scope sc_gae(ctx, LG_PROF_GAE);
    launch_adv_finalize(tot, tot + 1, (double)d.B * ctx->world, ctx->sc, d.T, ctx->st);  // (also advances s_base by T)
    CKL();
  }
  if (adv) CK(cudaMemcpyAsync(adv, ctx->buf[LG_BUF_ADV], (size_t)d.B * 4, cudaMemcpyDeviceToDevice, ctx->st));
  if (ret) CK(cudaMemcpyAsync(ret, ctx->buf[LG_BUF_RET], (size_t)d.B * 4, cudaMemcpyDeviceToDevice, ctx->st));
  return LG_OK;
}
static lg_status run_gae(lg_ctx* const* cs, int n, float* adv, float* ret) {
  lg_status s;
  for (int r = 0; r < n; ++r) if ((s = gae_local(cs[r])) != LG_OK) return s;
  if ((s = collective(cs, n, COLL_GAE_SUM)) != LG_OK) return s;
  for (int r = 0; r < n; ++r) if ((s = gae_var(cs[r])) != LG_OK) return s;
  if ((s = collective(cs, n, COLL_GAE_VAR)) != LG_OK) return s;
  for (int r = 0; r < n; ++r) if ((s = gae_finalize(cs[r], adv, ret)) != LG_OK) return s;
  return LG_OK;
}

lg_status storage_compute_gae(lg_ctx* ctx, float* adv, float* ret) {
  GUARD();
  lg_status s = solo_ok(ctx, "storage_compute_gae");
  if (s != LG_OK) return s;
  lg_ctx* cs[1] = {ctx};
  return run_gae(cs, 1, adv, ret);
}

// gradient of one minibatch (rows already gathered into the ACTIV minibatch arrays)
static GatherArgs gather_args(lg_ctx* ctx, int b);
static lg_status backward_chain(lg_ctx* ctx, int b, const uint32_t* next_perm);
// the loss epilogue fused into layer 3 (EPI 4): its weight-stationary schedule keeps W3 (H1 x 128 bf16 per net)
// resident, which fits for H1 <= 256
// the weight gradients leave their split-K reduction to Adam (single-rank ppo_update, S > 1 splits): no grid
// barrier and no reduction pass (dW1's is on the critical path); the multi-rank collective needs reduced gradients
static bool dw1_partial_ok(const lg_ctx* ctx) {
  static const bool off = [] { const char* e = getenv("LG_DW1_PARTIAL"); return e && e[0] == '0'; }();
  return !off && ctx->in_update && !multi_rank(ctx) && !ctx->group && ctx->L.dw1.S > 1;
}
// the same for the background layers 2 and 3 (LG_DW23_PARTIAL=0 switches it off; same-box A/B on C3: 4.38 ms with,
// 4.48 ms without -- Adam reads 16 MB more, the two background launches lose their barrier and reduction)
static bool dw23_partial_ok(const lg_ctx* ctx, const DwPlan& p) {
  static const bool off = [] { const char* e = getenv("LG_DW23_PARTIAL"); return e && e[0] == '0'; }();
  return !off && ctx->in_update && !multi_rank(ctx) && !ctx->group && p.S > 1;
}
static bool fused_loss_ok(const lg_ctx* ctx) {
  return ctx->d.H1 <= 256 && ctx->d.H2 <= 128 && !(ctx->cfg.flags & LG_F_UNFUSED_LOSS);
}

// One minibatch's gradient on gathered set b. With next_perm, the gather of the next minibatch (into set
// 1 - b) is launched on st right after dX2, beside the last weight-gradient GEMM on st2.
static lg_status minibatch_gradient(lg_ctx* ctx, int b, const uint32_t* next_perm) {
  const Dims& d = ctx->d;
  const Layout& L = ctx->L;
  void* W = ctx->buf[LG_BUF_WEIGHTS];
  void* A = ctx->buf[LG_BUF_ACTIV];
  void* K = ctx->buf[LG_BUF_WORK];
  float* grad = reinterpret_cast<float*>(ctx->buf[LG_BUF_GRAD]);
  GemmArgs l1 = b ? ctx->l1_upd_b1 : ctx->l1_upd;
  lg_status s;
  HeadReduceArgs hr;
  hr.HP = L.HP; hr.H2 = d.H2;
  hr.part = at<float>(K, L.k_lpart); hr.spart = at<double>(K, L.k_spart); hr.grad = grad;
  hr.off_W4a = ctx->cn.W4[0]; hr.off_b4a = ctx->cn.b4[0]; hr.off_W4c = ctx->cn.W4[1]; hr.off_b4c = ctx->cn.b4[1];
  hr.off_logstd = ctx->cn.logstd; hr.ent_coef = ctx->cfg.ent_coef; hr.payload = ctx->payload; hr.M = d.Mmb;
  if (fused_loss_ok(ctx)) {
    // layers 1, 2, then layer 3 with the PPO loss head in its epilogue (H3 stays on chip; output dZ3)
    g_gemm_cat = LG_PROF_GEMM_FWD;
    l1.M = d.Mmb;
    GemmArgs g2 = ctx->l2u;
    g2.M = d.Mmb;
    if ((s = gemm(ctx, GEMM_FWD, l1, ctx->bn1u, 1)) != LG_OK) return s;
    if ((s = gemm(ctx, GEMM_FWD, g2, ctx->bn2x, 2)) != LG_OK) return s;
    GemmArgs gl = ctx->l3loss;
    gl.M = d.Mmb;
    LossEpi& le = gl.le;
    le.W4a = at<float>(W, L.w_W4a); le.b4a = at<float>(W, L.w_b4a); le.W4c = at<float>(W, L.w_W4c);
    le.b4c = at<float>(W, L.w_b4c); le.logstd = at<float>(W, L.w_ls); le.logstd_old = at<float>(W, L.w_lso);
    le.act = at<float>(A, b ? L.b_act : L.a_act); le.mu_old = at<float>(A, b ? L.b_mu : L.a_mu);
    le.logp_old = at<float>(A, b ? L.b_logp : L.a_logp);
    le.V_old = at<float>(A, b ? L.b_V : L.a_V); le.adv = at<float>(A, b ? L.b_adv : L.a_adv);
    le.ret = at<float>(A, b ? L.b_ret : L.a_ret);
    le.clip = ctx->cfg.clip; le.vclip = ctx->cfg.vclip; le.vf_coef = ctx->cfg.vf_coef; le.invM = 1.0f / (float)d.Mmb;
    le.H2 = d.H2; le.payload = ctx->payload; le.part = at<float>(K, L.k_lpart); le.spart = at<double>(K, L.k_spart); le.HP = L.HP;
    int grid = 0;
    {
      Scope sc_(ctx, LG_PROF_LOSS);
      cudaError_t e = launch_gemm_loss(gl, &grid, ctx->st);
      if (e != cudaSuccess) return fail(ctx, LG_ERR_CUDA, "gemm_loss: %s", cudaGetErrorString(e));
    }
    hr.nblk = grid;
    // the head-gradient / statistics reduction feeds only Adam (and the collective): on the third stream beside
    // dX3 (the profiled pass keeps it on st so its duration is its own)
    const bool side = !ctx->prof && reduce_side();
    cudaStream_t sr = side ? ctx->st3 : ctx->st;
    if (side) {
      CK(cudaEventRecord(ctx->ev_fork3, ctx->st));
      CK(cudaStreamWaitEvent(ctx->st3, ctx->ev_fork3, 0));
    }
    { Scope sc_(ctx, LG_PROF_REDUCE, sr); launch_reduce_heads(hr, sr); }
    CKL();
    CK(cudaEventRecord(ctx->ev_heads, sr));
    if (side) CK(cudaEventRecord(ctx->ev_join3, ctx->st3));
    s = backward_chain(ctx, b, next_perm);
    if (s == LG_OK && side) CK(cudaStreamWaitEvent(ctx->st, ctx->ev_join3, 0));
    return s;
  }
  if ((s = forward_rows(ctx, l1, ctx->bn1u, d.Mmb)) != LG_OK) return s;
  LossArgs la;
  la.nd = NetDims{d.D, d.Dp, d.H0, d.H1, d.H2};
  la.M = d.Mmb;
  la.H3 = at<__nv_bfloat16>(A, L.a_H3);
  la.W4a = at<float>(W, L.w_W4a); la.b4a = at<float>(W, L.w_b4a); la.W4c = at<float>(W, L.w_W4c); la.b4c = at<float>(W, L.w_b4c);
  la.logstd = at<float>(W, L.w_ls); la.logstd_old = at<float>(W, L.w_lso);
  la.act = at<float>(A, b ? L.b_act : L.a_act); la.mu_old = at<float>(A, b ? L.b_mu : L.a_mu);
  la.logp_old = at<float>(A, b ? L.b_logp : L.a_logp);
  la.V_old = at<float>(A, b ? L.b_V : L.a_V); la.adv = at<float>(A, b ? L.b_adv : L.a_adv);
  la.ret = at<float>(A, b ? L.b_ret : L.a_ret);
  la.payload = ctx->payload;
  la.clip = ctx->cfg.clip; la.vclip = ctx->cfg.vclip; la.ent_coef = ctx->cfg.ent_coef; la.vf_coef = ctx->cfg.vf_coef;
  la.dZ3 = at<__nv_bfloat16>(A, L.a_dZ3);
  la.part = at<float>(K, L.k_lpart);
  la.spart = at<double>(K, L.k_spart);
  la.HP = L.HP;
  { Scope sc_(ctx, LG_PROF_LOSS); launch_loss_heads(la, ctx->st); }
  CKL();
  hr.nblk = loss_blocks(d.Mmb);
  // (measured: on the dW stream instead, the reduction delays dW3 -> dW1 by more than it saves here)
  { Scope sc_(ctx, LG_PROF_REDUCE); launch_reduce_heads(hr, ctx->st); }
  CKL();
  CK(cudaEventRecord(ctx->ev_heads, ctx->st));
  return backward_chain(ctx, b, next_perm);
}

// dZ3 -> dX3, dX2 (st) beside dW3, dW2, dW1 (st2); with next_perm the next minibatch's gather
static lg_status backward_chain(lg_ctx* ctx, int b, const uint32_t* next_perm) {
  const Dims& d = ctx->d;
  const Layout& L = ctx->L;
  float* grad = reinterpret_cast<float*>(ctx->buf[LG_BUF_GRAD]);
  lg_status s;
  // the weight-gradient chain runs on st2 beside the dX chain; the profiled pass (lg_profile, timing each
  // category) keeps everything on st so that every kernel's measured duration is its own
  cudaStream_t sdw = ctx->prof ? ctx->st : ctx->st2;
  auto dw = [&](const GemmArgs& g, const DwPlan& p, size_t koff, int cols, const long long* woff,
                const long long* boff, int row_split, bool partial = false) -> lg_status {
    DwOut o;
    memset(&o, 0, sizeof(o));
    o.partial_only = partial ? 1 : 0;
    o.part_bound = 3.4028234663852886e38f / (float)p.S;
    o.G = 1;
    o.part = at<float>(ctx->buf[LG_BUF_WORK], koff);
    o.cnt = at<int>(ctx->buf[LG_BUF_WORK], koff + p.part_bytes);
    o.grad = grad;
    o.w_off[0] = woff[0]; o.w_off[1] = woff[1]; o.b_off[0] = boff[0]; o.b_off[1] = boff[1];
    o.cols = cols;
    o.row_split = row_split;
    o.payload = ctx->payload;
    Scope sc_(ctx, LG_PROF_GEMM_DW, sdw);
    cudaError_t e = p.pair ? launch_gemm_dw_pair(p.bn, g, o, p.S, sdw) : launch_gemm_dw(p.bn, g, o, p.S, sdw);
    if (e != cudaSuccess) return fail(ctx, LG_ERR_CUDA, "gemm_dw: %s", cudaGetErrorString(e));
    return LG_OK;
  };
  // The dW chain runs on st2, forked after dZ_l is written: dW3 beside dX3, dW2 beside dX2, then dW1;
  // st waits for it before the gradient is reduced / applied.
  auto fork = [&](int k) -> lg_status {
    if (sdw == ctx->st) return LG_OK;
    CK(cudaEventRecord(ctx->ev_fork[k], ctx->st));
    CK(cudaStreamWaitEvent(ctx->st2, ctx->ev_fork[k], 0));
    return LG_OK;
  };
  // launch order inside a layer (measured, same box): dW3 before dX3, dX2 before dW2 (-0.3 %)
  // layer 3
  if ((s = fork(0)) != LG_OK) return s;
  if ((s = dw(ctx->dw3, L.dw3, L.k_dw3, d.H1, ctx->cn.W3, ctx->cn.b3, 0, dw23_partial_ok(ctx, L.dw3))) != LG_OK) return s;
  GemmArgs x3 = ctx->dx3;
  x3.M = d.Mmb;
  if ((s = gemm(ctx, GEMM_DX, x3, ctx->bnx3, 2)) != LG_OK) return s;
  // layer 2
  if ((s = fork(1)) != LG_OK) return s;
  GemmArgs x2 = ctx->dx2;
  x2.M = d.Mmb;
  if ((s = gemm(ctx, GEMM_DX, x2, ctx->bnx2, 2)) != LG_OK) return s;
  if ((s = dw(ctx->dw2, L.dw2, L.k_dw2, d.H0, ctx->cn.W2, ctx->cn.b2, 0, dw23_partial_ok(ctx, L.dw2))) != LG_OK) return s;
  if ((s = send_early_bucket(ctx)) != LG_OK) return s;  // NCCL ranks: layers 2-4 + heads beside dW1
  // layer 1 (both nets in one GEMM: rows [0,H0) actor, [H0,2H0) critic); only the first D columns are θ
  if ((s = fork(2)) != LG_OK) return s;
  if ((s = dw(b ? ctx->dw1_b1 : ctx->dw1, L.dw1, L.k_dw1, d.D, ctx->cn.W1, ctx->cn.b1, d.H0, dw1_partial_ok(ctx))) !=
      LG_OK)
    return s;
  if (next_perm) {  // the next minibatch's gather (set 1 - b) runs beside dW1
    GatherArgs g = gather_args(ctx, 1 - b);
    g.perm = next_perm;
    { Scope sc_(ctx, LG_PROF_GATHER); launch_gather(g, ctx->st); }
    CKL();
  }
  if (sdw != ctx->st) {
    CK(cudaEventRecord(ctx->ev_join, ctx->st2));
    CK(cudaStreamWaitEvent(ctx->st, ctx->ev_join, 0));
  }
  return LG_OK;
}

static GatherArgs gather_args(lg_ctx* ctx, int b) {
  const Dims& d = ctx->d;
  void* A = ctx->buf[LG_BUF_ACTIV];
  const Layout& L = ctx->L;
  GatherArgs g;
  memset(&g, 0, sizeof(g));
  g.M = d.Mmb; g.N = d.N; g.Dp = d.Dp;
  g.obs = reinterpret_cast<const __nv_bfloat16*>(ctx->buf[LG_BUF_OBS]);
  g.act = reinterpret_cast<const float*>(ctx->buf[LG_BUF_ACT]);
  g.mu = reinterpret_cast<const float*>(ctx->buf[LG_BUF_MU]);
  g.logp = reinterpret_cast<const float*>(ctx->buf[LG_BUF_LOGP]);
  g.V = reinterpret_cast<const float*>(ctx->buf[LG_BUF_VALUE]);
  g.A = reinterpret_cast<const float*>(ctx->buf[LG_BUF_ADV]);
  g.R = reinterpret_cast<const float*>(ctx->buf[LG_BUF_RET]);
  g.sc = ctx->sc;
  g.X = at<__nv_bfloat16>(A, b ? L.b_X : L.a_X);
  g.o_act = at<float>(A, b ? L.b_act : L.a_act); g.o_mu = at<float>(A, b ? L.b_mu : L.a_mu);
  g.o_logp = at<float>(A, b ? L.b_logp : L.a_logp);
  g.o_V = at<float>(A, b ? L.b_V : L.a_V); g.o_adv = at<float>(A, b ? L.b_adv : L.a_adv);
  g.o_ret = at<float>(A, b ? L.b_ret : L.a_ret);
  return g;
}

static void iter_begin(lg_ctx* ctx) {
  void* W = ctx->buf[LG_BUF_WEIGHTS];
  launch_iter_begin(ctx->sc, at<float>(W, ctx->L.w_lso), at<float>(W, ctx->L.w_ls), ctx->step_f + 4, ctx->cfg.adam_b1,
                    ctx->cfg.adam_b2, ctx->st);
}

lg_status ppo_shuffle(lg_ctx* ctx, int32_t epoch, uint32_t* perm) {
  GUARD();
  if (!perm || epoch < 0 || epoch >= ctx->d.E) return fail(ctx, LG_ERR_INVALID_ARG, "ppo_shuffle: bad arguments");
  PermArgs pa;
  pa.B = (uint32_t)ctx->d.B; pa.E = ctx->d.E; pa.epoch = epoch; pa.rank = ctx->cfg.rank;
  pa.seed_lo = (uint32_t)(ctx->cfg.seed & 0xFFFFFFFFu); pa.seed_hi = (uint32_t)(ctx->cfg.seed >> 32);
  pa.sc = ctx->sc; pa.perm = perm; pa.n_epochs = 1;
  launch_perm(pa, ctx->st);
  CKL();
  return LG_OK;
}

lg_status ppo_minibatch_grad(lg_ctx* ctx, const int32_t* idx, int32_t M_mb) {
  GUARD();
  const Dims& d = ctx->d;
  if (!idx || M_mb != d.Mmb) return fail(ctx, LG_ERR_SHAPE, "ppo_minibatch_grad: M_mb must equal N*T/K = %d", d.Mmb);
  iter_begin(ctx);
  CKL();
  GatherArgs g = gather_args(ctx, 0);
  g.idx = idx;
  launch_gather(g, ctx->st);
  CKL();
  return minibatch_gradient(ctx, 0, nullptr);
}

static AdamArgs adam_args(lg_ctx* ctx) {
  AdamArgs aa;
  memset(&aa, 0, sizeof(aa));
  aa.sh = ctx->shadow;
  aa.theta = reinterpret_cast<float*>(ctx->buf[LG_BUF_THETA]);
  aa.m = reinterpret_cast<float*>(ctx->buf[LG_BUF_ADAM_M]);
  aa.v = reinterpret_cast<float*>(ctx->buf[LG_BUF_ADAM_V]);
  aa.grad = reinterpret_cast<float*>(ctx->buf[LG_BUF_GRAD]);
  aa.b1 = ctx->cfg.adam_b1; aa.b2 = ctx->cfg.adam_b2; aa.eps = ctx->cfg.adam_eps;
  aa.inv_world = 1.0f / (float)ctx->world;
  aa.sc = ctx->sc;
  const Layout& L = ctx->L;
  auto part = [&](AdamPart& p, const DwPlan& pl, size_t koff, int m_tiles_z, int row_split, int cols,
                  const long long* w, const long long* b) {
    p.part = at<float>(ctx->buf[LG_BUF_WORK], koff);
    p.S = pl.S; p.rld = pl.bn + 20; p.bn = pl.bn; p.n_tiles = pl.n_tiles; p.m_tiles = m_tiles_z;
    p.row_split = row_split; p.cols = cols;
    p.w_off[0] = w[0]; p.w_off[1] = w[1]; p.b_off[0] = b[0]; p.b_off[1] = b[1];
  };
  const Dims& d = ctx->d;
  if (dw1_partial_ok(ctx)) part(aa.part[0], L.dw1, L.k_dw1, L.dw1.m_tiles, d.H0, d.D, ctx->cn.W1, ctx->cn.b1);
  if (dw23_partial_ok(ctx, L.dw2)) part(aa.part[1], L.dw2, L.k_dw2, L.dw2.m_tiles, 0, d.H0, ctx->cn.W2, ctx->cn.b2);
  if (dw23_partial_ok(ctx, L.dw3)) part(aa.part[2], L.dw3, L.k_dw3, L.dw3.m_tiles, 0, d.H1, ctx->cn.W3, ctx->cn.b3);
  return aa;
}
static uint32_t* perm_of(lg_ctx* ctx) { return at<uint32_t>(ctx->buf[LG_BUF_WORK], ctx->L.k_perm); }
// the permutation slice of minibatch k (epoch k / K, slice k % K of that epoch's permutation), or null past the end
static const uint32_t* mb_perm(lg_ctx* ctx, int k) {
  return k < ctx->d.E * ctx->d.K ? perm_of(ctx) + (size_t)k * ctx->d.Mmb : nullptr;
}
static bool gather_prefetch() {  // LG_GATHER_PREFETCH=1: next gather beside dW1 instead of inside the Adam launch
  static const bool v = [] { const char* e = getenv("LG_GATHER_PREFETCH"); return e && e[0] == '1'; }();
  return v;
}

// the Feistel permutations of all E epochs of the iteration (P:272 shuffled minibatches), one launch
static lg_status launch_perms(lg_ctx* ctx, cudaStream_t st) {
  const Dims& d = ctx->d;
  PermArgs pa;
  pa.B = (uint32_t)d.B; pa.E = d.E; pa.epoch = 0; pa.rank = ctx->cfg.rank;
  pa.seed_lo = (uint32_t)(ctx->cfg.seed & 0xFFFFFFFFu); pa.seed_hi = (uint32_t)(ctx->cfg.seed >> 32);
  pa.sc = ctx->sc; pa.perm = perm_of(ctx); pa.n_epochs = d.E;
  { Scope sc_(ctx, LG_PROF_GATHER, st); launch_perm(pa, st); }
  CKL();
  return LG_OK;
}
// ppo_update, per rank: Alg. 1 / Adam scalars of the iteration, the E shuffles, the first minibatch's gather
static lg_status update_begin(lg_ctx* ctx) {
  const Dims& d = ctx->d;
  { Scope sc_(ctx, LG_PROF_MISC); iter_begin(ctx); }
  CKL();
  if (ctx->perm_early) {  // computed beside the rollout (run_iteration)
    CK(cudaStreamWaitEvent(ctx->st, ctx->ev_perm, 0));
    ctx->perm_early = false;
  } else {  // the Feistel permutations of all E epochs (P:272 shuffled minibatches), one launch
    lg_status s = launch_perms(ctx, ctx->st);
    if (s != LG_OK) return s;
  }
  {  // the first minibatch's gather (later ones ride in the Adam launch, or beside dW1 with prefetch)
    GatherArgs g = gather_args(ctx, 0);
    g.perm = perm_of(ctx);
    { Scope sc_(ctx, LG_PROF_GATHER); launch_gather(g, ctx->st); }
    CKL();
  }
  return LG_OK;
}
// minibatch k, per rank: forward, loss, backward into [grad ‖ payload] (summed over the ranks next)
static lg_status update_gradient(lg_ctx* ctx, int k) {
  return minibatch_gradient(ctx, k & 1, gather_prefetch() ? mb_perm(ctx, k + 1) : nullptr);
}
// minibatch k, per rank, after the gradient collective: Alg. 1 on the rank-mean KL + Adam (+ next gather)
static lg_status update_adam(lg_ctx* ctx, int k) {
  AdamArgs aa = adam_args(ctx);
  const uint32_t* next = mb_perm(ctx, k + 1);
  Scope sc_adam(ctx, LG_PROF_ADAM);
  if (next && !gather_prefetch()) {  // Adam of minibatch k and the gather of minibatch k + 1 (other set) in one launch
    GatherArgs g = gather_args(ctx, (k + 1) & 1);
    g.perm = next;
    launch_adam_gather(aa, ctx->payload, ctx->cfg.kl_target, ctx->world, k, ctx->step_f + 4, g, ctx->st);
  } else {
    launch_adam(aa, ctx->payload, ctx->cfg.kl_target, ctx->world, k, ctx->step_f + 4, ctx->st);
  }
  CKL();
  return LG_OK;
}
// iteration end, per rank: statistics, α / Adam step write-back, o_T becomes o_0 of the next iteration
static lg_status update_end(lg_ctx* ctx, lg_update_stats* stats) {
  const Dims& d = ctx->d;
  const Layout& L = ctx->L;
  IterEndArgs ie;
  memset(&ie, 0, sizeof(ie));
  ie.sc = ctx->sc;
  ie.stats = stats ? (void*)stats : (void*)at<lg_update_stats>(ctx->buf[LG_BUF_WORK], L.k_stats);
  ie.n_mb = d.E * d.K; ie.T = d.T; ie.n_levels = d.L;
  ie.state = reinterpret_cast<const uint32_t*>(ctx->buf[LG_BUF_STATE]);
  ie.N = d.N;
  ie.logstd = at<float>(ctx->buf[LG_BUF_WEIGHTS], L.w_ls);
  Scope sc_end(ctx, LG_PROF_MISC);
  launch_iter_end(ie, ctx->step_f + 4, ctx->st);
  CKL();
  __nv_bfloat16* OBS = reinterpret_cast<__nv_bfloat16*>(ctx->buf[LG_BUF_OBS]);
  CK(cudaMemcpyAsync(OBS, OBS + (size_t)d.T * d.N * d.Dp, (size_t)d.N * d.Dp * 2, cudaMemcpyDeviceToDevice, ctx->st));
  return LG_OK;
}
static lg_status run_update(lg_ctx* const* cs, int n, lg_update_stats* const* stats) {
  lg_status s;
  struct Flag {  // in_update for the duration of the update (ppo_minibatch_grad keeps the reduced gradient)
    lg_ctx* const* cs; int n;
    Flag(lg_ctx* const* c, int k) : cs(c), n(k) { for (int r = 0; r < n; ++r) cs[r]->in_update = true; }
    ~Flag() { for (int r = 0; r < n; ++r) cs[r]->in_update = false; }
  } flag(cs, n);
  for (int r = 0; r < n; ++r) if ((s = update_begin(cs[r])) != LG_OK) return s;
  const int n_mb = cs[0]->d.E * cs[0]->d.K;
  for (int k = 0; k < n_mb; ++k) {
    for (int r = 0; r < n; ++r) if ((s = update_gradient(cs[r], k)) != LG_OK) return s;
    if ((s = collective(cs, n, COLL_GRAD)) != LG_OK) return s;
    for (int r = 0; r < n; ++r) if ((s = update_adam(cs[r], k)) != LG_OK) return s;
  }
  for (int r = 0; r < n; ++r) if ((s = update_end(cs[r], stats ? stats[r] : nullptr)) != LG_OK) return s;
  return LG_OK;
}

lg_status ppo_update(lg_ctx* ctx, lg_update_stats* stats) {
  GUARD();
  lg_status s = solo_ok(ctx, "ppo_update");
  if (s != LG_OK) return s;
  lg_ctx* cs[1] = {ctx};
  lg_update_stats* st[1] = {stats};
  return run_update(cs, 1, st);
}

// ------------------------------------------------------------------ multi-GPU
lg_status lg_terrain_generate(float* heightfield, int32_t n_levels, int32_t n_cols, uint64_t seed, void* stream) {
  if (!heightfield || n_levels < 1 || n_cols < 1) return LG_ERR_INVALID_ARG;
  if (n_levels > TERRAIN_MAX_LEVELS) return LG_ERR_RANGE;
  {
    int dev = 0;
    cudaDeviceProp prop;
    if (cudaGetDevice(&dev) != cudaSuccess || cudaGetDeviceProperties(&prop, dev) != cudaSuccess || prop.major != 10 ||
        prop.minor != 0)
      return LG_ERR_UNSUPPORTED;
  }
  TerrainArgs t;
  memset(&t, 0, sizeof(t));
  t.hf = heightfield;
  t.n_levels = n_levels; t.n_cols = n_cols;
  t.seed_lo = (uint32_t)(seed & 0xFFFFFFFFu); t.seed_hi = (uint32_t)(seed >> 32);
  for (int l = 0; l < n_levels; ++l) {  // slope pyramid gradient tan(25 deg * d_l), in double, rounded once
    const float d = n_levels > 1 ? (float)l / (float)(n_levels - 1) : 0.0f;
    t.slope[l] = (float)tan(25.0 * (3.14159265358979323846 / 180.0) * (double)d);
  }
  launch_terrain(t, reinterpret_cast<cudaStream_t>(stream));
  return cudaGetLastError() == cudaSuccess ? LG_OK : LG_ERR_CUDA;
}

lg_status lg_nccl_unique_id(uint8_t id_h[128]) {
  if (!id_h) return LG_ERR_INVALID_ARG;
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return LG_ERR_NCCL;
  memcpy(id_h, &id, 128);
  return LG_OK;
}

lg_status lg_set_nccl(lg_ctx* ctx, const uint8_t id_h[128]) {
  GUARD();
  if (!id_h) return fail(ctx, LG_ERR_INVALID_ARG, "null id");
  if (ctx->group) return fail(ctx, LG_ERR_STATE, "lg_set_nccl: the context is a rank of an lg_group");
  if (ctx->world <= 1 && !nccl_loopback()) return LG_OK;
  ncclUniqueId id;
  memcpy(&id, id_h, 128);
  CKN(ncclCommInitRank(&ctx->comm, ctx->world, id, ctx->cfg.rank));
  return LG_OK;
}

lg_status lg_broadcast_params(lg_ctx* ctx) {
  GUARD();
  if (multi_rank(ctx) && ctx->comm)
    CKN(ncclBroadcast(ctx->buf[LG_BUF_THETA], ctx->buf[LG_BUF_THETA], (size_t)ctx->d.P, ncclFloat32, 0, ctx->comm, ctx->st));
  return lg_params_sync(ctx);
}

// ------------------------------------------------------------------ whole iteration
static lg_status run_iteration(lg_ctx* ctx, lg_update_stats* stats) {
  lg_status s;
  static const bool perm_early = [] { const char* e = getenv("LG_PERM_EARLY"); return !(e && e[0] == '0'); }();
  if (perm_early && !ctx->prof) {  // the shuffles depend only on the iteration counter: beside the rollout
    CK(cudaEventRecord(ctx->ev_pfork, ctx->st));
    CK(cudaStreamWaitEvent(ctx->st3, ctx->ev_pfork, 0));
    if ((s = launch_perms(ctx, ctx->st3)) != LG_OK) return s;
    CK(cudaEventRecord(ctx->ev_perm, ctx->st3));
    ctx->perm_early = true;
  }
  for (int t = 0; t < ctx->d.T; ++t) {
    if ((s = policy_act(ctx, t, nullptr, nullptr, nullptr, nullptr)) != LG_OK) return s;
    if ((s = env_step_obs_reward(ctx, t, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr)) != LG_OK) return s;
  }
  if ((s = storage_compute_gae(ctx, nullptr, nullptr)) != LG_OK) return s;
  return ppo_update(ctx, stats);
}

lg_status lg_graph_capture_iteration(lg_ctx* ctx, lg_update_stats* stats) {
  GUARD();
  if (!ctx->reset_done) return fail(ctx, LG_ERR_STATE, "graph capture before env_reset");
  {
    lg_status s0 = solo_ok(ctx, "lg_graph_capture_iteration");
    if (s0 != LG_OK) return s0;
  }
  if (ctx->gexec) { cudaGraphExecDestroy(ctx->gexec); ctx->gexec = nullptr; }
  if (ctx->graph) { cudaGraphDestroy(ctx->graph); ctx->graph = nullptr; }
  CK(cudaStreamBeginCapture(ctx->st, cudaStreamCaptureModeThreadLocal));
  ctx->capturing = true;
  ctx->pairs.clear();
  ctx->evn = 0;
  lg_status s = run_iteration(ctx, stats);
  ctx->capturing = false;
  ctx->gpairs = ctx->pairs;
  ctx->pairs.clear();
  cudaGraph_t g = nullptr;
  cudaError_t e = cudaStreamEndCapture(ctx->st, &g);
  if (s != LG_OK) return s;
  if (e != cudaSuccess) return fail(ctx, LG_ERR_CUDA, "end capture: %s", cudaGetErrorString(e));
  ctx->graph = g;
  CK(cudaGraphInstantiate(&ctx->gexec, g, 0));
  return LG_OK;
}

lg_status lg_graph_launch(lg_ctx* ctx) {
  GUARD();
  if (!ctx->gexec) return fail(ctx, LG_ERR_STATE, "no captured graph");
  CK(cudaGraphLaunch(ctx->gexec, ctx->st));
  return LG_OK;
}

lg_status lg_graph_kernel_count(lg_ctx* ctx, int32_t* n_h) {
  GUARD();
  if (!n_h) return fail(ctx, LG_ERR_INVALID_ARG, "null output");
  if (!ctx->graph) return fail(ctx, LG_ERR_STATE, "no captured graph");
  size_t n = 0;
  CK(cudaGraphGetNodes(ctx->graph, nullptr, &n));
  std::vector<cudaGraphNode_t> nodes(n);
  CK(cudaGraphGetNodes(ctx->graph, nodes.data(), &n));
  int32_t k = 0;
  for (auto& nd : nodes) {
    cudaGraphNodeType ty;
    CK(cudaGraphNodeGetType(nd, &ty));
    if (ty == cudaGraphNodeTypeKernel) ++k;
  }
  *n_h = k;
  return LG_OK;
}

lg_status lg_iterate_host(lg_ctx* ctx, const uint8_t ctrl_h[16], lg_update_stats* stats_h) {
  GUARD();
  {
    lg_status s0 = solo_ok(ctx, "lg_iterate_host");
    if (s0 != LG_OK) return s0;
  }
  if (!ctrl_h || !stats_h) return fail(ctx, LG_ERR_INVALID_ARG, "iterate_host: null host buffer");
  void* K = ctx->buf[LG_BUF_WORK];
  CK(cudaMemcpyAsync(at<uint8_t>(K, ctx->L.k_ctrl), ctrl_h, 16, cudaMemcpyHostToDevice, ctx->st));
  lg_update_stats* dstats = at<lg_update_stats>(K, ctx->L.k_stats);
  lg_status s;
  if (ctx->gexec) {
    CK(cudaGraphLaunch(ctx->gexec, ctx->st));
  } else if ((s = run_iteration(ctx, dstats)) != LG_OK) {
    return s;
  }
  CK(cudaMemcpyAsync(stats_h, dstats, sizeof(lg_update_stats), cudaMemcpyDeviceToHost, ctx->st));
  CK(cudaStreamSynchronize(ctx->st));
  return LG_OK;
}

// ------------------------------------------------------------------ multi-rank group on one device
lg_status lg_group_create(lg_ctx* const* ctxs_h, int32_t n, lg_group** out_h) {
  if (!ctxs_h || !out_h || n < 1 || n > LG_MAX_GROUP) return LG_ERR_INVALID_ARG;
  for (int r = 0; r < n; ++r)
    if (!ctxs_h[r]) return LG_ERR_INVALID_ARG;
  // validation only returns a status: a refused grouping leaves the contexts usable (no sticky error)
  for (int r = 0; r < n; ++r) {
    lg_ctx* ctx = ctxs_h[r];
    if (ctx->err != LG_OK) return ctx->err;
    if (ctx->group || ctx->comm) return LG_ERR_STATE;
    if (ctx->cfg.world_size != n || ctx->cfg.rank != r) return LG_ERR_INVALID_ARG;
    if (ctx->st != ctxs_h[0]->st) return LG_ERR_INVALID_ARG;
    lg_config a = ctx->cfg, b = ctxs_h[0]->cfg;
    a.rank = b.rank = 0;
    if (memcmp(&a, &b, sizeof(a)) != 0) return LG_ERR_INVALID_ARG;
  }
  lg_group* g = new lg_group();
  g->n = n;
  for (int r = 0; r < n; ++r) { g->cs[r] = ctxs_h[r]; ctxs_h[r]->group = g; }
  *out_h = g;
  return LG_OK;
}

lg_status lg_group_destroy(lg_group* g) {
  if (!g) return LG_ERR_INVALID_ARG;
  for (int r = 0; r < g->n; ++r)
    if (g->cs[r]) g->cs[r]->group = nullptr;
  delete g;
  return LG_OK;
}

static lg_status group_guard(lg_group* g) {
  if (!g) return LG_ERR_INVALID_ARG;
  for (int r = 0; r < g->n; ++r) {
    if (!g->cs[r]) return LG_ERR_STATE;
    if (g->cs[r]->err != LG_OK) return g->cs[r]->err;
  }
  return LG_OK;
}

lg_status lg_group_broadcast_params(lg_group* g) {
  lg_status s = group_guard(g);
  if (s != LG_OK) return s;
  lg_ctx* c0 = g->cs[0];
  for (int r = 1; r < g->n; ++r) {
    lg_ctx* ctx = g->cs[r];
    CK(cudaMemcpyAsync(ctx->buf[LG_BUF_THETA], c0->buf[LG_BUF_THETA], (size_t)ctx->d.P * 4, cudaMemcpyDeviceToDevice,
                       ctx->st));
    launch_sync_shadow(ctx->shadow, reinterpret_cast<const float*>(ctx->buf[LG_BUF_THETA]), ctx->st);
    CKL();
  }
  return LG_OK;
}

lg_status lg_group_compute_gae(lg_group* g) {
  lg_status s = group_guard(g);
  if (s != LG_OK) return s;
  return run_gae(g->cs, g->n, nullptr, nullptr);
}

lg_status lg_group_ppo_update(lg_group* g, lg_update_stats* const* stats_h) {
  lg_status s = group_guard(g);
  if (s != LG_OK) return s;
  return run_update(g->cs, g->n, stats_h);
}

lg_status lg_group_iterate(lg_group* g, lg_update_stats* const* stats_h) {
  lg_status s = group_guard(g);
  if (s != LG_OK) return s;
  for (int r = 0; r < g->n; ++r) {
    lg_ctx* ctx = g->cs[r];
    if (!ctx->reset_done) return fail(ctx, LG_ERR_STATE, "lg_group_iterate before env_reset");
    for (int t = 0; t < ctx->d.T; ++t) {
      if ((s = policy_act(ctx, t, nullptr, nullptr, nullptr, nullptr)) != LG_OK) return s;
      if ((s = env_step_obs_reward(ctx, t, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr)) != LG_OK) return s;
    }
  }
  if ((s = run_gae(g->cs, g->n, nullptr, nullptr)) != LG_OK) return s;
  return run_update(g->cs, g->n, stats_h);
}

lg_status lg_profile(lg_ctx* ctx, int32_t enable) {
  GUARD();
  if (enable && ctx->ev.empty()) {
    ctx->ev.resize(8192);
    for (auto& e : ctx->ev) CK(cudaEventCreate(&e));
  }
  ctx->prof = enable != 0;
  ctx->pairs.clear();
  ctx->evn = 0;
  return LG_OK;
}

lg_status lg_profile_read(lg_ctx* ctx, float* ms_h, int32_t* count_h, int32_t n) {
  GUARD();
  if (!ms_h || !count_h || n < 1) return fail(ctx, LG_ERR_INVALID_ARG, "profile_read: bad arguments");
  const bool eager = !ctx->pairs.empty();
  const auto& pl = eager ? ctx->pairs : ctx->gpairs;
  for (const auto& p : pl) {
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, ctx->ev[p.a], ctx->ev[p.b]));
    if (p.cat < n) { ms_h[p.cat] += ms; count_h[p.cat] += 1; }
  }
  if (eager) { ctx->pairs.clear(); ctx->evn = 0; }
  return LG_OK;
}

lg_status lg_adv_normalization(lg_ctx* ctx, double* mean_h, double* inv_std_h) {
  GUARD();
  if (!mean_h || !inv_std_h) return fail(ctx, LG_ERR_INVALID_ARG, "null output");
  DevScalars s;
  CK(cudaMemcpyAsync(&s, ctx->sc, sizeof(s), cudaMemcpyDeviceToHost, ctx->st));
  CK(cudaStreamSynchronize(ctx->st));
  *mean_h = s.adv_mean;
  *inv_std_h = s.adv_inv_std;
  return LG_OK;
}

lg_status lg_device_scalars(lg_ctx* ctx, int32_t* out8_h) {
  GUARD();
  if (!out8_h) return fail(ctx, LG_ERR_INVALID_ARG, "null output");
  DevScalars s;
  CK(cudaMemcpyAsync(&s, ctx->sc, sizeof(s), cudaMemcpyDeviceToHost, ctx->st));
  CK(cudaStreamSynchronize(ctx->st));
  out8_h[0] = (int32_t)s.s_base; out8_h[1] = (int32_t)s.iteration; out8_h[2] = s.adam_t;
  memcpy(&out8_h[3], &s.alpha, 4);
  out8_h[4] = s.n_to_total; out8_h[5] = s.nonfinite_skips; out8_h[6] = s.applied;
  memcpy(&out8_h[7], &s.kl_last, 4);
  return LG_OK;
}

}  // extern "C"
