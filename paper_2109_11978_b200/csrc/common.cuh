// common.cuh -- device helpers of libleggedrl (written from DESIGN.md §3.1-§3.3; independent of oracle/).
#pragma once
#include <cstdint>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

namespace lg {

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

constexpr int NW = 66;  // state words per env
constexpr uint32_t TAG_RESET = 1u, TAG_OBS = 2u, TAG_ACTION = 3u, TAG_PUSH = 4u, TAG_CURR = 5u, TAG_SHUFFLE = 6u,
                   TAG_TERRAIN = 8u;
constexpr uint32_t F_CURRICULUM = 1u, F_NOISE = 2u, F_PUSH = 4u, F_BOOTSTRAP = 8u;

// state word indices
enum : int {
  S_P = 0, S_QUAT = 3, S_V = 7, S_W = 10, S_Q = 13, S_QD = 25, S_TAIR = 37, S_CMD = 41, S_APREV = 44, S_MU = 56,
  S_SPAWN = 57, S_CONTACT = 59, S_PUSH = 60, S_EPSTEP = 61, S_LEVEL = 62, S_COL = 63, S_CROSSED = 64, S_EPRET = 65
};

// device-resident scalars in the WORK buffer
struct DevScalars {
  uint32_t s_base;      // env step counter base: step t of the iteration uses s_base+t+1
  uint32_t iteration;   // PPO iterations completed (shuffle event = iteration*E + epoch)
  int32_t adam_t;       // applied Adam steps
  float alpha;          // Alg. 1 learning rate
  int32_t reserved0;
  int32_t nonfinite_skips;
  int32_t applied;
  int32_t pad0;
  double adv_mean, adv_inv_std;  // normalisation of the current batch
  float kl_last, pad1;
  // per-iteration episode statistics (accumulated by env steps): integer and fixed-point sums, so the totals do
  // not depend on the order in which the envs' atomics land (SPEC S:414 determinism)
  long long ep_return_fx;  // sum of finished episodes' returns, fixed point with 24 fraction bits
  long long ep_len_sum;    // sum of finished episodes' lengths (steps)
  int32_t episodes, promotions, demotions;
  int32_t nonfinite_envs;  // env steps whose state went non-finite (forced terminated + reset)
  int32_t level_hist[16];
  // Alg. 1 / Adam state per minibatch slot m of the iteration (read slot m&1, write slot (m+1)&1)
  float alpha_ring[2];
  int32_t adamt_ring[2];
  int32_t n_to_total;   // time-out rows compacted since the rollout began (batched bootstrap)
  float bc_ring[2][2];  // Adam bias corrections {1 - b1^t, 1 - b2^t} for minibatch slot m (read bc_ring[m & 1],
                        // written for slot m + 1 by Adam of slot m; slot 0 by iter_begin)
  int32_t n_to_slot[2]; // compacted time-out rows of env step event ev in slot ev & 1 (the step clears the other)
};

// ------------------------------------------------------------------ Philox4x32-10
struct U4 { uint32_t x, y, z, w; };

__device__ __forceinline__ U4 philox(uint32_t k0, uint32_t k1, uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    uint32_t hi0 = __umulhi(0xD2511F53u, c0), lo0 = 0xD2511F53u * c0;
    uint32_t hi1 = __umulhi(0xCD9E8D57u, c2), lo1 = 0xCD9E8D57u * c2;
    uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
    k0 += 0x9E3779B9u; k1 += 0xBB67AE85u;
  }
  return U4{c0, c1, c2, c3};
}

__device__ __forceinline__ uint32_t pick(const U4& u, uint32_t w) {
  return (w & 3u) == 0 ? u.x : (w & 3u) == 1 ? u.y : (w & 3u) == 2 ? u.z : u.w;
}

struct Rng {
  uint32_t k0, k1;
  __device__ __forceinline__ U4 block(uint32_t b, uint32_t id, uint32_t event, uint32_t tag) const {
    return philox(k0, k1, b, id, event, tag);
  }
  __device__ __forceinline__ uint32_t word(uint32_t id, uint32_t event, uint32_t tag, uint32_t w) const {
    return pick(philox(k0, k1, w >> 2, id, event, tag), w);
  }
};

__device__ __forceinline__ float u01(uint32_t x) { return __fmul_rn((float)(x >> 8), 0x1p-24f); }
__device__ __forceinline__ float usym(float s, uint32_t x) {
  float t = __fsub_rn(__fmul_rn(2.0f, u01(x)), 1.0f);
  return __fmul_rn(s, t);
}

// ------------------------------------------------------------------ polynomials
// (this translation unit family is compiled with -fmad=false; the explicit _rn intrinsics below
//  keep the no-contraction rule even if a file forgets the flag)
__device__ __forceinline__ float fm(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ float fa(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float fs(float a, float b) { return __fsub_rn(a, b); }

__device__ __forceinline__ void sincos_poly(float x, float& sn, float& cs) {
  float k = rintf(fm(x, 0x1.45f306p-1f));
  float r = fs(fs(x, fm(k, 0x1.92p0f)), fm(k, 0x1.fb5444p-12f));
  float r2 = fm(r, r);
  float ps = fa(fm(fa(fm(fa(fm(0x1.71de3ap-19f, r2), -0x1.a01a02p-13f), r2), 0x1.111112p-7f), r2), -0x1.555556p-3f);
  float s = fa(r, fm(fm(r, r2), ps));
  float pc = fa(fm(fa(fm(fa(fm(fa(fm(-0x1.27e4fcp-22f, r2), 0x1.a01a02p-16f), r2), -0x1.6c16c2p-10f), r2), 0x1.555556p-5f), r2), -0x1p-1f);
  float c = fa(1.0f, fm(r2, pc));
  int q = ((int)k) & 3;
  if (q == 0) { sn = s; cs = c; }
  else if (q == 1) { sn = c; cs = -s; }
  else if (q == 2) { sn = -s; cs = -c; }
  else { sn = -c; cs = s; }
}

__device__ __forceinline__ float clampf_(float v, float lo, float hi) { return fminf(fmaxf(v, lo), hi); }

__device__ __forceinline__ float exp_poly(float x) {
  x = clampf_(x, -87.0f, 88.0f);
  float k = rintf(fm(x, 0x1.715476p0f));
  float r = fs(fs(x, fm(k, 0x1.62e4p-1f)), fm(k, 0x1.7f7d1cp-20f));
  float p = 0x1.a01a02p-13f;
  p = fa(fm(p, r), 0x1.6c16c2p-10f);
  p = fa(fm(p, r), 0x1.111112p-7f);
  p = fa(fm(p, r), 0x1.555556p-5f);
  p = fa(fm(p, r), 0x1.555556p-3f);
  p = fa(fm(p, r), 0x1p-1f);
  p = fa(fm(p, r), 1.0f);
  p = fa(fm(p, r), 1.0f);
  int ki = (int)k;
  float two_k = __int_as_float((ki + 127) << 23);
  return fm(p, two_k);
}

__device__ __forceinline__ float log_poly(float x) {
  uint32_t bits = __float_as_uint(x);
  int e = (int)((bits >> 23) & 255u) - 127;
  float m = __uint_as_float((bits & 0x7fffffu) | 0x3f800000u);
  if (m > 0x1.6a09e6p0f) { m = fm(m, 0.5f); e = e + 1; }
  float s = __fdiv_rn(fs(m, 1.0f), fa(m, 1.0f));
  float s2 = fm(s, s);
  float p = fa(fm(fa(fm(fa(fm(fa(fm(s2, 0x1.c71c72p-4f), 0x1.24924ap-3f), s2), 0x1.99999ap-3f), s2), 0x1.555556p-2f), s2), 1.0f);
  return fa(fm(fm(2.0f, s), p), fm((float)e, 0x1.62e43p-1f));
}

// ------------------------------------------------------------------ height lookups
struct World {
  const float* hf;
  int R, C;
  float inv_cell;
};

__device__ __forceinline__ float h_plate(const World& w, float x, float y) {
  float fx = clampf_(fm(x, w.inv_cell), 0.0f, (float)w.R);
  float fy = clampf_(fm(y, w.inv_cell), 0.0f, (float)w.C);
  int i = (int)ceilf(fx) - 1;
  int j = (int)ceilf(fy) - 1;
  i = min(max(i, 0), w.R - 1);
  j = min(max(j, 0), w.C - 1);
  return __ldg(w.hf + (size_t)i * w.C + j);
}

__device__ __forceinline__ float h_bilinear(const World& w, float x, float y) {
  float fx = clampf_(fs(fm(x, w.inv_cell), 0.5f), 0.0f, (float)(w.R - 1));
  float fy = clampf_(fs(fm(y, w.inv_cell), 0.5f), 0.0f, (float)(w.C - 1));
  int i0 = min((int)floorf(fx), w.R - 2);
  int j0 = min((int)floorf(fy), w.C - 2);
  float tx = fs(fx, (float)i0), ty = fs(fy, (float)j0);
  const float* r0 = w.hf + (size_t)i0 * w.C + j0;
  const float* r1 = r0 + w.C;
  float h00 = __ldg(r0), h01 = __ldg(r0 + 1), h10 = __ldg(r1), h11 = __ldg(r1 + 1);
  float omx = fs(1.0f, tx);
  float lo = fa(fm(omx, h00), fm(tx, h10));
  float hi = fa(fm(omx, h01), fm(tx, h11));
  return fa(fm(fs(1.0f, ty), lo), fm(ty, hi));
}

// ------------------------------------------------------------------ Gaussian policy arithmetic
// Written with explicit roundings so every kernel that evaluates them (rollout heads, fused rollout policy,
// loss head) produces the same bits regardless of the translation unit's contraction choices.
// log-density term of one action dimension: 0.5 z^2 + log sigma, z = (a - mu) / sigma
__device__ __forceinline__ float logp_term_e(float a, float mu, float einv, float ls) {  // einv = expf(-ls)
  const float z = __fmul_rn(__fsub_rn(a, mu), einv);
  return __fadd_rn(__fmul_rn(__fmul_rn(0.5f, z), z), ls);
}
__device__ __forceinline__ float logp_term(float a, float mu, float ls) { return logp_term_e(a, mu, expf(-ls), ls); }
// action of dimension j from the ACTION Philox block j/4 of env g at event ev: a = mu + sigma * eps,
// eps = Box-Muller pair (2k, 2k+1), k = j/2 (cos for even j, sin for odd j)
// sigma * eps of that sample (independent of mu: the rollout policy computes it before its layers finish)
__device__ __forceinline__ float action_noise_b(const U4& b, int j, float ls) {  // b = block j/4
  const int k2 = (j & ~1) & 3;
  const uint32_t w0 = pick(b, (uint32_t)k2), w1 = pick(b, (uint32_t)k2 + 1u);
  const float u1 = (float)((w0 >> 8) + 1u) * 0x1p-24f;
  const float u2 = (float)(w1 >> 8) * 0x1p-24f;
  const float rr = sqrtf(-2.0f * log_poly(u1));
  float sn, cs;
  sincos_poly(0x1.921fb6p2f * u2, sn, cs);
  return __fmul_rn(expf(ls), __fmul_rn(rr, (j & 1) ? sn : cs));
}
__device__ __forceinline__ float sample_action_b(const U4& b, int j, float mu, float ls) {  // b = block j/4
  return __fadd_rn(mu, action_noise_b(b, j, ls));
}
__device__ __forceinline__ float sample_action(const Rng& rng, uint32_t g, uint32_t ev, int j, float mu, float ls) {
  return sample_action_b(rng.block((uint32_t)(j >> 2), g, ev, TAG_ACTION), j, mu, ls);
}

// ------------------------------------------------------------------ PPO loss of one sample
// Shared by the two loss-head kernels (k_loss_heads, and the layer-3 GEMM's loss epilogue), so the per-row
// quantities that feed dZ3 -- dL/dlogp and dL/dV -- are the same expressions (the same bits) on both paths.
// Clipped surrogate: returns dL/dlogp = -(A or 0) ratio / M; sv = the row's surrogate term.
__device__ __forceinline__ float ppo_dlogp(float ratio, float adv, float clip, float invM, float& sv, bool& clipped) {
  const float s1 = ratio * adv;
  const float rc = fminf(fmaxf(ratio, 1.0f - clip), 1.0f + clip);
  const float s2 = rc * adv;
  const bool take1 = s1 <= s2;
  const bool inside = ratio >= 1.0f - clip && ratio <= 1.0f + clip;
  sv = take1 ? s1 : s2;
  clipped = fabsf(ratio - 1.0f) > clip;
  return -(take1 ? adv : (inside ? adv : 0.0f)) * invM * ratio;
}
// PPO2 clipped value loss (reading R14): returns dL/dV; vv = the row's value-loss term
__device__ __forceinline__ float ppo_dvalue(float V, float Vo, float ret, float vclip, float vf_coef, float invM,
                                            float& vv) {
  const float vc = Vo + fminf(fmaxf(V - Vo, -vclip), vclip);
  const float e1 = (V - ret) * (V - ret), e2 = (vc - ret) * (vc - ret);
  const bool take_u = e1 >= e2;
  const bool vin = fabsf(V - Vo) <= vclip;
  vv = take_u ? e1 : e2;
  return vf_coef * (take_u ? 2.0f * (V - ret) : (vin ? 2.0f * (vc - ret) : 0.0f)) * invM;
}
// analytic KL(pi_old || pi) of one action dimension (reading R15): klc = the mu-independent part
__device__ __forceinline__ float kl_const(float ls, float lso, float iv) {
  return ls - lso + expf(2.0f * lso) * (0.5f * iv) - 0.5f;
}
__device__ __forceinline__ float kl_term(float klc, float dm, float iv) { return klc + dm * dm * (0.5f * iv); }
// d(-logp)/d(log sigma_j) factor of one dimension, times dL/dlogp
__device__ __forceinline__ float gls_term(float dLdlp, float d, float iv) { return dLdlp * (d * d * iv - 1.0f); }
// the 12-dimension sum of the warp-per-row kernels' dim_sum (term j on lane 2j, butterfly offsets 16..1),
// evaluated by one thread in the same addition order
__device__ __forceinline__ float dim_sum12(const float* t) {
  float e8[8];
#pragma unroll
  for (int m = 0; m < 4; ++m) e8[m] = t[m] + t[m + 8];
#pragma unroll
  for (int m = 4; m < 8; ++m) e8[m] = t[m] + 0.0f;
#pragma unroll
  for (int m = 0; m < 4; ++m) e8[m] = e8[m] + e8[m + 4];
  e8[0] = e8[0] + e8[2];
  e8[1] = e8[1] + e8[3];
  return (e8[0] + e8[1]) + 0.0f;
}

// ------------------------------------------------------------------ programmatic dependent launch
// Kernels launched with launch_pdl (kernels.h) let their dependent grid start launching as soon as all their
// CTAs are running (pdl_trigger), and block in pdl_wait until the preceding grid has completed and its memory
// is visible -- every such kernel calls pdl_wait before touching data a predecessor wrote, so completion stays
// transitive along the stream. Without the launch attribute both are no-ops.
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// ------------------------------------------------------------------ misc
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

}  // namespace lg
