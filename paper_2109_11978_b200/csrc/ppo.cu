// ppo.cu -- policy heads + Gaussian sampling, PPO loss head (fwd+bwd), GAE reverse scan, advantage
// statistics, Feistel shuffle, minibatch gather, deterministic gradient reductions, Alg. 1 + Adam.
// (§2.2, Table 3, Alg. 1; SPEC ppo/net.)
// Memory-bound kernels: one thread (or warp) per row/env, coalesced along the contiguous dimension;
// every cross-thread reduction uses a fixed tree order so results are run-to-run deterministic.
#include <algorithm>

#include "common.cuh"
#include "kernels.h"

namespace lg {

constexpr float SIX_LN_2PI = 11.027262398456072f;
constexpr float HALF_LN_2PI = 0.9189385332046727f;

// ------------------------------------------------------------------ heads (one warp per row)
// Lane l owns the H3 columns [4l, 4l+4) of the actor and of the critic half (H2 <= 128, a multiple of 32)
// and keeps the matching head weights in registers. The 13 head dot products (12 action means + value)
// are reduced over the warp by a 16-value butterfly (offsets 16, 8, 4, 2 halve the value set, offset 1
// finishes), after which lanes 2v and 2v+1 both hold total v (bit-identical: a+b == b+a). Lane 2j then
// owns action dimension j. The rollout (k_heads) and the update (k_loss_heads) use the same functions, so
// the ratio of the first minibatch of an iteration is exactly 1.
struct HeadRegs {
  float wa[12][4];
  float wc[4];
};

__device__ __forceinline__ void load_head_regs(const float* W4a, const float* W4c, int H2, int lane, HeadRegs& w) {
  const int c0 = 4 * lane;
  const bool on = c0 < H2;
#pragma unroll
  for (int j = 0; j < 12; ++j) {
    const float4 v = on ? *reinterpret_cast<const float4*>(W4a + j * H2 + c0) : make_float4(0.f, 0.f, 0.f, 0.f);
    w.wa[j][0] = v.x; w.wa[j][1] = v.y; w.wa[j][2] = v.z; w.wa[j][3] = v.w;
  }
  const float4 v = on ? *reinterpret_cast<const float4*>(W4c + c0) : make_float4(0.f, 0.f, 0.f, 0.f);
  w.wc[0] = v.x; w.wc[1] = v.y; w.wc[2] = v.z; w.wc[3] = v.w;
}

// this lane's 4 actor and 4 critic columns of row `hrow` (zeros for lanes beyond H2)
__device__ __forceinline__ void load_h3(const __nv_bfloat16* hrow, int H2, int lane, float* ha, float* hc) {
  const int c0 = 4 * lane;
  uint2 ua = make_uint2(0u, 0u), uc = make_uint2(0u, 0u);
  if (c0 < H2) {
    ua = *reinterpret_cast<const uint2*>(hrow + c0);
    uc = *reinterpret_cast<const uint2*>(hrow + H2 + c0);
  }
  float2 t;
  t = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&ua.x)); ha[0] = t.x; ha[1] = t.y;
  t = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&ua.y)); ha[2] = t.x; ha[3] = t.y;
  t = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&uc.x)); hc[0] = t.x; hc[1] = t.y;
  t = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&uc.y)); hc[2] = t.x; hc[3] = t.y;
}

// returns, on lanes 2v and 2v+1, the warp total of head product v (v < 12: mu_v - b4a_v; v = 12: V - b4c)
__device__ __forceinline__ float head_fwd_warp(const HeadRegs& w, const float* ha, const float* hc, int lane) {
  float v[16];
#pragma unroll
  for (int j = 0; j < 12; ++j) {
    float p = w.wa[j][0] * ha[0];
    p = fmaf(w.wa[j][1], ha[1], p);
    p = fmaf(w.wa[j][2], ha[2], p);
    v[j] = fmaf(w.wa[j][3], ha[3], p);
  }
  {
    float p = w.wc[0] * hc[0];
    p = fmaf(w.wc[1], hc[1], p);
    p = fmaf(w.wc[2], hc[2], p);
    v[12] = fmaf(w.wc[3], hc[3], p);
  }
  v[13] = v[14] = v[15] = 0.0f;
#pragma unroll
  for (int half = 8, off = 16; half >= 1; half >>= 1, off >>= 1) {
    const bool up = (lane & off) != 0;
#pragma unroll
    for (int i = 0; i < half; ++i) {
      const float send = up ? v[i] : v[i + half];
      const float keep = up ? v[i + half] : v[i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, off);
    }
  }
  return v[0] + __shfl_xor_sync(0xffffffffu, v[0], 1);
}

// sum over the action-dimension lanes (2j, j < 12) of x; fixed butterfly order, result on every lane
__device__ __forceinline__ float dim_sum(float x, int lane) {
  float s = (lane < 24 && (lane & 1) == 0) ? x : 0.0f;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  return s;
}

// log N(a | mu, exp(ls)) from the per-dimension lanes
__device__ __forceinline__ float logp_warp(float a_j, float mu_j, float ls_j, int lane) {
  return __fsub_rn(-dim_sum(logp_term(a_j, mu_j, ls_j), lane), SIX_LN_2PI);
}

constexpr int HEAD_WARPS = 8;      // rollout heads: warps per block
constexpr int HEAD_ROWS_PER_WARP = 4;

__global__ void __launch_bounds__(HEAD_WARPS * 32) k_heads(HeadArgs a) {
  pdl_trigger();
  pdl_wait();
  const int M = a.M_dev ? *a.M_dev : a.M;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int r0 = (blockIdx.x * HEAD_WARPS + warp) * HEAD_ROWS_PER_WARP;
  if (r0 >= M) return;  // warp-uniform (empty bootstrap launches)
  const int H2 = a.nd.H2;
  HeadRegs w;
  load_head_regs(a.W4a, a.W4c, H2, lane, w);
  const int j = lane >> 1;  // this lane's head output (valid for j <= 12)
  const float bias = j < 12 ? __ldg(a.b4a + j) : (j == 12 ? __ldg(a.b4c) : 0.0f);
  const float ls = j < 12 ? __ldg(a.logstd + j) : 0.0f;
  const int rend = min(r0 + HEAD_ROWS_PER_WARP, M);
  for (int r = r0; r < rend; ++r) {
    float ha[4], hc[4];
    load_h3(a.H3 + (size_t)r * 2 * H2, H2, lane, ha, hc);
    const float tot = head_fwd_warp(w, ha, hc, lane) + bias;  // lanes 2j: mu_j; lanes 24, 25: V
    const float V = __shfl_sync(0xffffffffu, tot, 24);
    const bool dl = lane < 24 && (lane & 1) == 0;               // dimension-owner lane
    if (a.mode == 1) {  // value scatter (time-out bootstrap or V(o_T))
      if (lane == 0) a.value[a.idx ? a.idx[r] : r] = V;
      continue;
    }
    if (a.mode == 2) {
      if (dl) a.mu[(size_t)r * 12 + j] = tot;
      if (lane == 0) a.value[r] = V;
      continue;
    }
    // act: a_j = mu_j + sigma_j eps_j, eps = Box-Muller pairs (2k, 2k+1) of the ACTION stream
    float act = 0.0f;
    if (dl) {
      Rng rng{a.seed_lo, a.seed_hi};
      act = a.deterministic ? tot
                            : sample_action(rng, (uint32_t)(a.rank * a.N + r), a.scalars->s_base + (uint32_t)a.t + 1u,
                                            j, tot, ls);
    }
    const float lp = logp_warp(act, tot, ls, lane);
    const size_t o = (size_t)r * 12 + j;
    if (dl) {
      a.act[o] = act;
      a.mu[o] = tot;
      if (a.u_act) a.u_act[o] = act;
      if (a.u_mu) a.u_mu[o] = tot;
    }
    if (lane == 0) {
      a.logp[r] = lp;
      a.value[r] = V;
      if (a.u_logp) a.u_logp[r] = lp;
      if (a.u_value) a.u_value[r] = V;
    }
  }
}

void launch_heads(const HeadArgs& a, cudaStream_t st) {
  const int rows_per_block = HEAD_WARPS * HEAD_ROWS_PER_WARP;
  launch_pdl(k_heads, dim3((a.M + rows_per_block - 1) / rows_per_block), dim3(HEAD_WARPS * 32), 0, st, a);
}

// ------------------------------------------------------------------ PPO loss head (fwd + bwd)
// Warp per row (head_fwd_warp), rows strided over all warps of the grid (fixed assignment). Each lane keeps
// its slice of the head/log-std gradients in registers (dW4a[12][4 cols], dW4c[4 cols]; lanes 2j: db4a_j,
// dlogstd_j; lane 0: db4c and the loss statistics in fp64) summed over its warp's rows in order; the warps
// of a block are then summed in warp order into the block partial (k_reduce_heads sums blocks in order).
constexpr int LOSS_WARPS = 12;       // one block per SM
constexpr int LOSS_MAX_BLOCKS = 148;
int loss_head_partial_floats(int H2) { return ((13 * H2 + 25) + 3) / 4 * 4; }
int loss_blocks(int M) { return std::max(1, std::min(LOSS_MAX_BLOCKS, (M + LOSS_WARPS - 1) / LOSS_WARPS)); }

__device__ __forceinline__ float elu_grad_from_out(float h) { return h > 0.0f ? 1.0f : h + 1.0f; }

__global__ void __launch_bounds__(LOSS_WARPS * 32, 1) k_loss_heads(LossArgs a) {
  pdl_trigger();
  pdl_wait();
  // first payload writer of the minibatch: clear the atomically accumulated non-finite counter (the other
  // slots are assigned by k_reduce_heads); the previous minibatch's Adam has consumed the payload already
  if (a.payload && blockIdx.x == 0 && threadIdx.x == 0) a.payload[4] = 0.0f;
  extern __shared__ float sacc[];  // [LOSS_WARPS][HP] warp partials, then [LOSS_WARPS][5] fp64 statistics
  const int H2 = a.nd.H2, HP = a.HP;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int gw = blockIdx.x * LOSS_WARPS + warp, TW = gridDim.x * LOSS_WARPS;
  HeadRegs w;
  load_head_regs(a.W4a, a.W4c, H2, lane, w);
  const int j = lane >> 1;
  const bool dl = lane < 24 && (lane & 1) == 0;
  const float bias = j < 12 ? __ldg(a.b4a + j) : (j == 12 ? __ldg(a.b4c) : 0.0f);
  const float ls = j < 12 ? __ldg(a.logstd + j) : 0.0f;
  const float lso = j < 12 ? __ldg(a.logstd_old + j) : 0.0f;
  const float iv = expf(-2.0f * ls);
  const float klc = kl_const(ls, lso, iv);  // KL terms independent of mu
  const float invM = 1.0f / (float)a.M;
  float gWa[12][4], gWc[4];
#pragma unroll
  for (int jj = 0; jj < 12; ++jj) gWa[jj][0] = gWa[jj][1] = gWa[jj][2] = gWa[jj][3] = 0.0f;
  gWc[0] = gWc[1] = gWc[2] = gWc[3] = 0.0f;
  float gb = 0.0f, gls = 0.0f, gbv = 0.0f;           // lanes 2j: db4a_j, dlogstd_j; lane 0: db4c
  double st0 = 0.0, st1 = 0.0, st2 = 0.0, st3 = 0.0, st4 = 0.0;
  // the next row's inputs are loaded while this row is computed (software pipelining: the row loop is
  // otherwise bound by the latency of its own loads)
  uint2 nua = make_uint2(0u, 0u), nuc = make_uint2(0u, 0u);
  float nact = 0.0f, nmuo = 0.0f, nlpo = 0.0f, nadv = 0.0f, nVo = 0.0f, nret = 0.0f;
  auto fetch = [&](int r) {
    if (r >= a.M) return;
    const __nv_bfloat16* hrow = a.H3 + (size_t)r * 2 * H2;
    if (4 * lane < H2) {
      nua = __ldg(reinterpret_cast<const uint2*>(hrow + 4 * lane));
      nuc = __ldg(reinterpret_cast<const uint2*>(hrow + H2 + 4 * lane));
    }
    nact = dl ? __ldg(a.act + (size_t)r * 12 + j) : 0.0f;
    nmuo = dl ? __ldg(a.mu_old + (size_t)r * 12 + j) : 0.0f;
    nlpo = __ldg(a.logp_old + r); nadv = __ldg(a.adv + r); nVo = __ldg(a.V_old + r); nret = __ldg(a.ret + r);
  };
  fetch(gw);
  for (int r = gw; r < a.M; r += TW) {
    const uint2 ua = nua, uc = nuc;
    const float act = nact, muo = nmuo, lpo = nlpo, adv = nadv, Vo = nVo, ret = nret;
    fetch(r + TW);
    float ha[4], hc[4];
    {
      float2 t2;
      t2 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&ua.x)); ha[0] = t2.x; ha[1] = t2.y;
      t2 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&ua.y)); ha[2] = t2.x; ha[3] = t2.y;
      t2 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&uc.x)); hc[0] = t2.x; hc[1] = t2.y;
      t2 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&uc.y)); hc[2] = t2.x; hc[3] = t2.y;
    }
    const float tot = head_fwd_warp(w, ha, hc, lane) + bias;
    const float V = __shfl_sync(0xffffffffu, tot, 24);
    const float lp = logp_warp(act, tot, ls, lane);
    // clipped surrogate (§2.2 / DESIGN.md §3.11); every lane evaluates the row scalars
    const float ratio = expf(lp - lpo);
    float svf, vvf;
    bool clipped;
    const float dLdlp = ppo_dlogp(ratio, adv, a.clip, invM, svf, clipped);
    const float dV = ppo_dvalue(V, Vo, ret, a.vclip, a.vf_coef, invM, vvf);
    const float d = act - tot;
    const float dmu = dLdlp * d * iv;
    const float dm = muo - tot;
    const float kl = dim_sum(kl_term(klc, dm, iv), lane);
    if (dl) {
      gb = gb + dmu;
      gls = gls + gls_term(dLdlp, d, iv);
    }
    if (lane == 0) {
      gbv = gbv + dV;
      const double sv = (double)svf, vv = (double)vvf, kv = (double)kl;
      st0 += sv; st1 += vv; st2 += kv;
      st3 += clipped ? 1.0 : 0.0;
      st4 += (isfinite(sv) && isfinite(vv) && isfinite(kv)) ? 0.0 : 1.0;
    }
    // dH3 = W4a^T dmu (actor), dV w4c (critic); dZ3 = dH3 * ELU'(H3); dW4 += dY h
    float dmuj[12];
#pragma unroll
    for (int jj = 0; jj < 12; ++jj) dmuj[jj] = __shfl_sync(0xffffffffu, dmu, 2 * jj);
    float za[4], zc[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      float acc = 0.0f;
#pragma unroll
      for (int jj = 0; jj < 12; ++jj) {
        acc = fmaf(dmuj[jj], w.wa[jj][e], acc);
        gWa[jj][e] = fmaf(dmuj[jj], ha[e], gWa[jj][e]);
      }
      za[e] = acc * elu_grad_from_out(ha[e]);
      zc[e] = dV * w.wc[e] * elu_grad_from_out(hc[e]);
      gWc[e] = fmaf(dV, hc[e], gWc[e]);
    }
    if (4 * lane < H2) {
      __nv_bfloat16* dz = a.dZ3 + (size_t)r * 2 * H2 + 4 * lane;
      const __nv_bfloat162 a0 = __floats2bfloat162_rn(za[0], za[1]), a1 = __floats2bfloat162_rn(za[2], za[3]);
      const __nv_bfloat162 c0 = __floats2bfloat162_rn(zc[0], zc[1]), c1 = __floats2bfloat162_rn(zc[2], zc[3]);
      *reinterpret_cast<uint2*>(dz) = make_uint2(*reinterpret_cast<const uint32_t*>(&a0), *reinterpret_cast<const uint32_t*>(&a1));
      *reinterpret_cast<uint2*>(dz + H2) = make_uint2(*reinterpret_cast<const uint32_t*>(&c0), *reinterpret_cast<const uint32_t*>(&c1));
    }
  }
  // warp partials -> smem (partial layout: W4a [12][H2], b4a [12], W4c [H2], b4c, logstd [12])
  float* my = sacc + warp * HP;
  if (4 * lane < H2) {
#pragma unroll
    for (int jj = 0; jj < 12; ++jj)
      *reinterpret_cast<float4*>(my + jj * H2 + 4 * lane) = make_float4(gWa[jj][0], gWa[jj][1], gWa[jj][2], gWa[jj][3]);
    *reinterpret_cast<float4*>(my + 12 * H2 + 12 + 4 * lane) = make_float4(gWc[0], gWc[1], gWc[2], gWc[3]);
  }
  if (dl) { my[12 * H2 + j] = gb; my[13 * H2 + 13 + j] = gls; }
  if (lane == 0) {
    my[13 * H2 + 12] = gbv;
    double* sd = reinterpret_cast<double*>(sacc + LOSS_WARPS * HP) + warp * 5;
    sd[0] = st0; sd[1] = st1; sd[2] = st2; sd[3] = st3; sd[4] = st4;
  }
  __syncthreads();
  float* out = a.part + (size_t)blockIdx.x * HP;
  for (int e = threadIdx.x; e < 13 * H2 + 25; e += blockDim.x) {
    float t = sacc[e];
#pragma unroll
    for (int ww = 1; ww < LOSS_WARPS; ++ww) t = t + sacc[ww * HP + e];
    out[e] = t;
  }
  if (threadIdx.x < 5) {
    const double* sd = reinterpret_cast<const double*>(sacc + LOSS_WARPS * HP);
    double t = sd[threadIdx.x];
    for (int ww = 1; ww < LOSS_WARPS; ++ww) t += sd[ww * 5 + threadIdx.x];
    a.spart[(size_t)blockIdx.x * 8 + threadIdx.x] = t;
  }
}

void launch_loss_heads(const LossArgs& a, cudaStream_t st) {
  const size_t smem = (size_t)LOSS_WARPS * a.HP * 4 + LOSS_WARPS * 5 * 8;
  static size_t set = 0;
  if (smem > set) {
    cudaFuncSetAttribute(k_loss_heads, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    set = smem;
  }
  launch_pdl(k_loss_heads, dim3(loss_blocks(a.M)), dim3(LOSS_WARPS * 32), smem, st, a);
}

// sums over blocks (fixed order) -> canonical gradient of heads/log-std + stats payload.
// Block = 32 warps x 32 elements; warp w sums partial rows b = w, w+32, ... (in order), then lane-wise the
// 32 warp sums are added in warp order: a fixed, run-to-run deterministic tree.
constexpr int RH_WARPS = 32;
constexpr int RH_UNROLL = 8;
__global__ void __launch_bounds__(RH_WARPS * 32) k_reduce_heads(HeadReduceArgs a) {
  pdl_trigger();
  pdl_wait();
  __shared__ float ssum[RH_WARPS][33];
  const int H2 = a.H2;
  const int nval = 13 * H2 + 25;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int e = blockIdx.x * 32 + lane;
  float s = 0.0f;
  if (e < nval) {
    // partial rows b = warp, warp + 32, ... summed in order; loads issued RH_UNROLL at a time
    for (int b0 = warp; b0 < a.nblk; b0 += RH_WARPS * RH_UNROLL) {
      float v[RH_UNROLL];
#pragma unroll
      for (int u = 0; u < RH_UNROLL; ++u) {
        const int b = b0 + u * RH_WARPS;
        v[u] = b < a.nblk ? __ldg(a.part + (size_t)b * a.HP + e) : 0.0f;
      }
#pragma unroll
      for (int u = 0; u < RH_UNROLL; ++u)
        if (b0 + u * RH_WARPS < a.nblk) s = s + v[u];
    }
  }
  ssum[warp][lane] = s;
  __syncthreads();
  if (warp == 0 && e < nval) {
    float t = 0.0f;
    for (int w = 0; w < RH_WARPS; ++w) t = t + ssum[w][lane];
    long long dst;
    if (e < 12 * H2) dst = a.off_W4a + e;
    else if (e < 12 * H2 + 12) dst = a.off_b4a + (e - 12 * H2);
    else if (e < 13 * H2 + 12) dst = a.off_W4c + (e - 12 * H2 - 12);
    else if (e == 13 * H2 + 12) dst = a.off_b4c;
    else { dst = a.off_logstd + (e - 13 * H2 - 13); t = t - a.ent_coef; }
    a.grad[dst] = t;
    if (!isfinite(t)) atomicAdd(&a.payload[4], 1.0f);
  }
  if (blockIdx.x == 0 && warp >= 1 && warp <= 5) {  // loss statistics: warp 1 + k sums statistic k
    const int k = warp - 1;
    const double invM = 1.0 / (double)a.M;
    double v = 0.0;
    for (int b0 = lane; b0 < a.nblk; b0 += 32 * RH_UNROLL) {
      double x[RH_UNROLL];
#pragma unroll
      for (int u = 0; u < RH_UNROLL; ++u) {
        const int b = b0 + 32 * u;
        x[u] = b < a.nblk ? a.spart[(size_t)b * 8 + k] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < RH_UNROLL; ++u) v += x[u];
    }
    v = warp_sum_d(v);
    if (lane == 0) {
      if (k == 0) a.payload[1] = (float)(v * invM);       // surrogate mean
      if (k == 1) a.payload[2] = (float)(v * invM);       // value loss mean
      if (k == 2) a.payload[0] = (float)(v * invM);       // KL mean (Alg. 1)
      if (k == 3) a.payload[3] = (float)(v * invM);       // clip fraction
      if (k == 4 && v > 0.0) atomicAdd(&a.payload[4], (float)v);
      if (k == 0) a.payload[5] = 1.0f;                    // rank count (allreduce sums it)
    }
  }
}

void launch_reduce_heads(const HeadReduceArgs& a, cudaStream_t st) {
  int n = 13 * a.H2 + 25;
  launch_pdl(k_reduce_heads, dim3((n + 31) / 32), dim3(RH_WARPS * 32), 0, st, a);
}

// split-K partials -> canonical W and b gradients. Block = 8 warps x 32 consecutive elements; warp w
// sums splits s = w, w+8, ... in order, then the 8 warp sums are added in warp order (deterministic).
__global__ void __launch_bounds__(256) k_reduce_dw(DwReduceArgs a) {
  __shared__ float ssum[8][33];
  const int z = blockIdx.z;
  const int per = a.cols + 1;  // cols + bias column
  const int total = a.rows * per;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int e = blockIdx.x * 32 + lane;
  float s = 0.0f;
  int r = 0, c = 0;
  if (e < total) {
    r = e / per;
    c = e - r * per;
    const int pc = c < a.cols ? c : a.bias_col;
    const float* p = a.part + z * a.zstride + (size_t)r * a.ld + pc;
    for (int k = warp; k < a.S; k += 8) s = s + __ldg(p + (size_t)k * a.sstride);
  }
  ssum[warp][lane] = s;
  __syncthreads();
  if (warp == 0 && e < total) {
    float t = 0.0f;
#pragma unroll
    for (int w = 0; w < 8; ++w) t = t + ssum[w][lane];
    int zz = z, rr = r;
    if (a.row_split > 0 && r >= a.row_split) { zz = 1; rr = r - a.row_split; }
    const long long wo = zz ? a.w_off[1] : a.w_off[0], bo = zz ? a.b_off[1] : a.b_off[0];  // no param indexing
    if (c < a.cols) a.grad[wo + (long long)rr * a.cols + c] = t;
    else a.grad[bo + rr] = t;
    if (!isfinite(t)) atomicAdd(&a.payload[4], 1.0f);
  }
}

void launch_reduce_dw(const DwReduceArgs& a, cudaStream_t st) {
  const int total = a.rows * (a.cols + 1);
  k_reduce_dw<<<dim3((total + 31) / 32, 1, a.nz), 256, 0, st>>>(a);
}

// ------------------------------------------------------------------ GAE (reverse time scan, thread per env)
constexpr int GAE_BLOCK = 256;
int gae_blocks(int N) { return (N + GAE_BLOCK - 1) / GAE_BLOCK; }

__device__ __forceinline__ double block_sum_d(double v, double* sred) {
  v = warp_sum_d(v);
  if ((threadIdx.x & 31) == 0) sred[threadIdx.x >> 5] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0)
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += sred[w];
  return s;
}

__global__ void __launch_bounds__(GAE_BLOCK) k_gae(GaeArgs a) {
  __shared__ double sred[GAE_BLOCK / 32];
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  double local = 0.0;
  if (i < a.N) {
    float nextA = 0.0f, nextV = a.VT[i];
    // the recurrence runs backwards in t; the inputs of GAE_PF steps are loaded before it consumes them
    constexpr int GAE_PF = 8;
    for (int t1 = a.T - 1; t1 >= 0; t1 -= GAE_PF) {
      float rr[GAE_PF], bb[GAE_PF], vv[GAE_PF];
      uint8_t ff[GAE_PF];
#pragma unroll
      for (int u = 0; u < GAE_PF; ++u) {
        const int t = t1 - u;
        if (t >= 0) {
          const size_t k = (size_t)t * a.N + i;
          rr[u] = __ldg(a.r + k); bb[u] = a.bootstrap ? __ldg(a.b + k) : 0.0f; vv[u] = __ldg(a.V + k);
          ff[u] = __ldg(a.flags + k);
        }
      }
#pragma unroll
      for (int u = 0; u < GAE_PF; ++u) {
        const int t = t1 - u;
        if (t < 0) break;
        const size_t k = (size_t)t * a.N + i;
        const float nd = (ff[u] & 3u) ? 0.0f : 1.0f;
        const float rt = a.bootstrap ? rr[u] + a.gamma * bb[u] : rr[u];
        const float v = vv[u];
        const float delta = rt + a.gamma * nd * nextV - v;
        const float A = delta + a.gamma * a.lam * nd * nextA;
        a.A[k] = A;
        a.R[k] = A + v;
        local += (double)A;
        nextA = A;
        nextV = v;
      }
    }
  }
  double s = block_sum_d(local, sred);
  if (threadIdx.x == 0) a.part[blockIdx.x] = s;
}

void launch_gae(const GaeArgs& a, cudaStream_t st) { k_gae<<<gae_blocks(a.N), GAE_BLOCK, 0, st>>>(a); }

__global__ void k_sum_partials(const double* part, int n, double* out) {
  __shared__ double sred[32];
  double s = 0.0;
  for (int k = threadIdx.x; k < n; k += blockDim.x) s += part[k];
  s = block_sum_d(s, sred);
  if (threadIdx.x == 0) *out = s;
}
void launch_sum_partials(const double* part, int n, double* out, cudaStream_t st) {
  k_sum_partials<<<1, 256, 0, st>>>(part, n, out);
}

constexpr int VAR_BLOCK = 256, VAR_PER = 8;
int var_blocks(int n) { return (n + VAR_BLOCK * VAR_PER - 1) / (VAR_BLOCK * VAR_PER); }
__global__ void k_var_partials(const float* A, int n, const double* mean_total, double count, double* part) {
  __shared__ double sred[VAR_BLOCK / 32];
  const double mean = *mean_total / count;
  double s = 0.0;
  const int base = blockIdx.x * VAR_BLOCK * VAR_PER;
  for (int k = 0; k < VAR_PER; ++k) {
    int i = base + k * VAR_BLOCK + threadIdx.x;
    if (i < n) { double d = (double)A[i] - mean; s += d * d; }
  }
  s = block_sum_d(s, sred);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}
void launch_var_partials(const float* A, int n, const double* mean_total, double count, double* part, cudaStream_t st) {
  k_var_partials<<<var_blocks(n), VAR_BLOCK, 0, st>>>(A, n, mean_total, count, part);
}

__global__ void k_adv_finalize(const double* sum_total, const double* sq_total, double count, DevScalars* sc, int T) {
  const double mean = *sum_total / count;
  const double var = count > 1.0 ? *sq_total / (count - 1.0) : 0.0;
  sc->adv_mean = mean;
  sc->adv_inv_std = 1.0 / (sqrt(var) + 1e-8);
  sc->s_base += (uint32_t)T;  // the rollout's T steps are consumed: the next rollout's events follow them
}
void launch_adv_finalize(const double* sum_total, const double* sq_total, double count, DevScalars* sc, int T,
                         cudaStream_t st) {
  k_adv_finalize<<<1, 1, 0, st>>>(sum_total, sq_total, count, sc, T);
}

// ------------------------------------------------------------------ Feistel shuffle
__device__ __forceinline__ uint32_t lowbias32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16;
  return x;
}

// grid.y = epochs computed by this launch (a.epoch + blockIdx.y), each writing perm + blockIdx.y * B
__global__ void k_perm(PermArgs a) {
  __shared__ uint32_t sKey[4];
  const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  const int epoch = a.epoch + (int)blockIdx.y;
  if (threadIdx.x == 0) {  // the epoch's round keys: one Philox block per thread block
    Rng rng{a.seed_lo, a.seed_hi};
    const uint32_t ev = a.sc->iteration * (uint32_t)a.E + (uint32_t)epoch;
    const U4 K = rng.block(0, (uint32_t)a.rank, ev, TAG_SHUFFLE);
    sKey[0] = K.x; sKey[1] = K.y; sKey[2] = K.z; sKey[3] = K.w;
  }
  __syncthreads();
  if (j >= a.B) return;
  const uint32_t Ks[4] = {sKey[0], sKey[1], sKey[2], sKey[3]};
  uint32_t k = 0;
  while ((1u << k) < a.B) ++k;
  if (k & 1u) ++k;
  if (k < 2) k = 2;
  const uint32_t half = k / 2u, mask = (1u << half) - 1u;
  uint32_t x = j;
  do {
    uint32_t L = x >> half, R = x & mask;
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      uint32_t nl = R;
      uint32_t nr = L ^ (lowbias32(R ^ Ks[r]) & mask);
      L = nl; R = nr;
    }
    x = (L << half) | R;
  } while (x >= a.B);
  a.perm[(size_t)blockIdx.y * a.B + j] = x;
}
void launch_perm(const PermArgs& a, cudaStream_t st) { k_perm<<<dim3((a.B + 255) / 256, a.n_epochs), 256, 0, st>>>(a); }

// ------------------------------------------------------------------ minibatch gather (warp per row)
constexpr int GATHER_ROWS = 2;  // rows per warp (even: the scalar fields go two rows per pass); see k_adam_gather
__device__ __forceinline__ void gather_body(const GatherArgs& a, int bid) {
  const int warp = (bid * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  const int r0 = warp * GATHER_ROWS;
  if (r0 >= a.M) return;
  const int nr = min(GATHER_ROWS, a.M - r0);
  uint32_t bl = 0;
  if (lane < nr) bl = a.idx ? (uint32_t)a.idx[r0 + lane] : a.perm[r0 + lane];
  uint32_t b[GATHER_ROWS];
#pragma unroll
  for (int k = 0; k < GATHER_ROWS; ++k) b[k] = __shfl_sync(0xffffffffu, bl, k);
  const int nq = a.Dp / 8;  // 16-B chunks per row
  uint4 v[GATHER_ROWS][2];
#pragma unroll
  for (int k = 0; k < GATHER_ROWS; ++k) {
    const uint4* src = reinterpret_cast<const uint4*>(a.obs + (size_t)b[k] * a.Dp);  // sample b = t N + i: row b of OBS
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int q = lane + 32 * h;
      if (k < nr && q < nq) v[k][h] = src[q];
    }
  }
  // scalar fields: lane 16k + f handles field f (< 16) of row k (two rows per pass)
  float sv[GATHER_ROWS / 2][2];
#pragma unroll
  for (int pss = 0; pss < GATHER_ROWS / 2; ++pss) {
    const int k = 2 * pss + (lane >> 4), f = lane & 15;
    const uint32_t bb = k == 2 * pss ? b[2 * pss] : b[2 * pss + 1];
    sv[pss][0] = sv[pss][1] = 0.0f;
    if (k < nr) {
      if (f < 12) { sv[pss][0] = a.act[(size_t)bb * 12 + f]; sv[pss][1] = a.mu[(size_t)bb * 12 + f]; }
      else if (f == 12) sv[pss][0] = a.logp[bb];
      else if (f == 13) sv[pss][0] = a.V[bb];
      else if (f == 14) sv[pss][0] = (float)(((double)a.A[bb] - a.sc->adv_mean) * a.sc->adv_inv_std);
      else sv[pss][0] = a.R[bb];
    }
  }
#pragma unroll
  for (int k = 0; k < GATHER_ROWS; ++k) {
    uint4* dst = reinterpret_cast<uint4*>(a.X + (size_t)(r0 + k) * a.Dp);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int q = lane + 32 * h;
      if (k < nr && q < nq) dst[q] = v[k][h];
    }
  }
#pragma unroll
  for (int pss = 0; pss < GATHER_ROWS / 2; ++pss) {
    const int k = 2 * pss + (lane >> 4), f = lane & 15;
    if (k >= nr) continue;
    const int w = r0 + k;
    if (f < 12) { a.o_act[(size_t)w * 12 + f] = sv[pss][0]; a.o_mu[(size_t)w * 12 + f] = sv[pss][1]; }
    else if (f == 12) a.o_logp[w] = sv[pss][0];
    else if (f == 13) a.o_V[w] = sv[pss][0];
    else if (f == 14) a.o_adv[w] = sv[pss][0];
    else a.o_ret[w] = sv[pss][0];
  }
}
__global__ void __launch_bounds__(256) k_gather(const __grid_constant__ GatherArgs a) {
  pdl_trigger();
  pdl_wait();
  gather_body(a, blockIdx.x);
}
static int gather_blocks(int M) {
  const long long warps = (M + GATHER_ROWS - 1) / GATHER_ROWS;
  return (int)((warps * 32 + 255) / 256);
}
void launch_gather(const GatherArgs& a, cudaStream_t st) {
  launch_pdl(k_gather, dim3((unsigned)gather_blocks(a.M)), dim3(256), 0, st, a);
}

// ------------------------------------------------------------------ Alg. 1 + Adam
// One kernel per minibatch m: thread 0 of every block evaluates Alg. 1 on the reduced KL of
// the payload and the bias corrections (same inputs -> same values in every block); block 0 publishes
// alpha/t into ring slot (m+1)&1 while every block reads slot m&1, so no block reads a value being written.
__device__ __forceinline__ void write_shadow(const ShadowArgs& sh, long long i, float th) {
  for (int s = 0; s < sh.nseg; ++s) {
    const Segment& g = sh.seg[s];
    const long long n = (long long)g.rows * g.cols;
    if (i >= g.off && i < g.off + n) {
      const uint32_t l = (uint32_t)(i - g.off);
      const int r = (int)(l / (uint32_t)g.cols), c = (int)(l - (uint32_t)r * (uint32_t)g.cols);
      if (g.kind == 0) reinterpret_cast<__nv_bfloat16*>(g.dst)[(size_t)r * g.dst_ld + c] = __float2bfloat16_rn(th);
      else reinterpret_cast<float*>(g.dst)[(size_t)r * g.dst_ld + c] = th;
      return;
    }
  }
}

// Grid: the parameter segments (ShadowArgs, one per weight / bias tensor) each get ceil(n / 512) blocks, so a
// block's 512 elements lie in one segment: its canonical range and its bf16 / fp32 GEMM shadow are found once.
constexpr int ADAM_PER_THREAD = ADAM_BLOCK_ELEMS / 256;
constexpr int ADAM_W = 6;  // split partials per element and pass
__device__ __forceinline__ void adam_body(const AdamArgs& a, const float* payload, float kl_target, int world, int m,
                                          float* acc, int bid) {
  __shared__ float s_step, s_ibc2;
  __shared__ int s_apply;
  int sg = 0;  // the block's segment: the last sg with blk0[sg] <= bid (block-uniform binary search)
  for (int hi = a.sh.nseg - 1; sg < hi;) {
    const int mid = (sg + hi + 1) >> 1;
    if (a.sh.blk0[mid] <= bid) sg = mid;
    else hi = mid - 1;
  }
  const Segment& G = a.sh.seg[sg];
  const int n = G.rows * G.cols;
  const int l0 = (bid - a.sh.blk0[sg]) * ADAM_BLOCK_ELEMS + threadIdx.x;
  // this thread's elements are loaded first, so their latency overlaps the Alg. 1 / bias-correction scalars
  float g[ADAM_PER_THREAD], mo[ADAM_PER_THREAD], vo[ADAM_PER_THREAD], tho[ADAM_PER_THREAD];
  // a weight / bias tensor whose gradient is still in its GEMM's split partials (AdamPart): summed here in split
  // order. The segment is block-uniform, so is its layer / net / kind.
  const AdamPart* PP = nullptr;
  int pz = 0;
  bool pbias = false;
  for (int li = 0; li < 3; ++li) {
    const AdamPart& q = a.part[li];
    if (!q.part) continue;
    for (int z = 0; z < 2; ++z) {
      if (G.off == q.w_off[z]) { PP = &q; pz = z; pbias = false; }
      if (G.off == q.b_off[z]) { PP = &q; pz = z; pbias = true; }
    }
  }
  // the state first (its latency overlaps the partial sums), then the gradient: the canonical vector, or the sum
  // of the GEMM's split partials in split order (AdamPart) -- both elements' loads of a pass in flight together
  // (2 x ADAM_W at once), addresses stepped by one split stride, no per-load predicate. Same-box A/B per C3
  // iteration against one element's six loads at a time: ADAM_W = 2 / 3 / 4 / 6 / 8 / 9 / 12: -0.7 / -1.1 / -1.3 /
  // -1.6 / -1.3 / -1.5 / -1.4 % (48 registers in every variant)
#pragma unroll
  for (int u = 0; u < ADAM_PER_THREAD; ++u) {
    const int l = l0 + u * 256;
    const long long i = G.off + l;
    g[u] = 0.0f;
    if (l < n) {
      mo[u] = a.m[i]; vo[u] = a.v[i]; tho[u] = a.theta[i];
      if (!PP) g[u] = a.grad[i];
    }
  }
  if (PP) {
    const float* p[ADAM_PER_THREAD];
    bool ok[ADAM_PER_THREAD];
#pragma unroll
    for (int u = 0; u < ADAM_PER_THREAD; ++u) {
      const int l = l0 + u * 256;
      ok[u] = l < n;
      int r, nt, col;
      if (!pbias) {
        r = l / PP->cols;
        const int c = l - r * PP->cols;
        nt = c / PP->bn;
        col = c - nt * PP->bn;
      } else {
        r = l;
        nt = 0;
        col = PP->bn;
      }
      const int R = PP->row_split ? pz * PP->row_split + r : r;
      const int mt = PP->row_split ? (R >> 7) : pz * PP->m_tiles + (R >> 7);
      p[u] = ok[u] ? PP->part + ((size_t)(mt * PP->n_tiles + nt) * PP->S * 128 + (R & 127)) * PP->rld + col : PP->part;
    }
    const size_t ss = (size_t)128 * PP->rld;
    const int S = PP->S;
    int s0 = 0;
#pragma unroll 1
    for (; s0 + ADAM_W <= S; s0 += ADAM_W) {
      float w[ADAM_PER_THREAD][ADAM_W];
#pragma unroll
      for (int u = 0; u < ADAM_PER_THREAD; ++u)
#pragma unroll
        for (int q = 0; q < ADAM_W; ++q) w[u][q] = __ldcg(p[u] + q * ss);
#pragma unroll
      for (int u = 0; u < ADAM_PER_THREAD; ++u) {
        g[u] = s0 == 0 ? w[u][0] : g[u] + w[u][0];
#pragma unroll
        for (int q = 1; q < ADAM_W; ++q) g[u] = g[u] + w[u][q];
        p[u] += ADAM_W * ss;
      }
    }
#pragma unroll 1
    for (; s0 < S; ++s0) {
#pragma unroll
      for (int u = 0; u < ADAM_PER_THREAD; ++u) {
        const float w = __ldcg(p[u]);
        g[u] = s0 == 0 ? w : g[u] + w;
        p[u] += ss;
      }
    }
  }
  if (threadIdx.x == 0) {
    DevScalars* sc = a.sc;
    const float W = (float)world;
    const float kl = payload[0] / W;
    const bool bad = payload[4] > 0.0f || !isfinite(kl);
    float alpha = sc->alpha_ring[m & 1];
    int t = sc->adamt_ring[m & 1];
    if (!bad) {
      if (kl > 2.0f * kl_target) alpha = fmaxf(1e-5f, alpha / 1.5f);
      else if (kl < 0.5f * kl_target) alpha = fminf(1e-2f, 1.5f * alpha);
      t = t + 1;
    }
    s_apply = bad ? 0 : 1;
    // alpha * m_hat / (sqrt(v_hat) + eps) = (alpha / bc1) * m / (sqrt(v / bc2) + eps), bc = 1 - b^t of the
    // applied step t (written by the previous Adam / iter_begin): the per-block scalars, one division left
    // per element
    s_step = alpha / sc->bc_ring[m & 1][0];
    s_ibc2 = 1.0f / sc->bc_ring[m & 1][1];
    if (bid == 0) {
      sc->alpha_ring[(m + 1) & 1] = alpha;
      sc->adamt_ring[(m + 1) & 1] = t;
      sc->bc_ring[(m + 1) & 1][0] = (float)(1.0 - pow((double)a.b1, (double)(t + 1)));
      sc->bc_ring[(m + 1) & 1][1] = (float)(1.0 - pow((double)a.b2, (double)(t + 1)));
      if (bad) {
        sc->nonfinite_skips += 1;
      } else {
        sc->applied += 1;
        sc->kl_last = kl;
        acc[0] += payload[1] / W; acc[1] += payload[2] / W; acc[2] += kl; acc[3] += payload[3] / W; acc[4] += 1.0f;
      }
    }
  }
  __syncthreads();
  if (!s_apply) return;
  const float step = s_step, ibc2 = s_ibc2;
  const bool dense = G.dst_ld == G.cols;  // shadow rows unpadded: shadow index = canonical index
#pragma unroll
  for (int u = 0; u < ADAM_PER_THREAD; ++u) {
    const int l = l0 + u * 256;
    if (l >= n) break;
    const long long i = G.off + l;
    const float gg = g[u] * a.inv_world;
    const float mm = a.b1 * mo[u] + (1.0f - a.b1) * gg;
    const float v = a.b2 * vo[u] + (1.0f - a.b2) * gg * gg;
    a.m[i] = mm;
    a.v[i] = v;
    const float th = tho[u] - step * mm / (sqrtf(v * ibc2) + a.eps);
    a.theta[i] = th;
    size_t o = (size_t)l;
    if (!dense) {
      const int r = l / G.cols, c = l - r * G.cols;
      o = (size_t)r * G.dst_ld + c;
    }
    if (G.kind == 0) reinterpret_cast<__nv_bfloat16*>(G.dst)[o] = __float2bfloat16_rn(th);
    else reinterpret_cast<float*>(G.dst)[o] = th;
  }
}
__global__ void __launch_bounds__(256) k_adam(const __grid_constant__ AdamArgs a, const float* payload, float kl_target,
                                              int world, int m, float* acc) {
  pdl_trigger();
  pdl_wait();
  adam_body(a, payload, kl_target, world, m, acc, blockIdx.x);
}
// Adam of minibatch m and the gather of minibatch m + 1 in one launch (blocks [0, nadam) update θ, the rest
// gather; both are memory bound, independent, and run side by side instead of as two dependent launches).
// Two rows per gather warp (45 registers, five blocks per SM, no spills): the random row reads want many
// warps in flight more than many rows per warp (same-box A/B per iteration: 4 rows at 58 registers = base,
// 4 rows capped at 48 registers -0.5 %, 2 rows -1.2 %, 8 rows +1.6 %)
__global__ void __launch_bounds__(256) k_adam_gather(const __grid_constant__ AdamArgs a, const float* payload,
                                                     float kl_target, int world, int m, float* acc,
                                                     const __grid_constant__ GatherArgs g, int nadam) {
  pdl_trigger();
  pdl_wait();
  if ((int)blockIdx.x < nadam) adam_body(a, payload, kl_target, world, m, acc, blockIdx.x);
  else gather_body(g, (int)blockIdx.x - nadam);
}

void launch_adam(const AdamArgs& a, const float* payload, float kl_target, int world, int m, float* acc, cudaStream_t st) {
  launch_pdl(k_adam, dim3((unsigned)a.sh.blk0[a.sh.nseg]), dim3(256), 0, st, a, payload, kl_target, world, m, acc);
}
void launch_adam_gather(const AdamArgs& a, const float* payload, float kl_target, int world, int m, float* acc,
                        const GatherArgs& g, cudaStream_t st) {
  const int nadam = a.sh.blk0[a.sh.nseg];
  launch_pdl(k_adam_gather, dim3((unsigned)(nadam + gather_blocks(g.M))), dim3(256), 0, st, a, payload, kl_target,
             world, m, acc, g, nadam);
}

__global__ void k_sync_shadow(ShadowArgs sh, const float* theta) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < sh.P; i += (long long)gridDim.x * blockDim.x)
    write_shadow(sh, i, theta[i]);
}
void launch_sync_shadow(const ShadowArgs& sh, const float* theta, cudaStream_t st) {
  int nb = (int)min((sh.P + 255) / 256, 148LL * 8);
  k_sync_shadow<<<nb, 256, 0, st>>>(sh, theta);
}

// ------------------------------------------------------------------ lg_group collective (single-device emulation)
// Every rank's element i is replaced by the rank-ordered sum of all ranks' element i: the allreduce(sum) of
// the one-process-per-GPU path, as one kernel over all ranks' buffers (no kernel waits for another).
template <typename T>
__global__ void k_group_sum(GroupSumArgs a) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < a.count; i += (long long)gridDim.x * blockDim.x) {
    T v[LG_MAX_GROUP];
#pragma unroll
    for (int r = 0; r < LG_MAX_GROUP; ++r)
      if (r < a.n) v[r] = reinterpret_cast<const T*>(a.p[r])[i];
    T s = v[0];
#pragma unroll
    for (int r = 1; r < LG_MAX_GROUP; ++r)
      if (r < a.n) s = s + v[r];
#pragma unroll
    for (int r = 0; r < LG_MAX_GROUP; ++r)
      if (r < a.n) reinterpret_cast<T*>(a.p[r])[i] = s;
  }
}
void launch_group_sum(const GroupSumArgs& a, cudaStream_t st) {
  const int nb = (int)std::min<long long>((a.count + 255) / 256, 148LL * 8);
  if (a.is_double) k_group_sum<double><<<nb, 256, 0, st>>>(a);
  else k_group_sum<float><<<nb, 256, 0, st>>>(a);
}

// ------------------------------------------------------------------ iteration bookkeeping
__global__ void k_iter_begin(DevScalars* sc, float* logstd_old, const float* logstd, float* iter_acc, float b1,
                             float b2) {
  const int j = threadIdx.x;
  if (j < 12) logstd_old[j] = logstd[j];
  if (j < 8) iter_acc[j] = 0.0f;
  if (j == 0) {
    sc->alpha_ring[0] = sc->alpha;
    sc->adamt_ring[0] = sc->adam_t;
    sc->bc_ring[0][0] = (float)(1.0 - pow((double)b1, (double)(sc->adam_t + 1)));
    sc->bc_ring[0][1] = (float)(1.0 - pow((double)b2, (double)(sc->adam_t + 1)));
  }
}
void launch_iter_begin(DevScalars* sc, float* logstd_old, const float* logstd, float* iter_acc, float b1, float b2,
                       cudaStream_t st) {
  k_iter_begin<<<1, 32, 0, st>>>(sc, logstd_old, logstd, iter_acc, b1, b2);
}

__global__ void k_iter_end(IterEndArgs a, const float* acc) {
  __shared__ int hist[16];
  if (threadIdx.x < 16) hist[threadIdx.x] = 0;
  __syncthreads();
  for (int i0 = 0; i0 < a.N; i0 += 4 * blockDim.x) {  // 4 level loads in flight per thread, then one ballot per bin
    int lv[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int i = i0 + u * (int)blockDim.x + (int)threadIdx.x;
      lv[u] = i < a.N ? min(max((int)__ldg(a.state + (size_t)S_LEVEL * a.N + i), 0), 15) : -1;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int bnum = 0; bnum < 16; ++bnum) {
        const int c = __popc(__ballot_sync(0xffffffffu, lv[u] == bnum));
        if ((threadIdx.x & 31) == 0 && c) atomicAdd(&hist[bnum], c);
      }
  }
  __syncthreads();
  // the statistics fields are written by separate threads (independent loads, no serial chain through
  // one thread); the counters are reset only after every thread has read them
  DevScalars* sc = a.sc;
  lg_update_stats_dev* s = a.stats ? reinterpret_cast<lg_update_stats_dev*>(a.stats) : nullptr;
  const int k = threadIdx.x;
  float alpha = 0.0f;
  if (k == 0) {
    alpha = sc->alpha_ring[a.n_mb & 1];
    sc->alpha = alpha;
    sc->adam_t = sc->adamt_ring[a.n_mb & 1];
    if (s) s->lr = alpha;
  }
  if (s) {
    if (k == 1) {
      const float n = fmaxf(acc[4], 1.0f);
      s->surrogate_loss = acc[0] / n; s->value_loss = acc[1] / n; s->mean_kl = acc[2] / n;
      s->clip_fraction = acc[3] / n; s->minibatches_applied = (int)acc[4];
    } else if (k == 2) {
      float H = 0.0f;
      for (int j = 0; j < 12; ++j) H += 0.5f + HALF_LN_2PI + a.logstd[j];
      s->entropy = H;
    } else if (k == 3) {
      const int ne = sc->episodes;
      s->mean_episode_return = ne > 0 ? (float)((double)sc->ep_return_fx * 0x1p-24 / (double)ne) : 0.0f;
      s->mean_episode_length = ne > 0 ? (float)((double)sc->ep_len_sum / (double)ne) : 0.0f;
      s->episodes = ne;
    } else if (k == 4) {
      s->promotions = sc->promotions; s->demotions = sc->demotions;
      s->nonfinite_skips = sc->nonfinite_skips; s->nonfinite_envs = sc->nonfinite_envs;
    } else if (k >= 32 && k < 48) {
      s->level_hist[k - 32] = hist[k - 32];
    }
  }
  __syncthreads();
  if (k == 0) {
    sc->ep_return_fx = 0; sc->ep_len_sum = 0; sc->episodes = 0; sc->promotions = 0; sc->demotions = 0;
    sc->nonfinite_envs = 0;
    sc->iteration += 1;
  }
}
void launch_iter_end(const IterEndArgs& a, const float* iter_acc, cudaStream_t st) {
  k_iter_end<<<1, 1024, 0, st>>>(a, iter_acc);
}


}  // namespace lg
