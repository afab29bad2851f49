// ppo.cu -- policy heads + Gaussian sampling, PPO loss head (fwd+bwd), GAE reverse scan, advantage
// statistics, Feistel shuffle, minibatch gather, deterministic gradient reductions, Alg. 1 + Adam.
// (§2.2, Table 3, Alg. 1; SPEC ppo/net.)
// Memory-bound kernels: one thread (or warp) per row/env, coalesced along the contiguous dimension;
// every cross-thread reduction uses a fixed tree order so results are run-to-run deterministic.
#include "common.cuh"
#include "kernels.h"

namespace lg {

constexpr float SIX_LN_2PI = 11.027262398456072f;
constexpr float HALF_LN_2PI = 0.9189385332046727f;

// ------------------------------------------------------------------ heads (4 threads per row)
// A "quad" of 4 consecutive threads owns one row; member q holds the columns [qC, qC+C) (C = H2/4) of
// the actor and of the critic half of H3. The 13 head dot products are reduced over the quad with two
// xor-shuffles and the quad leader's sums are broadcast, so all members hold bit-identical mu and V.
// The same head_fwd_quad serves the rollout (k_heads) and the update (k_loss_heads): the ratio of the
// first minibatch of an iteration is therefore exactly 1.
constexpr int MAXC = 32;  // H2 <= 128

__device__ __forceinline__ int wpad_index(int j, int col, int H2) {
  const int C = H2 >> 2, q = col / C, c = col - q * C;
  return j * (H2 + 16) + q * (C + 4) + c;  // 4 column groups, padded to stay bank-conflict free
}

__device__ __forceinline__ float quad_sum(float v) {
  v += __shfl_xor_sync(0xffffffffu, v, 1);
  v += __shfl_xor_sync(0xffffffffu, v, 2);
  return __shfl_sync(0xffffffffu, v, (threadIdx.x & 31) & ~3);
}

// ha/hc: this member's C columns; sW: padded [13][H2+16] (row 12 = critic W4c); returns mu[12], V
__device__ __forceinline__ void head_fwd_quad(const float* ha, const float* hc, int H2, int q, const float* sW,
                                              const float* sb4a, float b4c, float* mu, float& V) {
  const int C = H2 >> 2;
  const float* w0 = sW + q * (C + 4);
#pragma unroll
  for (int j = 0; j < 12; ++j) {
    float p = 0.0f;
#pragma unroll
    for (int c = 0; c < MAXC; c += 4)
      if (c < C) {
        const float4 w = *reinterpret_cast<const float4*>(w0 + j * (H2 + 16) + c);
        p = fmaf(w.x, ha[c], p); p = fmaf(w.y, ha[c + 1], p); p = fmaf(w.z, ha[c + 2], p); p = fmaf(w.w, ha[c + 3], p);
      }
    mu[j] = quad_sum(p) + sb4a[j];
  }
  float pv = 0.0f;
#pragma unroll
  for (int c = 0; c < MAXC; c += 4)
    if (c < C) {
      const float4 w = *reinterpret_cast<const float4*>(w0 + 12 * (H2 + 16) + c);
      pv = fmaf(w.x, hc[c], pv); pv = fmaf(w.y, hc[c + 1], pv); pv = fmaf(w.z, hc[c + 2], pv); pv = fmaf(w.w, hc[c + 3], pv);
    }
  V = quad_sum(pv) + b4c;
}

__device__ __forceinline__ float logp_gauss(const float* a, const float* mu, const float* ls) {
  float s = 0.0f;
#pragma unroll
  for (int j = 0; j < 12; ++j) {
    float z = (a[j] - mu[j]) * expf(-ls[j]);
    s = s + (0.5f * z * z + ls[j]);
  }
  return -s - SIX_LN_2PI;
}

__device__ __forceinline__ void load_head_weights(const float* W4a, const float* b4a, const float* W4c,
                                                  const float* b4c, const float* ls, int H2, float* sW,
                                                  float* sb4a, float* sls, float* sb4c) {
  for (int k = threadIdx.x; k < 13 * H2; k += blockDim.x) {
    const int j = k / H2, col = k - j * H2;
    sW[wpad_index(j, col, H2)] = j < 12 ? W4a[k] : W4c[col];
  }
  if (threadIdx.x < 12) { sb4a[threadIdx.x] = b4a[threadIdx.x]; sls[threadIdx.x] = ls[threadIdx.x]; }
  if (threadIdx.x == 12) *sb4c = *b4c;
}

__device__ __forceinline__ void bf16_cols(const __nv_bfloat16* p, int C, float* f) {
#pragma unroll
  for (int c = 0; c < MAXC; c += 8) {
    if (c < C) {
      uint4 u = *reinterpret_cast<const uint4*>(p + c);
      const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        float2 t = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w[e]));
        f[c + 2 * e] = t.x;
        f[c + 2 * e + 1] = t.y;
      }
    }
  }
}

constexpr int HEAD_ROWS = 16;  // rows per 64-thread block

__global__ void __launch_bounds__(64) k_heads(HeadArgs a) {
  extern __shared__ float sh[];
  const int M = a.M_dev ? *a.M_dev : a.M;
  if (blockIdx.x * HEAD_ROWS >= M) return;  // block-uniform, before any work (empty bootstrap launches)
  const int H2 = a.nd.H2, C = H2 >> 2;
  float* sW = sh;
  float* sb4a = sW + 13 * (H2 + 16);
  float* sls = sb4a + 12;
  float* sb4c = sls + 12;
  load_head_weights(a.W4a, a.b4a, a.W4c, a.b4c, a.logstd, H2, sW, sb4a, sls, sb4c);
  __syncthreads();
  const int q = threadIdx.x & 3;
  const int r = blockIdx.x * HEAD_ROWS + (threadIdx.x >> 2);
  const bool valid = r < M;
  float ha[MAXC], hc[MAXC];
  const __nv_bfloat16* hrow = a.H3 + (size_t)(valid ? r : 0) * 2 * H2;
  bf16_cols(hrow + q * C, C, ha);
  bf16_cols(hrow + H2 + q * C, C, hc);
  float mu[12], V;
  head_fwd_quad(ha, hc, H2, q, sW, sb4a, *sb4c, mu, V);
  if (!valid || q != 0) return;
  if (a.mode == 1) {  // value scatter (time-out bootstrap or V(o_T))
    a.value[a.idx ? a.idx[r] : r] = V;
    return;
  }
  if (a.mode == 2) {
    for (int j = 0; j < 12; ++j) a.mu[(size_t)r * 12 + j] = mu[j];
    a.value[r] = V;
    return;
  }
  // act: a = mu + sigma * eps, eps = Box-Muller pairs (2k, 2k+1) of the ACTION stream
  Rng rng{a.seed_lo, a.seed_hi};
  const uint32_t g = (uint32_t)(a.rank * a.N + r);
  const uint32_t ev = a.scalars->s_base + (uint32_t)a.t + 1u;
  const U4 b0 = rng.block(0, g, ev, TAG_ACTION), b1 = rng.block(1, g, ev, TAG_ACTION), b2 = rng.block(2, g, ev, TAG_ACTION);
  const uint32_t w[12] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w, b2.x, b2.y, b2.z, b2.w};
  float act[12];
#pragma unroll
  for (int k = 0; k < 6; ++k) {
    const float u1 = (float)((w[2 * k] >> 8) + 1u) * 0x1p-24f;
    const float u2 = (float)(w[2 * k + 1] >> 8) * 0x1p-24f;
    const float rr = sqrtf(-2.0f * log_poly(u1));
    float sn, cs;
    sincos_poly(0x1.921fb6p2f * u2, sn, cs);
    act[2 * k] = mu[2 * k] + expf(sls[2 * k]) * (rr * cs);
    act[2 * k + 1] = mu[2 * k + 1] + expf(sls[2 * k + 1]) * (rr * sn);
  }
  const float lp = logp_gauss(act, mu, sls);
  const size_t o = (size_t)r * 12;
#pragma unroll
  for (int j = 0; j < 12; ++j) {
    a.act[o + j] = act[j];
    a.mu[o + j] = mu[j];
  }
  a.logp[r] = lp;
  a.value[r] = V;
  if (a.u_act) for (int j = 0; j < 12; ++j) a.u_act[o + j] = act[j];
  if (a.u_mu) for (int j = 0; j < 12; ++j) a.u_mu[o + j] = mu[j];
  if (a.u_logp) a.u_logp[r] = lp;
  if (a.u_value) a.u_value[r] = V;
}

void launch_heads(const HeadArgs& a, cudaStream_t st) {
  int smem = (13 * (a.nd.H2 + 16) + 28) * 4;
  k_heads<<<(a.M + HEAD_ROWS - 1) / HEAD_ROWS, HEAD_ROWS * 4, smem, st>>>(a);
}

// ------------------------------------------------------------------ PPO loss head (fwd + bwd)
// Block = 256 threads = 64 rows x 4 members. The block's H3 rows (contiguous in memory) are staged in
// smem with coalesced 16-B loads; dmu/dV per row go to smem; the block then forms its partial of
// dW4 = dY^T H3 column-wise (each thread a few output columns, rows summed in order).
constexpr int LOSS_BLOCK = 64;
int loss_head_partial_floats(int H2) { return ((13 * H2 + 25) + 3) / 4 * 4; }
int loss_blocks(int M) { return (M + LOSS_BLOCK - 1) / LOSS_BLOCK; }

__device__ __forceinline__ float elu_grad_from_out(float h) { return h > 0.0f ? 1.0f : h + 1.0f; }

__global__ void __launch_bounds__(256, 2) k_loss_heads(LossArgs a) {
  extern __shared__ float sh[];
  const int H2 = a.nd.H2, C = H2 >> 2, HP = a.HP;
  const int SHLD = 2 * H2 + 8;  // bf16 row stride of the staged H3 tile
  float* sW = sh;
  float* sb4a = sW + 13 * (H2 + 16);
  float* sls = sb4a + 12;
  float* slso = sls + 12;
  float* sb4c = slso + 12;
  float* sdy = sb4c + 4;                       // [64][13] dmu | dV
  float* sdl = sdy + LOSS_BLOCK * 13;          // [64][12] dlogstd per row
  double* sst = reinterpret_cast<double*>(sdl + LOSS_BLOCK * 12);  // [64][5]
  __nv_bfloat16* sH = reinterpret_cast<__nv_bfloat16*>(sst + LOSS_BLOCK * 5);  // [64][SHLD]
  load_head_weights(a.W4a, a.b4a, a.W4c, a.b4c, a.logstd, H2, sW, sb4a, sls, sb4c);
  if (threadIdx.x < 12) slso[threadIdx.x] = a.logstd_old[threadIdx.x];
  const int row0 = blockIdx.x * LOSS_BLOCK;
  const int nrows = min(LOSS_BLOCK, a.M - row0);
  {  // stage H3 rows [row0, row0 + nrows) (contiguous) into smem
    const int v_per_row = (2 * H2) / 8;
    const uint4* src = reinterpret_cast<const uint4*>(a.H3 + (size_t)row0 * 2 * H2);
    for (int k = threadIdx.x; k < nrows * v_per_row; k += blockDim.x) {
      const int rr = k / v_per_row, cc = k - rr * v_per_row;
      *reinterpret_cast<uint4*>(sH + rr * SHLD + cc * 8) = src[k];
    }
  }
  __syncthreads();
  const int q = threadIdx.x & 3, rl = threadIdx.x >> 2;
  const int r = row0 + rl;
  const bool valid = rl < nrows;
  const float invM = 1.0f / (float)a.M;
  float ha[MAXC], hc[MAXC];
#pragma unroll
  for (int c = 0; c < MAXC; ++c) {
    ha[c] = c < C ? __bfloat162float(sH[rl * SHLD + q * C + c]) : 0.0f;
    hc[c] = c < C ? __bfloat162float(sH[rl * SHLD + H2 + q * C + c]) : 0.0f;
  }
  float mu[12], V;
  head_fwd_quad(ha, hc, H2, q, sW, sb4a, *sb4c, mu, V);
  float dmu[12], dV = 0.0f;
  if (valid) {
    float act[12];
#pragma unroll
    for (int j = 0; j < 12; ++j) act[j] = __ldg(a.act + (size_t)r * 12 + j);
    const float lp = logp_gauss(act, mu, sls);
    const float ratio = expf(lp - __ldg(a.logp_old + r));
    const float adv = __ldg(a.adv + r);
    const float s1 = ratio * adv;
    const float rc = fminf(fmaxf(ratio, 1.0f - a.clip), 1.0f + a.clip);
    const float s2 = rc * adv;
    const bool take1 = s1 <= s2;
    const bool inside = ratio >= 1.0f - a.clip && ratio <= 1.0f + a.clip;
    const float dLdlp = -(take1 ? adv : (inside ? adv : 0.0f)) * invM * ratio;
    const float Vo = __ldg(a.V_old + r), ret = __ldg(a.ret + r);
    const float vc = Vo + fminf(fmaxf(V - Vo, -a.vclip), a.vclip);
    const float e1 = (V - ret) * (V - ret), e2 = (vc - ret) * (vc - ret);
    const bool take_u = e1 >= e2;
    const bool vin = fabsf(V - Vo) <= a.vclip;
    dV = a.vf_coef * (take_u ? 2.0f * (V - ret) : (vin ? 2.0f * (vc - ret) : 0.0f)) * invM;
    float kl = 0.0f;
#pragma unroll
    for (int j = 0; j < 12; ++j) {
      const float d = act[j] - mu[j];
      const float iv = expf(-2.0f * sls[j]);
      dmu[j] = dLdlp * d * iv;
      const float dm = __ldg(a.mu_old + (size_t)r * 12 + j) - mu[j];
      kl += sls[j] - slso[j] + (expf(2.0f * slso[j]) + dm * dm) * (0.5f * iv) - 0.5f;
      if (q == 0) sdl[rl * 12 + j] = dLdlp * (d * d * iv - 1.0f);
    }
    if (q == 0) {
      for (int j = 0; j < 12; ++j) sdy[rl * 13 + j] = dmu[j];
      sdy[rl * 13 + 12] = dV;
      const double sv = (double)(take1 ? s1 : s2), vv = (double)(take_u ? e1 : e2), kv = (double)kl;
      double* s = sst + rl * 5;
      s[0] = sv; s[1] = vv; s[2] = kv;
      s[3] = fabsf(ratio - 1.0f) > a.clip ? 1.0 : 0.0;
      s[4] = (isfinite(sv) && isfinite(vv) && isfinite(kv)) ? 0.0 : 1.0;
    }
    // dZ3 = dH3 * ELU'(H3) for this member's columns (actor, then critic)
    const float* w0 = sW + q * (C + 4);
    __nv_bfloat16* dz = a.dZ3 + (size_t)r * 2 * H2 + q * C;
#pragma unroll
    for (int c = 0; c < MAXC; c += 4) {
      if (c < C) {
        float d0 = 0.0f, d1 = 0.0f, d2 = 0.0f, d3 = 0.0f;
#pragma unroll
        for (int j = 0; j < 12; ++j) {
          const float4 w = *reinterpret_cast<const float4*>(w0 + j * (H2 + 16) + c);
          d0 = fmaf(dmu[j], w.x, d0); d1 = fmaf(dmu[j], w.y, d1); d2 = fmaf(dmu[j], w.z, d2); d3 = fmaf(dmu[j], w.w, d3);
        }
        __nv_bfloat162 za = __floats2bfloat162_rn(d0 * elu_grad_from_out(ha[c]), d1 * elu_grad_from_out(ha[c + 1]));
        __nv_bfloat162 zb = __floats2bfloat162_rn(d2 * elu_grad_from_out(ha[c + 2]), d3 * elu_grad_from_out(ha[c + 3]));
        *reinterpret_cast<uint2*>(dz + c) = make_uint2(*reinterpret_cast<uint32_t*>(&za), *reinterpret_cast<uint32_t*>(&zb));
        const float4 wc = *reinterpret_cast<const float4*>(w0 + 12 * (H2 + 16) + c);
        __nv_bfloat162 ca = __floats2bfloat162_rn(dV * wc.x * elu_grad_from_out(hc[c]), dV * wc.y * elu_grad_from_out(hc[c + 1]));
        __nv_bfloat162 cb = __floats2bfloat162_rn(dV * wc.z * elu_grad_from_out(hc[c + 2]), dV * wc.w * elu_grad_from_out(hc[c + 3]));
        *reinterpret_cast<uint2*>(dz + H2 + c) = make_uint2(*reinterpret_cast<uint32_t*>(&ca), *reinterpret_cast<uint32_t*>(&cb));
      }
    }
  }
  __syncthreads();
  // block partial of the head/log-std gradients (rows in order)
  float* out = a.part + (size_t)blockIdx.x * HP;
  for (int e2 = threadIdx.x; e2 < 13 * H2 / 2; e2 += blockDim.x) {
    const int e = 2 * e2;
    const int j = e / H2, k = e - j * H2;
    const int col = j < 12 ? k : H2 + k;
    float acc0 = 0.0f, acc1 = 0.0f;
    for (int rr = 0; rr < nrows; ++rr) {
      const float dy = sdy[rr * 13 + j];
      const float2 h = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(sH + rr * SHLD + col));
      acc0 = fmaf(dy, h.x, acc0);
      acc1 = fmaf(dy, h.y, acc1);
    }
    const int o = j < 12 ? e : 12 * H2 + 12 + k;
    out[o] = acc0;
    out[o + 1] = acc1;
  }
  if (threadIdx.x < 13) {
    float sb = 0.0f;
    for (int rr = 0; rr < nrows; ++rr) sb = sb + sdy[rr * 13 + threadIdx.x];
    out[threadIdx.x < 12 ? 12 * H2 + threadIdx.x : 13 * H2 + 12] = sb;
  } else if (threadIdx.x >= 32 && threadIdx.x < 44) {
    const int j = threadIdx.x - 32;
    float sl = 0.0f;
    for (int rr = 0; rr < nrows; ++rr) sl = sl + sdl[rr * 12 + j];
    out[13 * H2 + 13 + j] = sl;
  } else if (threadIdx.x >= 64 && threadIdx.x < 69) {
    const int k = threadIdx.x - 64;
    double s = 0.0;
    for (int rr = 0; rr < nrows; ++rr) s += sst[rr * 5 + k];
    a.spart[(size_t)blockIdx.x * 8 + k] = s;
  }
}

void launch_loss_heads(const LossArgs& a, cudaStream_t st) {
  const int H2 = a.nd.H2;
  const size_t smem = (13 * (H2 + 16) + 40 + LOSS_BLOCK * 25) * 4 + 16 + LOSS_BLOCK * 5 * 8 +
                      (size_t)LOSS_BLOCK * (2 * H2 + 8) * 2 + 64;
  static size_t set = 0;
  if (smem > set) {
    cudaFuncSetAttribute(k_loss_heads, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    set = smem;
  }
  k_loss_heads<<<loss_blocks(a.M), 256, smem, st>>>(a);
}

// sums over blocks (fixed order) -> canonical gradient of heads/log-std + stats payload.
// Block = 32 warps x 32 elements; warp w sums partial rows b = w, w+32, ... (in order), then lane-wise the
// 32 warp sums are added in warp order: a fixed, run-to-run deterministic tree.
constexpr int RH_WARPS = 32;
__global__ void __launch_bounds__(RH_WARPS * 32) k_reduce_heads(HeadReduceArgs a) {
  __shared__ float ssum[RH_WARPS][33];
  const int H2 = a.H2;
  const int nval = 13 * H2 + 25;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int e = blockIdx.x * 32 + lane;
  float s = 0.0f;
  if (e < nval)
    for (int b = warp; b < a.nblk; b += RH_WARPS) s = s + a.part[(size_t)b * a.HP + e];
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
  if (blockIdx.x == 0 && warp == 1) {
    const double invM = 1.0 / (double)a.M;
    for (int k = 0; k < 5; ++k) {
      double v = 0.0;
      for (int b = lane; b < a.nblk; b += 32) v += a.spart[(size_t)b * 8 + k];
      v = warp_sum_d(v);
      if (lane == 0) {
        if (k == 0) a.payload[1] = (float)(v * invM);       // surrogate mean
        if (k == 1) a.payload[2] = (float)(v * invM);       // value loss mean
        if (k == 2) a.payload[0] = (float)(v * invM);       // KL mean (Alg. 1)
        if (k == 3) a.payload[3] = (float)(v * invM);       // clip fraction
        if (k == 4 && v > 0.0) atomicAdd(&a.payload[4], (float)v);
      }
    }
    if (lane == 0) a.payload[5] = 1.0f;                     // rank count (allreduce sums it)
  }
}

void launch_reduce_heads(const HeadReduceArgs& a, cudaStream_t st) {
  int n = 13 * a.H2 + 25;
  k_reduce_heads<<<(n + 31) / 32, RH_WARPS * 32, 0, st>>>(a);
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
    if (c < a.cols) a.grad[a.w_off[zz] + (long long)rr * a.cols + c] = t;
    else a.grad[a.b_off[zz] + rr] = t;
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
    for (int t = a.T - 1; t >= 0; --t) {
      const size_t k = (size_t)t * a.N + i;
      const float nd = (a.flags[k] & 3u) ? 0.0f : 1.0f;
      const float rt = a.bootstrap ? a.r[k] + a.gamma * a.b[k] : a.r[k];
      const float v = a.V[k];
      const float delta = rt + a.gamma * nd * nextV - v;
      const float A = delta + a.gamma * a.lam * nd * nextA;
      a.A[k] = A;
      a.R[k] = A + v;
      local += (double)A;
      nextA = A;
      nextV = v;
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

__global__ void k_adv_finalize(const double* sum_total, const double* sq_total, double count, DevScalars* sc) {
  const double mean = *sum_total / count;
  const double var = count > 1.0 ? *sq_total / (count - 1.0) : 0.0;
  sc->adv_mean = mean;
  sc->adv_inv_std = 1.0 / (sqrt(var) + 1e-8);
}
void launch_adv_finalize(const double* sum_total, const double* sq_total, double count, DevScalars* sc, cudaStream_t st) {
  k_adv_finalize<<<1, 1, 0, st>>>(sum_total, sq_total, count, sc);
}

// ------------------------------------------------------------------ Feistel shuffle
__device__ __forceinline__ uint32_t lowbias32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16;
  return x;
}

__global__ void k_perm(PermArgs a) {
  const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= a.B) return;
  Rng rng{a.seed_lo, a.seed_hi};
  const uint32_t ev = a.sc->iteration * (uint32_t)a.E + (uint32_t)a.epoch;
  U4 K = rng.block(0, (uint32_t)a.rank, ev, TAG_SHUFFLE);
  const uint32_t Ks[4] = {K.x, K.y, K.z, K.w};
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
  a.perm[j] = x;
}
void launch_perm(const PermArgs& a, cudaStream_t st) { k_perm<<<(a.B + 255) / 256, 256, 0, st>>>(a); }

// ------------------------------------------------------------------ minibatch gather (warp per row)
__global__ void k_gather(GatherArgs a) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= a.M) return;
  const uint32_t b = a.idx ? (uint32_t)a.idx[warp] : a.perm[warp];
  const uint32_t t = b / (uint32_t)a.N, i = b - t * (uint32_t)a.N;
  const uint4* src = reinterpret_cast<const uint4*>(a.obs + ((size_t)t * a.N + i) * a.Dp);
  uint4* dst = reinterpret_cast<uint4*>(a.X + (size_t)warp * a.Dp);
  for (int q = lane; q < a.Dp / 8; q += 32) dst[q] = src[q];
  if (lane < 12) {
    a.o_act[(size_t)warp * 12 + lane] = a.act[(size_t)b * 12 + lane];
    a.o_mu[(size_t)warp * 12 + lane] = a.mu[(size_t)b * 12 + lane];
  } else if (lane == 12) {
    a.o_logp[warp] = a.logp[b];
  } else if (lane == 13) {
    a.o_V[warp] = a.V[b];
  } else if (lane == 14) {
    a.o_adv[warp] = (float)(((double)a.A[b] - a.sc->adv_mean) * a.sc->adv_inv_std);
  } else if (lane == 15) {
    a.o_ret[warp] = a.R[b];
  }
}
void launch_gather(const GatherArgs& a, cudaStream_t st) {
  long long threads = (long long)a.M * 32;
  k_gather<<<(unsigned)((threads + 255) / 256), 256, 0, st>>>(a);
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
      const long long l = i - g.off;
      const int r = (int)(l / g.cols), c = (int)(l - (long long)r * g.cols);
      if (g.kind == 0) reinterpret_cast<__nv_bfloat16*>(g.dst)[(size_t)r * g.dst_ld + c] = __float2bfloat16_rn(th);
      else reinterpret_cast<float*>(g.dst)[(size_t)r * g.dst_ld + c] = th;
      return;
    }
  }
}

__global__ void k_adam(AdamArgs a, const float* payload, float kl_target, int world, int m, float* acc) {
  __shared__ float s_alpha, s_bc1, s_bc2;
  __shared__ int s_apply;
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
    s_alpha = alpha;
    s_bc1 = (float)(1.0 - pow((double)a.b1, (double)t));
    s_bc2 = (float)(1.0 - pow((double)a.b2, (double)t));
    if (blockIdx.x == 0) {
      sc->alpha_ring[(m + 1) & 1] = alpha;
      sc->adamt_ring[(m + 1) & 1] = t;
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
  const float alpha = s_alpha, bc1 = s_bc1, bc2 = s_bc2;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < a.sh.P; i += (long long)gridDim.x * blockDim.x) {
    const float g = a.grad[i] * a.inv_world;
    const float mm = a.b1 * a.m[i] + (1.0f - a.b1) * g;
    const float v = a.b2 * a.v[i] + (1.0f - a.b2) * g * g;
    a.m[i] = mm;
    a.v[i] = v;
    const float mh = mm / bc1, vh = v / bc2;
    const float th = a.theta[i] - alpha * mh / (sqrtf(vh) + a.eps);
    a.theta[i] = th;
    write_shadow(a.sh, i, th);
  }
}
void launch_adam(const AdamArgs& a, const float* payload, float kl_target, int world, int m, float* acc, cudaStream_t st) {
  int nb = (int)min((a.sh.P + 255) / 256, 148LL * 8);
  k_adam<<<nb, 256, 0, st>>>(a, payload, kl_target, world, m, acc);
}

__global__ void k_sync_shadow(ShadowArgs sh, const float* theta) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < sh.P; i += (long long)gridDim.x * blockDim.x)
    write_shadow(sh, i, theta[i]);
}
void launch_sync_shadow(const ShadowArgs& sh, const float* theta, cudaStream_t st) {
  int nb = (int)min((sh.P + 255) / 256, 148LL * 8);
  k_sync_shadow<<<nb, 256, 0, st>>>(sh, theta);
}

// ------------------------------------------------------------------ iteration bookkeeping
__global__ void k_iter_begin(DevScalars* sc, float* logstd_old, const float* logstd, float* iter_acc) {
  const int j = threadIdx.x;
  if (j < 12) logstd_old[j] = logstd[j];
  if (j < 8) iter_acc[j] = 0.0f;
  if (j == 0) { sc->alpha_ring[0] = sc->alpha; sc->adamt_ring[0] = sc->adam_t; }
}
void launch_iter_begin(DevScalars* sc, float* logstd_old, const float* logstd, float* iter_acc, cudaStream_t st) {
  k_iter_begin<<<1, 32, 0, st>>>(sc, logstd_old, logstd, iter_acc);
}

__global__ void k_iter_end(IterEndArgs a, const float* acc) {
  __shared__ int hist[16];
  if (threadIdx.x < 16) hist[threadIdx.x] = 0;
  __syncthreads();
  for (int i = threadIdx.x; i < a.N; i += blockDim.x) {
    int lv = (int)a.state[(size_t)S_LEVEL * a.N + i];
    atomicAdd(&hist[min(max(lv, 0), 15)], 1);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    DevScalars* sc = a.sc;
    sc->alpha = sc->alpha_ring[a.n_mb & 1];
    sc->adam_t = sc->adamt_ring[a.n_mb & 1];
    if (a.stats) {
      lg_update_stats_dev* s = reinterpret_cast<lg_update_stats_dev*>(a.stats);
      const float n = fmaxf(acc[4], 1.0f);
      s->surrogate_loss = acc[0] / n;
      s->value_loss = acc[1] / n;
      float H = 0.0f;
      for (int j = 0; j < 12; ++j) H += 0.5f + HALF_LN_2PI + a.logstd[j];
      s->entropy = H;
      s->mean_kl = acc[2] / n;
      s->lr = sc->alpha;
      s->clip_fraction = acc[3] / n;
      s->nonfinite_skips = sc->nonfinite_skips;
      s->minibatches_applied = (int)acc[4];
      const int ne = sc->episodes;
      s->mean_episode_return = ne > 0 ? sc->ep_return_sum / (float)ne : 0.0f;
      s->mean_episode_length = ne > 0 ? sc->ep_len_sum / (float)ne : 0.0f;
      s->episodes = ne;
      s->promotions = sc->promotions;
      s->demotions = sc->demotions;
      s->reserved = (int)sc->iteration + 1;
      for (int k = 0; k < 16; ++k) s->level_hist[k] = hist[k];
    }
    sc->ep_return_sum = 0.0f; sc->ep_len_sum = 0.0f; sc->episodes = 0; sc->promotions = 0; sc->demotions = 0;
    sc->iteration += 1;
  }
}
void launch_iter_end(const IterEndArgs& a, const float* iter_acc, cudaStream_t st) {
  k_iter_end<<<1, 256, 0, st>>>(a, iter_acc);
}

__global__ void k_advance_sbase(DevScalars* sc, int T) { sc->s_base += (uint32_t)T; }
void launch_advance_sbase(DevScalars* sc, int T, cudaStream_t st) { k_advance_sbase<<<1, 1, 0, st>>>(sc, T); }

}  // namespace lg
