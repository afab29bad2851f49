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

// ------------------------------------------------------------------ heads
__device__ __forceinline__ void bf16x8(const __nv_bfloat16* p, float* f) {
  uint4 u = *reinterpret_cast<const uint4*>(p);
  uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    float2 t = __bfloat1622float2(*reinterpret_cast<__nv_bfloat162*>(&w[e]));
    f[2 * e] = t.x;
    f[2 * e + 1] = t.y;
  }
}

// mu_j = (sum_k W4a[j][k] h_a[k]) + b4a_j, V = (sum_k W4c[k] h_c[k]) + b4c, sequential in k.
__device__ __forceinline__ void head_forward(const __nv_bfloat16* ha, const __nv_bfloat16* hc, int H2, const float* sW4a,
                                             const float* sb4a, const float* sW4c, float b4c, float* mu, float& V) {
  float acc[12];
#pragma unroll
  for (int j = 0; j < 12; ++j) acc[j] = 0.0f;
  float vac = 0.0f;
  for (int k = 0; k < H2; k += 8) {
    float h[8], g[8];
    bf16x8(ha + k, h);
    bf16x8(hc + k, g);
#pragma unroll
    for (int e = 0; e < 8; ++e) {
#pragma unroll
      for (int j = 0; j < 12; ++j) acc[j] = acc[j] + sW4a[j * H2 + k + e] * h[e];
      vac = vac + sW4c[k + e] * g[e];
    }
  }
#pragma unroll
  for (int j = 0; j < 12; ++j) mu[j] = acc[j] + sb4a[j];
  V = vac + b4c;
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

__global__ void k_heads(HeadArgs a) {
  extern __shared__ float sh[];
  const int H2 = a.nd.H2;
  float* sW4a = sh;
  float* sb4a = sW4a + 12 * H2;
  float* sW4c = sb4a + 12;
  float* sls = sW4c + H2;
  for (int k = threadIdx.x; k < 12 * H2; k += blockDim.x) sW4a[k] = a.W4a[k];
  for (int k = threadIdx.x; k < H2; k += blockDim.x) sW4c[k] = a.W4c[k];
  if (threadIdx.x < 12) { sb4a[threadIdx.x] = a.b4a[threadIdx.x]; sls[threadIdx.x] = a.logstd[threadIdx.x]; }
  __syncthreads();
  const int M = a.M_dev ? *a.M_dev : a.M;
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= M) return;
  const __nv_bfloat16* ha = a.H3 + (size_t)r * 2 * H2;
  float mu[12], V;
  head_forward(ha, ha + H2, H2, sW4a, sb4a, sW4c, __ldg(a.b4c), mu, V);
  if (a.mode == 1) {  // value scatter (time-out bootstrap or V(o_T))
    int dst = a.idx ? a.idx[r] : r;
    a.value[dst] = V;
    return;
  }
  if (a.mode == 2) {
    for (int j = 0; j < 12; ++j) a.mu[(size_t)r * 12 + j] = mu[j];
    a.value[r] = V;
    return;
  }
  // act: a = mu + sigma * eps (ACTION stream of env g at step s_base + t + 1), logp
  Rng rng{a.seed_lo, a.seed_hi};
  const uint32_t g = (uint32_t)(a.rank * a.N + r);
  const uint32_t ev = a.scalars->s_base + (uint32_t)a.t + 1u;
  U4 b0 = rng.block(0, g, ev, TAG_ACTION), b1 = rng.block(1, g, ev, TAG_ACTION), b2 = rng.block(2, g, ev, TAG_ACTION);
  uint32_t w[12] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w, b2.x, b2.y, b2.z, b2.w};
  float act[12];
#pragma unroll
  for (int k = 0; k < 6; ++k) {
    float u1 = (float)((w[2 * k] >> 8) + 1u) * 0x1p-24f;
    float u2 = (float)(w[2 * k + 1] >> 8) * 0x1p-24f;
    float rr = sqrtf(-2.0f * log_poly(u1));
    float sn, cs;
    sincos_poly(0x1.921fb6p2f * u2, sn, cs);
    act[2 * k] = mu[2 * k] + expf(sls[2 * k]) * (rr * cs);
    act[2 * k + 1] = mu[2 * k + 1] + expf(sls[2 * k + 1]) * (rr * sn);
  }
  float lp = logp_gauss(act, mu, sls);
  const size_t o = (size_t)r * 12;
  for (int j = 0; j < 12; ++j) { a.act[o + j] = act[j]; a.mu[o + j] = mu[j]; }
  a.logp[r] = lp;
  a.value[r] = V;
  if (a.u_act) for (int j = 0; j < 12; ++j) a.u_act[o + j] = act[j];
  if (a.u_mu) for (int j = 0; j < 12; ++j) a.u_mu[o + j] = mu[j];
  if (a.u_logp) a.u_logp[r] = lp;
  if (a.u_value) a.u_value[r] = V;
}

void launch_heads(const HeadArgs& a, cudaStream_t st) {
  int smem = (13 * a.nd.H2 + 24) * 4;
  int rows = a.M;
  k_heads<<<(rows + 127) / 128, 128, smem, st>>>(a);
}

// ------------------------------------------------------------------ PPO loss head (fwd + bwd)
constexpr int LOSS_BLOCK = 128;
int loss_head_partial_floats(int H2) { return ((13 * H2 + 25) + 3) / 4 * 4; }
int loss_blocks(int M) { return (M + LOSS_BLOCK - 1) / LOSS_BLOCK; }

__device__ __forceinline__ float elu_grad_from_out(float h) { return h > 0.0f ? 1.0f : h + 1.0f; }

__global__ void __launch_bounds__(LOSS_BLOCK) k_loss_heads(LossArgs a) {
  extern __shared__ float sh[];
  const int H2 = a.nd.H2;
  float* sW4a = sh;
  float* sb4a = sW4a + 12 * H2;
  float* sW4c = sb4a + 12;
  float* sls = sW4c + H2;       // 12
  float* slso = sls + 12;       // 12
  float* sdmu = slso + 12;      // [LOSS_BLOCK][12]
  float* sdls = sdmu + LOSS_BLOCK * 12;  // [LOSS_BLOCK][12]
  float* sdV = sdls + LOSS_BLOCK * 12;   // [LOSS_BLOCK]
  double* sst = reinterpret_cast<double*>(sdV + LOSS_BLOCK);  // [LOSS_BLOCK/32][5]
  for (int k = threadIdx.x; k < 12 * H2; k += blockDim.x) sW4a[k] = a.W4a[k];
  for (int k = threadIdx.x; k < H2; k += blockDim.x) sW4c[k] = a.W4c[k];
  if (threadIdx.x < 12) {
    sb4a[threadIdx.x] = a.b4a[threadIdx.x];
    sls[threadIdx.x] = a.logstd[threadIdx.x];
    slso[threadIdx.x] = a.logstd_old[threadIdx.x];
  }
  __syncthreads();
  const int row0 = blockIdx.x * LOSS_BLOCK;
  const int r = row0 + threadIdx.x;
  const float invM = 1.0f / (float)a.M;
  double st_surr = 0.0, st_vl = 0.0, st_kl = 0.0, st_clip = 0.0, st_bad = 0.0;
  float dmu[12], dls[12], dV = 0.0f;
#pragma unroll
  for (int j = 0; j < 12; ++j) { dmu[j] = 0.0f; dls[j] = 0.0f; }
  if (r < a.M) {
    const __nv_bfloat16* ha = a.H3 + (size_t)r * 2 * H2;
    float mu[12], V;
    head_forward(ha, ha + H2, H2, sW4a, sb4a, sW4c, __ldg(a.b4c), mu, V);
    float act[12];
#pragma unroll
    for (int j = 0; j < 12; ++j) act[j] = a.act[(size_t)r * 12 + j];
    const float lp = logp_gauss(act, mu, sls);
    const float ratio = expf(lp - a.logp_old[r]);
    const float adv = a.adv[r];
    const float s1 = ratio * adv;
    const float rc = fminf(fmaxf(ratio, 1.0f - a.clip), 1.0f + a.clip);
    const float s2 = rc * adv;
    const bool take1 = s1 <= s2;
    const bool inside = ratio >= 1.0f - a.clip && ratio <= 1.0f + a.clip;
    const float dLdr = -(take1 ? adv : (inside ? adv : 0.0f)) * invM;
    const float dLdlp = dLdr * ratio;
    const float Vo = a.V_old[r], ret = a.ret[r];
    const float vd = fminf(fmaxf(V - Vo, -a.vclip), a.vclip);
    const float vc = Vo + vd;
    const float e1 = (V - ret) * (V - ret), e2 = (vc - ret) * (vc - ret);
    const bool take_u = e1 >= e2;
    const bool vin = fabsf(V - Vo) <= a.vclip;
    dV = a.vf_coef * (take_u ? 2.0f * (V - ret) : (vin ? 2.0f * (vc - ret) : 0.0f)) * invM;
    float kl = 0.0f;
#pragma unroll
    for (int j = 0; j < 12; ++j) {
      const float d = act[j] - mu[j];
      const float is2 = expf(-2.0f * sls[j]);
      dmu[j] = dLdlp * d * is2;
      dls[j] = dLdlp * (d * d * is2 - 1.0f);
      const float dm = a.mu_old[(size_t)r * 12 + j] - mu[j];
      kl += sls[j] - slso[j] + (expf(2.0f * slso[j]) + dm * dm) * (0.5f * is2) - 0.5f;
    }
    st_surr = (double)(take1 ? s1 : s2);
    st_vl = (double)(take_u ? e1 : e2);
    st_kl = (double)kl;
    st_clip = fabsf(ratio - 1.0f) > a.clip ? 1.0 : 0.0;
    st_bad = (isfinite(st_surr) && isfinite(st_vl) && isfinite(st_kl)) ? 0.0 : 1.0;
    // dZ3 = (dH3) * ELU'(H3), actor columns then critic columns
    __nv_bfloat16* dz = a.dZ3 + (size_t)r * 2 * H2;
    for (int k = 0; k < H2; k += 8) {
      float h[8], g[8];
      bf16x8(ha + k, h);
      bf16x8(ha + H2 + k, g);
      uint32_t pa[4], pc[4];
#pragma unroll
      for (int e = 0; e < 8; e += 2) {
        float da0 = 0.0f, da1 = 0.0f;
#pragma unroll
        for (int j = 0; j < 12; ++j) {
          da0 = da0 + dmu[j] * sW4a[j * H2 + k + e];
          da1 = da1 + dmu[j] * sW4a[j * H2 + k + e + 1];
        }
        __nv_bfloat162 za = __floats2bfloat162_rn(da0 * elu_grad_from_out(h[e]), da1 * elu_grad_from_out(h[e + 1]));
        __nv_bfloat162 zc = __floats2bfloat162_rn(dV * sW4c[k + e] * elu_grad_from_out(g[e]),
                                                  dV * sW4c[k + e + 1] * elu_grad_from_out(g[e + 1]));
        pa[e / 2] = *reinterpret_cast<uint32_t*>(&za);
        pc[e / 2] = *reinterpret_cast<uint32_t*>(&zc);
      }
      *reinterpret_cast<uint4*>(dz + k) = make_uint4(pa[0], pa[1], pa[2], pa[3]);
      *reinterpret_cast<uint4*>(dz + H2 + k) = make_uint4(pc[0], pc[1], pc[2], pc[3]);
    }
  }
#pragma unroll
  for (int j = 0; j < 12; ++j) { sdmu[threadIdx.x * 12 + j] = dmu[j]; sdls[threadIdx.x * 12 + j] = dls[j]; }
  sdV[threadIdx.x] = dV;
  // block statistics (fixed butterfly order)
  st_surr = warp_sum_d(st_surr); st_vl = warp_sum_d(st_vl); st_kl = warp_sum_d(st_kl);
  st_clip = warp_sum_d(st_clip); st_bad = warp_sum_d(st_bad);
  const int wid = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    sst[wid * 5 + 0] = st_surr; sst[wid * 5 + 1] = st_vl; sst[wid * 5 + 2] = st_kl;
    sst[wid * 5 + 3] = st_clip; sst[wid * 5 + 4] = st_bad;
  }
  __syncthreads();
  float* out = a.part + (size_t)blockIdx.x * a.HP;
  const int nrows = min(LOSS_BLOCK, a.M - row0);
  // dW4a[j][k] = sum_r dmu[r][j] h_a[r][k]; dW4c[k] = sum_r dV[r] h_c[r][k]  (rows in order)
  for (int k = threadIdx.x; k < H2; k += blockDim.x) {
    float acc[12], accc = 0.0f;
#pragma unroll
    for (int j = 0; j < 12; ++j) acc[j] = 0.0f;
    for (int rr = 0; rr < nrows; ++rr) {
      const __nv_bfloat16* hrow = a.H3 + (size_t)(row0 + rr) * 2 * H2;
      const float h = __bfloat162float(hrow[k]), g = __bfloat162float(hrow[H2 + k]);
#pragma unroll
      for (int j = 0; j < 12; ++j) acc[j] = acc[j] + sdmu[rr * 12 + j] * h;
      accc = accc + sdV[rr] * g;
    }
#pragma unroll
    for (int j = 0; j < 12; ++j) out[j * H2 + k] = acc[j];
    out[12 * H2 + 12 + k] = accc;
  }
  if (threadIdx.x < 12) {
    const int j = threadIdx.x;
    float sb = 0.0f, sl = 0.0f;
    for (int rr = 0; rr < nrows; ++rr) { sb = sb + sdmu[rr * 12 + j]; sl = sl + sdls[rr * 12 + j]; }
    out[12 * H2 + j] = sb;
    out[13 * H2 + 13 + j] = sl;
  }
  if (threadIdx.x == 32) {
    float sv = 0.0f;
    for (int rr = 0; rr < nrows; ++rr) sv = sv + sdV[rr];
    out[13 * H2 + 12] = sv;
  }
  if (threadIdx.x < 5) {
    double s = 0.0;
    for (int w = 0; w < LOSS_BLOCK / 32; ++w) s += sst[w * 5 + threadIdx.x];
    a.spart[(size_t)blockIdx.x * 8 + threadIdx.x] = s;
  }
}

void launch_loss_heads(const LossArgs& a, cudaStream_t st) {
  int H2 = a.nd.H2;
  int smem = (13 * H2 + 36 + LOSS_BLOCK * 25) * 4 + 8 + (LOSS_BLOCK / 32) * 5 * 8;
  k_loss_heads<<<loss_blocks(a.M), LOSS_BLOCK, smem, st>>>(a);
}

// sums over blocks (fixed order) -> canonical gradient of heads/log-std + stats payload
__global__ void k_reduce_heads(HeadReduceArgs a) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  const int H2 = a.H2;
  const int nval = 13 * H2 + 25;
  if (e < nval) {
    float s = 0.0f;
    for (int b = 0; b < a.nblk; ++b) s = s + a.part[(size_t)b * a.HP + e];
    long long dst;
    if (e < 12 * H2) dst = a.off_W4a + e;
    else if (e < 12 * H2 + 12) dst = a.off_b4a + (e - 12 * H2);
    else if (e < 13 * H2 + 12) dst = a.off_W4c + (e - 12 * H2 - 12);
    else if (e == 13 * H2 + 12) dst = a.off_b4c;
    else { dst = a.off_logstd + (e - 13 * H2 - 13); s = s - a.ent_coef; }
    a.grad[dst] = s;
    if (!isfinite(s)) atomicAdd(&a.payload[4], 1.0f);
  }
  if (blockIdx.x == 0 && threadIdx.x < 5) {
    double s = 0.0;
    for (int b = 0; b < a.nblk; ++b) s += a.spart[(size_t)b * 8 + threadIdx.x];
    const double invM = 1.0 / (double)a.M;
    if (threadIdx.x == 0) a.payload[1] = (float)(s * invM);       // surrogate mean
    if (threadIdx.x == 1) a.payload[2] = (float)(s * invM);       // value loss mean
    if (threadIdx.x == 2) a.payload[0] = (float)(s * invM);       // KL mean (Alg. 1)
    if (threadIdx.x == 3) a.payload[3] = (float)(s * invM);       // clip fraction
    if (threadIdx.x == 4 && s > 0.0) atomicAdd(&a.payload[4], (float)s);
    if (threadIdx.x == 0) a.payload[5] = 1.0f;                    // rank count (allreduce sums it)
  }
}

void launch_reduce_heads(const HeadReduceArgs& a, cudaStream_t st) {
  int n = 13 * a.H2 + 25;
  k_reduce_heads<<<(n + 127) / 128, 128, 0, st>>>(a);
}

// split-K partials -> canonical W and b gradients (fixed split order)
__global__ void k_reduce_dw(DwReduceArgs a) {
  const int z = blockIdx.z;
  const int per = a.cols + 1;  // cols + bias column
  const long long total = (long long)a.rows * per;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total; e += (long long)gridDim.x * blockDim.x) {
    const int r = (int)(e / per), c = (int)(e % per);
    const int pc = c < a.cols ? c : a.bias_col;
    const float* p = a.part + z * a.zstride + (size_t)r * a.ld + pc;
    float s = 0.0f;
    for (int k = 0; k < a.S; ++k) s = s + p[k * a.sstride];
    int zz = z, rr = r;
    if (a.row_split > 0 && r >= a.row_split) { zz = 1; rr = r - a.row_split; }
    if (c < a.cols) a.grad[a.w_off[zz] + (long long)rr * a.cols + c] = s;
    else a.grad[a.b_off[zz] + rr] = s;
    if (!isfinite(s)) atomicAdd(&a.payload[4], 1.0f);
  }
}

void launch_reduce_dw(const DwReduceArgs& a, cudaStream_t st) {
  long long total = (long long)a.rows * (a.cols + 1);
  int nb = (int)min((total + 255) / 256, 2048LL);
  k_reduce_dw<<<dim3(nb, 1, a.nz), 256, 0, st>>>(a);
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
// step_f = {apply, alpha, bias-correction1, bias-correction2}; iteration accumulators in iter_acc
__global__ void k_alg1_prep(const float* payload, DevScalars* sc, float kl_target, int world, float b1, float b2,
                            float* step_f) {
  const float W = (float)world;
  const float kl = payload[0] / W;
  const bool bad = payload[4] > 0.0f || !isfinite(kl);
  float* acc = step_f + 4;  // iteration accumulators [surr, vloss, kl, clip, count]
  if (bad) {
    sc->nonfinite_skips += 1;
    step_f[0] = 0.0f;
    return;
  }
  float alpha = sc->alpha;
  if (kl > 2.0f * kl_target) alpha = fmaxf(1e-5f, alpha / 1.5f);
  else if (kl < 0.5f * kl_target) alpha = fminf(1e-2f, 1.5f * alpha);
  sc->alpha = alpha;
  sc->kl_last = kl;
  const int t = sc->adam_t + 1;
  sc->adam_t = t;
  sc->applied += 1;
  step_f[0] = 1.0f;
  step_f[1] = alpha;
  step_f[2] = (float)(1.0 - pow((double)b1, (double)t));
  step_f[3] = (float)(1.0 - pow((double)b2, (double)t));
  acc[0] += payload[1] / W; acc[1] += payload[2] / W; acc[2] += kl; acc[3] += payload[3] / W; acc[4] += 1.0f;
}
void launch_alg1_prep(const float* payload, DevScalars* sc, float kl_target, int world, float b1, float b2,
                      float* step_f, cudaStream_t st) {
  k_alg1_prep<<<1, 1, 0, st>>>(payload, sc, kl_target, world, b1, b2, step_f);
}

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

__global__ void k_adam(AdamArgs a, const float* step_f) {
  if (step_f[0] == 0.0f) return;
  const float alpha = step_f[1], bc1 = step_f[2], bc2 = step_f[3];
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < a.sh.P; i += (long long)gridDim.x * blockDim.x) {
    const float g = a.grad[i] * a.inv_world;
    const float m = a.b1 * a.m[i] + (1.0f - a.b1) * g;
    const float v = a.b2 * a.v[i] + (1.0f - a.b2) * g * g;
    a.m[i] = m;
    a.v[i] = v;
    const float mh = m / bc1, vh = v / bc2;
    const float th = a.theta[i] - alpha * mh / (sqrtf(vh) + a.eps);
    a.theta[i] = th;
    write_shadow(a.sh, i, th);
  }
}
void launch_adam(const AdamArgs& a, const float* step_f, cudaStream_t st) {
  int nb = (int)min((a.sh.P + 255) / 256, 148LL * 8);
  k_adam<<<nb, 256, 0, st>>>(a, step_f);
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
  (void)sc;
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
