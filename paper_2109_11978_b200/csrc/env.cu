// env.cu -- environment kernels: reset, transition, reward, flags, curriculum, observation + height
// scan + noise (§3, Tables 2/4; SPEC env/dynamics/curriculum).
// Compiled with -fmad=false: every a*b+c is two IEEE roundings, as in the oracle (R26).
//
// Layout: state SoA [66][N] (field-major, so every field access is coalesced across the warp).
// Kernel shape: k_env_step runs one thread per env for the per-env serial work (push, substeps, reward,
// flags, curriculum, reset) and writes a 256-B observation record per env; k_env_obs then spreads the
// observation rows over the whole GPU: one thread per item = 4 consecutive observation elements of one
// env = exactly one Philox block of noise, written as one 8-byte bf16x4 store (coalesced along a row).
#include "common.cuh"
#include "kernels.h"

namespace lg {

constexpr float M_BASE = 30.0f, GRAV = 9.81f, L_HIP = 0.08f, L_T = 0.35f, L_S = 0.35f;
constexpr float KP = 80.0f, KD = 2.0f, TAU_MAX = 80.0f, J_J = 0.25f, C_J = 0.5f;
constexpr float K_N = 5000.0f, C_N = 100.0f, C_T = 60.0f, R_B = 0.25f, DT_SIM = 0.005f, DT = 0.02f;

__constant__ float c_inertia[3] = {0.5f, 1.7f, 2.0f};
__constant__ float c_inertia_rc[3] = {(float)(1.0 / 0.5), (float)(1.0 / (double)1.7f), (float)(1.0 / 2.0)};

// x / c for the transition model's constant divisors (J_J, M_BASE, the inertias, 0.25, DT): q0 = RN(x rc),
// one fma residual and one fma correction (rc = RN(1/c)). On 2^-100 <= |x| <= 2^100 this equals the IEEE
// quotient RN(x / c) bit for bit for each of these c -- checked over all 2^32 inputs by tools/div_check.cu;
// +-0 keep their sign through q0 = x rc; everything else (denormals, huge, inf, NaN) takes the IEEE division.
// Same result as the oracle's plain x / c, without the division's slow-path branch.
__device__ __forceinline__ float div_const(float x, float c, float rc) {
  const float ax = fabsf(x);
  const float q0 = __fmul_rn(x, rc);
  const float r = __fmaf_rn(-q0, c, x);
  const float q = __fmaf_rn(r, rc, q0);
  if (ax == 0.0f) return q0;
  if (ax >= 0x1p-100f && ax <= 0x1p100f) return q;
  return __fdiv_rn(x, c);
}
constexpr float RC_J = (float)(1.0 / (double)J_J), RC_M = (float)(1.0 / (double)M_BASE),
                RC_DT = (float)(1.0 / (double)DT), RC_Q = (float)(1.0 / 0.25);
__constant__ float c_hip[4][3] = {{0.30f, 0.15f, 0.0f}, {0.30f, -0.15f, 0.0f}, {-0.30f, 0.15f, 0.0f}, {-0.30f, -0.15f, 0.0f}};
__constant__ float c_slat[4] = {1.0f, -1.0f, 1.0f, -1.0f};
__constant__ float c_qdef[12] = {0.0f, 0.7f, -1.4f, 0.0f, 0.7f, -1.4f, 0.0f, -0.7f, 1.4f, 0.0f, -0.7f, 1.4f};

struct St {  // registers of one env (DESIGN.md §3.4 record)
  float p[3], quat[4], v[3], w[3], q[12], qd[12], tair[4], cmd[3], aprev[12], mu, spawn[2];
  uint32_t contact;
  int32_t push_timer, ep_step, level, col;
  uint32_t crossed;
  float ep_return;
};

__device__ __forceinline__ void load_state(const uint32_t* __restrict__ S, int N, int i, St& s) {
  auto f = [&](int w) { return __uint_as_float(S[(size_t)w * N + i]); };
  for (int k = 0; k < 3; ++k) { s.p[k] = f(S_P + k); s.v[k] = f(S_V + k); s.w[k] = f(S_W + k); s.cmd[k] = f(S_CMD + k); }
  for (int k = 0; k < 4; ++k) { s.quat[k] = f(S_QUAT + k); s.tair[k] = f(S_TAIR + k); }
  for (int k = 0; k < 12; ++k) { s.q[k] = f(S_Q + k); s.qd[k] = f(S_QD + k); s.aprev[k] = f(S_APREV + k); }
  s.mu = f(S_MU); s.spawn[0] = f(S_SPAWN); s.spawn[1] = f(S_SPAWN + 1);
  s.contact = S[(size_t)S_CONTACT * N + i];
  s.push_timer = (int32_t)S[(size_t)S_PUSH * N + i];
  s.ep_step = (int32_t)S[(size_t)S_EPSTEP * N + i];
  s.level = (int32_t)S[(size_t)S_LEVEL * N + i];
  s.col = (int32_t)S[(size_t)S_COL * N + i];
  s.crossed = S[(size_t)S_CROSSED * N + i];
  s.ep_return = f(S_EPRET);
}

__device__ __forceinline__ void store_state(uint32_t* __restrict__ S, int N, int i, const St& s) {
  auto f = [&](int w, float v) { S[(size_t)w * N + i] = __float_as_uint(v); };
  for (int k = 0; k < 3; ++k) { f(S_P + k, s.p[k]); f(S_V + k, s.v[k]); f(S_W + k, s.w[k]); f(S_CMD + k, s.cmd[k]); }
  for (int k = 0; k < 4; ++k) { f(S_QUAT + k, s.quat[k]); f(S_TAIR + k, s.tair[k]); }
  for (int k = 0; k < 12; ++k) { f(S_Q + k, s.q[k]); f(S_QD + k, s.qd[k]); f(S_APREV + k, s.aprev[k]); }
  f(S_MU, s.mu); f(S_SPAWN, s.spawn[0]); f(S_SPAWN + 1, s.spawn[1]);
  S[(size_t)S_CONTACT * N + i] = s.contact;
  S[(size_t)S_PUSH * N + i] = (uint32_t)s.push_timer;
  S[(size_t)S_EPSTEP * N + i] = (uint32_t)s.ep_step;
  S[(size_t)S_LEVEL * N + i] = (uint32_t)s.level;
  S[(size_t)S_COL * N + i] = (uint32_t)s.col;
  S[(size_t)S_CROSSED * N + i] = s.crossed;
  f(S_EPRET, s.ep_return);
}

struct Mat3 { float m[3][3]; };

__device__ __forceinline__ Mat3 rot(const float* qt) {
  float w = qt[0], x = qt[1], y = qt[2], z = qt[3];
  Mat3 R;
  R.m[0][0] = 1.0f - 2.0f * (y * y + z * z);
  R.m[0][1] = 2.0f * (x * y - w * z);
  R.m[0][2] = 2.0f * (x * z + w * y);
  R.m[1][0] = 2.0f * (x * y + w * z);
  R.m[1][1] = 1.0f - 2.0f * (x * x + z * z);
  R.m[1][2] = 2.0f * (y * z - w * x);
  R.m[2][0] = 2.0f * (x * z - w * y);
  R.m[2][1] = 2.0f * (y * z + w * x);
  R.m[2][2] = 1.0f - 2.0f * (x * x + y * y);
  return R;
}
__device__ __forceinline__ void mv(const Mat3& R, const float* u, float* o) {
#pragma unroll
  for (int i = 0; i < 3; ++i) o[i] = (R.m[i][0] * u[0] + R.m[i][1] * u[1]) + R.m[i][2] * u[2];
}
__device__ __forceinline__ void mtv(const Mat3& R, const float* u, float* o) {
#pragma unroll
  for (int i = 0; i < 3; ++i) o[i] = (R.m[0][i] * u[0] + R.m[1][i] * u[1]) + R.m[2][i] * u[2];
}
__device__ __forceinline__ void cross3(const float* a, const float* b, float* o) {
  o[0] = a[1] * b[2] - a[2] * b[1];
  o[1] = a[2] * b[0] - a[0] * b[2];
  o[2] = a[0] * b[1] - a[1] * b[0];
}
__device__ __forceinline__ float dot3(const float* a, const float* b) { return (a[0] * b[0] + a[1] * b[1]) + a[2] * b[2]; }

// leg FK (+ Jacobian columns J[col][xyz]) in the base frame, DESIGN.md §3.5
__device__ __forceinline__ void leg_fk(int leg, const float* ql, float lsh, float* pt, float (*J)[3]) {
  float sa, ca, s1, c1, s12, c12;
  sincos_poly(ql[0], sa, ca);
  sincos_poly(ql[1], s1, c1);
  sincos_poly(ql[1] + ql[2], s12, c12);
  float fx = -L_T * s1 - lsh * s12;
  float fy = c_slat[leg] * L_HIP;
  float fz = -L_T * c1 - lsh * c12;
  pt[0] = c_hip[leg][0] + fx;
  pt[1] = c_hip[leg][1] + (fy * ca - fz * sa);
  pt[2] = c_hip[leg][2] + (fy * sa + fz * ca);
  if (J) {
    J[0][0] = 0.0f;
    J[0][1] = -sa * fy - ca * fz;
    J[0][2] = ca * fy - sa * fz;
    float dx = -L_T * c1 - lsh * c12, dz = L_T * s1 + lsh * s12;
    J[1][0] = dx; J[1][1] = -sa * dz; J[1][2] = ca * dz;
    float ex = -lsh * c12, ez = lsh * s12;
    J[2][0] = ex; J[2][1] = -sa * ez; J[2][2] = ca * ez;
  }
}

__device__ __forceinline__ void heading(const Mat3& R, float& c, float& s) {
  float f0 = R.m[0][0], f1 = R.m[1][0];
  float n = sqrtf(f0 * f0 + f1 * f1);
  if (n > 1e-6f) { c = f0 / n; s = f1 / n; } else { c = 1.0f; s = 0.0f; }
}

// reset of env g
__device__ void reset_env(const World& W, const Rng& rng, St& s, uint32_t g, uint32_t ev) {
  U4 b0 = rng.block(0, g, ev, TAG_RESET), b1 = rng.block(1, g, ev, TAG_RESET), b2 = rng.block(2, g, ev, TAG_RESET),
     b3 = rng.block(3, g, ev, TAG_RESET), b4 = rng.block(4, g, ev, TAG_RESET);
  uint32_t wd[20] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w, b2.x, b2.y,
                     b2.z, b2.w, b3.x, b3.y, b3.z, b3.w, b4.x, b4.y, b4.z, b4.w};
  float x = ((float)s.level * 8.0f + 4.0f) + usym(1.0f, wd[0]);
  float y = ((float)s.col * 8.0f + 4.0f) + usym(1.0f, wd[1]);
  float psi = usym(0x1.921fb6p1f, wd[2]);
  float sh, ch;
  sincos_poly(0.5f * psi, sh, ch);
  s.p[0] = x; s.p[1] = y; s.p[2] = h_plate(W, x, y) + 0.6f;
  s.quat[0] = ch; s.quat[1] = 0.0f; s.quat[2] = 0.0f; s.quat[3] = sh;
  for (int k = 0; k < 3; ++k) { s.v[k] = 0.0f; s.w[k] = 0.0f; }
  s.mu = 0.5f + 0.75f * u01(wd[3]);
  for (int k = 0; k < 3; ++k) s.cmd[k] = usym(1.0f, wd[4 + k]);
#pragma unroll
  for (int j = 0; j < 12; ++j) { s.q[j] = c_qdef[j] + usym(0.05f, wd[7 + j]); s.qd[j] = 0.0f; s.aprev[j] = 0.0f; }
  for (int l = 0; l < 4; ++l) s.tair[l] = 0.0f;
  s.contact = 0u; s.push_timer = 0; s.ep_step = 0; s.crossed = 0u;
  s.spawn[0] = x; s.spawn[1] = y; s.ep_return = 0.0f;
}

// per-env observation record for the cooperative phase
struct ObsRec {  // 64 words: everything the observation of one env needs (written by phase A)
  float pro[48];
  float px, py, pz, c, s;
  uint32_t g, word0;
  int32_t row;  // destination row (env index, or compacted terminal row)
  uint32_t pad[8];
};
static_assert(sizeof(ObsRec) == 256, "ObsRec layout");

__device__ __forceinline__ void fill_obs_rec(const St& s, ObsRec& o) {
  Mat3 R = rot(s.quat);
  float t3[3];
  mtv(R, s.v, t3);
  o.pro[0] = t3[0]; o.pro[1] = t3[1]; o.pro[2] = t3[2];
  o.pro[3] = s.w[0]; o.pro[4] = s.w[1]; o.pro[5] = s.w[2];
  o.pro[6] = -R.m[2][0]; o.pro[7] = -R.m[2][1]; o.pro[8] = -R.m[2][2];
  o.pro[9] = s.cmd[0]; o.pro[10] = s.cmd[1]; o.pro[11] = s.cmd[2];
  for (int j = 0; j < 12; ++j) { o.pro[12 + j] = s.q[j]; o.pro[24 + j] = s.qd[j]; o.pro[36 + j] = s.aprev[j]; }
  heading(R, o.c, o.s);
  o.px = s.p[0]; o.py = s.p[1]; o.pz = s.p[2];
}

// Observation rows (DESIGN.md §3.7 step 10): 64 threads per env row (2 rows per 128-thread block, no
// index division); thread gq owns the items gq, gq+64, ...; item gq = the 4 consecutive elements
// [4gq, 4gq+4) = one Philox block of noise words
// (two when a reset shifted the row's first word) and writes them as one 8-byte bf16x4 store. Proprioceptive
// items (4gq < 48) read one float4 of the record; scan items step through the scan grid incrementally.
// Blocks [0, ceil(N/2)) write the post-step rows of OBS slot `slot`; with `with_terminal` the next
// ceil(N/2) blocks write the pre-reset rows of this step's time-outs (records < n_to_slot[ev & 1]) into the rollout's
// compacted time-out buffer (row = the record's destination row).
__constant__ float c_noise_scale[48] = {0.01f, 0.01f, 0.01f, 0.2f, 0.2f, 0.2f, 0.05f, 0.05f, 0.05f, 0.0f, 0.0f, 0.0f,
                                        0.01f, 0.01f, 0.01f, 0.01f, 0.01f, 0.01f, 0.01f, 0.01f, 0.01f, 0.01f, 0.01f, 0.01f,
                                        1.5f, 1.5f, 1.5f, 1.5f, 1.5f, 1.5f, 1.5f, 1.5f, 1.5f, 1.5f, 1.5f, 1.5f,
                                        0.0f, 0.0f, 0.0f, 0.0f, 0.0f, 0.0f, 0.0f, 0.0f, 0.0f, 0.0f, 0.0f, 0.0f};
constexpr int OBS_ROWS_PER_BLOCK = 2;  // same-box A/B: 1 row +1.1 %, 4 rows +0.6 %

__global__ void __launch_bounds__(64 * OBS_ROWS_PER_BLOCK) k_env_obs(EnvParams P, int ev_off,
                                                                     __nv_bfloat16* __restrict__ dst_bf16,
                                                                     float* __restrict__ dst_f32, int with_terminal) {
  pdl_trigger();
  pdl_wait();
  const int D = P.obs_dim, Dp = P.obs_stride, G = Dp / 4;
  const uint32_t ev = P.scalars->s_base + (uint32_t)ev_off;
  const int nb_main = (P.N + OBS_ROWS_PER_BLOCK - 1) / OBS_ROWS_PER_BLOCK;
  int r = (int)blockIdx.x * OBS_ROWS_PER_BLOCK + (int)(threadIdx.x >> 6);
  const ObsRec* recs = reinterpret_cast<const ObsRec*>(P.recs);
  __nv_bfloat16* dst = dst_bf16;
  float* df = dst_f32;
  if ((int)blockIdx.x >= nb_main) {
    if (!with_terminal) return;
    r -= nb_main * OBS_ROWS_PER_BLOCK;
    if (r >= P.scalars->n_to_slot[ev & 1u]) return;
    recs = reinterpret_cast<const ObsRec*>(P.trecs);
    dst = P.term_obs;
    df = nullptr;
  } else if (r >= P.N) {
    return;
  }
  const ObsRec* o = recs + r;
  const int row = o->row;
  if (row < 0) return;  // time-out beyond the compacted buffer's capacity (not reachable for T <= 1000)
  for (int gq = threadIdx.x & 63; gq < G; gq += 64) {
  const int e0 = 4 * gq;
  float v[4] = {0.0f, 0.0f, 0.0f, 0.0f};
  float sc[4] = {0.0f, 0.0f, 0.0f, 0.0f};
  if (e0 < 48) {
    const float4 p4 = *reinterpret_cast<const float4*>(o->pro + e0);
    v[0] = p4.x; v[1] = p4.y; v[2] = p4.z; v[3] = p4.w;
#pragma unroll
    for (int j = 0; j < 4; ++j) sc[j] = c_noise_scale[e0 + j];
  } else {
    World W{P.hf, P.R, P.C, P.inv_cell};
    const float px = o->px, py = o->py, pz = o->pz, c = o->c, sn = o->s;
    const int k0 = e0 - 48;
    int ix = (int)(((uint32_t)k0 * P.ny_magic) >> 20), iy = k0 - ix * P.scan_ny;  // k0 / ny, exact (host check)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      if (e0 + j < D) {
        const float dx = (float)(ix - P.scan_nx / 2) * 0.1f;
        const float dy = (float)(iy - P.scan_ny / 2) * 0.1f;
        const float x = px + (c * dx - sn * dy);
        const float y = py + (sn * dx + c * dy);
        v[j] = pz - h_bilinear(W, x, y);
        sc[j] = 0.1f;
      }
      if (++iy == P.scan_ny) { iy = 0; ++ix; }
    }
  }
  if ((P.flags & F_NOISE) && (sc[0] != 0.0f || sc[1] != 0.0f || sc[2] != 0.0f || sc[3] != 0.0f)) {
    Rng rng{P.seed_lo, P.seed_hi};
    const uint32_t wbase = o->word0 + 4u * (uint32_t)gq;
    const U4 nb0 = rng.block(wbase >> 2, o->g, ev, TAG_OBS);
    // words wbase .. wbase+3 = the 4-word window at offset wbase % 4 of [nb0 | nb1] (the offset is the row's,
    // so uniform across the warp)
    uint32_t wd[4] = {nb0.x, nb0.y, nb0.z, nb0.w};
    const uint32_t sh = wbase & 3u;
    if (sh) {
      const U4 nb1 = rng.block((wbase >> 2) + 1, o->g, ev, TAG_OBS);
      if (sh == 1) { wd[0] = nb0.y; wd[1] = nb0.z; wd[2] = nb0.w; wd[3] = nb1.x; }
      else if (sh == 2) { wd[0] = nb0.z; wd[1] = nb0.w; wd[2] = nb1.x; wd[3] = nb1.y; }
      else { wd[0] = nb0.w; wd[1] = nb1.x; wd[2] = nb1.y; wd[3] = nb1.z; }
    }
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if (sc[j] != 0.0f) v[j] = v[j] + usym(sc[j], wd[j]);
  }
  if (df) {
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if (e0 + j < D) df[(size_t)row * D + e0 + j] = v[j];
  }
  __nv_bfloat162 lo = __floats2bfloat162_rn(v[0], v[1]), hi = __floats2bfloat162_rn(v[2], v[3]);
  uint2 pk;
  pk.x = *reinterpret_cast<uint32_t*>(&lo);
  pk.y = *reinterpret_cast<uint32_t*>(&hi);
  *reinterpret_cast<uint2*>(dst + (size_t)row * Dp + e0) = pk;
  }
}

static void launch_obs(const EnvParams& P, int ev_off, __nv_bfloat16* dst, float* f32, int with_terminal,
                       cudaStream_t st) {
  const int nb_main = (P.N + OBS_ROWS_PER_BLOCK - 1) / OBS_ROWS_PER_BLOCK;
  launch_pdl(k_env_obs, dim3(nb_main * (with_terminal ? 2 : 1)), dim3(64 * OBS_ROWS_PER_BLOCK), 0, st, P, ev_off, dst, f32,
             with_terminal);
}

// ------------------------------------------------------------------ kernels
__global__ void __launch_bounds__(ENV_BLOCK) k_env_reset(EnvParams P, const uint8_t* __restrict__ mask, int init) {
  World W{P.hf, P.R, P.C, P.inv_cell};
  Rng rng{P.seed_lo, P.seed_hi};
  const uint32_t ev = P.scalars->s_base;
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= P.N) return;
  St s;
  load_state(P.state, P.N, i, s);
  uint32_t g = (uint32_t)(P.rank * P.N + i);
  if (!mask || mask[i]) {
    if (init) { s.col = (int32_t)(g % (uint32_t)P.n_cols); s.level = 0; }
    reset_env(W, rng, s, g, ev);
    store_state(P.state, P.N, i, s);
  }
  ObsRec& rec = reinterpret_cast<ObsRec*>(P.recs)[i];
  fill_obs_rec(s, rec);
  rec.g = g; rec.word0 = 0u; rec.row = i;
}

// ------------------------------------------------------------------ leg-parallel transition
// k_env_step: a group of 4 consecutive lanes per env; lane l owns leg l (its 3 joints: targets, torques,
// FK/Jacobian, contact force, joint accelerations, air time). The base state is replicated in the 4 lanes
// and updated identically. Every sum the definition takes over legs or joints is formed in every lane of
// the group from group shuffles, in the definition's order (legs 0..3, joints 0..11), so the result is
// bit-identical to the sequential form (-fmad=false).
struct Com {  // per-env common state (identical copy in every lane of the group)
  float p[3], quat[4], v[3], w[3], cmd[3], mu, spawn[2];
  uint32_t contact;
  int32_t push_timer, ep_step, level, col;
  uint32_t crossed;
  float ep_return;
};
struct Leg {  // the lane's own leg
  float q[3], qd[3], aprev[3], tair;
};

__device__ __forceinline__ void load_com(const uint32_t* __restrict__ S, int N, int i, Com& c) {
  auto f = [&](int w) { return __uint_as_float(S[(size_t)w * N + i]); };
  for (int k = 0; k < 3; ++k) { c.p[k] = f(S_P + k); c.v[k] = f(S_V + k); c.w[k] = f(S_W + k); c.cmd[k] = f(S_CMD + k); }
  for (int k = 0; k < 4; ++k) c.quat[k] = f(S_QUAT + k);
  c.mu = f(S_MU); c.spawn[0] = f(S_SPAWN); c.spawn[1] = f(S_SPAWN + 1);
  c.contact = S[(size_t)S_CONTACT * N + i];
  c.push_timer = (int32_t)S[(size_t)S_PUSH * N + i];
  c.ep_step = (int32_t)S[(size_t)S_EPSTEP * N + i];
  c.level = (int32_t)S[(size_t)S_LEVEL * N + i];
  c.col = (int32_t)S[(size_t)S_COL * N + i];
  c.crossed = S[(size_t)S_CROSSED * N + i];
  c.ep_return = f(S_EPRET);
}
__device__ __forceinline__ void load_leg(const uint32_t* __restrict__ S, int N, int i, int l, Leg& g) {
  auto f = [&](int w) { return __uint_as_float(S[(size_t)w * N + i]); };
  for (int k = 0; k < 3; ++k) { g.q[k] = f(S_Q + 3 * l + k); g.qd[k] = f(S_QD + 3 * l + k); g.aprev[k] = f(S_APREV + 3 * l + k); }
  g.tair = f(S_TAIR + l);
}
__device__ __forceinline__ void store_com(uint32_t* __restrict__ S, int N, int i, const Com& c) {
  auto f = [&](int w, float v) { S[(size_t)w * N + i] = __float_as_uint(v); };
  for (int k = 0; k < 3; ++k) { f(S_P + k, c.p[k]); f(S_V + k, c.v[k]); f(S_W + k, c.w[k]); f(S_CMD + k, c.cmd[k]); }
  for (int k = 0; k < 4; ++k) f(S_QUAT + k, c.quat[k]);
  f(S_MU, c.mu); f(S_SPAWN, c.spawn[0]); f(S_SPAWN + 1, c.spawn[1]);
  S[(size_t)S_CONTACT * N + i] = c.contact;
  S[(size_t)S_PUSH * N + i] = (uint32_t)c.push_timer;
  S[(size_t)S_EPSTEP * N + i] = (uint32_t)c.ep_step;
  S[(size_t)S_LEVEL * N + i] = (uint32_t)c.level;
  S[(size_t)S_COL * N + i] = (uint32_t)c.col;
  S[(size_t)S_CROSSED * N + i] = c.crossed;
  f(S_EPRET, c.ep_return);
}
__device__ __forceinline__ void store_leg(uint32_t* __restrict__ S, int N, int i, int l, const Leg& g) {
  auto f = [&](int w, float v) { S[(size_t)w * N + i] = __float_as_uint(v); };
  for (int k = 0; k < 3; ++k) { f(S_Q + 3 * l + k, g.q[k]); f(S_QD + 3 * l + k, g.qd[k]); f(S_APREV + 3 * l + k, g.aprev[k]); }
  f(S_TAIR + l, g.tair);
}

// reset (same draws as reset_env): common part in every lane, joints of the own leg
__device__ void reset_group(const World& W, const Rng& rng, Com& c, Leg& g, int l, uint32_t gid, uint32_t ev) {
  U4 b0 = rng.block(0, gid, ev, TAG_RESET), b1 = rng.block(1, gid, ev, TAG_RESET), b2 = rng.block(2, gid, ev, TAG_RESET),
     b3 = rng.block(3, gid, ev, TAG_RESET), b4 = rng.block(4, gid, ev, TAG_RESET);
  uint32_t wd[20] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w, b2.x, b2.y,
                     b2.z, b2.w, b3.x, b3.y, b3.z, b3.w, b4.x, b4.y, b4.z, b4.w};
  float x = ((float)c.level * 8.0f + 4.0f) + usym(1.0f, wd[0]);
  float y = ((float)c.col * 8.0f + 4.0f) + usym(1.0f, wd[1]);
  float psi = usym(0x1.921fb6p1f, wd[2]);
  float sh, ch;
  sincos_poly(0.5f * psi, sh, ch);
  c.p[0] = x; c.p[1] = y; c.p[2] = h_plate(W, x, y) + 0.6f;
  c.quat[0] = ch; c.quat[1] = 0.0f; c.quat[2] = 0.0f; c.quat[3] = sh;
  for (int k = 0; k < 3; ++k) { c.v[k] = 0.0f; c.w[k] = 0.0f; }
  c.mu = 0.5f + 0.75f * u01(wd[3]);
  for (int k = 0; k < 3; ++k) c.cmd[k] = usym(1.0f, wd[4 + k]);
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const int j = 3 * l + k;
    // word 7 + j by selects on the leg (a lane-indexed wd[] would live in local memory)
    const uint32_t wq = l == 0 ? wd[7 + k] : (l == 1 ? wd[10 + k] : (l == 2 ? wd[13 + k] : wd[16 + k]));
    g.q[k] = c_qdef[j] + usym(0.05f, wq);
    g.qd[k] = 0.0f;
    g.aprev[k] = 0.0f;
  }
  g.tair = 0.0f;
  c.contact = 0u; c.push_timer = 0; c.ep_step = 0; c.crossed = 0u;
  c.spawn[0] = x; c.spawn[1] = y; c.ep_return = 0.0f;
}

// observation record: common part from lane 0 of the group, joint columns from every lane
__device__ __forceinline__ void fill_rec_group(const Com& c, const Leg& g, int l, ObsRec& o) {
  if (l == 0) {
    Mat3 R = rot(c.quat);
    float t3[3];
    mtv(R, c.v, t3);
    o.pro[0] = t3[0]; o.pro[1] = t3[1]; o.pro[2] = t3[2];
    o.pro[3] = c.w[0]; o.pro[4] = c.w[1]; o.pro[5] = c.w[2];
    o.pro[6] = -R.m[2][0]; o.pro[7] = -R.m[2][1]; o.pro[8] = -R.m[2][2];
    o.pro[9] = c.cmd[0]; o.pro[10] = c.cmd[1]; o.pro[11] = c.cmd[2];
    heading(R, o.c, o.s);
    o.px = c.p[0]; o.py = c.p[1]; o.pz = c.p[2];
  }
  for (int k = 0; k < 3; ++k) {
    o.pro[12 + 3 * l + k] = g.q[k];
    o.pro[24 + 3 * l + k] = g.qd[k];
    o.pro[36 + 3 * l + k] = g.aprev[k];
  }
}

// ordered sum over the 12 joints (j = 3L + k) of a per-lane triple, identical in every lane of the group
__device__ __forceinline__ float joint_sum(const float* x3, int gbase, unsigned gm) {
  float s = 0.0f;
#pragma unroll
  for (int L = 0; L < 4; ++L)
#pragma unroll
    for (int k = 0; k < 3; ++k) s = s + __shfl_sync(gm, x3[k], gbase + L);
  return s;
}

constexpr int STEP_THREADS = 64;  // 16 envs per block (256 blocks at 4096 envs: every SM gets one; same-box A/B -0.1 % vs 128)

__global__ void __launch_bounds__(STEP_THREADS) k_env_step(EnvParams P, int t, const float* __restrict__ actions,
                                                            float* __restrict__ rew_out,
                                                            uint8_t* __restrict__ term_out, uint8_t* __restrict__ to_out,
                                                            float* __restrict__ terms_out) {
  pdl_trigger();
  pdl_wait();
  World W{P.hf, P.R, P.C, P.inv_cell};
  Rng rng{P.seed_lo, P.seed_hi};
  const uint32_t ev = P.scalars->s_base + (uint32_t)t + 1u;
  if (blockIdx.x == 0 && threadIdx.x == 0) P.scalars->n_to_slot[(ev + 1u) & 1u] = 0;  // the next step's counter
  const int N = P.N;
  const int gt = blockIdx.x * blockDim.x + threadIdx.x;
  if ((gt & ~31) >= 4 * N) return;  // whole warps beyond the last env leave
  // every lane of a live warp runs the step (lanes past the last env shadow env N-1 and write nothing), so
  // the per-env group sums are full-warp shuffles: a shuffle with a 4-lane member mask compiles to a
  // vote / branch loop that cost ~25 % of the kernel's issue slots in branch resolution
  const bool live = (gt >> 2) < N;
  const int i = live ? gt >> 2 : N - 1, l = gt & 3;
  const int lane = threadIdx.x & 31, gbase = lane & ~3;
  const unsigned gm = 0xFu << gbase;  // the group's lanes (shuffles inside group-divergent branches)
  constexpr unsigned FULL = 0xffffffffu;
  Com c;
  Leg g;
  load_com(P.state, N, i, c);
  load_leg(P.state, N, i, l, g);
  const uint32_t gid = (uint32_t)(P.rank * N + i);
  float a[3], qstar[3], tau[3], qdd[3];
  const float* ap = actions + (size_t)i * 12 + 3 * l;
#pragma unroll
  for (int k = 0; k < 3; ++k) { a[k] = ap[k]; qstar[k] = c_qdef[3 * l + k] + 0.5f * a[k]; }
  if ((P.flags & F_PUSH) && c.push_timer >= 500) {
    U4 pb = rng.block(0, gid, ev, TAG_PUSH);
    c.v[0] = c.v[0] + usym(1.0f, pb.x);
    c.v[1] = c.v[1] + usym(1.0f, pb.y);
    c.push_timer = 0;
  }
  float airsum = 0.0f;
  int crash = 0;
  for (int sub = 0; sub < 4; ++sub) {
    Mat3 R = rot(c.quat);
    float ww[3];
    mv(R, c.w, ww);
#pragma unroll
    for (int k = 0; k < 3; ++k) tau[k] = clampf_(KP * (qstar[k] - g.q[k]) - KD * g.qd[k], -TAU_MAX, TAU_MAX);
    float f[3] = {0.0f, 0.0f, 0.0f}, rf[3];
    bool touch;
    {
      float fb[3], J[3][3], r[3], pf[3], jq[3], rj[3], cr[3], vf[3];
      leg_fk(l, g.q, L_S, fb, J);
      mv(R, fb, r);
      for (int k = 0; k < 3; ++k) pf[k] = c.p[k] + r[k];
      for (int k = 0; k < 3; ++k) jq[k] = (J[0][k] * g.qd[0] + J[1][k] * g.qd[1]) + J[2][k] * g.qd[2];
      cross3(ww, r, cr);
      mv(R, jq, rj);
      for (int k = 0; k < 3; ++k) vf[k] = (c.v[k] + cr[k]) + rj[k];
      float delta = h_plate(W, pf[0], pf[1]) - pf[2];
      touch = delta > 0.0f;
      if (touch) {
        float fn = fmaxf(0.0f, K_N * delta - C_N * vf[2]);
        float vt = sqrtf(vf[0] * vf[0] + vf[1] * vf[1]);
        float sc = vt > 0.0f ? fminf(C_T, (c.mu * fn) / vt) : 0.0f;
        f[0] = -sc * vf[0];
        f[1] = -sc * vf[1];
        f[2] = fn;
      }
      float fbb[3];
      mtv(R, f, fbb);
      float tc0 = dot3(J[0], fbb), tc1 = dot3(J[1], fbb), tc2 = dot3(J[2], fbb);
      qdd[0] = div_const((tau[0] + tc0) - C_J * g.qd[0], J_J, RC_J);
      qdd[1] = div_const((tau[1] + tc1) - C_J * g.qd[1], J_J, RC_J);
      qdd[2] = div_const((tau[2] + tc2) - C_J * g.qd[2], J_J, RC_J);
      cross3(r, f, rf);
    }
    const uint32_t contact = (__ballot_sync(FULL, touch) >> gbase) & 0xFu;
    float F[3] = {0.0f, 0.0f, 0.0f}, Tw[3] = {0.0f, 0.0f, 0.0f};
#pragma unroll
    for (int L = 0; L < 4; ++L)
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        F[k] = F[k] + __shfl_sync(FULL, f[k], gbase + L);
        Tw[k] = Tw[k] + __shfl_sync(FULL, rf[k], gbase + L);
      }
    F[2] = F[2] - M_BASE * GRAV;
    float tb[3], Iw[3], gy[3], wdot[3];
    mtv(R, Tw, tb);
    for (int k = 0; k < 3; ++k) Iw[k] = c_inertia[k] * c.w[k];
    cross3(c.w, Iw, gy);
    for (int k = 0; k < 3; ++k) wdot[k] = div_const(tb[k] - gy[k], c_inertia[k], c_inertia_rc[k]);
    for (int k = 0; k < 3; ++k) c.v[k] = c.v[k] + DT_SIM * div_const(F[k], M_BASE, RC_M);
    for (int k = 0; k < 3; ++k) c.w[k] = c.w[k] + DT_SIM * wdot[k];
#pragma unroll
    for (int k = 0; k < 3; ++k) g.qd[k] = g.qd[k] + DT_SIM * qdd[k];
    for (int k = 0; k < 3; ++k) c.p[k] = c.p[k] + DT_SIM * c.v[k];
#pragma unroll
    for (int k = 0; k < 3; ++k) g.q[k] = g.q[k] + DT_SIM * g.qd[k];
    {
      float h = 0.5f * DT_SIM;
      float w = c.quat[0], x = c.quat[1], y = c.quat[2], z = c.quat[3];
      float o0 = c.w[0], o1 = c.w[1], o2 = c.w[2];
      float w2 = w + h * (((-x * o0) - y * o1) - z * o2);
      float x2 = x + h * ((w * o0 + y * o2) - z * o1);
      float y2 = y + h * ((w * o1 + z * o0) - x * o2);
      float z2 = z + h * ((w * o2 + x * o1) - y * o0);
      float n = sqrtf(((w2 * w2 + x2 * x2) + y2 * y2) + z2 * z2);
      c.quat[0] = w2 / n; c.quat[1] = x2 / n; c.quat[2] = y2 / n; c.quat[3] = z2 / n;
    }
    {
      const uint32_t cn = (contact >> l) & 1u, cp = (c.contact >> l) & 1u;
      const bool td = cn && !cp;
      float term = 0.0f;
      if (td) { term = g.tair - 0.5f; g.tair = 0.0f; }
      else if (!cn) g.tair = g.tair + DT_SIM;
      const uint32_t tds = (__ballot_sync(FULL, td) >> gbase) & 0xFu;
#pragma unroll
      for (int L = 0; L < 4; ++L) {
        const float tL = __shfl_sync(FULL, term, gbase + L);
        if ((tds >> L) & 1u) airsum = airsum + tL;
      }
    }
    c.contact = contact;
    if (c.p[2] - h_plate(W, c.p[0], c.p[1]) < R_B) crash = 1;
  }
  // knees (R9)
  Mat3 R = rot(c.quat);
  int n_c;
  {
    float kb[3], r[3];
    leg_fk(l, g.q, 0.5f * L_S, kb, nullptr);
    mv(R, kb, r);
    float kx = c.p[0] + r[0], ky = c.p[1] + r[1], kz = c.p[2] + r[2];
    const bool kin = h_plate(W, kx, ky) - kz > 0.0f;
    n_c = __popc((__ballot_sync(FULL, kin) >> gbase) & 0xFu);
  }
  c.ep_step += 1;
  c.push_timer += 1;
  {
    float x0 = (float)c.level * 8.0f, y0 = (float)c.col * 8.0f;
    if (c.p[0] < x0 || c.p[0] >= x0 + 8.0f || c.p[1] < y0 || c.p[1] >= y0 + 8.0f) c.crossed = 1u;
  }
  bool fin = true;
  for (int k = 0; k < 3; ++k) fin = fin && isfinite(c.p[k]) && isfinite(c.v[k]) && isfinite(c.w[k]);
  for (int k = 0; k < 4; ++k) fin = fin && isfinite(c.quat[k]);
  for (int k = 0; k < 3; ++k) fin = fin && isfinite(g.q[k]) && isfinite(g.qd[k]);
  const bool finite = ((__ballot_sync(FULL, fin) >> gbase) & 0xFu) == 0xFu;
  // reward
  float rt[9];
  {
    float cc, sn, wv[3];
    heading(R, cc, sn);
    float vh0 = cc * c.v[0] + sn * c.v[1];
    float vh1 = -sn * c.v[0] + cc * c.v[1];
    float vh2 = c.v[2];
    mv(R, c.w, wv);
    float wh0 = cc * wv[0] + sn * wv[1];
    float wh1 = -sn * wv[0] + cc * wv[1];
    float wh2 = wv[2];
    float ex = c.cmd[0] - vh0, ey = c.cmd[1] - vh1, ez = c.cmd[2] - wh2;
    rt[0] = (1.0f * DT) * exp_poly(-div_const(ex * ex + ey * ey, 0.25f, RC_Q));
    rt[1] = (0.5f * DT) * exp_poly(-div_const(ez * ez, 0.25f, RC_Q));
    rt[2] = (-4.0f * DT) * (vh2 * vh2);
    rt[3] = (-0.05f * DT) * (wh0 * wh0 + wh1 * wh1);
    float x3[3];
    for (int k = 0; k < 3; ++k) x3[k] = qdd[k] * qdd[k];
    const float sa = joint_sum(x3, gbase, FULL);
    for (int k = 0; k < 3; ++k) x3[k] = g.qd[k] * g.qd[k];
    const float sb = joint_sum(x3, gbase, FULL);
    rt[4] = (-0.001f * DT) * (sa + sb);
    for (int k = 0; k < 3; ++k) x3[k] = tau[k] * tau[k];
    rt[5] = (-0.00002f * DT) * joint_sum(x3, gbase, FULL);
    for (int k = 0; k < 3; ++k) {
      float qprev = c_qdef[3 * l + k] + 0.5f * g.aprev[k];
      float d = div_const(qstar[k] - qprev, DT, RC_DT);
      x3[k] = d * d;
    }
    rt[6] = (-0.25f * DT) * joint_sum(x3, gbase, FULL);
    rt[7] = (-0.001f * DT) * (float)n_c;
    rt[8] = (2.0f * DT) * airsum;
  }
  float r = rt[0];
  for (int k = 1; k < 9; ++k) r = r + rt[k];
  if (!finite) { r = 0.0f; for (int k = 0; k < 9; ++k) rt[k] = 0.0f; }
  c.ep_return = c.ep_return + r;
  const bool terminated = crash || !finite;
  const bool to = (c.ep_step >= 1000) && !terminated;
  const bool done = terminated || to;
  for (int k = 0; k < 3; ++k) g.aprev[k] = a[k];
  if (!live) return;  // shadow lanes past the last env: no stores (no shuffles follow outside the group)
  const size_t ti = (size_t)t * N + i;
  if (l == 0) {
    P.reward[ti] = r;
    P.flags_out[ti] = (uint8_t)((terminated ? 1u : 0u) | (to ? 2u : 0u));
    P.boot[ti] = 0.0f;
    if (rew_out) rew_out[i] = r;
    if (term_out) term_out[i] = (uint8_t)terminated;
    if (to_out) to_out[i] = (uint8_t)to;
  }
  if (terms_out) {  // lane l writes terms l, l+4, l+8
#pragma unroll
    for (int k = 0; k < 9; ++k)  // constant indices keep rt[] in registers (a lane-indexed rt[k] put it in local memory)
      if ((k & 3) == l) terms_out[(size_t)i * 9 + k] = rt[k];
  }
  if (done) {  // group-uniform
    if (to && (P.flags & F_BOOTSTRAP)) {
      // record r of this step (k_env_obs writes its observation) -> row grow of the rollout's compacted
      // time-out buffer, evaluated by the critic once after the rollout (storage_compute_gae)
      int row = 0, grow = 0;
      if (l == 0) { row = atomicAdd(&P.scalars->n_to_slot[ev & 1u], 1); grow = atomicAdd(&P.scalars->n_to_total, 1); }
      row = __shfl_sync(gm, row, gbase);
      grow = __shfl_sync(gm, grow, gbase);
      ObsRec& tr = reinterpret_cast<ObsRec*>(P.trecs)[row];
      fill_rec_group(c, g, l, tr);
      if (l == 0) {
        tr.g = gid; tr.word0 = 0u;
        tr.row = grow < P.to_cap ? grow : -1;
        if (grow < P.to_cap) P.term_idx[grow] = t * N + i;
      }
    }
    if (l == 0) {  // episode statistics (stats only; float atomics)
      const float fx = c.ep_return * 16777216.0f;  // exact power-of-two scaling, then one rounding to an integer
      if (isfinite(fx) && fabsf(fx) < 9.0e18f)
        atomicAdd(reinterpret_cast<unsigned long long*>(&P.scalars->ep_return_fx), (unsigned long long)__float2ll_rn(fx));
      atomicAdd(reinterpret_cast<unsigned long long*>(&P.scalars->ep_len_sum), (unsigned long long)c.ep_step);
      if (!finite) atomicAdd(&P.scalars->nonfinite_envs, 1);
      atomicAdd(&P.scalars->episodes, 1);
    }
    if (P.flags & F_CURRICULUM) {
      int old = c.level;
      if (c.crossed) {
        c.level = c.level + 1;
        if (c.level > P.n_levels - 1) {
          uint32_t wrd = rng.block(0, gid, ev, TAG_CURR).x;
          c.level = (int32_t)(((uint64_t)wrd * (uint64_t)P.n_levels) >> 32);
        }
      } else {
        float dx = c.p[0] - c.spawn[0], dy = c.p[1] - c.spawn[1];
        float T = (float)c.ep_step * DT;
        float hh = 0.5f * T;
        if ((dx * dx + dy * dy) < (hh * hh) * (c.cmd[0] * c.cmd[0] + c.cmd[1] * c.cmd[1])) c.level = max(0, c.level - 1);
      }
      if (l == 0) {
        if (c.level > old) atomicAdd(&P.scalars->promotions, 1);
        if (c.level < old) atomicAdd(&P.scalars->demotions, 1);
      }
    }
    reset_group(W, rng, c, g, l, gid, ev);
  }
  if (l == 0) store_com(P.state, N, i, c);
  store_leg(P.state, N, i, l, g);
  ObsRec& rec = reinterpret_cast<ObsRec*>(P.recs)[i];
  fill_rec_group(c, g, l, rec);
  if (l == 0) { rec.g = gid; rec.word0 = done ? (uint32_t)P.obs_dim : 0u; rec.row = i; }
}

// standalone curriculum rule (DESIGN.md §3.7 step 9(ii))
__global__ void k_curriculum(int n, int n_levels, const uint8_t* crossed, const float* disp, const float* cmd,
                             const int32_t* ep_steps, const uint32_t* words, int32_t* level) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int lv = level[i];
  if (crossed[i]) {
    lv = lv + 1;
    if (lv > n_levels - 1) lv = (int32_t)(((uint64_t)words[i] * (uint64_t)n_levels) >> 32);
  } else {
    float dx = disp[2 * i], dy = disp[2 * i + 1], c0 = cmd[2 * i], c1 = cmd[2 * i + 1];
    float T = (float)ep_steps[i] * DT;
    float hh = 0.5f * T;
    if ((dx * dx + dy * dy) < (hh * hh) * (c0 * c0 + c1 * c1)) lv = max(0, lv - 1);
  }
  level[i] = lv;
}

// Gaussian ε for the policy head: eps[i][12] for step event ev
__device__ void action_eps(const Rng& rng, uint32_t g, uint32_t ev, float* eps) {
  U4 b0 = rng.block(0, g, ev, TAG_ACTION), b1 = rng.block(1, g, ev, TAG_ACTION), b2 = rng.block(2, g, ev, TAG_ACTION);
  uint32_t w[12] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w, b2.x, b2.y, b2.z, b2.w};
#pragma unroll
  for (int k = 0; k < 6; ++k) {
    float u1 = (float)((w[2 * k] >> 8) + 1u) * 0x1p-24f;
    float u2 = (float)(w[2 * k + 1] >> 8) * 0x1p-24f;
    float rr = sqrtf(-2.0f * log_poly(u1));
    float sn, cs;
    sincos_poly(0x1.921fb6p2f * u2, sn, cs);
    eps[2 * k] = rr * cs;
    eps[2 * k + 1] = rr * sn;
  }
}

__global__ void k_action_eps(int N, int rank, uint32_t seed_lo, uint32_t seed_hi, const DevScalars* sc, int t, float* eps) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N) return;
  Rng rng{seed_lo, seed_hi};
  action_eps(rng, (uint32_t)(rank * N + i), sc->s_base + (uint32_t)t + 1u, eps + (size_t)i * 12);
}

// World heightfield (reading R27): block (i, c, l) writes row i
// of tile (level l, column c), one thread per cell j; the obstacle boxes of the tile (10 Philox blocks) are
// drawn once per block into shared memory. fp32 with explicit rounding (this file is built -fmad=false).
__global__ void __launch_bounds__(128) k_terrain(const __grid_constant__ TerrainArgs a) {
  const int i = blockIdx.x, c = blockIdx.y, l = blockIdx.z, j = threadIdx.x;
  const int kind = c % 5;
  const uint32_t tile = (uint32_t)(l * a.n_cols + c);
  const Rng rng{a.seed_lo, a.seed_hi};
  const float d = a.n_levels > 1 ? __fdiv_rn((float)l, (float)(a.n_levels - 1)) : 0.0f;
  __shared__ int bi0[8], bi1[8], bj0[8], bj1[8];
  __shared__ float bh[8];
  if (kind == 3 && j < 8) {  // box b = j: words 5b .. 5b+4 = width, length, x0, y0, height
    uint32_t w[5];
#pragma unroll
    for (int k = 0; k < 5; ++k) {
      const uint32_t wi = 5u * (uint32_t)j + (uint32_t)k;
      w[k] = pick(rng.block(wi >> 2, tile, 0u, TAG_TERRAIN), wi);
    }
    const float wd = __fadd_rn(0.5f, __fmul_rn(1.5f, u01(w[0])));
    const float ln = __fadd_rn(0.5f, __fmul_rn(1.5f, u01(w[1])));
    const float x0 = __fmul_rn(8.0f, u01(w[2]));
    const float y0 = __fmul_rn(8.0f, u01(w[3]));
    bh[j] = usym(__fadd_rn(0.05f, __fmul_rn(0.15f, d)), w[4]);
    bi0[j] = (int)__fmul_rn(x0, 10.0f);
    bi1[j] = (int)__fmul_rn(fminf(8.0f, __fadd_rn(x0, wd)), 10.0f);
    bj0[j] = (int)__fmul_rn(y0, 10.0f);
    bj1[j] = (int)__fmul_rn(fminf(8.0f, __fadd_rn(y0, ln)), 10.0f);
  }
  __syncthreads();
  if (j >= 80) return;
  const float xc = __fmul_rn((float)(2 * i + 1), 0.05f), yc = __fmul_rn((float)(2 * j + 1), 0.05f);
  const float e = fminf(fminf(xc, __fsub_rn(8.0f, xc)), fminf(yc, __fsub_rn(8.0f, yc)));
  const float ep = fminf(e, 3.0f);
  float h = 0.0f;
  if (kind == 1) {
    h = __fmul_rn(a.slope[l], ep);
  } else if (kind == 2) {
    const uint32_t wi = (uint32_t)(i * 80 + j);
    const float half = __fmul_rn(0.5f, __fmul_rn(0.05f, __fadd_rn(1.0f, d)));
    h = usym(half, pick(rng.block(wi >> 2, tile, 0u, TAG_TERRAIN), wi));
  } else if (kind == 3) {
#pragma unroll
    for (int b = 0; b < 8; ++b)
      if (i >= bi0[b] && i < bi1[b] && j >= bj0[b] && j < bj1[b]) h = bh[b];
    if (e >= 3.0f) h = 0.0f;
  } else if (kind == 4) {
    h = __fmul_rn(__fadd_rn(0.05f, __fmul_rn(0.15f, d)), floorf(__fdiv_rn(ep, 0.3f)));
  }
  a.hf[(size_t)(l * 80 + i) * (size_t)(a.n_cols * 80) + (size_t)(c * 80 + j)] = h;
}

// ------------------------------------------------------------------ launchers
void launch_terrain(const TerrainArgs& a, cudaStream_t st) {
  k_terrain<<<dim3(80, a.n_cols, a.n_levels), 128, 0, st>>>(a);
}
void launch_env_reset(const EnvParams& P, const uint8_t* mask, int init, float* obs_f32, cudaStream_t st) {
  int nb = (P.N + ENV_BLOCK - 1) / ENV_BLOCK;
  k_env_reset<<<nb, ENV_BLOCK, 0, st>>>(P, mask, init);
  launch_obs(P, 0, P.obs_out, obs_f32, 0, st);  // noise event s_base
}
void launch_env_step(const EnvParams& P, int t, const float* actions, float* obs_f32, float* rew, uint8_t* term,
                     uint8_t* to, float* terms, cudaStream_t st) {
  const long long threads = 4LL * P.N;
  launch_pdl(k_env_step, dim3((unsigned)((threads + STEP_THREADS - 1) / STEP_THREADS)), dim3(STEP_THREADS), 0, st, P, t,
             actions, rew, term, to, terms);
  launch_obs(P, t + 1, P.obs_out + (size_t)(t + 1) * P.N * P.obs_stride, obs_f32, (P.flags & F_BOOTSTRAP) ? 1 : 0,
             st);  // noise event s_base + t + 1
}
void launch_curriculum(int n, int n_levels, const uint8_t* crossed, const float* disp, const float* cmd,
                       const int32_t* ep, const uint32_t* words, int32_t* level, cudaStream_t st) {
  k_curriculum<<<(n + 127) / 128, 128, 0, st>>>(n, n_levels, crossed, disp, cmd, ep, words, level);
}
void launch_action_eps(int N, int rank, uint32_t s0, uint32_t s1, const DevScalars* sc, int t, float* eps,
                       cudaStream_t st) {
  k_action_eps<<<(N + 127) / 128, 128, 0, st>>>(N, rank, s0, s1, sc, t, eps);
}

}  // namespace lg
