/*
 * oracle/env_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, single-threaded CPU oracle of the environment side of the hot path of
 * Rudin et al., "Learning to Walk in Minutes Using Massively Parallel Deep RL" (arXiv 2109.11978).
 * It is written from the frozen definitions in DESIGN.md §3 (which restate PAPER.md / SPEC.md; each
 * function cites the passage it follows) and shares no code with paper_2109_11978_b200/.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may load it.
 *
 * Arithmetic: IEEE fp32, round-to-nearest-even, compiled with -ffp-contract=off (no FMA), every
 * expression evaluated in the order DESIGN.md §3 writes it. (R26: the environment decides
 * integer outcomes -- contact, crash, curriculum level -- in the kernel's precision.)
 *
 * Pins (tests/test_oracle_env.py): Philox known-answer vectors; polynomial sin/cos/exp/log vs libm
 * within a few ulp; plate/bilinear hand grids; PD/contact/free-fall closed forms
 * (S:184-186); FK straight leg and yaw equivariance; settling to m·g
 * (S:204); reward examples; observation examples; curriculum examples
 * and exhaustive L=3 sequences; Feistel bijection.
 * Multi-step transition: pinned in flight by the closed forms of its integrator over 80 substeps (free fall,
 * torque-free spin about a principal axis, a PD-driven joint: test_flight_trajectory_closed_forms) and in contact
 * by the settling equilibrium. Between those, a contact-rich trajectory is "parity unpinned": it is fixed
 * only by DESIGN.md §3.5, which both sides implement (the GPU is bit-exact to it).
 */
#include <math.h>
#include <stdint.h>
#include <string.h>

#define OR_NW 66
#define OR_TAG_RESET 1u
#define OR_TAG_OBS 2u
#define OR_TAG_ACTION 3u
#define OR_TAG_PUSH 4u
#define OR_TAG_CURR 5u
#define OR_TAG_SHUFFLE 6u

#define OR_F_CURRICULUM 1u
#define OR_F_NOISE 2u
#define OR_F_PUSH 4u
#define OR_F_BOOTSTRAP 8u

typedef struct {
  int32_t n_envs;     /* envs on this rank */
  int32_t rank;       /* global env id g = rank*n_envs + i */
  int32_t n_levels;   /* tile rows (x) */
  int32_t n_cols;     /* tile columns (y) */
  int32_t scan_nx, scan_ny; /* 17, 11 (0,0 = flat, 48-dim obs) */
  uint32_t flags;
  uint32_t seed_lo, seed_hi;
  float inv_cell;     /* 10.0f, passed not computed */
} or_env_cfg;

typedef struct {
  float p[3], quat[4], v[3], w[3], q[12], qd[12], tair[4], cmd[3], aprev[12], mu, spawn[2];
  uint32_t contact;
  int32_t push_timer, ep_step, level, col;
  uint32_t crossed;
  float ep_return;
} or_state;

typedef char or_state_size_check[(sizeof(or_state) == OR_NW * 4) ? 1 : -1];

/* ---------------- DESIGN.md §3.1  Philox4x32-10 (Salmon et al. SC'11) ---------------- */
void or_philox(uint32_t k0, uint32_t k1, const uint32_t ctr[4], uint32_t out[4]) {
  uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
  for (int r = 0; r < 10; ++r) {
    uint64_t p0 = (uint64_t)0xD2511F53u * c0;
    uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
    uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    c0 = hi1 ^ c1 ^ k0;
    c1 = lo1;
    c2 = hi0 ^ c3 ^ k1;
    c3 = lo0;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* word w of stream (id, event, tag) */
uint32_t or_word(const or_env_cfg* cfg, uint32_t id, uint32_t event, uint32_t tag, uint32_t w) {
  uint32_t ctr[4] = {w / 4u, id, event, tag}, out[4];
  or_philox(cfg->seed_lo, cfg->seed_hi, ctr, out);
  return out[w % 4u];
}

static float u01(uint32_t x) { return (float)(x >> 8) * 0x1p-24f; }
static float usym(float s, uint32_t x) { float t = 2.0f * u01(x) - 1.0f; return s * t; }

/* ---------------- DESIGN.md §3.2 polynomial transcendentals ---------------- */
void or_sincos(float x, float* sn, float* cs) {
  float k = rintf(x * 0x1.45f306p-1f);
  float r = (x - k * 0x1.92p0f) - k * 0x1.fb5444p-12f;
  float r2 = r * r;
  float ps = ((0x1.71de3ap-19f * r2 + -0x1.a01a02p-13f) * r2 + 0x1.111112p-7f) * r2 + -0x1.555556p-3f;
  float s = r + (r * r2) * ps;
  float pc = (((-0x1.27e4fcp-22f * r2 + 0x1.a01a02p-16f) * r2 + -0x1.6c16c2p-10f) * r2 + 0x1.555556p-5f) * r2 + -0x1p-1f;
  float c = 1.0f + r2 * pc;
  int q = ((int)k) & 3;
  if (q == 0) { *sn = s; *cs = c; }
  else if (q == 1) { *sn = c; *cs = -s; }
  else if (q == 2) { *sn = -s; *cs = -c; }
  else { *sn = -c; *cs = s; }
}

static float clampf(float v, float lo, float hi) { return fminf(fmaxf(v, lo), hi); }

float or_exp(float x) {
  x = clampf(x, -87.0f, 88.0f);
  float k = rintf(x * 0x1.715476p0f);
  float r = (x - k * 0x1.62e4p-1f) - k * 0x1.7f7d1cp-20f;
  float p = 0x1.a01a02p-13f;
  p = p * r + 0x1.6c16c2p-10f;
  p = p * r + 0x1.111112p-7f;
  p = p * r + 0x1.555556p-5f;
  p = p * r + 0x1.555556p-3f;
  p = p * r + 0x1p-1f;
  p = p * r + 1.0f;
  p = p * r + 1.0f;
  int ki = (int)k;
  uint32_t bits = (uint32_t)(ki + 127) << 23;
  float two_k;
  memcpy(&two_k, &bits, 4);
  return p * two_k;
}

float or_log(float x) {
  uint32_t bits;
  memcpy(&bits, &x, 4);
  int e = (int)((bits >> 23) & 255u) - 127;
  uint32_t mb = (bits & 0x7fffffu) | 0x3f800000u;
  float m;
  memcpy(&m, &mb, 4);
  if (m > 0x1.6a09e6p0f) { m = m * 0.5f; e = e + 1; }
  float s = (m - 1.0f) / (m + 1.0f);
  float s2 = s * s;
  float p = (((s2 * 0x1.c71c72p-4f + 0x1.24924ap-3f) * s2 + 0x1.99999ap-3f) * s2 + 0x1.555556p-2f) * s2 + 1.0f;
  return (2.0f * s) * p + (float)e * 0x1.62e43p-1f;
}

/* ---------------- DESIGN.md §3.3 height lookups (S:62-70 plate; BJ bilinear) ---------------- */
float or_h_plate(const float* hf, int R, int C, float inv_cell, float x, float y) {
  float fx = clampf(x * inv_cell, 0.0f, (float)R);
  float fy = clampf(y * inv_cell, 0.0f, (float)C);
  int i = (int)ceilf(fx) - 1;
  int j = (int)ceilf(fy) - 1;
  if (i < 0) i = 0;
  if (i > R - 1) i = R - 1;
  if (j < 0) j = 0;
  if (j > C - 1) j = C - 1;
  return hf[(size_t)i * (size_t)C + (size_t)j];
}

float or_h_bilinear(const float* hf, int R, int C, float inv_cell, float x, float y) {
  float fx = clampf(x * inv_cell - 0.5f, 0.0f, (float)(R - 1));
  float fy = clampf(y * inv_cell - 0.5f, 0.0f, (float)(C - 1));
  int i0 = (int)floorf(fx);
  int j0 = (int)floorf(fy);
  if (i0 > R - 2) i0 = R - 2;
  if (j0 > C - 2) j0 = C - 2;
  float tx = fx - (float)i0;
  float ty = fy - (float)j0;
  float h00 = hf[(size_t)i0 * C + j0], h10 = hf[(size_t)(i0 + 1) * C + j0];
  float h01 = hf[(size_t)i0 * C + j0 + 1], h11 = hf[(size_t)(i0 + 1) * C + j0 + 1];
  float lo = (1.0f - tx) * h00 + tx * h10;
  float hi = (1.0f - tx) * h01 + tx * h11;
  return (1.0f - ty) * lo + ty * hi;
}

/* ---------------- DESIGN.md §3.5 model constants (S:222-226 + R24) ---------------- */
static const float M_BASE = 30.0f;
static const float INERTIA[3] = {0.5f, 1.7f, 2.0f};
static const float HIP[4][3] = {{0.30f, 0.15f, 0.0f}, {0.30f, -0.15f, 0.0f}, {-0.30f, 0.15f, 0.0f}, {-0.30f, -0.15f, 0.0f}};
static const float SLAT[4] = {1.0f, -1.0f, 1.0f, -1.0f};
static const float L_HIP = 0.08f, L_T = 0.35f, L_S = 0.35f;
static const float QDEF12[12] = {0.0f, 0.7f, -1.4f, 0.0f, 0.7f, -1.4f, 0.0f, -0.7f, 1.4f, 0.0f, -0.7f, 1.4f};
static const float KP = 80.0f, KD = 2.0f, TAU_MAX = 80.0f, J_J = 0.25f, C_J = 0.5f;
static const float K_N = 5000.0f, C_N = 100.0f, C_T = 60.0f, R_B = 0.25f, GRAV = 9.81f;
static const float DT_SIM = 0.005f, DT = 0.02f;
static float g_last_fz; /* diagnostic: sum of contact normal forces in the last substep */

static void rot_from_quat(const float* qt, float R[3][3]) {
  float w = qt[0], x = qt[1], y = qt[2], z = qt[3];
  R[0][0] = 1.0f - 2.0f * (y * y + z * z);
  R[0][1] = 2.0f * (x * y - w * z);
  R[0][2] = 2.0f * (x * z + w * y);
  R[1][0] = 2.0f * (x * y + w * z);
  R[1][1] = 1.0f - 2.0f * (x * x + z * z);
  R[1][2] = 2.0f * (y * z - w * x);
  R[2][0] = 2.0f * (x * z - w * y);
  R[2][1] = 2.0f * (y * z + w * x);
  R[2][2] = 1.0f - 2.0f * (x * x + y * y);
}
static void mv(const float R[3][3], const float* u, float* o) {
  for (int i = 0; i < 3; ++i) o[i] = (R[i][0] * u[0] + R[i][1] * u[1]) + R[i][2] * u[2];
}
static void mtv(const float R[3][3], const float* u, float* o) {
  for (int i = 0; i < 3; ++i) o[i] = (R[0][i] * u[0] + R[1][i] * u[1]) + R[2][i] * u[2];
}
static void cross3(const float* a, const float* b, float* o) {
  o[0] = a[1] * b[2] - a[2] * b[1];
  o[1] = a[2] * b[0] - a[0] * b[2];
  o[2] = a[0] * b[1] - a[1] * b[0];
}
static float dot3(const float* a, const float* b) { return (a[0] * b[0] + a[1] * b[1]) + a[2] * b[2]; }

/* Leg forward kinematics and Jacobian, DESIGN.md §3.5. lshank = L_S (foot) or 0.5*L_S (knee) */
void or_leg_fk(int leg, const float* ql, float lshank, float* pt, float J[3][3] /* J[col][xyz] */) {
  float sa, ca, s1, c1, s12, c12;
  or_sincos(ql[0], &sa, &ca);
  or_sincos(ql[1], &s1, &c1);
  or_sincos(ql[1] + ql[2], &s12, &c12);
  float fx = -L_T * s1 - lshank * s12;
  float fy = SLAT[leg] * L_HIP;
  float fz = -L_T * c1 - lshank * c12;
  pt[0] = HIP[leg][0] + fx;
  pt[1] = HIP[leg][1] + (fy * ca - fz * sa);
  pt[2] = HIP[leg][2] + (fy * sa + fz * ca);
  if (J) {
    J[0][0] = 0.0f;
    J[0][1] = -sa * fy - ca * fz;
    J[0][2] = ca * fy - sa * fz;
    float dx = -L_T * c1 - lshank * c12, dz = L_T * s1 + lshank * s12;
    J[1][0] = dx; J[1][1] = -sa * dz; J[1][2] = ca * dz;
    float ex = -lshank * c12, ez = lshank * s12;
    J[2][0] = ex; J[2][1] = -sa * ez; J[2][2] = ca * ez;
  }
}

/* Penalty contact: returns 1 if in contact, force f = ground reaction on the foot. */
int or_contact_force(float h_ground, const float* pf, const float* vf, float mu, float* f) {
  float delta = h_ground - pf[2];
  f[0] = 0.0f; f[1] = 0.0f; f[2] = 0.0f;
  if (delta > 0.0f) {
    float fn = fmaxf(0.0f, K_N * delta - C_N * vf[2]);
    float vt = sqrtf(vf[0] * vf[0] + vf[1] * vf[1]);
    float sc = vt > 0.0f ? fminf(C_T, (mu * fn) / vt) : 0.0f;
    f[0] = -sc * vf[0];
    f[1] = -sc * vf[1];
    f[2] = fn;
    return 1;
  }
  return 0;
}

static int finite_state(const or_state* st) {
  const float* f = st->p;
  for (int k = 0; k < 3 + 4 + 3 + 3 + 12 + 12; ++k)
    if (!isfinite(f[k])) return 0;
  return 1;
}

/* heading (c,s) from R·x̂ */
static void heading(const float R[3][3], float* c, float* s) {
  float f0 = R[0][0], f1 = R[1][0];
  float n = sqrtf(f0 * f0 + f1 * f1);
  if (n > 1e-6f) { *c = f0 / n; *s = f1 / n; }
  else { *c = 1.0f; *s = 0.0f; }
}

static const float NOISE_SCALE[5] = {0.01f, 0.2f, 0.05f, 0.01f, 1.5f};

static int obs_dim(const or_env_cfg* cfg) { return 48 + cfg->scan_nx * cfg->scan_ny; }

/* Observation, DESIGN.md §3.7 (Table 4). word0 = first noise word. */
static void env_obs_one(const or_env_cfg* cfg, const float* hf, const or_state* st, uint32_t g, uint32_t s,
                        uint32_t word0, float* o) {
  int R_ = cfg->n_levels * 80, C_ = cfg->n_cols * 80;
  float R[3][3];
  rot_from_quat(st->quat, R);
  float t3[3];
  mtv(R, st->v, t3);
  o[0] = t3[0]; o[1] = t3[1]; o[2] = t3[2];
  o[3] = st->w[0]; o[4] = st->w[1]; o[5] = st->w[2];
  o[6] = -R[2][0]; o[7] = -R[2][1]; o[8] = -R[2][2];
  o[9] = st->cmd[0]; o[10] = st->cmd[1]; o[11] = st->cmd[2];
  for (int j = 0; j < 12; ++j) { o[12 + j] = st->q[j]; o[24 + j] = st->qd[j]; o[36 + j] = st->aprev[j]; }
  int nx = cfg->scan_nx, ny = cfg->scan_ny;
  if (nx * ny > 0) {
    float c, sn;
    heading(R, &c, &sn);
    for (int ix = 0; ix < nx; ++ix)
      for (int iy = 0; iy < ny; ++iy) {
        int k = ny * ix + iy;
        float dx = (float)(ix - nx / 2) * 0.1f;
        float dy = (float)(iy - ny / 2) * 0.1f;
        float x = st->p[0] + (c * dx - sn * dy);
        float y = st->p[1] + (sn * dx + c * dy);
        o[48 + k] = st->p[2] - or_h_bilinear(hf, R_, C_, cfg->inv_cell, x, y);
      }
  }
  if (cfg->flags & OR_F_NOISE) {
    int D = obs_dim(cfg);
    for (int e = 0; e < D; ++e) {
      float sc;
      if (e < 3) sc = NOISE_SCALE[0];
      else if (e < 6) sc = NOISE_SCALE[1];
      else if (e < 9) sc = NOISE_SCALE[2];
      else if (e < 12) continue;
      else if (e < 24) sc = NOISE_SCALE[3];
      else if (e < 36) sc = NOISE_SCALE[4];
      else if (e < 48) continue;
      else sc = 0.1f;
      o[e] = o[e] + usym(sc, or_word(cfg, g, s, OR_TAG_OBS, word0 + (uint32_t)e));
    }
  }
}

/* Reset / spawn */
static void env_reset_one(const or_env_cfg* cfg, const float* hf, or_state* st, uint32_t g, uint32_t s) {
  int R_ = cfg->n_levels * 80, C_ = cfg->n_cols * 80;
  uint32_t wd[19];
  for (uint32_t w = 0; w < 19; ++w) wd[w] = or_word(cfg, g, s, OR_TAG_RESET, w);
  float x = ((float)st->level * 8.0f + 4.0f) + usym(1.0f, wd[0]);
  float y = ((float)st->col * 8.0f + 4.0f) + usym(1.0f, wd[1]);
  float psi = usym(0x1.921fb6p1f, wd[2]);
  float sh, ch;
  or_sincos(0.5f * psi, &sh, &ch);
  st->p[0] = x; st->p[1] = y; st->p[2] = or_h_plate(hf, R_, C_, cfg->inv_cell, x, y) + 0.6f;
  st->quat[0] = ch; st->quat[1] = 0.0f; st->quat[2] = 0.0f; st->quat[3] = sh;
  for (int k = 0; k < 3; ++k) { st->v[k] = 0.0f; st->w[k] = 0.0f; }
  st->mu = 0.5f + 0.75f * u01(wd[3]);
  for (int k = 0; k < 3; ++k) st->cmd[k] = usym(1.0f, wd[4 + k]);
  for (int j = 0; j < 12; ++j) {
    st->q[j] = QDEF12[j] + usym(0.05f, wd[7 + j]);
    st->qd[j] = 0.0f;
    st->aprev[j] = 0.0f;
  }
  for (int l = 0; l < 4; ++l) st->tair[l] = 0.0f;
  st->contact = 0u;
  st->push_timer = 0;
  st->ep_step = 0;
  st->crossed = 0u;
  st->spawn[0] = x; st->spawn[1] = y;
  st->ep_return = 0.0f;
}

/* Game-inspired curriculum, DESIGN.md §3.7 step 9(ii) */
int32_t or_curriculum_level(int32_t level, int32_t n_levels, uint32_t crossed, float dx, float dy,
                            float c0, float c1, int32_t ep_steps, uint32_t loop_word) {
  if (crossed) {
    level = level + 1;
    if (level > n_levels - 1) level = (int32_t)(((uint64_t)loop_word * (uint64_t)n_levels) >> 32);
    return level;
  }
  float T = (float)ep_steps * DT;
  float hh = 0.5f * T;
  if ((dx * dx + dy * dy) < (hh * hh) * (c0 * c0 + c1 * c1)) {
    level = level - 1;
    if (level < 0) level = 0;
  }
  return level;
}

/* Transition, DESIGN.md §3.5 -- returns nonfinite flag. */
static void transition_one(const or_env_cfg* cfg, const float* hf, or_state* st, const float* a, uint32_t g,
                           uint32_t s, float qstar[12], float tau[12], float qdd[12], float* airsum,
                           int* crash, int* n_c) {
  int R_ = cfg->n_levels * 80, C_ = cfg->n_cols * 80;
  for (int j = 0; j < 12; ++j) qstar[j] = QDEF12[j] + 0.5f * a[j];
  if ((cfg->flags & OR_F_PUSH) && st->push_timer >= 500) {
    st->v[0] = st->v[0] + usym(1.0f, or_word(cfg, g, s, OR_TAG_PUSH, 0));
    st->v[1] = st->v[1] + usym(1.0f, or_word(cfg, g, s, OR_TAG_PUSH, 1));
    st->push_timer = 0;
  }
  *airsum = 0.0f;
  *crash = 0;
  for (int sub = 0; sub < 4; ++sub) {
    float R[3][3], ww[3];
    rot_from_quat(st->quat, R);
    mv(R, st->w, ww);
    for (int j = 0; j < 12; ++j)
      tau[j] = clampf(KP * (qstar[j] - st->q[j]) - KD * st->qd[j], -TAU_MAX, TAU_MAX);
    float F[3] = {0.0f, 0.0f, 0.0f}, Tw[3] = {0.0f, 0.0f, 0.0f};
    uint32_t contact = 0u;
    for (int l = 0; l < 4; ++l) {
      float fb_[3], J[3][3];
      or_leg_fk(l, &st->q[3 * l], L_S, fb_, J);
      float r[3], pf[3], jq[3], rj[3], cr[3], vf[3];
      mv(R, fb_, r);
      for (int k = 0; k < 3; ++k) pf[k] = st->p[k] + r[k];
      const float* qdl = &st->qd[3 * l];
      for (int k = 0; k < 3; ++k) jq[k] = (J[0][k] * qdl[0] + J[1][k] * qdl[1]) + J[2][k] * qdl[2];
      cross3(ww, r, cr);
      mv(R, jq, rj);
      for (int k = 0; k < 3; ++k) vf[k] = (st->v[k] + cr[k]) + rj[k];
      float f[3];
      if (or_contact_force(or_h_plate(hf, R_, C_, cfg->inv_cell, pf[0], pf[1]), pf, vf, st->mu, f))
        contact |= (1u << l);
      float fbb[3], tc[3];
      mtv(R, f, fbb);
      tc[0] = dot3(J[0], fbb);
      tc[1] = dot3(J[1], fbb);
      tc[2] = dot3(J[2], fbb);
      for (int k = 0; k < 3; ++k) {
        int j = 3 * l + k;
        qdd[j] = ((tau[j] + tc[k]) - C_J * st->qd[j]) / J_J;
      }
      float rf[3];
      cross3(r, f, rf);
      for (int k = 0; k < 3; ++k) { F[k] = F[k] + f[k]; Tw[k] = Tw[k] + rf[k]; }
    }
    g_last_fz = F[2];
    F[2] = F[2] - M_BASE * GRAV;
    float tb[3], Iw[3], gy[3], wdot[3];
    mtv(R, Tw, tb);
    for (int k = 0; k < 3; ++k) Iw[k] = INERTIA[k] * st->w[k];
    cross3(st->w, Iw, gy);
    for (int k = 0; k < 3; ++k) wdot[k] = (tb[k] - gy[k]) / INERTIA[k];
    for (int k = 0; k < 3; ++k) st->v[k] = st->v[k] + DT_SIM * (F[k] / M_BASE);
    for (int k = 0; k < 3; ++k) st->w[k] = st->w[k] + DT_SIM * wdot[k];
    for (int j = 0; j < 12; ++j) st->qd[j] = st->qd[j] + DT_SIM * qdd[j];
    for (int k = 0; k < 3; ++k) st->p[k] = st->p[k] + DT_SIM * st->v[k];
    for (int j = 0; j < 12; ++j) st->q[j] = st->q[j] + DT_SIM * st->qd[j];
    {
      float h = 0.5f * DT_SIM;
      float w = st->quat[0], x = st->quat[1], y = st->quat[2], z = st->quat[3];
      float o0 = st->w[0], o1 = st->w[1], o2 = st->w[2];
      float w2 = w + h * (((-x * o0) - y * o1) - z * o2);
      float x2 = x + h * ((w * o0 + y * o2) - z * o1);
      float y2 = y + h * ((w * o1 + z * o0) - x * o2);
      float z2 = z + h * ((w * o2 + x * o1) - y * o0);
      float n = sqrtf(((w2 * w2 + x2 * x2) + y2 * y2) + z2 * z2);
      st->quat[0] = w2 / n; st->quat[1] = x2 / n; st->quat[2] = y2 / n; st->quat[3] = z2 / n;
    }
    for (int l = 0; l < 4; ++l) {
      int c_now = (contact >> l) & 1u, c_prev = (st->contact >> l) & 1u;
      if (c_now && !c_prev) { *airsum = *airsum + (st->tair[l] - 0.5f); st->tair[l] = 0.0f; }
      else if (!c_now) st->tair[l] = st->tair[l] + DT_SIM;
    }
    st->contact = contact;
    if (st->p[2] - or_h_plate(hf, R_, C_, cfg->inv_cell, st->p[0], st->p[1]) < R_B) *crash = 1;
  }
  /* collisions: knees below the plate after the last substep (R9) */
  {
    float R[3][3];
    rot_from_quat(st->quat, R);
    int nc = 0;
    for (int l = 0; l < 4; ++l) {
      float kb[3], r[3];
      or_leg_fk(l, &st->q[3 * l], 0.5f * L_S, kb, 0);
      mv(R, kb, r);
      float kx = st->p[0] + r[0], ky = st->p[1] + r[1], kz = st->p[2] + r[2];
      if (or_h_plate(hf, R_, C_, cfg->inv_cell, kx, ky) - kz > 0.0f) nc = nc + 1;
    }
    *n_c = nc;
  }
  st->ep_step += 1;
  st->push_timer += 1;
  {
    float x0 = (float)st->level * 8.0f, y0 = (float)st->col * 8.0f;
    if (st->p[0] < x0 || st->p[0] >= x0 + 8.0f || st->p[1] < y0 || st->p[1] >= y0 + 8.0f) st->crossed = 1u;
  }
}

/* Reward, DESIGN.md §3.6 (Table 2). terms[9] out. */
static float reward_one(const or_state* st, const float qstar[12], const float tau[12], const float qdd[12],
                        float airsum, int n_c, float* terms) {
  float R[3][3], c, s, ww[3];
  rot_from_quat(st->quat, R);
  heading(R, &c, &s);
  float vh0 = c * st->v[0] + s * st->v[1];
  float vh1 = -s * st->v[0] + c * st->v[1];
  float vh2 = st->v[2];
  mv(R, st->w, ww);
  float wh0 = c * ww[0] + s * ww[1];
  float wh1 = -s * ww[0] + c * ww[1];
  float wh2 = ww[2];
  float ex = st->cmd[0] - vh0, ey = st->cmd[1] - vh1, ez = st->cmd[2] - wh2;
  float r[9];
  r[0] = (1.0f * DT) * or_exp(-((ex * ex + ey * ey) / 0.25f));
  r[1] = (0.5f * DT) * or_exp(-((ez * ez) / 0.25f));
  r[2] = (-4.0f * DT) * (vh2 * vh2);
  r[3] = (-0.05f * DT) * (wh0 * wh0 + wh1 * wh1);
  float sa = 0.0f, sb = 0.0f, st_ = 0.0f, sr = 0.0f;
  for (int j = 0; j < 12; ++j) sa = sa + qdd[j] * qdd[j];
  for (int j = 0; j < 12; ++j) sb = sb + st->qd[j] * st->qd[j];
  r[4] = (-0.001f * DT) * (sa + sb);
  for (int j = 0; j < 12; ++j) st_ = st_ + tau[j] * tau[j];
  r[5] = (-0.00002f * DT) * st_;
  for (int j = 0; j < 12; ++j) {
    float qprev = QDEF12[j] + 0.5f * st->aprev[j];
    float d = (qstar[j] - qprev) / DT;
    sr = sr + d * d;
  }
  r[6] = (-0.25f * DT) * sr;
  r[7] = (-0.001f * DT) * (float)n_c;
  r[8] = (2.0f * DT) * airsum;
  float tot = r[0];
  for (int k = 1; k < 9; ++k) tot = tot + r[k];
  if (terms)
    for (int k = 0; k < 9; ++k) terms[k] = r[k];
  return tot;
}

/* ---------------- exported batch entry points ---------------- */

/* env_reset: mask==NULL -> all envs; init!=0 also sets col = g mod n_cols, level = 0. */
void or_env_reset(const or_env_cfg* cfg, const float* hf, or_state* st, const uint8_t* mask, int init,
                  uint32_t s, float* obs) {
  int D = obs_dim(cfg);
  for (int i = 0; i < cfg->n_envs; ++i) {
    if (mask && !mask[i]) continue;
    uint32_t g = (uint32_t)(cfg->rank * cfg->n_envs + i);
    if (init) {
      st[i].col = (int32_t)(g % (uint32_t)cfg->n_cols);
      st[i].level = 0;
    }
    env_reset_one(cfg, hf, &st[i], g, s);
    if (obs) env_obs_one(cfg, hf, &st[i], g, s, 0u, obs + (size_t)i * D);
  }
}

void or_env_obs(const or_env_cfg* cfg, const float* hf, const or_state* st, uint32_t s, uint32_t word0, float* obs) {
  int D = obs_dim(cfg);
  for (int i = 0; i < cfg->n_envs; ++i) {
    uint32_t g = (uint32_t)(cfg->rank * cfg->n_envs + i);
    env_obs_one(cfg, hf, &st[i], g, s, word0, obs + (size_t)i * D);
  }
}

/* env_step_obs_reward for step counter value s (already incremented by the caller).
 * term_obs: [N][D], written only for time-out rows when BOOTSTRAP is on (others untouched). */
void or_env_step(const or_env_cfg* cfg, const float* hf, or_state* st, const float* actions, uint32_t s,
                 float* obs, float* rew, uint8_t* term, uint8_t* timeout, float* terms, float* term_obs) {
  int D = obs_dim(cfg);
  for (int i = 0; i < cfg->n_envs; ++i) {
    uint32_t g = (uint32_t)(cfg->rank * cfg->n_envs + i);
    or_state* e = &st[i];
    const float* a = actions + (size_t)i * 12;
    float qstar[12], tau[12], qdd[12], airsum, tr[9];
    int crash, n_c;
    transition_one(cfg, hf, e, a, g, s, qstar, tau, qdd, &airsum, &crash, &n_c);
    int nonfinite = !finite_state(e);
    float r = reward_one(e, qstar, tau, qdd, airsum, n_c, tr);
    if (nonfinite) {
      r = 0.0f;
      for (int k = 0; k < 9; ++k) tr[k] = 0.0f;
    }
    e->ep_return = e->ep_return + r;
    int terminated = crash || nonfinite;
    int to = (e->ep_step >= 1000) && !terminated;
    int done = terminated || to;
    for (int j = 0; j < 12; ++j) e->aprev[j] = a[j];
    rew[i] = r;
    term[i] = (uint8_t)terminated;
    timeout[i] = (uint8_t)to;
    if (terms)
      for (int k = 0; k < 9; ++k) terms[(size_t)i * 9 + k] = tr[k];
    if (done) {
      if (to && (cfg->flags & OR_F_BOOTSTRAP) && term_obs) env_obs_one(cfg, hf, e, g, s, 0u, term_obs + (size_t)i * D);
      if (cfg->flags & OR_F_CURRICULUM) {
        e->level = or_curriculum_level(e->level, cfg->n_levels, e->crossed, e->p[0] - e->spawn[0],
                                       e->p[1] - e->spawn[1], e->cmd[0], e->cmd[1], e->ep_step,
                                       or_word(cfg, g, s, OR_TAG_CURR, 0));
      }
      env_reset_one(cfg, hf, e, g, s);
    }
    if (obs) env_obs_one(cfg, hf, e, g, s, done ? (uint32_t)D : 0u, obs + (size_t)i * D);
  }
}

/* Gaussian noise for action sampling: eps [N][12] */
void or_action_eps(const or_env_cfg* cfg, uint32_t s, float* eps) {
  for (int i = 0; i < cfg->n_envs; ++i) {
    uint32_t g = (uint32_t)(cfg->rank * cfg->n_envs + i);
    for (int k = 0; k < 6; ++k) {
      uint32_t x0 = or_word(cfg, g, s, OR_TAG_ACTION, 2u * k), x1 = or_word(cfg, g, s, OR_TAG_ACTION, 2u * k + 1u);
      float u1 = (float)((x0 >> 8) + 1u) * 0x1p-24f;
      float u2 = (float)(x1 >> 8) * 0x1p-24f;
      float rr = sqrtf(-2.0f * or_log(u1));
      float sn, cs;
      or_sincos(0x1.921fb6p2f * u2, &sn, &cs);
      eps[(size_t)i * 12 + 2 * k] = rr * cs;
      eps[(size_t)i * 12 + 2 * k + 1] = rr * sn;
    }
  }
}

/* ---------------- DESIGN.md §3.10 Feistel shuffle ---------------- */
static uint32_t lowbias32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16;
  return x;
}

void or_feistel_perm(uint32_t B, const uint32_t K[4], uint32_t* perm) {
  uint32_t k = 0;
  while ((1u << k) < B) ++k;
  if (k & 1u) ++k;
  if (k < 2) k = 2;
  uint32_t half = k / 2u, mask = (1u << half) - 1u;
  for (uint32_t i = 0; i < B; ++i) {
    uint32_t x = i;
    do {
      uint32_t L = x >> half, Rr = x & mask;
      for (int r = 0; r < 4; ++r) {
        uint32_t nl = Rr;
        uint32_t nr = L ^ (lowbias32(Rr ^ K[r]) & mask);
        L = nl; Rr = nr;
      }
      x = (L << half) | Rr;
    } while (x >= B);
    perm[i] = x;
  }
}

/* exported single-point helpers for pins */
void or_sincos_batch(int n, const float* x, float* s, float* c) { for (int i = 0; i < n; ++i) or_sincos(x[i], &s[i], &c[i]); }
void or_exp_batch(int n, const float* x, float* y) { for (int i = 0; i < n; ++i) y[i] = or_exp(x[i]); }
void or_log_batch(int n, const float* x, float* y) { for (int i = 0; i < n; ++i) y[i] = or_log(x[i]); }
void or_reward_terms(const or_state* st, const float* a, const float* tau, const float* qdd, float airsum, int n_c,
                     float* terms, float* total) {
  float qstar[12];
  for (int j = 0; j < 12; ++j) qstar[j] = QDEF12[j] + 0.5f * a[j];
  *total = reward_one(st, qstar, tau, qdd, airsum, n_c, terms);
}
void or_transition(const or_env_cfg* cfg, const float* hf, or_state* st, const float* a, uint32_t s,
                   float* tau, float* qdd, float* airsum, int* crash, int* n_c, float* fz) {
  float qstar[12];
  uint32_t g = (uint32_t)(cfg->rank * cfg->n_envs);
  transition_one(cfg, hf, st, a, g, s, qstar, tau, qdd, airsum, crash, n_c);
  *fz = g_last_fz;
}

/* ---------------- DESIGN.md §3.12  terrain generation (NEXT-4; reading R27) ----------------
 * The world of n_levels x n_cols tiles of 80 x 80 cells (8 m at 0.1 m): level l
 * along x (rows), column c along y; kind = c mod 5 (0 flat, 1 slope pyramid, 2 rough, 3 obstacles, 4 stairs
 * pyramid); difficulty d = l / (L - 1) (0 when L = 1). Written out cell by cell, in the definition's order.
 * Random words: Philox key = seed, counter (w / 4, tile id l * n_cols + c, 0, tag 8), word w mod 4. */
#define OR_TAG_TERRAIN 8u
static uint32_t terrain_word(uint32_t k0, uint32_t k1, uint32_t tile, uint32_t w) {
  uint32_t ctr[4] = {w / 4u, tile, 0u, OR_TAG_TERRAIN}, out[4];
  or_philox(k0, k1, ctr, out);
  return out[w % 4u];
}

void or_terrain_generate(float* hf, int n_levels, int n_cols, uint32_t seed_lo, uint32_t seed_hi) {
  const int C = n_cols * 80;
  for (int l = 0; l < n_levels; ++l) {
    const float d = n_levels > 1 ? (float)l / (float)(n_levels - 1) : 0.0f;
    /* slope: tan(25 deg * d), evaluated in double and rounded once */
    const float slope = (float)tan(25.0 * (3.14159265358979323846 / 180.0) * (double)d);
    const float rough_half = 0.5f * (0.05f * (1.0f + d)); /* rough: U(-a/2, a/2), a = 0.05 (1 + d) */
    const float hmax = 0.05f + 0.15f * d;                 /* obstacle heights U(-hmax, hmax) */
    const float riser = 0.05f + 0.15f * d;                /* stair riser */
    for (int c = 0; c < n_cols; ++c) {
      const int kind = c % 5;
      const uint32_t tile = (uint32_t)(l * n_cols + c);
      /* obstacles: 8 boxes, words 5b .. 5b+4 = width, length, x0, y0, height */
      int bi0[8], bi1[8], bj0[8], bj1[8];
      float bh[8];
      for (int b = 0; b < 8; ++b) {
        const float w = 0.5f + 1.5f * u01(terrain_word(seed_lo, seed_hi, tile, 5u * b + 0u));
        const float len = 0.5f + 1.5f * u01(terrain_word(seed_lo, seed_hi, tile, 5u * b + 1u));
        const float x0 = 8.0f * u01(terrain_word(seed_lo, seed_hi, tile, 5u * b + 2u));
        const float y0 = 8.0f * u01(terrain_word(seed_lo, seed_hi, tile, 5u * b + 3u));
        bh[b] = usym(hmax, terrain_word(seed_lo, seed_hi, tile, 5u * b + 4u));
        bi0[b] = (int)(x0 * 10.0f);
        bi1[b] = (int)(fminf(8.0f, x0 + w) * 10.0f);
        bj0[b] = (int)(y0 * 10.0f);
        bj1[b] = (int)(fminf(8.0f, y0 + len) * 10.0f);
      }
      for (int i = 0; i < 80; ++i) {
        for (int j = 0; j < 80; ++j) {
          const float xc = (float)(2 * i + 1) * 0.05f, yc = (float)(2 * j + 1) * 0.05f; /* cell centre */
          const float e = fminf(fminf(xc, 8.0f - xc), fminf(yc, 8.0f - yc));           /* to the border */
          const float ep = fminf(e, 3.0f);                                              /* 2 m plateau */
          float h = 0.0f;
          if (kind == 1) {
            h = slope * ep;
          } else if (kind == 2) {
            h = usym(rough_half, terrain_word(seed_lo, seed_hi, tile, (uint32_t)(i * 80 + j)));
          } else if (kind == 3) {
            for (int b = 0; b < 8; ++b)
              if (i >= bi0[b] && i < bi1[b] && j >= bj0[b] && j < bj1[b]) h = bh[b];
            if (e >= 3.0f) h = 0.0f;
          } else if (kind == 4) {
            h = riser * floorf(ep / 0.3f);
          }
          hf[(size_t)(l * 80 + i) * C + (size_t)(c * 80 + j)] = h;
        }
      }
    }
  }
}
