// gemm_probe.cu -- diagnostics for the tcgen05 GEMMs of libleggedrl (not part of the product path).
// Times the forward (K-major) and weight-gradient (MN-major, cluster split-K) kernels on synthetic bf16
// operands with CUDA events, with the probe bits of GemmArgs isolating the TMA load pipeline (skip MMA)
// and the MMA pipeline (skip TMA).
//
//   build: python tools/build_probe.py     run: tools/gemm_probe
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cmath>
#include <algorithm>
#include <vector>
#include <string>

#include "../paper_2109_11978_b200/csrc/kernels.h"

using namespace lg;

#define CK(x)                                                                                    \
  do {                                                                                           \
    cudaError_t e_ = (x);                                                                        \
    if (e_ != cudaSuccess) {                                                                     \
      fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_));         \
      exit(1);                                                                                   \
    }                                                                                            \
  } while (0)

static void fill(__nv_bfloat16* p, size_t n) {
  std::vector<__nv_bfloat16> h(n);
  uint32_t s = 12345u;
  for (size_t i = 0; i < n; ++i) {
    s = s * 1664525u + 1013904223u;
    h[i] = __float2bfloat16(((s >> 9) & 1023) / 1024.0f - 0.5f);
  }
  CK(cudaMemcpy(p, h.data(), n * 2, cudaMemcpyHostToDevice));
}

static char* g_flush = nullptr;
static bool g_do_flush = true;
static void flush(cudaStream_t st) {
  if (g_do_flush) CK(cudaMemsetAsync(g_flush, 1, 512u << 20, st));
}

static bool g_batch = false;  // time `reps` back-to-back launches between one event pair (steady state)

template <class F>
static float time_us(F f, cudaStream_t st, int reps = 20) {
  if (g_batch) {
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    for (int i = 0; i < 3; ++i) f();
    CK(cudaStreamSynchronize(st));
    CK(cudaEventRecord(a, st));
    for (int i = 0; i < reps; ++i) f();
    CK(cudaEventRecord(b, st));
    CK(cudaEventSynchronize(b));
    float ms;
    CK(cudaEventElapsedTime(&ms, a, b));
    return ms / reps * 1000.f;
  }
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  for (int i = 0; i < 3; ++i) f();
  CK(cudaStreamSynchronize(st));
  float tot = 0.f;
  for (int i = 0; i < reps; ++i) {
    flush(st);
    CK(cudaEventRecord(a, st));
    f();
    CK(cudaEventRecord(b, st));
    CK(cudaEventSynchronize(b));
    float ms;
    CK(cudaEventElapsedTime(&ms, a, b));
    tot += ms;
  }
  return tot / reps * 1000.f;
}

// forward: Y[M][N] = X[M][K] W[N][K]^T (+bias, ELU)
static void probe_fwd(int M, int N, int K, int bn, cudaStream_t st) {
  __nv_bfloat16 *X, *W, *Y;
  float* bias;
  CK(cudaMalloc(&X, (size_t)M * K * 2));
  CK(cudaMalloc(&W, (size_t)N * K * 2));
  CK(cudaMalloc(&Y, (size_t)M * N * 2));
  CK(cudaMalloc(&bias, N * 4));
  CK(cudaMemset(bias, 0, N * 4));
  fill(X, (size_t)M * K);
  fill(W, (size_t)N * K);
  GemmArgs g;
  memset(&g, 0, sizeof(g));
  make_tmap_bf16(&g.tmA[0], X, M, K, K, 128);
  make_tmap_bf16(&g.tmB[0], W, N, K, K, bn);
  make_tmap_bf16(&g.tmC[0], Y, M, N, N, 32);
  g.M = M; g.N = N; g.m_tiles = (M + 127) / 128; g.nz = 1;
  g.kb_total = (K + 63) / 64; g.kb_per_split = g.kb_total; g.n_tiles = (N + bn - 1) / bn; g.n_splits = 1;
  g.ldo = N; g.bias[0] = bias;
  const double fl = 2.0 * M * N * K;
  const int probes[6] = {0, 1, 2, 4, 5, 6};  // 5: loads only, 6: MMAs only
  for (int pi = 0; pi < 6; ++pi) {
    const int probe = probes[pi];
    g.probe = probe;
    float us = time_us([&] { CK(launch_gemm(GEMM_FWD, bn, g, st)); }, st);
    const double bytes = ((double)M * K + (double)g.m_tiles * 128.0 * 0 + (double)N * K * g.m_tiles) * 2.0;
    printf("fwd M=%d N=%d K=%d bn=%d probe=%d  %8.2f us  %7.1f TFLOP/s  operand-load %7.1f GB/s\n", M, N, K, bn,
           probe, us, fl / us * 1e-6, bytes / us * 1e-3);
  }
  CK(cudaFree(X)); CK(cudaFree(W)); CK(cudaFree(Y)); CK(cudaFree(bias));
}

// input gradient: dZp[M][N] = (dZ[M][K] W[K][N]) * ELU'(H[M][N])  (A K-major, B = W[out=K][in=N] MN-major)
static void probe_dx(int M, int N, int K, int bn, cudaStream_t st, bool once = false) {
  __nv_bfloat16 *dZ, *W, *H, *Y;
  CK(cudaMalloc(&dZ, (size_t)M * K * 2)); CK(cudaMalloc(&W, (size_t)K * N * 2));
  CK(cudaMalloc(&H, (size_t)M * N * 2)); CK(cudaMalloc(&Y, (size_t)M * N * 2));
  fill(dZ, (size_t)M * K); fill(W, (size_t)K * N); fill(H, (size_t)M * N);
  GemmArgs g;
  memset(&g, 0, sizeof(g));
  make_tmap_bf16(&g.tmA[0], dZ, M, K, K, 128);
  make_tmap_bf16(&g.tmB[0], W, K, N, N, 64);
  make_tmap_bf16(&g.tmC[0], Y, M, N, N, 32);
  g.M = M; g.N = N; g.m_tiles = (M + 127) / 128; g.nz = 1;
  g.kb_total = (K + 63) / 64; g.kb_per_split = g.kb_total; g.n_tiles = (N + bn - 1) / bn; g.n_splits = 1;
  g.ldo = N; g.aux[0] = H; g.ld_aux = N;
  const double fl = 2.0 * M * N * K;
  const int probes[4] = {0, 1, 2, 4};
  for (int pi = 0; pi < (once ? 1 : 4); ++pi) {
    const int probe = probes[pi];
    g.probe = probe;
    float us = time_us([&] { CK(launch_gemm(GEMM_DX, bn, g, st)); }, st);
    printf("dx M=%d N=%d K=%d bn=%d probe=%d  %8.2f us  %7.1f TFLOP/s\n", M, N, K, bn, probe, us, fl / us * 1e-6);
  }
  CK(cudaFree(dZ)); CK(cudaFree(W)); CK(cudaFree(H)); CK(cudaFree(Y));
}

// update layer 3 + fused PPO loss head (EPI 4): time it and print per-phase timestamps (tile 0 of the CTA with
// the latest finish) -- phases: 0 tile start, 1 A3 free, 2 accumulator ready, 3 head outputs read, 4 loss terms,
// 5 small sums done, 6 gradient MMAs complete, 7 dZ3 staged, 8 gradient MMAs issued, 9 after the loss barrier
static void probe_loss(int M, float frac, cudaStream_t st) {
  const int H1 = 256, H2 = 128;
  __nv_bfloat16 *H2a, *W3, *dZ3;
  float *b3, *W4a, *b4a, *W4c, *b4c, *ls, *lso, *act, *muo, *lpo, *Vo, *adv, *ret, *part, *payload;
  double* spart;
  unsigned long long* dbg;
  CK(cudaMalloc(&H2a, (size_t)M * 2 * H1 * 2)); fill(H2a, (size_t)M * 2 * H1);
  CK(cudaMalloc(&W3, (size_t)2 * H2 * H1 * 2)); fill(W3, (size_t)2 * H2 * H1);
  CK(cudaMalloc(&dZ3, (size_t)M * 2 * H2 * 2));
  auto fz = [&](float** p, size_t n, float v) {
    CK(cudaMalloc(p, n * 4));
    std::vector<float> h(n);
    uint32_t s = 777u + (uint32_t)n;
    for (size_t i = 0; i < n; ++i) { s = s * 1664525u + 1013904223u; h[i] = v * (((s >> 9) & 1023) / 512.0f - 1.0f); }
    CK(cudaMemcpy(*p, h.data(), n * 4, cudaMemcpyHostToDevice));
  };
  fz(&b3, 2 * H2, 0.1f); fz(&W4a, 12 * H2, 0.1f); fz(&b4a, 12, 0.1f); fz(&W4c, H2, 0.1f); fz(&b4c, 1, 0.1f);
  fz(&ls, 12, 0.1f); fz(&lso, 12, 0.1f); fz(&act, (size_t)M * 12, 1.0f); fz(&muo, (size_t)M * 12, 1.0f);
  fz(&lpo, M, 5.0f); fz(&Vo, M, 1.0f); fz(&adv, M, 1.0f); fz(&ret, M, 1.0f);
  CK(cudaMalloc(&part, (size_t)148 * (13 * H2 + 28) * 4));
  CK(cudaMalloc(&spart, (size_t)148 * 8 * 8));
  CK(cudaMalloc(&payload, 64));
  CK(cudaMalloc(&dbg, (size_t)148 * 128 * 8));
  CK(cudaMemset(dbg, 0, (size_t)148 * 128 * 8));
  GemmArgs g;
  memset(&g, 0, sizeof(g));
  for (int z = 0; z < 2; ++z) {
    make_tmap_bf16(&g.tmA[z], H2a + z * H1, M, H1, 2 * H1, 128);
    make_tmap_bf16(&g.tmB[z], W3 + (size_t)z * H2 * H1, H2, H1, H1, 128);
    make_tmap_bf16(&g.tmC[z], dZ3 + z * H2, M, H2, 2 * H2, 32);
    g.bias[z] = b3 + z * H2;
  }
  g.M = M; g.N = H2; g.kb_total = H1 / 64; g.kb_per_split = g.kb_total; g.n_tiles = 1; g.n_splits = 1;
  LossEpi& le = g.le;
  le.W4a = W4a; le.b4a = b4a; le.W4c = W4c; le.b4c = b4c; le.logstd = ls; le.logstd_old = lso;
  le.act = act; le.mu_old = muo; le.logp_old = lpo; le.V_old = Vo; le.adv = adv; le.ret = ret;
  le.clip = 0.2f; le.vclip = 0.2f; le.vf_coef = 1.0f; le.invM = 1.0f / M; le.H2 = H2; le.payload = payload;
  le.part = part; le.spart = spart; le.HP = (13 * H2 + 25 + 3) / 4 * 4;
  if (frac > 0) setenv("LG_LOSS_ACTOR_FRAC", std::to_string(frac).c_str(), 1);
  int grid = 0;
  float us = time_us([&] { CK(launch_gemm_loss(g, &grid, st)); }, st);
  printf("loss M=%d grid=%d  %8.2f us\n", M, grid, us);
  le.dbg = dbg;
  CK(launch_gemm_loss(g, &grid, st));
  CK(cudaStreamSynchronize(st));
  std::vector<unsigned long long> h((size_t)148 * 128);
  CK(cudaMemcpy(h.data(), dbg, h.size() * 8, cudaMemcpyDeviceToHost));
  unsigned long long t0 = ~0ull, tend = 0;
  int slow = 0;
  for (int b = 0; b < grid; ++b) {
    if (h[b * 128 + 8] && h[b * 128 + 8] < t0) t0 = h[b * 128 + 8];
    for (int k = 0; k < 128; ++k)
      if (h[b * 128 + k] > tend) { tend = h[b * 128 + k]; slow = b; }
  }
  printf("first stamp -> last stamp %.2f us; slowest CTA %d\n", (tend - t0) * 1e-3, slow);
  for (int b : {0, grid / 2, slow, grid - 1}) {
    printf("CTA %3d: entry %.2f exit %.2f", b, (h[b * 128 + 8] - t0) * 1e-3, (h[b * 128 + 9] - t0) * 1e-3);
    for (int t = 0; t < 8; ++t) {
      if (!h[(b * 8 + t) * 16]) break;
      printf(" |t%d", t);
      for (int k = 0; k < 8; ++k) printf(" %.2f", (h[(b * 8 + t) * 16 + k] - t0) * 1e-3);
    }
    printf("\n");
  }
}

// weight gradient: dW[N_out][N_in] = dZ[K][N_out]^T X[K][N_in], split-K over G clusters of S per tile
static std::vector<float> probe_dw(int Nout, int Nin, int K, int bn, int S, int G, cudaStream_t st, bool quiet = false) {
  __nv_bfloat16 *dZ, *X;
  float *grad, *part;
  int* cnt;
  const size_t gsz = (size_t)Nout * Nin + Nout + 64;
  CK(cudaMalloc(&dZ, (size_t)K * Nout * 2));
  CK(cudaMalloc(&X, (size_t)K * Nin * 2));
  CK(cudaMalloc(&grad, gsz * 4));
  fill(dZ, (size_t)K * Nout);
  fill(X, (size_t)K * Nin);
  GemmArgs g;
  memset(&g, 0, sizeof(g));
  make_tmap_bf16(&g.tmA[0], dZ, K, Nout, Nout, 64);
  make_tmap_bf16(&g.tmB[0], X, K, Nin, Nin, 64);
  g.M = Nout; g.N = Nin; g.m_tiles = (Nout + 127) / 128; g.nz = 1;
  g.kb_total = (K + 63) / 64; g.n_tiles = (Nin + bn - 1) / bn; g.n_splits = 1;
  const int tiles = g.m_tiles * g.n_tiles;
  S = S * G; G = 1;
  g.kb_per_split = (g.kb_total + S - 1) / S;
  S = (g.kb_total + g.kb_per_split - 1) / g.kb_per_split;
  CK(cudaMalloc(&part, (size_t)tiles * S * 128 * (bn + 20) * 4));
  CK(cudaMalloc(&cnt, 256));
  CK(cudaMemset(cnt, 0, 256));
  DwOut o;
  memset(&o, 0, sizeof(o));
  o.grad = grad; o.w_off[0] = 0; o.b_off[0] = (long long)Nout * Nin; o.cols = Nin; o.row_split = 0;
  o.payload = grad + (size_t)Nout * Nin + Nout;
  o.G = G; o.part = part; o.cnt = cnt;
  const double fl = 2.0 * Nout * Nin * K;
  for (int probe = 0; probe < (quiet ? 1 : 2); ++probe) {
    g.probe = probe;
    float us = time_us([&] { CK(launch_gemm_dw(bn, g, o, S, st)); }, st);
    const double bytes = ((double)K * Nout * g.n_tiles + (double)K * Nin * g.m_tiles) * 2.0;
    printf("dw  Nout=%d Nin=%d K=%d bn=%d S=%d G=%d ctas=%d probe=%d  %8.2f us  %7.1f TFLOP/s  operand-load %7.1f GB/s\n",
           Nout, Nin, K, bn, S, G, tiles * S * G, probe, us, fl / us * 1e-6, bytes / us * 1e-3);
  }
  g.probe = 0;
  CK(cudaMemset(grad, 0, gsz * 4));
  CK(launch_gemm_dw(bn, g, o, S, st));
  CK(cudaStreamSynchronize(st));
  std::vector<float> h(gsz);
  CK(cudaMemcpy(h.data(), grad, gsz * 4, cudaMemcpyDeviceToHost));
  CK(cudaFree(dZ)); CK(cudaFree(X)); CK(cudaFree(grad)); CK(cudaFree(part)); CK(cudaFree(cnt));
  return h;
}

// dW1-like problem from K-major (transposed) operand copies vs the MN-major originals
static void probe_dw_kmajor(int Nout, int Nin, int K, int bn, int S, int G, cudaStream_t st) {
  __nv_bfloat16 *dZ, *X, *dZT, *XT;
  float *g1, *g2, *part;
  int* cnt;
  const size_t gsz = (size_t)Nout * Nin + Nout + 64;
  CK(cudaMalloc(&dZ, (size_t)K * Nout * 2)); CK(cudaMalloc(&X, (size_t)K * Nin * 2));
  CK(cudaMalloc(&dZT, (size_t)K * Nout * 2)); CK(cudaMalloc(&XT, (size_t)K * Nin * 2));
  CK(cudaMalloc(&g1, gsz * 4)); CK(cudaMalloc(&g2, gsz * 4));
  std::vector<__nv_bfloat16> h1((size_t)K * Nout), h2((size_t)K * Nin), t1(h1.size()), t2(h2.size());
  uint32_t sd = 777u;
  for (auto& v : h1) { sd = sd * 1664525u + 1013904223u; v = __float2bfloat16(((sd >> 9) & 1023) / 1024.0f - 0.5f); }
  for (auto& v : h2) { sd = sd * 1664525u + 1013904223u; v = __float2bfloat16(((sd >> 9) & 1023) / 1024.0f - 0.5f); }
  for (int k = 0; k < K; ++k) {
    for (int o = 0; o < Nout; ++o) t1[(size_t)o * K + k] = h1[(size_t)k * Nout + o];
    for (int i = 0; i < Nin; ++i) t2[(size_t)i * K + k] = h2[(size_t)k * Nin + i];
  }
  CK(cudaMemcpy(dZ, h1.data(), h1.size() * 2, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(X, h2.data(), h2.size() * 2, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dZT, t1.data(), t1.size() * 2, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(XT, t2.data(), t2.size() * 2, cudaMemcpyHostToDevice));
  GemmArgs g, gt;
  memset(&g, 0, sizeof(g));
  make_tmap_bf16(&g.tmA[0], dZ, K, Nout, Nout, 64);
  make_tmap_bf16(&g.tmB[0], X, K, Nin, Nin, 64);
  g.M = Nout; g.N = Nin; g.m_tiles = (Nout + 127) / 128; g.nz = 1;
  g.kb_total = (K + 63) / 64; g.n_tiles = (Nin + bn - 1) / bn; g.n_splits = 1;
  const int tiles = g.m_tiles * g.n_tiles;
  S = S * G; G = 1;
  g.kb_per_split = (g.kb_total + S - 1) / S;
  S = (g.kb_total + g.kb_per_split - 1) / g.kb_per_split;
  gt = g;
  make_tmap_bf16(&gt.tmA[0], dZT, Nout, K, K, 128);
  make_tmap_bf16(&gt.tmB[0], XT, Nin, K, K, bn);
  CK(cudaMalloc(&part, (size_t)tiles * S * 128 * (bn + 20) * 4));
  CK(cudaMalloc(&cnt, 256));
  CK(cudaMemset(cnt, 0, 256));
  DwOut o;
  memset(&o, 0, sizeof(o));
  o.grad = g1; o.b_off[0] = (long long)Nout * Nin; o.cols = Nin; o.payload = g1 + (size_t)Nout * Nin + Nout;
  o.G = G; o.part = part; o.cnt = cnt;
  DwOut o2 = o;
  o2.grad = g2; o2.payload = g2 + (size_t)Nout * Nin + Nout;
  const double fl = 2.0 * Nout * Nin * K;
  for (int probe = 0; probe < 2; ++probe) {
    g.probe = gt.probe = probe;
    float u1 = time_us([&] { CK(launch_gemm_dw(bn, g, o, S, st)); }, st);
    float u2 = time_us([&] { CK(launch_gemm_dw_kmajor(bn, gt, o2, S, st)); }, st);
    printf("dw Nout=%d Nin=%d K=%d bn=%d S=%d G=%d probe=%d  MN-major %8.2f us (%6.1f TF)  K-major %8.2f us (%6.1f TF)\n",
           Nout, Nin, K, bn, S, G, probe, u1, fl / u1 * 1e-6, u2, fl / u2 * 1e-6);
  }
  g.probe = gt.probe = 0;
  CK(cudaMemset(g1, 0, gsz * 4)); CK(cudaMemset(g2, 0, gsz * 4));
  CK(launch_gemm_dw(bn, g, o, S, st));
  CK(launch_gemm_dw_kmajor(bn, gt, o2, S, st));
  CK(cudaStreamSynchronize(st));
  std::vector<float> a(gsz), b(gsz);
  CK(cudaMemcpy(a.data(), g1, gsz * 4, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(b.data(), g2, gsz * 4, cudaMemcpyDeviceToHost));
  double num = 0, den = 0;
  for (size_t i = 0; i + 64 < gsz; ++i) { num += (a[i] - b[i]) * (double)(a[i] - b[i]); den += (double)a[i] * a[i]; }
  printf("   K-major vs MN-major: rel l2 %.3e\n", std::sqrt(num / den));
  CK(cudaFree(dZ)); CK(cudaFree(X)); CK(cudaFree(dZT)); CK(cudaFree(XT)); CK(cudaFree(g1)); CK(cudaFree(g2));
  CK(cudaFree(part)); CK(cudaFree(cnt));
}

// phase timestamps of every CTA of one dW launch (globaltimer ns, relative to the earliest CTA start)
static void probe_dw_phases(int Nout, int Nin, int K, int bn, int S, int G, cudaStream_t st, int dmode = 0,
                            bool pair = false) {
  __nv_bfloat16 *dZ, *X;
  float *grad, *part;
  int* cnt;
  unsigned long long* dbg;
  const size_t gsz = (size_t)Nout * Nin + Nout + 64;
  CK(cudaMalloc(&dZ, (size_t)K * Nout * 2)); CK(cudaMalloc(&X, (size_t)K * Nin * 2)); CK(cudaMalloc(&grad, gsz * 4));
  fill(dZ, (size_t)K * Nout); fill(X, (size_t)K * Nin);
  GemmArgs g;
  memset(&g, 0, sizeof(g));
  make_tmap_bf16(&g.tmA[0], dZ, K, Nout, Nout, 64);
  make_tmap_bf16(&g.tmB[0], X, K, Nin, Nin, 64);
  g.M = Nout; g.N = Nin; g.m_tiles = (Nout + 127) / 128; g.nz = 1;
  g.kb_total = (K + 63) / 64; g.n_tiles = (Nin + bn - 1) / bn; g.n_splits = 1;
  const int tiles = g.m_tiles * g.n_tiles;
  S = S * G; G = 1;
  g.kb_per_split = (g.kb_total + S - 1) / S;
  S = (g.kb_total + g.kb_per_split - 1) / g.kb_per_split;
  const int nct = tiles * S * G;
  CK(cudaMalloc(&part, (size_t)tiles * S * 128 * (bn + 20) * 4));
  CK(cudaMalloc(&cnt, 256)); CK(cudaMemset(cnt, 0, 256));
  CK(cudaMalloc(&dbg, (size_t)nct * 8 * 8));
  DwOut o;
  memset(&o, 0, sizeof(o));
  o.grad = grad; o.b_off[0] = (long long)Nout * Nin; o.cols = Nin; o.payload = grad + (size_t)Nout * Nin + Nout;
  o.G = G; o.part = part; o.cnt = cnt; o.dbg = dbg; o.dbg_mode = dmode;
  for (int r = 0; r < 4; ++r) {
    if (pair) {
      GemmArgs gp = g;
      gp.kb_per_split = (g.kb_total + S - 1) / S;
      CK(launch_gemm_dw_pair(bn, gp, o, S, st));
    } else {
      CK(launch_gemm_dw(bn, g, o, S, st));
    }
  }
  CK(cudaStreamSynchronize(st));
  std::vector<unsigned long long> h((size_t)nct * 8);
  CK(cudaMemcpy(h.data(), dbg, h.size() * 8, cudaMemcpyDeviceToHost));
  unsigned long long t0 = ~0ull, tend = 0;
  for (int c = 0; c < nct; ++c) { t0 = std::min(t0, h[(size_t)c * 8]); tend = std::max(tend, h[(size_t)c * 8 + 7]); }
  double avg[8] = {0}, mx[8] = {0};
  for (int c = 0; c < nct; ++c)
    for (int k = 0; k < 8; ++k) {
      const double v = (h[(size_t)c * 8 + k] - t0) * 1e-3;
      avg[k] += v / nct;
      mx[k] = std::max(mx[k], v);
    }
  printf("dw phases%s Nout=%d Nin=%d K=%d S=%d G=%d ctas=%d kb/cta=%d dbg_mode=%d (us from first CTA start; avg | max):\n",
         pair ? " (CTA pair)" : "", Nout, Nin, K, S, G, nct, g.kb_per_split, dmode);
  const char* nm[8] = {"start", "tmem alloc", "mma done", "partial->smem", "partial->L2", "grid barrier", "reduced", "end"};
  for (int k = 0; k < 8; ++k) printf("   %-14s %8.2f | %8.2f\n", nm[k], avg[k], mx[k]);
  CK(cudaFree(dZ)); CK(cudaFree(X)); CK(cudaFree(grad)); CK(cudaFree(part)); CK(cudaFree(cnt)); CK(cudaFree(dbg));
}

// CTA-pair dW (launch_gemm_dw_pair, S splits per 256-row pair tile) vs the single-CTA kernel (2S splits)
static void probe_dw_pair(int Nout, int Nin, int K, int bn, int S, cudaStream_t st) {
  __nv_bfloat16 *dZ, *X;
  float *g1, *g2, *part;
  int* cnt;
  const size_t gsz = (size_t)Nout * Nin + Nout + 64;
  CK(cudaMalloc(&dZ, (size_t)K * Nout * 2)); CK(cudaMalloc(&X, (size_t)K * Nin * 2));
  CK(cudaMalloc(&g1, gsz * 4)); CK(cudaMalloc(&g2, gsz * 4));
  fill(dZ, (size_t)K * Nout); fill(X, (size_t)K * Nin);
  GemmArgs g;
  memset(&g, 0, sizeof(g));
  make_tmap_bf16(&g.tmA[0], dZ, K, Nout, Nout, 64);
  make_tmap_bf16(&g.tmB[0], X, K, Nin, Nin, 64);
  g.M = Nout; g.N = Nin; g.m_tiles = (Nout + 127) / 128; g.nz = 1;
  g.kb_total = (K + 63) / 64; g.n_tiles = (Nin + bn - 1) / bn; g.n_splits = 1;
  const int tiles = g.m_tiles * g.n_tiles;
  GemmArgs g1a = g, g2a = g;
  const int S1 = std::min(S, g.kb_total);  // single-CTA: 128-row tiles, same CTA count
  g1a.kb_per_split = (g.kb_total + S1 - 1) / S1;
  const int S1e = (g.kb_total + g1a.kb_per_split - 1) / g1a.kb_per_split;
  g2a.kb_per_split = (g.kb_total + S - 1) / S;
  const int S2e = (g.kb_total + g2a.kb_per_split - 1) / g2a.kb_per_split;
  const int Smax = std::max(S1e, S2e);
  CK(cudaMalloc(&part, (size_t)tiles * Smax * 128 * (bn + 20) * 4));
  CK(cudaMalloc(&cnt, 256)); CK(cudaMemset(cnt, 0, 256));
  DwOut o;
  memset(&o, 0, sizeof(o));
  o.grad = g1; o.b_off[0] = (long long)Nout * Nin; o.cols = Nin; o.payload = g1 + (size_t)Nout * Nin + Nout;
  o.G = 1; o.part = part; o.cnt = cnt;
  DwOut o2 = o;
  o2.grad = g2; o2.payload = g2 + (size_t)Nout * Nin + Nout;
  const double fl = 2.0 * Nout * Nin * K;
  printf("  [pair probe Nout=%d Nin=%d K=%d S=%d] single-CTA timing...\n", Nout, Nin, K, S);
  float u1 = time_us([&] { CK(launch_gemm_dw(bn, g1a, o, S1e, st)); }, st);
  printf("  one pair launch...\n");
  CK(launch_gemm_dw_pair(bn, g2a, o2, S2e, st));
  CK(cudaStreamSynchronize(st));
  printf("  pair timing...\n");
  float u2 = time_us([&] { CK(launch_gemm_dw_pair(bn, g2a, o2, S2e, st)); }, st);
  printf("dw Nout=%d Nin=%d K=%d bn=%d  single-CTA (%d splits, %d CTAs) %8.2f us (%6.1f TF)  CTA-pair (%d splits, %d CTAs) %8.2f us (%6.1f TF)\n",
         Nout, Nin, K, bn, S1e, S1e * tiles, u1, fl / u1 * 1e-6, S2e, 2 * S2e * tiles / 2, u2, fl / u2 * 1e-6);
  CK(cudaMemset(g1, 0, gsz * 4)); CK(cudaMemset(g2, 0, gsz * 4));
  CK(launch_gemm_dw(bn, g1a, o, S1e, st));
  CK(launch_gemm_dw_pair(bn, g2a, o2, S2e, st));
  CK(cudaStreamSynchronize(st));
  std::vector<float> a(gsz), b(gsz);
  CK(cudaMemcpy(a.data(), g1, gsz * 4, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(b.data(), g2, gsz * 4, cudaMemcpyDeviceToHost));
  double num = 0, den = 0, mx = 0;
  for (size_t i = 0; i + 64 < gsz; ++i) {
    num += (a[i] - b[i]) * (double)(a[i] - b[i]); den += (double)a[i] * a[i];
    mx = std::max(mx, (double)std::fabs(a[i] - b[i]));
  }
  printf("   pair vs single: rel l2 %.3e  max abs %.3e  (bias[0] %g vs %g)\n", std::sqrt(num / den), mx,
         a[(size_t)Nout * Nin], b[(size_t)Nout * Nin]);
  CK(cudaFree(dZ)); CK(cudaFree(X)); CK(cudaFree(g1)); CK(cudaFree(g2)); CK(cudaFree(part)); CK(cudaFree(cnt));
}

// fused rollout policy on synthetic data: timing and per-CTA phase stamps
static void probe_fused(int N, cudaStream_t st) {
  const int Dp = 240, H0 = 512, H1 = 256, H2 = 128;
  __nv_bfloat16 *X, *W1, *W2, *W3;
  float *b1, *b2, *b3, *W4a, *b4a, *W4c, *b4c, *ls, *out;
  unsigned long long* dbg;
  void* sc;
  CK(cudaMalloc(&X, (size_t)N * Dp * 2)); CK(cudaMalloc(&W1, (size_t)2 * H0 * Dp * 2));
  CK(cudaMalloc(&W2, (size_t)2 * H1 * H0 * 2)); CK(cudaMalloc(&W3, (size_t)2 * H2 * H1 * 2));
  fill(X, (size_t)N * Dp); fill(W1, (size_t)2 * H0 * Dp); fill(W2, (size_t)2 * H1 * H0); fill(W3, (size_t)2 * H2 * H1);
  CK(cudaMalloc(&b1, 4096 * 4)); CK(cudaMemset(b1, 0, 4096 * 4));
  b2 = b1 + 1024; b3 = b2 + 512; W4a = b3 + 256; b4a = W4a + 12 * 128; W4c = b4a + 16; b4c = W4c + 128; ls = b4c + 16;
  CK(cudaMalloc(&out, (size_t)N * 40 * 4));
  CK(cudaMalloc(&sc, 4096)); CK(cudaMemset(sc, 0, 4096));
  const int nct = ((N + 127) / 128) * 2;
  CK(cudaMalloc(&dbg, (size_t)nct * 16 * 8)); CK(cudaMemset(dbg, 0, (size_t)nct * 16 * 8));
  FusedPolicyArgs a;
  memset(&a, 0, sizeof(a));
  make_tmap_bf16(&a.tmX, X, N, Dp, Dp, 128);
  make_tmap_bf16(&a.tmW1, W1, 2 * H0, Dp, Dp, 256);
  for (int z = 0; z < 2; ++z) {
    make_tmap_bf16(&a.tmW2[z], W2 + (size_t)z * H1 * H0, H1, H0, H0, 256);
    make_tmap_bf16(&a.tmW3[z], W3 + (size_t)z * H2 * H1, H2, H1, H1, 128);
  }
  a.b1 = b1; a.b2 = b2; a.b3 = b3; a.W4a = W4a; a.b4a = b4a; a.W4c = W4c; a.b4c = b4c; a.logstd = ls;
  a.N = N; a.kb1 = 4; a.scalars = reinterpret_cast<const DevScalars*>(sc);
  a.act = out; a.mu = out + (size_t)N * 12; a.logp = out + (size_t)N * 24; a.value = out + (size_t)N * 25;
  float us = time_us([&] { CK(launch_policy_fused(a, st)); }, st);
  printf("fused policy N=%d: %.2f us per launch\n", N, us);
  a.dbg = dbg;
  for (int r = 0; r < 3; ++r) CK(launch_policy_fused(a, st));
  CK(cudaStreamSynchronize(st));
  std::vector<unsigned long long> h((size_t)nct * 16);
  CK(cudaMemcpy(h.data(), dbg, h.size() * 8, cudaMemcpyDeviceToHost));
  unsigned long long t0 = ~0ull;
  for (int c = 0; c < nct; ++c) t0 = std::min(t0, h[(size_t)c * 16]);
  const char* nm[9] = {"start", "prologue", "L1 mma done", "H1 written", "L2 mma done", "H2 written", "L3 mma done",
                       "head sums", "end"};
  for (int k = 0; k < 9; ++k) {
    double avg = 0, mx = 0;
    for (int c = 0; c < nct; ++c) {
      const double v = (h[(size_t)c * 16 + k] - t0) * 1e-3;
      avg += v / nct;
      mx = std::max(mx, v);
    }
    printf("   %-14s %8.2f | %8.2f\n", nm[k], avg, mx);
  }
}

// forward (kind 0) / input-gradient (kind 1) GEMM: CTA pair vs single CTA, timing and element-wise equality
static void probe_pair_gemm(int kind, int M, int N, int K, int bn, cudaStream_t st) {
  __nv_bfloat16 *A, *W, *H, *Y1, *Y2;
  float* bias;
  CK(cudaMalloc(&A, (size_t)M * K * 2)); CK(cudaMalloc(&W, (size_t)K * N * 2)); CK(cudaMalloc(&H, (size_t)M * N * 2));
  CK(cudaMalloc(&Y1, (size_t)M * N * 2)); CK(cudaMalloc(&Y2, (size_t)M * N * 2)); CK(cudaMalloc(&bias, N * 4));
  fill(A, (size_t)M * K); fill(W, (size_t)K * N); fill(H, (size_t)M * N);
  CK(cudaMemset(bias, 0, N * 4));
  GemmArgs g;
  memset(&g, 0, sizeof(g));
  make_tmap_bf16(&g.tmA[0], A, M, K, K, 128);
  if (kind == 0) {  // W [N][K] K-major
    make_tmap_bf16(&g.tmB[0], W, N, K, K, bn);
    make_tmap_bf16(&g.tmBp[0], W, N, K, K, bn / 2);
    g.bias[0] = bias;
  } else {          // W [K][N] read MN-major
    make_tmap_bf16(&g.tmB[0], W, K, N, N, 64);
    g.aux[0] = H; g.ld_aux = N;
  }
  g.M = M; g.N = N; g.m_tiles = (M + 127) / 128; g.nz = 1;
  g.kb_total = (K + 63) / 64; g.kb_per_split = g.kb_total; g.n_tiles = (N + bn - 1) / bn; g.n_splits = 1; g.ldo = N;
  GemmArgs g1 = g, g2 = g;
  make_tmap_bf16(&g1.tmC[0], Y1, M, N, N, 32);
  make_tmap_bf16(&g2.tmC[0], Y2, M, N, N, 32);
  g2.pair = 1;
  const GemmKind gk = kind == 0 ? GEMM_FWD : GEMM_DX;
  const double fl = 2.0 * M * N * K;
  float u1 = time_us([&] { CK(launch_gemm(gk, bn, g1, st)); }, st);
  float u2 = time_us([&] { CK(launch_gemm(gk, bn, g2, st)); }, st);
  CK(cudaStreamSynchronize(st));
  std::vector<uint16_t> y1((size_t)M * N), y2((size_t)M * N);
  CK(cudaMemcpy(y1.data(), Y1, y1.size() * 2, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(y2.data(), Y2, y2.size() * 2, cudaMemcpyDeviceToHost));
  size_t diff = 0;
  for (size_t i = 0; i < y1.size(); ++i) diff += y1[i] != y2[i];
  printf("%s M=%d N=%d K=%d bn=%d  single %8.2f us (%6.1f TF)  pair %8.2f us (%6.1f TF)  differing outputs %zu of %zu\n",
         kind == 0 ? "fwd" : "dx ", M, N, K, bn, u1, fl / u1 * 1e-6, u2, fl / u2 * 1e-6, diff, y1.size());
  CK(cudaFree(A)); CK(cudaFree(W)); CK(cudaFree(H)); CK(cudaFree(Y1)); CK(cudaFree(Y2)); CK(cudaFree(bias));
}

// forward (kind 0) / input-gradient (kind 1) GEMM: weight-stationary vs the tile-order schedule (timing and
// element-wise equality; nz = 2 column groups like the per-net layers)
static void probe_ws_gemm(int kind, int M, int N, int K, int bn, int nz, cudaStream_t st) {
  __nv_bfloat16 *A, *W, *H, *Y1, *Y2;
  float* bias;
  CK(cudaMalloc(&A, (size_t)M * K * 2 * nz)); CK(cudaMalloc(&W, (size_t)K * N * 2 * nz));
  CK(cudaMalloc(&H, (size_t)M * N * 2 * nz));
  CK(cudaMalloc(&Y1, (size_t)M * N * 2 * nz)); CK(cudaMalloc(&Y2, (size_t)M * N * 2 * nz)); CK(cudaMalloc(&bias, N * 4 * nz));
  fill(A, (size_t)M * K * nz); fill(W, (size_t)K * N * nz); fill(H, (size_t)M * N * nz);
  CK(cudaMemset(bias, 0, N * 4 * nz));
  GemmArgs g;
  memset(&g, 0, sizeof(g));
  for (int z = 0; z < nz; ++z) {
    make_tmap_bf16(&g.tmA[z], A + (size_t)z * K, M, K, (size_t)K * nz, 128);
    if (kind == 0) {
      make_tmap_bf16(&g.tmB[z], W + (size_t)z * N * K, N, K, K, bn);
      g.bias[z] = bias + z * N;
    } else {
      make_tmap_bf16(&g.tmB[z], W + (size_t)z * K * N, K, N, N, 64);
      g.aux[z] = H + (size_t)z * N; g.ld_aux = N * nz;
    }
  }
  g.M = M; g.N = N; g.m_tiles = (M + 127) / 128; g.nz = nz;
  g.kb_total = (K + 63) / 64; g.kb_per_split = g.kb_total; g.n_tiles = (N + bn - 1) / bn; g.n_splits = 1; g.ldo = N * nz;
  GemmArgs g1 = g, g2 = g;
  for (int z = 0; z < nz; ++z) {
    make_tmap_bf16(&g1.tmC[z], Y1 + (size_t)z * N, M, N, (size_t)N * nz, 32);
    make_tmap_bf16(&g2.tmC[z], Y2 + (size_t)z * N, M, N, (size_t)N * nz, 32);
  }
  g2.ws = 1;
  const GemmKind gk = kind == 0 ? GEMM_FWD : GEMM_DX;
  const double fl = 2.0 * M * N * K * nz;
  float u1 = time_us([&] { CK(launch_gemm(gk, bn, g1, st)); }, st);
  float u2 = time_us([&] { CK(launch_gemm(gk, bn, g2, st)); }, st);
  CK(cudaStreamSynchronize(st));
  std::vector<uint16_t> y1((size_t)M * N * nz), y2((size_t)M * N * nz);
  CK(cudaMemcpy(y1.data(), Y1, y1.size() * 2, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(y2.data(), Y2, y2.size() * 2, cudaMemcpyDeviceToHost));
  size_t diff = 0;
  for (size_t i = 0; i < y1.size(); ++i) diff += y1[i] != y2[i];
  printf("%s M=%d N=%d K=%d nz=%d bn=%d  tile-order %8.2f us (%6.1f TF)  weight-stationary %8.2f us (%6.1f TF)  differing %zu of %zu\n",
         kind == 0 ? "fwd" : "dx ", M, N, K, nz, bn, u1, fl / u1 * 1e-6, u2, fl / u2 * 1e-6, diff, y1.size());
  CK(cudaFree(A)); CK(cudaFree(W)); CK(cudaFree(H)); CK(cudaFree(Y1)); CK(cudaFree(Y2)); CK(cudaFree(bias));
}

static void check_dw(int Nout, int Nin, int K, int bn, int S, int G, cudaStream_t st) {
  std::vector<float> a = probe_dw(Nout, Nin, K, bn, 1, 1, st, true);  // unsplit K
  std::vector<float> b = probe_dw(Nout, Nin, K, bn, S, G, st, true);
  double num = 0, den = 0;
  for (size_t i = 0; i + 64 < a.size(); ++i) { num += (a[i] - b[i]) * (double)(a[i] - b[i]); den += (double)a[i] * a[i]; }
  printf("check dw Nout=%d Nin=%d S=%d vs S=1: rel l2 %.3e (payload %g)\n", Nout, Nin, S, std::sqrt(num / den),
         b[(size_t)Nout * Nin + Nout + 4]);
}

__global__ void k_empty(int* p) {
  extern __shared__ int sm[];
  if (p && threadIdx.x == 0) p[blockIdx.x] = sm[0];
}

int main(int argc, char** argv) {
  setvbuf(stdout, nullptr, _IONBF, 0);
  cudaStream_t st;
  CK(cudaStreamCreate(&st));
  CK(cudaMalloc(&g_flush, 512u << 20));
  const char* which = argc > 1 ? argv[1] : "all";
  if (argc > 2 && !strcmp(argv[2], "noflush")) g_do_flush = false;
  if (!strcmp(which, "one") || !strcmp(which, "onefwd") || !strcmp(which, "onedx")) g_do_flush = false;
  if (argc > 2 && !strcmp(argv[2], "batch")) { g_do_flush = false; g_batch = true; }
  printf("L2 flush between reps: %s\n", g_do_flush ? "yes" : "no");
  {
    CK(cudaFuncSetAttribute(k_empty, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    float us0 = time_us([&] { k_empty<<<1, 32, 0, st>>>(nullptr); }, st);
    float us1 = time_us([&] { k_empty<<<148, 384, 200 * 1024, st>>>(nullptr); }, st);
    printf("empty kernel: 1x32 %.2f us, 148x384 with 200 KB smem %.2f us\n", us0, us1);
  }
  if (!strcmp(which, "onefwd") && argc >= 6) {  // one forward config: onefwd M N K bn (for ncu)
    g_do_flush = false;
    probe_fwd(atoi(argv[2]), atoi(argv[3]), atoi(argv[4]), atoi(argv[5]), st);
    return 0;
  }
  if (!strcmp(which, "one") && argc >= 9) {  // one dW config: one Nout Nin K bn S G (for ncu)
    g_do_flush = false;
    probe_dw(atoi(argv[2]), atoi(argv[3]), atoi(argv[4]), atoi(argv[5]), atoi(argv[6]), atoi(argv[7]), st, true);
    return 0;
  }
  if (!strcmp(which, "epi")) {
    probe_fwd(24576, 1024, 256, 256, st);
    probe_fwd(24576, 256, 512, 256, st);
    probe_fwd(24576, 128, 256, 128, st);
    probe_dx(24576, 512, 256, 256, st);
    probe_dx(24576, 256, 128, 128, st);
    return 0;
  }
  if (!strcmp(which, "dx")) {
    probe_dx(24576, 512, 256, 256, st);   // dX2: dZ1 = dZ2 W2 (per net), K = H1 = 256
    probe_dx(24576, 512, 256, 128, st);
    probe_dx(24576, 256, 128, 256, st);   // dX3: dZ2 = dZ3 W3 (per net), K = H2 = 128
    probe_dx(24576, 256, 128, 128, st);
    return 0;
  }
  if (!strcmp(which, "onedx") && argc >= 6) {
    g_do_flush = false;
    probe_dx(atoi(argv[2]), atoi(argv[3]), atoi(argv[4]), atoi(argv[5]), st, true);
    return 0;
  }
  if (!strcmp(which, "loss")) {  // loss M [actor_frac]
    probe_loss(atoi(argv[2]), argc > 3 ? (float)atof(argv[3]) : 0.0f, st);
    return 0;
  }
  if (!strcmp(which, "roll")) {  // rollout-size forward GEMMs (M = 4096 envs) at different tile widths
    const int cfg[][4] = {{4096, 1024, 256, 256}, {4096, 1024, 256, 128}, {4096, 512, 256, 256}, {4096, 512, 256, 128},
                          {4096, 256, 512, 256}, {4096, 256, 512, 128}, {4096, 256, 512, 64},
                          {4096, 128, 256, 128}, {4096, 128, 256, 64}, {24576, 1024, 256, 128}, {24576, 256, 512, 128},
                          {24576, 128, 256, 64}};
    for (auto& c : cfg) probe_fwd(c[0], c[1], c[2], c[3], st);
    return 0;
  }
  if (!strcmp(which, "phases")) {
    probe_dw_phases(1024, 240, 24576, 256, 18, 1, st, 0, true);
    probe_dw_phases(512, 512, 24576, 256, 18, 1, st, 0, true);
    probe_dw_phases(1024, 240, 24576, 256, 18, 1, st);   // dW1 (both nets): 8 tiles x 18
    probe_dw_phases(512, 512, 24576, 256, 18, 1, st);    // dW2 both nets as 8 tiles
    probe_dw_phases(256, 256, 24576, 256, 74, 1, st);    // dW3 both nets as 2 tiles
    probe_dw_phases(128, 64, 64, 64, 1, 1, st);
    return 0;
  }
  if (!strcmp(which, "pairgemm")) {
    probe_pair_gemm(0, 24576, 1024, 256, 256, st);  // L1
    probe_pair_gemm(0, 24576, 256, 512, 256, st);   // L2 (one net)
    probe_pair_gemm(0, 24576, 128, 256, 128, st);   // L3 (one net)
    probe_pair_gemm(1, 24576, 512, 256, 256, st);   // dX2 (one net)
    probe_pair_gemm(1, 24576, 256, 128, 128, st);   // dX3 (one net)
    probe_pair_gemm(0, 1000, 256, 256, 256, st);    // odd tile count (8 tiles -> 4 pairs), ragged rows
    probe_pair_gemm(0, 900, 256, 256, 256, st);     // 8 tiles, ragged
    probe_pair_gemm(0, 700, 256, 256, 128, st);     // 6 tiles
    probe_pair_gemm(0, 300, 256, 256, 256, st);     // 3 tiles (odd)
    return 0;
  }
  if (!strcmp(which, "ws")) {
    probe_ws_gemm(0, 24576, 1024, 256, 256, 1, st);  // L1 (both nets), K = Dp padded
    probe_ws_gemm(0, 24576, 256, 512, 256, 2, st);   // L2 per net: tile order only (B 256 KB)
    probe_ws_gemm(0, 24576, 256, 512, 128, 2, st);   // L2 per net, 128-column blocks
    probe_ws_gemm(0, 24576, 128, 256, 128, 2, st);   // L3 per net
    probe_ws_gemm(1, 24576, 512, 256, 256, 2, st);   // dX2 per net
    probe_ws_gemm(1, 24576, 256, 128, 256, 2, st);   // dX3 per net
    probe_ws_gemm(1, 24576, 256, 128, 128, 2, st);
    probe_ws_gemm(0, 1000, 1024, 256, 256, 1, st);   // ragged rows
    probe_ws_gemm(1, 700, 512, 256, 256, 2, st);
    return 0;
  }
  if (!strcmp(which, "fused")) {
    probe_fused(4096, st);
    probe_fused(1024, st);
    return 0;
  }
  if (!strcmp(which, "pair")) {
    probe_dw_pair(256, 128, 640, 256, 2, st);       // small sanity: 1 pair tile, 2 splits
    probe_dw_pair(1024, 240, 24576, 256, 18, st);   // dW1 (both nets): 4 pair tiles x 18 splits = 144 CTAs
    probe_dw_pair(512, 512, 24576, 256, 18, st);    // dW2 both nets as 4 pair tiles
    probe_dw_pair(1024, 240, 24576, 256, 12, st);
    probe_dw_pair(512, 512, 24576, 256, 12, st);
    return 0;
  }
  if (!strcmp(which, "kmaj")) {
    probe_dw_kmajor(1024, 240, 24576, 256, 18, 1, st);
    probe_dw_kmajor(512, 512, 24576, 256, 18, 1, st);
    return 0;
  }
  if (!strcmp(which, "all") || !strcmp(which, "fwd")) {
    probe_fwd(16384, 8192, 8192, 256, st);   // large square-ish: pipeline/peak sanity
    probe_fwd(24576, 1024, 256, 256, st);    // layer 1 (both nets), K = Dp (256 padded)
    probe_fwd(24576, 256, 512, 256, st);     // layer 2 (one net)
    probe_fwd(24576, 128, 256, 128, st);     // layer 3 (one net)
    probe_fwd(128, 64, 64, 64, st);          // one tile, one k-block: fixed cost of a launch
    probe_fwd(4096, 1024, 256, 256, st);     // rollout layer 1 (both nets)
    probe_fwd(4096, 256, 512, 256, st);      // rollout layer 2 (one net)
  }
  if (!strcmp(which, "all") || !strcmp(which, "dw")) {
    const int sp1[] = {8, 12, 16, 18};
    for (int S : sp1) probe_dw(1024, 240, 24576, 256, S, 1, st);  // dW1 (both nets)
    for (int S : sp1) probe_dw(512, 512, 24576, 256, S, 1, st);   // dW2 both nets as 8 tiles
    const int sp3[] = {16, 32, 48, 74};
    for (int S : sp3) probe_dw(256, 256, 24576, 256, S, 1, st);   // dW3 both nets as 2 tiles
    probe_dw(128, 64, 64, 64, 1, 1, st);       // one CTA, one k-block: fixed cost of a launch
    check_dw(1024, 240, 24576, 256, 18, 1, st);
    check_dw(256, 256, 24576, 256, 74, 1, st);
    check_dw(200, 96, 1000, 128, 12, 1, st);
  }
  printf("done\n");
  return 0;
}
