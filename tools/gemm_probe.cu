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
#include <vector>

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
  for (int probe = 0; probe < 3; ++probe) {
    g.probe = probe;
    float us = time_us([&] { CK(launch_gemm(GEMM_FWD, bn, g, st)); }, st);
    const double bytes = ((double)M * K + (double)g.m_tiles * 128.0 * 0 + (double)N * K * g.m_tiles) * 2.0;
    printf("fwd M=%d N=%d K=%d bn=%d probe=%d  %8.2f us  %7.1f TFLOP/s  operand-load %7.1f GB/s\n", M, N, K, bn,
           probe, us, fl / us * 1e-6, bytes / us * 1e-3);
  }
  CK(cudaFree(X)); CK(cudaFree(W)); CK(cudaFree(Y)); CK(cudaFree(bias));
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
  g.kb_per_split = (g.kb_total + S * G - 1) / (S * G);
  CK(cudaMalloc(&part, (size_t)tiles * G * 128 * (bn + 4) * 4));
  CK(cudaMalloc(&cnt, (size_t)tiles * S * 4));
  CK(cudaMemset(cnt, 0, (size_t)tiles * S * 4));
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

static void check_dw(int Nout, int Nin, int K, int bn, int S, int G, cudaStream_t st) {
  std::vector<float> a = probe_dw(Nout, Nin, K, bn, S, 1, st, true);
  std::vector<float> b = probe_dw(Nout, Nin, K, bn, S, G, st, true);
  double num = 0, den = 0;
  for (size_t i = 0; i + 64 < a.size(); ++i) { num += (a[i] - b[i]) * (double)(a[i] - b[i]); den += (double)a[i] * a[i]; }
  printf("check dw Nout=%d Nin=%d G=%d vs G=1: rel l2 %.3e (payload %g)\n", Nout, Nin, G, std::sqrt(num / den),
         b[(size_t)Nout * Nin + Nout + 4]);
}

__global__ void k_empty(int* p) {
  extern __shared__ int sm[];
  if (p && threadIdx.x == 0) p[blockIdx.x] = sm[0];
}

int main(int argc, char** argv) {
  cudaStream_t st;
  CK(cudaStreamCreate(&st));
  CK(cudaMalloc(&g_flush, 512u << 20));
  const char* which = argc > 1 ? argv[1] : "all";
  if (argc > 2 && !strcmp(argv[2], "noflush")) g_do_flush = false;
  if (!strcmp(which, "one") || !strcmp(which, "onefwd")) g_do_flush = false;
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
    printf("max active clusters: bn256 S8 %d, S4 %d, S16 %d; bn128 S8 %d\n", dw_max_active_clusters(256, 8),
           dw_max_active_clusters(256, 4), dw_max_active_clusters(256, 16), dw_max_active_clusters(128, 8));
    const int cfgs[][2] = {{8, 1}, {4, 4}, {2, 8}, {1, 16}};
    for (auto& c : cfgs) probe_dw(1024, 240, 24576, 256, c[0], c[1], st);  // dW1 (both nets)
    for (auto& c : cfgs) probe_dw(256, 512, 24576, 256, c[0], c[1], st);   // dW2 (one net: x2 for both)
    probe_dw(512, 512, 24576, 256, 8, 2, st);                                // dW2 both nets as 4 tiles
    const int cfg3[][2] = {{8, 1}, {8, 4}, {8, 8}, {4, 16}};
    for (auto& c : cfg3) probe_dw(128, 256, 24576, 256, c[0], c[1], st);   // dW3 (one net)
    probe_dw(256, 256, 24576, 256, 8, 8, st);                                // dW3 both nets as 2 tiles
    probe_dw(128, 64, 64, 64, 1, 1, st);       // one CTA, one k-block: fixed cost of a launch
    probe_dw(128, 64, 1024, 64, 8, 1, st);     // one cluster of 8, 2 k-blocks each
    probe_dw(1024, 256, 4096, 256, 8, 1, st);  // 64 CTAs, 8 k-blocks each
    check_dw(1024, 240, 24576, 256, 8, 2, st);
    check_dw(128, 256, 24576, 256, 8, 8, st);
    check_dw(200, 96, 1000, 128, 4, 3, st);
  }
  printf("done\n");
  return 0;
}
