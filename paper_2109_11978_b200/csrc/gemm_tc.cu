// gemm_tc.cu -- persistent, warp-specialized tcgen05 bf16 GEMM for sm_100a (TMA operand staging,
// mbarrier pipelines, fp32 accumulators in TMEM, TMA stores), with the MLP's epilogues fused
// (the one dense contraction of the path, BJ north_star).
//
//   D[m][n] = sum_k A[m][k] * B[n][k]       (tile 128 x BN, K-blocks of 64 = one 128-B swizzle atom)
//
// Operand majorness (instruction-descriptor bits 15/16):
//   forward      Y = X W^T       A K-major (activations), B K-major (weights [out][in])
//   backward dX  dX = dZ W       A K-major (dZ),          B MN-major (W read as [k=out][n=in])
//   backward dW  dW = dZ^T X     A MN-major (dZ [batch][out]), B MN-major (X [batch][in]); split-K over
//                                the batch, plus a 16-column "ones" MMA that yields db = colsum(dZ) in the
//                                same pass (bias gradients for free).
// Epilogues: 0 = +bias, ELU -> bf16 ; 2 = * ELU'(saved activation) -> bf16 ; 3 = fp32 split-K partial.
//
// CTA = 12 warps, one CTA per SM, grid = min(tiles, #SMs), static round-robin tile schedule:
//   warp 0 lane 0: TMA producer (STAGES-deep smem ring, full/empty mbarriers)
//   warp 1 lane 0: tcgen05.mma issuer; accumulators double-buffered in TMEM (tmem_full/empty mbarriers)
//   warp 2      : TMEM allocation owner
//   warps 4..11 : epilogue; warp 4+e reads TMEM lanes 32(e%4).. and column half e/4, stages 32x64 bf16
//                 (or 32x32 fp32) sub-tiles in 128-B-swizzled smem and writes them with TMA stores, so the
//                 epilogue of tile i overlaps the MMA of tile i+1.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"

namespace lg {

// ------------------------------------------------------------------ PTX wrappers

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// mbarrier wait: a plain try_wait loop (mode 1). A suspend-time hint (mode 0) lets a waiting thread sleep
// until the hint expires when the phase is completed from the peer CTA of a pair (multicast tcgen05.commit /
// the peer's TMA complete_tx): the CTA-pair kernel then crawls. Mode 2 = test_wait spin, 3 = bounded (probe).
#ifndef LG_MBAR_MODE
#define LG_MBAR_MODE 1
#endif
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
#if LG_MBAR_MODE == 0
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n\t"
      "@P1 bra DONE_%=;\n\t"
      "bra WAIT_%=;\n\t"
      "DONE_%=:\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity), "r"(0x989680));
#elif LG_MBAR_MODE == 3
  // diagnostics build (tools/gemm_probe3): bounded wait that reports the stuck barrier and gives up
  uint32_t ok = 0;
  for (long long it = 0; it < (1ll << 22) && !ok; ++it) {
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, P1;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity));
  }
  if (!ok) {
    uint32_t rk;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rk));
    printf("mbar timeout: block (%d,%d) rank %u thread %d bar smem 0x%x parity %u\n", blockIdx.x, blockIdx.y, rk,
           threadIdx.x, smem_u32(bar), parity);
  }
#elif LG_MBAR_MODE == 1
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra DONE_%=;\n\t"
      "bra WAIT_%=;\n\t"
      "DONE_%=:\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity));
#else
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra DONE_%=;\n\t"
      "bra WAIT_%=;\n\t"
      "DONE_%=:\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity));
#endif
}
__device__ __forceinline__ void tma_load_2d(const CUtensorMap* map, uint64_t* bar, void* dst, int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(x), "r"(y)
      : "memory");
}
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, const void* src, int x, int y) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(smem_u32(src)), "r"(x), "r"(y)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read1() { asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tc_mma(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc));
}
// 32 consecutive fp32 columns of this thread's TMEM lane (no wait)
__device__ __forceinline__ void tmem_ld32_nowait(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,"
      "%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
// 16 consecutive fp32 columns of this thread's TMEM lane (no wait)
__device__ __forceinline__ void tmem_ld16_nowait(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}

// ---- CTA-pair (tcgen05 cta_group::2) helpers
__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t mapa_shared(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
__device__ __forceinline__ void cluster_barrier() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// TMA load into this CTA's smem, completing on an mbarrier of either CTA of the pair (shared::cluster address)
__device__ __forceinline__ void tma_load_2d_pair(const CUtensorMap* map, uint32_t mbar_cluster, void* dst, int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(mbar_cluster), "r"(x), "r"(y)
      : "memory");
}
__device__ __forceinline__ void tc_mma_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void tc_commit_pair(uint64_t* bar) {  // arrive on `bar` (same offset) in both CTAs
  asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                   smem_u32(bar)),
               "h"((uint16_t)3)
               : "memory");
}

// Shared-memory matrix descriptor (SM100 version 1), 128-byte swizzle.
//  K-major : rows of 128 B (64 bf16 of K), 8-row atoms 1024 B apart (SBO); LBO unused.
//  MN-major: rows of 128 B (64 bf16 of M or N) indexed by k; 8-k atoms 1024 B apart (SBO),
//            64-wide MN atoms LBO = 64 k-rows * 128 B = 8192 B apart.
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= 1ull << 46;  // version (sm100)
  d |= 2ull << 61;  // SWIZZLE_128B
  return d;
}

// Instruction descriptor, kind::f16: D f32, A/B bf16, majorness, N>>3, M>>4.
__host__ __device__ constexpr uint32_t idesc_bf16(int M, int N, bool a_mn, bool b_mn) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((a_mn ? 1u : 0u) << 15) | ((b_mn ? 1u : 0u) << 16) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

constexpr int GEMM_THREADS = 384;  // 4 control warps + 8 epilogue warps
constexpr int EPI_WARPS = 8;

// ------------------------------------------------------------------ the policy / value heads on the tensor core
// Shared by the rollout policy (k_policy_fused) and the update's loss epilogue (EPI 4) so both produce the same
// mu and V bits (the first minibatch's probability ratio is exactly 1):
//   D1[row][16p + j] = sum_c H3[row][c] W4_p[j][c],  head output j = (D1[j] + D1[16 + j]) + D1[32 + j]
// (M = 128 rows, N = 48, K = 128 H3 columns). W4 of one net is split into three bf16 parts whose sum is the fp32
// weight exactly (split3_bf16), so the tensor core sees the fp32 operands of the CUDA-core head. A = H3 as two
// K-major SW128 blocks of 64 columns 16 KB apart (the layer activation layout); B = the parts stacked as 48 rows
// (16p + j; rows j >= 12, or >= 1 for the critic, and columns >= H2 are zero) of 128 B in two 64-column SW128
// atoms 6 KB apart. The same atoms are the MN-major B (N = column, K = j; part p at row 16p, LBO 6 KB) of the
// head-input gradient dH3 = dmu W4.
__device__ __forceinline__ uint16_t bf16_bits(float x) {
  const __nv_bfloat16 b = __float2bfloat16_rn(x);
  return *reinterpret_cast<const uint16_t*>(&b);
}
// fp32 x = p0 + p1 + p2 exactly, each part a bf16 (8 significant bits): RNE to bf16, then the exact fp32 residual
__device__ __forceinline__ void split3_bf16(float x, uint16_t* p) {
  p[0] = bf16_bits(x);
  const float r1 = x - __uint_as_float((uint32_t)p[0] << 16);
  p[1] = bf16_bits(r1);
  p[2] = bf16_bits(r1 - __uint_as_float((uint32_t)p[1] << 16));
}
constexpr int W4_ATOM = 48 * 128;      // bytes of one 64-column atom (48 rows)
constexpr int W4_BYTES = 2 * W4_ATOM;  // the head-weight operand of one net
// element (j, c) part p: atom c / 64, row 16p + j, chunk (c % 64) / 8 ^ (j & 7). In two phases so that a caller's
// other prologue loads share one round trip: w4_load (elements t0 + i * nt, i < 8: nt >= 256 threads), w4_store.
__device__ __forceinline__ void w4_load(float* v, const float* W4a, const float* W4c, int H2, int z, int t0, int nt) {
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int k = t0 + i * nt, j = k >> 7, c = k & 127;
    v[i] = 0.0f;
    if (k < 16 * 128 && c < H2) v[i] = z == 0 ? (j < 12 ? __ldg(W4a + j * H2 + c) : 0.0f) : (j == 0 ? __ldg(W4c + c) : 0.0f);
  }
}
__device__ __forceinline__ void w4_store(uint8_t* w4, const float* v, int t0, int nt) {
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int k = t0 + i * nt, j = k >> 7, c = k & 127;
    if (k >= 16 * 128) break;
    uint16_t pt[3];
    split3_bf16(v[i], pt);
#pragma unroll
    for (int u = 0; u < 3; ++u)
      *reinterpret_cast<uint16_t*>(w4 + (c >> 6) * W4_ATOM + (16 * u + j) * 128 + ((((c & 63) >> 3) ^ (j & 7)) << 4) +
                                   2 * (c & 7)) = pt[u];
  }
}
__device__ __forceinline__ void build_w4_atoms(uint8_t* w4, const float* W4a, const float* W4c, int H2, int z, int t0,
                                               int nt) {
  float v[8];
  w4_load(v, W4a, W4c, H2, z, t0, nt);
  w4_store(w4, v, t0, nt);
}
// issued by one thread: the two 64-column blocks in K steps of 16
__device__ __forceinline__ void head_mma(uint32_t d1, uint32_t a3, uint32_t w4) {
  constexpr uint32_t id = idesc_bf16(128, 48, false, false);
#pragma unroll
  for (int kb = 0; kb < 2; ++kb)
#pragma unroll
    for (int k = 0; k < 4; ++k)
      tc_mma(d1, sdesc(a3 + kb * 16384u + 32u * k, 0u, 1024u), sdesc(w4 + kb * (uint32_t)W4_ATOM + 32u * k, 0u, 1024u),
             id, (kb > 0 || k > 0) ? 1u : 0u);
}
// head output j from the 48 accumulator columns of a row (fixed order)
__device__ __forceinline__ float head_out(const uint32_t* d, int j) {
  return (__uint_as_float(d[j]) + __uint_as_float(d[16 + j])) + __uint_as_float(d[32 + j]);
}

// EPI 4 (loss epilogue) shared-memory carve-up (offsets from a 1024-B aligned base):
//  A3     the tile's H3 [128 rows][128] bf16 as two K-major SW128 blocks of 64 columns: A of the head MMA (K-major,
//         M = row, K = column), MN-major A (M = column, K = row) of the head-weight gradient, and afterwards the
//         staging buffer of the dZ3 TMA stores (its 32-row x 64-column sub-tiles are SW128 store boxes)
//  DMU    dmu (actor) / dV (critic) per row as three bf16 parts (split3_bf16: their sum is the fp32 value), part p
//         of output j at column 16p + j of a 128-B row (columns >= 48 zero): K-major A (M = row, K = head output;
//         part p at K offset 16p) of dH3 = dmu W4, MN-major B (N = 48 part columns, K = row) of dW4
//  W4     the net's head weights as build_w4_atoms lays them out
//  REC    per-row records, column-major: [25][128] fp32 (dmu[12], dV, dlogstd terms[12]), [5][128] fp64 statistics
//  CST    per-dimension constants (log sigma, sigma^-2, KL constant, b4a, e^-log sigma); BIAS b3 of the CTA's net
namespace le {
constexpr int A3 = 0;
constexpr int DMU = A3 + 32768;  // [128 rows][128 B]: part p of dmu_j at column 16p + j
constexpr int W4 = DMU + 16384;  // build_w4_atoms
constexpr int REC = W4 + W4_BYTES;
constexpr int REC_NF = 25, REC_ND = 5;           // column-major: [25][128] fp32, then [5][128] fp64
constexpr int CST = REC + 128 * (REC_NF * 4 + REC_ND * 8);
constexpr int BIAS = CST + 64 * 4;
constexpr int BYTES = BIAS + 128 * 4;
// TMEM columns: the layer-3 accumulators use [0, 256)
constexpr int TM_D2 = 256;  // dH3 [row][128]
constexpr int TM_D3 = 384;  // dW4 accumulator [column][48] (part p of output j at 16p + j), across the CTA's tiles
constexpr int TM_D1 = 448;  // head outputs [row][48] (head_out)
static_assert(REC % 8 == 0 && BYTES % 16 == 0 && W4 % 1024 == 0, "loss epilogue smem alignment");
}  // namespace le

template <int BN, int EPI, bool PAIR = false, int WSKB = 0>
struct GemmCfg {
  static constexpr int BM = 128, BK = 64;
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int B_BYTES = (PAIR ? BN / 2 : BN) * BK * 2;  // a CTA of a pair holds half of B
  static constexpr int ONES_BYTES = EPI == 3 ? 16 * 128 : 0;  // 16 rows x 64 bf16 of 1.0 (bias column)
  static constexpr int EPI_BUF = 4096;         // one 32 x 128-B staging sub-tile
  // staging buffers per epilogue warp: EPI 4 stages dZ3 in its own smem; weight-stationary forward GEMMs have room
  // for one (their resident B takes the rest); the weight-stationary dX2 takes two and stages its saved activation
  // by coalesced cp.async like the other dX GEMMs (A ring 4 -> 2 stages; same-box A/B -0.3 % per C3 iteration
  // against one buffer with the activation loaded per row into registers and prefetched into L2)
  static constexpr int EPI_NBUF = EPI == 4 ? 0 : ((EPI == 3 || (WSKB && EPI != 2)) ? 1 : 2);
  static constexpr int BIAS_BYTES = EPI == 0 ? EPI_WARPS * 128 * 4 : 0;
  static constexpr int LOSS_BYTES = EPI == 4 ? le::BYTES : 0;
  static constexpr int BRES = WSKB * B_BYTES;  // weight-stationary: the resident column block of B
  static constexpr int FIXED = 1024 + ONES_BYTES + EPI_WARPS * EPI_NBUF * EPI_BUF + BIAS_BYTES + LOSS_BYTES + 512 + BRES;
  static constexpr int STAGE_BYTES = WSKB ? A_BYTES : A_BYTES + B_BYTES;
  static constexpr int STAGES_FIT = (232448 - FIXED) / STAGE_BYTES;
  static constexpr int STAGES = STAGES_FIT > 8 ? 8 : STAGES_FIT;
  static constexpr int ACC_COLS = ((BN + (EPI == 3 ? 16 : 0)) + 31) / 32 * 32;
  static constexpr int ACC_STAGES = 2 * ACC_COLS <= 512 ? 2 : 1;
  static constexpr int TMEM_NEED = ACC_STAGES * ACC_COLS;
  static constexpr int TMEM_COLS = EPI == 4 ? 512 : TMEM_NEED <= 32 ? 32 : TMEM_NEED <= 64 ? 64 : TMEM_NEED <= 128 ? 128 : TMEM_NEED <= 256 ? 256 : 512;
  static constexpr int SMEM = FIXED + STAGES * STAGE_BYTES;
  static_assert(STAGES >= 2, "operand ring");
  static_assert(EPI != 2 || EPI_NBUF == 2, "input-gradient epilogues stage the saved activation");
};

// ELU(x) = x > 0 ? x : e^x - 1, with e^x = 2^(x log2 e) from ex2.approx.ftz (one MUFU op, no subnormal
// rescaling path: the bf16 output cannot resolve e^x - 1 differences below 2^-126 anyway)
__device__ __forceinline__ float ex2_ftz(float t) {
  float e;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(t));
  return e;
}
__device__ __forceinline__ float elu_fast(float x) {
  const float e = ex2_ftz(x * 1.4426950408889634f) - 1.0f;
  return x > 0.0f ? x : e;
}
__device__ __forceinline__ float4 lds4(const float* p) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(smem_u32(p)));
  return v;
}

// write one thread's 128-byte row chunk (8 x 16 B) into a 32-row, 128-B-swizzled staging buffer
__device__ __forceinline__ void stage_row(uint8_t* buf, int lane, const uint32_t* w32) {
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    uint4 v = make_uint4(w32[4 * j], w32[4 * j + 1], w32[4 * j + 2], w32[4 * j + 3]);
    *reinterpret_cast<uint4*>(buf + lane * 128 + ((j ^ (lane & 7)) << 4)) = v;
  }
}

struct TileCoord {
  int z, m0, n0, split, ntile;
};

// dX epilogue: the saved activation H (for ELU'(x) = min(H + 1, 1)) of a warp's 32 rows x 64 columns,
// loaded with coalesced 16-B cp.async (8 lanes per 128-B row, 4 rows per instruction) into the warp's staging
// buffer in the swizzled layout stage_row writes (chunk j of row r at r * 128 + ((j ^ (r & 7)) << 4)), then
// read back row-per-lane. Thread-per-row global loads touch 32 lines per instruction; this touches 4.
__device__ __forceinline__ void aux_issue(uint8_t* buf, const __nv_bfloat16* aux, int ld, int row0, int M, int nb,
                                          int N, int lane) {
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int r = 4 * i + (lane >> 3), ch = lane & 7;
    const bool ok = row0 + r < M && nb + 8 * ch < N;
    const __nv_bfloat16* src = aux + (size_t)(ok ? row0 + r : 0) * ld + (ok ? nb + 8 * ch : 0);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(buf + r * 128 + ((ch ^ (r & 7)) << 4))),
                 "l"(src), "r"(ok ? 16 : 0)
                 : "memory");
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
}
__device__ __forceinline__ void aux_read(const uint8_t* buf, uint32_t* av, int lane) {
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  __syncwarp();
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const uint4 u = *reinterpret_cast<const uint4*>(buf + lane * 128 + ((j ^ (lane & 7)) << 4));
    av[4 * j] = u.x; av[4 * j + 1] = u.y; av[4 * j + 2] = u.z; av[4 * j + 3] = u.w;
  }
}
__device__ __forceinline__ TileCoord decode(const GemmArgs& a, int t, int m_tiles, int BN) {
  TileCoord c;
  c.ntile = t % a.n_tiles;
  int r = t / a.n_tiles;
  c.m0 = (r % m_tiles) * 128;
  r /= m_tiles;
  c.split = r % a.n_splits;
  c.z = r / a.n_splits;
  c.n0 = c.ntile * BN;
  return c;
}

// ------------------------------------------------------------------ EPI 4: the PPO loss head in the epilogue
// Layer 3 of the update (tile = 128 rows x 128 columns of one net: the CTA serves one net, z = 0 actor, 1 critic)
// ends the forward pass and starts the backward one in the same epilogue; H3 never goes to
// HBM. Per tile:
//  1. H3 = bf16(ELU(acc + b3)) into smem (A3; thread (row, h) writes columns 64h .. 64h+63).
//  2. one thread issues the head MMA (head_mma: mu - b4a or V - b4c, the rollout kernel's instruction sequence, so
//     the first minibatch's probability ratio is exactly 1); every thread reads its row's 16 outputs.
//  3. per row (both threads): log-probability (dim_sum12), ratio, clipped surrogate / value loss (the shared
//     ppo_dlogp / ppo_dvalue), KL; dmu_j = dL/dlogp (a_j - mu_j) / sigma_j^2, or dV -> smem as three bf16 parts
//     (split3_bf16: exact), so the tensor core sees the fp32 operands of the two-kernel path.
//  4. one thread issues dH3 = dmu W4 (K = 16; part products of order <= 2) into TMEM and dW4 += H3^T dmu (K = the
//     tile's 128 rows; N = the 48 part columns) into a TMEM accumulator that lives across the CTA's tiles;
//     meanwhile each warp sums its per-row record columns (head biases, log-std, loss statistics) over the rows.
//  5. dZ3 = dH3 * ELU'(H3) -> bf16 over H3 in A3 -> TMA stores.
// At the end the CTA writes its partial row (k_loss_heads layout) to le.part / le.spart; k_reduce_heads sums the
// rows in CTA order (deterministic). Ownership: dW4 = the D3 accumulator, TMEM lane c read by warps 4..7; record
// column col < 25 (dmu_j -> db4a, dV -> db4c, dlogstd terms; fp64 statistics surrogate, value loss, KL, clip
// count, non-finite rows) by lane 0 of epilogue warp col % 8.
constexpr float SIX_LN_2PI_F = 11.027262398456072f;
__device__ __forceinline__ float elu_grad_out(float h) { return h > 0.0f ? 1.0f : h + 1.0f; }
__device__ __forceinline__ void bar_epi() { asm volatile("bar.sync 1, 256;" ::: "memory"); }

__device__ __forceinline__ unsigned long long loss_gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define LOSS_STAMP(k)                                                                                          \
  do {                                                                                                         \
    if (L.dbg && et == 0) L.dbg[((size_t)blockIdx.x * 8 + (local - 1 < 7 ? local - 1 : 7)) * 16 + (k)] = loss_gtimer(); \
  } while (0)

// warp 3, one thread: per tile, the head MMA once the epilogue has staged H3 (lmma[2]), the gradient MMAs once it
// has staged dmu (lmma[3]); completions on lmma[0] / lmma[1]. (Issued from a converged control warp the
// descriptors stay on the uniform datapath; from an epilogue thread each MMA paid ~6 register-to-uniform moves.)
template <typename C, typename TileAt, typename Skip>
__device__ __forceinline__ void loss_mma(TileAt tile_at, Skip skip, uint32_t tmem, uint64_t* lmma, uint8_t* sLoss) {
  const uint32_t tD1 = tmem + le::TM_D1, tD2 = tmem + le::TM_D2, tD3 = tmem + le::TM_D3;
  constexpr uint32_t id2 = idesc_bf16(128, 128, false, true);  // dH3 [row][col] = dmu [row][j] . W4 [j][col]
  constexpr uint32_t id3 = idesc_bf16(128, 48, true, true);    // dW4 [col][16p+j] += H3^T [col][row] . dmu_p [row][j]
  const uint32_t a3 = smem_u32(sLoss + le::A3), dmu = smem_u32(sLoss + le::DMU), w4 = smem_u32(sLoss + le::W4);
  int local = 0;
  TileCoord tc;
  for (int it = 0; tile_at(it, tc); ++it) {
    if (skip(tc)) continue;
    const uint32_t ph = (uint32_t)(local & 1);
    const bool first = local == 0;
    ++local;
    mbar_wait(&lmma[2], ph);
    tc_fence_after();
    head_mma(tD1, a3, w4);
    tc_commit(&lmma[0]);
    mbar_wait(&lmma[3], ph);
    tc_fence_after();
    // dH3: the part products of order <= 2 (00, 01, 10, 02, 20, 11); the dropped ones are below 2^-24 relative.
    // dmu part p sits at K offset 16p of the DMU rows (32 B), W4 part p at row 16p of its atoms (2 KB)
    constexpr int PA[6] = {0, 0, 1, 0, 2, 1}, PB[6] = {0, 1, 0, 2, 0, 1};
#pragma unroll
    for (int t = 0; t < 6; ++t)
      tc_mma(tD2, sdesc(dmu + PA[t] * 32u, 0u, 1024u), sdesc(w4 + PB[t] * 2048u, (uint32_t)W4_ATOM, 1024u), id2,
             t > 0 ? 1u : 0u);
#pragma unroll
    for (int ks = 0; ks < 8; ++ks)  // K = the tile's 128 rows in steps of 16 (2 KB of 128-B rows)
      tc_mma(tD3, sdesc(a3 + ks * 2048u, 16384u, 1024u), sdesc(dmu + ks * 2048u, 16384u, 1024u), id3,
             (first && ks == 0) ? 0u : 1u);
    tc_commit(&lmma[1]);
  }
}

template <typename C, typename TileAt, typename Skip>
__device__ __forceinline__ void loss_epilogue(const GemmArgs& args, int M, TileAt tile_at, Skip skip, uint32_t tmem,
                                              uint64_t* tfull, uint64_t* tempty, uint64_t* lmma, uint8_t* sLoss,
                                              int z) {
  const LossEpi& L = args.le;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int e = warp - 4, q = e & 3, h = e >> 2;
  const int et = threadIdx.x - 128;
  uint8_t* sA3 = sLoss + le::A3;
  uint8_t* sD = sLoss + le::DMU;
  float* sRec = reinterpret_cast<float*>(sLoss + le::REC);
  float* sCst = reinterpret_cast<float*>(sLoss + le::CST);  // ls | sigma^-2 | KL constant | b4a | e^-ls ([12] each)
  float* sBias = reinterpret_cast<float*>(sLoss + le::BIAS);
  const int H2 = L.H2;
  if (L.dbg && et == 0) L.dbg[(size_t)blockIdx.x * 128 + 8] = loss_gtimer();  // (diagnostics: epilogue entry)
  // ---- once per CTA: the net's head weights (three bf16 parts), constants, b3, zeroed operands / records; every
  // global load of the prologue is issued first (one round trip instead of one per step)
  float w4v[8];
  w4_load(w4v, L.W4a, L.W4c, H2, z, et, 256);
  float ls = 0.0f, lso = 0.0f, b4a = 0.0f, b3 = 0.0f;
  if (et < 12) {
    ls = __ldg(L.logstd + et);
    lso = __ldg(L.logstd_old + et);
    b4a = __ldg(L.b4a + et);
  }
  if (et < args.N && et < 128) b3 = __ldg(args.bias[z] + et);
  const float b4c = __ldg(L.b4c);
  for (int k = et; k < 16384 / 16; k += 256) reinterpret_cast<uint4*>(sD)[k] = make_uint4(0u, 0u, 0u, 0u);
  for (int k = et; k < 128 * (le::REC_NF + 2 * le::REC_ND); k += 256) sRec[k] = 0.0f;  // columns a net never writes stay zero
  double* sRecD = reinterpret_cast<double*>(sRec + 128 * le::REC_NF);
  w4_store(sLoss + le::W4, w4v, et, 256);
  if (et < 12) {
    const float iv = expf(-2.0f * ls);
    sCst[et] = ls;
    sCst[12 + et] = iv;
    sCst[24 + et] = kl_const(ls, lso, iv);
    sCst[36 + et] = b4a;
    sCst[48 + et] = expf(-ls);  // the per-dimension factor of logp_term, once per CTA (same bits as per row)
  }
  if (et < 128) sBias[et] = b3;
  // the first payload writer of the minibatch clears the non-finite counter (the previous minibatch's Adam has
  // consumed it: this kernel runs after that minibatch's layers 1, 2)
  if (blockIdx.x == 0 && et == 0 && L.payload) L.payload[4] = 0.0f;
  // record-column sums (lane 0 of warp e owns float columns e, e + 8, e + 16, e + 24 (< 25) and fp64 statistic
  // e (< 5))
  float xf[4] = {0.0f, 0.0f, 0.0f, 0.0f};
  double xd = 0.0;
  fence_async_smem();
  bar_epi();
  const uint32_t tD1 = tmem + le::TM_D1, tD2 = tmem + le::TM_D2, tD3 = tmem + le::TM_D3;
  constexpr uint32_t id2 = idesc_bf16(128, 128, false, true);  // dH3 [row][col] = dmu [row][j] . W4 [j][col]
  constexpr uint32_t id3 = idesc_bf16(128, 48, true, true);    // dW4 [col][16p+j] += H3^T [col][row] . dmu_p [row][j]
  const int r = q * 32 + lane;
  const uint32_t lrow = (uint32_t)(q * 32) << 16;
  // 16-B chunk ch (columns 8ch .. 8ch+7) of this thread's 64 columns of row r in A3 (block h, swizzled by row)
  auto a3_chunk = [&](int ch) { return sA3 + h * 16384 + r * 128 + ((ch ^ (r & 7)) << 4); };
  int local = 0;
  TileCoord tc;
  for (int it = 0; tile_at(it, tc); ++it) {
    if (skip(tc)) continue;
    const int acc = local % C::ACC_STAGES;
    const uint32_t aph = (uint32_t)((local / C::ACC_STAGES) & 1);
    const uint32_t mph = (uint32_t)(local & 1);  // lmma[0], lmma[1] complete once per tile
    ++local;
    const int row = tc.m0 + r;
    const bool valid = row < M;
    // row inputs (independent of the accumulator: their loads overlap the waits below)
    float in_a[12], in_m[12];
    float lpo = 0.0f, adv = 0.0f, Vo = 0.0f, ret = 0.0f;
#pragma unroll
    for (int j = 0; j < 12; ++j) in_a[j] = in_m[j] = 0.0f;
    if (valid) {
      if (z == 0) {
        const float4* pa = reinterpret_cast<const float4*>(L.act + (size_t)row * 12);
        const float4* pm = reinterpret_cast<const float4*>(L.mu_old + (size_t)row * 12);
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          const float4 va = __ldg(pa + k), vm = __ldg(pm + k);
          in_a[4 * k] = va.x; in_a[4 * k + 1] = va.y; in_a[4 * k + 2] = va.z; in_a[4 * k + 3] = va.w;
          in_m[4 * k] = vm.x; in_m[4 * k + 1] = vm.y; in_m[4 * k + 2] = vm.z; in_m[4 * k + 3] = vm.w;
        }
        lpo = __ldg(L.logp_old + row);
        adv = __ldg(L.adv + row);
      } else {
        Vo = __ldg(L.V_old + row);
        ret = __ldg(L.ret + row);
      }
    }
    LOSS_STAMP(0);
    if (lane == 0) bulk_wait_read0();  // this warp's previous dZ3 store has read its A3 sub-tile
    __syncwarp();
    bar_epi();                         // every warp's: A3 is free
    LOSS_STAMP(1);
    mbar_wait(&tfull[acc], aph);
    __syncwarp();
    tc_fence_after();
    LOSS_STAMP(2);
    // (1) H3 = bf16(ELU(acc + b3)) of columns 64h .. 64h+63 into A3
    {
      const uint32_t tb = tmem + acc * C::ACC_COLS + lrow + 64 * h;
      uint32_t a32[2][32];
      tmem_ld32_nowait(tb, a32[0]);
      tmem_ld32_nowait(tb + 32, a32[1]);
      tmem_wait_ld();
#pragma unroll
      for (int ch = 0; ch < 8; ++ch) {
        uint32_t w[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int c = 8 * ch + 2 * k;
          const float2 b2 = *reinterpret_cast<const float2*>(sBias + 64 * h + c);
          const __nv_bfloat162 p = __floats2bfloat162_rn(elu_fast(__uint_as_float(a32[c >> 5][c & 31]) + b2.x),
                                                         elu_fast(__uint_as_float(a32[c >> 5][(c & 31) + 1]) + b2.y));
          w[k] = *reinterpret_cast<const uint32_t*>(&p);
        }
        *reinterpret_cast<uint4*>(a3_chunk(ch)) = make_uint4(w[0], w[1], w[2], w[3]);
      }
    }
    fence_async_smem();
    tc_fence_before();  // the accumulator stage is free once read: the next tile's layer-3 MMAs may start
    __syncwarp();
    if (lane == 0) {
      mbar_arrive(&tempty[acc]);
      mbar_arrive(&lmma[2]);  // H3 staged: warp 3 issues the head MMA
    }
    // (2) the head MMA
    mbar_wait(&lmma[0], mph);
    __syncwarp();
    tc_fence_after();
    uint32_t d1[48];
    tmem_ld32_nowait(tD1 + lrow, d1);
    tmem_ld16_nowait(tD1 + lrow + 32, d1 + 32);
    tmem_wait_ld();
    LOSS_STAMP(3);
    // (3) the row's loss terms; dmu / dV (the three parts: chunks 0..5 of the DMU row, 0..3 by the thread of h = 0,
    // 4, 5 by h = 1) and the row record
    float* rec = sRec + r;     // column col at rec[col * 128]
    double* rd = sRecD + r;    // statistic k at rd[k * 128]
    float dq[12];
    if (z == 0) {
      float mu[12], t[12];
#pragma unroll
      for (int j = 0; j < 12; ++j) {
        mu[j] = __fadd_rn(head_out(d1, j), sCst[36 + j]);
        t[j] = logp_term_e(in_a[j], mu[j], sCst[48 + j], sCst[j]);
      }
      const float lp = __fsub_rn(-dim_sum12(t), SIX_LN_2PI_F);
      const float ratio = expf(lp - lpo);
      float svf = 0.0f;
      bool clipped = false;
      const float dLdlp = valid ? ppo_dlogp(ratio, adv, L.clip, L.invM, svf, clipped) : 0.0f;
#pragma unroll
      for (int j = 0; j < 12; ++j) {
        const float d = in_a[j] - mu[j];
        dq[j] = dLdlp * d * sCst[12 + j];
        const float dm = in_m[j] - mu[j];
        t[j] = kl_term(sCst[24 + j], dm, sCst[12 + j]);
        if (h == 0) {
          rec[j * 128] = dq[j];
          rec[(13 + j) * 128] = valid ? gls_term(dLdlp, d, sCst[12 + j]) : 0.0f;
        }
      }
      const float kl = dim_sum12(t);
      if (h == 0) {
        const double sv = valid ? (double)svf : 0.0, kv = valid ? (double)kl : 0.0;
        rd[0] = sv;
        rd[2 * 128] = kv;
        rd[3 * 128] = valid && clipped ? 1.0 : 0.0;
        rd[4 * 128] = (isfinite(sv) && isfinite(kv)) ? 0.0 : 1.0;
      }
    } else {
      const float V = __fadd_rn(head_out(d1, 0), b4c);
      float vvf = 0.0f;
      const float dV = valid ? ppo_dvalue(V, Vo, ret, L.vclip, L.vf_coef, L.invM, vvf) : 0.0f;
      dq[0] = dV;
#pragma unroll
      for (int j = 1; j < 12; ++j) dq[j] = 0.0f;
      if (h == 0) {
        const double vv = valid ? (double)vvf : 0.0;
        rec[12 * 128] = dV;
        rd[128] = vv;
        rd[4 * 128] = isfinite(vv) ? 0.0 : 1.0;
      }
    }
    {  // row r of DMU: part p = columns 16p .. 16p+15 (j < 12 used) = 16-B chunks 2p, 2p+1, swizzled by r & 7
      uint32_t w[3][8];
#pragma unroll
      for (int k = 0; k < 6; ++k) {
        uint16_t p0[3], p1[3];
        split3_bf16(dq[2 * k], p0);
        split3_bf16(dq[2 * k + 1], p1);
#pragma unroll
        for (int u = 0; u < 3; ++u) w[u][k] = (uint32_t)p0[u] | ((uint32_t)p1[u] << 16);
      }
      uint8_t* drow = sD + r * 128;
#pragma unroll
      for (int u = 0; u < 3; ++u) {
        w[u][6] = w[u][7] = 0u;
#pragma unroll
        for (int hf = 0; hf < 2; ++hf) {
          const int ch = 2 * u + hf;
          if ((ch >= 4) != (h == 1)) continue;
          *reinterpret_cast<uint4*>(drow + ((ch ^ (r & 7)) << 4)) =
              make_uint4(w[u][4 * hf], w[u][4 * hf + 1], w[u][4 * hf + 2], w[u][4 * hf + 3]);
        }
      }
    }
    fence_async_smem();
    tc_fence_before();
    __syncwarp();
    LOSS_STAMP(4);
    if (lane == 0) mbar_arrive(&lmma[3]);  // dmu staged: warp 3 issues the gradient MMAs
    // (4) meanwhile each warp sums its record columns over the tile's rows: every lane keeps its rows' partial sums
    // (rows l, l + 32, l + 64, l + 96 of every tile, in order) and the warp adds its lanes once at the end
    bar_epi();                             // every row's record is written
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int col = e + 8 * k;
      if (col < 25) {
        const float* cp = sRec + col * 128 + lane;
        xf[k] = xf[k] + cp[0];
        xf[k] = xf[k] + cp[32];
        xf[k] = xf[k] + cp[64];
        xf[k] = xf[k] + cp[96];
      }
    }
    if (e < 5) {
      const double* d0 = sRecD + e * 128 + lane;
      xd += d0[0];
      xd += d0[32];
      xd += d0[64];
      xd += d0[96];
    }
    LOSS_STAMP(5);
    mbar_wait(&lmma[1], mph);
    __syncwarp();
    tc_fence_after();
    LOSS_STAMP(6);
    // (5) dZ3 = dH3 * ELU'(H3) of columns 64h .. 64h+63 -> bf16 over the H3 values in A3 (the MMAs have read
    // them): sub-tile (q, h) of the dZ3 stores is A3 + h * 16 KB + q * 4 KB
    {
      uint32_t a32[2][32];
      tmem_ld32_nowait(tD2 + lrow + 64 * h, a32[0]);
      tmem_ld32_nowait(tD2 + lrow + 64 * h + 32, a32[1]);
      tmem_wait_ld();
#pragma unroll
      for (int ch = 0; ch < 8; ++ch) {
        uint4* p = reinterpret_cast<uint4*>(a3_chunk(ch));
        const uint4 hv4 = *p;
        const uint32_t hw[4] = {hv4.x, hv4.y, hv4.z, hv4.w};
        uint32_t w[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int c = 8 * ch + 2 * k;
          const float g0 = __uint_as_float(a32[c >> 5][c & 31]) * elu_grad_out(__uint_as_float(hw[k] << 16));
          const float g1 = __uint_as_float(a32[c >> 5][(c & 31) + 1]) * elu_grad_out(__uint_as_float(hw[k] & 0xFFFF0000u));
          const __nv_bfloat162 pk = __floats2bfloat162_rn(g0, g1);
          w[k] = *reinterpret_cast<const uint32_t*>(&pk);
        }
        *p = make_uint4(w[0], w[1], w[2], w[3]);
      }
    }
    fence_async_smem();
    __syncwarp();
    LOSS_STAMP(7);
    if (lane == 0 && tc.n0 + 64 * h < args.N) {
      tma_store_2d(&args.tmC[z], sA3 + h * 16384 + q * 4096, tc.n0 + 64 * h, tc.m0 + q * 32);
      bulk_commit();
    }
    tc_fence_before();  // this tile's TMEM reads (D1, D2) precede the next tile's MMAs into them
  }
  // the CTA's partial row (k_loss_heads layout: W4a [12][H2] | b4a [12] | W4c [H2] | b4c | logstd [12])
  float* out = L.part + (size_t)blockIdx.x * L.HP;
  if (h == 0) {  // dW4: TMEM lane c of the D3 accumulator (zero when the CTA had no tile)
    const int c = q * 32 + lane;
    uint32_t d3[48];
    tc_fence_after();
    tmem_ld32_nowait(tD3 + lrow, d3);
    tmem_ld16_nowait(tD3 + lrow + 32, d3 + 32);
    tmem_wait_ld();
    if (c < H2) {
#pragma unroll
      for (int j = 0; j < 12; ++j) out[j * H2 + c] = (local > 0 && z == 0) ? head_out(d3, j) : 0.0f;
      out[12 * H2 + 12 + c] = (local > 0 && z == 1) ? head_out(d3, 0) : 0.0f;
    }
  }
#pragma unroll
  for (int k = 0; k < 4; ++k) xf[k] = warp_sum(xf[k]);  // (fixed butterfly, the same order on every lane)
  xd = warp_sum_d(xd);
  if (lane == 0) {  // record column col -> b4a (0..11), b4c (12), log-std (13..24: d/dlogstd, entropy added later)
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int col = e + 8 * k;
      if (col < 12) out[12 * H2 + col] = xf[k];
      else if (col == 12) out[13 * H2 + 12] = xf[k];
      else if (col < 25) out[13 * H2 + 13 + (col - 13)] = xf[k];
    }
    if (e < 5) L.spart[(size_t)blockIdx.x * 8 + e] = xd;
  }
  if (L.dbg && et == 0) L.dbg[(size_t)blockIdx.x * 128 + 9] = loss_gtimer();  // (diagnostics: epilogue exit)
  if (lane == 0) bulk_wait_all();
  __syncwarp();
}

// PAIR: a cluster of 2 CTAs computes 256-row tiles with tcgen05.mma.cta_group::2 -- each CTA loads its own
// 128 rows of A and half of B (so each SM receives 2/3 of the operand bytes of a 128 x BN tile), both CTAs'
// loads complete on the leader's full barrier, the leader issues the MMAs and multicasts its commits, and the
// peer's epilogue warps release the accumulator stage on the leader's tempty barrier (remote arrive).
// WSKB > 0 (weight-stationary, EPI 0 / 2): the grid is split into column blocks ("slices": n_tiles x nz); a CTA
// serves one slice, loads that slice's B (<= WSKB k-blocks) into shared memory once and streams only A tiles of
// its rows -- B is not re-read from L2 for every tile, so the operand traffic per tile drops to the A tile.
template <int BN, bool A_MN, bool B_MN, int EPI, bool PAIR = false, int WSKB = 0>
__global__ void __launch_bounds__(GEMM_THREADS, 1) k_gemm_tc(const __grid_constant__ GemmArgs args) {
  using C = GemmCfg<BN, EPI, PAIR, WSKB>;
  static_assert(!PAIR || (EPI != 3 && !A_MN && BN >= 128), "pairs: forward / input-gradient GEMMs only");
  static_assert(!WSKB || (!PAIR && EPI != 3), "weight-stationary: single-CTA forward / input-gradient GEMMs");
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = sA + C::STAGES * C::A_BYTES;                       // ring B stages, or the resident slice (WSKB)
  uint8_t* sEpi = sB + (WSKB ? C::BRES : C::STAGES * C::B_BYTES);
  uint8_t* sOnes = sEpi + EPI_WARPS * C::EPI_NBUF * C::EPI_BUF;
  float* sBias = reinterpret_cast<float*>(sOnes + C::ONES_BYTES);
  uint8_t* sLoss = sOnes + C::ONES_BYTES + C::BIAS_BYTES;  // EPI 4
  uint64_t* full = reinterpret_cast<uint64_t*>(sLoss + C::LOSS_BYTES);
  uint64_t* empty = full + C::STAGES;
  uint64_t* tfull = empty + C::STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* bfull = tempty + 2;  // WSKB: the resident B slice has landed
  uint64_t* lmma = bfull + 1;    // EPI 4: [0] head MMA done, [1] gradient MMAs done, [2] H3 staged, [3] dmu staged
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(lmma + 4);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  pdl_trigger();
  if (args.M_dev) pdl_wait();  // the device-side row count is a predecessor's output
  const int M = args.M_dev ? *args.M_dev : args.M;
  const uint32_t rank = PAIR ? cluster_ctarank() : 0u;
  // tile loop over (pair) tiles: a pair tile covers 128-row tiles 2u and 2u+1 of the same column block
  const int m_tiles = PAIR ? (args.m_tiles + 1) / 2 : args.m_tiles;
  const int cid = PAIR ? (int)(blockIdx.x >> 1) : (int)blockIdx.x;
  const int ncl = PAIR ? (int)(gridDim.x >> 1) : (int)gridDim.x;
  const int total = args.nz * m_tiles * args.n_tiles * args.n_splits;
  auto tile_of = [&](int t) {  // (pair) tile -> this CTA's coordinates; skip when the (pair) tile has no rows
    TileCoord c = decode(args, t, m_tiles, BN);
    if (PAIR) c.m0 = 2 * c.m0 + (int)rank * 128;
    return c;
  };
  // weight-stationary schedule: slice = cid % nsl (fixed column block of B), row tiles mi, mi + cps, ...; with
  // ws_split and two slices (the loss epilogue: actor rows cost more than critic rows) CTAs [0, ws_split) serve
  // slice 0 and the rest slice 1, each taking every (slice CTA count)-th row tile
  const int nsl = args.n_tiles * args.nz;
  const int cps = WSKB ? (int)gridDim.x / nsl : 1;
  const bool split2 = WSKB && args.ws_split > 0 && nsl == 2;
  const int wslice = WSKB ? (split2 ? (cid < args.ws_split ? 0 : 1) : cid % nsl) : 0;
  const int wfirst = split2 ? (wslice ? cid - args.ws_split : cid) : cid / nsl;
  const int wstride = split2 ? (wslice ? (int)gridDim.x - args.ws_split : args.ws_split) : cps;
  // the it-th tile of this CTA (false when there is none)
  auto tile_at = [&](int it, TileCoord& c) -> bool {
    if (WSKB) {
      const int m = wfirst + it * wstride;
      if (m >= m_tiles) return false;
      c.z = wslice / args.n_tiles; c.ntile = wslice - c.z * args.n_tiles; c.n0 = c.ntile * BN; c.split = 0;
      c.m0 = m * 128;
      return true;
    }
    const int t = cid + it * ncl;
    if (t >= total) return false;
    c = tile_of(t);
    return true;
  };
  auto skip = [&](const TileCoord& c) { return (PAIR ? c.m0 - (int)rank * 128 : c.m0) >= M; };
  bool has_tiles = true;
  if (!PAIR) {  // CTA-uniform early exit when none of this CTA's tiles has rows (device-sized M, e.g. no time-outs)
    bool any = false;
    TileCoord c0;
    for (int it = 0; !any && tile_at(it, c0); ++it) any = !skip(c0);
    if (!any && EPI != 4) return;  // (the loss epilogue still writes this CTA's -- zero -- partial row)
    has_tiles = any;
  }

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int s = 0; s < 2; ++s) { mbar_init(&tfull[s], 1); mbar_init(&tempty[s], (PAIR ? 2 : 1) * EPI_WARPS); }
    mbar_init(bfull, 1);
    mbar_init(&lmma[0], 1);
    mbar_init(&lmma[1], 1);
    mbar_init(&lmma[2], EPI_WARPS);
    mbar_init(&lmma[3], EPI_WARPS);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (EPI == 3) {  // 16 x 64 bf16 ones (any swizzle of a constant tile is the same tile)
    uint32_t* o = reinterpret_cast<uint32_t*>(sOnes);
    for (int k = threadIdx.x; k < C::ONES_BYTES / 4; k += blockDim.x) o[k] = 0x3F803F80u;
    fence_async_smem();
  }
  if (warp == 2) {
    if (PAIR) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                   "n"(C::TMEM_COLS));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                   "n"(C::TMEM_COLS));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
  }
  tc_fence_before();
  if (PAIR) cluster_barrier();  // the peer's barriers exist before any cross-CTA signal
  else __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_wait();  // the prologue above overlapped the preceding kernel; its outputs are read from here on

  if (warp == 0) {
    // ---------------------------------------------------------------- TMA producer
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      if (WSKB && has_tiles) {  // the slice's B column block, once (kb_total <= WSKB k-blocks, checked by the host)
        TileCoord c0;
        tile_at(0, c0);
        const CUtensorMap* tmB = &args.tmB[c0.z];
        mbar_expect_tx(bfull, args.kb_total * C::B_BYTES);
        for (int kb = 0; kb < args.kb_total; ++kb) {
          uint8_t* b = sB + kb * C::B_BYTES;
          if (!B_MN) {
            tma_load_2d(tmB, bfull, b, kb * C::BK, c0.n0);
          } else {
#pragma unroll
            for (int i = 0; i < BN / 64; ++i) tma_load_2d(tmB, bfull, b + i * 8192, c0.n0 + 64 * i, kb * C::BK);
          }
        }
      }
      TileCoord tc;
      for (int it = 0; tile_at(it, tc); ++it) {
        if (skip(tc)) continue;
        const CUtensorMap* tmA = &args.tmA[tc.z];
        const CUtensorMap* tmB = &args.tmB[tc.z];
        const int kb0 = tc.split * args.kb_per_split;
        const int nkb = min(args.kb_per_split, args.kb_total - kb0);
        for (int kb = 0; kb < nkb; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1u);
          const int k0 = (kb0 + kb) * C::BK;
          uint8_t* a = sA + stage * C::A_BYTES;
          uint8_t* b = sB + stage * C::B_BYTES;
          if (WSKB) {
            mbar_expect_tx(&full[stage], C::A_BYTES);
            if (!A_MN) {
              tma_load_2d(tmA, &full[stage], a, k0, tc.m0);
            } else {
              tma_load_2d(tmA, &full[stage], a, tc.m0, k0);
              tma_load_2d(tmA, &full[stage], a + 8192, tc.m0 + 64, k0);
            }
            if (++stage == C::STAGES) { stage = 0; phase ^= 1u; }
            continue;
          }
          if (PAIR) {
            if (rank == 0) mbar_expect_tx(&full[stage], 2 * (C::A_BYTES + C::B_BYTES));
            const uint32_t fb = mapa_shared(smem_u32(&full[stage]), 0);
            tma_load_2d_pair(tmA, fb, a, k0, tc.m0);
            const int nh = tc.n0 + (int)rank * (BN / 2);
            if (!B_MN) {
              tma_load_2d_pair(&args.tmBp[tc.z], fb, b, k0, nh);
            } else {
#pragma unroll
              for (int i = 0; i < BN / 128; ++i) tma_load_2d_pair(tmB, fb, b + i * 8192, nh + 64 * i, k0);
            }
            if (++stage == C::STAGES) { stage = 0; phase ^= 1u; }
            continue;
          }
          if (args.probe & 2) { mbar_arrive(&full[stage]); if (++stage == C::STAGES) { stage = 0; phase ^= 1u; } continue; }
          mbar_expect_tx(&full[stage], C::A_BYTES + C::B_BYTES);
          if (!A_MN) {
            tma_load_2d(tmA, &full[stage], a, k0, tc.m0);
          } else {
            tma_load_2d(tmA, &full[stage], a, tc.m0, k0);
            tma_load_2d(tmA, &full[stage], a + 8192, tc.m0 + 64, k0);
          }
          if (!B_MN) {
            tma_load_2d(tmB, &full[stage], b, k0, tc.n0);
          } else {
#pragma unroll
            for (int i = 0; i < BN / 64; ++i) tma_load_2d(tmB, &full[stage], b + i * 8192, tc.n0 + 64 * i, k0);
          }
          if (++stage == C::STAGES) { stage = 0; phase ^= 1u; }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ---------------------------------------------------------------- MMA issuer
    if (lane == 0 && rank == 0) {
      constexpr uint32_t idesc = idesc_bf16(PAIR ? 256 : 128, BN, A_MN, B_MN);
      constexpr uint32_t idesc_ones = idesc_bf16(128, 16, A_MN, false);
      const uint32_t a_lbo = A_MN ? 8192u : 0u, b_lbo = B_MN ? 8192u : 0u;
      const uint32_t a_step = A_MN ? 2048u : 32u, b_step = B_MN ? 2048u : 32u;  // bytes per UMMA_K = 16
      int stage = 0;
      uint32_t phase = 0;
      int local = 0;
      if (WSKB && has_tiles) {
        mbar_wait(bfull, 0);
        tc_fence_after();
      }
      TileCoord tc;
      for (int it = 0; tile_at(it, tc); ++it) {
        if (skip(tc)) continue;
        const int acc = local % C::ACC_STAGES;
        const uint32_t aph = (uint32_t)((local / C::ACC_STAGES) & 1);
        ++local;
        mbar_wait(&tempty[acc], aph ^ 1u);
        tc_fence_after();
        const uint32_t tacc = tmem + acc * C::ACC_COLS;
        const bool bias_col = (EPI == 3) && args.bias_col && tc.ntile == 0;
        const int kb0 = tc.split * args.kb_per_split;
        const int nkb = min(args.kb_per_split, args.kb_total - kb0);
        for (int kb = 0; kb < nkb; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          if (args.probe & 1) { mbar_arrive(&empty[stage]); if (++stage == C::STAGES) { stage = 0; phase ^= 1u; } continue; }
          const uint32_t a0 = smem_u32(sA + stage * C::A_BYTES);
          const uint32_t b0 = smem_u32(sB + (WSKB ? kb0 + kb : stage) * C::B_BYTES);
#pragma unroll
          for (int k = 0; k < C::BK / 16; ++k) {
            const uint64_t ad = sdesc(a0 + k * a_step, a_lbo, 1024u);
            const uint64_t bd = sdesc(b0 + k * b_step, b_lbo, 1024u);
            if (PAIR) {
              tc_mma_pair(tacc, ad, bd, idesc, (kb > 0 || k > 0) ? 1u : 0u);
            } else {
              tc_mma(tacc, ad, bd, idesc, (kb > 0 || k > 0) ? 1u : 0u);
              if (bias_col) {
                const uint64_t od = sdesc(smem_u32(sOnes) + k * 32u, 0u, 1024u);
                tc_mma(tacc + BN, ad, od, idesc_ones, (kb > 0 || k > 0) ? 1u : 0u);
              }
            }
          }
          if (PAIR) tc_commit_pair(&empty[stage]);
          else tc_commit(&empty[stage]);
          if (++stage == C::STAGES) { stage = 0; phase ^= 1u; }
        }
        if (PAIR) tc_commit_pair(&tfull[acc]);
        else tc_commit(&tfull[acc]);
      }
    }
    __syncwarp();
  } else if (warp == 3 && EPI == 4) {
    // ---------------------------------------------------------------- loss epilogue's MMA issuer
    if (lane == 0) loss_mma<C>(tile_at, skip, tmem, lmma, sLoss);
    __syncwarp();
  } else if (warp >= 4 && EPI == 4) {
    // ---------------------------------------------------------------- loss epilogue
    loss_epilogue<C>(args, M, tile_at, skip, tmem, tfull, tempty, lmma, sLoss, wslice);
  } else if (warp >= 4) {
    // ---------------------------------------------------------------- epilogue
    const int e = warp - 4, q = e & 3, h = e >> 2;
    uint8_t* mybuf = sEpi + e * C::EPI_NBUF * C::EPI_BUF;
    float* mybias = sBias + e * 128;
    constexpr int WCOLS = BN >= 128 ? BN / 2 : BN;  // columns handled by this warp
    const bool active = BN >= 128 || h == 0;
    int local = 0, nst = 0;
    TileCoord tc;
    for (int it = 0; tile_at(it, tc); ++it) {
      if (skip(tc)) continue;
      const int acc = local % C::ACC_STAGES;
      const uint32_t aph = (uint32_t)((local / C::ACC_STAGES) & 1);
      ++local;
      const int row = tc.m0 + q * 32 + lane;
      // work that does not depend on the accumulator, done while the MMA runs
      uint32_t av[32];
      if (EPI == 0 && active && (!WSKB || local == 1)) {  // (weight-stationary: one column block per CTA, once)
        const float* bias = args.bias[tc.z];
        for (int i = lane; i < WCOLS; i += 32) {
          const int n = tc.n0 + h * WCOLS + i;
          mybias[i] = n < args.N ? __ldg(bias + n) : 0.0f;
        }
        __syncwarp();
      }
      constexpr bool AUX_STAGED = EPI == 2 && C::EPI_NBUF == 2;
      if (AUX_STAGED && active) {  // this tile's first chunk of H into the staging buffer it will be stored from
        if (lane == 0) bulk_wait_read1();  // that buffer's previous store (two chunks ago) has been read out
        __syncwarp();
        aux_issue(mybuf + (nst & 1) * C::EPI_BUF, args.aux[tc.z], args.ld_aux, tc.m0 + q * 32, M, tc.n0 + h * WCOLS,
                  args.N, lane);
      }
      if (EPI == 2 && !AUX_STAGED && active) {
        const int nb = tc.n0 + h * WCOLS;
        const uint4* a4 = reinterpret_cast<const uint4*>(args.aux[tc.z] + (size_t)row * args.ld_aux + nb);
        if (row < M && nb + 64 <= args.N) {  // whole 64-column chunk in range (the common case)
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const uint4 u = __ldg(a4 + j);
            av[4 * j] = u.x; av[4 * j + 1] = u.y; av[4 * j + 2] = u.z; av[4 * j + 3] = u.w;
          }
        } else {
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            uint4 u = (row < M && nb + 8 * j < args.N) ? a4[j] : make_uint4(0, 0, 0, 0);
            av[4 * j] = u.x; av[4 * j + 1] = u.y; av[4 * j + 2] = u.z; av[4 * j + 3] = u.w;
          }
        }
      }
      mbar_wait(&tfull[acc], aph);
      __syncwarp();
      tc_fence_after();
      const uint32_t tbase = tmem + acc * C::ACC_COLS + ((uint32_t)(q * 32) << 16);
      if (active && !(args.probe & 4)) {
        if (EPI == 3) {
          // fp32 split-K partial: 32-column chunks
          const int prow = (tc.z * args.n_splits + tc.split) * args.part_rows + tc.m0 + q * 32;
#pragma unroll 1
          for (int c = h * WCOLS; c < (h + 1) * WCOLS; c += 32) {
            uint32_t r[32];
            tmem_ld32_nowait(tbase + c, r);
            tmem_wait_ld();
            uint8_t* buf = mybuf;
            if (lane == 0) bulk_wait_all();
            __syncwarp();
            stage_row(buf, lane, r);
            fence_async_smem();
            __syncwarp();
            if (lane == 0) { tma_store_2d(&args.tmC[0], buf, tc.n0 + c, prow); bulk_commit(); }
            ++nst;
          }
          if (args.bias_col && tc.ntile == 0 && h == 0) {
            uint32_t r[32];
            tmem_ld32_nowait(tbase + BN, r);
            tmem_wait_ld();
            if (row < M)
              args.part[(size_t)(prow + lane) * args.part_ld + args.part_bias_col] = __uint_as_float(r[0]);
          }
        } else {
          // bf16 outputs: 64-column chunks (two TMEM loads)
#pragma unroll 1
          for (int c = h * WCOLS; c < (h + 1) * WCOLS; c += 64) {
            uint32_t r0[32], r1[32];
            tmem_ld32_nowait(tbase + c, r0);
            tmem_ld32_nowait(tbase + c + 32, r1);
            tmem_wait_ld();
            uint32_t pk[32];
            const int nb = tc.n0 + c;
            if (EPI == 0) {
              const float* bb = mybias + (c - h * WCOLS);
#pragma unroll
              for (int k = 0; k < 64; k += 4) {
                const uint32_t* rr = k < 32 ? r0 : r1;
                const int kk = k & 31;
                const float4 b4 = lds4(bb + k);
                __nv_bfloat162 o0 = __floats2bfloat162_rn(elu_fast(__uint_as_float(rr[kk]) + b4.x),
                                                          elu_fast(__uint_as_float(rr[kk + 1]) + b4.y));
                __nv_bfloat162 o1 = __floats2bfloat162_rn(elu_fast(__uint_as_float(rr[kk + 2]) + b4.z),
                                                          elu_fast(__uint_as_float(rr[kk + 3]) + b4.w));
                pk[k / 2] = *reinterpret_cast<uint32_t*>(&o0);
                pk[k / 2 + 1] = *reinterpret_cast<uint32_t*>(&o1);
              }
            } else {
              if (AUX_STAGED) {
                aux_read(mybuf + (nst & 1) * C::EPI_BUF, av, lane);
                if (c + 64 < (h + 1) * WCOLS) {  // the next chunk's H into the other buffer (its store is done)
                  if (lane == 0) bulk_wait_read0();
                  __syncwarp();
                  aux_issue(mybuf + ((nst + 1) & 1) * C::EPI_BUF, args.aux[tc.z], args.ld_aux, tc.m0 + q * 32, M,
                            nb + 64, args.N, lane);
                }
              }
#pragma unroll
              for (int k = 0; k < 64; k += 2) {
                const uint32_t* rr = k < 32 ? r0 : r1;
                const int kk = k & 31;
                const uint32_t w = av[k / 2];
                // ELU'(x) from the saved output h = ELU(x) > -1: h > 0 ? 1 : h + 1 == min(h + 1, 1) (h + 1 exact)
                const float h0 = __uint_as_float(w << 16), h1 = __uint_as_float(w & 0xFFFF0000u);
                const float g0 = __uint_as_float(rr[kk]) * fminf(h0 + 1.0f, 1.0f);
                const float g1 = __uint_as_float(rr[kk + 1]) * fminf(h1 + 1.0f, 1.0f);
                __nv_bfloat162 o = __floats2bfloat162_rn(g0, g1);
                pk[k / 2] = *reinterpret_cast<uint32_t*>(&o);
              }
            }
            uint8_t* buf = mybuf + (C::EPI_NBUF == 2 ? (nst & 1) * C::EPI_BUF : 0);
            if (!AUX_STAGED) {  // (staged H: the buffer was freed before its H was loaded, and H is consumed)
              if (lane == 0) {
                if (C::EPI_NBUF == 2) bulk_wait_read1();
                else bulk_wait_read0();
              }
            }
            __syncwarp();
            stage_row(buf, lane, pk);
            fence_async_smem();
            __syncwarp();
            if (lane == 0) { tma_store_2d(&args.tmC[tc.z], buf, nb, tc.m0 + q * 32); bulk_commit(); }
            ++nst;
          }
        }
      }
      // release the accumulator stage to the MMA warp (the leader's barrier for a pair)
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (PAIR && rank != 0) {
          const uint32_t rb = mapa_shared(smem_u32(&tempty[acc]), 0);
          asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(rb) : "memory");
        } else {
          mbar_arrive(&tempty[acc]);
        }
      }
    }
    if (lane == 0) bulk_wait_all();
    __syncwarp();
  }
  tc_fence_before();
  if (PAIR) {
    cluster_barrier();  // both CTAs are done with the pair's TMEM
    if (warp == 2) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(C::TMEM_COLS));
  } else {
    __syncthreads();
    if (warp == 2) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(C::TMEM_COLS));
  }
}

// ------------------------------------------------------------------ dW: one-wave split-K with an L2 reduction
// dW = dZ^T X (+ db = colsum dZ via the ones MMA) for 128 x BN output tiles. Grid (S, tiles), one wave
// (cooperative launch: every CTA is resident). CTA (s, tile) contracts batch rows of k-blocks
// [s*kb_per_split, ...), copies its fp32 accumulator (+ bias column) TMEM -> smem -> an L2-resident partial
// buffer with coalesced 16-B stores, and arrives at a grid barrier. All CTAs then share the reduction: each
// output element is the sum of its S partials in split order 0..S-1 (deterministic), written straight into
// the canonical gradient vector. (DSMEM would move the same bytes at ~20 B/clk per SM; L2 is several times
// faster per SM, and the reduction is spread over the whole grid.)
__device__ __forceinline__ uint32_t ld_acquire_gpu(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define DW_STAMP(k)                                                                                         \
  do {                                                                                                      \
    if (out.dbg && threadIdx.x == 0) out.dbg[((size_t)blockIdx.y * gridDim.x + blockIdx.x) * 8 + (k)] = gtimer(); \
  } while (0)

// One reduced output item (tile t, row i, float4 column group g; g == BN/4 is the bias column) -> its
// canonical gradient destination, or !ok when it lies outside the real output (ragged rows / columns).
struct DwItem {
  float* dst;
  int nv;     // valid columns of the group (1..4)
  bool isb;   // bias item
  bool ok;
};
template <int BN>
__device__ __forceinline__ DwItem dw_item(const GemmArgs& args, const DwOut& out, int t, int i, int g) {
  DwItem d;
  d.ok = false; d.dst = nullptr; d.nv = 0; d.isb = false;
  const TileCoord c2 = decode(args, t, args.m_tiles, BN);
  if (i >= args.M - c2.m0) return d;
  const int cv = min(BN, out.cols - c2.n0);
  d.isb = g == BN / 4;
  if (d.isb ? c2.ntile != 0 : 4 * g >= cv) return d;
  int rr = c2.m0 + i;
  bool second = c2.z == 1;
  if (out.row_split > 0 && rr >= out.row_split) { second = true; rr -= out.row_split; }
  if (d.isb) {
    d.dst = out.grad + (second ? out.b_off[1] : out.b_off[0]) + rr;
    d.nv = 1;
  } else {
    d.dst = out.grad + (second ? out.w_off[1] : out.w_off[0]) + (long long)rr * out.cols + c2.n0 + 4 * g;
    d.nv = min(4, cv - 4 * g);
  }
  d.ok = true;
  return d;
}
__device__ __forceinline__ bool dw_emit(const DwItem& d, const float4& v) {
  if (d.isb) {
    d.dst[0] = v.x;
    return isfinite(v.x);
  }
  d.dst[0] = v.x;
  if (d.nv > 1) d.dst[1] = v.y;
  if (d.nv > 2) d.dst[2] = v.z;
  if (d.nv > 3) d.dst[3] = v.w;
  return isfinite(v.x) && isfinite(v.y) && isfinite(v.z) && isfinite(v.w);
}

// The split-K tail shared by the dW kernels. S == 1: the CTA holds its whole tile, which it writes straight
// from shared memory into the canonical gradient (no partial, no barrier). S > 1: the CTA's fp32 partial
// (128 rows x RLD, staged in smem `red`) -> the L2 buffer [tile][split][128][RLD] with one bulk copy; a grid
// barrier (cooperative launch: all CTAs resident; the counter only grows, the target is the next multiple of
// the grid size, so no reset is needed between launches); then the whole grid reduces: items (tile, row,
// column group) are split evenly over the CTAs and each sums its S partials in split order 0..S-1
// (deterministic) into the canonical gradient. Small S keeps several items' partial loads in flight per
// thread (the reduction is load-latency bound when the grid is small).
template <int BN>
__device__ __forceinline__ void dw_partial_barrier_reduce(const GemmArgs& args, const DwOut& out, const float* red,
                                                          int tile, int split, int S, int ntiles) {
  constexpr int RLD = BN + 20;
  constexpr int PER = BN / 4 + 1;  // float4 column groups + the bias group
  bool bad = false;
  if (S == 1) {
    for (int it = threadIdx.x; it < 128 * PER; it += blockDim.x) {
      const int i = it / PER, g = it - i * PER;
      const DwItem d = dw_item<BN>(args, out, tile, i, g);
      if (!d.ok) continue;
      bad |= !dw_emit(d, *reinterpret_cast<const float4*>(red + i * RLD + 4 * g));
    }
    if (bad) atomicAdd(out.payload + 4, 1.0f);
    DW_STAMP(6);
    return;
  }
  // partial -> L2 buffer [tile][split][128][RLD]: every thread copies 16-B chunks (coalesced, L2-only stores).
  // (One bulk async copy of the whole 128 x RLD tile by one thread streamed at ~25 B/clk per SM: 5-6 us of a
  // ~23 us launch; the all-thread copy runs near the SM's store rate.)
  float* part_me = out.part + ((size_t)tile * S + split) * 128 * RLD;
  __syncthreads();
  {
    const float4* src = reinterpret_cast<const float4*>(red);
    float4* dst = reinterpret_cast<float4*>(part_me);
    constexpr int NV = 128 * RLD / 4;
    const float bound = out.part_bound;
#pragma unroll 4
    for (int k = threadIdx.x; k < NV; k += blockDim.x) {
      const float4 w = src[k];
      __stcg(dst + k, w);
      // partial_only: the consumer (Adam) cannot see the reduced gradient before it applies the step, so the
      // non-finite rule is taken on the partials (|x| < FLT_MAX / S keeps the S-term sum finite)
      if (out.partial_only)
        bad |= !(fabsf(w.x) < bound && fabsf(w.y) < bound && fabsf(w.z) < bound && fabsf(w.w) < bound);
    }
  }
  if (out.partial_only) {
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicAdd(out.payload + 4, 1.0f);
    DW_STAMP(6);
    return;
  }
  __threadfence();
  __syncthreads();
  DW_STAMP(4);
  if (threadIdx.x == 0) {
    // generation barrier: cnt[0] counts arrivals and returns to 0 at every release, cnt[1] is the generation.
    // The generation is read before arriving (it cannot advance before this CTA arrives); the last CTA resets
    // the count and then publishes the next generation. No modular arithmetic on a growing counter, so
    // neither a counter wrap nor a grid size that changes between launches (another plan, a restored
    // checkpoint) can leave a CTA waiting for a target that is never reached.
    const uint32_t n = gridDim.x * gridDim.y * gridDim.z;
    uint32_t* cnt = reinterpret_cast<uint32_t*>(out.cnt);
    const uint32_t gen = ld_acquire_gpu(cnt + 1);
    const uint32_t old = atomicAdd(cnt, 1u);
    if (old == n - 1u) {
      cnt[0] = 0u;
      __threadfence();
      atomicAdd(cnt + 1, 1u);
    } else {
      while (ld_acquire_gpu(cnt + 1) == gen) __nanosleep(64);
    }
  }
  __syncthreads();
  DW_STAMP(5);

  const long long n_items = (long long)ntiles * 128 * PER;
  const int n_cta = gridDim.x * gridDim.y, cid = blockIdx.y * gridDim.x + blockIdx.x;
  const long long per_cta = (n_items + n_cta - 1) / n_cta;
  const long long lo = (long long)cid * per_cta, hi = min(n_items, lo + per_cta);
  auto src_of = [&](long long it) {
    const int t = (int)(it / (128 * PER));
    const int rem = (int)(it - (long long)t * 128 * PER);
    const int i = rem / PER, g = rem - i * PER;
    return out.part + ((size_t)t * S * 128 + i) * RLD + 4 * g;
  };
  auto item_of = [&](long long it) {
    const int t = (int)(it / (128 * PER));
    const int rem = (int)(it - (long long)t * 128 * PER);
    const int i = rem / PER, g = rem - i * PER;
    return dw_item<BN>(args, out, t, i, g);
  };
  if (S <= 6) {
    // 4 items per thread per pass, all 4*S partial loads in flight, each item summed in split order
    constexpr int J = 4;
    for (long long base = lo + threadIdx.x; base < hi; base += (long long)J * blockDim.x) {
      float4 w[J][6];
      DwItem d[J];
#pragma unroll
      for (int j = 0; j < J; ++j) {
        const long long it = base + (long long)j * blockDim.x;
        d[j].ok = false;
        if (it < hi) d[j] = item_of(it);
        if (d[j].ok) {
          const float* src = src_of(it);
#pragma unroll
          for (int q = 0; q < 6; ++q)
            if (q < S) w[j][q] = __ldcg(reinterpret_cast<const float4*>(src + (size_t)q * 128 * RLD));
        }
      }
#pragma unroll
      for (int j = 0; j < J; ++j) {
        if (!d[j].ok) continue;
        float4 v = w[j][0];
#pragma unroll
        for (int q = 1; q < 6; ++q)
          if (q < S) { v.x = v.x + w[j][q].x; v.y = v.y + w[j][q].y; v.z = v.z + w[j][q].z; v.w = v.w + w[j][q].w; }
        bad |= !dw_emit(d[j], v);
      }
    }
  } else {
    for (long long it = lo + threadIdx.x; it < hi; it += blockDim.x) {
      const DwItem d = item_of(it);
      if (!d.ok) continue;
      const float* src = src_of(it);
      // all S partials of the item in flight at once (S <= 24 in one pass), then summed in split order
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int s0 = 0; s0 < S; s0 += 24) {
        float4 w[24];
#pragma unroll
        for (int q = 0; q < 24; ++q)
          if (s0 + q < S) w[q] = __ldcg(reinterpret_cast<const float4*>(src + (size_t)(s0 + q) * 128 * RLD));
#pragma unroll
        for (int q = 0; q < 24; ++q)
          if (s0 + q < S) {
            if (s0 + q == 0) v = w[0];
            else { v.x = v.x + w[q].x; v.y = v.y + w[q].y; v.z = v.z + w[q].z; v.w = v.w + w[q].w; }
          }
      }
      bad |= !dw_emit(d, v);
    }
  }
  if (bad) atomicAdd(out.payload + 4, 1.0f);
  DW_STAMP(6);
}

template <int BN>
struct DwCfg {  // k_gemm_dw: no epilogue staging buffers, the operand ring is reused for the reduction
  static constexpr int BM = 128, BK = 64;
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int B_BYTES = BN * BK * 2;
  static constexpr int ONES_BYTES = 16 * 128;
  static constexpr int EPI_WARPS_ = EPI_WARPS;
  static constexpr int EPI_NBUF = 0, EPI_BUF = 0, BIAS_BYTES = 0;
  static constexpr int FIXED = 1024 + ONES_BYTES + 512;
  static constexpr int STAGES_FIT = (232448 - FIXED) / (A_BYTES + B_BYTES);
  static constexpr int STAGES = STAGES_FIT > 8 ? 8 : STAGES_FIT;
  static constexpr int ACC_COLS = ((BN + 16) + 31) / 32 * 32;
  static constexpr int TMEM_COLS = ACC_COLS <= 32 ? 32 : ACC_COLS <= 64 ? 64 : ACC_COLS <= 128 ? 128 : ACC_COLS <= 256 ? 256 : 512;
  static constexpr int SMEM = FIXED + STAGES * (A_BYTES + B_BYTES);
};

template <int BN, bool KMAJ = false>
__global__ void __launch_bounds__(GEMM_THREADS, 1) k_gemm_dw(const __grid_constant__ GemmArgs args, const DwOut out) {
  using C = DwCfg<BN>;
  constexpr int RLD = BN + 20;  // fp32 row stride of the reduction buffer (16-B rows, conflict-free float4 writes)
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = sA + C::STAGES * C::A_BYTES;
  float* red = reinterpret_cast<float*>(smem);  // reuses the operand ring after the last MMA
  uint8_t* sOnes = sB + C::STAGES * C::B_BYTES + EPI_WARPS * C::EPI_NBUF * C::EPI_BUF;
  uint64_t* full = reinterpret_cast<uint64_t*>(sOnes + C::ONES_BYTES + C::BIAS_BYTES);
  uint64_t* empty = full + C::STAGES;
  uint64_t* tfull = empty + C::STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tfull + 2);
  static_assert(128 * RLD * 4 <= C::STAGES * (C::A_BYTES + C::B_BYTES), "reduction buffer must fit the ring");

  DW_STAMP(0);
  pdl_trigger();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int S = gridDim.x;  // splits per tile
  const int tile = blockIdx.y;
  const uint32_t split = blockIdx.x;
  const TileCoord tc = decode(args, tile, args.m_tiles, BN);
  const bool bias_col = tc.ntile == 0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < C::STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    mbar_init(&tfull[0], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  {
    uint32_t* o = reinterpret_cast<uint32_t*>(sOnes);
    for (int k = threadIdx.x; k < C::ONES_BYTES / 4; k += blockDim.x) o[k] = 0x3F803F80u;
    fence_async_smem();
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "n"(C::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  DW_STAMP(1);
  pdl_wait();  // (partial_only launches use PDL: the prologue above overlapped the predecessor)
  const int kb0 = (int)split * args.kb_per_split;
  const int nkb = max(0, min(args.kb_per_split, args.kb_total - kb0));
  const CUtensorMap* tmA = &args.tmA[tc.z];
  const CUtensorMap* tmB = &args.tmB[tc.z];

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int kb = 0; kb < nkb; ++kb) {
        mbar_wait(&empty[stage], phase ^ 1u);
        const int k0 = (kb0 + kb) * C::BK;
        uint8_t* a = sA + stage * C::A_BYTES;
        uint8_t* b = sB + stage * C::B_BYTES;
        if (args.probe & 2) { mbar_arrive(&full[stage]); if (++stage == C::STAGES) { stage = 0; phase ^= 1u; } continue; }
        mbar_expect_tx(&full[stage], C::A_BYTES + C::B_BYTES);
        if (KMAJ) {  // operands stored transposed ([out][batch], [in][batch]): one K-major box each
          tma_load_2d(tmA, &full[stage], a, k0, tc.m0);
          tma_load_2d(tmB, &full[stage], b, k0, tc.n0);
        } else {
          tma_load_2d(tmA, &full[stage], a, tc.m0, k0);
          tma_load_2d(tmA, &full[stage], a + 8192, tc.m0 + 64, k0);
#pragma unroll
          for (int i = 0; i < BN / 64; ++i) tma_load_2d(tmB, &full[stage], b + i * 8192, tc.n0 + 64 * i, k0);
        }
        if (++stage == C::STAGES) { stage = 0; phase ^= 1u; }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = idesc_bf16(128, BN, !KMAJ, !KMAJ);
      constexpr uint32_t idesc_ones = idesc_bf16(128, 16, !KMAJ, false);
      constexpr uint32_t lbo = KMAJ ? 0u : 8192u, kstep = KMAJ ? 32u : 2048u;
      int stage = 0;
      uint32_t phase = 0;
      for (int kb = 0; kb < nkb; ++kb) {
        mbar_wait(&full[stage], phase);
        tc_fence_after();
        if (args.probe & 1) { mbar_arrive(&empty[stage]); if (++stage == C::STAGES) { stage = 0; phase ^= 1u; } continue; }
        const uint32_t a0 = smem_u32(sA + stage * C::A_BYTES), b0 = smem_u32(sB + stage * C::B_BYTES);
#pragma unroll
        for (int k = 0; k < C::BK / 16; ++k) {
          const uint64_t ad = sdesc(a0 + k * kstep, lbo, 1024u);
          const uint64_t bd = sdesc(b0 + k * kstep, lbo, 1024u);
          tc_mma(tmem, ad, bd, idesc, (kb > 0 || k > 0) ? 1u : 0u);
          if (bias_col) {
            const uint64_t od = sdesc(smem_u32(sOnes) + k * 32u, 0u, 1024u);
            tc_mma(tmem + BN, ad, od, idesc_ones, (kb > 0 || k > 0) ? 1u : 0u);
          }
        }
        tc_commit(&empty[stage]);
        if (++stage == C::STAGES) { stage = 0; phase ^= 1u; }
      }
      tc_commit(&tfull[0]);
    }
    __syncwarp();
  } else if (warp >= 4) {
    // TMEM -> smem partial (an empty split contributes zeros)
    const int e = warp - 4, q = e & 3, h = e >> 2;
    const int row = q * 32 + lane;
    if (nkb > 0) {
      mbar_wait(&tfull[0], 0);
      __syncwarp();
      tc_fence_after();
    }
    if (out.dbg && threadIdx.x == 128) out.dbg[((size_t)blockIdx.y * gridDim.x + blockIdx.x) * 8 + 2] = gtimer();
    const uint32_t tbase = tmem + ((uint32_t)(q * 32) << 16);
    for (int c = h * (BN / 2); c < (h + 1) * (BN / 2); c += 32) {
      uint32_t r[32];
      if (nkb > 0) {
        tmem_ld32_nowait(tbase + c, r);
        tmem_wait_ld();
      } else {
#pragma unroll
        for (int k = 0; k < 32; ++k) r[k] = 0u;
      }
#pragma unroll
      for (int k = 0; k < 32; k += 4)
        *reinterpret_cast<float4*>(red + row * RLD + c + k) =
            make_float4(__uint_as_float(r[k]), __uint_as_float(r[k + 1]), __uint_as_float(r[k + 2]), __uint_as_float(r[k + 3]));
    }
    if (h == 0) {
      uint32_t r[32];
      if (nkb > 0 && bias_col) {
        tmem_ld32_nowait(tbase + BN, r);
        tmem_wait_ld();
      }
      *reinterpret_cast<float4*>(red + row * RLD + BN) =
          make_float4((nkb > 0 && bias_col) ? __uint_as_float(r[0]) : 0.0f, 0.0f, 0.0f, 0.0f);
    }
  }
  tc_fence_before();
  __syncthreads();
  DW_STAMP(3);
  dw_partial_barrier_reduce<BN>(args, out, red, tile, split, S, (int)gridDim.y);
  DW_STAMP(7);
  if (warp == 2) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(C::TMEM_COLS));
}

// ------------------------------------------------------------------ dW with a CTA pair (tcgen05 cta_group::2)
// A thread-block cluster of 2 CTAs (one TPC) computes a 256 x BN output tile for one K-split: CTA r loads its
// own 128 output rows of A (dZ) and the r-th half of B (the BN/2 activation columns), so each SM receives
// 2/3 of the bytes of a 128 x BN single-CTA tile for the same MMA work (the per-SM TMA rate, not the tensor
// core, bounds these skinny GEMMs). Both CTAs' loads complete on the leader's full barrier; the leader alone
// issues tcgen05.mma.cta_group::2 (M = 256) and multicasts its commits to the empty / accumulator-full
// barriers of both CTAs; each CTA then drains its own TMEM half (its 128 rows) into the shared split-K tail.
template <int BN>
struct Dw2Cfg {
  static constexpr int BM = 128, BK = 64;
  static constexpr int A_BYTES = BM * BK * 2;        // own 128 rows
  static constexpr int B_BYTES = (BN / 2) * BK * 2;  // own half of the columns
  static constexpr int ONES_BYTES = 16 * 128;
  static constexpr int FIXED = 1024 + ONES_BYTES + 512;
  static constexpr int STAGES_FIT = (232448 - FIXED) / (A_BYTES + B_BYTES);
  static constexpr int STAGES = STAGES_FIT > 8 ? 8 : STAGES_FIT;
  static constexpr int ACC_COLS = ((BN + 16) + 31) / 32 * 32;
  static constexpr int TMEM_COLS = ACC_COLS <= 32 ? 32 : ACC_COLS <= 64 ? 64 : ACC_COLS <= 128 ? 128 : ACC_COLS <= 256 ? 256 : 512;
  static constexpr int SMEM = FIXED + STAGES * (A_BYTES + B_BYTES);
};

template <int BN>
__global__ void __launch_bounds__(GEMM_THREADS, 1) k_gemm_dw2(const __grid_constant__ GemmArgs args, const DwOut out) {
  using C = Dw2Cfg<BN>;
  constexpr int RLD = BN + 20;
  static_assert(BN % 128 == 0, "each CTA loads whole 64-column atoms of its half");
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = sA + C::STAGES * C::A_BYTES;
  float* red = reinterpret_cast<float*>(smem);  // reuses the operand ring after the last MMA
  uint8_t* sOnes = sB + C::STAGES * C::B_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sOnes + C::ONES_BYTES);
  uint64_t* empty = full + C::STAGES;
  uint64_t* tfull = empty + C::STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tfull + 2);
  static_assert(128 * RLD * 4 <= C::STAGES * (C::A_BYTES + C::B_BYTES), "reduction buffer must fit the ring");

  DW_STAMP(0);
  pdl_trigger();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const int S = gridDim.x / 2;  // splits per pair tile
  const int split = blockIdx.x >> 1;
  // pair tile blockIdx.y -> (z, m-pair, n-tile); this CTA's 128-row tile index in decode() order
  const int n_t = args.n_tiles;
  const int ntile = blockIdx.y % n_t;
  const int pr = blockIdx.y / n_t;
  const int mpairs = args.m_tiles / 2;
  const int mt = (pr % mpairs) * 2 + (int)rank, z = pr / mpairs;
  const int tile = (z * args.m_tiles + mt) * n_t + ntile;
  const int m0 = mt * 128, n0 = ntile * BN;
  const bool bias_col = ntile == 0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < C::STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    mbar_init(&tfull[0], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  {
    uint32_t* o = reinterpret_cast<uint32_t*>(sOnes);
    for (int k = threadIdx.x; k < C::ONES_BYTES / 4; k += blockDim.x) o[k] = 0x3F803F80u;
    fence_async_smem();
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "n"(C::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  cluster_barrier();  // both CTAs' barriers initialised and TMEM allocated before any cross-CTA signal
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  DW_STAMP(1);
  pdl_wait();  // (partial_only launches use PDL: the prologue above overlapped the predecessor)
  const int kb0 = split * args.kb_per_split;
  const int nkb = max(0, min(args.kb_per_split, args.kb_total - kb0));
  const CUtensorMap* tmA = &args.tmA[z];
  const CUtensorMap* tmB = &args.tmB[z];

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int kb = 0; kb < nkb; ++kb) {
        mbar_wait(&empty[stage], phase ^ 1u);
        const int k0 = (kb0 + kb) * C::BK;
        uint8_t* a = sA + stage * C::A_BYTES;
        uint8_t* b = sB + stage * C::B_BYTES;
        if (rank == 0) mbar_expect_tx(&full[stage], 2 * (C::A_BYTES + C::B_BYTES));
        const uint32_t fb = mapa_shared(smem_u32(&full[stage]), 0);
        tma_load_2d_pair(tmA, fb, a, m0, k0);
        tma_load_2d_pair(tmA, fb, a + 8192, m0 + 64, k0);
#pragma unroll
        for (int i = 0; i < BN / 128; ++i)
          tma_load_2d_pair(tmB, fb, b + i * 8192, n0 + (int)rank * (BN / 2) + 64 * i, k0);
        if (++stage == C::STAGES) { stage = 0; phase ^= 1u; }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0 && rank == 0) {
      constexpr uint32_t idesc = idesc_bf16(256, BN, true, true);
      constexpr uint32_t idesc_ones = idesc_bf16(256, 16, true, false);
      int stage = 0;
      uint32_t phase = 0;
      for (int kb = 0; kb < nkb; ++kb) {
        mbar_wait(&full[stage], phase);
        tc_fence_after();
        const uint32_t a0 = smem_u32(sA + stage * C::A_BYTES), b0 = smem_u32(sB + stage * C::B_BYTES);
#pragma unroll
        for (int k = 0; k < C::BK / 16; ++k) {
          const uint64_t ad = sdesc(a0 + k * 2048u, 8192u, 1024u);
          const uint64_t bd = sdesc(b0 + k * 2048u, 8192u, 1024u);
          tc_mma_pair(tmem, ad, bd, idesc, (kb > 0 || k > 0) ? 1u : 0u);
          if (bias_col) {
            const uint64_t od = sdesc(smem_u32(sOnes) + k * 32u, 0u, 1024u);
            tc_mma_pair(tmem + BN, ad, od, idesc_ones, (kb > 0 || k > 0) ? 1u : 0u);
          }
        }
        tc_commit_pair(&empty[stage]);
        if (++stage == C::STAGES) { stage = 0; phase ^= 1u; }
      }
      if (nkb > 0) tc_commit_pair(&tfull[0]);
    }
    __syncwarp();
  } else if (warp >= 4) {
    // TMEM (this CTA's 128 rows) -> smem partial (an empty split contributes zeros)
    const int e = warp - 4, q = e & 3, h = e >> 2;
    const int row = q * 32 + lane;
    if (nkb > 0) {
      mbar_wait(&tfull[0], 0);
      __syncwarp();
      tc_fence_after();
    }
    if (out.dbg && threadIdx.x == 128) out.dbg[((size_t)blockIdx.y * gridDim.x + blockIdx.x) * 8 + 2] = gtimer();
    const uint32_t tbase = tmem + ((uint32_t)(q * 32) << 16);
    for (int c = h * (BN / 2); c < (h + 1) * (BN / 2); c += 32) {
      uint32_t r[32];
      if (nkb > 0) {
        tmem_ld32_nowait(tbase + c, r);
        tmem_wait_ld();
      } else {
#pragma unroll
        for (int k = 0; k < 32; ++k) r[k] = 0u;
      }
#pragma unroll
      for (int k = 0; k < 32; k += 4)
        *reinterpret_cast<float4*>(red + row * RLD + c + k) =
            make_float4(__uint_as_float(r[k]), __uint_as_float(r[k + 1]), __uint_as_float(r[k + 2]), __uint_as_float(r[k + 3]));
    }
    if (h == 0) {
      uint32_t r[32];
      if (nkb > 0 && bias_col) {
        tmem_ld32_nowait(tbase + BN, r);
        tmem_wait_ld();
      }
      *reinterpret_cast<float4*>(red + row * RLD + BN) =
          make_float4((nkb > 0 && bias_col) ? __uint_as_float(r[0]) : 0.0f, 0.0f, 0.0f, 0.0f);
    }
  }
  tc_fence_before();
  __syncthreads();
  DW_STAMP(3);
  (void)m0;
  dw_partial_barrier_reduce<BN>(args, out, red, tile, split, S, args.nz * args.m_tiles * args.n_tiles);
  DW_STAMP(7);
  tc_fence_before();
  cluster_barrier();  // both CTAs are done with the pair's TMEM
  tc_fence_after();
  if (warp == 2) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(C::TMEM_COLS));
}

// launch of a weight-gradient GEMM that stores only its partials (no grid barrier): 0 cooperative (the default:
// the whole wave starts together), 1 plain, 2 programmatic dependent launch (LG_DW_PARTIAL_LAUNCH, measurement;
// same-box C3: PDL 4.72 ms vs cooperative 4.38 ms -- early-resident CTAs hold SMs the critical dX kernels need)
static int dw_partial_launch() {
  static const int m = [] { const char* e = getenv("LG_DW_PARTIAL_LAUNCH"); return e ? atoi(e) : 0; }();
  return m;
}
template <int BN>
static cudaError_t launch_dw2_bn(const GemmArgs& a, const DwOut& o, int S, cudaStream_t st) {
  using C = Dw2Cfg<BN>;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(k_gemm_dw2<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  const int pair_tiles = a.nz * (a.m_tiles / 2) * a.n_tiles;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(2 * S, pair_tiles, 1);
  cfg.blockDim = dim3(GEMM_THREADS, 1, 1);
  cfg.dynamicSmemBytes = C::SMEM;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  if (o.partial_only && dw_partial_launch() != 0) {  // no grid barrier: plain (1) or PDL (2) cluster launch
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
  } else {
    attr[1].id = cudaLaunchAttributeCooperative;  // the grid barrier needs every CTA resident
    attr[1].val.cooperative = 1;
  }
  cfg.attrs = attr;
  cfg.numAttrs = (o.partial_only && dw_partial_launch() == 1) ? 1 : 2;
  return cudaLaunchKernelEx(&cfg, k_gemm_dw2<BN>, a, o);
}

// CTA-pair variant (requires an even number of 128-row tiles per z and BN in {128, 256}); S = splits per pair
// tile, 2 * S * pair_tiles <= #SMs
static int g_dw_max_ctas();
cudaError_t launch_gemm_dw_pair(int bn, const GemmArgs& a, const DwOut& o, int S, cudaStream_t st) {
  if (S < 1 || (a.m_tiles & 1) || 2 * S * a.nz * (a.m_tiles / 2) * a.n_tiles > g_dw_max_ctas()) return cudaErrorInvalidValue;
  switch (bn) {
    case 128: return launch_dw2_bn<128>(a, o, S, st);
    case 256: return launch_dw2_bn<256>(a, o, S, st);
    default: return cudaErrorInvalidValue;
  }
}

// ------------------------------------------------------------------ fused rollout policy
// Shared memory: R1 (8 x 16 KB K-major SW128 A-operand blocks: the X tile, then H1, then H2), a 2-stage ring
// of 32 KB weight chunks, biases, head weights and the cross-thread head exchange.
namespace fp {
constexpr int H0 = 512, H1 = 256, H2 = 128, BK = 64;
constexpr int ABLK = 128 * BK * 2;     // one 128-row x 64-col bf16 A block (16 KB)
constexpr int R1_BYTES = 8 * ABLK;     // H1 = 8 blocks
constexpr int STAGE = 256 * BK * 2;    // one 256-row weight chunk (32 KB)
constexpr int NSTAGE = 2;
constexpr int OFF_RING = R1_BYTES;
constexpr int OFF_BIAS = OFF_RING + NSTAGE * STAGE;           // b1 (512) | b2 (256) | b3 (128) fp32
constexpr int OFF_W4 = OFF_BIAS + 4096;                         // the net's head weights, build_w4_atoms
constexpr int OFF_XCH = OFF_W4 + W4_BYTES;                      // [128 rows][2][13] log-density terms
constexpr int OFF_BAR = OFF_XCH + 128 * 26 * 4;
constexpr int SMEM = 1024 + OFF_BAR + 24 * 8;
static_assert(OFF_W4 % 1024 == 0 && (H0 + H1 + H2) * 4 <= 4096, "fused policy smem layout");
}  // namespace fp

// bf16 pack of 32 fp32 values after bias + ELU, written into a K-major SW128 A block (row r, columns c..c+31
// of the layer output = k-block c/64, 16-B chunks (c%64)/8 .. +3)
__device__ __forceinline__ void store_act_block(uint8_t* R1, int r, int c, const uint32_t* acc, const float* bias) {
  uint32_t pk[16];
#pragma unroll
  for (int k = 0; k < 32; k += 4) {
    const float4 b4 = *reinterpret_cast<const float4*>(bias + k);  // 16-B aligned: c is a multiple of 32
    __nv_bfloat162 o0 = __floats2bfloat162_rn(elu_fast(__uint_as_float(acc[k]) + b4.x),
                                              elu_fast(__uint_as_float(acc[k + 1]) + b4.y));
    __nv_bfloat162 o1 = __floats2bfloat162_rn(elu_fast(__uint_as_float(acc[k + 2]) + b4.z),
                                              elu_fast(__uint_as_float(acc[k + 3]) + b4.w));
    pk[k / 2] = *reinterpret_cast<uint32_t*>(&o0);
    pk[k / 2 + 1] = *reinterpret_cast<uint32_t*>(&o1);
  }
  uint8_t* blk = R1 + (c >> 6) * fp::ABLK + r * 128;
  const int ch0 = (c & 63) >> 3;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int ch = ch0 + q;
    *reinterpret_cast<uint4*>(blk + ((ch ^ (r & 7)) << 4)) = make_uint4(pk[4 * q], pk[4 * q + 1], pk[4 * q + 2], pk[4 * q + 3]);
  }
}

#define FP_STAMP(k)                                                                                        \
  do {                                                                                                     \
    if (a.dbg) a.dbg[((size_t)blockIdx.y * gridDim.x + blockIdx.x) * 16 + (k)] = gtimer();                \
  } while (0)

__global__ void __launch_bounds__(GEMM_THREADS, 1) k_policy_fused(const __grid_constant__ FusedPolicyArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* R1 = smem;
  uint8_t* ring = smem + fp::OFF_RING;
  float* sB1 = reinterpret_cast<float*>(smem + fp::OFF_BIAS);
  float* sB2 = sB1 + fp::H0;
  float* sB3 = sB2 + fp::H1;
  uint8_t* sW4 = smem + fp::OFF_W4;  // build_w4_atoms
  float* sX = reinterpret_cast<float*>(smem + fp::OFF_XCH);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + fp::OFF_BAR);
  uint64_t* xfull = bars + 0;
  uint64_t* full = bars + 1;           // [4]
  uint64_t* empty = bars + 5;          // [4]
  uint64_t* tfull = bars + 9;          // [5]: layer 1 columns 0-255, 256-511, layer 2, layer 3, heads
  uint64_t* h1ready = bars + 14;       // [2]: H1 columns 0-255 / 256-511 staged
  uint64_t* h2ready = bars + 16;       // [4]: H2 k-block kb staged
  uint64_t* h3ready = bars + 20;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 21);
  // The layers overlap: the H1 epilogue of columns 0-255 runs beside the layer-1 MMAs of columns 256-511, layer 2
  // starts on k-blocks 0-3 once columns 0-255 are staged (beside the epilogue of 256-511), and layer 3 takes each
  // H2 k-block as soon as it is staged. R1 blocks: the observation tile occupies 0..kb1-1 (<= 3) until layer 1 is
  // done, so H1 columns 0-255 go to blocks 4-7 and columns 256-511 to blocks 0-3 (layer 2 reads k-block kb from
  // block (kb + 4) % 8: the same MMAs in the same order, bit-identical). Weight-chunk slots: 0, 1 = the ring;
  // 2, 3 = R1 blocks 4-5 and 6-7, free until H1 columns 0-255 are staged: W1's first half streams four chunks deep
  auto slot_ptr = [&](int sl) { return sl < 2 ? ring + sl * fp::STAGE : R1 + (4 + 2 * (sl - 2)) * fp::ABLK; };
  auto w1_slot = [&](int g) { return g < 4 ? (g & 3) : (g & 1); };  // chunk g of W1 (g < 4: columns 0-255)

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int z = a.z0 + (int)blockIdx.y;
  const int m0 = blockIdx.x * 128;
  if (threadIdx.x == 0) FP_STAMP(0);
  pdl_trigger();
  if (threadIdx.x == 0) {
    mbar_init(xfull, 1);
    for (int s2 = 0; s2 < 4; ++s2) { mbar_init(&full[s2], 1); mbar_init(&empty[s2], 1); }
    for (int s2 = 0; s2 < 5; ++s2) mbar_init(&tfull[s2], 1);
    for (int s2 = 0; s2 < 2; ++s2) mbar_init(&h1ready[s2], EPI_WARPS);
    for (int s2 = 0; s2 < 4; ++s2) mbar_init(&h2ready[s2], EPI_WARPS);
    mbar_init(h3ready, EPI_WARPS);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)), "n"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_wait();  // observation rows and weights are predecessors' outputs
  if (threadIdx.x == 0) FP_STAMP(1);

  if (warp == 0) {
    // ---------------------------------------------------------------- TMA producer
    if (lane == 0) {
      mbar_expect_tx(xfull, a.kb1 * fp::ABLK);
      for (int kb = 0; kb < a.kb1; ++kb) tma_load_2d(&a.tmX, xfull, R1 + kb * fp::ABLK, kb * fp::BK, m0);
      uint32_t ph = 0;  // bit sl: phase parity of slot sl
      auto load = [&](int sl, const CUtensorMap* map, int x, int y, uint32_t bytes) {
        mbar_wait(&empty[sl], ((ph >> sl) & 1u) ^ 1u);
        mbar_expect_tx(&full[sl], bytes);
        tma_load_2d(map, &full[sl], slot_ptr(sl), x, y);
        ph ^= 1u << sl;
      };
      int g = 0;
      for (int nh = 0; nh < 2; ++nh)
        for (int kb = 0; kb < a.kb1; ++kb, ++g) load(w1_slot(nh * 4 + kb), &a.tmW1, kb * fp::BK, z * fp::H0 + nh * 256, fp::STAGE);
      int rr = 0;
      for (int kb = 0; kb < fp::H0 / fp::BK; ++kb, ++rr) load(rr & 1, &a.tmW2[z], kb * fp::BK, 0, fp::STAGE);
      for (int kb = 0; kb < fp::H1 / fp::BK; ++kb, ++rr) load(rr & 1, &a.tmW3[z], kb * fp::BK, 0, fp::STAGE / 2);
    }
    __syncwarp();
  } else if (warp == 1) {
    // ---------------------------------------------------------------- MMA issuer
    if (lane == 0) {
      constexpr uint32_t id256 = idesc_bf16(128, 256, false, false);
      constexpr uint32_t id128 = idesc_bf16(128, 128, false, false);
      uint32_t ph = 0;  // bit sl: phase parity of slot sl (the producer's schedule)
      auto take = [&](int sl) {
        mbar_wait(&full[sl], (ph >> sl) & 1u);
        tc_fence_after();
        return smem_u32(slot_ptr(sl));
      };
      auto release = [&](int sl) {
        tc_commit(&empty[sl]);
        ph ^= 1u << sl;
      };
      mbar_wait(xfull, 0);
      tc_fence_after();
      // layer 1: two 256-column halves of this net's 512 outputs, K = kb1 blocks of the observation
      for (int nh = 0; nh < 2; ++nh) {
        for (int kb = 0; kb < a.kb1; ++kb) {
          const int sl = w1_slot(nh * 4 + kb);
          const uint32_t b0 = take(sl);
          const uint32_t a0 = smem_u32(R1 + kb * fp::ABLK);
#pragma unroll
          for (int k = 0; k < fp::BK / 16; ++k)
            tc_mma(tmem + nh * 256, sdesc(a0 + k * 32u, 0u, 1024u), sdesc(b0 + k * 32u, 0u, 1024u), id256,
                   (kb > 0 || k > 0) ? 1u : 0u);
          release(sl);
        }
        tc_commit(&tfull[nh]);
      }
      // layer 2: A = H1 (k-block kb in R1 block (kb + 4) % 8), N = 256 into TMEM columns [0, 256) -- free once
      // H1 columns 0-255 are read (h1ready[0]); k-blocks 4-7 wait for columns 256-511 (h1ready[1])
      int rr = 0;
      for (int kb = 0; kb < fp::H0 / fp::BK; ++kb, ++rr) {
        if (kb == 0 || kb == 4) {
          mbar_wait(&h1ready[kb >> 2], 0);
          tc_fence_after();
        }
        const int sl = rr & 1;
        const uint32_t b0 = take(sl);
        const uint32_t a0 = smem_u32(R1 + ((kb + 4) & 7) * fp::ABLK);
#pragma unroll
        for (int k = 0; k < fp::BK / 16; ++k)
          tc_mma(tmem, sdesc(a0 + k * 32u, 0u, 1024u), sdesc(b0 + k * 32u, 0u, 1024u), id256, (kb > 0 || k > 0) ? 1u : 0u);
        release(sl);
      }
      tc_commit(&tfull[2]);
      // layer 3: A = H2 (4 blocks in R1, each as soon as it is staged), N = 128 into TMEM columns [256, 384)
      for (int kb = 0; kb < fp::H1 / fp::BK; ++kb, ++rr) {
        mbar_wait(&h2ready[kb], 0);
        tc_fence_after();
        const int sl = rr & 1;
        const uint32_t b0 = take(sl);
        const uint32_t a0 = smem_u32(R1 + kb * fp::ABLK);
#pragma unroll
        for (int k = 0; k < fp::BK / 16; ++k)
          tc_mma(tmem + 256, sdesc(a0 + k * 32u, 0u, 1024u), sdesc(b0 + k * 32u, 0u, 1024u), id128,
                 (kb > 0 || k > 0) ? 1u : 0u);
        release(sl);
      }
      tc_commit(&tfull[3]);
      // the heads: H3 (bf16, in R1 blocks 0, 1) . W4^T into TMEM columns [384, 432)
      mbar_wait(h3ready, 0);
      tc_fence_after();
      head_mma(tmem + 384, smem_u32(R1), smem_u32(sW4));
      tc_commit(&tfull[4]);
    }
    __syncwarp();
  } else if (warp >= 4) {
    // ---------------------------------------------------------------- epilogues
    const int e = warp - 4, q = e & 3, h = e >> 2;
    const int r = q * 32 + lane;  // TMEM lane = tile row
    const uint32_t tb = tmem + ((uint32_t)(q * 32) << 16);
    // biases (16-B cp.async chunks, all in flight at once) and the net's head weights (three bf16 parts) are
    // staged here, while the producer and the MMA warp run layer 1
    {
      const int et = threadIdx.x - 128, nt = EPI_WARPS * 32;
      constexpr int C1 = fp::H0 / 4, C2 = C1 + fp::H1 / 4, C3 = C2 + fp::H2 / 4;
      for (int k = et; k < C3; k += nt) {
        const float* src;
        float* dst;
        if (k < C1) { src = a.b1 + z * fp::H0 + 4 * k; dst = sB1 + 4 * k; }
        else if (k < C2) { src = a.b2 + z * fp::H1 + 4 * (k - C1); dst = sB2 + 4 * (k - C1); }
        else { src = a.b3 + z * fp::H2 + 4 * (k - C2); dst = sB3 + 4 * (k - C2); }
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
      build_w4_atoms(sW4, a.W4a, a.W4c, fp::H2, z, et, nt);
      asm volatile("cp.async.wait_group 0;" ::: "memory");
      asm volatile("bar.sync 1, %0;" ::"n"(EPI_WARPS * 32));
    }
    // the actor's per-row sampling terms do not depend on the layers: sigma * eps (ACTION Philox), e^-log sigma,
    // log sigma and b4a of this thread's six action dimensions, computed while layer 1 runs (the same operations
    // as sample_action_b / logp_term: the same bits)
    const int hs = (warp - 4) >> 2;
    float pre_se[6], pre_ei[6], pre_ls[6], pre_b4[6];
#pragma unroll
    for (int jj = 0; jj < 6; ++jj) pre_se[jj] = pre_ei[jj] = pre_ls[jj] = pre_b4[jj] = 0.0f;
    if (z == 0 && m0 + r < a.N) {
      Rng rng{a.seed_lo, a.seed_hi};
      const uint32_t gid = (uint32_t)(a.rank * a.N + m0 + r);
      const uint32_t ev = a.scalars->s_base + (uint32_t)a.t + 1u;
      const U4 blk0 = rng.block((uint32_t)(hs == 0 ? 0 : 1), gid, ev, TAG_ACTION);
      const U4 blk1 = rng.block((uint32_t)(hs == 0 ? 1 : 2), gid, ev, TAG_ACTION);
#pragma unroll
      for (int jj = 0; jj < 6; ++jj) {
        const int j = 6 * hs + jj;
        pre_ls[jj] = __ldg(a.logstd + j);
        pre_b4[jj] = __ldg(a.b4a + j);
        pre_ei[jj] = expf(-pre_ls[jj]);
        const bool first = (j >> 2) == (hs == 0 ? 0 : 1);
        pre_se[jj] = action_noise_b(first ? blk0 : blk1, j, pre_ls[jj]);
      }
    }
    // layer 1 -> H1 (bias + ELU, bf16): columns 0-255 into R1 blocks 4-7 as soon as their MMAs are done (beside
    // the MMAs of columns 256-511), then columns 256-511 into blocks 0-3 (the observation tile is dead by then);
    // each half: thread (q, h) takes columns 128h .. 128h+127 of it
    for (int nh = 0; nh < 2; ++nh) {
      mbar_wait(&tfull[nh], 0);
      __syncwarp();
      tc_fence_after();
      if (threadIdx.x == 128) FP_STAMP(2 + nh);
      uint8_t* dst = nh == 0 ? R1 + 4 * fp::ABLK : R1 - 4 * fp::ABLK;  // block (c >> 6) + 4 or - 4
      for (int c = nh * 256 + h * 128; c < nh * 256 + h * 128 + 128; c += 32) {
        uint32_t acc[32];
        tmem_ld32_nowait(tb + c, acc);
        tmem_wait_ld();
        store_act_block(dst, r, c, acc, sB1 + c);
      }
      fence_async_smem();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&h1ready[nh]);
    }
    // layer 2 -> H2 into R1 blocks 0-3 (H1 is dead once tfull[2] fired), one k-block at a time for layer 3:
    // thread (q, h) takes columns 64kb + 32h .. +31 of block kb
    mbar_wait(&tfull[2], 0);
    __syncwarp();
    tc_fence_after();
    if (threadIdx.x == 128) FP_STAMP(4);
    for (int kb = 0; kb < fp::H1 / fp::BK; ++kb) {
      const int c = 64 * kb + 32 * h;
      uint32_t acc[32];
      tmem_ld32_nowait(tb + c, acc);
      tmem_wait_ld();
      store_act_block(R1, r, c, acc, sB2 + c);
      fence_async_smem();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&h2ready[kb]);
    }
    if (threadIdx.x == 128) FP_STAMP(5);
    // layer 3 -> H3 (bf16, as the unfused path stores it) into R1 blocks 0, 1 (H2 is dead once tfull[3] fired)
    // -> the head MMA (head_mma: the loss epilogue's instruction sequence) -> mu - b4a / V - b4c in TMEM
    mbar_wait(&tfull[3], 0);
    __syncwarp();
    tc_fence_after();
    if (threadIdx.x == 128) FP_STAMP(6);
    for (int c = h * 64; c < h * 64 + 64; c += 32) {
      uint32_t acc[32];
      tmem_ld32_nowait(tb + 256 + c, acc);
      tmem_wait_ld();
      store_act_block(R1, r, c, acc, sB3 + c);
    }
    fence_async_smem();
    tc_fence_before();
    __syncwarp();
    if (lane == 0) mbar_arrive(h3ready);
    mbar_wait(&tfull[4], 0);
    __syncwarp();
    tc_fence_after();
    uint32_t d1[48];
    tmem_ld32_nowait(tb + 384, d1);
    tmem_ld16_nowait(tb + 416, d1 + 32);
    tmem_wait_ld();
    const int nval = z == 0 ? 12 : 1;
    (void)nval;
    // the two threads of a row split the action dimensions: h = 0 takes j < 6 (ACTION Philox blocks 0, 1),
    // h = 1 takes j >= 6 (blocks 1, 2); their log-density terms meet in smem for the fixed-order sum.
    if (threadIdx.x == 128) FP_STAMP(7);
    float* xrow = sX + r * 26;
    const int row = m0 + r;
    if (z == 1) {
      if (hs == 0 && row < a.N) {
        const float V = __fadd_rn(head_out(d1, 0), __ldg(a.b4c));
        a.value[row] = V;
        if (a.u_value) a.u_value[row] = V;
      }
    } else {
      float* trow = xrow;  // reused for the 12 log-density terms after the sums are consumed
      float tm[6];
      if (row < a.N) {
#pragma unroll
        for (int jj = 0; jj < 6; ++jj) {
          const int j = 6 * hs + jj;
          const float dj = hs == 0 ? head_out(d1, jj) : head_out(d1, 6 + jj);  // constant indices: d1[] in registers
          const float mu = __fadd_rn(dj, pre_b4[jj]);
          const float act = a.deterministic ? mu : __fadd_rn(mu, pre_se[jj]);
          tm[jj] = logp_term_e(act, mu, pre_ei[jj], pre_ls[jj]);
          a.act[(size_t)row * 12 + j] = act;
          a.mu[(size_t)row * 12 + j] = mu;
          if (a.u_act) a.u_act[(size_t)row * 12 + j] = act;
          if (a.u_mu) a.u_mu[(size_t)row * 12 + j] = mu;
        }
      }
#pragma unroll
      for (int jj = 0; jj < 6; ++jj) trow[6 * hs + jj] = tm[jj];
      asm volatile("bar.sync 1, %0;" ::"n"(EPI_WARPS * 32));
      if (hs == 0 && row < a.N) {
        float t[12];
#pragma unroll
        for (int j = 0; j < 12; ++j) t[j] = trow[j];
        // log-probability: dim_sum's butterfly (term j on lane 2j, zeros elsewhere), same additions in order:
        // offsets 16, 8, 4, 2, 1 pair lanes (2m, 2m+16), (2m, 2m+8), (2m, 2m+4), (0, 2), (0, 1)
        float e8[8];
#pragma unroll
        for (int m = 0; m < 4; ++m) e8[m] = t[m] + t[m + 8];
#pragma unroll
        for (int m = 4; m < 8; ++m) e8[m] = t[m] + 0.0f;
#pragma unroll
        for (int m = 0; m < 4; ++m) e8[m] = e8[m] + e8[m + 4];
        e8[0] = e8[0] + e8[2];
        e8[1] = e8[1] + e8[3];
        const float k01 = e8[0] + e8[1];
        const float lp = __fsub_rn(-(k01 + 0.0f), 11.027262398456072f);
        a.logp[row] = lp;
        if (a.u_logp) a.u_logp[row] = lp;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) FP_STAMP(8);
  if (warp == 2) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(512));
}

cudaError_t launch_policy_fused(const FusedPolicyArgs& a, cudaStream_t st) {
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(k_policy_fused, cudaFuncAttributeMaxDynamicSharedMemorySize, fp::SMEM);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  if (a.kb1 < 1 || a.kb1 > 4) return cudaErrorInvalidValue;
  if (a.z0 < 0 || a.z0 > 1) return cudaErrorInvalidValue;
  dim3 grid((a.N + 127) / 128, 2 - a.z0, 1);
  return launch_pdl(k_policy_fused, grid, dim3(GEMM_THREADS), fp::SMEM, st, a);
}

// ------------------------------------------------------------------ host side
bool pdl_enabled() {
  static const bool on = [] {
    const char* e = getenv("LG_NO_PDL");
    return !(e && e[0] == '1');
  }();
  return on;
}

static PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
static int g_num_sms = 0;
static int g_dw_max_ctas() {  // one k_gemm_dw CTA per SM (its shared memory allows no more)
  if (!g_num_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_num_sms <= 0) g_num_sms = 148;
  }
  return g_num_sms;
}

bool tma_init() {
  if (g_encode) return true;
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn) return false;
  g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  return true;
}

static bool encode(CUtensorMap* map, CUtensorMapDataType dt, int esize, const void* base, uint64_t rows, uint64_t cols,
                   uint64_t ld, uint32_t box_cols, uint32_t box_rows) {
  if (!tma_init()) return false;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {ld * (uint64_t)esize};
  cuuint32_t box[2] = {box_cols, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = g_encode(map, dt, 2, const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// 2D bf16 tensor [rows][cols] with row stride ld (elements); box {64, box_rows}; 128-B swizzle; OOB = 0
bool make_tmap_bf16(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols, uint64_t ld, uint32_t box_rows) {
  return encode(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, base, rows, cols, ld, 64, box_rows);
}
// 2D fp32 tensor, box {32, box_rows} (128 B inner), 128-B swizzle
bool make_tmap_f32(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols, uint64_t ld, uint32_t box_rows) {
  return encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, base, rows, cols, ld, 32, box_rows);
}

template <int BN, bool A_MN, bool B_MN, int EPI, bool PAIR = false, int WSKB = 0>
static cudaError_t launch_one(const GemmArgs& a, cudaStream_t st) {
  using C = GemmCfg<BN, EPI, PAIR, WSKB>;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(k_gemm_tc<BN, A_MN, B_MN, EPI, PAIR, WSKB>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  if (!g_num_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_num_sms <= 0) g_num_sms = 148;
  }
  if (PAIR) {
    const int total = a.nz * ((a.m_tiles + 1) / 2) * a.n_tiles * a.n_splits;
    const int pairs = total < g_num_sms / 2 ? total : g_num_sms / 2;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(2 * pairs, 1, 1);
    cfg.blockDim = dim3(GEMM_THREADS, 1, 1);
    cfg.dynamicSmemBytes = C::SMEM;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 2 : 1;
    return cudaLaunchKernelEx(&cfg, k_gemm_tc<BN, A_MN, B_MN, EPI, PAIR>, a);
  }
  if (WSKB) {  // cps CTAs per column block (slice), every CTA of a slice takes every cps-th row tile
    const int nsl = a.n_tiles * a.nz;
    const int cps = std::min(a.m_tiles, g_num_sms / nsl);
    return launch_pdl(k_gemm_tc<BN, A_MN, B_MN, EPI, false, WSKB>, dim3(cps * nsl), dim3(GEMM_THREADS), C::SMEM, st, a);
  }
  const int total = a.nz * a.m_tiles * a.n_tiles * a.n_splits;
  const int grid = total < g_num_sms ? total : g_num_sms;
  return launch_pdl(k_gemm_tc<BN, A_MN, B_MN, EPI>, dim3(grid), dim3(GEMM_THREADS), C::SMEM, st, a);
}

// weight-stationary eligibility: one split, the slice count fits the grid, the resident block fits WSKB
static bool ws_ok(const GemmArgs& a) {
  static const bool off = [] { const char* e = getenv("LG_NO_WS"); return e && e[0] == '1'; }();
  if (!g_num_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_num_sms <= 0) g_num_sms = 148;
  }
  return !off && a.ws && !a.pair && !a.M_dev && a.n_splits == 1 && a.kb_per_split == a.kb_total &&
         a.n_tiles * a.nz <= g_num_sms / 2;
}

template <bool A_MN, bool B_MN, int EPI>
static cudaError_t dispatch_bn(int bn, const GemmArgs& a, cudaStream_t st) {
  if constexpr (EPI != 3 && !A_MN) {
    if (ws_ok(a)) {  // resident B: <= 128 KB (BN 256: 4 k-blocks, BN 128: 8); smaller blocks leave a deeper A ring
      const int kb = a.kb_total;
      if (bn == 256 && kb <= 2) return launch_one<256, A_MN, B_MN, EPI, false, 2>(a, st);
      if (bn == 256 && kb <= 4) return launch_one<256, A_MN, B_MN, EPI, false, 4>(a, st);
      if (bn == 128 && kb <= 4) return launch_one<128, A_MN, B_MN, EPI, false, 4>(a, st);
      if (bn == 128 && kb <= 8) return launch_one<128, A_MN, B_MN, EPI, false, 8>(a, st);
    }
    if (a.pair) {
      switch (bn) {
        case 128: return launch_one<128, A_MN, B_MN, EPI, true>(a, st);
        case 256: return launch_one<256, A_MN, B_MN, EPI, true>(a, st);
        default: break;
      }
    }
  }
  switch (bn) {
    case 64: return launch_one<64, A_MN, B_MN, EPI>(a, st);
    case 128: return launch_one<128, A_MN, B_MN, EPI>(a, st);
    case 256: return launch_one<256, A_MN, B_MN, EPI>(a, st);
    default: return cudaErrorInvalidValue;
  }
}

template <int BN, bool KMAJ = false>
static cudaError_t launch_dw_bn(const GemmArgs& a, const DwOut& o, int S, cudaStream_t st) {
  using C = DwCfg<BN>;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(k_gemm_dw<BN, KMAJ>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  const int tiles = a.nz * a.m_tiles * a.n_tiles;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(S, tiles, 1);
  cfg.blockDim = dim3(GEMM_THREADS, 1, 1);
  cfg.dynamicSmemBytes = C::SMEM;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  if (o.partial_only && dw_partial_launch() != 0) {  // no grid barrier: plain (1) or PDL (2) launch
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
  } else {
    attr[0].id = cudaLaunchAttributeCooperative;  // the grid barrier needs every CTA resident
    attr[0].val.cooperative = 1;
  }
  cfg.attrs = attr;
  cfg.numAttrs = (o.partial_only && dw_partial_launch() == 1) ? 0 : 1;
  return cudaLaunchKernelEx(&cfg, k_gemm_dw<BN, KMAJ>, a, o);
}

// diagnostics (tools/gemm_probe): dW from transposed, K-major operand copies
cudaError_t launch_gemm_dw_kmajor(int bn, const GemmArgs& a, const DwOut& o, int S, cudaStream_t st) {
  switch (bn) {
    case 128: return launch_dw_bn<128, true>(a, o, S, st);
    case 256: return launch_dw_bn<256, true>(a, o, S, st);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_gemm_dw(int bn, const GemmArgs& a, const DwOut& o, int S, cudaStream_t st) {
  if (S < 1 || S * a.nz * a.m_tiles * a.n_tiles > g_dw_max_ctas()) return cudaErrorInvalidValue;  // one wave
  switch (bn) {
    case 64: return launch_dw_bn<64>(a, o, S, st);
    case 128: return launch_dw_bn<128>(a, o, S, st);
    case 256: return launch_dw_bn<256>(a, o, S, st);
    default: return cudaErrorInvalidValue;
  }
}

// EPI 4: the update's layer 3 + PPO loss head. Weight-stationary (each CTA keeps its net's W3, <= 4 k-blocks);
// the grid covers min(m_tiles, #SMs / 2) CTAs per net, split between the nets by the epilogue cost of their rows
// (an actor row does 12 head outputs, its KL and 12 x 128 head-gradient products; a critic row one) --
// LG_LOSS_ACTOR_FRAC overrides the share (measurement only). Every CTA owns at least one tile.
int gemm_loss_grid(const GemmArgs& a) {
  const int m_tiles = (a.M + 127) / 128;
  return 2 * std::min(m_tiles, g_dw_max_ctas() / 2);
}
cudaError_t launch_gemm_loss(const GemmArgs& a0, int* grid_out, cudaStream_t st) {
  using C = GemmCfg<128, 4, false, 4>;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(k_gemm_tc<128, false, false, 4, false, 4>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  static const double frac = [] { const char* e = getenv("LG_LOSS_ACTOR_FRAC"); return e ? atof(e) : -1.0; }();
  GemmArgs a = a0;
  a.m_tiles = (a.M + 127) / 128;
  a.nz = 2; a.n_tiles = 1; a.n_splits = 1; a.kb_per_split = a.kb_total;
  if (a.kb_total < 1 || a.kb_total > 4 || a.N > 128 || a.le.H2 != a.N || a.M_dev) return cudaErrorInvalidValue;
  const int grid = gemm_loss_grid(a);
  const int lo = std::max(1, grid - a.m_tiles), hi = std::min(a.m_tiles, grid - 1);
  int split;
  if (frac > 0) {
    split = std::max(lo, std::min(hi, (int)std::lround(frac * grid)));
  } else {
    // the busiest CTA's tiles x per-tile cost (tools/gemm_probe loss stamps: an actor tile ~5.0 us, a critic tile
    // ~4.1 us); ties go to the split that balances the nets' average load (C3: 64..84 actor CTAs of 148 all give
    // 3 tiles per CTA; same-box A/B 4.32 ms against 4.37 with the previous fixed 65 % actor share)
    constexpr double CA = 1.22, CC = 1.0;
    double best = 1e30, bal = 1e30;
    split = lo;
    for (int s = lo; s <= hi; ++s) {
      const double ta = CA * ((a.m_tiles + s - 1) / s), tc = CC * ((a.m_tiles + grid - s - 1) / (grid - s));
      const double mx = std::max(ta, tc), b = std::fabs(CA * a.m_tiles / s - CC * a.m_tiles / (grid - s));
      if (mx < best - 1e-9 || (mx < best + 1e-9 && b < bal)) { best = mx; bal = b; split = s; }
    }
  }
  a.ws_split = split;
  if (grid_out) *grid_out = grid;
  return launch_pdl(k_gemm_tc<128, false, false, 4, false, 4>, dim3(grid), dim3(GEMM_THREADS), C::SMEM, st, a);
}

cudaError_t launch_gemm(GemmKind kind, int bn, const GemmArgs& a, cudaStream_t st) {
  switch (kind) {
    case GEMM_FWD: return dispatch_bn<false, false, 0>(bn, a, st);
    case GEMM_DX: return dispatch_bn<false, true, 2>(bn, a, st);
    case GEMM_DW: return dispatch_bn<true, true, 3>(bn, a, st);
  }
  return cudaErrorInvalidValue;
}

}  // namespace lg
