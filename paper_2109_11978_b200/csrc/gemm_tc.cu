// gemm_tc.cu -- tcgen05 (5th-gen tensor core) bf16 GEMM for sm_100a with TMA operand staging,
// an mbarrier producer/consumer pipeline and the fp32 accumulator in TMEM, with the MLP's epilogues
// fused (the one dense contraction of the path, BJ north_star).
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
// Warp roles (128 threads): warp 0 lane 0 issues TMA, warp 1 lane 0 issues tcgen05.mma, warp 2 owns
// the TMEM allocation, all four warps run the epilogue (warp w reads TMEM lanes 32w..32w+31 = rows).
#include <cuda.h>
#include <cudaTypedefs.h>

#include "common.cuh"
#include "kernels.h"

namespace lg {

// ------------------------------------------------------------------ PTX wrappers
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n\t"
      "@P1 bra DONE_%=;\n\t"
      "bra WAIT_%=;\n\t"
      "DONE_%=:\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity), "r"(0x989680));
}
__device__ __forceinline__ void tma_load_2d(const CUtensorMap* map, uint64_t* bar, void* dst, int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(x), "r"(y)
      : "memory");
}
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
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float* v) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,"
      "%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int k = 0; k < 32; ++k) v[k] = __uint_as_float(r[k]);
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

template <int BN>
struct GemmCfg {
  static constexpr int BM = 128, BK = 64;
  static constexpr int STAGES = BN >= 256 ? 4 : (BN >= 128 ? 6 : 8);
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int B_BYTES = (BN < 64 ? 64 : BN) * BK * 2;  // MN-major B pads to one 64-wide atom
  template <bool B_MN>
  static constexpr int b_load_bytes() { return B_MN ? B_BYTES : BN * BK * 2; }
  static constexpr int ONES_BYTES = 16 * 128;                    // 16 rows x 64 bf16 of 1.0
  static constexpr int SMEM = 1024 + STAGES * (A_BYTES + B_BYTES) + ONES_BYTES + 256;
  static constexpr int TMEM_COLS = (BN + 16) <= 32 ? 32 : (BN + 16) <= 64 ? 64 : (BN + 16) <= 128 ? 128 : (BN + 16) <= 256 ? 256 : 512;
};

__device__ __forceinline__ float elu(float x) { return x > 0.0f ? x : expm1f(x); }

template <int BN, bool A_MN, bool B_MN, int EPI>
__global__ void __launch_bounds__(128, 1) k_gemm_tc(const __grid_constant__ GemmArgs args) {
  using C = GemmCfg<BN>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + C::STAGES * C::A_BYTES;
  uint8_t* sOnes = sB + C::STAGES * C::B_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sOnes + C::ONES_BYTES);
  uint64_t* empty = full + C::STAGES;
  uint64_t* accb = empty + C::STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(accb + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int z = blockIdx.z;
  const int m0 = blockIdx.x * C::BM;
  const int ntile = blockIdx.y % args.n_tiles, split = blockIdx.y / args.n_tiles;
  const int n0 = ntile * BN;
  const int M = args.M_dev ? *args.M_dev : args.M;
  if (m0 >= M) return;  // uniform early exit (device-sized M)
  const int kb0 = split * args.kb_per_split;
  const int nkb = min(args.kb_per_split, args.kb_total - kb0);
  const bool bias_col = (EPI == 3) && args.bias_col && ntile == 0;

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    mbar_init(accb, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (EPI == 3) {  // 16 x 64 bf16 ones (any swizzle of a constant tile is the same tile)
    uint32_t* o = reinterpret_cast<uint32_t*>(sOnes);
    for (int k = threadIdx.x; k < C::ONES_BYTES / 4; k += blockDim.x) o[k] = 0x3F803F80u;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
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
        mbar_expect_tx(&full[stage], C::A_BYTES + C::template b_load_bytes<B_MN>());
        if (!A_MN) {
          tma_load_2d(tmA, &full[stage], a, k0, m0);
        } else {
          tma_load_2d(tmA, &full[stage], a, m0, k0);
          tma_load_2d(tmA, &full[stage], a + 8192, m0 + 64, k0);
        }
        if (!B_MN) {
          tma_load_2d(tmB, &full[stage], b, k0, n0);
        } else {
#pragma unroll
          for (int i = 0; i < (BN < 64 ? 1 : BN / 64); ++i) tma_load_2d(tmB, &full[stage], b + i * 8192, n0 + 64 * i, k0);
        }
        if (++stage == C::STAGES) { stage = 0; phase ^= 1u; }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = idesc_bf16(128, BN, A_MN, B_MN);
      constexpr uint32_t idesc_ones = idesc_bf16(128, 16, A_MN, false);
      const uint32_t a_lbo = A_MN ? 8192u : 0u, b_lbo = B_MN ? 8192u : 0u;
      const uint32_t a_step = A_MN ? 2048u : 32u, b_step = B_MN ? 2048u : 32u;  // bytes per UMMA_K = 16
      int stage = 0;
      uint32_t phase = 0;
      for (int kb = 0; kb < nkb; ++kb) {
        mbar_wait(&full[stage], phase);
        tc_fence_after();
        const uint32_t a0 = smem_u32(sA + stage * C::A_BYTES), b0 = smem_u32(sB + stage * C::B_BYTES);
#pragma unroll
        for (int k = 0; k < C::BK / 16; ++k) {
          uint64_t ad = sdesc(a0 + k * a_step, a_lbo, 1024u);
          uint64_t bd = sdesc(b0 + k * b_step, b_lbo, 1024u);
          tc_mma(tmem, ad, bd, idesc, (kb > 0 || k > 0) ? 1u : 0u);
          if (bias_col) {
            uint64_t od = sdesc(smem_u32(sOnes) + k * 32u, 0u, 1024u);
            tc_mma(tmem + BN, ad, od, idesc_ones, (kb > 0 || k > 0) ? 1u : 0u);
          }
        }
        tc_commit(&empty[stage]);
        if (++stage == C::STAGES) { stage = 0; phase ^= 1u; }
      }
      tc_commit(accb);
    }
    __syncwarp();
  }

  // ---------------- epilogue: TMEM -> registers -> global
  mbar_wait(accb, 0);
  __syncwarp();
  tc_fence_after();
  const int row = m0 + warp * 32 + lane;
  const bool row_ok = row < M;
  const uint32_t tbase = tmem + ((uint32_t)(warp * 32) << 16);
  const int ncols = min(BN, args.N - n0);
#pragma unroll 1
  for (int c = 0; c < BN; c += 32) {
    float v[32];
    tmem_ld32(tbase + c, v);
    if (!row_ok || c >= ncols) continue;
    if (EPI == 0) {
      const float* bias = args.bias[z] + n0 + c;
      __nv_bfloat16* dst = reinterpret_cast<__nv_bfloat16*>(args.out[z]) + (size_t)row * args.ldo + n0 + c;
      uint32_t pk[16];
#pragma unroll
      for (int k = 0; k < 32; k += 2) {
        __nv_bfloat162 h = __floats2bfloat162_rn(elu(v[k] + __ldg(bias + k)), elu(v[k + 1] + __ldg(bias + k + 1)));
        pk[k / 2] = *reinterpret_cast<uint32_t*>(&h);
      }
      uint4* d4 = reinterpret_cast<uint4*>(dst);
#pragma unroll
      for (int q = 0; q < 4; ++q) d4[q] = make_uint4(pk[4 * q], pk[4 * q + 1], pk[4 * q + 2], pk[4 * q + 3]);
    } else if (EPI == 2) {
      const __nv_bfloat16* aux = args.aux[z] + (size_t)row * args.ld_aux + n0 + c;
      __nv_bfloat16* dst = reinterpret_cast<__nv_bfloat16*>(args.out[z]) + (size_t)row * args.ldo + n0 + c;
      const uint4* a4 = reinterpret_cast<const uint4*>(aux);
      uint32_t pk[16];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        uint4 u = a4[q];
        uint32_t w4[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          __nv_bfloat162 hb = *reinterpret_cast<__nv_bfloat162*>(&w4[e]);
          float2 hf = __bfloat1622float2(hb);
          int k = 8 * q + 2 * e;
          float g0 = v[k] * (hf.x > 0.0f ? 1.0f : hf.x + 1.0f);
          float g1 = v[k + 1] * (hf.y > 0.0f ? 1.0f : hf.y + 1.0f);
          __nv_bfloat162 o = __floats2bfloat162_rn(g0, g1);
          pk[k / 2] = *reinterpret_cast<uint32_t*>(&o);
        }
      }
      uint4* d4 = reinterpret_cast<uint4*>(dst);
#pragma unroll
      for (int q = 0; q < 4; ++q) d4[q] = make_uint4(pk[4 * q], pk[4 * q + 1], pk[4 * q + 2], pk[4 * q + 3]);
    } else {
      float* dst = args.part + (size_t)z * args.part_zstride + (size_t)split * args.part_sstride +
                   (size_t)row * args.part_ld + n0 + c;
      float4* d4 = reinterpret_cast<float4*>(dst);
#pragma unroll
      for (int q = 0; q < 8; ++q) d4[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
    }
  }
  if (EPI == 3 && args.bias_col) {
    float v[32];
    if (bias_col) tmem_ld32(tbase + BN, v);  // (warp-uniform branch)
    if (bias_col && row_ok) {
      float* dst = args.part + (size_t)z * args.part_zstride + (size_t)split * args.part_sstride +
                   (size_t)row * args.part_ld + args.part_bias_col;
      *dst = v[0];
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(C::TMEM_COLS));
}

// ------------------------------------------------------------------ host side
static PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;

bool tma_init() {
  if (g_encode) return true;
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn) return false;
  g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  return true;
}

// 2D bf16 tensor [rows][cols] with row stride ld (elements); box {64, box_rows}; 128-B swizzle; OOB = 0
bool make_tmap_bf16(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols, uint64_t ld, uint32_t box_rows) {
  if (!tma_init()) return false;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {ld * 2};
  cuuint32_t box[2] = {64, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = g_encode(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

template <int BN, bool A_MN, bool B_MN, int EPI>
static cudaError_t launch_one(const GemmArgs& a, int m_tiles, int nz, cudaStream_t st) {
  using C = GemmCfg<BN>;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(k_gemm_tc<BN, A_MN, B_MN, EPI>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  dim3 grid(m_tiles, a.n_tiles * a.n_splits, nz);
  k_gemm_tc<BN, A_MN, B_MN, EPI><<<grid, 128, C::SMEM, st>>>(a);
  return cudaGetLastError();
}

template <bool A_MN, bool B_MN, int EPI>
static cudaError_t dispatch_bn(int bn, const GemmArgs& a, int m_tiles, int nz, cudaStream_t st) {
  switch (bn) {
    case 32: return launch_one<32, A_MN, B_MN, EPI>(a, m_tiles, nz, st);
    case 64: return launch_one<64, A_MN, B_MN, EPI>(a, m_tiles, nz, st);
    case 128: return launch_one<128, A_MN, B_MN, EPI>(a, m_tiles, nz, st);
    case 256: return launch_one<256, A_MN, B_MN, EPI>(a, m_tiles, nz, st);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_gemm(GemmKind kind, int bn, const GemmArgs& a, int m_tiles, int nz, cudaStream_t st) {
  switch (kind) {
    case GEMM_FWD: return dispatch_bn<false, false, 0>(bn, a, m_tiles, nz, st);
    case GEMM_DX: return dispatch_bn<false, true, 2>(bn, a, m_tiles, nz, st);
    case GEMM_DW: return dispatch_bn<true, true, 3>(bn, a, m_tiles, nz, st);
  }
  return cudaErrorInvalidValue;
}

}  // namespace lg
