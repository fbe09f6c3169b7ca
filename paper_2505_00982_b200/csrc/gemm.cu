// Split-BF16x3 GEMMs for the MLP contractions (HVP forward/R-forward, backward/R-backward,
// weight-gradient accumulation; SURVEY.md §2 kernel table):
//
//     C[M x N] = alpha * (Ah*Bh^T + Ah*Bl^T + Al*Bh^T),   A: M x K, B: N x K, both K-major.
//
// gemm3_tc   : sm_100a tcgen05.mma (kind::f16, BF16 in, FP32 accumulate in TMEM), operands
//              staged by TMA (SWIZZLE_128B) through a multi-stage mbarrier pipeline; one
//              elected thread issues MMAs, 4 epilogue warps drain TMEM with tcgen05.ld.
// gemm3_simt : CUDA-core reference kernel with identical split arithmetic (fp32 FMA); used as
//              the in-device cross-check of the tensor-core path and selectable via
//              dho2g_ctx_set_option("gemm", 1).
#include <cudaTypedefs.h>

#include "internal.h"

namespace dho2g {

// =============================================================================== CUDA-core path
namespace {
constexpr int ST_BM = 64, ST_BN = 64, ST_BK = 16;

__global__ void __launch_bounds__(256) gemm3_simt_kernel(int M, int N, int K, const bf16* __restrict__ Ahi,
                                                         const bf16* __restrict__ Alo, int lda,
                                                         const bf16* __restrict__ Bhi, const bf16* __restrict__ Blo,
                                                         int ldb, float* __restrict__ C, int ldc, float alpha) {
  __shared__ float sAh[ST_BK][ST_BM + 4], sAl[ST_BK][ST_BM + 4], sBh[ST_BK][ST_BN + 4], sBl[ST_BK][ST_BN + 4];
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  const int m0 = blockIdx.y * ST_BM, n0 = blockIdx.x * ST_BN;
  float acc[4][4] = {};
  for (int k0 = 0; k0 < K; k0 += ST_BK) {
    for (int e = threadIdx.x; e < ST_BM * ST_BK; e += 256) {
      const int r = e / ST_BK, kk = e % ST_BK;
      const int gm = m0 + r, gk = k0 + kk;
      float ah = 0.f, al = 0.f;
      if (gm < M && gk < K) {
        ah = __bfloat162float(Ahi[(size_t)gm * lda + gk]);
        al = __bfloat162float(Alo[(size_t)gm * lda + gk]);
      }
      sAh[kk][r] = ah;
      sAl[kk][r] = al;
      const int gn = n0 + r;
      float bh = 0.f, bl = 0.f;
      if (gn < N && gk < K) {
        bh = __bfloat162float(Bhi[(size_t)gn * ldb + gk]);
        bl = __bfloat162float(Blo[(size_t)gn * ldb + gk]);
      }
      sBh[kk][r] = bh;
      sBl[kk][r] = bl;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < ST_BK; ++kk) {
      float ah[4], al[4], bh[4], bl[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        ah[i] = sAh[kk][ty * 4 + i];
        al[i] = sAl[kk][ty * 4 + i];
        bh[i] = sBh[kk][tx * 4 + i];
        bl[i] = sBl[kk][tx * 4 + i];
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          acc[i][j] = fmaf(ah[i], bh[j], acc[i][j]);
          acc[i][j] = fmaf(ah[i], bl[j], acc[i][j]);
          acc[i][j] = fmaf(al[i], bh[j], acc[i][j]);
        }
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int gm = m0 + ty * 4 + i;
    if (gm >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int gn = n0 + tx * 4 + j;
      if (gn < N) C[(size_t)gm * ldc + gn] = alpha * acc[i][j];
    }
  }
}
}  // namespace

void gemm3_simt(cudaStream_t s, int M, int N, int K, const bf16* Ahi, const bf16* Alo, int lda, const bf16* Bhi,
                const bf16* Blo, int ldb, float* C, int ldc, float alpha) {
  dim3 grid(cdiv(N, ST_BN), cdiv(M, ST_BM));
  gemm3_simt_kernel<<<grid, 256, 0, s>>>(M, N, K, Ahi, Alo, lda, Bhi, Blo, ldb, C, ldc, alpha);
  DHO2G_LAUNCH();
}

// =============================================================================== tcgen05 path
namespace tc {

constexpr int BM = 128;  // UMMA_M (cta_group::1): TMEM lane i <-> output row i
constexpr int BK = 64;   // one 128-byte swizzle row of bf16
constexpr int UK = 16;   // K per tcgen05.mma kind::f16

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(smem_u32(b)), "r"(parity)
        : "memory");
  } while (!done);
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// UMMA shared-memory descriptor, K-major SWIZZLE_128B canonical layout (8 rows x 128 B atoms):
// start>>4 [0,14), LBO>>4 [16,30) (unused for SW128 K-major: 1), SBO>>4 [32,46) = 1024 B,
// version [46,48) = 1 (sm_100), layout [61,64) = 2 (SWIZZLE_128B).
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  uint64_t d = (uint64_t)((saddr & 0x3FFFFu) >> 4);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

__device__ __forceinline__ void mma_bf16(uint32_t tmem, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
      "l"(da), "l"(db), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

template <int BN, int STAGES>
struct Cfg {
  static constexpr uint32_t A_BYTES = BM * BK * 2;
  static constexpr uint32_t B_BYTES = BN * BK * 2;
  static constexpr uint32_t STAGE_BYTES = 2 * A_BYTES + 2 * B_BYTES;
  static constexpr uint32_t SMEM = STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;
  static constexpr uint32_t TMEM_COLS = BN < 32 ? 32 : BN;
  // instruction descriptor, kind::f16: D=F32 [4,6), A=BF16 [7,10), B=BF16 [10,13), K-major both,
  // N>>3 [17,23), M>>4 [24,29)
  static constexpr uint32_t IDESC =
      (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
};

template <int BN, int STAGES>
__global__ void __launch_bounds__(256, 1)
    gemm3_tc_kernel(const __grid_constant__ CUtensorMap mAh, const __grid_constant__ CUtensorMap mAl,
                    const __grid_constant__ CUtensorMap mBh, const __grid_constant__ CUtensorMap mBl,
                    float* __restrict__ C, int ldc, int M, int N, int K, float alpha) {
  using CF = Cfg<BN, STAGES>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * CF::STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* accf = empty + STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(accf + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  const int nk = (K + BK - 1) / BK;

  if (threadIdx.x == 0) {
#pragma unroll
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(accf, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mAh)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mBh)) : "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(CF::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0 && lane == 0) {
    // ---------------- TMA producer
    for (int kb = 0; kb < nk; ++kb) {
      const int s = kb % STAGES;
      const uint32_t ph = (kb / STAGES) & 1;
      mbar_wait(&empty[s], ph ^ 1);
      uint8_t* st = smem + s * CF::STAGE_BYTES;
      mbar_expect_tx(&full[s], CF::STAGE_BYTES);
      tma_load_2d(st, &mAh, kb * BK, m0, &full[s]);
      tma_load_2d(st + CF::A_BYTES, &mAl, kb * BK, m0, &full[s]);
      tma_load_2d(st + 2 * CF::A_BYTES, &mBh, kb * BK, n0, &full[s]);
      tma_load_2d(st + 2 * CF::A_BYTES + CF::B_BYTES, &mBl, kb * BK, n0, &full[s]);
    }
  } else if (warp == 1 && lane == 0) {
    // ---------------- MMA issuer (single thread)
    for (int kb = 0; kb < nk; ++kb) {
      const int s = kb % STAGES;
      const uint32_t ph = (kb / STAGES) & 1;
      mbar_wait(&full[s], ph);
      fence_after();
      const uint32_t base = smem_u32(smem + s * CF::STAGE_BYTES);
#pragma unroll
      for (int kk = 0; kk < BK / UK; ++kk) {
        const uint64_t dAh = sw128_desc(base + kk * 32);
        const uint64_t dAl = sw128_desc(base + CF::A_BYTES + kk * 32);
        const uint64_t dBh = sw128_desc(base + 2 * CF::A_BYTES + kk * 32);
        const uint64_t dBl = sw128_desc(base + 2 * CF::A_BYTES + CF::B_BYTES + kk * 32);
        mma_bf16(tmem, dAh, dBh, CF::IDESC, (kb | kk) != 0);
        mma_bf16(tmem, dAh, dBl, CF::IDESC, 1u);
        mma_bf16(tmem, dAl, dBh, CF::IDESC, 1u);
      }
      mma_commit(&empty[s]);  // frees the stage once these MMAs have read it
    }
    mma_commit(accf);  // accumulator complete
  } else if (warp >= 4) {
    // ---------------- epilogue: TMEM -> registers -> global (row = TMEM lane)
    mbar_wait(accf, 0);
    fence_after();
    const int ew = warp - 4;
    const int row = m0 + ew * 32 + lane;
    float* crow = C + (size_t)row * ldc;
#pragma unroll 1
    for (int c0 = 0; c0 < BN; c0 += 16) {
      uint32_t r[16];
      tmem_ld16(tmem + ((uint32_t)(ew * 32) << 16) + (uint32_t)c0, r);
      if (row < M) {
        const int col = n0 + c0;
        if (col + 16 <= N && ((reinterpret_cast<uintptr_t>(crow + col) & 15) == 0)) {
#pragma unroll
          for (int j = 0; j < 16; j += 4) {
            float4 v = make_float4(alpha * __uint_as_float(r[j]), alpha * __uint_as_float(r[j + 1]),
                                   alpha * __uint_as_float(r[j + 2]), alpha * __uint_as_float(r[j + 3]));
            *reinterpret_cast<float4*>(crow + col + j) = v;
          }
        } else {
#pragma unroll
          for (int j = 0; j < 16; ++j)
            if (col + j < N) crow[col + j] = alpha * __uint_as_float(r[j]);
        }
      }
    }
  }
  fence_before();
  __syncthreads();
  if (warp == 2) {
    fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(CF::TMEM_COLS));
  }
}

CUtensorMap make_map(void* encode_fn, const bf16* ptr, uint64_t inner, uint64_t outer, uint64_t ld, uint32_t box_outer) {
  CUtensorMap m;
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {ld * sizeof(bf16)};
  cuuint32_t box[2] = {(cuuint32_t)BK, box_outer};
  cuuint32_t estr[2] = {1, 1};
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(encode_fn);
  CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<bf16*>(ptr), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    fail(DHO2G_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ") inner=" + std::to_string(inner) +
                         " outer=" + std::to_string(outer) + " ld=" + std::to_string(ld));
  return m;
}

template <int BN, int STAGES>
void launch(dho2g_ctx* ctx, int M, int N, int K, const bf16* Ahi, const bf16* Alo, int lda, const bf16* Bhi,
            const bf16* Blo, int ldb, float* C, int ldc, float alpha) {
  using CF = Cfg<BN, STAGES>;
  static bool attr_set = false;
  if (!attr_set) {
    DHO2G_CUDA(cudaFuncSetAttribute(gemm3_tc_kernel<BN, STAGES>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)CF::SMEM));
    attr_set = true;
  }
  const CUtensorMap mAh = make_map(ctx->encode_fn, Ahi, K, M, lda, BM);
  const CUtensorMap mAl = make_map(ctx->encode_fn, Alo, K, M, lda, BM);
  const CUtensorMap mBh = make_map(ctx->encode_fn, Bhi, K, N, ldb, BN);
  const CUtensorMap mBl = make_map(ctx->encode_fn, Blo, K, N, ldb, BN);
  dim3 grid(cdiv(N, BN), cdiv(M, BM));
  gemm3_tc_kernel<BN, STAGES><<<grid, 256, CF::SMEM, ctx->stream>>>(mAh, mAl, mBh, mBl, C, ldc, M, N, K, alpha);
  DHO2G_LAUNCH();
}

}  // namespace tc

bool gemm3_tc(dho2g_ctx* ctx, int M, int N, int K, const bf16* Ahi, const bf16* Alo, int lda, const bf16* Bhi,
              const bf16* Blo, int ldb, float* C, int ldc, float alpha) {
  if (!ctx->encode_fn) fail(DHO2G_CUDA, "cuTensorMapEncodeTiled entry point unavailable");
  if ((lda % 8) || (ldb % 8) || (reinterpret_cast<uintptr_t>(Ahi) & 15) || (reinterpret_cast<uintptr_t>(Alo) & 15) ||
      (reinterpret_cast<uintptr_t>(Bhi) & 15) || (reinterpret_cast<uintptr_t>(Blo) & 15))
    fail(DHO2G_ARGUMENT, "gemm3_tc: operands must be 16-byte aligned with ld % 8 == 0");
  tc::launch<128, 3>(ctx, M, N, K, Ahi, Alo, lda, Bhi, Blo, ldb, C, ldc, alpha);
  return true;
}

void gemm3(dho2g_ctx* ctx, int M, int N, int K, const bf16* Ahi, const bf16* Alo, int lda, const bf16* Bhi,
           const bf16* Blo, int ldb, float* C, int ldc, float alpha) {
  if (M <= 0 || N <= 0) return;
  if (K <= 0) {
    DHO2G_CUDA(cudaMemset2DAsync(C, (size_t)ldc * sizeof(float), 0, (size_t)N * sizeof(float), M, ctx->stream));
    return;
  }
  ctx->bump("gemm_calls", 1);
  ctx->bump("gemm_flops_issued", 3.0 * 2.0 * double(M) * double(N) * double(K));
  const int slot = ctx->kt_begin();
  if (ctx->gemm_backend == 1)
    gemm3_simt(ctx->stream, M, N, K, Ahi, Alo, lda, Bhi, Blo, ldb, C, ldc, alpha);
  else
    gemm3_tc(ctx, M, N, K, Ahi, Alo, lda, Bhi, Blo, ldb, C, ldc, alpha);
  ctx->kt_end(slot, ctx->gemm_backend == 1 ? "gemm3_simt" : "gemm3_tcgen05", 2.0 * double(M) * double(N) * double(K));
}

}  // namespace dho2g
