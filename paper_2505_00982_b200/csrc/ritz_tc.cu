// Ritz vectors on the tensor cores (extract_ese, reference dist_lanczos.cpp:121-158 / lanczos.cpp:96-120):
//
//     V_hat[:, c] = D[:, :me] U'[:, c]        D: rows x me fp32 (column-major basis), U': me x r
//
// as a tcgen05 kind::tf32 GEMM with a 3-term split (3xTF32): x = hi + lo with hi = x rounded to tf32
// and lo = x - hi rounded to tf32; D U' ~= Dh Uh + Dh Ul + Dl Uh with fp32 accumulation in TMEM
// (error ~2^-21 relative, the level of the fp32 CUDA-core kernel it replaces). A 128-row tile of the
// basis is brought in by one TMA (rows contiguous), and the split warps write hi / lo transposed into
// the K-major SWIZZLE_128B layout the MMA reads (16-byte chunks, conflict-free); U' is split on the host
// side of the launch and loaded K-major once per CTA. The r <= 64 Ritz columns leave through TMEM ->
// registers -> coalesced stores. The CUDA-core form is FMA/LDS-bound (2 rows.m.r FMAs); this one is
// HBM-bound.
//
// Persistent: one CTA per SM walks 128-row tiles as one stream of 32-wide K-chunks. The basis streams through
// a ring of NCS 16 KB K-chunk stages (128 rows x 32 columns, NCS = what shared memory leaves) and the split
// hi/lo operands through a ring of NSL chunk slots (2 x 16 KB each, 4 at C4), so the split runs up to NSL
// chunks ahead of the MMAs instead of alternating with them (round 2: 0.55 -> see DESIGN §9 of HBM at C4).
// Warp 0 TMA producer, warp 1 MMA issuer, warp 2 TMEM owner, warps 4-11 split (two threads per row), warps
// 12-15 epilogue (TMEM lane quadrant = warp % 4).
#include <cudaTypedefs.h>

#include "internal.h"
#include "tcgen05.cuh"

namespace dho2g {
namespace rtc {
using namespace tc;

constexpr int TM = 128;  // rows per tile (UMMA M)

constexpr uint32_t CB = TM * 32 * 4;  // one staged K-chunk: 128 rows x 32 basis columns fp32 (16 KB)
constexpr int kMaxStages = 8;
constexpr int kMaxSlots = 2;

struct Geo {
  int KP, NP;  // padded K (= me, multiple of 32) and N (= r, 32 or 64)
  int NCS;     // K-chunk staging ring depth (what is left of shared memory, <= kMaxStages)
  int NSL;     // hi/lo chunk slots (4, or 2 when U is large)
  __host__ __device__ uint32_t ubytes() const { return (uint32_t)NP * KP * 4; }  // one U (hi or lo)
  // chunk stages, hi slots, lo slots, Uh, Ul, barriers
  __host__ __device__ uint32_t smem() const { return NCS * CB + 2 * NSL * CB + 2 * ubytes() + 1024 + 1024; }
};

inline Geo make_geo(int me, int r) {
  Geo g{(int)round_up((size_t)me, 32), r <= 32 ? 32 : 64, 0, kMaxSlots};
  for (;;) {
    const long long left = 227LL * 1024 - 2LL * g.NSL * CB - 2LL * g.ubytes() - 2048;
    g.NCS = (int)std::max(0LL, std::min<long long>(kMaxStages, left / (long long)CB));
    if (g.NCS >= 2 || g.NSL <= 2) break;
    g.NSL = 2;
  }
  return g;
}

// Round to the nearest tf32 (10-bit mantissa) value, kept in an fp32 container. Both split terms are
// rounded (not truncated), so what the tensor core drops is centred: ~2^-22 relative per product,
// unbiased across the K sum.
__device__ __forceinline__ float rn_tf32(float x) {
  return __uint_as_float((__float_as_uint(x) + 0x1000u) & 0xFFFFE000u);
}

// instruction descriptor, kind::tf32: D=F32 [4,6), A=TF32 [7,10) = 2, B=TF32 [10,13) = 2, K-major both
__device__ __forceinline__ uint32_t idesc_tf32(int N) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(TM >> 4) << 24);
}

__global__ void __launch_bounds__(512, 1)
    ritz_tc_kernel(const __grid_constant__ CUtensorMap mD, const __grid_constant__ CUtensorMap mUh,
                   const __grid_constant__ CUtensorMap mUl, Geo g, int r, size_t rows, float* __restrict__ V,
                   size_t ldv, int ntiles) {
  extern __shared__ uint8_t smem_raw[];
  // 1024-byte aligned, derived from smem_raw by pointer arithmetic so that the compiler keeps the shared
  // address space (LDS / STS instead of generic loads and stores in the split)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const uint32_t UB = g.ubytes();
  const int NCS = g.NCS, NSL = g.NSL;
  uint8_t* stg0 = smem;               // [NCS] K-chunk stages, [32 k][128 rows] fp32 (TMA, no swizzle)
  uint8_t* Ah = smem + NCS * CB;      // [NSL] hi chunk slots, K-major SW128 (128 rows x 32 elems, 16 KB each)
  uint8_t* Al = Ah + NSL * CB;        // [NSL] lo chunk slots
  uint8_t* Uh = Al + NSL * CB;   // K-major SW128: K-chunk kc at kc * NP * 128
  uint8_t* Ul = Uh + UB;
  uint64_t* bars = reinterpret_cast<uint64_t*>(Ul + UB);
  uint64_t* full = bars;                     // [NCS] chunk stage landed
  uint64_t* sfree = bars + kMaxStages;       // [NCS] chunk stage consumed by the split
  uint64_t* tfull = sfree + kMaxStages;      // [2] accumulator ready
  uint64_t* tempty = tfull + 2;              // [2] accumulator drained
  uint64_t* ufull = tempty + 2;              // U landed
  uint64_t* hready = ufull + 1;              // [NSL] hi/lo chunk slot written
  uint64_t* hfree = hready + kMaxSlots;      // [NSL] MMAs done reading that slot
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(hfree + kMaxSlots);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t tmem_cols = 2 * (uint32_t)g.NP;  // 64 or 128
  const int nkc = g.KP / 32;

  if (threadIdx.x == 0) {
    for (int s = 0; s < NCS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&sfree[s], 4);  // one split group (4 warps) per chunk
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], 4);
    }
    mbar_init(ufull, 1);
    for (int c = 0; c < kMaxSlots; ++c) {
      mbar_init(&hready[c], 4);
      mbar_init(&hfree[c], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(tmem_cols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = *tmem_slot;
  // each CTA walks one contiguous range of row tiles (consecutive loads of a basis column are adjacent in
  // memory: longer DRAM bursts than a grid-strided walk)
  const int tpc = (ntiles + (int)gridDim.x - 1) / (int)gridDim.x;
  const int t0 = (int)blockIdx.x * tpc, t1 = min(ntiles, t0 + tpc);

  if (warp == 0 && lane == 0) {
    // ---------------- producer: U (hi, lo) once, then the tiles' 128 x 32 K-chunks through an NCS-deep ring
    // (up to NCS x 16 KB of the basis in flight per SM)
    mbar_expect_tx(ufull, 2 * UB);
    for (int kc = 0; kc < nkc; ++kc) {
      tma_load_2d<false>(Uh + kc * g.NP * 128, &mUh, kc * 32, 0, ufull);
      tma_load_2d<false>(Ul + kc * g.NP * 128, &mUl, kc * 32, 0, ufull);
    }
    uint32_t it = 0;
    for (int t = t0; t < t1; ++t)
      for (int kc = 0; kc < nkc; ++kc, ++it) {
        const uint32_t s = it % NCS;
        mbar_wait(&sfree[s], ((it / NCS) & 1) ^ 1);
        mbar_expect_tx(&full[s], CB);
        tma_load_2d<false>(stg0 + s * CB, &mD, t * TM, kc * 32, &full[s]);
      }
  } else if (warp == 1 && lane == 0) {
    // ---------------- MMA issuer: Dh Uh + Dh Ul + Dl Uh, one K-chunk (4 k-steps of 8) as soon as it is split
    const uint32_t ID = idesc_tf32(g.NP);
    mbar_wait(ufull, 0);
    fence_after();
    const uint32_t ah = smem_u32(Ah), al = smem_u32(Al), uh = smem_u32(Uh), ul = smem_u32(Ul);
    uint32_t i = 0, it = 0;
    for (int t = t0; t < t1; ++t, ++i) {
      const uint32_t ab = i & 1;
      mbar_wait(&tempty[ab], ((i >> 1) & 1) ^ 1);
      const uint32_t acc = tmem + ab * (uint32_t)g.NP;
      for (int kc = 0; kc < nkc; ++kc, ++it) {
        const uint32_t h = it % NSL;
        mbar_wait(&hready[h], (it / NSL) & 1);
        fence_after();
        for (int s4 = 0; s4 < 4; ++s4) {
          const uint32_t ao = h * CB + (uint32_t)s4 * 32u;
          const uint32_t uo = (uint32_t)kc * (uint32_t)g.NP * 128u + (uint32_t)s4 * 32u;
          const uint64_t aH = sw128_desc(ah + ao, 16, 1024), aL = sw128_desc(al + ao, 16, 1024);
          const uint64_t bH = sw128_desc(uh + uo, 16, 1024), bL = sw128_desc(ul + uo, 16, 1024);
          const uint32_t first = (kc > 0 || s4 > 0) ? 1u : 0u;
          asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(acc),
              "l"(aH), "l"(bH), "r"(ID), "r"(first));
          asm volatile("tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, 1;" ::"r"(acc), "l"(aH), "l"(bL),
                       "r"(ID));
          asm volatile("tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, 1;" ::"r"(acc), "l"(aL), "l"(bH),
                       "r"(ID));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                         smem_u32(&hfree[h]))
                     : "memory");
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                       smem_u32(&tfull[ab]))
                   : "memory");
    }
  } else if (warp >= 4 && warp < 12) {
    // ---------------- transpose-split: two groups of 4 warps take alternate chunks (two chunks in flight),
    // thread = row m, all 8 16-byte slots of the chunk's 128-byte row
    const int q = threadIdx.x - 128;  // 0..255
    const int grp = q >> 7, m = q & 127;
    const uint32_t rowoff = (uint32_t)(m >> 3) * 1024u + (uint32_t)(m & 7) * 128u;
    uint32_t it = 0;
    for (int t = t0; t < t1; ++t) {
      for (int kc = 0; kc < nkc; ++kc, ++it) {
        if ((int)(it & 1) != grp) continue;
        const uint32_t s = it % NCS, h = it % NSL;
        mbar_wait(&full[s], (it / NCS) & 1);
        const float* stg = reinterpret_cast<const float*>(stg0 + s * CB);
        mbar_wait(&hfree[h], ((it / NSL) & 1) ^ 1);  // the MMAs of this slot's previous chunk are done
        float x[32];
#pragma unroll
        for (int k = 0; k < 32; ++k) x[k] = stg[k * TM + m];
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const float4 hi = make_float4(rn_tf32(x[4 * c]), rn_tf32(x[4 * c + 1]), rn_tf32(x[4 * c + 2]),
                                        rn_tf32(x[4 * c + 3]));
          const uint32_t off = h * CB + rowoff + (uint32_t)((c ^ (m & 7)) * 16);
          *reinterpret_cast<float4*>(Ah + off) = hi;
          *reinterpret_cast<float4*>(Al + off) = make_float4(rn_tf32(x[4 * c] - hi.x), rn_tf32(x[4 * c + 1] - hi.y),
                                                             rn_tf32(x[4 * c + 2] - hi.z), rn_tf32(x[4 * c + 3] - hi.w));
        }
        // generic-proxy smem writes -> visible to the tensor core (async proxy)
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(&hready[h]);
          mbar_arrive(&sfree[s]);  // the stage is free for the next chunk load
        }
      }
    }
  } else if (warp >= 12) {
    // ---------------- epilogue: TMEM lane quadrant = warp % 4
    const int sw = warp & 3;
    uint32_t i = 0;
    for (int t = t0; t < t1; ++t, ++i) {
      const uint32_t ab = i & 1;
      mbar_wait(&tfull[ab], (i >> 1) & 1);
      fence_after();
      const size_t row = (size_t)t * TM + sw * 32 + lane;
      const uint32_t tb = tmem + ((uint32_t)(sw * 32) << 16) + ab * (uint32_t)g.NP;
      for (int cc = 0; cc < g.NP; cc += 16) {
        float v[16];
        tmem_ld16(tb + (uint32_t)cc, v);
        if (row < rows) {
#pragma unroll
          for (int j = 0; j < 16; ++j)
            if (cc + j < r) V[(size_t)(cc + j) * ldv + row] = v[j];
        }
      }
      fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[ab]);
    }
  }
  fence_before();
  __syncthreads();
  if (warp == 2) {
    fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(tmem_cols));
  }
}

// U' (me x r, row-major, sigma folded) -> zero-padded K-major [NP][KP] hi / lo (round-to-nearest tf32 split)
__global__ void u_split_kernel(const float* __restrict__ U, int me, int r, int KP, int NP, float* __restrict__ Uh,
                               float* __restrict__ Ul) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= KP * NP) return;
  const int c = i / KP, k = i % KP;
  const float x = (k < me && c < r) ? U[(size_t)k * r + c] : 0.f;
  const float hi = rtc::rn_tf32(x);
  Uh[i] = hi;
  Ul[i] = rtc::rn_tf32(x - hi);
}

CUtensorMap map_f32(void* encode_fn, const float* ptr, uint64_t inner, uint64_t outer, uint64_t ld, uint32_t bi,
                    uint32_t bo, CUtensorMapSwizzle sw) {
  CUtensorMap m;
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {ld * sizeof(float)};
  cuuint32_t box[2] = {bi, bo};
  cuuint32_t estr[2] = {1, 1};
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(encode_fn);
  if (enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(ptr), dims, strides, box, estr,
          CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    fail(DHO2G_CUDA, "ritz_tc: cuTensorMapEncodeTiled failed");
  return m;
}

}  // namespace rtc

bool ritz_tc_supported(int me, int r) {
  if (me < 1 || r < 1 || r > 64) return false;
  const rtc::Geo g = rtc::make_geo(me, r);
  return g.KP <= 256 && g.NCS >= 2 && g.smem() <= 227 * 1024;
}

// V[:, 0:r] = D[:, 0:me] U' (U' device me x r row-major); rows < rows written, ldv / ldd chunk padded.
void ritz_tc(dho2g_ctx* ctx, const float* D, size_t ldd, int me, const float* U, int r, float* V, size_t ldv,
             size_t rows, DevBuf<float>& uscratch) {
  using namespace rtc;
  if (!ctx->encode_fn) fail(DHO2G_CUDA, "cuTensorMapEncodeTiled entry point unavailable");
  const Geo g = make_geo(me, r);
  cudaStream_t st = ctx->stream;
  uscratch.ensure((size_t)2 * g.KP * g.NP);
  float* Uh = uscratch.p;
  float* Ul = uscratch.p + (size_t)g.KP * g.NP;
  u_split_kernel<<<cdiv((size_t)g.KP * g.NP, 256), 256, 0, st>>>(U, me, r, g.KP, g.NP, Uh, Ul);
  DHO2G_LAUNCH();
  // D: inner = rows, outer = basis columns (beyond me: zero fill); 128-row x 32-column boxes, no swizzle
  const CUtensorMap mD = map_f32(ctx->encode_fn, D, ldd, (uint64_t)me, ldd, TM, 32, CU_TENSOR_MAP_SWIZZLE_NONE);
  // U hi / lo: K-major [NP][KP]; boxes of 32 K x NP rows, SWIZZLE_128B (the K-major canonical layout)
  const CUtensorMap mUh = map_f32(ctx->encode_fn, Uh, (uint64_t)g.KP, (uint64_t)g.NP, (uint64_t)g.KP, 32, (uint32_t)g.NP,
                                  CU_TENSOR_MAP_SWIZZLE_128B);
  const CUtensorMap mUl = map_f32(ctx->encode_fn, Ul, (uint64_t)g.KP, (uint64_t)g.NP, (uint64_t)g.KP, 32, (uint32_t)g.NP,
                                  CU_TENSOR_MAP_SWIZZLE_128B);
  const uint32_t smem = g.smem();
  static uint32_t smem_set = 0;
  if (smem > smem_set) {
    DHO2G_CUDA(cudaFuncSetAttribute(ritz_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    smem_set = smem;
  }
  const int ntiles = (int)(ldd / TM);
  const int grid = std::min(ntiles, ctx->sm_count);
  ritz_tc_kernel<<<grid, 512, smem, st>>>(mD, mUh, mUl, g, r, rows, V, ldv, ntiles);
  DHO2G_LAUNCH();
}

}  // namespace dho2g
