// Ritz vectors on the tensor cores (extract_ese, reference dist_lanczos.cpp:121-158 / lanczos.cpp:96-120):
//
//     V_hat[:, c] = D[:, :me] U'[:, c]        D: rows x me fp32 (column-major basis), U': me x r
//
// as a tcgen05 kind::f16 GEMM on power-of-two-scaled fp16 (hi, lo) pairs (22 significant bits, the scheme of
// the MLP GEMMs, §5): basis column k is scaled by s_k = 2^(4 - round(log2(1 / (sigma_k sqrt(rows))))) (its
// entries' typical magnitude, from the lazy normalisation sigma_k, to ~16) and U' row k by usc / s_k, so
//     D U' = sum_k (D_k s_k)(U'_k usc / s_k) / usc       exactly (powers of two)
// and D U' ~= Dh Uh + Dh Ul + Dl Uh with fp32 accumulation in TMEM (dropped: Dl Ul, ~2^-22 relative).
// Round 2: the tf32 form (K = 8 per MMA, 12 MMAs per 32 basis columns) was bound by the tensor pipe's
// per-instruction cost at N = 32 (profiles/r02_ritz.txt: 0.55 of HBM; without the MMAs the same pipeline
// streams at HBM speed); kind::f16 takes K = 16 per MMA and 64-wide K-chunks: half the instructions.
//
// Persistent: one CTA per SM walks a contiguous range of 128-row tiles as one stream of 64-wide K-chunks:
// a ring of NCS 32 KB fp32 stages (TMA, 128 rows x 64 columns), a ring of NSL hi/lo fp16 slots (2 x 16 KB,
// K-major SWIZZLE_128B), two TMEM accumulators. Warp 0 TMA producer, warp 1 MMA issuer, warp 2 TMEM owner,
// warps 4-11 split (two groups of 4 warps on alternate chunks, one thread per row), warps 12-19 epilogue (two per TMEM lane quadrant, one per column half)
// (TMEM lane quadrant = warp % 4).
#include <cudaTypedefs.h>

#include "internal.h"
#include "tcgen05.cuh"

namespace dho2g {
namespace rtc {
using namespace tc;

constexpr int TM = 128;                     // rows per tile (UMMA M)
constexpr int KC = 64;                      // basis columns per K-chunk (one 128-byte fp16 row)
constexpr uint32_t CB = TM * KC * 4;        // one staged fp32 K-chunk (32 KB)
constexpr uint32_t HB = TM * KC * 2;        // one fp16 operand chunk, hi or lo (16 KB)
constexpr int kMaxStages = 6;
constexpr int kMaxSlots = 2;

struct Geo {
  int KP, NP;  // padded K (multiple of 64) and N (= r, 32 or 64)
  int NCS;     // fp32 staging ring depth (what is left of shared memory)
  int NSL;     // hi/lo chunk slots
  __host__ __device__ uint32_t ubytes() const { return (uint32_t)NP * KP * 2; }  // one U (hi or lo), fp16
  // stages, hi slots, lo slots, Uh, Ul, column scales, barriers
  __host__ __device__ uint32_t smem() const {
    return NCS * CB + 2 * NSL * HB + 2 * ubytes() + (uint32_t)KP * 4 + 1024 + 1024;
  }
};

inline Geo make_geo(int me, int r) {
  Geo g{(int)round_up((size_t)me, KC), r <= 32 ? 32 : 64, 0, kMaxSlots};
  const long long left = 227LL * 1024 - 2LL * g.NSL * HB - 2LL * g.ubytes() - (long long)g.KP * 4 - 2048;
  g.NCS = (int)std::max(0LL, std::min<long long>(kMaxStages, left / (long long)CB));
  return g;
}

// instruction descriptor, kind::f16: D=F32 [4,6), A=F16 [7,10) = 0, B=F16 [10,13) = 0, K-major both
__device__ __forceinline__ uint32_t idesc_f16(int N) {
  return (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(TM >> 4) << 24);
}

constexpr int kThreads = 640;  // 20 warps: producer, MMA, TMEM owner, idle, 8 split, 8 epilogue

__global__ void __launch_bounds__(kThreads, 1)
    ritz_tc_kernel(const __grid_constant__ CUtensorMap mD, const __grid_constant__ CUtensorMap mUh,
                   const __grid_constant__ CUtensorMap mUl, const float* __restrict__ colscale, float inv_usc, Geo g,
                   int me, int r, size_t rows, float* __restrict__ V, size_t ldv, int ntiles) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-byte aligned, derived from smem_raw by pointer arithmetic (the compiler keeps the shared address space)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const uint32_t UB = g.ubytes();
  const int NCS = g.NCS, NSL = g.NSL;
  uint8_t* stg0 = smem;               // [NCS] fp32 stages, [64 k][128 rows] (TMA, no swizzle)
  uint8_t* Ah = smem + NCS * CB;      // [NSL] hi chunk slots, fp16 K-major SW128 (128 rows x 128 B)
  uint8_t* Al = Ah + NSL * HB;        // [NSL] lo chunk slots
  uint8_t* Uh = Al + NSL * HB;        // fp16 K-major SW128: K-chunk kc at kc * NP * 128
  uint8_t* Ul = Uh + UB;
  float* csc = reinterpret_cast<float*>(Ul + UB);  // [KP] column scales
  uint64_t* bars = reinterpret_cast<uint64_t*>(csc + g.KP);
  uint64_t* full = bars;                     // [NCS] stage landed
  uint64_t* sfree = bars + kMaxStages;       // [NCS] stage consumed by the split
  uint64_t* tfull = sfree + kMaxStages;      // [2] accumulator ready
  uint64_t* tempty = tfull + 2;              // [2] accumulator drained
  uint64_t* ufull = tempty + 2;              // U landed
  uint64_t* hready = ufull + 1;              // [NSL] hi/lo slot written
  uint64_t* hfree = hready + kMaxSlots;      // [NSL] MMAs done reading that slot
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(hfree + kMaxSlots);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t tmem_cols = 2 * (uint32_t)g.NP;  // 64 or 128
  const int nkc = g.KP / KC;
  const int tpc = (ntiles + (int)gridDim.x - 1) / (int)gridDim.x;
  const int t0 = (int)blockIdx.x * tpc, t1 = min(ntiles, t0 + tpc);

  for (int k = threadIdx.x; k < g.KP; k += blockDim.x) csc[k] = colscale[k];
  if (threadIdx.x == 0) {
    for (int s = 0; s < NCS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&sfree[s], 8);  // the eight split warps
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], 8);  // eight epilogue warps
    }
    mbar_init(ufull, 1);
    for (int c = 0; c < kMaxSlots; ++c) {
      mbar_init(&hready[c], 8);
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

  if (warp == 0 && lane == 0) {
    // ---------------- producer: U (hi, lo) once, then the tiles' 128 x 64 K-chunks through the stage ring
    mbar_expect_tx(ufull, 2 * UB);
    for (int kc = 0; kc < nkc; ++kc) {
      tma_load_2d<false>(Uh + kc * g.NP * 128, &mUh, kc * KC, 0, ufull);
      tma_load_2d<false>(Ul + kc * g.NP * 128, &mUl, kc * KC, 0, ufull);
    }
    uint32_t it = 0;
    for (int t = t0; t < t1; ++t)
      for (int kc = 0; kc < nkc; ++kc, ++it) {
        const uint32_t s = it % NCS;
        mbar_wait(&sfree[s], ((it / NCS) & 1) ^ 1);
        mbar_expect_tx(&full[s], CB);
        tma_load_2d<false>(stg0 + s * CB, &mD, t * TM, kc * KC, &full[s]);
      }
  } else if (warp == 1 && lane == 0) {
    // ---------------- MMA issuer: Dh Uh + Dh Ul + Dl Uh, 4 k-steps of 16 per K-chunk, as soon as it is split
    const uint32_t ID = idesc_f16(g.NP);
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
        const int nks = min(KC, me - kc * KC + 15) / 16;  // k-steps holding basis columns (the rest is padding)
        for (int s4 = 0; s4 < nks; ++s4) {
          const uint32_t ao = h * HB + (uint32_t)s4 * 32u;
          const uint32_t uo = (uint32_t)kc * (uint32_t)g.NP * 128u + (uint32_t)s4 * 32u;
          const uint64_t aH = sw128_desc(ah + ao, 16, 1024), aL = sw128_desc(al + ao, 16, 1024);
          const uint64_t bH = sw128_desc(uh + uo, 16, 1024), bL = sw128_desc(ul + uo, 16, 1024);
          const uint32_t first = (kc > 0 || s4 > 0) ? 1u : 0u;
          asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(acc),
              "l"(aH), "l"(bH), "r"(ID), "r"(first));
          asm volatile("tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, 1;" ::"r"(acc), "l"(aH), "l"(bL),
                       "r"(ID));
          asm volatile("tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, 1;" ::"r"(acc), "l"(aL), "l"(bH),
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
    // ---------------- scale + split: all eight warps on every chunk, thread = row m; group grp takes the
    // odd or even 16-byte column slots, and only the slots the MMAs read (a short last chunk is trimmed)
    const int q = threadIdx.x - 128;  // 0..255
    const int grp = q >> 7, m = q & 127;
    const uint32_t rowoff = (uint32_t)(m >> 3) * 1024u + (uint32_t)(m & 7) * 128u;
    uint32_t it = 0;
    for (int t = t0; t < t1; ++t) {
      for (int kc = 0; kc < nkc; ++kc, ++it) {
        const int cmax = 2 * (min(KC, me - kc * KC + 15) / 16);  // valid 8-column slots
        const uint32_t s = it % NCS, h = it % NSL;
        mbar_wait(&full[s], (it / NCS) & 1);
        const float* stg = reinterpret_cast<const float*>(stg0 + s * CB);
        mbar_wait(&hfree[h], ((it / NSL) & 1) ^ 1);  // the MMAs of this slot's previous chunk are done
#pragma unroll
        for (int j = 0; j < KC / 16; ++j) {  // 16-byte slot c: 8 fp16 of columns 8c .. 8c+7
          const int c = 2 * j + grp;
          if (c >= cmax) break;
          uint32_t hw[4], lw[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) {  // pairs: one packed conversion each for hi and lo
            const int k0 = 8 * c + 2 * e;
            const float2 sc2 = *reinterpret_cast<const float2*>(&csc[kc * KC + k0]);
            const float2 x = make_float2(stg[k0 * TM + m] * sc2.x, stg[(k0 + 1) * TM + m] * sc2.y);
            const __half2 h2 = __float22half2_rn(x);
            const float2 hf = __half22float2(h2);
            const __half2 l2 = __float22half2_rn(make_float2(x.x - hf.x, x.y - hf.y));
            hw[e] = *reinterpret_cast<const uint32_t*>(&h2);
            lw[e] = *reinterpret_cast<const uint32_t*>(&l2);
          }
          const uint32_t off = h * HB + rowoff + (uint32_t)((c ^ (m & 7)) * 16);
          *reinterpret_cast<uint4*>(Ah + off) = make_uint4(hw[0], hw[1], hw[2], hw[3]);
          *reinterpret_cast<uint4*>(Al + off) = make_uint4(lw[0], lw[1], lw[2], lw[3]);
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
    // ---------------- epilogue: 8 warps, TMEM lane quadrant = warp % 4, column half = (warp - 12) / 4; undo U's
    // power-of-two scale
    const int sw = warp & 3, half = (warp - 12) >> 2;
    const int c0 = half * (g.NP / 2), c1 = c0 + g.NP / 2;
    uint32_t i = 0;
    for (int t = t0; t < t1; ++t, ++i) {
      const uint32_t ab = i & 1;
      mbar_wait(&tfull[ab], (i >> 1) & 1);
      fence_after();
      const size_t row = (size_t)t * TM + sw * 32 + lane;
      const uint32_t tb = tmem + ((uint32_t)(sw * 32) << 16) + ab * (uint32_t)g.NP;
      for (int cc = c0; cc < c1; cc += 16) {
        float v[16];
        tmem_ld16(tb + (uint32_t)cc, v);
        if (row < rows) {
#pragma unroll
          for (int j = 0; j < 16; ++j)
            if (cc + j < r) V[(size_t)(cc + j) * ldv + row] = v[j] * inv_usc;
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

// Column scales s_k (powers of two) from the lazy normalisation: D_k's entries are ~ 1 / (sigma_k sqrt(rows));
// U' (me x r, row-major, sigma folded) -> zero-padded fp16 K-major [NP][KP] hi / lo of U'[k][c] usc / s_k.
__global__ void u_split_kernel(const float* __restrict__ U, const float* __restrict__ sigma, int me, int r, int KP,
                               int NP, float lrows, float usc, __half* __restrict__ Uh, __half* __restrict__ Ul,
                               float* __restrict__ colscale) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < KP) {
    float s = 1.f;
    if (i < me) {
      const float sg = sigma[i];
      if (sg > 0.f && isfinite(sg)) s = exp2f(4.f - rintf(-log2f(sg) - 0.5f * lrows));
    }
    colscale[i] = s;
  }
  if (i >= KP * NP) return;
  const int c = i / KP, k = i % KP;
  float s = 1.f;
  if (k < me) {
    const float sg = sigma[k];
    if (sg > 0.f && isfinite(sg)) s = exp2f(4.f - rintf(-log2f(sg) - 0.5f * lrows));
  }
  const float x = (k < me && c < r) ? U[(size_t)k * r + c] * (usc / s) : 0.f;
  const __half hi = __float2half_rn(x);
  Uh[i] = hi;
  Ul[i] = __float2half_rn(x - __half2float(hi));
}

CUtensorMap map_2d(void* encode_fn, const void* ptr, CUtensorMapDataType dt, size_t esz, uint64_t inner,
                   uint64_t outer, uint64_t ld, uint32_t bi, uint32_t bo, CUtensorMapSwizzle sw) {
  CUtensorMap m;
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {ld * esz};
  cuuint32_t box[2] = {bi, bo};
  cuuint32_t estr[2] = {1, 1};
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(encode_fn);
  if (enc(&m, dt, 2, const_cast<void*>(ptr), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    fail(DHO2G_CUDA, "ritz_tc: cuTensorMapEncodeTiled failed");
  return m;
}

}  // namespace rtc

bool ritz_tc_supported(int me, int r) {
  if (me < 1 || r < 1 || r > 64) return false;
  const rtc::Geo g = rtc::make_geo(me, r);
  return g.KP <= 256 && g.NCS >= 2 && g.smem() <= 227 * 1024;
}

// V[:, 0:r] = D[:, 0:me] U' (U' device me x r row-major, sigma = the Lanczos sigma_j of the basis columns);
// rows < rows written, ldv / ldd chunk padded.
void ritz_tc(dho2g_ctx* ctx, const float* D, size_t ldd, int me, const float* U, const float* sigma, int r, float* V,
             size_t ldv, size_t rows, DevBuf<float>& uscratch) {
  using namespace rtc;
  if (!ctx->encode_fn) fail(DHO2G_CUDA, "cuTensorMapEncodeTiled entry point unavailable");
  const Geo g = make_geo(me, r);
  cudaStream_t st = ctx->stream;
  // fp16 Uh, Ul (KP x NP each) and the column scales (KP floats), in one float scratch
  uscratch.ensure((size_t)g.KP * g.NP + (size_t)g.KP);
  __half* Uh = reinterpret_cast<__half*>(uscratch.p);
  __half* Ul = Uh + (size_t)g.KP * g.NP;
  float* colscale = uscratch.p + (size_t)g.KP * g.NP;
  const float lrows = log2f((float)std::max<size_t>(rows, 1));
  const float usc = exp2f(14.f + rintf(0.5f * lrows));  // |U' usc / s_k| ~ 2^10 |Z| (|Z| <= 1)
  u_split_kernel<<<cdiv((size_t)g.KP * g.NP, 256), 256, 0, st>>>(U, sigma, me, r, g.KP, g.NP, lrows, usc, Uh, Ul,
                                                                  colscale);
  DHO2G_LAUNCH();
  // D: inner = rows, outer = basis columns (beyond me: zero fill); 128-row x 64-column boxes, no swizzle
  const CUtensorMap mD = map_2d(ctx->encode_fn, D, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, ldd, (uint64_t)me, ldd, TM, KC,
                                CU_TENSOR_MAP_SWIZZLE_NONE);
  // U hi / lo: fp16 K-major [NP][KP]; boxes of 64 K x NP rows, SWIZZLE_128B (the K-major canonical layout)
  const CUtensorMap mUh = map_2d(ctx->encode_fn, Uh, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, (uint64_t)g.KP,
                                 (uint64_t)g.NP, (uint64_t)g.KP, KC, (uint32_t)g.NP, CU_TENSOR_MAP_SWIZZLE_128B);
  const CUtensorMap mUl = map_2d(ctx->encode_fn, Ul, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, (uint64_t)g.KP,
                                 (uint64_t)g.NP, (uint64_t)g.KP, KC, (uint32_t)g.NP, CU_TENSOR_MAP_SWIZZLE_128B);
  const uint32_t smem = g.smem();
  static uint32_t smem_set = 0;
  if (smem > smem_set) {
    DHO2G_CUDA(cudaFuncSetAttribute(ritz_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    smem_set = smem;
  }
  const int ntiles = (int)(ldd / TM);
  const int grid = std::min(ntiles, ctx->sm_count);
  ritz_tc_kernel<<<grid, kThreads, smem, st>>>(mD, mUh, mUl, colscale, 1.f / usc, g, me, r, rows, V, ldv, ntiles);
  DHO2G_LAUNCH();
}

}  // namespace dho2g
