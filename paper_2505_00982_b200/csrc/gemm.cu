// Split-BF16x3 GEMMs for the MLP contractions (HVP forward/R-forward, backward/R-backward,
// weight-gradient accumulation; SURVEY.md §2 kernel table):
//
//     acc[M x N] = Ah*Bh^T + Ah*Bl^T + Al*Bh^T,   A: M x K, B: N x K, both K-major (bf16 hi/lo)
//
// followed by a fused epilogue (Epi, internal.h): plain fp32 store (with the bias-column redirect
// used by the weight-gradient GEMMs) or the MLP layer epilogues — bias + tanh/relu (+ R-term),
// back-propagated delta (+ R-delta) — writing fp32 activations and the next GEMMs' bf16 hi/lo
// operands in both row-major and transposed layouts.
//
// gemm3_tc   : sm_100a persistent kernel. One CTA per SM walks a static work list of
//              (split, tile) units; a TMA producer warp streams A/B (hi, lo) tiles through a
//              3-stage mbarrier ring (SWIZZLE_128B); one elected thread issues tcgen05.mma
//              (kind::f16, M=128, N=128, FP32 accumulate) into one of two TMEM accumulators;
//              4 epilogue warps drain the other accumulator with tcgen05.ld (epilogue of unit
//              i overlaps the MMAs of unit i+1). Small-M GEMMs (the HVP at B=1024) are split
//              along K; the split partials are combined in a fixed order through a global
//              workspace + release/acquire flags, so results are deterministic.
// gemm3_simt : CUDA-core reference kernel with identical split arithmetic (fp32 FMA) + the same
//              epilogue device function, selectable via dho2g_ctx_set_option("gemm", 1).
#include <cudaTypedefs.h>

#include "internal.h"
#include "tcgen05.cuh"

namespace dho2g {

// =============================================================================== epilogue
__device__ __forceinline__ float act_prime(bool relu, float a) { return relu ? (a > 0.f ? 1.f : 0.f) : 1.f - a * a; }

// Inputs an element's epilogue reads besides the accumulator (split from the math so the
// warp-cooperative form can issue all of a block's loads before the first use).
struct EpiIn {
  float p0 = 0.f, p1 = 0.f, p2 = 0.f;
};
__device__ __forceinline__ EpiIn epi_load(const Epi& e, int row, int col) {
  EpiIn in;
  const size_t ei = (size_t)row * e.N + col;
  if (e.mode == EPI_STORE) return in;
  if (e.mode == EPI_FWD || e.mode == EPI_FWD_OUT) {
    if (e.do0) {
      in.p0 = __ldg(e.bias + col);
    } else {
      in.p0 = __ldg(e.vbias + col);
      if (e.mode == EPI_FWD) in.p1 = __ldg(e.a_in + ei);
    }
  } else {
    in.p1 = __ldg(e.a_in + ei);
    if (e.do1) {
      in.p0 = __ldg(e.u_in + ei);
      if (!e.relu) in.p2 = __ldg(e.ra_in + ei);
    }
  }
  return in;
}

// One output element (row < M, col < N): mode-specific math, fp32 side outputs and the row-major
// (hi, lo) pair; returns the value that goes to the transposed pair (0 when nothing does).
__device__ __forceinline__ float epi_elem(const Epi& e, int row, int col, float acc, float vsc, const EpiIn& in) {
  const size_t ei = (size_t)row * e.N + col;
  float v;
  if (e.mode == EPI_STORE) {
    v = e.alpha * acc;
    if (e.route) {
      const long long flat = e.route_flat0 + (long long)row * e.ldc + col;
      const long long q = flat / e.route_base;
      e.route[q][e.route_rank * e.route_base + (flat - q * e.route_base)] = v;
    } else if (e.bias_out && col == e.N - 1) {
      e.bias_out[row] = v;
    } else {
      e.C[(size_t)row * e.ldc + col] = v;
    }
    return 0.f;
  }
  if (e.mode == EPI_FWD || e.mode == EPI_FWD_OUT) {
    // oracle.cpp:548-563: a = act(z), z = W a + b ; ra = act'(a) (V a + W ra + v_b)
    if (e.do0) {
      const float z = acc + in.p0;
      v = e.mode == EPI_FWD_OUT ? z : (e.relu ? fmaxf(z, 0.f) : tanhf(z));
      if (e.f0) e.f0[ei] = v;
    } else {
      const float rz = acc + vsc * in.p0;
      v = e.mode == EPI_FWD_OUT ? rz : act_prime(e.relu, in.p1) * rz;
      if (e.f1) e.f1[ei] = v;
    }
  } else {  // EPI_BWD, oracle.cpp:626-635: d = u act'(a); rd = ru act'(a) + u (-2 a ra) (tanh)
    const float a = in.p1;
    const float ap = act_prime(e.relu, a);
    if (e.do0) {
      v = acc * ap;
      if (e.f0) e.f0[ei] = v;
      if (e.u_out) e.u_out[ei] = acc;
    } else {
      const float rap = (!e.relu && ap != 0.f) ? -2.f * a * in.p2 : 0.f;
      v = acc * ap + in.p0 * rap;
      if (e.f1) e.f1[ei] = v;
    }
  }
  if (e.Rh) {
    const size_t r = (size_t)row * (2 * e.P) + (size_t)e.hR * e.P + col;
    split_bf16(v, e.Rh[r], e.Rl[r]);
  }
  return v;
}

// Per-thread form (CUDA-core backend): 16 consecutive columns of one row; x receives the values.
__device__ __forceinline__ float acc_unscale(const Epi& e) { return e.sa ? 1.f / (*e.sa * *e.sb) : 1.f; }
__device__ __forceinline__ void amax_warp(const Epi& e, float m) {  // m >= 0 per lane
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0 && m > 0.f) atomicMax(e.amax, __float_as_uint(m));
}

__device__ __forceinline__ void epi_apply16(const Epi& e, int row, int col0, const float (&acc)[16], float (&x)[16]) {
  const float vsc = (e.do1 && e.vscale) ? *e.vscale : 1.f;
  const float inv = acc_unscale(e);
  float m = 0.f;
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    x[j] = (row < e.M && col0 + j < e.N) ? epi_elem(e, row, col0 + j, acc[j] * inv, vsc, epi_load(e, row, col0 + j))
                                         : 0.f;
    m = fmaxf(m, fabsf(x[j]));
  }
  if (e.amax && e.mode != EPI_STORE && m > 0.f) atomicMax(e.amax, __float_as_uint(m));
  if (e.mode != EPI_STORE && e.Th && row < e.Bp) {  // transposed pair; pad rows [M, Bp) get zeros
    const size_t base = (size_t)e.hT * e.Bp + row;
#pragma unroll
    for (int j = 0; j < 16; ++j)
      if (col0 + j < e.N) split_bf16(x[j], e.Th[(size_t)(col0 + j) * e.ldT + base], e.Tl[(size_t)(col0 + j) * e.ldT + base]);
  }
}

// Compile-time-mode forms used by the tcgen05 kernels (the mode is a template parameter of the kernel, so
// each epilogue compiles to its own straight-line code; the generic forms above serve the CUDA-core path).
template <int MODE>
__device__ __forceinline__ EpiIn epi_load_t(const Epi& e, int row, int col) {
  EpiIn in;
  const size_t ei = (size_t)row * e.N + col;
  if (MODE == EPI_FWD || MODE == EPI_FWD_OUT) {
    if (e.do0) {
      in.p0 = __ldg(e.bias + col);
    } else {
      in.p0 = __ldg(e.vbias + col);
      if (MODE == EPI_FWD) in.p1 = __ldg(e.a_in + ei);
    }
  } else if (MODE == EPI_BWD) {
    in.p1 = __ldg(e.a_in + ei);
    if (e.do1) {
      in.p0 = __ldg(e.u_in + ei);
      if (!e.relu) in.p2 = __ldg(e.ra_in + ei);
    }
  }
  return in;
}

template <int MODE>
__device__ __forceinline__ float epi_elem_t(const Epi& e, int row, int col, float acc, float vsc, const EpiIn& in) {
  const size_t ei = (size_t)row * e.N + col;
  float v;
  if (MODE == EPI_FWD || MODE == EPI_FWD_OUT) {
    // oracle.cpp:548-563: a = act(z), z = W a + b ; ra = act'(a) (V a + W ra + v_b)
    if (e.do0) {
      const float z = acc + in.p0;
      v = MODE == EPI_FWD_OUT ? z : (e.relu ? fmaxf(z, 0.f) : tanhf(z));
      if (e.f0) e.f0[ei] = v;
    } else {
      const float rz = acc + vsc * in.p0;
      v = MODE == EPI_FWD_OUT ? rz : act_prime(e.relu, in.p1) * rz;
      if (e.f1) e.f1[ei] = v;
    }
  } else {  // EPI_BWD, oracle.cpp:626-635: d = u act'(a); rd = ru act'(a) + u (-2 a ra) (tanh)
    const float a = in.p1;
    const float ap = act_prime(e.relu, a);
    if (e.do0) {
      v = acc * ap;
      if (e.f0) e.f0[ei] = v;
      if (e.u_out) e.u_out[ei] = acc;
    } else {
      const float rap = (!e.relu && ap != 0.f) ? -2.f * a * in.p2 : 0.f;
      v = acc * ap + in.p0 * rap;
      if (e.f1) e.f1[ei] = v;
    }
  }
  if (e.Rh) {
    const size_t r = (size_t)row * (2 * e.P) + (size_t)e.hR * e.P + col;
    split_bf16(v, e.Rh[r], e.Rl[r]);
  }
  return v;
}

// Warp-cooperative epilogue of a 32 x 16 accumulator block (lane l holds row row0 + l, columns
// [col0, col0 + 16)). EPI_STORE writes each lane's 64 contiguous bytes directly (four 16-byte stores);
// the layer epilogues restage the block through shared memory (sm: 32 x 17 floats) so that their
// row-major inputs / outputs / bf16 pairs are coalesced, and write the transposed pair from the
// lane = row layout.
// Forward epilogues without a transposed or pair-split output: lane = row, its 16 consecutive columns with
// vector loads and stores (64 contiguous bytes per row), no restage through shared memory.
// (Measured: R-forward 146 -> 137 us at C4. The backward epilogues read three arrays and write column sums:
// there lanes = rows cost 4x the L1 wavefronts of the restaged 2-row pattern and measured 5-23 % slower; they
// use 8-row x 16-byte vectors after the restage instead: R-backward 157-162 -> 147 us.)
template <int MODE>
__device__ __forceinline__ bool epi_lane_rows(const Epi& e, int col0) {
  return MODE == EPI_FWD && !e.Rh && !e.Th && !e.csum && col0 + 16 <= e.N && (e.N & 3) == 0;
}

// The layer epilogues' inputs of a 32 x 16 block (lane: rows row0 + 2 it + lane / 16, column col0 + lane % 16),
// loaded apart from the math so a caller can have them in flight with its accumulator reads.
template <int MODE>
__device__ __forceinline__ void epi_load_block(const Epi& e, int row0, int col0, EpiIn (&in)[16]) {
  if (MODE == EPI_STORE || epi_lane_rows<MODE>(e, col0)) return;
  if (MODE == EPI_BWD && !e.Rh && !e.Th && col0 + 16 <= e.N && (e.N & 3) == 0) return;  // (vector path)
  const int lane = threadIdx.x & 31;
  const int col = col0 + (lane & 15);
#pragma unroll
  for (int it = 0; it < 16; ++it) {
    const int row = row0 + 2 * it + (lane >> 4);
    if (row < e.M && col < e.N) in[it] = epi_load_t<MODE>(e, row, col);
  }
}
// L2 prefetch of one lane's row of a 32 x 128 epilogue block's inputs (4 lines of 128 bytes per array)
template <int MODE>
__device__ __forceinline__ void epi_prefetch_row(const Epi& e, int row, int col0) {
  if (MODE == EPI_STORE || row >= e.M) return;
  auto pf = [&](const float* base) {
    if (!base) return;
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if (col0 + 32 * q < e.N)
        asm volatile("prefetch.global.L2 [%0];" ::"l"(base + (size_t)row * e.N + col0 + 32 * q));
  };
  if (MODE == EPI_FWD) {
    if (!e.do0) pf(e.a_in);
  } else if (MODE == EPI_BWD) {
    pf(e.a_in);
    if (e.do1) {
      pf(e.u_in);
      if (!e.relu) pf(e.ra_in);
    }
  }
}

// mx_out: the lane's max |x| is folded into *mx_out instead of a per-block atomicMax on e.amax (the caller
// publishes one max per CTA: ~10^4 same-address atomics per launch serialised at the end of the R-GEMMs)
template <int MODE>
__device__ __forceinline__ void epi_warp16_t(const Epi& e, int row0, int col0, const float (&acc_in)[16], float* sm,
                                             const EpiIn (&in)[16], float* mx_out = nullptr);
template <int MODE>
__device__ __forceinline__ void epi_warp16_t(const Epi& e, int row0, int col0, const float (&acc_in)[16], float* sm) {
  EpiIn in[16];
  if (MODE != EPI_STORE) epi_load_block<MODE>(e, row0, col0, in);
  epi_warp16_t<MODE>(e, row0, col0, acc_in, sm, in);
}
template <int MODE>
__device__ __forceinline__ void epi_warp16_t(const Epi& e, int row0, int col0, const float (&acc_in)[16], float* sm,
                                             const EpiIn (&in)[16], float* mx_out) {
  const int lane = threadIdx.x & 31;
  float acc[16];
  const float inv = acc_unscale(e);
#pragma unroll
  for (int j = 0; j < 16; ++j) acc[j] = acc_in[j] * inv;
  if (MODE == EPI_BWD && !e.Rh && !e.Th && col0 + 16 <= e.N && (e.N & 3) == 0) {
    // Backward: restage the accumulator block through shared memory, then lane = (row 8 q + lane / 4,
    // columns 4 (lane % 4) .. + 3): 16-byte loads / stores of 8 rows x 64 bytes per instruction (4x fewer
    // memory instructions than the scalar 2-row pattern, the same lines). Same per-element arithmetic as
    // epi_elem_t.
#pragma unroll
    for (int j = 0; j < 16; ++j) sm[lane * 17 + j] = acc[j];
    __syncwarp();
    const int c4 = (lane & 3) * 4;
    float mx = 0.f;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int rl = 8 * q + (lane >> 2), row = row0 + rl;
      float xo[4] = {0.f, 0.f, 0.f, 0.f};
      if (row < e.M) {
        const size_t ei = (size_t)row * e.N + col0 + c4;
        const float4 a4 = __ldg(reinterpret_cast<const float4*>(e.a_in + ei));
        const float a[4] = {a4.x, a4.y, a4.z, a4.w};
        float ac[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) ac[j] = sm[rl * 17 + c4 + j];
        if (e.do0) {  // d = u act'(a)
#pragma unroll
          for (int j = 0; j < 4; ++j) xo[j] = ac[j] * act_prime(e.relu, a[j]);
          if (e.f0) *reinterpret_cast<float4*>(e.f0 + ei) = make_float4(xo[0], xo[1], xo[2], xo[3]);
          if (e.u_out) *reinterpret_cast<float4*>(e.u_out + ei) = make_float4(ac[0], ac[1], ac[2], ac[3]);
        } else {  // rd = ru act'(a) + u (-2 a ra) (tanh)
          const float4 u4 = __ldg(reinterpret_cast<const float4*>(e.u_in + ei));
          const float4 r4 = e.relu ? make_float4(0.f, 0.f, 0.f, 0.f) : __ldg(reinterpret_cast<const float4*>(e.ra_in + ei));
          const float u[4] = {u4.x, u4.y, u4.z, u4.w}, ra[4] = {r4.x, r4.y, r4.z, r4.w};
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const float ap = act_prime(e.relu, a[j]);
            const float rap = (!e.relu && ap != 0.f) ? -2.f * a[j] * ra[j] : 0.f;
            xo[j] = ac[j] * ap + u[j] * rap;
          }
          if (e.f1) *reinterpret_cast<float4*>(e.f1 + ei) = make_float4(xo[0], xo[1], xo[2], xo[3]);
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) mx = fmaxf(mx, fabsf(xo[j]));
      }
      if (e.csum) {
        __syncwarp();  // (every lane has read its accumulators of row rl before they are overwritten)
#pragma unroll
        for (int j = 0; j < 4; ++j) sm[rl * 17 + c4 + j] = xo[j];
      }
    }
    if (e.amax) {
      if (mx_out) *mx_out = fmaxf(*mx_out, mx);
      else amax_warp(e, mx);
    }
    __syncwarp();
    if (e.csum && row0 < e.M && lane < 16) {  // column sums of this 32-row block (rows >= M hold 0)
      float t = 0.f;
#pragma unroll 8
      for (int rl = 0; rl < 32; ++rl) t += sm[rl * 17 + lane];
      e.csum[(size_t)(row0 >> 5) * e.N + col0 + lane] = t;
    }
    __syncwarp();
    return;
  }
  if (MODE == EPI_FWD && epi_lane_rows<MODE>(e, col0)) {  // (the same per-element arithmetic as epi_elem_t)
    const int row = row0 + lane;
    float mx = 0.f;
    if (row < e.M) {
      const size_t base = (size_t)row * e.N + col0;
      float x[16];
      if (e.do0) {  // a = act(z), z = W a + b
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const float z = acc[j] + __ldg(e.bias + col0 + j);
          x[j] = e.relu ? fmaxf(z, 0.f) : tanhf(z);
        }
        if (e.f0)
#pragma unroll
          for (int q = 0; q < 4; ++q)
            *reinterpret_cast<float4*>(e.f0 + base + 4 * q) = make_float4(x[4 * q], x[4 * q + 1], x[4 * q + 2], x[4 * q + 3]);
      } else {  // ra = act'(a) (V a + W ra + v_b)
        const float vsc = e.vscale ? *e.vscale : 1.f;
        float a[16];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float4 t = __ldg(reinterpret_cast<const float4*>(e.a_in + base) + q);
          a[4 * q] = t.x; a[4 * q + 1] = t.y; a[4 * q + 2] = t.z; a[4 * q + 3] = t.w;
        }
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const float rz = acc[j] + vsc * __ldg(e.vbias + col0 + j);
          x[j] = act_prime(e.relu, a[j]) * rz;
        }
        if (e.f1)
#pragma unroll
          for (int q = 0; q < 4; ++q)
            *reinterpret_cast<float4*>(e.f1 + base + 4 * q) = make_float4(x[4 * q], x[4 * q + 1], x[4 * q + 2], x[4 * q + 3]);
      }
#pragma unroll
      for (int j = 0; j < 16; ++j) mx = fmaxf(mx, fabsf(x[j]));
    }
    if (e.amax) {
      if (mx_out) *mx_out = fmaxf(*mx_out, mx);
      else amax_warp(e, mx);
    }
    return;
  }
  if (MODE == EPI_STORE) {
    const int row = row0 + lane;
    if (row >= e.M) return;
    if (e.route) {  // fused reduce-scatter: each element straight into its owner's slot for this rank
      const long long f0 = e.route_flat0 + (long long)row * e.ldc + col0;
      long long q = f0 / e.route_base;
      long long edge = (q + 1) * e.route_base;  // a 16-element run crosses at most one shard edge
      float* dst = e.route[q] + e.route_rank * e.route_base - q * e.route_base;
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        if (col0 + j >= e.N) break;
        const long long f = f0 + j;
        if (f >= edge) {
          ++q;
          edge += e.route_base;
          dst = e.route[q] + e.route_rank * e.route_base - q * e.route_base;
        }
        dst[f] = e.alpha * acc[j];
      }
      return;
    }
    float* c = e.C + (size_t)row * e.ldc + col0;
    if (!e.bias_out && col0 + 16 <= e.N && (reinterpret_cast<uintptr_t>(c) & 15) == 0) {
#pragma unroll
      for (int q = 0; q < 4; ++q)
        *reinterpret_cast<float4*>(c + 4 * q) =
            make_float4(e.alpha * acc[4 * q], e.alpha * acc[4 * q + 1], e.alpha * acc[4 * q + 2], e.alpha * acc[4 * q + 3]);
    } else {
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        if (col0 + j >= e.N) break;
        const float v = e.alpha * acc[j];
        if (e.bias_out && col0 + j == e.N - 1) e.bias_out[row] = v;
        else c[j] = v;
      }
    }
    return;
  }
  const float vsc = (e.do1 && e.vscale) ? *e.vscale : 1.f;
#pragma unroll
  for (int j = 0; j < 16; ++j) sm[lane * 17 + j] = acc[j];
  __syncwarp();
  const int rr = lane >> 4, cc = lane & 15;
  const int col = col0 + cc;
  float mx = 0.f;
#pragma unroll
  for (int it = 0; it < 16; ++it) {
    const int rl = 2 * it + rr;
    const int row = row0 + rl;
    float x = 0.f;
    if (row < e.M && col < e.N) x = epi_elem_t<MODE>(e, row, col, sm[rl * 17 + cc], vsc, in[it]);
    sm[rl * 17 + cc] = x;
    mx = fmaxf(mx, fabsf(x));
  }
  if (e.amax) {
    if (mx_out) *mx_out = fmaxf(*mx_out, mx);
    else amax_warp(e, mx);
  }
  __syncwarp();
  if (e.csum && row0 < e.M && lane < 16 && col0 + lane < e.N) {  // column sums of this 32-row block (rows >= M hold 0)
    float t = 0.f;
#pragma unroll 8
    for (int rl = 0; rl < 32; ++rl) t += sm[rl * 17 + lane];
    e.csum[(size_t)(row0 >> 5) * e.N + col0 + lane] = t;
  }
  if (e.Th) {
    const int row = row0 + lane;
    if (row < e.Bp) {
      const size_t base = (size_t)e.hT * e.Bp + row;
#pragma unroll
      for (int j = 0; j < 16; ++j)
        if (col0 + j < e.N) split_bf16(sm[lane * 17 + j], e.Th[(size_t)(col0 + j) * e.ldT + base],
                                       e.Tl[(size_t)(col0 + j) * e.ldT + base]);
    }
  }
  __syncwarp();
}

namespace {
// standalone epilogue over an fp32 accumulator matrix (CUDA-core backend)
// blockDim (8, 32): 32 rows x 128 columns per block, so the 32-row column sums are a block reduction
__global__ void epi_kernel(Epi e, const float* __restrict__ acc, int ldacc, int rows_pad) {
  __shared__ float red[32][129];
  const int row = blockIdx.y * blockDim.y + threadIdx.y;
  const int col0 = (blockIdx.x * blockDim.x + threadIdx.x) * 16;
  float x[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) x[j] = 0.f;
  if (row < rows_pad && col0 < e.N) {
    float v[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) v[j] = (row < e.M && col0 + j < e.N) ? acc[(size_t)row * ldacc + col0 + j] : 0.f;
    epi_apply16(e, row, col0, v, x);
  }
  if (!e.csum || (int)(blockIdx.y * blockDim.y) >= e.M) return;
#pragma unroll
  for (int j = 0; j < 16; ++j) red[threadIdx.y][threadIdx.x * 16 + j] = (row < e.M) ? x[j] : 0.f;
  __syncthreads();
  if (threadIdx.y == 0) {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      if (col0 + j >= e.N) break;
      float t = 0.f;
      for (int rl = 0; rl < 32; ++rl) t += red[rl][threadIdx.x * 16 + j];
      e.csum[(size_t)blockIdx.y * e.N + col0 + j] = t;
    }
  }
}
}  // namespace

// =============================================================================== operand windows
__host__ __device__ __forceinline__ void gop_coord(const GOp& op, int mn, int k, int kseg, int& in, int& out) {
  const int seg = k >= kseg ? 1 : 0;
  const int kk = k - (seg ? kseg : 0);
  if (op.mn_major) {
    in = mn + op.off_in[seg];
    out = kk + op.off_out[seg];
  } else {
    in = kk + op.off_in[seg];
    out = mn + op.off_out[seg];
  }
}

GOp gop_k(const bf16* hi, const bf16* lo, int ld, int K, int rows) {
  GOp g{};
  g.hi = hi;
  g.lo = lo;
  g.ld = ld;
  g.mn_major = 0;
  g.inner = K;
  g.outer = rows;
  return g;
}

// =============================================================================== CUDA-core path
namespace {
constexpr int ST_BM = 64, ST_BN = 64, ST_BK = 16;

__device__ __forceinline__ void gop_load(const GOp& op, int mn, int MN, int k, int K, int kseg, float& h, float& l) {
  h = l = 0.f;
  if (mn >= MN || k >= K) return;
  int in, out;
  gop_coord(op, mn, k, kseg, in, out);
  if (in < 0 || in >= op.inner || out < 0 || out >= op.outer) return;
  const size_t i = (size_t)out * op.ld + in;
  if (op.f16) {
    h = f16_bits_to_float(op.hi[i]);
    l = f16_bits_to_float(op.lo[i]);
  } else {
    h = __bfloat162float(op.hi[i]);
    l = __bfloat162float(op.lo[i]);
  }
}

__global__ void __launch_bounds__(256) gemm3_simt_kernel(int M, int N, int K, int kseg, const GOp A, const GOp B,
                                                         float* __restrict__ C, int ldc) {
  __shared__ float sAh[ST_BK][ST_BM + 4], sAl[ST_BK][ST_BM + 4], sBh[ST_BK][ST_BN + 4], sBl[ST_BK][ST_BN + 4];
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  const int m0 = blockIdx.y * ST_BM, n0 = blockIdx.x * ST_BN;
  float acc[4][4] = {};
  for (int k0 = 0; k0 < K; k0 += ST_BK) {
    for (int e = threadIdx.x; e < ST_BM * ST_BK; e += 256) {
      const int r = e / ST_BK, kk = e % ST_BK;
      gop_load(A, m0 + r, M, k0 + kk, K, kseg, sAh[kk][r], sAl[kk][r]);
      gop_load(B, n0 + r, N, k0 + kk, K, kseg, sBh[kk][r], sBl[kk][r]);
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
      if (gn < N) C[(size_t)gm * ldc + gn] = acc[i][j];
    }
  }
}
}  // namespace

static void gemm3_simt(dho2g_ctx* ctx, int M, int N, int K, int kseg, const GOp& A, const GOp& B, const Epi& e) {
  ctx->simt_ws.ensure_g((size_t)M * N + 16);
  float* acc = ctx->simt_ws.p;
  dim3 grid(cdiv(N, ST_BN), cdiv(M, ST_BM));
  gemm3_simt_kernel<<<grid, 256, 0, ctx->stream>>>(M, N, K, kseg, A, B, acc, N);
  DHO2G_LAUNCH();
  const int rows_pad = e.mode == EPI_STORE ? M : std::max(M, e.Bp);
  dim3 eb(8, 32);
  dim3 eg(cdiv(cdiv(N, 16), 8), cdiv(rows_pad, 32));
  epi_kernel<<<eg, eb, 0, ctx->stream>>>(e, acc, N, rows_pad);
  DHO2G_LAUNCH();
}

// =============================================================================== tcgen05 common
namespace tc {

constexpr int BK = 64;   // one 128-byte swizzle row of bf16 (K-major) / 64 K-rows per stage (MN-major)
constexpr int UK = 16;   // K per tcgen05.mma kind::f16
constexpr int ACC = 2;   // TMEM accumulator buffers
constexpr uint32_t OP_BYTES = 128 * BK * 2;      // one 128-row (hi or lo) operand tile
constexpr uint32_t EPI_SMEM = 8 * 32 * 17 * 4;  // per epilogue warp: 32 x 16 restaging block (+1 pad)
// instruction descriptor, kind::f16: D=F32 [4,6), A=BF16 [7,10), B=BF16 [10,13), A/B major [15], [16],
// N>>3 [17,23), M>>4 [24,29)
__host__ __device__ constexpr uint32_t idesc(int M, int N, bool amn, bool bmn) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((amn ? 1u : 0u) << 15) | ((bmn ? 1u : 0u) << 16) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
// the same with F16 operands (A / B format fields 0) for the scaled-fp16 pairs
__host__ __device__ constexpr uint32_t idesc_fmt(uint32_t id, bool f16) {
  return f16 ? (id & ~((7u << 7) | (7u << 10))) : id;
}

struct OpOff {  // per-segment coordinate offsets of one operand (GOp minus pointers / extents)
  int off_in[2], off_out[2];
};
inline OpOff op_off(const GOp& g) {
  OpOff o;
  for (int s = 0; s < 2; ++s) {
    o.off_in[s] = g.off_in[s];
    o.off_out[s] = g.off_out[s];
  }
  return o;
}

// Descriptor of the kk-th K=16 slice of a staged operand tile whose stage depth is BKT K-elements:
//  MN-major: panels of 64 MN x BKT K-rows (128-byte rows, SW128): LBO = panel stride = BKT * 128 B,
//            SBO = 1024 B, slice kk at +2 KB * kk;
//  K-major, BKT = 64: 128-byte rows (SW128), SBO = 1024 B, slice at +32 B * kk;
//  K-major, BKT = 32: 64-byte rows (SW64, layout 4), SBO = 512 B, slice at +32 B * kk.
template <bool MN, int BKT = 64>
__device__ __forceinline__ uint64_t op_desc(uint32_t tile_base, int kk) {
  if (MN) return sw128_desc(tile_base + kk * 2048, BKT * 128, 1024);
  if (BKT == 64) return sw128_desc(tile_base + kk * 32, 16, 1024);
  return umma_desc(tile_base + kk * 32, 16, 512, 4);
}

// Stage one 128-row (M or N) x 64-K operand tile (hi or lo) into smem through its map.
// PANELS2: 2 = 128 MN rows (MN-major: two 64-wide boxes), 1 = 64 rows (the B half of a 128-wide pair tile;
// K-major maps are then built with 64-row boxes).
template <bool MN, bool PAIR, int PANELS2 = 2, int BKT = 64>
__device__ __forceinline__ void load_op(uint8_t* dst, const CUtensorMap* map, const OpOff& o, int mn0, int kb,
                                        int kseg, uint64_t* bar) {
  const int k = kb * BKT;
  const int seg = k >= kseg ? 1 : 0;
  const int kk = k - (seg ? kseg : 0);
  if (MN) {  // 64(MN) x BKT(K) boxes
    tma_load_2d<PAIR>(dst, map, mn0 + o.off_in[seg], kk + o.off_out[seg], bar);
    if (PANELS2 == 2) tma_load_2d<PAIR>(dst + BKT * 128, map, mn0 + 64 + o.off_in[seg], kk + o.off_out[seg], bar);
  } else {  // one BKT(K) x (64 PANELS2)(MN) box
    tma_load_2d<PAIR>(dst, map, kk + o.off_in[seg], mn0 + o.off_out[seg], bar);
  }
}

CUtensorMap make_map(void* encode_fn, const bf16* ptr, uint64_t inner, uint64_t outer, uint64_t ld, uint32_t box_inner,
                     uint32_t box_outer, CUtensorMapSwizzle sw = CU_TENSOR_MAP_SWIZZLE_128B) {
  CUtensorMap m;
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {ld * sizeof(bf16)};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(encode_fn);
  CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<bf16*>(ptr), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    fail(DHO2G_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ") inner=" + std::to_string(inner) +
                         " outer=" + std::to_string(outer) + " ld=" + std::to_string(ld));
  return m;
}
// hi / lo maps of one operand: K-major boxes bk(K) x rows (SW128 for bk = 64, SW64 for bk = 32),
// MN-major boxes 64(MN) x bk(K) (SW128)
void op_maps(void* encode_fn, const GOp& g, CUtensorMap& mh, CUtensorMap& ml, uint32_t rows = 128, uint32_t bk = 64) {
  const uint32_t bi = g.mn_major ? 64 : bk, bo = g.mn_major ? bk : rows;
  const CUtensorMapSwizzle sw = (!g.mn_major && bk == 32) ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B;
  mh = make_map(encode_fn, g.hi, (uint64_t)g.inner, (uint64_t)g.outer, (uint64_t)g.ld, bi, bo, sw);
  ml = make_map(encode_fn, g.lo, (uint64_t)g.inner, (uint64_t)g.outer, (uint64_t)g.ld, bi, bo, sw);
}
void check_op(const GOp& g, const char* what) {
  auto al16 = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  if ((g.ld % 8) || !al16(g.hi) || !al16(g.lo))
    fail(DHO2G_ARGUMENT, std::string("gemm3: operand ") + what + " must be 16-byte aligned with ld % 8 == 0");
  if (g.inner <= 0 || g.outer <= 0) fail(DHO2G_ARGUMENT, std::string("gemm3: empty operand window ") + what);
}

}  // namespace tc

// =============================================================================== single-CTA kernel
// One CTA per SM walks a static work list of (split, tile) units (128 x 128 tiles). A TMA producer
// warp streams A/B (hi, lo) tiles through a 3-stage mbarrier ring; one elected thread issues
// tcgen05.mma (M = 128, N = 128) into one of two TMEM accumulators; 8 epilogue warps drain the other
// (epilogue of unit i overlaps the MMAs of unit i+1). Small-M GEMMs are split along K; split
// partials are combined in a fixed order through a global workspace + release/acquire flags.
namespace tc1 {
using namespace tc;
constexpr size_t kTc1Tickets = 4096;  // offset of the split-K tickets in ctx->gemm_flags
// Optional per-CTA timeline (test hook, investigation only): globaltimer ns at [0] entry, [1] setup done,
// [2] first stage landed (MMA thread), [3] last MMA committed, [4] final accumulator ready (epilogue),
// [5] epilogue done, [6] CTA joined, [7] TMEM freed.
__device__ unsigned long long* g_tc1_trace = nullptr;
__device__ __forceinline__ unsigned long long gtimer1() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
constexpr int BM = 128, BN = 128, STAGES = 3;
constexpr uint32_t STAGE_BYTES = 4 * OP_BYTES;
constexpr uint32_t SMEM = STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/ + EPI_SMEM;
constexpr uint32_t TMEM_COLS = 4 * BN;  // two accumulators + the chunked-accumulation running sum (+ spare)
constexpr uint32_t SUM_COL = ACC * BN;

struct Sched {
  int mt, nt, tiles, splits, units, nkb, kseg;  // nkb: k-blocks total
  int chunk;  // k-blocks per TMEM accumulation chunk (drained into an fp32 running sum), >= unit length: off
  __device__ __forceinline__ void unit(int u, int& m0, int& n0, int& split, int& tile, int& kb0, int& kb1) const {
    split = u / tiles;
    tile = u - split * tiles;
    m0 = (tile / nt) * BM;  // row-major tile order: consecutive CTAs share the A rows
    n0 = (tile % nt) * BN;
    kb0 = (int)((long long)nkb * split / splits);
    kb1 = (int)((long long)nkb * (split + 1) / splits);
  }
};

template <bool AMN, bool BMN, int MODE>
__global__ void __launch_bounds__(384, 1)
    gemm3_tc_kernel(const __grid_constant__ CUtensorMap mAh, const __grid_constant__ CUtensorMap mAl,
                    const __grid_constant__ CUtensorMap mBh, const __grid_constant__ CUtensorMap mBl, Sched sc,
                    OpOff oa, OpOff ob, const __grid_constant__ Epi e, float* __restrict__ ws,
                    unsigned* __restrict__ flags, unsigned epoch) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;  // [ACC]
  uint64_t* tempty = tfull + ACC;    // [ACC]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + ACC);
  __shared__ int s_last;
  __shared__ float s_mx1[8];  // epilogue warps' max |x| (one e.amax update per CTA)
  unsigned long long* trace = g_tc1_trace ? g_tc1_trace + (size_t)blockIdx.x * 8 : nullptr;
  if (trace && threadIdx.x == 0) trace[0] = gtimer1();

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
#pragma unroll
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
#pragma unroll
    for (int a = 0; a < ACC; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 8);  // one arrive per epilogue warp
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mAh)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mAl)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mBh)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mBl)) : "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = *tmem_slot;
  if (trace && threadIdx.x == 0) trace[1] = gtimer1();

  if (warp == 0 && lane == 0) {
    // ---------------- TMA producer: continuous ring over all k-blocks of this CTA's units
    uint32_t it = 0;
    for (int u = blockIdx.x; u < sc.units; u += gridDim.x) {
      int m0, n0, split, tile, kb0, kb1;
      sc.unit(u, m0, n0, split, tile, kb0, kb1);
      for (int kb = kb0; kb < kb1; ++kb, ++it) {
        const int s = it % STAGES;
        mbar_wait(&empty[s], ((it / STAGES) & 1) ^ 1);
        uint8_t* st = smem + s * STAGE_BYTES;
        mbar_expect_tx(&full[s], STAGE_BYTES);
        load_op<AMN, false>(st, &mAh, oa, m0, kb, sc.kseg, &full[s]);
        load_op<AMN, false>(st + OP_BYTES, &mAl, oa, m0, kb, sc.kseg, &full[s]);
        load_op<BMN, false>(st + 2 * OP_BYTES, &mBh, ob, n0, kb, sc.kseg, &full[s]);
        load_op<BMN, false>(st + 3 * OP_BYTES, &mBl, ob, n0, kb, sc.kseg, &full[s]);
      }
    }
  } else if (warp == 1 && lane == 0) {
    // ---------------- MMA issuer (single thread), accumulator double-buffered in TMEM
    const uint32_t ID = idesc_fmt(idesc(BM, BN, AMN, BMN), e.f16 != 0);
    uint32_t it = 0, uc = 0;
    for (int u = blockIdx.x; u < sc.units; u += gridDim.x) {
      int m0, n0, split, tile, kb0, kb1;
      sc.unit(u, m0, n0, split, tile, kb0, kb1);
     for (int c0 = kb0; c0 < kb1 || c0 == kb0; c0 += sc.chunk, ++uc) {  // one accumulator per chunk
      const int c1 = min(kb1, c0 + sc.chunk);
      const uint32_t ab = uc % ACC;
      mbar_wait(&tempty[ab], ((uc / ACC) & 1) ^ 1);  // epilogue drained this buffer
      fence_after();
      const uint32_t acc_addr = tmem + ab * BN;
      for (int kb = c0; kb < c1; ++kb, ++it) {
        const int s = it % STAGES;
        mbar_wait(&full[s], (it / STAGES) & 1);
        fence_after();
        if (trace && it == 0) trace[2] = gtimer1();
        const uint32_t base = smem_u32(smem + s * STAGE_BYTES);
#pragma unroll
        for (int kk = 0; kk < BK / UK; ++kk) {
          const uint64_t dAh = op_desc<AMN>(base, kk);
          const uint64_t dAl = op_desc<AMN>(base + OP_BYTES, kk);
          const uint64_t dBh = op_desc<BMN>(base + 2 * OP_BYTES, kk);
          const uint64_t dBl = op_desc<BMN>(base + 3 * OP_BYTES, kk);
          const uint32_t first = (kb > c0 || kk > 0) ? 1u : 0u;
          asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(acc_addr),
              "l"(dAh), "l"(dBh), "r"(ID), "r"(first));
          asm volatile("tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, 1;" ::"r"(acc_addr), "l"(dAh), "l"(dBl),
                       "r"(ID));
          asm volatile("tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, 1;" ::"r"(acc_addr), "l"(dAl), "l"(dBh),
                       "r"(ID));
        }
        // frees the stage once these MMAs have read it
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                         smem_u32(&empty[s]))
                     : "memory");
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                       smem_u32(&tfull[ab]))
                   : "memory");  // accumulator ready for the epilogue
     }
    }
    if (trace) trace[3] = gtimer1();
  } else if (warp >= 4) {
    // ---------------- epilogue warps: TMEM -> registers -> (split-K combine) -> fused epilogue
    // 8 warps: warp w reads TMEM lane quadrant w % 4 (hardware rule) and column half (w - 4) / 4.
    const int ew = warp & 3;
    const int chalf = (warp - 4) >> 2;
    float* esm = reinterpret_cast<float*>(smem + STAGES * STAGE_BYTES + 256) + (warp - 4) * (32 * 17);
    uint32_t uc = 0;
    float wmx = 0.f;  // this lane's max |x| over all its units (one e.amax update per CTA, at the end)
    const uint32_t tsum = tmem + ((uint32_t)(ew * 32) << 16) + SUM_COL;  // chunk running sum (TMEM)
    for (int u = blockIdx.x; u < sc.units; u += gridDim.x, ++uc) {
      int m0, n0, split, tile, kb0, kb1;
      sc.unit(u, m0, n0, split, tile, kb0, kb1);
      // chunks before the last: running sum (TMEM) += chunk (round-to-nearest fp32), free the accumulator
      const int nchunks = kb1 > kb0 ? (kb1 - kb0 + sc.chunk - 1) / sc.chunk : 1;
      for (int c = 0; c + 1 < nchunks; ++c, ++uc) {
        const uint32_t ab = uc % ACC;
        mbar_wait(&tfull[ab], (uc / ACC) & 1);
        fence_after();
        const uint32_t tb = tmem + ((uint32_t)(ew * 32) << 16) + ab * BN;
#pragma unroll 1
        for (int c0 = chalf * (BN / 2); c0 < (chalf + 1) * (BN / 2); c0 += 32)
          tmem_drain32(tb + (uint32_t)c0, tsum + (uint32_t)c0, c > 0);
        tmem_wait_st();
        fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[ab]);
      }
      const uint32_t ab = uc % ACC;
      mbar_wait(&tfull[ab], (uc / ACC) & 1);
      fence_after();
      if (trace && threadIdx.x == 128) trace[4] = gtimer1();
      const uint32_t tbase = tmem + ((uint32_t)(ew * 32) << 16) + ab * BN;
      auto acc16 = [&](int c0, float (&v)[16]) {  // this unit's sum: TMEM chunk (+ the earlier chunks)
        tmem_ld16(tbase + (uint32_t)c0, v);
        if (nchunks > 1) {
          float t[16];
          tmem_ld16(tsum + (uint32_t)c0, t);
#pragma unroll
          for (int j = 0; j < 16; ++j) v[j] += t[j];
        }
      };
      if (sc.splits == 1) {
#pragma unroll 1
        for (int c0 = chalf * (BN / 2); c0 < (chalf + 1) * (BN / 2); c0 += 16) {
          float v[16];
          acc16(c0, v);
          EpiIn in[16];
          epi_load_block<MODE>(e, m0 + ew * 32, n0 + c0, in);
          epi_warp16_t<MODE>(e, m0 + ew * 32, n0 + c0, v, esm, in, &wmx);
        }
        fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[ab]);
        continue;
      }
      // split-K: every split publishes its partial (private layout [split][warp slot][chunk][q][lane][4], each
      // warp float4 access one contiguous 512 B segment) and takes a ticket; the LAST split to arrive adds all
      // partials in split order (deterministic: the order does not depend on who arrives last) and runs the
      // epilogue. No split waits for another, so the latency is one mainloop plus one exchange.
      const size_t slot_off = (size_t)(ew + 4 * chalf) * (32 * BN / 2) + (size_t)lane * 4;
      auto part = [&](int s2) { return ws + ((size_t)tile * sc.splits + s2) * BM * BN + slot_off; };
#pragma unroll 1
      for (int c0 = chalf * (BN / 2); c0 < (chalf + 1) * (BN / 2); c0 += 16) {
        float v[16];
        acc16(c0, v);
        float* p = part(split) + (size_t)((c0 - chalf * (BN / 2)) / 16) * (4 * 32 * 4);
#pragma unroll
        for (int q = 0; q < 4; ++q)
          __stcg(reinterpret_cast<float4*>(p + q * 128), make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]));
      }
      fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[ab]);
      __threadfence();
      epi_bar();
      if (threadIdx.x == 128) s_last = atomicAdd(flags + tile, 1u) == (unsigned)(sc.splits - 1);
      epi_bar();
      if (!s_last) continue;
      __threadfence();
#pragma unroll 1
      for (int c0 = chalf * (BN / 2); c0 < (chalf + 1) * (BN / 2); c0 += 16) {
        float v[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] = 0.f;
        const size_t blk = (size_t)((c0 - chalf * (BN / 2)) / 16) * (4 * 32 * 4);
        int s2 = 0;
        for (; s2 + 4 <= sc.splits; s2 += 4) {  // 16 loads in flight, then the adds in split order
          float4 t[4][4];
#pragma unroll
          for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int q = 0; q < 4; ++q) t[u][q] = __ldcg(reinterpret_cast<const float4*>(part(s2 + u) + blk + q * 128));
#pragma unroll
          for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              v[4 * q] += t[u][q].x; v[4 * q + 1] += t[u][q].y; v[4 * q + 2] += t[u][q].z; v[4 * q + 3] += t[u][q].w;
            }
        }
        for (; s2 < sc.splits; ++s2) {
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const float4 t = __ldcg(reinterpret_cast<const float4*>(part(s2) + blk + q * 128));
            v[4 * q] += t.x; v[4 * q + 1] += t.y; v[4 * q + 2] += t.z; v[4 * q + 3] += t.w;
          }
        }
        EpiIn in[16];
        epi_load_block<MODE>(e, m0 + ew * 32, n0 + c0, in);
        epi_warp16_t<MODE>(e, m0 + ew * 32, n0 + c0, v, esm, in, &wmx);
      }
      if (threadIdx.x == 128) flags[tile] = 0u;  // ticket back to zero for the next launch
    }
    if (MODE != EPI_STORE && e.amax) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) wmx = fmaxf(wmx, __shfl_xor_sync(0xffffffffu, wmx, o));
      if (lane == 0) s_mx1[warp - 4] = wmx;
      epi_bar();
      if (threadIdx.x == 128) {
        float m = s_mx1[0];
#pragma unroll
        for (int q = 1; q < 8; ++q) m = fmaxf(m, s_mx1[q]);
        if (m > 0.f) atomicMax(e.amax, __float_as_uint(m));
      }
    }
    if (trace && threadIdx.x == 128) trace[5] = gtimer1();
  }
  fence_before();
  __syncthreads();
  if (trace && threadIdx.x == 0) trace[6] = gtimer1();
  if (warp == 2) {
    fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
    if (trace && lane == 0) trace[7] = gtimer1();
  }
}

// split-K factor that best fills the persistent grid (work quantization), >= 8 k-blocks per split
int pick_splits(int tiles, int nkb, int sms) {
  // Few tiles (the small-M GEMMs of small problems): split K for latency — the splits run concurrently and the
  // last one to finish combines them — keeping >= 2 k-blocks per split.
  // (Measured per-CTA timelines at M = 128, K = 1568: 4-8 splits minimise the launch; beyond, the last
  // split's combine costs more than the shorter mainloops save.)
  if (tiles * 4 <= sms) return std::max(1, std::min(std::min(sms / tiles, nkb / 4), 8));
  // Split only when whole-tile scheduling leaves the persistent grid badly quantised (the HVP GEMMs at
  // M = B = 1024: 224 tiles on 148 SMs); each extra split costs ~5% (partial write + read).
  // Measured on B200: profiles/r01_gemm_splits.txt.
  auto eff_of = [&](int s) {
    const int units = tiles * s;
    const int waves = (units + sms - 1) / sms;
    return (double)units / ((double)waves * sms) - 0.05 * (s - 1);
  };
  if (eff_of(1) >= 0.85) return 1;
  int best = 1;
  double best_eff = 0.0;
  for (int s = 1; s <= 3; ++s) {
    if (s > 1 && nkb / s < 8) break;
    const double eff = eff_of(s);
    if (eff > best_eff + 1e-9) {
      best_eff = eff;
      best = s;
    }
  }
  return best;
}

template <bool AMN, bool BMN, int MODE>
void launch(dho2g_ctx* ctx, const CUtensorMap* maps, const Sched& sc, const OpOff& oa, const OpOff& ob, const Epi& e,
            float* ws, unsigned* flags, unsigned epoch) {
  static bool attr_set = false;
  if (!attr_set) {
    DHO2G_CUDA(cudaFuncSetAttribute(gemm3_tc_kernel<AMN, BMN, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)SMEM));
    attr_set = true;
  }
  const int ctas = ctx->gemm_worker_cap > 0 ? std::min(ctx->sm_count, 2 * ctx->gemm_worker_cap) : ctx->sm_count;
  const int grid = std::min(sc.units, ctas);
  gemm3_tc_kernel<AMN, BMN, MODE><<<grid, 384, SMEM, ctx->stream>>>(maps[0], maps[1], maps[2], maps[3], sc, oa, ob,
                                                                    e, ws, flags, epoch);
  DHO2G_LAUNCH();
}

template <int MODE>
void launch_mode(dho2g_ctx* ctx, bool amn, bool bmn, const CUtensorMap* maps, const Sched& sc, const OpOff& oa,
                 const OpOff& ob, const Epi& e, float* ws, unsigned* flags, unsigned epoch) {
  if (amn && bmn) launch<true, true, MODE>(ctx, maps, sc, oa, ob, e, ws, flags, epoch);
  else if (amn) launch<true, false, MODE>(ctx, maps, sc, oa, ob, e, ws, flags, epoch);
  else if (bmn) launch<false, true, MODE>(ctx, maps, sc, oa, ob, e, ws, flags, epoch);
  else launch<false, false, MODE>(ctx, maps, sc, oa, ob, e, ws, flags, epoch);
}

int run(dho2g_ctx* ctx, int M, int N, int K, int kseg, const GOp& A, const GOp& B, const Epi& e) {
  Sched sc;
  sc.mt = (int)cdiv(M, BM);
  sc.nt = (int)cdiv(N, BN);
  sc.tiles = sc.mt * sc.nt;
  sc.nkb = (int)cdiv(K, BK);
  sc.kseg = kseg;
  const int ctas = ctx->gemm_worker_cap > 0 ? std::min(ctx->sm_count, 2 * ctx->gemm_worker_cap) : ctx->sm_count;
  sc.splits = ctx->gemm_splits > 0 ? std::min(ctx->gemm_splits, std::max(1, sc.nkb)) : pick_splits(sc.tiles, sc.nkb, ctas);
  sc.units = sc.tiles * sc.splits;
  const int per_unit = (sc.nkb + sc.splits - 1) / sc.splits;
  sc.chunk = (ctx->gemm_chunk_kb1 > 0 && ctx->gemm_chunk_kb1 < per_unit) ? ctx->gemm_chunk_kb1 : std::max(per_unit, 1);
  float* ws = nullptr;
  unsigned* flags = nullptr;
  unsigned epoch = 0;
  if (sc.splits > 1) {
    // one partial per (tile, split); tickets past the pair kernel's flags (they return to zero after each use)
    ctx->gemm_ws.ensure_g((size_t)sc.tiles * sc.splits * BM * BN);
    ctx->gemm_flags.ensure_g(kTc1Tickets + (size_t)sc.tiles);
    ws = ctx->gemm_ws.p;
    flags = ctx->gemm_flags.p + kTc1Tickets;
  }
  CUtensorMap maps[4];
  op_maps(ctx->encode_fn, A, maps[0], maps[1]);
  op_maps(ctx->encode_fn, B, maps[2], maps[3]);
  const OpOff oa = op_off(A), ob = op_off(B);
  const bool amn = A.mn_major != 0, bmn = B.mn_major != 0;
  switch (e.mode) {
    case EPI_STORE: launch_mode<EPI_STORE>(ctx, amn, bmn, maps, sc, oa, ob, e, ws, flags, epoch); break;
    case EPI_FWD: launch_mode<EPI_FWD>(ctx, amn, bmn, maps, sc, oa, ob, e, ws, flags, epoch); break;
    case EPI_FWD_OUT: launch_mode<EPI_FWD_OUT>(ctx, amn, bmn, maps, sc, oa, ob, e, ws, flags, epoch); break;
    default: launch_mode<EPI_BWD>(ctx, amn, bmn, maps, sc, oa, ob, e, ws, flags, epoch); break;
  }
  return sc.splits;
}

}  // namespace tc1

// =============================================================================== CTA-pair kernel
// cta_group::2: a cluster of two CTAs (one TPC) computes a 256 x Nt pair tile (Nt <= 256). CTA r
// stages rows [m0 + 128 r, +128) of A and rows [n0 + r Nt/2, +Nt/2) of B; the leader (rank 0)
// issues tcgen05.mma.cta_group::2 (M = 256, N = Nt) over both CTAs' shared memory, each CTA's TMEM
// receiving its 128 output rows. Per SM this halves the shared-memory operand reads and the L2->SM
// operand traffic per flop relative to the single-CTA 128 x 128 kernel.
//
// Work is distributed stream-K: the (tile, k-block) iteration space is cut into `workers` equal
// contiguous ranges, one per pair. A range starting inside a tile begins with a non-head segment,
// whose fp32 partial goes to the pair's workspace slot (flag = ready); the head segment's owner
// (which processes it last) adds the later segments' partials in segment order and runs the fused
// epilogue. The combine order is fixed by the schedule, so results are deterministic.
namespace tc2 {
// Optional per-CTA timeline of one pair-GEMM launch (option gemm_trace; investigation only): globaltimer
// ns at [0] start of work (after the prologue), [1] last MMA issued (leader), [2] start of the last
// segment's epilogue work, [3] end, per CTA slot blockIdx.x.
__device__ unsigned long long* g_gemm_trace = nullptr;
// which launches write it: 0 all, 1 R-forward (EPI_FWD, R half), 2 R-backward (EPI_BWD, R half), 3 EPI_STORE
__device__ int g_gemm_trace_filter = 0;
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
using namespace tc;

constexpr int BM = 128;   // output rows per CTA (pair tile 256)
constexpr int NT = 256;   // pair tile width (UMMA N)
constexpr int BKT = 64;   // K-block depth (one 128-byte SW128 row of bf16)
constexpr int STAGES = 3;
constexpr uint32_t STAGE_BYTES = 4 * OP_BYTES;  // A hi/lo (128 rows) + B hi/lo (128 = NT/2 rows)
constexpr uint32_t SMEM = STAGES * STAGE_BYTES + 1024 + 256 + EPI_SMEM;
constexpr uint32_t PART_MAX = BM * 256;  // one CTA's partial tile (NT = 256)

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void commit2(uint64_t* bar) {  // arrive on this offset's barrier in both CTAs
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"((uint16_t)3)
      : "memory");
}
__device__ __forceinline__ void arrive_leader(uint64_t* bar) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(smem_u32(bar) & 0xFEFFFFFFu)
               : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* b, uint32_t parity) {
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(smem_u32(b)), "r"(parity)
        : "memory");
  } while (!done);
}

// Tile schedule (m-major tile order, tile = m * nt + n): the first `dp` tiles are data-parallel — worker
// w takes whole tiles w, w + W, ..., so the tiles in flight at any time are consecutive and share their
// A rows (a working set that fits L2; measured 9x operand re-reads from HBM on the gradient GEMMs with
// stream-K over the whole space); the remaining tiles (about one wave) are stream-K: the
// (tile, k-block) space is cut into W equal contiguous ranges.
// Group mode (grp = mt > 1, no data-parallel part): the workers form workers / grp groups of grp pairs; a
// group's pairs walk the same contiguous range of the (n-tile, k-block) space, pair `sub` of the group on
// m-tile `sub`. The grp pairs that need a B slab (n, k) load it at about the same time, so it comes from
// DRAM once and from L2 for the others (plain stream-K over (tile, k) puts the m-tiles of one column at
// unrelated k offsets: the R-GEMMs re-read B ~4x from DRAM). A segment boundary splits tile (sub, n)
// between groups g and g + 1, whose pair `sub` does the fix-up as in plain stream-K.
struct Work {
  int mt, nt, nkb, workers, N, kseg, nround;  // nround: MMA N granularity (16; 128 for an MN-major B)
  int dp;                                      // data-parallel tiles
  int chunk;  // k-blocks per TMEM accumulation chunk (drained into an fp32 running sum); >= nkb: off
  int grp;    // pairs per group (1: plain stream-K)
  __device__ __forceinline__ int groups() const { return workers / grp; }
  __device__ __forceinline__ long long sk_total() const {
    return grp > 1 ? (long long)nt * nkb : (long long)(mt * nt - dp) * nkb;
  }
  // start of group (plain: worker) g's stream-K range
  __device__ __forceinline__ long long begin(int /*phase*/, int g) const { return sk_total() * g / groups(); }
};
struct Seg {
  int phase, tile, k0, k1;  // phase 0: data-parallel (tile = global index); 1: stream-K (tile = index after dp)
  int mtile, ntile;
};
// Iterates one worker's segments: its data-parallel tiles, then its stream-K range.
struct Cursor {
  int p, w, t, sub;
  long long a, end;
  __device__ __forceinline__ void init(const Work& wk, int worker) {
    w = worker;
    p = 0;
    t = worker;
    sub = worker % wk.grp;
    a = wk.begin(1, worker / wk.grp);
    end = wk.begin(1, worker / wk.grp + 1);
  }
  __device__ __forceinline__ bool next(const Work& wk, Seg& s) {
    int g;
    if (p == 0 && t < wk.dp) {
      s.phase = 0;
      s.tile = g = t;
      s.k0 = 0;
      s.k1 = wk.nkb;
      t += wk.workers;
    } else {
      p = 1;
      if (a >= end) return false;
      s.phase = 1;
      s.tile = (int)(a / wk.nkb);
      s.k0 = (int)(a - (long long)s.tile * wk.nkb);
      s.k1 = (int)((long long)s.k0 + (end - a) < wk.nkb ? s.k0 + (end - a) : wk.nkb);
      a += s.k1 - s.k0;
      if (wk.grp > 1) {  // group mode: s.tile is the n-tile, the m-tile is this pair's place in its group
        s.mtile = sub;
        s.ntile = s.tile;
        return true;
      }
      g = wk.dp + s.tile;
    }
    s.mtile = g / wk.nt;
    s.ntile = g % wk.nt;
    return true;
  }
};
template <int NT>
__device__ __forceinline__ int tile_cols(const Work& wk, int n0) {  // MMA N of a tile (<= NT)
  const int c = wk.N - n0;
  return c >= NT ? NT : ((c + wk.nround - 1) / wk.nround) * wk.nround;
}

// NT: pair tile width (256, or 128 when 256-wide tiles would leave pairs with less than ~2 tiles)
template <bool AMN, bool BMN, int MODE>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(384, 1)
    gemm3_tc2_kernel(const __grid_constant__ CUtensorMap mAh, const __grid_constant__ CUtensorMap mAl,
                     const __grid_constant__ CUtensorMap mBh, const __grid_constant__ CUtensorMap mBl, Work wk,
                     OpOff oa, OpOff ob, const __grid_constant__ Epi e, float* __restrict__ ws,
                     unsigned* __restrict__ flags, unsigned ready) {
  extern __shared__ uint8_t smem_raw[];
  __shared__ float s_mx[8];  // epilogue warps' max |x| (one e.amax update per CTA and tile)
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + ACC;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + ACC);

  constexpr uint32_t TMEM_COLS = ACC * NT;
  constexpr uint32_t PART_FLOATS = BM * NT;
  constexpr uint32_t B_BYTES = (NT / 2) * BKT * 2;  // one (hi or lo) B half-tile
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const int worker = blockIdx.x >> 1;

  if (threadIdx.x == 0) {
#pragma unroll
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
#pragma unroll
    for (int a = 0; a < ACC; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 16);  // 8 epilogue warps x 2 CTAs (leader copy is the one used)
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mAh)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mAl)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mBh)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mBl)) : "memory");
  }
  cluster_sync();
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  fence_before();
  cluster_sync();
  fence_after();
  const uint32_t tmem = *tmem_slot;
  // Programmatic dependent launch: everything above (barriers, tensor-map prefetch, TMEM allocation)
  // may overlap the previous kernel's tail; no global memory is touched before the previous grid has
  // completed and flushed (a no-op when launched without the attribute).
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int tf = g_gemm_trace_filter;
  const bool traced = tf == 0 || (tf == 1 && MODE == EPI_FWD && e.do1) || (tf == 2 && MODE == EPI_BWD && e.do1) ||
                      (tf == 3 && MODE == EPI_STORE);
  unsigned long long* trace = (g_gemm_trace && traced) ? g_gemm_trace + (size_t)blockIdx.x * 8 : nullptr;
  if (trace && threadIdx.x == 0) trace[0] = gtimer();

  if (warp == 0 && lane == 0) {
    // ---------------- TMA producer (both CTAs): this CTA's halves of A and B into its ring
    uint32_t it = 0;
    Cursor cur;
    cur.init(wk, worker);
    Seg sg;
    while (cur.next(wk, sg)) {
      const int m0 = sg.mtile * 256 + (int)rank * BM, n0 = sg.ntile * NT;
      const int nb = n0 + (int)rank * (tile_cols<NT>(wk, n0) / 2);
      for (int kb = sg.k0; kb < sg.k1; ++kb, ++it) {
        const int s = it % STAGES;
        mbar_wait(&empty[s], ((it / STAGES) & 1) ^ 1);
        uint8_t* st = smem + s * STAGE_BYTES;
        if (rank == 0) mbar_expect_tx(&full[s], 2 * (2 * OP_BYTES + 2 * B_BYTES));
        load_op<AMN, true, 2, BKT>(st, &mAh, oa, m0, kb, wk.kseg, &full[s]);
        load_op<AMN, true, 2, BKT>(st + OP_BYTES, &mAl, oa, m0, kb, wk.kseg, &full[s]);
        load_op<BMN, true, NT / 128, BKT>(st + 2 * OP_BYTES, &mBh, ob, nb, kb, wk.kseg, &full[s]);
        load_op<BMN, true, NT / 128, BKT>(st + 3 * OP_BYTES, &mBl, ob, nb, kb, wk.kseg, &full[s]);
      }
    }
    // all operand loads issued: the next kernel in the stream may start its prologue on freed SMs
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  } else if (warp == 1 && lane == 0 && rank == 0) {
    // ---------------- MMA issuer (leader CTA only)
    uint32_t it = 0, uc = 0;
    Cursor cur;
    cur.init(wk, worker);
    Seg sg;
    while (cur.next(wk, sg)) {
      const int n0 = sg.ntile * NT;
      const uint32_t ID = idesc_fmt(idesc(256, tile_cols<NT>(wk, n0), AMN, BMN), e.f16 != 0);
     for (int c0 = sg.k0; c0 < sg.k1; c0 += wk.chunk) {  // one accumulator per chunk
      const int c1 = min(sg.k1, c0 + wk.chunk);
      // double-buffered (a chunked accumulation keeps its running sum in the epilogue warps' registers)
      const uint32_t ab = uc % ACC;
      mbar_wait_cluster(&tempty[ab], ((uc / ACC) & 1) ^ 1);
      fence_after();
      const uint32_t acc_addr = tmem + ab * NT;
      for (int kb = c0; kb < c1; ++kb, ++it) {
        const int s = it % STAGES;
        mbar_wait(&full[s], (it / STAGES) & 1);
        fence_after();
        const uint32_t base = smem_u32(smem + s * STAGE_BYTES);
#pragma unroll
        for (int kk = 0; kk < BKT / UK; ++kk) {
          const uint64_t dAh = op_desc<AMN, BKT>(base, kk);
          const uint64_t dAl = op_desc<AMN, BKT>(base + OP_BYTES, kk);
          const uint64_t dBh = op_desc<BMN, BKT>(base + 2 * OP_BYTES, kk);
          const uint64_t dBl = op_desc<BMN, BKT>(base + 3 * OP_BYTES, kk);
          const uint32_t first = (kb > c0 || kk > 0) ? 1u : 0u;
          asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(acc_addr),
              "l"(dAh), "l"(dBh), "r"(ID), "r"(first));
          asm volatile("tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, 1;" ::"r"(acc_addr), "l"(dAh), "l"(dBl),
                       "r"(ID));
          asm volatile("tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, 1;" ::"r"(acc_addr), "l"(dAl), "l"(dBh),
                       "r"(ID));
        }
        commit2(&empty[s]);
      }
      commit2(&tfull[ab]);
      ++uc;
     }
    }
    if (trace) trace[1] = gtimer();
  } else if (warp >= 4) {
    // ---------------- epilogue warps (both CTAs): 8 warps = 4 TMEM lane quadrants x 2 column halves
    const int ew = warp & 3;
    const int chalf = (warp - 4) >> 2;
    float* esm = reinterpret_cast<float*>(smem + STAGES * STAGE_BYTES + 256) + (warp - 4) * (32 * 17);
    const size_t slot_off = (size_t)(ew + 4 * chalf) * (32 * NT / 2) + (size_t)lane * 4;
    uint32_t uc = 0;
    Cursor cur;
    cur.init(wk, worker);
    Seg sg;
    const uint32_t nacc = (uint32_t)ACC;
    const int cbase = chalf * (NT / 2);
    while (cur.next(wk, sg)) {
      const int m0 = sg.mtile * 256 + (int)rank * BM, n0 = sg.ntile * NT;
      const int ncols = tile_cols<NT>(wk, n0);
      // chunks before the last: running sum (this thread's row x 128 columns, in registers) += chunk
      // (round-to-nearest fp32), then free the accumulator for the MMAs of the chunk after next. Columns
      // past the MMA's N hold unused values.
      const int nchunks = (sg.k1 - sg.k0 + wk.chunk - 1) / wk.chunk;
      // a head segment runs the layer epilogue: its inputs into L2 while the last chunk's MMAs run
      const bool head = sg.k0 == 0;
      if (head && nchunks == 1) epi_prefetch_row<MODE>(e, m0 + ew * 32 + lane, n0 + cbase);
      if (nchunks > 1) {
        float rs[NT / 2];
#pragma unroll
        for (int j = 0; j < NT / 2; ++j) rs[j] = 0.f;
        for (int c = 0; c + 1 < nchunks; ++c, ++uc) {
          const uint32_t ab = uc % nacc;
          mbar_wait(&tfull[ab], (uc / nacc) & 1);
          fence_after();
          const uint32_t tb = tmem + ((uint32_t)(ew * 32) << 16) + ab * NT + (uint32_t)cbase;
#pragma unroll
          for (int q = 0; q < NT / 32; ++q) {
            uint32_t r[16];
            tmem_ld16_nowait(tb + (uint32_t)(16 * q), r);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
            for (int j = 0; j < 16; ++j) rs[16 * q + j] += __uint_as_float(r[j]);
          }
          fence_before();
          __syncwarp();
          if (lane == 0) arrive_leader(&tempty[ab]);
        }
        // fold the running sum into the last chunk's accumulator: acc = last + sum
        if (head) epi_prefetch_row<MODE>(e, m0 + ew * 32 + lane, n0 + cbase);
        const uint32_t ab = uc % nacc;
        mbar_wait(&tfull[ab], (uc / nacc) & 1);
        fence_after();
        const uint32_t tb = tmem + ((uint32_t)(ew * 32) << 16) + ab * NT + (uint32_t)cbase;
#pragma unroll
        for (int q = 0; q < NT / 32; ++q) {
          uint32_t r[16];
          tmem_ld16_nowait(tb + (uint32_t)(16 * q), r);
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
          float v[16];
#pragma unroll
          for (int j = 0; j < 16; ++j) v[j] = __uint_as_float(r[j]) + rs[16 * q + j];
          tmem_st16(tb + (uint32_t)(16 * q), v);
        }
        tmem_wait_st();
      }
      const uint32_t ab = uc % nacc;
      mbar_wait(&tfull[ab], (uc / nacc) & 1);
      fence_after();
      if (trace && threadIdx.x == 128) trace[2] = gtimer();
      const uint32_t tbase = tmem + ((uint32_t)(ew * 32) << 16) + ab * NT;
      if (sg.k0 != 0) {
        // non-head segment (first of this worker): publish the raw partial
        float* p = ws + ((size_t)(sg.phase * wk.workers + worker) * 2 + rank) * PART_FLOATS + slot_off;
#pragma unroll 1
        for (int c0 = chalf * (NT / 2); c0 < (chalf + 1) * (NT / 2); c0 += 16) {
          if (c0 >= ncols) break;
          float v[16];
          tmem_ld16(tbase + (uint32_t)c0, v);
          float* q = p + (size_t)((c0 - chalf * (NT / 2)) / 16) * (4 * 32 * 4);
#pragma unroll
          for (int j = 0; j < 4; ++j)
            __stcg(reinterpret_cast<float4*>(q + j * 128), make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]));
        }
        fence_before();
        __syncwarp();
        if (lane == 0) arrive_leader(&tempty[ab]);
        __threadfence();
        epi_bar();
        if (threadIdx.x == 128) st_release(flags + (sg.phase * wk.workers + worker) * 2 + rank, ready);
      } else {
        // head segment: later segments of this tile are the first segments of workers worker+1, ...
        // (group mode: the groups after this one, their pair of the same m-tile: worker + grp, + 2 grp, ...)
        const long long tile_end = (long long)(sg.tile + 1) * wk.nkb;
        const int sbase = sg.phase * wk.workers;
        const int gw = worker / wk.grp;
        int glast = gw;
        if (sg.k1 < wk.nkb) {
          while (glast + 1 < wk.groups() && wk.begin(sg.phase, glast + 1) < tile_end) ++glast;
          if (threadIdx.x == 128)
            for (int g2 = gw + 1; g2 <= glast; ++g2)
              while (ld_acquire(flags + (sbase + worker + (g2 - gw) * wk.grp) * 2 + rank) != ready) __nanosleep(64);
          epi_bar();
        }
        if (trace && threadIdx.x == 128) trace[4] = gtimer();
        const int wlast = worker + (glast - gw) * wk.grp;
        float wmx = 0.f;  // this lane's max |x| over the tile (e.amax)
#pragma unroll 1
        for (int c0 = chalf * (NT / 2); c0 < (chalf + 1) * (NT / 2); c0 += 16) {
          if (c0 >= ncols) break;
          // the block's epilogue inputs in flight together with the accumulator and partial reads
          EpiIn in[16];
          epi_load_block<MODE>(e, m0 + ew * 32, n0 + c0, in);
          float v[16];
          tmem_ld16(tbase + (uint32_t)c0, v);
          for (int w2 = worker + wk.grp; w2 <= wlast; w2 += wk.grp) {
            const float* q = ws + ((size_t)(sbase + w2) * 2 + rank) * PART_FLOATS + slot_off +
                             (size_t)((c0 - chalf * (NT / 2)) / 16) * (4 * 32 * 4);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const float4 t = __ldcg(reinterpret_cast<const float4*>(q + j * 128));
              v[4 * j] += t.x; v[4 * j + 1] += t.y; v[4 * j + 2] += t.z; v[4 * j + 3] += t.w;
            }
          }
          epi_warp16_t<MODE>(e, m0 + ew * 32, n0 + c0, v, esm, in, &wmx);
        }
        if (MODE != EPI_STORE && e.amax) {  // one atomicMax per CTA and tile
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) wmx = fmaxf(wmx, __shfl_xor_sync(0xffffffffu, wmx, o));
          if (lane == 0) s_mx[warp - 4] = wmx;
          epi_bar();
          if (threadIdx.x == 128) {
            float m = s_mx[0];
#pragma unroll
            for (int q = 1; q < 8; ++q) m = fmaxf(m, s_mx[q]);
            if (m > 0.f) atomicMax(e.amax, __float_as_uint(m));
          }
          epi_bar();  // s_mx is rewritten by the next tile's epilogue
        }
        if (trace && threadIdx.x == 128) trace[5] = gtimer();
        fence_before();
        __syncwarp();
        if (lane == 0) arrive_leader(&tempty[ab]);
      }
      ++uc;
    }
  }
  fence_before();
  __syncthreads();
  if (trace && threadIdx.x == 0) trace[3] = gtimer();
  cluster_sync();
  if (warp == 2) {
    fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
  }
}

template <bool AMN, bool BMN, int MODE>
int max_pairs(dho2g_ctx* ctx) {
  static int pairs = 0;
  if (pairs > 0) return pairs;
  DHO2G_CUDA(cudaFuncSetAttribute(gemm3_tc2_kernel<AMN, BMN, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(2 * (ctx->sm_count / 2));
  cfg.blockDim = dim3(384);
  cfg.dynamicSmemBytes = SMEM;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int clusters = 0;
  DHO2G_CUDA(cudaOccupancyMaxActiveClusters(&clusters, gemm3_tc2_kernel<AMN, BMN, MODE>, &cfg));
  if (clusters < 1) fail(DHO2G_CUDA, "gemm3_tc2: no CTA pair can be resident");
  pairs = clusters;
  return pairs;
}

template <bool AMN, bool BMN, int MODE>
int launch(dho2g_ctx* ctx, const CUtensorMap* maps, Work wk, const OpOff& oa, const OpOff& ob, const Epi& e) {
  const int pairs = max_pairs<AMN, BMN, MODE>(ctx);
  // every worker gets >= gemm_min_kb k-blocks (shorter segments are mostly fix-up traffic)
  const long long tiles = (long long)wk.mt * wk.nt;
  ctx->pairs_total = pairs;
  const int cap = ctx->gemm_worker_cap > 0 ? std::min(ctx->gemm_worker_cap, pairs) : pairs;
  wk.workers = (int)std::min<long long>(cap, std::max<long long>(1, tiles * wk.nkb / std::max(1, ctx->gemm_min_kb)));
  // data-parallel waves, keeping the last ~1-2 waves of tiles for stream-K balancing (option gemm_dp = 0
  // turns the data-parallel part off)
  const long long waves = tiles / wk.workers;
  wk.dp = (ctx->gemm_dp && waves >= 2) ? (int)((waves - 1) * wk.workers) : 0;
  wk.grp = 1;
  if (ctx->gemm_group && waves < 2 && wk.mt > 1 && 2 * wk.mt <= wk.workers) {  // few m-tiles: group mode
    wk.grp = wk.mt;
    wk.workers -= wk.workers % wk.mt;
    wk.dp = 0;
  }
  // stream-K partial slots (2 schedule parts x workers x 2 CTAs)
  ctx->gemm_ws.ensure_g((size_t)2 * wk.workers * 2 * PART_MAX);
  ctx->gemm_flags.ensure_g((size_t)2 * wk.workers * 2 + 16);
  wk.chunk = (e.chunk_kb > 0 && e.chunk_kb < wk.nkb) ? e.chunk_kb : wk.nkb;
  unsigned epoch = ++ctx->gemm_epoch;
  if (epoch >= (1u << 27)) {  // flags hold epoch * 16 + 15 here (epoch * 16 + split in tc1): recycle
    DHO2G_CUDA(cudaMemsetAsync(ctx->gemm_flags.p, 0, ctx->gemm_flags.n * sizeof(unsigned), ctx->stream));
    ctx->gemm_epoch = epoch = 1;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(2 * wk.workers);
  cfg.blockDim = dim3(384);
  cfg.dynamicSmemBytes = SMEM;
  cfg.stream = ctx->stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = ctx->gemm_pdl ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  DHO2G_CUDA(cudaLaunchKernelEx(&cfg, gemm3_tc2_kernel<AMN, BMN, MODE>, maps[0], maps[1], maps[2], maps[3], wk, oa,
                                ob, e, ctx->gemm_ws.p, ctx->gemm_flags.p, epoch * 16u + 15u));
  DHO2G_LAUNCH();
  return wk.workers;
}

template <int MODE>
int launch_mode(dho2g_ctx* ctx, const CUtensorMap* maps, const Work& wk, const OpOff& oa, const OpOff& ob,
                const Epi& e, bool amn, bool bmn) {
  if (amn && bmn) return launch<true, true, MODE>(ctx, maps, wk, oa, ob, e);
  if (amn) return launch<true, false, MODE>(ctx, maps, wk, oa, ob, e);
  if (bmn) return launch<false, true, MODE>(ctx, maps, wk, oa, ob, e);
  return launch<false, false, MODE>(ctx, maps, wk, oa, ob, e);
}

int run(dho2g_ctx* ctx, int M, int N, int K, int kseg, const GOp& A, const GOp& B, const Epi& e) {
  Work wk;
  wk.mt = (int)cdiv(M, 256);
  wk.nt = (int)cdiv(N, NT);
  wk.nkb = (int)cdiv(K, BKT);
  wk.N = N;
  wk.kseg = kseg;
  wk.nround = B.mn_major ? 128 : 16;
  wk.workers = 1;
  wk.dp = 0;  // set in launch() once the worker count is known
  CUtensorMap maps[4];
  op_maps(ctx->encode_fn, A, maps[0], maps[1]);
  op_maps(ctx->encode_fn, B, maps[2], maps[3], NT / 2);
  const OpOff oa = op_off(A), ob = op_off(B);
  const bool amn = A.mn_major != 0, bmn = B.mn_major != 0;
  switch (e.mode) {
    case EPI_STORE: return launch_mode<EPI_STORE>(ctx, maps, wk, oa, ob, e, amn, bmn);
    case EPI_FWD: return launch_mode<EPI_FWD>(ctx, maps, wk, oa, ob, e, amn, bmn);
    case EPI_FWD_OUT: return launch_mode<EPI_FWD_OUT>(ctx, maps, wk, oa, ob, e, amn, bmn);
    default: return launch_mode<EPI_BWD>(ctx, maps, wk, oa, ob, e, amn, bmn);
  }
}

}  // namespace tc2

void gemm_presize(dho2g_ctx* ctx) {
  // both lanes' stream-K partials (2 schedule parts x pairs x 2 CTAs x 128 x 256) and flags; covers the
  // single-CTA kernel's split-K partials for the small-M GEMMs too
  const size_t pairs = (size_t)std::max(1, ctx->sm_count / 2);
  ctx->gemm_ws.ensure_g(2 * pairs * 2 * tc2::PART_MAX);
  ctx->gemm_flags.ensure_g(tc1::kTc1Tickets + 2048);  // pair-kernel flags, then the single-CTA tickets
  ctx->gemm_ws2.ensure_g(2 * pairs * 2 * tc2::PART_MAX);
  ctx->gemm_flags2.ensure_g(tc1::kTc1Tickets + 2048);
}

// =============================================================================== dispatch
void gemm3x(dho2g_ctx* ctx, int M, int N, int K, int kseg, const GOp& A, const GOp& B, const Epi& e) {
  if (M <= 0 || N <= 0) return;
  if (K <= 0) fail(DHO2G_ARGUMENT, "gemm3: empty reduction dimension");
  if (kseg < K && (kseg <= 0 || kseg % tc::BK)) fail(DHO2G_ARGUMENT, "gemm3: K segment boundary must be a multiple of 64");
  tc::check_op(A, "A");
  tc::check_op(B, "B");
  if (A.f16 != B.f16 || (A.f16 != 0) != (e.f16 != 0)) fail(DHO2G_ARGUMENT, "gemm3: operand formats differ");
  ctx->bump("gemm_calls", 1);
  ctx->bump("gemm_flops_issued", 3.0 * 2.0 * double(M) * double(N) * double(K));
  const int slot = ctx->kt_begin();
  int splits = 1, pair_nt = 0;
  bool pair = false;
  if (ctx->gemm_backend == 1) {
    gemm3_simt(ctx, M, N, K, kseg, A, B, e);
  } else {
    if (!ctx->encode_fn) fail(DHO2G_CUDA, "cuTensorMapEncodeTiled entry point unavailable");
    // CTA pairs (256-row tiles) for the big shapes; M <= 512 or K <= 1024 run as 128 x 128 single-CTA tiles:
    // with few 256 x 256 tiles per pair each pair ends on an exposed full-tile epilogue (C3, M = 512: fwdR 72 ->
    // 51 us, the weight blocks at K = 512 46 -> 38 us, 102 -> 118 steps/s; C4 keeps the pairs: 10.5 vs 9.3).
    // Short-K weight blocks with both operands MN-major can also take the single-CTA kernel (gemm_mm_tc1).
    const bool short_mm = A.mn_major && B.mn_major && K <= 2048 && ctx->gemm_mm_tc1;
    pair = ctx->gemm_cta == 2 || (ctx->gemm_cta == 0 && M > 512 && K > 1024 && !short_mm);
    splits = pair ? tc2::run(ctx, M, N, K, kseg, A, B, e) : tc1::run(ctx, M, N, K, kseg, A, B, e);
    pair_nt = pair ? tc2::NT : 0;
  }
  if (slot >= 0) {  // name: backend:epilogue(+R)[operand majors]/(splits | pair), aggregated by prefix in the bench
    static const char* modes[] = {"store", "fwd", "fwdout", "bwd"};
    char lay[8] = "";
    if (A.mn_major || B.mn_major) std::snprintf(lay, sizeof(lay), "[%c%c]", A.mn_major ? 'm' : 'k', B.mn_major ? 'm' : 'k');
    char name[80];
    if (pair)
      std::snprintf(name, sizeof(name), "gemm3_tcgen05:%s%s%s/pair%d", modes[e.mode], e.do1 ? "R" : "", lay, pair_nt);
    else
      std::snprintf(name, sizeof(name), "%s:%s%s%s/s%d", ctx->gemm_backend == 1 ? "gemm3_simt" : "gemm3_tcgen05",
                    modes[e.mode], e.do1 ? "R" : "", lay, splits);
    ctx->kt_end(slot, name, 2.0 * double(M) * double(N) * double(K));
  }
}

void gemm3(dho2g_ctx* ctx, int M, int N, int K, const bf16* Ahi, const bf16* Alo, int lda, const bf16* Bhi,
           const bf16* Blo, int ldb, const Epi& e) {
  gemm3x(ctx, M, N, K, K, gop_k(Ahi, Alo, lda, K, M), gop_k(Bhi, Blo, ldb, K, N), e);
}

void gemm3_store(dho2g_ctx* ctx, int M, int N, int K, const bf16* Ahi, const bf16* Alo, int lda, const bf16* Bhi,
                 const bf16* Blo, int ldb, float* C, int ldc, float alpha, float* bias_out) {
  Epi e{};
  e.mode = EPI_STORE;
  e.M = M;
  e.N = N;
  e.C = C;
  e.ldc = ldc;
  e.alpha = alpha;
  e.bias_out = bias_out;
  gemm3(ctx, M, N, K, Ahi, Alo, lda, Bhi, Blo, ldb, e);
}

}  // namespace dho2g

// Test hook (option gemm_trace): route the next pair-GEMM launches' per-CTA timelines into buf (4 u64 per
// CTA slot); buf = nullptr switches tracing off.
namespace dho2g {
void gemm_trace_set(unsigned long long* buf, int filter) {
  DHO2G_CUDA(cudaMemcpyToSymbol(tc2::g_gemm_trace, &buf, sizeof(buf)));
  DHO2G_CUDA(cudaMemcpyToSymbol(tc2::g_gemm_trace_filter, &filter, sizeof(filter)));
}
void gemm_trace1_set(unsigned long long* buf) {
  DHO2G_CUDA(cudaMemcpyToSymbol(tc1::g_tc1_trace, &buf, sizeof(buf)));
}
}  // namespace dho2g
