// Device MLP oracle (reference: proj/src/oracle.cpp:288-687) — forward, backward and the
// Pearlmutter R-op as batched split-BF16x3 GEMMs plus fused tile epilogues.
//
// Layout (reference oracle.cpp:304-324): flat params, per layer W (out x in, row-major) then b.
// Per layer t with in = s_t, out = s_{t+1} the contractions are (B = batch):
//   forward    Z  = A W^T            RZ = [A | RA] [V | W]^T         (K = in, 2 in)
//   backward   U  = D W              RU = D V + RD W                 (K = out, two K segments)
//   weight     hvW = RD^T A + D^T RA                                 (K = B, two K segments)
// Every operand is stored once, row-major, as (hi, lo) bf16 pairs: [a | ra] and [d | rd] by sample,
// [V | W] by output unit. The forward GEMMs read them K-major; the backward and weight GEMMs read
// the same buffers MN-major through TMA windows (GOp), so no transposed copies are written.
//
// A Lanczos refresh applies H at ONE point w on ONE curvature batch m times, so everything that
// does not depend on the direction v (A, Z, softmax, D, U for every layer) is computed once by
// mlp_prepare_point() and cached; each mlp_hvp_dev() then only runs the R-GEMMs (RZ, RU) and the
// weight-block GEMM: 6 of the 8 per-layer GEMM units of oracle.cpp:524-647 (2 of 3 at layer 0).
#include <cmath>

#include "internal.h"
#include "mlp_dev.cuh"

using namespace dho2g;

void dho2g_mlp::ensure_batch(size_t B) {
  if (B <= Bcap) return;
  ++g_graph_gen;
  const size_t nB = round_up(B, 128);
  const int Ls = L;
  AR_hi.resize(Ls); AR_lo.resize(Ls);
  DR_hi.resize(Ls + 1); DR_lo.resize(Ls + 1);
  a32.resize(Ls + 1); ra32.resize(Ls + 1); d32.resize(Ls + 1); rd32.resize(Ls + 1); u32.resize(Ls + 1);
  for (int j = 0; j <= Ls; ++j) {
    const size_t s = sizes[j], P = round_up(s, 8), D = round_up(s, 64);
    if (j < Ls) {
      AR_hi[j].alloc(nB * 2 * P); AR_lo[j].alloc(nB * 2 * P);
    }
    if (j >= 1) {
      DR_hi[j].alloc(nB * 2 * D); DR_lo[j].alloc(nB * 2 * D);
      a32[j].alloc(nB * s); ra32[j].alloc(nB * s); d32[j].alloc(nB * s); rd32[j].alloc(nB * s);
      if (j < Ls) u32[j].alloc(nB * s);
    }
  }
  Z.alloc(nB * smax);
  RZ.alloc(nB * smax);
  lab.alloc(nB);
  sample_loss.alloc(nB);
  sample_correct.alloc(nB);
  Bcap = nB;
  prepared = nullptr;
}

namespace {

// ------------------------------------------------------------------ weight operand packing
// WV[t][o][half*Pin + k] = scale * p(o, k), k < in (pads [in, Pin) stay zero). One row o per
// blockIdx.y; each thread packs 8 elements (8 independent loads in flight), coalesced across the warp.
constexpr int kPackPer = 8;  // elements per thread: 4 pairs
__global__ void pack_weights_kernel(const float* __restrict__ p, const float* __restrict__ pscale, int in, int out,
                                    int Pin, int half, bf16* __restrict__ WVh, bf16* __restrict__ WVl) {
  // thread t of the block owns column pairs (k, k+1), k = k0 + 2 t + 2 u blockDim for u < 4: coalesced fp32
  // reads, 4-byte bf16x2 writes (k is even and so are Pin and the row base)
  const int k0 = blockIdx.x * (blockDim.x * kPackPer) + 2 * threadIdx.x;
  const float sc = pscale ? *pscale : 1.0f;
  for (int o = blockIdx.y; o < out; o += gridDim.y) {
    const float* row = p + (size_t)o * in;
    float x[kPackPer];
#pragma unroll
    for (int u = 0; u < kPackPer / 2; ++u) {
      const int k = k0 + 2 * u * blockDim.x;
      x[2 * u] = k < in ? __ldg(row + k) : 0.f;
      x[2 * u + 1] = k + 1 < in ? __ldg(row + k + 1) : 0.f;
    }
    const size_t base = (size_t)o * (2 * Pin) + (size_t)half * Pin;
#pragma unroll
    for (int u = 0; u < kPackPer / 2; ++u) {
      const int k = k0 + 2 * u * blockDim.x;
      if (k < in) {
        bf16 h0, l0, h1, l1;
        split_bf16(x[2 * u] * sc, h0, l0);
        split_bf16(x[2 * u + 1] * sc, h1, l1);
        if (k + 1 < in) {
          *reinterpret_cast<__nv_bfloat162*>(WVh + base + k) = __halves2bfloat162(h0, h1);
          *reinterpret_cast<__nv_bfloat162*>(WVl + base + k) = __halves2bfloat162(l0, l1);
        } else {
          WVh[base + k] = h0;
          WVl[base + k] = l0;
        }
      }
    }
  }
}

// ------------------------------------------------------------------ row-major operand packing
// Level-0 input rows (x0 = X[idx[b]], half 0) or output-layer deltas (x0 = d -> half 0, x1 = rd ->
// half 1) into a row-major (hi, lo) pair buffer of half-width P; pad columns [s, P) get zeros.
__global__ void pack_rows_kernel(int B, int s, int P, const float* __restrict__ X, const int64_t* __restrict__ idx,
                                 int ldX, const float* __restrict__ x1src, bf16* __restrict__ Rh,
                                 bf16* __restrict__ Rl) {
  const int b = blockIdx.y;
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B || k >= P) return;
  const size_t r = (size_t)b * (2 * P) + k;
  bf16 h, l;
  if (X) {
    const int64_t row = idx ? idx[b] : b;
    split_bf16(k < s ? X[(size_t)row * ldX + k] : 0.f, h, l);
    Rh[r] = h;
    Rl[r] = l;
  }
  if (x1src) {
    split_bf16(k < s ? x1src[(size_t)b * s + k] : 0.f, h, l);
    Rh[r + P] = h;
    Rl[r + P] = l;
  }
}

// ------------------------------------------------------------------ scaled-fp16 operands (gemm_f16)
// max |x| into a slot (float bits; nonnegative floats order like their bit patterns)
__device__ __forceinline__ void slot_max(unsigned* slot, float m) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0 && m > 0.f) atomicMax(slot, __float_as_uint(m));
}
__global__ void absmax_kernel(const float* __restrict__ p, size_t n, unsigned* slot) {
  float m = 0.f;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    m = fmaxf(m, fabsf(__ldg(p + i)));
  slot_max(slot, m);
}
__global__ void absmax_rows_kernel(const float* __restrict__ X, const int64_t* __restrict__ idx, int ldX, int B, int s,
                                   unsigned* slot) {
  float m = 0.f;
  for (int b = blockIdx.y; b < B; b += gridDim.y) {
    const float* row = X + (size_t)(idx ? idx[b] : b) * ldX;
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < s; k += gridDim.x * blockDim.x) m = fmaxf(m, fabsf(row[k]));
  }
  slot_max(slot, m);
}

// [V | W] packing as scaled fp16: the W half (half 1) picks the scale from max |W| and the bound on the
// direction halves that will share it, and publishes it; the V half (half 0) uses the published scale.
__global__ void pack_weights_f16_kernel(const float* __restrict__ p, const float* __restrict__ pscale, int in, int out,
                                        int Pin, int half, const unsigned* __restrict__ wmax, float vbound,
                                        float* __restrict__ sout, bf16* __restrict__ WVh, bf16* __restrict__ WVl) {
  const int k0 = blockIdx.x * (blockDim.x * kPackPer) + 2 * threadIdx.x;
  float sc;
  if (half == 1) {
    sc = pow2_scale(fmaxf(__uint_as_float(*wmax), vbound));
    if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) *sout = sc;
  } else {
    sc = *sout;
  }
  const float ps = pscale ? *pscale : 1.0f;
  for (int o = blockIdx.y; o < out; o += gridDim.y) {
    const float* row = p + (size_t)o * in;
    float x[kPackPer];
#pragma unroll
    for (int u = 0; u < kPackPer / 2; ++u) {
      const int k = k0 + 2 * u * blockDim.x;
      x[2 * u] = k < in ? __ldg(row + k) : 0.f;
      x[2 * u + 1] = k + 1 < in ? __ldg(row + k + 1) : 0.f;
    }
    const size_t base = (size_t)o * (2 * Pin) + (size_t)half * Pin;
#pragma unroll
    for (int u = 0; u < kPackPer / 2; ++u) {
      const int k = k0 + 2 * u * blockDim.x;
      if (k < in) {
        bf16 h0, l0, h1, l1;
        split_f16(x[2 * u] * ps, sc, h0, l0);
        split_f16(x[2 * u + 1] * ps, sc, h1, l1);
        if (k + 1 < in) {
          *reinterpret_cast<__nv_bfloat162*>(WVh + base + k) = __halves2bfloat162(h0, h1);
          *reinterpret_cast<__nv_bfloat162*>(WVl + base + k) = __halves2bfloat162(l0, l1);
        } else {
          WVh[base + k] = h0;
          WVl[base + k] = l0;
        }
      }
    }
  }
}

// One level's [x | rx] pair buffer (rows b, half-width P, pads [s, P) zero) from fp32 sources as scaled
// fp16: x from X rows (idx-gathered, level 0) or x32 (B x s), rx from rx32. One scale covers both halves:
//   x only (the point / gradient passes): s = pow2_scale(max |x|), written, and recorded in *sx;
//   x and rx (an HVP: x is the point's cached value, already in the buffer at scale *sx): the x half is
//   rewritten only when max(|x|, |rx|) needs a smaller scale than *sx (then *sx shrinks); otherwise only
//   rx is written, at *sx. *sx is read by every block at its start and updated by the last block to finish
//   (ticket), so no block sees a half-updated value.
// Block 0 publishes the scale for the consuming GEMMs (*sout). 2D grid: rows over y, 8-column groups over x.
__device__ __forceinline__ void load8(const float* row, int k, int s, bool vec, float (&x)[8]) {
  if (vec && k + 7 < s) {
    const float4 a = *reinterpret_cast<const float4*>(row + k), b = *reinterpret_cast<const float4*>(row + k + 4);
    x[0] = a.x; x[1] = a.y; x[2] = a.z; x[3] = a.w; x[4] = b.x; x[5] = b.y; x[6] = b.z; x[7] = b.w;
  } else {
#pragma unroll
    for (int u = 0; u < 8; ++u) x[u] = k + u < s ? row[k + u] : 0.f;
  }
}
__device__ __forceinline__ void split8(const float (&x)[8], float sc, bf16* h, bf16* l) {
  bf16 hh[8], ll[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) split_f16(x[u], sc, hh[u], ll[u]);
  *reinterpret_cast<uint4*>(h) = *reinterpret_cast<const uint4*>(hh);
  *reinterpret_cast<uint4*>(l) = *reinterpret_cast<const uint4*>(ll);
}
__global__ void __launch_bounds__(128) split_pair_kernel(int B, int s, int P, const float* __restrict__ X,
                                                         const int64_t* __restrict__ idx, int ldX,
                                                         const float* __restrict__ x32, const float* __restrict__ rx32,
                                                         const unsigned* __restrict__ mxx,
                                                         const unsigned* __restrict__ mxr, float* __restrict__ sout,
                                                         float* sx, unsigned* ticket, bf16* __restrict__ Rh,
                                                         bf16* __restrict__ Rl) {
  // launched as a programmatic dependent of the producing GEMM: nothing is read or written before that grid
  // has completed (a no-op without the launch attribute)
  asm volatile("griddepcontrol.wait;" ::: "memory");
  float mx = 0.f;
  if (mxx) mx = fmaxf(mx, __uint_as_float(*mxx));
  if (mxr) mx = fmaxf(mx, __uint_as_float(*mxr));
  const float s_need = pow2_scale(mx);
  const bool has_x = X != nullptr || x32 != nullptr;
  bool wx = has_x;
  float sc = s_need;
  if (has_x && rx32) {
    const float s_have = *sx;
    wx = !(s_have > 0.f) || s_need < s_have;
    sc = wx ? s_need : s_have;
  }
  if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) *sout = sc;
  const int G = P / 8;  // P is a multiple of 8
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  const bool vx = X ? (ldX % 4 == 0) : (s % 4 == 0), vr = s % 4 == 0;
  if (g < G) {
    const int k = g * 8;
    // two rows per step, all four loads issued before the first split (one memory latency per two rows)
    for (int b = blockIdx.y; b < B; b += 2 * gridDim.y) {
      const int b2 = b + gridDim.y;
      const bool two = b2 < B;
      float x0[8], x1[8], r0[8], r1[8];
      if (wx) {
        load8(X ? X + (size_t)(idx ? idx[b] : b) * ldX : x32 + (size_t)b * s, k, s, vx, x0);
        if (two) load8(X ? X + (size_t)(idx ? idx[b2] : b2) * ldX : x32 + (size_t)b2 * s, k, s, vx, x1);
      }
      if (rx32) {
        load8(rx32 + (size_t)b * s, k, s, vr, r0);
        if (two) load8(rx32 + (size_t)b2 * s, k, s, vr, r1);
      }
      const size_t o0 = (size_t)b * (2 * P) + k, o1 = (size_t)b2 * (2 * P) + k;
      if (wx) {
        split8(x0, sc, Rh + o0, Rl + o0);
        if (two) split8(x1, sc, Rh + o1, Rl + o1);
      }
      if (rx32) {
        split8(r0, sc, Rh + o0 + P, Rl + o0 + P);
        if (two) split8(r1, sc, Rh + o1 + P, Rl + o1 + P);
      }
    }
  }
  if (wx) {  // record the x half's scale once every block is done with *sx
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      if (atomicAdd(ticket, 1u) == gridDim.x * gridDim.y - 1) {
        *sx = sc;
        *ticket = 0u;
      }
    }
  }
}

// ------------------------------------------------------------------ output layer delta
// (output_delta_row: mlp_dev.cuh)
__global__ void output_delta_kernel(int B, int O, int mse, int ncls, int do0, int do1, double scale,
                                    const float* __restrict__ z, const float* __restrict__ rz,
                                    const float* __restrict__ lab, float* __restrict__ d, float* __restrict__ rd,
                                    double* __restrict__ loss, int* __restrict__ correct, unsigned* mxd,
                                    unsigned* mxrd) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (mxd || mxrd) {  // max |d|, |rd| for the scaled-fp16 split (this thread's row, after the deltas below)
    float md = 0.f, mr = 0.f;
    if (b < B) {
      output_delta_row<false>(b, O, mse, ncls, do0, do1, scale, z, rz, lab, d, rd, loss, correct);
      for (int j = 0; j < O; ++j) {
        if (do0) md = fmaxf(md, fabsf(d[(size_t)b * O + j]));
        if (do1) mr = fmaxf(mr, fabsf(rd[(size_t)b * O + j]));
      }
    }
    if (mxd) slot_max(mxd, md);
    if (mxrd) slot_max(mxrd, mr);
    return;
  }
  if (b >= B) return;
  output_delta_row<false>(b, O, mse, ncls, do0, do1, scale, z, rz, lab, d, rd, loss, correct);
}

// Bias block as a column sum of a row-major pair buffer: out[o] = sum_{b < B} (hi + lo)[b][off + o].
// Blocks of 64 columns (2 per lane, bf16x2 loads) x 8 row groups over one of kColChunks row chunks
// write fp64 partials part[chunk][o]; the last block of each column block (ticket) adds the chunks
// in order (deterministic, one launch).
constexpr int kColChunks = 32;
// (src32: the same sums over an fp32 B x cols source instead of the pairs — the scaled-fp16 mode, where the
// exact fp32 deltas are at hand)
__global__ void colsum_pairs_kernel(const bf16* __restrict__ hi, const bf16* __restrict__ lo, int ld, int off,
                                    int cols, int B, double* __restrict__ part, unsigned* __restrict__ tickets,
                                    float* __restrict__ out, const float* __restrict__ src32) {
  __shared__ double sh[8][64];
  __shared__ bool last;
  const int c = blockIdx.x * 64 + 2 * threadIdx.x;
  const int rows_per = (B + kColChunks - 1) / kColChunks;
  const int r0 = blockIdx.y * rows_per, r1 = min(B, r0 + rows_per);
  float a0 = 0.f, a1 = 0.f;
  if (src32) {
    if (c < cols)
      for (int b = r0 + threadIdx.y; b < r1; b += 8) {
        a0 += src32[(size_t)b * cols + c];
        if (c + 1 < cols) a1 += src32[(size_t)b * cols + c + 1];
      }
  } else if (c < cols) {
#pragma unroll 4
    for (int b = r0 + threadIdx.y; b < r1; b += 8) {
      const size_t i = (size_t)b * ld + off + c;
      const __nv_bfloat162 h = *reinterpret_cast<const __nv_bfloat162*>(hi + i);
      const __nv_bfloat162 l = *reinterpret_cast<const __nv_bfloat162*>(lo + i);
      a0 += __bfloat162float(h.x) + __bfloat162float(l.x);
      a1 += __bfloat162float(h.y) + __bfloat162float(l.y);
    }
  }
  sh[threadIdx.y][2 * threadIdx.x] = a0;
  sh[threadIdx.y][2 * threadIdx.x + 1] = a1;
  __syncthreads();
  const int tid = threadIdx.y * 32 + threadIdx.x;
  if (tid < 64) {
    const int cc = blockIdx.x * 64 + tid;
    double t = 0.0;
    for (int g = 0; g < 8; ++g) t += sh[g][tid];
    if (cc < cols) part[(size_t)blockIdx.y * cols + cc] = t;
  }
  __threadfence();
  __syncthreads();
  if (tid == 0) last = atomicAdd(&tickets[blockIdx.x], 1u) == gridDim.y - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  if (tid < 64) {
    const int cc = blockIdx.x * 64 + tid;
    if (cc < cols) {
      double t = 0.0;
      for (int k = 0; k < (int)gridDim.y; ++k) t += __ldcg(part + (size_t)k * cols + cc);
      out[cc] = (float)t;
    }
  }
  if (tid == 0) tickets[blockIdx.x] = 0u;
}

// Bias block from the per-32-row column sums the producing epilogue wrote: out[o] = sum_rb csum[rb][o]
// (fixed order, fp64).
__global__ void csum_final_kernel(const float* __restrict__ csum, int nrb, int cols, float* __restrict__ out) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= cols) return;
  double t = 0.0;
  for (int rb = 0; rb < nrb; ++rb) t += (double)csum[(size_t)rb * cols + c];
  out[c] = (float)t;
}

// batch rows X[idx[b]] (and labels) into a dense device copy
__global__ void gather_rows_kernel(const float* __restrict__ X, const float* __restrict__ y, const int64_t* __restrict__ idx,
                                   int B, int s, float* __restrict__ out, float* __restrict__ yout) {
  for (int b = blockIdx.y; b < B; b += gridDim.y) {
    const int64_t r = idx ? idx[b] : b;
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c < s) out[(size_t)b * s + c] = X[(size_t)r * s + c];
    if (blockIdx.x == 0 && threadIdx.x == 0) yout[b] = y[r];
  }
}

// label gather
__global__ void gather_labels_kernel(int B, const float* __restrict__ y, const int64_t* __restrict__ idx,
                                     float* __restrict__ out) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b < B) out[b] = y[idx ? idx[b] : b];
}

// deterministic single-CTA sum of per-sample loss / correct into acc2[0], acc2[1] (+=)
__global__ void eval_reduce_kernel(int B, const double* __restrict__ loss, const int* __restrict__ correct,
                                   double* __restrict__ acc2) {
  __shared__ double sh[32];
  double l = 0.0, c = 0.0;
  for (int b = threadIdx.x; b < B; b += blockDim.x) {
    l += loss[b];
    c += correct[b];
  }
  const double L = block_sum(l, sh);
  const double Cc = block_sum(c, sh);
  if (threadIdx.x == 0) {
    acc2[0] += L;
    acc2[1] += Cc;
  }
}

}  // namespace

namespace dho2g {

// Packs the [V | W] halves. With the side lane enabled the packing kernels run on ctx->stream2 (forked
// from the main stream, one event per layer) and forward() waits for layer t's event just before layer
// t's GEMMs, so the bandwidth-bound packing of later layers overlaps the tensor-core GEMMs of earlier ones.
static void pack_params(dho2g_mlp* m, const float* p, const float* pscale, int half) {
  dho2g_ctx* ctx = m->ctx;
  const bool async = ctx->bwd_overlap && ctx->gemm_backend == 0;
  cudaStream_t main = ctx->stream;
  if (async) {
    if (!ctx->stream2) DHO2G_CUDA(cudaStreamCreateWithFlags(&ctx->stream2, cudaStreamNonBlocking));
    while (m->pack_ev.size() < (size_t)m->L + 1) {
      cudaEvent_t ev;
      DHO2G_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
      m->pack_ev.push_back(ev);
    }
    DHO2G_CUDA(cudaEventRecord(m->pack_ev[m->L], main));  // fork: p and the previous readers of WV
    DHO2G_CUDA(cudaStreamWaitEvent(ctx->stream2, m->pack_ev[m->L], 0));
    ctx->stream = ctx->stream2;
  }
  for (int t = 0; t < m->L; ++t) {
    const LayerDesc& ld = m->layers[t];
    if (m->f16 && half == 1) {  // the W half fixes the layer's scale: max |W| first
      if (t == 0) DHO2G_CUDA(cudaMemsetAsync(m->mx_w(0), 0, m->L * sizeof(unsigned), ctx->stream));
      const size_t nw = (size_t)ld.in * ld.out;
      absmax_kernel<<<(int)std::min<size_t>(cdiv(nw, 256), (size_t)ctx->sm_count * 8), 256, 0, ctx->stream>>>(
          p + ld.w_off, nw, m->mx_w(t));
      DHO2G_LAUNCH();
    }
    const int slot = ctx->kt_begin();
    // one wave of resident blocks striding over the rows (short-lived per-row blocks cost more than the copy)
    const int gx = (int)cdiv(ld.in, 128 * kPackPer);
    const int gy = std::max(1, std::min(ld.out, ctx->sm_count * 16 / gx));
    if (m->f16)
      pack_weights_f16_kernel<<<dim3(gx, gy), 128, 0, ctx->stream>>>(p + ld.w_off, pscale, ld.in, ld.out, ld.Pin, half,
                                                                     m->mx_w(t), m->wv_vbound, m->s_wv(t),
                                                                     m->WV_hi[t].p, m->WV_lo[t].p);
    else
      pack_weights_kernel<<<dim3(gx, gy), 128, 0, ctx->stream>>>(p + ld.w_off, pscale, ld.in, ld.out, ld.Pin, half,
                                                                 m->WV_hi[t].p, m->WV_lo[t].p);
    DHO2G_LAUNCH();
    // algorithmic bytes: read fp32 (4) + write hi/lo (4)
    ctx->kt_end(slot, "pack_params", (double)ld.in * ld.out * 8.0);
    if (async) DHO2G_CUDA(cudaEventRecord(m->pack_ev[t], ctx->stream));
  }
  if (async) {
    ctx->stream = main;
    m->pack_pending = true;
  }
}

// The operand format follows the ctx option; a change invalidates everything packed in the old one.
static void sync_format(dho2g_mlp* m) {
  const int f = m->ctx->gemm_f16 ? 1 : 0;
  if (m->f16 == f) return;
  m->f16 = f;
  m->w_cur = nullptr;
  m->wv_packed = nullptr;
  m->input_packed = false;
  m->input_owner = nullptr;
  m->prepared = nullptr;
}

// The W halves are packed on first use by the tensor-core path (the small-model path reads w directly).
void mlp_load_weights(dho2g_mlp* m, const float* w) {
  sync_format(m);
  m->w_cur = w;
  m->wv_packed = nullptr;
  m->prepared = nullptr;
  if (m->wv_vbound < 1.0f) m->wv_vbound = 1.0f;  // unit Lanczos directions
}

static void ensure_weights_packed(dho2g_mlp* m, bool force = false) {
  if (!force && m->wv_packed == m->w_cur) return;
  pack_params(m, m->w_cur, nullptr, 1);
  m->wv_packed = m->w_cur;
}

void mlp_load_direction(dho2g_mlp* m, const float* v, const float* vscale) { pack_params(m, v, vscale, 0); }

void mlp_presize(dho2g_mlp* m, size_t B) {
  m->ensure_batch(B);
  mlp_small_presize(m, B);
  m->csum.ensure_g((size_t)2 * cdiv(B, 32) * m->smax);
  m->colpart.ensure_g((size_t)kColChunks * m->smax);
  m->coltickets.ensure_g(cdiv(m->smax, 64));
}

static void pack_rows(dho2g_ctx* ctx, int B, int s, int P, const float* X, const int64_t* idx, int ldX,
                      const float* x1, bf16* Rh, bf16* Rl) {
  const int slot = ctx->kt_begin();
  pack_rows_kernel<<<dim3(cdiv(P, 128), B), 128, 0, ctx->stream>>>(B, s, P, X, idx, ldX, x1, Rh, Rl);
  DHO2G_LAUNCH();
  ctx->kt_end(slot, "pack_rows", (double)B * s * 4.0 * ((X ? 2.0 : 0.0) + (x1 ? 2.0 : 0.0)));
}

// level-j pair buffer as scaled fp16 from fp32 sources (see split_pair_kernel)
static void split_pair(dho2g_mlp* m, int B, int s, int P, const float* X, const int64_t* idx, int ldX, const float* x32,
                       const float* rx32, const unsigned* mxx, const unsigned* mxr, float* sout, bf16* Rh, bf16* Rl) {
  dho2g_ctx* ctx = m->ctx;
  const int slot = ctx->kt_begin();
  const int gx = (int)cdiv((size_t)(P / 8), 128);
  // one wave of resident blocks (12 of 128 threads per SM at this kernel's register count), rows strided
  const int gy = (int)std::max<size_t>(1, std::min<size_t>((size_t)B, std::max<size_t>(1, (size_t)ctx->sm_count * 12 / gx)));
  const size_t bi = (size_t)(sout - m->scl.p);  // this buffer's x-half scale and ticket
  // programmatic dependent launch (option gemm_pdl): the launch and block scheduling overlap the producing
  // GEMM's tail; the kernel waits for that grid before touching memory
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(gx, gy);
  cfg.blockDim = dim3(128);
  cfg.stream = ctx->stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = ctx->gemm_pdl ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  DHO2G_CUDA(cudaLaunchKernelEx(&cfg, split_pair_kernel, B, s, P, X, idx, ldX, x32, rx32, mxx, mxr, sout,
                                m->sclx.p + bi, m->sticket.p + bi, Rh, Rl));
  DHO2G_LAUNCH();
  // algorithmic bytes: rx always, x when this call may rewrite it (counted as written: an upper bound)
  ctx->kt_end(slot, "split_pair", (double)B * s * 8.0 * ((rx32 ? 1.0 : 0.0) + ((X || x32) && !rx32 ? 1.0 : 0.0)));
}

static void ensure_input_packed(dho2g_mlp* m);

// Records the batch; the tensor-core path's level-0 operands are packed here unless the small-model path
// (which reads X and y directly) takes batches of this size.
void mlp_set_input(dho2g_mlp* m, const float* X, const float* y, const int64_t* idx, size_t B, bool /*with_r*/) {
  sync_format(m);
  m->ensure_batch(B);
  m->input_owner = nullptr;
  m->prepared = nullptr;
  m->x_src = X;
  m->x_idx = idx;
  m->y_src = y;
  m->x_B = B;
  m->input_packed = false;
  if (!mlp_small_eligible(m, B)) {
    ensure_input_packed(m);
    return;
  }
  // The small-model path reads X in every pass: a batch in host memory (the end-to-end mode's dataset,
  // mapped pinned) is gathered to the device once here instead of crossing PCIe in every HVP.
  cudaPointerAttributes pa{};
  if (cudaPointerGetAttributes(&pa, X) != cudaSuccess) cudaGetLastError();
  if (pa.type != cudaMemoryTypeDevice && pa.type != cudaMemoryTypeManaged) {
    const size_t s0 = m->sizes[0];
    m->x0.ensure_g(round_up(B, 128) * s0);
    m->y0.ensure_g(round_up(B, 128));
    gather_rows_kernel<<<dim3((unsigned)cdiv(s0, 128), (unsigned)std::min<size_t>(B, 65535)), 128, 0, m->ctx->stream>>>(
        X, y, idx, (int)B, (int)s0, m->x0.p, m->y0.p);
    DHO2G_LAUNCH();
    m->x_src = m->x0.p;
    m->y_src = m->y0.p;
    m->x_idx = nullptr;
  }
}

static void ensure_input_packed(dho2g_mlp* m) {
  if (m->input_packed) return;
  m->input_packed = true;
  const float* X = m->x_src;
  const float* y = m->y_src;
  const int64_t* idx = m->x_idx;
  const size_t B = m->x_B;
  const int s0 = (int)m->sizes[0];
  if (m->f16) {
    dho2g_ctx* ctx = m->ctx;
    DHO2G_CUDA(cudaMemsetAsync(m->mx_x(), 0, sizeof(unsigned), ctx->stream));
    absmax_rows_kernel<<<dim3((unsigned)cdiv(s0, 256), (unsigned)std::min<size_t>(B, 1024)), 256, 0, ctx->stream>>>(
        X, idx, s0, (int)B, s0, m->mx_x());
    DHO2G_LAUNCH();
    split_pair(m, (int)B, s0, (int)round_up(s0, 8), X, idx, s0, nullptr, nullptr, m->mx_x(), nullptr, m->s_ar(0),
               m->AR_hi[0].p, m->AR_lo[0].p);
  } else {
    pack_rows(m->ctx, (int)B, s0, (int)round_up(s0, 8), X, idx, s0, nullptr, m->AR_hi[0].p, m->AR_lo[0].p);
  }
  gather_labels_kernel<<<cdiv(B, 256), 256, 0, m->ctx->stream>>>((int)B, y, idx, m->lab.p);
  DHO2G_LAUNCH();
}

// Forward pass. do0: plain activations (Z GEMM + fused bias/act epilogue). do1: R-activations
// (RZ GEMM + fused R-epilogue over the cached activations).
static void forward(dho2g_mlp* m, const float* w, size_t B, bool do0, bool do1) {
  dho2g_ctx* ctx = m->ctx;
  if (m->f16) {  // max slots of the levels this pass writes (a or ra, levels 1..L), one memset
    if (do0) DHO2G_CUDA(cudaMemsetAsync(m->mx_a(1), 0, m->L * sizeof(unsigned), ctx->stream));
    if (do1) DHO2G_CUDA(cudaMemsetAsync(m->mx_ra(1), 0, m->L * sizeof(unsigned), ctx->stream));
  }
  for (int t = 0; t < m->L; ++t) {
    const LayerDesc& ld = m->layers[t];
    if (m->pack_pending) DHO2G_CUDA(cudaStreamWaitEvent(ctx->stream, m->pack_ev[t], 0));  // layer t packed
    const bool last = t + 1 == m->L;
    const int lda = 2 * ld.Pin;
    for (int pass = 0; pass < 2; ++pass) {
      const bool r = pass == 1;
      if ((r && !do1) || (!r && !do0)) continue;
      Epi e{};
      e.chunk_kb = m->chunk_kb;
      e.mode = last ? EPI_FWD_OUT : EPI_FWD;
      e.M = (int)B;
      e.N = ld.out;
      e.do0 = !r;
      e.do1 = r;
      e.relu = m->act == 1;
      e.bias = w + ld.b_off;
      e.vbias = r ? m->v_bias_ptr + ld.b_off : nullptr;
      e.vscale = m->v_scale_ptr;
      e.a_in = m->a32[t + 1].p;
      e.f0 = m->a32[t + 1].p;
      e.f1 = m->ra32[t + 1].p;
      if (m->f16) {  // fp32 outputs + max |.|, split below with the scale that covers them
        e.f16 = 1;
        e.sa = m->s_ar(t);
        e.sb = m->s_wv(t);
        if (!last) e.amax = r ? m->mx_ra(t + 1) : m->mx_a(t + 1);  // (cleared at the top)
      } else if (!last) {
        e.Rh = m->AR_hi[t + 1].p; e.Rl = m->AR_lo[t + 1].p; e.P = ld.Pout; e.hR = r ? 1 : 0;
      }
      const int K = r ? (t == 0 ? ld.in : 2 * ld.Pin) : ld.in;
      // Z = A W^T ; RZ = [A | RA] [V | W]^T (ra = 0 at the input layer: K = in only)
      GOp A = gop_k(m->AR_hi[t].p, m->AR_lo[t].p, lda, K, (int)B);
      GOp W = r ? gop_k(m->WV_hi[t].p, m->WV_lo[t].p, lda, K, ld.out)
                : gop_k(m->WV_hi[t].p + ld.Pin, m->WV_lo[t].p + ld.Pin, lda, K, ld.out);
      A.f16 = W.f16 = m->f16;
      gemm3x(ctx, (int)B, ld.out, K, K, A, W, e);
      if (m->f16 && !last)  // [a | ra] of level t+1: the R pass rewrites a too, so both halves share one scale
        split_pair(m, (int)B, ld.out, ld.Pout, nullptr, nullptr, 0, m->a32[t + 1].p, r ? m->ra32[t + 1].p : nullptr,
                   m->mx_a(t + 1), r ? m->mx_ra(t + 1) : nullptr, m->s_ar(t + 1), m->AR_hi[t + 1].p,
                   m->AR_lo[t + 1].p);
    }
  }
  m->pack_pending = false;  // every layer's event has been waited on by the main stream
}

static void output_delta(dho2g_mlp* m, size_t B, size_t ncls, double scale, bool do0, bool do1) {
  const int L = m->L;
  const int O = (int)m->sizes[L];
  cudaStream_t st = m->ctx->stream;
  unsigned* mxd = (m->f16 && do0) ? m->mx_d(L) : nullptr;
  unsigned* mxrd = (m->f16 && do1) ? m->mx_rd(L) : nullptr;
  if (mxd) DHO2G_CUDA(cudaMemsetAsync(mxd, 0, sizeof(unsigned), st));
  if (mxrd) DHO2G_CUDA(cudaMemsetAsync(mxrd, 0, sizeof(unsigned), st));
  output_delta_kernel<<<cdiv(B, 128), 128, 0, st>>>((int)B, O, m->loss, (int)ncls, do0, do1, scale, m->a32[L].p,
                                                    m->ra32[L].p, m->lab.p, m->d32[L].p, m->rd32[L].p,
                                                    m->sample_loss.p, m->sample_correct.p, mxd, mxrd);
  DHO2G_LAUNCH();
  if (m->f16)  // [d | rd]: the R pass rewrites d (cached) so both halves share one scale
    split_pair(m, (int)B, O, (int)round_up(O, 64), nullptr, nullptr, 0, m->d32[L].p, do1 ? m->rd32[L].p : nullptr,
               m->mx_d(L), do1 ? m->mx_rd(L) : nullptr, m->s_dr(L), m->DR_hi[L].p, m->DR_lo[L].p);
  else
    pack_rows(m->ctx, (int)B, O, (int)round_up(O, 64), do0 ? m->d32[L].p : nullptr, nullptr, O,
              do1 ? m->rd32[L].p : nullptr, m->DR_hi[L].p, m->DR_lo[L].p);
}

static void bias_colsum(dho2g_mlp* m, const bf16* hi, const bf16* lo, int ld, int off, int cols, int B, float* out,
                        const float* src32 = nullptr) {
  dho2g_ctx* ctx = m->ctx;
  m->colpart.ensure_g((size_t)kColChunks * cols);
  m->coltickets.ensure_g(cdiv(cols, 64));  // zeroed at allocation; each launch leaves them zero
  const int slot = ctx->kt_begin();
  colsum_pairs_kernel<<<dim3(cdiv(cols, 64), kColChunks), dim3(32, 8), 0, ctx->stream>>>(
      hi, lo, ld, off, cols, B, m->colpart.p, m->coltickets.p, out, src32);
  DHO2G_LAUNCH();
  ctx->kt_end(slot, "bias_colsum", 4.0 * cols * (double)B);  // algorithmic bytes: hi + lo
}

// Side lane: while active, the library's launches go to ctx->stream2 with the second GEMM workspace and a
// CTA-pair budget, so a GEMM issued here runs concurrently with one issued on the main stream.
struct SideLane {
  dho2g_ctx* c;
  cudaStream_t main;
  int cap_saved;
  SideLane(dho2g_ctx* ctx, int cap) : c(ctx), main(ctx->stream), cap_saved(ctx->gemm_worker_cap) {
    c->stream = c->stream2;
    std::swap(c->gemm_ws, c->gemm_ws2);
    std::swap(c->gemm_flags, c->gemm_flags2);
    c->gemm_worker_cap = cap;
  }
  ~SideLane() {
    c->stream = main;
    std::swap(c->gemm_ws, c->gemm_ws2);
    std::swap(c->gemm_flags, c->gemm_flags2);
    c->gemm_worker_cap = cap_saved;
  }
};

static cudaEvent_t lane_event(dho2g_ctx* ctx, size_t i) {
  while (ctx->lane_events.size() <= i) {
    cudaEvent_t ev;
    DHO2G_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    ctx->lane_events.push_back(ev);
  }
  return ctx->lane_events[i];
}

// Backward pass. do0: deltas d (U GEMMs + fused act' epilogue) and, if wgrad, the gradient blocks.
// do1: R-deltas (RU GEMMs + fused R-epilogue) and the Hessian blocks into `out`. The weight blocks
// are GEMMs over the batch (both operands MN-major windows of the row-major pair buffers); the bias
// blocks are column sums of the delta pairs.
static void backward(dho2g_mlp* m, size_t B, float* out, bool do0, bool do1, bool wgrad) {
  dho2g_ctx* ctx = m->ctx;
  const int L = m->L;
  const int Bi = (int)B;
  const int nrb = (int)cdiv(B, 32);
  if (m->f16 && L > 1) {  // max slots of the hidden levels this pass writes (d or rd), one memset
    if (do0) DHO2G_CUDA(cudaMemsetAsync(m->mx_d(1), 0, (L - 1) * sizeof(unsigned), ctx->stream));
    if (do1) DHO2G_CUDA(cudaMemsetAsync(m->mx_rd(1), 0, (L - 1) * sizeof(unsigned), ctx->stream));
  }
  // the bias block of layer t is the batch sum of level t+1's deltas: the epilogue that writes them (layer
  // t+1's backward GEMM) also writes per-32-row column sums into m->csum (two buffers, by level parity);
  // the output level's deltas come from the loss kernel and are summed by colsum_pairs_kernel
  const bool need_bias = do1 || wgrad;
  if (need_bias) m->csum.ensure_g((size_t)2 * nrb * m->smax);
  auto csum_buf = [&](int level) { return m->csum.p + (size_t)(level & 1) * nrb * m->smax; };
  // Weight blocks (and bias blocks) of layer t only read level t+1's deltas and level t's activations, so
  // they run on the side lane concurrently with the delta GEMM of layer t (main lane), the two sharing
  // the CTA pairs in proportion to their flops. Fork: the side lane waits for level t+1's deltas; the
  // main lane's next delta GEMM waits for the bias kernel that reads the csum buffer it will overwrite;
  // join at the end.
  const bool overlap = need_bias && ctx->bwd_overlap && ctx->gemm_backend == 0 && ctx->world >= 1 && L > 1;
  if (overlap && !ctx->stream2) DHO2G_CUDA(cudaStreamCreateWithFlags(&ctx->stream2, cudaStreamNonBlocking));
  size_t evn = 0;
  cudaEvent_t bias_done = nullptr;
  int csum_level = -1;
  for (int t = L - 1; t >= 0; --t) {
    const LayerDesc& ld = m->layers[t];
    const int j = t + 1;
    const int ldD = 2 * ld.Dout, ldA = 2 * ld.Pin;
    // flops of this layer's delta GEMM (0 at t = 0) and weight GEMM, for the CTA-pair split
    const double f_delta = t == 0 ? 0.0 : (double)Bi * ld.in * (do1 ? 2.0 * ld.Dout : (double)ld.out);
    const double f_weight = (double)ld.out * ld.in * (do1 && t > 0 ? 2.0 * Bi : (double)Bi);
    if (need_bias) {
      GOp A{}, X{};
      A.hi = m->DR_hi[j].p; A.lo = m->DR_lo[j].p; A.ld = ldD; A.mn_major = 1; A.inner = ldD; A.outer = Bi;
      X.hi = m->AR_hi[t].p; X.lo = m->AR_lo[t].p; X.ld = ldA; X.mn_major = 1; X.inner = ldA; X.outer = Bi;
      A.f16 = X.f16 = m->f16;
      int K, kseg;
      if (do1) {  // hvW = RD^T A + D^T RA ; hv_b = sum_b rd (oracle.cpp:606-613)
        A.off_in[0] = ld.Dout; A.off_in[1] = 0;
        X.off_in[0] = 0; X.off_in[1] = ld.Pin;
        if (t == 0) {  // ra = 0 at the input layer
          K = kseg = Bi;
        } else {
          kseg = (int)round_up((size_t)Bi, 64);
          K = kseg + Bi;
        }
      } else {  // gW = D^T A ; g_b = sum_b d (oracle.cpp:497-504)
        K = kseg = Bi;
      }
      Epi e{};
      e.chunk_kb = m->chunk_kb;
      e.mode = EPI_STORE;
      e.M = ld.out;
      e.N = ld.in;
      e.C = out + ld.w_off;
      e.ldc = ld.in;
      e.alpha = 1.0f;
      if (m->f16) {
        e.f16 = 1;
        e.sa = m->s_dr(j);
        e.sb = m->s_ar(t);
      }
      if (m->route) {  // fused reduce-scatter (dho2g_op::apply, hvp_route)
        e.route = m->route;
        e.route_flat0 = (long long)ld.w_off;
        e.route_base = m->route_base;
        e.route_rank = m->route_rank;
      }
      auto weight_and_bias = [&]() {
        if (csum_level == j) {
          const int slot = ctx->kt_begin();
          csum_final_kernel<<<cdiv(ld.out, 128), 128, 0, ctx->stream>>>(csum_buf(j), nrb, ld.out, out + ld.b_off);
          DHO2G_LAUNCH();
          ctx->kt_end(slot, "bias_sum", 4.0 * nrb * (double)ld.out);
        } else {  // (scaled fp16: the exact fp32 deltas)
          bias_colsum(m, m->DR_hi[j].p, m->DR_lo[j].p, ldD, do1 ? ld.Dout : 0, ld.out, Bi, out + ld.b_off,
                      m->f16 ? (do1 ? m->rd32[j].p : m->d32[j].p) : nullptr);
        }
        if (overlap) {
          bias_done = lane_event(ctx, evn++);
          DHO2G_CUDA(cudaEventRecord(bias_done, ctx->stream));
        }
        gemm3x(ctx, ld.out, ld.in, K, kseg, A, X, e);
      };
      if (overlap) {
        cudaEvent_t fork = lane_event(ctx, evn++);
        DHO2G_CUDA(cudaEventRecord(fork, ctx->stream));
        DHO2G_CUDA(cudaStreamWaitEvent(ctx->stream2, fork, 0));
        const int pairs = ctx->pairs_total > 0 ? ctx->pairs_total : ctx->sm_count / 2;
        const int side = t == 0 ? 0 : std::max(1, std::min(pairs - 1, (int)std::lround(pairs * f_weight /
                                                                                          (f_weight + f_delta))));
        SideLane lane(ctx, side);
        weight_and_bias();
      } else {
        weight_and_bias();
      }
      if (overlap && t > 0) {
        // the delta GEMM below writes csum_buf(t), which the bias kernel of layer t+1 read (same parity):
        // wait for the side lane up to this layer's bias kernel (recorded before this layer's weight
        // GEMM, so the two GEMMs of layer t still run concurrently)
        DHO2G_CUDA(cudaStreamWaitEvent(ctx->stream, bias_done, 0));
        const int pairs = ctx->pairs_total > 0 ? ctx->pairs_total : ctx->sm_count / 2;
        const int side = std::max(1, std::min(pairs - 1, (int)std::lround(pairs * f_weight / (f_weight + f_delta))));
        ctx->gemm_worker_cap = pairs - side;
      }
    }
    if (t == 0) continue;
    for (int pass = 0; pass < 2; ++pass) {
      const bool r = pass == 1;
      if ((r && !do1) || (!r && !do0)) continue;
      Epi e{};
      e.chunk_kb = m->chunk_kb;
      e.mode = EPI_BWD;
      e.M = Bi;
      e.N = ld.in;
      e.do0 = !r;
      e.do1 = r;
      e.relu = m->act == 1;
      e.a_in = m->a32[t].p;
      e.ra_in = m->ra32[t].p;
      e.u_in = m->u32[t].p;
      e.u_out = wgrad ? nullptr : m->u32[t].p;  // U is only re-read by the R-epilogue of the HVP
      if (m->f16) {  // fp32 deltas + max |.|, split below with the scale that covers them
        e.f16 = 1;
        e.sa = m->s_dr(j);
        e.sb = m->s_wv(t);
        e.f0 = m->d32[t].p;
        e.f1 = m->rd32[t].p;
        e.amax = r ? m->mx_rd(t) : m->mx_d(t);  // (levels 1..L-1 cleared at the top)
      } else {
        e.f0 = nullptr;  // fp32 deltas of hidden levels are not re-read (bias blocks come from the pairs)
        e.f1 = nullptr;
        e.Rh = m->DR_hi[t].p; e.Rl = m->DR_lo[t].p; e.P = ld.Din; e.hR = r ? 1 : 0;
      }
      // column sums of the deltas this epilogue writes: rd for the Hessian's bias block, d for the gradient's
      const bool sums = (r && do1) || (!r && wgrad && !do1);
      e.csum = sums ? csum_buf(t) : nullptr;
      if (sums) csum_level = t;
      // A = [d | rd] (K-major, K = out per segment), W = [V | W] rows o read MN-major (K = out)
      GOp A = gop_k(m->DR_hi[j].p, m->DR_lo[j].p, ldD, r ? ldD : ld.Dout, Bi);
      GOp W{};
      W.hi = m->WV_hi[t].p; W.lo = m->WV_lo[t].p; W.ld = ldA; W.mn_major = 1; W.inner = ldA; W.outer = ld.out;
      A.f16 = W.f16 = m->f16;
      if (!r) {  // U = D W
        W.off_in[0] = ld.Pin;
        gemm3x(ctx, Bi, ld.in, ld.out, ld.out, A, W, e);
      } else {  // RU = D V + RD W
        A.off_in[0] = 0; A.off_in[1] = ld.Dout;
        W.off_in[0] = 0; W.off_in[1] = ld.Pin;
        gemm3x(ctx, Bi, ld.in, ld.Dout + ld.out, ld.Dout, A, W, e);
      }
      if (m->f16)  // [d | rd] of level t
        split_pair(m, Bi, ld.in, ld.Din, nullptr, nullptr, 0, m->d32[t].p, r ? m->rd32[t].p : nullptr, m->mx_d(t),
                   r ? m->mx_rd(t) : nullptr, m->s_dr(t), m->DR_hi[t].p, m->DR_lo[t].p);
    }
    if (overlap) ctx->gemm_worker_cap = 0;
  }
  if (overlap) {  // join: the caller's next launches (GS, reductions) read every weight / bias block
    cudaEvent_t join = lane_event(ctx, evn++);
    DHO2G_CUDA(cudaEventRecord(join, ctx->stream2));
    DHO2G_CUDA(cudaStreamWaitEvent(ctx->stream, join, 0));
  }
}

void mlp_grad_dev(dho2g_mlp* m, const float* w, const float* X, const float* y, const int64_t* idx, size_t B,
                  size_t ncls, double scale, float* g) {
  mlp_set_input(m, X, y, idx, B, false);
  if (mlp_small_eligible(m, B)) {
    mlp_small_run(m, 0, B, w, nullptr, nullptr, g, ncls, scale);
    return;
  }
  ensure_weights_packed(m);
  forward(m, w, B, true, false);
  output_delta(m, B, ncls, scale, true, false);
  backward(m, B, g, true, false, true);
}

// The curvature GEMMs (the HVP point and the HVPs) run with chunked TMEM accumulation (ctx gemm_chunk_kb).
struct ChunkScope {
  dho2g_mlp* m;
  explicit ChunkScope(dho2g_mlp* mm) : m(mm) { m->chunk_kb = m->ctx->gemm_chunk_kb; }
  ~ChunkScope() { m->chunk_kb = 0; }
};

void mlp_prepare_point(dho2g_mlp* m, size_t B, size_t ncls, double scale) {
  // input and weights must already be loaded (mlp_set_input / mlp_load_weights)
  if (mlp_small_eligible(m, B)) {
    mlp_small_run(m, 1, B, m->w_cur, nullptr, nullptr, nullptr, ncls, scale);
    m->prepared = m->w_cur;
    m->prepared_small = true;
    return;
  }
  ensure_input_packed(m);
  ensure_weights_packed(m);
  m->prepared_small = false;
  ChunkScope cs(m);
  forward(m, m->w_cur, B, true, false);
  output_delta(m, B, ncls, scale, true, false);
  backward(m, B, nullptr, true, false, false);
  m->prepared = m->w_cur;
}

void mlp_hvp_dev(dho2g_mlp* m, const float* v, const float* vscale, size_t B, size_t ncls, double scale, float* hv,
                 float vbound) {
  if (mlp_small_eligible(m, B)) {
    if (m->prepared != m->w_cur || !m->prepared_small) mlp_prepare_point(m, B, ncls, scale);
    mlp_small_run(m, 2, B, m->w_cur, v, vscale, hv, ncls, scale);
    return;
  }
  if (m->f16 && vbound > m->wv_vbound) {  // the W halves' scale must also cover this direction
    m->wv_vbound = vbound;
    ensure_weights_packed(m, true);
  }
  if (m->prepared != m->w_cur || m->prepared_small) mlp_prepare_point(m, B, ncls, scale);
  ChunkScope cs(m);
  m->v_bias_ptr = v;
  m->v_scale_ptr = vscale;
  mlp_load_direction(m, v, vscale);
  forward(m, m->w_cur, B, false, true);
  output_delta(m, B, ncls, scale, false, true);
  backward(m, B, hv, false, true, false);
}

void mlp_eval_dev(dho2g_mlp* m, const float* w, const float* X, const float* y, const int64_t* idx, size_t B,
                  size_t ncls, double* acc2) {
  mlp_set_input(m, X, y, idx, B, false);
  if (mlp_small_eligible(m, B)) {
    mlp_small_run(m, 3, B, w, nullptr, nullptr, nullptr, ncls, 1.0);
  } else {
    ensure_weights_packed(m);
    forward(m, w, B, true, false);
    output_delta(m, B, ncls, 1.0, true, false);
  }
  eval_reduce_kernel<<<1, 1024, 0, m->ctx->stream>>>((int)B, m->sample_loss.p, m->sample_correct.p, acc2);
  DHO2G_LAUNCH();
}

void mlp_loss_sum(dho2g_mlp* m, size_t B, double* acc2) {
  DHO2G_CUDA(cudaMemsetAsync(acc2, 0, 2 * sizeof(double), m->ctx->stream));
  eval_reduce_kernel<<<1, 1024, 0, m->ctx->stream>>>((int)B, m->sample_loss.p, m->sample_correct.p, acc2);
  DHO2G_LAUNCH();
}

}  // namespace dho2g
