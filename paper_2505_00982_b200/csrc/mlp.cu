// Device MLP oracle (reference: proj/src/oracle.cpp:288-687) — forward, backward and the
// Pearlmutter R-op as batched split-BF16x3 GEMMs plus fused tile epilogues.
//
// Layout (reference oracle.cpp:304-324): flat params, per layer W (out x in, row-major) then b.
// Per layer t with in = s_t, out = s_{t+1} the contractions are (B = batch):
//   forward    Z  = A W^T            RZ = [A | RA] [V | W]^T         (K = in, 2 in)
//   backward   U  = D W              RU = [D | RD] [V^T | W^T]^T     (K = out, 2 out)
//   weight     hvW = [RD^T | D^T] [A^T | RA^T]^T                     (K = 2B)
// with every operand stored K-major as (hi, lo) bf16 pairs so all GEMMs are "TN" for tcgen05.
//
// A Lanczos refresh applies H at ONE point w on ONE curvature batch m times, so everything that
// does not depend on the direction v (A, Z, softmax, D, U for every layer) is computed once by
// mlp_prepare_point() and cached; each mlp_hvp_cached() then only runs the R-GEMMs (RZ, RU) and the
// weight-block GEMM: 6 of the 8 per-layer GEMM units of oracle.cpp:524-647 (2 of 3 at layer 0).
#include <cmath>

#include "internal.h"

using namespace dho2g;

void dho2g_mlp::ensure_batch(size_t B) {
  if (B <= Bcap) return;
  const size_t nB = round_up(B, 128);
  const size_t nBp = round_up(nB, 8);
  const int Ls = L;
  AR_hi.resize(Ls); AR_lo.resize(Ls); ART_hi.resize(Ls); ART_lo.resize(Ls);
  DR_hi.resize(Ls + 1); DR_lo.resize(Ls + 1); DRT_hi.resize(Ls + 1); DRT_lo.resize(Ls + 1);
  a32.resize(Ls + 1); ra32.resize(Ls + 1); d32.resize(Ls + 1); rd32.resize(Ls + 1); u32.resize(Ls + 1);
  for (int j = 0; j <= Ls; ++j) {
    const size_t s = sizes[j], P = round_up(s, 8);
    if (j < Ls) {
      AR_hi[j].alloc(nB * 2 * P); AR_lo[j].alloc(nB * 2 * P);
      ART_hi[j].alloc((s + 1) * 2 * nBp); ART_lo[j].alloc((s + 1) * 2 * nBp);  // + ones row (bias grads)
    }
    if (j >= 1) {
      DR_hi[j].alloc(nB * 2 * P); DR_lo[j].alloc(nB * 2 * P);
      DRT_hi[j].alloc(s * 2 * nBp); DRT_lo[j].alloc(s * 2 * nBp);
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
  Bpcap = nBp;
  prepared = nullptr;
  ones_B = 0;
}

namespace {

constexpr int TILE = 32;

// ------------------------------------------------------------------ weight operand packing
// WV[t][o][h*Pin + k] = p(o,k) (k < in, zero-padded to Pin); WVt[t][k][h*Pout + o] likewise.
__global__ void pack_weights_kernel(const float* __restrict__ p, const float* __restrict__ pscale, int in, int out,
                                    int Pin, int Pout, int half, bf16* __restrict__ WVh, bf16* __restrict__ WVl,
                                    bf16* __restrict__ WVth, bf16* __restrict__ WVtl) {
  __shared__ float sh[TILE][TILE + 1];
  const int k0 = blockIdx.x * TILE, o0 = blockIdx.y * TILE;
  const float sc = pscale ? *pscale : 1.0f;
  for (int i = threadIdx.y; i < TILE; i += blockDim.y) {
    const int o = o0 + i, k = k0 + threadIdx.x;
    float x = 0.f;
    if (o < out && k < in) x = p[(size_t)o * in + k] * sc;
    sh[i][threadIdx.x] = x;
    if (o < out && k < Pin) {
      bf16 h, l;
      split_bf16(x, h, l);
      const size_t idx = (size_t)o * (2 * Pin) + (size_t)half * Pin + k;
      WVh[idx] = h;
      WVl[idx] = l;
    }
  }
  if (!WVth) return;
  __syncthreads();
  for (int i = threadIdx.y; i < TILE; i += blockDim.y) {
    const int k = k0 + i, o = o0 + threadIdx.x;
    if (k < in && o < Pout) {
      const float x = sh[threadIdx.x][i];
      bf16 h, l;
      split_bf16(x, h, l);
      const size_t idx = (size_t)k * (2 * Pout) + (size_t)half * Pout + o;
      WVth[idx] = h;
      WVtl[idx] = l;
    }
  }
}

// ------------------------------------------------------------------ activation tile epilogues
enum Mode { M_INPUT = 0, M_FWD = 1, M_FWD_OUT = 2, M_BWD = 3, M_DPACK = 4 };

struct TileArgs {
  int B, s, P, Bp, ldT;  // batch, width, half width, padded batch, transposed row stride
  bool do0, do1, relu;   // compute/pack the plain (x0) and/or the R (x1) quantity
  // sources
  const float* X; const int64_t* idx; int ldX;  // M_INPUT
  const float* Zs; const float* RZs;             // GEMM outputs (B x s): Z or U, RZ or RU
  const float* bias; const float* vbias; const float* vscale;
  const float* a_in; const float* ra_in;         // cached activations of this level
  const float* u_in;                             // cached U (M_BWD with !do0)
  const float* d_in; const float* rd_in;         // M_DPACK
  // fp32 outputs (B x s)
  float* o0; float* o1; float* u_out;
  // packed outputs
  bf16 *Rh, *Rl;   // row-major pairs (B x 2P): x0 -> half 0, x1 -> half 1
  bf16 *Th, *Tl;   // transposed pairs (s x ldT): x0 -> half t0, x1 -> half t1
  int t0, t1;
};

template <int MODE>
__global__ void tile_epilogue_kernel(TileArgs a) {
  __shared__ float s0[TILE][TILE + 1], s1[TILE][TILE + 1];
  const int k0 = blockIdx.x * TILE, b0 = blockIdx.y * TILE;
  const float vsc = (a.vscale && a.do1) ? *a.vscale : 1.0f;
  for (int i = threadIdx.y; i < TILE; i += blockDim.y) {
    const int b = b0 + i, k = k0 + threadIdx.x;
    float x0 = 0.f, x1 = 0.f;
    if (b < a.B && k < a.s) {
      const size_t e = (size_t)b * a.s + k;
      if (MODE == M_INPUT) {
        const int64_t row = a.idx ? a.idx[b] : b;
        x0 = a.X[(size_t)row * a.ldX + k];
      } else if (MODE == M_FWD || MODE == M_FWD_OUT) {
        // oracle.cpp:548-563: z = b + W a ; a' = act(z) ; ra' = act'(a') (v_b + V a + W ra)
        if (a.do0) {
          const float z = a.Zs[e] + a.bias[k];
          x0 = MODE == M_FWD_OUT ? z : (a.relu ? fmaxf(z, 0.f) : tanhf(z));
          a.o0[e] = x0;
        } else {
          x0 = a.a_in[e];
        }
        if (a.do1) {
          const float rz = a.RZs[e] + vsc * a.vbias[k];
          if (MODE == M_FWD_OUT) {
            x1 = rz;
          } else {
            const float ap = a.relu ? (x0 > 0.f ? 1.f : 0.f) : 1.f - x0 * x0;
            x1 = ap * rz;
          }
          a.o1[e] = x1;
        }
      } else if (MODE == M_BWD) {
        // oracle.cpp:626-635: d = u act'(a); rd = ru act'(a) + u (-2 a ra) (tanh only)
        const float av = a.a_in[e];
        const float ap = a.relu ? (av > 0.f ? 1.f : 0.f) : 1.f - av * av;
        float u;
        if (a.do0) {
          u = a.Zs[e];
          x0 = u * ap;
          a.o0[e] = x0;
          if (a.u_out) a.u_out[e] = u;
        } else {
          u = a.u_in[e];
        }
        if (a.do1) {
          float rap = 0.f;
          if (!a.relu && ap != 0.f) rap = -2.f * av * a.ra_in[e];
          x1 = a.RZs[e] * ap + u * rap;
          a.o1[e] = x1;
        }
      } else {  // M_DPACK
        if (a.do0) x0 = a.d_in[e];
        if (a.do1) x1 = a.rd_in[e];
      }
    }
    if (MODE == M_FWD_OUT) continue;
    s0[i][threadIdx.x] = x0;
    s1[i][threadIdx.x] = x1;
    if (b < a.B && k < a.P && a.Rh) {
      bf16 h, l;
      const size_t r = (size_t)b * (2 * a.P) + k;
      if (a.do0) {
        split_bf16(x0, h, l);
        a.Rh[r] = h;
        a.Rl[r] = l;
      }
      if (a.do1) {
        split_bf16(x1, h, l);
        a.Rh[r + a.P] = h;
        a.Rl[r + a.P] = l;
      }
    }
  }
  if (MODE == M_FWD_OUT || !a.Th) return;
  __syncthreads();
  for (int i = threadIdx.y; i < TILE; i += blockDim.y) {
    const int k = k0 + i, b = b0 + threadIdx.x;
    if (k < a.s && b < a.Bp) {
      const size_t r = (size_t)k * a.ldT + b;
      bf16 h, l;
      if (a.do0 && a.t0 >= 0) {
        split_bf16(s0[threadIdx.x][i], h, l);
        a.Th[r + (size_t)a.t0 * a.Bp] = h;
        a.Tl[r + (size_t)a.t0 * a.Bp] = l;
      }
      if (a.do1 && a.t1 >= 0) {
        split_bf16(s1[threadIdx.x][i], h, l);
        a.Th[r + (size_t)a.t1 * a.Bp] = h;
        a.Tl[r + (size_t)a.t1 * a.Bp] = l;
      }
    }
  }
}

template <int MODE>
void launch_tile(dho2g_ctx* ctx, const TileArgs& a) {
  dim3 grid(cdiv(std::max(a.P, a.s), TILE), cdiv(std::max(a.Bp, a.B), TILE));
  const int slot = ctx->kt_begin();
  tile_epilogue_kernel<MODE><<<grid, dim3(TILE, 8), 0, ctx->stream>>>(a);
  DHO2G_LAUNCH();
  ctx->kt_end(slot, "tile_epilogue", 0.0);
}

// ------------------------------------------------------------------ output layer delta
// oracle.cpp:476-495 (delta) and :572-599 (R-delta); also per-sample loss / correctness.
__global__ void output_delta_kernel(int B, int O, int mse, int ncls, int do0, int do1, double scale,
                                    const float* __restrict__ z, const float* __restrict__ rz,
                                    const float* __restrict__ lab, float* __restrict__ d, float* __restrict__ rd,
                                    double* __restrict__ loss, int* __restrict__ correct) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  const float* o = z + (size_t)b * O;
  const float* ro = do1 ? rz + (size_t)b * O : nullptr;
  float* dd = d + (size_t)b * O;
  float* rdd = do1 ? rd + (size_t)b * O : nullptr;
  const float y = lab[b];
  int best = 0;
  for (int j = 1; j < O; ++j)
    if (o[j] > o[best]) best = j;
  if (do0) correct[b] = (ncls > 0 && best == (int)y) ? 1 : 0;
  if (!mse) {
    const int lbl = (int)y;
    const float mx = o[best];
    double den = 0.0;
    for (int j = 0; j < O; ++j) den += exp((double)o[j] - (double)mx);
    double sdot = 0.0;
    for (int j = 0; j < O; ++j) {
      const double soft = exp((double)o[j] - (double)mx) / den;
      if (do0) dd[j] = (float)((soft - (j == lbl ? 1.0 : 0.0)) * scale);
      if (do1) sdot += soft * ro[j];
    }
    if (do1)
      for (int j = 0; j < O; ++j) {
        const double soft = exp((double)o[j] - (double)mx) / den;
        rdd[j] = (float)(soft * (ro[j] - sdot) * scale);
      }
    if (do0) loss[b] = (double)mx + log(den) - (double)o[lbl];
  } else {
    double acc = 0.0;
    for (int j = 0; j < O; ++j) {
      const float t = ncls > 0 ? (j == (int)y ? 1.f : 0.f) : (j == 0 ? y : 0.f);
      const float df = o[j] - t;
      if (do0) dd[j] = (float)(df * scale);
      if (do1) rdd[j] = (float)(ro[j] * scale);
      acc += 0.5 * (double)df * (double)df;
    }
    if (do0) loss[b] = acc;
  }
}

__global__ void ones_row_kernel(bf16* __restrict__ hi, bf16* __restrict__ lo, int len, int B) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= len) return;
  hi[i] = __float2bfloat16_rn(i < B ? 1.f : 0.f);
  lo[i] = __float2bfloat16_rn(0.f);
}

// Bias gradient as a row sum of the weight GEMM's A operand pair: out[o] = alpha * sum_k (hi + lo)[o][k]
// over k < K (K % 8 == 0, rows 16-byte aligned). One warp per row, fp64 accumulation, fixed order.
__global__ void rowsum_pairs_kernel(const bf16* __restrict__ hi, const bf16* __restrict__ lo, int ld, int rows, int K,
                                    float alpha, float* __restrict__ out) {
  const int o = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (o >= rows) return;
  const uint4* ph = reinterpret_cast<const uint4*>(hi + (size_t)o * ld);
  const uint4* pl = reinterpret_cast<const uint4*>(lo + (size_t)o * ld);
  double acc = 0.0;
#pragma unroll 4
  for (int i = lane; i < K / 8; i += 32) {
    const uint4 a = __ldg(ph + i), b = __ldg(pl + i);
    const bf16* ha = reinterpret_cast<const bf16*>(&a);
    const bf16* hb = reinterpret_cast<const bf16*>(&b);
    float f = 0.f;
#pragma unroll
    for (int j = 0; j < 8; ++j) f += __bfloat162float(ha[j]) + __bfloat162float(hb[j]);
    acc += (double)f;
  }
  acc = warp_sum(acc);
  if (lane == 0) out[o] = (float)(alpha * acc);
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

static void pack_params(dho2g_mlp* m, const float* p, const float* pscale, int half) {
  cudaStream_t st = m->ctx->stream;
  for (int t = 0; t < m->L; ++t) {
    const LayerDesc& ld = m->layers[t];
    dim3 grid(cdiv(std::max(ld.Pin, ld.in), TILE), cdiv(std::max(ld.Pout, ld.out), TILE));
    const int slot = m->ctx->kt_begin();
    pack_weights_kernel<<<grid, dim3(TILE, 8), 0, st>>>(p + ld.w_off, pscale, ld.in, ld.out, ld.Pin, ld.Pout, half,
                                                        m->WV_hi[t].p, m->WV_lo[t].p, t > 0 ? m->WVt_hi[t].p : nullptr,
                                                        t > 0 ? m->WVt_lo[t].p : nullptr);
    DHO2G_LAUNCH();
    // algorithmic bytes: read fp32 (4) + write hi/lo to both layouts (2 x 4)
    m->ctx->kt_end(slot, "pack_params", (double)ld.in * ld.out * (t > 0 ? 12.0 : 8.0));
  }
}

void mlp_load_weights(dho2g_mlp* m, const float* w) {
  m->w_cur = w;
  m->prepared = nullptr;
  pack_params(m, w, nullptr, 1);
}

void mlp_load_direction(dho2g_mlp* m, const float* v, const float* vscale) { pack_params(m, v, vscale, 0); }

void mlp_set_input(dho2g_mlp* m, const float* X, const float* y, const int64_t* idx, size_t B, bool /*with_r*/) {
  m->ensure_batch(B);
  m->input_owner = nullptr;
  m->prepared = nullptr;
  cudaStream_t st = m->ctx->stream;
  TileArgs a{};
  const int s0 = (int)m->sizes[0];
  a.B = (int)B; a.s = s0; a.P = (int)round_up(s0, 8); a.Bp = (int)round_up(B, 8); a.ldT = (int)(2 * m->Bpcap);
  a.do0 = true; a.do1 = false;
  a.X = X; a.idx = idx; a.ldX = s0;
  a.Rh = m->AR_hi[0].p; a.Rl = m->AR_lo[0].p; a.Th = m->ART_hi[0].p; a.Tl = m->ART_lo[0].p;
  a.t0 = 0; a.t1 = -1;
  launch_tile<M_INPUT>(m->ctx, a);
  if (m->ones_B != B) {  // ones row of every transposed activation buffer: [1 (B) 0 (Bp-B) | 0 (Bp)]
    for (int j = 0; j < m->L; ++j)
      ones_row_kernel<<<cdiv(2 * m->Bpcap, 256), 256, 0, st>>>(m->ART_hi[j].p + m->sizes[j] * 2 * m->Bpcap,
                                                              m->ART_lo[j].p + m->sizes[j] * 2 * m->Bpcap,
                                                              (int)(2 * m->Bpcap), (int)B);
    DHO2G_LAUNCH();
    m->ones_B = B;
  }
  gather_labels_kernel<<<cdiv(B, 256), 256, 0, st>>>((int)B, y, idx, m->lab.p);
  DHO2G_LAUNCH();
}

// Forward pass. do0: plain activations (Z GEMM + fused bias/act epilogue). do1: R-activations
// (RZ GEMM + fused R-epilogue over the cached activations).
static void forward(dho2g_mlp* m, const float* w, size_t B, bool do0, bool do1) {
  dho2g_ctx* ctx = m->ctx;
  const int Bp = (int)round_up(B, 8);
  for (int t = 0; t < m->L; ++t) {
    const LayerDesc& ld = m->layers[t];
    const bool last = t + 1 == m->L;
    const int lda = 2 * ld.Pin;
    for (int pass = 0; pass < 2; ++pass) {
      const bool r = pass == 1;
      if ((r && !do1) || (!r && !do0)) continue;
      Epi e{};
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
      if (!last) {
        e.Rh = m->AR_hi[t + 1].p; e.Rl = m->AR_lo[t + 1].p; e.P = ld.Pout; e.hR = r ? 1 : 0;
        e.Th = m->ART_hi[t + 1].p; e.Tl = m->ART_lo[t + 1].p; e.ldT = (int)(2 * m->Bpcap); e.Bp = Bp; e.hT = r ? 1 : 0;
      }
      if (!r)  // Z = A W^T
        gemm3(ctx, (int)B, ld.out, ld.in, m->AR_hi[t].p, m->AR_lo[t].p, lda, m->WV_hi[t].p + ld.Pin,
              m->WV_lo[t].p + ld.Pin, lda, e);
      else  // RZ = [A | RA] [V | W]^T (ra = 0 at the input layer: K = in only)
        gemm3(ctx, (int)B, ld.out, t == 0 ? ld.in : 2 * ld.Pin, m->AR_hi[t].p, m->AR_lo[t].p, lda, m->WV_hi[t].p,
              m->WV_lo[t].p, lda, e);
    }
  }
}

static void output_delta(dho2g_mlp* m, size_t B, size_t ncls, double scale, bool do0, bool do1) {
  const int L = m->L;
  const int O = (int)m->sizes[L];
  output_delta_kernel<<<cdiv(B, 128), 128, 0, m->ctx->stream>>>((int)B, O, m->loss, (int)ncls, do0, do1, scale,
                                                                   m->a32[L].p, m->ra32[L].p, m->lab.p, m->d32[L].p,
                                                                   m->rd32[L].p, m->sample_loss.p,
                                                                   m->sample_correct.p);
  DHO2G_LAUNCH();
  TileArgs a{};
  const int s = O;
  a.B = (int)B; a.s = s; a.P = (int)round_up(s, 8); a.Bp = (int)round_up(B, 8); a.ldT = (int)(2 * m->Bpcap);
  a.do0 = do0; a.do1 = do1;
  a.Rh = m->DR_hi[L].p; a.Rl = m->DR_lo[L].p; a.Th = m->DRT_hi[L].p; a.Tl = m->DRT_lo[L].p;
  a.t0 = 1; a.t1 = 0;  // transposed pair is [rd^T | d^T]
  a.d_in = m->d32[L].p; a.rd_in = m->rd32[L].p;
  launch_tile<M_DPACK>(m->ctx, a);
}

// Backward pass. do0: deltas d (U GEMMs + fused act' epilogue) and, if wgrad, the gradient blocks.
// do1: R-deltas (RU GEMMs + fused R-epilogue) and the Hessian blocks into `out`. The weight-block
// GEMMs take the bias column from the ones row appended to the transposed activations
// (N = in + 1: column `in` = sum_b rd (or d), routed to out[b_off + o]).
static void bias_rowsum(dho2g_ctx* ctx, const bf16* hi, const bf16* lo, int ld, int rows, int K, float* out) {
  const int slot = ctx->kt_begin();
  rowsum_pairs_kernel<<<cdiv(rows, 8), 256, 0, ctx->stream>>>(hi, lo, ld, rows, K, 1.0f, out);
  DHO2G_LAUNCH();
  ctx->kt_end(slot, "bias_rowsum", 4.0 * rows * (double)K);  // algorithmic bytes: hi + lo
}

static void backward(dho2g_mlp* m, size_t B, float* out, bool do0, bool do1, bool wgrad) {
  dho2g_ctx* ctx = m->ctx;
  const int L = m->L;
  const int Bp = (int)round_up(B, 8);
  const int ldT = (int)(2 * m->Bpcap);
  for (int t = L - 1; t >= 0; --t) {
    const LayerDesc& ld = m->layers[t];
    const int j = t + 1;
    // weight block by GEMM; the bias block (sum over the batch of the A operand's first half) by a
    // row sum, which keeps the GEMM's N a multiple of the tile width
    if (do1) {  // hvW = [RD^T | D^T] [A^T | RA^T]^T ; hv_b = sum_b rd (oracle.cpp:606-613)
      gemm3_store(ctx, ld.out, ld.in, t == 0 ? Bp : 2 * Bp, m->DRT_hi[j].p, m->DRT_lo[j].p, ldT, m->ART_hi[t].p,
                  m->ART_lo[t].p, ldT, out + ld.w_off, ld.in, 1.0f);
      bias_rowsum(ctx, m->DRT_hi[j].p, m->DRT_lo[j].p, ldT, ld.out, Bp, out + ld.b_off);
    } else if (wgrad) {  // gW = D^T A ; g_b = sum_b d (oracle.cpp:497-504)
      gemm3_store(ctx, ld.out, ld.in, Bp, m->DRT_hi[j].p + Bp, m->DRT_lo[j].p + Bp, ldT, m->ART_hi[t].p,
                  m->ART_lo[t].p, ldT, out + ld.w_off, ld.in, 1.0f);
      bias_rowsum(ctx, m->DRT_hi[j].p + Bp, m->DRT_lo[j].p + Bp, ldT, ld.out, Bp, out + ld.b_off);
    }
    if (t == 0) continue;
    const int lda = 2 * ld.Pout;
    for (int pass = 0; pass < 2; ++pass) {
      const bool r = pass == 1;
      if ((r && !do1) || (!r && !do0)) continue;
      Epi e{};
      e.mode = EPI_BWD;
      e.M = (int)B;
      e.N = ld.in;
      e.do0 = !r;
      e.do1 = r;
      e.relu = m->act == 1;
      e.a_in = m->a32[t].p;
      e.ra_in = m->ra32[t].p;
      e.u_in = m->u32[t].p;
      e.u_out = wgrad ? nullptr : m->u32[t].p;  // U is only re-read by the R-epilogue of the HVP
      e.f0 = nullptr;  // fp32 deltas of hidden levels are not re-read (bias grads come from the GEMM)
      e.f1 = nullptr;
      e.Rh = m->DR_hi[t].p; e.Rl = m->DR_lo[t].p; e.P = ld.Pin; e.hR = r ? 1 : 0;
      e.Th = m->DRT_hi[t].p; e.Tl = m->DRT_lo[t].p; e.ldT = ldT; e.Bp = Bp; e.hT = r ? 0 : 1;  // [rd^T | d^T]
      if (!r)  // U = D W
        gemm3(ctx, (int)B, ld.in, ld.out, m->DR_hi[j].p, m->DR_lo[j].p, lda, m->WVt_hi[t].p + ld.Pout,
              m->WVt_lo[t].p + ld.Pout, lda, e);
      else  // RU = [D | RD] [V^T | W^T]^T
        gemm3(ctx, (int)B, ld.in, 2 * ld.Pout, m->DR_hi[j].p, m->DR_lo[j].p, lda, m->WVt_hi[t].p, m->WVt_lo[t].p, lda,
              e);
    }
  }
}

void mlp_grad_dev(dho2g_mlp* m, const float* w, const float* X, const float* y, const int64_t* idx, size_t B,
                  size_t ncls, double scale, float* g) {
  mlp_set_input(m, X, y, idx, B, false);
  forward(m, w, B, true, false);
  output_delta(m, B, ncls, scale, true, false);
  backward(m, B, g, true, false, true);
}

void mlp_prepare_point(dho2g_mlp* m, size_t B, size_t ncls, double scale) {
  // input and weights must already be loaded (mlp_set_input / mlp_load_weights)
  forward(m, m->w_cur, B, true, false);
  output_delta(m, B, ncls, scale, true, false);
  backward(m, B, nullptr, true, false, false);
  m->prepared = m->w_cur;
}

void mlp_hvp_dev(dho2g_mlp* m, const float* v, const float* vscale, size_t B, size_t ncls, double scale, float* hv) {
  if (m->prepared != m->w_cur) mlp_prepare_point(m, B, ncls, scale);
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
  forward(m, w, B, true, false);
  output_delta(m, B, ncls, 1.0, true, false);
  eval_reduce_kernel<<<1, 1024, 0, m->ctx->stream>>>((int)B, m->sample_loss.p, m->sample_correct.p, acc2);
  DHO2G_LAUNCH();
}

void mlp_loss_sum(dho2g_mlp* m, size_t B, double* acc2) {
  DHO2G_CUDA(cudaMemsetAsync(acc2, 0, 2 * sizeof(double), m->ctx->stream));
  eval_reduce_kernel<<<1, 1024, 0, m->ctx->stream>>>((int)B, m->sample_loss.p, m->sample_correct.p, acc2);
  DHO2G_LAUNCH();
}

}  // namespace dho2g
