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

// Bias block as a column sum of a row-major pair buffer: out[o] = sum_{b < B} (hi + lo)[b][off + o].
// Blocks of 64 columns (2 per lane, bf16x2 loads) x 8 row groups over one of kColChunks row chunks
// write fp64 partials part[chunk][o]; the last block of each column block (ticket) adds the chunks
// in order (deterministic, one launch).
constexpr int kColChunks = 32;
__global__ void colsum_pairs_kernel(const bf16* __restrict__ hi, const bf16* __restrict__ lo, int ld, int off,
                                    int cols, int B, double* __restrict__ part, unsigned* __restrict__ tickets,
                                    float* __restrict__ out) {
  __shared__ double sh[8][64];
  __shared__ bool last;
  const int c = blockIdx.x * 64 + 2 * threadIdx.x;
  const int rows_per = (B + kColChunks - 1) / kColChunks;
  const int r0 = blockIdx.y * rows_per, r1 = min(B, r0 + rows_per);
  float a0 = 0.f, a1 = 0.f;
  if (c < cols) {
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
    const int slot = ctx->kt_begin();
    // one wave of resident blocks striding over the rows (short-lived per-row blocks cost more than the copy)
    const int gx = (int)cdiv(ld.in, 128 * kPackPer);
    const int gy = std::max(1, std::min(ld.out, ctx->sm_count * 16 / gx));
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

void mlp_load_weights(dho2g_mlp* m, const float* w) {
  m->w_cur = w;
  m->prepared = nullptr;
  pack_params(m, w, nullptr, 1);
}

void mlp_load_direction(dho2g_mlp* m, const float* v, const float* vscale) { pack_params(m, v, vscale, 0); }

void mlp_presize(dho2g_mlp* m, size_t B) {
  m->ensure_batch(B);
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

void mlp_set_input(dho2g_mlp* m, const float* X, const float* y, const int64_t* idx, size_t B, bool /*with_r*/) {
  m->ensure_batch(B);
  m->input_owner = nullptr;
  m->prepared = nullptr;
  const int s0 = (int)m->sizes[0];
  pack_rows(m->ctx, (int)B, s0, (int)round_up(s0, 8), X, idx, s0, nullptr, m->AR_hi[0].p, m->AR_lo[0].p);
  gather_labels_kernel<<<cdiv(B, 256), 256, 0, m->ctx->stream>>>((int)B, y, idx, m->lab.p);
  DHO2G_LAUNCH();
}

// Forward pass. do0: plain activations (Z GEMM + fused bias/act epilogue). do1: R-activations
// (RZ GEMM + fused R-epilogue over the cached activations).
static void forward(dho2g_mlp* m, const float* w, size_t B, bool do0, bool do1) {
  dho2g_ctx* ctx = m->ctx;
  for (int t = 0; t < m->L; ++t) {
    const LayerDesc& ld = m->layers[t];
    if (m->pack_pending) DHO2G_CUDA(cudaStreamWaitEvent(ctx->stream, m->pack_ev[t], 0));  // layer t packed
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
      }
      if (!r)  // Z = A W^T
        gemm3(ctx, (int)B, ld.out, ld.in, m->AR_hi[t].p, m->AR_lo[t].p, lda, m->WV_hi[t].p + ld.Pin,
              m->WV_lo[t].p + ld.Pin, lda, e);
      else  // RZ = [A | RA] [V | W]^T (ra = 0 at the input layer: K = in only)
        gemm3(ctx, (int)B, ld.out, t == 0 ? ld.in : 2 * ld.Pin, m->AR_hi[t].p, m->AR_lo[t].p, lda, m->WV_hi[t].p,
              m->WV_lo[t].p, lda, e);
    }
  }
  m->pack_pending = false;  // every layer's event has been waited on by the main stream
}

static void output_delta(dho2g_mlp* m, size_t B, size_t ncls, double scale, bool do0, bool do1) {
  const int L = m->L;
  const int O = (int)m->sizes[L];
  output_delta_kernel<<<cdiv(B, 128), 128, 0, m->ctx->stream>>>((int)B, O, m->loss, (int)ncls, do0, do1, scale,
                                                                   m->a32[L].p, m->ra32[L].p, m->lab.p, m->d32[L].p,
                                                                   m->rd32[L].p, m->sample_loss.p,
                                                                   m->sample_correct.p);
  DHO2G_LAUNCH();
  pack_rows(m->ctx, (int)B, O, (int)round_up(O, 64), do0 ? m->d32[L].p : nullptr, nullptr, O,
            do1 ? m->rd32[L].p : nullptr, m->DR_hi[L].p, m->DR_lo[L].p);
}

static void bias_colsum(dho2g_mlp* m, const bf16* hi, const bf16* lo, int ld, int off, int cols, int B, float* out) {
  dho2g_ctx* ctx = m->ctx;
  m->colpart.ensure_g((size_t)kColChunks * cols);
  m->coltickets.ensure_g(cdiv(cols, 64));  // zeroed at allocation; each launch leaves them zero
  const int slot = ctx->kt_begin();
  colsum_pairs_kernel<<<dim3(cdiv(cols, 64), kColChunks), dim3(32, 8), 0, ctx->stream>>>(
      hi, lo, ld, off, cols, B, m->colpart.p, m->coltickets.p, out);
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
      e.mode = EPI_STORE;
      e.M = ld.out;
      e.N = ld.in;
      e.C = out + ld.w_off;
      e.ldc = ld.in;
      e.alpha = 1.0f;
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
        } else {
          bias_colsum(m, m->DR_hi[j].p, m->DR_lo[j].p, ldD, do1 ? ld.Dout : 0, ld.out, Bi, out + ld.b_off);
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
      e.f0 = nullptr;  // fp32 deltas of hidden levels are not re-read (bias blocks come from the pairs)
      e.f1 = nullptr;
      e.Rh = m->DR_hi[t].p; e.Rl = m->DR_lo[t].p; e.P = ld.Din; e.hR = r ? 1 : 0;
      // column sums of the deltas this epilogue writes: rd for the Hessian's bias block, d for the gradient's
      const bool sums = (r && do1) || (!r && wgrad && !do1);
      e.csum = sums ? csum_buf(t) : nullptr;
      if (sums) csum_level = t;
      // A = [d | rd] (K-major, K = out per segment), W = [V | W] rows o read MN-major (K = out)
      GOp A = gop_k(m->DR_hi[j].p, m->DR_lo[j].p, ldD, r ? ldD : ld.Dout, Bi);
      GOp W{};
      W.hi = m->WV_hi[t].p; W.lo = m->WV_lo[t].p; W.ld = ldA; W.mn_major = 1; W.inner = ldA; W.outer = ld.out;
      if (!r) {  // U = D W
        W.off_in[0] = ld.Pin;
        gemm3x(ctx, Bi, ld.in, ld.out, ld.out, A, W, e);
      } else {  // RU = D V + RD W
        A.off_in[0] = 0; A.off_in[1] = ld.Dout;
        W.off_in[0] = 0; W.off_in[1] = ld.Pin;
        gemm3x(ctx, Bi, ld.in, ld.Dout + ld.out, ld.Dout, A, W, e);
      }
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
