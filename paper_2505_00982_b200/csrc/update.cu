// FOSI / ADMM split update with the base optimizer (reference: proj/src/optimizer.cpp:37-154),
// fused into three bandwidth-bound passes over this rank's rows:
//   P1  c = V^T (g + pi)                                    reads V, g, pi
//   P2  g2 = g~ - V c ; s = base_step(g2) ; sc = V^T s       reads V, g, pi, moments(, w); writes moments, s
//   P3  w_a += (s - V sc) + (-alpha V (c / den))             reads V, s, w_a; writes w_a
// with the r-length reductions (c, sc) as fp64 partials + all_gather + rank-ordered sums.
#include <cmath>

#include "internal.h"

using namespace dho2g;

namespace {

constexpr int kT = 256;
constexpr int kW = kT / 32;
constexpr int kCh = 1024;  // rows staged per chunk

__device__ __forceinline__ double floored_den(double a, double fl, double sigma) {  // optimizer.cpp:75-79, :94-98
  double f;
  if (a == 0.0) f = fl;
  else {
    const double mag = fabs(a) > fl ? fabs(a) : fl;
    f = a < 0.0 ? -mag : mag;
  }
  double den = f + sigma;
  if (fabs(den) < fl) den = den < 0.0 ? -fl : fl;
  return den;
}

// grid-level deterministic reduction helper: per-CTA partial rows -> rank partial via ticket
__device__ void finish_partials(const double* acc_w /* [kW][nj] */, int nj, double* part, double* rankp,
                                unsigned* ticket) {
  __shared__ bool is_last;
  for (int j = threadIdx.x; j < nj; j += kT) {
    double t = 0.0;
    for (int w = 0; w < kW; ++w) t += acc_w[w * nj + j];
    part[(size_t)blockIdx.x * nj + j] = t;
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) is_last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!is_last) return;
  __threadfence();
  for (int j = threadIdx.x; j < nj; j += kT) {
    double t = 0.0;
    for (int b = 0; b < (int)gridDim.x; ++b) t += part[(size_t)b * nj + j];
    rankp[j] = t;
  }
  if (threadIdx.x == 0) *ticket = 0u;
}

// chunk-staged dots: acc[w][j] += V_j[chunk] . x[chunk] for x staged in smem
__device__ __forceinline__ void chunk_dots(const float* __restrict__ V, size_t ldv, size_t r0, int R,
                                           const float* xs, double* acc) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int items = R * (kCh / 128);
  for (int it = warp; it < items; it += kW) {
    const int j = it / (kCh / 128), q = it % (kCh / 128);
    const int rb = q * 128 + lane * 4;
    const float4 x = __ldg(reinterpret_cast<const float4*>(V + (size_t)j * ldv + r0 + rb));
    const float4 y = *reinterpret_cast<const float4*>(xs + rb);
    double s = (double)x.x * y.x + (double)x.y * y.y + (double)x.z * y.z + (double)x.w * y.w;
    s = warp_sum(s);
    if (lane == 0) acc[warp * R + j] += s;
  }
}

// ---- P1: c = V^T (g + pi)
__global__ void __launch_bounds__(kT) upd_p1_kernel(const float* __restrict__ V, size_t ldv, int R, size_t rows,
                                                    const float* __restrict__ g, const float* __restrict__ pi,
                                                    double* part, double* rankp, unsigned* ticket) {
  extern __shared__ __align__(16) unsigned char smem[];
  float* xs = reinterpret_cast<float*>(smem);
  double* acc = reinterpret_cast<double*>(smem + kCh * sizeof(float));
  for (int e = threadIdx.x; e < kW * R; e += kT) acc[e] = 0.0;
  const size_t nch = cdiv(rows, kCh);
  for (size_t c = blockIdx.x; c < nch; c += gridDim.x) {
    const size_t r0 = c * kCh;
    __syncthreads();
    for (int e = threadIdx.x; e < kCh; e += kT) {
      const size_t r = r0 + e;
      xs[e] = r < rows ? g[r] + (pi ? pi[r] : 0.f) : 0.f;
    }
    __syncthreads();
    chunk_dots(V, ldv, r0, R, xs, acc);
  }
  __syncthreads();
  finish_partials(acc, R, part, rankp, ticket);
}

struct BaseHyper {
  int kind;
  float lr, wd, b1, b2, omb1, omb2, eps, mom;  // omb = 1 - beta, formed in fp64 on the host
  float bc1, bc2;
};

// ---- P2: g2, base step (moments), s, and sc = V^T s
__global__ void __launch_bounds__(kT) upd_p2_kernel(const float* __restrict__ V, size_t ldv, int R, size_t rows,
                                                    const float* __restrict__ g, const float* __restrict__ pi,
                                                    const float* __restrict__ w, const double* __restrict__ all1,
                                                    int world, BaseHyper hp, float* __restrict__ m,
                                                    float* __restrict__ v, float* __restrict__ s_out, double* part,
                                                    double* rankp, unsigned* ticket, int* bad) {
  extern __shared__ __align__(16) unsigned char smem[];
  float* xs = reinterpret_cast<float*>(smem);
  double* c = reinterpret_cast<double*>(smem + kCh * sizeof(float));
  double* acc = c + R;
  for (int j = threadIdx.x; j < R; j += kT) {
    double t = 0.0;
    for (int r = 0; r < world; ++r) t += all1[(size_t)r * R + j];
    c[j] = t;
  }
  for (int e = threadIdx.x; e < kW * R; e += kT) acc[e] = 0.0;
  const size_t nch = cdiv(rows, kCh);
  int local_bad = 0;
  for (size_t ch = blockIdx.x; ch < nch; ch += gridDim.x) {
    const size_t r0 = ch * kCh;
    __syncthreads();
    for (int e = threadIdx.x; e < kCh; e += kT) {
      const size_t r = r0 + e;
      float sv = 0.f;
      if (r < rows) {
        double g2 = (double)g[r] + (pi ? (double)pi[r] : 0.0);
        for (int j = 0; j < R; ++j) g2 -= (double)__ldg(V + (size_t)j * ldv + r) * c[j];
        const float gf = (float)g2;
        if (!isfinite(gf)) local_bad = 1;
        // BaseOptimizer::step (optimizer.cpp:37-71)
        if (hp.kind == 0) {
          sv = -hp.lr * gf;
        } else if (hp.kind == 1) {
          const float mm = hp.mom * m[r] + gf;
          m[r] = mm;
          sv = -hp.lr * mm;
        } else {
          const float mm = hp.b1 * m[r] + hp.omb1 * gf;
          const float vv = hp.b2 * v[r] + hp.omb2 * gf * gf;
          m[r] = mm;
          v[r] = vv;
          sv = -hp.lr * (mm / hp.bc1) / (sqrtf(vv / hp.bc2) + hp.eps);
          if (hp.kind == 3) sv -= hp.lr * hp.wd * w[r];
        }
        s_out[r] = sv;
      }
      xs[e] = sv;
    }
    __syncthreads();
    if (R > 0) chunk_dots(V, ldv, r0, R, xs, acc);
  }
  if (local_bad) atomicOr(bad, 1);
  __syncthreads();
  if (R > 0) finish_partials(acc, R, part, rankp, ticket);
}

// ---- P3: w_a += base + newton (optionally materialized)
__global__ void __launch_bounds__(kT) upd_p3_kernel(const float* __restrict__ V, size_t ldv, int R, size_t rows,
                                                    const float* __restrict__ s, const double* __restrict__ all1,
                                                    const double* __restrict__ all2, int world,
                                                    const double* __restrict__ eigvals, double alpha, double sigma,
                                                    double fl, float* __restrict__ w_a, float* __restrict__ newton_out,
                                                    float* __restrict__ base_out) {
  extern __shared__ __align__(16) unsigned char smem[];
  double* sc = reinterpret_cast<double*>(smem);
  double* nb = sc + R;  // alpha c_j / den_j
  for (int j = threadIdx.x; j < R; j += kT) {
    double c = 0.0, t = 0.0;
    for (int r = 0; r < world; ++r) {
      c += all1[(size_t)r * R + j];
      t += all2[(size_t)r * R + j];
    }
    sc[j] = t;
    nb[j] = alpha * (c / floored_den(eigvals[j], fl, sigma));
  }
  __syncthreads();
  for (size_t r = blockIdx.x * (size_t)kT + threadIdx.x; r < rows; r += (size_t)gridDim.x * kT) {
    double base = s[r], newton = 0.0;
    for (int j = 0; j < R; ++j) {
      const double x = __ldg(V + (size_t)j * ldv + r);
      base -= x * sc[j];
      newton -= x * nb[j];
    }
    const float bf = (float)base, nf = (float)newton;
    if (newton_out) newton_out[r] = nf;
    if (base_out) base_out[r] = bf;
    if (w_a) {
      float wv = w_a[r] + bf;  // trainer.cpp:240-241 order: base, then newton
      if (R > 0) wv += nf;
      w_a[r] = wv;
    }
  }
}

__global__ void admm_w_kernel(size_t n, float inv_sigma, const float* __restrict__ w_a, const float* __restrict__ pi,
                              float* __restrict__ w) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    w[i] = w_a[i] + pi[i] * inv_sigma;
}
__global__ void admm_dual_kernel(size_t n, float sigma, const float* __restrict__ w_a, const float* __restrict__ w,
                                 float* __restrict__ pi) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    pi[i] += sigma * (w_a[i] - w[i]);
}
__global__ void f64_to_f32_kernel(const double* __restrict__ s, float* __restrict__ d, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    d[i] = (float)s[i];
}
__global__ void f32_to_f64_kernel(const float* __restrict__ s, double* __restrict__ d, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    d[i] = (double)s[i];
}

int grid_ew(size_t n) { return (int)std::max<size_t>(1, std::min<size_t>(cdiv(n, 256), 148 * 8)); }

}  // namespace

namespace dho2g {

void dev_copy_f64_to_f32(cudaStream_t s, const double* src, float* dst, size_t n) {
  if (!n) return;
  f64_to_f32_kernel<<<grid_ew(n), 256, 0, s>>>(src, dst, n);
  DHO2G_LAUNCH();
}
void dev_copy_f32_to_f64(cudaStream_t s, const float* src, double* dst, size_t n) {
  if (!n) return;
  f32_to_f64_kernel<<<grid_ew(n), 256, 0, s>>>(src, dst, n);
  DHO2G_LAUNCH();
}

void opt_alloc(dho2g_opt* o, dho2g_ctx* ctx, const dho2g_base_cfg& cfg, size_t rows) {
  if (rows == 0 && ctx->world == 1) fail(DHO2G_ARGUMENT, "BaseOptimizer: zero dimension");
  if (cfg.lr < 0.0) fail(DHO2G_ARGUMENT, "BaseOptimizer: negative learning rate");
  if (cfg.kind < 0 || cfg.kind > 3) fail(DHO2G_ARGUMENT, "base optimizer: expected sgd|momentum|adam|adamw");
  o->ctx = ctx;
  o->cfg = cfg;
  o->n = rows;
  o->t = 0;
  if (cfg.kind != 0) o->m.alloc(rows);
  if (cfg.kind >= 2) o->v.alloc(rows);
  o->s.alloc(rows);
  o->ticket.alloc(2);
  o->bad.alloc(1);
}

void split_update(dho2g_opt* o, const dho2g_ese* ese, const UpdateArgs& a) {
  dho2g_ctx* ctx = o->ctx;
  cudaStream_t st = ctx->stream;
  const int R = ese ? (int)ese->r : 0;
  const size_t rows = o->n;
  const size_t ldv = R ? ese->ldv : 0;
  const float* V = R ? ese->V.p : nullptr;
  const int world = ctx->world;
  const int gp = (int)std::max<size_t>(1, std::min<size_t>(cdiv(rows, kCh), (size_t)ctx->sm_count * 4));
  const int R1 = std::max(R, 1);
  o->part.ensure((size_t)gp * R1 + 8);
  o->rank1.ensure(R1);
  o->rank2.ensure(R1);
  o->all1.ensure((size_t)R1 * world);
  o->all2.ensure((size_t)R1 * world);
  const double* all1 = world > 1 ? o->all1.p : o->rank1.p;
  const double* all2 = world > 1 ? o->all2.p : o->rank2.p;
  const double rb = 4.0 * (double)rows;
  const bool adam = o->cfg.kind >= 2;
  if (R > 0) {
    const int k1 = ctx->kt_begin();
    upd_p1_kernel<<<gp, kT, kCh * sizeof(float) + (size_t)kW * R * sizeof(double), st>>>(V, ldv, R, rows, a.g, a.pi,
                                                                                         o->part.p, o->rank1.p,
                                                                                         o->ticket.p);
    DHO2G_LAUNCH();
    ctx->kt_end(k1, "upd_p1", rb * (R + 1 + (a.pi ? 1 : 0)));
    if (world > 1) ctx->allgather_f64(o->rank1.p, o->all1.p, R);
  }
  ++o->t;
  BaseHyper hp;
  hp.kind = o->cfg.kind;
  hp.lr = (float)o->cfg.lr;
  hp.wd = (float)o->cfg.weight_decay;
  hp.b1 = (float)o->cfg.beta1;
  hp.b2 = (float)o->cfg.beta2;
  hp.omb1 = (float)(1.0 - o->cfg.beta1);
  hp.omb2 = (float)(1.0 - o->cfg.beta2);
  hp.eps = (float)o->cfg.eps;
  hp.mom = (float)o->cfg.momentum;
  hp.bc1 = (float)(1.0 - std::pow(o->cfg.beta1, (double)o->t));
  hp.bc2 = (float)(1.0 - std::pow(o->cfg.beta2, (double)o->t));
  const int k2 = ctx->kt_begin();
  upd_p2_kernel<<<gp, kT, kCh * sizeof(float) + (size_t)R * sizeof(double) + (size_t)kW * R * sizeof(double), st>>>(
      V, ldv, R, rows, a.g, a.pi, a.w_decay ? a.w_decay : a.w_a, all1, world, hp, o->m.p, o->v.p, o->s.p, o->part.p, o->rank2.p,
      o->ticket.p + 1, o->bad.p);
  DHO2G_LAUNCH();
  ctx->kt_end(k2, "upd_p2", rb * (R + 2 + (a.pi ? 1 : 0) + (adam ? 4 : (o->cfg.kind == 1 ? 2 : 0)) +
                                  (o->cfg.kind == 3 ? 1 : 0)));
  if (R > 0 && world > 1) ctx->allgather_f64(o->rank2.p, o->all2.p, R);
  const int g3 = (int)std::max<size_t>(1, std::min<size_t>(cdiv(rows, kT), (size_t)ctx->sm_count * 8));
  const int k3 = ctx->kt_begin();
  upd_p3_kernel<<<g3, kT, (size_t)2 * R1 * sizeof(double), st>>>(V, ldv, R, rows, o->s.p, all1, all2, world,
                                                                  R ? ese->ev_dev.p : nullptr, a.alpha, a.sigma,
                                                                  a.floor, a.w_a, a.newton_out, a.base_out);
  DHO2G_LAUNCH();
  ctx->kt_end(k3, "upd_p3", rb * (R + 1 + (a.w_a ? 2 : 0) + (a.newton_out ? 1 : 0) + (a.base_out ? 1 : 0)));
}

void check_opt_flags(dho2g_opt* o) {
  int bad = 0;
  DHO2G_CUDA(cudaMemcpyAsync(&bad, o->bad.p, sizeof(int), cudaMemcpyDeviceToHost, o->ctx->stream));
  DHO2G_CUDA(cudaStreamSynchronize(o->ctx->stream));
  if (bad) {
    DHO2G_CUDA(cudaMemsetAsync(o->bad.p, 0, sizeof(int), o->ctx->stream));
    fail(DHO2G_NUMERIC, "BaseOptimizer: non-finite gradient");
  }
}

void admm_w_update_dev(cudaStream_t s, size_t n, double sigma, const float* w_a, const float* pi, float* w) {
  if (sigma <= 0.0) fail(DHO2G_ARGUMENT, "admm_w_update: sigma must be positive");
  if (!n) return;
  admm_w_kernel<<<grid_ew(n), 256, 0, s>>>(n, (float)(1.0 / sigma), w_a, pi, w);
  DHO2G_LAUNCH();
}

void admm_dual_update_dev(cudaStream_t s, size_t n, double sigma, const float* w_a, const float* w, float* pi) {
  if (!n) return;
  admm_dual_kernel<<<grid_ew(n), 256, 0, s>>>(n, (float)sigma, w_a, w, pi);
  DHO2G_LAUNCH();
}

}  // namespace dho2g
