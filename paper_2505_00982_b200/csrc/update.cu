// FOSI / ADMM split update with the base optimizer (reference: proj/src/optimizer.cpp:37-154),
// fused into three bandwidth-bound passes over this rank's rows:
//   P1  c = V^T (g + pi)                                    reads V, g, pi
//   P2  g2 = g~ - V c ; s = base_step(g2) ; sc = V^T s       reads V, g, pi, moments(, w); writes moments, s
//   P3  w_a += (s - V sc) + (-alpha V (c / den))             reads V, s, w_a; writes w_a
// with the r-length reductions (c, sc) as fp64 partials + all_gather + rank-ordered sums.
//
// Access pattern follows the Gram-Schmidt passes (lanczos.cu): row chunks of 2048 staged through
// shared memory; "dot" work is split into (column, 512-row block) items so every warp streams
// 2 KB contiguous per column; "axpy" work keeps 4 rows per thread with float4 loads.
#include <cudaTypedefs.h>

#include <cmath>

#include "internal.h"
#include "coop.cuh"

using namespace dho2g;

namespace {

constexpr int kT = 256;
constexpr int kW = kT / 32;
constexpr int kCh = 2048;            // rows staged per chunk
constexpr int kSubRows = 512;        // rows per warp dot item (32 lanes x 4 float4)

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

__device__ __forceinline__ float4 ld4(const float* p, size_t r, size_t rows) {
  if (r + 3 < rows) return *reinterpret_cast<const float4*>(p + r);
  float4 x = make_float4(0.f, 0.f, 0.f, 0.f);
  if (r < rows) x.x = p[r];
  if (r + 1 < rows) x.y = p[r + 1];
  if (r + 2 < rows) x.z = p[r + 2];
  return x;
}
__device__ __forceinline__ void st4(float* p, size_t r, size_t rows, float4 x) {
  if (r + 3 < rows) {
    *reinterpret_cast<float4*>(p + r) = x;
    return;
  }
  if (r < rows) p[r] = x.x;
  if (r + 1 < rows) p[r + 1] = x.y;
  if (r + 2 < rows) p[r + 2] = x.z;
}

// acc[w][j] -> CTA partials -> (last CTA, fixed order) rank partial
__device__ void finish_partials(const double* acc, int nj, double* part, double* rankp, unsigned* ticket) {
  __shared__ bool is_last;
  __syncthreads();
  for (int j = threadIdx.x; j < nj; j += kT) {
    double t = 0.0;
    for (int w = 0; w < kW; ++w) t += acc[w * nj + j];
    part[(size_t)blockIdx.x * nj + j] = t;
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) is_last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!is_last) return;
  __threadfence();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int j = warp; j < nj; j += kW) {  // a warp per value, lanes over the CTA partials (fixed order)
    const double t = warp_fold(part + j, (int)gridDim.x, (size_t)nj);
    if (lane == 0) rankp[j] = t;
  }
  if (threadIdx.x == 0) *ticket = 0u;
}

// acc[w][j] += V_j[r0 : r0 + CH] . xs (xs staged in smem); V is padded to whole chunks
template <int CH = kCh>
__device__ __forceinline__ void chunk_dots(const float* __restrict__ V, size_t ldv, size_t r0, int R,
                                           const float* xs, double* acc) {
  constexpr int kItems = CH / kSubRows;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int items = R * kItems;
  for (int it = warp; it < items; it += kW) {
    const int j = it / kItems, q = it % kItems;
    const int rb = q * kSubRows + lane * 4;
    const float* col = V + (size_t)j * ldv + r0;
    float4 x[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) x[k] = __ldg(reinterpret_cast<const float4*>(col + rb + k * 128));
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float4 y = *reinterpret_cast<const float4*>(xs + rb + k * 128);
      s += (double)(x[k].x * y.x + x[k].y * y.y + x[k].z * y.z + x[k].w * y.w);  // fp32 4-term, fp64 above
    }
    s = warp_sum(s);
    if (lane == 0) acc[warp * R + j] += s;
  }
}

// acc[w][j] += V_j[r0 : r0 + kCh] . xs with xs in fp64 and fp64 products: c feeds g2 = g~ - V c, which
// cancels to ~1e-8 of |g~| on some rows, and Adam's m/sqrt(v) is steep there (slope lr/eps at |g2| ~ eps),
// so c needs ~1e-10 relative accuracy; fp32 products over 1e8 rows give ~1e-7.
__device__ __forceinline__ void chunk_dots_f64(const float* __restrict__ V, size_t ldv, size_t r0, int R,
                                               const double* xs, double* acc) {
  constexpr int kItems = kCh / kSubRows;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int items = R * kItems;
  for (int it = warp; it < items; it += kW) {
    const int j = it / kItems, q = it % kItems;
    const int rb = q * kSubRows + lane * 4;
    const float* col = V + (size_t)j * ldv + r0;
    float4 x[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) x[k] = __ldg(reinterpret_cast<const float4*>(col + rb + k * 128));
    double s0 = 0.0, s1 = 0.0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const double2 a = *reinterpret_cast<const double2*>(xs + rb + k * 128);
      const double2 b = *reinterpret_cast<const double2*>(xs + rb + k * 128 + 2);
      s0 = fma((double)x[k].x, a.x, s0);
      s1 = fma((double)x[k].y, a.y, s1);
      s0 = fma((double)x[k].z, b.x, s0);
      s1 = fma((double)x[k].w, b.y, s1);
    }
    const double s = warp_sum(s0 + s1);
    if (lane == 0) acc[warp * R + j] += s;
  }
}

// ---- P1: c = V^T (g + pi), g~ formed in fp64 (optimizer.cpp:91) and fp64 products
__global__ void __launch_bounds__(kT) upd_p1_kernel(const float* __restrict__ V, size_t ldv, int R, size_t rows,
                                                    const float* __restrict__ g, const float* __restrict__ pi,
                                                    double* part, double* rankp, unsigned* ticket) {
  extern __shared__ __align__(16) unsigned char smem[];
  double* xs = reinterpret_cast<double*>(smem);
  double* acc = xs + kCh;
  for (int e = threadIdx.x; e < kW * R; e += kT) acc[e] = 0.0;
  const size_t nch = cdiv(rows, kCh);
  for (size_t c = blockIdx.x; c < nch; c += gridDim.x) {
    const size_t r0 = c * kCh;
    __syncthreads();
    for (int e = threadIdx.x; e < kCh / 4; e += kT) {
      const float4 x = ld4(g, r0 + 4 * e, rows);
      double2 a = make_double2(x.x, x.y), b = make_double2(x.z, x.w);
      if (pi) {
        const float4 p = ld4(pi, r0 + 4 * e, rows);
        a.x += p.x; a.y += p.y; b.x += p.z; b.y += p.w;
      }
      reinterpret_cast<double2*>(xs)[2 * e] = a;
      reinterpret_cast<double2*>(xs)[2 * e + 1] = b;
    }
    __syncthreads();
    chunk_dots_f64(V, ldv, r0, R, xs, acc);
  }
  finish_partials(acc, R, part, rankp, ticket);
}

struct BaseHyper {
  int kind;
  float lr, wd, b1, b2, omb1, omb2, eps, mom;  // omb = 1 - beta, formed in fp64 on the host
  float bc1, bc2;
};

__device__ __forceinline__ float base_step(const BaseHyper& hp, float gf, float& m, float& v, float w) {
  // BaseOptimizer::step (optimizer.cpp:37-71)
  if (hp.kind == 0) return -hp.lr * gf;
  if (hp.kind == 1) {
    m = hp.mom * m + gf;
    return -hp.lr * m;
  }
  m = hp.b1 * m + hp.omb1 * gf;
  v = hp.b2 * v + hp.omb2 * gf * gf;
  float s = -hp.lr * (m / hp.bc1) / (sqrtf(v / hp.bc2) + hp.eps);
  if (hp.kind == 3) s -= hp.lr * hp.wd * w;
  return s;
}

// ---- P2: g2 = g~ - V c, base step (moments), s, and sc = V^T s. Chunks of kCh2 = 1024 rows: the dots
// re-read the chunk's V columns right after the correction pass read them, and with all resident
// CTAs' chunks (~592 x R x 4 KB) inside the 126 MB L2 that re-read is an L2 hit.
constexpr int kCh2 = 1024;
__global__ void __launch_bounds__(kT) upd_p2_kernel(const float* __restrict__ V, size_t ldv, int R, size_t rows,
                                                    const float* __restrict__ g, const float* __restrict__ pi,
                                                    const float* __restrict__ w, const double* __restrict__ all1,
                                                    int world, BaseHyper hp, float* __restrict__ m,
                                                    float* __restrict__ v, float* __restrict__ s_out, double* part,
                                                    double* rankp, unsigned* ticket, int* bad) {
  extern __shared__ __align__(16) unsigned char smem[];
  float* xs = reinterpret_cast<float*>(smem);
  double* c = reinterpret_cast<double*>(smem + kCh2 * sizeof(float));
  double* acc = c + R;
  for (int j = threadIdx.x; j < R; j += kT) {
    double t = 0.0;
    for (int r = 0; r < world; ++r) t += all1[(size_t)r * R + j];
    c[j] = t;
  }
  for (int e = threadIdx.x; e < kW * R; e += kT) acc[e] = 0.0;
  const bool need_m = hp.kind != 0, need_v = hp.kind >= 2, need_w = hp.kind == 3;
  const size_t nch = cdiv(rows, kCh2);
  int local_bad = 0;
  for (size_t ch = blockIdx.x; ch < nch; ch += gridDim.x) {
    const size_t r0 = ch * kCh2;
    __syncthreads();
    for (int e = threadIdx.x; e < kCh2 / 4; e += kT) {
      const size_t r = r0 + 4 * (size_t)e;
      const float4 x = ld4(g, r, rows);
      double g0 = x.x, g1 = x.y, g2 = x.z, g3 = x.w;
      if (pi) {  // g~ = g + pi in fp64 (optimizer.cpp:91)
        const float4 p = ld4(pi, r, rows);
        g0 += p.x; g1 += p.y; g2 += p.z; g3 += p.w;
      }
      int j = 0;
      for (; j + 4 <= R; j += 4) {
        float4 d[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) d[u] = __ldg(reinterpret_cast<const float4*>(V + (size_t)(j + u) * ldv + r));
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const double cj = c[j + u];
          g0 -= (double)d[u].x * cj; g1 -= (double)d[u].y * cj; g2 -= (double)d[u].z * cj; g3 -= (double)d[u].w * cj;
        }
      }
      for (; j < R; ++j) {
        const float4 d = __ldg(reinterpret_cast<const float4*>(V + (size_t)j * ldv + r));
        const double cj = c[j];
        g0 -= (double)d.x * cj; g1 -= (double)d.y * cj; g2 -= (double)d.z * cj; g3 -= (double)d.w * cj;
      }
      const float4 gm = make_float4((float)g0, (float)g1, (float)g2, (float)g3);
      float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
      if (r < rows) {
        if (!isfinite(gm.x) || !isfinite(gm.y) || !isfinite(gm.z) || !isfinite(gm.w)) local_bad = 1;
        float4 mm = need_m ? ld4(m, r, rows) : make_float4(0.f, 0.f, 0.f, 0.f);
        float4 vm = need_v ? ld4(v, r, rows) : make_float4(0.f, 0.f, 0.f, 0.f);
        const float4 ww = need_w ? ld4(w, r, rows) : make_float4(0.f, 0.f, 0.f, 0.f);
        s.x = base_step(hp, gm.x, mm.x, vm.x, ww.x);
        s.y = r + 1 < rows ? base_step(hp, gm.y, mm.y, vm.y, ww.y) : 0.f;
        s.z = r + 2 < rows ? base_step(hp, gm.z, mm.z, vm.z, ww.z) : 0.f;
        s.w = r + 3 < rows ? base_step(hp, gm.w, mm.w, vm.w, ww.w) : 0.f;
        if (need_m) st4(m, r, rows, mm);
        if (need_v) st4(v, r, rows, vm);
        st4(s_out, r, rows, s);
      }
      reinterpret_cast<float4*>(xs)[e] = s;
    }
    __syncthreads();
    if (R > 0) chunk_dots<kCh2>(V, ldv, r0, R, xs, acc);
  }
  if (local_bad) atomicOr(bad, 1);
  if (R > 0) finish_partials(acc, R, part, rankp, ticket);
}

// ---- P2 (bulk-copy staged): same math as upd_p2_kernel for R <= kP2MaxR. Each chunk of CH rows of
// V (R columns) and of the row streams (g, pi, m, v, w) is brought into shared memory by
// cp.async.bulk (double-buffered, one mbarrier per stage), so V is read from HBM exactly once for
// both the correction g - V c and the dots V^T s (the register-staged kernel re-reads V for the dots
// and loses the L2 race at large R x CH). Dot partials stay in per-lane fp64 registers until the end.
constexpr int kP2MaxR = 48;

constexpr int kP2Streams = 5;  // g, pi, m, v, w

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_addr(dst)),
               "l"(src), "r"(bytes), "r"(smem_addr(bar))
               : "memory");
}
__device__ __forceinline__ void bar_wait(uint64_t* b, uint32_t parity) {
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(smem_addr(b)), "r"(parity)
        : "memory");
  } while (!done);
}

// Two CTAs per SM, each double-buffered: ~4 stages of (R + 5) x 1 KB in flight per SM.
// ROWDOT (R <= 32): each thread also accumulates its rows' contributions to V_hat^T s in 32 fp64
// registers while the row is at hand (no second pass over the stage, one barrier per chunk); the block
// reduction happens once at the end.
template <int CH, int NS, int MINB, bool ROWDOT = false>
__global__ void __launch_bounds__(kT, MINB) upd_p2_tma_kernel(const __grid_constant__ CUtensorMap mapV, int R, size_t rows,
                                                          const float* __restrict__ g, const float* __restrict__ pi,
                                                          const float* __restrict__ w,
                                                          const double* __restrict__ all1, int world, BaseHyper hp,
                                                          float* __restrict__ m, float* __restrict__ v,
                                                          float* __restrict__ s_out, double* part, double* rankp,
                                                          unsigned* ticket, int* bad) {
  extern __shared__ __align__(16) unsigned char smem[];
  const size_t stage_floats = (size_t)(R + kP2Streams) * CH;
  // tensor-copy destinations need 128-byte alignment
  float* stg0 = reinterpret_cast<float*>((reinterpret_cast<uintptr_t>(smem) + 127) & ~uintptr_t(127));
  float* xs = stg0 + NS * stage_floats;
  double* c = reinterpret_cast<double*>(xs + CH);
  double* acc = c + R;  // [kW][R]
  uint64_t* bar = reinterpret_cast<uint64_t*>(acc + kW * R);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool need_m = hp.kind != 0, need_v = hp.kind >= 2, need_w = hp.kind == 3;
  const size_t nch = cdiv(rows, CH);

  auto issue = [&](size_t i) {  // thread 0: stage i % NS <- chunk blockIdx.x + i * gridDim.x
    const size_t ch = blockIdx.x + i * gridDim.x;
    if (ch >= nch) return;
    float* st = stg0 + (i % NS) * stage_floats;
    const size_t r0 = ch * CH;
    const bool full = r0 + CH <= rows;
    uint32_t bytes = (uint32_t)R * CH * 4u;
    if (full) bytes += (uint32_t)(1 + (pi ? 1 : 0) + (need_m ? 1 : 0) + (need_v ? 1 : 0) + (need_w ? 1 : 0)) * CH * 4u;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // prior generic reads of the stage
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(&bar[i % NS])), "r"(bytes)
                 : "memory");
    // all R columns of the chunk in one tensor copy (column-major in smem): a 2D box CH rows x R columns,
    // or for CH > 256 (the box-dimension limit) a 3D box 256 x CH/256 x R over rows viewed as 256-row blocks
    if constexpr (CH <= 256) {
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::
              "r"(smem_addr(st)),
          "l"(reinterpret_cast<uint64_t>(&mapV)), "r"((int)r0), "r"(0), "r"(smem_addr(&bar[i % NS]))
          : "memory");
    } else {
      asm volatile(
          "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
          "[%5];" ::"r"(smem_addr(st)),
          "l"(reinterpret_cast<uint64_t>(&mapV)), "r"(0), "r"((int)(r0 / 256)), "r"(0), "r"(smem_addr(&bar[i % NS]))
          : "memory");
    }
    if (full) {
      float* ss = st + (size_t)R * CH;
      bulk_g2s(ss, g + r0, CH * 4u, &bar[i % NS]);
      if (pi) bulk_g2s(ss + CH, pi + r0, CH * 4u, &bar[i % NS]);
      if (need_m) bulk_g2s(ss + 2 * CH, m + r0, CH * 4u, &bar[i % NS]);
      if (need_v) bulk_g2s(ss + 3 * CH, v + r0, CH * 4u, &bar[i % NS]);
      if (need_w) bulk_g2s(ss + 4 * CH, w + r0, CH * 4u, &bar[i % NS]);
    }
  };

  if (threadIdx.x == 0) {
    for (int q = 0; q < NS; ++q) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(&bar[q])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int j = threadIdx.x; j < R; j += kT) {
    double t = 0.0;
    for (int r = 0; r < world; ++r) t += all1[(size_t)r * R + j];
    c[j] = t;
  }
  __syncthreads();
  if (threadIdx.x == 0)
    for (int q = 0; q < NS; ++q) issue(q);
  double lacc[kP2MaxR / kW];
#pragma unroll
  for (int q = 0; q < kP2MaxR / kW; ++q) lacc[q] = 0.0;
  constexpr int kRowR = ROWDOT ? 32 : 1;
  double pacc[kRowR];
#pragma unroll
  for (int q = 0; q < kRowR; ++q) pacc[q] = 0.0;
  int local_bad = 0;
  for (size_t i = 0; blockIdx.x + i * gridDim.x < nch; ++i) {
    const size_t r0 = (blockIdx.x + i * gridDim.x) * CH;
    const bool full = r0 + CH <= rows;
    float* st = stg0 + (i % NS) * stage_floats;
    bar_wait(&bar[i % NS], (uint32_t)((i / NS) & 1));
    for (int t = threadIdx.x; t < CH; t += kT) {  // phase A: rows r0 + t
      const size_t r = r0 + t;
      const bool in = r < rows;
      const float* ss = st + (size_t)R * CH;
      // g~ = g + pi in fp64 (optimizer.cpp:91 adds in fp64): an fp32 sum rounds away bits that matter
      // where g2 = g~ - V c nearly cancels and Adam's m/sqrt(v) is steep
      double x = full ? ss[t] : (in ? g[r] : 0.f);
      if (pi) x += (double)(full ? ss[CH + t] : (in ? pi[r] : 0.f));
      // four independent fp64 partial sums (short dependency chains), combined in a fixed order
      double g0 = x, g1 = 0.0, g2 = 0.0, g3 = 0.0;
      int j = 0;
      for (; j + 4 <= R; j += 4) {
        g0 -= (double)st[(size_t)j * CH + t] * c[j];
        g1 -= (double)st[(size_t)(j + 1) * CH + t] * c[j + 1];
        g2 -= (double)st[(size_t)(j + 2) * CH + t] * c[j + 2];
        g3 -= (double)st[(size_t)(j + 3) * CH + t] * c[j + 3];
      }
      for (; j < R; ++j) g0 -= (double)st[(size_t)j * CH + t] * c[j];
      const float gm = (float)((g0 + g1) + (g2 + g3));
      float sv = 0.f;
      if (in) {
        if (!isfinite(gm)) local_bad = 1;
        float mm = need_m ? (full ? ss[2 * CH + t] : m[r]) : 0.f;
        float vm = need_v ? (full ? ss[3 * CH + t] : v[r]) : 0.f;
        const float ww = need_w ? (full ? ss[4 * CH + t] : w[r]) : 0.f;
        sv = base_step(hp, gm, mm, vm, ww);
        if (need_m) m[r] = mm;
        if (need_v) v[r] = vm;
        s_out[r] = sv;
      }
      if constexpr (ROWDOT) {
#pragma unroll
        for (int q = 0; q < kRowR; ++q)
          if (q < R) pacc[q] += (double)st[(size_t)q * CH + t] * (double)sv;
      } else {
        xs[t] = sv;
      }
    }
    __syncthreads();
    // phase B: column j = warp + kW q, lanes stride the chunk with float4
#pragma unroll
    for (int q = 0; q < (ROWDOT ? 0 : kP2MaxR / kW); ++q) {
      const int j = warp + kW * q;
      if (j < R) {
        const float* col = st + (size_t)j * CH;
        float f = 0.f;
#pragma unroll
        for (int k = 0; k < CH / 128; ++k) {
          const float4 a = *reinterpret_cast<const float4*>(col + 4 * lane + 128 * k);
          const float4 b = *reinterpret_cast<const float4*>(xs + 4 * lane + 128 * k);
          f += a.x * b.x + a.y * b.y + a.z * b.z + a.w * b.w;
        }
        lacc[q] += (double)f;
      }
    }
    if constexpr (!ROWDOT) __syncthreads();  // stage (i % NS) and xs free (ROWDOT: the barrier above)
    if (threadIdx.x == 0) issue(i + NS);
  }
  if (local_bad) atomicOr(bad, 1);
  if constexpr (ROWDOT) {
#pragma unroll
    for (int q = 0; q < kRowR; ++q) {
      const double t = warp_sum(pacc[q]);
      if (q < R && lane == 0) acc[warp * R + q] = t;
    }
  } else {
#pragma unroll
    for (int q = 0; q < kP2MaxR / kW; ++q) {
      const int j = warp + kW * q;
      const double t = warp_sum(lacc[q]);
      if (j < R && lane == 0) acc[warp * R + j] = t;
    }
    for (int e = threadIdx.x; e < kW * R; e += kT)  // warps without column j contribute 0
      if (e / R != (e % R) % kW) acc[e] = 0.0;
  }
  finish_partials(acc, R, part, rankp, ticket);
}

// ---- small n (world 1, r <= 32): P1, P2 and P3 as ONE cooperative launch. Each CTA owns a contiguous slice of
// rows (rs rows, float4 groups g = tid + kT q); the r-length reductions are per-CTA partial rows + a grid
// barrier + the fixed-order cross-CTA sum that every CTA performs (reduce_rows): no tickets, no launches
// between the passes. Same per-element arithmetic as upd_p1 / upd_p2 / upd_p3 (c in fp64 products of
// g~ = g + pi formed in fp64; V^T s as fp32 4-term products summed in fp64).
constexpr int kSmallR = 32;
__global__ void __launch_bounds__(kT) upd_small_kernel(const float* __restrict__ V, size_t ldv, int R, size_t rows,
                                                       int rs, const float* __restrict__ g, const float* __restrict__ pi,
                                                       const float* __restrict__ w, BaseHyper hp, float* __restrict__ m,
                                                       float* __restrict__ v, float* __restrict__ s_out,
                                                       const double* __restrict__ eigvals, double alpha, double sigma,
                                                       double fl, float* __restrict__ w_a, float* __restrict__ newton_out,
                                                       float* __restrict__ base_out, double* part1, double* part2,
                                                       unsigned long long* bar, int* bad) {
  __shared__ double c[kSmallR], sc[kSmallR], nbv[kSmallR];
  __shared__ double sacc[kW * kSmallR];
  __shared__ unsigned long long bar_next;
  const unsigned nb = gridDim.x;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) bar_next = 0ull;
  const size_t r0 = (size_t)blockIdx.x * rs, r1 = min(rows, r0 + (size_t)rs);
  const int ng = r1 > r0 ? (int)((r1 - r0 + 3) / 4) : 0;
  const bool need_m = hp.kind != 0, need_v = hp.kind >= 2, need_w = hp.kind == 3;
  auto cta_row = [&](const double (&acc)[kSmallR], double* part) {  // warp sums -> this CTA's partial row
#pragma unroll
    for (int j = 0; j < kSmallR; ++j) {
      if (j >= R) break;
      const double t = warp_sum(acc[j]);
      if (lane == 0) sacc[warp * kSmallR + j] = t;
    }
    __syncthreads();
    if (tid < R) {
      double t = 0.0;
      for (int q = 0; q < kW; ++q) t += sacc[q * kSmallR + tid];
      __stcg(part + (size_t)blockIdx.x * kSmallR + tid, t);
    }
  };
  // ---- P1: c = V^T (g + pi)
  {
    double acc[kSmallR];
#pragma unroll
    for (int j = 0; j < kSmallR; ++j) acc[j] = 0.0;
    for (int q = tid; q < ng; q += kT) {
      const size_t r = r0 + 4 * (size_t)q;
      const float4 x = ld4(g, r, rows);
      double g0 = x.x, g1 = x.y, g2 = x.z, g3 = x.w;
      if (pi) {
        const float4 p = ld4(pi, r, rows);
        g0 += p.x; g1 += p.y; g2 += p.z; g3 += p.w;
      }
#pragma unroll
      for (int j = 0; j < kSmallR; ++j) {
        if (j >= R) break;
        const float4 d = __ldg(reinterpret_cast<const float4*>(V + (size_t)j * ldv + r));
        acc[j] = fma((double)d.x, g0, acc[j]);
        acc[j] = fma((double)d.y, g1, acc[j]);
        acc[j] = fma((double)d.z, g2, acc[j]);
        acc[j] = fma((double)d.w, g3, acc[j]);
      }
    }
    cta_row(acc, part1);
  }
  grid_barrier(bar, nb, &bar_next);
  reduce_rows<kT>(part1, (int)nb, kSmallR, R, sacc, c);
  // ---- P2: g2 = g~ - V c, base step, s; sc partials = V^T s
  int local_bad = 0;
  {
    double acc[kSmallR];
#pragma unroll
    for (int j = 0; j < kSmallR; ++j) acc[j] = 0.0;
    for (int q = tid; q < ng; q += kT) {
      const size_t r = r0 + 4 * (size_t)q;
      const float4 x = ld4(g, r, rows);
      double g0 = x.x, g1 = x.y, g2 = x.z, g3 = x.w;
      if (pi) {
        const float4 p = ld4(pi, r, rows);
        g0 += p.x; g1 += p.y; g2 += p.z; g3 += p.w;
      }
      float4 d[kSmallR];
#pragma unroll
      for (int j = 0; j < kSmallR; ++j)
        if (j < R) d[j] = __ldg(reinterpret_cast<const float4*>(V + (size_t)j * ldv + r));
#pragma unroll
      for (int j = 0; j < kSmallR; ++j) {
        if (j >= R) break;
        const double cj = c[j];
        g0 -= (double)d[j].x * cj; g1 -= (double)d[j].y * cj; g2 -= (double)d[j].z * cj; g3 -= (double)d[j].w * cj;
      }
      const float4 gm = make_float4((float)g0, (float)g1, (float)g2, (float)g3);
      if (!isfinite(gm.x) || !isfinite(gm.y) || !isfinite(gm.z) || !isfinite(gm.w)) local_bad = 1;
      float4 mm = need_m ? ld4(m, r, rows) : make_float4(0.f, 0.f, 0.f, 0.f);
      float4 vm = need_v ? ld4(v, r, rows) : make_float4(0.f, 0.f, 0.f, 0.f);
      const float4 ww = need_w ? ld4(w, r, rows) : make_float4(0.f, 0.f, 0.f, 0.f);
      float4 sv;
      sv.x = base_step(hp, gm.x, mm.x, vm.x, ww.x);
      sv.y = r + 1 < rows ? base_step(hp, gm.y, mm.y, vm.y, ww.y) : 0.f;
      sv.z = r + 2 < rows ? base_step(hp, gm.z, mm.z, vm.z, ww.z) : 0.f;
      sv.w = r + 3 < rows ? base_step(hp, gm.w, mm.w, vm.w, ww.w) : 0.f;
      if (need_m) st4(m, r, rows, mm);
      if (need_v) st4(v, r, rows, vm);
      st4(s_out, r, rows, sv);
#pragma unroll
      for (int j = 0; j < kSmallR; ++j) {
        if (j >= R) break;
        acc[j] += (double)(d[j].x * sv.x + d[j].y * sv.y + d[j].z * sv.z + d[j].w * sv.w);  // fp32 4-term
      }
    }
    if (local_bad) atomicOr(bad, 1);
    cta_row(acc, part2);
  }
  grid_barrier(bar, nb, &bar_next);
  reduce_rows<kT>(part2, (int)nb, kSmallR, R, sacc, sc);
  if (tid < R) nbv[tid] = alpha * (c[tid] / floored_den(eigvals[tid], fl, sigma));
  __syncthreads();
  // ---- P3: w_a += (s - V sc) + (-V (alpha c / den))
  for (int q = tid; q < ng; q += kT) {
    const size_t r = r0 + 4 * (size_t)q;
    const float4 s4 = ld4(s_out, r, rows);  // (this thread wrote it in P2)
    double b0 = s4.x, b1 = s4.y, b2 = s4.z, b3 = s4.w, n0 = 0, n1 = 0, n2 = 0, n3 = 0;
#pragma unroll
    for (int j = 0; j < kSmallR; ++j) {
      if (j >= R) break;
      const float4 d = __ldg(reinterpret_cast<const float4*>(V + (size_t)j * ldv + r));
      const double a = sc[j], b = nbv[j];
      b0 -= (double)d.x * a; b1 -= (double)d.y * a; b2 -= (double)d.z * a; b3 -= (double)d.w * a;
      n0 -= (double)d.x * b; n1 -= (double)d.y * b; n2 -= (double)d.z * b; n3 -= (double)d.w * b;
    }
    const float4 bf = make_float4((float)b0, (float)b1, (float)b2, (float)b3);
    const float4 nf = make_float4((float)n0, (float)n1, (float)n2, (float)n3);
    if (newton_out) st4(newton_out, r, rows, nf);
    if (base_out) st4(base_out, r, rows, bf);
    if (w_a) {
      float4 wv = ld4(w_a, r, rows);
      wv.x += bf.x; wv.y += bf.y; wv.z += bf.z; wv.w += bf.w;  // trainer.cpp:240-241 order: base, then newton
      wv.x += nf.x; wv.y += nf.y; wv.z += nf.z; wv.w += nf.w;
      st4(w_a, r, rows, wv);
    }
  }
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
  const size_t ng = cdiv(rows, 4);
  for (size_t q = blockIdx.x * (size_t)kT + threadIdx.x; q < ng; q += (size_t)gridDim.x * kT) {
    const size_t r = 4 * q;
    const float4 s4 = ld4(s, r, rows);
    double b0 = s4.x, b1 = s4.y, b2 = s4.z, b3 = s4.w, n0 = 0, n1 = 0, n2 = 0, n3 = 0;
    int j = 0;
    for (; j + 4 <= R; j += 4) {
      float4 d[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) d[u] = __ldg(reinterpret_cast<const float4*>(V + (size_t)(j + u) * ldv + r));
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const double a = sc[j + u], b = nb[j + u];
        b0 -= (double)d[u].x * a; b1 -= (double)d[u].y * a; b2 -= (double)d[u].z * a; b3 -= (double)d[u].w * a;
        n0 -= (double)d[u].x * b; n1 -= (double)d[u].y * b; n2 -= (double)d[u].z * b; n3 -= (double)d[u].w * b;
      }
    }
    for (; j < R; ++j) {
      const float4 d = __ldg(reinterpret_cast<const float4*>(V + (size_t)j * ldv + r));
      const double a = sc[j], b = nb[j];
      b0 -= (double)d.x * a; b1 -= (double)d.y * a; b2 -= (double)d.z * a; b3 -= (double)d.w * a;
      n0 -= (double)d.x * b; n1 -= (double)d.y * b; n2 -= (double)d.z * b; n3 -= (double)d.w * b;
    }
    const float4 bf = make_float4((float)b0, (float)b1, (float)b2, (float)b3);
    const float4 nf = make_float4((float)n0, (float)n1, (float)n2, (float)n3);
    if (newton_out) st4(newton_out, r, rows, nf);
    if (base_out) st4(base_out, r, rows, bf);
    if (w_a) {
      float4 wv = ld4(w_a, r, rows);
      wv.x += bf.x; wv.y += bf.y; wv.z += bf.z; wv.w += bf.w;  // trainer.cpp:240-241 order: base, then newton
      if (R > 0) {
        wv.x += nf.x; wv.y += nf.y; wv.z += nf.z; wv.w += nf.w;
      }
      st4(w_a, r, rows, wv);
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

BaseHyper make_hyper(const dho2g_base_cfg& cfg, size_t t) {
  BaseHyper hp;
  hp.kind = cfg.kind;
  hp.lr = (float)cfg.lr;
  hp.wd = (float)cfg.weight_decay;
  hp.b1 = (float)cfg.beta1;
  hp.b2 = (float)cfg.beta2;
  hp.omb1 = (float)(1.0 - cfg.beta1);
  hp.omb2 = (float)(1.0 - cfg.beta2);
  hp.eps = (float)cfg.eps;
  hp.mom = (float)cfg.momentum;
  hp.bc1 = (float)(1.0 - std::pow(cfg.beta1, (double)t));  // optimizer.cpp:54-55
  hp.bc2 = (float)(1.0 - std::pow(cfg.beta2, (double)t));
  return hp;
}

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
  if (R > 0 && ldv < round_up(std::max<size_t>(rows, 1), kCh)) fail(DHO2G_DIMENSION, "deltas: V_hat not chunk padded");
  auto al16 = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  if (!al16(a.g) || !al16(a.pi) || !al16(a.w_a) || !al16(a.w_decay) || !al16(a.newton_out) || !al16(a.base_out))
    fail(DHO2G_ARGUMENT, "split_update: vectors must be 16-byte aligned");
  const size_t smem_p1 = kCh * sizeof(double) + (size_t)kW * R * sizeof(double);
  const size_t smem_p2 = kCh2 * sizeof(float) + (size_t)R * sizeof(double) + (size_t)kW * R * sizeof(double);
  const int gp = std::min(one_wave_grid(upd_p1_kernel, kT, smem_p1, ctx->sm_count, cdiv(rows, kCh)),
                          one_wave_grid(upd_p2_kernel, kT, smem_p2, ctx->sm_count, cdiv(rows, kCh2)));
  const int R1 = std::max(R, 1);
  o->part.ensure((size_t)4 * gp * R1 + 8);  // the staged pass 2 may run up to 4 gp CTAs
  o->rank1.ensure(R1);
  o->rank2.ensure(R1);
  o->all1.ensure((size_t)R1 * world);
  o->all2.ensure((size_t)R1 * world);
  const double* all1 = world > 1 ? o->all1.p : o->rank1.p;
  const double* all2 = world > 1 ? o->all2.p : o->rank2.p;
  const double rb = 4.0 * (double)rows;  // algorithmic bytes per row-vector pass
  const bool adam = o->cfg.kind >= 2;
  if (world == 1 && R > 0 && R <= kSmallR && ctx->upd_small && rows <= (size_t)ctx->upd_small_max_rows) {
    // one cooperative launch for the three passes (small n: the three launches' fixed costs dominate)
    ++o->t;
    const BaseHyper hp = make_hyper(o->cfg, o->t);
    const int nbk = ctx->sm_count;
    const int rs = (int)round_up(cdiv(rows, (size_t)nbk), 4);
    o->part.ensure((size_t)2 * nbk * kSmallR);
    o->sbar.ensure_g((size_t)kBarShards * kBarStride);
    if (o->sbar_nb != nbk) {
      DHO2G_CUDA(cudaMemsetAsync(o->sbar.p, 0, o->sbar.n * sizeof(unsigned long long), st));
      o->sbar_nb = nbk;
    }
    const float* wdec = a.w_decay ? a.w_decay : a.w_a;
    double* p1 = o->part.p;
    double* p2 = o->part.p + (size_t)nbk * kSmallR;
    const double* ev = ese->ev_dev.p;
    float* s_out = o->s.p;
    unsigned long long* barp = o->sbar.p;
    int* badp = o->bad.p;
    void* args[] = {(void*)&V, (void*)&ldv, (void*)&R, (void*)&rows, (void*)&rs, (void*)&a.g, (void*)&a.pi,
                    (void*)&wdec, (void*)&hp, (void*)&o->m.p, (void*)&o->v.p, (void*)&s_out, (void*)&ev,
                    (void*)&a.alpha, (void*)&a.sigma, (void*)&a.floor, (void*)&a.w_a, (void*)&a.newton_out,
                    (void*)&a.base_out, (void*)&p1, (void*)&p2, (void*)&barp, (void*)&badp};
    const int k0 = ctx->kt_begin();
    DHO2G_CUDA(cudaLaunchCooperativeKernel((void*)upd_small_kernel, dim3((unsigned)nbk), dim3(kT), args, 0, st));
    DHO2G_LAUNCH();
    ctx->kt_end(k0, "upd_small", rb * (3.0 * R + 5.0 + (a.pi ? 2 : 0) + (adam ? 4 : (o->cfg.kind == 1 ? 2 : 0)) +
                                       (o->cfg.kind == 3 ? 1 : 0) + (a.w_a ? 2 : 0)));
    return;
  }
  if (R > 0) {
    const int k1 = ctx->kt_begin();
    upd_p1_kernel<<<gp, kT, smem_p1, st>>>(V, ldv, R, rows, a.g, a.pi,
                                                                                         o->part.p, o->rank1.p,
                                                                                         o->ticket.p);
    DHO2G_LAUNCH();
    ctx->kt_end(k1, "upd_p1", rb * (R + 1 + (a.pi ? 1 : 0)));
    if (world > 1) ctx->allgather_f64(o->rank1.p, o->all1.p, R, "all_reduce");
  }
  ++o->t;
  const BaseHyper hp = make_hyper(o->cfg, o->t);
  const int k2 = ctx->kt_begin();
  if (R > 0 && R <= kP2MaxR && ctx->upd_p2_staged) {
    // stage shape / depth / CTAs per SM (option upd_p2_variant). Default 5: 256-row stages, double-buffered,
    // two CTAs per SM, V_hat^T s accumulated per row in registers (C4, r = 32: 93 % of HBM peak vs 78 % for
    // the separate column-dot phase of variant 0)
    int var = (ctx->upd_p2_variant == 4 && ldv % 256) ? 0 : ctx->upd_p2_variant;  // 3D view needs 256 | ldv
    if (var == 5 && R > 32) var = 0;                                                  // row dots: R <= 32
    const int CH = (var == 0 || var == 5) ? 256 : (var == 4 ? 512 : 128);
    const int NS = var == 2 ? 3 : (var == 3 ? 4 : 2);
    const size_t smem_t = ((size_t)NS * (R + kP2Streams) * CH + CH) * sizeof(float) +
                          (size_t)(R + kW * R) * sizeof(double) + NS * sizeof(uint64_t) + 128;
    auto kern = var == 1 ? upd_p2_tma_kernel<128, 2, 4>
              : var == 2 ? upd_p2_tma_kernel<128, 3, 3>
              : var == 3 ? upd_p2_tma_kernel<128, 4, 2>
              : var == 4 ? upd_p2_tma_kernel<512, 2, 1>
              : var == 5 ? upd_p2_tma_kernel<256, 2, 2, true>
                         : upd_p2_tma_kernel<256, 2, 2>;
    if (smem_t > 227 * 1024) fail(DHO2G_ARGUMENT, "split_update: staged pass 2 does not fit shared memory");
    DHO2G_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_t));
    const int gt = std::min(gp * 4, one_wave_grid(kern, kT, smem_t, ctx->sm_count, cdiv(rows, CH)));
    // V_hat as a 2D fp32 tensor: inner = rows (stride 1), outer = R columns (stride ldv); box CH x R
    CUtensorMap mapV;
    {
      auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ctx->encode_fn);
      CUresult rc = CUDA_ERROR_INVALID_VALUE;
      if (CH <= 256) {
        cuuint64_t dims[2] = {(cuuint64_t)ldv, (cuuint64_t)R};
        cuuint64_t strides[1] = {(cuuint64_t)ldv * sizeof(float)};
        cuuint32_t box[2] = {(cuuint32_t)CH, (cuuint32_t)R};
        cuuint32_t estr[2] = {1, 1};
        if (enc)
          rc = enc(&mapV, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(V), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      } else {  // rows as (256, ldv / 256) blocks (ldv is a multiple of the 2048-row GS chunk)
        cuuint64_t dims[3] = {256, (cuuint64_t)(ldv / 256), (cuuint64_t)R};
        cuuint64_t strides[2] = {256 * sizeof(float), (cuuint64_t)ldv * sizeof(float)};
        cuuint32_t box[3] = {256, (cuuint32_t)(CH / 256), (cuuint32_t)R};
        cuuint32_t estr[3] = {1, 1, 1};
        if (enc)
          rc = enc(&mapV, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(V), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      }
      if (rc != CUDA_SUCCESS) fail(DHO2G_CUDA, "split_update: cuTensorMapEncodeTiled failed for V_hat");
    }
    kern<<<gt, kT, smem_t, st>>>(mapV, R, rows, a.g, a.pi, a.w_decay ? a.w_decay : a.w_a, all1, world, hp, o->m.p,
                                 o->v.p, o->s.p, o->part.p, o->rank2.p, o->ticket.p + 1, o->bad.p);
  } else {
    upd_p2_kernel<<<gp, kT, smem_p2, st>>>(
        V, ldv, R, rows, a.g, a.pi, a.w_decay ? a.w_decay : a.w_a, all1, world, hp, o->m.p, o->v.p, o->s.p, o->part.p,
        o->rank2.p, o->ticket.p + 1, o->bad.p);
  }
  DHO2G_LAUNCH();
  ctx->kt_end(k2, "upd_p2", rb * (R + 2 + (a.pi ? 1 : 0) + (adam ? 4 : (o->cfg.kind == 1 ? 2 : 0)) +
                                  (o->cfg.kind == 3 ? 1 : 0)));
  if (R > 0 && world > 1) ctx->allgather_f64(o->rank2.p, o->all2.p, R, "all_reduce");
  const int g3 = one_wave_grid(upd_p3_kernel, kT, (size_t)2 * R1 * sizeof(double), ctx->sm_count, cdiv(cdiv(rows, 4), kT));
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
  wait_stream(o->ctx, o->ctx->stream);
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
