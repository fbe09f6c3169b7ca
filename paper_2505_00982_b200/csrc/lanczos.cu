// Sharded Lanczos with full reorthogonalisation (reference: proj/src/dist_lanczos.cpp:31-119,
// lanczos.cpp:28-70), device tridiagonal eigensolve + Ritz extraction (dist_lanczos.cpp:121-158,
// linalg.cpp:140-226, lanczos.cpp:72-94).
//
// Per iteration i on this rank's basis rows (D column-major, lazily normalised: v_j = sigma_j D_j):
//   all_gather(D_i)  ->  h = H v_i (operator)  ->
//   pass 1: r_j = D_j^T h (j <= i), hh = ||h||^2           one read of D[:, 0..i] + h
//   [all_gather of the (i+2) fp64 partials, rank-ordered sum]
//   pass 2: h' = h - sum_j D_j e_j, ||h'||^2                one read of D[:, 0..i] + h, one write
// with e_j = sigma_j^2 r_j (classical Gram-Schmidt, the reference's arithmetic) or, by default, the
// recurrence-first form below.
//
// Recurrence-first projection (ctx option lanczos_recurrence, default on). The reference projects
// the raw h = H v_i against all of V in one classical Gram-Schmidt pass. With a basis whose
// orthogonality error is E (V^T V = I + E) that leaves V^T h' = -E V^T h, and V^T h is dominated by
// (alpha_i, beta_{i-1}) ~ ||H||, so the error grows by ~||H||/beta every iteration: from the fp32
// storage floor (1e-8) it reaches O(1) within ~25 iterations on spectra without a large gap (the
// fp64 reference itself does so within ~50). Here pass 1 also accumulates
// G_j = D_j^T D_i in the same sweep (D_i comes from L1: no extra HBM bytes), and pass 2 projects
// h - alpha v_i - beta v_{i-1} (the three-term recurrence) against V with coefficients
//   c_j = sigma_j (r_j - alpha sigma_i G_j - beta sigma_{i-1} G'_j),  G'_j = D_j^T D_{i-1} (kept
// from the previous iteration), i.e. the same single sweep with
//   e_j = sigma_j c_j + [j = i] alpha sigma_i + [j = i-1] beta sigma_{i-1}.
// Now V^T h' = -E c with c = O(E ||H||): orthogonality stays at the fp32 floor. alpha (= v_i^T h,
// pre-projection), pre-norm, beta = ||h'|| and the safeguard / breakdown rules are the reference's.
//   [all_gather of ||h'||^2 partials] -> decide (safeguard / breakdown / beta) on device
// The launch sequence is fixed (safeguard passes and post-breakdown iterations are predicated on
// device flags), so the whole refresh needs no host round trip.
#include <cmath>
#include <cstring>

#include "internal.h"

using namespace dho2g;

namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kSub = 512;  // rows per warp work item (32 lanes x 4 float4)
constexpr int kP2Unroll = 4;  // basis columns in flight per pass-2 thread (x 4 float4)

// ------------------------------------------------------------------ start vector
// seeded_unit_gaussian (lanczos.cpp:18-26): Rng(seed*phi + 0x1234567).fill_normal, computed
// counter-wise (SplitMix64 output i = mix(state0 + (i+1) phi); Box-Muller pairs (2p, 2p+1)).
__device__ __forceinline__ uint64_t splitmix_at(uint64_t s0, uint64_t i) {
  uint64_t z = s0 + (i + 1) * 0x9e3779b97f4a7c15ULL;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

__global__ void gauss_kernel(uint64_t s0, const uint64_t* __restrict__ s0p, size_t begin, size_t rows,
                             float* __restrict__ out, double* __restrict__ part) {
  __shared__ double sh[32];
  if (s0p) s0 = *s0p;  // graph replays read the refresh's seed from device memory
  double ss = 0.0;
  for (size_t r = blockIdx.x * (size_t)blockDim.x + threadIdx.x; r < rows; r += (size_t)gridDim.x * blockDim.x) {
    const size_t i = begin + r;
    const size_t p = i >> 1;
    const double u1 = ((double)(splitmix_at(s0, 2 * p) >> 11) + 1.0) * 0x1.0p-53;
    const double u2 = (double)(splitmix_at(s0, 2 * p + 1) >> 11) * 0x1.0p-53;
    const double radius = sqrt(-2.0 * log(u1));
    const double angle = 2.0 * 3.141592653589793 * u2;
    const double x = (i & 1) ? radius * sin(angle) : radius * cos(angle);
    out[r] = (float)x;
    ss += x * x;
  }
  const double t = block_sum(ss, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = t;
}

__global__ void gauss_norm_kernel(const double* __restrict__ part, int nb, double* __restrict__ rankp) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double s = 0.0;
    for (int b = 0; b < nb; ++b) s += part[b];
    rankp[0] = s;
  }
}

__global__ void lz_init_kernel(LzDev* st, const double* __restrict__ allp, int world, int stride) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double s = 0.0;
  for (int r = 0; r < world; ++r) s += allp[(size_t)r * stride];
  st->sigma[0] = (float)(1.0 / sqrt(s));
  st->iters = 0;
  st->stopped = 0;
  st->breakdown = 0;
  st->safeguards = 0;
  st->need_sg = 0;
  st->sg_cols = 0;
  st->nonfinite = 0;
  st->pre = 0.0;
  st->beta = 0.0;
}

// ------------------------------------------------------------------ GS pass 1: dots
// rankp[j] = D_j^T h (j < active), rankp[active] = h^T h, fp64, deterministic order.
// GRAM also accumulates G_j = D_j^T D_{active-1} (j < active) into rankp[goff + j].
//
// (butterfly_sum / butterfly_index: common.cuh)
template <bool GRAM>
__global__ void __launch_bounds__(kThreads) gs_pass1_kernel(const float* __restrict__ D, size_t ldd,
                                                            const float* __restrict__ h, int active, int nchunks,
                                                            int stride, double* __restrict__ part,
                                                            double* __restrict__ rankp, unsigned* ticket,
                                                            const LzDev* st, int safeguard_pass, int goff) {
  if (st->stopped || (safeguard_pass && !st->need_sg)) return;
  extern __shared__ __align__(16) unsigned char smem[];
  double* acc = reinterpret_cast<double*>(smem);  // [kWarps][active+1 (+active)]
  __shared__ bool is_last;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nj = active + 1;
  const int rowlen = nj + (GRAM ? active : 0);
  for (int e = threadIdx.x; e < kWarps * rowlen; e += kThreads) acc[e] = 0.0;
  __syncthreads();
  // Each warp owns one 512-row quarter q of every chunk of this CTA (kWarps / 4 warps per quarter,
  // splitting the columns j <= active between them, kCols columns per step). Its h segment (and
  // D_i's, for G) is loaded into registers once per chunk; per column only D_j's 2 KB segment is
  // streamed, so the sweep moves exactly the algorithmic bytes. 4-term products in fp32,
  // everything above in fp64.
  constexpr int kQuarters = kGsChunk / kSub;
  constexpr int kPerQuarter = kWarps / kQuarters;
  constexpr int kCols = 4;  // columns in flight per warp (4 x 2 KB)
  const int q = warp % kQuarters, j0 = warp / kQuarters;
  const int rb = q * kSub + lane * 4;
  const int my_chunks = blockIdx.x < nchunks ? (nchunks - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
  double* myacc = acc + warp * rowlen;
  for (int cl = 0; cl < my_chunks; ++cl) {
    const size_t r0 = ((size_t)blockIdx.x + (size_t)cl * gridDim.x) * kGsChunk;
    float4 y[4], z[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) y[k] = __ldg(reinterpret_cast<const float4*>(h + r0 + rb + k * 128));
    if (GRAM) {
      const float* zc = D + (size_t)(active - 1) * ldd + r0 + rb;
#pragma unroll
      for (int k = 0; k < 4; ++k) z[k] = __ldg(reinterpret_cast<const float4*>(zc + k * 128));
    }
    for (int ja = j0; ja <= active; ja += kCols * kPerQuarter) {
      constexpr int kVals = GRAM ? 2 * kCols : kCols;
      // all kCols segments in flight before any arithmetic (j == active is the ||h||^2 item: x = y)
      float4 x[kCols][4];
#pragma unroll
      for (int u = 0; u < kCols; ++u) {
        const int j = ja + u * kPerQuarter;
        const float* col = D + (size_t)min(j, active - 1) * ldd + r0 + rb;  // always a valid column
#pragma unroll
        for (int k = 0; k < 4; ++k) x[u][k] = __ldg(reinterpret_cast<const float4*>(col + k * 128));
        if (j >= active) {
#pragma unroll
          for (int k = 0; k < 4; ++k) x[u][k] = j == active ? y[k] : make_float4(0.f, 0.f, 0.f, 0.f);
        }
      }
      double v[kVals];
#pragma unroll
      for (int u = 0; u < kCols; ++u) {
        double sv = 0.0, gv = 0.0;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          sv += (double)(x[u][k].x * y[k].x + x[u][k].y * y[k].y + x[u][k].z * y[k].z + x[u][k].w * y[k].w);
          if (GRAM)  // G_j = D_j^T D_i
            gv += (double)(x[u][k].x * z[k].x + x[u][k].y * z[k].y + x[u][k].z * z[k].z + x[u][k].w * z[k].w);
        }
        if (GRAM) {
          v[2 * u] = sv;
          v[2 * u + 1] = gv;
        } else {
          v[u] = sv;
        }
      }
      const double t = butterfly_sum<kVals>(v, lane);
      if (lane < kVals) {
        const int idx = butterfly_index<kVals>(lane);
        const int u = GRAM ? idx >> 1 : idx;
        const int j = ja + u * kPerQuarter;
        if (GRAM && (idx & 1)) {
          if (j < active) myacc[nj + j] += t;
        } else if (j <= active) {
          myacc[j] += t;
        }
      }
    }
  }
  __syncthreads();
  for (int j = threadIdx.x; j < rowlen; j += kThreads) {
    double t = 0.0;
    for (int w = 0; w < kWarps; ++w) t += acc[w * rowlen + j];
    part[(size_t)blockIdx.x * stride + (j < nj ? j : goff + (j - nj))] = t;
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) is_last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!is_last) return;
  __threadfence();
  if (rowlen <= 4 * kWarps) {  // few values: a warp per value, lanes over the CTA partials
    for (int jj = warp; jj < rowlen; jj += kWarps) {
      const int j = jj < nj ? jj : goff + (jj - nj);
      const double t = warp_fold(part + j, (int)gridDim.x, (size_t)stride);
      if (lane == 0) rankp[j] = t;
    }
  } else {  // many values (long bases): a thread per value, its chain over the partials in CTA order
    for (int jj = threadIdx.x; jj < rowlen; jj += kThreads) {
      const int j = jj < nj ? jj : goff + (jj - nj);
      double t = 0.0;
      for (int b = 0; b < (int)gridDim.x; ++b) t += part[(size_t)b * stride + j];
      rankp[j] = t;
    }
  }
  if (threadIdx.x == 0) *ticket = 0u;
}

// ------------------------------------------------------------------ GS pass 2: projection
// dst = hsrc - sum_j D_j e_j with e_j = sigma_j^2 r_j (r_j rank-ordered sums of pass-1 partials);
// rankb[0] = ||dst||^2 for this rank. First pass also records alpha_i = diag[i] and pre.
__global__ void __launch_bounds__(kThreads) gs_pass2_kernel(const float* __restrict__ D, size_t ldd,
                                                            const float* hsrc, float* dst, int active, size_t ngroups,
                                                            const double* __restrict__ allp, int world, int stride,
                                                            double* __restrict__ part, double* __restrict__ rankb,
                                                            unsigned* ticket, LzDev* st, int it, int safeguard_pass,
                                                            int gram, int goff) {
  if (st->stopped || (safeguard_pass && !st->need_sg)) return;
  extern __shared__ __align__(16) unsigned char smem[];
  double* e = reinterpret_cast<double*>(smem);  // [active+1]
  double* gj = e + (active + 1);                // [active] (recurrence-first form)
  __shared__ double red[kWarps];
  __shared__ double alpha_s;
  __shared__ bool is_last;
  const bool rec = gram && !safeguard_pass;
  for (int j = threadIdx.x; j <= active; j += kThreads) {
    double r = 0.0;
    for (int w = 0; w < world; ++w) r += allp[(size_t)w * stride + j];
    if (j < active) {
      const double sg = (double)st->sigma[j];
      e[j] = rec ? r : sg * sg * r;
      if (j == it) alpha_s = sg * r;
      if (!safeguard_pass && j == it && blockIdx.x == 0) st->diag[it] = sg * r;  // alpha = v_i^T h
      if (rec) {
        double g = 0.0;
        for (int w = 0; w < world; ++w) g += allp[(size_t)w * stride + goff + j];
        gj[j] = g;
        if (blockIdx.x == 0) st->gram[it & 1][j] = g;  // G'_j of the next iteration
      }
    } else if (!safeguard_pass && blockIdx.x == 0) {
      st->pre = sqrt(r);
    }
  }
  __syncthreads();
  if (rec) {  // recurrence-first coefficients (header comment)
    const double alpha = alpha_s;
    const double si = (double)st->sigma[it];
    const double beta = it > 0 ? st->off[it - 1] : 0.0;
    const double sp = it > 0 ? (double)st->sigma[it - 1] : 0.0;
    for (int j = threadIdx.x; j < active; j += kThreads) {
      const double sj = (double)st->sigma[j];
      const double gp = it == 0 ? 0.0 : (j < it ? st->gram[(it - 1) & 1][j] : gj[it - 1]);
      const double c = sj * (e[j] - alpha * si * gj[j] - beta * sp * gp);
      double ej = sj * c;
      if (j == it) ej += alpha * si;
      if (j == it - 1) ej += beta * sp;
      e[j] = ej;
    }
    __syncthreads();
  }
  // Each warp owns super-groups of 128 float4 groups (512 rows): per basis column it streams one
  // contiguous 2 KB segment (lane l reads groups l, l+32, l+64, l+96), like pass 1's work items.
  double ss = 0.0;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const size_t nsg = ngroups / 128;
  for (size_t sgi = (size_t)blockIdx.x * kWarps + warp; sgi < nsg; sgi += (size_t)gridDim.x * kWarps) {
    const size_t g0 = sgi * 128 + lane;
    double a[4][4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float4 h4 = reinterpret_cast<const float4*>(hsrc)[g0 + 32 * q];
      a[q][0] = h4.x; a[q][1] = h4.y; a[q][2] = h4.z; a[q][3] = h4.w;
    }
    int j = 0;
    for (; j + kP2Unroll <= active; j += kP2Unroll) {
      float4 d[kP2Unroll][4];
#pragma unroll
      for (int u = 0; u < kP2Unroll; ++u)
#pragma unroll
        for (int q = 0; q < 4; ++q)
          d[u][q] = __ldg(reinterpret_cast<const float4*>(D + (size_t)(j + u) * ldd) + g0 + 32 * q);
#pragma unroll
      for (int u = 0; u < kP2Unroll; ++u) {
        const double c = e[j + u];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          a[q][0] -= (double)d[u][q].x * c;
          a[q][1] -= (double)d[u][q].y * c;
          a[q][2] -= (double)d[u][q].z * c;
          a[q][3] -= (double)d[u][q].w * c;
        }
      }
    }
    for (; j < active; ++j) {
      const double c = e[j];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float4 dd = __ldg(reinterpret_cast<const float4*>(D + (size_t)j * ldd) + g0 + 32 * q);
        a[q][0] -= (double)dd.x * c;
        a[q][1] -= (double)dd.y * c;
        a[q][2] -= (double)dd.z * c;
        a[q][3] -= (double)dd.w * c;
      }
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float4 o = make_float4((float)a[q][0], (float)a[q][1], (float)a[q][2], (float)a[q][3]);
      reinterpret_cast<float4*>(dst)[g0 + 32 * q] = o;
      ss += (double)o.x * o.x + (double)o.y * o.y + (double)o.z * o.z + (double)o.w * o.w;
    }
  }
  const double t = block_sum(ss, red);
  if (threadIdx.x == 0) part[blockIdx.x] = t;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) is_last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!is_last || warp != 0) return;
  __threadfence();
  const double s = warp_fold(part, (int)gridDim.x, 1);
  if (lane == 0) {
    rankb[0] = s;
    *ticket = 0u;
  }
}

// ------------------------------------------------------------------ decide (dist_lanczos.cpp:91-111)
__global__ void lz_decide_kernel(LzDev* st, const double* __restrict__ allb, int world, int stride, int it,
                                 int safeguard_pass, int safeguard_on, double ratio, double rtol) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  if (st->stopped || (safeguard_pass && !st->need_sg)) return;
  double b2 = 0.0;
  for (int w = 0; w < world; ++w) b2 += allb[(size_t)w * stride];
  const double beta = sqrt(b2);
  const double pre = st->pre;
  // dist_lanczos.cpp:80-82: a non-finite HVP stops the run (NaN fails every comparison below, so without
  // this it would flow into B and surface only as a non-converging eigensolve)
  if (!isfinite(pre) || !isfinite(beta) || !isfinite(st->diag[it])) {
    st->nonfinite = 1;
    st->stopped = 1;
    st->iters = it;
    return;
  }
  // fp32 adaptation of the reference thresholds (fp64 there): h and D are stored in fp32, so an
  // exactly invariant subspace leaves a residual at the fp32 rounding floor (~3e-8 pre), never at
  // 1e-10 pre; and a projection that cancels beyond ~1e-3 loses orthogonality at eps32/ratio.
  rtol = fmax(rtol, kBreakdownFloor32);
  ratio = fmax(ratio, kSafeguardFloor32);
  st->beta = beta;
  if (!safeguard_pass && safeguard_on && beta > rtol * pre && beta < ratio * pre) {
    st->need_sg = 1;
    st->safeguards += 1;
    st->sg_cols += it + 1;
    return;
  }
  st->need_sg = 0;
  if (beta <= rtol * pre) {  // invariant subspace: truncate (:99-108)
    st->breakdown = 1;
    st->stopped = 1;
    st->iters = it + 1;
    return;
  }
  st->off[it] = beta;
  st->sigma[it + 1] = (float)(1.0 / beta);
  st->iters = it + 1;
}

// ------------------------------------------------------------------ operators
__global__ void diag_apply_kernel(const float* __restrict__ spec, const float* __restrict__ v, const float* vscale,
                                  float* __restrict__ h, size_t rows) {
  const float sc = vscale ? *vscale : 1.f;
  for (size_t r = blockIdx.x * (size_t)blockDim.x + threadIdx.x; r < rows; r += (size_t)gridDim.x * blockDim.x)
    h[r] = (float)((double)spec[r] * (double)(sc * v[r]));
}

// out[r] = rs[r] * <M[:, r], vscale * v> for r < rows: one warp per column of a column-major
// n x rows panel (coalesced 128-B reads), fp64 accumulation. The dense operator (H symmetric, so
// row i == column i) and both GEMVs of the rotated quadratic (Q x with Q^T stored column-major,
// then Q^T y) are this kernel; it streams the panel once, so it is HBM-bound at 4 B per element.
__global__ void gemv_cols_kernel(const float* __restrict__ M, size_t n, size_t rows, const float* __restrict__ v,
                                 const float* vscale, const float* __restrict__ rs, float* __restrict__ out) {
  const float sc = vscale ? *vscale : 1.f;
  const int lane = threadIdx.x & 31;
  const size_t nwarps = ((size_t)gridDim.x * blockDim.x) >> 5;
  for (size_t r = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < rows; r += nwarps) {
    const float* col = M + r * n;
    double s0 = 0.0, s1 = 0.0;
    size_t j = lane;
    for (; j + 32 < n; j += 64) {
      s0 += (double)__ldg(col + j) * (double)(sc * v[j]);
      s1 += (double)__ldg(col + j + 32) * (double)(sc * v[j + 32]);
    }
    if (j < n) s0 += (double)__ldg(col + j) * (double)(sc * v[j]);
    const double s = warp_sum(s0 + s1);
    if (lane == 0) out[r] = (float)(rs ? (double)rs[r] * s : s);
  }
}

// out[0] = scale * <a, b> over `rows` (one CTA, fixed order: deterministic). Used for the quadratic
// oracle's value w^T H w / 2 on this rank's rows (O(n) next to the O(n^2) apply).
__global__ void __launch_bounds__(1024) dot_one_cta_kernel(const float* __restrict__ a, const float* __restrict__ b,
                                                           size_t rows, double scale, double* __restrict__ out) {
  __shared__ double red[32];
  double s = 0.0;
  for (size_t i = threadIdx.x; i < rows; i += blockDim.x) s += (double)a[i] * (double)b[i];
  const double t = block_sum(s, red);
  if (threadIdx.x == 0) out[0] = scale * t;
}

// ------------------------------------------------------------------ fused HVP -> reduce-scatter helpers
// (the weight-block GEMM epilogues store their elements into the owners' receive slots directly; these
// move the rest: bias blocks, an empty batch slice's zeros, and each owner's ordered sum of its slots)
__global__ void route_copy_kernel(const float* __restrict__ src, long long flat0, long long count,
                                  float* const* __restrict__ route, long long base, int rank) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < count; i += (long long)gridDim.x * blockDim.x) {
    const long long f = flat0 + i;
    const long long q = f / base;
    route[q][rank * base + (f - q * base)] = src ? src[f] : 0.f;
  }
}

__global__ void slot_sum_kernel(const float* __restrict__ recv, long long base, int world, long long rows,
                                float* __restrict__ h) {
  for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < rows; r += (long long)gridDim.x * blockDim.x) {
    float s = recv[r];
    for (int q = 1; q < world; ++q) s += recv[(long long)q * base + r];  // ascending rank order
    h[r] = s;
  }
}

// ------------------------------------------------------------------ tridiagonal eigensolve
// Single CTA, fp64 implicit-shift QL (linalg.cpp:140-226). Thread 0 runs the scalar recurrence
// of each sweep and records its Givens rotations; every thread then applies the sweep's
// rotations, in the reference's order, to its rows of Z (global, column-major n x n).
// Then stable ascending order (:199-212), extreme selection (lanczos.cpp:72-80) and
// U'[j][c] = sigma_j * Z[j, idx_c] (folds the lazy basis normalisation into the Ritz GEMM).
__global__ void tql2_kernel(const LzDev* st, int n, int keff, int leff, double* __restrict__ Z,
                            float* __restrict__ Usel, double* __restrict__ evsel, double* __restrict__ evall,
                            int* __restrict__ status) {
  extern __shared__ double sh[];
  double* d = sh;
  double* e = d + n;
  double* cs = e + n;
  double* sn = cs + n;
  int* order = reinterpret_cast<int*>(sn + n);
  __shared__ int s_mm, s_cnt, s_fail;
  const int tid = threadIdx.x;
  for (int i = tid; i < n; i += blockDim.x) {
    d[i] = st->diag[i];
    e[i] = (i + 1 < n) ? st->off[i] : 0.0;
  }
  for (size_t q = tid; q < (size_t)n * n; q += blockDim.x) Z[q] = ((q / n) == (q % n)) ? 1.0 : 0.0;
  if (tid == 0) s_fail = 0;
  __syncthreads();
  const double eps = 2.220446049250313e-16;
  if (tid == 0) s_mm = n - 1;
  __syncthreads();
  for (int l = 0; l < n && n > 1; ++l) {
    int iter = 0;
    for (;;) {
      // mm = first index >= l with a negligible off-diagonal (n-1 if none): every thread tests its
      // indices, the smallest wins (the reference scans serially, linalg.cpp:160-164; same result)
      for (int q = l + tid; q + 1 < n; q += blockDim.x)
        if (fabs(e[q]) <= eps * (fabs(d[q]) + fabs(d[q + 1]))) atomicMin(&s_mm, q);
      __syncthreads();
      if (tid == 0) {
        const int mm = s_mm;
        s_cnt = 0;
        if (mm != l) {
          if (iter++ == 60) {
            s_fail = 1;
          } else {
            double g = (d[l + 1] - d[l]) / (2.0 * e[l]);
            double r = sqrt(fma(g, g, 1.0));
            g = d[mm] - d[l] + e[l] / (g + copysign(r, g));
            double s = 1.0, c = 1.0, p = 0.0;
            bool under = false;
            int cnt = 0;
            // the serial chain is this kernel's latency: d[ii+1] is carried in a register and the next
            // e / d entries (untouched by this step) are read one step ahead
            double dk = d[mm], ek = e[mm - 1], dn = d[mm - 1];
            for (int ii = mm - 1; ii >= l; --ii) {
              const double en = ii > l ? e[ii - 1] : 0.0, dnn = ii > l ? d[ii - 1] : 0.0;
              const double f = s * ek;
              const double b = c * ek;
              // 1/sqrt(f^2 + g^2) instead of hypot and a division: the entries of a Lanczos tridiagonal
              // are O(||H||), far from fp64 over/underflow
              const double h2 = fma(f, f, g * g);
              if (h2 == 0.0) {
                e[ii + 1] = 0.0;
                d[ii + 1] = dk - p;
                e[mm] = 0.0;
                under = true;
                break;
              }
              const double gb2 = 2.0 * g * b;  // 2 c b = (2 g b) / r: off the rsqrt's critical path
              const double ir = rsqrt(h2);
              r = h2 * ir;
              e[ii + 1] = r;
              s = f * ir;
              c = g * ir;
              g = dk - p;
              r = fma(dn - g, s, gb2 * ir);
              p = s * r;
              d[ii + 1] = g + p;
              g = c * r - b;
              cs[cnt] = c;
              sn[cnt] = s;
              ++cnt;
              dk = dn;
              dn = dnn;
              ek = en;
            }
            s_cnt = cnt;
            if (!under) {
              d[l] -= p;
              e[l] = g;
              e[mm] = 0.0;
            }
          }
        }
      }
      __syncthreads();
      const int mm = s_mm, cnt = s_cnt, failed = s_fail;
      __syncthreads();  // everyone has read the sweep descriptor before it is rewritten
      if (tid == 0) s_mm = n - 1;  // reset for the next scan
      __syncthreads();
      if (failed) {
        if (tid == 0) *status = 1;
        return;
      }
      if (mm == l) break;
      for (int k = tid; k < n; k += blockDim.x) {
        // rotation q turns rows (ii, ii+1), ii = mm-1-q: row ii+1 is final after it and row ii is carried
        // (in a register) into rotation q+1, so only the untouched row ii-1 is loaded per step
        if (cnt > 0) {
          double f = Z[(size_t)mm * n + k];
          double z0 = Z[(size_t)(mm - 1) * n + k];
          for (int q = 0; q < cnt; ++q) {
            const int ii = mm - 1 - q;
            const double zn = q + 1 < cnt ? Z[(size_t)(ii - 1) * n + k] : 0.0;
            const double c = cs[q], s = sn[q];
            Z[(size_t)(ii + 1) * n + k] = s * z0 + c * f;
            f = c * z0 - s * f;
            z0 = zn;
          }
          Z[(size_t)(mm - cnt) * n + k] = f;
        }
      }
      __syncthreads();
    }
  }
  __syncthreads();
  // stable ascending order
  for (int i = tid; i < n; i += blockDim.x) {
    int rank = 0;
    const double di = d[i];
    for (int j = 0; j < n; ++j) rank += (d[j] < di) || (d[j] == di && j < i);
    order[rank] = i;
  }
  __syncthreads();
  for (int i = tid; i < n; i += blockDim.x) evall[i] = d[order[i]];
  const int r = keff + leff;
  for (int c = 0; c < r; ++c) {
    const int idx = c < keff ? order[n - 1 - c] : order[c - keff];
    if (tid == 0) evsel[c] = d[idx];
    for (int j = tid; j < n; j += blockDim.x)
      Usel[(size_t)j * r + c] = (float)((double)st->sigma[j] * Z[(size_t)idx * n + j]);
  }
  if (tid == 0) *status = 0;
}

// Split form of tql2_kernel (ctx option tql2_split): the same QL sweeps and rotations, with the
// rotation stream decoupled from its application. Every component k of the eigenvector slots is rotated
// independently of the others, so the application only has to follow the recorded stream:
//   tql2_pipe_kernel   1 + ceil(n / T) CTAs of 32 threads. The first CTA to start (ticket 0) is the
//                      producer: one warp runs the implicit-shift QL chain (linalg.cpp:140-197) with a
//                      warp-ballot deflation scan and appends each sweep's (mm, cnt, offset) and its
//                      rotations (c, s) to a log in HBM (worst case 30 n (n-1) rotations: at most 60
//                      sweeps per l before the reference's iteration limit), publishing the sweep count
//                      with st.release every >= 256 rotations. Every other CTA is a consumer: lane t < T
//                      owns component k of all n slots in shared memory (n * T * 8 bytes), stages each
//                      published sweep's rotations into shared memory (coalesced L2 loads, all lanes) and
//                      replays them with the register-carried order of tql2_kernel (same arithmetic).
//                      The producer never waits on a consumer and is the first CTA running, so the spin
//                      cannot deadlock; the replay overlaps the chain and trails it by one batch.
//   tql2_select_kernel stable ascending order, extreme selection and U' (as the tail of tql2_kernel).
// The single-CTA kernel alternates the chain with an L2-bound application (512 threads x 16 B per
// rotation through one SM at m = 512); here the eigensolve costs the chain alone.
__device__ __forceinline__ int ld_acquire_gpu(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_gpu(int* p, int v) {
  asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// sync[0] ticket, sync[1] published sweeps, sync[2] done (zeroed before the launch)
// status: 1 = no convergence within the reference's 60 sweeps per l, 2 = the rotation log (cap entries) is full
// (the host reruns the eigensolve with the single-CTA kernel)
__global__ void __launch_bounds__(32) tql2_pipe_kernel(const LzDev* st, int n, int T, double2* __restrict__ rot,
                                                       long long cap, int4* __restrict__ sweep,
                                                       int* __restrict__ sync, double* __restrict__ dout,
                                                       int* __restrict__ status, double* __restrict__ Z) {
  extern __shared__ double sh[];
  __shared__ int s_role;
  const int lane = threadIdx.x;
  if (lane == 0) s_role = atomicAdd(sync, 1);
  __syncwarp();
  const int role = s_role;
  if (role == 0) {  // ------------------------------------------------ producer: the QL chain
    double* d = sh;
    double* e = d + n;
    for (int i = lane; i < n; i += 32) {
      d[i] = st->diag[i];
      e[i] = (i + 1 < n) ? st->off[i] : 0.0;
    }
    __syncwarp();
    const double eps = 2.220446049250313e-16;
    int ns = 0, off = 0, pub = 0, fail = 0;
    for (int l = 0; l < n && n > 1 && !fail; ++l) {
      int iter = 0;
      for (;;) {
        // first q >= l with a negligible e[q] (linalg.cpp:160-164), n - 1 if none
        int mm = n - 1;
        for (int q0 = l; q0 + 1 < n; q0 += 32) {
          const int q = q0 + lane;
          const bool hit = q + 1 < n && fabs(e[q]) <= eps * (fabs(d[q]) + fabs(d[q + 1]));
          const unsigned b = __ballot_sync(0xffffffffu, hit);
          if (b) {
            mm = q0 + __ffs(b) - 1;
            break;
          }
        }
        if (mm == l) break;
        if (iter++ == 60) {
          fail = 1;
          break;
        }
        if ((long long)off + (mm - l) > cap) {  // this sweep could overflow the log
          fail = 2;
          break;
        }
        int cnt = 0;
        if (lane == 0) {
          double g = (d[l + 1] - d[l]) / (2.0 * e[l]);
          double r = sqrt(fma(g, g, 1.0));
          g = d[mm] - d[l] + e[l] / (g + copysign(r, g));
          double s = 1.0, c = 1.0, p = 0.0;
          bool under = false;
          double dk = d[mm], ek = e[mm - 1], dn = d[mm - 1];
          double2* out = rot + off;
          for (int ii = mm - 1; ii >= l; --ii) {
            const double en = ii > l ? e[ii - 1] : 0.0, dnn = ii > l ? d[ii - 1] : 0.0;
            const double f = s * ek;
            const double b = c * ek;
            const double h2 = fma(f, f, g * g);
            if (h2 == 0.0) {
              e[ii + 1] = 0.0;
              d[ii + 1] = dk - p;
              e[mm] = 0.0;
              under = true;
              break;
            }
            const double gb2 = 2.0 * g * b;  // 2 c b = (2 g b) / r: off the rsqrt's critical path
            const double ir = rsqrt(h2);
            r = h2 * ir;
            e[ii + 1] = r;
            s = f * ir;
            c = g * ir;
            g = dk - p;
            r = fma(dn - g, s, gb2 * ir);
            p = s * r;
            d[ii + 1] = g + p;
            g = c * r - b;
            out[cnt] = make_double2(c, s);
            ++cnt;
            dk = dn;
            dn = dnn;
            ek = en;
          }
          if (!under) {
            d[l] -= p;
            e[l] = g;
            e[mm] = 0.0;
          }
          if (cnt > 0) {
            sweep[ns] = make_int4(mm, cnt, off, 0);
            if (off + cnt - pub >= 256) {  // batch the publications (each release drains the stores)
              st_release_gpu(sync + 1, ns + 1);
              pub = off + cnt;
            }
          }
        }
        cnt = __shfl_sync(0xffffffffu, cnt, 0);
        if (cnt > 0) {
          ++ns;
          off += cnt;
        }
        __syncwarp();  // lane 0's d / e updates are visible to the next scan
      }
    }
    for (int i = lane; i < n; i += 32) dout[i] = d[i];
    if (lane == 0) {
      *status = fail;
      st_release_gpu(sync + 1, ns);
      st_release_gpu(sync + 2, 1);
    }
    return;
  }
  // ------------------------------------------------------------------ consumer: replay the log
  double* zs = sh;                                              // zs[i * T + t]: slot i, component k
  double2* stage = reinterpret_cast<double2*>(zs + (size_t)n * T);  // one sweep's rotations
  const int k = (role - 1) * T + lane;
  const bool own = lane < T && k < n;
  if (own)
    for (int i = 0; i < n; ++i) zs[(size_t)i * T + lane] = (i == k) ? 1.0 : 0.0;
  int w = 0;
  for (;;) {
    int avail = ld_acquire_gpu(sync + 1);
    if (w >= avail) {
      if (!ld_acquire_gpu(sync + 2)) {
        __nanosleep(128);
        continue;
      }
      avail = ld_acquire_gpu(sync + 1);  // final count (released before done)
      if (w >= avail) break;
    }
    for (; w < avail; ++w) {
      const int4 sw = __ldcg(sweep + w);
      const int mm = sw.x, cnt = sw.y;
      for (int q = lane; q < cnt; q += 32) stage[q] = __ldcg(rot + sw.z + q);
      __syncwarp();
      if (own) {
        double f = zs[(size_t)mm * T + lane];
        double z0 = zs[(size_t)(mm - 1) * T + lane];
#pragma unroll 4
        for (int q = 0; q < cnt; ++q) {
          const int ii = mm - 1 - q;
          const double zn = q + 1 < cnt ? zs[(size_t)(ii - 1) * T + lane] : 0.0;
          const double2 cs = stage[q];
          const double c = cs.x, s = cs.y;
          zs[(size_t)(ii + 1) * T + lane] = s * z0 + c * f;
          f = c * z0 - s * f;
          z0 = zn;
        }
        zs[(size_t)(mm - cnt) * T + lane] = f;
      }
      __syncwarp();  // the stage is rewritten by the next sweep
    }
  }
  if (own)
    for (int i = 0; i < n; ++i) Z[(size_t)i * n + k] = zs[(size_t)i * T + lane];
}

__global__ void tql2_select_kernel(const LzDev* st, int n, int keff, int leff, const double* __restrict__ dall,
                                   const double* __restrict__ Z, float* __restrict__ Usel,
                                   double* __restrict__ evsel, double* __restrict__ evall,
                                   const int* __restrict__ status) {
  extern __shared__ double sh[];
  double* d = sh;
  int* order = reinterpret_cast<int*>(d + n);
  const int tid = threadIdx.x;
  if (*status != 0) return;
  for (int i = tid; i < n; i += blockDim.x) d[i] = dall[i];
  __syncthreads();
  for (int i = tid; i < n; i += blockDim.x) {
    int rank = 0;
    const double di = d[i];
    for (int j = 0; j < n; ++j) rank += (d[j] < di) || (d[j] == di && j < i);
    order[rank] = i;
  }
  __syncthreads();
  for (int i = tid; i < n; i += blockDim.x) evall[i] = d[order[i]];
  const int r = keff + leff;
  for (int c = 0; c < r; ++c) {
    const int idx = c < keff ? order[n - 1 - c] : order[c - keff];
    if (tid == 0) evsel[c] = d[idx];
    for (int j = tid; j < n; j += blockDim.x)
      Usel[(size_t)j * r + c] = (float)((double)st->sigma[j] * Z[(size_t)idx * n + j]);
  }
}

// ------------------------------------------------------------------ Ritz vectors
// V[:, c0:c0+RC] = D[:, 0:me] U'[:, c0:c0+RC]  (bandwidth-bound tall-skinny GEMM)
constexpr int RC = 32;
__global__ void __launch_bounds__(256) ritz_kernel(const float* __restrict__ D, size_t ldd, int me,
                                                   const float* __restrict__ Usel, int r, int c0,
                                                   float* __restrict__ V, size_t ldv, size_t rows) {
  // V[:, c0 + c] = D[:, :me] Usel[:, c0 + c]. Each thread owns 2 adjacent rows (float2 loads of D),
  // so every broadcast shared-memory read of Usel feeds 8 FMAs; basis columns go in groups of 8
  // with all loads issued before the FMAs (groups of 8). Rows are padded to whole chunks (ldd, ldv even).
  extern __shared__ __align__(16) float us[];  // me x RC
  const int nc = min(RC, r - c0);
  for (int q = threadIdx.x; q < me * RC; q += blockDim.x) {
    const int j = q / RC, c = q % RC;
    us[q] = c < nc ? Usel[(size_t)j * r + c0 + c] : 0.f;
  }
  __syncthreads();
  const size_t npairs = (rows + 1) / 2;
  for (size_t pr = blockIdx.x * (size_t)blockDim.x + threadIdx.x; pr < npairs; pr += (size_t)gridDim.x * blockDim.x) {
    const size_t row = 2 * pr;
    float a0[RC], a1[RC];
#pragma unroll
    for (int c = 0; c < RC; ++c) a0[c] = a1[c] = 0.f;
    int j = 0;
    for (; j + 8 <= me; j += 8) {
      float2 x[8];
#pragma unroll
      for (int t = 0; t < 8; ++t) x[t] = __ldg(reinterpret_cast<const float2*>(D + (size_t)(j + t) * ldd + row));
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        const float4* u4 = reinterpret_cast<const float4*>(us + (j + t) * RC);
#pragma unroll
        for (int q = 0; q < RC / 4; ++q) {
          const float4 u = u4[q];
          a0[4 * q] = fmaf(x[t].x, u.x, a0[4 * q]);
          a0[4 * q + 1] = fmaf(x[t].x, u.y, a0[4 * q + 1]);
          a0[4 * q + 2] = fmaf(x[t].x, u.z, a0[4 * q + 2]);
          a0[4 * q + 3] = fmaf(x[t].x, u.w, a0[4 * q + 3]);
          a1[4 * q] = fmaf(x[t].y, u.x, a1[4 * q]);
          a1[4 * q + 1] = fmaf(x[t].y, u.y, a1[4 * q + 1]);
          a1[4 * q + 2] = fmaf(x[t].y, u.z, a1[4 * q + 2]);
          a1[4 * q + 3] = fmaf(x[t].y, u.w, a1[4 * q + 3]);
        }
      }
    }
    for (; j < me; ++j) {
      const float2 x = __ldg(reinterpret_cast<const float2*>(D + (size_t)j * ldd + row));
      const float4* u4 = reinterpret_cast<const float4*>(us + j * RC);
#pragma unroll
      for (int q = 0; q < RC / 4; ++q) {
        const float4 u = u4[q];
        a0[4 * q] = fmaf(x.x, u.x, a0[4 * q]);
        a0[4 * q + 1] = fmaf(x.x, u.y, a0[4 * q + 1]);
        a0[4 * q + 2] = fmaf(x.x, u.z, a0[4 * q + 2]);
        a0[4 * q + 3] = fmaf(x.x, u.w, a0[4 * q + 3]);
        a1[4 * q] = fmaf(x.y, u.x, a1[4 * q]);
        a1[4 * q + 1] = fmaf(x.y, u.y, a1[4 * q + 1]);
        a1[4 * q + 2] = fmaf(x.y, u.z, a1[4 * q + 2]);
        a1[4 * q + 3] = fmaf(x.y, u.w, a1[4 * q + 3]);
      }
    }
    const bool two = row + 1 < rows;
#pragma unroll
    for (int c = 0; c < RC; ++c)
      if (c < nc) {
        float* dst = V + (size_t)(c0 + c) * ldv + row;
        if (two) *reinterpret_cast<float2*>(dst) = make_float2(a0[c], a1[c]);
        else dst[0] = a0[c];
      }
  }
}

// per-column argmax |x| with the lowest index on ties (lanczos.cpp:82-94): blocks own contiguous
// row segments of one column; partials (maxabs, global index, value) merged in segment order.
constexpr int kArgThreads = 256;
__global__ void col_argmax_kernel(const float* __restrict__ V, size_t ldv, size_t rows, size_t begin, size_t seg,
                                  double* __restrict__ part /* [c][blk][3] */) {
  const int c = blockIdx.y;
  const float* col = V + (size_t)c * ldv;
  const size_t r0 = blockIdx.x * seg, r1 = min(rows, r0 + seg);
  float best = -1.f;
  size_t bi = r0;
  float bv = 0.f;
  for (size_t r = r0 + threadIdx.x; r < r1; r += kArgThreads) {
    const float x = col[r];
    const float a = fabsf(x);
    if (a > best) {
      best = a;
      bi = r;
      bv = x;
    }
  }
  __shared__ float sb[kArgThreads];
  __shared__ size_t si[kArgThreads];
  __shared__ float sv[kArgThreads];
  sb[threadIdx.x] = best;
  si[threadIdx.x] = bi;
  sv[threadIdx.x] = bv;
  __syncthreads();
  for (int s = kArgThreads / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      const float ob = sb[threadIdx.x + s];
      const size_t oi = si[threadIdx.x + s];
      if (ob > sb[threadIdx.x] || (ob == sb[threadIdx.x] && oi < si[threadIdx.x])) {
        sb[threadIdx.x] = ob;
        si[threadIdx.x] = oi;
        sv[threadIdx.x] = sv[threadIdx.x + s];
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    double* o = part + ((size_t)c * gridDim.x + blockIdx.x) * 3;
    o[0] = sb[0];
    o[1] = (double)(begin + si[0]);
    o[2] = sv[0];
  }
}

__global__ void col_argmax_final_kernel(const double* __restrict__ part, int nblk, double* __restrict__ out) {
  const int c = blockIdx.x;
  if (threadIdx.x != 0) return;
  const double* p = part + (size_t)c * nblk * 3;
  double best = p[0], bidx = p[1], bval = p[2];
  for (int b = 1; b < nblk; ++b)  // later segments win only on a strictly larger |x|
    if (p[3 * b] > best) {
      best = p[3 * b];
      bidx = p[3 * b + 1];
      bval = p[3 * b + 2];
    }
  out[3 * c] = best;
  out[3 * c + 1] = bidx;
  out[3 * c + 2] = bval;
}

int grid_for(dho2g_ctx* ctx, size_t work, int threads, int per_sm = 4) {
  const size_t want = cdiv(work, threads);
  const size_t cap = (size_t)ctx->sm_count * per_sm;
  return (int)std::max<size_t>(1, std::min(want, cap));
}

}  // namespace

// ------------------------------------------------------------------ dho2g_op::apply
void dho2g_op::load_mlp_input() {
  dho2g_mlp* m = mlp;
  // a rank whose slice of the curvature batch is empty (B < G) contributes zeros and runs no HVP
  if (b1 > b0 && (m->w_cur != wptr || !weights_loaded || m->input_owner != this ||
                  m->f16 != (ctx->gemm_f16 ? 1 : 0))) {
    if (idx.p) mlp_set_input(m, Xptr, yptr, idx.p + b0, b1 - b0, true);
    else mlp_set_input(m, Xptr + b0 * m->sizes[0], yptr + b0, nullptr, b1 - b0, true);
    mlp_load_weights(m, wptr);
    m->input_owner = this;
    weights_loaded = true;
  }
}

void dho2g_op::apply(const float* vfull, const float* vscale, float* h_shard, size_t begin, size_t rows, size_t base) {
  cudaStream_t st = ctx->stream;
  if (kind == 0) {
    dho2g_mlp* m = mlp;
    load_mlp_input();
    float* out = ctx->world == 1 ? h_shard : hfull.p;
    if (ctx->world > 1 && ctx->hvp_route) {
      // fused reduce-scatter: the weight-block GEMMs write every W element straight into its owner's
      // receive slot for this rank (peer memory); bias blocks and an empty slice are routed by copies;
      // after a barrier each owner sums its slots in rank order
      if (b1 > b0) {
        route_begin(base);
        try {
          mlp_hvp_dev(m, vfull, vscale, b1 - b0, ncls, scale, out);
        } catch (...) {
          m->route = nullptr;
          throw;
        }
      }
      route_end(out, b1 <= b0, h_shard, rows, base);
      return;
    }
    if (b1 > b0) {
      mlp_hvp_dev(m, vfull, vscale, b1 - b0, ncls, scale, out);
    } else {
      DHO2G_CUDA(cudaMemsetAsync(out, 0, n * sizeof(float), st));
    }
    if (ctx->world > 1) ctx->reduce_scatter_f32(hfull.p, h_shard, base);
    return;
  }
  if (kind == 1) {
    diag_apply_kernel<<<grid_for(ctx, rows, 256), 256, 0, st>>>(mat.p + begin, vfull + begin, vscale, h_shard, rows);
    DHO2G_LAUNCH();
    return;
  }
  if (kind == 2) {
    if (rows) {
      gemv_cols_kernel<<<grid_for(ctx, rows * 32, 256, 8), 256, 0, st>>>(mat.p + begin * n, n, rows, vfull, vscale,
                                                                        nullptr, h_shard);
      DHO2G_LAUNCH();
    }
    return;
  }
  if (kind == 4) {  // QuadraticOracle::apply_h, rotated (oracle.cpp:269-271): Q^T (spec o (Q v))
    if (begin != q_begin || rows != q_rows) fail(DHO2G_ARGUMENT, "quadratic operator: sharding changed since creation");
    float* yl = ctx->world == 1 ? qy.p : qy_loc.p;
    if (rows) {
      gemv_cols_kernel<<<grid_for(ctx, rows * 32, 256, 8), 256, 0, st>>>(qrot_t.p, n, rows, vfull, vscale,
                                                                        mat.p + begin, yl);
      DHO2G_LAUNCH();
    }
    if (ctx->world > 1) ctx->allgather_f32(qy_loc.p, qy.p, base);  // base == ceil(n/G): padded == global index
    if (rows) {
      gemv_cols_kernel<<<grid_for(ctx, rows * 32, 256, 8), 256, 0, st>>>(qrot.p, n, rows, qy.p, nullptr, nullptr,
                                                                        h_shard);
      DHO2G_LAUNCH();
    }
    return;
  }
  // host callback (tests / reference HvpFn adapters)
  pin.ensure(n + 1);
  DHO2G_CUDA(cudaMemcpyAsync(pin.p, vfull, n * sizeof(float), cudaMemcpyDeviceToHost, st));
  if (vscale) DHO2G_CUDA(cudaMemcpyAsync(pin.p + n, vscale, sizeof(float), cudaMemcpyDeviceToHost, st));
  DHO2G_CUDA(cudaStreamSynchronize(st));
  const double sc = vscale ? pin.p[n] : 1.0;
  hv_in.resize(n);
  hv_out.assign(n, 0.0);
  for (size_t i = 0; i < n; ++i) hv_in[i] = sc * (double)pin.p[i];
  fn(user, hv_in.data(), hv_out.data(), n);
  for (size_t r = 0; r < rows; ++r) pin.p[r] = (float)hv_out[begin + r];
  DHO2G_CUDA(cudaMemcpyAsync(h_shard, pin.p, rows * sizeof(float), cudaMemcpyHostToDevice, st));
  DHO2G_CUDA(cudaStreamSynchronize(st));
}

// Receive buffer (world slots of base floats) and the table of every rank's buffer: raw pointers on the
// in-process fabric (one address space), CUDA IPC handles exchanged through the communicator otherwise
// (peer access over NVLink).
void dho2g_op::route_setup(size_t base) {
  const int G = ctx->world;
  if (recv.p && recv.n >= base * G && route_tab.p) return;
  if (recv.p) {
    // growing: every rank is here (route_setup is collective); once all ranks have finished with the old
    // receive buffers (barrier) the stale peer mappings are closed before the owners free them
    ctx->barrier();
    dho2g::wait_stream(ctx, ctx->stream);
    for (void* p : ipc_opened) cudaIpcCloseMemHandle(p);
    ipc_opened.clear();
  }
  recv.alloc(base * G);
  route_tab.alloc(G);
  std::vector<float*> tab(G, nullptr);
  dho2g::DevBuf<double> ex(16 * (size_t)(G + 1));
  if (ctx->fabric) {
    double mine;
    const float* p = recv.p;
    std::memcpy(&mine, &p, sizeof(mine));
    DHO2G_CUDA(cudaMemcpyAsync(ex.p, &mine, sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    ctx->allgather_f64(ex.p, ex.p + 16, 1, "all_gather");
    std::vector<double> all(G);
    DHO2G_CUDA(cudaMemcpyAsync(all.data(), ex.p + 16, G * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    dho2g::wait_stream(ctx, ctx->stream);
    for (int q = 0; q < G; ++q) std::memcpy(&tab[q], &all[q], sizeof(float*));
  } else {
    static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
    cudaIpcMemHandle_t h;
    DHO2G_CUDA(cudaIpcGetMemHandle(&h, recv.p));
    double mine[8];
    std::memcpy(mine, &h, 64);
    DHO2G_CUDA(cudaMemcpyAsync(ex.p, mine, 64, cudaMemcpyHostToDevice, ctx->stream));
    ctx->allgather_f64(ex.p, ex.p + 16, 8, "all_gather");
    std::vector<double> all(8 * (size_t)G);
    DHO2G_CUDA(cudaMemcpyAsync(all.data(), ex.p + 16, all.size() * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    dho2g::wait_stream(ctx, ctx->stream);
    for (int q = 0; q < G; ++q) {
      if (q == ctx->rank) {
        tab[q] = recv.p;
        continue;
      }
      cudaIpcMemHandle_t hq;
      std::memcpy(&hq, &all[8 * (size_t)q], 64);
      void* ptr = nullptr;
      DHO2G_CUDA(cudaIpcOpenMemHandle(&ptr, hq, cudaIpcMemLazyEnablePeerAccess));
      ipc_opened.push_back(ptr);
      tab[q] = static_cast<float*>(ptr);
    }
  }
  DHO2G_CUDA(cudaMemcpyAsync(route_tab.p, tab.data(), G * sizeof(float*), cudaMemcpyHostToDevice, ctx->stream));
  dho2g::wait_stream(ctx, ctx->stream);
}

void dho2g_op::route_begin(size_t base) {
  route_setup(base);
  mlp->route = route_tab.p;
  mlp->route_base = (long long)base;
  mlp->route_rank = ctx->rank;
}

void dho2g_op::route_end(const float* full, bool empty, float* shard, size_t rows, size_t base) {
  cudaStream_t st = ctx->stream;
  route_setup(base);
  mlp->route = nullptr;
  if (!empty) {
    for (const LayerDesc& ld : mlp->layers)
      route_copy_kernel<<<grid_for(ctx, ld.out, 256), 256, 0, st>>>(full, (long long)ld.b_off, ld.out, route_tab.p,
                                                                 (long long)base, ctx->rank);
  } else {
    route_copy_kernel<<<grid_for(ctx, n, 256), 256, 0, st>>>(nullptr, 0, (long long)n, route_tab.p, (long long)base,
                                                          ctx->rank);
  }
  DHO2G_LAUNCH();
  ctx->barrier();  // every rank's stores into this rank's slots are complete
  slot_sum_kernel<<<grid_for(ctx, rows, 256), 256, 0, st>>>(recv.p, (long long)base, ctx->world, (long long)rows,
                                                            shard);
  DHO2G_LAUNCH();
}

dho2g_op::~dho2g_op() {
  for (void* p : ipc_opened) cudaIpcCloseMemHandle(p);
}

namespace dho2g {

void dot_dev(cudaStream_t st, const float* a, const float* b, size_t rows, double scale, double* out) {
  dot_one_cta_kernel<<<1, 1024, 0, st>>>(a, b, rows, scale, out);
  DHO2G_LAUNCH();
}

void lanczos_alloc(dho2g_lanczos* lz, dho2g_ctx* ctx, size_t n, size_t m) {
  lz->ctx = ctx;
  lz->n = n;
  lz->m = m;
  shard_range(n, ctx->world, ctx->rank, &lz->begin, &lz->end);
  lz->rows = lz->end - lz->begin;
  lz->base = cdiv(n, (size_t)ctx->world);
  lz->ldd = round_up(std::max<size_t>(lz->base, 1), kGsChunk);
  lz->D.alloc(lz->ldd * (m + 1));
  lz->h.alloc(lz->ldd);
  if (ctx->world > 1) lz->vfull.alloc(lz->base * ctx->world);
  lz->st.alloc(1);
  const int g1 = ctx->sm_count * 8;  // upper bound of the one-wave grids (256-thread CTAs, <= 8 per SM)
  const int g2 = ctx->sm_count * 8;
  // per-CTA / per-rank partial rows: [r_0..r_i, ||h||^2] at 0, [G_0..G_{i-1}] at m + 2
  lz->part.alloc((size_t)std::max(g1, g2) * 2 * (m + 2) + 8);
  lz->rankp.alloc(2 * (m + 2));
  lz->allp.alloc(2 * (m + 2) * ctx->world);
  const size_t smem1_max = (size_t)kWarps * (2 * m + 2) * sizeof(double);
  if (smem1_max > 48 * 1024) {
    DHO2G_CUDA(cudaFuncSetAttribute(gs_pass1_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem1_max));
    DHO2G_CUDA(cudaFuncSetAttribute(gs_pass1_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem1_max));
  }
  lz->ticket.alloc(2);
  // SlotMeter names of dist_lanczos.cpp:41-84 (logical slots; the basis is stored padded to ldd rows)
  ctx->meter("D_shard", (int64_t)(lz->rows * (m + 1)));
  ctx->meter("B", (int64_t)(2 * m + 1));
  ctx->meter("h_shard", (int64_t)lz->rows);
  if (ctx->world > 1) ctx->meter("v_full", (int64_t)n);
  ++g_graph_gen;
}

// The refresh's launch sequence (v1, then m x [HVP, GS pass 1, GS pass 2, decide] with device-resident
// predication) depends on the host only through the seed, so at world 1 it is captured once into a CUDA
// graph and replayed; the seed goes through device memory. Captures are invalidated by any device
// (re)allocation (pointers baked into the graph) and the split-K / stream-K flags are cleared inside the
// graph (their epoch values are baked too).
static void lanczos_enqueue(dho2g_lanczos* lz, dho2g_op* op, uint64_t s0, const uint64_t* s0p) {
  dho2g_ctx* ctx = lz->ctx;
  cudaStream_t st = ctx->stream;
  const size_t m = lz->m;
  const int world = ctx->world;
  const int stride = (int)(2 * (m + 2));
  const int goff = (int)(m + 2);
  const int gram = ctx->lanczos_recurrence ? 1 : 0;
  // v1 (lanczos.cpp:18-26) into column 0, raw; sigma_0 = 1/||v1||
  {
    const int gb = grid_for(ctx, lz->rows, 256);
    gauss_kernel<<<gb, 256, 0, st>>>(s0, s0p, lz->begin, lz->rows, lz->D.p, lz->part.p);
    gauss_norm_kernel<<<1, 32, 0, st>>>(lz->part.p, gb, lz->rankp.p);
    DHO2G_LAUNCH();
    ctx->allgather_f64(lz->rankp.p, lz->allp.p, 1, "all_reduce");
    lz_init_kernel<<<1, 32, 0, st>>>(lz->st.p, lz->allp.p, world, 1);
    DHO2G_LAUNCH();
  }

  if (lanczos_small_eligible(lz, op)) {  // small MLP operator: the m iterations as one persistent launch
    lanczos_small_run(lz, op);
    return;
  }
  const int nchunks = (int)(lz->ldd / kGsChunk);
  const size_t ngroups = lz->ldd / 4;
  const double* allp = world > 1 ? lz->allp.p : lz->rankp.p;
  const double* allb = world > 1 ? lz->allp.p : lz->rankp.p;

  for (size_t i = 0; i < m; ++i) {
    const int active = (int)i + 1;
    float* Di = lz->D.p + i * lz->ldd;
    float* Dn = lz->D.p + (i + 1) * lz->ldd;
    const float* vfull = Di;
    if (world > 1) {
      ctx->allgather_f32(Di, lz->vfull.p, lz->base);
      vfull = lz->vfull.p;
    }
    op->apply(vfull, &lz->st.p->sigma[i], lz->h.p, lz->begin, lz->rows, lz->base);
    const size_t smem1 = (size_t)kWarps * (active + 1 + (gram ? active : 0)) * sizeof(double);
    const size_t smem2 = (size_t)(2 * active + 1) * sizeof(double);
    const int gs_sms = ctx->gs_sm_cap > 0 ? std::min(ctx->gs_sm_cap, ctx->sm_count) : ctx->sm_count;
    const int g1 = one_wave_grid(gram ? gs_pass1_kernel<true> : gs_pass1_kernel<false>, kThreads, smem1, gs_sms,
                                 (size_t)nchunks);
    const int g2 = one_wave_grid(gs_pass2_kernel, kThreads, smem2, gs_sms, cdiv(ngroups / 128, kWarps));
    for (int pass = 0; pass < (lz->opts.reorth_safeguard ? 2 : 1); ++pass) {
      const float* hsrc = pass == 0 ? lz->h.p : Dn;
      // algorithmic bytes: active columns of D + h (pass 1); + h' write (pass 2)
      const double gsb = 4.0 * (double)lz->rows * (double)(active + 1);
      int ks = pass == 0 ? ctx->kt_begin() : -1;
      auto* k1 = pass == 0 && gram ? gs_pass1_kernel<true> : gs_pass1_kernel<false>;
      k1<<<g1, kThreads, smem1, st>>>(lz->D.p, lz->ldd, hsrc, active, nchunks, stride, lz->part.p, lz->rankp.p,
                                      lz->ticket.p, lz->st.p, pass, goff);
      DHO2G_LAUNCH();
      ctx->kt_end(ks, "gs_pass1", gsb);
      if (world > 1) ctx->allgather_f64(lz->rankp.p, lz->allp.p, stride, "all_reduce");
      ks = pass == 0 ? ctx->kt_begin() : -1;
      gs_pass2_kernel<<<g2, kThreads, smem2, st>>>(lz->D.p, lz->ldd, hsrc, Dn, active, ngroups, allp, world, stride,
                                                    lz->part.p, lz->rankp.p, lz->ticket.p + 1, lz->st.p, (int)i, pass,
                                                    gram, goff);
      DHO2G_LAUNCH();
      ctx->kt_end(ks, "gs_pass2", gsb + 4.0 * (double)lz->rows);
      if (world > 1) ctx->allgather_f64(lz->rankp.p, lz->allp.p, 1, "all_reduce");
      lz_decide_kernel<<<1, 32, 0, st>>>(lz->st.p, allb, world, world > 1 ? 1 : 1, (int)i, pass,
                                         lz->opts.reorth_safeguard, lz->opts.safeguard_ratio, lz->opts.breakdown_rtol);
      DHO2G_LAUNCH();
    }
  }
}

// launch = false: capture / instantiate only (done right after the first, eager refresh, so that the
// capture's host cost falls in that refresh rather than in a later one).
static bool lanczos_graph(dho2g_lanczos* lz, dho2g_op* op, uint64_t s0, bool launch = true) {
  dho2g_ctx* ctx = lz->ctx;
  cudaStream_t st = ctx->stream;
  // multi-rank: NCCL collectives are captured with the kernels (dho2g_test_collectives_graph); the in-process
  // fabric's / host communicator's host rendezvous cannot be
  if (!ctx->use_graphs || (ctx->world != 1 && (ctx->host_rendezvous() || !ctx->graphs_multirank)) || ctx->ktimers ||
      op->kind == 3 || lz->graph_failed)
    return false;
  lz->seed_dev.ensure(1);
  lz->seed_host.ensure(1);
  const bool valid = lz->gexec && lz->gop == op && lz->gm == lz->m && lz->ggen == g_graph_gen &&
                     lz->gflags == ctx->gemm_flags.p && lz->gflags2 == ctx->gemm_flags2.p;
  if (!valid) {
    if (!lz->seen_eager) return false;  // first refresh runs eagerly (allocates every buffer)
    if (lz->gexec) {
      cudaGraphExecDestroy(lz->gexec);
      lz->gexec = nullptr;
    }
    const unsigned long long gen0 = g_graph_gen;
    cudaGraph_t g = nullptr;
    if (cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
      cudaGetLastError();
      lz->graph_failed = true;
      return false;
    }
    bool ok = true;
    const unsigned long long l0 = g_launches;
    try {
      if (ctx->gemm_flags.p)
        DHO2G_CUDA(cudaMemsetAsync(ctx->gemm_flags.p, 0, ctx->gemm_flags.n * sizeof(unsigned), st));
      if (ctx->gemm_flags2.p)  // the side lane's split / stream-K flags (baked epochs too)
        DHO2G_CUDA(cudaMemsetAsync(ctx->gemm_flags2.p, 0, ctx->gemm_flags2.n * sizeof(unsigned), st));
      lanczos_enqueue(lz, op, 0, lz->seed_dev.p);
    } catch (...) {
      ok = false;
    }
    const cudaError_t ec = cudaStreamEndCapture(st, &g);
    if (!ok || ec != cudaSuccess || g == nullptr || g_graph_gen != gen0) {
      cudaGetLastError();
      if (g) cudaGraphDestroy(g);
      lz->graph_failed = true;
      return false;
    }
    const cudaError_t ei = cudaGraphInstantiate(&lz->gexec, g, 0);
    cudaGraphDestroy(g);
    if (ei != cudaSuccess) {
      cudaGetLastError();
      lz->gexec = nullptr;
      lz->graph_failed = true;
      return false;
    }
    lz->gop = op;
    lz->gm = lz->m;
    lz->ggen = g_graph_gen;
    lz->gflags = ctx->gemm_flags.p;
    lz->gflags2 = ctx->gemm_flags2.p;
    lz->glaunches = g_launches - l0;
    g_launches = l0;  // captured, not launched
    ctx->bump("lanczos_graph_captures", 1);
  }
  if (!launch) return true;
  lz->seed_host.p[0] = s0;
  DHO2G_CUDA(cudaMemcpyAsync(lz->seed_dev.p, lz->seed_host.p, sizeof(uint64_t), cudaMemcpyHostToDevice, st));
  DHO2G_CUDA(cudaGraphLaunch(lz->gexec, st));
  g_launches += lz->glaunches;  // the graph's kernel launches
  ctx->bump("lanczos_graph_launches", 1);
  return true;
}

void lanczos_run_into(dho2g_lanczos* lz, dho2g_op* op, uint64_t seed) {
  dho2g_ctx* ctx = lz->ctx;
  cudaStream_t st = ctx->stream;
  const size_t m = lz->m;
  if (ctx->world > 1) {
    // v1 is drawn from the shared seed on every rank; a mismatched seed would silently blend slices of
    // different vectors (dist_lanczos.cpp:47-52 checks the same with a hash of v1): compare the seeds
    lz->seed_chk.ensure(2 + 2 * (size_t)ctx->world);
    double mine[2] = {(double)(uint32_t)(seed >> 32), (double)(uint32_t)seed};
    DHO2G_CUDA(cudaMemcpyAsync(lz->seed_chk.p, mine, sizeof(mine), cudaMemcpyHostToDevice, st));
    ctx->allgather_f64(lz->seed_chk.p, lz->seed_chk.p + 2, 2, "hash_check");
    std::vector<double> all(2 * (size_t)ctx->world);
    DHO2G_CUDA(cudaMemcpyAsync(all.data(), lz->seed_chk.p + 2, all.size() * sizeof(double), cudaMemcpyDeviceToHost,
                               st));
    wait_stream(ctx, st);
    for (int r = 0; r < ctx->world; ++r)
      if (all[2 * r] != mine[0] || all[2 * r + 1] != mine[1])
        fail(DHO2G_DIVERGENCE, "lanczos_distributed: seed mismatch across ranks");
  }
  cudaEvent_t e0, e1;
  DHO2G_CUDA(cudaEventCreate(&e0));
  DHO2G_CUDA(cudaEventCreate(&e1));
  DHO2G_CUDA(cudaEventRecord(e0, st));
  const uint64_t s0 = seed * 0x9e3779b97f4a7c15ULL + 0x1234567ULL;
  bool eager = false;
  if (!lanczos_graph(lz, op, s0)) {
    lanczos_enqueue(lz, op, s0, nullptr);
    lz->seen_eager = eager = true;
  }
  DHO2G_CUDA(cudaEventRecord(e1, st));
  DHO2G_CUDA(cudaMemcpyAsync(&lz->host, lz->st.p, sizeof(LzDev), cudaMemcpyDeviceToHost, st));
  wait_stream(lz->ctx, st);
  float ms = 0.f;
  DHO2G_CUDA(cudaEventElapsedTime(&ms, e0, e1));
  lz->ms = ms;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  if (lz->host.nonfinite) fail(DHO2G_NUMERIC, "lanczos_distributed: hvp returned non-finite values");
  if (lz->host.stopped == 0) lz->host.iters = (int)m;
  if (ctx->hash_checks) {  // dist_lanczos.cpp:104 / :113, checked once for the whole B (no round trip per step)
    const size_t it = (size_t)lz->host.iters;
    if (!ranks_all_equal(ctx, tridiag_hash_host(lz->host.diag, lz->host.off, it)))
      fail(DHO2G_DIVERGENCE, "lanczos_distributed: B diverged across ranks (seed mismatch?)");
  }
  ctx->bump("lanczos_runs", 1);
  ctx->bump("lanczos_ms", ms);
  if (eager && !lz->gexec) {
    // pre-capture the next refresh from the host state a refresh starts in (operator weights reloaded)
    const bool wl = op->weights_loaded;
    op->weights_loaded = false;
    lanczos_graph(lz, op, s0, false);
    op->weights_loaded = wl || op->weights_loaded;
  }
}

void extract_ese_into(dho2g_ctx* ctx, dho2g_lanczos* lz, size_t k, size_t l, dho2g_ese* ese) {
  cudaStream_t st = ctx->stream;
  const int me = lz->host.iters;
  ese->ctx = ctx;
  ese->n = lz->n;
  ese->rows = lz->rows;
  ese->begin = lz->begin;
  ese->end = lz->end;
  ese->ldv = lz->ldd;
  if (k + l == 0) {
    ese->r = 0;
    return;
  }
  if (me < 1) fail(DHO2G_ARGUMENT, "extract_ese_distributed: empty Lanczos state");
  if (k + l > (size_t)me) fail(DHO2G_ARGUMENT, "extract_ese_distributed: k+l exceeds the filled block");
  if (ctx->hash_checks && !ranks_all_equal(ctx, tridiag_hash_host(lz->host.diag, lz->host.off, (size_t)me)))
    fail(DHO2G_DIVERGENCE, "extract_ese_distributed: B differs across ranks");  // dist_lanczos.cpp:134
  const int r = (int)(k + l);
  ese->r = r;
  // scratch persists in the Lanczos state (no allocation, hence no implicit device sync, per refresh)
  DevBuf<double>& Z = lz->xZ;
  DevBuf<float>& U = lz->xU;
  DevBuf<double>& evall = lz->xev;
  DevBuf<int>& status = lz->xstatus;
  Z.ensure((size_t)me * me);
  U.ensure((size_t)me * r);
  evall.ensure(me);
  status.ensure(1);
  ese->ev_dev.ensure(r);
  const int threads = (int)std::min<size_t>(1024, round_up((size_t)me, 32));
  const int kx = ctx->kt_begin();
  const int kq = ctx->kt_begin();
  if (ctx->tql2_split) {
    // log capacity: QL takes ~1-2 sweeps of <= n - 1 - l rotations per l, ~n^2 rotations in all; 2 n^2 is
    // kept (the reference's limit, 60 sweeps per l, would need 30 n (n - 1): 500 MB at m = 1023). A log that
    // fills up makes the kernel stop with status 2 and the single-CTA kernel redoes the eigensolve.
    const size_t cap = ctx->tql2_log_cap > 0 ? (size_t)ctx->tql2_log_cap : (size_t)2 * me * me + 4096;
    lz->xrot.ensure(cap);
    lz->xsweep.ensure((size_t)60 * me + 1);
    lz->xnsweep.ensure(4);
    lz->xd.ensure(me);
    DHO2G_CUDA(cudaMemsetAsync(lz->xnsweep.p, 0, 4 * sizeof(int), st));
    const int T = me <= 800 ? 32 : 16;  // consumer: n * T * 8 bytes of slots + n * 16 bytes of staging
    const size_t sp = std::max((size_t)me * T * sizeof(double) + (size_t)me * sizeof(double2),
                               (size_t)me * 2 * sizeof(double));
    if (sp > 48 * 1024)
      DHO2G_CUDA(cudaFuncSetAttribute(tql2_pipe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sp));
    const int k1 = ctx->kt_begin();
    tql2_pipe_kernel<<<(unsigned)(1 + cdiv((size_t)me, (size_t)T)), 32, sp, st>>>(
        lz->st.p, me, T, lz->xrot.p, (long long)cap, lz->xsweep.p, lz->xnsweep.p, lz->xd.p, status.p, Z.p);
    DHO2G_LAUNCH();
    ctx->kt_end(k1, "eig.pipe", 0.0);
    const int k3 = ctx->kt_begin();
    tql2_select_kernel<<<1, threads, (size_t)me * (sizeof(double) + sizeof(int)), st>>>(
        lz->st.p, me, (int)k, (int)l, lz->xd.p, Z.p, U.p, ese->ev_dev.p, evall.p, status.p);
    DHO2G_LAUNCH();
    ctx->kt_end(k3, "eig.select", 0.0);
  } else {
    const size_t smem = (size_t)me * 4 * sizeof(double) + (size_t)me * sizeof(int);
    if (smem > 48 * 1024)
      DHO2G_CUDA(cudaFuncSetAttribute(tql2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    tql2_kernel<<<1, threads, smem, st>>>(lz->st.p, me, (int)k, (int)l, Z.p, U.p, ese->ev_dev.p, evall.p, status.p);
    DHO2G_LAUNCH();
  }
  ctx->kt_end(kq, "extract.tql2", 0.0);
  ese->V.ensure(ese->ldv * r);  // padded rows stay zero (Ritz writes rows < rows only)
  ctx->meter("vhat_partial", (int64_t)(lz->rows * r));  // V_hat stays row-sharded: no "vhat" assembly
  const int kr = ctx->kt_begin();
  if (ctx->ritz_tc && ritz_tc_supported(me, r)) {
    ritz_tc(ctx, lz->D.p, lz->ldd, me, U.p, &lz->st.p->sigma[0], r, ese->V.p, ese->ldv, lz->rows, lz->xUs);
  } else {
    for (int c0 = 0; c0 < r; c0 += RC) {
      const size_t sm = (size_t)me * RC * sizeof(float);
      if (sm > 48 * 1024)
        DHO2G_CUDA(cudaFuncSetAttribute(ritz_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
      ritz_kernel<<<one_wave_grid(ritz_kernel, 256, sm, ctx->sm_count, cdiv(cdiv(lz->rows, 2), 256)), 256, sm, st>>>(
          lz->D.p, lz->ldd, me, U.p, r, c0, ese->V.p, ese->ldv, lz->rows);
      DHO2G_LAUNCH();
    }
  }
  ctx->kt_end(kr, "extract.ritz", 4.0 * (double)lz->rows * (double)(me + r));
  DevBuf<double>& am = lz->xam;
  DevBuf<double>& amall = lz->xamall;
  am.ensure((size_t)3 * r);
  amall.ensure((size_t)3 * r * ctx->world);
  {
    const int nblk = (int)std::max<size_t>(1, std::min<size_t>(cdiv(lz->rows, 4 * kArgThreads), 256));
    const size_t seg = cdiv(std::max<size_t>(lz->rows, 1), (size_t)nblk);
    DevBuf<double>& part = lz->xpart;
    part.ensure((size_t)3 * r * nblk);
    const int ka = ctx->kt_begin();
    col_argmax_kernel<<<dim3(nblk, r), kArgThreads, 0, st>>>(ese->V.p, ese->ldv, lz->rows, lz->begin, seg, part.p);
    col_argmax_final_kernel<<<r, 32, 0, st>>>(part.p, nblk, am.p);
    DHO2G_LAUNCH();
    ctx->kt_end(ka, "extract.argmax", 4.0 * (double)lz->rows * (double)r);
  }
  // tql2 + Ritz (reads D[:, :m_eff], writes V_hat) + argmax (reads V_hat): algorithmic bytes
  ctx->kt_end(kx, "extract_ese", 4.0 * (double)lz->rows * (double)(me + 2 * r));
  ctx->allgather_f64(am.p, amall.p, (size_t)3 * r);
  std::vector<double> h_am((size_t)3 * r * ctx->world);
  int h_status = 0;
  ese->eigvals.resize(r);
  DHO2G_CUDA(cudaMemcpyAsync(h_am.data(), amall.p, h_am.size() * sizeof(double), cudaMemcpyDeviceToHost, st));
  DHO2G_CUDA(cudaMemcpyAsync(ese->eigvals.data(), ese->ev_dev.p, r * sizeof(double), cudaMemcpyDeviceToHost, st));
  DHO2G_CUDA(cudaMemcpyAsync(&h_status, status.p, sizeof(int), cudaMemcpyDeviceToHost, st));
  wait_stream(lz->ctx, st);
  if (h_status == 2 && ctx->tql2_split) {  // rotation log full: the single-CTA eigensolve (bit-identical)
    ctx->bump("tql2_log_overflows", 1);
    ctx->tql2_split = 0;
    try {
      extract_ese_into(ctx, lz, k, l, ese);
    } catch (...) {
      ctx->tql2_split = 1;
      throw;
    }
    ctx->tql2_split = 1;
    return;
  }
  if (h_status) fail(DHO2G_NUMERIC, "tridiag_eig: QL iteration did not converge");
  ese->sign.assign(r, 1.f);
  for (int c = 0; c < r; ++c) {
    double best = -1.0, bidx = 0.0, bval = 0.0;
    for (int w = 0; w < ctx->world; ++w) {
      const double* p = h_am.data() + (size_t)w * 3 * r + 3 * c;
      if (p[0] > best || (p[0] == best && p[1] < bidx)) {
        best = p[0];
        bidx = p[1];
        bval = p[2];
      }
    }
    ese->sign[c] = bval < 0.0 ? -1.f : 1.f;
  }
}

}  // namespace dho2g
