// Cooperative-grid helpers shared by the one-launch kernels (mlp_small.cu, update.cu): a grid barrier that
// needs no per-launch initialisation and a fixed-order reduction of per-CTA partial rows.
#pragma once
#include "common.cuh"

namespace dho2g {

// Grid barrier on kBarShards monotonically increasing 64-bit arrival counters, 128 bytes apart (CTA b arrives
// on counter b mod kBarShards, so the arrivals do not serialise on one L2 line; each shard then has
// cnt_l = ceil((nb - l) / kBarShards) arrivals per barrier). Counters are never reset: a launch starts with
// every counter at K0 cnt_l for the same K0 (the grid size is fixed between resets), which the first barrier
// of a launch learns from its own ticket (atom.release); later arrivals only add (red.release, no round trip).
// Lanes 0..kBarShards-1 of warp 0 each poll one shard (relaxed) up to (K0 + k + 1) cnt_l, then an acquire fence.
// st[0] = K0 + k (the completed-barrier count of this launch, 0 before the first barrier: K0 unknown).
constexpr int kBarShards = 8;
constexpr int kBarStride = 16;  // 128 bytes
__device__ __forceinline__ void grid_barrier(unsigned long long* bar, unsigned nb, unsigned long long* st) {
  __syncthreads();
  if (threadIdx.x < 32) {
    const unsigned lane = threadIdx.x;
    const unsigned j = blockIdx.x % kBarShards;
    const unsigned long long cj = (nb - j + kBarShards - 1) / kBarShards;
    unsigned long long k;
    if (lane == 0) {
      if (*st == 0ull) {
        unsigned long long t;
        asm volatile("atom.add.release.gpu.global.u64 %0, [%1], 1;" : "=l"(t) : "l"(bar + j * kBarStride) : "memory");
        k = t / cj;  // K0
      } else {
        asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(bar + j * kBarStride) : "memory");
        k = *st;
      }
      *st = k + 1;
    }
    k = __shfl_sync(0xffffffffu, k, 0);
    if (lane < kBarShards && lane < nb) {
      const unsigned long long cl = (nb - lane + kBarShards - 1) / kBarShards;
      const unsigned long long target = (k + 1) * cl;
      unsigned long long v;
      do {
        asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(bar + lane * kBarStride) : "memory");
      } while (v < target);
    }
    __syncwarp();
    if (lane == 0) asm volatile("fence.acq_rel.gpu;" ::: "memory");
  }
  __syncthreads();
}

// Every CTA: out[e] = sum over the ngs partial rows. Warp w adds the rows of its block of CTAs (CTA order,
// lanes over values: coalesced), then the warp sums are added in warp order: a fixed order, identical in every
// CTA.
template <int kThr>
__device__ void reduce_rows(const double* part, int ngs, int stride, int rowlen, double* sacc, double* out) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = kThr / 32;
  const int per = (ngs + nw - 1) / nw, q0 = warp * per, q1 = min(ngs, q0 + per);
  for (int e0 = 0; e0 < rowlen; e0 += 32) {
    const int e = e0 + lane;
    double t = 0.0;
    if (e < rowlen) {
      for (int q = q0; q < q1; q += 20) {  // (one block for up to 160 CTAs: every load in flight)
        double vals[20];
#pragma unroll
        for (int u = 0; u < 20; ++u) vals[u] = q + u < q1 ? __ldcg(part + (size_t)(q + u) * stride + e) : 0.0;
#pragma unroll
        for (int u = 0; u < 20; ++u) t += vals[u];
      }
      sacc[warp * rowlen + e] = t;
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < rowlen; e += kThr) {
    double t = 0.0;
    for (int w = 0; w < nw; ++w) t += sacc[w * rowlen + e];
    out[e] = t;
  }
  __syncthreads();
}

}  // namespace dho2g
