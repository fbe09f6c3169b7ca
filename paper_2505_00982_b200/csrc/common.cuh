// Shared internals of libdho2gpu.so: error plumbing, device buffers, small device helpers.
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <nccl.h>

#include <cstdint>
#include <cstdio>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/dho2gpu.h"

namespace dho2g {

// Internal exception carrying a dho2g_status; converted at the C boundary (capi.cu).
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] inline void fail(int code, const std::string& msg) { throw Error(code, msg); }

#define DHO2G_CUDA(expr)                                                                        \
  do {                                                                                          \
    cudaError_t e__ = (expr);                                                                   \
    if (e__ != cudaSuccess)                                                                     \
      ::dho2g::fail(DHO2G_CUDA, std::string(#expr) + ": " + cudaGetErrorString(e__) + " @" +    \
                                    __FILE__ + ":" + std::to_string(__LINE__));                 \
  } while (0)

// NCCL is resolved at run time (dlopen of libnccl.so.2) so the library never pins a NCCL build:
// inside a torch process it binds to the NCCL torch already loaded.
struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*);
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int);
  ncclResult_t (*CommInitRankConfig)(ncclComm_t*, int, ncclUniqueId, int, ncclConfig_t*);
  ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t*);
  ncclResult_t (*CommAbort)(ncclComm_t);
  ncclResult_t (*CommDestroy)(ncclComm_t);
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t);
  ncclResult_t (*ReduceScatter)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t);
  const char* (*GetErrorString)(ncclResult_t);
};
const NcclApi& nccl();

#define DHO2G_NCCLCHK(expr)                                                                    \
  do {                                                                                         \
    ncclResult_t r__ = (expr);                                                                 \
    if (r__ != ncclSuccess)                                                                    \
      ::dho2g::fail(DHO2G_NCCL, std::string(#expr) + ": " + ::dho2g::nccl().GetErrorString(r__)); \
  } while (0)

// Every kernel launch of the library goes through DHO2G_LAUNCH(): counts it (bench evidence of
// device work, "gpu_launches") and surfaces launch errors.
extern unsigned long long g_launches;
#define DHO2G_LAUNCH()              \
  do {                              \
    ++::dho2g::g_launches;          \
    DHO2G_CUDA(cudaGetLastError()); \
  } while (0)

__host__ __device__ inline size_t round_up(size_t x, size_t m) { return (x + m - 1) / m * m; }
__host__ __device__ inline size_t cdiv(size_t a, size_t b) { return (a + b - 1) / b; }

// Incremented when a buffer that a captured refresh graph may reference is (re)allocated (ensure_g,
// MLP batch buffers, Lanczos state): captured CUDA graphs hold raw pointers and are rebuilt on change.
extern unsigned long long g_graph_gen;

// RAII device allocation (cudaMalloc, zero-initialised).
template <typename T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  DevBuf() = default;
  explicit DevBuf(size_t count) { alloc(count); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p(o.p), n(o.n) { o.p = nullptr; o.n = 0; }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) { release(); p = o.p; n = o.n; o.p = nullptr; o.n = 0; }
    return *this;
  }
  ~DevBuf() { release(); }
  void alloc(size_t count) {
    release();
    n = count;
    if (count == 0) return;
    DHO2G_CUDA(cudaMalloc(&p, count * sizeof(T)));
    // cudaMemset runs on the legacy stream, which does not order with the library's non-blocking
    // stream: complete it before any kernel can touch the buffer.
    DHO2G_CUDA(cudaMemset(p, 0, count * sizeof(T)));
    DHO2G_CUDA(cudaStreamSynchronize(0));
  }
  void ensure(size_t count) { if (count > n) alloc(count); }
  void ensure_g(size_t count) {  // ensure() for buffers a captured CUDA graph may hold pointers to
    if (count > n) {
      alloc(count);
      ++g_graph_gen;
    }
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
  T* get() const { return p; }
};

// Pinned host allocation.
template <typename T>
struct HostBuf {
  T* p = nullptr;
  size_t n = 0;
  HostBuf() = default;
  HostBuf(const HostBuf&) = delete;
  HostBuf& operator=(const HostBuf&) = delete;
  ~HostBuf() { if (p) cudaFreeHost(p); }
  void ensure(size_t count) {
    if (count <= n) return;
    if (p) cudaFreeHost(p);
    p = nullptr;
    DHO2G_CUDA(cudaHostAlloc(&p, count * sizeof(T), cudaHostAllocPortable | cudaHostAllocMapped));
    n = count;
  }
};

typedef __nv_bfloat16 bf16;

// Grid for a grid-stride (persistent-style) kernel: exactly one wave of resident CTAs, capped by
// the work. A second partial wave of such a kernel idles most SMs for a whole CTA lifetime.
template <typename Kernel>
inline int one_wave_grid(Kernel kernel, int threads, size_t smem, int sm_count, size_t work_blocks) {
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, smem) != cudaSuccess || per_sm < 1)
    per_sm = 1;
  const size_t cap = (size_t)per_sm * (size_t)sm_count;
  return (int)(work_blocks < 1 ? 1 : (work_blocks < cap ? work_blocks : cap));
}

// ----------------------------------------------------------------------------- device helpers
__device__ __forceinline__ void split_bf16(float x, bf16& hi, bf16& lo) {
  hi = __float2bfloat16_rn(x);
  lo = __float2bfloat16_rn(x - __bfloat162float(hi));
}
// Scaled-fp16 pair: x s = hi + lo with 11 + 11 significant bits (vs 8 + 8 for bf16) for |x s| in
// [2^-3, 2^15); s is a power of two chosen from max |x| (pow2_scale), so the scaling is exact and
// elements far below the maximum lose bits only at the 2^-25 / s absolute level. Stored in the same
// 16-bit buffers as the bf16 pairs.
__device__ __forceinline__ void split_f16(float x, float s, bf16& hi, bf16& lo) {
  const float y = x * s;
  const __half h = __float2half_rn(y);
  const __half l = __float2half_rn(y - __half2float(h));
  hi = __ushort_as_bfloat16(__half_as_ushort(h));
  lo = __ushort_as_bfloat16(__half_as_ushort(l));
}
__device__ __forceinline__ float f16_bits_to_float(bf16 x) {
  return __half2float(__ushort_as_half(__bfloat16_as_ushort(x)));
}
// Largest power of two s with mx * s < 2^14 (a 4x margin below the fp16 maximum); 1 for mx == 0.
__host__ __device__ __forceinline__ float pow2_scale(float mx) {
  if (!(mx > 0.f)) return 1.f;
  int e;
  frexpf(mx, &e);  // mx < 2^e
  e = 14 - e;
  e = e > 100 ? 100 : (e < -100 ? -100 : e);
  return ldexpf(1.f, e);
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
// Deterministic fold of n strided partials by one warp: lane l adds x[b * stride] for b = l, l + 32, ... in
// order, then the fixed xor-butterfly; every lane returns the total. The order depends only on n, never
// on timing, and n / 32 loads per lane are in flight instead of one thread's n-long dependent chain.
__device__ __forceinline__ double warp_fold(const double* x, int n, size_t stride) {
  const int lane = threadIdx.x & 31;
  double t = 0.0;
#pragma unroll 4
  for (int b = lane; b < n; b += 32) t += __ldcg(x + (size_t)b * stride);
  return warp_sum(t);
}
__device__ __forceinline__ float warp_sumf(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Deterministic block reduction of one double per thread (fixed tree order). Result valid in
// thread 0. `sh` needs blockDim.x/32 doubles.
__device__ __forceinline__ double block_sum(double v, double* sh) {
  v = warp_sum(v);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) sh[wid] = v;
  __syncthreads();
  double r = 0.0;
  if (threadIdx.x == 0)
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) r += sh[i];
  return r;
}

// Butterfly reduction of K per-lane values at once: at each of the first log2(K) levels every lane
// keeps half of its values and trades the other half with its partner, so K = 8 values take 9 fp64
// shuffles (4 + 2 + 1 + 2) instead of 40. Lane l ends up holding value
// sum_L ((l >> L) & 1) * (K >> (L + 1)), for l < K.
template <int K>
__device__ __forceinline__ double butterfly_sum(double (&v)[K], int lane) {
  int n = K, level = 0;
#pragma unroll
  for (; n > 1; n >>= 1, ++level) {
    const bool b = (lane >> level) & 1;
#pragma unroll
    for (int i = 0; i < n / 2; ++i) {
      const double send = b ? v[i] : v[i + n / 2];
      const double keep = b ? v[i + n / 2] : v[i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, 1 << level);
    }
  }
  double u = v[0];
#pragma unroll
  for (; level < 5; ++level) u += __shfl_xor_sync(0xffffffffu, u, 1 << level);
  return u;
}
template <int K>
__device__ __forceinline__ int butterfly_index(int lane) {
  int idx = 0;
#pragma unroll
  for (int L = 0; (K >> (L + 1)) > 0; ++L) idx += ((lane >> L) & 1) * (K >> (L + 1));
  return idx;
}

}  // namespace dho2g
