// Host-side bookkeeping that must be bit-exact with the reference (rng, shards, budget,
// permutations, sample/curvature indices) and the context's collectives.
#include <dlfcn.h>

#include <algorithm>
#include <cmath>
#include <chrono>
#include <condition_variable>
#include <mutex>
#include <numeric>
#include <thread>

#include <cstring>

#include "internal.h"

namespace dho2g {
unsigned long long g_graph_gen = 0;
}  // namespace dho2g

namespace dho2g {

unsigned long long g_launches = 0;

// rng.hpp:18-23 SplitMix64
uint64_t Rng::next_u64() {
  uint64_t z = (state += 0x9e3779b97f4a7c15ULL);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
// rng.hpp:26
double Rng::uniform() { return static_cast<double>(next_u64() >> 11) * 0x1.0p-53; }
// rng.hpp:29-35
uint64_t Rng::uniform_below(uint64_t bound) {
  const uint64_t threshold = (0 - bound) % bound;
  for (;;) {
    const uint64_t r = next_u64();
    if (r >= threshold) return r % bound;
  }
}
// rng.hpp:37-50
double Rng::normal() {
  if (have_spare) {
    have_spare = false;
    return spare;
  }
  const double u1 = (static_cast<double>(next_u64() >> 11) + 1.0) * 0x1.0p-53;
  const double u2 = uniform();
  const double radius = std::sqrt(-2.0 * std::log(u1));
  const double angle = 2.0 * 3.141592653589793 * u2;
  spare = radius * std::sin(angle);
  have_spare = true;
  return radius * std::cos(angle);
}

// QuadraticOracle rotation (oracle.cpp:241-257): Rng(seed*phi) normals filled column-major, then
// per column two modified Gram-Schmidt passes against the earlier columns and a normalisation.
// Operator construction (setup, O(n^3) like the reference's "desk-scale" constructor), not a
// per-iteration cost: every apply_h afterwards runs on the device.
bool quadratic_rotation(size_t n, uint64_t rotation_seed, double* Q) {
  Rng rng(rotation_seed * 0x9e3779b97f4a7c15ULL);
  for (size_t i = 0; i < n * n; ++i) Q[i] = rng.normal();
  for (size_t j = 0; j < n; ++j) {
    double* col = Q + j * n;
    for (int pass = 0; pass < 2; ++pass)
      for (size_t i = 0; i < j; ++i) {
        const double* qi = Q + i * n;
        double c = 0.0;
        for (size_t t = 0; t < n; ++t) c += qi[t] * col[t];
        for (size_t t = 0; t < n; ++t) col[t] += -c * qi[t];
      }
    double nn = 0.0;
    for (size_t t = 0; t < n; ++t) nn += col[t] * col[t];
    const double nrm = std::sqrt(nn);
    if (nrm < 1e-12) return false;
    const double inv = 1.0 / nrm;
    for (size_t t = 0; t < n; ++t) col[t] *= inv;
  }
  return true;
}

// rng.hpp:56-62 Fisher-Yates over iota
void shuffle_iota(uint64_t seed, size_t n, uint64_t* out) {
  for (size_t i = 0; i < n; ++i) out[i] = i;
  Rng r(seed);
  for (size_t i = n; i > 1; --i) {
    const size_t j = static_cast<size_t>(r.uniform_below(i));
    std::swap(out[i - 1], out[j]);
  }
}

const NcclApi& nccl() {
  static NcclApi api = [] {
    NcclApi a{};
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) fail(DHO2G_NCCL, std::string("cannot load libnccl.so.2: ") + dlerror());
    auto sym = [&](const char* n) {
      void* p = dlsym(h, n);
      if (!p) fail(DHO2G_NCCL, std::string("libnccl.so.2 lacks ") + n);
      return p;
    };
    a.GetUniqueId = reinterpret_cast<decltype(a.GetUniqueId)>(sym("ncclGetUniqueId"));
    a.CommInitRank = reinterpret_cast<decltype(a.CommInitRank)>(sym("ncclCommInitRank"));
    a.CommDestroy = reinterpret_cast<decltype(a.CommDestroy)>(sym("ncclCommDestroy"));
    a.CommInitRankConfig = reinterpret_cast<decltype(a.CommInitRankConfig)>(sym("ncclCommInitRankConfig"));
    a.CommGetAsyncError = reinterpret_cast<decltype(a.CommGetAsyncError)>(sym("ncclCommGetAsyncError"));
    a.CommAbort = reinterpret_cast<decltype(a.CommAbort)>(sym("ncclCommAbort"));
    a.AllGather = reinterpret_cast<decltype(a.AllGather)>(sym("ncclAllGather"));
    a.ReduceScatter = reinterpret_cast<decltype(a.ReduceScatter)>(sym("ncclReduceScatter"));
    a.GetErrorString = reinterpret_cast<decltype(a.GetErrorString)>(sym("ncclGetErrorString"));
    return a;
  }();
  return api;
}

// collectives.cpp:10-20
void shard_range(size_t n, int world, int rank, size_t* begin, size_t* end) {
  if (world < 1) fail(DHO2G_ARGUMENT, "Shard: world_size must be >= 1");
  if (rank < 0 || rank >= world) fail(DHO2G_ARGUMENT, "Shard: rank out of range");
  const size_t base = (n + static_cast<size_t>(world) - 1) / static_cast<size_t>(world);
  *begin = std::min(base * static_cast<size_t>(rank), n);
  *end = std::min(*begin + base, n);
}

// lanczos.cpp:10-16
size_t lanczos_budget(size_t k, size_t l, size_t n) {
  if (n < 1) fail(DHO2G_ARGUMENT, "lanczos_budget: n must be >= 1");
  if (k + l < 1) fail(DHO2G_ARGUMENT, "lanczos_budget: k+l must be >= 1");
  if (k + l > n) fail(DHO2G_ARGUMENT, "lanczos_budget: k+l exceeds the dimension");
  const auto log_term = static_cast<size_t>(std::ceil(2.0 * std::log(static_cast<double>(n))));
  return std::min(n, std::max(4 * (k + l), log_term));
}


}  // namespace dho2g

// ------------------------------------------------------------------------- context collectives
void dho2g_ctx::sync() { dho2g::wait_stream(this, stream); }
void dho2g_ctx::check_usable() const {
  if (failed)
    dho2g::fail(DHO2G_NCCL, "context unusable after a failed collective (" + failed_msg +
                                "); create a new context and communicator");
}

namespace dho2g {
// Failure detection (the reference's DeadlockError, collectives.cpp:257-262): with a communicator,
// host waits poll the stream and NCCL's asynchronous error state instead of blocking, so a rank that
// never arrives (or a failed peer) surfaces as DEADLOCK / NCCL after ctx->nccl_timeout_s instead of
// a hang; the communicator is aborted first (its kernels are released) and the context is marked failed
// (it does not go on as a single rank with the failed group's shards).
static void nccl_give_up(dho2g_ctx* ctx, int code, const std::string& msg) {
  if (ctx->comm) nccl().CommAbort(ctx->comm);
  ctx->comm = nullptr;
  ctx->failed = true;  // every later call on this context raises (dho2g_ctx::check_usable)
  ctx->failed_msg = msg;
  fail(code, msg);
}

static void nccl_poll(dho2g_ctx* ctx, const char* what, std::chrono::steady_clock::time_point t0, int spin) {
  ncclResult_t ae = ncclSuccess;
  nccl().CommGetAsyncError(ctx->comm, &ae);
  if (ae != ncclSuccess && ae != ncclInProgress)
    nccl_give_up(ctx, DHO2G_NCCL, std::string(what) + ": " + nccl().GetErrorString(ae));
  const double el = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  if (el > ctx->nccl_timeout_s)
    nccl_give_up(ctx, DHO2G_DEADLOCK, std::string("collective '") + what + "' timed out on rank " +
                                          std::to_string(ctx->rank) + ": a rank is missing from the round");
  if (spin > 2000) std::this_thread::sleep_for(std::chrono::microseconds(50));
  else std::this_thread::yield();
}

void nccl_settle(dho2g_ctx* ctx, const char* what) {
  const auto t0 = std::chrono::steady_clock::now();
  for (int spin = 0;; ++spin) {
    ncclResult_t ae = ncclSuccess;
    nccl().CommGetAsyncError(ctx->comm, &ae);
    if (ae == ncclSuccess) return;
    nccl_poll(ctx, what, t0, spin);
  }
}

void nccl_call(dho2g_ctx* ctx, ncclResult_t r, const char* what) {
  if (r == ncclSuccess) return;
  if (r == ncclInProgress) return nccl_settle(ctx, what);  // non-blocking communicator
  nccl_give_up(ctx, DHO2G_NCCL, std::string(what) + ": " + nccl().GetErrorString(r));
}

void wait_stream(dho2g_ctx* ctx, cudaStream_t s) {
  if (!ctx->comm) {
    DHO2G_CUDA(cudaStreamSynchronize(s));
    return;
  }
  const auto t0 = std::chrono::steady_clock::now();
  for (int spin = 0;; ++spin) {
    const cudaError_t e = cudaStreamQuery(s);
    if (e == cudaSuccess) return;
    if (e != cudaErrorNotReady) DHO2G_CUDA(e);
    nccl_poll(ctx, "stream wait", t0, spin);
  }
}
}  // namespace dho2g

int dho2g_ctx::kt_begin() {
  if (!ktimers) return -1;
  cudaEvent_t a, b;
  if (kpool.size() >= 2) {
    a = kpool.back(); kpool.pop_back();
    b = kpool.back(); kpool.pop_back();
  } else {
    DHO2G_CUDA(cudaEventCreate(&a));
    DHO2G_CUDA(cudaEventCreate(&b));
  }
  DHO2G_CUDA(cudaEventRecord(a, stream));
  const int id = knext++;
  kpend[id] = {std::string(), a, b, 0.0, false};
  return id;
}

void dho2g_ctx::kt_end(int slot, const char* name, double work) {
  if (slot < 0) return;
  auto it = kpend.find(slot);
  if (it == kpend.end()) return;
  KPending& p = it->second;
  p.name = name;
  p.work = work;
  p.ended = true;
  DHO2G_CUDA(cudaEventRecord(p.b, stream));
  if (kpend.size() > 4096) kt_flush();
}

void dho2g_ctx::kt_flush() {
  if (kpend.empty()) return;
  DHO2G_CUDA(cudaStreamSynchronize(stream));
  for (auto it = kpend.begin(); it != kpend.end();) {
    KPending& p = it->second;
    if (!p.ended) {  // still open (an enclosing phase timer): keep
      ++it;
      continue;
    }
    float ms = 0.f;
    DHO2G_CUDA(cudaEventElapsedTime(&ms, p.a, p.b));
    KStat& k = kstats[p.name];
    k.ms += ms;
    k.count += 1;
    k.work += p.work;
    kpool.push_back(p.a);
    kpool.push_back(p.b);
    it = kpend.erase(it);
  }
}

// ------------------------------------------------------------------ in-process fabric (test backend)
// Ranks are contexts on one GPU, each driven by its own host thread. A collective is: record "ready" on
// the caller's stream, rendezvous (host), copy / reduce every rank's deposit on the caller's stream after
// waiting for the depositor's "ready" event, record "done", rendezvous, and make the caller's stream wait
// for every rank's "done" (so no rank overwrites a send buffer a peer still reads). Only host threads and
// stream events synchronise: no kernel waits on another rank.

namespace {
__global__ void fabric_sum_kernel(const float* __restrict__ parts, float* __restrict__ out, size_t count, int world) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < count; i += (size_t)gridDim.x * blockDim.x) {
    float s = parts[i];
    for (int r = 1; r < world; ++r) s += parts[(size_t)r * count + i];  // ascending rank order
    out[i] = s;
  }
}
}  // namespace

// kind 0: all-gather (recv = world x count, rank q's block from q); kind 1: reduce-scatter of float
// (recv = count, sum over ranks of their block `rank`)
static void fabric_collective(dho2g_ctx* ctx, const void* send, void* recv, size_t count, size_t elem, int kind) {
  dho2g_fabric* f = ctx->fabric;
  const int W = f->world, r = ctx->rank;
  DHO2G_CUDA(cudaEventRecord(f->ready[r], ctx->stream));
  f->send[r] = send;
  f->barrier();
  if (kind == 0) {
    for (int q = 0; q < W; ++q) {
      DHO2G_CUDA(cudaStreamWaitEvent(ctx->stream, f->ready[q], 0));
      char* dst = static_cast<char*>(recv) + (size_t)q * count * elem;
      if (dst != f->send[q])
        DHO2G_CUDA(cudaMemcpyAsync(dst, f->send[q], count * elem, cudaMemcpyDeviceToDevice, ctx->stream));
    }
  } else {
    ctx->fabric_scratch.ensure((size_t)W * count);
    for (int q = 0; q < W; ++q) {
      DHO2G_CUDA(cudaStreamWaitEvent(ctx->stream, f->ready[q], 0));
      DHO2G_CUDA(cudaMemcpyAsync(ctx->fabric_scratch.p + (size_t)q * count,
                                 static_cast<const float*>(f->send[q]) + (size_t)r * count, count * sizeof(float),
                                 cudaMemcpyDeviceToDevice, ctx->stream));
    }
    fabric_sum_kernel<<<(unsigned)std::min<size_t>(dho2g::cdiv(count, 256), 1184), 256, 0, ctx->stream>>>(
        ctx->fabric_scratch.p, static_cast<float*>(recv), count, W);
    DHO2G_LAUNCH();
  }
  DHO2G_CUDA(cudaEventRecord(f->done[r], ctx->stream));
  f->barrier();
  for (int q = 0; q < W; ++q) DHO2G_CUDA(cudaStreamWaitEvent(ctx->stream, f->done[q], 0));
  f->barrier();  // every rank has issued its waits before any "done" / "ready" is recorded again
}

// Host-transport communicator: send -> pinned host, the caller's all-gather, pinned host -> recv (all-gather) or
// the ascending-rank sum of this rank's slices (reduce-scatter, fabric_sum_kernel).
static void host_collective(dho2g_ctx* ctx, const void* send, void* recv, size_t count, size_t elem, int kind) {
  const int W = ctx->world, r = ctx->rank;
  const size_t bytes = count * elem * (kind == 0 ? 1 : (size_t)W);  // reduce-scatter: the full-length partial
  ctx->host_ag_buf.ensure(bytes * (size_t)(W + 1));
  char* hs = ctx->host_ag_buf.p;
  char* hr = hs + bytes;
  DHO2G_CUDA(cudaMemcpyAsync(hs, send, bytes, cudaMemcpyDeviceToHost, ctx->stream));
  dho2g::wait_stream(ctx, ctx->stream);
  if (ctx->host_ag(ctx->host_ag_user, hs, hr, bytes) != 0) {
    ctx->failed = true;
    ctx->failed_msg = "host communicator: all-gather callback failed";
    dho2g::fail(DHO2G_NCCL, ctx->failed_msg);
  }
  if (kind == 0) {
    DHO2G_CUDA(cudaMemcpyAsync(recv, hr, bytes * W, cudaMemcpyHostToDevice, ctx->stream));
  } else {
    ctx->fabric_scratch.ensure((size_t)W * count);
    for (int q = 0; q < W; ++q)
      DHO2G_CUDA(cudaMemcpyAsync(ctx->fabric_scratch.p + (size_t)q * count, hr + (size_t)q * bytes + (size_t)r * count * 4,
                                 count * sizeof(float), cudaMemcpyHostToDevice, ctx->stream));
    fabric_sum_kernel<<<(unsigned)std::min<size_t>(dho2g::cdiv(count, 256), 1184), 256, 0, ctx->stream>>>(
        ctx->fabric_scratch.p, static_cast<float*>(recv), count, W);
    DHO2G_LAUNCH();
  }
  dho2g::wait_stream(ctx, ctx->stream);  // the staging buffer is reused by the next collective
}

namespace dho2g {
uint64_t tridiag_hash_host(const double* diag, const double* off, size_t upto) {
  uint64_t h = 0xcbf29ce484222325ULL;
  auto mix = [&h](double x) {
    uint64_t b;
    std::memcpy(&b, &x, sizeof(b));
    h ^= b;
    h *= 0x100000001b3ULL;
  };
  for (size_t i = 0; i < upto; ++i) mix(diag[i]);
  for (size_t i = 0; i < upto; ++i) mix(off[i]);
  return h;
}

// FNV-1a over the fp32 bits: one thread per 4096-element chunk, then the chunk hashes in order (one thread)
__global__ void hash_chunks_kernel(const float* __restrict__ v, size_t n, unsigned long long* __restrict__ ch,
                                   size_t nch) {
  const size_t c = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (c >= nch) return;
  unsigned long long h = 0xcbf29ce484222325ULL;
  const size_t e = min(n, (c + 1) * 4096);
  for (size_t i = c * 4096; i < e; ++i) {
    h ^= (unsigned long long)__float_as_uint(v[i]);
    h *= 0x100000001b3ULL;
  }
  ch[c] = h;
}
__global__ void hash_final_kernel(const unsigned long long* __restrict__ ch, size_t nch, double* out2) {
  unsigned long long h = 0xcbf29ce484222325ULL;
  for (size_t c = 0; c < nch; ++c) {
    h ^= ch[c];
    h *= 0x100000001b3ULL;
  }
  out2[0] = (double)(unsigned)(h >> 32);
  out2[1] = (double)(unsigned)h;
}

uint64_t device_hash_f32(dho2g_ctx* ctx, const float* v, size_t n) {
  const size_t nch = std::max<size_t>(1, cdiv(n, 4096));
  DevBuf<unsigned long long> ch(nch);
  DevBuf<double> o(2);
  hash_chunks_kernel<<<(unsigned)cdiv(nch, 256), 256, 0, ctx->stream>>>(v, n, ch.p, nch);
  hash_final_kernel<<<1, 1, 0, ctx->stream>>>(ch.p, nch, o.p);
  DHO2G_LAUNCH();
  double h[2];
  DHO2G_CUDA(cudaMemcpyAsync(h, o.p, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream));
  wait_stream(ctx, ctx->stream);
  return ((uint64_t)(unsigned)h[0] << 32) | (uint64_t)(unsigned)h[1];
}

// Worker::all_equal (collectives.cpp): every rank's value equal to every other's
bool ranks_all_equal(dho2g_ctx* ctx, uint64_t h) {
  if (ctx->world == 1) return true;
  if (ctx->hash_checks == 2) h ^= (uint64_t)ctx->rank;  // test hook: a simulated divergence on ranks > 0
  DevBuf<double> ex(2 + 2 * (size_t)ctx->world);
  const double mine[2] = {(double)(uint32_t)(h >> 32), (double)(uint32_t)h};
  DHO2G_CUDA(cudaMemcpyAsync(ex.p, mine, sizeof(mine), cudaMemcpyHostToDevice, ctx->stream));
  ctx->allgather_f64(ex.p, ex.p + 2, 2, "hash_check");
  std::vector<double> all(2 * (size_t)ctx->world);
  DHO2G_CUDA(cudaMemcpyAsync(all.data(), ex.p + 2, all.size() * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  wait_stream(ctx, ctx->stream);
  for (int r = 1; r < ctx->world; ++r)
    if (all[2 * r] != all[0] || all[2 * r + 1] != all[1]) return false;
  return true;
}
}  // namespace dho2g

void dho2g_ctx::allgather_f64(const double* send, double* recv, size_t count, const char* op) {
  check_usable();
  if (world == 1 && !nccl_force) {
    if (send != recv) DHO2G_CUDA(cudaMemcpyAsync(recv, send, count * sizeof(double), cudaMemcpyDeviceToDevice, stream));
    return;
  }
  if (fabric) fabric_collective(this, send, recv, count, sizeof(double), 0);
  else if (host_ag) host_collective(this, send, recv, count, sizeof(double), 0);
  else dho2g::nccl_call(this, dho2g::nccl().AllGather(send, recv, count, ncclDouble, comm, stream), "all_gather");
  bump("nccl_calls", 1);
  bump("nccl_bytes", double(count) * 8 * world);
  const int64_t c = (int64_t)count, w1 = world - 1;
  if (std::string(op) == "all_reduce") ledger_add(op, c, c * w1, c * w1);  // collectives.cpp:306-319 model
  else ledger_add(op, c * world, c * w1, c * w1);
}

void dho2g_ctx::allgather_f32(const float* send, float* recv, size_t count, const char* op) {
  check_usable();
  if (world == 1 && !nccl_force) {
    if (send != recv) DHO2G_CUDA(cudaMemcpyAsync(recv, send, count * sizeof(float), cudaMemcpyDeviceToDevice, stream));
    return;
  }
  if (fabric) fabric_collective(this, send, recv, count, sizeof(float), 0);
  else if (host_ag) host_collective(this, send, recv, count, sizeof(float), 0);
  else dho2g::nccl_call(this, dho2g::nccl().AllGather(send, recv, count, ncclFloat, comm, stream), "all_gather");
  bump("nccl_calls", 1);
  bump("nccl_bytes", double(count) * 4 * world);
  const int64_t c = (int64_t)count, w1 = world - 1;
  ledger_add(op, c * world, c * w1, c * w1);
}

void dho2g_ctx::reduce_scatter_f32(const float* send, float* recv, size_t count) {
  check_usable();
  if (world == 1 && !nccl_force) {
    if (send != recv) DHO2G_CUDA(cudaMemcpyAsync(recv, send, count * sizeof(float), cudaMemcpyDeviceToDevice, stream));
    return;
  }
  if (fabric) fabric_collective(this, send, recv, count, sizeof(float), 1);
  else if (host_ag) host_collective(this, send, recv, count, sizeof(float), 1);
  else dho2g::nccl_call(this, dho2g::nccl().ReduceScatter(send, recv, count, ncclFloat, ncclSum, comm, stream),
                        "reduce_scatter");
  bump("nccl_calls", 1);
  bump("nccl_bytes", double(count) * 4 * world);
  const int64_t c = (int64_t)count, w1 = world - 1;
  ledger_add("reduce_scatter", c * world, c * w1, c * w1);
}

namespace {
__global__ void ordered_sum_kernel(const double* __restrict__ all, double* __restrict__ out, size_t count, int world) {
  for (size_t i = blockIdx.x * blockDim.x + threadIdx.x; i < count; i += size_t(gridDim.x) * blockDim.x) {
    double s = all[i];
    for (int r = 1; r < world; ++r) s += all[size_t(r) * count + i];  // ascending rank (collectives.cpp:310-324)
    out[i] = s;
  }
}
}  // namespace

void dho2g_ctx::barrier() {
  if (world == 1) return;
  barrier_buf.ensure(1 + (size_t)world);
  allgather_f64(barrier_buf.p, barrier_buf.p + 1, 1, "barrier");
}

void dho2g_ctx::allreduce_sum_f64_ordered(double* inout, size_t count) {
  if (world == 1 && !nccl_force) return;
  gather_f64.ensure(count * world);
  allgather_f64(inout, gather_f64.p, count, "all_reduce");
  ordered_sum_kernel<<<(unsigned)std::min<size_t>(dho2g::cdiv(count, 256), 1024), 256, 0, stream>>>(
      gather_f64.p, inout, count, world);
  DHO2G_LAUNCH();
}
