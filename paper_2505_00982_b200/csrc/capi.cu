// extern "C" boundary of libdho2gpu.so (include/dho2gpu.h). Every entry point converts internal
// exceptions into a dho2g_status + thread-local message, mirroring the reference's exception
// types (proj/include/dho2/errors.hpp:8-36).
#include <cudaTypedefs.h>

#include <cmath>
#include <cstring>
#include <thread>

#include "internal.h"

using namespace dho2g;

namespace {
thread_local std::string g_err;

template <typename F>
int guard(F&& f) {
  try {
    f();
    return DHO2G_OK;
  } catch (const Error& e) {
    g_err = e.what();
    return e.code;
  } catch (const std::bad_alloc& e) {
    g_err = std::string("host allocation failed: ") + e.what();
    return DHO2G_CUDA;
  } catch (const std::exception& e) {
    g_err = e.what();
    return DHO2G_ARGUMENT;
  }
}

void check_ctx(dho2g_ctx* c) {
  if (!c) fail(DHO2G_ARGUMENT, "null context");
  c->check_usable();
  DHO2G_CUDA(cudaSetDevice(c->device));
}

std::vector<float> to_f32(const double* p, size_t n) {
  std::vector<float> f(n);
  for (size_t i = 0; i < n; ++i) f[i] = (float)p[i];
  return f;
}

void upload(DevBuf<float>& buf, const double* p, size_t n, cudaStream_t s) {
  buf.ensure(std::max<size_t>(n, 1));
  if (!n) return;
  const auto f = to_f32(p, n);
  DHO2G_CUDA(cudaMemcpyAsync(buf.p, f.data(), n * sizeof(float), cudaMemcpyHostToDevice, s));
  DHO2G_CUDA(cudaStreamSynchronize(s));  // host vector f goes out of scope
}

void download(const float* d, double* p, size_t n, cudaStream_t s) {
  std::vector<float> f(n);
  DHO2G_CUDA(cudaMemcpyAsync(f.data(), d, n * sizeof(float), cudaMemcpyDeviceToHost, s));
  DHO2G_CUDA(cudaStreamSynchronize(s));
  for (size_t i = 0; i < n; ++i) p[i] = f[i];
}

// oracle.cpp:326-343
void check_batch(const dho2g_mlp* m, size_t B, size_t ncls) {
  if (B == 0) fail(DHO2G_ARGUMENT, "mlp oracle: empty batch");
  const size_t out = m->sizes.back();
  if (m->loss == 0) {
    if (ncls == 0 || ncls != out) fail(DHO2G_ARGUMENT, "mlp oracle: softmax_ce needs n_classes == output layer size");
  } else if (ncls > 0) {
    if (ncls != out) fail(DHO2G_ARGUMENT, "mlp oracle: mse one-hot targets need n_classes == output layer size");
  } else if (out != 1) {
    fail(DHO2G_ARGUMENT, "mlp oracle: regression targets need output layer size 1");
  }
}

uint64_t splitmix_at(uint64_t s0, uint64_t i) {
  uint64_t z = s0 + (i + 1) * 0x9e3779b97f4a7c15ULL;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
// normal number i of Rng(s0) (rng.hpp:37-50): pair p = i/2, cos for even i, sin (spare) for odd i
double normal_at(uint64_t s0, uint64_t i) {
  const uint64_t p = i >> 1;
  const double u1 = (static_cast<double>(splitmix_at(s0, 2 * p) >> 11) + 1.0) * 0x1.0p-53;
  const double u2 = static_cast<double>(splitmix_at(s0, 2 * p + 1) >> 11) * 0x1.0p-53;
  const double radius = std::sqrt(-2.0 * std::log(u1));
  const double angle = 2.0 * 3.141592653589793 * u2;
  return (i & 1) ? radius * std::sin(angle) : radius * std::cos(angle);
}
}  // namespace

extern "C" {

const char* dho2g_last_error(void) { return g_err.c_str(); }

int dho2g_ctx_create(int device, dho2g_ctx** out) {
  return guard([&] {
    auto c = std::make_unique<dho2g_ctx>();
    c->device = device;
    DHO2G_CUDA(cudaSetDevice(device));
    DHO2G_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    DHO2G_CUDA(cudaDeviceGetAttribute(&c->sm_count, cudaDevAttrMultiProcessorCount, device));
    int major = 0, minor = 0;
    DHO2G_CUDA(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device));
    DHO2G_CUDA(cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, device));
    if (major != 10) fail(DHO2G_CUDA, "libdho2gpu is built for sm_100a (B200); device is sm_" +
                                          std::to_string(major) + std::to_string(minor));
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    DHO2G_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
    if (q != cudaDriverEntryPointSuccess || !fn) fail(DHO2G_CUDA, "cuTensorMapEncodeTiled unavailable");
    c->encode_fn = fn;
    *out = c.release();
  });
}

int dho2g_ctx_destroy(dho2g_ctx* ctx) {
  return guard([&] {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    if (ctx->stream2) {
      cudaStreamSynchronize(ctx->stream2);
      cudaStreamDestroy(ctx->stream2);
    }
    for (cudaEvent_t ev : ctx->lane_events) cudaEventDestroy(ev);
    if (ctx->comm) dho2g::nccl().CommAbort(ctx->comm);  // non-blocking communicator: abort frees at once
    cudaStreamDestroy(ctx->stream);
    delete ctx;
  });
}

int dho2g_ctx_set_option(dho2g_ctx* ctx, const char* key, double value) {
  return guard([&] {
    check_ctx(ctx);
    const std::string k = key ? key : "";
    if (k == "gemm") ctx->gemm_backend = (int)value;
    else if (k == "gemm_splits") ctx->gemm_splits = (int)value;
    else if (k == "gemm_cta") ctx->gemm_cta = (int)value;
    else if (k == "gemm_dp") ctx->gemm_dp = (int)value;
    else if (k == "gemm_group") ctx->gemm_group = (int)value;
    else if (k == "gemm_min_kb") ctx->gemm_min_kb = (int)value;
    else if (k == "gemm_mm_tc1") ctx->gemm_mm_tc1 = (int)value;
    else if (k == "bwd_overlap") ctx->bwd_overlap = (int)value;
    else if (k == "gemm_chunk_kb") {
      ctx->gemm_chunk_kb = (int)value;
      ++g_graph_gen;  // baked into captured refresh graphs
    }
    else if (k == "gemm_chunk_kb1") {
      ctx->gemm_chunk_kb1 = (int)value;
      ++g_graph_gen;  // baked into captured refresh graphs
    }
    else if (k == "gemm_f16") {
      ctx->gemm_f16 = (int)value;
      ++g_graph_gen;  // baked into captured refresh graphs
    }
    else if (k == "mlp_small") {
      ctx->mlp_small = (int)value;
      ++g_graph_gen;  // baked into captured refresh graphs
    }
    else if (k == "hash_checks") ctx->hash_checks = (int)value;
    else if (k == "upd_small") ctx->upd_small = (int)value;
    else if (k == "upd_small_max_rows") ctx->upd_small_max_rows = value;
    else if (k == "lanczos_small") {
      ctx->lanczos_small = (int)value;
      ++g_graph_gen;
    }
    else if (k == "lanczos_small_max_n") {
      ctx->lanczos_small_max_n = value;
      ++g_graph_gen;
    }
    else if (k == "mlp_small_mflop") {
      ctx->mlp_small_mflop = value;
      ++g_graph_gen;
    }
    else if (k == "mlp_small_ctas_per_sm") {
      ctx->mlp_small_ctas_per_sm = (int)value;
      ++g_graph_gen;
    }
    else if (k == "hvp_route") ctx->hvp_route = (int)value;
    else if (k == "upd_p2_variant") ctx->upd_p2_variant = (int)value;
    else if (k == "gemm_pdl") {
      ctx->gemm_pdl = (int)value;
      ++g_graph_gen;  // baked into captured refresh graphs
    }
    else if (k == "nccl_timeout_s") ctx->nccl_timeout_s = value;
    else if (k == "lanczos_recurrence") {
      ctx->lanczos_recurrence = (int)value;
      ++g_graph_gen;  // baked into captured refresh graphs
    }
    else if (k == "upd_p2_staged") ctx->upd_p2_staged = (int)value;
    else if (k == "ritz_tc") ctx->ritz_tc = (int)value;
    else if (k == "tql2_split") ctx->tql2_split = (int)value;
    else if (k == "tql2_log_cap") ctx->tql2_log_cap = (long long)value;
    else if (k == "gs_sm_cap") ctx->gs_sm_cap = (int)value;
    else if (k == "graphs") ctx->use_graphs = (int)value;
    else if (k == "graphs_multirank") ctx->graphs_multirank = (int)value;
    else if (k == "ktimers") {
      ctx->kt_flush();
      ctx->ktimers = value != 0.0;
    } else if (k == "ktimers_reset") {
      ctx->kt_flush();
      ctx->kstats.clear();
    }
    else fail(DHO2G_ARGUMENT, "unknown option '" + k + "'");
  });
}

int dho2g_ctx_get_stat(dho2g_ctx* ctx, const char* key, double* value) {
  return guard([&] {
    if (!ctx) fail(DHO2G_ARGUMENT, "null context");
    const std::string k = key ? key : "";
    if (k.rfind("kt.", 0) == 0) {  // kt.<kernel>.ms | .count | .work
      ctx->kt_flush();
      const size_t dot = k.rfind('.');
      const std::string name = k.substr(3, dot - 3), field = k.substr(dot + 1);
      auto it = ctx->kstats.find(name);
      if (it == ctx->kstats.end()) *value = 0.0;
      else *value = field == "ms" ? it->second.ms : field == "count" ? it->second.count : it->second.work;
      return;
    }
    if (k == "kt_names") {  // number of timed kernels; names via dho2g_ctx_kernel_name
      ctx->kt_flush();
      *value = (double)ctx->kstats.size();
      return;
    }
    if (k == "launches") *value = (double)g_launches;
    else if (k == "sm_count") *value = ctx->sm_count;
    else if (k == "world") *value = ctx->world;
    else if (k == "rank") *value = ctx->rank;
    else {
      auto it = ctx->stats.find(k);
      *value = it == ctx->stats.end() ? 0.0 : it->second;
    }
  });
}

int dho2g_ctx_kernel_name(dho2g_ctx* ctx, int i, char* buf, size_t len) {
  return guard([&] {
    ctx->kt_flush();
    if (i < 0 || (size_t)i >= ctx->kstats.size()) fail(DHO2G_ARGUMENT, "kernel index out of range");
    auto it = ctx->kstats.begin();
    std::advance(it, i);
    std::snprintf(buf, len, "%s", it->first.c_str());
  });
}

int dho2g_timer_mark(dho2g_ctx* ctx, int id) {
  return guard([&] {
    check_ctx(ctx);
    if (id < 0 || id > 1023) fail(DHO2G_ARGUMENT, "timer id out of range");
    while ((int)ctx->marks.size() <= id) {
      cudaEvent_t e;
      DHO2G_CUDA(cudaEventCreate(&e));
      ctx->marks.push_back(e);
    }
    DHO2G_CUDA(cudaEventRecord(ctx->marks[id], ctx->stream));
  });
}

int dho2g_timer_ms(dho2g_ctx* ctx, int id0, int id1, double* ms) {
  return guard([&] {
    check_ctx(ctx);
    if (id0 < 0 || id1 < 0 || id0 >= (int)ctx->marks.size() || id1 >= (int)ctx->marks.size())
      fail(DHO2G_ARGUMENT, "timer id not marked");
    DHO2G_CUDA(cudaEventSynchronize(ctx->marks[id1]));
    float f = 0.f;
    DHO2G_CUDA(cudaEventElapsedTime(&f, ctx->marks[id0], ctx->marks[id1]));
    *ms = f;
  });
}

int dho2g_synchronize(dho2g_ctx* ctx) {
  return guard([&] {
    check_ctx(ctx);
    ctx->sync();
  });
}

int dho2g_nccl_unique_id(void* id_out_128) {
  return guard([&] {
    ncclUniqueId id;
    DHO2G_NCCLCHK(dho2g::nccl().GetUniqueId(&id));
    std::memcpy(id_out_128, &id, sizeof(id));
  });
}

int dho2g_comm_init(dho2g_ctx* ctx, const void* nccl_id_128, int rank, int world) {
  return guard([&] {
    check_ctx(ctx);
    if (world < 1 || rank < 0 || rank >= world) fail(DHO2G_ARGUMENT, "Shard: rank out of range");
    ctx->rank = rank;
    ctx->world = world;
    if (world == 1) return;
    ncclUniqueId id;
    std::memcpy(&id, nccl_id_128, sizeof(id));
    // non-blocking init + polling: a rank that never joins is a DeadlockError after nccl_timeout_s
    // (test_collectives.cpp:245-258), not a hang
    ncclConfig_t cfg = NCCL_CONFIG_INITIALIZER;
    cfg.blocking = 0;
    dho2g::nccl_call(ctx, dho2g::nccl().CommInitRankConfig(&ctx->comm, world, id, rank, &cfg), "comm_init");
    dho2g::nccl_settle(ctx, "comm_init");
  });
}

// ------------------------------------------------------------------ accounting (CommLedger / SlotMeter)
size_t dho2g_ctx_ledger_rows(dho2g_ctx* ctx) { return ctx ? ctx->ledger.size() : 0; }
int dho2g_ctx_ledger_row(dho2g_ctx* ctx, size_t i, int64_t* event, char* op, size_t op_len, int64_t* floats,
                         int* rank, int64_t* sent, int64_t* received) {
  return guard([&] {
    if (!ctx || i >= ctx->ledger.size()) fail(DHO2G_ARGUMENT, "ledger: row out of range");
    const auto& r = ctx->ledger[i];
    if (event) *event = r.event;
    if (op && op_len) {
      std::strncpy(op, r.op.c_str(), op_len - 1);
      op[op_len - 1] = 0;
    }
    if (floats) *floats = r.floats;
    if (rank) *rank = r.rank;
    if (sent) *sent = r.sent;
    if (received) *received = r.received;
  });
}
size_t dho2g_ctx_memory_count(dho2g_ctx* ctx) { return ctx ? ctx->slots.size() : 0; }
int dho2g_ctx_memory_entry(dho2g_ctx* ctx, size_t i, char* name, size_t name_len, int64_t* slots) {
  return guard([&] {
    if (!ctx || i >= ctx->slots.size()) fail(DHO2G_ARGUMENT, "memory: entry out of range");
    auto it = ctx->slots.begin();
    std::advance(it, (long)i);
    if (name && name_len) {
      std::strncpy(name, it->first.c_str(), name_len - 1);
      name[name_len - 1] = 0;
    }
    if (slots) *slots = it->second;
  });
}
int dho2g_ctx_accounting_reset(dho2g_ctx* ctx) {
  return guard([&] {
    if (!ctx) fail(DHO2G_ARGUMENT, "null context");
    ctx->ledger.clear();
    ctx->ledger_next = 0;
    ctx->ledger_sent = 0;
    ctx->slots.clear();
  });
}

int dho2g_local_fabric_create(int world, dho2g_fabric** out) {
  return guard([&] {
    if (world < 1 || !out) fail(DHO2G_ARGUMENT, "local fabric: world_size must be >= 1");
    *out = new dho2g_fabric(world);
  });
}
int dho2g_local_fabric_destroy(dho2g_fabric* fab) {
  return guard([&] { delete fab; });
}
int dho2g_comm_init_local(dho2g_ctx* ctx, dho2g_fabric* fab, int rank) {
  return guard([&] {
    check_ctx(ctx);
    if (!fab) fail(DHO2G_ARGUMENT, "local fabric: null");
    if (rank < 0 || rank >= fab->world) fail(DHO2G_ARGUMENT, "Shard: rank out of range");
    if (ctx->comm) fail(DHO2G_ARGUMENT, "local fabric: context already has a communicator");
    ctx->rank = rank;
    ctx->world = fab->world;
    ctx->fabric = fab->world > 1 ? fab : nullptr;
  });
}

int dho2g_comm_init_host(dho2g_ctx* ctx, int rank, int world, dho2g_host_allgather fn, void* user) {
  return guard([&] {
    check_ctx(ctx);
    if (!fn) fail(DHO2G_ARGUMENT, "host communicator: null all-gather");
    if (world < 1 || rank < 0 || rank >= world) fail(DHO2G_ARGUMENT, "Shard: rank out of range");
    if (ctx->comm || ctx->fabric) fail(DHO2G_ARGUMENT, "host communicator: context already has a communicator");
    ctx->rank = rank;
    ctx->world = world;
    if (world > 1) {
      ctx->host_ag = fn;
      ctx->host_ag_user = user;
    }
  });
}

int dho2g_comm_rank(dho2g_ctx* ctx, int* rank, int* world) {
  return guard([&] {
    if (!ctx) fail(DHO2G_ARGUMENT, "null context");
    *rank = ctx->rank;
    *world = ctx->world;
  });
}

// ------------------------------------------------------------------ host bookkeeping
void dho2g_rng_u64(uint64_t seed, size_t n, uint64_t* out) {
  Rng r(seed);
  for (size_t i = 0; i < n; ++i) out[i] = r.next_u64();
}
void dho2g_rng_normal(uint64_t seed, size_t n, double* out) {
  Rng r(seed);
  for (size_t i = 0; i < n; ++i) out[i] = r.normal();
}
void dho2g_shuffle_iota(uint64_t seed, size_t n, uint64_t* out) { shuffle_iota(seed, n, out); }
uint64_t dho2g_mix_seed(uint64_t seed, uint64_t salt) {  // trainer.cpp:41-46
  uint64_t z = seed + 0x9e3779b97f4a7c15ULL * (salt + 1);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
int dho2g_shard(size_t n, int world, int rank, size_t* begin, size_t* end) {
  return guard([&] { shard_range(n, world, rank, begin, end); });
}
int dho2g_lanczos_budget(size_t k, size_t l, size_t n, size_t* m) {
  return guard([&] { *m = lanczos_budget(k, l, n); });
}
int dho2g_synthetic_dataset(const char* kind, size_t n_samples, uint64_t seed, double* X, double* y, size_t* dim,
                            size_t* ncls) {
  return guard([&] {
    const std::string k = kind ? kind : "";
    uint64_t code;  // DatasetKind enumerators (oracle.hpp)
    if (k == "two-gaussians") code = 0;
    else if (k == "concentric-rings") code = 1;
    else if (k == "linear-regression") code = 2;
    else fail(DHO2G_ARGUMENT, "unknown dataset kind: '" + k + "'");
    if (n_samples == 0) fail(DHO2G_ARGUMENT, "generate_synthetic_dataset: n_samples must be >= 1");
    Rng rng(seed * 0x2545f4914f6cdd1dULL + code + 1);
    if (code == 0) {  // alternating classes at means -1.5 / +1.5
      for (size_t i = 0; i < n_samples; ++i) {
        const double mean = (i % 2) == 0 ? -1.5 : 1.5;
        X[2 * i] = mean + rng.normal();
        X[2 * i + 1] = mean + rng.normal();
        y[i] = (double)(i % 2);
      }
      *dim = 2;
      *ncls = 2;
    } else if (code == 1) {  // rings of radius 1 / 2.5
      for (size_t i = 0; i < n_samples; ++i) {
        const double radius = ((i % 2) == 0 ? 1.0 : 2.5) + 0.15 * rng.normal();
        const double theta = 2.0 * 3.141592653589793 * rng.uniform();
        X[2 * i] = radius * std::cos(theta);
        X[2 * i + 1] = radius * std::sin(theta);
        y[i] = (double)(i % 2);
      }
      *dim = 2;
      *ncls = 2;
    } else {  // y = beta^T x + 0.05 N(0,1), d = 3
      double beta[3];
      for (double& b : beta) b = rng.normal();
      for (size_t i = 0; i < n_samples; ++i) {
        double dot = 0.0;
        for (size_t j = 0; j < 3; ++j) {
          X[i * 3 + j] = rng.normal();
          dot += beta[j] * X[i * 3 + j];
        }
        y[i] = dot + 0.05 * rng.normal();
      }
      *dim = 3;
      *ncls = 0;
    }
  });
}

void dho2g_epoch_permutation(size_t N, uint64_t shuffle_seed, uint64_t epoch, uint64_t* out) {
  shuffle_iota(shuffle_seed * 0x9e3779b97f4a7c15ULL + epoch + 1, N, out);
}
void dho2g_curvature_indices(size_t N, size_t want, uint64_t seed, uint64_t refresh, uint64_t* out) {
  std::vector<uint64_t> all(N);
  shuffle_iota(dho2g_mix_seed(seed, 0xc0ffee + refresh), N, all.data());
  std::copy(all.begin(), all.begin() + std::min(want, N), out);
}
int dho2g_batch_indices(const uint64_t* perm, size_t N, int workers, int worker, size_t round, size_t batch,
                        uint64_t* out) {
  return guard([&] {
    size_t sb, se;
    shard_range(N, workers, worker, &sb, &se);
    const size_t len = se - sb;
    if (len == 0) fail(DHO2G_ARGUMENT, "train: fewer samples than workers");
    for (size_t j = 0; j < batch; ++j) out[j] = perm[sb + (round * batch + j) % len];
  });
}
void dho2g_blobs_dataset(size_t N, size_t D, size_t n_classes, uint64_t seed, double* X, double* y) {
  const uint64_t s0 = seed * 0x2545F4914F6CDD1DULL + 0xB10B5ULL;
  const size_t nmu = n_classes * D;
  std::vector<double> mu(nmu);
  for (size_t i = 0; i < nmu; ++i) mu[i] = normal_at(s0, i);
  const unsigned nt = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
  std::vector<std::thread> th;
  for (unsigned t = 0; t < nt; ++t)
    th.emplace_back([&, t] {
      for (size_t i = t; i < N; i += nt) {
        const size_t c = n_classes ? i % n_classes : 0;
        for (size_t k = 0; k < D; ++k) X[i * D + k] = mu[c * D + k] + normal_at(s0, nmu + i * D + k);
        y[i] = (double)c;
      }
    });
  for (auto& x : th) x.join();
}

// ------------------------------------------------------------------ MLP plugin
int dho2g_mlp_create(dho2g_ctx* ctx, const size_t* sizes, int n_sizes, int act, int loss, dho2g_mlp** out) {
  return guard([&] {
    check_ctx(ctx);
    if (n_sizes < 3) fail(DHO2G_ARGUMENT, "mlp oracle: need at least one hidden layer");
    for (int i = 0; i < n_sizes; ++i)
      if (sizes[i] == 0) fail(DHO2G_ARGUMENT, "mlp oracle: zero layer size");
    if (act < 0 || act > 1) fail(DHO2G_ARGUMENT, "activation: expected tanh|relu");
    if (loss < 0 || loss > 1) fail(DHO2G_ARGUMENT, "loss: expected mse|softmax_ce");
    auto m = std::make_unique<dho2g_mlp>();
    m->ctx = ctx;
    m->sizes.assign(sizes, sizes + n_sizes);
    m->act = act;
    m->loss = loss;
    m->L = n_sizes - 1;
    size_t off = 0;
    for (int t = 0; t < m->L; ++t) {
      LayerDesc ld;
      ld.in = (int)sizes[t];
      ld.out = (int)sizes[t + 1];
      ld.Pin = (int)round_up(sizes[t], 8);
      ld.Pout = (int)round_up(sizes[t + 1], 8);
      ld.Din = (int)round_up(sizes[t], 64);
      ld.Dout = (int)round_up(sizes[t + 1], 64);
      ld.w_off = off;
      off += sizes[t] * sizes[t + 1];
      ld.b_off = off;
      off += sizes[t + 1];
      m->layers.push_back(ld);
    }
    m->dim = off;
    for (size_t s : m->sizes) m->smax = std::max(m->smax, s);
    m->WV_hi.resize(m->L); m->WV_lo.resize(m->L);
    for (int t = 0; t < m->L; ++t) {
      const LayerDesc& ld = m->layers[t];
      m->WV_hi[t].alloc((size_t)ld.out * 2 * ld.Pin);
      m->WV_lo[t].alloc((size_t)ld.out * 2 * ld.Pin);
    }
    m->scl.alloc((size_t)3 * m->L);
    m->sclx.alloc((size_t)3 * m->L);
    m->sticket.alloc((size_t)3 * m->L);
    m->amax.alloc((size_t)5 * (m->L + 1));
    *out = m.release();
  });
}

int dho2g_mlp_destroy(dho2g_mlp* mlp) {
  return guard([&] {
    if (!mlp) return;
    cudaSetDevice(mlp->ctx->device);
    cudaStreamSynchronize(mlp->ctx->stream);
    delete mlp;
  });
}

size_t dho2g_mlp_dim(const dho2g_mlp* mlp) { return mlp ? mlp->dim : 0; }

int dho2g_mlp_init_params(const dho2g_mlp* mlp, uint64_t seed, double* w) {  // oracle.cpp:386-394
  return guard([&] {
    std::fill(w, w + mlp->dim, 0.0);
    Rng rng(seed * 0x9e3779b97f4a7c15ULL + 17);
    for (const LayerDesc& l : mlp->layers) {
      const double sd = 1.0 / std::sqrt(static_cast<double>(l.in));
      for (size_t k = 0; k < (size_t)l.in * l.out; ++k) w[l.w_off + k] = sd * rng.normal();
    }
  });
}

// The same draw from the layer sizes alone (no context / device): layer-major W then b (oracle.cpp:312-323).
int dho2g_init_params(const size_t* sizes, int n_sizes, uint64_t seed, double* w, size_t* dim) {
  return guard([&] {
    if (!sizes || n_sizes < 3) fail(DHO2G_ARGUMENT, "mlp oracle: need at least one hidden layer");
    size_t off = 0;
    std::vector<size_t> w_off;
    for (int t = 0; t + 1 < n_sizes; ++t) {
      if (sizes[t] == 0 || sizes[t + 1] == 0) fail(DHO2G_ARGUMENT, "mlp oracle: zero layer size");
      w_off.push_back(off);
      off += sizes[t] * sizes[t + 1] + sizes[t + 1];
    }
    *dim = off;
    if (!w) return;
    std::fill(w, w + off, 0.0);
    Rng rng(seed * 0x9e3779b97f4a7c15ULL + 17);
    for (int t = 0; t + 1 < n_sizes; ++t) {
      const double sd = 1.0 / std::sqrt(static_cast<double>(sizes[t]));
      for (size_t k = 0; k < sizes[t] * sizes[t + 1]; ++k) w[w_off[t] + k] = sd * rng.normal();
    }
  });
}

static void mlp_stage(dho2g_mlp* m, const double* w, const double* X, const double* y, size_t B) {
  cudaStream_t s = m->ctx->stream;
  upload(m->w32, w, m->dim, s);
  upload(m->X32, X, B * m->sizes[0], s);
  upload(m->y32, y, B, s);
}

int dho2g_mlp_value(dho2g_mlp* m, const double* w, const double* X, const double* y, size_t B, size_t ncls,
                    double* out) {
  return guard([&] {
    check_ctx(m->ctx);
    std::lock_guard<std::mutex> lk(m->ctx->api_mu);
    check_batch(m, B, ncls);
    mlp_stage(m, w, X, y, B);
    m->red.ensure(2 * 16);
    DHO2G_CUDA(cudaMemsetAsync(m->red.p, 0, 2 * sizeof(double), m->ctx->stream));
    mlp_load_weights(m, m->w32.p);
    mlp_eval_dev(m, m->w32.p, m->X32.p, m->y32.p, nullptr, B, ncls, m->red.p);
    double h[2];
    DHO2G_CUDA(cudaMemcpyAsync(h, m->red.p, 2 * sizeof(double), cudaMemcpyDeviceToHost, m->ctx->stream));
    DHO2G_CUDA(cudaStreamSynchronize(m->ctx->stream));
    *out = h[0] / (double)B;
  });
}

int dho2g_mlp_accuracy(dho2g_mlp* m, const double* w, const double* X, const double* y, size_t B, size_t ncls,
                       double* acc) {
  return guard([&] {
    check_ctx(m->ctx);
    std::lock_guard<std::mutex> lk(m->ctx->api_mu);
    if (ncls == 0) {  // oracle.cpp:650: nullopt for regression
      *acc = -1.0;
      return;
    }
    check_batch(m, B, ncls);
    mlp_stage(m, w, X, y, B);
    m->red.ensure(2 * 16);
    DHO2G_CUDA(cudaMemsetAsync(m->red.p, 0, 2 * sizeof(double), m->ctx->stream));
    mlp_load_weights(m, m->w32.p);
    mlp_eval_dev(m, m->w32.p, m->X32.p, m->y32.p, nullptr, B, ncls, m->red.p);
    double h[2];
    DHO2G_CUDA(cudaMemcpyAsync(h, m->red.p, 2 * sizeof(double), cudaMemcpyDeviceToHost, m->ctx->stream));
    DHO2G_CUDA(cudaStreamSynchronize(m->ctx->stream));
    *acc = h[1] / (double)B;
  });
}

int dho2g_mlp_grad(dho2g_mlp* m, const double* w, const double* X, const double* y, size_t B, size_t ncls,
                   double* g) {
  return guard([&] {
    check_ctx(m->ctx);
    std::lock_guard<std::mutex> lk(m->ctx->api_mu);
    check_batch(m, B, ncls);
    mlp_stage(m, w, X, y, B);
    m->out32.ensure(m->dim);
    mlp_load_weights(m, m->w32.p);
    mlp_grad_dev(m, m->w32.p, m->X32.p, m->y32.p, nullptr, B, ncls, 1.0 / (double)B, m->out32.p);
    download(m->out32.p, g, m->dim, m->ctx->stream);
  });
}

int dho2g_mlp_hvp(dho2g_mlp* m, const double* w, const double* v, const double* X, const double* y, size_t B,
                  size_t ncls, double* hv) {
  return guard([&] {
    check_ctx(m->ctx);
    std::lock_guard<std::mutex> lk(m->ctx->api_mu);
    check_batch(m, B, ncls);
    mlp_stage(m, w, X, y, B);
    upload(m->v32, v, m->dim, m->ctx->stream);
    m->out32.ensure(m->dim);
    mlp_set_input(m, m->X32.p, m->y32.p, nullptr, B, true);
    mlp_load_weights(m, m->w32.p);
    double vmax = 0.0;  // the fp16 operand scale of the direction halves is sized from max |v|
    for (size_t i = 0; i < m->dim; ++i) vmax = std::max(vmax, std::fabs(v[i]));
    mlp_hvp_dev(m, m->v32.p, nullptr, B, ncls, 1.0 / (double)B, m->out32.p, (float)std::max(vmax, 1e-30));
    download(m->out32.p, hv, m->dim, m->ctx->stream);
  });
}

// ------------------------------------------------------------------ operators
int dho2g_op_mlp(dho2g_ctx* ctx, dho2g_mlp* mlp, const double* w, const double* X, const double* y, size_t B,
                 size_t ncls, dho2g_op** out) {
  return guard([&] {
    check_ctx(ctx);
    check_batch(mlp, B, ncls);
    auto op = std::make_unique<dho2g_op>();
    op->ctx = ctx;
    op->kind = 0;
    op->n = mlp->dim;
    op->mlp = mlp;
    upload(op->w, w, mlp->dim, ctx->stream);
    upload(op->X, X, B * mlp->sizes[0], ctx->stream);
    upload(op->y, y, B, ctx->stream);
    op->wptr = op->w.p;
    op->Xptr = op->X.p;
    op->yptr = op->y.p;
    op->B = B;
    op->ncls = ncls;
    shard_range(B, ctx->world, ctx->rank, &op->b0, &op->b1);
    op->scale = 1.0 / (double)B;
    if (ctx->world > 1) op->hfull.alloc(cdiv(op->n, (size_t)ctx->world) * ctx->world);
    *out = op.release();
  });
}

int dho2g_op_diag(dho2g_ctx* ctx, const double* spectrum, size_t n, dho2g_op** out) {
  return guard([&] {
    check_ctx(ctx);
    if (n == 0) fail(DHO2G_ARGUMENT, "quadratic oracle: empty spectrum");
    auto op = std::make_unique<dho2g_op>();
    op->ctx = ctx;
    op->kind = 1;
    op->n = n;
    upload(op->mat, spectrum, n, ctx->stream);
    *out = op.release();
  });
}

// QuadraticOracle(spectrum, rotation_seed) (oracle.cpp:233-260) as a device operator.
int dho2g_op_quadratic(dho2g_ctx* ctx, const double* spectrum, size_t n, uint64_t rotation_seed, dho2g_op** out) {
  return guard([&] {
    check_ctx(ctx);
    if (n == 0 || !spectrum) fail(DHO2G_ARGUMENT, "quadratic oracle: empty spectrum");
    for (size_t i = 0; i < n; ++i)
      if (spectrum[i] == 0.0 || !std::isfinite(spectrum[i]))
        fail(DHO2G_ARGUMENT, "quadratic oracle: spectrum entries must be nonzero and finite");
    auto op = std::make_unique<dho2g_op>();
    op->ctx = ctx;
    op->kind = rotation_seed ? 4 : 1;
    op->n = n;
    upload(op->mat, spectrum, n, ctx->stream);
    if (rotation_seed) {
      // the rotation is dense (n^2 fp64 on the host, O(n^3) to build, 8 n^2 bytes in HBM): desk-scale
      // problems only, like the reference's constructor (oracle.cpp:246)
      if (n > 32768) fail(DHO2G_ARGUMENT, "quadratic oracle: a rotated spectrum is limited to n <= 32768");
      std::vector<double> Q(n * n);
      if (!quadratic_rotation(n, rotation_seed, Q.data())) fail(DHO2G_NUMERIC, "quadratic oracle: degenerate rotation draw");
      size_t b, e;
      shard_range(n, ctx->world, ctx->rank, &b, &e);
      op->q_begin = b;
      op->q_rows = e - b;
      // this rank's columns: Q^T[:, i] = row i of Q (for Q v) and Q[:, i] (for Q^T y), i in [b, e)
      std::vector<double> qt(n * op->q_rows), qc(n * op->q_rows);
      for (size_t i = b; i < e; ++i)
        for (size_t j = 0; j < n; ++j) {
          qt[(i - b) * n + j] = Q[j * n + i];
          qc[(i - b) * n + j] = Q[i * n + j];
        }
      upload(op->qrot_t, qt.data(), qt.size(), ctx->stream);
      upload(op->qrot, qc.data(), qc.size(), ctx->stream);
      const size_t base = cdiv(n, (size_t)ctx->world);
      op->qy.alloc(base * ctx->world);
      op->qy_loc.alloc(std::max<size_t>(base, 1));
    }
    *out = op.release();
  });
}

// apply_h on host buffers: out = H x (full n, every rank), value = x^T H x / 2 (oracle.cpp:274-276).
int dho2g_op_apply(dho2g_op* op, const double* x, double* out, double* value) {
  return guard([&] {
    if (!op || !x) fail(DHO2G_ARGUMENT, "op_apply: null operator or input");
    dho2g_ctx* ctx = op->ctx;
    check_ctx(ctx);
    const size_t n = op->n;
    const size_t base = cdiv(n, (size_t)ctx->world);
    size_t b, e;
    shard_range(n, ctx->world, ctx->rank, &b, &e);
    DevBuf<float> xd(base * ctx->world), hd(base * ctx->world), hs(std::max<size_t>(base, 1));
    DevBuf<double> val(1);
    const auto xf = to_f32(x, n);
    cudaStream_t st = ctx->stream;
    DHO2G_CUDA(cudaMemcpyAsync(xd.p, xf.data(), n * sizeof(float), cudaMemcpyHostToDevice, st));
    float* own = ctx->world == 1 ? hd.p : hs.p;
    op->apply(xd.p, nullptr, own, b, e - b, base);
    if (value) {
      dot_dev(st, xd.p + b, own, e - b, 0.5, val.p);
      ctx->allreduce_sum_f64_ordered(val.p, 1);
    }
    if (ctx->world > 1) ctx->allgather_f32(hs.p, hd.p, base);
    if (out) download(hd.p, out, n, st);
    if (value) {
      DHO2G_CUDA(cudaMemcpyAsync(value, val.p, sizeof(double), cudaMemcpyDeviceToHost, st));
      DHO2G_CUDA(cudaStreamSynchronize(st));
    }
  });
}

int dho2g_op_dense(dho2g_ctx* ctx, const double* mat, size_t n, dho2g_op** out) {
  return guard([&] {
    check_ctx(ctx);
    if (n == 0) fail(DHO2G_ARGUMENT, "dense operator: empty");
    auto op = std::make_unique<dho2g_op>();
    op->ctx = ctx;
    op->kind = 2;
    op->n = n;
    upload(op->mat, mat, n * n, ctx->stream);
    *out = op.release();
  });
}

int dho2g_op_host(dho2g_ctx* ctx, dho2g_host_hvp fn, void* user, size_t n, dho2g_op** out) {
  return guard([&] {
    check_ctx(ctx);
    if (!fn || n == 0) fail(DHO2G_ARGUMENT, "host operator: null callback or empty");
    auto op = std::make_unique<dho2g_op>();
    op->ctx = ctx;
    op->kind = 3;
    op->n = n;
    op->fn = fn;
    op->user = user;
    *out = op.release();
  });
}

int dho2g_op_destroy(dho2g_op* op) {
  return guard([&] {
    if (!op) return;
    if (op->mlp && op->mlp->input_owner == op) op->mlp->input_owner = nullptr;
    cudaStreamSynchronize(op->ctx->stream);
    delete op;
  });
}

// ------------------------------------------------------------------ Lanczos / ESE
int dho2g_lanczos_run(dho2g_ctx* ctx, dho2g_op* op, size_t m, uint64_t seed, const dho2g_lanczos_opts* opts,
                      dho2g_lanczos** out) {
  return guard([&] {
    check_ctx(ctx);
    if (!op) fail(DHO2G_ARGUMENT, "null operator");
    if (m < 1 || m > op->n) fail(DHO2G_ARGUMENT, "lanczos_distributed: need 1 <= m <= n");
    if (m >= (size_t)kMaxLanczos) fail(DHO2G_ARGUMENT, "lanczos: m exceeds the device limit (1023)");
    auto lz = std::make_unique<dho2g_lanczos>();
    if (opts) lz->opts = *opts;
    lanczos_alloc(lz.get(), ctx, op->n, m);
    lanczos_run_into(lz.get(), op, seed);
    *out = lz.release();
  });
}

int dho2g_lanczos_result(const dho2g_lanczos* lz, double* diag, double* off, size_t* iters, int* breakdown,
                         size_t* safeguard_passes, size_t* shard_begin, size_t* shard_end) {
  return guard([&] {
    const int it = lz->host.iters;
    if (diag)
      for (int i = 0; i < it; ++i) diag[i] = lz->host.diag[i];
    const int noff = lz->host.breakdown ? it - 1 : it;
    if (off)
      for (int i = 0; i < noff; ++i) off[i] = lz->host.off[i];
    if (iters) *iters = (size_t)it;
    if (breakdown) *breakdown = lz->host.breakdown;
    if (safeguard_passes) *safeguard_passes = (size_t)lz->host.safeguards;
    if (shard_begin) *shard_begin = lz->begin;
    if (shard_end) *shard_end = lz->end;
  });
}

int dho2g_lanczos_basis(const dho2g_lanczos* lz, double* basis_shard) {
  return guard([&] {
    const int it = lz->host.iters;
    const int cols = lz->host.breakdown ? it : it + 1;
    DHO2G_CUDA(cudaStreamSynchronize(lz->ctx->stream));  // legacy-stream copies below do not order with it
    std::vector<float> f(lz->rows);
    for (int j = 0; j < cols; ++j) {
      if (lz->rows)
        DHO2G_CUDA(cudaMemcpy(f.data(), lz->D.p + (size_t)j * lz->ldd, lz->rows * sizeof(float),
                              cudaMemcpyDeviceToHost));
      const double sg = lz->host.sigma[j];
      for (size_t r = 0; r < lz->rows; ++r) basis_shard[(size_t)j * lz->rows + r] = sg * (double)f[r];
    }
  });
}

int dho2g_lanczos_destroy(dho2g_lanczos* lz) {
  return guard([&] { delete lz; });
}

int dho2g_extract_ese(dho2g_ctx* ctx, dho2g_lanczos* lz, size_t k, size_t l, dho2g_ese** out) {
  return guard([&] {
    check_ctx(ctx);
    auto e = std::make_unique<dho2g_ese>();
    extract_ese_into(ctx, lz, k, l, e.get());
    *out = e.release();
  });
}

size_t dho2g_ese_count(const dho2g_ese* ese) { return ese ? ese->r : 0; }

int dho2g_ese_eigvals(const dho2g_ese* ese, double* vals) {
  return guard([&] {
    for (size_t i = 0; i < ese->r; ++i) vals[i] = ese->eigvals[i];
  });
}

int dho2g_ese_eigvecs(const dho2g_ese* ese, double* vecs) {
  return guard([&] {
    if (ese->ctx) DHO2G_CUDA(cudaStreamSynchronize(ese->ctx->stream));
    std::vector<float> f(ese->rows);
    for (size_t c = 0; c < ese->r; ++c) {
      if (ese->rows)
        DHO2G_CUDA(cudaMemcpy(f.data(), ese->V.p + c * ese->ldv, ese->rows * sizeof(float), cudaMemcpyDeviceToHost));
      for (size_t r = 0; r < ese->rows; ++r) vecs[c * ese->rows + r] = (double)(ese->sign[c] * f[r]);
    }
  });
}

// The full V_hat (n x r, column-major) on every rank: extract_ese_distributed's gather_rows
// (dist_lanczos.cpp:148-156) for callers that need the reference's EseResult shape. One all-gather of
// each column's padded shard (equal counts on every rank), rows reassembled by Shard::for_rank.
int dho2g_ese_gather(const dho2g_ese* ese, double* vecs_full) {
  return guard([&] {
    dho2g_ctx* ctx = ese->ctx;
    check_ctx(ctx);
    const int W = ctx->world;
    if (W == 1) {
      DHO2G_CUDA(cudaStreamSynchronize(ctx->stream));
      std::vector<float> f(ese->rows);
      for (size_t c = 0; c < ese->r; ++c) {
        if (ese->rows)
          DHO2G_CUDA(cudaMemcpy(f.data(), ese->V.p + c * ese->ldv, ese->rows * sizeof(float), cudaMemcpyDeviceToHost));
        for (size_t i = 0; i < ese->rows; ++i) vecs_full[c * ese->n + i] = (double)(ese->sign[c] * f[i]);
      }
      return;
    }
    DevBuf<float> all((size_t)W * ese->ldv);
    std::vector<float> h((size_t)W * ese->ldv);
    for (size_t c = 0; c < ese->r; ++c) {
      ctx->allgather_f32(ese->V.p + c * ese->ldv, all.p, ese->ldv, "gather_rows");
      DHO2G_CUDA(cudaMemcpyAsync(h.data(), all.p, h.size() * sizeof(float), cudaMemcpyDeviceToHost, ctx->stream));
      ctx->sync();
      for (int q = 0; q < W; ++q) {
        size_t b, e;
        shard_range(ese->n, W, q, &b, &e);
        for (size_t i = 0; i < e - b; ++i)
          vecs_full[c * ese->n + b + i] = (double)(ese->sign[c] * h[(size_t)q * ese->ldv + i]);
      }
    }
  });
}

// This rank's V_hat rows (signs applied) into a caller-owned device fp32 buffer (column-major, leading dimension
// ld >= rows): for checks that keep a 101 M x 32 V_hat on the device.
__global__ void ese_copy_kernel(const float* __restrict__ V, size_t ldv, size_t rows, float sign, float* dst) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < rows; i += (size_t)gridDim.x * blockDim.x)
    dst[i] = sign * V[i];
}
int dho2g_ese_eigvecs_device(const dho2g_ese* ese, float* dst, size_t ld) {
  return guard([&] {
    check_ctx(ese->ctx);
    if (ld < ese->rows) fail(DHO2G_ARGUMENT, "ese_eigvecs_device: leading dimension < rows");
    for (size_t c = 0; c < ese->r; ++c)
      ese_copy_kernel<<<(unsigned)std::max<size_t>(1, std::min<size_t>(cdiv(ese->rows, 256), 4096)), 256, 0,
                        ese->ctx->stream>>>(ese->V.p + c * ese->ldv, ese->ldv, ese->rows, ese->sign[c], dst + c * ld);
    DHO2G_LAUNCH();
    DHO2G_CUDA(cudaStreamSynchronize(ese->ctx->stream));
  });
}

int dho2g_ese_from_host(dho2g_ctx* ctx, const double* eigvals, const double* V, size_t n, size_t r, dho2g_ese** out) {
  return guard([&] {
    check_ctx(ctx);
    auto e = std::make_unique<dho2g_ese>();
    e->ctx = ctx;
    e->n = n;
    e->r = r;
    shard_range(n, ctx->world, ctx->rank, &e->begin, &e->end);
    e->rows = e->end - e->begin;
    e->ldv = round_up(std::max<size_t>(cdiv(n, (size_t)ctx->world), 1), kGsChunk);
    e->eigvals.assign(eigvals, eigvals + r);
    e->sign.assign(r, 1.f);
    e->V.alloc(e->ldv * std::max<size_t>(r, 1));
    e->ev_dev.alloc(std::max<size_t>(r, 1));
    std::vector<float> col(e->rows);
    for (size_t c = 0; c < r; ++c) {
      for (size_t i = 0; i < e->rows; ++i) col[i] = (float)V[c * n + e->begin + i];
      if (e->rows)
        DHO2G_CUDA(cudaMemcpyAsync(e->V.p + c * e->ldv, col.data(), e->rows * sizeof(float), cudaMemcpyHostToDevice,
                                   ctx->stream));  // stream-ordered before any use (pageable source staged)
    }
    if (r) DHO2G_CUDA(cudaMemcpyAsync(e->ev_dev.p, eigvals, r * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    DHO2G_CUDA(cudaStreamSynchronize(ctx->stream));
    *out = e.release();
  });
}

// The same EseResult from a device-resident fp32 V (column-major, leading dimension ld_src >= n): this
// rank's rows are copied device to device, so a caller that already holds V_hat in HBM (a 101 M x 32
// basis is 13 GB) does not stage it through the host.
int dho2g_ese_from_device(dho2g_ctx* ctx, const double* eigvals, const float* V_dev, size_t ld_src, size_t n, size_t r,
                          dho2g_ese** out) {
  return guard([&] {
    check_ctx(ctx);
    if (ld_src < n) fail(DHO2G_ARGUMENT, "ese_from_device: leading dimension < n");
    auto e = std::make_unique<dho2g_ese>();
    e->ctx = ctx;
    e->n = n;
    e->r = r;
    shard_range(n, ctx->world, ctx->rank, &e->begin, &e->end);
    e->rows = e->end - e->begin;
    e->ldv = round_up(std::max<size_t>(cdiv(n, (size_t)ctx->world), 1), kGsChunk);
    e->eigvals.assign(eigvals, eigvals + r);
    e->sign.assign(r, 1.f);
    e->V.alloc(e->ldv * std::max<size_t>(r, 1));
    e->ev_dev.alloc(std::max<size_t>(r, 1));
    if (r && e->rows)
      DHO2G_CUDA(cudaMemcpy2DAsync(e->V.p, e->ldv * sizeof(float), V_dev + e->begin, ld_src * sizeof(float),
                                   e->rows * sizeof(float), r, cudaMemcpyDeviceToDevice, ctx->stream));
    if (r) DHO2G_CUDA(cudaMemcpyAsync(e->ev_dev.p, eigvals, r * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    DHO2G_CUDA(cudaStreamSynchronize(ctx->stream));
    *out = e.release();
  });
}

int dho2g_ese_destroy(dho2g_ese* ese) {
  return guard([&] { delete ese; });
}

// ------------------------------------------------------------------ optimizer (rank rows of host vectors)
int dho2g_opt_create(dho2g_ctx* ctx, const dho2g_base_cfg* cfg, size_t n, dho2g_opt** out) {
  return guard([&] {
    check_ctx(ctx);
    if (n == 0) fail(DHO2G_ARGUMENT, "BaseOptimizer: zero dimension");
    auto o = std::make_unique<dho2g_opt>();
    size_t b, e;
    shard_range(n, ctx->world, ctx->rank, &b, &e);
    opt_alloc(o.get(), ctx, *cfg, e - b);
    *out = o.release();
  });
}

int dho2g_opt_destroy(dho2g_opt* opt) {
  return guard([&] { delete opt; });
}

struct HostUpd {
  DevBuf<float> g, pi, w, nw, bs;
};

static void run_host_update(dho2g_opt* o, const dho2g_ese* ese, const double* g, const double* pi, const double* w,
                            double alpha, double sigma, double fl, double* newton, double* base) {
  cudaStream_t s = o->ctx->stream;
  const size_t rows = o->n;
  HostUpd h;
  upload(h.g, g, rows, s);
  if (pi) upload(h.pi, pi, rows, s);
  upload(h.w, w, rows, s);
  h.nw.alloc(std::max<size_t>(rows, 1));
  h.bs.alloc(std::max<size_t>(rows, 1));
  UpdateArgs a{};
  a.g = h.g.p;
  a.pi = pi ? h.pi.p : nullptr;
  a.w_a = nullptr;
  a.w_decay = h.w.p;
  a.newton_out = h.nw.p;
  a.base_out = h.bs.p;
  a.alpha = alpha;
  a.sigma = sigma;
  a.floor = fl;
  if (ese && ese->r > 0 && ese->rows != rows) fail(DHO2G_DIMENSION, "deltas: eigenvector rows != gradient length");
  split_update(o, (ese && ese->r > 0) ? ese : nullptr, a);
  check_opt_flags(o);
  if (newton) download(h.nw.p, newton, rows, s);
  if (base) download(h.bs.p, base, rows, s);
}

int dho2g_opt_step(dho2g_opt* opt, const double* g, const double* w, double* d) {
  return guard([&] {
    check_ctx(opt->ctx);
    run_host_update(opt, nullptr, g, nullptr, w, 0.0, 0.0, 1e-6, nullptr, d);
  });
}

int dho2g_deltas(dho2g_opt* opt, const dho2g_ese* ese, const double* g, const double* pi, const double* w, double alpha,
                 double sigma, double eigval_floor, double* newton, double* base) {
  return guard([&] {
    check_ctx(opt->ctx);
    run_host_update(opt, ese, g, pi, w, alpha, sigma, eigval_floor, newton, base);
    if (!ese || ese->r == 0)
      if (newton) std::fill(newton, newton + opt->n, 0.0);
  });
}

int dho2g_admm_w_update(dho2g_ctx* ctx, size_t n, double sigma, const double* w_a, const double* pi, double* w) {
  return guard([&] {
    check_ctx(ctx);
    if (sigma <= 0.0) fail(DHO2G_ARGUMENT, "admm_w_update: sigma must be positive");
    DevBuf<float> a, p, o;
    upload(a, w_a, n, ctx->stream);
    upload(p, pi, n, ctx->stream);
    o.alloc(std::max<size_t>(n, 1));
    admm_w_update_dev(ctx->stream, n, sigma, a.p, p.p, o.p);
    download(o.p, w, n, ctx->stream);
  });
}

int dho2g_admm_dual_update(dho2g_ctx* ctx, size_t n, double sigma, const double* w_a, const double* w, double* pi) {
  return guard([&] {
    check_ctx(ctx);
    DevBuf<float> a, b, p;
    upload(a, w_a, n, ctx->stream);
    upload(b, w, n, ctx->stream);
    upload(p, pi, n, ctx->stream);
    admm_dual_update_dev(ctx->stream, n, sigma, a.p, b.p, p.p);
    download(p.p, pi, n, ctx->stream);
  });
}

// ------------------------------------------------------------------ trainer
int dho2g_trainer_create(dho2g_ctx* ctx, const dho2g_train_cfg* cfg, dho2g_mlp* mlp, const double* X, const double* y,
                         size_t N, size_t ncls, uint64_t dataset_seed, const double* w0, int workers, int host_resident,
                         dho2g_trainer** out) {
  return guard([&] {
    check_ctx(ctx);
    *out = trainer_create(ctx, cfg, mlp, X, y, N, ncls, dataset_seed, w0, workers, host_resident);
  });
}
// train() on Problem{QuadraticOracle, Dataset::dummy(n_samples), w0} (test_trainer.cpp:14-21):
// Dataset::dummy is oracle.cpp:64-68 (one zero feature, no classes, shuffle seed 0).
int dho2g_trainer_create_quadratic(dho2g_ctx* ctx, const dho2g_train_cfg* cfg, dho2g_op* quad, size_t n_samples,
                                   const double* w0, int workers, dho2g_trainer** out) {
  return guard([&] {
    check_ctx(ctx);
    if (!quad) fail(DHO2G_ARGUMENT, "train: null operator");
    if (n_samples == 0) fail(DHO2G_ARGUMENT, "Dataset::dummy: need at least one sample");
    const std::vector<double> zeros(n_samples, 0.0);
    *out = trainer_create(ctx, cfg, nullptr, zeros.data(), zeros.data(), n_samples, 0, 0, w0, workers, 0, quad);
  });
}
int dho2g_trainer_destroy(dho2g_trainer* tr) {
  return guard([&] { trainer_destroy(tr); });
}
int dho2g_trainer_step(dho2g_trainer* tr, size_t steps, int with_eval) {
  return guard([&] {
    check_ctx(trainer_ctx(tr));
    trainer_step(tr, steps, with_eval);
  });
}
int dho2g_trainer_run(dho2g_trainer* tr) {
  return guard([&] {
    check_ctx(trainer_ctx(tr));
    trainer_run(tr);
  });
}
int dho2g_trainer_params(dho2g_trainer* tr, double* w) {
  return guard([&] { trainer_params(tr, w); });
}
size_t dho2g_trainer_rows(dho2g_trainer* tr) { return tr ? trainer_rows(tr) : 0; }
int dho2g_trainer_metrics(dho2g_trainer* tr, size_t max_rows, double* loss, double* acc, double* resid, int64_t* epoch,
                          int* refresh) {
  return guard([&] { trainer_metrics(tr, max_rows, loss, acc, resid, epoch, refresh); });
}
int dho2g_trainer_metrics_ex(dho2g_trainer* tr, size_t max_rows, int64_t* outer, int64_t* inner, double* wallclock) {
  return guard([&] { trainer_metrics_ex(tr, max_rows, outer, inner, wallclock); });
}
int dho2g_trainer_last_loss(dho2g_trainer* tr, double* loss) {
  return guard([&] { *loss = trainer_last_loss(tr); });
}
int dho2g_trainer_stat(dho2g_trainer* tr, const char* key, double* value) {
  return guard([&] {
    if (!trainer_stat(tr, key ? key : "", value)) fail(DHO2G_ARGUMENT, std::string("unknown trainer stat ") + key);
  });
}
int dho2g_trainer_eigvals(dho2g_trainer* tr, double* vals, size_t* count) {
  return guard([&] { trainer_eigvals(tr, vals, count); });
}

// ------------------------------------------------------------------ test hook
namespace {
__global__ void split_rows_kernel(const float* __restrict__ src, int rows, int K, int ld, bf16* __restrict__ hi,
                                  bf16* __restrict__ lo, int f16, float sc) {
  const size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (i >= (size_t)rows * ld) return;
  const int r = (int)(i / ld), k = (int)(i % ld);
  const float x = k < K ? src[(size_t)r * K + k] : 0.f;
  if (f16) split_f16(x, sc, hi[i], lo[i]);
  else split_bf16(x, hi[i], lo[i]);
}
float host_absmax(const float* x, size_t n) {
  float m = 0.f;
  for (size_t i = 0; i < n; ++i) m = std::max(m, std::fabs(x[i]));
  return m;
}
}  // namespace

int dho2g_test_gemm(dho2g_ctx* ctx, int M, int N, int K, const float* A, const float* B, float* Cout, int backend) {
  return guard([&] {
    check_ctx(ctx);
    const int ld = (int)round_up(std::max(K, 1), 8);
    DevBuf<float> a((size_t)M * K), b((size_t)N * K), c((size_t)M * N);
    DevBuf<bf16> ah((size_t)M * ld), al((size_t)M * ld), bh((size_t)N * ld), bl((size_t)N * ld);
    DHO2G_CUDA(cudaMemcpyAsync(a.p, A, sizeof(float) * M * K, cudaMemcpyHostToDevice, ctx->stream));
    DHO2G_CUDA(cudaMemcpyAsync(b.p, B, sizeof(float) * N * K, cudaMemcpyHostToDevice, ctx->stream));
    // operand format as the MLP uses it (ctx option gemm_f16): power-of-two scales from max |A|, max |B|
    const int f16 = ctx->gemm_f16 ? 1 : 0;
    const float sc[2] = {f16 ? pow2_scale(host_absmax(A, (size_t)M * K)) : 1.f,
                         f16 ? pow2_scale(host_absmax(B, (size_t)N * K)) : 1.f};
    DevBuf<float> scd(2);
    DHO2G_CUDA(cudaMemcpyAsync(scd.p, sc, sizeof(sc), cudaMemcpyHostToDevice, ctx->stream));
    split_rows_kernel<<<cdiv((size_t)M * ld, 256), 256, 0, ctx->stream>>>(a.p, M, K, ld, ah.p, al.p, f16, sc[0]);
    split_rows_kernel<<<cdiv((size_t)N * ld, 256), 256, 0, ctx->stream>>>(b.p, N, K, ld, bh.p, bl.p, f16, sc[1]);
    DHO2G_LAUNCH();
    const int saved = ctx->gemm_backend;
    ctx->gemm_backend = backend;
    Epi e{};
    e.mode = EPI_STORE;
    e.M = M;
    e.N = N;
    e.C = c.p;
    e.ldc = N;
    e.alpha = 1.0f;
    e.f16 = f16;
    e.sa = f16 ? scd.p : nullptr;
    e.sb = f16 ? scd.p + 1 : nullptr;
    GOp ga = gop_k(ah.p, al.p, ld, K, M), gb = gop_k(bh.p, bl.p, ld, K, N);
    ga.f16 = gb.f16 = f16;
    try {
      gemm3x(ctx, M, N, K, K, ga, gb, e);
    } catch (...) {
      ctx->gemm_backend = saved;
      throw;
    }
    ctx->gemm_backend = saved;
    DHO2G_CUDA(cudaStreamSynchronize(ctx->stream));
    DHO2G_CUDA(cudaMemcpy(Cout, c.p, sizeof(float) * M * N, cudaMemcpyDeviceToHost));
  });
}

// Physical operand for the segmented test: X0 (MN x K0), X1 (MN x K1) row-major logical.
static GOp test_operand(dho2g_ctx* ctx, int MN, int K0, int K1, int kseg, const float* X0, const float* X1, int mn_major,
                        DevBuf<bf16>& hi, DevBuf<bf16>& lo, float* sc) {
  std::vector<float> h;
  GOp g{};
  g.mn_major = mn_major;
  if (!mn_major) {  // rows mn: [X0 | 0 .. kseg | X1 | 0]
    const int w = (int)round_up((size_t)(kseg + std::max(K1, 1)), 8);
    h.assign((size_t)MN * w, 0.f);
    for (int r = 0; r < MN; ++r) {
      for (int k = 0; k < K0; ++k) h[(size_t)r * w + k] = X0[(size_t)r * K0 + k];
      for (int k = 0; k < K1; ++k) h[(size_t)r * w + kseg + k] = X1[(size_t)r * K1 + k];
    }
    g.ld = w;
    g.inner = w;
    g.outer = MN;
    g.off_in[0] = 0;
    g.off_in[1] = kseg;
  } else {  // rows k: [X0^T | X1^T], halves of MNp
    const int MNp = (int)round_up((size_t)MN, 8), rows = std::max(K0, K1);
    const int w = 2 * MNp;
    h.assign((size_t)rows * w, 0.f);
    for (int r = 0; r < MN; ++r) {
      for (int k = 0; k < K0; ++k) h[(size_t)k * w + r] = X0[(size_t)r * K0 + k];
      for (int k = 0; k < K1; ++k) h[(size_t)k * w + MNp + r] = X1[(size_t)r * K1 + k];
    }
    g.ld = w;
    g.inner = w;
    g.outer = rows;
    g.off_in[0] = 0;
    g.off_in[1] = MNp;
  }
  DevBuf<float> f(h.size());
  hi.alloc(h.size());
  lo.alloc(h.size());
  // stream-ordered upload: a pageable cudaMemcpy may return before its DMA lands, and the split
  // kernel runs on the library's (non-blocking) stream
  DHO2G_CUDA(cudaMemcpyAsync(f.p, h.data(), sizeof(float) * h.size(), cudaMemcpyHostToDevice, ctx->stream));
  const int rows = (int)(h.size() / g.ld);
  g.f16 = ctx->gemm_f16 ? 1 : 0;
  *sc = g.f16 ? pow2_scale(host_absmax(h.data(), h.size())) : 1.f;
  split_rows_kernel<<<cdiv(h.size(), 256), 256, 0, ctx->stream>>>(f.p, rows, g.ld, g.ld, hi.p, lo.p, g.f16, *sc);
  DHO2G_LAUNCH();
  DHO2G_CUDA(cudaStreamSynchronize(ctx->stream));
  g.hi = hi.p;
  g.lo = lo.p;
  return g;
}

int dho2g_test_gemm_seg(dho2g_ctx* ctx, int M, int N, int K0, int K1, const float* A0, const float* A1,
                        const float* B0, const float* B1, float* Cout, int backend, int a_mn, int b_mn) {
  return guard([&] {
    check_ctx(ctx);
    if (M <= 0 || N <= 0 || K0 <= 0 || K1 < 0) fail(DHO2G_ARGUMENT, "test_gemm_seg: bad shape");
    const int kseg = K1 > 0 ? (int)round_up((size_t)K0, 64) : K0;
    const int K = K1 > 0 ? kseg + K1 : K0;
    DevBuf<bf16> ah, al, bh, bl;
    float sc[2];
    const GOp A = test_operand(ctx, M, K0, K1, kseg, A0, A1, a_mn, ah, al, &sc[0]);
    const GOp B = test_operand(ctx, N, K0, K1, kseg, B0, B1, b_mn, bh, bl, &sc[1]);
    DevBuf<float> c((size_t)M * N), scd(2);
    DHO2G_CUDA(cudaMemcpyAsync(scd.p, sc, sizeof(sc), cudaMemcpyHostToDevice, ctx->stream));
    Epi e{};
    e.mode = EPI_STORE;
    e.M = M;
    e.N = N;
    e.C = c.p;
    e.ldc = N;
    e.alpha = 1.0f;
    e.f16 = A.f16;
    e.sa = A.f16 ? scd.p : nullptr;
    e.sb = A.f16 ? scd.p + 1 : nullptr;
    const int saved = ctx->gemm_backend;
    ctx->gemm_backend = backend;
    try {
      gemm3x(ctx, M, N, K, K1 > 0 ? kseg : K, A, B, e);
    } catch (...) {
      ctx->gemm_backend = saved;
      throw;
    }
    ctx->gemm_backend = saved;
    DHO2G_CUDA(cudaStreamSynchronize(ctx->stream));
    DHO2G_CUDA(cudaMemcpy(Cout, c.p, sizeof(float) * M * N, cudaMemcpyDeviceToHost));
  });
}

}  // extern "C"

// Test hook: every collective wrapper through a 1-rank NCCL communicator on this GPU (the NCCL
// plumbing — run-time binding, communicator init, datatypes, counts, stream order, ledger rows —
// exercised on a one-GPU box). Returns the worst element error in *max_err (exact copies: 0).
int dho2g_test_collectives(dho2g_ctx* ctx, double* max_err) {
  return guard([&] {
    check_ctx(ctx);
    if (ctx->world != 1 || ctx->comm) fail(DHO2G_ARGUMENT, "test_collectives: needs a context without a communicator");
    ncclUniqueId id;
    DHO2G_NCCLCHK(dho2g::nccl().GetUniqueId(&id));
    // the same non-blocking communicator dho2g_comm_init creates (collectives may return ncclInProgress)
    ncclConfig_t cfg = NCCL_CONFIG_INITIALIZER;
    cfg.blocking = 0;
    dho2g::nccl_call(ctx, dho2g::nccl().CommInitRankConfig(&ctx->comm, 1, id, 0, &cfg), "comm_init");
    dho2g::nccl_settle(ctx, "comm_init");
    ctx->nccl_force = true;
    double err = 0.0;
    try {
      cudaStream_t st = ctx->stream;
      const size_t n = 4099;
      std::vector<float> hf(n);
      std::vector<double> hd(n);
      for (size_t i = 0; i < n; ++i) {
        hf[i] = (float)(i % 97) - 48.5f;
        hd[i] = 1.0 / (double)(i + 1);
      }
      DevBuf<float> a(n), b(n);
      DevBuf<double> c(n), e(n);
      DHO2G_CUDA(cudaMemcpyAsync(a.p, hf.data(), n * sizeof(float), cudaMemcpyHostToDevice, st));
      DHO2G_CUDA(cudaMemcpyAsync(c.p, hd.data(), n * sizeof(double), cudaMemcpyHostToDevice, st));
      std::vector<float> of(n);
      std::vector<double> od(n);
      ctx->allgather_f32(a.p, b.p, n);
      DHO2G_CUDA(cudaMemcpyAsync(of.data(), b.p, n * sizeof(float), cudaMemcpyDeviceToHost, st));
      DHO2G_CUDA(cudaStreamSynchronize(st));
      for (size_t i = 0; i < n; ++i) err = std::max(err, (double)std::fabs(of[i] - hf[i]));
      DHO2G_CUDA(cudaMemsetAsync(b.p, 0, n * sizeof(float), st));
      ctx->reduce_scatter_f32(a.p, b.p, n);
      DHO2G_CUDA(cudaMemcpyAsync(of.data(), b.p, n * sizeof(float), cudaMemcpyDeviceToHost, st));
      DHO2G_CUDA(cudaStreamSynchronize(st));
      for (size_t i = 0; i < n; ++i) err = std::max(err, (double)std::fabs(of[i] - hf[i]));
      ctx->allgather_f64(c.p, e.p, n, "all_reduce");
      ctx->allreduce_sum_f64_ordered(c.p, n);
      DHO2G_CUDA(cudaMemcpyAsync(od.data(), c.p, n * sizeof(double), cudaMemcpyDeviceToHost, st));
      DHO2G_CUDA(cudaStreamSynchronize(st));
      for (size_t i = 0; i < n; ++i) err = std::max(err, std::fabs(od[i] - hd[i]));
      DHO2G_CUDA(cudaMemcpyAsync(od.data(), e.p, n * sizeof(double), cudaMemcpyDeviceToHost, st));
      DHO2G_CUDA(cudaStreamSynchronize(st));
      for (size_t i = 0; i < n; ++i) err = std::max(err, std::fabs(od[i] - hd[i]));
      ctx->sync();  // the polled wait of a context with a communicator
    } catch (...) {
      ctx->nccl_force = false;
      if (ctx->comm) dho2g::nccl().CommAbort(ctx->comm);
      ctx->comm = nullptr;
      throw;
    }
    ctx->nccl_force = false;
    dho2g::nccl().CommAbort(ctx->comm);  // non-blocking communicator: abort releases it at once
    ctx->comm = nullptr;
    *max_err = err;
  });
}

// Test hook: the same collectives captured into a CUDA graph (as the multi-rank refresh graph captures
// them), instantiated and replayed twice on a 1-rank NCCL communicator. *max_err: worst element error.
int dho2g_test_collectives_graph(dho2g_ctx* ctx, double* max_err) {
  return guard([&] {
    check_ctx(ctx);
    if (ctx->world != 1 || ctx->comm) fail(DHO2G_ARGUMENT, "test_collectives: needs a context without a communicator");
    ncclUniqueId id;
    DHO2G_NCCLCHK(dho2g::nccl().GetUniqueId(&id));
    ncclConfig_t cfg = NCCL_CONFIG_INITIALIZER;
    cfg.blocking = 0;
    dho2g::nccl_call(ctx, dho2g::nccl().CommInitRankConfig(&ctx->comm, 1, id, 0, &cfg), "comm_init");
    dho2g::nccl_settle(ctx, "comm_init");
    ctx->nccl_force = true;
    cudaGraph_t g = nullptr;
    cudaGraphExec_t ge = nullptr;
    double err = 0.0;
    try {
      cudaStream_t st = ctx->stream;
      const size_t n = 4099;
      std::vector<float> hf(n), of(n);
      std::vector<double> hd(n), od(n);
      for (size_t i = 0; i < n; ++i) {
        hf[i] = (float)(i % 89) - 44.5f;
        hd[i] = 1.0 / (double)(i + 3);
      }
      DevBuf<float> a(n), b(n), c(n);
      DevBuf<double> x(n);
      DHO2G_CUDA(cudaMemcpyAsync(a.p, hf.data(), n * sizeof(float), cudaMemcpyHostToDevice, st));
      DHO2G_CUDA(cudaMemcpyAsync(x.p, hd.data(), n * sizeof(double), cudaMemcpyHostToDevice, st));
      DHO2G_CUDA(cudaStreamSynchronize(st));
      ctx->gather_f64.ensure(n);  // allocation outside the capture
      DHO2G_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
      ctx->allgather_f32(a.p, b.p, n);
      ctx->reduce_scatter_f32(b.p, c.p, n);
      ctx->allreduce_sum_f64_ordered(x.p, n);
      DHO2G_CUDA(cudaStreamEndCapture(st, &g));
      DHO2G_CUDA(cudaGraphInstantiate(&ge, g, 0));
      for (int rep = 0; rep < 2; ++rep) {
        DHO2G_CUDA(cudaMemsetAsync(c.p, 0, n * sizeof(float), st));
        DHO2G_CUDA(cudaGraphLaunch(ge, st));
        DHO2G_CUDA(cudaMemcpyAsync(of.data(), c.p, n * sizeof(float), cudaMemcpyDeviceToHost, st));
        DHO2G_CUDA(cudaMemcpyAsync(od.data(), x.p, n * sizeof(double), cudaMemcpyDeviceToHost, st));
        ctx->sync();
        for (size_t i = 0; i < n; ++i) {
          err = std::max(err, (double)std::fabs(of[i] - hf[i]));
          err = std::max(err, std::fabs(od[i] - hd[i]));
        }
      }
      ctx->bump("test_graph_nodes", 1);
    } catch (...) {
      if (ge) cudaGraphExecDestroy(ge);
      if (g) cudaGraphDestroy(g);
      ctx->nccl_force = false;
      if (ctx->comm) dho2g::nccl().CommAbort(ctx->comm);
      ctx->comm = nullptr;
      throw;
    }
    cudaGraphExecDestroy(ge);
    cudaGraphDestroy(g);
    ctx->nccl_force = false;
    dho2g::nccl().CommAbort(ctx->comm);
    ctx->comm = nullptr;
    *max_err = err;
  });
}

// Test hook: per-CTA timelines of pair-GEMM launches (gemm.cu g_gemm_trace). on = 1 arms a zeroed buffer
// of n_ctas x 4 u64 (each later pair-GEMM launch overwrites it); on = 0 copies it to out and disarms.
int dho2g_test_gemm_trace(dho2g_ctx* ctx, int on, unsigned long long* out, size_t n_ctas) {
  return guard([&] {
    check_ctx(ctx);
    // on: 1 arms the pair kernel's trace (8 stamps per CTA: [0] start, [1] last MMA issued, [2] last segment's
    // accumulator ready, [3] end, [4] head fix-up wait done, [5] head epilogue done), 3 / 4 / 5 the same for
    // R-forward / R-backward / store-epilogue launches only; 2 the single-CTA kernel's (8 stamps per CTA); 0
    // disarms all and copies the buffer out
    static DevBuf<unsigned long long> buf;
    if (on) {
      buf.alloc(n_ctas * 8);
      if (on == 2) gemm_trace1_set(buf.p);
      else gemm_trace_set(buf.p, on >= 3 ? on - 2 : 0);
    } else {
      DHO2G_CUDA(cudaStreamSynchronize(ctx->stream));
      gemm_trace_set(nullptr, 0);
      gemm_trace1_set(nullptr);
      if (out && buf.p)
        DHO2G_CUDA(cudaMemcpy(out, buf.p, std::min(n_ctas * 8, buf.n) * sizeof(unsigned long long),
                              cudaMemcpyDeviceToHost));
    }
  });
}

// Host-level all-gather of `count` doubles per rank through the context's collectives (rank order), e.g.
// for run artifacts that list per-rank accounting. Every rank must call it.
int dho2g_ctx_allgather_host(dho2g_ctx* ctx, const double* in, size_t count, double* out) {
  return guard([&] {
    check_ctx(ctx);
    DevBuf<double> a(std::max<size_t>(count, 1)), b(std::max<size_t>(count * ctx->world, 1));
    DHO2G_CUDA(cudaMemcpyAsync(a.p, in, count * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    ctx->allgather_f64(a.p, b.p, count);
    DHO2G_CUDA(cudaMemcpyAsync(out, b.p, count * ctx->world * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    wait_stream(ctx, ctx->stream);
  });
}
