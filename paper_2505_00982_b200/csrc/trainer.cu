// Device DHO2 / FOSI / first-order loops (reference: proj/src/trainer.cpp:51-298).
//
// One trainer per GPU (rank). Parameters w_a are replicated (the MLP needs all of them);
// gradient, ADMM primal w, multiplier pi, optimizer moments, Lanczos basis and V_hat are
// row-sharded with Shard::for_rank(n, G, g) semantics. Per step: the rank's logical workers'
// gradient (batched into one GEMM pass) -> reduce_scatter -> fused split update on the shard ->
// all_gather(w_a). Per refresh: curvature batch split over ranks -> sharded Lanczos ->
// replicated eigensolve -> sharded Ritz vectors.
#include <chrono>
#include <cmath>
#include <condition_variable>
#include <cstring>
#include <exception>
#include <mutex>
#include <thread>

#include "internal.h"

using namespace dho2g;

struct MetricsRowH {
  int64_t outer = -1, inner = -1, epoch = 0;
  double loss = 0, acc = NAN, resid = NAN;
  double wallclock = 0;  // modeled clock (trainer.cpp:137-148)
  int refresh = 0;
};

// End-to-end mode (dataset in pinned host memory): the next step's batch is gathered on a host thread
// into a pinned staging slot and copied to the device by the copy engine while the current step
// computes, instead of being read over PCIe by the packing kernel on the critical path. Every step's
// inputs still cross PCIe once, inside the step that precedes it.
struct BatchPrefetch {
  std::thread th;
  std::mutex mu;
  std::condition_variable cv;
  bool quit = false;
  bool pending = false;  // a job is queued or running
  // job
  std::vector<int64_t> idx;
  int slot = 0;
  int64_t epoch = -1;
  size_t round = 0;
  // per slot: what it holds, pinned host staging, device copy, events
  int64_t key_epoch[2] = {-1, -1};
  size_t key_round[2] = {0, 0};
  size_t rows[2] = {0, 0};
  dho2g::HostBuf<float> hx[2], hy[2];
  dho2g::DevBuf<float> dx[2], dy[2];
  cudaEvent_t copied[2] = {}, consumed[2] = {};
  cudaStream_t cs = nullptr;
  std::exception_ptr err;
  int next = 0;
};

struct dho2g_trainer {
  dho2g_ctx* ctx = nullptr;
  dho2g_train_cfg cfg{};
  dho2g_mlp* mlp = nullptr;
  dho2g_op* quad = nullptr;  // QuadraticOracle problem (kind 1 / 4): grad = H w on every batch, no dataset reads
  size_t N = 0, D = 0, ncls = 0, n = 0;
  uint64_t dataset_seed = 0;
  int C = 1;
  int host_resident = 0;
  // dataset
  DevBuf<float> Xd, yd;
  HostBuf<float> Xh, yh;
  const float* Xptr = nullptr;
  const float* yptr = nullptr;
  // sharding
  size_t base = 0, begin = 0, end = 0, rows = 0;
  int c0 = 0, c1 = 1;  // logical workers on this rank
  // parameters / state
  DevBuf<float> w_a_full, g_full, w_a_sh, g_sh, w_sh, pi_sh, hw_sh;
  float* w_a_shard = nullptr;
  float* g_shard = nullptr;
  dho2g_opt opt;
  dho2g_op op;
  dho2g_lanczos lz;
  dho2g_ese ese;
  bool have_ese = false;
  // schedule (trainer.cpp:211-249)
  size_t rounds = 0, k_outer = 0, l_inner = 0, r = 0, iter = 0, epoch_fo = 0;
  bool outer_started = false;
  std::vector<uint64_t> perm;
  int64_t perm_epoch = -1;
  size_t refreshes = 0, safeguards = 0, steps = 0;
  int64_t gs_flops = 0;     // reference accounting (dist_lanczos.cpp:73): 4 active rows + rows per projection
  double sent_host = 0;     // staging for the all-rank floats-sent total of the modeled clock
  cudaEvent_t eval_ev[2] = {};
  double eval_ms_last = 0;  // device time of the last epoch_end evaluation
  size_t eval_count = 0;
  double refresh_ms_last = 0, refresh_ms_total = 0;
  bool refreshed_this_epoch = false;
  bool done = false;
  // staging
  static constexpr int kSlots = 4;
  HostBuf<int64_t> idx_pin[kSlots];
  cudaEvent_t idx_ev[kSlots] = {};
  int slot = 0;
  DevBuf<int64_t> idx_dev;
  DevBuf<double> acc2, stepacc;
  std::vector<MetricsRowH> metrics;
  size_t B_local = 0;
  double h2d_bytes = 0, d2h_bytes = 0;
  std::vector<double> last_eigvals;

  BatchPrefetch pf;

  ~dho2g_trainer() {
    if (pf.th.joinable()) {
      {
        std::lock_guard<std::mutex> lk(pf.mu);
        pf.quit = true;
      }
      pf.cv.notify_all();
      pf.th.join();
    }
    for (int q = 0; q < 2; ++q) {
      if (pf.copied[q]) cudaEventDestroy(pf.copied[q]);
      if (pf.consumed[q]) cudaEventDestroy(pf.consumed[q]);
    }
    if (pf.cs) {
      cudaStreamSynchronize(pf.cs);
      cudaStreamDestroy(pf.cs);
    }
    for (auto& e : idx_ev)
      if (e) cudaEventDestroy(e);
    for (auto& e : eval_ev)
      if (e) cudaEventDestroy(e);
  }

  // this rank's sample indices of one step (trainer.cpp:94-98)
  void step_indices(const std::vector<uint64_t>& pm, size_t round, std::vector<int64_t>& idx) const {
    const size_t b = cfg.batch_size;
    idx.clear();
    idx.reserve((size_t)(c1 - c0) * b);
    for (int c = c0; c < c1; ++c) {
      size_t sb, se;
      shard_range(N, C, c, &sb, &se);
      const size_t len = se - sb;
      for (size_t j = 0; j < b; ++j) idx.push_back((int64_t)pm[sb + (round * b + j) % len]);
    }
  }

  void prefetch_worker() {
    cudaSetDevice(ctx->device);
    for (;;) {
      std::unique_lock<std::mutex> lk(pf.mu);
      pf.cv.wait(lk, [&] { return pf.quit || pf.pending; });
      if (pf.quit) return;
      const int q = pf.slot;
      std::vector<int64_t> idx = pf.idx;
      lk.unlock();
      try {
        DHO2G_CUDA(cudaEventSynchronize(pf.copied[q]));  // the slot's previous host->device copy is done
        const size_t B = idx.size();
        for (size_t j = 0; j < B; ++j) {
          std::memcpy(pf.hx[q].p + j * D, Xh.p + (size_t)idx[j] * D, D * sizeof(float));
          pf.hy[q].p[j] = yh.p[idx[j]];
        }
        DHO2G_CUDA(cudaStreamWaitEvent(pf.cs, pf.consumed[q], 0));  // the step that read the slot is done
        DHO2G_CUDA(cudaMemcpyAsync(pf.dx[q].p, pf.hx[q].p, B * D * sizeof(float), cudaMemcpyHostToDevice, pf.cs));
        DHO2G_CUDA(cudaMemcpyAsync(pf.dy[q].p, pf.hy[q].p, B * sizeof(float), cudaMemcpyHostToDevice, pf.cs));
        DHO2G_CUDA(cudaEventRecord(pf.copied[q], pf.cs));
      } catch (...) {
        lk.lock();
        pf.err = std::current_exception();
        pf.pending = false;
        pf.cv.notify_all();
        continue;
      }
      lk.lock();
      pf.key_epoch[q] = pf.epoch;
      pf.key_round[q] = pf.round;
      pf.rows[q] = idx.size();
      pf.pending = false;
      pf.cv.notify_all();
    }
  }

  void prefetch_init() {
    const size_t cap = (size_t)(c1 - c0) * cfg.batch_size;
    for (int q = 0; q < 2; ++q) {
      pf.hx[q].ensure(std::max<size_t>(cap * D, 1));
      pf.hy[q].ensure(std::max<size_t>(cap, 1));
      pf.dx[q].alloc(std::max<size_t>(cap * D, 1));
      pf.dy[q].alloc(std::max<size_t>(cap, 1));
      DHO2G_CUDA(cudaEventCreateWithFlags(&pf.copied[q], cudaEventDisableTiming));
      DHO2G_CUDA(cudaEventCreateWithFlags(&pf.consumed[q], cudaEventDisableTiming));
      DHO2G_CUDA(cudaEventRecord(pf.copied[q], ctx->stream));
      DHO2G_CUDA(cudaEventRecord(pf.consumed[q], ctx->stream));
    }
    DHO2G_CUDA(cudaStreamCreateWithFlags(&pf.cs, cudaStreamNonBlocking));
    pf.th = std::thread([this] { prefetch_worker(); });
  }

  // queue the gather + copy of the step that will run at (epoch, round)
  void prefetch(int64_t epoch, size_t round) {
    std::vector<uint64_t> pm;
    const std::vector<uint64_t>* use = &perm;
    if (epoch != perm_epoch) {
      pm.resize(N);
      dho2g_epoch_permutation(N, dataset_seed, (uint64_t)epoch, pm.data());
      use = &pm;
    }
    std::vector<int64_t> idx;
    step_indices(*use, round, idx);
    std::unique_lock<std::mutex> lk(pf.mu);
    pf.cv.wait(lk, [&] { return !pf.pending; });
    pf.idx.swap(idx);
    pf.slot = pf.next;
    pf.next ^= 1;
    pf.epoch = epoch;
    pf.round = round;
    pf.key_epoch[pf.slot] = -1;
    pf.pending = true;
    h2d_bytes += (double)pf.idx.size() * (D + 1) * sizeof(float);
    lk.unlock();
    pf.cv.notify_all();
  }

  // the staged slot holding (epoch, round), or -1
  int prefetched(int64_t epoch, size_t round) {
    std::unique_lock<std::mutex> lk(pf.mu);
    pf.cv.wait(lk, [&] { return !pf.pending; });
    if (pf.err) std::rethrow_exception(std::exchange(pf.err, nullptr));
    for (int q = 0; q < 2; ++q)
      if (pf.key_epoch[q] == epoch && pf.key_round[q] == round) return q;
    return -1;
  }

  const int64_t* upload_indices(const std::vector<int64_t>& idx) {
    const int s = slot;
    slot = (slot + 1) % kSlots;
    if (idx_ev[s]) DHO2G_CUDA(cudaEventSynchronize(idx_ev[s]));
    idx_pin[s].ensure(idx.size());
    std::memcpy(idx_pin[s].p, idx.data(), idx.size() * sizeof(int64_t));
    const size_t off = (size_t)s * idx_stride;
    DHO2G_CUDA(cudaMemcpyAsync(idx_dev.p + off, idx_pin[s].p, idx.size() * sizeof(int64_t), cudaMemcpyHostToDevice,
                               ctx->stream));
    if (!idx_ev[s]) DHO2G_CUDA(cudaEventCreateWithFlags(&idx_ev[s], cudaEventDisableTiming));
    DHO2G_CUDA(cudaEventRecord(idx_ev[s], ctx->stream));
    h2d_bytes += (double)idx.size() * sizeof(int64_t);
    return idx_dev.p + off;
  }
  size_t idx_stride = 0;

  void ensure_perm(int64_t epoch) {
    if (perm_epoch == epoch) return;
    perm.resize(N);
    dho2g_epoch_permutation(N, dataset_seed, (uint64_t)epoch, perm.data());  // oracle.cpp:56-62
    perm_epoch = epoch;
  }

  // mean_gradient (trainer.cpp:92-103): this rank's workers' samples batched into one pass;
  // reduce_scatter sums over ranks; the 1/(b C) mean is folded into the output delta.
  void mean_gradient(size_t round) {
    const size_t b = cfg.batch_size;
    std::vector<int64_t> idx;
    step_indices(perm, round, idx);
    B_local = idx.size();
    const double scale = (1.0 / (double)b) * (1.0 / (double)C);
    const int ph = ctx->kt_begin();
    if (quad) {  // QuadraticOracle::grad = apply_h(w) for every worker's batch: the 1/C mean of C equal terms
      quad->apply(w_a_full.p, nullptr, g_shard, begin, rows, base);
      dot_dev(ctx->stream, w_a_shard, g_shard, rows, 0.5, stepacc.p);  // value(w) = w^T H w / 2
      if (ctx->world > 1) ctx->allreduce_sum_f64_ordered(stepacc.p, 1);
      ctx->kt_end(ph, "phase.grad", 0.0);
      return;
    }
    const bool routed = ctx->world > 1 && ctx->hvp_route;  // fused gradient reduce-scatter (peer memory)
    if (B_local > 0) {
      const int q = pf.th.joinable() ? prefetched(perm_epoch, round) : -1;
      mlp_load_weights(mlp, w_a_full.p);
      if (routed) op.route_begin(base);
      if (q >= 0 && pf.rows[q] == B_local) {  // batch staged on the device by the previous step
        DHO2G_CUDA(cudaStreamWaitEvent(ctx->stream, pf.copied[q], 0));
        mlp_grad_dev(mlp, w_a_full.p, pf.dx[q].p, pf.dy[q].p, nullptr, B_local, ncls, scale, g_full.p);
        DHO2G_CUDA(cudaEventRecord(pf.consumed[q], ctx->stream));
      } else {
        const int64_t* di = upload_indices(idx);
        mlp_grad_dev(mlp, w_a_full.p, Xptr, yptr, di, B_local, ncls, scale, g_full.p);
        if (host_resident) h2d_bytes += (double)B_local * (D + 1) * sizeof(float);
      }
      mlp_loss_sum(mlp, B_local, stepacc.p);
    } else if (!routed) {
      DHO2G_CUDA(cudaMemsetAsync(g_full.p, 0, n * sizeof(float), ctx->stream));
    }
    if (routed) op.route_end(g_full.p, B_local == 0, g_shard, rows, base);
    else if (ctx->world > 1) ctx->reduce_scatter_f32(g_full.p, g_shard, base);
    ctx->kt_end(ph, "phase.grad", 0.0);
  }

  // refresh_ese (trainer.cpp:105-135)
  void refresh() {
    const auto t0 = std::chrono::steady_clock::now();
    const int ph = ctx->kt_begin();
    if (!quad) {
      const size_t want = std::min<size_t>(cfg.curvature_batch, N);
      std::vector<uint64_t> all(N);
      dho2g_curvature_indices(N, want, cfg.seed, refreshes, all.data());
      std::vector<int64_t> cidx(all.begin(), all.begin() + want);
      op.idx.ensure_g(want);
      DHO2G_CUDA(cudaMemcpyAsync(op.idx.p, cidx.data(), want * sizeof(int64_t), cudaMemcpyHostToDevice, ctx->stream));
      if (host_resident) h2d_bytes += (double)want * (D + 1) * sizeof(float) + want * sizeof(int64_t);
      op.B = want;
      shard_range(want, ctx->world, ctx->rank, &op.b0, &op.b1);  // HVP batch split across ranks
      op.scale = 1.0 / (double)want;
      op.weights_loaded = false;  // w_a changed since the last refresh
    }
    const size_t m = cfg.lanczos_m ? cfg.lanczos_m : lanczos_budget(cfg.k, cfg.l, n);
    if (m < 1 || m > n) fail(DHO2G_ARGUMENT, "lanczos_distributed: need 1 <= m <= n");
    if (m > (size_t)kMaxLanczos - 1) fail(DHO2G_ARGUMENT, "lanczos: m exceeds the device limit");
    if (lz.m != m) lanczos_alloc(&lz, ctx, n, m);
    lanczos_run_into(&lz, quad ? quad : &op, dho2g_mix_seed(cfg.seed, 0xbeef + refreshes));
    const size_t iters = (size_t)lz.host.iters;
    const size_t keff = std::min(cfg.k, iters);
    const size_t leff = std::min(cfg.l, iters - keff);
    extract_ese_into(ctx, &lz, keff, leff, &ese);
    have_ese = ese.r > 0;
    ctx->kt_end(ph, "phase.refresh", 0.0);
    last_eigvals = ese.eigvals;
    safeguards += (size_t)lz.host.safeguards;
    {
      const int64_t it = (int64_t)lz.host.iters, r = (int64_t)lz.rows;
      gs_flops += 4 * r * (it * (it + 1) / 2) + it * r;                                  // one projection per iteration
      gs_flops += 4 * r * (int64_t)lz.host.sg_cols + (int64_t)lz.host.safeguards * r;  // safeguard passes
    }
    ++refreshes;
    refresh_ms_last = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    refresh_ms_total += refresh_ms_last;
    refreshed_this_epoch = true;
  }

  void allgather_params() {
    if (ctx->world > 1) ctx->allgather_f32(w_a_shard, w_a_full.p, base);
  }

  void update(bool use_pi, double sigma_eff) {
    UpdateArgs a{};
    a.g = g_shard;
    a.pi = use_pi ? pi_sh.p : nullptr;
    a.w_a = w_a_shard;
    a.alpha = cfg.alpha;
    a.sigma = sigma_eff;
    a.floor = cfg.eigval_floor;
    const int ph = ctx->kt_begin();
    split_update(&opt, have_ese ? &ese : nullptr, a);
    allgather_params();
    ctx->kt_end(ph, "phase.update", 0.0);
  }

  // epoch_end (trainer.cpp:150-172)
  void epoch_end(int64_t outer, int64_t inner, int64_t epoch, bool refreshed, bool with_resid) {
    // full-dataset evaluation, timed on the device (reported apart from steps/s)
    if (!eval_ev[0]) {
      DHO2G_CUDA(cudaEventCreate(&eval_ev[0]));
      DHO2G_CUDA(cudaEventCreate(&eval_ev[1]));
    }
    DHO2G_CUDA(cudaEventRecord(eval_ev[0], ctx->stream));
    size_t sb, se;
    shard_range(N, ctx->world, ctx->rank, &sb, &se);
    DHO2G_CUDA(cudaMemsetAsync(acc2.p, 0, 4 * sizeof(double), ctx->stream));
    if (quad) {  // QuadraticOracle::value (oracle.cpp:274-276); accuracy is nullopt
      quad->apply(w_a_full.p, nullptr, hw_sh.p, begin, rows, base);
      dot_dev(ctx->stream, w_a_shard, hw_sh.p, rows, 0.5, acc2.p);
    } else {
      mlp_load_weights(mlp, w_a_full.p);
      const size_t chunk = std::max<size_t>(mlp->Bcap, 1024);
      for (size_t s0 = sb; s0 < se; s0 += chunk) {
        const size_t cnt = std::min(chunk, se - s0);
        if (host_resident) h2d_bytes += (double)cnt * (D + 1) * sizeof(float);
        mlp_eval_dev(mlp, w_a_full.p, Xptr + s0 * D, yptr + s0, nullptr, cnt, ncls, acc2.p);
      }
    }
    if (with_resid) residual_partial(acc2.p + 2);
    sent_host = (double)ctx->ledger_sent;  // this rank's ledger traffic; summed over ranks below
    DHO2G_CUDA(cudaMemcpyAsync(acc2.p + 3, &sent_host, sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    ctx->allreduce_sum_f64_ordered(acc2.p, 4);
    double h[4];
    DHO2G_CUDA(cudaMemcpyAsync(h, acc2.p, 4 * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    wait_stream(ctx, ctx->stream);
    d2h_bytes += 4 * sizeof(double);
    MetricsRowH row;
    row.outer = outer;
    row.inner = inner;
    row.epoch = epoch;
    row.loss = quad ? h[0] : h[0] / (double)N;
    // a non-finite gradient raises the reference's NumericError (optimizer.cpp:38-40) before the loss check
    // can report the divergence it causes
    check_opt_flags(&opt);
    if (!std::isfinite(row.loss))
      fail(DHO2G_DIVERGED, "non-finite loss at epoch " + std::to_string(epoch) + " (trainer " +
                               (cfg.trainer == 2 ? "dho2" : cfg.trainer == 1 ? "fosi" : "sgd") + ")");
    if (ctx->hash_checks && !ranks_all_equal(ctx, device_hash_f32(ctx, w_a_full.p, n)))  // trainer.cpp:157
      fail(DHO2G_DIVERGENCE, "train: parameter replicas diverged at epoch " + std::to_string(epoch));
    row.acc = ncls > 0 ? h[1] / (double)N : NAN;
    row.resid = with_resid ? std::sqrt(h[2]) : NAN;
    row.refresh = refreshed ? 1 : 0;
    {  // modeled_ms (trainer.cpp:137-148): ledger floats x 8 B over the modeled bandwidth + GS flops
      const double world = (double)ctx->world;
      const double bw = cfg.model_bandwidth_gbps > 0 ? cfg.model_bandwidth_gbps : 50.0;
      const double gf = cfg.model_gflops > 0 ? cfg.model_gflops : 10.0;
      row.wallclock = h[3] * 8.0 / (bw * 1.25e5 * world) + (double)gs_flops / (gf * 1e6 * world);
    }
    metrics.push_back(row);
    DHO2G_CUDA(cudaEventRecord(eval_ev[1], ctx->stream));
    DHO2G_CUDA(cudaEventSynchronize(eval_ev[1]));
    float ems = 0.f;
    DHO2G_CUDA(cudaEventElapsedTime(&ems, eval_ev[0], eval_ev[1]));
    eval_ms_last = ems;
    ++eval_count;
    check_opt_flags(&opt);
  }

  void residual_partial(double* out);

  void step_one(bool with_eval) {
    const bool curvature = cfg.k + cfg.l > 0;
    if (cfg.trainer == 2) {  // run_dho2 (trainer.cpp:211-249)
      const bool red = cfg.sigma_zero_reduction != 0;
      const double sigma_state = red ? 1.0 : cfg.sigma;
      const double sigma_eff = red ? 0.0 : cfg.sigma;
      if (k_outer >= cfg.outer_rounds) {
        done = true;
        return;
      }
      if (r == 0 && l_inner == 0) {
        have_ese = false;
        if (curvature) refresh();
        if (red) DHO2G_CUDA(cudaMemcpyAsync(w_sh.p, w_a_shard, rows * sizeof(float), cudaMemcpyDeviceToDevice, ctx->stream));
        else admm_w_update_dev(ctx->stream, rows, sigma_state, w_a_shard, pi_sh.p, w_sh.p);
        DHO2G_CUDA(cudaMemcpyAsync(w_a_shard, w_sh.p, rows * sizeof(float), cudaMemcpyDeviceToDevice, ctx->stream));
        allgather_params();
      }
      const int64_t epoch = (int64_t)(k_outer * cfg.inner_epochs + l_inner);
      ensure_perm(epoch);
      mean_gradient(r);
      update(!red, sigma_eff);
      ++r;
      ++steps;
      if (r == rounds) {
        if (with_eval) epoch_end((int64_t)k_outer, (int64_t)l_inner, epoch, l_inner == 0 && curvature, true);
        r = 0;
        ++l_inner;
        if (l_inner == cfg.inner_epochs) {
          if (!red) admm_dual_update_dev(ctx->stream, rows, sigma_state, w_a_shard, w_sh.p, pi_sh.p);
          l_inner = 0;
          ++k_outer;
          if (k_outer >= cfg.outer_rounds) done = true;
        }
      }
      if (pf.th.joinable() && !done) prefetch((int64_t)(k_outer * cfg.inner_epochs + l_inner), r);
    } else {  // run_fosi (:187-209) / run_first_order (:174-185)
      if (epoch_fo >= cfg.epochs) {
        done = true;
        return;
      }
      if (r == 0) refreshed_this_epoch = false;
      ensure_perm((int64_t)epoch_fo);
      if (cfg.trainer == 1 && curvature) {
        const size_t interval = cfg.refresh_interval > 0 ? cfg.refresh_interval : rounds;
        if (iter % interval == 0) refresh();
      }
      mean_gradient(r);
      update(false, 0.0);
      ++r;
      ++iter;
      ++steps;
      if (r == rounds) {
        if (with_eval) epoch_end(-1, -1, (int64_t)epoch_fo, refreshed_this_epoch, false);
        r = 0;
        ++epoch_fo;
        if (epoch_fo >= cfg.epochs) done = true;
      }
      if (pf.th.joinable() && !done) prefetch((int64_t)epoch_fo, r);
    }
  }
};

namespace {
__global__ void resid_kernel(size_t n, const float* __restrict__ a, const float* __restrict__ b, double* __restrict__ out) {
  __shared__ double sh[32];
  double s = 0.0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const double d = (double)a[i] - (double)b[i];
    s += d * d;
  }
  const double t = block_sum(s, sh);
  if (threadIdx.x == 0) out[blockIdx.x] = t;
}
__global__ void sum_kernel(const double* __restrict__ part, int nb, double* __restrict__ out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double s = 0.0;
    for (int b = 0; b < nb; ++b) s += part[b];
    *out = s;
  }
}
}  // namespace

void dho2g_trainer::residual_partial(double* out) {
  const int nb = (int)std::max<size_t>(1, std::min<size_t>(cdiv(rows, 256), 296));
  DevBuf<double> part(nb);
  resid_kernel<<<nb, 256, 0, ctx->stream>>>(rows, w_a_shard, w_sh.p, part.p);
  sum_kernel<<<1, 32, 0, ctx->stream>>>(part.p, nb, out);
  DHO2G_LAUNCH();
  wait_stream(ctx, ctx->stream);
}

namespace dho2g {

dho2g_trainer* trainer_create(dho2g_ctx* ctx, const dho2g_train_cfg* cfg, dho2g_mlp* mlp, const double* X,
                              const double* y, size_t N, size_t ncls, uint64_t dataset_seed, const double* w0,
                              int workers, int host_resident, dho2g_op* quad) {
  if (!quad && !mlp) fail(DHO2G_ARGUMENT, "train: null oracle");
  if (quad && quad->kind != 1 && quad->kind != 4) fail(DHO2G_ARGUMENT, "train: operator is not a QuadraticOracle");
  if (quad && quad->ctx != ctx) fail(DHO2G_ARGUMENT, "train: operator belongs to another context");
  if (cfg->batch_size == 0) fail(DHO2G_ARGUMENT, "train: batch_size must be >= 1");
  if (workers < 1) fail(DHO2G_ARGUMENT, "run_workers: world_size must be >= 1");
  if (N < (size_t)workers) fail(DHO2G_ARGUMENT, "train: fewer samples than workers");
  if (cfg->trainer == 2 && !cfg->sigma_zero_reduction && cfg->sigma <= 0.0)
    fail(DHO2G_ARGUMENT, "dho2: sigma must be positive");
  auto t = std::make_unique<dho2g_trainer>();
  t->ctx = ctx;
  t->cfg = *cfg;
  ctx->hash_checks = cfg->debug_hash_checks ? 1 : 0;  // trainer.cpp:120 / :128 / :157 (context-wide)
  t->mlp = mlp;
  t->quad = quad;
  t->N = N;
  t->D = quad ? 1 : mlp->sizes[0];
  t->ncls = quad ? 0 : ncls;
  t->n = quad ? quad->n : mlp->dim;
  t->dataset_seed = dataset_seed;
  t->C = workers;
  t->host_resident = host_resident;
  const size_t n = t->n;
  cudaStream_t st = ctx->stream;
  // dataset: fp32 copy, device resident (or pinned + mapped host memory in end-to-end mode)
  std::vector<float> Xf(N * t->D), yf(N);
  for (size_t i = 0; i < N * t->D; ++i) Xf[i] = (float)X[i];
  for (size_t i = 0; i < N; ++i) yf[i] = (float)y[i];
  if (host_resident) {
    t->Xh.ensure(Xf.size());
    t->yh.ensure(yf.size());
    std::memcpy(t->Xh.p, Xf.data(), Xf.size() * sizeof(float));
    std::memcpy(t->yh.p, yf.data(), yf.size() * sizeof(float));
    float *dx = nullptr, *dy = nullptr;
    DHO2G_CUDA(cudaHostGetDevicePointer((void**)&dx, t->Xh.p, 0));
    DHO2G_CUDA(cudaHostGetDevicePointer((void**)&dy, t->yh.p, 0));
    t->Xptr = dx;
    t->yptr = dy;
  } else {
    t->Xd.alloc(Xf.size());
    t->yd.alloc(yf.size());
    // stream-ordered uploads (a pageable cudaMemcpy may return before its DMA lands)
    DHO2G_CUDA(cudaMemcpyAsync(t->Xd.p, Xf.data(), Xf.size() * sizeof(float), cudaMemcpyHostToDevice, ctx->stream));
    DHO2G_CUDA(cudaMemcpyAsync(t->yd.p, yf.data(), yf.size() * sizeof(float), cudaMemcpyHostToDevice, ctx->stream));
    t->Xptr = t->Xd.p;
    t->yptr = t->yd.p;
  }
  // sharding over GPUs
  t->base = cdiv(n, (size_t)ctx->world);
  shard_range(n, ctx->world, ctx->rank, &t->begin, &t->end);
  t->rows = t->end - t->begin;
  {
    size_t a, b;
    shard_range((size_t)workers, ctx->world, ctx->rank, &a, &b);
    t->c0 = (int)a;
    t->c1 = (int)b;
  }
  size_t sb, se;
  shard_range(N, workers, 0, &sb, &se);
  t->rounds = (se - sb + cfg->batch_size - 1) / cfg->batch_size;  // trainer.cpp:66-69
  const size_t full = t->base * ctx->world;
  t->w_a_full.alloc(full);
  t->g_full.alloc(full);
  std::vector<float> w0f(n);
  for (size_t i = 0; i < n; ++i) w0f[i] = (float)w0[i];
  DHO2G_CUDA(cudaMemcpyAsync(t->w_a_full.p, w0f.data(), n * sizeof(float), cudaMemcpyHostToDevice, ctx->stream));
  if (ctx->world == 1) {
    t->w_a_shard = t->w_a_full.p;
    t->g_shard = t->g_full.p;
  } else {
    t->w_a_sh.alloc(std::max<size_t>(t->base, 1));
    t->g_sh.alloc(std::max<size_t>(t->base, 1));
    t->w_a_shard = t->w_a_sh.p;
    t->g_shard = t->g_sh.p;
    if (t->rows)
      DHO2G_CUDA(cudaMemcpyAsync(t->w_a_shard, t->w_a_full.p + t->begin, t->rows * sizeof(float), cudaMemcpyDeviceToDevice, st));
  }
  t->w_sh.alloc(std::max<size_t>(t->base, 1));
  t->pi_sh.alloc(std::max<size_t>(t->base, 1));
  if (t->rows)
    DHO2G_CUDA(cudaMemcpyAsync(t->w_sh.p, t->w_a_shard, t->rows * sizeof(float), cudaMemcpyDeviceToDevice, st));  // make_admm_state
  opt_alloc(&t->opt, ctx, cfg->base, t->rows);
  // SlotMeter names of trainer.cpp:70-71 (w_a replicated; moments row-sharded)
  ctx->meter("w", (int64_t)n);
  ctx->meter("moments", (int64_t)(t->rows * (cfg->base.kind == 0 ? 0 : cfg->base.kind == 1 ? 1 : 2)));
  if (ctx->world > 1) ctx->meter("h_full", (int64_t)n);
  // Steady-state sizes for everything a refresh touches (MLP batch buffers for the larger of the step,
  // curvature and evaluation batches; both GEMM lanes' workspaces; the Lanczos state), so the refresh
  // graph captured right after the first, eager refresh stays valid through the gradient steps.
  {
    const size_t b_step = (size_t)(t->c1 - t->c0) * cfg->batch_size;
    size_t cb, ce;
    shard_range(std::min<size_t>(cfg->curvature_batch, N), ctx->world, ctx->rank, &cb, &ce);
    size_t eb, ee;
    shard_range(N, ctx->world, ctx->rank, &eb, &ee);
    const size_t b_eval = std::min<size_t>(ee - eb, 1024);
    if (!quad) mlp_presize(mlp, std::max(std::max(b_step, ce - cb), std::max(b_eval, (size_t)1)));
    else t->hw_sh.alloc(std::max<size_t>(t->base, 1));
    gemm_presize(ctx);
    if (cfg->trainer != 0 && (cfg->lanczos_m || (cfg->k + cfg->l >= 1 && cfg->k + cfg->l <= n))) {
      const size_t m = cfg->lanczos_m ? cfg->lanczos_m : lanczos_budget(cfg->k, cfg->l, n);
      if (m >= 1 && m <= n && m <= (size_t)kMaxLanczos - 1) lanczos_alloc(&t->lz, ctx, n, m);
    }
  }
  // curvature operator bound to (w_a, curvature batch) like the trainer.cpp:116 lambda
  t->op.ctx = ctx;
  t->op.kind = 0;
  t->op.n = n;
  t->op.mlp = mlp;
  t->op.ncls = ncls;
  t->op.wptr = t->w_a_full.p;
  t->op.Xptr = t->Xptr;
  t->op.yptr = t->yptr;
  if (ctx->world > 1) t->op.hfull.alloc(full);
  t->idx_stride = round_up((size_t)(t->c1 - t->c0) * cfg->batch_size + 1, 64);
  t->idx_dev.alloc(t->idx_stride * dho2g_trainer::kSlots);
  t->acc2.alloc(4);
  t->stepacc.alloc(2);
  if (host_resident && !quad && N > 0) t->prefetch_init();
  wait_stream(ctx, st);
  return t.release();
}

}  // namespace dho2g

namespace dho2g {
dho2g_ctx* trainer_ctx(dho2g_trainer* tr) {
  if (!tr) fail(DHO2G_ARGUMENT, "null trainer");
  return tr->ctx;
}
void trainer_step(dho2g_trainer* tr, size_t steps, int with_eval) {
  for (size_t s = 0; s < steps && !tr->done; ++s) tr->step_one(with_eval != 0);
}
void trainer_run(dho2g_trainer* tr) {
  while (!tr->done) tr->step_one(true);
  tr->ctx->sync();
  check_opt_flags(&tr->opt);
}
void trainer_params(dho2g_trainer* tr, double* w) {
  std::vector<float> f(tr->n);
  DHO2G_CUDA(cudaMemcpyAsync(f.data(), tr->w_a_full.p, tr->n * sizeof(float), cudaMemcpyDeviceToHost, tr->ctx->stream));
  wait_stream(tr->ctx, tr->ctx->stream);
  for (size_t i = 0; i < tr->n; ++i) w[i] = f[i];
}
size_t trainer_rows(dho2g_trainer* tr) { return tr->metrics.size(); }
void trainer_metrics_ex(dho2g_trainer* tr, size_t max_rows, int64_t* outer, int64_t* inner, double* wallclock) {
  for (size_t i = 0; i < tr->metrics.size() && i < max_rows; ++i) {
    const auto& m = tr->metrics[i];
    if (outer) outer[i] = m.outer;
    if (inner) inner[i] = m.inner;
    if (wallclock) wallclock[i] = m.wallclock;
  }
}
void trainer_metrics(dho2g_trainer* tr, size_t max_rows, double* loss, double* acc, double* resid, int64_t* epoch,
                     int* refresh) {
  for (size_t i = 0; i < tr->metrics.size() && i < max_rows; ++i) {
    const auto& m = tr->metrics[i];
    if (loss) loss[i] = m.loss;
    if (acc) acc[i] = m.acc;
    if (resid) resid[i] = m.resid;
    if (epoch) epoch[i] = m.epoch;
    if (refresh) refresh[i] = m.refresh;
  }
}
double trainer_last_loss(dho2g_trainer* tr) {
  double h[2] = {0, 0};
  DHO2G_CUDA(cudaMemcpyAsync(h, tr->stepacc.p, 2 * sizeof(double), cudaMemcpyDeviceToHost, tr->ctx->stream));
  wait_stream(tr->ctx, tr->ctx->stream);
  tr->d2h_bytes += 2 * sizeof(double);
  if (tr->quad) return h[0];
  return tr->B_local ? h[0] / (double)tr->B_local : 0.0;
}
bool trainer_stat(dho2g_trainer* tr, const std::string& key, double* v) {
  if (key == "refreshes") *v = (double)tr->refreshes;
  else if (key == "safeguard_passes") *v = (double)tr->safeguards;
  else if (key == "gs_flops") *v = (double)tr->gs_flops;
  else if (key == "eval_ms_last") *v = tr->eval_ms_last;
  else if (key == "eval_count") *v = (double)tr->eval_count;
  else if (key == "steps") *v = (double)tr->steps;
  else if (key == "refresh_ms_last") *v = tr->refresh_ms_last;
  else if (key == "refresh_ms_total") *v = tr->refresh_ms_total;
  else if (key == "lanczos_ms_last") *v = tr->lz.ms;
  else if (key == "h2d_bytes") *v = tr->h2d_bytes;
  else if (key == "d2h_bytes") *v = tr->d2h_bytes;
  else if (key == "rounds_per_epoch") *v = (double)tr->rounds;
  else if (key == "batch_local") *v = (double)tr->B_local;
  else if (key == "done") *v = tr->done ? 1.0 : 0.0;
  else if (key == "lanczos_m") *v = (double)tr->lz.m;
  else if (key == "lanczos_iters") *v = (double)tr->lz.host.iters;
  else if (key == "ese_count") *v = (double)(tr->have_ese ? tr->ese.r : 0);
  else return false;
  return true;
}
void trainer_eigvals(dho2g_trainer* tr, double* vals, size_t* count) {
  *count = tr->last_eigvals.size();
  if (vals)
    for (size_t i = 0; i < tr->last_eigvals.size(); ++i) vals[i] = tr->last_eigvals[i];
}
void trainer_destroy(dho2g_trainer* tr) { delete tr; }
}  // namespace dho2g
