// Drop-in check from the reference side: the UNMODIFIED reference's own train() (trainer.cpp:273-298)
// run twice on one problem — with its MlpOracle (CPU, fp64) and with GpuMlpOracle (integration/gpu_oracle.hpp
// over libdho2gpu.so). Every Oracle call of the reference loop (mean_gradient's per-worker grads from
// `workers` threads at once, trainer.cpp:92-103; the refresh's HvpFn lambda, trainer.cpp:116, called by
// lanczos_distributed on every worker, dist_lanczos.cpp:79; epoch_end's value / accuracy) goes to the GPU.
// Also one refresh through gpu_refresh() against lanczos_distributed + extract_ese_distributed.
// Prints one JSON line. Built by integration/Makefile into oracle/_ref/drop_in_train (test binary).
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "dho2/collectives.hpp"
#include "dho2/dist_lanczos.hpp"
#include "dho2/rng.hpp"
#include "dho2/trainer.hpp"
#include "gpu_oracle.hpp"

using namespace dho2;

namespace {
std::vector<std::size_t> parse_sizes(const char* s) {
  std::vector<std::size_t> v;
  for (const char* p = s; *p;) {
    v.push_back(std::strtoull(p, const_cast<char**>(&p), 10));
    if (*p == ',') ++p;
  }
  return v;
}
double ms_since(std::chrono::steady_clock::time_point t0) {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
}
std::string rows_json(const TrainResult& r) {
  std::string s = "[";
  for (std::size_t i = 0; i < r.metrics.size(); ++i) {
    char b[96];
    std::snprintf(b, sizeof b, "%s[%.17g,%.17g]", i ? "," : "", r.metrics[i].train_loss, r.metrics[i].train_acc);
    s += b;
  }
  return s + "]";
}
}  // namespace

int main(int argc, char** argv) {
  std::vector<std::size_t> sizes{784, 64, 10};
  std::size_t N = 640, b = 32, curv = 128, k = 6, outer = 2;
  int workers = 4;
  std::string base = "momentum";
  for (int i = 1; i + 1 < argc; i += 2) {
    const std::string a = argv[i];
    if (a == "--sizes") sizes = parse_sizes(argv[i + 1]);
    else if (a == "--N") N = std::strtoull(argv[i + 1], nullptr, 10);
    else if (a == "--b") b = std::strtoull(argv[i + 1], nullptr, 10);
    else if (a == "--curv") curv = std::strtoull(argv[i + 1], nullptr, 10);
    else if (a == "--k") k = std::strtoull(argv[i + 1], nullptr, 10);
    else if (a == "--outer") outer = std::strtoull(argv[i + 1], nullptr, 10);
    else if (a == "--workers") workers = std::atoi(argv[i + 1]);
    else if (a == "--base") base = argv[i + 1];
  }
  const std::size_t D = sizes.front(), K = sizes.back();
  // blobs-D from the reference's Rng: class means N(0,1), x = mu_y + N(0,1), y = i mod K
  Rng rng(7 * 0x2545F4914F6CDD1DULL + 0xB10B5ULL);
  std::vector<double> mu(K * D), X(N * D), y(N);
  for (double& m : mu) m = rng.normal();
  for (std::size_t i = 0; i < N; ++i) {
    y[i] = (double)(i % K);
    for (std::size_t j = 0; j < D; ++j) X[i * D + j] = mu[(i % K) * D + j] + rng.normal();
  }
  auto cpu = std::make_shared<MlpOracle>(sizes, Activation::Tanh, LossKind::SoftmaxCrossEntropy);
  dho2g_ctx* ctx = nullptr;
  gpu_check(dho2g_ctx_create(0, &ctx));
  auto gpu = std::make_shared<GpuMlpOracle>(ctx, sizes, Activation::Tanh, LossKind::SoftmaxCrossEntropy);

  TrainerConfig cfg;
  cfg.kind = TrainerKind::Dho2;
  cfg.base.kind = base == "adamw" ? BaseKind::AdamW : (base == "adam" ? BaseKind::Adam : BaseKind::Momentum);
  cfg.k = k;
  cfg.curvature_batch = curv;
  cfg.outer_rounds = outer;
  cfg.inner_epochs = 1;
  cfg.batch_size = b;
  cfg.seed = 1;
  Problem pc{cpu, Dataset(D, K, X, y, 7), cpu->init_params(1)};
  Problem pg{gpu, Dataset(D, K, X, y, 7), cpu->init_params(1)};  // (pg.oracle released before ctx)

  const bool dbg = std::getenv("DROPIN_DEBUG") != nullptr;
  if (dbg) {  // one call of each Oracle entry point first
    std::vector<std::size_t> i8{0, 1, 2, 3, 4, 5, 6, 7};
    const Batch b8 = pc.dataset.batch(i8);
    std::fprintf(stderr, "value cpu %.9g gpu %.9g\n", cpu->value(pc.w0, b8), gpu->value(pc.w0, b8));
    const Vector g1 = cpu->grad(pc.w0, b8), g2 = gpu->grad(pc.w0, b8);
    std::fprintf(stderr, "grad %.9g %.9g\n", g1[0], g2[0]);
    const Vector h1 = cpu->hvp(pc.w0, g1, b8), h2 = gpu->hvp(pc.w0, g1, b8);
    std::fprintf(stderr, "hvp %.9g %.9g\n", h1[0], h2[0]);
    std::fprintf(stderr, "acc %.9g %.9g\n", *cpu->accuracy(pc.w0, b8), *gpu->accuracy(pc.w0, b8));
  }
  auto t0 = std::chrono::steady_clock::now();
  const TrainResult rc = train(cfg, pc, workers, Schedule::round_robin(), nullptr);
  if (dbg) std::fprintf(stderr, "cpu train done\n");
  const double cpu_ms = ms_since(t0);
  t0 = std::chrono::steady_clock::now();
  const TrainResult rg = train(cfg, pg, workers, Schedule::round_robin(), nullptr);
  const double gpu_ms = ms_since(t0);
  if (dbg) std::fprintf(stderr, "gpu train done\n");

  double num = 0.0, den = 0.0, mx = 0.0;
  for (std::size_t i = 0; i < rc.w_final.size(); ++i) {
    const double d = rg.w_final[i] - rc.w_final[i];
    num += d * d;
    den += rc.w_final[i] * rc.w_final[i];
    mx = std::max(mx, std::fabs(d));
  }

  // one refresh through gpu_refresh vs the reference's lanczos_distributed + extract_ese_distributed on the
  // same operator (the final weights, the first curv samples)
  std::vector<std::size_t> idx(curv);
  for (std::size_t i = 0; i < curv; ++i) idx[i] = i;
  const Batch cb = pc.dataset.batch(idx);
  const std::size_t m = lanczos_budget(k, 0, cpu->dim());
  const Vector& w = rc.w_final;
  EseResult ref;
  run_workers(1, Schedule::round_robin(), nullptr, [&](Worker& wk) {
    const HvpFn h = [&](const Vector& v) { return cpu->hvp(w, v, cb); };
    auto st = lanczos_distributed(wk, m, h, cpu->dim(), 4242, DistLanczosOptions{});
    ref = extract_ese_distributed(wk, st, std::min(k, st.iterations), 0);
  });
  if (dbg) std::fprintf(stderr, "reference refresh done: %zu pairs\n", ref.eigvals.size());
  const EseResult ge = gpu_refresh(ctx, gpu->handle(), w, cb, m, 4242, k, 0, LanczosOptions{});
  if (dbg) std::fprintf(stderr, "gpu refresh done: %zu pairs, %zu rows\n", ge.eigvals.size(), ge.eigvecs.rows());
  double ev_rel = 0.0, pa = 0.0, pb = 0.0, pc2 = 0.0;
  const std::size_t n = cpu->dim(), r = ref.eigvals.size();
  for (std::size_t j = 0; j < r && j < ge.eigvals.size(); ++j)
    ev_rel = std::max(ev_rel, std::fabs(ge.eigvals[j] - ref.eigvals[j]) / std::fabs(ref.eigvals[j]));
  for (std::size_t a = 0; a < r; ++a)
    for (std::size_t c = 0; c < r; ++c) {  // ||V V^T - R R^T||_F^2 = |V^TV|^2 + |R^TR|^2 - 2 |V^TR|^2
      double vv = 0, rr = 0, vr = 0;
      for (std::size_t i = 0; i < n; ++i) {
        vv += ge.eigvecs(i, a) * ge.eigvecs(i, c);
        rr += ref.eigvecs(i, a) * ref.eigvecs(i, c);
        vr += ge.eigvecs(i, a) * ref.eigvecs(i, c);
      }
      pa += vv * vv;
      pb += rr * rr;
      pc2 += vr * vr;
    }
  const double proj = std::sqrt(std::max(pa + pb - 2 * pc2, 0.0));

  std::printf(
      "{\"n\": %zu, \"workers\": %d, \"rows\": [%zu, %zu], \"refreshes\": [%zu, %zu], \"params_rel_l2\": %.6e, "
      "\"params_max_abs\": %.6e, \"cpu_loss_acc\": %s, \"gpu_loss_acc\": %s, \"cpu_ms\": %.1f, \"gpu_ms\": %.1f, "
      "\"refresh_m\": %zu, \"refresh_eig_rel\": %.6e, \"refresh_projector\": %.6e, \"vhat_rows\": %zu}\n",
      cpu->dim(), workers, rc.metrics.size(), rg.metrics.size(), rc.ese_refreshes, rg.ese_refreshes,
      std::sqrt(num / den), mx, rows_json(rc).c_str(), rows_json(rg).c_str(), cpu_ms, gpu_ms, m, ev_rel, proj,
      ge.eigvecs.rows());
  pg.oracle.reset();  // every GpuMlpOracle reference goes before its context
  gpu.reset();
  dho2g_ctx_destroy(ctx);
  return 0;
}
