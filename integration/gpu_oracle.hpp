// Reference-side adapter: the code a maintainer of the reference adds (e.g. as src/gpu_oracle.cpp) to drop
// the B200 path into the UNMODIFIED reference library. It implements the reference's own plugin interfaces
// over the C ABI of libdho2gpu.so (include/dho2gpu.h):
//   GpuMlpOracle        : dho2::Oracle (oracle.hpp:72-80), drop-in for MlpOracle (oracle.hpp:113-141)
//   GpuQuadraticOracle  : dho2::Oracle, drop-in for QuadraticOracle (oracle.hpp:84-102)
//   gpu_refresh()       : lanczos_distributed + extract_ese_distributed (dist_lanczos.hpp:32-41) on a
//                         device-resident operator, returning the reference's EseResult shape (full V_hat)
// Compiled against /root/reference/proj/include by integration/Makefile and exercised by
// integration/drop_in_train.cpp, which runs the reference's own train() with GpuMlpOracle.
#pragma once

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

#include "dho2/dist_lanczos.hpp"
#include "dho2/errors.hpp"
#include "dho2/lanczos.hpp"
#include "dho2/oracle.hpp"
#include "dho2/trainer.hpp"
#include "dho2gpu.h"

namespace dho2 {

// status -> the reference's exception types (errors.hpp:8-36, trainer.hpp:22-24)
inline void gpu_check(int rc) {
  if (rc == DHO2G_OK) return;
  const std::string msg = dho2g_last_error();
  switch (rc) {
    case DHO2G_DIMENSION: throw DimensionError(msg);
    case DHO2G_ARGUMENT: throw ArgumentError(msg);
    case DHO2G_NUMERIC: throw NumericError(msg);
    case DHO2G_DIVERGENCE: throw DivergenceError(msg);
    case DHO2G_DEADLOCK: throw DeadlockError(msg);
    case DHO2G_DIVERGED: throw TrainingDiverged(msg);
    default: throw std::runtime_error("dho2gpu: " + msg);
  }
}

// Drop-in for MlpOracle: same layer sizes, activation, loss and flat parameter layout. Pure and safe for
// concurrent use by all worker threads (oracle.hpp:70-71): the library serialises the calls per context.
class GpuMlpOracle final : public Oracle {
 public:
  GpuMlpOracle(dho2g_ctx* ctx, std::vector<std::size_t> sizes, Activation act, LossKind loss) {
    gpu_check(dho2g_mlp_create(ctx, sizes.data(), (int)sizes.size(), act == Activation::Relu ? 1 : 0,
                               loss == LossKind::Mse ? 1 : 0, &mlp_));
  }
  GpuMlpOracle(const GpuMlpOracle&) = delete;
  GpuMlpOracle& operator=(const GpuMlpOracle&) = delete;
  ~GpuMlpOracle() override { dho2g_mlp_destroy(mlp_); }
  std::size_t dim() const override { return dho2g_mlp_dim(mlp_); }
  double value(const Vector& w, const Batch& b) const override {
    double v;
    gpu_check(dho2g_mlp_value(mlp_, w.data(), b.features.data(), b.labels.data(), b.size, b.n_classes, &v));
    return v;
  }
  Vector grad(const Vector& w, const Batch& b) const override {
    Vector g(dim());
    gpu_check(dho2g_mlp_grad(mlp_, w.data(), b.features.data(), b.labels.data(), b.size, b.n_classes, g.data()));
    return g;
  }
  Vector hvp(const Vector& w, const Vector& v, const Batch& b) const override {
    Vector hv(dim());
    gpu_check(dho2g_mlp_hvp(mlp_, w.data(), v.data(), b.features.data(), b.labels.data(), b.size, b.n_classes,
                            hv.data()));
    return hv;
  }
  std::optional<double> accuracy(const Vector& w, const Batch& b) const override {
    double a;
    gpu_check(dho2g_mlp_accuracy(mlp_, w.data(), b.features.data(), b.labels.data(), b.size, b.n_classes, &a));
    return a < 0 ? std::nullopt : std::optional<double>(a);
  }
  dho2g_mlp* handle() const { return mlp_; }

 private:
  dho2g_mlp* mlp_ = nullptr;
};

// Drop-in for QuadraticOracle: H = Q^T diag(spectrum) Q on the device.
class GpuQuadraticOracle final : public Oracle {
 public:
  GpuQuadraticOracle(dho2g_ctx* ctx, const Vector& spectrum, std::uint64_t rotation_seed) : n_(spectrum.size()) {
    gpu_check(dho2g_op_quadratic(ctx, spectrum.data(), spectrum.size(), rotation_seed, &op_));
  }
  GpuQuadraticOracle(const GpuQuadraticOracle&) = delete;
  GpuQuadraticOracle& operator=(const GpuQuadraticOracle&) = delete;
  ~GpuQuadraticOracle() override { dho2g_op_destroy(op_); }
  std::size_t dim() const override { return n_; }
  Vector apply_h(const Vector& x) const {
    if (x.size() != n_) throw DimensionError("quadratic oracle: dimension mismatch");
    Vector out(n_);
    gpu_check(dho2g_op_apply(op_, x.data(), out.data(), nullptr));
    return out;
  }
  double value(const Vector& w, const Batch&) const override {
    double v;
    gpu_check(dho2g_op_apply(op_, w.data(), nullptr, &v));
    return v;
  }
  Vector grad(const Vector& w, const Batch&) const override { return apply_h(w); }
  Vector hvp(const Vector&, const Vector& v, const Batch&) const override { return apply_h(v); }
  dho2g_op* op() const { return op_; }

 private:
  std::size_t n_;
  dho2g_op* op_ = nullptr;
};

// Drop-in for lanczos_distributed + extract_ese_distributed on the device operator of (w, curvature batch):
// returns the reference's EseResult, the full V_hat assembled on every rank (dist_lanczos.cpp:148-156).
inline EseResult gpu_refresh(dho2g_ctx* ctx, dho2g_mlp* mlp, const Vector& w, const Batch& curv, std::size_t m,
                             std::uint64_t seed, std::size_t k, std::size_t l, const LanczosOptions& o) {
  dho2g_op* op;
  gpu_check(dho2g_op_mlp(ctx, mlp, w.data(), curv.features.data(), curv.labels.data(), curv.size, curv.n_classes,
                         &op));
  dho2g_lanczos_opts lo{o.reorth_safeguard ? 1 : 0, o.safeguard_ratio, o.breakdown_rtol};
  dho2g_lanczos* lz = nullptr;
  dho2g_ese* ese = nullptr;
  EseResult out;
  try {
    gpu_check(dho2g_lanczos_run(ctx, op, m, seed, &lo, &lz));
    if (std::getenv("DROPIN_DEBUG")) std::fprintf(stderr, "gpu_refresh: lanczos ok\n");
    std::size_t iters, sg, b, e;
    int bd;
    gpu_check(dho2g_lanczos_result(lz, nullptr, nullptr, &iters, &bd, &sg, &b, &e));
    const std::size_t keff = std::min(k, iters), leff = std::min(l, iters - keff);  // trainer.cpp:125-126
    gpu_check(dho2g_extract_ese(ctx, lz, keff, leff, &ese));
    out.k = keff;
    out.l = leff;
    out.eigvals.resize(keff + leff);
    gpu_check(dho2g_ese_eigvals(ese, out.eigvals.data()));
    out.eigvecs = TallMatrix(w.size(), keff + leff);
    gpu_check(dho2g_ese_gather(ese, out.eigvecs.data().data()));
  } catch (...) {
    if (ese) dho2g_ese_destroy(ese);
    if (lz) dho2g_lanczos_destroy(lz);
    dho2g_op_destroy(op);
    throw;
  }
  dho2g_ese_destroy(ese);
  dho2g_lanczos_destroy(lz);
  dho2g_op_destroy(op);
  return out;
}

}  // namespace dho2
