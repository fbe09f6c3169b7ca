// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// A thin extern "C" shim over the UNMODIFIED reference library
// (/root/reference/proj/src/*.cpp, compiled in place by oracle/Makefile into
// oracle/_ref/libdho2ref.so). It lets the Python tests, __graft_entry__.smoke()
// and bench.py's cpu_baseline / --impl reference leg call the reference's own
// C++ API with plain pointers. Nothing here re-implements arithmetic: every
// number comes from the reference functions named in each comment.
#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <memory>
#include <numeric>
#include <string>
#include <vector>

#include <json.hpp>

#include "dho2/collectives.hpp"
#include "dho2/dist_lanczos.hpp"
#include "dho2/errors.hpp"
#include "dho2/harness.hpp"
#include "dho2/kernels.hpp"
#include "dho2/lanczos.hpp"
#include "dho2/linalg.hpp"
#include "dho2/optimizer.hpp"
#include "dho2/oracle.hpp"
#include "dho2/rng.hpp"
#include "dho2/trainer.hpp"

using namespace dho2;

namespace {

thread_local std::string g_err;

// status codes shared with include/dho2gpu.h (DHO2G_*)
enum { OK = 0, E_DIMENSION = 1, E_ARGUMENT = 2, E_NUMERIC = 3, E_DIVERGENCE = 4, E_DEADLOCK = 5,
       E_OTHER = 9 };

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return OK;
  } catch (const DimensionError& e) {
    g_err = e.what();
    return E_DIMENSION;
  } catch (const ArgumentError& e) {
    g_err = e.what();
    return E_ARGUMENT;
  } catch (const DivergenceError& e) {
    g_err = e.what();
    return E_DIVERGENCE;
  } catch (const DeadlockError& e) {
    g_err = e.what();
    return E_DEADLOCK;
  } catch (const NumericError& e) {
    g_err = e.what();
    return E_NUMERIC;
  } catch (const std::exception& e) {
    g_err = e.what();
    return E_OTHER;
  }
}

Batch make_batch(const double* X, const double* y, std::size_t B, std::size_t D, std::size_t ncls) {
  Batch b;
  b.size = B;
  b.feature_dim = D;
  b.n_classes = ncls;
  b.features.assign(X, X + B * D);
  b.labels.assign(y, y + B);
  return b;
}

std::vector<std::size_t> sizes_vec(const std::size_t* sizes, int nl) {
  return std::vector<std::size_t>(sizes, sizes + nl);
}

Activation act_of(int a) { return a == 1 ? Activation::Relu : Activation::Tanh; }
LossKind loss_of(int l) { return l == 1 ? LossKind::Mse : LossKind::SoftmaxCrossEntropy; }

}  // namespace

extern "C" {

struct ref_op {
  int kind;  // 0 dense symmetric (n*n, column-major), 1 diagonal spectrum, 2 MLP hvp
  std::size_t n;
  const double* mat;
  const std::size_t* sizes;
  int n_sizes;
  int act;
  int loss;
  const double* w;
  const double* X;
  const double* y;
  std::size_t B;
  std::size_t ncls;
  std::uint64_t rot_seed;  // kind 1: QuadraticOracle(mat, rot_seed)
  const double* rot;       // (the port's precomputed rotation; unused here)
};

struct ref_base_cfg {
  int kind;  // 0 sgd 1 momentum 2 adam 3 adamw
  double lr, weight_decay, beta1, beta2, eps, momentum;
};

struct ref_train_cfg {
  int trainer;  // 0 sgd 1 fosi 2 dho2
  ref_base_cfg base;
  std::size_t k, l;
  double alpha, eigval_floor;
  std::size_t refresh_interval, curvature_batch;
  int reorth_safeguard;
  double safeguard_ratio, breakdown_rtol;
  double sigma;
  std::size_t outer_rounds, inner_epochs;
  int sigma_zero_reduction;
  std::size_t epochs, batch_size;
  std::uint64_t seed;
};

const char* ref_last_error() { return g_err.c_str(); }
void ref_set_parallel(int on) { kernels::set_parallel(on != 0); }
int ref_max_threads() { return kernels::max_threads(); }

// rng.hpp:14-68
void ref_rng_u64(std::uint64_t seed, std::size_t n, std::uint64_t* out) {
  Rng r(seed);
  for (std::size_t i = 0; i < n; ++i) out[i] = r.next_u64();
}
void ref_rng_normal(std::uint64_t seed, std::size_t n, double* out) {
  Rng r(seed);
  for (std::size_t i = 0; i < n; ++i) out[i] = r.normal();
}
void ref_rng_uniform(std::uint64_t seed, std::size_t n, double* out) {
  Rng r(seed);
  for (std::size_t i = 0; i < n; ++i) out[i] = r.uniform();
}
void ref_rng_shuffle_iota(std::uint64_t seed, std::size_t n, std::uint64_t* out) {
  std::vector<std::size_t> v(n);
  std::iota(v.begin(), v.end(), 0);
  Rng r(seed);
  r.shuffle(v);
  for (std::size_t i = 0; i < n; ++i) out[i] = v[i];
}

// collectives.cpp:10-20
int ref_shard(std::size_t n, int world, int rank, std::size_t* begin, std::size_t* end) {
  return guarded([&] {
    const Shard s = Shard::for_rank(n, world, rank);
    *begin = s.begin;
    *end = s.end;
  });
}

// lanczos.cpp:10-16
int ref_lanczos_budget(std::size_t k, std::size_t l, std::size_t n, std::size_t* m) {
  return guarded([&] { *m = lanczos_budget(k, l, n); });
}

// lanczos.cpp:18-26
int ref_seeded_unit_gaussian(std::size_t n, std::uint64_t seed, double* out) {
  return guarded([&] {
    const Vector v = seeded_unit_gaussian(n, seed);
    std::copy(v.begin(), v.end(), out);
  });
}

// oracle.cpp:56-62
int ref_epoch_permutation(std::size_t N, std::uint64_t shuffle_seed, std::uint64_t epoch,
                          std::uint64_t* out) {
  return guarded([&] {
    std::vector<double> f(N, 0.0), y(N, 0.0);
    const Dataset ds(1, 0, f, y, shuffle_seed);
    const auto p = ds.epoch_permutation(epoch);
    for (std::size_t i = 0; i < N; ++i) out[i] = p[i];
  });
}

// oracle.cpp:304-324
int ref_mlp_dim(const std::size_t* sizes, int nl, std::size_t* dim) {
  return guarded([&] {
    const MlpOracle mlp(sizes_vec(sizes, nl), Activation::Tanh, LossKind::SoftmaxCrossEntropy);
    *dim = mlp.dim();
  });
}

// oracle.cpp:386-394
int ref_mlp_init(const std::size_t* sizes, int nl, std::uint64_t seed, double* w) {
  return guarded([&] {
    const MlpOracle mlp(sizes_vec(sizes, nl), Activation::Tanh, LossKind::SoftmaxCrossEntropy);
    const Vector v = mlp.init_params(seed);
    std::copy(v.begin(), v.end(), w);
  });
}

// oracle.cpp:400-449
int ref_mlp_value(const std::size_t* sizes, int nl, int act, int loss, const double* w,
                  const double* X, const double* y, std::size_t B, std::size_t ncls, double* out) {
  return guarded([&] {
    const MlpOracle mlp(sizes_vec(sizes, nl), act_of(act), loss_of(loss));
    const Vector wv(w, w + mlp.dim());
    *out = mlp.value(wv, make_batch(X, y, B, sizes[0], ncls));
  });
}

// oracle.cpp:451-522
int ref_mlp_grad(const std::size_t* sizes, int nl, int act, int loss, const double* w,
                 const double* X, const double* y, std::size_t B, std::size_t ncls, double* g) {
  return guarded([&] {
    const MlpOracle mlp(sizes_vec(sizes, nl), act_of(act), loss_of(loss));
    const Vector wv(w, w + mlp.dim());
    const Vector out = mlp.grad(wv, make_batch(X, y, B, sizes[0], ncls));
    std::copy(out.begin(), out.end(), g);
  });
}

// oracle.cpp:524-647
int ref_mlp_hvp(const std::size_t* sizes, int nl, int act, int loss, const double* w,
                const double* v, const double* X, const double* y, std::size_t B, std::size_t ncls,
                double* hv) {
  return guarded([&] {
    const MlpOracle mlp(sizes_vec(sizes, nl), act_of(act), loss_of(loss));
    const Vector wv(w, w + mlp.dim());
    const Vector vv(v, v + mlp.dim());
    const Vector out = mlp.hvp(wv, vv, make_batch(X, y, B, sizes[0], ncls));
    std::copy(out.begin(), out.end(), hv);
  });
}

// oracle.cpp:649-685
int ref_mlp_accuracy(const std::size_t* sizes, int nl, int act, int loss, const double* w,
                     const double* X, const double* y, std::size_t B, std::size_t ncls,
                     double* acc) {
  return guarded([&] {
    const MlpOracle mlp(sizes_vec(sizes, nl), act_of(act), loss_of(loss));
    const Vector wv(w, w + mlp.dim());
    const auto a = mlp.accuracy(wv, make_batch(X, y, B, sizes[0], ncls));
    *acc = a ? *a : -1.0;
  });
}

// linalg.cpp:140-226
int ref_tridiag_eig(std::size_t n, const double* diag, const double* off, double* vals,
                    double* vecs) {
  return guarded([&] {
    TridiagMatrix b(n);
    std::copy(diag, diag + n, b.diag.begin());
    if (n > 1) std::copy(off, off + n - 1, b.offdiag.begin());
    const auto e = linalg::tridiag_eig(b);
    std::copy(e.values.begin(), e.values.end(), vals);
    std::copy(e.vectors.data().begin(), e.vectors.data().end(), vecs);
  });
}

// linalg.cpp:117-134 (coefficient pass + update pass over the leading columns)
int ref_project_out(std::size_t n, std::size_t cols, const double* d, std::size_t active,
                    const double* h, double* out) {
  return guarded([&] {
    TallMatrix dm(n, cols);
    std::copy(d, d + n * cols, dm.data().begin());
    const Vector hv(h, h + n);
    const Vector r = linalg::project_out(hv, dm, active);
    std::copy(r.begin(), r.end(), out);
  });
}

static HvpFn make_hvp(const ref_op* op, std::shared_ptr<void>& keep) {
  if (op->kind == 0) {
    auto m = std::make_shared<std::vector<double>>(op->mat, op->mat + op->n * op->n);
    keep = m;
    const std::size_t n = op->n;
    return [m, n](const Vector& v) {
      Vector out(n, 0.0);
      for (std::size_t i = 0; i < n; ++i) {
        double acc = 0.0;
        for (std::size_t j = 0; j < n; ++j) acc += (*m)[j * n + i] * v[j];
        out[i] = acc;
      }
      return out;
    };
  }
  if (op->kind == 1) {
    // QuadraticOracle(spectrum, rot_seed).apply_h (oracle.cpp:262-272); seed 0 is the
    // bench_main.cpp:84-88 diagonal operator
    auto q = std::make_shared<QuadraticOracle>(Vector(op->mat, op->mat + op->n), op->rot_seed);
    keep = q;
    return [q](const Vector& v) { return q->apply_h(v); };
  }
  struct MlpCtx {
    MlpOracle mlp;
    Vector w;
    Batch batch;
  };
  auto c = std::make_shared<MlpCtx>(MlpCtx{
      MlpOracle(sizes_vec(op->sizes, op->n_sizes), act_of(op->act), loss_of(op->loss)),
      Vector(), make_batch(op->X, op->y, op->B, op->sizes[0], op->ncls)});
  c->w.assign(op->w, op->w + c->mlp.dim());
  keep = c;
  return [c](const Vector& v) { return c->mlp.hvp(c->w, v, c->batch); };
}

// dist_lanczos.cpp:31-119 + :121-158 under run_workers (collectives.cpp:461), round-robin schedule
int ref_lanczos(const ref_op* op, int workers, std::size_t m, std::uint64_t seed, int safeguard,
                double safeguard_ratio, double breakdown_rtol, std::size_t k, std::size_t l,
                double* diag, double* off, std::size_t* iters, int* breakdown,
                std::size_t* safeguard_passes, double* basis, double* eigvals, double* eigvecs,
                double* wall_ms) {
  return guarded([&] {
    std::shared_ptr<void> keep;
    const HvpFn hvp = make_hvp(op, keep);
    const std::size_t n = op->n;
    DistLanczosOptions opts;
    opts.lanczos.reorth_safeguard = safeguard != 0;
    opts.lanczos.safeguard_ratio = safeguard_ratio;
    opts.lanczos.breakdown_rtol = breakdown_rtol;
    const auto t0 = std::chrono::steady_clock::now();
    run_workers(workers, Schedule::round_robin(), nullptr, [&](Worker& w) {
      auto st = lanczos_distributed(w, m, hvp, n, seed, opts);
      TallMatrix full;
      if (basis != nullptr) full = w.gather_rows(st.basis_shard, st.shard);
      EseResult ese;
      if (k + l > 0) ese = extract_ese_distributed(w, st, std::min(k, st.iterations),
                                                  std::min(l, st.iterations - std::min(k, st.iterations)));
      if (w.rank() == 0) {
        std::fill(diag, diag + m + 1, 0.0);
        std::fill(off, off + m, 0.0);
        std::copy(st.tridiag.diag.begin(), st.tridiag.diag.end(), diag);
        std::copy(st.tridiag.offdiag.begin(), st.tridiag.offdiag.end(), off);
        *iters = st.iterations;
        *breakdown = st.breakdown ? 1 : 0;
        *safeguard_passes = st.safeguard_passes;
        if (basis != nullptr) std::copy(full.data().begin(), full.data().end(), basis);
        if (k + l > 0) {
          std::copy(ese.eigvals.begin(), ese.eigvals.end(), eigvals);
          std::copy(ese.eigvecs.data().begin(), ese.eigvecs.data().end(), eigvecs);
        }
      }
    });
    const auto t1 = std::chrono::steady_clock::now();
    if (wall_ms) *wall_ms = std::chrono::duration<double, std::milli>(t1 - t0).count();
  });
}

static BaseConfig base_cfg(const ref_base_cfg* c) {
  BaseConfig b;
  b.kind = static_cast<BaseKind>(c->kind);
  b.lr = c->lr;
  b.weight_decay = c->weight_decay;
  b.beta1 = c->beta1;
  b.beta2 = c->beta2;
  b.eps = c->eps;
  b.momentum = c->momentum;
  return b;
}

// optimizer.cpp:37-71 — T consecutive steps from zero moments
int ref_base_steps(const ref_base_cfg* c, std::size_t n, int T, const double* g, const double* w,
                   double* d_out) {
  return guarded([&] {
    BaseOptimizer opt(base_cfg(c), n);
    const Vector wv(w, w + n);
    for (int t = 0; t < T; ++t) {
      const Vector gv(g + static_cast<std::size_t>(t) * n, g + static_cast<std::size_t>(t + 1) * n);
      const Vector d = opt.step(gv, wv);
      std::copy(d.begin(), d.end(), d_out + static_cast<std::size_t>(t) * n);
    }
  });
}

// optimizer.cpp:81-129 — T consecutive fosi/admm splits sharing one BaseOptimizer.
// pi == nullptr selects fosi_deltas. w advances by base+newton after every step when
// advance != 0 (the trainer's w_a += d.base; w_a += d.newton, trainer.cpp:240-241).
int ref_deltas_seq(const ref_base_cfg* c, std::size_t n, std::size_t r, const double* eigvals,
                   const double* eigvecs, int T, const double* g, const double* pi, double* w,
                   double alpha, double sigma, double floor, int advance, double* newton_out,
                   double* base_out) {
  return guarded([&] {
    BaseOptimizer opt(base_cfg(c), n);
    EseResult ese;
    ese.k = r;
    ese.eigvals.assign(eigvals, eigvals + r);
    ese.eigvecs = TallMatrix(n, r);
    std::copy(eigvecs, eigvecs + n * r, ese.eigvecs.data().begin());
    Vector wv(w, w + n);
    const Vector piv = pi ? Vector(pi, pi + n) : Vector();
    for (int t = 0; t < T; ++t) {
      const Vector gv(g + static_cast<std::size_t>(t) * n, g + static_cast<std::size_t>(t + 1) * n);
      const Deltas d = pi ? admm_deltas(gv, piv, ese, opt, wv, alpha, sigma, floor)
                          : fosi_deltas(gv, ese, opt, wv, alpha, floor);
      if (newton_out) std::copy(d.newton.begin(), d.newton.end(), newton_out + t * n);
      if (base_out) std::copy(d.base.begin(), d.base.end(), base_out + t * n);
      if (advance) {
        linalg::axpy(1.0, d.base, wv);
        if (ese.count() > 0) linalg::axpy(1.0, d.newton, wv);
      }
    }
    std::copy(wv.begin(), wv.end(), w);
  });
}

// Parity-at-scale input generator (tests/scale_inputs.py h24_np / unif_np, same bits): a 24-bit counter
// hash, so a 100,989,962 x 32 V_hat can be built inside this process (no second 26 GB copy) and on the
// device by the GPU test. Values are 24-bit integers times powers of two: exact in fp32.
static inline std::int64_t h24(std::int64_t i, std::int64_t salt) {
  const std::int64_t M = 0xFFFFFF;
  std::int64_t x = ((i & M) * 0x9E3779 + (i >> 24) * 0x7F4A7D + salt * 0x2545F5 + 0x1234) & M;
  x = ((x ^ (x >> 12)) * 0x2C1B3D) & M;
  x = ((x ^ (x >> 11)) * 0x297A2D) & M;
  return x ^ (x >> 13);
}
static inline double unif24(std::int64_t i, std::int64_t salt, double scale) {
  return static_cast<double>(h24(i, salt) - (1 << 23)) * (scale * 0x1p-23);
}

// optimizer.cpp:81-129 on hashed inputs: T consecutive admm_deltas (one BaseOptimizer, w advanced by
// base + newton after each step as in trainer.cpp:240-241). V_hat[:, j] = unif(i, salt_v + j) * v_scale,
// g_t = unif(i, salt_g + t) * g_scale, pi = unif(i, salt_pi) * pi_scale, w0 = unif(i, salt_w) * w_scale.
// Returns newton_t, base_t and w after the T steps at the n_idx sampled indices, plus full-vector
// sums of squares (norm2 per step for newton and base).
int ref_deltas_hashed(const ref_base_cfg* c, std::size_t n, std::size_t r, const double* eigvals, int T,
                      double alpha, double sigma, double floor, std::int64_t salt_v, double v_scale,
                      std::int64_t salt_g, double g_scale, std::int64_t salt_pi, double pi_scale,
                      std::int64_t salt_w, double w_scale, const std::int64_t* idx, std::size_t n_idx,
                      double* newton_at, double* base_at, double* w_at, double* sq_newton, double* sq_base) {
  return guarded([&] {
    BaseOptimizer opt(base_cfg(c), n);
    EseResult ese;
    ese.k = r;
    ese.eigvals.assign(eigvals, eigvals + r);
    ese.eigvecs = TallMatrix(n, r);
    double* V = ese.eigvecs.data().data();
#pragma omp parallel for schedule(static)
    for (std::int64_t i = 0; i < static_cast<std::int64_t>(n); ++i)
      for (std::size_t j = 0; j < r; ++j) V[j * n + i] = unif24(i, salt_v + static_cast<std::int64_t>(j), v_scale);
    Vector wv(n), piv(n), gv(n);
#pragma omp parallel for schedule(static)
    for (std::int64_t i = 0; i < static_cast<std::int64_t>(n); ++i) {
      wv[i] = unif24(i, salt_w, w_scale);
      piv[i] = unif24(i, salt_pi, pi_scale);
    }
    for (int t = 0; t < T; ++t) {
#pragma omp parallel for schedule(static)
      for (std::int64_t i = 0; i < static_cast<std::int64_t>(n); ++i) gv[i] = unif24(i, salt_g + t, g_scale);
      const Deltas d = admm_deltas(gv, piv, ese, opt, wv, alpha, sigma, floor);
      for (std::size_t q = 0; q < n_idx; ++q) {
        newton_at[t * n_idx + q] = d.newton[idx[q]];
        base_at[t * n_idx + q] = d.base[idx[q]];
      }
      sq_newton[t] = linalg::dot(d.newton, d.newton);
      sq_base[t] = linalg::dot(d.base, d.base);
      linalg::axpy(1.0, d.base, wv);
      linalg::axpy(1.0, d.newton, wv);
    }
    for (std::size_t q = 0; q < n_idx; ++q) w_at[q] = wv[idx[q]];
  });
}

// optimizer.cpp:131-154
int ref_admm_round(std::size_t n, double sigma, const double* w_a, const double* pi, double* w_out,
                   const double* w_a_after, double* pi_out) {
  return guarded([&] {
    AdmmState st = make_admm_state(Vector(w_a, w_a + n), sigma);
    st.pi.assign(pi, pi + n);
    admm_w_update(st);
    std::copy(st.w.begin(), st.w.end(), w_out);
    if (w_a_after && pi_out) {
      st.w_a.assign(w_a_after, w_a_after + n);
      admm_dual_update(st);
      std::copy(st.pi.begin(), st.pi.end(), pi_out);
    }
  });
}

// trainer.cpp:273-298 — full trajectory on an MLP problem over a caller-supplied dataset
int ref_train_mlp(const ref_train_cfg* c, const std::size_t* sizes, int nl, int act, int loss,
                  const double* X, const double* y, std::size_t N, std::size_t ncls,
                  std::uint64_t dataset_seed, const double* w0, int workers, double* w_final,
                  std::size_t max_rows, std::size_t* n_rows, double* row_loss, double* row_acc,
                  double* row_resid, std::int64_t* row_epoch, std::size_t* refreshes,
                  std::size_t* safeguards, double* wall_ms) {
  return guarded([&] {
    TrainerConfig cfg;
    cfg.kind = static_cast<TrainerKind>(c->trainer);
    cfg.base = base_cfg(&c->base);
    cfg.k = c->k;
    cfg.l = c->l;
    cfg.alpha = c->alpha;
    cfg.eigval_floor = c->eigval_floor;
    cfg.refresh_interval = c->refresh_interval;
    cfg.curvature_batch = c->curvature_batch;
    cfg.lanczos.reorth_safeguard = c->reorth_safeguard != 0;
    cfg.lanczos.safeguard_ratio = c->safeguard_ratio;
    cfg.lanczos.breakdown_rtol = c->breakdown_rtol;
    cfg.sigma = c->sigma;
    cfg.outer_rounds = c->outer_rounds;
    cfg.inner_epochs = c->inner_epochs;
    cfg.sigma_zero_reduction = c->sigma_zero_reduction != 0;
    cfg.epochs = c->epochs;
    cfg.batch_size = c->batch_size;
    cfg.seed = c->seed;
    Problem p;
    auto mlp = std::make_shared<MlpOracle>(sizes_vec(sizes, nl), act_of(act), loss_of(loss));
    p.w0.assign(w0, w0 + mlp->dim());
    p.oracle = mlp;
    p.dataset = Dataset(sizes[0], ncls, std::vector<double>(X, X + N * sizes[0]),
                        std::vector<double>(y, y + N), dataset_seed);
    const auto res = train(cfg, p, workers, Schedule::round_robin(), nullptr);
    std::copy(res.w_final.begin(), res.w_final.end(), w_final);
    *n_rows = res.metrics.size();
    for (std::size_t i = 0; i < res.metrics.size() && i < max_rows; ++i) {
      row_loss[i] = res.metrics[i].train_loss;
      row_acc[i] = res.metrics[i].train_acc;
      row_resid[i] = res.metrics[i].residual_norm;
      row_epoch[i] = res.metrics[i].epoch;
    }
    *refreshes = res.ese_refreshes;
    *safeguards = res.safeguard_passes;
    *wall_ms = res.raw_wallclock_ms;
  });
}

// QuadraticOracle (oracle.cpp:233-286): rotation, apply_h, value
int ref_quadratic_rotation(std::size_t n, std::uint64_t rotation_seed, double* Q) {
  return guarded([&] {
    const QuadraticOracle q(Vector(n, 1.0), rotation_seed);
    if (q.rotated()) std::copy(q.rotation().data().begin(), q.rotation().data().end(), Q);
  });
}

int ref_quadratic_apply(const double* spec, std::size_t n, std::uint64_t rotation_seed, const double* x,
                        double* out, double* value) {
  return guarded([&] {
    const QuadraticOracle q(Vector(spec, spec + n), rotation_seed);
    const Vector xv(x, x + n);
    const Vector h = q.apply_h(xv);
    std::copy(h.begin(), h.end(), out);
    if (value) *value = q.value(xv, Dataset::dummy(1).full_batch());
  });
}

// trainer.cpp:273-298 on Problem{QuadraticOracle, Dataset::dummy(N), w0} (test_trainer.cpp:14-21)
int ref_train_quadratic(const ref_train_cfg* c, const double* spec, std::size_t n, std::uint64_t rotation_seed,
                        std::size_t N, const double* w0, int workers, double* w_final, std::size_t max_rows,
                        std::size_t* n_rows, double* row_loss, double* row_acc, double* row_resid,
                        std::int64_t* row_epoch, std::size_t* refreshes, std::size_t* safeguards,
                        double* wall_ms) {
  return guarded([&] {
    TrainerConfig cfg;
    cfg.kind = static_cast<TrainerKind>(c->trainer);
    cfg.base = base_cfg(&c->base);
    cfg.k = c->k;
    cfg.l = c->l;
    cfg.alpha = c->alpha;
    cfg.eigval_floor = c->eigval_floor;
    cfg.refresh_interval = c->refresh_interval;
    cfg.curvature_batch = c->curvature_batch;
    cfg.lanczos.reorth_safeguard = c->reorth_safeguard != 0;
    cfg.lanczos.safeguard_ratio = c->safeguard_ratio;
    cfg.lanczos.breakdown_rtol = c->breakdown_rtol;
    cfg.sigma = c->sigma;
    cfg.outer_rounds = c->outer_rounds;
    cfg.inner_epochs = c->inner_epochs;
    cfg.sigma_zero_reduction = c->sigma_zero_reduction != 0;
    cfg.epochs = c->epochs;
    cfg.batch_size = c->batch_size;
    cfg.seed = c->seed;
    Problem p;
    p.oracle = std::make_shared<QuadraticOracle>(Vector(spec, spec + n), rotation_seed);
    p.dataset = Dataset::dummy(N);
    p.w0.assign(w0, w0 + n);
    const auto res = train(cfg, p, workers, Schedule::round_robin(), nullptr);
    std::copy(res.w_final.begin(), res.w_final.end(), w_final);
    *n_rows = res.metrics.size();
    for (std::size_t i = 0; i < res.metrics.size() && i < max_rows; ++i) {
      row_loss[i] = res.metrics[i].train_loss;
      row_acc[i] = res.metrics[i].train_acc;
      row_resid[i] = res.metrics[i].residual_norm;
      row_epoch[i] = res.metrics[i].epoch;
    }
    *refreshes = res.ese_refreshes;
    *safeguards = res.safeguard_passes;
    *wall_ms = res.raw_wallclock_ms;
  });
}

// ---- harness (harness.cpp): config parsing, problem construction, artifacts, reports ----------
static int copy_out(const std::string& text, char* buf, std::size_t len, std::size_t* needed) {
  if (needed) *needed = text.size() + 1;
  if (buf && len) {
    const std::size_t k = std::min(len - 1, text.size());
    std::memcpy(buf, text.data(), k);
    buf[k] = 0;
  }
  return 0;
}

// parse_config_text (harness.cpp:181-247) -> every parsed field as JSON (test comparison)
int ref_parse_config_json(const char* text, const char* origin, char* buf, std::size_t len, std::size_t* needed) {
  return guarded([&] {
    const ExperimentConfig c = parse_config_text(text, origin);
    const TrainerConfig t = build_trainer_config(c);
    nlohmann::json j;
    j["trainer"] = c.trainer;
    j["workers"] = c.workers;
    j["seed"] = c.seed;
    j["schedule"] = c.schedule;
    j["out_dir"] = c.out_dir;
    j["loss_target"] = c.loss_target;
    const auto& p = c.problem;
    j["problem"] = {{"kind", p.kind}, {"n", p.n}, {"condition", p.condition}, {"rotation_seed", p.rotation_seed},
                    {"spectrum", p.spectrum}, {"dataset", p.dataset}, {"csv_path", p.csv_path},
                    {"label_col", p.label_col}, {"feature_cols", p.feature_cols}, {"samples", p.samples},
                    {"dataset_seed", p.dataset_seed}, {"layers", p.layers}, {"activation", p.activation},
                    {"loss", p.loss}};
    j["train"] = {{"kind", static_cast<int>(t.kind)}, {"base_kind", static_cast<int>(t.base.kind)},
                  {"lr", t.base.lr}, {"weight_decay", t.base.weight_decay}, {"beta1", t.base.beta1},
                  {"beta2", t.base.beta2}, {"eps", t.base.eps}, {"momentum", t.base.momentum}, {"k", t.k},
                  {"l", t.l}, {"alpha", t.alpha}, {"eigval_floor", t.eigval_floor},
                  {"refresh_interval", t.refresh_interval}, {"curvature_batch", t.curvature_batch},
                  {"reorth_safeguard", t.lanczos.reorth_safeguard}, {"safeguard_ratio", t.lanczos.safeguard_ratio},
                  {"breakdown_rtol", t.lanczos.breakdown_rtol}, {"sigma", t.sigma},
                  {"outer_rounds", t.outer_rounds}, {"inner_epochs", t.inner_epochs},
                  {"sigma_zero_reduction", t.sigma_zero_reduction}, {"epochs", t.epochs},
                  {"batch_size", t.batch_size}, {"seed", t.seed}, {"debug_hash_checks", t.debug_hash_checks},
                  {"model_bandwidth_gbps", t.model_bandwidth_gbps}, {"model_gflops", t.model_gflops}};
    copy_out(j.dump(), buf, len, needed);
  });
}

// build_problem (harness.cpp:267-309): w0 and the data the problem trains on (n <= max_n)
int ref_build_problem(const char* text, std::size_t max_n, double* w0, std::size_t* n, std::size_t max_samples,
                      double* X, double* y, std::size_t* samples, std::size_t* dim, std::size_t* ncls) {
  return guarded([&] {
    const ExperimentConfig c = parse_config_text(text, "<text>");
    const Problem p = build_problem(c);
    *n = p.w0.size();
    if (w0 && p.w0.size() <= max_n) std::copy(p.w0.begin(), p.w0.end(), w0);
    *samples = p.dataset.size();
    *dim = p.dataset.feature_dim();
    *ncls = p.dataset.n_classes();
    if (X && p.dataset.size() <= max_samples) {
      std::copy(p.dataset.features().begin(), p.dataset.features().end(), X);
      std::copy(p.dataset.labels().begin(), p.dataset.labels().end(), y);
    }
  });
}

// generate_synthetic_dataset (oracle.cpp:77-127)
int ref_synthetic_dataset(const char* kind, std::size_t n_samples, std::uint64_t seed, double* X, double* y,
                          std::size_t* dim, std::size_t* ncls) {
  return guarded([&] {
    const Dataset d = generate_synthetic_dataset(parse_dataset_kind(kind), n_samples, seed);
    std::copy(d.features().begin(), d.features().end(), X);
    std::copy(d.labels().begin(), d.labels().end(), y);
    *dim = d.feature_dim();
    *ncls = d.n_classes();
  });
}

// run_experiment (harness.cpp:364-440) on a config text; *rc = its return value (0, or 2 if aborted)
int ref_run_experiment_text(const char* text, int* rc) {
  return guarded([&] { *rc = run_experiment(parse_config_text(text, "<text>")); });
}

int ref_memory_report(const char** dirs, int ndirs, char* buf, std::size_t len, std::size_t* needed) {
  return guarded([&] {
    std::vector<std::string> d(dirs, dirs + ndirs);
    copy_out(memory_report(d), buf, len, needed);
  });
}

int ref_comm_report(const char* dir, char* buf, std::size_t len, std::size_t* needed) {
  return guarded([&] { copy_out(comm_report(dir), buf, len, needed); });
}

}  // extern "C"
