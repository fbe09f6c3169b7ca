/*
 * dho2gpu.h — C ABI of the B200-native DHO2 curvature-and-update hot path.
 *
 * Plain pointers and sizes only (no torch / STL types). Host buffers are fp64 like the
 * reference's dho2::Vector; device state is fp32 (three tensor-core MMAs per product on
 * power-of-two-scaled fp16 (hi, lo) operand pairs for the MLP contractions, fp64 accumulation
 * for every reduction, fp64 tridiagonal eigensolve).
 * Every entry point returns a dho2g_status; the matching reference exception type is named
 * beside each code, and dho2g_last_error() returns the message (thread-local).
 *
 * Each group below names the reference interface it replaces (paths relative to
 * /root/reference/proj). The reference-side bindings a maintainer adds are in INTEGRATION.md.
 */
#ifndef DHO2GPU_H
#define DHO2GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes <-> include/dho2/errors.hpp:8-36 (+ trainer.hpp:22-24 TrainingDiverged). */
typedef enum {
  DHO2G_OK = 0,
  DHO2G_DIMENSION = 1,  /* dho2::DimensionError */
  DHO2G_ARGUMENT = 2,   /* dho2::ArgumentError */
  DHO2G_NUMERIC = 3,    /* dho2::NumericError */
  DHO2G_DIVERGENCE = 4, /* dho2::DivergenceError */
  DHO2G_DEADLOCK = 5,   /* dho2::DeadlockError (collective timeout) */
  DHO2G_CUDA = 6,       /* CUDA runtime / launch failure */
  DHO2G_NCCL = 7,       /* NCCL failure */
  DHO2G_DIVERGED = 8    /* dho2::TrainingDiverged (non-finite loss) */
} dho2g_status;

typedef struct dho2g_ctx dho2g_ctx;        /* one per GPU / rank (collectives.hpp:88 Worker) */
typedef struct dho2g_mlp dho2g_mlp;        /* MlpOracle (oracle.hpp:113-141) */
typedef struct dho2g_op dho2g_op;          /* HvpFn (lanczos.hpp:11) bound to a device operator */
typedef struct dho2g_lanczos dho2g_lanczos;/* ShardedLanczosResult (dist_lanczos.hpp:21-30) */
typedef struct dho2g_ese dho2g_ese;        /* EseResult (lanczos.hpp:45-52), V_hat row-sharded */
typedef struct dho2g_opt dho2g_opt;        /* BaseOptimizer (optimizer.hpp:28-46) */
typedef struct dho2g_trainer dho2g_trainer;/* TrainerRun (trainer.cpp:51-269) */
typedef struct dho2g_fabric dho2g_fabric;  /* in-process rendezvous for several ranks on one GPU (test backend) */

/* ---- context, errors, collectives (collectives.hpp:88-125) ---------------------------- */
const char* dho2g_last_error(void);
int dho2g_ctx_create(int device, dho2g_ctx** out);
int dho2g_ctx_destroy(dho2g_ctx* ctx);
/* Optional knobs: "gemm" = 0 tcgen05 (default) / 1 CUDA-core reference kernel;
 * "graphs" = 1 capture per-iteration launch sequences in CUDA graphs. */
int dho2g_ctx_set_option(dho2g_ctx* ctx, const char* key, double value);
int dho2g_ctx_get_stat(dho2g_ctx* ctx, const char* key, double* value);
int dho2g_synchronize(dho2g_ctx* ctx);
/* Device timing: marks are CUDA events recorded on the context stream; "ktimers" = 1 makes every
 * library kernel launch record an event pair (stats "kt.<kernel>.ms|count|work"). */
int dho2g_timer_mark(dho2g_ctx* ctx, int id);
int dho2g_timer_ms(dho2g_ctx* ctx, int id0, int id1, double* ms);
int dho2g_ctx_kernel_name(dho2g_ctx* ctx, int i, char* buf, size_t len);
/* NCCL communicator over `world` GPUs (one process or thread per GPU). id = 128 bytes. */
int dho2g_nccl_unique_id(void* id_out_128);
int dho2g_comm_init(dho2g_ctx* ctx, const void* nccl_id_128, int rank, int world);
int dho2g_comm_rank(dho2g_ctx* ctx, int* rank, int* world);
/* Test backend for the multi-rank data path on fewer GPUs than ranks (the reference's in-process
 * run_workers, collectives.hpp:124-125): `world` contexts, one host thread each, share a fabric; every
 * collective is a host-side rendezvous plus stream-ordered device copies between the ranks' buffers
 * (events, no kernel ever waits on another rank). Sums are in ascending rank order. */
int dho2g_local_fabric_create(int world, dho2g_fabric** out);
int dho2g_local_fabric_destroy(dho2g_fabric* fab);
int dho2g_comm_init_local(dho2g_ctx* ctx, dho2g_fabric* fab, int rank);
/* Host-transport communicator: ranks in separate processes (possibly on the SAME GPU) whose collectives go
 * through a caller-supplied host all-gather (e.g. a gloo process group): fn(user, send, recv, bytes) must
 * gather `bytes` from every rank into recv (world x bytes, rank order) and return 0. Every collective is a
 * device->host copy, the callback and a host->device copy (reduce-scatter sums in ascending rank order on
 * the device). For tests of the multi-process data path without NCCL — notably the CUDA-IPC peer pointers
 * of the fused HVP -> reduce-scatter (option hvp_route), which need separate processes. */
typedef int (*dho2g_host_allgather)(void* user, const void* send, void* recv, size_t bytes);
int dho2g_comm_init_host(dho2g_ctx* ctx, int rank, int world, dho2g_host_allgather fn, void* user);
/* Accounting. Communication ledger (CommLedger, collectives.hpp:55-83): one row per
 * collective round this rank took part in — event index, op ("all_gather", "reduce_scatter",
 * "all_reduce"), logical floats, rank, modeled floats sent / received. Empty on a single GPU.
 * Peak float slots per named device object (SlotMeter, accounting.hpp:11-27; names of
 * dist_lanczos.cpp:41-84 and trainer.cpp:70-71, "vhat_partial" for the row-sharded V_hat). */
size_t dho2g_ctx_ledger_rows(dho2g_ctx* ctx);
int dho2g_ctx_ledger_row(dho2g_ctx* ctx, size_t i, int64_t* event, char* op, size_t op_len, int64_t* floats,
                         int* rank, int64_t* sent, int64_t* received);
size_t dho2g_ctx_memory_count(dho2g_ctx* ctx);
int dho2g_ctx_memory_entry(dho2g_ctx* ctx, size_t i, char* name, size_t name_len, int64_t* slots);
int dho2g_ctx_accounting_reset(dho2g_ctx* ctx);
/* All-gather of `count` host doubles per rank (rank order) through the context's collectives; every rank calls. */
int dho2g_ctx_allgather_host(dho2g_ctx* ctx, const double* in, size_t count, double* out);

/* ---- host bookkeeping, bit-exact with the reference (no device needed) ---------------- */
void dho2g_rng_u64(uint64_t seed, size_t n, uint64_t* out);           /* rng.hpp:18-23 */
void dho2g_rng_normal(uint64_t seed, size_t n, double* out);          /* rng.hpp:37-50 */
void dho2g_shuffle_iota(uint64_t seed, size_t n, uint64_t* out);      /* rng.hpp:56-62 */
uint64_t dho2g_mix_seed(uint64_t seed, uint64_t salt);                /* trainer.cpp:41-46 */
int dho2g_shard(size_t n, int world, int rank, size_t* begin, size_t* end); /* collectives.cpp:10-20 */
int dho2g_lanczos_budget(size_t k, size_t l, size_t n, size_t* m);    /* lanczos.cpp:10-16 */
void dho2g_epoch_permutation(size_t N, uint64_t shuffle_seed, uint64_t epoch, uint64_t* out); /* oracle.cpp:56-62 */
/* generate_synthetic_dataset (oracle.cpp:77-127): kind "two-gaussians" | "concentric-rings" |
 * "linear-regression"; X holds n_samples x 3 doubles (row-major, *dim used), y n_samples. */
int dho2g_synthetic_dataset(const char* kind, size_t n_samples, uint64_t seed, double* X, double* y, size_t* dim,
                            size_t* ncls);
/* Curvature batch indices of refresh number `refresh` (trainer.cpp:108-114). */
void dho2g_curvature_indices(size_t N, size_t want, uint64_t seed, uint64_t refresh, uint64_t* out);
/* Per-worker sample indices of round `round` (trainer.cpp:92-99). */
int dho2g_batch_indices(const uint64_t* perm, size_t N, int workers, int worker, size_t round, size_t batch,
                        uint64_t* out);
/* Build-defined "blobs-D" synthetic data, row-major fp64. */
void dho2g_blobs_dataset(size_t N, size_t D, size_t n_classes, uint64_t seed, double* X, double* y);

/* ---- model/loss plugin: Oracle (oracle.hpp:72-80), MlpOracle (oracle.hpp:113-141) ----- */
/* act: 0 tanh, 1 relu. loss: 0 softmax_ce, 1 mse (oracle.hpp:103-107). */
int dho2g_mlp_create(dho2g_ctx* ctx, const size_t* layer_sizes, int n_sizes, int act, int loss,
                     dho2g_mlp** out);
int dho2g_mlp_destroy(dho2g_mlp* mlp);
size_t dho2g_mlp_dim(const dho2g_mlp* mlp);
int dho2g_mlp_init_params(const dho2g_mlp* mlp, uint64_t seed, double* w);   /* oracle.cpp:386-394 */
/* The same from the layer sizes alone (host only); *dim = parameter count, w may be NULL to query it. */
int dho2g_init_params(const size_t* sizes, int n_sizes, uint64_t seed, double* w, size_t* dim);
/* Synchronous host-buffer calls with the reference's semantics (pure, caller-owned fp64). */
int dho2g_mlp_value(dho2g_mlp* mlp, const double* w, const double* X, const double* y, size_t B, size_t ncls,
                    double* out);
int dho2g_mlp_grad(dho2g_mlp* mlp, const double* w, const double* X, const double* y, size_t B, size_t ncls,
                   double* g);
int dho2g_mlp_hvp(dho2g_mlp* mlp, const double* w, const double* v, const double* X, const double* y, size_t B,
                  size_t ncls, double* hv);
int dho2g_mlp_accuracy(dho2g_mlp* mlp, const double* w, const double* X, const double* y, size_t B, size_t ncls,
                       double* acc);

/* ---- operators (HvpFn, lanczos.hpp:11) ----------------------------------------------- */
/* Device MLP Hessian at (w, curvature batch); n = mlp dim. Data are copied to the device. */
int dho2g_op_mlp(dho2g_ctx* ctx, dho2g_mlp* mlp, const double* w, const double* X, const double* y, size_t B,
                 size_t ncls, dho2g_op** out);
/* QuadraticOracle(spectrum, 0).apply_h: diagonal operator (oracle.cpp:262-268). */
int dho2g_op_diag(dho2g_ctx* ctx, const double* spectrum, size_t n, dho2g_op** out);
/* Dense symmetric n x n operator (column-major), the reference tests' matrix_hvp. */
int dho2g_op_dense(dho2g_ctx* ctx, const double* mat, size_t n, dho2g_op** out);
/* QuadraticOracle(spectrum, rotation_seed) (oracle.hpp:84-102, oracle.cpp:233-286): H = diag(spectrum)
 * (rotation_seed 0) or Q^T diag(spectrum) Q with Q the reference's seeded Gram-Schmidt rotation.
 * ARGUMENT for an empty spectrum or a zero / non-finite entry, NUMERIC for a degenerate rotation.
 * With a communicator, create it after dho2g_comm_init (each rank keeps its columns of Q). */
int dho2g_op_quadratic(dho2g_ctx* ctx, const double* spectrum, size_t n, uint64_t rotation_seed, dho2g_op** out);
/* QuadraticOracle::apply_h / hvp / grad (the HvpFn of any operator) on host buffers: out = H x
 * (full length on every rank; null to skip), *value = x^T H x / 2 (QuadraticOracle::value; null to skip). */
int dho2g_op_apply(dho2g_op* op, const double* x, double* out, double* value);
/* Host callback operator: out = H v, fp64 host buffers of length n. */
typedef void (*dho2g_host_hvp)(void* user, const double* v, double* out, size_t n);
int dho2g_op_host(dho2g_ctx* ctx, dho2g_host_hvp fn, void* user, size_t n, dho2g_op** out);
int dho2g_op_destroy(dho2g_op* op);

/* ---- sharded Lanczos (dist_lanczos.hpp:32-41, lanczos.hpp:17-26) --------------------- */
typedef struct {
  int reorth_safeguard;   /* default 1 */
  double safeguard_ratio; /* default 1e-6 */
  double breakdown_rtol;  /* default 1e-10 */
} dho2g_lanczos_opts;
int dho2g_lanczos_run(dho2g_ctx* ctx, dho2g_op* op, size_t m, uint64_t seed, const dho2g_lanczos_opts* opts,
                      dho2g_lanczos** out);
/* B (fp64, bitwise identical on every rank): diag[0..iters), off[0..iters-1 or iters). */
int dho2g_lanczos_result(const dho2g_lanczos* lz, double* diag, double* off, size_t* iters, int* breakdown,
                         size_t* safeguard_passes, size_t* shard_begin, size_t* shard_end);
/* This rank's basis rows D[s:e, 0:cols) normalized, column-major fp64 (cols = iters+1, or iters
 * after breakdown). */
int dho2g_lanczos_basis(const dho2g_lanczos* lz, double* basis_shard);
int dho2g_lanczos_destroy(dho2g_lanczos* lz);
/* extract_ese_distributed (dist_lanczos.cpp:121-158): device tql2 + selection + Ritz vectors. */
int dho2g_extract_ese(dho2g_ctx* ctx, dho2g_lanczos* lz, size_t k, size_t l, dho2g_ese** out);
size_t dho2g_ese_count(const dho2g_ese* ese);
int dho2g_ese_eigvals(const dho2g_ese* ese, double* vals);
/* This rank's rows of V_hat (sign convention of lanczos.cpp:82-94 applied), column-major. */
int dho2g_ese_eigvecs(const dho2g_ese* ese, double* vecs_shard);
/* The full V_hat (n x r, column-major) on every rank, as extract_ese_distributed returns it after its
 * gather_rows (dist_lanczos.cpp:148-156). Collective: every rank calls it. */
int dho2g_ese_gather(const dho2g_ese* ese, double* vecs_full);
/* This rank's V_hat rows (signs applied) into a caller-owned device fp32 buffer, column-major with
 * leading dimension ld >= rows (checks that keep a large V_hat on the device). */
int dho2g_ese_eigvecs_device(const dho2g_ese* ese, float* dst, size_t ld);
/* Build an ESE from host data (tests feed the reference's eigenpairs): V is n x r column-major. */
int dho2g_ese_from_host(dho2g_ctx* ctx, const double* eigvals, const double* V, size_t n, size_t r,
                        dho2g_ese** out);
/* The same from a device-resident fp32 V (column-major, leading dimension ld_src >= n); this rank's rows
 * are copied device to device (a caller holding V_hat in HBM does not stage 13 GB through the host). */
int dho2g_ese_from_device(dho2g_ctx* ctx, const double* eigvals, const float* V_dev, size_t ld_src, size_t n,
                          size_t r, dho2g_ese** out);
int dho2g_ese_destroy(dho2g_ese* ese);

/* ---- update step (optimizer.hpp:16-80) ---------------------------------------------- */
typedef struct {
  int kind; /* 0 sgd, 1 momentum, 2 adam, 3 adamw (optimizer.hpp:11) */
  double lr, weight_decay, beta1, beta2, eps, momentum;
} dho2g_base_cfg;
int dho2g_opt_create(dho2g_ctx* ctx, const dho2g_base_cfg* cfg, size_t n, dho2g_opt** out);
int dho2g_opt_destroy(dho2g_opt* opt);
/* BaseOptimizer::step (optimizer.cpp:37-71): d = step(g, w). */
int dho2g_opt_step(dho2g_opt* opt, const double* g, const double* w, double* d);
/* fosi_deltas (pi == NULL) / admm_deltas (optimizer.cpp:81-129), materialized Deltas. ese may
 * be NULL (empty ESE). Advances the optimizer's moments like the reference. */
int dho2g_deltas(dho2g_opt* opt, const dho2g_ese* ese, const double* g, const double* pi, const double* w,
                 double alpha, double sigma, double eigval_floor, double* newton, double* base);
/* admm_w_update / admm_dual_update (optimizer.cpp:141-154) over host buffers. */
int dho2g_admm_w_update(dho2g_ctx* ctx, size_t n, double sigma, const double* w_a, const double* pi, double* w);
int dho2g_admm_dual_update(dho2g_ctx* ctx, size_t n, double sigma, const double* w_a, const double* w, double* pi);

/* ---- the trainer (trainer.hpp:26-96): DHO2 / FOSI / first-order loops on device -------- */
typedef struct {
  int trainer; /* 0 sgd, 1 fosi, 2 dho2 */
  dho2g_base_cfg base;
  size_t k, l;
  double alpha, eigval_floor;
  size_t refresh_interval, curvature_batch;
  int reorth_safeguard;
  double safeguard_ratio, breakdown_rtol;
  double sigma;
  size_t outer_rounds, inner_epochs;
  int sigma_zero_reduction;
  size_t epochs, batch_size;
  uint64_t seed;
  size_t lanczos_m; /* 0 = lanczos_budget(k, l, n) (trainer.cpp:117); else explicit m (C4) */
  /* modeled clock of MetricsRow::wallclock_ms (trainer.cpp:137-148); 0 = the reference defaults 50 / 10 */
  double model_bandwidth_gbps, model_gflops;
  /* TrainerConfig::debug_hash_checks (trainer.cpp:120, :128, :157): sets the context's hash_checks option —
   * B compared across ranks after each refresh and at extraction, the parameter replicas at every epoch end
   * (DivergenceError on a mismatch) */
  int debug_hash_checks;
} dho2g_train_cfg;
/* Dataset (oracle.hpp:25-54) is uploaded once (device resident) unless host_resident != 0, in
 * which case every step gathers its batch from pinned host memory (end-to-end mode). */
int dho2g_trainer_create(dho2g_ctx* ctx, const dho2g_train_cfg* cfg, dho2g_mlp* mlp, const double* X,
                         const double* y, size_t N, size_t ncls, uint64_t dataset_seed, const double* w0,
                         int workers, int host_resident, dho2g_trainer** out);
/* The same loops on a QuadraticOracle problem (dho2g_op_quadratic; test_trainer.cpp:14-21): the
 * dataset is Dataset::dummy(n_samples) (oracle.cpp:64-68), every gradient is H w, epoch_end's loss is
 * w^T H w / 2 and accuracy is NaN. */
int dho2g_trainer_create_quadratic(dho2g_ctx* ctx, const dho2g_train_cfg* cfg, dho2g_op* quad, size_t n_samples,
                                   const double* w0, int workers, dho2g_trainer** out);
int dho2g_trainer_destroy(dho2g_trainer* tr);
/* Advance `steps` DHO2 steps (inner rounds, trainer.cpp:233-242) including every refresh and
 * ADMM w/dual update the schedule puts inside them. epoch_end evaluation (full-dataset loss,
 * accuracy, residual; trainer.cpp:150-172) runs when with_eval != 0. Asynchronous on the ctx
 * stream; errors surface at the next synchronizing call. */
int dho2g_trainer_step(dho2g_trainer* tr, size_t steps, int with_eval);
/* Run the whole configured schedule (train(), trainer.cpp:273-298) with evaluation. */
int dho2g_trainer_run(dho2g_trainer* tr);
int dho2g_trainer_params(dho2g_trainer* tr, double* w);      /* current w_a (trainer final_params) */
size_t dho2g_trainer_rows(dho2g_trainer* tr);                /* MetricsRow count */
int dho2g_trainer_metrics(dho2g_trainer* tr, size_t max_rows, double* loss, double* acc, double* resid,
                          int64_t* epoch, int* refresh);
/* The remaining MetricsRow fields (trainer.hpp:68-77): outer_k / inner_l (-1 outside DHO2) and the
 * modeled wallclock_ms (ledger floats x 8 B / bandwidth + GS flops / GFLOP/s, trainer.cpp:137-148). */
int dho2g_trainer_metrics_ex(dho2g_trainer* tr, size_t max_rows, int64_t* outer, int64_t* inner, double* wallclock);
/* Mean minibatch loss of the last step (device->host read of the step's result). */
int dho2g_trainer_last_loss(dho2g_trainer* tr, double* loss);
/* Counters: "refreshes", "safeguard_passes", "steps", "refresh_ms_last", "h2d_bytes", ... */
int dho2g_trainer_stat(dho2g_trainer* tr, const char* key, double* value);
/* Last refresh's eigenvalues (k+l) and tridiagonal matrix. */
int dho2g_trainer_eigvals(dho2g_trainer* tr, double* vals, size_t* count);

/* ---- test hook: one split (hi, lo) GEMM C = A B^T (operand format per ctx option gemm_f16) over host fp32 (A: M x K, B: N x K, row-major).
 * backend 0 = tcgen05 kernel, 1 = CUDA-core reference kernel. ------------------------------- */
int dho2g_test_gemm(dho2g_ctx* ctx, int M, int N, int K, const float* A, const float* B, float* C, int backend);
/* Two-segment form C = A0 B0^T + A1 B1^T (A0: M x K0, A1: M x K1, B0: N x K0, B1: N x K1; K1 = 0: one
 * segment) with each operand stored K-major (a_mn / b_mn = 0) or MN-major (1), the layouts the MLP's
 * concatenated contractions use. */
/* ---- test hook: each collective wrapper through a 1-rank NCCL communicator (plumbing check on one GPU).
 * The context must have no communicator; *max_err = worst element error (0 expected). */
int dho2g_test_collectives(dho2g_ctx* ctx, double* max_err);
/* The same collectives captured into a CUDA graph and replayed (the multi-rank refresh graph captures
 * its NCCL calls this way). */
int dho2g_test_collectives_graph(dho2g_ctx* ctx, double* max_err);
/* ---- test hook: per-CTA timelines (globaltimer ns: start, last MMA, last epilogue start, end) of pair-GEMM
 * launches; on = 1 arms a buffer for n_ctas CTA slots, on = 0 copies it to out and disarms. */
int dho2g_test_gemm_trace(dho2g_ctx* ctx, int on, unsigned long long* out, size_t n_ctas);
int dho2g_test_gemm_seg(dho2g_ctx* ctx, int M, int N, int K0, int K1, const float* A0, const float* A1,
                        const float* B0, const float* B1, float* C, int backend, int a_mn, int b_mn);

#ifdef __cplusplus
}
#endif
#endif /* DHO2GPU_H */
