// Internal object layouts shared by the translation units of libdho2gpu.so.
#pragma once

#include <chrono>
#include <condition_variable>
#include <map>
#include <mutex>
#include <memory>
#include <string>
#include <vector>

#include "common.cuh"

namespace dho2g {

constexpr int kMaxLanczos = 1024;  // m <= 1023 (C5 sweep needs 512)
// fp32 adaptation of the reference's breakdown / safeguard thresholds (lz_decide_kernel)
constexpr double kBreakdownFloor32 = 4e-6;
constexpr double kSafeguardFloor32 = 1e-3;
constexpr int kGsChunk = 2048;     // rows per GS pass-1 chunk; shard rows are padded to this

// ------------------------------------------------------------------------- host bookkeeping
struct Rng {  // rng.hpp:14-68 (SplitMix64 + Box-Muller with spare)
  uint64_t state;
  double spare = 0.0;
  bool have_spare = false;
  explicit Rng(uint64_t s) : state(s) {}
  uint64_t next_u64();
  double uniform();
  uint64_t uniform_below(uint64_t bound);
  double normal();
};
void shuffle_iota(uint64_t seed, size_t n, uint64_t* out);
void shard_range(size_t n, int world, int rank, size_t* begin, size_t* end);
size_t lanczos_budget(size_t k, size_t l, size_t n);
bool quadratic_rotation(size_t n, uint64_t rotation_seed, double* Q);  // false: degenerate draw

}  // namespace dho2g

// ------------------------------------------------------------------------- context
struct dho2g_ctx {
  int device = 0;
  int sm_count = 148;
  cudaStream_t stream = nullptr;
  int gemm_backend = 0;  // 0 tcgen05, 1 CUDA-core reference kernel
  int gemm_splits = 0;   // 0 = automatic split-K for small-M GEMMs (single-CTA kernel)
  int gemm_cta = 0;      // tcgen05 kernel: 0 auto, 1 single-CTA 128x128 tiles, 2 CTA-pair 256x256 tiles
  int gemm_dp = 1;       // pair kernel: data-parallel waves before the stream-K remainder (0: all stream-K)
  int gemm_group = 1;    // pair kernel, few m-tiles (the HVP's M = 1024): m-tile groups of pairs walk the same
                         // (n, k) ranges, so each B slab is read from DRAM once (0: plain stream-K)
  int gemm_mm_tc1 = 0;   // auto: short-K MN-major x MN-major GEMMs on the single-CTA kernel (off: measured slower since the
                         // compile-time epilogues)
  int gemm_min_kb = 4;   // pair kernel: minimum k-blocks per CTA pair (caps the worker count of small GEMMs)
  int gemm_worker_cap = 0;  // pair kernel: at most this many CTA pairs (0: all co-resident pairs)
  int lanczos_recurrence = 1;  // Lanczos: recurrence-first projection (1) or the reference's plain CGS (0)
  int gemm_pdl = 1;      // CTA-pair GEMMs launched with programmatic dependent launch (prologue overlaps the
                         // previous kernel's tail)
  int hvp_route = 0;      // world > 1: batch-split HVP partials stored straight into the owners' buffers
                         // (peer memory) instead of a reduce-scatter after the HVP
  int bwd_overlap = 1;   // backward: weight-block GEMM on a side stream, concurrent with the delta GEMM
  int gemm_chunk_kb = 8;  // HVP (curvature) GEMMs on the CTA-pair kernel: drain the TMEM accumulator into an
                         // fp32 running sum every this many 64-deep k-blocks (0: never). The tensor core's
                         // accumulation truncates, so its error grows with the chain length (measured: linear);
                         // short chains + round-to-nearest fp32 sums bound it.
  int gemm_chunk_kb1 = 8; // the same for the single-CTA kernel (small-M GEMMs: C1/C2 HVPs and gradients), where
                         // the drains are cheap
  int gemm_f16 = 1;      // MLP GEMM operands as power-of-two-scaled fp16 (hi, lo) pairs (22 significant bits)
                         // instead of bf16 pairs (16 bits); same tcgen05 kind::f16 rate
  int mlp_small = 1;      // MLP passes of small models (HVP <= mlp_small_mflop MFLOP) as one persistent CUDA-core
                         // launch each (mlp_small.cu) instead of the tcgen05 GEMM sequence
  double mlp_small_mflop = 2000.0;
  int upd_small = 1;  // world 1, r <= 32, rows <= upd_small_max_rows: the update's three passes as one launch
  double upd_small_max_rows = 4e6;
  int lanczos_small = 1;  // world 1, small MLP operator (2: also diagonal), m <= 512: the whole refresh as one launch
  double lanczos_small_max_n = 4e6;
  int mlp_small_ctas_per_sm = 1;
  cudaStream_t stream2 = nullptr;                 // side lane (created on first use)
  dho2g::DevBuf<float> gemm_ws2;                  // its GEMM workspace / flags (swapped in by SideLane)
  dho2g::DevBuf<unsigned> gemm_flags2;
  std::vector<cudaEvent_t> lane_events;           // fork / join events (created on first use)
  int pairs_total = 0;                            // co-resident CTA pairs of the pair kernel
  dho2g::DevBuf<float> gemm_ws, simt_ws;  // split-K partials / CUDA-core accumulators
  dho2g::DevBuf<unsigned> gemm_flags;
  unsigned gemm_epoch = 0;
  int use_graphs = 1;     // capture the Lanczos refresh into a CUDA graph (world 1)
  int gs_sm_cap = 0;     // Gram-Schmidt grids sized for at most this many SMs (0: all; experiments)
  int ritz_tc = 1;        // Ritz vectors on the tensor cores when supported (0: CUDA-core kernel)
  int tql2_split = 1;     // eigensolve: 1 QL chain with a concurrent shared-memory rotation replay, then
                          // selection (1.3x at m = 40-80, 2.0x at 512, 2.7x at 1000); 0 single-CTA tql2
  int upd_p2_staged = 1;  // update pass 2: 1 bulk-copy staged (R <= 48), 0 register-staged
  int upd_p2_variant = 5; // staged pass 2: 5 row-dot (R <= 32, else 0), 0 256-row x2 stages x2 CTAs/SM +
                          // column-dot phase, 1 128x2x4, 2 128x3x3, 3 128x4x2, 4 512x2x1
  ncclComm_t comm = nullptr;
  dho2g_fabric* fabric = nullptr;  // in-process test backend (dho2g_comm_init_local) instead of NCCL
  dho2g_host_allgather host_ag = nullptr;  // host-transport backend (dho2g_comm_init_host) instead of NCCL
  void* host_ag_user = nullptr;
  dho2g::HostBuf<char> host_ag_buf;        // its pinned staging (send, then world x recv)
  bool host_rendezvous() const { return fabric != nullptr || host_ag != nullptr; }  // collectives on the host
  dho2g::DevBuf<float> fabric_scratch;
  int rank = 0, world = 1;
  long long tql2_log_cap = 0;  // split eigensolve's rotation-log entries (0: 2 m^2 + 4096); tests shrink it
  int graphs_multirank = 1;  // refresh CUDA graph also at world > 1 (NCCL communicator; not the fabric)
  int hash_checks = 0;  // debug cross-rank checks (DistLanczosOptions::hash_checks / debug_hash_checks):
                        // B after a refresh and at extraction, the parameter replicas at every epoch end
                        // (2: test hook, ranks > 0 perturb their hash — a simulated divergence)
  bool nccl_force = false;  // test hook: route world-1 collectives through a 1-rank NCCL communicator
  // Set when a collective failed (DEADLOCK / NCCL): the communicator is aborted and every later call on
  // this context raises (its shards, offsets and buffers belong to the failed group, so it must not go on
  // as a single rank). The reference throws out of the failed round the same way (collectives.cpp:257-262).
  bool failed = false;
  std::string failed_msg;
  // Serialises the host-API oracle entry points (dho2g_mlp_value/grad/hvp/accuracy) on this context: they
  // stage through the model's buffers and the context stream, and the reference calls Oracle::grad / hvp
  // from every worker thread at once (trainer.cpp:92-103, dist_lanczos.cpp:79; "safe for concurrent use",
  // oracle.hpp:70-71).
  std::mutex api_mu;
  void check_usable() const;
  double nccl_timeout_s = 600.0;  // host waits with a communicator give up (DEADLOCK) after this long
  void* encode_fn = nullptr;  // PFN_cuTensorMapEncodeTiled
  std::map<std::string, double> stats;
  // Per-kernel device timers (CUDA events on this stream), enabled by option "ktimers".
  bool ktimers = false;
  struct KPending { std::string name; cudaEvent_t a, b; double work; bool ended; };
  std::map<int, KPending> kpend;  // open (nested) and ended timers, by id
  int knext = 0;
  std::vector<cudaEvent_t> kpool;
  struct KStat { double ms = 0, count = 0, work = 0; };
  std::map<std::string, KStat> kstats;
  std::vector<cudaEvent_t> marks;  // user timer marks
  int kt_begin();                  // returns slot or -1
  void kt_end(int slot, const char* name, double work);
  void kt_flush();                 // synchronize and fold pending events into kstats
  dho2g::DevBuf<double> gather_f64;  // world * count scratch for ordered all-reduces
  dho2g::DevBuf<double> pinned_dummy;

  // Collectives (NCCL over NVLink at world > 1; identity at world == 1). `op` names the logical
  // collective in the communication ledger (an all-gather of partials that every rank then sums in
  // rank order is the reference's "all_reduce").
  void allgather_f64(const double* send, double* recv, size_t count, const char* op = "all_gather");
  void allgather_f32(const float* send, float* recv, size_t count, const char* op = "all_gather");
  void reduce_scatter_f32(const float* send, float* recv, size_t count);
  void allreduce_sum_f64_ordered(double* inout, size_t count);  // all_gather + rank-ordered sum
  void barrier();  // stream-ordered: returns on each rank's stream once every rank's prior work is done
  dho2g::DevBuf<double> barrier_buf;
  // Communication ledger (CommLedger, collectives.hpp:55-83): one row per collective this rank took
  // part in (world > 1 only: a single GPU communicates nothing). floats = the round's logical result
  // length; sent / received model ring traffic of this rank, in floats.
  struct LedgerRow {
    int64_t event;
    std::string op;
    int64_t floats;
    int rank;
    int64_t sent, received;
  };
  std::vector<LedgerRow> ledger;
  int64_t ledger_next = 0;
  int64_t ledger_sent = 0;  // this rank's floats sent, all rounds
  void ledger_add(const char* op, int64_t floats, int64_t sent, int64_t received) {
    ledger.push_back({ledger_next++, op, floats, rank, sent, received});
    ledger_sent += sent;
  }
  // Peak float-slot accounting per named device object (SlotMeter, accounting.hpp:11-27).
  std::map<std::string, int64_t> slots;
  void meter(const char* name, int64_t n) {
    auto& p = slots[name];
    if (n > p) p = n;
  }
  void sync();
  void bump(const char* key, double v) { stats[key] += v; }
};

// ------------------------------------------------------------------------- MLP (oracle.hpp:113)
struct LayerDesc {
  int in = 0, out = 0;    // sizes[t], sizes[t+1]
  int Pin = 0, Pout = 0;  // round_up(., 8): half-width of the [a | ra] and [V | W] operand pairs
  int Din = 0, Dout = 0;  // round_up(., 64): half-width of the [d | rd] pairs (= their K segment length)
  size_t w_off = 0, b_off = 0;
};

struct dho2g_mlp {
  dho2g_ctx* ctx = nullptr;
  std::vector<size_t> sizes;
  std::vector<LayerDesc> layers;
  size_t dim = 0;
  int act = 0, loss = 0;
  int L = 0;
  // Weight operands per layer t: WV[t] = [V | W] rows o (out x 2Pin). The forward GEMMs read it K-major
  // (K = in), the backward GEMMs MN-major (K = out) — no transposed copy.
  std::vector<dho2g::DevBuf<dho2g::bf16>> WV_hi, WV_lo;
  // Batch operands per activation level j (width s_j = sizes[j], half-width P_j), row-major by sample:
  //  AR[j] = [a | ra] rows b (Bcap x 2P_j), j = 0..L-1
  //  DR[j] = [d | rd] rows b (Bcap x 2D_j, D_j = round_up(s_j, 64)), j = 1..L
  // K-major operands of the forward / backward GEMMs and MN-major operands (K = batch) of the
  // weight-block GEMMs.
  std::vector<dho2g::DevBuf<dho2g::bf16>> AR_hi, AR_lo, DR_hi, DR_lo;
  std::vector<dho2g::DevBuf<float>> a32, ra32, d32, rd32, u32;  // fp32 B x s_j (u32: cached U = D W)
  dho2g::DevBuf<float> Z, RZ;                               // GEMM outputs (Bcap x max s)
  dho2g::DevBuf<float> lab;                                 // gathered labels (Bcap)
  dho2g::DevBuf<double> sample_loss;                        // per-sample loss (Bcap)
  dho2g::DevBuf<int> sample_correct;
  size_t Bcap = 0;
  size_t smax = 0;
  // host-API staging
  dho2g::DevBuf<float> w32, v32, X32, y32, out32;
  dho2g::DevBuf<int64_t> idx;
  dho2g::DevBuf<double> red;
  dho2g::DevBuf<double> colpart;      // bias column-sum partials
  dho2g::DevBuf<float> csum;          // per-32-row column sums written by the backward epilogues
  std::vector<cudaEvent_t> pack_ev;   // per-layer 'packed' events of the side-lane weight packing (+ fork)
  bool pack_pending = false;          // forward() must wait for pack_ev before each layer
  dho2g::DevBuf<unsigned> coltickets;  // their per-column-block completion tickets
  const float* w_cur = nullptr;        // params whose W halves are loaded
  const float* v_bias_ptr = nullptr;   // direction whose V halves are loaded (bias part read directly)
  const float* v_scale_ptr = nullptr;  // device scalar multiplying the direction (lazy Lanczos norm)
  const void* input_owner = nullptr;   // operator whose curvature batch is packed at level 0
  const float* prepared = nullptr;     // w whose v-independent HVP quantities are cached
  // fused HVP -> reduce-scatter: the weight-block GEMMs store straight into the owners' receive slots
  float* const* route = nullptr;
  long long route_base = 0;
  int route_rank = 0;
  // Scaled-fp16 operand state (ctx option gemm_f16): one power-of-two scale per pair buffer
  //   scl[t] AR[t] (t < L), scl[L + j - 1] DR[j] (1 <= j <= L), scl[2L + t] WV[t]
  // and max |x| slots (float bits) of the fp32 tensors the pairs are split from
  //   amax[j] a_j, amax[(L+1) + j] ra_j, amax[2(L+1) + j] d_j, amax[3(L+1) + j] rd_j (j <= L),
  //   amax[4(L+1) + t] W_t, amax[4(L+1) + L] the level-0 input batch.
  int f16 = 0;              // format of the currently packed operands
  int chunk_kb = 0;         // Epi::chunk_kb of the GEMMs being issued (the HVP path sets it)
  float wv_vbound = 0.f;    // bound on |direction| the WV scales were chosen for
  dho2g::DevBuf<float> scl;
  dho2g::DevBuf<float> sclx;        // scale of the x half of each pair buffer (split_pair_kernel), same index
  dho2g::DevBuf<unsigned> sticket;  // its update tickets
  dho2g::DevBuf<unsigned> amax;
  float* s_ar(int t) { return scl.p + t; }
  float* s_dr(int j) { return scl.p + L + j - 1; }
  float* s_wv(int t) { return scl.p + 2 * L + t; }
  unsigned* mx_a(int j) { return amax.p + j; }
  unsigned* mx_ra(int j) { return amax.p + (L + 1) + j; }
  unsigned* mx_d(int j) { return amax.p + 2 * (L + 1) + j; }
  unsigned* mx_rd(int j) { return amax.p + 3 * (L + 1) + j; }
  unsigned* mx_w(int t) { return amax.p + 4 * (L + 1) + t; }
  unsigned* mx_x() { return amax.p + 4 * (L + 1) + L; }

  // Lazily packed operands: the W halves of w_cur (wv_packed == w_cur once packed for the current load) and
  // the level-0 batch (input_packed); the small-model path reads fp32 directly and never packs them.
  const float* wv_packed = nullptr;
  bool input_packed = false;
  const float* x_src = nullptr;  // current batch: rows X[idx[b]] (idx null: b), labels y likewise
  const int64_t* x_idx = nullptr;
  const float* y_src = nullptr;
  size_t x_B = 0;
  bool prepared_small = false;   // the cached point quantities came from the small-model path
  dho2g::DevBuf<float> x0, y0;   // small-model path: device copy of a host-resident batch
  dho2g::DevBuf<float> sm_part;  // small-model path: split partials, tickets, grid-barrier words
  dho2g::DevBuf<unsigned> sm_tickets;
  dho2g::DevBuf<unsigned long long> sm_bar;
  int sm_bar_nb = 0;  // grid size the barrier counter is a multiple of

  void ensure_batch(size_t B);
  ~dho2g_mlp() {
    for (cudaEvent_t ev : pack_ev) cudaEventDestroy(ev);
  }
};

namespace dho2g {
// MLP device operations (mlp.cu). All stream-ordered on mlp->ctx->stream.
void mlp_load_weights(dho2g_mlp* m, const float* w);
void mlp_load_direction(dho2g_mlp* m, const float* v, const float* vscale /* device scalar or null */);
// Pack level-0 operands from dataset rows X[idx[b]] (idx null: b itself); labels likewise.
void mlp_set_input(dho2g_mlp* m, const float* X, const float* y, const int64_t* idx, size_t B, bool with_r);
// Convenience compositions.
void mlp_grad_dev(dho2g_mlp* m, const float* w, const float* X, const float* y, const int64_t* idx, size_t B,
                  size_t ncls, double scale, float* g);
// Caches A, Z, softmax, D and U at the loaded point (Lanczos applies H m times at one point).
void mlp_prepare_point(dho2g_mlp* m, size_t B, size_t ncls, double scale);
// vbound: an upper bound on |vscale * v| (1 for the unit Lanczos directions); sizes the fp16 operand scale
void mlp_hvp_dev(dho2g_mlp* m, const float* v, const float* vscale, size_t B, size_t ncls, double scale, float* hv,
                 float vbound = 1.0f);
// Forward-only evaluation: adds sum of per-sample loss and correct count into acc[0], acc[1] (fp64).
void mlp_eval_dev(dho2g_mlp* m, const float* w, const float* X, const float* y, const int64_t* idx, size_t B,
                  size_t ncls, double* acc2);

void mlp_loss_sum(dho2g_mlp* m, size_t B, double* acc2);
// Debug hash checks (dist_lanczos.cpp:11-29): the reference's FNV-1a of the fp64 bits of B's entries, and a
// chunked FNV of a device vector's fp32 bits; all_equal across ranks (an all-gather of the two 32-bit halves).
uint64_t tridiag_hash_host(const double* diag, const double* off, size_t upto);
uint64_t device_hash_f32(dho2g_ctx* ctx, const float* v, size_t n);
bool ranks_all_equal(dho2g_ctx* ctx, uint64_t h);
// Small-model path (mlp_small.cu): eligibility (ctx option mlp_small, HVP flops at batch B), one persistent
// launch per pass (mode 0 gradient, 1 point preparation, 2 HVP, 3 evaluation), scratch presizing.
bool mlp_small_eligible(const dho2g_mlp* m, size_t B);
void mlp_small_run(dho2g_mlp* m, int mode, size_t B, const float* w, const float* v, const float* vscale, float* out,
                   size_t ncls, double scale);
void mlp_small_presize(dho2g_mlp* m, size_t B);
bool lanczos_small_eligible(const dho2g_lanczos* lz, const dho2g_op* op);
void lanczos_small_run(dho2g_lanczos* lz, dho2g_op* op);  // m iterations (after v1 / lz_init) in one launch  // acc2 = {sum loss, sum correct} of last batch
// Allocates the batch-dependent buffers for batches up to B up front (graph-stable pointers).
void mlp_presize(dho2g_mlp* m, size_t B);

// GEMM epilogues (gemm.cu). One accumulator element (row, col) of a GEMM tile is turned into:
//  EPI_STORE   C[row*ldc + col] = alpha*acc (column N-1 -> bias_out[row] when bias_out != null)
//  EPI_FWD     hidden layer: do0: a = act(acc + bias) ; do1: ra = act'(a_in) (acc + vscale*vbias)
//  EPI_FWD_OUT output layer: do0: z = acc + bias ; do1: rz = acc + vscale*vbias   (fp32 only)
//  EPI_BWD     do0: d = acc act'(a_in), u_out = acc ; do1: rd = acc act'(a_in) + u_in (-2 a_in ra_in)
// writing the fp32 value (f0 / f1, B x N) and its bf16 (hi, lo) split into the row-major pair
// buffer (R, half hR) and the transposed pair buffer (T, half hT; rows [M, Bp) get zeros), and, when
// csum is set, fixed-order column sums of the values per 32-row block (the next layer's bias block).
enum EpiMode { EPI_STORE = 0, EPI_FWD = 1, EPI_FWD_OUT = 2, EPI_BWD = 3 };
struct Epi {
  int mode, M, N;
  float alpha;
  float* C;
  int ldc;
  float* bias_out;
  int do0, do1, relu;
  const float* bias;
  const float* vbias;
  const float* vscale;
  const float* a_in;
  const float* ra_in;
  const float* u_in;
  float* f0;
  float* f1;
  float* u_out;
  bf16* Rh;
  bf16* Rl;
  int P, hR;
  bf16* Th;
  bf16* Tl;
  int ldT, Bp, hT;
  float* csum;  // optional: per 32-row block column sums of the epilogue values, [ceil(M/32)][N]
  // EPI_STORE routed to the owning ranks (fused GEMM -> reduce-scatter over peer memory): element
  // (row, col) has flat index route_flat0 + row*ldc + col; its owner q = flat / route_base receives it at
  // route[q][route_rank * route_base + flat - q * route_base]. C is unused when route is set.
  float* const* route;
  long long route_flat0;
  long long route_base;
  int route_rank;
  // Scaled-fp16 operands (option gemm_f16): f16 selects the fp16 operand format of the MMAs; sa / sb are
  // the device power-of-two scales of the A / B pair buffers (acc is multiplied by 1 / (sa sb) before the
  // epilogue math, exactly); amax, if set, receives max |value| over the values the epilogue writes
  // (float bits, atomicMax) for the split that turns them into the next operand.
  int f16;
  const float* sa;
  const float* sb;
  unsigned* amax;
  // CTA-pair kernel: k-blocks per TMEM accumulation chunk, drained into an fp32 running sum in TMEM (0: one
  // chain per segment). Set for the curvature (HVP) GEMMs, whose precision the Lanczos refresh needs.
  int chunk_kb;
};
// One GEMM operand: a (hi, lo) bf16 pair buffer read through a TMA-style window. K-major: rows are
// the M (or N) index, K contiguous; MN-major: rows are the K index, M (or N) contiguous. The K range
// may be two segments, [0, kseg) and [kseg, K), read at different offsets of the same buffer (the
// MLP's [x | rx] concatenations). Logical element (mn, k): seg = k >= kseg, kk = k - seg * kseg;
//   K-major : inner = kk + off_in[seg], outer = mn + off_out[seg]
//   MN-major: inner = mn + off_in[seg], outer = kk + off_out[seg]
// and address outer * ld + inner; coordinates outside [0, inner) x [0, outer) read as zero.
struct GOp {
  const bf16* hi;  // (hi, lo) 16-bit pairs: bf16, or fp16 scaled by a power of two when f16 is set
  const bf16* lo;
  int ld;
  int mn_major;
  int inner, outer;
  int off_in[2], off_out[2];
  int f16;
};
GOp gop_k(const bf16* hi, const bf16* lo, int ld, int K, int rows);  // plain K-major, one segment
void gemm_presize(dho2g_ctx* ctx);  // both lanes' GEMM workspaces at their maximum size
// acc = A[M x K] B[N x K]^T in split-BF16x3 (hi*hi + hi*lo + lo*hi), then the epilogue.
// kseg: segment boundary (a multiple of 64) or >= K for a single segment.
void gemm3x(dho2g_ctx* ctx, int M, int N, int K, int kseg, const GOp& A, const GOp& B, const Epi& e);
void gemm3(dho2g_ctx* ctx, int M, int N, int K, const bf16* Ahi, const bf16* Alo, int lda, const bf16* Bhi,
           const bf16* Blo, int ldb, const Epi& e);  // both K-major
void gemm3_store(dho2g_ctx* ctx, int M, int N, int K, const bf16* Ahi, const bf16* Alo, int lda, const bf16* Bhi,
                 const bf16* Blo, int ldb, float* C, int ldc, float alpha, float* bias_out = nullptr);

// fp32 elementwise helpers (update.cu)
void dev_copy_f64_to_f32(cudaStream_t s, const double* src, float* dst, size_t n);
void dev_copy_f32_to_f64(cudaStream_t s, const float* src, double* dst, size_t n);
}  // namespace dho2g

// ------------------------------------------------------------------------- operators / Lanczos
struct dho2g_op {
  dho2g_ctx* ctx = nullptr;
  int kind = 0;  // 0 mlp, 1 diag (quadratic, rotation_seed 0), 2 dense, 3 host, 4 rotated quadratic
  size_t n = 0;
  dho2g_mlp* mlp = nullptr;
  dho2g::DevBuf<float> w, X, y, mat;
  const float* wptr = nullptr;  // params the Hessian is taken at (own copy `w` or the trainer's w_a)
  const float* Xptr = nullptr;  // dataset rows (own copy `X` or the trainer's resident dataset)
  const float* yptr = nullptr;
  dho2g::DevBuf<int64_t> idx;
  dho2g::DevBuf<float> hfull;  // full-length partial (padded to world * base)
  // fused HVP -> reduce-scatter (ctx option hvp_route, world > 1): this rank's receive buffer (one
  // base-long slot per sender), the device table of every rank's receive buffer, IPC-opened peers
  dho2g::DevBuf<float> recv;
  dho2g::DevBuf<float*> route_tab;
  std::vector<void*> ipc_opened;
  void route_setup(size_t base);
  // fused reduce-scatter around any MLP pass that writes a full-length partial (HVP, gradient):
  // route_begin arms the weight-block GEMM epilogues of `mlp`; route_end routes the bias blocks of `full`
  // (or zeros when this rank computed nothing), runs the barrier and sums this rank's slots into `shard`
  void route_begin(size_t base);
  void route_end(const float* full, bool empty, float* shard, size_t rows, size_t base);
  ~dho2g_op();
  // kind 4: this rank's columns of Q^T and Q (n x rows each, column-major), spec in `mat`, and the
  // intermediate y = spec o (Q v) (own rows, then all-gathered to world * ceil(n/G))
  dho2g::DevBuf<float> qrot_t, qrot, qy, qy_loc;
  size_t q_begin = 0, q_rows = 0;
  size_t B = 0, ncls = 0, b0 = 0, b1 = 0;  // this rank's slice of the curvature batch
  double scale = 1.0;
  dho2g_host_hvp fn = nullptr;
  void* user = nullptr;
  std::vector<double> hv_in, hv_out;
  dho2g::HostBuf<float> pin;
  bool weights_loaded = false;
  void load_mlp_input();  // kind 0: this rank's curvature batch and the weights into the model (once per point)
  // h_shard[r] = (H (vscale * vfull))[begin + r]
  void apply(const float* vfull, const float* vscale, float* h_shard, size_t begin, size_t rows, size_t base);
};

namespace dho2g {
struct LzDev {  // device-resident Lanczos scalars (fixed launch sequence; no host round trips)
  double diag[kMaxLanczos + 1];
  double off[kMaxLanczos + 1];
  float sigma[kMaxLanczos + 2];  // lazy column normalisation: v_j = sigma_j * D[:, j]
  double pre, beta;
  int iters, stopped, breakdown, safeguards, need_sg;
  int nonfinite;  // the operator returned non-finite values (dist_lanczos.cpp:80-82): stop, raise on the host
  long long sg_cols;  // sum over safeguard passes of the active column count (gs_flops accounting)
  double gram[2][kMaxLanczos + 1];  // G_j = D_j^T D_i of the last two iterations (recurrence-first form)
};
}  // namespace dho2g

struct dho2g_lanczos {
  dho2g_ctx* ctx = nullptr;
  size_t n = 0, m = 0, begin = 0, end = 0, rows = 0, ldd = 0, base = 0;
  dho2g::DevBuf<float> D;       // ldd x (m+1) column-major, raw (scale sigma_j)
  dho2g::DevBuf<float> h;       // ldd
  dho2g::DevBuf<float> vfull;   // world * base (all_gather target)
  dho2g::DevBuf<dho2g::LzDev> st;
  dho2g::DevBuf<double> part;   // per-CTA partials
  dho2g::DevBuf<double> rankp;  // this rank's partial vector (m+2)
  dho2g::DevBuf<double> allp;   // world x (m+2)
  dho2g::DevBuf<unsigned> ticket;
  dho2g::LzDev host{};          // copy after run
  dho2g_lanczos_opts opts{1, 1e-6, 1e-10};
  dho2g::DevBuf<double> xZ, xev, xam, xamall, xpart;  // extract_ese scratch
  dho2g::DevBuf<float> xU, xUs;
  dho2g::DevBuf<int> xstatus;
  dho2g::DevBuf<double2> xrot;  // split tql2: rotation log (c, s)
  dho2g::DevBuf<int4> xsweep;   // split tql2: per-sweep (mm, cnt, log offset)
  dho2g::DevBuf<int> xnsweep;
  dho2g::DevBuf<double> xd;     // split tql2: eigenvalues in slot order
  dho2g::DevBuf<double> sm_part1, sm_part2;  // fused refresh: per-CTA Gram-Schmidt partials
  dho2g::DevBuf<unsigned long long> sm_bar;  // fused refresh of a diagonal operator: grid-barrier words
  int sm_bar_nb = 0;
  double ms = 0.0;
  // CUDA graph of the refresh launch sequence (world 1)
  cudaGraphExec_t gexec = nullptr;
  const void* gop = nullptr;
  size_t gm = 0;
  unsigned long long ggen = 0;
  const unsigned* gflags = nullptr;
  const unsigned* gflags2 = nullptr;
  bool seen_eager = false, graph_failed = false;
  unsigned long long glaunches = 0;  // kernel launches recorded in the graph
  dho2g::DevBuf<uint64_t> seed_dev;
  dho2g::HostBuf<uint64_t> seed_host;
  dho2g::DevBuf<double> seed_chk;  // [2] own seed halves, [2 world] gathered (multi-rank seed check)
  ~dho2g_lanczos() {
    if (gexec) cudaGraphExecDestroy(gexec);
  }
};

struct dho2g_ese {
  dho2g_ctx* ctx = nullptr;
  size_t n = 0, r = 0, rows = 0, begin = 0, end = 0, ldv = 0;
  dho2g::DevBuf<float> V;  // ldv x r column-major (column signs in `sign`)
  std::vector<double> eigvals;
  std::vector<float> sign;
  dho2g::DevBuf<double> ev_dev;
};

namespace dho2g {
void lanczos_run_into(dho2g_lanczos* lz, dho2g_op* op, uint64_t seed);
// Host waits that notice a missing / failed rank (NCCL async errors, timeout) when a communicator exists.
void wait_stream(dho2g_ctx* ctx, cudaStream_t s);
void nccl_call(dho2g_ctx* ctx, ncclResult_t r, const char* what);
void nccl_settle(dho2g_ctx* ctx, const char* what);
void gemm_trace_set(unsigned long long* buf, int filter);  // test hook (gemm.cu)
void gemm_trace1_set(unsigned long long* buf);  // the same for the single-CTA kernel (8 stamps per CTA)
// out[0] = scale * <a, b> over rows (single CTA, deterministic)
void dot_dev(cudaStream_t st, const float* a, const float* b, size_t rows, double scale, double* out);
void lanczos_alloc(dho2g_lanczos* lz, dho2g_ctx* ctx, size_t n, size_t m);
void extract_ese_into(dho2g_ctx* ctx, dho2g_lanczos* lz, size_t k, size_t l, dho2g_ese* ese);
// Ritz vectors on the tensor cores (3xTF32, ritz_tc.cu); supported for r <= 64, me <= 96.
bool ritz_tc_supported(int me, int r);
void ritz_tc(dho2g_ctx* ctx, const float* D, size_t ldd, int me, const float* U, const float* sigma, int r, float* V,
             size_t ldv, size_t rows, DevBuf<float>& uscratch);
}  // namespace dho2g

// ------------------------------------------------------------------------- optimizer / update
struct dho2g_opt {
  dho2g_ctx* ctx = nullptr;
  dho2g_base_cfg cfg{};
  size_t n = 0;  // local rows
  size_t t = 0;
  dho2g::DevBuf<float> m, v, s;
  dho2g::DevBuf<double> part, rank1, rank2, all1, all2;
  dho2g::DevBuf<unsigned> ticket;
  dho2g::DevBuf<int> bad;  // non-finite gradient flag
  dho2g::DevBuf<unsigned long long> sbar;  // small-n fused update: grid-barrier words
  int sbar_nb = 0;
};

namespace dho2g {
struct UpdateArgs {
  const float* g;    // rows (shard)
  const float* pi;   // rows or null
  float* w_a;        // rows, updated in place (null: only materialize)
  const float* w_decay;  // rows, w read by the AdamW term (null: w_a)
  float* newton_out; // optional materialized newton (rows)
  float* base_out;   // optional materialized base (rows)
  double alpha, sigma, floor;
};
void opt_alloc(dho2g_opt* o, dho2g_ctx* ctx, const dho2g_base_cfg& cfg, size_t rows);
// One split update (optimizer.cpp:81-117 + BaseOptimizer::step) on this rank's rows.
void split_update(dho2g_opt* o, const dho2g_ese* ese, const UpdateArgs& a);
void admm_w_update_dev(cudaStream_t s, size_t n, double sigma, const float* w_a, const float* pi, float* w);
void admm_dual_update_dev(cudaStream_t s, size_t n, double sigma, const float* w_a, const float* w, float* pi);
void check_opt_flags(dho2g_opt* o);
}  // namespace dho2g

struct dho2g_trainer;
namespace dho2g {
dho2g_ctx* trainer_ctx(dho2g_trainer* tr);
dho2g_trainer* trainer_create(dho2g_ctx* ctx, const dho2g_train_cfg* cfg, dho2g_mlp* mlp, const double* X,
                              const double* y, size_t N, size_t ncls, uint64_t dataset_seed, const double* w0,
                              int workers, int host_resident, dho2g_op* quad = nullptr);
void trainer_step(dho2g_trainer* tr, size_t steps, int with_eval);
void trainer_run(dho2g_trainer* tr);
void trainer_params(dho2g_trainer* tr, double* w);
size_t trainer_rows(dho2g_trainer* tr);
void trainer_metrics_ex(dho2g_trainer* tr, size_t max_rows, int64_t* outer, int64_t* inner, double* wallclock);
void trainer_metrics(dho2g_trainer* tr, size_t max_rows, double* loss, double* acc, double* resid, int64_t* epoch,
                     int* refresh);
double trainer_last_loss(dho2g_trainer* tr);
bool trainer_stat(dho2g_trainer* tr, const std::string& key, double* v);
void trainer_eigvals(dho2g_trainer* tr, double* vals, size_t* count);
void trainer_destroy(dho2g_trainer* tr);
}  // namespace dho2g

// In-process rendezvous for several ranks on one GPU (dho2g_comm_init_local; collectives in host.cu).
struct dho2g_fabric {
  int world = 1;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  unsigned long long gen = 0;
  std::vector<const void*> send;
  std::vector<cudaEvent_t> ready, done;
  explicit dho2g_fabric(int w) : world(w), send(w, nullptr), ready(w, nullptr), done(w, nullptr) {
    for (int r = 0; r < w; ++r) {
      DHO2G_CUDA(cudaEventCreateWithFlags(&ready[r], cudaEventDisableTiming));
      DHO2G_CUDA(cudaEventCreateWithFlags(&done[r], cudaEventDisableTiming));
    }
  }
  ~dho2g_fabric() {
    for (int r = 0; r < world; ++r) {
      cudaEventDestroy(ready[r]);
      cudaEventDestroy(done[r]);
    }
  }
  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    const unsigned long long g = gen;
    if (++arrived == world) {
      arrived = 0;
      ++gen;
      cv.notify_all();
    } else {
      if (!cv.wait_for(lk, std::chrono::seconds(600), [&] { return gen != g; }))
        dho2g::fail(DHO2G_DEADLOCK, "local fabric: a rank is missing from the round");
    }
  }
};
