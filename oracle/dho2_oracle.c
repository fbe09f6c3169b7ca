/*
 * TEST INFRASTRUCTURE ONLY — the CPU checker for the DHO2 curvature-and-update path.
 *
 * A plain-C, fp64 restatement of the reference algorithm (/root/reference/proj, cited
 * file:line below, paths relative to proj/). It is never linked into the product and
 * never measured as the product: only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg load it. Parity is PINNED: tests/test_oracle_pin.py checks every
 * function here bit-for-bit (or to the reference test's own tolerance) against the
 * unmodified reference library compiled into oracle/_ref/libdho2ref.so, and against the
 * known-answer cases of the reference's own doctest suites.
 *
 * Arithmetic order follows the reference exactly (left-to-right serial dots, 16-sample
 * chunk partials merged in chunk order, ascending-rank collective sums) so that results
 * are bitwise identical, which is what the pin tests assert.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_OK 0
#define ORC_DIMENSION 1
#define ORC_ARGUMENT 2
#define ORC_NUMERIC 3

static const char* g_err = "";
const char* orc_last_error(void) { return g_err; }
#define FAIL(code, msg) \
  do {                  \
    g_err = (msg);      \
    return (code);      \
  } while (0)

/* ------------------------------------------------------------------ rng.hpp:14-68 */
typedef struct {
  uint64_t state;
  double spare;
  int have_spare;
} orc_rng;

static void rng_init(orc_rng* r, uint64_t seed) {
  r->state = seed;
  r->spare = 0.0;
  r->have_spare = 0;
}
static uint64_t rng_u64(orc_rng* r) { /* SplitMix64, rng.hpp:18-23 */
  uint64_t z = (r->state += 0x9e3779b97f4a7c15ULL);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
static double rng_uniform(orc_rng* r) { return (double)(rng_u64(r) >> 11) * 0x1.0p-53; }
static uint64_t rng_below(orc_rng* r, uint64_t bound) { /* rng.hpp:29-35 */
  const uint64_t threshold = (0 - bound) % bound;
  for (;;) {
    const uint64_t x = rng_u64(r);
    if (x >= threshold) return x % bound;
  }
}
static double rng_normal(orc_rng* r) { /* Box-Muller with spare, rng.hpp:37-50 */
  if (r->have_spare) {
    r->have_spare = 0;
    return r->spare;
  }
  const double u1 = ((double)(rng_u64(r) >> 11) + 1.0) * 0x1.0p-53;
  const double u2 = rng_uniform(r);
  const double radius = sqrt(-2.0 * log(u1));
  const double angle = 2.0 * 3.141592653589793 * u2;
  r->spare = radius * sin(angle);
  r->have_spare = 1;
  return radius * cos(angle);
}
static void rng_shuffle(orc_rng* r, uint64_t* v, size_t n) { /* Fisher-Yates, rng.hpp:56-62 */
  for (size_t i = n; i > 1; --i) {
    const size_t j = (size_t)rng_below(r, i);
    const uint64_t t = v[i - 1];
    v[i - 1] = v[j];
    v[j] = t;
  }
}

void orc_rng_u64(uint64_t seed, size_t n, uint64_t* out) {
  orc_rng r;
  rng_init(&r, seed);
  for (size_t i = 0; i < n; ++i) out[i] = rng_u64(&r);
}
void orc_rng_normal(uint64_t seed, size_t n, double* out) {
  orc_rng r;
  rng_init(&r, seed);
  for (size_t i = 0; i < n; ++i) out[i] = rng_normal(&r);
}
void orc_rng_uniform(uint64_t seed, size_t n, double* out) {
  orc_rng r;
  rng_init(&r, seed);
  for (size_t i = 0; i < n; ++i) out[i] = rng_uniform(&r);
}
void orc_rng_shuffle_iota(uint64_t seed, size_t n, uint64_t* out) {
  orc_rng r;
  rng_init(&r, seed);
  for (size_t i = 0; i < n; ++i) out[i] = i;
  rng_shuffle(&r, out, n);
}

/* trainer.cpp:41-46 (file-local in the reference, restated) */
uint64_t orc_mix_seed(uint64_t seed, uint64_t salt) {
  uint64_t z = seed + 0x9e3779b97f4a7c15ULL * (salt + 1);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

/* oracle.cpp:56-62 */
void orc_epoch_permutation(size_t N, uint64_t shuffle_seed, uint64_t epoch, uint64_t* out) {
  orc_rng_shuffle_iota(shuffle_seed * 0x9e3779b97f4a7c15ULL + epoch + 1, N, out);
}

/* collectives.cpp:10-20 */
int orc_shard(size_t n, int world, int rank, size_t* begin, size_t* end) {
  if (world < 1) FAIL(ORC_ARGUMENT, "Shard: world_size must be >= 1");
  if (rank < 0 || rank >= world) FAIL(ORC_ARGUMENT, "Shard: rank out of range");
  const size_t base = (n + (size_t)world - 1) / (size_t)world;
  size_t b = base * (size_t)rank;
  if (b > n) b = n;
  size_t e = b + base;
  if (e > n) e = n;
  *begin = b;
  *end = e;
  return ORC_OK;
}

/* lanczos.cpp:10-16 */
int orc_lanczos_budget(size_t k, size_t l, size_t n, size_t* m) {
  if (n < 1) FAIL(ORC_ARGUMENT, "lanczos_budget: n must be >= 1");
  if (k + l < 1) FAIL(ORC_ARGUMENT, "lanczos_budget: k+l must be >= 1");
  if (k + l > n) FAIL(ORC_ARGUMENT, "lanczos_budget: k+l exceeds the dimension");
  const size_t log_term = (size_t)ceil(2.0 * log((double)n));
  size_t v = 4 * (k + l);
  if (log_term > v) v = log_term;
  *m = v < n ? v : n;
  return ORC_OK;
}

/* linalg.cpp:34-39: serial left-to-right */
static double dot(const double* a, const double* b, size_t n) {
  double acc = 0.0;
  for (size_t i = 0; i < n; ++i) acc += a[i] * b[i];
  return acc;
}
static int all_finite(const double* v, size_t n) {
  for (size_t i = 0; i < n; ++i)
    if (!isfinite(v[i])) return 0;
  return 1;
}

/* lanczos.cpp:18-26 */
int orc_seeded_unit_gaussian(size_t n, uint64_t seed, double* v) {
  orc_rng_normal(seed * 0x9e3779b97f4a7c15ULL + 0x1234567ULL, n, v);
  const double nrm = sqrt(dot(v, v, n));
  if (nrm == 0.0) FAIL(ORC_NUMERIC, "seeded_unit_gaussian: zero draw");
  const double inv = 1.0 / nrm;
  for (size_t i = 0; i < n; ++i) v[i] *= inv;
  return ORC_OK;
}

/* ------------------------------------------------------------ MLP oracle.cpp:288-687 */
typedef struct {
  int nl; /* number of layer sizes (layers = nl-1) */
  const size_t* sizes;
  size_t w_off[64], b_off[64];
  size_t dim;
  int relu;    /* 0 tanh, 1 relu */
  int mse;     /* 0 softmax-CE, 1 MSE */
} mlp_t;

static int mlp_make(mlp_t* m, const size_t* sizes, int nl, int act, int loss) {
  if (nl < 3) FAIL(ORC_ARGUMENT, "mlp oracle: need at least one hidden layer");
  if (nl > 64) FAIL(ORC_ARGUMENT, "mlp oracle: too many layers for the oracle");
  for (int i = 0; i < nl; ++i)
    if (sizes[i] == 0) FAIL(ORC_ARGUMENT, "mlp oracle: zero layer size");
  m->nl = nl;
  m->sizes = sizes;
  size_t off = 0; /* layer-major, W (out x in row-major) then b: oracle.cpp:312-323 */
  for (int t = 0; t + 1 < nl; ++t) {
    m->w_off[t] = off;
    off += sizes[t] * sizes[t + 1];
    m->b_off[t] = off;
    off += sizes[t + 1];
  }
  m->dim = off;
  m->relu = act == 1;
  m->mse = loss == 1;
  return ORC_OK;
}

int orc_mlp_dim(const size_t* sizes, int nl, size_t* dim) {
  mlp_t m;
  int rc = mlp_make(&m, sizes, nl, 0, 0);
  if (rc) return rc;
  *dim = m.dim;
  return ORC_OK;
}

/* oracle.cpp:386-394 */
int orc_mlp_init(const size_t* sizes, int nl, uint64_t seed, double* w) {
  mlp_t m;
  int rc = mlp_make(&m, sizes, nl, 0, 0);
  if (rc) return rc;
  memset(w, 0, m.dim * sizeof(double));
  orc_rng r;
  rng_init(&r, seed * 0x9e3779b97f4a7c15ULL + 17);
  for (int t = 0; t + 1 < nl; ++t) {
    const double sd = 1.0 / sqrt((double)sizes[t]);
    for (size_t k = 0; k < sizes[t] * sizes[t + 1]; ++k) w[m.w_off[t] + k] = sd * rng_normal(&r);
  }
  return ORC_OK;
}

static inline double act_apply(const mlp_t* m, double z) { return m->relu ? (z > 0.0 ? z : 0.0) : tanh(z); }
static inline double act_prime(const mlp_t* m, double a) { return m->relu ? (a > 0.0 ? 1.0 : 0.0) : 1.0 - a * a; }

static int check_batch(const mlp_t* m, size_t B, size_t ncls) {
  if (B == 0) FAIL(ORC_ARGUMENT, "mlp oracle: empty batch");
  const size_t out = m->sizes[m->nl - 1];
  if (!m->mse) {
    if (ncls == 0 || ncls != out) FAIL(ORC_ARGUMENT, "mlp oracle: softmax_ce needs n_classes == output layer size");
  } else if (ncls > 0) {
    if (ncls != out) FAIL(ORC_ARGUMENT, "mlp oracle: mse one-hot targets need n_classes == output layer size");
  } else if (out != 1) {
    FAIL(ORC_ARGUMENT, "mlp oracle: regression targets need output layer size 1");
  }
  return ORC_OK;
}

/* per-sample scratch: a[t], ra[t], delta[t], rdelta[t] for t = 0..L */
typedef struct {
  double **a, **ra, **d, **rd;
  double* target;
  double* pool;
} scratch_t;

static int scratch_alloc(scratch_t* s, const mlp_t* m) {
  size_t tot = 0;
  for (int t = 0; t < m->nl; ++t) tot += m->sizes[t];
  s->pool = (double*)calloc(4 * tot + m->sizes[m->nl - 1], sizeof(double));
  s->a = (double**)malloc(4 * (size_t)m->nl * sizeof(double*));
  if (!s->pool || !s->a) return 0;
  s->ra = s->a + m->nl;
  s->d = s->ra + m->nl;
  s->rd = s->d + m->nl;
  double* p = s->pool;
  for (int t = 0; t < m->nl; ++t) { s->a[t] = p; p += m->sizes[t]; }
  for (int t = 0; t < m->nl; ++t) { s->ra[t] = p; p += m->sizes[t]; }
  for (int t = 0; t < m->nl; ++t) { s->d[t] = p; p += m->sizes[t]; }
  for (int t = 0; t < m->nl; ++t) { s->rd[t] = p; p += m->sizes[t]; }
  s->target = p;
  return 1;
}
static void scratch_free(scratch_t* s) {
  free(s->pool);
  free(s->a);
}

static void forward(const mlp_t* m, const double* w, scratch_t* s) { /* oracle.cpp:413-421 */
  const int L = m->nl - 1;
  for (int t = 0; t < L; ++t) {
    const size_t in = m->sizes[t], out = m->sizes[t + 1];
    const int last = t + 1 == L;
    for (size_t o = 0; o < out; ++o) {
      double z = w[m->b_off[t] + o];
      const double* wr = w + m->w_off[t] + o * in;
      for (size_t k = 0; k < in; ++k) z += wr[k] * s->a[t][k];
      s->a[t + 1][o] = last ? z : act_apply(m, z);
    }
  }
}

static void set_target(const mlp_t* m, scratch_t* s, double label, size_t ncls) {
  const size_t out = m->sizes[m->nl - 1];
  for (size_t o = 0; o < out; ++o) s->target[o] = 0.0;
  if (ncls > 0) s->target[(size_t)label] = 1.0;
  else s->target[0] = label;
}

#define CHUNK 16 /* kernels.hpp:22 kBatchChunk */

/* oracle.cpp:400-449 */
int orc_mlp_value(const size_t* sizes, int nl, int act, int loss, const double* w, const double* X,
                  const double* y, size_t B, size_t ncls, double* out_val) {
  mlp_t m;
  int rc = mlp_make(&m, sizes, nl, act, loss);
  if (rc) return rc;
  if ((rc = check_batch(&m, B, ncls))) return rc;
  scratch_t s;
  if (!scratch_alloc(&s, &m)) FAIL(ORC_NUMERIC, "oom");
  const size_t D = sizes[0], L = (size_t)nl - 1, O = sizes[nl - 1];
  double total = 0.0;
  for (size_t c0 = 0; c0 < B; c0 += CHUNK) {
    double acc = 0.0;
    const size_t c1 = c0 + CHUNK < B ? c0 + CHUNK : B;
    for (size_t i = c0; i < c1; ++i) {
      memcpy(s.a[0], X + i * D, D * sizeof(double));
      forward(&m, w, &s);
      const double* o = s.a[L];
      if (!m.mse) {
        const size_t lbl = (size_t)y[i];
        double mx = o[0];
        for (size_t j = 0; j < O; ++j) mx = o[j] > mx ? o[j] : mx;
        double lse = 0.0;
        for (size_t j = 0; j < O; ++j) lse += exp(o[j] - mx);
        acc += mx + log(lse) - o[lbl];
      } else {
        set_target(&m, &s, y[i], ncls);
        for (size_t j = 0; j < O; ++j) {
          const double d = o[j] - s.target[j];
          acc += 0.5 * d * d;
        }
      }
    }
    total += acc;
  }
  scratch_free(&s);
  *out_val = total / (double)B;
  return ORC_OK;
}

/* oracle.cpp:649-685 */
int orc_mlp_accuracy(const size_t* sizes, int nl, int act, int loss, const double* w, const double* X,
                     const double* y, size_t B, size_t ncls, double* acc_out) {
  if (ncls == 0) {
    *acc_out = -1.0;
    return ORC_OK;
  }
  mlp_t m;
  int rc = mlp_make(&m, sizes, nl, act, loss);
  if (rc) return rc;
  if ((rc = check_batch(&m, B, ncls))) return rc;
  scratch_t s;
  if (!scratch_alloc(&s, &m)) FAIL(ORC_NUMERIC, "oom");
  const size_t D = sizes[0], L = (size_t)nl - 1, O = sizes[nl - 1];
  size_t correct = 0;
  for (size_t i = 0; i < B; ++i) {
    memcpy(s.a[0], X + i * D, D * sizeof(double));
    forward(&m, w, &s);
    size_t best = 0;
    for (size_t j = 1; j < O; ++j)
      if (s.a[L][j] > s.a[L][best]) best = j;
    if (best == (size_t)y[i]) ++correct;
  }
  scratch_free(&s);
  *acc_out = (double)correct / (double)B;
  return ORC_OK;
}

/* output-layer delta (oracle.cpp:476-495) and, when rd != NULL, R{delta} (:572-599) */
static void output_delta(const mlp_t* m, scratch_t* s, double label, size_t ncls, double inv_b, int with_r) {
  const int L = m->nl - 1;
  const size_t O = m->sizes[L];
  double* dl = s->d[L];
  const double* o = s->a[L];
  if (!m->mse) {
    const size_t lbl = (size_t)label;
    double mx = o[0];
    for (size_t j = 0; j < O; ++j) mx = o[j] > mx ? o[j] : mx;
    double den = 0.0;
    for (size_t j = 0; j < O; ++j) den += exp(o[j] - mx);
    if (!with_r) {
      for (size_t j = 0; j < O; ++j) dl[j] = (exp(o[j] - mx) / den - (j == lbl ? 1.0 : 0.0)) * inv_b;
      return;
    }
    double sdot = 0.0;
    const double* ro = s->ra[L];
    for (size_t j = 0; j < O; ++j) {
      const double soft = exp(o[j] - mx) / den;
      dl[j] = (soft - (j == lbl ? 1.0 : 0.0)) * inv_b;
      s->target[j] = soft;
      sdot += soft * ro[j];
    }
    for (size_t j = 0; j < O; ++j) s->rd[L][j] = s->target[j] * (ro[j] - sdot) * inv_b;
  } else {
    set_target(m, s, label, ncls);
    for (size_t j = 0; j < O; ++j) dl[j] = (o[j] - s->target[j]) * inv_b;
    if (with_r)
      for (size_t j = 0; j < O; ++j) s->rd[L][j] = s->ra[L][j] * inv_b;
  }
}

/* oracle.cpp:451-522 */
int orc_mlp_grad(const size_t* sizes, int nl, int act, int loss, const double* w, const double* X,
                 const double* y, size_t B, size_t ncls, double* g) {
  mlp_t m;
  int rc = mlp_make(&m, sizes, nl, act, loss);
  if (rc) return rc;
  if ((rc = check_batch(&m, B, ncls))) return rc;
  scratch_t s;
  if (!scratch_alloc(&s, &m)) FAIL(ORC_NUMERIC, "oom");
  double* part = (double*)malloc(m.dim * sizeof(double));
  const size_t D = sizes[0];
  const int L = nl - 1;
  const double inv_b = 1.0 / (double)B;
  memset(g, 0, m.dim * sizeof(double));
  for (size_t c0 = 0; c0 < B; c0 += CHUNK) {
    memset(part, 0, m.dim * sizeof(double));
    const size_t c1 = c0 + CHUNK < B ? c0 + CHUNK : B;
    for (size_t i = c0; i < c1; ++i) {
      memcpy(s.a[0], X + i * D, D * sizeof(double));
      forward(&m, w, &s);
      output_delta(&m, &s, y[i], ncls, inv_b, 0);
      for (int t = L - 1; t >= 0; --t) {
        const size_t in = sizes[t], out = sizes[t + 1];
        const double* d = s.d[t + 1];
        for (size_t o = 0; o < out; ++o) {
          const double dv = d[o];
          double* gr = part + m.w_off[t] + o * in;
          for (size_t k = 0; k < in; ++k) gr[k] += dv * s.a[t][k];
          part[m.b_off[t] + o] += dv;
        }
        if (t > 0) {
          for (size_t k = 0; k < in; ++k) {
            double u = 0.0;
            for (size_t o = 0; o < out; ++o) u += w[m.w_off[t] + o * in + k] * d[o];
            s.d[t][k] = u * act_prime(&m, s.a[t][k]);
          }
        }
      }
    }
    for (size_t i = 0; i < m.dim; ++i) g[i] += part[i]; /* chunk-order merge, :517-520 */
  }
  free(part);
  scratch_free(&s);
  return ORC_OK;
}

/* oracle.cpp:524-647 (Pearlmutter forward-over-reverse) */
int orc_mlp_hvp(const size_t* sizes, int nl, int act, int loss, const double* w, const double* v,
                const double* X, const double* y, size_t B, size_t ncls, double* hv) {
  mlp_t m;
  int rc = mlp_make(&m, sizes, nl, act, loss);
  if (rc) return rc;
  if ((rc = check_batch(&m, B, ncls))) return rc;
  scratch_t s;
  if (!scratch_alloc(&s, &m)) FAIL(ORC_NUMERIC, "oom");
  double* part = (double*)malloc(m.dim * sizeof(double));
  const size_t D = sizes[0];
  const int L = nl - 1;
  const double inv_b = 1.0 / (double)B;
  const int tanh_act = !m.relu;
  memset(hv, 0, m.dim * sizeof(double));
  for (size_t c0 = 0; c0 < B; c0 += CHUNK) {
    memset(part, 0, m.dim * sizeof(double));
    const size_t c1 = c0 + CHUNK < B ? c0 + CHUNK : B;
    for (size_t i = c0; i < c1; ++i) {
      memcpy(s.a[0], X + i * D, D * sizeof(double));
      for (size_t k = 0; k < D; ++k) s.ra[0][k] = 0.0;
      for (int t = 0; t < L; ++t) { /* forward + R-forward :544-565 */
        const size_t in = sizes[t], out = sizes[t + 1];
        const int last = t + 1 == L;
        for (size_t o = 0; o < out; ++o) {
          double z = w[m.b_off[t] + o];
          double rz = v[m.b_off[t] + o];
          const double* wr = w + m.w_off[t] + o * in;
          const double* vr = v + m.w_off[t] + o * in;
          for (size_t k = 0; k < in; ++k) {
            z += wr[k] * s.a[t][k];
            rz += vr[k] * s.a[t][k] + wr[k] * s.ra[t][k];
          }
          if (last) {
            s.a[t + 1][o] = z;
            s.ra[t + 1][o] = rz;
          } else {
            const double a = act_apply(&m, z);
            s.a[t + 1][o] = a;
            s.ra[t + 1][o] = act_prime(&m, a) * rz;
          }
        }
      }
      output_delta(&m, &s, y[i], ncls, inv_b, 1);
      for (int t = L - 1; t >= 0; --t) { /* backward + R-backward :602-638 */
        const size_t in = sizes[t], out = sizes[t + 1];
        const double* d = s.d[t + 1];
        const double* rd = s.rd[t + 1];
        for (size_t o = 0; o < out; ++o) {
          const double dv = d[o], rdv = rd[o];
          double* hr = part + m.w_off[t] + o * in;
          for (size_t k = 0; k < in; ++k) hr[k] += rdv * s.a[t][k] + dv * s.ra[t][k];
          part[m.b_off[t] + o] += rdv;
        }
        if (t > 0) {
          for (size_t k = 0; k < in; ++k) {
            double u = 0.0, ru = 0.0;
            for (size_t o = 0; o < out; ++o) {
              const double wk = w[m.w_off[t] + o * in + k];
              const double vk = v[m.w_off[t] + o * in + k];
              u += wk * d[o];
              ru += vk * d[o] + wk * rd[o];
            }
            const double a = s.a[t][k];
            const double ap = act_prime(&m, a);
            s.d[t][k] = u * ap;
            double rap_rz = 0.0;
            if (tanh_act && ap != 0.0) rap_rz = -2.0 * a * s.ra[t][k];
            s.rd[t][k] = ru * ap + u * rap_rz;
          }
        }
      }
    }
    for (size_t i = 0; i < m.dim; ++i) hv[i] += part[i];
  }
  free(part);
  scratch_free(&s);
  return ORC_OK;
}

/* ---------------------------------------------- tridiagonal eigensolve linalg.cpp:140-226 */
/* Implicit-shift QL (EISPACK tql2 structure); z is n x n column-major. */
static int ql_implicit(double* d, double* e /* length n, e[n-1] scratch */, double* z, size_t n) {
  if (n <= 1) return ORC_OK;
  const double eps = 2.220446049250313e-16;
  e[n - 1] = 0.0;
  for (size_t l = 0; l < n; ++l) {
    int iter = 0;
    size_t mm;
    do {
      for (mm = l; mm + 1 < n; ++mm) {
        const double dd = fabs(d[mm]) + fabs(d[mm + 1]);
        if (fabs(e[mm]) <= eps * dd) break;
      }
      if (mm != l) {
        if (iter++ == 60) FAIL(ORC_NUMERIC, "tridiag_eig: QL iteration did not converge");
        double g = (d[l + 1] - d[l]) / (2.0 * e[l]);
        double r = hypot(g, 1.0);
        g = d[mm] - d[l] + e[l] / (g + copysign(r, g));
        double s = 1.0, c = 1.0, p = 0.0;
        int underflow = 0;
        for (size_t ii = mm; ii-- > l;) {
          double f = s * e[ii];
          const double b = c * e[ii];
          r = hypot(f, g);
          e[ii + 1] = r;
          if (r == 0.0) {
            d[ii + 1] -= p;
            e[mm] = 0.0;
            underflow = 1;
            break;
          }
          s = f / r;
          c = g / r;
          g = d[ii + 1] - p;
          r = (d[ii] - g) * s + 2.0 * c * b;
          p = s * r;
          d[ii + 1] = g + p;
          g = c * r - b;
          double* z0 = z + ii * n;
          double* z1 = z + (ii + 1) * n;
          for (size_t k = 0; k < n; ++k) {
            f = z1[k];
            z1[k] = s * z0[k] + c * f;
            z0[k] = c * z0[k] - s * f;
          }
        }
        if (underflow) continue;
        d[l] -= p;
        e[l] = g;
        e[mm] = 0.0;
      }
    } while (mm != l);
  }
  return ORC_OK;
}

int orc_tridiag_eig(size_t n, const double* diag, const double* off, double* vals, double* vecs) {
  if (n == 0) FAIL(ORC_ARGUMENT, "tridiag_eig: empty matrix");
  if (!all_finite(diag, n) || (n > 1 && !all_finite(off, n - 1))) FAIL(ORC_NUMERIC, "tridiag_eig: non-finite entries");
  double* d = (double*)malloc(n * sizeof(double));
  double* e = (double*)malloc(n * sizeof(double));
  double* z = (double*)calloc(n * n, sizeof(double));
  size_t* order = (size_t*)malloc(n * sizeof(size_t));
  memcpy(d, diag, n * sizeof(double));
  if (n > 1) memcpy(e, off, (n - 1) * sizeof(double));
  for (size_t i = 0; i < n; ++i) z[i * n + i] = 1.0;
  int rc = ql_implicit(d, e, z, n);
  if (rc == ORC_OK) {
    /* stable ascending order (insertion sort is stable) */
    for (size_t i = 0; i < n; ++i) {
      size_t j = i;
      while (j > 0 && d[i] < d[order[j - 1]]) {
        order[j] = order[j - 1];
        --j;
      }
      order[j] = i;
    }
    for (size_t j = 0; j < n; ++j) {
      vals[j] = d[order[j]];
      memcpy(vecs + j * n, z + order[j] * n, n * sizeof(double));
    }
  }
  free(d);
  free(e);
  free(z);
  free(order);
  return rc;
}

/* ------------------------------------------- QuadraticOracle (oracle.cpp:233-286) */
/* Constructor checks (:234-240) on the spectrum. */
int orc_quadratic_check(const double* spec, size_t n) {
  if (n == 0) FAIL(ORC_ARGUMENT, "quadratic oracle: empty spectrum");
  for (size_t i = 0; i < n; ++i)
    if (spec[i] == 0.0 || !isfinite(spec[i]))
      FAIL(ORC_ARGUMENT, "quadratic oracle: spectrum entries must be nonzero and finite");
  return ORC_OK;
}

/* Rotation Q (n x n column-major, :241-257): Rng(seed*phi) normals, then per column two passes
 * of modified Gram-Schmidt against the earlier columns and a normalisation. */
int orc_quadratic_rotation(size_t n, uint64_t rotation_seed, double* Q) {
  orc_rng_normal(rotation_seed * 0x9e3779b97f4a7c15ULL, n * n, Q);
  for (size_t j = 0; j < n; ++j) {
    double* col = Q + j * n;
    for (int pass = 0; pass < 2; ++pass)
      for (size_t i = 0; i < j; ++i) {
        const double* qi = Q + i * n;
        const double c = dot(qi, col, n);
        for (size_t t = 0; t < n; ++t) col[t] += -c * qi[t];
      }
    const double nrm = sqrt(dot(col, col, n));
    if (nrm < 1e-12) FAIL(ORC_NUMERIC, "quadratic oracle: degenerate rotation draw");
    const double inv = 1.0 / nrm;
    for (size_t t = 0; t < n; ++t) col[t] *= inv;
  }
  return ORC_OK;
}

/* apply_h (:262-272): diag(spec) x, or Q^T (spec o (Q x)) when rotated (Q != NULL). */
void orc_quadratic_apply(size_t n, const double* spec, const double* Q, const double* x, double* out) {
  if (!Q) {
    for (size_t i = 0; i < n; ++i) out[i] = spec[i] * x[i];
    return;
  }
  double* qx = (double*)malloc(n * sizeof(double));
  for (size_t i = 0; i < n; ++i) { /* linalg::matvec: row i of column-major Q */
    double acc = 0.0;
    for (size_t j = 0; j < n; ++j) acc += Q[j * n + i] * x[j];
    qx[i] = acc * spec[i];
  }
  for (size_t j = 0; j < n; ++j) out[j] = dot(Q + j * n, qx, n); /* matvec_transpose */
  free(qx);
}

/* ------------------------------------------- operators for the Lanczos checker */
typedef struct {
  int kind; /* 0 dense symmetric col-major, 1 diagonal / rotated quadratic, 2 MLP hvp */
  size_t n;
  const double* mat;
  const size_t* sizes;
  int n_sizes, act, loss;
  const double* w;
  const double* X;
  const double* y;
  size_t B, ncls;
  uint64_t rot_seed;  /* kind 1: QuadraticOracle(mat, rot_seed) */
  const double* rot;  /* kind 1, rot_seed != 0: its rotation Q (orc_quadratic_rotation) */
} orc_op;

static int apply_op(const orc_op* op, const double* v, double* out) {
  const size_t n = op->n;
  if (op->kind == 0) {
    for (size_t i = 0; i < n; ++i) {
      double acc = 0.0;
      for (size_t j = 0; j < n; ++j) acc += op->mat[j * n + i] * v[j];
      out[i] = acc;
    }
    return ORC_OK;
  }
  if (op->kind == 1) { /* QuadraticOracle::apply_h, oracle.cpp:262-272 */
    orc_quadratic_apply(n, op->mat, op->rot_seed ? op->rot : NULL, v, out);
    return ORC_OK;
  }
  return orc_mlp_hvp(op->sizes, op->n_sizes, op->act, op->loss, op->w, v, op->X, op->y, op->B, op->ncls, out);
}

/* lanczos.cpp:82-94 */
static void sign_normalize(double* V, size_t n, size_t cols) {
  for (size_t j = 0; j < cols; ++j) {
    double* c = V + j * n;
    size_t best = 0;
    for (size_t i = 1; i < n; ++i)
      if (fabs(c[i]) > fabs(c[best])) best = i;
    if (c[best] < 0.0)
      for (size_t i = 0; i < n; ++i) c[i] *= -1.0;
  }
}

/*
 * dist_lanczos.cpp:31-119 with C simulated ranks (collectives.cpp:310-324 ascending-rank sums)
 * followed by extract_ese_distributed (:121-158). C == 1 is lanczos_single + extract_ese.
 * basis (optional) receives the assembled n x (m+1) column-major D (iters+1 columns filled,
 * iters columns after breakdown). eigvecs is n x (k_eff+l_eff).
 */
int orc_lanczos(const orc_op* op, int C, size_t m, uint64_t seed, int safeguard, double safeguard_ratio,
                double breakdown_rtol, size_t k, size_t l, double* diag, double* off, size_t* iters_out,
                int* breakdown_out, size_t* safeguards_out, double* basis, double* eigvals, double* eigvecs) {
  const size_t n = op->n;
  if (m < 1 || m > n) FAIL(ORC_ARGUMENT, "lanczos_distributed: need 1 <= m <= n");
  if (C < 1) FAIL(ORC_ARGUMENT, "run_workers: world_size must be >= 1");
  double* D = (double*)calloc(n * (m + 1), sizeof(double)); /* global index space; rank r owns rows [b_r,e_r) */
  double* h = (double*)malloc(n * sizeof(double));
  double* v = (double*)malloc(n * sizeof(double));
  double* coeffs = (double*)malloc((m + 1) * sizeof(double));
  double* partial = (double*)malloc((m + 1) * sizeof(double));
  double* next = (double*)malloc(n * sizeof(double));
  size_t* sb = (size_t*)malloc(2 * (size_t)C * sizeof(size_t));
  int rc = ORC_OK;
  for (int r = 0; r < C; ++r) orc_shard(n, C, r, &sb[2 * r], &sb[2 * r + 1]);
  memset(diag, 0, (m + 1) * sizeof(double));
  memset(off, 0, m * sizeof(double));
  size_t iters = m, safeguards = 0;
  int breakdown = 0;
  if ((rc = orc_seeded_unit_gaussian(n, seed, D))) goto done;

  for (size_t i = 0; i < m; ++i) {
    memcpy(v, D + i * n, n * sizeof(double)); /* all_gather of column i: exact concatenation */
    if ((rc = apply_op(op, v, h))) goto done;
    if (!all_finite(h, n)) {
      rc = ORC_NUMERIC;
      g_err = "lanczos_distributed: hvp returned non-finite values";
      goto done;
    }
    diag[i] = dot(h, v, n);
    const double pre = sqrt(dot(h, h, n));
    double beta = 0.0;
    for (int pass = 0; pass < 2; ++pass) {
      const size_t active = i + 1; /* project_shard (:58-74) */
      for (int r = 0; r < C; ++r) {
        const size_t b = sb[2 * r], len = sb[2 * r + 1] - b;
        for (size_t j = 0; j <= m; ++j) partial[j] = 0.0;
        for (size_t j = 0; j < active; ++j) partial[j] = dot(D + j * n + b, h + b, len);
        if (r == 0) memcpy(coeffs, partial, (m + 1) * sizeof(double));
        else
          for (size_t j = 0; j <= m; ++j) coeffs[j] += partial[j];
      }
      for (int r = 0; r < C; ++r) {
        const size_t b = sb[2 * r], e = sb[2 * r + 1];
        for (size_t row = b; row < e; ++row) {
          double acc = h[row];
          for (size_t j = 0; j < active; ++j) acc -= D[j * n + row] * coeffs[j];
          next[row] = acc;
        }
      }
      memcpy(h, next, n * sizeof(double));
      double bsq = 0.0; /* all_reduce of per-rank ||h_shard||^2, ascending rank */
      for (int r = 0; r < C; ++r) {
        const size_t b = sb[2 * r], len = sb[2 * r + 1] - b;
        const double loc = dot(h + b, h + b, len);
        bsq = r == 0 ? loc : bsq + loc;
      }
      beta = sqrt(bsq);
      if (pass == 0 && safeguard && beta > breakdown_rtol * pre && beta < safeguard_ratio * pre) {
        ++safeguards;
        continue;
      }
      break;
    }
    if (beta <= breakdown_rtol * pre) {
      iters = i + 1;
      breakdown = 1;
      off[i] = 0.0; /* leading_block(i+1) drops the trailing entries */
      break;
    }
    off[i] = beta;
    for (size_t row = 0; row < n; ++row) D[(i + 1) * n + row] = h[row] / beta;
  }
  if (breakdown) {
    diag[iters] = 0.0;
  }
  *iters_out = iters;
  *breakdown_out = breakdown;
  *safeguards_out = safeguards;
  if (basis) memcpy(basis, D, n * (breakdown ? iters : iters + 1) * sizeof(double));

  if (k + l > 0) { /* extract_ese_distributed :121-158 */
    const size_t me = iters;
    const size_t keff = k < me ? k : me;
    const size_t leff = l < me - keff ? l : me - keff;
    const size_t rr = keff + leff;
    double* vals = (double*)malloc(me * sizeof(double));
    double* U = (double*)malloc(me * me * sizeof(double));
    double* usel = (double*)malloc(me * rr * sizeof(double));
    rc = orc_tridiag_eig(me, diag, off, vals, U);
    if (rc == ORC_OK) {
      for (size_t c = 0; c < rr; ++c) { /* select_extreme_indices lanczos.cpp:72-80 */
        const size_t idx = c < keff ? me - 1 - c : c - keff;
        eigvals[c] = vals[idx];
        memcpy(usel + c * me, U + idx * me, me * sizeof(double));
      }
      /* matmul linalg.cpp:104-115 per shard rows (row blocks are independent) */
      memset(eigvecs, 0, n * rr * sizeof(double));
      for (size_t j = 0; j < rr; ++j)
        for (size_t kk = 0; kk < me; ++kk) {
          const double bkj = usel[j * me + kk];
          if (bkj == 0.0) continue;
          for (size_t row = 0; row < n; ++row) eigvecs[j * n + row] += D[kk * n + row] * bkj;
        }
      sign_normalize(eigvecs, n, rr);
    }
    free(vals);
    free(U);
    free(usel);
  }
done:
  free(D);
  free(h);
  free(v);
  free(coeffs);
  free(partial);
  free(next);
  free(sb);
  return rc;
}

/* ----------------------------------------------------- optimizer.cpp:37-154 */
typedef struct {
  int kind; /* 0 sgd 1 momentum 2 adam 3 adamw */
  double lr, weight_decay, beta1, beta2, eps, momentum;
} orc_base_cfg;

typedef struct {
  orc_base_cfg cfg;
  size_t n, t;
  double *m, *v;
} base_opt;

static void base_init(base_opt* o, const orc_base_cfg* c, size_t n) {
  o->cfg = *c;
  o->n = n;
  o->t = 0;
  o->m = c->kind != 0 ? (double*)calloc(n, sizeof(double)) : NULL;
  o->v = c->kind >= 2 ? (double*)calloc(n, sizeof(double)) : NULL;
}
static void base_free(base_opt* o) {
  free(o->m);
  free(o->v);
}
static int base_step(base_opt* o, const double* g, const double* w, double* d) { /* :37-71 */
  const size_t n = o->n;
  if (!all_finite(g, n)) FAIL(ORC_NUMERIC, "BaseOptimizer: non-finite gradient");
  ++o->t;
  const orc_base_cfg* c = &o->cfg;
  if (c->kind == 0) {
    for (size_t i = 0; i < n; ++i) d[i] = -c->lr * g[i];
  } else if (c->kind == 1) {
    for (size_t i = 0; i < n; ++i) {
      o->m[i] = c->momentum * o->m[i] + g[i];
      d[i] = -c->lr * o->m[i];
    }
  } else {
    const double bc1 = 1.0 - pow(c->beta1, (double)o->t);
    const double bc2 = 1.0 - pow(c->beta2, (double)o->t);
    for (size_t i = 0; i < n; ++i) {
      o->m[i] = c->beta1 * o->m[i] + (1.0 - c->beta1) * g[i];
      o->v[i] = c->beta2 * o->v[i] + (1.0 - c->beta2) * g[i] * g[i];
      const double mhat = o->m[i] / bc1;
      const double vhat = o->v[i] / bc2;
      d[i] = -c->lr * mhat / (sqrt(vhat) + c->eps);
    }
    if (c->kind == 3)
      for (size_t i = 0; i < n; ++i) d[i] -= c->lr * c->weight_decay * w[i];
  }
  return ORC_OK;
}

int orc_base_steps(const orc_base_cfg* c, size_t n, int T, const double* g, const double* w, double* d_out) {
  if (n == 0) FAIL(ORC_ARGUMENT, "BaseOptimizer: zero dimension");
  if (c->lr < 0.0) FAIL(ORC_ARGUMENT, "BaseOptimizer: negative learning rate");
  base_opt o;
  base_init(&o, c, n);
  int rc = ORC_OK;
  for (int t = 0; t < T && rc == ORC_OK; ++t) rc = base_step(&o, g + (size_t)t * n, w, d_out + (size_t)t * n);
  base_free(&o);
  return rc;
}

static double floored_eigval(double a, double fl) { /* :75-79 */
  if (a == 0.0) return fl;
  const double mag = fabs(a) > fl ? fabs(a) : fl;
  return a < 0.0 ? -mag : mag;
}

/* split_deltas :81-117; pi == NULL is fosi_deltas */
static int split_deltas(const double* g, const double* pi, size_t r, const double* eigvals, const double* V,
                        base_opt* base, const double* w, double alpha, double sigma, double fl, double* newton,
                        double* basev, double* work /* 3n + 3r */) {
  const size_t n = base->n;
  double* gt = work;
  double* g2 = work + n;
  double* s = work + 2 * n;
  double* c = work + 3 * n;
  double* nc = c + r;
  double* sc = nc + r;
  for (size_t i = 0; i < n; ++i) gt[i] = pi ? g[i] + pi[i] : g[i];
  if (r > 0) {
    for (size_t j = 0; j < r; ++j) c[j] = dot(V + j * n, gt, n);
    for (size_t j = 0; j < r; ++j) {
      double den = floored_eigval(eigvals[j], fl) + sigma;
      if (fabs(den) < fl) den = den < 0.0 ? -fl : fl;
      nc[j] = c[j] / den;
    }
    for (size_t i = 0; i < n; ++i) {
      double acc = 0.0;
      for (size_t j = 0; j < r; ++j) acc += V[j * n + i] * nc[j];
      newton[i] = acc * -alpha;
    }
    for (size_t i = 0; i < n; ++i) {
      double acc = 0.0;
      for (size_t j = 0; j < r; ++j) acc += V[j * n + i] * c[j];
      g2[i] = gt[i] - acc;
    }
  } else {
    for (size_t i = 0; i < n; ++i) {
      newton[i] = 0.0;
      g2[i] = gt[i];
    }
  }
  int rc = base_step(base, g2, w, s);
  if (rc) return rc;
  if (r > 0) {
    for (size_t j = 0; j < r; ++j) sc[j] = dot(V + j * n, s, n);
    for (size_t i = 0; i < n; ++i) {
      double acc = 0.0;
      for (size_t j = 0; j < r; ++j) acc += V[j * n + i] * sc[j];
      basev[i] = s[i] - acc;
    }
  } else {
    memcpy(basev, s, n * sizeof(double));
  }
  return ORC_OK;
}

int orc_deltas_seq(const orc_base_cfg* c, size_t n, size_t r, const double* eigvals, const double* V, int T,
                   const double* g, const double* pi, double* w, double alpha, double sigma, double fl, int advance,
                   double* newton_out, double* base_out) {
  base_opt o;
  base_init(&o, c, n);
  double* work = (double*)malloc((3 * n + 3 * r + 3) * sizeof(double));
  double* nw = (double*)malloc(n * sizeof(double));
  double* bs = (double*)malloc(n * sizeof(double));
  int rc = ORC_OK;
  for (int t = 0; t < T && rc == ORC_OK; ++t) {
    rc = split_deltas(g + (size_t)t * n, pi, r, eigvals, V, &o, w, alpha, sigma, fl, nw, bs, work);
    if (rc) break;
    if (newton_out) memcpy(newton_out + (size_t)t * n, nw, n * sizeof(double));
    if (base_out) memcpy(base_out + (size_t)t * n, bs, n * sizeof(double));
    if (advance) {
      for (size_t i = 0; i < n; ++i) w[i] += 1.0 * bs[i];
      if (r > 0)
        for (size_t i = 0; i < n; ++i) w[i] += 1.0 * nw[i];
    }
  }
  free(work);
  free(nw);
  free(bs);
  base_free(&o);
  return rc;
}

/* admm_w_update :141-147 and admm_dual_update :149-154 */
int orc_admm_round(size_t n, double sigma, const double* w_a, const double* pi, double* w_out,
                   const double* w_a_after, double* pi_out) {
  if (sigma <= 0.0) FAIL(ORC_ARGUMENT, "AdmmState: sigma must be positive");
  for (size_t i = 0; i < n; ++i) w_out[i] = w_a[i] + pi[i] / sigma;
  if (w_a_after && pi_out)
    for (size_t i = 0; i < n; ++i) pi_out[i] = pi[i] + sigma * (w_a_after[i] - w_out[i]);
  return ORC_OK;
}

/* ------------------------------------------------------ trainer.cpp:51-298 */
typedef struct {
  int trainer; /* 0 sgd 1 fosi 2 dho2 */
  orc_base_cfg base;
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
} orc_train_cfg;

typedef struct {
  const orc_train_cfg* cfg;
  const size_t* sizes;
  int nl, act, loss;
  const double* X;
  const double* y;
  size_t N, D, ncls, n;
  uint64_t dataset_seed;
  int C;
  size_t rounds;
  /* outputs */
  size_t max_rows, n_rows, refreshes, safeguards;
  double *row_loss, *row_acc, *row_resid;
  int64_t* row_epoch;
  /* scratch */
  double *Xb, *yb, *gl, *g;
  uint64_t* perm;
  /* QuadraticOracle problem (grad = H w for every batch; value = w^T H w / 2; no accuracy) */
  const double* qspec;
  const double* qrot;
} trun;

static void gather_batch(trun* R, const uint64_t* idx, size_t cnt) {
  for (size_t j = 0; j < cnt; ++j) {
    memcpy(R->Xb + j * R->D, R->X + idx[j] * R->D, R->D * sizeof(double));
    R->yb[j] = R->y[idx[j]];
  }
}

/* mean_gradient :92-103 over C simulated workers, ascending-rank sum then * (1/C) */
static int mean_gradient(trun* R, const double* at, size_t round) {
  const size_t b = R->cfg->batch_size;
  uint64_t* idx = (uint64_t*)malloc(b * sizeof(uint64_t));
  int rc = ORC_OK;
  for (int r = 0; r < R->C && rc == ORC_OK; ++r) {
    size_t sb, se;
    orc_shard(R->N, R->C, r, &sb, &se);
    const size_t len = se - sb;
    for (size_t j = 0; j < b; ++j) idx[j] = R->perm[sb + (round * b + j) % len];
    if (R->qspec) {
      orc_quadratic_apply(R->n, R->qspec, R->qrot, at, r == 0 ? R->g : R->gl);
    } else {
      gather_batch(R, idx, b);
      rc = orc_mlp_grad(R->sizes, R->nl, R->act, R->loss, at, R->Xb, R->yb, b, R->ncls, r == 0 ? R->g : R->gl);
    }
    if (rc == ORC_OK && r > 0)
      for (size_t i = 0; i < R->n; ++i) R->g[i] += R->gl[i];
  }
  const double inv = 1.0 / (double)R->C;
  for (size_t i = 0; i < R->n; ++i) R->g[i] *= inv;
  free(idx);
  return rc;
}

/* refresh_ese :105-135 -> eigvals (r), V (n x r); returns r via *rr */
static int refresh_ese(trun* R, const double* at, double* eigvals, double* V, size_t* rr) {
  const orc_train_cfg* c = R->cfg;
  const size_t want = c->curvature_batch < R->N ? c->curvature_batch : R->N;
  uint64_t* idx = (uint64_t*)malloc(R->N * sizeof(uint64_t));
  orc_rng_shuffle_iota(orc_mix_seed(c->seed, 0xc0ffee + R->refreshes), R->N, idx);
  double* Xc = (double*)malloc(want * R->D * sizeof(double));
  double* yc = (double*)malloc(want * sizeof(double));
  for (size_t j = 0; j < want; ++j) {
    memcpy(Xc + j * R->D, R->X + idx[j] * R->D, R->D * sizeof(double));
    yc[j] = R->y[idx[j]];
  }
  size_t m;
  int rc = orc_lanczos_budget(c->k, c->l, R->n, &m);
  if (rc == ORC_OK) {
    orc_op op = {2, R->n, NULL, R->sizes, R->nl, R->act, R->loss, at, Xc, yc, want, R->ncls, 0, NULL};
    if (R->qspec) {
      op.kind = 1;
      op.mat = R->qspec;
      op.rot_seed = R->qrot ? 1 : 0;
      op.rot = R->qrot;
    }
    double* dg = (double*)malloc((m + 1) * sizeof(double));
    double* of = (double*)malloc((m + 1) * sizeof(double));
    size_t iters, sg;
    int bd;
    rc = orc_lanczos(&op, R->C, m, orc_mix_seed(c->seed, 0xbeef + R->refreshes), c->reorth_safeguard,
                     c->safeguard_ratio, c->breakdown_rtol, c->k, c->l, dg, of, &iters, &bd, &sg, NULL, eigvals, V);
    const size_t keff = c->k < iters ? c->k : iters;
    const size_t leff = c->l < iters - keff ? c->l : iters - keff;
    *rr = keff + leff;
    R->safeguards += sg;
    free(dg);
    free(of);
  }
  ++R->refreshes;
  free(idx);
  free(Xc);
  free(yc);
  return rc;
}

/* epoch_end :150-172 */
static int epoch_end(trun* R, const double* at, int64_t epoch, const double* resid_against) {
  double loss, acc = NAN;
  int rc = ORC_OK;
  if (R->qspec) { /* QuadraticOracle::value, oracle.cpp:274-276 */
    orc_quadratic_apply(R->n, R->qspec, R->qrot, at, R->gl);
    loss = 0.5 * dot(at, R->gl, R->n);
  } else {
    rc = orc_mlp_value(R->sizes, R->nl, R->act, R->loss, at, R->X, R->y, R->N, R->ncls, &loss);
    if (rc) return rc;
  }
  if (!isfinite(loss)) FAIL(ORC_NUMERIC, "non-finite loss");
  if (!R->qspec) {
    rc = orc_mlp_accuracy(R->sizes, R->nl, R->act, R->loss, at, R->X, R->y, R->N, R->ncls, &acc);
    if (rc) return rc;
  }
  if (R->n_rows < R->max_rows) {
    R->row_loss[R->n_rows] = loss;
    R->row_acc[R->n_rows] = R->ncls > 0 ? acc : NAN;
    R->row_epoch[R->n_rows] = epoch;
    double rn = NAN;
    if (resid_against) {
      double s = 0.0;
      for (size_t i = 0; i < R->n; ++i) {
        const double d = at[i] - resid_against[i];
        s += d * d;
      }
      rn = sqrt(s);
    }
    R->row_resid[R->n_rows] = rn;
  }
  ++R->n_rows;
  return ORC_OK;
}

static int train_common(const orc_train_cfg* c, const size_t* sizes, int nl, int act, int loss, const double* X,
                        const double* y, size_t N, size_t ncls, uint64_t dataset_seed, const double* w0, int workers,
                        double* w_final, size_t max_rows, size_t* n_rows, double* row_loss, double* row_acc,
                        double* row_resid, int64_t* row_epoch, size_t* refreshes, size_t* safeguards, size_t n,
                        const double* qspec, const double* qrot) {
  int rc = ORC_OK;
  if (c->batch_size == 0) FAIL(ORC_ARGUMENT, "train: batch_size must be >= 1");
  if (N < (size_t)workers) FAIL(ORC_ARGUMENT, "train: fewer samples than workers");
  trun R;
  memset(&R, 0, sizeof(R));
  R.cfg = c;
  R.sizes = sizes;
  R.nl = nl;
  R.act = act;
  R.loss = loss;
  R.X = X;
  R.y = y;
  R.N = N;
  R.D = qspec ? 1 : sizes[0];
  R.ncls = ncls;
  R.n = n;
  R.dataset_seed = dataset_seed;
  R.C = workers;
  R.qspec = qspec;
  R.qrot = qrot;
  size_t sb, se;
  orc_shard(N, workers, 0, &sb, &se);
  R.rounds = (se - sb + c->batch_size - 1) / c->batch_size;
  R.max_rows = max_rows;
  R.row_loss = row_loss;
  R.row_acc = row_acc;
  R.row_resid = row_resid;
  R.row_epoch = row_epoch;
  R.Xb = (double*)malloc(c->batch_size * R.D * sizeof(double));
  R.yb = (double*)malloc(c->batch_size * sizeof(double));
  R.gl = (double*)malloc(n * sizeof(double));
  R.g = (double*)malloc(n * sizeof(double));
  R.perm = (uint64_t*)malloc(N * sizeof(uint64_t));
  const size_t rmax = c->k + c->l;
  double* eigvals = (double*)calloc(rmax + 1, sizeof(double));
  double* V = (double*)calloc(n * (rmax + 1), sizeof(double));
  double* wa = (double*)malloc(n * sizeof(double));
  double* w = (double*)malloc(n * sizeof(double));
  double* pi = (double*)calloc(n, sizeof(double));
  double* nw = (double*)malloc(n * sizeof(double));
  double* bs = (double*)malloc(n * sizeof(double));
  double* work = (double*)malloc((3 * n + 3 * rmax + 3) * sizeof(double));
  memcpy(wa, w0, n * sizeof(double));
  base_opt opt;
  base_init(&opt, &c->base, n);
  size_t r = 0;
  const int curvature = c->k + c->l > 0;

  if (c->trainer == 0) { /* run_first_order :174-185 */
    for (size_t e = 0; e < c->epochs && rc == ORC_OK; ++e) {
      orc_epoch_permutation(N, dataset_seed, e, R.perm);
      for (size_t rd = 0; rd < R.rounds && rc == ORC_OK; ++rd) {
        if ((rc = mean_gradient(&R, wa, rd))) break;
        if ((rc = base_step(&opt, R.g, wa, bs))) break;
        for (size_t i = 0; i < n; ++i) wa[i] += 1.0 * bs[i];
      }
      if (rc == ORC_OK) rc = epoch_end(&R, wa, (int64_t)e, NULL);
    }
  } else if (c->trainer == 1) { /* run_fosi :187-209 */
    const size_t interval = c->refresh_interval > 0 ? c->refresh_interval : R.rounds;
    size_t iter = 0;
    for (size_t e = 0; e < c->epochs && rc == ORC_OK; ++e) {
      orc_epoch_permutation(N, dataset_seed, e, R.perm);
      for (size_t rd = 0; rd < R.rounds && rc == ORC_OK; ++rd, ++iter) {
        if (curvature && iter % interval == 0)
          if ((rc = refresh_ese(&R, wa, eigvals, V, &r))) break;
        if ((rc = mean_gradient(&R, wa, rd))) break;
        if ((rc = split_deltas(R.g, NULL, r, eigvals, V, &opt, wa, c->alpha, 0.0, c->eigval_floor, nw, bs, work)))
          break;
        for (size_t i = 0; i < n; ++i) wa[i] += 1.0 * bs[i];
        if (r > 0)
          for (size_t i = 0; i < n; ++i) wa[i] += 1.0 * nw[i];
      }
      if (rc == ORC_OK) rc = epoch_end(&R, wa, (int64_t)e, NULL);
    }
  } else { /* run_dho2 :211-249 */
    const int red = c->sigma_zero_reduction;
    if (!red && c->sigma <= 0.0) {
      rc = ORC_ARGUMENT;
      g_err = "dho2: sigma must be positive";
    }
    const double sigma_state = red ? 1.0 : c->sigma;
    const double sigma_eff = red ? 0.0 : c->sigma;
    memcpy(w, wa, n * sizeof(double));
    for (size_t ko = 0; ko < c->outer_rounds && rc == ORC_OK; ++ko) {
      r = 0;
      if (curvature)
        if ((rc = refresh_ese(&R, wa, eigvals, V, &r))) break;
      if (red) memcpy(w, wa, n * sizeof(double));
      else
        for (size_t i = 0; i < n; ++i) w[i] = wa[i] + pi[i] / sigma_state;
      memcpy(wa, w, n * sizeof(double));
      for (size_t li = 0; li < c->inner_epochs && rc == ORC_OK; ++li) {
        const int64_t epoch = (int64_t)(ko * c->inner_epochs + li);
        orc_epoch_permutation(N, dataset_seed, (uint64_t)epoch, R.perm);
        for (size_t rd = 0; rd < R.rounds && rc == ORC_OK; ++rd) {
          if ((rc = mean_gradient(&R, wa, rd))) break;
          if ((rc = split_deltas(R.g, red ? NULL : pi, r, eigvals, V, &opt, wa, c->alpha, sigma_eff,
                                 c->eigval_floor, nw, bs, work)))
            break;
          for (size_t i = 0; i < n; ++i) wa[i] += 1.0 * bs[i];
          if (r > 0)
            for (size_t i = 0; i < n; ++i) wa[i] += 1.0 * nw[i];
        }
        if (rc == ORC_OK) rc = epoch_end(&R, wa, epoch, w);
      }
      if (rc == ORC_OK && !red)
        for (size_t i = 0; i < n; ++i) pi[i] += sigma_state * (wa[i] - w[i]);
    }
  }
  memcpy(w_final, wa, n * sizeof(double));
  *n_rows = R.n_rows;
  *refreshes = R.refreshes;
  *safeguards = R.safeguards;
  base_free(&opt);
  free(R.Xb);
  free(R.yb);
  free(R.gl);
  free(R.g);
  free(R.perm);
  free(eigvals);
  free(V);
  free(wa);
  free(w);
  free(pi);
  free(nw);
  free(bs);
  free(work);
  return rc;
}

int orc_train_mlp(const orc_train_cfg* c, const size_t* sizes, int nl, int act, int loss, const double* X,
                  const double* y, size_t N, size_t ncls, uint64_t dataset_seed, const double* w0, int workers,
                  double* w_final, size_t max_rows, size_t* n_rows, double* row_loss, double* row_acc,
                  double* row_resid, int64_t* row_epoch, size_t* refreshes, size_t* safeguards) {
  size_t n;
  int rc = orc_mlp_dim(sizes, nl, &n);
  if (rc) return rc;
  return train_common(c, sizes, nl, act, loss, X, y, N, ncls, dataset_seed, w0, workers, w_final, max_rows, n_rows,
                      row_loss, row_acc, row_resid, row_epoch, refreshes, safeguards, n, NULL, NULL);
}

/* train() on Problem{QuadraticOracle(spec, rotation_seed), Dataset::dummy(N), w0}
 * (tests/test_trainer.cpp:14-21; Dataset::dummy is oracle.cpp:64-68: D = 1, no classes, seed 0). */
int orc_train_quadratic(const orc_train_cfg* c, const double* spec, size_t n, uint64_t rotation_seed, size_t N,
                        const double* w0, int workers, double* w_final, size_t max_rows, size_t* n_rows,
                        double* row_loss, double* row_acc, double* row_resid, int64_t* row_epoch,
                        size_t* refreshes, size_t* safeguards) {
  int rc = orc_quadratic_check(spec, n);
  if (rc) return rc;
  if (N == 0) FAIL(ORC_ARGUMENT, "Dataset::dummy: need at least one sample");
  double* Q = NULL;
  if (rotation_seed != 0) {
    Q = (double*)malloc(n * n * sizeof(double));
    rc = orc_quadratic_rotation(n, rotation_seed, Q);
  }
  double* X = (double*)calloc(N, sizeof(double));
  double* y = (double*)calloc(N, sizeof(double));
  if (rc == ORC_OK)
    rc = train_common(c, NULL, 0, 0, 0, X, y, N, 0, 0, w0, workers, w_final, max_rows, n_rows, row_loss, row_acc,
                      row_resid, row_epoch, refreshes, safeguards, n, spec, Q);
  free(Q);
  free(X);
  free(y);
  return rc;
}

/* QuadraticOracle(spec, rotation_seed): apply_h(x) and value(x) = x^T H x / 2 (oracle.cpp:274-276);
 * same signature as the reference shim's ref_quadratic_apply. */
int orc_quadratic_apply_seeded(const double* spec, size_t n, uint64_t rotation_seed, const double* x, double* out,
                               double* value) {
  int rc = orc_quadratic_check(spec, n);
  if (rc) return rc;
  double* Q = NULL;
  if (rotation_seed != 0) {
    Q = (double*)malloc(n * n * sizeof(double));
    rc = orc_quadratic_rotation(n, rotation_seed, Q);
  }
  if (rc == ORC_OK) {
    orc_quadratic_apply(n, spec, Q, x, out);
    if (value) *value = 0.5 * dot(x, out, n);
  }
  free(Q);
  return rc;
}
