// Small-model MLP passes as ONE persistent launch each (the C1/C2 models, 784-256-10 at batch 128-512).
//
// At these sizes an HVP is ~0.3 GFLOP: the tcgen05 path's per-GEMM fixed costs (TMEM allocation, TMA
// descriptor fetch, pipeline fill, split-K combine; ~7-15 us per GEMM, profiles/r02_tc1_timeline.txt) and
// the ~20 launches of one pass (operand splits, packing, bias sums) are the whole cost. Here a cooperative
// grid (one CTA per SM) walks the pass's phases, separated by grid barriers:
//   forward    layer t = 0..L-1   Z / RZ tiles + the layer epilogue          (oracle.cpp:548-563)
//   output     one thread per sample: delta / R-delta, loss, correctness      (oracle.cpp:476-495, 572-599)
//   backward   layer t = L-1..0   weight block (+ bias column) and, t > 0, the delta / R-delta tiles of
//                                 level t — both read level t+1 only, so they share one phase
//                                 (oracle.cpp:497-504, 606-637)
// Every contraction is a 32 x 32 output tile over 32-deep K chunks, all of a unit's chunks in flight at once
// (cp.async ring of kStages chunks: at these sizes the loads' latency, not bandwidth, is the cost), fp32
// FMA with the chunk partials added into a running sum (two-level summation); tiles with few units per SM are split
// along K and the split partials are added in split order by the last unit to finish (ticket), so results
// are deterministic. The arithmetic is the reference's (fp32 products of fp32 operands, no operand
// splitting). Semantics, inputs and outputs are those of the GEMM path in mlp.cu (same cached a / d / u
// buffers, same flat gradient / HVP layout and optional fused reduce-scatter routing).
#include "internal.h"
#include "coop.cuh"
#include "mlp_dev.cuh"

namespace dho2g {
namespace {

constexpr int kT = 32;      // tile edge (M, N) and K chunk
constexpr int kThr = 256;   // 16 x 16 threads, 2 x 2 outputs each
constexpr int kMaxL = 8;

enum SmallMode { SM_GRAD = 0, SM_PREP = 1, SM_HVP = 2, SM_EVAL = 3 };
enum SmallEpi { SE_FWD0 = 0, SE_FWDR = 1, SE_BWD0 = 2, SE_BWDR = 3, SE_WB = 4 };

struct SmallNet {  // by value in the kernel parameters
  int L, relu, mse;
  int s[kMaxL + 1];
  long long w_off[kMaxL], b_off[kMaxL];
  float* a32[kMaxL + 1];
  float* ra32[kMaxL + 1];
  float* d32[kMaxL + 1];
  float* rd32[kMaxL + 1];
  float* u32[kMaxL + 1];
};

struct SmallCall {
  int mode, B, ncls, ldx, cache_u;
  double scale;
  const float* w;
  const float* v;
  const float* vscale;
  float* out;
  const float* X;
  const int64_t* idx;
  const float* y;
  float* lab;
  double* loss;
  int* correct;
  float* part;
  unsigned* tickets;
  unsigned long long* bar;
  float* const* route;
  long long route_base;
  int route_rank;
  unsigned long long* trace;  // debug (env DHO2G_SMALL_TRACE): per CTA %globaltimer at each phase edge
  int trace_t;                // the forward layer whose units are traced
};

__device__ __forceinline__ void stamp(const SmallCall& c, int i) {
  if (c.trace && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    c.trace[blockIdx.x * 32 + i] = t;
  }
}

// One K segment of an operand: element (r, k) at p[r * sr + k * sk] (times sc, applied to the chunk partial);
// gather 1: r -> idx[r], gather 2: k -> idx[k] (the input batch rows X[idx[b]]).
struct Seg {
  const float* p;
  int sr, sk;  // (products are formed in 64 bits)
  float sc;
  int gather;
};
// Operand of R rows (the M or N side); row `ones` reads 1 in the first segment and 0 in the second (the bias
// column of the weight blocks).
struct Opnd {
  Seg s0, s1;
  int R, ones;
};
__device__ __forceinline__ Seg pick(const Opnd& o, int seg) {  // by value: stays in registers
  Seg s;
  s.p = seg ? o.s1.p : o.s0.p;
  s.sr = seg ? o.s1.sr : o.s0.sr;
  s.sk = seg ? o.s1.sk : o.s0.sk;
  s.sc = seg ? o.s1.sc : o.s0.sc;
  s.gather = seg ? o.s1.gather : o.s0.gather;
  return s;
}
// acc[M x N] = sum_k A(m, k) B(n, k) over two K segments of lengths K0, K1 (K1 = 0: one). The second
// segment starts at the logical offset Kp0 = round_up(K0, kT), so every kT-deep chunk lies in one segment;
// K is the logical length.
struct SGemm {
  int M, N, K, K0, K1, Kp0, S, Kc, tn, units;
  Opnd A, B;
  int epi, t;
};
__device__ __forceinline__ void set_k(SGemm& g, int K0, int K1) {
  g.K0 = K0;
  g.K1 = K1;
  g.Kp0 = K1 ? (int)round_up(K0, kT) : K0;
  g.K = g.Kp0 + K1;
}

__device__ __forceinline__ float act_f(bool relu, float z) { return relu ? fmaxf(z, 0.f) : tanhf(z); }
__device__ __forceinline__ float act_p(bool relu, float a) { return relu ? (a > 0.f ? 1.f : 0.f) : 1.f - a * a; }

// Stage slots. An operand whose rows are contiguous in memory (sr == 1: "K-major" here) is staged [k][row]
// (row stride kLdK); a K-contiguous one (sk == 1) [row][k] with the 16-byte k-blocks XOR-swizzled by row so
// that both the 16-byte cp.async writes and the compute's float4 reads are conflict-free.
constexpr int kLdK = kT + 4;
constexpr int kStages = 8;   // two rounds of kGroups chunks in flight
constexpr int kGroups = 4;   // K groups per CTA: 64 threads each, 4 x 4 outputs per thread, chunk gr of a round
struct Stage {
  float A[kT * kLdK];
  float B[kT * kLdK];
};
constexpr size_t kSmem = sizeof(Stage) * kStages;
__device__ __forceinline__ int rmaj(int r, int k) { return r * kT + ((((k >> 2) ^ ((r >> 2) & 7))) << 2) + (k & 3); }

__device__ __forceinline__ void cp16(float* dst, const float* src) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(src) : "memory");
}
__device__ __forceinline__ void cp4(float* dst, const float* src) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(d), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

__device__ __forceinline__ bool seg_vec(const Seg& s) {
  const bool fast = s.sk == 1;
  return ((reinterpret_cast<uintptr_t>(s.p) & 15u) == 0) && (fast ? (s.sr & 3) == 0 : (s.sr == 1 && (s.sk & 3) == 0));
}

// Issues this thread's float4 slot of an operand's chunk [kc, kc + kT) (logical k; split end k1): K-contiguous:
// row f / 8, k 4 (f % 8) .. + 3; row-contiguous: k f / 8, rows 4 (f % 8) .. + 3. One 16-byte cp.async (L2) when
// the slot is whole and aligned, else 4-byte ones / zeros / the bias row's ones. (Data written earlier in this
// launch: the grid barrier's acquire fence invalidated L1.)
__device__ __noinline__ void issue_slot(const SGemm& g, const Opnd& o, const int64_t* idx, int r0, int kc, int k1,
                                        float* slot) {
  const int seg = (g.K1 && kc >= g.Kp0) ? 1 : 0;
  const Seg s = pick(o, seg);
  const int kb = kc - (seg ? g.Kp0 : 0);
  const int lim = min(min(kT, k1 - kc), (seg ? g.K1 : g.K0) - kb);
  const float onev = seg ? 0.f : 1.f;
  const int f = threadIdx.x;
  if (s.sk == 1) {
    const int i = f >> 3, kq = (f & 7) * 4, r = r0 + i;
    float* dst = slot + rmaj(i, kq);
    if (r >= o.R || kq >= lim || r == o.ones) {
      const float fill = r == o.ones && r < o.R ? onev : 0.f;
#pragma unroll
      for (int e = 0; e < 4; ++e) dst[e] = kq + e < lim ? fill : 0.f;
      return;
    }
    const long long rr = (s.gather == 1 && idx) ? idx[r] : r;
    const float* rp = s.p + rr * (long long)s.sr + kb + kq;
    if (kq + 4 <= lim && seg_vec(s)) {
      cp16(dst, rp);
    } else {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        if (kq + e < lim) cp4(dst + e, rp + e);
        else dst[e] = 0.f;
      }
    }
    return;
  }
  const int kk = f >> 3, rq = r0 + (f & 7) * 4;
  float* dst = slot + kk * kLdK + (f & 7) * 4;
  if (kk >= lim || rq >= o.R) {
    *reinterpret_cast<float4*>(dst) = make_float4(0.f, 0.f, 0.f, 0.f);
    return;
  }
  const long long k = kb + kk;
  const long long kx = (s.gather == 2 && idx) ? idx[k] : k;
  if (rq + 3 < o.R && (o.ones < rq || o.ones > rq + 3) && s.gather != 1 && seg_vec(s)) {
    cp16(dst, s.p + kx * (long long)s.sk + rq);
    return;
  }
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const int r = rq + e;
    if (r >= o.R) {
      dst[e] = 0.f;
    } else if (r == o.ones) {
      dst[e] = onev;
    } else {
      const long long rr = (s.gather == 1 && idx) ? idx[r] : r;
      cp4(dst + e, s.p + rr * (long long)s.sr + kx * (long long)s.sk);
    }
  }
}

// The common case of issue_slot with the per-segment address arithmetic hoisted: this thread's slot base
// pointer (row-gathered input rows resolved), its k stride, and whether the slot is whole-row and 16-byte
// aligned; chunks that are not (segment tails, the bias row, unaligned operands) take issue_slot.
struct OpIss {
  const float* base;
  long long sk;
  int seg, fast, vec, gidx;
};
__device__ __forceinline__ void iss_setup(OpIss& st, const Opnd& o, const int64_t* idx, int r0, int seg) {
  const Seg s = pick(o, seg);
  const int f = threadIdx.x;
  st.seg = seg;
  st.fast = s.sk == 1;
  if (st.fast) {
    const int r = r0 + (f >> 3);
    const bool on = r < o.R && r != o.ones;
    const long long rr = (s.gather == 1 && idx && on) ? idx[r] : r;
    st.base = s.p + rr * (long long)s.sr + (f & 7) * 4;
    st.sk = 1;
    st.gidx = 0;
    st.vec = on && seg_vec(s);
  } else {
    const int rq = r0 + (f & 7) * 4;
    st.base = s.p + rq;
    st.sk = s.sk;
    st.gidx = s.gather == 2 && idx;
    st.vec = rq + 3 < o.R && (o.ones < rq || o.ones > rq + 3) && s.gather != 1 && seg_vec(s);
  }
}
__device__ __forceinline__ void issue_fast(OpIss& st, const SGemm& g, const Opnd& o, const int64_t* idx, int r0,
                                           int kc, int k1, float* slot) {
  const int seg = (g.K1 && kc >= g.Kp0) ? 1 : 0;
  if (seg != st.seg) iss_setup(st, o, idx, r0, seg);
  const int kb = kc - (seg ? g.Kp0 : 0);
  const int lim = min(min(kT, k1 - kc), (seg ? g.K1 : g.K0) - kb);
  const int f = threadIdx.x;
  if (st.fast) {
    const int kq = (f & 7) * 4;
    if (st.vec && kq + 4 <= lim) {
      cp16(slot + rmaj(f >> 3, kq), st.base + kb);
      return;
    }
  } else {
    const int kk = f >> 3;
    if (st.vec && kk < lim) {
      const long long k = kb + kk;
      cp16(slot + kk * kLdK + (f & 7) * 4, st.base + (st.gidx ? idx[k] : k) * st.sk);
      return;
    }
  }
  issue_slot(g, o, idx, r0, kc, k1, slot);
}

// p[i][j] += sum_k A(ry + i, k) B(cx + j, k) over one staged chunk, k ascending (AK / BK: [k][row] staging)
template <bool AK, bool BK>
__device__ __forceinline__ void chunk_mma(const float* sa, const float* sb, int ry, int cx, float (&p)[4][4]) {
#pragma unroll 2
  for (int k = 0; k < kT; k += 4) {
    float a[4][4], b[4][4];  // [row][k]
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float4 ta = AK ? *reinterpret_cast<const float4*>(&sa[(k + e) * kLdK + ry])
                           : *reinterpret_cast<const float4*>(&sa[rmaj(ry + e, k)]);
      const float4 tb = BK ? *reinterpret_cast<const float4*>(&sb[(k + e) * kLdK + cx])
                           : *reinterpret_cast<const float4*>(&sb[rmaj(cx + e, k)]);
      if (AK) { a[0][e] = ta.x; a[1][e] = ta.y; a[2][e] = ta.z; a[3][e] = ta.w; }
      else { a[e][0] = ta.x; a[e][1] = ta.y; a[e][2] = ta.z; a[e][3] = ta.w; }
      if (BK) { b[0][e] = tb.x; b[1][e] = tb.y; b[2][e] = tb.z; b[3][e] = tb.w; }
      else { b[e][0] = tb.x; b[e][1] = tb.y; b[e][2] = tb.z; b[e][3] = tb.w; }
    }
#pragma unroll
    for (int e = 0; e < 4; ++e)
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) p[i][j] = fmaf(a[i][e], b[j][e], p[i][j]);
  }
}

// The element epilogues (gemm.cu epi_elem: the same math per mode), split into the loads of an element's
// inputs (issued for all of a thread's elements before any math) and the math + store.
struct EIn {
  float p0, p1, p2;
};
__device__ __forceinline__ EIn epi_in(const SGemm& g, const SmallNet& net, const SmallCall& c, const float* v, int r,
                                      int col) {
  EIn in{0.f, 0.f, 0.f};
  if (r >= g.M || col >= g.N) return in;
  const int t = g.t;
  const size_t e = (size_t)r * g.N + col;
  switch (g.epi) {
    case SE_FWD0: in.p0 = __ldg(c.w + net.b_off[t] + col); break;
    case SE_FWDR:
      in.p0 = __ldcg(v + net.b_off[t] + col);
      if (t + 1 != net.L) in.p1 = __ldcg(net.a32[t + 1] + e);
      break;
    case SE_BWD0: in.p0 = __ldcg(net.a32[t] + e); break;
    case SE_BWDR:
      in.p0 = __ldcg(net.a32[t] + e);
      if (!net.relu) in.p1 = __ldcg(net.ra32[t] + e);
      in.p2 = __ldcg(net.u32[t] + e);
      break;
    default: break;
  }
  return in;
}
__device__ void epi_store(const SGemm& g, const SmallNet& net, const SmallCall& c, float vsc, int r, int col, float x,
                          EIn in) {
  if (r >= g.M || col >= g.N) return;
  const int t = g.t;
  const bool last = t + 1 == net.L;
  const size_t e = (size_t)r * g.N + col;
  switch (g.epi) {
    case SE_FWD0: {  // z = acc + b ; a = act(z) (output layer: z)
      const float z = x + in.p0;
      net.a32[t + 1][e] = last ? z : act_f(net.relu, z);
      break;
    }
    case SE_FWDR: {  // rz = acc + vscale v_b ; ra = act'(a) rz (output layer: rz)
      const float rz = x + vsc * in.p0;
      net.ra32[t + 1][e] = last ? rz : act_p(net.relu, in.p1) * rz;
      break;
    }
    case SE_BWD0:  // level t: d = u act'(a), u cached for the R-delta
      net.d32[t][e] = x * act_p(net.relu, in.p0);
      if (c.cache_u) net.u32[t][e] = x;
      break;
    case SE_BWDR: {  // level t: rd = ru act'(a) + u (-2 a ra) (tanh)
      const float a = in.p0;
      const float ap = act_p(net.relu, a);
      const float rap = (!net.relu && ap != 0.f) ? -2.f * a * in.p1 : 0.f;
      net.rd32[t][e] = x * ap + in.p2 * rap;
      break;
    }
    default: {  // weight block row o = r, column i = col (col == in: the bias)
      const int in_ = net.s[t];
      if (col == in_) {
        c.out[net.b_off[t] + r] = x;
      } else {
        const long long flat = net.w_off[t] + (long long)r * in_ + col;
        if (c.route) {
          const long long q = flat / c.route_base;
          c.route[q][c.route_rank * c.route_base + (flat - q * c.route_base)] = x;
        } else {
          c.out[flat] = x;
        }
      }
    }
  }
}

// One work unit (tile, split) of g: the tile's partial over its K range. Rounds of kGroups chunks, two rounds in
// flight (cp.async); K group gr (64 threads, 4 x 4 outputs each) multiplies chunk gr of a round; the group
// partials are added in group order into the tile T (shared memory). Split partials are combined by the last
// unit of the tile in split order. Then the epilogue, element e = tid + kThr q of T.
__device__ bool run_unit(const SGemm& g, const SmallNet& net, const SmallCall& c, const float* v, float vsc, int u,
                         float* part, unsigned* tickets, Stage* ring, unsigned& s_last) {
  const int tile = u / g.S, s = u - tile * g.S;
  const int m0 = (tile / g.tn) * kT, n0 = (tile % g.tn) * kT;
  const int k0 = s * g.Kc, k1 = min(g.K, k0 + g.Kc);
  const int nc = (int)cdiv(max(k1 - k0, 0), kT);
  const int tid = threadIdx.x, gr = tid >> 6, gt = tid & 63, ry = (gt >> 3) * 4, cx = (gt & 7) * 4;
  const bool tr = c.trace && g.epi == SE_FWDR && g.t == c.trace_t;  // debug timeline of one forward phase
  if (tr) stamp(c, 16);
  float acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;
  // the epilogue's inputs do not depend on this unit's sums: loaded now, in flight during the GEMM
  EIn in[kT * kT / kThr];
#pragma unroll
  for (int q = 0; q < kT * kT / kThr; ++q) {
    const int e = tid + kThr * q;
    in[q] = epi_in(g, net, c, v, m0 + (e >> 5), n0 + (e & 31));
  }
  const int rounds = (int)cdiv(nc, kGroups);
  OpIss ia, ib;
  ia.seg = ib.seg = -1;
  auto issue_round = [&](int r) {
#pragma unroll 1
    for (int q = 0; q < kGroups; ++q) {
      const int ci = r * kGroups + q;
      if (ci >= nc) break;
      Stage& st = ring[ci % kStages];
      issue_fast(ia, g, g.A, c.idx, m0, k0 + ci * kT, k1, st.A);
      issue_fast(ib, g, g.B, c.idx, n0, k0 + ci * kT, k1, st.B);
    }
  };
  issue_round(0);
  cp_commit();
  issue_round(1);
  cp_commit();
  if (tr) stamp(c, 17);
#pragma unroll 1
  for (int r = 0; r < rounds; ++r) {
    cp_wait<1>();
    __syncthreads();
    const int ci = r * kGroups + gr;
    if (ci < nc) {
      const Stage& st = ring[ci % kStages];
      const int kc = k0 + ci * kT;
      const int seg = (g.K1 && kc >= g.Kp0) ? 1 : 0;
      const bool ak = (seg ? g.A.s1.sk : g.A.s0.sk) != 1, bk = (seg ? g.B.s1.sk : g.B.s0.sk) != 1;
      float p[4][4];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) p[i][j] = 0.f;
      if (ak) {
        if (bk) chunk_mma<true, true>(st.A, st.B, ry, cx, p);
        else chunk_mma<true, false>(st.A, st.B, ry, cx, p);
      } else {
        if (bk) chunk_mma<false, true>(st.A, st.B, ry, cx, p);
        else chunk_mma<false, false>(st.A, st.B, ry, cx, p);
      }
      const float f = (seg ? g.A.s1.sc : g.A.s0.sc) * (seg ? g.B.s1.sc : g.B.s0.sc);  // the direction's scale
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(p[i][j], f, acc[i][j]);
    }
    __syncthreads();  // this round's slots are refilled by round r + 2
    issue_round(r + 2);
    cp_commit();
    if (tr && r < 2) stamp(c, 18 + r);
  }
  cp_wait<0>();
  // group partials -> the tile T (group order)
  float* red = reinterpret_cast<float*>(ring);
  float* T = red + (kGroups - 1) * kT * kT;
  if (gr > 0) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
      *reinterpret_cast<float4*>(&red[(gr - 1) * kT * kT + (ry + i) * kT + cx]) =
          make_float4(acc[i][0], acc[i][1], acc[i][2], acc[i][3]);
  }
  __syncthreads();
  if (gr == 0) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      float4 t = make_float4(acc[i][0], acc[i][1], acc[i][2], acc[i][3]);
#pragma unroll
      for (int q = 0; q < kGroups - 1; ++q) {
        const float4 y = *reinterpret_cast<const float4*>(&red[q * kT * kT + (ry + i) * kT + cx]);
        t.x += y.x; t.y += y.y; t.z += y.z; t.w += y.w;
      }
      *reinterpret_cast<float4*>(&T[(ry + i) * kT + cx]) = t;
    }
  }
  __syncthreads();
  if (g.S > 1) {
    float4* mine = reinterpret_cast<float4*>(part + (size_t)u * (kT * kT));
    __stcg(mine + tid, reinterpret_cast<const float4*>(T)[tid]);
    __threadfence();
    __syncthreads();
    if (tid == 0) s_last = atomicAdd(&tickets[tile], 1u) == (unsigned)(g.S - 1);
    __syncthreads();
    if (!s_last) return false;
    __threadfence();
    const float4* base = reinterpret_cast<const float4*>(part + (size_t)tile * g.S * (kT * kT));
    // the S partials' loads in flight together (groups of 8), added in split order
    float4 x = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int q0 = 0; q0 < g.S; q0 += 8) {
      float4 y[8];
#pragma unroll
      for (int q = 0; q < 8; ++q)
        if (q0 + q < g.S) y[q] = __ldcg(base + (size_t)(q0 + q) * (kT * kT / 4) + tid);
#pragma unroll
      for (int q = 0; q < 8; ++q)
        if (q0 + q < g.S) {
          if (q0 + q == 0) x = y[q];
          else { x.x += y[q].x; x.y += y[q].y; x.z += y[q].z; x.w += y[q].w; }
        }
    }
    reinterpret_cast<float4*>(T)[tid] = x;
    if (tid == 0) tickets[tile] = 0u;  // reused by the next phase (after a grid barrier)
    __syncthreads();
  }
  if (tr) stamp(c, 28);
#pragma unroll
  for (int q = 0; q < kT * kT / kThr; ++q) {
    const int e = tid + kThr * q;
    epi_store(g, net, c, vsc, m0 + (e >> 5), n0 + (e & 31), T[e], in[q]);
  }
  if (tr) stamp(c, 29);
  __syncthreads();  // T aliases the stage ring
  return true;  // this unit completed the tile
}

__device__ __forceinline__ Seg seg(const float* p, int sr, int sk, float sc = 1.f, int gather = 0) {
  Seg s;
  s.p = p; s.sr = sr; s.sk = sk; s.sc = sc; s.gather = gather;
  return s;
}

// K splits for a GEMM given the CTAs it may occupy: >= 64-deep splits, about one unit per CTA
__device__ __forceinline__ void plan(SGemm& g, int ctas) {
  const int tiles = (int)(cdiv(g.M, kT) * cdiv(g.N, kT));
  g.tn = (int)cdiv(g.N, kT);
  int S = max(1, min((int)cdiv(g.K, 64), ctas / max(tiles, 1)));
  g.Kc = (int)round_up(cdiv(g.K, S), kT);
  g.S = (int)cdiv(g.K, g.Kc);
  if (g.K == 0) { g.S = 1; g.Kc = kT; }
  g.units = tiles * g.S;
}

// forward layer t (R: the R-pass)
__device__ __forceinline__ void fwd_gemm(SGemm& g, const SmallNet& net, const SmallCall& c, const float* v, int t,
                                         bool R, float vsc) {
  const int in = net.s[t], out = net.s[t + 1];
  g.M = c.B; g.N = out; g.t = t;
  const float* W = c.w + net.w_off[t];
  // A: level-t activations by sample (the input batch at t = 0)
  g.A.s0 = t == 0 ? seg(c.X, c.ldx, 1, 1.f, 1) : seg(net.a32[t], in, 1);
  g.A.R = c.B; g.A.ones = -1;
  g.B.R = out; g.B.ones = -1;
  if (!R) {  // Z = A W^T
    set_k(g, in, 0);
    g.B.s0 = seg(W, in, 1);
    g.epi = SE_FWD0;
  } else {   // RZ = [A | RA] [vscale V | W]^T (RA = 0 at the input layer)
    set_k(g, in, t == 0 ? 0 : in);
    g.A.s1 = seg(net.ra32[t], in, 1);
    g.B.s0 = seg(v + net.w_off[t], in, 1, vsc);
    g.B.s1 = seg(W, in, 1);
    g.epi = SE_FWDR;
  }
}

// weight block of layer t (M = out rows o, N = in + 1 columns, K = batch)
__device__ __forceinline__ void wb_gemm(SGemm& g, const SmallNet& net, const SmallCall& c, int t, bool R) {
  const int in = net.s[t], out = net.s[t + 1];
  g.M = out; g.N = in + 1; g.t = t; g.epi = SE_WB;
  g.A.R = out; g.A.ones = -1; g.B.R = in + 1; g.B.ones = in;
  // B(i, b) = level-t activation of sample b (input rows gathered at t = 0)
  g.B.s0 = t == 0 ? seg(c.X, 1, c.ldx, 1.f, 2) : seg(net.a32[t], 1, in);
  if (!R || t == 0) {  // gW = D^T A ; hvW (t = 0) = RD^T X
    set_k(g, c.B, 0);
    g.A.s0 = seg(R ? net.rd32[t + 1] : net.d32[t + 1], 1, out);
  } else {             // hvW = RD^T A + D^T RA
    set_k(g, c.B, c.B);
    g.A.s0 = seg(net.rd32[t + 1], 1, out);
    g.A.s1 = seg(net.d32[t + 1], 1, out);
    g.B.s1 = seg(net.ra32[t], 1, in);
  }
}

// delta of level t >= 1 (M = batch, N = in, K = out): U = D W ; RU = D (vscale V) + RD W
__device__ __forceinline__ void bwd_gemm(SGemm& g, const SmallNet& net, const SmallCall& c, const float* v, int t,
                                         bool R, float vsc) {
  const int in = net.s[t], out = net.s[t + 1];
  g.M = c.B; g.N = in; g.t = t;
  g.A.R = c.B; g.A.ones = -1; g.B.R = in; g.B.ones = -1;
  const float* W = c.w + net.w_off[t];
  g.A.s0 = seg(net.d32[t + 1], out, 1);
  if (!R) {
    set_k(g, out, 0);
    g.B.s0 = seg(W, 1, in);
    g.epi = SE_BWD0;
  } else {
    set_k(g, out, out);
    g.A.s1 = seg(net.rd32[t + 1], out, 1);
    g.B.s0 = seg(v + net.w_off[t], 1, in, vsc);
    g.B.s1 = seg(W, 1, in);
    g.epi = SE_BWDR;
  }
}

// output_delta_row (mlp_dev.cuh) for kOR samples b0 + q (q < kOR, b < b1) at once, lane j owning output j:
// the same per-element formulas, the row sums (softmax denominator, R-dot, MSE loss) as fixed-order warp
// reductions, argmax = lowest index of the max; the samples' fp64 chains are independent (ILP).
constexpr int kOR = 4;
__device__ void output_delta_warp(int b0, int b1, int O, int mse, int ncls, int do0, int do1, double scale,
                                  const float* z, const float* rz, const float* lab, float* __restrict__ d,
                                  float* __restrict__ rd, double* __restrict__ loss, int* __restrict__ correct) {
  const int j = threadIdx.x & 31;
  const bool on = j < O;
  float o[kOR], ro[kOR], y[kOR];
  bool rv[kOR];
#pragma unroll
  for (int q = 0; q < kOR; ++q) {
    const int b = b0 + q;
    rv[q] = b < b1;
    const size_t e = (size_t)b * O + j;
    o[q] = (rv[q] && on) ? __ldcg(z + e) : -INFINITY;
    ro[q] = (rv[q] && on && do1) ? __ldcg(rz + e) : 0.f;
    y[q] = rv[q] ? __ldcg(lab + b) : 0.f;
  }
  float bv[kOR];
  int bi[kOR];
#pragma unroll
  for (int q = 0; q < kOR; ++q) {
    bv[q] = o[q];
    bi[q] = on ? j : 0x7fffffff;
  }
#pragma unroll
  for (int s = 16; s > 0; s >>= 1)
#pragma unroll
    for (int q = 0; q < kOR; ++q) {
      const float ov = __shfl_xor_sync(0xffffffffu, bv[q], s);
      const int oi = __shfl_xor_sync(0xffffffffu, bi[q], s);
      if (ov > bv[q] || (ov == bv[q] && oi < bi[q])) {
        bv[q] = ov;
        bi[q] = oi;
      }
    }
  if (!mse) {
    double ex[kOR], den[kOR];
#pragma unroll
    for (int q = 0; q < kOR; ++q) ex[q] = (rv[q] && on) ? exp((double)o[q] - (double)bv[q]) : 0.0;
#pragma unroll
    for (int q = 0; q < kOR; ++q) den[q] = ex[q];
#pragma unroll
    for (int s = 16; s > 0; s >>= 1)
#pragma unroll
      for (int q = 0; q < kOR; ++q) den[q] += __shfl_xor_sync(0xffffffffu, den[q], s);
    double soft[kOR], sd[kOR];
#pragma unroll
    for (int q = 0; q < kOR; ++q) {
      soft[q] = ex[q] / den[q];
      sd[q] = (on && do1) ? soft[q] * ro[q] : 0.0;
    }
    if (do1) {
#pragma unroll
      for (int s = 16; s > 0; s >>= 1)
#pragma unroll
        for (int q = 0; q < kOR; ++q) sd[q] += __shfl_xor_sync(0xffffffffu, sd[q], s);
    }
#pragma unroll
    for (int q = 0; q < kOR; ++q) {
      if (!rv[q]) continue;
      const int b = b0 + q;
      const size_t e = (size_t)b * O + j;
      const int lbl = (int)y[q];
      if (do0 && on) d[e] = (float)((soft[q] - (j == lbl ? 1.0 : 0.0)) * scale);
      if (do1 && on) rd[e] = (float)(soft[q] * (ro[q] - sd[q]) * scale);
    }
#pragma unroll
    for (int q = 0; q < kOR; ++q) {
      const int lbl = (int)y[q];
      const float olbl = __shfl_sync(0xffffffffu, o[q], lbl & 31);
      if (do0 && j == 0 && rv[q]) {
        loss[b0 + q] = (double)bv[q] + log(den[q]) - (double)olbl;
        correct[b0 + q] = (ncls > 0 && bi[q] == lbl) ? 1 : 0;
      }
    }
  } else {
    double l[kOR];
#pragma unroll
    for (int q = 0; q < kOR; ++q) {
      const float t = ncls > 0 ? (j == (int)y[q] ? 1.f : 0.f) : (j == 0 ? y[q] : 0.f);
      const float df = (rv[q] && on) ? o[q] - t : 0.f;
      const size_t e = (size_t)(b0 + q) * O + j;
      if (rv[q] && do0 && on) d[e] = (float)(df * scale);
      if (rv[q] && do1 && on) rd[e] = (float)(ro[q] * scale);
      l[q] = 0.5 * (double)df * (double)df;
    }
#pragma unroll
    for (int s = 16; s > 0; s >>= 1)
#pragma unroll
      for (int q = 0; q < kOR; ++q) l[q] += __shfl_xor_sync(0xffffffffu, l[q], s);
#pragma unroll
    for (int q = 0; q < kOR; ++q)
      if (do0 && j == 0 && rv[q]) {
        loss[b0 + q] = l[q];
        correct[b0 + q] = (ncls > 0 && bi[q] == (int)y[q]) ? 1 : 0;
      }
  }
}

__device__ __forceinline__ double gflops(const SGemm& g) { return (double)g.M * g.N * g.K; }

// Output layer rows b in [b0, b1): a warp per sample (O <= 32; global warp index base_w + warp, stride sw), else
// a thread per sample (base_t + threadIdx.x, stride stt).
__device__ void output_rows(const SmallNet& net, const SmallCall& c, bool R, int b0, int b1, int base_w, int sw,
                            int base_t, int stt) {
  const int L = net.L, O = net.s[L];
  if (O <= 32) {  // groups of kOR consecutive samples per warp
    for (int b = b0 + (base_w + (int)(threadIdx.x >> 5)) * kOR; b < b1; b += sw * kOR)
      output_delta_warp(b, b1, O, net.mse, c.ncls, !R, R, c.scale, net.a32[L], net.ra32[L], c.lab, net.d32[L],
                        net.rd32[L], c.loss, c.correct);
  } else {
    for (int b = b0 + base_t + (int)threadIdx.x; b < b1; b += stt)
      output_delta_row<true>(b, O, net.mse, c.ncls, !R, R, c.scale, net.a32[L], net.ra32[L], c.lab, net.d32[L],
                             net.rd32[L], c.loss, c.correct);
  }
}

// All phases of one pass (mode c.mode; the direction v with scale vsc for the HVP), grid barriers between them
// (none after the last):
//   forward t = 0..L-1 | output (when the output layer is wider than a tile) | backward t = L-1..tlow
// The phase's GEMM descriptors live in shared memory (sg[2], built by thread 0). When the output layer has at
// most kT units its forward GEMM runs unsplit on 32-sample tiles and the CTA that finishes a tile applies the
// output delta to those samples (no separate output phase).
__device__ void pass_phases(const SmallNet& net, const SmallCall& c, const float* v, float vsc, Stage* ring,
                            unsigned& s_last, SGemm* sg, unsigned long long* bar_next) {
  const unsigned nb = gridDim.x;
  const bool R = c.mode == SM_HVP;
  const int L = net.L;
  const bool fuse_out = net.s[L] <= kT;
  const int tlow = c.mode == SM_PREP ? 1 : 0;
  const int nbwd = c.mode == SM_EVAL ? 0 : max(0, L - tlow);
  const int nph = L + (fuse_out ? 0 : 1) + nbwd;
  // labels of the batch (read by the output step, after at least one barrier or in the same CTA)
  if (c.mode != SM_HVP)
    for (int b = blockIdx.x * kThr + threadIdx.x; b < c.B; b += nb * kThr)
      c.lab[b] = __ldg(c.y + (c.idx ? c.idx[b] : b));
  stamp(c, 0);
  for (int ph = 0; ph < nph; ++ph) {
    const bool fwd = ph < L, outp = !fwd && !fuse_out && ph == L;
    const int t = fwd ? ph : L - 1 - (ph - L - (fuse_out ? 0 : 1));
    const bool fused_out = fwd && t == L - 1 && fuse_out;
    __syncthreads();  // sg of the previous phase is no longer read
    if (threadIdx.x == 0) {
      sg[0].units = sg[1].units = 0;
      if (fwd) {
        fwd_gemm(sg[0], net, c, v, t, R, vsc);
        plan(sg[0], (int)nb);
      } else if (!outp) {
        const bool wb = c.mode != SM_PREP;
        double fw = 0.0, fd = 0.0;
        if (wb) { wb_gemm(sg[0], net, c, t, R); fw = gflops(sg[0]); }
        if (t > 0) { bwd_gemm(sg[1], net, c, v, t, R, vsc); fd = gflops(sg[1]); }
        if (wb) plan(sg[0], max(1, (int)(nb * fw / (fw + fd))));
        if (t > 0) plan(sg[1], max(1, (int)(nb * fd / (fw + fd))));
        if (!wb) sg[0].units = 0;
        if (t == 0) sg[1].units = 0;
      }
    }
    __syncthreads();
    if (outp) {
      output_rows(net, c, R, 0, c.B, blockIdx.x * (kThr / 32), nb * (kThr / 32), blockIdx.x * kThr, nb * kThr);
    } else {
      const int u0 = sg[0].units, tot = u0 + sg[1].units;
      const size_t poff = (size_t)u0 * (kT * kT);
      const int toff = u0 ? (int)(cdiv(sg[0].M, kT) * cdiv(sg[0].N, kT)) : 0;
      for (int u = blockIdx.x; u < tot; u += nb) {
        const bool first = u < u0;
        const bool done = run_unit(first ? sg[0] : sg[1], net, c, v, vsc, first ? u : u - u0,
                                   first ? c.part : c.part + poff, first ? c.tickets : c.tickets + toff, ring, s_last);
        if (fused_out && done) {  // this unit completed the tile: its samples' output delta, here
          const int b0 = (u / sg[0].S / sg[0].tn) * kT;
          output_rows(net, c, R, b0, min(c.B, b0 + kT), 0, kThr / 32, 0, kThr);
          __syncthreads();
          if (c.trace && c.trace_t == t) stamp(c, 30);
        }
      }
    }
    stamp(c, 1 + 2 * ph);
    if (ph + 1 < nph) {
      grid_barrier(c.bar, nb, bar_next);
      stamp(c, 2 + 2 * ph);
    }
  }
}

__global__ void __launch_bounds__(kThr) mlp_small_kernel(const SmallNet net_p, const SmallCall c_p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ unsigned s_last;
  __shared__ SGemm sg[2];
  __shared__ SmallNet net;
  __shared__ SmallCall c;
  __shared__ unsigned long long bar_next;
  if (threadIdx.x == 0) {
    net = net_p;
    c = c_p;
    bar_next = 0ull;
  }
  __syncthreads();
  const float vsc = (c.mode == SM_HVP && c.vscale) ? __ldg(c.vscale) : 1.f;
  pass_phases(net, c, c.v, vsc, reinterpret_cast<Stage*>(smem_raw), s_last, sg, &bar_next);
}

// ------------------------------------------------------------------ fused small-model Lanczos refresh
// The whole recurrence of lanczos.cu (lanczos_enqueue: HVP, GS pass 1, GS pass 2, decide; the safeguard
// pass; breakdown) for a world-1 small-MLP operator as ONE persistent launch of m iterations. Per iteration:
//   HVP            pass_phases (v = sigma_i D_i), h complete at a grid barrier
//   pass 1         the first ngs CTAs own contiguous row slices: fp64 partial dots D_j^T h (j <= i),
//                  h^T h and (recurrence-first) G_j = D_j^T D_i, one row of partials per CTA; barrier
//   coefficients   every CTA adds the ngs partial rows in CTA order (identical in every CTA) and forms the
//                  projection coefficients (gs_pass2_kernel's formulas)
//   pass 2         D_{i+1} = h - sum_j D_j e_j on the slices, partial ||.||^2; barrier
//   decide         every CTA adds the norm partials in CTA order and applies lz_decide_kernel's rules, so
//                  all CTAs agree on sigma_{i+1} / stop / safeguard without another barrier; CTA 0 records
//                  the state (LzDev) for the host.
// Three barriers per iteration besides the HVP's own; no launches, no host round trips.
struct LzArgs {
  float* D;
  long long ldd;
  float* h;
  LzDev* st;
  double* part1;  // [ngs][stride]
  double* part2;  // [ngs]
  int n, m, gram, sg_on, stride, goff, ngs, rs;
  int sv_off;  // byte offset of the per-CTA arrays: after the stage ring / the pass-1 scratch, whichever is larger
  double ratio, rtol;  // floored on the host (fp32 adaptation, lanczos.cu)
  int kind;            // operator: 0 small MLP (pass_phases), 1 diagonal (h = spec o (sigma_i D_i), diag_apply_kernel)
  const float* spec;
};

// This CTA's slice: rows [blockIdx.x rs, min(n, (blockIdx.x + 1) rs)), float4 groups g = tid + kThr q
// (rs <= 2 kThr 4 rows: q < 2). Rows >= n of D and h are zero.
constexpr int kGsq = 2;

// Pass 1 partial row of this CTA: [0, active) D_j^T y, [active] y^T y, then (gram) D_j^T D_i; D_j read once
// for both dots, 8 columns x kGsq groups of loads in flight, fp64 sums of fp32 products, the 16 values of a
// column batch reduced across the warp by one butterfly; warps added in warp order.
__device__ void gs_dots(const LzArgs& a, const float* y, int active, int it, bool gram, double* sacc, double* srow) {
  const long long r0 = (long long)blockIdx.x * a.rs, r1 = min((long long)a.n, r0 + a.rs);
  const int ng = (int)max(0LL, (r1 - r0 + 3) / 4);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nj = active + 1, rowlen = nj + (gram ? active : 0);
  for (int e = lane; e < rowlen; e += 32) sacc[warp * rowlen + e] = 0.0;  // warp-private rows
  __syncwarp();
  // row tiles of kThr kGsq float4 groups: y (and D_i) in registers per tile, columns in batches of 8
  for (int g0 = 0; g0 < ng; g0 += kThr * kGsq) {
    float4 yv[kGsq], zv[kGsq];
#pragma unroll
    for (int q = 0; q < kGsq; ++q) {
      const int g = g0 + tid + kThr * q;
      const bool on = g < ng;
      yv[q] = on ? __ldcg(reinterpret_cast<const float4*>(y + r0) + g) : make_float4(0.f, 0.f, 0.f, 0.f);
      zv[q] = (on && gram) ? __ldcg(reinterpret_cast<const float4*>(a.D + (long long)it * a.ldd + r0) + g)
                           : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    for (int j0 = 0; j0 < nj; j0 += 8) {
      float4 x[8][kGsq];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int j = j0 + u;
#pragma unroll
        for (int q = 0; q < kGsq; ++q) {
          const int g = g0 + tid + kThr * q;
          if (j < active && g < ng) x[u][q] = __ldcg(reinterpret_cast<const float4*>(a.D + (long long)j * a.ldd + r0) + g);
          else x[u][q] = j == active ? yv[q] : make_float4(0.f, 0.f, 0.f, 0.f);
        }
      }
      double v[16];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        double sy = 0.0, sz = 0.0;
#pragma unroll
        for (int q = 0; q < kGsq; ++q) {
          sy += (double)x[u][q].x * yv[q].x + (double)x[u][q].y * yv[q].y + (double)x[u][q].z * yv[q].z +
                (double)x[u][q].w * yv[q].w;
          sz += (double)x[u][q].x * zv[q].x + (double)x[u][q].y * zv[q].y + (double)x[u][q].z * zv[q].z +
                (double)x[u][q].w * zv[q].w;
        }
        v[2 * u] = sy;
        v[2 * u + 1] = sz;
      }
      const double t = butterfly_sum<16>(v, lane);
      if (lane < 16) {
        const int idx = butterfly_index<16>(lane);
        const int j = j0 + (idx >> 1);
        if (idx & 1) {
          if (gram && j < active) sacc[warp * rowlen + nj + j] += t;
        } else if (j < nj) {
          sacc[warp * rowlen + j] += t;
        }
      }
    }
  }
  __syncthreads();
  for (int e = tid; e < rowlen; e += kThr) {
    double t = 0.0;
    for (int w = 0; w < kThr / 32; ++w) t += sacc[w * rowlen + e];
    srow[e] = t;
  }
}

__global__ void __launch_bounds__(kThr) lanczos_small_kernel(const SmallNet net_p, const SmallCall c_p, const LzArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ unsigned s_last;
  __shared__ double s_b2;
  __shared__ SGemm sg[2];
  __shared__ SmallNet net;
  __shared__ SmallCall c;
  __shared__ unsigned long long bar_next;
  if (threadIdx.x == 0) {
    net = net_p;
    c = c_p;
    bar_next = 0ull;
  }
  __syncthreads();
  Stage* ring = reinterpret_cast<Stage*>(smem_raw);
  const int mm = a.m;
  double* sv = reinterpret_cast<double*>(smem_raw + a.sv_off);  // [2 mm + 2] this CTA's pass-1 row, then sums
  double* se = sv + (2 * mm + 2);                              // [mm + 1] coefficients
  double* gcur = se + (mm + 1);                                // [mm + 1] G_j of this iteration
  double* gprev = gcur + (mm + 1);                             // [mm + 1] G_j of the previous one
  float* sig = reinterpret_cast<float*>(gprev + (mm + 1));     // [mm + 2] sigma_j
  const unsigned nb = gridDim.x;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  LzDev* st = a.st;
  if (tid == 0) sig[0] = __ldcg(&st->sigma[0]);
  __syncthreads();
  const bool gs_cta = (int)blockIdx.x < a.ngs;
  double beta_prev = 0.0;  // off[it - 1]
  double pre = 0.0;
  int sg_count = 0;
  long long sg_cols = 0;
  for (int it = 0; it < mm; ++it) {
    const int active = it + 1;
    // ---- HVP: h = H (sigma_it D_it)
    const bool trace_it = it == 20;
    if (trace_it) stamp(c, 20);
    if (a.kind == 0) {
      pass_phases(net, c, a.D + (long long)it * a.ldd, sig[it], ring, s_last, sg, &bar_next);
    } else {  // diagonal operator (diag_apply_kernel's arithmetic)
      const float sc = sig[it];
      const float* vi = a.D + (long long)it * a.ldd;
      for (long long r = (long long)blockIdx.x * kThr + tid; r < a.n; r += (long long)nb * kThr)
        a.h[r] = (float)((double)__ldg(a.spec + r) * (double)(sc * __ldcg(vi + r)));
    }
    grid_barrier(c.bar, nb, &bar_next);
    if (trace_it) stamp(c, 21);
    float* Dn = a.D + (long long)(it + 1) * a.ldd;
    bool stop = false, need_sg = false;
    double alpha = 0.0, alpha0 = 0.0, beta = 0.0;
    for (int pass = 0; pass < (a.sg_on ? 2 : 1); ++pass) {
      if (pass == 1 && !need_sg) break;
      const float* hsrc = pass == 0 ? a.h : Dn;
      const bool rec = a.gram && pass == 0;
      const int nj = active + 1, rowlen = nj + (rec ? active : 0);
      // ---- pass 1: this slice's partial row
      double* sacc = reinterpret_cast<double*>(ring);  // the HVP's stage ring is free until the next HVP
      if (gs_cta) {
        gs_dots(a, hsrc, active, it, rec, sacc, sv);
        __syncthreads();
        for (int e = tid; e < rowlen; e += kThr) __stcg(a.part1 + (size_t)blockIdx.x * a.stride + e, sv[e]);
      }
      if (trace_it && pass == 0) stamp(c, 22);
      grid_barrier(c.bar, nb, &bar_next);
      if (trace_it && pass == 0) stamp(c, 23);
      // ---- every CTA: the partial rows added in a fixed order
      reduce_rows<kThr>(a.part1, a.ngs, a.stride, rowlen, sacc, sv);
      if (trace_it && pass == 0) stamp(c, 24);
      // ---- coefficients (gs_pass2_kernel)
      const double sgi = (double)sig[it];
      alpha = sgi * sv[it];
      if (pass == 0) {
        alpha0 = alpha;
        pre = sqrt(sv[active]);
      }
      for (int j = tid; j < active; j += kThr) {
        const double sj = (double)sig[j];
        const double r = sv[j];
        if (rec) {
          const double g = sv[nj + j];
          gcur[j] = g;
          const double sp = it > 0 ? (double)sig[it - 1] : 0.0;
          const double gp = it == 0 ? 0.0 : (j < it ? gprev[j] : sv[nj + it - 1]);
          const double cc = sj * (r - alpha * sgi * g - beta_prev * sp * gp);
          double ej = sj * cc;
          if (j == it) ej += alpha * sgi;
          if (j == it - 1) ej += beta_prev * sp;
          se[j] = ej;
        } else {
          se[j] = sj * sj * r;
        }
      }
      __syncthreads();
      if (blockIdx.x == 0 && tid == 0 && pass == 0) {
        st->diag[it] = alpha;
        st->pre = pre;
      }
      if (blockIdx.x == 0 && rec)
        for (int j = tid; j < active; j += kThr) st->gram[it & 1][j] = gcur[j];
      // ---- pass 2: Dn = hsrc - sum_j D_j e_j on this slice (8 columns x kGsq groups of loads in flight),
      // partial ||Dn||^2
      if (gs_cta) {
        const long long r0 = (long long)blockIdx.x * a.rs, r1 = min((long long)a.n, r0 + a.rs);
        const int ng = (int)max(0LL, (r1 - r0 + 3) / 4);
        double ss = 0.0;
        for (int g0 = 0; g0 < ng; g0 += kThr * kGsq) {
          double acc[kGsq][4];
#pragma unroll
          for (int q = 0; q < kGsq; ++q) {
            const int g = g0 + tid + kThr * q;
            const float4 h4 = g < ng ? __ldcg(reinterpret_cast<const float4*>(hsrc + r0) + g) : make_float4(0.f, 0.f, 0.f, 0.f);
            acc[q][0] = h4.x; acc[q][1] = h4.y; acc[q][2] = h4.z; acc[q][3] = h4.w;
          }
          for (int j0 = 0; j0 < active; j0 += 8) {
            float4 d[8][kGsq];
#pragma unroll
            for (int u = 0; u < 8; ++u)
#pragma unroll
              for (int q = 0; q < kGsq; ++q) {
                const int g = g0 + tid + kThr * q;
                d[u][q] = (j0 + u < active && g < ng)
                              ? __ldcg(reinterpret_cast<const float4*>(a.D + (long long)(j0 + u) * a.ldd + r0) + g)
                              : make_float4(0.f, 0.f, 0.f, 0.f);
              }
#pragma unroll
            for (int u = 0; u < 8; ++u) {
              const double cj = j0 + u < active ? se[j0 + u] : 0.0;
#pragma unroll
              for (int q = 0; q < kGsq; ++q) {
                acc[q][0] -= (double)d[u][q].x * cj;
                acc[q][1] -= (double)d[u][q].y * cj;
                acc[q][2] -= (double)d[u][q].z * cj;
                acc[q][3] -= (double)d[u][q].w * cj;
              }
            }
          }
#pragma unroll
          for (int q = 0; q < kGsq; ++q) {
            const int g = g0 + tid + kThr * q;
            if (g < ng) {
              const float4 o = make_float4((float)acc[q][0], (float)acc[q][1], (float)acc[q][2], (float)acc[q][3]);
              __stcg(reinterpret_cast<float4*>(Dn + r0) + g, o);
              ss += (double)o.x * o.x + (double)o.y * o.y + (double)o.z * o.z + (double)o.w * o.w;
            }
          }
        }
        ss = warp_sum(ss);
        __syncthreads();  // sv (the row sums) is reused below
        if (lane == 0) sv[warp] = ss;
        __syncthreads();
        if (tid == 0) {
          double t = 0.0;
          for (int w = 0; w < kThr / 32; ++w) t += sv[w];
          __stcg(a.part2 + blockIdx.x, t);
        }
      }
      if (trace_it && pass == 0) stamp(c, 25);
      grid_barrier(c.bar, nb, &bar_next);
      if (trace_it && pass == 0) stamp(c, 26);
      // ---- decide (lz_decide_kernel), identically in every CTA
      if (warp == 0) {
        double t = 0.0;
        for (int q = lane; q < a.ngs; q += 32) t += __ldcg(a.part2 + q);
        t = warp_sum(t);
        if (lane == 0) s_b2 = t;
      }
      __syncthreads();
      beta = sqrt(s_b2);
      need_sg = false;
      if (!isfinite(pre) || !isfinite(beta) || !isfinite(alpha0)) {
        if (blockIdx.x == 0 && tid == 0) {
          st->nonfinite = 1;
          st->stopped = 1;
          st->iters = it;
        }
        stop = true;
        break;
      }
      if (blockIdx.x == 0 && tid == 0) st->beta = beta;
      if (pass == 0 && a.sg_on && beta > a.rtol * pre && beta < a.ratio * pre) {
        need_sg = true;
        sg_count += 1;
        sg_cols += it + 1;
        if (blockIdx.x == 0 && tid == 0) {
          st->need_sg = 1;
          st->safeguards = sg_count;
          st->sg_cols = sg_cols;
        }
        continue;
      }
      if (blockIdx.x == 0 && tid == 0) st->need_sg = 0;
      if (beta <= a.rtol * pre) {  // invariant subspace: truncate
        if (blockIdx.x == 0 && tid == 0) {
          st->breakdown = 1;
          st->stopped = 1;
          st->iters = it + 1;
        }
        stop = true;
        break;
      }
      break;
    }
    if (stop) break;
    if (tid == 0) sig[it + 1] = (float)(1.0 / beta);
    if (blockIdx.x == 0 && tid == 0) {
      st->off[it] = beta;
      st->sigma[it + 1] = (float)(1.0 / beta);
      st->iters = it + 1;
    }
    beta_prev = beta;
    if (a.gram)
      for (int j = tid; j < active; j += kThr) gprev[j] = gcur[j];
    __syncthreads();
  }
}
}  // namespace

// ------------------------------------------------------------------ host side
bool mlp_small_eligible(const dho2g_mlp* m, size_t B) {
  const dho2g_ctx* ctx = m->ctx;
  if (!ctx->mlp_small || ctx->gemm_backend != 0 || m->L > kMaxL || B == 0) return false;
  double f = 0.0;  // HVP flops
  for (int t = 0; t < m->L; ++t) f += 2.0 * (double)B * (5 + 3 * (t > 0)) * (double)m->sizes[t] * m->sizes[t + 1];
  return f <= ctx->mlp_small_mflop * 1e6;
}

// Scratch: split partials and tickets sized for the largest phase (units <= ctas x ~2 per GEMM plus the
// tiles of unsplit GEMMs), the barrier words.
static void small_scratch(dho2g_mlp* m, size_t B) {
  size_t units = 0, tiles = 0;
  for (int t = 0; t < m->L; ++t) {
    const size_t in = m->sizes[t], out = m->sizes[t + 1];
    const size_t tf = cdiv(B, kT) * cdiv(out, kT), tw = cdiv(out, kT) * cdiv(in + 1, kT), td = cdiv(B, kT) * cdiv(in, kT);
    const size_t cap = (size_t)m->ctx->sm_count * 4;
    units = std::max(units, std::max(tf, cap) + std::max(tw, cap) + std::max(td, cap));
    tiles = std::max(tiles, tf + tw + td);
  }
  // (zeroed at allocation; every launch leaves the tickets and the barrier count at zero)
  m->sm_part.ensure_g(units * kT * kT);
  m->sm_tickets.ensure_g(tiles + 2);
  m->sm_bar.ensure_g((size_t)kBarShards * kBarStride);
}

void mlp_small_presize(dho2g_mlp* m, size_t B) { small_scratch(m, B); }

static void setup_call(dho2g_mlp* m, int mode, size_t B, const float* w, const float* v, const float* vscale,
                       float* out, size_t ncls, double scale, SmallNet& net, SmallCall& c) {
  m->ensure_batch(B);
  small_scratch(m, B);
  net = SmallNet{};
  net.L = m->L;
  net.relu = m->act == 1;
  net.mse = m->loss;
  for (int j = 0; j <= m->L; ++j) {
    net.s[j] = (int)m->sizes[j];
    if (j >= 1) {
      net.a32[j] = m->a32[j].p; net.ra32[j] = m->ra32[j].p; net.d32[j] = m->d32[j].p; net.rd32[j] = m->rd32[j].p;
      net.u32[j] = j < m->L ? m->u32[j].p : nullptr;
    }
  }
  for (int t = 0; t < m->L; ++t) {
    net.w_off[t] = (long long)m->layers[t].w_off;
    net.b_off[t] = (long long)m->layers[t].b_off;
  }
  c = SmallCall{};
  c.mode = mode;
  c.B = (int)B;
  c.ncls = (int)ncls;
  c.ldx = (int)m->sizes[0];
  c.cache_u = mode == SM_PREP;
  c.scale = scale;
  c.w = w;
  c.v = v;
  c.vscale = vscale;
  c.out = out;
  c.X = m->x_src;
  c.idx = m->x_idx;
  c.y = m->y_src;
  c.lab = m->lab.p;
  c.loss = m->sample_loss.p;
  c.correct = m->sample_correct.p;
  c.part = m->sm_part.p;
  c.tickets = m->sm_tickets.p;
  c.bar = m->sm_bar.p;
  c.route = mode == SM_GRAD || mode == SM_HVP ? m->route : nullptr;
  c.route_base = m->route_base;
  c.route_rank = m->route_rank;
}

// Cooperative launch of `kernel` on ctas CTAs (kThr threads, smem dynamic bytes); the barrier counter is reset
// when the grid size changes (generations are counted in units of it).
template <typename... Args>
static void coop_launch(dho2g_ctx* ctx, void (*kernel)(Args...), int ctas, size_t smem, Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)ctas);
  cfg.blockDim = dim3(kThr);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = ctx->stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;  // co-residency of every CTA (grid barriers)
  at[0].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  DHO2G_CUDA(cudaLaunchKernelEx(&cfg, kernel, args...));
  DHO2G_LAUNCH();
}

// CTAs of a cooperative grid: ctx option mlp_small_ctas_per_sm per SM, capped by the occupancy at smem bytes
template <typename K>
static int coop_ctas(dho2g_ctx* ctx, K kernel, size_t smem, size_t* attr_set) {
  if (*attr_set < smem) {
    DHO2G_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    *attr_set = smem;
  }
  int per_sm = 0;
  DHO2G_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, kThr, smem));
  if (per_sm < 1) fail(DHO2G_CUDA, "small-model path: kernel does not fit on an SM");
  return ctx->sm_count * std::min(std::max(1, ctx->mlp_small_ctas_per_sm), per_sm);
}

void mlp_small_run(dho2g_mlp* m, int mode, size_t B, const float* w, const float* v, const float* vscale, float* out,
                   size_t ncls, double scale) {
  dho2g_ctx* ctx = m->ctx;
  SmallNet net;
  SmallCall c;
  setup_call(m, mode, B, w, v, vscale, out, ncls, scale, net, c);
  static size_t attr = 0;
  static int ctas_cached = 0, opt_cached = -1;
  if (opt_cached != ctx->mlp_small_ctas_per_sm) {
    ctas_cached = coop_ctas(ctx, mlp_small_kernel, kSmem, &attr);
    opt_cached = ctx->mlp_small_ctas_per_sm;
  }
  const int ctas = ctas_cached;
  static const char* names[] = {"mlp_small.grad", "mlp_small.prep", "mlp_small.hvp", "mlp_small.eval"};
  static const bool tracing = getenv("DHO2G_SMALL_TRACE") != nullptr;
  static DevBuf<unsigned long long> tbuf;
  if (tracing) {
    tbuf.ensure((size_t)ctas * 32);
    DHO2G_CUDA(cudaMemsetAsync(tbuf.p, 0, (size_t)ctas * 32 * 8, ctx->stream));
    c.trace = tbuf.p;
  }
  const int slot = ctx->kt_begin();
  if (m->sm_bar_nb != ctas) {  // barrier generations are counted in units of the grid size
    DHO2G_CUDA(cudaMemsetAsync(m->sm_bar.p, 0, m->sm_bar.n * sizeof(unsigned long long), ctx->stream));
    m->sm_bar_nb = ctas;
  }
  coop_launch(ctx, mlp_small_kernel, ctas, kSmem, net, c);
  ctx->kt_end(slot, names[mode], 0.0);
  if (tracing) {
    std::vector<unsigned long long> h((size_t)ctas * 32);
    DHO2G_CUDA(cudaMemcpyAsync(h.data(), tbuf.p, h.size() * 8, cudaMemcpyDeviceToHost, ctx->stream));
    DHO2G_CUDA(cudaStreamSynchronize(ctx->stream));
    unsigned long long t0 = ~0ull;
    for (int b = 0; b < ctas; ++b) t0 = std::min(t0, h[(size_t)b * 32]);
    fprintf(stderr, "[small %s B=%zu ctas=%d]", names[mode], B, ctas);
    for (int i = 1; i < 32; ++i) {
      double mx = 0, sum = 0;
      int cnt = 0;
      for (int b = 0; b < ctas; ++b) {
        const unsigned long long v = h[(size_t)b * 32 + i];
        if (!v) continue;
        mx = std::max(mx, (v - t0) * 1e-3);
        sum += (v - t0) * 1e-3;
        ++cnt;
      }
      if (cnt) fprintf(stderr, " %d:%.1f/%.1f", i, sum / cnt, mx);
    }
    fprintf(stderr, "\n");
  }
}

// ------------------------------------------------------------------ fused refresh (host side)
// [ring | pass-1 scratch (8 warps x rowlen, or rowlen x CTA chunks)] then sv, se, gcur, gprev (doubles), sig
static size_t lz_small_scratch(size_t m) {
  const size_t rowlen = 2 * m + 1;
  return round_up(std::max(kSmem, (size_t)8 * rowlen * sizeof(double)), 16);
}
static size_t lz_small_smem(size_t m) {
  return lz_small_scratch(m) + (2 * m + 2 + 3 * (m + 1)) * sizeof(double) + (m + 2) * sizeof(float);
}

bool lanczos_small_eligible(const dho2g_lanczos* lz, const dho2g_op* op) {
  const dho2g_ctx* ctx = lz->ctx;
  if (!ctx->lanczos_small || ctx->world != 1 || lz->m > 512 || lz->rows != lz->n) return false;  // (m: smem)
  // diagonal operator: supported (kind 1), but only on request (lanczos_small 2): at n >= 1e6 the
  // launch-per-step Gram-Schmidt kernels stream HBM faster (measured: profiles/r02_c5_fused.txt)
  if (op->kind == 1) return ctx->lanczos_small == 2 && lz->n <= (size_t)ctx->lanczos_small_max_n;
  if (op->kind != 0 || op->b1 <= op->b0) return false;
  return lz->n <= (size_t)ctx->lanczos_small_max_n && mlp_small_eligible(op->mlp, op->b1 - op->b0);
}

void lanczos_small_run(dho2g_lanczos* lz, dho2g_op* op) {
  dho2g_ctx* ctx = lz->ctx;
  SmallNet net{};
  SmallCall c{};
  dho2g_mlp* m = op->kind == 0 ? op->mlp : nullptr;
  if (m) {
    const size_t B = op->b1 - op->b0;
    op->load_mlp_input();
    if (m->prepared != m->w_cur || !m->prepared_small) mlp_prepare_point(m, B, op->ncls, op->scale);
    setup_call(m, SM_HVP, B, m->w_cur, nullptr, nullptr, lz->h.p, op->ncls, op->scale, net, c);
  } else {  // diagonal operator: the launch only needs the barrier words (kept on the Lanczos state)
    if (!lz->sm_bar.p) lz->sm_bar.ensure_g((size_t)kBarShards * kBarStride);
    c.bar = lz->sm_bar.p;
  }
  const size_t smem = lz_small_smem(lz->m);
  static size_t attr = 0;
  const int ctas = coop_ctas(ctx, lanczos_small_kernel, smem, &attr);
  LzArgs a{};
  a.D = lz->D.p;
  a.ldd = (long long)lz->ldd;
  a.h = lz->h.p;
  a.st = lz->st.p;
  a.n = (int)lz->n;
  a.m = (int)lz->m;
  a.gram = ctx->lanczos_recurrence ? 1 : 0;
  a.sg_on = lz->opts.reorth_safeguard ? 1 : 0;
  a.stride = (int)(2 * (lz->m + 2));
  a.goff = (int)(lz->m + 2);
  a.ngs = (int)std::min<size_t>((size_t)ctas, std::max<size_t>(1, cdiv(lz->n, 256)));  // >= 64 groups per slice
  a.rs = (int)round_up(cdiv(lz->n, (size_t)a.ngs), 4);
  a.sv_off = (int)lz_small_scratch(lz->m);
  a.kind = op->kind;
  a.spec = op->kind == 1 ? op->mat.p + lz->begin : nullptr;
  a.ratio = std::max(lz->opts.safeguard_ratio, kSafeguardFloor32);
  a.rtol = std::max(lz->opts.breakdown_rtol, kBreakdownFloor32);
  lz->sm_part1.ensure_g((size_t)a.ngs * a.stride);
  lz->sm_part2.ensure_g((size_t)a.ngs);
  a.part1 = lz->sm_part1.p;
  a.part2 = lz->sm_part2.p;
  static const bool tracing = getenv("DHO2G_SMALL_TRACE") != nullptr;
  static DevBuf<unsigned long long> tbuf;
  if (tracing) {
    tbuf.ensure((size_t)ctas * 32);
    DHO2G_CUDA(cudaMemsetAsync(tbuf.p, 0, (size_t)ctas * 32 * 8, ctx->stream));
    c.trace = tbuf.p;
    c.trace_t = getenv("DHO2G_SMALL_TRACE")[0] - '0';
  }
  const int slot = ctx->kt_begin();
  int& bar_nb = m ? m->sm_bar_nb : lz->sm_bar_nb;
  if (bar_nb != ctas) {  // barrier generations are counted in units of the grid size
    DHO2G_CUDA(cudaMemsetAsync(c.bar, 0, (size_t)kBarShards * kBarStride * sizeof(unsigned long long), ctx->stream));
    bar_nb = ctas;
  }
  coop_launch(ctx, lanczos_small_kernel, ctas, smem, net, c, a);
  if (tracing) {  // iteration 20: 20 start, 21 h complete, 22 pass-1 partials, 23 barrier, 24 sums, 25 pass 2, 26 barrier
    std::vector<unsigned long long> hb((size_t)ctas * 32);
    DHO2G_CUDA(cudaMemcpyAsync(hb.data(), tbuf.p, hb.size() * 8, cudaMemcpyDeviceToHost, ctx->stream));
    DHO2G_CUDA(cudaStreamSynchronize(ctx->stream));
    unsigned long long t0 = ~0ull;
    for (int b = 0; b < ctas; ++b) t0 = std::min(t0, hb[(size_t)b * 32 + 20]);
    fprintf(stderr, "[lanczos_small it=20 ctas=%d ngs=%d]", ctas, a.ngs);
    for (int i = 0; i < 32; ++i) {
      double mx = -1e30, sum = 0;
      int cnt = 0;
      for (int b = 0; b < ctas; ++b) {
        const unsigned long long v = hb[(size_t)b * 32 + i];
        if (!v || v < t0) continue;
        mx = std::max(mx, (v - t0) * 1e-3);
        sum += (v - t0) * 1e-3;
        ++cnt;
      }
      if (cnt) fprintf(stderr, " %d:%.1f/%.1f", i, sum / cnt, mx);
    }
    fprintf(stderr, "\n");
  }
  // algorithmic bytes of the Gram-Schmidt sweeps (the §8d figure, as gs_pass1 / gs_pass2 count them: pass 1
  // reads the active columns and h, pass 2 the same plus the new column), m iterations; the HVPs are not counted
  double gsb = 0.0;
  for (size_t i = 0; i < lz->m; ++i) gsb += 4.0 * (double)lz->n * (2.0 * (double)(i + 2) + 1.0);
  ctx->kt_end(slot, "lanczos_small", gsb);
}

}  // namespace dho2g
