// MLP device helpers shared by the GEMM-epilogue path (mlp.cu) and the persistent small-model path
// (mlp_small.cu).
#pragma once
#include "common.cuh"

namespace dho2g {

// COH: the inputs were written earlier in the same launch by other CTAs, so they are read through L2
// (ld.global.cg) instead of a possibly stale L1 line.
template <bool COH>
__device__ __forceinline__ float odl(const float* p) {
  if constexpr (COH) return __ldcg(p);
  else return *p;
}

// Output layer delta for sample b: oracle.cpp:476-495 (delta) and :572-599 (R-delta); also the
// per-sample loss and correctness.
template <bool COH>
__device__ __forceinline__ void output_delta_row(int b, int O, int mse, int ncls, int do0, int do1, double scale,
                                                 const float* z, const float* rz, const float* lab,
                                                 float* __restrict__ d, float* __restrict__ rd,
                                                 double* __restrict__ loss, int* __restrict__ correct) {
  const float* o = z + (size_t)b * O;
  const float* ro = do1 ? rz + (size_t)b * O : nullptr;
  float* dd = d + (size_t)b * O;
  float* rdd = do1 ? rd + (size_t)b * O : nullptr;
  const float y = odl<COH>(lab + b);
  int best = 0;
  float ob = odl<COH>(o);
  for (int j = 1; j < O; ++j) {
    const float oj = odl<COH>(o + j);
    if (oj > ob) {
      best = j;
      ob = oj;
    }
  }
  if (do0) correct[b] = (ncls > 0 && best == (int)y) ? 1 : 0;
  if (!mse) {
    const int lbl = (int)y;
    const float mx = ob;
    double den = 0.0;
    for (int j = 0; j < O; ++j) den += exp((double)odl<COH>(o + j) - (double)mx);
    double sdot = 0.0;
    for (int j = 0; j < O; ++j) {
      const double soft = exp((double)odl<COH>(o + j) - (double)mx) / den;
      if (do0) dd[j] = (float)((soft - (j == lbl ? 1.0 : 0.0)) * scale);
      if (do1) sdot += soft * odl<COH>(ro + j);
    }
    if (do1)
      for (int j = 0; j < O; ++j) {
        const double soft = exp((double)odl<COH>(o + j) - (double)mx) / den;
        rdd[j] = (float)(soft * (odl<COH>(ro + j) - sdot) * scale);
      }
    if (do0) loss[b] = (double)mx + log(den) - (double)odl<COH>(o + lbl);
  } else {
    double acc = 0.0;
    for (int j = 0; j < O; ++j) {
      const float t = ncls > 0 ? (j == (int)y ? 1.f : 0.f) : (j == 0 ? y : 0.f);
      const float df = odl<COH>(o + j) - t;
      if (do0) dd[j] = (float)(df * scale);
      if (do1) rdd[j] = (float)(odl<COH>(ro + j) * scale);
      acc += 0.5 * (double)df * (double)df;
    }
    if (do0) loss[b] = acc;
  }
}

}  // namespace dho2g
