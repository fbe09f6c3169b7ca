// Latency probe for the tridiagonal QL chain (tql2_ql_kernel): cycles per rotation of the recorded
// sweep loop vs its pieces (dependent DFMA / DMUL chain, rsqrt(double) chain).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ql_probe scripts/ql_chain_probe.cu && /tmp/ql_probe
#include <cstdio>
#include <cuda_runtime.h>

__global__ void chain_dfma(double* out, long long* cyc, int n) {
  double a = out[0], b = out[1];
  const long long t0 = clock64();
  for (int i = 0; i < n; ++i) a = fma(a, b, 1e-9);
  const long long t1 = clock64();
  out[2] = a;
  cyc[0] = t1 - t0;
}

__global__ void chain_rsqrt(double* out, long long* cyc, int n) {
  double a = out[0] + 2.0;
  const long long t0 = clock64();
  for (int i = 0; i < n; ++i) a = rsqrt(a) + 1.5;
  const long long t1 = clock64();
  out[2] = a;
  cyc[0] = t1 - t0;
}

// one QL sweep of length n over smem d / e, `store` selects the rotation log store
template <bool STORE>
__global__ void sweep(const double* din, double2* rot, long long* cyc, int n, int reps) {
  extern __shared__ double sh[];
  double* d = sh;
  double* e = d + n;
  for (int i = 0; i < n; ++i) {
    d[i] = din[i];
    e[i] = 0.3 + 0.01 * (i % 7);
  }
  long long tot = 0;
  double acc = 0.0;
  for (int rep = 0; rep < reps; ++rep) {
    const int l = 0, mm = n - 1;
    const long long t0 = clock64();
    double g = (d[l + 1] - d[l]) / (2.0 * e[l]);
    double r = sqrt(fma(g, g, 1.0));
    g = d[mm] - d[l] + e[l] / (g + copysign(r, g));
    double s = 1.0, c = 1.0, p = 0.0;
    double dk = d[mm], ek = e[mm - 1], dn = d[mm - 1];
    int cnt = 0;
    for (int ii = mm - 1; ii >= l; --ii) {
      const double en = ii > l ? e[ii - 1] : 0.0, dnn = ii > l ? d[ii - 1] : 0.0;
      const double f = s * ek;
      const double b = c * ek;
      const double h2 = fma(f, f, g * g);
      if (h2 == 0.0) break;
      const double ir = rsqrt(h2);
      r = h2 * ir;
      e[ii + 1] = r;
      s = f * ir;
      c = g * ir;
      g = dk - p;
      r = (dn - g) * s + 2.0 * c * b;
      p = s * r;
      d[ii + 1] = g + p;
      g = c * r - b;
      if (STORE) rot[cnt] = make_double2(c, s);
      ++cnt;
      dk = dn;
      dn = dnn;
      ek = en;
    }
    d[l] -= p;
    e[l] = g;
    tot += clock64() - t0;
    acc += d[0];
    for (int i = 0; i < n; ++i) e[i] = 0.3 + 0.01 * (i % 7);
  }
  cyc[0] = tot;
  if (acc == 12345.0) cyc[1] = 1;
}

int main() {
  double* buf;
  long long* cyc;
  double2* rot;
  const int n = 512, reps = 20;
  cudaMalloc(&buf, 4096 * sizeof(double));
  cudaMalloc(&cyc, 16);
  cudaMalloc(&rot, n * sizeof(double2));
  double h[4096];
  for (int i = 0; i < 4096; ++i) h[i] = 1.0 + 0.001 * i;
  cudaMemcpy(buf, h, sizeof(h), cudaMemcpyHostToDevice);
  long long c;
  const int N = 100000;
  chain_dfma<<<1, 1>>>(buf, cyc, N);
  chain_dfma<<<1, 1>>>(buf, cyc, N);
  cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  printf("dependent DFMA        %6.1f cycles\n", (double)c / N);
  chain_rsqrt<<<1, 1>>>(buf, cyc, N);
  chain_rsqrt<<<1, 1>>>(buf, cyc, N);
  cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  printf("rsqrt(double) + DADD  %6.1f cycles\n", (double)c / N);
  sweep<true><<<1, 1, 2 * n * 8>>>(buf, rot, cyc, n, reps);
  sweep<true><<<1, 1, 2 * n * 8>>>(buf, rot, cyc, n, reps);
  cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  printf("QL sweep, log stored  %6.1f cycles per rotation\n", (double)c / reps / (n - 1));
  sweep<false><<<1, 1, 2 * n * 8>>>(buf, rot, cyc, n, reps);
  cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  printf("QL sweep, no log      %6.1f cycles per rotation\n", (double)c / reps / (n - 1));
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
