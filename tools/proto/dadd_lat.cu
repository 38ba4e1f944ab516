// Microbenchmark: latency of a dependent fp64 add chain on one thread, and
// of the same chain with the binade-key test of the exact-order engine.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void chain(const double* v, int n, double* out, long long* cyc) {
  double s = 1.0;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) s = __dadd_rn(s, v[i & 1023]);
  long long t1 = clock64();
  double a = 1.0, b = 1.0 + 2.220446049250313e-16;
  unsigned key = (unsigned)((unsigned long long)__double_as_longlong(a) >> 52);
  int bad = 0;
  for (int i = 0; i < n; i += 4) {
    double q[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) { a = __dadd_rn(a, v[(i + k) & 1023]); b = __dadd_rn(b, v[(i + k) & 1023]); q[k] = a; }
#pragma unroll
    for (int k = 0; k < 4; ++k) bad += ((unsigned)((unsigned long long)__double_as_longlong(q[k]) >> 52)) != key;
  }
  long long t2 = clock64();
  double z = 0;
  for (int i = 0; i < n; ++i) z = __dadd_rn(z, __ldcg(v + i));
  long long t3 = clock64();
  out[0] = s + a + b + bad + z;
  cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2;
}
int main() {
  int n = 1 << 16;
  double *v, *o; long long* c;
  cudaMalloc(&v, sizeof(double) * n); cudaMemset(v, 0, sizeof(double) * n);
  cudaMalloc(&o, 8); cudaMalloc(&c, 24);
  chain<<<1, 1>>>(v, n, o, c); cudaDeviceSynchronize();
  chain<<<1, 1>>>(v, n, o, c);
  long long h[3]; cudaMemcpy(h, c, 24, cudaMemcpyDeviceToHost);
  printf("dadd chain: %.2f cyc/step; 2 chains + key test (x4 unrolled): %.2f cyc/step; ldcg+dadd: %.2f cyc/step\n",
         (double)h[0] / n, (double)h[1] / n, (double)h[2] / n);
}
