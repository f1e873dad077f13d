// Latency microbenchmarks (diagnostic): dependent chains of FP64 ops on one warp.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ double rcp_nr(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double t = fma(-x, r, 1.0);
  r = fma(r, t, r);
  t = fma(-x, r, 1.0);
  return fma(r, t, r);
}
__device__ __forceinline__ double rsqrt_nr(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double hx = 0.5 * x;
  y = y * fma(-hx * y, y, 1.5);
  y = y * fma(-hx * y, y, 1.5);
  return y;
}
__global__ void lat(double* out, long long* cyc, double a) {
  __shared__ double sm[64];
  const int lane = threadIdx.x;
  sm[lane] = a + lane;
  sm[lane + 32] = a - lane;
  __syncwarp();
  double v = a + lane * 1e-3;
  long long t0, t1;
  const int N = 256;
  // 0: DFMA chain
  t0 = clock64();
  for (int i = 0; i < N; ++i) v = fma(v, 0.999999, 1e-7);
  t1 = clock64(); if (lane == 0) cyc[0] = (t1 - t0) / N;
  // 1: DADD chain
  t0 = clock64();
  for (int i = 0; i < N; ++i) v = v + 1e-9;
  t1 = clock64(); if (lane == 0) cyc[1] = (t1 - t0) / N;
  // 2: rcp_nr chain
  t0 = clock64();
  for (int i = 0; i < N; ++i) v = rcp_nr(v) + 1.0;
  t1 = clock64(); if (lane == 0) cyc[2] = (t1 - t0) / N;
  // 3: rsqrt_nr chain
  t0 = clock64();
  for (int i = 0; i < N; ++i) v = rsqrt_nr(v) + 1.0;
  t1 = clock64(); if (lane == 0) cyc[3] = (t1 - t0) / N;
  // 4: IEEE division chain
  t0 = clock64();
  for (int i = 0; i < N; ++i) v = 1.0 / v + 1.0;
  t1 = clock64(); if (lane == 0) cyc[4] = (t1 - t0) / N;
  // 5: sqrt chain
  t0 = clock64();
  for (int i = 0; i < N; ++i) v = sqrt(v) + 1.0;
  t1 = clock64(); if (lane == 0) cyc[5] = (t1 - t0) / N;
  // 6: shared load -> dependent (pointer chase through an index)
  int idx = lane;
  t0 = clock64();
  for (int i = 0; i < N; ++i) { const double w = sm[idx & 63]; idx = (int)w & 63; }
  t1 = clock64(); if (lane == 0) cyc[6] = (t1 - t0) / N;
  v += idx;
  // 7: shfl of a double, dependent
  t0 = clock64();
  for (int i = 0; i < N; ++i) v = __shfl_sync(0xffffffffu, v, (lane + 1) & 31) * 1.0000001;
  t1 = clock64(); if (lane == 0) cyc[7] = (t1 - t0) / N;
  // 8: store + syncwarp + load round trip
  t0 = clock64();
  for (int i = 0; i < N; ++i) { sm[lane] = v; __syncwarp(); v = sm[(lane + 1) & 31] * 1.0000001; __syncwarp(); }
  t1 = clock64(); if (lane == 0) cyc[8] = (t1 - t0) / N;
  // 9: DMUL chain
  t0 = clock64();
  for (int i = 0; i < N; ++i) v = v * 1.0000001;
  t1 = clock64(); if (lane == 0) cyc[9] = (t1 - t0) / N;
  out[lane] = v;
}
int main() {
  double* out; long long* cyc;
  cudaMalloc(&out, 64 * sizeof(double));
  cudaMallocManaged(&cyc, 16 * sizeof(long long));
  for (int r = 0; r < 3; ++r) {
    lat<<<1, 32>>>(out, cyc, 1.5);
    cudaDeviceSynchronize();
  }
  const char* nm[] = {"dfma", "dadd", "rcp_nr", "rsqrt_nr", "div", "sqrt", "lds_chase", "shfl_f64", "st_sync_ld", "dmul"};
  for (int i = 0; i < 10; ++i) printf("%-12s %lld cycles\n", nm[i], cyc[i]);
  return 0;
}
