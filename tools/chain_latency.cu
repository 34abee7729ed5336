// Dependent-chain latencies that bound a one-warp banded sweep step
// (level-1 sweeps, banded.cu): DFMA, SHFL, SHFL+DFMA, SHFL+DMUL+DFMA, LDS+DFMA.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/chain_latency tools/chain_latency.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int N = 4096;

__global__ void k(double* out, long long* cyc, double a, double b) {
  __shared__ double sm[64];
  const int lane = threadIdx.x;
  sm[lane] = a;
  sm[lane + 32] = b;
  __syncwarp();
  double x = a + lane;
  long long t0, t1;
  // 0: DFMA chain
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) x = fma(x, b, a);
  t1 = clock64();
  if (lane == 0) cyc[0] = t1 - t0;
  // 1: SHFL chain (64-bit = 2 SHFL in parallel)
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) x = __shfl_sync(0xffffffffu, x, (i + 1) & 31);
  t1 = clock64();
  if (lane == 0) cyc[1] = t1 - t0;
  // 2: SHFL + DFMA
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) {
    const double w = __shfl_sync(0xffffffffu, x, (i + 1) & 31);
    x = fma(-b, w, x);
  }
  t1 = clock64();
  if (lane == 0) cyc[2] = t1 - t0;
  // 3: DMUL + SHFL + DFMA
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) {
    const double w = __shfl_sync(0xffffffffu, x * a, (i + 1) & 31);
    x = fma(-b, w, x);
  }
  t1 = clock64();
  if (lane == 0) cyc[3] = t1 - t0;
  // 4: LDS (address from the chain) + DFMA
  int idx = lane;
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) {
    const double m = sm[idx & 63];
    x = fma(m, b, x);
    idx = (int)(__double_as_longlong(x) & 31);
  }
  t1 = clock64();
  if (lane == 0) cyc[4] = t1 - t0;
  // 5: SHFL.32 chain
  int y = lane;
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) y = __shfl_sync(0xffffffffu, y, (y + 1) & 31);
  t1 = clock64();
  if (lane == 0) cyc[5] = t1 - t0;
  // 6: 4 independent DFMA per step + SHFL chain (a sweep step's FMA group)
  double c0 = x, c1 = x + 1, c2 = x + 2, c3 = x + 3;
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) {
    const double w = __shfl_sync(0xffffffffu, c0, (i + 1) & 31);
    c0 = fma(-b, w, c0);
    c1 = fma(-a, w, c1);
    c2 = fma(-b, w, c2);
    c3 = fma(-a, w, c3);
  }
  t1 = clock64();
  if (lane == 0) cyc[6] = t1 - t0;
  out[lane] = x + y + c0 + c1 + c2 + c3;
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 32 * sizeof(double));
  cudaMallocManaged(&cyc, 8 * sizeof(long long));
  for (int rep = 0; rep < 2; ++rep) {
    k<<<1, 32>>>(out, cyc, 1.0000001, 0.9999999);
    cudaDeviceSynchronize();
  }
  const char* names[] = {"DFMA", "SHFL.64", "SHFL+DFMA", "DMUL+SHFL+DFMA", "LDS+DFMA+cvt", "SHFL.32", "SHFL+4DFMA"};
  printf("{");
  for (int i = 0; i < 7; ++i) printf("\"%s\": %.1f%s", names[i], (double)cyc[i] / N, i < 6 ? ", " : "");
  printf("}\n");
  return 0;
}
