// Dependent-chain latency of FP64 instructions on one warp (clock64), and throughput with 8 warps.
#include <cstdio>
__global__ void lat(double* out, long long* cyc, double a, double b, int n) {
  double x = a, y = b;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    x = __dsub_rn(x, y);
    x = __dsub_rn(x, y);
    x = __dsub_rn(x, y);
    x = __dsub_rn(x, y);
  }
  long long t1 = clock64();
  double z = x;
  for (int i = 0; i < n; ++i) {
    z = __dmul_rn(z, b);
    z = __dmul_rn(z, b);
    z = __dmul_rn(z, b);
    z = __dmul_rn(z, b);
  }
  long long t2 = clock64();
  double f = z;
  for (int i = 0; i < n; ++i) {
    f = fma(f, a, b);
    f = fma(f, a, b);
    f = fma(f, a, b);
    f = fma(f, a, b);
  }
  long long t3 = clock64();
  float s = (float)f;
  for (int i = 0; i < n; ++i) {
    s = __fsub_rn(s, (float)b);
    s = __fsub_rn(s, (float)b);
    s = __fsub_rn(s, (float)b);
    s = __fsub_rn(s, (float)b);
  }
  long long t4 = clock64();
  if (threadIdx.x == 0) {
    cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3;
  }
  out[threadIdx.x] = f + s;
}
int main() {
  double* out; long long* cyc;
  cudaMalloc(&out, 1024 * 8); cudaMallocManaged(&cyc, 64);
  const int n = 4096;
  for (int w : {1, 2, 8, 32}) {
    lat<<<1, 32 * w>>>(out, cyc, 1.0000001, 1e-9, n);
    cudaDeviceSynchronize();
    lat<<<1, 32 * w>>>(out, cyc, 1.0000001, 1e-9, n);
    cudaDeviceSynchronize();
    printf("warps %2d: cycles per dependent op: DADD %.1f  DMUL %.1f  DFMA %.1f  FADD %.1f\n", w, cyc[0] / (4.0 * n),
           cyc[1] / (4.0 * n), cyc[2] / (4.0 * n), cyc[3] / (4.0 * n));
  }
  return 0;
}
