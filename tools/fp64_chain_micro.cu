// Per-term cost of the pending-term chain variants (v = fl(v - fl(a*b)) in order).
#include <cstdio>
template <int V>
__global__ void __launch_bounds__(256, 1) kern(double* out, long long* cyc, int reps) {
  __shared__ double sb[64];
  if (threadIdx.x < 64) sb[threadIdx.x] = 1.0 + threadIdx.x * 1e-3;
  __syncthreads();
  double a[32], b[32], p[32];
#pragma unroll
  for (int q = 0; q < 32; ++q) { a[q] = out[q] + threadIdx.x; b[q] = out[32 + q] * 0.5; p[q] = a[q] * b[q]; }
  double v = out[64 + threadIdx.x];
  double s = v;
#pragma unroll
  for (int q = 0; q < 32; ++q) s += a[q] + b[q] + p[q];
  if (s == 1234.5) out[0] = s;
  __syncwarp();
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
#pragma unroll
    for (int q = 0; q < 32; ++q) {
      if (V == 1) v = __dsub_rn(v, p[q]);
      if (V == 2) v = __dsub_rn(v, __dmul_rn(a[q], b[q]));
      if (V == 3) v = __dsub_rn(v, __dmul_rn(a[q], sb[q]));
      if (V == 4) v = fma(-a[q], b[q], v);
    }
  }
  __syncwarp();
  long long t1 = clock64();
  out[1024 + blockIdx.x * 256 + threadIdx.x] = v;
  if ((threadIdx.x & 31) == 0) atomicMax((unsigned long long*)cyc, (unsigned long long)(t1 - t0));
}
int main() {
  double* out; long long* cyc;
  cudaMalloc(&out, (1024 + 16 * 256) * 8); cudaMemset(out, 0, (1024 + 16 * 256) * 8);
  cudaMallocManaged(&cyc, 8);
  const int reps = 64;
  for (int thr : {32, 64, 256}) {
    void (*ks[4])(double*, long long*, int) = {kern<1>, kern<2>, kern<3>, kern<4>};
    const char* nm[4] = {"DADD chain (products in regs)", "DMUL+DADD (regs)", "DMUL+DADD (b from smem)", "DFMA chain"};
    for (int v = 0; v < 4; ++v) {
      for (int rep = 0; rep < 2; ++rep) { *cyc = 0; ks[v]<<<16, thr>>>(out, cyc, reps); cudaDeviceSynchronize(); }
      printf("threads %3d  %-30s %.1f cycles/term\n", thr, nm[v], *cyc / (32.0 * reps));
    }
  }
  return 0;
}
