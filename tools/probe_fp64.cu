// FP64 throughput probe for B200 (sm_100a): DMMA (mma.sync m8n8k4 f64) vs DFMA.
// Off the hot path: calibrates the FP64 roofline denominator.
#include <cstdio>
#include <cuda_runtime.h>

template <int CHAINS>
__global__ void dmma_loop(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[CHAINS][2];
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) { c[i][0] = 0.0; c[i][1] = 0.0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.0) out[threadIdx.x] = s;
}

template <int CHAINS>
__global__ void dfma_loop(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[CHAINS];
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) c[i] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) c[i] = fma(a, c[i], b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) s += c[i];
  if (s == 12345.0) out[threadIdx.x] = s;
}

int main() {
  double* out; cudaMalloc(&out, 4096 * sizeof(double));
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("SMs %d clock(kHz) %d\n", sms, clk);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 20000;
  for (int bpsm = 1; bpsm <= 4; bpsm *= 2) {
    for (int threads = 128; threads <= 512; threads *= 2) {
      int grid = sms * bpsm;
      dmma_loop<16><<<grid, threads>>>(out, 100);
      cudaEventRecord(e0);
      dmma_loop<16><<<grid, threads>>>(out, iters);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double flops = (double)grid * (threads / 32) * iters * 16 * 512.0;
      printf("DMMA m8n8k4 grid=%d threads=%d : %.2f TFLOP/s\n", grid, threads, flops / ms / 1e9);
      dfma_loop<16><<<grid, threads>>>(out, 100);
      cudaEventRecord(e0);
      dfma_loop<16><<<grid, threads>>>(out, iters);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      flops = (double)grid * threads * iters * 16 * 2.0;
      printf("DFMA        grid=%d threads=%d : %.2f TFLOP/s\n", grid, threads, flops / ms / 1e9);
    }
  }
  cudaError_t err = cudaGetLastError();
  printf("err: %s\n", cudaGetErrorString(err));
  return 0;
}
