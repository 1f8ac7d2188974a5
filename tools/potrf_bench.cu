// Times potrf_inv_kernel phases on one 128x128 SPD tile (dbg bits skip phases).
#include "../paper_2503_04424_b200/csrc/kernels.cu"
#include <cstdio>
#include <vector>
using namespace b2d;
int main() {
  std::vector<double> h(TILE_ELEMS);
  for (int r = 0; r < T; ++r) for (int c = 0; c < T; ++c) h[elem(r, c)] = (r == c ? 200.0 : 1.0 / (1 + r + c));
  double *t, *inv, *ell, *dg; unsigned long long* f;
  cudaMalloc(&t, TILE_BYTES); cudaMalloc(&inv, TILE_BYTES); cudaMalloc(&ell, 1024); cudaMalloc(&dg, 1024); cudaMalloc(&f, 8);
  cudaFuncSetAttribute(potrf_inv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, POTRF_SMEM);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int cases[] = {0};
  for (int dbg : cases) {
    cudaMemcpy(t, h.data(), TILE_BYTES, cudaMemcpyHostToDevice);
    potrf_inv_kernel<<<1, POTRF_THREADS, POTRF_SMEM>>>(t, inv, ell, dg, f, 0, T);
    cudaEventRecord(e0);
    for (int i = 0; i < 20; ++i) {
      potrf_inv_kernel<<<1, POTRF_THREADS, POTRF_SMEM>>>(t, inv, ell, dg, f, 0, T);
    }
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("dbg=%2d (skip A1:%d A2:%d A3:%d B:%d)  %.1f us\n", dbg, dbg & 1, !!(dbg & 2), !!(dbg & 4), !!(dbg & 8), ms * 1000 / 20);
  }
  long long* pr; cudaMalloc(&pr, 16 * 8); cudaMemset(pr, 0, 128);
  cudaMemcpy(t, h.data(), TILE_BYTES, cudaMemcpyHostToDevice);
  potrf_inv_kernel<<<1, POTRF_THREADS, POTRF_SMEM>>>(t, inv, ell, dg, f, 0, T, pr);
  long long hp[16]; cudaMemcpy(hp, pr, 128, cudaMemcpyDeviceToHost);
  const char* names[] = {"start", "loaded", "diag0", "A2(c0=0)", "A3 diag upd", "diag8", "A3(c0=0) end", "phaseA", "phaseB", "stored"};
  for (int i = 1; i < 10; ++i) printf("%-14s %8lld cycles (cum %8lld)\n", names[i], hp[i] - hp[i - 1], hp[i] - hp[0]);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
