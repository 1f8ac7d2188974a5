// Per-phase cycle counts of ldl_panel_cluster_kernel (built with -DLDL_PROF): one n x n block
// (random symmetric, strong diagonal so every step pivots) factored panel by panel exactly as
// ooc_ldl_factor does; prints the cycles per step of each phase (CTA 0, thread 0) and the
// panel / bulk kernel times.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DLDL_PROF -o tools/ldl_prof tools/ldl_prof.cu
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>
#include <random>
#include <cmath>
#include "../paper_2503_04424_b200/csrc/ldl.cu"

using namespace b2d;

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

int main(int argc, char** argv) {
  const int64_t n = argc > 1 ? atoll(argv[1]) : 4096, ld = n;
  std::vector<double> h((size_t)n * n);
  std::mt19937_64 rng(1);
  std::normal_distribution<double> nd;
  for (int64_t j = 0; j < n; ++j)
    for (int64_t i = j; i < n; ++i) h[j * ld + i] = h[i * ld + j] = nd(rng) * (i == j ? 100.0 : 1.0);
  double amax = 0;
  for (double v : h) amax = fmax(amax, fabs(v));
  double *A, *C, *W, *diag, *col, *d;
  uint8_t* tag;
  int64_t* swaps;
  unsigned long long *fail, *amax_bits;
  CK(cudaMalloc(&A, n * n * 8));
  CK(cudaMalloc(&tag, n * n));
  CK(cudaMalloc(&C, LDL_NB * ld * 8));
  CK(cudaMalloc(&W, LDL_NB * ld * 8));
  CK(cudaMalloc(&diag, n * 8));
  CK(cudaMalloc(&col, n * 8));
  CK(cudaMalloc(&d, n * 8));
  CK(cudaMalloc(&swaps, n * 8));
  CK(cudaMalloc(&fail, 8));
  CK(cudaMalloc(&amax_bits, 8));
  unsigned long long ab;
  memcpy(&ab, &amax, 8);
  CK(cudaMemcpy(amax_bits, &ab, 8, cudaMemcpyHostToDevice));
  CK(cudaFuncSetAttribute(ldl_panel_cluster_kernel<false>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  const size_t smem = ldl_cluster_smem((int)((n + LC - 1) / LC));
  CK(cudaFuncSetAttribute(ldl_panel_cluster_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const LdlArgs g{A, tag, C, W, diag, col, d, swaps, fail, amax_bits, ld, n, 0};
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int rep = 0; rep < 2; ++rep) {
    CK(cudaMemcpy(A, h.data(), n * n * 8, cudaMemcpyHostToDevice));
    CK(cudaMemset(tag, 0, n * n));
    CK(cudaMemset(fail, 0xff, 8));
    long long zero[16] = {0};
    CK(cudaMemcpyToSymbol(ldl_prof, zero, sizeof(zero)));
    ldl_diag_init_kernel<<<(unsigned)((n + 255) / 256), 256>>>(g);
    float tp = 0, tb = 0, ts = 0;
    for (int64_t r0 = 0; r0 < n; r0 += LDL_NB) {
      const int nbk = (int)std::min<int64_t>(LDL_NB, n - r0);
      cudaLaunchConfig_t cfg = {};
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = LC;
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      cfg.gridDim = dim3(LC);
      cfg.blockDim = dim3(LC_THREADS);
      cfg.dynamicSmemBytes = smem;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      cudaEventRecord(e0);
      CK(cudaLaunchKernelEx(&cfg, ldl_panel_cluster_kernel<false>, g, r0, nbk, (unsigned*)nullptr, 0u, (double*)nullptr));
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      tp += ms;
      const int64_t mt = (n - r0 - nbk + LDL_BT - 1) / LDL_BT, ntile = mt * (mt + 1) / 2;
      const int64_t nswap = r0 > 0 ? std::min<int64_t>(148, (r0 + 63) / 64) : 0;
      cudaEventRecord(e0);
      if (ntile + nswap > 0) ldl_bulk_kernel<<<(unsigned)(ntile + nswap), 256>>>(g, r0, nbk, ntile, (unsigned*)nullptr, 0u);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      tb += ms;
    }
    CK(cudaDeviceSynchronize());
    unsigned long long f;
    CK(cudaMemcpy(&f, fail, 8, cudaMemcpyDeviceToHost));
    long long prof[16];
    CK(cudaMemcpyFromSymbol(prof, ldl_prof, sizeof(prof)));
    std::vector<double> dd(n);
    CK(cudaMemcpy(dd.data(), d, n * 8, cudaMemcpyDeviceToHost));
    double ld_sum = 0;
    for (double v : dd) ld_sum += log(fabs(v));
    printf("n=%lld fail=%llx panel %.2f ms (%.2f us/step) store %.2f ms bulk %.2f ms  logabsdet %.10e\n", (long long)n,
           f, tp, tp * 1e3 / n, ts, tb, ld_sum);
    const char* names[6] = {"loop top", "cand push", "cluster sync", "reduce+push", "row wait", "row loop"};
    long long tot = 0;
    for (int i = 0; i < 6; ++i) tot += prof[i];
    for (int i = 0; i < 6; ++i) printf("  %-14s %8.0f cyc/step\n", names[i], (double)prof[i] / n);
    printf("  total          %8.0f cyc/step\n", (double)tot / n);
  }
  // the one-launch cluster factor
  CK(cudaFuncSetAttribute(ldl_factor_cluster_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  const size_t fsm = ldl_factor_smem((int)((n + LC - 1) / LC));
  CK(cudaFuncSetAttribute(ldl_factor_cluster_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fsm));
  for (int rep = 0; rep < 2; ++rep) {
    CK(cudaMemcpy(A, h.data(), n * n * 8, cudaMemcpyHostToDevice));
    CK(cudaMemset(tag, 0, n * n));
    CK(cudaMemset(fail, 0xff, 8));
    long long zero[16] = {0};
    CK(cudaMemcpyToSymbol(ldl_prof, zero, sizeof(zero)));
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = LC;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3(LC);
    cfg.blockDim = dim3(LC_THREADS);
    cfg.dynamicSmemBytes = fsm;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaEventRecord(e0);
    CK(cudaLaunchKernelEx(&cfg, ldl_factor_cluster_kernel, g));
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    long long prof[16];
    CK(cudaMemcpyFromSymbol(prof, ldl_prof, sizeof(prof)));
    std::vector<double> dd(n);
    CK(cudaMemcpy(dd.data(), d, n * 8, cudaMemcpyDeviceToHost));
    double ld_sum = 0;
    for (double v : dd) ld_sum += log(fabs(v));
    printf("one-launch factor n=%lld: %.2f ms  logabsdet %.10e\n", (long long)n, ms, ld_sum);
    const char* fn[5] = {"panel steps", "writeback+sync", "store/swap", "bulk", "sync"};
    for (int i = 0; i < 5; ++i) printf("  %-16s %8.2f ms (CTA 0 @1.9GHz)\n", fn[i], prof[9 + i] / 1.9e6);
  }
  return 0;
}
