// Probe: FP64 Schur update C -= P_I P_J^T emulated on the int8 tensor cores (tcgen05 kind::i8,
// Ozaki scheme: 8 balanced signed slices per row-scaled operand, the 36 slice products with
// s + t <= 9 accumulated exactly in int32 TMEM, one accumulator per s + t, reconstructed in
// FP64).  Standalone: checks the result against a CPU long-double reference and measures the
// throughput against the DMMA path's 35 TFLOP/s.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/ozaki_probe tools/ozaki_probe.cu
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s (line %d)\n", #x, cudaGetErrorString(e), __LINE__); exit(1); } } while (0)

constexpr int T = 128;
constexpr int S = 8;                    // slices per operand
constexpr int NG = S;                   // groups g = s + t = 2 .. S + 1
constexpr int BM = 128, BN = 64;        // CTA tile: 128 rows of C x 64 columns (half a C tile)
constexpr int KSTEP = 32;               // bytes of K per MMA
constexpr int STAGES = 4;
constexpr int A_STAGE = S * BM * KSTEP;  // 32 KB: 8 slices x 128 rows x 32 B
constexpr int B_STAGE = S * BN * KSTEP;  // 16 KB
constexpr int THREADS = 192;

__host__ __device__ __forceinline__ int perm8(int c) { return ((c & 3) << 1) | (c >> 2); }
__host__ __device__ __forceinline__ int elem(int r, int c) { return ((c >> 3) << 10) + (r << 3) + perm8(c & 7); }

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t n) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(n)); }
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t bytes) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory"); }
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile("{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W_%=;\n}\n" ::"r"(smem_u32(b)), "r"(parity) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) | ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46);
}
constexpr uint32_t IDESC = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);

// ---------------------------------------------------------------- slicing
// Panel P: rows tiles [0, rt) x K tiles [0, kt), octet-layout tiles, tile (i, p) at P + (i*kt + p)*T*T.
// Row exponent e_r: |P[r, :]| < 2^e_r.  Slices d_s (s = 1..8), x = P 2^-e = sum_s d_s 2^-7s + O(2^-56).
// A layout: [s][tile128][kstep][chunk][128 rows][16 B]; B layout: [s][tile64][kstep][chunk][64 rows][16 B].
__global__ void __launch_bounds__(256) slice_kernel(const double* __restrict__ P, int rt, int kt, int8_t* __restrict__ SA,
                                                    int8_t* __restrict__ SB, int* __restrict__ expo) {
  const int it = blockIdx.x;  // row tile
  const int K = kt * T, nks = K / KSTEP;
  __shared__ int se[T];
  __shared__ double smax[2][T];
  const int r = threadIdx.x & 127, half = threadIdx.x >> 7;
  double m = 0.0;
  for (int c16 = half; c16 < K / 16; c16 += 2) {
    const int k0 = c16 * 16, p = k0 / T, kc = k0 % T;
    const double* t = P + ((size_t)it * kt + p) * T * T;
#pragma unroll
    for (int u = 0; u < 16; ++u) m = fmax(m, fabs(t[elem(r, kc + u)]));
  }
  smax[half][r] = m;
  __syncthreads();
  if (half == 0) {
    const double mm = fmax(smax[0][r], smax[1][r]);
    se[r] = mm > 0.0 ? ilogb(mm) + 2 : 0;
    expo[it * T + r] = se[r];
  }
  __syncthreads();
  const int e = se[r];
  const int nT64 = rt * 2;
  for (int c16 = half; c16 < K / 16; c16 += 2) {
    const int k0 = c16 * 16, p = k0 / T, kc = k0 % T;
    const double* t = P + ((size_t)it * kt + p) * T * T;
    double x[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) x[u] = scalbn(t[elem(r, kc + u)], -e);
    const int ks = k0 / KSTEP, ch = (k0 % KSTEP) / 16;
    for (int s = 0; s < S; ++s) {
      int8_t d[16];
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        const double y = x[u] * 128.0;
        const double q = rint(y);
        d[u] = (int8_t)q;
        x[u] = y - q;
      }
      const uint4 v = *reinterpret_cast<const uint4*>(d);
      // A: 128-row tile it
      *reinterpret_cast<uint4*>(SA + ((((size_t)s * rt + it) * nks + ks) * 2 + ch) * (BM * 16) + (size_t)r * 16) = v;
      // B: 64-row tile (2 it + r / 64)
      const int t64 = it * 2 + (r >> 6), r64 = r & 63;
      *reinterpret_cast<uint4*>(SB + ((((size_t)s * nT64 + t64) * nks + ks) * 2 + ch) * (BN * 16) + (size_t)r64 * 16) = v;
    }
  }
}

// ---------------------------------------------------------------- Ozaki Schur update, N = 128, two passes
// CTA b: full C tile (I, J) (lower triangle).  Pass 0: groups g = 2..5 (10 products, slices
// 1..4); pass 1: g = 6..9 (26 products, slices 1..8); 4 TMEM accumulators x 128 columns.
constexpr int BN2 = 128;
constexpr int STAGE2 = 2 * S * BM * KSTEP;  // 64 KB (A and B, all 8 slices)
constexpr int STAGES2 = 3;
constexpr int THREADS2 = 320;               // producer, MMA, 8 epilogue warps
constexpr uint32_t IDESC2 = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BN2 >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);

__global__ void __launch_bounds__(THREADS2, 1) ozaki2_kernel(const int8_t* __restrict__ SA, const int* __restrict__ expo,
                                                             double* __restrict__ C, int rt, int kt) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + STAGES2 * STAGE2);
  uint64_t* empty = full + STAGES2;
  uint64_t* done = empty + STAGES2;     // [2]
  uint64_t* drained = done + 2;         // [1]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(drained + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int K = kt * T, nks = K / KSTEP;
  int b = blockIdx.x, J = 0;
  while (b >= rt - J) { b -= rt - J; ++J; }
  const int I = J + b;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES2; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    mbar_init(&done[0], 1); mbar_init(&done[1], 1); mbar_init(drained, 8 * 32);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)), "n"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *tmem_slot;
  if (warp == 0 && lane == 0) {
    int it = 0;
    for (int pass = 0; pass < 2; ++pass) {
      const int ns = pass == 0 ? 4 : S;
      for (int ks = 0; ks < nks; ++ks, ++it) {
        const int st = it % STAGES2;
        if (it >= STAGES2) mbar_wait(&empty[st], ((it / STAGES2) - 1) & 1);
        mbar_expect(&full[st], 2 * ns * BM * KSTEP);
        uint8_t* base = sm + st * STAGE2;
        for (int s = 0; s < ns; ++s) {
          bulk_g2s(base + s * (BM * KSTEP), SA + (((size_t)s * rt + I) * nks + ks) * (BM * KSTEP), BM * KSTEP, &full[st]);
          bulk_g2s(base + (S + s) * (BM * KSTEP), SA + (((size_t)s * rt + J) * nks + ks) * (BM * KSTEP), BM * KSTEP, &full[st]);
        }
      }
    }
  } else if (warp == 1 && lane == 0) {
    int it = 0;
    for (int pass = 0; pass < 2; ++pass) {
      if (pass == 1) {  // the accumulators must be drained first
        mbar_wait(drained, 0);
        asm volatile("tcgen05.fence::after_thread_sync;");
      }
      const int g0 = pass == 0 ? 2 : 6;
      for (int ks = 0; ks < nks; ++ks, ++it) {
        const int st = it % STAGES2;
        mbar_wait(&full[st], (it / STAGES2) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;");
        const uint32_t base = smem_u32(sm + st * STAGE2);
#pragma unroll
        for (int gg = 0; gg < 4; ++gg) {
          const int g = g0 + gg;
          const int s_first = g - S > 1 ? g - S : 1;
#pragma unroll
          for (int s = 1; s <= S; ++s) {
            const int t = g - s;
            if (t < 1 || t > S) continue;
            const uint64_t da = sdesc(base + (s - 1) * (BM * KSTEP), BM * 16, 8 * 16);
            const uint64_t db = sdesc(base + (S + t - 1) * (BM * KSTEP), BM * 16, 8 * 16);
            const uint32_t acc = (ks > 0 || s > s_first) ? 1u : 0u;
            asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                         "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n"
                         ::"r"(tmem + (uint32_t)(gg * BN2)), "l"(da), "l"(db), "r"(IDESC2), "r"(acc));
          }
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&empty[st])) : "memory");
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&done[pass])) : "memory");
    }
  } else if (warp >= 2) {
    const int q = warp & 3, hh = (warp - 2) >> 2;  // TMEM lane quadrant, column half
    const int r = q * 32 + lane;
    const int ei = expo[I * T + r];
    double* Ct = C + ((size_t)I * rt + J) * T * T;
    for (int pass = 0; pass < 2; ++pass) {
      mbar_wait(&done[pass], 0);
      asm volatile("tcgen05.fence::after_thread_sync;");
      const int g0 = pass == 0 ? 2 : 6;
      double part[2][32];
#pragma unroll
      for (int ch = 0; ch < 2; ++ch) {
#pragma unroll
        for (int j = 0; j < 32; ++j) part[ch][j] = 0.0;
        for (int gg = 3; gg >= 0; --gg) {  // smallest contributions first
          const double w = ldexp(1.0, -7 * (g0 + gg));
          uint32_t v[32];
          const uint32_t taddr = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(gg * BN2 + 64 * hh + 32 * ch);
          asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                       "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                       : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                         "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
                         "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
                         "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
                       : "r"(taddr));
          asm volatile("tcgen05.wait::ld.sync.aligned;");
#pragma unroll
          for (int j = 0; j < 32; ++j) part[ch][j] = fma((double)(int32_t)v[j], w, part[ch][j]);
        }
      }
      if (pass == 0) {  // TMEM read: pass 1 may overwrite the accumulators while C is updated
        asm volatile("tcgen05.fence::before_thread_sync;");
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(drained)) : "memory");
      }
#pragma unroll
      for (int ch = 0; ch < 2; ++ch)
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const int col = 64 * hh + 32 * ch + j;
          const int o = elem(r, col);
          Ct[o] = Ct[o] - ldexp(part[ch][j], ei + expo[J * T + col]);
        }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp == 2) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(512));
}

int main(int argc, char** argv) {
  const int rt = argc > 1 ? atoi(argv[1]) : 4, kt = argc > 2 ? atoi(argv[2]) : 16;
  const int n = rt * T, K = kt * T;
  std::mt19937_64 rng(7);
  std::normal_distribution<double> nd;
  // panel rows with mixed magnitudes (per-row scale 2^[-20, 20] and per-column decay)
  std::vector<double> p((size_t)n * K);
  for (int r = 0; r < n; ++r) {
    const double rs = ldexp(1.0, (int)(rng() % 41) - 20);
    for (int k = 0; k < K; ++k) p[(size_t)r * K + k] = nd(rng) * rs * (1.0 + 0.5 * std::sin(0.01 * k));
  }
  std::vector<double> ptiles((size_t)n * K);
  for (int r = 0; r < n; ++r)
    for (int k = 0; k < K; ++k) {
      const int i = r / T, pp = k / T;
      ptiles[((size_t)i * kt + pp) * T * T + elem(r % T, k % T)] = p[(size_t)r * K + k];
    }
  double *dP, *dC;
  int8_t *dA, *dB;
  int* dE;
  CK(cudaMalloc(&dP, ptiles.size() * 8));
  CK(cudaMalloc(&dC, (size_t)rt * rt * T * T * 8));
  CK(cudaMalloc(&dA, (size_t)S * n * K));
  CK(cudaMalloc(&dB, (size_t)S * n * K));
  CK(cudaMalloc(&dE, n * 4));
  CK(cudaMemcpy(dP, ptiles.data(), ptiles.size() * 8, cudaMemcpyHostToDevice));
  CK(cudaMemset(dC, 0, (size_t)rt * rt * T * T * 8));
  const size_t smem = STAGES2 * STAGE2 + (2 * STAGES2 + 3) * 8 + 16;
  CK(cudaFuncSetAttribute(ozaki2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int ntile = rt * (rt + 1) / 2;
  slice_kernel<<<rt, 256>>>(dP, rt, kt, dA, dB, dE);
  ozaki2_kernel<<<ntile, THREADS2, smem>>>(dA, dE, dC, rt, kt);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  std::vector<double> c((size_t)rt * rt * T * T);
  CK(cudaMemcpy(c.data(), dC, c.size() * 8, cudaMemcpyDeviceToHost));
  // check a sample of entries against long double
  double worst = 0, worst_dgemm_bound = 0;
  for (int trial = 0; trial < 4000; ++trial) {
    const int i = rng() % n, j = rng() % (i + 1);
    long double ref = 0, absdot = 0;
    for (int k = 0; k < K; ++k) {
      ref += (long double)p[(size_t)i * K + k] * p[(size_t)j * K + k];
      absdot += fabsl((long double)p[(size_t)i * K + k] * p[(size_t)j * K + k]);
    }
    const double got = -c[((size_t)(i / T) * rt + j / T) * T * T + elem(i % T, j % T)];
    const double err = fabs((double)((long double)got - ref)) / (double)absdot;
    worst = fmax(worst, err);
  }
  printf("n=%d K=%d: max |ozaki - exact| / sum|a b| over 4000 entries = %.3e (u = 1.1e-16)\n", n, K, worst);
  if (argc > 3) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int reps = 5;
    cudaEventRecord(e0);
    for (int r = 0; r < reps; ++r) ozaki2_kernel<<<ntile, THREADS2, smem>>>(dA, dE, dC, rt, kt);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double flops = 2.0 * T * T * K * (double)ntile;  // FP64-equivalent
    printf("ozaki update: %d tiles, %.3f ms/launch, %.1f FP64-equivalent TFLOP/s, %.1f int8 TOPS\n", ntile, ms / reps,
           flops / (ms / reps * 1e-3) / 1e12, flops * 36 / (ms / reps * 1e-3) / 1e12);
    cudaEventRecord(e0);
    for (int r = 0; r < reps; ++r) slice_kernel<<<rt, 256>>>(dP, rt, kt, dA, dB, dE);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    printf("slicing: %.3f ms/launch (%.1f GB/s of panel)\n", ms / reps, (double)n * K * 8 / (ms / reps * 1e-3) / 1e9);
  }
  return 0;
}
