// Probe: tcgen05 kind::i8 GEMM on sm_100a (standalone; not part of the engine).
// C[M x N] (int32) = A[M x K] (int8) * B[N x K]^T, K-major operands in the UMMA canonical
// SWIZZLE_NONE layout staged by cp.async.bulk, accumulators in TMEM.  Checks exactness against
// the CPU and measures throughput.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/imma_probe tools/imma_probe.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s (line %d)\n", #x, cudaGetErrorString(e), __LINE__); exit(1); } } while (0)

constexpr int BM = 128, BN = 64;       // CTA tile (one tcgen05.mma M=128 N=64)
constexpr int KC = 16;                  // bytes per K chunk (one core-matrix row)
constexpr int KSTAGE = 128;             // bytes of K per pipeline stage
constexpr int CHUNKS = KSTAGE / KC;     // 8
constexpr int STAGES = 6;
constexpr int A_STAGE = BM * KSTAGE;    // 16 KB
constexpr int B_STAGE = BN * KSTAGE;    // 8 KB
constexpr int THREADS = 192;            // warp 0 producer, warp 1 MMA, warps 2-5 epilogue

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(n));
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile("{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W_%=;\n}\n"
               ::"r"(smem_u32(b)), "r"(parity) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
// SWIZZLE_NONE K-major smem descriptor: start, LBO (next 16-byte K chunk), SBO (next 8-row group)
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // version (Blackwell)
  return d;                // base offset 0, lbo mode 0, layout SWIZZLE_NONE (0)
}
// kind::i8 instruction descriptor: D s32, A/B signed, K-major, N = BN, M = BM
constexpr uint32_t IDESC = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);

__global__ void __launch_bounds__(THREADS, 1) imma_kernel(const int8_t* __restrict__ A, const int8_t* __restrict__ B,
                                                          int32_t* __restrict__ C, int M, int N, int K) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* sA = sm;
  uint8_t* sB = sm + STAGES * A_STAGE;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + STAGES * B_STAGE);
  uint64_t* empty = full + STAGES;
  uint64_t* done = empty + STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int mt = blockIdx.x % (M / BM), nt = blockIdx.x / (M / BM);
  const int nst = K / KSTAGE;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    mbar_init(done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)), "n"(64));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *tmem_slot;
  // global operand layout: [tile][K chunk][rows][16 B]; a stage is CHUNKS consecutive chunks
  const int8_t* gA = A + (size_t)mt * BM * K;
  const int8_t* gB = B + (size_t)nt * BN * K;
  if (warp == 0 && lane == 0) {
    for (int st = 0; st < nst; ++st) {
      const int s = st % STAGES;
      if (st >= STAGES) mbar_wait(&empty[s], ((st / STAGES) - 1) & 1);
      mbar_expect(&full[s], A_STAGE + B_STAGE);
      bulk_g2s(sA + s * A_STAGE, gA + (size_t)st * A_STAGE, A_STAGE, &full[s]);
      bulk_g2s(sB + s * B_STAGE, gB + (size_t)st * B_STAGE, B_STAGE, &full[s]);
    }
  } else if (warp == 1 && lane == 0) {
    for (int st = 0; st < nst; ++st) {
      const int s = st % STAGES;
      mbar_wait(&full[s], (st / STAGES) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;");
      const uint32_t a0 = smem_u32(sA + s * A_STAGE), b0 = smem_u32(sB + s * B_STAGE);
#pragma unroll
      for (int j = 0; j < CHUNKS / 2; ++j) {  // one MMA per 32 bytes of K (2 chunks)
        const uint64_t da = sdesc(a0 + j * 2 * BM * KC, BM * KC, 8 * KC);
        const uint64_t db = sdesc(b0 + j * 2 * BN * KC, BN * KC, 8 * KC);
        const uint32_t acc = (st > 0 || j > 0) ? 1u : 0u;
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                     "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n"
                     ::"r"(tmem), "l"(da), "l"(db), "r"(IDESC), "r"(acc));
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                   ::"r"(smem_u32(&empty[s])) : "memory");
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                 ::"r"(smem_u32(done)) : "memory");
  } else if (warp >= 2) {
    mbar_wait(done, 0);
    asm volatile("tcgen05.fence::after_thread_sync;");
    const int q = warp & 3;  // lanes 32q .. 32q+31 of TMEM
    const int row = mt * BM + q * 32 + lane;
    for (int c0 = 0; c0 < BN; c0 += 32) {
      uint32_t v[32];
      const uint32_t taddr = tmem + ((uint32_t)(q * 32) << 16) + c0;
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                   "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                   : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                     "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
                     "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
                     "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
                   : "r"(taddr));
      asm volatile("tcgen05.wait::ld.sync.aligned;");
      for (int j = 0; j < 32; ++j) C[(size_t)row * N + nt * BN + c0 + j] = (int32_t)v[j];
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp == 2) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(64));
}

// host: row-major int8 X[rows][K] -> [tile][K chunk][rows_in_tile][16 B]
static std::vector<int8_t> to_umma(const std::vector<int8_t>& x, int rows, int K, int tile) {
  std::vector<int8_t> y(x.size());
  for (int r = 0; r < rows; ++r)
    for (int k = 0; k < K; ++k) {
      const int t = r / tile, rr = r % tile, c = k / KC, b = k % KC;
      y[(size_t)t * tile * K + (size_t)c * tile * KC + rr * KC + b] = x[(size_t)r * K + k];
    }
  return y;
}

int main(int argc, char** argv) {
  const size_t smem = STAGES * (A_STAGE + B_STAGE) + (2 * STAGES + 1) * 8 + 16;
  CK(cudaFuncSetAttribute(imma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  for (int pass = 0; pass < 2; ++pass) {
    const int M = pass == 0 ? 256 : 148 * 8 * BM / 8 * 2, N = pass == 0 ? 128 : 2048, K = pass == 0 ? 1024 : 4096;
    std::vector<int8_t> a((size_t)M * K), b((size_t)N * K);
    uint32_t s = 12345;
    for (auto& v : a) { s = s * 1664525u + 1013904223u; v = (int8_t)((s >> 24) & 0xff); }
    for (auto& v : b) { s = s * 1664525u + 1013904223u; v = (int8_t)((s >> 24) & 0xff); }
    auto ua = to_umma(a, M, K, BM), ub = to_umma(b, N, K, BN);
    int8_t *dA, *dB;
    int32_t* dC;
    CK(cudaMalloc(&dA, a.size()));
    CK(cudaMalloc(&dB, b.size()));
    CK(cudaMalloc(&dC, (size_t)M * N * 4));
    CK(cudaMemcpy(dA, ua.data(), a.size(), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dB, ub.data(), b.size(), cudaMemcpyHostToDevice));
    const int grid = (M / BM) * (N / BN);
    imma_kernel<<<grid, THREADS, smem>>>(dA, dB, dC, M, N, K);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    if (pass == 0) {
      std::vector<int32_t> c((size_t)M * N);
      CK(cudaMemcpy(c.data(), dC, c.size() * 4, cudaMemcpyDeviceToHost));
      long bad = 0;
      for (int i = 0; i < M; ++i)
        for (int j = 0; j < N; ++j) {
          int64_t ref = 0;
          for (int k = 0; k < K; ++k) ref += (int32_t)a[(size_t)i * K + k] * (int32_t)b[(size_t)j * K + k];
          if (ref != c[(size_t)i * N + j] && bad++ < 5)
            printf("mismatch (%d,%d): %d vs %lld\n", i, j, c[(size_t)i * N + j], (long long)ref);
        }
      printf("exactness M=%d N=%d K=%d: %ld mismatches\n", M, N, K, bad);
    } else {
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      cudaEventRecord(e0);
      const int reps = 10;
      for (int r = 0; r < reps; ++r) imma_kernel<<<grid, THREADS, smem>>>(dA, dB, dC, M, N, K);
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      const double ops = 2.0 * M * N * K * reps;
      printf("throughput M=%d N=%d K=%d grid=%d: %.3f ms/launch, %.1f TOPS (int8)\n", M, N, K, grid, ms / reps,
             ops / (ms * 1e-3) / 1e12);
    }
    cudaFree(dA);
    cudaFree(dB);
    cudaFree(dC);
  }
  return 0;
}
