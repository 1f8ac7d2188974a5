// FP64 Schur update on the int8 tensor cores (tcgen05 kind::i8), Ozaki scheme.
//
// The trailing update C(i, j) -= sum_p L(i, p) L(j, p)^T of one outer panel (K = 128 W) is
// the dominant kernel.  sm_100a has no FP64 tcgen05 kind; its DMMA (mma.sync m8n8k4 f64) peaks
// at 37 TFLOP/s, while the int8 tcgen05 path peaks at 4.5 POPS.  The panel rows are split into
// 8 signed slices each, after scaling every row by a power of two 2^-e_r (|L(r, :)| < 2^(e_r - 1)):
//     L(r, k) 2^-e_r = sum_{s=1..8} d_s(r, k) 2^-7s + delta,   |d_s| <= 64, |delta| <= 2^-57
// with balanced digits (each d_s the nearest integer of an exact power-of-two rescaling of the
// remainder, so every step is exact in FP64; balanced digits make the dropped products 4x
// smaller than truncated ones and of random sign), and
//     sum_k L(i, k) L(j, k) = 2^(e_i + e_j) sum_{g=2..9} 2^-7g acc_g + O(2^-53 K 2^(e_i + e_j)),
//     acc_g = sum_{s + t = g} sum_k d_s(i, k) d_t(j, k)                       (int32, exact)
// The 36 slice products with s + t <= 9 are tcgen05 MMAs (M = 128, N = 64, K = 32) into 8 TMEM
// accumulators of 64 columns (all 512 TMEM columns); the epilogue reconstructs in FP64 from the
// smallest group up and subtracts from C.  Measured error relative to sum_k |L(i,k) L(j,k)|:
// ~3.3e-16 (3 u) at K = 2048 (tools/ozaki_probe.cu), DGEMM-class.  int32 exactness needs
// 8 * 64^2 * K < 2^31 (K <= 65536); OZ_KMAX keeps a margin.
//
//   oz_expo_kernel    per-row exponents e_r of the panel rows
//   oz_slice_kernel   the 8 slices in the UMMA K-major SWIZZLE_NONE layout, once as 128-row A
//                     tiles and once as 64-row B tiles ([s][tile][kstep][chunk][rows][16 B])
//   oz_update_kernel  one CTA per (128 x 64) half of an output tile: cp.async.bulk producer warp,
//                     single-thread tcgen05.mma issuer, 4 epilogue warps (tcgen05.ld)

namespace b2d {

constexpr int OZ_S = 8;                      // slices per operand
constexpr int OZ_BM = 128, OZ_BN = 64;       // CTA tile (rows of C x columns of C)
constexpr int OZ_KSTEP = 32;                 // bytes of K per MMA
constexpr int OZ_STAGES = 4;
constexpr int OZ_A_STAGE = OZ_S * OZ_BM * OZ_KSTEP;  // 32 KB
constexpr int OZ_B_STAGE = OZ_S * OZ_BN * OZ_KSTEP;  // 16 KB
constexpr int OZ_THREADS = 192;              // warp 0 producer, warp 1 MMA, warps 2-5 epilogue
constexpr int OZ_KMAX = 32768;               // K bound (int32 exactness holds to 65536)
constexpr size_t OZ_SMEM = (size_t)OZ_STAGES * (OZ_A_STAGE + OZ_B_STAGE) + (2 * OZ_STAGES + 1) * 8 + 16;
// kind::i8 instruction descriptor: D s32 (bits 4-5 = 2), A and B signed (bits 7, 10), K-major,
// N >> 3 at bit 17, M >> 4 at bit 24
constexpr uint32_t OZ_IDESC = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(OZ_BN >> 3) << 17) |
                              ((uint32_t)(OZ_BM >> 4) << 24);

// Slices of panel rows [r0 tiles, r0 + rt) x K tiles [p0, p0 + kt) of `map`.
struct OzPanel {
  TileMap map;
  int r0, rt, p0, kt;
  int8_t* sa;  // [s][rt][nks][2][128][16]
  int8_t* sb;  // [s][2 rt][nks][2][64][16]
  int* expo;   // [rt * 128]
};

__device__ __forceinline__ uint64_t oz_sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  // SWIZZLE_NONE K-major: start, LBO = next 16-byte K chunk, SBO = next 8-row group, version 1
  return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46);
}

__global__ void __launch_bounds__(256) oz_expo_kernel(OzPanel P) {
  const int it = blockIdx.x;
  const int r = threadIdx.x & 127, half = threadIdx.x >> 7;
  __shared__ double smax[2][T];
  double m = 0.0;
  for (int p = half; p < P.kt; p += 2) {
    const double* t = P.map.tile(P.r0 + it, P.p0 + p);
    for (int c = 0; c < T; ++c) m = fmax(m, fabs(t[elem(r, c)]));
  }
  smax[half][r] = m;
  __syncthreads();
  if (half == 0) {
    const double mm = fmax(smax[0][r], smax[1][r]);
    P.expo[it * T + r] = mm > 0.0 ? ilogb(mm) + 2 : 0;  // |row| < 2^(e - 1): balanced digits fit
  }
}

// grid (rt, kt): one CTA per panel tile; thread (r, 16-column chunk pair)
__global__ void __launch_bounds__(256) oz_slice_kernel(OzPanel P) {
  const int it = blockIdx.x, p = blockIdx.y;
  const int K = P.kt * T, nks = K / OZ_KSTEP;
  const double* t = P.map.tile(P.r0 + it, P.p0 + p);
  const int r = threadIdx.x & 127;
  const int e = P.expo[it * T + r];
  for (int cc = threadIdx.x >> 7; cc < T / 16; cc += 2) {
    double x[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) x[u] = scalbn(t[elem(r, cc * 16 + u)], -e);
    const int k0 = p * T + cc * 16, ks = k0 / OZ_KSTEP, ch = (k0 % OZ_KSTEP) / 16;
    const int t64 = it * 2 + (r >> 6), r64 = r & 63;
#pragma unroll
    for (int s = 0; s < OZ_S; ++s) {
      int8_t d[16];
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        const double y = x[u] * 128.0;
        const double q = rint(y);  // |y| <= 64: a balanced digit, y - q exact
        d[u] = (int8_t)q;
        x[u] = y - q;
      }
      const uint4 v = *reinterpret_cast<const uint4*>(d);
      *reinterpret_cast<uint4*>(P.sa + ((((size_t)s * P.rt + it) * nks + ks) * 2 + ch) * (OZ_BM * 16) + (size_t)r * 16) = v;
      *reinterpret_cast<uint4*>(P.sb + ((((size_t)s * 2 * P.rt + t64) * nks + ks) * 2 + ch) * (OZ_BN * 16) + (size_t)r64 * 16) = v;
    }
  }
}

// C(i, j) -= L(i, .) L(j, .)^T over the tile set `out` (rows and columns index the panel rows:
// panel row tile = tile index - P.r0).  CTA b: tile tile_order(b / 2), columns 64 (b % 2) + [0, 64).
__global__ void __launch_bounds__(OZ_THREADS, 1) oz_update_kernel(OzPanel P, TileMap C, TileSet out) {
  extern __shared__ __align__(1024) double oz_smem[];  // (same symbol type as the other kernels')
  uint8_t* sA = reinterpret_cast<uint8_t*>(oz_smem);
  uint8_t* sB = sA + OZ_STAGES * OZ_A_STAGE;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + OZ_STAGES * OZ_B_STAGE);
  uint64_t* empty = full + OZ_STAGES;
  uint64_t* done = empty + OZ_STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nks = P.kt * T / OZ_KSTEP;
  int I, J;
  tile_order(blockIdx.x >> 1, out, 8, &I, &J);
  const int h = blockIdx.x & 1;
  const int ia = I - P.r0, t64 = 2 * (J - P.r0) + h;
  if (threadIdx.x == 0) {
    for (int s = 0; s < OZ_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(done, 1);
    fence_mbar_init();
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
    for (int ks = 0; ks < nks; ++ks) {
      const int st = ks % OZ_STAGES;
      if (ks >= OZ_STAGES) mbar_wait(&empty[st], ((ks / OZ_STAGES) - 1) & 1);
      mbar_arrive_expect_tx(&full[st], OZ_A_STAGE + OZ_B_STAGE);
#pragma unroll
      for (int s = 0; s < OZ_S; ++s) {
        bulk_g2s(sA + st * OZ_A_STAGE + s * (OZ_BM * OZ_KSTEP),
                 P.sa + (((size_t)s * P.rt + ia) * nks + ks) * (OZ_BM * OZ_KSTEP), OZ_BM * OZ_KSTEP, &full[st]);
        bulk_g2s(sB + st * OZ_B_STAGE + s * (OZ_BN * OZ_KSTEP),
                 P.sb + (((size_t)s * 2 * P.rt + t64) * nks + ks) * (OZ_BN * OZ_KSTEP), OZ_BN * OZ_KSTEP, &full[st]);
      }
    }
  } else if (warp == 1 && lane == 0) {
    for (int ks = 0; ks < nks; ++ks) {
      const int st = ks % OZ_STAGES;
      mbar_wait(&full[st], (ks / OZ_STAGES) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;");
      const uint32_t a0 = smem_u32(sA + st * OZ_A_STAGE), b0 = smem_u32(sB + st * OZ_B_STAGE);
#pragma unroll
      for (int g = 2; g <= OZ_S + 1; ++g) {
        const int s_first = g - OZ_S > 1 ? g - OZ_S : 1;
#pragma unroll
        for (int s = 1; s <= OZ_S; ++s) {
          const int t = g - s;
          if (t < 1 || t > OZ_S) continue;
          const uint64_t da = oz_sdesc(a0 + (s - 1) * (OZ_BM * OZ_KSTEP), OZ_BM * 16, 8 * 16);
          const uint64_t db = oz_sdesc(b0 + (t - 1) * (OZ_BN * OZ_KSTEP), OZ_BN * 16, 8 * 16);
          const uint32_t accum = (ks > 0 || s > s_first) ? 1u : 0u;  // the first product of g overwrites
          asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                       "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n"
                       ::"r"(tmem + (uint32_t)((g - 2) * OZ_BN)), "l"(da), "l"(db), "r"(OZ_IDESC), "r"(accum));
        }
      }
      // frees the stage once these MMAs have read it
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                   ::"r"(smem_u32(&empty[st])) : "memory");
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                 ::"r"(smem_u32(done)) : "memory");
  } else if (warp >= 2) {
    mbar_wait(done, 0);
    asm volatile("tcgen05.fence::after_thread_sync;");
    const int q = warp & 3;        // TMEM lanes 32q .. 32q + 31
    const int r = q * 32 + lane;   // row of the output tile
    double acc[OZ_BN];
#pragma unroll
    for (int c = 0; c < OZ_BN; ++c) acc[c] = 0.0;
    for (int g = OZ_S + 1; g >= 2; --g) {  // smallest contributions first
      const double w = ldexp(1.0, -7 * g);
#pragma unroll
      for (int c0 = 0; c0 < OZ_BN; c0 += 32) {
        uint32_t v[32];
        const uint32_t taddr = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)((g - 2) * OZ_BN + c0);
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                     "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                     : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                       "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
                       "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
                       "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
                     : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;");
#pragma unroll
        for (int j = 0; j < 32; ++j) acc[c0 + j] = fma((double)(int32_t)v[j], w, acc[c0 + j]);
      }
    }
    const int ei = P.expo[ia * T + r];
    const int* ej = P.expo + (J - P.r0) * T + h * OZ_BN;
    double* ct = C.tile(I, J);
#pragma unroll
    for (int c = 0; c < OZ_BN; ++c) {
      const int o = elem(r, h * OZ_BN + c);
      ct[o] = ct[o] - ldexp(acc[c], ei + ej[c]);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp == 2) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(512));
}

}  // namespace b2d
