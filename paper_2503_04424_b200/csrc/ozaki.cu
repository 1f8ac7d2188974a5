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
// The 36 slice products with s + t <= 9 are tcgen05 MMAs (M = 128, N = 128, K = 32), one CTA per
// output tile, in two passes over K so that 4 accumulators of 128 columns fill the 512 TMEM
// columns: pass 0 the groups g = 2..5 (10 products, slices 1..4), pass 1 g = 6..9 (26 products).
// The epilogue warps drain each pass (from the smallest group up, in FP64) and subtract it from
// C; pass 1's MMAs start as soon as pass 0's accumulators are read, and its operands are already
// prefetched.  Measured error relative to sum_k |L(i,k) L(j,k)|:
// ~3.3e-16 (3 u) at K = 2048 (tools/ozaki_probe.cu), DGEMM-class.  int32 exactness needs
// 8 * 64^2 * K < 2^31 (K <= 65536); OZ_KMAX keeps a margin.
//
//   oz_expo_kernel    per-row exponents e_r of the panel rows
//   oz_slice_kernel   the 8 slices in the UMMA K-major SWIZZLE_NONE layout of 128-row tiles
//                     ([s][tile][kstep][chunk][128 rows][16 B]; both MMA operands use it)
//   oz_update_kernel  one CTA per output tile: cp.async.bulk producer warp, single-thread
//                     tcgen05.mma issuer, 8 epilogue warps (tcgen05.ld, 4 lane quadrants x 2
//                     column halves)

#include <type_traits>

namespace b2d {

constexpr int OZ_S = 8;                      // slices per operand
constexpr int OZ_BM = 128, OZ_BN = 128;      // CTA tile = one output tile
constexpr int OZ_KSTEP = 32;                 // bytes of K per MMA
constexpr int OZ_STAGES = 3;
constexpr int OZ_SLICE = OZ_BM * OZ_KSTEP;   // 4 KB: one slice of one operand for one K step
constexpr int OZ_STAGE = 2 * OZ_S * OZ_SLICE;  // 64 KB: 8 slices of A and of B
constexpr int OZ_THREADS = 320;              // warp 0 producer, warp 1 MMA, warps 2-9 epilogue
#ifndef OZ_RASTER_G
#define OZ_RASTER_G 8
#endif
constexpr int OZ_KMAX = 32768;               // K bound (int32 exactness holds to 65536)
constexpr size_t OZ_SMEM = (size_t)OZ_STAGES * OZ_STAGE + (2 * OZ_STAGES + 3) * 8 + 16;
// kind::i8 instruction descriptor: D s32 (bits 4-5 = 2), A and B signed (bits 7, 10), K-major,
// N >> 3 at bit 17, M >> 4 at bit 24
constexpr uint32_t OZ_IDESC = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(OZ_BN >> 3) << 17) |
                              ((uint32_t)(OZ_BM >> 4) << 24);

// Slices of panel rows [r0 tiles, r0 + rt) x K tiles [p0, p0 + kt) of `map`.
struct OzPanel {
  TileMap map;
  int r0, rt, p0, kt;
  int8_t* sa;  // [s][rt][nks][2][128][16]
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
    }
  }
}

// C(i, j) -= L(i, .) L(j, .)^T over the tile set `out` (panel row tile = tile index - P.r0),
// one CTA per output tile (tile_order).
// Two passes: the products with s + t <= 9.  (A third pass for s + t = 10 would cut the
// truncation error ~64x but streams every slice again for only 7 MMAs per K step: ~50% slower.)
constexpr int NPASS = 2;
__global__ void __launch_bounds__(OZ_THREADS, 1) oz_update_kernel(OzPanel P, TileMap C, TileSet out) {
  extern __shared__ __align__(1024) double oz_smem[];
  uint8_t* sm8 = reinterpret_cast<uint8_t*>(oz_smem);
  uint64_t* full = reinterpret_cast<uint64_t*>(sm8 + OZ_STAGES * OZ_STAGE);
  uint64_t* empty = full + OZ_STAGES;
  uint64_t* done = empty + OZ_STAGES;  // [2]: each pass's accumulators complete
  uint64_t* drained = done + 2;        // pass 0's accumulators read by the epilogue
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(drained + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nks = P.kt * T / OZ_KSTEP;
  int I, J;
  tile_order(blockIdx.x, out, OZ_RASTER_G, &I, &J);
  const int ia = I - P.r0, ja = J - P.r0;
  // each CTA walks K from its own offset: neighbouring CTAs (which share operand rows) then read
  // different K steps at any moment instead of all hammering the same L2 lines; int32
  // accumulation is exact, so the order does not change the result
  const int rot = (int)((blockIdx.x * 7u) % (unsigned)nks);
  if (threadIdx.x == 0) {
    for (int s = 0; s < OZ_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(&done[0], 1);
    mbar_init(&done[1], 1);
    mbar_init(drained, 8 * 32);
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
  // pass p (compile time): groups g = G0(p) .. G0(p) + 3 from slices 1 .. NS(p)
  constexpr int G0[2] = {2, 6}, NGR[2] = {4, 4}, NSL[2] = {4, OZ_S};
  if (warp == 0 && lane == 0) {
    // stage = slices [0, ns) of A (rows I) at slot s, of B (rows J) at slot 8 + s
    int it = 0;
    auto produce = [&](auto pass_c) {
      constexpr int ns = NSL[decltype(pass_c)::value];
      for (int ks = 0; ks < nks; ++ks, ++it) {
        const int st = it % OZ_STAGES;
        if (it >= OZ_STAGES) mbar_wait(&empty[st], ((it / OZ_STAGES) - 1) & 1);
        mbar_arrive_expect_tx(&full[st], 2 * ns * OZ_SLICE);
        uint8_t* base = sm8 + st * OZ_STAGE;
        const int kk = ks + rot < nks ? ks + rot : ks + rot - nks;
#pragma unroll
        for (int s = 0; s < ns; ++s) {
          bulk_g2s(base + s * OZ_SLICE, P.sa + (((size_t)s * P.rt + ia) * nks + kk) * OZ_SLICE, OZ_SLICE, &full[st]);
          bulk_g2s(base + (OZ_S + s) * OZ_SLICE, P.sa + (((size_t)s * P.rt + ja) * nks + kk) * OZ_SLICE, OZ_SLICE,
                   &full[st]);
        }
      }
    };
    produce(std::integral_constant<int, 0>{});
    produce(std::integral_constant<int, 1>{});
  } else if (warp == 1 && lane == 0) {
    int it = 0;
    auto mma = [&](auto pass_c) {
      constexpr int pass = decltype(pass_c)::value;
      if (pass > 0) {  // the accumulators are reused: the previous pass's must have been read
        mbar_wait(drained, (pass - 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;");
      }
      for (int ks = 0; ks < nks; ++ks, ++it) {
        const int st = it % OZ_STAGES;
        mbar_wait(&full[st], (it / OZ_STAGES) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;");
        const uint32_t base = smem_u32(sm8 + st * OZ_STAGE);
#pragma unroll
        for (int gg = 0; gg < NGR[pass]; ++gg) {
          const int g = G0[pass] + gg;
          const int s_first = g - OZ_S > 1 ? g - OZ_S : 1;
#pragma unroll
          for (int s = 1; s <= OZ_S; ++s) {
            const int t = g - s;
            if (t < 1 || t > OZ_S) continue;
            const uint64_t da = oz_sdesc(base + (s - 1) * OZ_SLICE, OZ_BM * 16, 8 * 16);
            const uint64_t db = oz_sdesc(base + (OZ_S + t - 1) * OZ_SLICE, OZ_BN * 16, 8 * 16);
            const uint32_t accum = (ks > 0 || s > s_first) ? 1u : 0u;  // the first product of g overwrites
            asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                         "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n"
                         ::"r"(tmem + (uint32_t)(gg * OZ_BN)), "l"(da), "l"(db), "r"(OZ_IDESC), "r"(accum));
          }
        }
        // frees the stage once these MMAs have read it
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                     ::"r"(smem_u32(&empty[st])) : "memory");
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                   ::"r"(smem_u32(&done[pass])) : "memory");
    };
    mma(std::integral_constant<int, 0>{});
    mma(std::integral_constant<int, 1>{});
  } else if (warp >= 2) {
    const int q = warp & 3, hh = (warp - 2) >> 2;  // TMEM lane quadrant, column half
    const int r = q * 32 + lane;                   // row of the output tile
    const int ei = P.expo[ia * T + r];
    const int* ej = P.expo + ja * T + 64 * hh;
    double* ct = C.tile(I, J);
    auto drain = [&](auto pass_c) {
      constexpr int pass = decltype(pass_c)::value;
      mbar_wait(&done[pass], 0);
      asm volatile("tcgen05.fence::after_thread_sync;");
      double part[2][32];
#pragma unroll
      for (int ch = 0; ch < 2; ++ch) {
#pragma unroll
        for (int j = 0; j < 32; ++j) part[ch][j] = 0.0;
#pragma unroll 1
        for (int gg = NGR[pass] - 1; gg >= 0; --gg) {  // smallest contributions first
          const double w = ldexp(1.0, -7 * (G0[pass] + gg));
          uint32_t v[32];
          const uint32_t taddr = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(gg * OZ_BN + 64 * hh + 32 * ch);
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
      if (pass + 1 < NPASS) {  // TMEM read: the next pass may overwrite it while C is updated
        asm volatile("tcgen05.fence::before_thread_sync;");
        mbar_arrive(drained);
      }
#pragma unroll
      for (int ch = 0; ch < 2; ++ch)
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const int c = 32 * ch + j;
          const int o = elem(r, 64 * hh + c);
          // explicit global accesses (a TileMap pointer is generic to the compiler)
          __stcg(ct + o, __ldg(ct + o) - ldexp(part[ch][j], ei + __ldg(ej + c)));
        }
    };
    drain(std::integral_constant<int, 0>{});
    drain(std::integral_constant<int, 1>{});
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp == 2) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(512));
}

}  // namespace b2d
