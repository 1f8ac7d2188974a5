// Device kernels of the B200 MEMDET engine (sm_100a).
//
//   pack_tiles_kernel   row-major MEMDET01 data (f64/f32, device) -> packed lower tile triangle
//   potrf_inv_kernel    diagonal tile: Cholesky (= unpivoted LDL^T, D = L_ii^2), fused
//                       2 log L_ii, NotSpd detection, and L_kk^{-1} for the panel solve
//   gemm_kernel         DMMA (FP64 tensor core) tile GEMM, cp.async.bulk + mbarrier pipeline:
//                         MODE_UPDATE: C(i,j) -= sum_p L(i,p) L(j,p)^T  (Schur update)
//                         MODE_TRSM:   L(i,k)  = A(i,k) L_kk^{-T}       (panel solve)
//   prefix_kernel       compensated (double-double) prefix scan of 2 log L_ii -> every
//                       leading-principal-minor logdet
//   gen_rbf_kernel      C2 input generator (off the timed path)
//
// Reference call sites these replace: kernels/dense.py:84-91 (potrf), :94-99 (trtrs),
// :109-116 (schur_update), memdet.py:406-407,428 (cumsum of log d).
#include "tile.cuh"

namespace b2d {

// ------------------------------------------------------------------------------ pack

// Packs tile-columns [j_lo, j_hi) (all tiles (I, J), I >= J) from a row-major source whose
// first stored row is `row_base` (0 for a whole matrix, 128*J for a strip buffer).
// Tile element (r, c) = src[C][R] (R = 128I + r, C = 128J + c): the row-major UPPER triangle,
// i.e. the (i <= j) tiles the reference reads (memdet.py:364, 376, 384); identity padding
// beyond m.
// Two passes of 64 columns keep shared memory at 66 KB, so a pack CTA co-resides with a
// Schur-update CTA (128 KB) on one SM while host strips stream in under the factorisation.
constexpr int PACK_THREADS = 256;
constexpr int PACK_LD = 130;  // staging row pitch: conflict-free octet-order reads (2c + r mod 16)
constexpr size_t PACK_SMEM = (size_t)64 * PACK_LD * 8;

// One 128 x 128 tile through shared memory: element (r, c) = ld(r, c), where a tile column c
// is a contiguous source row.  NLOAD loads per thread are issued before the first use, so a
// CTA keeps 256 * NLOAD * 8 bytes in flight; the octet-layout writes are contiguous.
template <int NLOAD, typename F>
__device__ __forceinline__ void pack_tile_body(double* sm, double* __restrict__ dst, F ld) {
  const int tid = threadIdx.x;
  for (int half = 0; half < 2; ++half) {
    for (int k0 = 0; k0 < 32; k0 += NLOAD) {
      double v[NLOAD];
#pragma unroll
      for (int k = 0; k < NLOAD; ++k) {
        const int idx = tid + (k0 + k) * PACK_THREADS;
        v[k] = ld(idx & 127, 64 * half + (idx >> 7));
      }
#pragma unroll
      for (int k = 0; k < NLOAD; ++k) {
        const int idx = tid + (k0 + k) * PACK_THREADS;
        sm[(idx >> 7) * PACK_LD + (idx & 127)] = v[k];
      }
    }
    __syncthreads();
    // octets 8*half .. 8*half+7 are the contiguous half-tile [half*8192, half*8192 + 8192)
#pragma unroll 8
    for (int o = tid; o < 64 * T; o += PACK_THREADS) {
      const int r = (o >> 3) & 127;
      const int c = ((o >> 10) << 3) + iperm8(o & 7);  // 0..63 within this half
      dst[half * 64 * T + o] = sm[c * PACK_LD + r];
    }
    __syncthreads();
  }
}

// NLOAD = 32: whole-matrix pack from HBM (nothing else runs; 2 CTAs per SM); NLOAD = 8 keeps
// 64 registers so that strip packs co-reside with Schur-update CTAs during host ingest.
template <typename Tin, int NLOAD>
__global__ void __launch_bounds__(PACK_THREADS, NLOAD >= 32 ? 2 : 4)
    pack_tiles_kernel(const Tin* __restrict__ src, int64_t lda, int64_t row_base, int64_t m,
                      double* __restrict__ tiles, int nt, int j_lo, int i_lo = 0) {
  extern __shared__ double sm[];  // [64][PACK_LD]: sm[c*PACK_LD + r] for the current 64 columns
  // tiles (I, J), J >= j_lo, I >= max(J, i_lo), column by column
  int64_t b = blockIdx.x;
  int J = j_lo;
  while (b >= nt - max(J, i_lo)) { b -= nt - max(J, i_lo); ++J; }
  const int I = max(J, i_lo) + (int)b;
  const int64_t R0 = (int64_t)I * T, C0 = (int64_t)J * T;
  pack_tile_body<NLOAD>(sm, tiles + tile_index(I, J, nt) * TILE_ELEMS, [&](int r, int c) {
    const int64_t R = R0 + r, C = C0 + c;
    return (R < m && C < m) ? (double)src[(C - row_base) * lda + R] : ((R == C) ? 1.0 : 0.0);
  });
}

// Distributed ingest: the tiles of a TileSet (rows possibly local indices of a row-cyclic
// distribution, global row = i * stride + off) from a row-major source (first stored row
// row_base) into map `out` at (local row, column).  Same element rule as pack_tiles_kernel.
template <typename Tin>
__global__ void __launch_bounds__(PACK_THREADS, 4) pack_set_kernel(const Tin* __restrict__ src, int64_t lda,
                                                                int64_t row_base, int64_t m, TileMap out,
                                                                TileSet set) {
  extern __shared__ double sm[];
  int li, J;
  tile_order(blockIdx.x, set, 1, &li, &J);
  const int st = set.stride > 1 ? set.stride : 1;
  const int I = li * st + set.off;
  const int64_t R0 = (int64_t)I * T, C0 = (int64_t)J * T;
  pack_tile_body<8>(sm, out.tile(li, J), [&](int r, int c) {
    const int64_t R = R0 + r, C = C0 + c;
    return (R < m && C < m) ? (double)src[(C - row_base) * lda + R] : ((R == C) ? 1.0 : 0.0);
  });
}

// Out-of-core block ingest: one 128-row strip of the row-major file (rows = the block's
// tile-column J, columns = the block's rows) into tile-column J of a grid block.  Local row R
// of the block is valid below rows_valid, local column C below cols_valid; the padding is the
// identity on a diagonal block and zero elsewhere.  src points at element (first strip row,
// first block row) of the file, leading dimension lda.
template <typename Tin>
__global__ void __launch_bounds__(PACK_THREADS, 4) pack_block_kernel(const Tin* __restrict__ src,
                                                                  int64_t lda, int64_t rows_valid,
                                                                  int64_t cols_valid, int diag,
                                                                  TileMap out, int J) {
  extern __shared__ double sm[];
  const int I = blockIdx.x;
  const int64_t R0 = (int64_t)I * T, C0 = (int64_t)J * T;
  pack_tile_body<8>(sm, out.tile(I, J), [&](int r, int c) {
    const int64_t R = R0 + r, C = C0 + c;
    return (R < rows_valid && C < cols_valid) ? (double)src[(C - C0) * lda + R] : ((diag && R == C) ? 1.0 : 0.0);
  });
}

// Gram formation helpers.  init: packed lower tiles = jitter * I (identity beyond m, so the
// padding factors to 1).  pack_rect: a row-major m x k device chunk G into an nt x kt tile grid
// scaled by `scale` (zero beyond m / k), G's rows along tile rows.
__global__ void packed_init_kernel(double* __restrict__ tiles, int nt, int64_t m, double jitter) {
  const int64_t ntiles = n_packed_tiles(nt);
  for (int64_t tix = blockIdx.x; tix < ntiles; tix += gridDim.x) {
    // tile-column j: the largest j with col_offset(j, nt) <= tix (quadratic root, then fix up)
    const double a = nt + 0.5;
    int j = (int)(a - sqrt(a * a - 2.0 * (double)tix));
    if (j < 0) j = 0;
    while (j > 0 && col_offset(j, nt) > tix) --j;
    while (j + 1 < nt && col_offset(j + 1, nt) <= tix) ++j;
    const int i = j + (int)(tix - col_offset(j, nt));
    double* t = tiles + tix * TILE_ELEMS;
    for (int o = threadIdx.x; o < TILE_ELEMS; o += blockDim.x) {
      double v = 0.0;
      if (i == j) {
        const int r = (o >> 3) & 127, c = ((o >> 10) << 3) + iperm8(o & 7);
        if (r == c) v = ((int64_t)i * T + r < m) ? jitter : 1.0;
      }
      t[o] = v;
    }
  }
}

__global__ void __launch_bounds__(256) pack_rect_kernel(const double* __restrict__ g, int64_t ldg, int64_t m,
                                                        int64_t k, double scale, TileMap out, int kt) {
  __shared__ double sm[32][129];
  const int I = blockIdx.x / kt, P = blockIdx.x % kt;
  double* dst = out.tile(I, P);
  for (int qtr = 0; qtr < 4; ++qtr) {
    for (int idx = threadIdx.x; idx < 32 * T; idx += 256) {  // rows r, 32 columns: coalesced in c
      const int r = idx >> 5, c = idx & 31;
      const int64_t R = (int64_t)I * T + r, C = (int64_t)P * T + 32 * qtr + c;
      sm[c][r] = (R < m && C < k) ? g[R * ldg + C] * scale : 0.0;
    }
    __syncthreads();
    for (int o = threadIdx.x; o < 32 * T; o += 256) {  // octets 4*qtr .. 4*qtr+3
      const int r = (o >> 3) & 127;
      const int c = ((o >> 10) << 3) + iperm8(o & 7);
      dst[qtr * 32 * T + o] = sm[c][r];
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------------------------ potrf + inverse

// One CTA of 256 threads factors diagonal tile (k, k) in shared memory M[128][129].
// Phase A (Cholesky, right-looking over 8-column blocks, two barriers per block):
//   A2  one thread per row solves the block column below the current 8x8 diagonal block;
//   A3  all threads apply the rank-8 update to the trailing lower triangle in 4x4 register
//       blocks, while thread 0 updates AND factors the next 8x8 diagonal block (look-ahead,
//       so the serial rsqrt chain hides under the update).
// Phase B (X = L^{-1}): row blocks of 8 in order; per block, 256 threads form the partial
//   products L[rb, :rb] X[:rb, c] (two threads per column), then one thread per column does
//   the 8x8 forward substitution.  X[r][c] (r > c) lives transposed in the free upper
//   triangle M[c][r]; X[c][c] = dinv[c].
// Outputs: L_kk back to its tile (lower, zero upper), X to `inv` (tile layout, B operand of
// the panel solve), ell[g] = 2 log L_gg (memdet.py:428), diag[g] = L_gg, fail = first global
// row with a non-positive pivot (atomicMin; dense.py:86-89 raises NotSpdError there).
constexpr int POTRF_THREADS = 256;
constexpr int MLD = 129;
constexpr size_t POTRF_SMEM = (size_t)(T * MLD + 8 * T) * 8;

// Serial Cholesky of the 8x8 block at rows/cols c0..c0+7 (one thread, registers only).
__device__ __forceinline__ void factor_diag8(double* M, double* dinv, int c0) {
  double a[8][8];
#pragma unroll
  for (int r = 0; r < 8; ++r)
#pragma unroll
    for (int c = 0; c <= r; ++c) a[r][c] = M[(c0 + r) * MLD + c0 + c];
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const double rq = rsqrt(a[q][q]);
    a[q][q] *= rq;
    dinv[c0 + q] = rq;
#pragma unroll
    for (int r = q + 1; r < 8; ++r) a[r][q] *= rq;
#pragma unroll
    for (int r = q + 1; r < 8; ++r)
#pragma unroll
      for (int c = q + 1; c <= r; ++c) a[r][c] = fma(-a[r][q], a[c][q], a[r][c]);
  }
#pragma unroll
  for (int r = 0; r < 8; ++r)
#pragma unroll
    for (int c = 0; c <= r; ++c) M[(c0 + r) * MLD + c0 + c] = a[r][c];
}

// tile: the diagonal tile; g0: global index of its first row (ell/diag/fail), m: global order
__global__ void __launch_bounds__(POTRF_THREADS) potrf_inv_kernel(double* __restrict__ tile,
                                                                  double* __restrict__ inv,
                                                                  double* __restrict__ ell,
                                                                  double* __restrict__ diag,
                                                                  unsigned long long* __restrict__ fail,
                                                                  int64_t g0, int64_t m,
                                                                  long long* prof = nullptr) {
#define PROF(i) if (prof && tid == 0) prof[i] = clock64();
  extern __shared__ double M[];   // [T][MLD], then S[8][T] scratch
  double* S = M + T * MLD;
  __shared__ double dinv[T];
  const int tid = threadIdx.x;
  PROF(0)
  {
    double2 v[TILE_ELEMS / 2 / POTRF_THREADS];  // all 32 loads in flight
#pragma unroll
    for (int u = 0; u < TILE_ELEMS / 2 / POTRF_THREADS; ++u)
      v[u] = reinterpret_cast<const double2*>(tile)[tid + u * POTRF_THREADS];
#pragma unroll
    for (int u = 0; u < TILE_ELEMS / 2 / POTRF_THREADS; ++u) {
      const int o = 2 * (tid + u * POTRF_THREADS);  // positions (o, o+1): columns c and c+4
      const int r = (o >> 3) & 127;
      const int c = ((o >> 10) << 3) + iperm8(o & 7);
      M[r * MLD + c] = v[u].x;
      M[r * MLD + c + 4] = v[u].y;
    }
  }
  __syncthreads();
  PROF(1)
  if (tid == 0) factor_diag8(M, dinv, 0);
  __syncthreads();
  PROF(2)

  for (int c0 = 0; c0 + 8 < T; c0 += 8) {
    // A2: block column below the (already factored) diagonal block
    {
      const int i = c0 + 8 + tid;
      if (i < T) {
        double s[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) s[q] = M[i * MLD + c0 + q];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          double v = s[q];
#pragma unroll
          for (int q2 = 0; q2 < q; ++q2) v = fma(-s[q2], M[(c0 + q) * MLD + c0 + q2], v);
          s[q] = v * dinv[c0 + q];
        }
#pragma unroll
        for (int q = 0; q < 8; ++q) M[i * MLD + c0 + q] = s[q];
      }
    }
    __syncthreads();
    if (c0 == 0) PROF(3)
    // A3: rank-8 trailing update in 4x4 blocks; thread 0 takes the next diagonal 8x8 block
    {
      const int base = c0 + 8;
      if (tid < 32) {
        // warp 0: the 36 lower entries of the next diagonal block, then lane 0 factors it
        for (int e = tid; e < 36; e += 32) {
          int r = (int)((sqrtf(8.0f * e + 1.0f) - 1.0f) * 0.5f);
          while ((r + 1) * (r + 2) / 2 <= e) ++r;
          while (r * (r + 1) / 2 > e) --r;
          const int c = e - r * (r + 1) / 2;
          double lr[8], lc[8];
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            lr[q] = M[(base + r) * MLD + c0 + q];
            lc[q] = M[(base + c) * MLD + c0 + q];
          }
          double v = M[(base + r) * MLD + base + c];
#pragma unroll
          for (int q = 0; q < 8; ++q) v = fma(-lr[q], lc[q], v);
          M[(base + r) * MLD + base + c] = v;
        }
        __syncwarp();
        if (c0 == 0) PROF(4)
        if (tid == 0) factor_diag8(M, dinv, base);
        if (c0 == 0) PROF(5)
      }
      // warps 0 and 4 share SMSP 0: keep that scheduler for the serial diagonal chain
      const int w = tid >> 5;
      const int nb4 = (T - base) >> 2;
      const int nblk = nb4 * (nb4 + 1) / 2;
      const int slot = w < 4 ? tid - 32 : tid - 64;  // 0..191 over warps 1-3, 5-7
      for (int b = 3 + slot; (w & 3) != 0 && b < nblk; b += 192) {  // 0..2: next diag 8x8
        int bi = (int)((sqrtf(8.0f * b + 1.0f) - 1.0f) * 0.5f);
        while ((bi + 1) * (bi + 2) / 2 <= b) ++bi;
        while (bi * (bi + 1) / 2 > b) --bi;
        const int bj = b - bi * (bi + 1) / 2;
        const int i0 = base + 4 * bi, j0 = base + 4 * bj;
        double li[4][8], lj[4][8];
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            li[r][q] = M[(i0 + r) * MLD + c0 + q];
            lj[r][q] = M[(j0 + r) * MLD + c0 + q];
          }
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
          for (int cc = 0; cc < 4; ++cc) {
            double v = M[(i0 + r) * MLD + j0 + cc];
#pragma unroll
            for (int q = 0; q < 8; ++q) v = fma(-li[r][q], lj[cc][q], v);
            M[(i0 + r) * MLD + j0 + cc] = v;
          }
      }
    }
    __syncthreads();
    if (c0 == 0) PROF(6)
  }
  PROF(7)

  // Phase B: thread t pairs columns j and 127-j (balanced work), rows 2h, 2h+1 per block
  {
    const int j = tid & 63, h = tid >> 6;
    const int cA = j, cB = 127 - j;
    const int pwA = cA & ~31, pwB = cB & ~31;  // warp-uniform starts (broadcast L reads)
    const double dA = dinv[cA], dB = dinv[cB];
    for (int r0 = 0; r0 < T; r0 += 8) {
      const double* L0 = M + (r0 + 2 * h) * MLD;
#pragma unroll
      for (int side = 0; side < 2; ++side) {
        const int c = side ? cB : cA;
        const int pw = side ? pwB : pwA;
        const double dc = side ? dB : dA;
        if (r0 + 7 < pw) continue;
        const double* Xc = M + c * MLD;
        double s0 = 0.0, s1 = 0.0;
        for (int p0 = pw; p0 < r0; p0 += 8) {
          double x[8], l0[8], l1[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int p = p0 + u;
            const double xv = Xc[p];
            x[u] = p < c ? 0.0 : (p == c ? dc : xv);
            l0[u] = L0[p];
            l1[u] = L0[MLD + p];
          }
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            s0 = fma(l0[u], x[u], s0);
            s1 = fma(l1[u], x[u], s1);
          }
        }
        S[(2 * h) * T + c] = s0;
        S[(2 * h + 1) * T + c] = s1;
      }
      __syncthreads();
      if (tid < T && r0 + 7 > tid) {
        const int c = tid;
        const double dc = dinv[c];
        double ld[8][8], sv[8], di[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          sv[q] = (r0 + 7 >= (c & ~31)) ? S[q * T + c] : 0.0;
          di[q] = dinv[r0 + q];
#pragma unroll
          for (int q2 = 0; q2 < q; ++q2) ld[q][q2] = M[(r0 + q) * MLD + r0 + q2];
        }
        double xq[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const int r = r0 + q;
          double acc = sv[q];
#pragma unroll
          for (int q2 = 0; q2 < q; ++q2) acc = fma(ld[q][q2], xq[q2], acc);
          const double v = r < c ? 0.0 : (r == c ? dc : -acc * di[q]);
          if (r > c) M[c * MLD + r] = v;
          xq[q] = v;
        }
      }
      __syncthreads();
    }
  }
  PROF(8)
  if (tid < T) {
    // pivots: log, diagonal, and the NotSpd check, off the serial chain
    const int r = tid;
    const int64_t g = g0 + r;
    const double l = M[r * MLD + r];
    if (!(l > 0.0) && g < m) atomicMin(fail, (unsigned long long)g);
    ell[g] = 2.0 * log(l);
    diag[g] = l;
  }
#pragma unroll 8
  for (int o2 = tid; o2 < TILE_ELEMS / 2; o2 += POTRF_THREADS) {
    const int o = 2 * o2;
    const int r = (o >> 3) & 127;
    const int c = ((o >> 10) << 3) + iperm8(o & 7);
    double2 lv, xv;
    lv.x = c < r ? M[r * MLD + c] : (c == r ? M[r * MLD + r] : 0.0);
    lv.y = c + 4 < r ? M[r * MLD + c + 4] : (c + 4 == r ? M[r * MLD + r] : 0.0);
    xv.x = c < r ? M[c * MLD + r] : (c == r ? dinv[r] : 0.0);
    xv.y = c + 4 < r ? M[(c + 4) * MLD + r] : (c + 4 == r ? dinv[r] : 0.0);
    reinterpret_cast<double2*>(tile)[o2] = lv;
    reinterpret_cast<double2*>(inv)[o2] = xv;
  }
  __syncthreads();
  PROF(9)
#undef PROF
}

// ------------------------------------------------------------------------------ DMMA GEMM

enum { MODE_UPDATE = 0, MODE_TRSM = 1 };

// sign flip on the integer pipe (no FP64 pipe slot)
__device__ __forceinline__ double neg(double x) {
  return __longlong_as_double(__double_as_longlong(x) ^ (long long)0x8000000000000000ULL);
}

struct GemmTask {
  TileMap a, b, c;      // A(i, p), B(j, p), C(i, j); MODE_TRSM: A = C = c at (i, k)
  const double* binv;   // MODE_TRSM: L_kk^{-1} tile (B operand)
  TileSet out;          // output tiles
  int p0, p1;           // K tile-columns (MODE_UPDATE)
  int k;                // MODE_TRSM panel column
};

constexpr int KC = 16;                  // columns per pipeline stage (two octets)
constexpr int STAGE_ELEMS = T * KC;     // 2048 doubles = 16 KB per operand
#ifndef B2D_GEMM_STAGES
#define B2D_GEMM_STAGES 4
#endif
constexpr int STAGES = B2D_GEMM_STAGES;
constexpr int GEMM_THREADS = 288;       // 8 consumer warps + 1 producer warp
#ifndef B2D_RASTER_G
#define B2D_RASTER_G 32  // 8 -> 32: C2 344.2 -> 343.1 ms, C3 2691 -> 2669 ms (A rows re-read once per band)
#endif
constexpr int RASTER_G = B2D_RASTER_G;  // super-tile edge of the CTA raster (tile_order)
constexpr size_t GEMM_SMEM = (size_t)STAGES * 2 * STAGE_ELEMS * 8 + 2 * STAGES * 8 + 128;

template <int MODE>
__global__ void __launch_bounds__(GEMM_THREADS, 1) gemm_kernel(GemmTask t) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* sA = reinterpret_cast<double*>(smem_raw);
  double* sB = sA + STAGES * STAGE_ELEMS;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + STAGES * STAGE_ELEMS);
  uint64_t* empty = full + STAGES;

  // output tile (i, j) of this CTA, in L2-friendly super-tile order
  int i, j;
  tile_order(blockIdx.x, t.out, RASTER_G, &i, &j);
  const int jout = (MODE == MODE_TRSM) ? t.k : j;
  const int nchunks = (MODE == MODE_TRSM) ? (T / KC) : (t.p1 - t.p0) * (T / KC);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // B read in place from other ranks' grids (multi-GPU peer mode): those k-chunks move with
  // 16-byte cp.async by the whole producer warp (plain global loads through the peer aperture),
  // each lane's completion counted on the stage barrier; A (own rows) keeps the bulk copy
  const bool bpeer = MODE == MODE_UPDATE && t.b.npeer > 0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], bpeer ? 33 : 1);
      mbar_init(&empty[s], 8);
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (warp == 8 && bpeer) {
    for (int c = 0; c < nchunks; ++c) {
      const int s = c % STAGES;
      if (c >= STAGES) mbar_wait(&empty[s], ((c / STAGES) - 1) & 1);
      const int p = t.p0 + c / (T / KC);
      const int off = (c % (T / KC)) * STAGE_ELEMS;
      if (lane == 0) {
        mbar_arrive_expect_tx(&full[s], STAGE_ELEMS * 8);
        bulk_g2s(sA + s * STAGE_ELEMS, t.a.tile(i, p) + off, STAGE_ELEMS * 8, &full[s]);
      }
      const double* gb = t.b.tile(j, p) + off;
      const uint32_t sb = smem_u32(sB + s * STAGE_ELEMS);
#pragma unroll 8
      for (int q = lane; q < STAGE_ELEMS / 2; q += 32)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sb + q * 16), "l"(gb + 2 * q) : "memory");
      asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(smem_u32(&full[s])) : "memory");
    }
    asm volatile("cp.async.wait_all;\n" ::: "memory");
    return;
  }
  if (warp == 8) {
    // ---------------- producer: one elected lane streams K-chunks with the bulk-copy engine
    if (lane == 0) {
      for (int c = 0; c < nchunks; ++c) {
        const int s = c % STAGES;
        if (c >= STAGES) mbar_wait(&empty[s], ((c / STAGES) - 1) & 1);
        const double* ga;
        const double* gb;
        if (MODE == MODE_TRSM) {
          ga = t.c.tile(i, t.k) + c * STAGE_ELEMS;
          gb = t.binv + c * STAGE_ELEMS;
        } else {
          const int p = t.p0 + c / (T / KC);
          const int off = (c % (T / KC)) * STAGE_ELEMS;
          ga = t.a.tile(i, p) + off;
          gb = t.b.tile(j, p) + off;
        }
        mbar_arrive_expect_tx(&full[s], 2 * STAGE_ELEMS * 8);
        bulk_g2s(sA + s * STAGE_ELEMS, ga, STAGE_ELEMS * 8, &full[s]);
        bulk_g2s(sB + s * STAGE_ELEMS, gb, STAGE_ELEMS * 8, &full[s]);
      }
    }
    return;
  }

  // ---------------- consumers: 8 warps, warp tile 64 x 32, DMMA m8n8k4
  const int wm = warp >> 2, wn = warp & 3;
  double* C = t.c.tile(i, jout);
  // MODE_UPDATE: the accumulators start as the C tile (64 independent loads issued before the
  // first stage lands, so their latency hides under the pipeline fill) and the B fragments are
  // negated, giving acc = C - A B^T with a store-only epilogue.
  double acc[8][4][2];
#pragma unroll
  for (int g = 0; g < 8; ++g) {
    const int r = wm * 64 + g * 8 + (lane >> 2);
#pragma unroll
    for (int h = 0; h < 4; ++h)
#pragma unroll
      for (int e = 0; e < 2; ++e)
        acc[g][h][e] = (MODE == MODE_UPDATE) ? C[elem(r, wn * 32 + h * 8 + (lane & 3) * 2 + e)] : 0.0;
  }

  const int fr = (lane >> 2) * 8 + (lane & 3) * 2;  // fragment offset inside an octet
  for (int c = 0; c < nchunks; ++c) {
    const int s = c % STAGES;
    mbar_wait(&full[s], (c / STAGES) & 1);
    const double* a_st = sA + s * STAGE_ELEMS + wm * 64 * 8 + fr;
    const double* b_st = sB + s * STAGE_ELEMS + wn * 32 * 8 + fr;
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
      // k-step kk of the chunk: octet kk>>1, half kk&1 of each lane's 16-byte fragment pair.
      // One k-step's 8 A + 4 B fragments stay in registers (168-register cap of a 9-warp CTA)
      // and the 32 DMMAs of a k-step are independent, so dependent DMMAs are 32 issues apart.
      const int off = (kk >> 1) * OCTET_ELEMS + (kk & 1);
      double af[8], bf[4];
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        bf[h] = b_st[off + h * 64];
        if (MODE == MODE_UPDATE) bf[h] = neg(bf[h]);
      }
#pragma unroll
      for (int g = 0; g < 8; ++g) af[g] = a_st[off + g * 64];
#pragma unroll
      for (int g = 0; g < 8; ++g)
#pragma unroll
        for (int h = 0; h < 4; ++h) dmma(acc[g][h][0], acc[g][h][1], af[g], bf[h]);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }

  // ---------------- epilogue: straight to HBM in tile layout
#pragma unroll
  for (int g = 0; g < 8; ++g) {
    const int r = wm * 64 + g * 8 + (lane >> 2);
#pragma unroll
    for (int h = 0; h < 4; ++h)
#pragma unroll
      for (int e = 0; e < 2; ++e) C[elem(r, wn * 32 + h * 8 + (lane & 3) * 2 + e)] = acc[g][h][e];
  }
}

// ------------------------------------------------------------------------------ prefix scan

struct dd { double hi, lo; };
__device__ __forceinline__ dd two_sum(double a, double b) {
  const double s = a + b;
  const double bb = s - a;
  return {s, (a - (s - bb)) + (b - bb)};
}
__device__ __forceinline__ dd dd_add(dd a, dd b) {
  dd s = two_sum(a.hi, b.hi);
  const double e = s.lo + a.lo + b.lo;
  const double h = s.hi + e;
  return {h, e - (h - s.hi)};
}
__device__ __forceinline__ dd dd_add_d(dd a, double b) {
  dd s = two_sum(a.hi, b);
  const double e = s.lo + a.lo;
  const double h = s.hi + e;
  return {h, e - (h - s.hi)};
}

// One CTA: prefix[q] = sum_{g<=q} ell[g] in double-double, rounded once (the reference
// accumulates with a plain sequential np.cumsum, memdet.py:406, 428).
__global__ void __launch_bounds__(1024) prefix_kernel(const double* __restrict__ ell, int64_t n,
                                                      double* __restrict__ prefix) {
  __shared__ double shi[32], slo[32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t chunk = (n + 1023) / 1024;
  const int64_t lo = tid * chunk, hi = min(n, lo + chunk);
  dd run = {0.0, 0.0};
  for (int64_t g = lo; g < hi; ++g) run = dd_add_d(run, ell[g]);
  // inclusive warp scan
  dd inc = run;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    dd o;
    o.hi = __shfl_up_sync(0xffffffffu, inc.hi, off);
    o.lo = __shfl_up_sync(0xffffffffu, inc.lo, off);
    if (lane >= off) inc = dd_add(o, inc);
  }
  if (lane == 31) { shi[warp] = inc.hi; slo[warp] = inc.lo; }
  __syncthreads();
  if (warp == 0) {
    dd w = {shi[lane], slo[lane]};
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      dd o;
      o.hi = __shfl_up_sync(0xffffffffu, w.hi, off);
      o.lo = __shfl_up_sync(0xffffffffu, w.lo, off);
      if (lane >= off) w = dd_add(o, w);
    }
    shi[lane] = w.hi;
    slo[lane] = w.lo;
  }
  __syncthreads();
  dd ex;
  ex.hi = __shfl_up_sync(0xffffffffu, inc.hi, 1);
  ex.lo = __shfl_up_sync(0xffffffffu, inc.lo, 1);
  if (lane == 0) ex = {0.0, 0.0};
  if (warp > 0) ex = dd_add({shi[warp - 1], slo[warp - 1]}, ex);
  for (int64_t g = lo; g < hi; ++g) {
    ex = dd_add_d(ex, ell[g]);
    prefix[g] = ex.hi + ex.lo;
  }
}

// ------------------------------------------------------------------------------ generators

// K_ij = exp(-(sum_c (x_ic - x_jc)^2) / (2 l^2)) + jitter*delta_ij, rows [row0, row0+nrows),
// written row-major with leading dimension n.  Unfused mul/add in coordinate order, the same
// order as the host generator (gen.rbf), so the result is bit-symmetric.
__global__ void gen_rbf_kernel(const double* __restrict__ x, int64_t n, int d, double inv2l2,
                               double jitter, double* __restrict__ out, int64_t row0) {
  const int64_t row = row0 + blockIdx.y;
  const int64_t col = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (col >= n) return;
  double sq = 0.0;
  for (int c = 0; c < d; ++c) {
    const double diff = __dsub_rn(x[row * d + c], x[col * d + c]);
    sq = __dadd_rn(sq, __dmul_rn(diff, diff));
  }
  double v = exp(__dmul_rn(-sq, inv2l2));
  if (row == col) v = __dadd_rn(v, jitter);
  out[(int64_t)blockIdx.y * n + col] = v;
}

}  // namespace b2d

namespace b2d {
// ------------------------------------------------------------------------------ FP64 peak probe
// 16 independent DMMA accumulator chains per warp; every SM busy.  Calibrates the roofline
// denominator (B200 has no FP64 entry in MEASURED_PEAKS.json).
__global__ void __launch_bounds__(256) dmma_probe_kernel(double* out, int iters) {
  const double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[16][2];
#pragma unroll
  for (int i = 0; i < 16; ++i) c[i][0] = c[i][1] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) dmma(c[i][0], c[i][1], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.0) out[threadIdx.x] = s;
}
}  // namespace b2d
