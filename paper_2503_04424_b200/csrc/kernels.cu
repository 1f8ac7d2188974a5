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
template <typename Tin>
__global__ void __launch_bounds__(512) pack_tiles_kernel(const Tin* __restrict__ src, int64_t lda,
                                                         int64_t row_base, int64_t m,
                                                         double* __restrict__ tiles, int nt,
                                                         int j_lo) {
  extern __shared__ double sm[];  // [128][129]: sm[c*129 + r]
  int64_t b = blockIdx.x;
  int J = j_lo;
  while (b >= nt - J) { b -= nt - J; ++J; }
  const int I = J + (int)b;
  const int tid = threadIdx.x;
  const int64_t R0 = (int64_t)I * T, C0 = (int64_t)J * T;
#pragma unroll 4
  for (int idx = tid; idx < TILE_ELEMS; idx += 512) {
    const int c = idx >> 7, r = idx & 127;
    const int64_t R = R0 + r, C = C0 + c;
    double v;
    if (R < m && C < m) v = (double)src[(C - row_base) * lda + R];
    else v = (R == C) ? 1.0 : 0.0;
    sm[c * 129 + r] = v;
  }
  __syncthreads();
  double* out = tiles + tile_index(I, J, nt) * TILE_ELEMS;
#pragma unroll 4
  for (int o = tid; o < TILE_ELEMS; o += 512) {
    const int r = (o >> 3) & 127;
    const int c = ((o >> 10) << 3) + iperm8(o & 7);
    out[o] = sm[c * 129 + r];
  }
}

// ------------------------------------------------------------------------------ potrf + inverse

// One CTA of 128 threads factors diagonal tile (k, k) in shared memory.
// Cholesky: left-looking over 8-column blocks, one thread per row; the 8x8 diagonal block is
// factored warp-synchronously with shuffles.  Then X = L^{-1} in place (row-major, one thread
// per column) and X is written to `inv` in tile layout as the B operand of the panel solve.
// ell[g] = 2*log(L_gg) (the reference's per-row prefix increment, memdet.py:428),
// diag[g] = L_gg; fail = first global row whose pivot is not positive (atomicMin).
__global__ void __launch_bounds__(128) potrf_inv_kernel(double* __restrict__ tiles, int nt, int k,
                                                        double* __restrict__ inv,
                                                        double* __restrict__ ell,
                                                        double* __restrict__ diag,
                                                        unsigned long long* __restrict__ fail,
                                                        int64_t m) {
  extern __shared__ double L[];  // [128][129] row-major: L[r*129 + c]
  __shared__ double dinv[T];
  constexpr int LD = 129;
  const int i = threadIdx.x;  // row owned in the factorization, column owned in the inverse
  const int lane = i & 31, warp = i >> 5;
  const double* tile = tiles + tile_index(k, k, nt) * TILE_ELEMS;
  for (int o = i; o < TILE_ELEMS; o += T) {
    const int r = (o >> 3) & 127;
    const int c = ((o >> 10) << 3) + iperm8(o & 7);
    L[r * LD + c] = tile[o];
  }
  __syncthreads();

  for (int c0 = 0; c0 < T; c0 += 8) {
    double s[8];
    if (i >= c0) {
#pragma unroll
      for (int q = 0; q < 8; ++q) s[q] = L[i * LD + c0 + q];
      for (int p = 0; p < c0; ++p) {
        const double lp = L[i * LD + p];
#pragma unroll
        for (int q = 0; q < 8; ++q) s[q] = fma(-lp, L[(c0 + q) * LD + p], s[q]);
      }
    }
    if (warp == (c0 >> 5)) {
      const int base = c0 & 31;
      const int t = lane - base;  // row within the 8x8 diagonal block if 0 <= t < 8
      const bool mine = (t >= 0 && t < 8);
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const double dq = __shfl_sync(0xffffffffu, s[q], base + q);
        const double lqq = sqrt(dq);
        const double rq = 1.0 / lqq;
        if (mine) {
          if (t == q) {
            const int64_t g = (int64_t)k * T + c0 + q;
            if (!(dq > 0.0) && g < m) atomicMin(fail, (unsigned long long)g);
            s[q] = lqq;
            ell[g] = 2.0 * log(lqq);
            diag[g] = lqq;
            dinv[c0 + q] = rq;
          } else if (t > q) {
            s[q] *= rq;
          }
        }
#pragma unroll
        for (int q2 = q + 1; q2 < 8; ++q2) {
          const double l2 = __shfl_sync(0xffffffffu, s[q], base + q2);
          if (mine && t > q) s[q2] = fma(-s[q], l2, s[q2]);
        }
      }
      if (mine) {
#pragma unroll
        for (int q = 0; q < 8; ++q) L[i * LD + c0 + q] = s[q];
      }
    }
    __syncthreads();
    if (i >= c0 + 8) {
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        double v = s[q];
#pragma unroll
        for (int q2 = 0; q2 < q; ++q2) v = fma(-s[q2], L[(c0 + q) * LD + c0 + q2], v);
        s[q] = v * dinv[c0 + q];
      }
#pragma unroll
      for (int q = 0; q < 8; ++q) L[i * LD + c0 + q] = s[q];
    }
    __syncthreads();
  }

  // L_kk back to its tile (lower triangle, zero upper) so the packed storage holds the factor
  {
    double* out = tiles + tile_index(k, k, nt) * TILE_ELEMS;
    for (int o = i; o < TILE_ELEMS; o += T) {
      const int r = (o >> 3) & 127;
      const int cc = ((o >> 10) << 3) + iperm8(o & 7);
      out[o] = cc <= r ? L[r * LD + cc] : 0.0;
    }
  }
  __syncthreads();

  // In-place inverse, row by row: X[r][c] = -(sum_{p<r} L[r][p] X[p][c]) / L[r][r] (c < r).
  const int c = i;
  const int p_start = warp * 32;  // X[p][c] == 0 for p < c, so a warp may start at its min c
  for (int r = 0; r < T; ++r) {
    double x = 0.0;
    if (c < r) {
      double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
      int p = p_start;
      for (; p + 3 < r; p += 4) {
        a0 = fma(L[r * LD + p], L[p * LD + c], a0);
        a1 = fma(L[r * LD + p + 1], L[(p + 1) * LD + c], a1);
        a2 = fma(L[r * LD + p + 2], L[(p + 2) * LD + c], a2);
        a3 = fma(L[r * LD + p + 3], L[(p + 3) * LD + c], a3);
      }
      for (; p < r; ++p) a0 = fma(L[r * LD + p], L[p * LD + c], a0);
      x = -((a0 + a1) + (a2 + a3)) * dinv[r];
    } else if (c == r) {
      x = dinv[r];
    }
    __syncthreads();
    L[r * LD + c] = x;
    __syncthreads();
  }
  for (int o = i; o < TILE_ELEMS; o += T) {
    const int r = (o >> 3) & 127;
    const int cc = ((o >> 10) << 3) + iperm8(o & 7);
    inv[o] = L[r * LD + cc];
  }
}

// ------------------------------------------------------------------------------ DMMA GEMM

enum { MODE_UPDATE = 0, MODE_TRSM = 1 };

// sign flip on the integer pipe (no FP64 pipe slot)
__device__ __forceinline__ double neg(double x) {
  return __longlong_as_double(__double_as_longlong(x) ^ (long long)0x8000000000000000ULL);
}

struct GemmTask {
  double* tiles;
  const double* binv;  // MODE_TRSM: L_kk^{-1} tile
  int nt;
  int j0, j1;     // output tile-columns [j0, j1)
  int row_off;    // output rows i in [j + row_off, nt)
  int p0, p1;     // K tile-columns (MODE_UPDATE)
  int k;          // MODE_TRSM panel column
};

constexpr int KC = 16;                  // columns per pipeline stage (two octets)
constexpr int STAGE_ELEMS = T * KC;     // 2048 doubles = 16 KB per operand
constexpr int STAGES = 4;
constexpr int GEMM_THREADS = 288;       // 8 consumer warps + 1 producer warp
constexpr size_t GEMM_SMEM = (size_t)STAGES * 2 * STAGE_ELEMS * 8 + 2 * STAGES * 8 + 128;

template <int MODE>
__global__ void __launch_bounds__(GEMM_THREADS, 1) gemm_kernel(GemmTask t) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* sA = reinterpret_cast<double*>(smem_raw);
  double* sB = sA + STAGES * STAGE_ELEMS;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + STAGES * STAGE_ELEMS);
  uint64_t* empty = full + STAGES;

  // decode the output tile (i, j) of this CTA
  int b = blockIdx.x, j = t.j0;
  while (b >= t.nt - j - t.row_off) { b -= t.nt - j - t.row_off; ++j; }
  const int i = j + t.row_off + b;
  const int jout = (MODE == MODE_TRSM) ? t.k : j;
  const int nchunks = (MODE == MODE_TRSM) ? (T / KC) : (t.p1 - t.p0) * (T / KC);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 8);
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (warp == 8) {
    // ---------------- producer: one elected lane streams K-chunks with the bulk-copy engine
    if (lane == 0) {
      for (int c = 0; c < nchunks; ++c) {
        const int s = c % STAGES;
        if (c >= STAGES) mbar_wait(&empty[s], ((c / STAGES) - 1) & 1);
        const double* ga;
        const double* gb;
        if (MODE == MODE_TRSM) {
          ga = t.tiles + tile_index(i, t.k, t.nt) * TILE_ELEMS + c * STAGE_ELEMS;
          gb = t.binv + c * STAGE_ELEMS;
        } else {
          const int p = t.p0 + c / (T / KC);
          const int off = (c % (T / KC)) * STAGE_ELEMS;
          ga = t.tiles + tile_index(i, p, t.nt) * TILE_ELEMS + off;
          gb = t.tiles + tile_index(j, p, t.nt) * TILE_ELEMS + off;
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
  double* C = t.tiles + tile_index(i, jout, t.nt) * TILE_ELEMS;
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
    for (int o = 0; o < 2; ++o) {
      // B fragments for two k-steps stay in registers; A fragments stream one row-group at a
      // time (keeps the live set under the 168-register cap of a 9-warp CTA)
      double2 bf[4];
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        bf[h] = *reinterpret_cast<const double2*>(b_st + o * OCTET_ELEMS + h * 64);
        if (MODE == MODE_UPDATE) { bf[h].x = neg(bf[h].x); bf[h].y = neg(bf[h].y); }
      }
#pragma unroll
      for (int g = 0; g < 8; ++g) {
        const double2 af = *reinterpret_cast<const double2*>(a_st + o * OCTET_ELEMS + g * 64);
#pragma unroll
        for (int h = 0; h < 4; ++h) dmma(acc[g][h][0], acc[g][h][1], af.x, bf[h].x);
#pragma unroll
        for (int h = 0; h < 4; ++h) dmma(acc[g][h][0], acc[g][h][1], af.y, bf[h].y);
      }
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
