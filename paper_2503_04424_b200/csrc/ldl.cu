// Block-pivoted LDL^T kernels (memdet_ldl semantics, reference kernels/_ldl.pyx:21-61 and
// memdet.py:349-371): the diagonal block of each reference stage is factored with 1x1 pivots
// (largest |a_ii| of the trailing diagonal, lowest index on ties, fail below 64*eps*max|A|),
// the row-k blocks are permuted by the block-local permutation, solved with the unit factor,
// and the Schur update runs with one operand scaled by D^{-1}.
//
//   unpack_block_kernel    tile grid -> dense column-major block (lower triangle)
//   block_absmax_kernel    max |a_ij| over the block's lower triangle (the tolerance scale)
//   ldl_pivot_kernel       cooperative, one column per step: grid-wide argmax, symmetric swap,
//                          rank-1 trailing update (the reference's a_ij -= c_i * (c_j / p))
//   ldl_finish_kernel      swaps -> permutation, log|d|, d, global perm
//   pack_unit_lower_kernel dense unit-lower L -> tile grid
//   tile_inv_unit_kernel   inverse of a unit-lower 128 x 128 tile (TRSM operand)
//   permute_cols_kernel    panel block columns by the block permutation (rows of B in the ref)
//   scale_cols_kernel      panel block columns / d (B /= d, memdet.py:371)
#include <cooperative_groups.h>

#include "tile.cuh"

namespace b2d {
namespace cg = cooperative_groups;

__global__ void __launch_bounds__(256) unpack_block_kernel(TileMap src, int ntiles, double* __restrict__ dense,
                                                           int64_t ld) {
  __shared__ double sm[32][129];
  int I, J;
  const TileSet all{0, ntiles, 0, ntiles, 1, 0, 0, 0};
  tile_order(blockIdx.x, all, 1, &I, &J);
  const double* t = src.tile(I, J);
  for (int qtr = 0; qtr < 4; ++qtr) {
    // columns 32*qtr .. 32*qtr+31 of the tile = octets 4*qtr .. 4*qtr+3 (contiguous)
    for (int o = threadIdx.x; o < 32 * T; o += 256) {
      const int r = (o >> 3) & 127;
      const int c = ((o >> 10) << 3) + iperm8(o & 7);
      sm[c][r] = t[qtr * 32 * T + o];
    }
    __syncthreads();
    for (int idx = threadIdx.x; idx < 32 * T; idx += 256) {
      const int c = idx >> 7, r = idx & 127;
      dense[(int64_t)(J * T + 32 * qtr + c) * ld + I * T + r] = sm[c][r];
    }
    __syncthreads();
  }
}

__global__ void block_absmax_kernel(const double* __restrict__ dense, int64_t ld, int64_t n,
                                    unsigned long long* __restrict__ amax_bits) {
  double best = 0.0;
  const int64_t total = n * n;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = e / n, i = e % n;
    if (i >= j) best = fmax(best, fabs(dense[j * ld + i]));
  }
  for (int off = 16; off; off >>= 1) best = fmax(best, __shfl_xor_sync(0xffffffffu, best, off));
  // non-negative doubles order like their bit patterns
  if ((threadIdx.x & 31) == 0) atomicMax(amax_bits, (unsigned long long)__double_as_longlong(best));
}

struct ArgMax {
  double v;
  int64_t i;
};
__device__ __forceinline__ ArgMax better(ArgMax a, ArgMax b) {
  // larger |value| wins; ties go to the lower index (the reference's "first max", _ldl.pyx:31-36)
  if (b.v > a.v || (b.v == a.v && b.i < a.i)) return b;
  return a;
}
__device__ __forceinline__ ArgMax warp_argmax(ArgMax a) {
  for (int off = 16; off; off >>= 1) {
    ArgMax o{__shfl_xor_sync(0xffffffffu, a.v, off), __shfl_xor_sync(0xffffffffu, a.i, off)};
    a = better(a, o);
  }
  return a;
}

constexpr int LDL_THREADS = 256;

// Dense column-major block A (ld), valid order n; factored in place: strictly lower = unit L,
// d = pivots, swaps = LAPACK-style swap list.  tol = 64 * eps * amax (amax_bits holds the bits of
// max |a|).  *fail = g0 + first failing step (atomicMin), and the kernel stops there.
__global__ void __launch_bounds__(LDL_THREADS) ldl_pivot_kernel(double* __restrict__ A, int64_t ld, int64_t n,
                                                                const unsigned long long* __restrict__ amax_bits,
                                                                double* __restrict__ d, int64_t* __restrict__ swaps,
                                                                ArgMax* __restrict__ part,
                                                                unsigned long long* __restrict__ fail, int64_t g0) {
  cg::grid_group grid = cg::this_grid();
  __shared__ ArgMax sred[LDL_THREADS / 32];
  __shared__ int64_t s_t;
  const int tid = threadIdx.x, lane = tid & 31, wib = tid >> 5;
  const int64_t gtid = (int64_t)blockIdx.x * LDL_THREADS + tid;
  const int64_t gthreads = (int64_t)gridDim.x * LDL_THREADS;
  const int64_t gwarp = gtid >> 5, nwarps = gthreads >> 5;
  const double tol = 64.0 * 2.220446049250313e-16 * __longlong_as_double((long long)*amax_bits);
  auto block_argmax = [&](ArgMax a) {
    a = warp_argmax(a);
    if (lane == 0) sred[wib] = a;
    __syncthreads();
    if (wib == 0) {
      ArgMax b = lane < LDL_THREADS / 32 ? sred[lane] : ArgMax{-1.0, INT64_MAX};
      b = warp_argmax(b);
      if (lane == 0) part[blockIdx.x] = b;
    }
    __syncthreads();
  };
  // initial pivot candidates
  {
    ArgMax a{-1.0, INT64_MAX};
    for (int64_t i = gtid; i < n; i += gthreads) a = better(a, ArgMax{fabs(A[i * ld + i]), i});
    block_argmax(a);
  }
  grid.sync();
  // Two grid barriers per column: S(r) finishes column r-1 (L = c / p) while swapping r <-> t,
  // U(r) checks the pivot and applies the rank-1 update with the unscaled column r.
  for (int64_t r = 0; r < n; ++r) {
    // --- S: pivot t = argmax over the partials, symmetric swap r <-> t (_ldl.pyx:38-46)
    if (wib == 0) {
      ArgMax b{-1.0, INT64_MAX};
      for (int q = lane; q < (int)gridDim.x; q += 32) b = better(b, part[q]);
      b = warp_argmax(b);
      if (lane == 0) s_t = b.i;
    }
    __syncthreads();
    const int64_t t = s_t;
    if (gtid == 0) swaps[r] = t;
    const int64_t q = r - 1;                       // column finished in this phase
    const double invq = q >= 0 ? 1.0 / d[q] : 1.0;  // d[q] written by gtid 0 in U(q), visible after the sync
    if (q >= 0) {
      // a_iq = a_iq * (1/p) for i > q (_ldl.pyx:59-60), rows r and t via the swap below
      for (int64_t i = q + 1 + gtid; i < n; i += gthreads)
        if (i != r && i != t) A[q * ld + i] = __dmul_rn(A[q * ld + i], invq);
    }
    if (t != r) {
      for (int64_t j = gtid; j < r; j += gthreads) {  // rows r and t of the L part
        double x = A[j * ld + r], y = A[j * ld + t];
        if (j == q) {
          x = __dmul_rn(x, invq);
          y = __dmul_rn(y, invq);
        }
        A[j * ld + r] = y;
        A[j * ld + t] = x;
      }
      if (gtid == 0) {
        const double x = A[r * ld + r];
        A[r * ld + r] = A[t * ld + t];
        A[t * ld + t] = x;
      }
      for (int64_t i = r + 1 + gtid; i < t; i += gthreads) {  // column r below r <-> row t
        const double x = A[r * ld + i];
        A[r * ld + i] = A[i * ld + t];
        A[i * ld + t] = x;
      }
      for (int64_t i = t + 1 + gtid; i < n; i += gthreads) {  // below t: columns r and t
        const double x = A[r * ld + i];
        A[r * ld + i] = A[t * ld + i];
        A[t * ld + i] = x;
      }
    } else if (q >= 0 && gtid == 0) {
      A[q * ld + r] = __dmul_rn(A[q * ld + r], invq);
    }
    grid.sync();
    // --- U: pivot check, rank-1 update of the trailing lower triangle, next candidates
    const double p = A[r * ld + r];
    if (!(fabs(p) >= tol)) {
      if (gtid == 0) atomicMin(fail, (unsigned long long)(g0 + r));
      return;  // uniform: every thread read the same p
    }
    if (gtid == 0) d[r] = p;
    const double invp = 1.0 / p;
    ArgMax cand{-1.0, INT64_MAX};
    for (int64_t j = r + 1 + gwarp; j < n; j += nwarps) {
      const double wj = __dmul_rn(A[r * ld + j], invp);  // work[j] = a_jr * (1/p)
      double* colj = A + j * ld;
      const double* colr = A + r * ld;
      for (int64_t i = j + lane; i < n; i += 32) colj[i] = __dsub_rn(colj[i], __dmul_rn(colr[i], wj));
      if (lane == 0) cand = better(cand, ArgMax{fabs(colj[j]), j});
    }
    block_argmax(cand);
    grid.sync();
  }
  // the last column has no rows below it; column n-2 was finished in S(n-1)
}

// swaps -> block permutation (kernels/dense.py:25-30), global perm (memdet.py:352-353),
// ell = log|d| (memdet.py:406) and the D values; one thread walks the swaps, all fill the rest.
__global__ void ldl_finish_kernel(const int64_t* __restrict__ swaps, const double* __restrict__ d, int64_t n,
                                  int64_t g0, int64_t* __restrict__ perm_local, int64_t* __restrict__ perm_global,
                                  double* __restrict__ ell, double* __restrict__ dout) {
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    for (int64_t i = 0; i < n; ++i) perm_local[i] = i;
    for (int64_t r = 0; r < n; ++r) {
      const int64_t t = swaps[r];
      if (t != r) {
        const int64_t x = perm_local[r];
        perm_local[r] = perm_local[t];
        perm_local[t] = x;
      }
    }
    for (int64_t i = 0; i < n; ++i) perm_global[g0 + i] = g0 + perm_local[i];
  }
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    ell[g0 + i] = log(fabs(d[i]));
    dout[g0 + i] = d[i];
  }
}

// Dense unit-lower factor -> tile grid (identity padding beyond n; upper tiles untouched).
__global__ void __launch_bounds__(256) pack_unit_lower_kernel(const double* __restrict__ dense, int64_t ld,
                                                              int64_t n, TileMap dst, int ntiles) {
  int I, J;
  const TileSet all{0, ntiles, 0, ntiles, 1, 0, 0, 0};
  tile_order(blockIdx.x, all, 1, &I, &J);
  double* t = dst.tile(I, J);
  for (int o = threadIdx.x; o < TILE_ELEMS; o += 256) {
    const int r = (o >> 3) & 127;
    const int c = ((o >> 10) << 3) + iperm8(o & 7);
    const int64_t R = (int64_t)I * T + r, C = (int64_t)J * T + c;
    double v;
    if (R == C) v = 1.0;
    else if (R > C && R < n) v = dense[C * ld + R];
    else v = 0.0;
    t[o] = v;
  }
}

// X = L^{-1} of a unit-lower 128 x 128 tile: one thread per column, forward substitution in
// 8-row blocks; X[r][c] (r > c) kept transposed in the upper triangle of the staging array.
__global__ void __launch_bounds__(128) tile_inv_unit_kernel(const double* __restrict__ tile, double* __restrict__ inv) {
  extern __shared__ double M[];  // [T][129]
  const int c = threadIdx.x;
  for (int o = c; o < TILE_ELEMS; o += T) {
    const int r = (o >> 3) & 127;
    const int cc = ((o >> 10) << 3) + iperm8(o & 7);
    if (cc < r) M[r * 129 + cc] = tile[o];
  }
  __syncthreads();
  // X[r][c] = -sum_{c <= p < r} L[r][p] X[p][c], X[c][c] = 1
  for (int r = c + 1; r < T; ++r) {
    double acc = M[r * 129 + c];  // p = c term, X[c][c] = 1
    for (int p = c + 1; p < r; ++p) acc = fma(M[r * 129 + p], M[c * 129 + p], acc);
    M[c * 129 + r] = -acc;
  }
  __syncthreads();
  for (int o = c; o < TILE_ELEMS; o += T) {
    const int r = (o >> 3) & 127;
    const int cc = ((o >> 10) << 3) + iperm8(o & 7);
    inv[o] = cc < r ? M[cc * 129 + r] : (cc == r ? 1.0 : 0.0);
  }
}

// dst(i, c) = src(i, perm[c]) for c < n (columns of a panel block = rows of the reference's
// row-k tile, memdet.py:365-366, 378-379); padding columns copied as they are.
__global__ void permute_cols_kernel(TileMap src, TileMap dst, int rtiles, int ctiles, int64_t n,
                                    const int64_t* __restrict__ perm) {
  const int64_t rows = (int64_t)rtiles * T, cols = (int64_t)ctiles * T;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < rows * cols; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = e / rows, i = e % rows;
    const int64_t sc = c < n ? perm[c] : c;
    const double v = src.tile((int)(i / T), (int)(sc / T))[elem((int)(i % T), (int)(sc % T))];
    dst.tile((int)(i / T), (int)(c / T))[elem((int)(i % T), (int)(c % T))] = v;
  }
}

// dst(i, c) = src(i, c) / d[c] for c < n (B /= d, memdet.py:371); padding copied.
__global__ void scale_cols_kernel(TileMap src, TileMap dst, int rtiles, int ctiles, int64_t n,
                                  const double* __restrict__ d) {
  const int64_t rows = (int64_t)rtiles * T, cols = (int64_t)ctiles * T;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < rows * cols; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = e / rows, i = e % rows;
    const int off = elem((int)(i % T), (int)(c % T));
    const double v = src.tile((int)(i / T), (int)(c / T))[off];
    dst.tile((int)(i / T), (int)(c / T))[off] = c < n ? v / d[c] : v;
  }
}

}  // namespace b2d
