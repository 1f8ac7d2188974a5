// Block-pivoted LDL^T kernels (memdet_ldl semantics, reference kernels/_ldl.pyx:21-61 and
// memdet.py:349-371): the diagonal block of each reference stage is factored with 1x1 pivots
// (largest |a_ii| of the trailing diagonal, lowest index on ties, fail below 64*eps*max|A|),
// the row-k blocks are permuted by the block-local permutation, solved with the unit factor,
// and the Schur update runs with one operand scaled by D^{-1}.
//
//   unpack_block_kernel    tile grid -> dense column-major block (lower triangle)
//   block_absmax_kernel    max |a_ij| over the block's lower triangle (the tolerance scale)
//   ldl_panel_kernel       NB pivot steps in one CTA: argmax of the eager diagonal (lowest index
//                          on ties), symmetric interchange, pivot column with pending terms
//   ldl_bulk_kernel        the panel's NB steps applied to the trailing matrix (the reference's
//                          a_ij -= c_i * (c_j / p), same order and roundings)
//   ldl_finish_kernel      swaps -> permutation, log|d|, d, global perm
//   pack_unit_lower_kernel dense unit-lower L -> tile grid
//   tile_inv_unit_kernel   inverse of a unit-lower 128 x 128 tile (TRSM operand)
//   permute_cols_kernel    panel block columns by the block permutation (rows of B in the ref)
//   scale_cols_kernel      panel block columns / d (B /= d, memdet.py:371)
#include <cooperative_groups.h>

#include "tile.cuh"

namespace b2d {
namespace cg = cooperative_groups;

// lower = 1: the lower tile triangle (symmetric blocks); 0: every tile (generic blocks).
__global__ void __launch_bounds__(256) unpack_block_kernel(TileMap src, int ntiles, double* __restrict__ dense,
                                                           int64_t ld, int lower) {
  __shared__ double sm[32][129];
  int I, J;
  const TileSet all{0, ntiles, 0, ntiles, lower, 0, 0, 0};
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

// ---------------------------------------------------------------------------------------------
// Pivoted LDL^T of a dense column-major block, blocked with delayed updates and bit-identical to
// the reference's unblocked loop (_ldl.pyx:21-61; oracle/ldl_tile.c).
//
// The reference applies, at step q, a_ij -= c_i * w_j (c = the updated column q, w = c / p_q)
// to every trailing element, one step at a time.  Here the steps of a block of NB columns are
// kept as columns of C (c) and W (w) and applied to the trailing matrix once per block, in the
// same order and with the same two roundings per term, by ldl_bulk_kernel.  In between, a
// panel kernel (one CTA) runs the NB pivot steps:
//   * pivot search over an eagerly updated copy of the diagonal (diag_i -= c_i w_i per step is
//     exactly the reference's update of a_ii);
//   * the pivot column is computed from the raw (not yet updated) entries plus their pending
//     terms, each with the association of the position it held (row index -> C, column index -> W);
//   * the symmetric interchange moves raw entries with their pending terms.  The interchange
//     moves entries of column r into row t (r < i < t), where the pending terms would change
//     association (c_t w_i vs c_i w_t, equal in exact arithmetic, not in floating point); those
//     entries are brought up to date at the move and carry a tag = number of the block's steps
//     already applied, which the bulk update and later column computations honour.
// Every entry therefore sees the reference's sequence of roundings, and the pivot order, D and L
// are bit-identical to the unblocked kernel.
constexpr int LDL_NB = 32;             // steps per panel (columns of C / W)
constexpr int LDL_PANEL_THREADS = 1024;

struct LdlArgs {
  double* A;      // dense block, column-major, leading dimension ld
  uint8_t* tag;   // per-entry count of this panel's steps already applied (same layout as A)
  double* C;      // [LDL_NB][ld] unscaled pivot columns of the current panel
  double* W;      // [LDL_NB][ld] scaled pivot columns (c / p)
  double* diag;   // eagerly updated diagonal
  double* col;    // scratch: the pivot column being formed
  double* d;      // pivots
  int64_t* swaps; // LAPACK-style interchanges (block-local)
  unsigned long long* fail;
  const unsigned long long* amax_bits;
  int64_t ld, n, g0;
};

__global__ void ldl_diag_init_kernel(LdlArgs g) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < g.n; i += (int64_t)gridDim.x * blockDim.x)
    g.diag[i] = g.A[i * g.ld + i];
}

// One panel of nbk pivot steps starting at r0 (one CTA).
__global__ void __launch_bounds__(LDL_PANEL_THREADS, 1) ldl_panel_kernel(LdlArgs g, int64_t r0, int nbk) {
  if (*g.fail != ~0ull) return;  // an earlier step failed
  __shared__ ArgMax sred[LDL_PANEL_THREADS / 32];
  __shared__ int64_t s_t;
  const int tid = threadIdx.x, lane = tid & 31, wib = tid >> 5;
  const int64_t n = g.n, ld = g.ld;
  double* __restrict__ A = g.A;
  uint8_t* __restrict__ tag = g.tag;
  const double* __restrict__ C = g.C;
  const double* __restrict__ W = g.W;
  const double tol = 64.0 * 2.220446049250313e-16 * __longlong_as_double((long long)*g.amax_bits);
  // entry (row, col) brought up to date with the panel's steps [tag, k) in its own association
  auto upd = [&](int64_t row, int64_t col, int k) {
    double v = A[col * ld + row];
    for (int q = tag[col * ld + row]; q < k; ++q) v = __dsub_rn(v, __dmul_rn(C[q * ld + row], W[q * ld + col]));
    return v;
  };
  for (int k = 0; k < nbk; ++k) {
    const int64_t r = r0 + k;
    // pivot: largest |diag| over [r, n), lowest index on ties (_ldl.pyx:30-36)
    ArgMax a{-1.0, INT64_MAX};
    for (int64_t i = r + tid; i < n; i += LDL_PANEL_THREADS) a = better(a, ArgMax{fabs(g.diag[i]), i});
    a = warp_argmax(a);
    if (lane == 0) sred[wib] = a;
    __syncthreads();
    if (wib == 0) {
      ArgMax b = sred[lane];
      b = warp_argmax(b);
      if (lane == 0) s_t = b.i;
    }
    __syncthreads();
    const int64_t t = s_t;
    // interchange r <-> t (_ldl.pyx:38-46) and the new column r, from the pre-interchange entries
    for (int64_t i = r + 1 + tid; i < n; i += LDL_PANEL_THREADS) {
      double v;
      if (t == r) {
        v = upd(i, r, k);
      } else if (i < t) {
        v = upd(t, i, k);                      // (t, i) -> (i, r)
        A[i * ld + t] = upd(i, r, k);          // (i, r) -> (t, i), association changes: bring up to date
        tag[i * ld + t] = (uint8_t)k;
      } else if (i == t) {
        v = upd(t, r, k);                      // (t, r) stays
      } else {
        v = upd(i, t, k);                      // (i, t) -> (i, r)
        A[t * ld + i] = A[r * ld + i];         // (i, r) -> (i, t), same association: move raw + tag
        tag[t * ld + i] = tag[r * ld + i];
      }
      g.col[i] = v;
    }
    if (t != r)
      for (int64_t j = tid; j < r0; j += LDL_PANEL_THREADS) {  // rows r, t of the finished L columns
        const double x = A[j * ld + r];
        A[j * ld + r] = A[j * ld + t];
        A[j * ld + t] = x;
      }
    __syncthreads();
    if (t != r) {
      for (int q = tid; q < 2 * k; q += LDL_PANEL_THREADS) {  // rows r, t of this panel's C / W
        double* B = (q & 1) ? g.W : g.C;
        const int qq = q >> 1;
        const double x = B[qq * ld + r];
        B[qq * ld + r] = B[qq * ld + t];
        B[qq * ld + t] = x;
      }
      if (tid == 0) {
        const double x = g.diag[r];
        g.diag[r] = g.diag[t];
        g.diag[t] = x;
        A[t * ld + t] = A[r * ld + r];  // (r, r) -> (t, t) with its pending terms
        tag[t * ld + t] = tag[r * ld + r];
      }
    }
    if (tid == 0) g.swaps[r] = t;
    __syncthreads();
    const double p = g.diag[r];
    if (!(fabs(p) >= tol)) {
      if (tid == 0) atomicMin(g.fail, (unsigned long long)(g.g0 + r));
      return;  // uniform: every thread read the same p
    }
    if (tid == 0) g.d[r] = p;
    const double invp = 1.0 / p;
    for (int64_t i = r + 1 + tid; i < n; i += LDL_PANEL_THREADS) {
      const double c = g.col[i];
      const double w = __dmul_rn(c, invp);  // work[i] = a_ir * (1/p)
      g.C[k * ld + i] = c;
      g.W[k * ld + i] = w;
      g.diag[i] = __dsub_rn(g.diag[i], __dmul_rn(c, w));
    }
    __syncthreads();
  }
}

// The same panel on a cluster of LC CTAs (one per SM) with the panel's C / W rows, the eager
// diagonal and the pivot column in distributed shared memory: row i lives in CTA i % LC at
// local row i / LC.  Per step: local argmax -> candidates pushed to every CTA -> barrier ->
// every CTA reads rows r and t (C, W, diag) from their owners -> barrier -> local rows of the
// new column, interchange, update.  Entry arithmetic is the single-CTA kernel's exactly.
// Raw entries and tags stay in global memory (read through L2: other CTAs wrote them).
constexpr int LC = 16;                 // CTAs per cluster (non-portable size)
constexpr int LC_THREADS = 256;
constexpr int LC_LD = LDL_NB + 1;      // padded smem row (conflict-free column access)
constexpr int LC_RMAX = 384;           // local rows per CTA (n <= LC * LC_RMAX)
__host__ __device__ constexpr size_t ldl_cluster_smem(int rows) { return (size_t)rows * (2 * LC_LD + 2) * 8; }

__global__ void __launch_bounds__(LC_THREADS, 1) ldl_panel_cluster_kernel(LdlArgs g, int64_t r0, int nbk) {
  if (*g.fail != ~0ull) return;  // uniform: written by earlier kernels only
  cg::cluster_group cl = cg::this_cluster();
  const int c = (int)cl.block_rank();
  extern __shared__ double sm[];
  const int64_t n = g.n, ld = g.ld;
  const int R = (int)((n + LC - 1) / LC);
  double* Cs = sm;                      // [R][LC_LD]
  double* Ws = Cs + (size_t)R * LC_LD;  // [R][LC_LD]
  double* dg = Ws + (size_t)R * LC_LD;  // [R] eager diagonal
  double* col = dg + R;                 // [R] pivot column being formed
  __shared__ ArgMax cand[2][LC];
  __shared__ ArgMax sred[LC_THREADS / 32];
  __shared__ double bCr[LDL_NB], bWr[LDL_NB], bCt[LDL_NB], bWt[LDL_NB], bd[2];
  const int tid = threadIdx.x, lane = tid & 31, wib = tid >> 5;
  double* __restrict__ A = g.A;
  uint8_t* __restrict__ tag = g.tag;
  const double tol = 64.0 * 2.220446049250313e-16 * __longlong_as_double((long long)*g.amax_bits);
  for (int li = tid; li < R; li += LC_THREADS) {
    const int64_t i = (int64_t)li * LC + c;
    dg[li] = i < n ? g.diag[i] : 0.0;
  }
  // (row, col) up to date with steps [tag, k): cr = C row of `row`, wc = W row of `col`
  // raw entry v with pending steps [tg, k) applied: cr = C row of its row, wc = W row of its column
  auto chain = [&](double v, int tg, const double* cr, const double* wc, int k) {
    for (int q = tg; q < k; ++q) v = __dsub_rn(v, __dmul_rn(cr[q], wc[q]));
    return v;
  };
  for (int k = 0; k < nbk; ++k) {
    const int64_t r = r0 + k;
    ArgMax a{-1.0, INT64_MAX};
    for (int li = tid; li < R; li += LC_THREADS) {
      const int64_t i = (int64_t)li * LC + c;
      if (i >= r && i < n) a = better(a, ArgMax{fabs(dg[li]), i});
    }
    a = warp_argmax(a);
    if (lane == 0) sred[wib] = a;
    __syncthreads();
    if (wib == 0) {
      ArgMax b = lane < LC_THREADS / 32 ? sred[lane] : ArgMax{-1.0, INT64_MAX};
      b = warp_argmax(b);
      if (lane < LC) *cl.map_shared_rank(&cand[k & 1][c], lane) = b;  // push to every CTA
    }
    cl.sync();  // A: candidates (and the previous step's rows) visible cluster-wide
    ArgMax b{-1.0, INT64_MAX};
    for (int q = 0; q < LC; ++q) b = better(b, cand[k & 1][q]);
    const int64_t t = b.i;
    const int orr = (int)(r % LC), ort = (int)(t % LC);
    const int lr = (int)(r / LC), lt = (int)(t / LC);
    for (int q = tid; q < k; q += LC_THREADS) {
      bCr[q] = cl.map_shared_rank(Cs, orr)[(size_t)lr * LC_LD + q];
      bWr[q] = cl.map_shared_rank(Ws, orr)[(size_t)lr * LC_LD + q];
      bCt[q] = cl.map_shared_rank(Cs, ort)[(size_t)lt * LC_LD + q];
      bWt[q] = cl.map_shared_rank(Ws, ort)[(size_t)lt * LC_LD + q];
    }
    if (tid == 0) {
      bd[0] = cl.map_shared_rank(dg, orr)[lr];
      bd[1] = cl.map_shared_rank(dg, ort)[lt];
    }
    cl.sync();  // B: rows r, t read everywhere; their owners may overwrite them
    for (int li = tid; li < R; li += LC_THREADS) {
      const int64_t i = (int64_t)li * LC + c;
      if (i <= r || i >= n) continue;
      const double* Ci = Cs + (size_t)li * LC_LD;
      const double* Wi = Ws + (size_t)li * LC_LD;
      // every raw entry and tag this row needs is loaded before any chain runs (one L2 round)
      double v;
      if (t == r) {
        const double a0 = __ldcg(A + r * ld + i);
        const int g0 = __ldcg(tag + r * ld + i);
        v = chain(a0, g0, Ci, bWr, k);
      } else if (i < t) {
        const double a0 = __ldcg(A + i * ld + t), a1 = __ldcg(A + r * ld + i);
        const int g0 = __ldcg(tag + i * ld + t), g1 = __ldcg(tag + r * ld + i);
        v = chain(a0, g0, bCt, Wi, k);        // (t, i) -> (i, r)
        A[i * ld + t] = chain(a1, g1, Ci, bWr, k);  // (i, r) -> (t, i): brought up to date, tagged
        tag[i * ld + t] = (uint8_t)k;
      } else if (i == t) {
        const double a0 = __ldcg(A + r * ld + t), ad = __ldcg(A + r * ld + r);
        const int g0 = __ldcg(tag + r * ld + t), gd = __ldcg(tag + r * ld + r);
        v = chain(a0, g0, bCt, bWr, k);       // (t, r) stays
        A[t * ld + t] = ad;                   // (r, r) -> (t, t) with its pending terms
        tag[t * ld + t] = (uint8_t)gd;
      } else {
        const double a0 = __ldcg(A + t * ld + i), a1 = __ldcg(A + r * ld + i);
        const int g0 = __ldcg(tag + t * ld + i), g1 = __ldcg(tag + r * ld + i);
        v = chain(a0, g0, Ci, bWt, k);        // (i, t) -> (i, r)
        A[t * ld + i] = a1;                   // (i, r) -> (i, t) with its tag
        tag[t * ld + i] = (uint8_t)g1;
      }
      col[li] = v;
    }
    if (t != r)
      for (int64_t j = (int64_t)c * LC_THREADS + tid; j < r0; j += (int64_t)LC * LC_THREADS) {
        const double x = __ldcg(A + j * ld + r);
        A[j * ld + r] = __ldcg(A + j * ld + t);
        A[j * ld + t] = x;
      }
    __syncthreads();
    if (t != r) {
      if (c == orr) {
        for (int q = tid; q < k; q += LC_THREADS) {
          Cs[(size_t)lr * LC_LD + q] = bCt[q];
          Ws[(size_t)lr * LC_LD + q] = bWt[q];
        }
        if (tid == 0) dg[lr] = bd[1];
      }
      if (c == ort) {
        for (int q = tid; q < k; q += LC_THREADS) {
          Cs[(size_t)lt * LC_LD + q] = bCr[q];
          Ws[(size_t)lt * LC_LD + q] = bWr[q];
        }
        if (tid == 0) dg[lt] = bd[0];  // (the raw (r, r) -> (t, t) move is in the row loop above)
      }
    }
    const double p = t == r ? bd[0] : bd[1];
    if (!(fabs(p) >= tol)) {
      if (c == 0 && tid == 0) atomicMin(g.fail, (unsigned long long)(g.g0 + r));
      return;  // uniform across the cluster: every thread read the same p
    }
    if (c == 0 && tid == 0) {
      g.d[r] = p;
      g.swaps[r] = t;
    }
    const double invp = 1.0 / p;
    __syncthreads();
    for (int li = tid; li < R; li += LC_THREADS) {
      const int64_t i = (int64_t)li * LC + c;
      if (i <= r || i >= n) continue;
      const double cv = col[li];
      const double w = __dmul_rn(cv, invp);  // work[i] = a_ir * (1/p)
      Cs[(size_t)li * LC_LD + k] = cv;
      Ws[(size_t)li * LC_LD + k] = w;
      dg[li] = __dsub_rn(dg[li], __dmul_rn(cv, w));
    }
    __syncthreads();
  }
  // C, W and the diagonal back to global memory for the bulk update and the next panel
  for (int li = tid; li < R; li += LC_THREADS) {
    const int64_t i = (int64_t)li * LC + c;
    if (i >= n || i <= r0) continue;
    for (int q = 0; q < nbk; ++q) {
      g.C[q * ld + i] = Cs[(size_t)li * LC_LD + q];
      g.W[q * ld + i] = Ws[(size_t)li * LC_LD + q];
    }
    g.diag[i] = dg[li];
  }
}

// Finished columns [r0, r0 + nbk): L = W below the diagonal (_ldl.pyx:59-60).
__global__ void ldl_store_l_kernel(LdlArgs g, int64_t r0, int nbk) {
  if (*g.fail != ~0ull) return;
  const int64_t rows = g.n - r0;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < rows * nbk; e += (int64_t)gridDim.x * blockDim.x) {
    const int k = (int)(e / rows);
    const int64_t i = r0 + e % rows, r = r0 + k;
    if (i > r) g.A[r * g.ld + i] = g.W[k * g.ld + i];
  }
}

// Trailing update with the panel's nbk steps: a_ij -= c_i^q w_j^q for q = tag_ij .. nbk-1, in
// order, for j >= r0 + nbk, i >= j; tags reset.  64 x 64 entry tiles, 4 x 4 per thread.
constexpr int LDL_BT = 64;
__global__ void __launch_bounds__(256) ldl_bulk_kernel(LdlArgs g, int64_t r0, int nbk) {
  if (*g.fail != ~0ull) return;
  __shared__ double sC[LDL_NB][LDL_BT], sW[LDL_NB][LDL_BT];
  const int64_t re = r0 + nbk, m = g.n - re, ld = g.ld;
  // lower-triangular tile (bi >= bj) of blockIdx.x
  int64_t b = blockIdx.x, bj = 0;
  const int64_t nbt = (m + LDL_BT - 1) / LDL_BT;
  while (b >= nbt - bj) { b -= nbt - bj; ++bj; }
  const int64_t bi = bj + b;
  const int64_t i0 = re + bi * LDL_BT, j0 = re + bj * LDL_BT;
  for (int e = threadIdx.x; e < nbk * LDL_BT; e += 256) {
    const int q = e / LDL_BT, x = e % LDL_BT;
    sC[q][x] = i0 + x < g.n ? g.C[q * ld + i0 + x] : 0.0;
    sW[q][x] = j0 + x < g.n ? g.W[q * ld + j0 + x] : 0.0;
  }
  __syncthreads();
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  double v[4][4];
  int tg[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int64_t i = i0 + tx + 16 * a, j = j0 + ty + 16 * c;
      const bool ok = i < g.n && j < g.n && i >= j;
      v[a][c] = ok ? g.A[j * ld + i] : 0.0;
      tg[a][c] = ok ? g.tag[j * ld + i] : 255;
    }
  for (int q = 0; q < nbk; ++q) {
    double cc[4], ww[4];
#pragma unroll
    for (int a = 0; a < 4; ++a) cc[a] = sC[q][tx + 16 * a];
#pragma unroll
    for (int c = 0; c < 4; ++c) ww[c] = sW[q][ty + 16 * c];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int c = 0; c < 4; ++c)
        if (q >= tg[a][c]) v[a][c] = __dsub_rn(v[a][c], __dmul_rn(cc[a], ww[c]));
  }
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int64_t i = i0 + tx + 16 * a, j = j0 + ty + 16 * c;
      if (i < g.n && j < g.n && i >= j) {
        g.A[j * ld + i] = v[a][c];
        if (tg[a][c]) g.tag[j * ld + i] = 0;
      }
    }
}

// swaps -> block permutation (kernels/dense.py:25-30), global perm (memdet.py:352-353),
// ell = log|d| (memdet.py:406) and the D values.  One thread walks the swaps (sequential by
// definition) on a shared-memory copy of the permutation when it fits (LDL_FINISH_SMEM_MAX rows).
constexpr int64_t LDL_FINISH_SMEM_MAX = 24576;
__global__ void ldl_finish_kernel(const int64_t* __restrict__ swaps, const double* __restrict__ d, int64_t n,
                                  int64_t g0, int64_t* __restrict__ perm_local, int64_t* __restrict__ perm_global,
                                  double* __restrict__ ell, double* __restrict__ dout) {
  extern __shared__ int64_t sperm[];
  if (blockIdx.x == 0) {
    const bool sm = n <= LDL_FINISH_SMEM_MAX;
    int64_t* pl = sm ? sperm : perm_local;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) pl[i] = i;
    __syncthreads();
    auto walk = [&](int64_t* __restrict__ q) {
      for (int64_t r = 0; r < n; ++r) {
        const int64_t t = __ldg(swaps + r);
        if (t > r && t < n) {  // (entries past a failed step are stale: never valid there)
          const int64_t x = q[r];
          q[r] = q[t];
          q[t] = x;
        }
      }
    };
    if (threadIdx.x == 0) {
      if (sm) walk(sperm);
      else walk(perm_local);
    }
    __syncthreads();
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
      if (sm) perm_local[i] = pl[i];
      perm_global[g0 + i] = g0 + pl[i];
    }
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
// One CTA per diagonal tile q of `map` (blockIdx.x = q): inv + q * TILE_ELEMS = L_qq^{-1}.
__global__ void __launch_bounds__(128) tile_inv_unit_kernel(TileMap map, double* __restrict__ inv_base) {
  extern __shared__ double M[];  // [T][129]
  const double* __restrict__ tile = map.tile(blockIdx.x, blockIdx.x);
  double* __restrict__ inv = inv_base + (int64_t)blockIdx.x * TILE_ELEMS;
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
