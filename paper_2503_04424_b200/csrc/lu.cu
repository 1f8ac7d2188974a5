// Block-local LU with partial pivoting (memdet_lu, reference memdet.py:268-319 and
// kernels/dense.py:38-54, 102-106): each stage's diagonal block is factored P A = L U with the
// pivot of each column the largest |a| below the diagonal inside the block; the row-k blocks
// are permuted and solved with the unit L, the column blocks solved against U, and the Schur
// update runs on full tiles.  |det| and its sign do not depend on which valid pivot sequence
// is taken, so the pivots need not reproduce LAPACK's (the reference's result is the logdet and
// the sign only, memdet.py:202-205).
//
//   lu_panel_cluster_kernel  LU_NB columns of the dense block on a 16-CTA cluster, the panel's
//                            rows in distributed shared memory (row i in CTA i mod 16)
//   lu_swap_rows_kernel      the panel's interchanges applied to the columns outside it
//   lu_u12_kernel            U12 = L11^{-1} A12 (unit-lower forward substitution per column)
//   lu_bulk_kernel           A22 -= L21 U12 (rank-LU_NB, FP64 FMA)
//   pack_upper_t_kernel      U^T (lower, non-unit) -> tile grid (the factor of the column solves)
//   tile_inv_lower_kernel    inverses of the lower non-unit diagonal tiles of U^T
//   pack_block_nt_kernel     row-major file strip -> tiles, not transposed (generic blocks)

namespace b2d {

constexpr int LU_NB = 32;
constexpr int LU_LD = LU_NB + 1;  // padded smem row of the panel
__host__ __device__ constexpr size_t lu_panel_smem(int rows) { return (size_t)rows * LU_LD * 8; }

struct LuArgs {
  double* A;                  // dense block, column-major, leading dimension ld
  double* u;                  // pivots u_rr (block-local row index)
  int64_t* swaps;             // LAPACK-style interchanges (block-local)
  unsigned long long* fail;   // first global row with a zero pivot (singular block)
  int64_t ld, n, g0;
};

__global__ void __launch_bounds__(LC_THREADS, 1) lu_panel_cluster_kernel(LuArgs g, int64_t r0, int nbk) {
  if (*g.fail != ~0ull) return;  // uniform: written by earlier kernels only
  cg::cluster_group cl = cg::this_cluster();
  const int c = (int)cl.block_rank();
  extern __shared__ double sm[];
  const int64_t n = g.n, ld = g.ld;
  const int R = (int)((n + LC - 1) / LC);
  double* P = sm;  // [R][LU_LD]: row li*LC + c of the panel
  __shared__ ArgMax cand[2][LC];
  __shared__ ArgMax sred[LC_THREADS / 32];
  __shared__ double bR[LU_NB], bT[LU_NB];
  const int tid = threadIdx.x, lane = tid & 31, wib = tid >> 5;
  double* __restrict__ A = g.A;
  for (int e = tid; e < R * nbk; e += LC_THREADS) {
    const int q = e / R, li = e % R;
    const int64_t i = (int64_t)li * LC + c;
    P[li * LU_LD + q] = (i >= r0 && i < n) ? A[(r0 + q) * ld + i] : 0.0;
  }
  for (int k = 0; k < nbk; ++k) {
    const int64_t r = r0 + k;
    ArgMax a{-1.0, INT64_MAX};
    for (int li = tid; li < R; li += LC_THREADS) {
      const int64_t i = (int64_t)li * LC + c;
      if (i >= r && i < n) a = better(a, ArgMax{fabs(P[li * LU_LD + k]), i});
    }
    a = warp_argmax(a);
    if (lane == 0) sred[wib] = a;
    __syncthreads();
    if (wib == 0) {
      ArgMax b = lane < LC_THREADS / 32 ? sred[lane] : ArgMax{-1.0, INT64_MAX};
      b = warp_argmax(b);
      if (lane < LC) *cl.map_shared_rank(&cand[k & 1][c], lane) = b;
    }
    cl.sync();  // A: candidates and the previous step's rows visible cluster-wide
    ArgMax b{-1.0, INT64_MAX};
    for (int q = 0; q < LC; ++q) b = better(b, cand[k & 1][q]);
    const int64_t t = b.i;
    const int orr = (int)(r % LC), ort = (int)(t % LC), lr = (int)(r / LC), lt = (int)(t / LC);
    for (int q = tid; q < nbk; q += LC_THREADS) {
      bR[q] = cl.map_shared_rank(P, orr)[(size_t)lr * LU_LD + q];
      bT[q] = cl.map_shared_rank(P, ort)[(size_t)lt * LU_LD + q];
    }
    cl.sync();  // B: rows r, t read everywhere; their owners may overwrite them
    const double p = bT[k];  // the pivot: row t's entry in column k
    if (p == 0.0) {
      if (c == 0 && tid == 0) atomicMin(g.fail, (unsigned long long)(g.g0 + r));
      return;  // uniform: a zero column below the diagonal, the block is singular
    }
    if (t != r) {
      if (c == orr)
        for (int q = tid; q < nbk; q += LC_THREADS) P[(size_t)lr * LU_LD + q] = bT[q];
      if (c == ort)
        for (int q = tid; q < nbk; q += LC_THREADS) P[(size_t)lt * LU_LD + q] = bR[q];
    }
    if (c == 0 && tid == 0) {
      g.u[r] = p;
      g.swaps[r] = t;
    }
    __syncthreads();
    const double inv = 1.0 / p;
    for (int li = tid; li < R; li += LC_THREADS) {
      const int64_t i = (int64_t)li * LC + c;
      if (i <= r || i >= n) continue;
      double* Pi = P + (size_t)li * LU_LD;
      const double l = Pi[k] * inv;
      Pi[k] = l;
      for (int q = k + 1; q < nbk; ++q) Pi[q] = fma(-l, bT[q], Pi[q]);
    }
    __syncthreads();
  }
  for (int e = tid; e < R * nbk; e += LC_THREADS) {
    const int q = e / R, li = e % R;
    const int64_t i = (int64_t)li * LC + c;
    if (i >= r0 && i < n) A[(r0 + q) * ld + i] = P[li * LU_LD + q];
  }
}

// Columns outside [r0, r0 + nbk): the panel's interchanges, in order.
__global__ void lu_swap_rows_kernel(LuArgs g, int64_t r0, int nbk) {
  if (*g.fail != ~0ull) return;
  for (int64_t col = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; col < g.n; col += (int64_t)gridDim.x * blockDim.x) {
    if (col >= r0 && col < r0 + nbk) continue;
    double* a = g.A + col * g.ld;
    for (int k = 0; k < nbk; ++k) {
      const int64_t r = r0 + k, t = g.swaps[r];
      if (t != r) {
        const double x = a[r];
        a[r] = a[t];
        a[t] = x;
      }
    }
  }
}

// U12 = L11^{-1} A12 for columns [r0 + nbk, n): one thread per column, L11 (unit lower) in smem.
__global__ void __launch_bounds__(128) lu_u12_kernel(LuArgs g, int64_t r0, int nbk) {
  if (*g.fail != ~0ull) return;
  __shared__ double L[LU_NB][LU_NB + 1];
  const int64_t ld = g.ld;
  for (int e = threadIdx.x; e < nbk * nbk; e += blockDim.x) {
    const int q = e % nbk, qq = e / nbk;  // L[q][qq] = A(r0 + q, r0 + qq)
    L[q][qq] = g.A[(r0 + qq) * ld + r0 + q];
  }
  __syncthreads();
  const int64_t col = r0 + nbk + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (col >= g.n) return;
  double* a = g.A + col * ld + r0;
  double u[LU_NB];
#pragma unroll
  for (int q = 0; q < LU_NB; ++q) u[q] = q < nbk ? a[q] : 0.0;
#pragma unroll
  for (int q = 1; q < LU_NB; ++q) {
    double v = u[q];
#pragma unroll
    for (int qq = 0; qq < q; ++qq) v = fma(-L[q][qq], u[qq], v);
    u[q] = q < nbk ? v : 0.0;
  }
#pragma unroll
  for (int q = 0; q < LU_NB; ++q)
    if (q < nbk) a[q] = u[q];
}

// A22 -= L21 U12 over rows and columns [r0 + nbk, n): 64 x 64 entry tiles, 4 x 4 per thread.
__global__ void __launch_bounds__(256) lu_bulk_kernel(LuArgs g, int64_t r0, int nbk) {
  if (*g.fail != ~0ull) return;
  __shared__ double sL[LU_NB][64], sU[LU_NB][64 + 1];
  const int64_t re = r0 + nbk, m = g.n - re, ld = g.ld;
  const int64_t nbt = (m + 63) / 64;
  const int64_t bi = blockIdx.x % nbt, bj = blockIdx.x / nbt;
  const int64_t i0 = re + bi * 64, j0 = re + bj * 64;
  for (int e = threadIdx.x; e < nbk * 64; e += 256) {
    const int q = e / 64, x = e % 64;
    sL[q][x] = i0 + x < g.n ? g.A[(r0 + q) * ld + i0 + x] : 0.0;
  }
  for (int e = threadIdx.x; e < nbk * 64; e += 256) {
    const int q = e % nbk, y = e / nbk;  // U12(r0 + q, j0 + y): contiguous in q
    sU[q][y] = j0 + y < g.n ? g.A[(j0 + y) * ld + r0 + q] : 0.0;
  }
  __syncthreads();
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  double v[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int64_t i = i0 + tx + 16 * a, j = j0 + ty + 16 * b;
      v[a][b] = (i < g.n && j < g.n) ? g.A[j * ld + i] : 0.0;
    }
  for (int q = 0; q < nbk; ++q) {
    double l[4], u[4];
#pragma unroll
    for (int a = 0; a < 4; ++a) l[a] = sL[q][tx + 16 * a];
#pragma unroll
    for (int b = 0; b < 4; ++b) u[b] = sU[q][ty + 16 * b];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) v[a][b] = fma(-l[a], u[b], v[a][b]);
  }
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int64_t i = i0 + tx + 16 * a, j = j0 + ty + 16 * b;
      if (i < g.n && j < g.n) g.A[j * ld + i] = v[a][b];
    }
}

// U^T -> tile grid: tile element (R, C) = U(C, R) for R >= C (lower, non-unit), identity beyond
// n, zero above the diagonal.
__global__ void __launch_bounds__(256) pack_upper_t_kernel(const double* __restrict__ dense, int64_t ld, int64_t n,
                                                           TileMap dst, int ntiles) {
  int I, J;
  const TileSet all{0, ntiles, 0, ntiles, 1, 0, 0, 0};
  tile_order(blockIdx.x, all, 1, &I, &J);
  double* t = dst.tile(I, J);
  for (int o = threadIdx.x; o < TILE_ELEMS; o += 256) {
    const int r = (o >> 3) & 127;
    const int c = ((o >> 10) << 3) + iperm8(o & 7);
    const int64_t R = (int64_t)I * T + r, C = (int64_t)J * T + c;
    double v;
    if (R >= n || C >= n) v = R == C ? 1.0 : 0.0;
    else v = R >= C ? dense[R * ld + C] : 0.0;
    t[o] = v;
  }
}

// One CTA per diagonal tile q of `map` (blockIdx.x = q): inv + q * TILE_ELEMS = L_qq^{-1} for a
// lower non-unit tile; one thread per column, forward substitution.
__global__ void __launch_bounds__(128) tile_inv_lower_kernel(TileMap map, double* __restrict__ inv_base) {
  extern __shared__ double M[];  // [T][129]: L below and on the diagonal, X^T above
  const double* __restrict__ tile = map.tile(blockIdx.x, blockIdx.x);
  double* __restrict__ inv = inv_base + (int64_t)blockIdx.x * TILE_ELEMS;
  const int c = threadIdx.x;
  for (int o = c; o < TILE_ELEMS; o += T) {
    const int r = (o >> 3) & 127;
    const int cc = ((o >> 10) << 3) + iperm8(o & 7);
    if (cc <= r) M[r * 129 + cc] = tile[o];
  }
  __syncthreads();
  // X[c][c] = 1 / L[c][c]; X[r][c] = -(sum_{c <= p < r} L[r][p] X[p][c]) / L[r][r]
  const double xcc = 1.0 / M[c * 129 + c];
  for (int r = c + 1; r < T; ++r) {
    double acc = M[r * 129 + c] * xcc;
    for (int p = c + 1; p < r; ++p) acc = fma(M[r * 129 + p], M[c * 129 + p], acc);
    M[c * 129 + r] = -acc / M[r * 129 + r];
  }
  __syncthreads();
  for (int o = c; o < TILE_ELEMS; o += T) {
    const int r = (o >> 3) & 127;
    const int cc = ((o >> 10) << 3) + iperm8(o & 7);
    inv[o] = cc < r ? M[cc * 129 + r] : (cc == r ? 1.0 / M[r * 129 + r] : 0.0);
  }
}

// Generic block ingest without transposition: one 128-row strip of the row-major file (block
// rows [128 J, 128 J + 128)) into tile row J of a grid block; rows valid below rows_valid,
// columns below cols_valid; identity padding on a diagonal block, zero elsewhere.
template <typename Tin>
__global__ void __launch_bounds__(256) pack_block_nt_kernel(const Tin* __restrict__ src, int64_t lda,
                                                            int64_t rows_valid, int64_t cols_valid, int diag,
                                                            TileMap out, int J) {
  const int I = blockIdx.x;  // tile column
  double* dst = out.tile(J, I);
  for (int idx = threadIdx.x; idx < TILE_ELEMS; idx += 256) {
    const int r = idx >> 7, cc = idx & 127;
    const int64_t R = (int64_t)J * T + r, C = (int64_t)I * T + cc;
    double v;
    if (R < rows_valid && C < cols_valid) v = (double)src[(int64_t)r * lda + C];
    else v = (diag && R == C) ? 1.0 : 0.0;
    dst[elem(r, cc)] = v;
  }
}

// dst tile (J, I) = src tile (I, J)^T over rtiles x ctiles source tiles (a generic block
// written as the next stage's row block is kept transposed, the form the row solves use).
constexpr size_t TRANSPOSE_SMEM = (size_t)T * (T + 1) * 8;
__global__ void __launch_bounds__(256) transpose_block_kernel(TileMap src, TileMap dst, int rtiles, int ctiles) {
  extern __shared__ double S[];  // [T][T + 1]
  const int I = blockIdx.x % rtiles, J = blockIdx.x / rtiles;
  const double* a = src.tile(I, J);
  double* b = dst.tile(J, I);
  for (int o = threadIdx.x; o < TILE_ELEMS; o += 256) {
    const int r = (o >> 3) & 127;
    const int c = ((o >> 10) << 3) + iperm8(o & 7);
    S[r * (T + 1) + c] = a[o];
  }
  __syncthreads();
  for (int o = threadIdx.x; o < TILE_ELEMS; o += 256) {
    const int r = (o >> 3) & 127;
    const int c = ((o >> 10) << 3) + iperm8(o & 7);
    b[o] = S[c * (T + 1) + r];
  }
}

}  // namespace b2d
