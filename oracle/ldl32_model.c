/* ORACLE — TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).
 *
 * The reference's memdet_ldl on a float32 file (memdet.py:322-412) with every f32 operation in
 * the exact order of the third-party code it calls on the golden host, so the results are
 * bit-identical to the unmodified reference there (checked by tests/test_oracle_golden.py
 * against tests/golden/f32.*):
 *
 *   ldl tile       _ldl.pyx:21-61 (Cython `floating` = float, compiled without FMA contraction:
 *                  a_ij = fl(a_ij - fl(c_i * w_j)), w_j = fl(a_jr * fl(1 / p)))
 *   solve_lower    dense.py:94-99 -> SciPy ?trtrs -> OpenBLAS STRSM (Left, Lower, NoTrans, Unit),
 *                  OpenBLAS 0.3.3x as bundled with SciPy 1.18 (DYNAMIC_ARCH, SAPPHIRERAPIDS /
 *                  SKYLAKEX kernels): rows in GEMM_Q = 448 blocks; inside a block, rows in
 *                  unroll-16 groups (halving for the remainder): each group first subtracts one
 *                  FMA chain (from 0) over the block's earlier rows, then solves in place with
 *                  x_k = fma(-x_i, l_ki, x_k); after a block, every row below subtracts one chain
 *                  over the block.
 *   schur_update   dense.py:109-116 -> NumPy f32 matmul -> OpenBLAS SGEMM: tmp = C^T B with one
 *                  FMA chain (from 0) per K-block, K split as level3_thread.c does (GEMM_Q = 448:
 *                  K >= 2Q -> Q, Q < K < 2Q -> ceil(K/2)), the block chains added in order; then
 *                  T = fl(T - tmp).
 *   D^-1 scaling   memdet.py:368-371: fl(B / d).
 *
 * (Those BLAS orders were identified by bit-exact comparison with NumPy / SciPy on this host;
 * the engine's f32 kernels, ldl32.cu, follow this model.)
 *
 * Matrix: row-major m x m float (only the reference's (i <= j) blocks are used; updated in
 * place).  Outputs: d (m), perm (m, global), returns -1 or the failing global pivot.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define GEMM_Q 448
#define UNROLL_M 16

/* _ldl.pyx:21-61 on a row-major n x n block (leading dimension ld), float arithmetic. */
static int64_t ldl_tile32(float* a, int64_t ld, int64_t n, int64_t* swaps, float* d, float* work, double tol) {
#define A(i, j) a[(i) * ld + (j)]
  for (int64_t r = 0; r < n; ++r) {
    int64_t t = r;
    float best = fabsf(A(r, r));
    for (int64_t i = r + 1; i < n; ++i)
      if (fabsf(A(i, i)) > best) {
        best = fabsf(A(i, i));
        t = i;
      }
    swaps[r] = t;
    if (t != r) {
      float tmp;
      for (int64_t j = 0; j < r; ++j) { tmp = A(r, j); A(r, j) = A(t, j); A(t, j) = tmp; }
      tmp = A(r, r); A(r, r) = A(t, t); A(t, t) = tmp;
      for (int64_t i = r + 1; i < t; ++i) { tmp = A(i, r); A(i, r) = A(t, i); A(t, i) = tmp; }
      for (int64_t i = t + 1; i < n; ++i) { tmp = A(i, r); A(i, r) = A(i, t); A(i, t) = tmp; }
    }
    const float p = A(r, r);
    if (fabs((double)p) < tol) return r;
    d[r] = p;
    volatile float one = 1.0f;
    const float invp = one / p;
    for (int64_t i = r + 1; i < n; ++i) {
      volatile float w = A(i, r) * invp;
      work[i] = w;
    }
    for (int64_t i = r + 1; i < n; ++i) {
      const float ci = A(i, r);
      for (int64_t j = r + 1; j <= i; ++j) {
        volatile float prod = ci * work[j];
        A(i, j) = A(i, j) - prod;
      }
    }
    for (int64_t i = r + 1; i < n; ++i) A(i, r) = work[i];
  }
  return -1;
#undef A
}

/* X <- L^{-1} X, L unit lower (row-major, ldl), X n x w row-major (ldx): OpenBLAS STRSM order. */
static void trsm32(const float* L, int64_t ldl, float* X, int64_t ldx, int64_t n, int64_t w) {
  for (int64_t j = 0; j < w; ++j) {
    for (int64_t ls = 0; ls < n; ls += GEMM_Q) {
      const int64_t le = ls + GEMM_Q < n ? ls + GEMM_Q : n;
      int64_t r0 = ls, u = UNROLL_M;
      while (r0 < le) {
        while (u > 1 && r0 + u > le) u >>= 1;
        const int64_t r1 = r0 + u;
        if (r0 > ls)
          for (int64_t r = r0; r < r1; ++r) {
            float acc = 0.f;
            for (int64_t k = ls; k < r0; ++k) acc = fmaf(L[r * ldl + k], X[k * ldx + j], acc);
            X[r * ldx + j] = X[r * ldx + j] - acc;
          }
        for (int64_t i = r0; i < r1; ++i) {
          const float xi = X[i * ldx + j];
          for (int64_t k = i + 1; k < r1; ++k) X[k * ldx + j] = fmaf(-xi, L[k * ldl + i], X[k * ldx + j]);
        }
        r0 = r1;
      }
      for (int64_t r = le; r < n; ++r) {
        float acc = 0.f;
        for (int64_t k = ls; k < le; ++k) acc = fmaf(L[r * ldl + k], X[k * ldx + j], acc);
        X[r * ldx + j] = X[r * ldx + j] - acc;
      }
    }
  }
}

/* K-block boundaries of OpenBLAS's threaded level-3 driver (GEMM_Q = 448). */
static int kblocks(int64_t K, int64_t* bnd) {
  int nb = 0;
  int64_t ls = 0;
  bnd[nb++] = 0;
  while (ls < K) {
    int64_t ml = K - ls;
    if (ml >= 2 * GEMM_Q) ml = GEMM_Q;
    else if (ml > GEMM_Q) ml = (ml + 1) / 2;
    ls += ml;
    bnd[nb++] = ls;
  }
  return nb;
}

/* T (wi x wj, ldt) -= C^T S with C (K x wi, ldc), S (K x wj, lds): OpenBLAS SGEMM order. */
static void schur32(float* T, int64_t ldt, const float* C, int64_t ldc, const float* S, int64_t lds, int64_t K,
                    int64_t wi, int64_t wj) {
  int64_t bnd[64];
  const int nb = kblocks(K, bnd);
  for (int64_t p = 0; p < wi; ++p)
    for (int64_t q = 0; q < wj; ++q) {
      float tmp = 0.f;
      for (int b = 0; b + 1 < nb; ++b) {
        float acc = 0.f;
        for (int64_t k = bnd[b]; k < bnd[b + 1]; ++k) acc = fmaf(C[k * ldc + p], S[k * lds + q], acc);
        tmp = b == 0 ? acc : tmp + acc;
      }
      T[p * ldt + q] = T[p * ldt + q] - tmp;
    }
}

/* memdet.py:322-389 (scaled = True) on a row-major float matrix, in place. */
int64_t oracle_memdet_ldl32(float* M, int64_t m, int64_t nb, int64_t b, float* d_all, int64_t* perm_all) {
  float* work = (float*)malloc(sizeof(float) * (size_t)b);
  int64_t* swaps = (int64_t*)malloc(sizeof(int64_t) * (size_t)b);
  int64_t* perm = (int64_t*)malloc(sizeof(int64_t) * (size_t)b);
  float* X = NULL;
  float* S = NULL;
  float* dense = (float*)malloc(sizeof(float) * (size_t)b * b);
  int64_t fail = -1;
  for (int64_t k = 0; k < nb && fail < 0; ++k) {
    const int64_t k0 = k * b, hk = k == nb - 1 ? m - k0 : b;
    /* the diagonal block as its own array (the reference's A buffer), tolerance over all of it */
    float amax = 0.f;
    for (int64_t i = 0; i < hk; ++i)
      for (int64_t j = 0; j < hk; ++j) {
        dense[i * hk + j] = M[(k0 + i) * m + k0 + j];
        if (fabsf(dense[i * hk + j]) > amax) amax = fabsf(dense[i * hk + j]);
      }
    if (amax == 0.f) return k0;
    const double tol = 64.0 * 1.1920928955078125e-07 * (double)amax;
    const int64_t f = ldl_tile32(dense, hk, hk, swaps, d_all + k0, work, tol);
    if (f >= 0) { fail = k0 + f; break; }
    for (int64_t i = 0; i < hk; ++i) perm[i] = i;
    for (int64_t r = 0; r < hk; ++r)
      if (swaps[r] != r) { int64_t x = perm[r]; perm[r] = perm[swaps[r]]; perm[swaps[r]] = x; }
    for (int64_t i = 0; i < hk; ++i) perm_all[k0 + i] = k0 + perm[i];
    if (k == nb - 1) break;
    const int64_t c0 = k0 + b, W = m - c0;
    if (!X) {
      X = (float*)malloc(sizeof(float) * (size_t)b * W);
      S = (float*)malloc(sizeof(float) * (size_t)b * W);
    }
    /* row-k blocks: permute rows, solve, keep unscaled X, S = X / d (memdet.py:361-381) */
    for (int64_t i = 0; i < b; ++i) memcpy(X + i * W, M + (k0 + perm[i]) * m + c0, sizeof(float) * (size_t)W);
    trsm32(dense, hk, X, W, b, W);
    for (int64_t i = 0; i < b; ++i)
      for (int64_t j = 0; j < W; ++j) S[i * W + j] = X[i * W + j] / d_all[k0 + i];
    /* T(i, j) -= X_i^T S_j for every trailing block i <= j (memdet.py:385) */
    for (int64_t bi = k + 1; bi < nb; ++bi)
      for (int64_t bj = bi; bj < nb; ++bj) {
        const int64_t ri = bi * b, rj = bj * b;
        const int64_t wi = bi == nb - 1 ? m - ri : b, wj = bj == nb - 1 ? m - rj : b;
        schur32(M + ri * m + rj, m, X + (ri - c0), W, S + (rj - c0), W, b, wi, wj);
      }
  }
  free(work); free(swaps); free(perm); free(X); free(S); free(dense);
  return fail;
}
