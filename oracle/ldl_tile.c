/*
 * ORACLE — TEST INFRASTRUCTURE ONLY.  Never linked into or called by the product path.
 *
 * C restatement of the reference's compiled tile LDL^T with 1x1 diagonal pivoting,
 * oocdet/kernels/_ldl.pyx:21-61 (algorithm), driven as in kernels/dense.py:57-81.
 *   - pivot: largest |a_ii| over the trailing diagonal, lowest index on ties (_ldl.pyx:30-36)
 *   - symmetric swap of r and t touching only the lower triangle (_ldl.pyx:38-46)
 *   - fail if |pivot| < tol, returning the step index (_ldl.pyx:47-50)
 *   - update a_ij -= a_ir * (a_jr / p) for r < j <= i (_ldl.pyx:52-60)
 * The matrix is row-major with leading dimension lda; only the lower triangle is used.
 * Returns -1 on success or the failing step index.
 */
#include <math.h>
#include <stdint.h>

#define A(i, j) a[(int64_t)(i) * lda + (j)]

int64_t oracle_ldl_tile_f64(double *a, int64_t n, int64_t lda, int64_t *swaps, double *d,
                            double *work, double tol) {
  for (int64_t r = 0; r < n; ++r) {
    int64_t t = r;
    double best = fabs(A(r, r));
    for (int64_t i = r + 1; i < n; ++i) {
      double v = fabs(A(i, i));
      if (v > best) { best = v; t = i; }
    }
    swaps[r] = t;
    if (t != r) {
      for (int64_t j = 0; j < r; ++j) { double x = A(r, j); A(r, j) = A(t, j); A(t, j) = x; }
      { double x = A(r, r); A(r, r) = A(t, t); A(t, t) = x; }
      for (int64_t i = r + 1; i < t; ++i) { double x = A(i, r); A(i, r) = A(t, i); A(t, i) = x; }
      for (int64_t i = t + 1; i < n; ++i) { double x = A(i, r); A(i, r) = A(i, t); A(i, t) = x; }
    }
    double p = A(r, r);
    if (fabs(p) < tol) return r;
    d[r] = p;
    double invp = 1.0 / p;
    for (int64_t i = r + 1; i < n; ++i) work[i] = A(i, r) * invp;
    for (int64_t i = r + 1; i < n; ++i) {
      double ci = A(i, r);
      for (int64_t j = r + 1; j <= i; ++j) A(i, j) -= ci * work[j];
    }
    for (int64_t i = r + 1; i < n; ++i) A(i, r) = work[i];
  }
  return -1;
}

int64_t oracle_ldl_tile_f32(float *a, int64_t n, int64_t lda, int64_t *swaps, float *d,
                            float *work, double tol) {
  for (int64_t r = 0; r < n; ++r) {
    int64_t t = r;
    float best = fabsf(A(r, r));
    for (int64_t i = r + 1; i < n; ++i) {
      float v = fabsf(A(i, i));
      if (v > best) { best = v; t = i; }
    }
    swaps[r] = t;
    if (t != r) {
      for (int64_t j = 0; j < r; ++j) { float x = A(r, j); A(r, j) = A(t, j); A(t, j) = x; }
      { float x = A(r, r); A(r, r) = A(t, t); A(t, t) = x; }
      for (int64_t i = r + 1; i < t; ++i) { float x = A(i, r); A(i, r) = A(t, i); A(t, i) = x; }
      for (int64_t i = t + 1; i < n; ++i) { float x = A(i, r); A(i, r) = A(i, t); A(i, t) = x; }
    }
    float p = A(r, r);
    if (fabsf(p) < tol) return r;
    d[r] = p;
    float invp = 1.0f / p;
    for (int64_t i = r + 1; i < n; ++i) work[i] = A(i, r) * invp;
    for (int64_t i = r + 1; i < n; ++i) {
      float ci = A(i, r);
      for (int64_t j = r + 1; j <= i; ++j) A(i, j) -= ci * work[j];
    }
    for (int64_t i = r + 1; i < n; ++i) A(i, r) = work[i];
  }
  return -1;
}
