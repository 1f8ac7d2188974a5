// The reference's own rounding sequence on the GPU, in the file dtype (memdet.py:322-412 and the
// tile kernels it calls: the Cython `floating` LDL kernel, SciPy's ?trtrs, NumPy's matmul).  Two
// users:
//   * float32 memdet_ldl (engine.cu run_ldl32): the reference factors a float32 file in float32,
//     so its pivots differ from the same values factored in f64; this path gives its permutation,
//     D and prefixes (oracle/ldl32_model.c, bit-identical to the reference on the golden host);
//   * the tile seam (b2d_tile_* host entries, paper_2503_04424_b200/kernels.py): the reference's
//     kernel module on the GPU, float64 or float32 tiles.
// Every operation follows the third-party order on the golden host (OpenBLAS 0.3.3x in SciPy /
// NumPy, identified by bit-exact comparison): GEMM = one FMA chain (from 0) per K-block, K split
// as OpenBLAS's threaded level-3 driver (K >= 2Q -> Q, Q < K < 2Q -> ceil(K/2)), the blocks added
// in order, then C = fl(C - tmp); TRSM = Q-row blocks, 16-row unroll groups (halving at the end):
// a group subtracts one chain over its block's earlier rows, then solves in place with
// x_i *= fl(1 / l_ii) (non-unit) and x_k = fma(-x_i, l_ki, x_k); after a block every row below
// subtracts one chain over it.  Q = 448 (single precision), 384 (double).
//
//   l32_block_in_kernel   diagonal block (row-major) -> column-major dense block, max|A| over it
//   l32_step_kernel       one pivot step of _ldl.pyx:30-58 and the L column of the previous step
//   l32_update_kernel     the step's trailing update a_ij = fl(a_ij - fl(c_i w_j))
//   l32_finish_kernel     swaps -> permutation, log|d|, d
//   l32_gather_kernel     row-k blocks, rows permuted (memdet.py:365-366)
//   l32_trsm_diag_kernel  TRSM inside one Q-row block
//   l32_gemm_kernel       C -= sum of per-K-block FMA chains (GEMM order; TRSM below-updates)
//   l32_scale_kernel      S = X / d (memdet.py:371)
#include "tile.cuh"

namespace b2d {

template <typename E> struct Blas;
template <> struct Blas<float> {
  static constexpr int Q = 448;  // OpenBLAS GEMM_Q, SGEMM / STRSM
  static constexpr double EPS = 1.1920928955078125e-07;
  __device__ static float add(float a, float b) { return __fadd_rn(a, b); }
  __device__ static float sub(float a, float b) { return __fsub_rn(a, b); }
  __device__ static float mul(float a, float b) { return __fmul_rn(a, b); }
  __device__ static float div(float a, float b) { return __fdiv_rn(a, b); }
  __device__ static float fma(float a, float b, float c) { return __fmaf_rn(a, b, c); }
};
template <> struct Blas<double> {
  static constexpr int Q = 384;  // OpenBLAS GEMM_Q, DGEMM / DTRSM
  static constexpr double EPS = 2.220446049250313e-16;
  __device__ static double add(double a, double b) { return __dadd_rn(a, b); }
  __device__ static double sub(double a, double b) { return __dsub_rn(a, b); }
  __device__ static double mul(double a, double b) { return __dmul_rn(a, b); }
  __device__ static double div(double a, double b) { return __ddiv_rn(a, b); }
  __device__ static double fma(double a, double b, double c) { return __fma_rn(a, b, c); }
};

constexpr int L32_Q = 448;   // float32 memdet_ldl (engine.cu)
constexpr int L32_QMAX = 448;
constexpr int L32_U = 16;    // TRSM row unroll
constexpr int L32_MAXKB = 64;

// dense(i, j) (column-major, ldd) = M[(k0 + i) * ldm + k0 + j]; amax = max |.| over the block,
// kept as the bits of a non-negative double (they order like the values)
template <typename E>
__global__ void __launch_bounds__(256) l32_block_in_kernel(const E* __restrict__ M, int64_t ldm, int64_t k0,
                                                           int64_t n, E* __restrict__ dense, int64_t ldd,
                                                           unsigned long long* __restrict__ amax_bits) {
  __shared__ E sm[32][33];
  const int64_t bi = blockIdx.y * 32, bj = blockIdx.x * 32;  // row / column tile origin of the block
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  double best = 0.0;
  for (int r = ty; r < 32; r += 8) {
    const int64_t i = bi + r, j = bj + tx;
    E v = 0;
    if (i < n && j < n) v = M[(k0 + i) * ldm + k0 + j];
    best = fmax(best, fabs((double)v));
    sm[r][tx] = v;
  }
  __syncthreads();
  for (int cidx = ty; cidx < 32; cidx += 8) {
    const int64_t j = bj + cidx, i = bi + tx;
    if (i < n && j < n) dense[j * ldd + i] = sm[tx][cidx];
  }
  for (int off = 16; off; off >>= 1) best = fmax(best, __shfl_xor_sync(0xffffffffu, best, off));
  if (tx == 0) atomicMax(amax_bits, (unsigned long long)__double_as_longlong(best));
}

template <typename E>
struct L32Step {
  E* a;  // dense column-major block, a(i, j) = a[j * ld + i]
  int64_t ld, n, g0;
  E* work;
  E* d;
  int64_t* swaps;
  unsigned long long* fail;
  const unsigned long long* amax_bits;
  double tol;  // >= 0: the caller's tolerance; < 0: PIVOT_TOL_SCALE * eps(E) * max|A| (dense.py:73)
};

struct ArgMaxE {
  double v;
  int64_t i;
};
__device__ __forceinline__ ArgMaxE better_e(ArgMaxE a, ArgMaxE b) {
  // larger |a_ii| wins; ties go to the lower index (the reference's "first max", _ldl.pyx:31-36)
  if (b.v > a.v || (b.v == a.v && b.i < a.i)) return b;
  return a;
}

// Step r (one CTA of 1024 threads).
template <typename E>
__global__ void __launch_bounds__(1024) l32_step_kernel(L32Step<E> g, int64_t r) {
  if (*g.fail != ~0ull) return;
  __shared__ ArgMaxE sred[32];
  __shared__ int64_t s_t;
  const int tid = threadIdx.x, lane = tid & 31, wib = tid >> 5;
  const int64_t n = g.n, ld = g.ld;
  E* __restrict__ a = g.a;
  const double amax = __longlong_as_double((long long)*g.amax_bits);
  if (amax == 0.0) {  // "LDL on an all-zero tile" (dense.py:71-72)
    if (tid == 0) atomicMin(g.fail, (unsigned long long)g.g0);
    return;
  }
  // the L column of step r - 1 (_ldl.pyx:59-60), before this step's interchange moves row r
  if (r > 0)
    for (int64_t i = r + tid; i < n; i += 1024) a[(r - 1) * ld + i] = g.work[i];
  // pivot: largest |a_ii| over [r, n), lowest index on ties (|E| is exact in double)
  ArgMaxE best{-1.0, INT64_MAX};
  for (int64_t i = r + tid; i < n; i += 1024) best = better_e(best, ArgMaxE{fabs((double)a[i * ld + i]), i});
  for (int off = 16; off; off >>= 1) {
    ArgMaxE o{__shfl_xor_sync(0xffffffffu, best.v, off), __shfl_xor_sync(0xffffffffu, best.i, off)};
    best = better_e(best, o);
  }
  if (lane == 0) sred[wib] = best;
  __syncthreads();
  if (wib == 0) {
    ArgMaxE b = sred[lane];
    for (int off = 16; off; off >>= 1) {
      ArgMaxE o{__shfl_xor_sync(0xffffffffu, b.v, off), __shfl_xor_sync(0xffffffffu, b.i, off)};
      b = better_e(b, o);
    }
    if (lane == 0) s_t = b.i;
  }
  __syncthreads();
  const int64_t t = s_t;
  if (t != r) {  // symmetric interchange within the lower triangle (_ldl.pyx:38-46): disjoint sets
    for (int64_t q = tid; q < n; q += 1024) {
      E x;
      if (q < r) {  // a(r, q) <-> a(t, q)
        x = a[q * ld + r]; a[q * ld + r] = a[q * ld + t]; a[q * ld + t] = x;
      } else if (q == r) {  // a(r, r) <-> a(t, t)
        x = a[r * ld + r]; a[r * ld + r] = a[t * ld + t]; a[t * ld + t] = x;
      } else if (q < t) {  // a(q, r) <-> a(t, q)
        x = a[r * ld + q]; a[r * ld + q] = a[q * ld + t]; a[q * ld + t] = x;
      } else if (q > t) {  // a(q, r) <-> a(q, t)
        x = a[r * ld + q]; a[r * ld + q] = a[t * ld + q]; a[t * ld + q] = x;
      }
    }
  }
  if (tid == 0) g.swaps[r] = t;
  __syncthreads();
  const E p = a[r * ld + r];
  const double tol = g.tol >= 0.0 ? g.tol : 64.0 * Blas<E>::EPS * amax;  // PIVOT_TOL_SCALE * eps * max|A|
  if (fabs((double)p) < tol) {
    if (tid == 0) atomicMin(g.fail, (unsigned long long)(g.g0 + r));
    return;
  }
  if (tid == 0) g.d[r] = p;
  const E invp = Blas<E>::div((E)1, p);
  for (int64_t i = r + 1 + tid; i < n; i += 1024) g.work[i] = Blas<E>::mul(a[r * ld + i], invp);
}

// a(i, j) -= a(i, r) * w_j for r < j <= i < n; one CTA per column j.
template <typename E>
__global__ void __launch_bounds__(256) l32_update_kernel(L32Step<E> g, int64_t r) {
  if (*g.fail != ~0ull) return;
  const int64_t j = r + 1 + blockIdx.x, ld = g.ld;
  const E w = g.work[j];
  const E* __restrict__ cr = g.a + r * ld;
  E* __restrict__ cj = g.a + j * ld;
  for (int64_t i = j + threadIdx.x; i < g.n; i += 256) cj[i] = Blas<E>::sub(cj[i], Blas<E>::mul(cr[i], w));
}

// swaps -> block permutation (dense.py:25-30), global perm (memdet.py:352-353), ell = log|d|, d.
template <typename E>
__global__ void l32_finish_kernel(const int64_t* __restrict__ swaps, const E* __restrict__ d, int64_t n,
                                  int64_t g0, int64_t* __restrict__ perm_local, int64_t* __restrict__ perm_global,
                                  double* __restrict__ ell, double* __restrict__ dout,
                                  const unsigned long long* __restrict__ fail) {
  if (blockIdx.x == 0) {
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) perm_local[i] = i;
    __syncthreads();
    if (threadIdx.x == 0 && *fail == ~0ull)
      for (int64_t r = 0; r < n; ++r) {
        const int64_t t = swaps[r];
        if (t != r) {
          const int64_t x = perm_local[r];
          perm_local[r] = perm_local[t];
          perm_local[t] = x;
        }
      }
    __syncthreads();
    if (perm_global)
      for (int64_t i = threadIdx.x; i < n; i += blockDim.x) perm_global[g0 + i] = g0 + perm_local[i];
  }
  if (!ell) return;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    ell[g0 + i] = log(fabs((double)d[i]));
    dout[g0 + i] = (double)d[i];
  }
}

// X[i][c] = M[(k0 + perm[i]) * ldm + c0 + c], i < rows, c < W
template <typename E>
__global__ void l32_gather_kernel(const E* __restrict__ M, int64_t ldm, int64_t k0, int64_t c0,
                                  const int64_t* __restrict__ perm, int64_t rows, int64_t W, E* __restrict__ X,
                                  int64_t ldx) {
  for (int64_t i = blockIdx.y; i < rows; i += gridDim.y) {
    const E* src = M + (k0 + perm[i]) * ldm + c0;
    for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < W; c += (int64_t)gridDim.x * blockDim.x)
      X[i * ldx + c] = src[c];
  }
}

template <typename E>
__global__ void l32_scale_kernel(const E* __restrict__ X, E* __restrict__ S, int64_t ldx, int64_t rows, int64_t W,
                                 const E* __restrict__ d) {
  for (int64_t i = blockIdx.y; i < rows; i += gridDim.y) {
    const E di = d[i];
    for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < W; c += (int64_t)gridDim.x * blockDim.x)
      S[i * ldx + c] = Blas<E>::div(X[i * ldx + c], di);
  }
}

// TRSM inside the row block [ls, le) (<= Q rows) for TW columns per CTA: rows in unroll groups of
// 16 (halving for the remainder); each group first subtracts one FMA chain (from 0) over the
// block's earlier rows, then solves in place (non-unit: x_i *= fl(1 / l_ii) first).
// L = lower factor in a column-major dense block (l(r, k) = L[k * ldl + r]).
template <typename E> struct TrsmTW;
template <> struct TrsmTW<float> { static constexpr int v = 64; };
template <> struct TrsmTW<double> { static constexpr int v = 32; };
template <typename E>
constexpr size_t l32_trsm_smem() {
  return ((size_t)L32_QMAX * TrsmTW<E>::v + (size_t)L32_U * L32_QMAX + L32_U * L32_U + L32_U) * sizeof(E);
}
constexpr size_t L32_TRSM_SMEM = l32_trsm_smem<float>();
template <typename E>
__global__ void __launch_bounds__(256) l32_trsm_diag_kernel(const E* __restrict__ L, int64_t ldl, E* __restrict__ X,
                                                            int64_t ldx, int64_t W, int64_t ls, int64_t le, int unit,
                                                            const unsigned long long* __restrict__ fail) {
  if (*fail != ~0ull) return;
  constexpr int TW = TrsmTW<E>::v;
  extern __shared__ __align__(16) unsigned char smem_raw32[];
  E* xs = reinterpret_cast<E*>(smem_raw32);  // [QMAX][TW]
  E* Ls = xs + L32_QMAX * TW;                 // [U][QMAX]: rows of the group, columns [ls, r0)
  E* Lu = Ls + L32_U * L32_QMAX;              // [U][U]: the group's own triangle
  E* Li = Lu + L32_U * L32_U;                 // [U]: fl(1 / l_ii) of the group (non-unit)
  const int tid = threadIdx.x;
  const int64_t c0 = (int64_t)blockIdx.x * TW;
  const int cw = (int)(W - c0 < TW ? W - c0 : TW);
  const int nq = (int)(le - ls);
  for (int e = tid; e < nq * TW; e += 256) {
    const int i = e / TW, c = e % TW;
    xs[e] = c < cw ? X[(ls + i) * ldx + c0 + c] : (E)0;
  }
  __syncthreads();
  int u = L32_U;
  for (int r0 = 0; r0 < nq;) {
    while (u > 1 && r0 + u > nq) u >>= 1;
    const int r1 = r0 + u;
    // stage the group's rows of L: columns [0, r0) of the block (relative) and its own triangle
    for (int e = tid; e < u * r1; e += 256) {
      const int k = e / u, rr = e % u;  // coalesced: consecutive rows of column k
      const E v = L[(ls + k) * ldl + ls + r0 + rr];
      if (k < r0) Ls[rr * L32_QMAX + k] = v;
      else Lu[rr * L32_U + (k - r0)] = v;
    }
    if (!unit && tid < u) Li[tid] = Blas<E>::div((E)1, L[(ls + r0 + tid) * ldl + ls + r0 + tid]);
    __syncthreads();
    if (r0 > 0) {
      // chains for (row, column) pairs of the group
      for (int e = tid; e < u * TW; e += 256) {
        const int rr = e / TW, c = e % TW;
        E acc = 0;
        const E* lr = Ls + rr * L32_QMAX;
        for (int k = 0; k < r0; ++k) acc = Blas<E>::fma(lr[k], xs[k * TW + c], acc);
        xs[(r0 + rr) * TW + c] = Blas<E>::sub(xs[(r0 + rr) * TW + c], acc);
      }
      __syncthreads();
    }
    // in-group forward substitution, one thread per column
    if (tid < TW) {
      const int c = tid;
      for (int i = 0; i < u; ++i) {
        E xi = xs[(r0 + i) * TW + c];
        if (!unit) {
          xi = Blas<E>::mul(xi, Li[i]);
          xs[(r0 + i) * TW + c] = xi;
        }
        for (int k = i + 1; k < u; ++k)
          xs[(r0 + k) * TW + c] = Blas<E>::fma(-xi, Lu[k * L32_U + i], xs[(r0 + k) * TW + c]);
      }
    }
    __syncthreads();
    r0 = r1;
  }
  for (int e = tid; e < nq * TW; e += 256) {
    const int i = e / TW, c = e % TW;
    if (c < cw) X[(ls + i) * ldx + c0 + c] = xs[e];
  }
}

// C[p][q] = fl(C[p][q] - tmp), tmp = sum over K-blocks (in order) of the FMA chain (from 0)
// sum_{k in block} A[k][p] * B[k][q].  With tri, only elements whose reference block row
// (roff + p) / blk <= block column (coff + q) / blk.
template <typename E>
struct GT {
  const E* A;
  int64_t lda;
  const E* B;
  int64_t ldb;
  E* C;
  int64_t ldc;
  int64_t Mr, Nc;
  int nkb;
  int kb[L32_MAXKB + 1];
  int tri;
  int64_t blk, roff, coff;
};
using G32 = GT<float>;
template <typename E> struct GemmTM;  // rows per thread: 8 (float: 128 accumulators), 4 (double)
template <> struct GemmTM<float> { static constexpr int v = 8; };
template <> struct GemmTM<double> { static constexpr int v = 4; };
constexpr int G32_BN = 128, G32_KC = 8;
template <typename E>
constexpr int gemm_bm() { return 16 * GemmTM<E>::v; }
constexpr int G32_BM = 128;
template <typename E>
__global__ void __launch_bounds__(256) l32_gemm_kernel(GT<E> g, const unsigned long long* __restrict__ fail) {
  if (*fail != ~0ull) return;
  constexpr int TM = GemmTM<E>::v, BM = 16 * TM, BN = G32_BN, KC = G32_KC;
  __shared__ E As[2][KC][BM];
  __shared__ E Bs[2][KC][BN];
  const int64_t p0 = (int64_t)blockIdx.y * BM, q0 = (int64_t)blockIdx.x * BN;
  if (g.tri) {
    const int64_t pmin_blk = (g.roff + p0) / g.blk;
    const int64_t qmax_blk = (g.coff + (q0 + BN < g.Nc ? q0 + BN : g.Nc) - 1) / g.blk;
    if (pmin_blk > qmax_blk) return;  // wholly inside the strictly-lower block triangle
  }
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  // thread tile: rows ty + 16 a (a < TM), columns tx + 16 b (b < 8): strided, so shared reads are
  // conflict-free and coalesced stores need no vector alignment
  E acc[TM][8], tmp[TM][8];
#pragma unroll
  for (int a = 0; a < TM; ++a)
#pragma unroll
    for (int b = 0; b < 8; ++b) acc[a][b] = tmp[a][b] = (E)0;
  const int K = g.kb[g.nkb];
  constexpr int NA = KC * BM / 256, NB = KC * BN / 256;
  E ra[NA], rb[NB];
  auto load = [&](int k0) {
#pragma unroll
    for (int t = 0; t < NA; ++t) {
      const int e = tid + 256 * t, k = k0 + e / BM, p = e % BM;
      ra[t] = (k < K && p0 + p < g.Mr) ? g.A[(int64_t)k * g.lda + p0 + p] : (E)0;
    }
#pragma unroll
    for (int t = 0; t < NB; ++t) {
      const int e = tid + 256 * t, k = k0 + e / BN, q = e % BN;
      rb[t] = (k < K && q0 + q < g.Nc) ? g.B[(int64_t)k * g.ldb + q0 + q] : (E)0;
    }
  };
  auto store = [&](int buf) {
#pragma unroll
    for (int t = 0; t < NA; ++t) {
      const int e = tid + 256 * t;
      As[buf][e / BM][e % BM] = ra[t];
    }
#pragma unroll
    for (int t = 0; t < NB; ++t) {
      const int e = tid + 256 * t;
      Bs[buf][e / BN][e % BN] = rb[t];
    }
  };
  load(0);
  store(0);
  __syncthreads();
  int kbi = 0, next_b = g.kb[1];
  for (int k0 = 0, buf = 0; k0 < K; k0 += KC, buf ^= 1) {
    const bool more = k0 + KC < K;
    if (more) load(k0 + KC);
#pragma unroll
    for (int kk = 0; kk < KC; ++kk) {
      const int k = k0 + kk;
      if (k >= K) break;
      if (k == next_b) {  // K-block boundary: tmp = tmp + chain, new chain from 0
#pragma unroll
        for (int a = 0; a < TM; ++a)
#pragma unroll
          for (int b = 0; b < 8; ++b) {
            tmp[a][b] = kbi == 0 ? acc[a][b] : Blas<E>::add(tmp[a][b], acc[a][b]);
            acc[a][b] = (E)0;
          }
        ++kbi;
        next_b = g.kb[kbi + 1];
      }
      E ar[TM], br[8];
#pragma unroll
      for (int a = 0; a < TM; ++a) ar[a] = As[buf][kk][ty + 16 * a];
#pragma unroll
      for (int b = 0; b < 8; ++b) br[b] = Bs[buf][kk][tx + 16 * b];
#pragma unroll
      for (int a = 0; a < TM; ++a)
#pragma unroll
        for (int b = 0; b < 8; ++b) acc[a][b] = Blas<E>::fma(ar[a], br[b], acc[a][b]);
    }
    if (more) store(buf ^ 1);
    __syncthreads();
  }
#pragma unroll
  for (int a = 0; a < TM; ++a) {
    const int64_t p = p0 + ty + 16 * a;
    if (p >= g.Mr) continue;
    const int64_t pb = (g.roff + p) / g.blk;
#pragma unroll
    for (int b = 0; b < 8; ++b) {
      const int64_t q = q0 + tx + 16 * b;
      if (q >= g.Nc) continue;
      if (g.tri && pb > (g.coff + q) / g.blk) continue;
      const E t = kbi == 0 ? acc[a][b] : Blas<E>::add(tmp[a][b], acc[a][b]);
      E* cp = g.C + p * g.ldc + q;
      *cp = Blas<E>::sub(*cp, t);
    }
  }
}

// K-block boundaries of OpenBLAS's threaded level-3 driver: K >= 2Q -> Q, Q < K < 2Q -> ceil(K/2).
static int l32_kblocks(int64_t K, int* kb, int Q = L32_Q) {
  int nb = 0;
  int64_t ls = 0;
  kb[nb++] = 0;
  while (ls < K && nb <= L32_MAXKB) {
    int64_t ml = K - ls;
    if (ml >= 2 * Q) ml = Q;
    else if (ml > Q) ml = (ml + 1) / 2;
    ls += ml;
    kb[nb++] = (int)ls;
  }
  return nb - 1;
}

}  // namespace b2d
