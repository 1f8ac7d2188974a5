// float32 memdet_ldl in the reference's own f32 arithmetic (memdet.py:322-412 on a float32
// file: its Cython `floating` LDL kernel, SciPy's f32 ?trtrs and NumPy's f32 matmul).  Every
// operation follows oracle/ldl32_model.c, which is bit-identical to the unmodified reference on
// the golden host (tests/golden/f32.*), so the permutation, D and the prefixes are the
// reference's -- not those of the same values factored in f64, which pivot differently.
//
//   l32_block_in_kernel   diagonal block (row-major in M) -> column-major dense block, max|A|
//                         over the whole block (dense.py:70-73)
//   l32_step_kernel       one pivot step of _ldl.pyx:30-58 (argmax of the diagonal, lowest index
//                         on ties; symmetric interchange; tolerance; 1/p; w = c / p) and the L
//                         column of the previous step
//   l32_update_kernel     the step's trailing update a_ij = fl(a_ij - fl(c_i w_j))
//   l32_finish_kernel     swaps -> permutation, log|d|, d
//   l32_gather_kernel     row-k blocks, rows permuted (memdet.py:365-366)
//   l32_trsm_diag_kernel  STRSM (Left, Lower, Unit) inside one GEMM_Q row block, OpenBLAS order
//   l32_gemm_kernel       C -= sum of per-K-block FMA chains (SGEMM order; STRSM below-updates)
//   l32_scale_kernel      S = X / d (memdet.py:371)
#include "tile.cuh"

namespace b2d {

constexpr int L32_Q = 448;  // OpenBLAS GEMM_Q of SGEMM / STRSM (oracle/ldl32_model.c)
constexpr int L32_U = 16;   // STRSM row unroll
constexpr int L32_MAXKB = 64;

// dense(i, j) (column-major, ldd) = M[(k0 + i) * ldm + k0 + j]; amax = max |.| over the block
__global__ void __launch_bounds__(256) l32_block_in_kernel(const float* __restrict__ M, int64_t ldm, int64_t k0,
                                                           int64_t n, float* __restrict__ dense, int64_t ldd,
                                                           unsigned* __restrict__ amax_bits) {
  __shared__ float sm[32][33];
  const int64_t bi = blockIdx.y * 32, bj = blockIdx.x * 32;  // row / column tile origin of the block
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  float best = 0.f;
  for (int r = ty; r < 32; r += 8) {
    const int64_t i = bi + r, j = bj + tx;
    float v = 0.f;
    if (i < n && j < n) v = M[(k0 + i) * ldm + k0 + j];
    best = fmaxf(best, fabsf(v));
    sm[r][tx] = v;
  }
  __syncthreads();
  for (int cidx = ty; cidx < 32; cidx += 8) {
    const int64_t j = bj + cidx, i = bi + tx;
    if (i < n && j < n) dense[j * ldd + i] = sm[tx][cidx];
  }
  for (int off = 16; off; off >>= 1) best = fmaxf(best, __shfl_xor_sync(0xffffffffu, best, off));
  if (tx == 0) atomicMax(amax_bits, __float_as_uint(best));  // non-negative floats order as their bits
}

struct L32Step {
  float* a;  // dense column-major block, a(i, j) = a[j * ld + i]
  int64_t ld, n, g0;
  float* work;
  float* d;
  int64_t* swaps;
  unsigned long long* fail;
  const unsigned* amax_bits;
};

struct ArgMax32 {
  float v;
  int64_t i;
};
__device__ __forceinline__ ArgMax32 better32(ArgMax32 a, ArgMax32 b) {
  // larger |a_ii| wins; ties go to the lower index (the reference's "first max", _ldl.pyx:31-36)
  if (b.v > a.v || (b.v == a.v && b.i < a.i)) return b;
  return a;
}

// Step r (one CTA of 1024 threads).
__global__ void __launch_bounds__(1024) l32_step_kernel(L32Step g, int64_t r) {
  if (*g.fail != ~0ull) return;
  __shared__ ArgMax32 sred[32];
  __shared__ int64_t s_t;
  const int tid = threadIdx.x, lane = tid & 31, wib = tid >> 5;
  const int64_t n = g.n, ld = g.ld;
  float* __restrict__ a = g.a;
  const float amax = __uint_as_float(*g.amax_bits);
  if (amax == 0.f) {  // "LDL on an all-zero tile" (dense.py:71-72)
    if (tid == 0) atomicMin(g.fail, (unsigned long long)g.g0);
    return;
  }
  // the L column of step r - 1 (_ldl.pyx:59-60), before this step's interchange moves row r
  if (r > 0)
    for (int64_t i = r + tid; i < n; i += 1024) a[(r - 1) * ld + i] = g.work[i];
  // pivot: largest |a_ii| over [r, n), lowest index on ties
  ArgMax32 best{-1.f, INT64_MAX};
  for (int64_t i = r + tid; i < n; i += 1024) best = better32(best, ArgMax32{fabsf(a[i * ld + i]), i});
  for (int off = 16; off; off >>= 1) {
    ArgMax32 o{__shfl_xor_sync(0xffffffffu, best.v, off), __shfl_xor_sync(0xffffffffu, best.i, off)};
    best = better32(best, o);
  }
  if (lane == 0) sred[wib] = best;
  __syncthreads();
  if (wib == 0) {
    ArgMax32 b = sred[lane];
    for (int off = 16; off; off >>= 1) {
      ArgMax32 o{__shfl_xor_sync(0xffffffffu, b.v, off), __shfl_xor_sync(0xffffffffu, b.i, off)};
      b = better32(b, o);
    }
    if (lane == 0) s_t = b.i;
  }
  __syncthreads();
  const int64_t t = s_t;
  if (t != r) {  // symmetric interchange within the lower triangle (_ldl.pyx:38-46): disjoint sets
    for (int64_t q = tid; q < n; q += 1024) {
      float x;
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
  const float p = a[r * ld + r];
  const double tol = 64.0 * 1.1920928955078125e-07 * (double)amax;  // PIVOT_TOL_SCALE * eps(f32) * max|A|
  if (fabs((double)p) < tol) {
    if (tid == 0) atomicMin(g.fail, (unsigned long long)(g.g0 + r));
    return;
  }
  if (tid == 0) g.d[r] = p;
  const float invp = __fdiv_rn(1.0f, p);
  for (int64_t i = r + 1 + tid; i < n; i += 1024) g.work[i] = __fmul_rn(a[r * ld + i], invp);
}

// a(i, j) -= a(i, r) * w_j for r < j <= i < n; one CTA per column j.
__global__ void __launch_bounds__(256) l32_update_kernel(L32Step g, int64_t r) {
  if (*g.fail != ~0ull) return;
  const int64_t j = r + 1 + blockIdx.x, ld = g.ld;
  const float w = g.work[j];
  const float* __restrict__ cr = g.a + r * ld;
  float* __restrict__ cj = g.a + j * ld;
  for (int64_t i = j + threadIdx.x; i < g.n; i += 256) cj[i] = __fsub_rn(cj[i], __fmul_rn(cr[i], w));
}

// swaps -> block permutation (dense.py:25-30), global perm (memdet.py:352-353), ell = log|d|, d.
__global__ void l32_finish_kernel(const int64_t* __restrict__ swaps, const float* __restrict__ d, int64_t n,
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
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) perm_global[g0 + i] = g0 + perm_local[i];
  }
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    ell[g0 + i] = log(fabs((double)d[i]));
    dout[g0 + i] = (double)d[i];
  }
}

// X[i][c] = M[(k0 + perm[i]) * ldm + c0 + c], i < rows, c < W
__global__ void l32_gather_kernel(const float* __restrict__ M, int64_t ldm, int64_t k0, int64_t c0,
                                  const int64_t* __restrict__ perm, int64_t rows, int64_t W, float* __restrict__ X,
                                  int64_t ldx) {
  for (int64_t i = blockIdx.y; i < rows; i += gridDim.y) {
    const float* src = M + (k0 + perm[i]) * ldm + c0;
    for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < W; c += (int64_t)gridDim.x * blockDim.x)
      X[i * ldx + c] = src[c];
  }
}

__global__ void l32_scale_kernel(const float* __restrict__ X, float* __restrict__ S, int64_t ldx, int64_t rows,
                                 int64_t W, const float* __restrict__ d) {
  for (int64_t i = blockIdx.y; i < rows; i += gridDim.y) {
    const float di = d[i];
    for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < W; c += (int64_t)gridDim.x * blockDim.x)
      S[i * ldx + c] = __fdiv_rn(X[i * ldx + c], di);
  }
}

// STRSM inside the row block [ls, le) (<= L32_Q rows) for L32_TW columns per CTA: rows in unroll
// groups of 16 (halving for the remainder); each group first subtracts one FMA chain (from 0)
// over the block's earlier rows, then solves in place with x_k = fma(-x_i, l_ki, x_k).
// L = unit lower factor in the column-major dense block (l(r, k) = L[k * ldl + r]).
constexpr int L32_TW = 64;
constexpr size_t L32_TRSM_SMEM = ((size_t)L32_Q * L32_TW + (size_t)L32_U * L32_Q + L32_U * L32_U) * 4;
__global__ void __launch_bounds__(256) l32_trsm_diag_kernel(const float* __restrict__ L, int64_t ldl, float* __restrict__ X,
                                                            int64_t ldx, int64_t W, int64_t ls, int64_t le,
                                                            const unsigned long long* __restrict__ fail) {
  if (*fail != ~0ull) return;
  extern __shared__ float smem[];
  float* xs = smem;                      // [L32_Q][L32_TW]
  float* Ls = xs + L32_Q * L32_TW;       // [L32_U][L32_Q]: rows of the group, columns [ls, r0)
  float* Lu = Ls + L32_U * L32_Q;        // [L32_U][L32_U]: the group's own triangle
  const int tid = threadIdx.x;
  const int64_t c0 = (int64_t)blockIdx.x * L32_TW;
  const int cw = (int)(W - c0 < L32_TW ? W - c0 : L32_TW);
  const int nq = (int)(le - ls);
  for (int e = tid; e < nq * L32_TW; e += 256) {
    const int i = e / L32_TW, c = e % L32_TW;
    xs[e] = c < cw ? X[(ls + i) * ldx + c0 + c] : 0.f;
  }
  __syncthreads();
  int u = L32_U;
  for (int r0 = 0; r0 < nq;) {
    while (u > 1 && r0 + u > nq) u >>= 1;
    const int r1 = r0 + u;
    // stage the group's rows of L: columns [0, r0) of the block (relative) and its own triangle
    for (int e = tid; e < u * r1; e += 256) {
      const int k = e / u, rr = e % u;  // coalesced: consecutive rows of column k
      const float v = L[(ls + k) * ldl + ls + r0 + rr];
      if (k < r0) Ls[rr * L32_Q + k] = v;
      else Lu[rr * L32_U + (k - r0)] = v;
    }
    __syncthreads();
    if (r0 > 0) {
      // chains for (row, column) pairs of the group
      for (int e = tid; e < u * L32_TW; e += 256) {
        const int rr = e / L32_TW, c = e % L32_TW;
        float acc = 0.f;
        const float* lr = Ls + rr * L32_Q;
        for (int k = 0; k < r0; ++k) acc = __fmaf_rn(lr[k], xs[k * L32_TW + c], acc);
        xs[(r0 + rr) * L32_TW + c] = __fsub_rn(xs[(r0 + rr) * L32_TW + c], acc);
      }
      __syncthreads();
    }
    // in-group forward substitution, one thread per column
    if (tid < L32_TW) {
      const int c = tid;
      for (int i = 0; i < u; ++i) {
        const float xi = xs[(r0 + i) * L32_TW + c];
        for (int k = i + 1; k < u; ++k)
          xs[(r0 + k) * L32_TW + c] = __fmaf_rn(-xi, Lu[k * L32_U + i], xs[(r0 + k) * L32_TW + c]);
      }
    }
    __syncthreads();
    r0 = r1;
  }
  for (int e = tid; e < nq * L32_TW; e += 256) {
    const int i = e / L32_TW, c = e % L32_TW;
    if (c < cw) X[(ls + i) * ldx + c0 + c] = xs[e];
  }
}

// C[p][q] = fl(C[p][q] - tmp), tmp = sum over K-blocks (in order) of the FMA chain (from 0)
// sum_{k in block} A[k][p] * B[k][q]: NumPy / OpenBLAS SGEMM's rounding sequence.  With tri, only
// elements whose reference block row (roff + p) / blk <= block column (coff + q) / blk.
struct G32 {
  const float* A;
  int64_t lda;
  const float* B;
  int64_t ldb;
  float* C;
  int64_t ldc;
  int64_t Mr, Nc;
  int nkb;
  int kb[L32_MAXKB + 1];
  int tri;
  int64_t blk, roff, coff;
};
constexpr int G32_BM = 128, G32_BN = 128, G32_KC = 8;
__global__ void __launch_bounds__(256) l32_gemm_kernel(G32 g, const unsigned long long* __restrict__ fail) {
  if (*fail != ~0ull) return;
  __shared__ __align__(16) float As[2][G32_KC][G32_BM];
  __shared__ __align__(16) float Bs[2][G32_KC][G32_BN];
  const int64_t p0 = (int64_t)blockIdx.y * G32_BM, q0 = (int64_t)blockIdx.x * G32_BN;
  if (g.tri) {
    const int64_t pmin_blk = (g.roff + p0) / g.blk;
    const int64_t qmax_blk = (g.coff + (q0 + G32_BN < g.Nc ? q0 + G32_BN : g.Nc) - 1) / g.blk;
    if (pmin_blk > qmax_blk) return;  // wholly inside the strictly-lower block triangle
  }
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  // thread tile: rows ty*4 + {0..3} and 64 + ty*4 + {0..3}; columns tx*4 + {0..3}, 64 + tx*4 + {0..3}
  float acc[8][8], tmp[8][8];
#pragma unroll
  for (int a = 0; a < 8; ++a)
#pragma unroll
    for (int b = 0; b < 8; ++b) acc[a][b] = tmp[a][b] = 0.f;
  const int K = g.kb[g.nkb];
  // loader: 8 x 128 floats per operand per chunk = 1024 = 256 threads x 4
  const int lk = tid >> 5, lc = (tid & 31) * 4;
  auto load = [&](int k0, float4& av, float4& bv) {
    const int k = k0 + lk;
    av = make_float4(0.f, 0.f, 0.f, 0.f);
    bv = av;
    if (k < K) {
      const float* ap = g.A + (int64_t)k * g.lda + p0 + lc;
      const float* bp = g.B + (int64_t)k * g.ldb + q0 + lc;
      if (p0 + lc + 3 < g.Mr) av = *reinterpret_cast<const float4*>(ap);
      else {
        if (p0 + lc + 0 < g.Mr) av.x = ap[0];
        if (p0 + lc + 1 < g.Mr) av.y = ap[1];
        if (p0 + lc + 2 < g.Mr) av.z = ap[2];
      }
      if (q0 + lc + 3 < g.Nc) bv = *reinterpret_cast<const float4*>(bp);
      else {
        if (q0 + lc + 0 < g.Nc) bv.x = bp[0];
        if (q0 + lc + 1 < g.Nc) bv.y = bp[1];
        if (q0 + lc + 2 < g.Nc) bv.z = bp[2];
      }
    }
  };
  float4 av, bv;
  load(0, av, bv);
  *reinterpret_cast<float4*>(&As[0][lk][lc]) = av;
  *reinterpret_cast<float4*>(&Bs[0][lk][lc]) = bv;
  __syncthreads();
  int kbi = 0, next_b = g.kb[1];
  for (int k0 = 0, buf = 0; k0 < K; k0 += G32_KC, buf ^= 1) {
    const bool more = k0 + G32_KC < K;
    if (more) load(k0 + G32_KC, av, bv);
#pragma unroll
    for (int kk = 0; kk < G32_KC; ++kk) {
      const int k = k0 + kk;
      if (k >= K) break;
      if (k == next_b) {  // K-block boundary: tmp = tmp + chain, new chain from 0
#pragma unroll
        for (int a = 0; a < 8; ++a)
#pragma unroll
          for (int b = 0; b < 8; ++b) {
            tmp[a][b] = kbi == 0 ? acc[a][b] : __fadd_rn(tmp[a][b], acc[a][b]);
            acc[a][b] = 0.f;
          }
        ++kbi;
        next_b = g.kb[kbi + 1];
      }
      const float4 a0 = *reinterpret_cast<const float4*>(&As[buf][kk][ty * 4]);
      const float4 a1 = *reinterpret_cast<const float4*>(&As[buf][kk][64 + ty * 4]);
      const float4 b0 = *reinterpret_cast<const float4*>(&Bs[buf][kk][tx * 4]);
      const float4 b1 = *reinterpret_cast<const float4*>(&Bs[buf][kk][64 + tx * 4]);
      const float ar[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
      const float br[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
      for (int a = 0; a < 8; ++a)
#pragma unroll
        for (int b = 0; b < 8; ++b) acc[a][b] = __fmaf_rn(ar[a], br[b], acc[a][b]);
    }
    if (more) {
      *reinterpret_cast<float4*>(&As[buf ^ 1][lk][lc]) = av;
      *reinterpret_cast<float4*>(&Bs[buf ^ 1][lk][lc]) = bv;
    }
    __syncthreads();
  }
#pragma unroll
  for (int a = 0; a < 8; ++a) {
    const int64_t p = p0 + (a < 4 ? ty * 4 + a : 64 + ty * 4 + (a - 4));
    if (p >= g.Mr) continue;
    const int64_t pb = (g.roff + p) / g.blk;
#pragma unroll
    for (int b = 0; b < 8; ++b) {
      const int64_t q = q0 + (b < 4 ? tx * 4 + b : 64 + tx * 4 + (b - 4));
      if (q >= g.Nc) continue;
      if (g.tri && pb > (g.coff + q) / g.blk) continue;
      const float t = kbi == 0 ? acc[a][b] : __fadd_rn(tmp[a][b], acc[a][b]);
      float* cp = g.C + p * g.ldc + q;
      *cp = __fsub_rn(*cp, t);
    }
  }
}

// K-block boundaries of OpenBLAS's threaded level-3 driver: K >= 2Q -> Q, Q < K < 2Q -> ceil(K/2).
static int l32_kblocks(int64_t K, int* kb) {
  int nb = 0;
  int64_t ls = 0;
  kb[nb++] = 0;
  while (ls < K && nb <= L32_MAXKB) {
    int64_t ml = K - ls;
    if (ml >= 2 * L32_Q) ml = L32_Q;
    else if (ml > L32_Q) ml = (ml + 1) / 2;
    ls += ml;
    kb[nb++] = (int)ls;
  }
  return nb - 1;
}

}  // namespace b2d
