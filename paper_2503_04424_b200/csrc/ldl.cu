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

// B2D_LDL_TL (diagnostic): per-launch first-start / last-end %globaltimer of the panel (kind 0)
// and bulk (kind 1) launches, slot = 2 * ((g0 + r0) / LDL_NB) + kind; both fields are
// atomicMin'd (the end as its complement), the buffer starts all-ones.  Null: off.
__device__ unsigned long long* g_ldl_tl = nullptr;
__device__ __forceinline__ unsigned long long gtimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void tl_mark(int64_t slot, bool end) {
  unsigned long long* b = g_ldl_tl;
  if (b == nullptr || threadIdx.x != 0) return;
  const unsigned long long t = gtimer_ns();
  atomicMin(b + 2 * slot + (end ? 1 : 0), end ? ~t : t);
}

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u32(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}
// Panel / bulk pipeline (ldl_factor_block, B2D_LDL_PIPE): each panel kernel and each bulk
// update is launched ahead of its predecessor's completion -- panels on the factor's stream, bulks
// on a second one -- and waits in the kernel (thread 0 of every CTA polls a counter with acquire
// loads) instead of in the stream, so its CTAs take SMs while the predecessor still runs (a launch
// beside the trailing DMMA updates otherwise waits ~100 us for SMs, 256 times per 4096 block).
//   pipe[0] = panels done (panel p releases p + 1 after its writes; 0x7fffffff after a failure)
//   pipe[1] = bulk updates done (the last CTA of bulk p releases p + 1)
//   pipe[2] = CTAs of the running bulk update that finished (reset by its last CTA)
// Every kernel signals even when it returns early (an earlier failure), so nothing waits forever.
constexpr unsigned PIPE_FAIL = 0x7fffffffu;
__device__ __forceinline__ void pipe_wait(const unsigned* c, unsigned v) {
  if (threadIdx.x == 0)
    while (ld_acquire_u32(c) < v) __nanosleep(64);
  __syncthreads();
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
    if (!(fabs(p) >= tol) || tol == 0.0) {  // (tol = 0: an all-zero block, which the reference rejects)
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
#ifdef LDL_PROF  // tools/ldl_prof.cu: per-phase cycle counts of the cluster panel (CTA 0, thread 0)
__device__ long long ldl_prof[16];  // [0, 8): panel steps; [8, 16): one-launch factor phases
#define LDL_MARK(slot)                                   \
  if (c == 0 && tid == 0) {                              \
    const long long now = clock64();                     \
    prof_acc[slot] += now - prof_t;                      \
    prof_t = now;                                        \
  }
#else
#define LDL_MARK(slot)
#endif
constexpr int LC = 16;                 // CTAs per cluster (non-portable size)
constexpr int LC_THREADS = 256;
constexpr int LC_LD = LDL_NB + 1;      // padded smem row (conflict-free column access)
constexpr int LC_RMAX = 384;           // local rows per CTA (n <= LC * LC_RMAX)
#ifndef LDL_PANEL_MINB
#define LDL_PANEL_MINB 1
#endif
__host__ __device__ constexpr size_t ldl_cluster_smem(int rows) { return (size_t)rows * (2 * LC_LD + 2) * 8; }

// Cluster-panel helpers.  Candidates: (|d| bits as hi + 1 : lo, index); hi = 0 marks "none"
// (outside the trailing range, or NaN: a NaN never beats anything, as `better`).
struct Cand {
  uint32_t hi, lo, idx, pad;
};
__device__ __forceinline__ bool cand_better(const Cand& b, const Cand& a) {
  return b.hi > a.hi || (b.hi == a.hi && (b.lo > a.lo || (b.lo == a.lo && b.idx < a.idx)));
}
__device__ __forceinline__ Cand warp_best(const Cand& a) {
  const uint32_t mh = __reduce_max_sync(0xffffffffu, a.hi);
  const uint32_t ml = __reduce_max_sync(0xffffffffu, a.hi == mh ? a.lo : 0u);
  const uint32_t mi = __reduce_min_sync(0xffffffffu, a.hi == mh && a.lo == ml ? a.idx : 0xffffffffu);
  return Cand{mh, ml, mi, 0};
}
__device__ __forceinline__ uint32_t dsmem_map(uint32_t a, int rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}
// 8-byte store into a cluster CTA's shared memory completing 8 tx bytes on its mbarrier.
__device__ __forceinline__ void st_async_f64(uint32_t addr, double v, uint32_t bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];\n" ::"r"(addr),
               "l"(__double_as_longlong(v)), "r"(bar)
               : "memory");
}
__device__ __forceinline__ void mbar_wait_acq_cluster(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// v with the pending steps [tg, k) applied in order, each as fl(v - fl(c_q w_q)) (the reference's
// two roundings): the products are independent, so only the subtractions form the chain.
// Blocks of 8 terms: 8 independent products, then 8 subtractions.
__device__ __forceinline__ double chain_terms(double v, int tg, int k, const double* cr, const double* wc) {
  for (int q0 = tg & ~7; q0 < k; q0 += 8) {
    double p[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) p[u] = __dmul_rn(cr[q0 + u], wc[q0 + u]);
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (q0 + u >= tg && q0 + u < k) v = __dsub_rn(v, p[u]);
  }
  return v;
}
// Two independent chains over the same steps (interleaved).
__device__ __forceinline__ void chain_terms2(double& v, int tv, const double* cv, const double* wv, double& x, int tx,
                                             const double* cx, const double* wx, int k) {
  for (int q0 = min(tv, tx) & ~7; q0 < k; q0 += 8) {
    double p[8], s[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      p[u] = __dmul_rn(cv[q0 + u], wv[q0 + u]);
      s[u] = __dmul_rn(cx[q0 + u], wx[q0 + u]);
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      if (q0 + u >= tv && q0 + u < k) v = __dsub_rn(v, p[u]);
      if (q0 + u >= tx && q0 + u < k) x = __dsub_rn(x, s[u]);
    }
  }
}

// The panel on a cluster of LC CTAs (one per SM), row i in CTA i % LC at local row i / LC, the
// panel's C / W rows and the eager diagonal in shared memory.  One cluster barrier per step:
//   1. each warp's argmax candidate is stored into every CTA; cluster barrier (it also orders
//      the previous step's global writes: raw entries moved between CTAs' rows);
//   2. every warp reduces the candidates -> pivot t; the owners of rows r and t push those rows
//      (C, W, diagonal) into every CTA with st.async, completing on each CTA's mbarrier;
//   3. each thread forms the new column entry of its rows (the interchange, as the single-CTA
//      kernel), scales it and updates its C / W row and diagonal, and takes its candidate for the
//      next step.  A thread only touches its own rows' diagonal entries, so no CTA barrier.
// Rows r, t of the finished L columns (j < r0) are interchanged after the panel (ldl_store_part).
// Entry arithmetic is the single-CTA kernel's exactly.
constexpr int LC_NW = LC_THREADS / 32;
constexpr int LC_ROW = 2 * LDL_NB + 2;  // pushed row: C[0, NB), W[0, NB), diagonal, 1 / diagonal
struct ClusterShared {
  Cand cand[2][LC * LC_NW];
  double rows[2][2][LC_ROW];  // [step parity][0: row r, 1: row t]
  uint64_t bar[2];
  int64_t spos[2 * LDL_NB], ssrc[2 * LDL_NB];
};

__device__ __forceinline__ void cluster_shared_init(ClusterShared& sh) {
  if (threadIdx.x == 0) {
    mbar_init(&sh.bar[0], 1);
    mbar_init(&sh.bar[1], 1);
    fence_mbar_init();
  }
}

__device__ __forceinline__ Cand cand_of(int64_t i, double v) {
  Cand x{0u, 0u, 0xffffffffu, 0u};
  if (!isnan(v)) {
    const unsigned long long bits = (unsigned long long)__double_as_longlong(fabs(v));
    x = Cand{(uint32_t)(bits >> 32) + 1u, (uint32_t)bits, (uint32_t)i, 0u};
  }
  return x;
}

// The nbk steps of the panel at r0; gs0 = steps this kernel ran before (mbarrier phases and
// buffer parity).  Returns false if a step failed (uniform across the cluster, after a cluster
// barrier).  On return the C / W rows of the panel are final in shared memory.
// MRT: rows per thread (R <= MRT * LC_THREADS); Cs / Ws may be shared (<= LC_RMAX rows) or
// global memory (the big-block panel, ldl_panel_cluster_kernel<true>).
template <int MRT = (LC_RMAX + LC_THREADS - 1) / LC_THREADS>
__device__ __forceinline__ bool cluster_panel_steps(const LdlArgs& g, int64_t r0, int nbk, double* Cs, double* Ws,
                                                    double* dg, int R, ClusterShared& sh, int gs0) {
  cg::cluster_group cl = cg::this_cluster();
  const int c = (int)cl.block_rank();
  const int64_t n = g.n, ld = g.ld;
  const int tid = threadIdx.x, lane = tid & 31, wib = tid >> 5;
  double* __restrict__ A = g.A;
  uint8_t* __restrict__ tag = g.tag;
  const double tol = 64.0 * 2.220446049250313e-16 * __longlong_as_double((long long)*g.amax_bits);
  const uint32_t rows_u32 = smem_u32(&sh.rows[0][0][0]), bar_u32 = smem_u32(&sh.bar[0]);
  // step 0's candidate (later steps take theirs in the update)
  Cand my{0u, 0u, 0xffffffffu, 0u};
  for (int li = tid; li < R; li += LC_THREADS) {
    const int64_t i = (int64_t)li * LC + c;
    if (i >= r0 && i < n) {
      const Cand x = cand_of(i, dg[li]);
      if (cand_better(x, my)) my = x;
    }
  }
#ifdef LDL_PROF
  long long prof_acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  long long prof_t = clock64();
#endif
  for (int k = 0; k < nbk; ++k) {
    const int64_t r = r0 + k;
    const int gs = gs0 + k, buf = gs & 1;
    LDL_MARK(0);
    {
      const Cand w = warp_best(my);
      if (lane < LC) *cl.map_shared_rank(&sh.cand[buf][c * LC_NW + wib], lane) = w;
    }
    if (tid == 0) mbar_arrive_expect_tx(&sh.bar[buf], (2u * (2u * k + 1u) + 1u) * 8u);
    LDL_MARK(1);
    cl.sync();  // candidates and the previous step's writes visible cluster-wide
    LDL_MARK(2);
    // raw entries (i, r) of this thread's rows and their tags: every case needs them, and r is
    // known before the pivot (the loads overlap the reduction and the row exchange)
    constexpr int MR = MRT;
    double ar[MR], a2[MR];
    int gr[MR], g2[MR];
#pragma unroll
    for (int m = 0; m < MR; ++m) {
      const int li = tid + m * LC_THREADS;
      const int64_t i = (int64_t)li * LC + c;
      ar[m] = 0.0;
      gr[m] = 0;
      if (li < R && i > r && i < n) {
        ar[m] = __ldcg(A + r * ld + i);
        gr[m] = __ldcg(tag + r * ld + i);
      }
    }
    Cand b = sh.cand[buf][lane];
#pragma unroll
    for (int m = 1; m < LC * LC_NW / 32; ++m) {
      const Cand x = sh.cand[buf][lane + 32 * m];
      if (cand_better(x, b)) b = x;
    }
    b = warp_best(b);
    if (b.hi == 0) {  // no finite diagonal left: the step fails (uniform)
      if (c == 0 && tid == 0) atomicMin(g.fail, (unsigned long long)(g.g0 + r));
      cl.sync();
      return false;
    }
    const int64_t t = b.idx;
    const int orr = (int)(r % LC), ort = (int)(t % LC);
    const int lr = (int)(r / LC), lt = (int)(t / LC);
    // the pivot-dependent raw entries: (t, i) for i < t, (r, r) for i = t, (i, t) for i > t
#pragma unroll
    for (int m = 0; m < MR; ++m) {
      const int li = tid + m * LC_THREADS;
      const int64_t i = (int64_t)li * LC + c;
      a2[m] = 0.0;
      g2[m] = 0;
      if (li < R && i > r && i < n && t != r) {
        const int64_t o = i < t ? i * ld + t : i == t ? r * ld + r : t * ld + i;
        a2[m] = __ldcg(A + o);
        g2[m] = __ldcg(tag + o);
      }
    }
    // owners push rows r (slot 0) and t (slot 1): thread 128 * slot + e pushes element e
    {
      const int slot = tid >> 7, e = tid & 127;
      const int owner = slot ? ort : orr, lrow = slot ? lt : lr;
      if (slot < 2 && c == owner &&
          (e < k || (e >= LDL_NB && e < LDL_NB + k) || e == 2 * LDL_NB || (slot == 1 && e == 2 * LDL_NB + 1))) {
        const double v = e < LDL_NB       ? Cs[(size_t)lrow * LC_LD + e]
                         : e < 2 * LDL_NB ? Ws[(size_t)lrow * LC_LD + e - LDL_NB]
                         : e == 2 * LDL_NB ? dg[lrow]
                                           : 1.0 / dg[lrow];
        const uint32_t off = rows_u32 + (uint32_t)(((buf * 2 + slot) * LC_ROW + e) * 8);
        const uint32_t bo = bar_u32 + (uint32_t)(buf * 8);
#pragma unroll 4
        for (int d = 0; d < LC; ++d) st_async_f64(dsmem_map(off, d), v, dsmem_map(bo, d));
      }
    }
    LDL_MARK(3);
    mbar_wait_acq_cluster(&sh.bar[buf], (uint32_t)((gs >> 1) & 1));
    LDL_MARK(4);
    const double* rr = sh.rows[buf][0];
    const double* rt = sh.rows[buf][1];
    const double p = rt[2 * LDL_NB];  // row t's eager diagonal: the pivot
    if (!(fabs(p) >= tol) || tol == 0.0) {  // (tol = 0: an all-zero block, which the reference rejects)
      if (c == 0 && tid == 0) atomicMin(g.fail, (unsigned long long)(g.g0 + r));
      cl.sync();
      return false;  // uniform across the cluster: every thread read the same p
    }
    if (c == 0 && tid == 0) {
      g.d[r] = p;
      g.swaps[r] = t;
    }
    const double invp = rt[2 * LDL_NB + 1];
    // interchange in shared memory: row r's slot takes row t's C / W (row t's slot is rewritten
    // below with row r's, as its owner's row loop forms the new entry of position t)
    if (t != r) {
      if (c == orr && tid < k) {
        Cs[(size_t)lr * LC_LD + tid] = rt[tid];
        Ws[(size_t)lr * LC_LD + tid] = rt[LDL_NB + tid];
      }
      if (c == ort && tid >= 128 && tid < 128 + k) {
        Cs[(size_t)lt * LC_LD + tid - 128] = rr[tid - 128];
        Ws[(size_t)lt * LC_LD + tid - 128] = rr[LDL_NB + tid - 128];
      }
    }
    if (c == orr && tid == (lr % LC_THREADS)) dg[lr] = p;
    my = Cand{0u, 0u, 0xffffffffu, 0u};
#pragma unroll
    for (int m = 0; m < MR; ++m) {
      const int li = tid + m * LC_THREADS;
      const int64_t i = (int64_t)li * LC + c;
      if (li >= R || i <= r || i >= n) continue;
      const double* Ci = Cs + (size_t)li * LC_LD;
      const double* Wi = Ws + (size_t)li * LC_LD;
      double v, dnew = dg[li];
      if (t == r) {
        v = chain_terms(ar[m], gr[m], k, Ci, rr + LDL_NB);
      } else if (i < t) {
        // (t, i) -> (i, r); (i, r) -> (t, i): brought up to date, tagged
        v = a2[m];
        double x = ar[m];
        chain_terms2(v, g2[m], rt, Wi, x, gr[m], Ci, rr + LDL_NB, k);
        A[i * ld + t] = x;
        tag[i * ld + t] = (uint8_t)k;
      } else if (i == t) {
        v = chain_terms(ar[m], gr[m], k, rt, rr + LDL_NB);           // (t, r) stays
        A[t * ld + t] = a2[m];                                     // (r, r) -> (t, t) with its pending terms
        tag[t * ld + t] = (uint8_t)g2[m];
        dnew = rr[2 * LDL_NB];                                     // row r's diagonal moves to position t
      } else {
        v = chain_terms(a2[m], g2[m], k, Ci, rt + LDL_NB);           // (i, t) -> (i, r)
        A[t * ld + i] = ar[m];                                     // (i, r) -> (i, t) with its tag
        tag[t * ld + i] = (uint8_t)gr[m];
      }
      const double w = __dmul_rn(v, invp);  // work[i] = a_ir * (1/p)
      Cs[(size_t)li * LC_LD + k] = v;
      Ws[(size_t)li * LC_LD + k] = w;
      const double dn = __dsub_rn(dnew, __dmul_rn(v, w));
      dg[li] = dn;
      const Cand x = cand_of(i, dn);
      if (cand_better(x, my)) my = x;
    }
    LDL_MARK(5);
  }
  cl.sync();  // every push landed; C / W rows final
#ifdef LDL_PROF
  if (c == 0 && tid == 0)
    for (int q = 0; q < 8; ++q) ldl_prof[q] += prof_acc[q];
#endif
  return true;
}

// C and W rows of the panel (rows > r0) back to global memory for the store and bulk phases;
// with store_l also the finished L columns (L = W below the diagonal, _ldl.pyx:59-60).
__device__ __forceinline__ void cluster_panel_writeback(const LdlArgs& g, int64_t r0, int nbk, const double* Cs,
                                                        const double* Ws, int R, int c, bool store_l) {
  for (int li = threadIdx.x; li < R; li += LC_THREADS) {
    const int64_t i = (int64_t)li * LC + c;
    if (i >= g.n || i <= r0) continue;
    for (int q = 0; q < nbk; ++q) {
      const double w = Ws[(size_t)li * LC_LD + q];
      g.C[q * g.ld + i] = Cs[(size_t)li * LC_LD + q];
      g.W[q * g.ld + i] = w;
      if (store_l && i > r0 + q) g.A[(r0 + q) * g.ld + i] = w;
    }
  }
}

// BIG: blocks of up to LC * LC_RMAX_BIG rows (the reference's memory-sized blocks, C5: b = 39322):
// the rows' C / W histories live in global memory (`rows`, [LC][2][R][LC_LD], each CTA its own
// slab, read back through L2 after every step's barrier), only the eager diagonal stays in shared
// memory.  Same steps and arithmetic as the shared-memory panel.
constexpr int LC_RMAX_BIG = 2560;
__host__ __device__ constexpr size_t ldl_big_rows_bytes(int64_t n) {
  return (size_t)LC * 2 * (size_t)((n + LC - 1) / LC) * LC_LD * 8;
}
template <bool BIG>
__global__ void __launch_bounds__(LC_THREADS, LDL_PANEL_MINB) ldl_panel_cluster_kernel(LdlArgs g, int64_t r0, int nbk,
                                                                                   unsigned* pipe, unsigned pidx,
                                                                                   double* rows) {
  cg::cluster_group cl = cg::this_cluster();
  const int c = (int)cl.block_rank();
  if (pipe && pidx > 0) pipe_wait(pipe + 1, pidx);  // bulk update pidx - 1 done
  if (*g.fail != ~0ull) {  // uniform: written by earlier kernels only
    if (pipe && c == 0 && threadIdx.x == 0) st_release_u32(pipe, PIPE_FAIL);
    return;
  }
  const int64_t tls = 2 * ((g.g0 + r0) / LDL_NB);
  tl_mark(tls, false);
  extern __shared__ double sm[];
  const int R = (int)((g.n + LC - 1) / LC);
  double* Cs = BIG ? rows + (size_t)c * 2 * R * LC_LD : sm;  // [R][LC_LD]
  double* Ws = Cs + (size_t)R * LC_LD;                        // [R][LC_LD]
  double* dg = BIG ? sm : Ws + (size_t)R * LC_LD;             // [R] eager diagonal
  __shared__ ClusterShared sh;
  cluster_shared_init(sh);
  for (int li = threadIdx.x; li < R; li += LC_THREADS) {
    const int64_t i = (int64_t)li * LC + c;
    dg[li] = i < g.n ? g.diag[i] : 0.0;
  }
  __syncthreads();  // dg loaded, barriers initialised
  cl.sync();        // every CTA's barriers initialised before any remote arrive
  constexpr int MRT = BIG ? (LC_RMAX_BIG + LC_THREADS - 1) / LC_THREADS : (LC_RMAX + LC_THREADS - 1) / LC_THREADS;
  if (!cluster_panel_steps<MRT>(g, r0, nbk, Cs, Ws, dg, R, sh, 0)) {
    if (pipe && c == 0 && threadIdx.x == 0) st_release_u32(pipe, PIPE_FAIL);
    return;
  }
  cluster_panel_writeback(g, r0, nbk, Cs, Ws, R, c, true);
  for (int li = threadIdx.x; li < R; li += LC_THREADS) {
    const int64_t i = (int64_t)li * LC + c;
    if (i < g.n && i > r0) g.diag[i] = dg[li];
  }
  if (pipe) {  // every CTA's writes visible device-wide, then panel pidx is released
    __threadfence();
    cl.sync();
    if (c == 0 && threadIdx.x == 0) st_release_u32(pipe, pidx + 1);
  }
  tl_mark(tls, true);
}

// Finished columns [r0, r0 + nbk): L = W below the diagonal (_ldl.pyx:59-60); and the panel's
// interchanges applied to rows of the finished columns j < r0 (the reference swaps rows r, t of
// those columns at every step, _ldl.pyx:38-46): warp 0 folds the panel's swaps into one
// permutation of at most 2 * NB rows (spos / ssrc, in shared memory), then one warp per column
// gathers and scatters them.  Work item w of nw (CTA-granular).
__device__ __forceinline__ void ldl_swap_part(const LdlArgs& g, int64_t r0, int nbk, int64_t* spos, int64_t* ssrc,
                                              int64_t w, int64_t nw) {
  const int tid = threadIdx.x, lane = tid & 31;
  const int nthr = blockDim.x;
  if (r0 > 0 && tid < 32) {
    int64_t dcur = r0 + lane;        // row whose value ends at position r0 + lane
    int64_t xpos = -1, xcur = -1;    // extra position `lane` (beyond the panel) and its row
    int nx = 0;
    for (int k = 0; k < nbk; ++k) {
      const int64_t a = r0 + k, b = __ldcg(g.swaps + a);
      if (b == a) continue;
      const bool direct = b < r0 + nbk;
      int hb;
      if (direct) {
        hb = (int)(b - r0);
      } else {
        const unsigned m = __ballot_sync(0xffffffffu, xpos == b);
        if (m) {
          hb = __ffs(m) - 1;
        } else {
          hb = nx++;
          if (lane == hb) xpos = xcur = b;
        }
      }
      const int64_t va = __shfl_sync(0xffffffffu, dcur, k);
      const int64_t vb = direct ? __shfl_sync(0xffffffffu, dcur, hb) : __shfl_sync(0xffffffffu, xcur, hb);
      if (lane == k) dcur = vb;
      if (lane == hb) {
        if (direct) dcur = va;
        else xcur = va;
      }
    }
    const bool dv = lane < nbk && dcur != r0 + lane, xv = lane < nx && xcur != xpos;
    spos[lane] = dv ? r0 + lane : -1;
    ssrc[lane] = dcur;
    spos[32 + lane] = xv ? xpos : -1;
    ssrc[32 + lane] = xcur;
  }
  __syncthreads();
  if (r0 > 0) {
    const int64_t p0 = spos[lane], p1 = spos[32 + lane], s0 = ssrc[lane], s1 = ssrc[32 + lane];
    const int64_t ld = g.ld;
    for (int64_t j = (w * nthr + tid) >> 5; j < r0; j += (nw * nthr) >> 5) {
      double* colj = g.A + j * ld;
      const double v0 = p0 >= 0 ? __ldcg(colj + s0) : 0.0;
      const double v1 = p1 >= 0 ? __ldcg(colj + s1) : 0.0;
      __syncwarp();
      if (p0 >= 0) colj[p0] = v0;
      if (p1 >= 0) colj[p1] = v1;
    }
  }
}

__device__ __forceinline__ void ldl_store_part(const LdlArgs& g, int64_t r0, int nbk, int64_t* spos, int64_t* ssrc,
                                               int64_t w, int64_t nw) {
  ldl_swap_part(g, r0, nbk, spos, ssrc, w, nw);
  const int tid = threadIdx.x, nthr = blockDim.x;
  const int64_t rows = g.n - r0;
  for (int64_t e = w * nthr + tid; e < rows * nbk; e += nw * nthr) {
    const int k = (int)(e / rows);
    const int64_t i = r0 + e % rows, r = r0 + k;
    if (i > r) g.A[r * g.ld + i] = __ldcg(g.W + k * g.ld + i);
  }
}

__global__ void __launch_bounds__(256) ldl_store_l_kernel(LdlArgs g, int64_t r0, int nbk) {
  if (*g.fail != ~0ull) return;
  __shared__ int64_t spos[2 * LDL_NB], ssrc[2 * LDL_NB];
  ldl_store_part(g, r0, nbk, spos, ssrc, blockIdx.x, gridDim.x);
}

// Trailing update with the panel's nbk steps: a_ij -= c_i^q w_j^q for q = tag_ij .. nbk-1, in
// order, for j >= r0 + nbk, i >= j; tags reset.  64 x 64 entry tiles, 4 x 4 per thread (256
// threads); tile b of the lower tile triangle (column-major).
constexpr int LDL_BT = 64;
// 4 CTAs per SM worth of registers (<= 64 per thread): a bulk CTA then fits on an SM that runs a
// DMMA Schur-update CTA (288 threads x 168 registers, 128 KB shared), so the factor's bulk steps
// start at once beside the trailing updates instead of waiting for SMs to drain
#ifndef LDL_BULK_MINB
#define LDL_BULK_MINB 4
#endif
__device__ __forceinline__ void ldl_bulk_tile(const LdlArgs& g, int64_t r0, int nbk, int64_t b, double* sC,
                                              double* sW) {
  const int64_t re = r0 + nbk, m = g.n - re, ld = g.ld, n = g.n;
  const int64_t nbt = (m + LDL_BT - 1) / LDL_BT;
  // tile b of the column-major lower triangle: column bj = the largest j with
  // off(j) = j nbt - j (j - 1) / 2 <= b (closed form, then exact integer fix-up; a linear search
  // here was ~15% of the kernel's issue slots)
  const double qa = (double)(2 * nbt + 1);
  int64_t bj = (int64_t)((qa - sqrt(qa * qa - 8.0 * (double)b)) * 0.5);
  if (bj < 0) bj = 0;
  auto off = [nbt](int64_t j) { return j * nbt - j * (j - 1) / 2; };
  while (bj > 0 && off(bj) > b) --bj;
  while (bj + 1 < nbt && off(bj + 1) <= b) ++bj;
  b -= off(bj);
  const int64_t bi = bj + b;
  const int64_t i0 = re + bi * LDL_BT, j0 = re + bj * LDL_BT;
  // the panel's C / W rows of this tile staged with asynchronous 16-byte copies (zero-filled past
  // the block), in flight while the entries themselves are loaded (a register round trip per
  // element made every copy wait for its load)
  for (int e = threadIdx.x; e < nbk * (LDL_BT / 2); e += 256) {
    const int q = e / (LDL_BT / 2), x = 2 * (e % (LDL_BT / 2));
    const int64_t ci = i0 + x, wj = j0 + x;
    const uint32_t cb = ci < n ? (ci + 1 < n ? 16u : 8u) : 0u, wb = wj < n ? (wj + 1 < n ? 16u : 8u) : 0u;
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(sC + q * LDL_BT + x)),
                 "l"(g.C + q * ld + (cb ? ci : 0)), "r"(cb)
                 : "memory");
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(sW + q * LDL_BT + x)),
                 "l"(g.W + q * ld + (wb ? wj : 0)), "r"(wb)
                 : "memory");
  }
  asm volatile("cp.async.commit_group;\n" ::: "memory");
  // thread (tx, ty): rows i0 + 2 tx + (a & 1) + 32 (a >> 1), columns j0 + 4 ty + c (a, c < 4): the
  // C pairs (2 tx, 2 tx + 1) are conflict-free 16-byte shared loads (a stride of 4 rows per thread
  // made them 2-way bank conflicts, ncu: short-scoreboard stalls first)
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int64_t ib = i0 + 2 * tx, jb = j0 + 4 * ty;
  // per-thread base pointers and 32-bit column strides (the block has < 2^31 entries): fewer
  // 64-bit index registers under the kernel's 64-register cap
  double* const Ab = g.A + jb * ld + ib;
  uint8_t* const Tb = g.tag + jb * ld + ib;
  const int ldi = (int)ld;
  auto roff = [](int a) { return (a & 1) + 32 * (a >> 1); };
  // interior off-diagonal tiles: vector loads / stores (i0 is a multiple of 32, ld of 128)
  const bool vec = bi > bj && i0 + LDL_BT <= n && j0 + LDL_BT <= n;
  double v[4][4];
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const int64_t j = jb + c;
    if (vec) {
      const double2 x0 = __ldcg(reinterpret_cast<const double2*>(Ab + c * ldi));
      const double2 x1 = __ldcg(reinterpret_cast<const double2*>(Ab + c * ldi + 32));
      v[0][c] = x0.x;
      v[1][c] = x0.y;
      v[2][c] = x1.x;
      v[3][c] = x1.y;
    } else {
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        const int64_t i = ib + roff(a);
        const bool ok = i < n && j < n && i >= j;
        v[a][c] = ok ? __ldcg(Ab + c * ldi + roff(a)) : 0.0;
      }
    }
  }
  asm volatile("cp.async.wait_all;\n" ::: "memory");
  __syncthreads();
  uint32_t tw[4];  // tags of the 4 rows of column c, one byte each
  bool tagged = false;
  {
    // every term on every entry (the fast path); entries that already hold some of the panel's
    // steps (tag > 0, rare: rows / columns moved by the panel's interchanges) are redone below
    // from their loaded value with the terms [tag, nbk) only -- each entry still sees exactly
    // its terms, in order, with the reference's two roundings
    for (int q = 0; q < nbk; ++q) {
      const double2 c01 = *reinterpret_cast<const double2*>(sC + q * LDL_BT + 2 * tx);
      const double2 c23 = *reinterpret_cast<const double2*>(sC + q * LDL_BT + 32 + 2 * tx);
      const double2 w01 = *reinterpret_cast<const double2*>(sW + q * LDL_BT + 4 * ty);
      const double2 w23 = *reinterpret_cast<const double2*>(sW + q * LDL_BT + 4 * ty + 2);
      const double cc[4] = {c01.x, c01.y, c23.x, c23.y}, ww[4] = {w01.x, w01.y, w23.x, w23.y};
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int c = 0; c < 4; ++c) v[a][c] = __dsub_rn(v[a][c], __dmul_rn(cc[a], ww[c]));
    }
    // the tags (only read now: nothing before the terms needs them, and their loads would hold
    // registers or the first term)
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int64_t j = jb + c;
      if (vec) {
        tw[c] = (uint32_t)__ldcg(reinterpret_cast<const unsigned short*>(Tb + c * ldi)) |
                ((uint32_t)__ldcg(reinterpret_cast<const unsigned short*>(Tb + c * ldi + 32)) << 16);
      } else {
        tw[c] = 0;
#pragma unroll
        for (int a = 0; a < 4; ++a) {
          const int64_t i = ib + roff(a);
          const bool ok = i < n && j < n && i >= j;
          tw[c] |= (uint32_t)(ok ? __ldcg(Tb + c * ldi + roff(a)) : 0) << (8 * a);
        }
      }
      tagged |= tw[c] != 0;
    }
    if (tagged) {
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const int tg = (int)((tw[c] >> (8 * a)) & 0xffu);
          if (tg) {
            const int64_t i = ib + roff(a), j = jb + c;
            double x = __ldcg(Ab + c * ldi + roff(a));
            for (int q = tg; q < nbk; ++q)
              x = __dsub_rn(x, __dmul_rn(sC[q * LDL_BT + 2 * tx + roff(a)], sW[q * LDL_BT + 4 * ty + c]));
            v[a][c] = x;
          }
        }
    }
  }
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const int64_t j = jb + c;
    if (vec) {
      *reinterpret_cast<double2*>(Ab + c * ldi) = make_double2(v[0][c], v[1][c]);
      *reinterpret_cast<double2*>(Ab + c * ldi + 32) = make_double2(v[2][c], v[3][c]);
      if (tw[c] & 0xffffu) *reinterpret_cast<unsigned short*>(Tb + c * ldi) = 0;
      if (tw[c] >> 16) *reinterpret_cast<unsigned short*>(Tb + c * ldi + 32) = 0;
    } else {
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        const int64_t i = ib + roff(a);
        if (i < n && j < n && i >= j) {
          Ab[c * ldi + roff(a)] = v[a][c];
          if ((tw[c] >> (8 * a)) & 0xffu) Tb[c * ldi + roff(a)] = 0;
        }
      }
    }
  }
  __syncthreads();  // sC / sW reused by the next tile
}

// Blocks [0, ntile): the bulk tiles; blocks [ntile, gridDim.x): the panel's row interchanges on
// the finished L columns (after the cluster panel kernel, which stores the panel's L itself).
// pipeline: this CTA's writes visible device-wide; the last CTA of the launch releases bulk pidx
__device__ __forceinline__ void bulk_done(unsigned* pipe, unsigned pidx) {
  if (!pipe) return;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(pipe + 2, 1u) == gridDim.x - 1) {
      pipe[2] = 0u;  // (the next bulk launch is stream-ordered after this one)
      __threadfence();
      st_release_u32(pipe + 1, pidx + 1);
    }
  }
}
__global__ void __launch_bounds__(256, LDL_BULK_MINB) ldl_bulk_kernel(LdlArgs g, int64_t r0, int nbk, int64_t ntile,
                                                                     unsigned* pipe, unsigned pidx) {
  if (pipe) pipe_wait(pipe, pidx + 1);  // panel pidx done (or failed)
  if (*g.fail != ~0ull) {
    bulk_done(pipe, pidx);
    return;
  }
  const int64_t tls = 2 * ((g.g0 + r0) / LDL_NB) + 1;
  tl_mark(tls, false);
  __shared__ __align__(16) double sC[LDL_NB * LDL_BT];
  __shared__ __align__(16) double sW[LDL_NB * LDL_BT];
  if ((int64_t)blockIdx.x >= ntile) {
    __shared__ int64_t spos[2 * LDL_NB], ssrc[2 * LDL_NB];
    ldl_swap_part(g, r0, nbk, spos, ssrc, (int64_t)blockIdx.x - ntile, (int64_t)gridDim.x - ntile);
    tl_mark(tls, true);
    bulk_done(pipe, pidx);
    return;
  }
  // the first tile-column (the next panel's columns) last, so that it is L2-resident when the
  // next panel kernel reads it
  ldl_bulk_tile(g, r0, nbk, ntile - 1 - blockIdx.x, sC, sW);
  tl_mark(tls, true);
  bulk_done(pipe, pidx);
}

// The whole pivoted factorisation of the block on one 16-CTA cluster (one launch): per panel
// the cluster steps, then the store / interchange and the bulk update spread over the cluster's
// CTAs, with cluster barriers between the phases.  It holds its 16 SMs from start to end, so it
// runs beside the trailing DMMA updates of the previous stage at full speed (the per-panel
// kernels would each wait for SMs there).  Same arithmetic as the per-panel kernels.
__host__ __device__ constexpr size_t ldl_factor_smem(int rows) {
  return ((size_t)rows + 1 + (2 * (size_t)rows * LC_LD > 2 * (size_t)LDL_NB * LDL_BT ? 2 * (size_t)rows * LC_LD
                                                                                  : 2 * (size_t)LDL_NB * LDL_BT)) * 8;
}
__global__ void __launch_bounds__(LC_THREADS, 1) ldl_factor_cluster_kernel(LdlArgs g) {
  if (*g.fail != ~0ull) return;
  cg::cluster_group cl = cg::this_cluster();
  const int c = (int)cl.block_rank();
  extern __shared__ double sm[];
  const int64_t n = g.n, ld = g.ld;
  const int R = (int)((n + LC - 1) / LC);
  double* dg = sm;                      // [R] eager diagonal (kept across panels)
  double* Cs = dg + ((R + 1) & ~1);     // [R][LC_LD] (panel phase) / bulk staging C (16-byte aligned)
  double* Ws = Cs + (size_t)R * LC_LD;  // [R][LC_LD]
  double* sC = Cs;                      // bulk phase: [NB][BT] x 2
  double* sW = Cs + LDL_NB * LDL_BT;
  __shared__ ClusterShared sh;
  cluster_shared_init(sh);
  for (int li = threadIdx.x; li < R; li += LC_THREADS) {
    const int64_t i = (int64_t)li * LC + c;
    dg[li] = i < n ? g.A[i * ld + i] : 0.0;
  }
  __syncthreads();
  cl.sync();
#ifdef LDL_PROF
  const int tid = threadIdx.x;
  long long prof_acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  long long prof_t = clock64();
#define FMARK(slot) LDL_MARK(slot)
#else
#define FMARK(slot)
#endif
  for (int64_t r0 = 0; r0 < n; r0 += LDL_NB) {
    const int nbk = (int)(n - r0 < LDL_NB ? n - r0 : LDL_NB);
    FMARK(0);
    if (!cluster_panel_steps(g, r0, nbk, Cs, Ws, dg, R, sh, (int)r0)) return;
    FMARK(1);
    cluster_panel_writeback(g, r0, nbk, Cs, Ws, R, c, false);
    cl.sync();  // C / W rows and the panel's interchanges visible cluster-wide
    FMARK(2);
    ldl_store_part(g, r0, nbk, sh.spos, sh.ssrc, c, LC);
    FMARK(3);
    const int64_t m = n - r0 - nbk;
    if (m > 0) {
      const int64_t nbt = (m + LDL_BT - 1) / LDL_BT, ntile = nbt * (nbt + 1) / 2;
      for (int64_t b = c; b < ntile; b += LC) ldl_bulk_tile(g, r0, nbk, ntile - 1 - b, sC, sW);
    }
    FMARK(4);
    cl.sync();  // the trailing block up to date before the next panel reads it
    FMARK(5);
  }
#ifdef LDL_PROF
  if (c == 0 && tid == 0)
    for (int q = 0; q < 8; ++q) ldl_prof[8 + q] += prof_acc[q];
#endif
#undef FMARK
}

// Panel server: the block's panels on one 16-CTA cluster that holds its SMs for the whole factor
// (so the latency-bound pivot steps never share an SM with the trailing DMMA updates), while each
// panel's bulk update runs as an ordinary kernel on every SM (ldl_bulk_kernel: <= 64 registers,
// so its CTAs fit beside a Schur-update CTA).  Hand-off through two counters in global memory:
// flags[0] = panels finished (the server releases it after the panel's L columns and row
// interchanges are stored; the host gates panel p's bulk launch on it with a stream wait-value),
// flags[1] = bulk updates finished (a stream write-value after each bulk launch; the server
// acquires it before the next panel).  Same steps, same arithmetic as the per-panel kernels.
__global__ void __launch_bounds__(LC_THREADS, 1) ldl_panel_server_kernel(LdlArgs g, unsigned* flags) {
  cg::cluster_group cl = cg::this_cluster();
  const int c = (int)cl.block_rank();
  extern __shared__ double sm[];
  const int64_t n = g.n, ld = g.ld;
  const int R = (int)((n + LC - 1) / LC);
  double* Cs = sm;                      // [R][LC_LD]
  double* Ws = Cs + (size_t)R * LC_LD;  // [R][LC_LD]
  double* dg = Ws + (size_t)R * LC_LD;  // [R] eager diagonal (kept across panels)
  __shared__ ClusterShared sh;
  cluster_shared_init(sh);
  if (*g.fail != ~0ull) {  // an earlier block failed: release every gated bulk launch
    if (c == 0 && threadIdx.x == 0) st_release_u32(flags, 0x7fffffffu);
    return;
  }
  for (int li = threadIdx.x; li < R; li += LC_THREADS) {
    const int64_t i = (int64_t)li * LC + c;
    dg[li] = i < n ? __ldcg(g.A + i * ld + i) : 0.0;
  }
  __syncthreads();
  cl.sync();
  unsigned p = 0;
  for (int64_t r0 = 0; r0 < n; r0 += LDL_NB, ++p) {
    const int nbk = (int)(n - r0 < LDL_NB ? n - r0 : LDL_NB);
    if (p > 0) {  // panel p - 1's bulk update is in
      if (threadIdx.x == 0)
        while (ld_acquire_u32(flags + 1) < p) __nanosleep(128);
      __syncthreads();
    }
    if (!cluster_panel_steps(g, r0, nbk, Cs, Ws, dg, R, sh, (int)r0)) {
      if (c == 0 && threadIdx.x == 0) st_release_u32(flags, 0x7fffffffu);
      return;
    }
    cluster_panel_writeback(g, r0, nbk, Cs, Ws, R, c, false);
    cl.sync();  // C / W rows and the panel's interchanges visible cluster-wide
    ldl_store_part(g, r0, nbk, sh.spos, sh.ssrc, c, LC);
    __threadfence();
    cl.sync();  // every CTA's stores done before the release
    if (c == 0 && threadIdx.x == 0) st_release_u32(flags, p + 1);
  }
}

// swaps -> block permutation (kernels/dense.py:25-30), global perm (memdet.py:352-353),
// ell = log|d| (memdet.py:406) and the D values.  One thread walks the swaps (sequential by
// definition) on a shared-memory copy of the permutation when it fits (LDL_FINISH_SMEM_MAX rows).
constexpr int64_t LDL_FINISH_SMEM_MAX = 24576;
__global__ void ldl_finish_kernel(const int64_t* __restrict__ swaps, const double* __restrict__ d, int64_t n,
                                  int64_t g0, int64_t* __restrict__ perm_local, int64_t* __restrict__ perm_global,
                                  double* __restrict__ ell, double* __restrict__ dout, int64_t perm_lo) {
  // perm_lo: block-permutation entries below it were already written by ldl_partial_perm_kernel
  // (group pipeline; shared-memory walk only) and may be in use: not rewritten
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
      if (sm && i >= perm_lo) perm_local[i] = pl[i];
      perm_global[g0 + i] = g0 + pl[i];
    }
  }
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    ell[g0 + i] = log(fabs(d[i]));
    dout[g0 + i] = d[i];
  }
}

// Group pipeline (engine.cu ldl_factor_block, B2D_LDL_GROUPS): entries [e0, e1) of the block
// permutation once steps [0, e1) are done -- step r interchanges positions r and t > r, so
// positions below e1 never change again (kernels/dense.py:25-30 applied to a prefix of the swaps).
__global__ void ldl_partial_perm_kernel(const int64_t* __restrict__ swaps, int64_t n, int64_t e0, int64_t e1,
                                        int64_t* __restrict__ perm_local) {
  extern __shared__ int64_t sperm[];  // n entries (n <= LDL_FINISH_SMEM_MAX)
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) sperm[i] = i;
  __syncthreads();
  if (threadIdx.x == 0)
    for (int64_t r = 0; r < e1; ++r) {
      const int64_t t = __ldcg(swaps + r);
      if (t > r && t < n) {
        const int64_t x = sperm[r];
        sperm[r] = sperm[t];
        sperm[t] = x;
      }
    }
  __syncthreads();
  for (int64_t i = e0 + threadIdx.x; i < e1; i += blockDim.x) perm_local[i] = sperm[i];
}

// Tile rows [I0, I0 + gridDim.x / ncol) of the dense unit-lower factor -> tile grid, tile columns
// J <= I (the rows of a finished column group: final once its last panel's interchanges are in).
__global__ void __launch_bounds__(256) pack_unit_lower_rows_kernel(const double* __restrict__ dense, int64_t ld,
                                                                   int64_t n, TileMap dst, int I0, int ncol) {
  const int I = I0 + (int)(blockIdx.x / (unsigned)ncol), J = (int)(blockIdx.x % (unsigned)ncol);
  if (J > I) return;
  double* t = dst.tile(I, J);
  for (int o = threadIdx.x; o < TILE_ELEMS; o += 256) {
    const int r = (o >> 3) & 127;
    const int c = ((o >> 10) << 3) + iperm8(o & 7);
    const int64_t R = (int64_t)I * T + r, C = (int64_t)J * T + c;
    double v;
    if (R == C) v = 1.0;
    else if (R > C && R < n) v = __ldcg(dense + C * ld + R);
    else v = 0.0;
    t[o] = v;
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
// One CTA per diagonal tile q = q0 + blockIdx.x of `map`: inv + q * TILE_ELEMS = L_qq^{-1}.
__global__ void __launch_bounds__(128) tile_inv_unit_kernel(TileMap map, double* __restrict__ inv_base, int q0) {
  extern __shared__ double M[];  // [T][129]
  const int q = q0 + (int)blockIdx.x;
  const double* __restrict__ tile = map.tile(q, q);
  double* __restrict__ inv = inv_base + (int64_t)q * TILE_ELEMS;
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

// The same for panel columns [c0, c0 + ctiles T) only (group pipeline: the permutation's entries
// of a finished column group are final before the factor ends); dst, perm and n are the whole panel's.
__global__ void permute_cols_range_kernel(TileMap src, TileMap dst, int rtiles, int64_t c0, int ctiles, int64_t n,
                                          const int64_t* __restrict__ perm) {
  const int64_t rows = (int64_t)rtiles * T, cols = (int64_t)ctiles * T;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < rows * cols; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = c0 + e / rows, i = e % rows;
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
