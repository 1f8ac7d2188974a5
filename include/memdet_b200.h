/*
 * memdet_b200.h — C ABI of the B200-native MEMDET engine (libmemdet_b200.so).
 *
 * The engine computes the blocked LDL^T / Cholesky log-determinant of a dense symmetric
 * positive-definite matrix on one B200 (sm_100a) and returns every leading-principal-minor
 * log-determinant (the "prefix").  Plain C types only; no torch types cross this boundary.
 *
 * Reference interfaces replaced (paths relative to the oocdet 0.1.0 package, pkg/src/oocdet):
 *   b2d_memdet_sym          <- memdet_cholesky   memdet.py:415-433  (mode B2D_MODE_CHOLESKY)
 *                              memdet_ldl        memdet.py:392-412  (mode B2D_MODE_LDL_*)
 *                              driver body       memdet.py:322-389  (_memdet_symmetric)
 *                              memdet_lu         memdet.py:268-319  (mode B2D_MODE_LU, the
 *                                                generic walk; reads every block)
 *   b2d_ctx_*               <- the same driver, split so inputs can stay resident in HBM
 *   return codes            <- oocdet.errors                 errors.py:8-51
 *
 * Matrices are row-major (the MEMDET01 data region, storage.py:3-16) with a leading dimension
 * in elements.  The symmetric modes read only the row-major upper tile triangle (the (i <= j)
 * tiles the reference reads); inputs are borrowed read-only and never modified.
 * Every call blocks until the device work it issued has finished, except
 * b2d_ctx_factor_device_async, which only enqueues on the caller's stream.
 */
#ifndef MEMDET_B200_H
#define MEMDET_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* return codes (map to oocdet.errors; errors.py:8-51) */
#define B2D_OK 0
#define B2D_ERR_USAGE 2        /* ValueError / usage (exit 2)                       */
#define B2D_ERR_NOT_SPD 3      /* NotSpdError (NumericalError, exit 3)              */
#define B2D_ERR_INDEFINITE 4   /* IndefiniteBlockError (NumericalError, exit 3)     */
#define B2D_ERR_CUDA 5         /* device / driver failure                           */
#define B2D_ERR_NOMEM 6        /* HBM budget exceeded                               */
#define B2D_ERR_UNSUPPORTED 7  /* feature not built                                 */
#define B2D_ERR_STORAGE 8      /* StorageError: scratchpad file (exit 4)            */

/* dtype codes: identical to the MEMDET01 header byte (storage.py:40-41) */
#define B2D_F64 0
#define B2D_F32 1

/* factorisation modes */
#define B2D_MODE_CHOLESKY 0    /* memdet_cholesky: d = diag(L), prefix = cumsum 2 log d     */
#define B2D_MODE_LDL_NOPIV 1   /* memdet_ldl without pivoting: d = L_ii^2, perm = identity  */
#define B2D_MODE_LDL_PIV 2     /* memdet_ldl with block-local 1x1 pivots (_ldl.pyx:30-46):
                                  the reference's b x b block walk, d = D, perm = pivots    */
#define B2D_MODE_LU 3          /* memdet_lu (generic matrix, memdet.py:268-319): block-local
                                  partial pivoting in the reference's generic block walk;
                                  d = U_ii, perm = pivots, prefix[m-1] = log|det|; a zero
                                  pivot (singular) sets fail_index and returns B2D_OK       */

typedef struct b2d_run_info {
  int64_t m;               /* matrix order                                                 */
  int64_t n_b, b, tail;    /* reference tiling (layout.py:13-62) from num_blocks / max_mem  */
  int64_t blocks_read;     /* reference-equivalent block transfers (cost.py:79-92)          */
  int64_t blocks_written;
  int64_t scratch_slots;   /* cost.py:95-101                                               */
  int64_t tile;            /* engine tile edge (128)                                        */
  int64_t n_tiles;         /* engine tiles per side                                          */
  int64_t h2d_bytes;       /* host->device bytes moved by this call                         */
  int64_t d2h_bytes;       /* device->host bytes moved by this call                         */
  int64_t kernel_launches; /* engine kernels launched by this call                          */
  double device_ms;        /* CUDA-event time of the device work                            */
  double wall_seconds;     /* host wall time of the call                                    */
  int64_t ooc_blocks;      /* out-of-core: engine block grid n_b (0 = in-core run)          */
  int64_t ooc_block;       /* out-of-core: engine block edge b                              */
  int64_t ooc_reads;       /* out-of-core: whole-block host->HBM loads actually performed   */
  int64_t ooc_writes;      /* out-of-core: whole-block HBM->host scratch writes performed   */
  int64_t ooc_scratch;     /* out-of-core: distinct scratch blocks used                      */
} b2d_run_info;

/* Engine options (b2d_ctx_create_ex). */
typedef struct b2d_options {
  int64_t hbm_budget;      /* bytes of HBM the engine may use; 0 = free memory less a margin */
  int64_t num_blocks;      /* reference n_b for the out-of-core tile walk; 0 = from max_mem  */
  int64_t max_mem;         /* reference byte budget (memdet.py:63-80) when num_blocks is 0   */
  int32_t force_out_of_core; /* 1: stream blocks through HBM even if the matrix fits          */
  int32_t host_scratch;    /* 1: keep the out-of-core scratchpad in pinned host memory even when
                              it fits in HBM next to the block slots (default: HBM if it fits) */
  int32_t emulation;       /* trailing Schur updates of the in-core driver: 0 FP64 DMMA tensor
                              cores (default); 1 FP64 emulated on the int8 tcgen05 tensor cores
                              (Ozaki scheme, 8 slices, error ~3 u relative to sum |a b|)      */
  int32_t f32_arith;       /* B2D_MODE_LDL_PIV on float32 inputs: 1 factors in float32 with the
                              reference's own f32 rounding sequence (memdet.py:337-338: d_all in
                              the file dtype; _ldl.pyx `floating`; tolerance 64 eps(f32) max|A|),
                              so perm / D / prefixes are the reference's; in core only.  The
                              context then takes B2D_F32 inputs only.  0: f32 inputs are
                              converted to f64 (round-1 behaviour)                             */
  int32_t ndev;            /* > 1: one context over several devices (devices[0 .. ndev)) in this
                              process: Cholesky / unpivoted LDL over 1-D block-cyclic outer panels,
                              each device ingesting only its own panels from host memory, panels
                              exchanged by peer copies over NVLink; the `device`
                              argument of b2d_ctx_create_ex is then ignored.  0 / 1: one device */
  int32_t devices[8];
  int32_t scratch_mode;    /* out-of-core scratchpad when it lives in host memory (storage.py:147-204):
                              0 auto (= 2); 1 pinned host memory allocated at context creation;
                              2 pageable memory, touched lazily, every transfer staged through a
                              small pinned ring by the library's host threads (no up-front
                              pinning: a one-shot call pays no pinning); 3 a file (mkstemp +
                              ftruncate in scratch_dir, memory-mapped, unlinked at once), staged
                              like 2 -- capacity bounded by disk, not RAM                       */
  const char *scratch_dir; /* mode 3 directory (NULL: $OOCDET_SCRATCH_DIR, else /tmp); a non-NULL
                              scratch_dir with mode 0 selects mode 3 (the reference's behaviour)  */
} b2d_options;

typedef struct b2d_ctx b2d_ctx;

int b2d_version(void);
const char *b2d_last_error(void);
int b2d_device_count(void);

/* One-shot driver: host matrix in, every output on the host.
 *   a        row-major m x m, element type `dtype`, leading dimension lda (elements)
 *   num_blocks / max_mem   reference tiling request (either may be <= 0 = absent; num_blocks
 *                          wins, memdet.py:249-255); reported in `info`, and used as the
 *                          pivoting domain by B2D_MODE_LDL_PIV
 *   d_out     (m) f64: diag(L) for CHOLESKY, D for LDL modes
 *   perm_out  (m) int64 or NULL; prefix_out (m) f64; sign_out (m) int64 or NULL
 *   devices / ndev  the devices to run on (NULL / 0: device 0); ndev > 1 shards the
 *            factorisation over them (modes CHOLESKY and LDL_NOPIV; b2d_options.ndev)
 *   fail_index  first failing global pivot (0-based) on B2D_ERR_NOT_SPD / _INDEFINITE
 */
int b2d_memdet_sym(const void *a, int64_t m, int64_t lda, int dtype, int mode, int64_t num_blocks,
                   int64_t max_mem, const int *devices, int ndev, double *d_out, int64_t *perm_out,
                   double *prefix_out, int64_t *sign_out, b2d_run_info *info,
                   int64_t *fail_index);

/* Context API: allocate once, factor many times (bench / repeated runs). */
int b2d_ctx_create(int device, int64_t m, int mode, b2d_ctx **out);
/* With options: an order whose packed lower triangle exceeds the HBM budget (or
 * force_out_of_core) gets the out-of-core plan — the reference tile walk (memdet.py:124-145,
 * 322-389) over b x b blocks streamed between host memory and HBM, prefetched on copy streams
 * against the DMMA work; b follows num_blocks / max_mem, grown until six blocks fit. */
int b2d_ctx_create_ex(int device, int64_t m, int mode, const b2d_options *opt, b2d_ctx **out);
/* 0 in-core; 1 out of core with the scratchpad in pinned host memory; 2 out of core with the
 * scratchpad in HBM.  Out-of-core contexts accept host inputs only. */
int b2d_ctx_is_out_of_core(b2d_ctx *ctx);
int b2d_ctx_destroy(b2d_ctx *ctx);
/* Enqueue pack + factorisation + prefix of a DEVICE-resident row-major matrix on `stream`
 * (a cudaStream_t, 0 = legacy default).  Results stay on the device until b2d_ctx_fetch. */
int b2d_ctx_factor_device_async(b2d_ctx *ctx, const void *dev_a, int64_t lda, int dtype,
                                void *stream);
/* Same, from HOST memory (pinned or pageable): streams the upper tile triangle in strips.
 * Pinned memory is read by DMA; pageable memory (a memory-mapped file, malloc'd memory) is
 * copied into pinned staging buffers by the library's host threads in stream order.  Either
 * way `host_a` is read after the call returns: keep it valid until b2d_ctx_fetch. */
int b2d_ctx_factor_host_async(b2d_ctx *ctx, const void *host_a, int64_t lda, int dtype,
                              void *stream);
/* Wait for the enqueued work, check for failure, copy the outputs to host (any may be NULL). */
int b2d_ctx_fetch(b2d_ctx *ctx, double *d_out, double *prefix_out, int64_t *fail_index,
                  b2d_run_info *info);
/* The permutation of the last factorisation (block-local pivots offset by the block origin,
 * memdet.py:352-353; identity for unpivoted modes), after b2d_ctx_fetch. */
int b2d_ctx_fetch_perm(b2d_ctx *ctx, int64_t *perm_out);
/* Device pointer of the prefix vector (m doubles), valid until the next factorisation. */
const double *b2d_ctx_device_prefix(b2d_ctx *ctx);
/* Dominant-kernel accounting: the trailing "rest" Schur-update GEMM launches of the last
 * factorisation (~75% of the flops): algorithmic flops, summed CUDA-event duration (ms) and
 * launch count.  b2d_ctx_set_profiling(ctx, mode): 0 off; 1 events around those launches in a
 * normal run (where they share the GPU with the panel streams); 2 the same in a serialised
 * replay (every launch on one stream, so each event pair times the kernel alone). */
int b2d_ctx_set_profiling(b2d_ctx *ctx, int on);
int b2d_ctx_update_stats(b2d_ctx *ctx, double *flops, double *ms, int64_t *launches);

/* Tile-level device API, the building blocks of multi-GPU drivers (paper_2503_04424_b200/
 * distributed.py).  All pointers are DEVICE pointers; work is enqueued on `stream` and not
 * waited for.  Tiles are 128 x 128 doubles in the engine's octet layout.
 *   b2d_tilemap: tile (i, j) lives at base + r*ld + j tiles, r = i, or with rmod > 0
 *                r = (i % rmod) * rstride + i / rmod (row-cyclic blocks gathered from ranks);
 *                with npeer = rmod > 0 at peer[i % rmod] + (i / rmod)*ld + j tiles instead
 *                (each rank's own grid, read in place over NVLink peer memory);
 *                packed_nt > 0 selects the packed lower triangle instead.
 *   b2d_tileset: columns [j0, j1), rows [lo(j), i1), lo = i0, or with lower = 1
 *                lo(j) = max(i0, ceil((j + row_off - off) / stride)) (rows may be local indices
 *                of a row-cyclic distribution, global row = i * stride + off). */
#define B2D_MAX_PEERS 8
typedef struct b2d_tilemap {
  double *base;
  int64_t ld;
  int32_t packed_nt;
  int32_t rmod;
  int64_t rstride;
  int32_t npeer;
  double *peer[B2D_MAX_PEERS];
} b2d_tilemap;
typedef struct b2d_tileset {
  int32_t i0, i1, j0, j1, lower, row_off, stride, off;
} b2d_tileset;
/* Diagonal tile: Cholesky in place (L, zero upper), inv = L^{-1}, ell[g0+r] = 2 log L_rr,
 * diag[g0+r] = L_rr, *fail = min(*fail, first global row g < m with a non-positive pivot). */
int b2d_tile_potrf_inv(double *tile, double *inv, double *ell, double *diag, uint64_t *fail,
                       int64_t g0, int64_t m, void *stream);
/* mode 0: C(i,j) -= sum_{p in [p0,p1)} A(i,p) B(j,p)^T over the tile set (Schur update);
 * mode 1: C(i,k) = C(i,k) binv^T over the tile set's rows (panel solve, k = column). */
int b2d_tile_gemm(int mode, const b2d_tilemap *a, const b2d_tilemap *b, const b2d_tilemap *c,
                  const double *binv, const b2d_tileset *out, int32_t p0, int32_t p1, int32_t k,
                  void *stream);
/* Pack the set's tiles from a row-major DEVICE matrix (f64/f32, leading dimension lda, first
 * stored row row_base; only the row-major upper tile triangle is read, identity beyond m). */
int b2d_pack_tiles(const void *src, int64_t lda, int dtype, int64_t row_base, int64_t m,
                   const b2d_tilemap *out, const b2d_tileset *set, void *stream);
/* Host -> device 2D copy on `stream` (bytes; cudaMemcpy2DAsync): the distributed driver's sharded
 * ingest, each rank copying only its own tile rows' column strips of a host matrix. */
int b2d_h2d_2d(void *dst, int64_t dpitch, const void *src, int64_t spitch, int64_t width, int64_t height,
               void *stream);
/* prefix[q] = sum_{g <= q} ell[g] (double-double, rounded once), q < m. */
int b2d_prefix_scan(const double *ell, int64_t m, double *prefix, void *stream);
/* Peer-shared device buffers for the multi-GPU driver (replaces the panel all-gather: every rank
 * reads the owners' solved panel tiles in place).  b2d_dev_alloc is a plain cudaMalloc on
 * `device`; b2d_ipc_get_handle writes the 64-byte cudaIpcMemHandle of such a buffer;
 * b2d_ipc_open_handle maps a peer's buffer into this process (peer access enabled). */
int b2d_dev_alloc(int device, int64_t bytes, void **out);
int b2d_dev_free(void *p);
int b2d_ipc_get_handle(void *p, void *handle_out);
int b2d_ipc_open_handle(int device, const void *handle, void **out);
int b2d_ipc_close_handle(void *p);

/* Tile seam: the reference's kernel module on the GPU (oocdet.kernels, kernels/__init__.py:24-45;
 * dense.py:57-116), HOST row-major tiles (leading dimension in elements) updated in place, in the
 * tile's dtype (B2D_F64 / B2D_F32) with the golden host's LAPACK / BLAS rounding sequence (LDL,
 * TRSM and GEMM bit-identical there; paper_2503_04424_b200/kernels.py wraps them so the
 * reference's own driver can be patched onto the engine).  Synchronous.
 *   b2d_tile_ldl_host          <- ldl_inplace / _ldl.pyx:21-61: lower triangle -> unit L (strict)
 *                                 and D (diagonal), swaps (LAPACK style), d; tol as dense.py:73;
 *                                 *fail_step = failing step or -1 (the caller raises)
 *   b2d_tile_cholesky_host     <- cholesky_inplace (dense.py:84-91): a = L (zeros above), diag
 *   b2d_tile_solve_lower_host  <- solve_lower_inplace (dense.py:94-99): B <- L^{-1} B
 *   b2d_tile_schur_update_host <- schur_update(s, c, b, "ct_b") (dense.py:109-116): S -= C^T B,
 *                                 S m x n, C k x m, B k x n */
int b2d_tile_ldl_host(void *a, int64_t n, int64_t lda, int dtype, double tol, int64_t *swaps, void *d,
                      int64_t *fail_step, int device);
int b2d_tile_cholesky_host(void *a, int64_t n, int64_t lda, int dtype, void *diag, int64_t *fail_step,
                           int device);
int b2d_tile_solve_lower_host(const void *l, int64_t n, int64_t ldl, void *b, int64_t w, int64_t ldb,
                              int dtype, int unit_diag, int device);
int b2d_tile_schur_update_host(void *s, int64_t m, int64_t n, int64_t lds, const void *c, int64_t ldc,
                               const void *b, int64_t ldb, int64_t k, int dtype, int device);

/* FP64 roofline calibration (off the timed path): sustained DMMA m8n8k4 rate over every SM for
 * about `seconds`, in TFLOP/s (2 flops per FMA). */
int b2d_probe_fp64_peak(int device, double seconds, double *tflops);

/* Gram formation straight into an in-core context's packed tiles (BASELINE C3-C5 style
 * K = G G^T * scale + jitter I, formed chunk by chunk on the device with the engine's own DMMA
 * Schur kernel; off the timed path): init sets the packed tiles to jitter * I (identity beyond
 * m), each accumulate adds scale * G G^T for a DEVICE row-major m x k chunk G (leading dimension
 * ldg), and factor_packed factors the tiles as they are (no input pack). */
int b2d_ctx_packed_init(b2d_ctx *ctx, double jitter, void *stream);
int b2d_ctx_gram_accumulate(b2d_ctx *ctx, const double *dev_g, int64_t ldg, int64_t k, double scale,
                            void *stream);
int b2d_ctx_factor_packed_async(b2d_ctx *ctx, void *stream);

/* Device input generator (off the timed path): C2 RBF Gram, row-major n x n into dev_out. */
int b2d_gen_rbf(const double *dev_x, int64_t n, int d, double ell, double jitter, double *dev_out,
                void *stream);

#ifdef __cplusplus
}
#endif
#endif /* MEMDET_B200_H */
