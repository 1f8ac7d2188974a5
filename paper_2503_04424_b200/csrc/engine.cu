// Host side of the B200 MEMDET engine: HBM planner, right-looking tiled factorisation driver
// with one-panel look-ahead on two prioritised streams, host->HBM strip streamer overlapped
// with the factorisation, the out-of-core block streamer (the reference tile walk over blocks
// that live in host memory), and the C ABI declared in include/memdet_b200.h.
//
// Reference driver mirrored: _memdet_symmetric (memdet.py:322-389).  The reference walks an
// n_b x n_b tile grid out of core with four resident b x b buffers; here the whole lower tile
// triangle is resident in HBM (packed, 128-wide tiles) and the same three steps run per
// 128-wide tile-column k:  factor the diagonal tile (dense.py:84-91), solve the panel
// (dense.py:94-99), Schur-update the trailing tiles (dense.py:109-116); the prefix is the
// running sum of 2 log L_ii (memdet.py:428).
#include <algorithm>
#include <cstdint>
#include <fcntl.h>
#include <sys/mman.h>
#include <unistd.h>
#include <atomic>
#include <condition_variable>
#include <functional>
#include <memory>
#include <mutex>
#include <thread>
#include <chrono>
#include <climits>
#include <cstdlib>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <map>
#include <set>
#include <string>
#include <utility>
#include <vector>

#include "../../include/memdet_b200.h"
#include "kernels.cu"
#include "ldl.cu"
#include "lu.cu"
#include "ozaki.cu"
#include "ldl32.cu"

namespace b2d {

typedef unsigned long long CUdeviceptr_v2_compat;  // CUdeviceptr (driver API) for the entry points

static thread_local std::string g_err;

static int set_err(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

#define CUDA_TRY(expr)                                                                   \
  do {                                                                                   \
    cudaError_t e_ = (expr);                                                             \
    if (e_ != cudaSuccess)                                                               \
      return set_err(B2D_ERR_CUDA, "%s failed: %s (%s:%d)", #expr, cudaGetErrorString(e_), \
                     __FILE__, __LINE__);                                                \
  } while (0)

// outer panel width in tiles: the trailing Schur update runs with K = panel_tiles * 128
// (default 16, narrowed to 8 for the last 64 tile-columns where the potrf chain is the critical
// path; B2D_PANEL_TILES / B2D_TAIL_TILES / B2D_TAIL_W override for tuning)
static int panel_tiles_default() {
  const char* e = getenv("B2D_PANEL_TILES");
  int w = e ? atoi(e) : 16;
  return w < 1 ? 1 : (w > 16 ? 16 : w);
}

constexpr int NSTAGE = 8;   // host-ingest staging strips in flight
constexpr int BAND = 4;     // tile-columns per ingest band
constexpr int NSLOT = 6;      // out-of-core: HBM block slots (A, B, C, T + two for prefetch)
constexpr int NSLOT_LDL = 9;  // pivoted LDL: A, B (scaled), B (unscaled), C, T, next A, two spare, permute temp
constexpr int MAXSLOT = 9;

// The lower tile triangle of an nt x nt tile matrix to factor in place: the whole packed
// matrix (in-core) or one diagonal block slot (out-of-core).  g0 = global index of its row 0.
// Host worker threads for staging pageable inputs (e.g. a memory-mapped MEMDET01 file) into
// pinned buffers: a parallel-for over task indices, run from a CUDA host callback.
class HostPool {
 public:
  explicit HostPool(int n) {
    for (int t = 0; t < n; ++t) th_.emplace_back([this] { work(); });
  }
  ~HostPool() {
    {
      std::lock_guard<std::mutex> g(m_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto& t : th_) t.join();
  }
  // f(0 .. ntask-1) on the workers and the calling thread; returns when all are done
  void run(int ntask, const std::function<void(int)>& f) {
    std::lock_guard<std::mutex> serial(run_m_);  // one parallel-for at a time (contexts share the pool)
    {
      std::lock_guard<std::mutex> g(m_);
      job_ = &f;
      ntask_ = ntask;
      next_ = 0;
      busy_ = (int)th_.size();
      ++gen_;
    }
    cv_.notify_all();
    for (int i; (i = next_.fetch_add(1)) < ntask;) f(i);
    std::unique_lock<std::mutex> g(m_);
    done_.wait(g, [this] { return busy_ == 0; });
    job_ = nullptr;
  }

 private:
  void work() {
    uint64_t seen = 0;
    for (;;) {
      const std::function<void(int)>* f;
      int n;
      {
        std::unique_lock<std::mutex> g(m_);
        cv_.wait(g, [&] { return stop_ || gen_ != seen; });
        if (stop_) return;
        seen = gen_;
        f = job_;
        n = ntask_;
      }
      for (int i; (i = next_.fetch_add(1)) < n;) (*f)(i);
      std::lock_guard<std::mutex> g(m_);
      if (--busy_ == 0) done_.notify_all();
    }
  }
  std::vector<std::thread> th_;
  std::mutex m_, run_m_;
  std::condition_variable cv_, done_;
  const std::function<void(int)>* job_ = nullptr;
  int ntask_ = 0, busy_ = 0;
  std::atomic<int> next_{0};
  uint64_t gen_ = 0;
  bool stop_ = false;
};

constexpr int NHBUF = 4;                       // pinned staging buffers for pageable inputs
constexpr size_t HBUF_BYTES = (size_t)64 << 20; // (at most; sized to the input's strips)
constexpr size_t STAGE_MIN_COPY = (size_t)2 << 20;  // smaller pageable copies go to the driver
static HostPool* host_pool() {  // shared by all contexts, created on first pageable input
  static HostPool* pool = [] {
    const unsigned hw = std::thread::hardware_concurrency();
    return new HostPool((int)std::max(1u, std::min(16u, hw ? hw : 4u) - 1));
  }();
  return pool;
}

struct FillJob {
  HostPool* pool;
  char* dst;
  const char* src;
  size_t spitch, width, rows;
  int fd = -1;      // file-backed scratchpad: pwrite(dst -> fd) / pread(fd -> dst) at foff instead
  int64_t foff = 0;
  int dir = 0;      // 0: memory copy; 1: src -> file (drain); 2: file -> dst (fill)
};
static void CUDART_CB fill_cb(void* p) {
  std::unique_ptr<FillJob> j(static_cast<FillJob*>(p));
  const size_t per = std::max<size_t>(1, ((size_t)1 << 20) / j->width);  // ~1 MB per task
  const int ntask = (int)((j->rows + per - 1) / per);
  j->pool->run(ntask, [&](int t) {
    const size_t r1 = std::min(j->rows, (size_t)(t + 1) * per);
    for (size_t r = (size_t)t * per; r < r1; ++r) memcpy(j->dst + r * j->width, j->src + r * j->spitch, j->width);
  });
}

struct FactorTarget {
  TileMap map;
  int nt;
  int64_t g0;
};

// Out-of-core state: b x b blocks of the reference tile grid stream between host memory (the
// input matrix, and a pinned scratchpad of updated blocks in the engine's tile format) and
// NSLOT HBM slots of nbt x nbt tiles.
struct Ooc {
  int nb = 0;
  int64_t b = 0, tail = 0;
  int nbt = 0;
  int nslot = NSLOT;
  double* slot[MAXSLOT] = {};
  cudaEvent_t ev_loaded[MAXSLOT] = {}, ev_used[MAXSLOT] = {}, ev_stored[MAXSLOT] = {};
  // pivoted LDL: dense diagonal block, pivots and permutations
  double* dense = nullptr;
  int64_t* swaps = nullptr;
  int64_t* perm_local = nullptr;
  int64_t* perm_global = nullptr;
  double* dblk = nullptr;
  unsigned long long* amax = nullptr;
  unsigned* lflags = nullptr;       // panel-server hand-off counters (ldl_panel_server_kernel)
  unsigned* lpipe = nullptr;        // panel / bulk pipeline counters (ldl.cu, B2D_LDL_PIPE)
  double* lrows = nullptr;          // big-block cluster panel: the rows' C / W histories
  size_t lrows_bytes = 0;
  cudaStream_t s_lalt = nullptr;    // pipeline: odd panels and their bulk updates
  cudaStream_t s_lgrp = nullptr;    // group pipeline: early outputs of finished column groups
  cudaEvent_t ev_lgrp = nullptr;
  cudaEvent_t ev_lpanel[2] = {nullptr, nullptr}, ev_lalt = nullptr;
  cudaStream_t s_bulk = nullptr;    // panel-server bulk launches (high priority)
  cudaEvent_t ev_lreset = nullptr, ev_lbulk = nullptr;
  uint8_t* ltag = nullptr;  // blocked pivoted LDL: per-entry tags, panel columns C / W, diagonal, pivot column
  double *lC = nullptr, *lW = nullptr, *ldiag = nullptr, *lcol = nullptr;
  double* inv2 = nullptr;  // LU: inverses of the diagonal tiles of U^T (column-block solves)
  // pivoted LDL look-ahead: the next stage's diagonal block is factored (on s_main) while the
  // current stage's solves and Schur updates run on s_work, so the per-stage outputs of the
  // factor (tile inverses, block permutation, D) are double-buffered by stage parity
  double* inv_odd = nullptr;
  double* inv2_odd = nullptr;
  int64_t* perm_odd = nullptr;
  double* dblk_odd = nullptr;
  cudaStream_t s_work = nullptr;  // block-walk solves / updates: s_main, or s_mid under look-ahead
  cudaEvent_t ev_fac = nullptr, ev_diag = nullptr, ev_work = nullptr;
  cudaStream_t s_h2d = nullptr, s_d2h = nullptr;
  cudaStream_t s_walk = nullptr;  // Cholesky walk under look-ahead (low priority)
  double* stage = nullptr;                         // one 128-row file strip
  std::map<std::pair<int, int>, double*> scratch;  // pinned host blocks (kept across runs)
  std::map<std::pair<int, int>, cudaEvent_t> ev_key;  // last store of each scratch block
  std::vector<double*> pool;                       // scratch slots, bound in first-write order
  bool dev_scratch = false;                        // pool in HBM (fits next to the slots) or pinned host
  // host scratchpad not pinned (scratch_mode 2 / 3): one mapping (anonymous or a temp file),
  // transfers staged through pinned rings by the host pool
  int scratch_mode = 1;
  int scratch_fd = -1;           // mode 3: the (unlinked) scratch file; pool entries are offsets
  char* scratch_map = nullptr;
  size_t scratch_map_bytes = 0;
  static constexpr int NDBUF = 4;
  cudaStream_t s_drain = nullptr;  // host drains of staged HBM -> scratch copies (not behind fills)
  void* dbuf[NDBUF] = {};
  cudaEvent_t ev_ddma[NDBUF] = {}, ev_dfree[NDBUF] = {};
  bool dbuf_used[NDBUF] = {};
  uint64_t dseq = 0;
  std::set<std::pair<int, int>> written;           // cache table of the current run
  int64_t reads = 0, writes = 0;
  int rr = 0;
  int64_t size(int k) const { return k == nb - 1 ? tail : b; }
  int tiles(int k) const { return (int)((size(k) + T - 1) / T); }
  TileMap map(int s) const { return TileMap{slot[s], nbt, 0}; }
  size_t slot_bytes() const { return (size_t)nbt * nbt * TILE_BYTES; }
  // row-ordered in-core LDL (B2D_LDL_ROWS): one set of factor outputs per stage, so a factor
  // never waits for the panel solves of the stage two before it
  bool use_ring = false;
  std::vector<double*> ring_inv, ring_dblk;
  std::vector<int64_t*> ring_perm;
  int64_t* perm_of(int k) const {
    if (use_ring) return ring_perm[k];
    return (k & 1) && perm_odd ? perm_odd : perm_local;
  }
  double* dblk_of(int k) const {
    if (use_ring) return ring_dblk[k];
    return (k & 1) && dblk_odd ? dblk_odd : dblk;
  }
  double* inv_of(int k, double* even) const {
    if (use_ring) return ring_inv[k];
    return (k & 1) && inv_odd ? inv_odd : even;
  }
};

struct MCtx;  // multi-device context (mgpu.cu)

struct Ctx {
  MCtx* mg = nullptr;  // set: a front for several devices (b2d_options.ndev > 1)
  uint64_t hseq_strip = 0;       // multi-device ingest: staging strip rotation
  bool strip_used[NSTAGE] = {};
  int device = 0;
  int64_t m = 0;
  int mode = B2D_MODE_CHOLESKY;
  int nt = 0;
  int W_TILES = 8;
  std::vector<int> bounds;  // outer-panel boundaries k0 of the current factorisation (+ nt)
  double* tiles = nullptr;   // packed lower tile triangle
  double* inv = nullptr;     // nt inverse diagonal tiles
  double* ell = nullptr;     // n_pad: 2 log L_ii
  double* diag = nullptr;    // n_pad: L_ii
  double* prefix = nullptr;  // n_pad
  unsigned long long* fail = nullptr;
  double* strip[NSTAGE] = {};  // host-ingest staging strips (128 x n_pad doubles each)
  // pageable host inputs: each 2D host->HBM copy goes through NHBUF pinned buffers, filled by
  // host worker threads in a callback on s_fill (stream-ordered, so the enqueue never blocks)
  bool src_pageable = false;
  // host-strip ingest cursor: pageable inputs are enqueued band by band as the factorisation is
  // enqueued (a deep queue of staging callbacks would block the host thread before any
  // factorisation work is queued); pinned inputs are enqueued up front
  struct Ingest {
    const void* a = nullptr;
    int64_t lda = 0;
    int dtype = 0, skip = 0, next = 0;
    bool active = false;
  } ing;
  void* hbuf[NHBUF] = {};
  cudaEvent_t ev_hfill[NHBUF] = {}, ev_hcopy[NHBUF] = {};
  bool hbuf_used[NHBUF] = {};
  cudaStream_t s_fill = nullptr;
  size_t hbuf_bytes = 0;
  uint64_t hseq = 0;
  double* gram_neg = nullptr;   // Gram formation: -scale * G chunk as tiles
  double* gram_pos = nullptr;   //                   G chunk as tiles
  int64_t gram_cap = 0;         // tiles allocated per buffer
  cudaStream_t s_main = nullptr, s_side = nullptr, s_copy = nullptr, s_pack = nullptr;
  cudaStream_t s_mid = nullptr;  // panel work off the potrf chain (rows below the panel block)
  cudaEvent_t ev_m2s = nullptr;  // s_main -> s_mid hand-off (potrf + in-block solve of a column)
  cudaEvent_t ev_start = nullptr, ev_stop = nullptr, ev_join = nullptr;
  std::vector<cudaEvent_t> ev_panel, ev_rest, ev_resta, ev_catch, ev_stage, ev_copied, ev_band, ev_ub;
  // band activation (host ingest): band b = tile-columns [b*BAND, (b+1)*BAND) joins the
  // right-looking updates at outer step act[b] (-1: from the start) after one catch-up update
  std::vector<int> act;
  bool trace = false;  // B2D_TRACE: print a per-step event timeline on fetch
  int profiling = 0;
  // Ozaki (int8 tcgen05) trailing updates: panel slices and row exponents
  bool oz = false;
  int8_t* oz_sa[2] = {};  // double-buffered by outer step
  int* oz_expo[2] = {};  // events on the rest updates: 1 in a normal step, 2 in a serialised replay
  std::vector<cudaEvent_t> prof_ev;
  std::vector<double> prof_flops;
  int64_t launches = 0;
  int64_t h2d = 0, d2h = 0;
  bool pending = false;
  std::chrono::steady_clock::time_point t0;
  bool ooc = false;
  Ooc o;
  // block-pivoted LDL in core (reference block size a multiple of the tile): the packed
  // triangle holds the matrix, o.* the block factor state; the stage's solved panel lives in
  // full-height grids of nt x nbt tiles, unscaled and D^{-1}-scaled, double-buffered by stage
  bool ldl_ic = false;
  // in-core pivoted LDL panel grids [stage % npan][0: unscaled, 1: scaled]: three for the column
  // schedule; the row schedule takes up to MAX_PAN when HBM allows (a stage's far rows read its
  // panel grid long after the next stages start)
  static constexpr int MAX_PAN = 16;
  double* pan[MAX_PAN][2] = {};
  int npan = 3;
  bool ldl_rows = false;  // in-core pivoted LDL: row-ordered schedule (B2D_LDL_ROWS)
  // generic LU in core (the same conditions): the matrix as a full nt x nt tile grid; per stage
  // parity the column panel X, the transposed row panel Y^T and a transpose buffer (nt x nbt
  // tiles each, rows = global tile index), and the U^T factor of the diagonal block
  bool lu_ic = false;
  double* grid = nullptr;
  double* lpan[2][3] = {};
  double* ublk[2] = {};
  double* bstage[2] = {};                     // host ingest: one reference block each
  std::vector<cudaEvent_t> ev_bstage, ev_cross;  // staging buffer free; stage k's blocks packed
  // in-core pivoted LDL: one low-priority stream per block column (mod LDL_COL_STREAMS): a block
  // column's updates are ordered by stage on its stream, independently of the other columns'
  std::vector<cudaStream_t> s_cols;
  std::vector<cudaEvent_t> ev_cols;
  // row-ordered schedule (B2D_LDL_ROWS): block rows at distance <= 2, 3, 4, 5 from the stage
  // on streams of falling priority (farther rows on s_cols); per block row the events after its
  // last update and after its panel rows of the current stage
  cudaStream_t s_pr[4] = {nullptr, nullptr, nullptr, nullptr};
  std::vector<cudaEvent_t> ev_row, ev_prow;
  cudaStream_t s_la[2] = {nullptr, nullptr};  // look-ahead solve of the critical block row
  std::vector<cudaEvent_t> ev_la;
  std::vector<std::vector<cudaEvent_t>> ev_grp;  // group pipeline: [stage][group] early factor outputs
  std::vector<cudaEvent_t> ev_rowg;  // group pipeline: block row r's latest solved group
  static constexpr int NCATCH = 8;
  cudaStream_t s_catch[NCATCH] = {};  // host ingest: eager catch-ups of bands not yet active (one stream per step, mod NCATCH)
  std::vector<cudaEvent_t> ev_caught;            // band b's latest eager catch-up
  cudaStream_t s_grpu = nullptr;     // group pipeline: the chain row's scaling + diagonal update
  cudaEvent_t ev_grpu = nullptr;
  // float32 memdet_ldl in f32 arithmetic (ldl32.cu): the matrix row-major in M, the diagonal
  // block column-major in dense, the stage's solved row-k blocks X and their D^{-1}-scaled copy S
  bool ldl32 = false;
  struct F32 {
    float* M = nullptr;
    int64_t ldm = 0;
    float* dense = nullptr;
    int64_t ldd = 0;
    float *X = nullptr, *S = nullptr;
    int64_t ldx = 0;
    float* work = nullptr;
    float* d = nullptr;
    unsigned long long* amax = nullptr;
  } f;
};

static int configure_kernels() {
  static bool done = false;
  if (done) return B2D_OK;
  CUDA_TRY(cudaFuncSetAttribute(gemm_kernel<MODE_UPDATE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)GEMM_SMEM));
  CUDA_TRY(cudaFuncSetAttribute(gemm_kernel<MODE_TRSM>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)GEMM_SMEM));
  CUDA_TRY(cudaFuncSetAttribute(potrf_inv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)POTRF_SMEM));
  CUDA_TRY(cudaFuncSetAttribute(pack_tiles_kernel<double, 32>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)PACK_SMEM));
  CUDA_TRY(cudaFuncSetAttribute(pack_tiles_kernel<float, 32>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)PACK_SMEM));
  CUDA_TRY(cudaFuncSetAttribute(pack_tiles_kernel<double, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)PACK_SMEM));
  CUDA_TRY(cudaFuncSetAttribute(pack_tiles_kernel<float, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)PACK_SMEM));
  CUDA_TRY(cudaFuncSetAttribute(pack_block_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)PACK_SMEM));
  CUDA_TRY(cudaFuncSetAttribute(pack_block_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)PACK_SMEM));
  CUDA_TRY(cudaFuncSetAttribute(pack_set_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)PACK_SMEM));
  CUDA_TRY(cudaFuncSetAttribute(tile_inv_unit_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, T * 129 * 8));
  CUDA_TRY(cudaFuncSetAttribute(ldl_panel_cluster_kernel<false>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  CUDA_TRY(cudaFuncSetAttribute(ldl_panel_cluster_kernel<true>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  CUDA_TRY(cudaFuncSetAttribute(ldl_factor_cluster_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  CUDA_TRY(cudaFuncSetAttribute(ldl_factor_cluster_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)ldl_factor_smem(LC_RMAX)));
  CUDA_TRY(cudaFuncSetAttribute(oz_update_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)OZ_SMEM));
  CUDA_TRY(cudaFuncSetAttribute(lu_panel_cluster_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  CUDA_TRY(cudaFuncSetAttribute(lu_panel_cluster_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)lu_panel_smem(LC_RMAX)));
  CUDA_TRY(cudaFuncSetAttribute(tile_inv_lower_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, T * 129 * 8));
  CUDA_TRY(cudaFuncSetAttribute(transpose_block_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)TRANSPOSE_SMEM));
  CUDA_TRY(cudaFuncSetAttribute(ldl_finish_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)(LDL_FINISH_SMEM_MAX * 8)));
  CUDA_TRY(cudaFuncSetAttribute(ldl_partial_perm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)(LDL_FINISH_SMEM_MAX * 8)));
  CUDA_TRY(cudaFuncSetAttribute(ldl_panel_cluster_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)ldl_cluster_smem(LC_RMAX)));
  CUDA_TRY(cudaFuncSetAttribute(pack_set_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)PACK_SMEM));
  CUDA_TRY(cudaFuncSetAttribute(l32_trsm_diag_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)l32_trsm_smem<float>()));
  CUDA_TRY(cudaFuncSetAttribute(l32_trsm_diag_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)l32_trsm_smem<double>()));
  CUDA_TRY(cudaFuncSetAttribute(ldl_panel_server_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  CUDA_TRY(cudaFuncSetAttribute(ldl_panel_server_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)ldl_cluster_smem(LC_RMAX)));
  {  // the server spins on the bulk kernel's progress: load it now, not lazily at its first launch
    cudaFuncAttributes fa{};
    CUDA_TRY(cudaFuncGetAttributes(&fa, ldl_bulk_kernel));
  }
  done = true;
  return B2D_OK;
}

static void mg_destroy(MCtx* M);
static void destroy(Ctx* c) {
  if (!c) return;
  if (c->mg) {
    mg_destroy(c->mg);
    delete c;
    return;
  }
  cudaSetDevice(c->device);
  if (c->s_fill) {
    cudaStreamSynchronize(c->s_fill);
    cudaStreamDestroy(c->s_fill);
  }
  for (int k = 0; k < NHBUF; ++k) {
    if (c->hbuf[k]) cudaFreeHost(c->hbuf[k]);
    if (c->ev_hfill[k]) cudaEventDestroy(c->ev_hfill[k]);
    if (c->ev_hcopy[k]) cudaEventDestroy(c->ev_hcopy[k]);
  }
  if (c->s_main) cudaStreamSynchronize(c->s_main);
  if (c->s_side) cudaStreamSynchronize(c->s_side);
  if (c->s_mid) cudaStreamSynchronize(c->s_mid);
  cudaFree(c->tiles);
  cudaFree(c->inv);
  cudaFree(c->ell);
  cudaFree(c->diag);
  cudaFree(c->prefix);
  cudaFree(c->fail);
  if (c->s_copy) cudaStreamSynchronize(c->s_copy);
  for (auto* p : c->strip) cudaFree(p);
  for (auto* p : c->bstage) cudaFree(p);
  for (auto* v : {&c->ev_bstage, &c->ev_cross})
    for (auto e : *v) cudaEventDestroy(e);
  cudaFree(c->gram_neg);
  cudaFree(c->gram_pos);
  for (int b = 0; b < 2; ++b) {
    cudaFree(c->oz_sa[b]);
    cudaFree(c->oz_expo[b]);
  }
  if (c->s_pack) cudaStreamSynchronize(c->s_pack);
  for (auto* v : {&c->ev_panel, &c->ev_rest, &c->ev_resta, &c->ev_catch, &c->ev_stage, &c->ev_copied, &c->ev_band, &c->ev_ub,
                  &c->prof_ev})
    for (auto e : *v) cudaEventDestroy(e);
  if (c->ev_start) cudaEventDestroy(c->ev_start);
  if (c->ev_stop) cudaEventDestroy(c->ev_stop);
  if (c->ev_join) cudaEventDestroy(c->ev_join);
  if (c->ev_m2s) cudaEventDestroy(c->ev_m2s);
  if (c->s_main) cudaStreamDestroy(c->s_main);
  if (c->s_mid) cudaStreamDestroy(c->s_mid);
  if (c->s_side) cudaStreamDestroy(c->s_side);
  if (c->s_copy) cudaStreamDestroy(c->s_copy);
  if (c->s_pack) cudaStreamDestroy(c->s_pack);
  for (auto st : c->s_cols) {
    cudaStreamSynchronize(st);
    cudaStreamDestroy(st);
  }
  for (auto st : c->s_pr)
    if (st) {
      cudaStreamSynchronize(st);
      cudaStreamDestroy(st);
    }
  for (auto st : c->s_la)
    if (st) {
      cudaStreamSynchronize(st);
      cudaStreamDestroy(st);
    }
  for (auto e : c->ev_la) cudaEventDestroy(e);
  for (auto& v : c->ev_grp)
    for (auto e : v) cudaEventDestroy(e);
  for (auto e : c->ev_rowg) cudaEventDestroy(e);
  for (auto& q : c->s_catch)
    if (q) {
      cudaStreamSynchronize(q);
      cudaStreamDestroy(q);
    }
  for (auto e : c->ev_caught) cudaEventDestroy(e);
  if (c->s_grpu) {
    cudaStreamSynchronize(c->s_grpu);
    cudaStreamDestroy(c->s_grpu);
  }
  if (c->ev_grpu) cudaEventDestroy(c->ev_grpu);
  for (auto* v : {&c->ev_row, &c->ev_prow})
    for (auto e : *v) cudaEventDestroy(e);
  for (auto e : c->ev_cols) cudaEventDestroy(e);
  Ooc& o = c->o;
  if (o.s_h2d) cudaStreamSynchronize(o.s_h2d);
  if (o.s_d2h) cudaStreamSynchronize(o.s_d2h);
  for (int s = 0; s < MAXSLOT; ++s) {
    cudaFree(o.slot[s]);
    if (o.ev_loaded[s]) cudaEventDestroy(o.ev_loaded[s]);
    if (o.ev_used[s]) cudaEventDestroy(o.ev_used[s]);
    if (o.ev_stored[s]) cudaEventDestroy(o.ev_stored[s]);
  }
  cudaFree(o.dense);
  cudaFree(o.swaps);
  cudaFree(o.perm_local);
  cudaFree(o.perm_global);
  cudaFree(o.dblk);
  cudaFree(o.amax);
  if (o.s_bulk) {
    cudaStreamSynchronize(o.s_bulk);
    cudaStreamDestroy(o.s_bulk);
  }
  cudaFree(o.lflags);
  cudaFree(o.lpipe);
  cudaFree(o.lrows);
  if (o.s_lalt) {
    cudaStreamSynchronize(o.s_lalt);
    cudaStreamDestroy(o.s_lalt);
  }
  if (o.s_lgrp) {
    cudaStreamSynchronize(o.s_lgrp);
    cudaStreamDestroy(o.s_lgrp);
  }
  if (o.ev_lgrp) cudaEventDestroy(o.ev_lgrp);
  for (cudaEvent_t e : {o.ev_lpanel[0], o.ev_lpanel[1], o.ev_lalt})
    if (e) cudaEventDestroy(e);
  if (o.ev_lreset) cudaEventDestroy(o.ev_lreset);
  if (o.ev_lbulk) cudaEventDestroy(o.ev_lbulk);
  cudaFree(o.ltag);
  cudaFree(o.lC);
  cudaFree(o.lW);
  cudaFree(o.ldiag);
  cudaFree(o.lcol);
  cudaFree(o.inv2);
  for (auto& pp : c->pan)
    for (double* q : pp) cudaFree(q);
  for (auto& pp : c->lpan)
    for (double* q : pp) cudaFree(q);
  for (double* q : c->ublk) cudaFree(q);
  cudaFree(c->grid);
  for (double* q : o.ring_inv) cudaFree(q);
  for (double* q : o.ring_dblk) cudaFree(q);
  for (int64_t* q : o.ring_perm) cudaFree(q);
  cudaFree(o.inv_odd);
  cudaFree(o.inv2_odd);
  cudaFree(o.perm_odd);
  cudaFree(o.dblk_odd);
  for (cudaEvent_t e : {o.ev_fac, o.ev_diag, o.ev_work})
    if (e) cudaEventDestroy(e);
  for (void* q : {(void*)c->f.M, (void*)c->f.dense, (void*)c->f.X, (void*)c->f.S, (void*)c->f.work, (void*)c->f.d,
                  (void*)c->f.amax})
    cudaFree(q);
  cudaFree(o.stage);
  if (o.s_drain) {
    cudaStreamSynchronize(o.s_drain);
    cudaStreamDestroy(o.s_drain);
  }
  if (o.scratch_fd >= 0) {
    close(o.scratch_fd);
  } else if (o.scratch_map) {
    munmap(o.scratch_map, o.scratch_map_bytes);
  } else {
    for (double* h : o.pool) {
      if (o.dev_scratch) cudaFree(h);
      else cudaFreeHost(h);
    }
  }
  for (int k = 0; k < Ooc::NDBUF; ++k) {
    if (o.dbuf[k]) cudaFreeHost(o.dbuf[k]);
    if (o.ev_ddma[k]) cudaEventDestroy(o.ev_ddma[k]);
    if (o.ev_dfree[k]) cudaEventDestroy(o.ev_dfree[k]);
  }
  for (auto& kv : o.ev_key) cudaEventDestroy(kv.second);
  if (o.s_h2d) cudaStreamDestroy(o.s_h2d);
  if (o.s_walk) cudaStreamDestroy(o.s_walk);
  if (o.s_d2h) cudaStreamDestroy(o.s_d2h);
  delete c;
}

// ---------------------------------------------------------------- reference tiling bookkeeping

static int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

static void ref_layout(int64_t m, int64_t nb, int64_t* n_b, int64_t* b, int64_t* tail) {
  // layout.py:35-51
  nb = std::min(nb, m);
  for (;;) {
    const int64_t bb = 1 + (m - 1) / nb;
    const int64_t need = ceil_div(m, bb);
    if (need == nb) {
      *n_b = nb;
      *b = bb;
      *tail = m - (nb - 1) * bb;
      return;
    }
    nb = need;
  }
}

static int64_t isqrt_u(unsigned __int128 x) {
  unsigned __int128 r = 0, bit = (unsigned __int128)1 << 126;
  while (bit > x) bit >>= 2;
  while (bit) {
    if (x >= r + bit) { x -= r + bit; r = (r >> 1) + bit; }
    else r >>= 1;
    bit >>= 2;
  }
  return (int64_t)r;
}

static int64_t ref_select_blocking(int64_t m, int64_t c, int64_t beta) {
  // memdet.py:63-80 (exact integer arithmetic)
  const unsigned __int128 msq = (unsigned __int128)m * m * beta;
  if (msq <= (unsigned __int128)c) return 1;
  if (3 * msq <= 4 * (unsigned __int128)c) return 2;
  const unsigned __int128 target = 4 * msq;
  int64_t q = isqrt_u(target / c);
  while ((unsigned __int128)q * q * c < target) ++q;
  return q;
}

static void fill_ref_info(b2d_run_info* info, int64_t m, int64_t num_blocks, int64_t max_mem, int esz,
                          bool generic = false) {
  int64_t nb = num_blocks > 0 ? num_blocks : (max_mem > 0 ? ref_select_blocking(m, max_mem, esz) : 1);
  int64_t n_b, b, tail;
  ref_layout(m, nb, &n_b, &b, &tail);
  info->n_b = n_b;
  info->b = b;
  info->tail = tail;
  const int64_t n = n_b;
  info->blocks_read = (2 * n * n * n - 3 * n * n + 7 * n) / 6;                       // cost.py:79-83
  info->blocks_written = n <= 2 ? 0 : (n * n * n + 3 * n * n - 22 * n + 24) / 6;     // cost.py:86-92
  info->scratch_slots = n <= 2 ? 0 : (n * n + n - 8) / 2;                            // cost.py:95-101
  if (generic) {  // the generic walk (memdet.py:97-121): cost.py:79-101, case "generic"
    info->blocks_read = (2 * n * n * n - 3 * n * n + 4 * n) / 3;
    info->blocks_written = n <= 2 ? 0 : (n * n * n - 4 * n - 3) / 3;
    info->scratch_slots = n <= 2 ? 0 : n * n - n - 1;
  }
}


static int create_streams_events(Ctx* c) {
  int lo = 0, hi = 0;
  cudaDeviceGetStreamPriorityRange(&lo, &hi);
  // panel chain (critical path) and ingest get the highest priority; trailing updates the lowest
  if (cudaStreamCreateWithPriority(&c->s_main, cudaStreamNonBlocking, hi) != cudaSuccess ||
      cudaStreamCreateWithPriority(&c->s_side, cudaStreamNonBlocking, lo) != cudaSuccess ||
      cudaStreamCreateWithPriority(&c->s_mid, cudaStreamNonBlocking, (lo + hi) / 2) != cudaSuccess ||
      cudaStreamCreateWithPriority(&c->s_copy, cudaStreamNonBlocking, hi) != cudaSuccess ||
      cudaStreamCreateWithPriority(&c->s_pack, cudaStreamNonBlocking, hi) != cudaSuccess)
    return set_err(B2D_ERR_CUDA, "stream creation failed");
  cudaEventCreate(&c->ev_start);
  cudaEventCreate(&c->ev_stop);
  cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&c->ev_m2s, cudaEventDisableTiming);
  const int nsteps = c->nt;  // enough for any panel-width schedule
  c->ev_panel.resize(nsteps);
  c->ev_rest.resize(nsteps);
  c->ev_resta.resize(nsteps);
  c->ev_ub.resize(nsteps);
  for (auto& e : c->ev_ub) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
  c->ev_catch.resize(nsteps);
  c->trace = getenv("B2D_TRACE") != nullptr;
  const unsigned evf = c->trace ? cudaEventDefault : cudaEventDisableTiming;
  for (int s = 0; s < nsteps; ++s) {
    cudaEventCreateWithFlags(&c->ev_panel[s], evf);
    cudaEventCreateWithFlags(&c->ev_rest[s], evf);
    cudaEventCreateWithFlags(&c->ev_resta[s], evf);
    cudaEventCreateWithFlags(&c->ev_catch[s], evf);
  }
  const int nbands = (c->nt + BAND - 1) / BAND;
  c->ev_band.resize(nbands);
  for (auto& e : c->ev_band) cudaEventCreateWithFlags(&e, evf);
  c->ev_stage.resize(NSTAGE);
  for (auto& e : c->ev_stage) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
  c->ev_copied.resize(NSTAGE);
  for (auto& e : c->ev_copied) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
  c->act.assign(nbands, -1);
  return B2D_OK;
}

// HBM planner.  In-core: the packed lower tile triangle, the inverse diagonal tiles, three
// n_pad vectors and NSTAGE ingest strips.  Out-of-core (budget exceeded or forced): NSLOT
// block slots of nbt^2 tiles; the block grid starts at the reference n_b (num_blocks, else
// select_blocking(max_mem), memdet.py:63-80, 249-255) and grows until the slots fit.
static int mg_create(const int* devices, int ndev, int64_t m, int mode, const b2d_options* opt, MCtx** out);
static int create(int device, int64_t m, int mode, const b2d_options* opt, Ctx** out) {
  if (m < 1) return set_err(B2D_ERR_USAGE, "matrix dimension must be >= 1, got %lld", (long long)m);
  if (opt && opt->ndev > 1) {
    if (opt->ndev > 8) return set_err(B2D_ERR_USAGE, "at most 8 devices (got %d)", opt->ndev);
    MCtx* M = nullptr;
    if (int rc = mg_create(opt->devices, opt->ndev, m, mode, opt, &M)) return rc;
    Ctx* c = new Ctx();
    c->mg = M;
    c->device = opt->devices[0];
    c->m = m;
    c->mode = mode;
    *out = c;
    return B2D_OK;
  }
  if (mode != B2D_MODE_CHOLESKY && mode != B2D_MODE_LDL_NOPIV && mode != B2D_MODE_LDL_PIV && mode != B2D_MODE_LU)
    return set_err(B2D_ERR_USAGE, "unknown mode %d", mode);
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    return set_err(B2D_ERR_CUDA, "no CUDA device visible: the B200 engine has no CPU fallback");
  if (device < 0 || device >= ndev) return set_err(B2D_ERR_USAGE, "bad device %d", device);
  CUDA_TRY(cudaSetDevice(device));
  int rc = configure_kernels();
  if (rc) return rc;
  size_t free_b = 0, total_b = 0;
  cudaMemGetInfo(&free_b, &total_b);
  const size_t margin = (size_t)1 << 30;
  size_t budget = free_b > margin ? free_b - margin : 0;
  if (opt && opt->hbm_budget > 0) budget = std::min(budget, (size_t)opt->hbm_budget);

  Ctx* c = new Ctx();
  c->device = device;
  c->m = m;
  c->mode = mode;
  c->W_TILES = panel_tiles_default();
  const int nt_full = (int)((m + T - 1) / T);
  const int64_t npad_full = (int64_t)nt_full * T;
  const size_t incore_need = (size_t)n_packed_tiles(nt_full) * TILE_BYTES + (size_t)nt_full * TILE_BYTES +
                             3 * (size_t)npad_full * 8 + (size_t)NSTAGE * T * npad_full * 8;
  // block-pivoted LDL pivots inside the reference's b x b diagonal blocks, and the generic LU
  // runs the reference's generic walk: always the block walk
  const bool pivoted = mode == B2D_MODE_LDL_PIV || mode == B2D_MODE_LU;
  bool force = (opt && opt->force_out_of_core) || pivoted;
  // block-pivoted LDL in core: the reference's blocks (num_blocks, else select_blocking(max_mem))
  // must start on tile boundaries; needs the packed triangle plus four nt x nbt panel grids and
  // the dense block state
  int64_t ic_nb = 0, ic_b = 0, ic_tail = 0;
  if (mode == B2D_MODE_LU && !(opt && opt->force_out_of_core)) {
    int64_t nb0 = 1;
    if (opt && opt->num_blocks > 0) nb0 = opt->num_blocks;
    else if (opt && opt->max_mem > 0) nb0 = ref_select_blocking(m, opt->max_mem, 8);
    ref_layout(m, std::max<int64_t>(1, nb0), &ic_nb, &ic_b, &ic_tail);
    const int64_t bt = (ic_b + T - 1) / T, ldb = bt * T;
    const size_t ic_need = (size_t)nt_full * nt_full * TILE_BYTES + 6 * (size_t)nt_full * bt * TILE_BYTES +
                           (size_t)(nt_full + 5 * bt) * TILE_BYTES + (size_t)ldb * ldb * 8 +
                           3 * (size_t)npad_full * 8 + (size_t)NSTAGE * T * npad_full * 8 + (size_t)(m + 8 * ldb) * 8;
    // the cluster LU panel holds the block's rows in distributed shared memory
    if ((ic_b % T == 0 || ic_nb == 1) && ic_b <= (int64_t)LC * LC_RMAX && ic_need <= budget) force = false;
  }
  if (mode == B2D_MODE_LDL_PIV && !(opt && opt->force_out_of_core)) {
    int64_t nb0 = 1;
    if (opt && opt->num_blocks > 0) nb0 = opt->num_blocks;
    else if (opt && opt->max_mem > 0) nb0 = ref_select_blocking(m, opt->max_mem, 8);
    ref_layout(m, std::max<int64_t>(1, nb0), &ic_nb, &ic_b, &ic_tail);
    const int64_t bt = (ic_b + T - 1) / T, ldb = bt * T;
    const size_t ic_need = (size_t)n_packed_tiles(nt_full) * TILE_BYTES + 6 * (size_t)nt_full * bt * TILE_BYTES +
                           (size_t)(nt_full + bt) * TILE_BYTES + (size_t)ldb * ldb * 9 + 3 * (size_t)npad_full * 8 +
                           (size_t)NSTAGE * T * npad_full * 8 + (size_t)(m + 8 * ldb) * 8;
    if ((ic_b % T == 0 || ic_nb == 1) && ic_need <= budget) force = false;
  }
  const int nslot = pivoted ? NSLOT_LDL : NSLOT;
  int64_t vec_len = npad_full;
#define ALLOC(ptr, bytes)                                        \
  do {                                                           \
    cudaError_t e_ = cudaMalloc((void**)&(ptr), (bytes));        \
    if (e_ != cudaSuccess) {                                     \
      destroy(c);                                                \
      return set_err(B2D_ERR_NOMEM, "cudaMalloc(%zu) failed: %s", (size_t)(bytes), cudaGetErrorString(e_)); \
    }                                                            \
  } while (0)
  // Schur-update arithmetic: FP64 DMMA (default) or the Ozaki int8 emulation (opt->emulation = 1,
  // or B2D_SCHUR=ozaki / dmma to override)
  bool oz = opt && opt->emulation == 1;
  if (const char* e = getenv("B2D_SCHUR")) oz = strcmp(e, "ozaki") == 0 ? true : (strcmp(e, "dmma") == 0 ? false : oz);
  const size_t oz_need = oz ? 2 * ((size_t)OZ_S * npad_full * (size_t)(16 * T) + (size_t)npad_full * 4) : 0;
  const char* fa_env = getenv("B2D_F32_ARITH");
  const bool f32a = mode == B2D_MODE_LDL_PIV && opt && opt->f32_arith && (fa_env ? atoi(fa_env) != 0 : true);
  if (f32a) {
    // float32 memdet_ldl in the reference's f32 arithmetic (ldl32.cu), in core: the matrix
    // row-major, the stage's row-k blocks X and S, the dense diagonal block
    Ooc& o = c->o;
    c->ldl32 = true;
    c->nt = nt_full;
    int64_t nb0 = 1;
    if (opt->num_blocks > 0) nb0 = opt->num_blocks;
    else if (opt->max_mem > 0) nb0 = ref_select_blocking(m, opt->max_mem, 4);
    int64_t n_b, b, tail;
    ref_layout(m, std::max<int64_t>(1, nb0), &n_b, &b, &tail);
    o.nb = (int)n_b;
    o.b = b;
    o.tail = tail;
    auto r32 = [](int64_t x) { return (x + 31) / 32 * 32; };
    Ctx::F32& f = c->f;
    f.ldm = r32(m);
    f.ldd = r32(b);
    f.ldx = r32(std::max<int64_t>(1, m - b));
    const size_t need = (size_t)m * f.ldm * 4 + (n_b > 1 ? 2 * (size_t)b * f.ldx * 4 : 0) + (size_t)b * f.ldd * 4 +
                        (size_t)(m + 2 * b) * 16 + 3 * (size_t)npad_full * 8;
    if (need > budget) {
      destroy(c);
      return set_err(B2D_ERR_NOMEM,
                     "float32 memdet_ldl runs in core in f32 arithmetic: needs %.2f GB of HBM, the budget is %.2f GB",
                     need / 1e9, budget / 1e9);
    }
    ALLOC(f.M, (size_t)m * f.ldm * 4);
    ALLOC(f.dense, (size_t)b * f.ldd * 4);
    if (n_b > 1) {
      ALLOC(f.X, (size_t)b * f.ldx * 4);
      ALLOC(f.S, (size_t)b * f.ldx * 4);
    }
    ALLOC(f.work, (size_t)b * 4);
    ALLOC(f.d, (size_t)m * 4);
    ALLOC(f.amax, 8);
    ALLOC(o.swaps, (size_t)b * 8);
    ALLOC(o.perm_local, (size_t)b * 8);
    ALLOC(o.perm_global, (size_t)m * 8);
  } else if (!force && mode == B2D_MODE_LU) {
    Ooc& o = c->o;
    c->lu_ic = true;
    c->nt = nt_full;
    o.nb = (int)ic_nb;
    o.b = ic_b;
    o.tail = ic_tail;
    o.nbt = (int)((ic_b + T - 1) / T);
    const int64_t ld = (int64_t)o.nbt * T;
    ALLOC(c->grid, (size_t)c->nt * c->nt * TILE_BYTES);
    ALLOC(c->inv, (size_t)c->nt * TILE_BYTES);
    for (auto& pp : c->lpan)
      for (double*& q : pp) ALLOC(q, (size_t)c->nt * o.nbt * TILE_BYTES);
    for (double*& q : c->ublk) ALLOC(q, (size_t)o.nbt * o.nbt * TILE_BYTES);
    ALLOC(o.dense, (size_t)ld * ld * 8);
    ALLOC(o.swaps, (size_t)ld * 8);
    ALLOC(o.perm_local, (size_t)ld * 8);
    ALLOC(o.perm_global, (size_t)(m + ld) * 8);
    ALLOC(o.dblk, (size_t)ld * 8);
    ALLOC(o.inv2, (size_t)o.nbt * TILE_BYTES);
    ALLOC(o.inv_odd, (size_t)o.nbt * TILE_BYTES);
    ALLOC(o.inv2_odd, (size_t)o.nbt * TILE_BYTES);
    ALLOC(o.perm_odd, (size_t)ld * 8);
    ALLOC(o.dblk_odd, (size_t)ld * 8);
    cudaEventCreateWithFlags(&o.ev_fac, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&o.ev_diag, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&o.ev_work, cudaEventDisableTiming);
  } else if (!force && mode == B2D_MODE_LDL_PIV) {
    Ooc& o = c->o;
    c->ldl_ic = true;
    c->nt = nt_full;
    o.nb = (int)ic_nb;
    o.b = ic_b;
    o.tail = ic_tail;
    o.nbt = (int)((ic_b + T - 1) / T);
    const int64_t ld = (int64_t)o.nbt * T;
    ALLOC(c->tiles, (size_t)n_packed_tiles(c->nt) * TILE_BYTES);
    ALLOC(c->inv, (size_t)c->nt * TILE_BYTES);
    {
      // panel grids: three, plus up to half of the HBM left over (one pair per further stage)
      const size_t pair = 2 * (size_t)c->nt * o.nbt * TILE_BYTES;
      const int64_t bt = o.nbt;
      const size_t ic_need = (size_t)n_packed_tiles(nt_full) * TILE_BYTES + 6 * (size_t)nt_full * bt * TILE_BYTES +
                             (size_t)(nt_full + bt) * TILE_BYTES + (size_t)ld * ld * 9 + 3 * (size_t)npad_full * 8 +
                             (size_t)NSTAGE * T * npad_full * 8 + (size_t)(m + 8 * ld) * 8;
      const size_t spare = budget > ic_need ? (budget - ic_need) / 2 : 0;
      // B2D_LDL_ROWS: 1 = row-ordered schedule, 0 = column schedule; unset: rows for <= 8 blocks, and
      // for <= 16 blocks of at most 6144 rows (the blocks whose factors hand out column groups)
      // (with the factors' group pipeline, B2D_LDL_GROUPS, and one-launch trailing updates the row
      // schedule wins at C2, 431 -> 418 ms, and at C3, 2833 -> 2798 ms; before the group pipeline
      // the column schedule kept more of the DMMA throughput at 16 blocks: 2876 vs 2950 ms)
      const char* re = getenv("B2D_LDL_ROWS");
      c->ldl_rows = re ? atoi(re) != 0 : o.nb <= 8 || (o.nb <= 16 && o.b <= (int64_t)LC * LC_RMAX);
      c->npan = c->ldl_rows ? (int)std::min<int64_t>({(int64_t)Ctx::MAX_PAN, std::max<int64_t>(3, o.nb),
                                                      3 + (int64_t)(spare / pair)})
                            : 3;
      for (int q = 0; q < c->npan; ++q)
        for (double*& pq : c->pan[q]) ALLOC(pq, (size_t)c->nt * o.nbt * TILE_BYTES);
    }
    ALLOC(o.dense, (size_t)ld * ld * 8);
    ALLOC(o.swaps, (size_t)ld * 8);
    ALLOC(o.perm_local, (size_t)ld * 8);
    ALLOC(o.perm_global, (size_t)(m + ld) * 8);
    ALLOC(o.dblk, (size_t)ld * 8);
    ALLOC(o.amax, 8);
    ALLOC(o.ltag, (size_t)ld * ld);
    ALLOC(o.lC, (size_t)LDL_NB * ld * 8);
    ALLOC(o.lW, (size_t)LDL_NB * ld * 8);
    ALLOC(o.ldiag, (size_t)ld * 8);
    ALLOC(o.lcol, (size_t)ld * 8);
    ALLOC(o.inv_odd, (size_t)o.nbt * TILE_BYTES);
    ALLOC(o.perm_odd, (size_t)ld * 8);
    ALLOC(o.dblk_odd, (size_t)ld * 8);
    cudaEventCreateWithFlags(&o.ev_fac, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&o.ev_diag, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&o.ev_work, cudaEventDisableTiming);
  } else if (!force && incore_need + oz_need <= budget) {
    c->nt = nt_full;
    ALLOC(c->tiles, (size_t)n_packed_tiles(c->nt) * TILE_BYTES);
    ALLOC(c->inv, (size_t)c->nt * TILE_BYTES);
    if (oz) {  // slices of an outer panel (rows <= n_pad, K <= 16 tiles), two in flight
      c->oz = true;
      for (int b = 0; b < 2; ++b) {
        ALLOC(c->oz_sa[b], (size_t)OZ_S * npad_full * (16 * T));
        ALLOC(c->oz_expo[b], (size_t)npad_full * 4);
      }
    }
  } else {
    Ooc& o = c->o;
    c->ooc = true;
    int64_t nb = 2;
    if (opt && opt->num_blocks > 0) nb = opt->num_blocks;
    else if (opt && opt->max_mem > 0) nb = ref_select_blocking(m, opt->max_mem, 8);
    nb = std::max<int64_t>(1, nb);
    for (;;) {
      int64_t n_b, b, tail;
      ref_layout(m, nb, &n_b, &b, &tail);
      const int nbt = (int)((b + T - 1) / T);
      const size_t need = (size_t)(nslot + (pivoted ? 1 : 0)) * nbt * nbt * TILE_BYTES +
                          (size_t)nbt * TILE_BYTES +
                          (size_t)T * nbt * T * 8 + 3 * (size_t)(m + (int64_t)(nbt + 1) * T) * 8;
      // LU pivots inside the reference's diagonal blocks (block-local partial pivoting,
      // dense.py:38-54), so a finer grid would change the result (a zero leading block of a
      // finer grid is singular where the reference's block is not) -- never grow it either
      if (mode == B2D_MODE_LU && b > (int64_t)LC * LC_RMAX) {
        destroy(c);
        return set_err(B2D_ERR_UNSUPPORTED,
                       "generic LU factors the reference's %lld-row diagonal blocks with a cluster panel kernel "
                       "that holds at most %d rows: use num_blocks >= %lld (or a smaller max_mem)",
                       (long long)b, LC * LC_RMAX, (long long)ceil_div(m, (int64_t)LC * LC_RMAX));
      }
      if (mode == B2D_MODE_LU && need > budget) {
        destroy(c);
        return set_err(B2D_ERR_NOMEM,
                       "generic LU keeps the reference's %lld blocks of %lld rows (its pivots depend on them): "
                       "the out-of-core walk needs %.2f GB of HBM, the budget is %.2f GB",
                       (long long)n_b, (long long)b, need / 1e9, budget / 1e9);
      }
      // pivoted LDL: the pivots are searched inside the reference's blocks (block-local 1x1
      // pivoting, _ldl.pyx), so a finer grid would change perm and the prefixes -- never grow
      if (mode == B2D_MODE_LDL_PIV && need > budget) {
        destroy(c);
        return set_err(B2D_ERR_NOMEM,
                       "block-pivoted LDL keeps the reference's %lld blocks of %lld rows (its pivots depend on "
                       "them): the out-of-core walk needs %.2f GB of HBM, the budget is %.2f GB (raise hbm_budget, "
                       "or use more num_blocks / a smaller max_mem, or pivoting='none')",
                       (long long)n_b, (long long)b, need / 1e9, budget / 1e9);
      }
      if (need <= budget || n_b >= m) {
        if (need > budget) {
          destroy(c);
          return set_err(B2D_ERR_NOMEM, "no out-of-core plan fits %.2f GB of HBM", budget / 1e9);
        }
        o.nb = (int)n_b;
        o.b = b;
        o.tail = tail;
        o.nbt = nbt;
        break;
      }
      nb = n_b + 1;
    }
    c->nt = o.nbt;  // the in-core machinery factors one diagonal block at a time
    vec_len = m + (int64_t)(o.nbt + 1) * T;
    o.nslot = nslot;
    for (int s = 0; s < nslot; ++s) {
      ALLOC(o.slot[s], o.slot_bytes());
      cudaEventCreateWithFlags(&o.ev_loaded[s], cudaEventDisableTiming);
      cudaEventCreateWithFlags(&o.ev_used[s], cudaEventDisableTiming);
      cudaEventCreateWithFlags(&o.ev_stored[s], cudaEventDisableTiming);
    }
    ALLOC(o.stage, (size_t)T * o.nbt * T * 8);
    ALLOC(c->inv, (size_t)o.nbt * TILE_BYTES);
    if (!pivoted) ALLOC(o.inv_odd, (size_t)o.nbt * TILE_BYTES);  // stage parity (walk look-ahead)
    if (pivoted) {
      const int64_t ld = (int64_t)o.nbt * T;
      ALLOC(o.dense, (size_t)ld * ld * 8);
      ALLOC(o.swaps, (size_t)ld * 8);
      ALLOC(o.perm_local, (size_t)ld * 8);
      ALLOC(o.perm_global, (size_t)(m + ld) * 8);
      ALLOC(o.dblk, (size_t)ld * 8);
      ALLOC(o.amax, 8);
      ALLOC(o.ltag, (size_t)ld * ld);
      ALLOC(o.lC, (size_t)LDL_NB * ld * 8);
      ALLOC(o.lW, (size_t)LDL_NB * ld * 8);
      ALLOC(o.ldiag, (size_t)ld * 8);
      ALLOC(o.lcol, (size_t)ld * 8);
      if (mode == B2D_MODE_LU) ALLOC(o.inv2, (size_t)o.nbt * TILE_BYTES);
      if (mode == B2D_MODE_LDL_PIV) {
        ALLOC(o.inv_odd, (size_t)o.nbt * TILE_BYTES);
        ALLOC(o.perm_odd, (size_t)ld * 8);
        ALLOC(o.dblk_odd, (size_t)ld * 8);
      }
    }
    // scratchpad: exactly the reference capacity (cost.py:95-101), allocated up front; in HBM
    // when it fits beside the slots (scratch traffic then moves at HBM instead of PCIe speed),
    // otherwise in pinned host memory
    const int64_t nsc = o.nb <= 2 ? 0
                        : mode == B2D_MODE_LU ? (int64_t)o.nb * o.nb - o.nb - 1        // cost.py, generic
                                              : ((int64_t)o.nb * o.nb + o.nb - 8) / 2;
    size_t used = 0, fb = 0, tb = 0;
    cudaMemGetInfo(&fb, &tb);
    used = free_b > fb ? free_b - fb : 0;
    const char* hse = getenv("B2D_HOST_SCRATCH");  // 1: keep the scratchpad in host memory (tests)
    const bool host_scr = (opt && opt->host_scratch) || (hse && atoi(hse) != 0);
    o.dev_scratch = !host_scr && used + (size_t)nsc * o.slot_bytes() <= budget;
    // host scratchpad: pinned up front (mode 1), or pageable / a temp file staged through pinned
    // rings (modes 2 / 3, the default: nothing is pinned up front, so a one-shot call does not
    // pay for pinning the whole scratchpad; a file bounds the capacity by disk, as the
    // reference's mkstemp scratchpad, storage.py:147-204).  B2D_SCRATCH=pinned|staged|file.
    int smode = opt ? opt->scratch_mode : 0;
    if (smode == 0) smode = (opt && opt->scratch_dir && opt->scratch_dir[0]) ? 3 : 2;
    if (const char* e = getenv("B2D_SCRATCH"))
      smode = strcmp(e, "pinned") == 0 ? 1 : strcmp(e, "file") == 0 ? 3 : strcmp(e, "staged") == 0 ? 2 : smode;
    o.scratch_mode = smode;
    if (!o.dev_scratch && smode >= 2 && nsc > 0) {
      const size_t bytes = (size_t)nsc * o.slot_bytes();
      int fd = -1;
      if (smode == 3) {
        std::string dir = opt && opt->scratch_dir && opt->scratch_dir[0] ? opt->scratch_dir : "";
        if (dir.empty()) {
          const char* env = getenv("OOCDET_SCRATCH_DIR");  // storage.py:200-204
          dir = env && env[0] ? env : "/tmp";
        }
        std::string tmpl = dir + "/oocdet-b200-scratch-XXXXXX";
        std::vector<char> path(tmpl.begin(), tmpl.end());
        path.push_back('\0');
        fd = mkstemp(path.data());
        if (fd < 0) {
          destroy(c);
          return set_err(B2D_ERR_STORAGE, "scratchpad file in %s: %s", dir.c_str(), strerror(errno));
        }
        unlink(path.data());  // the mapping keeps it; nothing is left behind on any exit
        if (ftruncate(fd, (off_t)bytes) != 0) {
          close(fd);
          destroy(c);
          return set_err(B2D_ERR_STORAGE, "scratchpad file of %.2f GB in %s: %s", bytes / 1e9, dir.c_str(),
                         strerror(errno));
        }
      }
      if (fd >= 0) {
        // read / written with pread / pwrite by the host pool (no page-fault storm on a fresh file
        // mapping); pool entries are byte offsets into the file
        o.scratch_fd = fd;
        for (int64_t q = 0; q < nsc; ++q) o.pool.push_back((double*)(uintptr_t)((size_t)q * o.slot_bytes()));
      } else {
        void* mp = mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS | MAP_NORESERVE, -1, 0);
        if (mp == MAP_FAILED) {
          destroy(c);
          return set_err(B2D_ERR_NOMEM, "scratchpad mapping of %.2f GB failed: %s", bytes / 1e9, strerror(errno));
        }
        madvise(mp, bytes, MADV_HUGEPAGE);
        o.scratch_map = (char*)mp;
        o.scratch_map_bytes = bytes;
        for (int64_t q = 0; q < nsc; ++q) o.pool.push_back((double*)(o.scratch_map + (size_t)q * o.slot_bytes()));
      }
    } else {
      for (int64_t q = 0; q < nsc; ++q) {
        double* h = nullptr;
        const cudaError_t e = o.dev_scratch ? cudaMalloc((void**)&h, o.slot_bytes())
                                            : cudaHostAlloc((void**)&h, o.slot_bytes(), cudaHostAllocDefault);
        if (e != cudaSuccess) {
          destroy(c);
          return set_err(B2D_ERR_NOMEM, "scratchpad of %lld x %.2f GB failed", (long long)nsc, o.slot_bytes() / 1e9);
        }
        o.pool.push_back(h);
      }
    }
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    cudaStreamCreateWithPriority(&o.s_h2d, cudaStreamNonBlocking, hi);
    cudaStreamCreateWithPriority(&o.s_d2h, cudaStreamNonBlocking, hi);
    cudaStreamCreateWithPriority(&o.s_walk, cudaStreamNonBlocking, lo);
    cudaEventCreateWithFlags(&o.ev_fac, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&o.ev_diag, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&o.ev_work, cudaEventDisableTiming);
  }
  ALLOC(c->ell, vec_len * 8);
  ALLOC(c->diag, vec_len * 8);
  ALLOC(c->prefix, vec_len * 8);
  ALLOC(c->fail, 8);
#undef ALLOC
  rc = create_streams_events(c);
  if (rc) {
    destroy(c);
    return rc;
  }
  *out = c;
  return B2D_OK;
}

static void launch_gemm(Ctx* c, cudaStream_t s, int mode, const GemmTask& t, bool prof, double flops) {
  const int64_t ntile = t.out.count();
  if (ntile <= 0) return;
  if (mode == MODE_UPDATE && t.p1 <= t.p0) return;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (c->profiling && prof) {
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0, s);
  }
  if (mode == MODE_UPDATE)
    gemm_kernel<MODE_UPDATE><<<(unsigned)ntile, GEMM_THREADS, GEMM_SMEM, s>>>(t);
  else
    gemm_kernel<MODE_TRSM><<<(unsigned)ntile, GEMM_THREADS, GEMM_SMEM, s>>>(t);
  c->launches++;
  if (e0) {
    cudaEventRecord(e1, s);
    c->prof_ev.push_back(e0);
    c->prof_ev.push_back(e1);
    c->prof_flops.push_back(flops);
  }
}

// The trailing ("rest") update of a stage that runs beside the next diagonal factor, issued as
// sequential launches over K chunks of `rest_kchunk()` tile-columns: each CTA then holds its SM
// for K = 128 * chunk instead of the whole block width, so the factor's cluster and bulk
// launches find free SMs sooner.  Exact: the accumulators start from C and the chunks continue
// the same k order, and a stored FP64 accumulator reloads unchanged.
// K chunk (tile-columns) of the in-core LDL / LU trailing updates: B2D_REST_KCHUNK, else 32 for
// the pivoted LDL (one launch per 4096-row block; 16 was best before the factors' group pipeline
// gave the chain its slack: C2 422.6 -> 418.5 ms, C3 2821 -> 2798 ms) and 8 for the LU
static int rest_kchunk(int dflt = 8) {
  const char* e = getenv("B2D_REST_KCHUNK");
  return e ? atoi(e) : dflt;
}
static void launch_update_kchunked(Ctx* c, cudaStream_t s, GemmTask u, int dflt = 8) {
  const int kcv = rest_kchunk(dflt);
  const int p0 = u.p0, p1 = u.p1, kc = kcv > 0 ? kcv : p1 - p0;
  for (int q = p0; q < p1; q += kc) {
    u.p0 = q;
    u.p1 = std::min(p1, q + kc);
    launch_gemm(c, s, MODE_UPDATE, u, true, (double)u.out.count() * 2.0 * T * T * (double)(u.p1 - u.p0) * T);
  }
}

// Schur update of the output tiles `out` of the target with K tile-columns [p0, p1)
static void launch_update_set(Ctx* c, cudaStream_t s, const FactorTarget& ft, const TileSet& out, int p0, int p1,
                              bool prof) {
  GemmTask t{};
  t.a = t.b = t.c = ft.map;
  t.out = out;
  t.p0 = p0;
  t.p1 = p1;
  // algorithmic flops: off-diagonal tiles 2*T*T*K, diagonal (SYRK, lower half) T*(T+1)*K
  const double K = (double)(p1 - p0) * T;
  const int64_t ntile = t.out.count();
  int64_t ndiag = 0;
  for (int j = out.j0; j < out.j1; ++j) ndiag += j >= out.lo(j) && j < out.i1;
  launch_gemm(c, s, MODE_UPDATE, t, prof, (double)(ntile - ndiag) * 2.0 * T * T * K + (double)ndiag * T * (T + 1.0) * K);
}

// Slices of panel rows [P.r0, P.r0 + P.rt) over K tiles [P.p0, P.p0 + P.kt) (ozaki.cu).
static void launch_oz_slices(Ctx* c, cudaStream_t s, const OzPanel& P) {
  oz_expo_kernel<<<P.rt, 256, 0, s>>>(P);
  oz_slice_kernel<<<dim3(P.rt, P.kt), 256, 0, s>>>(P);
  c->launches += 2;
}

// The Schur update of `out` emulated on the int8 tensor cores from the slices P (ozaki.cu):
// one CTA per output tile.
static void launch_update_oz(Ctx* c, cudaStream_t s, const FactorTarget& ft, const OzPanel& P, const TileSet& out,
                             bool prof) {
  const int64_t ntile = out.count();
  if (ntile <= 0) return;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (prof && c->profiling) {
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0, s);
  }
  oz_update_kernel<<<(unsigned)ntile, OZ_THREADS, OZ_SMEM, s>>>(P, ft.map, out);
  c->launches++;
  if (e0) {
    const double K = (double)P.kt * T;
    int64_t ndiag = 0;
    for (int j = out.j0; j < out.j1; ++j) ndiag += j >= out.lo(j) && j < out.i1;
    cudaEventRecord(e1, s);
    c->prof_ev.push_back(e0);
    c->prof_ev.push_back(e1);
    c->prof_flops.push_back((double)(ntile - ndiag) * 2.0 * T * T * K + (double)ndiag * T * (T + 1.0) * K);
  }
}

// Schur update of the target's lower tiles in tile-columns [j0, j1) with K tile-columns [p0, p1)
static void launch_update(Ctx* c, cudaStream_t s, const FactorTarget& ft, int j0, int j1, int p0, int p1,
                          bool prof) {
  launch_update_set(c, s, ft, TileSet{0, ft.nt, j0, std::min(j1, ft.nt), 1, 0}, p0, p1, prof);
}

// Outer-panel schedule: W tile-columns per panel, narrowed to head_w for the first head tiles
// (host ingest: the chain runs ahead of the arriving strips) and to tail_w once no more than
// tail tiles remain (the chain-bound end).  B2D_HEAD_TILES/W, B2D_TAIL_TILES/W override.
static int env_int(const char* name, int dflt) {
  const char* e = getenv(name);
  return e ? atoi(e) : dflt;
}

static void make_bounds(Ctx* c, int nt, bool host) {
  const int W = c->W_TILES;
  const int head = env_int(host ? "B2D_HEAD_TILES" : "B2D_DEV_HEAD_TILES", 0), head_w = std::max(1, env_int("B2D_HEAD_W", 4));
  const int tail = env_int("B2D_TAIL_TILES", 64), tail_w = std::max(1, env_int("B2D_TAIL_W", 8));
  c->bounds.clear();
  int k = 0;
  while (k < nt) {
    c->bounds.push_back(k);
    int w = W;
    if (k < head) w = head_w;
    if (nt - k <= tail) w = tail_w;
    k = std::min(nt, k + w);
  }
  c->bounds.push_back(nt);
}

// Latest step at which a band starting at tile-column col may join: -1 if the first panel
// reads it, else the first step whose next-cols update reaches it.
static int band_deadline(const Ctx* c, int col) {
  if (col < c->bounds[1]) return -1;
  const int nsteps = (int)c->bounds.size() - 1;
  for (int s = 0; s < nsteps; ++s) {
    const int ne = s + 2 <= nsteps ? c->bounds[s + 2] : c->bounds[nsteps];
    if (ne > col) return s;
  }
  return nsteps - 1;
}

static void launch_potrf(Ctx* c, cudaStream_t s, const FactorTarget& ft, int p) {
  potrf_inv_kernel<<<1, POTRF_THREADS, POTRF_SMEM, s>>>(ft.map.tile(p, p), c->inv + (int64_t)p * TILE_ELEMS, c->ell,
                                                         c->diag, c->fail, ft.g0 + (int64_t)p * T, c->m);
  c->launches++;
}

// L(i, p) = A(i, p) L_pp^-T for rows i in [i0, i1)
static void launch_trsm(Ctx* c, cudaStream_t s, const FactorTarget& ft, int p, int i0, int i1) {
  if (i1 <= i0) return;
  GemmTask t{};
  t.c = ft.map;
  t.binv = c->inv + (int64_t)p * TILE_ELEMS;
  t.out = TileSet{i0, i1, p, p + 1, 0, 0};
  t.k = p;
  launch_gemm(c, s, MODE_TRSM, t, false, 0.0);
}

// The factorisation proper of ft (streams s_main / s_side, joined back into s_main).
// In the in-core host-ingest path, tile-columns of bands with act[b] == -1 are waited for before
// first use; a band with act[b] = s >= 0 first receives one catch-up update with every panel of
// steps < s (K = 128*k0, on s_side, after its band event), then joins the regular next-cols /
// rest updates from step s on.  act[b] <= the step whose next-cols update first touches band b,
// so every column is current before it is factored.
static void enqueue_factor(Ctx* c, const FactorTarget& ft, bool wait_bands,
                           const std::function<void(int)>* step_hook = nullptr) {
  // profiling mode 2: every launch on s_main (serialised replay: per-launch event times are the
  // kernel's own, nothing runs beside it)
  struct Restore {
    Ctx* c;
    cudaStream_t side, mid;
    ~Restore() { c->s_side = side; c->s_mid = mid; }
  } restore{c, c->s_side, c->s_mid};
  if (c->profiling == 2) c->s_side = c->s_mid = c->s_main;
  const int nt = ft.nt;
  if (c->bounds.empty() || c->bounds.back() != nt) make_bounds(c, nt, false);
  const int nsteps = (int)c->bounds.size() - 1;
  const int nbands = (nt + BAND - 1) / BAND;
  cudaEventRecord(c->ev_join, c->s_main);
  cudaStreamWaitEvent(c->s_side, c->ev_join, 0);
  cudaStreamWaitEvent(c->s_mid, c->ev_join, 0);
  if (wait_bands) {
    for (int b = 0; b < nbands; ++b)
      if (c->act[b] < 0) cudaStreamWaitEvent(c->s_side, c->ev_band[b], 0);
  }
  // B2D_EAGER_CATCH (default 1; pinned host input, whose strips are all enqueued up front): a
  // band that joins at step s takes the panels of steps t < s one by one, each as soon as that
  // panel is solved and the band has arrived (low-priority streams, one per step; a band's
  // pieces ordered by its event), instead of one K = 128 k0 catch-up when it joins -- the pieces
  // fill the SMs while the first panels' chains run with few bands active.  Same k order with
  // exact FP64 continuation across launches: bit-identical.
  // Pageable inputs enqueue their strips band by band (the step hook), so a band takes its first
  // piece once it is enqueued (its event is then this run's): K = every panel solved so far.
  const bool eager = wait_bands && c->ing.active && c->profiling != 2 &&
                     env_int("B2D_EAGER_CATCH", 1) != 0 && (c->ing.next >= nt || env_int("B2D_EAGER_PAGEABLE", 1) != 0);
  std::vector<int> caught((size_t)nbands, 0);  // K tile-columns [0, caught[b]) already applied to band b
  // one stream per step that issues pieces (a step's queue ends with the last band to arrive, so a
  // later step's pieces must not sit behind it): B2D_EAGER_STREAMS, default the plan's depth
  int max_act = 0;
  if (wait_bands)
    for (int b = 0; b < nbands; ++b) max_act = std::max(max_act, c->act[b]);
  const int ncatch = std::max(1, std::min((int)Ctx::NCATCH, env_int("B2D_EAGER_STREAMS", std::max(2, max_act))));
  if (eager) {
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    for (int q = 0; q < ncatch; ++q) {
      if (!c->s_catch[q]) cudaStreamCreateWithPriority(&c->s_catch[q], cudaStreamNonBlocking, lo);
      cudaStreamWaitEvent(c->s_catch[q], c->ev_join, 0);
    }
    while ((int)c->ev_caught.size() < nbands) {
      cudaEvent_t e;
      cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
      c->ev_caught.push_back(e);
    }
  }
  int main_waited = 0;  // initial bands s_main has waited for (waited lazily, per panel)
  // B2D_LEFT_BELOW (default 1): the rows below each panel are updated left-looking per column
  const char* lbe = getenv("B2D_LEFT_BELOW");
  const bool left_below = lbe ? atoi(lbe) != 0 : true;
  for (int st = 0; st < nsteps; ++st) {
    if (step_hook) (*step_hook)(st);  // host ingest of the bands this step may wait for
    const int k0 = c->bounds[st];
    const int ke = c->bounds[st + 1];
    // panel(k0): its columns were last touched by next-cols(st-1) and rest(st-2)
    if (st >= 2) cudaStreamWaitEvent(c->s_main, c->ev_rest[st - 2], 0);
    // The panel's diagonal block [k0, ke)^2 is factored on s_main (potrf, in-block solve and
    // in-block update per column: the critical chain touches at most W(W+1)/2 tiles); the rows
    // below it ([ke, nt): solve and update) follow each column on s_mid.  Every tile still
    // sees the same launches in the same order, so results do not depend on the split.
    for (int p = k0; p < ke; ++p) {
      if (wait_bands) {
        // an initial band must be in HBM before the first panel column that reads it (the
        // panel's updates touch columns up to ke-1)
        const int need = std::min(nbands, (ke - 1) / BAND + 1);
        while (main_waited < need && c->act[main_waited] < 0)
          cudaStreamWaitEvent(c->s_main, c->ev_band[main_waited++], 0);
      }
      launch_potrf(c, c->s_main, ft, p);
      launch_trsm(c, c->s_main, ft, p, p + 1, ke);
      cudaEventRecord(c->ev_m2s, c->s_main);
      cudaStreamWaitEvent(c->s_mid, c->ev_m2s, 0);
      if (left_below) {
        // rows below, left-looking inside the panel: column p takes the panel's columns
        // [k0, p) in ONE launch (K = 128 (p - k0)) right before its solve -- each tile is read
        // and written once per panel instead of once per column, with the same k order (the
        // FP64 accumulators start from C), so the result is bit-identical
        if (ke < nt && p > k0) launch_update_set(c, c->s_mid, ft, TileSet{ke, nt, p, p + 1, 0, 0}, k0, p, false);
        launch_trsm(c, c->s_mid, ft, p, ke, nt);
        if (p + 1 < ke) launch_update_set(c, c->s_main, ft, TileSet{p + 1, ke, p + 1, ke, 1, 0}, p, p + 1, false);
        continue;
      }
      launch_trsm(c, c->s_mid, ft, p, ke, nt);
      if (p + 1 < ke) {
        launch_update_set(c, c->s_main, ft, TileSet{p + 1, ke, p + 1, ke, 1, 0}, p, p + 1, false);
        if (ke < nt) launch_update_set(c, c->s_mid, ft, TileSet{ke, nt, p + 1, ke, 0, 0}, p, p + 1, false);
      }
    }
    // the whole panel is solved once s_mid gets here (s_mid waited for every in-block solve).
    // Ozaki mode: slice its rows [ke, nt) once for the next-cols remainder and the rest update
    // (buffer st % 2: the step that used it last, st - 2, finished before this panel started)
    const bool ozs = c->oz && ft.map.packed_nt > 0 && (ke - k0) <= 16 && ke < nt;
    OzPanel P{};
    if (ozs) {
      P = OzPanel{ft.map, ke, nt - ke, k0, ke - k0, c->oz_sa[st & 1], c->oz_expo[st & 1]};
      launch_oz_slices(c, c->s_mid, P);
    }
    cudaEventRecord(c->ev_panel[st], c->s_mid);
    if (ke >= nt) break;
    if (eager) {
      cudaStream_t cs = c->s_catch[st % ncatch];
      bool first = true;
      for (int b = 0; b < nbands; ++b) {
        if (c->act[b] <= st) continue;  // active, or joining at this step
        if (std::min(nt, (b + 1) * BAND) > c->ing.next) continue;  // strips not enqueued yet
        if (first) cudaStreamWaitEvent(cs, c->ev_panel[st], 0);
        first = false;
        cudaStreamWaitEvent(cs, c->ev_band[b], 0);
        if (caught[(size_t)b] > 0) cudaStreamWaitEvent(cs, c->ev_caught[b], 0);  // its previous piece (other stream)
        launch_update(c, cs, ft, b * BAND, std::min(nt, (b + 1) * BAND), caught[(size_t)b], ke, false);
        caught[(size_t)b] = ke;
        cudaEventRecord(c->ev_caught[b], cs);
      }
    }
    const int ne = c->bounds[st + 2 <= nsteps ? st + 2 : nsteps];
    // catch-up of the bands that join at this step (panels of steps < st, already factored).
    // Bands the next-cols update reads (deadline st) go before ev_catch; the others after it,
    // so the next panel's chain does not wait for bands it does not touch yet.
    int end_active = nt;
    if (wait_bands) {
      end_active = 0;
      for (int b = 0; b < nbands; ++b)
        if (c->act[b] <= st) end_active = std::min(nt, (b + 1) * BAND);
      for (int pass = 0; pass < 2; ++pass) {
        if (pass == 1) cudaEventRecord(c->ev_catch[st], c->s_side);
        for (int b = 0; b < nbands; ++b) {
          if (c->act[b] != st || (band_deadline(c, b * BAND) <= st) != (pass == 0)) continue;
          // panels already applied piece by piece as they were solved: wait for the last piece
          if (caught[(size_t)b] > 0) cudaStreamWaitEvent(c->s_side, c->ev_caught[b], 0);
          if (caught[(size_t)b] >= k0 && st > 0) continue;
          cudaStreamWaitEvent(c->s_side, c->ev_band[b], 0);
          launch_update(c, c->s_side, ft, b * BAND, std::min(nt, (b + 1) * BAND), caught[(size_t)b], k0, false);
        }
      }
    } else {
      cudaEventRecord(c->ev_catch[st], c->s_side);
    }
    // next-cols(k0): the next panel's columns [ke, ne); its diagonal block on s_main (the next
    // potrf chain starts as soon as it is done), the rows below on s_mid.  Both follow rest(st-1)
    // and the catch-ups (ev_catch) and the whole panel solve (ev_panel).
    cudaStreamWaitEvent(c->s_main, c->ev_catch[st], 0);
    cudaStreamWaitEvent(c->s_main, c->ev_panel[st], 0);
    launch_update_set(c, c->s_main, ft, TileSet{ke, ne, ke, ne, 1, 0}, k0, ke, false);
    cudaStreamWaitEvent(c->s_mid, c->ev_catch[st], 0);
    if (ne < nt) {
      if (ozs) launch_update_oz(c, c->s_mid, ft, P, TileSet{ne, nt, ke, ne, 0, 0}, false);
      else launch_update_set(c, c->s_mid, ft, TileSet{ne, nt, ke, ne, 0, 0}, k0, ke, false);
    }
    // rest(k0): active columns right of the next panel, overlapping the next panel
    cudaStreamWaitEvent(c->s_side, c->ev_panel[st], 0);
    if (ozs)
      launch_update_oz(c, c->s_side, ft, P, TileSet{0, nt, ne, std::max(ne, end_active), 1, 0}, true);
    else
      launch_update(c, c->s_side, ft, ne, std::max(ne, end_active), k0, ke, true);
    cudaEventRecord(c->ev_rest[st], c->s_side);
  }
  if (step_hook) (*step_hook)(INT_MAX);
  // join the side streams
  if (eager)
    for (int q = 0; q < ncatch; ++q) {
      cudaEventRecord(c->ev_join, c->s_catch[q]);
      cudaStreamWaitEvent(c->s_main, c->ev_join, 0);
    }
  cudaEventRecord(c->ev_join, c->s_side);
  cudaStreamWaitEvent(c->s_main, c->ev_join, 0);
  cudaEventRecord(c->ev_join, c->s_mid);
  cudaStreamWaitEvent(c->s_main, c->ev_join, 0);
}

static void enqueue_prefix(Ctx* c) {
  prefix_kernel<<<1, 1024, 0, c->s_main>>>(c->ell, c->m, c->prefix);
  c->launches++;
}

static void begin(Ctx* c, cudaStream_t user) {
  for (auto e : c->prof_ev) cudaEventDestroy(e);
  c->prof_ev.clear();
  c->prof_flops.clear();
  c->launches = 0;
  c->h2d = c->d2h = 0;
  c->t0 = std::chrono::steady_clock::now();
  cudaEventRecord(c->ev_start, user);
  cudaStreamWaitEvent(c->s_main, c->ev_start, 0);
  cudaStreamWaitEvent(c->s_side, c->ev_start, 0);
  cudaStreamWaitEvent(c->s_mid, c->ev_start, 0);
  cudaStreamWaitEvent(c->s_copy, c->ev_start, 0);
  cudaStreamWaitEvent(c->s_pack, c->ev_start, 0);
  cudaMemsetAsync(c->fail, 0xff, 8, c->s_main);
}

static void end(Ctx* c, cudaStream_t user) {
  cudaEventRecord(c->ev_join, c->s_main);
  cudaStreamWaitEvent(user, c->ev_join, 0);
  cudaEventRecord(c->ev_stop, user);
  c->pending = true;
}

static int run_ldl_incore(Ctx* c, const void* a, int64_t lda, int dtype, bool host, cudaStream_t user);
static int run_ldl32(Ctx* c, const void* a, int64_t lda, int dtype, bool host, cudaStream_t user);
static int h2d_2d(Ctx* c, void* dst, size_t dpitch, const void* src, size_t spitch, size_t width, size_t height,
                  cudaStream_t s);
static int run_lu_incore(Ctx* c, const void* a, int64_t lda, int dtype, bool host, cudaStream_t user);

static int mg_factor(MCtx* M, const void* a, int64_t lda, int dtype, bool host, cudaStream_t user);
static int mg_fetch(MCtx* M, double* d_out, double* prefix_out, int64_t* fail_index, b2d_run_info* info);
static int factor_device(Ctx* c, const void* a, int64_t lda, int dtype, cudaStream_t user) {
  if (c->mg) return mg_factor(c->mg, a, lda, dtype, false, user);
  if (dtype != B2D_F64 && dtype != B2D_F32) return set_err(B2D_ERR_USAGE, "dtype code %d", dtype);
  if (lda < c->m) return set_err(B2D_ERR_USAGE, "lda %lld < m", (long long)lda);
  if (c->ldl32) return run_ldl32(c, a, lda, dtype, false, user);
  if (c->ooc)
    return set_err(B2D_ERR_UNSUPPORTED, "out-of-core contexts take host inputs (the matrix exceeds the HBM budget)");
  if (c->ldl_ic) return run_ldl_incore(c, a, lda, dtype, false, user);
  if (c->lu_ic) return run_lu_incore(c, a, lda, dtype, false, user);
  CUDA_TRY(cudaSetDevice(c->device));
  begin(c, user);
  const unsigned ntiles = (unsigned)n_packed_tiles(c->nt);
  if (dtype == B2D_F64)
    pack_tiles_kernel<double, 32><<<ntiles, PACK_THREADS, PACK_SMEM, c->s_main>>>(
        (const double*)a, lda, 0, c->m, c->tiles, c->nt, 0);
  else
    pack_tiles_kernel<float, 32><<<ntiles, PACK_THREADS, PACK_SMEM, c->s_main>>>(
        (const float*)a, lda, 0, c->m, c->tiles, c->nt, 0);
  c->launches++;
  // Lazy trailing updates: band b (BAND tile-columns) joins the right-looking updates only
  // `lazy` outer steps before its first use, after one catch-up GEMM with every panel factored
  // so far (K = 128 * k0).  Same flops; far bands get few large-K updates instead of one K = 128*W
  // update per step (B2D_LAZY_STEPS; default -1 = eager, which measured faster at C2 and C3).
  const char* ls = getenv("B2D_LAZY_STEPS");
  const int lazy = ls ? atoi(ls) : -1;
  make_bounds(c, c->nt, false);
  const int nb = (c->nt + BAND - 1) / BAND;
  for (int b = 0; b < nb; ++b) {
    const int deadline = band_deadline(c, b * BAND);
    c->act[b] = lazy < 0 ? -1 : std::max(-1, deadline - lazy);
  }
  cudaEventRecord(c->ev_join, c->s_main);
  for (auto& e : c->ev_band) cudaEventRecord(e, c->s_main);  // everything is resident already
  enqueue_factor(c, FactorTarget{TileMap{c->tiles, 0, c->nt}, c->nt, 0}, true);
  enqueue_prefix(c);
  end(c, user);
  CUDA_TRY(cudaGetLastError());
  return B2D_OK;
}

// Band activation schedule for host ingest (static, data-independent => deterministic).
// A small event simulation of the pipeline: bands arrive at a modelled PCIe rate (~52 GB/s);
// each outer step costs its panel chain plus its update flops at ~34 TFLOP/s; a band joins at
// the first step that starts after its arrival, and never later than the step whose next-cols
// update first touches it (then the device waits for it).  Deferred panels are applied by one
// catch-up update when the band joins, so early steps are not held up by late strips.
static void plan_bands(Ctx* c, size_t esz) {
  const int nt = c->nt;
  make_bounds(c, nt, true);
  const int nbands = (nt + BAND - 1) / BAND;
  const int nsteps = (int)c->bounds.size() - 1;
  const double m = (double)c->m, rate = 34e12, chain_rate = 20e12;
  // ingest rate of the model: PCIe for pinned inputs; for pageable ones the host staging copies
  // (measured ~15 GB/s from a memory-mapped file with 16 threads) are the bound
  const char* rate_env = getenv(c->src_pageable ? "B2D_STAGE_GBS" : "B2D_PCIE_GBS");
  const double pcie = rate_env ? atof(rate_env) * 1e9 : (c->src_pageable ? 14e9 : 48e9);
  const double col_lat = getenv("B2D_COL_LAT_US") ? atof(getenv("B2D_COL_LAT_US")) * 1e-6 : 900e-6;
  const double tile_flops = 2.0 * T * T * T;
  std::vector<double> arrival(nbands);
  double bytes = 0.0;
  for (int b = 0; b < nbands; ++b) {
    for (int J = b * BAND; J < std::min(nt, (b + 1) * BAND); ++J) {
      const double r0 = (double)J * T;
      bytes += std::max(0.0, std::min((double)T, m - r0)) * std::max(0.0, m - r0) * (double)esz;
    }
    arrival[b] = bytes / pcie;
  }
  auto tiles = [nt](int j0, int j1) {
    double n = 0;
    for (int j = j0; j < std::min(j1, nt); ++j) n += nt - j;
    return n;
  };
  auto deadline = [&](int b) { return band_deadline(c, b * BAND); };
  double t = 0.0;
  int next = 0;
  while (next < nbands && deadline(next) < 0) {  // needed by step 0's panel / next-cols
    c->act[next] = -1;
    t = std::max(t, arrival[next]);
    ++next;
  }
  for (int st = 0; st < nsteps && next < nbands; ++st) {
    const int k0 = c->bounds[st], ke = c->bounds[st + 1];
    const int ne = c->bounds[st + 2 <= nsteps ? st + 2 : nsteps];
    const int W = ke - k0;
    // critical chain of the step (s_main): panel columns + intra-panel and next-cols updates
    const double chain = W * col_lat +
                         (0.5 * W * (W - 1) * (nt - k0) * tile_flops + tiles(ke, ne) * tile_flops * W) /
                             chain_rate;
    double side = 0.0;  // s_side: catch-ups of joining bands + rest over active bands
    while (next < nbands && (arrival[next] <= t || deadline(next) <= st)) {
      c->act[next] = st;
      t = std::max(t, arrival[next]);
      side += tiles(next * BAND, (next + 1) * BAND) * tile_flops * k0;
      ++next;
    }
    const int end_active = std::min(nt, next * BAND);
    side += tiles(ne, std::max(ne, end_active)) * tile_flops * W;
    t += std::max(chain, side / rate);
  }
}

// Host ingest: row strip J (rows [128J, 128J+128), columns [128J, m)) = tile-column J of the
// packed lower triangle.  Strips stream through NSTAGE staging buffers on s_copy (H2D copy,
// then a pack kernel that co-resides with the Schur-update CTAs); each band of BAND strips
// records an event, and the factorisation waits per band, so PCIe overlaps the DMMA work.
static int run_ooc(Ctx* c, const void* a, int64_t lda, int dtype, cudaStream_t user);

// The strips of a host matrix into the packed triangle (s_copy / s_pack); ev_band[b] is recorded
// on s_pack once tile-columns [b * BAND, (b + 1) * BAND) are packed.  skip > 0: the leading
// skip x skip tiles are already in (their strips bring only the columns from skip * 128 on).
// Host -> HBM 2D copy of a host input on stream s.  Pinned sources go straight to the copy
// engine; pageable ones (a memory-mapped file, a plain ndarray) are staged: rows are copied into
// one of NHBUF pinned buffers by the host pool in a callback on s_fill, and the DMA from that
// buffer waits for the fill (the next fill of a buffer waits for its DMA), so host copies and
// PCIe transfers overlap each other and the factorisation.
static int h2d_2d(Ctx* c, void* dst, size_t dpitch, const void* src, size_t spitch, size_t width, size_t height,
                  cudaStream_t s) {
  if (width == 0 || height == 0) return B2D_OK;
  if (!c->src_pageable || width * height < STAGE_MIN_COPY) {
    CUDA_TRY(cudaMemcpy2DAsync(dst, dpitch, src, spitch, width, height, cudaMemcpyHostToDevice, s));
    return B2D_OK;
  }
  if (!c->s_fill) {
    // buffers of two 128-row strips of the matrix (at most HBUF_BYTES): a small input does not
    // pin 256 MB
    c->hbuf_bytes = std::min(HBUF_BYTES, std::max(STAGE_MIN_COPY, (size_t)2 * T * (size_t)c->m * 8));
    CUDA_TRY(cudaStreamCreateWithFlags(&c->s_fill, cudaStreamNonBlocking));
    for (int k = 0; k < NHBUF; ++k) {
      CUDA_TRY(cudaHostAlloc(&c->hbuf[k], c->hbuf_bytes, cudaHostAllocDefault));
      cudaEventCreateWithFlags(&c->ev_hfill[k], cudaEventDisableTiming);
      cudaEventCreateWithFlags(&c->ev_hcopy[k], cudaEventDisableTiming);
    }
  }
  const size_t per = std::max<size_t>(1, c->hbuf_bytes / width);
  for (size_t r0 = 0; r0 < height; r0 += per) {
    const size_t rows = std::min(per, height - r0);
    const int k = (int)(c->hseq++ % NHBUF);
    if (c->hbuf_used[k]) cudaStreamWaitEvent(c->s_fill, c->ev_hcopy[k], 0);
    auto* job = new FillJob{host_pool(), (char*)c->hbuf[k], (const char*)src + r0 * spitch, spitch, width, rows};
    if (cudaLaunchHostFunc(c->s_fill, fill_cb, job) != cudaSuccess) {
      delete job;
      return set_err(B2D_ERR_CUDA, "cudaLaunchHostFunc failed");
    }
    cudaEventRecord(c->ev_hfill[k], c->s_fill);
    cudaStreamWaitEvent(s, c->ev_hfill[k], 0);
    CUDA_TRY(cudaMemcpy2DAsync((char*)dst + r0 * dpitch, dpitch, c->hbuf[k], width, width, rows,
                               cudaMemcpyHostToDevice, s));
    cudaEventRecord(c->ev_hcopy[k], s);
    c->hbuf_used[k] = true;
  }
  return B2D_OK;
}

static int ingest_host_strips(Ctx* c, const void* a, int64_t lda, int dtype, int skip, int J0, int J1) {
  const int64_t npad = (int64_t)c->nt * T;
  const size_t esz = dtype == B2D_F64 ? 8 : 4;
  for (int J = J0; J < J1; ++J) {
    const int b = J % NSTAGE;
    const int64_t r0 = (int64_t)J * T;
    const int64_t rows = std::min<int64_t>(T, c->m - r0);
    const int i_lo = J < skip ? skip : 0;
    const int64_t c0 = std::max<int64_t>(r0, (int64_t)i_lo * T);
    const int64_t cols = c->m - c0;  // columns [c0, m): the upper triangle of this strip
    // staging buffer b is free once the pack of strip J - NSTAGE has run
    if (J >= NSTAGE) cudaStreamWaitEvent(c->s_copy, c->ev_stage[b], 0);
    if (cols > 0) {
      const char* src = (const char*)a + (size_t)(r0 * lda + c0) * esz;
      // staged with leading dimension npad, offset so that column c0 lands at index c0
      char* dst = (char*)c->strip[b] + (size_t)c0 * esz;
      if (int rc = h2d_2d(c, dst, (size_t)npad * esz, src, (size_t)lda * esz, (size_t)cols * esz, (size_t)rows,
                          c->s_copy))
        return rc;
      c->h2d += rows * cols * (int64_t)esz;
    }
    cudaEventRecord(c->ev_copied[b], c->s_copy);
    cudaStreamWaitEvent(c->s_pack, c->ev_copied[b], 0);
    const unsigned ntile = (unsigned)(c->nt - std::max(J, i_lo));
    if (ntile > 0) {
      if (dtype == B2D_F64)
        pack_tiles_kernel<double, 8><<<ntile, PACK_THREADS, PACK_SMEM, c->s_pack>>>(
            (const double*)c->strip[b], npad, r0, c->m, c->tiles, c->nt, J, i_lo);
      else
        pack_tiles_kernel<float, 8><<<ntile, PACK_THREADS, PACK_SMEM, c->s_pack>>>(
            (const float*)c->strip[b], npad, r0, c->m, c->tiles, c->nt, J, i_lo);
    }
    c->launches++;
    cudaEventRecord(c->ev_stage[b], c->s_pack);
    if ((J + 1) % BAND == 0 || J + 1 == c->nt) cudaEventRecord(c->ev_band[J / BAND], c->s_pack);
  }
  return B2D_OK;
}

// Enqueue the host strips [ing.next, J1) (whole bands) of the run's input.
static int ingest_upto(Ctx* c, int J1) {
  if (!c->ing.active) return B2D_OK;
  J1 = std::min(c->nt, ((J1 + BAND - 1) / BAND) * BAND);
  if (J1 <= c->ing.next) return B2D_OK;
  const int rc = ingest_host_strips(c, c->ing.a, c->ing.lda, c->ing.dtype, c->ing.skip, c->ing.next, J1);
  if (rc) {
    c->ing.active = false;  // strips from ing.next on were not all enqueued: no later wait may pass
    return rc;
  }
  c->ing.next = J1;
  return B2D_OK;
}
static int ingest_start(Ctx* c, const void* a, int64_t lda, int dtype, int skip) {
  c->ing = Ctx::Ingest{a, lda, dtype, skip, 0, true};
  const char* pe = getenv("B2D_INGEST_PROGRESSIVE");
  const bool progressive = pe ? atoi(pe) != 0 : c->src_pageable;
  return progressive ? B2D_OK : ingest_upto(c, c->nt);
}

static int factor_host_impl(Ctx* c, const void* a, int64_t lda, int dtype, cudaStream_t user);
// An enqueue that fails half-way may leave staging callbacks pending on s_fill; they read the
// caller's buffer, so they finish before the error returns (the caller may free it).
// DMA copies already enqueued on the ingest streams read it too (pinned inputs always, small
// pageable copies through the driver), so every stream that may touch it is drained.
static int factor_host(Ctx* c, const void* a, int64_t lda, int dtype, cudaStream_t user) {
  const int rc = factor_host_impl(c, a, lda, dtype, user);
  if (rc != B2D_OK) {
    for (cudaStream_t s : {c->s_fill, c->s_copy, c->s_pack, c->o.s_h2d, c->s_main, c->s_mid, c->s_side, c->o.s_walk})
      if (s) cudaStreamSynchronize(s);
    c->ing.active = false;
    c->pending = false;
  }
  return rc;
}
static int factor_host_impl(Ctx* c, const void* a, int64_t lda, int dtype, cudaStream_t user) {
  if (c->mg) return mg_factor(c->mg, a, lda, dtype, true, user);
  if (dtype != B2D_F64 && dtype != B2D_F32) return set_err(B2D_ERR_USAGE, "dtype code %d", dtype);
  if (lda < c->m) return set_err(B2D_ERR_USAGE, "lda %lld < m", (long long)lda);
  {
    // pageable input (not page-locked): staged through pinned buffers (h2d_2d); B2D_HOST_STAGING=0
    // leaves it to the driver's pageable copies
    cudaPointerAttributes pa{};
    const bool known = cudaPointerGetAttributes(&pa, a) == cudaSuccess;
    cudaGetLastError();
    const char* hs = getenv("B2D_HOST_STAGING");
    c->src_pageable = (hs ? atoi(hs) != 0 : true) && (!known || pa.type == cudaMemoryTypeUnregistered);
  }
  if (c->ldl32) return run_ldl32(c, a, lda, dtype, true, user);
  if (c->ooc) return run_ooc(c, a, lda, dtype, user);
  if (c->ldl_ic) return run_ldl_incore(c, a, lda, dtype, true, user);
  if (c->lu_ic) return run_lu_incore(c, a, lda, dtype, true, user);
  CUDA_TRY(cudaSetDevice(c->device));
  const int64_t npad = (int64_t)c->nt * T;
  const size_t esz = dtype == B2D_F64 ? 8 : 4;
  for (int b = 0; b < NSTAGE; ++b)
    if (!c->strip[b]) CUDA_TRY(cudaMalloc(&c->strip[b], (size_t)T * npad * 8));
  begin(c, user);
  plan_bands(c, esz);
  int rc = ingest_start(c, a, lda, dtype, 0);
  if (rc) return rc;
  // pageable: the bands step 0 waits for now, then each step enqueues the bands that join the
  // updates up to two steps ahead (enqueue_factor's hook runs before the step's waits)
  const int nbands = (c->nt + BAND - 1) / BAND;
  auto bands_upto = [&](int st) {
    int b = 0;
    while (b < nbands && c->act[b] <= st) ++b;
    return b * BAND;
  };
  if ((rc = ingest_upto(c, bands_upto(-1)))) return rc;
  int hook_rc = 0;
  const std::function<void(int)> hook = [&](int st) {
    if (!hook_rc) hook_rc = ingest_upto(c, st == INT_MAX ? c->nt : bands_upto(st + 2));
  };
  enqueue_factor(c, FactorTarget{TileMap{c->tiles, 0, c->nt}, c->nt, 0}, true, &hook);
  if (hook_rc) return hook_rc;
  c->ing.active = false;
  enqueue_prefix(c);
  cudaEventRecord(c->ev_join, c->s_pack);
  cudaStreamWaitEvent(c->s_main, c->ev_join, 0);
  end(c, user);
  CUDA_TRY(cudaGetLastError());
  return B2D_OK;
}

// ---------------------------------------------------------------- out-of-core block streamer

// One visit of the reference's symmetric tile walk, stage k (memdet.py:83-145).
struct Visit {
  int i, j;
  bool col_start, load_b, load_c, solve_c, write_c, next_diag;
};

static std::vector<Visit> stage_visits(int nb, int k) {
  std::vector<Visit> v;
  for (int j = nb - 1; j > k; --j) {
    const bool last_col = j == nb - 1;
    std::vector<int> rows{j};
    for (int i = k + 1; i < j; ++i) rows.push_back(i);
    for (size_t pos = 0; pos < rows.size(); ++pos) {
      const int i = rows[pos];
      const bool off = i != j;
      v.push_back(Visit{i, j, pos == 0, pos == 0 && last_col, off, off && last_col,
                        off && last_col && nb > 2 && i < j - 1, i == k + 1 && j == k + 1});
    }
  }
  return v;
}

// Load reference block (ri, rj), ri <= rj (the row-major upper tile the reference reads), into
// slot s as the engine's lower block (rj, ri): from the scratchpad if it was written this run
// (the reference cache table, storage.py:134-144), else from the input in 128-row strips
// (H2D + pack_block_kernel).  Waits until the slot's previous contents are consumed and stored.
// Staged scratchpad transfers (scratch_mode 2 / 3): contiguous ranges split into pinned-buffer
// sized pieces.  HBM -> scratch: the DMA into ring buffer k (on `s`), then a host callback on
// s_fill drains it into the pageable / file mapping with the host pool; the buffer is reused once
// drained (callbacks on s_drain).  Scratch -> HBM: h2d_linear through the input-staging ring (fill
// callback on s_fill, then DMA); a load of a stored block waits for its last drain (ev_key), so
// it reads the drained bytes.  Returns after enqueueing; `drained` (optional) is recorded
// after the last drain.
static void CUDART_CB drain_cb(void* p) {
  std::unique_ptr<FillJob> j(static_cast<FillJob*>(p));
  const size_t per = (size_t)1 << 20;
  const int ntask = (int)((j->width + per - 1) / per);
  j->pool->run(ntask, [&](int t) {
    const size_t off = (size_t)t * per, n = std::min(per, j->width - off);
    if (j->dir == 1) {
      for (size_t w = 0; w < n;) {
        const ssize_t r = pwrite(j->fd, j->src + off + w, n - w, (off_t)(j->foff + off + w));
        if (r <= 0) break;
        w += (size_t)r;
      }
    } else if (j->dir == 2) {
      for (size_t w = 0; w < n;) {
        const ssize_t r = pread(j->fd, j->dst + off + w, n - w, (off_t)(j->foff + off + w));
        if (r <= 0) {
          memset(j->dst + off + w, 0, n - w);
          break;
        }
        w += (size_t)r;
      }
    } else {
      memcpy(j->dst + off, j->src + off, n);
    }
  });
}
static int ensure_staging(Ctx* c) {
  if (c->s_fill) return B2D_OK;
  c->hbuf_bytes = HBUF_BYTES;
  CUDA_TRY(cudaStreamCreateWithFlags(&c->s_fill, cudaStreamNonBlocking));
  for (int k = 0; k < NHBUF; ++k) {
    CUDA_TRY(cudaHostAlloc(&c->hbuf[k], c->hbuf_bytes, cudaHostAllocDefault));
    cudaEventCreateWithFlags(&c->ev_hfill[k], cudaEventDisableTiming);
    cudaEventCreateWithFlags(&c->ev_hcopy[k], cudaEventDisableTiming);
  }
  return B2D_OK;
}
static int d2h_linear(Ctx* c, void* dst, const void* src, size_t bytes, cudaStream_t s, cudaEvent_t drained) {
  Ooc& o = c->o;
  if (int rc = ensure_staging(c)) return rc;
  if (!o.s_drain) CUDA_TRY(cudaStreamCreateWithFlags(&o.s_drain, cudaStreamNonBlocking));
  if (!o.dbuf[0])
    for (int k = 0; k < Ooc::NDBUF; ++k) {
      CUDA_TRY(cudaHostAlloc(&o.dbuf[k], HBUF_BYTES, cudaHostAllocDefault));
      cudaEventCreateWithFlags(&o.ev_ddma[k], cudaEventDisableTiming);
      cudaEventCreateWithFlags(&o.ev_dfree[k], cudaEventDisableTiming);
    }
  for (size_t off = 0; off < bytes; off += HBUF_BYTES) {
    const size_t n = std::min(HBUF_BYTES, bytes - off);
    const int k = (int)(o.dseq++ % Ooc::NDBUF);
    if (o.dbuf_used[k]) cudaStreamWaitEvent(s, o.ev_dfree[k], 0);
    CUDA_TRY(cudaMemcpyAsync(o.dbuf[k], (const char*)src + off, n, cudaMemcpyDeviceToHost, s));
    cudaEventRecord(o.ev_ddma[k], s);
    cudaStreamWaitEvent(o.s_drain, o.ev_ddma[k], 0);
    auto* job = new FillJob{host_pool(), (char*)dst + off, (const char*)o.dbuf[k], 0, n, 1};
    if (o.scratch_fd >= 0) {
      job->fd = o.scratch_fd;
      job->foff = (int64_t)(uintptr_t)dst + (int64_t)off;
      job->dst = nullptr;
      job->dir = 1;
    }
    if (cudaLaunchHostFunc(o.s_drain, drain_cb, job) != cudaSuccess) {
      delete job;
      return set_err(B2D_ERR_CUDA, "cudaLaunchHostFunc failed");
    }
    cudaEventRecord(o.ev_dfree[k], o.s_drain);
    o.dbuf_used[k] = true;
  }
  if (drained) cudaEventRecord(drained, o.s_drain);
  return B2D_OK;
}
static int h2d_linear(Ctx* c, void* dst, const void* src, size_t bytes, cudaStream_t s) {
  if (int rc = ensure_staging(c)) return rc;
  for (size_t off = 0; off < bytes; off += c->hbuf_bytes) {
    const size_t n = std::min(c->hbuf_bytes, bytes - off);
    const int k = (int)(c->hseq++ % NHBUF);
    if (c->hbuf_used[k]) cudaStreamWaitEvent(c->s_fill, c->ev_hcopy[k], 0);
    auto* job = new FillJob{host_pool(), (char*)c->hbuf[k], (const char*)src + off, 0, n, 1};
    if (c->o.scratch_fd >= 0) {
      job->fd = c->o.scratch_fd;
      job->foff = (int64_t)(uintptr_t)src + (int64_t)off;
      job->src = nullptr;
      job->dir = 2;
    }
    if (cudaLaunchHostFunc(c->s_fill, drain_cb, job) != cudaSuccess) {
      delete job;
      return set_err(B2D_ERR_CUDA, "cudaLaunchHostFunc failed");
    }
    cudaEventRecord(c->ev_hfill[k], c->s_fill);
    cudaStreamWaitEvent(s, c->ev_hfill[k], 0);
    CUDA_TRY(cudaMemcpyAsync((char*)dst + off, c->hbuf[k], n, cudaMemcpyHostToDevice, s));
    cudaEventRecord(c->ev_hcopy[k], s);
    c->hbuf_used[k] = true;
  }
  return B2D_OK;
}

static int ooc_load(Ctx* c, int ri, int rj, int s, const void* a, int64_t lda, int dtype, bool trans = true) {
  Ooc& o = c->o;
  cudaStreamWaitEvent(o.s_h2d, o.ev_used[s], 0);
  cudaStreamWaitEvent(o.s_h2d, o.ev_stored[s], 0);
  auto key = std::make_pair(ri, rj);
  if (o.written.count(key)) {
    cudaStreamWaitEvent(o.s_h2d, o.ev_key[key], 0);  // the scratch copy must have landed
    if (o.scratch_map || o.scratch_fd >= 0) {
      cudaStreamWaitEvent(c->s_fill, o.ev_key[key], 0);  // the host reads it only once drained
      if (int rc = h2d_linear(c, o.slot[s], o.scratch[key], o.slot_bytes(), o.s_h2d)) return rc;
    } else {
      CUDA_TRY(cudaMemcpyAsync(o.slot[s], o.scratch[key], o.slot_bytes(), cudaMemcpyDefault, o.s_h2d));
    }
    if (!o.dev_scratch) c->h2d += (int64_t)o.slot_bytes();
  } else if (!trans) {
    // generic blocks (LU): reference block (ri, rj) as the engine block (ri, rj), strip J of
    // its rows -> tile row J
    const size_t esz = dtype == B2D_F64 ? 8 : 4;
    const int64_t rows_blk = o.size(ri), cols_blk = o.size(rj);
    const int64_t ld_stage = (int64_t)o.nbt * T;
    for (int J = 0; J < o.tiles(ri); ++J) {
      const int64_t frow = (int64_t)ri * o.b + (int64_t)J * T;
      const int64_t nrows = std::min<int64_t>(T, rows_blk - (int64_t)J * T);
      const char* src = (const char*)a + ((size_t)frow * lda + (size_t)rj * o.b) * esz;
      if (int rc = h2d_2d(c, o.stage, (size_t)ld_stage * esz, src, (size_t)lda * esz, (size_t)cols_blk * esz,
                          (size_t)nrows, o.s_h2d))
        return rc;
      c->h2d += nrows * cols_blk * (int64_t)esz;
      if (dtype == B2D_F64)
        pack_block_nt_kernel<double><<<o.tiles(rj), 256, 0, o.s_h2d>>>(
            (const double*)o.stage, ld_stage, rows_blk, cols_blk, ri == rj, o.map(s), J);
      else
        pack_block_nt_kernel<float><<<o.tiles(rj), 256, 0, o.s_h2d>>>(
            (const float*)o.stage, ld_stage, rows_blk, cols_blk, ri == rj, o.map(s), J);
      c->launches++;
    }
  } else {
    const size_t esz = dtype == B2D_F64 ? 8 : 4;
    const int64_t rows_blk = o.size(rj), cols_blk = o.size(ri);  // engine block: rows of rj, cols of ri
    const int64_t ld_stage = (int64_t)o.nbt * T;
    for (int J = 0; J < o.tiles(ri); ++J) {
      const int64_t frow = (int64_t)ri * o.b + (int64_t)J * T;            // first file row of the strip
      const int64_t nrows = std::min<int64_t>(T, cols_blk - (int64_t)J * T);
      const char* src = (const char*)a + ((size_t)frow * lda + (size_t)rj * o.b) * esz;
      if (int rc = h2d_2d(c, o.stage, (size_t)ld_stage * esz, src, (size_t)lda * esz, (size_t)rows_blk * esz,
                          (size_t)nrows, o.s_h2d))
        return rc;
      c->h2d += nrows * rows_blk * (int64_t)esz;
      if (dtype == B2D_F64)
        pack_block_kernel<double><<<o.tiles(rj), PACK_THREADS, PACK_SMEM, o.s_h2d>>>(
            (const double*)o.stage, ld_stage, rows_blk, cols_blk, ri == rj, o.map(s), J);
      else
        pack_block_kernel<float><<<o.tiles(rj), PACK_THREADS, PACK_SMEM, o.s_h2d>>>(
            (const float*)o.stage, ld_stage, rows_blk, cols_blk, ri == rj, o.map(s), J);
      c->launches++;
    }
  }
  cudaEventRecord(o.ev_loaded[s], o.s_h2d);
  o.reads++;
  return B2D_OK;
}

// Write slot s to the scratchpad as reference block (ri, rj) (storage.py:258-263).
static int ooc_store(Ctx* c, int ri, int rj, int s) {
  Ooc& o = c->o;
  auto key = std::make_pair(ri, rj);
  auto it = o.scratch.find(key);
  if (it == o.scratch.end()) {
    // slots are bound in first-write order and never reassigned (storage.py:167-181)
    if (o.scratch.size() >= o.pool.size())
      return set_err(B2D_ERR_CUDA, "scratchpad full (%zu slots) writing block (%d, %d)", o.pool.size(), ri, rj);
    it = o.scratch.emplace(key, o.pool[o.scratch.size()]).first;
  }
  cudaStreamWaitEvent(o.s_d2h, o.ev_used[s], 0);
  auto ek = o.ev_key.find(key);
  if (ek == o.ev_key.end()) {
    cudaEvent_t e;
    cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    ek = o.ev_key.emplace(key, e).first;
  }
  if (o.scratch_map || o.scratch_fd >= 0) {
    // the slot is free once its DMA pieces are out; the block is in the scratchpad once drained
    if (int rc = d2h_linear(c, it->second, o.slot[s], o.slot_bytes(), o.s_d2h, ek->second)) return rc;
    cudaEventRecord(o.ev_stored[s], o.s_d2h);
  } else {
    CUDA_TRY(cudaMemcpyAsync(it->second, o.slot[s], o.slot_bytes(), cudaMemcpyDefault, o.s_d2h));
    cudaEventRecord(o.ev_stored[s], o.s_d2h);
    cudaEventRecord(ek->second, o.s_d2h);
  }
  if (!o.dev_scratch) c->d2h += (int64_t)o.slot_bytes();
  o.written.insert(key);
  o.writes++;
  return B2D_OK;
}

// Panel solve X <- X L^{-T} of R x Q tiles against the factored diagonal block lkk (Q x Q tiles,
// unit or not per inv): right-looking over L's tile-columns in groups of W (dense.py:94-99).
// Wg: group width in tile-columns (0 = the panel width W_TILES).  Any grouping gives every tile
// its k-chunks in increasing order, so the result does not depend on it; narrow groups shorten
// the chain of left-looking launches (R tiles each) for a solve on the critical path.
static void trsm_panel(Ctx* c, cudaStream_t s, const TileMap& x, int R, const TileMap& lkk, int Q,
                       const double* inv, int Wg = 0) {
  const int W = Wg > 0 ? Wg : c->W_TILES;
  const char* lbe = getenv("B2D_LEFT_BELOW");
  const bool left = lbe ? atoi(lbe) != 0 : true;
  for (int q0 = 0; q0 < Q; q0 += W) {
    const int qe = std::min(q0 + W, Q);
    for (int q = q0; q < qe; ++q) {
      if (left && q > q0) {
        // left-looking inside the group: column q takes columns [q0, q) in one launch right
        // before its solve (same k order as the right-looking K = 128 updates: bit-identical)
        GemmTask u{};
        u.a = x;
        u.b = lkk;
        u.c = x;
        u.out = TileSet{0, R, q, q + 1, 0, 0};
        u.p0 = q0;
        u.p1 = q;
        launch_gemm(c, s, MODE_UPDATE, u, false, 0.0);
      }
      GemmTask t{};
      t.c = x;
      t.binv = inv + (int64_t)q * TILE_ELEMS;
      t.out = TileSet{0, R, q, q + 1, 0, 0};
      t.k = q;
      launch_gemm(c, s, MODE_TRSM, t, false, 0.0);
      if (!left && q + 1 < qe) {
        GemmTask u{};
        u.a = x;
        u.b = lkk;
        u.c = x;
        u.out = TileSet{0, R, q + 1, qe, 0, 0};
        u.p0 = q;
        u.p1 = q + 1;
        launch_gemm(c, s, MODE_UPDATE, u, false, 0.0);
      }
    }
    if (qe < Q) {
      GemmTask u{};
      u.a = x;
      u.b = lkk;
      u.c = x;
      u.out = TileSet{0, R, qe, Q, 0, 0};
      u.p0 = q0;
      u.p1 = qe;
      launch_gemm(c, s, MODE_UPDATE, u, false, 0.0);
    }
  }
}

// Look-ahead panel solve of the critical block row (the rows of block k+1: factor k -> these
// rows -> the update of diagonal block (k+1, k+1) -> factor k+1), with that diagonal update
// folded in.  The row's Q tile-columns go in groups G_0, G_1, ... of Wg; U(g -> h) is the update
// of group h by the solved group g (K = 128 Wg).  Stream A carries the chain: solve(g) (left-
// looking inside the group), then U(g -> g+1); stream B the rest of each group's updates
// U(g -> h >= g+2); stream C the D^{-1} scaling of group g and its K-chunk of the diagonal update
// (du: output tiles = the diagonal block, A = ps, B = pu).  Every tile still receives its K-chunks
// in increasing order -- the FP64 accumulators continue exactly across launches -- so pu, ps and
// the diagonal block equal those of trsm_panel + scale_cols + one K = 128 Q update bit for bit.
// On return A has joined B and C.
static int trsm_panel_la(Ctx* c, cudaStream_t A, const TileMap& pu, const TileMap& ps, int R, const TileMap& lkk,
                         int Q, const double* inv, int Wg, int64_t nsize, const double* dblk, GemmTask du) {
  if (!c->s_la[0]) {
    int pr = 0;
    cudaStreamGetPriority(A, &pr);
    for (auto& st : c->s_la) CUDA_TRY(cudaStreamCreateWithPriority(&st, cudaStreamNonBlocking, pr));
  }
  const int G = (Q + Wg - 1) / Wg;
  while ((int)c->ev_la.size() < 2 * G + 2) {
    cudaEvent_t e;
    CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    c->ev_la.push_back(e);
  }
  cudaStream_t B = c->s_la[0], C = c->s_la[1];
  cudaEvent_t* es = c->ev_la.data();      // es[g]: group g solved (A)
  cudaEvent_t* er = es + G;               // er[g]: U(g -> h >= g+2) done (B)
  cudaEvent_t ec = c->ev_la[2 * G], eb = c->ev_la[2 * G + 1];
  auto gcol = [&](int g) { return std::min(Q, g * Wg); };
  auto upd = [&](cudaStream_t st, int g, int h0, int h1) {  // U(g -> columns [h0, h1))
    if (h1 <= h0) return;
    GemmTask u{};
    u.a = pu;
    u.b = lkk;
    u.c = pu;
    u.out = TileSet{0, R, h0, h1, 0, 0};
    u.p0 = gcol(g);
    u.p1 = gcol(g + 1);
    launch_gemm(c, st, MODE_UPDATE, u, false, 0.0);
  };
  for (int g = 0; g < G; ++g) {
    const int q0 = gcol(g), qe = gcol(g + 1);
    if (g >= 1) {
      // U(g-1 -> g) on the chain, after every earlier update of group g (B's U(g-2 -> g))
      if (g >= 2) cudaStreamWaitEvent(A, er[g - 2], 0);
      upd(A, g - 1, q0, qe);
    }
    for (int q = q0; q < qe; ++q) {
      if (q > q0) {
        GemmTask u{};
        u.a = pu;
        u.b = lkk;
        u.c = pu;
        u.out = TileSet{0, R, q, q + 1, 0, 0};
        u.p0 = q0;
        u.p1 = q;
        launch_gemm(c, A, MODE_UPDATE, u, false, 0.0);
      }
      GemmTask t{};
      t.c = pu;
      t.binv = inv + (int64_t)q * TILE_ELEMS;
      t.out = TileSet{0, R, q, q + 1, 0, 0};
      t.k = q;
      launch_gemm(c, A, MODE_TRSM, t, false, 0.0);
    }
    cudaEventRecord(es[g], A);
    // B: the rest of group g's updates (groups g+2 ..), after group g is solved
    cudaStreamWaitEvent(B, es[g], 0);
    upd(B, g, gcol(g + 2), Q);
    cudaEventRecord(er[g], B);
    // C: scale group g, then its K-chunk of the diagonal update
    cudaStreamWaitEvent(C, es[g], 0);
    TileMap su = pu, ss = ps;
    su.base += (int64_t)q0 * TILE_ELEMS;
    ss.base += (int64_t)q0 * TILE_ELEMS;
    const int64_t nrem = std::max<int64_t>(0, nsize - (int64_t)q0 * T);
    scale_cols_kernel<<<1024, 256, 0, C>>>(su, ss, R, qe - q0, nrem, dblk + (int64_t)q0 * T);
    c->launches++;
    du.p0 = q0;
    du.p1 = qe;
    launch_gemm(c, C, MODE_UPDATE, du, true, (double)du.out.count() * 2.0 * T * T * (qe - q0) * T);
  }
  cudaEventRecord(ec, C);
  cudaEventRecord(eb, B);
  cudaStreamWaitEvent(A, ec, 0);
  cudaStreamWaitEvent(A, eb, 0);
  return B2D_OK;
}

// Panel solve of slot s (engine lower block (x, k), x's rows) against the factored diagonal
// block in slot sa.
static void ooc_trsm(Ctx* c, int s, int x, int sa, int k, const double* inv = nullptr) {
  Ooc& o = c->o;
  if (!inv) inv = c->inv;
  cudaStreamWaitEvent(o.s_work, o.ev_loaded[s], 0);
  trsm_panel(c, o.s_work, o.map(s), o.tiles(x), o.map(sa), o.tiles(k), inv);
  cudaEventRecord(o.ev_used[s], o.s_work);
  cudaEventRecord(o.ev_used[sa], o.s_work);
}

// Schur update of slot st (engine block (j, i)) -= L(j,k) L(i,k)^T (dense.py:109-116).
static void ooc_schur(Ctx* c, int st, int j, int i, int sbj, int sci, int k) {
  Ooc& o = c->o;
  for (int x : {st, sbj, sci}) cudaStreamWaitEvent(o.s_work, o.ev_loaded[x], 0);
  GemmTask t{};
  t.a = o.map(sbj);
  t.b = o.map(sci);
  t.c = o.map(st);
  t.out = TileSet{0, o.tiles(j), 0, o.tiles(i), i == j ? 1 : 0, 0};
  t.p0 = 0;
  t.p1 = o.tiles(k);
  const double K = (double)t.p1 * T;
  launch_gemm(c, o.s_work, MODE_UPDATE, t, true, (double)t.out.count() * 2.0 * T * T * K);
  cudaEventRecord(o.ev_used[st], o.s_work);
  cudaEventRecord(o.ev_used[sbj], o.s_work);
  cudaEventRecord(o.ev_used[sci], o.s_work);
}

// Pivoted LDL^T of the diagonal block in slot sa (stage k): dense copy, tolerance scale, the
// cooperative 1x1-pivot factorisation, permutation / log|d| bookkeeping, then the unit factor
// back into the slot and the inverses of its diagonal tiles for the panel solves.
// Stream memory operations (driver API, through the runtime's entry-point lookup: no -lcuda).
typedef int (*PFN_streamValue32)(cudaStream_t, CUdeviceptr_v2_compat, unsigned, unsigned);
static PFN_streamValue32 stream_wait_value32() {
  static PFN_streamValue32 fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &p, cudaEnableDefault, &q) != cudaSuccess) p = nullptr;
    return (PFN_streamValue32)p;
  }();
  return fn;
}
static PFN_streamValue32 stream_write_value32() {
  static PFN_streamValue32 fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &p, cudaEnableDefault, &q) != cudaSuccess) p = nullptr;
    return (PFN_streamValue32)p;
  }();
  return fn;
}
constexpr unsigned B2D_STREAM_WAIT_VALUE_GEQ = 0;  // CU_STREAM_WAIT_VALUE_GEQ

// The block factor with the panel server (ldl_panel_server_kernel) on s and the bulk updates on
// o.s_bulk, each gated on the server's panel counter and bumping the bulk counter.
static int ldl_server_factor(Ctx* c, const LdlArgs& g, cudaStream_t s) {
  Ooc& o = c->o;
  auto waitv = stream_wait_value32();
  auto writev = stream_write_value32();
  if (!waitv || !writev) return set_err(B2D_ERR_UNSUPPORTED, "stream memory operations unavailable");
  if (!o.lflags) {
    CUDA_TRY(cudaMalloc((void**)&o.lflags, 8));
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    CUDA_TRY(cudaStreamCreateWithPriority(&o.s_bulk, cudaStreamNonBlocking, hi));
    cudaEventCreateWithFlags(&o.ev_lreset, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&o.ev_lbulk, cudaEventDisableTiming);
  }
  const int64_t n = g.n;
  cudaMemsetAsync(o.lflags, 0, 8, s);
  cudaEventRecord(o.ev_lreset, s);
  cudaStreamWaitEvent(o.s_bulk, o.ev_lreset, 0);  // the counters are reset (and the block is ready)
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = LC;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.gridDim = dim3(LC);
  cfg.blockDim = dim3(LC_THREADS);
  cfg.dynamicSmemBytes = ldl_cluster_smem((int)((n + LC - 1) / LC));
  cfg.stream = s;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  CUDA_TRY(cudaLaunchKernelEx(&cfg, ldl_panel_server_kernel, g, o.lflags));
  c->launches++;
  const CUdeviceptr_v2_compat panels = (CUdeviceptr_v2_compat)(uintptr_t)o.lflags;
  const CUdeviceptr_v2_compat bulks = panels + 4;
  unsigned p = 0;
  for (int64_t r0 = 0; r0 < n; r0 += LDL_NB, ++p) {
    const int nbk = (int)std::min<int64_t>(LDL_NB, n - r0);
    const int64_t mt = (n - r0 - nbk + LDL_BT - 1) / LDL_BT, ntile = mt * (mt + 1) / 2;
    if (waitv(o.s_bulk, panels, p + 1, B2D_STREAM_WAIT_VALUE_GEQ) != 0)
      return set_err(B2D_ERR_CUDA, "cuStreamWaitValue32 failed");
    if (ntile > 0) {
      ldl_bulk_kernel<<<(unsigned)ntile, 256, 0, o.s_bulk>>>(g, r0, nbk, ntile, (unsigned*)nullptr, 0u);
      c->launches++;
    }
    if (writev(o.s_bulk, bulks, p + 1, 0) != 0) return set_err(B2D_ERR_CUDA, "cuStreamWriteValue32 failed");
  }
  cudaEventRecord(o.ev_lbulk, o.s_bulk);
  cudaStreamWaitEvent(s, o.ev_lbulk, 0);
  return B2D_OK;
}

// Group pipeline of the pivoted factor (B2D_LDL_GROUPS, default on; in-core row schedule): the
// finished column groups of gw tile-columns are handed out while the factor is still running --
// after the last panel of group g (and its bulk launch, which carries the row interchanges of the
// finished columns) rows < e1 = (g + 1) gw T of L, the pivots and D of steps < e1 and the block
// permutation's entries < e1 are final (step r only touches rows >= r), so the group's L tile rows,
// its diagonal-tile inverses and its permutation entries are written on a side stream and ev[g]
// recorded; the panel rows of the stage then solve and apply group g while the factor works on
// group g + 1 (factor 0 no longer runs alone on the GPU; the chain row's solve hides behind the
// factor).  `count` groups were handed out early; the remaining ones are ready with the factor.
struct LdlGroups {
  int gw = 4;
  std::vector<cudaEvent_t>* ev = nullptr;
  int count = 0;
};
static int ldl_factor_block(Ctx* c, const TileMap& blk, int k, cudaStream_t s, bool overlapped = false,
                            LdlGroups* grp = nullptr) {
  Ooc& o = c->o;
  const int nt = o.tiles(k);
  int64_t n = o.size(k);
  const int64_t ld = (int64_t)o.nbt * T, g0 = (int64_t)k * o.b;
  double* dblk = o.dblk_of(k);
  int64_t* perm = o.perm_of(k);
  double* inv = o.inv_of(k, c->inv);
  const unsigned ntri = (unsigned)(nt * (nt + 1) / 2);
  bool groups = false;
  if (grp) grp->count = 0;
  unpack_block_kernel<<<ntri, 256, 0, s>>>(blk, nt, o.dense, ld, 1);
  cudaMemsetAsync(o.amax, 0, 8, s);
  block_absmax_kernel<<<std::max<int64_t>(1, std::min<int64_t>(4096, (n * n + 255) / 256)), 256, 0, s>>>(o.dense, ld, n, o.amax);
  // blocked pivoted LDL: panels of LDL_NB steps (one CTA), then the delayed trailing update
  const LdlArgs g{o.dense, o.ltag, o.lC, o.lW, o.ldiag, o.lcol, dblk, o.swaps, c->fail, o.amax, ld, n, g0};
  cudaMemsetAsync(o.ltag, 0, (size_t)ld * ld, s);
  ldl_diag_init_kernel<<<(unsigned)std::max<int64_t>(1, (n + 255) / 256), 256, 0, s>>>(g);
  c->launches += 1;
  // B2D_LDL_SINGLE_CTA forces the one-CTA panel kernel (the path for blocks above 16*384 rows)
  const bool single_cta = getenv("B2D_LDL_SINGLE_CTA") != nullptr;
  // B2D_LDL_PERSIST: 0 (default) = per-panel kernels; 1 = the one-launch cluster factor when
  // the factor runs beside other work (it holds its 16 SMs, but its bulk updates run on those
  // 16 SMs only: 58 ms vs 23 ms alone at b = 4096, so it loses at C2); 2 = always
  const char* pe = getenv("B2D_LDL_PERSIST");
  const int persist = pe ? atoi(pe) : 0;
  // B2D_LDL_SERVER (1: beside other work, 2: always; default 0 -- measured slower at C2, 467 vs 453
  // ms: the bulk steps then share the FP64 pipe with the DMMA updates): the panel server (one cluster holding its SMs)
  // with each panel's bulk update gated by stream memory operations on s_bulk
  const char* sve = getenv("B2D_LDL_SERVER");
  const int server = sve ? atoi(sve) : 0;
  if (n <= (int64_t)LC * LC_RMAX && !single_cta && persist == 0 && (server == 2 || (server == 1 && overlapped))) {
    if (int rc = ldl_server_factor(c, g, s)) return rc;
  } else
  if (n <= (int64_t)LC * LC_RMAX && !single_cta && (persist == 2 || (persist == 1 && overlapped))) {
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = LC;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3(LC);
    cfg.blockDim = dim3(LC_THREADS);
    cfg.dynamicSmemBytes = ldl_factor_smem((int)((n + LC - 1) / LC));
    cfg.stream = s;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    CUDA_TRY(cudaLaunchKernelEx(&cfg, ldl_factor_cluster_kernel, g));
    c->launches += 1;
  } else {
  // B2D_LDL_PIPE (default 1): panel p+1 is launched as soon as panel p is done, on the other of
  // two streams, and waits in the kernel for bulk update p (ldl.cu pipe_wait): its cluster takes
  // its SMs while bulk p runs, instead of after it (beside the trailing DMMA updates a launch
  // waits ~100 us for SMs).  Bulk p follows panel p on the panel's stream.
  // clusters: the rows' C / W in shared memory up to LC * LC_RMAX rows, in global memory up to
  // LC * LC_RMAX_BIG (B2D_LDL_BIG=0: the one-CTA panel above LC * LC_RMAX, as round 1)
  const char* bge = getenv("B2D_LDL_BIG");
  const bool big = n > (int64_t)LC * LC_RMAX && n <= (int64_t)LC * LC_RMAX_BIG && (bge ? atoi(bge) != 0 : true);
  const bool clus = (n <= (int64_t)LC * LC_RMAX || big) && !single_cta;
  if (big && o.lrows_bytes < ldl_big_rows_bytes(n)) {
    cudaFree(o.lrows);
    o.lrows = nullptr;
    o.lrows_bytes = 0;
    CUDA_TRY(cudaMalloc((void**)&o.lrows, ldl_big_rows_bytes(n)));
    o.lrows_bytes = ldl_big_rows_bytes(n);
  }
  const char* pie = getenv("B2D_LDL_PIPE");
  const bool pipe = (pie ? atoi(pie) != 0 : true) && clus;
  cudaStream_t pst[2] = {s, s};
  if (pipe) {
    if (!o.lpipe) {
      CUDA_TRY(cudaMalloc((void**)&o.lpipe, 16));
      int lo = 0, hi = 0;
      cudaDeviceGetStreamPriorityRange(&lo, &hi);
      int sp = hi;
      cudaStreamGetPriority(s, &sp);
      CUDA_TRY(cudaStreamCreateWithPriority(&o.s_lalt, cudaStreamNonBlocking, sp));
      for (auto* e : {&o.ev_lpanel[0], &o.ev_lpanel[1], &o.ev_lalt})
        CUDA_TRY(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
    }
    pst[1] = o.s_lalt;
    CUDA_TRY(cudaMemsetAsync(o.lpipe, 0, 16, s));
    cudaEventRecord(o.ev_lalt, s);
    cudaStreamWaitEvent(o.s_lalt, o.ev_lalt, 0);  // counters reset, block state ready
  }
  groups = grp && grp->ev && grp->gw > 0 && clus && !big && n <= LDL_FINISH_SMEM_MAX;
  if (groups && !o.s_lgrp) {
    int sp = 0;
    cudaStreamGetPriority(s, &sp);
    CUDA_TRY(cudaStreamCreateWithPriority(&o.s_lgrp, cudaStreamNonBlocking, sp));
    CUDA_TRY(cudaEventCreateWithFlags(&o.ev_lgrp, cudaEventDisableTiming));
  }
  unsigned pidx = 0;
  for (int64_t r0 = 0; r0 < n; r0 += LDL_NB, ++pidx) {
    const int nbk = (int)std::min<int64_t>(LDL_NB, n - r0);
    if (clus) {
      cudaStream_t ps = pst[pidx & 1];
      if (pipe && pidx > 0) cudaStreamWaitEvent(ps, o.ev_lpanel[(pidx - 1) & 1], 0);  // panel pidx-1 done
      // the panel on a 16-CTA cluster with its rows in distributed shared memory
      cudaLaunchConfig_t cfg = {};
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = LC;
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      cfg.gridDim = dim3(LC);
      cfg.blockDim = dim3(LC_THREADS);
      cfg.dynamicSmemBytes = big ? (size_t)((n + LC - 1) / LC) * 8 : ldl_cluster_smem((int)((n + LC - 1) / LC));
      cfg.stream = ps;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      unsigned* pp = pipe ? o.lpipe : nullptr;
      if (big)
        CUDA_TRY(cudaLaunchKernelEx(&cfg, ldl_panel_cluster_kernel<true>, g, r0, nbk, pp, pidx, o.lrows));
      else
        CUDA_TRY(cudaLaunchKernelEx(&cfg, ldl_panel_cluster_kernel<false>, g, r0, nbk, pp, pidx, (double*)nullptr));
      if (pipe) cudaEventRecord(o.ev_lpanel[pidx & 1], ps);
      // the cluster kernel stored the panel's L; the row interchanges of the finished columns
      // ride along the bulk update as extra blocks
      const int64_t mt = (n - r0 - nbk + LDL_BT - 1) / LDL_BT, ntile = mt * (mt + 1) / 2;
      const int64_t nswap = r0 > 0 ? std::min<int64_t>(148, (r0 + 63) / 64) : 0;
      if (ntile + nswap > 0) {
        ldl_bulk_kernel<<<(unsigned)(ntile + nswap), 256, 0, ps>>>(g, r0, nbk, ntile, pp, pidx);
        c->launches += 1;
      }
      c->launches += 1;
      if (groups) {
        const int64_t e1 = r0 + nbk, gcols = (int64_t)grp->gw * T;
        if (e1 < n && e1 % gcols == 0) {
          const int gi = (int)(e1 / gcols) - 1, I0 = gi * grp->gw, I1 = I0 + grp->gw;
          while ((int)grp->ev->size() <= gi) {
            cudaEvent_t e;
            CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            grp->ev->push_back(e);
          }
          // bulk pidx done => panel pidx done => bulk pidx-1 done (pipe_wait): everything up to e1
          cudaEventRecord(o.ev_lgrp, ps);
          cudaStreamWaitEvent(o.s_lgrp, o.ev_lgrp, 0);
          ldl_partial_perm_kernel<<<1, 256, (size_t)n * 8, o.s_lgrp>>>(o.swaps, n, e1 - gcols, e1, perm);
          pack_unit_lower_rows_kernel<<<(unsigned)(grp->gw * I1), 256, 0, o.s_lgrp>>>(o.dense, ld, n, blk, I0, I1);
          tile_inv_unit_kernel<<<grp->gw, T, T * 129 * 8, o.s_lgrp>>>(blk, inv, I0);
          cudaEventRecord((*grp->ev)[gi], o.s_lgrp);
          c->launches += 3;
          grp->count = gi + 1;
        }
      }
      continue;
    }
    ldl_panel_kernel<<<1, LDL_PANEL_THREADS, 0, s>>>(g, r0, nbk);
    const int64_t st_ctas = std::max<int64_t>(((n - r0) * nbk + 255) / 256, (r0 + 7) / 8);
    ldl_store_l_kernel<<<(unsigned)std::max<int64_t>(1, std::min<int64_t>(1024, st_ctas)), 256, 0, s>>>(g, r0, nbk);
    const int64_t mt = (n - r0 - nbk + LDL_BT - 1) / LDL_BT, ntile = mt * (mt + 1) / 2;
    if (ntile > 0) ldl_bulk_kernel<<<(unsigned)ntile, 256, 0, s>>>(g, r0, nbk, ntile, (unsigned*)nullptr, 0u);
    c->launches += ntile > 0 ? 3 : 2;
  }
  if (pipe) {  // the odd panels' stream joins the factor's stream
    cudaEventRecord(o.ev_lalt, o.s_lalt);
    cudaStreamWaitEvent(s, o.ev_lalt, 0);
  }
  }
  // the groups handed out early keep their outputs (the panel rows may be reading them)
  const int gdone = groups ? grp->count * grp->gw : 0;
  ldl_finish_kernel<<<(unsigned)std::max<int64_t>(1, (n + 255) / 256), 256,
                      n <= LDL_FINISH_SMEM_MAX ? (size_t)n * 8 : 0, s>>>(o.swaps, dblk, n, g0, perm,
                                                                        o.perm_global, c->ell, c->diag,
                                                                        (int64_t)gdone * T);
  if (gdone > 0) {
    pack_unit_lower_rows_kernel<<<(unsigned)((nt - gdone) * nt), 256, 0, s>>>(o.dense, ld, n, blk, gdone, nt);
    tile_inv_unit_kernel<<<nt - gdone, T, T * 129 * 8, s>>>(blk, inv, gdone);
    cudaStreamWaitEvent(s, (*grp->ev)[grp->count - 1], 0);  // the factor's end covers every group
  } else {
    pack_unit_lower_kernel<<<ntri, 256, 0, s>>>(o.dense, ld, n, blk, nt);
    tile_inv_unit_kernel<<<nt, T, T * 129 * 8, s>>>(blk, inv, 0);
  }
  c->launches += 7;
  return B2D_OK;
}

static int ooc_ldl_factor(Ctx* c, int sa, int k, cudaStream_t s) {
  Ooc& o = c->o;
  cudaStreamWaitEvent(s, o.ev_loaded[sa], 0);
  const int rc = ldl_factor_block(c, o.map(sa), k, s);
  cudaEventRecord(o.ev_used[sa], s);
  return rc;
}

// Generic (LU) diagonal block in slot sa (stage k), reference lu_inplace (dense.py:38-54):
// dense copy, blocked LU with block-local partial pivoting, pivots / permutation / log|u_ii|,
// then L (unit lower) back into slot sa and U^T (lower) into slot su with the inverses of
// their diagonal tiles for the row-block and column-block solves.
static int lu_factor_block(Ctx* c, const TileMap& blk, const TileMap& umap, int k, cudaStream_t s) {
  Ooc& o = c->o;
  const int nt = o.tiles(k);
  const int64_t n = o.size(k);
  const int64_t ld = (int64_t)o.nbt * T, g0 = (int64_t)k * o.b;
  double* dblk = o.dblk_of(k);
  int64_t* perm = o.perm_of(k);
  double* inv = (k & 1) && o.inv_odd ? o.inv_odd : c->inv;
  double* inv2 = (k & 1) && o.inv2_odd ? o.inv2_odd : o.inv2;
  unpack_block_kernel<<<(unsigned)(nt * nt), 256, 0, s>>>(blk, nt, o.dense, ld, 0);
  const LuArgs g{o.dense, dblk, o.swaps, c->fail, ld, n, g0};
  const int cols_grid = (int)std::max<int64_t>(1, (n + 255) / 256);
  for (int64_t r0 = 0; r0 < n; r0 += LU_NB) {
    const int nbk = (int)std::min<int64_t>(LU_NB, n - r0);
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = LC;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3(LC);
    cfg.blockDim = dim3(LC_THREADS);
    cfg.dynamicSmemBytes = lu_panel_smem((int)((n + LC - 1) / LC));
    cfg.stream = s;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    CUDA_TRY(cudaLaunchKernelEx(&cfg, lu_panel_cluster_kernel, g, r0, nbk));
    lu_swap_rows_kernel<<<cols_grid, 256, 0, s>>>(g, r0, nbk);
    const int64_t rest = n - r0 - nbk;
    if (rest > 0) {
      lu_u12_kernel<<<(unsigned)((rest + 127) / 128), 128, 0, s>>>(g, r0, nbk);
      const int64_t mt = (rest + 63) / 64;
      lu_bulk_kernel<<<(unsigned)(mt * mt), 256, 0, s>>>(g, r0, nbk);
    }
    c->launches += rest > 0 ? 4 : 2;
  }
  ldl_finish_kernel<<<(unsigned)std::max<int64_t>(1, (n + 255) / 256), 256,
                      n <= LDL_FINISH_SMEM_MAX ? (size_t)n * 8 : 0, s>>>(o.swaps, dblk, n, g0, perm,
                                                                        o.perm_global, c->ell, c->diag, 0);
  const unsigned ntri = (unsigned)(nt * (nt + 1) / 2);
  pack_unit_lower_kernel<<<ntri, 256, 0, s>>>(o.dense, ld, n, blk, nt);
  pack_upper_t_kernel<<<ntri, 256, 0, s>>>(o.dense, ld, n, umap, nt);
  tile_inv_unit_kernel<<<nt, T, T * 129 * 8, s>>>(blk, inv, 0);
  tile_inv_lower_kernel<<<nt, T, T * 129 * 8, s>>>(umap, inv2);
  c->launches += 7;
  return B2D_OK;
}

static int ooc_lu_factor(Ctx* c, int sa, int su, int k) {
  Ooc& o = c->o;
  cudaStream_t s = c->s_main;
  cudaStreamWaitEvent(s, o.ev_loaded[sa], 0);
  cudaStreamWaitEvent(s, o.ev_used[su], 0);
  cudaStreamWaitEvent(s, o.ev_stored[su], 0);
  const int rc = lu_factor_block(c, o.map(sa), o.map(su), k, s);
  cudaEventRecord(o.ev_used[sa], s);
  cudaEventRecord(o.ev_used[su], s);
  return rc;
}

// One visit of the reference's generic walk, stage k (memdet.py:97-121): rows bottom-up, the
// column direction alternating so one of B / C is reused between consecutive visits.
struct GVisit {
  int i, j;
  bool new_row, load_b, solve_b, write_b, next_diag;
};

static std::vector<GVisit> generic_visits(int nb, int k) {
  std::vector<GVisit> v;
  const int t = nb - 1 - k;
  for (int i = nb - 1; i > k; --i) {
    const bool asc = (i - k) % 2 == 0;
    const int first = asc ? k + 1 : nb - 1, last = asc ? nb - 1 : k + 1;
    for (int step = 0; step < nb - 1 - k; ++step) {
      const int j = asc ? k + 1 + step : nb - 1 - step;
      const bool bottom = i == nb - 1;
      v.push_back(GVisit{i, j, j == first, bottom || j != first, bottom, bottom && (t > 2 || j != last),
                         i == k + 1 && j == k + 1});
    }
  }
  return v;
}

// Slot x (engine block of `rows` x `cols` blocks) replaced by its transpose, through the
// permute temp slot (pointer swap, as ooc_permute).
static void ooc_transpose(Ctx* c, int x, int rows, int cols) {
  Ooc& o = c->o;
  const int tmp = o.nslot - 1;
  transpose_block_kernel<<<(unsigned)(o.tiles(rows) * o.tiles(cols)), 256, TRANSPOSE_SMEM, o.s_work>>>(
      o.map(x), o.map(tmp), o.tiles(rows), o.tiles(cols));
  c->launches++;
  std::swap(o.slot[x], o.slot[tmp]);
  cudaEventRecord(o.ev_used[x], o.s_work);  // the store of slot x must follow the transpose
}

// Generic Schur update of slot st (block (i, j)) -= X_i Y_j: X_i in slot sx (rows of i, the
// column block solved against U), Y_j^T in slot sy (rows of j, the row block solved with L).
static void ooc_schur_full(Ctx* c, int st, int i, int j, int sx, int sy, int k) {
  Ooc& o = c->o;
  for (int x : {st, sx, sy}) cudaStreamWaitEvent(o.s_work, o.ev_loaded[x], 0);
  GemmTask t{};
  t.a = o.map(sx);
  t.b = o.map(sy);
  t.c = o.map(st);
  t.out = TileSet{0, o.tiles(i), 0, o.tiles(j), 0, 0};
  t.p0 = 0;
  t.p1 = o.tiles(k);
  const double K = (double)t.p1 * T;
  launch_gemm(c, o.s_work, MODE_UPDATE, t, true, (double)t.out.count() * 2.0 * T * T * K);
  cudaEventRecord(o.ev_used[st], o.s_work);
  cudaEventRecord(o.ev_used[sx], o.s_work);
  cudaEventRecord(o.ev_used[sy], o.s_work);
}

// Panel block in slot x (engine rows of block `rows`): columns permuted by the stage's block
// permutation into the temp slot, which then takes slot x's place (memdet.py:365-366, 378-379).
static void ooc_permute(Ctx* c, int x, int rows, int k) {
  Ooc& o = c->o;
  const int tmp = o.nslot - 1;
  cudaStreamWaitEvent(o.s_work, o.ev_loaded[x], 0);
  permute_cols_kernel<<<2048, 256, 0, o.s_work>>>(o.map(x), o.map(tmp), o.tiles(rows), o.tiles(k), o.size(k),
                                                   o.perm_of(k));
  c->launches++;
  std::swap(o.slot[x], o.slot[tmp]);
}

// dst = src * D^{-1} over the stage's columns (memdet.py:368-371: B /= d, the unscaled copy kept).
static void ooc_scale(Ctx* c, int src, int dst, int rows, int k) {
  Ooc& o = c->o;
  cudaStreamWaitEvent(o.s_work, o.ev_stored[dst], 0);
  scale_cols_kernel<<<2048, 256, 0, o.s_work>>>(o.map(src), o.map(dst), o.tiles(rows), o.tiles(k), o.size(k),
                                                 o.dblk_of(k));
  c->launches++;
  cudaEventRecord(o.ev_used[src], o.s_work);
  cudaEventRecord(o.ev_used[dst], o.s_work);
}

// The reference driver (memdet.py:322-389) with HBM slots for its A/B/C/S buffers: every read
// and scratch write the reference performs happens here too (so the transfer counters are the
// reference's), issued on copy streams that run ahead of the DMMA work by the spare slots.
static int run_ooc(Ctx* c, const void* a, int64_t lda, int dtype, cudaStream_t user) {
  Ooc& o = c->o;
  CUDA_TRY(cudaSetDevice(c->device));
  begin(c, user);
  cudaStreamWaitEvent(o.s_h2d, c->ev_start, 0);
  cudaStreamWaitEvent(o.s_d2h, c->ev_start, 0);
  o.written.clear();
  o.reads = o.writes = 0;
  o.rr = 0;
  // pivoted LDL: factors on s_main (high priority), the walk's solves / updates on s_mid
  const bool look = c->mode == B2D_MODE_LDL_PIV && getenv("B2D_LDL_NO_LOOKAHEAD") == nullptr;
  // Cholesky: the same look-ahead with the walk on its own stream (the diagonal factor is the
  // in-core multi-stream driver on s_main / s_mid / s_side); B2D_OOC_NO_LOOKAHEAD disables it
  const bool clook = c->mode != B2D_MODE_LDL_PIV && c->mode != B2D_MODE_LU && o.s_walk && o.inv_odd &&
                     getenv("B2D_OOC_NO_LOOKAHEAD") == nullptr;
  o.s_work = look ? c->s_mid : clook ? o.s_walk : c->s_main;
  auto alloc = [&](std::initializer_list<int> busy) {
    const int pool = c->mode == B2D_MODE_LDL_PIV || c->mode == B2D_MODE_LU ? o.nslot - 1 : o.nslot;  // last: permute temp
    for (int tries = 0; tries < pool; ++tries) {
      const int s = o.rr;
      o.rr = (o.rr + 1) % pool;
      bool ok = true;
      for (int x : busy) ok = ok && x != s;
      if (ok) return s;
    }
    return -1;
  };
  const bool piv = c->mode == B2D_MODE_LDL_PIV;
  int rc = 0;
  if (c->mode == B2D_MODE_LU) {
    // the reference's generic walk (memdet.py:268-319); blocks (i, k), (i, j), (k, k) are held
    // as themselves, row-k blocks (k, j) transposed so that T -= X_i Y_j is the engine's
    // C -= A B^T
    int sa = alloc({});
    if ((rc = ooc_load(c, 0, 0, sa, a, lda, dtype, false))) return rc;
    for (int k = 0; k < o.nb; ++k) {
      const int su = alloc({sa});
      if ((rc = ooc_lu_factor(c, sa, su, k))) return rc;
      if (k == o.nb - 1) break;
      int sx = -1, sy = -1, next_a = -1;
      for (const GVisit& v : generic_visits(o.nb, k)) {
        if (v.new_row) {
          sx = alloc({sa, su, sy, sx});
          if ((rc = ooc_load(c, v.i, k, sx, a, lda, dtype, false))) return rc;
          ooc_trsm(c, sx, v.i, su, k, o.inv2);  // X_i = A(i, k) U^{-1}    (dense.py:102-106)
        }
        if (v.load_b) {
          sy = alloc({sa, su, sy, sx});
          if ((rc = ooc_load(c, k, v.j, sy, a, lda, dtype))) return rc;
          if (v.solve_b) {
            ooc_permute(c, sy, v.j, k);         // Y_j^T = (P A(k, j))^T L^{-T} (dense.py:94-99)
            ooc_trsm(c, sy, v.j, sa, k);
            if (v.write_b && (rc = ooc_store(c, k, v.j, sy))) return rc;
          }
        }
        const int st = alloc({sa, su, sx, sy});
        if ((rc = ooc_load(c, v.i, v.j, st, a, lda, dtype, false))) return rc;
        ooc_schur_full(c, st, v.i, v.j, sx, sy, k);  // dense.py:109-116, "ct_b"
        // (k+1, j > k+1) is next stage's row block: kept transposed, the form its solve uses
        if (v.i == k + 1 && v.j > k + 1) ooc_transpose(c, st, v.i, v.j);
        if (v.next_diag) next_a = st;
        else if ((rc = ooc_store(c, v.i, v.j, st))) return rc;
      }
      sa = next_a;
    }
    enqueue_prefix(c);
    cudaEventRecord(c->ev_join, o.s_d2h);
    cudaStreamWaitEvent(c->s_main, c->ev_join, 0);
    end(c, user);
    CUDA_TRY(cudaGetLastError());
    return B2D_OK;
  }
  int sa = alloc({});
  rc = ooc_load(c, 0, 0, sa, a, lda, dtype);
  if (rc) return rc;
  // pivoted LDL: factor the stage's diagonal block on s_main; s_work waits for it
  // B2D_LDL_TRACE: per-stage factor start / end and walk progress (timing events, printed here)
  const bool ltrace = piv && getenv("B2D_LDL_TRACE") != nullptr;
  std::vector<cudaEvent_t> tev;
  auto tmark = [&](cudaStream_t st) {
    if (!ltrace) return;
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, st);
    tev.push_back(e);
  };
  auto factor_ldl = [&](int slot, int k) -> int {
    if (o.s_work != c->s_main) {
      cudaEventRecord(o.ev_diag, o.s_work);  // the block's last Schur update
      cudaStreamWaitEvent(c->s_main, o.ev_diag, 0);
    }
    tmark(c->s_main);
    int r = ooc_ldl_factor(c, slot, k, c->s_main);
    tmark(c->s_main);
    cudaEventRecord(o.ev_fac, c->s_main);
    return r;
  };
  // Cholesky under look-ahead: the in-core driver on the block's tile grid, tile inverses in the
  // stage-parity buffer (the walk of stage k still reads stage k's while k+1 is factored)
  auto factor_chol = [&](int slot, int k) {
    cudaEventRecord(o.ev_diag, o.s_work);  // the block's last Schur update
    cudaStreamWaitEvent(c->s_main, o.ev_diag, 0);
    cudaStreamWaitEvent(c->s_main, o.ev_loaded[slot], 0);
    make_bounds(c, o.tiles(k), false);
    double* inv0 = c->inv;
    if (k & 1) c->inv = o.inv_odd;
    enqueue_factor(c, FactorTarget{o.map(slot), o.tiles(k), (int64_t)k * o.b}, false);
    c->inv = inv0;
    cudaEventRecord(o.ev_used[slot], c->s_main);
    cudaEventRecord(o.ev_fac, c->s_main);
  };
  if (piv && (rc = factor_ldl(sa, 0))) return rc;
  if (clook) factor_chol(sa, 0);
  for (int k = 0; k < o.nb; ++k) {
    if (piv || clook) {
      cudaStreamWaitEvent(o.s_work, o.ev_fac, 0);  // stage k's factor (issued ahead)
    } else {
      cudaStreamWaitEvent(c->s_main, o.ev_loaded[sa], 0);
      make_bounds(c, o.tiles(k), false);
      enqueue_factor(c, FactorTarget{o.map(sa), o.tiles(k), (int64_t)k * o.b}, false);
      cudaEventRecord(o.ev_used[sa], c->s_main);
    }
    if (k == o.nb - 1) break;
    const double* inv_k = (piv || clook) && (k & 1) && o.inv_odd ? o.inv_odd : c->inv;
    // bx: the column's solved row-k block (unscaled); by: its D^{-1}-scaled copy (LDL) or bx
    int bx = -1, by = -1, sc = -1, next_a = -1;
    bool early = false;  // look-ahead: block (k+1, k+1) updated and its factor issued
    for (const Visit& v : stage_visits(o.nb, k)) {
      if (early && v.next_diag) continue;  // done ahead (one update per stage: same result)
      if (v.col_start) {
        if (v.load_b) {
          bx = alloc({sa, bx, by, sc, next_a});
          if ((rc = ooc_load(c, k, v.j, bx, a, lda, dtype))) return rc;
          if (piv) ooc_permute(c, bx, v.j, k);
          ooc_trsm(c, bx, v.j, sa, k, inv_k);
        } else {
          bx = sc;  // the previous visit's C is this column's row-k block (memdet.py:359-360)
        }
        if (piv) {
          by = alloc({sa, bx, sc, next_a});
          ooc_scale(c, bx, by, v.j, k);
        } else {
          by = bx;
        }
      }
      if (v.load_c) {
        sc = alloc({sa, bx, by, sc, next_a});
        if ((rc = ooc_load(c, k, v.i, sc, a, lda, dtype))) return rc;
        if (v.solve_c) {
          if (piv) ooc_permute(c, sc, v.i, k);
          ooc_trsm(c, sc, v.i, sa, k, inv_k);
        }
        if (v.write_c && (rc = ooc_store(c, k, v.i, sc))) return rc;
      }
      const int st = alloc({sa, bx, by, sc, next_a});
      if ((rc = ooc_load(c, v.i, v.j, st, a, lda, dtype))) return rc;
      // T(j, i) -= [D^{-1}] L(j, k) * L(i, k)^T (the unscaled copy on the diagonal visit)
      ooc_schur(c, st, v.j, v.i, by, v.i == v.j ? bx : sc, k);
      if (v.next_diag) next_a = st;
      else if ((rc = ooc_store(c, v.i, v.j, st))) return rc;
      if (clook && !early && v.j == o.nb - 1 && v.i == k + 1 && v.i != v.j) {
        // as below, unscaled: T(k+1, k+1) -= L(k+1, k) L(k+1, k)^T, the diagonal visit's operands
        const int sd = alloc({sa, bx, by, sc});
        if ((rc = ooc_load(c, k + 1, k + 1, sd, a, lda, dtype))) return rc;
        ooc_schur(c, sd, k + 1, k + 1, sc, sc, k);
        next_a = sd;
        early = true;
        factor_chol(next_a, k + 1);
      }
      if (look && !early && v.j == o.nb - 1 && v.i == k + 1 && v.i != v.j) {
        // L(k+1, k) was just solved (slot sc): update block (k+1, k+1) now, the walk's last
        // visit, and factor it on s_main while the rest of the stage runs on s_work
        const int by2 = alloc({sa, bx, by, sc});
        ooc_scale(c, sc, by2, k + 1, k);
        const int sd = alloc({sa, bx, by, sc, by2});
        if ((rc = ooc_load(c, k + 1, k + 1, sd, a, lda, dtype))) return rc;
        ooc_schur(c, sd, k + 1, k + 1, by2, sc, k);
        next_a = sd;
        early = true;
        if ((rc = factor_ldl(next_a, k + 1))) return rc;
      }
    }
    if (piv && !early && (rc = factor_ldl(next_a, k + 1))) return rc;
    if (clook && !early) factor_chol(next_a, k + 1);
    tmark(o.s_work);  // end of stage k's walk
    sa = next_a;
  }
  if (ltrace) {
    cudaDeviceSynchronize();
    // events: f0s f0e, then per stage k < nb-1: f(k+1)s f(k+1)e walk_end(k)
    float ms = 0;
    for (size_t q = 1; q < tev.size(); ++q) {
      cudaEventElapsedTime(&ms, tev[0], tev[q]);
      fprintf(stderr, "[ldl trace] event %zu at %.2f ms\n", q, ms);
    }
    for (auto e : tev) cudaEventDestroy(e);
  }
  if (o.s_work != c->s_main) {
    cudaEventRecord(o.ev_work, o.s_work);
    cudaStreamWaitEvent(c->s_main, o.ev_work, 0);
  }
  enqueue_prefix(c);
  cudaEventRecord(c->ev_join, o.s_d2h);
  cudaStreamWaitEvent(c->s_main, c->ev_join, 0);
  end(c, user);
  CUDA_TRY(cudaGetLastError());
  return B2D_OK;
}

// Block-pivoted LDL^T in core (memdet_ldl; memdet.py:322-389, kernels/_ldl.pyx:21-61): the
// reference's stages over its b x b blocks with the matrix resident in the packed triangle.
// Stage k: the diagonal block is factored with block-local pivoting (s_main); the panel below
// it is permuted, solved and D^{-1}-scaled into the stage's panel grids (s_mid); block column
// k+1 is updated first (s_mid) so that the next factor starts at once, and the rest of the
// trailing triangle takes one large DMMA update (s_side) while it runs.  Every tile receives
// the walk's updates with the same operands and K, so the results equal the block walk's.
static int run_ldl_incore(Ctx* c, const void* a, int64_t lda, int dtype, bool host, cudaStream_t user) {
  if (dtype != B2D_F64 && dtype != B2D_F32) return set_err(B2D_ERR_USAGE, "dtype code %d", dtype);
  if (lda < c->m) return set_err(B2D_ERR_USAGE, "lda %lld < m", (long long)lda);
  Ooc& o = c->o;
  CUDA_TRY(cudaSetDevice(c->device));
  const int nt = c->nt, nb = o.nb;
  const int64_t npad = (int64_t)nt * T;
  if (host)
    for (int b = 0; b < NSTAGE; ++b)
      if (!c->strip[b]) CUDA_TRY(cudaMalloc(&c->strip[b], (size_t)T * npad * 8));
  begin(c, user);
  const int skip = host && nb > 1 ? o.tiles(0) : 0;
  if (host) {
    // the first diagonal block ahead of the strips (factor 0 starts on it alone): one b x b 2D
    // copy, packed strip by strip into its lower tiles
    if (skip > 0) {
      const int64_t ldb = (int64_t)o.nbt * T, b0 = o.size(0);
      const size_t esz = dtype == B2D_F64 ? 8 : 4;
      if (!c->bstage[0]) CUDA_TRY(cudaMalloc(&c->bstage[0], (size_t)ldb * ldb * 8));
      cudaStreamWaitEvent(c->s_copy, c->ev_start, 0);
      if (int rc = h2d_2d(c, c->bstage[0], (size_t)ldb * esz, a, (size_t)lda * esz, (size_t)b0 * esz, (size_t)b0,
                          c->s_copy))
        return rc;
      c->h2d += b0 * b0 * (int64_t)esz;
      cudaEventRecord(c->ev_copied[0], c->s_copy);
      cudaStreamWaitEvent(c->s_pack, c->ev_copied[0], 0);
      for (int J = 0; J < skip; ++J) {
        if (dtype == B2D_F64)
          pack_tiles_kernel<double, 8><<<(unsigned)(skip - J), PACK_THREADS, PACK_SMEM, c->s_pack>>>(
              (const double*)c->bstage[0], ldb, 0, c->m, c->tiles, nt, J);
        else
          pack_tiles_kernel<float, 8><<<(unsigned)(skip - J), PACK_THREADS, PACK_SMEM, c->s_pack>>>(
              (const float*)c->bstage[0], ldb, 0, c->m, c->tiles, nt, J);
        c->launches++;
      }
      cudaEventRecord(o.ev_fac, c->s_pack);
    }
    int rc = ingest_start(c, a, lda, dtype, skip);
    if (rc) return rc;
  } else {
    const unsigned ntiles = (unsigned)n_packed_tiles(nt);
    if (dtype == B2D_F64)
      pack_tiles_kernel<double, 32><<<ntiles, PACK_THREADS, PACK_SMEM, c->s_pack>>>((const double*)a, lda, 0, c->m,
                                                                                  c->tiles, nt, 0);
    else
      pack_tiles_kernel<float, 32><<<ntiles, PACK_THREADS, PACK_SMEM, c->s_pack>>>((const float*)a, lda, 0, c->m,
                                                                                 c->tiles, nt, 0);
    c->launches++;
    for (auto& e : c->ev_band) cudaEventRecord(e, c->s_pack);
  }
  auto wait_cols = [&](cudaStream_t st, int j1) -> int {  // tile-columns [0, j1) packed
    if (host)
      if (int e = ingest_upto(c, j1)) return e;  // pageable input: enqueued as needed
    const int b = std::min((int)c->ev_band.size(), (j1 + BAND - 1) / BAND) - 1;
    if (b >= 0) cudaStreamWaitEvent(st, c->ev_band[b], 0);
    return B2D_OK;
  };
  auto col0 = [&](int k) { return (int)((int64_t)k * o.b / T); };
  const TileMap packed{c->tiles, 0, nt};
  auto diag_map = [&](int k) {
    TileMap t = packed;
    t.roff = t.coff = col0(k);
    return t;
  };
  int rc = 0;
  // column streams (urgent schedule): block column q on s_cols[q % n]
  if (c->s_cols.empty()) {
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    const int ncs = std::max(1, std::min(16, env_int("B2D_LDL_COL_STREAMS", 8)));
    c->s_cols.resize(ncs);
    c->ev_cols.resize(ncs);
    for (int q = 0; q < ncs; ++q) {
      cudaStreamCreateWithPriority(&c->s_cols[q], cudaStreamNonBlocking, lo);
      cudaEventCreateWithFlags(&c->ev_cols[q], cudaEventDisableTiming);
    }
  }
  for (auto cs : c->s_cols) cudaStreamWaitEvent(cs, c->ev_start, 0);
  auto col_stream = [&](int q) { return c->s_cols[q % c->s_cols.size()]; };
  // `st` waits for everything enqueued so far on block column q's stream
  auto col_sync = [&](int q, cudaStream_t st) {
    const int i = q % (int)c->s_cols.size();
    cudaEventRecord(c->ev_cols[i], c->s_cols[i]);
    cudaStreamWaitEvent(st, c->ev_cols[i], 0);
  };
  // B2D_LDL_TRACE: timing events (name, stage) printed after the run
  const bool ltrace = getenv("B2D_LDL_TRACE") != nullptr;
  std::vector<std::pair<std::string, cudaEvent_t>> tev;
  auto tmark = [&](const char* what, int k, cudaStream_t st) {
    if (!ltrace) return;
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, st);
    tev.emplace_back(std::string(what) + " " + std::to_string(k), e);
  };
  // B2D_LDL_TL=<file>: per-launch globaltimer spans of the panel / bulk kernels (diagnostic)
  const char* tl_path = getenv("B2D_LDL_TL");
  unsigned long long* tl_buf = nullptr;
  const size_t tl_n = 4 * ((size_t)c->m / LDL_NB + 4);
  if (tl_path) {
    CUDA_TRY(cudaDeviceSynchronize());
    CUDA_TRY(cudaMalloc(&tl_buf, tl_n * 8));
    CUDA_TRY(cudaMemset(tl_buf, 0xff, tl_n * 8));
    CUDA_TRY(cudaMemcpyToSymbol(g_ldl_tl, &tl_buf, sizeof(tl_buf)));
  }
  tmark("start", 0, c->s_main);
  if (skip > 0) cudaStreamWaitEvent(c->s_main, o.ev_fac, 0);
  else if ((rc = wait_cols(c->s_main, col0(0) + o.tiles(0)))) return rc;
  const bool rows_sched = c->ldl_rows && !getenv("B2D_LDL_SCHED") &&
                          (getenv("B2D_LDL_URGENT") ? atoi(getenv("B2D_LDL_URGENT")) != 0 : true) &&
                          (getenv("B2D_LDL_SPLIT") ? atoi(getenv("B2D_LDL_SPLIT")) != 0 : true);
  // one set of factor outputs per stage (row schedule), selected until this function returns
  struct RingOff {
    Ooc& o;
    ~RingOff() { o.use_ring = false; }
  } ring_off{o};
  // B2D_LDL_GROUPS (tile-columns per group, default 4; 0 = off): the factors hand out their
  // finished column groups early (LdlGroups) -- stage 0's panel rows and trailing updates then run
  // beside factor 0, and every stage's chain row (block row k+1) is solved behind its factor
  const int grp_w = rows_sched && nb > 1 ? std::max(0, env_int("B2D_LDL_GROUPS", 4)) : 0;
  std::vector<int> grp_count((size_t)nb, 0);
  auto factor = [&](int k, bool overlapped) -> int {
    LdlGroups lg;
    lg.gw = grp_w;
    if (grp_w > 0) {
      if ((int)c->ev_grp.size() < nb) c->ev_grp.resize((size_t)nb);
      lg.ev = &c->ev_grp[(size_t)k];
    }
    const int e = ldl_factor_block(c, diag_map(k), k, c->s_main, overlapped, grp_w > 0 && k + 1 < nb ? &lg : nullptr);
    grp_count[(size_t)k] = lg.count;
    return e;
  };
  if (rows_sched && nb > 1) {
    if ((int)o.ring_inv.size() < nb) {
      for (int q = (int)o.ring_inv.size(); q < nb; ++q) {
        double *iv = nullptr, *db = nullptr;
        int64_t* pm = nullptr;
        CUDA_TRY(cudaMalloc(&iv, (size_t)o.nbt * TILE_BYTES));
        CUDA_TRY(cudaMalloc(&db, (size_t)o.nbt * T * 8));
        CUDA_TRY(cudaMalloc(&pm, (size_t)o.nbt * T * 8));
        o.ring_inv.push_back(iv);
        o.ring_dblk.push_back(db);
        o.ring_perm.push_back(pm);
      }
    }
    o.use_ring = true;
    if (!c->s_pr[0]) {
      int lo = 0, hi = 0;
      cudaDeviceGetStreamPriorityRange(&lo, &hi);
      // four row levels: priorities one below s_main's downwards (clamped to the range)
      for (int q = 0; q < 4; ++q) {
        const int pr = std::min(lo, hi + 1 + q);
        CUDA_TRY(cudaStreamCreateWithPriority(&c->s_pr[q], cudaStreamNonBlocking, pr));
      }
    }
    for (auto* v : {&c->ev_row, &c->ev_prow})
      while ((int)v->size() < std::max(nb, 2)) {
        cudaEvent_t e;
        CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        v->push_back(e);
      }
    // row r's last update so far: none (recorded before factor 0, which the rows wait for
    // themselves -- as a whole, or group by group)
    for (int r = 0; r < nb; ++r) cudaEventRecord(c->ev_row[r], c->s_main);
  }
  tmark("factor-begin", 0, c->s_main);
  if ((rc = factor(0, false))) return rc;
  tmark("factor-end", 0, c->s_main);
  cudaEventRecord(c->ev_catch[0], c->s_main);
  // Row-ordered schedule (c->ldl_rows, B2D_LDL_ROWS): stage k's work is issued block row by block
  // row r = k+1 .. nb-1 -- the panel rows of block r (permuted, solved, D^{-1}-scaled), then the
  // tiles (r, k+1 .. r) -- each row on a stream whose priority falls with its distance d = r - k
  // from the stage (d = 1, 2, 3, 4: s_pr[0..3]; farther rows one low-priority stream per row):
  // the factor of block r needs block row r complete, so the rows are needed in that order.  A
  // row's work is ordered across stages by its event (ev_row), a row's update waits for the panel
  // rows of the blocks before it (ev_prow); every tile receives its stages' updates in order with
  // the same operands and K: bit-identical to the column schedule and to the block walk.  The
  // factors' outputs (L_kk^{-1} tiles, block permutation, D) get one buffer per stage, and up to
  // MAX_PAN panel grids decouple the stages' far rows from the next stages' panels.  In the
  // column schedule (below) the nearest rows' updates could queue behind whole-column work.
  if (rows_sched && nb > 1) {
    for (auto st : c->s_pr) cudaStreamWaitEvent(st, c->ev_start, 0);
    auto bstart = [&](int q) { return std::min(nt, col0(q)); };
    auto bend = [&](int q) { return q + 1 < nb ? std::min(nt, col0(q + 1)) : nt; };
    // block row r at distance d = r - k: streams of falling priority, then one stream per row
    // B2D_LDL_NEXT_W: solve group width of block row k+1 (the chain factor k -> factor k+1)
    const int next_w = env_int("B2D_LDL_NEXT_W", 0);
    // B2D_LDL_LA: group width of the look-ahead solve of block row k+1 (0 = trsm_panel); 4
    // measured best (C2 432.6 -> 431.0 ms, C3 2837 -> 2831 ms; 2 and 8 no better)
    const int la_w = env_int("B2D_LDL_LA", 4);
    // B2D_LDL_PRMAP: 1 (default) = one priority level per distance 1 .. 4, farther rows on their
    // low-priority row streams; 0 = distances 1-2 share the first level (3, 4, 5 the next ones).
    // C2 419.9 -> 417.0 ms, C3 neutral; two coarser maps measured slower (421 ms)
    const int prmap = env_int("B2D_LDL_PRMAP", 1);
    auto dstream = [&](int r, int k) {
      const int d = r - k;
      if (prmap == 1) return d <= 4 ? c->s_pr[d - 1] : col_stream(r);
      return d <= 2 ? c->s_pr[0] : d <= 5 ? c->s_pr[d - 2] : col_stream(r);
    };
    // Group pipeline (grp_w > 0): block rows k+1 .. rlast of stage k solved and applied column
    // group by column group as factor k hands the groups out (group-major, so rows that share a
    // stream interleave): per group and row the permuted columns, the left-looking update by the
    // groups before (K = q0 T), the group's solves, the D^{-1} scaling; then the row's tiles
    // (r, k+1 .. r) take the K-chunk of the group (far rows: every front_ue groups).  Every entry
    // still receives its terms in increasing k through exact FP64 continuation across launches:
    // bit-identical to the whole-panel path.  Block row k+1 ends with the next factor's launch.
    const int front_ue = std::max(1, env_int("B2D_LDL_FRONT_UE", 4));
    // B2D_LDL_FRONT: stage 0 groups every block row (1) or only the chain row (0).  Default 1 for
    // device-resident input; 0 for host input -- there stage 0's far rows wait for their own
    // columns to arrive, and on the streams they share with the chain row those waits would hold
    // the chain's next group (C2 from pinned memory: 459 ms with, 443 ms without)
    const bool front_all = env_int("B2D_LDL_FRONT", host ? 0 : 1) != 0;
    const bool host_cols = env_int("B2D_LDL_HOST_COLS", 1) != 0;
    if (grp_w > 0 && !c->s_grpu) {
      int pr = 0;
      cudaStreamGetPriority(c->s_pr[0], &pr);
      CUDA_TRY(cudaStreamCreateWithPriority(&c->s_grpu, cudaStreamNonBlocking, pr));
      CUDA_TRY(cudaEventCreateWithFlags(&c->ev_grpu, cudaEventDisableTiming));
    }
    if (c->s_grpu) cudaStreamWaitEvent(c->s_grpu, c->ev_start, 0);
    while (grp_w > 0 && (int)c->ev_rowg.size() < nb) {
      cudaEvent_t e;
      CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      c->ev_rowg.push_back(e);
    }
    auto stage_rows_grouped = [&](int k, int rlast) -> int {
      const int k0 = col0(k), kb = o.tiles(k), i0 = k0 + kb;
      const double* inv_k = o.inv_of(k, c->inv);
      const int np = c->npan, pb = k % np;
      const int G = (kb + grp_w - 1) / grp_w;
      const TileMap lkk = diag_map(k);
      std::vector<int> pend((size_t)nb, 0);
      GemmTask u{};
      u.a = TileMap{c->pan[pb][1], o.nbt, 0};  // rows indexed by global tile row
      u.b = TileMap{c->pan[pb][0], o.nbt, 0};
      u.c = packed;
      for (int r = k + 1; r <= rlast; ++r) {
        cudaStream_t st = dstream(r, k);
        if (k >= np) cudaStreamWaitEvent(st, c->ev_rest[k - np], 0);
        if (int e = wait_cols(st, i0)) return e;
        cudaStreamWaitEvent(st, c->ev_row[r], 0);
        if (r == k + 1) tmark("p1-ready", k, st);
      }
      // solve of group [q0, qe) for block row r on st (permute, left-looking update, in-group solves)
      auto solve_group = [&](int r, cudaStream_t st, int q0, int qe, cudaEvent_t ready) {
        const int r0 = bstart(r), R = bend(r) - r0;
        cudaStreamWaitEvent(st, ready, 0);
        TileMap src = packed;
        src.roff = r0;
        src.coff = k0;
        const TileMap pu{c->pan[pb][0] + (size_t)r0 * o.nbt * TILE_ELEMS, o.nbt, 0};
        permute_cols_range_kernel<<<1024, 256, 0, st>>>(src, pu, R, (int64_t)q0 * T, qe - q0, o.size(k), o.perm_of(k));
        c->launches++;
        if (q0 > 0) {
          GemmTask w{};
          w.a = pu;
          w.b = lkk;
          w.c = pu;
          w.out = TileSet{0, R, q0, qe, 0, 0};
          w.p0 = 0;
          w.p1 = q0;
          launch_gemm(c, st, MODE_UPDATE, w, false, 0.0);
        }
        for (int q = q0; q < qe; ++q) {
          if (q > q0) {
            GemmTask w{};
            w.a = pu;
            w.b = lkk;
            w.c = pu;
            w.out = TileSet{0, R, q, q + 1, 0, 0};
            w.p0 = q0;
            w.p1 = q;
            launch_gemm(c, st, MODE_UPDATE, w, false, 0.0);
          }
          GemmTask t{};
          t.c = pu;
          t.binv = inv_k + (int64_t)q * TILE_ELEMS;
          t.out = TileSet{0, R, q, q + 1, 0, 0};
          t.k = q;
          launch_gemm(c, st, MODE_TRSM, t, false, 0.0);
        }
        cudaEventRecord(c->ev_rowg[r], st);  // the group's unscaled columns (what other rows read)
      };
      // D^{-1} scaling of the group, then tiles (r, k+1 .. r) take K = [pend, qe) on st
      auto scale_group = [&](int r, cudaStream_t st, int q0, int qe) {
        const int r0 = bstart(r), R = bend(r) - r0;
        TileMap su{c->pan[pb][0] + (size_t)r0 * o.nbt * TILE_ELEMS, o.nbt, 0};
        TileMap ss{c->pan[pb][1] + (size_t)r0 * o.nbt * TILE_ELEMS, o.nbt, 0};
        su.base += (int64_t)q0 * TILE_ELEMS;
        ss.base += (int64_t)q0 * TILE_ELEMS;
        const int64_t nrem = std::max<int64_t>(0, o.size(k) - (int64_t)q0 * T);
        scale_cols_kernel<<<1024, 256, 0, st>>>(su, ss, R, qe - q0, nrem, o.dblk_of(k) + (int64_t)q0 * T);
        c->launches++;
      };
      auto update_row = [&](int r, cudaStream_t st, int qe) -> int {
        const int r0 = bstart(r), r1 = bend(r);
        if (pend[(size_t)r] == 0)
          if (int e = wait_cols(st, r1)) return e;  // host input: the row's own columns are in
        u.out = TileSet{r0, r1, i0, r1, 1, 0};
        u.p0 = pend[(size_t)r];
        u.p1 = qe;
        launch_gemm(c, st, MODE_UPDATE, u, true, (double)u.out.count() * 2.0 * T * T * (double)(qe - pend[(size_t)r]) * T);
        pend[(size_t)r] = qe;
        return B2D_OK;
      };
      const int rc1 = k + 1;  // the chain row: its scaling and diagonal update on a side stream
      cudaStream_t sc1 = dstream(rc1, k);
      for (int g = 0; g < G; ++g) {
        const int q0 = g * grp_w, qe = std::min(kb, q0 + grp_w);
        cudaEvent_t ready = g < grp_count[(size_t)k] ? c->ev_grp[(size_t)k][(size_t)g] : c->ev_catch[k];
        const bool last = g == G - 1;
        solve_group(rc1, sc1, q0, qe, ready);
        cudaStreamWaitEvent(c->s_grpu, c->ev_rowg[rc1], 0);
        scale_group(rc1, c->s_grpu, q0, qe);
        if (int e = update_row(rc1, c->s_grpu, qe)) return e;
        if (last) {
          cudaEventRecord(c->ev_grpu, c->s_grpu);
          cudaStreamWaitEvent(sc1, c->ev_grpu, 0);
          cudaEventRecord(c->ev_prow[rc1], sc1);
          cudaEventRecord(c->ev_row[rc1], sc1);
          tmark("next-col-end", k, sc1);
          cudaEventRecord(o.ev_diag, sc1);
          cudaStreamWaitEvent(c->s_main, o.ev_diag, 0);
          tmark("factor-begin", k + 1, c->s_main);
          if (int e = factor(k + 1, k + 2 < nb)) return e;
          tmark("factor-end", k + 1, c->s_main);
          cudaEventRecord(c->ev_catch[k + 1], c->s_main);
        }
        for (int r = k + 2; r <= rlast; ++r) {
          cudaStream_t st = dstream(r, k);
          solve_group(r, st, q0, qe, ready);
          scale_group(r, st, q0, qe);
        }
        for (int r = k + 2; r <= rlast; ++r) {
          const int ue = r - k <= 2 ? 1 : front_ue;
          if (!last && (g + 1) % ue != 0) continue;
          cudaStream_t st = dstream(r, k);
          for (int q = k + 1; q < r; ++q)
            if (dstream(q, k) != st) cudaStreamWaitEvent(st, c->ev_rowg[q], 0);
          if (int e = update_row(r, st, qe)) return e;
          if (!last) continue;
          cudaEventRecord(c->ev_prow[r], st);
          cudaEventRecord(c->ev_row[r], st);
          if (r == k + 2) tmark("urgent-end", k, st);
        }
      }
      return B2D_OK;
    };
    for (int k = 0; k + 1 < nb; ++k) {
      const int k0 = col0(k), kb = o.tiles(k), i0 = k0 + kb;
      const double* inv_k = o.inv_of(k, c->inv);
      const int np = c->npan, pb = k % np;  // panel grids: stage k waits for the readers of stage k-np
      // grouped rows: all of stage 0's (nothing else runs beside factor 0), the chain row after
      // (a factor that handed nothing out early -- a big block, a single group -- keeps the whole-panel path)
      const int rgrp = grp_w > 0 && grp_count[(size_t)k] > 0 ? (k == 0 && front_all ? nb - 1 : k + 1) : k;
      if (rgrp > k)
        if ((rc = stage_rows_grouped(k, rgrp))) return rc;
      auto panel_rows = [&](cudaStream_t st, int r0, int r1, int wg) {  // global tile rows [r0, r1)
        TileMap src = packed;
        src.roff = r0;
        src.coff = k0;
        const TileMap pu{c->pan[pb][0] + (size_t)r0 * o.nbt * TILE_ELEMS, o.nbt, 0};
        const TileMap ps{c->pan[pb][1] + (size_t)r0 * o.nbt * TILE_ELEMS, o.nbt, 0};
        permute_cols_kernel<<<2048, 256, 0, st>>>(src, pu, r1 - r0, kb, o.size(k), o.perm_of(k));
        trsm_panel(c, st, pu, r1 - r0, diag_map(k), kb, inv_k, wg);
        scale_cols_kernel<<<2048, 256, 0, st>>>(pu, ps, r1 - r0, kb, o.size(k), o.dblk_of(k));
        c->launches += 2;
      };
      GemmTask u{};
      u.a = TileMap{c->pan[pb][1], o.nbt, 0};  // rows indexed by global tile row
      u.b = TileMap{c->pan[pb][0], o.nbt, 0};
      u.c = packed;
      u.p0 = 0;
      u.p1 = kb;
      const double K = (double)kb * T;
      for (int r = rgrp + 1; r < nb; ++r) {
        const int r0 = bstart(r), r1 = bend(r);
        cudaStream_t st = dstream(r, k);
        // the stage's factor, free panel grids, row r's previous update
        cudaStreamWaitEvent(st, c->ev_catch[k], 0);
        if (k >= np) cudaStreamWaitEvent(st, c->ev_rest[k - np], 0);
        if ((rc = wait_cols(st, i0))) return rc;
        cudaStreamWaitEvent(st, c->ev_row[r], 0);
        if (r == k + 1) tmark("p1-ready", k, st);
        u.out = TileSet{r0, r1, i0, r1, 1, 0};
        const bool la = r == k + 1 && la_w > 0;
        if (la) {
          // block row k+1 with its diagonal update folded into the look-ahead solve
          if ((rc = wait_cols(st, r1))) return rc;
          TileMap src = packed;
          src.roff = r0;
          src.coff = k0;
          const TileMap pu{c->pan[pb][0] + (size_t)r0 * o.nbt * TILE_ELEMS, o.nbt, 0};
          const TileMap ps{c->pan[pb][1] + (size_t)r0 * o.nbt * TILE_ELEMS, o.nbt, 0};
          permute_cols_kernel<<<2048, 256, 0, st>>>(src, pu, r1 - r0, kb, o.size(k), o.perm_of(k));
          c->launches++;
          if ((rc = trsm_panel_la(c, st, pu, ps, r1 - r0, diag_map(k), kb, inv_k, la_w, o.size(k), o.dblk_of(k), u)))
            return rc;
        } else
          panel_rows(st, r0, r1, r == k + 1 ? next_w : 0);
        cudaEventRecord(c->ev_prow[r], st);
        if (r == k + 1) tmark("panel-end", k, st);
        // tiles (r, k+1 .. r): the panel rows of every block up to r
        for (int q = k + 1; q < r; ++q)
          if (dstream(q, k) != st) cudaStreamWaitEvent(st, c->ev_prow[q], 0);
        // B2D_LDL_HOST_COLS (default 1): stage 0 from host memory -- a far row's tiles go block
        // column by block column, each as soon as that column's strips are in, instead of the
        // whole row after its last column (disjoint tiles, same operands and K: bit-identical)
        const bool by_cols = host && k == 0 && r > k + 1 && host_cols;
        if (!by_cols)
          if ((rc = wait_cols(st, r1))) return rc;
        if (r == k + 1) {
          if (!la) launch_gemm(c, st, MODE_UPDATE, u, true, (double)u.out.count() * 2.0 * T * T * K);
          cudaEventRecord(c->ev_row[r], st);
          tmark("next-col-end", k, st);
          cudaEventRecord(o.ev_diag, st);
          cudaStreamWaitEvent(c->s_main, o.ev_diag, 0);
          tmark("factor-begin", k + 1, c->s_main);
          if ((rc = factor(k + 1, k + 2 < nb))) return rc;
          tmark("factor-end", k + 1, c->s_main);
          cudaEventRecord(c->ev_catch[k + 1], c->s_main);
        } else {
          if (by_cols) {
            for (int q = k + 1; q <= r; ++q) {
              if ((rc = wait_cols(st, bend(q)))) return rc;
              GemmTask uq = u;
              uq.out = TileSet{r0, r1, bstart(q), bend(q), 1, 0};
              launch_update_kchunked(c, st, uq, 32);
            }
          } else
            launch_update_kchunked(c, st, u, 32);
          cudaEventRecord(c->ev_row[r], st);
          if (r == k + 2) tmark("urgent-end", k, st);
        }
      }
      // ev_rest[k]: every reader of stage k's panel buffers (panel k+np reuses them)
      for (int r = k + 1; r < nb; ++r) cudaStreamWaitEvent(c->s_side, c->ev_row[r], 0);
      cudaEventRecord(c->ev_rest[k], c->s_side);
      tmark("rest-end", k, c->s_side);
    }
    for (int r = 0; r < nb; ++r) cudaStreamWaitEvent(c->s_main, c->ev_row[r], 0);
    for (auto st : {c->s_pr[0], c->s_pr[1], c->s_pr[2], c->s_pr[3], c->s_side}) {
      cudaEventRecord(o.ev_work, st);
      cudaStreamWaitEvent(c->s_main, o.ev_work, 0);
    }
  } else
  for (int k = 0; k + 1 < nb; ++k) {
    const int par = k & 1;
    const int k0 = col0(k), kb = o.tiles(k), i0 = k0 + kb, kb1 = o.tiles(k + 1);
    const double* inv_k = par && o.inv_odd ? o.inv_odd : c->inv;
    // panel: rows [i0, nt) of block column k, permuted by the stage's pivots (memdet.py:365-366),
    // solved with the unit factor (dense.py:94-99), and its D^{-1}-scaled copy (memdet.py:368-371)
    cudaStreamWaitEvent(c->s_mid, c->ev_catch[k], 0);
    const int pb = k % 3;  // panel buffers: three, so panel k waits only for rest k-3
    if (k >= 3) cudaStreamWaitEvent(c->s_mid, c->ev_rest[k - 3], 0);  // last reader of pan[pb]
    if ((rc = wait_cols(c->s_mid, i0))) return rc;
    // B2D_LDL_SPLIT (default 1): the rows of block k+1 are solved and its diagonal block
    // updated first, so the next factor starts on them while the rows below are solved
    const char* spe = getenv("B2D_LDL_SPLIT");
    const int r_split = (spe ? atoi(spe) != 0 : true) ? i0 + kb1 : nt;
    auto panel_rows = [&](int r0, int r1, int wg) {  // global tile rows [r0, r1) of the panel
      TileMap src = packed;
      src.roff = r0;
      src.coff = k0;
      const TileMap pu{c->pan[pb][0] + (size_t)r0 * o.nbt * TILE_ELEMS, o.nbt, 0};
      const TileMap ps{c->pan[pb][1] + (size_t)r0 * o.nbt * TILE_ELEMS, o.nbt, 0};
      permute_cols_kernel<<<2048, 256, 0, c->s_mid>>>(src, pu, r1 - r0, kb, o.size(k), o.perm_of(k));
      trsm_panel(c, c->s_mid, pu, r1 - r0, diag_map(k), kb, inv_k, wg);
      scale_cols_kernel<<<2048, 256, 0, c->s_mid>>>(pu, ps, r1 - r0, kb, o.size(k), o.dblk_of(k));
      c->launches += 2;
    };
    // B2D_LDL_LA: block row k+1 by the look-ahead solve, its diagonal update folded in
    const int la_w = r_split == i0 + kb1 ? env_int("B2D_LDL_LA", 4) : 0;
    GemmTask u{};
    u.a = TileMap{c->pan[pb][1], o.nbt, 0};  // rows indexed by global tile row
    u.b = TileMap{c->pan[pb][0], o.nbt, 0};
    u.c = packed;
    u.p0 = 0;
    u.p1 = kb;
    const double K = (double)kb * T;
    if (la_w > 0) {
      if ((rc = wait_cols(c->s_mid, i0 + kb1))) return rc;
      TileMap src = packed;
      src.roff = i0;
      src.coff = k0;
      const TileMap pu{c->pan[pb][0] + (size_t)i0 * o.nbt * TILE_ELEMS, o.nbt, 0};
      const TileMap ps{c->pan[pb][1] + (size_t)i0 * o.nbt * TILE_ELEMS, o.nbt, 0};
      permute_cols_kernel<<<2048, 256, 0, c->s_mid>>>(src, pu, r_split - i0, kb, o.size(k), o.perm_of(k));
      c->launches++;
      u.out = TileSet{i0, r_split, i0, i0 + kb1, 1, 0};
      if ((rc = trsm_panel_la(c, c->s_mid, pu, ps, r_split - i0, diag_map(k), kb, inv_k, la_w, o.size(k),
                              o.dblk_of(k), u)))
        return rc;
    } else
      panel_rows(i0, r_split, env_int("B2D_LDL_NEXT_W", 0));
    tmark("panel-end", k, c->s_mid);
    // T -= (L D^{-1})_rows L_cols^T (dense.py:109-116) over block column k+1 first (its
    // diagonal block first of all)
    // B2D_LDL_URGENT (default 1): each stage's update of block column k+2 runs on s_mid right
    // after its panel (U_k below), so block column k+1 is current here by stream order; without
    // it, that update heads the trailing update on s_side and queues behind the previous stage's
    const char* ue = getenv("B2D_LDL_URGENT");
    const bool urgent = (ue ? atoi(ue) != 0 : true) && !getenv("B2D_LDL_SCHED");
    if (!urgent && k >= 1) cudaStreamWaitEvent(c->s_mid, c->ev_resta[k - 1], 0);  // block column k+1 current
    if ((rc = wait_cols(c->s_mid, i0 + kb1))) return rc;
    u.out = TileSet{i0, r_split, i0, i0 + kb1, 1, 0};
    if (la_w == 0) launch_gemm(c, c->s_mid, MODE_UPDATE, u, true, (double)u.out.count() * 2.0 * T * T * K);
    tmark("next-col-end", k, c->s_mid);
    cudaEventRecord(o.ev_diag, c->s_mid);
    cudaStreamWaitEvent(c->s_main, o.ev_diag, 0);
    tmark("factor-begin", k + 1, c->s_main);
    // B2D_LDL_SCHED: 0 (default) = the next factor beside the rest update; 1 = the factor alone
    // on the GPU, then the rest update beside the next panel solve (measured slower at C2)
    const char* se = getenv("B2D_LDL_SCHED");
    const bool serial = se ? atoi(se) != 0 : false;
    if ((rc = ldl_factor_block(c, diag_map(k + 1), k + 1, c->s_main, !serial && i0 + kb1 < nt))) return rc;
    tmark("factor-end", k + 1, c->s_main);
    cudaEventRecord(c->ev_catch[k + 1], c->s_main);
    if (r_split < nt) {  // the rows below block k+1: solve, then their block-column k+1 update
      panel_rows(r_split, nt, 0);
      if (urgent) col_sync(k + 1, c->s_mid);  // stage k-1's update of those rows (column stream)
      u.out = TileSet{r_split, nt, i0, i0 + kb1, 1, 0};
      launch_gemm(c, c->s_mid, MODE_UPDATE, u, true, (double)u.out.count() * 2.0 * T * T * K);
      tmark("below-end", k, c->s_mid);
    }
    cudaEventRecord(c->ev_panel[k], c->s_mid);
    if (i0 + kb1 < nt && urgent) {
      // U_k: the diagonal block of block column k+2 on s_mid (the factor after next needs it),
      // after every earlier update of that column; the rest of stage k's trailing update --
      // block column j on its own low-priority column stream, after the whole panel -- so a
      // column's stages are ordered on its stream and no column waits behind another's.
      const int i2 = k + 2 < nb ? std::min(nt, i0 + kb1 + o.tiles(k + 2)) : nt;
      if (k + 2 < nb) {
        col_sync(k + 2, c->s_mid);
        if ((rc = wait_cols(c->s_mid, i2))) return rc;
        u.out = TileSet{i0 + kb1, i2, i0 + kb1, i2, 1, 0};
        launch_update_kchunked(c, c->s_mid, u, 32);
      }
      tmark("urgent-end", k, c->s_mid);
      for (int q = k + 2, j0 = i0 + kb1; q < nb && j0 < nt; j0 += o.tiles(q), ++q) {
        const int j1 = std::min(nt, j0 + o.tiles(q));
        cudaStream_t cs = col_stream(q);
        cudaStreamWaitEvent(cs, c->ev_panel[k], 0);
        if ((rc = wait_cols(cs, j1))) return rc;
        // block column k+2: its rows below the diagonal block (the diagonal block went above)
        u.out = q == k + 2 ? TileSet{j1, nt, j0, j1, 0, 0} : TileSet{j0, nt, j0, j1, 1, 0};
        if (u.out.count() > 0) launch_update_kchunked(c, cs, u, 32);
      }
      // join stage k's readers of its panel buffers on s_side (ev_rest[k]: panel k+3 reuses them)
      for (int q = k + 2; q < nb; ++q) col_sync(q, c->s_side);
    } else if (i0 + kb1 < nt) {
      // after the whole panel (issued after the next factor, which takes its SMs first)
      cudaStreamWaitEvent(c->s_side, c->ev_panel[k], 0);
      if (serial) cudaStreamWaitEvent(c->s_side, c->ev_catch[k + 1], 0);
      // block column k+2 first (the next stage's next-col update waits for it alone), then the
      // rest: launches over disjoint tiles, each tile's operands and K unchanged.  Host input,
      // stage 0: the rest goes block column by block column, each as soon as its strips are in
      // (the matrix is still streaming in)
      const int i2 = k + 2 < nb ? std::min(nt, i0 + kb1 + o.tiles(k + 2)) : nt;
      const bool by_cols = host && k == 0;
      if ((rc = wait_cols(c->s_side, by_cols ? i2 : nt))) return rc;
      u.out = TileSet{i0 + kb1, nt, i0 + kb1, i2, 1, 0};
      launch_update_kchunked(c, c->s_side, u, 32);
      cudaEventRecord(c->ev_resta[k], c->s_side);
      if (by_cols) {
        for (int q = k + 3, j0 = i2; q < nb && j0 < nt; j0 += o.tiles(q), ++q) {
          const int j1 = std::min(nt, j0 + o.tiles(q));
          if ((rc = wait_cols(c->s_side, j1))) return rc;
          u.out = TileSet{j0, nt, j0, j1, 1, 0};
          launch_update_kchunked(c, c->s_side, u, 32);
        }
      } else if (i2 < nt) {
        u.out = TileSet{i2, nt, i2, nt, 1, 0};
        launch_update_kchunked(c, c->s_side, u, 32);
      }
    } else {
      cudaEventRecord(c->ev_resta[k], c->s_side);
    }
    tmark("rest-end", k, c->s_side);
    cudaEventRecord(c->ev_rest[k], c->s_side);
  }
  cudaEventRecord(o.ev_work, c->s_mid);
  cudaStreamWaitEvent(c->s_main, o.ev_work, 0);
  cudaEventRecord(o.ev_diag, c->s_side);
  cudaStreamWaitEvent(c->s_main, o.ev_diag, 0);
  for (int q = 0; q < (int)c->s_cols.size(); ++q) col_sync(q, c->s_main);
  cudaEventRecord(c->ev_join, c->s_pack);
  cudaStreamWaitEvent(c->s_main, c->ev_join, 0);
  enqueue_prefix(c);
  tmark("end", nb, c->s_main);
  end(c, user);
  if (ltrace) {
    cudaDeviceSynchronize();
    {
      int plo = 0, phi = 0, pm = 0, pd = 0, pf = 0;
      cudaDeviceGetStreamPriorityRange(&plo, &phi);
      if (c->s_pr[0]) cudaStreamGetPriority(c->s_pr[0], &pm);
      if (c->s_pr[1]) cudaStreamGetPriority(c->s_pr[1], &pd);
      if (c->s_pr[3]) cudaStreamGetPriority(c->s_pr[3], &pf);
      fprintf(stderr, "[ldl trace] priorities: range [%d, %d], d<=2 %d, d=3 %d, d=5 %d, npan %d\n", plo, phi, pm, pd, pf,
              c->npan);
    }
    for (size_t q = 1; q < tev.size(); ++q) {
      float ms = 0;
      cudaEventElapsedTime(&ms, tev[0].second, tev[q].second);
      fprintf(stderr, "[ldl trace] %-14s %8.2f ms\n", tev[q].first.c_str(), ms);
    }
    for (auto& e : tev) cudaEventDestroy(e.second);
  }
  if (tl_buf) {
    CUDA_TRY(cudaDeviceSynchronize());
    std::vector<unsigned long long> h(tl_n);
    CUDA_TRY(cudaMemcpy(h.data(), tl_buf, tl_n * 8, cudaMemcpyDeviceToHost));
    unsigned long long* null_buf = nullptr;
    CUDA_TRY(cudaMemcpyToSymbol(g_ldl_tl, &null_buf, sizeof(null_buf)));
    cudaFree(tl_buf);
    if (FILE* f = fopen(tl_path, "a")) {
      fprintf(f, "# run m=%lld b=%lld: row kind start_ns end_ns\n", (long long)c->m, (long long)o.b);
      for (size_t q = 0; 2 * q + 1 < tl_n; ++q)
        if (h[2 * q] != ~0ull)
          fprintf(f, "%lld %d %llu %llu\n", (long long)((q / 2) * LDL_NB), (int)(q & 1), h[2 * q], ~h[2 * q + 1]);
      fclose(f);
    }
  }
  CUDA_TRY(cudaGetLastError());
  return B2D_OK;
}

// float32 memdet_ldl in the reference's f32 arithmetic (memdet.py:322-412 on a float32 file;
// ldl32.cu, oracle/ldl32_model.c).  All on s_main, stage by stage: the diagonal block factored
// one pivot step at a time (the reference's unblocked loop), the row-k blocks gathered in pivot
// order, solved in STRSM's row blocks, scaled by D^{-1}, and every trailing block (i <= j) updated
// in SGEMM's K-block order.
static int run_ldl32(Ctx* c, const void* a, int64_t lda, int dtype, bool host, cudaStream_t user) {
  if (dtype != B2D_F32)
    return set_err(B2D_ERR_USAGE, "this context factors float32 inputs in f32 arithmetic (got dtype code %d)", dtype);
  if (lda < c->m) return set_err(B2D_ERR_USAGE, "lda %lld < m", (long long)lda);
  CUDA_TRY(cudaSetDevice(c->device));
  Ooc& o = c->o;
  Ctx::F32& f = c->f;
  const int64_t m = c->m, b = o.b;
  const int nb = o.nb;
  cudaStream_t s = c->s_main;
  begin(c, user);
  // the reference reads the (i <= j) blocks: block row i, columns [i * b, m)
  for (int bi = 0; bi < nb; ++bi) {
    const int64_t r0 = (int64_t)bi * b, rows = o.size(bi), cols = m - r0;
    float* dst = f.M + r0 * f.ldm + r0;
    const float* src = (const float*)a + r0 * lda + r0;
    if (host) {
      if (int rc = h2d_2d(c, dst, (size_t)f.ldm * 4, src, (size_t)lda * 4, (size_t)cols * 4, (size_t)rows, s)) return rc;
      c->h2d += rows * cols * 4;
    } else {
      CUDA_TRY(cudaMemcpy2DAsync(dst, (size_t)f.ldm * 4, src, (size_t)lda * 4, (size_t)cols * 4, (size_t)rows,
                                 cudaMemcpyDeviceToDevice, s));
    }
  }
  int kb[L32_MAXKB + 1];
  const int nkb = l32_kblocks(b, kb);
  for (int k = 0; k < nb; ++k) {
    const int64_t k0 = (int64_t)k * b, hk = o.size(k);
    cudaMemsetAsync(f.amax, 0, 8, s);
    const dim3 gb((unsigned)((hk + 31) / 32), (unsigned)((hk + 31) / 32));
    l32_block_in_kernel<float><<<gb, 256, 0, s>>>(f.M, f.ldm, k0, hk, f.dense, f.ldd, f.amax);
    const L32Step<float> g{f.dense, f.ldd, hk, k0, f.work, f.d + k0, o.swaps, c->fail, f.amax, -1.0};
    for (int64_t r = 0; r < hk; ++r) {
      l32_step_kernel<float><<<1, 1024, 0, s>>>(g, r);
      if (r + 1 < hk) l32_update_kernel<float><<<(unsigned)(hk - r - 1), 256, 0, s>>>(g, r);
    }
    l32_finish_kernel<float><<<(unsigned)std::max<int64_t>(1, std::min<int64_t>(64, (hk + 255) / 256)), 256, 0, s>>>(
        o.swaps, f.d + k0, hk, k0, o.perm_local, o.perm_global, c->ell, c->diag, c->fail);
    c->launches += 3 + 2 * hk - 1;
    if (k == nb - 1) break;
    const int64_t c0 = k0 + b, W = m - c0;
    // row-k blocks in pivot order (memdet.py:365-366, 378-379), solved (dense.py:94-99)
    l32_gather_kernel<float><<<dim3((unsigned)std::min<int64_t>(64, (W + 255) / 256), (unsigned)std::min<int64_t>(b, 65535)),
                        256, 0, s>>>(f.M, f.ldm, k0, c0, o.perm_local, b, W, f.X, f.ldx);
    for (int64_t ls = 0; ls < b; ls += L32_Q) {
      const int64_t le = std::min<int64_t>(b, ls + L32_Q);
      l32_trsm_diag_kernel<float><<<(unsigned)((W + TrsmTW<float>::v - 1) / TrsmTW<float>::v), 256,
                                    l32_trsm_smem<float>(), s>>>(f.dense, f.ldd, f.X, f.ldx, W, ls, le, 1, c->fail);
      c->launches++;
      if (le < b) {  // rows below the row block: X -= L(le:, ls:le) X(ls:le, :), one chain each
        G32 u{};
        u.A = f.dense + ls * f.ldd + le;
        u.lda = f.ldd;
        u.B = f.X + ls * f.ldx;
        u.ldb = f.ldx;
        u.C = f.X + le * f.ldx;
        u.ldc = f.ldx;
        u.Mr = b - le;
        u.Nc = W;
        u.nkb = 1;
        u.kb[0] = 0;
        u.kb[1] = (int)(le - ls);
        u.blk = 1;
        l32_gemm_kernel<float><<<dim3((unsigned)((W + G32_BN - 1) / G32_BN), (unsigned)((b - le + G32_BM - 1) / G32_BM)),
                                 256, 0, s>>>(u, c->fail);
        c->launches++;
      }
    }
    // S = X / d (memdet.py:368-371); T(i, j) -= X_i^T S_j for every trailing block i <= j (memdet.py:385)
    l32_scale_kernel<float><<<dim3((unsigned)std::min<int64_t>(64, (W + 255) / 256), (unsigned)std::min<int64_t>(b, 65535)), 256, 0,
                       s>>>(f.X, f.S, f.ldx, b, W, f.d + k0);
    G32 u{};
    u.A = f.X;
    u.lda = f.ldx;
    u.B = f.S;
    u.ldb = f.ldx;
    u.C = f.M + c0 * f.ldm + c0;
    u.ldc = f.ldm;
    u.Mr = W;
    u.Nc = W;
    u.nkb = nkb;
    for (int q = 0; q <= nkb; ++q) u.kb[q] = kb[q];
    u.tri = 1;
    u.blk = b;
    u.roff = u.coff = c0;
    l32_gemm_kernel<float><<<dim3((unsigned)((W + G32_BN - 1) / G32_BN), (unsigned)((W + G32_BM - 1) / G32_BM)), 256, 0,
                             s>>>(u, c->fail);
    c->launches += 4;
  }
  enqueue_prefix(c);
  end(c, user);
  CUDA_TRY(cudaGetLastError());
  return B2D_OK;
}

// Generic LU in core (memdet_lu; memdet.py:268-319, kernels/dense.py:38-54, 94-106): the
// reference's stages over its b x b blocks with the matrix resident as a full tile grid.  Stage
// k: the diagonal block is factored P A = L U with block-local partial pivoting (s_main; L back
// into the grid's diagonal block, U^T into a block grid); the column panel X = A(i, k) U^{-1}
// and the transposed, permuted row panel Y^T = (P A(k, j))^T L^{-T} are formed in full-height
// panel grids (s_mid); block column and block row k+1 are updated first so the next factor
// starts at once, and the rest of the trailing square takes one DMMA update T -= X Y (s_side)
// beside it.  The same kernels, operands and K per tile as the generic block walk.
static int run_lu_incore(Ctx* c, const void* a, int64_t lda, int dtype, bool host, cudaStream_t user) {
  if (dtype != B2D_F64 && dtype != B2D_F32) return set_err(B2D_ERR_USAGE, "dtype code %d", dtype);
  if (lda < c->m) return set_err(B2D_ERR_USAGE, "lda %lld < m", (long long)lda);
  Ooc& o = c->o;
  CUDA_TRY(cudaSetDevice(c->device));
  const int nt = c->nt, nb = o.nb;
  const size_t esz = dtype == B2D_F64 ? 8 : 4;
  const TileMap full{c->grid, nt, 0};
  begin(c, user);
  // ingest, reference block by block in the stages' cross order -- (k, k), block row k, block
  // column k -- so that stage k starts once its blocks are in: ev_cross[k] after the last of
  // them; ev_diag_in = block (0, 0) (the first factor starts on it alone).  Host blocks go
  // through two staging buffers (2D copies of b x b, then pack_block_nt per 128-row strip).
  auto col0 = [&](int k) { return (int)((int64_t)k * o.b / T); };
  const int64_t ldb = (int64_t)o.nbt * T;
  if (host) {
    for (auto*& q : c->bstage)
      if (!q) CUDA_TRY(cudaMalloc(&q, (size_t)ldb * ldb * 8));
  }
  if ((int)c->ev_cross.size() < nb) {
    while ((int)c->ev_cross.size() < nb) {
      cudaEvent_t e;
      cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
      c->ev_cross.push_back(e);
    }
    while (c->ev_bstage.size() < 2) {
      cudaEvent_t e;
      cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
      c->ev_bstage.push_back(e);
    }
  }
  int nblk = 0;
  auto ingest = [&](int I, int J) -> int {
    const int64_t rows = o.size(I), cols = o.size(J);
    const TileMap dst{c->grid + ((size_t)col0(I) * nt + col0(J)) * TILE_ELEMS, nt, 0};
    const char* src;
    int64_t sld;
    if (host) {
      const int sb = nblk & 1;
      if (nblk >= 2) cudaStreamWaitEvent(c->s_copy, c->ev_bstage[sb], 0);
      if (int rc = h2d_2d(c, c->bstage[sb], (size_t)ldb * esz,
                          (const char*)a + ((size_t)I * o.b * lda + (size_t)J * o.b) * esz, (size_t)lda * esz,
                          (size_t)cols * esz, (size_t)rows, c->s_copy))
        return rc;
      cudaEventRecord(c->ev_copied[sb], c->s_copy);
      cudaStreamWaitEvent(c->s_pack, c->ev_copied[sb], 0);
      c->h2d += rows * cols * (int64_t)esz;
      src = (const char*)c->bstage[sb];
      sld = ldb;
    } else {
      src = (const char*)a + ((size_t)I * o.b * lda + (size_t)J * o.b) * esz;
      sld = lda;
    }
    for (int r = 0; r < o.tiles(I); ++r) {
      const char* sr = src + (size_t)r * T * sld * esz;
      if (dtype == B2D_F64)
        pack_block_nt_kernel<double><<<o.tiles(J), 256, 0, c->s_pack>>>((const double*)sr, sld, rows, cols, I == J,
                                                                         dst, r);
      else
        pack_block_nt_kernel<float><<<o.tiles(J), 256, 0, c->s_pack>>>((const float*)sr, sld, rows, cols, I == J,
                                                                        dst, r);
      c->launches++;
    }
    if (host) cudaEventRecord(c->ev_bstage[nblk & 1], c->s_pack);
    ++nblk;
    return B2D_OK;
  };
  int rc = 0;
  // host input: cross sets enqueued up to `upto` (pinned: all at once; pageable: as the stages
  // need them, since the staging callbacks would otherwise block this thread before the first
  // factor is queued)
  int crosses = 0;
  auto ingest_crosses = [&](int upto) -> int {
    for (int k = crosses; k < std::min(upto, nb); ++k) {
      int r;
      if ((r = ingest(k, k))) return r;
      if (k == 0) cudaEventRecord(o.ev_fac, c->s_pack);  // block (0, 0)
      for (int j = k + 1; j < nb; ++j)
        if ((r = ingest(k, j))) return r;
      for (int i = k + 1; i < nb; ++i)
        if ((r = ingest(i, k))) return r;
      cudaEventRecord(c->ev_cross[k], c->s_pack);
      crosses = k + 1;
    }
    return B2D_OK;
  };
  if (host) {
    if ((rc = ingest_crosses(getenv("B2D_LU_ALL_CROSSES") ? nb : 2))) return rc;
  } else {  // resident: one pack launch per 128-row strip
    for (int J = 0; J < nt; ++J) {
      const char* sr = (const char*)a + (size_t)J * T * lda * esz;
      if (dtype == B2D_F64)
        pack_block_nt_kernel<double><<<nt, 256, 0, c->s_pack>>>((const double*)sr, lda, c->m, c->m, 1, full, J);
      else
        pack_block_nt_kernel<float><<<nt, 256, 0, c->s_pack>>>((const float*)sr, lda, c->m, c->m, 1, full, J);
      c->launches++;
    }
    cudaEventRecord(o.ev_fac, c->s_pack);
    for (int k = 0; k < nb; ++k) cudaEventRecord(c->ev_cross[k], c->s_pack);
  }
  auto blk = [&](int k) { return TileMap{c->grid + ((size_t)col0(k) * nt + col0(k)) * TILE_ELEMS, nt, 0}; };
  auto umap = [&](int k) { return TileMap{c->ublk[k & 1], o.nbt, 0}; };
  cudaStreamWaitEvent(c->s_main, o.ev_fac, 0);
  if ((rc = lu_factor_block(c, blk(0), umap(0), 0, c->s_main))) return rc;
  cudaEventRecord(c->ev_catch[0], c->s_main);
  for (int k = 0; k + 1 < nb; ++k) {
    const int par = k & 1;
    const int k0 = col0(k), kb = o.tiles(k), i0 = k0 + kb, R = nt - i0, kb1 = o.tiles(k + 1);
    const double* inv_l = par && o.inv_odd ? o.inv_odd : c->inv;
    const double* inv_u = par && o.inv2_odd ? o.inv2_odd : o.inv2;
    cudaStreamWaitEvent(c->s_mid, c->ev_catch[k], 0);
    if (k >= 2) cudaStreamWaitEvent(c->s_mid, c->ev_rest[k - 2], 0);  // last reader of lpan[par]
    cudaStreamWaitEvent(c->s_mid, c->ev_cross[k], 0);                 // block row / column k in
    const size_t poff = (size_t)i0 * o.nbt * TILE_ELEMS;
    const TileMap X{c->lpan[par][0] + poff, o.nbt, 0}, Yt{c->lpan[par][1] + poff, o.nbt, 0},
        Tt{c->lpan[par][2] + poff, o.nbt, 0};
    // X = A(i, k) U^{-1} (dense.py:102-106): tile rows [i0, nt) of block column k
    CUDA_TRY(cudaMemcpy2DAsync(c->lpan[par][0] + poff, (size_t)o.nbt * TILE_BYTES,
                               c->grid + ((size_t)i0 * nt + k0) * TILE_ELEMS, (size_t)nt * TILE_BYTES,
                               (size_t)kb * TILE_BYTES, (size_t)R, cudaMemcpyDeviceToDevice, c->s_mid));
    trsm_panel(c, c->s_mid, X, R, umap(k), kb, inv_u);
    // Y^T = (P A(k, j))^T L^{-T} (dense.py:94-99, memdet.py:365-366): block row k transposed,
    // its (block-local) rows permuted, solved with the unit L
    transpose_block_kernel<<<(unsigned)(kb * R), 256, TRANSPOSE_SMEM, c->s_mid>>>(
        TileMap{c->grid + ((size_t)k0 * nt + i0) * TILE_ELEMS, nt, 0}, Tt, kb, R);
    permute_cols_kernel<<<2048, 256, 0, c->s_mid>>>(Tt, Yt, R, kb, o.size(k), o.perm_of(k));
    trsm_panel(c, c->s_mid, Yt, R, blk(k), kb, inv_l);
    c->launches += 2;
    cudaEventRecord(c->ev_panel[k], c->s_mid);
    // T(i, j) -= X_i Y_j (dense.py:109-116, "ct_b"): block column and block row k+1 first
    GemmTask u{};
    u.a = TileMap{c->lpan[par][0], o.nbt, 0};  // rows indexed by global tile row
    u.b = TileMap{c->lpan[par][1], o.nbt, 0};  // rows indexed by global tile column
    u.c = full;
    u.p0 = 0;
    u.p1 = kb;
    const double K = (double)kb * T;
    if (k >= 1) cudaStreamWaitEvent(c->s_mid, c->ev_resta[k - 1], 0);  // cross k+1 current
    if (host && (rc = ingest_crosses(k + 2))) return rc;
    cudaStreamWaitEvent(c->s_mid, c->ev_cross[k + 1], 0);
    u.out = TileSet{i0, nt, i0, i0 + kb1, 0, 0};
    launch_gemm(c, c->s_mid, MODE_UPDATE, u, true, (double)u.out.count() * 2.0 * T * T * K);
    if (i0 + kb1 < nt) {
      u.out = TileSet{i0, i0 + kb1, i0 + kb1, nt, 0, 0};
      launch_gemm(c, c->s_mid, MODE_UPDATE, u, true, (double)u.out.count() * 2.0 * T * T * K);
    }
    cudaEventRecord(o.ev_diag, c->s_mid);
    cudaStreamWaitEvent(c->s_main, o.ev_diag, 0);
    if ((rc = lu_factor_block(c, blk(k + 1), umap(k + 1), k + 1, c->s_main))) return rc;
    cudaEventRecord(c->ev_catch[k + 1], c->s_main);
    if (i0 + kb1 < nt) {
      cudaStreamWaitEvent(c->s_side, o.ev_diag, 0);
      if (k > 0 || !host) {
        if (host && (rc = ingest_crosses(nb))) return rc;
        cudaStreamWaitEvent(c->s_side, c->ev_cross[nb - 1], 0);
        // block column and block row k+2 first (the next stage's cross update waits for them
        // alone), then the rest of the square: disjoint tiles, operands and K unchanged
        const int i2 = k + 2 < nb ? std::min(nt, i0 + kb1 + o.tiles(k + 2)) : nt;
        u.out = TileSet{i0 + kb1, nt, i0 + kb1, i2, 0, 0};
        launch_update_kchunked(c, c->s_side, u);
        if (i2 < nt) {
          u.out = TileSet{i0 + kb1, i2, i2, nt, 0, 0};
          launch_update_kchunked(c, c->s_side, u);
        }
        cudaEventRecord(c->ev_resta[k], c->s_side);
        if (i2 < nt) {
          u.out = TileSet{i2, nt, i2, nt, 0, 0};
          launch_update_kchunked(c, c->s_side, u);
        }
      } else {
        // stage 0 runs while the matrix streams in: the rest of the trailing square in the
        // cross sets of the later stages (block (s, s), row s, column s), each as it arrives
        for (int st = 2; st < nb; ++st) {
          const int s0 = col0(st), s1 = s0 + o.tiles(st);
          if ((rc = ingest_crosses(st + 1))) return rc;
          cudaStreamWaitEvent(c->s_side, c->ev_cross[st], 0);
          u.out = TileSet{s0, s1, s0, nt, 0, 0};
          launch_gemm(c, c->s_side, MODE_UPDATE, u, true, (double)u.out.count() * 2.0 * T * T * K);
          if (s1 < nt) {
            u.out = TileSet{s1, nt, s0, s1, 0, 0};
            launch_gemm(c, c->s_side, MODE_UPDATE, u, true, (double)u.out.count() * 2.0 * T * T * K);
          }
        }
      }
    }
    cudaEventRecord(c->ev_rest[k], c->s_side);
    if (!(i0 + kb1 < nt && (k > 0 || !host))) cudaEventRecord(c->ev_resta[k], c->s_side);
  }
  cudaEventRecord(o.ev_work, c->s_mid);
  cudaStreamWaitEvent(c->s_main, o.ev_work, 0);
  cudaEventRecord(o.ev_diag, c->s_side);
  cudaStreamWaitEvent(c->s_main, o.ev_diag, 0);
  cudaEventRecord(c->ev_join, c->s_pack);
  cudaStreamWaitEvent(c->s_main, c->ev_join, 0);
  enqueue_prefix(c);
  end(c, user);
  CUDA_TRY(cudaGetLastError());
  return B2D_OK;
}

static int fetch(Ctx* c, double* d_out, double* prefix_out, int64_t* fail_index, b2d_run_info* info) {
  if (c->mg) return mg_fetch(c->mg, d_out, prefix_out, fail_index, info);
  if (!c->pending) return set_err(B2D_ERR_USAGE, "no factorisation enqueued");
  CUDA_TRY(cudaSetDevice(c->device));
  CUDA_TRY(cudaEventSynchronize(c->ev_stop));
  c->pending = false;
  CUDA_TRY(cudaGetLastError());
  unsigned long long fail = ULLONG_MAX;
  CUDA_TRY(cudaMemcpy(&fail, c->fail, 8, cudaMemcpyDeviceToHost));
  float ms = 0.f;
  cudaEventElapsedTime(&ms, c->ev_start, c->ev_stop);
  if (prefix_out) {
    CUDA_TRY(cudaMemcpy(prefix_out, c->prefix, c->m * 8, cudaMemcpyDeviceToHost));
    c->d2h += c->m * 8;
  }
  if (d_out) {
    CUDA_TRY(cudaMemcpy(d_out, c->diag, c->m * 8, cudaMemcpyDeviceToHost));
    c->d2h += c->m * 8;
    if (c->mode == B2D_MODE_LDL_NOPIV)
      for (int64_t g = 0; g < c->m; ++g) d_out[g] = d_out[g] * d_out[g];
  }
  if (info) {
    info->m = c->m;
    info->tile = T;
    info->n_tiles = c->nt;
    info->h2d_bytes = c->h2d;
    info->d2h_bytes = c->d2h;
    info->kernel_launches = c->launches;
    info->device_ms = ms;
    info->ooc_blocks = c->ooc ? c->o.nb : 0;
    info->ooc_block = c->ooc ? c->o.b : 0;
    info->ooc_reads = c->ooc ? c->o.reads : 0;
    info->ooc_writes = c->ooc ? c->o.writes : 0;
    info->ooc_scratch = c->ooc ? (int64_t)c->o.written.size() : 0;
    info->wall_seconds =
        std::chrono::duration<double>(std::chrono::steady_clock::now() - c->t0).count();
  }
  if (c->trace) {
    const int nsteps = (int)c->ev_panel.size();
    auto at = [&](cudaEvent_t e) {
      float x = -1.f;
      if (cudaEventElapsedTime(&x, c->ev_start, e) != cudaSuccess) { cudaGetLastError(); x = -1.f; }
      return x;
    };
    fprintf(stderr, "[b2d trace] total %.2f ms\n", ms);
    for (size_t b = 0; b < c->ev_band.size(); ++b)
      fprintf(stderr, "[b2d trace] band %zu act %d arrived %.2f\n", b, c->act[b], at(c->ev_band[b]));
    for (int st = 0; st < nsteps; ++st)
      fprintf(stderr, "[b2d trace] step %d panel %.2f catch %.2f rest %.2f\n", st, at(c->ev_panel[st]),
              at(c->ev_catch[st]), at(c->ev_rest[st]));
  }
  if (fail_index) *fail_index = fail == ULLONG_MAX ? -1 : (int64_t)fail;
  if (c->mode == B2D_MODE_LU) return B2D_OK;  // a zero pivot means det = 0 (fail_index), not an error
  if (fail != ULLONG_MAX && c->mode == B2D_MODE_LDL_PIV)
    return set_err(B2D_ERR_INDEFINITE, "LDL pivot %lld below tolerance (block-local 1x1 pivoting)",
                   (long long)fail);
  if (fail != ULLONG_MAX)
    return set_err(B2D_ERR_NOT_SPD, "leading minor of order %lld is not positive definite",
                   (long long)fail + 1);
  return B2D_OK;
}

static int mg_fetch_perm(MCtx* M, int64_t* perm);
static int fetch_perm(Ctx* c, int64_t* perm) {
  if (!perm) return set_err(B2D_ERR_USAGE, "null perm");
  if (c->mg) return mg_fetch_perm(c->mg, perm);
  if ((c->mode == B2D_MODE_LDL_PIV || c->mode == B2D_MODE_LU) && c->o.perm_global) {
    CUDA_TRY(cudaMemcpy(perm, c->o.perm_global, c->m * 8, cudaMemcpyDeviceToHost));
  } else {
    for (int64_t g = 0; g < c->m; ++g) perm[g] = g;
  }
  return B2D_OK;
}

#include "mgpu.cu"

}  // namespace b2d

using namespace b2d;

struct b2d_ctx : public Ctx {};

extern "C" {

int b2d_version(void) { return 100; }
const char* b2d_last_error(void) { return g_err.c_str(); }
int b2d_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
  return n;
}

int b2d_ctx_create(int device, int64_t m, int mode, b2d_ctx** out) {
  return b2d_ctx_create_ex(device, m, mode, nullptr, out);
}

int b2d_ctx_is_out_of_core(b2d_ctx* ctx) { return ctx && ctx->ooc ? (ctx->o.dev_scratch ? 2 : 1) : 0; }

int b2d_ctx_create_ex(int device, int64_t m, int mode, const b2d_options* opt, b2d_ctx** out) {
  if (!out) return set_err(B2D_ERR_USAGE, "null out pointer");
  Ctx* c = nullptr;
  int rc = create(device, m, mode, opt, &c);
  if (rc) return rc;
  *out = static_cast<b2d_ctx*>(c);
  return B2D_OK;
}

int b2d_ctx_destroy(b2d_ctx* ctx) {
  destroy(ctx);
  return B2D_OK;
}

int b2d_ctx_factor_device_async(b2d_ctx* ctx, const void* dev_a, int64_t lda, int dtype, void* stream) {
  if (!ctx || !dev_a) return set_err(B2D_ERR_USAGE, "null argument");
  return factor_device(ctx, dev_a, lda, dtype, (cudaStream_t)stream);
}

int b2d_ctx_factor_host_async(b2d_ctx* ctx, const void* host_a, int64_t lda, int dtype, void* stream) {
  if (!ctx || !host_a) return set_err(B2D_ERR_USAGE, "null argument");
  return factor_host(ctx, host_a, lda, dtype, (cudaStream_t)stream);
}

int b2d_ctx_fetch(b2d_ctx* ctx, double* d_out, double* prefix_out, int64_t* fail_index, b2d_run_info* info) {
  if (!ctx) return set_err(B2D_ERR_USAGE, "null ctx");
  return fetch(ctx, d_out, prefix_out, fail_index, info);
}

const double* b2d_ctx_device_prefix(b2d_ctx* ctx) {
  if (ctx && ctx->mg) return ctx->mg->r[0].c->prefix;
  return ctx ? ctx->prefix : nullptr;
}

int b2d_ctx_fetch_perm(b2d_ctx* ctx, int64_t* perm_out) {
  if (!ctx) return set_err(B2D_ERR_USAGE, "null ctx");
  return fetch_perm(ctx, perm_out);
}

int b2d_ctx_set_profiling(b2d_ctx* ctx, int on) {
  if (!ctx) return set_err(B2D_ERR_USAGE, "null ctx");
  ctx->profiling = on < 0 ? 0 : (on > 2 ? 2 : on);
  return B2D_OK;
}

int b2d_ctx_update_stats(b2d_ctx* ctx, double* flops, double* ms, int64_t* launches) {
  if (!ctx) return set_err(B2D_ERR_USAGE, "null ctx");
  double f = 0, t = 0;
  for (size_t i = 0; i + 1 < ctx->prof_ev.size(); i += 2) {
    float x = 0.f;
    if (cudaEventElapsedTime(&x, ctx->prof_ev[i], ctx->prof_ev[i + 1]) != cudaSuccess)
      return set_err(B2D_ERR_CUDA, "profiling events not complete");
    t += x;
    f += ctx->prof_flops[i / 2];
  }
  if (flops) *flops = f;
  if (ms) *ms = t;
  if (launches) *launches = (int64_t)ctx->prof_flops.size();
  return B2D_OK;
}

int b2d_memdet_sym(const void* a, int64_t m, int64_t lda, int dtype, int mode, int64_t num_blocks,
                   int64_t max_mem, const int* devices, int ndev, double* d_out, int64_t* perm_out,
                   double* prefix_out, int64_t* sign_out, b2d_run_info* info, int64_t* fail_index) {
  if (ndev > 8) return set_err(B2D_ERR_USAGE, "at most 8 devices (got %d)", ndev);
  if (ndev > 0 && !devices) return set_err(B2D_ERR_USAGE, "null devices with ndev %d", ndev);
  const int device = ndev > 0 ? devices[0] : 0;
  if (!a || !prefix_out) return set_err(B2D_ERR_USAGE, "null argument");
  if (dtype != B2D_F64 && dtype != B2D_F32) return set_err(B2D_ERR_USAGE, "dtype code %d", dtype);
  const int esz = dtype == B2D_F64 ? 8 : 4;
  if (num_blocks <= 0 && max_mem <= 0)
    return set_err(B2D_ERR_USAGE, "either max_mem or num_blocks is required");
  if (num_blocks <= 0 && max_mem < 3 * esz)
    return set_err(B2D_ERR_USAGE, "budget %lld B below minimum %d B", (long long)max_mem, 3 * esz);
  auto t0 = std::chrono::steady_clock::now();
  Ctx* c = nullptr;
  b2d_options opt{};
  opt.num_blocks = num_blocks;
  opt.max_mem = max_mem;
  opt.f32_arith = dtype == B2D_F32 && mode == B2D_MODE_LDL_PIV;
  opt.ndev = ndev > 1 ? ndev : 0;
  for (int d = 0; d < ndev && ndev > 1; ++d) opt.devices[d] = devices[d];
  int rc = create(device, m, mode, &opt, &c);
  if (rc) return rc;
  rc = factor_host(c, a, lda, dtype, 0);
  b2d_run_info local{};
  std::vector<double> dtmp;
  if (rc == B2D_OK) {
    if (!d_out && sign_out) {
      dtmp.resize(m);
      d_out = dtmp.data();
    }
    rc = fetch(c, d_out, prefix_out, fail_index, &local);
  }
  if (rc == B2D_OK && perm_out) rc = fetch_perm(c, perm_out);
  destroy(c);
  if (rc != B2D_OK && rc != B2D_ERR_NOT_SPD) return rc;
  fill_ref_info(&local, m, num_blocks, max_mem, esz, mode == B2D_MODE_LU);
  local.wall_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  if (info) *info = local;
  if (rc == B2D_OK && sign_out) {
    // cumprod(sign d) (memdet.py:407); Cholesky pivots are positive.  LU: sign of det(U) only
    // (the permutation parity is the caller's, from perm_out)
    int64_t sg = 1;
    for (int64_t g = 0; g < m; ++g) {
      if (mode == B2D_MODE_LDL_PIV || mode == B2D_MODE_LU) sg *= d_out[g] > 0 ? 1 : (d_out[g] < 0 ? -1 : 0);
      sign_out[g] = sg;
    }
  }
  return rc;
}

}  // extern "C"

extern "C" int b2d_gen_rbf(const double* dev_x, int64_t n, int d, double ell, double jitter,
                           double* dev_out, void* stream) {
  if (!dev_x || !dev_out || n < 1 || d < 1) return set_err(B2D_ERR_USAGE, "bad arguments");
  const double inv2l2 = 1.0 / (2.0 * ell * ell);
  const unsigned gx = (unsigned)((n + 255) / 256);
  // rows in chunks of 65535 (grid.y limit)
  for (int64_t r0 = 0; r0 < n; r0 += 65535) {
    const unsigned rows = (unsigned)std::min<int64_t>(65535, n - r0);
    gen_rbf_kernel<<<dim3(gx, rows), 256, 0, (cudaStream_t)stream>>>(dev_x, n, d, inv2l2, jitter,
                                                                     dev_out + r0 * n, r0);
  }
  CUDA_TRY(cudaGetLastError());
  return B2D_OK;
}

extern "C" int b2d_probe_fp64_peak(int device, double seconds, double* tflops) {
  if (!tflops) return set_err(B2D_ERR_USAGE, "null output");
  CUDA_TRY(cudaSetDevice(device));
  int sms = 0;
  CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
  double* out = nullptr;
  CUDA_TRY(cudaMalloc(&out, 256 * sizeof(double)));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  int iters = 2000;
  float ms = 0.f;
  dmma_probe_kernel<<<sms * 2, 256>>>(out, 100);
  for (;;) {
    cudaEventRecord(e0);
    dmma_probe_kernel<<<sms * 2, 256>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms >= 1000.0 * seconds || iters > (1 << 26)) break;
    iters = (int)std::min<double>(1 << 26, iters * std::max(2.0, 1000.0 * seconds / std::max(ms, 0.01f)));
  }
  const double flops = (double)sms * 2 * 8 * iters * 16 * 512.0;
  *tflops = flops / (ms * 1e-3) / 1e12;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(out);
  CUDA_TRY(cudaGetLastError());
  return B2D_OK;
}

static TileMap to_map(const b2d_tilemap* m) {
  TileMap t{};
  if (!m) return t;
  t.base = m->base;
  t.ld = m->ld;
  t.packed_nt = m->packed_nt;
  t.rmod = m->rmod;
  t.rstride = m->rstride;
  t.npeer = std::max(0, std::min<int>(m->npeer, MAX_PEERS));
  for (int r = 0; r < t.npeer; ++r) t.peer[r] = m->peer[r];
  return t;
}
static TileSet to_set(const b2d_tileset* t) {
  return TileSet{t->i0, t->i1, t->j0, t->j1, t->lower, t->row_off, t->stride, t->off};
}

extern "C" int b2d_tile_potrf_inv(double* tile, double* inv, double* ell, double* diag, uint64_t* fail,
                                  int64_t g0, int64_t m, void* stream) {
  if (!tile || !inv || !ell || !diag || !fail) return set_err(B2D_ERR_USAGE, "null argument");
  int rc = configure_kernels();
  if (rc) return rc;
  potrf_inv_kernel<<<1, POTRF_THREADS, POTRF_SMEM, (cudaStream_t)stream>>>(
      tile, inv, ell, diag, (unsigned long long*)fail, g0, m);
  CUDA_TRY(cudaGetLastError());
  return B2D_OK;
}

extern "C" int b2d_tile_gemm(int mode, const b2d_tilemap* a, const b2d_tilemap* b, const b2d_tilemap* c,
                             const double* binv, const b2d_tileset* out, int32_t p0, int32_t p1, int32_t k,
                             void* stream) {
  if (!c || !out || (mode == MODE_UPDATE && (!a || !b)) || (mode == MODE_TRSM && !binv) ||
      (mode != MODE_UPDATE && mode != MODE_TRSM))
    return set_err(B2D_ERR_USAGE, "bad b2d_tile_gemm arguments");
  int rc = configure_kernels();
  if (rc) return rc;
  GemmTask t{};
  t.a = to_map(a);
  t.b = to_map(b);
  t.c = to_map(c);
  t.binv = binv;
  t.out = to_set(out);
  t.p0 = p0;
  t.p1 = p1;
  t.k = k;
  const int64_t n = t.out.count();
  if (n <= 0 || (mode == MODE_UPDATE && p1 <= p0)) return B2D_OK;
  if (mode == MODE_UPDATE)
    gemm_kernel<MODE_UPDATE><<<(unsigned)n, GEMM_THREADS, GEMM_SMEM, (cudaStream_t)stream>>>(t);
  else
    gemm_kernel<MODE_TRSM><<<(unsigned)n, GEMM_THREADS, GEMM_SMEM, (cudaStream_t)stream>>>(t);
  CUDA_TRY(cudaGetLastError());
  return B2D_OK;
}

// Device memory shared with peer ranks (multi-GPU driver: each rank's tile grid is read in place
// by the others over NVLink).  Plain cudaMalloc allocations, so an IPC handle covers exactly one
// buffer and opens at offset 0.
extern "C" int b2d_dev_alloc(int device, int64_t bytes, void** out) {
  if (!out || bytes <= 0) return set_err(B2D_ERR_USAGE, "bad b2d_dev_alloc arguments");
  CUDA_TRY(cudaSetDevice(device));
  if (cudaMalloc(out, (size_t)bytes) != cudaSuccess) {
    cudaGetLastError();
    return set_err(B2D_ERR_NOMEM, "cudaMalloc of %lld bytes failed", (long long)bytes);
  }
  return B2D_OK;
}

extern "C" int b2d_dev_free(void* p) {
  if (p) CUDA_TRY(cudaFree(p));
  return B2D_OK;
}

extern "C" int b2d_ipc_get_handle(void* p, void* handle_out) {
  if (!p || !handle_out) return set_err(B2D_ERR_USAGE, "bad b2d_ipc_get_handle arguments");
  cudaIpcMemHandle_t h;
  CUDA_TRY(cudaIpcGetMemHandle(&h, p));
  memcpy(handle_out, &h, sizeof(h));
  return B2D_OK;
}

extern "C" int b2d_ipc_open_handle(int device, const void* handle, void** out) {
  if (!handle || !out) return set_err(B2D_ERR_USAGE, "bad b2d_ipc_open_handle arguments");
  CUDA_TRY(cudaSetDevice(device));
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  CUDA_TRY(cudaIpcOpenMemHandle(out, h, cudaIpcMemLazyEnablePeerAccess));
  return B2D_OK;
}

extern "C" int b2d_ipc_close_handle(void* p) {
  if (p) CUDA_TRY(cudaIpcCloseMemHandle(p));
  return B2D_OK;
}

extern "C" int b2d_pack_tiles(const void* src, int64_t lda, int dtype, int64_t row_base, int64_t m,
                              const b2d_tilemap* out, const b2d_tileset* set, void* stream) {
  if (!src || !out || !set || (dtype != B2D_F64 && dtype != B2D_F32))
    return set_err(B2D_ERR_USAGE, "bad b2d_pack_tiles arguments");
  int rc = configure_kernels();
  if (rc) return rc;
  const TileSet ts = to_set(set);
  const int64_t n = ts.count();
  if (n <= 0) return B2D_OK;
  if (dtype == B2D_F64)
    pack_set_kernel<double><<<(unsigned)n, PACK_THREADS, PACK_SMEM, (cudaStream_t)stream>>>(
        (const double*)src, lda, row_base, m, to_map(out), ts);
  else
    pack_set_kernel<float><<<(unsigned)n, PACK_THREADS, PACK_SMEM, (cudaStream_t)stream>>>(
        (const float*)src, lda, row_base, m, to_map(out), ts);
  CUDA_TRY(cudaGetLastError());
  return B2D_OK;
}

extern "C" int b2d_h2d_2d(void* dst, int64_t dpitch, const void* src, int64_t spitch, int64_t width, int64_t height,
                          void* stream) {
  if (!dst || !src || width < 0 || height < 0) return set_err(B2D_ERR_USAGE, "bad b2d_h2d_2d arguments");
  if (width == 0 || height == 0) return B2D_OK;
  CUDA_TRY(cudaMemcpy2DAsync(dst, (size_t)dpitch, src, (size_t)spitch, (size_t)width, (size_t)height,
                             cudaMemcpyHostToDevice, (cudaStream_t)stream));
  return B2D_OK;
}

extern "C" int b2d_prefix_scan(const double* ell, int64_t m, double* prefix, void* stream) {
  if (!ell || !prefix || m < 1) return set_err(B2D_ERR_USAGE, "bad b2d_prefix_scan arguments");
  prefix_kernel<<<1, 1024, 0, (cudaStream_t)stream>>>(ell, m, prefix);
  CUDA_TRY(cudaGetLastError());
  return B2D_OK;
}

extern "C" int b2d_ctx_packed_init(b2d_ctx* ctx, double jitter, void* stream) {
  if (!ctx || ctx->ooc) return set_err(B2D_ERR_USAGE, "packed formation needs an in-core context");
  CUDA_TRY(cudaSetDevice(ctx->device));
  packed_init_kernel<<<8 * 148, 256, 0, (cudaStream_t)stream>>>(ctx->tiles, ctx->nt, ctx->m, jitter);
  CUDA_TRY(cudaGetLastError());
  return B2D_OK;
}

extern "C" int b2d_ctx_gram_accumulate(b2d_ctx* ctx, const double* dev_g, int64_t ldg, int64_t k, double scale,
                                       void* stream) {
  if (!ctx || ctx->ooc || !dev_g || k < 1 || ldg < k) return set_err(B2D_ERR_USAGE, "bad gram_accumulate arguments");
  CUDA_TRY(cudaSetDevice(ctx->device));
  int rc = configure_kernels();
  if (rc) return rc;
  const int nt = ctx->nt;
  const int kt = (int)((k + T - 1) / T);
  const int64_t need = (int64_t)nt * kt;
  if (need > ctx->gram_cap) {
    cudaFree(ctx->gram_neg);
    cudaFree(ctx->gram_pos);
    ctx->gram_neg = ctx->gram_pos = nullptr;
    CUDA_TRY(cudaMalloc(&ctx->gram_neg, (size_t)need * TILE_BYTES));
    CUDA_TRY(cudaMalloc(&ctx->gram_pos, (size_t)need * TILE_BYTES));
    ctx->gram_cap = need;
  }
  cudaStream_t s = (cudaStream_t)stream;
  const TileMap gneg{ctx->gram_neg, kt, 0, 0, 0}, gpos{ctx->gram_pos, kt, 0, 0, 0};
  pack_rect_kernel<<<(unsigned)need, 256, 0, s>>>(dev_g, ldg, ctx->m, k, -scale, gneg, kt);
  pack_rect_kernel<<<(unsigned)need, 256, 0, s>>>(dev_g, ldg, ctx->m, k, 1.0, gpos, kt);
  // K -= (-scale G) G^T over the packed lower tiles: the engine's DMMA Schur kernel
  GemmTask t{};
  t.a = gneg;
  t.b = gpos;
  t.c = TileMap{ctx->tiles, 0, nt, 0, 0};
  t.out = TileSet{0, nt, 0, nt, 1, 0, 0, 0};
  t.p0 = 0;
  t.p1 = kt;
  gemm_kernel<MODE_UPDATE><<<(unsigned)t.out.count(), GEMM_THREADS, GEMM_SMEM, s>>>(t);
  CUDA_TRY(cudaGetLastError());
  return B2D_OK;
}

extern "C" int b2d_ctx_factor_packed_async(b2d_ctx* ctx, void* stream) {
  if (!ctx || ctx->ooc) return set_err(B2D_ERR_USAGE, "factor_packed needs an in-core context");
  CUDA_TRY(cudaSetDevice(ctx->device));
  cudaStream_t user = (cudaStream_t)stream;
  begin(ctx, user);
  make_bounds(ctx, ctx->nt, false);
  std::fill(ctx->act.begin(), ctx->act.end(), -1);
  enqueue_factor(ctx, FactorTarget{TileMap{ctx->tiles, 0, ctx->nt}, ctx->nt, 0}, false);
  enqueue_prefix(ctx);
  end(ctx, user);
  CUDA_TRY(cudaGetLastError());
  return B2D_OK;
}

// ---------------------------------------------------------------- tile seam: oocdet.kernels on the GPU
// Host tiles in, host tiles out (the reference's kernel module, kernels/__init__.py:24-45,
// dense.py:57-116): each call uploads its operands, runs the ldl32.cu kernels in the file dtype
// with the golden host's BLAS / LAPACK rounding sequence (LDL, TRSM, GEMM: bit-identical there),
// and writes the results back in place.  Synchronous; for the reference's own driver patched
// onto this engine (paper_2503_04424_b200/kernels.py), not the hot path.
namespace b2d {

template <typename E>
__global__ void seam_lower_to_rowmajor_kernel(const E* __restrict__ dense, int64_t n, E* __restrict__ M, int zero_upper) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n * n; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / n, j = e % n;
    if (j <= i) M[e] = dense[j * n + i];
    else if (zero_upper) M[e] = (E)0;
  }
}

// Unblocked right-looking Cholesky step j on a column-major block: l_jj = sqrt(a_jj) (fail when
// a_jj is not positive), l_ij = a_ij / l_jj; then the trailing update a_ik -= l_ij l_kj.
template <typename E>
__global__ void seam_chol_step_kernel(E* a, int64_t n, int64_t j, unsigned long long* fail) {
  __shared__ E piv;
  if (*fail != ~0ull) return;
  if (threadIdx.x == 0) {
    const E v = a[j * n + j];
    piv = v > (E)0 ? sqrt(v) : (E)-1;
    if (!(v > (E)0)) atomicMin(fail, (unsigned long long)j);
    else a[j * n + j] = piv;
  }
  __syncthreads();
  if (piv < (E)0) return;
  for (int64_t i = j + 1 + threadIdx.x; i < n; i += blockDim.x) a[j * n + i] = Blas<E>::div(a[j * n + i], piv);
}
template <typename E>
__global__ void seam_chol_update_kernel(E* a, int64_t n, int64_t j, const unsigned long long* fail) {
  if (*fail != ~0ull) return;
  const int64_t k = j + 1 + blockIdx.x;
  const E lkj = a[j * n + k];
  for (int64_t i = k + threadIdx.x; i < n; i += blockDim.x) a[k * n + i] = Blas<E>::fma(-a[j * n + i], lkj, a[k * n + i]);
}

struct SeamMem {
  std::vector<void*> p;
  ~SeamMem() {
    for (void* q : p) cudaFree(q);
  }
  template <typename X>
  X* get(size_t count) {
    void* q = nullptr;
    if (cudaMalloc(&q, std::max<size_t>(count, 1) * sizeof(X)) != cudaSuccess) return nullptr;
    p.push_back(q);
    return (X*)q;
  }
};

template <typename E>
static int seam_ldl(E* a, int64_t n, int64_t lda, double tol, int64_t* swaps, E* d, int64_t* fail_step) {
  SeamMem mem;
  E *M = mem.get<E>(n * n), *dense = mem.get<E>(n * n), *work = mem.get<E>(n), *dd = mem.get<E>(n);
  int64_t *sw = mem.get<int64_t>(n);
  unsigned long long *fail = mem.get<unsigned long long>(1), *amax = mem.get<unsigned long long>(1);
  if (!M || !dense || !work || !dd || !sw || !fail || !amax) return set_err(B2D_ERR_NOMEM, "tile seam: device allocation");
  CUDA_TRY(cudaMemcpy2D(M, n * sizeof(E), a, lda * sizeof(E), n * sizeof(E), n, cudaMemcpyHostToDevice));
  cudaMemset(fail, 0xff, 8);
  cudaMemset(amax, 0, 8);
  const dim3 gb((unsigned)((n + 31) / 32), (unsigned)((n + 31) / 32));
  l32_block_in_kernel<E><<<gb, 256>>>(M, n, 0, n, dense, n, amax);
  const L32Step<E> g{dense, n, n, 0, work, dd, sw, fail, amax, tol};
  for (int64_t r = 0; r < n; ++r) {
    l32_step_kernel<E><<<1, 1024>>>(g, r);
    if (r + 1 < n) l32_update_kernel<E><<<(unsigned)(n - r - 1), 256>>>(g, r);
  }
  unsigned long long f = ~0ull;
  CUDA_TRY(cudaMemcpy(&f, fail, 8, cudaMemcpyDeviceToHost));
  *fail_step = f == ~0ull ? -1 : (int64_t)f;
  if (f != ~0ull) return B2D_OK;  // the caller raises (dense.py:74-80)
  seam_lower_to_rowmajor_kernel<E><<<1024, 256>>>(dense, n, M, 0);  // the strict upper part stays the input's
  CUDA_TRY(cudaMemcpy2D(a, lda * sizeof(E), M, n * sizeof(E), n * sizeof(E), n, cudaMemcpyDeviceToHost));
  CUDA_TRY(cudaMemcpy(swaps, sw, n * 8, cudaMemcpyDeviceToHost));
  CUDA_TRY(cudaMemcpy(d, dd, n * sizeof(E), cudaMemcpyDeviceToHost));
  CUDA_TRY(cudaGetLastError());
  return B2D_OK;
}

template <typename E>
static int seam_cholesky(E* a, int64_t n, int64_t lda, E* diag, int64_t* fail_step) {
  SeamMem mem;
  E *M = mem.get<E>(n * n), *dense = mem.get<E>(n * n);
  unsigned long long *fail = mem.get<unsigned long long>(1), *amax = mem.get<unsigned long long>(1);
  if (!M || !dense || !fail || !amax) return set_err(B2D_ERR_NOMEM, "tile seam: device allocation");
  CUDA_TRY(cudaMemcpy2D(M, n * sizeof(E), a, lda * sizeof(E), n * sizeof(E), n, cudaMemcpyHostToDevice));
  cudaMemset(fail, 0xff, 8);
  const dim3 gb((unsigned)((n + 31) / 32), (unsigned)((n + 31) / 32));
  l32_block_in_kernel<E><<<gb, 256>>>(M, n, 0, n, dense, n, amax);
  for (int64_t j = 0; j < n; ++j) {
    seam_chol_step_kernel<E><<<1, 256>>>(dense, n, j, fail);
    if (j + 1 < n) seam_chol_update_kernel<E><<<(unsigned)(n - j - 1), 256>>>(dense, n, j, fail);
  }
  unsigned long long f = ~0ull;
  CUDA_TRY(cudaMemcpy(&f, fail, 8, cudaMemcpyDeviceToHost));
  *fail_step = f == ~0ull ? -1 : (int64_t)f;
  if (f != ~0ull) return B2D_OK;
  seam_lower_to_rowmajor_kernel<E><<<1024, 256>>>(dense, n, M, 1);  // L, zeros above (scipy's lower factor)
  CUDA_TRY(cudaMemcpy2D(a, lda * sizeof(E), M, n * sizeof(E), n * sizeof(E), n, cudaMemcpyDeviceToHost));
  for (int64_t j = 0; j < n; ++j) diag[j] = a[j * lda + j];
  CUDA_TRY(cudaGetLastError());
  return B2D_OK;
}

template <typename E>
static int seam_trsm(const E* l, int64_t n, int64_t ldl, E* b, int64_t w, int64_t ldb, int unit) {
  SeamMem mem;
  E *M = mem.get<E>(n * n), *dense = mem.get<E>(n * n), *X = mem.get<E>(n * w);
  unsigned long long *fail = mem.get<unsigned long long>(1), *amax = mem.get<unsigned long long>(1);
  if (!M || !dense || !X || !fail || !amax) return set_err(B2D_ERR_NOMEM, "tile seam: device allocation");
  CUDA_TRY(cudaMemcpy2D(M, n * sizeof(E), l, ldl * sizeof(E), n * sizeof(E), n, cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy2D(X, w * sizeof(E), b, ldb * sizeof(E), w * sizeof(E), n, cudaMemcpyHostToDevice));
  cudaMemset(fail, 0xff, 8);
  const dim3 gb((unsigned)((n + 31) / 32), (unsigned)((n + 31) / 32));
  l32_block_in_kernel<E><<<gb, 256>>>(M, n, 0, n, dense, n, amax);  // L column-major
  constexpr int Q = Blas<E>::Q, TW = TrsmTW<E>::v;
  for (int64_t ls = 0; ls < n; ls += Q) {
    const int64_t le = std::min<int64_t>(n, ls + Q);
    l32_trsm_diag_kernel<E><<<(unsigned)((w + TW - 1) / TW), 256, l32_trsm_smem<E>()>>>(dense, n, X, w, w, ls, le, unit,
                                                                                      fail);
    if (le < n) {
      GT<E> u{};
      u.A = dense + ls * n + le;
      u.lda = n;
      u.B = X + ls * w;
      u.ldb = w;
      u.C = X + le * w;
      u.ldc = w;
      u.Mr = n - le;
      u.Nc = w;
      u.nkb = 1;
      u.kb[1] = (int)(le - ls);
      u.blk = 1;
      l32_gemm_kernel<E><<<dim3((unsigned)((w + G32_BN - 1) / G32_BN), (unsigned)((n - le + gemm_bm<E>() - 1) / gemm_bm<E>())),
                           256>>>(u, fail);
    }
  }
  CUDA_TRY(cudaMemcpy2D(b, ldb * sizeof(E), X, w * sizeof(E), w * sizeof(E), n, cudaMemcpyDeviceToHost));
  CUDA_TRY(cudaGetLastError());
  return B2D_OK;
}

template <typename E>
static int seam_schur(E* s, int64_t m, int64_t nn, int64_t lds, const E* c, int64_t ldc, const E* b, int64_t ldb,
                      int64_t K) {
  SeamMem mem;
  E *S = mem.get<E>(m * nn), *C = mem.get<E>(K * m), *B = mem.get<E>(K * nn);
  unsigned long long* fail = mem.get<unsigned long long>(1);
  if (!S || !C || !B || !fail) return set_err(B2D_ERR_NOMEM, "tile seam: device allocation");
  CUDA_TRY(cudaMemcpy2D(S, nn * sizeof(E), s, lds * sizeof(E), nn * sizeof(E), m, cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy2D(C, m * sizeof(E), c, ldc * sizeof(E), m * sizeof(E), K, cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy2D(B, nn * sizeof(E), b, ldb * sizeof(E), nn * sizeof(E), K, cudaMemcpyHostToDevice));
  cudaMemset(fail, 0xff, 8);
  GT<E> u{};
  u.A = C;
  u.lda = m;
  u.B = B;
  u.ldb = nn;
  u.C = S;
  u.ldc = nn;
  u.Mr = m;
  u.Nc = nn;
  u.nkb = l32_kblocks(K, u.kb, Blas<E>::Q);
  u.blk = 1;
  if (K > 0)
    l32_gemm_kernel<E><<<dim3((unsigned)((nn + G32_BN - 1) / G32_BN), (unsigned)((m + gemm_bm<E>() - 1) / gemm_bm<E>())),
                         256>>>(u, fail);
  CUDA_TRY(cudaMemcpy2D(s, lds * sizeof(E), S, nn * sizeof(E), nn * sizeof(E), m, cudaMemcpyDeviceToHost));
  CUDA_TRY(cudaGetLastError());
  return B2D_OK;
}

static int seam_begin(int device, int dtype) {
  if (dtype != B2D_F64 && dtype != B2D_F32) return set_err(B2D_ERR_USAGE, "dtype code %d", dtype);
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    return set_err(B2D_ERR_CUDA, "no CUDA device visible: the B200 engine has no CPU fallback");
  if (device < 0 || device >= ndev) return set_err(B2D_ERR_USAGE, "bad device %d", device);
  CUDA_TRY(cudaSetDevice(device));
  return configure_kernels();
}

}  // namespace b2d

extern "C" int b2d_tile_ldl_host(void* a, int64_t n, int64_t lda, int dtype, double tol, int64_t* swaps, void* d,
                                 int64_t* fail_step, int device) {
  if (!a || !swaps || !d || !fail_step || n < 0 || lda < n) return set_err(B2D_ERR_USAGE, "bad b2d_tile_ldl_host arguments");
  if (int rc = seam_begin(device, dtype)) return rc;
  *fail_step = -1;
  if (n == 0) return B2D_OK;
  return dtype == B2D_F64 ? seam_ldl<double>((double*)a, n, lda, tol, swaps, (double*)d, fail_step)
                          : seam_ldl<float>((float*)a, n, lda, tol, swaps, (float*)d, fail_step);
}

extern "C" int b2d_tile_cholesky_host(void* a, int64_t n, int64_t lda, int dtype, void* diag, int64_t* fail_step,
                                      int device) {
  if (!a || !diag || !fail_step || n < 0 || lda < n) return set_err(B2D_ERR_USAGE, "bad b2d_tile_cholesky_host arguments");
  if (int rc = seam_begin(device, dtype)) return rc;
  *fail_step = -1;
  if (n == 0) return B2D_OK;
  return dtype == B2D_F64 ? seam_cholesky<double>((double*)a, n, lda, (double*)diag, fail_step)
                          : seam_cholesky<float>((float*)a, n, lda, (float*)diag, fail_step);
}

extern "C" int b2d_tile_solve_lower_host(const void* l, int64_t n, int64_t ldl, void* b, int64_t w, int64_t ldb, int dtype,
                                         int unit_diag, int device) {
  if (!l || !b || n < 0 || w < 0 || ldl < n || ldb < w) return set_err(B2D_ERR_USAGE, "bad b2d_tile_solve_lower_host arguments");
  if (int rc = seam_begin(device, dtype)) return rc;
  if (n == 0 || w == 0) return B2D_OK;
  return dtype == B2D_F64 ? seam_trsm<double>((const double*)l, n, ldl, (double*)b, w, ldb, unit_diag)
                          : seam_trsm<float>((const float*)l, n, ldl, (float*)b, w, ldb, unit_diag);
}

extern "C" int b2d_tile_schur_update_host(void* s, int64_t m, int64_t n, int64_t lds, const void* c, int64_t ldc,
                                          const void* b, int64_t ldb, int64_t k, int dtype, int device) {
  if (!s || !c || !b || m < 0 || n < 0 || k < 0 || lds < n || ldc < m || ldb < n)
    return set_err(B2D_ERR_USAGE, "bad b2d_tile_schur_update_host arguments");
  if (int rc = seam_begin(device, dtype)) return rc;
  if (m == 0 || n == 0) return B2D_OK;
  return dtype == B2D_F64 ? seam_schur<double>((double*)s, m, n, lds, (const double*)c, ldc, (const double*)b, ldb, k)
                          : seam_schur<float>((float*)s, m, n, lds, (const float*)c, ldc, (const float*)b, ldb, k);
}
