// Host side of the B200 MEMDET engine: HBM planner, right-looking tiled factorisation driver
// with one-panel look-ahead on two prioritised streams, host<->HBM strip streamer, and the
// C ABI declared in include/memdet_b200.h.
//
// Reference driver mirrored: _memdet_symmetric (memdet.py:322-389).  The reference walks an
// n_b x n_b tile grid out of core with four resident b x b buffers; here the whole lower tile
// triangle is resident in HBM (packed, 128-wide tiles) and the same three steps run per
// 128-wide tile-column k:  factor the diagonal tile (dense.py:84-91), solve the panel
// (dense.py:94-99), Schur-update the trailing tiles (dense.py:109-116); the prefix is the
// running sum of 2 log L_ii (memdet.py:428).
#include <algorithm>
#include <chrono>
#include <climits>
#include <cstdlib>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/memdet_b200.h"
#include "kernels.cu"

namespace b2d {

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
// (default 8; B2D_PANEL_TILES overrides for tuning)
static int panel_tiles_default() {
  const char* e = getenv("B2D_PANEL_TILES");
  int w = e ? atoi(e) : 8;
  return w < 1 ? 1 : (w > 16 ? 16 : w);
}

constexpr int NSTAGE = 8;   // host-ingest staging strips in flight
constexpr int BAND = 4;     // tile-columns per ingest band

struct Ctx {
  int device = 0;
  int64_t m = 0;
  int mode = B2D_MODE_CHOLESKY;
  int nt = 0;
  int W_TILES = 8;
  double* tiles = nullptr;   // packed lower tile triangle
  double* inv = nullptr;     // nt inverse diagonal tiles
  double* ell = nullptr;     // n_pad: 2 log L_ii
  double* diag = nullptr;    // n_pad: L_ii
  double* prefix = nullptr;  // n_pad
  unsigned long long* fail = nullptr;
  double* strip[NSTAGE] = {};  // host-ingest staging strips (128 x n_pad doubles each)
  cudaStream_t s_main = nullptr, s_side = nullptr, s_copy = nullptr, s_pack = nullptr;
  cudaEvent_t ev_start = nullptr, ev_stop = nullptr, ev_join = nullptr;
  std::vector<cudaEvent_t> ev_panel, ev_rest, ev_catch, ev_stage, ev_copied, ev_band;
  // band activation (host ingest): band b = tile-columns [b*BAND, (b+1)*BAND) joins the
  // right-looking updates at outer step act[b] (-1: from the start) after one catch-up update
  std::vector<int> act;
  bool trace = false;  // B2D_TRACE: print a per-step event timeline on fetch
  bool profiling = false;
  std::vector<cudaEvent_t> prof_ev;
  std::vector<double> prof_flops;
  int64_t launches = 0;
  int64_t h2d = 0, d2h = 0;
  bool pending = false;
  std::chrono::steady_clock::time_point t0;
};

static int configure_kernels() {
  static bool done = false;
  if (done) return B2D_OK;
  CUDA_TRY(cudaFuncSetAttribute(gemm_kernel<MODE_UPDATE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)GEMM_SMEM));
  CUDA_TRY(cudaFuncSetAttribute(gemm_kernel<MODE_TRSM>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)GEMM_SMEM));
  CUDA_TRY(cudaFuncSetAttribute(potrf_inv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)POTRF_SMEM));
  CUDA_TRY(cudaFuncSetAttribute(pack_tiles_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)PACK_SMEM));
  CUDA_TRY(cudaFuncSetAttribute(pack_tiles_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)PACK_SMEM));
  done = true;
  return B2D_OK;
}

static void destroy(Ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  if (c->s_main) cudaStreamSynchronize(c->s_main);
  if (c->s_side) cudaStreamSynchronize(c->s_side);
  cudaFree(c->tiles);
  cudaFree(c->inv);
  cudaFree(c->ell);
  cudaFree(c->diag);
  cudaFree(c->prefix);
  cudaFree(c->fail);
  if (c->s_copy) cudaStreamSynchronize(c->s_copy);
  for (auto* p : c->strip) cudaFree(p);
  if (c->s_pack) cudaStreamSynchronize(c->s_pack);
  for (auto* v : {&c->ev_panel, &c->ev_rest, &c->ev_catch, &c->ev_stage, &c->ev_copied, &c->ev_band,
                  &c->prof_ev})
    for (auto e : *v) cudaEventDestroy(e);
  if (c->ev_start) cudaEventDestroy(c->ev_start);
  if (c->ev_stop) cudaEventDestroy(c->ev_stop);
  if (c->ev_join) cudaEventDestroy(c->ev_join);
  if (c->s_main) cudaStreamDestroy(c->s_main);
  if (c->s_side) cudaStreamDestroy(c->s_side);
  if (c->s_copy) cudaStreamDestroy(c->s_copy);
  if (c->s_pack) cudaStreamDestroy(c->s_pack);
  delete c;
}

static int create(int device, int64_t m, int mode, Ctx** out) {
  if (m < 1) return set_err(B2D_ERR_USAGE, "matrix dimension must be >= 1, got %lld", (long long)m);
  if (mode == B2D_MODE_LDL_PIV)
    return set_err(B2D_ERR_UNSUPPORTED, "block-pivoted LDL is not built in this engine version");
  if (mode != B2D_MODE_CHOLESKY && mode != B2D_MODE_LDL_NOPIV)
    return set_err(B2D_ERR_USAGE, "unknown mode %d", mode);
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    return set_err(B2D_ERR_CUDA, "no CUDA device visible: the B200 engine has no CPU fallback");
  if (device < 0 || device >= ndev) return set_err(B2D_ERR_USAGE, "bad device %d", device);
  CUDA_TRY(cudaSetDevice(device));
  int rc = configure_kernels();
  if (rc) return rc;
  Ctx* c = new Ctx();
  c->device = device;
  c->m = m;
  c->mode = mode;
  c->nt = (int)((m + T - 1) / T);
  c->W_TILES = panel_tiles_default();
  const int64_t npad = (int64_t)c->nt * T;
  const size_t tile_bytes = (size_t)n_packed_tiles(c->nt) * TILE_BYTES;
  size_t free_b = 0, total_b = 0;
  cudaMemGetInfo(&free_b, &total_b);
  const size_t need = tile_bytes + (size_t)c->nt * TILE_BYTES + 3 * npad * 8 + 2 * (size_t)T * npad * 8;
  if (need + (size_t)(1 << 28) > free_b) {
    destroy(c);
    return set_err(B2D_ERR_NOMEM,
                   "in-core plan needs %.2f GB of HBM (%.2f GB free); the out-of-core streamer is not "
                   "built in this engine version",
                   need / 1e9, free_b / 1e9);
  }
#define ALLOC(ptr, bytes)                                        \
  do {                                                           \
    cudaError_t e_ = cudaMalloc((void**)&(ptr), (bytes));        \
    if (e_ != cudaSuccess) {                                     \
      destroy(c);                                                \
      return set_err(B2D_ERR_NOMEM, "cudaMalloc(%zu) failed: %s", (size_t)(bytes), cudaGetErrorString(e_)); \
    }                                                            \
  } while (0)
  ALLOC(c->tiles, tile_bytes);
  ALLOC(c->inv, (size_t)c->nt * TILE_BYTES);
  ALLOC(c->ell, npad * 8);
  ALLOC(c->diag, npad * 8);
  ALLOC(c->prefix, npad * 8);
  ALLOC(c->fail, 8);
#undef ALLOC
  int lo = 0, hi = 0;
  cudaDeviceGetStreamPriorityRange(&lo, &hi);
  // panel chain (critical path) gets the highest priority; trailing updates the lowest
  if (cudaStreamCreateWithPriority(&c->s_main, cudaStreamNonBlocking, hi) != cudaSuccess ||
      cudaStreamCreateWithPriority(&c->s_side, cudaStreamNonBlocking, lo) != cudaSuccess ||
      cudaStreamCreateWithPriority(&c->s_copy, cudaStreamNonBlocking, hi) != cudaSuccess ||
      cudaStreamCreateWithPriority(&c->s_pack, cudaStreamNonBlocking, hi) != cudaSuccess) {
    destroy(c);
    return set_err(B2D_ERR_CUDA, "stream creation failed");
  }
  cudaEventCreate(&c->ev_start);
  cudaEventCreate(&c->ev_stop);
  cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming);
  const int nsteps = (c->nt + c->W_TILES - 1) / c->W_TILES;
  c->ev_panel.resize(nsteps);
  c->ev_rest.resize(nsteps);
  c->ev_catch.resize(nsteps);
  c->trace = getenv("B2D_TRACE") != nullptr;
  const unsigned evf = c->trace ? cudaEventDefault : cudaEventDisableTiming;
  for (int s = 0; s < nsteps; ++s) {
    cudaEventCreateWithFlags(&c->ev_panel[s], evf);
    cudaEventCreateWithFlags(&c->ev_rest[s], evf);
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
  *out = c;
  return B2D_OK;
}

static int64_t tiles_in(int nt, int j0, int j1, int row_off) {
  int64_t n = 0;
  for (int j = j0; j < j1; ++j) n += std::max(0, nt - j - row_off);
  return n;
}

// MODE_UPDATE over output tile-columns [j0, j1) with K tile-columns [p0, p1)
static void launch_update(Ctx* c, cudaStream_t s, int j0, int j1, int p0, int p1, bool prof) {
  const int64_t ntile = tiles_in(c->nt, j0, j1, 0);
  if (ntile <= 0 || p1 <= p0) return;
  GemmTask t{};
  t.tiles = c->tiles;
  t.nt = c->nt;
  t.j0 = j0;
  t.j1 = j1;
  t.row_off = 0;
  t.p0 = p0;
  t.p1 = p1;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (prof && c->profiling) {
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0, s);
  }
  gemm_kernel<MODE_UPDATE><<<(unsigned)ntile, GEMM_THREADS, GEMM_SMEM, s>>>(t);
  c->launches++;
  if (e0) {
    cudaEventRecord(e1, s);
    c->prof_ev.push_back(e0);
    c->prof_ev.push_back(e1);
    // algorithmic flops: off-diagonal tiles 2*T*T*K, diagonal (SYRK, lower half) T*(T+1)*K
    const double K = (double)(p1 - p0) * T;
    const int64_t ndiag = j1 - j0;
    c->prof_flops.push_back((double)(ntile - ndiag) * 2.0 * T * T * K + (double)ndiag * T * (T + 1.0) * K);
  }
}

static void launch_panel_column(Ctx* c, cudaStream_t s, int p) {
  const int nt = c->nt;
  double* invp = c->inv + (int64_t)p * TILE_ELEMS;
  potrf_inv_kernel<<<1, POTRF_THREADS, POTRF_SMEM, s>>>(c->tiles, nt, p, invp, c->ell, c->diag, c->fail, c->m);
  c->launches++;
  if (p + 1 < nt) {
    GemmTask t{};
    t.tiles = c->tiles;
    t.binv = invp;
    t.nt = nt;
    t.j0 = p;
    t.j1 = p + 1;
    t.row_off = 1;
    t.k = p;
    gemm_kernel<MODE_TRSM><<<nt - p - 1, GEMM_THREADS, GEMM_SMEM, s>>>(t);
    c->launches++;
  }
}

// The factorisation proper.  Tile-columns of bands with act[b] == -1 are in HBM (or their
// band event is waited on) before step 0; a band with act[b] = s >= 0 first receives one
// catch-up update with every panel of steps < s (K = 128*k0, on s_side, after its band event),
// then joins the regular next-cols / rest updates from step s on.  act[b] <= the step whose
// next-cols update first touches band b, so every column is current before it is factored.
static void enqueue_factor(Ctx* c, bool wait_bands) {
  const int nt = c->nt;
  const int W_TILES = c->W_TILES;
  const int nsteps = (nt + W_TILES - 1) / W_TILES;
  const int nbands = (nt + BAND - 1) / BAND;
  if (wait_bands) {
    for (int b = 0; b < nbands; ++b)
      if (c->act[b] < 0) cudaStreamWaitEvent(c->s_side, c->ev_band[b], 0);
  }
  int main_waited = 0;  // initial bands s_main has waited for (waited lazily, per panel column)
  for (int st = 0; st < nsteps; ++st) {
    const int k0 = st * W_TILES;
    const int ke = std::min(k0 + W_TILES, nt);
    // panel(k0): its columns were last touched by next-cols(st-1) (same stream) and rest(st-2)
    if (st >= 2) cudaStreamWaitEvent(c->s_main, c->ev_rest[st - 2], 0);
    for (int p = k0; p < ke; ++p) {
      if (wait_bands) {
        // an initial band must be in HBM before the first panel column that reads it (the
        // intra-panel update touches columns up to ke-1)
        const int need = std::min(nbands, (ke - 1) / BAND + 1);
        while (main_waited < need && c->act[main_waited] < 0)
          cudaStreamWaitEvent(c->s_main, c->ev_band[main_waited++], 0);
      }
      launch_panel_column(c, c->s_main, p);
      if (p + 1 < ke) launch_update(c, c->s_main, p + 1, ke, p, p + 1, false);
    }
    cudaEventRecord(c->ev_panel[st], c->s_main);
    if (ke >= nt) break;
    const int ne = std::min(ke + W_TILES, nt);
    // catch-up of the bands that join at this step (panels of steps < st, already factored)
    int end_active = 0;
    for (int b = 0; b < nbands; ++b) {
      if (c->act[b] == st) {
        if (wait_bands) cudaStreamWaitEvent(c->s_side, c->ev_band[b], 0);
        launch_update(c, c->s_side, b * BAND, std::min(nt, (b + 1) * BAND), 0, k0, false);
      }
      if (c->act[b] <= st) end_active = std::min(nt, (b + 1) * BAND);
    }
    cudaEventRecord(c->ev_catch[st], c->s_side);
    // next-cols(k0): the next panel's columns, on the critical path
    cudaStreamWaitEvent(c->s_main, c->ev_catch[st], 0);
    launch_update(c, c->s_main, ke, ne, k0, ke, false);
    // rest(k0): active columns right of the next panel, overlapping the next panel
    cudaStreamWaitEvent(c->s_side, c->ev_panel[st], 0);
    launch_update(c, c->s_side, ne, std::max(ne, end_active), k0, ke, true);
    cudaEventRecord(c->ev_rest[st], c->s_side);
  }
  // join the side stream, then the prefix scan
  cudaEventRecord(c->ev_join, c->s_side);
  cudaStreamWaitEvent(c->s_main, c->ev_join, 0);
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

static int factor_device(Ctx* c, const void* a, int64_t lda, int dtype, cudaStream_t user) {
  if (dtype != B2D_F64 && dtype != B2D_F32) return set_err(B2D_ERR_USAGE, "dtype code %d", dtype);
  if (lda < c->m) return set_err(B2D_ERR_USAGE, "lda %lld < m", (long long)lda);
  CUDA_TRY(cudaSetDevice(c->device));
  begin(c, user);
  const unsigned ntiles = (unsigned)n_packed_tiles(c->nt);
  if (dtype == B2D_F64)
    pack_tiles_kernel<double><<<ntiles, PACK_THREADS, PACK_SMEM, c->s_main>>>(
        (const double*)a, lda, 0, c->m, c->tiles, c->nt, 0);
  else
    pack_tiles_kernel<float><<<ntiles, PACK_THREADS, PACK_SMEM, c->s_main>>>(
        (const float*)a, lda, 0, c->m, c->tiles, c->nt, 0);
  c->launches++;
  cudaEventRecord(c->ev_join, c->s_main);
  cudaStreamWaitEvent(c->s_side, c->ev_join, 0);
  std::fill(c->act.begin(), c->act.end(), -1);
  enqueue_factor(c, false);
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
  const int nt = c->nt, W = c->W_TILES;
  const int nbands = (nt + BAND - 1) / BAND;
  const int nsteps = (nt + W - 1) / W;
  const double m = (double)c->m, pcie = 48e9, rate = 34e12, chain_rate = 20e12, col_lat = 200e-6;
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
  double t = 0.0;
  int next = 0;
  while (next < nbands && (next * BAND) / W - 1 < 0) {  // needed by step 0's panel / next-cols
    c->act[next] = -1;
    t = std::max(t, arrival[next]);
    ++next;
  }
  for (int st = 0; st < nsteps && next < nbands; ++st) {
    const int k0 = st * W, ke = std::min(k0 + W, nt), ne = std::min(ke + W, nt);
    // critical chain of the step (s_main): panel columns + intra-panel and next-cols updates
    const double chain = W * col_lat +
                         (0.5 * W * (W - 1) * (nt - k0) * tile_flops + tiles(ke, ne) * tile_flops * W) /
                             chain_rate;
    double side = 0.0;  // s_side: catch-ups of joining bands + rest over active bands
    while (next < nbands && (arrival[next] <= t || (next * BAND) / W - 1 <= st)) {
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
static int factor_host(Ctx* c, const void* a, int64_t lda, int dtype, cudaStream_t user) {
  if (dtype != B2D_F64 && dtype != B2D_F32) return set_err(B2D_ERR_USAGE, "dtype code %d", dtype);
  if (lda < c->m) return set_err(B2D_ERR_USAGE, "lda %lld < m", (long long)lda);
  CUDA_TRY(cudaSetDevice(c->device));
  const int64_t npad = (int64_t)c->nt * T;
  const size_t esz = dtype == B2D_F64 ? 8 : 4;
  for (int b = 0; b < NSTAGE; ++b)
    if (!c->strip[b]) CUDA_TRY(cudaMalloc(&c->strip[b], (size_t)T * npad * 8));
  begin(c, user);
  plan_bands(c, esz);
  for (int J = 0; J < c->nt; ++J) {
    const int b = J % NSTAGE;
    const int64_t r0 = (int64_t)J * T;
    const int64_t rows = std::min<int64_t>(T, c->m - r0);
    const int64_t cols = c->m - r0;  // columns [r0, m): the upper triangle of this strip
    // staging buffer b is free once the pack of strip J - NSTAGE has run
    if (J >= NSTAGE) cudaStreamWaitEvent(c->s_copy, c->ev_stage[b], 0);
    const char* src = (const char*)a + (size_t)(r0 * lda + r0) * esz;
    // staged with leading dimension npad, offset so that column r0 lands at index r0
    char* dst = (char*)c->strip[b] + (size_t)r0 * esz;
    CUDA_TRY(cudaMemcpy2DAsync(dst, (size_t)npad * esz, src, (size_t)lda * esz, (size_t)cols * esz,
                               (size_t)rows, cudaMemcpyHostToDevice, c->s_copy));
    cudaEventRecord(c->ev_copied[b], c->s_copy);
    c->h2d += rows * cols * (int64_t)esz;
    cudaStreamWaitEvent(c->s_pack, c->ev_copied[b], 0);
    const unsigned ntile = (unsigned)(c->nt - J);
    if (dtype == B2D_F64)
      pack_tiles_kernel<double><<<ntile, PACK_THREADS, PACK_SMEM, c->s_pack>>>(
          (const double*)c->strip[b], npad, r0, c->m, c->tiles, c->nt, J);
    else
      pack_tiles_kernel<float><<<ntile, PACK_THREADS, PACK_SMEM, c->s_pack>>>(
          (const float*)c->strip[b], npad, r0, c->m, c->tiles, c->nt, J);
    c->launches++;
    cudaEventRecord(c->ev_stage[b], c->s_pack);
    if ((J + 1) % BAND == 0 || J + 1 == c->nt) cudaEventRecord(c->ev_band[J / BAND], c->s_pack);
  }
  enqueue_factor(c, true);
  cudaEventRecord(c->ev_join, c->s_pack);
  cudaStreamWaitEvent(c->s_main, c->ev_join, 0);
  end(c, user);
  CUDA_TRY(cudaGetLastError());
  return B2D_OK;
}

static int fetch(Ctx* c, double* d_out, double* prefix_out, int64_t* fail_index, b2d_run_info* info) {
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
  if (fail != ULLONG_MAX)
    return set_err(B2D_ERR_NOT_SPD, "leading minor of order %lld is not positive definite",
                   (long long)fail + 1);
  return B2D_OK;
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

static void fill_ref_info(b2d_run_info* info, int64_t m, int64_t num_blocks, int64_t max_mem, int esz) {
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
}

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
  if (!out) return set_err(B2D_ERR_USAGE, "null out pointer");
  Ctx* c = nullptr;
  int rc = create(device, m, mode, &c);
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

const double* b2d_ctx_device_prefix(b2d_ctx* ctx) { return ctx ? ctx->prefix : nullptr; }

int b2d_ctx_set_profiling(b2d_ctx* ctx, int on) {
  if (!ctx) return set_err(B2D_ERR_USAGE, "null ctx");
  ctx->profiling = on != 0;
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
                   int64_t max_mem, int device, double* d_out, int64_t* perm_out, double* prefix_out,
                   int64_t* sign_out, b2d_run_info* info, int64_t* fail_index) {
  if (!a || !prefix_out) return set_err(B2D_ERR_USAGE, "null argument");
  if (dtype != B2D_F64 && dtype != B2D_F32) return set_err(B2D_ERR_USAGE, "dtype code %d", dtype);
  const int esz = dtype == B2D_F64 ? 8 : 4;
  if (num_blocks <= 0 && max_mem <= 0)
    return set_err(B2D_ERR_USAGE, "either max_mem or num_blocks is required");
  if (num_blocks <= 0 && max_mem < 3 * esz)
    return set_err(B2D_ERR_USAGE, "budget %lld B below minimum %d B", (long long)max_mem, 3 * esz);
  auto t0 = std::chrono::steady_clock::now();
  Ctx* c = nullptr;
  int rc = create(device, m, mode, &c);
  if (rc) return rc;
  rc = factor_host(c, a, lda, dtype, 0);
  b2d_run_info local{};
  if (rc == B2D_OK) rc = fetch(c, d_out, prefix_out, fail_index, &local);
  destroy(c);
  if (rc != B2D_OK && rc != B2D_ERR_NOT_SPD) return rc;
  fill_ref_info(&local, m, num_blocks, max_mem, esz);
  local.wall_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  if (info) *info = local;
  if (rc == B2D_OK) {
    if (perm_out)
      for (int64_t g = 0; g < m; ++g) perm_out[g] = g;
    if (sign_out)
      for (int64_t g = 0; g < m; ++g) sign_out[g] = 1;
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
