// Multi-device MEMDET in one process (included by engine.cu inside namespace b2d): the drop-in
// entry's `devices=[...]` / b2d_memdet_sym(devices, ndev).  SURVEY §8(e), memdet.py:322-389.
//
// Layout: 1-D block-cyclic over outer panels.  The lower tile triangle is cut into outer panels
// of W tile-columns (panel s = tile-columns [sW, sW + W)); panel s lives on rank s mod P as a
// grid of its rows [sW, nt) x W tiles.  The deal balances the triangle (nt / W >> P panels) and
// makes host ingest sharded: panel s is the file's row strips [sW*128, (sW + W)*128) from
// column sW*128 on, so each rank reads 1/P of the upper triangle from host memory and never
// holds the matrix.  Communication volume: every rank receives every panel's
// rows below its own columns once -- at most n^2/2 doubles per rank per factorisation (C4 at
// P = 8: <= 69 GB, ~0.1 s of NVLink at 700 GB/s, against 2.7 s of DMMA work per rank); a 2-D
// P_r x P_c grid would cut that by ~sqrt(P) but adds a second broadcast and a row reduction per
// step, and with NVSwitch giving every pair full bandwidth the volume is not the bound.
//
// Step s, on every rank (one host thread per rank, enqueue only):
//   owner of s:  factor panel s on s_main / s_mid (potrf chain, in-panel solves and updates,
//                rows below left-looking per column -- the single-device panel code on the
//                panel's grid), record ev_ready[s];
//   others:      s_copy waits ev_ready[s] (a cross-device event) and pulls the panel's rows
//                below its first own column into a double-buffered receive grid
//                (cudaMemcpyPeerAsync over NVLink);
//   owner of s+1: next-cols update of panel s+1 with panel s (s_main: its factor is next);
//   everyone:    the rest of its own panels right of s+1 (s_side, low priority) -- overlapping
//                the factor of panel s+1 on its owner (one-panel look-ahead).
// Ranks synchronise on the host only for event ordering (a rank waits until the owner's thread
// has RECORDED ev_ready[s] before enqueueing a wait on it); the device work is ordered by events
// alone.  2 log L_ii land in the owners' ell vectors and are gathered into rank 0's, which runs
// the prefix scan.
//
// Block-pivoted LDL (memdet_ldl, _ldl.pyx:21-61): the outer panels are the reference's blocks
// (b a multiple of 128, or one block), so stage k is panel k on rank k mod P: its owner factors
// the diagonal block with block-local 1x1 pivoting (ldl_factor_block, the single-device kernels)
// and forms the stage's row-k blocks -- permuted, solved, and D^{-1}-scaled (memdet.py:361-371) --
// as full-height grids that the other ranks copy; every trailing tile receives the same update
// (same operands, K and order) as on one device, so perm, D and the prefixes are bit-identical
// to the single-device run.  Distributing whole reference blocks balances poorly when there are
// few blocks per rank (C3: 16 blocks over 8 ranks); sub-block distribution with a gather of each
// block column to its stage owner is the next step.  Ranks may share a device (tests run P = 2, 3 on one GPU): every dependency
// is a stream-event wait, never a kernel spinning on another rank's kernel.

struct MRank {
  Ctx* c = nullptr;
  std::map<int, double*> pan;  // owned step -> panel grid (rows [k0, nt) x W tiles)
  double* recv[2] = {};
  // block-pivoted LDL: each owned stage's row-k blocks, unscaled / D^{-1}-scaled (rows [ke, nt) x W
  // tiles, never overwritten, so the other ranks may copy them any time); received ones in
  // recv_u / recv_s (full height, tile (i, p) at base + (i W + p))
  std::map<int, double*> pu, ps;
  double *recv_u[2] = {}, *recv_s[2] = {};
  int first_own = INT_MAX;     // first owned step
  std::vector<cudaEvent_t> ev_ready, ev_in, ev_src_done;
  cudaEvent_t ev_free[2] = {};
  cudaEvent_t ev_done = nullptr;
};

struct MCtx {
  int P = 0;
  int64_t m = 0;
  int nt = 0, W = 16, mode = 0;
  bool ldl = false;  // block-pivoted LDL: panels = the reference's blocks
  std::vector<int> devs;
  std::vector<int> bounds;  // panel boundaries (tile-columns), nsteps + 1 entries
  std::vector<MRank> r;
  // host event-ordering fabric
  std::mutex mu;
  std::condition_variable cv;
  std::vector<int> recorded;  // per step: the owner's thread has recorded ev_ready[s]
  int nsteps() const { return (int)bounds.size() - 1; }
  int owner(int s) const { return s % P; }
};

static void mg_destroy(MCtx* M) {
  if (!M) return;
  for (auto& R : M->r) {
    if (!R.c) continue;
    cudaSetDevice(R.c->device);
    cudaDeviceSynchronize();
    for (auto& kv : R.pan) cudaFree(kv.second);
    for (double* q : R.recv) cudaFree(q);
    for (auto* mp : {&R.pu, &R.ps})
      for (auto& kv : *mp) cudaFree(kv.second);
    for (double* q : {R.recv_u[0], R.recv_u[1], R.recv_s[0], R.recv_s[1]}) cudaFree(q);
    for (auto* v : {&R.ev_ready, &R.ev_in, &R.ev_src_done})
      for (auto e : *v)
        if (e) cudaEventDestroy(e);
    for (auto e : R.ev_free)
      if (e) cudaEventDestroy(e);
    if (R.ev_done) cudaEventDestroy(R.ev_done);
    destroy(R.c);
  }
  delete M;
}

// A per-device shell context: streams, events, inverse diagonal tiles, ell / diag / prefix,
// fail flag (no matrix storage).
static int create_shell(int device, int64_t m, int mode, Ctx** out) {
  CUDA_TRY(cudaSetDevice(device));
  if (int rc = configure_kernels()) return rc;
  Ctx* c = new Ctx();
  c->device = device;
  c->m = m;
  c->mode = mode;
  c->W_TILES = panel_tiles_default();
  c->nt = (int)((m + T - 1) / T);
  const int64_t npad = (int64_t)c->nt * T;
  bool ok = cudaMalloc((void**)&c->inv, (size_t)c->nt * TILE_BYTES) == cudaSuccess &&
            cudaMalloc((void**)&c->ell, npad * 8) == cudaSuccess && cudaMalloc((void**)&c->diag, npad * 8) == cudaSuccess &&
            cudaMalloc((void**)&c->prefix, npad * 8) == cudaSuccess && cudaMalloc((void**)&c->fail, 8) == cudaSuccess;
  if (!ok) {
    destroy(c);
    return set_err(B2D_ERR_NOMEM, "multi-device: shell context allocation failed on device %d", device);
  }
  if (int rc = create_streams_events(c)) {
    destroy(c);
    return rc;
  }
  *out = c;
  return B2D_OK;
}

static int mg_create(const int* devices, int ndev, int64_t m, int mode, const b2d_options* opt, MCtx** out) {
  if (mode != B2D_MODE_CHOLESKY && mode != B2D_MODE_LDL_NOPIV && mode != B2D_MODE_LDL_PIV)
    return set_err(B2D_ERR_UNSUPPORTED, "multi-device runs Cholesky and LDL (mode %d requested)", mode);
  int64_t ref_nb = 1, ref_b = m, ref_tail = m;
  if (mode == B2D_MODE_LDL_PIV) {
    if (opt && opt->f32_arith)
      return set_err(B2D_ERR_UNSUPPORTED, "float32 memdet_ldl (f32 arithmetic) is single-device");
    int64_t nb0 = 1;
    if (opt && opt->num_blocks > 0) nb0 = opt->num_blocks;
    else if (opt && opt->max_mem > 0) nb0 = ref_select_blocking(m, opt->max_mem, 8);
    ref_layout(m, std::max<int64_t>(1, nb0), &ref_nb, &ref_b, &ref_tail);
    if (ref_nb > 1 && ref_b % T != 0)
      return set_err(B2D_ERR_UNSUPPORTED,
                     "multi-device block-pivoted LDL needs the reference's blocks on 128-row boundaries "
                     "(b = %lld; use num_blocks with m / num_blocks a multiple of 128, or one device)",
                     (long long)ref_b);
  }
  int nvis = 0;
  if (cudaGetDeviceCount(&nvis) != cudaSuccess || nvis == 0)
    return set_err(B2D_ERR_CUDA, "no CUDA device visible: the B200 engine has no CPU fallback");
  for (int d = 0; d < ndev; ++d)
    if (devices[d] < 0 || devices[d] >= nvis) return set_err(B2D_ERR_USAGE, "bad device %d", devices[d]);
  MCtx* M = new MCtx();
  M->P = ndev;
  M->m = m;
  M->mode = mode;
  M->devs.assign(devices, devices + ndev);
  M->nt = (int)((m + T - 1) / T);
  M->ldl = mode == B2D_MODE_LDL_PIV;
  M->W = M->ldl ? (int)((ref_b + T - 1) / T) : std::max(1, env_int("B2D_MG_PANEL_TILES", 16));
  for (int k = 0; k < M->nt; k += M->W) M->bounds.push_back(k);
  M->bounds.push_back(M->nt);
  const int S = M->nsteps(), nt = M->nt, W = M->W;
  // peer access between distinct devices (NVLink / NVSwitch); a rank's panel is read by copy
  for (int a : M->devs)
    for (int b : M->devs) {
      if (a == b) continue;
      int can = 0;
      cudaDeviceCanAccessPeer(&can, a, b);
      if (can) {
        cudaSetDevice(a);
        const cudaError_t e = cudaDeviceEnablePeerAccess(b, 0);
        if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) {
          cudaGetLastError();
        }
        cudaGetLastError();
      }
    }
  M->r.resize(ndev);
  const int64_t budget = opt && opt->hbm_budget > 0 ? opt->hbm_budget : INT64_MAX;
  for (int d = 0; d < ndev; ++d) {
    MRank& R = M->r[d];
    if (int rc = create_shell(M->devs[d], m, mode, &R.c)) {
      mg_destroy(M);
      return rc;
    }
    size_t need = 2 * (size_t)nt * W * TILE_BYTES + (size_t)NSTAGE * T * nt * T * 8;
    const int64_t ldb = (int64_t)W * T;
    if (M->ldl) {  // row-k block grids (2 per own stage + 4 receive), the dense block and its state
      need += 4 * (size_t)nt * W * TILE_BYTES + (size_t)ldb * ldb * 9 + (size_t)(m + 8 * ldb) * 8 +
              2 * (size_t)W * TILE_BYTES;
      for (int s = d; s < S; s += ndev) need += 2 * (size_t)(nt - M->bounds[s + 1]) * W * TILE_BYTES;
    }
    for (int s = d; s < S; s += ndev) need += (size_t)(nt - M->bounds[s]) * W * TILE_BYTES;
    if ((int64_t)need > budget) {
      mg_destroy(M);
      return set_err(B2D_ERR_NOMEM, "multi-device: rank %d needs %.2f GB of HBM, the budget is %.2f GB", d,
                     need / 1e9, budget / 1e9);
    }
    cudaSetDevice(M->devs[d]);
    bool ok = true;
    for (int s = d; s < S && ok; s += ndev) {
      double* p = nullptr;
      ok = cudaMalloc((void**)&p, (size_t)(nt - M->bounds[s]) * W * TILE_BYTES) == cudaSuccess;
      R.pan[s] = p;
      R.first_own = std::min(R.first_own, s);
    }
    if (ndev > 1)
      for (double*& q : R.recv) ok = ok && cudaMalloc((void**)&q, (size_t)nt * W * TILE_BYTES) == cudaSuccess;
    for (int b = 0; b < NSTAGE && ok; ++b) ok = cudaMalloc(&R.c->strip[b], (size_t)T * nt * T * 8) == cudaSuccess;
    if (M->ldl && ok) {
      // the block factor's state (ldl_factor_block), as the single-device in-core LDL has it
      Ooc& o = R.c->o;
      o.nb = (int)ref_nb;
      o.b = ref_b;
      o.tail = ref_tail;
      o.nbt = W;
      const size_t tiles = (size_t)nt * W * TILE_BYTES;
      for (int s = d; s < S && ok; s += ndev) {
        const size_t rows = (size_t)(nt - M->bounds[s + 1]);
        double *u = nullptr, *v = nullptr;
        if (rows > 0)
          ok = cudaMalloc((void**)&u, rows * W * TILE_BYTES) == cudaSuccess &&
               cudaMalloc((void**)&v, rows * W * TILE_BYTES) == cudaSuccess;
        R.pu[s] = u;
        R.ps[s] = v;
      }
      if (ndev > 1)
        for (double** q : {&R.recv_u[0], &R.recv_u[1], &R.recv_s[0], &R.recv_s[1]})
          ok = ok && cudaMalloc((void**)q, tiles) == cudaSuccess;
      ok = ok && cudaMalloc((void**)&o.dense, (size_t)ldb * ldb * 8) == cudaSuccess &&
           cudaMalloc((void**)&o.swaps, (size_t)ldb * 8) == cudaSuccess &&
           cudaMalloc((void**)&o.perm_local, (size_t)ldb * 8) == cudaSuccess &&
           cudaMalloc((void**)&o.perm_global, (size_t)(m + ldb) * 8) == cudaSuccess &&
           cudaMalloc((void**)&o.dblk, (size_t)ldb * 8) == cudaSuccess && cudaMalloc((void**)&o.amax, 8) == cudaSuccess &&
           cudaMalloc((void**)&o.ltag, (size_t)ldb * ldb) == cudaSuccess &&
           cudaMalloc((void**)&o.lC, (size_t)LDL_NB * ldb * 8) == cudaSuccess &&
           cudaMalloc((void**)&o.lW, (size_t)LDL_NB * ldb * 8) == cudaSuccess &&
           cudaMalloc((void**)&o.ldiag, (size_t)ldb * 8) == cudaSuccess &&
           cudaMalloc((void**)&o.lcol, (size_t)ldb * 8) == cudaSuccess &&
           cudaMalloc((void**)&o.inv_odd, (size_t)W * TILE_BYTES) == cudaSuccess &&
           cudaMalloc((void**)&o.perm_odd, (size_t)ldb * 8) == cudaSuccess &&
           cudaMalloc((void**)&o.dblk_odd, (size_t)ldb * 8) == cudaSuccess;
    }
    if (!ok) {
      const cudaError_t e = cudaGetLastError();
      size_t fb = 0, tb = 0;
      cudaMemGetInfo(&fb, &tb);
      mg_destroy(M);
      return set_err(B2D_ERR_NOMEM, "multi-device: allocation failed on device %d (rank %d, need %.2f GB, %.2f GB free): %s",
                     devices[d], d, need / 1e9, fb / 1e9, cudaGetErrorString(e));
    }
    for (auto* v : {&R.ev_ready, &R.ev_in, &R.ev_src_done}) {
      v->resize(S);
      for (auto& e : *v) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    }
    for (auto& e : R.ev_free) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&R.ev_done, cudaEventDisableTiming);
  }
  *out = M;
  return B2D_OK;
}

// Panel s's grid as a map over global tile indices: tile (i, j) at base + ((i - k0) W + (j - k0)).
static TileMap mg_panel_map(const MCtx* M, double* base, int s) {
  const int k0 = M->bounds[s];
  TileMap t{};
  t.base = base - ((int64_t)k0 * M->W + k0) * TILE_ELEMS;
  t.ld = M->W;
  return t;
}

// Pack panel s of rank d from the input: row strips J in [k0, ke) (file rows [128 J, 128 J + 128),
// columns from 128 J on) into tile-column J of the panel grid.  Host inputs stream through the
// rank's staging strips (pinned: DMA; pageable: the library's staging threads); device inputs
// are read in place (peer reads when the input lives on another device).
static int mg_ingest_panel(MCtx* M, int d, int s, const void* a, int64_t lda, int dtype, bool host) {
  MRank& R = M->r[d];
  Ctx* c = R.c;
  const int k0 = M->bounds[s], ke = M->bounds[s + 1], nt = M->nt;
  const int64_t npad = (int64_t)nt * T;
  const size_t esz = dtype == B2D_F64 ? 8 : 4;
  const TileMap pm = mg_panel_map(M, R.pan.at(s), s);
  for (int J = k0; J < ke; ++J) {
    const TileSet set{J, nt, J, J + 1, 1, 0, 0, 0};
    const unsigned n = (unsigned)set.count();
    if (!host) {
      if (dtype == B2D_F64)
        pack_set_kernel<double><<<n, PACK_THREADS, PACK_SMEM, c->s_pack>>>((const double*)a, lda, 0, M->m, pm, set);
      else
        pack_set_kernel<float><<<n, PACK_THREADS, PACK_SMEM, c->s_pack>>>((const float*)a, lda, 0, M->m, pm, set);
      c->launches++;
      continue;
    }
    const int b = (int)(c->hseq_strip++ % NSTAGE);
    const int64_t r0 = (int64_t)J * T;
    const int64_t rows = std::max<int64_t>(0, std::min<int64_t>(T, M->m - r0));
    const int64_t cols = M->m - r0;
    if (c->strip_used[b]) cudaStreamWaitEvent(c->s_copy, c->ev_stage[b], 0);
    if (rows > 0 && cols > 0) {
      const char* src = (const char*)a + (size_t)(r0 * lda + r0) * esz;
      char* dst = (char*)c->strip[b] + (size_t)r0 * esz;
      if (int rc = h2d_2d(c, dst, (size_t)npad * esz, src, (size_t)lda * esz, (size_t)cols * esz, (size_t)rows, c->s_copy))
        return rc;
      c->h2d += rows * cols * (int64_t)esz;
    }
    cudaEventRecord(c->ev_copied[b], c->s_copy);
    cudaStreamWaitEvent(c->s_pack, c->ev_copied[b], 0);
    if (dtype == B2D_F64)
      pack_set_kernel<double><<<n, PACK_THREADS, PACK_SMEM, c->s_pack>>>((const double*)c->strip[b], npad, r0, M->m,
                                                                         pm, set);
    else
      pack_set_kernel<float><<<n, PACK_THREADS, PACK_SMEM, c->s_pack>>>((const float*)c->strip[b], npad, r0, M->m,
                                                                        pm, set);
    c->launches++;
    cudaEventRecord(c->ev_stage[b], c->s_pack);
    c->strip_used[b] = true;
  }
  cudaEventRecord(R.ev_in[s], c->s_pack);
  return B2D_OK;
}

// Factor panel s on its owner (the single-device panel loop, on the panel grid):
// potrf + in-block solve and update on s_main (the chain), rows below left-looking per column on
// s_mid; ev_ready[s] on s_mid once the whole panel is solved.
static void mg_factor_panel(MCtx* M, int d, int s) {
  MRank& R = M->r[d];
  Ctx* c = R.c;
  const int k0 = M->bounds[s], ke = M->bounds[s + 1], nt = M->nt;
  const FactorTarget ft{mg_panel_map(M, R.pan.at(s), s), nt, 0};
  for (int p = k0; p < ke; ++p) {
    launch_potrf(c, c->s_main, ft, p);
    launch_trsm(c, c->s_main, ft, p, p + 1, ke);
    cudaEventRecord(c->ev_m2s, c->s_main);
    cudaStreamWaitEvent(c->s_mid, c->ev_m2s, 0);
    if (ke < nt && p > k0) launch_update_set(c, c->s_mid, ft, TileSet{ke, nt, p, p + 1, 0, 0}, k0, p, false);
    launch_trsm(c, c->s_mid, ft, p, ke, nt);
    if (p + 1 < ke) launch_update_set(c, c->s_main, ft, TileSet{p + 1, ke, p + 1, ke, 1, 0}, p, p + 1, false);
  }
  cudaEventRecord(c->ev_join, c->s_main);
  cudaStreamWaitEvent(c->s_mid, c->ev_join, 0);
  cudaEventRecord(R.ev_ready[s], c->s_mid);
}

// Block-pivoted LDL stage s on its owner (run_ldl_incore's stage on the panel grid): factor the
// diagonal block with block-local 1x1 pivots, then the row-k blocks below it -- permuted by the
// stage's pivots (memdet.py:365-366), solved with the unit factor (dense.py:94-99) into pu and
// D^{-1}-scaled into ps (memdet.py:368-371), rows indexed by global tile row.
static int mg_ldl_stage(MCtx* M, int d, int s) {
  MRank& R = M->r[d];
  Ctx* c = R.c;
  Ooc& o = c->o;
  const int k0 = M->bounds[s], ke = M->bounds[s + 1], nt = M->nt, W = M->W, kb = ke - k0;
  const TileMap blk{R.pan.at(s), W, 0};  // block-local tile (I, J) of the diagonal block
  if (int rc = ldl_factor_block(c, blk, s, c->s_main)) return rc;
  if (ke < nt) {
    const double* inv_k = (s & 1) && o.inv_odd ? o.inv_odd : c->inv;
    const TileMap src{R.pan.at(s) + (size_t)kb * W * TILE_ELEMS, W, 0};  // panel rows [ke, nt)
    const TileMap pu{R.pu.at(s), W, 0};
    const TileMap ps{R.ps.at(s), W, 0};
    permute_cols_kernel<<<2048, 256, 0, c->s_main>>>(src, pu, nt - ke, kb, o.size(s), o.perm_of(s));
    trsm_panel(c, c->s_main, pu, nt - ke, blk, kb, inv_k);
    scale_cols_kernel<<<2048, 256, 0, c->s_main>>>(pu, ps, nt - ke, kb, o.size(s), o.dblk_of(s));
    c->launches += 2;
  }
  cudaEventRecord(R.ev_ready[s], c->s_main);
  return B2D_OK;
}

// T(own panel t) -= L(., s) L(., s)^T over the tiles of t (rows >= its first column), K = panel s.
// LDL: T -= (L D^{-1})(., s) L(., s)^T from the stage's scaled / unscaled grids (a = ps, b = pu).
static void mg_update(MCtx* M, int d, cudaStream_t st, const TileMap& src, int s, int t,
                      const TileMap* scaled = nullptr) {
  MRank& R = M->r[d];
  const int k0 = M->bounds[s], ke = M->bounds[s + 1], t0 = M->bounds[t], t1 = M->bounds[t + 1];
  GemmTask u{};
  u.a = u.b = src;
  u.p0 = k0;
  u.p1 = ke;
  if (scaled) {
    u.a = *scaled;
    u.p0 = 0;
    u.p1 = ke - k0;
  }
  u.c = mg_panel_map(M, R.pan.at(t), t);
  u.out = TileSet{t0, M->nt, t0, t1, 1, 0};
  cudaStreamWaitEvent(st, R.ev_in[t], 0);  // the target panel has arrived
  launch_gemm(R.c, st, MODE_UPDATE, u, s + 1 != t, (double)u.out.count() * 2.0 * T * T * (double)(ke - k0) * T);
}

static void mg_wait_recorded(MCtx* M, int s) {
  std::unique_lock<std::mutex> lk(M->mu);
  M->cv.wait(lk, [&] { return M->recorded[s] != 0; });
}

// Everything rank d enqueues for one factorisation (runs on its own host thread).
static int mg_rank_run(MCtx* M, int d, const void* a, int64_t lda, int dtype, bool host, cudaEvent_t start) {
  MRank& R = M->r[d];
  Ctx* c = R.c;
  CUDA_TRY(cudaSetDevice(c->device));
  const int S = M->nsteps(), nt = M->nt, P = M->P;
  for (cudaStream_t st : {c->s_main, c->s_mid, c->s_side, c->s_copy, c->s_pack}) cudaStreamWaitEvent(st, start, 0);
  if (d != 0) {  // rank 0's vectors are cleared before `start` (other ranks copy into them)
    cudaMemsetAsync(c->fail, 0xff, 8, c->s_main);
    cudaMemsetAsync(c->ell, 0, (size_t)nt * T * 8, c->s_main);
    cudaMemsetAsync(c->diag, 0, (size_t)nt * T * 8, c->s_main);
  }
  int rc = B2D_OK;
  for (auto& kv : R.pan)
    if ((rc = mg_ingest_panel(M, d, kv.first, a, lda, dtype, host))) break;
  bool used[2] = {false, false};
  for (int s = 0; s < S && !rc; ++s) {
    const int o = M->owner(s);
    const bool own = o == d;
    const int ke = M->bounds[s + 1];
    if (own) {
      cudaStreamWaitEvent(c->s_main, R.ev_in[s], 0);                    // ingested
      if (s >= 2) cudaStreamWaitEvent(c->s_main, R.ev_src_done[s - 2], 0);  // rest updates of s-2
      if (M->ldl) {
        if ((rc = mg_ldl_stage(M, d, s))) {
          std::lock_guard<std::mutex> lk(M->mu);
          M->recorded[s] = 1;
          M->cv.notify_all();
          break;
        }
      } else {
        mg_factor_panel(M, d, s);
      }
      {
        std::lock_guard<std::mutex> lk(M->mu);
        M->recorded[s] = 1;
      }
      M->cv.notify_all();
    }
    if (s + 1 >= S) break;
    // does this rank own a panel right of s?
    int last_own = -1;
    for (auto& kv : R.pan) last_own = std::max(last_own, kv.first);
    if (last_own <= s) {
      cudaEventRecord(R.ev_src_done[s], c->s_side);
      continue;
    }
    TileMap src, src_s;
    cudaEvent_t src_ev;
    if (own) {
      src = mg_panel_map(M, R.pan.at(s), s);
      if (M->ldl) {  // rows indexed by global tile row: base shifted back by ke rows
        src = TileMap{R.pu.at(s) - (size_t)ke * M->W * TILE_ELEMS, M->W, 0};
        src_s = TileMap{R.ps.at(s) - (size_t)ke * M->W * TILE_ELEMS, M->W, 0};
      }
      src_ev = R.ev_ready[s];
    } else {
      mg_wait_recorded(M, s);
      // the panel's rows from this rank's first own column right of s
      int first = INT_MAX;
      for (auto& kv : R.pan)
        if (kv.first > s) first = std::min(first, M->bounds[kv.first]);
      const int k0 = M->bounds[s], W = M->W;
      double* buf = R.recv[s & 1];
      if (used[s & 1]) cudaStreamWaitEvent(c->s_copy, R.ev_free[s & 1], 0);
      cudaStreamWaitEvent(c->s_copy, M->r[o].ev_ready[s], 0);
      const size_t bytes = (size_t)(nt - first) * W * TILE_BYTES;
      auto pull = [&](double* dst, const double* from) -> int {
        if (c->device == M->r[o].c->device)
          CUDA_TRY(cudaMemcpyAsync(dst, from, bytes, cudaMemcpyDeviceToDevice, c->s_copy));
        else
          CUDA_TRY(cudaMemcpyPeerAsync(dst, c->device, from, M->r[o].c->device, bytes, c->s_copy));
        return B2D_OK;
      };
      if (M->ldl) {  // the stage's row-k block grids (rows indexed by global tile row)
        const size_t off = (size_t)first * W * TILE_ELEMS, soff = (size_t)(first - ke) * W * TILE_ELEMS;
        if ((rc = pull(R.recv_u[s & 1] + off, M->r[o].pu.at(s) + soff))) break;
        if ((rc = pull(R.recv_s[s & 1] + off, M->r[o].ps.at(s) + soff))) break;
        src = TileMap{R.recv_u[s & 1], W, 0};
        src_s = TileMap{R.recv_s[s & 1], W, 0};
      } else {
        const size_t off = (size_t)(first - k0) * W * TILE_ELEMS;
        if ((rc = pull(buf + off, M->r[o].pan.at(s) + off))) break;
        src = mg_panel_map(M, buf, s);
      }
      cudaEventRecord(c->ev_catch[s], c->s_copy);
      src_ev = c->ev_catch[s];
      used[s & 1] = true;
    }
    // next-cols: the panel the next factor needs (its owner's critical path)
    if (M->owner(s + 1) == d) {
      cudaStreamWaitEvent(c->s_main, src_ev, 0);
      mg_update(M, d, c->s_main, src, s, s + 1, M->ldl ? &src_s : nullptr);
      cudaEventRecord(c->ev_panel[s], c->s_main);
    }
    // the rest of this rank's panels (low priority, beside the next factor)
    cudaStreamWaitEvent(c->s_side, src_ev, 0);
    for (auto& kv : R.pan)
      if (kv.first > s + 1) mg_update(M, d, c->s_side, src, s, kv.first, M->ldl ? &src_s : nullptr);
    if (M->owner(s + 1) == d) cudaStreamWaitEvent(c->s_side, c->ev_panel[s], 0);
    cudaEventRecord(R.ev_src_done[s], c->s_side);
    if (!own) cudaEventRecord(R.ev_free[s & 1], c->s_side);
    (void)ke;
    (void)P;
  }
  // join, then the owners' 2 log L_ii / L_ii segments into rank 0's vectors
  cudaEventRecord(c->ev_join, c->s_side);
  cudaStreamWaitEvent(c->s_main, c->ev_join, 0);
  cudaEventRecord(c->ev_join, c->s_mid);
  cudaStreamWaitEvent(c->s_main, c->ev_join, 0);
  cudaEventRecord(c->ev_join, c->s_pack);
  cudaStreamWaitEvent(c->s_main, c->ev_join, 0);
  Ctx* c0 = M->r[0].c;
  if (d != 0 && !rc) {
    for (auto& kv : R.pan) {
      const int64_t g0 = (int64_t)M->bounds[kv.first] * T, g1 = std::min<int64_t>(M->m, (int64_t)M->bounds[kv.first + 1] * T);
      if (g1 <= g0) continue;
      std::vector<std::pair<void*, const void*>> segs{{c0->ell + g0, c->ell + g0}, {c0->diag + g0, c->diag + g0}};
      if (M->ldl) segs.emplace_back(c0->o.perm_global + g0, c->o.perm_global + g0);
      for (auto& sg : segs) {
        if (c->device == c0->device) cudaMemcpyAsync(sg.first, sg.second, (g1 - g0) * 8, cudaMemcpyDeviceToDevice, c->s_main);
        else cudaMemcpyPeerAsync(sg.first, c0->device, sg.second, c->device, (g1 - g0) * 8, c->s_main);
      }
    }
  }
  cudaEventRecord(R.ev_done, c->s_main);
  if (!rc) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) rc = set_err(B2D_ERR_CUDA, "multi-device rank %d: %s", d, cudaGetErrorString(e));
  }
  return rc;
}

static int mg_factor(MCtx* M, const void* a, int64_t lda, int dtype, bool host, cudaStream_t user) {
  if (dtype != B2D_F64 && dtype != B2D_F32) return set_err(B2D_ERR_USAGE, "dtype code %d", dtype);
  if (lda < M->m) return set_err(B2D_ERR_USAGE, "lda %lld < m", (long long)lda);
  Ctx* c0 = M->r[0].c;
  CUDA_TRY(cudaSetDevice(c0->device));
  for (auto& R : M->r) {
    R.c->launches = 0;
    R.c->h2d = R.c->d2h = 0;
    R.c->hseq_strip = 0;
    std::fill(std::begin(R.c->strip_used), std::end(R.c->strip_used), false);
    if (host) {
      cudaPointerAttributes pa{};
      const bool known = cudaPointerGetAttributes(&pa, a) == cudaSuccess;
      cudaGetLastError();
      const char* hs = getenv("B2D_HOST_STAGING");
      R.c->src_pageable = (hs ? atoi(hs) != 0 : true) && (!known || pa.type == cudaMemoryTypeUnregistered);
    }
  }
  c0->t0 = std::chrono::steady_clock::now();
  cudaMemsetAsync(c0->fail, 0xff, 8, user);
  cudaMemsetAsync(c0->ell, 0, (size_t)M->nt * T * 8, user);
  cudaMemsetAsync(c0->diag, 0, (size_t)M->nt * T * 8, user);
  cudaEventRecord(c0->ev_start, user);
  {
    std::lock_guard<std::mutex> lk(M->mu);
    M->recorded.assign(M->nsteps(), 0);
  }
  std::vector<int> rcs(M->P, B2D_OK);
  std::vector<std::string> errs(M->P);
  std::vector<std::thread> th;
  for (int d = 0; d < M->P; ++d)
    th.emplace_back([&, d] {
      rcs[d] = mg_rank_run(M, d, a, lda, dtype, host, c0->ev_start);
      if (rcs[d]) errs[d] = g_err;
      if (rcs[d]) {  // unblock ranks waiting on this rank's steps
        std::lock_guard<std::mutex> lk(M->mu);
        std::fill(M->recorded.begin(), M->recorded.end(), 1);
        M->cv.notify_all();
      }
    });
  for (auto& t : th) t.join();
  for (int d = 0; d < M->P; ++d)
    if (rcs[d]) {
      for (auto& R : M->r) {
        cudaSetDevice(R.c->device);
        cudaDeviceSynchronize();
      }
      cudaGetLastError();
      return set_err(rcs[d], "%s", errs[d].c_str());
    }
  cudaSetDevice(c0->device);
  for (int d = 1; d < M->P; ++d) cudaStreamWaitEvent(c0->s_main, M->r[d].ev_done, 0);
  prefix_kernel<<<1, 1024, 0, c0->s_main>>>(c0->ell, M->m, c0->prefix);
  c0->launches++;
  cudaEventRecord(c0->ev_join, c0->s_main);
  cudaStreamWaitEvent(user, c0->ev_join, 0);
  cudaEventRecord(c0->ev_stop, user);
  c0->pending = true;
  CUDA_TRY(cudaGetLastError());
  return B2D_OK;
}

static int mg_fetch(MCtx* M, double* d_out, double* prefix_out, int64_t* fail_index, b2d_run_info* info) {
  Ctx* c0 = M->r[0].c;
  if (!c0->pending) return set_err(B2D_ERR_USAGE, "no factorisation enqueued");
  CUDA_TRY(cudaSetDevice(c0->device));
  CUDA_TRY(cudaEventSynchronize(c0->ev_stop));
  c0->pending = false;
  unsigned long long fail = ULLONG_MAX;
  int64_t launches = 0, h2d = 0;
  for (auto& R : M->r) {
    unsigned long long f = ULLONG_MAX;
    cudaSetDevice(R.c->device);
    CUDA_TRY(cudaMemcpy(&f, R.c->fail, 8, cudaMemcpyDeviceToHost));
    fail = std::min(fail, f);
    launches += R.c->launches;
    h2d += R.c->h2d;
  }
  cudaSetDevice(c0->device);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, c0->ev_start, c0->ev_stop);
  if (prefix_out) CUDA_TRY(cudaMemcpy(prefix_out, c0->prefix, M->m * 8, cudaMemcpyDeviceToHost));
  if (d_out) {
    CUDA_TRY(cudaMemcpy(d_out, c0->diag, M->m * 8, cudaMemcpyDeviceToHost));
    if (M->mode == B2D_MODE_LDL_NOPIV)
      for (int64_t g = 0; g < M->m; ++g) d_out[g] = d_out[g] * d_out[g];
  }
  if (info) {
    info->m = M->m;
    info->tile = T;
    info->n_tiles = M->nt;
    info->h2d_bytes = h2d;
    info->d2h_bytes = (prefix_out ? M->m * 8 : 0) + (d_out ? M->m * 8 : 0);
    info->kernel_launches = launches;
    info->device_ms = ms;
    info->wall_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - c0->t0).count();
  }
  if (fail_index) *fail_index = fail == ULLONG_MAX ? -1 : (int64_t)fail;
  if (fail != ULLONG_MAX && M->ldl)
    return set_err(B2D_ERR_INDEFINITE, "LDL pivot %lld below tolerance (block-local 1x1 pivoting)", (long long)fail);
  if (fail != ULLONG_MAX)
    return set_err(B2D_ERR_NOT_SPD, "leading minor of order %lld is not positive definite", (long long)fail + 1);
  return B2D_OK;
}

static int mg_fetch_perm(MCtx* M, int64_t* perm) {
  if (!M->ldl) {
    for (int64_t g = 0; g < M->m; ++g) perm[g] = g;
    return B2D_OK;
  }
  CUDA_TRY(cudaSetDevice(M->r[0].c->device));
  CUDA_TRY(cudaMemcpy(perm, M->r[0].c->o.perm_global, M->m * 8, cudaMemcpyDeviceToHost));
  return B2D_OK;
}
