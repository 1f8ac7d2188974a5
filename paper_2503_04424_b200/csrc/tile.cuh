// Tile geometry, HBM layout and sm_100a PTX helpers shared by every kernel of the engine.
//
// HBM layout ("packed lower tile triangle"): the n_pad x n_pad matrix (n padded to a multiple
// of T = 128 with an identity tail) is cut into nt x nt tiles; only tiles (i, j) with i >= j
// are stored, tile-column by tile-column, so tile-column j (the panel of step j) is one
// contiguous run of (nt - j) tiles:
//     tile_index(i, j) = j*nt - j*(j-1)/2 + (i - j)
// Each tile is 128 x 128 doubles (128 KB) in the "octet" layout: the 16 column-octets are
// stored one after another, each octet row-major (128 rows x 8 doubles), with the 8 columns of
// an octet permuted so that columns q and q+4 sit side by side:
//     elem(r, c) = (c >> 3) * 1024 + r * 8 + perm8(c & 7),   perm8(c) = ((c & 3) << 1) | (c >> 2)
// A warp's DMMA m8n8k4 A- or B-fragments for two consecutive k-steps are then ONE conflict-free
// 16-byte shared-memory load per lane (512 contiguous bytes per warp), and a k-chunk of 16
// columns is a single contiguous 16 KB run that one cp.async.bulk moves into shared memory.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace b2d {

constexpr int T = 128;                 // tile edge
constexpr int TILE_ELEMS = T * T;      // 16384 doubles
constexpr int TILE_BYTES = TILE_ELEMS * 8;
constexpr int OCTET_ELEMS = T * 8;     // 1024 doubles per column-octet

__host__ __device__ __forceinline__ int perm8(int c) { return ((c & 3) << 1) | (c >> 2); }
__host__ __device__ __forceinline__ int iperm8(int p) { return (p >> 1) | ((p & 1) << 2); }
__host__ __device__ __forceinline__ int elem(int r, int c) {
  return ((c >> 3) << 10) + (r << 3) + perm8(c & 7);
}
__host__ __device__ __forceinline__ int64_t col_offset(int j, int nt) {
  return (int64_t)j * nt - (int64_t)j * (j - 1) / 2;
}
__host__ __device__ __forceinline__ int64_t tile_index(int i, int j, int nt) {
  return col_offset(j, nt) + (i - j);
}
__host__ __device__ __forceinline__ int64_t n_packed_tiles(int nt) {
  return (int64_t)nt * (nt + 1) / 2;
}

constexpr int MAX_PEERS = 8;  // ranks whose tile grids one map can address (one NVLink domain)

// Where a tile lives: the packed lower triangle (packed_nt > 0) or a row-major grid of tiles
// with `ld` tiles per row (out-of-core blocks).
// A sub-block of the packed triangle (a diagonal block, or the panel below it) is addressed with
// block-local indices through (roff, coff).
// Row-cyclic storage over several ranks (rmod = ranks): tile row i belongs to rank i % rmod at
// local row i / rmod, either gathered into one buffer of rank-major blocks of rstride rows
// (base, npeer = 0), or read in place from each rank's own grid over NVLink peer memory
// (npeer = rmod, peer[r] = rank r's grid as mapped into this process).
struct TileMap {
  double* base;
  int64_t ld;
  int packed_nt;
  int rmod;
  int64_t rstride;
  int npeer;
  double* peer[MAX_PEERS];
  int roff = 0, coff = 0;  // packed triangle: tile (i, j) of the map is packed tile (i + roff, j + coff)
  __host__ __device__ __forceinline__ double* tile(int i, int j) const {
    if (packed_nt > 0) return base + tile_index(i + roff, j + coff, packed_nt) * TILE_ELEMS;
    if (npeer > 0) return peer[i % rmod] + ((int64_t)(i / rmod) * ld + j) * TILE_ELEMS;
    const int64_t r = rmod > 0 ? (int64_t)(i % rmod) * rstride + i / rmod : (int64_t)i;
    return base + (r * ld + j) * TILE_ELEMS;
  }
};

// Output-tile set of a GEMM launch: columns j in [j0, j1), rows i in [lo(j), i1) with
// lo(j) = max(i0, j + row_off) when `lower`, else i0.  Rows may be local indices of a
// row-cyclic distribution (global row = i * stride + off; stride 0 means 1): then `lower`
// keeps global rows >= j + row_off, i.e. lo(j) = max(i0, ceil((j + row_off - off) / stride)).
// CTAs walk column bands of G tiles; inside a band the triangular head first (rows below the
// band's last lo), then row blocks of G rows (column-major inside a block), so a wave of ~148
// CTAs touches ~2-3 G x G super-tiles and its A/B operand tiles stay L2-resident.
// Bijective onto the set (tests/test_tile_order.py).
struct TileSet {
  int i0, i1, j0, j1, lower, row_off;
  int stride, off;
  __host__ __device__ __forceinline__ int lo(int j) const {
    if (!lower) return i0;
    const int x = j + row_off - off;
    int l = x;
    if (stride > 1) l = x <= 0 ? -((-x) / stride) : (x + stride - 1) / stride;  // no division on the
    return l > i0 ? l : i0;                                                         // single-GPU path
  }
  __host__ __device__ inline int64_t count() const {
    int64_t n = 0;
    for (int j = j0; j < j1; ++j) n += i1 > lo(j) ? i1 - lo(j) : 0;
    return n;
  }
};

__host__ __device__ inline void tile_order(int64_t b, const TileSet& s, int G, int* out_i, int* out_j) {
  for (int jb0 = s.j0; jb0 < s.j1; jb0 += G) {
    const int wb = (s.j1 - jb0) < G ? (s.j1 - jb0) : G;
    int head_end = s.lo(jb0 + wb - 1);
    if (head_end > s.i1) head_end = s.i1;
    int64_t tri = 0;
    for (int j = jb0; j < jb0 + wb; ++j) tri += head_end > s.lo(j) ? head_end - s.lo(j) : 0;
    const int64_t rows = s.i1 > head_end ? s.i1 - head_end : 0;
    const int64_t band = tri + rows * wb;
    if (b >= band) { b -= band; continue; }
    if (b < tri) {
      for (int j = jb0; j < jb0 + wb; ++j) {
        const int cnt = head_end > s.lo(j) ? head_end - s.lo(j) : 0;
        if (b < cnt) { *out_i = s.lo(j) + (int)b; *out_j = j; return; }
        b -= cnt;
      }
    }
    b -= tri;
    const int64_t rb = b / ((int64_t)G * wb);
    const int64_t e = b - rb * G * wb;
    const int64_t rows_here = (rows - rb * G) < G ? (rows - rb * G) : G;
    *out_j = jb0 + (int)(e / rows_here);
    *out_i = head_end + (int)(rb * G + e % rows_here);
    return;
  }
  *out_i = -1;
  *out_j = -1;
}

// ------------------------------------------------------------------ PTX helpers (sm_90+)

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t addr = smem_u32(bar);
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(addr),
      "r"(parity)
      : "memory");
}

// 1-D bulk async copy global -> shared (TMA engine, SASS UBLKCP), completes tx on `bar`.
__device__ __forceinline__ void bulk_g2s(void* dst_smem, const void* src_gmem, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_u32(dst_smem)),
      "l"(src_gmem), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// FP64 tensor-core MMA (SASS DMMA.8x8x4): D = A(8x4, row) * B(4x8, col) + C.
//   a = A[lane>>2][lane&3], b = B[k=lane&3][n=lane>>2], c = C[lane>>2][2*(lane&3) + {0,1}]
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

}  // namespace b2d
