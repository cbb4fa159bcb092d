// K1 — tile/mask selection on bit-packed masks.
//
// Replaces, with exact bit semantics:
//   upscale_mask                       fileio.py:430-436
//   LevelMaskSet.from_pixel_mask       wavelets.py:272-306 (downmap2 :243, binary_dilate :214)
//   foveation window cascades          decoding.py:124-152, wavelets.py:295-304
//   footprint cascade                  wavelets.py:380-392
//   inclusion_grid + per-block any     wavelets.py:337-348, decoding.py:265-268
//   bytes_loaded / records_processed   decoding.py:212-234, :271-285
// and emits the compacted K2 block work list and the per-level K3 tile lists.
//
// Masks are rows of 32-bit words, bit i of word w = column 32w+i; bits past
// the row width are kept 0.  The full-resolution pixel mask is never
// materialised: its rows repeat, so only the mh distinct rows are built and
// row y reads row (y*mh)/H.
#include "wv_common.cuh"

namespace wv {
namespace {

__device__ __forceinline__ uint32_t last_word_mask(int cols, int w) {
  int rem = cols - 32 * w;
  return rem >= 32 ? 0xFFFFFFFFu : (rem <= 0 ? 0u : (0xFFFFFFFFu >> (32 - rem)));
}

// bits [c0, c1) of a word w as a mask
__device__ __forceinline__ uint32_t range_mask(int c0, int c1, int w) {
  int lo = max(c0 - 32 * w, 0), hi = min(c1 - 32 * w, 32);
  if (lo >= hi) return 0u;
  uint32_t m = hi >= 32 ? 0xFFFFFFFFu : ((1u << hi) - 1u);
  return m & (0xFFFFFFFFu << lo);
}

// OR of adjacent bit pairs of a 64-bit run -> 32 bits (2:1 column pooling)
__device__ __forceinline__ uint32_t pool_pairs(uint64_t v) {
  uint64_t t = (v | (v >> 1)) & 0x5555555555555555ull;
  t = (t | (t >> 1)) & 0x3333333333333333ull;
  t = (t | (t >> 2)) & 0x0F0F0F0F0F0F0F0Full;
  t = (t | (t >> 4)) & 0x00FF00FF00FF00FFull;
  t = (t | (t >> 8)) & 0x0000FFFF0000FFFFull;
  t = (t | (t >> 16)) & 0x00000000FFFFFFFFull;
  return (uint32_t)t;
}

// 16 bits -> 32 bits, each bit doubled (2x column upsampling)
__device__ __forceinline__ uint32_t double_bits(uint32_t x) {
  uint32_t t = x & 0xFFFFu;
  t = (t | (t << 8)) & 0x00FF00FFu;
  t = (t | (t << 4)) & 0x0F0F0F0Fu;
  t = (t | (t << 2)) & 0x33333333u;
  t = (t | (t << 1)) & 0x55555555u;
  return t | (t << 1);
}

// horizontal OR-spread by DIL columns
__device__ __forceinline__ uint32_t spread(uint32_t p, uint32_t c, uint32_t n) {
  uint32_t x = c;
#pragma unroll
  for (int k = 1; k <= DIL; ++k) x |= (c << k) | (p >> (32 - k)) | (c >> k) | (n << (32 - k));
  return x;
}

// horizontal AND-shrink by DIL columns (outside counts as set: pass ~0)
__device__ __forceinline__ uint32_t shrink(uint32_t p, uint32_t c, uint32_t n) {
  uint32_t x = c;
#pragma unroll
  for (int k = 1; k <= DIL; ++k) x &= ((c << k) | (p >> (32 - k))) & ((c >> k) | (n << (32 - k)));
  return x;
}

// ---------------------------------------------------------------- mask rows
// Distinct pixel-mask rows R[my] (nearest column map, fileio.py:435) and the
// row map rowmap[y] = (y*mh)/H (fileio.py:434).
__global__ void k_mask_rows(const wv_frame_args* __restrict__ fa, uint32_t* __restrict__ R,
                            uint32_t* __restrict__ rowmap, uint32_t* __restrict__ counters, int mh,
                            int mw, int W, int H, int wpr0, int full, uint32_t* __restrict__ mbits) {
  pdl_sync();
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  const uint8_t* __restrict__ mask = fa->d_mask;
  if (idx == 0) *fa->d_result = wv_frame_result{};
  if (idx < 64) counters[idx] = 0u;   // work-list counters of this call
  if (idx < H) rowmap[idx] = ((uint32_t)idx * (uint32_t)mh) / (uint32_t)H;
  {
    // the low-res mask as bit rows (direct cascade source)
    const int mwpr = (mw + 31) >> 5;
    if (!full && idx < mh * mwpr) {
      const int my = idx / mwpr, k = idx - (idx / mwpr) * mwpr;
      uint32_t b = 0;
      for (int i = 0; i < 32 && 32 * k + i < mw; ++i)
        b |= (mask[(uint64_t)my * mw + 32 * k + i] ? 1u : 0u) << i;
      mbits[idx] = b;
    }
  }
  if (idx >= mh * wpr0) return;
  const int my = idx / wpr0, w = idx % wpr0;
  // the word's pixels map to a few runs of mask columns: pixel x -> floor(x*mw/W)
  // (fileio.py:435); mask column mx starts at pixel ceil(mx*W/mw)
  const int x0 = 32 * w, x1 = min(x0 + 32, W);
  uint32_t bits = 0;
  int mx = (int)(((uint32_t)x0 * (uint32_t)mw) / (uint32_t)W);   // < 2^32 (checked on host)
  for (int xs = x0; xs < x1; ++mx) {
    const int nx = min(x1, (int)(((uint64_t)(mx + 1) * W + mw - 1) / mw));
    if (full || mask[(uint64_t)my * mw + mx]) bits |= range_mask(xs, nx, w);
    xs = nx;
  }
  R[idx] = bits;
}

// ------------------------------------------------------------- cascade step
// C_j = dilate4(downmap2(C_{j-1})) on a 32-row x 32-word output tile (each
// thread 4 words of one row): the pooled words of the tile plus a 4-row /
// 1-word apron are staged in shared memory once, then each thread ORs its
// 9-row neighbourhood.  The CTA that produces the final detail mask D_j also
// pools it into one bit per 32x32 cell (used by the block selection when
// block_size is 32).
constexpr int CT_R = 32, CT_W = 32, CT_TW = 8;   // tile rows, tile words, threads per row
#ifndef WV_K1_DIRECT
#define WV_K1_DIRECT 1     // all cascade levels in one launch as box ORs of the low-res mask (0: one launch per level)
#endif
#ifndef WV_K1_DIRECT_RPW_WARPS
#define WV_K1_DIRECT_RPW_WARPS 32   // warps per 32-row band of the direct cascade (one row each)
#endif
#ifndef WV_K1_FOV_RECT
#define WV_K1_FOV_RECT 1   // skip gaze-window cascade tiles outside the window's level-j bound
#endif   // tile rows, tile words, threads per row

struct CascadeArgs {
  int j, L, H;
  int rows, cols, wpr;        // output level j
  int prow_n, pcols, pwpr;    // source level j-1
  const uint32_t* src;        // j > 1: stack[j-1]
  uint64_t src_stride;        // words per batch mask
  const uint32_t* R;          // j == 1: pixel rows
  const uint32_t* rowmap;
  uint32_t* dst;
  uint64_t dst_stride;
  int nbatch;
  int batch[WV_MAX_LEVELS + 1];
  const wv_frame_args* fa;         // j == 1 foveated windows: fa->fovea[batch id - 1]
  int fov;                         // foveated: batch j also ANDs with batch 0
  uint32_t* pooled;                // one word per tile: bit w = any bit in (32 rows x word w)
  int pool_wpr;                    // tiles per row of the level
  const uint32_t* src_pooled;      // viewport, j > 1: level j-1's pooled occupancy (else null)
  int src_pool_wpr;
  int mh, mw;                      // j == 1: low-res mask size (fa->d_mask)
};

// Can the tile (rows r0.., words w0.. of level j, with its dilation apron)
// receive any set bit?  j == 1: the low-res mask cells under it; j > 1
// (viewport): level j-1's pooled occupancy.  A zero answer is exact: the
// cascade of an all-zero source region is zero (foveated windows are
// subsets of the request, so the test holds for every batch at j == 1).
__device__ bool cascade_tile_live(const CascadeArgs& a, int r0, int w0) {
  bool hit = false;
  if (a.j == 1) {
    const int py0 = max(0, 2 * (r0 - DIL)), py1 = min(a.prow_n, 2 * (r0 + CT_R + DIL));
    const int px0 = max(0, 64 * (w0 - 1)), px1 = min(a.pcols, 64 * (w0 + CT_W + 1));
    if (py0 < py1 && px0 < px1) {
      const int m0 = (int)(((uint32_t)py0 * (uint32_t)a.mh) / (uint32_t)a.prow_n);
      const int m1 = (int)(((uint32_t)(py1 - 1) * (uint32_t)a.mh) / (uint32_t)a.prow_n);
      const int c0 = (int)(((uint32_t)px0 * (uint32_t)a.mw) / (uint32_t)a.pcols);
      const int c1 = (int)(((uint32_t)(px1 - 1) * (uint32_t)a.mw) / (uint32_t)a.pcols);
      const int nc = c1 - c0 + 1, cells = (m1 - m0 + 1) * nc;
      const uint8_t* mask = a.fa->d_mask;
      for (int e = threadIdx.x; e < cells; e += blockDim.x)
        hit |= mask[(uint64_t)(m0 + e / nc) * a.mw + c0 + e % nc] != 0;
    }
  } else {
    const int sr0 = max(0, 2 * (r0 - DIL)), sr1 = min(a.prow_n, 2 * (r0 + CT_R + DIL));
    const int sw0 = max(0, 2 * (w0 - 1)), sw1 = min(a.pwpr, 2 * (w0 + CT_W + 1));
    if (sr0 < sr1 && sw0 < sw1) {
      const int t0 = sr0 / CT_R, t1 = (sr1 - 1) / CT_R, q0 = sw0 / CT_W, q1 = (sw1 - 1) / CT_W;
      const int nq = q1 - q0 + 1;
      for (int e = threadIdx.x; e < (t1 - t0 + 1) * nq; e += blockDim.x) {
        const int tr = t0 + e / nq, tq = q0 + e % nq;
        const int lo = max(sw0 - tq * CT_W, 0), hi = min(sw1 - tq * CT_W, 32);
        const uint32_t m = (hi >= 32 ? 0xFFFFFFFFu : ((1u << hi) - 1u)) & (0xFFFFFFFFu << lo);
        hit |= (a.src_pooled[(uint64_t)tr * a.src_pool_wpr + tq] & m) != 0u;
      }
    }
  }
  return __syncthreads_or(hit) != 0;
}

__device__ __forceinline__ uint32_t cas_src(const CascadeArgs& a, const int4& rect, int b,
                                            int rr, int ww) {
  if (ww >= a.pwpr || rr >= a.prow_n) return 0u;
  if (a.j == 1) {
    uint32_t v = a.R[(uint64_t)a.rowmap[rr] * a.pwpr + ww];
    if (b > 0) {
      if (rr < rect.x || rr >= rect.y) return 0u;
      v &= range_mask(rect.z, rect.w, ww);
    }
    return v;
  }
  return a.src[(uint64_t)b * a.src_stride + (uint64_t)rr * a.pwpr + ww];
}

// downmapped word at output level (row r, word w), both in range
__device__ __forceinline__ uint32_t cas_down(const CascadeArgs& a, const int4& rect, int b,
                                             int r, int w) {
  const uint32_t lo = cas_src(a, rect, b, 2 * r, 2 * w) | cas_src(a, rect, b, 2 * r + 1, 2 * w);
  const uint32_t hi =
      cas_src(a, rect, b, 2 * r, 2 * w + 1) | cas_src(a, rect, b, 2 * r + 1, 2 * w + 1);
  return pool_pairs((uint64_t)lo | ((uint64_t)hi << 32));
}

__global__ void __launch_bounds__(256) k_cascade(CascadeArgs a) {
  pdl_sync();
  __shared__ uint32_t dm[2][CT_R + 2 * DIL][CT_W + 2];
  __shared__ uint32_t vor[2][CT_R][CT_W + 2];
  __shared__ uint32_t pool[CT_W];
  const int b = a.batch[blockIdx.y];
  const bool both = a.fov && b == a.j;
  const bool final_mask = a.fov ? (b == a.j) : (b == 0);
  const int r0 = blockIdx.z * CT_R, w0 = blockIdx.x * CT_W;
  int4 rect = make_int4(0, 0, 0, 0);
  if (a.j == 1 && b > 0) {
    const int32_t* f = a.fa->fovea[b - 1];
    rect = make_int4(f[0], f[1], f[2], f[3]);
  }
  const int4 none = make_int4(0, 0, 0, 0);
  // a gaze-window batch (b > 0) lives inside its pixel window scaled to level
  // j and grown by the dilations: rows [r0 / 2^j - 8, r1 / 2^j + 8) (each
  // level halves, then dilates by DIL = 4; 9 with rounding), columns alike
  bool outside = false;
  if (WV_K1_FOV_RECT && b > 0) {
    const int32_t* f = a.fa->fovea[b - 1];
    const int s = a.j, up = (1 << a.j) - 1;
    const int lr0 = (f[0] >> s) - 9, lr1 = ((f[1] + up) >> s) + 9;
    const int lc0 = (f[2] >> s) - 9, lc1 = ((f[3] + up) >> s) + 9;
    outside = r0 >= lr1 || r0 + CT_R <= lr0 || 32 * w0 >= lc1 || 32 * (w0 + CT_W) <= lc0;
  }
  if (outside || ((a.j == 1 || a.src_pooled) && !cascade_tile_live(a, r0, w0))) {
    // nothing can reach this tile: zero words, zero pooled cell
    for (int e = threadIdx.x; e < CT_R * CT_W; e += blockDim.x) {
      const int r = r0 + e / CT_W, w = w0 + e % CT_W;
      if (r < a.rows && w < a.wpr) a.dst[(uint64_t)b * a.dst_stride + (uint64_t)r * a.wpr + w] = 0u;
    }
    if (final_mask && a.pooled && threadIdx.x == 0)
      a.pooled[(uint64_t)blockIdx.z * a.pool_wpr + blockIdx.x] = 0u;
    return;
  }
  if (threadIdx.x < CT_W) pool[threadIdx.x] = 0;
  for (int e = threadIdx.x; e < (CT_R + 2 * DIL) * (CT_W + 2); e += blockDim.x) {
    const int lr = e / (CT_W + 2), lw = e % (CT_W + 2);
    const int r = r0 - DIL + lr, w = w0 - 1 + lw;
    uint32_t v0 = 0, v1 = 0;
    if (r >= 0 && r < a.rows && w >= 0 && w < a.wpr) {
      v0 = cas_down(a, rect, b, r, w);
      if (both) v1 = cas_down(a, none, 0, r, w);
    }
    dm[0][lr][lw] = v0;
    if (both) dm[1][lr][lw] = v1;
  }
  __syncthreads();
  // vertical 9-row OR of every apron column, once (the horizontal spread
  // then reads 3 of them per output word)
  for (int e = threadIdx.x; e < CT_R * (CT_W + 2); e += blockDim.x) {
    const int lr = e / (CT_W + 2), lw = e % (CT_W + 2);
    uint32_t v0 = 0, v1 = 0;
#pragma unroll
    for (int k = 0; k <= 2 * DIL; ++k) {
      v0 |= dm[0][lr + k][lw];
      if (both) v1 |= dm[1][lr + k][lw];
    }
    vor[0][lr][lw] = v0;
    if (both) vor[1][lr][lw] = v1;
  }
  __syncthreads();
  const int tr = threadIdx.x / CT_TW, tq = threadIdx.x % CT_TW;
  const int r = r0 + tr;
  if (r < a.rows) {
#pragma unroll
    for (int q = 0; q < CT_W / CT_TW; ++q) {
      const int lw = tq + q * CT_TW, w = w0 + lw;
      if (w >= a.wpr) break;
      uint32_t v = spread(vor[0][tr][lw], vor[0][tr][lw + 1], vor[0][tr][lw + 2]);
      if (both) v &= spread(vor[1][tr][lw], vor[1][tr][lw + 1], vor[1][tr][lw + 2]);
      v &= last_word_mask(a.cols, w);
      a.dst[(uint64_t)b * a.dst_stride + (uint64_t)r * a.wpr + w] = v;
      if (final_mask && v) atomicOr(&pool[lw], 1u);
    }
  }
  if (final_mask && a.pooled) {
    __syncthreads();
    if (threadIdx.x < 32) {
      const uint32_t bits = __ballot_sync(0xFFFFFFFFu, threadIdx.x < CT_W && pool[threadIdx.x]);
      if (threadIdx.x == 0) a.pooled[(uint64_t)blockIdx.z * a.pool_wpr + blockIdx.x] = bits;
    }
  }
}

// ------------------------------------------------- direct cascade (one launch)
// C_j = dilate4(downmap2(C_{j-1})) with C_0 the upscaled pixel mask is an OR
// over a box: downmap2 ORs pixel pairs and dilate4 ORs a 9 x 9 box, both
// separable, so C_j(y, x) = OR of C_0 over rows [2^j y - A_j, 2^j y + B_j]
// and the same columns, A_j = 8 (2^j - 1), B_j = 9 (2^j - 1), clipped to the
// frame (out-of-range cells contribute nothing at every level, exactly as in
// the step-by-step cascade).  A gaze-window batch b > 0 starts from C_0 ∩
// its pixel window, i.e. the box is clipped to the window too.  C_0 is the
// nearest upscale of the low-res mask (fileio.py:430-436), so a box reduces
// to an OR of low-res bit rows and, per set cell, an interval of output
// bits.  One CTA per (level, batch, 32-row band), one warp per row; the
// final masks are also pooled per 32 x 32 cell as the step kernel does.
struct DirectArgs {
  int L, H, W, mh, mw, mwpr, fov;
  const uint32_t* mbits;
  const wv_frame_args* fa;
  int nitems;                       // entries used in the tables below
  int first_cta[WV_MAX_LEVELS * (WV_MAX_LEVELS + 1) + 1];
  uint8_t lev[WV_MAX_LEVELS * (WV_MAX_LEVELS + 1)], bat[WV_MAX_LEVELS * (WV_MAX_LEVELS + 1)];
  uint32_t* dst[WV_MAX_LEVELS + 1];
  uint64_t dst_stride[WV_MAX_LEVELS + 1];   // words per batch mask
  int wpr[WV_MAX_LEVELS + 1];
  uint32_t* pooled[WV_MAX_LEVELS + 1];      // null: not pooled
  int pool_wpr[WV_MAX_LEVELS + 1];
};

// Row y of C_j for batch window win = (r0, r1, c0, c1) (pixels, half open;
// the whole frame for the request): srow gets the OR of the low-res bit rows
// under the box; returns whether any of them is set (warp-uniform).
__device__ __forceinline__ bool direct_prep(const DirectArgs& a, int j, int y, int4 win,
                                            uint32_t* srow, int lane) {
  const int A = 8 * ((1 << j) - 1), B = 9 * ((1 << j) - 1);
  const int p0 = max(max((y << j) - A, 0), win.x), p1 = min(min((y << j) + B, a.H - 1), win.y - 1);
  uint32_t rowor = 0;
  if (p0 <= p1 && lane < a.mwpr) {
    const int m0 = (int)(((uint32_t)p0 * (uint32_t)a.mh) / (uint32_t)a.H);
    const int m1 = (int)(((uint32_t)p1 * (uint32_t)a.mh) / (uint32_t)a.H);
    for (int m = m0; m <= m1; ++m) rowor |= a.mbits[(uint64_t)m * a.mwpr + lane];
  }
  if (lane < a.mwpr) srow[lane] = rowor;
  return __any_sync(0xFFFFFFFFu, rowor != 0u);
}

// word w of that row: each set low-res cell under the box sets the output
// bits whose box [x 2^j - A, x 2^j + B] meets the cell's pixels (clipped to
// the window)
__device__ __forceinline__ uint32_t direct_word(const DirectArgs& a, int j, int4 win,
                                                const uint32_t* srow, const int* cell_x0, int w) {
  const int A = 8 * ((1 << j) - 1), B = 9 * ((1 << j) - 1);
  const int ncols = a.W >> j;
  const int x0 = 32 * w, x1 = min(32 * w + 31, ncols - 1);
  const int q0 = max(max((x0 << j) - A, 0), win.z), q1 = min(min((x1 << j) + B, a.W - 1), win.w - 1);
  if (q0 > q1) return 0u;
  const int cA = (int)(((uint32_t)q0 * (uint32_t)a.mw) / (uint32_t)a.W);
  const int cB = (int)(((uint32_t)q1 * (uint32_t)a.mw) / (uint32_t)a.W);
  uint32_t v = 0;
  // set cells of srow in [cA, cB], word by word (find-first-set)
  for (int cw = cA >> 5; cw <= (cB >> 5); ++cw) {
   uint32_t bits = srow[cw] & range_mask(cA, cB + 1, cw);
   while (bits) {
    const int c = 32 * cw + __ffs(bits) - 1;
    bits &= bits - 1u;
    // pixels x of cell c: floor(x mw / W) == c (table of cell starts)
    int s0 = cell_x0[c];
    int s1 = cell_x0[c + 1] - 1;
    s0 = max(s0, win.z);
    s1 = min(s1, win.w - 1);
    if (s0 > s1) continue;
    const int lo = max((s0 - B + (1 << j) - 1) >> j, 0);   // ceil((s0 - B) / 2^j), s0 - B >= -B
    const int hi = min((s1 + A) >> j, ncols - 1);
    v |= range_mask(lo, hi + 1, w);
   }
  }
  return v;
}

// The row's output as intervals: every run of consecutive set cells of srow
// maps to one interval of level-j columns (the per-cell intervals of
// adjacent cells abut or overlap), clipped to the window and the frame.
// Lane 0 scans the runs; returns the interval count (warp-uniform), or -1
// if there are more than kMaxIv (the caller then takes the per-cell path).
constexpr int kMaxIv = 16;
__device__ __forceinline__ int direct_intervals(const DirectArgs& a, int j, int4 win,
                                                const uint32_t* srow, const int* cell_x0,
                                                int2* iv, int lane) {
  int n = 0;
  if (lane == 0) {
    const int A = 8 * ((1 << j) - 1), B = 9 * ((1 << j) - 1);
    const int ncols = a.W >> j;
    int c = 0;
    while (c < a.mw && n >= 0) {
      // next set cell at or after c
      int w = c >> 5;
      uint32_t bits = srow[w] & (0xFFFFFFFFu << (c & 31));
      while (!bits && ++w < a.mwpr) bits = srow[w];
      if (!bits) break;
      const int c0 = 32 * w + __ffs(bits) - 1;
      // end of the run: next clear cell after c0
      int e = c0 + 1;
      while (e < a.mw) {
        const uint32_t clr = ~srow[e >> 5] & (0xFFFFFFFFu << (e & 31));
        if (clr) {
          e = min(a.mw, 32 * (e >> 5) + __ffs(clr) - 1);
          break;
        }
        e = 32 * ((e >> 5) + 1);
      }
      e = min(e, a.mw);
      const int s0 = max(cell_x0[c0], win.z), s1 = min(cell_x0[e] - 1, win.w - 1);
      if (s0 <= s1) {
        const int lo = max((s0 - B + (1 << j) - 1) >> j, 0);
        const int hi = min((s1 + A) >> j, ncols - 1);
        if (lo <= hi) {
          if (n == kMaxIv) {
            n = -1;
            break;
          }
          iv[n++] = make_int2(lo, hi);
        }
      }
      c = e;
    }
  }
  return __shfl_sync(0xFFFFFFFFu, n, 0);
}

__device__ __forceinline__ uint32_t intervals_word(const int2* iv, int n, int w) {
  uint32_t v = 0;
  for (int i = 0; i < n; ++i) v |= range_mask(iv[i].x, iv[i].y + 1, w);
  return v;
}

// direct_word with the candidate cells split over the warp's lanes (coarse
// levels: a word's box spans tens of cells); every lane gets the word
__device__ __forceinline__ uint32_t direct_word_warp(const DirectArgs& a, int j, int4 win,
                                                     const uint32_t* srow, const int* cell_x0,
                                                     int w, int lane) {
  const int A = 8 * ((1 << j) - 1), B = 9 * ((1 << j) - 1);
  const int ncols = a.W >> j;
  const int x0 = 32 * w, x1 = min(32 * w + 31, ncols - 1);
  const int q0 = max(max((x0 << j) - A, 0), win.z), q1 = min(min((x1 << j) + B, a.W - 1), win.w - 1);
  uint32_t v = 0;
  if (q0 <= q1) {
    const int cA = (int)(((uint32_t)q0 * (uint32_t)a.mw) / (uint32_t)a.W);
    const int cB = (int)(((uint32_t)q1 * (uint32_t)a.mw) / (uint32_t)a.W);
    for (int c = cA + lane; c <= cB; c += 32) {
      if (!((srow[c >> 5] >> (c & 31)) & 1u)) continue;
      const int s0 = max(cell_x0[c], win.z), s1 = min(cell_x0[c + 1] - 1, win.w - 1);
      if (s0 > s1) continue;
      const int lo = max((s0 - B + (1 << j) - 1) >> j, 0);
      const int hi = min((s1 + A) >> j, ncols - 1);
      v |= range_mask(lo, hi + 1, w);
    }
  }
  return __reduce_or_sync(0xFFFFFFFFu, v);
}

__global__ void __launch_bounds__(32 * WV_K1_DIRECT_RPW_WARPS) k_cascade_direct(DirectArgs a) {
  pdl_sync();
  __shared__ uint32_t srow[WV_K1_DIRECT_RPW_WARPS][2][32];
  __shared__ int2 siv[WV_K1_DIRECT_RPW_WARPS][2][kMaxIv];
  __shared__ uint32_t s_pool[64];
  // which (level, batch) item this CTA serves
  int it = 0;
  while (it + 1 < a.nitems && (int)blockIdx.x >= a.first_cta[it + 1]) ++it;
  const int j = a.lev[it], b = a.bat[it];
  const int band = blockIdx.x - a.first_cta[it];
  const int rows = a.H >> j, wpr = a.wpr[j];
  const bool final_mask = a.fov ? (b == j) : (b == 0);
  uint32_t* pooled = final_mask ? a.pooled[j] : nullptr;
  const int npw = (wpr + 31) >> 5;   // pooled words of this band
  for (int k = threadIdx.x; k < npw; k += blockDim.x) s_pool[k] = 0u;
  __shared__ int cell_x0[1025];   // first pixel of low-res column c: ceil(c W / mw)
  for (int c = threadIdx.x; c <= a.mw; c += blockDim.x)
    cell_x0[c] = (int)(((uint32_t)c * (uint32_t)a.W + a.mw - 1) / (uint32_t)a.mw);
  __syncthreads();
  const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
  const int4 full = make_int4(0, a.H, 0, a.W);
  int4 win = full;
  if (b > 0) {
    const int32_t* f = a.fa->fovea[b - 1];
    win = make_int4(f[0], f[1], f[2], f[3]);
  }
  const bool both = a.fov && b == j;   // D_j = C_j(window j) & C_j(request)
  constexpr int RPW = 32 / WV_K1_DIRECT_RPW_WARPS;   // rows per warp of the 32-row band
  for (int r = 0; r < RPW; ++r) {
    const int y = band * 32 + wp * RPW + r;
    if (y >= rows) break;
    const bool anyA = direct_prep(a, j, y, win, srow[wp][0], lane);
    const bool anyB = both ? direct_prep(a, j, y, full, srow[wp][1], lane) : true;
    __syncwarp();
    uint32_t* out = a.dst[j] + (uint64_t)b * a.dst_stride[j] + (uint64_t)y * wpr;
    const int nA = anyA ? direct_intervals(a, j, win, srow[wp][0], cell_x0, siv[wp][0], lane) : 0;
    const int nB = (both && anyB) ? direct_intervals(a, j, full, srow[wp][1], cell_x0, siv[wp][1],
                                                     lane)
                                  : 0;
    __syncwarp();
    if (nA >= 0 && nB >= 0) {
      // runs of set cells -> at most kMaxIv intervals per row: one word per lane
      for (int w = lane; w < wpr; w += 32) {
        uint32_t v = intervals_word(siv[wp][0], nA, w);
        if (both) v &= intervals_word(siv[wp][1], nB, w);
        out[w] = v;
        if (pooled && v) atomicOr(&s_pool[w >> 5], 1u << (w & 31));
      }
    } else if (wpr > 8) {
      // enough words for the lanes: one word per lane
      for (int w = lane; w < wpr; w += 32) {
        uint32_t v = anyA ? direct_word(a, j, win, srow[wp][0], cell_x0, w) : 0u;
        if (both && v) v &= anyB ? direct_word(a, j, full, srow[wp][1], cell_x0, w) : 0u;
        out[w] = v;
        if (pooled && v) atomicOr(&s_pool[w >> 5], 1u << (w & 31));
      }
    } else {
      // coarsest levels: few words, tens of cells each, split over the lanes
      for (int w = 0; w < wpr; ++w) {
        uint32_t v = anyA ? direct_word_warp(a, j, win, srow[wp][0], cell_x0, w, lane) : 0u;
        if (both && v) v &= anyB ? direct_word_warp(a, j, full, srow[wp][1], cell_x0, w, lane) : 0u;
        if (lane == 0) {
          out[w] = v;
          if (pooled && v) atomicOr(&s_pool[w >> 5], 1u << (w & 31));
        }
      }
    }
    __syncwarp();
  }
  if (pooled) {
    __syncthreads();
    for (int k = threadIdx.x; k < npw; k += blockDim.x)
      pooled[(uint64_t)band * a.pool_wpr[j] + k] = s_pool[k];
  }
}

// ----------------------------------------------------------- footprint step
// V_{j-1} = shrink4(upsample2(V_j & D_j)) (outside the grid counts as set),
// levels j = L..2; the finest step (j = 1, ANDed with the request) is
// k_footprint_tiles.  Upsampling duplicates rows, so the
// 9-row AND is taken over the 5 distinct source rows before bit doubling.
struct FootArgs {
  int j, L, H;
  int rows, cols, wpr;        // output level j-1
  int srows, swpr;            // source level j
  const uint32_t* V;          // valid at level j (nullptr: all ones)
  const uint32_t* D;          // detail mask level j
  uint32_t* out;              // level j-1 (finest step: fa->d_footprint)
  const uint32_t* R;          // finest step: requested rows
  const uint32_t* rowmap;
  const wv_frame_args* fa;
  const uint32_t* dpool;      // pooled occupancy of D_j (bs == 32), else null
  int dpool_wpr;
};

constexpr int FP_SR = CT_R / 2 + DIL + 1;  // source rows staged per tile (21)
constexpr int FP_SW = CT_W / 2 + 2;        // source words staged per tile (18)

__global__ void __launch_bounds__(256) k_footprint(FootArgs a) {
  pdl_sync();
  __shared__ uint32_t sv[FP_SR][FP_SW];
  const int r0 = blockIdx.z * CT_R, w0 = blockIdx.x * CT_W;
  const int sr0 = (r0 - DIL) >> 1, sw0 = (w0 >> 1) - 1;
  if (a.dpool) {
    // every output bit ANDs its own (in-range) source bit of V_j & D_j: a
    // tile whose in-range sources see no D_j bit is zero
    const int q0 = max(sr0, 0), q1 = min(sr0 + FP_SR, a.srows);
    const int u0 = max(sw0, 0), u1 = min(sw0 + FP_SW, a.swpr);
    bool hit = false;
    if (q0 < q1 && u0 < u1) {
      const int t0 = q0 / CT_R, t1 = (q1 - 1) / CT_R, c0 = u0 / CT_W, c1 = (u1 - 1) / CT_W;
      const int nc = c1 - c0 + 1;
      for (int e = threadIdx.x; e < (t1 - t0 + 1) * nc; e += blockDim.x) {
        const int tr = t0 + e / nc, tc = c0 + e % nc;
        const int lo = max(u0 - tc * CT_W, 0), hi = min(u1 - tc * CT_W, 32);
        const uint32_t m = (hi >= 32 ? 0xFFFFFFFFu : ((1u << hi) - 1u)) & (0xFFFFFFFFu << lo);
        hit |= (a.dpool[(uint64_t)tr * a.dpool_wpr + tc] & m) != 0u;
      }
    }
    if (!__syncthreads_or(hit)) {
      for (int e = threadIdx.x; e < CT_R * CT_W; e += blockDim.x) {
        const int r = r0 + e / CT_W, w = w0 + e % CT_W;
        if (r < a.rows && w < a.wpr) a.out[(uint64_t)r * a.wpr + w] = 0u;
      }
      return;
    }
  }
  for (int e = threadIdx.x; e < FP_SR * FP_SW; e += blockDim.x) {
    const int lr = e / FP_SW, lw = e % FP_SW;
    const int sr = sr0 + lr, sw = sw0 + lw;
    uint32_t v = 0xFFFFFFFFu;
    if (sr >= 0 && sr < a.srows && sw >= 0 && sw < a.swpr) {
      v = a.D[(uint64_t)sr * a.swpr + sw];
      if (a.V) v &= a.V[(uint64_t)sr * a.swpr + sw];
    }
    sv[lr][lw] = v;
  }
  __syncthreads();
  // AND over each output row's 4-5 source rows, once per staged source word
  __shared__ uint32_t va[CT_R][FP_SW];
  for (int e = threadIdx.x; e < CT_R * FP_SW; e += blockDim.x) {
    const int lr = e / FP_SW, lw = e - (e / FP_SW) * FP_SW;
    const int rr = r0 + lr;
    const int s_lo = ((rr - DIL) >> 1) - sr0, s_hi = ((rr + DIL) >> 1) - sr0;
    uint32_t v = 0xFFFFFFFFu;
    for (int k = s_lo; k <= s_hi; ++k) v &= sv[k][lw];
    va[lr][lw] = v;
  }
  __syncthreads();
  const int tr = threadIdx.x / CT_TW, tq = threadIdx.x % CT_TW;
  const int r = r0 + tr;
  if (r >= a.rows) return;
#pragma unroll
  for (int q = 0; q < CT_W / CT_TW; ++q) {
    const int w = w0 + tq + q * CT_TW;
    if (w >= a.wpr) break;
    uint32_t nb[3];
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      const int ww = w - 1 + d;
      if (ww < 0 || ww >= a.wpr) {
        nb[d] = 0xFFFFFFFFu;
        continue;
      }
      const uint32_t v = va[tr][(ww >> 1) - sw0];
      nb[d] = double_bits(v >> (16 * (ww & 1))) | ~last_word_mask(a.cols, ww);
    }
    a.out[(uint64_t)r * a.wpr + w] = shrink(nb[0], nb[1], nb[2]) & last_word_mask(a.cols, w);
  }
}

// Finest footprint step restricted to the level-1 synthesis tiles: the
// footprint is ANDed with the request, so it is zero outside the tiles that
// touch the request; tiles that left the request (ZERO_FLAG) are cleared.
// One CTA-iteration per OUT_H x OUT_W-pixel tile: 64 rows x FT_OW words, one
// word per thread; source: 37 rows x FT_SW words of V_1 & D_1.  Tiles are not
// word aligned (OUT_W = 56), so a word can straddle two listed tiles: each
// tile updates only the bits of its own pixel columns (atomicAnd to clear,
// atomicOr to set -- neighbouring tiles touch disjoint bits).
constexpr int FT_OW = (OUT_W + 31) / 32 + (OUT_W % 32 ? 1 : 0);   // output words a tile touches
constexpr int FT_SR = OUT_H / 2 + DIL + 1, FT_SW = FT_OW / 2 + 2;   // source rows / words
constexpr int FT_THREADS = OUT_H * FT_OW;
static_assert(FT_SW * 2 >= FT_OW + 2, "source window covers the tile's words and neighbours");

__global__ void __launch_bounds__(FT_THREADS) k_footprint_tiles(FootArgs a, const uint32_t* list,
                                                                const uint32_t* count, int ntx1) {
  pdl_sync();
  __shared__ uint32_t sv[FT_SR][FT_SW];
  const uint32_t n = *count;
  uint32_t* out = a.fa->d_footprint;
  const int tid = threadIdx.x;
  for (uint32_t it = blockIdx.x; it < n; it += gridDim.x) {
    const uint32_t e = list[it];
    const int tile = (int)(e & ~ZERO_FLAG);
    const int ty = tile / ntx1, tx = tile - (tile / ntx1) * ntx1;
    const int r0 = ty * OUT_H, c0 = tx * OUT_W, c1 = min(c0 + OUT_W, a.cols);
    const int wa = c0 >> 5;
    const int lr = tid / FT_OW, lw = tid - (tid / FT_OW) * FT_OW;
    const int r = r0 + lr, w = wa + lw;
    const uint32_t own = (r < a.rows && w < a.wpr) ? range_mask(c0, c1, w) : 0u;
    if (e & ZERO_FLAG) {
      if (own) atomicAnd(&out[(uint64_t)r * a.wpr + w], ~own);
      continue;   // no shared memory touched
    }
    const int sr0 = (r0 - DIL) >> 1, sw0 = (wa - 1) >> 1;
    for (int i = tid; i < FT_SR * FT_SW; i += blockDim.x) {
      const int ir = i / FT_SW, iw = i - (i / FT_SW) * FT_SW;
      const int sr = sr0 + ir, sw = sw0 + iw;
      uint32_t v = 0xFFFFFFFFu;
      if (sr >= 0 && sr < a.srows && sw >= 0 && sw < a.swpr) {
        v = a.D[(uint64_t)sr * a.swpr + sw];
        if (a.V) v &= a.V[(uint64_t)sr * a.swpr + sw];
      }
      sv[ir][iw] = v;
    }
    __syncthreads();
    if (own) {
      // AND over the output row's 4-5 source rows for each source word the
      // thread's neighbourhood (words w-1 .. w+1) reads
      const int s_lo = ((r - DIL) >> 1) - sr0, s_hi = ((r + DIL) >> 1) - sr0;
      const int q0 = ((w - 1) >> 1) - sw0;   // the words are q0, q0 + 1 (< FT_SW)
      uint32_t va0 = 0xFFFFFFFFu, va1 = 0xFFFFFFFFu;
      for (int k = s_lo; k <= s_hi; ++k) {
        va0 &= sv[k][q0];
        va1 &= sv[k][q0 + 1];
      }
      uint32_t nb[3];
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        const int ww = w - 1 + d;
        if (ww < 0 || ww >= a.wpr) {
          nb[d] = 0xFFFFFFFFu;
          continue;
        }
        const uint32_t v = ((ww >> 1) - sw0) > q0 ? va1 : va0;
        nb[d] = double_bits(v >> (16 * (ww & 1))) | ~last_word_mask(a.cols, ww);
      }
      uint32_t v = shrink(nb[0], nb[1], nb[2]) & last_word_mask(a.cols, w);
      v &= a.R[(uint64_t)a.rowmap[r] * a.wpr + w];
      uint32_t* o = &out[(uint64_t)r * a.wpr + w];
      if (own == 0xFFFFFFFFu) {
        *o = v;
      } else {
        atomicAnd(o, ~own);
        if (v & own) atomicOr(o, v & own);
      }
    }
    __syncthreads();
  }
}

// -------------------------------------------------------------- block select
// One warp per 32x32 coefficient block (lane = block row); 8 blocks per CTA
// aggregate their list appends and statistics before touching global
// counters.
struct BlockArgs {
  int L, H, W, bs, nbx, NB, n, rs;
  const uint32_t* D[WV_MAX_LEVELS + 1];
  int dwpr[WV_MAX_LEVELS + 1];
  const wv_frame_args* fa;          // payload / cache entry / result of this call
  unsigned long long table_bytes;   // n * NB * 8
  uint32_t* sel;
  uint32_t* prev_sel;
  uint32_t* list;
  uint32_t* list_count;
  int account_only;
  int full;                                    // decode_full: every block selected
  const uint8_t* bstate;                       // K2's per-block "plane may be nonzero"
  int fetch;                                   // WV_FLAG_FETCH: list blocks whose records are absent
  uint32_t* flist;
  uint32_t* fcount;
  const uint32_t* pooled[WV_MAX_LEVELS + 1];   // nullptr: scan rows
  int pool_wpr[WV_MAX_LEVELS + 1];
};

__device__ __forceinline__ bool row_any(const uint32_t* row, int c0, int c1) {
  if (c0 >= c1) return false;
  for (int w = c0 >> 5; w <= ((c1 - 1) >> 5); ++w)
    if (row[w] & range_mask(c0, c1, w)) return true;
  return false;
}

__device__ bool incl_row_any(const BlockArgs& a, int y, int x0, int x1) {
  if (y < (a.H >> a.L) && x0 < (a.W >> a.L)) return true;
  for (int k = 1; k <= a.L; ++k) {
    const int bh = a.H >> k, bw = a.W >> k;
    if (y < bh) {
      if (row_any(a.D[k] + (uint64_t)y * a.dwpr[k], max(x0, bw) - bw, min(x1, 2 * bw) - bw))
        return true;
    } else if (y < 2 * bh) {
      const uint32_t* row = a.D[k] + (uint64_t)(y - bh) * a.dwpr[k];
      if (row_any(row, x0, min(x1, bw))) return true;
      if (row_any(row, max(x0, bw) - bw, min(x1, 2 * bw) - bw)) return true;
    }
  }
  return false;
}

// Thread per block.  A block lying inside one subband quadrant of one level
// reads its "any" bit from the level's 32x32-pooled mask (block_size 32 with
// 32-aligned subbands: every block at the 8K configuration); other blocks
// scan their rows.  A warp owns 32 consecutive blocks = one bitmap word.
__device__ bool block_any(const BlockArgs& a, int b) {
  const int by = b / a.nbx, bx = b - (b / a.nbx) * a.nbx;
  const int y0 = by * a.bs, x0 = bx * a.bs, y1 = y0 + a.bs, x1 = x0 + a.bs;
  if (y0 < (a.H >> a.L) && x0 < (a.W >> a.L)) return true;
  for (int k = 1; k <= a.L; ++k) {
    const int bh = a.H >> k, bw = a.W >> k;
    const bool top = y1 <= bh, bot = y0 >= bh && y1 <= 2 * bh;
    const bool left = x1 <= bw, right = x0 >= bw && x1 <= 2 * bw;
    if ((top && right) || (bot && (left || right))) {
      const int r0 = bot ? y0 - bh : y0, c0 = right ? x0 - bw : x0;
      if (a.pooled[k] && !(r0 & 31) && !(c0 & 31)) {
        const int w = c0 >> 5;
        return (a.pooled[k][(uint64_t)(r0 >> 5) * a.pool_wpr[k] + (w >> 5)] >> (w & 31)) & 1u;
      }
      break;
    }
    if (!(y1 <= bh && x1 <= bw)) break;   // straddles quadrants: scan rows
  }
  for (int r = y0; r < y1; ++r)
    if (incl_row_any(a, r, x0, x1)) return true;
  return false;
}

__global__ void __launch_bounds__(256) k_blocks(BlockArgs a) {
  pdl_sync();
  const unsigned long long* __restrict__ ends = (const unsigned long long*)a.fa->d_payload;
  const unsigned long long rec_bytes = a.fa->payload_bytes - a.table_bytes;
  uint32_t* loaded = a.fa->d_set_loaded;
  unsigned long long* set_bytes = a.fa->d_set_bytes;
  wv_frame_result* res = a.fa->d_result;
  const int lane = threadIdx.x & 31;
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  const bool valid = b < a.NB;
  const bool sel = valid && (a.full || block_any(a, b));
  unsigned long long bytes = 0, recs = 0;
  uint32_t err = 0;
  if (sel) {
    unsigned long long prev = b ? ends[b - 1] : 0ull;
    for (int t = 0; t < a.n; ++t) {
      const uint64_t i = (uint64_t)t * a.NB + b;
      const unsigned long long e = ends[i];
      const unsigned long long st = t ? ends[i - 1] : prev;
      if (e < st || e > rec_bytes || (e - st) % a.rs ||
          (e - st) / a.rs > (unsigned long long)a.bs * a.bs)
        err |= WV_DERR_TABLE;
      else {
        bytes += e - st;
        recs += (e - st) / a.rs;
      }
    }
  }
  const uint32_t word = (uint32_t)(blockIdx.x * blockDim.x + (threadIdx.x & ~31)) >> 5;
  const uint32_t selmask = __ballot_sync(0xFFFFFFFFu, sel);
  uint32_t prevw = 0, loadw = 0;
  if (lane == 0 && (word << 5) < (uint32_t)a.NB) {
    prevw = a.prev_sel[word];
    loadw = loaded[word];
  }
  prevw = __shfl_sync(0xFFFFFFFFu, prevw, 0);
  loadw = __shfl_sync(0xFFFFFFFFu, loadw, 0);
  const bool prev = valid && ((prevw >> lane) & 1u);
  const bool was = (loadw >> lane) & 1u;
  const bool missing = sel && !was;
  // K2 work: selected blocks with records (all are offset-checked) or with
  // stale nonzeros; blocks that left the selection and still hold nonzeros.
  // A selected block without records whose plane block is zero needs nothing.
  const bool dirty = valid && a.bstate[b] != 0;
  const bool emit = !a.account_only && ((sel && (recs > 0 || dirty)) || (!sel && prev && dirty));
  const uint32_t emask = __ballot_sync(0xFFFFFFFFu, emit);
  uint32_t base = 0;
  if (lane == 0 && emask) base = atomicAdd(a.list_count, (uint32_t)__popc(emask));
  base = __shfl_sync(0xFFFFFFFFu, base, 0);
  if (emit)
    a.list[base + __popc(emask & ((1u << lane) - 1u))] = sel ? (uint32_t)b : ((uint32_t)b | ZERO_FLAG);
  unsigned long long newb = missing ? bytes : 0ull;
  const uint32_t nmiss = __popc(__ballot_sync(0xFFFFFFFFu, missing));
  for (int o = 16; o; o >>= 1) {
    recs += __shfl_xor_sync(0xFFFFFFFFu, recs, o);
    newb += __shfl_xor_sync(0xFFFFFFFFu, newb, o);
    err |= __shfl_xor_sync(0xFFFFFFFFu, err, o);
  }
  if (a.fetch) {
    // records of selected blocks not yet in HBM: list them for k_fetch
    uint32_t fw = 0;
    if (lane == 0 && (word << 5) < (uint32_t)a.NB) fw = a.fa->d_fetched[word];
    fw = __shfl_sync(0xFFFFFFFFu, fw, 0);
    const uint32_t need = selmask & ~fw;
    uint32_t fb = 0;
    if (lane == 0 && need) {
      fb = atomicAdd(a.fcount, (uint32_t)__popc(need));
      a.fa->d_fetched[word] = fw | need;
    }
    fb = __shfl_sync(0xFFFFFFFFu, fb, 0);
    if ((need >> lane) & 1u) a.flist[fb + __popc(need & ((1u << lane) - 1u))] = (uint32_t)b;
  }
  if (lane == 0 && (word << 5) < (uint32_t)a.NB) {
    a.sel[word] = selmask;
    if (!a.account_only) a.prev_sel[word] = selmask;
    loaded[word] = loadw | selmask;
    if (recs) atomicAdd(&res->records, recs);
    if (newb) {
      atomicAdd(&res->new_bytes, newb);
      atomicAdd(set_bytes, newb);
    }
    if (nmiss) atomicAdd(&res->n_missing, nmiss);
    if (selmask) atomicAdd(&res->n_selected, (uint32_t)__popc(selmask));
    if (err) atomicOr(&res->error, err);
  }
}

// The fetch list (and its length) to the caller's pinned host buffers, so a
// stream-ordered host function can read exactly those spans from the file
// before k_fetch copies them to HBM (plain stores over PCIe; no-op without
// h_fetch_list).
__global__ void __launch_bounds__(256) k_list_to_host(const wv_frame_args* __restrict__ fa,
                                                      const uint32_t* __restrict__ flist,
                                                      const uint32_t* __restrict__ fcount) {
  pdl_sync();
  uint32_t* hl = fa->h_fetch_list;
  if (!hl || !fa->h_fetch_count) return;
  const uint32_t n = *fcount;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    hl[i] = flist[i];
  if (blockIdx.x == 0 && threadIdx.x == 0) *fa->h_fetch_count = n;
  __threadfence_system();
}

// --------------------------------------------------------------- span fetch
// VideoReader.load_blocks (fileio.py:346-390) for one decode: copy the record
// spans of the listed blocks, all temporal indices, from the set payload in
// pinned host memory (read by the SMs over PCIe, UVA) to the same offsets of
// the HBM payload.  One warp per (block, t) span; 16-byte chunks covering the
// span (both payload buffers are padded to 16 bytes, and bytes outside the
// span are the file's own bytes, so over-copying is harmless).
__global__ void __launch_bounds__(256) k_fetch(const wv_frame_args* __restrict__ fa,
                                               const uint32_t* __restrict__ flist,
                                               const uint32_t* __restrict__ fcount, int n, int NB,
                                               unsigned long long table_bytes) {
  pdl_sync();
  const uint32_t nspans = *fcount * (uint32_t)n;
  const unsigned long long* __restrict__ ends = (const unsigned long long*)fa->d_payload;
  const uint4* src = reinterpret_cast<const uint4*>(fa->h_payload);
  uint4* dst = reinterpret_cast<uint4*>(const_cast<void*>(fa->d_payload));
  const unsigned long long size = fa->payload_bytes;
  const int lane = threadIdx.x & 31;
  const uint32_t warps = gridDim.x * (blockDim.x >> 5);
  unsigned long long copied = 0;
  for (uint32_t sp = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); sp < nspans; sp += warps) {
    const uint32_t b = flist[sp / n];
    const int t = (int)(sp % n);
    const uint64_t fi = (uint64_t)t * NB + b;
    const unsigned long long en = ends[fi], st = fi ? ends[fi - 1] : 0ull;
    if (en <= st) continue;
    const unsigned long long lo = table_bytes + st, hi = min(table_bytes + en, size);
    if (lo >= hi) continue;   // (k_blocks flags inconsistent tables)
    for (unsigned long long c = (lo >> 4) + lane; c < (hi + 15) >> 4; c += 32) dst[c] = src[c];
    copied += hi - lo;
  }
  if (lane == 0 && copied) atomicAdd(&fa->d_result->fetched_bytes, copied);
}

// -------------------------------------------------------------- tile lists
// Level 1 (output pixels): a 64x64 tile is needed iff it touches the request;
// tiles needed last frame but not now are listed with ZERO_FLAG so the
// canvas is cleared there.  Level k >= 2: tile u is needed iff a needed
// level-(k-1) tile reads its rows; unrolled to level 1 this is the need-bit
// rectangle [2^m u - (2^m-1), 2^m u + 2(2^m-1)] (m = k-1) in each axis.
struct TileArgs {
  int L, H, W;
  int wpr0;
  const uint32_t* R;
  const uint32_t* rowmap;
  int full;
  int nty[WV_MAX_LEVELS + 1], ntx[WV_MAX_LEVELS + 1];
  uint32_t* need1;                   // bit rows: nty[1] x nwords1
  int nwords1;
  uint32_t* list[WV_MAX_LEVELS + 1];
  uint8_t* prev_need;
  uint32_t* counters;                // CNT_TILES + k
  const wv_frame_args* fa;
};

__global__ void __launch_bounds__(256) k_tiles1(TileArgs a) {
  pdl_sync();
  const int nt1 = a.nty[1] * a.ntx[1];
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  bool nd = false, pv = false;
  if (t < nt1) {
    const int ty = t / a.ntx[1], tx = t % a.ntx[1];
    nd = a.full != 0;
    const int ro0 = a.fa->out_row0, ro1 = a.fa->out_row1;
    const bool in_rows = ro1 <= ro0 || (ty * OUT_H < ro1 && min((ty + 1) * OUT_H, a.H) > ro0);
    if (!in_rows) {
      nd = false;
    } else if (!nd) {
      const int y0 = ty * OUT_H, y1 = min(y0 + OUT_H, a.H);
      const int c0 = tx * OUT_W, c1 = min(c0 + OUT_W, a.W);
      const uint32_t m0 = a.rowmap[y0], m1 = a.rowmap[y1 - 1];
      for (uint32_t m = m0; m <= m1 && !nd; ++m) {
        const uint32_t* row = a.R + (uint64_t)m * a.wpr0;
        for (int w = c0 >> 5; w <= ((c1 - 1) >> 5); ++w)
          if (row[w] & range_mask(c0, c1, w)) { nd = true; break; }
      }
    }
    pv = a.prev_need[t] != 0;
    a.prev_need[t] = nd;
    if (nd) atomicOr(&a.need1[ty * a.nwords1 + (tx >> 5)], 1u << (tx & 31));
    else atomicAnd(&a.need1[ty * a.nwords1 + (tx >> 5)], ~(1u << (tx & 31)));
  }
  const bool emit = nd || pv;
  const uint32_t m = __ballot_sync(0xFFFFFFFFu, emit);
  const uint32_t mn = __ballot_sync(0xFFFFFFFFu, nd);
  const int lane = threadIdx.x & 31;
  uint32_t base = 0;
  if (lane == 0 && m) base = atomicAdd(&a.counters[CNT_TILES + 1], (uint32_t)__popc(m));
  base = __shfl_sync(0xFFFFFFFFu, base, 0);
  if (emit) a.list[1][base + __popc(m & ((1u << lane) - 1u))] = (uint32_t)t | (nd ? 0u : ZERO_FLAG);
  if (lane == 0 && mn) atomicAdd(&a.fa->d_result->n_tiles, (uint32_t)__popc(mn));
}

// Coarser levels in one CTA: need maps live as bit rows in shared memory and
// level k is derived from level k-1 (rows 2u-1..2u+2 x cols 2v-1..2v+2).
__global__ void __launch_bounds__(1024) k_tiles_up(TileArgs a) {
  pdl_sync();
  extern __shared__ uint32_t nbits[];
  __shared__ uint32_t cnt;
  int off[WV_MAX_LEVELS + 2];
  off[1] = 0;
  for (int k = 1; k <= a.L; ++k) off[k + 1] = off[k] + a.nty[k] * wpr(a.ntx[k]);
  for (int i = threadIdx.x; i < off[a.L + 1]; i += blockDim.x)
    nbits[i] = i < off[2] ? a.need1[i] : 0u;
  __syncthreads();
  for (int k = 2; k <= a.L; ++k) {
    if (threadIdx.x == 0) cnt = 0;
    __syncthreads();
    const int ntx = a.ntx[k], nt = a.nty[k] * ntx;
    const int fy = a.nty[k - 1], fx = a.ntx[k - 1], fw = wpr(fx);
    const uint32_t* prev = nbits + off[k - 1];
    for (int t = threadIdx.x; t < nt; t += blockDim.x) {
      const int u = t / ntx, v = t - (t / ntx) * ntx;
      const int x0 = max(2 * v - 1, 0), x1 = min(2 * v + 2, fx - 1);
      bool nd = false;
      for (int ty = max(2 * u - 1, 0); ty <= min(2 * u + 2, fy - 1) && !nd; ++ty)
        for (int w = x0 >> 5; w <= (x1 >> 5); ++w)
          if (prev[ty * fw + w] & range_mask(x0, x1 + 1, w)) { nd = true; break; }
      if (nd) {
        atomicOr(&nbits[off[k] + u * wpr(ntx) + (v >> 5)], 1u << (v & 31));
        a.list[k][atomicAdd(&cnt, 1u)] = (uint32_t)t;
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) a.counters[CNT_TILES + k] = cnt;
  }
}

// decode_full: the footprint is the whole frame (LevelMaskSet.full,
// wavelets.py:267-270), no mask cascades are needed
__global__ void k_fill_footprint(const wv_frame_args* __restrict__ fa, int rows, int cols,
                                 int wpr) {
  pdl_sync();
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= rows * wpr) return;
  const int w = idx % wpr;
  fa->d_footprint[idx] = last_word_mask(cols, w);
}

__global__ void k_finalize(const wv_frame_args* fa) {
  pdl_sync();
  fa->d_result->set_bytes = *fa->d_set_bytes;
}

}  // namespace

int launch_select(const Layout& lo, const wv_geometry* g, int mode, int flags,
                  const wv_frame_args* fa, uint8_t* ws, cudaStream_t s, int stages) {
  const int L = lo.L, H = lo.H, W = lo.W;
  const bool full = mode == WV_MODE_FULL;
  const bool fov = mode == WV_MODE_FOVEATED;
  const bool acct = (flags & WV_FLAG_ACCOUNT_ONLY) != 0;
  uint32_t* R = (uint32_t*)(ws + lo.mrows);
  uint32_t* rowmap = (uint32_t*)(ws + lo.rowmap);
  uint32_t* counters = (uint32_t*)(ws + lo.counters);
  const bool st_rows = stages & WV_STAGE_ROWS, st_cas = stages & WV_STAGE_CASCADES;
  const bool st_fp = stages & WV_STAGE_FOOTPRINT, st_blocks = stages & WV_STAGE_BLOCKS;
  const bool st_tiles = stages & WV_STAGE_TILES, st_fpt = stages & WV_STAGE_FOOTPRINT_TILES;
  if (st_rows) {
    const int n = max(lo.mh * lo.wpr_[0], H);
    WV_CUDA(launch_k(k_mask_rows, dim3(cdiv(n, 256)), dim3(256), 0, s, fa, R, rowmap, counters,
                     lo.mh, lo.mw, W, H, lo.wpr_[0], (int)full, (uint32_t*)(ws + lo.mbits)));
  }
  // level cascades (batch 0: request closure; batches k>=j: gaze windows);
  // a full-frame decode needs none of them
  const bool direct = WV_K1_DIRECT && lo.mw <= 1024 && !full && st_cas;
  if (direct) {
    DirectArgs d{};
    d.L = L; d.H = H; d.W = W; d.mh = lo.mh; d.mw = lo.mw; d.mwpr = (lo.mw + 31) / 32;
    d.fov = fov;
    d.mbits = (const uint32_t*)(ws + lo.mbits);
    d.fa = fa;
    int ctas = 0;
    for (int j = 1; j <= L; ++j) {
      d.dst[j] = (uint32_t*)(ws + lo.stack[j]);
      d.dst_stride[j] = lo.stack_stride[j] / 4;
      d.wpr[j] = lo.wpr_[j];
      d.pooled[j] = lo.bs == 32 ? (uint32_t*)(ws + lo.pooled[j]) : nullptr;
      d.pool_wpr[j] = cdiv(lo.wpr_[j], CT_W);
      const int bands = cdiv(H >> j, 32);
      auto add = [&](int bb) {
        d.lev[d.nitems] = (uint8_t)j;
        d.bat[d.nitems] = (uint8_t)bb;
        d.first_cta[d.nitems] = ctas;
        ++d.nitems;
        ctas += bands;
      };
      add(0);
      if (fov)
        for (int k = j; k <= L; ++k) add(k);
    }
    d.first_cta[d.nitems] = ctas;
    WV_CUDA(launch_k(k_cascade_direct, dim3(ctas), dim3(32 * WV_K1_DIRECT_RPW_WARPS), 0, s, d));
  }
  for (int j = 1; j <= L && !full && st_cas && !direct; ++j) {
    CascadeArgs c{};
    c.j = j; c.L = L; c.H = H;
    c.rows = H >> j; c.cols = W >> j; c.wpr = lo.wpr_[j];
    c.prow_n = H >> (j - 1); c.pcols = W >> (j - 1); c.pwpr = lo.wpr_[j - 1];
    c.src = j > 1 ? (const uint32_t*)(ws + lo.stack[j - 1]) : nullptr;
    c.src_stride = j > 1 ? lo.stack_stride[j - 1] / 4 : 0;
    c.R = R; c.rowmap = rowmap;
    c.dst = (uint32_t*)(ws + lo.stack[j]);
    c.dst_stride = lo.stack_stride[j] / 4;
    c.fov = fov;
    c.fa = fa;
    c.nbatch = 0;
    c.batch[c.nbatch++] = 0;
    if (fov)
      for (int k = j; k <= L; ++k) c.batch[c.nbatch++] = k;
    c.pooled = lo.bs == 32 ? (uint32_t*)(ws + lo.pooled[j]) : nullptr;
    c.pool_wpr = cdiv(c.wpr, CT_W);
    // zero-tile skipping: j == 1 from the low-res mask; j > 1 from level
    // j-1's pooled occupancy (viewport only: a foveated D_{j-1} is not an
    // upper bound of the request cascade)
    c.src_pooled = (j > 1 && !fov && lo.bs == 32) ? (const uint32_t*)(ws + lo.pooled[j - 1]) : nullptr;
    c.src_pool_wpr = cdiv(lo.wpr_[j - 1], CT_W);
    c.mh = lo.mh; c.mw = lo.mw;
    dim3 grid(cdiv(c.wpr, CT_W), c.nbatch, cdiv(c.rows, CT_R));
    WV_CUDA(launch_k(k_cascade, dim3(grid), dim3(256), 0, s, c));
  }
  auto Dptr = [&](int k) -> uint32_t* {
    return (uint32_t*)(ws + lo.stack[k] + (fov ? (uint64_t)k * lo.stack_stride[k] : 0));
  };
  // footprint: V_L = ones; V_{j-1} = shrink(up(V_j & D_j)); last & request
  if (full && !acct && st_fp)
    WV_CUDA(launch_k(k_fill_footprint, dim3(cdiv(H * lo.wpr_[0], 256)), dim3(256), 0, s, fa, H, W,
                     lo.wpr_[0]));
  for (int j = L; j >= 2 && !acct && !full && st_fp; --j) {
    FootArgs f{};
    f.j = j; f.L = L; f.H = H;
    f.rows = H >> (j - 1); f.cols = W >> (j - 1); f.wpr = lo.wpr_[j - 1];
    f.srows = H >> j; f.swpr = lo.wpr_[j];
    f.V = j == L ? nullptr : (const uint32_t*)(ws + lo.fp[j]);
    f.D = Dptr(j);
    f.out = (uint32_t*)(ws + lo.fp[j - 1]);
    f.R = R; f.rowmap = rowmap; f.fa = fa;
    f.dpool = lo.bs == 32 ? (const uint32_t*)(ws + lo.pooled[j]) : nullptr;
    f.dpool_wpr = cdiv(lo.wpr_[j], CT_W);
    dim3 grid(cdiv(f.wpr, CT_W), 1, cdiv(f.rows, CT_R));
    WV_CUDA(launch_k(k_footprint, dim3(grid), dim3(256), 0, s, f));
  }
  if (st_blocks) {
    BlockArgs b{};
    b.L = L; b.H = H; b.W = W; b.bs = lo.bs; b.nbx = lo.nbx; b.NB = lo.NB; b.n = lo.n;
    b.rs = 2 + lo.C * (g->float_mode ? 4 : 1);
    for (int k = 1; k <= L; ++k) { b.D[k] = Dptr(k); b.dwpr[k] = lo.wpr_[k]; }
    b.fa = fa;
    b.table_bytes = (unsigned long long)lo.n * lo.NB * 8;
    b.sel = (uint32_t*)(ws + lo.sel);
    b.prev_sel = (uint32_t*)(ws + lo.prev_sel);
    b.list = (uint32_t*)(ws + lo.blist);
    b.list_count = counters + CNT_BLOCKS;
    b.account_only = acct;
    b.full = full;
    b.bstate = ws + lo.bstate;
    b.fetch = (flags & WV_FLAG_FETCH) != 0;
    b.flist = (uint32_t*)(ws + lo.flist);
    b.fcount = counters + CNT_FETCH;
    for (int k = 1; k <= L; ++k) {
      const bool ok = lo.bs == 32 && ((H >> k) % 32) == 0 && ((W >> k) % 32) == 0;
      b.pooled[k] = ok ? (const uint32_t*)(ws + lo.pooled[k]) : nullptr;
      b.pool_wpr[k] = cdiv(lo.wpr_[k], CT_W);
    }
    WV_CUDA(launch_k(k_blocks, dim3(cdiv(lo.NB, 256)), dim3(256), 0, s, b));
    if (b.fetch)
      WV_CUDA(launch_k(k_list_to_host, dim3(8), dim3(256), 0, s, fa, (const uint32_t*)b.flist,
                       (const uint32_t*)b.fcount));
  }
  if (acct && st_blocks) {
    WV_CUDA(launch_k(k_finalize, dim3(1), dim3(1), 0, s, fa));
  } else if (!acct) {
    TileArgs t{};
    t.L = L; t.H = H; t.W = W; t.wpr0 = lo.wpr_[0]; t.R = R; t.rowmap = rowmap; t.full = full;
    for (int k = 1; k <= L; ++k) {
      t.nty[k] = lo.nty[k]; t.ntx[k] = lo.ntx[k];
      t.list[k] = (uint32_t*)(ws + lo.tlist[k]);
    }
    t.need1 = (uint32_t*)(ws + lo.need[1]);
    t.nwords1 = wpr(lo.ntx[1]);
    t.prev_need = ws + lo.prev_need;
    t.counters = counters;
    t.fa = fa;
    const int nt1 = lo.nty[1] * lo.ntx[1];
    if (st_tiles) WV_CUDA(launch_k(k_tiles1, dim3(cdiv(nt1, 256)), dim3(256), 0, s, t));
    if (!full && st_fpt) {
      // finest footprint step on the level-1 tiles only (zero elsewhere)
      FootArgs f{};
      f.j = 1; f.L = L; f.H = H;
      f.rows = H; f.cols = W; f.wpr = lo.wpr_[0];
      f.srows = H >> 1; f.swpr = lo.wpr_[1];
      f.V = L == 1 ? nullptr : (const uint32_t*)(ws + lo.fp[1]);
      f.D = Dptr(1);
      f.R = R; f.rowmap = rowmap; f.fa = fa;
      int dev = 0, sms = 148;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      WV_CUDA(launch_k(k_footprint_tiles, dim3(min(nt1, 8 * sms)), dim3(FT_THREADS), 0, s, f,
                       (const uint32_t*)t.list[1], (const uint32_t*)(counters + CNT_TILES + 1),
                       lo.ntx[1]));
    }
    if (L >= 2 && st_tiles) {
      size_t words = 0;
      for (int k = 1; k <= L; ++k) words += (size_t)lo.nty[k] * wpr(lo.ntx[k]);
      if (words * 4 > 200 * 1024) return WV_ERR_UNSUPPORTED;
      if (words * 4 > 48 * 1024)
        WV_CUDA(cudaFuncSetAttribute(k_tiles_up, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)(words * 4)));
      WV_CUDA(launch_k(k_tiles_up, dim3(1), dim3(1024), words * 4, s, t));
    }
  }
  WV_CUDA(cudaGetLastError());
  return WV_OK;
}

// WV_STAGE_FETCH: the listed blocks' records, all temporal indices, host -> HBM
int launch_fetch(const Layout& lo, const wv_frame_args* fa, uint8_t* ws, cudaStream_t s) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const uint32_t* counters = (const uint32_t*)(ws + lo.counters);
  WV_CUDA(launch_k(k_fetch, dim3(4 * sms), dim3(256), 0, s, fa, (const uint32_t*)(ws + lo.flist),
                   counters + CNT_FETCH, lo.n, lo.NB, (unsigned long long)lo.n * lo.NB * 8));
  WV_CUDA(cudaGetLastError());
  return WV_OK;
}

// ------------------------------------------------------ compact BlockEnd table
// ends[i] = rs * (counts[0] + ... + counts[i]) (the BlockEnd table's
// cumulative record ends, fileio.py:157-162), rebuilt on the device from
// per-(t, block) record counts so span residency uploads 2 bytes per entry
// instead of 8.  One CTA: each thread sums a contiguous run of entries, a
// block-wide exclusive scan of the run sums, then each thread writes its run.
__global__ void __launch_bounds__(1024) k_table_expand(const uint16_t* __restrict__ counts,
                                                       uint64_t n, int rs,
                                                       unsigned long long* __restrict__ ends) {
  __shared__ unsigned long long wsum[32];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const uint64_t per = (n + blockDim.x - 1) / blockDim.x;
  const uint64_t b0 = min(n, (uint64_t)tid * per), b1 = min(n, b0 + per);
  unsigned long long s = 0;
  for (uint64_t i = b0; i < b1; ++i) s += counts[i];
  unsigned long long inc = s;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long u = __shfl_up_sync(0xFFFFFFFFu, inc, o);
    if (lane >= o) inc += u;
  }
  if (lane == 31) wsum[wid] = inc;
  __syncthreads();
  if (wid == 0) {
    unsigned long long w = lane < (int)(blockDim.x >> 5) ? wsum[lane] : 0ull;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long u = __shfl_up_sync(0xFFFFFFFFu, w, o);
      if (lane >= o) w += u;
    }
    wsum[lane] = w;   // inclusive over warps
  }
  __syncthreads();
  unsigned long long run = inc - s + (wid ? wsum[wid - 1] : 0ull);   // exclusive prefix
  for (uint64_t i = b0; i < b1; ++i) {
    run += counts[i];
    ends[i] = run * (unsigned long long)rs;
  }
}

int launch_table_expand(const uint16_t* d_counts, uint64_t n, int rs, uint64_t* d_table,
                        cudaStream_t s) {
  WV_CUDA(launch_k(k_table_expand, dim3(1), dim3(1024), 0, s, d_counts, n, rs,
                   (unsigned long long*)d_table));
  WV_CUDA(cudaGetLastError());
  return WV_OK;
}

}  // namespace wv
