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
__global__ void k_mask_rows(const uint8_t* __restrict__ mask, uint32_t* __restrict__ R, int mh,
                            int mw, int W, int wpr0, int full) {
  int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= mh * wpr0) return;
  int my = idx / wpr0, w = idx % wpr0;
  uint32_t bits = 0;
  for (int i = 0; i < 32; ++i) {
    int x = 32 * w + i;
    if (x >= W) break;
    int mx = (int)(((long long)x * mw) / W);
    if (full || mask[(long long)my * mw + mx]) bits |= 1u << i;
  }
  R[idx] = bits;
}

// ------------------------------------------------------------- cascade step
struct CascadeArgs {
  int j, L, H;
  int rows, cols, wpr;        // output level j
  int prow_n, pcols, pwpr;    // source level j-1
  const uint32_t* src;        // j > 1: stack[j-1]
  uint64_t src_stride;        // words per batch mask
  const uint32_t* R;          // j == 1: pixel rows
  int mh;
  uint32_t* dst;
  uint64_t dst_stride;
  int nbatch;
  int batch[WV_MAX_LEVELS + 1];
  int rect[WV_MAX_LEVELS + 1][4];  // j == 1 foveated windows, by batch id
  int fov;                         // foveated: batch j also ANDs with batch 0
};

__device__ __forceinline__ uint32_t cas_src(const CascadeArgs& a, int b, int rr, int ww) {
  if (ww < 0 || ww >= a.pwpr || rr < 0 || rr >= a.prow_n) return 0u;
  if (a.j == 1) {
    uint32_t v = a.R[(long long)((long long)rr * a.mh / a.H) * a.pwpr + ww];
    if (b > 0) {
      const int* r = a.rect[b];
      if (rr < r[0] || rr >= r[1]) return 0u;
      v &= range_mask(r[2], r[3], ww);
    }
    return v;
  }
  return a.src[(uint64_t)b * a.src_stride + (uint64_t)rr * a.pwpr + ww];
}

// downmapped word at output level (row r, word w)
__device__ __forceinline__ uint32_t cas_down(const CascadeArgs& a, int b, int r, int w) {
  if (w < 0 || w >= a.wpr) return 0u;
  uint32_t lo = cas_src(a, b, 2 * r, 2 * w) | cas_src(a, b, 2 * r + 1, 2 * w);
  uint32_t hi = cas_src(a, b, 2 * r, 2 * w + 1) | cas_src(a, b, 2 * r + 1, 2 * w + 1);
  return pool_pairs((uint64_t)lo | ((uint64_t)hi << 32));
}

__device__ uint32_t cas_word(const CascadeArgs& a, int b, int r, int w) {
  uint32_t p = 0, c = 0, n = 0;
  int r0 = max(r - DIL, 0), r1 = min(r + DIL, a.rows - 1);
  for (int rr = r0; rr <= r1; ++rr) {
    p |= cas_down(a, b, rr, w - 1);
    c |= cas_down(a, b, rr, w);
    n |= cas_down(a, b, rr, w + 1);
  }
  return spread(p, c, n) & last_word_mask(a.cols, w);
}

__global__ void k_cascade(CascadeArgs a) {
  int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= a.rows * a.wpr) return;
  int b = a.batch[blockIdx.y];
  int r = idx / a.wpr, w = idx % a.wpr;
  uint32_t v = cas_word(a, b, r, w);
  if (a.fov && b == a.j) v &= cas_word(a, 0, r, w);
  a.dst[(uint64_t)b * a.dst_stride + idx] = v;
}

// ----------------------------------------------------------- footprint step
struct FootArgs {
  int j, L, H;
  int rows, cols, wpr;        // output level j-1
  int srows, swpr;            // source level j
  const uint32_t* V;          // valid at level j (nullptr: all ones)
  const uint32_t* D;          // detail mask level j
  uint32_t* out;              // level j-1
  const uint32_t* R;          // j == 1: requested rows
  int mh;
};

__device__ __forceinline__ uint32_t fp_up(const FootArgs& a, int r, int w) {
  // upsampled (V_j & D_j) word at level j-1, outside the grid = all set
  if (r < 0 || r >= a.rows || w < 0 || w >= a.wpr) return 0xFFFFFFFFu;
  int sr = r >> 1, sw = w >> 1;
  uint32_t s = a.D[(uint64_t)sr * a.swpr + sw];
  if (a.V) s &= a.V[(uint64_t)sr * a.swpr + sw];
  uint32_t v = double_bits(s >> (16 * (w & 1)));
  return v | ~last_word_mask(a.cols, w);
}

__global__ void k_footprint(FootArgs a) {
  int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= a.rows * a.wpr) return;
  int r = idx / a.wpr, w = idx % a.wpr;
  uint32_t p = ~0u, c = ~0u, n = ~0u;
  for (int rr = r - DIL; rr <= r + DIL; ++rr) {
    p &= fp_up(a, rr, w - 1);
    c &= fp_up(a, rr, w);
    n &= fp_up(a, rr, w + 1);
  }
  uint32_t v = shrink(p, c, n) & last_word_mask(a.cols, w);
  if (a.j == 1) v &= a.R[(uint64_t)((long long)r * a.mh / a.H) * a.wpr + w];
  a.out[idx] = v;
}

// -------------------------------------------------------------- block select
struct BlockArgs {
  int L, H, W, bs, nbx, NB, n, rs;
  const uint32_t* D[WV_MAX_LEVELS + 1];
  int dwpr[WV_MAX_LEVELS + 1];
  const unsigned long long* ends;   // (n, NB) u64
  unsigned long long rec_bytes;     // bytes after the table
  uint32_t* sel;
  uint32_t* prev_sel;
  uint32_t* loaded;
  uint32_t* list;
  uint32_t* list_count;
  unsigned long long* set_bytes;
  wv_frame_result* res;
  int account_only;
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
    int bh = a.H >> k, bw = a.W >> k;
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

__global__ void k_blocks(BlockArgs a) {
  const int lane = threadIdx.x & 31;
  const int wid = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int b0 = wid * 32;
  if (b0 >= a.NB) return;
  uint32_t selmask = 0;
  for (int i = 0; i < 32 && b0 + i < a.NB; ++i) {
    int b = b0 + i;
    int by = b / a.nbx, bx = b % a.nbx;
    int x0 = bx * a.bs, x1 = x0 + a.bs;
    bool any = false;
    for (int r = lane; r < a.bs; r += 32) any |= incl_row_any(a, by * a.bs + r, x0, x1);
    if (__any_sync(0xFFFFFFFFu, any)) selmask |= 1u << i;
  }
  const int b = b0 + lane;
  const bool valid = b < a.NB;
  const bool sel = valid && ((selmask >> lane) & 1u);
  const uint32_t word = b0 >> 5;
  const uint32_t prevw = a.prev_sel[word];
  const uint32_t loadw = a.loaded[word];
  const bool prev = valid && ((prevw >> lane) & 1u);
  const bool was = (loadw >> lane) & 1u;
  unsigned long long bytes = 0, recs = 0;
  uint32_t err = 0;
  if (sel) {
    for (int t = 0; t < a.n; ++t) {
      uint64_t i = (uint64_t)t * a.NB + b;
      unsigned long long e = a.ends[i];
      unsigned long long s = i ? a.ends[i - 1] : 0ull;
      if (e < s || e > a.rec_bytes || (e - s) % a.rs || (e - s) / a.rs > (unsigned long long)a.bs * a.bs)
        err |= WV_DERR_TABLE;
      else {
        bytes += e - s;
        recs += (e - s) / a.rs;
      }
    }
  }
  const bool missing = sel && !was;
  unsigned long long newb = missing ? bytes : 0ull;
  const bool emit = !a.account_only && (sel || prev);
  uint32_t emask = __ballot_sync(0xFFFFFFFFu, emit);
  uint32_t base = 0;
  if (lane == 0 && emask) base = atomicAdd(a.list_count, (uint32_t)__popc(emask));
  base = __shfl_sync(0xFFFFFFFFu, base, 0);
  if (emit) a.list[base + __popc(emask & ((1u << lane) - 1u))] = sel ? (uint32_t)b : ((uint32_t)b | ZERO_FLAG);
  uint32_t nmiss = __popc(__ballot_sync(0xFFFFFFFFu, missing));
  for (int o = 16; o; o >>= 1) {
    recs += __shfl_xor_sync(0xFFFFFFFFu, recs, o);
    newb += __shfl_xor_sync(0xFFFFFFFFu, newb, o);
    err |= __shfl_xor_sync(0xFFFFFFFFu, err, o);
  }
  if (lane == 0) {
    a.sel[word] = selmask;
    if (!a.account_only) a.prev_sel[word] = selmask;
    a.loaded[word] = loadw | selmask;
    if (recs) atomicAdd(&a.res->records, recs);
    if (newb) {
      atomicAdd(&a.res->new_bytes, newb);
      atomicAdd(a.set_bytes, newb);
    }
    if (nmiss) atomicAdd(&a.res->n_missing, nmiss);
    if (selmask) atomicAdd(&a.res->n_selected, (uint32_t)__popc(selmask));
    if (err) atomicOr(&a.res->error, err);
  }
}

// -------------------------------------------------------------- tile lists
struct TileArgs {
  int L, H, W, mh;
  int wpr0;
  const uint32_t* R;
  int full;
  int nty[WV_MAX_LEVELS + 1], ntx[WV_MAX_LEVELS + 1];
  uint8_t* need[WV_MAX_LEVELS + 1];
  uint32_t* list[WV_MAX_LEVELS + 1];
  uint8_t* prev_need;
  uint32_t* counters;                // CNT_TILES + k
};

__global__ void k_tiles(TileArgs a) {
  __shared__ uint32_t cnt;
  // level 1: tiles of the output pixels that touch the request
  const int nt1 = a.nty[1] * a.ntx[1];
  if (threadIdx.x == 0) cnt = 0;
  __syncthreads();
  for (int t = threadIdx.x; t < nt1; t += blockDim.x) {
    int ty = t / a.ntx[1], tx = t % a.ntx[1];
    bool nd = a.full != 0;
    if (!nd) {
      int y0 = ty * OUT_H, y1 = min(y0 + OUT_H, a.H);
      int c0 = tx * OUT_W, c1 = min(c0 + OUT_W, a.W);
      int m0 = (int)((long long)y0 * a.mh / a.H), m1 = (int)((long long)(y1 - 1) * a.mh / a.H);
      for (int m = m0; m <= m1 && !nd; ++m) {
        const uint32_t* row = a.R + (uint64_t)m * a.wpr0;
        for (int w = c0 >> 5; w <= ((c1 - 1) >> 5); ++w)
          if (row[w] & range_mask(c0, c1, w)) { nd = true; break; }
      }
    }
    bool pv = a.prev_need[t] != 0;
    a.need[1][t] = nd;
    a.prev_need[t] = nd;
    if (nd || pv) {
      uint32_t pos = atomicAdd(&cnt, 1u);
      a.list[1][pos] = (uint32_t)t | (nd ? 0u : ZERO_FLAG);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) a.counters[CNT_TILES + 1] = cnt;
  // coarser levels: a tile is needed if a needed finer tile reads its rows
  for (int k = 2; k <= a.L; ++k) {
    __syncthreads();
    if (threadIdx.x == 0) cnt = 0;
    __syncthreads();
    const int nt = a.nty[k] * a.ntx[k];
    const int fy = a.nty[k - 1], fx = a.ntx[k - 1];
    for (int t = threadIdx.x; t < nt; t += blockDim.x) {
      int u = t / a.ntx[k], v = t % a.ntx[k];
      bool nd = false;
      for (int ty = max(2 * u - 1, 0); ty <= min(2 * u + 2, fy - 1) && !nd; ++ty)
        for (int tx = max(2 * v - 1, 0); tx <= min(2 * v + 2, fx - 1); ++tx)
          if (a.need[k - 1][ty * fx + tx]) { nd = true; break; }
      a.need[k][t] = nd;
      if (nd) a.list[k][atomicAdd(&cnt, 1u)] = (uint32_t)t;
    }
    __syncthreads();
    if (threadIdx.x == 0) a.counters[CNT_TILES + k] = cnt;
  }
}

// result finalisation: cache-entry total after this call, level-1 tile count
__global__ void k_finalize(const uint8_t* need1, int nt1, const unsigned long long* set_bytes,
                           wv_frame_result* res) {
  __shared__ uint32_t c;
  if (threadIdx.x == 0) c = 0;
  __syncthreads();
  uint32_t mine = 0;
  if (need1)
    for (int t = threadIdx.x; t < nt1; t += blockDim.x) mine += need1[t] != 0;
  atomicAdd(&c, mine);
  __syncthreads();
  if (threadIdx.x == 0) {
    res->n_tiles = c;
    res->set_bytes = *set_bytes;
  }
}

}  // namespace

int launch_select(const Layout& lo, const wv_geometry* g, const wv_frame_args* a, uint8_t* ws,
                  cudaStream_t s) {
  const int L = lo.L, H = lo.H, W = lo.W;
  const bool full = a->mode == WV_MODE_FULL;
  const bool fov = a->mode == WV_MODE_FOVEATED;
  const bool acct = (a->flags & WV_FLAG_ACCOUNT_ONLY) != 0;
  if (!full && !a->d_mask) return WV_ERR_ARG;
  uint32_t* R = (uint32_t*)(ws + lo.mrows);
  uint32_t* counters = (uint32_t*)(ws + lo.counters);
  WV_CUDA(cudaMemsetAsync(counters, 0, 64 * 4, s));
  WV_CUDA(cudaMemsetAsync(a->d_result, 0, sizeof(wv_frame_result), s));
  {
    int n = lo.mh * lo.wpr_[0];
    k_mask_rows<<<cdiv(n, 256), 256, 0, s>>>(a->d_mask, R, lo.mh, lo.mw, W, lo.wpr_[0], full);
  }
  // level cascades (batch 0: request closure; batches k>=j: gaze windows)
  for (int j = 1; j <= L; ++j) {
    CascadeArgs c{};
    c.j = j; c.L = L; c.H = H;
    c.rows = H >> j; c.cols = W >> j; c.wpr = lo.wpr_[j];
    c.prow_n = H >> (j - 1); c.pcols = W >> (j - 1); c.pwpr = lo.wpr_[j - 1];
    c.src = j > 1 ? (const uint32_t*)(ws + lo.stack[j - 1]) : nullptr;
    c.src_stride = j > 1 ? lo.stack_stride[j - 1] / 4 : 0;
    c.R = R; c.mh = lo.mh;
    c.dst = (uint32_t*)(ws + lo.stack[j]);
    c.dst_stride = lo.stack_stride[j] / 4;
    c.fov = fov;
    c.nbatch = 0;
    c.batch[c.nbatch++] = 0;
    if (fov) {
      for (int k = j; k <= L; ++k) c.batch[c.nbatch++] = k;
      for (int k = 1; k <= L; ++k)
        for (int q = 0; q < 4; ++q) c.rect[k][q] = a->fovea[k - 1][q];
    }
    int n = c.rows * c.wpr;
    dim3 grid(cdiv(n, 256), c.nbatch);
    k_cascade<<<grid, 256, 0, s>>>(c);
  }
  auto Dptr = [&](int k) -> uint32_t* {
    return (uint32_t*)(ws + lo.stack[k] + (fov ? (uint64_t)k * lo.stack_stride[k] : 0));
  };
  // footprint: V_L = ones; V_{j-1} = shrink(up(V_j & D_j)); last & request
  for (int j = L; j >= 1 && !acct; --j) {
    FootArgs f{};
    f.j = j; f.L = L; f.H = H;
    f.rows = H >> (j - 1); f.cols = W >> (j - 1); f.wpr = lo.wpr_[j - 1];
    f.srows = H >> j; f.swpr = lo.wpr_[j];
    f.V = j == L ? nullptr : (const uint32_t*)(ws + lo.fp[j]);
    f.D = Dptr(j);
    f.out = j == 1 ? a->d_footprint : (uint32_t*)(ws + lo.fp[j - 1]);
    f.R = R; f.mh = lo.mh;
    int n = f.rows * f.wpr;
    k_footprint<<<cdiv(n, 256), 256, 0, s>>>(f);
  }
  {
    BlockArgs b{};
    b.L = L; b.H = H; b.W = W; b.bs = lo.bs; b.nbx = lo.nbx; b.NB = lo.NB; b.n = lo.n;
    b.rs = 2 + lo.C * (g->float_mode ? 4 : 1);
    for (int k = 1; k <= L; ++k) { b.D[k] = Dptr(k); b.dwpr[k] = lo.wpr_[k]; }
    uint64_t table = (uint64_t)lo.n * lo.NB * 8;
    if (a->payload_bytes < table) return WV_ERR_ARG;
    b.ends = (const unsigned long long*)a->d_payload;
    b.rec_bytes = a->payload_bytes - table;
    b.sel = (uint32_t*)(ws + lo.sel);
    b.prev_sel = (uint32_t*)(ws + lo.prev_sel);
    b.loaded = a->d_set_loaded;
    b.list = (uint32_t*)(ws + lo.blist);
    b.list_count = counters + CNT_BLOCKS;
    b.set_bytes = a->d_set_bytes;
    b.res = a->d_result;
    b.account_only = acct;
    int warps = cdiv(lo.NB, 32);
    k_blocks<<<cdiv(warps * 32, 256), 256, 0, s>>>(b);
  }
  if (acct) {
    k_finalize<<<1, 32, 0, s>>>(nullptr, 0, a->d_set_bytes, a->d_result);
  } else {
    TileArgs t{};
    t.L = L; t.H = H; t.W = W; t.mh = lo.mh; t.wpr0 = lo.wpr_[0]; t.R = R; t.full = full;
    for (int k = 1; k <= L; ++k) {
      t.nty[k] = lo.nty[k]; t.ntx[k] = lo.ntx[k];
      t.need[k] = ws + lo.need[k];
      t.list[k] = (uint32_t*)(ws + lo.tlist[k]);
    }
    t.prev_need = ws + lo.prev_need;
    t.counters = counters;
    k_tiles<<<1, 1024, 0, s>>>(t);
    k_finalize<<<1, 256, 0, s>>>(ws + lo.need[1], lo.nty[1] * lo.ntx[1], a->d_set_bytes,
                                 a->d_result);
  }
  WV_CUDA(cudaGetLastError());
  return WV_OK;
}

}  // namespace wv
