// K2 — fused dequantisation + inverse temporal Haar + inclusion masking.
//
// One CTA-iteration per work-list block (persistent grid).  For display time
// t the reference adds, per coefficient position, the signed records of the
// log2(n)+1 live temporal indices in ascending index order starting from
// +0.0 (decoding.py:53-90: weights :72-80, np.add.at :87-89), after
// dequantising each record as cmin + (q/255)*(cmax-cmin) with per-coefficient
// approx/detail extrema (decoding.py:37-50).  The block is accumulated in
// shared memory in exactly that order with IEEE round-to-nearest ops (no
// FMA contraction), multiplied by the inclusion bit of its level mask
// (wavelets.py:372-378) and written to the planar C x H x W coefficient
// plane with 16-byte coalesced stores.  Blocks selected last frame but not
// this one are zero-filled instead, so every unselected block of the plane is
// zero and the synthesis kernels read the plane without a selection lookup.
#include "wv_common.cuh"

namespace wv {
namespace {

struct TemporalArgs {
  int L, H, W, C, bs, bs_log2, nbx, n, rs, float_mode;
  const wv_frame_args* fa;          // t, payload (table + records), extrema, result
  unsigned long long table_bytes;
  const uint32_t* D[WV_MAX_LEVELS + 1];
  int dwpr[WV_MAX_LEVELS + 1];
  const uint32_t* list;
  const uint32_t* count;
  int NB;
  float* plane;
  uint8_t* bstate;                  // per block: the plane block may hold nonzeros
  int all_included;                 // full-frame decode: every inclusion bit is set
};

// inclusion bit of plane position (y, x) (LevelMaskSet.inclusion_grid)
__device__ __forceinline__ uint32_t included(const TemporalArgs& a, int y, int x) {
  for (int k = 1; k <= a.L; ++k) {
    const int bh = a.H >> k, bw = a.W >> k;
    if (y >= bh || x >= bw) {
      const int r = y >= bh ? y - bh : y;
      const int c = x >= bw ? x - bw : x;
      return (a.D[k][(uint64_t)r * a.dwpr[k] + (c >> 5)] >> (c & 31)) & 1u;
    }
  }
  return 1u;  // approximation band: always included
}

// Where a whole block sits inside one subband quadrant of one level (or in
// the approximation band) its inclusion bits are a straight slice of that
// level's mask rows; blocks straddling quadrants use the per-position path.
struct BlockIncl {
  int mode;            // 0: all included, 1: slice of D[k], 2: per position
  const uint32_t* rows;
  int wpr, r0, c0;
};

__device__ __forceinline__ BlockIncl classify(const TemporalArgs& a, int y0, int x0) {
  BlockIncl bi{2, nullptr, 0, 0, 0};
  const int y1 = y0 + a.bs, x1 = x0 + a.bs;
  if (y1 <= (a.H >> a.L) && x1 <= (a.W >> a.L)) { bi.mode = 0; return bi; }
  for (int k = 1; k <= a.L; ++k) {
    const int bh = a.H >> k, bw = a.W >> k;
    const bool top = y1 <= bh, bot = y0 >= bh && y1 <= 2 * bh;
    const bool left = x1 <= bw, right = x0 >= bw && x1 <= 2 * bw;
    if ((top && right) || (bot && (left || right))) {
      bi.mode = 1;
      bi.rows = a.D[k];
      bi.wpr = a.dwpr[k];
      bi.r0 = bot ? y0 - bh : y0;
      bi.c0 = right ? x0 - bw : x0;
      return bi;
    }
    if (!(y1 <= bh && x1 <= bw)) return bi;   // straddles this level's quadrants
  }
  return bi;
}

// temporal Mallat index ti contributes to display time t with sign
// (+1/-1) or not at all (0) (encoding.py:187-195, decoding.py:72-80)
__device__ __forceinline__ int tweight(int ti, int t, int n) {
  if (ti == 0) return 1;
  const int big = 31 - __clz(n);
  const int lvl = big - (31 - __clz(ti));
  if ((t >> lvl) != ti - (1 << (big - lvl))) return 0;
  return ((t >> (lvl - 1)) & 1) ? -1 : 1;
}

// One CTA (256 threads) per work-list block (K1 lists only blocks with
// records or with stale nonzeros).  Warp 0 reads the block's BlockEnd spans
// and prefix-sums them; blocks without a record of a contributing temporal
// index are zero (cleared only if the plane block still holds nonzeros).
// Otherwise the records are added into a shared-memory block temporal index
// by temporal index (ascending, the np.add.at order), all records of one
// index concurrently, and the inclusion-masked block is written with 16-byte
// stores.
#ifndef WV_K2_THREADS
#define WV_K2_THREADS 256
#endif
constexpr int K2_THREADS = WV_K2_THREADS;
#ifndef WV_K2_STAGED
#define WV_K2_STAGED 0   // staged K2 (k_temporal_staged) where the geometry allows
#endif
constexpr int K2_MAXN = 32;

__global__ void __launch_bounds__(K2_THREADS) k_temporal(TemporalArgs a) {
  pdl_sync();
  const int t_disp = a.fa->t;
  const unsigned long long* __restrict__ ends = (const unsigned long long*)a.fa->d_payload;
  const uint8_t* __restrict__ recs = (const uint8_t*)a.fa->d_payload + a.table_bytes;
  const float* __restrict__ extrema = a.fa->d_extrema;
  extern __shared__ float4 smem4[];
  float* acc = reinterpret_cast<float*>(smem4);              // C x bs*bs
  __shared__ unsigned long long s_start[K2_MAXN];
  __shared__ int s_pre[K2_MAXN + 1];
  __shared__ int s_w[K2_MAXN];
  __shared__ uint32_t s_mrow[32];
  __shared__ int s_live;
  __shared__ float s_q255[256];   // q / 255.0f, IEEE division (encoding.py:270-271)
  for (int q = threadIdx.x; q < 256; q += blockDim.x) s_q255[q] = __fdiv_rn((float)q, 255.0f);
  const int tid = threadIdx.x;
  const int npos = a.bs * a.bs;
  const int nq = (a.C * npos) >> 2;                           // float4 per block
  const uint32_t count = *a.count;
  // cache entry total after this call's block selection (decoding.py:231)
  if (blockIdx.x == 0 && threadIdx.x == 0) a.fa->d_result->set_bytes = *a.fa->d_set_bytes;
  const int ah = a.H >> a.L, aw = a.W >> a.L;
  const int bmask = a.bs - 1;
  uint32_t err = 0;
  for (uint32_t item = blockIdx.x; item < count; item += gridDim.x) {
    const uint32_t e = a.list[item];
    const int b = (int)(e & ~ZERO_FLAG);
    const int by = b / a.nbx;
    const int y0 = by * a.bs, x0 = (b - by * a.nbx) * a.bs;
    const bool dirty = a.bstate[b] != 0;
    auto zero_block = [&]() {
      for (int q = tid; q < nq; q += K2_THREADS) {
        const int c = (q << 2) >> (2 * a.bs_log2), i = (q << 2) & (npos - 1);
        float* dst = a.plane + ((uint64_t)c * a.H + y0 + (i >> a.bs_log2)) * a.W + x0 + (i & bmask);
        *reinterpret_cast<float4*>(dst) = make_float4(0.f, 0.f, 0.f, 0.f);
      }
    };
    if (e & ZERO_FLAG) {
      // block left the selection: clear it unless it is already all zero
      if (dirty) {
        zero_block();
        __syncthreads();   // every thread has read the state byte
        if (tid == 0) a.bstate[b] = 0;
      }
      continue;
    }
    // spans of the block's records per temporal index; warp 0 prefix-sums
    // the counts (n <= 32) and the weights of display time t
    if (tid < 32) {
      int cnt = 0, w = 0;
      unsigned long long st = 0;
      if (tid < a.n) {
        const uint64_t fi = (uint64_t)tid * a.NB + b;
        const unsigned long long en = ends[fi];
        st = fi ? ends[fi - 1] : 0ull;
        // spans past the record bytes or misaligned are skipped (k_blocks
        // reports them as WV_DERR_TABLE)
        if (en >= st && en <= a.fa->payload_bytes - a.table_bytes && (en - st) % a.rs == 0)
          cnt = (int)min((en - st) / a.rs, (unsigned long long)npos);
        w = tweight(tid, t_disp, a.n);
      }
      int inc = cnt, live = w ? cnt : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int u = __shfl_up_sync(0xFFFFFFFFu, inc, o), l = __shfl_up_sync(0xFFFFFFFFu, live, o);
        if (tid >= o) {
          inc += u;
          live += l;
        }
      }
      if (tid < a.n) {
        s_start[tid] = st;
        s_pre[tid + 1] = inc;
        s_w[tid] = w;
      }
      if (tid == 0) s_pre[0] = 0;
      if (tid == 31) s_live = live;
    }
    __syncthreads();
    const int total = s_pre[a.n];
    if (s_live == 0) {
      // no record of a contributing temporal index: the block is zero
      // (offsets of the other records are still validated, decoding.py:64-69)
      for (int i = tid; i < total; i += K2_THREADS) {
        int ti = 0;
        while (s_pre[ti + 1] <= i) ++ti;
        const uint8_t* rp = recs + s_start[ti] + (uint64_t)(i - s_pre[ti]) * a.rs;
        if (((int)rp[0] | ((int)rp[1] << 8)) >= npos) err |= WV_DERR_OFFSET;
      }
      if (dirty) zero_block();
      __syncthreads();
      if (tid == 0 && dirty) a.bstate[b] = 0;
      continue;
    }
    const BlockIncl bi = a.all_included ? BlockIncl{0, nullptr, 0, 0, 0} : classify(a, y0, x0);
    if (bi.mode == 1 && a.bs <= 32 && tid < a.bs) {
      const int cc = bi.c0;
      const uint32_t* row = bi.rows + (uint64_t)(bi.r0 + tid) * bi.wpr;
      const uint32_t lo = row[cc >> 5];
      const uint32_t hi = ((cc & 31) + a.bs > 32) ? row[(cc >> 5) + 1] : 0u;
      s_mrow[tid] = (uint32_t)(((((uint64_t)hi) << 32) | lo) >> (cc & 31));
    }
    for (int q = tid; q < nq; q += K2_THREADS)
      smem4[q] = make_float4(0.f, 0.f, 0.f, 0.f);
    __syncthreads();
    if (tid == 0 && !dirty) a.bstate[b] = 1;
    // temporal index by temporal index, ascending (the np.add.at order);
    // within one index every position has at most one record, so its
    // records are added concurrently
    for (int tt = 0; tt < a.n; ++tt) {
      const int cnt = s_pre[tt + 1] - s_pre[tt];
      if (cnt == 0) continue;
      const int w = s_w[tt];
      const uint8_t* rbase = recs + s_start[tt];
      if (!w) {
        // not summed for this display time; offsets are still validated
        for (int i = tid; i < cnt; i += K2_THREADS) {
          const uint8_t* rp = rbase + (uint64_t)i * a.rs;
          if (((int)rp[0] | ((int)rp[1] << 8)) >= npos) err |= WV_DERR_OFFSET;
        }
        continue;
      }
      float lo_a[4], d_a[4], lo_d[4], d_d[4];   // cmin, cmax - cmin: approx / detail
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        lo_a[c] = d_a[c] = lo_d[c] = d_d[c] = 0.0f;
        if (c < a.C && !a.float_mode) {
          const float* ex = extrema + ((uint64_t)tt * a.C + c) * 4;
          lo_a[c] = ex[0];
          d_a[c] = __fsub_rn(ex[1], ex[0]);
          lo_d[c] = ex[2];
          d_d[c] = __fsub_rn(ex[3], ex[2]);
        }
      }
#pragma unroll 4
      for (int i = tid; i < cnt; i += K2_THREADS) {
        const uint8_t* rp = rbase + (uint64_t)i * a.rs;
        const int off = (int)rp[0] | ((int)rp[1] << 8);
        if (off >= npos) {
          err |= WV_DERR_OFFSET;
          continue;
        }
        const int yy = y0 + (off >> a.bs_log2), xx = x0 + (off & bmask);
        const bool appr = yy < ah && xx < aw;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          if (c < a.C) {
            float x;
            if (a.float_mode) {
              const uint8_t* q = rp + 2 + 4 * c;
              x = __uint_as_float((uint32_t)q[0] | ((uint32_t)q[1] << 8) |
                                  ((uint32_t)q[2] << 16) | ((uint32_t)q[3] << 24));
            } else {
              // cmin + (q / 255) * (cmax - cmin), q / 255 from the IEEE table
              x = __fadd_rn(appr ? lo_a[c] : lo_d[c],
                            __fmul_rn(s_q255[rp[2 + c]], appr ? d_a[c] : d_d[c]));
            }
            acc[c * npos + off] = __fadd_rn(acc[c * npos + off], w > 0 ? x : -x);
          }
        }
      }
      __syncthreads();
    }
    // write: inclusion-masked, 4 consecutive positions per thread-step; the
    // block's mask rows (bs <= 32) were staged in shared memory up front
    const int npos_log2 = 2 * a.bs_log2;
    for (int q = tid; q < nq; q += K2_THREADS) {
      const int e4 = q << 2;
      const int c = e4 >> npos_log2, i = e4 & (npos - 1);
      const int ly = i >> a.bs_log2, lx = i & bmask;
      const int yy = y0 + ly, xx = x0 + lx;
      uint32_t m4;
      if (bi.mode == 0) {
        m4 = 0xFu;
      } else if (bi.mode == 1 && a.bs <= 32) {
        m4 = (s_mrow[ly] >> lx) & 0xFu;
      } else if (bi.mode == 1) {
        const int cc = bi.c0 + lx;
        const uint32_t* row = bi.rows + (uint64_t)(bi.r0 + ly) * bi.wpr;
        const uint32_t lo = row[cc >> 5];
        const uint32_t hi = (cc & 31) > 28 ? row[(cc >> 5) + 1] : 0u;
        m4 = (uint32_t)(((((uint64_t)hi) << 32) | lo) >> (cc & 31)) & 0xFu;
      } else {
        m4 = included(a, yy, xx) | (included(a, yy, xx + 1) << 1) |
             (included(a, yy, xx + 2) << 2) | (included(a, yy, xx + 3) << 3);
      }
      const float4 v = smem4[q];
      float4 o;
      o.x = __fmul_rn(v.x, (m4 & 1u) ? 1.0f : 0.0f);
      o.y = __fmul_rn(v.y, (m4 & 2u) ? 1.0f : 0.0f);
      o.z = __fmul_rn(v.z, (m4 & 4u) ? 1.0f : 0.0f);
      o.w = __fmul_rn(v.w, (m4 & 8u) ? 1.0f : 0.0f);
      *reinterpret_cast<float4*>(a.plane + ((uint64_t)c * a.H + yy) * a.W + xx) = o;
    }
    __syncthreads();
  }
  for (int o = 16; o; o >>= 1) err |= __shfl_xor_sync(0xFFFFFFFFu, err, o);
  if ((tid & 31) == 0 && err) atomicOr(&a.fa->d_result->error, err);
}

// ------------------------------------------------------------ K2, staged
// Default K2 (bs <= 32, records staged in shared memory).  Per work-list
// block, one 128-thread CTA iteration:
//   1. warp 0 reads the n BlockEnd spans, validates them against the record
//      bytes (a span past the payload or misaligned is skipped and flagged
//      WV_DERR_TABLE), and lays the spans out in a shared staging buffer;
//   2. all threads copy the spans' covering 16-byte chunks with 128-bit
//      loads (one pass over the block's records, every span in flight at
//      once);
//   3. every record's offset is checked (offset >= bs^2 -> WV_DERR_OFFSET)
//      and, for the temporal indices that contribute to display time t, its
//      staging position is scattered into that index's slot table (within
//      one temporal index positions are unique);
//   4. each thread owns 4 consecutive positions and sums, per channel, the
//      present records of the contributing indices in ascending index order
//      from +0.0 -- exactly the np.add.at order of the reference
//      (decoding.py:87-89) -- dequantising on the fly (decoding.py:37-50),
//      then applies the inclusion mask and stores float4s.
// Three barriers per block, none per temporal index.
constexpr int K2S_THREADS = 128;
constexpr int K2S_MAXLIVE = 6;      // log2(32) + 1 contributing indices at most

struct K2Smem {
  unsigned long long st[K2_MAXN];   // span start (record bytes)
  uint32_t sbase[K2_MAXN];          // staging byte offset of the span's first record
  uint32_t cpre[K2_MAXN + 1];       // 16-byte chunks before span k
  uint32_t rpre[K2_MAXN + 1];       // records before span k
  uint32_t c0[K2_MAXN];             // first payload chunk of span k
  int slot[K2_MAXN];                // contributing slot of span k, or -1
  int w[K2_MAXN];
  int nlive, anylive;
  float ext[K2S_MAXLIVE][4][4];     // per slot, channel: cmin_a, dmax_a, cmin_d, dmax_d
  float q255[256];
};

__global__ void __launch_bounds__(K2S_THREADS) k_temporal_staged(TemporalArgs a, int stage_bytes) {
  pdl_sync();
  const int t_disp = a.fa->t;
  const unsigned long long* __restrict__ ends = (const unsigned long long*)a.fa->d_payload;
  const uint4* __restrict__ pay4 = (const uint4*)a.fa->d_payload;
  const unsigned long long tb = a.table_bytes;
  const unsigned long long rec_bytes = a.fa->payload_bytes - tb;
  const float* __restrict__ extrema = a.fa->d_extrema;
  extern __shared__ uint4 dyn4[];
  uint8_t* stage = reinterpret_cast<uint8_t*>(dyn4);
  uint16_t* idx = reinterpret_cast<uint16_t*>(stage + stage_bytes);   // [slot][npos]
  __shared__ K2Smem sm;
  __shared__ uint32_t s_mrow[32];
  const int tid = threadIdx.x;
  for (int q = tid; q < 256; q += K2S_THREADS) sm.q255[q] = __fdiv_rn((float)q, 255.0f);
  const int npos = a.bs * a.bs;
  const int bmask = a.bs - 1;
  const int nq = (a.C * npos) >> 2;
  const uint32_t count = *a.count;
  if (blockIdx.x == 0 && tid == 0) a.fa->d_result->set_bytes = *a.fa->d_set_bytes;
  const int ah = a.H >> a.L, aw = a.W >> a.L;
  uint32_t err = 0;
  for (uint32_t item = blockIdx.x; item < count; item += gridDim.x) {
    const uint32_t e = a.list[item];
    const int b = (int)(e & ~ZERO_FLAG);
    const int by = b / a.nbx;
    const int y0 = by * a.bs, x0 = (b - by * a.nbx) * a.bs;
    const bool dirty = a.bstate[b] != 0;
    float* const pblk = a.plane + (uint64_t)y0 * a.W + x0;
    auto zero_block = [&]() {
      for (int q = tid; q < nq; q += K2S_THREADS) {
        const int c = (q << 2) >> (2 * a.bs_log2), i = (q << 2) & (npos - 1);
        *reinterpret_cast<float4*>(pblk + ((uint64_t)c * a.H + (i >> a.bs_log2)) * a.W +
                                   (i & bmask)) = make_float4(0.f, 0.f, 0.f, 0.f);
      }
    };
    if (e & ZERO_FLAG) {
      if (dirty) {
        zero_block();
        __syncthreads();
        if (tid == 0) a.bstate[b] = 0;
      }
      continue;
    }
    // 1. spans (warp 0; n <= 32)
    if (tid < 32) {
      int cnt = 0, w = 0;
      uint32_t nch = 0, c0 = 0;
      unsigned long long st = 0;
      if (tid < a.n) {
        const uint64_t fi = (uint64_t)tid * a.NB + b;
        const unsigned long long en = ends[fi];
        st = fi ? ends[fi - 1] : 0ull;
        if (en < st || en > rec_bytes || (en - st) % a.rs ||
            (en - st) / a.rs > (unsigned long long)npos) {
          err |= WV_DERR_TABLE;
        } else if (en > st) {
          cnt = (int)((en - st) / a.rs);
          c0 = (uint32_t)((tb + st) >> 4);
          nch = (uint32_t)(((tb + en + 15) >> 4) - c0);
        }
        w = tweight(tid, t_disp, a.n);
      }
      uint32_t cinc = nch, rinc = (uint32_t)cnt, linc = w != 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t u = __shfl_up_sync(0xFFFFFFFFu, cinc, o);
        const uint32_t v = __shfl_up_sync(0xFFFFFFFFu, rinc, o);
        const uint32_t l = __shfl_up_sync(0xFFFFFFFFu, linc, o);
        if (tid >= o) {
          cinc += u;
          rinc += v;
          linc += l;
        }
      }
      const bool live = w != 0 && cnt > 0;
      const uint32_t anyl = __ballot_sync(0xFFFFFFFFu, live);
      if (tid < a.n) {
        sm.st[tid] = st;
        sm.c0[tid] = c0;
        sm.cpre[tid + 1] = cinc;
        sm.rpre[tid + 1] = rinc;
        sm.sbase[tid] = 16u * (cinc - nch) + (uint32_t)((tb + st) & 15u);
        sm.w[tid] = w;
        sm.slot[tid] = w ? (int)linc - 1 : -1;
        if (w) {
          // dequantisation constants of this temporal index (decoding.py:44-49)
          for (int c = 0; c < a.C; ++c) {
            const float* ex = extrema + ((uint64_t)tid * a.C + c) * 4;
            float* d = sm.ext[linc - 1][c];
            if (a.float_mode) {
              d[0] = d[1] = d[2] = d[3] = 0.0f;
            } else {
              d[0] = ex[0];
              d[1] = __fsub_rn(ex[1], ex[0]);
              d[2] = ex[2];
              d[3] = __fsub_rn(ex[3], ex[2]);
            }
          }
        }
      }
      if (tid == 0) {
        sm.cpre[0] = 0;
        sm.rpre[0] = 0;
      }
      if (tid == 31) {
        sm.nlive = (int)linc;
        sm.anylive = anyl != 0;
      }
    }
    __syncthreads();
    const int n = a.n;
    const uint32_t nchunks = sm.cpre[n], nrec = sm.rpre[n];
    if (!sm.anylive) {
      // no record of a contributing temporal index: the block is zero
      // (the other records' offsets are still validated, decoding.py:64-69)
      for (uint32_t i = tid; i < nrec; i += K2S_THREADS) {
        int k = 0;
        while (sm.rpre[k + 1] <= i) ++k;
        const uint8_t* rp = (const uint8_t*)a.fa->d_payload + tb + sm.st[k] +
                            (uint64_t)(i - sm.rpre[k]) * a.rs;
        if (((int)rp[0] | ((int)rp[1] << 8)) >= npos) err |= WV_DERR_OFFSET;
      }
      if (dirty) zero_block();
      __syncthreads();
      if (tid == 0 && dirty) a.bstate[b] = 0;
      continue;
    }
    // 2. stage the spans (128-bit loads) and clear the slot tables
    for (uint32_t q = tid; q < nchunks; q += K2S_THREADS) {
      int k = 0;
      while (sm.cpre[k + 1] <= q) ++k;
      dyn4[q] = pay4[sm.c0[k] + (q - sm.cpre[k])];
    }
    const int nlive = sm.nlive;
    {
      uint4* id4 = reinterpret_cast<uint4*>(idx);
      const int n4 = (nlive * npos) >> 3;
      for (int q = tid; q < n4; q += K2S_THREADS) id4[q] = make_uint4(~0u, ~0u, ~0u, ~0u);
    }
    const BlockIncl bi = a.all_included ? BlockIncl{0, nullptr, 0, 0, 0} : classify(a, y0, x0);
    if (bi.mode == 1 && tid < a.bs) {
      const int cc = bi.c0;
      const uint32_t* row = bi.rows + (uint64_t)(bi.r0 + tid) * bi.wpr;
      const uint32_t lo = row[cc >> 5];
      const uint32_t hi = ((cc & 31) + a.bs > 32) ? row[(cc >> 5) + 1] : 0u;
      s_mrow[tid] = (uint32_t)(((((uint64_t)hi) << 32) | lo) >> (cc & 31));
    }
    __syncthreads();
    if (tid == 0 && !dirty) a.bstate[b] = 1;
    // 3. offsets: validate all, scatter the contributing ones
    for (uint32_t i = tid; i < nrec; i += K2S_THREADS) {
      int k = 0;
      while (sm.rpre[k + 1] <= i) ++k;
      const uint32_t pos = sm.sbase[k] + (i - sm.rpre[k]) * a.rs;
      const int off = (int)stage[pos] | ((int)stage[pos + 1] << 8);
      if (off >= npos) {
        err |= WV_DERR_OFFSET;
        continue;
      }
      const int sl = sm.slot[k];
      if (sl >= 0) idx[sl * npos + off] = (uint16_t)pos;
    }
    __syncthreads();
    // 4. per position: ascending contributing indices, then inclusion + store
    for (int g = tid; g < (npos >> 2); g += K2S_THREADS) {
      const int i0 = g << 2;
      const int ly = i0 >> a.bs_log2, lx = i0 & bmask;
      const int yy = y0 + ly, xx = x0 + lx;
      float acc[4][4];
#pragma unroll
      for (int c = 0; c < 4; ++c)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[c][j] = 0.0f;
      for (int k = 0; k < n; ++k) {
        const int sl = sm.slot[k];
        if (sl < 0) continue;
        const bool neg = sm.w[k] < 0;
        const uint2 pp = *reinterpret_cast<const uint2*>(idx + sl * npos + i0);
        const uint32_t ps[4] = {pp.x & 0xFFFFu, pp.x >> 16, pp.y & 0xFFFFu, pp.y >> 16};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          if (ps[j] == 0xFFFFu) continue;
          const bool ap = yy < ah && xx + j < aw;   // approximation band (decoding.py:44)
          const uint8_t* rp = stage + ps[j] + 2;
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            if (c < a.C) {
              float x;
              if (a.float_mode) {
                const uint8_t* q = rp + 4 * c;
                x = __uint_as_float((uint32_t)q[0] | ((uint32_t)q[1] << 8) |
                                    ((uint32_t)q[2] << 16) | ((uint32_t)q[3] << 24));
              } else {
                const float* ex = sm.ext[sl][c];
                x = __fadd_rn(ap ? ex[0] : ex[2], __fmul_rn(sm.q255[rp[c]], ap ? ex[1] : ex[3]));
              }
              acc[c][j] = __fadd_rn(acc[c][j], neg ? -x : x);
            }
          }
        }
      }
      uint32_t m4;
      if (bi.mode == 0) {
        m4 = 0xFu;
      } else if (bi.mode == 1) {
        m4 = (s_mrow[ly] >> lx) & 0xFu;
      } else {
        m4 = included(a, yy, xx) | (included(a, yy, xx + 1) << 1) |
             (included(a, yy, xx + 2) << 2) | (included(a, yy, xx + 3) << 3);
      }
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        if (c < a.C) {
          float4 o;
          o.x = __fmul_rn(acc[c][0], (m4 & 1u) ? 1.0f : 0.0f);
          o.y = __fmul_rn(acc[c][1], (m4 & 2u) ? 1.0f : 0.0f);
          o.z = __fmul_rn(acc[c][2], (m4 & 4u) ? 1.0f : 0.0f);
          o.w = __fmul_rn(acc[c][3], (m4 & 8u) ? 1.0f : 0.0f);
          *reinterpret_cast<float4*>(pblk + ((uint64_t)c * a.H + ly) * a.W + lx) = o;
        }
      }
    }
    __syncthreads();
  }
  for (int o = 16; o; o >>= 1) err |= __shfl_xor_sync(0xFFFFFFFFu, err, o);
  if ((tid & 31) == 0 && err) atomicOr(&a.fa->d_result->error, err);
}

}  // namespace

int launch_temporal(const Layout& lo, const wv_geometry* g, int mode, const wv_frame_args* fa,
                    uint8_t* ws, cudaStream_t s) {
  if (lo.bs < 4) return WV_ERR_UNSUPPORTED;
  if (lo.n > K2_MAXN) return WV_ERR_UNSUPPORTED;
  TemporalArgs t{};
  t.L = lo.L; t.H = lo.H; t.W = lo.W; t.C = lo.C; t.bs = lo.bs; t.nbx = lo.nbx; t.n = lo.n;
  t.bs_log2 = 31 - __builtin_clz((unsigned)lo.bs);
  t.float_mode = g->float_mode; t.rs = 2 + lo.C * (g->float_mode ? 4 : 1);
  t.NB = lo.NB;
  t.fa = fa;
  t.table_bytes = (unsigned long long)lo.n * lo.NB * 8;
  const bool fov = mode == WV_MODE_FOVEATED;
  t.all_included = mode == WV_MODE_FULL;
  for (int k = 1; k <= lo.L; ++k) {
    t.D[k] = (const uint32_t*)(ws + lo.stack[k] + (fov ? (uint64_t)k * lo.stack_stride[k] : 0));
    t.dwpr[k] = lo.wpr_[k];
  }
  t.list = (const uint32_t*)(ws + lo.blist);
  t.count = (const uint32_t*)(ws + lo.counters) + CNT_BLOCKS;
  t.plane = (float*)(ws + lo.plane);
  t.bstate = ws + lo.bstate;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  // staged kernel: the block's spans (<= n * bs^2 records) fit the staging
  // buffer with 16-bit positions
  const int rs = t.rs, npos = lo.bs * lo.bs;
  const int nlive = (31 - __builtin_clz((unsigned)lo.n)) + 1;
  const long stage_bytes = ((long)lo.n * npos * rs + 32L * lo.n + 15) & ~15L;
  const long staged_smem = stage_bytes + (long)nlive * npos * 2;
  if (WV_K2_STAGED && lo.bs <= 32 && nlive <= K2S_MAXLIVE && stage_bytes < 65536 &&
      staged_smem <= 160 * 1024) {
    static int occ_s = 0;
    static long occ_smem = -1;
    if (occ_smem != staged_smem) {
      WV_CUDA(cudaFuncSetAttribute(k_temporal_staged, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)staged_smem));
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_s, k_temporal_staged, K2S_THREADS,
                                                    (size_t)staged_smem);
      occ_smem = staged_smem;
    }
    const int grid = max(1, min(lo.NB, sms * max(occ_s, 1)));
    WV_CUDA(launch_k(k_temporal_staged, dim3(grid), dim3(K2S_THREADS), (size_t)staged_smem, s, t,
                     (int)stage_bytes));
    WV_CUDA(cudaGetLastError());
    return WV_OK;
  }
  const size_t smem = (size_t)lo.C * lo.bs * lo.bs * 4;
  if (smem > 48 * 1024)
    WV_CUDA(cudaFuncSetAttribute(k_temporal, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int occ = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_temporal, K2_THREADS, smem);
  const int grid = max(1, min(lo.NB, sms * max(occ, 1)));
  WV_CUDA(launch_k(k_temporal, dim3(grid), dim3(K2_THREADS), smem, s, t));
  WV_CUDA(cudaGetLastError());
  return WV_OK;
}

}  // namespace wv
