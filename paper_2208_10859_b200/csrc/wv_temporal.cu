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
        if (en >= st && (en - st) % a.rs == 0) cnt = (int)min((en - st) / a.rs, (unsigned long long)npos);
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
