// Encoder for one inter-frame set: the mirror of the decode path
// (SURVEY.md §8f row 2).
//
// Reference: encode_video (encoding.py:377-425) per set -- frames/255,
// analyze_2d (wavelets.py:128-149, analyze_1d :44-65), sparsify
// (encoding.py:118-135), haar_time_forward (:153-169), temporal_threshold
// (:198-236), compute_extrema (:239-254), quantize (:296-332) with records
// sorted by (t, block, layer, offset), and the BlockEnd counts
// (fileio.py:142-165).  Every float32 operation is a separately rounded
// IEEE op in the reference's order (this TU is built with --fmad=false and
// uses explicit _rn intrinsics), so the payload bytes equal the reference's.
//
// Kernels (one set, n frames, C channels, H x W; 2L + 7 launches):
//   E1 k_rows_u8   level-1 row lifting straight from the u8 frames (x / 255
//                  from a table of the IEEE quotients), warp chunks staged in
//                  shared memory for coalesced loads and stores
//   E2 k_rows /    levels 2..L rows (planes -> tmp, same warp chunks) and
//      k_cols      every level's columns (tmp -> planes, adjacent threads on
//                  adjacent columns); each lane lifts a 16-pair segment from
//                  a 2-pair halo (the analysis support)
//   E3 k_point     per 32x32 block, per position: spatial threshold of each
//                  frame (channel max magnitude vs level threshold + H(y)),
//                  temporal Haar forward in Mallat order, temporal
//                  threshold; emits nonzero bits, (t, block) record counts
//                  and the per-(t, c) approximation / detail extrema
//   E4 k_scan*     exclusive scan of the counts -> first record of each block
//   E5 k_emit      per (t, block) with records: rank by (layer, offset),
//                  quantise, write
#include <cuda_runtime.h>

#include <cstdint>

#include "wavevid_b200.h"
#include "wv_common.cuh"

namespace wv {
namespace {

// analyze_1d constants (wavelets.py:16-22) as float32, like the reference's
// numpy float32 arithmetic with Python-float scalars
constexpr float kA = (float)-1.586134342059924;
constexpr float kB = (float)-0.052980118572961;
constexpr float kG = (float)0.882911075530934;
constexpr float kD = (float)0.443506852043971;
constexpr float kK = (float)1.230174104914001;
constexpr float kIK = (float)(1.0 / 1.230174104914001);

constexpr int SEG = 16;         // output pairs per lifting segment
constexpr int LOC = SEG + 4;    // local pairs: 2-pair halo left, 2 right

struct EncLayout {
  size_t planes, tmp, starts, ext_bits, partials, nzbits, total;
};

__host__ __device__ inline int nb_x(const wv_encode_params& p) { return p.width / p.block_size; }
__host__ __device__ inline int nb_all(const wv_encode_params& p) {
  return (p.width / p.block_size) * (p.height / p.block_size);
}

EncLayout enc_layout(const wv_encode_params& p) {
  EncLayout L{};
  size_t off = 0;
  auto take = [&](size_t bytes) {
    const size_t o = off;
    off += (bytes + 255) / 256 * 256;
    return o;
  };
  const size_t plane = (size_t)p.width * p.height;
  const size_t nblk = (size_t)p.inter_size * nb_all(p);
  L.planes = take(plane * p.channels * p.inter_size * 4);
  L.tmp = take(plane * p.channels * p.inter_size * 4);
  L.starts = take(nblk * 8);
  L.ext_bits = take((size_t)p.inter_size * p.channels * 4 * 4);
  L.partials = take(((nblk + 1023) / 1024 + 1) * 8);
  L.nzbits = take(nblk * ((size_t)(p.block_size * p.block_size + 31) / 32) * 4);
  L.total = off;
  return L;
}

// ---------------------------------------------------------------- E1 / E2

// CDF 9/7 analysis (wavelets.py:44-65) of pairs [a, a + SEG) of a line of M
// pairs: d += A(s + s[i+1]); s += B(d[i-1] + d); d += G(s + s[i+1]);
// s += D(d[i-1] + d); s *= 1/K; d *= K, with s[M] = s[M-1] and d[-1] = d[0]
// (the reference's edge-clamped shifts).  Local pair j is global a - 2 + j.
template <class Load, class Store>
__device__ __forceinline__ void analyze_segment(int M, int a, Load load, Store store) {
  float s[LOC], d[LOC];
  const int lo = a - 2;
  const int jl = lo < 0 ? -lo : 0;                 // first valid local pair
  const int jh = M - lo < LOC ? M - lo : LOC;      // one past the last
#pragma unroll
  for (int j = 0; j < LOC; ++j) {
    s[j] = 0.0f;
    d[j] = 0.0f;
    if (j >= jl && j < jh) load(lo + j, s[j], d[j]);
  }
  // neighbours with the border clamp (interior segment edges produce values
  // that never reach the emitted pairs)
#pragma unroll
  for (int j = 0; j < LOC; ++j) {
    const float sn = (j + 1 < LOC && j + 1 < jh) ? s[j + 1 < LOC ? j + 1 : j] : s[j];
    d[j] = __fadd_rn(d[j], __fmul_rn(kA, __fadd_rn(s[j], sn)));
  }
#pragma unroll
  for (int j = LOC - 1; j >= 0; --j) {
    const float dp = (j >= 1 && j - 1 >= jl) ? d[j >= 1 ? j - 1 : 0] : d[j];
    s[j] = __fadd_rn(s[j], __fmul_rn(kB, __fadd_rn(dp, d[j])));
  }
#pragma unroll
  for (int j = 0; j < LOC; ++j) {
    const float sn = (j + 1 < LOC && j + 1 < jh) ? s[j + 1 < LOC ? j + 1 : j] : s[j];
    d[j] = __fadd_rn(d[j], __fmul_rn(kG, __fadd_rn(s[j], sn)));
  }
#pragma unroll
  for (int j = LOC - 1; j >= 0; --j) {
    const float dp = (j >= 1 && j - 1 >= jl) ? d[j >= 1 ? j - 1 : 0] : d[j];
    s[j] = __fadd_rn(s[j], __fmul_rn(kD, __fadd_rn(dp, d[j])));
  }
#pragma unroll
  for (int j = 2; j < SEG + 2; ++j)
    if (lo + j < M) store(lo + j, __fmul_rn(s[j], kIK), __fmul_rn(d[j], kK));
}

// Row pass of one level: every row of the h x w region of every plane.  A
// warp takes a chunk of RCH pairs of one row: it stages the chunk plus its
// 2-pair halos in shared memory with coalesced loads, each lane lifts one
// 16-pair segment from there, and the s / d halves go back through shared
// memory to coalesced stores.  Shared pair index p is padded to p + p / 16
// (conflict-free 8-byte accesses per half-warp).
constexpr int RCH = 32 * SEG;                       // pairs per warp chunk
constexpr int RSM = RCH + 4 + (RCH + 4) / 16 + 1;   // padded float2 slots
__device__ __forceinline__ int rpad(int p) { return p + (p >> 4); }

__global__ void __launch_bounds__(256) k_rows(const float* __restrict__ src, float* __restrict__ dst,
                                              int planes, int H, int W, int h, int w) {
  __shared__ float2 sm[8][RSM];
  const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
  float2* buf = sm[wp];
  float* outs = reinterpret_cast<float*>(buf);            // reused for the outputs
  const int M = w / 2, nch = (M + RCH - 1) / RCH;
  const size_t total = (size_t)planes * h * nch;
  for (size_t it = (size_t)blockIdx.x * 8 + wp; it < total; it += (size_t)gridDim.x * 8) {
    const int ch = (int)(it % nch);
    const size_t row = it / nch;
    const size_t pl = row / h, y = row - pl * h;
    const float2* in = reinterpret_cast<const float2*>(src + (pl * H + y) * W);
    float* out = dst + (pl * H + y) * W;
    const int c0 = ch * RCH;                 // first pair of the chunk
    // stage pairs [c0 - 2, c0 + RCH + 2) (in range only)
    for (int q = lane; q < RCH + 4; q += 32) {
      const int g = c0 - 2 + q;
      if (g >= 0 && g < M) buf[rpad(q)] = in[g];
    }
    __syncwarp();
    float sv[SEG], dv[SEG];
    const int a = c0 + lane * SEG;
    if (a < M) {
      analyze_segment(
          M, a,
          [&](int g, float& s, float& d) {
            const float2 v = buf[rpad(g - (c0 - 2))];
            s = v.x;
            d = v.y;
          },
          [&](int g, float s, float d) {
            sv[g - a] = s;
            dv[g - a] = d;
          });
    }
    __syncwarp();
    // outputs: s at pair slots [0, RCH), d at [RCH, 2 RCH) of the float view
    if (a < M) {
#pragma unroll
      for (int j = 0; j < SEG; ++j) {
        if (a + j < M) {
          outs[rpad(lane * SEG + j)] = sv[j];
          outs[RSM + rpad(lane * SEG + j)] = dv[j];
        }
      }
    }
    __syncwarp();
    const int cnt = min(RCH, M - c0);
    for (int q = lane; q < cnt; q += 32) {
      out[c0 + q] = outs[rpad(q)];
      out[M + c0 + q] = outs[RSM + rpad(q)];
    }
    __syncwarp();
  }
}

// Level-1 row pass fused with the u8 load (E1): a warp takes a chunk of one
// frame row, stages its bytes (all C channels interleaved, as stored) once,
// and lifts every channel from them; x / 255 comes from a 256-entry table of
// the IEEE quotients (chunk / 255, encoding.py:413).  4 warps per CTA.
constexpr int UCH = RCH;                               // pairs per warp chunk
__global__ void __launch_bounds__(128) k_rows_u8(const uint8_t* __restrict__ frames,
                                                 float* __restrict__ dst, int n, int C, int H,
                                                 int W) {
  __shared__ float s_q[256];
  __shared__ __align__(16) uint8_t sb[4][(UCH + 4) * 2 * 4 + 16];
  __shared__ float so[4][2 * RSM];
  for (int i = threadIdx.x; i < 256; i += 128) s_q[i] = __fdiv_rn((float)i, 255.0f);
  __syncthreads();
  const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
  uint8_t* bb = sb[wp];
  float* outs = so[wp];
  const int M = W / 2, nch = (M + UCH - 1) / UCH;
  const size_t plane = (size_t)H * W;
  const size_t total = (size_t)n * H * nch;
  for (size_t it = (size_t)blockIdx.x * 4 + wp; it < total; it += (size_t)gridDim.x * 4) {
    const int ch = (int)(it % nch);
    const size_t row = it / nch;               // t * H + y
    const size_t t = row / H, y = row - t * H;
    const int c0 = ch * UCH;
    const int g0 = c0 - 2 < 0 ? 0 : c0 - 2;                 // first staged pair
    const int g1 = c0 + UCH + 2 > M ? M : c0 + UCH + 2;     // one past the last
    const uint8_t* src = frames + ((t * H + y) * W + 2 * (size_t)g0) * C;
    const int nbytes = (g1 - g0) * 2 * C;
    // 4-byte words from the aligned-down start; byte b of the chunk is bb[mis + b]
    const int mis = (int)(reinterpret_cast<uintptr_t>(src) & 3u);
    const uint32_t* wsrc = reinterpret_cast<const uint32_t*>(src - mis);
    const int nw = (mis + nbytes + 3) >> 2;
    for (int q = lane; q < nw; q += 32) reinterpret_cast<uint32_t*>(bb)[q] = wsrc[q];
    __syncwarp();
    const int a = c0 + lane * SEG;
    for (int c = 0; c < C; ++c) {
      float sv[SEG], dv[SEG];
      if (a < M) {
        analyze_segment(
            M, a,
            [&](int g, float& sx, float& dx) {
              const int b = mis + (g - g0) * 2 * C + c;
              sx = s_q[bb[b]];
              dx = s_q[bb[b + C]];
            },
            [&](int g, float sx, float dx) {
              sv[g - a] = sx;
              dv[g - a] = dx;
            });
#pragma unroll
        for (int j = 0; j < SEG; ++j) {
          if (a + j < M) {
            outs[rpad(lane * SEG + j)] = sv[j];
            outs[RSM + rpad(lane * SEG + j)] = dv[j];
          }
        }
      }
      __syncwarp();
      float* out = dst + (t * C + c) * plane + y * W;
      const int cnt = min(UCH, M - c0);
      for (int q = lane; q < cnt; q += 32) {
        out[c0 + q] = outs[rpad(q)];
        out[M + c0 + q] = outs[RSM + rpad(q)];
      }
      __syncwarp();
    }
  }
}

// Column pass: thread = (column, segment of rows); adjacent threads take
// adjacent columns (coalesced).
__global__ void k_cols(const float* __restrict__ src, float* __restrict__ dst, int planes, int H,
                       int W, int h, int w) {
  const int M = h / 2, nseg = (M + SEG - 1) / SEG;
  const size_t total = (size_t)planes * nseg * w;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total;
       i += (size_t)gridDim.x * blockDim.x) {
    const int x = (int)(i % w);
    const size_t r = i / w;
    const int sg = (int)(r % nseg);
    const size_t pl = r / nseg;
    const float* in = src + pl * H * W + x;
    float* out = dst + pl * H * W + x;
    analyze_segment(
        M, sg * SEG,
        [&](int g, float& s, float& d) {
          s = in[(size_t)(2 * g) * W];
          d = in[(size_t)(2 * g + 1) * W];
        },
        [&](int g, float s, float d) {
          out[(size_t)g * W] = s;
          out[(size_t)(M + g) * W] = d;
        });
  }
}

// ---------------------------------------------------------------- E3

// Level of a Mallat position (0 = approximation) and the row inside its
// subband (wavelets.py:202-211, encoding.py:101-115).
__device__ __forceinline__ int position_level(int y, int x, int H, int W, int L, int& yy) {
  for (int k = 1; k <= L; ++k) {
    const int hh = H >> k, hw = W >> k;
    if (y < hh && x >= hw && x < 2 * hw) {
      yy = y;
      return k;
    }
    if (y >= hh && y < 2 * hh && x < 2 * hw) {
      yy = y - hh;
      return k;
    }
  }
  yy = 0;
  return 0;
}

// float -> unsigned key with the float order (for atomicMin / atomicMax)
__device__ __forceinline__ uint32_t fkey(float f) {
  const uint32_t b = __float_as_uint(f);
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ float unkey(uint32_t k) {
  return __uint_as_float((k & 0x80000000u) ? (k & 0x7FFFFFFFu) : ~k);
}

// keys: (n, C, 4) = approx min, approx max, detail min, detail max
__global__ void k_ext_init(uint32_t* keys, int count) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < count) keys[i] = (i & 1) ? 0u : 0xFFFFFFFFu;
}

__global__ void k_ext_final(const uint32_t* keys, float* ext, int count) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < count) ext[i] = unkey(keys[i]);
}

// E3-E5, one CTA per 32x32 (bs x bs) block at a time (grid-stride), 256
// threads, position o = r * 256 + tid of the block.  Per position: sparsify
// each frame (encoding.py:118-135: keep iff the channel max magnitude
// exceeds level threshold + H(y); the approximation is kept), temporal Haar
// forward in Mallat order (:153-169: a = (x0 + x1) * 0.5, d = (x0 - x1) *
// 0.5, the finest temporal level's details last), then zero temporal
// details whose channel max magnitude is <= their threshold (:198-236; the
// approximation band is exempt).  The final values go back to the planes;
// their nonzero flags (any channel != 0, encoding.py:306) become one bit per
// (t, position) and the (t, block) record counts (warp atomics: the warps
// of a CTA never wait for each other); the per-(t, c) extrema
// (:239-254) are reduced on the way (detail in registers, the rare
// approximation positions through shared-memory atomics).
// NT = n, CT = C at compile time (register arrays), or 0 = run time
template <int NT, int CT>
__global__ void __launch_bounds__(256) k_point(float* __restrict__ planes,
                                               const float* __restrict__ row_factor,
                                               uint32_t* __restrict__ nzbits,
                                               uint32_t* __restrict__ counts,
                                               uint32_t* __restrict__ keys, wv_encode_params p) {
  constexpr int NA = NT ? NT : WV_ENC_MAX_N;
  constexpr int CA = CT ? CT : 4;
  const int H = p.height, W = p.width, C = CT ? CT : p.channels, n = NT ? NT : p.inter_size;
  const int L = p.levels;
  const int bs = p.block_size, nbx = W / bs, NB = nbx * (H / bs);
  const int npos = bs * bs, nwords = (npos + 31) / 32;
  const size_t plane = (size_t)H * W;
  const int tid = threadIdx.x, lane = tid & 31, wp = tid >> 5;
  __shared__ uint32_t s_keys[WV_ENC_MAX_N * 4 * 4];
  for (int k = tid; k < n * C * 4; k += 256) s_keys[k] = (k & 1) ? 0u : 0xFFFFFFFFu;
  float dmin[NA][CA], dmax[NA][CA];
#pragma unroll
  for (int t = 0; t < NA; ++t)
#pragma unroll
    for (int c = 0; c < CA; ++c) {
      dmin[t][c] = INFINITY;
      dmax[t][c] = -INFINITY;
    }
  __syncthreads();
  for (int b = blockIdx.x; b < NB; b += gridDim.x) {
    const int by = b / nbx, bx = b - by * nbx;
    uint32_t cnt[NA];
#pragma unroll
    for (int t = 0; t < NA; ++t) cnt[t] = 0;
    for (int o0 = 0; o0 < npos; o0 += 256) {
      const int o = o0 + tid;
      const bool live = o < npos;
      const int y = by * bs + (live ? o / bs : 0), x = bx * bs + (live ? o % bs : 0);
      const size_t i = (size_t)y * W + x;
      int yy;
      const int k = position_level(y, x, H, W, L, yy);
      float v[NA][CA];
#pragma unroll
      for (int t = 0; t < NA; ++t) {
        if (t >= n) break;
        float m = 0.0f;
#pragma unroll
        for (int c = 0; c < CA; ++c) {
          v[t][c] = 0.0f;
          if (c < C && live) {
            v[t][c] = planes[(size_t)(t * C + c) * plane + i];
            m = fmaxf(m, fabsf(v[t][c]));
          }
        }
        if (k > 0) {
          const int ry = min(yy << k, H - 1);
          const float thr = __fadd_rn(p.level_threshold[k - 1], row_factor[ry]);
          if (!(m > thr)) {
#pragma unroll
            for (int c = 0; c < CA; ++c) v[t][c] = 0.0f;
          }
        }
      }
      float out[NA][CA];
      int end = n;
#pragma unroll
      for (int cur = NA; cur > 1; cur >>= 1) {
        if (cur > n) continue;
        const int half = cur >> 1;
#pragma unroll
        for (int q = 0; q < NA / 2; ++q) {
          if (q >= half) break;
#pragma unroll
          for (int c = 0; c < CA; ++c) {
            const float a0 = v[2 * q][c], a1 = v[2 * q + 1][c];
            out[end - half + q][c] = __fmul_rn(__fsub_rn(a0, a1), 0.5f);
            v[q][c] = __fmul_rn(__fadd_rn(a0, a1), 0.5f);
          }
        }
        end -= half;
      }
#pragma unroll
      for (int c = 0; c < CA; ++c) out[0][c] = v[0][c];
      const bool approx = k == 0;
#pragma unroll
      for (int t = 0; t < NA; ++t) {
        if (t >= n) break;
        bool kill = false;
        if (t >= 1 && !approx) {
          float m = 0.0f;
#pragma unroll
          for (int c = 0; c < CA; ++c)
            if (c < C) m = fmaxf(m, fabsf(out[t][c]));
          kill = m <= p.temporal_threshold[t];
        }
        bool nz = false;
#pragma unroll
        for (int c = 0; c < CA; ++c)
          if (c < C && live) nz |= !kill && out[t][c] != 0.0f;
#pragma unroll
        for (int c = 0; c < CA; ++c) {
          if (c < C && live) {
            const float r = kill ? 0.0f : out[t][c];
            // only positions with a record are read again (k_emit, via nzbits)
            if (nz) planes[(size_t)(t * C + c) * plane + i] = r;
            if (approx) {
              atomicMin(&s_keys[(t * C + c) * 4 + 0], fkey(r));
              atomicMax(&s_keys[(t * C + c) * 4 + 1], fkey(r));
            } else {
              dmin[t][c] = fminf(dmin[t][c], r);
              dmax[t][c] = fmaxf(dmax[t][c], r);
            }
          }
        }
        const uint32_t bits = __ballot_sync(0xFFFFFFFFu, nz);
        if (lane == 0 && (o0 >> 5) + wp < nwords) {
          // positions o0 + 32 wp .. +31 of the block (masked to the block for bs < 8)
          const uint32_t mk = npos - (o0 + 32 * wp) >= 32 ? 0xFFFFFFFFu
                                                           : ((1u << (npos - (o0 + 32 * wp))) - 1u);
          nzbits[((size_t)t * NB + b) * nwords + (o0 >> 5) + wp] = bits & mk;
          cnt[t] += __popc(bits & mk);
        }
      }
    }
    if (lane == 0) {
#pragma unroll
      for (int t = 0; t < NA; ++t)
        if (t < n && cnt[t]) atomicAdd(&counts[(size_t)t * NB + b], cnt[t]);
    }
  }
  // detail extrema: warp reduce, shared atomics, then one global atomic per key
#pragma unroll
  for (int t = 0; t < NA; ++t) {
    if (t >= n) break;
#pragma unroll
    for (int c = 0; c < CA; ++c) {
      if (c >= C) break;
      float mn = dmin[t][c], mx = dmax[t][c];
      for (int o = 16; o; o >>= 1) {
        mn = fminf(mn, __shfl_xor_sync(0xFFFFFFFFu, mn, o));
        mx = fmaxf(mx, __shfl_xor_sync(0xFFFFFFFFu, mx, o));
      }
      if (lane == 0 && mn <= mx) {
        atomicMin(&s_keys[(t * C + c) * 4 + 2], fkey(mn));
        atomicMax(&s_keys[(t * C + c) * 4 + 3], fkey(mx));
      }
    }
  }
  __syncthreads();
  for (int k = tid; k < n * C * 4; k += 256) {
    const uint32_t v = s_keys[k];
    if (k & 1) {
      if (v != 0u) atomicMax(&keys[k], v);
    } else if (v != 0xFFFFFFFFu) {
      atomicMin(&keys[k], v);
    }
  }
}

// ---------------------------------------------------------------- E4 / E5

// Storage layer of a position (wavelets.py:202-211): 0 approx, L - k + 1 for
// level-k detail.
__device__ __forceinline__ int position_layer(int y, int x, int H, int W, int L) {
  int yy;
  const int k = position_level(y, x, H, W, L, yy);
  return k == 0 ? 0 : L - k + 1;
}

// Exclusive scan of the (n * NB) counts in 1024-element tiles: tile sums,
// a serial scan of the (few hundred) tile sums, then the in-tile scan.
__global__ void k_scan_tiles(const uint32_t* counts, uint64_t* partials, int total) {
  __shared__ uint64_t ws[32];
  const int i = blockIdx.x * 1024 + threadIdx.x;
  uint64_t v = 0;
  for (int k = 0; k < 4; ++k) {
    const int j = i + k * 256;
    if (j < total) v += counts[j];
  }
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint64_t s = 0;
    for (int w = 0; w < 8; ++w) s += ws[w];
    partials[blockIdx.x] = s;
  }
}

__global__ void k_scan_partials(uint64_t* partials, int ntiles, uint64_t* d_num_records) {
  if (threadIdx.x != 0) return;
  uint64_t s = 0;
  for (int i = 0; i < ntiles; ++i) {
    const uint64_t v = partials[i];
    partials[i] = s;
    s += v;
  }
  *d_num_records = s;
}

__global__ void k_scan_apply(const uint32_t* counts, const uint64_t* partials, uint64_t* starts,
                             int total) {
  // 256 threads x 4 consecutive elements
  __shared__ uint64_t ws[8];
  const int base = blockIdx.x * 1024 + threadIdx.x * 4;
  uint32_t c[4];
  uint64_t loc = 0;
  for (int k = 0; k < 4; ++k) {
    c[k] = base + k < total ? counts[base + k] : 0u;
    loc += c[k];
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint64_t inc = loc;
  for (int o = 1; o < 32; o <<= 1) {
    const uint64_t u = __shfl_up_sync(0xFFFFFFFFu, inc, o);
    if (lane >= o) inc += u;
  }
  if (lane == 31) ws[warp] = inc;
  __syncthreads();
  uint64_t wbase = 0;
  for (int w = 0; w < warp; ++w) wbase += ws[w];
  uint64_t run = partials[blockIdx.x] + wbase + inc - loc;
  for (int k = 0; k < 4; ++k) {
    if (base + k < total) starts[base + k] = run;
    run += c[k];
  }
}

// Records of one (t, block) in (layer, offset) order (encoding.py:296-332):
// u16 offset, then C quantised bytes (cmin/cmax of the position's band:
// floor((v - lo) / span * 255 + 0.5), 0 when span == 0) or C float32.
__global__ void k_emit(const float* __restrict__ planes, const float* __restrict__ ext,
                       const uint64_t* __restrict__ starts, const uint32_t* __restrict__ nzbits,
                       uint8_t* __restrict__ payload, wv_encode_params p) {
  const int bs = p.block_size, nbx = nb_x(p), NB = nb_all(p);
  const int H = p.height, W = p.width, C = p.channels, L = p.levels;
  const int t = blockIdx.x / NB, b = blockIdx.x - t * NB;
  const int by = b / nbx, bx = b - by * nbx;
  const size_t plane = (size_t)H * W;
  const int npos = bs * bs;
  const int rs = p.quantize ? 2 + C : 2 + 4 * C;
  __shared__ int s_layer_count[WV_MAX_LEVELS + 1];
  __shared__ int s_warp[8];
  if (starts[blockIdx.x + 1 < (unsigned)(p.inter_size * NB) ? blockIdx.x + 1 : blockIdx.x] ==
          starts[blockIdx.x] &&
      blockIdx.x + 1 < (unsigned)(p.inter_size * NB))
    return;   // no records in this (t, block)
  if (threadIdx.x <= WV_MAX_LEVELS) s_layer_count[threadIdx.x] = 0;
  __syncthreads();
  // 4 consecutive offsets per thread (npos <= 1024)
  int lay[4];
  bool nz[4];
  for (int k = 0; k < 4; ++k) {
    const int o = threadIdx.x * 4 + k;
    nz[k] = false;
    lay[k] = 0;
    if (o < npos) {
      nz[k] = (nzbits[(size_t)blockIdx.x * ((npos + 31) / 32) + (o >> 5)] >> (o & 31)) & 1u;
      if (nz[k]) {
        const int y = by * bs + o / bs, x = bx * bs + o % bs;
        lay[k] = position_layer(y, x, H, W, L);
        atomicAdd(&s_layer_count[lay[k]], 1);
      }
    }
  }
  __syncthreads();
  uint64_t rec_base = starts[blockIdx.x];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int l = 0; l <= L; ++l) {
    if (s_layer_count[l] == 0) continue;   // CTA-uniform
    // exclusive rank among this layer's nonzero positions in offset order
    int mine = 0;
    for (int k = 0; k < 4; ++k) mine += nz[k] && lay[k] == l;
    int inc = mine;
    for (int o = 1; o < 32; o <<= 1) {
      const int u = __shfl_up_sync(0xFFFFFFFFu, inc, o);
      if (lane >= o) inc += u;
    }
    if (lane == 31) s_warp[warp] = inc;
    __syncthreads();
    int r = inc - mine;
    for (int w = 0; w < warp; ++w) r += s_warp[w];
    for (int k = 0; k < 4; ++k) {
      if (!(nz[k] && lay[k] == l)) continue;
      const int o = threadIdx.x * 4 + k;
      const int y = by * bs + o / bs, x = bx * bs + o % bs;
      const size_t pix = (size_t)y * W + x;
      uint8_t* dst = payload + (rec_base + r) * rs;
      dst[0] = (uint8_t)(o & 0xFF);
      dst[1] = (uint8_t)(o >> 8);
      const bool in_appr = lay[k] == 0;
      for (int c = 0; c < C; ++c) {
        const float v = planes[(size_t)(t * C + c) * plane + pix];
        if (!p.quantize) {
          const uint32_t u = __float_as_uint(v);
          dst[2 + 4 * c] = (uint8_t)u;
          dst[3 + 4 * c] = (uint8_t)(u >> 8);
          dst[4 + 4 * c] = (uint8_t)(u >> 16);
          dst[5 + 4 * c] = (uint8_t)(u >> 24);
        } else {
          const float* e = ext + (size_t)(t * C + c) * 4;
          const float lo = in_appr ? e[0] : e[2], hi = in_appr ? e[1] : e[3];
          const float span = __fsub_rn(hi, lo);
          float q = 0.0f;
          if (span > 0.0f)
            q = floorf(__fadd_rn(__fmul_rn(__fdiv_rn(__fsub_rn(v, lo), span), 255.0f), 0.5f));
          dst[2 + c] = (uint8_t)fminf(fmaxf(q, 0.0f), 255.0f);
        }
      }
      ++r;
    }
    rec_base += s_layer_count[l];
    __syncthreads();   // s_warp reuse
  }
}

int check_params(const wv_encode_params* p) {
  if (!p) return WV_ERR_ARG;
  const int n = p->inter_size, bs = p->block_size;
  if (p->width < 1 || p->height < 1 || p->channels < 1 || p->channels > 4) return WV_ERR_ARG;
  if (p->levels < 1 || p->levels > WV_MAX_LEVELS) return WV_ERR_ARG;
  if (n < 1 || n > WV_ENC_MAX_N || (n & (n - 1))) return WV_ERR_ARG;
  if (bs < 1 || bs > 32 || (bs & (bs - 1))) return WV_ERR_ARG;
  if (p->width % (1 << p->levels) || p->height % (1 << p->levels)) return WV_ERR_ARG;
  if (p->width % bs || p->height % bs) return WV_ERR_ARG;
  if (bs * bs > 65536) return WV_ERR_ARG;
  return WV_OK;
}

int grid_for(size_t work, int threads) {
  const size_t b = (work + threads - 1) / threads;
  return (int)(b < 148 * 16 ? (b ? b : 1) : 148 * 16);
}

}  // namespace
}  // namespace wv

using namespace wv;

extern "C" int wv_encode_workspace_bytes(const wv_encode_params* p, uint64_t* bytes) {
  if (check_params(p) != WV_OK || !bytes) return WV_ERR_ARG;
  *bytes = enc_layout(*p).total;
  return WV_OK;
}

extern "C" int wv_encode_payload_capacity(const wv_encode_params* p, uint64_t* bytes) {
  if (check_params(p) != WV_OK || !bytes) return WV_ERR_ARG;
  const uint64_t rs = p->quantize ? 2 + p->channels : 2 + 4 * p->channels;
  *bytes = (uint64_t)p->inter_size * p->width * p->height * rs;
  return WV_OK;
}

extern "C" int wv_encode_set(const wv_encode_params* p, const uint8_t* d_frames,
                             const float* d_row_factor, void* d_workspace,
                             uint64_t workspace_bytes, float* d_extrema, uint32_t* d_counts,
                             uint8_t* d_payload, uint64_t payload_capacity,
                             uint64_t* d_num_records, void* stream) {
  if (check_params(p) != WV_OK) return WV_ERR_ARG;
  if (!d_frames || !d_row_factor || !d_workspace || !d_extrema || !d_counts || !d_payload ||
      !d_num_records)
    return WV_ERR_ARG;
  const EncLayout lo = enc_layout(*p);
  uint64_t cap = 0;
  wv_encode_payload_capacity(p, &cap);
  if (workspace_bytes < lo.total || payload_capacity < cap) return WV_ERR_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  uint8_t* ws = (uint8_t*)d_workspace;
  float* planes = (float*)(ws + lo.planes);
  float* tmp = (float*)(ws + lo.tmp);
  uint64_t* starts = (uint64_t*)(ws + lo.starts);
  uint32_t* keys = (uint32_t*)(ws + lo.ext_bits);
  uint64_t* partials = (uint64_t*)(ws + lo.partials);
  uint32_t* nzbits = (uint32_t*)(ws + lo.nzbits);
  const int H = p->height, W = p->width, C = p->channels, n = p->inter_size;
  const int planes_n = n * C;
  constexpr int T = 256;

  int h = H, w = W;
  for (int k = 0; k < p->levels; ++k) {
    if (k == 0) {
      const size_t work = (size_t)n * H * ((W / 2 + UCH - 1) / UCH);   // warps
      k_rows_u8<<<grid_for(work * 32, 128), 128, 0, s>>>(d_frames, tmp, n, C, H, W);
    } else {
      const size_t rows_work = (size_t)planes_n * h * ((w / 2 + RCH - 1) / RCH);   // warps
      k_rows<<<grid_for(rows_work * 32, T), T, 0, s>>>(planes, tmp, planes_n, H, W, h, w);
    }
    const size_t cols_work = (size_t)planes_n * ((h / 2 + SEG - 1) / SEG) * w;
    k_cols<<<grid_for(cols_work, T), T, 0, s>>>(tmp, planes, planes_n, H, W, h, w);
    h /= 2;
    w /= 2;
  }
  const int nkeys = planes_n * 4;
  const int nblk = n * nb_all(*p);
  k_ext_init<<<(nkeys + T - 1) / T, T, 0, s>>>(keys, nkeys);
  WV_CUDA(cudaMemsetAsync(d_counts, 0, (size_t)nblk * 4, s));
  {
    const int g = nb_all(*p) < 148 * 8 ? nb_all(*p) : 148 * 8;
#define WV_POINT(NTV, CTV) \
  k_point<NTV, CTV><<<g, T, 0, s>>>(planes, d_row_factor, nzbits, d_counts, keys, *p)
    if (n == 4 && C == 3) WV_POINT(4, 3);
    else if (n == 4 && C == 1) WV_POINT(4, 1);
    else if (n == 1) WV_POINT(1, 0);
    else if (n == 2) WV_POINT(2, 0);
    else if (n == 4) WV_POINT(4, 0);
    else if (n == 8) WV_POINT(8, 0);
    else WV_POINT(0, 0);
#undef WV_POINT
  }
  k_ext_final<<<(nkeys + T - 1) / T, T, 0, s>>>(keys, d_extrema, nkeys);
  const int ntiles = (nblk + 1023) / 1024;
  k_scan_tiles<<<ntiles, 256, 0, s>>>(d_counts, partials, nblk);
  k_scan_partials<<<1, 32, 0, s>>>(partials, ntiles, d_num_records);
  k_scan_apply<<<ntiles, 256, 0, s>>>(d_counts, partials, starts, nblk);
  k_emit<<<nblk, T, 0, s>>>(planes, d_extrema, starts, nzbits, d_payload, *p);
  WV_CUDA(cudaGetLastError());
  return WV_OK;
}
