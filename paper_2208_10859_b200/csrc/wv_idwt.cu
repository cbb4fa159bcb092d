// K3 — per-level inverse 2-D CDF 9/7 synthesis, TMA-fed, column+row lifting
// fused in shared memory; the finest level fuses the u8 colour conversion
// and request masking (K4 colour step).
//
// Reference: synthesize_2d_region (wavelets.py:355-444) -> synthesize_1d
// (wavelets.py:68-91) per level, columns (y) first then rows (x), and
// decoding.py:301 for clip(rint(x*255)).  Inside the requested area the
// reference's windowed result equals a full-frame synthesis of the masked
// pyramid (verified by tests/test_oracle_golden.py), so each 32x32 coefficient
// tile is computed independently from a 2-coefficient halo: outputs equal the
// full-frame values bit for bit.  Boundary symmetric extension is applied at
// every lifting step at the true level borders only (index clamp, as numpy's
// _shift_left/_shift_right do).
//
// Per (tile, channel) item (TY = 32 rows x TX = 28 columns of each subband ->
// 64 x 56 outputs), 4 warps, one per 8-row-pair segment: one elected thread
// issues four TMA box loads (LL, HL, LH, HH; 36 x 36 f32 each, far-edge
// out-of-range zero-filled) completing on an mbarrier.  Lane l of a warp owns
// coefficient column ax - 2 + l: the 28 output columns plus 2 halo columns on
// each side, so a warp's 32 lanes hold everything its row lifting needs.  The
// column pass streams the lane's column down the segment (the L-half LL/LH and
// H-half HL/HH lines packed as float2, Blackwell's paired FP32 ops
// __fadd2_rn and products as __ffma2_rn(a, b, -0.0), each rounded like numpy) and keeps the 8 emitted row pairs in
// registers; the row pass then lifts each row pair (two rows packed) across
// the lanes, neighbour values exchanged by warp shuffles -- no shared column
// buffer and one barrier per item (the boxes are free once every warp's
// column pass is done, and the next item's TMA loads go out then).  Mid
// levels store f32 pairs per lane, the finest level converts to u8 in
// registers and stores 2-pixel pairs request-masked straight to the canvas.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstdlib>

#include "wv_common.cuh"

namespace wv {
namespace {

constexpr int BOX_FLOATS = BOX_W * BOX_H;
constexpr int BOX_SLOT = ((BOX_FLOATS * 4 + 127) / 128) * 128;  // bytes
#ifndef WV_K3_CVT_U8
#define WV_K3_CVT_U8 1
#endif
#ifndef WV_K3_UNMASKED
#define WV_K3_UNMASKED 1   // fully requested tiles skip the per-pixel masking
#endif
#ifndef WV_K3_MINB
#define WV_K3_MINB 8   // 64 registers: 8 CTAs (32 warps) per SM, the shared-memory limit too
#endif
#if WV_K3_MINB > 0 && WV_K3_STRIPS > 1
#define K3_BOUNDS __launch_bounds__(NTHREADS, WV_K3_MINB / WV_K3_STRIPS)
#elif WV_K3_MINB > 0
#define K3_BOUNDS __launch_bounds__(NTHREADS, WV_K3_MINB)
#else
#define K3_BOUNDS __launch_bounds__(NTHREADS)
#endif
#ifndef WV_K3_MID_PREFETCH
#define WV_K3_MID_PREFETCH 1   // mid levels also load the next item during the row pass
#endif
constexpr int SEG = 8;                 // output row pairs per warp (column-pass segment)
#ifndef WV_K3_RP
#define WV_K3_RP 2   // row pairs lifted together in the row pass (shuffle latency overlap)
#endif
constexpr int RP = WV_K3_RP;
static_assert(SEG % RP == 0, "row-pass groups tile the segment");
constexpr int NSTRIP = WV_K3_STRIPS;
constexpr int NWARP = TY / SEG * NSTRIP;   // 4 per strip
constexpr int NTHREADS = 32 * NWARP;       // 128 per strip
static_assert(TXS + 2 * HALO == 32, "a warp's lanes are its strip's columns plus the halo");
static_assert(BOX_W >= TX + 2 * XPAD, "the box covers the halo columns");

__device__ __forceinline__ float2 f2(float v) { return make_float2(v, v); }
// clip(rint(x), 0, 255) (decoding.py:301; rint is round-half-even): one
// saturating convert (F2IP.U8) instead of F2I + min
__device__ __forceinline__ uint32_t u8_rint(float x) {
#if WV_K3_CVT_U8
  uint32_t u;
  asm("cvt.rni.sat.u8.f32 %0, %1;" : "=r"(u) : "f"(x));
  return u;   // zero-extended to 32 bits
#else
  return min(__float2uint_rn(x), 255u);
#endif
}
// RN products as fma.rn.f32x2(a, b, z) with z = -0.0 supplied at run time
// (a kernel argument): a*b + (-0) rounds exactly like mul.rn (a -0 addend
// changes no product, +0 included), and an FMA result is never contracted
// into a following add -- ptxas (CUDA 12.9) contracts a paired mul.rn.f32x2
// feeding add.rn.f32x2 into FFMA2 despite the .rn, and it folds a literal
// -0 addend back into a multiply.  So every lifting step is three paired
// instructions: add, "multiply", add, each rounded once like numpy's.
__device__ __forceinline__ float2 pmul(float2 a, float2 b, float2 z) { return __ffma2_rn(a, b, z); }
// x - k*(y1 + y2), written as x + (-k)*(y1+y2): identical rounding.
__device__ __forceinline__ float2 lstep(float2 x, float2 nk, float2 y1, float2 y2, float2 z) {
  return __fadd2_rn(x, pmul(nk, __fadd2_rn(y1, y2), z));
}

// Interior segment (no level border inside [g0, g0 + LEN + 4)): the same
// stream with a compile-time trip count, fully unrolled -- no loop counter,
// no emission tests, constant shared-memory offsets.  Local indices: inputs
// 0 .. LEN+3, emitted pairs 2 .. LEN+1.
template <int LEN, class Load, class Emit>
__device__ __forceinline__ void lift_interior(float2 z, Load load, Emit emit) {
  const float2 KS = f2(__uint_as_float(0x3f9d7658u));
  const float2 IK = f2(__uint_as_float(0x3f5019c3u));
  const float2 ND = f2(-__uint_as_float(0x3ee31355u));
  const float2 NG = f2(-__uint_as_float(0x3f620676u));
  const float2 NB = f2(-__uint_as_float(0xbd5901aeu));
  const float2 NA = f2(-__uint_as_float(0xbfcb0673u));
  float2 sr, dr;
  load(0, sr, dr);
  float2 d1m = pmul(dr, IK, z);
  float2 s2m = pmul(sr, KS, z);         // s2[0] is a halo value: never emitted
  load(1, sr, dr);
  float2 d1 = pmul(dr, IK, z);
  float2 s2 = lstep(pmul(sr, KS, z), ND, d1m, d1, z);
  float2 d2mm = lstep(d1m, NG, s2m, s2, z);   // d2[0] (halo)
  float2 s3mm = s2;                        // s3[0] (halo)
  d1m = d1;
  s2m = s2;
#pragma unroll
  for (int j = 2; j < LEN + 4; ++j) {
    load(j, sr, dr);
    d1 = pmul(dr, IK, z);
    s2 = lstep(pmul(sr, KS, z), ND, d1m, d1, z);   // s2[j]
    const float2 d2 = lstep(d1m, NG, s2m, s2, z);     // d2[j-1]
    const float2 s3 = lstep(s2m, NB, d2mm, d2, z);    // s3[j-1]
    if (j >= 4) emit(j - 2, s3mm, lstep(d2mm, NA, s3mm, s3, z));   // d3[j-2]
    d2mm = d2;
    s3mm = s3;
    d1m = d1;
    s2m = s2;
  }
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(phase)
        : "memory");
  }
}

__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int x, int y, int z,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
      : "memory");
}

// n / d by multiply-high with m = ceil(2^32 / d) (exact for n * d < 2^32,
// far above any item or tile index here); d = 1 is the identity.
struct FastDiv {
  uint32_t d, m;
};
__host__ __device__ inline FastDiv fast_div(uint32_t d) {
  return FastDiv{d, d > 1 ? (uint32_t)((0x100000000ull + d - 1) / d) : 0u};
}
__device__ __forceinline__ uint32_t operator/(uint32_t n, FastDiv f) {
  return f.d > 1 ? __umulhi(n, f.m) : n;
}

struct LevelArgs {
  int k, bh, bw, C, ntx;
  FastDiv divC, divN;  // by C and by ntx
  const uint32_t* list;
  const uint32_t* count;
  float* out;          // non-final: Y_{k-1} planar C x 2bh x out_pitch
  int out_pitch;       // floats
  const wv_frame_args* fa;   // final: fa->d_canvas, planar C x H x W u8
  const uint32_t* R;   // final: requested-mask rows (mh x wpr0)
  const uint32_t* rowmap;  // final: pixel row -> mask row
  int wpr0;
  int use_tma;         // subband width is a multiple of 4 floats (TMA inner coordinate
                       // alignment); else the boxes are filled with plain loads
  const float* ll_ptr; int ll_pitch, ll_rows;   // LDG fallback sources
  const float* plane; int plane_w, plane_h;
  float neg_zero;      // -0.0f (see pmul)
};

// Items are (tile, channel), 4 warps per item, warp w = output row pairs
// [8w, 8w+8) of the tile.  The finest level stages the tile's request-mask
// words (two dependent loads per row) while the boxes load and ANDs them
// over the tile: a fully requested tile stores unmasked.  Once every warp's
// column pass is done (the one barrier per item) the boxes are dead and the
// next item's four loads go out, overlapping this item's row pass.  21 KB
// of boxes + 2 KB of request staging and 64 registers: 8 CTAs per SM.
constexpr int BOXSET = 4 * BOX_SLOT;
constexpr int RQ_USED = (30 + 2 * TX + 31) / 32;   // request words a tile row can touch
constexpr int RQ_WORDS = RQ_USED <= 4 ? 4 : 8;      // staged per row (16-B stores)
constexpr int RQ_SLOT = OUT_H * RQ_WORDS;       // u32 per staging slot
constexpr int SMEM_MID = BOXSET;
constexpr int SMEM_FIN = BOXSET + 2 * RQ_SLOT * 4;

template <bool FINAL>
__global__ void K3_BOUNDS k_level(const __grid_constant__ CUtensorMap tm_ll,
                                                    const __grid_constant__ CUtensorMap tm_det,
                                                    LevelArgs a) {
  pdl_sync();
  extern __shared__ __align__(128) uint8_t smem[];
  uint8_t* canvas = FINAL ? a.fa->d_canvas : nullptr;
  float* box = reinterpret_cast<float*>(smem);
  const float* bLL = box;
  const float* bHL = box + BOX_SLOT / 4;
  const float* bLH = box + 2 * BOX_SLOT / 4;
  const float* bHH = box + 3 * BOX_SLOT / 4;
  uint32_t* rq_stage = reinterpret_cast<uint32_t*>(smem + BOXSET);   // final: 2 slots
  __shared__ uint64_t bar;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) mbar_init(&bar, 1);
  __syncthreads();
  uint32_t phase = 0u;
  const int C = a.C;
  const uint32_t nitems = *a.count * (uint32_t)C;
  const int H = 2 * a.bh, W = 2 * a.bw;
  const float2 KS = f2(__uint_as_float(0x3f9d7658u));    // K
  const float2 IK = f2(__uint_as_float(0x3f5019c3u));    // 1/K
  const float2 ND = f2(-__uint_as_float(0x3ee31355u));   // -delta
  const float2 NG = f2(-__uint_as_float(0x3f620676u));   // -gamma
  const float2 NB = f2(-__uint_as_float(0xbd5901aeu));   // -beta
  const float2 NA = f2(-__uint_as_float(0xbfcb0673u));   // -alpha
  const float2 z = f2(a.neg_zero);                       // -0.0, opaque to ptxas

  // issue the four box loads of an item (elected thread)
  auto issue = [&](uint32_t it) {
    if (tid != 0) return;
    const uint32_t itile = it / a.divC;
    const uint32_t tile = a.list[itile] & ~ZERO_FLAG;
    const int ty = (int)(tile / a.divN), tx = (int)tile - ty * a.ntx;
    // TMA faults on unaligned/negative innermost box coordinates (observed on
    // B200, driver 580): x starts at ax-4 (ax = 28 tx: 16-byte aligned) clamped to 0
    const int oy = max(ty * TY - HALO, 0), ox = max(tx * TX - XPAD, 0);
    const int c = (int)(it - itile * C);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    mbar_expect_tx(&bar, 4u * BOX_FLOATS * 4u);
    tma_load_3d(box, &tm_ll, ox, oy, c, &bar);
    tma_load_3d(box + BOX_SLOT / 4, &tm_det, a.bw + ox, oy, c, &bar);
    tma_load_3d(box + 2 * BOX_SLOT / 4, &tm_det, ox, a.bh + oy, c, &bar);
    tma_load_3d(box + 3 * BOX_SLOT / 4, &tm_det, a.bw + ox, a.bh + oy, c, &bar);
  };

  bool issued = false;   // the current item's boxes are already in flight
  int slot = 0;          // final: request-staging slot of this item
  for (uint32_t item = blockIdx.x; item < nitems; item += gridDim.x) {
    const uint32_t itile = item / a.divC;
    const uint32_t entry = a.list[itile];
    const int c = (int)(item - itile * C);
    const uint32_t tile = entry & ~ZERO_FLAG;
    const int ty = (int)(tile / a.divN), tx = (int)tile - ty * a.ntx;
    const int ay = ty * TY, ax = tx * TX;
    const int by = min(ay + TY, a.bh), bx = min(ax + TX, a.bw);
    const int ny = 2 * (by - ay), nx = 2 * (bx - ax);
    if (FINAL && (entry & ZERO_FLAG)) {
      // tile left the request: clear what an earlier frame wrote there
      const int qw = nx >> 1;   // u16 pairs per row (56-px tiles start 8-byte aligned)
      for (int idx = tid; idx < ny * qw; idx += NTHREADS) {
        const int r = idx / qw, q = idx - (idx / qw) * qw;
        *reinterpret_cast<uint16_t*>(canvas + ((uint64_t)c * H + 2 * ay + r) * W + 2 * ax + 2 * q) = 0;
      }
      continue;
    }
    const int oy = max(ay - HALO, 0), ox = max(ax - XPAD, 0);
    const uint32_t nxt = item + gridDim.x;
    uint32_t nxt_entry = ZERO_FLAG;
    if ((FINAL || WV_K3_MID_PREFETCH) && tid == 0 && a.use_tma && nxt < nitems) nxt_entry = a.list[nxt / a.divC];
    // the boxes go out before the request words are staged (the elected
    // thread would otherwise wait for its staging loads first)
    if (FINAL && a.use_tma && !issued) issue(item);
    uint32_t* rq = rq_stage + slot * RQ_SLOT;
    const int w0 = (2 * ax) >> 5;   // first request word of the tile's pixel columns
    bool rq_all = true;             // final: the whole tile is requested (no masking)
    if (FINAL) {
      // the tile's request-mask words, one output row per thread (row map ->
      // mask row, then the row's 3 words), staged while the boxes load; a
      // 56-px tile starting at bit 2ax & 31 spans at most 3 words
      if (tid < ny) {
        const uint32_t* Rrow = a.R + (uint64_t)a.rowmap[2 * ay + tid] * a.wpr0;
        uint32_t v[RQ_WORDS];
#pragma unroll
        for (int k = 0; k < RQ_WORDS; ++k) {
          const int w = w0 + k;
          v[k] = (k < RQ_USED && w < a.wpr0) ? Rrow[w] : 0u;
          // the tile's pixel columns [2ax, 2ax + nx) inside this word
          const int lo = max(2 * ax - 32 * w, 0), hi = min(2 * ax + nx - 32 * w, 32);
          const uint32_t need =
              lo >= hi ? 0u : ((hi >= 32 ? 0xFFFFFFFFu : ((1u << hi) - 1u)) & (0xFFFFFFFFu << lo));
          rq_all &= (v[k] & need) == need;
        }
#pragma unroll
        for (int k = 0; k < RQ_WORDS; k += 4)
          *reinterpret_cast<uint4*>(rq + tid * RQ_WORDS + k) =
              make_uint4(v[k], v[k + 1], v[k + 2], v[k + 3]);
      }
    }
    if (a.use_tma) {
      if (!FINAL && !issued) issue(item);
      mbar_wait(&bar, phase);
      phase ^= 1u;
    } else {
      // tiny levels whose subband width is not a multiple of 4 floats
      for (int i = tid; i < 4 * BOX_FLOATS; i += NTHREADS) {
        const int q = i / BOX_FLOATS, e = i % BOX_FLOATS;
        const int yy = oy + e / BOX_W, xx = ox + e % BOX_W;
        float v = 0.0f;
        if (yy < a.bh && xx < a.bw) {
          const bool ll = q == 0;
          const float* src = ll ? a.ll_ptr : a.plane;
          const int pitch = ll ? a.ll_pitch : a.plane_w;
          const int rows = ll ? a.ll_rows : a.plane_h;
          const int gy = yy + ((q >= 2) ? a.bh : 0), gx = xx + ((q & 1) ? a.bw : 0);
          v = src[((uint64_t)c * rows + gy) * pitch + gx];
        }
        box[q * (BOX_SLOT / 4) + e] = v;
      }
      __syncthreads();
    }
    issued = false;

    // column pass: lane = column x, warp = segment of SEG output row pairs;
    // the 8 pairs (L and H halves packed) stay in registers
    const int strip = warp % NSTRIP, seg = warp / NSTRIP;
    const int x = ax + TXS * strip - HALO + lane;
    const int pa = ay + SEG * seg, pb = min(pa + SEG, by);
    float2 cs[SEG], cd[SEG];   // (s3, d3) of pair q: .x = L half, .y = H half
    const bool col_live = x >= 0 && x < min(bx + HALO, a.bw) && pa < pb;
    if (col_live) {
      const int lc = x - ox;
      auto emit = [&](int p, float2 s3, float2 d3) {
        cs[p - HALO] = s3;   // compile-time index after unrolling
        cd[p - HALO] = d3;
      };
      if (pa >= HALO && pa + SEG + HALO <= a.bh) {
        const int rb = pa - HALO - oy;
        lift_interior<SEG>(
            z,
            [&](int j, float2& s_, float2& d_) {
              const int o = (rb + j) * BOX_W + lc;
              WV_ASSERT(o >= 0 && o < BOX_FLOATS);
              s_ = make_float2(bLL[o], bHL[o]);
              d_ = make_float2(bLH[o], bHH[o]);
            },
            emit);
      } else {
        // a level border inside the segment: whole-sample symmetric extension
        // of the interleaved line (x[-k] = x[k], x[2N-1+k] = x[2N-1-k]) is
        // carried through every lifting step unchanged, so loading mirrored
        // coefficients equals the reference's per-step extension
        // (wavelets.py:82-101) bit for bit: s[-k] = s[k], d[-k] = d[k-1],
        // s[N+m] = s[N-1-m], d[N+m] = d[N-2-m].  Pairs past the border are
        // computed from rows clamped into the box and never emitted.
        const int g0 = pa - HALO, N = a.bh;
        const int glo = oy, ghi = min(N, oy + BOX_H) - 1;   // rows held by the box
        lift_interior<SEG>(
            z,
            [&](int j, float2& s_, float2& d_) {
              const int g = g0 + j;
              int gs = g, gd = g;
              if (g < 0) {
                gs = -g;
                gd = -g - 1;
              } else if (g >= N) {
                gs = 2 * N - 1 - g;
                gd = 2 * N - 2 - g;
              }
              gs = min(max(gs, glo), ghi);
              gd = min(max(gd, glo), ghi);
              const int os = (gs - oy) * BOX_W + lc, od = (gd - oy) * BOX_W + lc;
              WV_ASSERT(os >= 0 && os < BOX_FLOATS && od >= 0 && od < BOX_FLOATS);
              s_ = make_float2(bLL[os], bHL[os]);
              d_ = make_float2(bLH[od], bHH[od]);
            },
            emit);
      }
    }
    // every warp is done with the boxes (and the staged request words)
    const bool unmasked = __syncthreads_and(rq_all) != 0 && WV_K3_UNMASKED;
    if ((FINAL || WV_K3_MID_PREFETCH) && a.use_tma) {
      // the boxes are consumed: start the next item's loads now (only the
      // elected thread read nxt_entry and issues)
      issued = !(nxt_entry & ZERO_FLAG);   // meaningful for the elected thread only
      if (issued) issue(nxt);
    }
    // row pass: each row pair (two output rows packed) lifted across the
    // lanes; neighbours by shuffle, symmetric extension at the level borders
    // (wavelets.py:94-101) by reading the lane's own value there.  Lanes
    // 2..29 emit; 0, 1, 30, 31 are the halo.  All eight pairs are lifted
    // unconditionally (the shuffles stay warp-converged); pairs past the
    // segment's end are not stored.
    const int up = x == 0 ? lane : lane - 1;          // source of d[x-1]
    const int dn = x == a.bw - 1 ? lane : lane + 1;   // source of s[x+1]
    const bool emit = lane >= HALO && lane < 32 - HALO && x < bx;
    const int npairs = pb - pa;   // <= SEG, may be <= 0
    auto sh2 = [](float2 v, int src) {
      return make_float2(__shfl_sync(0xFFFFFFFFu, v.x, src), __shfl_sync(0xFFFFFFFFu, v.y, src));
    };
    auto cv = [](float v) { return u8_rint(__fmul_rn(v, 255.0f)); };
    // final: this lane's request bits (pixels 2x, 2x+1) sit at bit px & 31 of
    // staged word (px >> 5) - w0 of each output row
    const int px = 2 * x;
    const uint32_t* rql = rq + (2 * (pa - ay)) * RQ_WORDS + ((px >> 5) - w0);
    const int rsh = px & 31;
    uint8_t* crow = FINAL ? canvas + ((uint64_t)c * H + 2 * pa) * W + px : nullptr;
    float* orow = FINAL ? nullptr : a.out + ((uint64_t)c * H + 2 * pa) * a.out_pitch + 2 * x;
    // lift pair q across the lanes -> (s3, d3): .x = row 2p, .y = row 2p+1
    // lift RP row pairs q .. q+RP-1 across the lanes, stage by stage, so
    // their shuffle round trips overlap -> (s3, d3): .x = row 2p, .y = 2p+1
    auto lift_pairs = [&](int q, float2 (&s3)[RP], float2 (&d3)[RP]) {
      float2 s2[RP], d1[RP], d2[RP];
#pragma unroll
      for (int r = 0; r < RP; ++r) {
        d1[r] = pmul(make_float2(cs[q + r].y, cd[q + r].y), IK, z);   // H half
        s2[r] = pmul(make_float2(cs[q + r].x, cd[q + r].x), KS, z);   // L half (s1)
      }
#pragma unroll
      for (int r = 0; r < RP; ++r) s2[r] = lstep(s2[r], ND, sh2(d1[r], up), d1[r], z);
#pragma unroll
      for (int r = 0; r < RP; ++r) d2[r] = lstep(d1[r], NG, s2[r], sh2(s2[r], dn), z);
#pragma unroll
      for (int r = 0; r < RP; ++r) s3[r] = lstep(s2[r], NB, sh2(d2[r], up), d2[r], z);
#pragma unroll
      for (int r = 0; r < RP; ++r) d3[r] = lstep(d2[r], NA, s3[r], sh2(s3[r], dn), z);
    };
    // one unrolled loop per store kind (a branch inside the loop would keep
    // both epilogues' registers live)
    if (!FINAL) {
#pragma unroll
      for (int q0 = 0; q0 < SEG; q0 += RP) {
        float2 s3v[RP], d3v[RP];
        lift_pairs(q0, s3v, d3v);
#pragma unroll
        for (int r = 0; r < RP; ++r) {
          const int q = q0 + r;
          const float2 s3 = s3v[r], d3 = d3v[r];
          if (emit && q < npairs) {
            *reinterpret_cast<float2*>(orow + (2 * q) * (size_t)a.out_pitch) = make_float2(s3.x, d3.x);
            *reinterpret_cast<float2*>(orow + (2 * q + 1) * (size_t)a.out_pitch) =
                make_float2(s3.y, d3.y);
          }
        }
      }
    } else {
      // clip(rint(x*255)) (decoding.py:301), request-masked unless the whole
      // tile is requested; 2 pixels per row
#pragma unroll
      for (int q0 = 0; q0 < SEG; q0 += RP) {
        float2 s3v[RP], d3v[RP];
        lift_pairs(q0, s3v, d3v);
#pragma unroll
        for (int r = 0; r < RP; ++r) {
          const int q = q0 + r;
          const float2 s3 = s3v[r], d3 = d3v[r];
          if (emit && q < npairs) {
            uint32_t m0 = 0xFFFFu, m1 = 0xFFFFu;
            if (!unmasked) {
              const uint32_t b0 = (rql[(2 * q) * RQ_WORDS] >> rsh) & 3u;
              const uint32_t b1 = (rql[(2 * q + 1) * RQ_WORDS] >> rsh) & 3u;
              // bits (0, 1) -> byte masks (0x00FF, 0xFF00)
              m0 = ((b0 | (b0 << 7)) & 0x101u) * 0xFFu;
              m1 = ((b1 | (b1 << 7)) & 0x101u) * 0xFFu;
            }
            const uint32_t v0 = (cv(s3.x) | (cv(d3.x) << 8)) & m0;
            const uint32_t v1 = (cv(s3.y) | (cv(d3.y) << 8)) & m1;
            *reinterpret_cast<uint16_t*>(crow + (2 * q) * (size_t)W) = (uint16_t)v0;
            *reinterpret_cast<uint16_t*>(crow + (2 * q + 1) * (size_t)W) = (uint16_t)v1;
          }
        }
      }
    }
    slot ^= 1;
  }
}

PFN_cuTensorMapEncodeTiled_v12000 get_encoder() {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess)
    return nullptr;
  return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
}

int make_map(CUtensorMap* m, const float* base, int cols, int rows, int pitch, int chans,
             int box_w = BOX_W, int box_h = BOX_H) {
  static PFN_cuTensorMapEncodeTiled_v12000 enc = get_encoder();  // immutable after init
  if (!enc) return WV_ERR_CUDA;
  cuuint64_t dims[3] = {(cuuint64_t)cols, (cuuint64_t)rows, (cuuint64_t)chans};
  cuuint64_t strides[2] = {(cuuint64_t)pitch * 4, (cuuint64_t)pitch * 4 * rows};
  cuuint32_t box[3] = {(cuuint32_t)box_w, (cuuint32_t)box_h, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, (void*)base, dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? WV_OK : WV_ERR_CUDA;
}

// one level with the per-tile TMA-box kernel (k_level)
int launch_tiles(const Layout& lo, const wv_frame_args* fa, uint8_t* ws, cudaStream_t s, int k,
                 int sms, float* f32_out = nullptr) {
  const int L = lo.L, C = lo.C;
  float* plane = (float*)(ws + lo.plane);
  const uint32_t* counters = (const uint32_t*)(ws + lo.counters);
  static int occ_mid = 0, occ_fin = 0;   // per-process constants of the kernels
  if (!occ_fin) {
    WV_CUDA(cudaFuncSetAttribute(k_level<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 SMEM_MID));
    WV_CUDA(cudaFuncSetAttribute(k_level<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 SMEM_FIN));
    int om = 1, of = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&om, k_level<false>, NTHREADS, SMEM_MID);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&of, k_level<true>, NTHREADS, SMEM_FIN);
    occ_mid = max(om, 1);
    occ_fin = max(of, 1);
  }
  CUtensorMap tm_plane;
  if (make_map(&tm_plane, plane, lo.W, lo.H, lo.W, C) != WV_OK) return WV_ERR_CUDA;
  CUtensorMap tm_ll = tm_plane;
  if (k < L) {
    if (make_map(&tm_ll, (const float*)(ws + lo.ybuf[k]), lo.W >> k, lo.H >> k, lo.ypitch[k], C) !=
        WV_OK)
      return WV_ERR_CUDA;
  }
  LevelArgs la{};
  la.neg_zero = -0.0f;
  la.k = k; la.bh = lo.H >> k; la.bw = lo.W >> k; la.C = C; la.ntx = lo.ntx[k];
  la.divC = fast_div((uint32_t)C);
  la.divN = fast_div((uint32_t)lo.ntx[k]);
  la.use_tma = (la.bw % 4) == 0;
  la.ll_ptr = k < L ? (const float*)(ws + lo.ybuf[k]) : plane;
  la.ll_pitch = k < L ? lo.ypitch[k] : lo.W;
  la.ll_rows = k < L ? (lo.H >> k) : lo.H;
  la.plane = plane; la.plane_w = lo.W; la.plane_h = lo.H;
  la.list = (const uint32_t*)(ws + lo.tlist[k]);
  la.count = counters + CNT_TILES + k;
  const int ntiles = lo.nty[k] * lo.ntx[k];
  if (k > 1 || f32_out) {
    // mid levels into the next level's LL buffer; with f32_out level 1 too
    // (wv_synthesize_2d: a float32 frame instead of the u8 canvas)
    la.out = k > 1 ? (float*)(ws + lo.ybuf[k - 1]) : f32_out;
    la.out_pitch = k > 1 ? lo.ypitch[k - 1] : lo.W;
    const int grid = max(1, min(ntiles * C, sms * occ_mid));
    WV_CUDA(launch_k(k_level<false>, dim3(grid), dim3(NTHREADS), (size_t)SMEM_MID, s, tm_ll,
                     tm_plane, la));
  } else {
    la.fa = fa;
    la.R = (const uint32_t*)(ws + lo.mrows);
    la.rowmap = (const uint32_t*)(ws + lo.rowmap);
    la.wpr0 = lo.wpr_[0];
    const int grid = max(1, min(ntiles * C, sms * occ_fin));
    WV_CUDA(launch_k(k_level<true>, dim3(grid), dim3(NTHREADS), (size_t)SMEM_FIN, s, tm_ll,
                     tm_plane, la));
  }
  WV_CUDA(cudaGetLastError());
  return WV_OK;
}

}  // namespace

int launch_synthesis(const Layout& lo, const wv_geometry* g, const wv_frame_args* fa, uint8_t* ws,
                     cudaStream_t s, int only_level) {
  (void)g;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  for (int k = lo.L; k >= 1; --k) {
    if (only_level && k != only_level) continue;
    const int st = launch_tiles(lo, fa, ws, s, k, sms);
    if (st != WV_OK) return st;
  }
  return WV_OK;
}

// Full-frame float32 synthesis of a Mallat pyramid already in the plane
// (wv_synthesize_2d): the per-tile kernel for every level, level 1 into f32_out.
int launch_synthesis_f32(const Layout& lo, const wv_frame_args* fa, uint8_t* ws, float* f32_out,
                         cudaStream_t s) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  for (int k = lo.L; k >= 1; --k) {
    const int st = launch_tiles(lo, fa, ws, s, k, sms, k == 1 ? f32_out : nullptr);
    if (st != WV_OK) return st;
  }
  return WV_OK;
}

}  // namespace wv
