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
// Per (tile, channel) item: one elected thread issues four TMA box loads
// (LL, HL, LH, HH; 40x36 f32 each, far-edge out-of-range zero-filled) completing on an
// mbarrier.  The column pass streams each box column through registers with
// the L-half (LL/LH) and H-half (HL/HH) lines packed as float2 and lifted with
// Blackwell's paired FP32 ops (__fadd2_rn/__fmul2_rn, RN, no FMA); results land
// row-pair-interleaved so the row pass again lifts two output rows per
// thread as one float2 stream.  Mid levels stage the f32 output tile in shared
// memory and write it with coalesced stores; the finest level converts to u8
// in registers and stores each 16-pixel row segment, request-masked, straight
// to the canvas.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstdlib>

#include "wv_common.cuh"

namespace wv {
namespace {

constexpr int BOX_FLOATS = BOX_W * BOX_H;
constexpr int BOX_SLOT = ((BOX_FLOATS * 4 + 127) / 128) * 128;  // bytes
constexpr int CB_PITCH = BOX_W + 1;   // float2 units, odd -> conflict-free row pass
constexpr int OB_PITCH = OUT_W + 1;   // float2 units (row pairs), odd
// line segments: every column (row) lifting stream covers SEGLEN_C
// (SEGLEN_R) output pairs plus its own 2-pair halo on each side
#ifndef WV_K3_CVT_U8
#define WV_K3_CVT_U8 1
#endif
#ifndef WV_SEGLEN_C
#define WV_SEGLEN_C 8
#endif
#ifndef WV_SEGLEN_R
#define WV_SEGLEN_R 8
#endif
#ifndef WV_SEGLEN_RF
#define WV_SEGLEN_RF 8    // finest level row segments (16 measured slower)
#endif
constexpr int SEGLEN_C = WV_SEGLEN_C, SEGLEN_R = WV_SEGLEN_R, SEGLEN_RF = WV_SEGLEN_RF;
constexpr int COL_SEGS = TY / SEGLEN_C, ROW_SEGS = TX / SEGLEN_R;
static_assert(SEGLEN_RF % 8 == 0 && SEGLEN_RF <= TX, "finest row segments store 16-pixel chunks");
constexpr int NTHREADS_MIN = (COL_SEGS * BOX_W > ROW_SEGS * TY ? COL_SEGS * BOX_W : ROW_SEGS * TY);
#ifdef WV_K3_THREADS
constexpr int NTHREADS = WV_K3_THREADS;
#else
constexpr int NTHREADS = NTHREADS_MIN <= 64 ? 64 : (NTHREADS_MIN <= 128 ? 128 : (NTHREADS_MIN + 31) / 32 * 32);
#endif
static_assert(NTHREADS >= NTHREADS_MIN, "every segment needs a thread");
static_assert(TY * OB_PITCH * 8 <= 4 * BOX_SLOT, "output tile must fit in the box region");

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
// d * (1/K) feeds the packed add (d[i-1] + d[i]) of the next lifting step; a
// packed multiply there would be contracted into FFMA2 by ptxas, so the
// scale is two scalar round-to-nearest multiplies (never contracted).
__device__ __forceinline__ float2 dscale(float2 d, float2 ik) {
  return make_float2(__fmul_rn(d.x, ik.x), __fmul_rn(d.y, ik.y));
}
// x - k*(y1 + y2), written as x + (-k)*(y1+y2): identical rounding.  The
// final add is issued as two scalar FADDs: ptxas contracts a paired
// mul.rn.f32x2 feeding add.rn.f32x2 into FFMA2 (observed with CUDA 12.9),
// which would change the rounding; scalar adds keep the product rounded.
__device__ __forceinline__ float2 lstep(float2 x, float2 nk, float2 y1, float2 y2) {
  const float2 t = __fmul2_rn(nk, __fadd2_rn(y1, y2));
  return make_float2(__fadd_rn(x.x, t.x), __fadd_rn(x.y, t.y));
}

// Inverse CDF 9/7 lifting of one line (two packed lines) over global
// coefficient indices [g0, g1) of a level of length N; emits pairs p in
// [a, b) as (s3[p], d3[p]).  Left/right symmetric extension applies only when
// g0 == 0 / g1 == N (wavelets.py:82-91, :94-101).
template <class Load, class Emit>
__device__ __forceinline__ void lift_line(int g0, int g1, int N, int a, int b, Load load,
                                          Emit emit) {
  const float2 KS = f2(__uint_as_float(0x3f9d7658u));    // K
  const float2 IK = f2(__uint_as_float(0x3f5019c3u));    // 1/K
  const float2 ND = f2(-__uint_as_float(0x3ee31355u));   // -delta
  const float2 NG = f2(-__uint_as_float(0x3f620676u));   // -gamma
  const float2 NB = f2(-__uint_as_float(0xbd5901aeu));   // -beta
  const float2 NA = f2(-__uint_as_float(0xbfcb0673u));   // -alpha
  float2 sr, dr;
  // j = g0 (at the left border d1[-1] = d1[0]; elsewhere the value is a halo)
  load(g0, sr, dr);
  float2 d1m = dscale(dr, IK);
  float2 s2m = lstep(__fmul2_rn(sr, KS), ND, d1m, d1m);
  float2 d2mm = d1m, s3mm = s2m;
  if (g1 - g0 >= 2) {
    // j = g0 + 1 (at the left border d2[-1] = d2[0])
    load(g0 + 1, sr, dr);
    float2 d1 = dscale(dr, IK);
    float2 s2 = lstep(__fmul2_rn(sr, KS), ND, d1m, d1);
    float2 d2 = lstep(d1m, NG, s2m, s2);
    s3mm = lstep(s2m, NB, d2, d2);
    d2mm = d2;
    d1m = d1;
    s2m = s2;
#pragma unroll 4
    for (int j = g0 + 2; j < g1; ++j) {
      load(j, sr, dr);
      d1 = dscale(dr, IK);
      s2 = lstep(__fmul2_rn(sr, KS), ND, d1m, d1);   // s2[j]
      d2 = lstep(d1m, NG, s2m, s2);                   // d2[j-1]
      float2 s3 = lstep(s2m, NB, d2mm, d2);           // s3[j-1]
      float2 d3 = lstep(d2mm, NA, s3mm, s3);          // d3[j-2]
      const int p = j - 2;
      if (p >= a && p < b) emit(p, s3mm, d3);
      d2mm = d2;
      s3mm = s3;
      d1m = d1;
      s2m = s2;
    }
  }
  if (g1 == N) {
    float2 d2 = lstep(d1m, NG, s2m, s2m);                     // d2[N-1]
    float2 s3 = lstep(s2m, NB, N == 1 ? d2 : d2mm, d2);       // s3[N-1]
    if (N >= 2 && N - 2 >= a && N - 2 < b) emit(N - 2, s3mm, lstep(d2mm, NA, s3mm, s3));
    if (N - 1 >= a && N - 1 < b) emit(N - 1, s3, lstep(d2, NA, s3, s3));
  }
}

// Interior segment (no level border inside [g0, g0 + LEN + 4)): the same
// stream with a compile-time trip count, fully unrolled -- no loop counter,
// no emission tests, constant shared-memory offsets.  Local indices: inputs
// 0 .. LEN+3, emitted pairs 2 .. LEN+1.
template <int LEN, class Load, class Emit>
__device__ __forceinline__ void lift_interior(Load load, Emit emit) {
  const float2 KS = f2(__uint_as_float(0x3f9d7658u));
  const float2 IK = f2(__uint_as_float(0x3f5019c3u));
  const float2 ND = f2(-__uint_as_float(0x3ee31355u));
  const float2 NG = f2(-__uint_as_float(0x3f620676u));
  const float2 NB = f2(-__uint_as_float(0xbd5901aeu));
  const float2 NA = f2(-__uint_as_float(0xbfcb0673u));
  float2 sr, dr;
  load(0, sr, dr);
  float2 d1m = dscale(dr, IK);
  float2 s2m = __fmul2_rn(sr, KS);         // s2[0] is a halo value: never emitted
  load(1, sr, dr);
  float2 d1 = dscale(dr, IK);
  float2 s2 = lstep(__fmul2_rn(sr, KS), ND, d1m, d1);
  float2 d2mm = lstep(d1m, NG, s2m, s2);   // d2[0] (halo)
  float2 s3mm = s2;                        // s3[0] (halo)
  d1m = d1;
  s2m = s2;
#pragma unroll
  for (int j = 2; j < LEN + 4; ++j) {
    load(j, sr, dr);
    d1 = dscale(dr, IK);
    s2 = lstep(__fmul2_rn(sr, KS), ND, d1m, d1);   // s2[j]
    const float2 d2 = lstep(d1m, NG, s2m, s2);      // d2[j-1]
    const float2 s3 = lstep(s2m, NB, d2mm, d2);     // s3[j-1]
    if (j >= 4) emit(j - 2, s3mm, lstep(d2mm, NA, s3mm, s3));   // d3[j-2]
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
};

// Items are (tile, channel).  Column pass: TY/SEGLEN_C segments x BOX_W
// columns (each segment lifts SEGLEN_C output row pairs from its own 2-row
// halo); row pass: TX/SEGLEN_R segments x TY row pairs.  Mid levels stage the
// f32 output tile in the box region (dead after the column pass) and store it
// coalesced.  The finest level needs no output tile: each row-pass thread
// keeps its 2 x 16 output bytes in registers and writes them with the
// request mask applied, so the box region is free as soon as the column pass
// ends and the next item's four TMA boxes are issued there, loading while
// this item's row pass runs (43 KB of shared memory: 5 CTAs per SM).
constexpr int BOXSET = 4 * BOX_SLOT;
constexpr int COL_BYTES = 2 * TY * CB_PITCH * 8;
#ifndef WV_K3_PAIRSEG
#define WV_K3_PAIRSEG 1  // finest row pass: a warp = 16 row pairs x 2 adjacent segments, so
                         // each 16-B store pair fills whole 32-B sectors
#endif
// row-pass thread -> (row pair i, segment sg)
template <bool FINAL>
__device__ __forceinline__ void row_map(int tid, int& i, int& sg) {
  if (FINAL && WV_K3_PAIRSEG && TY == 32) {
    const int w = tid >> 5, l = tid & 31;
    i = 16 * (w & 1) + (l & 15);
    sg = 2 * (w >> 1) + (l >> 4);
  } else {
    i = tid % TY;
    sg = tid / TY;
  }
}
#ifndef WV_K3_OUT4
#define WV_K3_OUT4 1   // mid-level output tile as float4 (s3.x, d3.x, s3.y, d3.y) per pair:
                       // one conflict-free 16-B shared store / load instead of two 8-B ones
#endif
constexpr int OB4_PITCH = TX + 1;     // float4 units, odd
static_assert(TY * OB4_PITCH * 16 <= 4 * BOX_SLOT, "float4 output tile must fit in the box region");
constexpr int SMEM_MID = BOXSET + COL_BYTES;
constexpr int SMEM_FIN = BOXSET + COL_BYTES;   // the u8 tile goes from registers to HBM

template <bool FINAL>
__global__ void __launch_bounds__(NTHREADS) k_level(const __grid_constant__ CUtensorMap tm_ll,
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
  float2* colL = reinterpret_cast<float2*>(smem + BOXSET);  // [TY][CB_PITCH]
  float2* colH = colL + TY * CB_PITCH;
  // mid levels: the f32 output tile aliases the boxes
  float2* outb = reinterpret_cast<float2*>(smem);
  constexpr bool PF = FINAL;   // next item's boxes issued after the column pass
  __shared__ uint64_t bar;

  const int tid = threadIdx.x;
  if (tid == 0) mbar_init(&bar, 1);
  __syncthreads();
  uint32_t phase = 0u;
  const int C = a.C;
  const uint32_t nitems = *a.count * (uint32_t)C;
  const int H = 2 * a.bh, W = 2 * a.bw;

  // issue the four box loads of an item (elected thread)
  auto issue = [&](uint32_t it) {
    if (tid != 0) return;
    const uint32_t itile = it / a.divC;
    const uint32_t tile = a.list[itile] & ~ZERO_FLAG;
    const int ty = (int)(tile / a.divN), tx = (int)tile - ty * a.ntx;
    // TMA faults on unaligned/negative innermost box coordinates (observed on
    // B200, driver 580): x starts at ax-4 clamped to 0
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
      const int qw = nx >> 2;
      for (int idx = tid; idx < ny * qw; idx += NTHREADS) {
        const int r = idx / qw, q = idx % qw;
        *reinterpret_cast<uint32_t*>(canvas + ((uint64_t)c * H + 2 * ay + r) * W + 2 * ax +
                                     4 * q) = 0u;
      }
      continue;
    }
    const int oy = max(ay - HALO, 0), ox = max(ax - XPAD, 0);
    // finest level: fetch this thread's request-mask words (rowmap -> R, two
    // dependent global loads) and the next item's list entry now, so their
    // latency hides behind the box wait and the column pass
    constexpr int SR = FINAL ? SEGLEN_RF : SEGLEN_R;
    uint32_t rq[2][SR / 8];
    uint32_t nxt_entry = ZERO_FLAG;
    const uint32_t nxt = item + gridDim.x;
    if (FINAL) {
      int i, sg;
      row_map<FINAL>(tid, i, sg);
      const int pa = ax + sg * SR;
      if (tid < (TX / SR) * TY && i < by - ay && pa < bx) {
#pragma unroll
        for (int rr = 0; rr < 2; ++rr) {
          const uint32_t* req = a.R + (uint64_t)a.rowmap[2 * ay + 2 * i + rr] * a.wpr0;
#pragma unroll
          for (int k = 0; k < SR / 8; ++k) {
            const int px = 2 * pa + 16 * k;
            rq[rr][k] = px < W ? req[px >> 5] : 0u;
          }
        }
      }
    }
    if (PF && tid == 0 && a.use_tma && nxt < nitems) nxt_entry = a.list[nxt / a.divC];
    if (a.use_tma) {
      if (!issued) issue(item);
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

    // column pass: (segment, box column) per thread, L and H halves packed
    if (tid < COL_SEGS * BOX_W) {
      const int lc = tid % BOX_W, sg = tid / BOX_W;
      const int cg = ox + lc;
      const int pa = ay + sg * SEGLEN_C, pb = min(pa + SEGLEN_C, by);
      if (pa < pb && cg >= max(ax - HALO, 0) && cg < min(bx + HALO, a.bw)) {
        if (pa >= HALO && pb + HALO <= a.bh && pb - pa == SEGLEN_C) {
          const int rb = pa - HALO - oy;          // local box row of input 0
          const int qb = pa - HALO - ay;          // output pair of input 0
          lift_interior<SEGLEN_C>(
              [&](int j, float2& s, float2& d) {
                const int o = (rb + j) * BOX_W + lc;
                WV_ASSERT(o >= 0 && o < BOX_FLOATS);
                s = make_float2(bLL[o], bHL[o]);
                d = make_float2(bLH[o], bHH[o]);
              },
              [&](int p, float2 s3, float2 d3) {
                WV_ASSERT(qb + p >= 0 && qb + p < TY && lc < CB_PITCH);
                colL[(qb + p) * CB_PITCH + lc] = make_float2(s3.x, d3.x);
                colH[(qb + p) * CB_PITCH + lc] = make_float2(s3.y, d3.y);
              });
        } else {
          lift_line(
              max(pa - HALO, 0), min(pb + HALO, a.bh), a.bh, pa, pb,
              [&](int j, float2& s, float2& d) {
                const int o = (j - oy) * BOX_W + lc;
                WV_ASSERT(o >= 0 && o < BOX_FLOATS);
                s = make_float2(bLL[o], bHL[o]);
                d = make_float2(bLH[o], bHH[o]);
              },
              [&](int p, float2 s3, float2 d3) {
                const int q = p - ay;
                WV_ASSERT(q >= 0 && q < TY && lc < CB_PITCH);
                colL[q * CB_PITCH + lc] = make_float2(s3.x, d3.x);
                colH[q * CB_PITCH + lc] = make_float2(s3.y, d3.y);
              });
        }
      }
    }
    __syncthreads();
    if (PF && a.use_tma) {
      // the boxes are consumed: start the next item's loads now (only the
      // elected thread read nxt_entry and issues)
      issued = !(nxt_entry & ZERO_FLAG);   // meaningful for the elected thread only
      if (issued) issue(nxt);
    }
    // row pass: (segment, output row pair) per thread, two rows packed
    if (tid < (TX / SR) * TY) {
      int i, sg;
      row_map<FINAL>(tid, i, sg);
      const int pa = ax + sg * SR, pb = min(pa + SR, bx);
      if (i < by - ay && pa < pb) {
        // finest level: clip(rint(x*255)) (decoding.py:301; rint is
        // round-half-even like __float2uint_rn, which also saturates below 0)
        // of the segment's 2 x 16 output pixels, kept in registers and
        // written to the canvas with the request mask applied
        auto cv = [](float v) { return u8_rint(__fmul_rn(v, 255.0f)); };
        uint32_t w0[SR / 2] = {}, w1[SR / 2] = {};   // rows 2i, 2i+1
        uint8_t* crow = FINAL ? canvas + ((uint64_t)c * H + 2 * ay + 2 * i) * W : nullptr;
        // mid levels: f32 pairs into outb
        auto emit_mid = [&](int q, float2 s3, float2 d3) {
          WV_ASSERT(q >= 0 && q < TX && i < TY);
          if (WV_K3_OUT4) {
            reinterpret_cast<float4*>(outb)[i * OB4_PITCH + q] = make_float4(s3.x, d3.x, s3.y, d3.y);
          } else {
            outb[i * OB_PITCH + 2 * q] = s3;
            outb[i * OB_PITCH + 2 * q + 1] = d3;
          }
        };
        if (pa >= HALO && pb + HALO <= a.bw && pb - pa == SR) {
          const int cb = pa - HALO - ox, qb = pa - HALO - ax;
          lift_interior<SR>(
              [&](int j, float2& s, float2& d) {
                WV_ASSERT(cb + j >= 0 && cb + j < CB_PITCH);
                s = colL[i * CB_PITCH + cb + j];
                d = colH[i * CB_PITCH + cb + j];
              },
              [&](int p, float2 s3, float2 d3) {
                if (!FINAL) {
                  emit_mid(qb + p, s3, d3);
                } else {
                  // p - HALO is the segment-local pair: compile-time after unrolling
                  const int lq = p - HALO;
                  w0[lq >> 1] |= (cv(s3.x) | (cv(d3.x) << 8)) << (16 * (lq & 1));
                  w1[lq >> 1] |= (cv(s3.y) | (cv(d3.y) << 8)) << (16 * (lq & 1));
                }
              });
          if (FINAL) {
            // 16-pixel chunks of each row: request bits -> byte masks, 16-byte stores
            auto bm = [](uint32_t b4) { return ((b4 * 0x00204081u) & 0x01010101u) * 0xFFu; };
#pragma unroll
            for (int rr = 0; rr < 2; ++rr) {
              const uint32_t* wr = rr ? w1 : w0;
#pragma unroll
              for (int k = 0; k < SR / 8; ++k) {
                const int px = 2 * pa + 16 * k;
                const uint32_t bits = (rq[rr][k] >> (px & 31)) & 0xFFFFu;
                const uint4 v = make_uint4(wr[4 * k] & bm(bits & 0xFu),
                                           wr[4 * k + 1] & bm((bits >> 4) & 0xFu),
                                           wr[4 * k + 2] & bm((bits >> 8) & 0xFu),
                                           wr[4 * k + 3] & bm(bits >> 12));
                uint8_t* dst = crow + (uint64_t)rr * W + px;
                if ((W & 15) == 0) {
                  *reinterpret_cast<uint4*>(dst) = v;
                } else {
                  uint32_t* d4 = reinterpret_cast<uint32_t*>(dst);
                  d4[0] = v.x;
                  d4[1] = v.y;
                  d4[2] = v.z;
                  d4[3] = v.w;
                }
              }
            }
          }
        } else {
          lift_line(
              max(pa - HALO, 0), min(pb + HALO, a.bw), a.bw, pa, pb,
              [&](int j, float2& s, float2& d) {
                WV_ASSERT(j - ox >= 0 && j - ox < CB_PITCH);
                s = colL[i * CB_PITCH + (j - ox)];
                d = colH[i * CB_PITCH + (j - ox)];
              },
              [&](int p, float2 s3, float2 d3) {
                if (!FINAL) {
                  emit_mid(p - ax, s3, d3);
                } else {
                  // level borders: two pixels per row straight to the canvas
                  const int px = 2 * p;
#pragma unroll
                  for (int rr = 0; rr < 2; ++rr) {
                    const int y = 2 * ay + 2 * i + rr;
                    const uint32_t bits =
                        (a.R[(uint64_t)a.rowmap[y] * a.wpr0 + (px >> 5)] >> (px & 31)) & 3u;
                    const uint32_t lo = rr ? cv(s3.y) : cv(s3.x), hi = rr ? cv(d3.y) : cv(d3.x);
                    *reinterpret_cast<uint16_t*>(crow + (uint64_t)rr * W + px) =
                        (uint16_t)(((bits & 1u) ? lo : 0u) | (((bits >> 1) & 1u) ? hi << 8 : 0u));
                  }
                }
              });
        }
      }
    }
    __syncthreads();   // mid: outb complete; final: colL / colH free for the next item
    if (!FINAL) {
      float* base = a.out + ((uint64_t)c * H + 2 * ay) * a.out_pitch + 2 * ax;
      if (nx == OUT_W && ny == OUT_H) {
        // full tile: 32 row pairs x 32 float2 columns, shifts only
        for (int idx = tid; idx < TY * TX; idx += NTHREADS) {
          const int i = idx / TX, x2 = idx % TX;
          float* r0 = base + (uint64_t)(2 * i) * a.out_pitch + 2 * x2;
          if (WV_K3_OUT4) {
            const float4 t = reinterpret_cast<const float4*>(outb)[i * OB4_PITCH + x2];
            *reinterpret_cast<float2*>(r0) = make_float2(t.x, t.y);
            *reinterpret_cast<float2*>(r0 + a.out_pitch) = make_float2(t.z, t.w);
          } else {
            const float2 u = outb[i * OB_PITCH + 2 * x2];
            const float2 v = outb[i * OB_PITCH + 2 * x2 + 1];
            *reinterpret_cast<float2*>(r0) = make_float2(u.x, v.x);
            *reinterpret_cast<float2*>(r0 + a.out_pitch) = make_float2(u.y, v.y);
          }
        }
      } else {
        const int half = nx >> 1;   // float2 columns per row
        for (int idx = tid; idx < (ny >> 1) * half; idx += NTHREADS) {
          const int i = idx / half, x2 = idx % half;
          float* r0 = base + (uint64_t)(2 * i) * a.out_pitch + 2 * x2;
          if (WV_K3_OUT4) {
            const float4 t = reinterpret_cast<const float4*>(outb)[i * OB4_PITCH + x2];
            *reinterpret_cast<float2*>(r0) = make_float2(t.x, t.y);
            *reinterpret_cast<float2*>(r0 + a.out_pitch) = make_float2(t.z, t.w);
          } else {
            const float2 u = outb[i * OB_PITCH + 2 * x2];
            const float2 v = outb[i * OB_PITCH + 2 * x2 + 1];
            *reinterpret_cast<float2*>(r0) = make_float2(u.x, v.x);
            *reinterpret_cast<float2*>(r0 + a.out_pitch) = make_float2(u.y, v.y);
          }
        }
      }
      __syncthreads();
    }
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
