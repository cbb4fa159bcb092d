// Shared device/host definitions for the B200 decode path.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/wavevid_b200.h"

namespace wv {

// synthesis tile: TY x TX coefficients per subband -> (2TY) x (2TX) outputs
#ifndef WV_TILE_Y
#define WV_TILE_Y 32
#endif
constexpr int TY = WV_TILE_Y;
#ifndef WV_K3_STRIPS
#define WV_K3_STRIPS 1
#endif
constexpr int TXS = 28;               // columns of one warp strip (+ 2 halo each side = 32 lanes)
constexpr int TX = TXS * WV_K3_STRIPS;   // tile width: WV_K3_STRIPS strips side by side
constexpr int HALO = 2;               // lifting support per side
// TMA box: the innermost box coordinate must be 16-byte aligned (unaligned or
// negative-unaligned starts raise an illegal-instruction fault on B200), so
// the box starts at ax-4 (ax is a multiple of 28 floats = 112 bytes) and
// spans 36 floats.
constexpr int XPAD = 4;
constexpr int BOX_W = TX + 2 * XPAD;
constexpr int BOX_H = TY + 2 * HALO;
constexpr int OUT_H = 2 * TY;
constexpr int OUT_W = 2 * TX;
constexpr uint32_t ZERO_FLAG = 0x80000000u;  // work-list entry: zero-fill only
constexpr int DIL = 4;                // WaveletKind.CDF97.half_width (wavelets.py:30-32)

__host__ __device__ inline int wpr(int cols) { return (cols + 31) >> 5; }
__host__ __device__ inline int cdiv(int a, int b) { return (a + b - 1) / b; }

// Offsets of every workspace region (bytes from the workspace base).
struct Layout {
  int L, C, H, W, NB, nbx, bs, n;
  int mh, mw;
  int wpr_[WV_MAX_LEVELS + 1];           // words per bit row at level j
  uint64_t mrows;                        // mask rows at full width (mh x wpr0)
  uint64_t rowmap;                       // u32[H]: pixel row -> mask row (fileio.py:434)
  uint64_t stack[WV_MAX_LEVELS + 1];     // level j (1..L): (L+1) masks
  uint64_t stack_stride[WV_MAX_LEVELS + 1];
  uint64_t fp[WV_MAX_LEVELS + 1];        // footprint intermediates, level 1..L-1
  uint64_t pooled[WV_MAX_LEVELS + 1];    // D_j pooled to 32x32 cells: one word per 32x1024 tile
  uint64_t sel, prev_sel;                // NB-bit bitmaps
  uint64_t blist;                        // NB u32 entries
  uint64_t bstate;                       // u8[NB]: plane block may hold nonzeros (K2)
  uint64_t flist;                        // NB u32: blocks whose records are fetched (WV_FLAG_FETCH)
  int nty[WV_MAX_LEVELS + 1], ntx[WV_MAX_LEVELS + 1];  // tile grid of synthesis level k
  uint64_t need[WV_MAX_LEVELS + 1];      // u8 per tile
  uint64_t prev_need;                    // level 1, u8 per tile
  uint64_t tlist[WV_MAX_LEVELS + 1];     // u32 per tile
  uint64_t counters;                     // u32[64]
  uint64_t desc;                         // device wv_frame_args + 4 wv_view_args + mask bytes
  uint64_t desc_mask, desc_bytes;        // mask offset inside the slot, slot size
  uint64_t plane;                        // C x H x W f32
  uint64_t ybuf[WV_MAX_LEVELS + 1];      // level k (1..L-1): C x (H>>k) x pitch[k] f32
  int ypitch[WV_MAX_LEVELS + 1];
  uint64_t mbits;                        // low-res mask as bit rows: mh x ceil(mw/32) u32
  uint64_t select_bytes;                 // prefix holding all selection state (wv_select alone)
  uint64_t total;
};

// counter slots
enum { CNT_BLOCKS = 0, CNT_TILES = 1 /* + level */, CNT_FETCH = 40 };

inline int build_layout(const wv_geometry* g, Layout* o) {
  if (!g || !o) return WV_ERR_ARG;
  const int L = g->levels, W = g->width, H = g->height, C = g->channels;
  const int bs = g->block_size, n = g->inter_size;
  if (L < 1 || L > WV_MAX_LEVELS - 1 || C < 1 || C > 4 || bs < 1 || bs > 64 || n < 1 ||
      n > 256 || W < 2 || H < 2 || (W % (1 << L)) || (H % (1 << L)) || (W % bs) || (H % bs) ||
      g->mask_w < 1 || g->mask_h < 1 || (bs & (bs - 1)) || (n & (n - 1)))
    return WV_ERR_ARG;
  if ((W % 4) != 0) return WV_ERR_UNSUPPORTED;  // TMA row strides need 16-B multiples
  // 32-bit index maps in the mask kernels
  if ((uint64_t)W * g->mask_w >= (1ull << 32) || (uint64_t)H * g->mask_h >= (1ull << 32))
    return WV_ERR_UNSUPPORTED;
  o->L = L; o->C = C; o->H = H; o->W = W; o->bs = bs; o->n = n;
  o->nbx = W / bs; o->NB = (W / bs) * (H / bs);
  o->mh = g->mask_h; o->mw = g->mask_w;
  uint64_t off = 0;
  auto take = [&](uint64_t bytes) { uint64_t r = off; off += (bytes + 255) & ~uint64_t(255); return r; };
  for (int j = 0; j <= L; ++j) o->wpr_[j] = wpr(W >> j);
  o->mrows = take(uint64_t(g->mask_h) * o->wpr_[0] * 4);
  o->rowmap = take(uint64_t(H) * 4);
  for (int j = 1; j <= L; ++j) {
    uint64_t one = uint64_t(H >> j) * o->wpr_[j] * 4;
    one = (one + 255) & ~uint64_t(255);
    o->stack_stride[j] = one;
    o->stack[j] = take(one * (L + 1));
  }
  for (int j = 1; j < L; ++j) o->fp[j] = take(uint64_t(H >> j) * o->wpr_[j] * 4);
  for (int j = 1; j <= L; ++j)
    o->pooled[j] = take(uint64_t(cdiv(H >> j, 32)) * cdiv(o->wpr_[j], 32) * 4);
  o->sel = take(uint64_t(wpr(o->NB)) * 4);
  o->prev_sel = take(uint64_t(wpr(o->NB)) * 4);
  o->blist = take(uint64_t(o->NB) * 4);
  o->bstate = take(uint64_t(o->NB));
  o->flist = take(uint64_t(o->NB) * 4);
  for (int k = 1; k <= L; ++k) {
    o->nty[k] = cdiv(H >> k, TY);
    o->ntx[k] = cdiv(W >> k, TX);
    uint64_t nt = uint64_t(o->nty[k]) * o->ntx[k];
    // level 1: need bits (rows of tiles); other levels unused
    o->need[k] = take(k == 1 ? uint64_t(o->nty[1]) * wpr(o->ntx[1]) * 4 : 4);
    o->tlist[k] = take(nt * 4 * (k == 1 ? 2 : 1));
  }
  o->prev_need = take(uint64_t(o->nty[1]) * o->ntx[1]);
  o->counters = take(64 * 4);
  o->desc_mask = (sizeof(wv_frame_args) + 4 * sizeof(wv_view_args) + 15) & ~size_t(15);
  o->desc_bytes = o->desc_mask + (uint64_t(g->mask_h) * g->mask_w + 15) / 16 * 16;
  o->desc = take(o->desc_bytes);
  o->mbits = take(uint64_t(g->mask_h) * ((g->mask_w + 31) / 32) * 4);
  // everything above is selection state; the synthesis buffers come last, so
  // a selection-only workspace (prefetch accounting) is a prefix
  o->select_bytes = off;
  o->plane = take(uint64_t(C) * H * W * 4);
  for (int k = 1; k < L; ++k) {
    int cols = W >> k;
    o->ypitch[k] = (cols + 3) & ~3;
    o->ybuf[k] = take(uint64_t(C) * (H >> k) * o->ypitch[k] * 4);
  }
  o->total = off;
  return WV_OK;
}

// Debug builds (-DWV_CHECK=1, e.g. build.build(defines=["WV_CHECK=1"], ...)
// + WV_LIB) trap on out-of-range shared-memory indices in K3/K4; release
// builds compile the checks away.
#if defined(WV_CHECK) && WV_CHECK
#define WV_ASSERT(c)                 \
  do {                               \
    if (!(c)) __trap();              \
  } while (0)
#else
#define WV_ASSERT(c) \
  do {               \
  } while (0)
#endif

// Programmatic dependent launch (WV_PDL=1): kernels of the decode sequence
// are launched with programmatic stream serialization; each first waits for
// its predecessor grid (griddepcontrol.wait: completion + memory visibility)
// and then lets its successor launch.  Measured slower end to end on B200
// (serial frame latency +0.1-0.25 ms, early-resident successor CTAs), so it
// is off by default; the launch path is shared.
#ifndef WV_PDL
#define WV_PDL 0
#endif
__device__ __forceinline__ void pdl_sync() {
#if WV_PDL
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
}

template <typename... KArgs, typename... Args>
inline cudaError_t launch_k(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                            cudaStream_t s, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = WV_PDL;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<Args&&>(args)...);
}

#define WV_CUDA(x)                                   \
  do {                                               \
    cudaError_t e_ = (x);                            \
    if (e_ != cudaSuccess) return WV_ERR_CUDA;       \
  } while (0)

// ---- kernel launchers (defined in the .cu files) ----
// Launchers take the frame arguments as a DEVICE pointer (the descriptor slot
// of the workspace): kernels read every per-frame value from it, so the launch
// sequence of a mode is fixed and can be captured in a CUDA graph.
int launch_select(const Layout& lo, const wv_geometry* g, int mode, int flags,
                  const wv_frame_args* d_fa, uint8_t* ws, cudaStream_t s,
                  int stages = WV_STAGE_SELECT);
int launch_fetch(const Layout& lo, const wv_frame_args* fa, uint8_t* ws, cudaStream_t s);
int launch_table_expand(const uint16_t* d_counts, uint64_t n, int rs, uint64_t* d_table,
                        cudaStream_t s);
int launch_temporal(const Layout& lo, const wv_geometry* g, int mode, const wv_frame_args* d_fa,
                    uint8_t* ws, cudaStream_t s);
int launch_synthesis(const Layout& lo, const wv_geometry* g, const wv_frame_args* d_fa,
                     uint8_t* ws, cudaStream_t s, int only_level = 0);
int launch_synthesis_f32(const Layout& lo, const wv_frame_args* fa, uint8_t* ws, float* f32_out,
                         cudaStream_t s);
int launch_perspective(const wv_view_args* v, int n, cudaStream_t s);
int launch_perspective_dev(const wv_view_args* d_views, int n, int max_w, int max_h,
                           int shared_geometry, cudaStream_t s);

}  // namespace wv
