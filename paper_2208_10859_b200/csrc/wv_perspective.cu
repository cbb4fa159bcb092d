// K4 — equirectangular -> perspective writeout with footprint coverage check.
//
// Reference: render_perspective (projection.py:111-172).  Per output pixel:
// camera ray through the pixel centre, normalised, rotated to world
// (float64), lon/lat via atan2/asin, fractional source position, bilinear
// blend of the u8 canvas in float32 with the reference's operation order,
// rint, clamp.  Any tap outside the decoded footprint counts as uncovered
// (the caller raises CoverageError).  The parity bar for this stage is
// +-1 LSB.
#include "wv_common.cuh"

namespace wv {
namespace {

#ifndef WV_K4_GEO2
#define WV_K4_GEO2 1     // tap geometry two rows per paired-FP32 stream (0: scalar, ~1% slower)
#endif

constexpr double kRad2Deg = 57.29577951308232;  // numpy.degrees factor 180/pi

constexpr int kMaxViews = 4;
struct Views {
  wv_view_args v[kMaxViews];
};

struct Taps {
  int x0, y0;
  float ax, ay;
};

// Exact-as-reference tap selection in float64 (the reference geometry).
__device__ __noinline__ Taps taps_f64(const wv_view_args& v, int x, int y) {
  const double u = __dsub_rn(__dmul_rn(__ddiv_rn(__dadd_rn((double)x, 0.5), (double)v.out_w), 2.0), 1.0);
  const double w = __dsub_rn(1.0, __dmul_rn(__ddiv_rn(__dadd_rn((double)y, 0.5), (double)v.out_h), 2.0));
  double rx = __dmul_rn(u, v.tan_h), ry = __dmul_rn(w, v.tan_v), rz = 1.0;
  const double nrm = sqrt(__dadd_rn(__dadd_rn(__dmul_rn(rx, rx), __dmul_rn(ry, ry)), 1.0));
  rx = __ddiv_rn(rx, nrm);
  ry = __ddiv_rn(ry, nrm);
  rz = __ddiv_rn(rz, nrm);
  const double* R = v.rot;
  const double wx = __dadd_rn(__dadd_rn(__dmul_rn(rx, R[0]), __dmul_rn(ry, R[1])), __dmul_rn(rz, R[2]));
  const double wy = __dadd_rn(__dadd_rn(__dmul_rn(rx, R[3]), __dmul_rn(ry, R[4])), __dmul_rn(rz, R[5]));
  const double wz = __dadd_rn(__dadd_rn(__dmul_rn(rx, R[6]), __dmul_rn(ry, R[7])), __dmul_rn(rz, R[8]));
  const double lon = __dmul_rn(atan2(wx, wz), kRad2Deg);
  const double lat = __dmul_rn(asin(fmin(fmax(wy, -1.0), 1.0)), kRad2Deg);
  const double fx = __dsub_rn(__dmul_rn(__ddiv_rn(__dadd_rn(lon, 180.0), 360.0), (double)v.width), 0.5);
  const double fy = __dsub_rn(__dmul_rn(__ddiv_rn(__dsub_rn(90.0, lat), 180.0), (double)v.rows), 0.5);
  const double flx = floor(fx), fly = floor(fy);
  Taps t;
  t.x0 = (int)flx;
  t.y0 = (int)fly;
  t.ax = (float)__dsub_rn(fx, flx);
  t.ay = (float)__dsub_rn(fy, fly);
  return t;
}

__device__ __forceinline__ int wrapx(int x, int n) { return x < 0 ? x + n : (x >= n ? x - n : x); }

// atan2 for finite arguments, not both zero: octant reduction + degree-15 odd
// minimax polynomial (max error 1.1e-7 rad in float32, i.e. < 2e-4 px of the
// 8K source; the coverage margin kNear is 4e-3 px).
__device__ __forceinline__ float rcp_approx(float x) {   // MUFU.RCP, no denormal fix-up
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float sqrt_approx(float x) {   // MUFU.SQRT; sqrt(0) = 0
  float r;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

#if !WV_K4_GEO2
__device__ __forceinline__ float fast_atan2(float y, float x) {
  const float ax = fabsf(x), ay = fabsf(y);
  const float mx = fmaxf(ax, ay), mn = fminf(ax, ay);
  const float a = mx > 1e-30f ? mn * rcp_approx(mx) : 0.0f;   // atan2(0, 0) = 0
  const float s = a * a;
  float p = -0.004054488614201546f;
  p = fmaf(p, s, 0.021862687543034554f);
  p = fmaf(p, s, -0.05591195821762085f);
  p = fmaf(p, s, 0.09642171859741211f);
  p = fmaf(p, s, -0.13908620178699493f);
  p = fmaf(p, s, 0.19946563243865967f);
  p = fmaf(p, s, -0.33329859375953674f);
  p = fmaf(p, s, 0.9999993443489075f);
  float r = a * p;
  r = ay > ax ? 1.5707963267948966f - r : r;
  r = x < 0.0f ? 3.141592653589793f - r : r;
  return copysignf(r, y);
}
#endif

// bits of columns [c0, c1) that fall in word w
__device__ __forceinline__ uint32_t range_bits(int c0, int c1, int w) {
  const int lo = max(c0 - 32 * w, 0), hi = min(c1 - 32 * w, 32);
  if (lo >= hi) return 0u;
  return (hi >= 32 ? 0xFFFFFFFFu : ((1u << hi) - 1u)) & (0xFFFFFFFFu << lo);
}

// Geometry in float32 (|fx| error < 1e-3 px at 8K); the bilinear value is
// continuous in (fx, fy), so this stays within +-1 LSB of the float64
// reference.  The coverage test must pick the reference's taps exactly: when
// a coordinate lies within kNear of an integer the union of both candidate
// tap sets is tested, and only if that union is not fully covered is the
// float64 reference geometry evaluated for the pixel.
constexpr float kNear = 4e-3f;

__device__ __noinline__ uint32_t fp_bits_wrap(const uint32_t* row, int x0, int len, int n) {
  uint32_t r = 0;
  for (int i = 0; i < len; ++i) {
    int xx = x0 + i;
    xx = xx < 0 ? xx + n : (xx >= n ? xx - n : xx);
    r |= ((__ldg(row + (xx >> 5)) >> (xx & 31)) & 1u) << i;
  }
  return r;
}

// bits [x0, x0+len) of a footprint row (len <= 4), wrapping in longitude
__device__ __forceinline__ uint32_t fp_bits(const uint32_t* row, int x0, int len, int n) {
  if (x0 >= 0 && x0 + len <= n) {
    const int w = x0 >> 5, sh = x0 & 31;
    uint64_t v = __ldg(row + w);
    if (sh + len > 32) v |= (uint64_t)__ldg(row + w + 1) << 32;
    return (uint32_t)(v >> sh) & ((1u << len) - 1u);
  }
  return fp_bits_wrap(row, x0, len, n);
}

struct ViewConst {
  float r[9];
  float tan_h, tan_v, inv_w, inv_h, sx, sy;
  int out_w, out_h, m, n, C, wpr0;
  uint32_t plane;
};

// One CTA renders a K4_TY x K4_TX output tile (16 x 32: 4 warps, K4_PPT = 4
// pixels per thread, rows ty + 4k; 8 CTAs of 22.5 KB per SM -- measured
// 4% faster than 32 x 32 tiles with 8 warps and 4 CTAs/SM).
// Phases: (1) float32 geometry of every pixel and the CTA's candidate-tap box; (2) the box is tested against the footprint;
// (3) the box of all C canvas planes is read with 4-byte loads and stored
// channel-interleaved (one 32-bit word per source pixel) in shared memory;
// (4) four shared loads per pixel feed the bilinear blend; (5) the tile's
// (rows, K4_TX*C) bytes are staged and written with 16-byte stores.  For a
// stereo pair the window holds both eyes' boxes at once when they fit, so
// phases (2)-(5) run once for the pair (one round of staging loads in flight,
// half the barriers).  Boxes that wrap in longitude, clamp at a pole or exceed
// the window use direct global gathers (projection.py:146-149 semantics).
#ifndef K4_TILE_Y
#define K4_TILE_Y 16
#endif
#ifndef K4_WARPS
#define K4_WARPS 4
#endif
constexpr int K4_NW = K4_WARPS, K4_NTH = 32 * K4_WARPS;   // warps / threads per CTA
constexpr int K4_TX = 32, K4_TY = K4_TILE_Y, K4_PPT = K4_TY / K4_NW;
static_assert(K4_PPT % 2 == 0, "channel 2 is blended for pixel pairs");
static_assert(K4_NW == 4 || K4_NW == 8, "the coverage reduction reads 4 or 8 warp words");
#ifndef K4_WIN_WORDS
#define K4_WIN_WORDS (9216 * K4_TILE_Y / 32)
#endif
constexpr int WIN_WORDS = K4_WIN_WORDS;         // window capacity, source pixels (32-bit words)
constexpr int BOX_MAX_W = 128;                  // widest box the footprint test covers
constexpr int OST_PITCH = K4_TX * 4;            // bytes per staged output row (C <= 4)
constexpr int OST_VIEW = K4_TY * OST_PITCH;
constexpr int K4_SMEM = WIN_WORDS * 4 + 2 * OST_VIEW;
#ifndef K4_MIN_BLOCKS
#define K4_MIN_BLOCKS 8
#endif


// clip(rint(v)) of the bilinear blend (projection.py:150-170) from the four
// taps' biased channel values.  v is a convex combination of bytes, rounded
// once per FMA, so it lies in [0, 255] up to 1e-5 and needs no clamp;
// adding 2^23 rounds half-to-even like np.rint and leaves the byte in the
// low mantissa bits.
__device__ __forceinline__ uint32_t blend(float b00, float b01, float b10, float b11, float ax,
                                          float ay) {
  const float top = fmaf(ax, b01 - b00, b00 - 8388608.0f);
  const float bot = fmaf(ax, b11 - b10, b10 - 8388608.0f);
  return __float_as_uint(fmaf(ay, bot - top, top) + 8388608.0f) & 0xFFu;
}

// blend() of two lanes at once with paired FP32 operations (each lane
// rounds exactly like the scalar code), per-lane weights; the taps are
// 2^23-biased channel values.  Returns byte x | byte y << 8.
__device__ __forceinline__ uint32_t blend_v2(float2 b00, float2 b01, float2 b10, float2 b11,
                                             float2 A, float2 B) {
  const float2 nk = make_float2(-8388608.0f, -8388608.0f);
  auto neg = [](float2 v) { return make_float2(-v.x, -v.y); };
  const float2 top = __ffma2_rn(A, __fadd2_rn(b01, neg(b00)), __fadd2_rn(b00, nk));
  const float2 bot = __ffma2_rn(A, __fadd2_rn(b11, neg(b10)), __fadd2_rn(b10, nk));
  const float2 v = __fadd2_rn(__ffma2_rn(B, __fadd2_rn(bot, neg(top)), top), neg(nk));
  return __byte_perm(__float_as_uint(v.x), __float_as_uint(v.y), 0x0040u);
}

// 2^23 + byte s of tap word w (selector: byte s, zeros, 0x4B)
__device__ __forceinline__ float biased(uint32_t w, uint32_t s) {
  return __uint_as_float(__byte_perm(0x4B000000u, w, 0x3004u + s));
}

// blend() of channels 0 and 1 of one pixel; returns byte 0 | byte 1 << 8.
__device__ __forceinline__ uint32_t blend2(uint32_t w00, uint32_t w01, uint32_t w10, uint32_t w11,
                                           float ax, float ay) {
  auto b = [](uint32_t w) { return make_float2(biased(w, 0), biased(w, 1)); };
  return blend_v2(b(w00), b(w01), b(w10), b(w11), make_float2(ax, ax), make_float2(ay, ay));
}

// t / d and t % d for 0 <= t <= 256 and 1 <= d <= 64 without an integer
// division: (t + 0.5) / d is at least 1/128 away from an integer, far beyond
// the float error, so the truncation is exact.
struct SmallDiv {
  int q, r;
};
__device__ __forceinline__ SmallDiv small_div(int t, int d, float inv_d) {
  const int q = __float2int_rz(((float)t + 0.5f) * inv_d);
  return SmallDiv{q, t - q * d};
}

// region pointers of a view, derived where they are used (keeping them live
// across the phases costs registers)
__device__ __forceinline__ const uint32_t* view_fp(const wv_view_args& w, int wpr0) {
  return w.d_footprint + (uint64_t)w.row0 * wpr0;
}
__device__ __forceinline__ const uint8_t* view_img(const wv_view_args& w) {
  return w.d_canvas + (uint64_t)w.row0 * w.width;
}

// float32 geometry of output column x: the camera ray's x component through
// the rotation.
struct ColGeo {
  float cx, cy, cz;
};
__device__ __forceinline__ ColGeo col_geo(const ViewConst& vc, int x) {
  const float u = ((float)x + 0.5f) * vc.inv_w - 1.0f;
  const float rx = u * vc.tan_h;
  return ColGeo{rx * vc.r[0] + vc.r[2], rx * vc.r[3] + vc.r[5], rx * vc.r[6] + vc.r[8]};
}
__device__ __forceinline__ float2 f2v(float v) { return make_float2(v, v); }
__device__ __forceinline__ float2 neg2(float2 v) { return make_float2(-v.x, -v.y); }
__device__ __forceinline__ float sel(bool c, float a, float b) { return c ? a : b; }

// fast_atan2 of two lanes, the arithmetic as paired FP32 operations (the
// per-lane selects, min/max and reciprocals stay scalar)
__device__ __forceinline__ float2 fast_atan2_x2(float2 y, float2 x) {
  const float2 ax = make_float2(fabsf(x.x), fabsf(x.y)), ay = make_float2(fabsf(y.x), fabsf(y.y));
  const float2 mx = make_float2(fmaxf(ax.x, ay.x), fmaxf(ax.y, ay.y));
  const float2 mn = make_float2(fminf(ax.x, ay.x), fminf(ax.y, ay.y));
  float2 a = __fmul2_rn(mn, make_float2(rcp_approx(mx.x), rcp_approx(mx.y)));
  a = make_float2(sel(mx.x > 1e-30f, a.x, 0.0f), sel(mx.y > 1e-30f, a.y, 0.0f));   // atan2(0, 0) = 0
  const float2 s = __fmul2_rn(a, a);
  float2 p = f2v(-0.004054488614201546f);
  p = __ffma2_rn(p, s, f2v(0.021862687543034554f));
  p = __ffma2_rn(p, s, f2v(-0.05591195821762085f));
  p = __ffma2_rn(p, s, f2v(0.09642171859741211f));
  p = __ffma2_rn(p, s, f2v(-0.13908620178699493f));
  p = __ffma2_rn(p, s, f2v(0.19946563243865967f));
  p = __ffma2_rn(p, s, f2v(-0.33329859375953674f));
  p = __ffma2_rn(p, s, f2v(0.9999993443489075f));
  float2 r = __fmul2_rn(a, p);
  const float2 rc = __fadd2_rn(f2v(1.5707963267948966f), neg2(r));
  r = make_float2(sel(ay.x > ax.x, rc.x, r.x), sel(ay.y > ax.y, rc.y, r.y));
  const float2 rp = __fadd2_rn(f2v(3.141592653589793f), neg2(r));
  r = make_float2(sel(x.x < 0.0f, rp.x, r.x), sel(x.y < 0.0f, rp.y, r.y));
  return make_float2(copysignf(r.x, y.x), copysignf(r.y, y.y));
}

// float32 tap geometry of the thread's K4_PPT pixels (column x, rows
// ybase + 8k) (WV_K4_GEO2: two rows per paired-FP32 stream).  The fast path and the
// general path both use this function, so they see identical taps.
__device__ __forceinline__ void geo_all(const ViewConst& vc, int x, int ybase, int (&x0)[K4_PPT],
                                        int (&y0)[K4_PPT], float (&ax)[K4_PPT],
                                        float (&ay)[K4_PPT]) {
  const ColGeo cg = col_geo(vc, x);
  const float kdeg = 57.29577951308232f;
#if !WV_K4_GEO2
#pragma unroll
  for (int k = 0; k < K4_PPT; ++k) {
    const float w = 1.0f - ((float)(ybase + K4_NW * k) + 0.5f) * vc.inv_h;
    const float ry = w * vc.tan_v;
    const float wx = fmaf(ry, vc.r[1], cg.cx), wy = fmaf(ry, vc.r[4], cg.cy),
                wz = fmaf(ry, vc.r[7], cg.cz);
    // lon = atan2(x, z); lat = asin(y/|w|) = atan2(y, hypot(x, z))
    const float lon = fast_atan2(wx, wz) * kdeg;
    const float hz = wx * wx + wz * wz;
    // (at the poles hz = 0 and fast_atan2(wy, 0) = +-pi/2)
    const float lat = fast_atan2(wy, sqrt_approx(hz)) * kdeg;
    const float fx = (lon + 180.0f) * vc.sx - 0.5f;
    const float fy = (90.0f - lat) * vc.sy - 0.5f;
    const float flx = floorf(fx), fly = floorf(fy);
    x0[k] = (int)flx;
    y0[k] = (int)fly;
    ax[k] = fx - flx;
    ay[k] = fy - fly;
  }
#else
#pragma unroll
  for (int k = 0; k < K4_PPT; k += 2) {
    const float2 yc = __fadd2_rn(make_float2((float)(ybase + K4_NW * k), (float)(ybase + K4_NW * k + K4_NW)),
                                 f2v(0.5f));
    const float2 w = __ffma2_rn(neg2(yc), f2v(vc.inv_h), f2v(1.0f));
    const float2 ry = __fmul2_rn(w, f2v(vc.tan_v));
    const float2 wx = __ffma2_rn(ry, f2v(vc.r[1]), f2v(cg.cx));
    const float2 wy = __ffma2_rn(ry, f2v(vc.r[4]), f2v(cg.cy));
    const float2 wz = __ffma2_rn(ry, f2v(vc.r[7]), f2v(cg.cz));
    // lon = atan2(x, z); lat = asin(y/|w|) = atan2(y, hypot(x, z))
    const float2 lon = __fmul2_rn(fast_atan2_x2(wx, wz), f2v(kdeg));
    const float2 hz = __ffma2_rn(wx, wx, __fmul2_rn(wz, wz));
    // (at the poles hz = 0 and fast_atan2(wy, 0) = +-pi/2)
    const float2 lat = __fmul2_rn(
        fast_atan2_x2(wy, make_float2(sqrt_approx(hz.x), sqrt_approx(hz.y))), f2v(kdeg));
    const float2 fx = __ffma2_rn(__fadd2_rn(lon, f2v(180.0f)), f2v(vc.sx), f2v(-0.5f));
    const float2 fy = __ffma2_rn(__fadd2_rn(f2v(90.0f), neg2(lat)), f2v(vc.sy), f2v(-0.5f));
    const float2 fl = make_float2(floorf(fx.x), floorf(fx.y));
    const float2 gl = make_float2(floorf(fy.x), floorf(fy.y));
    const float2 fa = __fadd2_rn(fx, neg2(fl)), ga = __fadd2_rn(fy, neg2(gl));
    x0[k] = (int)fl.x;
    x0[k + 1] = (int)fl.y;
    y0[k] = (int)gl.x;
    y0[k + 1] = (int)gl.y;
    ax[k] = fa.x;
    ax[k + 1] = fa.y;
    ay[k] = ga.x;
    ay[k + 1] = ga.y;
  }
#endif
}

// Phase 4 for one view when the CTA-uniform fast path does not apply:
// per-pixel coverage (only when the box test failed; a pixel whose float32
// candidate taps are not all covered takes the reference's float64 taps),
// longitude wrap / pole clamp, partial tiles.  Re-evaluates the pixel
// geometry instead of receiving it, so the caller keeps nothing live across
// the call.
template <int CT>
__device__ __noinline__ void general_view(const ViewConst& vc, const wv_view_args& v,
                                          const wv_view_args& w, const uint32_t* wj, uint8_t* oj,
                                          int P, int rows, int yl, int wx0, bool use_win,
                                          bool covered, int x, int ybase) {
  const int C = CT ? CT : vc.C;
  const int m = vc.m, n = vc.n, out_w = vc.out_w, out_h = vc.out_h;
  const uint32_t K = 0x4B000000u;
  int gx0[K4_PPT], gy0[K4_PPT];
  float gax[K4_PPT], gay[K4_PPT];
  geo_all(vc, x, ybase, gx0, gy0, gax, gay);
  unsigned n_unc = 0;
#pragma unroll
  for (int k = 0; k < K4_PPT; ++k) {
    const int y = ybase + K4_NW * k;
    const bool live = x < out_w && y < out_h;
    bool uncovered = false;
    if (live) {
      int tx0 = gx0[k], ty0 = gy0[k];
      float tax = gax[k], tay = gay[k];
      if (!covered) {
        const uint32_t* F = view_fp(w, vc.wpr0);
        const int wpr0 = vc.wpr0;
        const int cl = tax < kNear ? tx0 - 1 : tx0, ch = tax > 1.0f - kNear ? tx0 + 2 : tx0 + 1;
        const int rl = tay < kNear ? ty0 - 1 : ty0, rh = tay > 1.0f - kNear ? ty0 + 2 : ty0 + 1;
        const int len = ch - cl + 1;
        const uint32_t full = (1u << len) - 1u;
        bool ok = true;
        for (int yy = rl; yy <= rh; ++yy)
          ok = ok && fp_bits(F + (uint32_t)min(max(yy, 0), m - 1) * wpr0, cl, len, n) == full;
        if (!ok) {
          const Taps t = taps_f64(v, x, y);
          tx0 = t.x0;
          ty0 = t.y0;
          tax = t.ax;
          tay = t.ay;
          const uint32_t* r0 = F + (uint32_t)min(max(ty0, 0), m - 1) * wpr0;
          const uint32_t* r1 = F + (uint32_t)min(max(ty0 + 1, 0), m - 1) * wpr0;
          uncovered = (fp_bits(r0, tx0, 2, n) & fp_bits(r1, tx0, 2, n)) != 3u;
        }
      }
      uint32_t w00, w01, w10, w11;
      if (use_win) {
        WV_ASSERT(ty0 - yl >= 0 && ty0 + 1 - yl < rows && tx0 - wx0 >= 0 && tx0 + 1 - wx0 < P);
        const uint32_t* p = wj + (ty0 - yl) * P + (tx0 - wx0);
        w00 = p[0];
        w01 = p[1];
        w10 = p[P];
        w11 = p[P + 1];
      } else {
        // longitude wrap / pole clamp (projection.py:146-149)
        const int xa = wrapx(tx0, n), xb = wrapx(tx0 + 1, n);
        const int ya = min(max(ty0, 0), m - 1), yb = min(max(ty0 + 1, 0), m - 1);
        const uint32_t o00 = (uint32_t)ya * n + xa, o01 = (uint32_t)ya * n + xb;
        const uint32_t o10 = (uint32_t)yb * n + xa, o11 = (uint32_t)yb * n + xb;
        w00 = w01 = w10 = w11 = 0u;
        const uint8_t* pc = view_img(w);
        for (int c = 0; c < C; ++c, pc += vc.plane) {
          w00 |= (uint32_t)__ldg(pc + o00) << (8 * c);
          w01 |= (uint32_t)__ldg(pc + o01) << (8 * c);
          w10 |= (uint32_t)__ldg(pc + o10) << (8 * c);
          w11 |= (uint32_t)__ldg(pc + o11) << (8 * c);
        }
      }
      uint8_t* o = oj + (threadIdx.y + K4_NW * k) * OST_PITCH + threadIdx.x * C;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        if (c < C) {
          // 2^23 + byte c of each tap (selector: byte c of the tap, zeros, 0x4B)
          const uint32_t sel = 0x3004u + c;
          const float b00 = __uint_as_float(__byte_perm(K, w00, sel));
          const float b01 = __uint_as_float(__byte_perm(K, w01, sel));
          const float b10 = __uint_as_float(__byte_perm(K, w10, sel));
          const float b11 = __uint_as_float(__byte_perm(K, w11, sel));
          o[c] = (uint8_t)blend(b00, b01, b10, b11, tax, tay);
        }
      }
    }
    n_unc += __popc(__ballot_sync(0xFFFFFFFFu, uncovered));
  }
  if (threadIdx.x == 0 && n_unc) atomicAdd(w.d_uncovered, n_unc);
}

// Phases 2-5 for NV views sharing the geometry (NV = 2: a stereo pair staged
// together), CT channels (CT = 0: any C in 1..4, read at run time).
template <int CT, int NV>
__device__ __forceinline__ void finish(const ViewConst& vc, const wv_view_args& v,
                                       const wv_view_args* const (&vp)[NV], uint32_t* win, uint8_t* ost,
                                       uint32_t* s_ok, const int (&off)[K4_PPT],
                                       const float (&ax)[K4_PPT],
                                       const float (&ay)[K4_PPT], int x, int ybase, int xl,
                                       int xh, int yl, int yh, int wx0, int ww, bool box_ok,
                                       bool use_win, int tid) {
  const int C = CT ? CT : vc.C;
  const int n = vc.n, out_w = vc.out_w, out_h = vc.out_h;
  const int rows = yh - yl + 1;
  const int P = 4 * ww;           // window pitch (words)
  const int VW = rows * P;        // words per view in the window
  // (2) footprint test of the box and (3) staging of the box, channels
  // interleaved (byte c of word = channel c).  Thread t owns word t % nwords
  // of rows t / nwords + k * (256 / nwords): one division per CTA, not per word.
  uint32_t okb = box_ok ? (1u << NV) - 1u : 0u;   // bit j: view j's box covered so far
  if (box_ok) {
    const int w0 = xl >> 5, nw = (xh >> 5) - w0 + 1;
    const float inv = rcp_approx((float)nw);
    const SmallDiv dq = small_div(tid, nw, inv);
    const int q = dq.r, rstep = small_div(K4_NTH, nw, inv).q, wd = w0 + q;
    const uint32_t mk = ~range_bits(xl, xh + 1, wd);
    const uint32_t o = (uint32_t)yl * vc.wpr0 + wd;
    if (tid < rstep * nw)
      for (int r = dq.q; r < rows; r += rstep) {
#pragma unroll
        for (int j = 0; j < NV; ++j)
          if ((__ldg(view_fp(*vp[j], vc.wpr0) + o + (uint32_t)r * vc.wpr0) | mk) != 0xFFFFFFFFu) okb &= ~(1u << j);
      }
  }
  if (use_win) {
    const uint32_t plane = vc.plane;
    const float inv = rcp_approx((float)ww);
    const SmallDiv dq = small_div(tid, ww, inv);
    const int q = dq.r, rstep = small_div(K4_NTH, ww, inv).q;
    const uint32_t so = (uint32_t)yl * n + wx0 + 4 * q;
    if (tid < rstep * ww) {
      for (int r = dq.q; r < rows; r += rstep) {
#pragma unroll
        for (int j = 0; j < NV; ++j) {
          const uint8_t* src = view_img(*vp[j]) + so + (uint32_t)r * n;
          const uint32_t R = __ldg(reinterpret_cast<const uint32_t*>(src));
          const uint32_t G = C > 1 ? __ldg(reinterpret_cast<const uint32_t*>(src + plane)) : 0u;
          const uint32_t B = C > 2 ? __ldg(reinterpret_cast<const uint32_t*>(src + 2 * plane)) : 0u;
          const uint32_t A = C > 3 ? __ldg(reinterpret_cast<const uint32_t*>(src + 3 * plane)) : 0u;
          const uint32_t rg_lo = __byte_perm(R, G, 0x5140), rg_hi = __byte_perm(R, G, 0x7362);
          const uint32_t ba_lo = __byte_perm(B, A, 0x5140), ba_hi = __byte_perm(B, A, 0x7362);
          WV_ASSERT(j * VW + r * P + 4 * q + 3 < WIN_WORDS);
          *reinterpret_cast<uint4*>(win + j * VW + r * P + 4 * q) =
              make_uint4(__byte_perm(rg_lo, ba_lo, 0x5410), __byte_perm(rg_lo, ba_lo, 0x7632),
                         __byte_perm(rg_hi, ba_hi, 0x5410), __byte_perm(rg_hi, ba_hi, 0x7632));
        }
      }
    }
  }
  {
    const uint32_t wb = __reduce_and_sync(0xFFFFFFFFu, okb);
    if (threadIdx.x == 0) s_ok[threadIdx.y] = wb;
  }
  __syncthreads();
  uint32_t cov;
  {
    const uint4 a = *reinterpret_cast<const uint4*>(s_ok);
    cov = a.x & a.y & a.z & a.w;
    if (K4_NW > 4) {
      const uint4 b = *reinterpret_cast<const uint4*>(s_ok + 4);
      cov &= b.x & b.y & b.z & b.w;
    }
  }
  const uint32_t K = 0x4B000000u;
  const int tx0 = x - (int)threadIdx.x, ty0 = ybase - (int)threadIdx.y;   // tile origin
  const bool full_tile = tx0 + K4_TX <= out_w && ty0 + K4_TY <= out_h;
#pragma unroll
  for (int j = 0; j < NV; ++j) {
    const uint32_t* wj = win + j * VW;
    uint8_t* oj = ost + j * OST_VIEW;
    const bool covered = (cov >> j) & 1u;
    // (4a) common case, uniform over the CTA: whole tile inside the output,
    // box covered by the footprint and staged -- taps straight from the window
    if (covered && use_win && full_tile) {
      uint32_t pw[4];   // CT == 3: taps of the previous (even) pixel
#pragma unroll
      for (int k = 0; k < K4_PPT; ++k) {
        WV_ASSERT(off[k] >= 0 && off[k] + P + 1 < rows * P);
        const uint32_t* p = wj + off[k];
        const uint32_t w00 = p[0], w01 = p[1], w10 = p[P], w11 = p[P + 1];
        uint8_t* o = oj + (threadIdx.y + K4_NW * k) * OST_PITCH + threadIdx.x * C;
        if (CT == 3) {
          // channels 0 and 1 as one paired-FP32 stream (same per-lane rounding
          // as blend()); channel 2 paired with channel 2 of the thread's next
          // pixel (k odd: done with pixel k-1)
          const uint32_t rg = blend2(w00, w01, w10, w11, ax[k], ay[k]);
          o[0] = (uint8_t)rg;
          o[1] = (uint8_t)(rg >> 8);
          if (k & 1) {
            const uint32_t bb = blend_v2(
                make_float2(biased(pw[0], 2), biased(w00, 2)), make_float2(biased(pw[1], 2), biased(w01, 2)),
                make_float2(biased(pw[2], 2), biased(w10, 2)),
                make_float2(biased(pw[3], 2), biased(w11, 2)), make_float2(ax[k - 1], ax[k]),
                make_float2(ay[k - 1], ay[k]));
            o[2 - K4_NW * OST_PITCH] = (uint8_t)bb;
            o[2] = (uint8_t)(bb >> 8);
          } else {
            pw[0] = w00;
            pw[1] = w01;
            pw[2] = w10;
            pw[3] = w11;
          }
        } else {
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            if (c < C) {
              const uint32_t sel = 0x3004u + c;
              o[c] = (uint8_t)blend(__uint_as_float(__byte_perm(K, w00, sel)),
                                    __uint_as_float(__byte_perm(K, w01, sel)),
                                    __uint_as_float(__byte_perm(K, w10, sel)),
                                    __uint_as_float(__byte_perm(K, w11, sel)), ax[k], ay[k]);
            }
          }
        }
      }
    } else {
      // (4b) general case, out of line (its registers stay out of the fast path)
      general_view<CT>(vc, v, *vp[j], wj, oj, P, rows, yl, wx0, use_win, covered, x, ybase);
    }
  }
  __syncthreads();
  // (5) tile rows -> (out_h, out_w, C) with 16-byte stores where aligned
  const int nx = min(K4_TX, out_w - tx0);
  const int ny = min(K4_TY, out_h - ty0);
  const int rowb = nx * C;
  const uint64_t gpitch = (uint64_t)out_w * C;
  const uint64_t gofs = ((uint64_t)ty0 * out_w + tx0) * C;
#pragma unroll
  for (int j = 0; j < NV; ++j) {
    uint8_t* gbase = vp[j]->d_out + gofs;
    const uint8_t* oj = ost + j * OST_VIEW;
    if (((reinterpret_cast<uintptr_t>(gbase) | gpitch | rowb) & 15) == 0) {
      const int nv = rowb >> 4;
      for (int idx = tid; idx < ny * nv; idx += K4_NTH) {
        // nv = 6 (RGB, full tile): constant divisor, no division instructions
        const int r = nv == 6 ? idx / 6 : idx / nv, q = idx - r * nv;
        __stcs(reinterpret_cast<uint4*>(gbase + r * gpitch) + q,
               *reinterpret_cast<const uint4*>(oj + r * OST_PITCH + 16 * q));
      }
    } else {
      for (int idx = tid; idx < ny * rowb; idx += K4_NTH) {
        const int r = idx / rowb, b = idx - (idx / rowb) * rowb;
        gbase[r * gpitch + b] = oj[r * OST_PITCH + b];
      }
    }
  }
}

template <int NV>
__device__ __forceinline__ void finish_c(const ViewConst& vc, const wv_view_args& v,
                                         const wv_view_args* const (&vp)[NV], uint32_t* win, uint8_t* ost,
                                         uint32_t* s_ok, const int (&off)[K4_PPT],
                                         const float (&ax)[K4_PPT],
                                         const float (&ay)[K4_PPT], int x, int ybase, int xl,
                                         int xh, int yl, int yh, int wx0, int ww, bool box_ok,
                                         bool use_win, int tid) {
  if (vc.C == 3)
    finish<3, NV>(vc, v, vp, win, ost, s_ok, off, ax, ay, x, ybase, xl, xh, yl, yh, wx0, ww,
                  box_ok, use_win, tid);
  else
    finish<0, NV>(vc, v, vp, win, ost, s_ok, off, ax, ay, x, ybase, xl, xh, yl, yh, wx0, ww,
                  box_ok, use_win, tid);
}

// shared_n == 0: CTA (x, y, z) renders view z.  shared_n > 0: the views
// share pose, FOV, region size and output size (a stereo pair), so the CTA
// evaluates the geometry once and renders all shared_n views from it.
template <bool DEV>
__global__ void __launch_bounds__(K4_NTH, K4_MIN_BLOCKS) k_perspective(const __grid_constant__ Views views,
                                                     const wv_view_args* __restrict__ d_views,
                                                     int shared_n) {
  pdl_sync();
  __shared__ ViewConst vc;
  // window + staged output tiles in dynamic shared memory (K4_SMEM bytes)
  extern __shared__ __align__(16) uint32_t k4_dyn[];
  uint32_t* win = k4_dyn;
  uint8_t* ost = reinterpret_cast<uint8_t*>(k4_dyn + WIN_WORDS);
  __shared__ __align__(16) uint32_t s_ok[8];   // one word per warp (<= 8 warps)
  __shared__ int s_box[2][4];   // candidate-tap box: xmin, xmax, ymin, ymax
  const int vz = shared_n > 0 ? 0 : blockIdx.z;
  const wv_view_args& v = DEV ? d_views[vz] : views.v[vz];
  const int tid = threadIdx.y * 32 + threadIdx.x;
  if (tid == 0) {
    for (int i = 0; i < 9; ++i) vc.r[i] = (float)v.rot[i];
    vc.tan_h = (float)v.tan_h;
    vc.tan_v = (float)v.tan_v;
    vc.out_w = v.out_w;
    vc.out_h = v.out_h;
    vc.inv_w = 2.0f / (float)v.out_w;
    vc.inv_h = 2.0f / (float)v.out_h;
    vc.m = v.rows;
    vc.n = v.width;
    vc.sx = (float)v.width * (1.0f / 360.0f);
    vc.sy = (float)v.rows * (1.0f / 180.0f);
    vc.C = v.channels;
    vc.wpr0 = (v.width + 31) >> 5;
    vc.plane = (uint32_t)v.canvas_h * (uint32_t)v.width;
    s_box[0][0] = s_box[0][2] = 0x7FFFFFFF;
    s_box[0][1] = s_box[0][3] = -0x7FFFFFFF;
  }
  __syncthreads();
  const int out_w = vc.out_w, out_h = vc.out_h;
  const int m = vc.m, n = vc.n;
  const int ntx = (out_w + K4_TX - 1) / K4_TX, ntiles = ntx * ((out_h + K4_TY - 1) / K4_TY);
  // persistent CTAs: the view constants are set up once, tiles round-robin;
  // the candidate-tap box alternates between two shared slots, so the next
  // tile's slot is reset while the current one is in use (no extra barrier)
  int it = 0;
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
    int* box = s_box[it & 1];
    const int tby = tile / ntx, tbx = tile - tby * ntx;
    const int x = tbx * K4_TX + threadIdx.x;
    const int ybase = tby * K4_TY + threadIdx.y;

    // (1) geometry
    int x0[K4_PPT], y0[K4_PPT];
    float ax[K4_PPT], ay[K4_PPT];
    int bx0 = 0x7FFFFFFF, bx1 = -0x7FFFFFFF, by0 = 0x7FFFFFFF, by1 = -0x7FFFFFFF;
    geo_all(vc, x, ybase, x0, y0, ax, ay);
#pragma unroll
    for (int k = 0; k < K4_PPT; ++k) {
      const int y = ybase + K4_NW * k;
      if (x < out_w && y < out_h) {
        bx0 = min(bx0, x0[k] - 1);
        bx1 = max(bx1, x0[k] + 2);
        by0 = min(by0, y0[k] - 1);
        by1 = max(by1, y0[k] + 2);
      }
    }
    // candidate-tap box of the tile (both tap choices near integer boundaries)
    bx0 = __reduce_min_sync(0xFFFFFFFFu, bx0);
    bx1 = __reduce_max_sync(0xFFFFFFFFu, bx1);
    by0 = __reduce_min_sync(0xFFFFFFFFu, by0);
    by1 = __reduce_max_sync(0xFFFFFFFFu, by1);
    if (threadIdx.x == 0) {
      atomicMin(&box[0], bx0);
      atomicMax(&box[1], bx1);
      atomicMin(&box[2], by0);
      atomicMax(&box[3], by1);
    }
    if (tid == 0) {   // the other slot: last read before the previous tile's barriers
      int* nb = s_box[(it + 1) & 1];
      nb[0] = nb[2] = 0x7FFFFFFF;
      nb[1] = nb[3] = -0x7FFFFFFF;
    }
    __syncthreads();
    const int xl = box[0], xh = box[1], yl = box[2], yh = box[3];
    const bool inside = xl >= 0 && xh < n && yl >= 0 && yh < m && xl <= xh;
    const int wx0 = xl & ~3;
    const int ww = ((xh | 3) - wx0 + 1) >> 2;   // 4-pixel words per window row
    const int vwords = inside ? (yh - yl + 1) * 4 * ww : 0x7FFFFFFF;
    const bool box_ok = inside && (xh - xl) < BOX_MAX_W;
    // window offset of each pixel's (x0, y0) tap (used only when staged; the
    // general path re-evaluates its geometry)
    int off[K4_PPT];
#pragma unroll
    for (int k = 0; k < K4_PPT; ++k) off[k] = (y0[k] - yl) * (4 * ww) + (x0[k] - wx0);
    const bool stage = inside && (n & 3) == 0;
    const int nv = shared_n > 0 ? shared_n : 1;
    auto vargs = [&](int vi) -> const wv_view_args* {
      return shared_n > 0 ? (DEV ? d_views + vi : &views.v[vi]) : &v;
    };
    for (int vi = 0; vi < nv;) {
      if (vi + 1 < nv && stage && 2 * vwords <= WIN_WORDS) {
        const wv_view_args* const vp[2] = {vargs(vi), vargs(vi + 1)};
        finish_c<2>(vc, v, vp, win, ost, s_ok, off, ax, ay, x, ybase, xl, xh, yl, yh, wx0, ww,
                    box_ok, true, tid);
        vi += 2;
      } else {
        const wv_view_args* const vp[1] = {vargs(vi)};
        finish_c<1>(vc, v, vp, win, ost, s_ok, off, ax, ay, x, ybase, xl, xh, yl, yh, wx0, ww,
                    box_ok, stage && vwords <= WIN_WORDS, tid);
        vi += 1;
      }
    }
  }
}

}  // namespace

// resident CTAs for the persistent K4 grid (at most one per tile)
template <class K>
int persistent_grid(K kernel, int ntiles) {
  int dev = 0, sms = 148, occ = K4_MIN_BLOCKS;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, K4_SMEM);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, K4_NTH, K4_SMEM);
  return max(1, min(ntiles, sms * max(occ, 1)));
}

int launch_perspective(const wv_view_args* views, int n, cudaStream_t s) {
  if (n < 1 || n > kMaxViews) return WV_ERR_ARG;
  Views pv{};
  int mw = 0, mh = 0;
  for (int i = 0; i < n; ++i) {
    const wv_view_args& v = views[i];
    if (!v.d_canvas || !v.d_footprint || !v.d_out || !v.d_uncovered || v.out_w < 1 ||
        v.out_h < 1 || v.channels < 1 || v.width < 1 || v.rows < 1 ||
        v.canvas_h < v.row0 + v.rows)
      return WV_ERR_ARG;
    pv.v[i] = v;
    mw = max(mw, v.out_w);
    mh = max(mh, v.out_h);
  }
  // one geometry evaluation for views that differ only in their canvas rows
  bool shared = n > 1;
  for (int i = 1; i < n && shared; ++i) {
    const wv_view_args &a = views[0], &b = views[i];
    shared = a.out_w == b.out_w && a.out_h == b.out_h && a.width == b.width &&
             a.rows == b.rows && a.channels == b.channels && a.canvas_h == b.canvas_h &&
             a.tan_h == b.tan_h && a.tan_v == b.tan_v;
    for (int k = 0; k < 9 && shared; ++k) shared = a.rot[k] == b.rot[k];
  }
  dim3 block(32, K4_NW);
  dim3 grid(persistent_grid(k_perspective<false>, cdiv(mw, K4_TX) * cdiv(mh, K4_TY)), 1,
            shared ? 1 : n);
  WV_CUDA(launch_k(k_perspective<false>, dim3(grid), dim3(block), (size_t)K4_SMEM, s, pv, nullptr,
                   shared ? n : 0));
  WV_CUDA(cudaGetLastError());
  return WV_OK;
}

int launch_perspective_dev(const wv_view_args* d_views, int n, int max_w, int max_h,
                           int shared_geometry, cudaStream_t s) {
  if (!d_views || n < 1 || n > kMaxViews || max_w < 1 || max_h < 1) return WV_ERR_ARG;
  Views none{};
  const bool shared = shared_geometry && n > 1;
  dim3 block(32, K4_NW);
  dim3 grid(persistent_grid(k_perspective<true>, cdiv(max_w, K4_TX) * cdiv(max_h, K4_TY)), 1,
            shared ? 1 : n);
  WV_CUDA(launch_k(k_perspective<true>, dim3(grid), dim3(block), (size_t)K4_SMEM, s, none, d_views,
                   shared ? n : 0));
  WV_CUDA(cudaGetLastError());
  return WV_OK;
}

}  // namespace wv
