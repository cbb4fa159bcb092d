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
__device__ __forceinline__ float fast_atan2(float y, float x) {
  const float ax = fabsf(x), ay = fabsf(y);
  const float mx = fmaxf(ax, ay), mn = fminf(ax, ay);
  const float a = __fdividef(mn, mx);
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
#ifndef K4_MIN_BLOCKS
#define K4_MIN_BLOCKS 8
#endif

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
  const uint32_t* F;
  const uint8_t* img;
  uint8_t* out;
  uint32_t* uncovered;
  int xmin, xmax, ymin, ymax;   // candidate-tap bounding box of the CTA
  int covered;                  // that whole box lies inside the footprint
};

// This translation unit is compiled with FMA contraction enabled: the float32
// geometry is approximate by design, and the bilinear blend's lerps may round
// differently from the reference by < 1e-4 LSB; both stay inside the +-1 LSB
// bar.  The float64 fallback uses explicit __d*_rn intrinsics.
template <bool DEV>
__global__ void __launch_bounds__(256, K4_MIN_BLOCKS) k_perspective(const __grid_constant__ Views views,
                                                     const wv_view_args* __restrict__ d_views) {
  __shared__ ViewConst vc;
  const wv_view_args& v = DEV ? d_views[blockIdx.z] : views.v[blockIdx.z];
  if (threadIdx.x == 0 && threadIdx.y == 0) {
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
    vc.F = v.d_footprint + (uint64_t)v.row0 * vc.wpr0;
    vc.img = v.d_canvas + (uint64_t)v.row0 * v.width;
    vc.out = v.d_out;
    vc.uncovered = v.d_uncovered;
    vc.xmin = vc.ymin = 0x7FFFFFFF;
    vc.xmax = vc.ymax = -0x7FFFFFFF;
  }
  __syncthreads();
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int y = blockIdx.y * blockDim.y + threadIdx.y;
  const bool live = x < vc.out_w && y < vc.out_h;
  bool uncovered = false;
  const int m = vc.m, n = vc.n, wpr0 = vc.wpr0;
  int x0 = 0, y0 = 0;
  float ax = 0.f, ay = 0.f;
  if (live) {
    const float u = ((float)x + 0.5f) * vc.inv_w - 1.0f;
    const float w = 1.0f - ((float)y + 0.5f) * vc.inv_h;
    const float rx = u * vc.tan_h, ry = w * vc.tan_v;
    const float wx = rx * vc.r[0] + ry * vc.r[1] + vc.r[2];
    const float wy = rx * vc.r[3] + ry * vc.r[4] + vc.r[5];
    const float wz = rx * vc.r[6] + ry * vc.r[7] + vc.r[8];
    // lon = atan2(x, z); lat = asin(y/|w|) = atan2(y, hypot(x, z))
    const float lon = fast_atan2(wx, wz) * 57.29577951308232f;
    const float hz = wx * wx + wz * wz;
    const float lat = (hz > 0.0f ? fast_atan2(wy, hz * rsqrtf(hz)) : copysignf(1.5707963f, wy)) *
                      57.29577951308232f;
    const float fx = (lon + 180.0f) * vc.sx - 0.5f;
    const float fy = (90.0f - lat) * vc.sy - 0.5f;
    const float flx = floorf(fx), fly = floorf(fy);
    x0 = (int)flx;
    y0 = (int)fly;
    ax = fx - flx;
    ay = fy - fly;
  }
  {
    // candidate-tap box of the CTA (both tap choices near integer boundaries):
    // warp reductions, one shared atomic per warp, one warp tests its rows
    const int bx0 = __reduce_min_sync(0xFFFFFFFFu, live ? x0 - 1 : 0x7FFFFFFF);
    const int bx1 = __reduce_max_sync(0xFFFFFFFFu, live ? x0 + 2 : -0x7FFFFFFF);
    const int by0 = __reduce_min_sync(0xFFFFFFFFu, live ? y0 - 1 : 0x7FFFFFFF);
    const int by1 = __reduce_max_sync(0xFFFFFFFFu, live ? y0 + 2 : -0x7FFFFFFF);
    if ((threadIdx.x & 31) == 0) {
      atomicMin(&vc.xmin, bx0);
      atomicMax(&vc.xmax, bx1);
      atomicMin(&vc.ymin, by0);
      atomicMax(&vc.ymax, by1);
    }
  }
  __syncthreads();
  const int tid = threadIdx.y * blockDim.x + threadIdx.x;
  if (tid < 32) {
    const int xl = vc.xmin, xh = vc.xmax, yl = vc.ymin, yh = vc.ymax;
    bool ok = xl >= 0 && xh < n && yl >= 0 && yh < m && xl <= xh && (xh - xl) < 96;
    for (int yy = yl + tid; ok && yy <= yh; yy += 32) {
      const uint32_t* row = vc.F + (uint32_t)yy * wpr0;
      for (int wd = xl >> 5; ok && wd <= (xh >> 5); ++wd)
        ok = (__ldg(row + wd) | ~range_bits(xl, xh + 1, wd)) == 0xFFFFFFFFu;
    }
    const bool all = __all_sync(0xFFFFFFFFu, ok);
    if (tid == 0) vc.covered = all;
  }
  __syncthreads();
  if (live) {
    if (!vc.covered) {
      const uint32_t* F = vc.F;
      const int xl = ax < kNear ? x0 - 1 : x0, xh = ax > 1.0f - kNear ? x0 + 2 : x0 + 1;
      const int yl = ay < kNear ? y0 - 1 : y0, yh = ay > 1.0f - kNear ? y0 + 2 : y0 + 1;
      const int len = xh - xl + 1;
      const uint32_t full = (1u << len) - 1u;
      bool ok = true;
      for (int yy = yl; yy <= yh; ++yy)
        ok = ok && fp_bits(F + (uint32_t)min(max(yy, 0), m - 1) * wpr0, xl, len, n) == full;
      if (!ok) {
        const Taps t = taps_f64(v, x, y);
        x0 = t.x0;
        y0 = t.y0;
        ax = t.ax;
        ay = t.ay;
        const uint32_t* r0 = F + (uint32_t)min(max(y0, 0), m - 1) * wpr0;
        const uint32_t* r1 = F + (uint32_t)min(max(y0 + 1, 0), m - 1) * wpr0;
        uncovered = (fp_bits(r0, x0, 2, n) & fp_bits(r1, x0, 2, n)) != 3u;
      }
    }
    const int C = vc.C;
    uint8_t* out = vc.out + ((uint32_t)y * vc.out_w + x) * C;
    // u8 <-> f32 without the conversion pipe: 2^23 + b has b in its mantissa
    auto u2f = [](uint32_t b) { return __uint_as_float(0x4B000000u | b) - 8388608.0f; };
    auto f2u = [](float v) {   // clip(rint(v)), round-half-even like np.rint
      return __float_as_uint(fminf(fmaxf(v, 0.0f), 255.0f) + 8388608.0f) & 0xFFu;
    };
    if (x0 >= 0 && x0 + 1 < n && y0 >= 0 && y0 + 1 < m) {
      // interior taps: (y0, x0), (y0, x0+1), (y0+1, x0), (y0+1, x0+1)
      const uint8_t* p0 = vc.img + (uint32_t)y0 * n + x0;
      const uint8_t* p1 = p0 + n;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        if (c < C) {
          const float p00 = u2f(__ldg(p0)), p01 = u2f(__ldg(p0 + 1));
          const float p10 = u2f(__ldg(p1)), p11 = u2f(__ldg(p1 + 1));
          const float top = fmaf(ax, p01 - p00, p00);
          const float bot = fmaf(ax, p11 - p10, p10);
          __stcs(out + c, (unsigned char)f2u(fmaf(ay, bot - top, top)));
          p0 += vc.plane;
          p1 += vc.plane;
        }
      }
    } else {
      // longitude wrap / pole clamp (projection.py:146-149)
      const int xa = wrapx(x0, n), xb = wrapx(x0 + 1, n);
      const int ya = min(max(y0, 0), m - 1), yb = min(max(y0 + 1, 0), m - 1);
      const uint32_t o00 = (uint32_t)ya * n + xa, o01 = (uint32_t)ya * n + xb;
      const uint32_t o10 = (uint32_t)yb * n + xa, o11 = (uint32_t)yb * n + xb;
      const uint8_t* pc = vc.img;
      for (int c = 0; c < C; ++c, pc += vc.plane) {
        const float p00 = u2f(__ldg(pc + o00)), p01 = u2f(__ldg(pc + o01));
        const float p10 = u2f(__ldg(pc + o10)), p11 = u2f(__ldg(pc + o11));
        const float top = fmaf(ax, p01 - p00, p00);
        const float bot = fmaf(ax, p11 - p10, p10);
        __stcs(out + c, (unsigned char)f2u(fmaf(ay, bot - top, top)));
      }
    }
  }
  const unsigned cnt = __popc(__ballot_sync(0xFFFFFFFFu, uncovered));
  if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(vc.uncovered, cnt);
}

}  // namespace

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
  dim3 block(32, 8);
  dim3 grid(cdiv(mw, 32), cdiv(mh, 8), n);
  k_perspective<false><<<grid, block, 0, s>>>(pv, nullptr);
  WV_CUDA(cudaGetLastError());
  return WV_OK;
}

int launch_perspective_dev(const wv_view_args* d_views, int n, int max_w, int max_h,
                           int shared_geometry, cudaStream_t s) {
  // shared_geometry is a hint; evaluating the geometry once per stereo pair
  // measured slower than one thread per (pixel, view) (latency-bound gathers)
  (void)shared_geometry;
  if (!d_views || n < 1 || n > kMaxViews || max_w < 1 || max_h < 1) return WV_ERR_ARG;
  Views none{};
  dim3 block(32, 8);
  dim3 grid(cdiv(max_w, 32), cdiv(max_h, 8), n);
  k_perspective<true><<<grid, block, 0, s>>>(none, d_views);
  WV_CUDA(cudaGetLastError());
  return WV_OK;
}

}  // namespace wv
