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
  int L, H, W, C, bs, nbx, n, t, rs, float_mode;
  const unsigned long long* ends;   // (n, NB)
  const uint8_t* recs;              // records region
  const float* extrema;             // (n, C, 4)
  const uint32_t* D[WV_MAX_LEVELS + 1];
  int dwpr[WV_MAX_LEVELS + 1];
  const uint32_t* list;
  const uint32_t* count;
  int NB;
  float* plane;
  wv_frame_result* res;
};

// inclusion bit of plane position (y, x) (LevelMaskSet.inclusion_grid)
__device__ __forceinline__ bool included(const TemporalArgs& a, int y, int x) {
  for (int k = 1; k <= a.L; ++k) {
    int bh = a.H >> k, bw = a.W >> k;
    if (y >= bh || x >= bw) {
      int r = y >= bh ? y - bh : y;
      int c = x >= bw ? x - bw : x;
      return (a.D[k][(uint64_t)r * a.dwpr[k] + (c >> 5)] >> (c & 31)) & 1u;
    }
  }
  return true;  // approximation band: always included
}

// temporal Mallat index ti contributes to display time t with sign
// (+1/-1) or not at all (0) (encoding.py:187-195, decoding.py:72-80)
__device__ __forceinline__ int tweight(int ti, int t, int n) {
  if (ti == 0) return 1;
  int big = 31 - __clz(n);
  int lvl = big - (31 - __clz(ti));
  if ((t >> lvl) != ti - (1 << (big - lvl))) return 0;
  return ((t >> (lvl - 1)) & 1) ? -1 : 1;
}

__global__ void __launch_bounds__(256) k_temporal(TemporalArgs a) {
  extern __shared__ float acc[];        // C x bs*bs
  const int npos = a.bs * a.bs;
  const uint32_t count = *a.count;
  const int tid = threadIdx.x;
  const int ah = a.H >> a.L, aw = a.W >> a.L;
  uint32_t err = 0;
  for (uint32_t item = blockIdx.x; item < count; item += gridDim.x) {
    const uint32_t e = a.list[item];
    const int b = (int)(e & ~ZERO_FLAG);
    const int y0 = (b / a.nbx) * a.bs, x0 = (b % a.nbx) * a.bs;
    const bool zero_only = (e & ZERO_FLAG) != 0;
    if (!zero_only) {
      for (int i = tid; i < a.C * npos; i += blockDim.x) acc[i] = 0.0f;
      __syncthreads();
      for (int ti = 0; ti < a.n; ++ti) {
        const int wgt = tweight(ti, a.t, a.n);
        const uint64_t fi = (uint64_t)ti * a.NB + b;
        const unsigned long long s = fi ? a.ends[fi - 1] : 0ull;
        const unsigned long long en = a.ends[fi];
        if (en < s || (en - s) % a.rs) continue;  // flagged by K1
        const int cnt = (int)min((en - s) / a.rs, (unsigned long long)npos);
        const uint8_t* base = a.recs + s;
        for (int r = tid; r < cnt; r += blockDim.x) {
          const uint8_t* rp = base + (uint64_t)r * a.rs;
          const int off = (int)rp[0] | ((int)rp[1] << 8);
          if (off >= npos) { err |= WV_DERR_OFFSET; continue; }
          if (!wgt) continue;
          const int yy = y0 + off / a.bs, xx = x0 + off % a.bs;
          const bool appr = yy < ah && xx < aw;
          for (int c = 0; c < a.C; ++c) {
            float v;
            if (a.float_mode) {
              uint32_t u = (uint32_t)rp[2 + 4 * c] | ((uint32_t)rp[3 + 4 * c] << 8) |
                           ((uint32_t)rp[4 + 4 * c] << 16) | ((uint32_t)rp[5 + 4 * c] << 24);
              v = __uint_as_float(u);
            } else {
              const float* ex = a.extrema + ((uint64_t)ti * a.C + c) * 4 + (appr ? 0 : 2);
              const float lo = ex[0], hi = ex[1];
              v = __fadd_rn(lo, __fmul_rn(__fdiv_rn((float)rp[2 + c], 255.0f), __fsub_rn(hi, lo)));
            }
            float* cell = acc + c * npos + off;
            *cell = __fadd_rn(*cell, wgt > 0 ? v : -v);
          }
        }
        if (wgt) __syncthreads();
      }
    }
    // write the block: 4 consecutive positions per thread-step
    for (int i = tid * 4; i < npos; i += blockDim.x * 4) {
      const int yy = y0 + i / a.bs, xx = x0 + i % a.bs;
      float4 m;
      if (zero_only) {
        m = make_float4(0.f, 0.f, 0.f, 0.f);
      } else {
        m.x = included(a, yy, xx) ? 1.0f : 0.0f;
        m.y = included(a, yy, xx + 1) ? 1.0f : 0.0f;
        m.z = included(a, yy, xx + 2) ? 1.0f : 0.0f;
        m.w = included(a, yy, xx + 3) ? 1.0f : 0.0f;
      }
      for (int c = 0; c < a.C; ++c) {
        float4 v;
        if (zero_only) {
          v = m;
        } else {
          const float* p = acc + c * npos + i;
          v = make_float4(__fmul_rn(p[0], m.x), __fmul_rn(p[1], m.y), __fmul_rn(p[2], m.z),
                          __fmul_rn(p[3], m.w));
        }
        float* dst = a.plane + ((uint64_t)c * a.H + yy) * a.W + xx;
        *reinterpret_cast<float4*>(dst) = v;
      }
    }
    __syncthreads();
  }
  for (int o = 16; o; o >>= 1) err |= __shfl_xor_sync(0xFFFFFFFFu, err, o);
  if ((tid & 31) == 0 && err) atomicOr(&a.res->error, err);
}

// block_size < 4: scalar writer (tiny test geometries only)


}  // namespace

int launch_temporal(const Layout& lo, const wv_geometry* g, const wv_frame_args* a, uint8_t* ws,
                    cudaStream_t s) {
  if (lo.bs < 4) return WV_ERR_UNSUPPORTED;
  if (a->t < 0 || a->t >= lo.n) return WV_ERR_ARG;
  TemporalArgs t{};
  t.L = lo.L; t.H = lo.H; t.W = lo.W; t.C = lo.C; t.bs = lo.bs; t.nbx = lo.nbx; t.n = lo.n;
  t.t = a->t; t.float_mode = g->float_mode; t.rs = 2 + lo.C * (g->float_mode ? 4 : 1);
  t.NB = lo.NB;
  t.ends = (const unsigned long long*)a->d_payload;
  t.recs = (const uint8_t*)a->d_payload + (uint64_t)lo.n * lo.NB * 8;
  t.extrema = a->d_extrema;
  const bool fov = a->mode == WV_MODE_FOVEATED;
  for (int k = 1; k <= lo.L; ++k) {
    t.D[k] = (const uint32_t*)(ws + lo.stack[k] + (fov ? (uint64_t)k * lo.stack_stride[k] : 0));
    t.dwpr[k] = lo.wpr_[k];
  }
  t.list = (const uint32_t*)(ws + lo.blist);
  t.count = (const uint32_t*)(ws + lo.counters) + CNT_BLOCKS;
  t.plane = (float*)(ws + lo.plane);
  t.res = a->d_result;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  size_t smem = (size_t)lo.C * lo.bs * lo.bs * 4;
  if (smem > 48 * 1024)
    WV_CUDA(cudaFuncSetAttribute(k_temporal, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int grid = min(lo.NB, sms * 8);
  k_temporal<<<grid, 256, smem, s>>>(t);
  WV_CUDA(cudaGetLastError());
  return WV_OK;
}

}  // namespace wv
