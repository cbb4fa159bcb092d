// C ABI entry points (include/wavevid_b200.h): argument checks, workspace
// carving and the K1 -> K2 -> K3 launch sequence of one decode call
// (DecodeSession._decode, decoding.py:260-307).  No allocation, no global
// mutable state: everything lives in the caller's workspace.
#include "wv_common.cuh"

using namespace wv;

namespace {

int check(const wv_geometry* g, const wv_frame_args* a, Layout* lo) {
  if (!g || !a) return WV_ERR_ARG;
  int st = build_layout(g, lo);
  if (st != WV_OK) return st;
  if (a->mode < WV_MODE_FULL || a->mode > WV_MODE_FOVEATED) return WV_ERR_ARG;
  if (a->t < 0 || a->t >= g->inter_size) return WV_ERR_ARG;
  if (!a->d_payload || !a->d_extrema || !a->d_set_loaded || !a->d_set_bytes || !a->d_canvas ||
      !a->d_footprint || !a->d_result)
    return WV_ERR_ARG;
  if (reinterpret_cast<uintptr_t>(a->d_payload) & 15) return WV_ERR_ARG;
  if (a->mode != WV_MODE_FULL && !a->d_mask) return WV_ERR_ARG;
  return WV_OK;
}

}  // namespace

extern "C" {

int wv_abi_version(void) { return WV_ABI_VERSION; }

const char* wv_status_string(int status) {
  switch (status) {
    case WV_OK: return "ok";
    case WV_ERR_ARG: return "invalid argument";
    case WV_ERR_CUDA: return "CUDA error";
    case WV_ERR_UNSUPPORTED: return "unsupported geometry";
    default: return "unknown status";
  }
}

int wv_workspace_bytes(const wv_geometry* g, uint64_t* bytes) {
  Layout lo;
  if (!bytes) return WV_ERR_ARG;
  int st = build_layout(g, &lo);
  if (st != WV_OK) return st;
  *bytes = lo.total;
  return WV_OK;
}

int wv_workspace_reset(const wv_geometry* g, void* ws, void* stream) {
  Layout lo;
  int st = build_layout(g, &lo);
  if (st != WV_OK) return st;
  if (!ws) return WV_ERR_ARG;
  WV_CUDA(cudaMemsetAsync(ws, 0, lo.total, (cudaStream_t)stream));
  return WV_OK;
}

int wv_select(const wv_geometry* g, const wv_frame_args* a, void* ws, void* stream) {
  Layout lo;
  int st = check(g, a, &lo);
  if (st != WV_OK) return st;
  if (!ws) return WV_ERR_ARG;
  return launch_select(lo, g, a, (uint8_t*)ws, (cudaStream_t)stream);
}

int wv_dequant_temporal(const wv_geometry* g, const wv_frame_args* a, void* ws, void* stream) {
  Layout lo;
  int st = check(g, a, &lo);
  if (st != WV_OK) return st;
  if (!ws) return WV_ERR_ARG;
  return launch_temporal(lo, g, a, (uint8_t*)ws, (cudaStream_t)stream);
}

int wv_synthesize(const wv_geometry* g, const wv_frame_args* a, void* ws, void* stream) {
  Layout lo;
  int st = check(g, a, &lo);
  if (st != WV_OK) return st;
  if (!ws) return WV_ERR_ARG;
  return launch_synthesis(lo, g, a, (uint8_t*)ws, (cudaStream_t)stream);
}

int wv_decode_frame(const wv_geometry* g, const wv_frame_args* a, void* ws, void* stream) {
  Layout lo;
  int st = check(g, a, &lo);
  if (st != WV_OK) return st;
  if (!ws) return WV_ERR_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  if ((st = launch_select(lo, g, a, (uint8_t*)ws, s)) != WV_OK) return st;
  if ((st = launch_temporal(lo, g, a, (uint8_t*)ws, s)) != WV_OK) return st;
  return launch_synthesis(lo, g, a, (uint8_t*)ws, s);
}

int wv_synthesize_level(const wv_geometry* g, const wv_frame_args* a, void* ws, int level,
                        void* stream) {
  Layout lo;
  int st = check(g, a, &lo);
  if (st != WV_OK) return st;
  if (!ws || level < 1 || level > lo.L) return WV_ERR_ARG;
  return launch_synthesis(lo, g, a, (uint8_t*)ws, (cudaStream_t)stream, level);
}

int wv_render_perspective(const wv_view_args* views, int n_views, void* stream) {
  if (!views) return WV_ERR_ARG;
  return launch_perspective(views, n_views, (cudaStream_t)stream);
}

int wv_plane_view(const wv_geometry* g, void* ws, float** d_plane) {
  Layout lo;
  int st = build_layout(g, &lo);
  if (st != WV_OK) return st;
  if (!ws || !d_plane) return WV_ERR_ARG;
  *d_plane = (float*)((uint8_t*)ws + lo.plane);
  return WV_OK;
}

int wv_level_mask_view(const wv_geometry* g, void* ws, int level, uint32_t** d_bits,
                       int32_t* words_per_row) {
  Layout lo;
  int st = build_layout(g, &lo);
  if (st != WV_OK) return st;
  if (!ws || !d_bits || !words_per_row || level < 1 || level > lo.L) return WV_ERR_ARG;
  // viewport/full masks sit in batch 0 of the level stack; foveated masks in batch `level`
  *d_bits = (uint32_t*)((uint8_t*)ws + lo.stack[level]);
  *words_per_row = lo.wpr_[level];
  return WV_OK;
}

int wv_block_list_view(const wv_geometry* g, void* ws, uint32_t** d_list, uint32_t** d_count) {
  Layout lo;
  int st = build_layout(g, &lo);
  if (st != WV_OK) return st;
  if (!ws || !d_list || !d_count) return WV_ERR_ARG;
  *d_list = (uint32_t*)((uint8_t*)ws + lo.blist);
  *d_count = (uint32_t*)((uint8_t*)ws + lo.counters) + CNT_BLOCKS;
  return WV_OK;
}

}  // extern "C"
