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
  if ((a->flags & WV_FLAG_FETCH) &&
      (!a->h_payload || !a->d_fetched || (reinterpret_cast<uintptr_t>(a->h_payload) & 15)))
    return WV_ERR_ARG;
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
    case WV_ERR_FORMAT: return "malformed or unsupported .wvv data";
    case WV_ERR_IO: return "file missing or truncated";
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

int wv_workspace_bytes_select(const wv_geometry* g, uint64_t* bytes) {
  Layout lo;
  if (!bytes) return WV_ERR_ARG;
  int st = build_layout(g, &lo);
  if (st != WV_OK) return st;
  *bytes = lo.select_bytes;
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

// Host-argument entry points: copy the arguments into the workspace
// descriptor slot (stream-ordered) and run the launch sequence reading it.
static int stage(const wv_geometry* g, const wv_frame_args* a, void* ws, void* stream,
                 Layout* lo, wv_frame_args** d_fa) {
  int st = check(g, a, lo);
  if (st != WV_OK) return st;
  if (!ws) return WV_ERR_ARG;
  if (a->payload_bytes < (uint64_t)lo->n * lo->NB * 8) return WV_ERR_ARG;
  *d_fa = (wv_frame_args*)((uint8_t*)ws + lo->desc);
  WV_CUDA(cudaMemcpyAsync(*d_fa, a, sizeof(wv_frame_args), cudaMemcpyHostToDevice,
                          (cudaStream_t)stream));
  return WV_OK;
}

// the fetch stage right after selection, unless the caller streams the spans
// from the file in between (h_fetch_list set: it runs WV_STAGE_FETCH itself)
static int select_and_fetch(const Layout& lo, const wv_geometry* g, const wv_frame_args* a,
                            const wv_frame_args* d, uint8_t* ws, cudaStream_t s) {
  int st = launch_select(lo, g, a->mode, a->flags, d, ws, s);
  if (st != WV_OK) return st;
  if ((a->flags & WV_FLAG_FETCH) && !a->h_fetch_list) return launch_fetch(lo, d, ws, s);
  return WV_OK;
}

int wv_select(const wv_geometry* g, const wv_frame_args* a, void* ws, void* stream) {
  Layout lo;
  wv_frame_args* d;
  int st = stage(g, a, ws, stream, &lo, &d);
  if (st != WV_OK) return st;
  return select_and_fetch(lo, g, a, d, (uint8_t*)ws, (cudaStream_t)stream);
}

int wv_dequant_temporal(const wv_geometry* g, const wv_frame_args* a, void* ws, void* stream) {
  Layout lo;
  wv_frame_args* d;
  int st = stage(g, a, ws, stream, &lo, &d);
  if (st != WV_OK) return st;
  return launch_temporal(lo, g, a->mode, d, (uint8_t*)ws, (cudaStream_t)stream);
}

int wv_synthesize(const wv_geometry* g, const wv_frame_args* a, void* ws, void* stream) {
  Layout lo;
  wv_frame_args* d;
  int st = stage(g, a, ws, stream, &lo, &d);
  if (st != WV_OK) return st;
  return launch_synthesis(lo, g, d, (uint8_t*)ws, (cudaStream_t)stream);
}

int wv_decode_frame(const wv_geometry* g, const wv_frame_args* a, void* ws, void* stream) {
  Layout lo;
  wv_frame_args* d;
  int st = stage(g, a, ws, stream, &lo, &d);
  if (st != WV_OK) return st;
  cudaStream_t s = (cudaStream_t)stream;
  if ((st = select_and_fetch(lo, g, a, d, (uint8_t*)ws, s)) != WV_OK) return st;
  if (a->flags & WV_FLAG_ACCOUNT_ONLY) return WV_OK;
  if ((st = launch_temporal(lo, g, a->mode, d, (uint8_t*)ws, s)) != WV_OK) return st;
  return launch_synthesis(lo, g, d, (uint8_t*)ws, s);
}

int wv_synthesize_level(const wv_geometry* g, const wv_frame_args* a, void* ws, int level,
                        void* stream) {
  Layout lo;
  wv_frame_args* d;
  int st = stage(g, a, ws, stream, &lo, &d);
  if (st != WV_OK) return st;
  if (level < 1 || level > lo.L) return WV_ERR_ARG;
  return launch_synthesis(lo, g, d, (uint8_t*)ws, (cudaStream_t)stream, level);
}

int wv_synthesize_level_desc(const wv_geometry* g, void* ws, int level, void* stream) {
  Layout lo;
  int st = build_layout(g, &lo);
  if (st != WV_OK) return st;
  if (!ws || level < 1 || level > lo.L) return WV_ERR_ARG;
  const wv_frame_args* d = (const wv_frame_args*)((uint8_t*)ws + lo.desc);
  return launch_synthesis(lo, g, d, (uint8_t*)ws, (cudaStream_t)stream, level);
}

int wv_desc_view(const wv_geometry* g, void* ws, void** d_desc) {
  Layout lo;
  int st = build_layout(g, &lo);
  if (st != WV_OK) return st;
  if (!ws || !d_desc) return WV_ERR_ARG;
  *d_desc = (uint8_t*)ws + lo.desc;
  return WV_OK;
}

int wv_decode_frame_desc(const wv_geometry* g, int mode, int flags, void* ws, void* stream) {
  Layout lo;
  int st = build_layout(g, &lo);
  if (st != WV_OK) return st;
  if (!ws || mode < WV_MODE_FULL || mode > WV_MODE_FOVEATED) return WV_ERR_ARG;
  const wv_frame_args* d = (const wv_frame_args*)((uint8_t*)ws + lo.desc);
  cudaStream_t s = (cudaStream_t)stream;
  if ((st = launch_select(lo, g, mode, flags, d, (uint8_t*)ws, s)) != WV_OK) return st;
  if ((flags & WV_FLAG_FETCH) && (st = launch_fetch(lo, d, (uint8_t*)ws, s)) != WV_OK) return st;
  if (flags & WV_FLAG_ACCOUNT_ONLY) return WV_OK;
  if ((st = launch_temporal(lo, g, mode, d, (uint8_t*)ws, s)) != WV_OK) return st;
  return launch_synthesis(lo, g, d, (uint8_t*)ws, s);
}

int wv_decode_stages_desc(const wv_geometry* g, int mode, int flags, int stages, void* ws,
                          void* stream) {
  Layout lo;
  int st = build_layout(g, &lo);
  if (st != WV_OK) return st;
  if (!ws || mode < WV_MODE_FULL || mode > WV_MODE_FOVEATED || (stages & ~WV_STAGE_ALL))
    return WV_ERR_ARG;
  const wv_frame_args* d = (const wv_frame_args*)((uint8_t*)ws + lo.desc);
  cudaStream_t s = (cudaStream_t)stream;
  if (stages & WV_STAGE_SELECT)
    if ((st = launch_select(lo, g, mode, flags, d, (uint8_t*)ws, s, stages & WV_STAGE_SELECT)) !=
        WV_OK)
      return st;
  if ((stages & WV_STAGE_FETCH) && (flags & WV_FLAG_FETCH) &&
      (st = launch_fetch(lo, d, (uint8_t*)ws, s)) != WV_OK)
    return st;
  if (flags & WV_FLAG_ACCOUNT_ONLY) return WV_OK;
  if ((stages & WV_STAGE_DEQUANT) &&
      (st = launch_temporal(lo, g, mode, d, (uint8_t*)ws, s)) != WV_OK)
    return st;
  if (stages & WV_STAGE_SYNTH) return launch_synthesis(lo, g, d, (uint8_t*)ws, s);
  return WV_OK;
}

int wv_render_perspective_desc(const wv_view_args* d_views, int n_views, int max_out_w,
                               int max_out_h, int shared_geometry, void* stream) {
  return launch_perspective_dev(d_views, n_views, max_out_w, max_out_h, shared_geometry,
                                (cudaStream_t)stream);
}

int wv_render_perspective(const wv_view_args* views, int n_views, void* stream) {
  if (!views) return WV_ERR_ARG;
  return launch_perspective(views, n_views, (cudaStream_t)stream);
}

int wv_enqueue_frame(void* d_desc, const void* h_desc, uint64_t desc_bytes, void* graph_exec,
                     void* stream, const void* d_result, void* h_result, void* event) {
  if (!d_desc || !h_desc || !graph_exec || !d_result || !h_result) return WV_ERR_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  WV_CUDA(cudaMemcpyAsync(d_desc, h_desc, desc_bytes, cudaMemcpyHostToDevice, s));
  WV_CUDA(cudaGraphLaunch((cudaGraphExec_t)graph_exec, s));
  WV_CUDA(cudaMemcpyAsync(h_result, d_result, sizeof(wv_frame_result), cudaMemcpyDeviceToHost, s));
  if (event) WV_CUDA(cudaEventRecord((cudaEvent_t)event, s));
  return WV_OK;
}

int wv_synthesize_2d(const wv_geometry* g, const float* d_pyramid, float* d_out, void* ws,
                     void* d_result, void* stream) {
  Layout lo;
  int st = build_layout(g, &lo);
  if (st != WV_OK) return st;
  if (!d_pyramid || !d_out || !ws || !d_result) return WV_ERR_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  uint8_t* w = (uint8_t*)ws;
  WV_CUDA(cudaMemcpyAsync(w + lo.plane, d_pyramid, (size_t)lo.C * lo.H * lo.W * 4,
                          cudaMemcpyDeviceToDevice, s));
  // a full-frame descriptor: every tile of every level (LevelMaskSet.full)
  wv_frame_args fa{};
  fa.mode = WV_MODE_FULL;
  fa.d_result = (wv_frame_result*)d_result;
  wv_frame_args* d_fa = (wv_frame_args*)(w + lo.desc);
  WV_CUDA(cudaMemcpyAsync(d_fa, &fa, sizeof(fa), cudaMemcpyHostToDevice, s));
  if ((st = launch_select(lo, g, WV_MODE_FULL, 0, d_fa, w, s, WV_STAGE_ROWS | WV_STAGE_TILES)) !=
      WV_OK)
    return st;
  return launch_synthesis_f32(lo, d_fa, w, d_out, s);
}

int wv_table_expand(const uint16_t* d_counts, uint64_t n_entries, int record_size,
                    uint64_t* d_table, void* stream) {
  if (!d_counts || !d_table || record_size < 1 || n_entries == 0) return WV_ERR_ARG;
  return launch_table_expand(d_counts, n_entries, record_size, d_table, (cudaStream_t)stream);
}

int wv_desc_layout(const wv_geometry* g, uint64_t* mask_offset, uint64_t* slot_bytes) {
  Layout lo;
  int st = build_layout(g, &lo);
  if (st != WV_OK) return st;
  if (!mask_offset || !slot_bytes) return WV_ERR_ARG;
  *mask_offset = lo.desc_mask;
  *slot_bytes = lo.desc_bytes;
  return WV_OK;
}

int wv_synthesis_tile(int* ty, int* tx) {
  if (!ty || !tx) return WV_ERR_ARG;
  *ty = TY;
  *tx = TX;
  return WV_OK;
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

int wv_fetch_list_view(const wv_geometry* g, void* ws, uint32_t** d_list, uint32_t** d_count) {
  Layout lo;
  int st = build_layout(g, &lo);
  if (st != WV_OK) return st;
  if (!ws || !d_list || !d_count) return WV_ERR_ARG;
  *d_list = (uint32_t*)((uint8_t*)ws + lo.flist);
  *d_count = (uint32_t*)((uint8_t*)ws + lo.counters) + CNT_FETCH;
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
