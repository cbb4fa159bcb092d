/*
 * wavevid_b200.h — C ABI of the B200 decode hot path for the wavelet
 * 360-degree video codec of arXiv 2208.10859 (reference package `wavevid`,
 * citations relative to /root/reference).
 *
 * The reference is pure Python; its decode seam is the Python method
 * DecodeSession._decode (pkg/src/wavevid/decoding.py:260-307), reached from
 * decode_viewport / decode_foveated / decode_full (decoding.py:309-331).
 * Each entry point below replaces one stage of that method:
 *
 *   wv_select            LevelMaskSet.from_pixel_mask      wavelets.py:272-306
 *                        foveation_masks                   decoding.py:124-152
 *                        upscale_mask                      fileio.py:430-436
 *                        inclusion_grid + block ids        wavelets.py:337-348,
 *                                                          decoding.py:265-268
 *                        footprint cascade                 wavelets.py:380-392
 *                        bytes_loaded / records_processed  decoding.py:271-285
 *   wv_dequant_temporal  dequantize_records                decoding.py:37-50
 *                        temporal_inverse_sparse           decoding.py:53-90
 *                        inclusion masking                 wavelets.py:372-378
 *   wv_synthesize        synthesize_2d_region synthesis    wavelets.py:396-443
 *                        + u8 conversion                   decoding.py:301
 *   wv_decode_frame      DecodeSession._decode (all of the above)
 *   wv_render_perspective render_perspective               projection.py:111-172
 *   wv_encode_set        encode_video, one set (mirror path) encoding.py:377-425
 *
 * Conventions: plain pointers and sizes only.  Every pointer named d_* or
 * documented as "device" is CUDA device memory owned by the caller; the
 * library allocates nothing and keeps no global mutable state.  `stream` is
 * a cudaStream_t passed as void*.  Calls are asynchronous on that stream and
 * return a WV_* status for argument/launch errors; data-dependent errors
 * (corrupt stream, coverage) are reported through device-side result words
 * the caller reads after synchronising.
 */
#ifndef WAVEVID_B200_H
#define WAVEVID_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define WV_ABI_VERSION 4
#define WV_MAX_LEVELS 12

enum wv_status {
  WV_OK = 0,
  WV_ERR_ARG = 1,          /* invalid geometry / argument */
  WV_ERR_CUDA = 2,         /* a CUDA runtime call or launch failed */
  WV_ERR_UNSUPPORTED = 3,  /* geometry outside what the kernels handle */
  WV_ERR_FORMAT = 4,       /* malformed or unsupported .wvv data (FormatError, fileio.py:34) */
  WV_ERR_IO = 5            /* file missing / truncated read */
};

enum wv_mode { WV_MODE_FULL = 0, WV_MODE_VIEWPORT = 1, WV_MODE_FOVEATED = 2 };

/* wv_frame_args.flags */
enum wv_flags {
  WV_FLAG_ACCOUNT_ONLY = 1,  /* wv_select only: update the set's cache accounting
                                (DecodeSession.advance prefetch, decoding.py:335-354);
                                no work lists, no footprint, dirty maps untouched */
  WV_FLAG_FETCH = 2          /* span streaming (VideoReader.load_blocks, fileio.py:346-390):
                                d_payload holds the BlockEnd table but records only for
                                blocks whose d_fetched bit is set; the records of newly
                                selected blocks are copied from h_payload (pinned host
                                memory, read by the GPU over PCIe) before K2 runs */
};

/* device error word bits (wv_frame_result.error) */
enum wv_device_error {
  WV_DERR_OFFSET = 1,      /* record offset >= block_size^2 -> CorruptStreamError */
  WV_DERR_TABLE = 2        /* BlockEnd span outside payload / misaligned */
};

/* Decode geometry = the .wvv header fields the kernels need
 * (fileio.py:38-61). */
typedef struct wv_geometry {
  int32_t width, height, channels, levels;
  int32_t inter_size, block_size, float_mode;
  int32_t mask_w, mask_h;
} wv_geometry;

/* Device-side per-call result (caller allocates, library overwrites). */
typedef struct wv_frame_result {
  unsigned long long new_bytes;   /* span bytes of blocks newly added to the set's cache entry */
  unsigned long long set_bytes;   /* cache entry total after this call (decoding.py:231) */
  unsigned long long records;     /* records_processed (decoding.py:284) */
  uint32_t n_missing;             /* blocks newly added to the entry */
  uint32_t n_selected;            /* blocks selected by the level masks */
  uint32_t error;                 /* WV_DERR_* bits */
  uint32_t n_tiles;               /* level-1 synthesis tiles computed */
  unsigned long long fetched_bytes;/* WV_FLAG_FETCH: record bytes copied host -> HBM by this call */
} wv_frame_result;

typedef struct wv_frame_args {
  int32_t mode;                   /* wv_mode */
  int32_t t;                      /* display time inside the set, 0 <= t < inter_size */
  int32_t flags;                  /* wv_flags */
  int32_t reserved;
  const uint8_t* d_mask;          /* (mask_h, mask_w) bytes 0/1; unused for FULL */
  int32_t fovea[WV_MAX_LEVELS][4];/* FOVEATED: detail level k at [k-1]: r0, r1, c0, c1
                                     pixel window, half-open (decoding.py:147-150) */
  const void* d_payload;          /* set payload: BlockEnd table (n*NB u64) + packed records, 16-B aligned
                                     and readable up to the next 16-byte boundary past payload_bytes
                                     (K2 stages record spans in 16-byte chunks) */
  uint64_t payload_bytes;
  const float* d_extrema;         /* (n, C, 4) float32 (fileio.py:123) */
  uint32_t* d_set_loaded;         /* NB-bit block bitmap of the set's cache entry */
  unsigned long long* d_set_bytes;/* the entry's cumulative bytes */
  uint8_t* d_canvas;              /* planar (C, H, W) u8 output; must persist across calls of one workspace */
  uint32_t* d_footprint;          /* (H, ceil(W/32)) bit rows output, bit i of word w = column 32w+i;
                                     like d_canvas it is updated incrementally (only the 64x64 tiles
                                     that touch or left the request are rewritten): zero it once and
                                     pass the same buffer to every call of one workspace */
  wv_frame_result* d_result;
  const void* h_payload;          /* WV_FLAG_FETCH: the set payload in pinned host memory (UVA
                                     pointer, same layout as d_payload) */
  uint32_t* d_fetched;            /* WV_FLAG_FETCH: NB-bit bitmap, records of block b are in
                                     d_payload; zero it when d_payload is (re)filled */
  uint32_t* h_fetch_list;         /* WV_FLAG_FETCH, optional: host (pinned) buffers that receive
                                     this call's fetch list -- the blocks whose records are not yet
                                     in HBM (NB u32) -- and its length, before the fetch stage
                                     (span streaming from the file, wv_span_queue_enqueue) */
  uint32_t* h_fetch_count;
  int32_t out_row0, out_row1;     /* output pixel rows this call must produce, half open
                                     (0, 0 = the whole frame).  A stereo eye split
                                     ([0, H/2) or [H/2, H)) synthesises only the tiles those
                                     rows depend on; its pixels and footprint inside the rows
                                     equal a whole-frame decode's.  Masks, block selection,
                                     K2 and the stats are unchanged. */
} wv_frame_args;

/* One perspective view (projection.py:111-172). */
typedef struct wv_view_args {
  const uint8_t* d_canvas;        /* planar (C, canvas_h, W) u8 */
  const uint32_t* d_footprint;    /* bit rows of the same canvas */
  int32_t row0, rows;             /* equirect region = canvas rows [row0, row0+rows) (a stereo eye) */
  int32_t width, channels;
  int32_t canvas_h, reserved;
  double rot[9];                  /* world-from-camera rotation, row major (projection.py:39-52) */
  double tan_h, tan_v;            /* tan(fov_h/2), tan(fov_v/2) */
  int32_t out_w, out_h;
  uint8_t* d_out;                 /* (out_h, out_w, C) u8 */
  uint32_t* d_uncovered;          /* device counter: output pixels with a tap outside the footprint */
} wv_view_args;

int wv_abi_version(void);
const char* wv_status_string(int status);

/* Bytes of device workspace one decode stream needs for this geometry. */
int wv_workspace_bytes(const wv_geometry* g, uint64_t* bytes);
/* Bytes of a selection-only workspace: enough for wv_select with
 * WV_FLAG_ACCOUNT_ONLY (and WV_STAGE_FETCH through wv_decode_stages_desc) on
 * a second stream, e.g. prefetching the next set beside the current decodes
 * (DecodeSession.advance, decoding.py:335-354).  Zero it once. */
int wv_workspace_bytes_select(const wv_geometry* g, uint64_t* bytes);
/* Zero the workspace (coefficient plane, dirty maps). Call once after allocation. */
int wv_workspace_reset(const wv_geometry* g, void* d_workspace, void* stream);

int wv_select(const wv_geometry* g, const wv_frame_args* a, void* d_workspace, void* stream);
int wv_dequant_temporal(const wv_geometry* g, const wv_frame_args* a, void* d_workspace, void* stream);
int wv_synthesize(const wv_geometry* g, const wv_frame_args* a, void* d_workspace, void* stream);
int wv_decode_frame(const wv_geometry* g, const wv_frame_args* a, void* d_workspace, void* stream);
/* One synthesis level k (1 = finest, writes the u8 canvas) of wv_synthesize;
 * levels must run L..1 after wv_select/wv_dequant_temporal (timing, profiling). */
int wv_synthesize_level(const wv_geometry* g, const wv_frame_args* a, void* d_workspace,
                        int level, void* stream);
/* The same level reading the frame arguments already in the workspace
 * descriptor (no argument copy on the stream: per-kernel timing). */
int wv_synthesize_level_desc(const wv_geometry* g, void* d_workspace, int level, void* stream);

int wv_render_perspective(const wv_view_args* views, int n_views, void* stream);

/* Graph-capturable variants.  Per-frame inputs live in device memory: the
 * frame arguments in the workspace descriptor slot (wv_desc_view; a
 * wv_frame_args followed by room for 4 wv_view_args), so the launch sequence
 * of a mode is fixed and can be recorded once in a CUDA graph and replayed
 * after a single H2D copy of the slot per frame. */
int wv_desc_view(const wv_geometry* g, void* d_workspace, void** d_desc);
int wv_decode_frame_desc(const wv_geometry* g, int mode, int flags, void* d_workspace,
                         void* stream);
/* Stages of one decode (bit mask) for callers that overlap independent
 * stages on several streams (e.g. inside a CUDA graph).  Dependencies:
 * CASCADES, TILES <- ROWS; FOOTPRINT, BLOCKS <- CASCADES; DEQUANT <- BLOCKS;
 * SYNTH <- DEQUANT, TILES; FOOTPRINT_TILES <- FOOTPRINT, TILES.  The
 * footprint (only the writeout needs it) and the tile lists can therefore run
 * beside block selection -> K2.  wv_decode_frame_desc runs all stages in
 * order. */
enum wv_stage {
  WV_STAGE_ROWS = 1,              /* distinct request-mask rows, row map, counters (K1) */
  WV_STAGE_CASCADES = 2,          /* level-mask cascades (K1) */
  WV_STAGE_FOOTPRINT = 4,         /* footprint cascade levels L..2 (K1) */
  WV_STAGE_BLOCKS = 8,            /* block selection + accounting, span fetch (K1) */
  WV_STAGE_TILES = 16,            /* synthesis tile lists (K1) */
  WV_STAGE_FOOTPRINT_TILES = 32,  /* finest footprint on the level-1 tiles (K1) */
  WV_STAGE_DEQUANT = 64,          /* K2 */
  WV_STAGE_SYNTH = 128,           /* K3, all levels */
  WV_STAGE_FETCH = 256,           /* WV_FLAG_FETCH: copy the listed blocks' records host -> HBM
                                     (k_fetch) <- BLOCKS; DEQUANT waits for it */
  WV_STAGE_SELECT = 63,
  WV_STAGE_ALL = 511
};
int wv_decode_stages_desc(const wv_geometry* g, int mode, int flags, int stages,
                          void* d_workspace, void* stream);

/* One frame of a captured decode graph in a single call (the per-frame host
 * path of DecodeSession): copy the frame's descriptor -- wv_frame_args, the
 * wv_view_args and the request-mask bytes, laid out as in the workspace
 * descriptor slot -- from pinned host memory to the slot (d_desc, from
 * wv_desc_view), launch the graph (a cudaGraphExec_t recorded from
 * wv_decode_stages_desc / wv_render_perspective_desc reading that slot),
 * copy the frame's wv_frame_result back to pinned host memory and record
 * `event` (a cudaEvent_t, may be NULL), all on `stream`.  Replaces the
 * decode call of DecodeSession._decode (decoding.py:260-307) for callers
 * that pipeline frames. */
int wv_enqueue_frame(void* d_desc, const void* h_desc, uint64_t desc_bytes, void* graph_exec,
                     void* stream, const void* d_result, void* h_result, void* event);
/* Bytes of the descriptor slot: wv_frame_args, 4 wv_view_args, then the
 * mask bytes (mask_h * mask_w) at wv_desc_mask_offset(). */
int wv_desc_layout(const wv_geometry* g, uint64_t* mask_offset, uint64_t* slot_bytes);
/* The synthesis tile of the inverse-DWT kernels: ty x tx coefficients of each
 * subband per work item (2 ty x 2 tx output samples); tile counts reported
 * by the decode (wv_block_list_view counters) are in these units. */
int wv_synthesis_tile(int* ty, int* tx);

/* shared_geometry != 0: all views share pose, FOV, region size and output
 * size (a stereo pair rendered with one head pose) -- the ray geometry is
 * computed once per output pixel and applied to every view. */
int wv_render_perspective_desc(const wv_view_args* d_views, int n_views, int max_out_w,
                               int max_out_h, int shared_geometry, void* stream);

/* ---- .wvv container reader (fileio.py:28-193, read_header :240-261) ----
 * Host-only, stateless (each call opens, reads and closes the file), no
 * allocation: a C-ABI consumer (e.g. a native player) gets the decode
 * geometry, the set directory and set payloads without Python. */
typedef struct wv_file_info {
  wv_geometry geom;               /* decode geometry of the header */
  int32_t frame_count, pad_frames, num_sets, stereo;
  float fps;
  uint32_t version;
  uint64_t table_bytes;           /* BlockEnd table bytes per set: inter_size * num_blocks * 8 */
} wv_file_info;

typedef struct wv_set_info {
  uint64_t payload_offset, payload_length, record_count;
} wv_set_info;

/* Parse and validate the 64-byte header and the SetMeta directory. */
int wv_file_info_read(const char* path, wv_file_info* info);
/* Directory entry of one set; its extrema (inter_size, C, 4) f32 into
 * `extrema` when not NULL (fileio.py:118-138). */
int wv_file_set_read(const char* path, int set_index, wv_set_info* set, float* extrema);
/* One set's payload (BlockEnd table + packed records) into `buf`
 * (>= payload_length bytes; pinned host memory serves both a whole-set
 * upload and WV_FLAG_FETCH's h_payload). */
int wv_file_payload_read(const char* path, int set_index, void* buf, uint64_t buf_bytes);

/* ---- Span streaming from the file ----
 * VideoReader.load_blocks (fileio.py:346-390) for a block list made on the
 * GPU: for every temporal index and every run of consecutive ids, the span
 * (end of the previous (t, block) entry, end of the run's last block)
 * (block_range_bytes, fileio.py:168-181) of the record data is read from
 * `fd` into the same payload offset of `dst` (widened to whole 16-byte
 * chunks, which the fetch kernel copies); ranges are merged through gaps
 * <= coalesce_gap (COALESCE_GAP 4096, fileio.py:31, :264-274), one pread
 * per merged range.  bytes_read: the reference's coalesced read of the
 * exact spans (VideoReader.io_trace), bytes_spans: bytes of the requested
 * spans. */
#define WV_SPAN_QUEUE 64
typedef struct wv_span_job {
  int32_t fd;                     /* open .wvv file */
  int32_t n, nb;                  /* inter_size, blocks per frame */
  int32_t status;                 /* out: WV_* of the read */
  uint64_t payload_offset;        /* file offset of the set's payload (its BlockEnd table) */
  uint64_t payload_bytes;         /* payload length */
  uint64_t table_bytes;           /* n * nb * 8 */
  const uint64_t* table;          /* host BlockEnd table of the set, n * nb u64 */
  uint8_t* dst;                   /* host buffer mirroring the payload (16-byte chunks of
                                     every requested span are filled from the file) */
  const uint32_t* ids;            /* host block list (any order) ... */
  const uint32_t* count;          /* ... and its length */
  uint64_t coalesce_gap;
  uint64_t bytes_read, bytes_spans;   /* out */
  int32_t done, reserved;         /* out: 1 once read */
} wv_span_job;
/* FIFO of jobs consumed by stream-ordered reads (caller-owned host memory,
 * zero-initialised; one producer, the stream's host-function thread as the
 * consumer). */
typedef struct wv_span_queue {
  wv_span_job jobs[WV_SPAN_QUEUE];
  uint32_t fifo[WV_SPAN_QUEUE];
  uint32_t head, tail;
} wv_span_queue;
int wv_spans_read(const wv_span_job* job, uint64_t* bytes_read, uint64_t* bytes_spans);
/* Append a copy of *job (stored in jobs[slot]) to the queue. */
int wv_span_queue_push(wv_span_queue* q, const wv_span_job* job, uint32_t slot);
/* Enqueue on `stream` a host function that runs the oldest queued job
 * (cudaLaunchHostFunc; capturable into a CUDA graph, where every replay
 * consumes the next job). */
int wv_span_queue_enqueue(wv_span_queue* q, void* stream);
/* The BlockEnd table from per-(t, block) record counts (n_entries = n * NB,
 * row major): d_table[i] = record_size * (counts[0] + ... + counts[i]), the
 * cumulative ends of fileio.py:157-162.  Span residency uploads the 2-byte
 * counts (a quarter of the table) and rebuilds the table in HBM. */
int wv_table_expand(const uint16_t* d_counts, uint64_t n_entries, int record_size,
                    uint64_t* d_table, void* stream);
/* Device views of the fetch list of the last select (k_blocks output). */
int wv_fetch_list_view(const wv_geometry* g, void* d_workspace, uint32_t** d_list,
                       uint32_t** d_count);

/* ---- Encoder: one inter-frame set ----
 * Replaces the per-set body of the reference encoder, encode_video
 * (encoding.py:377-425): analyze_2d (wavelets.py:128-149), sparsify
 * (encoding.py:118-135), haar_time_forward (:153-169), temporal_threshold
 * (:198-236), compute_extrema (:239-254), quantize (:296-332) and the record
 * order / BlockEnd counts (fileio.py:142-165).  Output bytes equal the
 * reference's (the golden sha256 manifest).  Thresholds are passed as the
 * float32 values the reference compares against:
 *   level_threshold[k-1] = float32(threshold_value(alpha, k-1, levels)), k = 1..levels
 *   row_factor[y]        = float32 equirect H(y) (encoding.py:359-362), or 0 (no mapping)
 *   temporal_threshold[t] = float32(threshold_value(inter_threshold,
 *                             temporal_level_of(t, n) - 1, log2 n)), t = 1..n-1 */
#define WV_ENC_MAX_N 64
typedef struct wv_encode_params {
  int32_t width, height, channels;  /* frame size (width, height divisible by 2^levels and block_size) */
  int32_t levels;                   /* spatial DWT levels, 1..WV_MAX_LEVELS */
  int32_t inter_size;               /* n frames per set: power of two, <= WV_ENC_MAX_N */
  int32_t block_size;               /* power of two dividing width and height, <= 32 */
  int32_t quantize;                 /* 1: u8 records, 0: float32 records (FLAG_FLOAT) */
  int32_t reserved;
  float level_threshold[WV_MAX_LEVELS];
  float temporal_threshold[WV_ENC_MAX_N];
} wv_encode_params;

/* Device workspace bytes for wv_encode_set, and the payload capacity that
 * can never overflow (every coefficient a record). */
int wv_encode_workspace_bytes(const wv_encode_params* p, uint64_t* bytes);
int wv_encode_payload_capacity(const wv_encode_params* p, uint64_t* bytes);
/* d_frames: n x H x W x C u8 (device), d_row_factor: H float32 (device).
 * Outputs (device): d_extrema (n, C, 4) float32, d_counts (n, NB) u32
 * records per (temporal index, block), d_payload packed records in
 * (t, block, layer, offset) order, d_num_records (1 x u64). */
int wv_encode_set(const wv_encode_params* p, const uint8_t* d_frames, const float* d_row_factor,
                  void* d_workspace, uint64_t workspace_bytes, float* d_extrema,
                  uint32_t* d_counts, uint8_t* d_payload, uint64_t payload_capacity,
                  uint64_t* d_num_records, void* stream);

/* Full inverse 2-D CDF 9/7 of a float32 Mallat pyramid (synthesize_2d,
 * wavelets.py:167-182) with the K3 kernels: d_pyramid and d_out are planar
 * (C, H, W) float32 device buffers (geometry: width, height, channels,
 * levels; the other fields only size the workspace), d_result a device
 * wv_frame_result scratch.  Bit-exact with the reference (same lifting,
 * columns then rows, one rounding per operation).  Uses the workspace's
 * coefficient plane, so it must not run concurrently with a decode on the
 * same workspace. */
int wv_synthesize_2d(const wv_geometry* g, const float* d_pyramid, float* d_out, void* d_workspace,
                     void* d_result, void* stream);

/* Views into the workspace for parity tests (no launches). */
int wv_plane_view(const wv_geometry* g, void* d_workspace, float** d_plane);
int wv_level_mask_view(const wv_geometry* g, void* d_workspace, int level,
                       uint32_t** d_bits, int32_t* words_per_row);
int wv_block_list_view(const wv_geometry* g, void* d_workspace,
                       uint32_t** d_list, uint32_t** d_count);

#ifdef __cplusplus
}
#endif
#endif /* WAVEVID_B200_H */
