// .wvv container reader for C-ABI consumers (include/wavevid_b200.h).
//
// Reference: fileio.py:28-193 (header struct "<4sHHIIIfBBBBHHB31x" :28,
// SetMeta :118-138, BlockEnd tables :141-165) and read_header :240-261 with
// its validation (magic, version, divisibility, whole sets, contiguous
// payloads, record_count vs payload length, table inside the payload).
// Stateless: every call opens and closes the file.
#include <cstdio>
#include <cstring>

#include "../../include/wavevid_b200.h"

namespace {

constexpr int kHeaderSize = 64;

struct File {
  FILE* f = nullptr;
  explicit File(const char* path) : f(path ? std::fopen(path, "rb") : nullptr) {}
  ~File() {
    if (f) std::fclose(f);
  }
  bool read(void* dst, size_t n) { return f && std::fread(dst, 1, n, f) == n; }
  bool seek(uint64_t off) { return f && fseeko(f, (off_t)off, SEEK_SET) == 0; }
};

template <class T>
T le(const unsigned char* p) {   // little-endian field (the format is "<")
  T v;
  std::memcpy(&v, p, sizeof(T));
  return v;
}

int parse_header(File& fh, wv_file_info* info) {
  unsigned char h[kHeaderSize];
  if (!fh.read(h, sizeof h)) return WV_ERR_IO;
  if (std::memcmp(h, "WVVC", 4) != 0) return WV_ERR_FORMAT;
  const uint16_t version = le<uint16_t>(h + 4), flags = le<uint16_t>(h + 6);
  if (version != 1) return WV_ERR_FORMAT;
  wv_file_info o{};
  o.version = version;
  o.geom.width = (int32_t)le<uint32_t>(h + 8);
  o.geom.height = (int32_t)le<uint32_t>(h + 12);
  o.frame_count = (int32_t)le<uint32_t>(h + 16);
  o.fps = le<float>(h + 20);
  o.geom.channels = h[24];
  o.geom.levels = h[25];
  const int n_log2 = h[26], bs_log2 = h[27];
  if (n_log2 > 16 || bs_log2 > 15) return WV_ERR_FORMAT;
  o.geom.inter_size = 1 << n_log2;
  o.geom.block_size = 1 << bs_log2;
  o.geom.mask_w = le<uint16_t>(h + 28);
  o.geom.mask_h = le<uint16_t>(h + 30);
  o.pad_frames = h[32];
  o.stereo = (flags & 1) != 0;
  o.geom.float_mode = (flags & 2) != 0;
  const wv_geometry& g = o.geom;
  if (g.levels > 30 || g.width <= 0 || g.height <= 0 || g.channels <= 0) return WV_ERR_FORMAT;
  if ((g.width % (1 << g.levels)) || (g.height % (1 << g.levels))) return WV_ERR_FORMAT;
  if ((g.width % g.block_size) || (g.height % g.block_size)) return WV_ERR_FORMAT;
  if ((o.frame_count + o.pad_frames) % g.inter_size) return WV_ERR_FORMAT;
  o.num_sets = (o.frame_count + o.pad_frames) / g.inter_size;
  const uint64_t nb = (uint64_t)(g.width / g.block_size) * (g.height / g.block_size);
  o.table_bytes = (uint64_t)g.inter_size * nb * 8;
  *info = o;
  return WV_OK;
}

size_t meta_size(const wv_file_info& i) { return 24 + (size_t)i.geom.inter_size * i.geom.channels * 16; }

// Reads directory entries 0..upto (validating each against its predecessor);
// fills `want` for entry upto.
int walk_meta(File& fh, const wv_file_info& info, int upto, wv_set_info* want, float* extrema) {
  const size_t ms = meta_size(info);
  const uint64_t rs = 2 + (uint64_t)info.geom.channels * (info.geom.float_mode ? 4 : 1);
  unsigned char head[24];
  wv_set_info prev{};
  for (int i = 0; i <= upto; ++i) {
    if (!fh.read(head, 24)) return WV_ERR_IO;
    wv_set_info m{le<uint64_t>(head), le<uint64_t>(head + 8), le<uint64_t>(head + 16)};
    const size_t ext_bytes = ms - 24;
    if (i == upto && extrema) {
      if (!fh.read(extrema, ext_bytes)) return WV_ERR_IO;
    } else if (!fh.seek((uint64_t)ftello(fh.f) + ext_bytes)) {
      return WV_ERR_IO;
    }
    if (i && m.payload_offset != prev.payload_offset + prev.payload_length) return WV_ERR_FORMAT;
    // record_count * rs > payload_length, without the u64 wrap-around
    if (m.record_count > m.payload_length / (uint64_t)rs) return WV_ERR_FORMAT;
    if (m.payload_length < info.table_bytes) return WV_ERR_FORMAT;
    prev = m;
  }
  if (want) *want = prev;
  return WV_OK;
}

}  // namespace

extern "C" {

int wv_file_info_read(const char* path, wv_file_info* info) {
  if (!path || !info) return WV_ERR_ARG;
  File fh(path);
  if (!fh.f) return WV_ERR_IO;
  wv_file_info i;
  int st = parse_header(fh, &i);
  if (st != WV_OK) return st;
  if (i.num_sets > 0 && (st = walk_meta(fh, i, i.num_sets - 1, nullptr, nullptr)) != WV_OK)
    return st;
  *info = i;
  return WV_OK;
}

int wv_file_set_read(const char* path, int set_index, wv_set_info* set, float* extrema) {
  if (!path || !set) return WV_ERR_ARG;
  File fh(path);
  if (!fh.f) return WV_ERR_IO;
  wv_file_info i;
  int st = parse_header(fh, &i);
  if (st != WV_OK) return st;
  if (set_index < 0 || set_index >= i.num_sets) return WV_ERR_ARG;
  return walk_meta(fh, i, set_index, set, extrema);
}

int wv_file_payload_read(const char* path, int set_index, void* buf, uint64_t buf_bytes) {
  if (!buf) return WV_ERR_ARG;
  wv_set_info m;
  int st = wv_file_set_read(path, set_index, &m, nullptr);
  if (st != WV_OK) return st;
  if (buf_bytes < m.payload_length) return WV_ERR_ARG;
  File fh(path);
  if (!fh.seek(m.payload_offset) || !fh.read(buf, m.payload_length)) return WV_ERR_IO;
  return WV_OK;
}

}  // extern "C"
