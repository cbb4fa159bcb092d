// Storage -> host span reads for span-streaming residency (SURVEY.md §8f
// row 1): VideoReader.load_blocks (fileio.py:346-390) restated for a list of
// block ids produced on the GPU.  For every temporal index and every run of
// consecutive block ids the byte span is (end of the previous (t, block)
// entry, end of the run's last block) (block_range_bytes, fileio.py:168-181,
// _id_runs :420-427); spans are sorted and merged through gaps of up to
// COALESCE_GAP = 4096 bytes (_coalesce :264-274) and each merged range is
// one pread into a host buffer that mirrors the set's payload, so the GPU
// finds every record at its file offset.  bytes_read is the io_trace
// figure (read-through slack included), bytes_spans the requested bytes.
//
// wv_span_queue_enqueue runs one read as a stream-ordered host function
// (cudaLaunchHostFunc, capturable in a CUDA graph): the frame's block list,
// written to host memory by the GPU just before, is read from the file while
// the stream waits, and the span fetch kernel that follows copies the bytes
// to HBM.  Jobs are consumed in the order they were pushed, which is the
// stream order of the frames that carry them.
#include <cuda_runtime.h>
#include <unistd.h>

#include <algorithm>
#include <cstring>
#include <vector>

#include "../../include/wavevid_b200.h"

namespace {

int read_spans(const wv_span_job& j, uint64_t* bytes_read, uint64_t* bytes_spans) {
  *bytes_read = *bytes_spans = 0;
  const uint32_t n_ids = *j.count;
  if (n_ids == 0) return WV_OK;
  if (j.n < 1 || j.nb < 1 || n_ids > (uint32_t)j.nb) return WV_ERR_ARG;
  std::vector<uint32_t> ids(j.ids, j.ids + n_ids);
  std::sort(ids.begin(), ids.end());
  ids.erase(std::unique(ids.begin(), ids.end()), ids.end());
  if (ids.back() >= (uint32_t)j.nb) return WV_ERR_ARG;
  // runs of consecutive ids
  std::vector<std::pair<uint32_t, uint32_t>> runs;
  for (size_t i = 0; i < ids.size();) {
    size_t e = i;
    while (e + 1 < ids.size() && ids[e + 1] == ids[e] + 1) ++e;
    runs.emplace_back(ids[i], ids[e]);
    i = e + 1;
  }
  // spans in payload coordinates (after the BlockEnd table)
  const uint64_t tb = j.table_bytes;
  std::vector<std::pair<uint64_t, uint64_t>> spans;
  spans.reserve(runs.size() * j.n);
  for (int t = 0; t < j.n; ++t)
    for (const auto& r : runs) {
      const uint64_t si = (uint64_t)t * j.nb + r.first, ei = (uint64_t)t * j.nb + r.second;
      const uint64_t st = si ? j.table[si - 1] : 0, en = j.table[ei];
      if (en < st || tb + en > j.payload_bytes) return WV_ERR_FORMAT;
      if (en > st) spans.emplace_back(tb + st, tb + en);
      *bytes_spans += en - st;
    }
  std::sort(spans.begin(), spans.end());
  auto merge = [&](const std::vector<std::pair<uint64_t, uint64_t>>& in) {
    std::vector<std::pair<uint64_t, uint64_t>> out;
    for (const auto& s : in) {
      if (!out.empty() && s.first <= out.back().second + j.coalesce_gap)
        out.back().second = std::max(out.back().second, s.second);
      else
        out.push_back(s);
    }
    return out;
  };
  // the io_trace figure: the reference's coalesced reads of the exact spans
  for (const auto& m : merge(spans)) *bytes_read += m.second - m.first;
  // the reads themselves cover whole 16-byte payload chunks, because the
  // fetch kernel copies 16-byte chunks: every chunk a span touches holds
  // file bytes in the host buffer
  std::vector<std::pair<uint64_t, uint64_t>> aligned;
  aligned.reserve(spans.size());
  for (const auto& s : spans)
    aligned.emplace_back(s.first & ~uint64_t(15), std::min((s.second + 15) & ~uint64_t(15),
                                                           j.payload_bytes));
  for (const auto& m : merge(aligned)) {
    uint64_t off = m.first;
    while (off < m.second) {
      const ssize_t got = pread(j.fd, j.dst + off, (size_t)(m.second - off),
                                (off_t)(j.payload_offset + off));
      if (got <= 0) return WV_ERR_IO;
      off += (uint64_t)got;
    }
  }
  return WV_OK;
}

void CUDART_CB run_next_job(void* user) {
  wv_span_queue* q = static_cast<wv_span_queue*>(user);
  const uint32_t h = __atomic_load_n(&q->head, __ATOMIC_RELAXED);
  if (h == __atomic_load_n(&q->tail, __ATOMIC_ACQUIRE)) return;   // no job: nothing to read
  wv_span_job& j = q->jobs[q->fifo[h % WV_SPAN_QUEUE]];
  j.status = read_spans(j, &j.bytes_read, &j.bytes_spans);
  __atomic_store_n(&j.done, 1, __ATOMIC_RELEASE);
  __atomic_store_n(&q->head, h + 1, __ATOMIC_RELEASE);
}

}  // namespace

extern "C" {

int wv_spans_read(const wv_span_job* job, uint64_t* bytes_read, uint64_t* bytes_spans) {
  if (!job || !bytes_read || !bytes_spans || !job->table || !job->dst || !job->ids ||
      !job->count)
    return WV_ERR_ARG;
  return read_spans(*job, bytes_read, bytes_spans);
}

int wv_span_queue_push(wv_span_queue* q, const wv_span_job* job, uint32_t slot) {
  if (!q || !job || slot >= WV_SPAN_QUEUE) return WV_ERR_ARG;
  const uint32_t t = __atomic_load_n(&q->tail, __ATOMIC_RELAXED);
  if (t - __atomic_load_n(&q->head, __ATOMIC_ACQUIRE) >= WV_SPAN_QUEUE) return WV_ERR_ARG;   // full
  q->jobs[slot] = *job;
  q->jobs[slot].done = 0;
  q->jobs[slot].status = 0;
  q->fifo[t % WV_SPAN_QUEUE] = slot;
  __atomic_store_n(&q->tail, t + 1, __ATOMIC_RELEASE);
  return WV_OK;
}

int wv_span_queue_enqueue(wv_span_queue* q, void* stream) {
  if (!q) return WV_ERR_ARG;
  return cudaLaunchHostFunc((cudaStream_t)stream, run_next_job, q) == cudaSuccess ? WV_OK
                                                                                   : WV_ERR_CUDA;
}

}  // extern "C"
