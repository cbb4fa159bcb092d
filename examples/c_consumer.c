/* A C-only consumer of the decode library: reads a .wvv header and set
 * directory with the C++ reader, sizes the decode workspace, and (when a
 * GPU is present) decodes one full frame of set 0 through the C ABI.
 *
 *   gcc -std=c11 -I include examples/c_consumer.c \
 *       -L paper_2208_10859_b200 -l:_wvb200.so -Wl,-rpath,paper_2208_10859_b200 -o c_consumer
 *   ./c_consumer tests/golden/smooth_hq.wvv [--decode]
 */
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "wavevid_b200.h"

int main(int argc, char** argv) {
  if (argc < 2) {
    fprintf(stderr, "usage: %s file.wvv\n", argv[0]);
    return 2;
  }
  wv_file_info info;
  int st = wv_file_info_read(argv[1], &info);
  if (st != WV_OK) {
    fprintf(stderr, "wv_file_info_read: %s\n", wv_status_string(st));
    return 1;
  }
  uint64_t ws = 0;
  st = wv_workspace_bytes(&info.geom, &ws);
  printf("%dx%d C%d L%d n%d bs%d frames %d sets %d stereo %d table %llu workspace %llu (%s)\n",
         info.geom.width, info.geom.height, info.geom.channels, info.geom.levels,
         info.geom.inter_size, info.geom.block_size, info.frame_count, info.num_sets,
         info.stereo, (unsigned long long)info.table_bytes, (unsigned long long)ws,
         wv_status_string(st));
  for (int s = 0; s < info.num_sets; ++s) {
    wv_set_info si;
    if ((st = wv_file_set_read(argv[1], s, &si, NULL)) != WV_OK) return 1;
    void* buf = malloc(si.payload_length);
    if (!buf || (st = wv_file_payload_read(argv[1], s, buf, si.payload_length)) != WV_OK) return 1;
    printf("set %d: offset %llu payload %llu records %llu\n", s,
           (unsigned long long)si.payload_offset, (unsigned long long)si.payload_length,
           (unsigned long long)si.record_count);
    free(buf);
  }
  return 0;
}
