/*
 * bmatch_b200_io.h — graph files on the host: Matrix Market ingest/export
 * and a binary CSC container. Not on the
 * matching hot path; this is the step before bm_upload_csc.
 *
 * Matrix Market. bm_mm_load is a drop-in for the reference's
 * load_matrix_market / read_matrix_market (matrix_market.cpp:29-108): the same
 * accepted headers (coordinate; pattern|real|integer; general|symmetric, with
 * symmetric off-diagonal entries mirrored), the same 1-based -> 0-based
 * transcription (matrix rows -> row vertices, matrix columns -> column
 * vertices), the same sorted, de-duplicated CSC as from_edge_list
 * (csr_graph.cpp:10-43), and the same errors: BM_ERR_PARSE with the
 * reference's message and 1-based line number (*err_line) for anything
 * read_matrix_market rejects, BM_ERR_INVALID_ARG for what from_edge_list
 * rejects (a mirrored entry outside a non-square matrix), BM_ERR_IO when the
 * file cannot be opened. The file is memory-mapped and parsed by every host
 * core (the reference parses one line at a time through iostreams).
 * bm_mm_write emits exactly the bytes of write_matrix_market
 * (matrix_market.cpp:111-118), formatted in parallel.
 *
 * Binary CSC ("BMCSC001"): a 40-byte header {char magic[8]; int32 nc, nr;
 * int64 nedges; uint64 checksum; uint64 reserved} followed by cxadj[nc+1]
 * (int64, little-endian) and cadj[nedges] (int32). The checksum covers both
 * arrays; bm_csc_read verifies it and the CSC invariants (check_csr,
 * csr_graph.cpp:45-64) before returning. Reads and writes are parallel.
 *
 * Protocol as in bmatch_b200_gen.h: *_info first to size the caller's
 * cxadj[nc+1] / cadj[capacity]; `threads` <= 0 uses every host core.
 * err_line may be NULL.
 */
#ifndef BMATCH_B200_IO_H
#define BMATCH_B200_IO_H

#include <stdint.h>

#include "bmatch_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct bm_mm_header {
  int32_t nrows;     /* matrix rows    = row vertices (nr)    */
  int32_t ncols;     /* matrix columns = column vertices (nc) */
  int64_t entries;   /* declared entry count */
  int32_t symmetric; /* 1: off-diagonal entries are mirrored */
  int32_t field;     /* 0 pattern, 1 real, 2 integer (values are discarded) */
  int64_t capacity;  /* cadj elements bm_mm_load needs before de-duplication */
} bm_mm_header;

bm_status bm_mm_info(const char* path, bm_mm_header* header, int64_t* err_line);
bm_status bm_mm_load(const char* path, int32_t threads, int64_t capacity, int64_t* cxadj, int32_t* cadj,
                     int64_t* nedges, int64_t* err_line);
/* Same, from a memory buffer (read_matrix_market on a stream). */
bm_status bm_mm_parse_info(const char* text, int64_t length, bm_mm_header* header, int64_t* err_line);
bm_status bm_mm_parse(const char* text, int64_t length, int32_t threads, int64_t capacity, int64_t* cxadj,
                      int32_t* cadj, int64_t* nedges, int64_t* err_line);
bm_status bm_mm_write(const char* path, int32_t nc, int32_t nr, const int64_t* cxadj, const int32_t* cadj,
                      int32_t threads);

bm_status bm_csc_write(const char* path, int32_t nc, int32_t nr, const int64_t* cxadj, const int32_t* cadj,
                       int32_t threads);
bm_status bm_csc_info(const char* path, int32_t* nc, int32_t* nr, int64_t* nedges);
bm_status bm_csc_read(const char* path, int32_t threads, int64_t capacity, int64_t* cxadj, int32_t* cadj);

#ifdef __cplusplus
}
#endif

#endif /* BMATCH_B200_IO_H */
