/*
 * maskmul_mmio — native Matrix Market coordinate reader
 *
 * Replaces the line-by-line Python parser of the reference,
 * read_matrix_market (pkg/src/maskmul/mmio.py:27-101), for the kinds it
 * supports: "%%MatrixMarket matrix coordinate {real|integer|pattern}
 * {general|symmetric}".  Host code only (file text in host memory); the
 * canonical CSR is then built on the device by mm_csr_from_coo
 * (maskmul_b200.h) or on the host by from_arrays.
 *
 * Errors mirror MatrixMarketError (mmio.py:19-24): status MMX_ERR_FORMAT with
 * the offending 1-based line number in *err_line and the message in msg, the
 * same line the reference reports (first failing line in file order).
 * MMX_ERR_OVERFLOW: an integer value outside int64 (the reference raises
 * OverflowError from numpy at mmio.py:88).
 *
 * Line model: lines end at '\n'; '\r' and the other ASCII whitespace
 * characters Python's str.split()/strip() drop (\t \v \f \r \x1c-\x1f, space)
 * separate tokens.  Lone '\r' line breaks (classic Mac files) are not lines.
 */
#ifndef MASKMUL_MMIO_H
#define MASKMUL_MMIO_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { MMX_OK = 0, MMX_ERR_FORMAT = 2, MMX_ERR_OVERFLOW = 5 };
enum { MMX_FIELD_REAL = 0, MMX_FIELD_INTEGER = 1, MMX_FIELD_PATTERN = 2 };

typedef struct {
    int32_t field;       /* MMX_FIELD_* (mmio.py:15) */
    int32_t symmetric;   /* 0 general, 1 symmetric (mmio.py:16) */
    int64_t nrows, ncols, nnz;
    int64_t data_offset; /* byte offset of the first line after the size line */
    int64_t data_line;   /* line number of the size line */
} mmx_header_t;

/* Banner + size line (mmio.py:28-61). */
int mmx_read_header(const char* text, int64_t len, mmx_header_t* h, int64_t* err_line, char* msg,
                    int msg_cap);

/* Entry lines (mmio.py:63-94): rows/cols 0-based int64[nnz]; vals float64[nnz]
 * (real) or int64[nnz] (integer), NULL for pattern (the caller fills ones).
 * nthreads >= 1 host threads parse disjoint line ranges. */
int mmx_read_entries(const char* text, int64_t len, const mmx_header_t* h, int64_t* rows, int64_t* cols,
                     void* vals, int nthreads, int64_t* err_line, char* msg, int msg_cap);

#ifdef __cplusplus
}
#endif

#endif
