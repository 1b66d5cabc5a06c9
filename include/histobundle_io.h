/* histobundle_io.h -- host-side bulk polyline export / import
 * (libhb_io.so; replaces the per-number Python formatting/parsing of the
 * reference's io.export_polylines / io.read_polylines, io.py:136-171).
 *
 * Text format (identical bytes to the reference):
 *   # histobundle polylines v1
 *   # edges <E>
 *   <edge_index> <bin> <weight %.9g> <n> <x0 %.9g> <y0 %.9g> ...   per edge
 * world: packed (N,2) float64 polylines, starts: (E+1) int64 offsets;
 * bins/weights are indexed by the edge's graph index (index[e], or e when
 * index is NULL); NULL bins/weights mean 0 / 1.0.
 */
#ifndef HISTOBUNDLE_IO_H
#define HISTOBUNDLE_IO_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Records [e_lo, e_hi) into buf (capacity cap bytes); stops before the first
 * record that does not fit.  Returns the records written, bytes in *used. */
int64_t hb_io_format(const double *world, const int64_t *starts, const int64_t *bins,
                     const double *weights, const int64_t *index, int64_t e_lo,
                     int64_t e_hi, char *buf, int64_t cap, int64_t *used);

/* Header + all records written to fd in edge order, formatted by `threads`
 * threads.  0 or -errno. */
int hb_io_export_fd(int fd, const double *world, const int64_t *starts,
                    const int64_t *bins, const double *weights, const int64_t *index,
                    int64_t n_edges, int threads);

/* Two-pass parse of an export (fill = 0: count *n_records / *n_coords;
 * fill = 1: write edge_index, bins, weights (n_records), starts
 * (n_records+1) and coords (n_coords)).  0 = ok; 1 = a token only Python's
 * int()/float() accept (caller parses in Python); -1 = malformed record,
 * -2 = coordinate count mismatch (*err_a expected, *err_b found); *err_line
 * is the 1-based line. */
int hb_io_parse(const char *text, int64_t len, int fill, int64_t *n_records,
                int64_t *n_coords, int64_t *edge_index, int64_t *bins, double *weights,
                int64_t *starts, double *coords, int64_t *err_line, int64_t *err_a,
                int64_t *err_b);

#ifdef __cplusplus
}
#endif
#endif
