/*
 * lmdtw_b200.h -- C ABI of the B200-native exact linear-memory DTW library
 * (liblmdtw_b200.so).  Plain pointers and sizes only; no torch types.
 *
 * Each entry point replaces one function of the reference package `lmdtw`
 * (paths relative to /root/reference/pkg/src/lmdtw):
 *
 *   lmdtw_half_pass   == diagonal.diag_dtw      (diagonal.py:172-223,
 *                        kernel _advance         diagonal.py:74-122)
 *   lmdtw_find_pivot  == divide.find_pivot      (divide.py:97-145)
 *   lmdtw_dtw_full    == oracle.dtw_full        (oracle.py:105-131, with
 *                        _dtw_fill oracle.py:40-82 and backtrace :85-102);
 *                        with D_out != NULL also accumulated_cost_table
 *                        (oracle.py:134-141)
 *   lmdtw_align       == divide.linmdtw         (divide.py:181-213, recursion
 *                        _solve :148-178, final cost core.path_cost
 *                        core.py:182-197)
 *   lmdtw_align_batch == many independent linmdtw calls fused level by level
 *   lmdtw_path_cost   == core.path_cost         (core.py:182-197)
 *
 * Building blocks of the multi-GPU recursion (paper_2008_02734_b200/
 * distributed.py): one recursion level's find_pivot calls on sub-blocks
 * (lmdtw_pivot_nodes == divide.find_pivot on X.view/Y.view, divide.py:158-167),
 * the leaf dtw_full calls (lmdtw_leaf_nodes == divide._solve's leaf branch,
 * divide.py:153-157), and the split-point combine of two half passes computed
 * on different GPUs (lmdtw_pivot_combine == divide.py:122-145).
 *
 * Memory: every entry takes `mem`: LMDTW_MEM_HOST means X/Y/outputs are host
 * pointers (the library stages them through pinned memory, copies included in
 * the call); LMDTW_MEM_DEVICE means X/Y are device pointers on `device`
 * (float32, row-major, C-contiguous) and outputs are still host pointers
 * unless stated otherwise.  Features are always float32 in storage, as in
 * the reference (core.py:35); accumulation dtype is `precision` (32 or 64).
 *
 * Errors: every int-returning entry returns LMDTW_OK (0) or a negative status;
 * lmdtw_last_error() returns a thread-local message for the last failure.
 * The Python layer maps EINVAL -> InvalidInputError, ENOMEM -> MemoryError,
 * ECUDA/EINTERNAL -> RuntimeError, the reference's exception classes.
 *
 * Threading: reentrant.  Calls on the same device serialise on a per-device
 * workspace mutex; calls on different devices run concurrently.  The
 * progress callback runs on the calling thread between recursion levels.
 */
#ifndef LMDTW_B200_H
#define LMDTW_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LMDTW_OK 0
#define LMDTW_EINVAL (-1)
#define LMDTW_ENOMEM (-2)
#define LMDTW_ECUDA (-3)
#define LMDTW_EINTERNAL (-4)

#define LMDTW_MEM_HOST 0
#define LMDTW_MEM_DEVICE 1

/* Backpointer / move codes (oracle.py:23). */
#define LMDTW_LEFT 0
#define LMDTW_UP 1
#define LMDTW_DIAG 2
#define LMDTW_SELF 3

/* LinMdtwConfig (divide.py:44-57). */
typedef struct {
    int32_t min_dim;        /* >= 2; default 500 */
    int32_t precision;      /* 32 or 64; default 64 */
    int32_t tie[3];         /* move precedence codes, default {DIAG, LEFT, UP} */
    int32_t pivot_highest;  /* 0 = "lowest" (default), 1 = "highest" */
    int32_t reserved[4];
} lmdtw_config_t;

/* One entry of AlignmentResult.pivot_trace (divide.py:160-164). */
typedef struct {
    int64_t i, j, i_off, j_off, M, N, sub_i, sub_j, diagonal_k;
    double total_at_pivot;
} lmdtw_pivot_t;

/* Scalar fields of AlignmentResult (core.py:133-155) plus run statistics. */
typedef struct {
    double cost;
    int64_t path_len;
    int64_t cells_processed;
    int64_t cells_budget;
    int64_t peak_diag_values;
    int64_t peak_table_cells;
    int64_t n_pivots;
    int64_t n_levels;
    int64_t gpu_launches;      /* kernels this call launched */
    int64_t h2d_bytes, d2h_bytes;
} lmdtw_align_info_t;

/* progress(cells_done, budget=2MN, user): divide.py:73-82 cadence. */
typedef void (*lmdtw_progress_fn)(int64_t done, int64_t budget, void *user);

/* Opaque result of lmdtw_align; read with the accessors, free with _free. */
typedef struct lmdtw_result lmdtw_result_t;

const char *lmdtw_version(void);
const char *lmdtw_last_error(void);
int lmdtw_device_count(void);
/* Largest feature dimension the kernels accept for a precision. */
int lmdtw_max_dim(int32_t precision);

/* diag_dtw: run diagonals 0..kstop of the (optionally reversed) grid and
 * return the last three accumulated (out_d) and raw (out_c) diagonals,
 * k = kstop-2+s in slot s, each of length diag_length(k,M,N), as `precision`
 * floats into HOST buffers.  *cells = sum_{k<=kstop} L(k). */
int lmdtw_half_pass(int device, const float *X, int64_t M, const float *Y, int64_t N,
                    int32_t d, int64_t kstop, int32_t reverse, int32_t precision,
                    int32_t mem, void *out_d[3], void *out_c[3], int64_t *cells);

/* find_pivot: forward pass to ceil((M+N-1)/2), reverse pass to the matching
 * diagonal, combine (Df + Db) - Cf on the three shared diagonals and take the
 * lexicographic argmin.  Writes (i, j, diagonal_k), total, cells, peak. */
int lmdtw_find_pivot(int device, const float *X, int64_t M, const float *Y, int64_t N,
                     int32_t d, int32_t precision, int32_t pivot_highest, int32_t mem,
                     int64_t *i, int64_t *j, int64_t *diagonal_k, double *total,
                     int64_t *cells, int64_t *peak);

/* dtw_full: textbook DP with backpointers (tie precedence `tie`, strict <) and
 * a backtrace from (M-1,N-1).  path_out holds >= M+N-1 (i,j) int64 pairs;
 * *path_len receives K.  *cost = D[M-1,N-1].  If D_out != NULL it receives
 * the full M*N accumulated-cost table (host, `precision` floats). */
int lmdtw_dtw_full(int device, const float *X, int64_t M, const float *Y, int64_t N,
                   int32_t d, const int32_t tie[3], int32_t precision, int32_t mem,
                   double *cost, int64_t *path_out, int64_t *path_len, void *D_out);

/* linmdtw: the whole divide-and-conquer recursion on the device, one batched
 * launch per recursion level, leaves solved by the batched textbook solver,
 * cost = sequential path_cost in `precision`. */
int lmdtw_align(int device, const float *X, int64_t M, const float *Y, int64_t N, int32_t d,
                const lmdtw_config_t *cfg, int32_t mem, lmdtw_progress_fn progress,
                void *user, lmdtw_result_t **result);

/* Many independent alignments (pairs p: X[p] M[p] x Y[p] N[p], same d and
 * config) fused: every recursion level of every pair shares one launch. */
int lmdtw_align_batch(int device, int32_t npairs, const float *const *X, const int64_t *M,
                      const float *const *Y, const int64_t *N, int32_t d,
                      const lmdtw_config_t *cfg, int32_t mem, lmdtw_result_t **results);

/* find_pivot on n sub-blocks sub[4q..4q+3] = (i_off, j_off, Mq, Nq) of X x Y
 * in one batched launch: out[5q..5q+4] = (i, j, diagonal_k, cells, peak) in
 * sub-block coordinates, totals[q] = total_at_pivot. */
int lmdtw_pivot_nodes(int device, const float *X, int64_t M, const float *Y, int64_t N, int32_t d,
                      int32_t n, const int64_t *sub, int32_t precision, int32_t pivot_highest,
                      int32_t mem, int64_t *out, double *totals);

/* dtw_full on n sub-blocks in one batched launch: the local paths (forward
 * order, sub-block coordinates) are concatenated into path_out (room for
 * sum(Mq + Nq - 1) (i,j) int64 pairs), path_len[q] = Kq. */
int lmdtw_leaf_nodes(int device, const float *X, int64_t M, const float *Y, int64_t N, int32_t d,
                     int32_t n, const int64_t *sub, const int32_t tie[3], int32_t precision,
                     int32_t mem, int64_t *path_out, int64_t *path_len);

/* Split point from a forward and a reverse half pass computed elsewhere (host
 * buffers from lmdtw_half_pass: fwd to kf = ceil((M+N-1)/2), reverse to kb):
 * (Df + Db[idx_b]) - Cf with the lexicographic (value, k, idx) argmin
 * ("lowest") or (value, -k, -idx) ("highest").  ijk = (i, j, diagonal_k). */
int lmdtw_pivot_combine(int32_t precision, int64_t M, int64_t N, int32_t pivot_highest,
                        const void *const fwd_d[3], const void *const fwd_c[3],
                        const void *const bwd_d[3], int64_t *ijk, double *total);

/* The same combine on `device` (pivot_kernel): the nine diagonals may be
 * device pointers (e.g. NCCL all-gather outputs; lmdtw_half_pass and
 * lmdtw_half_pass_shard accept device output pointers) or host pointers.
 * Bit-identical to lmdtw_pivot_combine. */
int lmdtw_pivot_combine_device(int device, int32_t precision, int64_t M, int64_t N, int32_t pivot_highest,
                               const void *const fwd_d[3], const void *const fwd_c[3],
                               const void *const bwd_d[3], int64_t *ijk, double *total);

/* One shard of a half pass for the multi-GPU layout: strips
 * [strip_lo, strip_hi) of diag_dtw(X, Y, kstop, reverse), strips being
 * lmdtw_strip_height() grid rows.  bnd_local: caller-owned device buffer of
 * lmdtw_handoff_words(N) 64-bit words, set to all ones before ANY shard of the
 * pass starts; this shard's strips publish their bottom rows there.  bnd_prev:
 * the previous shard's bnd_local (a peer GPU's memory mapped with CUDA IPC),
 * NULL for strip_lo = 0; read with system-scope loads.  The entries of the last
 * three diagonals that belong to rows [strip_lo H, strip_hi H) are written to
 * the host buffers (other entries untouched); *cells = the shard's cells. */
int lmdtw_half_pass_shard(int device, const float *X, int64_t M, const float *Y, int64_t N, int32_t d,
                          int64_t kstop, int32_t reverse, int32_t precision, int32_t mem, int32_t strip_lo,
                          int32_t strip_hi, void *bnd_local, const void *bnd_prev, void *out_d[3],
                          void *out_c[3], int64_t *cells);
int64_t lmdtw_handoff_words(int64_t N, int32_t precision);
/* Handoff buffers shared between the processes of a sharded pass (CUDA IPC):
 * allocate + export a 64-byte handle, open a peer's handle (peer access
 * enabled), close, free, and set every byte to 0xFF (synchronously). */
int lmdtw_ipc_alloc(int device, int64_t bytes, void **ptr, unsigned char handle[64]);
int lmdtw_ipc_open(int device, const unsigned char handle[64], void **ptr);
int lmdtw_ipc_close(int device, void *ptr);
int lmdtw_ipc_free(int device, void *ptr);
int lmdtw_fill_ones(int device, void *ptr, int64_t bytes);
int32_t lmdtw_strip_height(int32_t precision, int32_t d);

int lmdtw_result_info(const lmdtw_result_t *r, lmdtw_align_info_t *info);
/* Copies K (i,j) int64 pairs. */
int lmdtw_result_path(const lmdtw_result_t *r, int64_t *path_out);
/* Copies n_pivots entries in pre-order DFS (divide.py:160-175). */
int lmdtw_result_pivots(const lmdtw_result_t *r, lmdtw_pivot_t *pivots_out);
void lmdtw_result_free(lmdtw_result_t *r);

/* path_cost on host data: costs in `precision`, summed sequentially from 0. */
int lmdtw_path_cost(const float *X, int64_t M, const float *Y, int64_t N, int32_t d,
                    const int64_t *path, int64_t K, int32_t precision, double *cost);

/* Closed forms used by the instrumentation (diagonal.py:29-33, :160-169). */
int64_t lmdtw_diag_length(int64_t k, int64_t M, int64_t N);
int64_t lmdtw_cells_upto(int64_t kstop, int64_t M, int64_t N);
int64_t lmdtw_peak_retained_values(int64_t kstop, int64_t M, int64_t N);

/* Library-wide statistics: total kernels launched since load (for bench). */
int64_t lmdtw_launch_count(void);

/* ---- per-path steps either side of the aligner ---------- */

/* approx.constrained_dtw (approx.py:180-220; fill _window_fill :130-177):
 * optimal path among those inside the monotone staircase window
 * lo[i] <= j <= hi[i] (M entries each, validated as approx.Window.validate,
 * approx.py:52-63: EINVAL with the reference's messages).  path_out holds
 * M+N-1 (i, j) pairs; *cells = window size (cells_processed).  A backtrace
 * that meets SELF before (0, 0) returns EINTERNAL ("backtrace escaped the
 * window"), the reference's RuntimeError. */
int lmdtw_window_dtw(int device, const float *X, int64_t M, const float *Y, int64_t N, int32_t d,
                     const int64_t *lo, const int64_t *hi, const int32_t tie[3], int32_t precision,
                     int32_t mem, double *cost, int64_t *path_out, int64_t *path_len, int64_t *cells);

/* core.frame_costs (core.py:167-179): out[q] = cost(A[q], B[q]) in
 * `precision` (out is a host array of K floats or doubles). */
int lmdtw_frame_costs(int device, const float *A, const float *B, int64_t K, int32_t d,
                      int32_t precision, int32_t mem, void *out);

/* core.path_cost (core.py:182-197) for npaths (X, Y, path) triples at once:
 * per-cell costs in parallel, each path's sequential sum from 0 in
 * `precision`; costs_out[p] as double.  X/Y per `mem`, paths on the host. */
int lmdtw_path_cost_batch(int device, int32_t npaths, const float *const *X, const int64_t *M,
                          const float *const *Y, const int64_t *N, int32_t d,
                          const int64_t *const *paths, const int64_t *K, int32_t precision,
                          int32_t mem, double *costs_out);

/* metrics.discrepancy (metrics.py:44-63): errors_out[0..K1) row errors and
 * errors_out[K1..2K1) column errors of path p1 against p2 (host arrays of
 * (i, j) int64 pairs); EINVAL on mismatched endpoints. */
int lmdtw_discrepancy(int device, const int64_t *p1, int64_t K1, const int64_t *p2, int64_t K2,
                      int64_t *errors_out);

#ifdef __cplusplus
}
#endif
#endif /* LMDTW_B200_H */
