/*
 * lmdtw_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference's exact linear-memory DTW path
 * (arXiv 2008.02734, package `lmdtw` under /root/reference/pkg/src/lmdtw).
 * It is the checker for the CUDA product path and the CPU baseline leg of
 * bench.py.  Nothing in paper_2008_02734_b200/ may link or call it.
 *
 * Parity pin: tests/test_oracle_golden.py checks every function here against
 * golden vectors produced by the real reference (tests/golden/make_golden.py).
 *
 * Arithmetic contract (follows the reference's numba codegen, which has no
 * FMA contraction and uses a correctly rounded sqrt):
 *   cost(i,j) = sqrt( (((0 + d0*d0) + d1*d1) + ...) ),  d_t = x_t - y_t,
 *   each operation rounded in the accumulation dtype T (float or double).
 * Build with -ffp-contract=off (see oracle/Makefile).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

#define LMIN(a, b) ((a) < (b) ? (a) : (b))
#define LMAX(a, b) ((a) > (b) ? (a) : (b))

/* diagonal.py:29-33 */
int64_t orc_diag_length(int64_t k, int64_t M, int64_t N) {
    if (k < 0 || k > M + N - 2) return 0;
    int64_t v = LMIN(LMIN(k, M - 1), LMIN(N - 1, M + N - 2 - k));
    return v + 1;
}

/* diagonal.py:160-169 (closed loop form; O(kstop)) */
int64_t orc_peak_retained_values(int64_t kstop, int64_t M, int64_t N) {
    int64_t peak = 0;
    for (int64_t k = 0; k <= kstop; k++) {
        int64_t w = 0;
        for (int64_t kk = k - 2; kk <= k; kk++)
            if (kk >= 0 && kk <= M + N - 2) w += orc_diag_length(kk, M, N);
        if (2 * w > peak) peak = 2 * w;
    }
    return peak;
}

/* oracle.py:23 */
enum { ORC_LEFT = 0, ORC_UP = 1, ORC_DIAG = 2, ORC_SELF = 3 };

typedef struct {
    int64_t i, j, i_off, j_off, M, N, sub_i, sub_j, diagonal_k;
    double total_at_pivot;
} orc_pivot_t;

typedef struct {
    int min_dim;
    int tie[3];
    int pivot_highest;   /* 0 = "lowest", 1 = "highest" */
} orc_cfg_t;

typedef struct {
    int64_t cells;
    int64_t peak_diag_values;
    int64_t peak_table_cells;
    orc_pivot_t *pivots;
    int64_t npivots, cap_pivots;
} orc_inst_t;

static void inst_add_pivot(orc_inst_t *st, const orc_pivot_t *p) {
#ifdef _OPENMP
#pragma omp critical(orc_pivots)
#endif
    {
        if (st->npivots == st->cap_pivots) {
            st->cap_pivots = st->cap_pivots ? 2 * st->cap_pivots : 64;
            st->pivots = (orc_pivot_t *)realloc(st->pivots, st->cap_pivots * sizeof(orc_pivot_t));
        }
        st->pivots[st->npivots++] = *p;
    }
}

/* ------------------------------------------------------------------ */
/* Type-generic body, instantiated for float (f32) and double (f64).   */
/* ------------------------------------------------------------------ */
#define ORC_DEFINE(T, SFX, SQRT)                                                          \
                                                                                          \
/* Cell cost (diagonal.py:99-103, oracle.py:50-54): sequential, no FMA. */                \
static inline T cost_##SFX(const float *x, const float *y, int d) {                     \
    T s = (T)0;                                                                           \
    for (int t = 0; t < d; t++) {                                                         \
        T diff = (T)x[t] - (T)y[t];                                                       \
        T sq = diff * diff;                                                               \
        s = s + sq;                                                                       \
    }                                                                                     \
    return SQRT(s);                                                                       \
}                                                                                         \
                                                                                          \
/* Half pass (diag_dtw, diagonal.py:172-223 with _advance :74-122).                  */   \
/* X rows xs[0..M), Y rows ys[0..N) are addressed via strides so reversed views      */   \
/* (negative stride) need no copy. Outputs: out_d[s], out_c[s] for k=kstop-2+s,      */   \
/* lengths L(k).  Returns cells processed.                                           */   \
int64_t orc_half_pass_##SFX(const float *X, int64_t xstride, const float *Y,             \
                            int64_t ystride, int64_t M, int64_t N, int d, int64_t kstop,  \
                            T *out_d[3], T *out_c[3]) {                                   \
    int64_t Lmax = LMIN(M, N);                                                            \
    T *bufD[3], *bufC[3];                                                                 \
    for (int s = 0; s < 3; s++) {                                                         \
        bufD[s] = (T *)malloc(sizeof(T) * (Lmax + 1));                                    \
        bufC[s] = (T *)malloc(sizeof(T) * (Lmax + 1));                                    \
    }                                                                                     \
    /* rotating: slot for k is k % 3 */                                                   \
    int64_t cells = 0;                                                                    \
    for (int64_t k = 0; k <= kstop; k++) {                                                \
        int64_t L = orc_diag_length(k, M, N);                                             \
        T *D2 = bufD[k % 3], *C2 = bufC[k % 3];                                           \
        const T *Dm1 = bufD[(k + 2) % 3], *Dm2 = bufD[(k + 1) % 3];                       \
        int64_t i0 = LMIN(k, M - 1), i0m1 = LMIN(k - 1, M - 1), i0m2 = LMIN(k - 2, M - 1); \
        /* cells of one diagonal are independent: long diagonals are split    */         \
        /* into tasks (inside the linmdtw parallel region); results never     */         \
        /* depend on the thread count                                         */         \
        _Pragma("omp taskloop grainsize(4096) if(L >= 16384)")                            \
        for (int64_t idx = 0; idx < L; idx++) {                                           \
            int64_t i = i0 - idx, j = k - i;                                              \
            T c = cost_##SFX(X + i * xstride, Y + j * ystride, d);                         \
            C2[idx] = c;                                                                  \
            if (k == 0) { D2[idx] = c; continue; }                                        \
            T best = (T)0;                                                                \
            int have = 0;                                                                 \
            if (j > 0) { best = Dm1[i0m1 - i]; have = 1; }                                \
            if (i > 0) {                                                                  \
                T v = Dm1[i0m1 - (i - 1)];                                                \
                if (!have || v < best) best = v;                                          \
            }                                                                             \
            if (i > 0 && j > 0) {                                                         \
                T v = Dm2[i0m2 - (i - 1)];                                                \
                if (v < best) best = v;                                                   \
            }                                                                             \
            D2[idx] = best + c;                                                           \
        }                                                                                 \
        cells += L;                                                                       \
        if (k >= kstop - 2) {                                                             \
            int s = (int)(k - (kstop - 2));                                               \
            memcpy(out_d[s], D2, sizeof(T) * L);                                          \
            memcpy(out_c[s], C2, sizeof(T) * L);                                          \
        }                                                                                 \
    }                                                                                     \
    for (int s = 0; s < 3; s++) { free(bufD[s]); free(bufC[s]); }                         \
    return cells;                                                                         \
}                                                                                         \
                                                                                          \
/* Full table fill (_dtw_fill, oracle.py:40-82). D, P are M*N row-major; D may be NULL  */ \
/* only if the caller just wants P; here both are required.                          */   \
void orc_dtw_fill_##SFX(const float *X, int64_t xstride, const float *Y, int64_t ystride,  \
                        int64_t M, int64_t N, int d, const int tie[3], T *D, uint8_t *P) { \
    for (int64_t i = 0; i < M; i++) {                                                     \
        for (int64_t j = 0; j < N; j++) {                                                 \
            T c = cost_##SFX(X + i * xstride, Y + j * ystride, d);                         \
            if (i == 0 && j == 0) { D[0] = c; P[0] = ORC_SELF; continue; }                \
            T best = (T)0; int have = 0; int move = ORC_SELF;                             \
            for (int m = 0; m < 3; m++) {                                                 \
                int code = tie[m]; T v;                                                   \
                if (code == ORC_LEFT) { if (j == 0) continue; v = D[i * N + j - 1]; }     \
                else if (code == ORC_UP) { if (i == 0) continue; v = D[(i - 1) * N + j]; } \
                else { if (i == 0 || j == 0) continue; v = D[(i - 1) * N + j - 1]; }      \
                if (!have || v < best) { best = v; move = code; have = 1; }               \
            }                                                                             \
            D[i * N + j] = best + c;                                                      \
            P[i * N + j] = (uint8_t)move;                                                 \
        }                                                                                 \
    }                                                                                     \
}                                                                                         \
                                                                                          \
/* dtw_full (oracle.py:105-131) + backtrace (oracle.py:85-102).  path must hold M+N-1   */ \
/* pairs. Returns path length, or -1 on SELF-before-origin, -2 on OOM.              */    \
int64_t orc_dtw_full_##SFX(const float *X, int64_t xstride, const float *Y,               \
                           int64_t ystride, int64_t M, int64_t N, int d, const int tie[3], \
                           double *cost_out, int64_t *path) {                             \
    T *D = (T *)malloc(sizeof(T) * M * N);                                                \
    uint8_t *P = (uint8_t *)malloc((size_t)(M * N));                                      \
    if (!D || !P) { free(D); free(P); return -2; }                                        \
    orc_dtw_fill_##SFX(X, xstride, Y, ystride, M, N, d, tie, D, P);                       \
    if (cost_out) *cost_out = (double)D[M * N - 1];                                       \
    int64_t i = M - 1, j = N - 1, n = 0;                                                  \
    int64_t cap = M + N - 1;                                                              \
    path[2 * n] = i; path[2 * n + 1] = j; n++;                                            \
    while (!(i == 0 && j == 0)) {                                                         \
        int mv = P[i * N + j];                                                            \
        if (mv == ORC_LEFT) j -= 1;                                                       \
        else if (mv == ORC_UP) i -= 1;                                                    \
        else if (mv == ORC_DIAG) { i -= 1; j -= 1; }                                      \
        else { free(D); free(P); return -1; }                                             \
        if (n >= cap) { free(D); free(P); return -1; }                                    \
        path[2 * n] = i; path[2 * n + 1] = j; n++;                                        \
    }                                                                                     \
    /* reverse in place */                                                                \
    for (int64_t a = 0, b = n - 1; a < b; a++, b--) {                                     \
        int64_t ti = path[2 * a], tj = path[2 * a + 1];                                   \
        path[2 * a] = path[2 * b]; path[2 * a + 1] = path[2 * b + 1];                     \
        path[2 * b] = ti; path[2 * b + 1] = tj;                                           \
    }                                                                                     \
    free(D); free(P);                                                                     \
    return n;                                                                             \
}                                                                                         \
                                                                                          \
/* find_pivot (divide.py:97-145).  Returns 0, or -1 if too small.                    */   \
int orc_find_pivot_##SFX(const float *X, const float *Y, int64_t M, int64_t N, int d,     \
                         int highest, int64_t *pi, int64_t *pj, double *total_out,        \
                         int64_t *k_out, int64_t *cells_out, int64_t *peak_out) {        \
    if (M + N - 2 < 2) return -1;                                                         \
    int64_t K = M + N - 1;                                                                \
    int64_t kf = (K + 1) / 2;                                                             \
    int64_t kb = (K % 2 == 0) ? kf + 1 : kf;                                              \
    T *fd[3], *fc[3], *bd[3], *bc[3];                                                     \
    for (int s = 0; s < 3; s++) {                                                         \
        int64_t Lf = orc_diag_length(kf - 2 + s, M, N), Lb = orc_diag_length(kb - 2 + s, M, N); \
        fd[s] = (T *)malloc(sizeof(T) * (Lf + 1)); fc[s] = (T *)malloc(sizeof(T) * (Lf + 1)); \
        bd[s] = (T *)malloc(sizeof(T) * (Lb + 1)); bc[s] = (T *)malloc(sizeof(T) * (Lb + 1)); \
    }                                                                                     \
    int64_t cf = 0, cb = 0;                                                               \
    int64_t d64 = d;                                                                      \
    _Pragma("omp task shared(cf)")                                                        \
    cf = orc_half_pass_##SFX(X, d64, Y, d64, M, N, d, kf, fd, fc);                        \
    _Pragma("omp task shared(cb)")                                                        \
    cb = orc_half_pass_##SFX(X + (M - 1) * d64, -d64, Y + (N - 1) * d64, -d64, M, N, d, kb, bd, bc); \
    _Pragma("omp taskwait")                                                               \
    if (cells_out) *cells_out = cf + cb;                                                  \
    if (peak_out) {                                                                       \
        int64_t p1 = orc_peak_retained_values(kf, M, N), p2 = orc_peak_retained_values(kb, M, N); \
        *peak_out = LMAX(p1, p2);                                                         \
    }                                                                                     \
    int have = 0; T bt = 0; int64_t bk = 0, bidx = 0;                                     \
    for (int m = 0; m < 3; m++) {                                                         \
        int64_t k = kf - 2 + m;                                                           \
        int64_t L = orc_diag_length(k, M, N);                                             \
        const T *df = fd[m], *cfv = fc[m], *db = bd[2 - m];                               \
        int64_t i0 = LMIN(k, M - 1), ib0 = LMIN(M + N - 2 - k, M - 1);                    \
        /* first argmin in (possibly reversed) order: np.argmin semantics */             \
        int cand_have = 0; T ct = 0; int64_t cidx = 0;                                    \
        for (int64_t q = 0; q < L; q++) {                                                 \
            int64_t idx = highest ? (L - 1 - q) : q;                                      \
            int64_t i = i0 - idx;                                                         \
            int64_t idx_b = ib0 - (M - 1 - i);                                            \
            T tot = df[idx] + db[idx_b];                                                  \
            tot = tot - cfv[idx];                                                         \
            if (!cand_have || tot < ct) { ct = tot; cidx = idx; cand_have = 1; }          \
        }                                                                                 \
        if (!have) { bt = ct; bk = k; bidx = cidx; have = 1; }                            \
        else if (!highest) { if ((double)ct < (double)bt) { bt = ct; bk = k; bidx = cidx; } } \
        else { if ((double)ct <= (double)bt) { bt = ct; bk = k; bidx = cidx; } }          \
    }                                                                                     \
    int64_t i = LMIN(bk, M - 1) - bidx;                                                   \
    *pi = i; *pj = bk - i; *total_out = (double)bt; *k_out = bk;                          \
    for (int s = 0; s < 3; s++) { free(fd[s]); free(fc[s]); free(bd[s]); free(bc[s]); }   \
    return 0;                                                                             \
}                                                                                         \
                                                                                          \
/* _solve (divide.py:148-178): returns path length written at path (caller sized M+N-1). */ \
static int64_t solve_##SFX(const float *X, const float *Y, int64_t M, int64_t N, int d,   \
                           const orc_cfg_t *cfg, orc_inst_t *st, int64_t i_off,          \
                           int64_t j_off, int64_t *path, int depth) {                     \
    if (M < cfg->min_dim || N < cfg->min_dim || M + N <= 5) {                             \
        double c;                                                                         \
        int64_t n = orc_dtw_full_##SFX(X, d, Y, d, M, N, d, cfg->tie, &c, path);          \
        _Pragma("omp atomic")                                                             \
        st->cells += M * N;                                                               \
        _Pragma("omp critical(orc_peak)")                                                 \
        { if (M * N > st->peak_table_cells) st->peak_table_cells = M * N; }               \
        return n;                                                                         \
    }                                                                                     \
    int64_t pi, pj, kk, cells, peak; double tot;                                          \
    orc_find_pivot_##SFX(X, Y, M, N, d, cfg->pivot_highest, &pi, &pj, &tot, &kk, &cells, &peak); \
    _Pragma("omp atomic")                                                                 \
    st->cells += cells;                                                                   \
    _Pragma("omp critical(orc_peak)")                                                     \
    { if (peak > st->peak_diag_values) st->peak_diag_values = peak; }                     \
    orc_pivot_t pv = {i_off + pi, j_off + pj, i_off, j_off, M, N, pi, pj, kk, tot};      \
    /* appended in completion order; linmdtw restores pre-order DFS afterwards */         \
    inst_add_pivot(st, &pv);                                                              \
    int64_t *lp = path;                                                                   \
    int64_t *rp = (int64_t *)malloc(sizeof(int64_t) * 2 * ((M - pi) + (N - pj) - 1));     \
    int64_t nl = 0, nr = 0;                                                               \
    _Pragma("omp task shared(nl) if(depth < 12)")                                         \
    nl = solve_##SFX(X, Y, pi + 1, pj + 1, d, cfg, st, i_off, j_off, lp, depth + 1);      \
    _Pragma("omp task shared(nr) if(depth < 12)")                                         \
    nr = solve_##SFX(X + pi * (int64_t)d, Y + pj * (int64_t)d, M - pi, N - pj, d, cfg, st, \
                     i_off + pi, j_off + pj, rp, depth + 1);                              \
    _Pragma("omp taskwait")                                                               \
    for (int64_t q = 1; q < nr; q++) {                                                    \
        path[2 * (nl + q - 1)] = rp[2 * q] + pi;                                          \
        path[2 * (nl + q - 1) + 1] = rp[2 * q + 1] + pj;                                  \
    }                                                                                     \
    free(rp);                                                                             \
    return nl + nr - 1;                                                                   \
}                                                                                         \
                                                                                          \
/* constrained_dtw (approx.py:180-220): _window_fill (approx.py:130-177) over rows     */   \
/* lo[i]..hi[i], row-major, moves in tie order with strict <; no valid move -> inf    */   \
/* and SELF; backtrace from the corner.  Returns the path length (path holds M+N-1   */   \
/* pairs), -1 if the backtrace meets SELF early, -2 on OOM.                          */   \
int64_t orc_window_dtw_##SFX(const float *X, const float *Y, int64_t M, int64_t N, int d,   \
                             const int64_t *lo, const int64_t *hi, const int tie[3],        \
                             double *cost_out, int64_t *path, int64_t *cells_out) {        \
    int64_t *off = (int64_t *)malloc(sizeof(int64_t) * (M + 1));                          \
    if (!off) return -2;                                                                  \
    off[0] = 0;                                                                           \
    for (int64_t i = 0; i < M; i++) off[i + 1] = off[i] + (hi[i] - lo[i] + 1);            \
    T *D = (T *)malloc(sizeof(T) * off[M]);                                               \
    uint8_t *P = (uint8_t *)malloc((size_t)off[M]);                                       \
    if (!D || !P) { free(off); free(D); free(P); return -2; }                             \
    for (int64_t i = 0; i < M; i++) {                                                     \
        for (int64_t j = lo[i]; j <= hi[i]; j++) {                                        \
            int64_t pos = off[i] + (j - lo[i]);                                           \
            T c = cost_##SFX(X + i * (int64_t)d, Y + j * (int64_t)d, d);                   \
            if (i == 0 && j == 0) { D[pos] = c; P[pos] = ORC_SELF; continue; }            \
            T best = (T)0; int have = 0; int move = ORC_SELF;                             \
            for (int m = 0; m < 3; m++) {                                                 \
                int code = tie[m]; T v;                                                   \
                if (code == ORC_LEFT) {                                                   \
                    if (j - 1 < lo[i]) continue;                                          \
                    v = D[pos - 1];                                                       \
                } else if (code == ORC_UP) {                                              \
                    if (i == 0 || j < lo[i - 1] || j > hi[i - 1]) continue;               \
                    v = D[off[i - 1] + (j - lo[i - 1])];                                  \
                } else {                                                                  \
                    if (i == 0 || j - 1 < lo[i - 1] || j - 1 > hi[i - 1]) continue;       \
                    v = D[off[i - 1] + (j - 1 - lo[i - 1])];                              \
                }                                                                         \
                if (!have || v < best) { best = v; move = code; have = 1; }               \
            }                                                                             \
            D[pos] = have ? best + c : (T)INFINITY;                                       \
            P[pos] = (uint8_t)move;                                                       \
        }                                                                                 \
    }                                                                                     \
    if (cost_out) *cost_out = (double)D[off[M] - 1];                                      \
    if (cells_out) *cells_out = off[M];                                                   \
    int64_t i = M - 1, j = N - 1, n = 0;                                                  \
    path[0] = i; path[1] = j; n = 1;                                                      \
    while (!(i == 0 && j == 0)) {                                                         \
        int mv = P[off[i] + (j - lo[i])];                                                 \
        if (mv == ORC_LEFT) j -= 1;                                                       \
        else if (mv == ORC_UP) i -= 1;                                                    \
        else if (mv == ORC_DIAG) { i -= 1; j -= 1; }                                      \
        else { n = -1; break; }                                                           \
        path[2 * n] = i; path[2 * n + 1] = j; n++;                                        \
    }                                                                                     \
    free(off); free(D); free(P);                                                          \
    if (n < 0) return -1;                                                                 \
    for (int64_t a = 0, b = n - 1; a < b; a++, b--) {                                     \
        int64_t ti = path[2 * a], tj = path[2 * a + 1];                                   \
        path[2 * a] = path[2 * b]; path[2 * a + 1] = path[2 * b + 1];                     \
        path[2 * b] = ti; path[2 * b + 1] = tj;                                           \
    }                                                                                     \
    return n;                                                                             \
}                                                                                         \
                                                                                          \
/* path_cost (core.py:182-197): per-cell costs in T, summed sequentially from 0.     */   \
double orc_path_cost_##SFX(const float *X, const float *Y, int d, const int64_t *path,    \
                           int64_t K) {                                                   \
    T total = (T)0;                                                                       \
    for (int64_t q = 0; q < K; q++)                                                       \
        total = total + cost_##SFX(X + path[2 * q] * (int64_t)d, Y + path[2 * q + 1] * (int64_t)d, d); \
    return (double)total;                                                                 \
}

ORC_DEFINE(float, f32, sqrtf)
ORC_DEFINE(double, f64, sqrt)

/* Pre-order sort of the pivot trace: the recursion is a binary tree over disjoint   */
/* index boxes, and the reference appends pivots in pre-order DFS (left first).      */
/* With tasks the append order is nondeterministic, so we restore pre-order: a node  */
/* precedes everything inside its box, and left children (smaller offsets) precede  */
/* right children.  Key: (i_off + j_off ascending ... ) is not enough, so we rebuild */
/* the tree from containment.                                                        */
static int box_contains(const orc_pivot_t *a, const orc_pivot_t *b) {
    return b->i_off >= a->i_off && b->j_off >= a->j_off &&
           b->i_off + b->M <= a->i_off + a->M && b->j_off + b->N <= a->j_off + a->N &&
           !(a->i_off == b->i_off && a->j_off == b->j_off && a->M == b->M && a->N == b->N);
}
static int cmp_pre(const void *pa, const void *pb) {
    const orc_pivot_t *a = (const orc_pivot_t *)pa, *b = (const orc_pivot_t *)pb;
    if (box_contains(a, b)) return -1;
    if (box_contains(b, a)) return 1;
    /* disjoint interiors: left subtree boxes end (at the pivot) where right ones start */
    int64_t ea = a->i_off + a->j_off, eb = b->i_off + b->j_off;
    return (ea < eb) ? -1 : (ea > eb) ? 1 : 0;
}

/* linmdtw (divide.py:181-213). prec = 32 or 64. tie: 3 codes. Returns path length (>0)  */
/* or <0 on error.  path must hold M+N-1 pairs.  Pivots are returned via *pivots_out  */
/* (malloc'd; caller frees with orc_free) in pre-order DFS.                          */
int64_t orc_linmdtw(const float *X, const float *Y, int64_t M, int64_t N, int d, int prec,
                    int min_dim, const int tie[3], int pivot_highest, int nthreads,
                    int64_t *path, double *cost_out, int64_t *cells_out,
                    int64_t *peak_diag_out, int64_t *peak_table_out,
                    orc_pivot_t **pivots_out, int64_t *npivots_out) {
    orc_cfg_t cfg;
    cfg.min_dim = min_dim;
    cfg.tie[0] = tie[0]; cfg.tie[1] = tie[1]; cfg.tie[2] = tie[2];
    cfg.pivot_highest = pivot_highest;
    orc_inst_t st;
    memset(&st, 0, sizeof(st));
    int64_t n = 0;
#ifdef _OPENMP
    if (nthreads <= 0) nthreads = omp_get_max_threads();
#pragma omp parallel num_threads(nthreads)
#pragma omp single
#endif
    {
        if (prec == 32) n = solve_f32(X, Y, M, N, d, &cfg, &st, 0, 0, path, 0);
        else n = solve_f64(X, Y, M, N, d, &cfg, &st, 0, 0, path, 0);
    }
    (void)nthreads;
    if (n < 0) { free(st.pivots); return n; }
    /* insertion sort by pre-order relation (partial order is total on a tree's DFS) */
    for (int64_t a = 1; a < st.npivots; a++) {
        orc_pivot_t key = st.pivots[a];
        int64_t b = a - 1;
        while (b >= 0 && cmp_pre(&st.pivots[b], &key) > 0) { st.pivots[b + 1] = st.pivots[b]; b--; }
        st.pivots[b + 1] = key;
    }
    if (cost_out)
        *cost_out = (prec == 32) ? orc_path_cost_f32(X, Y, d, path, n) : orc_path_cost_f64(X, Y, d, path, n);
    if (cells_out) *cells_out = st.cells;
    if (peak_diag_out) *peak_diag_out = st.peak_diag_values;
    if (peak_table_out) *peak_table_out = st.peak_table_cells;
    if (pivots_out) *pivots_out = st.pivots; else free(st.pivots);
    if (npivots_out) *npivots_out = st.npivots;
    return n;
}

void orc_free(void *p) { free(p); }

int orc_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
