// sm_100a kernels for the per-path steps either side of the exact aligner
// (SURVEY.md 8(f)):
//
//  * band_kernel      -- windowed DP of approx._window_fill (approx.py:130-177)
//                        over a monotone staircase window, 2-bit backpointers,
//                        D(M-1, N-1).  Replaces the numba row-major fill of
//                        constrained_dtw (approx.py:180-220).
//  * band_backtrace   -- constrained_dtw's backtrace (approx.py:203-217).
//  * frame_costs / path sums -- core.frame_costs (core.py:167-179) and
//                        core.path_cost (core.py:182-197) for batches of paths.
//  * discrepancy      -- metrics.discrepancy (metrics.py:44-63).
//
// Arithmetic contract as in kernels.cu: cost = sqrt(((d0*d0) + d1*d1) + ...),
// every op rounded separately in the accumulation dtype (the library builds
// with -fmad=false), sqrt correctly rounded; D = min(valid neighbours) + c;
// the move is the first code in tie order whose valid neighbour attains the
// minimum (== the reference's strict-< precedence scan, approx.py:152-171).
//
// Band engine.  The window's rows are cut into groups of 32; a warp owns one
// group (lane l = row 32g + l) and sweeps its columns in a systolic skew
// (lane l works on column B + s - l at step s, B = the group's first lo),
// the up-neighbour arriving by shuffle from lane l-1.  Groups go round-robin
// to the CTA's warps; group g hands its bottom row to group g+1 through two
// N-long slots of tagged 64-bit words (value | group index), read 32 columns
// at a time one block ahead -- the strip handoff of the main engine.  All warps
// of a problem live in one CTA, so the pipeline cannot deadlock.
#include <climits>
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
#include <math_constants.h>

#include "lmdtw_internal.h"

namespace lmdtw {
namespace {

typedef unsigned long long u64;
constexpr unsigned kFull = 0xffffffffu;

template <typename T> struct BNum;
template <> struct BNum<float> {
    static constexpr int W = 1;  // 64-bit handoff words per value
    static __device__ __forceinline__ float inf() { return CUDART_INF_F; }
    static __device__ __forceinline__ float sub(float a, float b) { return __fsub_rn(a, b); }
    static __device__ __forceinline__ float mul(float a, float b) { return __fmul_rn(a, b); }
    static __device__ __forceinline__ float add(float a, float b) { return __fadd_rn(a, b); }
    static __device__ __forceinline__ float sqrt_(float a) { return __fsqrt_rn(a); }
    static __device__ __forceinline__ void put(u64* p, float v, int tag) {
        const u64 w = ((u64)(unsigned)tag << 32) | (u64)__float_as_uint(v);
        asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(w) : "memory");
    }
    static __device__ __forceinline__ bool get(const u64* p, int tag, float& v) {
        u64 w;
        asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(w) : "l"(p) : "memory");
        v = __uint_as_float((unsigned)w);
        return (int)(w >> 32) == tag;
    }
};
template <> struct BNum<double> {
    static constexpr int W = 2;
    static __device__ __forceinline__ double inf() { return CUDART_INF; }
    static __device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }
    static __device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
    static __device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
    static __device__ __forceinline__ double sqrt_(double a) { return __dsqrt_rn(a); }
    static __device__ __forceinline__ void put(u64* p, double v, int tag) {
        const u64 b = (u64)__double_as_longlong(v);
        const u64 w0 = ((u64)(unsigned)tag << 32) | (b & 0xffffffffull);
        const u64 w1 = ((u64)(unsigned)tag << 32) | (b >> 32);
        asm volatile("st.relaxed.gpu.global.v2.b64 [%0], {%1, %2};" ::"l"(p), "l"(w0), "l"(w1) : "memory");
    }
    static __device__ __forceinline__ bool get(const u64* p, int tag, double& v) {
        u64 w0, w1;
        asm volatile("ld.relaxed.gpu.global.v2.b64 {%0, %1}, [%2];" : "=l"(w0), "=l"(w1) : "l"(p) : "memory");
        v = __longlong_as_double((long long)((w1 << 32) | (w0 & 0xffffffffull)));
        return (int)(w0 >> 32) == tag && (int)(w1 >> 32) == tag;
    }
};

__device__ __forceinline__ unsigned long long now_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
constexpr unsigned long long kBandWatchdogNs = 60000000000ull;

// Euclidean cost of rows x, y (float32 storage, accumulation dtype T).
template <typename T>
__device__ __forceinline__ T row_cost(const float* __restrict__ x, const float* __restrict__ y, int d) {
    typedef BNum<T> Nm;
    T s = T(0);
    for (int t = 0; t < d; t++) {
        const T df = Nm::sub((T)__ldg(x + t), (T)__ldg(y + t));
        const T q = Nm::mul(df, df);
        s = (t == 0) ? q : Nm::add(s, q);
    }
    return Nm::sqrt_(s);
}

template <typename T>
__global__ void band_kernel(const float* __restrict__ X, const float* __restrict__ Y, int d,
                            const BandDesc* __restrict__ probs, const int32_t* __restrict__ lo,
                            const int32_t* __restrict__ hi, const int64_t* __restrict__ woff, u64* bp, u64* bnd,
                            T* cost_out, int tie0, int tie1, int tie2) {
    typedef BNum<T> Nm;
    constexpr int W = Nm::W;
    const BandDesc P = probs[blockIdx.x];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    const int M = P.M, N = P.N;
    const int ngroups = (M + 31) / 32;
    const int32_t* L = lo + P.win_off;
    const int32_t* Hh = hi + P.win_off;
    const int64_t* WO = woff + P.win_off;
    const T INF = Nm::inf();
    auto rank_of = [&](int code) { return tie0 == code ? 0 : (tie1 == code ? 1 : 2); };
    const int keyL = (rank_of(0) << 2) | 0, keyU = (rank_of(1) << 2) | 1, keyD = (rank_of(2) << 2) | 2;
    const long long sstride = (long long)((N + 1) & ~1) * W;
    u64* slots = bnd + P.bnd_off;

    for (int g = warp; g < ngroups; g += nw) {
        const int i0 = 32 * g;
        const int i = i0 + lane;
        const bool row_ok = i < M;
        const int ilast = min(i0 + 31, M - 1);
        const int B = L[i0];
        const int E = Hh[ilast];
        const int lo_i = row_ok ? L[i] : INT_MAX, hi_i = row_ok ? Hh[i] : -1;
        const int lo_p = (row_ok && i > 0) ? L[i - 1] : INT_MAX, hi_p = (row_ok && i > 0) ? Hh[i - 1] : -1;
        const int lo_p0 = __shfl_sync(kFull, lo_p, 0), hi_p0 = __shfl_sync(kFull, hi_p, 0);
        const float* xr = X + (P.x_off + (long long)(row_ok ? i : 0)) * d;
        const int64_t wbase = row_ok ? P.bp_off + WO[i] - (lo_i >> 5) : 0;
        const u64* bin = slots + (long long)((g + 1) & 1) * sstride;  // group g-1's bottom row
        u64* bout = slots + (long long)(g & 1) * sstride;
        const bool publish = (lane == 31) && (g + 1 < ngroups);
        const int nsteps = E - B + 32;

        T cur = INF, top_prev = INF, bcur = INF, bnext = INF;
        bool nok = true;
        u64 acc = 0;
        // group g-1's bottom row, columns B + 32 blk + lane
        auto need_col = [&](int col) { return g > 0 && col >= lo_p0 && col <= hi_p0; };
        auto load_blk = [&](int blk, T& v) -> bool {
            const int col = B + 32 * blk + lane;
            if (!need_col(col)) return true;
            return Nm::get(bin + (long long)col * W, g - 1, v);
        };
        nok = load_blk(0, bnext);
        // lane 0's first diagonal neighbour: row i0-1 at column B-1 (the feed
        // starts at column B)
        if (lane == 0 && need_col(B - 1)) {
            const unsigned long long t0 = now_ns();
            while (!Nm::get(bin + (long long)(B - 1) * W, g - 1, top_prev)) {
                __nanosleep(64);
                if (now_ns() - t0 > kBandWatchdogNs) {
                    printf("lmdtw band watchdog: group %d corner stuck\n", g);
                    __trap();
                }
            }
        }
        for (int s = 0; s < nsteps; s++) {
            if ((s & 31) == 0) {
                const int blk = s >> 5;
                if (!__all_sync(kFull, nok)) {
                    const unsigned long long t0 = now_ns();
                    unsigned ns = 32;
                    for (;;) {
                        __nanosleep(ns);
                        ns = min(ns * 2, 512u);
                        nok = load_blk(blk, bnext);
                        if (__all_sync(kFull, nok)) break;
                        if (now_ns() - t0 > kBandWatchdogNs) {
                            if (lane == 0) printf("lmdtw band watchdog: group %d block %d stuck\n", g, blk);
                            __trap();
                        }
                    }
                }
                bcur = bnext;
                nok = load_blk(blk + 1, bnext);
            }
            const int j = B + s - lane;
            const T feed = __shfl_sync(kFull, bcur, s & 31);
            T top = __shfl_sync(kFull, cur, (lane + 31) & 31);
            top = (lane == 0) ? feed : top;
            const bool act = row_ok && j >= lo_i && j <= hi_i;
            if (act) {
                const T c = row_cost<T>(xr, Y + (P.y_off + (long long)j) * d, d);
                const bool okL = j - 1 >= lo_i;
                const bool okU = i > 0 && j >= lo_p && j <= hi_p;
                const bool okD = i > 0 && j - 1 >= lo_p && j - 1 <= hi_p;
                T m = INF;
                if (okL) m = fmin(m, cur);
                if (okU) m = fmin(m, top);
                if (okD) m = fmin(m, top_prev);
                const int kL = (okL && cur == m) ? keyL : 15;
                const int kU = (okU && top == m) ? keyU : 15;
                const int kD = (okD && top_prev == m) ? keyD : 15;
                const int mv = min(min(kL, kU), kD) & 3;  // 3 = SELF: no valid move
                const T D = (i == 0 && j == 0) ? c : Nm::add(m, c);
                acc |= (u64)mv << (2 * (j & 31));
                if ((j & 31) == 31 || j == hi_i) {
                    bp[wbase + (j >> 5)] = acc;
                    acc = 0;
                }
                cur = D;
                if (publish) Nm::put(bout + (long long)j * W, D, g);
                if (i == M - 1 && j == N - 1) cost_out[P.id] = D;
            }
            top_prev = top;
        }
    }
}

// One warp per problem: follow the 2-bit moves from (M-1, N-1), caching the
// backpointer words of 32 rows x one 32-column word (lane l: row ib - l).
__global__ void band_backtrace(const BandDesc* __restrict__ probs, int nprobs, const int32_t* __restrict__ lo,
                               const int64_t* __restrict__ woff, const u64* __restrict__ bp, int* path,
                               const int64_t* __restrict__ path_off, int* plen) {
    const int lane = threadIdx.x & 31;
    const int p = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (p >= nprobs) return;
    const BandDesc P = probs[p];
    const int32_t* L = lo + P.win_off;
    const int64_t* WO = woff + P.win_off;
    int* out = path + 2 * path_off[p];
    int i = P.M - 1, j = P.N - 1, n = 0;
    int ib = i, jw = j >> 5;
    auto word = [&](int r) -> u64 {
        if (r < 0) return 0ull;
        const int l0 = L[r] >> 5;
        return bp[P.bp_off + WO[r] + jw - l0];
    };
    u64 w = word(ib - lane);
    if (lane == 0) {
        out[0] = i;
        out[1] = j;
    }
    n = 1;
    bool bad = false;
    while (!(i == 0 && j == 0)) {
        const u64 wd = __shfl_sync(kFull, w, ib - i);
        const int mv = (int)((wd >> (2 * (j & 31))) & 3ull);
        if (mv == 0) {
            j -= 1;
        } else if (mv == 1) {
            i -= 1;
        } else if (mv == 2) {
            i -= 1;
            j -= 1;
        } else {
            bad = true;
            break;
        }
        if (i < ib - 31 || (j >> 5) != jw) {
            ib = i;
            jw = j >> 5;
            w = word(ib - lane);
        }
        if (lane == 0) {
            out[2 * n] = i;
            out[2 * n + 1] = j;
        }
        n++;
    }
    if (lane == 0) plen[p] = bad ? -1 : n;
}

// core.frame_costs over gathered rows: cost of (X[pi], Y[pj]) for every path
// cell of every path (grid-stride over all cells).
template <typename T>
__global__ void path_cell_costs(const float* __restrict__ X, const float* __restrict__ Y, int d,
                                const int64_t* __restrict__ cells, long long ncells,
                                const int64_t* __restrict__ cell_xoff, const int64_t* __restrict__ cell_yoff,
                                const int32_t* __restrict__ cell_path, T* costs) {
    for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < ncells;
         q += (long long)gridDim.x * blockDim.x) {
        // cells == nullptr: row q against row q (frame_costs of two frame arrays)
        const int p = cell_path ? cell_path[q] : 0;
        const long long xi = (cell_xoff ? cell_xoff[p] : 0) + (cells ? cells[2 * q] : q);
        const long long yj = (cell_yoff ? cell_yoff[p] : 0) + (cells ? cells[2 * q + 1] : q);
        costs[q] = row_cost<T>(X + xi * d, Y + yj * d, d);
    }
}

// core.path_cost: sequential sum from 0 in T, left to right (core.py:194-196).
// One warp per path: the warp stages 1024 costs in shared memory, lane 0 adds.
template <typename T>
__global__ void seq_sums(const T* __restrict__ costs, const int64_t* __restrict__ off, int npaths,
                         double* out) {
    __shared__ T buf[4][1024];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int p = blockIdx.x * 4 + w;
    if (p >= npaths) return;
    const long long a = off[p], b = off[p + 1];
    T total = T(0);
    for (long long c0 = a; c0 < b; c0 += 1024) {
        const int n = (int)((b - c0) < 1024 ? (b - c0) : 1024);
        for (int q = lane; q < n; q += 32) buf[w][q] = costs[c0 + q];
        __syncwarp();
        if (lane == 0)
            for (int q = 0; q < n; q++) total = BNum<T>::add(total, buf[w][q]);
        __syncwarp();
    }
    if (lane == 0) out[p] = (double)total;
}

// metrics.discrepancy: per-row / per-column [min, max] of path 2, then every
// cell of path 1 measured against them.
__global__ void path_intervals(const int64_t* __restrict__ p2, long long K2, long long* rlo, long long* rhi,
                               long long* clo, long long* chi) {
    for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < K2;
         q += (long long)gridDim.x * blockDim.x) {
        const long long i = p2[2 * q], j = p2[2 * q + 1];
        atomicMin(rlo + i, j);
        atomicMax(rhi + i, j);
        atomicMin(clo + j, i);
        atomicMax(chi + j, i);
    }
}
__global__ void path_offsets(const int64_t* __restrict__ p1, long long K1, const long long* __restrict__ rlo,
                             const long long* __restrict__ rhi, const long long* __restrict__ clo,
                             const long long* __restrict__ chi, long long* err) {
    for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < K1;
         q += (long long)gridDim.x * blockDim.x) {
        const long long i = p1[2 * q], j = p1[2 * q + 1];
        const long long re = max(0ll, max(rlo[i] - j, j - rhi[i]));
        const long long ce = max(0ll, max(clo[j] - i, i - chi[j]));
        err[q] = re;
        err[K1 + q] = ce;
    }
}
__global__ void fill_i64(long long* p, long long n, long long v) {
    for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < n;
         q += (long long)gridDim.x * blockDim.x)
        p[q] = v;
}

inline int grid_for(long long n, int block) {
    long long g = (n + block - 1) / block;
    if (g > 148 * 8) g = 148 * 8;
    return (int)(g < 1 ? 1 : g);
}

}  // namespace

cudaError_t launch_band(int precision, const float* X, const float* Y, int d, const BandDesc* probs, int nprobs,
                        int warps, const int32_t* lo, const int32_t* hi, const int64_t* woff,
                        unsigned long long* bp, unsigned long long* bnd, void* cost_out, const int tie[3],
                        cudaStream_t st) {
    if (nprobs <= 0) return cudaSuccess;
    if (precision == 32)
        band_kernel<float><<<nprobs, 32 * warps, 0, st>>>(X, Y, d, probs, lo, hi, woff, bp, bnd, (float*)cost_out,
                                                          tie[0], tie[1], tie[2]);
    else
        band_kernel<double><<<nprobs, 32 * warps, 0, st>>>(X, Y, d, probs, lo, hi, woff, bp, bnd,
                                                           (double*)cost_out, tie[0], tie[1], tie[2]);
    return cudaGetLastError();
}

cudaError_t launch_band_backtrace(const BandDesc* probs, int nprobs, const int32_t* lo, const int64_t* woff,
                                  const unsigned long long* bp, int* path, const int64_t* path_off, int* plen,
                                  cudaStream_t st) {
    if (nprobs <= 0) return cudaSuccess;
    band_backtrace<<<(nprobs + 3) / 4, 128, 0, st>>>(probs, nprobs, lo, woff, bp, path, path_off, plen);
    return cudaGetLastError();
}

cudaError_t launch_path_costs(int precision, const float* X, const float* Y, int d, const int64_t* cells,
                              long long ncells, const int64_t* cell_xoff, const int64_t* cell_yoff,
                              const int32_t* cell_path, void* costs, cudaStream_t st) {
    if (ncells <= 0) return cudaSuccess;
    if (precision == 32)
        path_cell_costs<float><<<grid_for(ncells, 256), 256, 0, st>>>(X, Y, d, cells, ncells, cell_xoff, cell_yoff,
                                                                     cell_path, (float*)costs);
    else
        path_cell_costs<double><<<grid_for(ncells, 256), 256, 0, st>>>(X, Y, d, cells, ncells, cell_xoff,
                                                                      cell_yoff, cell_path, (double*)costs);
    return cudaGetLastError();
}

cudaError_t launch_seq_sums(int precision, const void* costs, const int64_t* off, int npaths, double* out,
                            cudaStream_t st) {
    if (npaths <= 0) return cudaSuccess;
    if (precision == 32)
        seq_sums<float><<<(npaths + 3) / 4, 128, 0, st>>>((const float*)costs, off, npaths, out);
    else
        seq_sums<double><<<(npaths + 3) / 4, 128, 0, st>>>((const double*)costs, off, npaths, out);
    return cudaGetLastError();
}

cudaError_t launch_discrepancy(const int64_t* p1, long long K1, const int64_t* p2, long long K2, long long M,
                               long long N, long long* scratch, long long* err, cudaStream_t st) {
    long long* rlo = scratch;
    long long* rhi = rlo + M;
    long long* clo = rhi + M;
    long long* chi = clo + N;
    fill_i64<<<grid_for(M, 256), 256, 0, st>>>(rlo, M, LLONG_MAX);
    fill_i64<<<grid_for(M, 256), 256, 0, st>>>(rhi, M, -1);
    fill_i64<<<grid_for(N, 256), 256, 0, st>>>(clo, N, LLONG_MAX);
    fill_i64<<<grid_for(N, 256), 256, 0, st>>>(chi, N, -1);
    path_intervals<<<grid_for(K2, 256), 256, 0, st>>>(p2, K2, rlo, rhi, clo, chi);
    path_offsets<<<grid_for(K1, 256), 256, 0, st>>>(p1, K1, rlo, rhi, clo, chi, err);
    return cudaGetLastError();
}

}  // namespace lmdtw
