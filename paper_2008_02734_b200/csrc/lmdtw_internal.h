// Internal structures shared by the host scheduler and the sm_100a kernels.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace lmdtw {

// Zero rows padded before and after the device X / Y arrays: lets the strip
// engine walk row pointers past the sub-block edges without clamping.
constexpr int kPadRows = 256;

// One DP domain handled by the strip engine.  For a half pass it is the
// triangle {i + j <= kstop} of an M x N grid (optionally on the reversed
// series); for a leaf it is the whole grid plus 2-bit backpointers.
struct PassDesc {
    int64_t x_off, y_off;   // first row of the sub-block in the padded X / Y arrays
    int32_t M, N;           // sub-block shape
    int32_t kstop;          // last anti-diagonal (M+N-2 for leaves)
    int32_t reverse;        // 1: rows/cols indexed from the end (diag_dtw "reverse")
    int32_t rows;           // rows taking part: min(M, kstop+1)
    int32_t nstrips;        // ceil(rows / (32 R))
    int64_t out_off[6];     // half pass: D(k-2),D(k-1),D(k),C(k-2),C(k-1),C(k)
    int64_t bnd_off;        // 2 slots x N tagged 64-bit words (x2 for fp64): strip handoff
    int64_t bp_off;         // leaf: backpointer words (uint64, 32 cells each)
    int64_t tab_off;        // leaf: optional full D table (-1 = none)
    int32_t bp_ld;          // leaf: backpointer words per 32-column block (nstrips * H rows; block-major)
    int32_t leaf_id;        // leaf: index into per-leaf outputs
    int64_t lb_off;         // tile left boundaries: nstrips x (H + 1) values (set by the launcher)
    int64_t flag_off;       // tiles completed per strip: nstrips ints (set by the launcher)
    int32_t tile_w;         // columns per tile (set by the launcher)
    int32_t strip_lo;       // strips [strip_lo, strip_hi) run in this launch (a shard of the pass)
    int32_t strip_hi;
    int32_t sys_out;        // 1: strip strip_hi-1 publishes to a consumer on another GPU (system-scope stores)
    uint64_t bnd_in_first;  // != 0: strip strip_lo reads strip strip_lo-1's handoff slots here
                            // (another shard's buffer, e.g. a peer GPU's), system-scope loads
    int32_t win_first;      // extra diagonals this pass saves (WinDesc entries [win_first, +win_count))
    int32_t win_count;
};

// A run of consecutive diagonals [k_lo, k_hi] (pass coordinates) whose D and
// C values a half pass saves besides its last three: the diagonals the pass's
// descendants on its spine need (a left child's forward half pass is its
// parent's forward pass restricted to the top-left block, a right child's
// reverse pass likewise), so those descendants skip recomputing them.
// D(k, idx) lands at out[d_off + (k - k_lo) * stride + idx], C likewise.
struct WinDesc {
    int32_t k_lo, k_hi;
    int32_t stride;
    int32_t pad;
    int64_t d_off, c_off;
};

// Columns per work item: a strip is cut into tiles of kTileW columns so the
// persistent pipelines rotate over strips instead of holding one strip for
// its whole length (a multiple of 32 and of the ring chunk).
#ifndef LMDTW_TILE_W
#define LMDTW_TILE_W 8192  // measured: 2048 -> 8192 cfg3 36.3 -> 35.75 ms, cfg4 353 -> 344 ms
#endif
constexpr int kTileW = LMDTW_TILE_W;

// One tile: strip `strip` of pass `pass`, columns [blk * tile_w, ...).
struct WorkItem {
    int32_t pass;
    int32_t strip;
    int32_t blk;
    int32_t pad;
};

// Queue build input: strip `strip` of pass `pass` has `ntiles` tiles.
struct StripEnt {
    int32_t pass;
    int32_t strip;
    int32_t ntiles;
};
static_assert(sizeof(StripEnt) == 12, "StripEnt is staged as 3 int32");

// Pivot search input: the two passes of one internal node.
struct PivotDesc {
    int32_t fwd, bwd;       // PassDesc indices
    int32_t M, N;
    int32_t kf, kb;         // kstop of forward / reverse pass
    int32_t highest;
    int32_t pad;
};

struct PivotOut {
    int64_t i, j, k;
    double total;
};

// Leaf backtrace input/output.
struct LeafDesc {
    int64_t x_off, y_off;
    int32_t M, N;
    int32_t pass;           // PassDesc index of the fill
    int32_t pad;
    int64_t path_off;       // capacity M+N-1 (i,j) int32 pairs, written reversed
    int64_t bp_off;
    int32_t bp_ld;          // words per 32-column block (PassDesc::bp_ld)
    int32_t pad2;
};

// Kernel launchers (kernels.cu).  All are asynchronous on `stream`.
struct WaveLaunch {
    const void* X;          // padded features, dtype T, row stride dp
    const void* Y;
    int dp;                 // padded row length (elements)
    int wide;               // DimPlan::wide
    int precision;          // 32 / 64
    const PassDesc* passes;
    const WorkItem* items;
    int nitems;
    int* counter;           // [0] work queue head, [1] exit count: zero before the first launch
                            // on the buffer; the kernel leaves both at zero
    int tag_base;           // strip handoff tags are tag_base + strip (see Engine::next_tags)
    void* out;              // half-pass diagonal outputs
    void* bnd;              // strip handoff words (memset 0xFF = tag -1 by caller)
    unsigned long long* bp; // leaf backpointers
    void* tab;              // leaf full tables (may be null)
    void* leaf_cost;        // leaf D[M-1,N-1], one per leaf_id (may be null)
    int tie0, tie1, tie2;
    int leaf;               // 0 half pass, 1 leaf fill
    void* lb;               // tile left boundaries (dtype T)
    int* flags;             // tiles completed per strip (zeroed by caller)
    int dbg;                // probe mode (LMDTW_PROBES builds; 0 = normal)
    int active_np;          // pipelines per CTA taking work (0 = all)
    int grid_warps;         // persistent warps to launch (0 = auto)
    unsigned long long* trace;  // optional per-item timestamps (debug)
    int lat;                // 1: latency variant (strip height strip_height(.., 1))
    const WinDesc* wins;    // saved-diagonal windows of the passes (PassDesc::win_first/win_count)
};

// How feature rows of dimension d are laid out and which kernels run them:
// dp = padded row length in elements; wide = 0: register-resident kernels
// instantiated for dp; wide = 1: dimension-blocked kernels (dp a multiple of
// the block width).  dp = -1: unsupported d.
struct DimPlan {
    int dp;
    int wide;
};
constexpr int kMaxDim = 1 << 16;
DimPlan plan_dims(int precision, int d);
// lat = 1: the latency variant (half the rows per lane) for levels whose
// head strips are on the critical path
int strip_height(int precision, DimPlan dp, int lat = 0);  // grid rows per strip
int pipes_per_cta(int precision, DimPlan dp, int lat = 0);
cudaError_t launch_wave(const WaveLaunch& w, cudaStream_t stream);
// per-precision halves (kernels.cu compiled as two units, LMDTW_TU=32 / 64)
cudaError_t launch_wave_f32(const WaveLaunch& w, cudaStream_t stream);
cudaError_t launch_wave_f64(const WaveLaunch& w, cudaStream_t stream);
int max_resident_warps_f32(DimPlan dp, int leaf, int device, int lat);
int max_resident_warps_f64(DimPlan dp, int leaf, int device, int lat);
cudaError_t set_watchdog_ns_f64(unsigned long long ns);
// Tile queue: tile b of entry e goes to slot cursor[b*key_per_tile + strip]++
// (cursor = first slot of each key, consumed).
cudaError_t launch_scatter_items(const StripEnt* ents, int nents, int32_t* cursor, int key_per_tile,
                                 WorkItem* items, cudaStream_t stream);
cudaError_t launch_pivots(int precision, const PassDesc* passes, const PivotDesc* piv, int npiv,
                          const void* out, PivotOut* res, void* scratch, unsigned* done, cudaStream_t stream);
// scratch for launch_pivots; `done` holds npiv counters that must be zero on
// entry (the kernel leaves them at zero)
size_t pivot_scratch_bytes(int npiv);
cudaError_t launch_backtrace(int precision, DimPlan dp, const void* X, const void* Y, const LeafDesc* leaves,
                             int nleaves, const unsigned long long* bp, int* path, void* pcost,
                             int* plen, cudaStream_t stream);
// rows of src (float32, d columns) cast to the dtype and padded to dp
// columns at dst; `pre` zero rows before and `post` after are written too
cudaError_t launch_pad_cast(int precision, const float* src, int64_t rows, int d, int dp, void* dst,
                            cudaStream_t stream, int pre = 0, int post = 0);
int max_resident_warps(int precision, DimPlan dp, int leaf, int device, int lat = 0);

// ---- window.cu: windowed DP (approx._window_fill), path costs, discrepancy
// One constrained_dtw problem: rows [0, M) of a monotone staircase window
// lo[win_off + i] .. hi[win_off + i]; backpointer words of row i start at
// bp_off + woff[win_off + i] and cover the 32-column words lo>>5 .. hi>>5.
struct BandDesc {
    int64_t x_off, y_off;   // first row in the raw float32 X / Y arrays
    int32_t M, N;
    int64_t win_off;        // offset into lo / hi / woff
    int64_t bp_off;         // backpointer word offset
    int64_t bnd_off;        // handoff words: 2 slots x N (x2 for fp64)
    int32_t id;             // index of the D(M-1, N-1) output
    int32_t pad;
};
cudaError_t launch_band(int precision, const float* X, const float* Y, int d, const BandDesc* probs, int nprobs,
                        int warps, const int32_t* lo, const int32_t* hi, const int64_t* woff,
                        unsigned long long* bp, unsigned long long* bnd, void* cost_out, const int tie[3],
                        cudaStream_t stream);
cudaError_t launch_band_backtrace(const BandDesc* probs, int nprobs, const int32_t* lo, const int64_t* woff,
                                  const unsigned long long* bp, int* path, const int64_t* path_off, int* plen,
                                  cudaStream_t stream);
// per-cell costs of (X[x_off[p] + i], Y[y_off[p] + j]) for path cells (i, j);
// cells == nullptr: row q of X against row q of Y
cudaError_t launch_path_costs(int precision, const float* X, const float* Y, int d, const int64_t* cells,
                              long long ncells, const int64_t* cell_xoff, const int64_t* cell_yoff,
                              const int32_t* cell_path, void* costs, cudaStream_t stream);
// sequential sums of costs[off[p] .. off[p+1]) in the accumulation dtype
cudaError_t launch_seq_sums(int precision, const void* costs, const int64_t* off, int npaths, double* out,
                            cudaStream_t stream);
// scratch: 2M + 2N int64; err: 2 K1 int64 (row errors, then column errors)
cudaError_t launch_discrepancy(const int64_t* p1, long long K1, const int64_t* p2, long long K2, long long M,
                               long long N, long long* scratch, long long* err, cudaStream_t stream);
cudaError_t set_watchdog_ns(unsigned long long ns);  // per device (current device)
cudaError_t wait_stats(unsigned long long* cycles, unsigned long long* count, int reset);

}  // namespace lmdtw
