// Host side of liblmdtw_b200.so: device contexts, the level-batched
// recursion scheduler and the extern "C" ABI declared in include/lmdtw_b200.h.
//
// Scheduler (replaces divide._solve, divide.py:148-178).  The reference
// recurses depth-first, one pivot search at a time.  Here every recursion
// level is one batch: all internal nodes of the level (of every pair in a
// batch) launch their forward and reverse half passes as ONE persistent
// wave_kernel launch, then ONE pivot_kernel launch, then one 48-byte-per-node
// device->host copy of the pivots.  Leaves (divide.py:153-157) accumulate and
// are filled + backtraced in one batched launch at the end.  The pivot trace
// is re-emitted in the reference's pre-order DFS, the path is the in-order
// concatenation of leaf paths (divide.py:176-178), and the returned cost is
// the reference's path_cost: per-cell costs summed sequentially in the
// accumulation dtype (core.py:191-197).
#include <algorithm>
#include <chrono>
#include <functional>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include <cuda_runtime.h>

#include "lmdtw_b200.h"
#include "lmdtw_internal.h"

using namespace lmdtw;

struct lmdtw_result {
    lmdtw_align_info_t info;
    std::unique_ptr<int64_t[]> path;  // 2 * info.path_len, written once (no zero fill)
    std::vector<lmdtw_pivot_t> pivots;
};

namespace {

thread_local std::string g_err;
std::atomic<long long> g_launches{0};

struct Stats {
    std::mutex mu;
    double wave_ms = 0, leaf_ms = 0, pivot_ms = 0;
    long long wave_launches = 0, wave_cells = 0, leaf_cells = 0;
} g_stats;
std::atomic<int> g_profile{0};
cudaEvent_t g_last_sync_ev = nullptr;  // LMDTW_HOST_TIMING diagnostics

int set_err(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

int cuda_err(cudaError_t e, const char* what) {
    cudaGetLastError();
    if (e == cudaErrorMemoryAllocation)
        return set_err(LMDTW_ENOMEM, std::string("device out of memory in ") + what);
    return set_err(LMDTW_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

#define CU(x)                                        \
    do {                                             \
        cudaError_t _e = (x);                        \
        if (_e != cudaSuccess) return cuda_err(_e, #x); \
    } while (0)
#define TRY(x)                 \
    do {                       \
        int _r = (x);          \
        if (_r != LMDTW_OK) return _r; \
    } while (0)

struct DBuf {
    void* p = nullptr;
    size_t cap = 0;
    cudaError_t ensure(size_t n) {
        if (n <= cap && p) return cudaSuccess;
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
        size_t c = std::max<size_t>(n + n / 4, 4096);
        cudaError_t e = cudaMalloc(&p, c);
        if (e != cudaSuccess) {
            p = nullptr;
            cudaGetLastError();
            return e;
        }
        cap = c;
        return cudaSuccess;
    }
    // ensure, and fill a new allocation with `byte` (buffers the kernels
    // leave clean after every launch: queue counters, tile flags, pivot
    // counters; handoff words, whose stale tags never match -- Engine::next_tags)
    cudaError_t ensure_init(size_t n, int byte, cudaStream_t st) {
        if (n <= cap && p) return cudaSuccess;
        cudaError_t e = ensure(n);
        if (e == cudaSuccess) e = cudaMemsetAsync(p, byte, cap, st);
        return e;
    }
    template <typename T> T* as() const { return reinterpret_cast<T*>(p); }
    // Grow to n bytes keeping the first `used` bytes (offsets into the buffer
    // stay valid); stream-ordered copy, the old block freed after it.
    cudaError_t grow_keep(size_t n, size_t used, cudaStream_t st) {
        if (n <= cap && p) return cudaSuccess;
        void* q = nullptr;
        const size_t c = std::max<size_t>(n + n / 2, 1 << 20);
        cudaError_t e = cudaMalloc(&q, c);
        if (e != cudaSuccess) {
            cudaGetLastError();
            return e;
        }
        if (p && used) {
            e = cudaMemcpyAsync(q, p, used, cudaMemcpyDeviceToDevice, st);
            if (e == cudaSuccess) e = cudaStreamSynchronize(st);
            if (e != cudaSuccess) {
                cudaFree(q);
                return e;
            }
        }
        if (p) cudaFree(p);
        p = q;
        cap = c;
        return cudaSuccess;
    }
};

struct HBuf {
    void* p = nullptr;
    size_t cap = 0;
    cudaError_t ensure(size_t n) {
        if (n <= cap && p) return cudaSuccess;
        if (p) cudaFreeHost(p);
        p = nullptr;
        cap = 0;
        size_t c = std::max<size_t>(n + n / 4, 4096);
        cudaError_t e = cudaMallocHost(&p, c);
        if (e != cudaSuccess) {
            p = nullptr;
            cudaGetLastError();
            return e;
        }
        cap = c;
        return cudaSuccess;
    }
    template <typename T> T* as() const { return reinterpret_cast<T*>(p); }
};

// One in-flight batch of half passes (a set of recursion nodes): its stream
// and its buffers.  Batches run concurrently on their own streams, so the
// children of a node start while other nodes of its level still run.
// Host side of one host->device upload per launch batch: pass descriptors,
// the tile queue's build input, saved-window and pivot descriptors, packed at
// 16-byte aligned offsets (Engine::upload).
struct Staging {
    std::vector<char> h;
    size_t reserve(size_t n) {
        const size_t o = (h.size() + 15) & ~(size_t)15;
        h.resize(o + n);
        return o;
    }
    size_t add(const void* src, size_t n) {
        const size_t o = reserve(n);
        if (n) memcpy(h.data() + o, src, n);
        return o;
    }
    template <typename T> T* at(size_t o) { return reinterpret_cast<T*>(h.data() + o); }
};

struct Slot {
    cudaStream_t st = nullptr;
    cudaEvent_t done = nullptr;
    DBuf passes, items, counter, out, bnd, pdesc, pout, pscratch, pdone, trace, lb, flags, istage, wins;
    HBuf h_passes, h_items, h_istage, h_pdesc, h_pout, h_wins;
    Staging stg;       // the batch being built
    HBuf h_stage;      // its pinned copy
    DBuf d_stage;      // its device copy (valid until the slot's next upload)
    size_t passes_off = 0;  // PassDesc array of the last run_wave in d_stage
    int tag_next = 0;       // next free handoff tag base of `bnd`
    template <typename T> T* dev(size_t off) const { return reinterpret_cast<T*>((char*)d_stage.p + off); }
};

struct Ctx {
    int device = 0;
    int nsm = 148;  // SMs of the device
    std::mutex mu;
    cudaStream_t st = nullptr;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    Slot main;                                  // main.st == st
    std::vector<std::unique_ptr<Slot>> extra;   // more batch slots, created on demand
    DBuf xraw, yraw, xp, yp, ldesc, bp, path, pcost, plen, lcost, tab;
    DBuf arena;  // recursion outputs with stable offsets: last diagonals + saved windows (align_core)
    // window.cu entry points (constrained DTW, path costs, discrepancy)
    DBuf wlo, whi, woff, wbp, wbnd, wdesc, wcost, wpath, wpoff, wplen, pcells, pcost2, poffs, pxoff, pyoff, ppid,
        pout2, dsc;
    // leaf outputs, one device block and its pinned copy (one D2H copy):
    // reversed local paths (int pairs) | per-cell costs | lengths | D(M-1, N-1)
    DBuf lout;
    HBuf h_lout;
    size_t lo_pcost = 0, lo_plen = 0, lo_lcost = 0;
    const int* hpath() const { return h_lout.as<int>(); }
    template <typename T> const T* hpcost() const { return reinterpret_cast<const T*>(h_lout.as<char>() + lo_pcost); }
    const int* hplen() const { return reinterpret_cast<const int*>(h_lout.as<char>() + lo_plen); }
    template <typename T> const T* hlcost() const { return reinterpret_cast<const T*>(h_lout.as<char>() + lo_lcost); }
    long long call_launches = 0;
    long long h2d = 0, d2h = 0;
    // profiling (lmdtw_profile_enable): events around wave launches, read
    // back at the next stream sync, so timing never adds a host sync
    struct Pend {
        int e0, e1;
        long long cells;
        bool leaf;
    };
    std::vector<cudaEvent_t> evpool;
    std::vector<Pend> pend;
    int ev_used = 0;
    cudaError_t prof_event(int* idx) {
        if (ev_used == (int)evpool.size()) {
            cudaEvent_t e;
            cudaError_t r = cudaEventCreate(&e);
            if (r != cudaSuccess) return r;
            evpool.push_back(e);
        }
        *idx = ev_used++;
        return cudaSuccess;
    }
    // call after a stream sync: every pending event has completed
    void prof_collect();
};

void Ctx::prof_collect() {
    if (pend.empty()) {
        ev_used = 0;
        return;
    }
    // Launches of concurrent batches overlap: the time charged to waves and
    // to leaves is the union of their [start, end] intervals, measured from
    // the first pending event.
    std::vector<std::pair<float, float>> waves, leaves;
    long long wcells = 0, lcells = 0, wl = 0;
    const cudaEvent_t ref = evpool[pend[0].e0];
    for (const Pend& p : pend) {
        float a = 0, b = 0;
        if (cudaEventElapsedTime(&a, ref, evpool[p.e0]) != cudaSuccess ||
            cudaEventElapsedTime(&b, ref, evpool[p.e1]) != cudaSuccess) {
            cudaGetLastError();
            continue;
        }
        if (p.leaf) {
            leaves.emplace_back(a, b);
            lcells += p.cells;
        } else {
            waves.emplace_back(a, b);
            wcells += p.cells;
            wl++;
        }
    }
    auto span = [](std::vector<std::pair<float, float>>& v) {
        std::sort(v.begin(), v.end());
        double tot = 0, lo = 0, hi = -1e30;
        for (auto& iv : v) {
            if (iv.first > hi) {
                if (hi > lo) tot += hi - lo;
                lo = iv.first;
                hi = iv.second;
            } else {
                hi = std::max<double>(hi, iv.second);
            }
        }
        if (hi > lo) tot += hi - lo;
        return tot;
    };
    const double wms = span(waves), lms = span(leaves);
    {
        std::lock_guard<std::mutex> g(g_stats.mu);
        g_stats.wave_ms += wms;
        g_stats.wave_launches += wl;
        g_stats.wave_cells += wcells;
        g_stats.leaf_ms += lms;
        g_stats.leaf_cells += lcells;
    }
    pend.clear();
    ev_used = 0;
}

// Contexts: a per-device pool.  A call leases one context (stream, events,
// buffers) for its duration and returns it afterwards, so concurrent calls
// on one device run on separate streams with separate buffers (SPEC.md:287
// "safe for concurrent independent calls"), and a progress callback that
// calls back into the library (from inside a running alignment) gets a
// context of its own instead of deadlocking on the running call's.
struct DevPool {
    std::mutex mu;
    std::vector<std::unique_ptr<Ctx>> all;  // all[0]: the primary context (lmdtw_stream)
    std::vector<bool> busy;
};
std::mutex g_ctx_mu;
std::vector<std::unique_ptr<DevPool>> g_pools;

int make_ctx(int device, std::unique_ptr<Ctx>& out) {
    std::unique_ptr<Ctx> c(new Ctx());
    c->device = device;
    CU(cudaSetDevice(device));
    CU(cudaDeviceGetAttribute(&c->nsm, cudaDevAttrMultiProcessorCount, device));
    CU(cudaStreamCreateWithFlags(&c->st, cudaStreamNonBlocking));
    CU(cudaEventCreate(&c->ev0));
    CU(cudaEventCreate(&c->ev1));
    c->main.st = c->st;
    CU(cudaEventCreateWithFlags(&c->main.done, cudaEventDisableTiming));
    if (const char* w = getenv("LMDTW_WATCHDOG_S")) {
        const double sec = atof(w);  // 0 disables the watchdog
        if (sec >= 0) CU(set_watchdog_ns((unsigned long long)(sec * 1e9)));
    }
    out = std::move(c);
    return LMDTW_OK;
}

int get_pool(int device, DevPool** out) {
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess || n == 0) {
        cudaGetLastError();
        return set_err(LMDTW_ECUDA, "no CUDA device available (liblmdtw_b200 has no CPU fallback)");
    }
    if (device < 0 || device >= n) return set_err(LMDTW_EINVAL, "bad device index");
    std::lock_guard<std::mutex> g(g_ctx_mu);
    if ((int)g_pools.size() < n) g_pools.resize(n);
    if (!g_pools[device]) g_pools[device].reset(new DevPool());
    *out = g_pools[device].get();
    return LMDTW_OK;
}

struct CtxLease {
    Ctx* c = nullptr;
    DevPool* pool = nullptr;
    size_t slot = 0;
    Ctx* operator->() const { return c; }
    Ctx& operator*() const { return *c; }
    ~CtxLease() {
        if (c) {
            std::lock_guard<std::mutex> g(pool->mu);
            pool->busy[slot] = false;
        }
    }
};

// Lease the lowest-numbered free context of `device` (creating one if all
// are busy) and make `device` current.
int lease_ctx(int device, CtxLease& out) {
    DevPool* pool = nullptr;
    TRY(get_pool(device, &pool));
    std::lock_guard<std::mutex> g(pool->mu);
    size_t q = 0;
    while (q < pool->all.size() && pool->busy[q]) q++;
    if (q == pool->all.size()) {
        std::unique_ptr<Ctx> c;
        TRY(make_ctx(device, c));
        pool->all.push_back(std::move(c));
        pool->busy.push_back(false);
    }
    pool->busy[q] = true;
    out.c = pool->all[q].get();
    out.pool = pool;
    out.slot = q;
    CU(cudaSetDevice(device));
    return LMDTW_OK;
}

// The primary context's stream (created on first use).
int primary_stream(int device, cudaStream_t* st) {
    DevPool* pool = nullptr;
    TRY(get_pool(device, &pool));
    std::lock_guard<std::mutex> g(pool->mu);
    if (pool->all.empty()) {
        std::unique_ptr<Ctx> c;
        TRY(make_ctx(device, c));
        pool->all.push_back(std::move(c));
        pool->busy.push_back(false);
    }
    *st = pool->all[0]->st;
    return LMDTW_OK;
}

inline int64_t dlen(int64_t k, int64_t M, int64_t N) {
    if (k < 0 || k > M + N - 2) return 0;
    return std::min(std::min(k, M - 1), std::min(N - 1, M + N - 2 - k)) + 1;
}

// Number of cells (i,j), i<M, j<N with i+j <= kstop.
int64_t cells_upto(int64_t kstop, int64_t M, int64_t N) {
    if (kstop < 0) return 0;
    const int64_t imax = std::min(M - 1, kstop);
    int64_t total = 0;
    // rows with kstop - i + 1 >= N contribute N
    const int64_t ifull = std::min(imax, kstop - N + 1);
    int64_t start = 0;
    if (ifull >= 0) {
        total += (ifull + 1) * N;
        start = ifull + 1;
    }
    if (start <= imax) {
        // sum_{i=start}^{imax} (kstop - i + 1)
        const int64_t a = kstop - start + 1, b = kstop - imax + 1, cnt = imax - start + 1;
        total += (a + b) * cnt / 2;
    }
    return total;
}

// diagonal.py:160-169: max over k<=kstop of 2*(L(k-2)+L(k-1)+L(k)); the window
// sum is unimodal with its peak at k in [m, m+2], m = min(M,N)-1.
int64_t peak_values(int64_t kstop, int64_t M, int64_t N) {
    auto W = [&](int64_t k) { return dlen(k - 2, M, N) + dlen(k - 1, M, N) + dlen(k, M, N); };
    const int64_t m = std::min(M, N) - 1;
    int64_t best = W(kstop);
    for (int64_t k = m; k <= m + 2; k++)
        if (k >= 0 && k <= kstop) best = std::max(best, W(k));
    return 2 * best;
}

struct Inst {  // divide._Instrument (divide.py:60-94)
    int64_t cells = 0, budget = 0, next_report = 0, peak_diag = 0, peak_table = 0;
    lmdtw_progress_fn cb = nullptr;
    void* user = nullptr;
    void add(int64_t n) {
        cells += n;
        if (cb && cells >= next_report) {
            next_report = cells + std::max<int64_t>(1, budget / 100);
            cb(cells, budget, user);
        }
    }
    // A level is one "completed diagonal batch"; report it in <=1% slices.
    void add_batch(int64_t n) {
        const int64_t step = std::max<int64_t>(1, budget / 100);
        while (n > 0) {
            const int64_t s = std::min(n, step);
            add(s);
            n -= s;
        }
    }
};

struct Node {
    int64_t i_off, j_off, M, N;
    int pair;
    int left = -1, right = -1;
    int64_t pi = -1, pj = -1, k = -1;
    double total = 0;
    int leaf = -1;  // index into leaf list
    int depth = 0;  // recursion level (root 0)
    // half-pass reuse: the saved pass whose windows hold this node's forward /
    // reverse diagonals (-1: compute them), and the passes this node's own
    // children inherit from (set when the node's batch is built)
    int fsrc = -1, bsrc = -1, fpass = -1, bpass = -1;
};

// A computed half pass kept for the descendants on its spine: a forward pass
// of node n serves n.left, n.left.left, ... (same first cell), a reverse pass
// n.right, n.right.right, ... (same last cell).
struct SavedPass {
    int64_t M, N;                 // grid of the node that computed it
    std::vector<WinDesc> wins;    // arena offsets (element units)
};

// Diagonal ranges a pass's spine descendants may need, in the pass's
// coordinates.  Forward (left spine): a child's K = kpiv + 1 with the
// pivot's diagonal kpiv in [kf - 2, kf], kf = (K + 1) / 2; reverse (right
// spine): a child's K = K - kpiv.  A descendant with M' + N' < 2 min_dim is
// a leaf (no pivot), which ends the spine.
void spine_windows(int64_t K, int rev, int64_t min_dim, std::vector<std::pair<int64_t, int64_t>>& out) {
    int64_t lo = K, hi = K;
    for (int depth = 0; depth < 64; depth++) {
        int64_t clo = INT64_MAX, chi = -1;
        for (int64_t k = lo; k <= hi; k++) {
            const int64_t kf = (k + 1) / 2;
            clo = std::min(clo, rev ? k - kf : kf - 1);
            chi = std::max(chi, rev ? k - kf + 2 : kf + 1);
        }
        if (chi + 1 < 2 * min_dim || clo < 2) break;
        int64_t dlo = INT64_MAX, dhi = -1;
        for (int64_t k = clo; k <= chi; k++) {
            const int64_t kf = (k + 1) / 2, kstop = rev ? kf + ((k % 2 == 0) ? 1 : 0) : kf;
            dlo = std::min(dlo, kstop - 2);
            dhi = std::max(dhi, kstop);
        }
        out.push_back({std::max<int64_t>(dlo, 0), dhi});
        lo = clo;
        hi = chi;
    }
}

struct Engine {
    Ctx& c;
    int prec, d, dp, H;  // dp: padded row length (elements); H: strip height of the launch being built
    int lat = 0;         // the launch being built uses the latency variant (strip_height(.., 1))
    void* out_base = nullptr;  // diagonal outputs of run_wave (null: the slot's buffer)
    // half-pass reuse (align_core): saved passes and the arena fill (elements)
    bool reuse = false;
    int windows_policy = 1;  // LMDTW_WINDOWS: 1 not for latency-bound batches, 2 always
    int64_t min_dim = 500;
    std::vector<SavedPass> saved;
    int64_t arena_used = 0;
    int lat_policy = 1;  // LMDTW_LAT: 0 never, 1 latency-bound launches, 2 always
    void set_lat(int l) {
        (void)l;  // the latency variant is not dispatched (kernels.cu, WsCfg::R)
        lat = 0;
        H = strip_height(prec, dpl, lat);
    }
    // A launch is latency-bound when its longest strip has more serial tiles
    // than the launch has tiles per pipeline (twice over): the head strips'
    // chain, not the FMA pipes, then sets the time.
    bool latency_bound(const std::vector<PassDesc>& P) {
        const int nsm = c.nsm;
        int64_t head = 0, tiles = 0;
        for (const auto& p : P) {
            head = std::max<int64_t>(head, tiles_of(p, p.strip_lo, H));
            for (int a = p.strip_lo; a < p.strip_hi; a++) tiles += tiles_of(p, a, H);
        }
        return head > 2.0 * (double)tiles / ((double)pipes_per_cta(prec, dpl, lat) * nsm);
    }
    DimPlan dpl;
    size_t esz;
    int tie[3] = {2, 0, 1};
    Engine(Ctx& ctx, int precision, int dim) : c(ctx), prec(precision), d(dim) {
        dpl = plan_dims(prec, d);
        dp = dpl.dp;
        H = strip_height(prec, dpl);
        lat_policy = 0;  // the latency variant is not dispatched (see WsCfg::R)
        esz = prec == 32 ? 4 : 8;
    }

    // 64-bit words per boundary element (tagged handoff, see kernels.cu)
    int64_t bwords() const { return prec == 32 ? 1 : 2; }

    int launched(cudaError_t e, const char* what) {
        if (e != cudaSuccess) return cuda_err(e, what);
        c.call_launches++;
        g_launches++;
        return LMDTW_OK;
    }

    // Copy features (host or device float32) into the padded dtype arrays.
    int stage(const float* const* src, const int64_t* rows, int n, int mem, bool isx, std::vector<int64_t>& base) {
        int64_t total = 0;
        base.resize(n);
        for (int p = 0; p < n; p++) {
            base[p] = total;
            total += rows[p];
        }
        DBuf& raw = isx ? c.xraw : c.yraw;
        DBuf& pad = isx ? c.xp : c.yp;
        // kPadRows zero rows before and after (see kernels.cu); row r of the
        // concatenated series lives at padded row kPadRows + r.
        const size_t rowb = (size_t)dp * esz;
        CU(pad.ensure((size_t)(total + 2 * kPadRows) * rowb));
        char* body = (char*)pad.p + kPadRows * rowb;  // the guard rows: the first / last cast launch
        if (mem == LMDTW_MEM_HOST) {
            CU(raw.ensure((size_t)total * d * sizeof(float)));
            for (int p = 0; p < n; p++) {
                CU(cudaMemcpyAsync(raw.as<float>() + base[p] * d, src[p], (size_t)rows[p] * d * sizeof(float),
                                   cudaMemcpyHostToDevice, c.st));
                c.h2d += (long long)rows[p] * d * sizeof(float);
            }
            TRY(launched(launch_pad_cast(prec, raw.as<float>(), total, d, dp, body, c.st, kPadRows, kPadRows),
                         "pad_cast"));
        } else {
            for (int p = 0; p < n; p++) {
                char* dst = body + (size_t)base[p] * rowb;
                TRY(launched(launch_pad_cast(prec, src[p], rows[p], d, dp, dst, c.st, p == 0 ? kPadRows : 0,
                                             p == n - 1 ? kPadRows : 0),
                             "pad_cast"));
            }
        }
        for (int p = 0; p < n; p++) base[p] += kPadRows;
        return LMDTW_OK;
    }

    // Work queue of tiles (pass, strip a, column block b), ordered by the
    // tile's earliest start b*W + a*kLagKey: a strip trails the strip above
    // it by a short lag and its own previous tile by a tile width, so both
    // predecessors of a tile come earlier in the queue -- the persistent
    // kernel's deadlock freedom -- and pipelines rotate over the strips
    // instead of holding a long strip while shorter ones wait behind it.
    // LMDTW_LAG_KEY (experiments): a divisor of kTileW; default 128
    static int64_t lag_key() {
        static const int64_t v = [] {
            const char* e = getenv("LMDTW_LAG_KEY");
            const int64_t k = e ? atoll(e) : 128;
            return (k >= 16 && kTileW % k == 0) ? k : 128;
        }();
        return v;
    }
    static int64_t tiles_of(const PassDesc& p, int a, int H) {
        const int64_t jend = std::min<int64_t>(p.N - 1, (int64_t)p.kstop - (int64_t)a * H);
        return jend / kTileW + 1;
    }
    // Host side of the queue build: O(strips + keys) work.  The per-key counts
    // come from a difference array along each residue class m = a (mod kPer)
    // (strip a's tiles are the keys a, a+kPer, ..., a+(nb-1)*kPer); their
    // exclusive prefix sum is each key's first queue slot.  The tiles
    // themselves are scattered on the device (scatter_items_kernel), so the
    // host never touches the O(tiles) queue.  Returns the number of tiles.
    int64_t stage_items(Slot& S, const std::vector<PassDesc>& P, int64_t& nents, int64_t& nkeys, size_t& ents_off,
                        size_t& cur_off) {
        const int64_t kPer = kTileW / lag_key();
        int64_t mmax = 0, total = 0;
        nents = 0;
        for (const auto& p : P) {
            nents += p.strip_hi - p.strip_lo;
            for (int a = p.strip_lo; a < p.strip_hi; a++) {
                const int64_t nb = tiles_of(p, a, H);
                mmax = std::max<int64_t>(mmax, (nb - 1) * kPer + a);
                total += nb;
            }
        }
        nkeys = mmax + 1;
        ents_off = S.stg.reserve((size_t)nents * sizeof(StripEnt));
        cur_off = S.stg.reserve((size_t)(nkeys + kPer) * sizeof(int32_t));
        StripEnt* ents = S.stg.at<StripEnt>(ents_off);
        int32_t* cnt = S.stg.at<int32_t>(cur_off);
        std::fill(cnt, cnt + nkeys + kPer, 0);
        int64_t e = 0;
        for (size_t q = 0; q < P.size(); q++)
            for (int a = P[q].strip_lo; a < P[q].strip_hi; a++) {
                const int64_t nb = tiles_of(P[q], a, H);
                ents[e++] = StripEnt{(int32_t)q, a, (int32_t)nb};
                cnt[a]++;
                cnt[a + nb * kPer]--;
            }
        for (int64_t m = kPer; m < nkeys; m++) cnt[m] += cnt[m - kPer];  // per-key tile counts
        int64_t run = 0;
        for (int64_t m = 0; m < nkeys; m++) {  // exclusive scan: first slot of key m
            const int64_t n = cnt[m];
            cnt[m] = (int32_t)run;
            run += n;
        }
        if (run != total) return -1;
        return total;
    }

    // The slot's staged batch to the device: one pinned copy, one H2D copy on
    // the slot's stream; the staging is then empty for the next batch.  (The
    // slot's previous batch has completed: callers sync on it first.)
    int upload(Slot& S) {
        const size_t n = std::max<size_t>(S.stg.h.size(), 16);
        CU(S.h_stage.ensure(n));
        memcpy(S.h_stage.p, S.stg.h.data(), S.stg.h.size());
        CU(S.d_stage.ensure(n));
        CU(cudaMemcpyAsync(S.d_stage.p, S.h_stage.p, S.stg.h.size(), cudaMemcpyHostToDevice, S.st));
        S.stg.h.clear();
        return LMDTW_OK;
    }

    // Tile queue of passes P (staged, not yet uploaded): the scatter kernel
    // runs after upload() from the offsets recorded here.
    struct QueueStage {
        int64_t nitems = 0, nents = 0;
        size_t ents_off = 0, cur_off = 0;
    };
    int stage_queue(Slot& S, const std::vector<PassDesc>& P, QueueStage& q) {
        int64_t nkeys = 0;
        q.nitems = stage_items(S, P, q.nents, nkeys, q.ents_off, q.cur_off);
        if (q.nitems < 0 || q.nitems > INT32_MAX) return set_err(LMDTW_EINTERNAL, "tile queue size");
        CU(S.items.ensure((size_t)std::max<int64_t>(q.nitems, 1) * sizeof(WorkItem)));
        return LMDTW_OK;
    }
    int scatter_queue(Slot& S, const QueueStage& q) {
        return launched(launch_scatter_items(S.dev<StripEnt>(q.ents_off), (int)q.nents, S.dev<int32_t>(q.cur_off),
                                             (int)(kTileW / lag_key()), S.items.as<WorkItem>(), S.st),
                        "scatter_items_kernel");
    }

    // Build the tile queue of passes P in S.items (device), on S.st (entry
    // points that upload their own descriptors).
    int upload_queue(Slot& S, const std::vector<PassDesc>& P, int64_t& nitems) {
        QueueStage q;
        TRY(stage_queue(S, P, q));
        TRY(upload(S));
        nitems = q.nitems;
        return scatter_queue(S, q);
    }

    // Handoff tags of a launch over `bnd`: strip a of the launch tags its words
    // tag_base + a, above every tag an earlier launch on the buffer used, so
    // stale words never match and the buffer needs no reset between launches
    // (a new allocation is all tag -1; the base restarts, with a reset, near
    // 2^30).
    int next_tags(Slot& S, int64_t nstrips_max, int& tag_base) {
        const int64_t span = nstrips_max + 2;
        if ((int64_t)S.tag_next + span >= (1LL << 30)) {
            CU(cudaMemsetAsync(S.bnd.p, 0xFF, S.bnd.cap, S.st));
            S.tag_next = 0;
        }
        tag_base = S.tag_next;
        S.tag_next += (int)span;
        return LMDTW_OK;
    }

    // Host-built queue (debug entry points only): same order as the device
    // scatter up to the order of tiles that share a key.
    void make_items(Slot& S, const std::vector<PassDesc>& P, std::vector<WorkItem>& items) {
        const int64_t kPer = kTileW / lag_key();
        int64_t nents = 0, nkeys = 0;
        size_t ents_off = 0, cur_off = 0;
        const int64_t total = stage_items(S, P, nents, nkeys, ents_off, cur_off);
        std::vector<int32_t> cur(S.stg.at<int32_t>(cur_off), S.stg.at<int32_t>(cur_off) + nkeys);
        S.stg.h.clear();
        items.resize(std::max<int64_t>(total, 0));
        for (size_t q = 0; q < P.size(); q++)
            for (int a = P[q].strip_lo; a < P[q].strip_hi; a++)
                for (int64_t b = 0; b < tiles_of(P[q], a, H); b++)
                    items[cur[b * kPer + a]++] = WorkItem{(int)q, a, (int)b, 0};
    }

    // One wave launch over passes P0: stages its descriptors and tile queue
    // after whatever the caller staged in S.stg (wins_off: the caller's
    // WinDesc array there, or npos), uploads the batch in one copy, builds the
    // queue and launches.  The batch's device offsets stay valid until the
    // slot's next upload (S.passes_off: the PassDesc array).
    static constexpr size_t npos = ~(size_t)0;
    int run_wave(Slot& S, const std::vector<PassDesc>& P0, int64_t bnd_total, bool leaf, void* tab, void* lcost,
                 int64_t cells, size_t wins_off = npos) {
        const auto th0 = std::chrono::steady_clock::now();
        // tile bookkeeping: per strip H+1 boundary values and a completion count
        std::vector<PassDesc> P(P0);
        int64_t lb_total = 0, flag_total = 0;
        for (auto& p : P) {
            p.tile_w = kTileW;
            p.lb_off = lb_total;
            p.flag_off = flag_total;
            lb_total += (int64_t)p.nstrips * (H + 1);
            flag_total += p.nstrips;
        }
        // buffers the kernel leaves clean (flags, counters) or never needs
        // clean (handoff words, by their tags): initialised at allocation only
        CU(S.lb.ensure((size_t)std::max<int64_t>(lb_total, 1) * esz));
        CU(S.flags.ensure_init((size_t)std::max<int64_t>(flag_total, 1) * sizeof(int), 0, S.st));
        CU(S.counter.ensure_init(2 * sizeof(int), 0, S.st));
        CU(S.bnd.ensure_init((size_t)std::max<int64_t>(bnd_total, 1) * 8, 0xFF, S.st));
        int64_t smax = 0;
        for (const auto& p : P) smax = std::max<int64_t>(smax, p.nstrips);
        int tag_base = 0;
        TRY(next_tags(S, smax, tag_base));
        S.passes_off = S.stg.add(P.data(), P.size() * sizeof(PassDesc));
        QueueStage qs;
        TRY(stage_queue(S, P, qs));
        TRY(upload(S));
        TRY(scatter_queue(S, qs));
        const int64_t nitems = qs.nitems;
        WaveLaunch w{};
        w.tag_base = tag_base;
        w.X = c.xp.p;
        w.Y = c.yp.p;
        w.dp = dp;
        w.wide = dpl.wide;
        w.precision = prec;
        w.passes = S.dev<PassDesc>(S.passes_off);
        w.items = S.items.as<WorkItem>();
        w.nitems = (int)nitems;
        w.counter = S.counter.as<int>();
        w.out = out_base ? out_base : S.out.p;
        w.wins = wins_off == npos ? nullptr : S.dev<WinDesc>(wins_off);
        w.bnd = S.bnd.p;
        w.bp = c.bp.as<unsigned long long>();
        w.lb = S.lb.p;
        if (const char* d = getenv("LMDTW_PROBE")) w.dbg = atoi(d);  // LMDTW_PROBES builds only
        // Latency-bound level: the longest strip has more serial tiles than the
        // level has tiles per pipeline -> half the pipelines per SM, so the
        // head strips run with more of their SM (LMDTW_ACTIVE_NP overrides).
        {
            const int nsm = c.nsm;
            const int np = pipes_per_cta(prec, dpl, lat);
            int64_t head = 0;
            for (const auto& p : P) head = std::max<int64_t>(head, tiles_of(p, p.strip_lo, H));
            const double per_pipe = (double)nitems / ((double)np * nsm);
            // LMDTW_LAT_FACTOR (experiments): the head / per-pipeline tile ratio above which
            // a launch counts as latency-bound (default 2)
            static const double lat_factor = [] {
                const char* e = getenv("LMDTW_LAT_FACTOR");
                const double f = e ? atof(e) : 2.0;
                return f > 0 ? f : 2.0;
            }();
            w.active_np = (head > lat_factor * per_pipe && np >= 2) ? np / 2 : np;
            if (const char* a = getenv("LMDTW_ACTIVE_NP")) w.active_np = atoi(a);
        }
        w.flags = S.flags.as<int>();
        w.tab = tab;
        w.leaf_cost = lcost;
        w.tie0 = tie[0];
        w.tie1 = tie[1];
        w.tie2 = tie[2];
        w.leaf = leaf ? 1 : 0;
        w.grid_warps = 0;
        w.lat = lat;
        // LMDTW_TRACE_FILE: append per-strip DP start/end timestamps (debug)
        const char* trace_file = getenv("LMDTW_TRACE_FILE");
        if (trace_file) {
            CU(S.trace.ensure(nitems * 24));
            CU(cudaMemsetAsync(S.trace.p, 0, nitems * 24, S.st));
            w.trace = S.trace.as<unsigned long long>();
        }
        const bool prof = g_profile.load() != 0;
        if (getenv("LMDTW_HOST_TIMING"))
            fprintf(stderr, "lmdtw host: %lld items prepared in %.1f us\n", (long long)nitems,
                    std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - th0).count());
        int pe0 = -1, pe1 = -1;
        if (prof) {
            CU(c.prof_event(&pe0));
            CU(c.prof_event(&pe1));
            CU(cudaEventRecord(c.evpool[pe0], S.st));
        }
        if (getenv("LMDTW_HOST_TIMING")) {  // device-idle gap since the last sync point
            cudaEvent_t ev;
            cudaEventCreate(&ev);
            cudaEventRecord(ev, S.st);
            cudaEventSynchronize(ev);
            float ms = 0;
            if (g_last_sync_ev) cudaEventElapsedTime(&ms, g_last_sync_ev, ev);
            fprintf(stderr, "lmdtw host: device idle %.1f us before this wave launch\n", 1e3 * ms);
            cudaEventDestroy(ev);
        }
        TRY(launched(launch_wave(w, S.st), leaf ? "leaf wave_kernel" : "wave_kernel"));
        if (trace_file) {
            std::vector<unsigned long long> tr(nitems * 3);
            std::vector<WorkItem> items(nitems);
            CU(cudaMemcpyAsync(tr.data(), S.trace.p, tr.size() * 8, cudaMemcpyDeviceToHost, S.st));
            CU(cudaMemcpyAsync(items.data(), S.items.p, nitems * sizeof(WorkItem), cudaMemcpyDeviceToHost, S.st));
            CU(cudaStreamSynchronize(S.st));
            if (FILE* f = fopen(trace_file, "ab")) {
                const long long hdr[3] = {(long long)P.size(), (long long)items.size(), (long long)leaf};
                fwrite(hdr, sizeof hdr, 1, f);
                fwrite(P.data(), sizeof(PassDesc), P.size(), f);
                fwrite(items.data(), sizeof(WorkItem), items.size(), f);
                fwrite(tr.data(), 8, tr.size(), f);
                fclose(f);
            }
        }
        if (prof) {
            CU(cudaEventRecord(c.evpool[pe1], S.st));
            c.pend.push_back(Ctx::Pend{pe0, pe1, (long long)cells, leaf});
        }
        return LMDTW_OK;
    }

    PassDesc half_pass_desc(int64_t x_off, int64_t y_off, int64_t M, int64_t N, int64_t kstop, int rev,
                            int64_t& out_total, int64_t& bnd_total) {
        PassDesc p{};
        p.x_off = x_off;
        p.y_off = y_off;
        p.M = (int32_t)M;
        p.N = (int32_t)N;
        p.kstop = (int32_t)kstop;
        p.reverse = rev;
        p.rows = (int32_t)std::min<int64_t>(M, kstop + 1);
        p.nstrips = (p.rows + H - 1) / H;
        for (int s = 0; s < 3; s++) {
            p.out_off[s] = out_total;
            out_total += dlen(kstop - 2 + s, M, N);
        }
        for (int s = 0; s < 3; s++) {
            p.out_off[3 + s] = out_total;
            out_total += dlen(kstop - 2 + s, M, N);
        }
        p.bnd_off = bnd_total;
        bnd_total += 2 * ((N + 1) & ~1LL) * bwords();  // two slots, 16-byte aligned
        p.strip_lo = 0;
        p.strip_hi = p.nstrips;
        p.bnd_in_first = 0;
        p.sys_out = 0;
        p.bp_off = 0;
        p.tab_off = -1;
        p.bp_ld = 0;
        p.leaf_id = -1;
        p.win_first = 0;
        p.win_count = 0;
        return p;
    }

    // Batched find_pivot over `nodes` (indices into `all`).
    // pivot_launch: everything for one batch on slot S's stream, ending with
    // the pivots' device->host copy and S.done; pivot_collect reads them back
    // once S.done has completed.
    int pivot_launch(Slot& S, std::vector<Node>& all, const std::vector<int>& nodes, const std::vector<int64_t>& xb,
                     const std::vector<int64_t>& yb, std::vector<int64_t>* cells_out,
                     std::vector<int64_t>* peak_out, int highest) {
        std::vector<PassDesc> P;
        std::vector<PivotDesc> V;
        int64_t out_total = 0, bnd_total = 0, cells = 0;
        // latency variant for latency-bound batches (decided on the default strips)
        set_lat(0);
        if (lat_policy == 2) {
            set_lat(1);
        } else if (lat_policy == 1) {
            for (int q : nodes) {
                const Node& n = all[q];
                const int64_t K = n.M + n.N - 1, kf = (K + 1) / 2, kb = (K % 2 == 0) ? kf + 1 : kf;
                P.push_back(half_pass_desc(0, 0, n.M, n.N, kf, 0, out_total, bnd_total));
                P.push_back(half_pass_desc(0, 0, n.M, n.N, kb, 1, out_total, bnd_total));
            }
            const bool lb = latency_bound(P);
            P.clear();
            out_total = bnd_total = 0;
            set_lat(lb ? 1 : 0);
        }
        P.reserve(nodes.size() * 2);
        // Outputs: with reuse (align_core) every diagonal lives in the per-call
        // arena at a stable offset (saved windows outlive the batch);
        // otherwise in the slot's buffer from offset 0.
        const int64_t base0 = reuse ? arena_used : 0;
        out_total = base0;
        std::vector<WinDesc> W;
        int64_t computed = 0;  // cells the wave kernel actually updates
        // Windows put stores on the strips' DP path: a latency-bound batch
        // (its head strips set the time) saves none -- its children then
        // compute both half passes (inherited_pass finds no window).
        bool save_windows = reuse;
        if (reuse && windows_policy == 1) {
            std::vector<PassDesc> probe;
            int64_t o = 0, bt = 0;
            for (int q : nodes) {
                const Node& n = all[q];
                const int64_t K = n.M + n.N - 1, kf = (K + 1) / 2, kb = (K % 2 == 0) ? kf + 1 : kf;
                if (!(n.fsrc >= 0)) probe.push_back(half_pass_desc(0, 0, n.M, n.N, kf, 0, o, bt));
                if (!(n.bsrc >= 0)) probe.push_back(half_pass_desc(0, 0, n.M, n.N, kb, 1, o, bt));
            }
            save_windows = !latency_bound(probe);
        }
        auto computed_pass = [&](const Node& n, int64_t kstop, int rev) -> int {
            PassDesc p = half_pass_desc(xb[n.pair] + n.i_off, yb[n.pair] + n.j_off, n.M, n.N, kstop, rev,
                                        out_total, bnd_total);
            computed += cells_upto(kstop, n.M, n.N);
            if (!save_windows) {
                P.push_back(p);
                return -1;
            }
            std::vector<std::pair<int64_t, int64_t>> rng;
            spine_windows(n.M + n.N - 1, rev, min_dim, rng);
            // A window costs every strip of this pass ~8 chunks of stores on
            // its DP path; it saves one half pass of a descendant whose
            // M' + N' ~ 2 * (the window's middle k): keep it only where the
            // saved cells outweigh ~2x the cells of those chunks (measured:
            // storing all 8 windows of cfg3's root passes cost 3.6% of level 0)
            {
                const double cost = 2.0 * p.nstrips * 8.0 * 16.0 * H;
                std::vector<std::pair<int64_t, int64_t>> keep;
                for (auto& r : rng) {
                    const double half = (double)(r.first + r.second) / 2.0;  // ~ the descendant's kf ~ (M'+N')/2
                    const double saved_cells = half * half / 2.0;          // its half pass, ~square
                    if (saved_cells > cost) keep.push_back(r);
                }
                rng.swap(keep);
            }
            std::sort(rng.begin(), rng.end());  // the kernel walks windows in increasing k
            SavedPass sp;
            sp.M = n.M;
            sp.N = n.N;
            p.win_first = (int32_t)W.size();
            for (auto& r : rng) {
                if (r.second > kstop - 3) continue;  // never past the pass's own last diagonals
                WinDesc wd{};
                wd.k_lo = (int32_t)r.first;
                wd.k_hi = (int32_t)r.second;
                int64_t stride = 0;
                for (int64_t k = r.first; k <= r.second; k++) stride = std::max(stride, dlen(k, n.M, n.N));
                wd.stride = (int32_t)stride;
                wd.d_off = out_total;
                out_total += (r.second - r.first + 1) * stride;
                wd.c_off = out_total;
                out_total += (r.second - r.first + 1) * stride;
                W.push_back(wd);
                sp.wins.push_back(wd);
            }
            p.win_count = (int32_t)W.size() - p.win_first;
            P.push_back(p);
            saved.push_back(std::move(sp));
            return (int)saved.size() - 1;
        };
        // a pass inherited from a saved one: a descriptor the pivot kernel
        // reads (no strips), its offsets pointing into the saved windows
        auto inherited_pass = [&](const Node& n, int src, int64_t kstop) -> bool {
            const SavedPass& sp = saved[src];
            PassDesc p{};
            for (int s3 = 0; s3 < 3; s3++) {
                const int64_t k = kstop - 2 + s3;
                const WinDesc* w = nullptr;
                for (const auto& wd : sp.wins)
                    if (k >= wd.k_lo && k <= wd.k_hi) w = &wd;
                if (!w) return false;
                // the node's diag index idx is the saved pass's idx + shift
                const int64_t shift = std::min(k, sp.M - 1) - std::min(k, n.M - 1);
                p.out_off[s3] = w->d_off + (k - w->k_lo) * w->stride + shift;
                p.out_off[3 + s3] = w->c_off + (k - w->k_lo) * w->stride + shift;
            }
            p.M = (int32_t)n.M;
            p.N = (int32_t)n.N;
            p.kstop = (int32_t)kstop;
            P.push_back(p);
            return true;
        };
        for (int q : nodes) {
            Node& n = all[q];
            const int64_t K = n.M + n.N - 1;
            const int64_t kf = (K + 1) / 2;
            const int64_t kb = (K % 2 == 0) ? kf + 1 : kf;
            PivotDesc v{};
            v.fwd = (int)P.size();
            if (reuse && n.fsrc >= 0 && inherited_pass(n, n.fsrc, kf))
                n.fpass = n.fsrc;
            else
                n.fpass = computed_pass(n, kf, 0);
            v.bwd = (int)P.size();
            if (reuse && n.bsrc >= 0 && inherited_pass(n, n.bsrc, kb))
                n.bpass = n.bsrc;
            else
                n.bpass = computed_pass(n, kb, 1);
            v.M = (int)n.M;
            v.N = (int)n.N;
            v.kf = (int)kf;
            v.kb = (int)kb;
            v.highest = highest;
            V.push_back(v);
            const int64_t cl = cells_upto(kf, n.M, n.N) + cells_upto(kb, n.M, n.N);
            cells += cl;
            if (cells_out) cells_out->push_back(cl);
            if (peak_out)
                peak_out->push_back(std::max(peak_values(kf, n.M, n.N), peak_values(kb, n.M, n.N)));
        }
        if (reuse) {
            CU(c.arena.grow_keep((size_t)std::max<int64_t>(out_total, 1) * esz, (size_t)arena_used * esz, S.st));
            arena_used = out_total;
            out_base = c.arena.p;
        } else {
            CU(S.out.ensure((size_t)std::max<int64_t>(out_total, 1) * esz));
            out_base = S.out.p;
        }
        // one upload for the batch: windows and pivot descriptors ride with
        // run_wave's pass descriptors and queue input
        (void)cells;
        const size_t wins_off = W.empty() ? npos : S.stg.add(W.data(), W.size() * sizeof(WinDesc));
        const size_t pdesc_off = S.stg.add(V.data(), V.size() * sizeof(PivotDesc));
        TRY(run_wave(S, P, bnd_total, false, nullptr, nullptr, computed, wins_off));
        CU(S.pout.ensure(V.size() * sizeof(PivotOut)));
        CU(S.h_pout.ensure(V.size() * sizeof(PivotOut)));
        const size_t scb = pivot_scratch_bytes((int)V.size());
        CU(S.pscratch.ensure(scb));
        CU(S.pdone.ensure_init(V.size() * sizeof(unsigned), 0, S.st));  // the kernel leaves them at zero
        TRY(launched(launch_pivots(prec, S.dev<PassDesc>(S.passes_off), S.dev<PivotDesc>(pdesc_off), (int)V.size(),
                                   out_base, S.pout.as<PivotOut>(), S.pscratch.p, S.pdone.as<unsigned>(), S.st),
                     "pivot_kernel"));
        CU(cudaMemcpyAsync(S.h_pout.p, S.pout.p, V.size() * sizeof(PivotOut), cudaMemcpyDeviceToHost, S.st));
        c.d2h += V.size() * sizeof(PivotOut);
        CU(cudaEventRecord(S.done, S.st));
        return LMDTW_OK;
    }
    void pivot_collect(Slot& S, std::vector<Node>& all, const std::vector<int>& nodes) {
        const PivotOut* po = S.h_pout.as<PivotOut>();
        for (size_t q = 0; q < nodes.size(); q++) {
            Node& n = all[nodes[q]];
            n.pi = po[q].i;
            n.pj = po[q].j;
            n.k = po[q].k;
            n.total = po[q].total;
        }
    }
    // Synchronous batch (single-level entry points).
    int pivot_level(Slot& S, std::vector<Node>& all, const std::vector<int>& nodes, const std::vector<int64_t>& xb,
                    const std::vector<int64_t>& yb, std::vector<int64_t>* cells_out,
                    std::vector<int64_t>* peak_out, int highest) {
        TRY(pivot_launch(S, all, nodes, xb, yb, cells_out, peak_out, highest));
        CU(cudaEventSynchronize(S.done));
        pivot_collect(S, all, nodes);
        return LMDTW_OK;
    }

    // Batched dtw_full over leaf nodes.  Fills per-leaf reversed paths (local
    // coordinates), per-cell costs, lengths, and D[M-1,N-1].
    int leaves(const std::vector<Node>& all, const std::vector<int>& leafs, const std::vector<int64_t>& xb,
               const std::vector<int64_t>& yb, void* tab_host, std::vector<int64_t>& path_off,
               std::vector<int>& plen) {
        const int n = (int)leafs.size();
        {
            static const int leaf_lat = [] {
                const char* e = getenv("LMDTW_LAT_LEAF");  // leaves in the latency variant
                return e ? atoi(e) : 0;
            }();
            set_lat(leaf_lat);
        }
        std::vector<PassDesc> P(n);
        std::vector<LeafDesc> L(n);
        int64_t bnd_total = 0, bp_total = 0, path_total = 0, cells = 0;
        path_off.resize(n);
        for (int q = 0; q < n; q++) {
            const Node& nd = all[leafs[q]];
            PassDesc& p = P[q];
            p = PassDesc{};
            p.x_off = xb[nd.pair] + nd.i_off;
            p.y_off = yb[nd.pair] + nd.j_off;
            p.M = (int32_t)nd.M;
            p.N = (int32_t)nd.N;
            p.kstop = (int32_t)(nd.M + nd.N - 2);
            p.reverse = 0;
            p.rows = (int32_t)nd.M;
            p.nstrips = (p.rows + H - 1) / H;
            p.strip_lo = 0;
            p.strip_hi = p.nstrips;
            p.bnd_in_first = 0;
            p.sys_out = 0;
            p.bnd_off = bnd_total;
            bnd_total += 2 * ((nd.N + 1) & ~1LL) * bwords();  // two slots, 16-byte aligned
            // block-major words: block jw of row i at bp_off + jw * bp_ld + i,
            // rows padded to whole strips (a strip's row-less lanes store too)
            p.bp_ld = (int32_t)(p.nstrips * H);
            p.bp_off = bp_total;
            bp_total += (int64_t)p.bp_ld * ((nd.N + 31) / 32);
            p.tab_off = tab_host ? 0 : -1;
            p.leaf_id = q;
            LeafDesc& l = L[q];
            l = LeafDesc{};
            l.x_off = p.x_off;
            l.y_off = p.y_off;
            l.M = p.M;
            l.N = p.N;
            l.pass = q;
            l.path_off = path_total;
            l.bp_off = p.bp_off;
            l.bp_ld = p.bp_ld;
            path_off[q] = path_total;
            path_total += nd.M + nd.N - 1;
            cells += nd.M * nd.N;
        }
        CU(c.bp.ensure((size_t)std::max<int64_t>(bp_total, 1) * 8));
        auto al = [](size_t x) { return (x + 15) & ~(size_t)15; };
        c.lo_pcost = al((size_t)path_total * 2 * sizeof(int));
        c.lo_plen = c.lo_pcost + al((size_t)path_total * esz);
        c.lo_lcost = c.lo_plen + al((size_t)n * sizeof(int));
        const size_t lbytes = c.lo_lcost + (size_t)n * esz;
        CU(c.lout.ensure(lbytes));
        CU(c.h_lout.ensure(lbytes));
        char* lo = c.lout.as<char>();
        void* tab_dev = nullptr;
        if (tab_host) {
            CU(c.tab.ensure((size_t)all[leafs[0]].M * all[leafs[0]].N * esz));
            tab_dev = c.tab.p;
        }
        const size_t ldesc_off = c.main.stg.add(L.data(), n * sizeof(LeafDesc));  // uploaded with the fill's batch
        TRY(run_wave(c.main, P, bnd_total, true, tab_dev, lo + c.lo_lcost, cells));
        TRY(launched(launch_backtrace(prec, dpl, c.xp.p, c.yp.p, c.main.dev<LeafDesc>(ldesc_off), n,
                                      c.bp.as<unsigned long long>(), reinterpret_cast<int*>(lo), lo + c.lo_pcost,
                                      reinterpret_cast<int*>(lo + c.lo_plen), c.st),
                     "backtrace_kernel"));
        CU(cudaMemcpyAsync(c.h_lout.p, lo, lbytes, cudaMemcpyDeviceToHost, c.st));
        c.d2h += (long long)path_total * (2 * sizeof(int) + esz) + n * (sizeof(int) + esz);
        if (tab_host) {
            const size_t tb = (size_t)all[leafs[0]].M * all[leafs[0]].N * esz;
            CU(cudaMemcpyAsync(tab_host, tab_dev, tb, cudaMemcpyDeviceToHost, c.st));
            c.d2h += tb;
        }
        CU(cudaStreamSynchronize(c.st));
        c.prof_collect();
        plen.assign(c.hplen(), c.hplen() + n);
        for (int q = 0; q < n; q++)
            if (plen[q] < 0) {
                const Node& nd = all[leafs[q]];
                char buf[160];
                snprintf(buf, sizeof buf, "backtrace hit SELF before (0, 0) in %lldx%lld leaf",
                         (long long)nd.M, (long long)nd.N);
                return set_err(LMDTW_EINTERNAL, buf);
            }
        return LMDTW_OK;
    }

    double leaf_cost(int q) const {
        return prec == 32 ? (double)c.hlcost<float>()[q] : c.hlcost<double>()[q];
    }
};

template <typename T> double seq_sum(const std::vector<const T*>& parts, const std::vector<int>& lens) {
    T total = T(0);
    for (size_t p = 0; p < parts.size(); p++)
        for (int q = 0; q < lens[p]; q++) total = total + parts[p][q];
    return (double)total;
}

int validate_common(int64_t M, int64_t N, int d, int prec) {
    if (M < 1 || N < 1) return set_err(LMDTW_EINVAL, "series must have length >= 1");
    if (d < 1) return set_err(LMDTW_EINVAL, "feature dimension must be >= 1");
    if (prec != 32 && prec != 64) return set_err(LMDTW_EINVAL, "precision must be 32 or 64");
    if (plan_dims(prec, d).dp < 0) {
        char buf[128];
        snprintf(buf, sizeof buf, "feature dimension %d exceeds the supported maximum (%d)", d, lmdtw_max_dim(prec));
        return set_err(LMDTW_EINVAL, buf);
    }
    if (M + N > (int64_t)1 << 30) return set_err(LMDTW_EINVAL, "M + N too large (limit 2^30)");
    return LMDTW_OK;
}

int validate_tie(const int32_t* tie) {
    int seen = 0;
    for (int q = 0; q < 3; q++) {
        if (tie[q] < 0 || tie[q] > 2) return set_err(LMDTW_EINVAL, "tie codes must be a permutation of 0,1,2");
        seen |= 1 << tie[q];
    }
    if (seen != 7) return set_err(LMDTW_EINVAL, "tie codes must be a permutation of 0,1,2");
    return LMDTW_OK;
}

// Core of lmdtw_align / lmdtw_align_batch.
int align_core(int device, int npairs, const float* const* X, const int64_t* M, const float* const* Y,
               const int64_t* N, int d, const lmdtw_config_t& cfg, int mem, lmdtw_progress_fn progress, void* user,
               std::vector<lmdtw_result*>& results) {
    if (npairs < 1) return set_err(LMDTW_EINVAL, "npairs must be >= 1");
    for (int p = 0; p < npairs; p++) TRY(validate_common(M[p], N[p], d, cfg.precision));
    if (cfg.min_dim < 2) return set_err(LMDTW_EINVAL, "min_dim must be >= 2");
    TRY(validate_tie(cfg.tie));
    if (cfg.pivot_highest != 0 && cfg.pivot_highest != 1) return set_err(LMDTW_EINVAL, "unknown pivot_tie_rule");
    CtxLease c;
    TRY(lease_ctx(device, c));
    CU(cudaSetDevice(device));
    c->call_launches = 0;
    c->h2d = c->d2h = 0;
    Engine E(*c, cfg.precision, d);
    E.tie[0] = cfg.tie[0];
    E.tie[1] = cfg.tie[1];
    E.tie[2] = cfg.tie[2];
    // Half-pass reuse: a left child's forward half pass is its parent's
    // forward pass restricted to the top-left block (same first cell, the
    // same recurrence, bit-identical values), a right child's reverse pass
    // likewise; each pass saves the diagonals its spine descendants need, so
    // every node below the root computes one half pass instead of two.
    // cells_processed keeps the reference's count (both half passes of every
    // node, divide.py:148-178).  LMDTW_REUSE=0 computes both.
    {
        const char* e = getenv("LMDTW_REUSE");
        E.reuse = !(e && atoi(e) == 0);
        const char* w = getenv("LMDTW_WINDOWS");
        E.windows_policy = w ? atoi(w) : 1;
        E.min_dim = cfg.min_dim;
        E.arena_used = 0;
        E.saved.clear();
    }
    std::vector<int64_t> xb, yb;
    // LMDTW_PHASES=1: host timestamps of the phases of this call (diagnostics)
    const bool phases = getenv("LMDTW_PHASES") != nullptr;
    const auto tp0 = std::chrono::steady_clock::now();
    auto phase = [&](const char* what) {
        if (phases)
            fprintf(stderr, "lmdtw phase %-18s %8.1f us\n", what,
                    std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - tp0).count());
    };
    phase("leased");
    TRY(E.stage(X, M, npairs, mem, true, xb));
    TRY(E.stage(Y, N, npairs, mem, false, yb));

    std::vector<Inst> inst(npairs);
    std::vector<Node> nodes;
    std::vector<int> level;
    for (int p = 0; p < npairs; p++) {
        inst[p].budget = 2 * M[p] * N[p];
        inst[p].cb = (npairs == 1) ? progress : nullptr;
        inst[p].user = user;
        Node n;
        n.i_off = 0;
        n.j_off = 0;
        n.M = M[p];
        n.N = N[p];
        n.pair = p;
        nodes.push_back(n);
        level.push_back((int)nodes.size() - 1);
    }
    // Dataflow over the recursion (replaces the level-synchronous loop): the
    // internal nodes whose sub-blocks are known form batches; a batch is one
    // wave launch (both half passes of each node) + one pivot launch + one
    // small D2H copy on its own stream and buffers (a Slot), so up to
    // kMaxFlights batches run concurrently -- a node's children start as soon
    // as its own batch has finished, while slower nodes of its level still
    // run; persistent CTAs of a draining batch exit and free SMs for the next.
    // Results never depend on the schedule (every node is the same
    // find_pivot call); the trace and path are rebuilt from the tree below.
    std::vector<int> leafs, ready;
    int64_t nlevels = 0;
    auto classify = [&](int q) {
        const Node& n = nodes[q];
        if (n.M < cfg.min_dim || n.N < cfg.min_dim || n.M + n.N <= 5) {
            nodes[q].leaf = (int)leafs.size();
            leafs.push_back(q);
        } else {
            ready.push_back(q);
            nlevels = std::max<int64_t>(nlevels, n.depth + 1);
        }
    };
    for (int q : level) classify(q);
    static const int kMaxFlights = [] {
        const char* e = getenv("LMDTW_MAX_FLIGHTS");
        // 1: one batch per recursion level (default: concurrent persistent
        // grids serialise -- the first holds every SM while its wavefront
        // ramps, measured 36 -> 52 ms at cfg3 with 8 slots)
        const int v = e ? atoi(e) : 1;
        return v < 1 ? 1 : (v > 32 ? 32 : v);
    }();
    // features padded and cast on c->st; batch slots on other streams wait for it
    cudaEvent_t staged = nullptr;
    if (kMaxFlights > 1) {
        CU(cudaEventCreateWithFlags(&staged, cudaEventDisableTiming));
        CU(cudaEventRecord(staged, c->st));
    }
    struct Flight {
        Slot* S;
        std::vector<int> ids;
        std::vector<int64_t> cells, peaks;
    };
    std::vector<Flight> flights;
    std::vector<Slot*> free_slots;
    auto slot_for = [&](size_t k) -> Slot* {
        if (k == 0) return &c->main;
        while (c->extra.size() < k) {
            std::unique_ptr<Slot> s(new Slot());
            if (cudaStreamCreateWithFlags(&s->st, cudaStreamNonBlocking) != cudaSuccess ||
                cudaEventCreateWithFlags(&s->done, cudaEventDisableTiming) != cudaSuccess)
                return nullptr;
            c->extra.push_back(std::move(s));
        }
        return c->extra[k - 1].get();
    };
    for (int k = kMaxFlights - 1; k >= 0; k--) {
        Slot* s = slot_for(k);
        if (!s) {
            if (staged) cudaEventDestroy(staged);
            return cuda_err(cudaGetLastError(), "batch stream");
        }
        free_slots.push_back(s);
    }
    int rc = LMDTW_OK;
    while (rc == LMDTW_OK && (!ready.empty() || !flights.empty())) {
        if (!ready.empty() && !free_slots.empty()) {
            // split the ready nodes over the free slots, longest first (LPT by
            // cells), but never into batches of fewer than ~1/8 of the ready
            // work when many nodes are ready (launch count stays per level)
            std::vector<int> order(ready);
            std::sort(order.begin(), order.end(), [&](int a, int b) {
                const int64_t ca = nodes[a].M * nodes[a].N, cb = nodes[b].M * nodes[b].N;
                return ca != cb ? ca > cb : a < b;
            });
            const size_t nb = std::min(free_slots.size(), order.size());
            std::vector<std::vector<int>> groups(nb);
            std::vector<int64_t> load(nb, 0);
            for (int q : order) {
                size_t g = 0;
                for (size_t k = 1; k < nb; k++)
                    if (load[k] < load[g]) g = k;
                groups[g].push_back(q);
                load[g] += nodes[q].M * nodes[q].N;
            }
            ready.clear();
            for (auto& g : groups) {
                if (g.empty()) continue;
                Flight f;
                f.S = free_slots.back();
                free_slots.pop_back();
                std::sort(g.begin(), g.end());
                f.ids = g;
                if (staged && f.S->st != c->st && cudaStreamWaitEvent(f.S->st, staged, 0) != cudaSuccess) {
                    rc = cuda_err(cudaGetLastError(), "cudaStreamWaitEvent");
                    break;
                }
                phase("batch launch");
                rc = E.pivot_launch(*f.S, nodes, f.ids, xb, yb, &f.cells, &f.peaks, cfg.pivot_highest);
                phase("batch launched");
                if (rc != LMDTW_OK) break;
                flights.push_back(std::move(f));
            }
            continue;
        }
        // a finished batch: the first whose event completed, else wait for the oldest
        size_t k = flights.size();
        for (size_t q = 0; q < flights.size() && k == flights.size(); q++) {
            const cudaError_t e = cudaEventQuery(flights[q].S->done);
            if (e == cudaSuccess) k = q;
            else if (e != cudaErrorNotReady) rc = cuda_err(e, "batch");
        }
        if (rc != LMDTW_OK) break;
        if (k == flights.size()) {
            k = 0;
            const cudaError_t e = cudaEventSynchronize(flights[0].S->done);
            if (e != cudaSuccess) {
                rc = cuda_err(e, "batch");
                break;
            }
        }
        phase("batch done");
        Flight f = std::move(flights[k]);
        flights.erase(flights.begin() + k);
        E.pivot_collect(*f.S, nodes, f.ids);
        free_slots.push_back(f.S);
        for (size_t q = 0; q < f.ids.size(); q++) {
            const int id = f.ids[q];
            Node parent = nodes[id];
            Inst& in = inst[parent.pair];
            in.peak_diag = std::max(in.peak_diag, f.peaks[q]);
            in.add_batch(f.cells[q]);
            Node l, r;
            l.i_off = parent.i_off;
            l.j_off = parent.j_off;
            l.M = parent.pi + 1;
            l.N = parent.pj + 1;
            l.pair = parent.pair;
            l.depth = parent.depth + 1;
            l.fsrc = parent.fpass;  // same first cell: the parent's forward pass restricted
            r.i_off = parent.i_off + parent.pi;
            r.j_off = parent.j_off + parent.pj;
            r.M = parent.M - parent.pi;
            r.N = parent.N - parent.pj;
            r.pair = parent.pair;
            r.depth = parent.depth + 1;
            r.bsrc = parent.bpass;  // same last cell: the parent's reverse pass restricted
            nodes.push_back(l);
            nodes[id].left = (int)nodes.size() - 1;
            classify(nodes[id].left);
            nodes.push_back(r);
            nodes[id].right = (int)nodes.size() - 1;
            classify(nodes[id].right);
        }
    }
    // on error: drain what is in flight before the buffers are reused
    for (auto& f : flights) cudaEventSynchronize(f.S->done);
    if (staged) cudaEventDestroy(staged);
    if (rc != LMDTW_OK) return rc;
    if (leafs.empty()) c->prof_collect();  // else leaves() collects after its sync (off the critical path)
    // leaves, in node order (the stitching below walks the tree)
    std::vector<int64_t> poff;
    std::vector<int> plen;
    phase("recursion done");
    TRY(E.leaves(nodes, leafs, xb, yb, nullptr, poff, plen));
    phase("leaves done");

    const int* hpath = c->hpath();
    results.assign(npairs, nullptr);
    struct PhaseEnd {
        std::function<void()> f;
        ~PhaseEnd() { f(); }
    } phase_end{[&] { phase("results built"); }};
    // One result per pair; pairs are independent (the inputs are read-only,
    // inst[p] and results[p] belong to pair p), so a batch builds them on
    // host threads: the sequential cost sum over each path is a dependent add
    // chain, ~12 ms over cfg4's 256 paths on one thread.
    auto build_one = [&](int p) {
        std::unique_ptr<lmdtw_result> res(new lmdtw_result());
        Inst& in = inst[p];
        // pre-order DFS: pivots and leaf sequence
        std::vector<int> stack{p};  // root node index == p
        std::vector<int> leaf_seq;
        while (!stack.empty()) {
            const int id = stack.back();
            stack.pop_back();
            const Node& n = nodes[id];
            if (n.leaf >= 0) {
                leaf_seq.push_back(n.leaf);
                const int64_t cl = n.M * n.N;
                in.add_batch(cl);
                in.peak_table = std::max(in.peak_table, cl);
                continue;
            }
            lmdtw_pivot_t pv;
            pv.i = n.i_off + n.pi;
            pv.j = n.j_off + n.pj;
            pv.i_off = n.i_off;
            pv.j_off = n.j_off;
            pv.M = n.M;
            pv.N = n.N;
            pv.sub_i = n.pi;
            pv.sub_j = n.pj;
            pv.diagonal_k = n.k;
            pv.total_at_pivot = n.total;
            res->pivots.push_back(pv);
            stack.push_back(n.right);
            stack.push_back(n.left);
        }
        // path: leaf paths in order, first cell of every later leaf dropped;
        // cost: the sequential sum over the path in that order (core.py:191-197)
        // -- one pass, so the add chain's latency hides the path writes
        int64_t K = 0;
        for (size_t s = 0; s < leaf_seq.size(); s++) K += plen[leaf_seq[s]] - (s ? 1 : 0);
        res->path.reset(new int64_t[std::max<int64_t>(2 * K, 1)]);
        auto build = [&](auto zero, const auto* pc) {
            auto total = zero;
            int64_t* out = res->path.get();
            for (size_t s = 0; s < leaf_seq.size(); s++) {
                const int lf = leaf_seq[s];
                const Node& n = nodes[leafs[lf]];
                const int* lp = hpath + 2 * poff[lf];  // reversed: lp[0] is the corner
                const auto* cl = pc + poff[lf];
                const int64_t io = n.i_off, jo = n.j_off;
                for (int q = plen[lf] - 1 - (s ? 1 : 0); q >= 0; q--) {
                    out[0] = io + lp[2 * q];
                    out[1] = jo + lp[2 * q + 1];
                    out += 2;
                    total = total + cl[q];
                }
            }
            return (double)total;
        };
        res->info.cost = cfg.precision == 32 ? build(0.0f, c->hpcost<float>()) : build(0.0, c->hpcost<double>());
        if (in.cb) in.cb(in.cells, in.budget, in.user);
        res->info.path_len = K;
        res->info.cells_processed = in.cells;
        res->info.cells_budget = in.budget;
        res->info.peak_diag_values = in.peak_diag;
        res->info.peak_table_cells = in.peak_table;
        res->info.n_pivots = (int64_t)res->pivots.size();
        res->info.n_levels = nlevels;
        res->info.gpu_launches = c->call_launches;
        res->info.h2d_bytes = c->h2d;
        res->info.d2h_bytes = c->d2h;
        results[p] = res.release();
    };
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    const int nth = npairs >= 8 ? (int)std::min<unsigned>(std::min<unsigned>((unsigned)npairs / 4, 16u), hw) : 1;
    if (nth <= 1) {
        for (int p = 0; p < npairs; p++) build_one(p);
        return LMDTW_OK;
    }
    std::atomic<int> next{0};
    std::atomic<bool> failed{false};
    {
        std::vector<std::thread> pool;
        pool.reserve(nth);
        for (int t = 0; t < nth; t++)
            pool.emplace_back([&] {
                try {
                    for (int p; !failed.load() && (p = next.fetch_add(1)) < npairs;) build_one(p);
                } catch (...) {
                    failed.store(true);
                }
            });
        for (auto& t : pool) t.join();
    }
    if (failed.load()) {
        for (auto*& r : results) {
            delete r;
            r = nullptr;
        }
        return set_err(LMDTW_ENOMEM, "host allocation failed while building the results");
    }
    return LMDTW_OK;
}

}  // namespace

// Host split-point combine of divide.find_pivot (divide.py:122-145) for two
// half passes computed on different devices.
namespace {
template <typename T>
void combine_pivot(int64_t M, int64_t N, int highest, const void* const fd[3], const void* const fc[3],
                   const void* const bd[3], int64_t* ijk, double* total) {
    const int64_t K = M + N - 1;
    const int64_t kf = (K + 1) / 2;
    T best = T(0);
    int64_t bk = -1, bidx = -1;
    bool have = false;
    for (int m = 0; m < 3; m++) {
        const int64_t k = kf - 2 + m;
        const int64_t L = dlen(k, M, N);
        const T* df = static_cast<const T*>(fd[m]);
        const T* cf = static_cast<const T*>(fc[m]);
        const T* db = static_cast<const T*>(bd[2 - m]);
        for (int64_t idx = 0; idx < L; idx++) {
            const int64_t i = std::min(k, M - 1) - idx;
            const int64_t ib = std::min(M + N - 2 - k, M - 1) - (M - 1 - i);
            T t = df[idx] + db[ib];  // two roundings in the reference's order
            t = t - cf[idx];
            // lexicographic (t, k, idx) minimum, or (t, -k, -idx) for "highest"
            bool take;
            if (!have) take = true;
            else if (t < best) take = true;
            else if (t == best) take = highest ? (k > bk || (k == bk && idx > bidx)) : false;
            else take = false;
            if (take) {
                best = t;
                bk = k;
                bidx = idx;
                have = true;
            }
        }
    }
    const int64_t i = std::min(bk, M - 1) - bidx;
    ijk[0] = i;
    ijk[1] = bk - i;
    ijk[2] = bk;
    *total = (double)best;
}
}  // namespace

// ====================================================================== C ABI
extern "C" {

const char* lmdtw_version(void) { return "lmdtw_b200 0.1.0 (sm_100a)"; }
const char* lmdtw_last_error(void) { return g_err.c_str(); }

int lmdtw_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

int lmdtw_max_dim(int32_t precision) {
    (void)precision;
    return kMaxDim;
}

int64_t lmdtw_diag_length(int64_t k, int64_t M, int64_t N) { return dlen(k, M, N); }
int64_t lmdtw_cells_upto(int64_t kstop, int64_t M, int64_t N) { return cells_upto(kstop, M, N); }
int64_t lmdtw_peak_retained_values(int64_t kstop, int64_t M, int64_t N) { return peak_values(kstop, M, N); }
int64_t lmdtw_launch_count(void) { return g_launches.load(); }

void lmdtw_profile_enable(int on) { g_profile.store(on ? 1 : 0); }
void lmdtw_profile_reset(void) {
    std::lock_guard<std::mutex> g(g_stats.mu);
    g_stats.wave_ms = g_stats.leaf_ms = g_stats.pivot_ms = 0;
    g_stats.wave_launches = g_stats.wave_cells = g_stats.leaf_cells = 0;
}
// out[0]=wave_ms out[1]=wave_launches out[2]=wave_cells out[3]=leaf_ms out[4]=leaf_cells
void lmdtw_profile_get(double* out) {
    std::lock_guard<std::mutex> g(g_stats.mu);
    out[0] = g_stats.wave_ms;
    out[1] = (double)g_stats.wave_launches;
    out[2] = (double)g_stats.wave_cells;
    out[3] = g_stats.leaf_ms;
    out[4] = (double)g_stats.leaf_cells;
}
// Probe builds (LMDTW_WAITSTATS): blocked-wait cycles by tag (16 + 16 values).
int lmdtw_debug_wait_stats(unsigned long long* cycles, unsigned long long* count, int reset) {
    CU(wait_stats(cycles, count, reset));
    return LMDTW_OK;
}
// The stream of `device`'s primary context: every kernel of a call runs on
// it unless another call on the same device is in flight (for event timing).
void* lmdtw_stream(int device) {
    cudaStream_t st = nullptr;
    if (primary_stream(device, &st) != LMDTW_OK) return nullptr;
    return (void*)st;
}

// Benchmark hook (not part of the reference-facing ABI): `npasses`
// independent full-grid passes of one strip each (H x N), random features,
// `reps` launches; *ms = mean kernel time.  Measures the strip engine's
// per-warp step rate without strip-to-strip dependencies.
int lmdtw_debug_wave_independent(int device, int32_t precision, int32_t d, int32_t npasses, int32_t N,
                                 int32_t reps, double* ms) {
    CtxLease c;
    TRY(lease_ctx(device, c));
    CU(cudaSetDevice(device));
    Engine E(*c, precision, d);
    const int64_t M = E.H;
    std::vector<float> hx((size_t)M * d), hy((size_t)N * d);
    unsigned s = 12345u;
    for (auto& v : hx) { s = s * 1664525u + 1013904223u; v = (s >> 8) * (1.0f / 16777216.0f); }
    for (auto& v : hy) { s = s * 1664525u + 1013904223u; v = (s >> 8) * (1.0f / 16777216.0f); }
    const float* xp = hx.data();
    const float* yp = hy.data();
    int64_t Mv = M, Nv = N;
    std::vector<int64_t> xb, yb;
    TRY(E.stage(&xp, &Mv, 1, LMDTW_MEM_HOST, true, xb));
    TRY(E.stage(&yp, &Nv, 1, LMDTW_MEM_HOST, false, yb));
    int64_t out_total = 0, bnd_total = 0;
    std::vector<PassDesc> P;
    for (int q = 0; q < npasses; q++)
        P.push_back(E.half_pass_desc(xb[0], yb[0], M, N, M + N - 2, 0, out_total, bnd_total));
    CU(c->main.out.ensure((size_t)out_total * E.esz));
    double tot = 0;
    for (int r = 0; r < reps + 1; r++) {
        TRY(E.run_wave(c->main, P, bnd_total, false, nullptr, nullptr, 0));
        CU(cudaEventRecord(c->ev1, c->st));
        CU(cudaEventSynchronize(c->ev1));
        if (r == 0) continue;  // warm-up
    }
    // time the last `reps` launches as one block
    CU(cudaEventRecord(c->ev0, c->st));
    for (int r = 0; r < reps; r++) TRY(E.run_wave(c->main, P, bnd_total, false, nullptr, nullptr, 0));
    CU(cudaEventRecord(c->ev1, c->st));
    CU(cudaEventSynchronize(c->ev1));
    float f = 0;
    CU(cudaEventElapsedTime(&f, c->ev0, c->ev1));
    tot = f;
    *ms = tot / reps;
    return LMDTW_OK;
}

int64_t lmdtw_handoff_words(int64_t N, int32_t precision) { return 2 * ((N + 1) & ~1LL) * (precision == 32 ? 1 : 2); }

int32_t lmdtw_strip_height(int32_t precision, int32_t d) {
    const DimPlan dp = plan_dims(precision, d);
    return dp.dp < 0 ? -1 : strip_height(precision, dp);
}

int lmdtw_half_pass_shard(int device, const float* X, int64_t M, const float* Y, int64_t N, int32_t d, int64_t kstop,
                          int32_t reverse, int32_t precision, int32_t mem, int32_t strip_lo, int32_t strip_hi,
                          void* bnd_local, const void* bnd_prev, void* out_d[3], void* out_c[3], int64_t* cells) {
    TRY(validate_common(M, N, d, precision));
    if (kstop < 2 || kstop > M + N - 2) return set_err(LMDTW_EINVAL, "kstop out of range [2, M+N-2]");
    if (!bnd_local) return set_err(LMDTW_EINVAL, "bnd_local is required");
    CtxLease c;
    TRY(lease_ctx(device, c));
    CU(cudaSetDevice(device));
    c->call_launches = 0;
    Engine E(*c, precision, d);
    std::vector<int64_t> xb, yb;
    TRY(E.stage(&X, &M, 1, mem, true, xb));
    TRY(E.stage(&Y, &N, 1, mem, false, yb));
    int64_t out_total = 0, bnd_total = 0;
    PassDesc pd = E.half_pass_desc(xb[0], yb[0], M, N, kstop, reverse ? 1 : 0, out_total, bnd_total);
    if (strip_lo < 0 || strip_hi > pd.nstrips || strip_lo >= strip_hi)
        return set_err(LMDTW_EINVAL, "strip range outside the pass");
    if (strip_lo > 0 && !bnd_prev) return set_err(LMDTW_EINVAL, "bnd_prev is required after the first shard");
    const int H = E.H;
    pd.strip_lo = strip_lo;
    pd.strip_hi = strip_hi;
    pd.tile_w = kTileW;
    pd.lb_off = 0;
    pd.flag_off = 0;
    pd.bnd_off = 0;
    pd.bnd_in_first = strip_lo > 0 ? (uint64_t)(uintptr_t)bnd_prev : 0;
    pd.sys_out = strip_hi < pd.nstrips ? 1 : 0;  // the next shard may run on a peer GPU
    CU(c->main.out.ensure((size_t)out_total * E.esz));
    CU(c->main.passes.ensure(sizeof(PassDesc)));
    CU(c->main.counter.ensure(2 * sizeof(int)));
    CU(c->main.lb.ensure((size_t)pd.nstrips * (H + 1) * E.esz));
    CU(c->main.flags.ensure((size_t)pd.nstrips * sizeof(int)));
    CU(c->main.h_passes.ensure(sizeof(PassDesc)));
    memcpy(c->main.h_passes.p, &pd, sizeof(PassDesc));
    CU(cudaMemcpyAsync(c->main.passes.p, c->main.h_passes.p, sizeof(PassDesc), cudaMemcpyHostToDevice, c->st));
    int64_t nitems = 0;
    TRY(E.upload_queue(c->main, std::vector<PassDesc>{pd}, nitems));
    CU(cudaMemsetAsync(c->main.counter.p, 0, 2 * sizeof(int), c->st));
    CU(cudaMemsetAsync(c->main.flags.p, 0, (size_t)pd.nstrips * sizeof(int), c->st));
    WaveLaunch w{};
    w.X = c->xp.p;
    w.Y = c->yp.p;
    w.dp = E.dp;
    w.wide = E.dpl.wide;
    w.precision = precision;
    w.passes = c->main.passes.as<PassDesc>();
    w.items = c->main.items.as<WorkItem>();
    w.nitems = (int)nitems;
    w.counter = c->main.counter.as<int>();
    w.out = c->main.out.p;
    w.bnd = bnd_local;
    w.lb = c->main.lb.p;
    w.flags = c->main.flags.as<int>();
    w.tie0 = 2;
    w.tie1 = 0;
    w.tie2 = 1;
    TRY(E.launched(launch_wave(w, c->st), "wave_kernel (shard)"));
    // the shard's rows of the last three diagonals: idx = min(k, M-1) - i
    for (int s3 = 0; s3 < 3; s3++) {
        const int64_t k = kstop - 2 + s3, L = dlen(k, M, N);
        if (L <= 0) continue;
        const int64_t top = std::min<int64_t>(k, M - 1), ilo = std::max<int64_t>(0, k - (N - 1));
        const int64_t r0 = std::max<int64_t>((int64_t)strip_lo * H, ilo);
        const int64_t r1 = std::min<int64_t>((int64_t)strip_hi * H - 1, top);
        if (r1 < r0) continue;
        const int64_t i0 = top - r1, cnt = r1 - r0 + 1;
        if (out_d && out_d[s3])
            CU(cudaMemcpyAsync((char*)out_d[s3] + i0 * E.esz, (char*)c->main.out.p + (pd.out_off[s3] + i0) * E.esz,
                               cnt * E.esz, cudaMemcpyDefault, c->st));
        if (out_c && out_c[s3])
            CU(cudaMemcpyAsync((char*)out_c[s3] + i0 * E.esz, (char*)c->main.out.p + (pd.out_off[3 + s3] + i0) * E.esz,
                               cnt * E.esz, cudaMemcpyDefault, c->st));
    }
    CU(cudaStreamSynchronize(c->st));
    c->prof_collect();
    if (cells) {
        const int64_t ra = (int64_t)strip_lo * H, rb = std::min<int64_t>(pd.rows, (int64_t)strip_hi * H);
        *cells = cells_upto(kstop, rb, N) - cells_upto(kstop, ra, N);
    }
    return LMDTW_OK;
}

// Handoff buffers shared between the ranks of a sharded pass (CUDA IPC).
int lmdtw_ipc_alloc(int device, int64_t bytes, void** ptr, unsigned char handle[64]) {
    if (!ptr || !handle || bytes <= 0) return set_err(LMDTW_EINVAL, "bad ipc allocation request");
    CU(cudaSetDevice(device));
    CU(cudaMalloc(ptr, (size_t)bytes));
    cudaIpcMemHandle_t h;
    CU(cudaIpcGetMemHandle(&h, *ptr));
    memcpy(handle, &h, 64);
    return LMDTW_OK;
}
int lmdtw_ipc_open(int device, const unsigned char handle[64], void** ptr) {
    if (!ptr || !handle) return set_err(LMDTW_EINVAL, "bad ipc handle");
    CU(cudaSetDevice(device));
    cudaIpcMemHandle_t h;
    memcpy(&h, handle, 64);
    CU(cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess));
    return LMDTW_OK;
}
int lmdtw_ipc_close(int device, void* ptr) {
    CU(cudaSetDevice(device));
    CU(cudaIpcCloseMemHandle(ptr));
    return LMDTW_OK;
}
int lmdtw_ipc_free(int device, void* ptr) {
    CU(cudaSetDevice(device));
    CU(cudaFree(ptr));
    return LMDTW_OK;
}
// All bytes 0xFF (handoff tag -1), synchronously.
int lmdtw_fill_ones(int device, void* ptr, int64_t bytes) {
    CU(cudaSetDevice(device));
    CU(cudaMemset(ptr, 0xFF, (size_t)bytes));
    CU(cudaDeviceSynchronize());
    return LMDTW_OK;
}

// Test hook for strip sharding (not part of the reference-facing ABI): one
// half pass split into `nshards` contiguous strip ranges, each run by its own
// persistent wave kernel on its own stream and buffers, concurrently on one
// GPU; shard s reads the boundary row of shard s-1's last strip from shard
// s-1's handoff buffer (what a peer GPU's buffer is in the multi-GPU layout).
// The outputs are merged by row range into the host buffers of diag_dtw.
int lmdtw_debug_sharded_half_pass(int device, const float* X, int64_t M, const float* Y, int64_t N, int32_t d,
                                  int64_t kstop, int32_t reverse, int32_t precision, int32_t nshards, void* out_d[3],
                                  void* out_c[3]) {
    TRY(validate_common(M, N, d, precision));
    if (kstop < 2 || kstop > M + N - 2) return set_err(LMDTW_EINVAL, "kstop out of range [2, M+N-2]");
    if (nshards < 1) return set_err(LMDTW_EINVAL, "nshards must be >= 1");
    CtxLease c;
    TRY(lease_ctx(device, c));
    CU(cudaSetDevice(device));
    Engine E(*c, precision, d);
    std::vector<int64_t> xb, yb;
    TRY(E.stage(&X, &M, 1, LMDTW_MEM_HOST, true, xb));
    TRY(E.stage(&Y, &N, 1, LMDTW_MEM_HOST, false, yb));
    CU(cudaStreamSynchronize(c->st));
    c->prof_collect();
    int64_t out_total = 0, bnd_total = 0;
    const PassDesc base = E.half_pass_desc(xb[0], yb[0], M, N, kstop, reverse ? 1 : 0, out_total, bnd_total);
    const int S = base.nstrips, H = E.H;
    const int ns = std::min<int>(nshards, S);
    // contiguous strip ranges of about equal cell counts
    std::vector<int64_t> scells(S);
    int64_t all = 0;
    for (int a = 0; a < S; a++) {
        const int64_t r0 = (int64_t)a * H, r1 = std::min<int64_t>(base.rows, r0 + H);
        scells[a] = cells_upto(kstop, r1, N) - cells_upto(kstop, r0, N);
        all += scells[a];
    }
    std::vector<int> lo(ns + 1, S);
    lo[0] = 0;
    int64_t acc = 0;
    for (int a = 0, sh = 1; a < S && sh < ns; a++) {
        acc += scells[a];
        if (acc * ns >= all * sh && S - (a + 1) >= ns - sh) lo[sh++] = a + 1;
    }
    struct Shard {
        PassDesc pd;
        std::vector<WorkItem> items;
        DBuf passes, items_d, counter, bnd, lb, flags, out;
        cudaStream_t st = nullptr;
    };
    std::vector<Shard> sh(ns);
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device);
    int rc = LMDTW_OK;
    for (int q = 0; q < ns && rc == LMDTW_OK; q++) {
        Shard& z = sh[q];
        z.pd = base;
        z.pd.strip_lo = lo[q];
        z.pd.strip_hi = lo[q + 1];
        z.pd.tile_w = kTileW;
        z.pd.lb_off = 0;
        z.pd.flag_off = 0;
        E.make_items(c->main, std::vector<PassDesc>{z.pd}, z.items);
        if (z.bnd.ensure((size_t)bnd_total * 8) != cudaSuccess || z.out.ensure((size_t)out_total * E.esz) ||
            z.passes.ensure(sizeof(PassDesc)) || z.items_d.ensure(z.items.size() * sizeof(WorkItem)) ||
            z.counter.ensure(2 * sizeof(int)) || z.lb.ensure((size_t)S * (H + 1) * E.esz) ||
            z.flags.ensure((size_t)S * sizeof(int)) || cudaStreamCreateWithFlags(&z.st, cudaStreamNonBlocking))
            rc = set_err(LMDTW_ENOMEM, "sharded half pass: allocation failed");
    }
    if (rc == LMDTW_OK) {
        for (int q = 0; q < ns; q++) {
            Shard& z = sh[q];
            z.pd.bnd_in_first = q > 0 ? (uint64_t)(uintptr_t)sh[q - 1].bnd.p : 0;
            z.pd.sys_out = q + 1 < ns ? 1 : 0;
            cudaMemcpy(z.passes.p, &z.pd, sizeof(PassDesc), cudaMemcpyHostToDevice);
            cudaMemcpy(z.items_d.p, z.items.data(), z.items.size() * sizeof(WorkItem), cudaMemcpyHostToDevice);
            cudaMemset(z.counter.p, 0, 2 * sizeof(int));
            cudaMemset(z.bnd.p, 0xFF, (size_t)bnd_total * 8);  // tag -1
            cudaMemset(z.flags.p, 0, (size_t)S * sizeof(int));
        }
        CU(cudaDeviceSynchronize());  // every buffer initialised before any shard runs
        for (int q = 0; q < ns; q++) {
            Shard& z = sh[q];
            WaveLaunch w{};
            w.X = c->xp.p;
            w.Y = c->yp.p;
            w.dp = E.dp;
            w.wide = E.dpl.wide;
    w.wide = E.dpl.wide;
            w.precision = precision;
            w.passes = z.passes.as<PassDesc>();
            w.items = z.items_d.as<WorkItem>();
            w.nitems = (int)z.items.size();
            w.counter = z.counter.as<int>();
            w.out = z.out.p;
            w.bnd = z.bnd.p;
            w.lb = z.lb.p;
            w.flags = z.flags.as<int>();
            w.tie0 = 2;
            w.tie1 = 0;
            w.tie2 = 1;
            w.grid_warps = std::max(1, nsm / ns);  // CTAs: the shards share the SMs
            CU(launch_wave(w, z.st));
        }
        CU(cudaDeviceSynchronize());
        // merge the last three diagonals by row range: idx = min(k, M-1) - i
        for (int s3 = 0; s3 < 3; s3++) {
            const int64_t k = kstop - 2 + s3, L = dlen(k, M, N);
            if (L <= 0) continue;
            const int64_t top = std::min<int64_t>(k, M - 1), ilo = std::max<int64_t>(0, k - (N - 1));
            for (int q = 0; q < ns; q++) {
                const int64_t r0 = std::max<int64_t>((int64_t)lo[q] * H, ilo);
                const int64_t r1 = std::min<int64_t>((int64_t)lo[q + 1] * H - 1, top);
                if (r1 < r0) continue;
                const int64_t i0 = top - r1, cnt = r1 - r0 + 1;
                if (out_d && out_d[s3])
                    CU(cudaMemcpy((char*)out_d[s3] + i0 * E.esz, (char*)sh[q].out.p + (base.out_off[s3] + i0) * E.esz,
                                  cnt * E.esz, cudaMemcpyDeviceToHost));
                if (out_c && out_c[s3])
                    CU(cudaMemcpy((char*)out_c[s3] + i0 * E.esz,
                                  (char*)sh[q].out.p + (base.out_off[3 + s3] + i0) * E.esz, cnt * E.esz,
                                  cudaMemcpyDeviceToHost));
            }
        }
    }
    for (auto& z : sh) {
        if (z.st) cudaStreamDestroy(z.st);
        for (DBuf* b : {&z.passes, &z.items_d, &z.counter, &z.bnd, &z.lb, &z.flags, &z.out})
            if (b->p) cudaFree(b->p);
    }
    return rc;
}

int lmdtw_half_pass(int device, const float* X, int64_t M, const float* Y, int64_t N, int32_t d, int64_t kstop,
                    int32_t reverse, int32_t precision, int32_t mem, void* out_d[3], void* out_c[3],
                    int64_t* cells) {
    TRY(validate_common(M, N, d, precision));
    if (kstop < 2 || kstop > M + N - 2) return set_err(LMDTW_EINVAL, "kstop out of range [2, M+N-2]");
    CtxLease c;
    TRY(lease_ctx(device, c));
    CU(cudaSetDevice(device));
    c->call_launches = 0;
    Engine E(*c, precision, d);
    std::vector<int64_t> xb, yb;
    TRY(E.stage(&X, &M, 1, mem, true, xb));
    TRY(E.stage(&Y, &N, 1, mem, false, yb));
    int64_t out_total = 0, bnd_total = 0;
    std::vector<PassDesc> P{E.half_pass_desc(xb[0], yb[0], M, N, kstop, reverse ? 1 : 0, out_total, bnd_total)};
    CU(c->main.out.ensure((size_t)out_total * E.esz));
    const int64_t cl = cells_upto(kstop, M, N);
    TRY(E.run_wave(c->main, P, bnd_total, false, nullptr, nullptr, cl));
    for (int s = 0; s < 3; s++) {
        const int64_t L = dlen(kstop - 2 + s, M, N);
        if (L > 0 && out_d && out_d[s])
            CU(cudaMemcpyAsync(out_d[s], (char*)c->main.out.p + P[0].out_off[s] * E.esz, L * E.esz,
                               cudaMemcpyDefault, c->st));
        if (L > 0 && out_c && out_c[s])
            CU(cudaMemcpyAsync(out_c[s], (char*)c->main.out.p + P[0].out_off[3 + s] * E.esz, L * E.esz,
                               cudaMemcpyDefault, c->st));
    }
    CU(cudaStreamSynchronize(c->st));
    c->prof_collect();
    if (cells) *cells = cl;
    return LMDTW_OK;
}

int lmdtw_find_pivot(int device, const float* X, int64_t M, const float* Y, int64_t N, int32_t d,
                     int32_t precision, int32_t pivot_highest, int32_t mem, int64_t* i, int64_t* j,
                     int64_t* diagonal_k, double* total, int64_t* cells, int64_t* peak) {
    TRY(validate_common(M, N, d, precision));
    if (M + N - 2 < 2) return set_err(LMDTW_EINVAL, "too small for a pivot search; use dtw_full");
    CtxLease c;
    TRY(lease_ctx(device, c));
    CU(cudaSetDevice(device));
    c->call_launches = 0;
    Engine E(*c, precision, d);
    std::vector<int64_t> xb, yb;
    TRY(E.stage(&X, &M, 1, mem, true, xb));
    TRY(E.stage(&Y, &N, 1, mem, false, yb));
    std::vector<Node> nodes(1);
    nodes[0].i_off = 0;
    nodes[0].j_off = 0;
    nodes[0].M = M;
    nodes[0].N = N;
    nodes[0].pair = 0;
    std::vector<int64_t> cl, pk;
    TRY(E.pivot_level(c->main, nodes, std::vector<int>{0}, xb, yb, &cl, &pk, pivot_highest ? 1 : 0));
    if (i) *i = nodes[0].pi;
    if (j) *j = nodes[0].pj;
    if (diagonal_k) *diagonal_k = nodes[0].k;
    if (total) *total = nodes[0].total;
    if (cells) *cells = cl[0];
    if (peak) *peak = pk[0];
    return LMDTW_OK;
}

int lmdtw_dtw_full(int device, const float* X, int64_t M, const float* Y, int64_t N, int32_t d,
                   const int32_t tie[3], int32_t precision, int32_t mem, double* cost, int64_t* path_out,
                   int64_t* path_len, void* D_out) {
    TRY(validate_common(M, N, d, precision));
    TRY(validate_tie(tie));
    CtxLease c;
    TRY(lease_ctx(device, c));
    CU(cudaSetDevice(device));
    c->call_launches = 0;
    Engine E(*c, precision, d);
    E.tie[0] = tie[0];
    E.tie[1] = tie[1];
    E.tie[2] = tie[2];
    std::vector<int64_t> xb, yb;
    TRY(E.stage(&X, &M, 1, mem, true, xb));
    TRY(E.stage(&Y, &N, 1, mem, false, yb));
    std::vector<Node> nodes(1);
    nodes[0].i_off = 0;
    nodes[0].j_off = 0;
    nodes[0].M = M;
    nodes[0].N = N;
    nodes[0].pair = 0;
    std::vector<int64_t> poff;
    std::vector<int> plen;
    TRY(E.leaves(nodes, std::vector<int>{0}, xb, yb, D_out, poff, plen));
    const int* lp = c->hpath();
    const int len = plen[0];
    for (int q = 0; q < len; q++) {
        path_out[2 * q] = lp[2 * (len - 1 - q)];
        path_out[2 * q + 1] = lp[2 * (len - 1 - q) + 1];
    }
    if (path_len) *path_len = len;
    if (cost) *cost = E.leaf_cost(0);
    return LMDTW_OK;
}

int lmdtw_align(int device, const float* X, int64_t M, const float* Y, int64_t N, int32_t d,
                const lmdtw_config_t* cfg, int32_t mem, lmdtw_progress_fn progress, void* user,
                lmdtw_result_t** result) {
    if (!cfg || !result) return set_err(LMDTW_EINVAL, "null config/result");
    std::vector<lmdtw_result*> res;
    TRY(align_core(device, 1, &X, &M, &Y, &N, d, *cfg, mem, progress, user, res));
    *result = res[0];
    return LMDTW_OK;
}

int lmdtw_align_batch(int device, int32_t npairs, const float* const* X, const int64_t* M, const float* const* Y,
                      const int64_t* N, int32_t d, const lmdtw_config_t* cfg, int32_t mem,
                      lmdtw_result_t** results) {
    if (!cfg || !results) return set_err(LMDTW_EINVAL, "null config/results");
    std::vector<lmdtw_result*> res;
    TRY(align_core(device, npairs, X, M, Y, N, d, *cfg, mem, nullptr, nullptr, res));
    for (int p = 0; p < npairs; p++) results[p] = res[p];
    return LMDTW_OK;
}

int lmdtw_pivot_nodes(int device, const float* X, int64_t M, const float* Y, int64_t N, int32_t d, int32_t n,
                      const int64_t* sub, int32_t precision, int32_t pivot_highest, int32_t mem, int64_t* out,
                      double* totals) {
    TRY(validate_common(M, N, d, precision));
    if (n < 0 || (n > 0 && (!sub || !out || !totals))) return set_err(LMDTW_EINVAL, "bad node list");
    for (int q = 0; q < n; q++) {
        const int64_t* s = sub + 4 * q;
        if (s[0] < 0 || s[1] < 0 || s[2] < 1 || s[3] < 1 || s[0] + s[2] > M || s[1] + s[3] > N)
            return set_err(LMDTW_EINVAL, "sub-block outside the series");
        if (s[2] + s[3] - 2 < 2) return set_err(LMDTW_EINVAL, "sub-block too small for a pivot search");
    }
    if (n == 0) return LMDTW_OK;
    CtxLease c;
    TRY(lease_ctx(device, c));
    CU(cudaSetDevice(device));
    c->call_launches = 0;
    Engine E(*c, precision, d);
    std::vector<int64_t> xb, yb;
    TRY(E.stage(&X, &M, 1, mem, true, xb));
    TRY(E.stage(&Y, &N, 1, mem, false, yb));
    std::vector<Node> nodes(n);
    std::vector<int> ids(n);
    for (int q = 0; q < n; q++) {
        nodes[q].i_off = sub[4 * q];
        nodes[q].j_off = sub[4 * q + 1];
        nodes[q].M = sub[4 * q + 2];
        nodes[q].N = sub[4 * q + 3];
        nodes[q].pair = 0;
        ids[q] = q;
    }
    std::vector<int64_t> cl, pk;
    TRY(E.pivot_level(c->main, nodes, ids, xb, yb, &cl, &pk, pivot_highest ? 1 : 0));
    for (int q = 0; q < n; q++) {
        out[5 * q] = nodes[q].pi;
        out[5 * q + 1] = nodes[q].pj;
        out[5 * q + 2] = nodes[q].k;
        out[5 * q + 3] = cl[q];
        out[5 * q + 4] = pk[q];
        totals[q] = nodes[q].total;
    }
    return LMDTW_OK;
}

int lmdtw_leaf_nodes(int device, const float* X, int64_t M, const float* Y, int64_t N, int32_t d, int32_t n,
                     const int64_t* sub, const int32_t tie[3], int32_t precision, int32_t mem, int64_t* path_out,
                     int64_t* path_len) {
    TRY(validate_common(M, N, d, precision));
    TRY(validate_tie(tie));
    if (n < 0 || (n > 0 && (!sub || !path_out || !path_len))) return set_err(LMDTW_EINVAL, "bad node list");
    for (int q = 0; q < n; q++) {
        const int64_t* s = sub + 4 * q;
        if (s[0] < 0 || s[1] < 0 || s[2] < 1 || s[3] < 1 || s[0] + s[2] > M || s[1] + s[3] > N)
            return set_err(LMDTW_EINVAL, "sub-block outside the series");
    }
    if (n == 0) return LMDTW_OK;
    CtxLease c;
    TRY(lease_ctx(device, c));
    CU(cudaSetDevice(device));
    c->call_launches = 0;
    Engine E(*c, precision, d);
    E.tie[0] = tie[0];
    E.tie[1] = tie[1];
    E.tie[2] = tie[2];
    std::vector<int64_t> xb, yb;
    TRY(E.stage(&X, &M, 1, mem, true, xb));
    TRY(E.stage(&Y, &N, 1, mem, false, yb));
    std::vector<Node> nodes(n);
    std::vector<int> ids(n);
    for (int q = 0; q < n; q++) {
        nodes[q].i_off = sub[4 * q];
        nodes[q].j_off = sub[4 * q + 1];
        nodes[q].M = sub[4 * q + 2];
        nodes[q].N = sub[4 * q + 3];
        nodes[q].pair = 0;
        ids[q] = q;
    }
    std::vector<int64_t> poff;
    std::vector<int> plen;
    TRY(E.leaves(nodes, ids, xb, yb, nullptr, poff, plen));
    const int* hp = c->hpath();
    int64_t w = 0;
    for (int q = 0; q < n; q++) {
        const int len = plen[q];
        const int* lp = hp + 2 * poff[q];  // reversed: lp[0] is the corner
        for (int t = 0; t < len; t++) {
            path_out[2 * (w + t)] = lp[2 * (len - 1 - t)];
            path_out[2 * (w + t) + 1] = lp[2 * (len - 1 - t) + 1];
        }
        path_len[q] = len;
        w += len;
    }
    return LMDTW_OK;
}


int lmdtw_pivot_combine(int32_t precision, int64_t M, int64_t N, int32_t pivot_highest, const void* const fwd_d[3],
                        const void* const fwd_c[3], const void* const bwd_d[3], int64_t* ijk, double* total) {
    if (precision != 32 && precision != 64) return set_err(LMDTW_EINVAL, "precision must be 32 or 64");
    if (M < 1 || N < 1 || M + N - 2 < 2) return set_err(LMDTW_EINVAL, "too small for a pivot search");
    if (!fwd_d || !fwd_c || !bwd_d || !ijk || !total) return set_err(LMDTW_EINVAL, "null buffer");
    if (precision == 32)
        combine_pivot<float>(M, N, pivot_highest, fwd_d, fwd_c, bwd_d, ijk, total);
    else
        combine_pivot<double>(M, N, pivot_highest, fwd_d, fwd_c, bwd_d, ijk, total);
    return LMDTW_OK;
}

// divide.find_pivot's combine (divide.py:122-145) on the device: the three
// forward D and C diagonals and the three reverse D diagonals (device or host
// pointers; host pointers are staged) are gathered into one device buffer and
// reduced by pivot_kernel -- the multi-GPU path's combine after an NCCL
// all-gather of the diagonals, bit-identical to lmdtw_pivot_combine.
int lmdtw_pivot_combine_device(int device, int32_t precision, int64_t M, int64_t N, int32_t pivot_highest,
                               const void* const fwd_d[3], const void* const fwd_c[3], const void* const bwd_d[3],
                               int64_t* ijk, double* total) {
    if (precision != 32 && precision != 64) return set_err(LMDTW_EINVAL, "precision must be 32 or 64");
    if (M < 1 || N < 1 || M + N - 2 < 2) return set_err(LMDTW_EINVAL, "too small for a pivot search");
    if (!fwd_d || !fwd_c || !bwd_d || !ijk || !total) return set_err(LMDTW_EINVAL, "null buffer");
    CtxLease c;
    TRY(lease_ctx(device, c));
    const size_t esz = precision == 32 ? 4 : 8;
    const int64_t K = M + N - 1, kf = (K + 1) / 2, kb = (K % 2 == 0) ? kf + 1 : kf;
    PassDesc P[2] = {};
    int64_t off = 0;
    for (int s = 0; s < 3; s++) {  // fwd D, fwd C at kf-2+s; rev D at kb-2+s
        P[0].out_off[s] = off;
        off += dlen(kf - 2 + s, M, N);
    }
    for (int s = 0; s < 3; s++) {
        P[0].out_off[3 + s] = off;
        off += dlen(kf - 2 + s, M, N);
    }
    for (int s = 0; s < 3; s++) {
        P[1].out_off[s] = off;
        off += dlen(kb - 2 + s, M, N);
    }
    CU(c->main.out.ensure((size_t)std::max<int64_t>(off, 1) * esz));
    for (int s = 0; s < 3; s++) {
        const int64_t Lf = dlen(kf - 2 + s, M, N), Lb = dlen(kb - 2 + s, M, N);
        if (Lf > 0) {
            CU(cudaMemcpyAsync((char*)c->main.out.p + P[0].out_off[s] * esz, fwd_d[s], Lf * esz, cudaMemcpyDefault, c->st));
            CU(cudaMemcpyAsync((char*)c->main.out.p + P[0].out_off[3 + s] * esz, fwd_c[s], Lf * esz, cudaMemcpyDefault,
                               c->st));
        }
        if (Lb > 0)
            CU(cudaMemcpyAsync((char*)c->main.out.p + P[1].out_off[s] * esz, bwd_d[s], Lb * esz, cudaMemcpyDefault, c->st));
    }
    PivotDesc v{};
    v.fwd = 0;
    v.bwd = 1;
    v.M = (int32_t)M;
    v.N = (int32_t)N;
    v.kf = (int32_t)kf;
    v.kb = (int32_t)kb;
    v.highest = pivot_highest ? 1 : 0;
    CU(c->main.passes.ensure(sizeof P));
    CU(c->main.pdesc.ensure(sizeof v));
    CU(c->main.pout.ensure(sizeof(PivotOut)));
    CU(cudaMemcpyAsync(c->main.passes.p, P, sizeof P, cudaMemcpyHostToDevice, c->st));
    CU(cudaMemcpyAsync(c->main.pdesc.p, &v, sizeof v, cudaMemcpyHostToDevice, c->st));
    const size_t scb = pivot_scratch_bytes(1);
    CU(c->main.pscratch.ensure(scb));
    CU(c->main.pdone.ensure_init(sizeof(unsigned), 0, c->st));  // the kernel leaves it at zero
    CU(launch_pivots(precision, c->main.passes.as<PassDesc>(), c->main.pdesc.as<PivotDesc>(), 1, c->main.out.p,
                     c->main.pout.as<PivotOut>(), c->main.pscratch.p, c->main.pdone.as<unsigned>(), c->st));
    g_launches++;
    PivotOut po{};
    CU(cudaMemcpyAsync(&po, c->main.pout.p, sizeof po, cudaMemcpyDeviceToHost, c->st));
    CU(cudaStreamSynchronize(c->st));
    ijk[0] = po.i;
    ijk[1] = po.j;
    ijk[2] = po.k;
    *total = po.total;
    return LMDTW_OK;
}

int lmdtw_result_info(const lmdtw_result_t* r, lmdtw_align_info_t* info) {
    if (!r || !info) return set_err(LMDTW_EINVAL, "null result");
    *info = r->info;
    return LMDTW_OK;
}

int lmdtw_result_path(const lmdtw_result_t* r, int64_t* path_out) {
    if (!r || !path_out) return set_err(LMDTW_EINVAL, "null result");
    if (r->info.path_len > 0) memcpy(path_out, r->path.get(), (size_t)r->info.path_len * 2 * sizeof(int64_t));
    return LMDTW_OK;
}

int lmdtw_result_pivots(const lmdtw_result_t* r, lmdtw_pivot_t* pivots_out) {
    if (!r || (!pivots_out && !r->pivots.empty())) return set_err(LMDTW_EINVAL, "null result");
    if (!r->pivots.empty()) memcpy(pivots_out, r->pivots.data(), r->pivots.size() * sizeof(lmdtw_pivot_t));
    return LMDTW_OK;
}

void lmdtw_result_free(lmdtw_result_t* r) { delete r; }

int lmdtw_path_cost(const float* X, int64_t M, const float* Y, int64_t N, int32_t d, const int64_t* path,
                    int64_t K, int32_t precision, double* cost) {
    if (precision != 32 && precision != 64) return set_err(LMDTW_EINVAL, "precision must be 32 or 64");
    if (d < 1 || K < 1) return set_err(LMDTW_EINVAL, "empty path or bad dimension");
    for (int64_t q = 0; q < K; q++)
        if (path[2 * q] < 0 || path[2 * q] >= M || path[2 * q + 1] < 0 || path[2 * q + 1] >= N)
            return set_err(LMDTW_EINVAL, "path index out of range");
    if (precision == 32) {
        float total = 0.0f;
        for (int64_t q = 0; q < K; q++) {
            const float* x = X + path[2 * q] * d;
            const float* y = Y + path[2 * q + 1] * d;
            float s = 0.0f;
            for (int t = 0; t < d; t++) {
                const float df = x[t] - y[t];
                const float sq = df * df;
                s = s + sq;
            }
            total = total + std::sqrt(s);
        }
        *cost = (double)total;
    } else {
        double total = 0.0;
        for (int64_t q = 0; q < K; q++) {
            const float* x = X + path[2 * q] * d;
            const float* y = Y + path[2 * q + 1] * d;
            double s = 0.0;
            for (int t = 0; t < d; t++) {
                const double df = (double)x[t] - (double)y[t];
                const double sq = df * df;
                s = s + sq;
            }
            total = total + std::sqrt(s);
        }
        *cost = total;
    }
    return LMDTW_OK;
}

}  // extern "C"

// ------------------------------------------------ per-path steps (window.cu)
namespace {
// Raw float32 rows on the device: host rows copied into `buf`, device rows used in place.
int stage_raw(Ctx& c, DBuf& buf, const float* src, int64_t rows, int d, int mem, const float** out) {
    if (mem == LMDTW_MEM_DEVICE) {
        *out = src;
        return LMDTW_OK;
    }
    const size_t b = (size_t)std::max<int64_t>(rows, 1) * d * sizeof(float);
    CU(buf.ensure(b));
    CU(cudaMemcpyAsync(buf.p, src, (size_t)rows * d * sizeof(float), cudaMemcpyHostToDevice, c.st));
    c.h2d += (long long)rows * d * sizeof(float);
    *out = buf.as<float>();
    return LMDTW_OK;
}

// approx.Window.validate (approx.py:52-63), same checks and messages.
int validate_window(const int64_t* lo, const int64_t* hi, int64_t M, int64_t N) {
    if (M < 1) return set_err(LMDTW_EINVAL, "window lo/hi length mismatch");
    for (int64_t i = 0; i < M; i++)
        if (lo[i] < 0 || hi[i] >= N || lo[i] > hi[i]) return set_err(LMDTW_EINVAL, "window intervals empty or out of range");
    for (int64_t i = 1; i < M; i++)
        if (lo[i] < lo[i - 1] || hi[i] < hi[i - 1]) return set_err(LMDTW_EINVAL, "window staircase not monotone");
    if (lo[0] != 0 || hi[M - 1] != N - 1) return set_err(LMDTW_EINVAL, "window must contain (0,0) and (M-1,N-1)");
    for (int64_t i = 1; i < M; i++)
        if (lo[i] > hi[i - 1] + 1) return set_err(LMDTW_EINVAL, "window rows disconnected; no warping path fits");
    return LMDTW_OK;
}
}  // namespace

extern "C" {

int lmdtw_window_dtw(int device, const float* X, int64_t M, const float* Y, int64_t N, int32_t d,
                     const int64_t* lo, const int64_t* hi, const int32_t tie[3], int32_t precision, int32_t mem,
                     double* cost, int64_t* path_out, int64_t* path_len, int64_t* cells) {
    TRY(validate_common(M, N, d, precision));
    TRY(validate_tie(tie));
    TRY(validate_window(lo, hi, M, N));
    CtxLease c;
    TRY(lease_ctx(device, c));
    c->call_launches = 0;
    c->h2d = c->d2h = 0;
    const float *dX = nullptr, *dY = nullptr;
    TRY(stage_raw(*c, c->xraw, X, M, d, mem, &dX));
    TRY(stage_raw(*c, c->yraw, Y, N, d, mem, &dY));
    // window rows, backpointer word offsets, pipeline width
    std::vector<int32_t> lo32(M), hi32(M);
    std::vector<int64_t> wo(M + 1);
    int64_t ncell = 0, span = 0;
    wo[0] = 0;
    for (int64_t i = 0; i < M; i++) {
        lo32[i] = (int32_t)lo[i];
        hi32[i] = (int32_t)hi[i];
        wo[i + 1] = wo[i] + (hi[i] >> 5) - (lo[i] >> 5) + 1;
        ncell += hi[i] - lo[i] + 1;
    }
    for (int64_t g = 0; g * 32 < M; g++) span = std::max<int64_t>(span, hi[std::min(M - 1, 32 * g + 31)] - lo[32 * g] + 32);
    // groups in flight: a group trails its predecessor by >= 32 steps
    const int warps = (int)std::min<int64_t>(16, std::max<int64_t>(2, (span + 31) / 32 + 1));
    const int W = precision == 32 ? 1 : 2;
    const int64_t bnd_words = 2 * ((N + 1) & ~1LL) * W;
    CU(c->wlo.ensure(M * sizeof(int32_t)));
    CU(c->whi.ensure(M * sizeof(int32_t)));
    CU(c->woff.ensure((M + 1) * sizeof(int64_t)));
    CU(c->wbp.ensure((size_t)wo[M] * 8));
    CU(c->wbnd.ensure((size_t)bnd_words * 8));
    CU(c->wdesc.ensure(sizeof(BandDesc)));
    CU(c->wcost.ensure(8));
    CU(c->wpath.ensure((size_t)(M + N) * 2 * sizeof(int)));
    CU(c->wpoff.ensure(sizeof(int64_t)));
    CU(c->wplen.ensure(sizeof(int)));
    BandDesc bd{};
    bd.M = (int32_t)M;
    bd.N = (int32_t)N;
    const int64_t zero = 0;
    CU(cudaMemcpyAsync(c->wlo.p, lo32.data(), M * sizeof(int32_t), cudaMemcpyHostToDevice, c->st));
    CU(cudaMemcpyAsync(c->whi.p, hi32.data(), M * sizeof(int32_t), cudaMemcpyHostToDevice, c->st));
    CU(cudaMemcpyAsync(c->woff.p, wo.data(), (M + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, c->st));
    CU(cudaMemcpyAsync(c->wdesc.p, &bd, sizeof bd, cudaMemcpyHostToDevice, c->st));
    CU(cudaMemcpyAsync(c->wpoff.p, &zero, sizeof zero, cudaMemcpyHostToDevice, c->st));
    CU(cudaMemsetAsync(c->wbnd.p, 0xFF, (size_t)bnd_words * 8, c->st));  // tag -1
    const int tie_i[3] = {tie[0], tie[1], tie[2]};
    CU(launch_band(precision, dX, dY, d, c->wdesc.as<BandDesc>(), 1, warps, c->wlo.as<int32_t>(),
                   c->whi.as<int32_t>(), c->woff.as<int64_t>(), c->wbp.as<unsigned long long>(),
                   c->wbnd.as<unsigned long long>(), c->wcost.p, tie_i, c->st));
    CU(launch_band_backtrace(c->wdesc.as<BandDesc>(), 1, c->wlo.as<int32_t>(), c->woff.as<int64_t>(),
                             c->wbp.as<unsigned long long>(), c->wpath.as<int>(), c->wpoff.as<int64_t>(),
                             c->wplen.as<int>(), c->st));
    c->call_launches += 2;
    g_launches += 2;
    int plen = 0;
    double dcost = 0;
    float fcost = 0;
    std::vector<int> rev((size_t)(M + N) * 2);
    CU(cudaMemcpyAsync(&plen, c->wplen.p, sizeof(int), cudaMemcpyDeviceToHost, c->st));
    if (precision == 32)
        CU(cudaMemcpyAsync(&fcost, c->wcost.p, sizeof(float), cudaMemcpyDeviceToHost, c->st));
    else
        CU(cudaMemcpyAsync(&dcost, c->wcost.p, sizeof(double), cudaMemcpyDeviceToHost, c->st));
    CU(cudaMemcpyAsync(rev.data(), c->wpath.p, rev.size() * sizeof(int), cudaMemcpyDeviceToHost, c->st));
    CU(cudaStreamSynchronize(c->st));
    c->prof_collect();
    if (plen < 0) return set_err(LMDTW_EINTERNAL, "backtrace escaped the window; window was infeasible");
    for (int q = 0; q < plen; q++) {
        path_out[2 * q] = rev[2 * (plen - 1 - q)];
        path_out[2 * q + 1] = rev[2 * (plen - 1 - q) + 1];
    }
    if (path_len) *path_len = plen;
    if (cost) *cost = precision == 32 ? (double)fcost : dcost;
    if (cells) *cells = ncell;
    return LMDTW_OK;
}

int lmdtw_frame_costs(int device, const float* A, const float* B, int64_t K, int32_t d, int32_t precision,
                      int32_t mem, void* out) {
    if (precision != 32 && precision != 64) return set_err(LMDTW_EINVAL, "precision must be 32 or 64");
    if (d < 1 || K < 0) return set_err(LMDTW_EINVAL, "bad frame count or dimension");
    if (K == 0) return LMDTW_OK;
    CtxLease c;
    TRY(lease_ctx(device, c));
    const float *dA = nullptr, *dB = nullptr;
    TRY(stage_raw(*c, c->xraw, A, K, d, mem, &dA));
    TRY(stage_raw(*c, c->yraw, B, K, d, mem, &dB));
    const size_t esz = precision == 32 ? 4 : 8;
    CU(c->pcost2.ensure((size_t)K * esz));
    CU(launch_path_costs(precision, dA, dB, d, nullptr, K, nullptr, nullptr, nullptr, c->pcost2.p, c->st));
    g_launches++;
    CU(cudaMemcpyAsync(out, c->pcost2.p, (size_t)K * esz, cudaMemcpyDeviceToHost, c->st));
    CU(cudaStreamSynchronize(c->st));
    return LMDTW_OK;
}

int lmdtw_path_cost_batch(int device, int32_t npaths, const float* const* X, const int64_t* M,
                          const float* const* Y, const int64_t* N, int32_t d, const int64_t* const* paths,
                          const int64_t* K, int32_t precision, int32_t mem, double* costs_out) {
    if (precision != 32 && precision != 64) return set_err(LMDTW_EINVAL, "precision must be 32 or 64");
    if (npaths < 1 || d < 1) return set_err(LMDTW_EINVAL, "npaths must be >= 1 and d >= 1");
    int64_t ncell = 0, xrows = 0, yrows = 0;
    for (int p = 0; p < npaths; p++) {
        if (K[p] < 1) return set_err(LMDTW_EINVAL, "empty path");
        for (int64_t q = 0; q < K[p]; q++) {
            const int64_t i = paths[p][2 * q], j = paths[p][2 * q + 1];
            if (i < 0 || i >= M[p] || j < 0 || j >= N[p]) return set_err(LMDTW_EINVAL, "path index out of range");
        }
        ncell += K[p];
        xrows += M[p];
        yrows += N[p];
    }
    CtxLease c;
    TRY(lease_ctx(device, c));
    // features: concatenated raw rows (device inputs are gathered by copies)
    CU(c->xraw.ensure((size_t)xrows * d * 4));
    CU(c->yraw.ensure((size_t)yrows * d * 4));
    std::vector<int64_t> xo(npaths), yo(npaths), off(npaths + 1);
    std::vector<int32_t> pid((size_t)ncell);
    std::vector<int64_t> cells((size_t)ncell * 2);
    const cudaMemcpyKind kind = mem == LMDTW_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
    int64_t xr = 0, yr = 0, w = 0;
    for (int p = 0; p < npaths; p++) {
        xo[p] = xr;
        yo[p] = yr;
        off[p] = w;
        CU(cudaMemcpyAsync(c->xraw.as<float>() + xr * d, X[p], (size_t)M[p] * d * 4, kind, c->st));
        CU(cudaMemcpyAsync(c->yraw.as<float>() + yr * d, Y[p], (size_t)N[p] * d * 4, kind, c->st));
        xr += M[p];
        yr += N[p];
        memcpy(cells.data() + 2 * w, paths[p], (size_t)K[p] * 2 * sizeof(int64_t));
        std::fill(pid.begin() + w, pid.begin() + w + K[p], p);
        w += K[p];
    }
    off[npaths] = w;
    const size_t esz = precision == 32 ? 4 : 8;
    CU(c->pcells.ensure((size_t)ncell * 16));
    CU(c->ppid.ensure((size_t)ncell * 4));
    CU(c->pxoff.ensure((size_t)npaths * 8));
    CU(c->pyoff.ensure((size_t)npaths * 8));
    CU(c->poffs.ensure((size_t)(npaths + 1) * 8));
    CU(c->pcost2.ensure((size_t)ncell * esz));
    CU(c->pout2.ensure((size_t)npaths * 8));
    CU(cudaMemcpyAsync(c->pcells.p, cells.data(), (size_t)ncell * 16, cudaMemcpyHostToDevice, c->st));
    CU(cudaMemcpyAsync(c->ppid.p, pid.data(), (size_t)ncell * 4, cudaMemcpyHostToDevice, c->st));
    CU(cudaMemcpyAsync(c->pxoff.p, xo.data(), (size_t)npaths * 8, cudaMemcpyHostToDevice, c->st));
    CU(cudaMemcpyAsync(c->pyoff.p, yo.data(), (size_t)npaths * 8, cudaMemcpyHostToDevice, c->st));
    CU(cudaMemcpyAsync(c->poffs.p, off.data(), (size_t)(npaths + 1) * 8, cudaMemcpyHostToDevice, c->st));
    CU(launch_path_costs(precision, c->xraw.as<float>(), c->yraw.as<float>(), d, c->pcells.as<int64_t>(), ncell,
                         c->pxoff.as<int64_t>(), c->pyoff.as<int64_t>(), c->ppid.as<int32_t>(), c->pcost2.p, c->st));
    CU(launch_seq_sums(precision, c->pcost2.p, c->poffs.as<int64_t>(), npaths, c->pout2.as<double>(), c->st));
    g_launches += 2;
    CU(cudaMemcpyAsync(costs_out, c->pout2.p, (size_t)npaths * 8, cudaMemcpyDeviceToHost, c->st));
    CU(cudaStreamSynchronize(c->st));
    return LMDTW_OK;
}

int lmdtw_discrepancy(int device, const int64_t* p1, int64_t K1, const int64_t* p2, int64_t K2,
                      int64_t* errors_out) {
    if (K1 < 1 || K2 < 1) return set_err(LMDTW_EINVAL, "path must be a nonempty (K, 2) index array");
    if (p1[0] != p2[0] || p1[1] != p2[1] || p1[2 * (K1 - 1)] != p2[2 * (K2 - 1)] ||
        p1[2 * (K1 - 1) + 1] != p2[2 * (K2 - 1) + 1])
        return set_err(LMDTW_EINVAL, "paths have mismatched endpoints; not comparable");
    const int64_t M = p1[2 * (K1 - 1)] + 1, N = p1[2 * (K1 - 1) + 1] + 1;
    if (M < 1 || N < 1) return set_err(LMDTW_EINVAL, "path index out of range");
    for (int64_t q = 0; q < K1; q++)
        if (p1[2 * q] < 0 || p1[2 * q] >= M || p1[2 * q + 1] < 0 || p1[2 * q + 1] >= N)
            return set_err(LMDTW_EINVAL, "path index out of range");
    for (int64_t q = 0; q < K2; q++)
        if (p2[2 * q] < 0 || p2[2 * q] >= M || p2[2 * q + 1] < 0 || p2[2 * q + 1] >= N)
            return set_err(LMDTW_EINVAL, "path index out of range");
    CtxLease c;
    TRY(lease_ctx(device, c));
    // dsc: p1 | p2 | scratch 2M+2N | errors 2 K1 (int64 each)
    const size_t n64 = (size_t)(2 * K1 + 2 * K2 + 2 * M + 2 * N + 2 * K1);
    CU(c->dsc.ensure(n64 * 8));
    int64_t* d1 = c->dsc.as<int64_t>();
    int64_t* d2 = d1 + 2 * K1;
    long long* scr = reinterpret_cast<long long*>(d2 + 2 * K2);
    long long* err = scr + 2 * M + 2 * N;
    CU(cudaMemcpyAsync(d1, p1, (size_t)K1 * 16, cudaMemcpyHostToDevice, c->st));
    CU(cudaMemcpyAsync(d2, p2, (size_t)K2 * 16, cudaMemcpyHostToDevice, c->st));
    CU(launch_discrepancy(d1, K1, d2, K2, M, N, scr, err, c->st));
    g_launches += 6;
    CU(cudaMemcpyAsync(errors_out, err, (size_t)K1 * 16, cudaMemcpyDeviceToHost, c->st));
    CU(cudaStreamSynchronize(c->st));
    return LMDTW_OK;
}

}  // extern "C"
