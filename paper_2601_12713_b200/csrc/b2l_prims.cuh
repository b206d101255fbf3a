// Device-wide primitives for the trace-analysis pipeline (sm_100a, hand-written):
//   * stream-ordered scratch buffers (cudaMallocAsync pool)
//   * generic single-pass scan (decoupled look-back, one launch) over functor inputs/outputs,
//     with a segmented wrapper -- used for counts, prefix maxima, the max-plus
//     depth scan of alloc/delete pairing, run ids, compaction
//   * stable LSD radix sort of (multi-word u64 key, u32 value) records: 8-bit
//     digits, one histogram read for all digits, one Onesweep launch per digit
//     (warp __match_any_sync multisplit ranking, decoupled look-back, coalesced
//     digit-ordered scatter through shared memory); digit passes whose byte never
//     varies are skipped (planned from an OR-of-XOR reduction), so wide composite
//     keys cost only their live bytes
//   * segmented fix-up: records ordered by a key prefix become ordered by the full
//     key in one pass (runs found by head-bit scans), and the wide sort built on it
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <initializer_list>
#include <map>
#include <mutex>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <utility>
#include <thread>
#include <vector>

#include "b2l_common.cuh"

namespace b2l {

struct EngineErr {
    int code;
    std::string msg;
};
inline void ck(cudaError_t e, const char *what) {
    if (e != cudaSuccess)
        throw EngineErr{e == cudaErrorMemoryAllocation ? B2L_E_OOM : B2L_E_CUDA,
                        std::string(what) + ": " + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) + ")"};
}
#define CK(call) ::b2l::ck((call), #call)
#define CK_LAUNCH(what) ::b2l::ck(cudaGetLastError(), what)

// ---------------------------------------------------------------- scratch buffers
// B2L_TRACE: host time spent in the pool's allocate/free calls (diagnostics)
struct AllocStats {
    std::atomic<uint64_t> n{0}, ns{0};
    bool on = getenv("B2L_TRACE") != nullptr;
};
// B2L_SYNC_STATS: host round trips per analysis call (read-backs and stream waits), per thread
struct SyncStats {
    std::atomic<uint64_t> n{0}, ns{0}, ln{0}, lns{0};  // round trips; launches and their host time
    bool on = getenv("B2L_SYNC_STATS") != nullptr;
};
inline SyncStats &sync_stats() {
    static SyncStats a;
    return a;
}
// B2L_SYNC_STATS=2: also every round trip's caller line, host start and wait (printed per call)
struct SyncRec {
    int line;
    std::chrono::steady_clock::time_point t0;
    uint64_t ns;
    size_t thread;
};
inline std::mutex &sync_log_mu() {
    static std::mutex m;
    return m;
}
inline std::vector<SyncRec> &sync_log() {
    static std::vector<SyncRec> v;
    return v;
}
struct SyncTimer {
    bool on;
    int line;
    std::chrono::steady_clock::time_point t0;
    explicit SyncTimer(int ln = 0) : on(sync_stats().on), line(ln) {
        if (on) t0 = std::chrono::steady_clock::now();
    }
    ~SyncTimer() {
        if (!on) return;
        const uint64_t ns = (uint64_t)std::chrono::duration_cast<std::chrono::nanoseconds>(
            std::chrono::steady_clock::now() - t0).count();
        sync_stats().n++;
        sync_stats().ns += ns;
        static const bool detail = getenv("B2L_SYNC_STATS") && getenv("B2L_SYNC_STATS")[0] == '2';
        if (detail) {
            std::lock_guard<std::mutex> g(sync_log_mu());
            sync_log().push_back({line, t0, ns, std::hash<std::thread::id>()(std::this_thread::get_id())});
        }
    }
};
inline AllocStats &alloc_stats() {
    static AllocStats a;
    return a;
}
struct AllocTimer {
    std::chrono::steady_clock::time_point t0;
    bool on;
    AllocTimer() : on(alloc_stats().on) {
        if (on) t0 = std::chrono::steady_clock::now();
    }
    ~AllocTimer() {
        if (!on) return;
        alloc_stats().n++;
        alloc_stats().ns += (uint64_t)std::chrono::duration_cast<std::chrono::nanoseconds>(
                                std::chrono::steady_clock::now() - t0).count();
    }
};
// Call-scoped scratch arena: one pool allocation per engine call, carved by an atomic bump
// pointer and released as a whole.  An analysis call makes ~600 scratch allocations/frees; through
// the stream-ordered pool they cost ~1.5 ms of host time (three host threads contending on the
// driver), about the whole call at 1M events.  Buffers that do not fit fall back to the pool.
struct Arena {
    uint8_t *base = nullptr;
    size_t cap = 0;
    std::atomic<size_t> off{0};
    cudaStream_t s = nullptr;
    // A zeroed pool at the head of the arena (one fill when it opens) serves the small scratch
    // that must start at zero -- look-back flags and tile tickets of the scans -- so a scan is one
    // launch instead of a fill and a launch (~35 scans per analysis call).
    uint8_t *zbase = nullptr;
    size_t zcap = 0;
    bool mailbox = true;  // small read-backs through the mailbox (read_back); off for huge calls
    std::atomic<size_t> zoff{0};
    void open(size_t bytes, cudaStream_t st, size_t zero_bytes = size_t(64) << 10) {
        s = st;
        if (!bytes) return;
        zero_bytes = (zero_bytes + 255) & ~size_t(255);
        if (cudaMallocAsync((void **)&base, bytes + zero_bytes, st) != cudaSuccess) {
            cudaGetLastError();  // no arena: every buffer comes from the pool
            base = nullptr;
            return;
        }
        zbase = base, zcap = zero_bytes;
        base += zero_bytes;
        cap = bytes;
        zero_pool();
    }
    inline void zero_pool();
    void *take(size_t bytes) {
        bytes = (bytes + 255) & ~size_t(255);
        const size_t o = off.fetch_add(bytes, std::memory_order_relaxed);
        return o + bytes <= cap ? base + o : nullptr;
    }
    void *take_zeroed(size_t bytes) {
        if (!zbase) return nullptr;
        bytes = (bytes + 15) & ~size_t(15);
        const size_t o = zoff.fetch_add(bytes, std::memory_order_relaxed);
        return o + bytes <= zcap ? zbase + o : nullptr;
    }
    ~Arena() {
        if (zbase) cudaFreeAsync(zbase, s);
    }
};
// the arena the calling thread's buffers come from (set for the duration of an engine call, and in
// the side threads it spawns)
inline thread_local Arena *t_arena = nullptr;
struct ArenaUse {
    Arena *prev;
    explicit ArenaUse(Arena *a) : prev(t_arena) { t_arena = a; }
    ~ArenaUse() { t_arena = prev; }
};

// Programmatic dependent launch: kernels of a chain are launched with programmatic stream
// serialisation, enter with griddepcontrol.wait (every prerequisite grid complete, its memory
// visible) and immediately allow their own dependents to be scheduled, so the next kernel's
// launch processing overlaps this one instead of following its completion (small traces run
// ~50 dependent kernels per chain).  Kernels launched without the attribute are unaffected.
__device__ __forceinline__ void pdl_enter() {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
inline bool pdl_on() {
    static const bool on = !getenv("B2L_NO_PDL");
    return on;
}
template <typename... KArgs, typename... Args>
inline void launch_k(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid, cfg.blockDim = block, cfg.dynamicSmemBytes = smem, cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at, cfg.numAttrs = pdl_on() ? 1 : 0;
    if (!sync_stats().on) {
        ck(cudaLaunchKernelEx(&cfg, k, args...), "cudaLaunchKernelEx");
        return;
    }
    const auto t0 = std::chrono::steady_clock::now();
    ck(cudaLaunchKernelEx(&cfg, k, args...), "cudaLaunchKernelEx");
    sync_stats().ln += 1;
    sync_stats().lns += (uint64_t)std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now() - t0).count();
}

// Device-side fill / copy as kernels, never through a copy engine: the engines may be busy with a
// large host->device upload (analyze_many queues the next trace's upload beside this analysis), and
// a memset or device-to-device copy queued behind it would stall the whole dependent chain.
static __global__ void k_fill_bytes(uint8_t *__restrict__ p, size_t n, uint32_t v4) {
    pdl_enter();
    const size_t head = (16 - ((uintptr_t)p & 15)) & 15;
    const size_t h = head < n ? head : n;
    const size_t tid = (size_t)blockIdx.x * blockDim.x + threadIdx.x, stride = (size_t)gridDim.x * blockDim.x;
    for (size_t i = tid; i < h; i += stride) p[i] = (uint8_t)v4;
    const size_t nv = (n - h) / 16;
    uint4 *q = reinterpret_cast<uint4 *>(p + h);
    for (size_t i = tid; i < nv; i += stride) q[i] = make_uint4(v4, v4, v4, v4);
    for (size_t i = h + nv * 16 + tid; i < n; i += stride) p[i] = (uint8_t)v4;
}
static __global__ void k_copy_bytes(uint8_t *__restrict__ d, const uint8_t *__restrict__ s, size_t n) {
    pdl_enter();
    const size_t tid = (size_t)blockIdx.x * blockDim.x + threadIdx.x, stride = (size_t)gridDim.x * blockDim.x;
    if ((((uintptr_t)d | (uintptr_t)s) & 15) == 0) {
        const size_t nv = n / 16;
        for (size_t i = tid; i < nv; i += stride) reinterpret_cast<uint4 *>(d)[i] = reinterpret_cast<const uint4 *>(s)[i];
        for (size_t i = nv * 16 + tid; i < n; i += stride) d[i] = s[i];
    } else {
        for (size_t i = tid; i < n; i += stride) d[i] = s[i];
    }
}
inline unsigned fill_grid(size_t bytes) {
    const size_t b = (bytes / 16 + 255) / 256;
    return (unsigned)(b < 1 ? 1 : (b > 148 * 8 ? 148 * 8 : b));
}
inline void dev_memset(void *p, int v, size_t bytes, cudaStream_t s) {
    if (!bytes) return;
    const uint32_t b = (uint32_t)(v & 0xFF);
    launch_k(k_fill_bytes, fill_grid(bytes), 256, 0, s, (uint8_t *)p, bytes, b | (b << 8) | (b << 16) | (b << 24));
    CK(cudaGetLastError());
}
inline void Arena::zero_pool() { dev_memset(zbase, 0, zcap, s); }
// u64 words [0, n0) = 0, [n0, n0 + n1) = ~0, then n2 more zeros, in one launch (accumulators
// whose max / min slots start at the identity)
static __global__ void k_init_u64(uint64_t *__restrict__ p, size_t n0, size_t n1, size_t n2) {
    pdl_enter();
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n0 + n1 + n2; i += (size_t)gridDim.x * blockDim.x)
        p[i] = (i >= n0 && i < n0 + n1) ? ~0ull : 0ull;
}
inline void init_u64(void *p, size_t n0, size_t n1, size_t n2, cudaStream_t s) {
    if (!n0 && !n1 && !n2) return;
    launch_k(k_init_u64, fill_grid((n0 + n1 + n2) * 8), 256, 0, s, (uint64_t *)p, n0, n1, n2);
    CK(cudaGetLastError());
}
inline void dev_copy(void *d, const void *src, size_t bytes, cudaStream_t s) {
    if (!bytes) return;
    launch_k(k_copy_bytes, fill_grid(bytes), 256, 0, s, (uint8_t *)d, (const uint8_t *)src, bytes);
    CK(cudaGetLastError());
}

template <class T>
struct DBuf {
    T *p = nullptr;
    size_t n = 0;
    cudaStream_t s = nullptr;
    bool arena = false;  // carved from the call's arena: released with it
    DBuf() = default;
    DBuf(size_t n_, cudaStream_t st) { alloc(n_, st); }
    void alloc(size_t n_, cudaStream_t st) {
        release();
        s = st;
        n = n_;
        if (!n_) return;
        if (t_arena) {
            if (void *q = t_arena->take(n_ * sizeof(T))) {
                p = (T *)q;
                arena = true;
                return;
            }
        }
        AllocTimer at;
        CK(cudaMallocAsync((void **)&p, n_ * sizeof(T), st));
    }
    void zero() {
        if (n) dev_memset(p, 0, n * sizeof(T), s);
    }
    // zero-initialised: from the call arena's zeroed pool when it has room (no fill launch)
    void alloc_zeroed(size_t n_, cudaStream_t st) {
        release();
        s = st;
        n = n_;
        if (!n_) return;
        if (t_arena) {
            if (void *q = t_arena->take_zeroed(n_ * sizeof(T))) {
                p = (T *)q;
                arena = true;
                return;
            }
        }
        alloc(n_, st);
        zero();
    }
    void release() {
        if (p && !arena) {
            AllocTimer at;
            cudaFreeAsync(p, s);
        }
        p = nullptr;
        n = 0;
        arena = false;
    }
    ~DBuf() { release(); }
    DBuf(const DBuf &) = delete;
    DBuf &operator=(const DBuf &) = delete;
    DBuf(DBuf &&o) noexcept : p(o.p), n(o.n), s(o.s), arena(o.arena) { o.p = nullptr, o.n = 0, o.arena = false; }
    DBuf &operator=(DBuf &&o) noexcept {
        release();
        p = o.p, n = o.n, s = o.s, arena = o.arena;
        o.p = nullptr, o.n = 0, o.arena = false;
        return *this;
    }
    operator T *() const { return p; }
};

inline unsigned grid_for(size_t n, unsigned per_block, unsigned cap = 148u * 64u) {
    size_t g = (n + per_block - 1) / per_block;
    if (g < 1) g = 1;
    return (unsigned)(g < cap ? g : cap);
}

// ---------------------------------------------------------------- scan monoids
struct SumU32 {
    using T = uint32_t;
    static __device__ __forceinline__ T identity() { return 0; }
    static __device__ __forceinline__ T combine(T a, T b) { return a + b; }
};
struct SumU64 {
    using T = uint64_t;
    static __device__ __forceinline__ T identity() { return 0; }
    static __device__ __forceinline__ T combine(T a, T b) { return a + b; }
};
struct MaxU64 {
    using T = uint64_t;
    static __device__ __forceinline__ T identity() { return 0; }
    static __device__ __forceinline__ T combine(T a, T b) { return a > b ? a : b; }
};
struct MaxI64 {
    using T = long long;
    static __device__ __forceinline__ T identity() { return (long long)(-0x7fffffffffffffffll - 1); }
    static __device__ __forceinline__ T combine(T a, T b) { return a > b ? a : b; }
};
// Clamped-depth transfer functions f(d) = max(d + a, b) under composition (apply a then b):
// the alloc/delete LIFO depth d_i = max(d_{i-1} + x_i, 0) of prep.py:45-96 as a scan.
struct MaxPlus {
    struct T {
        long long a, b;
    };
    static __device__ __forceinline__ T identity() { return T{0, (long long)(-0x3fffffffffffffffll)}; }
    static __device__ __forceinline__ T combine(T f, T g) {
        long long bb = f.b + g.a;
        return T{f.a + g.a, bb > g.b ? bb : g.b};
    }
};
// Segmented wrapper: a set flag starts a new segment.
template <class Op>
struct Seg {
    struct T {
        uint32_t flag;
        typename Op::T v;
    };
    static __device__ __forceinline__ T identity() { return T{0u, Op::identity()}; }
    static __device__ __forceinline__ T combine(T a, T b) {
        return T{a.flag | b.flag, b.flag ? b.v : Op::combine(a.v, b.v)};
    }
};

// ---------------------------------------------------------------- generic tile scan
constexpr int SCAN_THREADS = 256;
constexpr int SCAN_ITEMS = 8;
constexpr int SCAN_TILE = SCAN_THREADS * SCAN_ITEMS;

template <class T>
__device__ __forceinline__ T shfl_up_t(T v, int off) {
    static_assert(sizeof(T) % 4 == 0, "scan values are whole words");
    unsigned *d = reinterpret_cast<unsigned *>(&v);
#pragma unroll
    for (int i = 0; i < (int)(sizeof(T) / 4); ++i) d[i] = __shfl_up_sync(0xffffffffu, d[i], off);
    return v;
}
// Exclusive block scan (256 threads): warp shuffle scans, then the 8 warp totals scanned by every
// thread from shared memory -- two barriers.  `sm` needs SCAN_THREADS / 32 + 1 entries.
template <class Op>
__device__ __forceinline__ typename Op::T block_excl_scan(typename Op::T v, typename Op::T *sm,
                                                          typename Op::T &total) {
    using T = typename Op::T;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    T x = v;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const T y = shfl_up_t(x, off);
        if (lane >= off) x = Op::combine(y, x);
    }
    if (lane == 31) sm[warp] = x;
    __syncthreads();
    T before = Op::identity(), tot = Op::identity();
#pragma unroll
    for (int w = 0; w < SCAN_THREADS / 32; ++w) {
        const T c = sm[w];
        if (w < warp) before = Op::combine(before, c);
        tot = Op::combine(tot, c);
    }
    total = tot;
    T ex = shfl_up_t(x, 1);
    ex = lane == 0 ? before : Op::combine(before, ex);
    __syncthreads();  // sm is reused by the caller
    return ex;
}


// In-place exclusive scan of per-tile partials by one CTA (the fused front pass).
template <class Op>
__global__ void __launch_bounds__(SCAN_THREADS) k_scan_partials(typename Op::T *partials, size_t np,
                                                                 typename Op::T *d_total) {
    pdl_enter();
    using T = typename Op::T;
    __shared__ T sm[SCAN_THREADS];
    T carry = Op::identity();
    for (size_t c0 = 0; c0 < np; c0 += SCAN_TILE) {
        const size_t base = c0 + (size_t)threadIdx.x * SCAN_ITEMS;
        T items[SCAN_ITEMS];
        T acc = Op::identity();
#pragma unroll
        for (int k = 0; k < SCAN_ITEMS; ++k) {
            items[k] = base + k < np ? partials[base + k] : Op::identity();
            acc = Op::combine(acc, items[k]);
        }
        T total;
        T ex = Op::combine(carry, block_excl_scan<Op>(acc, sm, total));
#pragma unroll
        for (int k = 0; k < SCAN_ITEMS; ++k) {
            if (base + k < np) partials[base + k] = ex;
            ex = Op::combine(ex, items[k]);
        }
        carry = Op::combine(carry, total);
    }
    if (threadIdx.x == 0 && d_total) *d_total = carry;
}

// ---------------------------------------------------------------- single-pass scan
// One launch per scan: tiles take ids in launch order, publish their aggregate, and a warp
// looks back over 32 predecessors per step (flags then values; values are written before
// their flag with a fence in between, read after it through L2), so inputs are read once.
constexpr uint32_t SP_AGG = 1, SP_INC = 2;
// look-back flags sit one per 128-byte line: every resident tile polls its predecessors' flags,
// and packed flags put tens of thousands of polling threads on a handful of L2 lines (measured:
// ~10 us per tile at 1M items, about 4x the whole scan's load and store work)
#ifndef B2L_FLAG_STRIDE
#define B2L_FLAG_STRIDE 32
#endif
constexpr uint32_t FS = B2L_FLAG_STRIDE;

template <class T>
__device__ __forceinline__ T ld_l2(const T *p) {
    static_assert(sizeof(T) % 4 == 0, "scan values are whole words");
    T v;
    const unsigned *q = reinterpret_cast<const unsigned *>(p);
    unsigned *d = reinterpret_cast<unsigned *>(&v);
#pragma unroll
    for (int i = 0; i < (int)(sizeof(T) / 4); ++i) d[i] = __ldcg(q + i);
    return v;
}
template <class T>
__device__ __forceinline__ T shfl_down_t(T v, int off) {
    unsigned *d = reinterpret_cast<unsigned *>(&v);
#pragma unroll
    for (int i = 0; i < (int)(sizeof(T) / 4); ++i) d[i] = __shfl_down_sync(0xffffffffu, d[i], off);
    return v;
}

// Decoupled look-back by the whole block (all SCAN_THREADS threads, called uniformly): publishes
// this tile's aggregate, then inspects 256 predecessors per step -- one flag and one value per
// thread -- until a window holds an inclusive prefix; returns this tile's exclusive prefix and
// publishes its inclusive one.  Flags are one per 128-byte line (FS) and polled with acquire
// loads.  Measured in isolation (tools/scan_bench.cu, u32 sum scan, B200): 1M items 29 -> 11 us,
// 10M 100 -> 41 us against the earlier warp-wide look-back over packed flags with full fences.
// Value stores before the flag: a release store orders them; the pollers read flags with acquire
// loads, so neither side needs a full fence.
__device__ __forceinline__ void publish_flag(uint32_t *f, uint32_t v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(f), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t acquire_flag(const uint32_t *f) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
    return v;
}
template <class Op>
__device__ __forceinline__ typename Op::T block_lookback(uint32_t tile, typename Op::T total, typename Op::T *agg,
                                                         typename Op::T *inc, uint32_t *flag) {
    using T = typename Op::T;
    constexpr int NW = SCAN_THREADS / 32;
    __shared__ T wv[NW];
    __shared__ int wfirst[NW];
    __shared__ T prefix_sh;
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    if (tile == 0) {
        if (t == 0) {
            inc[0] = total;
            publish_flag(flag, SP_INC);  // tile 0's flag: word 0
        }
        return Op::identity();
    }
    if (t == 0) {
        agg[tile] = total;
        publish_flag(flag + (size_t)tile * FS, SP_AGG);
    }
    T prefix = Op::identity();  // meaningful in thread 0
    for (int64_t base = (int64_t)tile - 1;; base -= SCAN_THREADS) {
        const int64_t jj = base - t;  // thread t holds tile base - t (older for higher t)
        uint32_t f = SP_INC;
        if (jj >= 0)
            do {
                f = acquire_flag(flag + jj * FS);
            } while (f == 0);
        T v = jj < 0 ? Op::identity() : (f == SP_INC ? ld_l2(inc + jj) : ld_l2(agg + jj));
        const uint32_t incm = __ballot_sync(0xffffffffu, f == SP_INC);
        if (lane == 0) wfirst[warp] = incm ? warp * 32 + __ffs(incm) - 1 : SCAN_THREADS;
        __syncthreads();
        int first = SCAN_THREADS;  // newest predecessor holding an inclusive prefix
#pragma unroll
        for (int w = 0; w < NW; ++w) first = wfirst[w] < first ? wfirst[w] : first;
        if (t > first) v = Op::identity();
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {  // ordered: lane 0 gets its warp's window, oldest first
            const T o = shfl_down_t(v, off);
            if (lane + off < 32) v = Op::combine(o, v);
        }
        if (lane == 0) wv[warp] = v;
        __syncthreads();
        if (t == 0) {
            T win = wv[NW - 1];
#pragma unroll
            for (int w = NW - 2; w >= 0; --w) win = Op::combine(win, wv[w]);
            prefix = Op::combine(win, prefix);
        }
        if (first < SCAN_THREADS) break;  // uniform: every thread read the same wfirst[]
        __syncthreads();                  // wfirst / wv are rewritten by the next window
    }
    if (t == 0) {
        inc[tile] = Op::combine(prefix, total);
        publish_flag(flag + (size_t)tile * FS, SP_INC);
        prefix_sh = prefix;
    }
    __syncthreads();
    return prefix_sh;
}

// Single-pass scan tiles: 256 threads x I items (I = 16 for values of up to 8 bytes, else 8).
// Loads are block-striped (item k*256 + t for thread t: every warp access is contiguous, and a
// thread's I loads -- gathers included -- are all in flight at once) and stay in registers; a
// copy goes to shared memory in a padded blocked layout (item j at slot (j / I) * (I + 1) + j % I)
// where each thread reduces its row, and after the look-back the row is rewritten as exclusive
// prefixes, which the striped store pass reads back beside the items it still holds.
// (Measured on B200, u32 sum scan: a blocked register layout -- thread t owning I consecutive
// items -- ran 2x slower at 1M-30M items: every load / store instruction touched 32 sectors.)
#ifndef B2L_SCAN_I
#define B2L_SCAN_I 0
#endif
template <class T>
__host__ __device__ constexpr int scan_items() {
    return B2L_SCAN_I ? B2L_SCAN_I : (sizeof(T) <= 8 ? 16 : 8);
}
template <class T>
constexpr size_t scan_smem() {
    return (size_t)SCAN_THREADS * (scan_items<T>() + 1) * sizeof(T);
}

#ifdef B2L_SCAN_PROF
__device__ long long g_scan_prof[65536 * 6];
#endif
template <class Op, class Load, class Store>
__global__ void __launch_bounds__(SCAN_THREADS) k_scan_1p(size_t n, Load ld, Store st, typename Op::T *agg,
                                                          typename Op::T *inc, uint32_t *flag, uint32_t *counter,
                                                          typename Op::T *d_total) {
    pdl_enter();
    using T = typename Op::T;
    constexpr int I = scan_items<T>();
    constexpr int TILE = SCAN_THREADS * I;
    extern __shared__ __align__(16) uint8_t scan_sm_raw[];
    T *tr = reinterpret_cast<T *>(scan_sm_raw);  // SCAN_THREADS * (I + 1) slots
    __shared__ T sm[SCAN_THREADS / 32 + 1];
    __shared__ uint32_t tile_s;
    if (threadIdx.x == 0) tile_s = atomicAdd(counter, 1u);
    __syncthreads();
    const uint32_t tile = tile_s;
    const size_t tb = (size_t)tile * TILE;
    const int t = threadIdx.x;
#ifdef B2L_SCAN_PROF
    long long c0 = clock64(), g0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
#endif
    T items[I];
#pragma unroll
    for (int k = 0; k < I; ++k) {
        const size_t i = tb + (size_t)k * SCAN_THREADS + t;
        items[k] = i < n ? ld(i) : Op::identity();
    }
#pragma unroll
    for (int k = 0; k < I; ++k) {
        const int j = k * SCAN_THREADS + t;
        tr[(j / I) * (I + 1) + j % I] = items[k];
    }
    __syncthreads();
    T *row = tr + t * (I + 1);
    T acc = Op::identity();
#pragma unroll
    for (int k = 0; k < I; ++k) acc = Op::combine(acc, row[k]);
    T total;
    T ex = block_excl_scan<Op>(acc, sm, total);
#ifdef B2L_SCAN_PROF
    long long c1 = clock64();
#endif
    const T prefix = block_lookback<Op>(tile, total, agg, inc, flag);
#ifdef B2L_SCAN_PROF
    long long c2 = clock64();
#endif
    if (d_total && t == 0 && tb + TILE >= n) *d_total = Op::combine(prefix, total);
    ex = Op::combine(prefix, ex);
#pragma unroll
    for (int k = 0; k < I; ++k) {  // exclusive prefixes over the own row, in place
        const T it = row[k];
        row[k] = ex;
        ex = Op::combine(ex, it);
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < I; ++k) {
        const int j = k * SCAN_THREADS + t;
        if (tb + j < n) st(tb + j, tr[(j / I) * (I + 1) + j % I], items[k]);
    }
#ifdef B2L_SCAN_PROF
    __syncthreads();
    if (t == 0 && tile < 65536) {
        long long c3 = clock64(), g3;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g3));
        g_scan_prof[tile * 6 + 0] = g0, g_scan_prof[tile * 6 + 1] = c1 - c0, g_scan_prof[tile * 6 + 2] = c2 - c1;
        g_scan_prof[tile * 6 + 3] = c3 - c2, g_scan_prof[tile * 6 + 4] = g3;
        unsigned smid;
        asm("mov.u32 %0, %%smid;" : "=r"(smid));
        g_scan_prof[tile * 6 + 5] = smid;
    }
#endif
}

// scan over n items: st(i, exclusive_prefix, item) for every i; optional device total.
template <class Op, class Load, class Store>
void scan(size_t n, Load ld, Store st, cudaStream_t s, typename Op::T *d_total = nullptr) {
    using T = typename Op::T;
    if (n == 0) {  // only sums are scanned with a device total over possibly-empty ranges
        if (d_total) dev_memset(d_total, 0, sizeof(T), s);
        return;
    }
    constexpr size_t TILE = (size_t)SCAN_THREADS * scan_items<T>();
    const size_t tiles = (n + TILE - 1) / TILE;
    // flags (one per line) + tile counter in one zeroed block; aggregates / inclusive prefixes beside them
    const size_t fwords = (tiles + 1) * FS;
    const size_t tv = (tiles * sizeof(T) + 15) & ~size_t(15);
    DBuf<uint8_t> ws(fwords * 4 + 2 * tv, s);
    uint32_t *flag = t_arena ? static_cast<uint32_t *>(t_arena->take_zeroed(fwords * 4)) : nullptr;
    if (!flag) {  // no zeroed pool left: this scan's own scratch, zeroed
        flag = reinterpret_cast<uint32_t *>(ws.p);
        dev_memset(flag, 0, fwords * 4, s);
    }
    T *agg = reinterpret_cast<T *>(ws.p + fwords * 4), *inc = reinterpret_cast<T *>(ws.p + fwords * 4 + tv);
    constexpr size_t smem = scan_smem<T>();
    if (smem > 48 * 1024) {
        static bool opted = false;  // per instantiation
        if (!opted) {
            CK(cudaFuncSetAttribute(k_scan_1p<Op, Load, Store>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            opted = true;
        }
    }
    launch_k(k_scan_1p<Op, Load, Store>, (unsigned)tiles, SCAN_THREADS, smem, s, n, ld, st, agg, inc, flag,
             flag + tiles * FS, d_total);
    CK_LAUNCH("k_scan_1p");
}

// ---------------------------------------------------------------- pinned readback staging
// A per-thread pinned buffer (grown, never per call): small device->host reads and the result
// arrays go through it, so no call pays cudaMallocHost / pageable-copy costs.
struct Pinned {
    uint8_t *p = nullptr;
    size_t cap = 0;
    uint8_t *reserve(size_t bytes) {
        if (bytes > cap) {
            if (p) cudaFreeHost(p);
            p = nullptr;
            cap = 0;
            size_t c = bytes < (1u << 20) ? (1u << 20) : bytes + bytes / 2;
            CK(cudaMallocHost(&p, c));
            cap = c;
        }
        return p;
    }
};
// One staging buffer per stream (a stream is driven by one host thread at a time), kept for the
// life of the process -- never allocated per call.
inline Pinned &pinned(cudaStream_t s) {
    static std::mutex mu;
    static std::map<cudaStream_t, Pinned> by_stream;
    std::lock_guard<std::mutex> lock(mu);
    return by_stream[s];
}
// Pinned result slabs: findings / sums arrays live in page-locked memory the engine owns and
// recycles (DMA'd straight into place, no malloc + memcpy; the Python side wraps them zero-copy).
struct SlabPool {
    std::mutex mu;
    std::multimap<size_t, uint8_t *> free_;
    uint8_t *acquire(size_t bytes, size_t &cap) {
        bytes = bytes < 4096 ? 4096 : bytes;
        {
            std::lock_guard<std::mutex> lock(mu);
            auto it = free_.lower_bound(bytes);
            if (it != free_.end() && it->first <= 4 * bytes) {
                cap = it->first;
                uint8_t *p = it->second;
                free_.erase(it);
                return p;
            }
        }
        size_t c = 4096;
        while (c < bytes) c <<= 1;
        uint8_t *p = nullptr;
        CK(cudaMallocHost(&p, c));
        cap = c;
        return p;
    }
    void release(uint8_t *p, size_t cap) {
        if (!p) return;
        std::lock_guard<std::mutex> lock(mu);
        free_.emplace(cap, p);
    }
};
inline SlabPool &slab_pool() {
    static SlabPool pool;
    return pool;
}

// Device->host reads go through the copy engine of that direction (it stays free while the
// other direction carries analyze_many's next upload; a kernel storing into mapped host memory
// would instead wait on the busy PCIe link for its write acknowledgements).
inline void to_host_async(void *h_pinned, const void *d_src, size_t bytes, cudaStream_t s) {
    if (bytes) CK(cudaMemcpyAsync(h_pinned, d_src, bytes, cudaMemcpyDeviceToHost, s));
}
// Small read-backs (the "how many?" counts that size the next step) of calls up to ~16M events
// (their arena says so; huge calls overlap many-MB result copies, behind which the mailbox
// kernel's host writes wait) go through a per-stream
// MAILBOX in mapped pinned memory: one tiny kernel copies the value there and then bumps a tag
// (__threadfence_system in between), the host spins on the tag.  A D2H copy + stream
// synchronisation costs ~23 us per round trip and ~60 us while a host->device upload shares the
// PCIe link (analyze_many uploads the next trace beside the current analysis); the mailbox costs
// ~8 / ~36 us (tools/pipe_exp4.py).  The tag lands after every earlier operation of the stream,
// so the read is also a stream barrier.  While spinning, cudaStreamQuery surfaces faults.
constexpr size_t MAILBOX_BYTES = 256;
struct Mailbox {
    uint8_t *host = nullptr;  // [0, 4): tag; [64, 64 + MAILBOX_BYTES): payload (mapped, UVA)
    uint32_t seq = 0;
};
inline Mailbox &mailbox(cudaStream_t s) {
    static std::mutex mu;
    static std::map<cudaStream_t, Mailbox> by_stream;
    std::lock_guard<std::mutex> lock(mu);
    Mailbox &m = by_stream[s];
    if (!m.host) {
        CK(cudaHostAlloc((void **)&m.host, 64 + MAILBOX_BYTES, cudaHostAllocMapped | cudaHostAllocPortable));
        memset(m.host, 0, 64 + MAILBOX_BYTES);
    }
    return m;
}
static __global__ void k_mailbox(const uint8_t *__restrict__ src, uint32_t bytes, uint8_t *box, uint32_t tag) {
    pdl_enter();
    for (uint32_t i = threadIdx.x; i < bytes; i += blockDim.x) box[64 + i] = src[i];
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence_system();
        *reinterpret_cast<volatile uint32_t *>(box) = tag;
    }
}
inline bool mailbox_on() {
    static const bool on = !getenv("B2L_NO_MAILBOX");
    return on;
}
// Spin on the tag without touching the driver (a cudaStreamQuery takes the driver lock the
// other chains' launches need); after ~200 us of waiting, fall back to a blocking stream sync,
// which also surfaces a fault (a faulted stream never delivers the tag).
inline void mailbox_wait(Mailbox &m, uint32_t tag, cudaStream_t s) {
    const volatile uint32_t *t = reinterpret_cast<volatile uint32_t *>(m.host);
    if (*t != tag) {
        const auto t0 = std::chrono::steady_clock::now();
        for (uint32_t spin = 1; *t != tag; ++spin) {
            if ((spin & 255u) == 0 && std::chrono::steady_clock::now() - t0 > std::chrono::microseconds(200)) {
                CK(cudaStreamSynchronize(s));  // long wait: block (the tag landed with the stream's work)
                while (*t != tag) {
                }
                break;
            }
        }
    }
    std::atomic_thread_fence(std::memory_order_acquire);
}
// Read `bytes` from device memory into host `dst` (synchronous).
inline void read_back(void *dst, const void *d_src, size_t bytes, cudaStream_t s, int line = __builtin_LINE()) {
    SyncTimer st_(line);
    if (bytes <= MAILBOX_BYTES && mailbox_on() && t_arena && t_arena->mailbox) {
        Mailbox &m = mailbox(s);
        const uint32_t tag = ++m.seq ? m.seq : ++m.seq;
        launch_k(k_mailbox, 1, 64, 0, s, static_cast<const uint8_t *>(d_src), (uint32_t)bytes, m.host, tag);
        CK(cudaGetLastError());
        mailbox_wait(m, tag, s);
        memcpy(dst, m.host + 64, bytes);
        return;
    }
    uint8_t *st = pinned(s).reserve(bytes);
    to_host_async(st, d_src, bytes, s);
    CK(cudaStreamSynchronize(s));
    memcpy(dst, st, bytes);
}
// Several small device values in one mailbox trip (up to 8 pieces, MAILBOX_BYTES in total).
struct ReadPiece {
    void *dst;
    const void *src;
    size_t bytes;
};
struct MailboxPieces {
    const uint8_t *src[8];
    uint32_t bytes[8];
    uint32_t n;
};
static __global__ void k_mailbox_multi(MailboxPieces p, uint8_t *box, uint32_t tag) {
    pdl_enter();
    uint32_t off = 0;
    for (uint32_t k = 0; k < p.n; ++k) {
        for (uint32_t i = threadIdx.x; i < p.bytes[k]; i += blockDim.x) box[64 + off + i] = p.src[k][i];
        off += p.bytes[k];
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence_system();
        *reinterpret_cast<volatile uint32_t *>(box) = tag;
    }
}
inline void read_back_multi(std::initializer_list<ReadPiece> pieces, cudaStream_t s, int line = __builtin_LINE()) {
    SyncTimer st_(line);
    size_t total = 0;
    for (const ReadPiece &q : pieces) total += q.bytes;
    if (!mailbox_on() || !t_arena || !t_arena->mailbox || pieces.size() > 8 || total > MAILBOX_BYTES) {
        uint8_t *st = pinned(s).reserve(total);
        size_t off = 0;
        for (const ReadPiece &q : pieces) to_host_async(st + off, q.src, q.bytes, s), off += q.bytes;
        CK(cudaStreamSynchronize(s));
        off = 0;
        for (const ReadPiece &q : pieces) memcpy(q.dst, st + off, q.bytes), off += q.bytes;
        return;
    }
    MailboxPieces mp{};
    for (const ReadPiece &q : pieces) mp.src[mp.n] = static_cast<const uint8_t *>(q.src), mp.bytes[mp.n++] = (uint32_t)q.bytes;
    Mailbox &m = mailbox(s);
    const uint32_t tag = ++m.seq ? m.seq : ++m.seq;
    launch_k(k_mailbox_multi, 1, 64, 0, s, mp, m.host, tag);
    CK(cudaGetLastError());
    mailbox_wait(m, tag, s);
    size_t off = 0;
    for (const ReadPiece &q : pieces) memcpy(q.dst, m.host + 64 + off, q.bytes), off += q.bytes;
}
// Wait until everything queued on `s` has run.  (Not through the mailbox: these waits follow
// large result copies, and a kernel writing into mapped host memory behind a device->host copy
// stream waits for that link -- at 100M events the chains slowed from 47 to 110 ms.)
inline void stream_wait(cudaStream_t s, int line = __builtin_LINE()) {
    SyncTimer st_(line);
    CK(cudaStreamSynchronize(s));
}

// ---------------------------------------------------------------- compaction
template <class Pred>
struct FlagLoad {
    Pred p;
    __device__ __forceinline__ uint32_t operator()(size_t i) const { return p(i) ? 1u : 0u; }
};
template <class Pred>
struct CompactStore {
    Pred p;
    uint32_t *out;
    __device__ __forceinline__ void operator()(size_t i, uint32_t ex, uint32_t item) const {
        if (item) out[ex] = (uint32_t)i;
    }
};
// Indices i in [0,n) with pred(i), ascending, into out (capacity n).  Count -> *d_count (device, u32).
template <class Pred>
void compact(size_t n, Pred pred, uint32_t *out, uint32_t *d_count, cudaStream_t s) {
    if (n == 0) {
        dev_memset(d_count, 0, sizeof(uint32_t), s);
        return;
    }
    scan<SumU32>(n, FlagLoad<Pred>{pred}, CompactStore<Pred>{pred, out}, s, d_count);
}

// ---------------------------------------------------------------- simple functors
struct LoadU32 {
    const uint32_t *c;
    __device__ __forceinline__ uint32_t operator()(size_t i) const { return c[i]; }
};
struct StoreExclU32 {
    uint32_t *c;
    __device__ __forceinline__ void operator()(size_t i, uint32_t ex, uint32_t) const { c[i] = ex; }
};

// ---------------------------------------------------------------- radix sort
constexpr int RS_THREADS = 256;

template <int KW>
struct KeyCols {
    uint64_t *w[KW];  // w[0] = most significant word
};

__device__ __forceinline__ uint32_t lanemask_lt() {
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// Histograms of every digit position of every key word in one read of the keys:
// hist[(w * 8 + byte) * 256 + digit].  Warp-aggregated (match_any) shared-memory counts.
template <int KW>
struct LiveBytes {
    uint8_t m[KW];  // bit b set: byte b of word w may differ between keys
};

template <int KW>
__global__ void __launch_bounds__(RS_THREADS) k_radix_hist_all(KeyCols<KW> k, size_t n, LiveBytes<KW> live,
                                                               uint32_t *__restrict__ hist) {
    pdl_enter();
    __shared__ uint32_t sh[KW * 8][256];
    for (int i = threadIdx.x; i < KW * 8 * 256; i += RS_THREADS) (&sh[0][0])[i] = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    constexpr int U = 4;  // keys per thread per step (loads issued together)
    const size_t stride = (size_t)gridDim.x * RS_THREADS * U;
    for (size_t base = (size_t)blockIdx.x * RS_THREADS * U; base < n; base += stride) {
#pragma unroll
        for (int w = 0; w < KW; ++w) {
            if (!live.m[w]) continue;
            uint64_t key[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const size_t i = base + (size_t)u * RS_THREADS + threadIdx.x;
                key[u] = i < n ? k.w[w][i] : 0;
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const bool valid = base + (size_t)u * RS_THREADS + threadIdx.x < n;
#pragma unroll
                for (int b = 0; b < 8; ++b) {
                    if (!((live.m[w] >> b) & 1)) continue;
                    const uint32_t d = (uint32_t)(key[u] >> (8 * b)) & 255u;
                    // a digit shared by the whole warp (skewed or sorted keys) is one add of 32
                    const uint32_t d0 = __shfl_sync(0xffffffffu, d, 0);
                    if (__all_sync(0xffffffffu, valid && d == d0)) {
                        if (lane == 0) atomicAdd(&sh[w * 8 + b][d0], 32u);
                    } else if (valid) {
                        atomicAdd(&sh[w * 8 + b][d], 1u);
                    }
                }
            }
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < KW * 8 * 256; i += RS_THREADS) {
        const uint32_t v = (&sh[0][0])[i];
        if (v) atomicAdd(hist + i, v);
    }
}

// One LSD pass, Onesweep style: tiles take ids in launch order, rank their keys stably
// (warp multisplit), publish per-digit tile counts, and resolve the exclusive prefix of
// every digit across preceding tiles by decoupled look-back -- one launch per pass.
// The tile is then reordered by digit in shared memory and written out run by run, so
// each warp store covers consecutive addresses of one digit's output range (coalesced),
// one key word at a time through a 32 KB staging buffer.
constexpr uint32_t LB_AGG = 1u << 30, LB_INC = 2u << 30, LB_VAL = (1u << 30) - 1;
constexpr int OS_THREADS = 256;
constexpr int OS_WARPS = OS_THREADS / 32;
constexpr int OS_ITEMS = 16;
constexpr int OS_TILE = OS_THREADS * OS_ITEMS;  // 4096 records per tile

// Exclusive scan of one u32 per thread across a 256-thread block (warp shuffles + one
// cross-warp step).  `wsum` is OS_WARPS words of shared scratch.  Returns the block total.
__device__ __forceinline__ uint32_t block256_excl(uint32_t v, uint32_t *wsum, uint32_t &total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) wsum[warp] = x;
    __syncthreads();
    uint32_t before = 0, tot = 0;
#pragma unroll
    for (int w = 0; w < OS_WARPS; ++w) {
        const uint32_t c = wsum[w];
        before += w < warp ? c : 0u;
        tot += c;
    }
    total = tot;
    return before + x - v;
}

template <int KW, int ITEMS>
__global__ void __launch_bounds__(OS_THREADS, 3) k_onesweep(KeyCols<KW> in, const uint32_t *__restrict__ vin,
                                                         KeyCols<KW> out, uint32_t *__restrict__ vout, size_t n,
                                                         int word, int shift, const uint32_t *__restrict__ hist,
                                                         uint32_t *status, uint32_t *tile_counter) {
    pdl_enter();
    __shared__ uint32_t tile_s;
    __shared__ uint32_t wsum[2][OS_WARPS];
    __shared__ uint32_t wcnt[OS_WARPS][256];  // per-warp digit counts -> tile positions of each warp's run
    __shared__ uint32_t gofs[256];            // output index of tile position j of digit d = gofs[d] + j
    __shared__ uint8_t sdig[(OS_THREADS * ITEMS)];         // digit of tile position j
    __shared__ uint64_t stage[(OS_THREADS * ITEMS)];
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    if (t == 0) tile_s = atomicAdd(tile_counter, 1u);
#pragma unroll
    for (int w = 0; w < OS_WARPS; ++w) wcnt[w][t] = 0;
    __syncthreads();
    const uint32_t tile = tile_s;
    const size_t tbase = (size_t)tile * (OS_THREADS * ITEMS);
    const size_t wbase = tbase + (size_t)warp * (32 * ITEMS) + lane;
    const uint64_t *kd = in.w[word];

    // ---- load the digit word (warp-striped: item i of lane l is wbase + 32 i) and rank per warp
    uint64_t key[ITEMS];
    uint32_t slot[ITEMS];  // (digit << 16) | rank within this warp's run of the digit; ~0 = past n
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
        const size_t pos = wbase + 32 * i;
        key[i] = pos < n ? kd[pos] : 0;
    }
    const uint32_t lt = lanemask_lt();
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
        const bool valid = wbase + 32 * i < n;
        const uint32_t d = valid ? (uint32_t)(key[i] >> shift) & 255u : 256u;
        const uint32_t peers = __match_any_sync(0xffffffffu, d);
        const uint32_t before = valid ? wcnt[warp][d] : 0u;
        __syncwarp();
        if (valid && lane == 31 - __clz(peers)) wcnt[warp][d] = before + __popc(peers);
        __syncwarp();
        slot[i] = valid ? ((d << 16) | (before + __popc(peers & lt))) : 0xFFFFFFFFu;
    }
    __syncthreads();
    // ---- digit t: counts per warp -> exclusive offsets across warps; tile total
    uint32_t cnt = 0;
#pragma unroll
    for (int w = 0; w < OS_WARPS; ++w) {
        const uint32_t c = wcnt[w][t];
        wcnt[w][t] = cnt;
        cnt += c;
    }
    volatile uint32_t *st = status;
    if (tile != 0) st[(size_t)tile * 256 + t] = LB_AGG | cnt;  // publish the aggregate early
    uint32_t tot;
    const uint32_t tstart = block256_excl(cnt, wsum[0], tot);  // tile position of digit t's run
    const uint32_t h = hist[t];
    const uint32_t dbase = block256_excl(h, wsum[1], tot) ;    // global start of digit t
    // ---- decoupled look-back for digit t
    uint32_t excl = 0;
    if (tile == 0) {
        st[t] = LB_INC | cnt;
    } else {
        // walk back over predecessors 4 at a time (independent loads), in order
        bool done = false;
        for (int64_t j = (int64_t)tile - 1; !done; j -= 4) {
            uint32_t v[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) v[u] = j - u >= 0 ? st[(size_t)(j - u) * 256 + t] : (uint32_t)LB_INC;
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                if (done) break;
                while ((v[u] & (LB_AGG | LB_INC)) == 0) v[u] = st[(size_t)(j - u) * 256 + t];
                excl += v[u] & LB_VAL;
                done = (v[u] & LB_INC) != 0;
            }
        }
        st[(size_t)tile * 256 + t] = LB_INC | (excl + cnt);
    }
    gofs[t] = dbase + excl - tstart;
#pragma unroll
    for (int w = 0; w < OS_WARPS; ++w) wcnt[w][t] += tstart;
    __syncthreads();
    // ---- tile positions; digit of each position
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
        if (slot[i] == 0xFFFFFFFFu) continue;
        const uint32_t d = slot[i] >> 16;
        const uint32_t p = wcnt[warp][d] + (slot[i] & 0xFFFFu);
        slot[i] = p;
        sdig[p] = (uint8_t)d;
        stage[p] = key[i];
    }
    __syncthreads();
    const uint32_t tn = (uint32_t)(n - tbase < (size_t)(OS_THREADS * ITEMS) ? n - tbase : (size_t)(OS_THREADS * ITEMS));
    {
        uint64_t *o = out.w[word];
        for (uint32_t j = t; j < tn; j += OS_THREADS) o[gofs[sdig[j]] + j] = stage[j];
    }
    // ---- the other key words and the value, through the same staging buffer
#pragma unroll
    for (int w = 0; w < KW; ++w) {
        if (w == word) continue;
        const uint64_t *src = in.w[w];
#pragma unroll
        for (int i = 0; i < ITEMS; ++i) key[i] = slot[i] != 0xFFFFFFFFu ? src[wbase + 32 * i] : 0;
        __syncthreads();
#pragma unroll
        for (int i = 0; i < ITEMS; ++i)
            if (slot[i] != 0xFFFFFFFFu) stage[slot[i]] = key[i];
        __syncthreads();
        uint64_t *o = out.w[w];
        for (uint32_t j = t; j < tn; j += OS_THREADS) o[gofs[sdig[j]] + j] = stage[j];
    }
    {
        uint32_t vv[ITEMS];
#pragma unroll
        for (int i = 0; i < ITEMS; ++i) vv[i] = slot[i] != 0xFFFFFFFFu ? vin[wbase + 32 * i] : 0u;
        uint32_t *st32 = reinterpret_cast<uint32_t *>(stage);
        __syncthreads();
#pragma unroll
        for (int i = 0; i < ITEMS; ++i)
            if (slot[i] != 0xFFFFFFFFu) st32[slot[i]] = vv[i];
        __syncthreads();
        for (uint32_t j = t; j < tn; j += OS_THREADS) vout[gofs[sdig[j]] + j] = st32[j];
    }
}

// Sorts that fit one tile (<= ST_TILE records): every live digit pass in ONE CTA, the records
// in shared memory between passes (the same warp-multisplit ranking as a Onesweep pass, without
// the global histogram and look-back) -- one launch instead of a histogram + a pass per digit.
// A small trace's analysis makes ~10 such sorts, each otherwise 3-5 launches.
constexpr int ST_THREADS = 256, ST_ITEMS = 16, ST_TILE = ST_THREADS * ST_ITEMS;
template <int KW>
constexpr size_t sort_tile_smem() {
    return (size_t)KW * ST_TILE * 8 + (size_t)ST_TILE * 4;
}
template <int KW>
__global__ void __launch_bounds__(ST_THREADS) k_sort_tile(KeyCols<KW> in, const uint32_t *__restrict__ vin,
                                                           KeyCols<KW> out, uint32_t *__restrict__ vout, uint32_t n,
                                                           LiveBytes<KW> live) {
    pdl_enter();
    extern __shared__ __align__(16) uint8_t st_raw[];
    uint64_t *sk = reinterpret_cast<uint64_t *>(st_raw);                         // [KW][ST_TILE]
    uint32_t *sv = reinterpret_cast<uint32_t *>(st_raw + (size_t)KW * ST_TILE * 8);  // [ST_TILE]
    __shared__ uint32_t wsum[OS_WARPS];
    __shared__ uint32_t wcnt[OS_WARPS][256];
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    for (uint32_t j = t; j < n; j += ST_THREADS) {
#pragma unroll
        for (int w = 0; w < KW; ++w) sk[(size_t)w * ST_TILE + j] = in.w[w][j];
        sv[j] = vin[j];
    }
    __syncthreads();
    const uint32_t wbase = (uint32_t)warp * (32 * ST_ITEMS) + lane;  // item i of lane l: wbase + 32 i
    for (int w = KW - 1; w >= 0; --w) {
        for (int byte = 0; byte < 8; ++byte) {
            if (!((live.m[w] >> byte) & 1)) continue;
            const int shift = 8 * byte;
#pragma unroll
            for (int ww = 0; ww < OS_WARPS; ++ww) wcnt[ww][t] = 0;
            __syncthreads();
            uint32_t slot[ST_ITEMS];
            const uint32_t lt = lanemask_lt();
#pragma unroll
            for (int i = 0; i < ST_ITEMS; ++i) {
                const uint32_t pos = wbase + 32 * i;
                const bool valid = pos < n;
                const uint32_t d = valid ? (uint32_t)(sk[(size_t)w * ST_TILE + pos] >> shift) & 255u : 256u;
                const uint32_t peers = __match_any_sync(0xffffffffu, d);
                const uint32_t before = valid ? wcnt[warp][d] : 0u;
                __syncwarp();
                if (valid && lane == 31 - __clz(peers)) wcnt[warp][d] = before + __popc(peers);
                __syncwarp();
                slot[i] = valid ? ((d << 16) | (before + __popc(peers & lt))) : 0xFFFFFFFFu;
            }
            __syncthreads();
            uint32_t cnt = 0;  // digit t: counts per warp -> exclusive offsets across warps
#pragma unroll
            for (int ww = 0; ww < OS_WARPS; ++ww) {
                const uint32_t c = wcnt[ww][t];
                wcnt[ww][t] = cnt;
                cnt += c;
            }
            uint32_t tot;
            const uint32_t dstart = block256_excl(cnt, wsum, tot);
#pragma unroll
            for (int ww = 0; ww < OS_WARPS; ++ww) wcnt[ww][t] += dstart;
            __syncthreads();
#pragma unroll
            for (int i = 0; i < ST_ITEMS; ++i)
                if (slot[i] != 0xFFFFFFFFu) slot[i] = wcnt[warp][slot[i] >> 16] + (slot[i] & 0xFFFFu);
            // permute every key word and the value in place: load all, barrier, store all
#pragma unroll
            for (int kw = 0; kw < KW; ++kw) {
                uint64_t v[ST_ITEMS];
#pragma unroll
                for (int i = 0; i < ST_ITEMS; ++i) v[i] = slot[i] != 0xFFFFFFFFu ? sk[(size_t)kw * ST_TILE + wbase + 32 * i] : 0;
                __syncthreads();
#pragma unroll
                for (int i = 0; i < ST_ITEMS; ++i)
                    if (slot[i] != 0xFFFFFFFFu) sk[(size_t)kw * ST_TILE + slot[i]] = v[i];
                __syncthreads();
            }
            {
                uint32_t v[ST_ITEMS];
#pragma unroll
                for (int i = 0; i < ST_ITEMS; ++i) v[i] = slot[i] != 0xFFFFFFFFu ? sv[wbase + 32 * i] : 0u;
                __syncthreads();
#pragma unroll
                for (int i = 0; i < ST_ITEMS; ++i)
                    if (slot[i] != 0xFFFFFFFFu) sv[slot[i]] = v[i];
                __syncthreads();
            }
        }
    }
    for (uint32_t j = t; j < n; j += ST_THREADS) {
#pragma unroll
        for (int w = 0; w < KW; ++w) out.w[w][j] = sk[(size_t)w * ST_TILE + j];
        vout[j] = sv[j];
    }
}

inline bool sort_tiles_on() {
    static const bool on = !getenv("B2L_NO_SORT_TILE");
    return on;
}
template <int KW>
struct SortBufs {
    KeyCols<KW> k[2];
    uint32_t *v[2];
    int cur = 0;  // which side holds the data
};

// Stable sort of n records (keys KW words, value u32) held in side `b.cur`; on return b.cur names
// the side holding the sorted records.  `live` names the key bytes that may vary (callers derive it
// from column-wide OR-of-XOR masks and known value ranges), so there is no host round trip: one
// histogram read of the keys, then one Onesweep launch per live digit position.
template <int KW>
void radix_sort(SortBufs<KW> &b, size_t n, LiveBytes<KW> live, cudaStream_t s) {
    if (n <= 1) return;
    if (n >= (size_t)LB_VAL) throw EngineErr{B2L_E_INVALID_ARG, "radix_sort: too many records"};
    int npass = 0;
    for (int w = 0; w < KW; ++w) npass += __builtin_popcount(live.m[w]);
    if (npass == 0) return;
    if (n <= (size_t)ST_TILE && sort_tiles_on()) {  // one CTA, every pass in shared memory
        constexpr size_t smem = sort_tile_smem<KW>();
        static bool opted = false;  // per instantiation
        if (!opted) {
            CK(cudaFuncSetAttribute(k_sort_tile<KW>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            opted = true;
        }
        launch_k(k_sort_tile<KW>, 1, ST_THREADS, smem, s, b.k[b.cur], (const uint32_t *)b.v[b.cur], b.k[b.cur ^ 1],
                 b.v[b.cur ^ 1], (uint32_t)n, live);
        CK_LAUNCH("k_sort_tile");
        b.cur ^= 1;
        return;
    }
    constexpr int NPOS = KW * 8;
    DBuf<uint32_t> hist_own;
    uint32_t *hist_p = t_arena ? static_cast<uint32_t *>(t_arena->take_zeroed((size_t)NPOS * 256 * 4)) : nullptr;
    if (!hist_p) {
        hist_own.alloc((size_t)NPOS * 256, s);
        hist_own.zero();
        hist_p = hist_own.p;
    }
    struct {
        uint32_t *p;
    } hist{hist_p};
    launch_k(k_radix_hist_all<KW>, grid_for(n, RS_THREADS * 4, 148 * 4), RS_THREADS, 0, s, b.k[b.cur], n, live, hist.p);
    CK_LAUNCH("k_radix_hist_all");
    // sorts under ~1.2M records use 1024-record tiles: four times the CTAs, so a pass is not a few
    // long tiles on part of the GPU
    const bool small = n < (size_t)OS_TILE * 296;  // fewer than two big tiles per SM
    const size_t tile = small ? (size_t)OS_THREADS * 4 : (size_t)OS_TILE;
    const unsigned ntiles = (unsigned)((n + tile - 1) / tile);
    const size_t stride = (size_t)ntiles * 256 + 32;  // status words + tile counter per pass
    DBuf<uint32_t> status_own;
    uint32_t *status_p = t_arena ? static_cast<uint32_t *>(t_arena->take_zeroed(stride * npass * 4)) : nullptr;
    if (!status_p) {
        status_own.alloc(stride * npass, s);
        status_own.zero();
        status_p = status_own.p;
    }
    struct {
        uint32_t *p;
    } status{status_p};
    int p = 0;
    for (int w = KW - 1; w >= 0; --w) {
        for (int byte = 0; byte < 8; ++byte) {
            if (!((live.m[w] >> byte) & 1)) continue;
            uint32_t *stp = status.p + stride * p++;
            if (small)
                launch_k(k_onesweep<KW, 4>, ntiles, OS_THREADS, 0, s, b.k[b.cur], (const uint32_t *)b.v[b.cur],
                         b.k[b.cur ^ 1], b.v[b.cur ^ 1], n, w, 8 * byte,
                         (const uint32_t *)(hist.p + (size_t)(w * 8 + byte) * 256), stp, stp + (size_t)ntiles * 256);
            else
                launch_k(k_onesweep<KW, OS_ITEMS>, ntiles, OS_THREADS, 0, s, b.k[b.cur], (const uint32_t *)b.v[b.cur],
                         b.k[b.cur ^ 1], b.v[b.cur ^ 1], n, w, 8 * byte,
                         (const uint32_t *)(hist.p + (size_t)(w * 8 + byte) * 256), stp, stp + (size_t)ntiles * 256);
            CK_LAUNCH("k_onesweep");
            b.cur ^= 1;
        }
    }
}

// Live-byte mask of a value range [0, v): the low bytes needed to represent v - 1.
inline uint8_t live_range(uint64_t v) {
    if (v <= 1) return 0;
    uint64_t x = v - 1;
    uint8_t m = 0;
    for (int b = 0; b < 8 && x; ++b, x >>= 8) m |= (uint8_t)(1u << b);
    return m;
}
// Live-byte mask from an OR-of-XOR column mask.
inline uint8_t live_mask(uint64_t vary) {
    uint8_t m = 0;
    for (int b = 0; b < 8; ++b)
        if ((vary >> (8 * b)) & 255ull) m |= (uint8_t)(1u << b);
    return m;
}

static __global__ void k_gather_kv(const uint32_t *__restrict__ P, size_t m, const uint64_t *__restrict__ k,
                            const uint32_t *__restrict__ v, uint64_t *__restrict__ ko, uint32_t *__restrict__ vo) {
    pdl_enter();
    for (size_t j = (size_t)blockIdx.x * blockDim.x + threadIdx.x; j < m; j += (size_t)gridDim.x * blockDim.x)
        ko[j] = k[P[j]], vo[j] = v[P[j]];
}
static __global__ void k_scatter_kv(const uint32_t *__restrict__ P, size_t m, const uint64_t *__restrict__ k,
                             const uint32_t *__restrict__ v, uint64_t *__restrict__ ko, uint32_t *__restrict__ vo) {
    pdl_enter();
    for (size_t j = (size_t)blockIdx.x * blockDim.x + threadIdx.x; j < m; j += (size_t)gridDim.x * blockDim.x)
        ko[P[j]] = k[j], vo[P[j]] = v[j];
}
// ---------------------------------------------------------------- segmented fix-up sort
// Records (u64 key, u32 value) already stably ordered by the key's prefix (key >> shift) become
// stably ordered by the full key in one pass: every run of equal prefixes of length <= FIX_T is
// ranked in place by each of its members (reads of the run only); longer runs are flagged and
// sorted afterwards by a full-key LSD sort of just their records.  Used where random keys have
// few records per prefix: the hash sort needs LSD passes over ~log2(n)+1 prefix bits instead of
// all 64, and records generated in hash-rank order need no LSD pass at all.
constexpr uint32_t FIX_T = 32;

constexpr int FX_THREADS = 256, FX_ITEMS = 8, FX_TILE = FX_THREADS * FX_ITEMS;
constexpr int FX_WIN = FX_TILE + 2 * FIX_T;   // tile plus halo, positions relative to lo
constexpr int FX_HW = FX_WIN / 32 + 2;        // head-bit words (+ end sentinel)
// One tile of positions plus a FIX_T halo on each side in shared memory, with a bitmask of run
// heads: each record finds its run [a, b) with two bit scans (no walking); runs longer than FIX_T
// are left in place and flagged, shorter ones are ranked from shared memory.
static __global__ void __launch_bounds__(FX_THREADS) k_seg_fixup(const uint64_t *__restrict__ kin,
                                                                 const uint32_t *__restrict__ vin,
                                                                 uint64_t *__restrict__ kout,
                                                                 uint32_t *__restrict__ vout, size_t n, int shift,
                                                                 uint8_t *__restrict__ big, uint32_t *big_count) {
    pdl_enter();
    __shared__ uint64_t sk[FX_WIN];
    __shared__ uint32_t hb[FX_HW];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const size_t t0 = (size_t)blockIdx.x * FX_TILE;
    const size_t lo = t0 >= FIX_T ? t0 - FIX_T : 0;
    const size_t hi = t0 + FX_TILE + FIX_T < n ? t0 + FX_TILE + FIX_T : n;
    const int wn = (int)(hi - lo);
    for (int j = threadIdx.x; j < wn; j += FX_THREADS) sk[j] = kin[lo + j];
    for (int j = threadIdx.x; j < FX_HW; j += FX_THREADS) hb[j] = 0;
    __syncthreads();
    // head bits: position lo + j starts a run (global position 0 always does; n is a sentinel)
    for (int w0 = warp * 32; w0 < wn + 1; w0 += FX_THREADS) {
        const int j = w0 + lane;
        bool h = false;
        if (j < wn) h = (lo + j == 0) || (j > 0 && (sk[j] >> shift) != (sk[j - 1] >> shift));
        else if (j == wn) h = hi == n;  // end of the keys: a run boundary
        const uint32_t m = __ballot_sync(0xffffffffu, h);
        if (lane == 0) hb[w0 >> 5] |= m;
    }
    __syncthreads();
    // position lo + j, j = 0, is a head when j == 0 would need the key before lo: compare it
    if (threadIdx.x == 0 && lo > 0 && (kin[lo - 1] >> shift) != (sk[0] >> shift)) hb[0] |= 1u;
    __syncthreads();
    uint32_t nbig = 0, nbreak = 0;
#pragma unroll 1
    for (int it = 0; it < FX_ITEMS; ++it) {
        const size_t i = t0 + (size_t)it * FX_THREADS + threadIdx.x;
        if (i >= n) break;
        const int rel = (int)(i - lo);
        // a = last head <= rel, searched in the word of rel and the one before
        int a = -1;
        {
            const int wi = rel >> 5, bi = rel & 31;
            const uint32_t m0 = hb[wi] & (bi == 31 ? 0xffffffffu : ((2u << bi) - 1u));
            if (m0) a = wi * 32 + 31 - __clz(m0);
            else if (wi > 0 && hb[wi - 1]) a = (wi - 1) * 32 + 31 - __clz(hb[wi - 1]);
        }
        // b = first head > rel, searched in the word of rel and the one after
        int b = -1;
        {
            const int wi = rel >> 5, bi = rel & 31;
            const uint32_t m0 = bi == 31 ? 0u : (hb[wi] & ~((2u << bi) - 1u));
            if (m0) b = wi * 32 + __ffs(m0) - 1;
            else if (wi + 1 < FX_HW && hb[wi + 1]) b = (wi + 1) * 32 + __ffs(hb[wi + 1]) - 1;
        }
        const bool isbig = a < 0 || b < 0 || b - a > (int)FIX_T;
        big[i] = isbig;
        const uint64_t key = sk[rel];
        if (isbig) {  // stays in place unless its run holds distinct keys (fixed up afterwards)
            ++nbig;
            // a break: same run as its predecessor (not a head), different full key
            if (i > 0 && !((hb[rel >> 5] >> (rel & 31)) & 1u) && (rel > 0 ? sk[rel - 1] : kin[i - 1]) != key) ++nbreak;
            kout[i] = key;
            vout[i] = vin[i];
            continue;
        }
        uint32_t rank = 0;
        for (int j = a; j < b; ++j) {
            const uint64_t kj = sk[j];
            rank += (kj < key || (kj == key && j < rel)) ? 1u : 0u;
        }
        kout[lo + a + rank] = key;
        vout[lo + a + rank] = vin[i];
    }
    if (nbig) atomicAdd(big_count, nbig);
    if (nbreak) atomicAdd(big_count + 1, nbreak);
}
static __global__ void k_compose_idx(const uint32_t *__restrict__ P, const uint32_t *__restrict__ S, size_t m,
                                     uint32_t *__restrict__ out) {
    pdl_enter();
    for (size_t j = (size_t)blockIdx.x * blockDim.x + threadIdx.x; j < m; j += (size_t)gridDim.x * blockDim.x)
        out[j] = P[S[j]];
}
// Over the long-run positions P (ascending): a run starts where positions jump or the prefix changes.
struct RunHeadLoad {
    const uint32_t *P;
    const uint64_t *k;
    int shift;
    __device__ uint32_t operator()(size_t j) const {
        return (j == 0 || P[j - 1] + 1 != P[j] || (k[P[j - 1]] >> shift) != (k[P[j]] >> shift)) ? 1u : 0u;
    }
};
struct RunIdStore {  // run id per long-run record; flag runs whose neighbours differ in the full key
    const uint32_t *P;
    const uint64_t *k;
    uint32_t *rid, *rflag;
    __device__ void operator()(size_t j, uint32_t ex, uint32_t it) const {
        const uint32_t r = ex + it - 1;
        rid[j] = r;
        if (!it && k[P[j - 1]] != k[P[j]]) rflag[r] = 1;
    }
};
struct RunFlagged {
    const uint32_t *rid, *rflag;
    __device__ bool operator()(size_t j) const { return rflag[rid[j]] != 0; }
};
struct BigPred {
    const uint8_t *big;
    __device__ bool operator()(size_t i) const { return big[i] != 0; }
};

// b.cur holds records ordered by key >> shift; on return b.cur holds them ordered by the full key.
// `live` = the key bytes that may vary (for the long-run fallback).
inline void seg_fixup(SortBufs<1> &b, size_t n, int shift, uint8_t live, cudaStream_t s) {
    if (n <= 1) return;
    DBuf<uint8_t> big(n, s);
    DBuf<uint32_t> cnt;  // [records in long runs, breaks inside long runs]
    cnt.alloc_zeroed(2, s);
    const uint64_t *kin = b.k[b.cur].w[0];
    const uint32_t *vin = b.v[b.cur];
    uint64_t *kout = b.k[b.cur ^ 1].w[0];
    uint32_t *vout = b.v[b.cur ^ 1];
    launch_k(k_seg_fixup, (unsigned)((n + FX_TILE - 1) / FX_TILE), FX_THREADS, 0, s, kin, vin, kout, vout, n, shift, big.p,
                                                                            cnt.p);
    CK_LAUNCH("k_seg_fixup");
    b.cur ^= 1;
    uint32_t nc[2] = {0, 0};
    read_back(nc, cnt.p, sizeof(nc), s);
    const uint32_t nbig = nc[0];
    if (!nbig || !nc[1]) return;  // no long run holds two distinct keys: all in order already
    // long runs: those holding one key repeated are already in order; the others (a "break": equal
    // prefix, different key, between neighbours) are gathered, full-key sorted, scattered back
    DBuf<uint32_t> pos(nbig, s), pc(1, s);
    compact(n, BigPred{big.p}, pos.p, pc.p, s);
    DBuf<uint32_t> rid(nbig, s), rflag, sel(nbig, s), nsel(1, s);
    rflag.alloc_zeroed(nbig, s);
    const uint32_t *P = pos.p;
    scan<SumU32>(nbig, RunHeadLoad{P, kin, shift}, RunIdStore{P, kin, rid.p, rflag.p}, s);
    compact(nbig, RunFlagged{rid.p, rflag.p}, sel.p, nsel.p, s);
    const uint32_t m = [&] {
        uint32_t v = 0;
        read_back(&v, nsel.p, sizeof(v), s);
        return v;
    }();
    if (!m) return;
    DBuf<uint64_t> k2[2] = {DBuf<uint64_t>(m, s), DBuf<uint64_t>(m, s)};
    DBuf<uint32_t> v2[2] = {DBuf<uint32_t>(m, s), DBuf<uint32_t>(m, s)}, P2(m, s);
    {
        const uint32_t *S = sel.p;
        uint32_t *p2 = P2.p;
        launch_k(k_compose_idx, grid_for(m, 256), 256, 0, s, P, S, (size_t)m, p2);
        CK_LAUNCH("k_compose_idx");
    }
    SortBufs<1> sb;
    sb.k[0].w[0] = k2[0].p, sb.k[1].w[0] = k2[1].p, sb.v[0] = v2[0].p, sb.v[1] = v2[1].p, sb.cur = 0;
    launch_k(k_gather_kv, grid_for(m, 256), 256, 0, s, (const uint32_t *)P2.p, (size_t)m, kin, vin, k2[0].p, v2[0].p);
    CK_LAUNCH("k_gather_kv");
    radix_sort<1>(sb, m, LiveBytes<1>{{live}}, s);
    launch_k(k_scatter_kv, grid_for(m, 256), 256, 0, s, (const uint32_t *)P2.p, (size_t)m, (const uint64_t *)sb.k[sb.cur].w[0],
             (const uint32_t *)sb.v[sb.cur], kout, vout);
    CK_LAUNCH("k_scatter_kv");
}

// Stable sort by a u64 key: LSD passes over the live bytes at and above `lowbyte` only, then the
// segmented fix-up orders runs of equal high parts by the full key.
inline void radix_sort_prefix(SortBufs<1> &b, size_t n, uint8_t live, int lowbyte, cudaStream_t s) {
    if (n <= 1 || !live) return;
    if (n <= (size_t)ST_TILE && sort_tiles_on()) {  // small: the whole key in one tile sort, no fix-up
        radix_sort<1>(b, n, LiveBytes<1>{{live}}, s);
        return;
    }
    const uint8_t top = (uint8_t)(live & (0xFFu << lowbyte));
    if (top == live || !top) {  // nothing below the prefix, or no prefix: plain LSD
        radix_sort<1>(b, n, LiveBytes<1>{{live}}, s);
        return;
    }
    radix_sort<1>(b, n, LiveBytes<1>{{top}}, s);
    seg_fixup(b, n, 8 * lowbyte, live, s);
}

// Random, well-spread keys (content hashes): LSD over just enough of the most significant live
// bytes for ~1 bit of slack over log2(n), then the fix-up (most runs have one record).
inline void radix_sort_wide(SortBufs<1> &b, size_t n, uint8_t live, cudaStream_t s) {
    if (n <= 1 || !live) return;
    if (n <= (size_t)ST_TILE && sort_tiles_on()) {
        radix_sort<1>(b, n, LiveBytes<1>{{live}}, s);
        return;
    }
    int need = 2;
    while (need < 64 && (1ull << need) < (uint64_t)n) ++need;
    const int nbytes = (need + 1 + 7) / 8;
    int got = 0, low = 0;
    for (int byte = 7; byte >= 0 && got < nbytes; --byte)
        if ((live >> byte) & 1) ++got, low = byte;
    radix_sort_prefix(b, n, live, low, s);
}

// Owning storage for a sort of n records.
template <int KW>
struct SortStore {
    DBuf<uint64_t> keys[2][KW];
    DBuf<uint32_t> vals[2];
    SortBufs<KW> b;
    SortStore(size_t n, cudaStream_t s) {
        for (int side = 0; side < 2; ++side) {
            for (int w = 0; w < KW; ++w) {
                keys[side][w].alloc(n ? n : 1, s);
                b.k[side].w[w] = keys[side][w].p;
            }
            vals[side].alloc(n ? n : 1, s);
            b.v[side] = vals[side].p;
        }
        b.cur = 0;
    }
    uint64_t *key(int w) const { return b.k[b.cur].w[w]; }
    uint32_t *val() const { return b.v[b.cur]; }
    uint64_t *in_key(int w) const { return b.k[0].w[w]; }
    uint32_t *in_val() const { return b.v[0]; }
};

}  // namespace b2l
