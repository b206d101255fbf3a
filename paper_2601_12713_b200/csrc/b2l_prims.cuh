// Device-wide primitives for the trace-analysis pipeline (sm_100a, hand-written):
//   * stream-ordered scratch buffers (cudaMallocAsync pool)
//   * generic tile scan (reduce-then-scan, 3 launches) over functor inputs/outputs,
//     with a segmented wrapper -- used for counts, prefix maxima, the max-plus
//     depth scan of alloc/delete pairing, run ids, compaction
//   * stable LSD radix sort of (multi-word u64 key, u32 value) records: 8-bit
//     digits, per-tile histograms + scanned digit offsets, stable tile ranking with
//     warp __match_any_sync multisplit; digit passes whose byte never varies are
//     skipped (planned from an OR-of-XOR reduction), so wide composite keys cost
//     only their live bytes.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <stdexcept>
#include <string>
#include <utility>

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
template <class T>
struct DBuf {
    T *p = nullptr;
    size_t n = 0;
    cudaStream_t s = nullptr;
    DBuf() = default;
    DBuf(size_t n_, cudaStream_t st) { alloc(n_, st); }
    void alloc(size_t n_, cudaStream_t st) {
        release();
        s = st;
        n = n_;
        if (n_) CK(cudaMallocAsync((void **)&p, n_ * sizeof(T), st));
    }
    void zero() {
        if (n) CK(cudaMemsetAsync(p, 0, n * sizeof(T), s));
    }
    void release() {
        if (p) cudaFreeAsync(p, s);
        p = nullptr;
        n = 0;
    }
    ~DBuf() { release(); }
    DBuf(const DBuf &) = delete;
    DBuf &operator=(const DBuf &) = delete;
    DBuf(DBuf &&o) noexcept : p(o.p), n(o.n), s(o.s) { o.p = nullptr, o.n = 0; }
    DBuf &operator=(DBuf &&o) noexcept {
        release();
        p = o.p, n = o.n, s = o.s;
        o.p = nullptr, o.n = 0;
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

template <class Op>
__device__ __forceinline__ typename Op::T block_excl_scan(typename Op::T v, typename Op::T *sm,
                                                          typename Op::T &total) {
    using T = typename Op::T;
    const int t = threadIdx.x;
    sm[t] = v;
    __syncthreads();
#pragma unroll 1
    for (int off = 1; off < SCAN_THREADS; off <<= 1) {
        T x = t >= off ? sm[t - off] : Op::identity();
        __syncthreads();
        if (t >= off) sm[t] = Op::combine(x, sm[t]);
        __syncthreads();
    }
    total = sm[SCAN_THREADS - 1];
    T ex = t ? sm[t - 1] : Op::identity();
    __syncthreads();
    return ex;
}

template <class Op, class Load>
__global__ void __launch_bounds__(SCAN_THREADS) k_scan_reduce(size_t n, Load ld, typename Op::T *partials) {
    using T = typename Op::T;
    __shared__ T sm[SCAN_THREADS];
    const size_t base = (size_t)blockIdx.x * SCAN_TILE + (size_t)threadIdx.x * SCAN_ITEMS;
    T acc = Op::identity();
#pragma unroll
    for (int k = 0; k < SCAN_ITEMS; ++k)
        if (base + k < n) acc = Op::combine(acc, ld(base + k));
    T total;
    block_excl_scan<Op>(acc, sm, total);
    if (threadIdx.x == 0) partials[blockIdx.x] = total;
}

template <class Op>
__global__ void __launch_bounds__(SCAN_THREADS) k_scan_partials(typename Op::T *partials, size_t np,
                                                                 typename Op::T *d_total) {
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

template <class Op, class Load, class Store>
__global__ void __launch_bounds__(SCAN_THREADS) k_scan_apply(size_t n, Load ld, Store st,
                                                             const typename Op::T *partials) {
    using T = typename Op::T;
    __shared__ T sm[SCAN_THREADS];
    const size_t base = (size_t)blockIdx.x * SCAN_TILE + (size_t)threadIdx.x * SCAN_ITEMS;
    T items[SCAN_ITEMS];
    T acc = Op::identity();
#pragma unroll
    for (int k = 0; k < SCAN_ITEMS; ++k) {
        items[k] = base + k < n ? ld(base + k) : Op::identity();
        acc = Op::combine(acc, items[k]);
    }
    T total;
    T ex = Op::combine(partials[blockIdx.x], block_excl_scan<Op>(acc, sm, total));
#pragma unroll
    for (int k = 0; k < SCAN_ITEMS; ++k) {
        if (base + k < n) st(base + k, ex, items[k]);
        ex = Op::combine(ex, items[k]);
    }
}

// scan over n items: st(i, exclusive_prefix, item) for every i; optional device total.
template <class Op, class Load, class Store>
void scan(size_t n, Load ld, Store st, cudaStream_t s, typename Op::T *d_total = nullptr) {
    using T = typename Op::T;
    if (n == 0) {  // only sums are scanned with a device total over possibly-empty ranges
        if (d_total) CK(cudaMemsetAsync(d_total, 0, sizeof(T), s));
        return;
    }
    const size_t tiles = (n + SCAN_TILE - 1) / SCAN_TILE;
    DBuf<T> part(tiles, s);
    k_scan_reduce<Op, Load><<<(unsigned)tiles, SCAN_THREADS, 0, s>>>(n, ld, part.p);
    CK_LAUNCH("k_scan_reduce");
    k_scan_partials<Op><<<1, SCAN_THREADS, 0, s>>>(part.p, tiles, d_total);
    CK_LAUNCH("k_scan_partials");
    k_scan_apply<Op, Load, Store><<<(unsigned)tiles, SCAN_THREADS, 0, s>>>(n, ld, st, part.p);
    CK_LAUNCH("k_scan_apply");
}

// ---------------------------------------------------------------- pinned scalar readback
struct HostScalars {
    uint64_t *h = nullptr;
    uint64_t *d = nullptr;
    int cap = 0;
    cudaStream_t s = nullptr;
    HostScalars(int n, cudaStream_t st) : cap(n), s(st) {
        CK(cudaMallocHost(&h, n * sizeof(uint64_t)));
        CK(cudaMallocAsync((void **)&d, n * sizeof(uint64_t), st));
        CK(cudaMemsetAsync(d, 0, n * sizeof(uint64_t), st));
    }
    ~HostScalars() {
        if (d) cudaFreeAsync(d, s);
        if (h) cudaFreeHost(h);
    }
    uint64_t *dev(int i) { return d + i; }
    // copy slots [0, k) back and wait
    void fetch(int k) {
        CK(cudaMemcpyAsync(h, d, k * sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
    }
};

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
        CK(cudaMemsetAsync(d_count, 0, sizeof(uint32_t), s));
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
constexpr int RS_ROUNDS = 16;
constexpr int RS_TILE = RS_THREADS * RS_ROUNDS;

template <int KW>
struct KeyCols {
    uint64_t *w[KW];  // w[0] = most significant word
};

__device__ __forceinline__ uint32_t lanemask_lt() {
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

template <int KW>
__global__ void k_key_vary(KeyCols<KW> k, size_t n, unsigned long long *vary) {
    unsigned long long acc[KW];
    uint64_t first[KW];
#pragma unroll
    for (int w = 0; w < KW; ++w) acc[w] = 0, first[w] = k.w[w][0];
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
#pragma unroll
        for (int w = 0; w < KW; ++w) acc[w] |= k.w[w][i] ^ first[w];
#pragma unroll
    for (int w = 0; w < KW; ++w) {
        unsigned long long v = acc[w];
        for (int o = 16; o; o >>= 1) v |= __shfl_xor_sync(0xffffffffu, v, o);
        if ((threadIdx.x & 31) == 0 && v) atomicOr(vary + w, v);
    }
}

__global__ void __launch_bounds__(RS_THREADS) k_radix_hist(const uint64_t *__restrict__ key, size_t n, int shift,
                                                           uint32_t *__restrict__ counts, unsigned ntiles) {
    __shared__ uint32_t hist[256];
    hist[threadIdx.x] = 0;
    __syncthreads();
    const size_t base = (size_t)blockIdx.x * RS_TILE;
    const int lane = threadIdx.x & 31;
#pragma unroll 4
    for (int r = 0; r < RS_ROUNDS; ++r) {
        const size_t pos = base + (size_t)r * RS_THREADS + threadIdx.x;
        const bool valid = pos < n;
        const uint32_t d = valid ? (uint32_t)(key[pos] >> shift) & 255u : 256u;
        const uint32_t peers = __match_any_sync(0xffffffffu, d);
        if (valid && lane == __ffs(peers) - 1) atomicAdd(&hist[d], (uint32_t)__popc(peers));
    }
    __syncthreads();
    counts[(size_t)threadIdx.x * ntiles + blockIdx.x] = hist[threadIdx.x];
}

template <int KW>
__global__ void __launch_bounds__(RS_THREADS) k_radix_scatter(KeyCols<KW> in, const uint32_t *__restrict__ vin,
                                                              KeyCols<KW> out, uint32_t *__restrict__ vout, size_t n,
                                                              int word, int shift,
                                                              const uint32_t *__restrict__ offs, unsigned ntiles) {
    __shared__ uint32_t base_off[256];
    __shared__ uint32_t running[256];
    __shared__ uint32_t wcnt[RS_THREADS / 32][256];
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    base_off[t] = offs[(size_t)t * ntiles + blockIdx.x];
    running[t] = 0;
    const size_t base = (size_t)blockIdx.x * RS_TILE;
    const uint64_t *kd = in.w[word];
    for (int r = 0; r < RS_ROUNDS; ++r) {
#pragma unroll
        for (int w = 0; w < RS_THREADS / 32; ++w) wcnt[w][t] = 0;
        __syncthreads();
        const size_t pos = base + (size_t)r * RS_THREADS + t;
        const bool valid = pos < n;
        const uint32_t d = valid ? (uint32_t)(kd[pos] >> shift) & 255u : 256u;
        const uint32_t peers = __match_any_sync(0xffffffffu, d);
        const uint32_t wrank = __popc(peers & lanemask_lt());
        if (valid && lane == __ffs(peers) - 1) wcnt[warp][d] = __popc(peers);
        __syncthreads();
        uint32_t run = running[t];
#pragma unroll
        for (int w = 0; w < RS_THREADS / 32; ++w) {
            uint32_t c = wcnt[w][t];
            wcnt[w][t] = run;
            run += c;
        }
        running[t] = run;
        __syncthreads();
        if (valid) {
            const uint32_t dst = base_off[d] + wcnt[warp][d] + wrank;
#pragma unroll
            for (int w = 0; w < KW; ++w) out.w[w][dst] = in.w[w][pos];
            vout[dst] = vin[pos];
        }
        __syncthreads();
    }
    (void)running;
}

template <int KW>
struct SortBufs {
    KeyCols<KW> k[2];
    uint32_t *v[2];
    int cur = 0;  // which side holds the data
};

// Stable sort of n records (keys KW words, value u32) held in side `b.cur`; on return b.cur names
// the side holding the sorted records.  One host sync (pass planning).
template <int KW>
void radix_sort(SortBufs<KW> &b, size_t n, cudaStream_t s) {
    if (n <= 1) return;
    DBuf<unsigned long long> vary(KW, s);
    vary.zero();
    k_key_vary<KW><<<grid_for(n, 256, 148 * 8), 256, 0, s>>>(b.k[b.cur], n, vary.p);
    CK_LAUNCH("k_key_vary");
    unsigned long long hv[KW];
    CK(cudaMemcpyAsync(hv, vary.p, sizeof(hv), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    const unsigned ntiles = (unsigned)((n + RS_TILE - 1) / RS_TILE);
    DBuf<uint32_t> counts((size_t)256 * ntiles, s);
    for (int w = KW - 1; w >= 0; --w) {
        for (int byte = 0; byte < 8; ++byte) {
            if (((hv[w] >> (8 * byte)) & 255ull) == 0) continue;  // digit constant over all keys: identity pass
            const int shift = 8 * byte;
            k_radix_hist<<<ntiles, RS_THREADS, 0, s>>>(b.k[b.cur].w[w], n, shift, counts.p, ntiles);
            CK_LAUNCH("k_radix_hist");
            uint32_t *cp = counts.p;
            scan<SumU32>((size_t)256 * ntiles, LoadU32{cp}, StoreExclU32{cp}, s);
            k_radix_scatter<KW><<<ntiles, RS_THREADS, 0, s>>>(b.k[b.cur], b.v[b.cur], b.k[b.cur ^ 1], b.v[b.cur ^ 1],
                                                              n, w, shift, counts.p, ntiles);
            CK_LAUNCH("k_radix_scatter");
            b.cur ^= 1;
        }
    }
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
