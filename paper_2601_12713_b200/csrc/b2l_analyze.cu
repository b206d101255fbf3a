// Trace-analysis pipeline on the B200: validate -> partition -> (DD, RT) ->
// LIFO pairing -> RA -> UA / UT, all as sort / segmented-scan / compaction
// passes over SoA event columns (no per-event sequential sweep).
//
// Reference semantics (paths under /root/reference/pkg/src/dmlens/):
//   validate        model.py:125-200        -> k_validate (rule bits per event)
//   analyze         detectors.py:274-326    -> analyze_impl (partition :296-312)
//   pairing         prep.py:45-96           -> pairs_step: stable sort by (dst_dev, dst_addr),
//                                              clamped-depth max-plus scan, (segment, level)
//                                              sort; alternating A,D at one level are pairs
//   DD              detectors.py:85-103     -> dd_rt_step: segments of the (hash, dev) sort
//   RT default      detectors.py:106-167    -> r_j = j + max_{i<=j}(f_i - i) over each queue
//   RT strict       detectors.py:139-160    -> k_rt_strict: one thread per hash, head pointers
//   RA              detectors.py:170-191    -> ra_step: stable sort of pairs by (addr, dev, bytes)
//   UA / UT         detectors.py:194-271    -> kernel cursor = lower_bound of the per-device
//                                              prefix max of kernel ends; UT run ids by scan
// Proofs of the reformulations: SURVEY.md Appendix A; the GPU tests check every step
// against oracle/analysis_ref.py and the reference's golden outputs.
#include <chrono>
#include <condition_variable>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <exception>
#include <functional>
#include <future>
#include <mutex>
#include <thread>
#include <type_traits>
#include <vector>

#include "b2l_prims.cuh"

namespace b2l {
namespace ana {

constexpr uint32_t NONE = 0xFFFFFFFFu;
constexpr int TPB = 256;

struct DevCols {
    size_t n;
    int ndev, host;
    const uint64_t *seq, *start, *end, *sa, *da, *nb, *h;
    const int32_t *src, *dst;
    const uint8_t *kind;
    const uint32_t *loc;
    const uint8_t *loc_flags;
    const uint32_t *loc_bucket;
    uint32_t nlocs, nbuckets;
};

// Which key bytes can vary (OR over events of x ^ x[0] per column) and value-range masks;
// computed once per trace so no sort needs a host round trip for pass planning.
struct Masks {
    uint8_t hash = 0xFF, sa = 0xFF, da = 0xFF, nb = 0xFF, sa_tt = 0xFF, dev = 0xFF, idx = 0xFF;
    const uint32_t *srank = nullptr;  // srank[i] = first index with start == start[i]
    uint64_t n = 0;                   // events
};
// Bits needed to hold values < v.
inline int bit_width(uint64_t v) {
    int b = 0;
    while (b < 64 && v > 1 && ((v - 1) >> b)) ++b;
    return b;
}
thread_local Masks g_masks;

// Owns device copies of host columns.
struct ColsUpload {
    std::vector<DBuf<uint8_t>> bufs;
    DevCols d{};
    template <class T>
    const T *up(const T *h, size_t n, cudaStream_t s) {
        if (!n) return nullptr;
        bufs.emplace_back(n * sizeof(T), s);
        CK(cudaMemcpyAsync(bufs.back().p, h, n * sizeof(T), cudaMemcpyHostToDevice, s));
        return reinterpret_cast<const T *>(bufs.back().p);
    }
    void load(const b2l_trace_cols *c, cudaStream_t s) {
        d.n = c->n_events;
        d.ndev = c->num_devices_total;
        d.host = c->host_device;
        d.nlocs = c->n_locs;
        d.nbuckets = c->n_buckets;
        if (c->device_resident) {
            d.seq = c->seq, d.start = c->start_ns, d.end = c->end_ns, d.sa = c->src_addr, d.da = c->dst_addr;
            d.nb = c->bytes, d.h = c->hash, d.src = c->src_device, d.dst = c->dst_device, d.kind = c->kind;
            d.loc = c->loc, d.loc_flags = c->loc_flags, d.loc_bucket = c->loc_bucket;
            return;
        }
        const size_t n = d.n;
        d.seq = up(c->seq, n, s), d.start = up(c->start_ns, n, s), d.end = up(c->end_ns, n, s);
        d.sa = up(c->src_addr, n, s), d.da = up(c->dst_addr, n, s), d.nb = up(c->bytes, n, s);
        d.h = up(c->hash, n, s), d.src = up(c->src_device, n, s), d.dst = up(c->dst_device, n, s);
        d.kind = up(c->kind, n, s), d.loc = up(c->loc, n, s);
        d.loc_flags = up(c->loc_flags, c->n_locs, s), d.loc_bucket = up(c->loc_bucket, c->n_locs, s);
    }
};

// ============================================================ validation (model.py:125-200)
// One event's fields, loaded with plain coalesced loads (the 64-B/event algorithmic read).
struct Row {
    uint64_t seq, start, end, nb, h, da;
    int32_t src, dst;
    uint8_t kind;
    uint32_t loc;
};
__device__ __forceinline__ Row load_row(const DevCols &c, size_t i) {
    Row r;
    r.seq = c.seq[i], r.start = c.start[i], r.end = c.end[i], r.nb = c.nb[i], r.h = c.h[i], r.da = c.da[i];
    r.src = c.src[i], r.dst = c.dst[i], r.kind = c.kind[i], r.loc = c.loc[i];
    return r;
}
// Rule bits of one event given the previous event's (start, seq) (has_prev false for event 0).
__device__ __forceinline__ uint32_t row_rules(const DevCols &c, const Row &r, bool has_prev, uint64_t ps, uint64_t pq) {
    uint32_t m = 0;
    if (r.start > r.end) m |= B2L_RULE_INTERVAL;
    if (r.src < 0 || r.src >= c.ndev) m |= B2L_RULE_SRC_DEVICE;
    if (r.dst < 0 || r.dst >= c.ndev) m |= B2L_RULE_DST_DEVICE;
    switch (r.kind) {
        case B2L_KIND_TRANSFER:
            if (r.nb > 0 && r.h == 0) m |= B2L_RULE_TRANSFER_HASH;
            break;
        case B2L_KIND_ALLOC:
            if (r.nb == 0) m |= B2L_RULE_ALLOC_BYTES;
            if (r.da == 0) m |= B2L_RULE_ALLOC_ADDR;
            break;
        case B2L_KIND_DELETE:
            if (r.da == 0) m |= B2L_RULE_DELETE_ADDR;
            break;
        default:
            if (r.src != r.dst) m |= B2L_RULE_KERNEL_DEVICE;
    }
    const uint8_t lf = c.loc_flags[r.loc];
    if (lf & B2L_LOC_FILE_NO_LINE) m |= B2L_RULE_LOC_FILE;
    if (lf & B2L_LOC_LINE_NONPOS) m |= B2L_RULE_LOC_LINE;
    if (has_prev) {
        if (r.start < ps || (r.start == ps && r.seq < pq)) m |= B2L_RULE_ORDER_SORT;
        if (r.seq <= pq) m |= B2L_RULE_ORDER_SEQ;
    }
    return m;
}
__device__ __forceinline__ uint32_t event_rules(const DevCols &c, size_t i) {
    const Row r = load_row(c, i);
    return row_rules(c, r, i > 0, i > 0 ? c.start[i - 1] : 0, i > 0 ? c.seq[i - 1] : 0);
}
__global__ void k_bad_rules(DevCols c, const uint32_t *bad, const uint32_t *count, uint32_t *rules) {
    const uint32_t nb = *count;
    for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < nb; k += gridDim.x * blockDim.x)
        rules[k] = event_rules(c, bad[k]);
}

// ============================================================ partition (detectors.py:296-312)

// ============================================================ fused front pass
// validate + partition + max data-op end + key-bit variation + start ranks in one
// reduce -> partials-scan -> apply sequence (3 launches, two reads of the columns):
//   reduce: per 4096-event tile, counts of {bad, H, TT, AD, A, TK} and the last start
//           change; block-reduced atomics for max end and the OR/AND masks;
//   apply:  order-preserving warp-ballot compaction of the five index lists (or of the
//           bad list when validation failed) and srank[i] = last start change <= i.
#ifndef B2L_FR_ITEMS
#define B2L_FR_ITEMS 16
#endif
#ifndef B2L_FR_MINB
#define B2L_FR_MINB 2
#endif
constexpr int FR_THREADS = 256, FR_ITEMS = B2L_FR_ITEMS, FR_TILE = FR_THREADS * FR_ITEMS, FR_NCAT = 6;
#ifndef B2L_FR_MINB_APPLY
#define B2L_FR_MINB_APPLY B2L_FR_MINB
#endif
constexpr int FR_MINB = B2L_FR_MINB;  // resident CTAs per SM the front kernels are compiled for
constexpr int FR_MINB_APPLY = B2L_FR_MINB_APPLY;
#ifndef B2L_FR_MINB_FUSED
#define B2L_FR_MINB_FUSED B2L_FR_MINB
#endif
constexpr int FR_MINB_FUSED = B2L_FR_MINB_FUSED;
#ifndef B2L_FR_BATCH_FUSED
#define B2L_FR_BATCH_FUSED 4
#endif
constexpr int FR_BATCH_FUSED = B2L_FR_BATCH_FUSED;  // rows whose loads the fused pass issues together
static_assert(FR_ITEMS % FR_BATCH_FUSED == 0 && FR_ITEMS % 4 == 0, "the load batches tile a thread's items");
enum : uint32_t { F_BAD = 1, F_H = 2, F_TT = 4, F_AD = 8, F_A = 16, F_TK = 32 };
struct FrontAcc {
    uint32_t c[FR_NCAT];
    uint32_t lastchg;  // max index j <= i with j == 0 or start[j] != start[j-1]
};
struct FrontOp {
    using T = FrontAcc;
    static __device__ __forceinline__ T identity() { return T{{0, 0, 0, 0, 0, 0}, 0}; }
    static __device__ __forceinline__ T combine(T a, T b) {
        T r;
#pragma unroll
        for (int k = 0; k < FR_NCAT; ++k) r.c[k] = a.c[k] + b.c[k];
        r.lastchg = a.lastchg > b.lastchg ? a.lastchg : b.lastchg;
        return r;
    }
};
__device__ __forceinline__ uint32_t part_flags(const DevCols &c, uint8_t k, int32_t dst, uint64_t nb, uint64_t h,
                                               bool raw) {
    uint32_t f = 0;
    if (k == B2L_KIND_TRANSFER && (raw || (nb > 0 && h != 0))) f |= F_H;
    if (k == B2L_KIND_TRANSFER && dst != c.host) f |= F_TT;
    if (k == B2L_KIND_ALLOC || k == B2L_KIND_DELETE) f |= F_AD;
    if (k == B2L_KIND_ALLOC) f |= F_A;
    if (k == B2L_KIND_KERNEL && dst != c.host) f |= F_TK;
    return f;
}
constexpr int FR_BATCH = 4;  // items whose loads are issued together (memory-level parallelism)

__global__ void __launch_bounds__(FR_THREADS, FR_MINB) k_front_reduce(DevCols c, bool validate, bool raw, FrontAcc *partials,
                                                             unsigned long long *agg /*[0] max end, [1..5] OR, [6..10] AND*/) {
    pdl_enter();
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const size_t wb = (size_t)blockIdx.x * FR_TILE + (size_t)warp * (32 * FR_ITEMS) + lane;
    const size_t last = c.n - 1;
    uint32_t cnt[FR_NCAT] = {0, 0, 0, 0, 0, 0}, lastchg = 0;
    unsigned long long me = 0, o[5] = {0, 0, 0, 0, 0}, a[5] = {~0ull, ~0ull, ~0ull, ~0ull, ~0ull};
#pragma unroll 1
    for (int k0 = 0; k0 < FR_ITEMS; k0 += FR_BATCH) {
        if (wb - lane + 32 * k0 > last) break;  // warp-uniform
        Row r[FR_BATCH];
        uint64_t sa[FR_BATCH], p0s = 0, p0q = 0;
#pragma unroll
        for (int b = 0; b < FR_BATCH; ++b) {
            const size_t i = wb + 32 * (k0 + b), ic = i < last ? i : last;
            r[b] = load_row(c, ic);
            sa[b] = c.sa[ic];
        }
        {
            const size_t i0 = wb + 32 * k0;  // lane 0's predecessor lives in the previous 32-run
            if (lane == 0 && i0 > 0 && i0 <= last) p0s = c.start[i0 - 1], p0q = c.seq[i0 - 1];
        }
#pragma unroll
        for (int b = 0; b < FR_BATCH; ++b) {
            const size_t i = wb + 32 * (k0 + b);
            uint64_t ps = __shfl_up_sync(0xffffffffu, r[b].start, 1), pq = __shfl_up_sync(0xffffffffu, r[b].seq, 1);
            if (lane == 0) {
                if (b == 0) ps = p0s, pq = p0q;
                else ps = c.start[i - 1 < last ? i - 1 : last], pq = c.seq[i - 1 < last ? i - 1 : last];
            }
            if (i > last) continue;
            uint32_t f = part_flags(c, r[b].kind, r[b].dst, r[b].nb, r[b].h, raw);
            if (validate && row_rules(c, r[b], i > 0, ps, pq)) f |= F_BAD;
#pragma unroll
            for (int q = 0; q < FR_NCAT; ++q) cnt[q] += (f >> q) & 1u;
            if (i == 0 || r[b].start != ps) lastchg = (uint32_t)i;  // i increases along the loop
            if (r[b].kind != B2L_KIND_KERNEL) me = r[b].end > me ? r[b].end : me;
            if (r[b].kind == B2L_KIND_TRANSFER) {
                o[0] |= r[b].h, a[0] &= r[b].h;  // superset of the hashed subset
                if (f & F_TT) o[4] |= sa[b], a[4] &= sa[b];
            } else if (f & F_AD) {
                o[1] |= r[b].da, a[1] &= r[b].da;
                if (f & F_A) o[2] |= sa[b], a[2] &= sa[b], o[3] |= r[b].nb, a[3] &= r[b].nb;
            }
        }
    }
    // warp reductions
#pragma unroll
    for (int off = 16; off; off >>= 1) {
#pragma unroll
        for (int q = 0; q < FR_NCAT; ++q) cnt[q] += __shfl_xor_sync(0xffffffffu, cnt[q], off);
        const uint32_t lc = __shfl_xor_sync(0xffffffffu, lastchg, off);
        lastchg = lc > lastchg ? lc : lastchg;
        const unsigned long long m2 = __shfl_xor_sync(0xffffffffu, me, off);
        me = m2 > me ? m2 : me;
#pragma unroll
        for (int q = 0; q < 5; ++q) {
            o[q] |= __shfl_xor_sync(0xffffffffu, o[q], off);
            a[q] &= __shfl_xor_sync(0xffffffffu, a[q], off);
        }
    }
    __shared__ uint32_t sc[FR_THREADS / 32][FR_NCAT + 1];
    __shared__ unsigned long long sm[FR_THREADS / 32][11];
    if (lane == 0) {
#pragma unroll
        for (int q = 0; q < FR_NCAT; ++q) sc[warp][q] = cnt[q];
        sc[warp][FR_NCAT] = lastchg;
        sm[warp][0] = me;
#pragma unroll
        for (int q = 0; q < 5; ++q) sm[warp][1 + q] = o[q], sm[warp][6 + q] = a[q];
    }
    __syncthreads();
    if (t < FR_NCAT + 1) {
        uint32_t v = 0;
        for (int w = 0; w < FR_THREADS / 32; ++w) v = t < FR_NCAT ? v + sc[w][t] : (sc[w][t] > v ? sc[w][t] : v);
        if (t < FR_NCAT) partials[blockIdx.x].c[t] = v;
        else partials[blockIdx.x].lastchg = v;
    } else if (t >= 32 && t < 32 + 11) {
        const int q = t - 32;
        unsigned long long v = q < 6 ? 0ull : ~0ull;
        for (int w = 0; w < FR_THREADS / 32; ++w) {
            const unsigned long long x = sm[w][q];
            v = q == 0 ? (x > v ? x : v) : q < 6 ? (v | x) : (v & x);
        }
        if (q == 0) {
            if (v) atomicMax(agg, v);
        } else if (q < 6) {
            if (v) atomicOr(agg + q, v);
        } else if (~v) {
            atomicAnd(agg + q, v);
        }
    }
}

struct FrontOut {
    uint32_t *list[FR_NCAT];  // bad, H, TT, AD, A, TK (nullptr: not written)
    uint32_t *srank;          // nullptr: not written
    // attribution record per event (fused savings; nullptr: not written): {duration | bucket << 40,
    // bytes} -- one 16-byte gather per finding member in k_attr instead of four column gathers
    // (loc, start, end, bytes); `nopack` is set when some duration >= 2^40 or bucket >= 2^24
    ulonglong2 *attr;
    unsigned *nopack;
    uint64_t *hd;  // per entry of the hashed-transfer list: src << 32 | dst (nullptr: not written)
};
// Warp-striped tiles (item k of lane l in warp w is base + w*32*ITEMS + 32k + l) keep index
// order under ballot ranking: a warp's items precede the next warp's, items precede items.
// bad_mode: only the bad list (validation failed); else the five partition lists + srank.
__global__ void __launch_bounds__(FR_THREADS, FR_MINB_APPLY) k_front_apply(DevCols c, bool bad_mode, bool raw,
                                                            const FrontAcc *__restrict__ prefix, FrontOut out) {
    pdl_enter();
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const size_t wb = (size_t)blockIdx.x * FR_TILE + (size_t)warp * (32 * FR_ITEMS) + lane;
    const size_t last = c.n - 1;
    const uint32_t lt = lanemask_lt();
    uint32_t fl[FR_ITEMS];  // bits 0..5 category flags, bit 6 start change
    uint32_t wc[FR_NCAT] = {0, 0, 0, 0, 0, 0};
    bool nopack = false;
#pragma unroll
    for (int k0 = 0; k0 < FR_ITEMS; k0 += FR_BATCH) {
        uint8_t kd[FR_BATCH];
        int32_t dst[FR_BATCH];
        uint64_t nb[FR_BATCH], h[FR_BATCH], st[FR_BATCH];
#pragma unroll
        for (int b = 0; b < FR_BATCH; ++b) {
            const size_t i = wb + 32 * (k0 + b), ic = i < last ? i : last;
            kd[b] = c.kind[ic], dst[b] = c.dst[ic], nb[b] = c.nb[ic], h[b] = c.h[ic], st[b] = c.start[ic];
        }
        if (out.attr) {
#pragma unroll
            for (int b = 0; b < FR_BATCH; ++b) {
                const size_t i = wb + 32 * (k0 + b);
                if (i > last) continue;
                const uint64_t d = c.end[i] - st[b];
                const uint32_t bk = c.nbuckets ? c.loc_bucket[c.loc[i]] : 0u;
                nopack |= (d >> 40) != 0 || (bk >> 24) != 0;
                out.attr[i] = make_ulonglong2(d | ((unsigned long long)bk << 40), nb[b]);
            }
        }
#pragma unroll
        for (int b = 0; b < FR_BATCH; ++b) {
            const size_t i = wb + 32 * (k0 + b);
            uint64_t ps = __shfl_up_sync(0xffffffffu, st[b], 1);
            if (lane == 0 && i > 0 && i <= last) ps = c.start[i - 1];
            uint32_t f = 0;
            if (i <= last) {
                if (bad_mode) {
                    f = event_rules(c, i) ? F_BAD : 0u;
                } else {
                    f = part_flags(c, kd[b], dst[b], nb[b], h[b], raw);
                    if (i == 0 || st[b] != ps) f |= 64u;
                }
            }
            fl[k0 + b] = f;
#pragma unroll
            for (int q = 0; q < FR_NCAT; ++q) wc[q] += __popc(__ballot_sync(0xffffffffu, (f >> q) & 1u));
        }
    }
    if (out.attr && __any_sync(0xffffffffu, nopack) && lane == 0) atomicOr(out.nopack, 1u);
    // srank: the last start change at or before each index (max scan of change positions)
    uint32_t chmax = 0;
#pragma unroll
    for (int k = 0; k < FR_ITEMS; ++k)
        if (fl[k] & 64u) chmax = (uint32_t)(wb + 32 * k);
#pragma unroll
    for (int off = 16; off; off >>= 1) {
        const uint32_t v = __shfl_xor_sync(0xffffffffu, chmax, off);
        chmax = v > chmax ? v : chmax;
    }
    __shared__ uint32_t swc[FR_THREADS / 32][FR_NCAT + 1];
    if (lane == 0) {
#pragma unroll
        for (int q = 0; q < FR_NCAT; ++q) swc[warp][q] = wc[q];
        swc[warp][FR_NCAT] = chmax;
    }
    __syncthreads();
    const FrontAcc pre = prefix[blockIdx.x];
    uint32_t run[FR_NCAT];
#pragma unroll
    for (int q = 0; q < FR_NCAT; ++q) {
        uint32_t b = pre.c[q];
        for (int w = 0; w < warp; ++w) b += swc[w][q];
        run[q] = b;
    }
    uint32_t carry = pre.lastchg;
    for (int w = 0; w < warp; ++w) carry = swc[w][FR_NCAT] > carry ? swc[w][FR_NCAT] : carry;
#pragma unroll
    for (int k = 0; k < FR_ITEMS; ++k) {
        const size_t i = wb + 32 * k;
#pragma unroll
        for (int q = 0; q < FR_NCAT; ++q) {
            const uint32_t m = __ballot_sync(0xffffffffu, (fl[k] >> q) & 1u);
            if (out.list[q] && ((fl[k] >> q) & 1u)) {
                out.list[q][run[q] + __popc(m & lt)] = (uint32_t)i;
                if (q == 1 && out.hd)  // (the columns were just read: cached)
                    out.hd[run[q] + __popc(m & lt)] = ((uint64_t)(uint32_t)c.src[i] << 32) | (uint32_t)c.dst[i];
            }
            run[q] += __popc(m);
        }
        if (out.srank) {
            uint32_t v = (fl[k] & 64u) ? (uint32_t)i : 0u;
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, v, off);
                if (lane >= off) v = y > v ? y : v;
            }
            v = v > carry ? v : carry;
            if (i <= last) out.srank[i] = v;
            carry = __shfl_sync(0xffffffffu, v, 31);
        }
    }
}

// Single-pass front (the normal path): reduce + apply in ONE read of the columns.  Tiles take
// ids in launch order; each reads its 4096 rows once (validation rules, partition flags, start
// changes, max data-op end, key masks, attribution records), publishes its counts by decoupled
// look-back (block_lookback: the same protocol as the single-pass scans) and compacts its five
// index lists + start ranks behind the exclusive prefix it gets back.  The bad list is not
// written: a trace with violations (total.c[0] > 0) takes the reduce/apply path above, once, to
// list them (an error path).  Columns are read once instead of twice (10M events: ~140 -> ~100
// B/event for the front pass).
__global__ void __launch_bounds__(FR_THREADS, FR_MINB_FUSED) k_front_fused(DevCols c, bool validate, bool raw,
                                                                     FrontOut out, FrontAcc *lb_agg,
                                                                     FrontAcc *lb_inc, uint32_t *lb_flag,
                                                                     uint32_t *counter, FrontAcc *d_total,
                                                                     unsigned long long *agg) {
    static_assert(FR_THREADS == SCAN_THREADS, "block_lookback runs on the whole block");
    pdl_enter();
    __shared__ uint32_t tile_s;
    if (threadIdx.x == 0) tile_s = atomicAdd(counter, 1u);
    __syncthreads();
    const uint32_t tile = tile_s;
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const size_t wb = (size_t)tile * FR_TILE + (size_t)warp * (32 * FR_ITEMS) + lane;
    const size_t last = c.n - 1;
    const uint32_t lt = lanemask_lt();
    uint32_t fl[FR_ITEMS];  // bits 0..5 category flags, bit 6 start change
    uint32_t wc[FR_NCAT] = {0, 0, 0, 0, 0, 0};
    bool nopack = false;
    unsigned long long me = 0, o[5] = {0, 0, 0, 0, 0}, a[5] = {~0ull, ~0ull, ~0ull, ~0ull, ~0ull};
#pragma unroll
    for (int k0 = 0; k0 < FR_ITEMS; k0 += FR_BATCH_FUSED) {
        Row r[FR_BATCH_FUSED];
        uint64_t sa[FR_BATCH_FUSED], p0s = 0, p0q = 0;
#pragma unroll
        for (int b = 0; b < FR_BATCH_FUSED; ++b) {
            const size_t i = wb + 32 * (k0 + b), ic = i < last ? i : last;
            r[b] = load_row(c, ic);
            sa[b] = c.sa[ic];
        }
        {
            const size_t i0 = wb + 32 * k0;  // lane 0's predecessor lives in the previous 32-run
            if (lane == 0 && i0 > 0 && i0 <= last) p0s = c.start[i0 - 1], p0q = c.seq[i0 - 1];
        }
#pragma unroll
        for (int b = 0; b < FR_BATCH_FUSED; ++b) {
            const size_t i = wb + 32 * (k0 + b);
            uint64_t ps = __shfl_up_sync(0xffffffffu, r[b].start, 1), pq = __shfl_up_sync(0xffffffffu, r[b].seq, 1);
            if (lane == 0) {
                if (b == 0) ps = p0s, pq = p0q;
                else ps = c.start[i - 1 < last ? i - 1 : last], pq = c.seq[i - 1 < last ? i - 1 : last];
            }
            uint32_t f = 0;
            if (i <= last) {
                f = part_flags(c, r[b].kind, r[b].dst, r[b].nb, r[b].h, raw);
                if (validate && row_rules(c, r[b], i > 0, ps, pq)) f |= F_BAD;
                if (i == 0 || r[b].start != ps) f |= 64u;
                if (r[b].kind != B2L_KIND_KERNEL) me = r[b].end > me ? r[b].end : me;
                if (r[b].kind == B2L_KIND_TRANSFER) {
                    o[0] |= r[b].h, a[0] &= r[b].h;  // superset of the hashed subset
                    if (f & F_TT) o[4] |= sa[b], a[4] &= sa[b];
                } else if (f & F_AD) {
                    o[1] |= r[b].da, a[1] &= r[b].da;
                    if (f & F_A) o[2] |= sa[b], a[2] &= sa[b], o[3] |= r[b].nb, a[3] &= r[b].nb;
                }
                if (out.attr) {
                    const uint64_t d = r[b].end - r[b].start;
                    const uint32_t bk = c.nbuckets ? c.loc_bucket[r[b].loc] : 0u;
                    nopack |= (d >> 40) != 0 || (bk >> 24) != 0;
                    out.attr[i] = make_ulonglong2(d | ((unsigned long long)bk << 40), r[b].nb);
                }
            }
            fl[k0 + b] = f;
#pragma unroll
            for (int q = 0; q < FR_NCAT; ++q) wc[q] += __popc(__ballot_sync(0xffffffffu, (f >> q) & 1u));
        }
    }
    if (out.attr && __any_sync(0xffffffffu, nopack) && lane == 0) atomicOr(out.nopack, 1u);
    uint32_t chmax = 0;
#pragma unroll
    for (int k = 0; k < FR_ITEMS; ++k)
        if (fl[k] & 64u) chmax = (uint32_t)(wb + 32 * k);
#pragma unroll
    for (int off = 16; off; off >>= 1) {
        const uint32_t v = __shfl_xor_sync(0xffffffffu, chmax, off);
        chmax = v > chmax ? v : chmax;
        const unsigned long long m2 = __shfl_xor_sync(0xffffffffu, me, off);
        me = m2 > me ? m2 : me;
#pragma unroll
        for (int q = 0; q < 5; ++q) {
            o[q] |= __shfl_xor_sync(0xffffffffu, o[q], off);
            a[q] &= __shfl_xor_sync(0xffffffffu, a[q], off);
        }
    }
    __shared__ uint32_t swc[FR_THREADS / 32][FR_NCAT + 1];
    __shared__ unsigned long long sm[FR_THREADS / 32][11];
    if (lane == 0) {
#pragma unroll
        for (int q = 0; q < FR_NCAT; ++q) swc[warp][q] = wc[q];
        swc[warp][FR_NCAT] = chmax;
        sm[warp][0] = me;
#pragma unroll
        for (int q = 0; q < 5; ++q) sm[warp][1 + q] = o[q], sm[warp][6 + q] = a[q];
    }
    __syncthreads();
    if (t >= 32 && t < 32 + 11) {  // key masks and max end: block-reduced atomics
        const int q = t - 32;
        unsigned long long v = q < 6 ? 0ull : ~0ull;
        for (int w = 0; w < FR_THREADS / 32; ++w) {
            const unsigned long long x = sm[w][q];
            v = q == 0 ? (x > v ? x : v) : q < 6 ? (v | x) : (v & x);
        }
        if (q == 0) {
            if (v) atomicMax(agg, v);
        } else if (q < 6) {
            if (v) atomicOr(agg + q, v);
        } else if (~v) {
            atomicAnd(agg + q, v);
        }
    }
    FrontAcc total = FrontOp::identity();
    for (int w = 0; w < FR_THREADS / 32; ++w) {
#pragma unroll
        for (int q = 0; q < FR_NCAT; ++q) total.c[q] += swc[w][q];
        total.lastchg = swc[w][FR_NCAT] > total.lastchg ? swc[w][FR_NCAT] : total.lastchg;
    }
    const FrontAcc pre = block_lookback<FrontOp>(tile, total, lb_agg, lb_inc, lb_flag);
    if (t == 0 && (size_t)(tile + 1) * FR_TILE > last) *d_total = FrontOp::combine(pre, total);
    uint32_t run[FR_NCAT];
#pragma unroll
    for (int q = 0; q < FR_NCAT; ++q) {
        uint32_t b = pre.c[q];
        for (int w = 0; w < warp; ++w) b += swc[w][q];
        run[q] = b;
    }
    uint32_t carry = pre.lastchg;
    for (int w = 0; w < warp; ++w) carry = swc[w][FR_NCAT] > carry ? swc[w][FR_NCAT] : carry;
#pragma unroll
    for (int k = 0; k < FR_ITEMS; ++k) {
        const size_t i = wb + 32 * k;
#pragma unroll
        for (int q = 1; q < FR_NCAT; ++q) {
            const uint32_t m = __ballot_sync(0xffffffffu, (fl[k] >> q) & 1u);
            if (out.list[q] && ((fl[k] >> q) & 1u)) {
                out.list[q][run[q] + __popc(m & lt)] = (uint32_t)i;
                if (q == 1 && out.hd)  // (the columns were just read: cached)
                    out.hd[run[q] + __popc(m & lt)] = ((uint64_t)(uint32_t)c.src[i] << 32) | (uint32_t)c.dst[i];
            }
            run[q] += __popc(m);
        }
        if (out.srank) {
            uint32_t v = (fl[k] & 64u) ? (uint32_t)i : 0u;
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, v, off);
                if (lane >= off) v = y > v ? y : v;
            }
            v = v > carry ? v : carry;
            if (i <= last) out.srank[i] = v;
            carry = __shfl_sync(0xffffffffu, v, 31);
        }
    }
}

// ============================================================ helpers
template <class F>
__global__ void k_for(size_t n, F f) {
    pdl_enter();
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) f(i);
}
template <class F>
void for_each(size_t n, F f, cudaStream_t s) {
    if (!n) return;
    launch_k(k_for<F>, grid_for(n, TPB), TPB, 0, s, n, f);
}

// Read a device u32 count (one sync).
uint32_t read_u32(const uint32_t *d, cudaStream_t s, int line = __builtin_LINE()) {
    uint32_t v = 0;
    read_back(&v, d, sizeof(v), s, line);
    return v;
}

// Segment heads of sorted keys.
template <int KW>
struct HeadPred {
    KeyCols<KW> k;
    __device__ bool operator()(size_t p) const {
        if (p == 0) return true;
#pragma unroll
        for (int w = 0; w < KW; ++w)
            if (k.w[w][p] != k.w[w][p - 1]) return true;
        return false;
    }
};

template <int KW>
struct HeadLoad {
    KeyCols<KW> k;
    __device__ uint32_t operator()(size_t p) const { return HeadPred<KW>{k}(p) ? 1u : 0u; }
};
struct SegStartStore {  // over head flags: segment id per position, start position per segment
    uint32_t *seg_of, *seg_start;
    uint32_t n;  // seg_start[#segments] = n is written by the last position
    __device__ void operator()(size_t i, uint32_t ex, uint32_t it) const {
        const uint32_t sg = ex + it - 1;
        seg_of[i] = sg;
        if (it) seg_start[sg] = (uint32_t)i;
        if (i + 1 == n) seg_start[sg + 1] = n;
    }
};
struct StoreInclMinus1 {
    uint32_t *o;
    __device__ void operator()(size_t i, uint32_t ex, uint32_t it) const { o[i] = ex + it - 1; }
};

// Group ordering: stable sort of group ids by the start time of each group's first
// event (ties keep the key order the groups were produced in) -- detectors.py:102,166,180.
struct GroupOrder {
    DBuf<uint32_t> order;  // final rank -> group id
    DBuf<uint32_t> rank;   // group id -> final rank
};
struct FirstStartKey {
    const uint32_t *srank;
    const uint32_t *first_event;
    uint64_t *key;
    uint32_t *val;
    __device__ void operator()(size_t g) const {
        key[g] = srank[first_event[g]];
        val[g] = (uint32_t)g;
    }
};
// Groups in key order: a stable sort by the start of their first event (as the rank of the first
// event with that start -- equal starts, equal ranks) gives the reference's (start, key...) order.
// Groups produced in another order pass `tie` (per group, ascending in the reference's key order)
// and are sorted by (start rank, tie).
GroupOrder order_groups(size_t ng, const uint64_t *start, const uint32_t *first_event, cudaStream_t s,
                        const uint64_t *tie = nullptr, uint64_t tie_bound = 0) {
    (void)start;
    GroupOrder go;
    go.order.alloc(ng ? ng : 1, s);
    go.rank.alloc(ng ? ng : 1, s);
    if (!ng) return go;
    const uint32_t *ordp;
    const bool narrow = !tie || bit_width(tie_bound) + bit_width(g_masks.n) <= 64;
    SortStore<1> st(narrow ? ng : 1, s);
    SortStore<2> st2(narrow ? 1 : ng, s);
    if (!tie) {
        for_each(ng, FirstStartKey{g_masks.srank, first_event, st.in_key(0), st.in_val()}, s);
        radix_sort<1>(st.b, ng, LiveBytes<1>{{g_masks.idx}}, s);
        ordp = st.val();
    } else if (bit_width(tie_bound) + bit_width(g_masks.n) <= 64) {
        // one key: start rank << tie bits | tie; LSD over the bytes holding the start rank, then
        // the segmented fix-up of equal-start runs (usually single groups)
        const int tb = bit_width(tie_bound);
        uint64_t *k0 = st.in_key(0);
        uint32_t *v = st.in_val();
        const uint32_t *sr = g_masks.srank, *fe = first_event;
        for_each(ng, [=] __device__(size_t g) {
            k0[g] = ((uint64_t)sr[fe[g]] << tb) | tie[g];
            v[g] = (uint32_t)g;
        }, s);
        radix_sort_prefix(st.b, ng, live_range((uint64_t)g_masks.n << tb), tb / 8, s);
        ordp = st.val();
    } else {
        for_each(ng, FirstStartKey{g_masks.srank, first_event, st2.in_key(0), st2.in_val()}, s);
        dev_copy(st2.in_key(1), tie, ng * sizeof(uint64_t), s);
        radix_sort<2>(st2.b, ng, LiveBytes<2>{{g_masks.idx, live_range(tie_bound)}}, s);
        ordp = st2.val();
    }
    dev_copy(go.order.p, ordp, ng * sizeof(uint32_t), s);
    uint32_t *ord = go.order.p, *rk = go.rank.p;
    for_each(ng, [=] __device__(size_t r) { rk[ord[r]] = (uint32_t)r; }, s);
    return go;
}

// Offsets of groups in final order from per-group sizes: off[r] = sum of sizes of ranks < r.
struct SizeByRank {
    const uint32_t *order;
    const uint32_t *size;
    __device__ uint64_t operator()(size_t r) const { return size[order[r]]; }
};
struct StoreOffset {
    uint64_t *off;
    __device__ void operator()(size_t r, uint64_t ex, uint64_t) const { off[r] = ex; }
};

// ============================================================ output container
void stream_after(cudaStream_t to, cudaStream_t from);
cudaStream_t engine_stream_n(int k);
struct HostSlab;
struct Internal {
    // the device findings of the call (first member: released after every buffer carved from it).
    // Sized from the partition counts' upper bounds (~30 B/event at most), so a live findings
    // object keeps only its results; the call's scratch arena is released when analyze returns.
    Arena keep;
    template <class T>
    void own(DBuf<T> &b, size_t n, cudaStream_t s) {
        ArenaUse au(&keep);
        b.alloc(n, s);
    }
    HostSlab *slab = nullptr;  // pinned host memory behind the b2l_findings arrays
    HostSlab *slab_pairs = nullptr, *slab_kern = nullptr, *slab_dd = nullptr;  // ... of the other chains
    // device copies of the trace columns (when they were uploaded from host) and their identity
    ColsUpload cols;
    const void *cols_key[3] = {nullptr, nullptr, nullptr};
    uint64_t cols_n = 0;
    // device copies of findings (for b2l_savings)
    DBuf<uint64_t> dd_off, rt_off, ra_off;
    DBuf<uint32_t> dd_mem, rt_tx, rt_rx, pair_alloc, pair_delete, ra_mem, ua, ut;
    uint64_t dd_groups = 0, dd_members = 0, rt_groups = 0, rt_trips = 0, ra_groups = 0, ra_members = 0;
    uint64_t n_pairs = 0, n_ua = 0, n_ut = 0, synth_end = 0;
    // savings computed by a fused analyze (B2L_ANALYZE_WITH_SAVINGS), handed to the first
    // b2l_savings_compute of the same columns
    b2l_savings *fused = nullptr;
    const void *fused_key[3] = {nullptr, nullptr, nullptr};
    uint64_t fused_n = 0;
};

template <class T>
T *host_copy(const T *d, size_t n, cudaStream_t s) {
    T *h = (T *)malloc((n ? n : 1) * sizeof(T));
    if (!h) throw EngineErr{B2L_E_OOM, "host allocation failed"};
    if (n) read_back(h, d, n * sizeof(T), s);
    return h;
}
// Many device->host result copies straight into one pinned slab with a single synchronisation.
struct HostSlab {
    uint8_t *p = nullptr;
    size_t cap = 0;
    ~HostSlab() { slab_pool().release(p, cap); }
};
// Segments packed into one staging block (HostBatch::flush_async): segment k at off[k].
struct PackSegs {
    static constexpr int MAX = 16;
    const uint8_t *src[MAX];
    size_t off[MAX], bytes[MAX];
    int n;
};
__global__ void k_pack_segs(PackSegs ps, uint8_t *__restrict__ dst) {
    pdl_enter();
    const size_t tid = (size_t)blockIdx.x * blockDim.x + threadIdx.x, stride = (size_t)gridDim.x * blockDim.x;
    for (int k = 0; k < ps.n; ++k) {
        const uint8_t *src = ps.src[k];
        uint8_t *d = dst + ps.off[k];
        const size_t b = ps.bytes[k];
        if ((((uintptr_t)src | (uintptr_t)d) & 15) == 0) {
            const size_t nv = b / 16;
            for (size_t i = tid; i < nv; i += stride) reinterpret_cast<uint4 *>(d)[i] = reinterpret_cast<const uint4 *>(src)[i];
            for (size_t i = nv * 16 + tid; i < b; i += stride) d[i] = src[i];
        } else {
            for (size_t i = tid; i < b; i += stride) d[i] = src[i];
        }
    }
}
struct HostBatch {
    struct Item {
        void **dst;
        const void *src;
        size_t bytes;
    };
    std::vector<Item> items;
    template <class T>
    void add(T **dst, const T *d, size_t n) {
        items.push_back(Item{(void **)dst, d, n * sizeof(T)});
    }
    // Queue the copies on `copy` once everything queued so far on `after` is done, into a fresh
    // slab; no synchronisation (the caller synchronises `copy` before reading).  Several arrays
    // are first packed (one kernel on `after`) into a device staging block laid out like the
    // slab, so the batch is ONE device->host copy instead of one per array (each costs the copy
    // engine ~5 us).  The staging block comes from the call's arena (the caller synchronises
    // `copy` before the arena is released).
    void flush_async(HostSlab &slab, cudaStream_t after, cudaStream_t copy) {
        size_t total = 0;
        for (auto &it : items) total += (it.bytes + 63) & ~size_t(63);
        slab.p = slab_pool().acquire(total, slab.cap);
        uint8_t *stage = items.size() > 1 && items.size() <= PackSegs::MAX && t_arena
                             ? static_cast<uint8_t *>(t_arena->take(total))
                             : nullptr;
        if (stage) {
            PackSegs ps{};
            size_t off = 0;
            for (auto &it : items) {
                ps.src[ps.n] = static_cast<const uint8_t *>(it.src), ps.off[ps.n] = off, ps.bytes[ps.n++] = it.bytes;
                *it.dst = slab.p + off;
                off += (it.bytes + 63) & ~size_t(63);
            }
            launch_k(k_pack_segs, grid_for(total / 16 + 1, 256, 148 * 4), 256, 0, after, ps, stage);
            stream_after(copy, after);
            to_host_async(slab.p, stage, total, copy);
            items.clear();
            return;
        }
        stream_after(copy, after);
        size_t off = 0;
        for (auto &it : items) {
            to_host_async(slab.p + off, it.src, it.bytes, copy);
            *it.dst = slab.p + off;
            off += (it.bytes + 63) & ~size_t(63);
        }
        items.clear();
    }
    void flush(HostSlab &slab, cudaStream_t s) {
        size_t total = 0;
        for (auto &it : items) total += (it.bytes + 63) & ~size_t(63);
        slab.p = slab_pool().acquire(total, slab.cap);
        size_t off = 0;
        for (auto &it : items) {
            to_host_async(slab.p + off, it.src, it.bytes, s);
            *it.dst = slab.p + off;
            off += (it.bytes + 63) & ~size_t(63);
        }
        stream_wait(s);
        items.clear();
    }
};

// B2L_TRACE=1: synchronise after each phase and print its wall time (diagnostics only).
// B2L_TRACE=ev: no synchronisation; each mark records a timing event on its stream and the host
// time it was queued, printed side by side when the call ends (ev_log_flush): where the GPU waits
// for the host and where the host waits for the GPU.
struct EvLog {
    struct Rec {
        const char *name;
        std::chrono::steady_clock::time_point host;
        cudaEvent_t ev;
        cudaStream_t s;
    };
    std::mutex mu;
    std::vector<Rec> recs;
};
inline EvLog &ev_log() {
    static EvLog l;
    return l;
}
inline int trace_mode() {
    static const int m = getenv("B2L_TRACE") ? (strcmp(getenv("B2L_TRACE"), "ev") == 0 ? 2 : 1) : 0;
    return m;
}
void ev_log_flush() {
    if (trace_mode() != 2) return;
    EvLog &l = ev_log();
    std::lock_guard<std::mutex> g(l.mu);
    if (l.recs.empty()) return;
    for (auto &r : l.recs) cudaEventSynchronize(r.ev);
    std::sort(l.recs.begin(), l.recs.end(), [](const EvLog::Rec &a, const EvLog::Rec &b) { return a.host < b.host; });
    const auto h0 = l.recs[0].host;
    const cudaEvent_t g0 = l.recs[0].ev;
    for (auto &r : l.recs) {
        float ms = 0;
        cudaEventElapsedTime(&ms, g0, r.ev);
        fprintf(stderr, "[b2l-ev] %-14s host %8.1f us  gpu %8.1f us  stream %p\n", r.name,
                std::chrono::duration<double, std::micro>(r.host - h0).count(), ms * 1e3, (void *)r.s);
    }
    for (auto &r : l.recs) cudaEventDestroy(r.ev);
    l.recs.clear();
}
struct PhaseClock {
    int on;
    cudaStream_t s;
    std::chrono::steady_clock::time_point t;
    explicit PhaseClock(cudaStream_t st) : on(trace_mode()), s(st), t(std::chrono::steady_clock::now()) {}
    void mark(const char *name) {
        if (!on) return;
        if (on == 2) {
            cudaEvent_t e;
            cudaEventCreate(&e);
            cudaEventRecord(e, s);
            EvLog &l = ev_log();
            std::lock_guard<std::mutex> g(l.mu);
            l.recs.push_back({name, std::chrono::steady_clock::now(), e, s});
            return;
        }
        cudaStreamSynchronize(s);
        auto now = std::chrono::steady_clock::now();
        fprintf(stderr, "[b2l] %-12s %8.3f ms\n", name, std::chrono::duration<double, std::milli>(now - t).count());
        t = now;
    }
};

// ============================================================ DD + RT (detectors.py:85-167)
struct RtRecordInit {  // record r = 2k + role over hashed transfer k: role 0 = reception, 1 = send
    DevCols c;            // generated in hash-rank order (q = 2p + role over hash-sorted position p)
    const uint32_t *H, *hsv, *hidp;  // hsv[p]: transfer at sorted position p; hidp[p]: its hash rank
    const uint64_t *hd;              // (src << 32 | dst) per hashed transfer (front pass) or nullptr
    uint64_t *k0;                    // key = device << 32 | rank: queues (device, hash)
    uint32_t *val;
    __device__ void operator()(size_t q) const {
        const size_t p = q >> 1;
        const uint32_t role = (uint32_t)(q & 1), k = hsv[p];
        uint32_t dev;
        if (hd) {  // one gather per record instead of three (H[k], then src or dst)
            const uint64_t sd = hd[k];
            dev = role ? (uint32_t)(sd >> 32) : (uint32_t)sd;
        } else {
            const uint32_t e = H[k];
            dev = (uint32_t)(role ? c.src[e] : c.dst[e]);
        }
        k0[q] = ((uint64_t)dev << 32) | hidp[p];
        val[q] = 2 * k + role;
    }
};
struct StoreHid {  // hash rank per sorted position and per hashed transfer
    const uint32_t *sval;
    uint32_t *hidp, *hid;
    __device__ void operator()(size_t p, uint32_t ex, uint32_t it) const {
        const uint32_t v = ex + it - 1;
        hidp[p] = v;
        hid[sval[p]] = v;
    }
};

// Per sorted record: segment head, reception/send counts (segmented + global).
struct QState {
    uint32_t head, seg, rx_seg, tx_seg, rx_glob;
};
struct QOp {
    using T = QState;
    static __device__ __forceinline__ T identity() { return T{0, 0, 0, 0, 0}; }
    static __device__ __forceinline__ T combine(T a, T b) {
        return T{a.head | b.head, a.seg + b.seg, b.head ? b.rx_seg : a.rx_seg + b.rx_seg,
                 b.head ? b.tx_seg : a.tx_seg + b.tx_seg, a.rx_glob + b.rx_glob};
    }
};
struct QLoad {
    const uint64_t *k;
    const uint32_t *val;
    __device__ QState operator()(size_t p) const {
        const bool head = p == 0 || k[p] != k[p - 1];
        const uint32_t rx = (val[p] & 1u) == 0;
        return QState{head, head, rx, 1u - rx, rx};
    }
};
struct QStore {
    const uint32_t *val;
    uint32_t *seg_of, *f_of, *j_of, *rxpos, *seg_start, *seg_rxbase;
    __device__ void operator()(size_t p, QState ex, QState it) const {
        const uint32_t seg = ex.seg + it.seg - 1;
        seg_of[p] = seg;
        const uint32_t f = it.head ? 0 : ex.rx_seg, j = it.head ? 0 : ex.tx_seg;
        f_of[p] = f;
        j_of[p] = j;
        if (it.head) {
            seg_start[seg] = (uint32_t)p;
            seg_rxbase[seg] = ex.rx_glob;
        }
        if ((val[p] & 1u) == 0) rxpos[ex.rx_glob] = (uint32_t)p;
    }
};
// r_j = j + max_{i<=j}(f_i - i) over the sends of one queue
struct RtMaxLoad {
    const uint64_t *k;
    const uint32_t *val, *f_of, *j_of;
    __device__ Seg<MaxI64>::T operator()(size_t p) const {
        const bool head = p == 0 || k[p] != k[p - 1];
        const bool tx = val[p] & 1u;
        return Seg<MaxI64>::T{head ? 1u : 0u, tx ? (long long)f_of[p] - (long long)j_of[p] : MaxI64::identity()};
    }
};
struct RtMatchStore {
    const uint32_t *val, *j_of, *seg_of, *seg_rxbase, *rxpos, *H;
    uint32_t *match;  // per hashed-transfer k: reception event or NONE
    __device__ void operator()(size_t p, Seg<MaxI64>::T ex, Seg<MaxI64>::T it) const {
        if (!(val[p] & 1u)) return;
        const long long pm = it.flag ? it.v : MaxI64::combine(ex.v, it.v);
        const long long r = (long long)j_of[p] + pm;
        const uint32_t seg = seg_of[p];
        const long long nrx = (long long)seg_rxbase[seg + 1] - (long long)seg_rxbase[seg];
        if (r < nrx) match[val[p] >> 1] = H[val[rxpos[seg_rxbase[seg] + r]] >> 1];
    }
};

// Strict pseudocode (detectors.py:139-160): per hash, sends in trace order peek the
// (hash, src) queue and pop the (hash, dst) queue.  Queues of one hash interact, so one
// thread walks each hash's events; different hashes run in parallel.
__device__ __forceinline__ int find_seg(const uint64_t *sk, uint32_t nseg, uint64_t key) {
    uint32_t lo = 0, hi = nseg;
    while (lo < hi) {
        uint32_t mid = (lo + hi) >> 1;
        if (sk[mid] < key)
            lo = mid + 1;
        else
            hi = mid;
    }
    return (lo < nseg && sk[lo] == key) ? (int)lo : -1;
}
__global__ void k_rt_strict(DevCols c, const uint32_t *H, const uint32_t *hsorted /*hashed-k sorted by hash*/,
                            const uint32_t *hseg_start, uint32_t nhseg, uint32_t nH, const uint32_t *hid,
                            const uint64_t *segk, uint32_t nseg, const uint32_t *seg_rxbase, const uint32_t *rxpos,
                            const uint32_t *sval, uint32_t *qhead, uint32_t *match) {
    pdl_enter();
    for (uint32_t g = blockIdx.x * blockDim.x + threadIdx.x; g < nhseg; g += gridDim.x * blockDim.x) {
        const uint32_t b = hseg_start[g], e = (g + 1 < nhseg) ? hseg_start[g + 1] : nH;
        for (uint32_t q = b; q < e; ++q) {
            const uint32_t k = hsorted[q];
            const uint32_t ev = H[k];
            const uint64_t hk = hid[k];
            const int sq = find_seg(segk, nseg, hk | ((uint64_t)(uint32_t)c.src[ev] << 32));
            if (sq < 0) continue;
            const uint32_t nrx = seg_rxbase[sq + 1] - seg_rxbase[sq];
            if (qhead[sq] >= nrx) continue;  // `if not q: continue`
            match[k] = H[sval[rxpos[seg_rxbase[sq] + qhead[sq]]] >> 1];
            const int so = find_seg(segk, nseg, hk | ((uint64_t)(uint32_t)c.dst[ev] << 32));
            if (so >= 0 && qhead[so] < seg_rxbase[so + 1] - seg_rxbase[so]) qhead[so] += 1;
        }
    }
}

// Persistent host workers for the side chains (spawning three threads per call cost tens of µs).
// Calls are serialised by g_mu, so at most three tasks are in flight; the pool is never torn down.
class Workers {
   public:
    explicit Workers(int n) {
        for (int i = 0; i < n; ++i) std::thread([this] { loop(); }).detach();
    }
    std::future<void> submit(std::function<void()> f) {
        auto task = std::make_shared<std::packaged_task<void()>>(std::move(f));
        std::future<void> fu = task->get_future();
        {
            std::lock_guard<std::mutex> l(m_);
            q_.emplace_back([task] { (*task)(); });
        }
        cv_.notify_one();
        return fu;
    }

   private:
    void loop() {
        for (;;) {
            std::function<void()> f;
            {
                std::unique_lock<std::mutex> l(m_);
                cv_.wait(l, [&] { return !q_.empty(); });
                f = std::move(q_.front());
                q_.pop_front();
            }
            f();
        }
    }
    std::mutex m_;
    std::condition_variable cv_;
    std::deque<std::function<void()>> q_;
};
inline Workers &workers() {
    static Workers *w = new Workers(4);
    return *w;
}

struct DdRt {
    uint64_t dd_groups = 0, rt_groups = 0, dd_members = 0, rt_trips = 0;
};

cudaStream_t engine_stream_n(int k);
void stream_after(cudaStream_t to, cudaStream_t from);

DdRt dd_rt_step(const DevCols &c, const uint32_t *H, const uint64_t *HD, uint32_t nH, bool strict, Internal &out,
                cudaStream_t s,
                b2l_findings *f = nullptr, cudaStream_t sc = nullptr) {
    DdRt r;
    const size_t R = 2ull * nH;
    if (nH == 0) {
        out.own(out.dd_off, 1, s), out.dd_off.zero(), out.own(out.dd_mem, 1, s);
        out.own(out.rt_off, 1, s), out.rt_off.zero(), out.own(out.rt_tx, 1, s), out.own(out.rt_rx, 1, s);
        return r;
    }
    PhaseClock pc(s);
    // ---- hashed transfers in hash order (stable) -> dense hash rank per transfer, so the
    // (hash, device) record sort runs on one narrow key: rank << db | device
    SortStore<1> hsort(nH, s);
    {
        uint64_t *k0 = hsort.in_key(0);
        uint32_t *v = hsort.in_val();
        const uint64_t *hh = c.h;
        for_each(nH, [=] __device__(size_t k) { k0[k] = hh[H[k]], v[k] = (uint32_t)k; }, s);
    }
    radix_sort_wide(hsort.b, nH, g_masks.hash, s);
    KeyCols<1> hk = hsort.b.k[hsort.b.cur];
    DBuf<uint32_t> hid(nH, s), hidp(nH, s);
    scan<SumU32>(nH, HeadLoad<1>{hk}, StoreHid{hsort.val(), hidp.p, hid.p}, s);
    int db = 0;
    while (db < 32 && (1ull << db) < (uint64_t)(c.ndev > 0 ? c.ndev : 1)) ++db;
    pc.mark(" hash-rank");
    // records generated in hash-rank order, then one stable pass over the device byte(s): queues
    // come out in (device, hash) order, trace order inside.  Group orders that break start ties by
    // the reference's (hash, device...) key take explicit tie keys below.
    SortStore<1> st(R, s);
    for_each(R, RtRecordInit{c, H, hsort.val(), hidp.p, HD, st.in_key(0), st.in_val()}, s);
    pc.mark(" rt-init");
    radix_sort<1>(st.b, R, LiveBytes<1>{{(uint8_t)(g_masks.dev << 4)}}, s);
    pc.mark(" rt-sort");
    const uint64_t *sk = st.key(0);
    const uint32_t *sval = st.val();

    DBuf<uint32_t> seg_of(R, s), f_of(R, s), j_of(R, s), rxpos(R, s), seg_start(R + 1, s), seg_rxbase(R + 1, s);
    DBuf<QState> tot(1, s);
    scan<QOp>(R, QLoad{sk, sval},
              QStore{sval, seg_of.p, f_of.p, j_of.p, rxpos.p, seg_start.p, seg_rxbase.p}, s, tot.p);
    QState qt{};
    read_back(&qt, tot.p, sizeof(qt), s);
    const uint32_t nseg = qt.seg, nrx = qt.rx_glob;
    dev_copy(seg_rxbase.p + nseg, &tot.p->rx_glob, sizeof(uint32_t), s);

    pc.mark(" q-scan");
    // ---- DD groups need only the queue scan: on small traces they run on their own stream (and
    // host thread) beside the RT matching and grouping, which are latency bound there
    static const uint64_t side_min = getenv("B2L_SIDE_MIN") ? strtoull(getenv("B2L_SIDE_MIN"), nullptr, 10) : 0;
    const bool dd_side = R <= (size_t(8) << 20) && R >= side_min;
    int dev = 0;
    CK(cudaGetDevice(&dev));
    const Masks masks = g_masks;
    cudaStream_t sd = dd_side ? engine_stream_n(3) : s;
    if (dd_side) stream_after(sd, s);
    EngineErr errd{0, ""};
    bool faild = false;
    Arena *const arena = t_arena;
    auto dd_groups = [&](cudaStream_t s) {
        ArenaUse au(arena);
        try {
            CK(cudaSetDevice(dev));
            g_masks = masks;
            // ---- DD groups: queue segments with >= 2 receptions (members = the receptions, trace order)
            {
                DBuf<uint32_t> gseg(nseg, s), gcount(1, s);
                const uint32_t *rb = seg_rxbase.p;
                compact(nseg, [=] __device__(size_t g) { return rb[g + 1] - rb[g] >= 2; }, gseg.p, gcount.p, s);
                const uint32_t ng = read_u32(gcount.p, s);
                r.dd_groups = ng;
                DBuf<uint32_t> first_ev(ng ? ng : 1, s), gsize(ng ? ng : 1, s), seg_group(nseg, s);
                DBuf<uint64_t> tie(ng ? ng : 1, s);
                dev_memset(seg_group.p, 0xFF, nseg * sizeof(uint32_t), s);
                {
                    const uint32_t *gs = gseg.p, *rp = rxpos.p, *ss = seg_start.p;
                    uint32_t *fe = first_ev.p, *sz = gsize.p, *sgp = seg_group.p;
                    uint64_t *tk = tie.p;
                    const int dbits = db;
                    for_each(ng, [=] __device__(size_t g) {
                        const uint32_t sg = gs[g];
                        fe[g] = H[sval[rp[rb[sg]]] >> 1];
                        sz[g] = rb[sg + 1] - rb[sg];
                        sgp[sg] = (uint32_t)g;
                        const uint64_t key = sk[ss[sg]];  // dst << 32 | hash rank
                        tk[g] = ((key & 0xFFFFFFFFull) << dbits) | (key >> 32);  // reference order (hash, dst)
                    }, s);
                }
                GroupOrder go = order_groups(ng, c.start, first_ev.p, s, tie.p, (uint64_t)nH << db);
                out.own(out.dd_off, ng + 1, s);
                DBuf<uint64_t> total(1, s);
                scan<SumU64>(ng, SizeByRank{go.order.p, gsize.p}, StoreOffset{out.dd_off.p}, s, total.p);
                if (ng) dev_copy(out.dd_off.p + ng, total.p, sizeof(uint64_t), s);
                else dev_memset(out.dd_off.p, 0, sizeof(uint64_t), s);
                out.own(out.dd_mem, nrx ? nrx : 1, s);  // members are receptions; count read after the scatter
                // every reception of a grouped segment lands at off[rank] + (its rank within the segment)
                const uint32_t *sgp = seg_group.p, *rk = go.rank.p, *so = seg_of.p, *rp = rxpos.p;
                const uint64_t *off = out.dd_off.p;
                uint32_t *mem = out.dd_mem.p;
                for_each(nrx, [=] __device__(size_t q) {
                    const uint32_t p = rp[q];
                    const uint32_t sg = so[p];
                    const uint32_t g = sgp[sg];
                    if (g == NONE) return;
                    mem[off[rk[g]] + (q - rb[sg])] = H[sval[p] >> 1];
                }, s);
                uint64_t nm = 0;
                if (ng) read_back(&nm, total.p, sizeof(nm), s);
                r.dd_members = nm;
                if (f && sc) {  // the DD results go to the host while RT still runs
                    HostBatch hb;
                    hb.add(&f->dd_offsets, (const uint64_t *)out.dd_off.p, (size_t)ng + 1);
                    hb.add(&f->dd_members, (const uint32_t *)out.dd_mem.p, (size_t)nm);
                    out.slab_dd = new HostSlab();
                    hb.flush_async(*out.slab_dd, s, sc);
                }
            }
            if (dd_side) stream_wait(s);
        } catch (const EngineErr &e) {
            errd = e;
            faild = true;
        }
    };
    std::future<void> td;
    if (dd_side) td = workers().submit([&] { dd_groups(sd); });
    else dd_groups(s);
    auto rt_groups = [&] {
        // ---- round trips: per send, the matched reception (or NONE)
        DBuf<uint32_t> match(nH, s);
        dev_memset(match.p, 0xFF, nH * sizeof(uint32_t), s);
        if (!strict) {
            scan<Seg<MaxI64>>(R, RtMaxLoad{sk, sval, f_of.p, j_of.p},
                              RtMatchStore{sval, j_of.p, seg_of.p, seg_rxbase.p, rxpos.p, H, match.p}, s);
        } else {
            DBuf<uint64_t> segk(nseg, s);
            {
                const uint32_t *ss = seg_start.p;
                uint64_t *a = segk.p;
                for_each(nseg, [=] __device__(size_t g) { a[g] = sk[ss[g]]; }, s);
            }
            // hashed transfers grouped by hash, trace order within a hash: the hash sort above
            DBuf<uint32_t> hstart(nH, s), hcount(1, s);
            compact(nH, HeadPred<1>{hk}, hstart.p, hcount.p, s);
            const uint32_t nhseg = read_u32(hcount.p, s);
            DBuf<uint32_t> qhead;
            qhead.alloc_zeroed(nseg, s);
            k_rt_strict<<<grid_for(nhseg, 128), 128, 0, s>>>(c, H, hsort.val(), hstart.p, nhseg, nH, hid.p, segk.p,
                                                             nseg, seg_rxbase.p, rxpos.p, sval, qhead.p, match.p);
            CK_LAUNCH("k_rt_strict");
        }

        pc.mark(" rt-match");
        // ---- RT groups: matched sends keyed (hash, src, dst); sends of one (hash, src) queue are
        // already in trace order in the record sort, so a stable sort by (queue segment, dst) groups them
        {
            DBuf<uint32_t> mpos(R, s), mcount(1, s);
            uint32_t *mt = match.p;
            compact(R, [=] __device__(size_t p) { return (sval[p] & 1u) && mt[sval[p] >> 1] != NONE; }, mpos.p,
                    mcount.p, s);
            const uint32_t nt = read_u32(mcount.p, s);
            r.rt_trips = nt;
            out.own(out.rt_tx, nt ? nt : 1, s);
            out.own(out.rt_rx, nt ? nt : 1, s);
            if (nt == 0) {
                out.own(out.rt_off, 1, s), out.rt_off.zero();
                return;
            }
            SortStore<1> ts(nt, s);
            {
                uint64_t *k0 = ts.in_key(0);
                uint32_t *v = ts.in_val();
                const uint32_t *mp = mpos.p, *so = seg_of.p;
                const int32_t *dst = c.dst;
                for_each(nt, [=] __device__(size_t t) {
                    const uint32_t p = mp[t];
                    k0[t] = ((uint64_t)so[p] << 32) | (uint32_t)dst[H[sval[p] >> 1]];
                    v[t] = p;
                }, s);
            }
            // trips come in record order, i.e. already ordered by queue: only runs of one queue need
            // ordering by dst (stable) -- the segmented fix-up, no digit passes
            seg_fixup(ts.b, nt, 32, (uint8_t)(g_masks.dev | (live_range(nseg) << 4)), s);
            KeyCols<1> tk = ts.b.k[ts.b.cur];
            const uint32_t *tv = ts.val();
            // one scan: group id of every sorted trip and the first trip of every group
            DBuf<uint32_t> gstart(nt + 1, s), gcount(1, s), trip_group(nt, s);
            scan<SumU32>(nt, HeadLoad<1>{tk}, SegStartStore{trip_group.p, gstart.p, nt}, s, gcount.p);
            const uint32_t ng = read_u32(gcount.p, s);
            r.rt_groups = ng;
            DBuf<uint32_t> first_ev(ng, s), gsize(ng, s);
            DBuf<uint64_t> tie(ng, s);
            {
                const uint32_t *gs = gstart.p;
                uint32_t *fe = first_ev.p, *sz = gsize.p;
                uint64_t *tk = tie.p;
                const uint32_t ntt = nt;
                const int dbits = db;
                const int32_t *dst = c.dst;
                for_each(ng, [=] __device__(size_t g) {
                    const uint32_t p = tv[gs[g]], e = H[sval[p] >> 1];
                    fe[g] = e;
                    sz[g] = ((g + 1 < ng) ? gs[g + 1] : ntt) - gs[g];
                    const uint64_t key = sk[p];  // src << 32 | hash rank
                    // reference order (hash, src, dst)
                    tk[g] = ((((key & 0xFFFFFFFFull) << dbits) | (key >> 32)) << dbits) | (uint64_t)(uint32_t)dst[e];
                }, s);
            }
            GroupOrder go = order_groups(ng, c.start, first_ev.p, s, tie.p, (uint64_t)nH << (2 * db));
            out.own(out.rt_off, ng + 1, s);
            DBuf<uint64_t> total(1, s);
            scan<SumU64>(ng, SizeByRank{go.order.p, gsize.p}, StoreOffset{out.rt_off.p}, s, total.p);
            dev_copy(out.rt_off.p + ng, total.p, sizeof(uint64_t), s);
            const uint32_t *tg = trip_group.p, *rk = go.rank.p, *gs = gstart.p;
            const uint64_t *off = out.rt_off.p;
            uint32_t *otx = out.rt_tx.p, *orx = out.rt_rx.p;
            for_each(nt, [=] __device__(size_t t) {
                const uint32_t g = tg[t];
                const uint64_t o = off[rk[g]] + (t - gs[g]);
                const uint32_t k = sval[tv[t]] >> 1;
                otx[o] = H[k];
                orx[o] = mt[k];
            }, s);
        }
    };
    try {
        rt_groups();
    } catch (...) {
        if (td.valid()) td.wait();
        throw;
    }
    if (td.valid()) td.wait();
    if (faild) throw errd;
    pc.mark(" dd-rt-groups");
    return r;
}


// ============================================================ LIFO pairing (prep.py:45-96)
struct UmPred {
    const uint8_t *um;
    __device__ bool operator()(size_t r) const { return um[r] != 0; }
};
template <class Pred>
struct MapCompactStore {  // compaction that stores map[i] instead of i
    Pred p;
    const uint32_t *map;
    uint32_t *out;
    __device__ __forceinline__ void operator()(size_t i, uint32_t ex, uint32_t item) const {
        if (item) out[ex] = map[i];
    }
};
struct PairOut {
    uint32_t n_pairs = 0, n_warn = 0;
    DBuf<uint32_t> wcount;  // device count of warnings (read at the end of the chain)
    DBuf<uint32_t> warn;  // unmatched deletes, trace order
};
// inclusive depth after an element from its (exclusive prefix, item) of the max-plus scan
__device__ __forceinline__ long long depth_of(const MaxPlus::T &f) { return f.a > f.b ? f.a : f.b; }
struct DepthLoad {
    KeyCols<2> k;
    const uint32_t *val, *AD;
    const uint8_t *kind;
    __device__ Seg<MaxPlus>::T operator()(size_t p) const {
        const bool head = p == 0 || k.w[0][p] != k.w[0][p - 1] || k.w[1][p] != k.w[1][p - 1];
        const bool is_alloc = kind[AD[val[p]]] == B2L_KIND_ALLOC;
        // alloc: d -> d + 1 ; delete: d -> max(d - 1, 0)
        MaxPlus::T f = is_alloc ? MaxPlus::T{1, MaxPlus::identity().b} : MaxPlus::T{-1, 0};
        return Seg<MaxPlus>::T{head ? 1u : 0u, f};
    }
};
struct DepthStore {  // level (>= 1) of allocs and matched deletes, 0 for unmatched deletes
    const uint32_t *val, *AD;
    const uint8_t *kind;
    uint32_t *level;
    __device__ void operator()(size_t p, Seg<MaxPlus>::T ex, Seg<MaxPlus>::T it) const {
        const long long before = it.flag ? 0 : depth_of(ex.v);
        const bool is_alloc = kind[AD[val[p]]] == B2L_KIND_ALLOC;
        level[p] = is_alloc ? (uint32_t)(before + 1) : (uint32_t)before;  // delete at depth 0: unmatched
    }
};

// Unmatched deletes (level 0) flagged by AD rank, and the largest level (block max, one atomic per
// block) so the (segment, level) sort key can be packed to its exact width.
__global__ void k_pair_unmatched(size_t n, const uint32_t *sv, const uint32_t *AD, const uint8_t *kind,
                                 const uint32_t *lv, uint8_t *um, unsigned *maxlv) {
    pdl_enter();
    __shared__ unsigned bm;
    if (threadIdx.x == 0) bm = 0;
    __syncthreads();
    unsigned m = 0;
    for (size_t p = (size_t)blockIdx.x * blockDim.x + threadIdx.x; p < n; p += (size_t)gridDim.x * blockDim.x) {
        const uint32_t l = lv[p];
        m = l > m ? l : m;
        if (l == 0 && kind[AD[sv[p]]] == B2L_KIND_DELETE) um[sv[p]] = 1;
    }
    m = __reduce_max_sync(0xffffffffu, m);
    if ((threadIdx.x & 31) == 0 && m) atomicMax(&bm, m);
    __syncthreads();
    if (threadIdx.x == 0 && bm) atomicMax(maxlv, bm);
}

PairOut pairs_step(const DevCols &c, const uint32_t *AD, uint32_t nAD, const uint32_t *A, uint32_t nA,
                   uint64_t synth_end, Internal &out, cudaStream_t s) {
    PairOut po;
    po.n_pairs = nA;
    out.own(out.pair_alloc, nA ? nA : 1, s);
    out.own(out.pair_delete, nA ? nA : 1, s);
    if (nA) dev_copy(out.pair_alloc.p, A, nA * sizeof(uint32_t), s);
    if (nA) dev_memset(out.pair_delete.p, 0xFF, nA * sizeof(uint32_t), s);  // synthetic unless matched
    po.warn.alloc(nAD ? nAD : 1, s);
    if (nAD == 0) return po;
    // event -> allocation rank (pairs are in allocation order, prep.py:95)
    DBuf<uint32_t> arank(c.n, s);
    {
        uint32_t *ar = arank.p;
        for_each(nA, [=] __device__(size_t r) { ar[A[r]] = (uint32_t)r; }, s);
    }
    SortStore<2> st(nAD, s);
    {
        uint64_t *k0 = st.in_key(0), *k1 = st.in_key(1);
        uint32_t *v = st.in_val();
        const int32_t *dst = c.dst;
        const uint64_t *da = c.da;
        for_each(nAD, [=] __device__(size_t r) {
            const uint32_t e = AD[r];
            k0[r] = (uint64_t)(uint32_t)dst[e];
            k1[r] = da[e];
            v[r] = (uint32_t)r;
        }, s);
    }
    radix_sort<2>(st.b, nAD, LiveBytes<2>{{g_masks.dev, g_masks.da}}, s);
    KeyCols<2> sk = st.b.k[st.b.cur];
    const uint32_t *sv = st.val();
    DBuf<uint32_t> level(nAD, s), seg(nAD, s), nseg_d(1, s), maxlv;
    maxlv.alloc_zeroed(1, s);
    scan<Seg<MaxPlus>>(nAD, DepthLoad{sk, sv, AD, c.kind}, DepthStore{sv, AD, c.kind, level.p}, s);
    scan<SumU32>(nAD, HeadLoad<2>{sk}, StoreInclMinus1{seg.p}, s, nseg_d.p);
    // unmatched deletes -> warnings in trace order (flag by AD rank, compact in AD order)
    {
        DBuf<uint8_t> unmatched;
        unmatched.alloc_zeroed(nAD, s);
        uint8_t *um = unmatched.p;
        launch_k(k_pair_unmatched, grid_for(nAD, TPB, 148 * 8), TPB, 0, s, (size_t)nAD, sv, AD, c.kind,
                 (const uint32_t *)level.p, um, maxlv.p);
        CK_LAUNCH("k_pair_unmatched");
        // compacted straight to event indices; the count is read at the end of the chain
        po.wcount.alloc(1, s);
        scan<SumU32>(nAD, FlagLoad<UmPred>{UmPred{um}}, MapCompactStore<UmPred>{UmPred{um}, AD, po.warn.p}, s,
                     po.wcount.p);
    }
    // (segment, level) sort of allocs and matched deletes: within one level of one address the
    // sequence alternates alloc, delete, alloc, ... and each alloc pairs with the delete after it
    DBuf<uint32_t> lp(nAD, s), lc(1, s);
    {
        const uint32_t *lv = level.p;
        compact(nAD, [=] __device__(size_t p) { return lv[p] != 0; }, lp.p, lc.p, s);
    }
    // one read-back sizes the sort exactly: the record count, and a key (segment << lb) | level
    // packed to the bits the segments and levels really use (typically 3 digit passes, not 6)
    uint32_t h[3];
    read_back_multi({{&h[0], lc.p, 4}, {&h[1], nseg_d.p, 4}, {&h[2], maxlv.p, 4}}, s);
    PhaseClock(s).mark(" pairs-rb");
    const uint32_t nl = h[0], nseg = h[1], maxl = h[2];
    if (nl == 0) return po;
    int lb = 0;
    while (lb < 32 && (uint64_t(1) << lb) <= maxl) ++lb;
    SortStore<1> ls(nl, s);
    {
        uint64_t *k0 = ls.in_key(0);
        uint32_t *v = ls.in_val();
        const uint32_t *lpp = lp.p, *lv = level.p, *sg = seg.p;
        for_each(nl, [=] __device__(size_t q) {
            const uint32_t p = lpp[q];
            k0[q] = ((uint64_t)sg[p] << lb) | lv[p];
            v[q] = p;
        }, s);
    }
    radix_sort<1>(ls.b, nl, LiveBytes<1>{{live_range((((uint64_t)(nseg ? nseg - 1 : 0)) << lb | maxl) + 1)}}, s);
    {
        const uint64_t *lk = ls.key(0);
        const uint32_t *lvv = ls.val();
        const uint8_t *kind = c.kind;
        const uint32_t *ar = arank.p;
        uint32_t *pd = out.pair_delete.p;
        const uint32_t nll = nl;
        for_each(nl, [=] __device__(size_t q) {
            const uint32_t e = AD[sv[lvv[q]]];
            if (kind[e] != B2L_KIND_ALLOC) return;
            if (q + 1 < nll && lk[q + 1] == lk[q]) {
                const uint32_t e2 = AD[sv[lvv[q + 1]]];
                if (kind[e2] == B2L_KIND_DELETE) pd[ar[e]] = e2;
            }
        }, s);
    }
    (void)synth_end;
    return po;
}

// ============================================================ RA (detectors.py:170-191)
void ra_step(const DevCols &c, uint32_t nP, Internal &out, cudaStream_t s) {
    out.ra_groups = out.ra_members = 0;
    if (nP < 2) {
        out.own(out.ra_off, 1, s), out.ra_off.zero(), out.own(out.ra_mem, 1, s);
        return;
    }
    const uint32_t *PA = out.pair_alloc.p;
    SortStore<3> st(nP, s);
    {
        uint64_t *k0 = st.in_key(0), *k1 = st.in_key(1), *k2 = st.in_key(2);
        uint32_t *v = st.in_val();
        const uint64_t *sa = c.sa, *nb = c.nb;
        const int32_t *dst = c.dst;
        for_each(nP, [=] __device__(size_t r) {
            const uint32_t a = PA[r];
            k0[r] = sa[a], k1[r] = (uint64_t)(uint32_t)dst[a], k2[r] = nb[a], v[r] = (uint32_t)r;
        }, s);
    }
    radix_sort<3>(st.b, nP, LiveBytes<3>{{g_masks.sa, g_masks.dev, g_masks.nb}}, s);
    KeyCols<3> sk = st.b.k[st.b.cur];
    const uint32_t *sv = st.val();
    // one scan: segment id of every sorted pair and the start of every segment; the segment count
    // stays on the device (the group compaction reads it), one synchronisation for the group count
    DBuf<uint32_t> sstart(nP + 1, s), scount(1, s), seg_of(nP, s);
    scan<SumU32>(nP, HeadLoad<3>{sk}, SegStartStore{seg_of.p, sstart.p, (uint32_t)nP}, s, scount.p);
    DBuf<uint32_t> gseg(nP, s), gc(1, s);
    const uint32_t *ss = sstart.p, *nsp = scount.p;
    compact(nP, [=] __device__(size_t g) { return g < *nsp && ss[g + 1] - ss[g] >= 2; }, gseg.p, gc.p, s);
    uint32_t cnts[2];
    {
        read_back_multi({{&cnts[0], scount.p, 4}, {&cnts[1], gc.p, 4}}, s);
    }
    PhaseClock(s).mark(" ra-rb");
    const uint32_t nseg = cnts[0], ng = cnts[1];
    out.ra_groups = ng;
    if (ng == 0) {
        out.own(out.ra_off, 1, s), out.ra_off.zero(), out.own(out.ra_mem, 1, s);
        return;
    }
    DBuf<uint32_t> first_ev(ng, s), gsize(ng, s), seg_group(nseg, s);
    dev_memset(seg_group.p, 0xFF, nseg * sizeof(uint32_t), s);
    {
        const uint32_t *gs = gseg.p;
        uint32_t *fe = first_ev.p, *sz = gsize.p, *sgp = seg_group.p;
        for_each(ng, [=] __device__(size_t g) {
            const uint32_t sg = gs[g];
            fe[g] = PA[sv[ss[sg]]];
            sz[g] = ss[sg + 1] - ss[sg];
            sgp[sg] = (uint32_t)g;
        }, s);
    }
    GroupOrder go = order_groups(ng, c.start, first_ev.p, s);
    out.own(out.ra_off, ng + 1, s);
    DBuf<uint64_t> total(1, s);
    scan<SumU64>(ng, SizeByRank{go.order.p, gsize.p}, StoreOffset{out.ra_off.p}, s, total.p);
    dev_copy(out.ra_off.p + ng, total.p, sizeof(uint64_t), s);
    out.own(out.ra_mem, nP, s);  // members <= pairs; the count is read once the scatter is queued
    const uint32_t *sgp = seg_group.p, *rk = go.rank.p, *so = seg_of.p;
    const uint64_t *off = out.ra_off.p;
    uint32_t *mem = out.ra_mem.p;
    for_each(nP, [=] __device__(size_t p) {
        const uint32_t sg = so[p];
        const uint32_t g = sgp[sg];
        if (g == NONE) return;
        mem[off[rk[g]] + (p - ss[sg])] = sv[p];
    }, s);
    uint64_t nm = 0;
    read_back(&nm, total.p, sizeof(nm), s);
    out.ra_members = nm;
}

// ============================================================ UA / UT (detectors.py:194-271)
// Kernels of the target devices, grouped by device in trace order, with PM = per-device
// prefix max of kernel ends.  The reference's forward cursor at a (non-decreasing) query
// time t is the first kernel with PM >= t.
struct KernelIndex {
    const uint64_t *kdev;  // sorted device key per kernel position
    const uint32_t *kev;   // kernel event per position
    const uint64_t *pm;
    uint32_t nk;
    const uint32_t *dlo, *dhi;  // per-device [lo, hi) when the device count is small, else null
    __device__ void range(uint64_t dev, uint32_t &lo, uint32_t &hi) const {
        if (dlo) {
            lo = dlo[dev], hi = dhi[dev];
            return;
        }
        uint32_t a = 0, b = nk;
        while (a < b) {
            uint32_t m = (a + b) >> 1;
            if (kdev[m] < dev) a = m + 1; else b = m;
        }
        lo = a;
        b = nk;
        while (a < b) {
            uint32_t m = (a + b) >> 1;
            if (kdev[m] <= dev) a = m + 1; else b = m;
        }
        hi = a;
    }
    __device__ uint32_t cursor(uint32_t lo, uint32_t hi, uint64_t t) const {
        while (lo < hi) {
            uint32_t m = (lo + hi) >> 1;
            if (pm[m] < t) lo = m + 1; else hi = m;
        }
        return lo;
    }
};
struct PmLoad {
    const uint64_t *kdev;
    const uint32_t *kev;
    const uint64_t *end;
    __device__ Seg<MaxU64>::T operator()(size_t p) const {
        return Seg<MaxU64>::T{(p == 0 || kdev[p] != kdev[p - 1]) ? 1u : 0u, end[kev[p]]};
    }
};
struct PmStore {
    uint64_t *pm;
    __device__ void operator()(size_t p, Seg<MaxU64>::T ex, Seg<MaxU64>::T it) const {
        pm[p] = Seg<MaxU64>::combine(ex, it).v;
    }
};

constexpr uint8_t CLS_GAP = 0, CLS_OVERLAP = 1, CLS_AFTER = 2;

struct RunLoad {  // run increments along one device's target transfers (trace order)
    const uint64_t *dk;  // sorted device key
    const uint32_t *dv;  // transfer rank per sorted position
    const uint32_t *cur;
    const uint8_t *cls;
    __device__ Seg<SumU32>::T operator()(size_t q) const {
        const bool head = q == 0 || dk[q] != dk[q - 1];
        uint32_t inc = 0;
        if (!head) {
            const uint32_t a = dv[q - 1], b = dv[q];
            inc = (cur[b] > cur[a] || cls[a] == CLS_OVERLAP) ? 1u : 0u;
        }
        return Seg<SumU32>::T{head ? 1u : 0u, inc};
    }
};
struct RunStore {
    const uint32_t *dv;
    uint32_t *run;
    __device__ void operator()(size_t q, Seg<SumU32>::T ex, Seg<SumU32>::T it) const {
        run[dv[q]] = Seg<SumU32>::combine(ex, it).v;
    }
};

// Target kernels grouped by device with the per-device prefix max of their ends: the cursor index
// shared by UA and UT (detectors.py:194-271).
struct KernelIndexStore {
    SortStore<1> ks;
    DBuf<uint64_t> pm;
    DBuf<uint32_t> kev, dlo, dhi;
    KernelIndex KI{};
    KernelIndexStore(uint32_t nK, cudaStream_t s) : ks(nK ? nK : 1, s), pm(nK ? nK : 1, s), kev(nK ? nK : 1, s) {}
};
void build_kernel_index(KernelIndexStore &X, const DevCols &c, const uint32_t *TK, uint32_t nK, cudaStream_t s) {
    SortStore<1> &ks = X.ks;
    DBuf<uint64_t> &pm = X.pm;
    DBuf<uint32_t> &kev = X.kev, &dlo = X.dlo, &dhi = X.dhi;
    {
        // ---- kernels grouped by device
        if (nK) {
            uint64_t *k0 = ks.in_key(0);
            uint32_t *v = ks.in_val();
            const int32_t *dst = c.dst;
            for_each(nK, [=] __device__(size_t r) { k0[r] = (uint64_t)(uint32_t)dst[TK[r]], v[r] = (uint32_t)r; }, s);
            radix_sort<1>(ks.b, nK, LiveBytes<1>{{g_masks.dev}}, s);
            uint32_t *ke = kev.p;
            const uint32_t *kv = ks.val();
            for_each(nK, [=] __device__(size_t p) { ke[p] = TK[kv[p]]; }, s);
            scan<Seg<MaxU64>>(nK, PmLoad{ks.key(0), kev.p, c.end}, PmStore{pm.p}, s);
        }
        // per-device kernel ranges (one lookup instead of two binary searches per query)
        const bool small_ndev = c.ndev > 0 && c.ndev <= (1 << 16);
        dlo.alloc_zeroed(small_ndev ? c.ndev : 1, s), dhi.alloc_zeroed(small_ndev ? c.ndev : 1, s);
        if (small_ndev) {
            uint32_t *lo = dlo.p, *hi = dhi.p;
            const uint64_t *kd = ks.key(0);
            const uint32_t nk = nK;
            for_each(nK, [=] __device__(size_t p) {
                if (p == 0 || kd[p] != kd[p - 1]) lo[kd[p]] = (uint32_t)p;
                if (p + 1 == nk || kd[p + 1] != kd[p]) hi[kd[p]] = (uint32_t)p + 1;
            }, s);
        }
        X.KI = KernelIndex{ks.key(0), kev.p, pm.p, nK, small_ndev ? dlo.p : nullptr, small_ndev ? dhi.p : nullptr};
    }
}

// UA: target pairs whose [alloc start, delete end] meets no kernel (detectors.py:194-229).
void ua_step(const DevCols &c, const KernelIndex &KI, Internal &out, cudaStream_t s) {
    {
        const uint32_t nP = (uint32_t)out.n_pairs;
        DBuf<uint32_t> ua, uc(1, s);
        out.own(ua, nP ? nP : 1, s);
        const uint32_t *PA = out.pair_alloc.p, *PD = out.pair_delete.p;
        const int32_t *dst = c.dst;
        const int host = c.host;
        const uint64_t *start = c.start, *end = c.end;
        const uint64_t se = out.synth_end;
        DBuf<uint8_t> uflag(nP ? nP : 1, s);
        uint8_t *uf = uflag.p;
        for_each(nP, [=] __device__(size_t r) {
            const uint32_t a = PA[r];
            uint8_t f = 0;
            if (dst[a] != host) {
                uint32_t lo, hi;
                KI.range((uint64_t)(uint32_t)dst[a], lo, hi);
                const uint32_t cc = KI.cursor(lo, hi, start[a]);
                const uint64_t del_end = PD[r] == NONE ? se : end[PD[r]];
                f = (cc == hi || start[KI.kev[cc]] > del_end) ? 1 : 0;
            }
            uf[r] = f;
        }, s);
        compact(nP, [=] __device__(size_t r) { return uf[r] != 0; }, ua.p, uc.p, s);
        out.n_ua = read_u32(uc.p, s);
        out.ua = std::move(ua);
    }

}

// UT (detectors.py:232-271).
void ut_step(const DevCols &c, const KernelIndex &KI, const uint32_t *TT, uint32_t nT, Internal &out,
             cudaStream_t s) {
    DBuf<uint8_t> flag;
    flag.alloc_zeroed(c.n ? c.n : 1, s);
    if (nT) {
        DBuf<uint32_t> cur(nT, s), run(nT, s);
        DBuf<uint8_t> cls(nT, s);
        {
            uint32_t *cu = cur.p;
            uint8_t *cl = cls.p, *fl = flag.p;
            const int32_t *dst = c.dst;
            const uint64_t *start = c.start;
            for_each(nT, [=] __device__(size_t t) {
                const uint32_t x = TT[t];
                uint32_t lo, hi;
                KI.range((uint64_t)(uint32_t)dst[x], lo, hi);
                const uint32_t cc = KI.cursor(lo, hi, start[x]);
                uint8_t k;
                if (cc == hi) k = CLS_AFTER;
                else if (start[KI.kev[cc]] > start[x]) k = CLS_GAP;
                else k = CLS_OVERLAP;
                cu[t] = cc;
                cl[t] = k;
                if (k == CLS_AFTER) fl[x] = 1;  // after the device's last kernel
            }, s);
        }
        SortStore<1> ds(nT, s);
        {
            uint64_t *k0 = ds.in_key(0);
            uint32_t *v = ds.in_val();
            const int32_t *dst = c.dst;
            for_each(nT, [=] __device__(size_t t) { k0[t] = (uint64_t)(uint32_t)dst[TT[t]], v[t] = (uint32_t)t; }, s);
        }
        radix_sort<1>(ds.b, nT, LiveBytes<1>{{g_masks.dev}}, s);
        scan<Seg<SumU32>>(nT, RunLoad{ds.key(0), ds.val(), cur.p, cls.p}, RunStore{ds.val(), run.p}, s);
        SortStore<2> as(nT, s);
        {
            uint64_t *k0 = as.in_key(0), *k1 = as.in_key(1);
            uint32_t *v = as.in_val();
            const int32_t *dst = c.dst;
            const uint64_t *sa = c.sa;
            for_each(nT, [=] __device__(size_t t) {
                k0[t] = (uint64_t)(uint32_t)dst[TT[t]], k1[t] = sa[TT[t]], v[t] = (uint32_t)t;
            }, s);
        }
        radix_sort<2>(as.b, nT, LiveBytes<2>{{g_masks.dev, g_masks.sa_tt}}, s);
        {
            const uint64_t *a0 = as.key(0), *a1 = as.key(1);
            const uint32_t *av = as.val(), *rn = run.p;
            const uint8_t *cl = cls.p;
            uint8_t *fl = flag.p;
            const uint32_t nt = nT;
            // a gap transfer overwritten in place by the next same-address transfer of the same run
            for_each(nT, [=] __device__(size_t q) {
                if (q + 1 >= nt || a0[q + 1] != a0[q] || a1[q + 1] != a1[q]) return;
                const uint32_t t1 = av[q], t2 = av[q + 1];
                if (cl[t1] == CLS_GAP && cl[t2] == CLS_GAP && rn[t1] == rn[t2]) fl[TT[t1]] = 1;
            }, s);
        }
    }
    DBuf<uint32_t> ut, utc(1, s);
    out.own(ut, c.n ? c.n : 1, s);
    const uint8_t *fl = flag.p;
    compact(c.n, [=] __device__(size_t i) { return fl[i] != 0; }, ut.p, utc.p, s);
    out.n_ut = read_u32(utc.p, s);
    out.ut = std::move(ut);
}

// ============================================================ analyze (detectors.py:274-326)
std::mutex g_mu;
cudaStream_t g_stream[64] = {nullptr};
// arena sizing: bytes of scratch per event as measured with B2L_TRACE (analyze 164-183 B/event on
// C2/C4 at 10k-4M events), plus slack; beyond 64M events buffers come from the pool (reused)
constexpr size_t ARENA_MAX_EVENTS = size_t(64) << 20, ARENA_BASE = size_t(4) << 20;
constexpr size_t ARENA_ANALYZE_PER_EVENT = 272, ARENA_SAVINGS_PER_EVENT = 96;  // savings: 5 B/event + a 69 B/event column upload

cudaStream_t engine_stream() {
    int dev = 0;
    CK(cudaGetDevice(&dev));
    if (!g_stream[dev & 63]) {
        CK(cudaStreamCreateWithFlags(&g_stream[dev & 63], cudaStreamNonBlocking));
        // keep freed scratch cached in the stream-ordered pool across calls (no re-mapping)
        cudaMemPool_t pool;
        CK(cudaDeviceGetDefaultMemPool(&pool, dev));
        uint64_t keep = ~0ull;
        CK(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
        // grow the pool once up front (one mapping instead of many small growths on the first
        // call; a one-shot CLI run pays the first call only)
        void *warm = nullptr;
        if (cudaMallocAsync(&warm, size_t(512) << 20, g_stream[dev & 63]) == cudaSuccess)
            cudaFreeAsync(warm, g_stream[dev & 63]);
        else
            cudaGetLastError();
    }
    return g_stream[dev & 63];
}
cudaStream_t g_streamx[4][64] = {{nullptr}};
cudaStream_t engine_stream_n(int k) {  // side streams 1..3: the chains that run beside DD/RT; 4: result copies
    int dev = 0;
    CK(cudaGetDevice(&dev));
    cudaStream_t &st = g_streamx[k - 1][dev & 63];
    if (!st) CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    return st;
}

// `to` waits for everything queued on `from` so far.  One cached event per host thread and device
// (an event may be re-recorded as soon as the wait is queued).
void stream_after(cudaStream_t to, cudaStream_t from) {
    thread_local cudaEvent_t ev[64] = {nullptr};
    int dev = 0;
    CK(cudaGetDevice(&dev));
    cudaEvent_t &e = ev[dev & 63];
    if (!e) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    CK(cudaEventRecord(e, from));
    CK(cudaStreamWaitEvent(to, e, 0));
}

// Declared right after a call's scratch arena: if the call unwinds with an exception, wait for
// the side streams before the arena goes back to the pool (kernels queued on them may still read
// or write scratch carved from it).  On success every chain has already been joined.
struct SideJoin {
    int unc = std::uncaught_exceptions();
    ~SideJoin() {
        if (std::uncaught_exceptions() <= unc) return;
        int dev = 0;
        if (cudaGetDevice(&dev) != cudaSuccess) return;
        for (int k = 0; k < 4; ++k)
            if (cudaStream_t st = g_streamx[k][dev & 63]) cudaStreamSynchronize(st);
        cudaGetLastError();
    }
};



// ============================================================ savings (estimator.py:61-130, report.py:44-95)
// Byte-granular atomic OR (the category bits of one event can come from several lists at once).
__device__ __forceinline__ void atomicOr_u8(uint8_t *p, uint32_t bits) {
    const uintptr_t a = (uintptr_t)p;
    atomicOr(reinterpret_cast<unsigned int *>(a & ~uintptr_t(3)), bits << (8 * (a & 3)));
}
// Overlap flag and union list in one scan: (max end so far, count of events in any category).
struct OvUn {
    using T = struct {
        unsigned long long mx;
        uint32_t cnt, pad;
    };
    static __device__ __forceinline__ T identity() { return T{0ull, 0u, 0u}; }
    static __device__ __forceinline__ T combine(T a, T b) { return T{a.mx > b.mx ? a.mx : b.mx, a.cnt + b.cnt, 0u}; }
};
struct OvUnLoad {
    const uint64_t *end;
    const uint8_t *cat;
    __device__ OvUn::T operator()(size_t i) const { return OvUn::T{end[i], cat[i] ? 1u : 0u, 0u}; }
};
struct OvUnStore {
    const uint64_t *start;
    const uint8_t *cat;
    uint32_t *flag, *uni;
    __device__ void operator()(size_t i, OvUn::T ex, OvUn::T) const {
        if (i > 0 && start[i] < ex.mx) *flag = 1;
        if (cat[i]) uni[ex.cnt] = (uint32_t)i;
    }
};
struct U128 {
    unsigned long long lo, hi;
};
__device__ __forceinline__ void add128(U128 &a, unsigned long long v) {
    a.lo += v;
    a.hi += (a.lo < v);
}
__device__ __forceinline__ U128 warp_sum128(U128 a) {
    for (int o = 16; o; o >>= 1) {
        unsigned long long lo = __shfl_xor_sync(0xffffffffu, a.lo, o), hi = __shfl_xor_sync(0xffffffffu, a.hi, o);
        const unsigned long long s = a.lo + lo;
        a.hi += hi + (s < lo);
        a.lo = s;
    }
    return a;
}
__device__ __forceinline__ void atomic_add128(unsigned long long *lohi, U128 v) {
    if (!v.lo && !v.hi) return;
    const unsigned long long old = atomicAdd(lohi, v.lo);
    const unsigned long long carry = (old + v.lo < old) ? 1ull : 0ull;
    if (v.hi + carry) atomicAdd(lohi + 1, v.hi + carry);
}

// per-event category bits: DD 1, RT 2, RA 4, UA 8, UT 16 (estimator.py:77-113)
__global__ void k_sums(DevCols c, const uint8_t *cat, unsigned long long *acc /*[6][2]*/, unsigned long long *nunion,
                       unsigned long long *minmax /*[2]: min start, max end*/) {
    pdl_enter();
    U128 a[6];
#pragma unroll
    for (int k = 0; k < 6; ++k) a[k] = U128{0, 0};
    unsigned long long cnt = 0, mn = ~0ull, mx = 0;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < c.n; i += (size_t)gridDim.x * blockDim.x) {
        const uint64_t t0 = c.start[i], t1 = c.end[i];
        mn = t0 < mn ? t0 : mn;
        mx = t1 > mx ? t1 : mx;
        const uint8_t m = cat[i];
        if (!m) continue;
        const unsigned long long d = t1 - t0;
#pragma unroll
        for (int k = 0; k < 5; ++k)
            if (m & (1u << k)) add128(a[k], d);
        add128(a[5], d);
        ++cnt;
    }
    // warp -> block (shared memory) -> one set of atomics per block: every warp hitting the same
    // nine L2 addresses serialises (~85k same-address atomics at 1M events otherwise)
    __shared__ unsigned long long part[32][15];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
#pragma unroll
    for (int k = 0; k < 6; ++k) {
        U128 w = warp_sum128(a[k]);
        if (lane == 0) part[warp][2 * k] = w.lo, part[warp][2 * k + 1] = w.hi;
    }
    for (int o = 16; o; o >>= 1) {
        cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
        unsigned long long x = __shfl_xor_sync(0xffffffffu, mn, o), y = __shfl_xor_sync(0xffffffffu, mx, o);
        mn = x < mn ? x : mn;
        mx = y > mx ? y : mx;
    }
    if (lane == 0) part[warp][12] = cnt, part[warp][13] = mn, part[warp][14] = mx;
    __syncthreads();
    if (warp != 0) return;
    U128 b[6];
    unsigned long long bc = 0, bmn = ~0ull, bmx = 0;
#pragma unroll
    for (int k = 0; k < 6; ++k) b[k] = U128{0, 0};
    if (lane < nwarps) {
#pragma unroll
        for (int k = 0; k < 6; ++k) b[k] = U128{part[lane][2 * k], part[lane][2 * k + 1]};
        bc = part[lane][12], bmn = part[lane][13], bmx = part[lane][14];
    }
#pragma unroll
    for (int k = 0; k < 6; ++k) {
        U128 w = warp_sum128(b[k]);
        if (lane == 0) atomic_add128(acc + 2 * k, w);
    }
    for (int o = 16; o; o >>= 1) {
        bc += __shfl_xor_sync(0xffffffffu, bc, o);
        unsigned long long x = __shfl_xor_sync(0xffffffffu, bmn, o), y = __shfl_xor_sync(0xffffffffu, bmx, o);
        bmn = x < bmn ? x : bmn;
        bmx = y > bmx ? y : bmx;
    }
    if (lane == 0) {
        if (bc) atomicAdd(nunion, bc);
        atomicMin(minmax, bmn);
        atomicMax(minmax + 1, bmx);
    }
}

// Attribution of one category's ordered multiset of finding events to location buckets
// (report.py:44-95): count, sum of durations, sum of bytes, first member (min position).
struct AttrAcc {
    unsigned long long *cnt, *ns, *by, *first;  // [nb], [2nb], [2nb], [nb]
    const ulonglong2 *rec;                       // packed per-event records (FrontOut::attr) or nullptr
    const unsigned *nopack;
};
template <class Elem>
__global__ void k_attr(DevCols c, size_t n_elem, Elem el, AttrAcc g) {
    pdl_enter();
    extern __shared__ unsigned long long sm[];
    const uint32_t nb = c.nbuckets;
    const bool local = nb <= 512;
    unsigned long long *scnt = sm, *sns = sm + nb, *sby = sm + 3 * nb, *sfirst = sm + 5 * nb;
    if (local) {
        for (uint32_t b = threadIdx.x; b < nb; b += blockDim.x)
            scnt[b] = 0, sns[2 * b] = sns[2 * b + 1] = 0, sby[2 * b] = sby[2 * b + 1] = 0, sfirst[b] = ~0ull;
        __syncthreads();
    }
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    const bool packed = g.rec && !*g.nopack;
    // warp-uniform trip count so every lane reaches the warp collectives below
    for (size_t base = (size_t)blockIdx.x * blockDim.x; base < n_elem; base += stride) {
        const size_t q = base + threadIdx.x;
        uint32_t ev[2];
        uint64_t pos[2];
        const int k = q < n_elem ? el(q, ev, pos) : 0;
        for (int j = 0; j < 2; ++j) {
            const bool have = j < k;
            const uint32_t e = have ? ev[j] : 0;
            uint32_t b = 0xFFFFFFFFu;
            unsigned long long d = 0, by = 0;
            if (have && packed) {
                const ulonglong2 r = g.rec[e];
                b = (uint32_t)(r.x >> 40), d = r.x & ((1ull << 40) - 1), by = r.y;
            } else if (have) {
                b = c.loc_bucket[c.loc[e]], d = c.end[e] - c.start[e], by = c.nb[e];
            }
            unsigned long long fp = have ? ((pos[j] << 32) | e) : ~0ull, cnt = have ? 1 : 0;
            const uint32_t peers = __match_any_sync(0xffffffffu, b);
            U128 sd{d, 0}, sb{by, 0};
            if (peers == 0xffffffffu) {
                // the whole warp hit one bucket (the common case: few code locations): reduce first
                sd = warp_sum128(sd);
                sb = warp_sum128(sb);
                for (int o = 16; o; o >>= 1) {
                    cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
                    const unsigned long long x = __shfl_xor_sync(0xffffffffu, fp, o);
                    fp = x < fp ? x : fp;
                }
                if ((threadIdx.x & 31) != 0) continue;
            }
            if (b == 0xFFFFFFFFu) continue;
            if (local) {
                atomicAdd(scnt + b, cnt);
                atomic_add128(sns + 2 * b, sd);
                atomic_add128(sby + 2 * b, sb);
                atomicMin(sfirst + b, fp);
            } else {
                atomicAdd(g.cnt + b, cnt);
                atomic_add128(g.ns + 2 * b, sd);
                atomic_add128(g.by + 2 * b, sb);
                atomicMin(g.first + b, fp);
            }
        }
    }
    if (local) {
        __syncthreads();
        for (uint32_t b = threadIdx.x; b < nb; b += blockDim.x) {
            if (!scnt[b]) continue;
            atomicAdd(g.cnt + b, scnt[b]);
            atomic_add128(g.ns + 2 * b, U128{sns[2 * b], sns[2 * b + 1]});
            atomic_add128(g.by + 2 * b, U128{sby[2 * b], sby[2 * b + 1]});
            atomicMin(g.first + b, sfirst[b]);
        }
    }
}
struct ElemList {  // plain event list (DD members, UT): position = index
    const uint32_t *ev;
    __device__ int operator()(size_t q, uint32_t *e, uint64_t *p) const {
        e[0] = ev[q], p[0] = q;
        return 1;
    }
};
struct ElemTrips {  // RT: (tx, rx) per trip
    const uint32_t *tx, *rx;
    __device__ int operator()(size_t q, uint32_t *e, uint64_t *p) const {
        e[0] = tx[q], e[1] = rx[q], p[0] = 2 * q, p[1] = 2 * q + 1;
        return 2;
    }
};
struct ElemPairs {  // RA / UA: alloc + non-synthetic delete per pair
    const uint32_t *pairs, *pa, *pd;
    __device__ int operator()(size_t q, uint32_t *e, uint64_t *p) const {
        const uint32_t r = pairs[q];
        e[0] = pa[r], p[0] = 2 * q;
        if (pd[r] == NONE) return 1;
        e[1] = pd[r], p[1] = 2 * q + 1;
        return 2;
    }
};

struct FindingsDev {  // device views of a findings set
    const uint64_t *dd_off, *ra_off;
    const uint32_t *dd_mem, *rt_tx, *rt_rx, *pa, *pd, *ra_mem, *ua, *ut;
    uint64_t dd_groups, dd_members, rt_trips, n_pairs, ra_groups, ra_members, n_ua, n_ut;
};

// One savings computation (estimator.py:61-130 integer part, report.py:44-95 aggregation),
// split so a fused analyze can feed it category by category as its chains finish: attribution
// and category bits of a category only need that category's findings; the sums and the
// overlap / union scan need all five.
struct SvRun {
    DevCols c{};
    size_t n = 0;
    uint32_t nb = 0;
    size_t smem = 0;
    DBuf<unsigned long long> at, acc;
    DBuf<uint8_t> cat;
    DBuf<uint32_t> ovl, uni, unic;
    DBuf<OvUn::T> ovt;
    const ulonglong2 *rec = nullptr;
    const unsigned *nopack = nullptr;
    AttrAcc acc_of(int cat_i) const {
        unsigned long long *base = at.p;
        return AttrAcc{base + (size_t)cat_i * nb, base + 5 * (size_t)nb + (size_t)cat_i * 2 * nb,
                       base + 15 * (size_t)nb + (size_t)cat_i * 2 * nb, base + 25 * (size_t)nb + (size_t)cat_i * nb,
                       rec, nopack};
    }
};

void sv_begin(SvRun &R, const DevCols &c, cudaStream_t s) {
    R.c = c;
    R.n = c.n;
    R.nb = c.nbuckets;
    R.at.alloc(5 * (size_t)R.nb * 6 + 1, s);
    init_u64(R.at.p, 5 * (size_t)R.nb * 5, 5 * (size_t)R.nb, 1, s);  // the first-member slots start at ~0
    R.smem = R.nb <= 512 ? (size_t)R.nb * 6 * sizeof(unsigned long long) : 0;
    R.cat.alloc_zeroed(((R.n ? R.n : 1) + 3) & ~size_t(3), s);  // whole words: byte atomics touch the word
}

// Attribution + category bits of category k (DD 0, RT 1, RA 2, UA 3, UT 4) on stream st.
void sv_add(SvRun &R, int k, const FindingsDev &F, cudaStream_t st) {
    const DevCols c = R.c;
    uint8_t *ct = R.cat.p;
    auto launch = [&](auto el, size_t ne) {
        if (!ne || !R.nb) return;
        launch_k(k_attr<decltype(el)>, grid_for(ne, TPB, 148 * 8), TPB, R.smem, st, c, ne, el, R.acc_of(k));
        CK_LAUNCH("k_attr");
    };
    if (k == 0) {  // DD: every member counts for attribution; all but the first of a group are eliminable
        launch(ElemList{F.dd_mem}, F.dd_members);
        const uint64_t *off = F.dd_off;
        const uint32_t *mem = F.dd_mem;
        const uint64_t ng = F.dd_groups;
        for_each(F.dd_members, [=] __device__(size_t q) {
            uint64_t lo = 0, hi = ng;  // group g with off[g] <= q < off[g+1]
            while (hi - lo > 1) {
                uint64_t m = (lo + hi) >> 1;
                if (off[m] <= q) lo = m; else hi = m;
            }
            if (off[lo] != q) atomicOr_u8(ct + mem[q], 1);
        }, st);
    } else if (k == 1) {  // RT: tx and rx attributed, the receptions eliminable
        launch(ElemTrips{F.rt_tx, F.rt_rx}, F.rt_trips);
        const uint32_t *rx = F.rt_rx;
        for_each(F.rt_trips, [=] __device__(size_t q) { atomicOr_u8(ct + rx[q], 2); }, st);
    } else if (k == 2) {  // RA: pairs after the first of a group (alloc + non-synthetic delete)
        launch(ElemPairs{F.ra_mem, F.pa, F.pd}, F.ra_members);
        const uint64_t *roff = F.ra_off;
        const uint32_t *rm = F.ra_mem, *pa = F.pa, *pd = F.pd;
        const uint64_t rng = F.ra_groups;
        for_each(F.ra_members, [=] __device__(size_t q) {
            uint64_t lo = 0, hi = rng;
            while (hi - lo > 1) {
                uint64_t m = (lo + hi) >> 1;
                if (roff[m] <= q) lo = m; else hi = m;
            }
            if (roff[lo] == q) return;  // first pair of a group is necessary
            const uint32_t r = rm[q];
            atomicOr_u8(ct + pa[r], 4);
            if (pd[r] != NONE) atomicOr_u8(ct + pd[r], 4);
        }, st);
    } else if (k == 3) {  // UA
        launch(ElemPairs{F.ua, F.pa, F.pd}, F.n_ua);
        const uint32_t *ua = F.ua, *pa = F.pa, *pd = F.pd;
        for_each(F.n_ua, [=] __device__(size_t q) {
            const uint32_t r = ua[q];
            atomicOr_u8(ct + pa[r], 8);
            if (pd[r] != NONE) atomicOr_u8(ct + pd[r], 8);
        }, st);
    } else {  // UT
        launch(ElemList{F.ut}, F.n_ut);
        const uint32_t *ut = F.ut;
        for_each(F.n_ut, [=] __device__(size_t q) { atomicOr_u8(ct + ut[q], 16); }, st);
    }
}

// Sums, overlap flag and union list once every category is in (all on s), then the results to
// the host: the small ones with one synchronisation of s, the arrays on `copy` (not synchronised).
void sv_finish(SvRun &R, b2l_savings *o, cudaStream_t s, cudaStream_t copy) {
    const size_t n = R.n;
    const DevCols c = R.c;
    R.acc.alloc(12 + 1 + 2, s);
    init_u64(R.acc.p, 13, 1, 1, s);  // min start := ~0 (max end stays 0)
    if (n) {
        launch_k(k_sums, grid_for(n, TPB, 148 * 4), TPB, 0, s, c, (const uint8_t *)R.cat.p, R.acc.p, R.acc.p + 12, R.acc.p + 13);
        CK_LAUNCH("k_sums");
    }
    // overlap: exists i >= 1 with start[i] < max(end[0..i-1])  (estimator.py:51-58)
    // ... and the union list, in the same scan
    R.ovl.alloc_zeroed(1, s);
    R.uni.alloc(n ? n : 1, s);
    R.unic.alloc(1, s);
    R.ovt.alloc(1, s);
    scan<OvUn>(n, OvUnLoad{c.end, R.cat.p}, OvUnStore{c.start, R.cat.p, R.ovl.p, R.uni.p}, s, R.ovt.p);
    if (n) dev_copy(R.unic.p, &R.ovt.p->cnt, 4, s);
    else R.unic.zero();
    unsigned long long h[15];
    uint32_t hov = 0, hun = 0;
    PhaseClock(s).mark(" sv-queued");
    {  // one synchronisation for the three small results
        read_back_multi({{h, R.acc.p, sizeof(h)}, {&hov, R.ovl.p, 4}, {&hun, R.unic.p, 4}}, s);
    }
    PhaseClock(s).mark(" sv-rb");
    for (int k = 0; k < 5; ++k) o->per_category_ns[k] = b2l_u128{h[2 * k], h[2 * k + 1]};
    o->union_ns = b2l_u128{h[10], h[11]};
    o->n_union = hun;
    o->has_overlaps = hov ? 1 : 0;
    o->min_start_ns = n ? h[13] : 0;
    o->max_end_ns = h[14];
    HostBatch hb;
    hb.add(&o->union_index, R.uni.p, hun);
    o->n_buckets = R.nb;
    const size_t nb5 = 5 * (size_t)R.nb;
    hb.add((unsigned long long **)&o->attr_count, R.at.p, nb5);
    hb.add((unsigned long long **)&o->attr_ns, R.at.p + nb5, 2 * nb5);
    hb.add((unsigned long long **)&o->attr_bytes, R.at.p + 3 * nb5, 2 * nb5);
    hb.add((unsigned long long **)&o->attr_first, R.at.p + 5 * nb5, nb5);
    HostSlab *slab = new HostSlab();
    o->internal = slab;
    hb.flush_async(*slab, s, copy);
}

FindingsDev findings_dev(const Internal &in) {
    FindingsDev F{};
    F.dd_off = in.dd_off.p, F.ra_off = in.ra_off.p, F.dd_mem = in.dd_mem.p, F.rt_tx = in.rt_tx.p;
    F.rt_rx = in.rt_rx.p, F.pa = in.pair_alloc.p, F.pd = in.pair_delete.p, F.ra_mem = in.ra_mem.p;
    F.ua = in.ua.p, F.ut = in.ut.p;
    F.dd_groups = in.dd_groups, F.dd_members = in.dd_members, F.rt_trips = in.rt_trips, F.n_pairs = in.n_pairs;
    F.ra_groups = in.ra_groups, F.ra_members = in.ra_members, F.n_ua = in.n_ua, F.n_ut = in.n_ut;
    return F;
}

int savings_impl(const b2l_trace_cols *cols, const b2l_findings *f, b2l_savings **outp) {
    // a fused analyze (B2L_ANALYZE_WITH_SAVINGS) of these very columns already computed them
    if (f && f->internal) {
        Internal *in = (Internal *)f->internal;
        if (in->fused && in->fused_n == cols->n_events && in->fused_key[0] == (const void *)cols->seq &&
            in->fused_key[1] == (const void *)cols->start_ns && in->fused_key[2] == (const void *)cols->hash &&
            in->fused->n_buckets == cols->n_buckets) {
            *outp = in->fused;
            in->fused = nullptr;
            return B2L_OK;
        }
    }
    b2l_savings *o = (b2l_savings *)calloc(1, sizeof(b2l_savings));
    if (!o) return fail(B2L_E_OOM, "host allocation failed");
    *outp = o;
    std::lock_guard<std::mutex> lock(g_mu);
    cudaStream_t s = engine_stream();
    Arena arena;  // this call's scratch (declared first: released last)
    SideJoin side_join;
    arena.open(cols->n_events <= ARENA_MAX_EVENTS ? ARENA_BASE + cols->n_events * ARENA_SAVINGS_PER_EVENT : 0, s,
               (size_t(1) << 20) + cols->n_events * 2);
    ArenaUse arena_use(&arena);
    ColsUpload up;
    const Internal *fin = (const Internal *)f->internal;
    DevCols c;
    if (fin && !cols->device_resident && fin->cols_n == cols->n_events && fin->cols_key[0] == (const void *)cols->seq &&
        fin->cols_key[1] == (const void *)cols->start_ns && fin->cols_key[2] == (const void *)cols->hash) {
        c = fin->cols.d;  // the same host columns analyze() uploaded: reuse the device copy
        c.nlocs = cols->n_locs, c.nbuckets = cols->n_buckets;
    } else {
        up.load(cols, s);
        c = up.d;
    }
    // findings on the device: reuse the engine's copies, or upload caller arrays
    FindingsDev F{};
    std::vector<DBuf<uint8_t>> keep;
    auto upl = [&](const auto *h, size_t cnt) {
        using T = std::remove_const_t<std::remove_pointer_t<decltype(h)>>;
        if (!cnt) return (const T *)nullptr;
        keep.emplace_back(cnt * sizeof(T), s);
        CK(cudaMemcpyAsync(keep.back().p, h, cnt * sizeof(T), cudaMemcpyHostToDevice, s));
        return (const T *)keep.back().p;
    };
    const uint64_t nm_dd = f->dd_groups ? f->dd_offsets[f->dd_groups] : 0;
    const uint64_t nt_rt = f->rt_groups ? f->rt_offsets[f->rt_groups] : 0;
    const uint64_t nm_ra = f->ra_groups ? f->ra_offsets[f->ra_groups] : 0;
    if (f->internal) {
        F = findings_dev(*(const Internal *)f->internal);
    } else {
        F.dd_off = upl(f->dd_offsets, f->dd_groups + 1), F.ra_off = upl(f->ra_offsets, f->ra_groups + 1);
        F.dd_mem = upl(f->dd_members, nm_dd), F.rt_tx = upl(f->rt_tx, nt_rt), F.rt_rx = upl(f->rt_rx, nt_rt);
        F.pa = upl(f->pair_alloc, f->n_pairs), F.pd = upl(f->pair_delete, f->n_pairs);
        F.ra_mem = upl(f->ra_pairs, nm_ra), F.ua = upl(f->ua_pairs, f->n_ua), F.ut = upl(f->ut_events, f->n_ut);
    }
    F.dd_groups = f->dd_groups, F.dd_members = nm_dd, F.rt_trips = nt_rt, F.n_pairs = f->n_pairs;
    F.ra_groups = f->ra_groups, F.ra_members = nm_ra, F.n_ua = f->n_ua, F.n_ut = f->n_ut;
    PhaseClock pc(s);
    pc.mark("sv-setup");
    SvRun R;
    sv_begin(R, c, s);
    // attribution and category bits: DD, RT, RA on a side stream, UA, UT on s
    cudaStream_t sa = engine_stream_n(1);
    stream_after(sa, s);
    for (int k = 0; k < 3; ++k) sv_add(R, k, F, sa);
    for (int k = 3; k < 5; ++k) sv_add(R, k, F, s);
    stream_after(s, sa);
    pc.mark("sv-attr");
    cudaStream_t sc = engine_stream_n(4);
    sv_finish(R, o, s, sc);
    stream_wait(sc);
    pc.mark("sv-d2h");
    if (alloc_stats().on)
        fprintf(stderr, "[b2l] savings arena %.1f of %.1f MB (%.0f B/event)\n", arena.off.load() / 1048576.0,
                arena.cap / 1048576.0, c.n ? (double)arena.off.load() / c.n : 0.0);
    return B2L_OK;
}

void savings_free(b2l_savings *o) {
    if (!o) return;
    delete (HostSlab *)o->internal;
    free(o);
}

int analyze_impl(const b2l_trace_cols *cols, uint32_t flags, uint64_t synth_end_override, b2l_findings **outp) {
    b2l_findings *f = (b2l_findings *)calloc(1, sizeof(b2l_findings));
    if (!f) return fail(B2L_E_OOM, "host allocation failed");
    *outp = f;
    f->n_events = cols->n_events;
    if (cols->n_events >= 0xFFFFFFFFull) return fail(B2L_E_INVALID_ARG, "trace too large for 32-bit event indices");
    std::lock_guard<std::mutex> lock(g_mu);
    cudaStream_t s = engine_stream();
    PhaseClock pc(s);
    pc.mark("start");
    Internal *in = new Internal();
    f->internal = in;
    ColsUpload &up = in->cols;
    up.load(cols, s);
    if (!cols->device_resident) {
        in->cols_key[0] = cols->seq, in->cols_key[1] = cols->start_ns, in->cols_key[2] = cols->hash;
        in->cols_n = cols->n_events;
    }
    const DevCols c = up.d;
    const size_t n = c.n;
    pc.mark("upload");
    // this call's scratch: one arena, released when the call returns (the device findings get
    // their own, smaller arena once the partition counts bound them)
    Arena arena;
    SideJoin side_join;
    // zeroed pool: the scans' flags and the radix passes' look-back status words (1-KiB status
    // per 1024-record tile under ~1.2M records, per 4096-record tile above)
    arena.open(n <= ARENA_MAX_EVENTS ? ARENA_BASE + n * ARENA_ANALYZE_PER_EVENT : 0, s,
               (size_t(1) << 20) + (n < (size_t(2) << 20) ? n * 20 : n * 4));
    arena.mailbox = n <= (size_t(16) << 20);
    ArenaUse arena_use(&arena);
    // ---- 1+2. validation, partition, max end, key-bit masks, start ranks (fused front pass)
    const bool validate = !(flags & B2L_ANALYZE_NO_VALIDATE), raw = (flags & B2L_ANALYZE_RAW_HASHED) != 0;
    const unsigned ftiles = (unsigned)((n + FR_TILE - 1) / FR_TILE);
    DBuf<FrontAcc> fpart(ftiles + 1, s);
    DBuf<unsigned long long> agg(11, s);  // [0] max data-op end, [1..5] subset OR, [6..10] subset AND
    init_u64(agg.p, 6, 5, 0, s);
    FrontAcc ftot{};
    unsigned long long hm[11] = {0, 0, 0, 0, 0, 0, ~0ull, ~0ull, ~0ull, ~0ull, ~0ull};
    // the five partition lists are sized n (an upper bound) so the apply pass is queued right
    // behind the reduce, before the one read-back of the counts and masks
    const bool only_validate = (flags & B2L_ANALYZE_VALIDATE_ONLY) != 0;
    const size_t nl = only_validate || !n ? 1 : n;
    DBuf<uint32_t> H(nl, s), TT(nl, s), AD(nl, s), A(nl, s), TK(nl, s);
    DBuf<uint64_t> HD(nl, s);
    DBuf<uint32_t> srank(nl, s);
    // fused savings: the attribution records come out of the apply pass
    const bool want_attr = (flags & B2L_ANALYZE_WITH_SAVINGS) != 0 && !only_validate && n && c.nbuckets;
    DBuf<ulonglong2> attr;
    DBuf<unsigned> nopack;
    if (want_attr) attr.alloc(n, s), nopack.alloc_zeroed(1, s);
    static const bool two_pass = getenv("B2L_FRONT_TWO_PASS") != nullptr;  // the r02 reduce/apply path
    const bool fused_front = n && !only_validate && !two_pass;
    if (fused_front) {  // one read of the columns (k_front_fused); the counts come back with the masks
        DBuf<uint32_t> lbf;  // look-back flags (one per 128-byte line) + the tile ticket, zeroed
        lbf.alloc_zeroed((ftiles + 1) * FS + 1, s);
        DBuf<FrontAcc> lb(2 * (size_t)ftiles, s);
        FrontOut fo{{nullptr, H.p, TT.p, AD.p, A.p, TK.p}, srank.p, attr.p, nopack.p, HD.p};
        launch_k(k_front_fused, ftiles, FR_THREADS, 0, s, c, validate, raw, fo, lb.p, lb.p + ftiles, lbf.p,
                 lbf.p + (ftiles + 1) * FS, fpart.p + ftiles, agg.p);
        CK_LAUNCH("k_front_fused");
        read_back_multi({{&ftot, fpart.p + ftiles, sizeof(FrontAcc)}, {hm, agg.p, sizeof(hm)}}, s);
    } else if (n) {
        launch_k(k_front_reduce, ftiles, FR_THREADS, 0, s, c, validate, raw, fpart.p, agg.p);
        CK_LAUNCH("k_front_reduce");
        launch_k(k_scan_partials<FrontOp>, 1, SCAN_THREADS, 0, s, fpart.p, (size_t)ftiles, fpart.p + ftiles);
        CK_LAUNCH("k_scan_partials<FrontOp>");
        if (!only_validate) {  // lists of an invalid trace are never read
            FrontOut fo{{nullptr, H.p, TT.p, AD.p, A.p, TK.p}, srank.p, attr.p, nopack.p, HD.p};
            launch_k(k_front_apply, ftiles, FR_THREADS, 0, s, c, false, raw, (const FrontAcc *)fpart.p, fo);
            CK_LAUNCH("k_front_apply");
        }
        read_back_multi({{&ftot, fpart.p + ftiles, sizeof(FrontAcc)}, {hm, agg.p, sizeof(hm)}}, s);
    }
    const uint32_t nbad = ftot.c[0];
    if (nbad && fused_front) {  // error path: per-tile bad counts for the bad list
        init_u64(agg.p, 6, 5, 0, s);
        launch_k(k_front_reduce, ftiles, FR_THREADS, 0, s, c, validate, raw, fpart.p, agg.p);
        CK_LAUNCH("k_front_reduce");
        launch_k(k_scan_partials<FrontOp>, 1, SCAN_THREADS, 0, s, fpart.p, (size_t)ftiles, fpart.p + ftiles);
        CK_LAUNCH("k_scan_partials<FrontOp>");
    }
    if (nbad) {
        DBuf<uint32_t> bad(nbad, s), rules(nbad, s), dcount(1, s);
        FrontOut fo{{bad.p, nullptr, nullptr, nullptr, nullptr, nullptr}, nullptr, nullptr, nullptr, nullptr};
        k_front_apply<<<ftiles, FR_THREADS, 0, s>>>(c, true, raw, fpart.p, fo);
        CK_LAUNCH("k_front_apply(bad)");
        CK(cudaMemcpyAsync(dcount.p, &nbad, sizeof(uint32_t), cudaMemcpyHostToDevice, s));
        k_bad_rules<<<grid_for(nbad, TPB), TPB, 0, s>>>(c, bad.p, dcount.p, rules.p);
        CK_LAUNCH("k_bad_rules");
        f->n_bad = nbad;
        HostBatch hb;
        hb.add(&f->bad_index, bad.p, nbad);
        hb.add(&f->bad_rules, rules.p, nbad);
        in->slab = new HostSlab();
        hb.flush(*in->slab, s);
        return fail(B2L_E_INVALID_TRACE, "trace fails validation");
    }
    pc.mark("validate");
    if (flags & B2L_ANALYZE_VALIDATE_ONLY) return B2L_OK;
    const uint32_t hc[FR_NCAT] = {0, ftot.c[1], ftot.c[2], ftot.c[3], ftot.c[4], ftot.c[5]};
    const unsigned long long me = (flags & B2L_ANALYZE_SYNTH_END) ? synth_end_override : hm[0];
    const bool ddrt = !(flags & B2L_ANALYZE_SKIP_DDRT), alloc = !(flags & B2L_ANALYZE_SKIP_ALLOC);
    const uint32_t nH = ddrt ? hc[1] : 0, nT = alloc ? hc[2] : 0, nAD = alloc ? hc[3] : 0, nA = alloc ? hc[4] : 0,
                   nK = alloc ? hc[5] : 0;
    g_masks.hash = live_mask(hm[1] ^ hm[6]), g_masks.da = live_mask(hm[2] ^ hm[7]);
    g_masks.sa = live_mask(hm[3] ^ hm[8]), g_masks.nb = live_mask(hm[4] ^ hm[9]);
    g_masks.sa_tt = live_mask(hm[5] ^ hm[10]);
    g_masks.dev = live_range((uint64_t)(c.ndev > 0 ? c.ndev : 1));
    g_masks.idx = live_range(n);
    g_masks.n = n;
    g_masks.srank = srank.p;

    pc.mark("partition");
    // fused savings: attribution / category bits of each category queued as its chain finishes
    const bool with_sv = (flags & B2L_ANALYZE_WITH_SAVINGS) != 0;
    SvRun R;
    if (with_sv) {
        sv_begin(R, c, s);
        R.rec = attr.p, R.nopack = nopack.p;
    }
    {  // upper bounds of the device findings: DD/RT offsets and members <= nH, pairs/RA/UA <= nA, UT <= n
        const size_t fb = 16 * (nH + 2) + 12 * (size_t)nH + 8 * (nA + 2) + 16 * (size_t)nA + 4 * n + 32 * 256;
        in->keep.open(n <= ARENA_MAX_EVENTS ? fb : 0, s, 0);
    }
    in->synth_end = me;
    in->n_pairs = nA;
    // ---- 3-6.  Three independent chains: hash-keyed (DD, RT), pairs -> RA, and the kernel index
    // -> UT (-> UA once the pairs exist).  Small traces run them on three streams from three host
    // threads (each keeps its own syncs and staging); traces past 16M events run them back to back
    // on one stream (measured r02: three streams win 7-8 % at 10M, tie at 30M, lose 9 % at 100M
    // where the chains' working sets evict each other from L2).
    int dev = 0;
    CK(cudaGetDevice(&dev));
    const Masks masks = g_masks;
    PairOut po;
    static const uint64_t overlap_min = getenv("B2L_OVERLAP_MIN") ? strtoull(getenv("B2L_OVERLAP_MIN"), nullptr, 10) : 0;
    static const uint64_t overlap_max = getenv("B2L_OVERLAP_MAX") ? strtoull(getenv("B2L_OVERLAP_MAX"), nullptr, 10) : (size_t(16) << 20);
    const bool overlap = n <= overlap_max && n >= overlap_min;
    cudaStream_t s2 = overlap ? engine_stream_n(1) : s, s3 = overlap ? engine_stream_n(2) : s;
    cudaStream_t sc = engine_stream_n(4);  // device -> host result copies, chain by chain
    if (overlap) {  // the partition lists and start ranks are produced on s
        stream_after(s2, s);
        stream_after(s3, s);
    }
    std::promise<cudaEvent_t> pairs_done;  // recorded on s2 after pairing (UA needs the pairs)
    std::shared_future<cudaEvent_t> pairs_ready = pairs_done.get_future().share();
    EngineErr err2{0, ""}, err3{0, ""};
    bool failed2 = false, failed3 = false, promised = false;
    auto pairs_chain = [&] {
        ArenaUse au(&arena);
        try {
            CK(cudaSetDevice(dev));
            g_masks = masks;
            PhaseClock pc2(s2);
            pc2.mark("pairs-start");
            po = pairs_step(c, AD.p, nAD, A.p, nA, me, *in, s2);
            cudaEvent_t ev;
            CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
            CK(cudaEventRecord(ev, s2));
            pairs_done.set_value(ev);
            promised = true;
            pc2.mark("pairs");
            ra_step(c, nA, *in, s2);
            if (po.wcount.p) po.n_warn = read_u32(po.wcount.p, s2);
            pc2.mark("ra");
            if (with_sv) sv_add(R, 2, findings_dev(*in), s2);
            {  // this chain's results go to the host while the other chains still run
                HostBatch hb;
                hb.add(&f->pair_alloc, in->pair_alloc.p, nA);
                hb.add(&f->pair_delete, in->pair_delete.p, nA);
                hb.add(&f->warn_index, po.warn.p, po.n_warn);
                hb.add(&f->ra_offsets, in->ra_off.p, in->ra_groups + 1);
                hb.add(&f->ra_pairs, in->ra_mem.p, in->ra_members);
                in->slab_pairs = new HostSlab();
                hb.flush_async(*in->slab_pairs, s2, sc);
            }
            if (overlap) stream_wait(s2);
        } catch (const EngineErr &e) {
            err2 = e;
            failed2 = true;
            if (!promised) pairs_done.set_value(nullptr);
        }
    };
    auto kernel_chain = [&] {
        ArenaUse au(&arena);
        try {
            CK(cudaSetDevice(dev));
            g_masks = masks;
            PhaseClock pc3(s3);
            pc3.mark("kern-start");
            KernelIndexStore kis(nK, s3);
            build_kernel_index(kis, c, TK.p, nK, s3);
            ut_step(c, kis.KI, TT.p, nT, *in, s3);
            pc3.mark("ut");
            cudaEvent_t ev = pairs_ready.get();
            if (!ev) return;  // pairing failed (reported by its chain)
            CK(cudaStreamWaitEvent(s3, ev, 0));
            ua_step(c, kis.KI, *in, s3);
            pc3.mark("ua");
            if (with_sv) {
                const FindingsDev F = findings_dev(*in);
                sv_add(R, 3, F, s3);
                sv_add(R, 4, F, s3);
            }
            {
                HostBatch hb;
                hb.add(&f->ua_pairs, in->ua.p, in->n_ua);
                hb.add(&f->ut_events, in->ut.p, in->n_ut);
                in->slab_kern = new HostSlab();
                hb.flush_async(*in->slab_kern, s3, sc);
            }
            if (overlap) stream_wait(s3);
        } catch (const EngineErr &e) {
            err3 = e;
            failed3 = true;
        }
    };
    std::future<void> t2, t3;
    if (overlap) {
        t2 = workers().submit(pairs_chain);
        t3 = workers().submit(kernel_chain);
    } else {
        pairs_chain();
        kernel_chain();
    }
    auto join = [&] {
        if (t2.valid()) t2.wait();
        if (t3.valid()) t3.wait();
        cudaEvent_t ev = pairs_ready.get();
        if (ev) cudaEventDestroy(ev);
    };
    try {
        DdRt dr = dd_rt_step(c, H.p, HD.p, nH, (flags & B2L_ANALYZE_STRICT_RT) != 0, *in, s, f, sc);
        in->dd_groups = dr.dd_groups, in->dd_members = dr.dd_members, in->rt_groups = dr.rt_groups,
        in->rt_trips = dr.rt_trips;
        if (with_sv) {
            const FindingsDev F = findings_dev(*in);
            sv_add(R, 0, F, s);
            sv_add(R, 1, F, s);
        }
    } catch (...) {
        join();
        throw;
    }
    join();
    if (failed2) throw err2;
    if (failed3) throw err3;
    pc.mark("detectors");

    // ---- results to the host: DD/RT now (the other chains queued theirs when they ended), then
    // one synchronisation of the copy stream
    HostBatch hb;
    f->dd_groups = in->dd_groups;
    if (!in->slab_dd) {  // (no hashed transfers: the DD chain queued nothing)
        hb.add(&f->dd_offsets, in->dd_off.p, in->dd_groups + 1);
        hb.add(&f->dd_members, in->dd_mem.p, in->dd_members);
    }
    f->rt_groups = in->rt_groups;
    hb.add(&f->rt_offsets, in->rt_off.p, in->rt_groups + 1);
    hb.add(&f->rt_tx, in->rt_tx.p, in->rt_trips);
    hb.add(&f->rt_rx, in->rt_rx.p, in->rt_trips);
    in->slab = new HostSlab();
    hb.flush_async(*in->slab, s, sc);
    f->n_pairs = nA;
    f->synthetic_end_ns = me;
    f->n_warnings = po.n_warn;
    f->ra_groups = in->ra_groups;
    f->n_ua = in->n_ua;
    f->n_ut = in->n_ut;
    if (with_sv) {  // every category is in: sums, overlap / union scan, results on the copy stream
        b2l_savings *o = (b2l_savings *)calloc(1, sizeof(b2l_savings));
        if (!o) throw EngineErr{B2L_E_OOM, "host allocation failed"};
        in->fused = o;
        in->fused_key[0] = cols->seq, in->fused_key[1] = cols->start_ns, in->fused_key[2] = cols->hash;
        in->fused_n = cols->n_events;
        sv_finish(R, o, s, sc);
    }
    pc.mark("queued");
    stream_wait(sc);
    pc.mark("d2h");
    ev_log_flush();
    if (alloc_stats().on) {
        fprintf(stderr, "[b2l] pool alloc/free calls %llu, host %.3f ms; arena %.1f of %.1f MB (%.0f B/event)\n",
                (unsigned long long)alloc_stats().n.load(), alloc_stats().ns.load() * 1e-6,
                arena.off.load() / 1048576.0, arena.cap / 1048576.0, n ? (double)arena.off.load() / n : 0.0);
        fprintf(stderr, "[b2l] findings arena %.1f of %.1f MB\n", in->keep.off.load() / 1048576.0,
                in->keep.cap / 1048576.0);
        alloc_stats().n = 0, alloc_stats().ns = 0;
    }
    if (sync_stats().on) {
        fprintf(stderr, "[b2l] host round trips %llu, %.3f ms waiting (all chains); %llu launches, %.3f ms host\n",
                (unsigned long long)sync_stats().n.load(), sync_stats().ns.load() * 1e-6,
                (unsigned long long)sync_stats().ln.load(), sync_stats().lns.load() * 1e-6);
        sync_stats().n = 0, sync_stats().ns = 0, sync_stats().ln = 0, sync_stats().lns = 0;
        std::lock_guard<std::mutex> g(sync_log_mu());
        auto &L = sync_log();
        if (!L.empty()) {
            std::sort(L.begin(), L.end(), [](const SyncRec &a, const SyncRec &b) { return a.t0 < b.t0; });
            std::vector<size_t> tids;
            for (auto &r : L) {
                size_t k = 0;
                while (k < tids.size() && tids[k] != r.thread) ++k;
                if (k == tids.size()) tids.push_back(r.thread);
                fprintf(stderr, "[b2l-rb] thread %zu line %5d at %8.1f us waited %6.1f us\n", k, r.line,
                        std::chrono::duration<double, std::micro>(r.t0 - L[0].t0).count(), r.ns * 1e-3);
            }
            L.clear();
        }
    }
    if (in->dd_groups == 0) f->dd_offsets[0] = 0;
    if (in->rt_groups == 0) f->rt_offsets[0] = 0;
    if (in->ra_groups == 0) f->ra_offsets[0] = 0;
    return B2L_OK;
}

void findings_free(b2l_findings *f) {
    if (!f) return;
    Internal *in = (Internal *)f->internal;
    if (in) {  // arrays live in the slabs
        if (in->fused) savings_free(in->fused);
        delete in->slab;
        delete in->slab_pairs;
        delete in->slab_kern;
        delete in->slab_dd;
    }
    delete in;
    free(f);
}

// seq -> trace position (binary search over the ascending seq column)
int lookup_impl(const b2l_trace_cols *cols, const uint64_t *seqs, uint64_t nq, uint32_t *out) {
    std::lock_guard<std::mutex> lock(g_mu);
    cudaStream_t s = engine_stream();
    ColsUpload up;
    const uint64_t *dseq;
    if (cols->device_resident) {
        dseq = cols->seq;
    } else {
        dseq = up.up(cols->seq, cols->n_events, s);
    }
    const size_t n = cols->n_events;
    DBuf<uint64_t> q(nq ? nq : 1, s);
    DBuf<uint32_t> r(nq ? nq : 1, s);
    if (nq) CK(cudaMemcpyAsync(q.p, seqs, nq * sizeof(uint64_t), cudaMemcpyHostToDevice, s));
    const uint64_t *qp = q.p;
    uint32_t *rp = r.p;
    for_each(nq, [=] __device__(size_t i) {
        const uint64_t v = qp[i];
        size_t lo = 0, hi = n;
        while (lo < hi) {
            size_t m = (lo + hi) >> 1;
            if (dseq[m] < v) lo = m + 1; else hi = m;
        }
        rp[i] = (lo < n && dseq[lo] == v) ? (uint32_t)lo : NONE;
    }, s);
    if (nq) CK(cudaMemcpyAsync(out, r.p, nq * sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    return B2L_OK;
}

}  // namespace ana
}  // namespace b2l

namespace b2l {
namespace ana {
// ============================================================ key-range sharding
// Rows exchanged between ranks: one i64 per field, ROW = 12:
//   [0] global event index | key space << 63, then seq, start, end, src_addr, dst_addr, bytes, hash,
//   src_device, dst_device, kind, loc (sharded.py FIELDS).
constexpr int SH_ROW = 12;
// Owner rank of a device-keyed record: ((mix * G) >> 64) on the top 32 bits of a splitmix64 mix
// of the key (sharded.py route_mix -- the host path routes identically).
__host__ __device__ __forceinline__ uint64_t route_splitmix(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
__host__ __device__ __forceinline__ uint64_t route_mix(uint64_t a, uint64_t b) { return route_splitmix(a ^ route_splitmix(b)); }
__host__ __device__ __forceinline__ uint32_t route_owner(uint64_t key, uint32_t G) {
    return (uint32_t)(((key >> 32) * (uint64_t)G) >> 32);
}
// Records of one event (the exchange of the key-range sharded analysis):
//  space 0: a hashed transfer -> the owner of its hash range (DD / RT: detectors.py:85-167);
//  space 1: an alloc or delete -> the pairing owner of (dst_device, dst_addr) (prep.py:58-70);
//           a target transfer -> the owner of (dst_device, src_addr) (UT's next-same-address
//           key, detectors.py:250-264); a target kernel -> every rank that needs it for exact
//           UA / UT cursors (detectors.py:208-212,251-253): the rank of each query (target
//           transfer or target alloc) whose cursor lands on it, and every rank for the first
//           kernel of each device in the shard (queries whose cursor lands on a later shard).
//           Cursors that land on an earlier shard are covered by a per-device carry kernel at
//           the head of every rank's block (sharded.py device_parts).
struct RouteKind {
    bool h, ad, tt, tk;
    __device__ RouteKind(const DevCols &c, size_t i, bool raw) {
        const uint8_t k = c.kind[i];
        h = k == B2L_KIND_TRANSFER && (raw || (c.nb[i] > 0 && c.h[i] != 0));
        ad = k == B2L_KIND_ALLOC || k == B2L_KIND_DELETE;
        tt = k == B2L_KIND_TRANSFER && c.dst[i] != c.host;
        tk = k == B2L_KIND_KERNEL && c.dst[i] != c.host;
    }
};
struct RouteKeys {
    DevCols c;
    uint32_t G;
    __device__ uint32_t pair_owner(size_t i) const {  // (dst + owner(mix(dst_addr))) % G
        return (uint32_t)(((uint64_t)(uint32_t)c.dst[i] + route_owner(route_splitmix(c.da[i]), G)) % G);
    }
    __device__ uint32_t ut_owner(size_t i) const {
        return route_owner(route_mix((uint64_t)(uint32_t)c.dst[i] ^ (1ull << 40), c.sa[i]), G);
    }
};
constexpr int NEED_W = 4;  // 64-bit words of the per-kernel rank mask (G <= 256)
struct RouteCtx {
    DevCols c;
    bool raw;
    uint32_t G, W;
    const uint32_t *kpos;   // event -> kernel position (target kernels), else NONE
    const uint64_t *need;   // [position][W] ranks that need the kernel
    __device__ uint32_t count(size_t i) const {
        const RouteKind r(c, i, raw);
        uint32_t n = (r.h ? 1u : 0u) + (r.ad || r.tt ? 1u : 0u);
        if (r.tk) {
            const uint64_t *m = need + (size_t)kpos[i] * W;
            for (uint32_t w = 0; w < W; ++w) n += __popcll(m[w]);
        }
        return n;
    }
};
struct RouteCount {
    RouteCtx x;
    __device__ uint32_t operator()(size_t i) const { return x.count(i); }
};
struct RouteStore {  // record keys (destination rank) and record ids (event << 1 | space)
    RouteCtx x;
    uint64_t *key;
    uint32_t *rec;
    __device__ void operator()(size_t i, uint32_t ex, uint32_t) const {
        const DevCols &c = x.c;
        const RouteKind r(c, i, x.raw);
        const RouteKeys K{c, x.G};
        uint32_t o = ex;
        if (r.h) {  // owner of the hash range: (hash * G) >> 64 on the top 32 bits
            key[o] = ((c.h[i] >> 32) * (uint64_t)x.G) >> 32;
            rec[o++] = (uint32_t)(i << 1);
        }
        const uint32_t id = (uint32_t)(i << 1) | 1u;
        if (r.ad) key[o] = K.pair_owner(i), rec[o++] = id;
        if (r.tt) key[o] = K.ut_owner(i), rec[o++] = id;
        if (r.tk) {
            const uint64_t *m = x.need + (size_t)x.kpos[i] * x.W;
            for (uint32_t w = 0; w < x.W; ++w)
                for (uint64_t b = m[w]; b; b &= b - 1) key[o] = 64 * w + __ffsll((long long)b) - 1, rec[o++] = id;
        }
    }
};
__global__ void k_route_total(RouteCtx x, unsigned long long *out) {
    unsigned long long t = 0;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < x.c.n; i += (size_t)gridDim.x * blockDim.x)
        t += x.count(i);
    for (int o = 16; o; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if ((threadIdx.x & 31) == 0 && t) atomicAdd(out, t);
}
// kernel position of every event (target kernels; NONE elsewhere)
__global__ void k_kernel_pos(const uint32_t *__restrict__ kev, uint32_t nk, uint32_t *__restrict__ kpos) {
    for (size_t p = (size_t)blockIdx.x * blockDim.x + threadIdx.x; p < nk; p += (size_t)gridDim.x * blockDim.x)
        kpos[kev[p]] = (uint32_t)p;
}
// first kernel of each device: every rank; each query's cursor kernel: the query's rank
struct NeedFirst {
    KernelIndex KI;
    uint32_t G, W;
    uint64_t *need;
    __device__ void operator()(size_t p) const {
        if (p == 0 || KI.kdev[p] != KI.kdev[p - 1])
            for (uint32_t g = 0; g < G; ++g) need[p * W + g / 64] |= 1ull << (g % 64);
    }
};
struct NeedCursor {
    DevCols c;
    KernelIndex KI;
    RouteKeys K;
    uint32_t W;
    const uint8_t *carry_has;
    const uint64_t *carry_max;
    uint64_t *need;
    __device__ void operator()(size_t i) const {
        const uint8_t k = c.kind[i];
        const bool tt = k == B2L_KIND_TRANSFER && c.dst[i] != c.host;
        const bool ta = k == B2L_KIND_ALLOC && c.dst[i] != c.host;
        if (!tt && !ta) return;
        const uint32_t dev = (uint32_t)c.dst[i];
        const uint64_t t = c.start[i];
        if (carry_has[dev] && carry_max[dev] >= t) return;  // the cursor lands on an earlier shard
        uint32_t lo, hi;
        KI.range(dev, lo, hi);
        const uint32_t p = KI.cursor(lo, hi, t);
        if (p >= hi) return;  // on a later shard (its first kernel goes to every rank)
        const uint32_t r = tt ? K.ut_owner(i) : K.pair_owner(i);
        atomicOr((unsigned long long *)&need[(size_t)p * W + r / 64], 1ull << (r % 64));
    }
};
// rows: rank r's block = its carry kernels, then its records (sorted by rank, event order inside)
__global__ void k_route_rows(DevCols c, uint64_t base, const int64_t *__restrict__ gid,
                             const uint64_t *__restrict__ key, const uint32_t *__restrict__ rec, uint64_t nrec,
                             uint32_t npseudo, int64_t *__restrict__ rows) {
    for (size_t r = (size_t)blockIdx.x * blockDim.x + threadIdx.x; r < nrec; r += (size_t)gridDim.x * blockDim.x) {
        const uint32_t x = rec[r], e = x >> 1;
        int64_t *o = rows + (r + (key[r] + 1) * npseudo) * SH_ROW;
        const uint64_t g = gid ? (uint64_t)gid[e] : base + e;
        o[0] = (int64_t)(g | ((uint64_t)(x & 1u) << 63));
        o[1] = (int64_t)c.seq[e], o[2] = (int64_t)c.start[e], o[3] = (int64_t)c.end[e];
        o[4] = (int64_t)c.sa[e], o[5] = (int64_t)c.da[e], o[6] = (int64_t)c.nb[e], o[7] = (int64_t)c.h[e];
        o[8] = c.src[e], o[9] = c.dst[e], o[10] = c.kind[e], o[11] = c.loc[e];
    }
}
// carry kernel rows (space 1) at the head of every rank's block: start = the shard's first start,
// end = the device's max kernel end on earlier shards
__global__ void k_route_carry_rows(DevCols c, uint64_t base, const unsigned long long *__restrict__ cnt,
                                   const uint32_t *__restrict__ pdev, const uint64_t *__restrict__ carry_max,
                                   uint32_t npseudo, uint32_t G, int64_t *__restrict__ rows) {
    const uint32_t r = blockIdx.x;
    uint64_t off = 0;
    for (uint32_t q = 0; q < r; ++q) off += cnt[q] + npseudo;
    for (uint32_t j = threadIdx.x; j < npseudo; j += blockDim.x) {
        const uint32_t d = pdev[j];
        int64_t *o = rows + (off + j) * SH_ROW;
        o[0] = (int64_t)(base | (1ull << 63));
        o[1] = (int64_t)c.seq[0], o[2] = (int64_t)c.start[0], o[3] = (int64_t)carry_max[d];
        o[4] = 0, o[5] = 0, o[6] = 0, o[7] = 0, o[8] = d, o[9] = d, o[10] = B2L_KIND_KERNEL, o[11] = c.loc[0];
    }
}
__global__ void k_max_data_end(DevCols c, unsigned long long *out) {  // max end over non-kernel events
    unsigned long long m = 0;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < c.n; i += (size_t)gridDim.x * blockDim.x)
        if (c.kind[i] != B2L_KIND_KERNEL && c.end[i] > m) m = c.end[i];
    for (int o = 16; o; o >>= 1) {
        const unsigned long long v = __shfl_xor_sync(0xffffffffu, m, o);
        m = v > m ? v : m;
    }
    if ((threadIdx.x & 31) == 0 && m) atomicMax(out, m);
}
// per target device: has kernels, max kernel end (the carry other shards need)
__global__ void k_kernel_summary(DevCols c, unsigned long long *has, unsigned long long *mx) {
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < c.n; i += (size_t)gridDim.x * blockDim.x)
        if (c.kind[i] == B2L_KIND_KERNEL && c.dst[i] != c.host) {
            const uint32_t d = (uint32_t)c.dst[i];
            if (!has[d]) atomicOr(&has[d], 1ull);
            atomicMax(&mx[d], (unsigned long long)c.end[i]);
        }
}
// OR and AND of two u64 columns (warp-reduced, one atomic per warp and value).
__global__ void k_or_and2(const uint64_t *__restrict__ a, const uint64_t *__restrict__ b, size_t n,
                          unsigned long long *m /*[or a, or b, and a, and b]*/) {
    unsigned long long oa = 0, ob = 0, aa = ~0ull, ab = ~0ull;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        oa |= a[i], ob |= b[i], aa &= a[i], ab &= b[i];
    for (int o = 16; o; o >>= 1) {
        oa |= __shfl_xor_sync(0xffffffffu, oa, o), ob |= __shfl_xor_sync(0xffffffffu, ob, o);
        aa &= __shfl_xor_sync(0xffffffffu, aa, o), ab &= __shfl_xor_sync(0xffffffffu, ab, o);
    }
    if ((threadIdx.x & 31) == 0) atomicOr(m, oa), atomicOr(m + 1, ob), atomicAnd(m + 2, aa), atomicAnd(m + 3, ab);
}
__global__ void k_route_counts(const uint64_t *__restrict__ key, uint64_t n, uint32_t G, unsigned long long *cnt) {
    __shared__ unsigned long long sc[256];
    for (uint32_t g = threadIdx.x; g < G; g += blockDim.x) sc[g] = 0;
    __syncthreads();
    for (size_t r = (size_t)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += (size_t)gridDim.x * blockDim.x)
        atomicAdd(&sc[key[r]], 1ull);
    __syncthreads();
    for (uint32_t g = threadIdx.x; g < G; g += blockDim.x)
        if (sc[g]) atomicAdd(cnt + g, sc[g]);
}
// records (key = destination rank, rec = event << 1 | space) -> rows grouped by destination, event
// order inside (one stable radix pass over the rank), npseudo carry rows ahead of every block;
// per-rank row counts to the host
void route_emit(const DevCols &c, uint64_t base, const int64_t *gid, uint64_t *key, uint32_t *rec, uint32_t nrec,
                uint32_t G, uint32_t npseudo, const uint32_t *pdev, const uint64_t *carry_max, int64_t *d_rows,
                unsigned long long *cnt, uint64_t *h_counts, cudaStream_t s) {
    SortBufs<1> sb;
    DBuf<uint64_t> k2(nrec ? nrec : 1, s);
    DBuf<uint32_t> v2(nrec ? nrec : 1, s);
    if (nrec) {
        sb.k[0].w[0] = key, sb.k[1].w[0] = k2.p, sb.v[0] = rec, sb.v[1] = v2.p, sb.cur = 0;
        radix_sort<1>(sb, nrec, LiveBytes<1>{{live_range(G)}}, s);
        k_route_counts<<<grid_for(nrec, 256, 148 * 4), 256, 0, s>>>(sb.k[sb.cur].w[0], nrec, G, cnt);
        CK_LAUNCH("k_route_counts");
        k_route_rows<<<grid_for(nrec, 256), 256, 0, s>>>(c, base, gid, sb.k[sb.cur].w[0], sb.v[sb.cur], nrec, npseudo,
                                                          d_rows);
        CK_LAUNCH("k_route_rows");
    }
    if (npseudo) {
        k_route_carry_rows<<<G, 64, 0, s>>>(c, base, cnt, pdev, carry_max, npseudo, G, d_rows);
        CK_LAUNCH("k_route_carry_rows");
    }
    std::vector<unsigned long long> hc(G);
    read_back(hc.data(), cnt, G * sizeof(unsigned long long), s);
    for (uint32_t g = 0; g < G; ++g) h_counts[g] = hc[g] + npseudo;
}

int shard_kernel_summary_impl(const b2l_trace_cols *cols, uint64_t *h_has, uint64_t *h_max) {
    if (!cols->device_resident) return fail(B2L_E_INVALID_ARG, "b2l_shard_kernel_summary: device columns only");
    std::lock_guard<std::mutex> lock(g_mu);
    cudaStream_t s = engine_stream();
    ColsUpload up;
    up.load(cols, s);
    const DevCols c = up.d;
    const uint32_t nd = c.ndev > 0 ? (uint32_t)c.ndev : 1;
    DBuf<unsigned long long> hm(2 * nd, s);
    hm.zero();
    if (c.n) {
        k_kernel_summary<<<grid_for(c.n, TPB, 148 * 8), TPB, 0, s>>>(c, hm.p, hm.p + nd);
        CK_LAUNCH("k_kernel_summary");
    }
    std::vector<unsigned long long> h(2 * nd);
    read_back(h.data(), hm.p, 2 * nd * sizeof(unsigned long long), s);
    for (uint32_t d = 0; d < (uint32_t)c.ndev; ++d) h_has[d] = h[d], h_max[d] = h[nd + d];
    return B2L_OK;
}

int shard_route_impl(const b2l_trace_cols *cols, uint32_t G, uint64_t base, uint32_t flags, const uint8_t *h_carry_has,
                     const uint64_t *h_carry_max, int64_t *d_rows, uint64_t *h_counts, uint64_t *h_nrec,
                     uint64_t *h_data_end) {
    if (!cols->device_resident) return fail(B2L_E_INVALID_ARG, "b2l_shard_route: columns must be device-resident");
    if (G == 0 || G > 64 * NEED_W) return fail(B2L_E_INVALID_ARG, "b2l_shard_route: 1..256 ranks");
    std::lock_guard<std::mutex> lock(g_mu);
    cudaStream_t s = engine_stream();
    Arena arena;  // call-scoped scratch (outputs go to the caller's buffers)
    arena.open(cols->n_events <= ARENA_MAX_EVENTS ? ARENA_BASE + cols->n_events * 96 : 0, s);
    ArenaUse arena_use(&arena);
    ColsUpload up;
    up.load(cols, s);
    const DevCols c = up.d;
    const size_t n = c.n;
    const bool raw = (flags & B2L_ANALYZE_RAW_HASHED) != 0;
    const uint32_t nd = c.ndev > 0 ? (uint32_t)c.ndev : 1, W = (G + 63) / 64;
    g_masks = Masks{};
    g_masks.dev = live_range(nd);
    g_masks.idx = live_range(n);
    g_masks.n = n;
    // carry per device (host arrays, NULL = none) and the devices that get a carry kernel
    std::vector<uint8_t> ch(nd, 0);
    std::vector<uint64_t> cm(nd, 0);
    std::vector<uint32_t> pd;
    uint64_t first_start = 0;
    if (n) read_back(&first_start, c.start, sizeof(uint64_t), s);
    for (uint32_t d = 0; d < (uint32_t)c.ndev; ++d) {
        ch[d] = h_carry_has ? h_carry_has[d] : 0, cm[d] = h_carry_max ? h_carry_max[d] : 0;
        if (ch[d] && cm[d] >= first_start && n) pd.push_back(d);
    }
    const uint32_t npseudo = (uint32_t)pd.size();
    DBuf<uint8_t> d_ch(nd, s);
    DBuf<uint64_t> d_cm(nd, s);
    DBuf<uint32_t> d_pd(npseudo ? npseudo : 1, s);
    // pageable sources: the copies are staged before cudaMemcpyAsync returns
    CK(cudaMemcpyAsync(d_ch.p, ch.data(), nd, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(d_cm.p, cm.data(), nd * sizeof(uint64_t), cudaMemcpyHostToDevice, s));
    if (npseudo) CK(cudaMemcpyAsync(d_pd.p, pd.data(), npseudo * sizeof(uint32_t), cudaMemcpyHostToDevice, s));
    DBuf<unsigned long long> cnt(G + 2, s);  // [G] = max data-op end, [G + 1] = records
    cnt.zero();
    // target kernels, grouped by device with their prefix-max ends; which ranks need which kernel
    DBuf<uint32_t> TK(n ? n : 1, s), nk_d(1, s), kpos(n ? n : 1, s);
    const int32_t *dst = c.dst;
    const uint8_t *kind = c.kind;
    const int32_t host = c.host;
    compact(n, [=] __device__(size_t i) { return kind[i] == B2L_KIND_KERNEL && dst[i] != host; }, TK.p, nk_d.p, s);
    const uint32_t nK = n ? read_u32(nk_d.p, s) : 0;
    KernelIndexStore kis(nK, s);
    build_kernel_index(kis, c, TK.p, nK, s);
    DBuf<uint64_t> need((size_t)(nK ? nK : 1) * W, s);
    need.zero();
    if (nK) {
        k_kernel_pos<<<grid_for(nK, TPB), TPB, 0, s>>>(kis.kev.p, nK, kpos.p);
        CK_LAUNCH("k_kernel_pos");
        for_each(nK, NeedFirst{kis.KI, G, W, need.p}, s);
        for_each(n, NeedCursor{c, kis.KI, RouteKeys{c, G}, W, d_ch.p, d_cm.p, need.p}, s);
    }
    const RouteCtx x{c, raw, G, W, kpos.p, need.p};
    if (n) {
        k_max_data_end<<<grid_for(n, TPB, 148 * 8), TPB, 0, s>>>(c, cnt.p + G);
        CK_LAUNCH("k_max_data_end");
        k_route_total<<<grid_for(n, TPB, 148 * 8), TPB, 0, s>>>(x, cnt.p + G + 1);
        CK_LAUNCH("k_route_total");
    }
    unsigned long long hv[2] = {0, 0};
    read_back(hv, cnt.p + G, sizeof(hv), s);
    *h_data_end = hv[0];
    if (hv[1] >= 0xFFFFFFFFull) return fail(B2L_E_INVALID_ARG, "b2l_shard_route: too many records for one call");
    const uint32_t nrec = (uint32_t)hv[1];
    *h_nrec = nrec + (uint64_t)G * npseudo;
    for (uint32_t g = 0; g < G; ++g) h_counts[g] = 0;
    if (!d_rows) return B2L_OK;  // sizing call
    DBuf<uint64_t> key(nrec ? nrec : 1, s);
    DBuf<uint32_t> rec(nrec ? nrec : 1, s);
    if (nrec) scan<SumU32>(n, RouteCount{x}, RouteStore{x, key.p, rec.p}, s);
    route_emit(c, base, nullptr, key.p, rec.p, nrec, G, npseudo, d_pd.p, d_cm.p, d_rows, cnt.p, h_counts, s);
    return B2L_OK;
}

// The second exchange: every event of a pair (the alloc, and its delete unless synthetic) of a
// device sub-trace goes to the owner of the pair's RA key (alloc src_addr, dst_device, bytes:
// detectors.py:170-176), as space-1 rows; global indices from gid[].
struct PairDestOp {
    DevCols c;
    const uint32_t *pa, *pd;
    uint32_t G;
    uint32_t *dest;
    __device__ void operator()(size_t p) const {
        const uint32_t a = pa[p];
        const uint32_t o = route_owner(route_mix(c.sa[a], route_mix((uint64_t)(uint32_t)c.dst[a], c.nb[a])), G);
        dest[a] = o;
        if (pd[p] != NONE) dest[pd[p]] = o;
    }
};
struct DestPred {
    const uint32_t *dest;
    __device__ bool operator()(size_t i) const { return dest[i] != NONE; }
};
int shard_route_pairs_impl(const b2l_trace_cols *cols, const int64_t *gid, const uint32_t *pa, const uint32_t *pd,
                           uint64_t np, uint32_t G, int64_t *d_rows, uint64_t *h_counts, uint64_t *h_nrec) {
    if (!cols->device_resident) return fail(B2L_E_INVALID_ARG, "b2l_shard_route_pairs: columns must be device-resident");
    if (G == 0 || G > 256) return fail(B2L_E_INVALID_ARG, "b2l_shard_route_pairs: 1..256 ranks");
    std::lock_guard<std::mutex> lock(g_mu);
    cudaStream_t s = engine_stream();
    ColsUpload up;
    up.load(cols, s);
    const DevCols c = up.d;
    const size_t n = c.n;
    for (uint32_t g = 0; g < G; ++g) h_counts[g] = 0;
    *h_nrec = 0;
    if (!n || !np) return B2L_OK;
    Arena arena;
    arena.open(n <= ARENA_MAX_EVENTS ? ARENA_BASE + n * 64 : 0, s);
    ArenaUse arena_use(&arena);
    DBuf<uint32_t> dest(n, s), rec(n, s), tot(1, s);
    dev_memset(dest.p, 0xFF, n * sizeof(uint32_t), s);
    for_each(np, PairDestOp{c, pa, pd, G, dest.p}, s);
    compact(n, DestPred{dest.p}, rec.p, tot.p, s);
    const uint32_t nrec = read_u32(tot.p, s);
    *h_nrec = nrec;
    if (!d_rows || !nrec) return B2L_OK;
    DBuf<uint64_t> key(nrec, s);
    {
        uint64_t *k = key.p;
        uint32_t *r = rec.p;
        const uint32_t *d = dest.p;
        for_each(nrec, [=] __device__(size_t q) {
            const uint32_t e = r[q];
            k[q] = d[e];
            r[q] = (e << 1) | 1u;
        }, s);
    }
    DBuf<unsigned long long> cnt(G, s);
    cnt.zero();
    route_emit(c, 0, gid, key.p, rec.p, nrec, G, 0, nullptr, nullptr, d_rows, cnt.p, h_counts, s);
    return B2L_OK;
}

// Received rows of one key space -> SoA device columns (rows arrive ordered by global index: each
// source rank sends its records in event order, ranks hold increasing seq ranges).
struct SpacePred {
    const int64_t *rows;
    uint32_t space;
    __device__ bool operator()(size_t r) const { return ((uint64_t)rows[r * SH_ROW] >> 63) == space; }
};
struct UnpackOut {
    int64_t *gid, *seq, *start, *end, *sa, *da, *nb, *h;
    int32_t *src, *dst;
    uint8_t *kind;
    int32_t *loc;
};
int shard_unpack_impl(const int64_t *d_rows, uint64_t nrows, uint32_t space, const UnpackOut &o, uint64_t *h_n) {
    std::lock_guard<std::mutex> lock(g_mu);
    cudaStream_t s = engine_stream();
    Arena arena;
    arena.open(nrows <= ARENA_MAX_EVENTS ? ARENA_BASE + nrows * 32 : 0, s);
    ArenaUse arena_use(&arena);
    DBuf<uint32_t> pos(nrows ? nrows : 1, s), cnt(1, s);
    compact(nrows, SpacePred{d_rows, space}, pos.p, cnt.p, s);
    uint32_t m = 0;
    read_back(&m, cnt.p, sizeof(m), s);
    const uint32_t *P = pos.p;
    const UnpackOut O = o;
    for_each(m, [=] __device__(size_t q) {
        const int64_t *r = d_rows + (size_t)P[q] * SH_ROW;
        O.gid[q] = r[0] & 0x7FFFFFFFFFFFFFFFll;
        O.seq[q] = r[1], O.start[q] = r[2], O.end[q] = r[3], O.sa[q] = r[4], O.da[q] = r[5], O.nb[q] = r[6];
        O.h[q] = r[7], O.src[q] = (int32_t)r[8], O.dst[q] = (int32_t)r[9], O.kind[q] = (uint8_t)r[10];
        O.loc[q] = (int32_t)r[11];
    }, s);
    CK(cudaStreamSynchronize(s));
    *h_n = m;
    return B2L_OK;
}

}  // namespace ana
}  // namespace b2l

extern "C" {

int b2l_analyze(const b2l_trace_cols *cols, uint32_t flags, b2l_findings **out) {
    if (!cols || !out) return b2l::fail(B2L_E_INVALID_ARG, "null argument");
    *out = nullptr;
    try {
        return b2l::ana::analyze_impl(cols, flags, 0, out);
    } catch (const b2l::EngineErr &e) {
        return b2l::fail(e.code, e.msg);
    } catch (const std::exception &e) {
        return b2l::fail(B2L_E_CUDA, e.what());
    }
}

int b2l_analyze_ex(const b2l_trace_cols *cols, uint32_t flags, uint64_t synthetic_end_ns, b2l_findings **out) {
    if (!cols || !out) return b2l::fail(B2L_E_INVALID_ARG, "null argument");
    *out = nullptr;
    try {
        return b2l::ana::analyze_impl(cols, flags, synthetic_end_ns, out);
    } catch (const b2l::EngineErr &e) {
        return b2l::fail(e.code, e.msg);
    } catch (const std::exception &e) {
        return b2l::fail(B2L_E_CUDA, e.what());
    }
}

void b2l_findings_free(b2l_findings *f) { b2l::ana::findings_free(f); }

int b2l_savings_compute(const b2l_trace_cols *cols, const b2l_findings *f, b2l_savings **out) {
    if (!cols || !f || !out) return b2l::fail(B2L_E_INVALID_ARG, "null argument");
    *out = nullptr;
    try {
        return b2l::ana::savings_impl(cols, f, out);
    } catch (const b2l::EngineErr &e) {
        return b2l::fail(e.code, e.msg);
    }
}

void b2l_savings_free(b2l_savings *s) { b2l::ana::savings_free(s); }

int b2l_stable_sort_u32(const uint32_t *keys, uint64_t n, uint32_t *out_perm) {
    if (n && (!keys || !out_perm)) return b2l::fail(B2L_E_INVALID_ARG, "null argument");
    if (n == 0) return B2L_OK;
    try {
        using namespace b2l;
        std::lock_guard<std::mutex> lock(ana::g_mu);
        cudaStream_t s = ana::engine_stream();
        DBuf<uint32_t> k32(n, s);
        CK(cudaMemcpyAsync(k32.p, keys, n * sizeof(uint32_t), cudaMemcpyHostToDevice, s));
        SortStore<1> st(n, s);
        uint64_t *k0 = st.in_key(0);
        uint32_t *v = st.in_val();
        const uint32_t *kk = k32.p;
        ana::for_each(n, [=] __device__(size_t i) { k0[i] = kk[i], v[i] = (uint32_t)i; }, s);
        radix_sort<1>(st.b, n, LiveBytes<1>{{0x0F}}, s);
        read_back(out_perm, st.val(), n * sizeof(uint32_t), s);
        return B2L_OK;
    } catch (const b2l::EngineErr &e) {
        return b2l::fail(e.code, e.msg);
    }
}

int b2l_stable_sort_u64(const uint64_t *keys, uint64_t n, uint32_t strategy, uint32_t *out_perm) {
    if (n && (!keys || !out_perm)) return b2l::fail(B2L_E_INVALID_ARG, "null argument");
    if (strategy > 1 && (strategy < 16 || strategy > 23)) return b2l::fail(B2L_E_INVALID_ARG, "unknown strategy");
    if (n == 0) return B2L_OK;
    try {
        using namespace b2l;
        std::lock_guard<std::mutex> lock(ana::g_mu);
        cudaStream_t s = ana::engine_stream();
        SortStore<1> st(n, s);
        CK(cudaMemcpyAsync(st.in_key(0), keys, n * sizeof(uint64_t), cudaMemcpyHostToDevice, s));
        uint32_t *v = st.in_val();
        ana::for_each(n, [=] __device__(size_t i) { v[i] = (uint32_t)i; }, s);
        uint64_t o = 0, a = ~0ull;
        for (uint64_t i = 0; i < n; ++i) o |= keys[i], a &= keys[i];
        const uint8_t live = live_mask(o ^ a);
        if (strategy == 0) radix_sort<1>(st.b, n, LiveBytes<1>{{live}}, s);
        else if (strategy == 1) radix_sort_wide(st.b, n, live, s);
        else radix_sort_prefix(st.b, n, live, (int)strategy - 16, s);
        read_back(out_perm, st.val(), n * sizeof(uint32_t), s);
        return B2L_OK;
    } catch (const b2l::EngineErr &e) {
        return b2l::fail(e.code, e.msg);
    }
}

int b2l_sort_u64_pairs_device(const uint64_t *d_k0, const uint64_t *d_k1, uint64_t n, uint32_t *d_perm) {
    if (n && (!d_k0 || !d_k1 || !d_perm)) return b2l::fail(B2L_E_INVALID_ARG, "null argument");
    if (n == 0) return B2L_OK;
    try {
        using namespace b2l;
        std::lock_guard<std::mutex> lock(ana::g_mu);
        cudaStream_t s = ana::engine_stream();
        CK(cudaStreamSynchronize(cudaStreamLegacy));  // inputs written on the caller's stream
        Arena arena;
        arena.open(n <= ana::ARENA_MAX_EVENTS ? ana::ARENA_BASE + n * 64 : 0, s);
        ArenaUse arena_use(&arena);
        SortStore<2> st(n, s);
        dev_copy(st.in_key(0), d_k0, n * sizeof(uint64_t), s);
        dev_copy(st.in_key(1), d_k1, n * sizeof(uint64_t), s);
        uint32_t *v = st.in_val();
        ana::for_each(n, [=] __device__(size_t i) { v[i] = (uint32_t)i; }, s);
        DBuf<unsigned long long> m(4, s);
        dev_memset(m.p, 0, 2 * sizeof(unsigned long long), s);
        dev_memset(m.p + 2, 0xFF, 2 * sizeof(unsigned long long), s);
        b2l::ana::k_or_and2<<<grid_for(n, 256, 148 * 4), 256, 0, s>>>(d_k0, d_k1, n, m.p);  // live digit bytes
        CK_LAUNCH("k_or_and2");
        unsigned long long hm[4];
        read_back(hm, m.p, sizeof(hm), s);
        radix_sort<2>(st.b, n, LiveBytes<2>{{live_mask(hm[0] ^ hm[2]), live_mask(hm[1] ^ hm[3])}}, s);
        dev_copy(d_perm, st.val(), n * sizeof(uint32_t), s);
        CK(cudaStreamSynchronize(s));
        return B2L_OK;
    } catch (const b2l::EngineErr &e) {
        return b2l::fail(e.code, e.msg);
    }
}

int b2l_sort_u64_pairs(const uint64_t *k0, const uint64_t *k1, uint64_t n, uint32_t *out_perm) {
    if (n && (!k0 || !k1 || !out_perm)) return b2l::fail(B2L_E_INVALID_ARG, "null argument");
    if (n == 0) return B2L_OK;
    try {
        using namespace b2l;
        std::lock_guard<std::mutex> lock(ana::g_mu);
        cudaStream_t s = ana::engine_stream();
        SortStore<2> st(n, s);
        CK(cudaMemcpyAsync(st.in_key(0), k0, n * sizeof(uint64_t), cudaMemcpyHostToDevice, s));
        CK(cudaMemcpyAsync(st.in_key(1), k1, n * sizeof(uint64_t), cudaMemcpyHostToDevice, s));
        uint32_t *v = st.in_val();
        ana::for_each(n, [=] __device__(size_t i) { v[i] = (uint32_t)i; }, s);
        // live digit bytes from an OR/AND pass over the (host) keys
        uint64_t o0 = 0, a0 = ~0ull, o1 = 0, a1 = ~0ull;
        for (uint64_t i = 0; i < n; ++i) o0 |= k0[i], a0 &= k0[i], o1 |= k1[i], a1 &= k1[i];
        radix_sort<2>(st.b, n, LiveBytes<2>{{live_mask(o0 ^ a0), live_mask(o1 ^ a1)}}, s);
        read_back(out_perm, st.val(), n * sizeof(uint32_t), s);
        return B2L_OK;
    } catch (const b2l::EngineErr &e) {
        return b2l::fail(e.code, e.msg);
    }
}

int b2l_shard_kernel_summary(const b2l_trace_cols *cols, uint64_t *has_kernels, uint64_t *max_kernel_end) {
    if (!cols || !has_kernels || !max_kernel_end) return b2l::fail(B2L_E_INVALID_ARG, "null argument");
    try {
        return b2l::ana::shard_kernel_summary_impl(cols, has_kernels, max_kernel_end);
    } catch (const b2l::EngineErr &e) {
        return b2l::fail(e.code, e.msg);
    }
}

int b2l_shard_route(const b2l_trace_cols *cols, uint32_t n_ranks, uint64_t base, uint32_t flags,
                    const uint8_t *carry_has, const uint64_t *carry_max_end, int64_t *d_rows, uint64_t *counts,
                    uint64_t *n_rows, uint64_t *data_end_ns) {
    if (!cols || !counts || !n_rows || !data_end_ns) return b2l::fail(B2L_E_INVALID_ARG, "null argument");
    try {
        return b2l::ana::shard_route_impl(cols, n_ranks, base, flags, carry_has, carry_max_end, d_rows, counts,
                                          n_rows, data_end_ns);
    } catch (const b2l::EngineErr &e) {
        return b2l::fail(e.code, e.msg);
    }
}

int b2l_shard_route_pairs(const b2l_trace_cols *cols, const int64_t *d_gid, const uint32_t *d_pair_alloc,
                          const uint32_t *d_pair_delete, uint64_t n_pairs, uint32_t n_ranks, int64_t *d_rows,
                          uint64_t *counts, uint64_t *n_rows) {
    if (!cols || !d_gid || (n_pairs && (!d_pair_alloc || !d_pair_delete)) || !counts || !n_rows)
        return b2l::fail(B2L_E_INVALID_ARG, "null argument");
    try {
        return b2l::ana::shard_route_pairs_impl(cols, d_gid, d_pair_alloc, d_pair_delete, n_pairs, n_ranks, d_rows,
                                                counts, n_rows);
    } catch (const b2l::EngineErr &e) {
        return b2l::fail(e.code, e.msg);
    }
}

int b2l_shard_unpack(const int64_t *d_rows, uint64_t n_rows, uint32_t space, int64_t *const *d_cols,
                     uint64_t *n_out) {
    if ((n_rows && !d_rows) || !d_cols || !n_out || space > 1) return b2l::fail(B2L_E_INVALID_ARG, "bad argument");
    try {
        b2l::ana::UnpackOut o{d_cols[0], d_cols[1], d_cols[2], d_cols[3], d_cols[4], d_cols[5], d_cols[6],
                              d_cols[7], (int32_t *)d_cols[8], (int32_t *)d_cols[9], (uint8_t *)d_cols[10],
                              (int32_t *)d_cols[11]};
        return b2l::ana::shard_unpack_impl(d_rows, n_rows, space, o, n_out);
    } catch (const b2l::EngineErr &e) {
        return b2l::fail(e.code, e.msg);
    }
}

int b2l_lookup_seqs(const b2l_trace_cols *cols, const uint64_t *seqs, uint64_t n, uint32_t *out_index) {
    if (!cols || (n && (!seqs || !out_index))) return b2l::fail(B2L_E_INVALID_ARG, "null argument");
    try {
        return b2l::ana::lookup_impl(cols, seqs, n, out_index);
    } catch (const b2l::EngineErr &e) {
        return b2l::fail(e.code, e.msg);
    }
}

}  // extern "C"
