// K1 hash_batch_seq: one sequential FNV fold per buffer, many buffers in flight.
//
// Reference semantics: dmlens.hashing._fold64 + make_hasher
// (/root/reference/pkg/src/dmlens/hashing.py:34-64).  The fold is a strict
// serial chain per buffer, so parallelism is across buffers: every lane owns
// one chain and walks a static, longest-first list of buffers (lane g takes
// order[g], order[g+T], ...).  Bytes reach the lane through a private ring of
// S shared-memory slots filled by 1-D TMA bulk copies (cp.async.bulk +
// per-slot mbarrier), so each HBM byte is read exactly once, in 16-B aligned
// bulk transactions, while the lane hashes the previous slot from SMEM with
// conflict-free 128-bit LDS.
//
// Alignment: the lane's byte stream of a buffer starts at the 16-B aligned
// address A0 <= start; words are re-formed from byte `start` with a funnel
// shift when start % 8 != 0.  Reads never leave the 16-B aligned segments
// that contain buffer bytes, so they never cross a page the buffer does not
// touch.
#include <algorithm>
#include <cstdlib>

#include "b2l_common.cuh"

namespace b2l {

namespace {


struct BufCursor {
    uint64_t idx;    // buffer index (for digests) ; UINT64_MAX = exhausted
    uint64_t a0;     // 16-B aligned stream start address
    uint64_t L;      // stream length in bytes (multiple of 16)
    uint64_t pos;    // next stream byte
    uint64_t n;      // payload length
    uint32_t m;      // start - a0  (0..15)
};

__device__ __forceinline__ void cursor_load(BufCursor &c, const uint64_t *__restrict__ ptrs,
                                            const uint64_t *__restrict__ lens,
                                            const uint32_t *__restrict__ order, uint64_t k, uint64_t n_bufs) {
    if (k >= n_bufs) {
        c.idx = ~0ull;
        return;
    }
    uint64_t idx = order ? (uint64_t)__ldg(order + k) : k;
    uint64_t start = __ldg(ptrs + idx);
    uint64_t len = __ldg(lens + idx);
    c.idx = idx;
    c.a0 = start & ~15ull;
    c.m = (uint32_t)(start - c.a0);
    c.n = len;
    c.L = len ? (((start + len + 15ull) & ~15ull) - c.a0) : 0;
    c.pos = 0;
}

// Hash one staged chunk (`bytes` stream bytes starting at stream offset cs.pos) into (h, prev).
// Word j of the payload is stream u64 q = q0 + j, or -- when start % 8 != 0 -- the funnel of
// stream u64s (q0+j, q0+j+1), emitted at q0+j+1.
// PF (one chain per warp, registers to spare): the whole chunk is loaded into registers before
// the chain starts, so no LDS latency lands on the chain's critical path.
template <int CH, bool PF = false>
__device__ __forceinline__ void consume_chunk(const BufCursor &cs, uint32_t bytes, const uint4 *__restrict__ src,
                                              uint64_t &h, uint64_t &prev) {
    const uint32_t r = cs.m & 7u;
    const uint64_t qb = (cs.m >> 3) + (r ? 1 : 0);
    const uint64_t nw = (cs.n + 7) >> 3;
    const uint64_t qe = qb + nw;  // exclusive
    const uint64_t qc = cs.pos >> 3;
    const uint32_t nu = bytes >> 3;
    const bool interior = qc >= qb && qc + nu < qe && cs.pos + bytes < cs.L;  // full, not the last chunk
    if (PF && r == 0 && interior) {
        uint4 v[CH / 16];
#pragma unroll
        for (int i = 0; i < CH / 16; ++i) v[i] = src[i];
        uint32_t hl = (uint32_t)h, hh = (uint32_t)(h >> 32);
#pragma unroll
        for (int i = 0; i < CH / 16; ++i) {
            fnv_step32_lat(hl, hh, v[i].x, v[i].y);
            fnv_step32_lat(hl, hh, v[i].z, v[i].w);
        }
        h = ((uint64_t)hh << 32) | hl;
    } else if (r == 0 && interior) {
        uint32_t hl = (uint32_t)h, hh = (uint32_t)(h >> 32);
#pragma unroll 8
        for (uint32_t i = 0; i < (uint32_t)CH / 16; ++i) {
            uint4 v = src[i];
            fnv_step32(hl, hh, v.x, v.y);
            fnv_step32(hl, hh, v.z, v.w);
        }
        h = ((uint64_t)hh << 32) | hl;
    } else if (r != 0 && interior) {
        const uint32_t sh = r * 8;
        uint32_t hl = (uint32_t)h, hh = (uint32_t)(h >> 32);
#pragma unroll 4
        for (uint32_t i = 0; i < (uint32_t)CH / 16; ++i) {
            uint4 v = src[i];
            uint64_t u0 = ((uint64_t)v.y << 32) | v.x, u1 = ((uint64_t)v.w << 32) | v.z;
            uint64_t w0 = (prev >> sh) | (u0 << (64 - sh));
            uint64_t w1 = (u0 >> sh) | (u1 << (64 - sh));
            if (PF) {
                fnv_step32_lat(hl, hh, (uint32_t)w0, (uint32_t)(w0 >> 32));
                fnv_step32_lat(hl, hh, (uint32_t)w1, (uint32_t)(w1 >> 32));
            } else {
                fnv_step32(hl, hh, (uint32_t)w0, (uint32_t)(w0 >> 32));
                fnv_step32(hl, hh, (uint32_t)w1, (uint32_t)(w1 >> 32));
            }
            prev = u1;
        }
        h = ((uint64_t)hh << 32) | hl;
    } else {
        const uint32_t sh = r * 8;
        const uint32_t tailb = (uint32_t)(cs.n & 7);
        for (uint32_t i = 0; i < nu; ++i) {
            const uint32_t *p32 = reinterpret_cast<const uint32_t *>(src) + 2 * i;
            uint64_t u = ((uint64_t)p32[1] << 32) | p32[0];
            uint64_t q = qc + i;
            if (q >= qb && q < qe) {
                uint64_t w = r ? ((prev >> sh) | (u << (64 - sh))) : u;
                if (q == qe - 1 && tailb) w &= (1ull << (8 * tailb)) - 1;
                h = fnv_step(h, w);
            }
            prev = u;
        }
        // misaligned payload whose last (partial) word lies wholly inside the final stream
        // u64: the stream ends before that word's emission point -- emit it here.
        if (r && qc + nu == (cs.L >> 3) && qe > (cs.L >> 3))
            h = fnv_step(h, (prev >> sh) & ((1ull << (8 * tailb)) - 1));
    }
}

__device__ __forceinline__ uint32_t chunk_bytes(const BufCursor &c, int ch) {
    uint64_t rem = c.L - c.pos;
    return rem < (uint64_t)ch ? (uint32_t)rem : (uint32_t)ch;
}

// ============================================================================ variant A
// Per-lane TMA ring: each lane issues its own cp.async.bulk per chunk (ptxas serialises the
// 32 lanes' bulk copies in a uniform-register loop), completion on a per-lane mbarrier.
template <int NT, int CH, int S>
struct HashSmem {
    static constexpr int SLOT = CH + 16;  // stride == 16 mod 128: conflict-free LDS.128 across 8 lanes
    static constexpr size_t data_bytes = (size_t)S * NT * SLOT;
    static constexpr size_t bytes = data_bytes + (size_t)S * NT * sizeof(uint64_t);
};

template <int NT, int CH, int S>
__global__ void __launch_bounds__(NT) k_hash_seq(const uint64_t *__restrict__ ptrs, const uint64_t *__restrict__ lens,
                                                 const uint32_t *__restrict__ order, uint64_t n_bufs,
                                                 uint64_t *__restrict__ digests) {
    using SM = HashSmem<NT, CH, S>;
    extern __shared__ __align__(128) uint8_t smem[];
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem + SM::data_bytes);
    const int tid = threadIdx.x;
    const uint64_t T = (uint64_t)gridDim.x * NT;
    const uint64_t g = (uint64_t)blockIdx.x * NT + tid;

#pragma unroll
    for (int s = 0; s < S; ++s) mbar_init(&bars[s * NT + tid], 1);
    fence_mbar_init();
    __syncthreads();

    const uint64_t policy = l2_policy_evict_first();
    auto slot_ptr = [&](int s) { return smem + ((size_t)s * NT + tid) * SM::SLOT; };

    BufCursor ld;  // loader: S chunks ahead of the consumer
    uint64_t ld_k = g;
    cursor_load(ld, ptrs, lens, order, ld_k, n_bufs);
    auto issue = [&](int s) {
        while (ld.idx != ~0ull && ld.pos >= ld.L) {
            ld_k += T;
            cursor_load(ld, ptrs, lens, order, ld_k, n_bufs);
        }
        if (ld.idx == ~0ull) return;
        const uint32_t bytes = chunk_bytes(ld, CH);
        uint64_t *bar = &bars[s * NT + tid];
        mbar_expect_tx(bar, bytes);
        bulk_g2s(slot_ptr(s), reinterpret_cast<const void *>(ld.a0 + ld.pos), bytes, bar, policy);
        ld.pos += bytes;
    };
#pragma unroll
    for (int s = 0; s < S; ++s) issue(s);

    BufCursor cs;
    uint64_t cs_k = g;
    cursor_load(cs, ptrs, lens, order, cs_k, n_bufs);
    uint64_t h = FNV_OFFSET, prev = 0;
    uint32_t phase_bits = 0;
    int s = 0;
    while (cs.idx != ~0ull) {
        if (cs.L == 0) {  // zero-length payload: reserved digest 0 (host raises EmptyPayload)
            digests[cs.idx] = 0;
            cs_k += T;
            cursor_load(cs, ptrs, lens, order, cs_k, n_bufs);
            continue;
        }
        const uint32_t bytes = chunk_bytes(cs, CH);
        mbar_wait(&bars[s * NT + tid], (phase_bits >> s) & 1u);
        phase_bits ^= 1u << s;
        consume_chunk<CH>(cs, bytes, reinterpret_cast<const uint4 *>(slot_ptr(s)), h, prev);
        cs.pos += bytes;
        issue(s);
        s = (s + 1 == S) ? 0 : s + 1;
        if (cs.pos >= cs.L) {
            digests[cs.idx] = finish_digest(h, cs.n);
            h = FNV_OFFSET;
            prev = 0;
            cs_k += T;
            cursor_load(cs, ptrs, lens, order, cs_k, n_bufs);
        }
    }
}

// ============================================================================ variant B
// Warp-cooperative ring: a warp moves the 32 lanes' next chunks with coalesced 16-B
// cp.async (LDGSTS, L1 bypass) -- each warp instruction covers 512 contiguous-per-buffer
// bytes of 32*16/CH buffers -- S-1 rounds ahead of the round being hashed.  No per-lane
// copy descriptors, so many more chains fit per SM than in variant A.
template <int WARPS, int CH, int S>
struct CoopSmem {
    static constexpr int SLOT = CH + 16;
    static constexpr size_t warp_bytes = (size_t)S * 32 * SLOT;
    static constexpr size_t bytes = warp_bytes * WARPS;
};

__device__ __forceinline__ void cp_async16(uint32_t dst, uint64_t src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

template <int WARPS, int CH, int S>
__global__ void __launch_bounds__(WARPS * 32) k_hash_coop(const uint64_t *__restrict__ ptrs,
                                                          const uint64_t *__restrict__ lens,
                                                          const uint32_t *__restrict__ order, uint64_t n_bufs,
                                                          uint64_t *__restrict__ digests) {
    static_assert(CH % 128 == 0 && CH <= 512 && S >= 2, "chunk must be 128..512 B");
    using SM = CoopSmem<WARPS, CH, S>;
    constexpr int PIECES = CH / 16;            // 16-B pieces per chunk
    constexpr int PER_INSTR = 32 / PIECES;     // chunks moved per warp instruction
    extern __shared__ __align__(128) uint8_t smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint64_t T = (uint64_t)gridDim.x * WARPS * 32;
    const uint64_t g = ((uint64_t)blockIdx.x * WARPS + warp) * 32 + lane;
    uint8_t *wbase = smem + warp * SM::warp_bytes;
    const uint32_t wbase_s = smem_u32(wbase);

    BufCursor ld;
    uint64_t ld_k = g;
    cursor_load(ld, ptrs, lens, order, ld_k, n_bufs);
    auto issue_round = [&](int stage) {
        while (ld.idx != ~0ull && ld.pos >= ld.L) {
            ld_k += T;
            cursor_load(ld, ptrs, lens, order, ld_k, n_bufs);
        }
        uint64_t my_addr = 0;
        uint32_t my_bytes = 0;
        if (ld.idx != ~0ull) {
            my_bytes = chunk_bytes(ld, CH);
            my_addr = ld.a0 + ld.pos;
            ld.pos += my_bytes;
        }
        const int p = lane % PIECES;
#pragma unroll
        for (int i = 0; i < PIECES; ++i) {
            const int j = i * PER_INSTR + lane / PIECES;
            const uint64_t a = __shfl_sync(0xffffffffu, my_addr, j);
            const uint32_t b = __shfl_sync(0xffffffffu, my_bytes, j);
            if ((uint32_t)(16 * p) < b)
                cp_async16(wbase_s + (uint32_t)((stage * 32 + j) * SM::SLOT + 16 * p), a + 16 * p);
        }
        cp_async_commit();
    };
#pragma unroll
    for (int s = 0; s < S - 1; ++s) issue_round(s);

    BufCursor cs;
    uint64_t cs_k = g;
    cursor_load(cs, ptrs, lens, order, cs_k, n_bufs);
    uint64_t h = FNV_OFFSET, prev = 0;
    int stage = 0;
    for (;;) {
        while (cs.idx != ~0ull && cs.L == 0) {  // zero-length payloads take no round
            digests[cs.idx] = 0;
            cs_k += T;
            cursor_load(cs, ptrs, lens, order, cs_k, n_bufs);
        }
        if (!__any_sync(0xffffffffu, cs.idx != ~0ull)) break;
        cp_async_wait<S - 2>();
        __syncwarp();
        issue_round(stage == 0 ? S - 1 : stage - 1);
        if (cs.idx != ~0ull) {
            const uint32_t bytes = chunk_bytes(cs, CH);
            consume_chunk<CH>(cs, bytes, reinterpret_cast<const uint4 *>(wbase + (stage * 32 + lane) * SM::SLOT), h,
                              prev);
            cs.pos += bytes;
            if (cs.pos >= cs.L) {
                digests[cs.idx] = finish_digest(h, cs.n);
                h = FNV_OFFSET;
                prev = 0;
                cs_k += T;
                cursor_load(cs, ptrs, lens, order, cs_k, n_bufs);
            }
        }
        stage = (stage + 1 == S) ? 0 : stage + 1;
    }
    cp_async_wait<0>();
}

// Launch configurations (lanes per CTA, chunk bytes, ring depth).  Selected at
// first use; B2L_HASH_CFG=<i> overrides (used by the tuning sweep).
// ============================================================================ variant W
// One WARP per buffer, for batches too small to fill the GPU with lanes (C1): all 32 lanes
// stream the buffer's next 512-B chunk with one coalesced 16-B cp.async each (one instruction
// per chunk instead of 32 shuffled ones), an S-deep ring per warp, and lane 0 runs the serial
// chain out of shared memory.  A lone chain is then bound by its own dependency latency, not by
// the cooperative ring's per-round issue cost (the longest C1 buffer sets the batch time).
template <int WARPS, int S>
__global__ void __launch_bounds__(WARPS * 32) k_hash_warp(const uint64_t *__restrict__ ptrs,
                                                          const uint64_t *__restrict__ lens,
                                                          const uint32_t *__restrict__ order, uint64_t n_bufs,
                                                          uint64_t *__restrict__ digests, uint64_t primary) {
    constexpr int CH = 512;
    extern __shared__ __align__(128) uint8_t smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint8_t *ring = smem + (size_t)warp * S * CH;
    const uint32_t ring_s = smem_u32(ring);
    // Round r of warp w takes list position r*W + w, or r*W + (W-1-w) on odd rounds (boustrophedon
    // over a longest-first order: the warp holding the longest buffer gets the shortest of the next
    // round, so per-warp totals stay close).  With `primary` = P > 0, warps 0..P-1 (the first CTA
    // of every SM) take the P longest buffers alone and the other warps deal out the rest, so the
    // longest chains share their schedulers only with short work.
    const uint64_t wg0 = (uint64_t)blockIdx.x * WARPS + warp;
    const bool prim = wg0 < primary;
    const uint64_t W = prim ? 1 : (uint64_t)gridDim.x * WARPS - primary;
    const uint64_t wg = prim ? 0 : wg0 - primary, base = prim ? wg0 : primary;
    const uint64_t rounds = prim ? 1 : ~0ull;
    for (uint64_t r = 0; r < rounds && base + r * W < n_bufs; ++r) {
        const uint64_t k = base + r * W + ((r & 1) ? W - 1 - wg : wg);
        if (k >= n_bufs) continue;
        BufCursor ld, cs;
        cursor_load(ld, ptrs, lens, order, k, n_bufs);
        cs = ld;
        if (cs.L == 0) {
            if (lane == 0) digests[cs.idx] = 0;
            continue;
        }
        auto issue = [&](int st) {
            if (ld.pos < ld.L) {
                const uint32_t b = chunk_bytes(ld, CH);
                if ((uint32_t)(16 * lane) < b) cp_async16(ring_s + (uint32_t)(st * CH + 16 * lane), ld.a0 + ld.pos + 16 * lane);
                ld.pos += b;
            }
            cp_async_commit();
        };
#pragma unroll
        for (int st = 0; st < S - 1; ++st) issue(st);
        uint64_t h = FNV_OFFSET, prev = 0;
        int st = 0;
        while (cs.pos < cs.L) {
            cp_async_wait<S - 2>();
            __syncwarp();
            issue(st == 0 ? S - 1 : st - 1);
            const uint32_t bytes = chunk_bytes(cs, CH);
            if (lane == 0) consume_chunk<CH, true>(cs, bytes, reinterpret_cast<const uint4 *>(ring + st * CH), h, prev);
            cs.pos += bytes;
            st = st + 1 == S ? 0 : st + 1;
            __syncwarp();  // the slot is re-filled only after lane 0 has read it
        }
        cp_async_wait<0>();
        __syncwarp();
        if (lane == 0) digests[cs.idx] = finish_digest(h, cs.n);
    }
}
constexpr int WARP_K_WARPS = 4, WARP_K_STAGES = 8;
constexpr size_t WARP_K_SMEM = (size_t)WARP_K_WARPS * WARP_K_STAGES * 512;

struct HashCfg {
    int nt, ch, s;
    size_t smem;
    const void *fn;
};
template <int NT, int CH, int S>
HashCfg make_tma() {
    return HashCfg{NT, CH, S, HashSmem<NT, CH, S>::bytes, (const void *)k_hash_seq<NT, CH, S>};
}
template <int W, int CH, int S>
HashCfg make_coop() {
    return HashCfg{W * 32, CH, S, CoopSmem<W, CH, S>::bytes, (const void *)k_hash_coop<W, CH, S>};
}
const HashCfg *cfg_table(int &count) {
    static const HashCfg tab[] = {
        make_coop<4, 128, 3>(),  make_coop<4, 256, 2>(), make_coop<4, 128, 4>(), make_coop<2, 256, 3>(),
        make_coop<8, 128, 3>(),  make_coop<4, 256, 3>(), make_coop<2, 512, 2>(), make_coop<1, 128, 3>(),
        make_tma<128, 384, 3>(), make_tma<128, 256, 4>(), make_tma<96, 512, 3>(),
        // deep rings for few, long chains (latency-bound batches): 5-7 chunks in flight per lane
        make_coop<1, 512, 6>(),  make_coop<1, 512, 8>(),  make_coop<1, 256, 8>(),
    };
    count = (int)(sizeof(tab) / sizeof(tab[0]));
    return tab;
}
constexpr int DEFAULT_CFG = 6;  // coop<2 warps, 512 B, 2 stages>: 96.5% of measured HBM on C2 (r01 sweep)
constexpr int LATENCY_CFG = 11;   // coop<1 warp, 512 B, 6 stages>: batches too small to fill the GPU
constexpr uint64_t LATENCY_MAX_BUFS = 148ull * 2 * 32;  // one lane per buffer fits the deep variant
constexpr uint64_t WARP_MAX_BUFS = 148ull * 32;          // one warp per buffer, all resident at once
constexpr uint64_t RAGGED_WARPS_PER_SMSP = 2;

struct HashLaunch {
    int cfg = -1;
    int ctas_per_sm = 0;
};
HashLaunch g_launch[64];
int setenv_variant = -1;  // b2l_hash_select_variant override

const HashCfg *active_cfg(int &ctas_per_sm) {
    int dev = 0;
    cudaGetDevice(&dev);
    HashLaunch &L = g_launch[dev & 63];
    int count;
    const HashCfg *tab = cfg_table(count);
    if (L.cfg < 0) {
        int c = DEFAULT_CFG;
        if (const char *e = getenv("B2L_HASH_CFG")) {
            int v = atoi(e);
            if (v >= 0 && v < count) c = v;
        }
        if (setenv_variant >= 0) c = setenv_variant;
        if (cudaFuncSetAttribute(tab[c].fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tab[c].smem) !=
            cudaSuccess)
            return nullptr;
        int nb = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, tab[c].fn, tab[c].nt, tab[c].smem) != cudaSuccess)
            return nullptr;
        L.ctas_per_sm = nb > 0 ? nb : 1;
        L.cfg = c;
    }
    ctas_per_sm = L.ctas_per_sm;
    return &tab[L.cfg];
}

int hash_grid(const HashCfg &c, int per_sm, uint64_t n) {
    uint64_t max_ctas = (uint64_t)sm_count() * (uint64_t)per_sm;
    uint64_t need = (n + c.nt - 1) / c.nt;
    uint64_t g = need < max_ctas ? need : max_ctas;
    return g < 1 ? 1 : (int)g;
}

// ---------------------------------------------------------------- synthetic payloads
__device__ __forceinline__ uint64_t splitmix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
// Same stream as oracle/hash_fold64.c orc_payload_word (the bench checks digests against it).
__device__ __forceinline__ uint64_t payload_word(uint64_t seed, uint64_t cid, uint64_t j) {
    return splitmix64(seed ^ splitmix64(cid * 0xD1B54A32D192ED03ull + j));
}

__global__ void k_fill_payloads(uint8_t *__restrict__ base, const uint64_t *__restrict__ offs,
                                const uint64_t *__restrict__ lens, const uint64_t *__restrict__ cids,
                                uint64_t n, uint64_t seed) {
    for (uint64_t b = blockIdx.x; b < n; b += gridDim.x) {
        uint8_t *dst = base + offs[b];
        const uint64_t len = lens[b], cid = cids[b];
        const uint64_t nw = len >> 3;
        if ((reinterpret_cast<uintptr_t>(dst) & 7) == 0) {
            uint64_t *d64 = reinterpret_cast<uint64_t *>(dst);
            for (uint64_t j = threadIdx.x; j < nw; j += blockDim.x) d64[j] = payload_word(seed, cid, j);
        } else {
            for (uint64_t j = threadIdx.x; j < nw; j += blockDim.x) {
                uint64_t w = payload_word(seed, cid, j);
#pragma unroll
                for (int k = 0; k < 8; ++k) dst[j * 8 + k] = (uint8_t)(w >> (8 * k));
            }
        }
        if ((len & 7) && threadIdx.x == 0) {
            uint64_t w = payload_word(seed, cid, nw);
            for (uint64_t k = 0; k < (len & 7); ++k) dst[nw * 8 + k] = (uint8_t)(w >> (8 * k));
        }
    }
}

}  // namespace

int hash_batch_launch(const uint64_t *d_ptrs, const uint64_t *d_lens, uint64_t n, uint64_t *d_digests,
                      const uint32_t *d_order, cudaStream_t stream) {
    if (n == 0) return B2L_OK;
    if (!d_ptrs || !d_lens || !d_digests) return fail(B2L_E_INVALID_ARG, "b2l_hash_batch: null array");
    int per_sm = 0;
    const HashCfg *c = active_cfg(per_sm);
    if (!c) return fail(B2L_E_CUDA, "b2l_hash_batch: cannot configure hash kernel");
    if (setenv_variant < 0 && !getenv("B2L_HASH_CFG") && n <= WARP_MAX_BUFS) {
        // few buffers: one warp each (every buffer's chain runs at its own latency)
        auto fn = k_hash_warp<WARP_K_WARPS, WARP_K_STAGES>;
        // ragged (longest-first order given): two warps per scheduler, buffers dealt out
        // boustrophedon; uniform: one warp per buffer, all in flight at once
        uint64_t warps = n;
        static const uint64_t wps = [] {  // B2L_RAGGED_WPS: tuning override
            const char *e = getenv("B2L_RAGGED_WPS");
            return e && atoi(e) > 0 ? (uint64_t)atoi(e) : RAGGED_WARPS_PER_SMSP;
        }();
        if (d_order) warps = std::min<uint64_t>(n, (uint64_t)sm_count() * 4 * wps);
        const unsigned grid = (unsigned)((warps + WARP_K_WARPS - 1) / WARP_K_WARPS);
        // ragged and two warps per scheduler: the first CTA of every SM holds the longest buffers
        static const bool prim_on = !getenv("B2L_HASH_NO_PRIMARY");
        const uint64_t primary =
            (d_order && prim_on && wps >= 2 && warps == (uint64_t)sm_count() * 4 * wps) ? (uint64_t)sm_count() * 4 : 0;
        fn<<<grid, WARP_K_WARPS * 32, WARP_K_SMEM, stream>>>(d_ptrs, d_lens, d_order, n, d_digests, primary);
        B2L_CHECK_LAUNCH("k_hash_warp");
        return B2L_OK;
    }
    if (setenv_variant < 0 && !getenv("B2L_HASH_CFG") && n <= LATENCY_MAX_BUFS) {
        // few buffers: every chain runs alone, so what matters is bytes in flight per lane
        int count;
        const HashCfg *tab = cfg_table(count);
        static int lat_per_sm[64] = {0};
        int dev = 0;
        cudaGetDevice(&dev);
        if (!lat_per_sm[dev & 63]) {
            int nb = 0;
            B2L_CUDA(cudaFuncSetAttribute(tab[LATENCY_CFG].fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)tab[LATENCY_CFG].smem));
            B2L_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, tab[LATENCY_CFG].fn, tab[LATENCY_CFG].nt,
                                                                   tab[LATENCY_CFG].smem));
            lat_per_sm[dev & 63] = nb > 0 ? nb : 1;
        }
        c = &tab[LATENCY_CFG];
        per_sm = lat_per_sm[dev & 63];
    }
    int grid = hash_grid(*c, per_sm, n);
    void *args[] = {(void *)&d_ptrs, (void *)&d_lens, (void *)&d_order, (void *)&n, (void *)&d_digests};
    B2L_CUDA(cudaLaunchKernel(c->fn, dim3(grid), dim3(c->nt), args, c->smem, stream));
    return B2L_OK;
}

int hash_select_variant(int v, int *count) {
    int n;
    cfg_table(n);
    if (count) *count = n;
    if (v == -1) return B2L_OK;  // query only
    if (v >= n || v < -2) return fail(B2L_E_INVALID_ARG, "hash variant out of range");
    for (auto &L : g_launch) L.cfg = -1;
    setenv_variant = v == -2 ? -1 : v;  // -2: back to the default
    return B2L_OK;
}

int hash_launch_info(uint64_t n, int *grid, int *block, int *smem) {
    int per_sm = 0;
    const HashCfg *c = active_cfg(per_sm);
    if (!c) return fail(B2L_E_CUDA, "hash kernel configuration failed");
    if (grid) *grid = hash_grid(*c, per_sm, n);
    if (block) *block = c->nt;
    if (smem) *smem = (int)c->smem;
    return B2L_OK;
}

int fill_payloads_launch(uint8_t *d_base, const uint64_t *d_offsets, const uint64_t *d_lens,
                         const uint64_t *d_cids, uint64_t n, uint64_t seed, cudaStream_t stream) {
    if (n == 0) return B2L_OK;
    int grid = (int)(n < (uint64_t)sm_count() * 16 ? n : (uint64_t)sm_count() * 16);
    k_fill_payloads<<<grid, 256, 0, stream>>>(d_base, d_offsets, d_lens, d_cids, n, seed);
    B2L_CHECK_LAUNCH("k_fill_payloads launch");
    return B2L_OK;
}

}  // namespace b2l
