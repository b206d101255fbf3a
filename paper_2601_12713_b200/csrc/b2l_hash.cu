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

#ifndef PF_STEP
#define PF_STEP fnv_step32_lat
#endif
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
            PF_STEP(hl, hh, v[i].x, v[i].y);
            PF_STEP(hl, hh, v[i].z, v[i].w);
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
                PF_STEP(hl, hh, (uint32_t)w0, (uint32_t)(w0 >> 32));
                PF_STEP(hl, hh, (uint32_t)w1, (uint32_t)(w1 >> 32));
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

// ============================================================================ split pair
// Two warps fold ONE long buffer.  h = (h ^ w) * P mod 2^64 with P = 2^40 + 435 splits into two
// 32-bit recurrences (hashing.py:38-40):
//   lo' = lo32(xl * 435)                                  xl = lo ^ wl  (needs only the low halves)
//   hi' = xh * 435 + c,   c = hi32(xl * 435) + (xl << 8)   xh = hi ^ wh
// Each is one LOP3 -> IMAD dependency (~10 cycles/word), but one thread running both, plus the
// IMAD.HI behind c (a quarter-rate op), needs ~16-20 cycles per word (tools/chain_bench.cu).
// So warp A runs the low chain and publishes every xl; warp B computes the c values of a whole
// chunk with 32 lanes at once (off its chain, interleaved with the previous chunk's fold) and
// runs the high chain one chunk behind.  Warp A streams the buffer through an S-slot smem ring
// (coalesced 16-B cp.async, D chunks in flight); per-slot mbarriers hand a chunk (payload + xl)
// from A to B ("full", 32 arrivals) and the slot back from B to A ("empty", 32 arrivals).  B
// finishes the digest.  Chunks are 2 KiB: a chunk's synchronisation (cp.async wait, mbarrier
// try_wait ~90 cycles even when complete, arrive) costs ~300 cycles, ~1 cycle/word at 256 words.
// Only 16-B aligned buffers take this path (the halves are then plain 32-bit words).
//
// Both roles run warp-uniform code (every lane computes the chain; lane 0's copy is the one
// stored), so side work sits in the chain's basic block and fills its dependency stalls.  A
// chunk is folded in 32-word blocks held in registers; the next block's shared-memory loads are
// issued before the current block is folded (program order: ptxas keeps loads behind earlier
// stores to the same array), and a block's xl values are stored after it is folded (stores
// interleaved with the chain stall it on register reuse).  The block loop stays rolled (two
// blocks per iteration): fully unrolled chunks made the warps stall on instruction fetch once
// more than ~40 SMs ran them (ncu: "no_instructions" 5% -> 31% of samples).
constexpr int SPLIT_S = 4, SPLIT_D = 1, SPLIT_CH = 4096;
#ifndef B2L_SPLIT_UNROLL
#define B2L_SPLIT_UNROLL 4
#endif
constexpr int SPLIT_UNROLL = B2L_SPLIT_UNROLL;  // block pairs per loop iteration
constexpr int SPLIT_BW = 32;                            // words per register block
constexpr int SPLIT_NB = SPLIT_CH / 8 / SPLIT_BW;        // blocks per chunk
constexpr int SPLIT_CW = SPLIT_CH / 8;                   // words per chunk
constexpr uint64_t SPLIT_MIN_BYTES = 64 << 10;
struct SplitBars {
    uint64_t full[SPLIT_S], empty[SPLIT_S];
};
// per-pair shared memory: payload ring, published xl per slot, c values (two chunks), lo states
constexpr size_t SPLIT_RING = (size_t)SPLIT_S * SPLIT_CH;
constexpr size_t SPLIT_XB = (size_t)SPLIT_S * SPLIT_CW * 4, SPLIT_CB = 2ull * SPLIT_CW * 4, SPLIT_HLB = 16 * 4;
constexpr size_t SPLIT_PAIR = SPLIT_RING + SPLIT_XB + SPLIT_CB + SPLIT_HLB;
#ifdef B2L_SPLIT_PROF  // tools/split_bench.cu: cycles each role spends waiting
__device__ long long g_split_wait[2];
#define SPLIT_WAIT(role, bar, par)                       \
    do {                                                 \
        long long t0_ = clock64();                       \
        mbar_wait(bar, par);                             \
        if (threadIdx.x % 32 == 0) atomicAdd((unsigned long long *)&g_split_wait[role], clock64() - t0_); \
    } while (0)
#else
#define SPLIT_WAIT(role, bar, par) mbar_wait(bar, par)
#endif
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ uint32_t split_words(uint64_t nwf, uint64_t k) {
    const uint64_t w0 = k * SPLIT_CW;
    return nwf > w0 ? (uint32_t)(nwf - w0 < (uint64_t)SPLIT_CW ? nwf - w0 : (uint64_t)SPLIT_CW) : 0u;
}
// 128-bit shared loads in program order (ptxas otherwise splits the strided halves into 32-bit
// LDS, one per word -- more in-flight loads than a warp's scoreboards cover, ~3.5 cycles/word)
__device__ __forceinline__ uint4 lds128(const void *p) {
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "r"(smem_u32(p)));
    return v;
}
// the low (HI = 0) or high (HI = 1) halves of block `blk` of chunk k
template <int HI>
__device__ __forceinline__ void split_load(uint32_t (&w)[SPLIT_BW], const uint8_t *ring, uint64_t k, int blk) {
    const uint8_t *src = ring + (k % SPLIT_S) * SPLIT_CH + blk * SPLIT_BW * 8;
#pragma unroll
    for (int j = 0; j < SPLIT_BW / 2; ++j) {
        const uint4 v = lds128(src + 16 * j);
        w[2 * j] = HI ? v.y : v.x;
        w[2 * j + 1] = HI ? v.w : v.z;
    }
}
__device__ __forceinline__ void split_lo_block(uint32_t &hl, const uint32_t (&w)[SPLIT_BW], uint32_t *xdst, bool st) {
    uint32_t x[SPLIT_BW];
#pragma unroll
    for (int j = 0; j < SPLIT_BW; ++j) {
        x[j] = hl ^ w[j];
        asm("mul.lo.u32 %0, %1, 435;" : "=r"(hl) : "r"(x[j]));
    }
    if (st) {
        uint4 *d4 = reinterpret_cast<uint4 *>(xdst);
#pragma unroll
        for (int j = 0; j < SPLIT_BW; j += 4) d4[j / 4] = make_uint4(x[j], x[j + 1], x[j + 2], x[j + 3]);
    }
}
__device__ __forceinline__ void split_c_load(uint32_t (&c)[SPLIT_BW], const uint32_t *cc, int blk) {
#pragma unroll
    for (int j = 0; j < SPLIT_BW / 4; ++j) {
        const uint4 v = lds128(cc + blk * SPLIT_BW + 4 * j);
        c[4 * j] = v.x, c[4 * j + 1] = v.y, c[4 * j + 2] = v.z, c[4 * j + 3] = v.w;
    }
}
__device__ __forceinline__ void split_hi_block(uint32_t &hh, const uint32_t (&w)[SPLIT_BW], const uint32_t (&c)[SPLIT_BW]) {
#pragma unroll
    for (int j = 0; j < SPLIT_BW; ++j) asm("mad.lo.u32 %0, %1, 435, %2;" : "=r"(hh) : "r"(hh ^ w[j]), "r"(c[j]));
}

// role 0 (warp A)
__device__ __forceinline__ void split_lo(const BufCursor &cur, int lane, uint8_t *pair_smem, SplitBars *b, uint64_t base) {
    uint8_t *ring = pair_smem;
    uint32_t *xb = reinterpret_cast<uint32_t *>(pair_smem + SPLIT_RING);
    uint32_t *hlb = reinterpret_cast<uint32_t *>(pair_smem + SPLIT_RING + SPLIT_XB + SPLIT_CB);
    const uint32_t ring_s = smem_u32(ring);
    const uint64_t nch = (cur.L + SPLIT_CH - 1) / SPLIT_CH, nwf = cur.n >> 3;
    auto issue = [&](uint64_t k) {
        if (k < nch) {
            const uint64_t g = base + k;  // pair-lifetime chunk number: slot and barrier phase
            if (g >= SPLIT_S) SPLIT_WAIT(0, &b->empty[g % SPLIT_S], (uint32_t)((g / SPLIT_S - 1) & 1));
            const uint64_t off = k * SPLIT_CH;
            const uint64_t rem = cur.L - off;
            const uint32_t bytes = rem < SPLIT_CH ? (uint32_t)rem : SPLIT_CH;
            const uint32_t dst = ring_s + (uint32_t)((g % SPLIT_S) * SPLIT_CH);
#pragma unroll
            for (int i = 0; i < SPLIT_CH / 512; ++i) {
                const uint32_t o = (uint32_t)(512 * i + 16 * lane);
                if (o < bytes) cp_async16(dst + o, cur.a0 + off + o);
            }
        }
        cp_async_commit();
    };
#pragma unroll
    for (int k = 0; k < SPLIT_D; ++k) issue(k);
    uint32_t hl = (uint32_t)FNV_OFFSET;
    uint32_t wa[SPLIT_BW], wb[SPLIT_BW];
    cp_async_wait<SPLIT_D - 1>();  // chunk 0 landed (this lane's pieces) ...
    __syncwarp();                  // ... and every lane's
    split_load<0>(wa, ring, base, 0);
    for (uint64_t k = 0; k < nch; ++k) {
        const int s = (int)((base + k) % SPLIT_S);
        const uint32_t words = split_words(nwf, k);
        uint32_t *xs = xb + s * SPLIT_CW;
        issue(k + SPLIT_D);
        if (words == SPLIT_CW) {
#pragma unroll(SPLIT_UNROLL)
            for (int blk = 0; blk < SPLIT_NB; blk += 2) {  // rolled: the whole GPU runs this code, so
                                                           // it must stay in the instruction caches
                split_load<0>(wb, ring, base + k, blk + 1);
                split_lo_block(hl, wa, xs + blk * SPLIT_BW, lane == 0);
                if (blk + 2 < SPLIT_NB) {
                    split_load<0>(wa, ring, base + k, blk + 2);
                } else if (k + 1 < nch) {
                    cp_async_wait<SPLIT_D - 1>();  // chunk k+1 landed (this lane's pieces) ...
                    __syncwarp();                  // ... and every lane's
                    split_load<0>(wa, ring, base + k + 1, 0);
                }
                split_lo_block(hl, wb, xs + (blk + 1) * SPLIT_BW, lane == 0);
            }
        } else {  // the last, partial chunk
            const uint32_t *s32 = reinterpret_cast<const uint32_t *>(ring + s * SPLIT_CH);
            for (uint32_t j = 0; j < words; ++j) {
                const uint32_t x = hl ^ s32[2 * j];
                if (lane == 0) xs[j] = x;
                hl = x * 435u;
            }
        }
        if (lane == 0) hlb[s] = hl;
        __syncwarp();
        mbar_arrive(&b->full[s]);
    }
    cp_async_wait<0>();
}

// role 1 (warp B)
__device__ __forceinline__ void split_hi(const BufCursor &cur, int lane, uint8_t *pair_smem, SplitBars *b,
                                         uint64_t *__restrict__ digests, uint64_t base) {
    const uint8_t *ring = pair_smem;
    const uint32_t *xb = reinterpret_cast<const uint32_t *>(pair_smem + SPLIT_RING);
    uint32_t *cb = reinterpret_cast<uint32_t *>(pair_smem + SPLIT_RING + SPLIT_XB);
    const uint32_t *hlb = reinterpret_cast<const uint32_t *>(pair_smem + SPLIT_RING + SPLIT_XB + SPLIT_CB);
    const uint64_t nch = (cur.L + SPLIT_CH - 1) / SPLIT_CH, nwf = cur.n >> 3;
    // c of chunk k into cb[k & 1] (chunk k's "full" already waited)
    auto make_c = [&](uint64_t k) {
        const uint32_t words = split_words(nwf, k);
        const uint32_t *x32 = xb + ((base + k) % SPLIT_S) * SPLIT_CW;
        uint32_t *c = cb + (k & 1) * SPLIT_CW;
#pragma unroll
        for (int h = 0; h < SPLIT_CW / 32; ++h) {
            const uint32_t j = (uint32_t)lane + 32u * h;
            if (j < words) {
                const uint32_t x = x32[j];
                c[j] = __umulhi(x, 435u) + (x << 8);
            }
        }
    };
    SPLIT_WAIT(1, &b->full[base % SPLIT_S], (uint32_t)((base / SPLIT_S) & 1));
    make_c(0);
    __syncwarp();
    uint32_t hh = (uint32_t)(FNV_OFFSET >> 32);
    uint32_t wa[SPLIT_BW], wb[SPLIT_BW], ca[SPLIT_BW], cr[SPLIT_BW];
    split_load<1>(wa, ring, base, 0);
    split_c_load(ca, cb, 0);
    for (uint64_t k = 0; k < nch; ++k) {
        const int s = (int)((base + k) % SPLIT_S);
        const uint32_t words = split_words(nwf, k);
        const uint32_t *cc = cb + (k & 1) * SPLIT_CW;
        if (k + 1 < nch) {  // the next chunk's c values, computed beside this chunk's chain
            SPLIT_WAIT(1, &b->full[(base + k + 1) % SPLIT_S], (uint32_t)(((base + k + 1) / SPLIT_S) & 1));
            make_c(k + 1);
        }
        if (words == SPLIT_CW) {
#pragma unroll(SPLIT_UNROLL)
            for (int blk = 0; blk < SPLIT_NB; blk += 2) {  // rolled: the whole GPU runs this code, so
                                                           // it must stay in the instruction caches
                split_load<1>(wb, ring, base + k, blk + 1);
                split_c_load(cr, cc, blk + 1);
                split_hi_block(hh, wa, ca);
                if (blk + 2 < SPLIT_NB) {
                    split_load<1>(wa, ring, base + k, blk + 2);
                    split_c_load(ca, cc, blk + 2);
                } else if (k + 1 < nch) {
                    __syncwarp();  // the next chunk's c values are in
                    split_load<1>(wa, ring, base + k + 1, 0);
                    split_c_load(ca, cb + ((k + 1) & 1) * SPLIT_CW, 0);
                }
                split_hi_block(hh, wb, cr);
            }
        } else {  // the last, partial chunk
            const uint32_t *s32 = reinterpret_cast<const uint32_t *>(ring + s * SPLIT_CH);
            for (uint32_t j = 0; j < words; ++j) hh = (hh ^ s32[2 * j + 1]) * 435u + cc[j];
        }
        if (k + 1 == nch && lane == 0) {  // both halves of the last full word are in: tail word + finish
            uint64_t h = ((uint64_t)hh << 32) | hlb[s];
            const uint32_t tailb = (uint32_t)(cur.n & 7);
            if (tailb) {
                const uint64_t *s64 = reinterpret_cast<const uint64_t *>(ring + s * SPLIT_CH);
                const uint64_t w = s64[(uint32_t)(nwf - k * SPLIT_CW)] & ((1ull << (8 * tailb)) - 1);
                h = fnv_step(h, w);
            }
            digests[cur.idx] = finish_digest(h, cur.n);
        }
        __syncwarp();  // this slot fully read
        mbar_arrive(&b->empty[s]);
    }
}

// Launch configurations (lanes per CTA, chunk bytes, ring depth).  Selected at
// first use; B2L_HASH_CFG=<i> overrides (used by the tuning sweep).
// ============================================================================ variant W
// One WARP per buffer, for batches too small to fill the GPU with lanes (C1): all 32 lanes
// stream the buffer's next 512-B chunk with one coalesced 16-B cp.async each (one instruction
// per chunk instead of 32 shuffled ones), an S-deep ring per warp, and lane 0 runs the serial
// chain out of shared memory.  A lone chain is then bound by its own dependency latency, not by
// the cooperative ring's per-round issue cost (the longest C1 buffer sets the batch time).
template <int S>
__device__ __forceinline__ void warp_fold(BufCursor ld, int lane, uint8_t *ring, uint64_t *__restrict__ digests) {
    constexpr int CH = 512;
    const uint32_t ring_s = smem_u32(ring);
    BufCursor cs = ld;
    if (cs.L == 0) {
        if (lane == 0) digests[cs.idx] = 0;
        return;
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

// Work is claimed dynamically from per-launch counters (`WarpSched`, zeroed before the launch):
// the first CTA to start on each SM (a per-SM ticket) is a LEAD CTA -- with `split` = P > 0 its
// two warp pairs claim list positions 0..P-1 (the longest buffers) one at a time and fold each
// as a split pair (lo chain on warp 2p, hi chain on warp 2p+1: different schedulers), or with
// warp A alone when a buffer is short or unaligned; every other warp, and the lead warps once
// those positions are gone, claims the next position of [P, n) and folds it alone.  Claiming a
// longest-first list in order is greedy LPT, whatever the CTA placement or residency.
struct WarpSched {
    unsigned int lead[256];        // per-SM tickets
    unsigned int pair_next;        // next position of [0, P)
    unsigned int pad;
    unsigned long long deal_next;  // next position of [P, n), minus P
};
__device__ __forceinline__ void named_bar(int id, int threads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}
// RAGGED = false compiles only the uniform path (one warp per buffer): without the split pairs'
// registers more CTAs fit per SM, so a uniform batch keeps every buffer in flight at once.
template <int WARPS, int S, bool RAGGED>
__global__ void __launch_bounds__(WARPS * 32) k_hash_warp(const uint64_t *__restrict__ ptrs,
                                                          const uint64_t *__restrict__ lens,
                                                          const uint32_t *__restrict__ order, uint64_t n_bufs,
                                                          uint64_t *__restrict__ digests, WarpSched *sch,
                                                          uint32_t split) {
    constexpr int CH = 512;
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ uint32_t s_lead, s_item[2];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint8_t *ring = smem + (size_t)warp * S * CH;
    if (!RAGGED || !sch) {  // uniform batch: one warp per buffer, all in flight at once
        const uint64_t k = (uint64_t)blockIdx.x * WARPS + warp;
        if (k < n_bufs) {
            BufCursor cur;
            cursor_load(cur, ptrs, lens, order, k, n_bufs);
            warp_fold<S>(cur, lane, ring, digests);
        }
        return;
    }
    if (split) {
        static_assert(WARPS == 4, "a lead CTA holds two split pairs");
        if (threadIdx.x == 0) {
            uint32_t smid;
            asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
            s_lead = atomicAdd(&sch->lead[smid & 255], 1u) == 0;  // every SM that runs a CTA has a lead
        }
        __syncthreads();
        if (s_lead) {
            SplitBars *bars = reinterpret_cast<SplitBars *>(smem + 2 * SPLIT_PAIR);
            const int pair = warp >> 1, role = warp & 1;
            if (lane == 0 && role == 0) {
                for (int i = 0; i < SPLIT_S; ++i) mbar_init(&bars[pair].full[i], 32), mbar_init(&bars[pair].empty[i], 32);
                fence_mbar_init();
            }
            __syncthreads();
            uint8_t *pr = smem + (size_t)pair * SPLIT_PAIR;
            uint64_t base = 0;  // chunks this pair has moved so far (ring slot / barrier phase)
            for (;;) {
                if (lane == 0 && role == 0) s_item[pair] = atomicAdd(&sch->pair_next, 1u);
                named_bar(1 + pair, 64);
                const uint64_t k = s_item[pair];
                named_bar(1 + pair, 64);  // both warps have read the item
                if (k >= split || k >= n_bufs) break;
                BufCursor cur;
                cursor_load(cur, ptrs, lens, order, k, n_bufs);
                if (cur.m == 0 && cur.n >= SPLIT_MIN_BYTES) {
                    if (role == 0) split_lo(cur, lane, pr, &bars[pair], base);
                    else split_hi(cur, lane, pr, &bars[pair], digests, base);
                    base += (cur.L + SPLIT_CH - 1) / SPLIT_CH;
                } else if (role == 0) {  // short or unaligned: warp A folds it alone
                    warp_fold<S>(cur, lane, pr, digests);
                }
                named_bar(1 + pair, 64);  // the pair's shared memory is free again
            }
            ring = pr + (size_t)role * S * CH;  // this pair's area, split between its two warps
        }
    }
    // claim the next position of [split, n) and fold it with this warp alone
    for (;;) {
        unsigned long long k = 0;
        if (lane == 0) k = atomicAdd(&sch->deal_next, 1ull);
        k = __shfl_sync(0xffffffffu, k, 0) + split;
        if (k >= n_bufs) break;
        BufCursor cur;
        cursor_load(cur, ptrs, lens, order, k, n_bufs);
        warp_fold<S>(cur, lane, ring, digests);
    }
}
constexpr int WARP_K_WARPS = 4, WARP_K_STAGES = 8;
constexpr size_t WARP_K_SMEM_DEAL = (size_t)WARP_K_WARPS * WARP_K_STAGES * 512;
constexpr size_t WARP_K_SMEM_SPLIT = 2 * SPLIT_PAIR + 2 * sizeof(SplitBars);
constexpr size_t WARP_K_SMEM = WARP_K_SMEM_DEAL > WARP_K_SMEM_SPLIT ? WARP_K_SMEM_DEAL : WARP_K_SMEM_SPLIT;

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
        auto fn = d_order ? k_hash_warp<WARP_K_WARPS, WARP_K_STAGES, true> : k_hash_warp<WARP_K_WARPS, WARP_K_STAGES, false>;
        static bool smem_set[64] = {false};
        int cur_dev = 0;
        B2L_CUDA(cudaGetDevice(&cur_dev));
        if (!smem_set[cur_dev & 63]) {  // the split pairs' rings exceed the 48 KiB default
            B2L_CUDA(cudaFuncSetAttribute(k_hash_warp<WARP_K_WARPS, WARP_K_STAGES, true>,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, (int)WARP_K_SMEM));
            smem_set[cur_dev & 63] = true;
        }
        // ragged (longest-first order given): three warps per scheduler claiming the list (the
        // lead CTAs' split pairs first); uniform: one warp per buffer, all in flight at once
        uint64_t warps = n;
        static const uint64_t wps = [] {  // B2L_RAGGED_WPS: tuning override
            const char *e = getenv("B2L_RAGGED_WPS");
            return e && atoi(e) > 0 ? (uint64_t)atoi(e) : RAGGED_WARPS_PER_SMSP;
        }();
        if (d_order) warps = std::min<uint64_t>(n, (uint64_t)sm_count() * 4 * wps);
        const unsigned grid = (unsigned)((warps + WARP_K_WARPS - 1) / WARP_K_WARPS);
        // ragged: the first CTA on every SM folds the longest buffers as split pairs
        // (B2L_HASH_NO_SPLIT: one warp each); the list is claimed dynamically (WarpSched)
        static const bool split_on = !getenv("B2L_HASH_NO_SPLIT");
        const uint32_t split = d_order && split_on ? 2u * (uint32_t)sm_count() : 0u;
        WarpSched *sch = nullptr;
        if (d_order) {
            B2L_CUDA(cudaMallocAsync((void **)&sch, sizeof(WarpSched), stream));
            B2L_CUDA(cudaMemsetAsync(sch, 0, sizeof(WarpSched), stream));
        }
        fn<<<grid, WARP_K_WARPS * 32, split ? WARP_K_SMEM : WARP_K_SMEM_DEAL, stream>>>(d_ptrs, d_lens, d_order, n,
                                                                                      d_digests, sch, split);
        const cudaError_t le = cudaGetLastError();
        if (sch) B2L_CUDA(cudaFreeAsync(sch, stream));
        if (le != cudaSuccess) return cuda_fail(le, "k_hash_warp");
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
