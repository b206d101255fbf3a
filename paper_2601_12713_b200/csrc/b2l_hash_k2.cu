// K2 hash_planes: the reference's serial FNV fold of ONE huge buffer, parallelised exactly
// across the whole GPU (in 4-bit groups instead of single bit planes).
//
// f_w(h) = (h ^ w) * P is a T-function: bits [k, k+4) of the output depend only on bits < k+4
// of the inputs.  Processing the 64-bit state in 16 groups of 4 bits, once bits < k of every
// intermediate state are known (x_i = h_i ^ w_i known mod 2^k, R_i = (x_i mod 2^k) * P),
// the 4-bit group of the chain obeys
//     h4_{i+1} = ((R_i >> k) + 3 * (h4_i ^ w4_i)) mod 16        (P = 2^40 + 435 = 3 mod 16)
// so every run of words is a map {0..15} -> {0..15}: a 16-byte table, built for all 16 inputs
// at once with byte-parallel arithmetic.  Tables compose associatively, so a group resolves by
// a prefix composition across threads (warp shuffles), warps, and CTAs; a second pass with the
// actual input state writes the resolved bits back.
//
// v5 layout: each word lives in shared memory as ONE u64 y_i whose bits < k already hold x_i
// (resolved) and bits >= k still hold w_i, so R_i's nibble is recomputed from y_i (one or two
// IMADs) instead of being kept in registers -- 24 Ki words per CTA per round (192 KiB of smem,
// 512 threads), fewer rounds.  Across CTAs every CTA publishes its aggregate map and composes
// all predecessors' aggregates itself (a warp reads them in parallel): no serial look-back
// chain through the grid.  Chunks beyond the co-resident grid are processed in rounds chained
// through a per-group carry.  Verified bit-exact against the serial fold (tests).
#include <algorithm>
#include <cstdlib>
#include <mutex>
#include <vector>
#include <cooperative_groups.h>

#include "b2l_common.cuh"

namespace b2l {
namespace k2 {

#ifndef K2_THREADS
#define K2_THREADS 256
#endif
constexpr int THREADS = K2_THREADS;
#ifndef K2_MIN_BLOCKS
#define K2_MIN_BLOCKS 3
#endif
constexpr int MIN_BLOCKS = K2_MIN_BLOCKS;  // co-resident CTAs per SM (three: up to 85 registers, 3 x 74 KiB of words)
constexpr int WARPS = THREADS / 32;
#ifndef K2_WPT
#define K2_WPT 36
#endif
constexpr int WPT = K2_WPT;                   // words per thread, resident in shared memory
// words per CTA per round (72 KiB; three CTAs per SM).  Measured (16 x 256 MiB / one 256 MiB):
// 24 words x 4 CTAs 164 / 143 GB/s, 32 x 3 186 / 156, 36 x 3 196 / 163, 48 x 2 191 / 159 -- the
// step count falls with the words resident per SM, and each step costs about the same.
static_assert(WPT % 4 == 0, "the table passes run four quarter chains per thread");
constexpr int CHUNK = THREADS * WPT;
constexpr int ROW = WPT + 1;              // padded row (u32 units): conflict-free column access
constexpr size_t SMEM = (size_t)2 * THREADS * ROW * sizeof(uint32_t);  // lo and hi planes

// Aggregate slots: a map is 16 bytes whose entries use only the low nibble, so the high
// nibble of byte 0 marks a published slot and map + mark travel in one 16-byte access.
constexpr uint32_t MARK = 0x10u;
// Each slot sits alone on a 128-byte line (uint4 units): up to ~600 CTAs' warps poll their
// predecessors' slots at once, and slots packed 8 to a line queue those polls on a few lines.
constexpr uint32_t SLOT_STRIDE = 8;
// Predecessor slots a lane loads at once before it starts composing (the rest one by one).
constexpr uint32_t PREFETCH = 1;
// Optional back-off between polls of an unpublished slot (-DK2_SPIN_NS=n).  Spin loops are ~25%
// of the kernel's instructions, but 64 or 400 ns of back-off measured no faster than none.
#ifndef K2_SPIN_NS
#define K2_SPIN_NS 0
#endif
constexpr unsigned SPIN_NS = K2_SPIN_NS;
__device__ __forceinline__ uint4 ld_slot(const uint4 *p) {
    uint4 v;
    asm volatile("ld.volatile.global.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p));
    return v;
}
__device__ __forceinline__ void st_slot(uint4 *p, uint4 v) {
    asm volatile("st.volatile.global.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(v.x | MARK), "r"(v.y), "r"(v.z),
                 "r"(v.w)
                 : "memory");
}
__device__ __forceinline__ uint4 unmark(uint4 v) {
    v.x &= 0x0F0F0F0Fu;
    return v;
}

// A map {0..15} -> {0..15} as 16 bytes (entry j = byte j): byte-parallel arithmetic never
// carries across bytes here, and composition is a byte gather done with PRMT.
struct Tab {
    uint32_t r[4];
};
__device__ __forceinline__ Tab tab_id() { return Tab{{0x03020100u, 0x07060504u, 0x0B0A0908u, 0x0F0E0D0Cu}}; }
// one word through all 16 candidate states: t -> ((R>>k)&15) + 3 * (t ^ w4)  (mod 16)
__device__ __forceinline__ void tab_step(Tab &T, uint32_t w4, uint32_t r4) {
    const uint32_t wb = w4 * 0x01010101u, rb = r4 * 0x01010101u;
#pragma unroll
    for (int m = 0; m < 4; ++m) T.r[m] = ((T.r[m] ^ wb) * 3u + rb) & 0x0F0F0F0Fu;
}
// The same step on an unmasked table (entries < 64): the mask folds into the XOR (one LOP3),
// so a step is LOP3 + IMAD per register; tab_mask() once after the run.
__device__ __forceinline__ void tab_step_lazy(Tab &T, uint32_t wb, uint32_t rb) {
#pragma unroll
    for (int m = 0; m < 4; ++m) T.r[m] = ((T.r[m] & 0x0F0F0F0Fu) ^ wb) * 3u + rb;
}
__device__ __forceinline__ void tab_mask(Tab &T) {
#pragma unroll
    for (int m = 0; m < 4; ++m) T.r[m] &= 0x0F0F0F0Fu;
}
// (first A, then B): out[j] = B[A[j]]
__device__ __forceinline__ Tab tab_compose(const Tab &A, const Tab &B) {
    Tab o;
#pragma unroll
    for (int m = 0; m < 4; ++m) {
        const uint32_t a = A.r[m];
        const uint32_t x = a & 0x07070707u;
        const uint32_t sx = x | (x >> 4);
        const uint32_t sel = (sx & 0xFFu) | ((sx >> 8) & 0xFF00u);
        const uint32_t lo = __byte_perm(B.r[0], B.r[1], sel), hi = __byte_perm(B.r[2], B.r[3], sel);
        const uint32_t mask = ((a >> 3) & 0x01010101u) * 0xFFu;
        o.r[m] = (lo & ~mask) | (hi & mask);
    }
    return o;
}
__device__ __forceinline__ uint32_t tab_apply(const Tab &T, uint32_t s) {
    const uint32_t v = (s & 8) ? ((s & 4) ? T.r[3] : T.r[2]) : ((s & 4) ? T.r[1] : T.r[0]);
    return (v >> (8 * (s & 3))) & 15u;
}
__device__ __forceinline__ Tab tab_shfl_up(const Tab &T, int d) {
    Tab o;
#pragma unroll
    for (int m = 0; m < 4; ++m) o.r[m] = __shfl_up_sync(0xffffffffu, T.r[m], d);
    return o;
}
__device__ __forceinline__ uint4 tab_pack(const Tab &T) { return make_uint4(T.r[0], T.r[1], T.r[2], T.r[3]); }
__device__ __forceinline__ Tab tab_unpack(uint4 v) { return Tab{{v.x, v.y, v.z, v.w}}; }

__device__ __forceinline__ uint64_t load_word(const uint8_t *buf, uint64_t n, uint64_t i) {
    const uint64_t start = (uint64_t)buf, a = start + 8 * i;
    const uint64_t end = start + n;  // exclusive
    uint64_t w;
    const uint32_t r = (uint32_t)(a & 7);
    const uint64_t lo = a - r;
    if (r == 0) {
        w = __ldg(reinterpret_cast<const unsigned long long *>(lo));
    } else {
        const uint64_t u0 = __ldg(reinterpret_cast<const unsigned long long *>(lo));
        const uint64_t u1 = (lo + 8 < end) ? __ldg(reinterpret_cast<const unsigned long long *>(lo + 8)) : 0ull;
        w = (u0 >> (8 * r)) | (u1 << (64 - 8 * r));
    }
    if (a + 8 > end) {  // zero-extended tail word
        const uint32_t valid = (uint32_t)(end - a);
        w &= (1ull << (8 * valid)) - 1;
    }
    return w;
}

// Bits [k, k+4) of R = (y mod 2^k) * P, P = 2^40 + 435, from the low / high 32-bit halves of y.
// k < 32 (HI false): the nibble lies in the low word, (y mod 2^k) * 435 mod 2^32.
// k >= 32 (HI true): the high word of the product: hi32(lo * 435) + (hi mod 2^(k-32)) * 435 + (lo << 8).
template <bool HI>
__device__ __forceinline__ uint32_t r_nib(uint32_t lo, uint32_t hi, int k) {
    if (!HI) {
        if (k == 0) return 0;
        return (((lo & ((1u << k) - 1u)) * 435u) >> k) & 15u;
    }
    const int kh = k - 32;
    const uint32_t hm = kh ? (hi & ((1u << kh) - 1u)) : 0u;
    const uint32_t hw = __umulhi(lo, 435u) + hm * 435u + (lo << 8);
    return (hw >> kh) & 15u;
}

struct Shared {
    uint4 warp_tab[WARPS];
    uint32_t warp_in[WARPS];
};

// One 4-bit group of one round: pass A (maps), the prefix across warps and CTAs, pass B
// (resolved nibbles written back into y).  HI: the group lies in the high 32 bits.
template <bool HI, bool FULL>
__device__ __forceinline__ void group_step(uint32_t *ylo, uint32_t *yhi, int nv, int k, uint64_t r, uint64_t slot,
                                           uint32_t c, uint32_t nc, uint32_t G, uint4 *aggs,
                                           unsigned long long *carry, Shared &sh) {
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    constexpr int Q = WPT / 4;
    const int ks = HI ? k - 32 : k;
    uint32_t *ymine = HI ? yhi : ylo;
    // ---- pass A: this thread's map over its words, four independent quarter chains
    Tab Tq[4] = {tab_id(), tab_id(), tab_id(), tab_id()};
#pragma unroll
    for (int j = 0; j < Q; ++j) {
#pragma unroll
        for (int h = 0; h < 4; ++h) {
            const int jj = h * Q + j;
            if (FULL || jj < nv) {
                const uint32_t lo = ylo[jj], hi = HI ? yhi[jj] : 0u;
                const uint32_t w4 = ((HI ? hi : lo) >> ks) & 15u, r4 = r_nib<HI>(lo, hi, k);
                tab_step_lazy(Tq[h], w4 * 0x01010101u, r4 * 0x01010101u);
            }
        }
    }
#pragma unroll
    for (int h = 0; h < 4; ++h) tab_mask(Tq[h]);
    const Tab T01 = tab_compose(Tq[0], Tq[1]);
    const Tab T012 = tab_compose(T01, Tq[2]);
    Tab T = tab_compose(T012, Tq[3]);
    // ---- inclusive prefix composition across the warp (lane order)
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const Tab o = tab_shfl_up(T, d);
        if (lane >= d) T = tab_compose(o, T);
    }
    const Tab excl_lane = tab_shfl_up(T, 1);
    if (lane == 31) sh.warp_tab[warp] = tab_pack(T);
    __syncthreads();
    if (warp == 0) {
        // prefix over the warps (lanes 0..WARPS-1), CTA aggregate in lane WARPS-1
        Tab W = lane < WARPS ? tab_unpack(sh.warp_tab[lane]) : tab_id();
#pragma unroll
        for (int d = 1; d < WARPS; d <<= 1) {
            const Tab o = tab_shfl_up(W, d);
            if (lane >= d) W = tab_compose(o, W);
        }
        const Tab wexcl = tab_shfl_up(W, 1);
        Tab agg;
#pragma unroll
        for (int m = 0; m < 4; ++m) agg.r[m] = __shfl_sync(0xffffffffu, W.r[m], WARPS - 1);
        uint4 *row = aggs + slot * G * SLOT_STRIDE;
        if (lane == 0 && c + 1 < nc) st_slot(&row[c * SLOT_STRIDE], tab_pack(agg));  // the last CTA's is never read
        // the carry into this round is needed only after the composition: its load goes out now
        unsigned long long cv = 0;
        if (lane == 0 && r != 0) cv = ((volatile unsigned long long *)carry)[slot - 16];
        // prefix of the predecessors' aggregates: lane l composes a contiguous block of them
        // (in order), then a warp scan composes the blocks.  The block's first PREFETCH slots
        // are loaded together (one L2 round trip, not one per slot); unpublished ones re-polled.
        const uint32_t per = (c + 31) / 32, b0 = lane * per, b1 = b0 + per < c ? b0 + per : c;
        Tab P = tab_id();
        uint4 pv[PREFETCH];
#pragma unroll
        for (uint32_t u = 0; u < PREFETCH; ++u)
            if (b0 + u < b1) pv[u] = ld_slot(&row[(b0 + u) * SLOT_STRIDE]);
#pragma unroll
        for (uint32_t u = 0; u < PREFETCH; ++u) {
            if (b0 + u < b1) {
                while (!(pv[u].x & MARK)) {
                    if (SPIN_NS) __nanosleep(SPIN_NS);
                    pv[u] = ld_slot(&row[(b0 + u) * SLOT_STRIDE]);
                }
                P = tab_compose(P, tab_unpack(unmark(pv[u])));
            }
        }
        for (uint32_t j = b0 + PREFETCH; j < b1; ++j) {
            uint4 v;
            for (v = ld_slot(&row[j * SLOT_STRIDE]); !(v.x & MARK); v = ld_slot(&row[j * SLOT_STRIDE]))
                if (SPIN_NS) __nanosleep(SPIN_NS);
            P = tab_compose(P, tab_unpack(unmark(v)));
        }
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const Tab o = tab_shfl_up(P, d);
            if (lane >= d) P = tab_compose(o, P);
        }
#pragma unroll
        for (int m = 0; m < 4; ++m) P.r[m] = __shfl_sync(0xffffffffu, P.r[m], 31);
        uint32_t s_cta = 0;
        if (lane == 0) {
            uint32_t s_round;  // the group's state entering this round
            if (r == 0) {
                s_round = (uint32_t)(FNV_OFFSET >> k) & 15u;
            } else {
                volatile unsigned long long *vcarry = carry;
                while (cv == 0) {
                    if (SPIN_NS) __nanosleep(SPIN_NS);
                    cv = vcarry[slot - 16];
                }
                s_round = (uint32_t)cv & 15u;
            }
            s_cta = tab_apply(P, s_round);
            if (c + 1 == nc) {  // last chunk of the round: carry its output state
                __threadfence();
                atomicExch(&carry[slot], 0x100ull | tab_apply(agg, s_cta));
            }
        }
        s_cta = __shfl_sync(0xffffffffu, s_cta, 0);
        if (lane < WARPS) sh.warp_in[lane] = lane == 0 ? s_cta : tab_apply(wexcl, s_cta);
    }
    __syncthreads();
    // ---- pass B with the actual input state, the four quarters at once (quarter h's input is
    // the composed map of the quarters before it applied to the thread's input); the resolved
    // nibble x4 = h4 ^ w4 replaces w4 in y: y ^= h4 << k
    const uint32_t sin = lane == 0 ? sh.warp_in[warp] : tab_apply(excl_lane, sh.warp_in[warp]);
    uint32_t sq[4] = {sin, tab_apply(Tq[0], sin), tab_apply(T01, sin), tab_apply(T012, sin)};
#pragma unroll
    for (int j = 0; j < Q; ++j) {
#pragma unroll
        for (int h = 0; h < 4; ++h) {
            const int jj = h * Q + j;
            if (FULL || jj < nv) {
                const uint32_t lo = ylo[jj], hi = HI ? yhi[jj] : 0u;
                const uint32_t mine = HI ? hi : lo;
                const uint32_t w4 = (mine >> ks) & 15u, r4 = r_nib<HI>(lo, hi, k);
                ymine[jj] = mine ^ (sq[h] << ks);
                sq[h] = (r4 + 3u * (sq[h] ^ w4)) & 15u;
            }
        }
    }
}

// One buffer of a launch.  A launch hashes up to MAX_JOBS buffers at once, each by its own
// `teams` teams of G CTAs (G = grid / (jobs * teams)), with its own slot and carry scratch.
// Independent buffers share every SM, so one buffer's cross-CTA waits are filled by the
// others' table passes, and a smaller G makes each (round, group) step cheaper.
struct Job {
    const uint8_t *buf;
    uint64_t nbytes;
    uint4 *aggs;
    unsigned long long *carry;
    uint64_t *digest;
};
constexpr int MAX_JOBS = 16;
struct Jobs {
    Job j[MAX_JOBS];
    uint32_t njobs, teams;
};

__global__ void __launch_bounds__(THREADS, MIN_BLOCKS) k_hash_planes(const __grid_constant__ Jobs J) {
    extern __shared__ uint32_t planes[];  // lo plane then hi plane, THREADS x ROW each
    __shared__ Shared sh;
    const int t = threadIdx.x;
    // `teams` teams of CTAs take a buffer's rounds in turn (team t the rounds r = t mod teams):
    // a round's CTAs wait on each other once per group, and with CTAs of several teams on each
    // SM, the other teams' table passes fill a team's waits (each team runs about one group
    // behind the previous one, on its carries).
    const uint32_t teams = J.teams, G = gridDim.x / (J.njobs * teams);
    const uint32_t unit = blockIdx.x / G, c = blockIdx.x % G;
    if (unit >= J.njobs * teams) return;
    const Job &jb = J.j[unit / teams];
    const uint32_t team = unit % teams;
    const uint8_t *buf = jb.buf;
    const uint64_t nbytes = jb.nbytes;
    uint4 *aggs = jb.aggs;
    unsigned long long *carry = jb.carry;
    const uint64_t nw = (nbytes + 7) >> 3;
    const uint64_t nchunks = (nw + CHUNK - 1) / CHUNK;
    const uint64_t rounds = (nchunks + G - 1) / G;
    uint32_t *plo = planes, *phi = planes + THREADS * ROW;

    for (uint64_t r = team; r < rounds; r += teams) {
        const uint64_t q = r * G + c;
        if (q >= nchunks) break;  // only the last round has idle CTAs, and nobody waits on them
        const uint32_t nc = (uint32_t)(nchunks - r * G < G ? nchunks - r * G : G);  // CTAs in this round
        const uint64_t base = q * CHUNK;
        for (int idx = t; idx < CHUNK; idx += THREADS) {
            const uint64_t i = base + idx;
            const uint64_t v = i < nw ? load_word(buf, nbytes, i) : 0ull;
            const int o = (idx / WPT) * ROW + idx % WPT;
            plo[o] = (uint32_t)v;
            phi[o] = (uint32_t)(v >> 32);
        }
        __syncthreads();
        uint32_t *ylo = plo + t * ROW, *yhi = phi + t * ROW;  // this thread's words, resident for the round
        const int64_t left = (int64_t)nw - (int64_t)(base + (uint64_t)t * WPT);
        const int nv = left <= 0 ? 0 : (left >= WPT ? WPT : (int)left);
        if (base + CHUNK <= nw) {  // a full chunk (CTA-uniform): the table passes run unpredicated
#pragma unroll 1
            for (int g = 0; g < 8; ++g)
                group_step<false, true>(ylo, yhi, nv, 4 * g, r, r * 16 + g, c, nc, G, aggs, carry, sh);
#pragma unroll 1
            for (int g = 8; g < 16; ++g)
                group_step<true, true>(ylo, yhi, nv, 4 * g, r, r * 16 + g, c, nc, G, aggs, carry, sh);
        } else {
#pragma unroll 1
            for (int g = 0; g < 8; ++g)
                group_step<false, false>(ylo, yhi, nv, 4 * g, r, r * 16 + g, c, nc, G, aggs, carry, sh);
#pragma unroll 1
            for (int g = 8; g < 16; ++g)
                group_step<true, false>(ylo, yhi, nv, 4 * g, r, r * 16 + g, c, nc, G, aggs, carry, sh);
        }
        __syncthreads();
    }
    // the final state is the carry of the last round; the buffer's first CTA finishes the digest
    if (team == 0 && c == 0 && threadIdx.x == 0) {
        volatile unsigned long long *vcarry = carry;
        uint64_t h = 0;
        const uint64_t last = rounds - 1;
        for (int g = 0; g < 16; ++g) {
            unsigned long long v;
            do {
                v = vcarry[last * 16 + g];
            } while (v == 0);
            h |= (uint64_t)(v & 15ull) << (4 * g);
        }
        *jb.digest = finish_digest(h, nbytes);
    }
}

// Per-device K2 state.  The status/carry scratch is shared by every K2 launch on the device,
// whatever stream it is queued on (hash_tensors on the caller's stream, b2l_hash_host's
// pipeline, the capture agent), so launches are chained: each new call's stream first waits
// on the event recorded after the previous launch, then resets the scratch.  This also keeps
// two whole-GPU cooperative grids from ever being resident at once.
struct Ctx {
    int grid = 0;
    uint4 *status = nullptr;
    unsigned long long *carry = nullptr;
    size_t status_cap = 0, carry_cap = 0;
    std::mutex mu;
    cudaEvent_t done = nullptr;  // recorded after the last K2 launch on this device
};
Ctx g_ctx[64];

}  // namespace k2

int k2_grid() {
    int dev = 0;
    cudaGetDevice(&dev);
    k2::Ctx &C = k2::g_ctx[dev & 63];
    if (!C.grid) {
        int nb = 0;
        if (cudaFuncSetAttribute(k2::k_hash_planes, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)k2::SMEM) !=
            cudaSuccess)
            return -1;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k2::k_hash_planes, k2::THREADS, k2::SMEM) !=
                cudaSuccess ||
            nb < 1)
            return -1;
        C.grid = nb * sm_count();
    }
    return C.grid;
}

static uint32_t env_u32(const char *name, uint32_t dflt) {
    const char *v = getenv(name);
    return v && *v ? (uint32_t)strtoul(v, nullptr, 10) : dflt;
}

// Digests of n device buffers with the whole GPU (cooperative launches: every CTA co-resident).
// Buffers go MAX_JOBS (or B2L_K2_JOBS) per launch, longest first; a lone buffer gets one team
// per co-resident CTA per SM.
int hash_planes_launch_many(const void *const *d_bufs, const uint64_t *lens, uint64_t n, uint64_t *d_digests,
                            cudaStream_t stream) {
    if (n == 0) return B2L_OK;
    int dev = 0;
    B2L_CUDA(cudaGetDevice(&dev));
    k2::Ctx &C = k2::g_ctx[dev & 63];
    const int grid = k2_grid();
    if (grid < 1) return fail(B2L_E_CUDA, "k_hash_planes: no occupancy");
    std::vector<uint64_t> order(n);
    for (uint64_t i = 0; i < n; ++i) order[i] = i;
    std::stable_sort(order.begin(), order.end(), [&](uint64_t a, uint64_t b) { return lens[a] > lens[b]; });
    const uint32_t per_sm = (uint32_t)(grid / sm_count()) ? (uint32_t)(grid / sm_count()) : 1u;
    const uint32_t max_jobs = std::min<uint32_t>(std::max<uint32_t>(env_u32("B2L_K2_JOBS", k2::MAX_JOBS), 1u),
                                                 (uint32_t)k2::MAX_JOBS);
    std::lock_guard<std::mutex> lock(C.mu);
    if (!C.done) B2L_CUDA(cudaEventCreateWithFlags(&C.done, cudaEventDisableTiming));
    B2L_CUDA(cudaStreamWaitEvent(stream, C.done, 0));  // the previous K2 is done with the scratch
    for (uint64_t i0 = 0; i0 < n;) {
        const uint32_t nj = (uint32_t)std::min<uint64_t>(max_jobs, n - i0);
        for (uint32_t k = 0; k < nj; ++k)
            if (lens[order[i0 + k]] == 0) return fail(B2L_E_EMPTY_PAYLOAD, "cannot hash a zero-byte payload");
        // teams per buffer: one per co-resident CTA per SM for a lone buffer, else B2L_K2_TEAMS (1)
        uint32_t teams = nj == 1 ? per_sm : std::max<uint32_t>(env_u32("B2L_K2_TEAMS", 1), 1u);
        uint64_t G = (uint64_t)grid / ((uint64_t)nj * teams);
        if (G < 1) teams = 1, G = (uint64_t)grid / nj;
        const uint64_t nch0 = ((lens[order[i0]] + 7) / 8 + k2::CHUNK - 1) / k2::CHUNK;  // the longest
        if (nj == 1 && nch0 < (uint64_t)sm_count() * teams) teams = 1, G = std::min<uint64_t>(nch0, grid);
        else if (nch0 < G) G = nch0;
        size_t need_st = 0, need_c = 0;
        k2::Jobs J{};
        J.njobs = nj;
        J.teams = teams;
        for (uint32_t k = 0; k < nj; ++k) {
            const uint64_t len = lens[order[i0 + k]];
            const uint64_t nch = ((len + 7) / 8 + k2::CHUNK - 1) / k2::CHUNK;
            const uint64_t rounds = (nch + G - 1) / G;
            J.j[k].buf = (const uint8_t *)d_bufs[order[i0 + k]];
            J.j[k].nbytes = len;
            J.j[k].digest = d_digests + order[i0 + k];
            J.j[k].aggs = (uint4 *)(uintptr_t)need_st;  // offsets until the scratch is sized
            J.j[k].carry = (unsigned long long *)(uintptr_t)need_c;
            need_st += rounds * 16 * G * k2::SLOT_STRIDE;
            need_c += rounds * 16;
        }
        if (C.status_cap < need_st) {
            if (C.status) {
                B2L_CUDA(cudaEventSynchronize(C.done));
                B2L_CUDA(cudaStreamSynchronize(stream));
                cudaFree(C.status);
            }
            C.status = nullptr;
            C.status_cap = 0;
            B2L_CUDA(cudaMalloc(&C.status, need_st * sizeof(uint4)));
            C.status_cap = need_st;
        }
        if (C.carry_cap < need_c) {
            if (C.carry) {
                B2L_CUDA(cudaEventSynchronize(C.done));
                B2L_CUDA(cudaStreamSynchronize(stream));
                cudaFree(C.carry);
            }
            C.carry = nullptr;
            C.carry_cap = 0;
            B2L_CUDA(cudaMalloc(&C.carry, need_c * sizeof(unsigned long long)));
            C.carry_cap = need_c;
        }
        for (uint32_t k = 0; k < nj; ++k) {
            J.j[k].aggs = C.status + (uintptr_t)J.j[k].aggs;
            J.j[k].carry = C.carry + (uintptr_t)J.j[k].carry;
        }
        B2L_CUDA(cudaMemsetAsync(C.status, 0, need_st * sizeof(uint4), stream));
        B2L_CUDA(cudaMemsetAsync(C.carry, 0, need_c * sizeof(unsigned long long), stream));
        void *args[] = {(void *)&J};
        B2L_CUDA(cudaLaunchCooperativeKernel((const void *)k2::k_hash_planes, dim3((unsigned)(G * nj * teams)),
                                             dim3(k2::THREADS), args, k2::SMEM, stream));
        i0 += nj;
    }
    B2L_CUDA(cudaEventRecord(C.done, stream));
    return B2L_OK;
}

// Digest of one device buffer with the whole GPU.
int hash_planes_launch(const void *d_buf, uint64_t nbytes, uint64_t *d_digest, cudaStream_t stream) {
    if (nbytes == 0) return B2L_OK;
    return hash_planes_launch_many(&d_buf, &nbytes, 1, d_digest, stream);
}

}  // namespace b2l
