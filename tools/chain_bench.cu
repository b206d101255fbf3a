// Lone FNV-chain latency microbenchmark (tools only, not product code).
// One warp per CTA, lane 0 folds a 1 MiB L2-resident buffer; cycles per 8-B word for several
// step formulations and load schedules.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3
//   -o chain_bench tools/chain_bench.cu ; run on a B200.
#include <cstdint>
#include <cstdio>
#include <vector>

__constant__ uint32_t c435 = 435u;
constexpr uint64_t P = 0x100000001B3ull;

template <int V>
__device__ __forceinline__ void step(uint32_t &hl, uint32_t &hh, uint32_t wl, uint32_t wh) {
    if constexpr (V == 0) {  // current latency form
        const uint32_t xl = hl ^ wl, xh = hh ^ wh;
        const uint32_t c = __umulhi(xl, c435) + (xl << 8);
        asm("mul.lo.u32 %0, %1, 435;" : "=r"(hl) : "r"(xl));
        asm("mad.lo.u32 %0, %1, 435, %2;" : "=r"(hh) : "r"(xh), "r"(c));
    } else if constexpr (V == 1) {  // IMAD.WIDE form
        const uint32_t xl = hl ^ wl, xh = hh ^ wh;
        const uint64_t p = (uint64_t)xl * 435u;
        const uint32_t c = (uint32_t)(p >> 32) + (xl << 8);
        hl = (uint32_t)p;
        asm("mad.lo.u32 %0, %1, 435, %2;" : "=r"(hh) : "r"(xh), "r"(c));
    } else if constexpr (V == 2) {  // plain 64-bit
        uint64_t h = ((uint64_t)hh << 32) | hl;
        h = (h ^ (((uint64_t)wh << 32) | wl)) * P;
        hl = (uint32_t)h, hh = (uint32_t)(h >> 32);
    } else if constexpr (V == 3) {  // shift on the ALU pipe (shf), add folded into the hi IMAD chain
        const uint32_t xl = hl ^ wl, xh = hh ^ wh;
        uint32_t hi, sh;
        asm("mul.hi.u32 %0, %1, %2;" : "=r"(hi) : "r"(xl), "r"(c435));
        asm("shf.l.clamp.b32 %0, 0, %1, 8;" : "=r"(sh) : "r"(xl));
        asm("mul.lo.u32 %0, %1, 435;" : "=r"(hl) : "r"(xl));
        uint32_t t;
        asm("mad.lo.u32 %0, %1, 435, %2;" : "=r"(t) : "r"(xh), "r"(hi));
        hh = t + sh;
    } else if constexpr (V == 5) {  // wide multiply, LEA-style add off the chain
        const uint32_t xl = hl ^ wl, xh = hh ^ wh;
        uint32_t lo, hi, c;
        asm("{.reg .b64 p; mul.wide.u32 p, %2, 435; mov.b64 {%0, %1}, p;}" : "=r"(lo), "=r"(hi) : "r"(xl));
        asm("{.reg .b32 t; shl.b32 t, %1, 8; add.u32 %0, %2, t;}" : "=r"(c) : "r"(xl), "r"(hi));
        hl = lo;
        asm("mad.lo.u32 %0, %1, 435, %2;" : "=r"(hh) : "r"(xh), "r"(c));
    } else if constexpr (V == 6) {  // one IMAD.WIDE with a 64-bit addend {0, xl<<8}: lo and c at once
        const uint32_t xl = hl ^ wl, xh = hh ^ wh;
        uint32_t lo, c;
        asm("{.reg .b64 p, a; .reg .b32 t; shl.b32 t, %2, 8; mov.b64 a, {0, t}; mad.wide.u32 p, %2, 435, a; "
            "mov.b64 {%0, %1}, p;}" : "=r"(lo), "=r"(c) : "r"(xl));
        hl = lo;
        asm("mad.lo.u32 %0, %1, 435, %2;" : "=r"(hh) : "r"(xh), "r"(c));
    } else if constexpr (V == 7) {  // lo chain + an off-chain IMAD.HI per word (folded into hh)
        const uint32_t xl = hl ^ wl;
        asm("mul.lo.u32 %0, %1, 435;" : "=r"(hl) : "r"(xl));
        hh ^= __umulhi(wh ^ xl, c435);
    } else if constexpr (V == 8) {  // lo chain + an off-chain plain IMAD per word
        const uint32_t xl = hl ^ wl;
        asm("mul.lo.u32 %0, %1, 435;" : "=r"(hl) : "r"(xl));
        uint32_t t;
        asm("mad.lo.u32 %0, %1, 437, %2;" : "=r"(t) : "r"(xl), "r"(wh));
        hh ^= t;
    } else if constexpr (V == 9) {  // lo chain + hi chain without the cross term (two LOP3->IMAD chains)
        const uint32_t xl = hl ^ wl, xh = hh ^ wh;
        asm("mul.lo.u32 %0, %1, 435;" : "=r"(hl) : "r"(xl));
        asm("mad.lo.u32 %0, %1, 435, %2;" : "=r"(hh) : "r"(xh), "r"(xl));
    } else {  // V == 4: lo chain only (the dependency floor of one 32-bit LOP3 -> IMAD chain)
        const uint32_t xl = hl ^ wl;
        asm("mul.lo.u32 %0, %1, 435;" : "=r"(hl) : "r"(xl));
        hh ^= wh;
    }
}

// L = 0: load a 64-word chunk into registers, then fold it.  L = 1: two 32-word halves, the next
// half's loads issued before the current half is folded.
template <int V, int L>
__global__ void k_chain(const uint4 *__restrict__ buf, uint64_t nvec, uint64_t *out, long long *cyc, int active) {
    if (threadIdx.x >= active) return;
    uint32_t hl = 0x84222325u, hh = 0xCBF29CE4u;
    long long t0 = clock64();
    if constexpr (L == 2) {  // no loads in the loop: 16 vectors reused (the arithmetic floor)
        uint4 a[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) a[j] = __ldg(buf + j);
        t0 = clock64();
        for (uint64_t i = 0; i < nvec; i += 16) {
#pragma unroll
            for (int j = 0; j < 16; ++j) {
                step<V>(hl, hh, a[j].x, a[j].y);
                step<V>(hl, hh, a[j].z, a[j].w);
            }
        }
    } else if constexpr (L == 0) {
        for (uint64_t i = 0; i < nvec; i += 32) {
            uint4 v[32];
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] = __ldg(buf + i + j);
#pragma unroll
            for (int j = 0; j < 32; ++j) {
                step<V>(hl, hh, v[j].x, v[j].y);
                step<V>(hl, hh, v[j].z, v[j].w);
            }
        }
    } else {
        uint4 a[16], b[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) a[j] = __ldg(buf + j);
        for (uint64_t i = 0; i < nvec; i += 32) {
#pragma unroll
            for (int j = 0; j < 16; ++j) b[j] = __ldg(buf + i + 16 + j);
#pragma unroll
            for (int j = 0; j < 16; ++j) {
                step<V>(hl, hh, a[j].x, a[j].y);
                step<V>(hl, hh, a[j].z, a[j].w);
            }
            const uint64_t nx = i + 32 < nvec ? i + 32 : 0;
#pragma unroll
            for (int j = 0; j < 16; ++j) a[j] = __ldg(buf + nx + j);
#pragma unroll
            for (int j = 0; j < 16; ++j) {
                step<V>(hl, hh, b[j].x, b[j].y);
                step<V>(hl, hh, b[j].z, b[j].w);
            }
        }
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) {
        out[blockIdx.x] = ((uint64_t)hh << 32) | hl;
        cyc[blockIdx.x] = t1 - t0;
    }
}

// Two lanes per chain: lane 0 folds the low 32-bit halves (s = (s ^ wl) * 435), lane 1 the high
// halves (s = (s ^ wh) * 435 + c) one 16-word block behind, c_i = hi32(xl_i * 435) + (xl_i << 8)
// handed over by shuffle.  Registers only (the arithmetic floor of the split).
__global__ void k_chain2(const uint4 *__restrict__ buf, uint64_t nvec, uint64_t *out, long long *cyc) {
    const int lane = threadIdx.x;
    if (lane > 1) return;
    uint32_t s = lane ? 0xCBF29CE4u : 0x84222325u;
    uint32_t w[32];
#pragma unroll
    for (int j = 0; j < 16; ++j) {
        uint4 v = __ldg(buf + j);
        w[2 * j] = lane ? v.y : v.x;
        w[2 * j + 1] = lane ? v.w : v.z;
    }
    const uint32_t keep = lane ? 0u : ~0u;
    uint32_t cq[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) cq[j] = 0;
    long long t0 = clock64();
    for (uint64_t i = 0; i < nvec; i += 16) {
#pragma unroll
        for (int j = 0; j < 32; ++j) {
            const uint32_t add = __shfl_sync(3u, cq[j], 0);  // lane 0's c of the previous block
            const uint32_t x = s ^ w[j];
            uint32_t t;
            asm("mad.lo.u32 %0, %1, 435, %2;" : "=r"(t) : "r"(x), "r"(lane ? add : 0u));
            s = t;
            cq[j] = (__umulhi(x, c435) + (x << 8)) & keep;
        }
    }
    long long t1 = clock64();
    out[blockIdx.x * 2 + lane] = s;
    if (lane == 0) cyc[blockIdx.x] = t1 - t0;
}

void run2(const uint4 *d, uint64_t nvec, uint64_t *dout, long long *dcyc) {
    for (int rep = 0; rep < 3; ++rep) {
        k_chain2<<<1, 32>>>(d, nvec, dout, dcyc);
        cudaDeviceSynchronize();
        long long cyc;
        cudaMemcpy(&cyc, dcyc, 8, cudaMemcpyDeviceToHost);
        if (rep == 2) printf("two-lane split, registers        %.2f cycles/word\n", (double)cyc / (nvec * 2));
    }
}

template <int V, int L>
void run(const uint4 *d, uint64_t nvec, uint64_t *dout, long long *dcyc, const char *name, int active = 1) {
    for (int rep = 0; rep < 3; ++rep) {
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0), cudaEventCreate(&e1);
        cudaEventRecord(e0);
        k_chain<V, L><<<1, 32>>>(d, nvec, dout, dcyc, active);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        long long cyc;
        uint64_t h;
        cudaMemcpy(&cyc, dcyc, 8, cudaMemcpyDeviceToHost);
        cudaMemcpy(&h, dout, 8, cudaMemcpyDeviceToHost);
        if (rep == 2)
            printf("V%d L%d a%d %-28s %.3f ms  %.2f cycles/word  h=%016llx\n", V, L, active, name, ms, (double)cyc / (nvec * 2),
                   (unsigned long long)h);
    }
}

int main() {
    const uint64_t bytes = 1 << 20, nvec = bytes / 16;
    std::vector<uint8_t> h(bytes);
    for (uint64_t i = 0; i < bytes; ++i) h[i] = (uint8_t)(i * 2654435761u >> 13);
    uint4 *d;
    uint64_t *dout;
    long long *dcyc;
    cudaMalloc(&d, bytes), cudaMalloc(&dout, 64), cudaMalloc(&dcyc, 64);
    cudaMemcpy(d, h.data(), bytes, cudaMemcpyHostToDevice);
    run<0, 2>(d, nvec, dout, dcyc, "lat form, registers");
    run<1, 2>(d, nvec, dout, dcyc, "wide form, registers");
    run<2, 2>(d, nvec, dout, dcyc, "u64, registers");
    run<3, 2>(d, nvec, dout, dcyc, "shf form, registers");
    run<4, 2>(d, nvec, dout, dcyc, "lo chain only, registers");
    run<4, 2>(d, nvec, dout, dcyc, "lo chain only, registers", 2);
    run<4, 2>(d, nvec, dout, dcyc, "lo chain only, registers", 32);
    run<0, 2>(d, nvec, dout, dcyc, "lat form, registers", 32);
    run<5, 2>(d, nvec, dout, dcyc, "wide+lea, registers");
    run<6, 2>(d, nvec, dout, dcyc, "wide 64-bit addend, registers");
    run<7, 2>(d, nvec, dout, dcyc, "lo + off-chain IMAD.HI");
    run<8, 2>(d, nvec, dout, dcyc, "lo + off-chain IMAD");
    run<9, 2>(d, nvec, dout, dcyc, "two chains, no cross term");
    run2(d, nvec, dout, dcyc);
    return 0;
    run<0, 0>(d, nvec, dout, dcyc, "lat form, chunk");
    run<0, 1>(d, nvec, dout, dcyc, "lat form, halves");
    run<1, 0>(d, nvec, dout, dcyc, "wide form, chunk");
    run<1, 1>(d, nvec, dout, dcyc, "wide form, halves");
    run<2, 0>(d, nvec, dout, dcyc, "u64, chunk");
    run<2, 1>(d, nvec, dout, dcyc, "u64, halves");
    run<3, 0>(d, nvec, dout, dcyc, "shf form, chunk");
    run<3, 1>(d, nvec, dout, dcyc, "shf form, halves");
    run<4, 0>(d, nvec, dout, dcyc, "lo chain only, chunk");
    run<4, 1>(d, nvec, dout, dcyc, "lo chain only, halves");
    return 0;
}
