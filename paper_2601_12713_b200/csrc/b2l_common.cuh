// Shared helpers for libb2l: error plumbing and small PTX wrappers (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <string>
#include "b2l.h"

namespace b2l {

// Thread-local last error (b2l_last_error()).
void set_error(const std::string &msg);
int fail(int code, const std::string &msg);
int cuda_fail(cudaError_t e, const char *what);

#define B2L_CUDA(call)                                   \
    do {                                                 \
        cudaError_t _e = (call);                         \
        if (_e != cudaSuccess) return ::b2l::cuda_fail(_e, #call); \
    } while (0)

#define B2L_CHECK_LAUNCH(what)                           \
    do {                                                 \
        cudaError_t _e = cudaGetLastError();             \
        if (_e != cudaSuccess) return ::b2l::cuda_fail(_e, what); \
    } while (0)

int sm_count();  // cached multiprocessor count of the current device

// ---------------------------------------------------------------- PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "W%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra W%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// 1-D TMA bulk copy global -> shared, completion signalled on `bar` (complete_tx).
// src and dst 16-B aligned, bytes a multiple of 16.
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar,
                                         uint64_t policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}
__device__ __forceinline__ uint64_t l2_policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}

// ---------------------------------------------------------------- hash constants
// dmlens.hashing: _FNV_OFFSET / _FNV_PRIME (hashing.py:23-24), fmix64 (hashing.py:46-51)
constexpr uint64_t FNV_OFFSET = 0xCBF29CE484222325ull;
constexpr uint64_t FNV_PRIME = 0x100000001B3ull;

__host__ __device__ __forceinline__ uint64_t fmix64(uint64_t h) {
    h ^= h >> 33;
    h *= 0xFF51AFD7ED558CCDull;
    h ^= h >> 33;
    h *= 0xC4CEB9FE1A85EC53ull;
    h ^= h >> 33;
    return h;
}
__host__ __device__ __forceinline__ uint64_t fnv_step(uint64_t h, uint64_t w) { return (h ^ w) * FNV_PRIME; }
// One FNV step on 32-bit halves.  P = 2^40 + 435, so
//   lo' = lo32(xl*435),  hi' = xh*435 + hi32(xl*435) + (xl << 8)
// and the hi recurrence is one IMAD (xh*435 + c) whose addend c comes off the lo chain.
__device__ __forceinline__ void fnv_step32(uint32_t &hl, uint32_t &hh, uint32_t wl, uint32_t wh) {
    const uint32_t xl = hl ^ wl, xh = hh ^ wh;
    const uint64_t p = (uint64_t)xl * 435u;
    const uint32_t c = (uint32_t)(p >> 32) + (xl << 8);
    hl = (uint32_t)p;
    // keep the hi recurrence a single IMAD on the critical path (stop re-association)
    asm("mad.lo.u32 %0, %1, 435, %2;" : "=r"(hh) : "r"(xh), "r"(c));
}
// Latency form for a lone chain: the lo recurrence is a plain IMAD (no IMAD.WIDE on the
// critical path); hi32(xl*435) comes from a separate IMAD.HI off the chain.
// (the IMAD.HI multiplier is read from constant memory so ptxas cannot re-fuse the pair into
// one IMAD.WIDE)
__constant__ static uint32_t c_fnv_prime_lo = 435u;
__device__ __forceinline__ void fnv_step32_lat(uint32_t &hl, uint32_t &hh, uint32_t wl, uint32_t wh) {
    const uint32_t xl = hl ^ wl, xh = hh ^ wh;
    const uint32_t c = __umulhi(xl, c_fnv_prime_lo) + (xl << 8);
    asm("mul.lo.u32 %0, %1, 435;" : "=r"(hl) : "r"(xl));
    asm("mad.lo.u32 %0, %1, 435, %2;" : "=r"(hh) : "r"(xh), "r"(c));
}
__host__ __device__ __forceinline__ uint64_t finish_digest(uint64_t h, uint64_t n) {
    h = fmix64(h ^ n);
    return h ? h : 1ull;
}

}  // namespace b2l
