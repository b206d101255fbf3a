// Collision audit on the device: replaces the reference's
// CollisionAuditStore.observe loop (hashing.py:70-92; used by `dmlens audit`,
// cli.py:206-236).  For observations (hash_i, payload_i) in order, the reference keeps
// the first payload per hash and counts every later observation whose payload differs:
//   stable sort of (hash, observation index) -> segments = distinct hashes; every
//   non-first member is compared with its segment's first payload (one CTA per
//   comparison, 8-byte words re-formed at any alignment) -> count of mismatches.
#include <mutex>

#include "b2l_prims.cuh"

namespace b2l {
namespace audit {

__device__ __forceinline__ uint64_t word_at(const uint8_t *buf, uint64_t n, uint64_t i) {
    const uint64_t start = (uint64_t)buf, a = start + 8 * i, end = start + n;
    const uint32_t r = (uint32_t)(a & 7);
    const uint64_t lo = a - r;
    uint64_t w;
    if (r == 0) {
        w = *reinterpret_cast<const unsigned long long *>(lo);
    } else {
        const uint64_t u0 = *reinterpret_cast<const unsigned long long *>(lo);
        const uint64_t u1 = (lo + 8 < end) ? *reinterpret_cast<const unsigned long long *>(lo + 8) : 0ull;
        w = (u0 >> (8 * r)) | (u1 << (64 - 8 * r));
    }
    if (a + 8 > end) w &= (1ull << (8 * (uint32_t)(end - a))) - 1;
    return w;
}

// one CTA per later observation: does its payload differ from its hash's first payload?
__global__ void k_compare(const uint64_t *__restrict__ sk, const uint32_t *__restrict__ sv, const uint64_t *ptrs,
                          const uint64_t *lens, uint64_t n, const uint32_t *__restrict__ first_pos,
                          unsigned long long *collisions) {
    __shared__ int differ;
    for (uint64_t p = blockIdx.x; p < n; p += gridDim.x) {
        const uint32_t f = first_pos[p];
        if (f == (uint32_t)p) continue;  // the stored (first) payload of this hash
        const uint32_t a = sv[f], b = sv[p];
        const uint64_t la = lens[a], lb = lens[b];
        if (threadIdx.x == 0) differ = la != lb;
        __syncthreads();
        if (!differ) {
            const uint8_t *pa = (const uint8_t *)ptrs[a], *pb = (const uint8_t *)ptrs[b];
            const uint64_t nw = (la + 7) >> 3;
            for (uint64_t i = threadIdx.x; i < nw && !differ; i += blockDim.x)
                if (word_at(pa, la, i) != word_at(pb, lb, i)) differ = 1;
        }
        __syncthreads();
        if (threadIdx.x == 0 && differ) atomicAdd(collisions, 1ull);
        __syncthreads();
    }
    (void)sk;
}

struct FirstPos {  // position of the first member of p's segment = max over heads <= p
    const uint64_t *k;
    __device__ uint64_t operator()(size_t p) const { return (p == 0 || k[p] != k[p - 1]) ? p : 0; }
};
struct StoreFirst {
    uint32_t *first;
    __device__ void operator()(size_t p, uint64_t ex, uint64_t it) const {
        first[p] = (uint32_t)(ex > it ? ex : it);
    }
};
struct IsHead {
    const uint64_t *k;
    __device__ uint32_t operator()(size_t p) const { return (p == 0 || k[p] != k[p - 1]) ? 1u : 0u; }
};
struct Nop {
    __device__ void operator()(size_t, uint32_t, uint32_t) const {}
};

__global__ void k_iota(uint32_t *v, size_t n) {
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        v[i] = (uint32_t)i;
}

std::mutex g_mu;

int audit_impl(const uint64_t *d_hashes, const uint64_t *d_ptrs, const uint64_t *d_lens, uint64_t n,
               uint64_t *collisions, uint64_t *distinct) {
    *collisions = 0, *distinct = 0;
    if (n == 0) return B2L_OK;
    if (n >= 0xFFFFFFFFull) return fail(B2L_E_INVALID_ARG, "too many observations");
    std::lock_guard<std::mutex> lock(g_mu);
    cudaStream_t s = nullptr;
    CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    struct StreamGuard {
        cudaStream_t s;
        ~StreamGuard() { cudaStreamDestroy(s); }
    } guard{s};
    {
        SortStore<1> st(n, s);
        CK(cudaMemcpyAsync(st.in_key(0), d_hashes, n * sizeof(uint64_t), cudaMemcpyDeviceToDevice, s));
        uint32_t *v = st.in_val();
        DBuf<uint32_t> first(n, s);
        DBuf<unsigned long long> acc(1, s);
        DBuf<uint32_t> nseg(1, s);
        acc.zero();
        // observation index as the sort payload
        k_iota<<<grid_for(n, 256), 256, 0, s>>>(v, n);
        CK_LAUNCH("k_iota");
        radix_sort<1>(st.b, n, LiveBytes<1>{{0xFF}}, s);
        scan<MaxU64>(n, FirstPos{st.key(0)}, StoreFirst{first.p}, s);
        scan<SumU32>(n, IsHead{st.key(0)}, Nop{}, s, nseg.p);
        k_compare<<<grid_for(n, 1, 148 * 16), 256, 0, s>>>(st.key(0), st.val(), d_ptrs, d_lens, n, first.p, acc.p);
        CK_LAUNCH("k_compare");
        unsigned long long c = 0;
        uint32_t d = 0;
        read_back(&c, acc.p, sizeof(c), s);
        read_back(&d, nseg.p, sizeof(d), s);
        *collisions = c, *distinct = d;
    }
    CK(cudaStreamSynchronize(s));
    return B2L_OK;
}

}  // namespace audit
}  // namespace b2l

extern "C" int b2l_audit_batch(const uint64_t *d_hashes, const uint64_t *d_ptrs, const uint64_t *d_lens, uint64_t n,
                               uint64_t *collisions, uint64_t *distinct) {
    if (!collisions || !distinct || (n && (!d_hashes || !d_ptrs || !d_lens)))
        return b2l::fail(B2L_E_INVALID_ARG, "null argument");
    try {
        return b2l::audit::audit_impl(d_hashes, d_ptrs, d_lens, n, collisions, distinct);
    } catch (const b2l::EngineErr &e) {
        return b2l::fail(e.code, e.msg);
    }
}
