// C ABI of libb2l (declared in include/b2l.h): error plumbing, device info,
// hashing entry points and the host-buffer (end-to-end) hashing pipeline.
#include <algorithm>
#include <cstring>
#include <mutex>
#include <numeric>
#include <string>
#include <vector>

#include "b2l_common.cuh"

namespace b2l {

static thread_local std::string t_last_error;

void set_error(const std::string &msg) { t_last_error = msg; }
int fail(int code, const std::string &msg) {
    t_last_error = msg;
    return code;
}
int cuda_fail(cudaError_t e, const char *what) {
    t_last_error = std::string(what) + ": " + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) + ")";
    return e == cudaErrorMemoryAllocation ? B2L_E_OOM : B2L_E_CUDA;
}

int sm_count() {
    static int cached[64] = {0};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
    if (!cached[dev]) {
        int v = 0;
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        cached[dev] = v > 0 ? v : 148;
    }
    return cached[dev];
}

// defined in b2l_hash.cu
int hash_batch_launch(const uint64_t *, const uint64_t *, uint64_t, uint64_t *, const uint32_t *, cudaStream_t);
int hash_launch_info(uint64_t, int *, int *, int *);
int hash_select_variant(int, int *);
int hash_planes_launch(const void *, uint64_t, uint64_t *, cudaStream_t);
int hash_planes_launch_many(const void *const *, const uint64_t *, uint64_t, uint64_t *, cudaStream_t);
constexpr uint64_t K2_MIN_BYTES = 32ull << 20;  // serial chain >= ~20 ms: the whole-GPU fold wins
constexpr uint64_t K2_SOLO_BYTES = 96ull << 10;  // a call hashing ONE buffer: K2 (~80 us floor) beats the 1.6 ns/B chain
int fill_payloads_launch(uint8_t *, const uint64_t *, const uint64_t *, const uint64_t *, uint64_t, uint64_t,
                         cudaStream_t);

// ------------------------------------------------------------------ host pipeline
// Double-buffered device ring: batch b's host->device copy (side stream) overlaps
// batch b-1's hashing (compute stream).  Contiguous host buffers are merged into
// one DMA.  One pipeline per device, serialized by that device's mutex.
namespace {

constexpr uint64_t RING_SLOT_BYTES = 512ull << 20;

struct Slot {
    uint8_t *d_data = nullptr;
    uint64_t cap = 0;
    uint64_t *h_meta = nullptr;  // pinned: [ptrs | lens] for the batch
    uint32_t *h_order = nullptr;
    uint64_t *d_meta = nullptr;
    uint32_t *d_order = nullptr;
    uint64_t meta_cap = 0;
    cudaEvent_t copied = nullptr, hashed = nullptr;
    bool used = false;
};

struct HostPipe {
    int device = -1;
    cudaStream_t copy = nullptr, comp = nullptr;
    Slot slot[2];
    uint64_t *d_digests = nullptr;
    uint64_t dig_cap = 0;
    uint8_t *h_small = nullptr, *d_small = nullptr;  // one-DMA staging for small calls (pinned / device)
};

// Small calls (the per-event HashFn drop-in: one payload of a few bytes to a few KiB) are
// latency-bound: the payloads are packed behind their (ptr, len) table in one pinned block,
// moved by ONE host->device copy, hashed, and the digests come back by one device->host copy.
constexpr uint64_t SMALL_MAX_BUFS = 64, SMALL_BYTES = 64ull << 10, ZERO_COPY_BYTES = 4096;
constexpr uint64_t SMALL_META = 16 * SMALL_MAX_BUFS, SMALL_CAP = SMALL_META + SMALL_BYTES + 8 * SMALL_MAX_BUFS;

std::mutex g_pipe_mu[64];  // one per device: pipelines of different GPUs run concurrently
HostPipe g_pipes[64];

int ensure_slot(Slot &s, uint64_t data_bytes, uint64_t nbuf) {
    if (!s.copied) {
        B2L_CUDA(cudaEventCreateWithFlags(&s.copied, cudaEventDisableTiming));
        B2L_CUDA(cudaEventCreateWithFlags(&s.hashed, cudaEventDisableTiming));
    }
    if (s.cap < data_bytes) {
        if (s.used) B2L_CUDA(cudaEventSynchronize(s.hashed));
        if (s.d_data) cudaFree(s.d_data);
        s.d_data = nullptr;
        s.cap = 0;
        B2L_CUDA(cudaMalloc(&s.d_data, data_bytes));
        s.cap = data_bytes;
    }
    if (s.meta_cap < nbuf) {
        if (s.used) B2L_CUDA(cudaEventSynchronize(s.hashed));
        if (s.h_meta) cudaFreeHost(s.h_meta);
        if (s.h_order) cudaFreeHost(s.h_order);
        if (s.d_meta) cudaFree(s.d_meta);
        if (s.d_order) cudaFree(s.d_order);
        s.h_meta = nullptr;
        s.h_order = nullptr;
        s.d_meta = nullptr;
        s.d_order = nullptr;
        s.meta_cap = 0;
        uint64_t cap = std::max<uint64_t>(nbuf, 4096);
        B2L_CUDA(cudaMallocHost(&s.h_meta, 2 * cap * sizeof(uint64_t)));
        B2L_CUDA(cudaMallocHost(&s.h_order, cap * sizeof(uint32_t)));
        B2L_CUDA(cudaMalloc(&s.d_meta, 2 * cap * sizeof(uint64_t)));
        B2L_CUDA(cudaMalloc(&s.d_order, cap * sizeof(uint32_t)));
        s.meta_cap = cap;
    }
    return B2L_OK;
}

inline uint64_t span_bytes(uint64_t start, uint64_t len) { return len + (start & 15) + 16; }

int hash_small(HostPipe &P, const void *const *h_bufs, const uint64_t *h_lens, uint64_t n, uint64_t *h_digests) {
    if (!P.h_small) {
        B2L_CUDA(cudaMallocHost(&P.h_small, SMALL_CAP));
        B2L_CUDA(cudaMalloc(&P.d_small, SMALL_CAP));
    }
    uint64_t total = 0;
    for (uint64_t i = 0; i < n; ++i) total += (h_lens[i] + 15) & ~15ull;
    // a few KiB: the kernel reads the pinned block in place and writes the digests back to it
    // (host-mapped memory through unified addressing): no copy launches at all
    const bool zero_copy = total <= ZERO_COPY_BYTES;
    uint8_t *const dev_view = zero_copy ? P.h_small : P.d_small;
    uint64_t *hp = (uint64_t *)P.h_small, *hl = hp + n;
    uint64_t off = SMALL_META;
    bool any_empty = false;
    for (uint64_t i = 0; i < n; ++i) {
        if (h_lens[i]) std::memcpy(P.h_small + off, h_bufs[i], h_lens[i]);
        any_empty |= h_lens[i] == 0;
        hp[i] = (uint64_t)(dev_view + off);
        hl[i] = h_lens[i];
        off += (h_lens[i] + 15) & ~15ull;
    }
    const uint64_t dig_off = SMALL_META + SMALL_BYTES;
    uint64_t *d_dig = (uint64_t *)(dev_view + dig_off), *h_dig = (uint64_t *)(P.h_small + dig_off);
    if (!zero_copy) B2L_CUDA(cudaMemcpyAsync(P.d_small, P.h_small, off, cudaMemcpyHostToDevice, P.comp));
    const uint64_t *d_meta = (const uint64_t *)dev_view;
    int rc = hash_batch_launch(d_meta, d_meta + n, n, d_dig, nullptr, P.comp);
    if (rc) return rc;
    if (!zero_copy) B2L_CUDA(cudaMemcpyAsync(h_dig, d_dig, n * sizeof(uint64_t), cudaMemcpyDeviceToHost, P.comp));
    B2L_CUDA(cudaStreamSynchronize(P.comp));
    std::memcpy(h_digests, h_dig, n * sizeof(uint64_t));
    if (any_empty) return fail(B2L_E_EMPTY_PAYLOAD, "cannot hash a zero-byte payload");
    return B2L_OK;
}

}  // namespace

int hash_host_impl(const void *const *h_bufs, const uint64_t *h_lens, uint64_t n, uint64_t *h_digests) {
    if (n == 0) return B2L_OK;
    if (!h_bufs || !h_lens || !h_digests) return fail(B2L_E_INVALID_ARG, "b2l_hash_host: null array");
    int dev = 0;
    B2L_CUDA(cudaGetDevice(&dev));
    if (dev < 0 || dev >= 64) return fail(B2L_E_INVALID_ARG, "device ordinal out of range");
    std::lock_guard<std::mutex> lock(g_pipe_mu[dev]);
    HostPipe &P = g_pipes[dev];
    if (!P.copy) {
        B2L_CUDA(cudaStreamCreateWithFlags(&P.copy, cudaStreamNonBlocking));
        B2L_CUDA(cudaStreamCreateWithFlags(&P.comp, cudaStreamNonBlocking));
        P.device = dev;
    }
    if (n <= SMALL_MAX_BUFS) {
        uint64_t tot = 0;
        for (uint64_t i = 0; i < n; ++i) tot += (h_lens[i] + 15) & ~15ull;
        if (tot <= SMALL_BYTES) return hash_small(P, h_bufs, h_lens, n, h_digests);
    }
    if (P.dig_cap < n) {
        if (P.d_digests) cudaFree(P.d_digests);
        P.d_digests = nullptr;
        P.dig_cap = 0;
        B2L_CUDA(cudaMalloc(&P.d_digests, n * sizeof(uint64_t)));
        P.dig_cap = n;
    }
    bool any_empty = false;
    uint64_t i0 = 0;
    int cur = 0;
    while (i0 < n) {
        // ---- form batch [i0, i1): fits one ring slot (a single oversized buffer gets its own, grown slot)
        uint64_t i1 = i0, bytes = 0;
        while (i1 < n) {
            // ring bytes of buffer i1 (with the gap a merged copy run carries; see the copy plan)
            uint64_t sb = span_bytes((uint64_t)h_bufs[i1], h_lens[i1]) + (i1 > i0 ? 4096 : 0);
            if (i1 > i0 && (bytes + sb > RING_SLOT_BYTES || h_lens[i1] >= K2_MIN_BYTES)) break;
            if (h_lens[i1] >= K2_MIN_BYTES) {  // huge buffers are hashed alone by K2
                bytes += sb;
                ++i1;
                break;
            }
            bytes += sb;
            ++i1;
        }
        const uint64_t nb = i1 - i0;
        Slot &S = P.slot[cur];
        int rc = ensure_slot(S, std::max(bytes, RING_SLOT_BYTES), nb);
        if (rc) return rc;
        if (S.used) B2L_CUDA(cudaEventSynchronize(S.hashed));  // ring slot + pinned meta free again
        // ---- copy plan: merge host-contiguous runs into one DMA, keep (addr mod 16) in the ring
        uint64_t *mp = S.h_meta, *ml = S.h_meta + nb;
        uint64_t off = 0;
        bool uniform = true;
        for (uint64_t k = i0; k < i1;) {
            uint64_t run_start = (uint64_t)h_bufs[k];
            uint64_t run_end = run_start + h_lens[k];
            uint64_t e = k + 1;
            // one DMA per run of buffers that follow each other in host memory: adjacent, or
            // separated by a gap that lies in pages the two buffers already touch (a page holding
            // any buffer byte is mapped -- and pinned, when the buffer is -- so copying the rest of
            // it is safe).  Thousands of separate copies of small buffers cost ~5 us each.
            auto joins = [&](uint64_t next) {
                if (next < run_end) return false;
                if (next == run_end) return true;
                const uint64_t last_page = (run_end - 1) >> 12, next_page = next >> 12;
                return run_end > run_start && next_page <= last_page + 1 && next - run_end <= 4096;
            };
            while (e < i1 && h_lens[e] && joins((uint64_t)h_bufs[e])) {
                run_end = (uint64_t)h_bufs[e] + h_lens[e];
                ++e;
            }
            off = ((off + 15) & ~15ull) + (run_start & 15);
            uint8_t *dst = S.d_data + off;
            if (run_end > run_start)
                B2L_CUDA(cudaMemcpyAsync(dst, (const void *)run_start, run_end - run_start, cudaMemcpyHostToDevice,
                                         P.copy));
            for (uint64_t j = k; j < e; ++j) {
                mp[j - i0] = (uint64_t)dst + ((uint64_t)h_bufs[j] - run_start);
                ml[j - i0] = h_lens[j];
                if (h_lens[j] == 0) any_empty = true;
                if (h_lens[j] != h_lens[i0]) uniform = false;
            }
            off += run_end - run_start;
            k = e;
        }
        const uint32_t *d_order = nullptr;
        if (!uniform) {  // longest-first processing order (static LPT over lanes)
            std::iota(S.h_order, S.h_order + nb, 0u);
            std::stable_sort(S.h_order, S.h_order + nb, [&](uint32_t a, uint32_t b) { return ml[a] > ml[b]; });
            B2L_CUDA(cudaMemcpyAsync(S.d_order, S.h_order, nb * sizeof(uint32_t), cudaMemcpyHostToDevice, P.copy));
            d_order = S.d_order;
        }
        B2L_CUDA(cudaMemcpyAsync(S.d_meta, S.h_meta, 2 * nb * sizeof(uint64_t), cudaMemcpyHostToDevice, P.copy));
        B2L_CUDA(cudaEventRecord(S.copied, P.copy));
        B2L_CUDA(cudaStreamWaitEvent(P.comp, S.copied, 0));
        if (nb == 1 && (h_lens[i0] >= K2_MIN_BYTES || (n == 1 && h_lens[i0] >= K2_SOLO_BYTES)))  // whole-GPU fold
            rc = hash_planes_launch((const void *)mp[0], h_lens[i0], P.d_digests + i0, P.comp);
        else
            rc = hash_batch_launch(S.d_meta, S.d_meta + nb, nb, P.d_digests + i0, d_order, P.comp);
        if (rc) return rc;
        B2L_CUDA(cudaEventRecord(S.hashed, P.comp));
        S.used = true;
        i0 = i1;
        cur ^= 1;
    }
    B2L_CUDA(cudaMemcpyAsync(h_digests, P.d_digests, n * sizeof(uint64_t), cudaMemcpyDeviceToHost, P.comp));
    B2L_CUDA(cudaStreamSynchronize(P.comp));
    if (any_empty) return fail(B2L_E_EMPTY_PAYLOAD, "cannot hash a zero-byte payload");
    return B2L_OK;
}

}  // namespace b2l

// =================================================================== extern "C"
extern "C" {

int b2l_abi_version(void) { return B2L_ABI_VERSION; }

const char *b2l_last_error(void) { return b2l::t_last_error.c_str(); }

int b2l_device_count(int *count) {
    if (!count) return b2l::fail(B2L_E_INVALID_ARG, "null count");
    cudaError_t e = cudaGetDeviceCount(count);
    if (e != cudaSuccess) {
        *count = 0;
        return b2l::cuda_fail(e, "cudaGetDeviceCount");
    }
    return B2L_OK;
}

int b2l_hash_batch(const uint64_t *d_ptrs, const uint64_t *d_lens, uint64_t n, uint64_t *d_digests,
                   const uint32_t *d_order, void *stream) {
    return b2l::hash_batch_launch(d_ptrs, d_lens, n, d_digests, d_order, (cudaStream_t)stream);
}

int b2l_hash_host(const void *const *h_bufs, const uint64_t *h_lens, uint64_t n, uint64_t *h_digests) {
    return b2l::hash_host_impl(h_bufs, h_lens, n, h_digests);
}

int b2l_hash_large(const void *d_buf, uint64_t len, uint64_t *d_digest, void *stream) {
    if (!d_buf || !d_digest) return b2l::fail(B2L_E_INVALID_ARG, "null argument");
    if (len == 0) return b2l::fail(B2L_E_EMPTY_PAYLOAD, "cannot hash a zero-byte payload");
    return b2l::hash_planes_launch(d_buf, len, d_digest, (cudaStream_t)stream);
}

int b2l_hash_large_many(const void *const *d_bufs, const uint64_t *lens, uint64_t n, uint64_t *d_digests,
                        void *stream) {
    if (n && (!d_bufs || !lens || !d_digests)) return b2l::fail(B2L_E_INVALID_ARG, "null argument");
    for (uint64_t i = 0; i < n; ++i) {
        if (lens[i] == 0) return b2l::fail(B2L_E_EMPTY_PAYLOAD, "cannot hash a zero-byte payload");
        if (!d_bufs[i]) return b2l::fail(B2L_E_INVALID_ARG, "null buffer");
    }
    return b2l::hash_planes_launch_many(d_bufs, lens, n, d_digests, (cudaStream_t)stream);
}

int b2l_hash_bytes(const void *h_buf, uint64_t len, uint64_t *digest) {
    if (!digest) return b2l::fail(B2L_E_INVALID_ARG, "null digest");
    if (len == 0) return b2l::fail(B2L_E_EMPTY_PAYLOAD, "cannot hash a zero-byte payload");
    if (!h_buf) return b2l::fail(B2L_E_INVALID_ARG, "null payload");
    const void *bufs[1] = {h_buf};
    return b2l::hash_host_impl(bufs, &len, 1, digest);
}

int b2l_fill_payloads(uint8_t *d_base, const uint64_t *d_offsets, const uint64_t *d_lens,
                      const uint64_t *d_content_ids, uint64_t n, uint64_t seed, void *stream) {
    if (!d_base || !d_offsets || !d_lens || !d_content_ids) return b2l::fail(B2L_E_INVALID_ARG, "null array");
    return b2l::fill_payloads_launch(d_base, d_offsets, d_lens, d_content_ids, n, seed, (cudaStream_t)stream);
}

int b2l_hash_select_variant(int variant, int *count) { return b2l::hash_select_variant(variant, count); }

int b2l_hash_launch_info(uint64_t n, int *grid, int *block, int *smem_bytes) {
    return b2l::hash_launch_info(n, grid, block, smem_bytes);
}

}  // extern "C"
