// Multi-GPU context in one process (8(e) "Hashing").
//
// Hashing shards naturally: digests of independent buffers.  Two splits:
//  * host batches (b2l_hash_host_multi): the batch is cut into contiguous, byte-balanced index
//    ranges, one per initialised device, so each device's pipeline still merges host-contiguous
//    buffers into single DMAs over its own PCIe link; one host thread per device drives
//    hash_host_impl on its range and writes its digests straight into the caller's array (the
//    gather is free: it is host memory);
//  * placement of buffers that will live on the devices (b2l_lpt_partition): LPT by size --
//    longest first, each to the least-loaded part -- so the largest serial chains spread out
//    and per-device byte loads differ by at most one buffer.
// Multi-process runs (one rank per GPU, torch.distributed) use the same LPT placement and gather
// the 8-B digests with one NCCL call (paper_2601_12713_b200/multigpu.py).
#include <algorithm>
#include <cstring>
#include <mutex>
#include <numeric>
#include <queue>
#include <thread>
#include <vector>

#include "b2l_common.cuh"

namespace b2l {
int hash_host_impl(const void *const *h_bufs, const uint64_t *h_lens, uint64_t n, uint64_t *h_digests);

namespace multi {
std::mutex g_mu;
std::vector<int> g_devs;  // initialised devices (empty: not initialised)
}  // namespace multi

// Balanced contiguous cut of a byte sequence into `parts` index ranges: range p ends at the first
// index whose prefix sum reaches (p+1)/parts of the total.
static void byte_ranges(const uint64_t *lens, uint64_t n, size_t parts, std::vector<uint64_t> &cut) {
    cut.assign(parts + 1, n);
    cut[0] = 0;
    long double total = 0;
    for (uint64_t i = 0; i < n; ++i) total += (long double)lens[i];
    long double acc = 0;
    size_t p = 1;
    for (uint64_t i = 0; i < n && p < parts; ++i) {
        acc += (long double)lens[i];
        while (p < parts && acc >= total * (long double)p / (long double)parts) cut[p++] = i + 1;
    }
    for (size_t q = 1; q <= parts; ++q) cut[q] = std::max(cut[q], cut[q - 1]);
}

}  // namespace b2l

extern "C" {

int b2l_init(int ngpus, const int *devs) {
    using namespace b2l;
    int count = 0;
    B2L_CUDA(cudaGetDeviceCount(&count));
    if (ngpus < 1 || ngpus > 64) return fail(B2L_E_INVALID_ARG, "b2l_init: ngpus must be in [1, 64]");
    std::vector<int> d(ngpus);
    for (int i = 0; i < ngpus; ++i) {
        d[i] = devs ? devs[i] : i;
        if (d[i] < 0 || d[i] >= count) return fail(B2L_E_INVALID_ARG, "b2l_init: device ordinal out of range");
    }
    int prev = 0;
    B2L_CUDA(cudaGetDevice(&prev));
    for (int x : d) {  // create the primary contexts up front (first-call latency off the hot path)
        B2L_CUDA(cudaSetDevice(x));
        B2L_CUDA(cudaFree(nullptr));
    }
    B2L_CUDA(cudaSetDevice(prev));
    std::lock_guard<std::mutex> l(multi::g_mu);
    multi::g_devs = d;
    return B2L_OK;
}

int b2l_shutdown(void) {
    using namespace b2l;
    std::vector<int> d;
    {
        std::lock_guard<std::mutex> l(multi::g_mu);
        d.swap(multi::g_devs);
    }
    int prev = 0;
    B2L_CUDA(cudaGetDevice(&prev));
    for (int x : d) {  // drain every device's queued work
        B2L_CUDA(cudaSetDevice(x));
        B2L_CUDA(cudaDeviceSynchronize());
    }
    B2L_CUDA(cudaSetDevice(prev));
    return B2L_OK;
}

int b2l_ngpus(int *n, int *devs, int cap) {
    using namespace b2l;
    if (!n) return fail(B2L_E_INVALID_ARG, "null count");
    std::lock_guard<std::mutex> l(multi::g_mu);
    *n = (int)multi::g_devs.size();
    for (int i = 0; devs && i < *n && i < cap; ++i) devs[i] = multi::g_devs[i];
    return B2L_OK;
}

int b2l_lpt_partition(const uint64_t *lens, uint64_t n, uint32_t parts, uint32_t *owner, uint64_t *load) {
    using namespace b2l;
    if ((n && (!lens || !owner)) || parts == 0) return fail(B2L_E_INVALID_ARG, "b2l_lpt_partition: bad argument");
    std::vector<uint64_t> ld(parts, 0);
    // longest first (stable: equal lengths keep index order, so equal sizes deal round robin)
    std::vector<uint32_t> ord(n);
    std::iota(ord.begin(), ord.end(), 0u);
    std::stable_sort(ord.begin(), ord.end(), [&](uint32_t a, uint32_t b) { return lens[a] > lens[b]; });
    using E = std::pair<uint64_t, uint32_t>;  // (load, part): least load, then lowest part
    std::priority_queue<E, std::vector<E>, std::greater<E>> heap;
    for (uint32_t p = 0; p < parts; ++p) heap.push({0, p});
    for (uint32_t i : ord) {
        E e = heap.top();
        heap.pop();
        owner[i] = e.second;
        e.first += lens[i];
        ld[e.second] = e.first;
        heap.push(e);
    }
    if (load) std::copy(ld.begin(), ld.end(), load);
    return B2L_OK;
}

int b2l_hash_host_multi(const void *const *h_bufs, const uint64_t *h_lens, uint64_t n, uint64_t *h_digests) {
    using namespace b2l;
    std::vector<int> d;
    {
        std::lock_guard<std::mutex> l(multi::g_mu);
        d = multi::g_devs;
    }
    if (d.empty()) return fail(B2L_E_INVALID_ARG, "b2l_hash_host_multi: call b2l_init first");
    if (n == 0) return B2L_OK;
    if (!h_bufs || !h_lens || !h_digests) return fail(B2L_E_INVALID_ARG, "b2l_hash_host_multi: null array");
    std::vector<uint64_t> cut;
    byte_ranges(h_lens, n, d.size(), cut);
    std::vector<int> rc(d.size(), B2L_OK);
    std::vector<std::string> err(d.size());
    std::vector<std::thread> th;
    for (size_t k = 0; k < d.size(); ++k) {
        if (cut[k + 1] == cut[k]) continue;
        th.emplace_back([&, k] {
            if (cudaSetDevice(d[k]) != cudaSuccess) {
                rc[k] = fail(B2L_E_CUDA, "cudaSetDevice");
            } else {
                rc[k] = hash_host_impl(h_bufs + cut[k], h_lens + cut[k], cut[k + 1] - cut[k], h_digests + cut[k]);
            }
            if (rc[k]) err[k] = b2l_last_error();
        });
    }
    for (auto &t : th) t.join();
    for (size_t k = 0; k < d.size(); ++k)  // the first failing range's error (empty payloads included)
        if (rc[k]) return fail(rc[k], err[k]);
    return B2L_OK;
}

}  // extern "C"
