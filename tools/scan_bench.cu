// Single-pass scan in isolation: device time of one scan<> launch at several sizes, with a
// sequential load and with a three-level gather load (like the pairing depth scan), against a
// plain copy of the same bytes.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --extended-lambda -I paper_2601_12713_b200/csrc -I include \
//        -o tools/scan_bench tools/scan_bench.cu
#include <cstdio>
#include <vector>

#include "b2l_prims.cuh"

using namespace b2l;

struct SeqLoad {
    const uint32_t *x;
    __device__ uint32_t operator()(size_t i) const { return x[i] & 1u; }
};
struct GatherLoad {  // x[perm[perm[i]]]: two dependent random reads, then the value
    const uint32_t *x, *perm;
    __device__ uint32_t operator()(size_t i) const { return x[perm[perm[i]]] & 1u; }
};
struct ExStore {
    uint32_t *out;
    __device__ void operator()(size_t i, uint32_t ex, uint32_t) const { out[i] = ex; }
};
struct ExStoreS {
    static constexpr bool kStriped = true;
    uint32_t *out;
    __device__ void operator()(size_t i, uint32_t ex, uint32_t) const { out[i] = ex; }
};
__global__ void k_copy(const uint32_t *a, uint32_t *b, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) b[i] = a[i];
}

template <class F>
static float time_it(cudaStream_t s, F f, int reps = 20) {
    cudaEvent_t a, b;
    cudaEventCreate(&a), cudaEventCreate(&b);
    float tot = 0;
    for (int r = 0; r < reps + 3; ++r) {
        Arena ar;
        ar.open(size_t(64) << 20, s, size_t(4) << 20);
        ArenaUse au(&ar);
        cudaEventRecord(a, s);
        f();
        cudaEventRecord(b, s);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (r >= 3) tot += ms;
    }
    return tot / reps * 1e3f;
}

int main() {
    cudaStream_t s;
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    for (size_t n : {size_t(100000), size_t(400000), size_t(1000000), size_t(4000000), size_t(10000000), size_t(30000000)}) {
        std::vector<uint32_t> h(n), p(n);
        uint64_t z = 88172645463325252ull;
        for (size_t i = 0; i < n; ++i) {
            z ^= z << 13, z ^= z >> 7, z ^= z << 17;
            h[i] = (uint32_t)z, p[i] = (uint32_t)i;
        }
        for (size_t i = n - 1; i > 0; --i) {
            z ^= z << 13, z ^= z >> 7, z ^= z << 17;
            std::swap(p[i], p[z % (i + 1)]);
        }
        uint32_t *x, *perm, *out;
        cudaMalloc(&x, n * 4), cudaMalloc(&perm, n * 4), cudaMalloc(&out, n * 4);
        cudaMemcpy(x, h.data(), n * 4, cudaMemcpyHostToDevice);
        cudaMemcpy(perm, p.data(), n * 4, cudaMemcpyHostToDevice);
        const float tc = time_it(s, [&] { k_copy<<<148 * 8, 256, 0, s>>>(x, out, n); });
        const float ts = time_it(s, [&] { scan<SumU32>(n, SeqLoad{x}, ExStore{out}, s); });
        const float tg = time_it(s, [&] { scan<SumU32>(n, GatherLoad{x, perm}, ExStore{out}, s); });
        const float ts2 = time_it(s, [&] { scan<SumU32>(n, SeqLoad{x}, ExStoreS{out}, s); });
        const float tg2 = time_it(s, [&] { scan<SumU32>(n, GatherLoad{x, perm}, ExStoreS{out}, s); });
        printf("n %9zu: copy %6.1f us | blocked: seq %6.1f us (%5.0f GB/s) gather %6.1f | striped: seq %6.1f us (%5.0f GB/s) gather %6.1f\n",
               n, tc, ts, 8.0 * n / ts * 1e-3, tg, ts2, 8.0 * n / ts2 * 1e-3, tg2);
        cudaFree(x), cudaFree(perm), cudaFree(out);
    }
    return 0;
}
