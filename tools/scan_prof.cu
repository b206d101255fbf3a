// Per-tile phase times of one single-pass scan (built with -DB2L_SCAN_PROF): load+local scan,
// look-back, store; and the tile start times (globaltimer) to see how tiles flow through the GPU.
#include <algorithm>
#include <cstdio>
#include <vector>

#include "b2l_prims.cuh"

using namespace b2l;
struct SeqLoad {
    const uint32_t *x;
    __device__ uint32_t operator()(size_t i) const { return x[i] & 1u; }
};
struct ExStore {
    uint32_t *out;
    __device__ void operator()(size_t i, uint32_t ex, uint32_t) const { out[i] = ex; }
};
int main(int argc, char **argv) {
    size_t n = argc > 1 ? strtoull(argv[1], nullptr, 10) : 10000000;
    cudaStream_t s;
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    uint32_t *x, *out;
    cudaMalloc(&x, n * 4), cudaMalloc(&out, n * 4);
    cudaMemset(x, 1, n * 4);
    for (int r = 0; r < 5; ++r) {
        Arena ar;
        ar.open(size_t(64) << 20, s, size_t(4) << 20);
        ArenaUse au(&ar);
        scan<SumU32>(n, SeqLoad{x}, ExStore{out}, s);
        cudaStreamSynchronize(s);
    }
    const size_t tiles = (n + SCAN_THREADS * scan_items<uint32_t>() - 1) / (SCAN_THREADS * scan_items<uint32_t>());
    std::vector<long long> h(tiles * 6);
    cudaMemcpyFromSymbol(h.data(), g_scan_prof, tiles * 6 * 8);
    long long g0 = h[0], gend = 0;
    double a = 0, b = 0, c = 0;
    for (size_t t = 0; t < tiles; ++t) {
        g0 = std::min(g0, h[t * 6]), gend = std::max(gend, h[t * 6 + 4]);
        a += h[t * 6 + 1], b += h[t * 6 + 2], c += h[t * 6 + 3];
    }
    printf("n %zu tiles %zu: span %.1f us; per tile (cycles): load+scan %.0f  lookback %.0f  store %.0f\n", n, tiles,
           (gend - g0) * 1e-3, a / tiles, b / tiles, c / tiles);
    for (size_t t : {size_t(0), size_t(1), size_t(100), size_t(500), size_t(1000), tiles / 2, tiles - 1})
        if (t < tiles)
            printf("  tile %6zu sm %3lld start %8.2f us end %8.2f us  load %6lld lb %6lld st %6lld cyc\n", t, h[t * 6 + 5],
                   (h[t * 6] - g0) * 1e-3, (h[t * 6 + 4] - g0) * 1e-3, h[t * 6 + 1], h[t * 6 + 2], h[t * 6 + 3]);
    // how many tiles were in flight at the midpoint
    long long mid = g0 + (gend - g0) / 2;
    int inflight = 0;
    for (size_t t = 0; t < tiles; ++t) inflight += h[t * 6] <= mid && h[t * 6 + 4] >= mid;
    printf("  in flight at mid-span: %d\n", inflight);
    return 0;
}
