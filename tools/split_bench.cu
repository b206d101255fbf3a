// Split-pair instrumentation (tools only): one 1 MiB buffer folded by a warp pair, total cycles
// per role and cycles each role spends waiting on the other.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --extended-lambda -DB2L_SPLIT_PROF
//   -I include -I paper_2601_12713_b200/csrc -o tools/split_bench tools/split_bench.cu
#include "b2l_hash.cu"
#include <cstdio>
#include <vector>
namespace b2l {
int fail(int code, const std::string &) { return code; }
int cuda_fail(cudaError_t, const char *) { return -1; }
int sm_count() { return 148; }
void set_error(const std::string &) {}
}  // namespace b2l
using namespace b2l;
__device__ long long g_role_cyc[2];
__device__ void hi_null(const BufCursor &cur, SplitBars *b) {  // B that only hands slots back
    const uint64_t nch = (cur.L + SPLIT_CH - 1) / SPLIT_CH;
    for (uint64_t k = 0; k < nch; ++k) {
        const int s = (int)(k % SPLIT_S);
        SPLIT_WAIT(1, &b->full[s], (uint32_t)((k / SPLIT_S) & 1));
        mbar_arrive(&b->empty[s]);
    }
}
__global__ void k_pair(const uint64_t *ptrs, const uint64_t *lens, uint64_t *dig, int mode) {
    extern __shared__ __align__(128) uint8_t smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    SplitBars *bars = reinterpret_cast<SplitBars *>(smem + 2 * SPLIT_PAIR);
    if (threadIdx.x == 0) {
        for (int p = 0; p < 2; ++p)
            for (int i = 0; i < SPLIT_S; ++i) mbar_init(&bars[p].full[i], 32), mbar_init(&bars[p].empty[i], 32);
        fence_mbar_init();
    }
    __syncthreads();
    BufCursor cur;
    cursor_load(cur, ptrs, lens, nullptr, 0, 1);
    if (mode >= 3) {  // a distinct buffer per pair (copies of the first)
        cur.a0 += (uint64_t)(blockIdx.x * 2 + (threadIdx.x >> 6)) * cur.n;
    }
    const int pair = warp >> 1, role = warp & 1;
    if (pair == 1 && mode < 2) return;  // mode 2, 3: two pairs per CTA
    uint8_t *pr = smem + pair * SPLIT_PAIR;
    long long t0 = clock64();
    if (role == 0) split_lo(cur, lane, pr, bars + pair, 0);
    else if (mode != 1) split_hi(cur, lane, pr, bars + pair, dig + blockIdx.x * 2 + pair, 0);
    else hi_null(cur, bars);
    if (lane == 0 && blockIdx.x == 0 && pair == 0) g_role_cyc[role] = clock64() - t0;
}
int main() {
    const uint64_t n = 1 << 20;
    std::vector<uint8_t> h(n);
    for (uint64_t i = 0; i < n; ++i) h[i] = (uint8_t)(i * 2654435761u >> 13);
    uint64_t hv = FNV_OFFSET;
    for (uint64_t i = 0; i < n / 8; ++i) { uint64_t w; memcpy(&w, &h[8 * i], 8); hv = (hv ^ w) * FNV_PRIME; }
    const uint64_t want = finish_digest(hv, n);
    uint8_t *d; uint64_t *dp, *dl, *dd;
    cudaMalloc(&d, n * 300); cudaMalloc(&dp, 8); cudaMalloc(&dl, 8); cudaMalloc(&dd, 8 * 1024);
    for (int i = 0; i < 300; ++i) cudaMemcpy(d + i * n, h.data(), n, cudaMemcpyHostToDevice);
    uint64_t p = (uint64_t)d;
    cudaMemcpy(dp, &p, 8, cudaMemcpyHostToDevice); cudaMemcpy(dl, &n, 8, cudaMemcpyHostToDevice);
    const int smem = 2 * SPLIT_PAIR + 2 * sizeof(SplitBars);
    cudaFuncSetAttribute(k_pair, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int modes[5] = {0, 1, 2, 2, 3}, grids[5] = {1, 1, 1, 148, 148};
    for (int rep = 0; rep < 5; ++rep) {
        long long z[2] = {0, 0};
        cudaMemcpyToSymbol(g_split_wait, z, 16);
        k_pair<<<grids[rep], 128, smem>>>(dp, dl, dd, modes[rep]);
        cudaDeviceSynchronize();
        long long cyc[2], wt[2];
        uint64_t got;
        cudaMemcpyFromSymbol(cyc, g_role_cyc, 16); cudaMemcpyFromSymbol(wt, g_split_wait, 16);
        cudaMemcpy(&got, dd, 8, cudaMemcpyDeviceToHost);
        printf("mode %d grid %d %s  A %.2f cyc/word (waits %.2f)  B %.2f cyc/word (waits %.2f)  %s\n", modes[rep], grids[rep], cudaGetErrorString(cudaGetLastError()),
               cyc[0] / (n / 8.0), wt[0] / (n / 8.0), cyc[1] / (n / 8.0), wt[1] / (n / 8.0), got == want ? "ok" : "MISMATCH");
    }
}
// CTA -> SM placement of a 2-CTA/SM launch (is the first CTA of every SM blockIdx < 148?)
__global__ void k_where(int *sm) {
    extern __shared__ uint8_t sm_[];
    if (threadIdx.x == 0) {
        int id;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(id));
        sm[blockIdx.x] = id;
        sm_[0] = 1;
    }
    long long t = clock64();
    while (clock64() - t < 200000) {}
}
struct Where {
    Where() {
        int *d;
        cudaMalloc(&d, 4096 * 4);
        const int smem = 100 << 10;
        cudaFuncSetAttribute(k_where, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        for (int grid : {296, 444}) {
            k_where<<<grid, 128, grid == 296 ? smem : 70 << 10>>>(d);
            std::vector<int> h(grid);
            cudaMemcpy(h.data(), d, grid * 4, cudaMemcpyDeviceToHost);
            std::vector<int> cnt(200, 0);
            for (int i = 0; i < 148; ++i) cnt[h[i]]++;
            int distinct = 0;
            for (int c : cnt) distinct += c > 0;
            printf("grid %d: first 148 CTAs on %d distinct SMs; ctas 0..7 on SMs", grid, distinct);
            for (int i = 0; i < 8; ++i) printf(" %d", h[i]);
            printf("\n");
        }
    }
};
