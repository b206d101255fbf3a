// Host cost of a kernel launch: <<<>>> vs cudaLaunchKernelEx (with / without the programmatic
// serialisation attribute), from 1 and 3 host threads on 3 streams.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o /tmp/lb tools/launch_bench.cu -lpthread
#include <cuda_runtime.h>
#include <chrono>
#include <cstdio>
#include <thread>
#include <vector>

__global__ void k_empty(int *p, int v) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;");
    if (p && threadIdx.x == 0 && blockIdx.x == 0 && v < 0) *p = v;
}

static double run(int mode, int threads, int per_thread) {
    std::vector<cudaStream_t> st(threads);
    for (auto &s : st) cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    auto body = [&](int t) {
        cudaStream_t s = st[t];
        for (int i = 0; i < per_thread; ++i) {
            if (mode == 0) {
                k_empty<<<148, 256, 0, s>>>(nullptr, i);
            } else {
                cudaLaunchConfig_t cfg = {};
                cfg.gridDim = 148, cfg.blockDim = 256, cfg.stream = s;
                cudaLaunchAttribute at[1];
                at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
                at[0].val.programmaticStreamSerializationAllowed = 1;
                cfg.attrs = at, cfg.numAttrs = mode == 2 ? 1 : 0;
                cudaLaunchKernelEx(&cfg, k_empty, (int *)nullptr, i);
            }
            if (i % 64 == 63) cudaStreamSynchronize(s);  // keep the queue short, like the engine
        }
        cudaStreamSynchronize(s);
    };
    body(0);  // warm
    auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> th;
    for (int t = 0; t < threads; ++t) th.emplace_back(body, t);
    for (auto &x : th) x.join();
    double us = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count();
    for (auto &s : st) cudaStreamDestroy(s);
    return us / (threads * per_thread);
}

int main() {
    cudaFree(0);
    const char *names[3] = {"<<<>>>", "LaunchKernelEx", "LaunchKernelEx+PDL"};
    for (int threads : {1, 3})
        for (int mode = 0; mode < 3; ++mode)
            printf("%-20s threads %d: %.2f us per launch (wall / launches)\n", names[mode], threads, run(mode, threads, 2048));
    return 0;
}
