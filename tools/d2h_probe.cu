// Device->host copy bandwidth of a C4-sized result (678 MB): page-locked by
// cudaHostAlloc vs malloc + cudaHostRegister (the result-block cache), one
// stream vs two, and pageable memory for comparison.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <cstring>

static float d2h(void* h, const void* d, size_t bytes, int ns, cudaStream_t* st) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e9f;
    for (int rep = 0; rep < 5; ++rep) {
        cudaEventRecord(e0, st[0]);
        for (int k = 1; k < ns; ++k) cudaStreamWaitEvent(st[k], e0, 0);
        const size_t part = bytes / ns;
        for (int k = 0; k < ns; ++k)
            cudaMemcpyAsync(static_cast<char*>(h) + k * part, static_cast<const char*>(d) + k * part, part,
                            cudaMemcpyDeviceToHost, st[k]);
        for (int k = 1; k < ns; ++k) {
            cudaEvent_t ek;
            cudaEventCreateWithFlags(&ek, cudaEventDisableTiming);
            cudaEventRecord(ek, st[k]);
            cudaStreamWaitEvent(st[0], ek, 0);
        }
        cudaEventRecord(e1, st[0]);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    return best;
}

int main() {
    const size_t bytes = size_t(678) << 20;
    void* d;
    cudaMalloc(&d, bytes);
    cudaMemset(d, 1, bytes);
    cudaStream_t st[2];
    for (auto& x : st) cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking);
    void* ha;
    cudaHostAlloc(&ha, bytes, cudaHostAllocPortable);
    void* hr = std::aligned_alloc(size_t(2) << 20, bytes);
    std::memset(hr, 0, bytes);
    cudaHostRegister(hr, bytes, cudaHostRegisterPortable);
    void* hp = std::aligned_alloc(size_t(2) << 20, bytes);
    std::memset(hp, 0, bytes);
    for (int ns : {1, 2}) {
        float a = d2h(ha, d, bytes, ns, st), r = d2h(hr, d, bytes, ns, st);
        std::printf("streams=%d hostalloc %.2f ms (%.1f GB/s)  registered %.2f ms (%.1f GB/s)\n", ns, a,
                    bytes / (a * 1e6), r, bytes / (r * 1e6));
    }
    float p = d2h(hp, d, bytes, 1, st);
    std::printf("pageable %.2f ms (%.1f GB/s)\n", p, bytes / (p * 1e6));
    std::printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
