// Host->device copy bandwidth from page-locked memory: one buffer split over
// 1, 2 or 4 streams (copy engines), sizes as a per-join collection upload.
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>

int main() {
    const size_t sizes[] = {size_t(2) << 20, size_t(10) << 20, size_t(64) << 20};
    void* h;
    void* d;
    cudaMallocHost(&h, size_t(64) << 20);
    cudaMalloc(&d, size_t(64) << 20);
    cudaStream_t st[4];
    for (auto& x : st) cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (size_t bytes : sizes) {
        for (int ns : {1, 2, 4}) {
            float best = 1e9f;
            for (int rep = 0; rep < 10; ++rep) {
                cudaEventRecord(e0, st[0]);
                for (int k = 1; k < ns; ++k) cudaStreamWaitEvent(st[k], e0, 0);
                const size_t part = bytes / ns;
                for (int k = 0; k < ns; ++k)
                    cudaMemcpyAsync(static_cast<char*>(d) + k * part, static_cast<char*>(h) + k * part, part,
                                    cudaMemcpyHostToDevice, st[k]);
                for (int k = 1; k < ns; ++k) {
                    cudaEvent_t ek;
                    cudaEventCreateWithFlags(&ek, cudaEventDisableTiming);
                    cudaEventRecord(ek, st[k]);
                    cudaStreamWaitEvent(st[0], ek, 0);
                    cudaEventDestroy(ek);
                }
                cudaEventRecord(e1, st[0]);
                cudaEventSynchronize(e1);
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                if (ms < best) best = ms;
            }
            std::printf("bytes=%zu streams=%d  %.3f ms  %.1f GB/s\n", bytes, ns, best, bytes / best / 1e6);
        }
    }
    return 0;
}
