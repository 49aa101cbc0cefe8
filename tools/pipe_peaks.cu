// Integer-pipe microbenchmark for the filter kernel's roofline: full-chip
// throughput of 32-bit POPC and of LOP3 on sm_100a, measured with CUDA events.
// Built by __graft_entry__.build() into paper_1711_07295_b200/lib/pipe_peaks;
// bench.py runs it on the GPU box and uses the POPC figure as the peak of the
// K2 filter (which issues b/32 POPC per pair comparison).
//   usage: pipe_peaks [device]   -> one JSON line on stdout
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

constexpr int kChains = 8;
constexpr int kIters = 4096;

__global__ void popc_loop(unsigned* out, unsigned seed) {
    unsigned a[kChains];
#pragma unroll
    for (int k = 0; k < kChains; ++k) a[k] = seed * (threadIdx.x + k * 7919u) + blockIdx.x;
    for (int it = 0; it < kIters; ++it) {
#pragma unroll
        for (int k = 0; k < kChains; ++k) a[k] = __popc(a[k]) + a[k];  // POPC + IADD
    }
    unsigned s = 0;
#pragma unroll
    for (int k = 0; k < kChains; ++k) s ^= a[k];
    if (s == 0x12345678u) out[0] = s;
}

__global__ void lop3_loop(unsigned* out, unsigned seed) {
    unsigned a[kChains];
#pragma unroll
    for (int k = 0; k < kChains; ++k) a[k] = seed * (threadIdx.x + k * 7919u) + blockIdx.x;
    const unsigned b = seed ^ 0x5bd1e995u, c = seed * 3u;
    for (int it = 0; it < kIters; ++it) {
#pragma unroll
        for (int k = 0; k < kChains; ++k)  // exactly one LOP3 per op (opaque to the optimiser)
            asm("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(a[k]) : "r"(b), "r"(c));
    }
    unsigned s = 0;
#pragma unroll
    for (int k = 0; k < kChains; ++k) s ^= a[k];
    if (s == 0x12345678u) out[0] = s;
}

template <typename K>
double run(K kernel, int sms, unsigned* d) {
    const int threads = 256, blocks = sms * 8;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    kernel<<<blocks, threads>>>(d, 3u);  // warm-up
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0);
        kernel<<<blocks, threads>>>(d, 3u + r);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    const double ops = double(blocks) * threads * kIters * kChains;
    return ops / (best * 1e-3);
}

int main(int argc, char** argv) {
    int dev = argc > 1 ? std::atoi(argv[1]) : 0;
    if (cudaSetDevice(dev) != cudaSuccess) {
        std::printf("{\"error\": \"no device\"}\n");
        return 1;
    }
    int sms = 0, clk_khz = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev);
    unsigned* d;
    cudaMalloc(&d, 64);
    const double popc = run(popc_loop, sms, d);
    const double lop3 = run(lop3_loop, sms, d);
    const double clk = clk_khz * 1e3;
    std::printf("{\"popc_ops_per_s\": %.6e, \"lop3_ops_per_s\": %.6e, \"sms\": %d, \"max_clock_hz\": %.6e, "
                "\"popc_per_clk_per_sm_at_max\": %.3f, \"lop3_per_clk_per_sm_at_max\": %.3f}\n",
                popc, lop3, sms, clk, popc / (sms * clk), lop3 / (sms * clk));
    cudaFree(d);
    return 0;
}
