// Integer-pipe microbenchmark for the filter kernel's roofline: full-chip
// throughput of 32-bit POPC and of LOP3 on sm_100a, measured with CUDA events.
// Built by __graft_entry__.build() into paper_1711_07295_b200/lib/pipe_peaks;
// bench.py runs it on the GPU box and uses the POPC figure as the peak of the
// K2 filter (which issues b/32 POPC per pair comparison).
//   usage: pipe_peaks [device]   -> one JSON line on stdout
#include <cuda_runtime.h>

#include <cstdint>
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


// ---- tcgen05 kind::i8 throughput: back-to-back M=128 x N=256 x K=32 MMAs
// from shared memory into TMEM, one CTA per SM (the filter kernel's shape).
__device__ __forceinline__ uint64_t pk_desc(uint32_t saddr, uint32_t sbo) {
    uint64_t d = static_cast<uint64_t>((saddr >> 4) & 0x3FFF);
    d |= static_cast<uint64_t>(128 >> 4) << 16;
    d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFF) << 32;
    d |= static_cast<uint64_t>(1) << 46;
    return d;
}

constexpr int kTcIters = 2048;  // groups of 8 MMAs

__global__ void __launch_bounds__(128, 1) tc_i8_loop(unsigned* out, uint32_t sbo, uint32_t lbo, uint32_t bofs) {
    extern __shared__ __align__(1024) uint8_t sm[];  // A and B tiles (zeros are fine)
    __shared__ __align__(8) uint64_t bar[2];
    __shared__ uint32_t tbase;
    const int warp = threadIdx.x >> 5;
    for (int k = threadIdx.x; k < 200 * 1024 / 4; k += blockDim.x) reinterpret_cast<uint32_t*>(sm)[k] = 0;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(
            static_cast<uint32_t>(__cvta_generic_to_shared(&tbase))));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 0) {
        for (int b = 0; b < 2; ++b)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(&bar[b]))));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (threadIdx.x == 0) {
        const uint32_t a0 = static_cast<uint32_t>(__cvta_generic_to_shared(sm));
        const uint32_t b0 = a0 + bofs;
        const uint32_t idesc = (2u << 4) | (0u << 7) | (1u << 10) | ((256u >> 3) << 17) | ((128u >> 4) << 24);
        uint64_t da = pk_desc(a0, sbo), db = pk_desc(b0, sbo);
        da = (da & ~(uint64_t(0x3FFF) << 16)) | (uint64_t((lbo >> 4) & 0x3FFF) << 16);
        db = (db & ~(uint64_t(0x3FFF) << 16)) | (uint64_t((lbo >> 4) & 0x3FFF) << 16);
        uint32_t phase[2] = {0, 0};
        for (int it = 0; it < kTcIters; ++it) {
            const int b = it & 1;
            if (it >= 2) {  // keep two groups in flight
                const uint32_t ba = static_cast<uint32_t>(__cvta_generic_to_shared(&bar[b]));
                asm volatile("{\n.reg .pred P1;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W;\n}\n"
                             ::"r"(ba), "r"(phase[b]) : "memory");
                phase[b] ^= 1;
            }
            for (int k = 0; k < 8; ++k)
                asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n"
                             ::"r"(tbase + b * 256), "l"(da), "l"(db), "r"(idesc), "r"(k));
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                static_cast<uint32_t>(__cvta_generic_to_shared(&bar[b]))) : "memory");
        }
        for (int b = 0; b < 2; ++b) {
            const uint32_t ba = static_cast<uint32_t>(__cvta_generic_to_shared(&bar[b]));
            asm volatile("{\n.reg .pred P1;\nW2:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W2;\n}\n"
                         ::"r"(ba), "r"(phase[b]) : "memory");
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tbase));
    if (threadIdx.x == 0 && out == nullptr) out[0] = 1;
}

double run_tc(int sms, uint32_t sbo = 256, uint32_t lbo = 128, uint32_t bofs = 128 * 32) {
    const int smem = 200 * 1024;
    cudaFuncSetAttribute(tc_i8_loop, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    unsigned* d;
    cudaMalloc(&d, 64);
    tc_i8_loop<<<sms, 128, smem>>>(d, sbo, lbo, bofs);
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0);
        tc_i8_loop<<<sms, 128, smem>>>(d, sbo, lbo, bofs);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    cudaFree(d);
    const double ops = double(sms) * kTcIters * 8 * 128.0 * 256.0 * 32.0 * 2.0;
    return ops / (best * 1e-3);
}

// ---- tcgen05 kind::mxf4 (block32 ue8m0 scales) throughput: back-to-back
// M=128 x N=256 x K=64 MMAs into one TMEM accumulator (the head-overlap
// kernel's instruction), unit scales in the TMEM columns after it.
__global__ void __launch_bounds__(128, 1) tc_f4_loop(unsigned* out, uint32_t sbo, uint32_t bofs) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ __align__(8) uint64_t bar[2];
    __shared__ uint32_t tbase;
    const int warp = threadIdx.x >> 5;
    for (int k = threadIdx.x; k < 200 * 1024 / 4; k += blockDim.x) reinterpret_cast<uint32_t*>(sm)[k] = 0;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
            static_cast<uint32_t>(__cvta_generic_to_shared(&tbase))));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 0) {
        for (int b = 0; b < 2; ++b)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(&bar[b]))));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    {  // unit scales (ue8m0 127) in columns 256..383 of every lane
        const uint32_t lanes = static_cast<uint32_t>(warp * 32) << 16;
        for (int c = 256; c < 384; c += 32) {
            const uint32_t v = 0x7F7F7F7Fu;
            asm volatile(
                "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,"
                "%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(tbase + lanes + c), "r"(v));
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (threadIdx.x == 0) {
        const uint32_t a0 = static_cast<uint32_t>(__cvta_generic_to_shared(sm));
        const uint32_t idesc = (1u << 7) | (1u << 10) | ((256u >> 3) << 17) | (1u << 23) | ((128u >> 4) << 24);
        const uint64_t da = pk_desc(a0, sbo), db = pk_desc(a0 + bofs, sbo);
        uint32_t phase[2] = {0, 0};
        for (int it = 0; it < kTcIters; ++it) {
            const int b = it & 1;
            if (it >= 2) {
                const uint32_t ba = static_cast<uint32_t>(__cvta_generic_to_shared(&bar[b]));
                asm volatile("{\n.reg .pred P1;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W;\n}\n"
                             ::"r"(ba), "r"(phase[b]) : "memory");
                phase[b] ^= 1;
            }
            for (int k = 0; k < 8; ++k)
                asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                             "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%6], p;\n}\n"
                             ::"r"(tbase), "l"(da), "l"(db), "r"(idesc), "r"(k), "r"(tbase + 256), "r"(tbase + 288));
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                static_cast<uint32_t>(__cvta_generic_to_shared(&bar[b]))) : "memory");
        }
        for (int b = 0; b < 2; ++b) {
            const uint32_t ba = static_cast<uint32_t>(__cvta_generic_to_shared(&bar[b]));
            asm volatile("{\n.reg .pred P1;\nW2:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W2;\n}\n"
                         ::"r"(ba), "r"(phase[b]) : "memory");
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tbase));
    if (threadIdx.x == 0 && out == nullptr) out[0] = 1;
}

double run_tc_f4(int sms) {
    const int smem = 200 * 1024;
    cudaFuncSetAttribute(tc_f4_loop, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    unsigned* d;
    cudaMalloc(&d, 64);
    tc_f4_loop<<<sms, 128, smem>>>(d, 256, 128 * 32);
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0);
        tc_f4_loop<<<sms, 128, smem>>>(d, 256, 128 * 32);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    cudaFree(d);
    const double ops = double(sms) * kTcIters * 8 * 128.0 * 256.0 * 64.0 * 2.0;
    return ops / (best * 1e-3);
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
    const double tci8 = run_tc(sms);
    const double tcf4 = run_tc_f4(sms);
    if (argc > 2) {  // layout sweep: SBO / LBO effect on tcgen05 operand reads
        const uint32_t sbos[] = {256, 640, 1408, 1536, 2048, 2816};
        for (uint32_t sb : sbos)
            std::printf("sbo=%u lbo=128: %.0f TOPS\n", sb, run_tc(sms, sb, 128, 16 * sb) / 1e12);
        std::printf("sbo=128 lbo=2048 (chunk-major): %.0f TOPS\n", run_tc(sms, 128, 2048, 65536) / 1e12);
        std::printf("sbo=128 lbo=4096 (chunk-major): %.0f TOPS\n", run_tc(sms, 128, 4096, 65536) / 1e12);
    }
    cudaError_t err = cudaGetLastError();
    const double clk = clk_khz * 1e3;
    std::printf("{\"popc_ops_per_s\": %.6e, \"lop3_ops_per_s\": %.6e, \"tc_i8_ops_per_s\": %.6e, \"sms\": %d, "
                "\"max_clock_hz\": %.6e, \"popc_per_clk_per_sm_at_max\": %.3f, \"lop3_per_clk_per_sm_at_max\": %.3f, "
                "\"tc_i8_ops_per_clk_per_sm_at_max\": %.1f, \"tc_f4_ops_per_s\": %.6e, \"error\": \"%s\"}\n",
                popc, lop3, tci8, sms, clk, popc / (sms * clk), lop3 / (sms * clk), tci8 / (sms * clk), tcf4,
                err == cudaSuccess ? "" : cudaGetErrorString(err));
    cudaFree(d);
    return 0;
}
