// cp.async.bulk (1-D TMA) throughput probe: one CTA per SM streams an
// L2-resident buffer into a shared-memory ring of `depth` slots of `bytes`
// each, refilling a slot as soon as its previous copy landed.
//   usage: bulk_probe  -> one line per (bytes, depth): TB/s chip-wide, B/clk/SM
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__global__ void stream(const uint8_t* src, size_t src_bytes, int bytes, int depth, int rounds, unsigned* sink) {
    extern __shared__ __align__(128) uint8_t ring[];
    __shared__ __align__(8) uint64_t bar[16];
    if (threadIdx.x == 0) {
        for (int s = 0; s < depth; ++s)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(&bar[s]))));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x != 0) return;
    uint32_t phase = 0;
    size_t off = (static_cast<size_t>(blockIdx.x) * 7919 * bytes) % (src_bytes - bytes);
    for (int r = 0; r < rounds; ++r) {
        for (int s = 0; s < depth; ++s) {
            const uint32_t b = static_cast<uint32_t>(__cvta_generic_to_shared(&bar[s]));
            if (r > 0) {
                const uint32_t par = (phase >> s) & 1u;
                asm volatile("{\n.reg .pred P1;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W;\n}\n"
                             ::"r"(b), "r"(par) : "memory");
                phase ^= 1u << s;
            }
            off = (off + 65536 + bytes) % (src_bytes - bytes);
            off &= ~size_t(127);
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes) : "memory");
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                             static_cast<uint32_t>(__cvta_generic_to_shared(ring + static_cast<size_t>(s) * bytes))),
                         "l"(src + off), "r"(bytes), "r"(b) : "memory");
        }
    }
    for (int s = 0; s < depth; ++s) {
        const uint32_t b = static_cast<uint32_t>(__cvta_generic_to_shared(&bar[s]));
        const uint32_t par = (phase >> s) & 1u;
        asm volatile("{\n.reg .pred P1;\nW2:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W2;\n}\n"
                     ::"r"(b), "r"(par) : "memory");
    }
    if (ring[0] == 0xAB && sink) sink[0] = 1;
}

int main() {
    int sms = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const size_t src_bytes = 32u << 20;  // L2 resident
    uint8_t* src;
    cudaMalloc(&src, src_bytes);
    cudaMemset(src, 1, src_bytes);
    cudaFuncSetAttribute(stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    const int sizes[] = {4096, 12288, 20480, 40960};
    const int depths[] = {1, 2, 4, 8, 12};
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int bytes : sizes)
        for (int depth : depths) {
            if (static_cast<size_t>(bytes) * depth > 200 * 1024) continue;
            const int rounds = static_cast<int>((64ll << 20) / (static_cast<long long>(bytes) * depth)) + 1;
            stream<<<sms, 32, bytes * depth>>>(src, src_bytes, bytes, depth, 4, nullptr);
            cudaEventRecord(e0);
            stream<<<sms, 32, bytes * depth>>>(src, src_bytes, bytes, depth, rounds, nullptr);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            const double total = double(sms) * rounds * depth * bytes;
            const double bps = total / (ms * 1e-3);
            std::printf("bytes=%6d depth=%2d  %.2f TB/s  %.1f B/clk/SM  %.0f cycles/copy\n", bytes, depth, bps / 1e12,
                        bps / sms / (clk * 1e3), (ms * 1e-3) * clk * 1e3 / (double(rounds) * depth));
        }
    std::printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
