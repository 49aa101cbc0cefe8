// Probe of the tcgen05 int8 path used by the tensor-core filter: one CTA loads
// a 128 x K u8 A tile and a 128 x K s8 B tile (core-matrix / SWIZZLE_NONE
// K-major layout) with cp.async.bulk, issues K/32 tcgen05.mma kind::i8
// (M=128, N=128) into TMEM, reads the accumulator back with tcgen05.ld and
// compares with a host GEMM.   usage: tc_probe  -> "tc_probe ok" or mismatches
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

__device__ __forceinline__ uint64_t smem_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFF);
    d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFF) << 16;
    d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFF) << 32;
    d |= static_cast<uint64_t>(1) << 46;  // sm100 descriptor version
    return d;                             // base offset 0, SWIZZLE_NONE
}

__global__ void probe(const uint8_t* A, const int8_t* B, int K, int* out) {
    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t* sA = smem;
    uint8_t* sB = smem + 128 * K;
    __shared__ __align__(8) uint64_t bar_load, bar_mma;
    __shared__ uint32_t tmem_base;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == 0) {
        uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(&tmem_base));
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(a));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 0) {
        uint32_t b1 = static_cast<uint32_t>(__cvta_generic_to_shared(&bar_load));
        uint32_t b2 = static_cast<uint32_t>(__cvta_generic_to_shared(&bar_mma));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b1));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b2));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = tmem_base;
    const uint32_t bl = static_cast<uint32_t>(__cvta_generic_to_shared(&bar_load));
    const uint32_t bm = static_cast<uint32_t>(__cvta_generic_to_shared(&bar_mma));
    if (threadIdx.x == 0) {
        const uint32_t bytes = 128u * K;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bl), "r"(2 * bytes) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         static_cast<uint32_t>(__cvta_generic_to_shared(sA))),
                     "l"(A), "r"(bytes), "r"(bl)
                     : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         static_cast<uint32_t>(__cvta_generic_to_shared(sB))),
                     "l"(B), "r"(bytes), "r"(bl)
                     : "memory");
    }
    asm volatile(
        "{\n.reg .pred P1;\nW1:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n@!P1 bra W1;\n}\n" ::"r"(bl)
        : "memory");
    if (threadIdx.x == 0) {
        const uint32_t KC = K / 16;
        const uint32_t idesc = (2u << 4) | (0u << 7) | (1u << 10) | ((128u >> 3) << 17) | ((128u >> 4) << 24);
        const uint32_t a0 = static_cast<uint32_t>(__cvta_generic_to_shared(sA));
        const uint32_t b0 = static_cast<uint32_t>(__cvta_generic_to_shared(sB));
        for (int s = 0; s < K / 32; ++s) {
            uint64_t da = smem_desc(a0 + s * 256, 128, KC * 128);
            uint64_t db = smem_desc(b0 + s * 256, 128, KC * 128);
            uint32_t acc = s > 0;
            asm volatile(
                "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
                "l"(da), "l"(db), "r"(idesc), "r"(acc));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bm) : "memory");
    }
    asm volatile(
        "{\n.reg .pred P1;\nW2:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n@!P1 bra W2;\n}\n" ::"r"(bm)
        : "memory");
    asm volatile("tcgen05.fence::after_thread_sync;");
    for (int c = 0; c < 4; ++c) {
        uint32_t r[32];
        const uint32_t taddr = tmem + ((warp * 32) << 16) + c * 32;
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
            "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
            : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
              "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
              "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
              "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),
              "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
            : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;");
        for (int k = 0; k < 32; ++k) out[(warp * 32 + lane) * 128 + c * 32 + k] = static_cast<int>(r[k]);
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tmem));
}

// row-major [rows][K] -> core matrices [rows/8][K/16][8][16]
template <typename T>
std::vector<T> to_core(const std::vector<T>& rm, int rows, int K) {
    std::vector<T> cm(rm.size());
    const int KC = K / 16;
    for (int r = 0; r < rows; ++r)
        for (int k = 0; k < K; ++k)
            cm[(((r / 8) * KC + k / 16) * 8 + r % 8) * 16 + k % 16] = rm[r * K + k];
    return cm;
}

int main() {
    const int K = 160;
    std::vector<uint8_t> A(128 * K);
    std::vector<int8_t> B(128 * K);
    srand(7);
    for (auto& x : A) x = rand() % 2;
    for (auto& x : B) x = static_cast<int8_t>((rand() % 3) - 1) * 2;
    for (int r = 0; r < 128; ++r) B[r * K + 130] = -100;  // a large negative extension value
    auto Ac = to_core(A, 128, K);
    auto Bc = to_core(B, 128, K);
    uint8_t* dA;
    int8_t* dB;
    int* dO;
    cudaMalloc(&dA, Ac.size());
    cudaMalloc(&dB, Bc.size());
    cudaMalloc(&dO, 128 * 128 * 4);
    cudaMemcpy(dA, Ac.data(), Ac.size(), cudaMemcpyHostToDevice);
    cudaMemcpy(dB, Bc.data(), Bc.size(), cudaMemcpyHostToDevice);
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * 128 * K);
    probe<<<1, 128, 2 * 128 * K>>>(dA, dB, K, dO);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        std::printf("tc_probe CUDA error: %s\n", cudaGetErrorString(e));
        return 1;
    }
    std::vector<int> O(128 * 128);
    cudaMemcpy(O.data(), dO, O.size() * 4, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int m = 0; m < 128; ++m)
        for (int n = 0; n < 128; ++n) {
            int ref = 0;
            for (int k = 0; k < K; ++k) ref += A[m * K + k] * B[n * K + k];
            if (ref != O[m * 128 + n] && bad++ < 10) std::printf("mismatch m=%d n=%d got %d want %d\n", m, n, O[m * 128 + n], ref);
        }
    std::printf(bad ? "tc_probe FAILED (%d mismatches)\n" : "tc_probe ok\n", bad);
    return bad != 0;
}
