// Probe of tcgen05.mma kind::mxf4 (packed e2m1, block-32 ue8m0 scales = 1.0):
// nibble order, scale-factor TMEM setup and instruction descriptor, checked
// against a host GEMM; then a throughput loop.   usage: tc_probe_fp4
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

constexpr int M = 128, N = 192;

__device__ __forceinline__ uint64_t smem_desc(uint32_t saddr, uint32_t sbo) {
    uint64_t d = static_cast<uint64_t>((saddr >> 4) & 0x3FFF);
    d |= static_cast<uint64_t>(128 >> 4) << 16;
    d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFF) << 32;
    d |= static_cast<uint64_t>(1) << 46;
    return d;
}

// block-scaled idesc: a/b format E2M1 (MXF4Format = 1), scale E8M0 (bit 23), M, N, K64
constexpr uint32_t kIdesc = (1u << 7) | (1u << 10) | ((N >> 3) << 17) | (1u << 23) | ((M >> 4) << 24);

__device__ __forceinline__ void sts_sf(uint32_t taddr) {
    const uint32_t v = 0x7F7F7F7Fu;
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,"
        "%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(taddr),
        "r"(v));
}

template <bool kLoop>
__global__ void probe(const uint8_t* A, const uint8_t* B, int Kbytes, float* out, int iters) {
    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t* sA = smem;
    uint8_t* sB = smem + M * Kbytes;
    __shared__ __align__(8) uint64_t bar_load, bar_mma;
    __shared__ uint32_t tmem_base;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
            static_cast<uint32_t>(__cvta_generic_to_shared(&tmem_base))));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(&bar_load))));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(&bar_mma))));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = tmem_base;
    const uint32_t sfa = tmem + 384, sfb = tmem + 448;  // 32 + 64 columns of scale factors (all 1.0)
    sts_sf(tmem + ((warp * 32) << 16) + 384);
    sts_sf(tmem + ((warp * 32) << 16) + 448);
    sts_sf(tmem + ((warp * 32) << 16) + 480);
    asm volatile("tcgen05.wait::st.sync.aligned;");
    const uint32_t bl = static_cast<uint32_t>(__cvta_generic_to_shared(&bar_load));
    const uint32_t bm = static_cast<uint32_t>(__cvta_generic_to_shared(&bar_mma));
    if (threadIdx.x == 0) {
        const uint32_t ba = M * Kbytes, bb = N * Kbytes;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bl), "r"(ba + bb) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         static_cast<uint32_t>(__cvta_generic_to_shared(sA))), "l"(A), "r"(ba), "r"(bl) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         static_cast<uint32_t>(__cvta_generic_to_shared(sB))), "l"(B), "r"(bb), "r"(bl) : "memory");
    }
    asm volatile("{\n.reg .pred P1;\nW1:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n@!P1 bra W1;\n}\n" ::"r"(bl) : "memory");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (threadIdx.x == 0) {
        const uint32_t KC = Kbytes / 16;
        const uint32_t a0 = static_cast<uint32_t>(__cvta_generic_to_shared(sA));
        const uint32_t b0 = static_cast<uint32_t>(__cvta_generic_to_shared(sB));
        for (int rep = 0; rep < (kLoop ? iters : 1); ++rep)
            for (int s = 0; s < Kbytes / 32; ++s) {
                uint64_t da = smem_desc(a0 + s * 256, KC * 128);
                uint64_t db = smem_desc(b0 + s * 256, KC * 128);
                uint32_t acc = s > 0;
                asm volatile(
                    "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                    "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%6], p;\n}\n" ::"r"(tmem),
                    "l"(da), "l"(db), "r"(kIdesc), "r"(acc), "r"(sfa), "r"(sfb));
            }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bm) : "memory");
    }
    asm volatile("{\n.reg .pred P1;\nW2:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n@!P1 bra W2;\n}\n" ::"r"(bm) : "memory");
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (!kLoop) {
        for (int c = 0; c < N / 32; ++c) {
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
            for (int k = 0; k < 32; ++k) out[(warp * 32 + lane) * N + c * 32 + k] = __uint_as_float(r[k]);
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

static const float kE2M1[16] = {0, 0.5f, 1, 1.5f, 2, 3, 4, 6, -0.f, -0.5f, -1, -1.5f, -2, -3, -4, -6};

// element-major [rows][K] nibbles -> packed core matrices [rows/8][Kbytes/16][8][16]
std::vector<uint8_t> to_core4(const std::vector<uint8_t>& nib, int rows, int K, bool low_first) {
    const int Kb = K / 2, KC = Kb / 16;
    std::vector<uint8_t> cm(static_cast<size_t>(rows) * Kb, 0);
    for (int r = 0; r < rows; ++r)
        for (int k = 0; k < K; ++k) {
            const int byte = k / 2;
            const size_t off = ((static_cast<size_t>(r / 8) * KC + byte / 16) * 8 + r % 8) * 16 + byte % 16;
            const int shift = ((k & 1) ^ (low_first ? 0 : 1)) * 4;
            cm[off] |= static_cast<uint8_t>(nib[static_cast<size_t>(r) * K + k] << shift);
        }
    return cm;
}

int main() {
    const int K = 192, Kbytes = K / 2;  // b = 128 + 64 extension
    std::vector<uint8_t> A(M * K), B(N * K);
    srand(11);
    for (auto& x : A) x = rand() % 2 ? 0x2 : 0x0;                    // {0, 1.0}
    const uint8_t bvals[6] = {0x0, 0x4, 0xF, 0xE, 0xD, 0xA};          // {0, 2, -6, -4, -3, -1}
    for (auto& x : B) x = bvals[rand() % 6];
    uint8_t *dA, *dB;
    float* dO;
    cudaMalloc(&dA, M * Kbytes);
    cudaMalloc(&dB, N * Kbytes);
    cudaMalloc(&dO, M * N * 4);
    const int smem = (M + N) * Kbytes;
    cudaFuncSetAttribute(probe<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(probe<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    int good_order = -1;
    for (int low_first = 1; low_first >= 0; --low_first) {
        auto Ac = to_core4(A, M, K, low_first), Bc = to_core4(B, N, K, low_first);
        cudaMemcpy(dA, Ac.data(), Ac.size(), cudaMemcpyHostToDevice);
        cudaMemcpy(dB, Bc.data(), Bc.size(), cudaMemcpyHostToDevice);
        probe<false><<<1, 128, smem>>>(dA, dB, Kbytes, dO, 1);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) {
            std::printf("tc_probe_fp4 CUDA error: %s\n", cudaGetErrorString(e));
            return 1;
        }
        std::vector<float> O(M * N);
        cudaMemcpy(O.data(), dO, O.size() * 4, cudaMemcpyDeviceToHost);
        int bad = 0;
        for (int m = 0; m < M; ++m)
            for (int n = 0; n < N; ++n) {
                float ref = 0;
                for (int k = 0; k < K; ++k) ref += kE2M1[A[m * K + k]] * kE2M1[B[n * K + k]];
                if (ref != O[m * N + n] && bad++ < 3)
                    std::printf("low_first=%d mismatch m=%d n=%d got %g want %g\n", low_first, m, n, O[m * N + n], ref);
            }
        std::printf("low_first=%d: %d mismatches\n", low_first, bad);
        if (!bad) good_order = low_first;
    }
    // throughput: 1 CTA per SM, back-to-back MMAs on resident tiles
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int iters = 4096;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    probe<true><<<sms, 128, smem>>>(dA, dB, Kbytes, dO, 16);
    cudaEventRecord(e0);
    probe<true><<<sms, 128, smem>>>(dA, dB, Kbytes, dO, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double flops = double(sms) * iters * (Kbytes / 32) * 2.0 * M * N * 64;
    std::printf("{\"tc_probe_fp4\": \"%s\", \"low_nibble_first\": %d, \"fp4_dense_tflops\": %.1f}\n",
                good_order >= 0 ? "ok" : "FAILED", good_order, flops / (ms * 1e-3) / 1e12);
    return good_order >= 0 ? 0 : 1;
}
