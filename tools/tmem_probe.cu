// TMEM read-bandwidth probe (tcgen05.ld): one CTA per SM allocates 512 TMEM
// columns and WARPS warps stream them back with tcgen05.ld.32x32b.xN (+ wait)
// in a loop; optionally .pack::16b.  Prints bytes/clk/SM of accumulator data
// (32-bit cells) moved to registers.   usage: tmem_probe
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

template <int N, bool PACK>
__device__ __forceinline__ uint32_t ld_cols(uint32_t taddr) {
    uint32_t r[N];
    if constexpr (N == 32 && !PACK) {
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
            "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
            : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
              "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
              "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]),
              "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]),
              "=r"(r[30]), "=r"(r[31])
            : "r"(taddr));
    } else if constexpr (N == 16 && PACK) {
        // 32 columns of 16-bit data packed into 16 registers
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.pack::16b.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
            : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
              "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
            : "r"(taddr));
    } else if constexpr (N == 16 && !PACK) {
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
            : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
              "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
            : "r"(taddr));
    }
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    uint32_t x = 0;
#pragma unroll
    for (int k = 0; k < N; ++k) x ^= r[k];
    return x;
}

// COLS: TMEM columns covered per tcgen05.ld (32 for both x32 forms)
template <int N, bool PACK>
__global__ void tmem_read(int iters, unsigned* sink, long long* cycles) {
    __shared__ uint32_t tbase;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
            static_cast<uint32_t>(__cvta_generic_to_shared(&tbase))));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t base = tbase + (static_cast<uint32_t>((warp & 3) * 32) << 16);
    const int nw = blockDim.x >> 5;
    const int part = warp >> 2, parts = nw >> 2;
    constexpr int kCols = (N == 16 && !PACK) ? 16 : 32;
    uint32_t acc = 0;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        for (int c = part * kCols; c < 512; c += parts * kCols) acc ^= ld_cols<N, PACK>(base + c);
    }
    long long t1 = clock64();
    if (acc == 0x12345678u) sink[0] = acc;
    if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tbase));
}

// Semantics check of .pack::16b: column c holds 0x10000*c + c; lane 0 prints
// the 16 packed registers read at column 0.
__global__ void pack_check(unsigned* out) {
    __shared__ uint32_t tbase;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(
            static_cast<uint32_t>(__cvta_generic_to_shared(&tbase))));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (warp == 0) {
        uint32_t v[32];
#pragma unroll
        for (int c = 0; c < 32; ++c) v[c] = 0x10000u * c + c + 0x100u;
        asm volatile(
            "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
            "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(tbase),
            "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
            "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]),
            "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]),
            "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31]));
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        uint32_t r[16];
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.pack::16b.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
            : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
              "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
            : "r"(tbase));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if (lane == 0)
            for (int k = 0; k < 16; ++k) out[k] = r[k];
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tbase));
}

template <int N, bool PACK>
void run(const char* name, int warps, int sms) {
    unsigned* sink;
    long long* cyc;
    cudaMalloc(&sink, 4);
    cudaMalloc(&cyc, sms * 8);
    const int iters = 2000;
    tmem_read<N, PACK><<<sms, warps * 32>>>(10, sink, cyc);
    tmem_read<N, PACK><<<sms, warps * 32>>>(iters, sink, cyc);
    cudaDeviceSynchronize();
    long long c = 0;
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    // cells read per CTA: 128 lanes x 512 columns x 4 B per iteration
    const double bytes = 128.0 * 512 * 4 * iters;
    std::printf("%-22s warps=%2d  %.1f B/clk/SM (32-bit cells)  %.0f clk per 128x256 tile\n", name, warps,
                bytes / c, 128.0 * 256 * 4 / (bytes / c));
    cudaFree(sink);
    cudaFree(cyc);
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    unsigned* pc;
    cudaMalloc(&pc, 64);
    pack_check<<<1, 128>>>(pc);
    unsigned h[16];
    cudaMemcpy(h, pc, 64, cudaMemcpyDeviceToHost);
    std::printf("pack::16b regs:");
    for (int k = 0; k < 16; ++k) std::printf(" %08x", h[k]);
    std::printf("\n");
    for (int w : {4, 8, 16}) {
        run<32, false>("32x32b.x32", w, sms);
        run<16, false>("32x32b.x16", w, sms);
        run<16, true>("32x32b.x16.pack::16b", w, sms);
    }
    std::printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
