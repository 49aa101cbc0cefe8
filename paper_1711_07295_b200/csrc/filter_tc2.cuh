// Tensor-core Bitmap Filter on a CTA pair (K2, tcgen05 cta_group::2).
// Included by engine.cu after filter_tc.cuh (shares its encoding and helpers).
//
// Same exact int8 GEMM as filter_tc_kernel (A_i = [bits(b_i) | 1,1],
// B_j = [2 bits(b_j) | -ceil(pc_j/2), -floor(pc_j/2)], D = 2<b_i,b_j> - pc_j,
// survive iff D > pc_i - T - 1), but two SMs of a TPC run ONE M=256 x N=256
// MMA per K step:
//   * CTA rank r of the pair owns rows [row0 + 128 r, +128) of a 256-row
//     super tile (its own A tile) and columns [col + 128 r, +128) of each
//     256-column tile (half of B); the MMA reads the peer's half over the pair
//     link, so every B byte is staged into shared memory once for two SMs.
//     Per SM and tile this halves the bulk-copy ingress and the shared-memory
//     traffic of the single-CTA kernel, which ran into the SM's shared-memory
//     bandwidth (MMA operand reads + TMA writes ~116 B/clk of 128).
//   * Each CTA's TMEM holds the accumulators of its own 128 rows x 256 columns,
//     so the epilogue is the single-CTA one (own rows, all 256 columns; the
//     256 column sizes come with every stage as a separate 1 KB copy).
// Roles (576 threads per CTA): warp 0 lane 0 producer (both CTAs; the leader
// also claims work items and hands them to the peer through its shared memory),
// warp 1 lane 0 MMA issuer (leader) / readiness relay (peer), warps 2..17
// epilogue.  Barriers that collect arrivals from the peer live in the leader.
#pragma once

#include "filter_tc.cuh"

namespace ssjb {
namespace dev {

__device__ __forceinline__ uint32_t cluster_ctarank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}

// shared::cluster address of the same shared variable in CTA `rank`
__device__ __forceinline__ uint32_t mapa_u32(uint32_t saddr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
    return r;
}

__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}

// Relaxed remote arrive: pure progress signals that publish no memory the
// receiver reads through ordinary loads (the TMEM slot an epilogue warp has
// finished loading; a stage the peer's bulk copy has completed -- the data
// is complete in the peer's shared memory before its barrier flips).  A
// .release arrive would first drain the thread's outstanding memory traffic.
__device__ __forceinline__ void mbar_arrive_cluster_relaxed(uint32_t cluster_addr) {
    asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}

// wait with cluster-scope acquire (barriers that receive arrivals from the peer)
__device__ __forceinline__ void mbar_wait_cl(uint32_t a, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra WAIT_%=;\n"
        "}\n" ::"r"(a),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ void st_cluster_u32(uint32_t cluster_addr, uint32_t v) {
    asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(cluster_addr), "r"(v) : "memory");
}

__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// kind::i8, cta_group::2: D s32, A u8, B s8, K-major both, M = 256, N = 256
__device__ __forceinline__ void umma_i8_pair(uint32_t tmem, uint64_t da, uint64_t db, uint32_t acc) {
    constexpr uint32_t idesc = (2u << 4) | (0u << 7) | (1u << 10) | ((256u >> 3) << 17) | ((256u >> 4) << 24);
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
        "l"(da), "l"(db), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void umma_commit_pair(uint32_t bar) {
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            bar),
        "h"(static_cast<uint16_t>(3))
        : "memory");
}

template <int KA, int NS>
struct Tc2Layout {
    static constexpr int kEpiWarps = 16;
    static constexpr int kThreads = 64 + 32 * kEpiWarps;
    static constexpr int NT = 256;               // columns per MMA tile (both CTAs)
    static constexpr int kColsPerWarp = 64;      // 4 column parts x 4 TMEM lane quarters
    static constexpr int kKCT = KA / 16;         // 16-byte K chunks per operand row
    static constexpr int kSbo = kKCT * 128;      // stride between 8-row core groups
    static constexpr int kA = 128 * KA;          // one A tile (own 128 rows)
    static constexpr int kB = 128 * KA;          // one B half tile (own 128 columns)
    static constexpr int kSz = NT * 4;           // the tile's 256 column sizes
    static constexpr int kQueue = kEpiWarps * kTcQueue * 8;
    static constexpr int kBytes = 2 * kA + NS * kB + NS * kSz + kQueue;
    static constexpr uint32_t kTmemCols = 512;   // 2 accumulator slots x 256 columns
    static_assert(kBytes + 1024 + 4 * kTcLut + 1024 <= 232448, "shared memory per CTA");
};

template <int KA, int NS>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__((Tc2Layout<KA, NS>::kThreads), 1)
    filter_tc2_kernel(TcParams P) {
    using L = Tc2Layout<KA, NS>;
    constexpr int NT = L::NT;
    constexpr int kRows2 = 2 * kRowTile;  // rows per work item (super tile)
    constexpr int kTcEpiWarps2 = L::kEpiWarps;
    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t* sA = smem;
    uint8_t* sB = smem + 2 * L::kA;
    const uint32_t* sSz = reinterpret_cast<const uint32_t*>(sB + NS * L::kB);
    uint2* sQ = reinterpret_cast<uint2*>(sB + NS * L::kB + NS * L::kSz);
    __shared__ __align__(8) uint64_t item_full[2], item_empty[2], a_full[2], a_peer[2], a_empty[2];
    __shared__ __align__(8) uint64_t b_full[NS], b_peer[NS], b_empty[NS], acc_full[2], acc_empty[2];
    __shared__ __align__(16) TcItem items[2];
    __shared__ uint32_t tmem_base_sh;
    __shared__ int32_t s_maxham[kTcLut];

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = cluster_ctarank();
    const bool leader = rank == 0;

    const bool lut_smem = P.maxham_len <= kTcLut;
    if (lut_smem)
        for (int k = threadIdx.x; k < P.maxham_len; k += blockDim.x) s_maxham[k] = P.maxham[k];
    const int32_t* maxham = lut_smem ? s_maxham : P.maxham;
    if (threadIdx.x == 0) {
        for (int s = 0; s < 2; ++s) {
            mbar_init(&item_full[s], 1);
            // leader: its MMA + 16 epilogue warps, the peer's producer, relay, 16 epilogue warps
            mbar_init(&item_empty[s], 1 + kTcEpiWarps2 + 2 + kTcEpiWarps2);
            mbar_init(&a_full[s], 1);
            mbar_init(&a_peer[s], 1);
            mbar_init(&a_empty[s], 1);
            mbar_init(&acc_full[s], 1);
            mbar_init(&acc_empty[s], 2 * kTcEpiWarps2);
        }
        for (int s = 0; s < NS; ++s) {
            mbar_init(&b_full[s], 1);
            mbar_init(&b_peer[s], 1);
            mbar_init(&b_empty[s], 1 + kTcEpiWarps2);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base_sh)),
                     "r"(L::kTmemCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    cluster_sync_all();  // both CTAs' barriers initialised before any remote arrive
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem_base = tmem_base_sh;
    const uint32_t peer = rank ^ 1u;
    // leader-side barriers as seen from this CTA (local address in the leader)
    const uint32_t L_item_empty = mapa_u32(smem_u32(&item_empty[0]), 0);
    const uint32_t L_acc_empty = mapa_u32(smem_u32(&acc_empty[0]), 0);
    const uint32_t L_a_peer = mapa_u32(smem_u32(&a_peer[0]), 0);
    const uint32_t L_b_peer = mapa_u32(smem_u32(&b_peer[0]), 0);

    if (warp == 0) {
        // ------------------------------------------------------------ producer
        if (lane == 0) {
            uint32_t iseq = 0, tseq = 0;
            unsigned long long nxt = 0;
            uint32_t nxt_tile = 0;
            if (leader) {
                nxt = P.item_begin + atomicAdd(&P.ctl->work_next, 1ull);
                nxt_tile = nxt < P.item_end ? P.item_tile[nxt] : 0u;
            }
            const uint32_t R_items = mapa_u32(smem_u32(&items[0]), peer);
            const uint32_t R_item_full = mapa_u32(smem_u32(&item_full[0]), peer);
            for (;;) {
                const int slot = iseq & 1;
                TcItem info{};
                if (leader) {
                    mbar_spin(&item_empty[slot], ((iseq >> 1) & 1) ^ 1);
                    const unsigned long long it = nxt;
                    info.item = it;
                    if (it >= P.item_end) {
                        info.done = 1;
                    } else {
                        const uint32_t tile = nxt_tile;
                        const uint32_t chunk = static_cast<uint32_t>(it - P.item_base[tile]);
                        const uint32_t row0 = P.row_begin + tile * kRows2;
                        const uint32_t rows_end = min(row0 + kRows2, P.row_end);
                        info.tile = tile;
                        info.c0 = P.tile_col_lo[tile] + chunk * kColChunk;
                        info.c1 = min(info.c0 + kColChunk, rows_end - 1);
                        info.ntiles = (info.c1 - info.c0 + NT - 1) / NT;
                    }
                    items[slot] = info;
                    // hand the item to the peer: its copy, then a release arrive
                    const uint32_t* w = reinterpret_cast<const uint32_t*>(&info);
                    const uint32_t dst = R_items + slot * sizeof(TcItem);
#pragma unroll
                    for (int k = 0; k < static_cast<int>(sizeof(TcItem) / 4); ++k) st_cluster_u32(dst + 4 * k, w[k]);
                    mbar_arrive_cluster(R_item_full + 8 * slot);
                    mbar_arrive(&item_full[slot]);
                    if (!info.done) {
                        nxt = P.item_begin + atomicAdd(&P.ctl->work_next, 1ull);
                        nxt_tile = nxt < P.item_end ? P.item_tile[nxt] : 0u;
                    }
                } else {
                    mbar_wait_cl(smem_u32(&item_full[slot]), (iseq >> 1) & 1);
                    info = items[slot];
                    mbar_arrive_cluster(L_item_empty + 8 * slot);
                }
                if (info.done) break;
                const uint32_t row0 = P.row_begin + info.tile * kRows2 + rank * kRowTile;
                const int aslot = iseq & 1;
                mbar_spin(&a_empty[aslot], ((iseq >> 1) & 1) ^ 1);
                mbar_expect_tx(&a_full[aslot], L::kA);
                tma_load_1d(sA + aslot * L::kA, P.opA + static_cast<uint64_t>(row0) * KA, L::kA, &a_full[aslot]);
                for (uint32_t t = 0; t < info.ntiles; ++t, ++tseq) {
                    const int st = tseq % NS;
                    mbar_spin(&b_empty[st], ((tseq / NS) & 1) ^ 1);
                    if (SSJB_TRACE && P.trace && blockIdx.x == 0 && tseq < 512) P.trace[tseq * 4 + 0] = clock64();
                    const uint32_t col = info.c0 + t * NT;
                    mbar_expect_tx(&b_full[st], L::kB + L::kSz);
                    tma_load_1d(sB + st * L::kB, P.opB + static_cast<uint64_t>(col + rank * kRowTile) * KA, L::kB,
                                &b_full[st]);
                    tma_load_1d(const_cast<uint32_t*>(sSz) + st * NT, P.sizes + col, L::kSz, &b_full[st]);
                }
                ++iseq;
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            uint32_t iseq = 0, tseq = 0, aseq = 0;
            for (;;) {
                const int slot = iseq & 1;
                if (leader) mbar_spin(&item_full[slot], (iseq >> 1) & 1);
                else mbar_wait_cl(smem_u32(&item_full[slot]), (iseq >> 1) & 1);
                const TcItem info = items[slot];
                if (leader) mbar_arrive(&item_empty[slot]);
                else mbar_arrive_cluster(L_item_empty + 8 * slot);
                if (info.done) break;
                const int aslot = iseq & 1;
                if (!leader) {
                    // --------------------------------------------------- relay
                    // tell the leader's MMA issuer when this CTA's halves landed
                    mbar_spin(&a_full[aslot], (iseq >> 1) & 1);
                    mbar_arrive_cluster_relaxed(L_a_peer + 8 * aslot);
                    for (uint32_t t = 0; t < info.ntiles; ++t, ++tseq) {
                        const int st = tseq % NS;
                        mbar_spin(&b_full[st], (tseq / NS) & 1);
                        mbar_arrive_cluster_relaxed(L_b_peer + 8 * st);
                    }
                    ++iseq;
                    continue;
                }
                // ------------------------------------------------------- MMA issuer
                mbar_spin(&a_full[aslot], (iseq >> 1) & 1);
                mbar_wait_cl(smem_u32(&a_peer[aslot]), (iseq >> 1) & 1);
                const uint32_t a0 = smem_u32(sA + aslot * L::kA);
                for (uint32_t t = 0; t < info.ntiles; ++t, ++tseq, ++aseq) {
                    const int st = tseq % NS;
                    const int as = aseq & 1;
                    mbar_spin(&b_full[st], (tseq / NS) & 1);
                    mbar_wait_cl(smem_u32(&b_peer[st]), (tseq / NS) & 1);
                    if (SSJB_TRACE && P.trace && blockIdx.x == 0 && tseq < 512) P.trace[tseq * 4 + 1] = clock64();
                    mbar_wait_cl(smem_u32(&acc_empty[as]), ((aseq >> 1) & 1) ^ 1);
                    if (SSJB_TRACE && P.trace && blockIdx.x == 0 && tseq < 512) P.trace[tseq * 4 + 2] = clock64();
                    asm volatile("tcgen05.fence::after_thread_sync;");
                    const uint32_t b0 = smem_u32(sB + st * L::kB);
                    const uint32_t d1 = tmem_base + as * NT;
#pragma unroll
                    for (int s = 0; s < KA / 32; ++s)
                        umma_i8_pair(d1, umma_desc(a0 + s * 256, L::kSbo), umma_desc(b0 + s * 256, L::kSbo), s > 0);
                    umma_commit_pair(smem_u32(&b_empty[st]));
                    umma_commit_pair(smem_u32(&acc_full[as]));
                }
                umma_commit_pair(smem_u32(&a_empty[aslot]));
                ++iseq;
            }
        }
    } else {
        // ------------------------------------------------------------ epilogue
        const int ew = warp - 2;
        const int quarter = warp & 3;          // TMEM lanes 32*quarter .. +31 (hardware rule)
        const int part = ew >> 2;              // this warp's 64-column range of each tile
        const int rit = quarter * 32 + lane;   // row in this CTA's 128-row tile
        const uint32_t lane_base = static_cast<uint32_t>(quarter * 32) << 16;
        uint2* q = sQ + ew * kTcQueue;
        int qlen = 0;
        uint32_t iseq = 0, st_idx = 0, st_phase = 0, acc_idx = 0, acc_phase = 0, tile_seq = 0;
        for (;;) {
            const int slot = iseq & 1;
            mbar_wait_cl(smem_u32(&item_full[slot]), (iseq >> 1) & 1);
            const TcItem info = items[slot];
            __syncwarp();
            if (lane == 0) {
                if (leader) mbar_arrive(&item_empty[slot]);
                else mbar_arrive_cluster(L_item_empty + 8 * slot);
            }
            if (info.done) break;
            const uint32_t row0 = P.row_begin + info.tile * kRows2 + rank * kRowTile;
            const uint32_t rows_end = min(row0 + kRowTile, P.row_end);
            const uint32_t i = row0 + rit;
            const bool valid = i < rows_end;
            uint32_t si = 0, j0 = 0;
            int pc = 0;
            bool bypass = false;
            if (valid) {
                si = P.sizes[i];
                j0 = P.wstart[si];
                bypass = static_cast<int64_t>(si) > P.cutoff;
                constexpr int kW = (KA - 32) / 64;
#pragma unroll
                for (int w = 0; w < kW; ++w) pc += __popcll(P.bits[static_cast<uint64_t>(i) * kW + w]);
            }
            const uint32_t lo_i = valid ? max(j0, info.c0) : info.c1;
            const uint32_t hi_i = valid ? min(i, info.c1) : info.c1;
            uint32_t lo_max = lo_i, hi_min = hi_i;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                lo_max = max(lo_max, __shfl_xor_sync(0xFFFFFFFFu, lo_max, o));
                hi_min = min(hi_min, __shfl_xor_sync(0xFFFFFFFFu, hi_min, o));
            }
            uint32_t cnt = 0;
            uint32_t last_sz = 0xFFFFFFFFu;
            int cim1 = 0;
            for (uint32_t t = 0; t < info.ntiles; ++t) {
                mbar_wait_u32(smem_u32(&b_full[0]) + 8 * st_idx, st_phase);
                mbar_wait_u32(smem_u32(&acc_full[0]) + 8 * acc_idx, acc_phase);
                asm volatile("tcgen05.fence::after_thread_sync;");
                if (SSJB_TRACE && P.trace && blockIdx.x == 0 && lane == 0 && tile_seq < 512)
                    P.trace[2048 + tile_seq * 16 + (warp - 2)] = clock64();
                const uint32_t* szs = sSz + st_idx * NT;
                const int cw = part * L::kColsPerWarp;
                const uint32_t wbase = info.c0 + t * NT + cw;
                const uint32_t szw0 = szs[cw], szw1 = szs[cw + L::kColsPerWarp - 1];
                const bool fast = szw0 == szw1 && wbase >= lo_max && wbase + L::kColsPerWarp <= hi_min;
                if (fast && szw0 != last_sz) {
                    last_sz = szw0;
                    cim1 = pc - maxham[si + szw0] - 1;
                }
                const uint32_t acc_col = tmem_base + lane_base + acc_idx * NT;
                if (fast) {
                    // interior: the warp's 64 columns in one packed load
                    uint32_t d[32];
                    tmem_ld64_pack16(acc_col + cw, d);
                    const int c16 = max(cim1, -32768);
                    if (__any_sync(0xFFFFFFFFu, bypass || any_above16(d, c16))) {
                        uint32_t m0 = 0xFFFFFFFFu, m1 = 0xFFFFFFFFu;
                        if (!bypass) masks16(d, c16, m0, m1);
                        cnt += __popc(m0) + __popc(m1);
                        if (__any_sync(0xFFFFFFFFu, m0 != 0)) tc_emit(m0, wbase, i, q, qlen, P, lane);
                        if (__any_sync(0xFFFFFFFFu, m1 != 0)) tc_emit(m1, wbase + 32, i, q, qlen, P, lane);
                    }
                } else {
#pragma unroll 1
                    for (int g = 0; g < 2; ++g) {
                        const int cl = cw + g * 32;
                        const uint32_t gbase = wbase + g * 32;
                        const int kl = static_cast<int>(lo_i) - static_cast<int>(gbase);
                        const int kh = static_cast<int>(hi_i) - static_cast<int>(gbase);
                        const uint32_t rm = low_mask(kh) & ~low_mask(kl);
                        if (!__any_sync(0xFFFFFFFFu, rm != 0)) continue;
                        uint32_t d[16];
                        tmem_ld32_pack16_nowait(acc_col + cl, d);
                        const uint32_t colsz = szs[cl + lane];
                        tmem_wait_ld();
                        int cmin = INT_MAX;
                        uint32_t rem = 0xFFFFFFFFu;
                        while (rem) {
                            const uint32_t sz = __shfl_sync(0xFFFFFFFFu, colsz, __ffs(rem) - 1);
                            rem &= ~__ballot_sync(0xFFFFFFFFu, colsz == sz);
                            cmin = min(cmin, pc - maxham[si + sz] - 1);
                        }
                        if (!__any_sync(0xFFFFFFFFu, bypass || (rm != 0 && any_above16_32(d, max(cmin, -32768)))))
                            continue;
                        // (all lanes run the run loop: its shuffles need the full warp)
                        uint32_t m = 0;
                        rem = 0xFFFFFFFFu;
                        while (rem) {
                            const uint32_t sz = __shfl_sync(0xFFFFFFFFu, colsz, __ffs(rem) - 1);
                            const uint32_t sel = __ballot_sync(0xFFFFFFFFu, colsz == sz);
                            rem &= ~sel;
                            m |= mask16_32(d, max(pc - maxham[si + sz] - 1, -32768)) & sel;
                        }
                        if (bypass) m = 0xFFFFFFFFu;
                        m &= rm;
                        cnt += __popc(m);
                        if (__any_sync(0xFFFFFFFFu, m != 0)) tc_emit(m, gbase, i, q, qlen, P, lane);
                    }
                }
                asm volatile("tcgen05.fence::before_thread_sync;");
                __syncwarp();
                if (lane == 0) {
                    if (SSJB_TRACE && P.trace && blockIdx.x == 0 && tile_seq < 512)
                        P.trace[2048 + 8192 + tile_seq * 16 + (warp - 2)] = clock64();
                    if (leader) mbar_arrive(&acc_empty[acc_idx]);
                    else mbar_arrive_cluster_relaxed(L_acc_empty + 8 * acc_idx);
                    mbar_arrive(&b_empty[st_idx]);
                }
                if (++st_idx == NS) {
                    st_idx = 0;
                    st_phase ^= 1u;
                }
                if (++acc_idx == 2) {
                    acc_idx = 0;
                    acc_phase ^= 1u;
                }
                ++tile_seq;
            }
            if (valid && cnt) atomicAdd(P.rowcnt + (i - P.row_begin), cnt);
            if (P.item_counts && cnt) atomicAdd(P.item_counts + info.item * kRows2 + rank * kRowTile + rit, cnt);
            ++iseq;
        }
        if (qlen) tc_flush(q, qlen, P, lane);
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    cluster_sync_all();  // the peer may still be arriving on this CTA's barriers / reading TMEM
    if (warp == 1)
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(L::kTmemCols));
}

}  // namespace dev
}  // namespace ssjb
