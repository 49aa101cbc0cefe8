// Tensor-core Bitmap Filter, two row tiles per column tile (K2, tcgen05,
// single CTA).  Included by engine.cu after filter_tc.cuh.
//
// Same exact int8 GEMM and operand layout as filter_tc_kernel (K = b + 32 with
// the popcount extension, 16-byte size chunk per row), but a work item covers
// 256 rows (two 128-row tiles, A0 and A1) and every staged 256-column B tile
// feeds two M=128 x N=256 MMA chains, one per row tile, into their own TMEM
// accumulators (columns 0..255 and 256..511).  Per window pair this halves the
// bulk-copy writes into shared memory -- the single-CTA kernel's per-tile
// shared-memory traffic (A and B reads by the MMA, B writes by the copy engine,
// ~105 KB per 32K pairs) drops to ~82 KB -- and the epilogue drains row tile 0
// while the MMAs of row tile 1 run (each accumulator is single-buffered, the
// two alternate).
// Roles (576 threads): warp 0 producer, warp 1 MMA issuer, warps 2..17 epilogue.
#pragma once

#include "filter_tc.cuh"

namespace ssjb {
namespace dev {

template <int KA, int NS>
struct TcmLayout {
    static constexpr int kEpiWarps = 16;
    static constexpr int kThreads = 64 + 32 * kEpiWarps;
    static constexpr int NT = 256;
    static constexpr int kColsPerWarp = 64;
    static constexpr int kWords = (KA - 32) / 64;
    static constexpr int kRow = KA + 16;         // operand row: L1 (+extension) | size chunk
    static constexpr int kKCT = kRow / 16;
    static constexpr int kSbo = kKCT * 128;
    static constexpr int kA = 128 * kRow;        // one row tile
    static constexpr int kB = NT * kRow;         // one column tile
    static constexpr int kQueue = kEpiWarps * kTcQueue * 8;
    static constexpr int kBytes = 2 * 2 * kA + NS * kB + kQueue;  // A: 2 items x 2 row tiles
    static_assert(kBytes + 1024 + 4 * kTcLut + 512 <= 232448, "shared memory per CTA");
};

// Per-row state of one 128-row tile in the epilogue (lane = row).
struct TcmRow {
    uint32_t i, si, lo, hi, lo_max, hi_min, cnt, last_sz;
    int pc, cim1;
    bool valid, bypass;
};

// One 128x256 accumulator block of one row tile: survivors of this warp's 64
// columns (packed s16 fast path, or per-size-run thresholds at window edges).
template <int KCT>
__device__ __forceinline__ void tcm_block(TcmRow& R, uint32_t acc_col, const uint8_t* stage, int cw, uint32_t wbase,
                                          uint32_t szw0, uint32_t szw1, const int32_t* maxham, uint2* q, int& qlen,
                                          const TcParams& P, int lane) {
    const bool fast = szw0 == szw1 && wbase >= R.lo_max && wbase + 64 <= R.hi_min;
    if (fast) {
        if (szw0 != R.last_sz) {
            R.last_sz = szw0;
            R.cim1 = R.pc - maxham[R.si + szw0] - 1;
        }
        uint32_t d[32];
        tmem_ld64_pack16(acc_col + cw, d);
        const int c16 = max(R.cim1, -32768);
        if (__any_sync(0xFFFFFFFFu, R.bypass || any_above16(d, c16))) {
            uint32_t m0 = 0xFFFFFFFFu, m1 = 0xFFFFFFFFu;
            if (P.bias > 0) {  // non-negative accumulators: 3-instruction SWAR masks, permuted bits
                if (!R.bypass) masks16_nonneg(d, R.cim1, m0, m1);
                R.cnt += __popc(m0) + __popc(m1);
                tc_emit64<true>(m0, m1, wbase, R.i, q, qlen, P, lane);
                return;
            }
            if (!R.bypass) masks16(d, c16, m0, m1);
            R.cnt += __popc(m0) + __popc(m1);
            if (__any_sync(0xFFFFFFFFu, m0 != 0)) tc_emit(m0, wbase, R.i, q, qlen, P, lane);
            if (__any_sync(0xFFFFFFFFu, m1 != 0)) tc_emit(m1, wbase + 32, R.i, q, qlen, P, lane);
        }
        return;
    }
#pragma unroll 1
    for (int g = 0; g < 2; ++g) {
        const int cl = cw + g * 32;
        const uint32_t gbase = wbase + g * 32;
        const int kl = static_cast<int>(R.lo) - static_cast<int>(gbase);
        const int kh = static_cast<int>(R.hi) - static_cast<int>(gbase);
        const uint32_t rm = low_mask(kh) & ~low_mask(kl);
        if (!__any_sync(0xFFFFFFFFu, rm != 0)) continue;
        uint32_t d[16];
        tmem_ld32_pack16_nowait(acc_col + cl, d);
        const uint32_t colsz = stage_size<KCT>(stage, cl + lane);
        tmem_wait_ld();
        int cmin = INT_MAX;
        uint32_t rem = 0xFFFFFFFFu;
        while (rem) {
            const uint32_t sz = __shfl_sync(0xFFFFFFFFu, colsz, __ffs(rem) - 1);
            rem &= ~__ballot_sync(0xFFFFFFFFu, colsz == sz);
            cmin = min(cmin, R.pc - maxham[R.si + sz] - 1);
        }
        if (!__any_sync(0xFFFFFFFFu, R.bypass || (rm != 0 && any_above16_32(d, max(cmin, -32768))))) continue;
        uint32_t m = 0;
        rem = 0xFFFFFFFFu;
        while (rem) {  // all lanes: the shuffles need the full warp
            const uint32_t sz = __shfl_sync(0xFFFFFFFFu, colsz, __ffs(rem) - 1);
            const uint32_t sel = __ballot_sync(0xFFFFFFFFu, colsz == sz);
            rem &= ~sel;
            m |= mask16_32(d, max(R.pc - maxham[R.si + sz] - 1, -32768)) & sel;
        }
        if (R.bypass) m = 0xFFFFFFFFu;
        m &= rm;
        R.cnt += __popc(m);
        if (__any_sync(0xFFFFFFFFu, m != 0)) tc_emit(m, gbase, R.i, q, qlen, P, lane);
    }
}

template <int KA, int NS>
__global__ void __launch_bounds__((TcmLayout<KA, NS>::kThreads), 1) filter_tcm_kernel(TcParams P) {
    using L = TcmLayout<KA, NS>;
    constexpr int NT = L::NT;
    constexpr int kRows2 = 2 * kRowTile;
    constexpr int kEpi = L::kEpiWarps;
    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t* sA = smem;                          // [2 items][2 row tiles][kA]
    uint8_t* sB = smem + 4 * L::kA;              // [NS][kB]
    uint2* sQ = reinterpret_cast<uint2*>(sB + NS * L::kB);
    __shared__ __align__(8) uint64_t item_full[2], item_empty[2], a_full[2], a_empty[2];
    __shared__ __align__(8) uint64_t b_full[NS], b_empty[NS], acc_full[2], acc_empty[2];
    __shared__ TcItem items[2];
    __shared__ uint32_t tmem_base_sh;
    __shared__ int32_t s_maxham[kTcLut];

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tmem_base_sh)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    const bool lut_smem = P.maxham_len <= kTcLut;
    if (lut_smem)
        for (int k = threadIdx.x; k < P.maxham_len; k += blockDim.x) s_maxham[k] = P.maxham[k];
    const int32_t* maxham = lut_smem ? s_maxham : P.maxham;
    if (threadIdx.x == 0) {
        for (int s = 0; s < 2; ++s) {
            mbar_init(&item_full[s], 1);
            mbar_init(&item_empty[s], 1 + kEpi);
            mbar_init(&a_full[s], 1);
            mbar_init(&a_empty[s], 1);
            mbar_init(&acc_full[s], 1);
            mbar_init(&acc_empty[s], kEpi);
        }
        for (int s = 0; s < NS; ++s) {
            mbar_init(&b_full[s], 1);
            mbar_init(&b_empty[s], 1 + kEpi);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem_base = tmem_base_sh;

    if (warp == 0) {
        // ------------------------------------------------------------ producer
        if (lane == 0) {
            uint32_t iseq = 0, tseq = 0;
            unsigned long long nxt = claim_tc(P);
            uint32_t nxt_tile = nxt != kNoItem ? P.item_tile[nxt] : 0u;
            for (;;) {
                const int slot = iseq & 1;
                mbar_spin(&item_empty[slot], ((iseq >> 1) & 1) ^ 1);
                const unsigned long long it = nxt;
                TcItem info{};
                info.item = it;
                if (it == kNoItem) {
                    info.done = 1;
                    items[slot] = info;
                    mbar_arrive(&item_full[slot]);
                    break;
                }
                const uint32_t tile = nxt_tile;
                const uint32_t chunk = static_cast<uint32_t>(it - P.item_base[tile]);
                const uint32_t row0 = P.row_begin + tile * kRows2;
                const uint32_t rows_end = min(row0 + kRows2, P.row_end);
                info.tile = tile;
                info.c0 = P.tile_col_lo[tile] + chunk * kColChunk;
                info.c1 = min(info.c0 + kColChunk, rows_end - 1);
                info.ntiles = (info.c1 - info.c0 + NT - 1) / NT;
                items[slot] = info;
                // both row tiles (256 consecutive operand rows) in one copy
                const int aslot = iseq & 1;
                mbar_spin(&a_empty[aslot], ((iseq >> 1) & 1) ^ 1);
                mbar_expect_tx(&a_full[aslot], 2 * L::kA);
                tma_load_1d(sA + aslot * 2 * L::kA, P.opA + static_cast<uint64_t>(row0) * L::kRow, 2 * L::kA,
                            &a_full[aslot]);
                mbar_arrive(&item_full[slot]);
                nxt = claim_tc(P);
                nxt_tile = nxt != kNoItem ? P.item_tile[nxt] : 0u;
                for (uint32_t t = 0; t < info.ntiles; ++t, ++tseq) {
                    const int st = tseq % NS;
                    mbar_spin(&b_empty[st], ((tseq / NS) & 1) ^ 1);
                    const uint32_t col = info.c0 + t * NT;
                    if (SSJB_TRACE && P.trace && blockIdx.x == 0 && tseq < 512) P.trace[tseq * 4 + 0] = clock64();
                    mbar_expect_tx(&b_full[st], L::kB);
                    tma_load_1d(sB + st * L::kB, P.opB + static_cast<uint64_t>(col) * L::kRow, L::kB, &b_full[st]);
                }
                ++iseq;
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------------------ MMA issuer
        // (warp-uniform loop, one elected lane issues: see filter_tc_kernel)
        const bool leader = elect_one();
        {
            uint32_t iseq = 0, tseq = 0, useq = 0;  // useq: uses of each accumulator
            for (;;) {
                const int slot = iseq & 1;
                mbar_spin(&item_full[slot], (iseq >> 1) & 1);
                const TcItem info = items[slot];
                __syncwarp();
                if (leader) mbar_arrive(&item_empty[slot]);
                if (info.done) break;
                const int aslot = iseq & 1;
                mbar_spin(&a_full[aslot], (iseq >> 1) & 1);
                const uint32_t a0 = smem_u32(sA + aslot * 2 * L::kA);
                const uint64_t da0 = umma_desc(a0, L::kSbo), da1 = umma_desc(a0 + L::kA, L::kSbo);
                for (uint32_t t = 0; t < info.ntiles; ++t, ++tseq, ++useq) {
                    const int st = tseq % NS;
                    mbar_spin(&b_full[st], (tseq / NS) & 1);
                    if (SSJB_TRACE && P.trace && blockIdx.x == 0 && tseq < 512) P.trace[tseq * 4 + 1] = clock64();
                    const uint64_t db0 = umma_desc(smem_u32(sB + st * L::kB), L::kSbo);
#pragma unroll
                    for (int r = 0; r < 2; ++r) {
                        mbar_spin(&acc_empty[r], (useq & 1) ^ 1);
                        asm volatile("tcgen05.fence::after_thread_sync;");
                        if (leader) {
                            const uint64_t dar = r ? da1 : da0;
#pragma unroll
                            for (int s = 0; s < KA / 32; ++s)
                                umma_i8<NT>(tmem_base + r * NT, umma_desc_step(dar, s), umma_desc_step(db0, s), s > 0);
                            umma_commit(&acc_full[r]);
                        }
                        __syncwarp();
                    }
                    if (leader) umma_commit(&b_empty[st]);
                    __syncwarp();
                    if (SSJB_TRACE && P.trace && blockIdx.x == 0 && tseq < 512) P.trace[tseq * 4 + 2] = clock64();
                }
                if (leader) umma_commit(&a_empty[aslot]);
                __syncwarp();
                ++iseq;
            }
        }
    } else {
        // ------------------------------------------------------------ epilogue
        const int ew = warp - 2;
        const int quarter = warp & 3;
        const int part = ew >> 2;
        const int rit = quarter * 32 + lane;
        const uint32_t lane_base = static_cast<uint32_t>(quarter * 32) << 16;
        uint2* q = sQ + ew * kTcQueue;
        int qlen = 0;
        uint32_t iseq = 0, st_idx = 0, st_phase = 0, useq = 0;
        for (;;) {
            const int slot = iseq & 1;
            mbar_wait(&item_full[slot], (iseq >> 1) & 1);
            const TcItem info = warp_item(items[slot], lane);
            __syncwarp();
            if (lane == 0) mbar_arrive(&item_empty[slot]);
            if (info.done) break;
            TcmRow R[2];
#pragma unroll
            for (int r = 0; r < 2; ++r) {
                const uint32_t row0 = P.row_begin + info.tile * kRows2 + r * kRowTile;
                const uint32_t i = row0 + rit;
                R[r].i = i;
                R[r].valid = i < P.row_end && row0 < P.row_end;
                R[r].si = 0;
                R[r].pc = 0;
                R[r].bypass = false;
                uint32_t j0 = 0;
                if (R[r].valid) {
                    R[r].si = P.sizes[i];
                    j0 = P.wstart[R[r].si];
                    R[r].bypass = static_cast<int64_t>(R[r].si) > P.cutoff;
#pragma unroll
                    for (int w = 0; w < L::kWords; ++w)
                        R[r].pc += __popcll(P.bits[static_cast<uint64_t>(i) * L::kWords + w]);
                    R[r].pc += P.bias;  // thresholds shift with the biased accumulators
                }
                R[r].lo = R[r].valid ? max(j0, info.c0) : info.c1;
                R[r].hi = R[r].valid ? min(i, info.c1) : info.c1;
                uint32_t lo_max = R[r].lo, hi_min = R[r].hi;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    lo_max = max(lo_max, __shfl_xor_sync(0xFFFFFFFFu, lo_max, o));
                    hi_min = min(hi_min, __shfl_xor_sync(0xFFFFFFFFu, hi_min, o));
                }
                R[r].lo_max = lo_max;
                R[r].hi_min = hi_min;
                R[r].cnt = 0;
                R[r].last_sz = 0xFFFFFFFFu;
                R[r].cim1 = 0;
            }
            for (uint32_t t = 0; t < info.ntiles; ++t, ++useq) {
                mbar_wait_u32(smem_u32(&b_full[0]) + 8 * st_idx, st_phase);
                const uint8_t* stage = sB + st_idx * L::kB;
                const int cw = part * L::kColsPerWarp;
                const uint32_t wbase = info.c0 + t * NT + cw;
                const uint32_t szw0 = stage_size<L::kKCT>(stage, cw);
                const uint32_t szw1 = stage_size<L::kKCT>(stage, cw + L::kColsPerWarp - 1);
#pragma unroll
                for (int r = 0; r < 2; ++r) {
                    mbar_wait_u32(smem_u32(&acc_full[0]) + 8 * r, useq & 1);
                    asm volatile("tcgen05.fence::after_thread_sync;");
                    if (r == 0 && P.trace && blockIdx.x == 0 && lane == 0 && useq < 512)
                        P.trace[2048 + useq * 16 + ew] = clock64();
                    tcm_block<L::kKCT>(R[r], tmem_base + lane_base + r * NT, stage, cw, wbase, szw0, szw1, maxham, q,
                                       qlen, P, lane);
                    asm volatile("tcgen05.fence::before_thread_sync;");
                    __syncwarp();
                    if (lane == 0) mbar_arrive_u32(smem_u32(&acc_empty[0]) + 8 * r);
                }
                if (SSJB_TRACE && P.trace && blockIdx.x == 0 && lane == 0 && useq < 512)
                    P.trace[2048 + 8192 + useq * 16 + ew] = clock64();
                if (lane == 0) mbar_arrive_u32(smem_u32(&b_empty[0]) + 8 * st_idx);
                if (++st_idx == NS) {
                    st_idx = 0;
                    st_phase ^= 1u;
                }
            }
#pragma unroll
            for (int r = 0; r < 2; ++r) {
                if (R[r].valid && R[r].cnt) atomicAdd(P.rowcnt + (R[r].i - P.row_begin), R[r].cnt);
                if (P.item_counts && R[r].cnt)
                    atomicAdd(P.item_counts + info.item * kRows2 + r * kRowTile + rit, R[r].cnt);
            }
            ++iseq;
        }
        if (qlen) tc_flush(q, qlen, P, lane);
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem_base));
}

}  // namespace dev
}  // namespace ssjb
