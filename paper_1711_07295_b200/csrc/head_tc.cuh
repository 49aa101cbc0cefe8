// K3a: exact head-token overlaps on the tensor cores, for the dense region
// of large records.  Included by engine.cu.
//
// Why.  For records of several hundred tokens and more, every b-bit Xor
// sketch saturates: at tau = 0.7 the allowed Hamming distance of a pair with
// |r|+|s| = 1000 is ~180 bits, more than a 256-bit sketch of two unrelated
// records differs by.  On the ORKUT-shaped C4 these pairs are 8e9 of the 8.1e9
// level-2 survivors, and merging them is 0.7 s of a 1 s join.
//
// What.  The K most frequent tokens of the region (its "head") get dense
// indices; every region record becomes an exact K-bit head indicator h_r and
// a tail count t_r = |r| - popcount(h_r).  For any pair
//
//     overlap(r, s) = <h_r, h_s> + |tail_r  ^  tail_s|  <=  <h_r, h_s> + min(t_r, t_s)
//
// and <h_r, h_s> is an exact int8 GEMM (operands 0/1, s32 accumulators).  A
// pair whose bound is below the required overlap minov[|r|+|s|] cannot match
// (the same integer threshold reference src/similarity.cpp:113-115 verifies
// against, src/similarity.cpp:168-185); the rest are emitted as survivors and
// verified exactly by K3 (verify_pairs).  The head is a property of the data,
// not of a hash: the bound is exact for the head and loses only on the tail,
// which for Zipf-like token laws is short where it matters.  Reference
// counters are unaffected: they come from the level-1 b-bit filter (K2), which
// still tests every window pair; K2 only stops EMITTING the pairs this kernel
// covers (j >= L0, see TcParams::emit_col_end).
//
// Region: rows i >= L0 (records are size-sorted, so L0 = the first record with
// |r| >= S0) and columns j in [max(L0, j0(i)), i).
//
// Layout.  The head operand is slice-major so one bulk copy moves a K-slice of
// a whole tile: element (row r, k) of K at
//     (((k / 128) * groups + (r - base) / 8) * 8 + (k % 128) / 16) * 128 + (r % 8) * 16 + k % 16
// i.e. per K-slice of 128 bytes, 8-row core groups of 8 K-major 128-byte core
// matrices (SBO = 1024 between groups, LBO = 128 between the two 16-byte K
// halves of one kind::i8 instruction).
//
// Kernel: persistent, one CTA per SM, warp-specialised like K2:
//   warp 0      bulk-copy producer: per 128 x 256 output tile, K/128 stages of
//               (A slice 16 KB + B slice 32 KB) into a 4-stage ring
//   warp 1      TMEM allocator + MMA issuer: tcgen05.mma kind::i8 M=128 N=256
//               K=32, 4 per stage, into 2 accumulator slots of 256 columns
//   warps 2-17  epilogue: packed s16 TMEM loads, a per-group pre-test against
//               the group's lowest threshold, exact per-pair test on the rare
//               candidates, warp-queued emission of survivors (j, i)
// Work items: (row tile, 4096-column chunk), ordered chunk-major so the SMs
// working at once share one column chunk (its B operand stays in L2).
#pragma once

#include "filter_tc.cuh"

namespace ssjb {
namespace dev {

constexpr int kHeadSliceK = 128;                       // K bytes per pipeline stage
constexpr int kHeadStages = 4;
constexpr int kHeadQueue = 128;                        // survivor staging per epilogue warp
constexpr int kHeadGroupBytes = 8 * kHeadSliceK;       // one 8-row core group of one slice (SBO)

// Per operand kind: int8 (0/1 bytes, s32 accumulators, N = 256, two slots =
// all 512 TMEM columns) or mxf4 (packed e2m1 1.0 codes, unit block scales,
// f32 accumulators, twice the elements per byte and per instruction; N = 192
// so two slots leave TMEM room for the scale factors).
template <int KIND>
struct HeadLayout {
    static constexpr int NT = KIND == kKindF4 ? 192 : 256;   // columns per MMA tile
    static constexpr int kEpiWarps = NT / 16;                // 64 columns x 32 rows each
    static constexpr int kThreads = 64 + 32 * kEpiWarps;
    static constexpr int kA = kRowTile * kHeadSliceK;         // 16 KB
    static constexpr int kB = NT * kHeadSliceK;
    static constexpr int kStage = kA + kB;
    static constexpr int kSmem = kHeadStages * kStage + kEpiWarps * kHeadQueue * 8;
    static constexpr uint32_t kSfCol = 2 * NT;               // fp4: A scales, then B scales (+32)
    static constexpr uint32_t kTmemCols = 512;
    static_assert(kSmem + 2048 <= 232448, "shared memory per CTA");
    static_assert(KIND == kKindI8 || 2 * NT + 128 <= 512, "TMEM: accumulators + scale factors");
};

struct HeadParams {
    const uint8_t* op;          // head operand rows [base, base + 8 * groups), slice-major core layout
    uint32_t base;              // first operand row (multiple of 8)
    uint32_t groups;            // 8-row groups per slice
    int kslices;                // K / kHeadSliceK
    const uint32_t* info;       // (|r| << 16) | tail per operand row
    const int32_t* minov;       // minov[|r| + |s|]
    const uint32_t* wstart;     // j0 per record size
    const uint2* items;         // (row tile, column chunk), chunk-major
    const uint32_t* tile_col_lo;  // first (8-aligned) column of each row tile's window span
    uint32_t tile0;             // first row of row tile 0 (multiple of 8, >= base)
    uint32_t L0;                // first region record
    uint32_t row_begin, row_end;  // this shard's rows
    uint2* surv;
    unsigned long long surv_cap, surv_soft;
    unsigned long long item_begin, item_end;
    Control* ctl;               // the head phase's own control block (survivors, work_next)
};

struct HeadItem {
    uint32_t row0, c0, ntiles, done;
};

// lane 0 reads the published item and broadcasts it (see warp_item, filter_tc.cuh)
__device__ __forceinline__ HeadItem warp_head_item(const HeadItem& slot, int lane) {
    HeadItem v{};
    if (lane == 0) v = slot;
    v.row0 = __shfl_sync(0xFFFFFFFFu, v.row0, 0);
    v.c0 = __shfl_sync(0xFFFFFFFFu, v.c0, 0);
    v.ntiles = __shfl_sync(0xFFFFFFFFu, v.ntiles, 0);
    v.done = __shfl_sync(0xFFFFFFFFu, v.done, 0);
    return v;
}

__device__ __forceinline__ void head_flush(uint2* q, int& qlen, const HeadParams& P, int lane) {
    unsigned long long base = 0;
    if (lane == 0) base = atomicAdd(&P.ctl->survivors, static_cast<unsigned long long>(qlen));
    base = __shfl_sync(0xFFFFFFFFu, base, 0);
    for (int k = lane; k < qlen; k += 32)
        if (base + k < P.surv_cap) P.surv[base + k] = q[k];
    qlen = 0;
    __syncwarp();
}

// lane's survivors of a 32-column group (bit k = column base_col + k) into the warp queue
__device__ __forceinline__ void head_emit(uint32_t m, uint32_t base_col, uint32_t row, uint2* q, int& qlen,
                                          const HeadParams& P, int lane) {
    const int c = __popc(m);
    int incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xFFFFFFFFu, incl, o);
        if (lane >= o) incl += v;
    }
    const int total = __shfl_sync(0xFFFFFFFFu, incl, 31);
    if (total == 0) return;
    if (qlen + total > kHeadQueue) head_flush(q, qlen, P, lane);
    if (total > kHeadQueue) {  // (at most 32 x 32: straight to global memory)
        unsigned long long base = 0;
        if (lane == 0) base = atomicAdd(&P.ctl->survivors, static_cast<unsigned long long>(total));
        base = __shfl_sync(0xFFFFFFFFu, base, 0) + (incl - c);
        while (m) {
            const int k = __ffs(m) - 1;
            m &= m - 1;
            if (base < P.surv_cap) P.surv[base] = make_uint2(base_col + k, row);
            ++base;
        }
        return;
    }
    int pos = qlen + incl - c;
    while (m) {
        const int k = __ffs(m) - 1;
        m &= m - 1;
        q[pos++] = make_uint2(base_col + k, row);
    }
    qlen += total;
    __syncwarp();
}

template <int KIND>
__global__ void __launch_bounds__(HeadLayout<KIND>::kThreads, 1) head_overlap_kernel(HeadParams P) {
    using L = HeadLayout<KIND>;
    constexpr int kHeadNT = L::NT;
    constexpr int kHeadEpiWarps = L::kEpiWarps;
    constexpr int kHeadA = L::kA, kHeadB = L::kB, kHeadStage = L::kStage;
    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t* sStage = smem;                                                        // [kHeadStages][A | B]
    uint2* sQ = reinterpret_cast<uint2*>(smem + kHeadStages * kHeadStage);         // [warps][kHeadQueue]
    __shared__ __align__(8) uint64_t item_full[2], item_empty[2];
    __shared__ __align__(8) uint64_t s_full[kHeadStages], s_empty[kHeadStages], acc_full[2], acc_empty[2];
    __shared__ HeadItem items[2];
    __shared__ uint32_t tmem_base_sh;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    constexpr uint32_t kTmemCols = L::kTmemCols;

    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base_sh)),
                     "r"(kTmemCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 0) {
        for (int s = 0; s < 2; ++s) {
            mbar_init(&item_full[s], 1);
            mbar_init(&item_empty[s], 1 + kHeadEpiWarps);
            mbar_init(&acc_full[s], 1);
            mbar_init(&acc_empty[s], kHeadEpiWarps);
        }
        for (int s = 0; s < kHeadStages; ++s) {
            mbar_init(&s_full[s], 1);
            mbar_init(&s_empty[s], 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem_base = tmem_base_sh;
    if constexpr (KIND == kKindF4) {
        // unit block scales (ue8m0 127 = 1.0) for every A and B scale slot the MMA may read
        if (warp >= 2 && warp < 6) {
            const uint32_t lanes = static_cast<uint32_t>((warp & 3) * 32) << 16;
#pragma unroll
            for (int c = 0; c < 128; c += 32) tmem_fill32(tmem_base + lanes + L::kSfCol + c, 0x7F7F7F7Fu);
            asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        }
        asm volatile("tcgen05.fence::before_thread_sync;");
        __syncthreads();
        asm volatile("tcgen05.fence::after_thread_sync;");
    }
    const uint64_t slice_stride = static_cast<uint64_t>(P.groups) * kHeadGroupBytes;

    if (warp == 0) {
        // ------------------------------------------------------------ producer
        if (lane == 0) {
            uint32_t iseq = 0, sseq = 0;
            for (;;) {
                const int slot = iseq & 1;
                mbar_spin(&item_empty[slot], ((iseq >> 1) & 1) ^ 1);
                const unsigned long long it = claim_item(P.ctl, P.item_begin, P.item_end, P.surv_soft);
                HeadItem info{};
                if (it >= P.item_end) {
                    info.done = 1;
                    items[slot] = info;
                    mbar_arrive(&item_full[slot]);
                    break;
                }
                const uint2 w = P.items[it];  // (row tile, column chunk)
                const uint32_t row0 = P.tile0 + w.x * kRowTile;
                const uint32_t rmax = min(row0 + kRowTile, P.row_end);  // columns j < i < rmax
                const uint32_t chunk0 = P.base + w.y * kColChunk;
                info.row0 = row0;
                info.c0 = max(P.tile_col_lo[w.x], chunk0);
                const uint32_t c1 = min(chunk0 + kColChunk, rmax > 0 ? rmax - 1 : 0);
                info.ntiles = c1 > info.c0 ? (c1 - info.c0 + kHeadNT - 1) / kHeadNT : 0;
                info.done = 0;
                items[slot] = info;
                mbar_arrive(&item_full[slot]);
                const uint8_t* a_src = P.op + static_cast<uint64_t>((row0 - P.base) >> 3) * kHeadGroupBytes;
                for (uint32_t t = 0; t < info.ntiles; ++t) {
                    const uint8_t* b_src =
                        P.op + static_cast<uint64_t>((info.c0 + t * kHeadNT - P.base) >> 3) * kHeadGroupBytes;
                    for (int s = 0; s < P.kslices; ++s, ++sseq) {
                        const int st = sseq % kHeadStages;
                        mbar_spin(&s_empty[st], ((sseq / kHeadStages) & 1) ^ 1);
                        uint8_t* dst = sStage + st * kHeadStage;
                        mbar_expect_tx(&s_full[st], kHeadStage);
                        tma_load_1d(dst, a_src + s * slice_stride, kHeadA, &s_full[st]);
                        tma_load_1d(dst + kHeadA, b_src + s * slice_stride, kHeadB, &s_full[st]);
                    }
                }
                ++iseq;
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------------------ MMA issuer
        // (warp-uniform loop, one elected lane issues: see filter_tc_kernel)
        const bool leader = elect_one();
        {
            uint32_t iseq = 0, sseq = 0, aseq = 0;
            for (;;) {
                const int slot = iseq & 1;
                mbar_spin(&item_full[slot], (iseq >> 1) & 1);
                const HeadItem info = items[slot];
                __syncwarp();
                if (leader) mbar_arrive(&item_empty[slot]);
                if (info.done) break;
                for (uint32_t t = 0; t < info.ntiles; ++t, ++aseq) {
                    const int as = aseq & 1;
                    mbar_spin(&acc_empty[as], ((aseq >> 1) & 1) ^ 1);
                    asm volatile("tcgen05.fence::after_thread_sync;");
                    const uint32_t d = tmem_base + as * kHeadNT;
                    for (int s = 0; s < P.kslices; ++s, ++sseq) {
                        const int st = sseq % kHeadStages;
                        mbar_spin(&s_full[st], (sseq / kHeadStages) & 1);
                        asm volatile("tcgen05.fence::after_thread_sync;");
                        if (leader) {
                            const uint32_t a0 = smem_u32(sStage + st * kHeadStage);
                            const uint64_t da0 = umma_desc(a0, kHeadGroupBytes);
                            const uint64_t db0 = umma_desc(a0 + kHeadA, kHeadGroupBytes);
#pragma unroll
                            for (int k = 0; k < kHeadSliceK / 32; ++k) {
                                const uint64_t da = umma_desc_step(da0, k);
                                const uint64_t db = umma_desc_step(db0, k);
                                if constexpr (KIND == kKindI8)
                                    umma_i8<kHeadNT>(d, da, db, (s | k) != 0);
                                else
                                    umma_f4<kHeadNT>(d, da, db, (s | k) != 0, tmem_base + L::kSfCol,
                                                     tmem_base + L::kSfCol + 32);
                            }
                            umma_commit(&s_empty[st]);
                        }
                        __syncwarp();
                    }
                    if (leader) umma_commit(&acc_full[as]);
                    __syncwarp();
                }
                ++iseq;
            }
        }
    } else {
        // ------------------------------------------------------------ epilogue
        const int ew = warp - 2;
        const int quarter = warp & 3;  // TMEM lanes 32*quarter .. +31 (hardware rule)
        const int part = ew >> 2;      // 64-column quarter of each tile
        const int rit = quarter * 32 + lane;
        const uint32_t lane_base = static_cast<uint32_t>(quarter * 32) << 16;
        uint2* q = sQ + ew * kHeadQueue;
        int qlen = 0;
        uint32_t iseq = 0, aseq = 0;
        for (;;) {
            const int slot = iseq & 1;
            mbar_wait(&item_full[slot], (iseq >> 1) & 1);
            const HeadItem info = warp_head_item(items[slot], lane);
            __syncwarp();
            if (lane == 0) mbar_arrive(&item_empty[slot]);
            if (info.done) break;
            const uint32_t i = info.row0 + rit;
            const bool valid = i >= max(P.L0, P.row_begin) && i < P.row_end;
            uint32_t si = 0, ti = 0, lo_i = 0, hi_i = 0;
            if (valid) {
                const uint32_t inf = P.info[i - P.base];
                si = inf >> 16;
                ti = inf & 0xFFFFu;
                lo_i = max(P.L0, P.wstart[si]);
                hi_i = i;
            }
            for (uint32_t t = 0; t < info.ntiles; ++t, ++aseq) {
                const int as = aseq & 1;
                const uint32_t gcol = info.c0 + t * kHeadNT + part * 64;  // warp's first column
                // sizes of the warp's two 32-column groups' first columns (pre-test thresholds)
                const uint32_t f0 = __ldg(P.info + (gcol - P.base));
                const uint32_t f1 = __ldg(P.info + (gcol + 32 - P.base));
                mbar_wait(&acc_full[as], (aseq >> 1) & 1);
                asm volatile("tcgen05.fence::after_thread_sync;");
                // the warp's 64 accumulator columns: packed s16 pairs (int8: values <= K)
                // or two loads of 32 f32 values (mxf4)
                uint32_t d[KIND == kKindI8 ? 32 : 64];
                if constexpr (KIND == kKindI8) {
                    uint32_t (&d32)[32] = *reinterpret_cast<uint32_t(*)[32]>(d);
                    tmem_ld64_pack16(tmem_base + lane_base + as * kHeadNT + part * 64, d32);
                } else {
                    uint32_t (&lo)[32] = *reinterpret_cast<uint32_t(*)[32]>(d);
                    uint32_t (&hi)[32] = *reinterpret_cast<uint32_t(*)[32]>(d + 32);
                    tmem_ld32(tmem_base + lane_base + as * kHeadNT + part * 64, lo);
                    tmem_ld32(tmem_base + lane_base + as * kHeadNT + part * 64 + 32, hi);
                }
                asm volatile("tcgen05.fence::before_thread_sync;");
                __syncwarp();
                if (lane == 0) mbar_arrive(&acc_empty[as]);  // accumulators are in registers
#if defined(SSJB_HEAD_PROBE)
                if (SSJB_HEAD_PROBE == 3) continue;  // (probe: no epilogue math)
#endif
#pragma unroll
                for (int g = 0; g < 2; ++g) {
                    const uint32_t gbase = gcol + 32 * g;
                    const uint32_t rm = valid ? (low_mask(static_cast<int>(hi_i) - static_cast<int>(gbase)) &
                                                 ~low_mask(static_cast<int>(lo_i) - static_cast<int>(gbase)))
                                              : 0u;
                    // the group's columns are size-sorted: minov[si + first size] - ti is
                    // a lower bound of every column's threshold minov[si+sj] - min(ti,tj)
                    const uint32_t sfirst = (g ? f1 : f0) >> 16;
                    const int thr = valid ? __ldg(P.minov + si + sfirst) - static_cast<int>(ti) : 0;
                    uint32_t cand = 0;
                    if constexpr (KIND == kKindI8) {
                        uint32_t dg[16];
#pragma unroll
                        for (int k = 0; k < 16; ++k) dg[k] = d[16 * g + k];
                        cand = rm ? rm & mask16_32(dg, min(max(thr - 1, -32768), 32767)) : 0u;
                    } else if (rm) {
                        // exact integers in f32, all >= 0: compare the bit patterns as ints
                        const int key = thr <= 0 ? INT_MIN : __float_as_int(static_cast<float>(thr));
#pragma unroll
                        for (int k = 0; k < 32; ++k) cand |= (static_cast<int>(d[32 * g + k]) >= key ? 1u : 0u) << k;
                        cand &= rm;
                    }
                    uint32_t e = 0;
#ifdef SSJB_HEAD_PROBE
                    if (SSJB_HEAD_PROBE == 1) {  // (probe: count candidates)
                        const int c = __reduce_add_sync(0xFFFFFFFFu, __popc(cand));
                        if (lane == 0 && c) atomicAdd(&P.ctl->verify_bytes, static_cast<unsigned long long>(c));
                    }
                    if (SSJB_HEAD_PROBE >= 1) cand = 0;
#endif
                    if (cand) {  // rare: exact per-pair test of the pre-test's candidates
#pragma unroll
                        for (int k = 0; k < 32; ++k) {
                            if (!((cand >> k) & 1u)) continue;
                            const uint32_t inf = __ldg(P.info + (gbase + k - P.base));
                            const int need = __ldg(P.minov + si + (inf >> 16));
                            int acc;
                            if constexpr (KIND == kKindI8) acc = static_cast<int>((d[16 * g + (k >> 1)] >> (16 * (k & 1))) & 0xFFFFu);
                            else acc = static_cast<int>(__uint_as_float(d[32 * g + k]));
                            if (acc + static_cast<int>(min(ti, inf & 0xFFFFu)) >= need) e |= 1u << k;
                        }
                    }
                    if (__any_sync(0xFFFFFFFFu, e != 0)) head_emit(e, gbase, i, q, qlen, P, lane);
                }
            }
            ++iseq;
        }
        if (qlen) head_flush(q, qlen, P, lane);
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(kTmemCols));
}

// ---------------------------------------------------------------- head setup
// Token counts over every stride-th record of the region [L0, n), one warp
// per record: cnt[t] += 1 per occurrence.  The head only has to be a good
// guess of the frequent tokens (any head set gives an exact bound), so a
// sample of the region's records is enough.
__global__ void head_count(const uint32_t* tokens, const uint64_t* offsets, uint32_t L0, uint32_t n, uint32_t stride,
                           uint32_t* cnt) {
    const uint32_t warps = gridDim.x * (blockDim.x >> 5);
    const int lane = threadIdx.x & 31;
    for (uint32_t w = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);; w += warps) {
        const uint64_t r = L0 + static_cast<uint64_t>(w) * stride;
        if (r >= n) break;
        const uint64_t b = offsets[r], e = offsets[r + 1];
        for (uint64_t k = b + lane; k < e; k += 32) atomicAdd(cnt + tokens[k], 1u);
    }
}

// Count-of-counts for the head selection: hist[min(c, 65535)] over tokens with c >= 2
// (a token in one region record cannot contribute to any pair's overlap).
// Small counts (the contended buckets) go through a per-block histogram.
__global__ void __launch_bounds__(256) head_hist(const uint32_t* cnt, uint32_t universe, uint32_t* hist) {
    __shared__ uint32_t sh[1024];
    for (int k = threadIdx.x; k < 1024; k += blockDim.x) sh[k] = 0;
    __syncthreads();
    const uint32_t stride = gridDim.x * blockDim.x;
    for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < universe; t += stride) {
        const uint32_t c = cnt[t];
        if (c < 2) continue;
        if (c < 1024) atomicAdd(sh + c, 1u);
        else atomicAdd(hist + min(c, 65535u), 1u);
    }
    __syncthreads();
    for (int k = threadIdx.x; k < 1024; k += blockDim.x)
        if (sh[k]) atomicAdd(hist + k, sh[k]);
}

// One block of 1024 threads: the smallest count c* >= 2 such that at most K
// tokens have count >= c* (out[0]).  hist has 65536 buckets; chunk t of 64
// buckets is summed by thread t, then thread 0 scans from the top.
__global__ void __launch_bounds__(1024) head_threshold(const uint32_t* hist, uint32_t K, uint32_t* out) {
    __shared__ uint32_t part[1024];
    const int t = threadIdx.x;
    uint32_t s = 0;
    for (int k = 0; k < 64; ++k) s += hist[t * 64 + k];
    part[t] = s;
    __syncthreads();
    if (t != 0) return;
    uint32_t acc = 0, thr = 2;
    for (int c = 1023; c >= 0; --c) {
        if (acc + part[c] <= K) {
            acc += part[c];
            continue;
        }
        for (int k = 63; k >= 0; --k) {  // the cut lies in this chunk
            const uint32_t h = hist[c * 64 + k];
            if (acc + h > K) {
                thr = static_cast<uint32_t>(c * 64 + k + 1);
                break;
            }
            acc += h;
        }
        break;
    }
    out[0] = thr < 2 ? 2u : thr;
}

// Dense head indices for tokens with count >= c* (order is immaterial: any
// token set gives an exact bound); map[t] = index or 0xFFFF.
__global__ void head_assign(const uint32_t* cnt, uint32_t universe, const uint32_t* thr, uint32_t K,
                            uint16_t* map, uint32_t* next) {
    const uint32_t c0 = thr[0];
    const uint32_t stride = gridDim.x * blockDim.x;
    for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < universe; t += stride) {
        const bool take = cnt[t] >= c0;
        const uint32_t bal = __ballot_sync(__activemask(), take);
        if (!take) continue;
        const int lane = threadIdx.x & 31;
        const int leader = __ffs(bal) - 1;
        uint32_t base = 0;
        if (lane == leader) base = atomicAdd(next, static_cast<uint32_t>(__popc(bal)));
        base = __shfl_sync(bal, base, leader) + __popc(bal & ((1u << lane) - 1u));
        map[t] = base < K ? static_cast<uint16_t>(base) : static_cast<uint16_t>(0xFFFFu);
    }
}

// One CTA per 8-row core group of operand rows [base + 8g, +8): the head
// indicator rows in the slice-major core layout -- int8 (one byte 0/1 per
// head token, K bytes) or mxf4 (e2m1 1.0 = 0x2 per head token, two per byte
// low nibble first, K/2 bytes) -- and info[] = (|r| << 16) | tail.  Rows
// outside [L0, n) stay zero (size 0).
template <int KIND>
__global__ void __launch_bounds__(256) head_expand(const uint32_t* tokens, const uint64_t* offsets, uint32_t n,
                                                   uint32_t L0, uint32_t base, uint32_t groups, int K,
                                                   const uint16_t* map, uint8_t* op, uint32_t* info) {
    extern __shared__ __align__(16) uint8_t rowbuf[];  // [8][RB]
    __shared__ uint32_t heads[8];
    const int RB = KIND == kKindI8 ? K : K / 2;         // operand bytes per row
    const uint32_t g = blockIdx.x;
    uint4* z = reinterpret_cast<uint4*>(rowbuf);
    for (int k = threadIdx.x; k < 8 * RB / 16; k += blockDim.x) z[k] = make_uint4(0, 0, 0, 0);
    if (threadIdx.x < 8) heads[threadIdx.x] = 0;
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t r = base + 8 * g + warp;  // one warp per row
    if (r >= L0 && r < n) {
        const uint64_t b = offsets[r], e = offsets[r + 1];
        uint32_t h = 0;
        for (uint64_t k = b + lane; k < e; k += 32) {
            const uint32_t m = map[tokens[k]];
            if (m != 0xFFFFu) {
                if constexpr (KIND == kKindI8) rowbuf[warp * RB + m] = 1;
                else atomicOr(reinterpret_cast<uint32_t*>(rowbuf + warp * RB) + (m >> 3), 0x2u << (4 * (m & 7)));
                ++h;
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) h += __shfl_xor_sync(0xFFFFFFFFu, h, o);
        if (lane == 0) heads[warp] = h;
    }
    __syncthreads();
    if (threadIdx.x < 8) {
        const uint32_t rr = base + 8 * g + threadIdx.x;
        const uint32_t sz = (rr >= L0 && rr < n) ? static_cast<uint32_t>(offsets[rr + 1] - offsets[rr]) : 0u;
        info[8 * g + threadIdx.x] = (sz << 16) | (sz - heads[threadIdx.x]);
    }
    // 16-byte units: unit u -> (slice s, chunk c, row q): u = (s * 8 + c) * 8 + q
    const int units = RB / 16 * 8;
    for (int u = threadIdx.x; u < units; u += blockDim.x) {
        const int q = u & 7, c = (u >> 3) & 7, s = u >> 6;
        const uint4 v = *reinterpret_cast<const uint4*>(rowbuf + q * RB + s * kHeadSliceK + c * 16);
        const uint64_t off = ((static_cast<uint64_t>(s) * groups + g) * 8 + c) * 128 + q * 16;
        *reinterpret_cast<uint4*>(op + off) = v;
    }
}

}  // namespace dev
}  // namespace ssjb
