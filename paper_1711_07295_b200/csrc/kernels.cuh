// sm_100a kernels of the Bitmap-Filter self-join (paper Alg. 8; reference
// hot loop src/parallel_join.cpp:61-136).  Included by engine.cu only.
//
//   K1 build_sketches   one b-bit sketch per record (Set / Xor / Next)
//   K2 filter           row tile x column chunk; TMA-staged column sketches,
//                       xor + POPC against an exact per-(|r|+|s|) threshold,
//                       survivors compacted through warp ballots
//   K2b rescan_saturated  position of the capacity-th survivor of rows whose
//                       reference buffer would saturate (counter semantics)
//   K3 verify           exact merge intersection with early exit
//   K4 radix sort       canonical (id_r, id_s) order of the matches
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace ssjb {
namespace dev {

constexpr int kRowTile = 128;     // rows per work item == threads per filter CTA
constexpr int kColSub = 256;      // columns per TMA stage
constexpr int kColChunk = 4096;   // columns per work item
constexpr int kWarpQueue = 512;   // survivor staging entries per warp
constexpr int kMaxInlineWords = 8;

struct Control {
    unsigned long long survivors;   // survivors emitted (may exceed capacity: overflow)
    unsigned long long results;     // matches emitted
    unsigned long long work_next;   // persistent-kernel work counter
    unsigned long long tested, pruned, verified, saturated;  // counter sums
    unsigned long long verify_bytes;  // algorithmic bytes of K3
    unsigned long long sat_rows;      // rows listed by find_saturated
    unsigned long long pad[6];
};

// Work-item claim of the persistent filters.  With a soft survivor cap the
// producer stops claiming once the batch's survivors pass it, so a launch
// always finishes with a prefix [item_begin, item_begin + work_next) of its
// items processed (every claimed item is processed) and the survivor buffer
// fills to about the cap instead of overflowing; the host resumes from there.
__device__ __forceinline__ unsigned long long claim_item(Control* ctl, unsigned long long item_begin,
                                                         unsigned long long item_end, unsigned long long soft) {
    if (soft) {
        unsigned long long cur;
        asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(cur) : "l"(&ctl->survivors));
        if (cur > soft) return item_end;
    }
    return item_begin + atomicAdd(&ctl->work_next, 1ull);
}

// ------------------------------------------------------------------ hashing
// reference src/bitmap.hpp:30-36
__device__ __forceinline__ uint32_t hash_token(uint32_t t, uint32_t width, int hash_mult, bool pow2) {
    if (hash_mult) {
        uint32_t h = static_cast<uint32_t>((static_cast<uint64_t>(t) * 0x9E3779B97F4A7C15ull) >> 33);
        return pow2 ? (h & (width - 1)) : (h % width);
    }
    return pow2 ? (t & (width - 1)) : (t % width);
}

// =============================================================== K1: sketches
struct BuildParams {
    const uint32_t* tokens;
    const uint64_t* offsets;
    uint64_t* bits;        // n * W words, row-major
    uint32_t n;
    uint32_t width;        // b
    int words;             // W = b / 64
    int method;            // 0 Set, 1 Xor, 2 Next
    int hash_mult;
    int pow2;
};

constexpr int kBuildRecs = 128;           // records (threads) per CTA
constexpr int kBuildStage = 8192;         // staged tokens per CTA (32 KB)

// One thread per record.  The CTA first stages the token range of its 128
// records into shared memory with coalesced 128-bit loads, then each thread
// folds its record into a register sketch.  Next (linear probing into the
// next free bit, reference src/bitmap.cpp:40-62) is insertion-order
// independent (reference tests/test_bitmap.cpp:108-122), so the probe order
// is free; a record with |s| >= b is all ones.
template <int W>
__global__ void __launch_bounds__(kBuildRecs) build_sketches(BuildParams P) {
    __shared__ __align__(16) uint32_t stage[kBuildStage + 8];
    const uint32_t r0 = blockIdx.x * kBuildRecs;
    const uint32_t r = r0 + threadIdx.x;
    const uint32_t rl = min(r0 + kBuildRecs, P.n);
    const uint64_t t_begin = P.offsets[r0];
    const uint64_t t_end = P.offsets[rl];
    const uint64_t a_begin = t_begin & ~uint64_t(3);  // 16-byte aligned start
    const bool staged = (t_end - a_begin) <= kBuildStage;
    if (staged) {
        const uint64_t nvec = (t_end - a_begin + 3) / 4;
        const uint4* src = reinterpret_cast<const uint4*>(P.tokens + a_begin);
        uint4* dst = reinterpret_cast<uint4*>(stage);
        for (uint64_t k = threadIdx.x; k < nvec; k += kBuildRecs) dst[k] = __ldg(src + k);
    }
    __syncthreads();
    if (r >= P.n) return;
    const uint64_t b = P.offsets[r], e = P.offsets[r + 1];
    const uint32_t cnt = static_cast<uint32_t>(e - b);
    const uint32_t* tok = staged ? stage + (b - a_begin) : P.tokens + b;
    const int words = W > 0 ? W : P.words;
    uint64_t row[W > 0 ? W : kMaxInlineWords];
    if constexpr (W > 0) {
#pragma unroll
        for (int w = 0; w < W; ++w) row[w] = 0;
        if (P.method == 2 && cnt >= P.width) {
#pragma unroll
            for (int w = 0; w < W; ++w) row[w] = ~0ull;
        } else {
            for (uint32_t k = 0; k < cnt; ++k) {
                uint32_t h = hash_token(tok[k], P.width, P.hash_mult, P.pow2);
                uint32_t hw = h >> 6;
                uint64_t bit = 1ull << (h & 63);
                if (P.method == 0) {
#pragma unroll
                    for (int w = 0; w < W; ++w) row[w] |= (hw == uint32_t(w)) ? bit : 0ull;
                } else if (P.method == 1) {
#pragma unroll
                    for (int w = 0; w < W; ++w) row[w] ^= (hw == uint32_t(w)) ? bit : 0ull;
                } else {
                    // first free bit at or after h, then wrap to the front
                    bool placed = false;
#pragma unroll
                    for (int w = 0; w < W; ++w) {
                        uint64_t fb = uint32_t(w) < hw ? 0ull : ~row[w];
                        if (uint32_t(w) == hw) fb &= ~0ull << (h & 63);
                        if (!placed && fb) {
                            row[w] |= fb & (~fb + 1);
                            placed = true;
                        }
                    }
#pragma unroll
                    for (int w = 0; w < W; ++w) {
                        uint64_t fb = ~row[w];
                        if (uint32_t(w) <= hw && !placed && fb) {
                            row[w] |= fb & (~fb + 1);
                            placed = true;
                        }
                    }
                }
            }
        }
        uint64_t* out = P.bits + static_cast<uint64_t>(r) * W;
#pragma unroll
        for (int w = 0; w < W; ++w) out[w] = row[w];
    } else {
        // Wide sketches (b > 512): build directly in global memory, one thread
        // per record; rare and off the hot path.
        uint64_t* out = P.bits + static_cast<uint64_t>(r) * words;
        for (int w = 0; w < words; ++w) out[w] = 0;
        if (P.method == 2 && cnt >= P.width) {
            for (int w = 0; w < words; ++w) out[w] = ~0ull;
        } else {
            for (uint32_t k = 0; k < cnt; ++k) {
                uint32_t h = hash_token(tok[k], P.width, P.hash_mult, P.pow2);
                if (P.method == 0) {
                    out[h >> 6] |= 1ull << (h & 63);
                } else if (P.method == 1) {
                    out[h >> 6] ^= 1ull << (h & 63);
                } else {
                    int word = static_cast<int>(h >> 6);
                    uint64_t fb = ~out[word] & (~0ull << (h & 63));
                    for (int step = 0; step <= words; ++step) {
                        if (fb) {
                            out[word] |= fb & (~fb + 1);
                            break;
                        }
                        word = (word + 1) % words;
                        fb = ~out[word];
                    }
                }
            }
        }
    }
}

// Set / Xor sketches with LPR lanes per record (LPR = 1..32, a power of two):
// lane k of a record's group folds 16-byte chunks k, k+LPR, ... into register
// sketches, then the group combines them with shuffles (OR for Set, XOR for
// Xor -- both order-independent, reference src/bitmap.cpp:70-81).  Token loads
// are coalesced across the group.  With W2 > 0 the same token pass also
// builds the level-2 Xor sketch (64*W2 bits) into bits2.
struct BuildParams2 {
    const uint32_t* tokens;
    const uint64_t* offsets;
    uint64_t* bits;        // n * W words
    uint64_t* bits2;       // n * W2 words (W2 > 0)
    uint32_t n;            // rows [row0, n) are built
    uint32_t row0;
    uint32_t width, width2;
    int method;            // 0 Set, 1 Xor
    int hash_mult;
    int pow2, pow2_2;
    int lpr_log2;          // log2(lanes per record)
    uint64_t total_tokens; // tokens in the array (bound of the 16-byte loads)
};

template <int W, int W2, bool XOR>
__global__ void __launch_bounds__(256) build_sketches_sub(BuildParams2 P) {
    const int lpr = 1 << P.lpr_log2;
    const uint32_t gtid = blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t r = P.row0 + (gtid >> P.lpr_log2);
    const int sub = static_cast<int>(gtid & (lpr - 1));
    const bool live = r < P.n;
    uint64_t row[W], row2[W2 > 0 ? W2 : 1];
#pragma unroll
    for (int w = 0; w < W; ++w) row[w] = 0;
#pragma unroll
    for (int w = 0; w < (W2 > 0 ? W2 : 1); ++w) row2[w] = 0;
    // widths are compile-time (64 W, 64 W2): the modulo of hash_token
    // (reference src/bitmap.hpp:30-36) folds to a mask or a multiply-shift
    auto fold = [&](uint32_t t) {
            const uint32_t hm = P.hash_mult ? static_cast<uint32_t>((static_cast<uint64_t>(t) * 0x9E3779B97F4A7C15ull) >> 33)
                                            : t;
            const uint32_t h = hm % (64u * W);
            const uint64_t bit = 1ull << (h & 63);
#pragma unroll
            for (int w = 0; w < W; ++w) {
                const uint64_t m = (W == 1 || (h >> 6) == uint32_t(w)) ? bit : 0ull;
                row[w] = XOR ? (row[w] ^ m) : (row[w] | m);
            }
            if constexpr (W2 > 0) {
                const uint32_t h2 = hm % (64u * W2);
                const uint64_t bit2 = 1ull << (h2 & 63);
#pragma unroll
                for (int w = 0; w < W2; ++w) row2[w] ^= (h2 >> 6) == uint32_t(w) ? bit2 : 0ull;
            }
    };
    if (live) {
        // the record's span as aligned 16-byte chunks, chunk c to lane c mod
        // lpr, four 128-bit loads in flight per lane before folding (a scalar
        // strided loop is bound by one load round trip per token)
        const uint64_t b = P.offsets[r], e = P.offsets[r + 1];
        // 32-bit offsets relative to the record's first aligned chunk
        const uint64_t a0 = b & ~uint64_t(3);
        const uint32_t lo = static_cast<uint32_t>(b - a0), hi = static_cast<uint32_t>(e - a0);
        const uint64_t rem = P.total_tokens - a0;
        const uint32_t lim = rem > 0xFFFFFFFFull ? 0xFFFFFFFFu : static_cast<uint32_t>(rem);
        const uint32_t* base = P.tokens + a0;
        for (uint32_t c = 4u * sub; c < hi; c += 16u * lpr) {
            uint4 v[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const uint32_t cc = c + 4u * lpr * u;
                if (cc + 4 <= lim) {
                    v[u] = cc < hi ? __ldg(reinterpret_cast<const uint4*>(base + cc)) : make_uint4(0, 0, 0, 0);
                } else {
                    v[u].x = cc < hi ? base[cc] : 0u;
                    v[u].y = cc + 1 < hi ? base[cc + 1] : 0u;
                    v[u].z = cc + 2 < hi ? base[cc + 2] : 0u;
                    v[u].w = 0u;
                }
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const uint32_t cc = c + 4u * lpr * u;
                if (cc >= lo && cc + 4 <= hi) {  // interior chunk: no per-token bounds
                    fold(v[u].x);
                    fold(v[u].y);
                    fold(v[u].z);
                    fold(v[u].w);
                } else if (cc < hi) {
                    const uint32_t t4[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
#pragma unroll
                    for (int q = 0; q < 4; ++q)
                        if (cc + q >= lo && cc + q < hi) fold(t4[q]);
                }
            }
        }
    }
    // group reduction (groups never straddle a warp: lpr divides 32)
    for (int o = lpr >> 1; o > 0; o >>= 1) {
#pragma unroll
        for (int w = 0; w < W; ++w) {
            const uint64_t v = __shfl_xor_sync(0xFFFFFFFFu, row[w], o);
            row[w] = XOR ? (row[w] ^ v) : (row[w] | v);
        }
        if constexpr (W2 > 0) {
#pragma unroll
            for (int w = 0; w < W2; ++w) row2[w] ^= __shfl_xor_sync(0xFFFFFFFFu, row2[w], o);
        }
    }
    if (!live) return;
    // lanes of the group store disjoint words
#pragma unroll
    for (int w = 0; w < W; ++w)
        if (w % lpr == sub) P.bits[static_cast<uint64_t>(r) * W + w] = row[w];
    if constexpr (W2 > 0) {
#pragma unroll
        for (int w = 0; w < W2; ++w)
            if (w % lpr == sub) P.bits2[static_cast<uint64_t>(r) * W2 + w] = row2[w];
    }
}

// Records too long for a lane group (sizes are sorted, so they are the tail
// rows of the build): one CTA per record, every thread folds 16-byte chunks
// (four in flight), then warp shuffles and a shared-memory combine.  Without
// this the last blocks of a heavy-tailed collection (C4: up to 40,425 tokens
// per record on 8 lanes) run alone long after the rest of the grid.
template <int W, int W2, bool XOR>
__global__ void __launch_bounds__(256) build_sketches_big(BuildParams2 P) {
    __shared__ uint64_t part[8][W + (W2 > 0 ? W2 : 0)];
    const uint32_t r = P.row0 + blockIdx.x;
    if (r >= P.n) return;
    uint64_t row[W], row2[W2 > 0 ? W2 : 1];
#pragma unroll
    for (int w = 0; w < W; ++w) row[w] = 0;
#pragma unroll
    for (int w = 0; w < (W2 > 0 ? W2 : 1); ++w) row2[w] = 0;
    auto fold = [&](uint32_t t) {
        const uint32_t hm = P.hash_mult ? static_cast<uint32_t>((static_cast<uint64_t>(t) * 0x9E3779B97F4A7C15ull) >> 33)
                                        : t;
        const uint32_t h = hm % (64u * W);
        const uint64_t bit = 1ull << (h & 63);
#pragma unroll
        for (int w = 0; w < W; ++w) {
            const uint64_t m = (W == 1 || (h >> 6) == uint32_t(w)) ? bit : 0ull;
            row[w] = XOR ? (row[w] ^ m) : (row[w] | m);
        }
        if constexpr (W2 > 0) {
            const uint32_t h2 = hm % (64u * W2);
            const uint64_t bit2 = 1ull << (h2 & 63);
#pragma unroll
            for (int w = 0; w < W2; ++w) row2[w] ^= (h2 >> 6) == uint32_t(w) ? bit2 : 0ull;
        }
    };
    const uint64_t b = P.offsets[r], e = P.offsets[r + 1];
    const uint64_t a0 = b & ~uint64_t(3);
    const uint32_t lo = static_cast<uint32_t>(b - a0), hi = static_cast<uint32_t>(e - a0);
    const uint64_t rem = P.total_tokens - a0;
    const uint32_t lim = rem > 0xFFFFFFFFull ? 0xFFFFFFFFu : static_cast<uint32_t>(rem);
    const uint32_t* base = P.tokens + a0;
    constexpr uint32_t T = 256;
    for (uint32_t c = 4u * threadIdx.x; c < hi; c += 16u * T) {
        uint4 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const uint32_t cc = c + 4u * T * u;
            if (cc + 4 <= lim) {
                v[u] = cc < hi ? __ldg(reinterpret_cast<const uint4*>(base + cc)) : make_uint4(0, 0, 0, 0);
            } else {
                v[u].x = cc < hi ? base[cc] : 0u;
                v[u].y = cc + 1 < hi ? base[cc + 1] : 0u;
                v[u].z = cc + 2 < hi ? base[cc + 2] : 0u;
                v[u].w = 0u;
            }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const uint32_t cc = c + 4u * T * u;
            if (cc >= lo && cc + 4 <= hi) {
                fold(v[u].x);
                fold(v[u].y);
                fold(v[u].z);
                fold(v[u].w);
            } else if (cc < hi) {
                const uint32_t t4[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    if (cc + q >= lo && cc + q < hi) fold(t4[q]);
            }
        }
    }
    for (int o = 16; o > 0; o >>= 1) {
#pragma unroll
        for (int w = 0; w < W; ++w) {
            const uint64_t v = __shfl_xor_sync(0xFFFFFFFFu, row[w], o);
            row[w] = XOR ? (row[w] ^ v) : (row[w] | v);
        }
        if constexpr (W2 > 0) {
#pragma unroll
            for (int w = 0; w < W2; ++w) row2[w] ^= __shfl_xor_sync(0xFFFFFFFFu, row2[w], o);
        }
    }
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) {
#pragma unroll
        for (int w = 0; w < W; ++w) part[warp][w] = row[w];
        if constexpr (W2 > 0) {
#pragma unroll
            for (int w = 0; w < W2; ++w) part[warp][W + w] = row2[w];
        }
    }
    __syncthreads();
    constexpr int kAll = W + (W2 > 0 ? W2 : 0);
    if (threadIdx.x < kAll) {
        const int w = threadIdx.x;
        uint64_t acc = part[0][w];
        for (int k = 1; k < 8; ++k) acc = (XOR || w >= W) ? (acc ^ part[k][w]) : (acc | part[k][w]);
        if (w < W) P.bits[static_cast<uint64_t>(r) * W + w] = acc;
        else P.bits2[static_cast<uint64_t>(r) * W2 + (w - W)] = acc;
    }
}

// ================================================================ K2: filter
struct FilterParams {
    const uint64_t* bits;        // sketches, n * W words (padded by kColSub rows)
    const uint64_t* bits2;       // level-2 Xor sketches, n * W2 words (W2 = 0: none)
    const uint32_t* sizes;       // |r| per record (padded)
    const int32_t* maxham;       // maxham[S] = S - 2*minov[S], S in [0, 2*max_size]
    const uint32_t* wstart;      // j0 per record size
    const uint64_t* item_base;   // work items per tile, prefix (ntiles + 1)
    const uint32_t* tile_col_lo; // first (32-aligned) column of each tile's span
    uint2* surv;                 // survivors (j, i)
    uint32_t* rowcnt;            // survivors per row (row - row_begin)
    uint32_t* item_counts;       // survivors per (item, row-in-tile) for the rescan, or null
    Control* ctl;
    unsigned long long surv_cap;
    unsigned long long surv_soft;  // stop claiming work items once this many survivors exist (0: never)
    unsigned long long item_begin, item_end;
    uint32_t tile_begin;         // tile index of item_begin's tile (search lower bound)
    uint32_t ntiles;
    uint32_t row_begin, row_end;
    int64_t cutoff;              // bypass the filter for rows with |r| > cutoff
    int words;
    int colsub;                  // columns per TMA stage for the generic-width kernel
    int bypass_all;              // bitmap disabled or NAIVE: every window pair survives
    int naive;                   // NAIVE: window [0, i)
};

__device__ __forceinline__ uint32_t low_mask(int x) {
    return x >= 32 ? 0xFFFFFFFFu : (x <= 0 ? 0u : ((1u << x) - 1u));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(bar));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(bar));
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(a), "r"(bytes) : "memory");
}

__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(dst));
    uint32_t b = static_cast<uint32_t>(__cvta_generic_to_shared(bar));
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(d),
        "l"(src), "r"(bytes), "r"(b)
        : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(bar));
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n"
        "@!P1 bra WAIT_%=;\n"
        "}\n" ::"r"(a),
        "r"(parity), "r"(0x989680u)  // suspend-time hint: sleep in hardware instead of spinning
        : "memory");
}

// Survivor emission for one 32-column group: lane l owns row i and the
// survivor bitmap m (bit k = column base+k).  Staged per warp in shared
// memory; flushed to the global survivor array with one atomic per flush.
__device__ __forceinline__ void warp_flush(uint2* q, int& qlen, const FilterParams& P, int lane) {
    unsigned long long base = 0;
    if (lane == 0) base = atomicAdd(&P.ctl->survivors, static_cast<unsigned long long>(qlen));
    base = __shfl_sync(0xFFFFFFFFu, base, 0);
    for (int k = lane; k < qlen; k += 32)
        if (base + k < P.surv_cap) P.surv[base + k] = q[k];
    qlen = 0;
    __syncwarp();
}

__device__ __forceinline__ void emit_group(uint32_t m, uint32_t base_col, uint32_t row, uint2* q, int& qlen,
                                           const FilterParams& P, int lane) {
    const int c = __popc(m);
    int incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int v = __shfl_up_sync(0xFFFFFFFFu, incl, o);
        if (lane >= o) incl += v;
    }
    const int total = __shfl_sync(0xFFFFFFFFu, incl, 31);
    const int excl = incl - c;
    if (total > kWarpQueue) {
        // bulk (bypassed rows): reserve directly in the global array
        unsigned long long base = 0;
        if (lane == 0) base = atomicAdd(&P.ctl->survivors, static_cast<unsigned long long>(total));
        base = __shfl_sync(0xFFFFFFFFu, base, 0) + excl;
        while (m) {
            int k = __ffs(m) - 1;
            m &= m - 1;
            if (base < P.surv_cap) P.surv[base] = make_uint2(base_col + k, row);
            ++base;
        }
        return;
    }
    if (qlen + total > kWarpQueue) warp_flush(q, qlen, P, lane);
    int pos = qlen + excl;
    while (m) {
        int k = __ffs(m) - 1;
        m &= m - 1;
        q[pos++] = make_uint2(base_col + k, row);
    }
    qlen += total;
    __syncwarp();
}

// Persistent filter kernel.  Work item = (tile of 128 consecutive rows, chunk
// of <= kColChunk columns of the tile's window span).  Thread t owns row
// i = tile*128 + t with its sketch in registers; the chunk's column sketches
// and sizes stream through a 2-stage TMA (cp.async.bulk) ring in shared
// memory and every lane reads the same column (smem broadcast).  Per pair:
// W x (2 LOP3 + 2 POPC) + IADD3 + SHF.  skip <=> popcount(b_i ^ b_j) >
// maxham[|r_i|+|r_j|], the exact integer form of reference
// src/bitmap.cpp:125-143 with src/similarity.cpp:113-115.
//
// Level 2 (W2 > 0): the level-1 mask m alone defines the reference counters
// (per-row survivors); pairs in m are additionally tested against a wider
// Xor sketch (b2 = 64*W2 bits, same exact threshold) before they are emitted
// for verification.  Both tests are sound upper bounds on the overlap, so the
// emitted set still contains every matching pair -- it only spares the
// verifier the pairs a b-bit sketch cannot reject (at tau = 0.5 on C2 with
// b = 128 that is 43% of all window pairs).  Dense groups test all 32 columns;
// sparse ones only the surviving columns of each lane.
template <int W, int W2>
__global__ void __launch_bounds__(kRowTile) filter_kernel(FilterParams P) {
    constexpr int WS = W > 0 ? W : 1;
    constexpr int WS2 = W2 > 0 ? W2 : 1;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int words = W > 0 ? W : P.words;
    const int colsub = W > 0 ? kColSub : P.colsub;  // columns per stage
    uint64_t* s_bits = reinterpret_cast<uint64_t*>(smem_raw);                  // [2][colsub*W]
    uint64_t* s_bits2 = s_bits + 2 * colsub * words;                           // [2][colsub*W2]
    uint32_t* s_size = reinterpret_cast<uint32_t*>(s_bits2 + 2 * colsub * W2);  // [2][colsub]
    uint2* s_queue = reinterpret_cast<uint2*>(s_size + 2 * colsub);            // [4][kWarpQueue]
    __shared__ __align__(8) uint64_t bars[2];
    __shared__ unsigned long long s_item;
    __shared__ uint32_t s_tile;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    uint2* q = s_queue + warp * kWarpQueue;
    int qlen = 0;
    if (tid == 0) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    uint32_t phase = 0;  // bit b = parity of stage buffer b

    for (;;) {
        if (tid == 0) {
            unsigned long long it = claim_item(P.ctl, P.item_begin, P.item_end, P.surv_soft);
            uint32_t t = 0;
            if (it < P.item_end) {
                uint32_t lo = P.tile_begin, hi = P.ntiles;  // largest t with item_base[t] <= it
                while (hi - lo > 1) {
                    uint32_t mid = (lo + hi) >> 1;
                    if (P.item_base[mid] <= it) lo = mid; else hi = mid;
                }
                t = lo;
            }
            s_item = it;
            s_tile = t;
        }
        __syncthreads();
        const unsigned long long item = s_item;
        const uint32_t tile = s_tile;
        if (item >= P.item_end) break;
        const uint32_t chunk = static_cast<uint32_t>(item - P.item_base[tile]);

        const uint32_t tile_row0 = P.row_begin + tile * kRowTile;
        const uint32_t tile_rows_end = min(tile_row0 + kRowTile, P.row_end);
        const uint32_t i = tile_row0 + tid;
        const bool valid = i < tile_rows_end;
        const uint32_t c0 = P.tile_col_lo[tile] + chunk * kColChunk;
        const uint32_t c1 = min(c0 + kColChunk, tile_rows_end - 1);  // columns < last row

        uint64_t mine[WS], mine2[WS2];
        uint32_t si = 0, j0 = 0;
        bool bypass = P.bypass_all != 0;
#pragma unroll
        for (int w = 0; w < WS; ++w) mine[w] = 0;
#pragma unroll
        for (int w = 0; w < WS2; ++w) mine2[w] = 0;
        if (valid) {
            si = P.sizes[i];
            j0 = P.naive ? 0u : P.wstart[si];
            if (static_cast<int64_t>(si) > P.cutoff) bypass = true;
            if constexpr (W > 0) {
#pragma unroll
                for (int w = 0; w < W; ++w) mine[w] = P.bits[static_cast<uint64_t>(i) * W + w];
            }
            if constexpr (W2 > 0) {
#pragma unroll
                for (int w = 0; w < W2; ++w) mine2[w] = P.bits2[static_cast<uint64_t>(i) * W2 + w];
            }
        }
        const uint32_t lo_i = valid ? max(j0, c0) : c1;
        const uint32_t hi_i = valid ? min(i, c1) : c1;
        uint32_t cnt = 0;

        const uint32_t nsub = (c1 - c0 + colsub - 1) / colsub;
        auto issue = [&](uint32_t s, int buf) {
            const uint32_t cs = c0 + s * colsub;
            const uint32_t ncol = min(static_cast<uint32_t>(colsub), c1 - cs);
            const uint32_t ncol4 = (ncol + 3) & ~3u;  // padded allocation keeps this in bounds
            const uint32_t bb = ncol4 * 8u * static_cast<uint32_t>(words);
            const uint32_t bb2 = ncol4 * 8u * static_cast<uint32_t>(W2);
            const uint32_t sb = ncol4 * 4u;
            mbar_expect_tx(&bars[buf], bb + bb2 + sb);
            tma_load_1d(s_bits + buf * colsub * words, P.bits + static_cast<uint64_t>(cs) * words, bb, &bars[buf]);
            if constexpr (W2 > 0)
                tma_load_1d(s_bits2 + buf * colsub * W2, P.bits2 + static_cast<uint64_t>(cs) * W2, bb2, &bars[buf]);
            tma_load_1d(s_size + buf * colsub, P.sizes + cs, sb, &bars[buf]);
        };
        if (tid == 0 && nsub > 0) issue(0, 0);

        for (uint32_t s = 0; s < nsub; ++s) {
            const int buf = s & 1;
            if (tid == 0 && s + 1 < nsub) issue(s + 1, buf ^ 1);
            mbar_wait(&bars[buf], (phase >> buf) & 1u);
            phase ^= 1u << buf;
            const uint32_t cs = c0 + s * colsub;
            const uint32_t ncol = min(static_cast<uint32_t>(colsub), c1 - cs);
            const uint64_t* cb = s_bits + buf * colsub * words;
            const uint64_t* cb2 = s_bits2 + buf * colsub * W2;
            const uint32_t* cz = s_size + buf * colsub;
            const uint32_t sz_first = cz[0], sz_last = cz[ncol - 1];
            const bool uniform = sz_first == sz_last;
            // d = h - T - 1 < 0  <=> survive;  T = maxham[si + sj]
            int negT1 = 0;
            if (uniform) negT1 = -P.maxham[si + sz_first] - 1;
            for (uint32_t g = 0; g < ncol; g += 32) {
                const uint32_t gbase = cs + g;
                const int kl = static_cast<int>(lo_i) - static_cast<int>(gbase);
                const int kh = static_cast<int>(hi_i) - static_cast<int>(gbase);
                const uint32_t rm = low_mask(kh) & ~low_mask(kl);
                uint32_t m = 0;
                if (__any_sync(0xFFFFFFFFu, rm != 0)) {
                    const int kmax = min(32, static_cast<int>(ncol - g));
                    if (uniform && kmax == 32) {
#pragma unroll 8
                        for (int k = 0; k < 32; ++k) {
                            const uint64_t* col = cb + (g + k) * words;
                            int h = 0;
                            if constexpr (W > 0) {
#pragma unroll
                                for (int w = 0; w < W; ++w) h += __popcll(mine[w] ^ col[w]);
                            } else {
                                const uint64_t* me = P.bits + static_cast<uint64_t>(i) * words;
                                for (int w = 0; w < words; ++w) h += __popcll(me[w] ^ col[w]);
                            }
                            m = __funnelshift_l(static_cast<uint32_t>(h + negT1), m, 1);
                        }
                        m = __brev(m);
                    } else {
                        for (int k = 0; k < kmax; ++k) {
                            const uint64_t* col = cb + (g + k) * words;
                            int h = 0;
                            if constexpr (W > 0) {
#pragma unroll
                                for (int w = 0; w < W; ++w) h += __popcll(mine[w] ^ col[w]);
                            } else {
                                const uint64_t* me = P.bits + static_cast<uint64_t>(i) * words;
                                for (int w = 0; w < words; ++w) h += __popcll(me[w] ^ col[w]);
                            }
                            const int T = __ldg(P.maxham + si + cz[g + k]);
                            m |= (h <= T ? 1u : 0u) << k;
                        }
                    }
                    m = bypass ? rm : (m & rm);
                    cnt += __popc(m);
                    uint32_t e = m;  // emitted for verification
                    if constexpr (W2 > 0) {
                        const uint32_t most = __reduce_max_sync(0xFFFFFFFFu, static_cast<uint32_t>(__popc(m)));
                        if (most > 8 && uniform && kmax == 32) {
                            uint32_t m2 = 0;
#pragma unroll 8
                            for (int k = 0; k < 32; ++k) {
                                const uint64_t* col = cb2 + (g + k) * W2;
                                int h = 0;
#pragma unroll
                                for (int w = 0; w < W2; ++w) h += __popcll(mine2[w] ^ col[w]);
                                m2 = __funnelshift_l(static_cast<uint32_t>(h + negT1), m2, 1);
                            }
                            e = m & __brev(m2);
                        } else if (most > 0) {
                            uint32_t mm = m;
                            e = 0;
                            while (mm) {
                                const int k = __ffs(mm) - 1;
                                mm &= mm - 1;
                                const uint64_t* col = cb2 + (g + k) * W2;
                                int h = 0;
#pragma unroll
                                for (int w = 0; w < W2; ++w) h += __popcll(mine2[w] ^ col[w]);
                                const int T = uniform ? -negT1 - 1 : __ldg(P.maxham + si + cz[g + k]);
                                e |= (h <= T ? 1u : 0u) << k;
                            }
                        }
                    }
                    if (__any_sync(0xFFFFFFFFu, e != 0)) emit_group(e, gbase, i, q, qlen, P, lane);
                }
            }
            __syncthreads();  // stage buffer free for the TMA issued next iteration
        }
        if (valid && cnt) atomicAdd(P.rowcnt + (i - P.row_begin), cnt);
        if (P.item_counts) P.item_counts[item * kRowTile + tid] = cnt;
        __syncthreads();  // s_item / s_tile / stage buffers are rewritten next item
    }
    if (qlen) warp_flush(q, qlen, P, lane);
}

// ======================================================= K2b: saturated rows
struct RescanParams {
    const uint64_t* bits;
    const uint32_t* sizes;
    const int32_t* maxham;
    const uint32_t* wstart;
    const uint32_t* rowcnt;
    const uint32_t* item_counts;  // per (item, row-in-tile) survivors, or null
    const uint64_t* item_base;    // per tile
    const uint32_t* tile_col_lo;
    uint32_t* jstar;              // capacity-th survivor column per row (row - row_begin)
    uint32_t row_begin, row_end;
    uint32_t capacity;
    int64_t cutoff;
    int words;
    int bypass_all;
    uint32_t tile_rows;           // rows per work item (128, or 256 for the CTA-pair filter)
    int maxham_len;
    const uint16_t* tile_counts;  // per (item, tile, part, row) survivors (tcgen05 filter), or null
    uint32_t tiles_per_item, tile_cols, tile_parts;
    const uint32_t* sat_list;     // rows (row - row_begin) whose count reaches the capacity
    const unsigned long long* sat_count;
};

// Saturated rows into a list (coalesced count reads, one atomic per warp), so
// the rescan runs one warp per listed row: no per-row scan of the whole shard
// (a chain of dependent loads per warp) when few or no rows saturate.
__global__ void find_saturated(const uint32_t* rowcnt, uint32_t nrows, uint32_t capacity, uint32_t* list,
                               Control* ctl) {
    const int lane = threadIdx.x & 31;
    for (uint32_t base = (blockIdx.x * blockDim.x + threadIdx.x) & ~31u; base < nrows;
         base += gridDim.x * blockDim.x) {
        const uint32_t r = base + lane;
        const bool sat = r < nrows && rowcnt[r] >= capacity;
        const uint32_t bal = __ballot_sync(0xFFFFFFFFu, sat);
        if (!bal) continue;
        unsigned long long at = 0;
        if (lane == 0) at = atomicAdd(&ctl->sat_rows, static_cast<unsigned long long>(__popc(bal)));
        at = __shfl_sync(0xFFFFFFFFu, at, 0);
        if (sat) list[at + __popc(bal & ((1u << lane) - 1u))] = r;
    }
}

constexpr int kRescanLut = 4096;  // maxham[] entries staged in shared memory

__device__ __forceinline__ uint32_t warp_inclusive_sum(uint32_t v, int lane) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t u = __shfl_up_sync(0xFFFFFFFFu, v, o);
        if (lane >= o) v += u;
    }
    return v;
}

// One warp per row whose survivor count reaches the capacity: locate the
// capacity-th survivor in window order (the reference's saturation point,
// src/parallel_join.cpp:83-94).  With per-item counts from the filter only the
// single 4096-column chunk holding it is rescanned; 128 columns per step.
__global__ void __launch_bounds__(256) rescan_saturated(RescanParams P) {
    __shared__ int32_t lut[kRescanLut];
    const bool lut_smem = P.maxham_len <= kRescanLut;
    if (lut_smem)
        for (int k = threadIdx.x; k < P.maxham_len; k += blockDim.x) lut[k] = P.maxham[k];
    __syncthreads();
    const int32_t* maxham = lut_smem ? lut : P.maxham;
    const int lane = threadIdx.x & 31;
    const uint32_t warps = (gridDim.x * blockDim.x) >> 5;
    const uint32_t nsat = static_cast<uint32_t>(*P.sat_count);
    for (uint32_t idx = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; idx < nsat; idx += warps) {
        const uint32_t r = P.sat_list[idx];
        const uint32_t i = P.row_begin + r;
        const uint32_t si = P.sizes[i];
        const uint32_t j0 = P.wstart[si];
        if (P.bypass_all || static_cast<int64_t>(si) > P.cutoff) {
            if (lane == 0) P.jstar[r] = j0 + P.capacity - 1;
            continue;
        }
        uint32_t start = j0, stop = i, seen = 0;
        if (P.item_counts) {
            // the work item (then the filter tile) holding the capacity-th
            // survivor: 32 items (tiles) per step, one per lane, located by a
            // warp prefix sum and a ballot instead of a chain of dependent loads
            const uint32_t tile = r / P.tile_rows, t = r % P.tile_rows;
            const uint64_t ib = P.item_base[tile], ie = P.item_base[tile + 1];
            for (uint64_t base = ib; base < ie; base += 32) {
                const uint64_t it = base + lane;
                const uint32_t cc = it < ie ? P.item_counts[it * P.tile_rows + t] : 0u;
                const uint32_t inc = warp_inclusive_sum(cc, lane);
                const uint32_t hit = __ballot_sync(0xFFFFFFFFu, seen + inc >= P.capacity);
                if (!hit) {
                    seen += __shfl_sync(0xFFFFFFFFu, inc, 31);
                    continue;
                }
                const int L = __ffs(hit) - 1;
                seen += __shfl_sync(0xFFFFFFFFu, inc - cc, L);
                const uint64_t itL = base + static_cast<uint64_t>(L);
                const uint32_t c0 = P.tile_col_lo[tile] + static_cast<uint32_t>(itL - ib) * kColChunk;
                start = max(j0, c0);
                stop = min(i, c0 + kColChunk);
                if (P.tile_counts) {  // narrow to the filter tile holding it (tiles_per_item <= 32)
                    uint32_t tc = 0;
                    if (static_cast<uint32_t>(lane) < P.tiles_per_item)
                        for (uint32_t pp = 0; pp < P.tile_parts; ++pp)
                            tc += P.tile_counts[((itL * P.tiles_per_item + lane) * 4 + pp) * P.tile_rows + t];
                    const uint32_t inc2 = warp_inclusive_sum(tc, lane);
                    // (slots past the item's last processed tile are not written, but
                    // they only follow the crossing lane, so no prefix before it sees them)
                    const uint32_t hit2 = __ballot_sync(
                        0xFFFFFFFFu, static_cast<uint32_t>(lane) < P.tiles_per_item && seen + inc2 >= P.capacity);
                    if (hit2) {
                        const int L2 = __ffs(hit2) - 1;
                        seen += __shfl_sync(0xFFFFFFFFu, inc2 - tc, L2);
                        start = max(j0, c0 + static_cast<uint32_t>(L2) * P.tile_cols);
                        stop = min(stop, c0 + static_cast<uint32_t>(L2 + 1) * P.tile_cols);
                    }
                }
                break;
            }
        }
        uint64_t me[kMaxInlineWords];
        const int words = min(P.words, kMaxInlineWords);
        for (int w = 0; w < words; ++w) me[w] = __ldg(P.bits + static_cast<uint64_t>(i) * P.words + w);
        // 128 columns per step in four lane-contiguous groups of 32 (coalesced
        // sketch and size loads: a group reads 32 consecutive sketch rows)
        for (uint32_t jb = start; jb < stop; jb += 128) {
            uint32_t bal[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const uint32_t j = jb + q * 32 + lane;
                bool surv = false;
                if (j < stop) {
                    const uint32_t sj = __ldg(P.sizes + j);
                    int h = 0;
                    if (P.words == 2) {
                        const ulonglong2 o = __ldg(reinterpret_cast<const ulonglong2*>(P.bits) + j);
                        h = __popcll(me[0] ^ o.x) + __popcll(me[1] ^ o.y);
                    } else if (P.words == 1) {
                        h = __popcll(me[0] ^ __ldg(P.bits + j));
                    } else if (P.words <= kMaxInlineWords) {
                        const uint64_t* o = P.bits + static_cast<uint64_t>(j) * P.words;
                        for (int w = 0; w < words; ++w) h += __popcll(me[w] ^ __ldg(o + w));
                    } else {
                        const uint64_t* o = P.bits + static_cast<uint64_t>(j) * P.words;
                        const uint64_t* mi = P.bits + static_cast<uint64_t>(i) * P.words;
                        for (int w = 0; w < P.words; ++w) h += __popcll(__ldg(mi + w) ^ __ldg(o + w));
                    }
                    surv = h <= maxham[si + sj];
                }
                bal[q] = __ballot_sync(0xFFFFFFFFu, surv);
            }
            bool done = false;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const uint32_t pc = __popc(bal[q]);
                if (!done && seen + pc >= P.capacity) {
                    uint32_t b2 = bal[q];  // drop the first (need-1) survivors of this group
                    for (uint32_t k = P.capacity - seen; k > 1; --k) b2 &= b2 - 1;
                    if (lane == 0) P.jstar[r] = jb + q * 32 + static_cast<uint32_t>(__ffs(b2) - 1);
                    done = true;
                }
                if (!done) seen += pc;
            }
            if (done) break;
        }
    }
}

// Counter reduction: per row, the reference's buffered/bypassed bookkeeping
// reconstructed from (window, survivors, capacity-th survivor position).
struct CountParams {
    const uint32_t* sizes;
    const uint32_t* wstart;
    const uint32_t* rowcnt;
    const uint32_t* jstar;
    Control* ctl;
    uint32_t row_begin, row_end;
    uint32_t capacity;
    int bitmap_enabled;
    int naive;
};

__global__ void reduce_counters(CountParams P) {
    unsigned long long tested = 0, pruned = 0, verified = 0, sat = 0;
    for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < P.row_end - P.row_begin;
         r += gridDim.x * blockDim.x) {
        const uint32_t i = P.row_begin + r;
        const uint32_t j0 = P.naive ? 0u : P.wstart[P.sizes[i]];
        const uint32_t w = j0 < i ? i - j0 : 0u;
        if (P.naive) {
            verified += w;
            continue;
        }
        const uint32_t s = P.rowcnt[r];
        if (s < P.capacity) {
            if (P.bitmap_enabled) {
                tested += w;
                pruned += w - s;
            }
            verified += s;
        } else {
            const uint32_t js = P.jstar[r];
            const uint32_t t = js - j0 + 1;
            if (P.bitmap_enabled) {
                tested += t;
                pruned += t - P.capacity;
            }
            verified += P.capacity + (i - js - 1);
            sat += 1;
        }
    }
    for (int o = 16; o > 0; o >>= 1) {
        tested += __shfl_down_sync(0xFFFFFFFFu, tested, o);
        pruned += __shfl_down_sync(0xFFFFFFFFu, pruned, o);
        verified += __shfl_down_sync(0xFFFFFFFFu, verified, o);
        sat += __shfl_down_sync(0xFFFFFFFFu, sat, o);
    }
    if ((threadIdx.x & 31) == 0) {
        if (tested) atomicAdd(&P.ctl->tested, tested);
        if (pruned) atomicAdd(&P.ctl->pruned, pruned);
        if (verified) atomicAdd(&P.ctl->verified, verified);
        if (sat) atomicAdd(&P.ctl->saturated, sat);
    }
}

// ================================================================ K3: verify
// Required overlap of a pair for the similarity functions the NAIVE join
// accepts (reference src/similarity.cpp:93-115).  Jaccard, Dice and Overlap
// depend on |r|+|s| only and come from the host-exact table minov[|r|+|s|];
// Cosine depends on |r|*|s| and is computed here with the reference's own
// 128-bit arithmetic: ceil(isqrt_ceil(p^2 |r| |s|) / q)
// (src/similarity.cpp:103-107, src/rational.cpp:43-71).
struct SimNeed {
    const int32_t* minov;  // minov[|r|+|s|]
    int cosine;            // 1: Cosine, minov unused
    long long cp, cq;      // reduced threshold p/q (Cosine)
};

__device__ __forceinline__ uint64_t isqrt_floor_u128(unsigned __int128 v) {
    // Newton from a double estimate, then exact correction (src/rational.cpp:51-65)
    if (v == 0) return 0;
    const double est = static_cast<double>(static_cast<uint64_t>(v >> 64)) * 18446744073709551616.0 +
                       static_cast<double>(static_cast<uint64_t>(v));
    unsigned __int128 x = static_cast<unsigned __int128>(sqrt(est));
    if (x == 0) x = 1;
    for (int it = 0; it < 6; ++it) {
        const unsigned __int128 nx = (x + v / x) >> 1;
        if (nx == x) break;
        x = nx;
    }
    while (x * x > v) --x;
    while ((x + 1) * (x + 1) <= v) ++x;
    return static_cast<uint64_t>(x);
}

__device__ __forceinline__ int32_t need_overlap(const SimNeed& N, uint32_t na, uint32_t nb) {
    if (!N.cosine) return N.minov[na + nb];
    unsigned __int128 target = static_cast<unsigned __int128>(N.cp) * static_cast<unsigned __int128>(N.cp);
    target *= static_cast<unsigned __int128>(na) * nb;
    const uint64_t root = target == 0 ? 0 : isqrt_floor_u128(target - 1) + 1;
    const __int128 q = N.cq;
    const long long v = static_cast<long long>((static_cast<__int128>(root) + q - 1) / q);
    return static_cast<int32_t>(max(1ll, min(v, 0x7FFFFFFFll)));
}

struct VerifyParams {
    const uint32_t* tokens;
    const uint64_t* offsets;
    SimNeed need;             // required overlap per (|r|, |s|)
    const uint2* surv;
    const unsigned long long* count_ptr;  // survivors emitted by K2 (device memory)
    unsigned long long count_cap;         // survivor buffer capacity
    unsigned long long* res_keys;  // (j << 32) | i
    uint32_t* res_ov;
    unsigned long long res_cap;
    Control* ctl;
    const uint64_t* bits2;    // level-2 Xor sketches (n x w2 words), or null
    const int32_t* maxham;    // maxham[|r|+|s|] (with bits2)
    int w2;
    int warp_mode;            // 1: warp per pair when the survivors are few; 2: always
    const uint64_t* bits3;    // level-3 512-bit Xor sketches (dense joins), or null
    uint32_t l3_min_sum;      // level 3 is tested when |r| + |s| >= this
};

// One thread per surviving pair: branch-free sorted merge with the
// reference's early exit (src/similarity.cpp:168-185).  A match's overlap is
// exact because the exit only fires on pairs that cannot reach minov.
// With bits2, a pair is first re-tested against the wider level-2 Xor sketch
// (the same exact bound, reference src/bitmap.cpp:125-143, at 64*w2 bits):
// level-1 survivors the wider sketch rejects cannot match and skip the merge.
// Survivor counts up to this are verified one warp per pair: the merge of a
// thread-per-pair kernel is a chain of ~|r|+|s| dependent loads, so a launch
// with few survivors costs that chain's latency (~30 us at C2's 86-token
// records) however few pairs it has.  A warp instead takes 32 tokens of the
// shorter record at a time, each lane binary-searches its token in the
// longer one (independent searches, ~log2|s| loads deep), and the ballot
// counts the overlap.  On a match the overlap is the full intersection, the
// same exact value the merge produces; the early exit (overlap + tokens left
// < required) only ever stops non-matching pairs, as in the reference's
// verify (src/similarity.cpp:174-175).
constexpr unsigned long long kWarpVerifyMax = 1ull << 15;

template <int W2>
__device__ __forceinline__ void verify_warp_mode(const VerifyParams& P, unsigned long long count, int lane) {
    const unsigned long long nwarps = static_cast<unsigned long long>(gridDim.x) * (blockDim.x >> 5);
    const unsigned long long gw = static_cast<unsigned long long>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
    for (unsigned long long k = gw; k < count; k += nwarps) {
        const uint2 pr = P.surv[k];
        const uint32_t j = pr.x, i = pr.y;
        const uint64_t ab = P.offsets[j], ae = P.offsets[j + 1];
        const uint64_t bb = P.offsets[i], be = P.offsets[i + 1];
        const uint32_t na = static_cast<uint32_t>(ae - ab), nb = static_cast<uint32_t>(be - bb);
        if constexpr (W2 > 0) {
            int h = 0;
            if (lane < W2) h = __popcll(__ldg(P.bits2 + static_cast<uint64_t>(j) * W2 + lane) ^
                                        __ldg(P.bits2 + static_cast<uint64_t>(i) * W2 + lane));
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) h += __shfl_xor_sync(0xFFFFFFFFu, h, o);
            if (h > P.maxham[na + nb]) continue;  // rejected by the level-2 sketch (warp-uniform)
        }
        const int32_t need = need_overlap(P.need, na, nb);
        const bool a_short = na <= nb;
        const uint32_t* S = P.tokens + (a_short ? ab : bb);
        const uint32_t* L = P.tokens + (a_short ? bb : ab);
        const uint32_t ns = a_short ? na : nb, nl = a_short ? nb : na;
        int32_t o = 0;
        for (uint32_t base = 0; base < ns; base += 32) {
            bool hit = false;
            if (base + lane < ns) {
                const uint32_t t = __ldg(S + base + lane);
                uint32_t lo = 0, len = nl;  // lower_bound of t in L
                while (len > 0) {
                    const uint32_t half = len >> 1;
                    if (__ldg(L + lo + half) < t) {
                        lo += half + 1;
                        len -= half + 1;
                    } else {
                        len = half;
                    }
                }
                hit = lo < nl && __ldg(L + lo) == t;
            }
            o += __popc(__ballot_sync(0xFFFFFFFFu, hit));
            const uint32_t left = ns - min(ns, base + 32);
            if (o + static_cast<int32_t>(left) < need) break;
        }
        const bool matched = o >= need;
        if (lane == 0) {
            atomicAdd(&P.ctl->verify_bytes, 4ull * (na + nb) + (matched ? 16ull : 0ull));
            if (matched) {
                const unsigned long long slot = atomicAdd(&P.ctl->results, 1ull);
                if (slot < P.res_cap) {
                    P.res_keys[slot] = (static_cast<unsigned long long>(j) << 32) | i;
                    P.res_ov[slot] = static_cast<uint32_t>(o);
                }
            }
        }
    }
}

// Chunked sorted-list intersection for the thread-per-pair verify: each
// round loads the next kVerifyChunk tokens of both records (independent
// loads, one memory round trip instead of one per merge step), counts the
// equal pairs among the tokens <= m = min(last of each chunk) with an all-
// pairs compare in registers, and consumes exactly the tokens <= m from each
// side -- the same positions a step-by-step merge reaches, so the overlap of
// every pair that runs to the end is the exact intersection.  The early exit
// (overlap + min(tokens left) < required, src/similarity.cpp:174-175) is
// tested once per round; it only ever stops pairs that cannot match.
// Positions past a record's end hold sentinels (0xFFFFFFFF in A's chunk,
// 0xFFFFFFFE in B's) that never compare equal to each other and sort above
// every smaller token; a chunk whose last real token is >= 0xFFFFFFFE (token
// ids the sentinels could alias) finishes on the step-by-step merge instead.
#ifndef SSJB_VERIFY_CHUNK
#define SSJB_VERIFY_CHUNK 8
#endif
constexpr int kVerifyChunk = SSJB_VERIFY_CHUNK;

__device__ __forceinline__ void step_merge(const uint32_t* A, uint32_t na, const uint32_t* B, uint32_t nb,
                                           int32_t need, uint32_t& ia, uint32_t& ib, int32_t& o) {
    while (ia < na && ib < nb) {
        const int32_t rest = static_cast<int32_t>(min(na - ia, nb - ib));
        if (o + rest < need) break;
        const uint32_t x = __ldg(A + ia), y = __ldg(B + ib);
        o += x == y;
        ia += x <= y;
        ib += y <= x;
    }
}

__device__ __forceinline__ void chunk_merge(const uint32_t* A, uint32_t na, const uint32_t* B, uint32_t nb,
                                            int32_t need, uint32_t& ia, uint32_t& ib, int32_t& o) {
    constexpr int Q = kVerifyChunk > 0 ? kVerifyChunk : 1;
    while (ia < na && ib < nb) {
        if (o + static_cast<int32_t>(min(na - ia, nb - ib)) < need) return;
        uint32_t qa[Q], qb[Q];
        bool alias = false;
#pragma unroll
        for (int k = 0; k < Q; ++k) {
            const bool va = ia + k < na, vb = ib + k < nb;
            qa[k] = va ? __ldg(A + ia + k) : 0xFFFFFFFFu;
            qb[k] = vb ? __ldg(B + ib + k) : 0xFFFFFFFEu;
            alias |= (va && qa[k] >= 0xFFFFFFFEu) || (vb && qb[k] >= 0xFFFFFFFEu);
        }
        if (alias) break;
        const uint32_t m = min(qa[Q - 1], qb[Q - 1]);
        uint32_t ca = 0, cb = 0;
        int32_t hits = 0;
#pragma unroll
        for (int k = 0; k < Q; ++k) {
            ca += qa[k] <= m;
            cb += qb[k] <= m;
#pragma unroll
            for (int l = 0; l < Q; ++l) hits += qa[k] == qb[l];
        }
        // (an equal pair above m cannot exist: it would need a token above the
        // last token of a full chunk, within that chunk)
        o += hits;
        ia = min(ia + ca, na);
        ib = min(ib + cb, nb);
    }
    step_merge(A, na, B, nb, need, ia, ib, o);
}

template <int W2>
__global__ void verify_pairs(VerifyParams P) {
    const int lane = threadIdx.x & 31;
    const unsigned long long count = min(*P.count_ptr, P.count_cap);
    // warp_mode 2: every pair one warp (the head-overlap survivors: long records,
    // where one lane's merge chain of thousands of tokens paces its warp)
    if ((count <= kWarpVerifyMax && P.warp_mode) || P.warp_mode == 2) {
        verify_warp_mode<W2>(P, count, lane);
        return;
    }
    // result slots are reserved once per block and iteration (one global
    // atomic for the block's matches, not one per warp: C3 matches 2e8 of its
    // 3.3e8 survivors, and same-address atomics serialise in L2); the verify
    // byte count is summed in registers and added once per warp at the end
    __shared__ uint32_t s_cnt[2][32];
    __shared__ unsigned long long s_base[2];
    const int warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    unsigned long long vbytes = 0;
    int par = 0;
    const unsigned long long stride = static_cast<unsigned long long>(gridDim.x) * blockDim.x;
    for (unsigned long long base = static_cast<unsigned long long>(blockIdx.x) * blockDim.x; base < count;
         base += stride, par ^= 1) {
        const unsigned long long k = base + threadIdx.x;
        bool matched = false, merged = false;
        uint32_t j = 0, i = 0, ov = 0;
        if (k < count) {
            const uint2 pr = P.surv[k];
            j = pr.x;
            i = pr.y;
            const uint64_t ab = P.offsets[j], ae = P.offsets[j + 1];
            const uint64_t bb = P.offsets[i], be = P.offsets[i + 1];
            const uint32_t na = static_cast<uint32_t>(ae - ab), nb = static_cast<uint32_t>(be - bb);
            const int32_t need = need_overlap(P.need, na, nb);
            const uint32_t* A = P.tokens + ab;
            const uint32_t* B = P.tokens + bb;
            uint32_t ia = 0, ib = 0;
            int32_t o = 0;
            bool l2_ok = true;
            if constexpr (W2 > 0) {
                const ulonglong2* sj = reinterpret_cast<const ulonglong2*>(P.bits2 + static_cast<uint64_t>(j) * W2);
                const ulonglong2* si = reinterpret_cast<const ulonglong2*>(P.bits2 + static_cast<uint64_t>(i) * W2);
                int h = 0;
#pragma unroll
                for (int w = 0; w < W2 / 2; ++w) {
                    const ulonglong2 x = __ldg(sj + w), y = __ldg(si + w);
                    h += __popcll(x.x ^ y.x) + __popcll(x.y ^ y.y);
                }
                l2_ok = h <= P.maxham[na + nb];
                if (!l2_ok) ia = na;  // skip the merge
            }
            if (l2_ok && P.bits3 && na + nb >= P.l3_min_sum) {
                // level 3: the wider sketch still discriminates where the 256-bit
                // one has saturated (large records); same sound bound
                const ulonglong2* sj = reinterpret_cast<const ulonglong2*>(P.bits3 + static_cast<uint64_t>(j) * 8);
                const ulonglong2* si = reinterpret_cast<const ulonglong2*>(P.bits3 + static_cast<uint64_t>(i) * 8);
                int h = 0;
#pragma unroll
                for (int w = 0; w < 4; ++w) {
                    const ulonglong2 x = __ldg(sj + w), y = __ldg(si + w);
                    h += __popcll(x.x ^ y.x) + __popcll(x.y ^ y.y);
                }
                if (h > P.maxham[na + nb]) {
                    l2_ok = false;
                    ia = na;  // skip the merge
                }
            }
            merged = l2_ok;
            if constexpr (kVerifyChunk > 0) chunk_merge(A, na, B, nb, need, ia, ib, o);
            else step_merge(A, na, B, nb, need, ia, ib, o);
            matched = o >= need;
            ov = static_cast<uint32_t>(o);
        }
        // algorithmic traffic: both token lists plus the 16-byte result record
        if (merged)
            vbytes += 4ull * (P.offsets[j + 1] - P.offsets[j] + P.offsets[i + 1] - P.offsets[i]) + (matched ? 16 : 0);
        const uint32_t bal = __ballot_sync(0xFFFFFFFFu, matched);
        if (lane == 0) s_cnt[par][warp] = __popc(bal);
        __syncthreads();
        if (threadIdx.x == 0) {
            unsigned long long tot = 0;
            for (int w = 0; w < nwarps; ++w) tot += s_cnt[par][w];
            s_base[par] = tot ? atomicAdd(&P.ctl->results, tot) : 0ull;
        }
        __syncthreads();
        if (bal) {
            unsigned long long slot = s_base[par];
            for (int w = 0; w < warp; ++w) slot += s_cnt[par][w];
            slot += __popc(bal & ((1u << lane) - 1u));
            if (matched && slot < P.res_cap) {
                P.res_keys[slot] = (static_cast<unsigned long long>(j) << 32) | i;
                P.res_ov[slot] = ov;
            }
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) vbytes += __shfl_down_sync(0xFFFFFFFFu, vbytes, o);
    if (lane == 0 && vbytes) atomicAdd(&P.ctl->verify_bytes, vbytes);
}

// ===================================================== K3 (RS): naive R x S
// NAIVE RS-join (reference src/join.cpp:110-121): every (r, s) in
// [r_begin, r_end) x [0, nS) is merged, no filter.  Pair index k enumerates
// the block row-major, k -> (r = k / nS, s = k % nS), so a warp shares one
// r-record (broadcast loads) and walks consecutive, size-sorted s-records;
// a contiguous k range yields keys (r << 32 | s) in one contiguous key range,
// so runs of consecutive launches concatenate in canonical order.
struct VerifyRsParams {
    const uint32_t* ta;
    const uint64_t* oa;   // R
    const uint32_t* tb;
    const uint64_t* ob;   // S
    unsigned long long nS;
    unsigned long long k0, k1;
    unsigned long long r_begin;
    SimNeed need;
    unsigned long long* res_keys;  // (r << 32) | s
    uint32_t* res_ov;
    unsigned long long res_cap;
    Control* ctl;
};

__global__ void verify_rs(VerifyRsParams P) {
    const int lane = threadIdx.x & 31;
    const unsigned long long stride = static_cast<unsigned long long>(gridDim.x) * blockDim.x;
    for (unsigned long long base = P.k0 + static_cast<unsigned long long>(blockIdx.x) * blockDim.x; base < P.k1;
         base += stride) {
        const unsigned long long k = base + threadIdx.x;
        bool matched = false;
        uint32_t r = 0, sidx = 0, ov = 0;
        unsigned long long vb = 0;
        if (k < P.k1) {
            r = static_cast<uint32_t>(P.r_begin + k / P.nS);
            sidx = static_cast<uint32_t>(k % P.nS);
            const uint64_t ab = P.oa[r], ae = P.oa[r + 1];
            const uint64_t bb = P.ob[sidx], be = P.ob[sidx + 1];
            const uint32_t na = static_cast<uint32_t>(ae - ab), nb = static_cast<uint32_t>(be - bb);
            const int32_t need = need_overlap(P.need, na, nb);
            const uint32_t* A = P.ta + ab;
            const uint32_t* B = P.tb + bb;
            uint32_t ia = 0, ib = 0;
            int32_t o = 0;
            while (ia < na && ib < nb) {  // early exit of src/similarity.cpp:174-175
                const int32_t rest = static_cast<int32_t>(min(na - ia, nb - ib));
                if (o + rest < need) break;
                const uint32_t x = __ldg(A + ia), y = __ldg(B + ib);
                o += x == y;
                ia += x <= y;
                ib += y <= x;
            }
            matched = o >= need;
            ov = static_cast<uint32_t>(o);
            vb = 4ull * (na + nb) + (matched ? 16 : 0);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) vb += __shfl_down_sync(0xFFFFFFFFu, vb, o);
        if (lane == 0 && vb) atomicAdd(&P.ctl->verify_bytes, vb);
        const uint32_t bal = __ballot_sync(0xFFFFFFFFu, matched);
        if (bal) {
            unsigned long long slot = 0;
            if (lane == 0) slot = atomicAdd(&P.ctl->results, static_cast<unsigned long long>(__popc(bal)));
            slot = __shfl_sync(0xFFFFFFFFu, slot, 0) + __popc(bal & ((1u << lane) - 1u));
            if (matched && slot < P.res_cap) {
                P.res_keys[slot] = (static_cast<unsigned long long>(r) << 32) | sidx;
                P.res_ov[slot] = ov;
            }
        }
    }
}

// ================================================ K2/K3 (RS): filtered R x S
// NAIVE RS-join through the Bitmap Filter (round 2): the reference verifies
// every (r, s) (src/join.cpp:110-121); here only the pairs that survive a
// length window (S is size-sorted: per R size an S index range) and the
// b-bit Xor sketch bound popcount(b_r ^ b_s) <= maxham[|r|+|s|] are merged.
// Both tests are sound for every similarity function whose required overlap
// depends on |r|+|s| (Jaccard, Dice, Overlap), so the matches -- and the
// NAIVE counters, candidates = verified = |R||S| -- are unchanged.
struct RsFilterParams {
    const uint64_t* bits_r;    // R sketches, words per row
    const uint64_t* bits_s;    // S sketches
    const uint32_t* sizes_r;
    const uint32_t* sizes_s;
    const uint32_t* s_lo;      // per R size: first S index of the length window
    const uint32_t* s_hi;      // per R size: end of the window
    const int32_t* maxham;     // maxham[|r| + |s|]
    const uint2* items;        // (R row tile, S column chunk of kColChunk)
    uint32_t r_begin, r_end, n_s;
    int words;                 // 1 or 2
    uint2* surv;               // (s, r)
    unsigned long long surv_cap, surv_soft;
    unsigned long long item_begin, item_end;
    Control* ctl;
};

constexpr int kRsCols = 1024;  // S columns staged in shared memory per step

__global__ void __launch_bounds__(kRowTile) rs_filter(RsFilterParams P) {
    __shared__ uint64_t s_bits[kRsCols * 2];
    __shared__ uint32_t s_size[kRsCols];
    __shared__ unsigned long long s_item;
    const int lane = threadIdx.x & 31;
    for (;;) {
        if (threadIdx.x == 0) s_item = claim_item(P.ctl, P.item_begin, P.item_end, P.surv_soft);
        __syncthreads();
        const unsigned long long it = s_item;
        __syncthreads();
        if (it >= P.item_end) break;
        const uint2 w = P.items[it];
        const uint32_t i = P.r_begin + w.x * kRowTile + threadIdx.x;
        const bool valid = i < P.r_end;
        uint32_t si = 0, lo = 0, hi = 0;
        uint64_t m0 = 0, m1 = 0;
        if (valid) {
            si = P.sizes_r[i];
            lo = P.s_lo[si];
            hi = P.s_hi[si];
            m0 = P.bits_r[static_cast<uint64_t>(i) * P.words];
            if (P.words == 2) m1 = P.bits_r[static_cast<uint64_t>(i) * 2 + 1];
        }
        const uint32_t c0 = w.y * kColChunk, c1 = min(c0 + kColChunk, P.n_s);
        for (uint32_t cb = c0; cb < c1; cb += kRsCols) {
            const uint32_t ce = min(cb + kRsCols, c1);
            for (uint32_t k = threadIdx.x; k < ce - cb; k += blockDim.x) {
                s_size[k] = P.sizes_s[cb + k];
                s_bits[2 * k] = P.bits_s[static_cast<uint64_t>(cb + k) * P.words];
                s_bits[2 * k + 1] = P.words == 2 ? P.bits_s[static_cast<uint64_t>(cb + k) * 2 + 1] : 0ull;
            }
            __syncthreads();
            const uint32_t jl = valid ? max(lo, cb) : ce, jh = valid ? min(hi, ce) : ce;
            uint32_t wl = jl, wh = jh;  // warp-uniform bounds
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                wl = min(wl, __shfl_xor_sync(0xFFFFFFFFu, wl, o));
                wh = max(wh, __shfl_xor_sync(0xFFFFFFFFu, wh, o));
            }
            for (uint32_t j = wl; j < wh; ++j) {
                const uint32_t k = j - cb;
                const int h = __popcll(m0 ^ s_bits[2 * k]) + __popcll(m1 ^ s_bits[2 * k + 1]);
                const bool pass = j >= jl && j < jh && h <= __ldg(P.maxham + si + s_size[k]);
                const uint32_t bal = __ballot_sync(0xFFFFFFFFu, pass);
                if (!bal) continue;
                unsigned long long base = 0;
                if (lane == __ffs(bal) - 1) base = atomicAdd(&P.ctl->survivors, static_cast<unsigned long long>(__popc(bal)));
                base = __shfl_sync(0xFFFFFFFFu, base, __ffs(bal) - 1) + __popc(bal & ((1u << lane) - 1u));
                if (pass && base < P.surv_cap) P.surv[base] = make_uint2(j, i);
            }
            __syncthreads();
        }
    }
}

// Exact verification of filtered RS survivors (s, r): thread per pair, the
// merge with early exit of reference src/similarity.cpp:168-185; matches
// keyed (r << 32) | s.
struct VerifyRsPairsParams {
    const uint32_t* ta;
    const uint64_t* oa;   // R
    const uint32_t* tb;
    const uint64_t* ob;   // S
    SimNeed need;
    const uint2* surv;
    const unsigned long long* count_ptr;
    unsigned long long count_cap;
    unsigned long long* res_keys;
    uint32_t* res_ov;
    unsigned long long res_cap;
    Control* ctl;
};

__global__ void verify_rs_pairs(VerifyRsPairsParams P) {
    const int lane = threadIdx.x & 31;
    const unsigned long long count = min(*P.count_ptr, P.count_cap);
    const unsigned long long stride = static_cast<unsigned long long>(gridDim.x) * blockDim.x;
    for (unsigned long long base = static_cast<unsigned long long>(blockIdx.x) * blockDim.x; base < count;
         base += stride) {
        const unsigned long long k = base + threadIdx.x;
        bool matched = false;
        uint32_t r = 0, sidx = 0, ov = 0;
        unsigned long long vb = 0;
        if (k < count) {
            const uint2 pr = P.surv[k];
            sidx = pr.x;
            r = pr.y;
            const uint64_t ab = P.oa[r], ae = P.oa[r + 1];
            const uint64_t bb = P.ob[sidx], be = P.ob[sidx + 1];
            const uint32_t na = static_cast<uint32_t>(ae - ab), nb = static_cast<uint32_t>(be - bb);
            const int32_t need = need_overlap(P.need, na, nb);
            const uint32_t* A = P.ta + ab;
            const uint32_t* B = P.tb + bb;
            uint32_t ia = 0, ib = 0;
            int32_t o = 0;
            while (ia < na && ib < nb) {
                const int32_t rest = static_cast<int32_t>(min(na - ia, nb - ib));
                if (o + rest < need) break;
                const uint32_t x = __ldg(A + ia), y = __ldg(B + ib);
                o += x == y;
                ia += x <= y;
                ib += y <= x;
            }
            matched = o >= need;
            ov = static_cast<uint32_t>(o);
            vb = 4ull * (na + nb) + (matched ? 16 : 0);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) vb += __shfl_down_sync(0xFFFFFFFFu, vb, o);
        if (lane == 0 && vb) atomicAdd(&P.ctl->verify_bytes, vb);
        const uint32_t bal = __ballot_sync(0xFFFFFFFFu, matched);
        if (bal) {
            unsigned long long slot = 0;
            if (lane == 0) slot = atomicAdd(&P.ctl->results, static_cast<unsigned long long>(__popc(bal)));
            slot = __shfl_sync(0xFFFFFFFFu, slot, 0) + __popc(bal & ((1u << lane) - 1u));
            if (matched && slot < P.res_cap) {
                P.res_keys[slot] = (static_cast<unsigned long long>(r) << 32) | sidx;
                P.res_ov[slot] = ov;
            }
        }
    }
}

// ============================================================ K4: radix sort
constexpr int kSortThreads = 256;
constexpr int kSortItems = 8;                       // keys per thread per tile
constexpr int kSortTile = kSortThreads * kSortItems;  // 2048 keys per tile

// Digit histogram of each tile: hist[digit * ntiles + tile].
__global__ void __launch_bounds__(kSortThreads) radix_hist(const unsigned long long* keys, unsigned long long n,
                                                          int shift, uint32_t* hist, uint32_t ntiles) {
    __shared__ uint32_t h[256];
    h[threadIdx.x] = 0;
    __syncthreads();
    const unsigned long long t0 = static_cast<unsigned long long>(blockIdx.x) * kSortTile;
    for (int k = 0; k < kSortItems; ++k) {
        unsigned long long idx = t0 + k * kSortThreads + threadIdx.x;
        if (idx < n) atomicAdd(&h[(keys[idx] >> shift) & 255], 1u);
    }
    __syncthreads();
    hist[threadIdx.x * ntiles + blockIdx.x] = h[threadIdx.x];
}

// Exclusive scan of a u32 array in place, three phases (block sums, a
// single-block scan of the sums, add-back).  Lengths here are 256 * ntiles.
constexpr int kScanBlock = 1024;

__device__ __forceinline__ uint32_t block_exclusive_scan(uint32_t v, uint32_t* tmp, uint32_t& total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t y = __shfl_up_sync(0xFFFFFFFFu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) tmp[warp] = x;
    __syncthreads();
    if (warp == 0) {
        uint32_t s = lane < static_cast<int>(blockDim.x >> 5) ? tmp[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t y = __shfl_up_sync(0xFFFFFFFFu, s, o);
            if (lane >= o) s += y;
        }
        tmp[lane] = s;
    }
    __syncthreads();
    total = tmp[(blockDim.x >> 5) - 1];
    uint32_t prefix = warp ? tmp[warp - 1] : 0;
    __syncthreads();
    return prefix + x - v;
}

__global__ void __launch_bounds__(kScanBlock) scan_blocks(uint32_t* data, uint32_t n, uint32_t* block_sums) {
    __shared__ uint32_t tmp[32];
    const uint32_t idx = blockIdx.x * kScanBlock + threadIdx.x;
    const uint32_t v = idx < n ? data[idx] : 0;
    uint32_t total;
    const uint32_t ex = block_exclusive_scan(v, tmp, total);
    if (idx < n) data[idx] = ex;
    if (threadIdx.x == 0) block_sums[blockIdx.x] = total;
}

__global__ void __launch_bounds__(kScanBlock) scan_single(uint32_t* data, uint32_t n) {
    __shared__ uint32_t tmp[32];
    uint32_t carry = 0;
    for (uint32_t base = 0; base < n; base += kScanBlock) {
        const uint32_t idx = base + threadIdx.x;
        const uint32_t v = idx < n ? data[idx] : 0;
        uint32_t total;
        const uint32_t ex = block_exclusive_scan(v, tmp, total);
        if (idx < n) data[idx] = ex + carry;
        carry += total;
    }
}

__global__ void __launch_bounds__(kScanBlock) scan_add(uint32_t* data, uint32_t n, const uint32_t* block_sums) {
    const uint32_t idx = blockIdx.x * kScanBlock + threadIdx.x;
    if (idx < n) data[idx] += block_sums[blockIdx.x];
}

// Stable scatter of one tile: keys are ranked in tile order (round by round,
// warp-major inside a round) with __match_any_sync, so equal digits keep
// their relative order -- the LSD invariant.
__global__ void __launch_bounds__(kSortThreads) radix_scatter(const unsigned long long* keys_in, const uint32_t* vals_in,
                                                             unsigned long long* keys_out, uint32_t* vals_out,
                                                             unsigned long long n, int shift, const uint32_t* hist,
                                                             uint32_t ntiles) {
    constexpr int kWarps = kSortThreads / 32;
    __shared__ uint32_t base[256];
    __shared__ uint32_t wcount[kWarps][256];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    base[threadIdx.x] = hist[threadIdx.x * ntiles + blockIdx.x];
    const unsigned long long t0 = static_cast<unsigned long long>(blockIdx.x) * kSortTile;
    for (int round = 0; round < kSortItems; ++round) {
        for (int w = 0; w < kWarps; ++w) wcount[w][threadIdx.x] = 0;
        __syncthreads();
        const unsigned long long idx = t0 + static_cast<unsigned long long>(round) * kSortThreads + threadIdx.x;
        const bool ok = idx < n;
        unsigned long long key = ok ? keys_in[idx] : 0ull;
        const uint32_t d = ok ? static_cast<uint32_t>((key >> shift) & 255) : 256u + lane;  // unique dummy
        const uint32_t peers = __match_any_sync(0xFFFFFFFFu, d);
        const uint32_t rank = __popc(peers & ((1u << lane) - 1u));
        if (ok && rank == 0) wcount[warp][d] = __popc(peers);
        __syncthreads();
        // per digit: prefix over warps, then advance the running base
        {
            const uint32_t dd = threadIdx.x;
            uint32_t run = 0;
            for (int w = 0; w < kWarps; ++w) {
                uint32_t c = wcount[w][dd];
                wcount[w][dd] = run;
                run += c;
            }
            __syncthreads();
            if (ok) {
                const uint32_t pos = base[d] + wcount[warp][d] + rank;
                keys_out[pos] = key;
                vals_out[pos] = vals_in[idx];
            }
            __syncthreads();
            base[dd] += run;
        }
        __syncthreads();
    }
}

}  // namespace dev
}  // namespace ssjb
