// Tensor-core Bitmap Filter (K2, tcgen05 path).  Included by engine.cu.
//
// The xor/popcount bound is a dot product:  popcount(b_i ^ b_j) =
// pc_i + pc_j - 2 <b_i, b_j>.  So the filter for a 128-row x 128-column tile
// is one int8 GEMM.  Operands are the sketches expanded to one byte per bit
// (kernel expand_operands), K-major, in the tcgen05 core-matrix layout
// (8 rows x 16 bytes per 128-byte core matrix), with a 32-byte extension block:
//
//   A_i = [ bit_k(b_i) in {0,1}  (k < b) | 1, 1, 0 ... ]                  (u8)
//   B_j = [ 2*bit_k(b_j) in {0,2} (k < b) | -ceil(pc_j/2), -floor(pc_j/2), 0...] (s8)
//   D_ij = sum_k A_ik B_jk = 2 <b_i, b_j> - pc_j                          (s32, TMEM)
//
// survive  <=>  popcount <= T(|r_i|+|r_j|)  <=>  D_ij >= pc_i - T  -- exact
// integers throughout, identical to the POPC kernel and to reference
// src/bitmap.cpp:125-143.
//
// Warp roles (320 threads, one CTA per SM, persistent over work items):
//   warp 0      TMA producer: row tile A (once per item), column tiles B
//               + sizes (+ level-2 sketches) into an NS-stage ring
//   warp 1      TMEM allocator and MMA issuer (one elected lane, kind::i8,
//               M=128, N=128, K=32 per instruction) into 2 accumulator slots
//   warps 2..9  epilogue: tcgen05.ld 32x32b.x32, exact threshold, survivor
//               masks, per-row counts, level-2 check, warp-queued emission
// Level 2 is either a second GEMM on the 256-bit Xor sketches (dense regimes,
// L2G) or a POPC check of the level-1 survivors against staged sketches.
#pragma once

#include <climits>

#include "kernels.cuh"

namespace ssjb {
namespace dev {

#ifndef SSJB_SUSPEND_NS
#define SSJB_SUSPEND_NS 8192u
#endif
#ifndef SSJB_EARLY_ACC
#define SSJB_EARLY_ACC 1
#endif
// pipeline trace probe (SSJB_TC_DEBUG=2) compiled in only with -DSSJB_TRACE=1:
// its per-tile checks cost the hot loops a handful of instructions each
#ifndef SSJB_TRACE
#define SSJB_TRACE 0
#endif
constexpr int kTcQueue = 128;      // survivor staging per epilogue warp
constexpr int kTcLut = 1536;       // shared-memory copy of maxham[] (entries)
constexpr int kKindI8 = 0;         // tcgen05 kind::i8, s32 accumulators
constexpr int kKindF4 = 1;         // tcgen05 kind::mxf4 (packed e2m1, unit block scales), f32 accumulators

struct TcParams {
    const uint8_t* opA;        // expanded rows, core layout, n_pad x (KA [+ K2] + 16): L1 | L2 | size
    const uint8_t* opB;        // expanded columns, same layout (B encoding)
    const uint64_t* bits;      // level-1 sketches (row popcounts)
    const uint64_t* bits2;     // level-2 Xor sketches (rows; staged columns for the POPC check)
    const uint32_t* sizes;
    const int32_t* maxham;
    int maxham_len;
    const uint32_t* wstart;
    const uint64_t* item_base;
    const uint32_t* item_tile;   // tile of each work item
    const uint32_t* tile_col_lo;
    uint2* surv;
    uint32_t* rowcnt;
    uint32_t* item_counts;     // per (item, row-in-tile), u32 (two column halves add)
    uint16_t* tile_counts;     // per (item, tile-in-item, column part, row-in-tile), or null: the
                               // rescan's 2nd level; every slot of a processed tile is written
    uint32_t tiles_per_item;   // slots per item (>= ceil(kColChunk / NT))
    Control* ctl;
    unsigned long long surv_cap;
    unsigned long long surv_soft;  // see claim_item (kernels.cuh)
    unsigned long long item_begin, item_end;
    uint32_t tile_begin, ntiles;
    uint32_t row_begin, row_end;
    int64_t cutoff;
    int neg1;                  // always -1 (keeps the epilogue subtraction an IMAD)
    const uint32_t* npc2;      // no-extension int8 operands: -pc of columns 2k, 2k+1 as s16x2
    int debug;                 // bit 0: skip the epilogue math (pipeline probe)
    int bias, bias2;           // added to every level-1 / level-2 accumulator by the operands'
                               // extension (non-negative accumulators: SWAR masks, masks16_nonneg)
    unsigned long long* trace; // CTA 0 event timestamps (pipeline probe), or null
    uint32_t emit_col_end;     // level-2 GEMM: survivors with column j >= this are counted but
                               // not emitted (the head-overlap kernel K3a covers them); ~0u: all
    const uint32_t* item_order;  // claim index -> work item id (column-chunk-major), or null: identity
};

constexpr unsigned long long kNoItem = ~0ull;

// Next work item of a persistent tcgen05 filter: the claim index (prefix
// semantics of claim_item) mapped through P.item_order to an item id, or
// kNoItem when the launch has none left.  The column-chunk-major order makes
// the CTAs working at once read the same column operands, which then stay in
// L2 instead of being re-read from HBM by every row tile of a wide window.
__device__ __forceinline__ unsigned long long claim_tc(const TcParams& P) {
    const unsigned long long k = claim_item(P.ctl, P.item_begin, P.item_end, P.surv_soft);
    if (k >= P.item_end) return kNoItem;
    return P.item_order ? static_cast<unsigned long long>(P.item_order[k]) : k;
}

// Columns base_col + k < end of a 32-column group as a mask, natural bit order
// (bit k = column k) or the masks16_nonneg order (PERM: bit k < 16 = column
// 2k, bit 16 + k = column 2k + 1).
template <bool PERM>
__device__ __forceinline__ uint32_t cols_below(uint32_t end, uint32_t base_col) {
    const int x = end > base_col ? static_cast<int>(min(end - base_col, 32u)) : 0;
    if constexpr (PERM) return low_mask((x + 1) >> 1) | (low_mask(x >> 1) << 16);
    else return low_mask(x);
}

// One lane of the (converged) warp: elect.sync
__device__ __forceinline__ bool elect_one() {
    uint32_t pred = 0;
    asm volatile(
        "{\n.reg .pred P;\nelect.sync _|P, 0xffffffff;\nselp.u32 %0, 1, 0, P;\n}\n"
        : "=r"(pred));
    return pred != 0;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_arrive_u32(uint32_t a) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(a) : "memory");
}

// Spin without a suspend hint (single-lane producer / MMA roles: wake-up
// latency is on the critical path there).
// try_wait suspend-time hint (8 us; a 1 ms hint stalled concurrent joins from
// several host threads): a waiting warp is parked until the phase
// completes (or this many ns pass) instead of re-issuing the probe, leaving
// issue slots to the epilogue warps that share the SM sub-partitions
constexpr uint32_t kSuspendNs = SSJB_SUSPEND_NS;

__device__ __forceinline__ void mbar_spin(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n"
        "@!P1 bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity), "r"(kSuspendNs)
        : "memory");
}

__device__ __forceinline__ void mbar_wait_u32(uint32_t a, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n"
        "@!P1 bra WAIT_%=;\n"
        "}\n" ::"r"(a),
        "r"(parity), "r"(kSuspendNs)
        : "memory");
}

// Descriptor of the K step s after `d` (K-major, SWIZZLE_NONE): the next two
// 16-byte K chunks start 256 bytes further, i.e. +16 in the 14-bit start
// address field (shared-memory addresses < 256 KB never carry out of it).
// The MMA issuer builds one descriptor per operand and tile and steps it with
// one add per instruction instead of re-encoding it (a chain of uniform-
// datapath ops per MMA that paced the single issuing thread).
__device__ __forceinline__ uint64_t umma_desc_step(uint64_t d, int s) {
    return d + static_cast<uint64_t>(16 * s);
}

__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t sbo) {
    // K-major, SWIZZLE_NONE: LBO = 128 B between the two 16-byte K halves of
    // an instruction, SBO = stride between 8-row core-matrix groups.
    uint64_t d = static_cast<uint64_t>((saddr >> 4) & 0x3FFF);
    d |= static_cast<uint64_t>(128 >> 4) << 16;
    d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFF) << 32;
    d |= static_cast<uint64_t>(1) << 46;  // sm100 descriptor version
    return d;
}

// kind::i8, D s32, A u8, B s8, K-major both, M = 128, N = NT
template <int NT>
__device__ __forceinline__ void umma_i8(uint32_t tmem, uint64_t da, uint64_t db, uint32_t acc) {
    constexpr uint32_t idesc = (2u << 4) | (0u << 7) | (1u << 10) | ((NT >> 3) << 17) | ((128u >> 4) << 24);
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
        "l"(da), "l"(db), "r"(idesc), "r"(acc));
}

// kind::mxf4.block_scale.block32: A/B packed e2m1 (MXF4 format 1), ue8m0 scales
// (bit 23) read from TMEM -- all 1.0 here -- f32 accumulate, K = 64 per instruction.
template <int NT>
__device__ __forceinline__ void umma_f4(uint32_t tmem, uint64_t da, uint64_t db, uint32_t acc, uint32_t sfa,
                                        uint32_t sfb) {
    constexpr uint32_t idesc = (1u << 7) | (1u << 10) | ((NT >> 3) << 17) | (1u << 23) | ((128u >> 4) << 24);
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%6], p;\n}\n" ::"r"(tmem),
        "l"(da), "l"(db), "r"(idesc), "r"(acc), "r"(sfa), "r"(sfb));
}

__device__ __forceinline__ void tmem_fill32(uint32_t taddr, uint32_t v) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,"
        "%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(taddr),
        "r"(v));
}

__device__ __forceinline__ void umma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]),
          "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]),
          "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// 64 accumulator columns in one load: the low 16 bits of columns 2k, 2k+1 in
// register k (tcgen05.ld .pack::16b).  Exact for the int8 filter: every
// accumulator lies in [-2b, 2b] and b <= 256.
__device__ __forceinline__ void tmem_ld64_pack16(uint32_t taddr, uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.pack::16b.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]),
          "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]),
          "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// max over 64 packed s16 accumulators > c (two independent VIMNMX3.S16x2 chains)
__device__ __forceinline__ bool any_above16(const uint32_t (&d)[32], int c) {
    uint32_t a = __vimax3_s16x2(d[0], d[1], d[2]);
    uint32_t b = __vimax3_s16x2(d[3], d[4], d[5]);
#pragma unroll
    for (int k = 6; k < 30; k += 4) {
        a = __vimax3_s16x2(a, d[k], d[k + 1]);
        b = __vimax3_s16x2(b, d[k + 2], d[k + 3]);
    }
    a = __vimax3_s16x2(a, b, __vimax3_s16x2(d[30], d[31], d[31]));
    const int hi = static_cast<int>(a) >> 16;
    const int lo = static_cast<int>(static_cast<int16_t>(a & 0xFFFFu));
    return max(hi, lo) > c;
}

// 32 accumulator columns packed into 16 registers, no wait (pair with tmem_wait_ld)
__device__ __forceinline__ void tmem_ld32_pack16_nowait(uint32_t taddr, uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.pack::16b.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
}

__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// max over 32 packed s16 accumulators > c
__device__ __forceinline__ bool any_above16_32(const uint32_t (&d)[16], int c) {
    uint32_t a = __vimax3_s16x2(d[0], d[1], d[2]);
    uint32_t b = __vimax3_s16x2(d[3], d[4], d[5]);
    a = __vimax3_s16x2(a, d[6], d[7]);
    b = __vimax3_s16x2(b, d[8], d[9]);
    a = __vimax3_s16x2(a, d[10], d[11]);
    b = __vimax3_s16x2(b, d[12], d[13]);
    a = __vimax3_s16x2(a, b, __vimax3_s16x2(d[14], d[15], d[15]));
    const int hi = static_cast<int>(a) >> 16;
    const int lo = static_cast<int>(static_cast<int16_t>(a & 0xFFFFu));
    return max(hi, lo) > c;
}

// survivor mask of 32 packed columns: bit k set iff accumulator k > c (c >= -32768)
__device__ __forceinline__ uint32_t mask16_32(const uint32_t (&d)[16], int c) {
    const uint32_t c2 = (static_cast<uint32_t>(c) & 0xFFFFu) * 0x10001u;
    uint32_t x = 0;
#pragma unroll
    for (int k = 0; k < 16; ++k) {
        const uint32_t v = __vcmpgts2(d[k], c2);
        x |= ((v & 1u) | ((v >> 30) & 2u)) << (2 * k);
    }
    return x;
}

// survivor masks of the two 32-column groups of a packed 64-column load:
// bit k of m[g] = column 32g + k, set iff its accumulator > c (c >= -32768)
__device__ __forceinline__ void masks16(const uint32_t (&d)[32], int c, uint32_t& m0, uint32_t& m1) {
    const uint32_t c2 = (static_cast<uint32_t>(c) & 0xFFFFu) * 0x10001u;
    uint32_t x0 = 0, x1 = 0;
#pragma unroll
    for (int k = 0; k < 16; ++k) {
        const uint32_t v0 = __vcmpgts2(d[k], c2);       // 0xFFFF per half that survives
        const uint32_t v1 = __vcmpgts2(d[16 + k], c2);
        x0 |= ((v0 & 1u) | ((v0 >> 30) & 2u)) << (2 * k);
        x1 |= ((v1 & 1u) | ((v1 >> 30) & 2u)) << (2 * k);
    }
    m0 = x0;
    m1 = x1;
}

// Survivor masks of a packed 64-column load whose accumulators are
// non-negative and below 0x8000 (biased operands): per register one
// subtraction whose halves cannot borrow into each other -- (c + 0x8000) - d
// has bit 15 clear exactly when d > c -- then one shift and one LOP3 place
// the two survivor bits.  Bit order per 32 columns: bit k (k < 16) = column
// 2k, bit 16 + k = column 2k + 1 (see mask_col<true>).  c < 0: all survive.
__device__ __forceinline__ void masks16_nonneg(const uint32_t (&d)[32], int c, uint32_t& m0, uint32_t& m1) {
    if (c < 0) {
        m0 = m1 = 0xFFFFFFFFu;
        return;
    }
    const uint32_t C2 = ((static_cast<uint32_t>(min(c, 0x7FFE)) | 0x8000u)) * 0x10001u;
    uint32_t x0 = 0, x1 = 0;
#pragma unroll
    for (int k = 0; k < 16; ++k) {
        const uint32_t bits = (1u << k) | (1u << (16 + k));
        x0 |= ~((C2 - d[k]) >> (15 - k)) & bits;
        x1 |= ~((C2 - d[16 + k]) >> (15 - k)) & bits;
    }
    m0 = x0;
    m1 = x1;
}

// 32-column version (16 packed registers) of masks16_nonneg, same bit order.
__device__ __forceinline__ uint32_t mask16_32_nonneg(const uint32_t (&d)[16], int c) {
    if (c < 0) return 0xFFFFFFFFu;
    const uint32_t C2 = ((static_cast<uint32_t>(min(c, 0x7FFE)) | 0x8000u)) * 0x10001u;
    uint32_t x = 0;
#pragma unroll
    for (int k = 0; k < 16; ++k) x |= ~((C2 - d[k]) >> (15 - k)) & ((1u << k) | (1u << (16 + k)));
    return x;
}

// Survivor mask of 32 accumulator columns: column k survives iff
// cim1_k - D_k < 0 (sign bit set).  Four independent funnel-shift chains
// (8 columns each) keep the ALU pipe fed; the subtraction is an IMAD on the
// FMA pipe (neg1 == -1 arrives as a kernel parameter so ptxas keeps it there).
// Result: bit k = column k.
template <bool kUniform, int KIND = kKindI8>
__device__ __forceinline__ uint32_t survivors32(const uint32_t (&d)[32], int cim1, const int (&cims)[32], int neg1) {
    uint32_t m0 = 0, m1 = 0, m2 = 0, m3 = 0;
    const float cf = static_cast<float>(cim1);
    const float nf = static_cast<float>(neg1);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        uint32_t v[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            const int kk = 8 * c + j;
            if constexpr (KIND == kKindI8) {
                const int cc = kUniform ? cim1 : cims[kk];
                v[c] = static_cast<uint32_t>(static_cast<int>(d[kk]) * neg1 + cc);
            } else {  // exact small integers in f32: FFMA keeps the sign semantics (x - x = +0)
                const float cc = kUniform ? cf : static_cast<float>(cims[kk]);
                v[c] = __float_as_uint(__fmaf_rn(__uint_as_float(d[kk]), nf, cc));
            }
        }
        m0 = __funnelshift_l(v[0], m0, 1);
        m1 = __funnelshift_l(v[1], m1, 1);
        m2 = __funnelshift_l(v[2], m2, 1);
        m3 = __funnelshift_l(v[3], m3, 1);
    }
    // m_c bit (7-j) = column 8c+j  ->  bit 31-k = column k  ->  brev
    return __brev((m0 << 24) | (m1 << 16) | (m2 << 8) | m3);
}

// Accumulator value as an exact integer (s32, or an integral f32).
template <int KIND>
__device__ __forceinline__ int acc_int(uint32_t d) {
    if constexpr (KIND == kKindI8) return static_cast<int>(d);
    else return static_cast<int>(__uint_as_float(d));
}

// max_k D_k > cim1 for 32 accumulators, 16 three-input maxima.  For f32
// accumulators the bit patterns are compared as signed integers: that order
// is exact among non-negative values and puts every negative value below
// them, so the test is exact whenever cim1 >= 0 (the caller treats cim1 < 0
// as "maybe").
template <int KIND>
__device__ __forceinline__ bool any_above(const uint32_t (&d)[32], int cim1) {
    int mx = __vimax3_s32(static_cast<int>(d[0]), static_cast<int>(d[1]), static_cast<int>(d[2]));
#pragma unroll
    for (int k = 3; k < 31; k += 2) mx = __vimax3_s32(mx, static_cast<int>(d[k]), static_cast<int>(d[k + 1]));
    mx = max(mx, static_cast<int>(d[31]));
    if constexpr (KIND == kKindI8) return mx > cim1;
    else return mx > cim1;  // caller passes the bit pattern of cim1 + 0.5f, or INT_MIN when cim1 < 0
}

// Column sizes live in the last 16-byte chunk of every operand row (one
// bulk copy per tile carries operands and sizes); KCT = chunks per row.
template <int KCT>
__device__ __forceinline__ uint32_t stage_size(const uint8_t* stage, int col) {
    return *reinterpret_cast<const uint32_t*>(stage + ((col >> 3) * KCT + (KCT - 1)) * 128 + (col & 7) * 16);
}

// Column size of a tile column: from the side ring (no-extension operands) or
// from the size chunk of the staged operand rows.
template <bool kNoExt, int KCT>
__device__ __forceinline__ uint32_t tile_col_size(const uint32_t* side, const uint8_t* stage, int col) {
    if constexpr (kNoExt) return side[col];
    else return stage_size<KCT>(stage, col);
}

// Non-uniform group (column sizes change inside it): per-column threshold.
template <int KIND, int KCT>
__device__ __forceinline__ uint32_t survivors_mixed(const uint32_t (&d)[32], int base, const int32_t* maxham,
                                                    uint32_t si, const uint8_t* stage, int cl) {
    uint32_t m = 0;
#pragma unroll
    for (int k = 0; k < 32; ++k)
        m |= ((base - maxham[si + stage_size<KCT>(stage, cl + k)] - 1 - acc_int<KIND>(d[k])) < 0 ? 1u : 0u) << k;
    return m;
}

// a column size from the shared side ring (SMEM) or from global memory (read-only path)
template <bool SMEM>
__device__ __forceinline__ uint32_t ld_sz(const uint32_t* p) {
    if constexpr (SMEM) return *p;
    else return __ldg(p);
}

// survivors_mixed with the tile's column sizes read from a plain u32 array
template <int KIND, bool SMEM>
__device__ __forceinline__ uint32_t survivors_mixed_g(const uint32_t (&d)[32], int base, const int32_t* maxham,
                                                      uint32_t si, const uint32_t* gsz, int cl) {
    uint32_t m = 0;
#pragma unroll
    for (int k = 0; k < 32; ++k)
        m |= ((base - maxham[si + ld_sz<SMEM>(gsz + cl + k)] - 1 - acc_int<KIND>(d[k])) < 0 ? 1u : 0u) << k;
    return m;
}

__device__ __forceinline__ void tc_flush(uint2* q, int& qlen, const TcParams& P, int lane) {
    unsigned long long base = 0;
    if (lane == 0) base = atomicAdd(&P.ctl->survivors, static_cast<unsigned long long>(qlen));
    base = __shfl_sync(0xFFFFFFFFu, base, 0);
    for (int k = lane; k < qlen; k += 32)
        if (base + k < P.surv_cap) P.surv[base + k] = q[k];
    qlen = 0;
    __syncwarp();
}

// Column of mask bit k: identity, or (PERM) the masks16_nonneg order where bit
// k < 16 is column 2k and bit 16 + k is column 2k + 1.
template <bool PERM>
__device__ __forceinline__ uint32_t mask_col(int k) {
    return PERM ? static_cast<uint32_t>(2 * (k & 15) + (k >> 4)) : static_cast<uint32_t>(k);
}

// Both 32-column masks of a 64-column block in one emission (one prefix scan
// instead of two): m0 covers columns base_col + [0, 32), m1 base_col + [32, 64).
template <bool PERM>
__device__ __forceinline__ void tc_emit64(uint32_t m0, uint32_t m1, uint32_t base_col, uint32_t row, uint2* q,
                                          int& qlen, const TcParams& P, int lane) {
    const int c = __popc(m0) + __popc(m1);
    int incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int v = __shfl_up_sync(0xFFFFFFFFu, incl, o);
        if (lane >= o) incl += v;
    }
    const int total = __shfl_sync(0xFFFFFFFFu, incl, 31);
    if (total == 0) return;
    const int excl = incl - c;
    if (total > kTcQueue) {
        unsigned long long base = 0;
        if (lane == 0) base = atomicAdd(&P.ctl->survivors, static_cast<unsigned long long>(total));
        base = __shfl_sync(0xFFFFFFFFu, base, 0) + excl;
        while (m0) {
            int k = __ffs(m0) - 1;
            m0 &= m0 - 1;
            if (base < P.surv_cap) P.surv[base] = make_uint2(base_col + mask_col<PERM>(k), row);
            ++base;
        }
        while (m1) {
            int k = __ffs(m1) - 1;
            m1 &= m1 - 1;
            if (base < P.surv_cap) P.surv[base] = make_uint2(base_col + 32 + mask_col<PERM>(k), row);
            ++base;
        }
        return;
    }
    if (qlen + total > kTcQueue) tc_flush(q, qlen, P, lane);
    int pos = qlen + excl;
    while (m0) {
        int k = __ffs(m0) - 1;
        m0 &= m0 - 1;
        q[pos++] = make_uint2(base_col + mask_col<PERM>(k), row);
    }
    while (m1) {
        int k = __ffs(m1) - 1;
        m1 &= m1 - 1;
        q[pos++] = make_uint2(base_col + 32 + mask_col<PERM>(k), row);
    }
    qlen += total;
    __syncwarp();
}

template <bool PERM = false>
__device__ __forceinline__ void tc_emit(uint32_t m, uint32_t base_col, uint32_t row, uint2* q, int& qlen,
                                        const TcParams& P, int lane) {
    const int c = __popc(m);
    int incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int v = __shfl_up_sync(0xFFFFFFFFu, incl, o);
        if (lane >= o) incl += v;
    }
    const int total = __shfl_sync(0xFFFFFFFFu, incl, 31);
    const int excl = incl - c;
    if (total > kTcQueue) {
        unsigned long long base = 0;
        if (lane == 0) base = atomicAdd(&P.ctl->survivors, static_cast<unsigned long long>(total));
        base = __shfl_sync(0xFFFFFFFFu, base, 0) + excl;
        while (m) {
            int k = __ffs(m) - 1;
            m &= m - 1;
            if (base < P.surv_cap) P.surv[base] = make_uint2(base_col + mask_col<PERM>(k), row);
            ++base;
        }
        return;
    }
    if (qlen + total > kTcQueue) tc_flush(q, qlen, P, lane);
    int pos = qlen + excl;
    while (m) {
        int k = __ffs(m) - 1;
        m &= m - 1;
        q[pos++] = make_uint2(base_col + mask_col<PERM>(k), row);
    }
    qlen += total;
    __syncwarp();
}

struct TcItem {
    unsigned long long item;
    uint32_t tile, c0, c1, ntiles, done;
};

// An epilogue warp's copy of a published work item: lane 0 alone reads the
// shared slot and broadcasts it, so the lane that releases the slot (its
// mbarrier arrive) is the only one that read it.
__device__ __forceinline__ TcItem warp_item(const TcItem& slot, int lane) {
    TcItem v{};
    if (lane == 0) v = slot;
    v.item = __shfl_sync(0xFFFFFFFFu, v.item, 0);
    v.tile = __shfl_sync(0xFFFFFFFFu, v.tile, 0);
    v.c0 = __shfl_sync(0xFFFFFFFFu, v.c0, 0);
    v.c1 = __shfl_sync(0xFFFFFFFFu, v.c1, 0);
    v.ntiles = __shfl_sync(0xFFFFFFFFu, v.ntiles, 0);
    v.done = __shfl_sync(0xFFFFFFFFu, v.done, 0);
    return v;
}

// KIND: operand kind; KA: level-1 operand bytes per row; K2: level-2 GEMM
// operand bytes (0: none); W2: level-2 Xor sketch words for the POPC check
// (used when K2 == 0); NS: B stages; NT: columns per MMA tile.
template <int KIND, int KA, int K2, int W2, int NS, int NT>
struct TcLayout {
    // int8 operands without the popcount extension (K = b): D = 2<b_i,b_j>, the
    // -pc_j term is added in the epilogue from a per-stage s16x2 array
    static constexpr bool kNoExt = KIND == kKindI8 && K2 == 0 && KA % 64 == 0;
    static constexpr int kWords = kNoExt ? KA / 64 : (KIND == kKindI8 ? (KA - 32) / 64 : (KA - 32) / 32);
    // no-extension operands carry no size chunk: the column sizes and -pc pairs of
    // each tile go to a separate, deeper "side" ring, so a B stage is released as
    // soon as its MMAs complete (the epilogue never holds it)
    // level-2 GEMM: a B stage is released when its MMAs complete, not when the
    // epilogue is done with the tile -- with only a few 51 KB stages fitting, a
    // stage's lifetime (copy + MMAs + epilogue) otherwise paces the pipeline.
    // The epilogue reads the tile's column sizes from global memory (L2);
    // SSJB_SIZE_RING=1 stages them in a small side ring instead (512 B per
    // tile, its own bulk copy, released by the epilogue warps) -- measured
    // slower on C4 (136.5 vs 128.1 ms K2, 4 or 7 slots alike), although the
    // global loads are the epilogue's largest single stall in ncu.
    static constexpr bool kEarlyB = K2 > 0;
#ifndef SSJB_L2_EPI_SETS
#define SSJB_L2_EPI_SETS 1
#endif
    static constexpr int kSets = (K2 > 0 && NT == 128) ? SSJB_L2_EPI_SETS : 1;
#ifndef SSJB_SIZE_RING
#define SSJB_SIZE_RING 0
#endif
    static constexpr bool kSizeRing = kEarlyB && kSets == 1 && SSJB_SIZE_RING;
    static constexpr int kSide = kNoExt ? NT * 4 + NT * 2 : (kSizeRing ? NT * 4 : 0);  // sizes u32[NT] | -pc pairs
#ifndef SSJB_SIZE_RING_SLOTS
#define SSJB_SIZE_RING_SLOTS 7
#endif
    // side-ring slots (size ring: enough that the producer's lead over the
    // epilogue stays that of the B stages plus accumulator slots)
    static constexpr int NE = kNoExt ? 2 * NS : (kSizeRing ? SSJB_SIZE_RING_SLOTS : 1);
    static constexpr bool kSideRing = kNoExt || kSizeRing;
    // epilogue warps (4 per column part, one per TMEM lane quarter): 64 columns
    // each for the level-2 GEMM's 128-column tiles (the per-tile fixed cost of a
    // warp -- barrier waits, column sizes, thresholds -- paid by 8 warps, not 16)
    static constexpr int kEpiWarps = NT == 192 ? 12 : 16;
    // level-2 GEMM kernel: SSJB_L2_EPI_SETS=2 splits the 16 epilogue warps into
    // two sets taking alternate tiles (accumulator slots), 64 columns per warp
    // and two tile intervals each; measured neutral on C4 (162 vs 160 ms), so
    // the default keeps every warp on every tile
    static constexpr int kSetWarps = kEpiWarps / kSets;      // warps per tile
    static constexpr int kParts = kSetWarps / 4;             // column parts per tile
    static constexpr int kThreads = 64 + 32 * kEpiWarps;
    static constexpr int kColsPerWarp = NT * 4 / kSetWarps;
    static constexpr int kRow = KA + K2 + (kNoExt ? 0 : 16);   // operand row: L1 | L2 | size chunk
    static constexpr int kKCT = kRow / 16;                     // 16-byte chunks per row
    static constexpr int kSbo = kKCT * 128;                    // stride between 8-row core groups
    static constexpr int kA = 128 * kRow;                      // one A slot
    static constexpr int kB = NT * kRow;                       // one B stage: a single bulk copy
    static constexpr int kAslots = K2 ? 1 : 2;
    static constexpr int kQueue = kEpiWarps * kTcQueue * 8;
    static constexpr int kBytes = kAslots * kA + NS * kB + (kSideRing ? NE * kSide : 0) + kQueue;
    // accumulator slots in flight: as many NT-column slots (x2 with the level-2
    // GEMM) as TMEM holds next to the fp4 scale factors, at most 4
    static constexpr int kAccSlots = (((KIND == kKindF4 ? 384 : 512) / (NT * (K2 ? 2 : 1))) < 4)
                                         ? ((KIND == kKindF4 ? 384 : 512) / (NT * (K2 ? 2 : 1))) : 4;
    static constexpr uint32_t kAccCols = (K2 ? 2 : 1) * kAccSlots * NT;
    static constexpr uint32_t kL2Col = kAccSlots * NT;        // level-2 accumulators follow level 1
    static constexpr uint32_t kSfCol = kAccCols;              // fp4: 32 columns of A scales, then B scales
    static constexpr uint32_t kTmemCols = KIND == kKindF4 ? 512 : (kAccCols <= 256 ? 256 : 512);
    static_assert(kColsPerWarp % 32 == 0, "epilogue column split");
    static_assert(kBytes + 1024 + 4 * kTcLut + 512 <= 232448, "shared memory per CTA");
    static_assert(KIND == kKindI8 || kAccCols + 128 <= 512, "TMEM: accumulators + scale factors");
    static_assert(kAccCols <= 512 && kAccSlots >= 2, "TMEM");
    static_assert(kSets == 1 || (kEarlyB && kAccSlots % kSets == 0), "epilogue sets need early B release");
};

template <int KIND, int KA, int K2, int W2, int NS, int NT>
__global__ void __launch_bounds__((TcLayout<KIND, KA, K2, W2, NS, NT>::kThreads), 1) filter_tc_kernel(TcParams P) {
    using L = TcLayout<KIND, KA, K2, W2, NS, NT>;
    constexpr int kTcEpiWarps = L::kEpiWarps;
    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t* sA = smem;                                   // [2][kA]
    uint8_t* sB = smem + L::kAslots * L::kA;              // [NS][kB]
    uint8_t* sSide = sB + NS * L::kB;                     // [NE][kSide] (no-extension operands)
    uint2* sQ = reinterpret_cast<uint2*>(sSide + (L::kSideRing ? L::NE * L::kSide : 0));  // [8][kTcQueue]
    __shared__ __align__(8) uint64_t item_full[2], item_empty[2], a_full[2], a_empty[2];
    __shared__ __align__(8) uint64_t b_full[NS], b_empty[NS], acc_full[L::kAccSlots], acc_empty[L::kAccSlots];
    __shared__ __align__(8) uint64_t e_full[L::NE], e_empty[L::NE];
    __shared__ TcItem items[2];
    __shared__ uint32_t tmem_base_sh;
    __shared__ int32_t s_maxham[kTcLut];  // maxham[] when it fits (2*max_size + 1 <= kTcLut)

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    constexpr uint32_t kTmemCols = L::kTmemCols;  // 2 slots x (L1 [+ L2]) x NT (+ fp4 scale factors)

    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base_sh)),
                     "r"(kTmemCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    const bool lut_smem = P.maxham_len <= kTcLut;
    if (lut_smem)
        for (int k = threadIdx.x; k < P.maxham_len; k += blockDim.x) s_maxham[k] = P.maxham[k];
    const int32_t* maxham = lut_smem ? s_maxham : P.maxham;
    if (threadIdx.x == 0) {
        for (int s = 0; s < 2; ++s) {
            mbar_init(&item_full[s], 1);
            mbar_init(&item_empty[s], 1 + kTcEpiWarps);
            mbar_init(&a_full[s], 1);
            mbar_init(&a_empty[s], 1);
        }
        for (int s = 0; s < L::kAccSlots; ++s) {
            mbar_init(&acc_full[s], 1);
            mbar_init(&acc_empty[s], L::kSetWarps);
        }
        for (int s = 0; s < L::NE; ++s) {
            mbar_init(&e_full[s], 1);
            mbar_init(&e_empty[s], kTcEpiWarps);
        }
        for (int s = 0; s < NS; ++s) {
            mbar_init(&b_full[s], 1);
            mbar_init(&b_empty[s], (L::kNoExt || L::kEarlyB) ? 1 : 1 + kTcEpiWarps);
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

    if (warp == 0) {
        // ------------------------------------------------------------ producer
        if (lane == 0) {
            uint32_t iseq = 0, tseq = 0;
            // the next work item is claimed and looked up while the current one's
            // column tiles are still streaming (hides the atomic + table latency)
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
                const uint32_t row0 = P.row_begin + tile * kRowTile;
                const uint32_t rows_end = min(row0 + kRowTile, P.row_end);
                info.tile = tile;
                info.c0 = P.tile_col_lo[tile] + chunk * kColChunk;
                info.c1 = min(info.c0 + kColChunk, rows_end - 1);
                info.ntiles = (info.c1 - info.c0 + NT - 1) / NT;
                info.done = 0;
                items[slot] = info;
                // row operand (A): 128 rows, contiguous in the core layout
                const int aslot = iseq % L::kAslots;
                mbar_spin(&a_empty[aslot], ((iseq / L::kAslots) & 1) ^ 1);
                mbar_expect_tx(&a_full[aslot], L::kA);
                tma_load_1d(sA + aslot * L::kA, P.opA + static_cast<uint64_t>(row0) * L::kRow, L::kA, &a_full[aslot]);
                mbar_arrive(&item_full[slot]);
                for (uint32_t t = 0; t < info.ntiles; ++t, ++tseq) {
                    const int st = tseq % NS;
                    mbar_spin(&b_empty[st], ((tseq / NS) & 1) ^ 1);
                    if (SSJB_TRACE && P.trace && blockIdx.x == 0 && tseq < 512) P.trace[tseq * 4 + 0] = clock64();
                    const uint32_t col = info.c0 + t * NT;
                    uint8_t* dst = sB + st * L::kB;
                    if constexpr (L::kSideRing) {
                        const int se = tseq % L::NE;
                        mbar_spin(&e_empty[se], ((tseq / L::NE) & 1) ^ 1);
                        uint8_t* side = sSide + se * L::kSide;
                        mbar_expect_tx(&e_full[se], L::kSide);
                        tma_load_1d(side, P.sizes + col, NT * 4, &e_full[se]);
                        if constexpr (L::kNoExt) tma_load_1d(side + NT * 4, P.npc2 + col / 2, NT * 2, &e_full[se]);
                    }
                    if ((P.debug & 8) && tseq >= NS) {  // (probe bit 8: stale B stages, no copies)
                        mbar_arrive(&b_full[st]);
                    } else {
                        mbar_expect_tx(&b_full[st], L::kB);
                        tma_load_1d(dst, P.opB + static_cast<uint64_t>(col) * L::kRow, L::kB, &b_full[st]);
                    }
                    if (t == 0) {
                        nxt = claim_tc(P);
                        nxt_tile = nxt != kNoItem ? P.item_tile[nxt] : 0u;
                    }
                }
                if (info.ntiles == 0) {
                    nxt = claim_tc(P);
                    nxt_tile = nxt != kNoItem ? P.item_tile[nxt] : 0u;
                }
                ++iseq;
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------------------ MMA issuer
        // The whole warp runs the loop (warp-uniform control flow: the tile
        // bookkeeping and descriptors live in uniform registers); one elected
        // lane issues each tcgen05 instruction and arrive.
        const bool leader = elect_one();
        {
            uint32_t iseq = 0, tseq = 0, aseq = 0;
            for (;;) {
                const int slot = iseq & 1;
                mbar_spin(&item_full[slot], (iseq >> 1) & 1);
                const TcItem info = items[slot];
                __syncwarp();
                if (leader) mbar_arrive(&item_empty[slot]);
                if (info.done) break;
                const int aslot = iseq % L::kAslots;
                mbar_spin(&a_full[aslot], (iseq / L::kAslots) & 1);
                const uint32_t a0 = smem_u32(sA + aslot * L::kA);
                const uint64_t da0 = umma_desc(a0, L::kSbo);
                const uint64_t da2 = umma_desc(a0 + KA * 8, L::kSbo);  // level-2 K range of the A rows
                // the NS stages' B descriptors (a stage's address never changes)
                uint64_t dbs[NS];
#pragma unroll
                for (int k = 0; k < NS; ++k) dbs[k] = umma_desc(smem_u32(sB + k * L::kB), L::kSbo);
                for (uint32_t t = 0; t < info.ntiles; ++t, ++tseq, ++aseq) {
                    const int st = tseq % NS;
                    const int as = aseq % L::kAccSlots;
                    uint64_t db0 = dbs[0];
#pragma unroll
                    for (int k = 1; k < NS; ++k) db0 = st == k ? dbs[k] : db0;
                    const uint64_t db2 = umma_desc_step(db0, KA / 32);  // (KA * 8 bytes further = KA/32 K steps)
                    mbar_spin(&b_full[st], (tseq / NS) & 1);
                    if (SSJB_TRACE && P.trace && blockIdx.x == 0 && tseq < 512) P.trace[tseq * 4 + 1] = clock64();
                    mbar_spin(&acc_empty[as], ((aseq / L::kAccSlots) & 1) ^ 1);
                    if (SSJB_TRACE && P.trace && blockIdx.x == 0 && tseq < 512) P.trace[tseq * 4 + 2] = clock64();
                    asm volatile("tcgen05.fence::after_thread_sync;");
                    const uint32_t d1 = tmem_base + as * NT;
                    if (leader) {
#pragma unroll
                        for (int s = 0; s < KA / 32; ++s) {
                            const uint64_t da = umma_desc_step(da0, s);
                            const uint64_t db = umma_desc_step(db0, s);
                            if constexpr (KIND == kKindI8)
                                umma_i8<NT>(d1, da, db, s > 0);
                            else
                                umma_f4<NT>(d1, da, db, s > 0, tmem_base + L::kSfCol, tmem_base + L::kSfCol + 32);
                        }
                        if constexpr (K2 > 0) {
                            const uint32_t d2 = tmem_base + L::kL2Col + as * NT;
#pragma unroll
                            for (int s = 0; s < ((P.debug & 4) ? 1 : K2 / 32); ++s)  // (probe bit 4: one L2 MMA)
                                umma_i8<NT>(d2, umma_desc_step(da2, s), umma_desc_step(db2, s), s > 0);
                        }
                        umma_commit(&b_empty[st]);
                        umma_commit(&acc_full[as]);
                    }
                    __syncwarp();
                }
                if (leader) umma_commit(&a_empty[aslot]);
                __syncwarp();
                ++iseq;
            }
        }
    } else {
        // ------------------------------------------------------------ epilogue
        const int ew = warp - 2;
        const int quarter = warp & 3;          // TMEM lanes 32*quarter .. +31 (hardware rule)
        const int eset = ew / L::kSetWarps;    // the tiles (accumulator slots) this warp takes
        const int part = (ew % L::kSetWarps) >> 2;  // this warp's column range of each tile
        const int rit = quarter * 32 + lane;   // row in tile
        const uint32_t lane_base = static_cast<uint32_t>(quarter * 32) << 16;
        uint2* q = sQ + ew * kTcQueue;
        int qlen = 0;
        uint32_t iseq = 0;
        uint32_t st_idx = 0, st_phase = 0, acc_idx = 0, acc_phase = 0;  // ring positions
        uint32_t se_idx = 0, se_phase = 0;                                 // side ring (no-extension)
        uint32_t tile_seq = 0;
        const uint32_t bfull_u32 = smem_u32(&b_full[0]), bempty_u32 = smem_u32(&b_empty[0]);
        const uint32_t accfull_u32 = smem_u32(&acc_full[0]), accempty_u32 = smem_u32(&acc_empty[0]);
        for (;;) {
            const int slot = iseq & 1;
            mbar_wait(&item_full[slot], (iseq >> 1) & 1);
            const TcItem info = warp_item(items[slot], lane);
            __syncwarp();
            if (lane == 0) mbar_arrive(&item_empty[slot]);
            if (info.done) break;
            const uint32_t row0 = P.row_begin + info.tile * kRowTile;
            const uint32_t rows_end = min(row0 + kRowTile, P.row_end);
            const uint32_t i = row0 + rit;
            const bool valid = i < rows_end;
            uint32_t si = 0, j0 = 0;
            int pc = 0;
            bool bypass = false;
            uint64_t mine2[W2 > 0 ? W2 : 1];
#pragma unroll
            for (int w = 0; w < (W2 > 0 ? W2 : 1); ++w) mine2[w] = 0;
            if (valid) {
                si = P.sizes[i];
                j0 = P.wstart[si];
                bypass = static_cast<int64_t>(si) > P.cutoff;
#pragma unroll
                for (int w = 0; w < L::kWords; ++w) pc += __popcll(P.bits[static_cast<uint64_t>(i) * L::kWords + w]);
                pc += P.bias;  // thresholds shift with the biased accumulators
                if constexpr (K2 > 0) {
#pragma unroll
                    for (int w = 0; w < W2; ++w) mine2[w] = P.bits2[static_cast<uint64_t>(i) * W2 + w];
                }
            }
            int pc2 = 0;
            if constexpr (K2 > 0) {
#pragma unroll
                for (int w = 0; w < W2; ++w) pc2 += __popcll(mine2[w]);
                pc2 += P.bias2;
            }
            const uint32_t lo_i = valid ? max(j0, info.c0) : info.c1;
            const uint32_t hi_i = valid ? min(i, info.c1) : info.c1;
            // warp-uniform interior: groups inside every lane's window need no mask
            uint32_t lo_max = lo_i, hi_min = hi_i;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                lo_max = max(lo_max, __shfl_xor_sync(0xFFFFFFFFu, lo_max, o));
                hi_min = min(hi_min, __shfl_xor_sync(0xFFFFFFFFu, hi_min, o));
            }
            uint32_t cnt = 0, cnt_tile0 = 0;
            uint32_t last_sz = 0xFFFFFFFFu;  // cim1 cache: sizes are sorted, so it rarely changes
            int cim1 = 0, cim1_2 = 0, cim1_key = 0;
            for (uint32_t t = 0; t < info.ntiles; ++t) {
                if constexpr (L::kSets > 1) {
                    if (static_cast<int>(acc_idx % L::kSets) != eset) {  // the other set's tile
                        if (++st_idx == NS) {
                            st_idx = 0;
                            st_phase ^= 1u;
                        }
                        if (++acc_idx == L::kAccSlots) {
                            acc_idx = 0;
                            acc_phase ^= 1u;
                        }
                        continue;
                    }
                }
                const int st = static_cast<int>(st_idx), as = static_cast<int>(acc_idx);
                if constexpr (L::kSideRing) mbar_wait_u32(smem_u32(&e_full[0]) + 8 * se_idx, se_phase);
                else if constexpr (!L::kEarlyB) mbar_wait_u32(bfull_u32 + 8 * st_idx, st_phase);
                // (early-released stages: the accumulator's completion implies the
                // operands arrived; sizes come from gsz below)
                // tile's column sizes: the side ring (kSizeRing, already waited on
                // above) or global memory (L2)
                const uint32_t* gsz = L::kSizeRing ? reinterpret_cast<const uint32_t*>(sSide + se_idx * L::kSide)
                                                   : P.sizes + info.c0 + t * NT;
                // level-2 GEMM kernel, one 32-column group per warp: the packed
                // group loads are the warp's only TMEM reads of the tile, so the slot
                // is released as soon as they land (SSJB_EARLY_ACC=0: at tile end)
                constexpr bool kEarlyAcc = K2 > 0 && KIND == kKindI8 && L::kColsPerWarp == 32 && SSJB_EARLY_ACC;
                bool acc_released = false;
                uint32_t pre0 = 0, pre1 = 0;
                if constexpr (L::kEarlyB) {  // issue the size loads before the accumulator wait
                    // (loading them one tile ahead measured slower: 151.7 vs 147.7 ms on C4)
                    pre0 = ld_sz<L::kSizeRing>(gsz + part * L::kColsPerWarp);
                    pre1 = ld_sz<L::kSizeRing>(gsz + part * L::kColsPerWarp + L::kColsPerWarp - 1);
                }
                mbar_wait_u32(accfull_u32 + 8 * acc_idx, acc_phase);
                asm volatile("tcgen05.fence::after_thread_sync;");
                if (SSJB_TRACE && P.trace && blockIdx.x == 0 && lane == 0 && tile_seq < 512) P.trace[2048 + tile_seq * 16 + (warp - 2)] = clock64();
                ++tile_seq;
                const uint8_t* stage = sB + st * L::kB;
                const uint32_t* side_sz = reinterpret_cast<const uint32_t*>(sSide + se_idx * L::kSide);
                const uint32_t* sNpc = side_sz + NT;  // -pc pairs of the tile's columns
                const int cw = part * L::kColsPerWarp;               // this warp's first column
                const uint32_t wbase = info.c0 + t * NT + cw;
                const uint32_t szw0 = L::kEarlyB ? pre0 : tile_col_size<L::kNoExt, L::kKCT>(side_sz, stage, cw);
                const uint32_t szw1 =
                    L::kEarlyB ? pre1 : tile_col_size<L::kNoExt, L::kKCT>(side_sz, stage, cw + L::kColsPerWarp - 1);
                // fast path: every group of this warp's range is inside all 32
                // windows and of one column size (the bulk of the pair space)
                const bool fast = szw0 == szw1 && wbase >= lo_max && wbase + L::kColsPerWarp <= hi_min;
                if (fast && szw0 != last_sz) {
                    last_sz = szw0;
                    const int T = maxham[si + szw0];
                    cim1 = pc - T - 1;
                    cim1_2 = pc2 - T - 1;
                    cim1_key = cim1 < 0 ? INT_MIN : __float_as_int(static_cast<float>(cim1) + 0.5f);
                }
                // per-group tail: counts, level-2 check, emission (m = level-1 survivors)
                auto finish = [&](int cl, uint32_t gbase, uint32_t m, bool uni) {
                    cnt += __popc(m);
                    if (!__any_sync(0xFFFFFFFFu, m != 0)) return;
                    uint32_t e = m;
                    if constexpr (K2 > 0) {
                        uint32_t d2[32];
                        int dummy2[32];
                        tmem_ld32(tmem_base + lane_base + L::kL2Col + as * NT + cl, d2);
                        e = m & (uni ? survivors32<true, KIND>(d2, cim1_2, dummy2, P.neg1)
                                     : (L::kEarlyB ? survivors_mixed_g<KIND, L::kSizeRing>(d2, pc2, maxham, si, gsz, cl)
                                                   : survivors_mixed<KIND, L::kKCT>(d2, pc2, maxham, si, stage, cl)));
                    }
                    // (without the level-2 GEMM, level-1 survivors are emitted and
                    // verify_pairs re-tests them against the level-2 sketch first)
                    if constexpr (K2 > 0) e &= cols_below<false>(P.emit_col_end, gbase);
                    if (__any_sync(0xFFFFFFFFu, e != 0)) tc_emit(e, gbase, i, q, qlen, P, lane);
                };
                bool groups_done = (P.debug & 1) != 0;
                if constexpr (KIND == kKindI8 && L::kColsPerWarp == 64 && K2 == 0) {
                    // interior fast path: the warp's 64 columns in ONE packed TMEM
                    // load (one load latency per tile instead of two)
                    if (fast && !groups_done) {
                        groups_done = true;
                        uint32_t d[32];
                        tmem_ld64_pack16(tmem_base + lane_base + as * NT + cw, d);
                        const int c16 = max(cim1, -32768);
                        if constexpr (L::kNoExt) {  // D = 2<b_i,b_j>: subtract pc_j per column first
                            const uint4* np = reinterpret_cast<const uint4*>(sNpc + cw / 2);
#pragma unroll
                            for (int k = 0; k < 8; ++k) {
                                const uint4 v = np[k];
                                d[4 * k] = __vadd2(d[4 * k], v.x);
                                d[4 * k + 1] = __vadd2(d[4 * k + 1], v.y);
                                d[4 * k + 2] = __vadd2(d[4 * k + 2], v.z);
                                d[4 * k + 3] = __vadd2(d[4 * k + 3], v.w);
                            }
                        }
                        if (__any_sync(0xFFFFFFFFu, bypass || any_above16(d, c16))) {
                            uint32_t m0 = 0xFFFFFFFFu, m1 = 0xFFFFFFFFu;
                            if (!bypass) masks16(d, c16, m0, m1);
                            finish(cw, wbase, m0, true);
                            finish(cw + 32, wbase + 32, m1, true);
                        }
                    }
                }
                // (the level-2 GEMM variant keeps the unpacked path below: it is bound
                // by shared-memory operand traffic, and the packed s16 masks cost more
                // ALU per group when most pairs survive level 1 -- 3.17 vs 2.68 ms, C2 tau=0.5)
                // (with biased operands the level-2 GEMM variant takes the packed
                // path too: non-negative accumulators make its masks 3 instructions
                // per register -- masks16_nonneg -- so the packed path wins there)
                const bool packed32 = K2 == 0 || (P.bias > 0 && P.bias2 > 0);
                if constexpr (KIND == kKindI8) {
                    // int8 groups of 32 columns: level-1 accumulators
                    // as packed s16 in one load latency.  Thresholds per run of equal
                    // column size (sizes are sorted, so a group holds 1-3 runs): a
                    // ballot over the lanes' column sizes gives each run's columns.
#pragma unroll 1
                    for (int g = 0; g < (groups_done || !packed32 ? 0 : L::kColsPerWarp / 32); ++g) {
                        const int cl = cw + g * 32;
                        const uint32_t gbase = wbase + g * 32;
                        uint32_t rm = 0xFFFFFFFFu;
                        if (!fast) {
                            const int kl = static_cast<int>(lo_i) - static_cast<int>(gbase);
                            const int kh = static_cast<int>(hi_i) - static_cast<int>(gbase);
                            rm = low_mask(kh) & ~low_mask(kl);
                            if (!__any_sync(0xFFFFFFFFu, rm != 0)) continue;
                        }
                        uint32_t d[16], d2[16];
                        tmem_ld32_pack16_nowait(tmem_base + lane_base + as * NT + cl, d);
                        if constexpr (K2 > 0) tmem_ld32_pack16_nowait(tmem_base + lane_base + L::kL2Col + as * NT + cl, d2);
                        const uint32_t colsz = fast ? 0u
                                                    : (L::kEarlyB ? ld_sz<L::kSizeRing>(gsz + cl + lane)
                                                                  : tile_col_size<L::kNoExt, L::kKCT>(side_sz, stage, cl + lane));
                        tmem_wait_ld();
                        if constexpr (kEarlyAcc) {
                            // the warp's only group is in registers: hand the accumulator
                            // slot back to the MMA issuer before the masks and emission
                            asm volatile("tcgen05.fence::before_thread_sync;");
                            __syncwarp();
                            if (lane == 0) mbar_arrive_u32(accempty_u32 + 8 * acc_idx);
                            acc_released = true;
                        }
                        if constexpr (L::kNoExt) {  // D - pc_j per column
                            const uint4* np = reinterpret_cast<const uint4*>(sNpc + cl / 2);
#pragma unroll
                            for (int k = 0; k < 4; ++k) {
                                const uint4 v = np[k];
                                d[4 * k] = __vadd2(d[4 * k], v.x);
                                d[4 * k + 1] = __vadd2(d[4 * k + 1], v.y);
                                d[4 * k + 2] = __vadd2(d[4 * k + 2], v.z);
                                d[4 * k + 3] = __vadd2(d[4 * k + 3], v.w);
                            }
                        }
                        // lowest threshold over the group's size runs (pre-test)
                        int cmin = cim1;
                        if (!fast) {
                            cmin = INT_MAX;
                            uint32_t rem = 0xFFFFFFFFu;
                            while (rem) {
                                const uint32_t sz = __shfl_sync(0xFFFFFFFFu, colsz, __ffs(rem) - 1);
                                rem &= ~__ballot_sync(0xFFFFFFFFu, colsz == sz);
                                cmin = min(cmin, pc - maxham[si + sz] - 1);
                            }
                        }
                        if (!__any_sync(0xFFFFFFFFu, bypass || (rm != 0 && any_above16_32(d, max(cmin, -32768)))))
                            continue;
                        uint32_t m = 0xFFFFFFFFu, e2 = 0xFFFFFFFFu;
                        bool perm = false;
                        if (fast && P.bias > 0 && (K2 == 0 || P.bias2 > 0)) {
                            // biased accumulators: SWAR masks in the permuted bit order
                            perm = true;
                            if (!bypass) m = mask16_32_nonneg(d, cim1);
                            if constexpr (K2 > 0) {
                                // level-2 survivors are rare: the mask only when a lane has one
                                // (max over the packed accumulators, three-input VIMNMX)
                                e2 = __any_sync(0xFFFFFFFFu, m != 0 && any_above16_32(d2, max(cim1_2, -32768)))
                                         ? mask16_32_nonneg(d2, cim1_2)
                                         : 0u;
                            }
                        } else if (fast) {
                            if (!bypass) m = mask16_32(d, max(cim1, -32768));
                            if constexpr (K2 > 0) e2 = mask16_32(d2, max(cim1_2, -32768));
                        } else {
                            uint32_t mm = 0, ee = 0, rem = 0xFFFFFFFFu;
                            while (rem) {
                                const uint32_t sz = __shfl_sync(0xFFFFFFFFu, colsz, __ffs(rem) - 1);
                                const uint32_t sel = __ballot_sync(0xFFFFFFFFu, colsz == sz);
                                rem &= ~sel;
                                const int T = maxham[si + sz];
                                mm |= mask16_32(d, max(pc - T - 1, -32768)) & sel;
                                if constexpr (K2 > 0) ee |= mask16_32(d2, max(pc2 - T - 1, -32768)) & sel;
                            }
                            if (!bypass) m = mm;
                            if constexpr (K2 > 0) e2 = ee;
                        }
                        m &= rm;  // (rm is all ones on the fast path, so the bit order is moot)
                        cnt += __popc(m);
                        uint32_t e = m & e2;
                        if constexpr (K2 > 0)
                            e &= perm ? cols_below<true>(P.emit_col_end, gbase) : cols_below<false>(P.emit_col_end, gbase);
                        if (__any_sync(0xFFFFFFFFu, e != 0)) {
                            if (perm) tc_emit<true>(e, gbase, i, q, qlen, P, lane);
                            else tc_emit(e, gbase, i, q, qlen, P, lane);
                        }
                    }
                    if (packed32) groups_done = true;
                }
#pragma unroll 1
                for (int g = 0; g < (groups_done ? 0 : L::kColsPerWarp / 32); ++g) {
                    const int cl = cw + g * 32;  // column within the tile
                    const uint32_t gbase = wbase + g * 32;
                    uint32_t d[32];
                    uint32_t m;
                    bool uni = true;
                    int dummy[32];
                    if (fast) {
                        tmem_ld32(tmem_base + lane_base + as * NT + cl, d);
                        // any survivor in the group <=> max_k D_k > cim1: 16 three-input
                        // maxima (VIMNMX3) decide most groups without building the mask
                        if (!__any_sync(0xFFFFFFFFu, bypass || any_above<KIND>(d, KIND == kKindI8 ? cim1 : cim1_key))) continue;
                        m = bypass ? 0xFFFFFFFFu : survivors32<true, KIND>(d, cim1, dummy, P.neg1);
                    } else {
                        const int kl = static_cast<int>(lo_i) - static_cast<int>(gbase);
                        const int kh = static_cast<int>(hi_i) - static_cast<int>(gbase);
                        const uint32_t rm = low_mask(kh) & ~low_mask(kl);
                        if (!__any_sync(0xFFFFFFFFu, rm != 0)) continue;
                        tmem_ld32(tmem_base + lane_base + as * NT + cl, d);
                        const uint32_t sz0 = L::kEarlyB ? ld_sz<L::kSizeRing>(gsz + cl) : stage_size<L::kKCT>(stage, cl);
                        uni = sz0 == (L::kEarlyB ? ld_sz<L::kSizeRing>(gsz + cl + 31) : stage_size<L::kKCT>(stage, cl + 31));
                        if (uni) {
                            if (sz0 != last_sz) {
                                last_sz = sz0;
                                const int T = maxham[si + sz0];
                                cim1 = pc - T - 1;
                                cim1_2 = pc2 - T - 1;
                                cim1_key = cim1 < 0 ? INT_MIN : __float_as_int(static_cast<float>(cim1) + 0.5f);
                            }
                            m = survivors32<true, KIND>(d, cim1, dummy, P.neg1);
                        } else {
                            m = L::kEarlyB ? survivors_mixed_g<KIND, L::kSizeRing>(d, pc, maxham, si, gsz, cl)
                                           : survivors_mixed<KIND, L::kKCT>(d, pc, maxham, si, stage, cl);
                        }
                        m = bypass ? rm : (m & rm);
                    }
                    finish(cl, gbase, m, uni);
                }
                if (P.tile_counts) {  // this warp's survivors in this tile, per row (rescan locator)
                    P.tile_counts[((info.item * P.tiles_per_item + t) * 4 + part) * kRowTile + rit] =
                        static_cast<uint16_t>(cnt - cnt_tile0);
                    cnt_tile0 = cnt;
                }
                asm volatile("tcgen05.fence::before_thread_sync;");
                __syncwarp();
                if (lane == 0) {
                    if (SSJB_TRACE && P.trace && blockIdx.x == 0 && tile_seq - 1 < 512) P.trace[2048 + 8192 + (tile_seq - 1) * 16 + (warp - 2)] = clock64();
                    if (!acc_released) mbar_arrive_u32(accempty_u32 + 8 * acc_idx);
                    if constexpr (L::kSideRing) mbar_arrive_u32(smem_u32(&e_empty[0]) + 8 * se_idx);
                    else if constexpr (!L::kEarlyB) mbar_arrive_u32(bempty_u32 + 8 * st_idx);
                }
                if (++st_idx == NS) {
                    st_idx = 0;
                    st_phase ^= 1u;
                }
                if (++se_idx == L::NE) {
                    se_idx = 0;
                    se_phase ^= 1u;
                }
                if (++acc_idx == L::kAccSlots) {
                    acc_idx = 0;
                    acc_phase ^= 1u;
                }
            }
            if (valid && cnt) atomicAdd(P.rowcnt + (i - P.row_begin), cnt);
            if (P.item_counts && cnt) atomicAdd(P.item_counts + info.item * kRowTile + rit, cnt);
            ++iseq;
        }
        if (qlen) tc_flush(q, qlen, P, lane);
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(kTmemCols));
}

// Expanded GEMM operands in the core-matrix layout (see the header comment).
// One thread per (row, 16-byte K chunk).
//   int8 (K = b + 32 bytes):  A = bit (u8), B = 2*bit (s8); extension
//     A = 1,1  B = -ceil(pc/2), -floor(pc/2)
//   fp4  (K = b + 64 e2m1 elements, packed two per byte, low nibble first):
//     A = 1.0*bit, B = 2.0*bit; extension A = 1.0 everywhere,
//     B = -6 (x floor(pc/6)) then the remainder as one or two of -1..-4 -- an
//     exact small-integer sum -pc_j in f32 accumulation.
struct ExpandParams {
    const uint64_t* bits;   // level-1 sketches, n_pad x W
    const uint64_t* bits2;  // level-2 Xor sketches (with_l2), n_pad x W2
    const uint32_t* sizes;  // |r| (padded)
    uint8_t* opA;
    uint8_t* opB;
    uint32_t rows;          // rows [row0, rows) are expanded (n_pad: multiple of 8)
    uint32_t row0;          // multiple of 8
    int words, words2;
    int K1;                 // level-1 bytes per row
    int K2;                 // level-2 bytes per row (0: none)
    int fp4;                // level-1 encoding
    int with_size;          // append the 16-byte size chunk (single-CTA kernels)
    int acc_bias, acc_bias2;  // bias the extension adds to level-1 / level-2 accumulators
};

__device__ __forceinline__ uint32_t e2m1_neg(int v) {  // codes of -1, -2, -3, -4, -6
    switch (v) {
        case 1: return 0xAu;
        case 2: return 0xCu;
        case 3: return 0xDu;
        case 4: return 0xEu;
        default: return 0xFu;
    }
}

// int8 segment chunk c (16 bytes = 16 elements) of a sketch with `words` words
// Extension chunk: A holds 1 in bytes [0, nb), B holds shares of
// (acc_bias - pc_j) in those bytes -- floor((v + k) / nb) for byte k, which
// sum to v exactly (Hermite's identity) -- so the GEMM adds acc_bias - pc_j to
// every accumulator of column j.  nb = 2 without a bias (shares -ceil(pc/2),
// -floor(pc/2)); 4 for the level-2 bias of 256 so every share fits an int8.
__device__ __forceinline__ int floor_div_int(int a, int b) { return a >= 0 ? a / b : -((-a + b - 1) / b); }

__device__ __forceinline__ void expand_i8(const uint64_t* row, int words, int c, uint32_t (&a)[4], uint32_t (&b)[4],
                                          int acc_bias = 0) {
    const int bitsn = 64 * words;
    if (16 * c < bitsn) {
        const uint32_t bits16 = static_cast<uint32_t>(row[(16 * c) / 64] >> ((16 * c) % 64)) & 0xFFFFu;
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            const uint32_t bit = (bits16 >> k) & 1u;
            a[k >> 2] |= bit << (8 * (k & 3));
            b[k >> 2] |= (bit * 2u) << (8 * (k & 3));
        }
    } else if (16 * c == bitsn) {
        int pcnt = 0;
        for (int w = 0; w < words; ++w) pcnt += __popcll(row[w]);
        const int nb = acc_bias > 128 ? 4 : 2;
        const int v = acc_bias - pcnt;
        for (int k = 0; k < nb; ++k) {
            a[0] |= 1u << (8 * k);
            b[0] |= static_cast<uint32_t>(static_cast<uint8_t>(floor_div_int(v + k, nb))) << (8 * k);
        }
    }
}

// fp4 segment chunk c (16 bytes = 32 e2m1 elements)
__device__ __forceinline__ void expand_f4(const uint64_t* row, int words, int c, uint32_t (&a)[4], uint32_t (&b)[4]) {
    const int bitsn = 64 * words;
    const int e0 = 32 * c;
    if (e0 < bitsn) {
        const uint32_t bits32 = static_cast<uint32_t>(row[e0 / 64] >> (e0 % 64));
#pragma unroll
        for (int k = 0; k < 32; ++k) {
            const uint32_t bit = (bits32 >> k) & 1u;
            a[k >> 3] |= (bit * 0x2u) << (4 * (k & 7));
            b[k >> 3] |= (bit * 0x4u) << (4 * (k & 7));
        }
    } else {
        int pcnt = 0;
        for (int w = 0; w < words; ++w) pcnt += __popcll(row[w]);
        const int sixes = pcnt / 6, rem = pcnt % 6;
#pragma unroll
        for (int k = 0; k < 32; ++k) {
            const int x = e0 - bitsn + k;  // extension element index
            uint32_t code = 0;
            if (x < sixes) code = 0xFu;
            else if (x == sixes && rem) code = e2m1_neg(rem == 5 ? 3 : rem);
            else if (x == sixes + 1 && rem == 5) code = e2m1_neg(2);
            a[k >> 3] |= 0x2u << (4 * (k & 7));
            b[k >> 3] |= code << (4 * (k & 7));
        }
    }
}

__global__ void expand_operands(ExpandParams P) {
    const int KCT = (P.K1 + P.K2) / 16 + P.with_size;
    const uint64_t idx = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    if (idx >= static_cast<uint64_t>(P.rows - P.row0) * KCT) return;
    const uint32_t r = P.row0 + static_cast<uint32_t>(idx / KCT);
    const int c = static_cast<int>(idx % KCT);
    uint32_t a[4] = {0, 0, 0, 0}, b[4] = {0, 0, 0, 0};
    if (c < P.K1 / 16) {
        const uint64_t* row = P.bits + static_cast<uint64_t>(r) * P.words;
        if (P.fp4) expand_f4(row, P.words, c, a, b);
        else expand_i8(row, P.words, c, a, b, P.acc_bias);
    } else if (c < (P.K1 + P.K2) / 16) {
        expand_i8(P.bits2 + static_cast<uint64_t>(r) * P.words2, P.words2, c - P.K1 / 16, a, b, P.acc_bias2);
    } else {
        a[0] = b[0] = P.sizes[r];  // the size chunk
    }
    const uint64_t off = ((static_cast<uint64_t>(r / 8) * KCT + c) * 8 + (r % 8)) * 16;
    *reinterpret_cast<uint4*>(P.opA + off) = make_uint4(a[0], a[1], a[2], a[3]);
    *reinterpret_cast<uint4*>(P.opB + off) = make_uint4(b[0], b[1], b[2], b[3]);
}

// Per-column data of the no-extension int8 operands: npc2[k] = (-pc(2k), -pc(2k+1))
// as s16x2 (padding rows have empty sketches: pc = 0).
__global__ void column_info(const uint64_t* bits, int words, uint32_t row0, uint32_t rows, uint32_t* npc2) {
    const uint32_t k = row0 / 2 + blockIdx.x * blockDim.x + threadIdx.x;
    if (2 * k >= rows) return;
    int pc[2] = {0, 0};
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const uint32_t r = 2 * k + h;
        if (r >= rows) break;
        for (int w = 0; w < words; ++w) pc[h] += __popcll(bits[static_cast<uint64_t>(r) * words + w]);
    }
    npc2[k] = (static_cast<uint32_t>(-pc[0]) & 0xFFFFu) | (static_cast<uint32_t>(-pc[1]) << 16);
}

}  // namespace dev
}  // namespace ssjb
