// Prefix-filter joins on the GPU: AllPairs / PPJoin / PPJoin+
// with the Bitmap Filter as filter2 (inside candidate generation) or filter3
// (after it), GroupJoin and AdaptJoin -- the reference's framework_join,
// group_join and adapt_join (src/join.cpp:132-420) and its probe
// (src/prefix_index.cpp:53-148), with the reference's counters.
//
// The reference probes one record r at a time, walking the postings of r's
// prefix tokens in prefix order and keeping per-candidate state (first touch,
// match count, prune cause) in a scratch array.  Every piece of that state is
// a function of the PAIR alone: the walk meets candidate s once per common
// prefix token, in increasing token order on both sides, and each filter
// decision uses only (r, s, the positions of that common token, the count so
// far).  So the GPU enumerates encounters -- (probe posting g, earlier posting
// a) of the same token list -- in parallel, keeps the one that is the pair's
// FIRST common prefix token (no common token in r[0..i) x s[0..pos)), and
// replays the pair's whole walk from there in one thread: the counters it adds
// are exactly the increments the reference's probe makes for that pair.
// Inverted index: postings (token << 32 | id, pos) sorted by the radix sort,
// so each token's list is id-ascending like the reference's (ids ascend with
// size, build_prefix_index src/prefix_index.cpp:7-27).
#pragma once

#include "kernels.cuh"

namespace ssjb {
namespace dev {

// counter slots (reference JoinCounters, src/prefix_index.hpp:80-94)
enum PfxCounter {
    kPcCandidates = 0,
    kPcPrunedLength,
    kPcPrunedPositional,
    kPcPrunedSuffix,
    kPcPrunedBitmap,
    kPcBitmapTested,
    kPcFilterEvals,
    kPcVerified,
    kPcMatched,
    kPcResults,   // result slots claimed (may exceed the buffer: overflow)
    kPcItems,     // group-pair expansion items claimed
    kPcCand,      // AdaptJoin candidate-list entries claimed
    kPcSlots
};

constexpr int kAdaptMaxEll = 16;  // ell_max supported by the AdaptJoin tallies

struct PrefixParams {
    const uint32_t* tokens;
    const uint64_t* offsets;
    const uint32_t* sizes;
    const uint32_t* rec;              // index id -> record (group representatives); null: identity
    const unsigned long long* pkey;   // sorted postings: token << 32 | index id
    const uint32_t* ppos;             // position of the token in that record
    const unsigned long long* eoff;   // encounter offsets per posting (P + 1 entries)
    unsigned long long P, E;
    const int32_t* plen;              // prefix length per record size (probe / index ell)
    const uint32_t* lower;            // length window per probe size (src/similarity.cpp:117-142)
    const uint32_t* upper;
    SimNeed need;
    int positional, suffix, suffix_depth;
    int f2, f3;                       // bitmap placement (src/join.cpp:143-144)
    const uint64_t* bits;             // sketches (n x words), or null
    int words;
    long long cutoff;
    // results: (s << 32 | r, overlap)
    unsigned long long* res_keys;
    uint32_t* res_ov;
    unsigned long long res_cap;
    unsigned long long* ctr;          // kPcSlots counters
    // GroupJoin: group sizes (grp_begin[g + 1] - grp_begin[g]) and the pair items
    int group_mode;
    const uint32_t* grp_begin;
    uint2* items;
    unsigned long long item_cap;
    // AdaptJoin (mode 2): per-(row, ell) tallies, ell_max prefixes per size
    int ell_max;
    const int32_t* plen_ell;          // plen_ell[(ell - 1) * (max_size + 1) + size]
    uint32_t max_size;
    uint32_t n_rows;
    uint32_t* a_touch;                // [ell_max][n] touched pairs per probe row
    uint32_t* a_alive;                // [ell_max][n] uncaused pairs with count >= ell
    uint32_t* a_len;                  // [ell_max][n] length-pruned (touched)
    uint32_t* a_bmp;                  // [ell_max][n] bitmap-pruned (touched)
    uint32_t* a_bt;                   // [n] bitmap predicate evaluations of the first walk
    const uint8_t* a_ell;             // [n] final ell per probe row (verify pass)
    uint2* a_cand;                    // tally pass: pairs (s, r) that survive some walk
    uint16_t* a_cmask;                // bit l: the pair is a candidate of the walk at ell = l + 1
    unsigned long long a_cand_cap;
};

__device__ __forceinline__ uint32_t pfx_rec(const PrefixParams& P, uint32_t id) {
    return P.rec ? P.rec[id] : id;
}

// true when the sorted spans a[0..na) and b[0..nb) share a token
__device__ __forceinline__ bool spans_intersect(const uint32_t* a, uint32_t na, const uint32_t* b, uint32_t nb) {
    uint32_t x = 0, y = 0;
    while (x < na && y < nb) {
        const uint32_t u = __ldg(a + x), v = __ldg(b + y);
        if (u == v) return true;
        x += u < v;
        y += v < u;
    }
    return false;
}

// next common token of a[ia..na) and b[ib..nb): positions in (ia, ib); false if none
__device__ __forceinline__ bool next_common(const uint32_t* a, uint32_t na, const uint32_t* b, uint32_t nb,
                                            uint32_t& ia, uint32_t& ib) {
    while (ia < na && ib < nb) {
        const uint32_t u = __ldg(a + ia), v = __ldg(b + ib);
        if (u == v) return true;
        ia += u < v;
        ib += v < u;
    }
    return false;
}

__device__ __forceinline__ uint32_t lower_bound_u32(const uint32_t* b, uint32_t nb, uint32_t t) {
    uint32_t lo = 0, len = nb;
    while (len > 0) {
        const uint32_t half = len >> 1;
        if (__ldg(b + lo + half) < t) {
            lo += half + 1;
            len -= half + 1;
        } else {
            len = half;
        }
    }
    return lo;
}

// PPJoin+ suffix filter (reference partition_bound, src/prefix_index.cpp:31-43)
__device__ long long partition_bound(const uint32_t* a, uint32_t na, const uint32_t* b, uint32_t nb, int depth) {
    const long long cap = static_cast<long long>(min(na, nb));
    if (cap == 0 || depth <= 0) return cap;
    const uint32_t mid = na / 2;
    const uint32_t probe = __ldg(a + mid);
    const uint32_t split = lower_bound_u32(b, nb, probe);
    const long long found = (split < nb && __ldg(b + split) == probe) ? 1 : 0;
    const long long left = partition_bound(a, mid, b, split, depth - 1);
    const long long right = partition_bound(a + mid + 1, na - mid - 1, b + split + found,
                                            nb - split - static_cast<uint32_t>(found), depth - 1);
    return min(cap, left + found + right);
}

// Reference bitmap_filter_skip (src/bitmap.cpp:138-143): size_r is the probe's.
__device__ __forceinline__ bool pfx_bitmap_skip(const PrefixParams& P, uint32_t rr, uint32_t ss, uint32_t nr,
                                                uint32_t ns, long long minov) {
    if (static_cast<long long>(nr) > P.cutoff) return false;
    const uint64_t* br = P.bits + static_cast<uint64_t>(rr) * P.words;
    const uint64_t* bs = P.bits + static_cast<uint64_t>(ss) * P.words;
    long long ham = 0;
    for (int w = 0; w < P.words; ++w) ham += __popcll(__ldg(br + w) ^ __ldg(bs + w));
    const long long slack = static_cast<long long>(nr) + ns - ham;
    const long long ub = slack <= 0 ? 0 : slack / 2;
    return ub < minov;
}

// Reference verify (src/similarity.cpp:168-185): merge with early exit.
__device__ __forceinline__ bool pfx_verify(const uint32_t* a, uint32_t na, const uint32_t* b, uint32_t nb,
                                           long long minov, uint32_t& overlap) {
    uint32_t i = 0, j = 0, o = 0;
    while (i < na && j < nb) {
        const long long best = static_cast<long long>(o) + min(na - i, nb - j);
        if (best < minov) return false;
        const uint32_t u = __ldg(a + i), v = __ldg(b + j);
        o += u == v;
        i += u <= v;
        j += v <= u;
    }
    overlap = o;
    return static_cast<long long>(o) >= minov;
}

__device__ __forceinline__ void pfx_count(unsigned long long* acc, int slot, unsigned long long v) {
    acc[slot] += v;
}

// One slot of a global counter per calling lane, one atomic per warp: the
// lanes active at the call (coalesced group) share the leader's claim.
__device__ __forceinline__ unsigned long long warp_claim(unsigned long long* counter) {
    const unsigned m = __activemask();
    const int lane = threadIdx.x & 31;
    const int leader = __ffs(m) - 1;
    unsigned long long base = 0;
    if (lane == leader) base = atomicAdd(counter, static_cast<unsigned long long>(__popc(m)));
    base = __shfl_sync(m, base, leader);
    return base + __popc(m & ((1u << lane) - 1u));
}

__device__ __forceinline__ void pfx_emit(const PrefixParams& P, uint32_t lo, uint32_t hi, uint32_t overlap) {
    const unsigned long long slot = warp_claim(P.ctr + kPcResults);
    if (slot < P.res_cap) {
        P.res_keys[slot] = (static_cast<unsigned long long>(lo) << 32) | hi;
        P.res_ov[slot] = overlap;
    }
}

// Warp-reduce the per-thread counters and add them with one atomic per slot.
__device__ __forceinline__ void pfx_flush(const PrefixParams& P, unsigned long long* acc) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int k = 0; k < kPcResults; ++k) {
        unsigned long long v = acc[k];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
        if (lane == 0 && v) atomicAdd(P.ctr + k, v);
    }
}

// Posting g of the sorted index -> (token, index id, pos); eoff[g]..eoff[g+1]
// are its encounters with the earlier postings of its list.
__device__ __forceinline__ uint64_t pfx_find_posting_from(const PrefixParams& P, unsigned long long e, uint64_t lo) {
    uint64_t len = P.P - lo;  // last g >= lo with eoff[g] <= e
    while (len > 0) {
        const uint64_t half = len >> 1;
        if (P.eoff[lo + half + 1] <= e) {
            lo += half + 1;
            len -= half + 1;
        } else {
            len = half;
        }
    }
    return lo;
}

// Called by all 32 lanes with consecutive encounters (e < E or not): lane 0
// binary-searches the warp's first encounter, the others step forward from
// it (a posting usually holds many encounters) and fall back to a search.
__device__ __forceinline__ uint64_t pfx_find_posting(const PrefixParams& P, unsigned long long e) {
    const unsigned long long e0 = __shfl_sync(0xFFFFFFFFu, e, 0);
    uint64_t g0 = 0;
    if ((threadIdx.x & 31) == 0) g0 = pfx_find_posting_from(P, min(e0, P.E - 1), 0);
    g0 = __shfl_sync(0xFFFFFFFFu, g0, 0);
    if (e >= P.E) return g0;
    uint64_t g = g0;
    for (int step = 0; step < 8; ++step) {
        if (P.eoff[g + 1] > e) return g;
        ++g;
    }
    return pfx_find_posting_from(P, e, g);
}

// AdaptJoin (src/join.cpp:330-420) per pair: the walks use prefixes of
// ell = 1..ell_max and the index holds ell_max prefixes, so the first common
// token is taken over those.  cnt[l]: common tokens inside both records'
// (l + 1)-prefixes = the pair's match count in the walk at ell = l + 1
// (touched iff > 0).  Causes: length (every walk), bitmap (pruned by the
// first walk's in-loop test, then killed on first touch by later walks).
__device__ __forceinline__ void adapt_pair(const PrefixParams& P, uint32_t rr, uint32_t ss, uint32_t nr, uint32_t ns,
                                           const uint32_t* Tr, const uint32_t* Ts, uint32_t i, uint32_t pos,
                                           uint32_t (&cnt)[kAdaptMaxEll], bool& inwin, bool& bskip,
                                           long long& minov) {
    const uint32_t ms1 = P.max_size + 1;
    const int L = P.ell_max;
    inwin = ns >= P.lower[nr] && ns <= P.upper[nr];
    minov = need_overlap(P.need, nr, ns);
    bskip = inwin && P.bits && pfx_bitmap_skip(P, rr, ss, nr, ns, minov);
#pragma unroll
    for (int l = 0; l < kAdaptMaxEll; ++l) cnt[l] = 0;
    uint32_t ii = i, pp = pos;
    const uint32_t plr = static_cast<uint32_t>(P.plen_ell[(L - 1) * ms1 + nr]);
    const uint32_t pls = static_cast<uint32_t>(P.plen_ell[(L - 1) * ms1 + ns]);
    do {
#pragma unroll
        for (int l = 0; l < kAdaptMaxEll; ++l)
            if (l < L && ii < static_cast<uint32_t>(P.plen_ell[l * ms1 + nr]) &&
                pp < static_cast<uint32_t>(P.plen_ell[l * ms1 + ns]))
                ++cnt[l];
        ++ii;
        ++pp;
    } while (next_common(Tr, plr, Ts, pls, ii, pp));
}

// One thread per encounter; the thread holding a pair's first common prefix
// token replays the pair's probe walk (src/prefix_index.cpp:70-133) and the
// join's candidate loop (src/join.cpp:160-181 / :300-326).
__global__ void __launch_bounds__(256, 4) prefix_encounters(PrefixParams P) {
    unsigned long long acc[kPcResults];
#pragma unroll
    for (int k = 0; k < kPcResults; ++k) acc[k] = 0;
    const unsigned long long stride = static_cast<unsigned long long>(gridDim.x) * blockDim.x;
    const unsigned long long start = static_cast<unsigned long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    const unsigned long long Eround = (P.E + 31) / 32 * 32;  // whole warps for the flush
    for (unsigned long long e = start; e < Eround; e += stride) {
        const uint64_t g = pfx_find_posting(P, e);
        if (e >= P.E) continue;
        const uint64_t k = P.eoff[g + 1] - P.eoff[g];
        const uint64_t a = g - k + (e - P.eoff[g]);
        const unsigned long long kg = P.pkey[g], ka = P.pkey[a];
        const uint32_t r = static_cast<uint32_t>(kg), s = static_cast<uint32_t>(ka);
        const uint32_t i = P.ppos[g], pos = P.ppos[a];
        const uint32_t rr = pfx_rec(P, r), ss = pfx_rec(P, s);
        const uint32_t nr = P.sizes[rr], ns = P.sizes[ss];
        const uint32_t* Tr = P.tokens + P.offsets[rr];
        const uint32_t* Ts = P.tokens + P.offsets[ss];
        // first common prefix token of the pair?  (tokens before i / pos are smaller)
        if (spans_intersect(Tr, i, Ts, pos)) continue;
        const unsigned long long factor =
            P.group_mode ? static_cast<unsigned long long>(P.grp_begin[r + 1] - P.grp_begin[r]) *
                               (P.grp_begin[s + 1] - P.grp_begin[s])
                         : 1ull;
        pfx_count(acc, kPcFilterEvals, 1);
        pfx_count(acc, kPcCandidates, factor);
        if (ns < P.lower[nr] || ns > P.upper[nr]) {
            pfx_count(acc, kPcPrunedLength, factor);
            continue;
        }
        const long long minov = need_overlap(P.need, nr, ns);
        const bool bskip = (P.f2 || P.f3) && pfx_bitmap_skip(P, rr, ss, nr, ns, minov);
        const uint32_t plr = static_cast<uint32_t>(P.plen[nr]), pls = static_cast<uint32_t>(P.plen[ns]);
        const bool walk = P.f2 || P.positional;  // decisions at every common token
        long long count = 0;
        int cause = 0;  // 1 positional, 2 suffix, 3 bitmap
        uint32_t ii = i, pp = pos;
        for (;;) {
            if (P.f2) {
                pfx_count(acc, kPcBitmapTested, 1);
                if (bskip) {
                    cause = 3;
                    break;
                }
            }
            if (P.positional) {
                pfx_count(acc, kPcFilterEvals, 1);
                const long long bound = count + 1 + min(static_cast<long long>(nr) - (ii + 1),
                                                        static_cast<long long>(ns) - (pp + 1));
                if (bound < minov) {
                    cause = 1;
                    break;
                }
            }
            if (P.suffix && count == 0) {
                pfx_count(acc, kPcFilterEvals, 1);
                const long long bound = 1 + partition_bound(Tr + ii + 1, nr - ii - 1, Ts + pp + 1, ns - pp - 1,
                                                            P.suffix_depth);
                if (bound < minov) {
                    cause = 2;
                    break;
                }
            }
            ++count;
            if (!walk) break;
            ++ii;
            ++pp;
            if (!next_common(Tr, plr, Ts, pls, ii, pp)) break;
        }
        if (cause) {
            pfx_count(acc, cause == 1 ? kPcPrunedPositional : cause == 2 ? kPcPrunedSuffix : kPcPrunedBitmap, factor);
            continue;
        }
        if (P.group_mode) {  // expanded to record pairs by group_expand
            const unsigned long long slot = warp_claim(P.ctr + kPcItems);
            if (slot < P.item_cap) P.items[slot] = make_uint2(r, s);
            continue;
        }
        if (P.f3) {
            pfx_count(acc, kPcBitmapTested, 1);
            if (bskip) {
                pfx_count(acc, kPcPrunedBitmap, 1);
                continue;
            }
        }
        pfx_count(acc, kPcVerified, 1);
        uint32_t ov = 0;
        if (pfx_verify(Ts, ns, Tr, nr, minov, ov)) {
            pfx_count(acc, kPcMatched, 1);
            pfx_emit(P, s, r, ov);
        }
    }
    pfx_flush(P, acc);
}

// AdaptJoin tally pass: per (probe row, ell) counts of touched, length-pruned,
// bitmap-pruned and surviving (count >= ell) pairs, and the first walk's
// bitmap evaluations.  Consecutive encounters mostly share the probe row, so
// lanes with the same row (__match_any_sync) reduce first and one lane adds.
__global__ void __launch_bounds__(256) adapt_tally(PrefixParams P) {
    const unsigned long long stride = static_cast<unsigned long long>(gridDim.x) * blockDim.x;
    const unsigned long long start = static_cast<unsigned long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    const unsigned long long Eround = (P.E + 31) / 32 * 32;
    const int L = P.ell_max;
    for (unsigned long long e = start; e < Eround; e += stride) {
        uint32_t key = 0xFFFFFFFFu, tmask = 0, amask = 0, btv = 0;
        bool lenp = false, bmpp = false;
        const uint64_t g = pfx_find_posting(P, e);
        if (e < P.E) {
            const uint64_t k = P.eoff[g + 1] - P.eoff[g];
            const uint64_t a = g - k + (e - P.eoff[g]);
            const uint32_t r = static_cast<uint32_t>(P.pkey[g]), s = static_cast<uint32_t>(P.pkey[a]);
            const uint32_t i = P.ppos[g], pos = P.ppos[a];
            const uint32_t nr = P.sizes[r], ns = P.sizes[s];
            const uint32_t* Tr = P.tokens + P.offsets[r];
            const uint32_t* Ts = P.tokens + P.offsets[s];
            if (!spans_intersect(Tr, i, Ts, pos)) {
                uint32_t cnt[kAdaptMaxEll];
                bool inwin, bskip;
                long long minov;
                adapt_pair(P, r, s, nr, ns, Tr, Ts, i, pos, cnt, inwin, bskip, minov);
                key = r;
                lenp = !inwin;
                bmpp = inwin && bskip && cnt[0] > 0;
                if (cnt[0] && inwin && P.bits) btv = bskip ? 1u : cnt[0];
#pragma unroll
                for (int l = 0; l < kAdaptMaxEll; ++l) {
                    if (l < L && cnt[l]) tmask |= 1u << l;
                    if (l < L && cnt[l] >= static_cast<uint32_t>(l + 1)) amask |= 1u << l;
                }
                if (P.a_cand && !lenp && !bmpp && amask) {  // verified iff its row ends on such a walk
                    const unsigned long long slot = warp_claim(P.ctr + kPcCand);
                    if (slot < P.a_cand_cap) {
                        P.a_cand[slot] = make_uint2(s, r);
                        P.a_cmask[slot] = static_cast<uint16_t>(amask);
                    }
                }
            }
        }
        const unsigned grp = __match_any_sync(0xFFFFFFFFu, key);
        if (key == 0xFFFFFFFFu) continue;
        const bool lead = (threadIdx.x & 31) == __ffs(grp) - 1;
        const uint32_t bt = __reduce_add_sync(grp, btv);
        if (lead && bt) atomicAdd(P.a_bt + key, bt);
        for (int l = 0; l < L; ++l) {
            const uint32_t t = (tmask >> l) & 1u;
            const uint32_t nt = __reduce_add_sync(grp, t);
            if (!nt) continue;  // uniform over the group
            const uint32_t nl = __reduce_add_sync(grp, t & (lenp ? 1u : 0u));
            const uint32_t nb = __reduce_add_sync(grp, t & (bmpp ? 1u : 0u));
            const uint32_t na = __reduce_add_sync(grp, t & (!lenp && !bmpp ? (amask >> l) & 1u : 0u));
            if (lead) {
                const uint64_t at = static_cast<uint64_t>(l) * P.n_rows + key;
                atomicAdd(P.a_touch + at, nt);
                if (nl) atomicAdd(P.a_len + at, nl);
                if (nb) atomicAdd(P.a_bmp + at, nb);
                if (na) atomicAdd(P.a_alive + at, na);
            }
        }
    }
}

// AdaptJoin verify pass: the candidates of each probe row's final walk.
__global__ void __launch_bounds__(256) adapt_verify(PrefixParams P) {
    unsigned long long acc[kPcResults];
#pragma unroll
    for (int k = 0; k < kPcResults; ++k) acc[k] = 0;
    const unsigned long long stride = static_cast<unsigned long long>(gridDim.x) * blockDim.x;
    const unsigned long long start = static_cast<unsigned long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    const unsigned long long Eround = (P.E + 31) / 32 * 32;
    for (unsigned long long e = start; e < Eround; e += stride) {
        const uint64_t g = pfx_find_posting(P, e);
        if (e >= P.E) continue;
        const uint64_t k = P.eoff[g + 1] - P.eoff[g];
        const uint64_t a = g - k + (e - P.eoff[g]);
        const uint32_t r = static_cast<uint32_t>(P.pkey[g]), s = static_cast<uint32_t>(P.pkey[a]);
        const uint32_t i = P.ppos[g], pos = P.ppos[a];
        const uint32_t nr = P.sizes[r], ns = P.sizes[s];
        const uint32_t* Tr = P.tokens + P.offsets[r];
        const uint32_t* Ts = P.tokens + P.offsets[s];
        if (spans_intersect(Tr, i, Ts, pos)) continue;
        uint32_t cnt[kAdaptMaxEll];
        bool inwin, bskip;
        long long minov;
        adapt_pair(P, r, s, nr, ns, Tr, Ts, i, pos, cnt, inwin, bskip, minov);
        const bool bpruned = bskip && cnt[0] > 0;
        const int ell = P.a_ell[r];  // the row's final walk
        if (!inwin || bpruned || cnt[ell - 1] < static_cast<uint32_t>(ell)) continue;
        // (verified is counted per row by adapt_rows)
        uint32_t ov = 0;
        if (pfx_verify(Ts, ns, Tr, nr, minov, ov)) {
            pfx_count(acc, kPcMatched, 1);
            pfx_emit(P, s, r, ov);
        }
    }
    pfx_flush(P, acc);
}

// AdaptJoin verify over the tally pass's candidate list (when it fit): the
// pairs whose probe row's final walk (a_ell) keeps them.
__global__ void __launch_bounds__(256) adapt_verify_list(PrefixParams P, unsigned long long count) {
    unsigned long long acc[kPcResults];
#pragma unroll
    for (int k = 0; k < kPcResults; ++k) acc[k] = 0;
    const unsigned long long stride = static_cast<unsigned long long>(gridDim.x) * blockDim.x;
    const unsigned long long cround = (count + 31) / 32 * 32;
    for (unsigned long long k = static_cast<unsigned long long>(blockIdx.x) * blockDim.x + threadIdx.x; k < cround;
         k += stride) {
        if (k >= count) continue;
        const uint2 pr = P.a_cand[k];
        const uint32_t s = pr.x, r = pr.y;
        const int ell = P.a_ell[r];
        if (!((P.a_cmask[k] >> (ell - 1)) & 1u)) continue;
        const uint32_t nr = P.sizes[r], ns = P.sizes[s];
        const long long minov = need_overlap(P.need, nr, ns);
        uint32_t ov = 0;
        if (pfx_verify(P.tokens + P.offsets[s], ns, P.tokens + P.offsets[r], nr, minov, ov)) {
            pfx_count(acc, kPcMatched, 1);
            pfx_emit(P, s, r, ov);
        }
    }
    pfx_flush(P, acc);
}

// ------------------------------------------------------------- index build
// Per index id: its prefix length (count of postings).
__global__ void prefix_counts(const uint32_t* sizes, const uint32_t* rec, const int32_t* plen, uint32_t U,
                              unsigned long long* cnt) {
    const uint32_t u = blockIdx.x * blockDim.x + threadIdx.x;
    if (u >= U) return;
    cnt[u] = static_cast<unsigned long long>(plen[sizes[rec ? rec[u] : u]]);
}

// Warp per index id: postings (token << 32 | id, pos) at base[u].
__global__ void prefix_emit(const uint32_t* tokens, const uint64_t* offsets, const uint32_t* sizes,
                            const uint32_t* rec, const int32_t* plen, uint32_t U, const unsigned long long* base,
                            unsigned long long* keys, uint32_t* pos) {
    const uint32_t u = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (u >= U) return;
    const uint32_t rr = rec ? rec[u] : u;
    const uint32_t L = static_cast<uint32_t>(plen[sizes[rr]]);
    const uint32_t* T = tokens + offsets[rr];
    const unsigned long long b = base[u];
    for (uint32_t i = lane; i < L; i += 32) {
        keys[b + i] = (static_cast<unsigned long long>(T[i]) << 32) | u;
        pos[b + i] = i;
    }
}

// Encounters of posting g: the earlier postings of its token's list.
__global__ void prefix_encounter_counts(const unsigned long long* keys, unsigned long long P,
                                        unsigned long long* cnt) {
    const unsigned long long g = static_cast<unsigned long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (g >= P) return;
    const unsigned long long t = keys[g] >> 32 << 32;
    unsigned long long lo = 0, len = g;  // first index with key >= t
    while (len > 0) {
        const unsigned long long half = len >> 1;
        if (keys[lo + half] < t) {
            lo += half + 1;
            len -= half + 1;
        } else {
            len = half;
        }
    }
    cnt[g] = g - lo;
}

// ------------------------------------------------------------ u64 scan
constexpr int kScan64Threads = 1024;
constexpr int kScan64Items = 4;
constexpr unsigned long long kScan64Tile = kScan64Threads * kScan64Items;

// Exclusive scan of each tile in place; tile totals to sums[blockIdx.x].
__global__ void __launch_bounds__(kScan64Threads) scan64_tiles(unsigned long long* d, unsigned long long n,
                                                               unsigned long long* sums) {
    __shared__ unsigned long long warp_tot[32];
    const unsigned long long base = static_cast<unsigned long long>(blockIdx.x) * kScan64Tile +
                                    static_cast<unsigned long long>(threadIdx.x) * kScan64Items;
    unsigned long long v[kScan64Items];
    unsigned long long t = 0;
#pragma unroll
    for (int k = 0; k < kScan64Items; ++k) {
        v[k] = base + k < n ? d[base + k] : 0ull;
        t += v[k];
    }
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    unsigned long long incl = t;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
        if (lane >= o) incl += y;
    }
    if (lane == 31) warp_tot[w] = incl;
    __syncthreads();
    if (w == 0) {
        unsigned long long x = warp_tot[lane];
        unsigned long long xi = x;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned long long y = __shfl_up_sync(0xFFFFFFFFu, xi, o);
            if (lane >= o) xi += y;
        }
        warp_tot[lane] = xi - x;  // exclusive warp offsets
        if (lane == 31) sums[blockIdx.x] = xi;
    }
    __syncthreads();
    unsigned long long run = warp_tot[w] + incl - t;
#pragma unroll
    for (int k = 0; k < kScan64Items; ++k) {
        if (base + k < n) d[base + k] = run;
        run += v[k];
    }
}

__global__ void scan64_add(unsigned long long* d, unsigned long long n, const unsigned long long* offs) {
    const unsigned long long i = static_cast<unsigned long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) d[i] += offs[i / kScan64Tile];
}

// ------------------------------------------------------------- GroupJoin
// Group starts (src/join.cpp:205-219): record i opens a group unless it has
// the size and the full prefix of record i - 1.
__global__ void group_flags(const uint32_t* tokens, const uint64_t* offsets, const uint32_t* sizes,
                            const int32_t* plen, uint32_t n, unsigned long long* flag) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    bool start = i == 0 || sizes[i] != sizes[i - 1];
    if (!start) {
        const uint32_t L = static_cast<uint32_t>(plen[sizes[i]]);
        const uint32_t* a = tokens + offsets[i];
        const uint32_t* b = tokens + offsets[i - 1];
        for (uint32_t k = 0; k < L; ++k)
            if (a[k] != b[k]) {
                start = true;
                break;
            }
    }
    flag[i] = start ? 1ull : 0ull;
}

// flag scanned (exclusive) -> group begin records; grp_begin[G] = n
__global__ void group_begins(const unsigned long long* scanned, uint32_t n, uint32_t* grp_begin,
                             const uint32_t* sizes, const uint32_t* tokens_unused) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const bool start = (i + 1 < n ? scanned[i + 1] : scanned[n]) != scanned[i];
    if (start) grp_begin[scanned[i]] = i;
    if (i == n - 1) grp_begin[scanned[n]] = n;
}

// Intra-group items (g, g) for groups of >= 2 records; candidates += C(size, 2)
// (src/join.cpp:301-305).
__global__ void group_intra(const uint32_t* grp_begin, uint32_t G, uint2* items, unsigned long long item_cap,
                            unsigned long long* ctr) {
    const uint32_t g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= G) return;
    const unsigned long long sz = grp_begin[g + 1] - grp_begin[g];
    if (sz < 2) return;
    atomicAdd(ctr + kPcCandidates, sz * (sz - 1) / 2);
    const unsigned long long slot = atomicAdd(ctr + kPcItems, 1ull);
    if (slot < item_cap) items[slot] = make_uint2(g, g);
}

__global__ void group_item_sizes(const uint2* items, unsigned long long m, const uint32_t* grp_begin,
                                 unsigned long long* f) {
    const unsigned long long k = static_cast<unsigned long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (k >= m) return;
    const uint2 it = items[k];
    const unsigned long long a = grp_begin[it.x + 1] - grp_begin[it.x];
    const unsigned long long b = grp_begin[it.y + 1] - grp_begin[it.y];
    f[k] = it.x == it.y ? a * (a - 1) / 2 : a * b;
}

// Record pairs of the group items (src/join.cpp:236-260 expand, :306-326
// intra-group): bitmap predicate, exact verification.
__global__ void __launch_bounds__(256) group_expand(PrefixParams P, const uint2* items, unsigned long long m,
                                                    const unsigned long long* foff, unsigned long long total) {
    unsigned long long acc[kPcResults];
#pragma unroll
    for (int k = 0; k < kPcResults; ++k) acc[k] = 0;
    const unsigned long long stride = static_cast<unsigned long long>(gridDim.x) * blockDim.x;
    const unsigned long long Tround = (total + 31) / 32 * 32;
    for (unsigned long long e = static_cast<unsigned long long>(blockIdx.x) * blockDim.x + threadIdx.x;
         e < Tround; e += stride) {
        if (e >= total) continue;
        unsigned long long lo = 0, len = m;  // last item with foff <= e
        while (len > 0) {
            const unsigned long long half = len >> 1;
            if (foff[lo + half + 1] <= e) {
                lo += half + 1;
                len -= half + 1;
            } else {
                len = half;
            }
        }
        const uint2 it = items[lo];
        const unsigned long long k = e - foff[lo];
        const uint32_t ba = P.grp_begin[it.x], bb = P.grp_begin[it.y];
        uint32_t rl, rh;
        if (it.x == it.y) {  // k-th pair (x < y) of the group, row-major by y
            unsigned long long y = static_cast<unsigned long long>((1.0 + sqrt(1.0 + 8.0 * static_cast<double>(k))) * 0.5);
            while (y * (y - 1) / 2 > k) --y;
            while ((y + 1) * y / 2 <= k) ++y;
            const unsigned long long x = k - y * (y - 1) / 2;
            rl = ba + static_cast<uint32_t>(x);
            rh = ba + static_cast<uint32_t>(y);
        } else {  // probe group it.x (later records) x touched group it.y
            const unsigned long long nb = P.grp_begin[it.y + 1] - bb;
            rh = ba + static_cast<uint32_t>(k / nb);
            rl = bb + static_cast<uint32_t>(k % nb);
        }
        const uint32_t nl = P.sizes[rl], nh = P.sizes[rh];
        const long long minov = need_overlap(P.need, nl, nh);
        if (P.bits) {
            pfx_count(acc, kPcBitmapTested, 1);
            if (pfx_bitmap_skip(P, rh, rl, nh, nl, minov)) {
                pfx_count(acc, kPcPrunedBitmap, 1);
                continue;
            }
        }
        pfx_count(acc, kPcVerified, 1);
        uint32_t ov = 0;
        if (pfx_verify(P.tokens + P.offsets[rl], nl, P.tokens + P.offsets[rh], nh, minov, ov)) {
            pfx_count(acc, kPcMatched, 1);
            pfx_emit(P, rl, rh, ov);
        }
    }
    pfx_flush(P, acc);
}

// ------------------------------------------------------------- AdaptJoin
struct AdaptRowParams {
    const uint32_t* tokens;
    const uint64_t* offsets;
    const uint32_t* sizes;
    const unsigned long long* pkey;  // the ell_max index
    unsigned long long P;
    const int32_t* plen_ell;
    const int32_t* ellcap;           // per probe size (src/join.cpp:368-371)
    uint32_t max_size;
    int ell_max;
    double avg;                      // mean record size (src/join.cpp:346)
    uint32_t n;
    const uint32_t *touch, *alive, *len, *bmp, *bt;
    uint8_t* ell_out;
    unsigned long long* ctr;
};

__device__ __forceinline__ unsigned long long pfx_key_bound(const unsigned long long* k, unsigned long long n,
                                                            unsigned long long key) {
    unsigned long long lo = 0, len = n;  // first index with k >= key
    while (len > 0) {
        const unsigned long long half = len >> 1;
        if (k[lo + half] < key) {
            lo += half + 1;
            len -= half + 1;
        } else {
            len = half;
        }
    }
    return lo;
}

// One thread per probe row: the row's ell loop (src/join.cpp:383-393) from
// the tallies, then the row's counters from its final walk (:395-400).
__global__ void adapt_rows(AdaptRowParams A) {
    const uint32_t r = blockIdx.x * blockDim.x + threadIdx.x;
    unsigned long long fe = 0, cand = 0, pl = 0, pb = 0, bt = 0, ver = 0;
    if (r < A.n) {
        const uint32_t nr = A.sizes[r];
        const uint32_t* T = A.tokens + A.offsets[r];
        const uint32_t ms1 = A.max_size + 1;
        const int cap = A.ellcap[nr];
        int ell = 1;
        while (ell < cap) {
            // probe_cost(r, ell + 1): postings of the (ell + 1)-prefix's tokens
            const uint32_t pl1 = static_cast<uint32_t>(A.plen_ell[ell * ms1 + nr]);
            unsigned long long cost = 0;
            for (uint32_t i = 0; i < pl1; ++i) {
                const unsigned long long t = static_cast<unsigned long long>(T[i]) << 32;
                cost += pfx_key_bound(A.pkey, A.P, t + 0x100000000ull) - pfx_key_bound(A.pkey, A.P, t);
            }
            const double c = static_cast<double>(A.alive[static_cast<uint64_t>(ell - 1) * A.n + r]);
            if (!(c * A.avg > static_cast<double>(cost))) break;
            ++ell;
        }
        A.ell_out[r] = static_cast<uint8_t>(ell);
        for (int l = 0; l < ell; ++l) fe += A.touch[static_cast<uint64_t>(l) * A.n + r];
        const uint64_t at = static_cast<uint64_t>(ell - 1) * A.n + r;
        pl = A.len[at];
        pb = A.bmp[at];
        ver = A.alive[at];
        cand = pl + pb + ver;
        bt = A.bt[r];
    }
    unsigned long long v[6] = {fe, cand, pl, pb, bt, ver};
    const int slot[6] = {kPcFilterEvals, kPcCandidates, kPcPrunedLength, kPcPrunedBitmap, kPcBitmapTested,
                         kPcVerified};
#pragma unroll
    for (int k = 0; k < 6; ++k) {
        unsigned long long x = v[k];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xFFFFFFFFu, x, o);
        if ((threadIdx.x & 31) == 0 && x) atomicAdd(A.ctr + slot[k], x);
    }
}

}  // namespace dev
}  // namespace ssjb
