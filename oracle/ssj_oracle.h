/* CPU ORACLE -- test infrastructure only.
 *
 * Plain-C restatement of the reference engine's data-parallel Bitmap-Filter
 * join (SSJ_ALGO_PAR_BITMAP) and of the brute-force NAIVE join, used by
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg as the
 * CHECKER.  The product library (paper_1711_07295_b200/lib/libssjoin.so)
 * never links, loads or calls anything declared here.
 *
 * Parity pinning: tests/test_oracle.py checks this restatement against the
 * reference's own golden vectors (proj/tests/test_bitmap.cpp:47-134,
 * test_similarity.cpp, test_parallel.cpp:73-84, test_capi.cpp:41-98) and
 * against fixtures produced by the UNMODIFIED reference compiled from its
 * sources (oracle/Makefile -> oracle/_ref/libssjoin_ref.so, fixtures written
 * by tests/golden/make_golden.py).
 *
 * All inputs are canonical collections in CSR form: record r owns
 * tokens[offsets[r] .. offsets[r+1]), strictly increasing, records sorted by
 * (size, token sequence) -- the order reference src/collection.cpp:44-54
 * produces; record id == position.
 */
#ifndef SSJ_ORACLE_H
#define SSJ_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct oracle_pair {
    uint32_t id_r;
    uint32_t id_s;
    int64_t overlap;
} oracle_pair;

typedef struct oracle_counters {
    uint64_t candidates;
    uint64_t pruned_bitmap;
    uint64_t bitmap_tested;
    uint64_t verified;
    uint64_t matched;
    uint64_t saturated_records;
} oracle_counters;

/* max(1, ceil(p*(sr+ss)/(p+q)))  -- reference src/similarity.cpp:99-100,113-115 */
int64_t oracle_required_overlap(int64_t p, int64_t q, int64_t sr, int64_t ss);

/* token -> bit index  -- reference src/bitmap.hpp:30-36 (hash 1 = multiplicative) */
uint32_t oracle_hash_token(uint32_t t, int width, int hash);

/* One sketch row of width/64 words. method 0 Set, 1 Xor, 2 Next
 * -- reference src/bitmap.cpp:40-88 */
void oracle_build_row(uint64_t* row, const uint32_t* tokens, size_t count, int method, int width,
                      int hash);

/* Sketch store for the whole collection, row r at out[r*width/64 ...]
 * -- reference src/bitmap.cpp:145-158 */
void oracle_build_bitmaps(const uint32_t* tokens, const uint64_t* offsets, size_t n, int method,
                          int width, int hash, uint64_t* out);

/* Exact merge with early exit; returns 1 when matched, overlap in *overlap
 * -- reference src/similarity.cpp:168-185 */
int oracle_verify(const uint32_t* a, size_t na, const uint32_t* b, size_t nb, int64_t minov,
                  int64_t* overlap);

/* Data-parallel Bitmap-Filter join restricted to rows [row_begin, row_end)
 * (all rows when row_end == 0), reference src/parallel_join.cpp:40-140.
 * bitmap_enabled 0 disables the filter (every window pair is verified).
 * cutoff: the resolved size guard (INT64_MAX = off).  *pairs is malloc'ed,
 * sorted by (id_r, id_s); free with oracle_free.  Returns 0 on success. */
int oracle_par_bitmap_join(const uint32_t* tokens, const uint64_t* offsets, size_t n, int64_t p,
                           int64_t q, int bitmap_enabled, int method, int width, int hash,
                           int64_t cutoff, int64_t capacity, size_t row_begin, size_t row_end,
                           oracle_pair** pairs, size_t* pair_count, oracle_counters* counters);

/* The same join with a prebuilt sketch store (oracle_build_bitmaps of the
 * whole collection at this method/width/hash; NULL: built here), so row blocks
 * of one join share one build. */
int oracle_par_bitmap_join_store(const uint32_t* tokens, const uint64_t* offsets, size_t n, int64_t p,
                                 int64_t q, int bitmap_enabled, int method, int width, int hash,
                                 int64_t cutoff, int64_t capacity, size_t row_begin, size_t row_end,
                                 const uint64_t* prebuilt, oracle_pair** pairs, size_t* pair_count,
                                 oracle_counters* counters);

/* Brute-force self-join, reference src/join.cpp:91-126. */
int oracle_naive_join(const uint32_t* tokens, const uint64_t* offsets, size_t n, int64_t p,
                      int64_t q, oracle_pair** pairs, size_t* pair_count,
                      oracle_counters* counters);

/* required_overlap for sim 0 Overlap / 1 Jaccard / 2 Cosine / 3 Dice
 * -- reference src/similarity.cpp:93-115 (Cosine via isqrt_ceil, src/rational.cpp:51-71) */
int64_t oracle_required_overlap_sim(int sim, int64_t p, int64_t q, int64_t sr, int64_t ss);

/* NAIVE join with any similarity, reference src/join.cpp:91-126: a self-join of
 * (rt, ro, rn) when self_join != 0 (s arguments ignored), else R x S. */
int oracle_naive_join_sim(const uint32_t* rt, const uint64_t* ro, size_t rn, const uint32_t* st,
                          const uint64_t* so, size_t sn, int self_join, int sim, int64_t p, int64_t q,
                          oracle_pair** pairs, size_t* pair_count, oracle_counters* counters);

/* Canonical order of a raw CSR collection (per-record sort + dedup, records by
 * (size, tokens)), reference src/collection.cpp:44-54.  Writes the canonical
 * CSR into out_tokens (capacity >= input token count) / out_offsets (n+1). */
void oracle_canonicalize(const uint32_t* tokens, const uint64_t* offsets, size_t n,
                         uint32_t* out_tokens, uint64_t* out_offsets);

/* Analytics used by cutoff_mode AUTO -- reference src/bounds.cpp:13-35,78-107 */
double oracle_expected_bound(int method, int b, int64_t n);
int64_t oracle_cutoff(int method, int b, int64_t num, int64_t den, int jaccard_space);

void oracle_free(void* p);

#ifdef __cplusplus
}
#endif

#endif
