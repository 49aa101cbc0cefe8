/* CPU ORACLE -- test infrastructure only (see ssj_oracle.h).
 *
 * A deliberately literal, scalar restatement of the reference algorithm; every
 * function cites the reference file:line it follows.  Speed is irrelevant here:
 * it runs on collections the tests size to finish in seconds, and as the
 * single-core "port" CPU baseline in bench.py. */
#include "ssj_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

typedef __int128 i128;

/* reference src/rational.cpp:43-45 */
static int64_t ceil_div(i128 a, i128 b) { return (int64_t)((a + b - 1) / b); }

int64_t oracle_required_overlap(int64_t p, int64_t q, int64_t sr, int64_t ss) {
    /* Jaccard branch of equivalent_overlap (src/similarity.cpp:99-100), then
     * the max(1, .) clamp of required_overlap (src/similarity.cpp:113-115). */
    int64_t o = ceil_div((i128)p * (sr + ss), (i128)p + q);
    return o < 1 ? 1 : o;
}

uint32_t oracle_hash_token(uint32_t t, int width, int hash) {
    if (hash == 1) { /* src/bitmap.hpp:31-33 */
        uint64_t h = (uint64_t)t * 0x9E3779B97F4A7C15ull;
        return (uint32_t)((h >> 33) % (uint64_t)width);
    }
    return t % (uint32_t)width; /* src/bitmap.hpp:35 */
}

/* Sequential circular next-free-bit probe, src/bitmap.cpp:40-62. */
static void build_next(uint64_t* row, const uint32_t* tokens, size_t count, int width, int hash) {
    int nwords = width / 64;
    if ((int64_t)count >= width) {
        for (int w = 0; w < nwords; ++w) row[w] = ~0ull;
        return;
    }
    for (size_t k = 0; k < count; ++k) {
        int bit = (int)oracle_hash_token(tokens[k], width, hash);
        int word = bit / 64;
        uint64_t free_bits = ~row[word] & (~0ull << (bit % 64));
        for (int step = 0; step <= nwords; ++step) {
            if (free_bits) {
                row[word] |= 1ull << __builtin_ctzll(free_bits);
                break;
            }
            word = (word + 1) % nwords;
            free_bits = ~row[word];
        }
    }
}

/* src/bitmap.cpp:66-88 */
void oracle_build_row(uint64_t* row, const uint32_t* tokens, size_t count, int method, int width,
                      int hash) {
    int nwords = width / 64;
    for (int w = 0; w < nwords; ++w) row[w] = 0;
    if (method == 2) {
        build_next(row, tokens, count, width, hash);
        return;
    }
    for (size_t k = 0; k < count; ++k) {
        uint32_t bit = oracle_hash_token(tokens[k], width, hash);
        if (method == 0)
            row[bit / 64] |= 1ull << (bit % 64);
        else
            row[bit / 64] ^= 1ull << (bit % 64);
    }
}

/* src/bitmap.cpp:145-158 */
void oracle_build_bitmaps(const uint32_t* tokens, const uint64_t* offsets, size_t n, int method,
                          int width, int hash, uint64_t* out) {
    size_t w = (size_t)(width / 64);
    for (size_t r = 0; r < n; ++r)
        oracle_build_row(out + r * w, tokens + offsets[r], (size_t)(offsets[r + 1] - offsets[r]),
                         method, width, hash);
}

/* hamming + overlap_upper_bound_words + bitmap_filter_skip,
 * src/bitmap.cpp:119-143 */
static int filter_skip(int64_t size_r, int64_t size_s, const uint64_t* br, const uint64_t* bs,
                       int nwords, int64_t minov, int64_t cutoff) {
    if (size_r > cutoff) return 0;
    int64_t ham = 0;
    for (int w = 0; w < nwords; ++w) ham += __builtin_popcountll(br[w] ^ bs[w]);
    int64_t slack = size_r + size_s - ham;
    int64_t bound = slack <= 0 ? 0 : slack / 2;
    return bound < minov;
}

/* src/similarity.cpp:168-185 */
int oracle_verify(const uint32_t* a, size_t na, const uint32_t* b, size_t nb, int64_t minov,
                  int64_t* overlap) {
    size_t i = 0, j = 0;
    int64_t o = 0;
    while (i < na && j < nb) {
        size_t ra = na - i, rb = nb - j;
        int64_t best = o + (int64_t)(ra < rb ? ra : rb);
        if (best < minov) {
            *overlap = o;
            return 0;
        }
        if (a[i] == b[j]) {
            ++o;
            ++i;
            ++j;
        } else if (a[i] < b[j]) {
            ++i;
        } else {
            ++j;
        }
    }
    *overlap = o;
    return o >= minov;
}

typedef struct pair_vec {
    oracle_pair* data;
    size_t size, cap;
} pair_vec;

static int push_pair(pair_vec* v, uint32_t r, uint32_t s, int64_t o) {
    if (v->size == v->cap) {
        size_t nc = v->cap ? v->cap * 2 : 256;
        oracle_pair* nd = (oracle_pair*)realloc(v->data, nc * sizeof(oracle_pair));
        if (!nd) return -1;
        v->data = nd;
        v->cap = nc;
    }
    v->data[v->size].id_r = r;
    v->data[v->size].id_s = s;
    v->data[v->size].overlap = o;
    v->size++;
    return 0;
}

/* ResultPair::operator<, src/report.hpp:16-19 */
static int pair_cmp(const void* x, const void* y) {
    const oracle_pair* a = (const oracle_pair*)x;
    const oracle_pair* b = (const oracle_pair*)y;
    if (a->id_r != b->id_r) return a->id_r < b->id_r ? -1 : 1;
    if (a->id_s != b->id_s) return a->id_s < b->id_s ? -1 : 1;
    return 0;
}

#define SIZE_OF(r) ((int64_t)(offsets[(r) + 1] - offsets[(r)]))

/* src/parallel_join.cpp:40-140, one worker (worker count is unobservable,
 * reference tests/test_parallel.cpp:37-59).  Verification is done inline in
 * the order the reference's serial pass would meet the pairs; the outcome is
 * identical because verification is a pure function of the pair. */
int oracle_par_bitmap_join(const uint32_t* tokens, const uint64_t* offsets, size_t n, int64_t p,
                           int64_t q, int bitmap_enabled, int method, int width, int hash,
                           int64_t cutoff, int64_t capacity, size_t row_begin, size_t row_end,
                           oracle_pair** pairs, size_t* pair_count, oracle_counters* counters) {
    return oracle_par_bitmap_join_store(tokens, offsets, n, p, q, bitmap_enabled, method, width, hash,
                                        cutoff, capacity, row_begin, row_end, NULL, pairs, pair_count,
                                        counters);
}

int oracle_par_bitmap_join_store(const uint32_t* tokens, const uint64_t* offsets, size_t n, int64_t p,
                                 int64_t q, int bitmap_enabled, int method, int width, int hash,
                                 int64_t cutoff, int64_t capacity, size_t row_begin, size_t row_end,
                                 const uint64_t* prebuilt, oracle_pair** pairs, size_t* pair_count,
                                 oracle_counters* counters) {
    memset(counters, 0, sizeof(*counters));
    *pairs = NULL;
    *pair_count = 0;
    if (capacity < 1) return -1;
    if (row_end == 0 || row_end > n) row_end = n;
    int nwords = width / 64;
    uint64_t* owned = NULL;
    const uint64_t* store = prebuilt;
    if (bitmap_enabled && !store) {
        owned = (uint64_t*)calloc(n * (size_t)nwords + 1, sizeof(uint64_t));
        if (!owned) return -1;
        oracle_build_bitmaps(tokens, offsets, n, method, width, hash, owned);
        store = owned;
    }
    pair_vec out = {0, 0, 0};
    for (size_t i = row_begin; i < row_end; ++i) {
        int64_t si = SIZE_OF(i);
        /* src/parallel_join.cpp:66-70: partition_point over [0, i) */
        int64_t min_size = ceil_div((i128)p * si, q);
        size_t lo = 0, hi = i;
        while (lo < hi) {
            size_t mid = lo + (hi - lo) / 2;
            if (SIZE_OF(mid) < min_size)
                lo = mid + 1;
            else
                hi = mid;
        }
        size_t j0 = lo;
        int64_t buffered = 0;
        for (size_t j = j0; j < i; ++j) {
            counters->candidates += 1;
            int64_t sj = SIZE_OF(j);
            int64_t minov = oracle_required_overlap(p, q, si, sj);
            if (bitmap_enabled) {
                counters->bitmap_tested += 1;
                if (filter_skip(si, sj, store + i * (size_t)nwords, store + j * (size_t)nwords,
                                nwords, minov, cutoff)) {
                    counters->pruned_bitmap += 1;
                    continue;
                }
            }
            /* buffered pair (j, i) -> verified */
            int64_t ov;
            counters->verified += 1;
            if (oracle_verify(tokens + offsets[j], (size_t)sj, tokens + offsets[i], (size_t)si,
                              minov, &ov)) {
                counters->matched += 1;
                if (push_pair(&out, (uint32_t)j, (uint32_t)i, ov)) goto oom;
            }
            if (++buffered == capacity) {
                counters->saturated_records += 1;
                if (j + 1 < i) {
                    counters->candidates += (uint64_t)(i - j - 1);
                    /* bypass: every remaining window pair is verified as-is */
                    for (size_t k = j + 1; k < i; ++k) {
                        int64_t sk = SIZE_OF(k);
                        int64_t mk = oracle_required_overlap(p, q, sk, si);
                        counters->verified += 1;
                        if (oracle_verify(tokens + offsets[k], (size_t)sk, tokens + offsets[i],
                                          (size_t)si, mk, &ov)) {
                            counters->matched += 1;
                            if (push_pair(&out, (uint32_t)k, (uint32_t)i, ov)) goto oom;
                        }
                    }
                }
                break;
            }
        }
    }
    free(owned);
    qsort(out.data, out.size, sizeof(oracle_pair), pair_cmp);
    *pairs = out.data;
    *pair_count = out.size;
    return 0;
oom:
    free(owned);
    free(out.data);
    return -1;
}

/* src/join.cpp:91-126 (self-join branch) */
int oracle_naive_join(const uint32_t* tokens, const uint64_t* offsets, size_t n, int64_t p,
                      int64_t q, oracle_pair** pairs, size_t* pair_count,
                      oracle_counters* counters) {
    memset(counters, 0, sizeof(*counters));
    pair_vec out = {0, 0, 0};
    for (size_t j = 1; j < n; ++j) {
        for (size_t i = 0; i < j; ++i) {
            counters->candidates += 1;
            counters->verified += 1;
            int64_t ov;
            int64_t minov = oracle_required_overlap(p, q, SIZE_OF(i), SIZE_OF(j));
            if (oracle_verify(tokens + offsets[i], (size_t)SIZE_OF(i), tokens + offsets[j],
                              (size_t)SIZE_OF(j), minov, &ov)) {
                counters->matched += 1;
                if (push_pair(&out, (uint32_t)i, (uint32_t)j, ov)) {
                    free(out.data);
                    return -1;
                }
            }
        }
    }
    qsort(out.data, out.size, sizeof(oracle_pair), pair_cmp);
    *pairs = out.data;
    *pair_count = out.size;
    return 0;
}

/* isqrt_ceil of src/rational.cpp:51-71 (Newton from a long double estimate,
 * exact correction) */
static uint64_t isqrt_ceil_u128(unsigned __int128 v) {
    if (v == 0) return 0;
    unsigned __int128 m = v - 1, x;
    if (m == 0) return 1;
    x = (unsigned __int128)sqrtl((long double)m);
    if (x == 0) x = 1;
    for (int i = 0; i < 6; ++i) {
        unsigned __int128 nx = (x + m / x) >> 1;
        if (nx == x) break;
        x = nx;
    }
    while (x * x > m) --x;
    while ((x + 1) * (x + 1) <= m) ++x;
    return (uint64_t)x + 1;
}

int64_t oracle_required_overlap_sim(int sim, int64_t p, int64_t q, int64_t sr, int64_t ss) {
    /* equivalent_overlap (src/similarity.cpp:93-111) for Overlap 0 / Jaccard 1 /
     * Cosine 2 / Dice 3, then the max(1, .) clamp (:113-115) */
    int64_t o = 0;
    switch (sim) {
        case 0: o = p; break;
        case 1: o = ceil_div((i128)p * (sr + ss), (i128)p + q); break;
        case 2: {
            unsigned __int128 target = (unsigned __int128)p * (unsigned __int128)p;
            target *= (unsigned __int128)sr * (unsigned __int128)ss;
            o = ceil_div((i128)isqrt_ceil_u128(target), (i128)q);
            break;
        }
        case 3: o = ceil_div((i128)p * (sr + ss), (i128)2 * q); break;
        default: return -1;
    }
    return o < 1 ? 1 : o;
}

int oracle_naive_join_sim(const uint32_t* rt, const uint64_t* ro, size_t rn, const uint32_t* st,
                          const uint64_t* so, size_t sn, int self_join, int sim, int64_t p, int64_t q,
                          oracle_pair** pairs, size_t* pair_count, oracle_counters* counters) {
    /* src/join.cpp:91-126: self (pairs (i, j), i < j) or R x S (pairs (r, s)) */
    memset(counters, 0, sizeof(*counters));
    pair_vec out = {0, 0, 0};
    if (self_join) {
        st = rt;
        so = ro;
        sn = rn;
    }
    for (size_t a = 0; a < (self_join ? sn : rn); ++a) {
        size_t bend = self_join ? a : sn;
        for (size_t b = 0; b < bend; ++b) {
            /* self: r = b (earlier), s = a; RS: r = a, s = b */
            size_t ri = self_join ? b : a, si = self_join ? a : b;
            int64_t nr = (int64_t)(ro[ri + 1] - ro[ri]), ns = (int64_t)(so[si + 1] - so[si]);
            int64_t ov, minov = oracle_required_overlap_sim(sim, p, q, nr, ns);
            counters->candidates += 1;
            counters->verified += 1;
            if (oracle_verify(rt + ro[ri], (size_t)nr, st + so[si], (size_t)ns, minov, &ov)) {
                counters->matched += 1;
                if (push_pair(&out, (uint32_t)ri, (uint32_t)si, ov)) {
                    free(out.data);
                    return -1;
                }
            }
        }
    }
    qsort(out.data, out.size, sizeof(oracle_pair), pair_cmp);
    *pairs = out.data;
    *pair_count = out.size;
    return 0;
}

static int u32_cmp(const void* x, const void* y) {
    uint32_t a = *(const uint32_t*)x, b = *(const uint32_t*)y;
    return a < b ? -1 : (a > b ? 1 : 0);
}

typedef struct rec_view {
    const uint32_t* t;
    size_t n;
} rec_view;

/* records by (size, lexicographic token sequence), src/collection.cpp:49-52 */
static int rec_cmp(const void* x, const void* y) {
    const rec_view* a = (const rec_view*)x;
    const rec_view* b = (const rec_view*)y;
    if (a->n != b->n) return a->n < b->n ? -1 : 1;
    for (size_t k = 0; k < a->n; ++k)
        if (a->t[k] != b->t[k]) return a->t[k] < b->t[k] ? -1 : 1;
    return 0;
}

/* src/collection.cpp:44-54 */
void oracle_canonicalize(const uint32_t* tokens, const uint64_t* offsets, size_t n,
                         uint32_t* out_tokens, uint64_t* out_offsets) {
    size_t total = n ? (size_t)offsets[n] : 0;
    uint32_t* tmp = (uint32_t*)malloc((total + 1) * sizeof(uint32_t));
    rec_view* views = (rec_view*)malloc((n + 1) * sizeof(rec_view));
    size_t w = 0;
    for (size_t r = 0; r < n; ++r) {
        size_t b = (size_t)offsets[r], e = (size_t)offsets[r + 1];
        size_t start = w;
        memcpy(tmp + w, tokens + b, (e - b) * sizeof(uint32_t));
        qsort(tmp + w, e - b, sizeof(uint32_t), u32_cmp);
        size_t k = 0;
        for (size_t x = 0; x < e - b; ++x)
            if (x == 0 || tmp[start + x] != tmp[start + x - 1]) tmp[start + k++] = tmp[start + x];
        views[r].t = tmp + start;
        views[r].n = k;
        w = start + (e - b);
    }
    qsort(views, n, sizeof(rec_view), rec_cmp);
    out_offsets[0] = 0;
    for (size_t r = 0; r < n; ++r) {
        memcpy(out_tokens + out_offsets[r], views[r].t, views[r].n * sizeof(uint32_t));
        out_offsets[r + 1] = out_offsets[r] + views[r].n;
    }
    free(views);
    free(tmp);
}

/* src/bounds.cpp:13-35 */
double oracle_expected_bound(int method, int b, int64_t n) {
    double bn = (double)b, nn = (double)n;
    if (method == 0) {
        double log_x = log1p(-1.0 / bn);
        return nn + bn * exp(2.0 * nn * log_x) - bn * exp(nn * log_x);
    }
    if (method == 1) {
        if (b == 1) return nn - 0.25 * (1.0 - ((2 * n) % 2 == 0 ? 1.0 : -1.0));
        double log_x = log1p(-2.0 / bn);
        return nn - bn / 4.0 * (1.0 - exp(2.0 * nn * log_x));
    }
    double v = nn * nn / bn;
    return v < nn ? v : nn;
}

/* src/bounds.cpp:78-107: doubling + bisection over the monotone predicate
 * E(b, n)/n <= tau, tau converted from Jaccard space by 2j/(1+j). */
int64_t oracle_cutoff(int method, int b, int64_t num, int64_t den, int jaccard_space) {
    int64_t tn = num, td = den;
    if (jaccard_space) {
        tn = 2 * num;
        td = num + den;
    }
    /* Rational normalisation does not change the double value except through
     * rounding of num/den; keep the reduced form as the reference does. */
    int64_t a = tn < 0 ? -tn : tn, c = td;
    while (c) {
        int64_t t = a % c;
        a = c;
        c = t;
    }
    if (a > 1) {
        tn /= a;
        td /= a;
    }
    double tau = (double)tn / (double)td;
    const int64_t cap = (int64_t)1 << 26;
#define PRED(x) (oracle_expected_bound(method, b, (x)) / (double)(x) <= tau)
    if (!PRED(1)) return 0;
    int64_t lo = 1, hi = 2;
    while (hi <= cap && PRED(hi)) {
        lo = hi;
        hi *= 2;
    }
    if (hi > cap) return INT64_MAX;
    while (lo + 1 < hi) {
        int64_t mid = lo + (hi - lo) / 2;
        if (PRED(mid))
            lo = mid;
        else
            hi = mid;
    }
#undef PRED
    return lo;
}

void oracle_free(void* p) { free(p); }
