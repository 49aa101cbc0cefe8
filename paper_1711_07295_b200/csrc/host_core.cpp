// Host-side core: see host_core.hpp.  Every behaviour that defines record
// ids, thresholds or error codes cites the reference line it reproduces.
#include "host_core.hpp"

#include <algorithm>
#include <charconv>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <fstream>
#include <functional>
#include <map>
#include <numeric>
#include <random>
#include <sstream>
#include <thread>
#include <unordered_map>
#include <unordered_set>

namespace ssjb {

// ================================================================ rational
Rational::Rational(int64_t n, int64_t d) : num(n), den(d) {
    // reference src/rational.hpp:21-26
    if (den == 0) throw std::invalid_argument("rational: zero denominator");
    if (den < 0) {
        num = -num;
        den = -den;
    }
    int64_t g = std::gcd(num < 0 ? -num : num, den);
    if (g > 1) {
        num /= g;
        den /= g;
    }
}

namespace {
int64_t parse_digits(const std::string& s, const char* what) {
    // <= 18 decimal digits, digits only (reference src/rational.cpp:10-19)
    if (s.empty() || s.size() > 18) throw std::invalid_argument(std::string("rational: bad ") + what);
    int64_t v = 0;
    for (char c : s) {
        if (c < '0' || c > '9') throw std::invalid_argument(std::string("rational: bad ") + what);
        v = v * 10 + (c - '0');
    }
    return v;
}
}  // namespace

Rational parse_rational(const std::string& text) {
    // reference src/rational.cpp:23-41
    size_t slash = text.find('/');
    if (slash != std::string::npos) {
        int64_t p = parse_digits(text.substr(0, slash), "numerator");
        int64_t q = parse_digits(text.substr(slash + 1), "denominator");
        if (q == 0) throw std::invalid_argument("rational: zero denominator");
        return Rational(p, q);
    }
    size_t dot = text.find('.');
    if (dot == std::string::npos) return Rational(parse_digits(text, "integer"), 1);
    std::string whole = text.substr(0, dot), frac = text.substr(dot + 1);
    if (frac.size() > 9) throw std::invalid_argument("rational: too many fractional digits");
    int64_t w = whole.empty() ? 0 : parse_digits(whole, "integer part");
    int64_t f = frac.empty() ? 0 : parse_digits(frac, "fractional part");
    int64_t scale = 1;
    for (size_t i = 0; i < frac.size(); ++i) scale *= 10;
    return Rational(w * scale + f, scale);
}

// ============================================================== similarity
void validate_threshold(Sim f, const Rational& t) {
    // reference src/similarity.cpp:18-27
    if (f == Sim::Overlap) {
        if (t.den != 1 || t.num < 1)
            throw std::invalid_argument("overlap threshold must be a positive integer");
    } else if (t.num <= 0 || Rational(1, 1) < t) {
        throw std::invalid_argument("normalized threshold must be in (0, 1]");
    }
}

Rational jaccard_space(Sim f, const Rational& t) {
    switch (f) {  // reference src/join.cpp:37-50
        case Sim::Jaccard: return t;
        case Sim::Dice:
        case Sim::Cosine: return Rational(t.num, 2 * t.den - t.num);
        case Sim::Overlap: break;
    }
    throw std::invalid_argument("no jaccard-space equivalent for overlap thresholds");
}

Method resolve_combined(Method m, const Rational& t) {
    if (m != Method::Combined) return m;  // reference src/bitmap.cpp:30-36
    if (t <= Rational(56, 100)) return Method::Next;
    if (t >= Rational(73, 100)) return Method::Xor;
    return Method::Set;
}

// =============================================================== analytics
double expected_bound(Method m, int b, int64_t n) {
    // reference src/bounds.cpp:13-35
    if (b < 1) throw std::invalid_argument("bitmap width must be >= 1");
    if (n < 0) throw std::invalid_argument("token count must be >= 0");
    const double bn = static_cast<double>(b), nn = static_cast<double>(n);
    switch (m) {
        case Method::Set: {
            double lx = std::log1p(-1.0 / bn);
            return nn + bn * std::exp(2.0 * nn * lx) - bn * std::exp(nn * lx);
        }
        case Method::Xor: {
            if (b == 1) return nn - 0.25 * (1.0 - ((2 * n) % 2 == 0 ? 1.0 : -1.0));
            double lx = std::log1p(-2.0 / bn);
            return nn - bn / 4.0 * (1.0 - std::exp(2.0 * nn * lx));
        }
        case Method::Next: return std::min(nn * nn / bn, nn);
        case Method::Combined: break;
    }
    throw std::invalid_argument("expected_bound needs a concrete method");
}

namespace {
// Largest n >= 1 with a monotone predicate true: doubling then bisection,
// capped at 2^26 (reference src/bounds.cpp:78-92).
int64_t largest_true(const std::function<bool(int64_t)>& pred) {
    constexpr int64_t kCap = int64_t{1} << 26;
    if (!pred(1)) return 0;
    int64_t lo = 1, hi = 2;
    while (hi <= kCap && pred(hi)) {
        lo = hi;
        hi *= 2;
    }
    if (hi > kCap) return kUnlimited;
    while (lo + 1 < hi) {
        int64_t mid = lo + (hi - lo) / 2;
        (pred(mid) ? lo : hi) = mid;
    }
    return lo;
}
}  // namespace

int64_t cutoff(Method m, int b, const Rational& t, bool space_jaccard) {
    // reference src/bounds.cpp:96-107
    if (t.num <= 0 || Rational(1, 1) < t)
        throw std::invalid_argument("cutoff threshold must be in (0, 1]");
    Rational tau = space_jaccard ? Rational(2 * t.num, t.num + t.den) : t;
    const double td = tau.to_double();
    return largest_true([&](int64_t n) { return expected_bound(m, b, n) / static_cast<double>(n) <= td; });
}

int64_t cutoff_for_overlap(Method m, int b, int64_t tau) {
    if (tau < 1) throw std::invalid_argument("overlap threshold must be >= 1");
    return largest_true([&](int64_t n) { return expected_bound(m, b, n) <= static_cast<double>(tau); });
}

namespace {
uint32_t hash_token(uint32_t t, int width, int hash) {
    if (hash == 1) return static_cast<uint32_t>(((static_cast<uint64_t>(t) * 0x9E3779B97F4A7C15ull) >> 33) %
                                                static_cast<uint64_t>(width));
    return t % static_cast<uint32_t>(width);
}

// Host sketch of one record: used only by the Monte-Carlo analytics entry point.
void host_sketch(std::vector<uint64_t>& row, const std::vector<uint32_t>& toks, int width, Method m) {
    std::fill(row.begin(), row.end(), 0);
    const int nw = width / 64;
    if (m == Method::Next) {
        if (static_cast<int64_t>(toks.size()) >= width) {
            std::fill(row.begin(), row.end(), ~0ull);
            return;
        }
        for (uint32_t t : toks) {
            int bit = static_cast<int>(hash_token(t, width, 0));
            int word = bit / 64;
            uint64_t fb = ~row[word] & (~0ull << (bit % 64));
            for (int step = 0; step <= nw; ++step) {
                if (fb) {
                    row[word] |= 1ull << __builtin_ctzll(fb);
                    break;
                }
                word = (word + 1) % nw;
                fb = ~row[word];
            }
        }
        return;
    }
    for (uint32_t t : toks) {
        uint32_t bit = hash_token(t, width, 0);
        if (m == Method::Set)
            row[bit / 64] |= 1ull << (bit % 64);
        else
            row[bit / 64] ^= 1ull << (bit % 64);
    }
}
}  // namespace

double monte_carlo_bound(Method m, int b, int64_t n, int64_t trials, uint64_t seed) {
    // reference src/bounds.cpp:37-71
    if (trials < 1) throw std::invalid_argument("trials must be >= 1");
    if (b <= 0 || b % 64 != 0) throw std::invalid_argument("bitmap width must be a positive multiple of 64");
    if (m == Method::Combined) throw std::invalid_argument("combined method must be resolved before building");
    if (n < 0) throw std::length_error("token count must be >= 0");
    std::mt19937_64 rng(seed);
    const size_t count = static_cast<size_t>(n);
    std::vector<uint32_t> tr(count), ts(count);
    std::vector<uint64_t> rr(b / 64), rs(b / 64);
    std::unordered_set<uint32_t> seen;
    seen.reserve(2 * count);
    double total = 0.0;
    for (int64_t t = 0; t < trials; ++t) {
        seen.clear();
        auto draw = [&]() {
            uint32_t v;
            do { v = static_cast<uint32_t>(rng()); } while (!seen.insert(v).second);
            return v;
        };
        for (size_t i = 0; i < count; ++i) tr[i] = draw();
        for (size_t i = 0; i < count; ++i) ts[i] = draw();
        host_sketch(rr, tr, b, m);
        host_sketch(rs, ts, b, m);
        int64_t ham = 0;
        for (size_t w = 0; w < rr.size(); ++w) ham += __builtin_popcountll(rr[w] ^ rs[w]);
        total += static_cast<double>(2 * n - ham) / 2.0;
    }
    return total / static_cast<double>(trials);
}

// ============================================================== collection
int64_t Collection::median_size() const {
    if (size() == 0) return 0;
    return rec_size((size() - 1) / 2);  // reference src/collection.cpp:13-17
}

double Collection::mean_size() const {
    if (size() == 0) return 0.0;
    return static_cast<double>(tokens.size()) / static_cast<double>(size());
}

// ------------------------------------------------------- host parallelism
// Host threads for ingest (parse, canonical sort, write): SSJB_HOST_THREADS or
// the hardware concurrency, at most 64.
unsigned host_threads() {
    static const unsigned t = []() {
        const char* v = std::getenv("SSJB_HOST_THREADS");
        long x = v && *v ? std::strtol(v, nullptr, 10) : static_cast<long>(std::thread::hardware_concurrency());
        return static_cast<unsigned>(std::max(1L, std::min(64L, x)));
    }();
    return t;
}

namespace {

// f(t, begin, end) over T contiguous slices of [0, n); serial below `grain`.
template <class F>
void parallel_for(size_t n, F&& f, size_t grain = 1 << 14) {
    const unsigned T = static_cast<unsigned>(std::max<size_t>(1, std::min<size_t>(host_threads(), n / grain)));
    if (T <= 1) {
        f(0u, size_t(0), n);
        return;
    }
    std::vector<std::thread> th;
    std::exception_ptr err;
    std::mutex mu;
    for (unsigned t = 0; t < T; ++t) {
        const size_t a = n * t / T, b = n * (t + 1) / T;
        th.emplace_back([&, t, a, b]() {
            try {
                f(t, a, b);
            } catch (...) {
                std::lock_guard<std::mutex> lk(mu);
                if (!err) err = std::current_exception();
            }
        });
    }
    for (auto& x : th) x.join();
    if (err) std::rethrow_exception(err);
}

// Parallel merge sort: T sorted slices, then rounds of pairwise merges.
template <class T, class Less>
void parallel_sort(std::vector<T>& v, Less less) {
    const size_t n = v.size();
    unsigned P = static_cast<unsigned>(std::max<size_t>(1, std::min<size_t>(host_threads(), n / (1 << 15))));
    if (P <= 1) {
        std::sort(v.begin(), v.end(), less);
        return;
    }
    std::vector<size_t> cut(P + 1);
    for (unsigned k = 0; k <= P; ++k) cut[k] = n * k / P;
    parallel_for(P, [&](unsigned, size_t a, size_t b) {
        for (size_t k = a; k < b; ++k) std::sort(v.begin() + cut[k], v.begin() + cut[k + 1], less);
    }, 1);
    std::vector<T> tmp(n);
    std::vector<T>* src = &v;
    std::vector<T>* dst = &tmp;
    while (cut.size() > 2) {
        std::vector<size_t> next;
        const size_t runs = cut.size() - 1;
        std::vector<std::thread> th;
        for (size_t k = 0; k < runs; k += 2) {
            next.push_back(cut[k]);
            if (k + 1 < runs) {
                th.emplace_back([=, &less]() {
                    std::merge(src->begin() + cut[k], src->begin() + cut[k + 1], src->begin() + cut[k + 1],
                               src->begin() + cut[k + 2], dst->begin() + cut[k], less);
                });
            } else {
                std::copy(src->begin() + cut[k], src->begin() + cut[k + 1], dst->begin() + cut[k]);
            }
        }
        for (auto& x : th) x.join();
        next.push_back(n);
        cut.swap(next);
        std::swap(src, dst);
    }
    if (src != &v) v.swap(*src);
}

}  // namespace

void canonicalize(Collection& c, std::vector<uint32_t>&& raw, const std::vector<uint64_t>& off) {
    // reference src/collection.cpp:44-54: per-record sort + dedup, then records
    // by (size, lexicographic tokens); id = position.  Host-parallel: records
    // are sorted in slices, the record order is a parallel merge sort over
    // (size, first two tokens, index) keys that touch the token array only on
    // ties, and the canonical CSR is filled by slices.
    const size_t n = off.size() - 1;
    std::vector<uint32_t> len(n);
    parallel_for(n, [&](unsigned, size_t a, size_t b) {
        for (size_t r = a; r < b; ++r) {
            auto rb = raw.begin() + static_cast<ptrdiff_t>(off[r]);
            auto re = raw.begin() + static_cast<ptrdiff_t>(off[r + 1]);
            std::sort(rb, re);
            len[r] = static_cast<uint32_t>(std::unique(rb, re) - rb);
        }
    }, 4096);
    struct Item {
        uint64_t key;  // (t0 << 32 | t1) of the deduplicated record (missing tokens 0)
        uint32_t len;
        uint32_t idx;
    };
    std::vector<Item> items(n);
    parallel_for(n, [&](unsigned, size_t a, size_t b) {
        for (size_t r = a; r < b; ++r) {
            const uint32_t* p = raw.data() + off[r];
            const uint64_t k = (len[r] > 0 ? static_cast<uint64_t>(p[0]) << 32 : 0) | (len[r] > 1 ? p[1] : 0u);
            items[r] = Item{k, len[r], static_cast<uint32_t>(r)};
        }
    });
    const uint32_t* rd = raw.data();
    const uint64_t* od = off.data();
    parallel_sort(items, [rd, od](const Item& x, const Item& y) {
        if (x.len != y.len) return x.len < y.len;
        if (x.key != y.key) return x.key < y.key;
        // same size, same first two tokens: the rest of the sequence, then
        // the input position (std::sort in the reference is not stable, but
        // equal records are indistinguishable in the canonical output)
        const uint32_t* pa = rd + od[x.idx];
        const uint32_t* pb = rd + od[y.idx];
        for (uint32_t k = 2; k < x.len; ++k)
            if (pa[k] != pb[k]) return pa[k] < pb[k];
        return x.idx < y.idx;
    });
    c.offsets.assign(n + 1, 0);
    uint64_t total = 0;
    uint32_t ms = 0;
    for (size_t k = 0; k < n; ++k) {
        total += items[k].len;
        c.offsets[k + 1] = total;
        ms = std::max(ms, items[k].len);
    }
    c.tokens.resize(total);
    c.max_size = ms;
    parallel_for(n, [&](unsigned, size_t a, size_t b) {
        for (size_t k = a; k < b; ++k)
            std::memcpy(c.tokens.data() + c.offsets[k], raw.data() + off[items[k].idx], items[k].len * sizeof(uint32_t));
    });
    // size index of the sorted collection (the length filter's window starts)
    c.first_ge.assign(static_cast<size_t>(c.max_size) + 2, static_cast<uint32_t>(n));
    for (size_t k = n; k-- > 0;) c.first_ge[c.rec_size(k)] = static_cast<uint32_t>(k);
    for (size_t s = c.max_size + 1; s-- > 0;) c.first_ge[s] = std::min(c.first_ge[s], c.first_ge[s + 1]);
}

Collection::~Collection() = default;

std::unique_ptr<Collection> collection_from_csr(const uint32_t* tokens, const uint64_t* offsets, size_t n) {
    std::vector<uint64_t> off(offsets, offsets + n + 1);
    if (off[0] != 0) {
        uint64_t base = off[0];
        for (auto& v : off) v -= base;
        tokens += base;
    }
    for (size_t r = 0; r < n; ++r)
        if (off[r + 1] < off[r]) throw std::invalid_argument("offsets must be non-decreasing");
    std::vector<uint32_t> raw(tokens, tokens + off[n]);
    uint32_t max_id = 0;
    for (uint32_t t : raw) max_id = std::max(max_id, t);
    auto c = std::make_unique<Collection>();
    c->universe = raw.empty() ? 0 : static_cast<uint64_t>(max_id) + 1;
    canonicalize(*c, std::move(raw), off);
    return c;
}

namespace {

// reference src/collection.cpp:97-137 (ids as-is; line-numbered parse errors).
// The file is read whole and cut at line boundaries into one slice per host
// thread; slices parse independently and the first error in file order wins.
std::unique_ptr<Collection> read_id_lines(const std::string& path) {
    std::vector<char> buf;
    {
        std::FILE* f = std::fopen(path.c_str(), "rb");
        if (!f) throw IoError("cannot open " + path);
        std::fseek(f, 0, SEEK_END);
        const long size = std::ftell(f);
        std::fseek(f, 0, SEEK_SET);
        buf.resize(size > 0 ? static_cast<size_t>(size) : 0);
        const size_t got = buf.empty() ? 0 : std::fread(buf.data(), 1, buf.size(), f);
        std::fclose(f);
        if (got != buf.size()) throw IoError("cannot read " + path);
    }
    const size_t L = buf.size();
    const char* d = buf.data();
    const unsigned T = static_cast<unsigned>(std::max<size_t>(1, std::min<size_t>(host_threads(), L >> 20)));
    std::vector<size_t> cut(T + 1, L);
    cut[0] = 0;
    for (unsigned t = 1; t < T; ++t) {  // slices start right after a newline
        size_t p = std::max(cut[t - 1], L * t / T);
        while (p < L && (p == 0 || d[p - 1] != '\n')) ++p;
        cut[t] = p;
    }
    struct Slice {
        std::vector<uint32_t> tokens;
        std::vector<uint64_t> ends;  // per line: token count so far
        uint32_t max_id = 0;
        bool any = false;
        size_t err_line = SIZE_MAX;  // 0-based line within the slice
        std::string err;
    };
    std::vector<Slice> sl(T);
    parallel_for(T, [&](unsigned, size_t ta, size_t tb) {
        for (size_t t = ta; t < tb; ++t) {
            Slice& S = sl[t];
            S.tokens.reserve((cut[t + 1] - cut[t]) / 3);
            size_t pos = cut[t];
            const size_t end = cut[t + 1];
            size_t line = 0;
            // getline semantics: every '\n' ends a line; trailing text without
            // one is a last line
            while (pos < end) {
                size_t eol = pos;
                while (eol < end && d[eol] != '\n') ++eol;
                size_t q = pos;
                while (q < eol) {
                    while (q < eol && d[q] == ' ') ++q;
                    if (q >= eol) break;
                    uint64_t value = 0;
                    while (q < eol && d[q] != ' ') {
                        const char ch = d[q];
                        if (ch < '0' || ch > '9' || value > 0xFFFFFFFFull) {
                            S.err_line = line;
                            S.err = "expected a token id";
                            return;
                        }
                        value = value * 10 + static_cast<uint64_t>(ch - '0');
                        ++q;
                    }
                    if (value > 0xFFFFFFFFull) {
                        S.err_line = line;
                        S.err = "token id out of range";
                        return;
                    }
                    S.tokens.push_back(static_cast<uint32_t>(value));
                    S.max_id = std::max(S.max_id, static_cast<uint32_t>(value));
                    S.any = true;
                }
                S.ends.push_back(S.tokens.size());
                ++line;
                pos = eol + 1;
            }
        }
    }, 1);
    size_t lines_before = 0;
    for (unsigned t = 0; t < T; ++t) {
        if (sl[t].err_line != SIZE_MAX)
            throw ParseError("parse error at line " + std::to_string(lines_before + sl[t].err_line + 1) + ": " +
                             sl[t].err);
        lines_before += sl[t].ends.size();
    }
    std::vector<uint64_t> tok_base(T + 1, 0), line_base(T + 1, 0);
    uint32_t max_id = 0;
    bool any = false;
    for (unsigned t = 0; t < T; ++t) {
        tok_base[t + 1] = tok_base[t] + sl[t].tokens.size();
        line_base[t + 1] = line_base[t] + sl[t].ends.size();
        max_id = std::max(max_id, sl[t].max_id);
        any |= sl[t].any;
    }
    std::vector<uint32_t> raw(tok_base[T]);
    std::vector<uint64_t> off(line_base[T] + 1, 0);
    parallel_for(T, [&](unsigned, size_t ta, size_t tb) {
        for (size_t t = ta; t < tb; ++t) {
            if (!sl[t].tokens.empty())
                std::memcpy(raw.data() + tok_base[t], sl[t].tokens.data(), sl[t].tokens.size() * 4);
            for (size_t k = 0; k < sl[t].ends.size(); ++k) off[line_base[t] + k + 1] = tok_base[t] + sl[t].ends[k];
            std::vector<uint32_t>().swap(sl[t].tokens);
        }
    }, 1);
    std::vector<char>().swap(buf);
    auto c = std::make_unique<Collection>();
    c->universe = any ? static_cast<uint64_t>(max_id) + 1 : 0;
    canonicalize(*c, std::move(raw), off);
    return c;
}

std::vector<std::string> tokenize(const std::string& text, int kind, int q) {
    // reference src/collection.cpp:26-40
    std::vector<std::string> out;
    if (kind == 0) {
        std::istringstream in(text);
        std::string w;
        while (in >> w) out.push_back(w);
        return out;
    }
    if (q < 1) throw std::invalid_argument("q-gram size must be >= 1");
    const size_t qq = static_cast<size_t>(q);
    if (text.size() < qq) return out;
    for (size_t i = 0; i + qq <= text.size(); ++i) out.push_back(text.substr(i, qq));
    return out;
}

// Rarest-first renumbering with ties broken by token text, then canonical
// order (reference src/collection.cpp:58-93).  Keys are any totally ordered
// token type whose order matches the reference's std::string order.
template <typename Key, typename KeyLess>
std::unique_ptr<Collection> build_renumbered(std::vector<std::vector<Key>>& sets, KeyLess key_less) {
    std::unordered_map<Key, uint64_t> freq;
    for (auto& rec : sets) {
        std::sort(rec.begin(), rec.end());  // any total order dedups; ids come from key_less below
        rec.erase(std::unique(rec.begin(), rec.end()), rec.end());
        for (const auto& t : rec) ++freq[t];
    }
    std::vector<std::pair<Key, uint64_t>> order(freq.begin(), freq.end());
    std::sort(order.begin(), order.end(), [&](const auto& a, const auto& b) {
        if (a.second != b.second) return a.second < b.second;
        return key_less(a.first, b.first);
    });
    std::unordered_map<Key, uint32_t> ids;
    ids.reserve(order.size());
    for (size_t k = 0; k < order.size(); ++k) ids.emplace(order[k].first, static_cast<uint32_t>(k));
    std::vector<uint32_t> raw;
    std::vector<uint64_t> off{0};
    for (const auto& rec : sets) {
        for (const auto& t : rec) raw.push_back(ids.at(t));
        off.push_back(raw.size());
    }
    auto c = std::make_unique<Collection>();
    c->universe = order.size();
    canonicalize(*c, std::move(raw), off);
    return c;
}

// Decimal-string order of non-negative integers: the order std::map<std::string>
// gives the reference generator's std::to_string tokens ("10" < "2").
// Digits are compared most-significant first without formatting.
int decimal_digits(uint64_t v, unsigned char* d) {
    int n = 0;
    do {
        d[n++] = static_cast<unsigned char>(v % 10);
        v /= 10;
    } while (v);
    return n;  // least significant first
}

bool decimal_less(int64_t a, int64_t b) {
    unsigned char da[24], db[24];
    const int la = decimal_digits(static_cast<uint64_t>(a), da);
    const int lb = decimal_digits(static_cast<uint64_t>(b), db);
    for (int k = 0; k < la && k < lb; ++k) {
        const unsigned char x = da[la - 1 - k], y = db[lb - 1 - k];
        if (x != y) return x < y;
    }
    return la < lb;
}

double uniform01(std::mt19937_64& rng) {
    return static_cast<double>(rng() >> 11) * 0x1.0p-53;  // reference src/collection.cpp:174-176
}

int64_t poisson_draw(std::mt19937_64& rng, double mean) {
    // Knuth with long double, reference src/collection.cpp:180-189
    long double limit = std::exp(static_cast<long double>(-mean));
    int64_t k = 0;
    long double p = 1.0L;
    do {
        ++k;
        p *= static_cast<long double>(uniform01(rng));
    } while (p > limit);
    return k - 1;
}

}  // namespace

std::unique_ptr<Collection> read_collection(const std::string& path, int input_format, int q) {
    if (input_format == 0) return read_id_lines(path);
    std::ifstream in(path);
    if (!in) throw IoError("cannot open " + path);
    // Any other code is text; q-grams only for SSJ_INPUT_QGRAMS (reference src/capi.cpp:134-140).
    const int kind = input_format == 2 ? 1 : 0;
    const int qq = input_format == 2 ? q : 2;
    std::vector<std::vector<std::string>> sets;
    std::string line;
    while (std::getline(in, line)) sets.push_back(tokenize(line, kind, qq));
    return build_renumbered(sets, std::less<std::string>());
}

void write_collection(const Collection& c, const std::string& path) {
    // reference src/collection.cpp:153-168: one line per record, tokens
    // separated by one space.  Record slices are formatted by the host threads
    // and written in order.
    std::FILE* f = std::fopen(path.c_str(), "wb");
    if (!f) throw IoError("cannot open " + path + " for writing");
    const size_t n = c.size();
    const size_t block = size_t(1) << 16;  // records per formatting task
    const unsigned T = host_threads();
    bool ok = true;
    for (size_t base = 0; base < n && ok; base += block * T) {
        const size_t span = std::min(n - base, block * T);
        std::vector<std::string> out(T);
        parallel_for(span, [&](unsigned t, size_t a, size_t b) {
            std::string& o = out[t];
            o.reserve((c.offsets[base + b] - c.offsets[base + a]) * 8 + (b - a));
            char num[16];
            for (size_t r = base + a; r < base + b; ++r) {
                for (uint64_t k = c.offsets[r]; k < c.offsets[r + 1]; ++k) {
                    if (k != c.offsets[r]) o.push_back(' ');
                    char* e = std::to_chars(num, num + sizeof num, c.tokens[k]).ptr;
                    o.append(num, static_cast<size_t>(e - num));
                }
                o.push_back('\n');
            }
        }, 1024);
        for (auto& o : out)
            if (!o.empty() && std::fwrite(o.data(), 1, o.size(), f) != o.size()) ok = false;
    }
    if (std::fclose(f) != 0) ok = false;
    if (!ok) throw IoError("write failed for " + path);
}

std::unique_ptr<Collection> generate(const GeneratorConfig& cfg) {
    // reference src/collection.cpp:193-254: same RNG stream, same draws, same
    // renumbering (tokens are the decimal strings of the drawn ranks).
    if (cfg.num_sets <= 0) throw std::invalid_argument("generator: num_sets must be > 0");
    if (cfg.mean_size <= 0) throw std::invalid_argument("generator: mean_size must be > 0");
    if (cfg.universe <= 0) throw std::invalid_argument("generator: universe must be > 0");
    std::mt19937_64 rng(cfg.seed);
    std::vector<double> cumulative;
    if (cfg.distribution == 1) {
        cumulative.resize(static_cast<size_t>(cfg.universe));
        double total = 0.0;
        for (int64_t k = 0; k < cfg.universe; ++k) {
            total += 1.0 / std::pow(static_cast<double>(k + 1), cfg.zipf_exponent);
            cumulative[static_cast<size_t>(k)] = total;
        }
        for (auto& v : cumulative) v /= total;
    }
    // guide table: u in [b/G, (b+1)/G) (exact, G a power of two) has its
    // upper_bound in [guide[b], guide[b+1]]; the search runs on that bracket
    constexpr int kGuideBits = 16;
    std::vector<uint32_t> guide;
    if (cfg.distribution == 1) {
        const size_t G = size_t(1) << kGuideBits;
        guide.resize(G + 1);
        for (size_t b = 0; b <= G; ++b)
            guide[b] = static_cast<uint32_t>(
                std::upper_bound(cumulative.begin(), cumulative.end(), std::ldexp(static_cast<double>(b), -kGuideBits)) -
                cumulative.begin());
    }
    const uint64_t span = static_cast<uint64_t>(cfg.universe);
    const uint64_t limit = std::numeric_limits<uint64_t>::max() - std::numeric_limits<uint64_t>::max() % span;
    auto draw_token = [&]() -> int64_t {
        if (cfg.distribution != 1) {
            uint64_t v;
            do { v = rng(); } while (v >= limit);
            return static_cast<int64_t>(v % span);
        }
        double u = uniform01(rng);
        const size_t b = static_cast<size_t>(std::ldexp(u, kGuideBits));  // u < 1
        auto it = std::upper_bound(cumulative.begin() + guide[b], cumulative.begin() + guide[b + 1], u);
        if (it == cumulative.end()) --it;
        return static_cast<int64_t>(it - cumulative.begin());
    };
    // Records as CSR of distinct ranks.  A record draws until it holds `size`
    // distinct ranks (the draw count depends on the repeats, so the stream is
    // consumed serially); membership is a bitmap over the universe with the
    // record's bits cleared afterwards.
    const bool dense = cfg.universe <= (int64_t(1) << 30);
    std::vector<uint64_t> seen(dense ? (static_cast<size_t>(cfg.universe) + 63) / 64 : 0, 0);
    std::unordered_set<int64_t> drawn;
    std::vector<std::vector<int64_t>> sparse;  // records of universes above 2^30
    std::vector<uint32_t> raw;
    std::vector<uint64_t> off{0};
    raw.reserve(static_cast<size_t>(cfg.num_sets * cfg.mean_size * 1.05) + 16);
    off.reserve(static_cast<size_t>(cfg.num_sets) + 1);
    for (int64_t i = 0; i < cfg.num_sets; ++i) {
        int64_t size = 0;
        while (size == 0) size = poisson_draw(rng, cfg.mean_size);
        size = std::min(size, cfg.universe);
        const size_t start = raw.size();
        if (!dense) sparse.emplace_back();
        int64_t have = 0, attempts = 0;
        const int64_t budget = 1000 * size + 1000;
        auto add = [&](int64_t t) {
            if (!dense) {
                if (drawn.insert(t).second) {
                    sparse.back().push_back(t);
                    ++have;
                }
                return;
            }
            uint64_t& w = seen[static_cast<size_t>(t) >> 6];
            const uint64_t bit = uint64_t(1) << (t & 63);
            if (!(w & bit)) {
                w |= bit;
                raw.push_back(static_cast<uint32_t>(t));
                ++have;
            }
        };
        while (have < size && attempts < budget) {
            add(draw_token());
            ++attempts;
        }
        for (int64_t t = 0; have < size; ++t) add(t);
        if (dense)
            for (size_t k = start; k < raw.size(); ++k) seen[raw[k] >> 6] = 0;
        else
            drawn.clear();
        off.push_back(raw.size());
    }
    if (!dense) return build_renumbered(sparse, decimal_less);  // the general renumbering
    // renumber rarest-first, ties by the decimal text of the rank
    // (reference src/collection.cpp:58-93 over std::to_string keys)
    std::vector<uint64_t> freq(static_cast<size_t>(cfg.universe), 0);
    for (uint32_t t : raw) ++freq[t];
    std::vector<uint32_t> order;
    for (size_t t = 0; t < freq.size(); ++t)
        if (freq[t]) order.push_back(static_cast<uint32_t>(t));
    std::sort(order.begin(), order.end(), [&](uint32_t a, uint32_t b) {
        if (freq[a] != freq[b]) return freq[a] < freq[b];
        return decimal_less(a, b);
    });
    std::vector<uint32_t> id(static_cast<size_t>(cfg.universe), 0);
    for (size_t k = 0; k < order.size(); ++k) id[order[k]] = static_cast<uint32_t>(k);
    for (auto& t : raw) t = id[t];
    auto c = std::make_unique<Collection>();
    c->universe = order.size();
    canonicalize(*c, std::move(raw), off);
    return c;
}

// ================================================================= options
ResolvedBitmap resolve_bitmap(const Collection& c, const Options& o) {
    // reference src/join.cpp:52-89
    ResolvedBitmap r;
    r.enabled = o.bitmap_enabled;
    if (!r.enabled) return r;
    r.width = o.bits > 0 ? o.bits : (c.median_size() > 64 ? 128 : 64);
    r.hash = o.hash;
    Method m = o.method;
    if (m == Method::Combined)
        m = o.sim == Sim::Overlap ? Method::Set : resolve_combined(m, jaccard_space(o.sim, o.threshold));
    switch (o.cutoff_mode) {
        case CutoffMode::Off: r.cutoff = kUnlimited; break;
        case CutoffMode::Explicit: r.cutoff = o.cutoff_value; break;
        case CutoffMode::Auto:
            r.cutoff = o.sim == Sim::Overlap ? cutoff_for_overlap(m, r.width, o.threshold.num)
                                             : cutoff(m, r.width, jaccard_space(o.sim, o.threshold), true);
            break;
    }
    r.method = m;
    return r;
}

// ==================================================================== plan
int64_t required_overlap(Sim f, const Rational& t, int64_t size_r, int64_t size_s) {
    // reference src/similarity.cpp:93-115
    const int64_t p = t.num, q = t.den;
    int64_t v = 0;
    switch (f) {
        case Sim::Overlap: v = p; break;
        case Sim::Jaccard: v = ceil_div(static_cast<__int128>(p) * (size_r + size_s), static_cast<__int128>(p) + q); break;
        case Sim::Dice: v = ceil_div(static_cast<__int128>(p) * (size_r + size_s), static_cast<__int128>(2) * q); break;
        case Sim::Cosine: {
            unsigned __int128 target = static_cast<unsigned __int128>(p) * static_cast<unsigned __int128>(p);
            target *= static_cast<unsigned __int128>(size_r) * static_cast<unsigned __int128>(size_s);
            uint64_t root = 0;
            if (target == 1) {
                root = 1;  // isqrt_floor(0) = 0 (src/rational.cpp:51-52)
            } else if (target != 0) {  // isqrt_ceil (src/rational.cpp:51-71)
                const unsigned __int128 m = target - 1;
                unsigned __int128 x = static_cast<unsigned __int128>(std::sqrt(static_cast<long double>(m)));
                if (x == 0) x = 1;
                for (int i = 0; i < 6; ++i) {
                    unsigned __int128 nx = (x + m / x) >> 1;
                    if (nx == x) break;
                    x = nx;
                }
                while (x * x > m) --x;
                while ((x + 1) * (x + 1) <= m) ++x;
                root = static_cast<uint64_t>(x) + 1;
            }
            v = ceil_div(static_cast<__int128>(root), q);
            break;
        }
    }
    return std::max<int64_t>(1, v);
}

LengthWindow length_window(Sim f, const Rational& t, int64_t size_r) {
    // reference src/similarity.cpp:117-142 (sizes and thresholds are non-negative)
    const __int128 p = t.num, q = t.den, n = size_r;
    const int64_t unbounded = std::numeric_limits<int64_t>::max();
    LengthWindow w;
    switch (f) {
        case Sim::Overlap:
            w.lower = t.num;
            w.upper = unbounded;
            break;
        case Sim::Jaccard:
            w.lower = ceil_div(n * p, q);
            w.upper = p == 0 ? unbounded : static_cast<int64_t>(n * q / p);
            break;
        case Sim::Cosine:
            w.lower = ceil_div(n * p * p, q * q);
            w.upper = static_cast<int64_t>(n * q * q / (p * p));
            break;
        case Sim::Dice:
            w.lower = ceil_div(n * p, 2 * q - p);
            w.upper = static_cast<int64_t>(n * (2 * q - p) / p);
            break;
    }
    if (w.lower < 0) w.lower = 0;
    return w;
}

int64_t prefix_length(Sim f, const Rational& t, int64_t size_r, int ell) {
    // reference src/similarity.cpp:144-166
    const __int128 p = t.num, q = t.den, n = size_r;
    int64_t base = 0;
    switch (f) {
        case Sim::Overlap: base = size_r - t.num + 1; break;
        case Sim::Jaccard: base = static_cast<int64_t>(n * (q - p) / q) + 1; break;
        case Sim::Cosine: base = static_cast<int64_t>(n * (q * q - p * p) / (q * q)) + 1; break;
        case Sim::Dice: base = static_cast<int64_t>(n * (2 * q - 2 * p) / (2 * q - p)) + 1; break;
    }
    const int64_t len = base + (ell - 1);
    return std::min<int64_t>(std::max<int64_t>(len, 0), size_r);
}

std::vector<int32_t> minov_table(Sim f, const Rational& t, size_t smax) {
    std::vector<int32_t> m(smax + 1, 1);
    if (f == Sim::Cosine) return m;  // depends on |r|*|s|: computed per pair
    for (size_t S = 0; S <= smax; ++S) {
        const int64_t v = required_overlap(f, t, static_cast<int64_t>(S), 0);
        m[S] = static_cast<int32_t>(std::min<int64_t>(v, std::numeric_limits<int32_t>::max()));
    }
    return m;
}

RsPlan make_rs_plan(const Collection& r, const Collection& s, const Options& o, size_t r_begin, size_t r_end) {
    RsPlan plan;
    plan.sim = o.sim;
    plan.p = o.threshold.num;
    plan.q = o.threshold.den;
    plan.r_begin = std::min(r_begin, r.size());
    plan.r_end = std::max(plan.r_begin, std::min(r_end, r.size()));
    plan.minov = minov_table(o.sim, o.threshold, static_cast<size_t>(r.max_size) + s.max_size);
    plan.cosine = o.sim == Sim::Cosine;
    return plan;
}

uint32_t window_start_of(const Collection& c, const JoinPlan& plan, size_t row) {
    return plan.naive ? 0u : plan.window_start[c.rec_size(row)];
}

JoinPlan make_plan(const Collection& c, const Options& o, size_t row_begin, size_t row_end) {
    JoinPlan plan;
    plan.naive = o.algorithm == Algo::Naive;
    const size_t n = c.size();
    plan.row_begin = std::min(row_begin, n);
    plan.row_end = std::min(row_end, n);
    if (plan.row_end < plan.row_begin) plan.row_end = plan.row_begin;
    plan.p = o.threshold.num;
    plan.q = o.threshold.den;
    plan.capacity = static_cast<uint32_t>(o.buffer_capacity);
    if (!plan.naive) plan.bitmap = resolve_bitmap(c, o);
    const uint32_t ms = c.max_size;
    // minov over S in [0, 2*max_size] (reference src/similarity.cpp:99-100,113-115);
    // NAIVE takes every similarity function (src/join.cpp:91-126)
    const Sim sim = plan.naive ? o.sim : Sim::Jaccard;
    plan.minov = minov_table(sim, o.threshold, 2 * static_cast<size_t>(ms));
    plan.cosine = sim == Sim::Cosine;
    // j0 per size from the collection's size index (reference src/parallel_join.cpp:65-70)
    const std::vector<uint32_t>& first_ge = c.first_ge;
    plan.window_start.resize(static_cast<size_t>(ms) + 1);
    for (size_t s = 0; s <= ms; ++s) {
        int64_t lo = ceil_div(static_cast<__int128>(plan.p) * static_cast<int64_t>(s), plan.q);
        plan.window_start[s] = lo > static_cast<int64_t>(ms) ? static_cast<uint32_t>(n)
                                                             : first_ge[static_cast<size_t>(lo)];
    }
    // sum over rows of (i - j0(i)), one arithmetic series per size class
    uint64_t w = 0;
    for (size_t s = 0; s <= ms; ++s) {
        const uint64_t a = std::max<uint64_t>(first_ge[s], plan.row_begin);
        const uint64_t b = std::min<uint64_t>(first_ge[s + 1], plan.row_end);
        if (a >= b) continue;
        const uint64_t j0 = plan.naive ? 0 : plan.window_start[s];
        const uint64_t from = std::max(a, j0 + 1);  // rows with a non-empty window
        if (from >= b) continue;
        const uint64_t cnt = b - from;
        w += cnt * (from - j0) + cnt * (cnt - 1) / 2;
    }
    plan.window_pairs = w;
    return plan;
}

std::vector<uint64_t> partition_rows(const Collection& c, const JoinPlan& plan, int parts, size_t row_begin,
                                     size_t row_end, uint32_t head_L0, double head_weight) {
    if (parts < 1) throw std::invalid_argument("parts must be >= 1");
    const size_t n = c.size();
    row_end = std::min(row_end, n);
    row_begin = std::min(row_begin, row_end);
    std::vector<uint64_t> bounds(static_cast<size_t>(parts) + 1, row_end);
    bounds[0] = row_begin;
    // per-row work: its window pairs (+1 so empty-window rows still spread),
    // plus head_weight x its pairs in the head-overlap region (rows and
    // columns >= head_L0: K3a's per-pair cost is several times K2's)
    auto work = [&](size_t i) {
        const uint32_t j0 = window_start_of(c, plan, i);
        double w = static_cast<double>(j0 < i ? i - j0 : 0) + 1.0;
        if (i >= head_L0) {
            const size_t lo = std::max<size_t>(head_L0, j0);
            if (i > lo) w += head_weight * static_cast<double>(i - lo);
        }
        return w;
    };
    double total = 0;
    for (size_t i = row_begin; i < row_end; ++i) total += work(i);
    const double per = total / parts;
    double run = 0;
    int g = 1;
    for (size_t i = row_begin; i < row_end && g < parts; ++i) {
        run += work(i);
        while (g < parts && run >= per * g) bounds[static_cast<size_t>(g++)] = i + 1;
    }
    // shard starts on 128-row tile boundaries (the filter's row tile and the
    // tensor-core operand layout want 8-aligned row blocks)
    for (int k = 1; k < parts; ++k) {
        uint64_t b = row_begin + ((bounds[static_cast<size_t>(k)] - row_begin) & ~uint64_t(127));
        bounds[static_cast<size_t>(k)] = std::max(b, bounds[static_cast<size_t>(k - 1)]);
    }
    return bounds;
}

}  // namespace ssjb
