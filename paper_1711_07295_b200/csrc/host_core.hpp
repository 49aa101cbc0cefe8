// Host-side core of the B200 Bitmap-Filter join: exact rationals, canonical
// CSR collections (load / write / generate), sketch analytics, option
// resolution and the per-join plan handed to the device engine.
//
// Namespace ssjb (never ssj) so the reference library can be loaded into the
// same process by the tests without ODR clashes.
#pragma once

#include <cstdint>
#include <limits>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

namespace ssjb {

// ---------------------------------------------------------------- errors --
// Mapped onto ssj_status by the C ABI exactly like reference src/capi.cpp:17-37.
struct ParseError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct IoError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct DeviceError : std::runtime_error {  // CUDA failures -> SSJ_ERROR_INTERNAL
    using std::runtime_error::runtime_error;
};

// -------------------------------------------------------------- rational --
// Reduced fraction with positive denominator (reference src/rational.hpp:14-43).
struct Rational {
    int64_t num = 0;
    int64_t den = 1;
    Rational() = default;
    Rational(int64_t n, int64_t d);
    double to_double() const { return static_cast<double>(num) / static_cast<double>(den); }
    friend bool operator<(const Rational& a, const Rational& b) {
        return static_cast<__int128>(a.num) * b.den < static_cast<__int128>(b.num) * a.den;
    }
    friend bool operator<=(const Rational& a, const Rational& b) { return !(b < a); }
    friend bool operator>=(const Rational& a, const Rational& b) { return !(a < b); }
};

// "p/q", integer, or decimal with <= 9 fractional digits (reference src/rational.cpp:23-41).
Rational parse_rational(const std::string& text);
// ceil(a/b) for a >= 0, b > 0 (reference src/rational.cpp:43-45).
inline int64_t ceil_div(__int128 a, __int128 b) { return static_cast<int64_t>((a + b - 1) / b); }

// ------------------------------------------------------------ similarity --
enum class Sim { Overlap = 0, Jaccard = 1, Cosine = 2, Dice = 3 };
enum class Method { Set = 0, Xor = 1, Next = 2, Combined = 3 };
enum class Algo { Naive = 0, AllPairs, PPJoin, PPJoinPlus, GroupJoin, AdaptJoin, ParBitmap };
enum class CutoffMode { Auto = 0, Off = 1, Explicit = 2 };

constexpr int64_t kUnlimited = std::numeric_limits<int64_t>::max();

// Threshold validation of reference src/similarity.cpp:18-27.
void validate_threshold(Sim f, const Rational& t);
// Jaccard-space threshold (reference src/join.cpp:37-50).
Rational jaccard_space(Sim f, const Rational& t);
// Combined -> concrete method (reference src/bitmap.cpp:30-36).
Method resolve_combined(Method m, const Rational& jaccard_t);

// ------------------------------------------------------------- analytics --
// Closed forms of reference src/bounds.cpp:13-35.
double expected_bound(Method m, int b, int64_t n);
// Reference src/bounds.cpp:96-107 (space_jaccard) / :109-114 (overlap).
int64_t cutoff(Method m, int b, const Rational& t, bool space_jaccard);
int64_t cutoff_for_overlap(Method m, int b, int64_t tau);
// Reference src/bounds.cpp:37-71.
double monte_carlo_bound(Method m, int b, int64_t n, int64_t trials, uint64_t seed);

// ------------------------------------------------------------ collection --
// Canonical collection in CSR form: record r owns tokens[offsets[r]..offsets[r+1]),
// strictly increasing; records sorted by (size, tokens); id == position
// (reference src/collection.hpp:25-40, src/collection.cpp:44-54).
struct DeviceReplica;  // engine-owned, per device

struct Collection {
    std::vector<uint32_t> tokens;
    std::vector<uint64_t> offsets{0};
    uint64_t universe = 0;   // token_frequency.size() of the reference
    uint32_t max_size = 0;
    std::vector<uint32_t> first_ge;  // first record index with size >= s, s in [0, max_size + 1]

    size_t size() const { return offsets.size() - 1; }
    uint32_t rec_size(size_t r) const { return static_cast<uint32_t>(offsets[r + 1] - offsets[r]); }
    int64_t median_size() const;  // lower median (reference src/collection.cpp:13-17)
    double mean_size() const;

    // Device-side state (resident replicas, host page registration), managed by the engine.
    mutable std::mutex dev_mu;
    mutable std::shared_ptr<DeviceReplica> pinned[16];
    mutable bool host_registered = false;
    // 16-bit copy of the tokens (universe <= 65536), page-locked: halves every upload
    mutable std::vector<uint16_t> tokens16;
    // Delta-coded copy for dense universes (<= 65536 and small gaps), page-locked:
    // record r occupies bytes [offsets[r] + r, offsets[r+1] + r + 1): its first
    // token as u16, then one byte per token holding the gap to the previous one
    // (1..254), 255 marking an exception whose absolute value is the next entry
    // of exc_val (record r's exceptions start at exc_start[r]).  ~1 byte per token.
    mutable std::vector<uint8_t> tokens8;
    mutable std::vector<uint32_t> exc_start;
    mutable std::vector<uint16_t> exc_val;
    mutable bool use_delta8 = false;
    // engine-owned host cache of the last join's work-item tiling (keyed by
    // the plan; repeated joins with the same options skip rebuilding it)
    mutable std::mutex plan_cache_mu;
    mutable std::shared_ptr<void> plan_cache;
    mutable std::shared_ptr<void> head_cache;
    ~Collection();
};

// Host threads used by ingest (env SSJB_HOST_THREADS, default: all cores).
unsigned host_threads();
// Canonicalises raw id records in place (per-record sort+dedup, record order).
void canonicalize(Collection& c, std::vector<uint32_t>&& raw_tokens,
                  const std::vector<uint64_t>& raw_offsets);
std::unique_ptr<Collection> collection_from_csr(const uint32_t* tokens, const uint64_t* offsets,
                                                size_t n);
// input_format: 0 ids, 1 words, 2 q-grams (reference src/capi.cpp:127-146).
std::unique_ptr<Collection> read_collection(const std::string& path, int input_format, int q);
void write_collection(const Collection& c, const std::string& path);

struct GeneratorConfig {
    int distribution = 0;  // 0 uniform, 1 zipf
    int64_t num_sets = 0;
    double mean_size = 0;
    int64_t universe = 0;
    uint64_t seed = 0;
    double zipf_exponent = 1.0;
};
// Bit-identical to reference src/collection.cpp:193-254 + build_collection :58-93.
std::unique_ptr<Collection> generate(const GeneratorConfig& cfg);

// --------------------------------------------------------------- options --
struct Options {
    Algo algorithm = Algo::AllPairs;
    Sim sim = Sim::Jaccard;
    Rational threshold{1, 2};
    bool bitmap_enabled = false;
    Method method = Method::Combined;
    int bits = 0;
    int hash = 0;  // 1 multiplicative
    CutoffMode cutoff_mode = CutoffMode::Auto;
    int64_t cutoff_value = 0;
    int workers = 1;
    int buffer_capacity = 2048;
    int placement = 0;     // 0 default (filter3), 1 filter2, 2 filter3 (reference src/join.hpp:13)
    int suffix_depth = 2;  // PPJoin+ partition rounds
    int ell_max = 3;       // AdaptJoin prefix extension cap
};

struct ResolvedBitmap {
    bool enabled = false;
    Method method = Method::Xor;
    int width = 64;
    int hash = 0;
    int64_t cutoff = kUnlimited;
};
// Reference src/join.cpp:52-89.
ResolvedBitmap resolve_bitmap(const Collection& c, const Options& o);

// ------------------------------------------------------------------ plan --
// Everything the device engine needs, precomputed exactly on the host with
// __int128 arithmetic so the kernels only do table lookups and integer compares.
struct JoinPlan {
    bool naive = false;          // NAIVE: window [0, i), no filter
    ResolvedBitmap bitmap;
    int64_t p = 1, q = 2;        // reduced Jaccard threshold
    uint32_t capacity = 2048;    // per-record buffer (counter semantics only)
    size_t row_begin = 0, row_end = 0;
    // minov[S] = max(1, ceil(p*S/(p+q))) for S = |r|+|s| in [0, 2*max_size]
    // (NAIVE with Dice / Overlap: that function's required overlap of S)
    std::vector<int32_t> minov;
    bool cosine = false;         // NAIVE with Cosine: required overlap computed per pair
    // j0 of a record of size s: first index whose size >= ceil(p*s/q)
    std::vector<uint32_t> window_start;
    uint64_t window_pairs = 0;   // sum over rows of (i - j0(i))
    int delivery = 0;            // 0 pairs to host, 1 count only, 2 sorted runs kept in HBM
};

// Required overlap of the similarity functions (reference src/similarity.cpp:93-115).
int64_t required_overlap(Sim f, const Rational& t, int64_t size_r, int64_t size_s);
// minov[S] for S in [0, smax] (Jaccard / Dice / Overlap; Cosine: all 1, unused).
std::vector<int32_t> minov_table(Sim f, const Rational& t, size_t smax);

// NAIVE RS-join (two collections) over R rows [r_begin, r_end) x all of S
// (reference src/join.cpp:110-121).
struct RsPlan {
    Sim sim = Sim::Jaccard;
    int64_t p = 1, q = 2;
    std::vector<int32_t> minov;  // minov[|r|+|s|]
    bool cosine = false;
    size_t r_begin = 0, r_end = 0;
    int delivery = 0;            // as JoinPlan::delivery
};
RsPlan make_rs_plan(const Collection& r, const Collection& s, const Options& o, size_t r_begin, size_t r_end);

// Prefix-filter bounds (reference src/similarity.cpp:117-166): the length
// window of a probe of size `size_r` (upper clamped to UINT32_MAX) and the
// prefix length at `ell`.
struct LengthWindow {
    int64_t lower = 0;
    int64_t upper = 0;
};
LengthWindow length_window(Sim f, const Rational& t, int64_t size_r);
int64_t prefix_length(Sim f, const Rational& t, int64_t size_r, int ell);

uint32_t window_start_of(const Collection& c, const JoinPlan& plan, size_t row);
JoinPlan make_plan(const Collection& c, const Options& o, size_t row_begin, size_t row_end);
// Row boundaries of `parts` shards of rows [row_begin, row_end) balancing the
// window pair count (+ head_weight x the pairs of the head-overlap region
// starting at record head_L0, when the join will run it).
std::vector<uint64_t> partition_rows(const Collection& c, const JoinPlan& plan, int parts, size_t row_begin = 0,
                                     size_t row_end = SIZE_MAX, uint32_t head_L0 = UINT32_MAX,
                                     double head_weight = 0.0);

}  // namespace ssjb
