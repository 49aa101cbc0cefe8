// C ABI of libssjoin.so: the reference's ssj_* surface (include/ssjoin.h)
// plus the ssjb_* extensions (include/ssjoin_b200.h).  Status codes, error
// texts and option validation follow reference src/capi.cpp; joins run on the
// GPU engine (engine.cu), split over several GPUs when configured.
#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "../../include/ssjoin.h"
#include "../../include/ssjoin_b200.h"
#include "engine.hpp"
#include "host_core.hpp"

#define SSJB_API extern "C" __attribute__((visibility("default")))

struct ssj_collection {
    std::unique_ptr<ssjb::Collection> c;
};

struct ssj_report {
    ssjb::PairVec pairs;  // same 16-byte layout as ssj_pair
    ssj_counters counters{};
    ssj_timings timings{};
    uint64_t saturated = 0;
    ssjb_stats stats{};
};

namespace {

thread_local std::string g_last_error;
void set_error(const std::string& m) { g_last_error = m; }

// Exception -> status mapping of reference src/capi.cpp:17-37.
template <typename Fn>
ssj_status guarded(Fn&& fn) {
    try {
        return fn();
    } catch (const ssjb::ParseError& e) {
        set_error(e.what());
        return SSJ_ERROR_PARSE;
    } catch (const ssjb::IoError& e) {
        set_error(e.what());
        return SSJ_ERROR_IO;
    } catch (const std::invalid_argument& e) {
        set_error(e.what());
        return SSJ_ERROR_INVALID_ARGUMENT;
    } catch (const std::exception& e) {
        set_error(e.what());
        return SSJ_ERROR_INTERNAL;
    } catch (...) {
        set_error("unknown failure");
        return SSJ_ERROR_INTERNAL;
    }
}

ssjb::Method to_method(int m) {
    switch (m) {
        case SSJ_BITMAP_SET: return ssjb::Method::Set;
        case SSJ_BITMAP_XOR: return ssjb::Method::Xor;
        case SSJ_BITMAP_NEXT: return ssjb::Method::Next;
        case SSJ_BITMAP_COMBINED: return ssjb::Method::Combined;
    }
    throw std::invalid_argument("unknown bitmap method code");
}

ssjb::Sim to_sim(int s) {
    if (s < SSJ_SIM_OVERLAP || s > SSJ_SIM_DICE) throw std::invalid_argument("unknown similarity function code");
    return static_cast<ssjb::Sim>(s);
}

ssjb::Algo to_algo(int a) {
    if (a < SSJ_ALGO_NAIVE || a > SSJ_ALGO_PAR_BITMAP) throw std::invalid_argument("unknown algorithm code");
    return static_cast<ssjb::Algo>(a);
}

const char* algo_name(ssjb::Algo a) {
    static const char* names[] = {"naive", "allpairs", "ppjoin", "ppjoin+", "groupjoin", "adaptjoin", "par-bitmap"};
    return names[static_cast<int>(a)];
}

// reference src/capi.cpp:82-110 (same validation, same messages)
ssjb::Options to_options(const ssj_join_options& in) {
    ssjb::Options o;
    o.algorithm = to_algo(in.algorithm);
    ssjb::Rational t(in.threshold_num, in.threshold_den);
    o.sim = to_sim(in.similarity);
    ssjb::validate_threshold(o.sim, t);
    o.threshold = t;
    o.bitmap_enabled = in.bitmap_enabled != 0;
    o.method = to_method(in.bitmap_method);
    o.bits = in.bitmap_bits;
    o.hash = in.bitmap_hash == SSJ_HASH_MULT ? 1 : 0;
    switch (in.cutoff_mode) {
        case SSJ_CUTOFF_AUTO: o.cutoff_mode = ssjb::CutoffMode::Auto; break;
        case SSJ_CUTOFF_OFF: o.cutoff_mode = ssjb::CutoffMode::Off; break;
        case SSJ_CUTOFF_EXPLICIT: o.cutoff_mode = ssjb::CutoffMode::Explicit; break;
        default: throw std::invalid_argument("unknown cutoff mode");
    }
    o.cutoff_value = in.cutoff_value;
    if (in.placement < SSJ_PLACEMENT_DEFAULT || in.placement > SSJ_PLACEMENT_FILTER3)
        throw std::invalid_argument("unknown placement");
    o.workers = in.workers;
    o.buffer_capacity = in.buffer_capacity;
    return o;
}

// Algorithms the GPU path runs; the reference's checks of
// src/parallel_join.cpp:41-44 for the data-parallel join.
void check_supported(const ssjb::Options& o) {
    if (o.algorithm == ssjb::Algo::Naive) return;
    if (o.algorithm != ssjb::Algo::ParBitmap)
        throw std::invalid_argument(std::string("algorithm ") + algo_name(o.algorithm) +
                                    " is not provided by the B200 build (PAR_BITMAP and NAIVE run on the GPU)");
    if (o.workers < 1) throw std::invalid_argument("workers must be >= 1");
    if (o.buffer_capacity < 1) throw std::invalid_argument("buffer capacity must be >= 1");
    if (o.sim != ssjb::Sim::Jaccard) throw std::invalid_argument("the data-parallel join takes a jaccard threshold");
}

int g_devices = 0;  // 0: not yet configured

int configured_devices() {
    if (g_devices > 0) return g_devices;
    const char* v = std::getenv("SSJ_GPUS");
    int d = v && *v ? std::atoi(v) : 1;
    return std::max(1, d);
}

void fill_report(ssj_report& rep, std::vector<ssjb::EngineResult>& parts, double total_s) {
    size_t total = 0;
    for (auto& p : parts) total += p.pairs.size();
    if (parts.size() == 1) {
        rep.pairs = std::move(parts[0].pairs);
    } else {
        // shards own disjoint id_s ranges; k-way merge by (id_r, id_s)
        ssjb::PairVec merged;
        merged.reserve(total);
        for (auto& p : parts) {
            ssjb::PairVec tmp;
            tmp.reserve(merged.size() + p.pairs.size());
            std::merge(merged.begin(), merged.end(), p.pairs.begin(), p.pairs.end(), std::back_inserter(tmp),
                       [](const ssjb::PairOut& x, const ssjb::PairOut& y) {
                           return x.id_r != y.id_r ? x.id_r < y.id_r : x.id_s < y.id_s;
                       });
            merged.swap(tmp);
        }
        rep.pairs = std::move(merged);
    }
    ssj_counters& c = rep.counters;
    std::memset(&c, 0, sizeof c);
    ssjb_stats& s = rep.stats;
    std::memset(&s, 0, sizeof s);
    for (auto& p : parts) {
        c.candidates += p.candidates;
        c.bitmap_tested += p.bitmap_tested;
        c.pruned_bitmap += p.pruned_bitmap;
        c.verified += p.verified;
        c.matched += p.matched;
        rep.saturated += p.saturated;
        rep.timings.index_s = std::max(rep.timings.index_s, p.index_s);
        rep.timings.candidates_s = std::max(rep.timings.candidates_s, p.candidates_s);
        s.window_pairs += p.stats.window_pairs;
        s.survivors += p.stats.survivors;
        s.batches += p.stats.batches;
        s.launches += p.stats.launches;
        s.h2d_bytes += p.stats.h2d_bytes;
        s.d2h_bytes += p.stats.d2h_bytes;
        s.verify_bytes += p.stats.verify_bytes;
        s.ms_upload = std::max(s.ms_upload, p.stats.ms_upload);
        s.ms_build = std::max(s.ms_build, p.stats.ms_build);
        s.ms_filter = std::max(s.ms_filter, p.stats.ms_filter);
        s.ms_rescan = std::max(s.ms_rescan, p.stats.ms_rescan);
        s.ms_verify = std::max(s.ms_verify, p.stats.ms_verify);
        s.ms_sort = std::max(s.ms_sort, p.stats.ms_sort);
        s.ms_download = std::max(s.ms_download, p.stats.ms_download);
        s.filter_kernel = p.stats.filter_kernel;
    }
    s.devices = static_cast<int>(parts.size());
    rep.timings.total_s = total_s;
    rep.timings.verify_s = std::max(0.0, total_s - rep.timings.index_s - rep.timings.candidates_s);
}

// Runs rows [row_begin, row_end) split over `devices` GPUs (first_device..).
std::unique_ptr<ssj_report> run_gpu_join(const ssjb::Collection& coll, const ssjb::Options& o, size_t row_begin,
                                         size_t row_end, int devices, int first_device) {
    const auto t0 = std::chrono::steady_clock::now();
    if (coll.size() >= (size_t(1) << 31)) throw std::invalid_argument("collections above 2^31 records are not supported");
    ssjb::JoinPlan whole = ssjb::make_plan(coll, o, row_begin, row_end);
    const int avail = ssjb::engine_device_count();
    if (avail <= 0) throw ssjb::DeviceError("no CUDA device available for the B200 join");
    devices = std::max(1, std::min(devices, avail - first_device));
    std::vector<ssjb::EngineResult> parts(static_cast<size_t>(devices));
    if (devices == 1) {
        ssjb::engine_join(coll, whole, first_device, parts[0]);
    } else {
        // balanced contiguous row blocks of the range (window-pair prefix sums)
        std::vector<uint64_t> bounds(static_cast<size_t>(devices) + 1);
        {
            std::vector<double> pre(row_end - row_begin + 1, 0.0);
            for (size_t i = row_begin; i < row_end; ++i) {
                uint32_t j0 = ssjb::window_start_of(coll, whole, i);
                pre[i - row_begin + 1] = pre[i - row_begin] + (j0 < i ? double(i - j0) : 0.0) + 1.0;
            }
            bounds[0] = row_begin;
            for (int g = 1; g < devices; ++g) {
                const double target = pre.back() * g / devices;
                uint64_t b = row_begin + (std::lower_bound(pre.begin(), pre.end(), target) - pre.begin());
                b = row_begin + ((b - row_begin) & ~uint64_t(127));  // 128-row tile boundaries
                bounds[g] = std::max(b, bounds[g - 1]);
            }
            bounds[devices] = row_end;
        }
        std::vector<std::thread> pool;
        std::vector<std::exception_ptr> errs(static_cast<size_t>(devices));
        for (int g = 0; g < devices; ++g) {
            pool.emplace_back([&, g]() {
                try {
                    ssjb::JoinPlan p = ssjb::make_plan(coll, o, bounds[g], bounds[g + 1]);
                    ssjb::engine_join(coll, p, first_device + g, parts[static_cast<size_t>(g)]);
                } catch (...) {
                    errs[static_cast<size_t>(g)] = std::current_exception();
                }
            });
        }
        for (auto& t : pool) t.join();
        for (auto& e : errs)
            if (e) std::rethrow_exception(e);
    }
    auto rep = std::make_unique<ssj_report>();
    const double total = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    fill_report(*rep, parts, total);
    return rep;
}

// NAIVE RS-join (reference src/capi.cpp:225-232 -> src/join.cpp:110-121): R rows
// split into contiguous blocks over `devices` GPUs; each block's pairs are
// (R id, S id)-sorted and the blocks' id_r ranges ascend, so they concatenate.
std::unique_ptr<ssj_report> run_gpu_join_rs(const ssjb::Collection& r, const ssjb::Collection& sc,
                                            const ssjb::Options& o, int devices) {
    const auto t0 = std::chrono::steady_clock::now();
    if (r.size() >= (size_t(1) << 31) || sc.size() >= (size_t(1) << 31))
        throw std::invalid_argument("collections above 2^31 records are not supported");
    const int avail = ssjb::engine_device_count();
    if (avail <= 0) throw ssjb::DeviceError("no CUDA device available for the B200 join");
    devices = std::max(1, std::min(devices, avail));
    if (r.size() < static_cast<size_t>(devices) * 1024) devices = 1;
    std::vector<ssjb::EngineResult> parts(static_cast<size_t>(devices));
    std::vector<std::thread> pool;
    std::vector<std::exception_ptr> errs(static_cast<size_t>(devices));
    for (int g = 0; g < devices; ++g) {
        const size_t b = r.size() * static_cast<size_t>(g) / devices, e = r.size() * static_cast<size_t>(g + 1) / devices;
        auto work = [&, g, b, e]() {
            try {
                ssjb::RsPlan p = ssjb::make_rs_plan(r, sc, o, b, e);
                ssjb::engine_join_rs(r, sc, p, g, parts[static_cast<size_t>(g)]);
            } catch (...) {
                errs[static_cast<size_t>(g)] = std::current_exception();
            }
        };
        if (devices == 1) work();
        else pool.emplace_back(work);
    }
    for (auto& t : pool) t.join();
    for (auto& e : errs)
        if (e) std::rethrow_exception(e);
    // blocks own ascending id_r ranges: concatenation is the canonical order
    ssjb::PairVec all;
    if (devices > 1) {
        size_t count = 0;
        for (auto& p : parts) count += p.pairs.size();
        all.resize(count);
        size_t at = 0;
        for (auto& p : parts) {
            if (!p.pairs.empty()) std::memcpy(all.data() + at, p.pairs.data(), p.pairs.size() * sizeof(ssjb::PairOut));
            at += p.pairs.size();
            p.pairs = ssjb::PairVec();
        }
    }
    auto rep = std::make_unique<ssj_report>();
    const double total = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    fill_report(*rep, parts, total);
    if (devices > 1) rep->pairs = std::move(all);
    rep->timings.index_s = rep->timings.candidates_s = 0;  // naive: all verify (src/join.cpp:124)
    rep->timings.verify_s = total;
    return rep;
}

}  // namespace

SSJB_API const char* ssj_last_error(void) { return g_last_error.c_str(); }

SSJB_API ssj_status ssj_collection_load(const char* path, int input_format, int qgram_size, ssj_collection** out) {
    return guarded([&]() {
        if (path == nullptr || out == nullptr) {
            set_error("null argument");
            return SSJ_ERROR_INVALID_ARGUMENT;
        }
        auto h = std::make_unique<ssj_collection>();
        h->c = ssjb::read_collection(path, input_format, qgram_size);
        *out = h.release();
        return SSJ_OK;
    });
}

SSJB_API ssj_status ssj_collection_write(const ssj_collection* coll, const char* path) {
    return guarded([&]() {
        if (coll == nullptr || path == nullptr) {
            set_error("null argument");
            return SSJ_ERROR_INVALID_ARGUMENT;
        }
        ssjb::write_collection(*coll->c, path);
        return SSJ_OK;
    });
}

SSJB_API void ssj_collection_free(ssj_collection* coll) {
    if (coll == nullptr) return;
    for (auto& p : coll->c->pinned) p.reset();
    ssjb::engine_release_host(*coll->c);
    delete coll;
}

SSJB_API size_t ssj_collection_size(const ssj_collection* coll) { return coll ? coll->c->size() : 0; }
SSJB_API int64_t ssj_collection_median_size(const ssj_collection* coll) { return coll ? coll->c->median_size() : 0; }
SSJB_API double ssj_collection_mean_size(const ssj_collection* coll) { return coll ? coll->c->mean_size() : 0.0; }
SSJB_API int64_t ssj_collection_max_size(const ssj_collection* coll) {
    if (coll == nullptr || coll->c->size() == 0) return 0;
    return coll->c->rec_size(coll->c->size() - 1);
}
SSJB_API int64_t ssj_collection_universe(const ssj_collection* coll) {
    return coll ? static_cast<int64_t>(coll->c->universe) : 0;
}

SSJB_API ssj_status ssj_collection_generate(const ssj_generator_config* config, ssj_collection** out) {
    return guarded([&]() {
        if (config == nullptr || out == nullptr) {
            set_error("null argument");
            return SSJ_ERROR_INVALID_ARGUMENT;
        }
        ssjb::GeneratorConfig g;
        g.distribution = config->distribution == SSJ_DIST_ZIPF ? 1 : 0;
        g.num_sets = config->num_sets;
        g.mean_size = config->mean_size;
        g.universe = config->universe;
        g.seed = config->seed;
        g.zipf_exponent = config->zipf_exponent > 0 ? config->zipf_exponent : 1.0;
        auto h = std::make_unique<ssj_collection>();
        h->c = ssjb::generate(g);
        *out = h.release();
        return SSJ_OK;
    });
}

SSJB_API void ssj_join_options_init(ssj_join_options* opts) {
    // reference src/capi.cpp:201-215
    if (opts == nullptr) return;
    std::memset(opts, 0, sizeof(*opts));
    opts->algorithm = SSJ_ALGO_ALLPAIRS;
    opts->similarity = SSJ_SIM_JACCARD;
    opts->threshold_num = 1;
    opts->threshold_den = 2;
    opts->bitmap_method = SSJ_BITMAP_COMBINED;
    opts->cutoff_mode = SSJ_CUTOFF_AUTO;
    opts->placement = SSJ_PLACEMENT_DEFAULT;
    opts->suffix_depth = 2;
    opts->ell_max = 3;
    opts->workers = 1;
    opts->buffer_capacity = 2048;
}

SSJB_API ssj_status ssj_join(const ssj_collection* r, const ssj_collection* s_or_null, const ssj_join_options* opts,
                             ssj_report** out) {
    return guarded([&]() {
        if (r == nullptr || opts == nullptr || out == nullptr) {
            set_error("null argument");
            return SSJ_ERROR_INVALID_ARGUMENT;
        }
        ssjb::Options o = to_options(*opts);
        if (s_or_null != nullptr && o.algorithm != ssjb::Algo::Naive) {
            set_error("RS-joins are only supported by the naive algorithm");
            return SSJ_ERROR_INVALID_ARGUMENT;
        }
        check_supported(o);
        if (s_or_null != nullptr) {
            *out = run_gpu_join_rs(*r->c, *s_or_null->c, o, configured_devices()).release();
            return SSJ_OK;
        }
        auto rep = run_gpu_join(*r->c, o, 0, r->c->size(), configured_devices(), 0);
        *out = rep.release();
        return SSJ_OK;
    });
}

SSJB_API ssj_status ssj_resolve_bitmap(const ssj_collection* coll, const ssj_join_options* opts, int* method,
                                       int* bits, int64_t* cutoff) {
    return guarded([&]() {
        if (coll == nullptr || opts == nullptr) {
            set_error("null argument");
            return SSJ_ERROR_INVALID_ARGUMENT;
        }
        ssjb::ResolvedBitmap rb = ssjb::resolve_bitmap(*coll->c, to_options(*opts));
        if (method) *method = static_cast<int>(rb.method);
        if (bits) *bits = rb.enabled ? rb.width : 0;
        if (cutoff) *cutoff = rb.enabled ? rb.cutoff : 0;
        return SSJ_OK;
    });
}

SSJB_API size_t ssj_report_pair_count(const ssj_report* report) { return report ? report->pairs.size() : 0; }
SSJB_API const ssj_pair* ssj_report_pairs(const ssj_report* report) {
    return report ? reinterpret_cast<const ssj_pair*>(report->pairs.data()) : nullptr;
}
SSJB_API void ssj_report_counters(const ssj_report* report, ssj_counters* out) {
    if (report == nullptr || out == nullptr) return;
    *out = report->counters;
}
SSJB_API void ssj_report_timings(const ssj_report* report, ssj_timings* out) {
    if (report == nullptr || out == nullptr) return;
    *out = report->timings;
}
SSJB_API uint64_t ssj_report_saturated_records(const ssj_report* report) { return report ? report->saturated : 0; }
SSJB_API void ssj_report_free(ssj_report* report) { delete report; }

SSJB_API ssj_status ssj_expected_bound(int method, int bits, int64_t n, double* out) {
    return guarded([&]() {
        if (out == nullptr) {
            set_error("null argument");
            return SSJ_ERROR_INVALID_ARGUMENT;
        }
        *out = ssjb::expected_bound(to_method(method), bits, n);
        return SSJ_OK;
    });
}

SSJB_API ssj_status ssj_monte_carlo_bound(int method, int bits, int64_t n, int64_t trials, uint64_t seed,
                                          double* out) {
    return guarded([&]() {
        if (out == nullptr) {
            set_error("null argument");
            return SSJ_ERROR_INVALID_ARGUMENT;
        }
        *out = ssjb::monte_carlo_bound(to_method(method), bits, n, trials, seed);
        return SSJ_OK;
    });
}

SSJB_API ssj_status ssj_cutoff(int method, int bits, int64_t threshold_num, int64_t threshold_den, int space,
                               int64_t* out) {
    return guarded([&]() {
        if (out == nullptr) {
            set_error("null argument");
            return SSJ_ERROR_INVALID_ARGUMENT;
        }
        *out = ssjb::cutoff(to_method(method), bits, ssjb::Rational(threshold_num, threshold_den),
                            space == SSJ_SPACE_JACCARD);
        return SSJ_OK;
    });
}

SSJB_API ssj_status ssj_parse_threshold(const char* text, int64_t* num, int64_t* den) {
    return guarded([&]() {
        if (text == nullptr || num == nullptr || den == nullptr) {
            set_error("null argument");
            return SSJ_ERROR_INVALID_ARGUMENT;
        }
        ssjb::Rational r = ssjb::parse_rational(text);
        *num = r.num;
        *den = r.den;
        return SSJ_OK;
    });
}

// ------------------------------------------------------------ extensions --
SSJB_API ssj_status ssjb_collection_from_csr(const uint32_t* tokens, const uint64_t* offsets, size_t n,
                                             ssj_collection** out) {
    return guarded([&]() {
        if (offsets == nullptr || out == nullptr || (tokens == nullptr && n && offsets[n] != offsets[0])) {
            set_error("null argument");
            return SSJ_ERROR_INVALID_ARGUMENT;
        }
        auto h = std::make_unique<ssj_collection>();
        h->c = ssjb::collection_from_csr(tokens, offsets, n);
        *out = h.release();
        return SSJ_OK;
    });
}

SSJB_API ssj_status ssjb_collection_csr(const ssj_collection* coll, const uint32_t** tokens, const uint64_t** offsets,
                                        size_t* n) {
    return guarded([&]() {
        if (coll == nullptr || tokens == nullptr || offsets == nullptr || n == nullptr) {
            set_error("null argument");
            return SSJ_ERROR_INVALID_ARGUMENT;
        }
        *tokens = coll->c->tokens.data();
        *offsets = coll->c->offsets.data();
        *n = coll->c->size();
        return SSJ_OK;
    });
}

SSJB_API ssj_status ssjb_collection_pin_device(const ssj_collection* coll, int device) {
    return guarded([&]() {
        if (coll == nullptr) {
            set_error("null argument");
            return SSJ_ERROR_INVALID_ARGUMENT;
        }
        ssjb::engine_pin(*coll->c, device < 0 ? 0 : device);
        return SSJ_OK;
    });
}

SSJB_API ssj_status ssjb_collection_unpin_device(const ssj_collection* coll, int device) {
    return guarded([&]() {
        if (coll == nullptr) {
            set_error("null argument");
            return SSJ_ERROR_INVALID_ARGUMENT;
        }
        ssjb::engine_unpin(*coll->c, device < 0 ? 0 : device);
        return SSJ_OK;
    });
}

SSJB_API ssj_status ssjb_join_rows(const ssj_collection* coll, const ssj_join_options* opts, size_t row_begin,
                                   size_t row_end, int device, ssj_report** out) {
    return guarded([&]() {
        if (coll == nullptr || opts == nullptr || out == nullptr) {
            set_error("null argument");
            return SSJ_ERROR_INVALID_ARGUMENT;
        }
        ssjb::Options o = to_options(*opts);
        check_supported(o);
        if (row_begin > row_end || row_end > coll->c->size())
            throw std::invalid_argument("row range outside the collection");
        auto rep = run_gpu_join(*coll->c, o, row_begin, row_end, 1, device < 0 ? 0 : device);
        *out = rep.release();
        return SSJ_OK;
    });
}

SSJB_API ssj_status ssjb_partition_rows(const ssj_collection* coll, const ssj_join_options* opts, int parts,
                                        uint64_t* bounds) {
    return guarded([&]() {
        if (coll == nullptr || opts == nullptr || bounds == nullptr) {
            set_error("null argument");
            return SSJ_ERROR_INVALID_ARGUMENT;
        }
        ssjb::Options o = to_options(*opts);
        check_supported(o);
        ssjb::JoinPlan plan = ssjb::make_plan(*coll->c, o, 0, coll->c->size());
        auto b = ssjb::partition_rows(*coll->c, plan, parts);
        std::copy(b.begin(), b.end(), bounds);
        return SSJ_OK;
    });
}

SSJB_API int ssjb_device_count(void) { return configured_devices(); }

SSJB_API ssj_status ssjb_set_devices(int count) {
    return guarded([&]() {
        if (count < 1) throw std::invalid_argument("device count must be >= 1");
        g_devices = count;
        return SSJ_OK;
    });
}

SSJB_API ssj_status ssjb_report_stats(const ssj_report* report, ssjb_stats* out) {
    return guarded([&]() {
        if (report == nullptr || out == nullptr) {
            set_error("null argument");
            return SSJ_ERROR_INVALID_ARGUMENT;
        }
        *out = report->stats;
        return SSJ_OK;
    });
}

SSJB_API ssj_status ssjb_build_bitmaps(const ssj_collection* coll, int method, int bits, int hash, int device,
                                       uint64_t* out_host) {
    return guarded([&]() {
        if (coll == nullptr || out_host == nullptr) {
            set_error("null argument");
            return SSJ_ERROR_INVALID_ARGUMENT;
        }
        ssjb::Method m = to_method(method);
        if (m == ssjb::Method::Combined) throw std::invalid_argument("combined method must be resolved before building");
        if (bits <= 0 || bits % 64 != 0) throw std::invalid_argument("bitmap width must be a positive multiple of 64");
        ssjb::engine_build_bitmaps(*coll->c, m, bits, hash == SSJ_HASH_MULT ? 1 : 0, device < 0 ? 0 : device, out_host);
        return SSJ_OK;
    });
}

SSJB_API const char* ssjb_version(void) { return "ssjoin-b200 0.1 (sm_100a)"; }
