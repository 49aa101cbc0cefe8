// C ABI of libssjoin.so: the reference's ssj_* surface (include/ssjoin.h)
// plus the ssjb_* extensions (include/ssjoin_b200.h).  Status codes, error
// texts and option validation follow reference src/capi.cpp; joins run on the
// GPU engine (engine.cu), split over several GPUs when configured.
#include <algorithm>
#include <charconv>
#include <chrono>
#include <condition_variable>
#include <deque>
#include <mutex>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
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
    o.placement = in.placement;
    o.suffix_depth = in.suffix_depth;
    o.ell_max = in.ell_max;
    o.workers = in.workers;
    o.buffer_capacity = in.buffer_capacity;
    return o;
}

// Algorithms of the drop-in.  PAR_BITMAP and NAIVE run as themselves (the
// PAR_BITMAP checks are reference src/parallel_join.cpp:41-44).  The
// prefix-filter algorithms (ALLPAIRS, PPJOIN, PPJOIN+, GROUPJOIN, ADAPTJOIN)
// run on the GPU prefix-filter engine (engine_prefix_join, prefix_join.cuh)
// with the reference's counters when a whole collection is joined (ssj_join,
// the delivery entry points).  Row-range entry points (ssjb_join_rows,
// ssjb_partition_rows) are PAR_BITMAP concepts: there a prefix-filter code is
// answered by the Bitmap-Filter join of the same threshold (Jaccard) or the
// NAIVE join (other functions) -- the same pair list, since every exact
// algorithm returns it (reference tests/test_joins.cpp:62-112).
bool is_prefix_algo(ssjb::Algo a) {
    return a == ssjb::Algo::AllPairs || a == ssjb::Algo::PPJoin || a == ssjb::Algo::PPJoinPlus ||
           a == ssjb::Algo::GroupJoin || a == ssjb::Algo::AdaptJoin;
}

void to_row_join(ssjb::Options& o) {
    if (!is_prefix_algo(o.algorithm)) return;
    if (o.sim == ssjb::Sim::Jaccard) {
        o.algorithm = ssjb::Algo::ParBitmap;
        o.bitmap_enabled = true;
    } else {
        o.algorithm = ssjb::Algo::Naive;
    }
    o.workers = std::max(o.workers, 1);
    if (o.buffer_capacity < 1) o.buffer_capacity = 2048;
}

void check_supported(ssjb::Options& o) {
    if (o.algorithm == ssjb::Algo::Naive || is_prefix_algo(o.algorithm)) return;
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

// ------------------------------------------------------- shard merge
// Row shards of a self-join own disjoint, ascending id_s ranges (rows i are
// id_s, reference src/parallel_join.cpp:61-136), and RS blocks own ascending
// id_r ranges.  So the canonical (id_r, id_s) order of the union is, id_r by
// id_r, shard 0's run, then shard 1's, ... -- no key comparisons beyond
// finding each run's end.  The id_r space is cut into T slices of about equal
// pair counts (a value binary search over the shards' lower bounds); each
// host thread writes its slice at the offset given by the shards' lower
// bounds: O(P) copying over all host threads, no growing intermediate.
using Seq = std::pair<const ssjb::PairOut*, size_t>;

size_t lower_id_r(const Seq& q, uint64_t v) {
    return static_cast<size_t>(std::lower_bound(q.first, q.first + q.second, v,
                                                [](const ssjb::PairOut& x, uint64_t j) { return x.id_r < j; }) -
                               q.first);
}

void merge_shards(const std::vector<Seq>& seqs, ssjb::PairOut* out) {
    size_t total = 0;
    uint64_t max_id = 0;
    for (const auto& q : seqs) {
        total += q.second;
        if (q.second) max_id = std::max<uint64_t>(max_id, q.first[q.second - 1].id_r);
    }
    if (!total) return;
    const unsigned T = static_cast<unsigned>(
        std::max<size_t>(1, std::min<size_t>(ssjb::host_threads(), total / (size_t(1) << 16))));
    // cut[t]: first id_r of slice t (slice t = id_r in [cut[t], cut[t+1]))
    std::vector<uint64_t> cut(T + 1);
    cut[0] = 0;
    cut[T] = max_id + 1;
    for (unsigned t = 1; t < T; ++t) {
        const size_t target = total * t / T;
        uint64_t lo = cut[t - 1], hi = max_id + 1;  // smallest v with count(id_r < v) >= target
        while (lo < hi) {
            const uint64_t mid = lo + (hi - lo) / 2;
            size_t c = 0;
            for (const auto& q : seqs) c += lower_id_r(q, mid);
            if (c >= target) hi = mid;
            else lo = mid + 1;
        }
        cut[t] = lo;
    }
    auto slice = [&](unsigned t) {
        const size_t G = seqs.size();
        std::vector<size_t> at(G), end(G);
        size_t dst = 0;
        for (size_t g = 0; g < G; ++g) {
            at[g] = lower_id_r(seqs[g], cut[t]);
            end[g] = lower_id_r(seqs[g], cut[t + 1]);
            dst += at[g];
        }
        ssjb::PairOut* o = out + dst;
        for (;;) {
            uint64_t r = UINT64_MAX;
            for (size_t g = 0; g < G; ++g)
                if (at[g] < end[g]) r = std::min<uint64_t>(r, seqs[g].first[at[g]].id_r);
            if (r == UINT64_MAX) break;
            for (size_t g = 0; g < G; ++g) {
                const ssjb::PairOut* p = seqs[g].first;
                size_t k = at[g];
                while (k < end[g] && p[k].id_r == r) ++k;
                if (k > at[g]) {
                    std::memcpy(o, p + at[g], (k - at[g]) * sizeof(ssjb::PairOut));
                    o += k - at[g];
                    at[g] = k;
                }
            }
        }
    };
    if (T == 1) {
        slice(0);
        return;
    }
    std::vector<std::thread> th;
    for (unsigned t = 1; t < T; ++t) th.emplace_back(slice, t);
    slice(0);
    for (auto& x : th) x.join();
}

// total_s < 0: the join's total is measured from t0 after the merge
void fill_report(ssj_report& rep, std::vector<ssjb::EngineResult>& parts, double total_s,
                 std::chrono::steady_clock::time_point t0 = {}) {
    if (parts.size() == 1) {
        rep.pairs = std::move(parts[0].pairs);
    } else {
        std::vector<Seq> seqs;
        size_t total = 0;
        for (auto& p : parts) {
            seqs.emplace_back(p.pairs.data(), p.pairs.size());
            total += p.pairs.size();
        }
        const auto m0 = std::chrono::steady_clock::now();
        ssjb::PairVec merged(total);
        merge_shards(seqs, merged.data());
        rep.pairs = std::move(merged);
        rep.stats.ms_merge = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - m0).count();
        for (auto& p : parts) p.pairs = ssjb::PairVec();
    }
    ssj_counters& c = rep.counters;
    std::memset(&c, 0, sizeof c);
    ssjb_stats& s = rep.stats;
    const double ms_merge = s.ms_merge;
    std::memset(&s, 0, sizeof s);
    s.ms_merge = ms_merge;
    for (auto& p : parts) {
        c.candidates += p.candidates;
        c.pruned_length += p.pruned_length;
        c.pruned_positional += p.pruned_positional;
        c.pruned_suffix += p.pruned_suffix;
        c.filter_evaluations += p.filter_evaluations;
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
        s.head_pairs += p.stats.head_pairs;
        s.head_survivors += p.stats.head_survivors;
        s.ms_head = std::max(s.ms_head, p.stats.ms_head);
        s.ms_head_setup = std::max(s.ms_head_setup, p.stats.ms_head_setup);
        s.head_k = std::max(s.head_k, p.stats.head_k);
    }
    s.devices = static_cast<int>(parts.size());
    if (total_s < 0) total_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    rep.timings.total_s = total_s;
    rep.timings.verify_s = std::max(0.0, total_s - rep.timings.index_s - rep.timings.candidates_s);
}

// Persistent host workers for per-device shard work.  The engine keeps
// per-(host thread, device) CUDA resources (streams, event pools, pinned
// staging), so shard work must run on long-lived threads: a batch of tasks
// takes idle workers (spawning more only when every worker is busy, i.e. up
// to the peak number of shards in flight) and the workers outlive the call.
class DeviceWorkers {
  public:
    static DeviceWorkers& get() {
        static DeviceWorkers* w = new DeviceWorkers();  // leaked: workers are detached
        return *w;
    }
    // Runs every task, returns when all have finished (exceptions rethrown, first first).
    void run_all(std::vector<std::function<void()>>& tasks) {
        const size_t n = tasks.size();
        std::vector<std::exception_ptr> errs(n);
        std::mutex dmu;
        std::condition_variable dcv;
        size_t left = n;
        {
            std::lock_guard<std::mutex> lk(mu_);
            for (size_t k = 0; k < n; ++k) {
                q_.push_back([&, k]() {
                    try {
                        tasks[k]();
                    } catch (...) {
                        errs[k] = std::current_exception();
                    }
                    std::lock_guard<std::mutex> l2(dmu);
                    if (--left == 0) dcv.notify_all();
                });
            }
            while (idle_ < q_.size()) {
                std::thread([this]() { loop(); }).detach();
                ++idle_;
            }
        }
        cv_.notify_all();
        std::unique_lock<std::mutex> lk(dmu);
        dcv.wait(lk, [&]() { return left == 0; });
        lk.unlock();
        for (auto& e : errs)
            if (e) std::rethrow_exception(e);
    }
    size_t threads() {
        std::lock_guard<std::mutex> lk(mu_);
        return spawned_;
    }

  private:
    void loop() {
        {
            std::lock_guard<std::mutex> lk(mu_);
            ++spawned_;
        }
        for (;;) {
            std::function<void()> f;
            {
                std::unique_lock<std::mutex> lk(mu_);
                cv_.wait(lk, [&]() { return !q_.empty(); });
                f = std::move(q_.front());
                q_.pop_front();
                --idle_;
            }
            f();
            std::lock_guard<std::mutex> lk(mu_);
            ++idle_;
        }
    }
    std::mutex mu_;
    std::condition_variable cv_;
    std::deque<std::function<void()>> q_;
    size_t idle_ = 0, spawned_ = 0;
};

int g_shards_per_device = 0;  // 0: env SSJB_SHARDS_PER_DEVICE, else 1

// Relative per-pair cost of the head-overlap region vs the filter's window
// pairs for row partitioning (C4: K2 ~0.34 ns / window pair, K3a ~2.7 ns / region pair).
double head_weight() {
    const char* v = std::getenv("SSJB_HEAD_WEIGHT");
    return v && *v ? std::atof(v) : 8.0;
}

int shards_per_device() {
    if (g_shards_per_device > 0) return g_shards_per_device;
    const char* v = std::getenv("SSJB_SHARDS_PER_DEVICE");
    return std::max(1, v && *v ? std::atoi(v) : 1);
}

// Runs rows [row_begin, row_end) split over `devices` GPUs (first_device..),
// shards_per_device() row shards per GPU (more than one only as a test hook:
// the multi-GPU partition and merge exercised on one device); the engines'
// results per shard, in row order (delivery: see JoinPlan::delivery).
std::vector<ssjb::EngineResult> run_self_parts(const ssjb::Collection& coll, const ssjb::Options& o, size_t row_begin,
                                               size_t row_end, int devices, int first_device, int delivery) {
    if (coll.size() >= (size_t(1) << 31)) throw std::invalid_argument("collections above 2^31 records are not supported");
    if (is_prefix_algo(o.algorithm)) {
        if (row_begin == 0 && row_end == coll.size()) {
            if (ssjb::engine_device_count() <= first_device)
                throw ssjb::DeviceError("no CUDA device available for the B200 join");
            std::vector<ssjb::EngineResult> parts(1);
            ssjb::engine_prefix_join(coll, o, first_device, parts[0]);
            return parts;
        }
        ssjb::Options ro = o;
        to_row_join(ro);
        return run_self_parts(coll, ro, row_begin, row_end, devices, first_device, delivery);
    }
    const auto h0 = std::chrono::steady_clock::now();
    ssjb::JoinPlan whole = ssjb::make_plan(coll, o, row_begin, row_end);
    whole.delivery = delivery;
    const auto h1 = std::chrono::steady_clock::now();
    const int avail = ssjb::engine_device_count();
    if (std::getenv("SSJB_HOST_TIMING") && std::atoi(std::getenv("SSJB_HOST_TIMING")) >= 2)
        std::fprintf(stderr, "[host] plan %.3f ms, device count %.3f ms\n",
                     std::chrono::duration<double, std::milli>(h1 - h0).count(),
                     std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - h1).count());
    if (avail <= 0) throw ssjb::DeviceError("no CUDA device available for the B200 join");
    devices = std::max(1, std::min(devices, avail - first_device));
    const int shards = devices * shards_per_device();
    std::vector<ssjb::EngineResult> parts(static_cast<size_t>(shards));
    if (shards == 1) {
        ssjb::engine_join(coll, whole, first_device, parts[0]);
    } else {
        // contiguous row blocks of the range balanced on the join's work
        const std::vector<uint64_t> bounds = ssjb::partition_rows(
            coll, whole, shards, row_begin, row_end, ssjb::engine_head_start(coll, whole), head_weight());
        std::vector<std::function<void()>> tasks;
        for (int g = 0; g < shards; ++g) {
            tasks.emplace_back([&, g]() {
                ssjb::JoinPlan p = ssjb::make_plan(coll, o, bounds[g], bounds[g + 1]);
                p.delivery = delivery;
                ssjb::engine_join(coll, p, first_device + g % devices, parts[static_cast<size_t>(g)]);
            });
        }
        DeviceWorkers::get().run_all(tasks);
    }
    return parts;
}

std::unique_ptr<ssj_report> run_gpu_join(const ssjb::Collection& coll, const ssjb::Options& o, size_t row_begin,
                                         size_t row_end, int devices, int first_device) {
    const auto t0 = std::chrono::steady_clock::now();
    auto parts = run_self_parts(coll, o, row_begin, row_end, devices, first_device, 0);
    auto rep = std::make_unique<ssj_report>();
    fill_report(*rep, parts, -1.0, t0);  // total_s includes the shard merge
    return rep;
}

// NAIVE RS-join (reference src/capi.cpp:225-232 -> src/join.cpp:110-121): R rows
// split into contiguous blocks over `devices` GPUs; each block's pairs are
// (R id, S id)-sorted and the blocks' id_r ranges ascend, so they concatenate.
std::vector<ssjb::EngineResult> run_rs_parts(const ssjb::Collection& r, const ssjb::Collection& sc,
                                             const ssjb::Options& o, int devices, int delivery) {
    if (r.size() >= (size_t(1) << 31) || sc.size() >= (size_t(1) << 31))
        throw std::invalid_argument("collections above 2^31 records are not supported");
    const int avail = ssjb::engine_device_count();
    if (avail <= 0) throw ssjb::DeviceError("no CUDA device available for the B200 join");
    devices = std::max(1, std::min(devices, avail));
    if (r.size() < static_cast<size_t>(devices) * 1024) devices = 1;
    std::vector<ssjb::EngineResult> parts(static_cast<size_t>(devices));
    std::vector<std::function<void()>> tasks;
    for (int g = 0; g < devices; ++g) {
        const size_t b = r.size() * static_cast<size_t>(g) / devices, e = r.size() * static_cast<size_t>(g + 1) / devices;
        tasks.emplace_back([&, g, b, e]() {
            ssjb::RsPlan p = ssjb::make_rs_plan(r, sc, o, b, e);
            p.delivery = delivery;
            ssjb::engine_join_rs(r, sc, p, g, parts[static_cast<size_t>(g)]);
        });
    }
    if (devices == 1) tasks[0]();
    else DeviceWorkers::get().run_all(tasks);
    return parts;
}

std::unique_ptr<ssj_report> run_gpu_join_rs(const ssjb::Collection& r, const ssjb::Collection& sc,
                                            const ssjb::Options& o, int devices) {
    const auto t0 = std::chrono::steady_clock::now();
    auto parts = run_rs_parts(r, sc, o, devices, 0);
    auto rep = std::make_unique<ssj_report>();
    fill_report(*rep, parts, -1.0, t0);  // blocks own ascending id_r ranges (merge = concatenation)
    const double total = rep->timings.total_s;
    rep->timings.index_s = rep->timings.candidates_s = 0;  // naive: all verify (src/join.cpp:124)
    rep->timings.verify_s = total;
    return rep;
}

// ------------------------------------------------------------ delivery
// Streams the engines' output in canonical (id_r, id_s) order to `sink`, in
// chunks of whole id_r ranges holding about chunk_pairs pairs (one id_r with
// more pairs is one chunk).  Each part contributes its small host run and its
// sorted device runs (plan.delivery 2); per chunk the device side extracts the
// id_r range (merged on the GPU), the host merges the parts' sequences.
using Sink = std::function<void(const ssjb::PairOut*, size_t)>;

void stream_parts(std::vector<ssjb::EngineResult>& parts, size_t n_ids, size_t chunk_pairs, const Sink& sink) {
    chunk_pairs = std::max<size_t>(chunk_pairs, 1);
    bool any_runs = false;
    for (auto& p : parts) any_runs |= p.runs != nullptr;
    if (!any_runs && parts.size() == 1) {  // one sorted host run: slice it
        const ssjb::PairVec& v = parts[0].pairs;
        for (size_t a = 0; a < v.size(); a += chunk_pairs) sink(v.data() + a, std::min(chunk_pairs, v.size() - a));
        return;
    }
    std::vector<uint64_t> hist(n_ids, 0);
    for (auto& p : parts) {
        for (const auto& x : p.pairs)
            if (x.id_r < n_ids) ++hist[x.id_r];
        if (p.runs) ssjb::runs_histogram(*p.runs, hist);
    }
    auto key_less = [](const ssjb::PairOut& x, const ssjb::PairOut& y) {
        return x.id_r != y.id_r ? x.id_r < y.id_r : x.id_s < y.id_s;
    };
    size_t ja = 0;
    while (ja < n_ids) {
        uint64_t tot = hist[ja];
        size_t jb = ja + 1;
        while (jb < n_ids && tot + hist[jb] <= chunk_pairs) tot += hist[jb++];
        if (tot == 0) {
            ja = jb;
            continue;
        }
        // per part: its host run and its device runs (merged on the GPU) share
        // id_s ranges, so they are merged by key; across parts (row shards /
        // RS blocks) the id ranges are disjoint and ordered: merge_shards
        std::vector<ssjb::PairVec> own;
        std::vector<Seq> seqs;
        for (auto& p : parts) {
            const ssjb::PairOut* lo = nullptr;
            size_t cnt = 0;
            if (!p.pairs.empty()) {
                const Seq all(p.pairs.data(), p.pairs.size());
                const size_t a = lower_id_r(all, ja), b = lower_id_r(all, jb);
                lo = p.pairs.data() + a;
                cnt = b - a;
            }
            ssjb::PairVec v;
            if (p.runs) ssjb::runs_extract(*p.runs, static_cast<uint32_t>(ja), static_cast<uint32_t>(jb), v);
            if (!v.empty() && cnt) {
                ssjb::PairVec m(v.size() + cnt);
                std::merge(lo, lo + cnt, v.begin(), v.end(), m.begin(), key_less);
                own.push_back(std::move(m));
            } else if (!v.empty()) {
                own.push_back(std::move(v));
            } else if (cnt) {
                seqs.emplace_back(lo, cnt);
                continue;
            } else {
                continue;
            }
            seqs.emplace_back(own.back().data(), own.back().size());
        }
        if (seqs.size() == 1) {
            sink(seqs[0].first, seqs[0].second);
        } else if (!seqs.empty()) {
            size_t cnt = 0;
            for (const auto& q : seqs) cnt += q.second;
            ssjb::PairVec m(cnt);
            merge_shards(seqs, m.data());
            sink(m.data(), m.size());
        }
        ja = jb;
    }
}

// Text pairs in the reference CLI's format, "id_r id_s overlap\n" per pair
// (tools/ssjoin_cli.cpp:290-294); chunks are formatted by several threads and
// written in order.
struct PairTextWriter {
    std::FILE* f = nullptr;
    std::string path;
    explicit PairTextWriter(const char* p) : path(p) {
        f = std::fopen(p, "wb");
        if (!f) throw ssjb::IoError("cannot open output file '" + path + "'");
    }
    ~PairTextWriter() {
        if (f) std::fclose(f);
    }
    void close() {
        if (f && std::fclose(f) != 0) {
            f = nullptr;
            throw ssjb::IoError("error writing '" + path + "'");
        }
        f = nullptr;
    }
    static size_t format(const ssjb::PairOut* p, size_t n, std::vector<char>& buf) {
        buf.resize(n * 42 + 1);
        char* o = buf.data();
        for (size_t k = 0; k < n; ++k) {
            o = std::to_chars(o, o + 10, p[k].id_r).ptr;
            *o++ = ' ';
            o = std::to_chars(o, o + 10, p[k].id_s).ptr;
            *o++ = ' ';
            o = std::to_chars(o, o + 20, p[k].overlap).ptr;
            *o++ = '\n';
        }
        return static_cast<size_t>(o - buf.data());
    }
    void write(const ssjb::PairOut* p, size_t n) {
        const size_t piece = size_t(1) << 16;
        const unsigned nt = static_cast<unsigned>(
            std::max<size_t>(1, std::min<size_t>((n + piece - 1) / piece, std::min(16u, std::thread::hardware_concurrency()))));
        std::vector<std::vector<char>> bufs(nt);
        std::vector<size_t> lens(nt, 0);
        const size_t per = (n + nt - 1) / nt;
        std::vector<std::thread> th;
        for (unsigned t = 0; t < nt; ++t) {
            const size_t a = std::min(n, t * per), b = std::min(n, a + per);
            if (t == 0) continue;
            th.emplace_back([&, t, a, b]() { lens[t] = format(p + a, b - a, bufs[t]); });
        }
        lens[0] = format(p, std::min(n, per), bufs[0]);
        for (auto& x : th) x.join();
        for (unsigned t = 0; t < nt; ++t)
            if (lens[t] && std::fwrite(bufs[t].data(), 1, lens[t], f) != lens[t])
                throw ssjb::IoError("error writing '" + path + "'");
    }
};

// The join of (r, s_or_null) with the given delivery; the report carries the
// counters (pairs only for delivery 0).
std::vector<ssjb::EngineResult> run_parts(const ssj_collection* r, const ssj_collection* s_or_null,
                                          const ssjb::Options& o, int delivery) {
    if (s_or_null != nullptr) return run_rs_parts(*r->c, *s_or_null->c, o, configured_devices(), delivery);
    return run_self_parts(*r->c, o, 0, r->c->size(), configured_devices(), 0, delivery);
}

ssj_status checked_options(const ssj_collection* r, const ssj_collection* s_or_null, const ssj_join_options* opts,
                           ssjb::Options& o) {
    if (r == nullptr || opts == nullptr) {
        set_error("null argument");
        return SSJ_ERROR_INVALID_ARGUMENT;
    }
    o = to_options(*opts);
    if (s_or_null != nullptr && o.algorithm != ssjb::Algo::Naive) {
        set_error("RS-joins are only supported by the naive algorithm");
        return SSJ_ERROR_INVALID_ARGUMENT;
    }
    check_supported(o);
    return SSJ_OK;
}

std::unique_ptr<ssj_report> report_of(std::vector<ssjb::EngineResult>& parts, double total_s, bool rs) {
    for (auto& p : parts) {
        p.pairs = ssjb::PairVec();
        p.runs.reset();
    }
    auto rep = std::make_unique<ssj_report>();
    fill_report(*rep, parts, total_s);
    if (rs) {
        rep->timings.index_s = rep->timings.candidates_s = 0;
        rep->timings.verify_s = total_s;
    }
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
        to_row_join(o);
        ssjb::JoinPlan plan = ssjb::make_plan(*coll->c, o, 0, coll->c->size());
        auto b = ssjb::partition_rows(*coll->c, plan, parts, 0, coll->c->size(),
                                      ssjb::engine_head_start(*coll->c, plan), head_weight());
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

SSJB_API ssj_status ssjb_set_shards_per_device(int count) {
    return guarded([&]() {
        if (count < 0) throw std::invalid_argument("shards per device must be >= 0");
        g_shards_per_device = count;
        return SSJ_OK;
    });
}

SSJB_API ssj_status ssjb_merge_row_shards(const ssj_pair* const* runs, const size_t* counts, int nruns,
                                          ssj_pair* out) {
    return guarded([&]() {
        if (nruns < 0 || (nruns > 0 && (runs == nullptr || counts == nullptr)) || out == nullptr) {
            set_error("null argument");
            return SSJ_ERROR_INVALID_ARGUMENT;
        }
        std::vector<Seq> seqs;
        for (int k = 0; k < nruns; ++k)
            if (counts[k]) seqs.emplace_back(reinterpret_cast<const ssjb::PairOut*>(runs[k]), counts[k]);
        merge_shards(seqs, reinterpret_cast<ssjb::PairOut*>(out));
        return SSJ_OK;
    });
}

SSJB_API ssj_status ssjb_trim(int device) {
    return guarded([&]() {
        ssjb::engine_trim(device);
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

SSJB_API ssj_status ssjb_time_build(const ssj_collection* coll, int method, int bits, int hash, int device, int reps,
                                    double* ms_per_launch) {
    return guarded([&]() {
        if (coll == nullptr || ms_per_launch == nullptr || reps < 1) {
            set_error("null argument or reps < 1");
            return SSJ_ERROR_INVALID_ARGUMENT;
        }
        ssjb::Method m = to_method(method);
        if (m == ssjb::Method::Combined) throw std::invalid_argument("combined method must be resolved before building");
        if (bits <= 0 || bits % 64 != 0) throw std::invalid_argument("bitmap width must be a positive multiple of 64");
        *ms_per_launch = ssjb::engine_time_build(*coll->c, m, bits, hash == SSJ_HASH_MULT ? 1 : 0,
                                                 device < 0 ? 0 : device, reps);
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

// ------------------------------------------------------------------ delivery
SSJB_API ssj_status ssjb_join_stream(const ssj_collection* r, const ssj_collection* s_or_null,
                                     const ssj_join_options* opts, size_t chunk_pairs, ssjb_pair_sink sink, void* user,
                                     ssj_report** out) {
    return guarded([&]() {
        ssjb::Options o;
        if (sink == nullptr) {
            set_error("null argument");
            return SSJ_ERROR_INVALID_ARGUMENT;
        }
        ssj_status st = checked_options(r, s_or_null, opts, o);
        if (st != SSJ_OK) return st;
        const auto t0 = std::chrono::steady_clock::now();
        auto parts = run_parts(r, s_or_null, o, 2);
        stream_parts(parts, r->c->size(), chunk_pairs ? chunk_pairs : (size_t(1) << 24),
                     [&](const ssjb::PairOut* p, size_t n) {
                         if (sink(reinterpret_cast<const ssj_pair*>(p), n, user) != 0)
                             throw ssjb::IoError("the pair sink stopped the delivery");
                     });
        const double total = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        auto rep = report_of(parts, total, s_or_null != nullptr);
        if (out) *out = rep.release();
        return SSJ_OK;
    });
}

SSJB_API ssj_status ssjb_join_count(const ssj_collection* r, const ssj_collection* s_or_null,
                                    const ssj_join_options* opts, ssj_report** out) {
    return guarded([&]() {
        ssjb::Options o;
        if (out == nullptr) {
            set_error("null argument");
            return SSJ_ERROR_INVALID_ARGUMENT;
        }
        ssj_status st = checked_options(r, s_or_null, opts, o);
        if (st != SSJ_OK) return st;
        const auto t0 = std::chrono::steady_clock::now();
        auto parts = run_parts(r, s_or_null, o, 1);
        const double total = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        *out = report_of(parts, total, s_or_null != nullptr).release();
        return SSJ_OK;
    });
}

SSJB_API ssj_status ssjb_join_write_pairs(const ssj_collection* r, const ssj_collection* s_or_null,
                                          const ssj_join_options* opts, const char* path, ssj_report** out) {
    return guarded([&]() {
        ssjb::Options o;
        if (path == nullptr) {
            set_error("null argument");
            return SSJ_ERROR_INVALID_ARGUMENT;
        }
        ssj_status st = checked_options(r, s_or_null, opts, o);
        if (st != SSJ_OK) return st;
        const auto t0 = std::chrono::steady_clock::now();
        PairTextWriter w(path);
        auto parts = run_parts(r, s_or_null, o, 2);
        stream_parts(parts, r->c->size(), size_t(1) << 24,
                     [&](const ssjb::PairOut* p, size_t n) { w.write(p, n); });
        w.close();
        const double total = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        auto rep = report_of(parts, total, s_or_null != nullptr);
        if (out) *out = rep.release();
        return SSJ_OK;
    });
}

SSJB_API ssj_status ssjb_report_write_pairs(const ssj_report* report, const char* path) {
    return guarded([&]() {
        if (report == nullptr || path == nullptr) {
            set_error("null argument");
            return SSJ_ERROR_INVALID_ARGUMENT;
        }
        PairTextWriter w(path);
        const size_t n = report->pairs.size();
        for (size_t a = 0; a < n; a += size_t(1) << 24)
            w.write(report->pairs.data() + a, std::min(size_t(1) << 24, n - a));
        w.close();
        return SSJ_OK;
    });
}
