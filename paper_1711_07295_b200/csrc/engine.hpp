// Device engine of the B200 Bitmap-Filter join (implemented in engine.cu).
//
// The host (capi.cpp / host_core.cpp) resolves options into a JoinPlan; the
// engine uploads the canonical CSR collection, runs the four sm_100a kernel
// stages (sketch build, windowed xor/popcount filter, exact verification,
// canonical ordering) over the plan's row range on one GPU and returns the
// sorted pairs plus reference-exact counters.
#pragma once

#include <cstdint>
#include <memory>
#include <utility>
#include <vector>

#include "host_core.hpp"

namespace ssjb {

struct PairOut {  // layout of ssj_pair (reference include/ssjoin.h:125-129)
    uint32_t id_r;
    uint32_t id_s;
    int64_t overlap;
};
static_assert(sizeof(PairOut) == 16, "ssj_pair layout");

// Large result blocks (>= 64 MB): a process-wide cache of page-locked host
// blocks (engine.cu).  A freed block is kept (pinned, pages already faulted
// in) up to SSJB_RESULT_CACHE_MB (default min(8 GB, RAM / 8)) and handed to the next large
// result, so repeated joins neither zero fresh pages nor stage their
// downloads: the device copies straight into the result.
void* result_block_alloc(size_t bytes);
void result_block_free(void* p);
bool result_block_pinned(const void* p, size_t bytes);  // p..p+bytes inside a pinned cached block
constexpr size_t kResultBlockMin = size_t(64) << 20;

// Allocator that leaves trivially-constructible elements uninitialised: result
// vectors of 1e8+ pairs are filled by device copies, not zeroed first.
template <class T>
struct DefaultInitAlloc : std::allocator<T> {
    template <class U>
    struct rebind {
        using other = DefaultInitAlloc<U>;
    };
    DefaultInitAlloc() = default;
    template <class U>
    DefaultInitAlloc(const DefaultInitAlloc<U>&) noexcept {}
    T* allocate(size_t n) {
        if (n * sizeof(T) >= kResultBlockMin) return static_cast<T*>(result_block_alloc(n * sizeof(T)));
        return std::allocator<T>::allocate(n);
    }
    void deallocate(T* p, size_t n) {
        if (n * sizeof(T) >= kResultBlockMin) return result_block_free(p);
        std::allocator<T>::deallocate(p, n);
    }
    template <class U>
    void construct(U* p) noexcept {
        ::new (static_cast<void*>(p)) U;
    }
    template <class U, class... A>
    void construct(U* p, A&&... a) {
        ::new (static_cast<void*>(p)) U(std::forward<A>(a)...);
    }
};
using PairVec = std::vector<PairOut, DefaultInitAlloc<PairOut>>;

struct EngineStats {
    uint64_t window_pairs = 0, survivors = 0, batches = 0, launches = 0;
    uint64_t h2d_bytes = 0, d2h_bytes = 0, verify_bytes = 0;
    double ms_upload = 0, ms_build = 0, ms_filter = 0, ms_rescan = 0, ms_verify = 0, ms_sort = 0,
           ms_download = 0;
    int filter_kernel = 0;
    // K3a head-overlap phase (dense joins): region window pairs, survivors, head tokens, device ms
    uint64_t head_pairs = 0, head_survivors = 0;
    int head_k = 0;
    double ms_head = 0, ms_head_setup = 0;
};

// Sorted result runs left in device memory (delivery mode 2): the streaming
// delivery extracts them id_r range by id_r range (engine.cu).
struct DeviceRuns;

struct EngineResult {
    PairVec pairs;  // sorted by (id_r, id_s)
    std::shared_ptr<DeviceRuns> runs;  // delivery 2: further sorted runs in HBM (null if none)
    uint64_t candidates = 0, bitmap_tested = 0, pruned_bitmap = 0, verified = 0, matched = 0;
    // prefix-filter joins only (engine_prefix_join)
    uint64_t pruned_length = 0, pruned_positional = 0, pruned_suffix = 0, filter_evaluations = 0;
    uint64_t saturated = 0;
    double index_s = 0, candidates_s = 0, verify_s = 0;
    EngineStats stats;
};

int engine_device_count();
// One shard (plan.row_begin..row_end) of a self-join on `device`.
void engine_join(const Collection& c, const JoinPlan& plan, int device, EngineResult& out);
// ALLPAIRS / PPJOIN / PPJOIN+ / GROUPJOIN / ADAPTJOIN self-join of the whole
// collection on `device` (reference src/join.cpp:132-420), reference counters.
void engine_prefix_join(const Collection& c, const Options& o, int device, EngineResult& out);
// NAIVE RS-join block (plan.r_begin..r_end of R) x S on `device`; pairs are
// (R id, S id), sorted.
void engine_join_rs(const Collection& r, const Collection& s, const RsPlan& plan, int device, EngineResult& out);
// Streaming delivery over device runs: per-id_r match counts added into
// hist[0..hist.size()), and the sorted pairs with id_r in [ja, jb) (all runs
// merged) appended to out.
void runs_histogram(const DeviceRuns& runs, std::vector<uint64_t>& hist);
void runs_extract(const DeviceRuns& runs, uint32_t ja, uint32_t jb, PairVec& out);
uint64_t runs_total(const DeviceRuns& runs);
// The sketch-build kernel alone; copies the store (n * width/64 words) to out_host.
void engine_build_bitmaps(const Collection& c, Method method, int width, int hash, int device,
                          uint64_t* out_host);
// Mean device time (ms) of the sketch-build kernel over `reps` launches, L2 flushed.
double engine_time_build(const Collection& c, Method method, int width, int hash, int device, int reps);
void engine_pin(const Collection& c, int device);
void engine_unpin(const Collection& c, int device);
void engine_release_host(const Collection& c);  // undo host page registration
void engine_trim(int device);                   // free idle join workspaces (-1: all devices)
// First record of the head-overlap region (K3a) the join of `plan` over the
// whole collection would use, or UINT32_MAX (for work-balanced row shards).
uint32_t engine_head_start(const Collection& c, const JoinPlan& plan);

}  // namespace ssjb
