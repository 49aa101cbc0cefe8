// Device engine: uploads the canonical CSR collection, runs K1-K4 on one GPU
// for one row shard of the self-join, and returns sorted pairs plus counters
// identical to the reference's SSJ_ALGO_PAR_BITMAP (src/parallel_join.cpp:40-140)
// or SSJ_ALGO_NAIVE (src/join.cpp:91-126).
#include <cuda_runtime.h>
#include <sys/mman.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <deque>
#include <condition_variable>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "engine.hpp"
#include "kernels.cuh"
#include "filter_tc.cuh"
#include "filter_tc2.cuh"
#include "filter_tcm.cuh"
#include "head_tc.cuh"
#include "prefix_join.cuh"

namespace ssjb {

namespace {

#define CK(expr)                                                                                   \
    do {                                                                                           \
        cudaError_t e_ = (expr);                                                                   \
        if (e_ != cudaSuccess)                                                                     \
            throw DeviceError(std::string("CUDA error: ") + cudaGetErrorString(e_) + " at " #expr); \
    } while (0)

constexpr uint32_t kPadRows = 256;  // sketch/size arrays are padded so TMA stages never read past the end

uint64_t env_u64(const char* name, uint64_t dflt) {
    const char* v = std::getenv(name);
    if (!v || !*v) return dflt;
    return std::strtoull(v, nullptr, 10);
}

void set_device(int device) {
    int count = 0;
    cudaError_t e = cudaGetDeviceCount(&count);
    if (e != cudaSuccess || count == 0)
        throw DeviceError(std::string("no CUDA device available for the B200 join (") +
                          (e == cudaSuccess ? "0 devices" : cudaGetErrorString(e)) + ")");
    if (device < 0 || device >= count)
        throw DeviceError("CUDA device " + std::to_string(device) + " out of range (" + std::to_string(count) +
                          " visible)");
    CK(cudaSetDevice(device));
    static std::once_flag pool_once[16];
    std::call_once(pool_once[device & 15], [device]() {
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
            uint64_t keep = UINT64_MAX;  // keep freed blocks cached for the next join
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
        }
    });
}

// Stream-ordered allocations freed when the scope ends.
struct Arena {
    cudaStream_t stream;
    std::vector<void*> blocks;
    explicit Arena(cudaStream_t s) : stream(s) {}
    template <typename T>
    T* alloc(size_t count) {
        void* p = nullptr;
        CK(cudaMallocAsync(&p, std::max<size_t>(count, 1) * sizeof(T), stream));
        blocks.push_back(p);
        return static_cast<T*>(p);
    }
    ~Arena() {
        for (void* p : blocks) cudaFreeAsync(p, stream);
        cudaStreamSynchronize(stream);
    }
};

// Small host tables of a join packed into one page-locked staging buffer and
// sent with a single copy (pageable cudaMemcpyAsync calls each cost a staged,
// synchronous transfer).  The buffer is per host thread; a join synchronises
// its stream before the next one reuses it.
struct TableStage {
    std::vector<std::pair<const void*, size_t>> parts;
    std::vector<void**> targets;
    size_t total = 0;
    template <typename T>
    void add(T** dev_ptr, const void* host, size_t bytes) {
        parts.push_back({host, bytes});
        targets.push_back(reinterpret_cast<void**>(dev_ptr));
        total += (bytes + 15) & ~size_t(15);
    }
    // one H2D of every part; sets the device pointers
    void flush(Arena& A, cudaStream_t s, uint64_t& h2d) {
        static thread_local uint8_t* host = nullptr;
        static thread_local size_t cap = 0;
        if (total == 0) return;
        if (total > cap) {
            if (host) cudaFreeHost(host);
            cap = std::max(total, size_t(1) << 20);
            CK(cudaHostAlloc(reinterpret_cast<void**>(&host), cap, cudaHostAllocPortable));
        }
        uint8_t* dev = A.alloc<uint8_t>(total);
        size_t off = 0;
        for (size_t k = 0; k < parts.size(); ++k) {
            if (parts[k].second) std::memcpy(host + off, parts[k].first, parts[k].second);
            *targets[k] = dev + off;
            off += (parts[k].second + 15) & ~size_t(15);
        }
        CK(cudaMemcpyAsync(dev, host, total, cudaMemcpyHostToDevice, s));
        h2d += total;
        parts.clear();
        targets.clear();
        total = 0;
    }
};

struct Timer {  // device-time spans on one stream; events recycled per host thread
    cudaStream_t stream;
    std::vector<cudaEvent_t> evs;
    int device = 0;
    static std::vector<cudaEvent_t>& pool(int dev) {
        static thread_local std::vector<cudaEvent_t> p[16];
        return p[dev & 15];
    }
    explicit Timer(cudaStream_t s) : stream(s) { cudaGetDevice(&device); }
    cudaEvent_t mark() {
        cudaEvent_t e;
        auto& p = pool(device);
        if (!p.empty()) {
            e = p.back();
            p.pop_back();
        } else {
            CK(cudaEventCreate(&e));
        }
        CK(cudaEventRecord(e, stream));
        evs.push_back(e);
        return e;
    }
    static double ms(cudaEvent_t a, cudaEvent_t b) {
        float f = 0;
        CK(cudaEventElapsedTime(&f, a, b));
        return f;
    }
    ~Timer() {
        auto& p = pool(device);  // per host thread and device
        for (auto e : evs) p.push_back(e);
    }
};

// Dynamic shared-memory opt-in, once per kernel and device.
void set_smem_once(const void* fn, int bytes) {
    static std::mutex mu;
    static std::vector<std::pair<std::pair<const void*, int>, int>> done;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(mu);
    for (auto& d : done)
        if (d.first.first == fn && d.first.second == dev && d.second >= bytes) return;
    CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    done.push_back({{fn, dev}, bytes});
}

bool narrow_tokens(const Collection& c) { return !c.tokens.empty() && c.universe <= 65536; }

// Builds the delta-coded token copy (see Collection::tokens8); true when it is
// worth using (at most 80% of the 16-bit copy's bytes).
bool build_delta8(const Collection& c) {
    const size_t n = c.size(), T = c.tokens.size();
    std::vector<uint8_t> bytes(T + n + 1);
    std::vector<uint32_t> start(n + 1, 0);
    std::vector<uint16_t> val;
    for (size_t r = 0; r < n; ++r) {
        start[r] = static_cast<uint32_t>(val.size());
        const uint64_t t0 = c.offsets[r], t1 = c.offsets[r + 1];
        uint8_t* b = bytes.data() + t0 + r;
        if (t0 == t1) {
            b[0] = 0;  // pad byte of an empty record
            continue;
        }
        uint32_t prev = c.tokens[t0];
        b[0] = static_cast<uint8_t>(prev & 0xFF);
        b[1] = static_cast<uint8_t>(prev >> 8);
        for (uint64_t t = t0 + 1; t < t1; ++t) {
            const uint32_t v = c.tokens[t], d = v - prev;
            if (d < 255) {
                b[t - t0 + 1] = static_cast<uint8_t>(d);
            } else {
                b[t - t0 + 1] = 255;
                val.push_back(static_cast<uint16_t>(v));
            }
            prev = v;
        }
    }
    start[n] = static_cast<uint32_t>(val.size());
    const double coded = double(bytes.size()) + 4.0 * double(start.size()) + 2.0 * double(val.size());
    if (coded > 0.8 * 2.0 * double(T)) return false;
    c.tokens8.swap(bytes);
    c.exc_start.swap(start);
    c.exc_val.swap(val);
    return true;
}

void register_host(const Collection& c) {
    // Page-lock the arrays that are uploaded so every upload is a pinned DMA
    // (portable: pinned for every device's context -- multi-GPU joins upload
    // the same collection to each device);
    // tokens of a universe <= 65536 travel as a delta-coded byte stream (dense
    // universes) or a 16-bit copy, built once here.
    if (c.host_registered) return;
    if (narrow_tokens(c) && c.universe <= 65535 && env_u64("SSJB_DELTA8", 1) != 0 && build_delta8(c)) {
        c.use_delta8 = true;
        cudaHostRegister(c.tokens8.data(), c.tokens8.size(), cudaHostRegisterPortable);
        cudaHostRegister(c.exc_start.data(), c.exc_start.size() * 4, cudaHostRegisterPortable);
        if (!c.exc_val.empty()) cudaHostRegister(c.exc_val.data(), c.exc_val.size() * 2, cudaHostRegisterPortable);
    } else if (narrow_tokens(c)) {
        c.tokens16.assign(c.tokens.begin(), c.tokens.end());
        cudaHostRegister(c.tokens16.data(), c.tokens16.size() * sizeof(uint16_t), cudaHostRegisterPortable);
    } else if (!c.tokens.empty()) {
        cudaHostRegister(const_cast<uint32_t*>(c.tokens.data()), c.tokens.size() * sizeof(uint32_t),
                         cudaHostRegisterPortable);
    }
    cudaHostRegister(const_cast<uint64_t*>(c.offsets.data()), c.offsets.size() * sizeof(uint64_t),
                     cudaHostRegisterPortable);
    cudaGetLastError();  // registration is an optimisation; ignore failures
    c.host_registered = true;
}

}  // namespace

// Sketch stores and expanded GEMM operands derived from a collection for one
// (method, width, hash).  Pinned replicas keep the last set, so a threshold
// sweep over a resident collection builds them once.
struct SketchSet {
    int device = -1;
    int method = -1, width = 0, hash = 0, words2 = 0;
    uint64_t* bits = nullptr;
    uint64_t* bits2 = nullptr;
    // expanded tcgen05 operand arrays (A, B) per variant: 0 int8, 1 int8 + level-2,
    // 2 fp4, 3 int8 without the size chunk (CTA-pair kernel), 4 int8 without the
    // popcount extension (+ per-column -pc pairs)
    uint8_t* opA[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};
    uint8_t* opB[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};
    uint32_t* npc2 = nullptr;
    bool owned = false;  // cudaMalloc'd (persistent) rather than arena memory
    ~SketchSet() {
        if (!owned) return;
        int cur = 0;
        cudaGetDevice(&cur);
        cudaSetDevice(device);
        cudaFree(bits);
        cudaFree(bits2);
        cudaFree(npc2);
        for (int v = 0; v < 5; ++v) {
            cudaFree(opA[v]);
            cudaFree(opB[v]);
        }
        cudaSetDevice(cur);
    }
};

// Device copy of a canonical collection: tokens, offsets and sizes (padded).
struct DeviceReplica {
    int device = -1;
    uint32_t* tokens = nullptr;
    uint64_t* offsets = nullptr;
    uint32_t* sizes = nullptr;
    size_t n = 0;
    uint64_t tokens_total = 0;
    uint64_t bytes = 0;
    const Collection* src = nullptr;  // host collection (sizes: first_ge) for launch shapes
    cudaStream_t stream = nullptr;  // set for per-join replicas: stream-ordered alloc/free
    std::shared_ptr<SketchSet> sketches;  // resident replicas only
    ~DeviceReplica() {
        if (device < 0) return;
        if (stream) {
            cudaFreeAsync(tokens, stream);
            cudaFreeAsync(offsets, stream);
            cudaFreeAsync(sizes, stream);
            return;
        }
        int cur = 0;
        cudaGetDevice(&cur);
        cudaSetDevice(device);
        cudaFree(tokens);
        cudaFree(offsets);
        cudaFree(sizes);
        cudaSetDevice(cur);
    }
};

namespace {

// |r| per record; the padding rows repeat the largest size so the array stays
// sorted (the filters test size-uniform column groups by their end points).
__global__ void sizes_from_offsets(const uint64_t* off, uint32_t* sizes, size_t n) {
    size_t r = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    if (r < n) sizes[r] = static_cast<uint32_t>(off[r + 1] - off[r]);
    else if (r < n + kPadRows + 8) sizes[r] = n ? static_cast<uint32_t>(off[n] - off[n - 1]) : 0u;
}

__global__ void widen_tokens(const uint16_t* in, uint32_t* out, size_t n) {
    size_t k = (blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x) * 4;
    if (k + 3 < n) {
        const ushort4 v = *reinterpret_cast<const ushort4*>(in + k);
        *reinterpret_cast<uint4*>(out + k) = make_uint4(v.x, v.y, v.z, v.w);
    } else {
        for (; k < n; ++k) out[k] = in[k];
    }
}

// Delta-coded tokens (Collection::tokens8) -> u32 tokens of records [r0, r1),
// one thread per record.
__global__ void decode_delta8(const uint8_t* bytes, const uint64_t* offsets, const uint32_t* exc_start,
                              const uint16_t* exc_val, uint32_t* out, uint32_t r0, uint32_t r1) {
    const uint32_t r = r0 + blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= r1) return;
    const uint64_t t0 = offsets[r], t1 = offsets[r + 1];
    if (t0 == t1) return;
    const uint8_t* b = bytes + t0 + r;
    uint32_t v = static_cast<uint32_t>(b[0]) | (static_cast<uint32_t>(b[1]) << 8);
    out[t0] = v;
    uint32_t e = exc_start[r];
    for (uint64_t t = t0 + 1; t < t1; ++t) {
        const uint32_t d = b[t - t0 + 1];
        if (d == 255) v = exc_val[e++];
        else v += d;
        out[t] = v;
    }
}

// Sub-warp variant: 2^lg lanes per record, each decoding a contiguous segment of
// the record's gap bytes.  A segment either adds its gaps to the value coming
// in, or (if it holds an exception) restarts from its last exception: a
// segmented scan over the lanes gives every segment its starting value, and an
// exclusive scan of exception counts its first exception index.
__global__ void decode_delta8_sub(const uint8_t* bytes, const uint64_t* offsets, const uint32_t* exc_start,
                                  const uint16_t* exc_val, uint32_t* out, uint32_t r0, uint32_t r1, int lg) {
    const int lpr = 1 << lg;
    const uint32_t gtid = blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t r = r0 + (gtid >> lg);
    const int sub = static_cast<int>(gtid & (lpr - 1));
    const bool live = r < r1;
    uint64_t t0 = 0, t1 = 0;
    if (live) {
        t0 = offsets[r];
        t1 = offsets[r + 1];
    }
    const uint32_t gaps = t1 > t0 ? static_cast<uint32_t>(t1 - t0 - 1) : 0u;  // gap bytes after the first token
    const uint32_t seg = (gaps + lpr - 1) >> lg;
    const uint32_t g0 = min(gaps, sub * seg), g1 = min(gaps, g0 + seg);
    const uint8_t* b = bytes + t0 + r + 2;  // gap k of the record at b[k]
    // pass 1: this segment's effect
    uint32_t sum = 0, nexc = 0;
    bool reset = false;
    for (uint32_t k = g0; k < g1; ++k) {
        const uint32_t d = b[k];
        if (d == 255) {
            ++nexc;
            reset = true;
            sum = 0;  // value restarts at the exception; the value itself is added below
        } else {
            sum += d;
        }
    }
    // exclusive scan of exception counts within the group
    uint32_t ex = nexc;
    for (int o = 1; o < lpr; o <<= 1) {
        const uint32_t v = __shfl_up_sync(0xFFFFFFFFu, ex, o, lpr);
        if (sub >= o) ex += v;
    }
    const uint32_t e_first = (live ? exc_start[r] : 0u) + ex - nexc;
    // segment transform: reset -> exc_val[last] + sum, else in + sum
    uint32_t val = sum + (reset ? exc_val[e_first + nexc - 1] : 0u);
    bool rs = reset;
    for (int o = 1; o < lpr; o <<= 1) {  // inclusive segmented scan
        const uint32_t pv = __shfl_up_sync(0xFFFFFFFFu, val, o, lpr);
        const bool pr = __shfl_up_sync(0xFFFFFFFFu, rs ? 1 : 0, o, lpr) != 0;
        if (sub >= o && !rs) {
            val += pv;
            rs = pr;
        }
    }
    // value entering this segment = inclusive result of the previous lane (+ first token)
    const uint32_t first = live && t1 > t0 ? (static_cast<uint32_t>(bytes[t0 + r]) |
                                              (static_cast<uint32_t>(bytes[t0 + r + 1]) << 8))
                                           : 0u;
    uint32_t prev_val = __shfl_up_sync(0xFFFFFFFFu, val, 1, lpr);
    const bool prev_rs = __shfl_up_sync(0xFFFFFFFFu, rs ? 1 : 0, 1, lpr) != 0;
    uint32_t v = sub == 0 ? first : (prev_rs ? prev_val : first + prev_val);
    if (!live || t1 == t0) return;
    if (sub == 0) out[t0] = first;
    uint32_t e = e_first;
    for (uint32_t k = g0; k < g1; ++k) {
        const uint32_t d = b[k];
        v = d == 255 ? exc_val[e++] : v + d;
        out[t0 + 1 + k] = v;
    }
}

struct Delta8Dev {
    uint8_t* bytes = nullptr;
    uint32_t* exc_start = nullptr;
    uint16_t* exc_val = nullptr;
};

// Device buffers for the delta-coded stream; the exception lists are uploaded here.
Delta8Dev alloc_delta8(const Collection& c, cudaStream_t stream, uint64_t& h2d) {
    Delta8Dev d;
    const size_t ne = c.exc_val.size();
    CK(cudaMallocAsync(reinterpret_cast<void**>(&d.bytes), c.tokens8.size() + 16, stream));
    CK(cudaMallocAsync(reinterpret_cast<void**>(&d.exc_start), c.exc_start.size() * 4, stream));
    CK(cudaMallocAsync(reinterpret_cast<void**>(&d.exc_val), std::max<size_t>(ne, 1) * 2, stream));
    CK(cudaMemcpyAsync(d.exc_start, c.exc_start.data(), c.exc_start.size() * 4, cudaMemcpyHostToDevice, stream));
    if (ne) CK(cudaMemcpyAsync(d.exc_val, c.exc_val.data(), ne * 2, cudaMemcpyHostToDevice, stream));
    h2d += c.exc_start.size() * 4 + ne * 2;
    return d;
}

void launch_decode(const Delta8Dev& d, const uint64_t* offsets, uint32_t* out, uint32_t r0, uint32_t r1,
                   cudaStream_t stream, uint64_t& launches, double mean_size = 0) {
    if (r1 <= r0) return;
    int lg = 0;  // about 6 gap bytes per lane
    while (lg < 5 && (1 << lg) * 6.0 < mean_size) ++lg;
    if (lg == 0) {
        decode_delta8<<<(r1 - r0 + 127) / 128, 128, 0, stream>>>(d.bytes, offsets, d.exc_start, d.exc_val, out, r0,
                                                                 r1);
    } else {
        const uint64_t threads = static_cast<uint64_t>(r1 - r0) << lg;
        decode_delta8_sub<<<static_cast<unsigned>((threads + 255) / 256), 256, 0, stream>>>(
            d.bytes, offsets, d.exc_start, d.exc_val, out, r0, r1, lg);
    }
    ++launches;
    CK(cudaGetLastError());
}

void free_delta8(Delta8Dev& d, cudaStream_t stream) {
    if (d.bytes) CK(cudaFreeAsync(d.bytes, stream));
    if (d.exc_start) CK(cudaFreeAsync(d.exc_start, stream));
    if (d.exc_val) CK(cudaFreeAsync(d.exc_val, stream));
    d = Delta8Dev{};
}

std::shared_ptr<DeviceReplica> upload(const Collection& c, int device, cudaStream_t stream, uint64_t& h2d,
                                      uint64_t& launches, bool resident = false) {
    register_host(c);
    auto rep = std::make_shared<DeviceReplica>();
    const size_t n = c.size();
    const size_t tok_bytes = std::max<size_t>(c.tokens.size(), 4) * sizeof(uint32_t) + 16;
    if (resident) {
        CK(cudaMalloc(&rep->tokens, tok_bytes));
        CK(cudaMalloc(&rep->offsets, (n + 1) * sizeof(uint64_t)));
        CK(cudaMalloc(&rep->sizes, (n + kPadRows + 8) * sizeof(uint32_t)));
    } else {
        rep->stream = stream;
        CK(cudaMallocAsync(reinterpret_cast<void**>(&rep->tokens), tok_bytes, stream));
        CK(cudaMallocAsync(reinterpret_cast<void**>(&rep->offsets), (n + 1) * sizeof(uint64_t), stream));
        CK(cudaMallocAsync(reinterpret_cast<void**>(&rep->sizes), (n + kPadRows + 8) * sizeof(uint32_t), stream));
    }
    rep->device = device;
    rep->n = n;
    rep->src = &c;
    rep->tokens_total = c.tokens.size();
    uint64_t tok_h2d = 0;
    CK(cudaMemcpyAsync(rep->offsets, c.offsets.data(), (n + 1) * sizeof(uint64_t), cudaMemcpyHostToDevice,
                       stream));
    if (c.use_delta8) {
        // ~1 byte per token, decoded on the device
        Delta8Dev d = alloc_delta8(c, stream, tok_h2d);
        CK(cudaMemcpyAsync(d.bytes, c.tokens8.data(), c.tokens8.size(), cudaMemcpyHostToDevice, stream));
        tok_h2d += c.tokens8.size();
        launch_decode(d, rep->offsets, rep->tokens, 0, static_cast<uint32_t>(n), stream, launches,
                      n ? static_cast<double>(c.tokens.size()) / static_cast<double>(n) : 0.0);
        free_delta8(d, stream);
    } else if (narrow_tokens(c)) {
        // 16-bit upload, widened on the device
        uint16_t* t16 = nullptr;
        const size_t T = c.tokens.size();
        CK(cudaMallocAsync(reinterpret_cast<void**>(&t16), T * sizeof(uint16_t), stream));
        CK(cudaMemcpyAsync(t16, c.tokens16.data(), T * sizeof(uint16_t), cudaMemcpyHostToDevice, stream));
        widen_tokens<<<static_cast<unsigned>((T + 1023) / 1024), 256, 0, stream>>>(t16, rep->tokens, T);
        ++launches;
        CK(cudaGetLastError());
        CK(cudaFreeAsync(t16, stream));
        tok_h2d = T * sizeof(uint16_t);
    } else if (!c.tokens.empty()) {
        CK(cudaMemcpyAsync(rep->tokens, c.tokens.data(), c.tokens.size() * sizeof(uint32_t),
                           cudaMemcpyHostToDevice, stream));
        tok_h2d = c.tokens.size() * sizeof(uint32_t);
    }
    rep->bytes = tok_h2d + (n + 1) * sizeof(uint64_t);
    h2d += rep->bytes;
    const size_t tot = n + kPadRows + 8;  // (n_pad = n + kPadRows rounded up to 8 rows)
    sizes_from_offsets<<<static_cast<unsigned>((tot + 255) / 256), 256, 0, stream>>>(rep->offsets, rep->sizes, n);
    ++launches;
    CK(cudaGetLastError());
    return rep;
}

std::shared_ptr<DeviceReplica> replica_for(const Collection& c, int device, cudaStream_t stream, uint64_t& h2d,
                                           uint64_t& launches) {
    {
        std::lock_guard<std::mutex> lk(c.dev_mu);
        if (c.pinned[device & 15] && c.pinned[device & 15]->device == device) return c.pinned[device & 15];
        register_host(c);
    }
    return upload(c, device, stream, h2d, launches);
}

// Streamed ingest for a per-join replica: offsets and sizes are uploaded on
// `stream` at once, the token array in row chunks (boundaries on multiples of
// `align_rows`, balanced by tokens) on the copy stream `cs`, one event per chunk.
// The join then builds sketches and filters chunk k while chunk k+1 is in
// flight: the window of row i only reaches columns j < i, so a chunk's work
// items never need rows of a later chunk.
struct IngestChunk {
    uint32_t r0 = 0, r1 = 0;
    uint64_t t0 = 0, t1 = 0;
    cudaEvent_t ev = nullptr;
};

std::shared_ptr<DeviceReplica> upload_streamed(const Collection& c, int device, cudaStream_t stream, cudaStream_t cs,
                                               uint32_t align_rows, int nchunks, uint64_t& h2d, uint64_t& launches,
                                               std::vector<IngestChunk>& chunks, uint16_t*& t16,
                                               Delta8Dev& d8) {
    {
        std::lock_guard<std::mutex> lk(c.dev_mu);
        register_host(c);
    }
    auto rep = std::make_shared<DeviceReplica>();
    const size_t n = c.size();
    const size_t T = c.tokens.size();
    const size_t tok_bytes = std::max<size_t>(T, 4) * sizeof(uint32_t) + 16;
    rep->stream = stream;
    rep->src = &c;
    CK(cudaMallocAsync(reinterpret_cast<void**>(&rep->tokens), tok_bytes, stream));
    CK(cudaMallocAsync(reinterpret_cast<void**>(&rep->offsets), (n + 1) * sizeof(uint64_t), stream));
    CK(cudaMallocAsync(reinterpret_cast<void**>(&rep->sizes), (n + kPadRows + 8) * sizeof(uint32_t), stream));
    const bool delta8 = c.use_delta8;
    const bool narrow = !delta8 && narrow_tokens(c);
    t16 = nullptr;
    uint64_t tok_h2d = 0;
    if (delta8) d8 = alloc_delta8(c, stream, tok_h2d);
    if (narrow) CK(cudaMallocAsync(reinterpret_cast<void**>(&t16), std::max<size_t>(T, 4) * 2 + 16, stream));
    rep->device = device;
    rep->n = n;
    rep->tokens_total = T;
    CK(cudaMemcpyAsync(rep->offsets, c.offsets.data(), (n + 1) * sizeof(uint64_t), cudaMemcpyHostToDevice, stream));
    sizes_from_offsets<<<static_cast<unsigned>((n + kPadRows + 8 + 255) / 256), 256, 0, stream>>>(rep->offsets,
                                                                                              rep->sizes, n);
    ++launches;
    CK(cudaGetLastError());
    cudaEvent_t ready;
    CK(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
    CK(cudaEventRecord(ready, stream));  // allocations done
    CK(cudaStreamWaitEvent(cs, ready, 0));
    CK(cudaEventDestroy(ready));
    chunks.clear();
    uint32_t r0 = 0;
    for (int k = 1; k <= nchunks && r0 < n; ++k) {
        uint32_t r1 = static_cast<uint32_t>(n);
        if (k < nchunks) {
            const uint64_t target = T * static_cast<uint64_t>(k) / nchunks;
            const size_t r = std::lower_bound(c.offsets.begin(), c.offsets.end(), target) - c.offsets.begin();
            r1 = static_cast<uint32_t>(std::min(n, (r + align_rows - 1) / align_rows * align_rows));
            if (r1 <= r0) continue;
        }
        IngestChunk ch;
        ch.r0 = r0;
        ch.r1 = r1;
        ch.t0 = c.offsets[r0];
        ch.t1 = c.offsets[r1];
        if (delta8) {
            const uint64_t b0 = ch.t0 + r0, b1 = (r1 < n ? ch.t1 + r1 : c.tokens8.size());
            if (b1 > b0)
                CK(cudaMemcpyAsync(d8.bytes + b0, c.tokens8.data() + b0, b1 - b0, cudaMemcpyHostToDevice, cs));
            tok_h2d += b1 - b0;
        } else if (ch.t1 > ch.t0) {
            tok_h2d += (ch.t1 - ch.t0) * (narrow ? 2 : 4);
            if (narrow)
                CK(cudaMemcpyAsync(t16 + ch.t0, c.tokens16.data() + ch.t0, (ch.t1 - ch.t0) * 2, cudaMemcpyHostToDevice,
                                   cs));
            else
                CK(cudaMemcpyAsync(rep->tokens + ch.t0, c.tokens.data() + ch.t0, (ch.t1 - ch.t0) * 4,
                                   cudaMemcpyHostToDevice, cs));
        }
        CK(cudaEventCreateWithFlags(&ch.ev, cudaEventDisableTiming));
        CK(cudaEventRecord(ch.ev, cs));
        chunks.push_back(ch);
        r0 = r1;
    }
    rep->bytes = tok_h2d + (n + 1) * sizeof(uint64_t);
    h2d += rep->bytes;
    return rep;
}

// ---------------------------------------------------------------- launchers
using FilterFn = void (*)(dev::FilterParams);
using BuildFn = void (*)(dev::BuildParams);

// Level-2 sketch words for a level-1 width (see filter_kernel): b <= 128 -> 256,
// b <= 256 -> 512, wider sketches filter well enough on their own.
int level2_words(int words) { return words <= 2 ? 4 : (words <= 4 ? 8 : 0); }

FilterFn filter_fn(int words, int words2) {
    if (words2 == 0) {
        switch (words) {
            case 1: return dev::filter_kernel<1, 0>;
            case 2: return dev::filter_kernel<2, 0>;
            case 3: return dev::filter_kernel<3, 0>;
            case 4: return dev::filter_kernel<4, 0>;
            case 5: return dev::filter_kernel<5, 0>;
            case 6: return dev::filter_kernel<6, 0>;
            case 7: return dev::filter_kernel<7, 0>;
            case 8: return dev::filter_kernel<8, 0>;
            default: return dev::filter_kernel<0, 0>;
        }
    }
    switch (words) {
        case 1: return dev::filter_kernel<1, 4>;
        case 2: return dev::filter_kernel<2, 4>;
        case 3: return dev::filter_kernel<3, 8>;
        case 4: return dev::filter_kernel<4, 8>;
    }
    throw DeviceError("no level-2 filter kernel for this width");
}

BuildFn build_fn(int words) {
    switch (words) {
        case 1: return dev::build_sketches<1>;
        case 2: return dev::build_sketches<2>;
        case 3: return dev::build_sketches<3>;
        case 4: return dev::build_sketches<4>;
        case 5: return dev::build_sketches<5>;
        case 6: return dev::build_sketches<6>;
        case 7: return dev::build_sketches<7>;
        case 8: return dev::build_sketches<8>;
        default: return dev::build_sketches<0>;
    }
}

int filter_colsub(int words) {
    if (words <= dev::kMaxInlineWords) return dev::kColSub;
    int c = (2048 / words) & ~31;
    return std::max(32, c);
}

size_t filter_smem(int words, int words2) {
    const size_t cs = static_cast<size_t>(filter_colsub(words));
    const size_t w2 = static_cast<size_t>(words2);
    return 2 * cs * (words + w2) * 8 + 2 * cs * 4 + 4 * dev::kWarpQueue * sizeof(uint2);
}

struct TcKernel {
    void (*fn)(dev::TcParams);
    int smem;
    int threads;
    int nt = 256;    // columns per MMA tile
    int parts = 4;   // epilogue column parts per tile (epilogue warps / 4)
};

template <int KIND, int KA, int K2, int W2, int NS, int NT>
TcKernel tc_kernel() {
    using L = dev::TcLayout<KIND, KA, K2, W2, NS, NT>;
    return TcKernel{dev::filter_tc_kernel<KIND, KA, K2, W2, NS, NT>, L::kBytes, L::kThreads, NT, L::kParts};
}

// Tensor-core filter instantiations: level-1 width b = 64*words.
//   fp4:  kind::mxf4, K = b + 64 e2m1 elements ((b+64)/2 bytes), 192-column tiles
//   i8:   kind::i8, K = b + 32 bytes, 256-column tiles; with the level-2
//         GEMM on 256-bit Xor sketches (l2gemm), 128-column tiles
TcKernel tc_select(int words, bool l2gemm, bool fp4, bool noext = false) {
    if (noext && !l2gemm && !fp4) {
        switch (words) {
            case 1: return tc_kernel<dev::kKindI8, 64, 0, 4, 6, 256>();
            case 2: return tc_kernel<dev::kKindI8, 128, 0, 4, 4, 256>();
        }
    }
    const char* nenv = std::getenv("SSJB_TC_N");  // tile width override (experiments)
    const int nt = nenv && *nenv ? std::atoi(nenv) : 0;
    if (l2gemm) {
        switch (words) {
            case 1: return tc_kernel<dev::kKindI8, 96, 288, 4, 3, 128>();
            case 2: return tc_kernel<dev::kKindI8, 160, 288, 4, 2, 128>();
        }
    } else if (fp4) {
        if (nt == 128) {
            switch (words) {
                case 1: return tc_kernel<dev::kKindF4, 64, 0, 4, 8, 128>();
                case 2: return tc_kernel<dev::kKindF4, 96, 0, 4, 12, 128>();
            }
        }
        switch (words) {
            case 1: return tc_kernel<dev::kKindF4, 64, 0, 4, 12, 192>();
            case 2: return tc_kernel<dev::kKindF4, 96, 0, 4, 8, 192>();
            case 3: return tc_kernel<dev::kKindF4, 128, 0, 8, 5, 192>();
            case 4: return tc_kernel<dev::kKindF4, 160, 0, 8, 4, 192>();
        }
    } else {
        if (nt == 128) {
            switch (words) {
                case 1: return tc_kernel<dev::kKindI8, 96, 0, 4, 8, 128>();
                case 2: return tc_kernel<dev::kKindI8, 160, 0, 4, 6, 128>();
            }
        }
        switch (words) {
            case 1: return tc_kernel<dev::kKindI8, 96, 0, 4, 4, 256>();
            case 2: return tc_kernel<dev::kKindI8, 160, 0, 4, 3, 256>();
            case 3: return tc_kernel<dev::kKindI8, 224, 0, 8, 2, 256>();
            case 4: return tc_kernel<dev::kKindI8, 288, 0, 8, 3, 128>();
        }
    }
    throw DeviceError("no tensor-core filter instantiation for this width");
}

// CTA-pair int8 filter (filter_tc2.cuh): level-1 width b = 64 * words <= 128.
template <int KA, int NS>
TcKernel tc2_kernel() {
    using L = dev::Tc2Layout<KA, NS>;
    return TcKernel{dev::filter_tc2_kernel<KA, NS>, L::kBytes, L::kThreads};
}

// Single-CTA int8 filter with two row tiles per staged column tile (filter_tcm.cuh).
template <int KA, int NS>
TcKernel tcm_kernel() {
    using L = dev::TcmLayout<KA, NS>;
    return TcKernel{dev::filter_tcm_kernel<KA, NS>, L::kBytes, L::kThreads, 256, 4};
}

TcKernel tcm_select(int words) {
    switch (words) {
        case 1: return tcm_kernel<96, 3>();
        case 2: return tcm_kernel<160, 2>();
    }
    throw DeviceError("no two-row-tile filter instantiation for this width");
}

TcKernel tc2_select(int words) {
    switch (words) {
        case 1: return tc2_kernel<96, 8>();
        case 2: return tc2_kernel<160, 6>();
    }
    throw DeviceError("no CTA-pair filter instantiation for this width");
}

size_t operand_bytes(int words, bool fp4) { return fp4 ? 32 * words + 32 : 64 * words + 32; }

// Operand row bytes of a variant: level 1 | level 2 (int8, 256-bit sketch) | 16-byte size chunk.
size_t operand_row(int words, int variant) {
    if (variant == 4) return 64 * words;
    return operand_bytes(words, variant == 2) + (variant == 1 ? 64 * 4 + 32 : 0) + (variant == 3 ? 0 : 16);
}

// Accumulator bias built into the int8 operands' extension bytes: with
// b <= 128, D = 2<b_i,b_j> - pc_j lies in [-b, b]; adding b (spread over the
// extension bytes, each still an int8) puts D + b in [0, 2b], so the epilogue
// can use borrow-free packed subtractions (masks16_nonneg).  Level 1 of
// variants 0 (level-1 GEMM) and 1 (level-1 + level-2 GEMM); level 2 of
// variant 1 (256-bit sketch: bias 256 over four bytes).
bool acc_bias_on() {
    static const bool on = env_u64("SSJB_BIAS", 1) != 0;
    return on;
}
int level1_acc_bias(int words, int variant) {
    return acc_bias_on() && (variant == 0 || variant == 1) && words <= 2 ? 64 * words : 0;
}
int level2_acc_bias(int words2, int variant) {
    return acc_bias_on() && variant == 1 && words2 == 4 ? 256 : 0;
}

void launch_expand(const uint64_t* bits, int words, const uint64_t* bits2, int words2, const uint32_t* sizes,
                   uint8_t* opA, uint8_t* opB, uint32_t rows, int variant, cudaStream_t s, uint64_t& launches,
                   uint32_t row0 = 0) {
    if (rows <= row0) return;
    dev::ExpandParams E{};
    E.row0 = row0;
    E.bits = bits;
    E.bits2 = bits2;
    E.sizes = sizes;
    E.opA = opA;
    E.opB = opB;
    E.rows = rows;
    E.words = words;
    E.words2 = variant == 1 ? words2 : 0;
    E.fp4 = variant == 2 ? 1 : 0;
    E.K1 = variant == 4 ? 64 * words : static_cast<int>(operand_bytes(words, variant == 2));
    E.K2 = variant == 1 ? 64 * words2 + 32 : 0;
    E.with_size = (variant == 3 || variant == 4) ? 0 : 1;
    E.acc_bias = level1_acc_bias(words, variant);
    E.acc_bias2 = level2_acc_bias(words2, variant);
    const int kct = (E.K1 + E.K2) / 16 + E.with_size;
    const uint64_t threads = static_cast<uint64_t>(rows - row0) * kct;
    dev::expand_operands<<<static_cast<unsigned>((threads + 255) / 256), 256, 0, s>>>(E);
    ++launches;
    CK(cudaGetLastError());
}

// Per-column data of the no-extension variant for rows [row0, rows).
void launch_column_info(const uint64_t* bits, int words, uint32_t row0, uint32_t rows, uint32_t* npc2,
                        cudaStream_t s, uint64_t& launches) {
    if (rows <= row0) return;
    const uint32_t pairs = (rows - row0 + 1) / 2;
    dev::column_info<<<(pairs + 255) / 256, 256, 0, s>>>(bits, words, row0, rows, npc2);
    ++launches;
    CK(cudaGetLastError());
}

void launch_build(const DeviceReplica& rep, uint64_t* bits, Method method, int width, int hash, cudaStream_t s,
                  uint64_t& launches) {
    if (rep.n == 0) return;
    dev::BuildParams P{};
    P.tokens = rep.tokens;
    P.offsets = rep.offsets;
    P.bits = bits;
    P.n = static_cast<uint32_t>(rep.n);
    P.width = static_cast<uint32_t>(width);
    P.words = width / 64;
    P.method = static_cast<int>(method);
    P.hash_mult = hash == 1 ? 1 : 0;
    P.pow2 = (width & (width - 1)) == 0;
    const unsigned grid = static_cast<unsigned>((rep.n + dev::kBuildRecs - 1) / dev::kBuildRecs);
    build_fn(P.words)<<<grid, dev::kBuildRecs, 0, s>>>(P);
    ++launches;
    CK(cudaGetLastError());
}

using BuildFn2 = void (*)(dev::BuildParams2);

// Set/Xor sketches (and the level-2 Xor sketch in the same token pass) with
// several lanes per record; null when the shape has no instantiation.
BuildFn2 build_sub_fn(int words, int words2, bool x, bool big = false) {
#define SSJB_SUB(W)                                      \
    case W:                                              \
        switch (words2) {                                \
            case 0: return big ? (x ? dev::build_sketches_big<W, 0, true> : dev::build_sketches_big<W, 0, false>) \
                               : (x ? dev::build_sketches_sub<W, 0, true> : dev::build_sketches_sub<W, 0, false>); \
            case 4: return big ? (x ? dev::build_sketches_big<W, 4, true> : dev::build_sketches_big<W, 4, false>) \
                               : (x ? dev::build_sketches_sub<W, 4, true> : dev::build_sketches_sub<W, 4, false>); \
            case 8: return big ? (x ? dev::build_sketches_big<W, 8, true> : dev::build_sketches_big<W, 8, false>) \
                               : (x ? dev::build_sketches_sub<W, 8, true> : dev::build_sketches_sub<W, 8, false>); \
        }                                                \
        break;
    switch (words) {
        SSJB_SUB(1)
        SSJB_SUB(2)
        SSJB_SUB(3)
        SSJB_SUB(4)
        SSJB_SUB(5)
        SSJB_SUB(6)
        SSJB_SUB(7)
        SSJB_SUB(8)
    }
#undef SSJB_SUB
    return nullptr;
}

// Level-1 Set/Xor sketch (+ level-2 Xor sketch when bits2) in one launch.
// Returns false when the method/width needs the one-thread-per-record kernel.
bool launch_build_sub(const DeviceReplica& rep, uint64_t* bits, uint64_t* bits2, Method method, int width,
                      int width2, int hash, cudaStream_t s, uint64_t& launches, uint32_t row0 = 0,
                      uint32_t row1 = UINT32_MAX) {
    if (method != Method::Set && method != Method::Xor) return false;
    BuildFn2 fn = build_sub_fn(width / 64, bits2 ? width2 / 64 : 0, method == Method::Xor);
    if (!fn) return false;
    row1 = std::min<uint32_t>(row1, static_cast<uint32_t>(rep.n));
    if (row1 <= row0) return true;
    dev::BuildParams2 P{};
    P.row0 = row0;
    P.tokens = rep.tokens;
    P.offsets = rep.offsets;
    P.bits = bits;
    P.bits2 = bits2;
    P.n = row1;
    P.width = static_cast<uint32_t>(width);
    P.width2 = static_cast<uint32_t>(width2);
    P.method = method == Method::Set ? 0 : 1;
    P.hash_mult = hash == 1 ? 1 : 0;
    P.pow2 = (width & (width - 1)) == 0;
    P.pow2_2 = (width2 & (width2 - 1)) == 0;
    // about four 16-byte chunks per lane: lanes per record = next power of two
    // of (mean/4 + 1)/4
    const double mean = static_cast<double>(rep.tokens_total) / static_cast<double>(rep.n);
    int lg = 0;
    while (lg < 5 && (1 << lg) * 4.0 < mean / 4.0 + 1.0) ++lg;
    P.lpr_log2 = lg;
    P.total_tokens = rep.tokens_total;
    // Size tiers (sizes ascend with the row, so each tier is a row range):
    // 2^k lanes for records of (8 << k, 16 << k] tokens -- about four 16-byte
    // chunks per lane, four loads in flight -- a warp up to 4096 tokens, one
    // CTA per record above.  Without sizes (no host collection) one launch
    // with lanes from the mean size.
    if (rep.src && !rep.src->first_ge.empty() && !env_u64("SSJB_BUILD_ONE_TIER", 0)) {
        auto first_above = [&](uint64_t z) {
            return z >= rep.src->max_size ? row1
                                          : std::max<uint32_t>(row0, std::min<uint32_t>(row1, rep.src->first_ge[z + 1]));
        };
        auto launch_tier = [&](uint32_t a, uint32_t b, int lgr) {
            if (b <= a) return;
            P.row0 = a;
            P.n = b;
            P.lpr_log2 = lgr;
            const uint64_t threads = static_cast<uint64_t>(b - a) << lgr;
            fn<<<static_cast<unsigned>((threads + 255) / 256), 256, 0, s>>>(P);
            ++launches;
            CK(cudaGetLastError());
        };
        uint32_t at = row0;
        for (int k = 0; k <= 5 && at < row1; ++k) {
            const uint32_t e = first_above(k < 5 ? (uint64_t(16) << k) : 4096);
            launch_tier(at, e, k);
            at = std::max(at, e);
        }
        if (at < row1) {
            P.row0 = at;
            P.n = row1;
            build_sub_fn(width / 64, bits2 ? width2 / 64 : 0, method == Method::Xor, true)<<<row1 - at, 256, 0, s>>>(P);
            ++launches;
            CK(cudaGetLastError());
        }
        return true;
    }
    const uint64_t threads = static_cast<uint64_t>(row1 - row0) << lg;
    fn<<<static_cast<unsigned>((threads + 255) / 256), 256, 0, s>>>(P);
    ++launches;
    CK(cudaGetLastError());
    return true;
}

// Sort keys/vals in place by key bits [0, 32+bits) skipping constant bytes;
// returns the buffer holding the result (a or b).
struct SortBufs {
    const unsigned long long* count;  // device-side element count (small-sort path)
    unsigned long long* count_store = nullptr;  // writable count slot (when count is not ctl->results)
    unsigned long long* ka;
    uint32_t* va;
    unsigned long long* kb;
    uint32_t* vb;
    uint32_t* hist;
    uint32_t* sums;
};

constexpr uint32_t kSmallSort = 4096;

// Sorted (j << 32 | i, overlap) results -> ssj_pair records (id_r, id_s, i64).
__global__ void pack_pairs(const unsigned long long* keys, const uint32_t* ov, PairOut* out, uint64_t count) {
    const uint64_t k = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    if (k >= count) return;
    const unsigned long long key = keys[k];
    out[k] = PairOut{static_cast<uint32_t>(key >> 32), static_cast<uint32_t>(key & 0xFFFFFFFFu),
                     static_cast<int64_t>(ov[k])};
}

// Device -> pageable host copy of a large buffer: double-buffered through
// pinned staging chunks, the host side copied out by several threads while the
// next chunk is in flight (a plain cudaMemcpy to pageable memory runs at a
// fraction of the link rate).
void d2h_staged(void* dst, const void* src, size_t bytes, cudaStream_t s) {
    constexpr size_t kChunk = size_t(64) << 20;
    if (bytes >= (size_t(16) << 20)) {
        // a fresh multi-GB result vector is first touched here: back it with
        // transparent huge pages so the copy-out does not take a page fault per 4 KB
        const uintptr_t a = (reinterpret_cast<uintptr_t>(dst) + (size_t(2) << 20) - 1) & ~((uintptr_t(2) << 20) - 1);
        const uintptr_t e = (reinterpret_cast<uintptr_t>(dst) + bytes) & ~((uintptr_t(2) << 20) - 1);
        if (e > a) madvise(reinterpret_cast<void*>(a), e - a, MADV_HUGEPAGE);
    }
    if (bytes <= kChunk) {
        if (bytes) CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        return;
    }
    static thread_local uint8_t* stage[2] = {nullptr, nullptr};
    static thread_local cudaEvent_t ev[2];
    if (!stage[0]) {
        for (int b = 0; b < 2; ++b) {
            CK(cudaHostAlloc(reinterpret_cast<void**>(&stage[b]), kChunk, cudaHostAllocPortable));
            CK(cudaEventCreateWithFlags(&ev[b], cudaEventDisableTiming));
        }
    }
    const size_t nchunks = (bytes + kChunk - 1) / kChunk;
    auto issue = [&](size_t k) {
        const size_t off = k * kChunk, len = std::min(kChunk, bytes - off);
        CK(cudaMemcpyAsync(stage[k & 1], static_cast<const uint8_t*>(src) + off, len, cudaMemcpyDeviceToHost, s));
        CK(cudaEventRecord(ev[k & 1], s));
    };
    static const unsigned max_threads = static_cast<unsigned>(env_u64("SSJB_D2H_THREADS", 32));  // host-memcpy bound: all cores
    const unsigned nthreads = std::max(1u, std::min(max_threads, std::thread::hardware_concurrency()));
    issue(0);
    for (size_t k = 0; k < nchunks; ++k) {
        if (k + 1 < nchunks) issue(k + 1);
        CK(cudaEventSynchronize(ev[k & 1]));
        const size_t off = k * kChunk, len = std::min(kChunk, bytes - off);
        const size_t piece = (len + nthreads - 1) / nthreads;
        const uint8_t* buf = stage[k & 1];  // (thread_local: resolve here, not in the workers)
        uint8_t* out = static_cast<uint8_t*>(dst) + off;
        std::vector<std::thread> th;
        for (unsigned t = 1; t < nthreads; ++t) {
            const size_t a = std::min(len, t * piece), b = std::min(len, a + piece);
            if (a < b) th.emplace_back([=]() { std::memcpy(out + a, buf + a, b - a); });
        }
        std::memcpy(out, buf, std::min(len, piece));
        for (auto& x : th) x.join();
    }
}

// ------------------------------------------------- result block cache
}  // namespace

namespace {
struct ResultBlockCache {
    std::mutex mu;
    std::map<void*, size_t> live;                 // block -> capacity
    std::multimap<size_t, void*> idle;            // capacity -> block
    std::map<void*, size_t> pinned;               // page-locked blocks (live or idle)
    std::map<void*, size_t> pinning;              // queued / being page-locked
    size_t idle_bytes = 0;
    // page-locking runs on a background thread: pinning a multi-GB block costs
    // ~0.1 s per GB and must not land inside the next join
    std::condition_variable cv;
    std::deque<std::pair<void*, size_t>> queue;
    bool worker = false;
};
ResultBlockCache& result_cache() {
    static ResultBlockCache* c = new ResultBlockCache();  // leaked: outlives static teardown
    return *c;
}
size_t result_cache_budget() {
    // SSJB_RESULT_CACHE_MB, default min(8 GB, 1/8 of physical memory)
    static const size_t b = [] {
        const uint64_t mb = env_u64("SSJB_RESULT_CACHE_MB", 0);
        if (mb) return static_cast<size_t>(mb) << 20;
        const long pages = sysconf(_SC_PHYS_PAGES), psz = sysconf(_SC_PAGE_SIZE);
        const size_t phys = pages > 0 && psz > 0 ? static_cast<size_t>(pages) * static_cast<size_t>(psz) : 0;
        return std::min<size_t>(size_t(8) << 30, phys / 8);
    }();
    return b;
}
}  // namespace

void* result_block_alloc(size_t bytes) {
    ResultBlockCache& C = result_cache();
    {
        std::lock_guard<std::mutex> lk(C.mu);
        auto it = C.idle.lower_bound(bytes);
        if (it != C.idle.end() && it->first <= 2 * bytes) {
            void* p = it->second;
            C.live[p] = it->first;
            C.idle_bytes -= it->first;
            C.idle.erase(it);
            return p;
        }
    }
    const size_t cap = (bytes + (size_t(2) << 20) - 1) & ~((size_t(2) << 20) - 1);
    void* p = std::aligned_alloc(size_t(2) << 20, cap);
    if (!p) throw std::bad_alloc();
    madvise(p, cap, MADV_HUGEPAGE);  // first touch in 2 MB pages
    std::lock_guard<std::mutex> lk(C.mu);
    C.live[p] = cap;
    return p;
}

void result_block_free(void* p) {
    if (!p) return;
    ResultBlockCache& C = result_cache();
    std::unique_lock<std::mutex> lk(C.mu);
    auto it = C.live.find(p);
    if (it == C.live.end()) return;
    const size_t cap = it->second;
    C.live.erase(it);
    if (C.idle_bytes + cap <= result_cache_budget()) {
        if (!C.pinned.count(p) && !C.pinning.count(p)) {
            // page-lock once (its pages are faulted in by now), in the background;
            // later results reuse it and the device copies into it directly
            C.pinning[p] = cap;
            C.queue.emplace_back(p, cap);
            if (!C.worker) {
                C.worker = true;
                std::thread([&C]() {
                    for (;;) {
                        std::pair<void*, size_t> job;
                        {
                            std::unique_lock<std::mutex> l2(C.mu);
                            C.cv.wait(l2, [&C]() { return !C.queue.empty(); });
                            job = C.queue.front();
                            C.queue.pop_front();
                        }
                        const bool ok = cudaHostRegister(job.first, job.second, cudaHostRegisterPortable) == cudaSuccess;
                        if (!ok) cudaGetLastError();
                        std::lock_guard<std::mutex> l2(C.mu);
                        C.pinning.erase(job.first);
                        if (ok) C.pinned[job.first] = job.second;
                    }
                }).detach();
            }
            C.cv.notify_one();
        }
        C.idle.emplace(cap, p);
        C.idle_bytes += cap;
        return;
    }
    // over budget: release it (after any page-locking in flight)
    while (C.pinning.count(p)) {
        lk.unlock();
        std::this_thread::sleep_for(std::chrono::milliseconds(1));
        lk.lock();
    }
    if (C.pinned.count(p)) {
        C.pinned.erase(p);
        lk.unlock();
        cudaHostUnregister(p);
    } else {
        lk.unlock();
    }
    std::free(p);
}

bool result_block_pinned(const void* p, size_t bytes) {
    ResultBlockCache& C = result_cache();
    std::lock_guard<std::mutex> lk(C.mu);
    auto it = C.pinned.upper_bound(const_cast<void*>(p));
    if (it == C.pinned.begin()) return false;
    --it;
    const uint8_t* b = static_cast<const uint8_t*>(it->first);
    return static_cast<const uint8_t*>(p) >= b && static_cast<const uint8_t*>(p) + bytes <= b + it->second;
}

namespace {

// Sorted (key, overlap) results straight to ssj_pair records in host memory:
// the keys (8 B) and overlaps (4 B) travel as they are -- 12 B per pair instead
// of the 16 B packed record -- through double-buffered pinned staging, and the
// host threads that copy each chunk out widen it into (id_r, id_s, i64) records.
void d2h_pairs_staged(PairOut* dst, const unsigned long long* keys, const uint32_t* ov, uint64_t n, cudaStream_t s,
                      PairOut* dev_scratch = nullptr) {
    if (dev_scratch && n && result_block_pinned(dst, n * sizeof(PairOut))) {
        // a cached, page-locked result block: pack on the device, one DMA into it
        pack_pairs<<<static_cast<unsigned>((n + 255) / 256), 256, 0, s>>>(keys, ov, dev_scratch, n);
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(dst, dev_scratch, n * sizeof(PairOut), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        return;
    }
    constexpr uint64_t kChunk = uint64_t(4) << 20;  // pairs per staging chunk (48 MB)
    if (n >= (uint64_t(1) << 20)) {
        // fresh multi-GB result vectors: transparent huge pages for the first touch
        const uintptr_t a = (reinterpret_cast<uintptr_t>(dst) + (size_t(2) << 20) - 1) & ~((uintptr_t(2) << 20) - 1);
        const uintptr_t e = (reinterpret_cast<uintptr_t>(dst) + n * sizeof(PairOut)) & ~((uintptr_t(2) << 20) - 1);
        if (e > a) madvise(reinterpret_cast<void*>(a), e - a, MADV_HUGEPAGE);
    }
    static thread_local uint8_t* stage[2] = {nullptr, nullptr};
    static thread_local cudaEvent_t ev[2];
    if (!stage[0]) {
        for (int b = 0; b < 2; ++b) {
            CK(cudaHostAlloc(reinterpret_cast<void**>(&stage[b]), kChunk * 12, cudaHostAllocPortable));
            CK(cudaEventCreateWithFlags(&ev[b], cudaEventDisableTiming));
        }
    }
    const uint64_t nchunks = (n + kChunk - 1) / kChunk;
    auto issue = [&](uint64_t k) {
        const uint64_t off = k * kChunk, len = std::min(kChunk, n - off);
        uint8_t* st = stage[k & 1];
        CK(cudaMemcpyAsync(st, keys + off, len * 8, cudaMemcpyDeviceToHost, s));
        CK(cudaMemcpyAsync(st + kChunk * 8, ov + off, len * 4, cudaMemcpyDeviceToHost, s));
        CK(cudaEventRecord(ev[k & 1], s));
    };
    static const unsigned max_threads = static_cast<unsigned>(env_u64("SSJB_D2H_THREADS", 32));
    const unsigned nthreads = std::max(1u, std::min(max_threads, std::thread::hardware_concurrency()));
    if (nchunks) issue(0);
    for (uint64_t k = 0; k < nchunks; ++k) {
        if (k + 1 < nchunks) issue(k + 1);
        CK(cudaEventSynchronize(ev[k & 1]));
        const uint64_t off = k * kChunk, len = std::min(kChunk, n - off);
        const unsigned long long* kk = reinterpret_cast<const unsigned long long*>(stage[k & 1]);
        const uint32_t* oo = reinterpret_cast<const uint32_t*>(stage[k & 1] + kChunk * 8);
        PairOut* out = dst + off;
        auto widen = [=](uint64_t a, uint64_t b) {
            for (uint64_t x = a; x < b; ++x)
                out[x] = PairOut{static_cast<uint32_t>(kk[x] >> 32), static_cast<uint32_t>(kk[x] & 0xFFFFFFFFu),
                                 static_cast<int64_t>(oo[x])};
        };
        const unsigned T = len >= (uint64_t(1) << 16) ? nthreads : 1u;
        const uint64_t piece = (len + T - 1) / T;
        std::vector<std::thread> th;
        for (unsigned t = 1; t < T; ++t) {
            const uint64_t a = std::min(len, t * piece), b = std::min(len, a + piece);
            if (a < b) th.emplace_back(widen, a, b);
        }
        widen(0, std::min(len, piece));
        for (auto& x : th) x.join();
    }
}

// Single-CTA bitonic sort of up to 4096 (key, value) pairs; the count comes
// from device memory so it runs in the same stream-ordered chain as the
// verifier (a larger count leaves the data for the radix path).
__global__ void small_sort(unsigned long long* keys, uint32_t* vals, const unsigned long long* count) {
    const unsigned long long cnt = *count;
    if (cnt <= 1 || cnt > kSmallSort) return;
    const uint32_t n = static_cast<uint32_t>(cnt);
    __shared__ unsigned long long k[kSmallSort];
    __shared__ uint32_t v[kSmallSort];
    uint32_t m = 1;
    while (m < n) m <<= 1;
    for (uint32_t t = threadIdx.x; t < m; t += blockDim.x) {
        k[t] = t < n ? keys[t] : ~0ull;
        v[t] = t < n ? vals[t] : 0u;
    }
    __syncthreads();
    for (uint32_t size = 2; size <= m; size <<= 1) {
        for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
            for (uint32_t t = threadIdx.x; t < m; t += blockDim.x) {
                uint32_t p = t ^ stride;
                if (p > t) {
                    bool up = (t & size) == 0;
                    if ((k[t] > k[p]) == up) {
                        unsigned long long tk = k[t];
                        k[t] = k[p];
                        k[p] = tk;
                        uint32_t tv = v[t];
                        v[t] = v[p];
                        v[p] = tv;
                    }
                }
            }
            __syncthreads();
        }
    }
    for (uint32_t t = threadIdx.x; t < n; t += blockDim.x) {
        keys[t] = k[t];
        vals[t] = v[t];
    }
}

// The fast path's single download: the counters block, then (when the
// matches fit kSmallSort) the sorted keys and overlaps, packed contiguously so
// one copy into a page-locked buffer returns everything the host needs.
struct SmallPack {
    dev::Control ctl;
    unsigned long long keys[kSmallSort];
    uint32_t ov[kSmallSort];
};

__global__ void small_sort_pack(const unsigned long long* keys, const uint32_t* vals, const dev::Control* ctl,
                                SmallPack* pack) {
    const unsigned long long cnt = ctl->results;
    if (threadIdx.x < sizeof(dev::Control) / 8)
        reinterpret_cast<unsigned long long*>(&pack->ctl)[threadIdx.x] =
            reinterpret_cast<const unsigned long long*>(ctl)[threadIdx.x];
    if (cnt == 0 || cnt > kSmallSort) return;
    const uint32_t n = static_cast<uint32_t>(cnt);
    __shared__ unsigned long long k[kSmallSort];
    __shared__ uint32_t v[kSmallSort];
    if (n <= 640) {  // (measured: rank sort wins below ~700 keys, bitonic above)
        // rank sort: keys are distinct (one per pair), so each key's rank is its
        // slot; one pass over the keys instead of log^2 n barrier stages
        const bool mine = threadIdx.x < n;
        const unsigned long long key = mine ? keys[threadIdx.x] : 0ull;
        if (mine) k[threadIdx.x] = key;
        __syncthreads();
        if (mine) {
            uint32_t rank = 0;
            const ulonglong2* k2 = reinterpret_cast<const ulonglong2*>(k);
            for (uint32_t t = 0; t < n / 2; ++t) {  // broadcast 16-byte reads
                const ulonglong2 q = k2[t];
                rank += (q.x < key) + (q.y < key);
            }
            if (n & 1) rank += k[n - 1] < key;
            pack->keys[rank] = key;
            pack->ov[rank] = vals[threadIdx.x];
        }
        return;
    }
    uint32_t m = 1;
    while (m < n) m <<= 1;
    for (uint32_t t = threadIdx.x; t < m; t += blockDim.x) {
        k[t] = t < n ? keys[t] : ~0ull;
        v[t] = t < n ? vals[t] : 0u;
    }
    __syncthreads();
    for (uint32_t size = 2; size <= m; size <<= 1) {
        for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
            for (uint32_t t = threadIdx.x; t < m; t += blockDim.x) {
                uint32_t p = t ^ stride;
                if (p > t) {
                    bool up = (t & size) == 0;
                    if ((k[t] > k[p]) == up) {
                        unsigned long long tk = k[t];
                        k[t] = k[p];
                        k[p] = tk;
                        uint32_t tv = v[t];
                        v[t] = v[p];
                        v[p] = tv;
                    }
                }
            }
            __syncthreads();
        }
    }
    for (uint32_t t = threadIdx.x; t < n; t += blockDim.x) {
        pack->keys[t] = k[t];
        pack->ov[t] = v[t];
    }
}

SmallPack* host_small_pack() {
    static thread_local SmallPack* p = nullptr;
    if (!p) CK(cudaHostAlloc(reinterpret_cast<void**>(&p), sizeof(SmallPack), cudaHostAllocPortable));
    return p;
}

bool sort_results(SortBufs& B, unsigned long long n, int idbits, cudaStream_t s, uint64_t& launches) {
    // returns true when the sorted data ended in (kb, vb)
    if (n <= 1) return false;
    if (n <= kSmallSort) {
        small_sort<<<1, 1024, 0, s>>>(B.ka, B.va, B.count);
        ++launches;
        CK(cudaGetLastError());
        return false;
    }
    const uint32_t ntiles = static_cast<uint32_t>((n + dev::kSortTile - 1) / dev::kSortTile);
    const uint32_t hlen = 256u * ntiles;
    const uint32_t nblk = (hlen + dev::kScanBlock - 1) / dev::kScanBlock;
    std::vector<int> shifts;
    for (int sh = 0; sh < idbits; sh += 8) shifts.push_back(sh);
    for (int sh = 0; sh < idbits; sh += 8) shifts.push_back(32 + sh);
    bool flip = false;
    for (int sh : shifts) {
        unsigned long long* kin = flip ? B.kb : B.ka;
        uint32_t* vin = flip ? B.vb : B.va;
        unsigned long long* kout = flip ? B.ka : B.kb;
        uint32_t* vout = flip ? B.va : B.vb;
        dev::radix_hist<<<ntiles, dev::kSortThreads, 0, s>>>(kin, n, sh, B.hist, ntiles);
        if (nblk == 1) {
            dev::scan_single<<<1, dev::kScanBlock, 0, s>>>(B.hist, hlen);
            launches += 1;
        } else {
            dev::scan_blocks<<<nblk, dev::kScanBlock, 0, s>>>(B.hist, hlen, B.sums);
            dev::scan_single<<<1, dev::kScanBlock, 0, s>>>(B.sums, nblk);
            dev::scan_add<<<nblk, dev::kScanBlock, 0, s>>>(B.hist, hlen, B.sums);
            launches += 3;
        }
        dev::radix_scatter<<<ntiles, dev::kSortThreads, 0, s>>>(kin, vin, kout, vout, n, sh, B.hist, ntiles);
        launches += 2;
        CK(cudaGetLastError());
        flip = !flip;
    }
    return flip;
}

struct Tiling {
    uint32_t tile_rows = dev::kRowTile;  // rows per work item
    uint32_t ntiles = 0;
    std::vector<uint64_t> item_base;  // ntiles + 1
    std::vector<uint32_t> col_lo;     // ntiles
    std::vector<uint32_t> item_tile;  // tile of each work item
    std::vector<uint32_t> order;      // claim order -> item id (column-chunk-major), empty: identity
};

Tiling make_tiling(const Collection& c, const JoinPlan& plan, uint32_t tile_rows, bool ordered = false,
                   uint32_t split_tile = 0) {
    Tiling t;
    t.tile_rows = tile_rows;
    const size_t rows = plan.row_end - plan.row_begin;
    t.ntiles = static_cast<uint32_t>((rows + tile_rows - 1) / tile_rows);
    t.item_base.assign(t.ntiles + 1, 0);
    t.col_lo.assign(t.ntiles, 0);
    for (uint32_t k = 0; k < t.ntiles; ++k) {
        const size_t r0 = plan.row_begin + static_cast<size_t>(k) * tile_rows;
        const size_t rl = std::min<size_t>(r0 + tile_rows, plan.row_end) - 1;  // last row
        const uint32_t j0 = window_start_of(c, plan, r0);                   // smallest j0 of the tile
        const uint32_t lo = j0 & ~31u;
        t.col_lo[k] = lo;
        uint64_t items = 0;
        if (rl > lo && j0 < rl) items = (rl - lo + dev::kColChunk - 1) / dev::kColChunk;
        t.item_base[k + 1] = t.item_base[k] + items;
    }
    t.item_tile.resize(t.item_base.back());
    for (uint32_t k = 0; k < t.ntiles; ++k)
        std::fill(t.item_tile.begin() + static_cast<ptrdiff_t>(t.item_base[k]),
                  t.item_tile.begin() + static_cast<ptrdiff_t>(t.item_base[k + 1]), k);
    if (ordered && !t.item_tile.empty()) {
        // claim order: items by the 4096-column bucket of their first column
        // (counting sort, stable in tile order), so the CTAs working at once
        // stream the same column operands from L2
        // (split_tile > 0: the items of tiles [0, split_tile) come first, each
        // group column-chunk-major -- a streamed join filters them while the
        // rest of the collection is still in flight)
        const size_t nb1 = c.size() / dev::kColChunk + 2;
        const size_t nb = split_tile ? 2 * nb1 : nb1;
        std::vector<uint64_t> at(nb + 1, 0);
        auto bucket = [&](uint32_t k, uint64_t item) {
            const size_t b = std::min<size_t>(nb1 - 1, (t.col_lo[k] + (item - t.item_base[k]) * dev::kColChunk) /
                                                           dev::kColChunk);
            return split_tile && k >= split_tile ? nb1 + b : b;
        };
        for (uint32_t k = 0; k < t.ntiles; ++k)
            for (uint64_t it = t.item_base[k]; it < t.item_base[k + 1]; ++it) ++at[bucket(k, it) + 1];
        for (size_t b = 0; b < nb; ++b) at[b + 1] += at[b];
        t.order.resize(t.item_tile.size());
        for (uint32_t k = 0; k < t.ntiles; ++k)
            for (uint64_t it = t.item_base[k]; it < t.item_base[k + 1]; ++it)
                t.order[at[bucket(k, it)]++] = static_cast<uint32_t>(it);
    }
    return t;
}

// The tiling of the collection's last join with the same rows, window and
// tile shape (host cache on the Collection: repeated joins skip rebuilding
// and re-ordering millions of work items).
struct TilingCacheEntry {
    size_t row_begin = 0, row_end = 0;
    int64_t p = 0, q = 0;
    uint32_t tile_rows = 0, split_tile = 0;
    bool ordered = false;
    Tiling tl;
};

std::shared_ptr<const Tiling> cached_tiling(const Collection& c, const JoinPlan& plan, uint32_t tile_rows,
                                            bool ordered, uint32_t split_tile = 0) {
    {
        std::lock_guard<std::mutex> lk(c.plan_cache_mu);
        auto e = std::static_pointer_cast<TilingCacheEntry>(c.plan_cache);
        if (e && e->row_begin == plan.row_begin && e->row_end == plan.row_end && e->p == plan.p && e->q == plan.q &&
            e->tile_rows == tile_rows && e->split_tile == split_tile && e->ordered == ordered && !plan.naive)
            return std::shared_ptr<const Tiling>(e, &e->tl);
    }
    auto e = std::make_shared<TilingCacheEntry>();
    e->tl = make_tiling(c, plan, tile_rows, ordered, split_tile);
    if (plan.naive) return std::shared_ptr<const Tiling>(e, &e->tl);
    e->row_begin = plan.row_begin;
    e->row_end = plan.row_end;
    e->p = plan.p;
    e->q = plan.q;
    e->tile_rows = tile_rows;
    e->split_tile = split_tile;
    e->ordered = ordered;
    std::lock_guard<std::mutex> lk(c.plan_cache_mu);
    c.plan_cache = e;
    return std::shared_ptr<const Tiling>(e, &e->tl);
}

// Zeroes the per-(item, row) survivor counts of the items at claim positions
// [k0, k1) of a column-chunk-major order (the items a batch has not processed).
__global__ void zero_item_counts(const uint32_t* order, uint64_t k0, uint64_t k1, uint32_t* counts,
                                 uint32_t tile_rows) {
    const uint64_t total = (k1 - k0) * tile_rows;
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    for (uint64_t x = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; x < total; x += stride)
        counts[static_cast<uint64_t>(order[k0 + x / tile_rows]) * tile_rows + x % tile_rows] = 0;
}

// ------------------------------------------------------------ K3a head plan
// Region and work items of the head-overlap kernel (head_tc.cuh) for one
// shard, computed on the host.  Eligible joins: Xor/Set sketches with the
// 256-bit level-2 check (b <= 128), a minov table (not Cosine), records
// below 2^16 tokens, universes up to 2^28.  SSJB_HEAD: 0 off, 1 auto (region
// of >= 2^30 window pairs), 2 forced (tests); SSJB_HEAD_MIN_SIZE: S0;
// SSJB_HEAD_K: head tokens (multiple of 128, <= 4096).
struct HeadPlan {
    bool ok = false;
    uint32_t S0 = 0, L0 = 0, base = 0, tile0 = 0, ntiles = 0, rows_pad = 0;
    int K = 0;                          // head tokens (GEMM depth in elements)
    int kind = dev::kKindF4;            // operand kind: kKindF4 (mxf4, K/2 bytes per row) or kKindI8
    int row_bytes() const { return kind == dev::kKindF4 ? K / 2 : K; }
    uint64_t pairs = 0;                 // region window pairs (the kernel's algorithmic work)
    std::vector<uint32_t> tile_col_lo;  // per row tile
    std::vector<uint2> items;           // (row tile, column chunk), chunk-major
};

HeadPlan make_head_plan(const Collection& c, const JoinPlan& plan, int W2) {
    HeadPlan h;
    const uint64_t mode = env_u64("SSJB_HEAD", 1);
    const size_t n = c.size();
    if (!mode || W2 != 4 || plan.naive || plan.cosine || !plan.bitmap.enabled || plan.row_end <= plan.row_begin ||
        c.max_size >= 65536 || c.universe > (uint64_t(1) << 28) || n >= (size_t(1) << 31))
        return h;
    const char* kenv = std::getenv("SSJB_HEAD_KIND");
    h.kind = kenv && std::string(kenv) == "i8" ? dev::kKindI8 : dev::kKindF4;
    // K: a multiple of one 128-byte pipeline slice (128 int8 / 256 e2m1 elements)
    const int kq = h.kind == dev::kKindF4 ? 2 * dev::kHeadSliceK : dev::kHeadSliceK;
    h.K = static_cast<int>(std::min<uint64_t>(4096, env_u64("SSJB_HEAD_K", 4096))) / kq * kq;
    if (h.K < kq) return h;
    // S0: the smallest size at which two records of that size may differ in
    // 64 sketch bits (maxham(2s) >= 64): from there on the 256-bit level-2
    // sketch stops pruning
    uint32_t S0 = static_cast<uint32_t>(env_u64("SSJB_HEAD_MIN_SIZE", 0));
    if (!S0) {
        S0 = 32;
        while (S0 <= c.max_size && 2 * size_t(S0) < plan.minov.size() &&
               2 * int64_t(S0) - 2 * int64_t(plan.minov[2 * S0]) < 64)
            ++S0;
    }
    if (S0 > c.max_size) return h;
    h.S0 = S0;
    h.L0 = c.first_ge[S0];
    const size_t r0 = std::max<size_t>(h.L0, plan.row_begin);
    if (r0 >= plan.row_end) return h;
    for (size_t i = r0; i < plan.row_end; ++i) {
        const size_t lo = std::max<size_t>(h.L0, window_start_of(c, plan, i));
        h.pairs += i > lo ? i - lo : 0;
    }
    if (h.pairs == 0 || (mode == 1 && h.pairs < (uint64_t(1) << 30))) return h;
    h.base = h.L0 & ~127u;
    h.tile0 = static_cast<uint32_t>(r0) & ~7u;
    h.ntiles = static_cast<uint32_t>((plan.row_end - h.tile0 + dev::kRowTile - 1) / dev::kRowTile);
    h.rows_pad = static_cast<uint32_t>(((n - h.base + 512) + 127) & ~size_t(127));
    h.tile_col_lo.assign(h.ntiles, 0);
    std::vector<std::pair<uint32_t, uint32_t>> it;  // (chunk, tile)
    for (uint32_t t = 0; t < h.ntiles; ++t) {
        const size_t first = std::max<size_t>(r0, size_t(h.tile0) + size_t(t) * dev::kRowTile);
        if (first >= plan.row_end) continue;
        const uint32_t lo = static_cast<uint32_t>(std::max<size_t>(h.L0, window_start_of(c, plan, first))) & ~7u;
        h.tile_col_lo[t] = std::max(lo, h.base);
        const size_t rmax = std::min<size_t>(size_t(h.tile0) + size_t(t + 1) * dev::kRowTile, plan.row_end);
        const size_t c1 = rmax - 1;  // columns j < i <= rmax - 1
        if (c1 <= h.tile_col_lo[t]) continue;
        for (size_t cc = (h.tile_col_lo[t] - h.base) / dev::kColChunk; cc <= (c1 - 1 - h.base) / dev::kColChunk; ++cc)
            it.emplace_back(static_cast<uint32_t>(cc), t);
    }
    std::sort(it.begin(), it.end());
    h.items.resize(it.size());
    for (size_t k = 0; k < it.size(); ++k) h.items[k] = make_uint2(it[k].second, it[k].first);
    h.ok = !h.items.empty();
    return h;
}

// make_head_plan of the collection's last join with the same rows, threshold,
// level-2 width and SSJB_HEAD* settings (host cache on the Collection, next to
// the tiling: the region's sampled token counts and work items are a few ms).
struct HeadPlanCacheEntry {
    size_t row_begin = 0, row_end = 0;
    std::vector<int32_t> minov;
    int W2 = 0;
    std::string env;
    std::shared_ptr<const HeadPlan> hp;
};

std::string head_env_key() {
    std::string k;
    for (const char* v : {"SSJB_HEAD", "SSJB_HEAD_KIND", "SSJB_HEAD_K", "SSJB_HEAD_MIN_SIZE"}) {
        const char* x = std::getenv(v);
        k += x ? x : "-";
        k += '|';
    }
    return k;
}

std::shared_ptr<const HeadPlan> cached_head_plan(const Collection& c, const JoinPlan& plan, int W2) {
    const std::string env = head_env_key();
    const bool cacheable = !plan.naive && !plan.cosine && plan.bitmap.enabled;
    {
        std::lock_guard<std::mutex> lk(c.plan_cache_mu);
        auto e = std::static_pointer_cast<HeadPlanCacheEntry>(c.head_cache);
        if (cacheable && e && e->row_begin == plan.row_begin && e->row_end == plan.row_end && e->W2 == W2 &&
            e->env == env && e->minov == plan.minov)
            return e->hp;
    }
    auto hp = std::make_shared<const HeadPlan>(make_head_plan(c, plan, W2));
    if (!cacheable) return hp;
    auto e = std::make_shared<HeadPlanCacheEntry>();
    e->row_begin = plan.row_begin;
    e->row_end = plan.row_end;
    e->minov = plan.minov;
    e->W2 = W2;
    e->env = env;
    e->hp = hp;
    std::lock_guard<std::mutex> lk(c.plan_cache_mu);
    c.head_cache = e;
    return hp;
}

// Device side of the head plan: head selection (token counts over the region,
// count threshold for the K most frequent, dense indices), the head operand
// and the per-row (size, tail) info.  Everything lives in the join's arena.
struct HeadDev {
    uint8_t* op = nullptr;
    uint32_t* info = nullptr;
    uint2* items = nullptr;
    uint32_t* col_lo = nullptr;
};

HeadDev head_setup(const DeviceReplica& rep, const Collection& c, const HeadPlan& h, Arena& A, cudaStream_t s,
                   int sms, uint64_t& launches) {
    HeadDev d;
    const uint32_t U = static_cast<uint32_t>(std::max<uint64_t>(c.universe, 1));
    const uint32_t n = static_cast<uint32_t>(c.size());
    uint32_t* cnt = A.alloc<uint32_t>(U);
    uint32_t* hist = A.alloc<uint32_t>(65536);
    uint32_t* thr = A.alloc<uint32_t>(2);
    uint16_t* map = A.alloc<uint16_t>(U);
    CK(cudaMemsetAsync(cnt, 0, size_t(U) * 4, s));
    CK(cudaMemsetAsync(hist, 0, 65536 * 4, s));
    CK(cudaMemsetAsync(thr, 0, 8, s));
    CK(cudaMemsetAsync(map, 0xFF, size_t(U) * 2, s));
    const unsigned g = static_cast<unsigned>(sms) * 8;
    // sample: about 2^24 region tokens (every stride-th region record)
    const uint64_t region_tokens = c.offsets[n] - c.offsets[h.L0];
    const uint32_t stride = static_cast<uint32_t>(std::max<uint64_t>(1, region_tokens >> 24));
    dev::head_count<<<g, 256, 0, s>>>(rep.tokens, rep.offsets, h.L0, n, stride, cnt);
    dev::head_hist<<<g, 256, 0, s>>>(cnt, U, hist);
    dev::head_threshold<<<1, 1024, 0, s>>>(hist, static_cast<uint32_t>(h.K), thr);
    dev::head_assign<<<g, 256, 0, s>>>(cnt, U, thr, static_cast<uint32_t>(h.K), map, thr + 1);
    d.op = A.alloc<uint8_t>(size_t(h.rows_pad) * h.row_bytes());
    d.info = A.alloc<uint32_t>(h.rows_pad);
    if (h.kind == dev::kKindF4)
        dev::head_expand<dev::kKindF4><<<h.rows_pad / 8, 256, 8 * h.row_bytes(), s>>>(
            rep.tokens, rep.offsets, n, h.L0, h.base, h.rows_pad / 8, h.K, map, d.op, d.info);
    else
        dev::head_expand<dev::kKindI8><<<h.rows_pad / 8, 256, 8 * h.row_bytes(), s>>>(
            rep.tokens, rep.offsets, n, h.L0, h.base, h.rows_pad / 8, h.K, map, d.op, d.info);
    launches += 5;
    CK(cudaGetLastError());
    d.items = A.alloc<uint2>(h.items.size());
    d.col_lo = A.alloc<uint32_t>(h.tile_col_lo.size());
    CK(cudaMemcpyAsync(d.items, h.items.data(), h.items.size() * sizeof(uint2), cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(d.col_lo, h.tile_col_lo.data(), h.tile_col_lo.size() * 4, cudaMemcpyHostToDevice, s));
    return d;
}

}  // namespace

// ------------------------------------------------------------ delivery
// Sorted result runs kept in HBM for the streaming delivery (plan.delivery 2):
// each run is (key = id_r << 32 | id_s, overlap) sorted by key.  A chunk of the
// canonical output is every pair with id_r in [ja, jb): per run a binary
// search bounds the segment, the segments are gathered, merged by K4 when
// there is more than one, packed to ssj_pair and downloaded.
struct DeviceRuns {
    int device = -1;
    int idbits = 1;
    std::vector<unsigned long long*> keys;
    std::vector<uint32_t*> ov;
    std::vector<uint64_t> len;
    ~DeviceRuns() {
        if (device < 0) return;
        int cur = 0;
        cudaGetDevice(&cur);
        cudaSetDevice(device);
        for (auto* p : keys) cudaFree(p);
        for (auto* p : ov) cudaFree(p);
        cudaSetDevice(cur);
    }
};

namespace {

void keep_device_run(EngineResult& out, int device, cudaStream_t s, const unsigned long long* keys,
                     const uint32_t* ov, uint64_t count, int idbits) {
    if (!count) return;
    if (!out.runs) {
        out.runs = std::make_shared<DeviceRuns>();
        out.runs->device = device;
    }
    DeviceRuns& R = *out.runs;
    R.idbits = std::max(R.idbits, idbits);
    unsigned long long* k = nullptr;
    uint32_t* v = nullptr;
    CK(cudaMalloc(&k, count * 8));
    CK(cudaMalloc(&v, count * 4));
    CK(cudaMemcpyAsync(k, keys, count * 8, cudaMemcpyDeviceToDevice, s));
    CK(cudaMemcpyAsync(v, ov, count * 4, cudaMemcpyDeviceToDevice, s));
    CK(cudaStreamSynchronize(s));
    R.keys.push_back(k);
    R.ov.push_back(v);
    R.len.push_back(count);
}

// per-id_r counts of one run
__global__ void run_histogram(const unsigned long long* keys, uint64_t n, unsigned int* hist, uint32_t hlen) {
    for (uint64_t k = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; k < n;
         k += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint32_t j = static_cast<uint32_t>(keys[k] >> 32);
        if (j < hlen) atomicAdd(hist + j, 1u);
    }
}

// lower_bound of key in each run: one thread per (run, bound)
struct RunTable {
    const unsigned long long* keys[64];
    uint64_t len[64];
};
__global__ void run_bounds(RunTable T, int nruns, unsigned long long lo_key, unsigned long long hi_key,
                           uint64_t* out) {
    const int t = threadIdx.x;
    if (t >= 2 * nruns) return;
    const int r = t >> 1;
    const unsigned long long key = (t & 1) ? hi_key : lo_key;
    uint64_t a = 0, b = T.len[r];
    while (a < b) {
        const uint64_t m = (a + b) >> 1;
        if (T.keys[r][m] < key) a = m + 1;
        else b = m;
    }
    out[t] = a;
}

cudaStream_t runs_stream(int device) {
    static thread_local cudaStream_t streams[16] = {};
    if (!streams[device & 15]) CK(cudaStreamCreateWithFlags(&streams[device & 15], cudaStreamNonBlocking));
    return streams[device & 15];
}

}  // namespace

uint64_t runs_total(const DeviceRuns& R) {
    uint64_t t = 0;
    for (uint64_t l : R.len) t += l;
    return t;
}

void runs_histogram(const DeviceRuns& R, std::vector<uint64_t>& hist) {
    if (R.keys.empty() || hist.empty()) return;
    set_device(R.device);
    cudaStream_t s = runs_stream(R.device);
    const uint32_t hlen = static_cast<uint32_t>(hist.size());
    unsigned int* d = nullptr;
    CK(cudaMallocAsync(&d, hlen * 4ull, s));
    CK(cudaMemsetAsync(d, 0, hlen * 4ull, s));
    for (size_t r = 0; r < R.keys.size(); ++r) {
        const unsigned g = static_cast<unsigned>(std::min<uint64_t>((R.len[r] + 255) / 256, 148 * 16));
        run_histogram<<<g, 256, 0, s>>>(R.keys[r], R.len[r], d, hlen);
        CK(cudaGetLastError());
    }
    std::vector<unsigned int> h(hlen);
    CK(cudaMemcpyAsync(h.data(), d, hlen * 4ull, cudaMemcpyDeviceToHost, s));
    CK(cudaFreeAsync(d, s));
    CK(cudaStreamSynchronize(s));
    for (uint32_t j = 0; j < hlen; ++j) hist[j] += h[j];
}

void runs_extract(const DeviceRuns& R, uint32_t ja, uint32_t jb, PairVec& out) {
    if (R.keys.empty() || ja >= jb) return;
    set_device(R.device);
    cudaStream_t s = runs_stream(R.device);
    // segment bounds per run (in groups of 64 runs)
    std::vector<uint64_t> lo(R.keys.size()), hi(R.keys.size());
    {
        uint64_t* d = nullptr;
        CK(cudaMallocAsync(&d, 128 * 8, s));
        for (size_t base = 0; base < R.keys.size(); base += 64) {
            RunTable T{};
            const int nr = static_cast<int>(std::min<size_t>(64, R.keys.size() - base));
            for (int r = 0; r < nr; ++r) {
                T.keys[r] = R.keys[base + r];
                T.len[r] = R.len[base + r];
            }
            run_bounds<<<1, 128, 0, s>>>(T, nr, static_cast<unsigned long long>(ja) << 32,
                                         static_cast<unsigned long long>(jb) << 32, d);
            CK(cudaGetLastError());
            uint64_t h[128];
            CK(cudaMemcpyAsync(h, d, 2 * nr * 8, cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s));
            for (int r = 0; r < nr; ++r) {
                lo[base + r] = h[2 * r];
                hi[base + r] = h[2 * r + 1];
            }
        }
        CK(cudaFreeAsync(d, s));
    }
    uint64_t total = 0;
    for (size_t r = 0; r < lo.size(); ++r) total += hi[r] - lo[r];
    if (!total) return;
    Arena A(s);
    uint64_t launches = 0;
    SortBufs SB{};
    SB.ka = A.alloc<unsigned long long>(total);
    SB.va = A.alloc<uint32_t>(total);
    uint64_t at = 0;
    int nonempty = 0;
    for (size_t r = 0; r < lo.size(); ++r) {
        const uint64_t len = hi[r] - lo[r];
        if (!len) continue;
        ++nonempty;
        CK(cudaMemcpyAsync(SB.ka + at, R.keys[r] + lo[r], len * 8, cudaMemcpyDeviceToDevice, s));
        CK(cudaMemcpyAsync(SB.va + at, R.ov[r] + lo[r], len * 4, cudaMemcpyDeviceToDevice, s));
        at += len;
    }
    bool inb = false;
    if (nonempty > 1) {  // merge the runs' segments (K4 over the gathered chunk)
        SB.kb = A.alloc<unsigned long long>(total);
        SB.vb = A.alloc<uint32_t>(total);
        const uint32_t max_tiles = static_cast<uint32_t>((total + dev::kSortTile - 1) / dev::kSortTile);
        SB.hist = A.alloc<uint32_t>(256ull * max_tiles);
        SB.sums = A.alloc<uint32_t>((256ull * max_tiles + dev::kScanBlock - 1) / dev::kScanBlock + 1);
        unsigned long long* cnt = A.alloc<unsigned long long>(1);
        const unsigned long long tot = total;
        CK(cudaMemcpyAsync(cnt, &tot, 8, cudaMemcpyHostToDevice, s));
        SB.count = cnt;
        inb = sort_results(SB, total, R.idbits, s, launches);
    }
    PairOut* packed = A.alloc<PairOut>(total);
    pack_pairs<<<static_cast<unsigned>((total + 255) / 256), 256, 0, s>>>(inb ? SB.kb : SB.ka, inb ? SB.vb : SB.va,
                                                                        packed, total);
    CK(cudaGetLastError());
    const size_t old = out.size();
    out.resize(old + total);
    d2h_staged(out.data() + old, packed, total * sizeof(PairOut), s);
}

int engine_device_count() {
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return count;
}

void engine_pin(const Collection& c, int device) {
    set_device(device);
    cudaStream_t s;
    CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    uint64_t h2d = 0, launches = 0;
    std::shared_ptr<DeviceReplica> rep;
    {
        std::lock_guard<std::mutex> lk(c.dev_mu);
        register_host(c);
    }
    rep = upload(c, device, s, h2d, launches, true);
    CK(cudaStreamSynchronize(s));
    cudaStreamDestroy(s);
    std::lock_guard<std::mutex> lk(c.dev_mu);
    c.pinned[device & 15] = rep;
}

void engine_unpin(const Collection& c, int device) {
    std::lock_guard<std::mutex> lk(c.dev_mu);
    c.pinned[device & 15].reset();
}

void engine_release_host(const Collection& c) {
    if (!c.host_registered) return;
    if (c.use_delta8) {
        cudaHostUnregister(c.tokens8.data());
        cudaHostUnregister(c.exc_start.data());
        if (!c.exc_val.empty()) cudaHostUnregister(c.exc_val.data());
    }
    else if (narrow_tokens(c)) cudaHostUnregister(c.tokens16.data());
    else if (!c.tokens.empty()) cudaHostUnregister(const_cast<uint32_t*>(c.tokens.data()));
    cudaHostUnregister(const_cast<uint64_t*>(c.offsets.data()));
    cudaGetLastError();
    c.host_registered = false;
}

void engine_build_bitmaps(const Collection& c, Method method, int width, int hash, int device,
                          uint64_t* out_host) {
    set_device(device);
    cudaStream_t s;
    CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    {
        uint64_t h2d = 0, launches = 0;
        auto rep = replica_for(c, device, s, h2d, launches);
        Arena A(s);
        const int W = width / 64;
        uint64_t* bits = A.alloc<uint64_t>((c.size() + kPadRows) * W);
        if (!launch_build_sub(*rep, bits, nullptr, method, width, 0, hash, s, launches))
            launch_build(*rep, bits, method, width, hash, s, launches);
        if (c.size())
            CK(cudaMemcpyAsync(out_host, bits, c.size() * W * sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
    }
    cudaStreamDestroy(s);
}

namespace {
// Reads a buffer larger than L2 (clean lines only: a write-based flush would
// leave ~126 MB of dirty lines whose write-back lands inside the timed kernel).
__global__ void l2_flush_read(const uint4* buf, size_t n16, unsigned int* sink) {
    uint32_t acc = 0;
    for (size_t k = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; k < n16;
         k += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const uint4 v = __ldcg(buf + k);
        acc ^= v.x ^ v.y ^ v.z ^ v.w;
    }
    if (acc == 0x9E3779B9u) atomicAdd(sink, 1u);  // keeps the loads alive
}
}  // namespace

double engine_time_build(const Collection& c, Method method, int width, int hash, int device, int reps) {
    // K1 alone on the device replica, L2 flushed (256 MiB read) before every
    // timed launch so the token stream comes from HBM; mean ms per launch
    set_device(device);
    cudaStream_t s;
    CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    double total = 0;
    {
        uint64_t h2d = 0, launches = 0;
        auto rep = replica_for(c, device, s, h2d, launches);
        Arena A(s);
        const int W = width / 64;
        uint64_t* bits = A.alloc<uint64_t>((c.size() + kPadRows) * W);
        const size_t flush_bytes = size_t(256) << 20;
        uint8_t* flush = A.alloc<uint8_t>(flush_bytes);
        unsigned int* sink = A.alloc<unsigned int>(1);
        CK(cudaMemsetAsync(flush, 0, flush_bytes, s));
        int sms = 148;
        CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
        Timer T(s);
        for (int r = 0; r < reps + 1; ++r) {
            l2_flush_read<<<static_cast<unsigned>(sms * 8), 512, 0, s>>>(reinterpret_cast<const uint4*>(flush),
                                                                     flush_bytes / 16, sink);
            CK(cudaGetLastError());
            cudaEvent_t a = T.mark();
            if (!launch_build_sub(*rep, bits, nullptr, method, width, 0, hash, s, launches))
                launch_build(*rep, bits, method, width, hash, s, launches);
            cudaEvent_t b = T.mark();
            CK(cudaStreamSynchronize(s));
            if (r > 0) total += Timer::ms(a, b);  // first launch: warm-up
        }
    }
    cudaStreamDestroy(s);
    return reps > 0 ? total / reps : 0.0;
}

namespace {
// Survivor and result buffers of one join in flight on one device, kept
// across joins (grown, never shrunk): per-join stream-ordered allocations of
// these multi-GB buffers from several threads at once make the memory pool
// map fresh pages, stalling concurrent joins.
struct JoinWorkspace {
    int device = -1;
    uint2* surv = nullptr;
    uint64_t surv_cap = 0;
    unsigned long long *ka = nullptr, *kb = nullptr;
    uint32_t *va = nullptr, *vb = nullptr, *hist = nullptr, *sums = nullptr;
    uint64_t res_cap = 0;
    ~JoinWorkspace() { release(); }
    void release() {
        if (device < 0) return;
        int cur = 0;
        cudaGetDevice(&cur);
        cudaSetDevice(device);
        cudaFree(surv);
        cudaFree(ka);
        cudaFree(kb);
        cudaFree(va);
        cudaFree(vb);
        cudaFree(hist);
        cudaFree(sums);
        cudaSetDevice(cur);
        surv = nullptr;
        ka = kb = nullptr;
        va = vb = hist = sums = nullptr;
        surv_cap = res_cap = 0;
    }
    uint64_t bytes() const { return surv_cap * sizeof(uint2) + res_cap * 24; }
    // (buffers may still be in use by the stream: callers synchronise it first).
    // Every pointer is nulled and its capacity zeroed as soon as it is freed, so
    // a failed (throwing) allocation leaves an empty workspace, never a stale
    // capacity over freed memory.
    void ensure(int dev, uint64_t scap, uint64_t rcap) {
        device = dev;
        if (scap > surv_cap) {
            cudaFree(surv);
            surv = nullptr;
            surv_cap = 0;
            CK(cudaMalloc(&surv, scap * sizeof(uint2)));
            surv_cap = scap;
        }
        if (rcap > res_cap) {
            for (void** p : {reinterpret_cast<void**>(&ka), reinterpret_cast<void**>(&kb),
                             reinterpret_cast<void**>(&va), reinterpret_cast<void**>(&vb),
                             reinterpret_cast<void**>(&hist), reinterpret_cast<void**>(&sums)}) {
                cudaFree(*p);
                *p = nullptr;
            }
            res_cap = 0;
            const uint64_t tiles = (rcap + dev::kSortTile - 1) / dev::kSortTile;
            CK(cudaMalloc(&ka, rcap * 8));
            CK(cudaMalloc(&kb, rcap * 8));
            CK(cudaMalloc(&va, rcap * 4));
            CK(cudaMalloc(&vb, rcap * 4));
            CK(cudaMalloc(&hist, 256ull * tiles * 4));
            CK(cudaMalloc(&sums, ((256ull * tiles + dev::kScanBlock - 1) / dev::kScanBlock + 1) * 4));
            res_cap = rcap;
        }
    }
};

// Workspaces live in a per-device pool: a join leases one (a concurrent join
// gets another), so short-lived host threads -- one per device in multi-GPU
// joins -- reuse buffers across calls instead of re-allocating them.
struct WorkspacePool {
    std::mutex mu;
    std::vector<std::unique_ptr<JoinWorkspace>> idle[16];
};
WorkspacePool& workspace_pool() {
    static WorkspacePool* p = new WorkspacePool();  // leaked: outlives thread/static teardown
    return *p;
}

// Idle workspace bytes kept per device (SSJB_WORKSPACE_KEEP_MB, default a
// quarter of the device's HBM): a dense join grows its workspace to tens of
// GB; beyond this budget a returned workspace is freed instead of pooled.
uint64_t workspace_keep_bytes(int device) {
    static uint64_t keep[16] = {};
    static std::once_flag once[16];
    std::call_once(once[device & 15], [device]() {
        const uint64_t mb = env_u64("SSJB_WORKSPACE_KEEP_MB", 0);
        size_t f = 0, t = 0;
        int cur = 0;
        cudaGetDevice(&cur);
        cudaSetDevice(device);
        if (cudaMemGetInfo(&f, &t) != cudaSuccess) t = 0;
        cudaSetDevice(cur);
        keep[device & 15] = mb ? (mb << 20) : t / 4;
    });
    return keep[device & 15];
}

struct WorkspaceLease {
    int device;
    cudaStream_t stream;
    std::unique_ptr<JoinWorkspace> ws;
    int uncaught;
    WorkspaceLease(int dev, cudaStream_t s) : device(dev), stream(s), uncaught(std::uncaught_exceptions()) {
        WorkspacePool& P = workspace_pool();
        std::lock_guard<std::mutex> lk(P.mu);
        auto& v = P.idle[dev & 15];
        if (!v.empty()) {
            ws = std::move(v.back());
            v.pop_back();
        } else {
            ws = std::make_unique<JoinWorkspace>();
        }
    }
    ~WorkspaceLease() {
        cudaStreamSynchronize(stream);  // nothing queued may still use the buffers
        // a join that failed (e.g. an allocation inside ensure) returns nothing
        // to the pool: its buffers are freed with it
        if (std::uncaught_exceptions() > uncaught) {
            ws->release();
            return;
        }
        WorkspacePool& P = workspace_pool();
        std::lock_guard<std::mutex> lk(P.mu);
        auto& v = P.idle[device & 15];
        uint64_t held = ws->bytes();
        for (auto& w : v) held += w->bytes();
        if (held > workspace_keep_bytes(device)) ws->release();  // keep the (empty) object
        v.push_back(std::move(ws));
    }
};
}  // namespace

uint32_t engine_head_start(const Collection& c, const JoinPlan& plan) {
    const int W = plan.bitmap.enabled ? plan.bitmap.width / 64 : 0;
    const bool set_or_xor = plan.bitmap.method == Method::Set || plan.bitmap.method == Method::Xor;
    if (!plan.bitmap.enabled || W < 1 || W > 2 || !set_or_xor || plan.bitmap.width % 64) return UINT32_MAX;
    const HeadPlan h = make_head_plan(c, plan, level2_words(W));
    return h.ok ? h.L0 : UINT32_MAX;
}

// Frees every idle join workspace of `device` (all devices for -1).
void engine_trim(int device) {
    WorkspacePool& P = workspace_pool();
    std::lock_guard<std::mutex> lk(P.mu);
    for (int d = 0; d < 16; ++d) {
        if (device >= 0 && d != (device & 15)) continue;
        for (auto& w : P.idle[d]) w->release();
        P.idle[d].clear();
    }
}

void engine_join(const Collection& c, const JoinPlan& plan, int device, EngineResult& out) {
    using Clock = std::chrono::steady_clock;
    const auto t_enter = Clock::now();
    set_device(device);
    // one non-blocking stream per (host thread, device), reused across joins
    static thread_local cudaStream_t streams[16] = {};
    if (!streams[device & 15]) CK(cudaStreamCreateWithFlags(&streams[device & 15], cudaStreamNonBlocking));
    cudaStream_t s = streams[device & 15];
    EngineStats& st = out.stats;
    st.window_pairs = plan.window_pairs;
    const auto t_start = Clock::now();
    // SSJB_HOST_TIMING=2: host timestamps of the join's phases (stderr)
    const bool host_trace = env_u64("SSJB_HOST_TIMING", 0) >= 2;
    std::vector<std::pair<const char*, Clock::time_point>> hmarks;
    auto hmark = [&](const char* what) {
        if (host_trace) hmarks.emplace_back(what, Clock::now());
    };
    Timer T(s);
    Arena A(s);

    const size_t n = c.size();
    const uint32_t rows = static_cast<uint32_t>(plan.row_end - plan.row_begin);
    const bool naive = plan.naive;
    const bool enabled = !naive && plan.bitmap.enabled;
    const int width = enabled ? plan.bitmap.width : 64;
    const int W = width / 64;
    if (enabled && (width <= 0 || width % 64 != 0))
        throw std::invalid_argument("bitmap width must be a positive multiple of 64");
    if (enabled && plan.bitmap.cutoff < 0) throw std::invalid_argument("bitmap cutoff must be >= 0");

    cudaEvent_t e0 = T.mark();
    // plan tables (staged, sent with the tiling tables in one copy below)
    TableStage stage;
    int32_t* d_maxham = nullptr;
    int32_t* d_minov = nullptr;
    uint32_t* d_wstart = nullptr;
    std::vector<int32_t> maxham(plan.minov.size());
    for (size_t S = 0; S < maxham.size(); ++S) maxham[S] = static_cast<int32_t>(S) - 2 * plan.minov[S];
    stage.add(&d_maxham, maxham.data(), maxham.size() * 4);
    stage.add(&d_minov, plan.minov.data(), plan.minov.size() * 4);
    stage.add(&d_wstart, plan.window_start.data(), plan.window_start.size() * 4);

    // K1: sketches (+ level-2 Xor sketches), reused from a resident replica's cache
    const int W2 = enabled ? level2_words(W) : 0;
    // K2 flavour: tcgen05 int8 GEMM filter where it applies, POPC otherwise
    const char* fenv = std::getenv("SSJB_FILTER");
    const bool tc_ok = enabled && W <= 4 && plan.row_begin % 8 == 0;
    const bool use_tc = tc_ok && !(fenv && std::string(fenv) == "popc");
    bool l2gemm = false;
    bool l2_auto = false;  // may switch to the level-2 GEMM when level-1 survivors overflow
    if (use_tc && W <= 2 && W2 == 4) {
        const char* genv = std::getenv("SSJB_L2GEMM");
        l2_auto = !(genv && *genv);
        if (genv && *genv) {
            l2gemm = std::atoi(genv) != 0;
        } else {
            // dense regime: the b-bit Xor sketch stops discriminating near the
            // median record size (the paper's cutoff analysis), so most window
            // pairs survive level 1 and the level-2 check runs as a GEMM too
            const int64_t cx = cutoff(Method::Xor, width, Rational(plan.p, plan.q), true);
            static const double factor = [] {
                const char* v = std::getenv("SSJB_L2GEMM_FACTOR");
                return v && *v ? std::atof(v) : 1.25;
            }();
            l2gemm = static_cast<double>(cx) < factor * static_cast<double>(c.median_size());
        }
    }
    // K3a: exact head-token overlaps for the large-record region of dense joins
    // (head_tc.cuh); active whenever the join runs the level-2 GEMM
    hmark("plan tables");
    std::shared_ptr<const HeadPlan> hplan_p =
        use_tc && W <= 2 && W2 == 4 ? cached_head_plan(c, plan, W2) : std::make_shared<const HeadPlan>();
    const HeadPlan& hplan = *hplan_p;
    hmark("head plan");
    // a head region of >= 2^30 window pairs of large records means a dense join:
    // start on the level-2 GEMM instead of discovering it by a level-1 pass
    // that overflows (C4: the discarded pass and its operands)
    if (l2_auto && !l2gemm && hplan.ok && env_u64("SSJB_HEAD_PREDICT", 1) != 0) l2gemm = true;
    bool head_active = l2gemm && hplan.ok;
    const bool head_upfront = head_active;  // batch mode from the start (no single-pass fast path)
    const char* kenv = std::getenv("SSJB_TC_KIND");
    // operand kind: fp4 (packed e2m1) halves the operand bytes and doubles the
    // MMA rate per element, which wins for b >= 192 (C2 b=256 sweep: 7.96 vs
    // 10.0 ms); at b <= 128 the int8 kernel's 256-column tiles are faster
    // (C2 b=128: 9.0 vs 22.5 ms).  SSJB_TC_KIND=i8|fp4 overrides.
    const bool fp4 = use_tc && !l2gemm &&
                     (kenv && *kenv ? std::string(kenv) == "fp4" : W >= 3);
    // int8 level-1-only filter on a CTA pair (M = 256): experimental, opt in with SSJB_TC2=1
    const bool use_tc2 = use_tc && !l2gemm && !fp4 && W <= 2 && env_u64("SSJB_TC2", 0) != 0;
    // single-CTA int8 level-1 filter without the popcount extension (K = b, the
    // -pc_j term added per column in the epilogue): 20% fewer MMA steps, but the
    // extra epilogue work (and register pressure at 96 registers x 576 threads)
    // outweighs them (C2 tau=0.7: 0.86 vs 0.69 ms) -- opt in with SSJB_NOEXT=1
    const bool noext = use_tc && !l2gemm && !fp4 && !use_tc2 && W <= 2 && env_u64("SSJB_NOEXT", 0) != 0;
    // two row tiles per staged column tile (256-row work items, one CTA)
    const bool use_tcm = use_tc && !l2gemm && !fp4 && !use_tc2 && !noext && W <= 2 && env_u64("SSJB_TCM", 1) != 0;

    // work items: (row tile, 4096-column chunk); the pair kernel takes 256-row tiles
    std::shared_ptr<const Tiling> tlp = std::make_shared<Tiling>();
    uint64_t* d_item_base = nullptr;
    uint32_t* d_col_lo = nullptr;
    uint32_t* d_item_tile = nullptr;
    uint32_t* d_item_order = nullptr;
    // column-chunk-major claim order for collections whose operands exceed L2
    // (tcgen05 single-CTA kernels; per-chunk streamed filter launches keep item order)
    const bool item_ordered = use_tc && !use_tc2 && n >= env_u64("SSJB_ORDER_MIN_ROWS", 262144) &&
                              env_u64("SSJB_STREAM", 1) < 2 && env_u64("SSJB_ITEM_ORDER", 1) != 0;
    // The collection on the device: a pinned replica, or uploaded for this join --
    // streamed in row chunks when the whole self-join runs here.  A dense join
    // (batch mode from the start) streams a small first chunk (1/16 of the
    // tokens, SSJB_STREAM_CHUNKS_BATCH) whose rows' work items (C4: ~57% of the
    // filter work) are claimed first and filtered while the rest is in flight.
    std::shared_ptr<DeviceReplica> rep;
    {
        std::lock_guard<std::mutex> lk(c.dev_mu);
        if (c.pinned[device & 15] && c.pinned[device & 15]->device == device) rep = c.pinned[device & 15];
    }
    const bool set_or_xor = plan.bitmap.method == Method::Set || plan.bitmap.method == Method::Xor;
    const bool will_stream = !rep && use_tc && set_or_xor && W <= 8 && plan.row_begin == 0 && plan.row_end == n &&
                             n >= env_u64("SSJB_STREAM_MIN_ROWS", 65536) && n > 0 && env_u64("SSJB_STREAM", 1) != 0;
    const bool two_phase = will_stream && head_upfront && env_u64("SSJB_STREAM", 1) < 2 &&
                           env_u64("SSJB_STREAM_PHASES", 1) != 0;
    const int stream_chunks = static_cast<int>(two_phase ? std::max<uint64_t>(2, env_u64("SSJB_STREAM_CHUNKS_BATCH", 16))
                                                         : env_u64("SSJB_STREAM_CHUNKS", 2));
    const uint32_t phase_tile_rows = use_tc2 || use_tcm ? 2 * dev::kRowTile : dev::kRowTile;
    uint32_t split_row = 0;  // first row of the second streaming phase (upload_streamed's first chunk end)
    if (two_phase) {
        const uint64_t target = c.tokens.size() / static_cast<uint64_t>(stream_chunks);
        const size_t r = std::lower_bound(c.offsets.begin(), c.offsets.end(), target) - c.offsets.begin();
        split_row = static_cast<uint32_t>(std::min<size_t>(n, (r + phase_tile_rows - 1) / phase_tile_rows * phase_tile_rows));
        if (split_row >= n) split_row = 0;
    }
    auto set_tiling = [&](uint32_t tile_rows) {
        tlp = cached_tiling(c, plan, tile_rows, item_ordered,
                            split_row && tile_rows == phase_tile_rows ? split_row / tile_rows : 0);
        stage.add(&d_item_base, tlp->item_base.data(), tlp->item_base.size() * 8);
        stage.add(&d_col_lo, tlp->col_lo.data(), tlp->col_lo.size() * 4);
        stage.add(&d_item_tile, tlp->item_tile.data(), tlp->item_tile.size() * 4);
        if (!tlp->order.empty()) stage.add(&d_item_order, tlp->order.data(), tlp->order.size() * 4);
        stage.flush(A, s, st.h2d_bytes);
    };
    set_tiling(use_tc2 || use_tcm ? 2 * dev::kRowTile : dev::kRowTile);
    hmark("tiling staged");

    std::vector<IngestChunk> ingest;
    uint16_t* ingest_t16 = nullptr;
    Delta8Dev ingest_d8;
    if (will_stream) {
        static thread_local cudaStream_t copy_streams[16] = {};
        if (!copy_streams[device & 15])
            CK(cudaStreamCreateWithFlags(&copy_streams[device & 15], cudaStreamNonBlocking));
        rep = upload_streamed(c, device, s, copy_streams[device & 15], tlp->tile_rows, stream_chunks, st.h2d_bytes,
                              st.launches, ingest, ingest_t16, ingest_d8);
    } else if (!rep) {
        rep = replica_for(c, device, s, st.h2d_bytes, st.launches);
    }
    const bool streamed = !ingest.empty();
    size_t ingest_pending = 0;  // first chunk whose ingest kernels are not enqueued yet (two-phase streaming)
    uint64_t phase_items = 0;   // claim positions [0, phase_items) read only the first chunk's rows
    uint64_t* l3_bits = nullptr;
    cudaEvent_t e_up = T.mark();
    const uint32_t n_pad = static_cast<uint32_t>(((n + kPadRows) + 7) & ~size_t(7));
    const bool resident = rep->stream == nullptr;
    std::shared_ptr<SketchSet> sk;
    // resident replicas build sketches/operands once, under the collection lock
    std::unique_lock<std::mutex> cache_lock(c.dev_mu, std::defer_lock);
    if (resident) {
        cache_lock.lock();
        sk = rep->sketches;
    }
    auto get = [&](size_t bytes) -> void* {
        void* p = nullptr;
        if (resident) CK(cudaMalloc(&p, bytes));
        else p = A.alloc<uint8_t>(bytes);
        return p;
    };
    const int mcode = enabled ? static_cast<int>(plan.bitmap.method) : -2;
    bool built = false;
    if (enabled && !(sk && sk->method == mcode && sk->width == width && sk->hash == plan.bitmap.hash &&
                     sk->words2 == W2)) {
        auto fresh = std::make_shared<SketchSet>();
        fresh->device = device;
        fresh->method = mcode;
        fresh->width = width;
        fresh->hash = plan.bitmap.hash;
        fresh->words2 = W2;
        fresh->owned = resident;
        fresh->bits = static_cast<uint64_t*>(get((n + kPadRows + 8) * W * 8));
        CK(cudaMemsetAsync(fresh->bits + n * W, 0, (kPadRows + 8) * W * 8, s));
        if (W2) {
            fresh->bits2 = static_cast<uint64_t*>(get((n + kPadRows + 8) * W2 * 8));
            CK(cudaMemsetAsync(fresh->bits2 + n * W2, 0, (kPadRows + 8) * W2 * 8, s));
        }
        // one token pass for both sketches where the sub-warp builder applies
        // (streamed ingest: built chunk by chunk before each chunk's filter work)
        if (streamed) {
        } else if (!launch_build_sub(*rep, fresh->bits, fresh->bits2, plan.bitmap.method, width, 64 * W2,
                                     plan.bitmap.hash, s, st.launches)) {
            launch_build(*rep, fresh->bits, plan.bitmap.method, width, plan.bitmap.hash, s, st.launches);
            if (W2 && !launch_build_sub(*rep, fresh->bits2, nullptr, Method::Xor, 64 * W2, 0, plan.bitmap.hash, s,
                                        st.launches))
                launch_build(*rep, fresh->bits2, Method::Xor, 64 * W2, plan.bitmap.hash, s, st.launches);
        }
        sk = fresh;
        built = true;
    }
    const int variant = !use_tc ? -1 : (l2gemm ? 1 : (fp4 ? 2 : (use_tc2 ? 3 : (noext ? 4 : 0))));
    if (variant == 4 && !sk->npc2) {
        sk->npc2 = static_cast<uint32_t*>(get(static_cast<size_t>(n_pad / 2 + 1) * 4));
        if (!streamed) launch_column_info(sk->bits, W, 0, n_pad, sk->npc2, s, st.launches);
        built = true;
    }
    if (variant >= 0 && !sk->opA[variant]) {
        const size_t rowb = operand_row(W, variant);
        sk->opA[variant] = static_cast<uint8_t*>(get(static_cast<size_t>(n_pad) * rowb));
        sk->opB[variant] = static_cast<uint8_t*>(get(static_cast<size_t>(n_pad) * rowb));
        if (streamed) {
            // tiles near the diagonal load (masked) columns of the next chunk
            // before it is expanded: keep them zero, i.e. size 0, a valid index
            CK(cudaMemsetAsync(sk->opA[variant], 0, static_cast<size_t>(n_pad) * rowb, s));
            CK(cudaMemsetAsync(sk->opB[variant], 0, static_cast<size_t>(n_pad) * rowb, s));
        } else {
            launch_expand(sk->bits, W, sk->bits2, W2, rep->sizes, sk->opA[variant], sk->opB[variant], n_pad, variant,
                          s, st.launches);
        }
        built = true;
    }
    if (resident) {
        if (built) {
            CK(cudaStreamSynchronize(s));  // publish only finished sketches
            rep->sketches = sk;
        }
        cache_lock.unlock();
    }
    uint64_t* d_bits = enabled ? sk->bits : A.alloc<uint64_t>((n + kPadRows + 8) * W);
    uint64_t* d_bits2 = enabled && W2 ? sk->bits2 : nullptr;
    uint8_t* d_opA = variant >= 0 ? sk->opA[variant] : nullptr;
    uint8_t* d_opB = variant >= 0 ? sk->opB[variant] : nullptr;
    cudaEvent_t e_build = T.mark();
    hmark("upload+build enqueued");

    // buffers
    // buffer sizing: survivors (8 B) and result sort buffers (24 B); a batch's
    // results must fit the result buffer, so res_cap >= surv_cap.  With the HBM
    // of a B200 free, larger buffers mean fewer filter batches / result runs.
    // free HBM when this device was first used (one query per device and process)
    static size_t free_at_first[16] = {};
    static std::once_flag mem_once[16];
    std::call_once(mem_once[device & 15], [device]() {
        size_t f = 0, t = 0;
        if (cudaMemGetInfo(&f, &t) == cudaSuccess) free_at_first[device & 15] = f;
    });
    const size_t free_b = free_at_first[device & 15];
    const uint64_t big = free_b >= (size_t(64) << 30) ? 1 : 0;
    // live free HBM for the optional large buffers below (queried only when a
    // decision depends on it: earlier joins may hold pooled workspaces, pins)
    size_t live_free_b = 0;
    auto live_free = [&]() -> size_t {
        if (!live_free_b) {
            size_t f = 0, t = 0;
            if (cudaMemGetInfo(&f, &t) == cudaSuccess) live_free_b = f;
        }
        return live_free_b;
    };
    uint64_t surv_cap =
        std::max<uint64_t>(env_u64("SSJB_SURVIVOR_CAP", uint64_t(1) << (27 + big)), 1u << 20);
    uint64_t res_cap = std::max<uint64_t>(env_u64("SSJB_RESULT_CAP", uint64_t(1) << 26), surv_cap);
    WorkspaceLease lease(device, s);
    hmark("workspace");
    JoinWorkspace& WS = *lease.ws;
    const bool use_ws = env_u64("SSJB_WORKSPACE", 1) != 0;
    if (use_ws) {
        CK(cudaStreamSynchronize(s));  // the previous join on this stream is done with them
        WS.ensure(device, surv_cap, res_cap);
    }
    uint2* d_surv = use_ws ? WS.surv : A.alloc<uint2>(surv_cap);
    uint32_t* d_rowcnt = A.alloc<uint32_t>(rows + 1);
    uint32_t* d_rowsnap = A.alloc<uint32_t>(rows + 1);
    uint32_t* d_jstar = A.alloc<uint32_t>(rows + 1);
    uint32_t* d_satlist = A.alloc<uint32_t>(rows + 1);
    // per-(item,row) survivor counts let the saturation rescan touch one chunk per row
    uint64_t n_items = tlp->item_base.back();
    const uint64_t ic_bytes = n_items * tlp->tile_rows * 4;
    const bool keep_item_counts =
        !naive && (ic_bytes <= (uint64_t(1) << 30) ||
                   (ic_bytes <= (uint64_t(16) << 30) && static_cast<double>(ic_bytes) <= 0.3 * double(live_free())));
    uint32_t* d_item_counts = keep_item_counts ? A.alloc<uint32_t>(n_items * tlp->tile_rows) : nullptr;
    // second level: per (item, filter tile, column part, row) counts written by the
    // tcgen05 epilogue (plain u16 stores, no memset: every slot of a processed
    // tile is written), so a saturated row's rescan covers one filter tile
    // instead of a 4096-column chunk (32 tiles per item covers widths >= 128)
    constexpr uint32_t kTilesPerItem = dev::kColChunk / 128;
    const uint64_t tc_bytes = n_items * kTilesPerItem * 4 * dev::kRowTile * 2;
    // (kept for the dense regime only -- the level-2 GEMM joins, where most rows
    // saturate; elsewhere the stores cost the filter more than the rescan saves)
    uint16_t* d_tile_counts = keep_item_counts && use_tc && l2gemm && !use_tc2 && tlp->tile_rows == dev::kRowTile &&
                                      tc_bytes <= std::min<uint64_t>(uint64_t(2) << 30, live_free() / 5)
                                  ? A.alloc<uint16_t>(n_items * kTilesPerItem * 4 * dev::kRowTile)
                                  : nullptr;
    dev::Control* d_ctl = A.alloc<dev::Control>(1);
    SortBufs SB{};
    auto alloc_results = [&]() {
        if (use_ws) {
            WS.ensure(device, surv_cap, res_cap);
            SB.ka = WS.ka;
            SB.kb = WS.kb;
            SB.va = WS.va;
            SB.vb = WS.vb;
            SB.hist = WS.hist;
            SB.sums = WS.sums;
            return;
        }
        SB.ka = A.alloc<unsigned long long>(res_cap);
        SB.va = A.alloc<uint32_t>(res_cap);
        SB.kb = A.alloc<unsigned long long>(res_cap);
        SB.vb = A.alloc<uint32_t>(res_cap);
        const uint32_t max_tiles = static_cast<uint32_t>((res_cap + dev::kSortTile - 1) / dev::kSortTile);
        SB.hist = A.alloc<uint32_t>(256ull * max_tiles);
        SB.sums = A.alloc<uint32_t>((256ull * max_tiles + dev::kScanBlock - 1) / dev::kScanBlock + 1);
    };
    alloc_results();
    CK(cudaMemsetAsync(d_rowcnt, 0, (rows + 1) * 4, s));
    CK(cudaMemsetAsync(d_ctl, 0, sizeof(dev::Control), s));
    dev::Control h_ctl{};

    // filter launch configuration
    const FilterFn ffn = filter_fn(W, W2);
    const size_t fsmem = filter_smem(W, W2);
    set_smem_once(reinterpret_cast<const void*>(ffn), static_cast<int>(fsmem));
    int sms = 0, per_sm = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, ffn, dev::kRowTile, fsmem));
    per_sm = std::max(per_sm, 1);

    dev::FilterParams FP{};
    FP.bits = d_bits;
    FP.bits2 = d_bits2;
    FP.sizes = rep->sizes;
    FP.maxham = d_maxham;
    FP.wstart = d_wstart;
    FP.item_base = d_item_base;
    FP.tile_col_lo = d_col_lo;
    FP.surv = d_surv;
    FP.rowcnt = d_rowcnt;
    FP.item_counts = d_item_counts;
    FP.ctl = d_ctl;
    FP.surv_cap = surv_cap;
    FP.ntiles = tlp->ntiles;
    FP.row_begin = static_cast<uint32_t>(plan.row_begin);
    FP.row_end = static_cast<uint32_t>(plan.row_end);
    FP.cutoff = enabled ? plan.bitmap.cutoff : kUnlimited;
    FP.words = W;
    FP.colsub = filter_colsub(W);
    FP.bypass_all = enabled ? 0 : 1;
    FP.naive = naive ? 1 : 0;

    dev::TcParams TP{};
    TcKernel tck{nullptr, 0};
    bool tc2_active = use_tc2;
    if (use_tc) {
        tck = use_tc2 ? tc2_select(W) : (use_tcm ? tcm_select(W) : tc_select(W, l2gemm, fp4, noext));
        set_smem_once(reinterpret_cast<const void*>(tck.fn), tck.smem);
        TP.opA = d_opA;
        TP.opB = d_opB;
        TP.bits = d_bits;
        TP.bits2 = d_bits2;
        TP.sizes = rep->sizes;
        TP.maxham = d_maxham;
        TP.maxham_len = static_cast<int>(maxham.size());
        TP.wstart = d_wstart;
        TP.item_base = d_item_base;
        TP.item_tile = d_item_tile;
        TP.item_order = item_ordered ? d_item_order : nullptr;
        TP.tile_col_lo = d_col_lo;
        TP.surv = d_surv;
        TP.rowcnt = d_rowcnt;
        TP.item_counts = d_item_counts;
        TP.tile_counts = d_tile_counts;
        TP.tiles_per_item = kTilesPerItem;
        TP.ctl = d_ctl;
        TP.surv_cap = surv_cap;
        TP.ntiles = tlp->ntiles;
        TP.row_begin = static_cast<uint32_t>(plan.row_begin);
        TP.row_end = static_cast<uint32_t>(plan.row_end);
        TP.cutoff = FP.cutoff;
        TP.neg1 = -1;
        TP.npc2 = noext ? sk->npc2 : nullptr;
        TP.debug = static_cast<int>(env_u64("SSJB_TC_DEBUG", 0));
        TP.bias = level1_acc_bias(W, variant);
        TP.bias2 = level2_acc_bias(W2, variant);
        TP.emit_col_end = head_active ? hplan.L0 : ~0u;
        if (TP.debug & 2) {
            TP.trace = A.alloc<unsigned long long>(2048 + 2 * 8192);
            CK(cudaMemsetAsync(TP.trace, 0, (2048 + 2 * 8192) * 8, s));
        }
        st.filter_kernel = l2gemm ? 2 : (fp4 ? 3 : 1);
    }

    dev::VerifyParams VP{};
    VP.tokens = rep->tokens;
    VP.offsets = rep->offsets;
    VP.need.minov = d_minov;
    VP.need.cosine = plan.cosine ? 1 : 0;
    VP.need.cp = plan.p;
    VP.need.cq = plan.q;
    VP.surv = d_surv;
    VP.res_keys = SB.ka;
    VP.res_ov = SB.va;
    VP.res_cap = res_cap;
    VP.ctl = d_ctl;
    VP.warp_mode = static_cast<int>(env_u64("SSJB_WARP_VERIFY", 1));
    if (W2 && !naive) {  // level-2 re-test of level-1 survivors before the merge
        VP.bits2 = d_bits2;
        VP.maxham = d_maxham;
        // (the level-2 GEMM emits level-2 survivors: no second test, which would
        // cost two random 32-byte sketch loads per survivor)
        VP.w2 = l2gemm ? 0 : W2;
    }
    // level 3 (512-bit Xor) for the dense regime's large records, built on demand
    auto enable_level3 = [&]() {
        if (VP.bits3 || W2 != 4 || naive || env_u64("SSJB_L3", 1) == 0) return;
        uint64_t* b3 = A.alloc<uint64_t>((n + kPadRows + 8) * 8);
        // (two-phase streaming: the rows still in flight are built by finish_ingest)
        launch_build_sub(*rep, b3, nullptr, Method::Xor, 512, 0, plan.bitmap.hash, s, st.launches, 0,
                         ingest_pending ? split_row : static_cast<uint32_t>(n));
        l3_bits = b3;
        VP.bits3 = b3;
        VP.maxham = d_maxham;
        VP.l3_min_sum = static_cast<uint32_t>(env_u64("SSJB_L3_MIN", 128));
    };
    // (tests: SSJB_L3_FORCE=1 enables level 3 from the first pass of any
    // non-streamed join with level-2 sketches)
    if (env_u64("SSJB_L3_FORCE", 0) != 0 && !streamed) enable_level3();

    std::vector<PairVec> runs;
    uint64_t res_count = 0;
    uint64_t resume_item = 0;  // first work item the batch phase still has to filter
    uint64_t fast_prefix = 0;  // items the first (soft-capped) pass filtered
    int idbits = 1;
    while ((uint64_t(1) << idbits) < n + 1) ++idbits;
    SB.count = &d_ctl->results;

    uint64_t counted = 0;  // matches in runs (every delivery mode)
    auto take_run = [&](const unsigned long long* keys, const uint32_t* ov, uint64_t count) {
        counted += count;
        if (plan.delivery == 1) return;
        PairVec run(count);
        for (uint64_t k = 0; k < count; ++k)
            run[k] = PairOut{static_cast<uint32_t>(keys[k] >> 32), static_cast<uint32_t>(keys[k] & 0xFFFFFFFFu),
                             static_cast<int64_t>(ov[k])};
        runs.push_back(std::move(run));
    };

    auto flush_results = [&](uint64_t count) {
        // K4 on the current result buffer, packed to ssj_pair records on the
        // device, then one (staged) download of the sorted run
        counted += count;
        if (plan.delivery == 1) {  // count only: nothing sorted or downloaded
            CK(cudaMemsetAsync(&d_ctl->results, 0, 8, s));
            return;
        }
        cudaEvent_t a = T.mark();
        bool inb = sort_results(SB, count, idbits, s, st.launches);
        if (plan.delivery == 2) {  // keep the sorted run in HBM for the streaming delivery
            cudaEvent_t b = T.mark();
            keep_device_run(out, device, s, inb ? SB.kb : SB.ka, inb ? SB.vb : SB.va, count, idbits);
            st.ms_sort += Timer::ms(a, b);
            CK(cudaMemsetAsync(&d_ctl->results, 0, 8, s));
            return;
        }
        cudaEvent_t b = T.mark();
        hmark("flush: sort enqueued");
        PairVec run(count);
        hmark("flush: result block");
        const bool direct = count && result_block_pinned(run.data(), count * sizeof(PairOut));
        d2h_pairs_staged(run.data(), inb ? SB.kb : SB.ka, inb ? SB.vb : SB.va, count, s,
                         direct ? A.alloc<PairOut>(count) : nullptr);
        cudaEvent_t d = T.mark();
        CK(cudaStreamSynchronize(s));
        st.d2h_bytes += count * (direct ? sizeof(PairOut) : 12);
        st.ms_sort += Timer::ms(a, b);
        st.ms_download += Timer::ms(b, d);
        hmark(direct ? "flush: downloaded (direct)" : "flush: downloaded (staged)");
        runs.push_back(std::move(run));
        CK(cudaMemsetAsync(&d_ctl->results, 0, 8, s));
    };

    uint64_t total_items = tlp->item_base.back();
    auto launch_filter = [&](uint64_t ib, uint64_t ie, uint32_t tb, bool keep_survivors = false,
                             bool zero_counts = true) {
        if (!keep_survivors) CK(cudaMemsetAsync(&d_ctl->survivors, 0, 8, s));
        CK(cudaMemsetAsync(&d_ctl->work_next, 0, 8, s));
        if (d_item_counts && ie > ib && zero_counts)
            CK(cudaMemsetAsync(d_item_counts + ib * tlp->tile_rows, 0, (ie - ib) * tlp->tile_rows * 4, s));
        if (ie <= ib) return;
        FP.item_begin = ib;
        FP.item_end = ie;
        FP.tile_begin = tb;
        if (use_tc) {
            TP.item_begin = ib;
            TP.item_end = ie;
            TP.tile_begin = tb;
            if (tc2_active) {
                // one CTA pair per TPC, the pair sharing each work item
                const uint64_t pairs = std::min<uint64_t>(ie - ib, static_cast<uint64_t>(sms / 2));
                tck.fn<<<static_cast<unsigned>(2 * pairs), tck.threads, tck.smem, s>>>(TP);
            } else {
                const uint64_t grid = std::min<uint64_t>(ie - ib, static_cast<uint64_t>(sms));
                tck.fn<<<static_cast<unsigned>(grid), tck.threads, tck.smem, s>>>(TP);
            }
        } else {
            const uint64_t grid = std::min<uint64_t>(ie - ib, static_cast<uint64_t>(sms) * per_sm);
            ffn<<<static_cast<unsigned>(grid), dev::kRowTile, fsmem, s>>>(FP);
        }
        ++st.launches;
        CK(cudaGetLastError());
    };
    auto launch_verify = [&](const unsigned long long* count_ptr = nullptr) {
        // survivor count read on the device: no host round trip between K2 and K3
        VP.count_ptr = count_ptr ? count_ptr : &d_ctl->survivors;
        VP.count_cap = surv_cap;
        static const unsigned vmul = static_cast<unsigned>(env_u64("SSJB_VERIFY_GRID", 32));  // latency-bound: more warps
        const unsigned vgrid = static_cast<unsigned>(sms) * vmul;
        if (VP.w2 == 4) dev::verify_pairs<4><<<vgrid, 256, 0, s>>>(VP);
        else if (VP.w2 == 8) dev::verify_pairs<8><<<vgrid, 256, 0, s>>>(VP);
        else dev::verify_pairs<0><<<vgrid, 256, 0, s>>>(VP);
        ++st.launches;
        CK(cudaGetLastError());
    };
    // K2b: the saturated-row rescan (on `rs`, default the join stream) and the
    // counter reduction (on the join stream; with reduce = false the caller
    // launches it later)
    auto launch_counters = [&](cudaStream_t rs = nullptr, bool rescan = true, bool reduce = true) {
        if (!rows) return;
        if (!rs) rs = s;
        if (!naive && rescan) {
            dev::RescanParams RP{};
            RP.bits = d_bits;
            RP.sizes = rep->sizes;
            RP.maxham = d_maxham;
            RP.maxham_len = static_cast<int>(maxham.size());
            RP.wstart = d_wstart;
            RP.rowcnt = d_rowcnt;
            RP.item_counts = d_item_counts;
            RP.tile_rows = tlp->tile_rows;
            RP.tile_counts = use_tc ? TP.tile_counts : nullptr;
            RP.tiles_per_item = kTilesPerItem;
            RP.tile_cols = static_cast<uint32_t>(tck.nt);
            RP.tile_parts = static_cast<uint32_t>(tck.parts);
            RP.item_base = d_item_base;
            RP.tile_col_lo = d_col_lo;
            RP.jstar = d_jstar;
            RP.row_begin = static_cast<uint32_t>(plan.row_begin);
            RP.row_end = static_cast<uint32_t>(plan.row_end);
            RP.capacity = plan.capacity;
            RP.cutoff = FP.cutoff;
            RP.words = W;
            RP.bypass_all = FP.bypass_all;
            RP.sat_list = d_satlist;
            RP.sat_count = &d_ctl->sat_rows;
            const unsigned gf = static_cast<unsigned>(std::min<uint64_t>((rows + 255) / 256, uint64_t(sms) * 8));
            dev::find_saturated<<<gf, 256, 0, rs>>>(d_rowcnt, rows, plan.capacity, d_satlist, d_ctl);
            const unsigned g = static_cast<unsigned>(std::min<uint64_t>((rows + 7) / 8, uint64_t(sms) * 8));
            dev::rescan_saturated<<<g, 256, 0, rs>>>(RP);
            st.launches += 2;
            CK(cudaGetLastError());
        }
        if (!reduce) return;
        dev::CountParams CP{};
        CP.sizes = rep->sizes;
        CP.wstart = d_wstart;
        CP.rowcnt = d_rowcnt;
        CP.jstar = d_jstar;
        CP.ctl = d_ctl;
        CP.row_begin = static_cast<uint32_t>(plan.row_begin);
        CP.row_end = static_cast<uint32_t>(plan.row_end);
        CP.capacity = plan.capacity;
        CP.bitmap_enabled = enabled ? 1 : 0;
        CP.naive = naive ? 1 : 0;
        const unsigned g = static_cast<unsigned>(std::min<uint64_t>((rows + 255) / 256, uint64_t(sms) * 4));
        dev::reduce_counters<<<g, 256, 0, s>>>(CP);
        ++st.launches;
        CK(cudaGetLastError());
    };

    // Fast path: the whole shard as one batch, K2 -> K3 -> K2b -> counters ->
    // K4 chained on the stream with a single host synchronisation.
    // Streamed ingest: per row chunk (as its tokens land) decode / widen, build
    // the sketches and expand the operands; with filter_chunks also launch the
    // chunk's filter work items.  Returns filter_chunks.
    auto stream_ingest = [&](bool filter_chunks, size_t k_begin = 0, size_t k_end = SIZE_MAX) {
            const int variant_s = variant;
            // per-chunk filter launches (SSJB_STREAM=2) overlap more of the transfer
            // but pay a launch tail per chunk; by default only the ingest kernels
            // (decode, sketches, operands) are chunked
            const bool stream_filter = filter_chunks;
            for (size_t k = k_begin; k < std::min(k_end, ingest.size()); ++k) {
                const IngestChunk& ch = ingest[k];
                CK(cudaStreamWaitEvent(s, ch.ev, 0));
                if (ingest_d8.bytes)
                    launch_decode(ingest_d8, rep->offsets, rep->tokens, ch.r0, ch.r1, s, st.launches,
                                  static_cast<double>(c.tokens.size()) / static_cast<double>(std::max<size_t>(n, 1)));
                if (ingest_t16 && ch.t1 > ch.t0) {
                    const uint64_t w0 = ch.t0 & ~uint64_t(3);  // 8-byte aligned vector loads
                    const uint64_t cnt = ch.t1 - w0;
                    widen_tokens<<<static_cast<unsigned>((cnt + 1023) / 1024), 256, 0, s>>>(ingest_t16 + w0,
                                                                                           rep->tokens + w0, cnt);
                    ++st.launches;
                    CK(cudaGetLastError());
                }
                launch_build_sub(*rep, sk->bits, sk->bits2, plan.bitmap.method, width, 64 * W2, plan.bitmap.hash, s,
                                 st.launches, ch.r0, ch.r1);
                const bool last = k + 1 == ingest.size();
                launch_expand(sk->bits, W, sk->bits2, W2, rep->sizes, d_opA, d_opB, last ? n_pad : ch.r1, variant_s,
                              s, st.launches, ch.r0);
                if (variant_s == 4)
                    launch_column_info(sk->bits, W, ch.r0, last ? n_pad : ch.r1, sk->npc2, s, st.launches);
                if (stream_filter) {  // filter work items of this chunk's row tiles
                    const uint32_t ta = ch.r0 / tlp->tile_rows;
                    const uint32_t tb2 = last ? tlp->ntiles : ch.r1 / tlp->tile_rows;
                    launch_filter(tlp->item_base[ta], tlp->item_base[tb2], ta, k > 0);
                }
            }
        return filter_chunks;
    };
    double ms_filter = 0, ms_verify = 0;
    bool done = false;
    const auto t_launch = Clock::now();  // host setup ends: the first filter launch
    auto t_synced = t_launch;
    // batch mode from the start: ingest only -- in two phases, the first chunk
    // now and the rest once the batches reach items outside it
    if (head_upfront && streamed) {
        if (two_phase && ingest.size() > 1 && ingest[0].r1 == split_row) {
            stream_ingest(false, 0, 1);
            ingest_pending = 1;
            phase_items = tlp->item_base[split_row / tlp->tile_rows];
        } else {
            stream_ingest(false);
        }
    }
    if (!head_upfront) {
        cudaEvent_t a = T.mark();
        if (streamed) {
            const bool stream_filter = stream_ingest(env_u64("SSJB_STREAM", 1) >= 2);
            if (!stream_filter) {
                FP.surv_soft = TP.surv_soft = std::max<uint64_t>(surv_cap / 2, 1);
                launch_filter(0, total_items, 0);  // one persistent launch after ingest
            }
        } else {
            // soft survivor cap: a join whose survivors would overflow the buffer
            // stops after an item prefix (kept, then continued in batches)
            FP.surv_soft = TP.surv_soft = std::max<uint64_t>(surv_cap / 2, 1);
            launch_filter(0, total_items, 0);
        }
        FP.surv_soft = TP.surv_soft = 0;
        cudaEvent_t b = T.mark();
        launch_verify();
        cudaEvent_t c1 = T.mark();
        launch_counters();
        cudaEvent_t r1 = T.mark();
        SmallPack* d_pack = A.alloc<SmallPack>(1);
        small_sort_pack<<<1, 1024, 0, s>>>(SB.ka, SB.va, d_ctl, d_pack);
        ++st.launches;
        CK(cudaGetLastError());
        cudaEvent_t so = T.mark();
        SmallPack* hp = host_small_pack();
        CK(cudaMemcpyAsync(hp, d_pack, sizeof(SmallPack), cudaMemcpyDeviceToHost, s));
        cudaEvent_t dl = T.mark();
        const auto t_enq = Clock::now();
        CK(cudaStreamSynchronize(s));
        t_synced = Clock::now();
        if (std::getenv("SSJB_HOST_TIMING"))
            std::fprintf(stderr, "[host] setup %.3f ms, enqueue %.3f ms\n",
                         std::chrono::duration<double, std::milli>(t_launch - t_start).count(),
                         std::chrono::duration<double, std::milli>(t_enq - t_launch).count());
        h_ctl = hp->ctl;
        const bool multi_launch = streamed && env_u64("SSJB_STREAM", 1) >= 2;
        const uint64_t fast_items = multi_launch ? total_items : std::min<uint64_t>(h_ctl.work_next, total_items);
        const bool partial = fast_items < total_items;
        fast_prefix = fast_items;
        const bool switch_l2 = l2_auto && use_tc && !l2gemm && !fp4;
        if (h_ctl.survivors <= surv_cap && partial && !switch_l2) {
            // soft-capped: the item prefix [0, fast_items) is filtered and its
            // survivors verified; keep its results and row/item counts, drop the
            // counters computed from partial rows (recomputed at the end), and
            // continue with the remaining items in batches
            ms_filter = Timer::ms(a, b);
            ms_verify = Timer::ms(b, c1);
            st.batches = 1;
            st.survivors = h_ctl.survivors;
            res_count = h_ctl.results;
            resume_item = fast_items;
            CK(cudaMemsetAsync(&d_ctl->tested, 0, 4 * sizeof(unsigned long long), s));
            CK(cudaMemsetAsync(&d_ctl->sat_rows, 0, sizeof(unsigned long long), s));
        } else if (h_ctl.survivors <= surv_cap && !partial) {
            done = true;
            ms_filter = Timer::ms(a, b);
            ms_verify = Timer::ms(b, c1);
            st.ms_rescan = Timer::ms(c1, r1);
            st.batches = 1;
            st.survivors = h_ctl.survivors;
            if (h_ctl.results <= kSmallSort) {
                st.ms_sort = Timer::ms(r1, so);
                st.ms_download = Timer::ms(so, dl);
                st.d2h_bytes += sizeof(SmallPack);
                take_run(hp->keys, hp->ov, h_ctl.results);
            } else {
                flush_results(h_ctl.results);
            }
        } else {
            // survivor buffer overflow, or a soft-capped level-1 pass that switches
            // to the level-2 GEMM: discard and redo in batches
            CK(cudaMemsetAsync(d_rowcnt, 0, (rows + 1) * 4ull, s));
            CK(cudaMemsetAsync(d_ctl, 0, sizeof(dev::Control), s));
            if (l2_auto && use_tc && !l2gemm && !fp4) {
                // level-1 survivors overflow: the b-bit sketch is saturated for this
                // collection, so re-test level 1 and level 2 together in the GEMM and
                // emit only level-2 survivors (operands built for this join only)
                const size_t rowb = operand_row(W, 1);
                uint8_t* a1 = A.alloc<uint8_t>(static_cast<size_t>(n_pad) * rowb);
                uint8_t* b1 = A.alloc<uint8_t>(static_cast<size_t>(n_pad) * rowb);
                launch_expand(sk->bits, W, sk->bits2, W2, rep->sizes, a1, b1, n_pad, 1, s, st.launches);
                l2gemm = true;
                if (tlp->tile_rows != dev::kRowTile) {
                    // the level-2 GEMM kernel takes 128-row work items
                    tc2_active = false;
                    set_tiling(dev::kRowTile);
                    total_items = n_items = tlp->item_base.back();
                    TP.item_base = d_item_base;
                    TP.item_tile = d_item_tile;
                    TP.item_order = item_ordered ? d_item_order : nullptr;
                    TP.tile_col_lo = d_col_lo;
                    TP.ntiles = tlp->ntiles;
                    if (d_item_counts && n_items * tlp->tile_rows * 4 <= ic_bytes) {
                        TP.item_counts = d_item_counts;  // same buffer, fewer/equal bytes
                    } else {
                        d_item_counts = nullptr;
                        TP.item_counts = nullptr;
                    }
                }
                tck = tc_select(W, true, false);
                set_smem_once(reinterpret_cast<const void*>(tck.fn), tck.smem);
                TP.opA = a1;
                TP.opB = b1;
                VP.w2 = 0;  // its survivors pass level 2 already
                TP.bias = level1_acc_bias(W, 1);  // the variant-1 operands' biases
                TP.bias2 = level2_acc_bias(W2, 1);
                st.filter_kernel = 2;
                head_active = hplan.ok;
                TP.emit_col_end = head_active ? hplan.L0 : ~0u;
            }
        }
    }

    auto finish_ingest = [&]() {
        if (ingest_pending) {
            stream_ingest(false, ingest_pending);
            if (l3_bits) launch_build_sub(*rep, l3_bits, nullptr, Method::Xor, 512, 0, plan.bitmap.hash, s, st.launches,
                                           split_row, static_cast<uint32_t>(n));
            ingest_pending = 0;
        }
        for (auto& ch : ingest) CK(cudaEventDestroy(ch.ev));
        ingest.clear();
        if (ingest_t16) CK(cudaFreeAsync(ingest_t16, s));
        ingest_t16 = nullptr;
        free_delta8(ingest_d8, s);
    };
    if (!ingest_pending) finish_ingest();

    if (!done) {
        // Survivor batches.  Grow the survivor / result buffers toward the first
        // pass's survivor count while HBM allows (8 + 24 bytes per entry), then
        // launch the filter over every remaining item with a soft survivor cap:
        // its producers stop claiming items once the cap is passed, so each
        // launch processes a prefix of the items, fills the buffer to about
        // the cap and never overflows it (only if the last claims overshoot
        // the margin is the launch rolled back and retried with a lower cap).
        {
            size_t fr = 0, tot = 0;
            cudaMemGetInfo(&fr, &tot);
            // survivors of the whole join, extrapolated from the first pass's prefix
            const double est = static_cast<double>(h_ctl.survivors) * static_cast<double>(total_items) /
                               static_cast<double>(std::max<uint64_t>(fast_prefix ? fast_prefix : total_items, 1));
            uint64_t want = surv_cap;
            while (static_cast<double>(want) < est && want < (uint64_t(1) << 30)) want <<= 1;
            const uint64_t limit = static_cast<uint64_t>(0.35 * static_cast<double>(fr)) / 32;
            while (want > surv_cap && want > limit) want >>= 1;
            if (want > surv_cap && env_u64("SSJB_SURVIVOR_CAP", 0) == 0 && env_u64("SSJB_RESULT_CAP", 0) == 0) {
                if (res_count) {  // the kept prefix's results leave the old buffer first
                    flush_results(res_count);
                    res_count = 0;
                }
                surv_cap = want;
                res_cap = std::max(res_cap, surv_cap);
                if (use_ws) CK(cudaStreamSynchronize(s));  // (regrown in place)
                d_surv = use_ws ? (WS.ensure(device, surv_cap, res_cap), WS.surv) : A.alloc<uint2>(surv_cap);
                alloc_results();
                FP.surv = d_surv;
                FP.surv_cap = surv_cap;
                TP.surv = d_surv;
                TP.surv_cap = surv_cap;
                VP.surv = d_surv;
                VP.res_keys = SB.ka;
                VP.res_ov = SB.va;
                VP.res_cap = res_cap;
            }
        }
        if (l2gemm) enable_level3();  // dense join: survivors in the billions, large records
        uint64_t soft = std::max<uint64_t>(surv_cap / 2, 1);
        uint64_t span = total_items;  // items per launch (halved only if the soft cap cannot help)
        uint64_t ib = resume_item;
        const bool ordered = use_tc && TP.item_order != nullptr;
        // the counts of the items a batch has not processed: claim positions [k0, total)
        auto zero_unprocessed = [&](uint64_t k0) {
            if (!d_item_counts || total_items <= k0) return;
            if (ordered) {
                const uint64_t cnt = (total_items - k0) * tlp->tile_rows;
                zero_item_counts<<<static_cast<unsigned>(std::min<uint64_t>((cnt + 255) / 256, uint64_t(sms) * 16)), 256,
                                   0, s>>>(TP.item_order, k0, total_items, d_item_counts, tlp->tile_rows);
                ++st.launches;
                CK(cudaGetLastError());
            } else {
                CK(cudaMemsetAsync(d_item_counts + k0 * tlp->tile_rows, 0, (total_items - k0) * tlp->tile_rows * 4, s));
            }
        };
        zero_unprocessed(ib);
        while (ib < total_items) {
            if (ingest_pending && ib >= phase_items) finish_ingest();
            const uint32_t tb = static_cast<uint32_t>(std::upper_bound(tlp->item_base.begin(), tlp->item_base.end(), ib) -
                                                      tlp->item_base.begin() - 1);
            const uint32_t rb = ordered ? 0u : tb * tlp->tile_rows;  // rows this launch may touch: [rb, rows)
            CK(cudaMemcpyAsync(d_rowsnap + rb, d_rowcnt + rb, (rows - rb) * 4ull, cudaMemcpyDeviceToDevice, s));
            FP.surv_soft = soft;
            TP.surv_soft = soft;
            cudaEvent_t a = T.mark();
            const uint64_t ie = std::min(ingest_pending ? phase_items : total_items, ib + span);
            launch_filter(ib, ie, tb, false, false);
            cudaEvent_t b = T.mark();
            CK(cudaMemcpyAsync(&h_ctl, d_ctl, sizeof(h_ctl), cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s));
            ms_filter += Timer::ms(a, b);
            const uint64_t S = h_ctl.survivors;
            const uint64_t processed = std::min<uint64_t>(h_ctl.work_next, ie - ib);
            if (S > surv_cap) {
                // the last claims overshot the margin: roll back this launch's
                // row and item counts, retry with a lower cap
                CK(cudaMemcpyAsync(d_rowcnt + rb, d_rowsnap + rb, (rows - rb) * 4ull, cudaMemcpyDeviceToDevice, s));
                zero_unprocessed(ib);
                if (soft > 1) soft = std::max<uint64_t>(soft / 4, 1);
                else span = std::max<uint64_t>(1, std::min(span, processed) / 2);  // kernels without the soft cap
                continue;
            }
            ++st.batches;
            st.survivors += S;
            if (S) {
                if (res_count + S > res_cap) {
                    flush_results(res_count);
                    res_count = 0;
                }
                cudaEvent_t c0 = T.mark();
                launch_verify();
                cudaEvent_t c1 = T.mark();
                CK(cudaMemcpyAsync(&h_ctl, d_ctl, sizeof(h_ctl), cudaMemcpyDeviceToHost, s));
                CK(cudaStreamSynchronize(s));
                ms_verify += Timer::ms(c0, c1);
                res_count = h_ctl.results;
            }
            ib += processed;
        }
        finish_ingest();  // (no-op unless every item fit the first phase)
        FP.surv_soft = 0;
        TP.surv_soft = 0;
        // with K3a to run, the saturated-row rescan (it reads only the filter's
        // row / item counts and the level-1 sketches) runs on a side stream
        // next to the head kernel; the counter reduction waits for it
        cudaStream_t side = nullptr;
        cudaEvent_t ev_side0 = nullptr, ev_side1 = nullptr;
        if (head_active && !naive && rows && env_u64("SSJB_RESCAN_SIDE", 1) != 0) {
            static thread_local cudaStream_t side_streams[16] = {};
            if (!side_streams[device & 15])
                CK(cudaStreamCreateWithFlags(&side_streams[device & 15], cudaStreamNonBlocking));
            side = side_streams[device & 15];
            CK(cudaEventCreate(&ev_side0));
            CK(cudaEventCreate(&ev_side1));
            CK(cudaEventRecord(ev_side0, s));
            CK(cudaStreamWaitEvent(side, ev_side0, 0));
            launch_counters(side, true, false);
            CK(cudaEventRecord(ev_side1, side));
        }
        if (head_active) {
            // K3a over the large-record region (K2 counted those pairs but did not
            // emit them): batches with a soft survivor cap, each verified by K3
            cudaEvent_t h0 = T.mark();
            const HeadDev hd = head_setup(*rep, c, hplan, A, s, sms, st.launches);
            hmark("head setup");
            dev::Control* d_hctl = A.alloc<dev::Control>(1);
            dev::HeadParams HP{};
            HP.op = hd.op;
            HP.base = hplan.base;
            HP.groups = hplan.rows_pad / 8;
            HP.kslices = hplan.row_bytes() / dev::kHeadSliceK;
            HP.info = hd.info;
            HP.minov = d_minov;
            HP.wstart = d_wstart;
            HP.items = hd.items;
            HP.tile_col_lo = hd.col_lo;
            HP.tile0 = hplan.tile0;
            HP.L0 = hplan.L0;
            HP.row_begin = static_cast<uint32_t>(plan.row_begin);
            HP.row_end = static_cast<uint32_t>(plan.row_end);
            HP.surv = d_surv;
            HP.surv_cap = surv_cap;
            HP.ctl = d_hctl;
            using HL8 = dev::HeadLayout<dev::kKindI8>;
            using HL4 = dev::HeadLayout<dev::kKindF4>;
            const bool hf4 = hplan.kind == dev::kKindF4;
            const void* hfn = hf4 ? reinterpret_cast<const void*>(dev::head_overlap_kernel<dev::kKindF4>)
                                  : reinterpret_cast<const void*>(dev::head_overlap_kernel<dev::kKindI8>);
            set_smem_once(hfn, hf4 ? HL4::kSmem : HL8::kSmem);
            cudaEvent_t h1 = T.mark();
            const uint64_t hitems = hplan.items.size();
            uint64_t hsoft = std::max<uint64_t>(surv_cap / 2, 1);
            uint64_t hspan = hitems;  // items per launch: halved when even a soft cap of 1 overshoots
            uint64_t hb = 0;
            dev::Control hc{};
            while (hb < hitems) {
                CK(cudaMemsetAsync(d_hctl, 0, sizeof(dev::Control), s));
                const uint64_t he = std::min(hitems, hb + hspan);
                HP.item_begin = hb;
                HP.item_end = he;
                HP.surv_soft = hsoft;
                cudaEvent_t a = T.mark();
                const unsigned hgrid = static_cast<unsigned>(std::min<uint64_t>(he - hb, sms));
                if (hf4) dev::head_overlap_kernel<dev::kKindF4><<<hgrid, HL4::kThreads, HL4::kSmem, s>>>(HP);
                else dev::head_overlap_kernel<dev::kKindI8><<<hgrid, HL8::kThreads, HL8::kSmem, s>>>(HP);
                ++st.launches;
                CK(cudaGetLastError());
                cudaEvent_t b = T.mark();
                CK(cudaMemcpyAsync(&hc, d_hctl, sizeof(hc), cudaMemcpyDeviceToHost, s));
                CK(cudaStreamSynchronize(s));
                st.ms_head += Timer::ms(a, b);
#ifdef SSJB_HEAD_PROBE
                std::fprintf(stderr, "head probe: candidates %llu\n", static_cast<unsigned long long>(hc.verify_bytes));
#endif
                const uint64_t S = hc.survivors;
                const uint64_t processed = std::min<uint64_t>(hc.work_next, he - hb);
                if (S > surv_cap) {  // overshoot: nothing was counted; redo with a lower cap / fewer items
                    if (hsoft > 1) hsoft = std::max<uint64_t>(hsoft / 4, 1);
                    else hspan = std::max<uint64_t>(1, std::min(hspan, std::max<uint64_t>(processed, 2)) / 2);
                    continue;
                }
                st.head_survivors += S;
                ++st.batches;
                if (S) {
                    if (res_count + S > res_cap) {
                        flush_results(res_count);
                        res_count = 0;
                    }
                    cudaEvent_t c0 = T.mark();
                    // (one warp per pair, SSJB_HEAD_WARP_VERIFY=1, measured slower on
                    // C4: 32.9 vs 14.1 ms -- the lanes' binary searches miss L2)
                    const int wm = VP.warp_mode;
                    if (env_u64("SSJB_HEAD_WARP_VERIFY", 0) != 0 && wm) VP.warp_mode = 2;
                    launch_verify(&d_hctl->survivors);
                    VP.warp_mode = wm;
                    cudaEvent_t c1 = T.mark();
                    CK(cudaMemcpyAsync(&h_ctl, d_ctl, sizeof(h_ctl), cudaMemcpyDeviceToHost, s));
                    CK(cudaStreamSynchronize(s));
                    ms_verify += Timer::ms(c0, c1);
                    res_count = h_ctl.results;
                }
                hb += processed;
            }
            CK(cudaStreamSynchronize(s));
            st.ms_head_setup += Timer::ms(h0, h1);
            st.head_pairs = hplan.pairs;
            st.head_k = hplan.K;
        }
        cudaEvent_t r0 = T.mark();
        if (side) {
            CK(cudaStreamWaitEvent(s, ev_side1, 0));
            launch_counters(s, false, true);
        } else {
            launch_counters();
        }
        cudaEvent_t r1 = T.mark();
        CK(cudaMemcpyAsync(&h_ctl, d_ctl, sizeof(h_ctl), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        st.ms_rescan = Timer::ms(r0, r1);
        if (side) {
            float side_ms = 0;
            CK(cudaEventElapsedTime(&side_ms, ev_side0, ev_side1));
            st.ms_rescan += side_ms;  // (overlapped with K3a)
            CK(cudaEventDestroy(ev_side0));
            CK(cudaEventDestroy(ev_side1));
        }
        flush_results(res_count);
    }

    hmark("results downloaded");
    // merge sorted runs (one run unless the result buffer overflowed)
    if (runs.size() == 1) {
        out.pairs = std::move(runs[0]);
    } else if (!runs.empty()) {
        PairVec merged;
        for (auto& r : runs) {
            PairVec tmp(merged.size() + r.size());
            std::merge(merged.begin(), merged.end(), r.begin(), r.end(), tmp.begin(),
                       [](const PairOut& x, const PairOut& y) {
                           return x.id_r != y.id_r ? x.id_r < y.id_r : x.id_s < y.id_s;
                       });
            merged.swap(tmp);
        }
        out.pairs = std::move(merged);
    }

    if (use_tc && TP.trace) {
        std::vector<unsigned long long> tr(2048 + 2 * 8192);
        CK(cudaMemcpy(tr.data(), TP.trace, tr.size() * 8, cudaMemcpyDeviceToHost));
        if (FILE* f = std::fopen("gpurun_out/tc_trace.txt", "a")) {
            for (int k = 0; k < 512; ++k) {
                std::fprintf(f, "%d %llu %llu %llu", k, tr[k * 4], tr[k * 4 + 1], tr[k * 4 + 2]);
                for (int w = 0; w < 16; ++w) std::fprintf(f, " %llu", tr[2048 + k * 16 + w]);
                for (int w = 0; w < 16; ++w) std::fprintf(f, " %llu", tr[2048 + 8192 + k * 16 + w]);
                std::fprintf(f, "\n");
            }
            std::fprintf(f, "---\n");
            std::fclose(f);
        }
    }
    out.candidates = plan.window_pairs;
    out.bitmap_tested = h_ctl.tested;
    out.pruned_bitmap = h_ctl.pruned;
    out.verified = h_ctl.verified;
    out.saturated = h_ctl.saturated;
    st.verify_bytes = h_ctl.verify_bytes;
    out.matched = counted;
    st.ms_upload = Timer::ms(e0, e_up);
    st.ms_build = Timer::ms(e_up, e_build);
    st.ms_filter = ms_filter;
    st.ms_verify = ms_verify;
    out.index_s = (st.ms_upload + st.ms_build) * 1e-3;
    out.candidates_s = (st.ms_filter + st.ms_rescan) * 1e-3;
    const double total = std::chrono::duration<double>(Clock::now() - t_start).count();
    if (std::getenv("SSJB_HOST_TIMING"))
        std::fprintf(stderr, "[host] after sync %.3f ms, total %.3f ms\n",
                     std::chrono::duration<double, std::milli>(Clock::now() - t_synced).count(), total * 1e3);
    out.verify_s = std::max(0.0, total - out.index_s - out.candidates_s);
    if (host_trace) {
        auto prev = t_start;
        for (auto& m : hmarks) {
            std::fprintf(stderr, "[host] %-24s +%8.3f ms (at %8.3f)\n", m.first,
                         std::chrono::duration<double, std::milli>(m.second - prev).count(),
                         std::chrono::duration<double, std::milli>(m.second - t_start).count());
            prev = m.second;
        }
        std::fprintf(stderr, "[host] engine total %.3f ms (+ %.3f ms device/stream setup before it)\n", total * 1e3,
                     std::chrono::duration<double, std::milli>(t_start - t_enter).count());
    }
}

// NAIVE RS-join block on one GPU: R rows [r_begin, r_end) x all of S
// (reference src/join.cpp:110-121).  No filter: launches of verify_rs over
// contiguous ranges of the row-major pair index, each sized so its matches
// fit the result buffer; every launch's matches are sorted (K4) and
// downloaded as one run, and consecutive runs are already in (id_r, id_s)
// order, so they concatenate.  Overflowing launches are redone smaller.
void engine_join_rs(const Collection& R, const Collection& Sc, const RsPlan& plan, int device, EngineResult& out) {
    using Clock = std::chrono::steady_clock;
    set_device(device);
    static thread_local cudaStream_t streams[16] = {};
    if (!streams[device & 15]) CK(cudaStreamCreateWithFlags(&streams[device & 15], cudaStreamNonBlocking));
    cudaStream_t s = streams[device & 15];
    EngineStats& st = out.stats;
    const auto t_start = Clock::now();
    Timer T(s);
    Arena A(s);
    const uint64_t nS = Sc.size();
    const uint64_t rows = plan.r_end - plan.r_begin;
    const uint64_t total = rows * nS;
    st.window_pairs = total;
    out.candidates = out.verified = total;
    if (total == 0) return;

    cudaEvent_t e0 = T.mark();
    auto repR = replica_for(R, device, s, st.h2d_bytes, st.launches);
    auto repS = &R == &Sc ? repR : replica_for(Sc, device, s, st.h2d_bytes, st.launches);
    TableStage stage;
    int32_t* d_minov = nullptr;
    stage.add(&d_minov, plan.minov.data(), plan.minov.size() * 4);
    stage.flush(A, s, st.h2d_bytes);
    cudaEvent_t e_up = T.mark();

    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
    const uint64_t res_cap = std::max<uint64_t>(env_u64("SSJB_RESULT_CAP", uint64_t(1) << 26), 1024);
    dev::Control* d_ctl = A.alloc<dev::Control>(1);
    SortBufs SB{};
    SB.ka = A.alloc<unsigned long long>(res_cap);
    SB.va = A.alloc<uint32_t>(res_cap);
    SB.kb = A.alloc<unsigned long long>(res_cap);
    SB.vb = A.alloc<uint32_t>(res_cap);
    const uint32_t max_tiles = static_cast<uint32_t>((res_cap + dev::kSortTile - 1) / dev::kSortTile);
    SB.hist = A.alloc<uint32_t>(256ull * max_tiles);
    SB.sums = A.alloc<uint32_t>((256ull * max_tiles + dev::kScanBlock - 1) / dev::kScanBlock + 1);
    SB.count = &d_ctl->results;
    CK(cudaMemsetAsync(d_ctl, 0, sizeof(dev::Control), s));
    int idbits = 1;
    while ((uint64_t(1) << idbits) < std::max<uint64_t>(R.size(), nS) + 1) ++idbits;

    dev::VerifyRsParams VP{};
    VP.ta = repR->tokens;
    VP.oa = repR->offsets;
    VP.tb = repS->tokens;
    VP.ob = repS->offsets;
    VP.nS = nS;
    VP.r_begin = plan.r_begin;
    VP.need.minov = d_minov;
    VP.need.cosine = plan.cosine ? 1 : 0;
    VP.need.cp = plan.p;
    VP.need.cq = plan.q;
    VP.res_keys = SB.ka;
    VP.res_ov = SB.va;
    VP.res_cap = res_cap;
    VP.ctl = d_ctl;

    std::vector<PairVec> runs;
    uint64_t counted = 0;
    SB.count_store = A.alloc<unsigned long long>(1);
    uint64_t k0 = 0;
    uint64_t batch = std::min<uint64_t>(total, env_u64("SSJB_RS_BATCH", uint64_t(1) << 32));
    double ms_verify = 0;
    dev::Control h_ctl{};
    uint64_t verify_bytes = 0;
    // Filtered path (round 2): length window + Xor-sketch bound on R x S tiles,
    // then exact verification of the survivors only.  Sound for every
    // similarity function whose required overlap depends on |r|+|s| (not
    // Cosine); NAIVE's counters are unchanged (candidates = verified = |R||S|).
    // SSJB_RS_FILTER: 0 off, 1 auto (|R||S| >= 2^24), 2 forced.
    const uint64_t rs_mode = env_u64("SSJB_RS_FILTER", 1);
    const bool filtered = !plan.cosine && rs_mode != 0 && (rs_mode == 2 || total >= (uint64_t(1) << 24)) &&
                          plan.delivery != 2 && R.max_size < (uint32_t(1) << 30);
    if (filtered) {
        const int words = std::max(R.median_size(), Sc.median_size()) > 64 ? 2 : 1;
        const uint32_t nR = static_cast<uint32_t>(R.size()), nS32 = static_cast<uint32_t>(nS);
        uint64_t* bits_r = A.alloc<uint64_t>((size_t(nR) + kPadRows + 8) * words);
        uint64_t* bits_s = &R == &Sc ? bits_r : A.alloc<uint64_t>((size_t(nS32) + kPadRows + 8) * words);
        if (!launch_build_sub(*repR, bits_r, nullptr, Method::Xor, 64 * words, 0, 0, s, st.launches))
            launch_build(*repR, bits_r, Method::Xor, 64 * words, 0, s, st.launches);
        if (bits_s != bits_r && !launch_build_sub(*repS, bits_s, nullptr, Method::Xor, 64 * words, 0, 0, s, st.launches))
            launch_build(*repS, bits_s, Method::Xor, 64 * words, 0, s, st.launches);
        // per R size x: the S index window of sizes y with minov[x+y] <= min(x, y)
        // (an overlap never exceeds the smaller record; minov steps by <= 1, so
        // the admissible y form one interval)
        const uint32_t mr = R.max_size, ms = Sc.max_size;
        std::vector<uint32_t> lo(mr + 1), hi(mr + 1);
        auto ok = [&](uint32_t x, uint32_t y) { return plan.minov[x + y] <= static_cast<int32_t>(std::min(x, y)); };
        for (uint32_t x = 0; x <= mr; ++x) {
            const uint32_t ym = std::min(x, ms);
            lo[x] = hi[x] = nS32;
            if (!ok(x, ym)) continue;  // no admissible size
            // y <= x: y - minov[x+y] is nondecreasing -> first admissible y by bisection
            uint32_t a = 0, b = ym;
            while (a < b) {
                const uint32_t m = (a + b) / 2;
                if (ok(x, m)) b = m;
                else a = m + 1;
            }
            const uint32_t ylo = a;
            // y >= x: minov[x+y] <= x holds on a prefix of [x, ms]
            uint32_t yhi = ms;
            if (x < ms) {
                a = x;
                b = ms;
                while (a < b) {
                    const uint32_t m = (a + b + 1) / 2;
                    if (ok(x, m)) a = m;
                    else b = m - 1;
                }
                yhi = a;
            }
            lo[x] = Sc.first_ge[ylo];
            hi[x] = std::max(lo[x], Sc.first_ge[yhi + 1]);
        }
        std::vector<int32_t> maxham(plan.minov.size());
        for (size_t S = 0; S < maxham.size(); ++S) maxham[S] = static_cast<int32_t>(S) - 2 * plan.minov[S];
        // work items: (R row tile, S column chunk) over each tile's window union
        std::vector<uint2> items;
        const uint32_t ntiles = static_cast<uint32_t>((rows + dev::kRowTile - 1) / dev::kRowTile);
        for (uint32_t t = 0; t < ntiles; ++t) {
            const size_t a = plan.r_begin + size_t(t) * dev::kRowTile;
            const size_t b = std::min<size_t>(a + dev::kRowTile, plan.r_end);
            uint32_t wlo = nS32, whi = 0;  // union of the rows' windows (empty ones excluded)
            for (size_t r = a; r < b; ++r) {
                const uint32_t x = R.rec_size(r);
                if (hi[x] > lo[x]) {
                    wlo = std::min(wlo, lo[x]);
                    whi = std::max(whi, hi[x]);
                }
            }
            if (whi <= wlo) continue;
            for (uint32_t cc = wlo / dev::kColChunk; cc <= (whi - 1) / dev::kColChunk; ++cc) items.push_back(make_uint2(t, cc));
        }
        uint32_t *d_lo = nullptr, *d_hi = nullptr;
        int32_t* d_maxham = nullptr;
        uint2* d_items = nullptr;
        TableStage fs;
        fs.add(&d_lo, lo.data(), lo.size() * 4);
        fs.add(&d_hi, hi.data(), hi.size() * 4);
        fs.add(&d_maxham, maxham.data(), maxham.size() * 4);
        if (!items.empty()) fs.add(&d_items, items.data(), items.size() * sizeof(uint2));
        fs.flush(A, s, st.h2d_bytes);
        const uint64_t surv_cap = std::max<uint64_t>(env_u64("SSJB_SURVIVOR_CAP", uint64_t(1) << 26), 1u << 20);
        uint2* d_surv = A.alloc<uint2>(surv_cap);
        dev::RsFilterParams FP{};
        FP.bits_r = bits_r;
        FP.bits_s = bits_s;
        FP.sizes_r = repR->sizes;
        FP.sizes_s = repS->sizes;
        FP.s_lo = d_lo;
        FP.s_hi = d_hi;
        FP.maxham = d_maxham;
        FP.items = d_items;
        FP.r_begin = static_cast<uint32_t>(plan.r_begin);
        FP.r_end = static_cast<uint32_t>(plan.r_end);
        FP.n_s = nS32;
        FP.words = words;
        FP.surv = d_surv;
        FP.surv_cap = surv_cap;
        FP.ctl = d_ctl;
        dev::VerifyRsPairsParams RP{};
        RP.ta = repR->tokens;
        RP.oa = repR->offsets;
        RP.tb = repS->tokens;
        RP.ob = repS->offsets;
        RP.need = VP.need;
        RP.surv = d_surv;
        RP.count_ptr = &d_ctl->survivors;
        RP.count_cap = surv_cap;
        RP.res_keys = SB.ka;
        RP.res_ov = SB.va;
        RP.res_cap = res_cap;
        RP.ctl = d_ctl;
        uint64_t res_count = 0, survivors = 0;
        auto flush = [&]() {  // sort + pack + download the result buffer as one run
            if (!res_count) return;
            const bool inb = sort_results(SB, res_count, idbits, s, st.launches);
            PairOut* packed = A.alloc<PairOut>(res_count);
            pack_pairs<<<static_cast<unsigned>((res_count + 255) / 256), 256, 0, s>>>(
                inb ? SB.kb : SB.ka, inb ? SB.vb : SB.va, packed, res_count);
            ++st.launches;
            CK(cudaGetLastError());
            counted += res_count;
            if (plan.delivery == 0) {
                PairVec run(res_count);
                d2h_staged(run.data(), packed, res_count * sizeof(PairOut), s);
                st.d2h_bytes += res_count * sizeof(PairOut);
                runs.push_back(std::move(run));
            }
            CK(cudaStreamSynchronize(s));
            CK(cudaMemsetAsync(&d_ctl->results, 0, 8, s));
            res_count = 0;
        };
        uint64_t soft = std::max<uint64_t>(surv_cap / 2, 1), span = items.size(), ib = 0;
        const uint64_t nitems = items.size();
        int per_sm = 0;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, dev::rs_filter, dev::kRowTile, 0));
        while (ib < nitems) {
            const uint64_t ie = std::min(nitems, ib + span);
            CK(cudaMemsetAsync(&d_ctl->survivors, 0, 8, s));
            CK(cudaMemsetAsync(&d_ctl->work_next, 0, 8, s));
            FP.item_begin = ib;
            FP.item_end = ie;
            FP.surv_soft = soft;
            cudaEvent_t a = T.mark();
            dev::rs_filter<<<static_cast<unsigned>(std::min<uint64_t>(ie - ib, uint64_t(sms) * std::max(per_sm, 1))),
                             dev::kRowTile, 0, s>>>(FP);
            ++st.launches;
            CK(cudaGetLastError());
            cudaEvent_t b = T.mark();
            CK(cudaMemcpyAsync(&h_ctl, d_ctl, sizeof(h_ctl), cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s));
            st.ms_filter += Timer::ms(a, b);
            const uint64_t S = h_ctl.survivors;
            const uint64_t processed = std::min<uint64_t>(h_ctl.work_next, ie - ib);
            if (S > surv_cap) {  // overshoot: nothing counted yet, retry with a lower cap / fewer items
                if (soft > 1) soft = std::max<uint64_t>(soft / 4, 1);
                else span = std::max<uint64_t>(1, std::min(span, std::max<uint64_t>(processed, 2)) / 2);
                continue;
            }
            ++st.batches;
            survivors += S;
            if (S) {
                if (res_count + S > res_cap) flush();
                cudaEvent_t c0 = T.mark();
                dev::verify_rs_pairs<<<static_cast<unsigned>(std::min<uint64_t>((S + 255) / 256, uint64_t(sms) * 16)),
                                       256, 0, s>>>(RP);
                ++st.launches;
                CK(cudaGetLastError());
                cudaEvent_t c1 = T.mark();
                CK(cudaMemcpyAsync(&h_ctl, d_ctl, sizeof(h_ctl), cudaMemcpyDeviceToHost, s));
                CK(cudaStreamSynchronize(s));
                ms_verify += Timer::ms(c0, c1);
                if (h_ctl.results > res_cap) throw DeviceError("RS result buffer overflow");
                res_count = h_ctl.results;
            }
            ib += processed;
        }
        flush();
        verify_bytes = h_ctl.verify_bytes;
        st.survivors = survivors;
        // runs are each sorted; batches follow the item order, which a row tile's
        // chunks may straddle: merge
        PairVec merged;
        for (auto& r : runs) {
            if (merged.empty()) {
                merged = std::move(r);
                continue;
            }
            PairVec tmp(merged.size() + r.size());
            std::merge(merged.begin(), merged.end(), r.begin(), r.end(), tmp.begin(),
                       [](const PairOut& x, const PairOut& y) {
                           return x.id_r != y.id_r ? x.id_r < y.id_r : x.id_s < y.id_s;
                       });
            merged.swap(tmp);
        }
        out.pairs = std::move(merged);
        out.matched = counted;
        st.verify_bytes = verify_bytes;
        st.ms_upload = Timer::ms(e0, e_up);
        st.ms_verify = ms_verify;
        out.index_s = 0;
        out.candidates_s = 0;
        out.verify_s = std::chrono::duration<double>(Clock::now() - t_start).count();
        return;
    }
    while (k0 < total) {
        const uint64_t k1 = std::min(total, k0 + std::max<uint64_t>(batch, 1));
        CK(cudaMemsetAsync(d_ctl, 0, sizeof(dev::Control), s));
        VP.k0 = k0;
        VP.k1 = k1;
        const uint64_t blocks = std::min<uint64_t>((k1 - k0 + 255) / 256, uint64_t(sms) * 16);
        cudaEvent_t a = T.mark();
        dev::verify_rs<<<static_cast<unsigned>(blocks), 256, 0, s>>>(VP);
        ++st.launches;
        CK(cudaGetLastError());
        cudaEvent_t b = T.mark();
        CK(cudaMemcpyAsync(&h_ctl, d_ctl, sizeof(h_ctl), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        ms_verify += Timer::ms(a, b);
        const uint64_t cnt = h_ctl.results;
        if (cnt > res_cap) {  // matches overflowed the buffer: redo a smaller range
            batch = std::max<uint64_t>(1, (k1 - k0) * res_cap / cnt * 7 / 10);
            continue;
        }
        verify_bytes += h_ctl.verify_bytes;
        ++st.batches;
        counted += cnt;
        if (cnt && plan.delivery == 2) {
            cudaEvent_t c0 = T.mark();
            const bool inb = sort_results(SB, cnt, idbits, s, st.launches);
            cudaEvent_t c1 = T.mark();
            keep_device_run(out, device, s, inb ? SB.kb : SB.ka, inb ? SB.vb : SB.va, cnt, idbits);
            st.ms_sort += Timer::ms(c0, c1);
        } else if (cnt && plan.delivery == 0) {
            cudaEvent_t c0 = T.mark();
            const bool inb = sort_results(SB, cnt, idbits, s, st.launches);
            PairOut* packed = A.alloc<PairOut>(cnt);
            pack_pairs<<<static_cast<unsigned>((cnt + 255) / 256), 256, 0, s>>>(inb ? SB.kb : SB.ka,
                                                                              inb ? SB.vb : SB.va, packed, cnt);
            ++st.launches;
            CK(cudaGetLastError());
            cudaEvent_t c1 = T.mark();
            PairVec run(cnt);
            d2h_staged(run.data(), packed, cnt * sizeof(PairOut), s);
            cudaEvent_t c2 = T.mark();
            CK(cudaStreamSynchronize(s));
            st.d2h_bytes += cnt * sizeof(PairOut);
            st.ms_sort += Timer::ms(c0, c1);
            st.ms_download += Timer::ms(c1, c2);
            runs.push_back(std::move(run));
        }
        k0 = k1;
    }
    size_t n_out = 0;
    for (auto& r : runs) n_out += r.size();
    if (runs.size() == 1) {
        out.pairs = std::move(runs[0]);
    } else if (n_out) {
        out.pairs.resize(n_out);
        size_t at = 0;
        for (auto& r : runs) {
            std::memcpy(out.pairs.data() + at, r.data(), r.size() * sizeof(PairOut));
            at += r.size();
        }
    }
    out.matched = counted;
    st.survivors = total;
    st.verify_bytes = verify_bytes;
    st.ms_upload = Timer::ms(e0, e_up);
    st.ms_verify = ms_verify;
    out.index_s = 0;
    out.candidates_s = 0;
    out.verify_s = std::chrono::duration<double>(Clock::now() - t_start).count();
}


// ---------------------------------------------------------------------------
// Prefix-filter joins: ALLPAIRS / PPJOIN / PPJOIN+ (reference
// framework_join, src/join.cpp:132-189), GROUPJOIN (:197-329) and ADAPTJOIN
// (:331-420) on the GPU with the reference's counters; kernels in
// prefix_join.cuh.
namespace {

// In-place exclusive scan of d[0..n) (u64).
void scan_u64(unsigned long long* d, uint64_t n, Arena& A, cudaStream_t s, uint64_t& launches) {
    if (n == 0) return;
    const uint64_t tiles = (n + dev::kScan64Tile - 1) / dev::kScan64Tile;
    unsigned long long* sums = A.alloc<unsigned long long>(tiles + 1);
    dev::scan64_tiles<<<static_cast<unsigned>(tiles), dev::kScan64Threads, 0, s>>>(d, n, sums);
    ++launches;
    CK(cudaGetLastError());
    if (tiles > 1) {
        scan_u64(sums, tiles, A, s, launches);
        dev::scan64_add<<<static_cast<unsigned>((n + 255) / 256), 256, 0, s>>>(d, n, sums);
        ++launches;
        CK(cudaGetLastError());
    }
}

uint64_t read_u64(const unsigned long long* d, cudaStream_t s) {
    unsigned long long h = 0;
    CK(cudaMemcpyAsync(&h, d, 8, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    return h;
}

unsigned grid_for(uint64_t work, int sms, unsigned per_sm) {
    return static_cast<unsigned>(std::max<uint64_t>(1, std::min<uint64_t>((work + 255) / 256, uint64_t(sms) * per_sm)));
}

}  // namespace

void engine_prefix_join(const Collection& c, const Options& o, int device, EngineResult& out) {
    using Clock = std::chrono::steady_clock;
    set_device(device);
    static thread_local cudaStream_t streams[16] = {};
    if (!streams[device & 15]) CK(cudaStreamCreateWithFlags(&streams[device & 15], cudaStreamNonBlocking));
    cudaStream_t s = streams[device & 15];
    EngineStats& st = out.stats;
    const auto t_start = Clock::now();
    const uint64_t n = c.size();
    if (n < 2) {
        out.index_s = out.candidates_s = out.verify_s = 0;
        return;
    }
    const bool group = o.algorithm == Algo::GroupJoin;
    const bool adapt = o.algorithm == Algo::AdaptJoin;
    const int L = adapt ? std::max(1, o.ell_max) : 1;  // index / tally prefix extension
    if (L > dev::kAdaptMaxEll)
        throw std::invalid_argument("ell_max above " + std::to_string(dev::kAdaptMaxEll) + " is not supported");
    Timer T(s);
    Arena A(s);
    cudaEvent_t e0 = T.mark();
    auto rep = replica_for(c, device, s, st.h2d_bytes, st.launches);

    // host tables over record sizes (exact, reference src/similarity.cpp)
    const uint32_t ms = c.max_size, ms1 = ms + 1;
    std::vector<int32_t> plen_ell(static_cast<size_t>(L) * ms1), ellcap(ms1, 1);
    std::vector<uint32_t> lower(ms1), upper(ms1);
    for (uint32_t z = 0; z <= ms; ++z) {
        for (int l = 1; l <= L; ++l)
            plen_ell[static_cast<size_t>(l - 1) * ms1 + z] = static_cast<int32_t>(prefix_length(o.sim, o.threshold, z, l));
        const LengthWindow w = length_window(o.sim, o.threshold, z);
        lower[z] = static_cast<uint32_t>(std::min<int64_t>(w.lower, UINT32_MAX));
        upper[z] = static_cast<uint32_t>(std::min<int64_t>(w.upper, UINT32_MAX));
        if (adapt) {
            const int64_t need = required_overlap(o.sim, o.threshold, z, std::max<int64_t>(w.lower, 0));
            ellcap[z] = static_cast<int32_t>(std::max<int64_t>(1, std::min<int64_t>(L, need)));
        }
    }
    std::vector<int32_t> minov = minov_table(o.sim, o.threshold, 2 * static_cast<size_t>(ms));
    int32_t *d_plen = nullptr, *d_minov = nullptr, *d_ellcap = nullptr;
    uint32_t *d_lower = nullptr, *d_upper = nullptr;
    TableStage stage;
    stage.add(&d_plen, plen_ell.data(), plen_ell.size() * 4);
    stage.add(&d_minov, minov.data(), minov.size() * 4);
    stage.add(&d_lower, lower.data(), lower.size() * 4);
    stage.add(&d_upper, upper.data(), upper.size() * 4);
    stage.add(&d_ellcap, ellcap.data(), ellcap.size() * 4);
    stage.flush(A, s, st.h2d_bytes);
    // the index holds ell = L prefixes; framework / group probes use ell = 1
    const int32_t* d_plen_index = d_plen + static_cast<size_t>(L - 1) * ms1;

    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));

    // sketches (src/join.cpp:139-140: every record, the resolved config)
    const ResolvedBitmap rb = resolve_bitmap(c, o);
    uint64_t* bits = nullptr;
    const int W = rb.width / 64;
    if (rb.enabled) {
        bits = A.alloc<uint64_t>((n + kPadRows) * W);
        if (!launch_build_sub(*rep, bits, nullptr, rb.method, rb.width, 0, rb.hash, s, st.launches))
            launch_build(*rep, bits, rb.method, rb.width, rb.hash, s, st.launches);
    }
    const bool f2 = !group && !adapt && rb.enabled && o.placement == 1;
    const bool f3 = !group && !adapt && rb.enabled && !f2;

    // GroupJoin groups: runs of equal (size, full prefix) (src/join.cpp:205-219)
    uint32_t* grp_begin = nullptr;
    uint64_t U = n;
    if (group) {
        unsigned long long* flag = A.alloc<unsigned long long>(n + 1);
        CK(cudaMemsetAsync(flag + n, 0, 8, s));
        dev::group_flags<<<static_cast<unsigned>((n + 255) / 256), 256, 0, s>>>(rep->tokens, rep->offsets, rep->sizes,
                                                                              d_plen, static_cast<uint32_t>(n), flag);
        ++st.launches;
        CK(cudaGetLastError());
        scan_u64(flag, n + 1, A, s, st.launches);
        U = read_u64(flag + n, s);
        grp_begin = A.alloc<uint32_t>(U + 1);
        dev::group_begins<<<static_cast<unsigned>((n + 255) / 256), 256, 0, s>>>(flag, static_cast<uint32_t>(n),
                                                                               grp_begin, rep->sizes, nullptr);
        ++st.launches;
        CK(cudaGetLastError());
    }

    // inverted prefix index: postings (token << 32 | id, pos), sorted
    unsigned long long* pcnt = A.alloc<unsigned long long>(U + 1);
    CK(cudaMemsetAsync(pcnt + U, 0, 8, s));
    dev::prefix_counts<<<static_cast<unsigned>((U + 255) / 256), 256, 0, s>>>(rep->sizes, grp_begin, d_plen_index,
                                                                            static_cast<uint32_t>(U), pcnt);
    ++st.launches;
    CK(cudaGetLastError());
    scan_u64(pcnt, U + 1, A, s, st.launches);
    const uint64_t P = read_u64(pcnt + U, s);
    if (P >= (uint64_t(1) << 32)) throw std::invalid_argument("prefix index above 2^32 postings is not supported");
    SortBufs IB{};
    IB.ka = A.alloc<unsigned long long>(P);
    IB.kb = A.alloc<unsigned long long>(P);
    IB.va = A.alloc<uint32_t>(P);
    IB.vb = A.alloc<uint32_t>(P);
    {
        const uint64_t ntiles = (P + dev::kSortTile - 1) / dev::kSortTile;
        IB.hist = A.alloc<uint32_t>(256ull * std::max<uint64_t>(ntiles, 1));
        IB.sums = A.alloc<uint32_t>((256ull * std::max<uint64_t>(ntiles, 1) + dev::kScanBlock - 1) / dev::kScanBlock + 1);
    }
    IB.count_store = pcnt + U;
    IB.count = pcnt + U;
    dev::prefix_emit<<<static_cast<unsigned>((U * 32 + 255) / 256), 256, 0, s>>>(
        rep->tokens, rep->offsets, rep->sizes, grp_begin, d_plen_index, static_cast<uint32_t>(U), pcnt, IB.ka, IB.va);
    ++st.launches;
    CK(cudaGetLastError());
    int idbits = 1;
    while ((uint64_t(1) << idbits) < std::max<uint64_t>(c.universe, U) + 1) ++idbits;
    const bool inb = sort_results(IB, P, idbits, s, st.launches);
    const unsigned long long* pkey = inb ? IB.kb : IB.ka;
    const uint32_t* ppos = inb ? IB.vb : IB.va;
    unsigned long long* eoff = A.alloc<unsigned long long>(P + 1);
    CK(cudaMemsetAsync(eoff + P, 0, 8, s));
    if (P)
        dev::prefix_encounter_counts<<<static_cast<unsigned>((P + 255) / 256), 256, 0, s>>>(pkey, P, eoff);
    ++st.launches;
    CK(cudaGetLastError());
    scan_u64(eoff, P + 1, A, s, st.launches);
    const uint64_t E = read_u64(eoff + P, s);
    cudaEvent_t e_index = T.mark();
    st.window_pairs = E;  // encounters (pair x common prefix token)

    unsigned long long* ctr = A.alloc<unsigned long long>(dev::kPcSlots);
    dev::PrefixParams PP{};
    PP.tokens = rep->tokens;
    PP.offsets = rep->offsets;
    PP.sizes = rep->sizes;
    PP.rec = grp_begin;  // group g's representative = its first record
    PP.pkey = pkey;
    PP.ppos = ppos;
    PP.eoff = eoff;
    PP.P = P;
    PP.E = E;
    PP.plen = d_plen_index;
    PP.lower = d_lower;
    PP.upper = d_upper;
    PP.need.minov = d_minov;
    PP.need.cosine = o.sim == Sim::Cosine ? 1 : 0;
    PP.need.cp = o.threshold.num;
    PP.need.cq = o.threshold.den;
    PP.positional = o.algorithm == Algo::PPJoin || o.algorithm == Algo::PPJoinPlus || group;
    PP.suffix = o.algorithm == Algo::PPJoinPlus;
    PP.suffix_depth = o.suffix_depth;
    PP.f2 = f2;
    PP.f3 = f3;
    PP.bits = rb.enabled ? bits : nullptr;
    PP.words = W;
    PP.cutoff = rb.cutoff;
    PP.ctr = ctr;
    PP.group_mode = group;
    PP.grp_begin = grp_begin;
    PP.ell_max = L;
    PP.plen_ell = d_plen;
    PP.max_size = ms;
    PP.n_rows = static_cast<uint32_t>(n);

    // result buffer: matches <= first encounters <= E; sized from free HBM
    // (40 B per result: keys / overlaps, sort buffers, packed pairs) so a
    // re-run after an overflow is the exception
    size_t free_b = 0, total_b = 0;
    CK(cudaMemGetInfo(&free_b, &total_b));
    uint64_t res_cap = std::min<uint64_t>(std::max<uint64_t>(E, 1024),
                                          std::max<uint64_t>(free_b / 2 / 40, uint64_t(1) << 20));
    res_cap = std::min<uint64_t>(res_cap, env_u64("SSJB_PREFIX_RESULT_CAP", ~uint64_t(0)));
    uint64_t item_cap = group ? std::min<uint64_t>(std::max<uint64_t>(E + U, 1024), uint64_t(1) << 26) : 0;
    unsigned long long h[dev::kPcSlots];
    double ms_filter = 0, ms_verify = 0;
    uint64_t R = 0;
    SortBufs RB{};
    for (;;) {  // re-run with larger buffers if the results / items overflowed
        CK(cudaMemsetAsync(ctr, 0, dev::kPcSlots * 8, s));
        RB = SortBufs{};
        RB.ka = A.alloc<unsigned long long>(res_cap);
        RB.va = A.alloc<uint32_t>(res_cap);
        PP.res_keys = RB.ka;
        PP.res_ov = RB.va;
        PP.res_cap = res_cap;
        PP.items = group ? A.alloc<uint2>(item_cap) : nullptr;
        PP.item_cap = item_cap;
        cudaEvent_t f0 = T.mark();
        if (adapt) {
            const uint64_t nL = n * static_cast<uint64_t>(L);
            uint32_t* tallies = A.alloc<uint32_t>(4 * nL + n);
            CK(cudaMemsetAsync(tallies, 0, (4 * nL + n) * 4, s));
            PP.a_touch = tallies;
            PP.a_alive = tallies + nL;
            PP.a_len = tallies + 2 * nL;
            PP.a_bmp = tallies + 3 * nL;
            PP.a_bt = tallies + 4 * nL;
            uint8_t* ell = A.alloc<uint8_t>(n);
            // candidate list of the tally pass (10 B per pair), bounded by free HBM;
            // if it overflows the verify pass re-enumerates the encounters instead
            {
                size_t fb = 0, tb = 0;
                CK(cudaMemGetInfo(&fb, &tb));
                PP.a_cand_cap = std::min<uint64_t>(std::max<uint64_t>(E, 1), fb / 4 / 10);
                PP.a_cand_cap = std::min<uint64_t>(PP.a_cand_cap, env_u64("SSJB_ADAPT_LIST_CAP", ~uint64_t(0)));
                PP.a_cand = A.alloc<uint2>(PP.a_cand_cap);
                PP.a_cmask = A.alloc<uint16_t>(PP.a_cand_cap);
            }
            if (E) dev::adapt_tally<<<grid_for(E, sms, 8), 256, 0, s>>>(PP);
            ++st.launches;
            CK(cudaGetLastError());
            dev::AdaptRowParams AR{};
            AR.tokens = rep->tokens;
            AR.offsets = rep->offsets;
            AR.sizes = rep->sizes;
            AR.pkey = pkey;
            AR.P = P;
            AR.plen_ell = d_plen;
            AR.ellcap = d_ellcap;
            AR.max_size = ms;
            AR.ell_max = L;
            AR.avg = c.mean_size();
            AR.n = static_cast<uint32_t>(n);
            AR.touch = PP.a_touch;
            AR.alive = PP.a_alive;
            AR.len = PP.a_len;
            AR.bmp = PP.a_bmp;
            AR.bt = PP.a_bt;
            AR.ell_out = ell;
            AR.ctr = ctr;
            dev::adapt_rows<<<static_cast<unsigned>((n + 255) / 256), 256, 0, s>>>(AR);
            ++st.launches;
            CK(cudaGetLastError());
            PP.a_ell = ell;
            const uint64_t ncand = read_u64(ctr + dev::kPcCand, s);
            if (ncand <= PP.a_cand_cap) {
                if (ncand) dev::adapt_verify_list<<<grid_for(ncand, sms, 8), 256, 0, s>>>(PP, ncand);
            } else if (E) {
                dev::adapt_verify<<<grid_for(E, sms, 8), 256, 0, s>>>(PP);
            }
            ++st.launches;
            CK(cudaGetLastError());
        } else if (E) {
            dev::prefix_encounters<<<grid_for(E, sms, 16), 256, 0, s>>>(PP);
            ++st.launches;
            CK(cudaGetLastError());
        }
        cudaEvent_t f1 = T.mark();
        if (group) {
            dev::group_intra<<<static_cast<unsigned>((U + 255) / 256), 256, 0, s>>>(grp_begin, static_cast<uint32_t>(U),
                                                                                  PP.items, item_cap, ctr);
            ++st.launches;
            CK(cudaGetLastError());
            const uint64_t m = read_u64(ctr + dev::kPcItems, s);
            if (m > item_cap) {
                item_cap = m;
                continue;
            }
            if (m) {
                unsigned long long* foff = A.alloc<unsigned long long>(m + 1);
                CK(cudaMemsetAsync(foff + m, 0, 8, s));
                dev::group_item_sizes<<<static_cast<unsigned>((m + 255) / 256), 256, 0, s>>>(PP.items, m, grp_begin, foff);
                ++st.launches;
                CK(cudaGetLastError());
                scan_u64(foff, m + 1, A, s, st.launches);
                const uint64_t total = read_u64(foff + m, s);
                if (total) dev::group_expand<<<grid_for(total, sms, 8), 256, 0, s>>>(PP, PP.items, m, foff, total);
                ++st.launches;
                CK(cudaGetLastError());
            }
        }
        cudaEvent_t f2e = T.mark();
        CK(cudaMemcpyAsync(h, ctr, sizeof h, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        ms_filter = Timer::ms(f0, f1);
        ms_verify = Timer::ms(f1, f2e);
        R = h[dev::kPcResults];
        if (R > res_cap) {
            res_cap = R;
            continue;
        }
        break;
    }
    out.candidates = h[dev::kPcCandidates];
    out.pruned_length = h[dev::kPcPrunedLength];
    out.pruned_positional = h[dev::kPcPrunedPositional];
    out.pruned_suffix = h[dev::kPcPrunedSuffix];
    out.pruned_bitmap = h[dev::kPcPrunedBitmap];
    out.bitmap_tested = h[dev::kPcBitmapTested];
    out.filter_evaluations = h[dev::kPcFilterEvals];
    out.verified = h[dev::kPcVerified];
    out.matched = h[dev::kPcMatched];
    st.survivors = out.verified;

    // canonical order (src/join.cpp:30-32), one packed download
    cudaEvent_t s0 = T.mark();
    if (R) {
        RB.kb = A.alloc<unsigned long long>(R);
        RB.vb = A.alloc<uint32_t>(R);
        const uint64_t ntiles = (R + dev::kSortTile - 1) / dev::kSortTile;
        RB.hist = A.alloc<uint32_t>(256ull * ntiles);
        RB.sums = A.alloc<uint32_t>((256ull * ntiles + dev::kScanBlock - 1) / dev::kScanBlock + 1);
        RB.count = ctr + dev::kPcResults;
        int rbits = 1;
        while ((uint64_t(1) << rbits) < n + 1) ++rbits;
        const bool rin = sort_results(RB, R, rbits, s, st.launches);
        PairOut* packed = A.alloc<PairOut>(R);
        pack_pairs<<<static_cast<unsigned>((R + 255) / 256), 256, 0, s>>>(rin ? RB.kb : RB.ka, rin ? RB.vb : RB.va,
                                                                          packed, R);
        ++st.launches;
        CK(cudaGetLastError());
        out.pairs.resize(R);
        d2h_staged(out.pairs.data(), packed, R * sizeof(PairOut), s);
        st.d2h_bytes += R * sizeof(PairOut);
    }
    cudaEvent_t s1 = T.mark();
    CK(cudaStreamSynchronize(s));
    st.ms_upload = Timer::ms(e0, e_index);
    st.ms_filter = ms_filter;
    st.ms_verify = ms_verify;
    st.ms_sort = Timer::ms(s0, s1);
    st.batches = 1;
    out.index_s = Timer::ms(e0, e_index) / 1e3;
    out.candidates_s = ms_filter / 1e3;
    out.verify_s = std::chrono::duration<double>(Clock::now() - t_start).count() - out.index_s - out.candidates_s;
}

}  // namespace ssjb
