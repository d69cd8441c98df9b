// engine.cu — engine lifetime, workspace, error plumbing, host RNG entry point.
#include <algorithm>
#include <cstring>
#include <stdexcept>
#include <vector>

#include "common.cuh"
#include "rng.cuh"

#include <map>
#include <mutex>
#include <tuple>
#include <set>
#include <utility>

namespace kt {

static thread_local std::string g_last_error;

void set_last_error(const std::string& msg) { g_last_error = msg; }

[[noreturn]] void fail(int code, const std::string& msg) { throw Error{code, msg}; }

// Raise a kernel's dynamic shared-memory limit to the device's opt-in maximum, once
// per (device, kernel).  Setting the limit per launch to that launch's size races
// when several host threads (several engines) launch the same kernel.
void allow_dynamic_smem(const void* kernel) {
    static std::mutex mu;
    static std::set<std::pair<int, const void*>> done;
    int dev = 0;
    KT_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(mu);
    if (done.count({dev, kernel})) return;
    int optin = 0;
    KT_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    cudaFuncAttributes fa{};
    KT_CUDA(cudaFuncGetAttributes(&fa, kernel));
    KT_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, optin - int(fa.sharedSizeBytes)));
    done.insert({dev, kernel});
}

// Launch-planning queries are constant per (device, kernel, shape): cached, because a driver
// round trip each (cudaOccupancy*, cudaFuncGetAttributes, cudaDeviceGetAttribute: ~5-20 us)
// on every launch of an adaptive_sample step left the GPU idle between kernels.
int occupancy_blocks(const void* kernel, int threads, size_t smem) {
    static std::mutex mu;
    static std::map<std::tuple<int, const void*, int, size_t>, int> cache;
    int dev = 0;
    KT_CUDA(cudaGetDevice(&dev));
    const auto key = std::make_tuple(dev, kernel, threads, smem);
    {
        std::lock_guard<std::mutex> lk(mu);
        auto it = cache.find(key);
        if (it != cache.end()) return it->second;
    }
    int blocks = 0;
    KT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, kernel, threads, smem));
    std::lock_guard<std::mutex> lk(mu);
    cache[key] = blocks;
    return blocks;
}

int smem_optin(int device) {
    static std::mutex mu;
    static std::map<int, int> cache;
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find(device);
    if (it != cache.end()) return it->second;
    int optin = 0;
    KT_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device));
    cache[device] = optin;
    return optin;
}

size_t static_smem(const void* kernel) {
    static std::mutex mu;
    static std::map<const void*, size_t> cache;
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find(kernel);
    if (it != cache.end()) return it->second;
    cudaFuncAttributes fa{};
    KT_CUDA(cudaFuncGetAttributes(&fa, kernel));
    cache[kernel] = fa.sharedSizeBytes;
    return fa.sharedSizeBytes;
}

RowFmt row_fmt(const int32_t* cards, int n) {
    if (n < 1 || n > kMaxKnobs) fail(KT_ERR_UNSUPPORTED, "the engine supports spaces of 1..8 knobs");
    RowFmt f{};
    int maxc = 1;
    for (int k = 0; k < n; ++k) {
        if (cards[k] < 1) fail(KT_ERR_VALUE, "knob cardinalities must be >= 1");
        maxc = std::max(maxc, int(cards[k]));
    }
    f.cmax = maxc - 1;
    if (maxc <= kMaxCard) {  // one byte per knob
        f.bytes = 1;
        for (int k = 0; k < kMaxKnobs; ++k) f.shift[k] = uint8_t(8 * k), f.width[k] = 8;
        return f;
    }
    if (maxc > 65535) fail(KT_ERR_UNSUPPORTED, "engine rows support knobs with at most 65535 settings");
    int pos = 0;
    for (int k = 0; k < n; ++k) {
        int w = 1;
        while ((1 << w) < cards[k]) ++w;
        f.shift[k] = uint8_t(pos);
        f.width[k] = uint8_t(w);
        pos += w;
    }
    // bit 63 stays clear, so no row can equal the all-ones empty-slot sentinel
    if (pos > 63) fail(KT_ERR_UNSUPPORTED, "the space's knob indices need more than 63 bits per row");
    return f;
}

}  // namespace kt

void* kt_engine::scratch(const std::string& name, size_t bytes) {
    if (bytes == 0) bytes = 16;
    Buf& b = dev[name];
    if (b.bytes < bytes) {
        if (b.ptr) KT_CUDA(cudaFreeAsync(b.ptr, stream));
        size_t grow = bytes + bytes / 4;
        KT_CUDA(cudaMallocAsync(&b.ptr, grow, stream));
        b.bytes = grow;
    }
    return b.ptr;
}

void* kt_engine::staging(const std::string& name, size_t bytes) {
    if (bytes == 0) bytes = 16;
    Buf& b = pinned[name];
    if (b.bytes < bytes) {
        if (b.ptr) {
            KT_CUDA(cudaStreamSynchronize(stream));
            KT_CUDA(cudaFreeHost(b.ptr));
        }
        size_t grow = bytes + bytes / 4;
        KT_CUDA(cudaMallocHost(&b.ptr, grow));
        b.bytes = grow;
    }
    return b.ptr;
}

namespace {
// one warp, few registers: it fits beside a resident Lloyd / GEMM block on a busy SM, so an engine's
// read-back never waits for another engine's cooperative launch to drain (concurrent engines)
__global__ void __launch_bounds__(32) readback_kernel(uint32_t* __restrict__ dst, const uint32_t* __restrict__ src,
                                                      size_t words) {
    for (size_t i = threadIdx.x; i < words; i += blockDim.x) dst[i] = src[i];
}
struct ReadbackList {
    uint32_t* dst[8];
    const uint32_t* src[8];
    uint32_t words[8];
    int n;
};
__global__ void __launch_bounds__(32) readback_list_kernel(ReadbackList l) {
    for (int r = 0; r < l.n; ++r)
        for (uint32_t i = threadIdx.x; i < l.words[r]; i += blockDim.x) l.dst[r][i] = l.src[r][i];
}
}  // namespace

void kt_engine::d2h(std::initializer_list<D2H> regions) {
    static const bool use_copy = std::getenv("KT_D2H_COPY") != nullptr;
    ReadbackList l{};
    for (const D2H& d : regions) {
        const bool ok = !use_copy && !(d.bytes & 3) && !(reinterpret_cast<uintptr_t>(d.dst) & 3) &&
                        !(reinterpret_cast<uintptr_t>(d.src) & 3) && d.bytes / 4 < (size_t(1) << 31) && l.n < 8;
        if (!ok) {
            KT_CUDA(cudaMemcpyAsync(d.dst, d.src, d.bytes, cudaMemcpyDeviceToHost, stream));
            continue;
        }
        if (!d.bytes) continue;
        l.dst[l.n] = static_cast<uint32_t*>(d.dst);
        l.src[l.n] = static_cast<const uint32_t*>(d.src);
        l.words[l.n] = uint32_t(d.bytes / 4);
        ++l.n;
    }
    if (!l.n) return;
    pre_launch("readback");
    readback_list_kernel<<<1, 32, 0, stream>>>(l);
    check_launch("readback");
}

void kt_engine::d2h(void* host_dst, const void* dev_src, size_t bytes) {
    // KT_D2H_COPY=1: plain cudaMemcpyAsync (A/B switch)
    static const bool use_copy = std::getenv("KT_D2H_COPY") != nullptr;
    if (use_copy || (bytes & 3) || (reinterpret_cast<uintptr_t>(host_dst) & 3) ||
        (reinterpret_cast<uintptr_t>(dev_src) & 3)) {
        KT_CUDA(cudaMemcpyAsync(host_dst, dev_src, bytes, cudaMemcpyDeviceToHost, stream));
        return;
    }
    if (bytes == 0) return;
    pre_launch("readback");
    readback_kernel<<<1, 32, 0, stream>>>(static_cast<uint32_t*>(host_dst), static_cast<const uint32_t*>(dev_src),
                                           bytes / 4);
    check_launch("readback");
}

cudaEvent_t kt_engine::take_event() {
    if (!event_pool.empty()) {
        cudaEvent_t ev = event_pool.back();
        event_pool.pop_back();
        return ev;
    }
    cudaEvent_t ev;
    KT_CUDA(cudaEventCreate(&ev));
    return ev;
}

void kt_engine::pre_launch(const char* what) {
    (void)what;
    if (!timing) return;
    open_start = take_event();
    KT_CUDA(cudaEventRecord(open_start, stream));
}

void kt_engine::check_launch(const char* what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) kt::fail(KT_ERR_CUDA, std::string("launch of ") + what + ": " + cudaGetErrorString(e));
    static const bool sync_check = std::getenv("KT_SYNC_CHECK") != nullptr;  // debugging: name the faulting kernel
    if (sync_check) {
        e = cudaStreamSynchronize(stream);
        if (e != cudaSuccess) kt::fail(KT_ERR_CUDA, std::string("kernel ") + what + ": " + cudaGetErrorString(e));
    }
    note_launch();
    if (timing && open_start) {
        cudaEvent_t stop = take_event();
        KT_CUDA(cudaEventRecord(stop, stream));
        pending.push_back({what, open_start, stop});
        open_start = nullptr;
    }
}

void kt_engine::flush_timing() {
    if (pending.empty()) return;
    KT_CUDA(cudaStreamSynchronize(stream));
    // KT_GAP_TRACE: idle time of the stream between consecutive timed launches, attributed to
    // the pair (host work / synchronisations between them), accumulated as "gap:<a>><b>"
    static const bool gaps = std::getenv("KT_GAP_TRACE") != nullptr;
    for (size_t i = 0; i < pending.size(); ++i) {
        auto& p = pending[i];
        float ms = 0.f;
        KT_CUDA(cudaEventElapsedTime(&ms, p.start, p.stop));
        Stat& s = stats[p.name];
        s.count += 1;
        s.ms += ms;
        if (gaps && i + 1 < pending.size()) {
            float g = 0.f;
            KT_CUDA(cudaEventElapsedTime(&g, p.stop, pending[i + 1].start));
            Stat& gs = stats[std::string("gap:") + p.name + ">" + pending[i + 1].name];
            gs.count += 1;
            gs.ms += g;
        }
    }
    for (auto& p : pending) {
        event_pool.push_back(p.start);
        event_pool.push_back(p.stop);
    }
    pending.clear();
}

void kt_engine::sync() { KT_CUDA(cudaStreamSynchronize(stream)); }

extern "C" {

const char* kt_last_error(void) { return kt::g_last_error.c_str(); }

const char* kt_version(void) { return "knobtuner_b200 0.1 (sm_100a)"; }

int kt_row_layout(const int32_t* cards, int n_knobs, int32_t* shift_out, int32_t* width_out) {
    KT_API_BEGIN
    const kt::RowFmt f = kt::row_fmt(cards, n_knobs);
    for (int k = 0; k < n_knobs; ++k) {
        shift_out[k] = f.shift[k];
        width_out[k] = f.width[k];
    }
    KT_API_END
}

int kt_engine_create(int device, kt_engine** out) {
    KT_API_BEGIN
    if (!out) kt::fail(KT_ERR_VALUE, "out is NULL");
    int count = 0;
    KT_CUDA(cudaGetDeviceCount(&count));
    if (device < 0 || device >= count) kt::fail(KT_ERR_VALUE, "no CUDA device " + std::to_string(device));
    KT_CUDA(cudaSetDevice(device));
    cudaDeviceProp prop;
    KT_CUDA(cudaGetDeviceProperties(&prop, device));
    if (prop.major < 10) kt::fail(KT_ERR_UNSUPPORTED, std::string("engine is built for sm_100a; device is ") + prop.name);
    auto* e = new kt_engine();
    e->device = device;
    e->num_sms = prop.multiProcessorCount;
    KT_CUDA(cudaStreamCreateWithFlags(&e->own_stream, cudaStreamNonBlocking));
    e->stream = e->own_stream;
    *out = e;
    KT_API_END
}

int kt_engine_destroy(kt_engine* e) {
    KT_API_BEGIN
    if (!e) return KT_OK;
    cudaSetDevice(e->device);
    cudaStreamSynchronize(e->stream);
    for (auto& kv : e->dev)
        if (kv.second.ptr) cudaFree(kv.second.ptr);
    for (auto& kv : e->pinned)
        if (kv.second.ptr) cudaFreeHost(kv.second.ptr);
    if (e->own_stream) cudaStreamDestroy(e->own_stream);
    delete e;
    KT_API_END
}

int kt_engine_set_stream(kt_engine* e, void* s) {
    KT_API_BEGIN
    KT_CUDA(cudaStreamSynchronize(e->stream));
    e->stream = s ? static_cast<cudaStream_t>(s) : e->own_stream;
    KT_API_END
}

// Cross-stream ordering without a host round trip: `after` = 0 makes the engine stream wait for
// everything enqueued so far on `other`; 1 makes `other` wait for the engine stream.
int kt_engine_order(kt_engine* e, void* other, int after) {
    KT_API_BEGIN
    auto* o = static_cast<cudaStream_t>(other);
    if (o == e->stream) return KT_OK;
    if (!e->order_event) KT_CUDA(cudaEventCreateWithFlags(&e->order_event, cudaEventDisableTiming));
    if (after == 0) {
        KT_CUDA(cudaEventRecord(e->order_event, o));
        KT_CUDA(cudaStreamWaitEvent(e->stream, e->order_event, 0));
    } else {
        KT_CUDA(cudaEventRecord(e->order_event, e->stream));
        KT_CUDA(cudaStreamWaitEvent(o, e->order_event, 0));
    }
    KT_API_END
}

int kt_engine_synchronize(kt_engine* e) {
    KT_API_BEGIN
    e->sync();
    KT_API_END
}

int64_t kt_engine_launch_count(const kt_engine* e) { return e ? e->launches : 0; }

int kt_engine_set_timing(kt_engine* e, int enabled) {
    KT_API_BEGIN
    e->flush_timing();
    e->timing = enabled != 0;
    KT_API_END
}

int kt_engine_kernel_stats(kt_engine* e, int capacity, char* names, int64_t* counts, double* total_ms,
                           int32_t* n_kernels, int reset) {
    KT_API_BEGIN
    e->flush_timing();
    int i = 0;
    for (auto& kv : e->stats) {
        if (i >= capacity) break;
        std::strncpy(names + size_t(i) * 32, kv.first.c_str(), 31);
        names[size_t(i) * 32 + 31] = '\0';
        counts[i] = kv.second.count;
        total_ms[i] = kv.second.ms;
        ++i;
    }
    *n_kernels = i;
    if (reset) e->stats.clear();
    KT_API_END
}

int kt_pcg64_draw(const uint32_t* entropy, int ne, const uint32_t* spawn, int ns, int kind,
                  uint64_t bound, int64_t count, void* out) {
    KT_API_BEGIN
    if (ne < 1 || ne > 16 || ns < 0 || ns > 16) kt::fail(KT_ERR_VALUE, "entropy/spawn word counts out of range");
    kt::Pcg64 g = kt::pcg64_from_seed_sequence(entropy, ne, spawn, ns);
    if (kind == 0) {
        double* o = static_cast<double*>(out);
        for (int64_t i = 0; i < count; ++i) o[i] = g.random();
    } else if (kind == 1) {
        if (bound == 0 || bound > 0x100000000ull) kt::fail(KT_ERR_VALUE, "bound must be in [1, 2^32]");
        int64_t* o = static_cast<int64_t*>(out);
        for (int64_t i = 0; i < count; ++i) o[i] = int64_t(g.bounded32(uint32_t(bound - 1)));
    } else {
        kt::fail(KT_ERR_VALUE, "kind must be 0 (random) or 1 (integers)");
    }
    KT_API_END
}

}  // extern "C"
