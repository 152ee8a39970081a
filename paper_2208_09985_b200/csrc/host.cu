// Host runtime behind the C ABI (include/scrooge_b200.h): validation,
// 2-bit packing (K4), per-device pipelines (H2D -> K1 -> K2 -> K3 -> D2H),
// static cost-balanced sharding over devices with one host thread each (K5),
// device-resident sessions, synthetic batches and run decoding.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <condition_variable>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <numeric>
#include <string>
#include <thread>
#include <type_traits>
#include <vector>

#include "../../include/scrooge_b200.h"
#include "synth.h"
#include "window_align.cuh"

namespace {

thread_local std::string g_last_error;

int set_error(int code, const char* fmt, ...) {
    char buf[1024];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_last_error = buf;
    return code;
}

}  // namespace

namespace sgk {
int set_error_msg(int code, const std::string& msg) {  // for io.cpp
    g_last_error = msg;
    return code;
}
}  // namespace sgk

namespace {

struct Fail {  // thrown inside the runtime, converted to a status at the ABI
    int code;
};

#define SG_CUDA_CHECK(expr)                                                             \
    do {                                                                                \
        cudaError_t e__ = (expr);                                                       \
        if (e__ != cudaSuccess) {                                                       \
            set_error(SG_CUDA, "CUDA error %s at %s:%d (%s)", cudaGetErrorString(e__), \
                      __FILE__, __LINE__, #expr);                                       \
            throw Fail{SG_CUDA};                                                        \
        }                                                                               \
    } while (0)

int hw_threads() {
    const unsigned h = std::thread::hardware_concurrency();
    return h ? static_cast<int>(std::min(h, 64u)) : 8;
}

// Worker threads for the host loops over the pairs, started once and kept (creating
// a thread costs ~0.2 ms on the GPU hosts: more than a pass over 100 k pairs). One
// parallel loop uses them at a time; a caller that finds them busy (another shard's
// host thread) runs its loop on threads of its own.
class WorkerPool {
  public:
    explicit WorkerPool(int workers) {
        for (int w = 0; w < workers; ++w) std::thread([this] { loop(); }).detach();
    }
    // job(t) for t in [0, tasks), the caller taking part; false when the pool is busy
    template <class Job>
    bool run(int tasks, Job&& job) {
        std::unique_lock<std::mutex> use(use_mu_, std::try_to_lock);
        if (!use.owns_lock()) return false;
        using JobT = typename std::remove_reference<Job>::type;
        struct Call {
            JobT* job;
            static void invoke(void* c, int t) { (*static_cast<Call*>(c)->job)(t); }
        } call{&job};
        unsigned gen;
        {
            std::lock_guard<std::mutex> lk(mu_);
            fn_ = &Call::invoke;
            ctx_ = &call;
            tasks_ = tasks;
            gen = ++gen_;
            next_.store(static_cast<uint64_t>(gen) << 32);
            left_ = tasks;
        }
        cv_.notify_all();
        drain(gen, tasks, &Call::invoke, &call);
        std::unique_lock<std::mutex> lk(mu_);
        done_.wait(lk, [this] { return left_ == 0; });
        fn_ = nullptr;
        return true;
    }

  private:
    // Tasks of generation `gen` only: the ticket carries the generation, so a worker
    // that wakes late never takes (or skips) a task of a later loop.
    void drain(unsigned gen, int tasks, void (*fn)(void*, int), void* ctx) {
        uint64_t cur = next_.load();
        for (;;) {
            if (static_cast<unsigned>(cur >> 32) != gen || static_cast<int>(cur & 0xFFFFFFFFu) >= tasks)
                return;
            if (!next_.compare_exchange_weak(cur, cur + 1)) continue;
            fn(ctx, static_cast<int>(cur & 0xFFFFFFFFu));
            {
                std::lock_guard<std::mutex> lk(mu_);
                if (--left_ == 0) done_.notify_all();
            }
            cur = next_.load();
        }
    }
    void loop() {
        unsigned seen = 0;
        for (;;) {
            void (*fn)(void*, int);
            void* ctx;
            int tasks;
            {
                std::unique_lock<std::mutex> lk(mu_);
                cv_.wait(lk, [&] { return gen_ != seen && fn_ != nullptr; });
                seen = gen_;
                fn = fn_;
                ctx = ctx_;
                tasks = tasks_;
            }
            drain(seen, tasks, fn, ctx);
        }
    }
    std::mutex use_mu_, mu_;
    std::condition_variable cv_, done_;
    void (*fn_)(void*, int) = nullptr;
    void* ctx_ = nullptr;
    int tasks_ = 0, left_ = 0;
    std::atomic<uint64_t> next_{0};  // (generation << 32) | next task
    unsigned gen_ = 0;
};

WorkerPool& worker_pool() {  // (leaked: its threads never outlive a destroyed object)
    static WorkerPool* pool = new WorkerPool(std::max(1, hw_threads() - 1));
    return *pool;
}

// f(lo, hi, chunk_index) over [0, n) in contiguous chunks (at most 64, at least
// `grain` items each).
template <class F>
void parallel_for(int64_t n, F&& f, int64_t grain = 1024) {
    int threads = hw_threads();
    threads = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(threads, n / grain)));
    if (threads <= 1) {
        f(int64_t{0}, n, 0);
        return;
    }
    const int64_t chunk = (n + threads - 1) / threads;
    auto task = [&](int t) {
        const int64_t lo = t * chunk, hi = std::min(n, lo + chunk);
        if (lo < hi) f(lo, hi, t);
    };
    if (worker_pool().run(threads, task)) return;
    std::vector<std::thread> pool;
    for (int t = 0; t < threads; ++t) pool.emplace_back([&task, t] { task(t); });
    for (auto& th : pool) th.join();
}

// ------------------------------------------------------------ options, device guard

std::mutex g_opt_mu;
sg_options g_opt = {SG_KERNEL_AUTO, 1, 1, 0, 0};

sg_options options() {
    std::lock_guard<std::mutex> lk(g_opt_mu);
    return g_opt;
}

// Restores the caller's current device when an ABI call returns: the library
// must not change the host application's CUDA device (a drop-in sits next to
// PyTorch and others that rely on it).
struct DeviceGuard {
    int prev = -1;
    DeviceGuard() {
        if (cudaGetDevice(&prev) != cudaSuccess) {
            prev = -1;
            cudaGetLastError();
        }
    }
    ~DeviceGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
    DeviceGuard(const DeviceGuard&) = delete;
    DeviceGuard& operator=(const DeviceGuard&) = delete;
};

// ------------------------------------------------------------ pinned host memory

// Grow-only pool so repeated calls do not re-pin memory inside timed regions.
// Without a device (host-only helpers such as sg_pack / sg_synth_* on a CPU
// box) it hands out pageable memory; computing still requires the GPU.
struct PinnedPool {
    std::mutex mu;
    std::vector<std::pair<void*, size_t>> free_list;
    std::vector<void*> pageable;  // blocks from malloc (never pinned)

    void* acquire(size_t bytes, size_t* got) {
        bytes = std::max<size_t>(bytes, 256);
        {
            std::lock_guard<std::mutex> lk(mu);
            size_t bi = SIZE_MAX;
            for (size_t k = 0; k < free_list.size(); ++k) {
                const size_t c = free_list[k].second;
                if (c >= bytes && c <= 2 * bytes + (size_t{64} << 20) &&
                    (bi == SIZE_MAX || c < free_list[bi].second))
                    bi = k;
            }
            if (bi != SIZE_MAX) {
                void* p = free_list[bi].first;
                *got = free_list[bi].second;
                free_list.erase(free_list.begin() + static_cast<long>(bi));
                return p;
            }
        }
        void* p = nullptr;
        if (cudaMallocHost(&p, bytes) != cudaSuccess) {
            cudaGetLastError();
            p = std::malloc(bytes);
            if (!p) {
                set_error(SG_INTERNAL, "out of host memory (%zu bytes)", bytes);
                throw Fail{SG_INTERNAL};
            }
            std::lock_guard<std::mutex> lk(mu);
            pageable.push_back(p);
        }
        *got = bytes;
        return p;
    }
    void release(void* p, size_t bytes) {
        if (!p) return;
        std::lock_guard<std::mutex> lk(mu);
        free_list.emplace_back(p, bytes);
    }
};

PinnedPool& pinned() {
    static PinnedPool* pool = new PinnedPool();  // process lifetime
    return *pool;
}

struct PinBuf {
    void* p = nullptr;
    size_t cap = 0;
    PinBuf() = default;
    PinBuf(const PinBuf&) = delete;
    PinBuf& operator=(const PinBuf&) = delete;
    void ensure(size_t bytes) {
        if (p && bytes <= cap) return;
        reset();
        p = pinned().acquire(bytes, &cap);
    }
    void reset() {
        if (p) pinned().release(p, cap);
        p = nullptr;
        cap = 0;
    }
    ~PinBuf() { reset(); }
    template <class T> T* as() const { return static_cast<T*>(p); }
};

// ------------------------------------------------------------ device memory

struct DevBuf {
    void* p = nullptr;
    size_t cap = 0;
    void ensure(size_t bytes) {
        bytes = std::max<size_t>(bytes, 256);
        if (p && bytes <= cap) return;
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
        SG_CUDA_CHECK(cudaMalloc(&p, bytes));
        cap = bytes;
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
    }
    template <class T> T* as() const { return static_cast<T*>(p); }
};

// Device buffers, stream and events of one pipeline on one device.
struct DevState {
    int device = 0;
    int sms = 0;
    cudaStream_t stream = nullptr;
    cudaEvent_t ev[3] = {};
    DevBuf seq, nmask, text_off, pat_off, text_len, pat_len, has_n, order;
    DevBuf distance, windows, status, out_bytes, counters, bound_off, scratch, bnd, next_pair;
    DevBuf ready;                    // per-chunk "sequence words arrived" flags (streamed upload)
    DevBuf bnd_ones, bnd_zeros;      // constant parked rows (one warp's slots, L = 4 size)
    cudaStream_t copy = nullptr;     // H2D of the sequence words, overlapping K1
    cudaEvent_t copy_go = nullptr;
    cudaEvent_t copy_done = nullptr; // the last piece of the upload (joined before K2)
    int64_t chunk_words = 1;
    int n_chunks = 1;                // pieces of the last sequence upload
    DevBuf dense_off, dense, scan_tmp;
    DevBuf ex_store, ex_hbuf, ex_store_off, ex_hbuf_off;  // K7 (exact global alignment)
    // K1 mixed (§3.8-3.10): hand-over queues, counters (remaining pairs, K0 count),
    // the handed pairs' state, K0's list of unrelated pairs
    DevBuf q_band, q_full, q_coop, q_std, mixed_ctr, resume_state, u_list, t_list;
    long long grid = 0, lanes = 0;
    // diagnostics (SG_DIAG_*) of the last launch on this device
    DevBuf diag_warp, diag_phase;
    int diag_warps = 0, diag_flags = 0;
    // sliced output (one-shot calls, §5): K2/K3 per slice of finished pairs on their
    // own stream while K1 runs, each slice's run bytes copied out as soon as it is ready
    static constexpr int kMaxSlices = 32;
    DevBuf slice_done;
    // pipelined launches of the mixed kernel (§3.12): per-slice list counts, hand-over
    // counts, queue heads and the error flag (kPipe* offsets, in 32-bit words)
    DevBuf pipe_ctr;
    static constexpr int kPipeT = 0, kPipeU = kMaxSlices, kPipeBody = 2 * kMaxSlices,
                         kPipeTailQ = 3 * kMaxSlices, kPipeFullQ = 4 * kMaxSlices,
                         kPipeErr = 5 * kMaxSlices, kPipeWords = 5 * kMaxSlices + 8;
    int tail_sms = 0;               // SMs the last pipelined launch left to the tail kernels
    cudaEvent_t k1_done = nullptr;  // the last slice's full-frame K1 (K1's end in a pipelined launch)
    cudaStream_t slice_stream = nullptr, d2h = nullptr;
    cudaEvent_t slice_go = nullptr, slices_done = nullptr, ev_slice[kMaxSlices] = {};
    int64_t* slice_info = nullptr;  // host-mapped [2 * kMaxSlices]: (first byte, bytes)
    int64_t runs_estimate = 0;      // run bytes of the last sliced call (staging size)

    void init(int dev) {
        device = dev;
        SG_CUDA_CHECK(cudaSetDevice(dev));
        SG_CUDA_CHECK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        SG_CUDA_CHECK(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
        SG_CUDA_CHECK(cudaStreamCreateWithFlags(&copy, cudaStreamNonBlocking));
        SG_CUDA_CHECK(cudaEventCreateWithFlags(&copy_go, cudaEventDisableTiming));
        SG_CUDA_CHECK(cudaEventCreateWithFlags(&copy_done, cudaEventDisableTiming));
        SG_CUDA_CHECK(cudaStreamCreateWithFlags(&slice_stream, cudaStreamNonBlocking));
        SG_CUDA_CHECK(cudaStreamCreateWithFlags(&d2h, cudaStreamNonBlocking));
        SG_CUDA_CHECK(cudaEventCreateWithFlags(&slice_go, cudaEventDisableTiming));
        SG_CUDA_CHECK(cudaEventCreateWithFlags(&slices_done, cudaEventDisableTiming));
        SG_CUDA_CHECK(cudaEventCreateWithFlags(&k1_done, cudaEventDisableTiming));
        for (auto& e : ev_slice) SG_CUDA_CHECK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        void* info = nullptr;
        SG_CUDA_CHECK(cudaHostAlloc(&info, 16 * kMaxSlices, cudaHostAllocMapped | cudaHostAllocPortable));
        slice_info = static_cast<int64_t*>(info);
        for (auto& e : ev) SG_CUDA_CHECK(cudaEventCreate(&e));
    }
    ~DevState() {
        if (!stream) return;
        cudaSetDevice(device);
        for (DevBuf* b : {&seq, &nmask, &text_off, &pat_off, &text_len, &pat_len, &has_n, &order,
                          &distance, &windows, &status, &out_bytes, &counters, &bound_off,
                          &scratch, &bnd, &next_pair, &ready, &bnd_ones, &bnd_zeros, &dense_off,
                          &dense, &scan_tmp, &ex_store, &ex_hbuf, &ex_store_off, &ex_hbuf_off,
                          &q_band, &q_full, &q_coop, &q_std, &mixed_ctr, &resume_state, &t_list,
                          &u_list, &diag_warp, &diag_phase, &slice_done, &pipe_ctr})
            b->release();
        if (k1_done) cudaEventDestroy(k1_done);
        if (slice_stream) cudaStreamDestroy(slice_stream);
        if (d2h) cudaStreamDestroy(d2h);
        if (slice_go) cudaEventDestroy(slice_go);
        if (slices_done) cudaEventDestroy(slices_done);
        for (auto& e : ev_slice)
            if (e) cudaEventDestroy(e);
        if (slice_info) cudaFreeHost(slice_info);
        if (copy) cudaStreamDestroy(copy);
        if (copy_go) cudaEventDestroy(copy_go);
        if (copy_done) cudaEventDestroy(copy_done);
        for (auto& e : ev)
            if (e) cudaEventDestroy(e);
        cudaStreamDestroy(stream);
    }
};

// One cached pipeline per device for the one-shot calls (serialised per device).
struct DevSlot {
    std::mutex mu;
    std::unique_ptr<DevState> st;
};
// Keyed by (device, occurrence): a device listed twice in one call gets two
// pipelines (own buffers), so shards never share or wait on each other.
// Intentionally leaked: no device teardown races the CUDA runtime at exit.
std::mutex g_slots_mu;
std::vector<std::vector<DevSlot*>>* g_slots = new std::vector<std::vector<DevSlot*>>();

DevSlot& dev_slot(int dev, int occurrence) {
    std::lock_guard<std::mutex> lk(g_slots_mu);
    while (static_cast<int>(g_slots->size()) <= dev) g_slots->emplace_back();
    auto& v = (*g_slots)[static_cast<size_t>(dev)];
    while (static_cast<int>(v.size()) <= occurrence) v.push_back(new DevSlot());
    return *v[static_cast<size_t>(occurrence)];
}

// ------------------------------------------------------------ validation

int limbs_for(int W) { return W <= 32 ? 1 : W <= 64 ? 2 : W <= 128 ? 4 : 0; }

int validate_cfg(const sg_config* c) {
    if (!c) return set_error(SG_CONFIG, "null config");
    // AlignerConfig::validate, proj/src/aligner.cpp:8-18
    if (c->W < 1 || c->W > 1024)
        return set_error(SG_CONFIG, "window size W out of range: %d", c->W);
    if (c->O < 0 || c->O >= c->W)
        return set_error(SG_CONFIG, "window overlap O must satisfy 0 <= O < W, got O=%d W=%d",
                         c->O, c->W);
    if (c->dent && c->single_window)
        return set_error(SG_CONFIG,
                         "trimmed table storage cannot back a full single-window traceback");
    if (c->single_window && (c->k_single < 0 || c->k_single > 1024))
        return set_error(SG_CONFIG, "k out of range: %d", c->k_single);
    return SG_OK;
}

constexpr int64_t kMaxSingle = 1024;     // BitVector::kMaxBits (bitvec.hpp:29)

// Host loops over the pairs run on several threads from this batch size on (a
// cfg2-sized call has 1 M pairs: each serial pass over them costs 1-7 ms).
constexpr int64_t kParGrain = 8192;

int validate_lengths(int64_t n, const int64_t* tl, const int64_t* pl, const sg_config* c) {
    // kind of the first (lowest-index) bad pair: 1 empty, 2 too long, 3 single-window cap
    auto check = [&](int64_t k) -> int {
        if (tl[k] <= 0 || pl[k] <= 0) return 1;  // batch.cpp:18-25
        if (tl[k] + pl[k] > (int64_t{1} << 30)) return 2;
        // aligner.cpp:92-94; run_batch reports it as an input error (batch.cpp:94-97)
        if (c->single_window && (tl[k] > kMaxSingle || pl[k] > kMaxSingle)) return 3;
        return 0;
    };
    std::vector<int64_t> first(64, INT64_MAX);
    parallel_for(n, [&](int64_t lo, int64_t hi, int t) {
        for (int64_t k = lo; k < hi; ++k)
            if (check(k)) {
                first[static_cast<size_t>(t)] = k;
                break;
            }
    }, kParGrain);
    const int64_t bad = *std::min_element(first.begin(), first.end());
    if (bad == INT64_MAX) return SG_OK;
    switch (check(bad)) {
        case 1: return set_error(SG_INPUT, "pair '%lld': empty sequence", static_cast<long long>(bad));
        case 2: return set_error(SG_INPUT, "pair '%lld': sequence too long for one GPU pair slot",
                                 static_cast<long long>(bad));
        default: return set_error(SG_INPUT,
                                  "pair '%lld': single-window mode requires sequences of at most "
                                  "1024 characters", static_cast<long long>(bad));
    }
}

// ------------------------------------------------------------ packing (K4)

// Owned packed batch (pinned, so it can be uploaded at full PCIe rate).
struct Packed {
    PinBuf seq, nmask, text_off, text_len, pat_off, pat_len;
    int64_t n_pairs = 0, seq_words = 0;
    bool any_n = false;
    sg_packed_pairs view() const {
        sg_packed_pairs v{};
        v.n_pairs = n_pairs;
        v.seq = seq.as<uint32_t>();
        v.seq_words = seq_words;
        v.nmask = any_n ? nmask.as<uint32_t>() : nullptr;
        v.text_off = text_off.as<int64_t>();
        v.text_len = text_len.as<int64_t>();
        v.pat_off = pat_off.as<int64_t>();
        v.pat_len = pat_len.as<int64_t>();
        return v;
    }
};

std::mutex g_owned_mu;
std::vector<Packed*>& packed_registry() {
    static auto* r = new std::vector<Packed*>();
    return *r;
}

// Pack one sequence of 1-byte codes into 16-base words; returns true if it
// holds a non-ACGT code (then nm, if given, receives its bits).
bool pack_seq(const uint8_t* src, int64_t len, uint32_t* dst, uint32_t* nm, int64_t base) {
    const int64_t words = (len + 15) / 16;
    bool n = false;
    int64_t k = 0;
    for (int64_t w = 0; w < words; ++w) {
        uint32_t v = 0;
        const int64_t hi = std::min(len, k + 16);
        for (int sh = 0; k < hi; ++k, sh += 2) {
            const uint32_t c = src[k];
            n |= c >= 4;
            v |= (c & 3u) << sh;
        }
        dst[w] = v;
    }
    if (n && nm)
        for (int64_t i = 0; i < len; ++i)
            if (src[i] >= 4) {
                const int64_t b = base + i;
                __atomic_fetch_or(&nm[b >> 5], 1u << (b & 31), __ATOMIC_RELAXED);
            }
    return n;
}

void layout_offsets(Packed& pk, int64_t n, const int64_t* tl, const int64_t* pl) {
    pk.n_pairs = n;
    const size_t n1 = static_cast<size_t>(std::max<int64_t>(n, 1));
    pk.text_off.ensure(8 * n1);
    pk.text_len.ensure(8 * n1);
    pk.pat_off.ensure(8 * n1);
    pk.pat_len.ensure(8 * n1);
    int64_t words = 0;
    for (int64_t k = 0; k < n; ++k) {
        pk.text_off.as<int64_t>()[k] = words * 16;
        pk.text_len.as<int64_t>()[k] = tl[k];
        words += (tl[k] + 15) / 16;
        pk.pat_off.as<int64_t>()[k] = words * 16;
        pk.pat_len.as<int64_t>()[k] = pl[k];
        words += (pl[k] + 15) / 16;
    }
    pk.seq_words = words;
    pk.seq.ensure(4 * static_cast<size_t>(words + 1));
    pk.seq.as<uint32_t>()[words] = 0;
}

void pack_pairs(const sg_pairs* in, Packed& pk) {
    const int64_t n = in->n_pairs;
    layout_offsets(pk, n, in->text_len, in->pat_len);
    std::atomic<bool> any{false};
    parallel_for(n, [&](int64_t lo, int64_t hi, int) {
        bool a = false;
        for (int64_t k = lo; k < hi && !a; ++k) {
            const uint8_t* t = in->text + in->text_off[k];
            const uint8_t* p = in->pattern + in->pat_off[k];
            for (int64_t i = 0; i < in->text_len[k] && !a; ++i) a = t[i] >= 4;
            for (int64_t i = 0; i < in->pat_len[k] && !a; ++i) a = p[i] >= 4;
        }
        if (a) any = true;
    });
    pk.any_n = any.load();
    uint32_t* nm = nullptr;
    if (pk.any_n) {
        const size_t nm_words = static_cast<size_t>((pk.seq_words * 16 + 31) / 32 + 2);
        pk.nmask.ensure(4 * nm_words);
        nm = pk.nmask.as<uint32_t>();
        std::memset(nm, 0, 4 * nm_words);
    }
    uint32_t* seq = pk.seq.as<uint32_t>();
    parallel_for(n, [&](int64_t lo, int64_t hi, int) {
        for (int64_t k = lo; k < hi; ++k) {
            const int64_t to = pk.text_off.as<int64_t>()[k], po = pk.pat_off.as<int64_t>()[k];
            pack_seq(in->text + in->text_off[k], in->text_len[k], seq + to / 16, nm, to);
            pack_seq(in->pattern + in->pat_off[k], in->pat_len[k], seq + po / 16, nm, po);
        }
    });
}

// ------------------------------------------------------------ results

struct ResultOwner {
    PinBuf distance, windows, found, cigar_off, runs, counters;
};

// `staged`: a pinned buffer that already holds the run bytes (the sliced D2H);
// the result takes it over instead of allocating its own.
void results_alloc(sg_results* out, int64_t n, int64_t run_bytes, PinBuf* staged = nullptr) {
    auto own = std::make_unique<ResultOwner>();
    const size_t n1 = static_cast<size_t>(std::max<int64_t>(n, 1));
    own->distance.ensure(8 * n1);
    own->windows.ensure(4 * n1);
    own->found.ensure(n1);
    own->cigar_off.ensure(8 * (n1 + 1));
    if (staged && staged->p) {
        std::swap(own->runs.p, staged->p);
        std::swap(own->runs.cap, staged->cap);
    }
    own->runs.ensure(static_cast<size_t>(std::max<int64_t>(run_bytes, 1)));
    own->counters.ensure(8 * SG_CNT_COUNT * n1);
    std::memset(out, 0, sizeof *out);
    out->n_pairs = n;
    out->distance = own->distance.as<int64_t>();
    out->windows = own->windows.as<int32_t>();
    out->found = own->found.as<uint8_t>();
    out->cigar_off = own->cigar_off.as<int64_t>();
    out->runs = own->runs.as<uint8_t>();
    out->counters = own->counters.as<uint64_t>();
    out->cigar_off[0] = 0;
    out->_owner = own.release();
}

// ------------------------------------------------------------ one shard

struct Shard {
    const sg_packed_pairs* in;
    int64_t lo, hi;
};

// Whether the mixed kernel (band frame first, §3.8-3.10) pays for this shard.
// It wins when pairs are long (most windows are band windows: cfg3 1.50x, cfg4 up
// to 2x) and loses when most windows are final / tail windows (cfg1, cfg2: short
// reads, 4x) or when many pairs are unrelated (cfg5: they leave the band frame at
// once). Decided per shard from the mean window count per pair and the unrelated
// fraction of a strided sample of <= 64 pairs (exact 8-base blocks of the first
// 256 text bases found in the pattern within +-16 diagonals: correlated reads give
// ~8, unrelated ones ~0.02; the sample costs ~0.1 ms of host time per call). Only the choice of kernel depends on it, never a result.
uint32_t bases8(const uint32_t* seq, int64_t a) {  // 8 bases (16 bits) from base a on
    const uint64_t w = static_cast<uint64_t>(seq[a >> 4]) | (static_cast<uint64_t>(seq[(a >> 4) + 1]) << 32);
    return static_cast<uint32_t>(w >> (2 * (a & 15))) & 0xFFFFu;
}

bool pair_related(const sg_packed_pairs* in, int64_t k, int64_t span = 256, int need = 2) {
    const int64_t n = in->text_len[k], m = in->pat_len[k];
    const int64_t len = std::min<int64_t>(std::min(n, m), span);
    if (len < 128) return true;
    const int64_t ta = in->text_off[k], pa = in->pat_off[k];
    int hits = 0;
    for (int64_t b = 0; b + 8 <= len; b += 8) {
        const uint32_t t = bases8(in->seq, ta + b);
        for (int64_t dl = -16; dl <= 16; ++dl) {
            const int64_t j = b + dl;
            if (j < 0 || j + 8 > m) continue;
            if (bases8(in->seq, pa + j) == t && ++hits >= need) return true;
        }
    }
    return false;
}

bool band_pays(const sg_packed_pairs* in, int64_t lo, int64_t hi, int W, int O) {
    const int kernel = options().kernel;
    if (kernel == SG_KERNEL_MIXED) return true;
    if (kernel == SG_KERNEL_FULL) return false;
    const int64_t n = hi - lo;
    if (n <= 0) return false;
    // the mixed kernel wins unless most pairs are a single final window (they go
    // straight to the full-frame K1 after it) or many are unrelated (K0, §3.10).
    // K1 on one B200, auto -> mixed: cfg2 9.4 -> 5.5 ms, cfg1 0.133 -> 0.103, cfg4 W=32
    // 6.0 -> 5.5; cfg5 (30 % unrelated) stays full frame: 134 against 160 ms
    std::vector<double> part(64, 0.0);
    parallel_for(n, [&](int64_t a, int64_t b, int t) {
        double acc = 0;
        for (int64_t k = lo + a; k < lo + b; ++k)
            acc += static_cast<double>(std::max(in->text_len[k], in->pat_len[k]));
        part[static_cast<size_t>(t)] = acc;
    }, kParGrain);
    double tot = 0;
    for (double v : part) tot += v;
    if (tot / static_cast<double>(n) <= W) return false;
    (void)O;
    const int64_t samples = std::min<int64_t>(n, 64);
    int tested = 0, unrelated = 0;
    for (int64_t i = 0; i < samples; ++i) {
        const int64_t k = lo + i * n / samples;
        if (std::min(in->text_len[k], in->pat_len[k]) < 128) continue;
        ++tested;
        unrelated += !pair_related(in, k);
    }
    return unrelated * 20 <= tested;
}

// Expected edits per window of W columns, from a strided sample of <= 16 pairs: the share
// r of exact 8-base blocks of the first 256 text bases found in the pattern within +-16
// diagonals estimates the per-base identity as r^(1/8) (cfg2, 2 % edits: r ~ 0.85; cfg3,
// 15 %: r ~ 0.27). Only K1 mixed's chunk schedule depends on it (band_subchunks), never
// a result. Returns -1 when no sampled pair is long enough.
double expected_window_edits(const sg_packed_pairs* in, int64_t lo, int64_t hi, int W) {
    const int64_t n = hi - lo;
    const int64_t samples = std::min<int64_t>(n, 16);
    int64_t blocks = 0, hits = 0;
    for (int64_t i = 0; i < samples; ++i) {
        const int64_t k = lo + i * n / samples;
        const int64_t nt = in->text_len[k], m = in->pat_len[k];
        const int64_t len = std::min<int64_t>(std::min(nt, m), 256);
        if (len < 64) continue;
        const int64_t ta = in->text_off[k], pa = in->pat_off[k];
        for (int64_t b = 0; b + 8 <= len; b += 8) {
            const uint32_t t = bases8(in->seq, ta + b);
            ++blocks;
            for (int64_t dl = -16; dl <= 16; ++dl) {
                const int64_t j = b + dl;
                if (j < 0 || j + 8 > m) continue;
                if (bases8(in->seq, pa + j) == t) {
                    ++hits;
                    break;
                }
            }
        }
    }
    if (blocks < 8) return -1.0;
    const double r = std::max(1e-3, static_cast<double>(hits) / static_cast<double>(blocks));
    return W * (1.0 - std::pow(r, 1.0 / 8.0));
}

// K1 mixed's band chunks per phase (§3.8): one 8-row chunk when the windows are expected
// to hold fewer than 4.5 edits and the pairs are at least three windows long, else the
// default two. K1 on one B200, two chunks -> one: cfg2 (1.3 edits expected) 5.52 -> 4.97
// ms, cfg4 W = 32 (3.2) 5.42 -> 4.19; the other way cfg4 W = 64 (6.4) 4.62 -> 4.78, cfg3
// (9.6) 17.7 -> 22.4.
int band_schedule(const sg_packed_pairs* in, int64_t lo, int64_t hi, int W) {
    const int64_t n = hi - lo;
    if (n <= 0) return 0;
    const int64_t samples = std::min<int64_t>(n, 16);
    double len = 0;
    for (int64_t i = 0; i < samples; ++i) {
        const int64_t k = lo + i * n / samples;
        len += static_cast<double>(std::max(in->text_len[k], in->pat_len[k]));
    }
    if (len / static_cast<double>(samples) < 3.0 * W) return 0;
    const double e = expected_window_edits(in, lo, hi, W);
    return e >= 0 && e < 4.5 ? 1 : 0;
}

// Host-side per-pair inputs of a shard: rebased offsets, lengths, bounds, order.
struct ShardPrep {
    PinBuf text_off, pat_off, text_len, pat_len, has_n, bound_off, order;
    int64_t n = 0;
    int64_t word_lo = 0, word_hi = 0;
    int64_t scratch_bytes = 0;
    bool any_n = false;
    bool ordered = false;
};

bool any_bits(const uint32_t* m, int64_t base, int64_t len) {  // any of bits [base, base + len)
    if (len <= 0) return false;
    const int64_t end = base + len;
    int64_t w = base >> 5;
    const int64_t wl = (end - 1) >> 5;
    uint32_t first = ~0u << (base & 31);
    const uint32_t last = ~0u >> (31 - ((end - 1) & 31));
    if (w == wl) return (m[w] & first & last) != 0u;
    if (m[w] & first) return true;
    for (++w; w < wl; ++w)
        if (m[w]) return true;
    return (m[wl] & last) != 0u;
}

// Packed words a shard's pairs use: [lo, hi), lo even (the N mask stays 32-bit
// aligned after rebasing).
void shard_words(const Shard& s, int64_t* lo, int64_t* hi) {
    const sg_packed_pairs* in = s.in;
    std::vector<int64_t> plo(64, INT64_MAX), phi(64, 0);
    parallel_for(s.hi - s.lo, [&](int64_t a, int64_t b, int t) {
        int64_t l = INT64_MAX, h = 0;
        for (int64_t k = s.lo + a; k < s.lo + b; ++k) {
            l = std::min({l, in->text_off[k] >> 4, in->pat_off[k] >> 4});
            h = std::max({h, (in->text_off[k] + in->text_len[k] + 15) >> 4,
                          (in->pat_off[k] + in->pat_len[k] + 15) >> 4});
        }
        plo[static_cast<size_t>(t)] = l;
        phi[static_cast<size_t>(t)] = h;
    }, kParGrain);
    int64_t wlo = *std::min_element(plo.begin(), plo.end());
    int64_t whi = *std::max_element(phi.begin(), phi.end());
    if (s.hi <= s.lo) wlo = whi = 0;
    *lo = wlo & ~int64_t{1};
    *hi = whi;
}

void prep_shard(const Shard& s, ShardPrep& pp, bool longest_first, int64_t split = 0,
                const int64_t* words = nullptr) {
    const sg_packed_pairs* in = s.in;
    const int64_t n = s.hi - s.lo;
    pp.n = n;
    int64_t wlo = 0, whi = 0;
    if (words) {
        wlo = words[0];
        whi = words[1];
    } else {
        shard_words(s, &wlo, &whi);
    }
    pp.word_lo = wlo;
    pp.word_hi = whi;
    const int64_t rebase = wlo * 16;
    const size_t n1 = static_cast<size_t>(std::max<int64_t>(n, 1));
    pp.text_off.ensure(8 * n1);
    pp.pat_off.ensure(8 * n1);
    pp.text_len.ensure(4 * n1);
    pp.pat_len.ensure(4 * n1);
    pp.has_n.ensure(n1);
    pp.bound_off.ensure(8 * n1);
    // run-byte bound of a pair: at most one byte per edit op, ops <= n + m
    auto bound_of = [&](int64_t g) {
        return ((in->text_len[g] + in->pat_len[g] + 3) & ~int64_t{3}) + 4;
    };
    // two passes over contiguous chunks: each chunk's bound total, then its pairs
    // from the chunk's base
    std::vector<int64_t> cbound(65, 0);
    std::vector<uint8_t> cn(64, 0);
    parallel_for(n, [&](int64_t a, int64_t b, int t) {
        int64_t acc = 0;
        for (int64_t k = a; k < b; ++k) acc += bound_of(s.lo + k);
        cbound[static_cast<size_t>(t) + 1] = acc;
    }, kParGrain);
    for (size_t t = 0; t < 64; ++t) cbound[t + 1] += cbound[t];
    parallel_for(n, [&](int64_t a, int64_t b, int t) {
        int64_t bound = cbound[static_cast<size_t>(t)];
        bool any = false;
        for (int64_t k = a; k < b; ++k) {
            const int64_t g = s.lo + k;
            pp.text_off.as<int64_t>()[k] = in->text_off[g] - rebase;
            pp.pat_off.as<int64_t>()[k] = in->pat_off[g] - rebase;
            pp.text_len.as<int32_t>()[k] = static_cast<int32_t>(in->text_len[g]);
            pp.pat_len.as<int32_t>()[k] = static_cast<int32_t>(in->pat_len[g]);
            bool hn = false;
            if (in->nmask)
                hn = any_bits(in->nmask, in->text_off[g], in->text_len[g]) ||
                     any_bits(in->nmask, in->pat_off[g], in->pat_len[g]);
            pp.has_n.as<uint8_t>()[k] = hn;
            any |= hn;
            pp.bound_off.as<int64_t>()[k] = bound;
            bound += bound_of(g);
        }
        cn[static_cast<size_t>(t)] = any;
    }, kParGrain);
    pp.any_n = std::any_of(cn.begin(), cn.end(), [](uint8_t v) { return v != 0; });
    pp.scratch_bytes = cbound[64];
    pp.ordered = longest_first && n > 1 && options().longest_first;
    if (pp.ordered) {
        pp.order.ensure(4 * static_cast<size_t>(n));
        int32_t* o = pp.order.as<int32_t>();
        // Longest first, ties in input order (a stable LSD radix sort on the
        // complemented length key, two 16-bit digits, O(n)). With a split, the
        // pairs before it (the first round of lanes, the first sequence words to
        // arrive in a streamed upload) are ordered among themselves, then the rest.
        auto lpt = [&](int64_t lo, int64_t hi) {
            const int64_t m = hi - lo;
            std::vector<uint32_t> key(static_cast<size_t>(m)), k2(static_cast<size_t>(m));
            std::vector<int32_t> tmp(static_cast<size_t>(m));
            for (int64_t k = 0; k < m; ++k) {
                o[lo + k] = static_cast<int32_t>(lo + k);
                key[k] = ~static_cast<uint32_t>(std::min<int64_t>(
                    in->text_len[s.lo + lo + k] + in->pat_len[s.lo + lo + k], 0xFFFFFFFFll));
            }
            for (int shift = 0; shift < 32; shift += 16) {
                std::vector<int64_t> cnt(65537, 0);
                for (int64_t k = 0; k < m; ++k) ++cnt[((key[k] >> shift) & 0xFFFF) + 1];
                for (int b = 0; b < 65536; ++b) cnt[b + 1] += cnt[b];
                for (int64_t k = 0; k < m; ++k) {
                    const int64_t dst = cnt[(key[k] >> shift) & 0xFFFF]++;
                    tmp[dst] = o[lo + k];
                    k2[dst] = key[k];
                }
                std::copy(tmp.begin(), tmp.end(), o + lo);
                key.swap(k2);
            }
        };
        const int64_t cut = split > 0 && split < n ? split : n;
        lpt(0, cut);
        if (cut < n) lpt(cut, n);
    }
}

struct RunConfig {
    int L, W, O, et, policy, single, k_single;
    bool wide;  // K6 (one warp per pair): windows wider than 128 bits
    bool band;  // K1b band pass first, full-frame K1 resumes what it defers (§3.8)
    int band_sub = 0;  // K1 mixed: band chunks per phase (0: the kernel's default)
    int wcap;   // K6: widest window in columns
};

// Single-window mode sizes the vectors by the longest sequence of the batch.
RunConfig run_config(const sg_config* c, int64_t n = 0, const int64_t* tl = nullptr,
                     const int64_t* pl = nullptr) {
    RunConfig r;
    r.L = limbs_for(c->W);
    r.single = c->single_window ? 1 : 0;
    r.k_single = c->k_single;
    r.wcap = c->W;
    if (r.single) {
        int64_t mx = 1;
        for (int64_t k = 0; k < n; ++k) mx = std::max(mx, std::max(tl[k], pl[k]));
        r.L = limbs_for(static_cast<int>(mx));
        r.wcap = static_cast<int>(mx);
    }
    // K6 takes what K1's limb counts do not cover; SG_KERNEL_WIDE routes every
    // batch through it (tests cross-check the two kernels)
    const int kernel = options().kernel;
    r.wide = r.L == 0 || kernel == SG_KERNEL_WIDE;
    r.W = c->W;
    r.O = c->O;
    r.et = c->early_termination ? 1 : 0;
    r.policy = c->dent ? 2 : c->sene ? 1 : 0;
    // The mixed kernel always stops a window at D(0, 0) (its band frame is exact only
    // up to row 30). Without early termination every window computes all K + 1 rows,
    // as compute_dc does (proj/src/dp.cpp:177,225): the full-frame K1 and K6 do.
    r.band = !r.wide && sgk::band_eligible(r.W, r.O, r.single) && kernel != SG_KERNEL_FULL &&
             c->early_termination;
    return r;
}

// Sequence words go in up to kChunks pieces of at least 2 MB (a small batch is one
// piece: every piece costs two API calls before K1 can launch). Streamed (one-shot calls): the pieces
// go on the copy stream, each followed by its ready flag, while K1 already runs
// on the main stream; a lane waits for the piece holding its pair's last word
// (K1 fetch). Otherwise (sessions) everything is copied and flagged up front.
constexpr int kChunks = 16;
constexpr int64_t kChunkMinWords = int64_t{1} << 19;

// The sequence words (the bulk of the H2D), issued before the host prepares the
// per-pair arrays so that they arrive earlier (one-shot calls stream them, §1).
int64_t upload_seq(DevState& st, const Shard& s, int64_t word_lo, int64_t word_hi, bool streamed) {
    const sg_packed_pairs* in = s.in;
    const int64_t words = word_hi - word_lo;
    int64_t h2d_bytes = 0;
    const size_t seq_bytes = 4 * static_cast<size_t>(words + 48);  // K1 reads up to 12 words past a start, K0 35
    st.seq.ensure(seq_bytes);
    st.ready.ensure(4 * kChunks);
    const int64_t avail = std::max<int64_t>(0, std::min<int64_t>(words + 48, in->seq_words - word_lo));
    st.n_chunks = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(kChunks, avail / kChunkMinWords)));
    st.chunk_words = std::max<int64_t>(1, (avail + st.n_chunks - 1) / st.n_chunks);
    cudaStream_t cs = streamed ? st.copy : st.stream;
    SG_CUDA_CHECK(cudaMemsetAsync(st.ready.p, 0, 4 * kChunks, st.stream));
    if (streamed) {
        SG_CUDA_CHECK(cudaEventRecord(st.copy_go, st.stream));
        SG_CUDA_CHECK(cudaStreamWaitEvent(st.copy, st.copy_go, 0));
    }
    if (static_cast<size_t>(4 * avail) < seq_bytes)
        SG_CUDA_CHECK(cudaMemsetAsync(static_cast<char*>(st.seq.p) + 4 * avail, 0,
                                      seq_bytes - 4 * static_cast<size_t>(avail), cs));
    for (int c = 0; c < st.n_chunks; ++c) {
        const int64_t lo = std::min<int64_t>(avail, c * st.chunk_words);
        const int64_t hi = std::min<int64_t>(avail, lo + st.chunk_words);
        if (hi > lo) {
            SG_CUDA_CHECK(cudaMemcpyAsync(st.seq.as<uint32_t>() + lo, in->seq + word_lo + lo,
                                          4 * static_cast<size_t>(hi - lo), cudaMemcpyHostToDevice, cs));
            h2d_bytes += 4 * (hi - lo);
        }
        SG_CUDA_CHECK(cudaMemsetAsync(st.ready.as<uint32_t>() + c, 1, 4, cs));
    }
    SG_CUDA_CHECK(cudaEventRecord(st.copy_done, cs));
    return h2d_bytes;
}

int64_t upload_shard(DevState& st, const Shard& s, const ShardPrep& pp, bool streamed = false,
                     bool seq_done = false) {
    const int64_t n = pp.n;
    const sg_packed_pairs* in = s.in;
    const int64_t words = pp.word_hi - pp.word_lo;
    int64_t h2d_bytes = seq_done ? 0 : upload_seq(st, s, pp.word_lo, pp.word_hi, streamed);
    if (pp.any_n) {
        const int64_t mlo = pp.word_lo / 2;
        const int64_t mwords = (words + 1) / 2 + 4;
        const int64_t mtot = (in->seq_words * 16 + 31) / 32;
        st.nmask.ensure(4 * static_cast<size_t>(mwords));
        SG_CUDA_CHECK(cudaMemsetAsync(st.nmask.p, 0, 4 * static_cast<size_t>(mwords), st.stream));
        const int64_t ma = std::min<int64_t>(mwords, mtot - mlo);
        if (ma > 0) {
            SG_CUDA_CHECK(cudaMemcpyAsync(st.nmask.p, in->nmask + mlo, 4 * static_cast<size_t>(ma),
                                          cudaMemcpyHostToDevice, st.stream));
            h2d_bytes += 4 * ma;
        }
    }
    const size_t n1 = static_cast<size_t>(std::max<int64_t>(n, 1));
    auto h2d = [&](DevBuf& d, const PinBuf& h, size_t elem) {
        d.ensure(elem * n1);
        if (n) {
            SG_CUDA_CHECK(cudaMemcpyAsync(d.p, h.p, elem * static_cast<size_t>(n),
                                          cudaMemcpyHostToDevice, st.stream));
            h2d_bytes += static_cast<int64_t>(elem) * n;
        }
    };
    h2d(st.text_off, pp.text_off, 8);
    h2d(st.pat_off, pp.pat_off, 8);
    h2d(st.text_len, pp.text_len, 4);
    h2d(st.pat_len, pp.pat_len, 4);
    h2d(st.has_n, pp.has_n, 1);
    h2d(st.bound_off, pp.bound_off, 8);
    if (pp.ordered) h2d(st.order, pp.order, 4);
    return h2d_bytes;
}

// Sizes the per-run buffers and launches K1, K2 (3 kernels) and K3.
// K1 grid for n pairs. Each lane aligns whole pairs one after another, so a
// batch takes about ceil(n / lanes) pair-times. Use the fewest lanes that keep
// that number of rounds (fewer warps per SM run each round faster).
long long k1_grid(const DevState& st, const RunConfig& rc, int64_t n, bool band_pass = false) {
    if (rc.wide) {  // K6: one warp per pair, persistent
        const int wpb = sgk::wide_warps_per_block();
        const long long bps = std::max(1, sgk::wide_max_blocks_per_sm());
        long long warps = std::min<long long>(std::max<int64_t>(n, 1), st.sms * bps * wpb);
        // parked row + events: keep the scratch within 4 GiB
        const long long per = sgk::wide_warp_words(rc.wcap) * 4;
        warps = std::max(1LL, std::min(warps, (4LL << 30) / per));
        return (warps + wpb - 1) / wpb;
    }
    int blocks_per_sm = band_pass ? sgk::mixed_max_blocks_per_sm(rc.L) : sgk::k1_max_blocks_per_sm(rc.L);
    if (blocks_per_sm < 1) blocks_per_sm = 1;
    // mixed: size by the band warps (they take the fresh pairs)
    const int wpb = band_pass ? sgk::mixed_band_warps() : sgk::k1_warps_per_block(rc.L);
    const long long max_grid = static_cast<long long>(st.sms) * blocks_per_sm;
    const long long max_lanes = max_grid * wpb * 32;
    const long long rounds = std::max(1LL, (static_cast<long long>(n) + max_lanes - 1) / max_lanes);
    const long long lanes_needed = (static_cast<long long>(n) + rounds - 1) / rounds;
    long long grid = (lanes_needed + 32LL * wpb - 1) / (32LL * wpb);
    return std::max(1LL, std::min(grid, max_grid));
}

// Band chunks per phase of the tail K1: its STD windows need rows 0..D with D ~ 33-64
// (a text of W bases against <= 31 pattern bases), so every lane runs chunk after chunk
// and the traceback phase waits until the warp has none left to run.
#ifndef SG_TAIL_SUB
#define SG_TAIL_SUB 8
#endif
constexpr int kTailSubChunks = SG_TAIL_SUB;

// K1 mixed: band warps that take pairs, spread over one block per SM; the others
// exit at once. Every slot when there are more pairs than lanes: unlike the
// full-frame kernel, whole rounds do not pay here (cfg3 100k: 3.02 rounds on all
// 1036 warps 28.7 ms, 4 whole rounds on 782 warps 33.7 ms) — the last pairs run
// on nearly idle SMs and hand their tails to the cooperative warps.
long long band_active_warps(const DevState& st, const RunConfig& rc, int64_t n, int sms = 0) {
    (void)rc;
    const long long max_warps = static_cast<long long>(sms > 0 ? sms : st.sms) * sgk::mixed_band_warps();
    const long long w = (static_cast<long long>(n) + 31) / 32;
    return std::max(1LL, std::min(w, max_warps));
}

// Pairs K1 / K6 work on at once (lanes / warps of the grid).
int64_t pairs_in_flight(const DevState& st, const RunConfig& rc, int64_t n) {
    if (rc.band) return band_active_warps(st, rc, n) * 32;
    const long long g = k1_grid(st, rc, n);
    return rc.wide ? g * sgk::wide_warps_per_block() : g * sgk::k1_warps_per_block(rc.L) * 32;
}

// Pipelined launches (§3.12): the SMs K1 mixed leaves to the tail K1 and the full-frame
// K1 of the slices, in proportion to the work they get. In band-window units (cfg3 /
// cfg2 on one B200: 0.096 SM-us per band window) an STD window of a pair's tail costs
// ~7 (D ~ 48 in the 32-bit standard frame) and a final window in the full-frame K1
// ~2.65. From a strided sample of the pairs; only the split depends on it.
int tail_sm_count(const DevState& st, const RunConfig& rc, const ShardPrep& pp) {
    const int64_t n = pp.n;
    const int64_t samples = std::min<int64_t>(n, 4096);
    const double step = std::max(1, rc.W - rc.O);
    double band = 0, tail = 0;
    for (int64_t i = 0; i < samples; ++i) {
        const int64_t k = i * n / samples;
        const double tl = pp.text_len.as<int32_t>()[k], pl = pp.pat_len.as<int32_t>()[k];
        band += std::max(0.0, std::max(tl, pl) - rc.W) / step;
        tail += tl - pl >= 32 ? 7.0 : 2.65;
    }
    const double share = tail / std::max(1.0, band + tail);
    const int t = static_cast<int>(std::ceil(1.1 * share * st.sms));
    return std::max(2, std::min(t, st.sms / 2));
}

// Output slices of a one-shot call (§3.12, §5): `early` slices of `per` pairs, then
// (K1 mixed, pipelined: the pairs of its last round) `late` slices of `per_late` pairs,
// the final one taking the rest.
struct SlicePlan {
    int early = 0, late = 0;
    int32_t per = 0, per_late = 0;
    int total() const { return early + late; }
    int64_t early_pairs(int64_t n) const { return std::min<int64_t>(n, int64_t{early} * per); }
    int64_t lo(int sl, int64_t n) const {
        if (sl < early) return std::min<int64_t>(n, int64_t{sl} * per);
        return std::min<int64_t>(n, early_pairs(n) + int64_t{sl - early} * per_late);
    }
    int64_t hi(int sl, int64_t n) const { return sl == total() - 1 ? n : lo(sl + 1, n); }
};

// Events: ev[0] before K1, ev[1] after K1, ev[2] after K3. Returns launches.
// slices > 0 (one-shot calls): K2/K3 run per slice of `slice_pairs` pairs on the
// slice stream while K1 runs; ev_slice[s] marks slice s's bytes dense on the device.
int launch_shard(DevState& st, const RunConfig& rc, const ShardPrep& pp, const SlicePlan& plan = SlicePlan{}) {
    const int slices = plan.total();
    const int32_t slice_pairs = plan.per;
    const int64_t n = pp.n;
    const size_t n1 = static_cast<size_t>(std::max<int64_t>(n, 1));
    st.distance.ensure(4 * n1);
    st.windows.ensure(4 * n1);
    st.status.ensure(4 * n1);
    st.out_bytes.ensure(4 * n1);
    st.counters.ensure(8 * SG_CNT_COUNT * n1);
    st.scratch.ensure(static_cast<size_t>(pp.scratch_bytes));
    st.next_pair.ensure(64);
    st.dense_off.ensure(8 * (n1 + 1));
    st.dense.ensure(static_cast<size_t>(pp.scratch_bytes));
    st.scan_tmp.ensure(sgk::cigar_offsets_temp_bytes(static_cast<int32_t>(n)) + 64);
    const int wpb = rc.wide ? sgk::wide_warps_per_block() : sgk::k1_warps_per_block(rc.L);
    const long long grid = k1_grid(st, rc, n);
    st.grid = grid;
    st.lanes = grid * wpb * (rc.wide ? 1 : 32);  // pairs in flight
    // pipelined (§3.12): K1 mixed on all SMs but `tsm`, the slices' tail / full-frame K1
    // and K2 / K3 beside it on the slice stream
    const bool piped = rc.band && slices > 0;
    const int tsm = piped ? tail_sm_count(st, rc, pp) : 0;
    st.tail_sms = tsm;
    const long long band_warps = rc.band ? band_active_warps(st, rc, n, st.sms - tsm) : 0;
    const long long grid_band = rc.band ? std::min<long long>(st.sms - tsm, band_warps) : 0;
    if (rc.band) {
        st.lanes = band_warps * 32;
        st.q_band.ensure(4 * (n1 + 32));
        st.q_full.ensure(4 * (n1 + 32));
        st.q_coop.ensure(4 * (n1 + 32));
        st.q_std.ensure(4 * (n1 + 32));
        st.mixed_ctr.ensure(64);
        st.resume_state.ensure(16 * n1);
    }
    st.bnd.ensure(rc.wide ? static_cast<size_t>(sgk::wide_warp_words(rc.wcap)) * 4 * grid * wpb
                          : sgk::bnd_scratch_bytes(rc.L, grid * wpb));
    if (!st.bnd_ones.p) {
        const size_t cb = sgk::bnd_scratch_bytes(4, 1);
        st.bnd_ones.ensure(cb);
        st.bnd_zeros.ensure(cb);
        SG_CUDA_CHECK(cudaMemsetAsync(st.bnd_ones.p, 0xFF, cb, st.stream));
        SG_CUDA_CHECK(cudaMemsetAsync(st.bnd_zeros.p, 0, cb, st.stream));
    }
    SG_CUDA_CHECK(cudaMemsetAsync(st.next_pair.p, 0, 64, st.stream));

    sgk::AlignParams p{};
    p.seq = st.seq.as<uint32_t>();
    p.nmask = pp.any_n ? st.nmask.as<uint32_t>() : nullptr;
    p.text_off = st.text_off.as<int64_t>();
    p.pat_off = st.pat_off.as<int64_t>();
    p.text_len = st.text_len.as<int32_t>();
    p.pat_len = st.pat_len.as<int32_t>();
    p.has_n = pp.any_n ? st.has_n.as<uint8_t>() : nullptr;
    p.order = pp.ordered ? st.order.as<int32_t>() : nullptr;
    p.n_pairs = static_cast<int32_t>(n);
    p.W = rc.W;
    p.O = rc.O;
    p.et = rc.et;
    p.policy = rc.policy;
    p.two = 2;
    p.single = rc.single;
    p.k_single = rc.k_single;
    p.distance = st.distance.as<int32_t>();
    p.windows = st.windows.as<int32_t>();
    p.status = st.status.as<int32_t>();
    p.out_bytes = st.out_bytes.as<int32_t>();
    p.counters = st.counters.as<uint64_t>();
    p.bound_off = st.bound_off.as<int64_t>();
    p.scratch = st.scratch.as<uint32_t>();
    p.bnd = st.bnd.as<uint32_t>();
    p.bnd_ones = st.bnd_ones.as<uint32_t>();
    p.bnd_zeros = st.bnd_zeros.as<uint32_t>();
    p.next_pair = st.next_pair.as<unsigned int>();
    p.ready = st.ready.as<unsigned int>();
    p.chunk_words = st.chunk_words;
    p.n_chunks = st.n_chunks;
    p.wcap = rc.wcap;
    p.phase_cycles = nullptr;
    p.warp_times = nullptr;
    st.diag_flags = options().diagnostics;
    if (st.diag_flags & SG_DIAG_WARP_TIMES) {
        st.diag_warps = static_cast<int>(std::min<long long>(
            8192, rc.band ? grid_band * sgk::mixed_warps_per_block()
                          : grid * wpb));
        st.diag_warp.ensure(8 * 3 * 8192);
        SG_CUDA_CHECK(cudaMemsetAsync(st.diag_warp.p, 0, 8 * 3 * 8192, st.stream));
        p.warp_times = st.diag_warp.as<unsigned long long>();
    }
    if (st.diag_flags & SG_DIAG_PHASE_CYCLES) {
        st.diag_phase.ensure(256);
        SG_CUDA_CHECK(cudaMemsetAsync(st.diag_phase.p, 0, 256, st.stream));
        p.phase_cycles = st.diag_phase.as<unsigned long long>();
    }

    if (slices > 0) {
        st.slice_done.ensure(4 * DevState::kMaxSlices);
        SG_CUDA_CHECK(cudaMemsetAsync(st.slice_done.p, 0, 4 * DevState::kMaxSlices, st.stream));
        SG_CUDA_CHECK(cudaMemsetAsync(st.dense_off.p, 0, 8, st.stream));
        p.slice_done = piped ? nullptr : st.slice_done.as<unsigned int>();
        p.slice_pairs = slice_pairs;
        if (piped) {
            st.pipe_ctr.ensure(4 * DevState::kPipeWords);
            SG_CUDA_CHECK(cudaMemsetAsync(st.pipe_ctr.p, 0, 4 * DevState::kPipeWords, st.stream));
        } else {
            SG_CUDA_CHECK(cudaEventRecord(st.slice_go, st.stream));
        }
    }
    int launches = 0;
    SG_CUDA_CHECK(cudaEventRecord(st.ev[0], st.stream));
    if (n > 0 && rc.band) {
        // K1 mixed: band warps take every pair first; windows the band frame
        // cannot take move with their pair to the block's full-frame warps and
        // back (§3.8)
        p.mixed = 1;
        p.band_active = static_cast<int32_t>(band_warps);
        p.band_subchunks = rc.band_sub;
        p.q_band = st.q_band.as<uint32_t>();
        p.q_full = st.q_full.as<uint32_t>();
        p.q_coop = st.q_coop.as<uint32_t>();
        p.q_std = st.q_std.as<uint32_t>();
        p.remaining = st.mixed_ctr.as<unsigned int>();
        p.resume_state = st.resume_state.as<int32_t>();
        SG_CUDA_CHECK(cudaMemsetAsync(st.q_band.p, 0, st.q_band.cap, st.stream));
        SG_CUDA_CHECK(cudaMemsetAsync(st.q_full.p, 0, st.q_full.cap, st.stream));
        SG_CUDA_CHECK(cudaMemsetAsync(st.q_coop.p, 0, st.q_coop.cap, st.stream));
        SG_CUDA_CHECK(cudaMemsetAsync(st.q_std.p, 0, st.q_std.cap, st.stream));
        SG_CUDA_CHECK(static_cast<cudaError_t>(sgk::launch_queue_init(
            p.q_band, p.q_full, p.q_coop, p.q_std, p.remaining, static_cast<int>(n), nullptr,
            st.stream)));
        // K0 (§3.10): band warps leave unrelated pairs to a full-frame K1 after them
        st.u_list.ensure(4 * n1);
        SG_CUDA_CHECK(cudaMemsetAsync(st.mixed_ctr.as<unsigned int>() + 8, 0, 12, st.stream));
        p.coop_out = st.mixed_ctr.as<unsigned int>() + 9;
        st.t_list.ensure(4 * n1);
        p.t_list = st.t_list.as<int32_t>();
        p.t_count = st.mixed_ctr.as<unsigned int>() + 10;
        p.u_list = st.u_list.as<int32_t>();
        p.u_count = st.mixed_ctr.as<unsigned int>() + 8;
        if (piped) {
            unsigned int* ctr = st.pipe_ctr.as<unsigned int>();
            p.t_count = ctr + DevState::kPipeT;
            p.u_count = ctr + DevState::kPipeU;
            p.body_done = ctr + DevState::kPipeBody;
            p.last_slice = slices - 1;  // (late slices are `per` pairs too: one division per pair)
            p.pipe_err = ctr + DevState::kPipeErr;
            // everything the slice stream's kernels read is set up before they start
            SG_CUDA_CHECK(cudaEventRecord(st.slice_go, st.stream));
            SG_CUDA_CHECK(cudaStreamWaitEvent(st.slice_stream, st.slice_go, 0));
            SG_CUDA_CHECK(static_cast<cudaError_t>(
                sgk::launch_mixed_align(rc.L, p, static_cast<int>(grid_band), st.stream)));
            ++launches;
            const int full_bps = std::max(1, sgk::k1_max_blocks_per_sm(rc.L));
            int64_t* info = nullptr;
            SG_CUDA_CHECK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&info), st.slice_info, 0));
            for (int sl = 0; sl < slices; ++sl) {
                const int32_t lo = static_cast<int32_t>(plan.lo(sl, n));
                const bool last = sl == slices - 1;
                const int32_t hi = static_cast<int32_t>(plan.hi(sl, n));
                // the slice's STD windows, once its pairs have left K1 mixed: on the SMs
                // K1 mixed leaves free (the last slice: on every SM, K1 mixed is ending)
                sgk::AlignParams pt = p;
                pt.warp_times = nullptr;
                pt.mixed = 0;
                pt.body_done = nullptr;
                pt.t_list = nullptr;
                pt.order = st.t_list.as<int32_t>() + lo;
                pt.n_fresh = reinterpret_cast<const int32_t*>(ctr + DevState::kPipeT + sl);
                pt.next_pair = ctr + DevState::kPipeTailQ + sl;
                pt.restore = 1;
                pt.band_active = 0x7FFFFFFF;
                pt.band_subchunks = kTailSubChunks;
                pt.u_list = st.u_list.as<int32_t>() + lo;
                pt.u_count = ctr + DevState::kPipeU + sl;
                pt.wait_count = ctr + DevState::kPipeBody + sl;
                pt.wait_target = static_cast<unsigned>(hi - lo);
                // (slices of the last round: K1 mixed's blocks are leaving, the grids grow
                // towards the whole device)
                int tgrid = last ? st.sms : tsm;
                if (sl >= plan.early && !last)
                    tgrid = tsm + static_cast<int>(static_cast<long long>(st.sms - tsm) * (sl - plan.early + 1) /
                                                   plan.late);
                SG_CUDA_CHECK(static_cast<cudaError_t>(
                    sgk::launch_tail_align(pt, tgrid, st.slice_stream)));
                // then the full-frame K1 over the slice's list: final windows, unrelated pairs
                sgk::AlignParams pu = p;
                pu.warp_times = nullptr;
                pu.mixed = 0;
                pu.body_done = nullptr;
                pu.u_list = nullptr;
                pu.t_list = nullptr;
                pu.order = st.u_list.as<int32_t>() + lo;
                pu.n_fresh = reinterpret_cast<const int32_t*>(ctr + DevState::kPipeU + sl);
                pu.next_pair = ctr + DevState::kPipeFullQ + sl;
                pu.restore = 1;
                const long long gfull = last ? grid : std::min<long long>(grid, static_cast<long long>(tgrid) * full_bps);
                SG_CUDA_CHECK(static_cast<cudaError_t>(
                    sgk::launch_window_align(rc.L, pu, static_cast<int>(gfull), wpb, st.slice_stream)));
                if (last) SG_CUDA_CHECK(cudaEventRecord(st.k1_done, st.slice_stream));
                SG_CUDA_CHECK(static_cast<cudaError_t>(sgk::launch_slice_scan(
                    st.out_bytes.as<int32_t>(), st.dense_off.as<int64_t>(), lo, hi, nullptr, sl, info,
                    st.slice_stream)));
                SG_CUDA_CHECK(static_cast<cudaError_t>(sgk::launch_slice_compact(
                    st.scratch.as<uint32_t>(), st.bound_off.as<int64_t>(), st.dense_off.as<int64_t>(),
                    st.out_bytes.as<int32_t>(), st.dense.as<uint8_t>(), lo, hi, st.slice_stream)));
                SG_CUDA_CHECK(cudaEventRecord(st.ev_slice[sl], st.slice_stream));
                launches += hi > lo ? 4 : 3;
            }
            SG_CUDA_CHECK(cudaEventRecord(st.slices_done, st.slice_stream));
            SG_CUDA_CHECK(cudaStreamWaitEvent(st.stream, st.k1_done, 0));
            SG_CUDA_CHECK(cudaEventRecord(st.ev[1], st.stream));
            SG_CUDA_CHECK(cudaStreamWaitEvent(st.stream, st.copy_done, 0));
            SG_CUDA_CHECK(cudaStreamWaitEvent(st.stream, st.slices_done, 0));
            SG_CUDA_CHECK(cudaEventRecord(st.ev[2], st.stream));
            return launches + 1;  // + the queue init
        }
        SG_CUDA_CHECK(static_cast<cudaError_t>(
            sgk::launch_mixed_align(rc.L, p, static_cast<int>(grid_band), st.stream)));
        // the tail K1: the pairs' STD windows in the band warps' single-word frame
        sgk::AlignParams pt = p;
        pt.warp_times = nullptr;
        pt.mixed = 0;
        pt.t_list = nullptr;
        pt.order = st.t_list.as<int32_t>();
        pt.n_fresh = reinterpret_cast<const int32_t*>(p.t_count);
        pt.next_pair = st.next_pair.as<unsigned int>() + 4;
        pt.restore = 1;
        pt.band_active = 0x7FFFFFFF;
        pt.band_subchunks = kTailSubChunks;  // (STD windows: D ~ 48, rows 0..D in one phase)
        SG_CUDA_CHECK(static_cast<cudaError_t>(
            sgk::launch_tail_align(pt, static_cast<int>(st.sms), st.stream)));
        sgk::AlignParams pu = p;
        pu.warp_times = nullptr;
        pu.mixed = 0;
        pu.u_list = nullptr;
        pu.order = st.u_list.as<int32_t>();
        pu.n_fresh = reinterpret_cast<const int32_t*>(p.u_count);
        pu.restore = 1;  // unrelated pairs from their start, the others from their tail
        pu.next_pair = st.next_pair.as<unsigned int>() + 8;
        SG_CUDA_CHECK(static_cast<cudaError_t>(
            sgk::launch_window_align(rc.L, pu, static_cast<int>(grid), wpb, st.stream)));
        launches += 4;
    } else if (n > 0) {
        SG_CUDA_CHECK(static_cast<cudaError_t>(
            rc.wide ? sgk::launch_wide_align(p, static_cast<int>(grid), st.stream)
                    : sgk::launch_window_align(rc.L, p, static_cast<int>(grid), wpb, st.stream)));
        ++launches;
    }
    SG_CUDA_CHECK(cudaEventRecord(st.ev[1], st.stream));
    // trailing pieces of a streamed upload no pair waited for finish before the call does
    SG_CUDA_CHECK(cudaStreamWaitEvent(st.stream, st.copy_done, 0));
    if (slices > 0) {
        SG_CUDA_CHECK(cudaStreamWaitEvent(st.slice_stream, st.slice_go, 0));
        for (int sl = 0; sl < slices; ++sl) {
            const int32_t lo = static_cast<int32_t>(plan.lo(sl, n));
            const int32_t hi = static_cast<int32_t>(plan.hi(sl, n));
            int64_t* info = nullptr;
            SG_CUDA_CHECK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&info), st.slice_info, 0));
            SG_CUDA_CHECK(static_cast<cudaError_t>(sgk::launch_slice_scan(
                st.out_bytes.as<int32_t>(), st.dense_off.as<int64_t>(), lo, hi,
                st.slice_done.as<unsigned>(), sl, info, st.slice_stream)));
            SG_CUDA_CHECK(static_cast<cudaError_t>(sgk::launch_slice_compact(
                st.scratch.as<uint32_t>(), st.bound_off.as<int64_t>(), st.dense_off.as<int64_t>(),
                st.out_bytes.as<int32_t>(), st.dense.as<uint8_t>(), lo, hi, st.slice_stream)));
            SG_CUDA_CHECK(cudaEventRecord(st.ev_slice[sl], st.slice_stream));
            launches += hi > lo ? 2 : 1;
        }
        SG_CUDA_CHECK(cudaEventRecord(st.slices_done, st.slice_stream));
        SG_CUDA_CHECK(cudaStreamWaitEvent(st.stream, st.slices_done, 0));
        SG_CUDA_CHECK(cudaEventRecord(st.ev[2], st.stream));
        return launches;
    }
    SG_CUDA_CHECK(static_cast<cudaError_t>(sgk::launch_cigar_offsets(
        st.out_bytes.as<int32_t>(), st.dense_off.as<int64_t>(), static_cast<int32_t>(n),
        st.scan_tmp.p, st.scan_tmp.cap, st.stream)));
    launches += n > 0 ? 3 : 0;
    SG_CUDA_CHECK(static_cast<cudaError_t>(sgk::launch_cigar_compact(
        st.scratch.as<uint32_t>(), st.bound_off.as<int64_t>(), st.dense_off.as<int64_t>(),
        st.out_bytes.as<int32_t>(), st.dense.as<uint8_t>(), static_cast<int32_t>(n), st.stream)));
    launches += n > 0 ? 1 : 0;
    SG_CUDA_CHECK(cudaEventRecord(st.ev[2], st.stream));
    return launches;
}

// Small per-pair outputs of a shard, staged in pinned memory.
struct ShardOut {
    PinBuf dist, win, status, doff, cnt, pipe_err;
    PinBuf runs;          // sliced calls: the run bytes, already copied out
    bool staged = false;
    int64_t run_bytes = 0;
    float device_ms = 0, k1_ms = 0;
    int launches = 0;
    int err = SG_OK;
    std::string msg;
    int64_t first_bad = -1;
    int32_t first_bad_status = 0;
    int64_t h2d_bytes = 0, d2h_bytes = 0;
};

thread_local const std::chrono::steady_clock::time_point* g_trace_t0 = nullptr;  // SG_DIAG_HOST_TRACE
void trace_point(const char* what) {
    if (g_trace_t0)
        std::fprintf(stderr, "[sg trace] %-10s %8.2f ms\n", what,
                     std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - *g_trace_t0).count());
}

// Issues the D2H of a shard's small per-pair outputs on its main stream (they wait
// for every kernel there); fetch_small_finish waits for them.
void fetch_small_issue(DevState& st, int64_t n, ShardOut& so) {
    const size_t n1 = static_cast<size_t>(std::max<int64_t>(n, 1));
    so.dist.ensure(4 * n1);
    so.win.ensure(4 * n1);
    so.status.ensure(4 * n1);
    so.doff.ensure(8 * (n1 + 1));
    so.cnt.ensure(8 * SG_CNT_COUNT * n1);
    auto d2h = [&](PinBuf& h, const DevBuf& d, size_t bytes) {
        if (bytes) {
            SG_CUDA_CHECK(cudaMemcpyAsync(h.p, d.p, bytes, cudaMemcpyDeviceToHost, st.stream));
            so.d2h_bytes += static_cast<int64_t>(bytes);
        }
    };
    const size_t un = static_cast<size_t>(n);
    d2h(so.dist, st.distance, 4 * un);
    d2h(so.win, st.windows, 4 * un);
    d2h(so.status, st.status, 4 * un);
    d2h(so.doff, st.dense_off, 8 * (un + 1));
    d2h(so.cnt, st.counters, 8 * SG_CNT_COUNT * un);
    so.pipe_err.ensure(4);
    *so.pipe_err.as<unsigned>() = 0;
    if (st.tail_sms > 0)
        SG_CUDA_CHECK(cudaMemcpyAsync(so.pipe_err.p, st.pipe_ctr.as<unsigned>() + DevState::kPipeErr, 4,
                                      cudaMemcpyDeviceToHost, st.stream));
}

void fetch_small_finish(DevState& st, int64_t n, ShardOut& so) {
    SG_CUDA_CHECK(cudaStreamSynchronize(st.stream));
    trace_point("small d2h");
    if (*so.pipe_err.as<unsigned>()) {
        set_error(SG_INTERNAL, "device pipeline: a slice's tail launch timed out waiting for K1 mixed");
        throw Fail{SG_INTERNAL};
    }
    so.run_bytes = so.doff.as<int64_t>()[n];
    std::vector<int64_t> bad(64, INT64_MAX);
    parallel_for(n, [&](int64_t lo, int64_t hi, int t) {
        const int32_t* stp = so.status.as<int32_t>();
        for (int64_t k = lo; k < hi; ++k)
            if (stp[k] != 0) {
                bad[static_cast<size_t>(t)] = k;
                break;
            }
    }, kParGrain);
    const int64_t fb = *std::min_element(bad.begin(), bad.end());
    if (fb != INT64_MAX) {
        so.first_bad = fb;
        so.first_bad_status = so.status.as<int32_t>()[fb];
    }
    float ms = 0, k1 = 0;
    SG_CUDA_CHECK(cudaEventElapsedTime(&ms, st.ev[0], st.ev[2]));
    SG_CUDA_CHECK(cudaEventElapsedTime(&k1, st.ev[0], st.ev[1]));
    so.device_ms = ms;
    so.k1_ms = k1;
}

void fetch_small(DevState& st, int64_t n, ShardOut& so) {
    fetch_small_issue(st, n, so);
    fetch_small_finish(st, n, so);
}

// The sliced D2H (§5): slice by slice, as soon as K2/K3 have made its bytes dense,
// the run bytes go to a pinned staging buffer on the d2h stream, overlapping K1.
// The buffer is sized from the last call (grown, rarely, when a batch needs more);
// the result takes it over.
void stream_runs(DevState& st, int slices, int64_t bound_total, ShardOut& o) {
    int64_t want = st.runs_estimate > 0 ? st.runs_estimate + st.runs_estimate / 8 + (int64_t{1} << 20)
                                        : std::max<int64_t>(int64_t{64} << 20, bound_total / 4);
    want = std::max<int64_t>(1, std::min(want, bound_total));
    o.runs.ensure(static_cast<size_t>(want));
    int64_t end = 0;
    for (int sl = 0; sl < slices; ++sl) {
        SG_CUDA_CHECK(cudaEventSynchronize(st.ev_slice[sl]));
        if (sl == slices - 1) trace_point("last k3");
        const volatile int64_t* info = st.slice_info;
        const int64_t base = info[2 * sl], bytes = info[2 * sl + 1];
        if (base + bytes > static_cast<int64_t>(o.runs.cap)) {
            SG_CUDA_CHECK(cudaStreamSynchronize(st.d2h));
            PinBuf bigger;
            bigger.ensure(static_cast<size_t>(std::max(bound_total, base + bytes)));
            if (base) std::memcpy(bigger.p, o.runs.p, static_cast<size_t>(base));
            std::swap(bigger.p, o.runs.p);
            std::swap(bigger.cap, o.runs.cap);
        }
        if (bytes)
            SG_CUDA_CHECK(cudaMemcpyAsync(o.runs.as<uint8_t>() + base, st.dense.as<uint8_t>() + base,
                                          static_cast<size_t>(bytes), cudaMemcpyDeviceToHost, st.d2h));
        end = base + bytes;
    }
    SG_CUDA_CHECK(cudaStreamSynchronize(st.d2h));
    st.runs_estimate = end;
    o.staged = true;
    o.d2h_bytes += end;
}

const char* status_detail(int32_t s) {
    switch (s & ~0xFFFF) {
        case sgk::kDetBudgetI: return "traceback: budget != remaining pattern";
        case sgk::kDetBudgetD: return "traceback: budget != remaining text";
        case sgk::kDetLeftover: return "traceback: finished with leftover budget";
        case sgk::kDetWatchdog: return "windowed alignment: window count exceeded watchdog cap";
        case sgk::kDetNoStep: return "traceback: no legal step";
        case sgk::kDetSegment: return "window continuation disagrees with the traceback budget";
        default: return "internal error";
    }
}

// Copies a shard's small outputs into the public result at pair `base`.
void scatter_small(sg_results* out, int64_t base, int64_t n, int64_t run_base, const ShardOut& so) {
    const int32_t* dist = so.dist.as<int32_t>();
    const int32_t* win = so.win.as<int32_t>();
    const int64_t* doff = so.doff.as<int64_t>();
    parallel_for(n, [&](int64_t lo, int64_t hi, int) {
        for (int64_t k = lo; k < hi; ++k) {
            out->distance[base + k] = dist[k];
            out->windows[base + k] = win[k];
            out->found[base + k] = dist[k] >= 0;  // single window: D > k is "not found"
            out->cigar_off[base + k] = run_base + doff[k];
        }
        std::memcpy(out->counters + (base + lo) * SG_CNT_COUNT, so.cnt.as<uint64_t>() + lo * SG_CNT_COUNT,
                    8 * SG_CNT_COUNT * static_cast<size_t>(hi - lo));
    }, kParGrain);
    out->cigar_off[base + n] = run_base + doff[n];
}

void finish_totals(sg_results* out) {
    std::vector<uint64_t> part(64 * SG_CNT_COUNT, 0);
    parallel_for(out->n_pairs, [&](int64_t lo, int64_t hi, int t) {
        uint64_t acc[SG_CNT_COUNT] = {};
        for (int64_t k = lo; k < hi; ++k)
            for (int c = 0; c < SG_CNT_COUNT; ++c) acc[c] += out->counters[k * SG_CNT_COUNT + c];
        for (int c = 0; c < SG_CNT_COUNT; ++c) part[static_cast<size_t>(t) * SG_CNT_COUNT + c] = acc[c];
    }, kParGrain);
    for (int c = 0; c < SG_CNT_COUNT; ++c) {
        out->total[c] = 0;
        for (size_t t = 0; t < 64; ++t) out->total[c] += part[t * SG_CNT_COUNT + c];
    }
}

// ------------------------------------------------------------ K5: shards over devices

// Estimated alignment cost of a pair for the device split: its length times the
// rows per window. An unrelated pair (cfg5's independent 30 %) runs ~36 rows per
// window against ~8 for a correlated read, ~4.7x the work.
constexpr float kUnrelatedCost = 4.7f;

// How the pairs of one call go to the devices. Pairs are
// independent, so there is no exchange and no collective: each device aligns its
// shard and the host puts the results back in input order (batch.cpp:28,45).
//  * one device, or pairs of near-equal length and relatedness (cfg2/3/4): contiguous
//    ranges of input order with balanced estimated cost, read in place;
//  * otherwise (cfg5's mix of 100..20k bp, 30 % unrelated): the pairs are sorted
//    into cost buckets (4 per octave, longest first, input order inside a bucket)
//    and dealt longest-processing-time-first to the least-loaded device; each
//    device's members are gathered into one packed batch, and the permutation
//    puts the results back.
struct ShardPlan {
    std::vector<int64_t> cut;                   // contiguous: shard d = [cut[d], cut[d+1])
    std::vector<std::vector<int64_t>> members;  // gathered: input indices of shard d, in order
    bool gathered = false;
};

ShardPlan plan_shards(const sg_packed_pairs* in, size_t nd) {
    ShardPlan plan;
    const int64_t n = in->n_pairs;
    plan.cut.assign(nd + 1, n);
    plan.cut[0] = 0;
    if (nd == 1 || n == 0) return plan;
    std::vector<float> cost(static_cast<size_t>(n));
    std::atomic<int64_t> unrelated{0};
    parallel_for(n, [&](int64_t lo, int64_t hi, int) {
        int64_t u = 0;
        for (int64_t k = lo; k < hi; ++k) {
            const bool rel = pair_related(in, k, 128, 1);
            u += !rel;
            cost[static_cast<size_t>(k)] =
                static_cast<float>(in->text_len[k] + in->pat_len[k]) * (rel ? 1.f : kUnrelatedCost);
        }
        unrelated += u;
    }, 4096);
    const auto mm = std::minmax_element(cost.begin(), cost.end());
    if (*mm.second <= 1.25f * *mm.first) {
        double total = 0;
        for (float c : cost) total += c;
        double acc = 0;
        size_t d = 1;
        for (int64_t k = 0; k < n && d < nd; ++k) {
            acc += cost[static_cast<size_t>(k)];
            while (d < nd && acc * static_cast<double>(nd) >= total * static_cast<double>(d))
                plan.cut[d++] = k + 1;
        }
        return plan;
    }
    plan.gathered = true;
    // buckets: 4 per octave of estimated cost, most expensive first (stable counting sort)
    constexpr int kBuckets = 4 * 40;
    std::vector<int> bucket(static_cast<size_t>(n));
    std::vector<int64_t> start(kBuckets + 1, 0);
    for (int64_t k = 0; k < n; ++k) {
        const int b = std::min(kBuckets - 1, std::max(0, static_cast<int>(4.0f * std::log2(
                                                      std::max(1.0f, cost[static_cast<size_t>(k)])))));
        bucket[static_cast<size_t>(k)] = kBuckets - 1 - b;
        ++start[static_cast<size_t>(kBuckets - b)];
    }
    for (int b = 0; b < kBuckets; ++b) start[b + 1] += start[b];
    std::vector<int64_t> sorted(static_cast<size_t>(n));
    for (int64_t k = 0; k < n; ++k) sorted[static_cast<size_t>(start[bucket[static_cast<size_t>(k)]]++)] = k;
    // LPT over the bucket order
    plan.members.assign(nd, {});
    std::vector<double> load(nd, 0.0);
    for (int64_t k : sorted) {
        const size_t d = static_cast<size_t>(std::min_element(load.begin(), load.end()) - load.begin());
        plan.members[d].push_back(k);
        load[d] += cost[static_cast<size_t>(k)];
    }
    return plan;
}

// Copies `len` bases starting at base `off` of src into dst from its base 0.
void copy_bases(const uint32_t* src, int64_t src_words, int64_t off, int64_t len, uint32_t* dst) {
    const int64_t words = (len + 15) / 16;
    const int64_t w0 = off >> 4;
    const int sh = static_cast<int>(2 * (off & 15));
    if (sh == 0) {
        std::memcpy(dst, src + w0, 4 * static_cast<size_t>(words));
    } else {
        for (int64_t w = 0; w < words; ++w) {
            const uint32_t lo = src[w0 + w] >> sh;
            const uint32_t hi = w0 + w + 1 < src_words ? src[w0 + w + 1] << (32 - sh) : 0u;
            dst[w] = lo | hi;
        }
    }
    if (len & 15) dst[words - 1] &= (1u << (2 * (len & 15))) - 1u;
}

// Packs the members of a gathered shard into one batch (pinned, word-aligned).
void gather_shard(const sg_packed_pairs* in, const std::vector<int64_t>& mem, Packed& pk) {
    const int64_t n = static_cast<int64_t>(mem.size());
    std::vector<int64_t> tl(static_cast<size_t>(n)), pl(static_cast<size_t>(n));
    for (int64_t k = 0; k < n; ++k) {
        tl[static_cast<size_t>(k)] = in->text_len[mem[static_cast<size_t>(k)]];
        pl[static_cast<size_t>(k)] = in->pat_len[mem[static_cast<size_t>(k)]];
    }
    layout_offsets(pk, n, tl.data(), pl.data());
    uint32_t* seq = pk.seq.as<uint32_t>();
    const int64_t* to = pk.text_off.as<int64_t>();
    const int64_t* po = pk.pat_off.as<int64_t>();
    std::vector<uint8_t> hn(static_cast<size_t>(n), 0);
    bool any_n = false;
    for (int64_t k = 0; k < n; ++k) {
        const int64_t g = mem[static_cast<size_t>(k)];
        copy_bases(in->seq, in->seq_words, in->text_off[g], in->text_len[g], seq + to[k] / 16);
        copy_bases(in->seq, in->seq_words, in->pat_off[g], in->pat_len[g], seq + po[k] / 16);
        if (in->nmask && (any_bits(in->nmask, in->text_off[g], in->text_len[g]) ||
                          any_bits(in->nmask, in->pat_off[g], in->pat_len[g]))) {
            hn[static_cast<size_t>(k)] = 1;
            any_n = true;
        }
    }
    pk.any_n = any_n;
    if (!any_n) return;
    const size_t nm_words = static_cast<size_t>((pk.seq_words * 16 + 31) / 32 + 2);
    pk.nmask.ensure(4 * nm_words);
    uint32_t* nm = pk.nmask.as<uint32_t>();
    std::memset(nm, 0, 4 * nm_words);
    auto copy_bits = [&](int64_t src, int64_t len, int64_t dst) {
        for (int64_t i = 0; i < len; ++i)
            if ((in->nmask[(src + i) >> 5] >> ((src + i) & 31)) & 1u)
                nm[(dst + i) >> 5] |= 1u << ((dst + i) & 31);
    };
    for (int64_t k = 0; k < n; ++k) {
        if (!hn[static_cast<size_t>(k)]) continue;
        const int64_t g = mem[static_cast<size_t>(k)];
        copy_bits(in->text_off[g], in->text_len[g], to[k]);
        copy_bits(in->pat_off[g], in->pat_len[g], po[k]);
    }
}

// All device threads of a call meet here between the kernels and the result copy;
// the last to arrive runs `on_last` (sizes and allocates the result) for all of them.
class Rendezvous {
  public:
    explicit Rendezvous(size_t n) : count_(n) {}
    template <class F> void arrive(F&& on_last) {
        std::unique_lock<std::mutex> lk(mu_);
        if (++waiting_ == count_) {
            on_last();
            done_ = true;
            cv_.notify_all();
        } else {
            cv_.wait(lk, [&] { return done_; });
        }
    }

  private:
    std::mutex mu_;
    std::condition_variable cv_;
    size_t count_, waiting_ = 0;
    bool done_ = false;
};

// ------------------------------------------------------------ batch driver

thread_local int64_t g_last_h2d = 0, g_last_d2h = 0;

double since_ms(std::chrono::steady_clock::time_point t0) {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
}

int align_packed_impl(const sg_config* cfg, const sg_packed_pairs* in, const int* devices,
                      int n_devices, sg_results* out) {
    const auto t0 = std::chrono::steady_clock::now();
    std::memset(out, 0, sizeof *out);
    int rc = validate_cfg(cfg);
    if (rc) return rc;
    if (!in || in->n_pairs < 0) return set_error(SG_INPUT, "null or negative pair batch");
    const int64_t n = in->n_pairs;
    if (n > INT32_MAX) return set_error(SG_INPUT, "too many pairs in one batch");
    rc = validate_lengths(n, in->text_len, in->pat_len, cfg);
    if (rc) return rc;
    int dev_default = 0;
    if (!devices || n_devices < 1) {
        devices = &dev_default;
        n_devices = 1;
    }
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count < 1)
        return set_error(SG_CUDA, "no CUDA device available (the GPU path has no CPU fallback)");
    for (int d = 0; d < n_devices; ++d)
        if (devices[d] < 0 || devices[d] >= count)
            return set_error(SG_CONFIG, "bad device index %d", devices[d]);
    DeviceGuard guard;
    const sg_options opt = options();
    const bool trace = (opt.diagnostics & SG_DIAG_HOST_TRACE) != 0;
    g_trace_t0 = trace && n_devices == 1 ? &t0 : nullptr;
    struct TraceReset {  // (t0 is this call's: no trace point may outlive it)
        ~TraceReset() { g_trace_t0 = nullptr; }
    } trace_reset;
    const RunConfig rcfg = run_config(cfg, n, in->text_len, in->pat_len);
    const size_t nd = static_cast<size_t>(n_devices);
    const ShardPlan plan = plan_shards(in, nd);
    if (trace) std::fprintf(stderr, "[sg trace] %-10s %8.2f ms\n", "plan", since_ms(t0));

    bool mixed = false;
    int64_t lmin = INT64_MAX, lmax = 0;
    {
        std::vector<int64_t> pmin(64, INT64_MAX), pmax(64, 0);
        parallel_for(n, [&](int64_t lo, int64_t hi, int t) {
            int64_t a = INT64_MAX, b = 0;
            for (int64_t k = lo; k < hi; ++k) {
                const int64_t l = in->text_len[k] + in->pat_len[k];
                a = std::min(a, l);
                b = std::max(b, l);
            }
            pmin[static_cast<size_t>(t)] = a;
            pmax[static_cast<size_t>(t)] = b;
        }, kParGrain);
        lmin = *std::min_element(pmin.begin(), pmin.end());
        lmax = *std::max_element(pmax.begin(), pmax.end());
    }
    mixed = n > 1 && lmax != lmin;
    // One device: the run bytes leave in slices while K1 still runs (§5). Slices are
    // ranges of input order, so near-equal pairs (cfg2/3/4) go in input order rather
    // than longest first: slices then finish roughly one after another.
    const bool sliced = nd == 1 && n >= 4096;
    const bool uniform = 4 * lmax <= 5 * lmin;

    std::vector<ShardOut> so(nd);
    std::vector<ShardPrep> prep(nd);
    std::vector<Packed> gathered(plan.gathered ? nd : 0);
    std::vector<sg_packed_pairs> views(nd);
    std::vector<PinBuf> stage(nd);  // gathered shards: run bytes before the scatter
    int fail_code = SG_OK;
    std::string fail_msg;
    int64_t run_total = 0;
    std::vector<int64_t> run_base(nd, 0);
    Rendezvous meet(nd);

    // Runs once, after every shard's kernels: errors, then the first failing pair
    // in input order (batch.cpp:94-97), then the result buffers and the CIGAR
    // offsets in input order.
    auto size_results = [&]() {
        for (auto& o : so)
            if (o.err && !fail_code) {
                fail_code = o.err;
                fail_msg = o.msg;
            }
        if (fail_code) return;
        int64_t bad = -1;
        int32_t bad_status = 0;
        for (size_t d = 0; d < nd; ++d) {
            const int64_t sn = plan.gathered ? static_cast<int64_t>(plan.members[d].size())
                                             : plan.cut[d + 1] - plan.cut[d];
            const int32_t* st = so[d].status.as<int32_t>();
            if (!plan.gathered) {  // contiguous shards: the first bad pair was found at the fetch
                if (so[d].first_bad >= 0 && (bad < 0 || plan.cut[d] + so[d].first_bad < bad)) {
                    bad = plan.cut[d] + so[d].first_bad;
                    bad_status = so[d].first_bad_status;
                }
                continue;
            }
            for (int64_t k = 0; k < sn; ++k) {
                if (!st[k]) continue;
                const int64_t g = plan.gathered ? plan.members[d][static_cast<size_t>(k)] : plan.cut[d] + k;
                if (bad < 0 || g < bad) {
                    bad = g;
                    bad_status = st[k];
                }
                if (!plan.gathered) break;
            }
        }
        if (bad >= 0) {
            fail_code = set_error(SG_INTERNAL, "pair '%lld': %s", static_cast<long long>(bad),
                                  status_detail(bad_status));
            fail_msg = g_last_error;
            return;
        }
        for (size_t d = 0; d < nd; ++d) {
            run_base[d] = run_total;
            run_total += so[d].run_bytes;
        }
        try {
            results_alloc(out, n, run_total, nd == 1 && so[0].staged ? &so[0].runs : nullptr);
        } catch (const Fail& f) {
            fail_code = f.code;
            fail_msg = g_last_error;
            return;
        }
        if (plan.gathered) {  // CIGAR offsets in input order from the shards' sizes
            for (size_t d = 0; d < nd; ++d) {
                const int64_t* doff = so[d].doff.as<int64_t>();
                const auto& mem = plan.members[d];
                for (size_t k = 0; k < mem.size(); ++k) out->cigar_off[mem[k] + 1] = doff[k + 1] - doff[k];
            }
            out->cigar_off[0] = 0;
            for (int64_t k = 0; k < n; ++k) out->cigar_off[k + 1] += out->cigar_off[k];
        }
    };

    // One host thread per shard runs it from upload to result copy, holding its
    // device pipeline throughout.
    auto body = [&](size_t d) {
        ShardOut& o = so[d];
        std::unique_lock<std::mutex> slot_lock;
        DevState* stp = nullptr;
        auto guarded = [&](auto&& f) {
            try {
                f();
            } catch (const Fail& f) {
                o.err = f.code;
                o.msg = g_last_error;
            } catch (const std::exception& e) {
                o.err = SG_INTERNAL;
                o.msg = e.what();
            } catch (...) {
                o.err = SG_INTERNAL;
                o.msg = "unknown exception in the device pipeline";
            }
        };
        guarded([&] {
            SG_CUDA_CHECK(cudaSetDevice(devices[d]));
            int occ = 0;
            for (size_t e = 0; e < d; ++e) occ += devices[e] == devices[d];
            DevSlot& slot = dev_slot(devices[d], occ);
            slot_lock = std::unique_lock<std::mutex>(slot.mu);
            if (!slot.st) {
                slot.st = std::make_unique<DevState>();
                slot.st->init(devices[d]);
            }
            DevState& st = *slot.st;
            stp = &st;
            Shard s{in, plan.cut[d], plan.cut[d + 1]};
            if (plan.gathered) {
                gather_shard(in, plan.members[d], gathered[d]);
                views[d] = gathered[d].view();
                s = Shard{&views[d], 0, static_cast<int64_t>(plan.members[d].size())};
                if (trace) std::fprintf(stderr, "[sg trace] %-10s %8.2f ms\n", "gather", since_ms(t0));
            }
            // streamed: the first round of lanes takes pairs from the front of memory
            const bool streamed = opt.stream_upload != 0;
            // the sequence words first: their copy overlaps the host prep below
            int64_t wlo = 0, whi = 0;
            shard_words(s, &wlo, &whi);
            o.h2d_bytes = upload_seq(st, s, wlo, whi, streamed);
            RunConfig rcs = rcfg;
            rcs.band = rcfg.band && band_pays(s.in, s.lo, s.hi, rcfg.W, rcfg.O);
            if (rcs.band) rcs.band_sub = band_schedule(s.in, s.lo, s.hi, rcfg.W);
            const int64_t split = streamed ? pairs_in_flight(st, rcs, s.hi - s.lo) : 0;
            const int64_t words[2] = {wlo, whi};
            prep_shard(s, prep[d], mixed && !(sliced && uniform), split, words);
            o.h2d_bytes += upload_shard(st, s, prep[d], streamed, true);
            if (trace) std::fprintf(stderr, "[sg trace] %-10s %8.2f ms\n", "upload", since_ms(t0));
            const int64_t sn = s.hi - s.lo;
            SlicePlan sp;
            // (K1 mixed leaves every pair's tail to the launches after it: pipelined,
            // they run per slice beside it on a few SMs, §3.12)
            if (sliced && !rcs.band) {
                sp.early = static_cast<int>(std::min<int64_t>(DevState::kMaxSlices, std::max<int64_t>(1, sn / 4096)));
                sp.per = static_cast<int32_t>((sn + sp.early - 1) / sp.early);
                sp.early = static_cast<int>((sn + sp.per - 1) / sp.per);
            } else if (sliced && !(opt.diagnostics & SG_DIAG_NO_PIPELINE) && !prep[d].ordered &&
                       st.sms >= 16 && tail_sm_count(st, rcs, prep[d]) * 10 <= st.sms) {
                // K1 mixed, pipelined (§3.12). Its lanes take the pairs in input order
                // and, the pairs being of near-equal length, finish them round by
                // round: the pairs of all rounds but the last leave it early and go
                // out in slices of >= 4096 pairs; those of the last round finish while
                // K1 mixed's blocks leave, in slices of the same size on growing grids. (Batches whose tail / final windows are a large share of the
                // work, cfg2: the kernels one after another on every SM are faster than
                // a static split of the SMs.)
                const int64_t lanes = std::max<int64_t>(
                    1, 32 * band_active_warps(st, rcs, sn, st.sms - tail_sm_count(st, rcs, prep[d])));
                const int64_t early = (sn / lanes - 1) * lanes;
                if (early >= 4096) {
                    // (the last round in slices of the same size: a second slice size
                    // in K1 mixed's pair -> slice mapping cost its window loop 2 %)
                    int es = static_cast<int>(std::min<int64_t>(DevState::kMaxSlices - 1, early / 4096));
                    int32_t per = static_cast<int32_t>((early + es - 1) / es);
                    while ((sn + per - 1) / per > DevState::kMaxSlices && es > 1) {
                        --es;
                        per = static_cast<int32_t>((early + es - 1) / es);
                    }
                    const int64_t tot = (sn + per - 1) / per;
                    if (tot <= DevState::kMaxSlices && tot > es) {
                        sp.early = es;
                        sp.per = sp.per_late = per;
                        sp.late = static_cast<int>(tot) - es;
                    }
                }
            }
            const int slices = sp.total();
            o.launches = launch_shard(st, rcs, prep[d], sp);
            fetch_small_issue(st, prep[d].n, o);  // (beside the last slices' run bytes)
            if (slices) {
                stream_runs(st, slices, prep[d].scratch_bytes, o);
                if (trace) std::fprintf(stderr, "[sg trace] %-10s %8.2f ms\n", "runs d2h", since_ms(t0));
            }
            fetch_small_finish(st, prep[d].n, o);
            if (trace) std::fprintf(stderr, "[sg trace] %-10s %8.2f ms\n", "kernels", since_ms(t0));
        });
        meet.arrive(size_results);
        if (fail_code || !stp) return;
        guarded([&] {
            DevState& st = *stp;
            if (plan.gathered) {
                stage[d].ensure(static_cast<size_t>(std::max<int64_t>(o.run_bytes, 1)));
                if (o.run_bytes)
                    SG_CUDA_CHECK(cudaMemcpyAsync(stage[d].p, st.dense.p, static_cast<size_t>(o.run_bytes),
                                                  cudaMemcpyDeviceToHost, st.stream));
                SG_CUDA_CHECK(cudaStreamSynchronize(st.stream));
                const auto& mem = plan.members[d];
                const int32_t* dist = o.dist.as<int32_t>();
                const int32_t* win = o.win.as<int32_t>();
                const int64_t* doff = o.doff.as<int64_t>();
                const uint64_t* cnt = o.cnt.as<uint64_t>();
                const uint8_t* src = stage[d].as<uint8_t>();
                for (size_t k = 0; k < mem.size(); ++k) {
                    const int64_t g = mem[k];
                    out->distance[g] = dist[k];
                    out->windows[g] = win[k];
                    out->found[g] = dist[k] >= 0;
                    std::memcpy(out->runs + out->cigar_off[g], src + doff[k],
                                static_cast<size_t>(doff[k + 1] - doff[k]));
                    std::memcpy(out->counters + g * SG_CNT_COUNT, cnt + k * SG_CNT_COUNT,
                                8 * SG_CNT_COUNT);
                }
            } else if (o.staged) {  // run bytes already in the result (sliced D2H)
                scatter_small(out, plan.cut[d], plan.cut[d + 1] - plan.cut[d], run_base[d], o);
            } else {
                if (o.run_bytes)
                    SG_CUDA_CHECK(cudaMemcpyAsync(out->runs + run_base[d], st.dense.p,
                                                  static_cast<size_t>(o.run_bytes),
                                                  cudaMemcpyDeviceToHost, st.stream));
                scatter_small(out, plan.cut[d], plan.cut[d + 1] - plan.cut[d], run_base[d], o);
                SG_CUDA_CHECK(cudaStreamSynchronize(st.stream));
            }
            if (!o.staged) o.d2h_bytes += o.run_bytes;
            if (trace) std::fprintf(stderr, "[sg trace] %-10s %8.2f ms\n", "results", since_ms(t0));
        });
    };
    if (nd == 1) {
        body(0);
    } else {
        std::vector<std::thread> th;
        th.reserve(nd);
        for (size_t d = 0; d < nd; ++d) th.emplace_back(body, d);
        for (auto& t : th) t.join();
    }
    if (!fail_code)
        for (auto& o : so)
            if (o.err) {
                fail_code = o.err;
                fail_msg = o.msg;
                break;
            }
    if (fail_code) {
        sg_results_free(out);
        return set_error(fail_code, "%s", fail_msg.c_str());
    }
    finish_totals(out);
    g_last_h2d = g_last_d2h = 0;
    for (auto& o : so) {
        out->device_ms = std::max(out->device_ms, static_cast<double>(o.device_ms));
        out->kernel_ms = std::max(out->kernel_ms, static_cast<double>(o.k1_ms));
        out->gpu_launches += o.launches;
        g_last_h2d += o.h2d_bytes;
        g_last_d2h += o.d2h_bytes;
    }
    out->align_seconds =
        std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return SG_OK;
}

// ------------------------------------------------------------ synthetic batches

// Generates pairs [first, first+count) of a BASELINE config in parallel.
// emit(k, text, n, pattern, m) is called once per pair, from worker threads.
template <class Emit>
int synth_each(const sg_synth_spec& spec, int64_t first, int64_t count, Emit&& emit) {
    std::atomic<int> bad{0};
    parallel_for(count, [&](int64_t lo, int64_t hi, int) {
        std::vector<uint8_t> tb(static_cast<size_t>(sg_synth_max_text(&spec)));
        std::vector<uint8_t> pb(static_cast<size_t>(sg_synth_max_pattern(&spec)));
        for (int64_t k = lo; k < hi; ++k) {
            int64_t n = 0, m = 0;
            if (sg_synth_pair(&spec, first + k, tb.data(), &n, pb.data(), &m)) {
                bad = 1;
                return;
            }
            emit(k, tb.data(), n, pb.data(), m);
        }
    }, 256);
    return bad.load() ? set_error(SG_INPUT, "bad synthetic spec") : SG_OK;
}

struct OwnedCodes {
    std::vector<uint8_t> text, pattern;
    std::vector<int64_t> text_off, text_len, pat_off, pat_len;
};
std::mutex g_codes_mu;
std::vector<OwnedCodes*>& codes_registry() {
    static auto* r = new std::vector<OwnedCodes*>();
    return *r;
}

}  // namespace

// ====================================================================== C ABI

struct sg_session {
    sg_config cfg;
    RunConfig rc;
    DevState st;
    ShardPrep prep;
    int64_t n = 0;
    int launches = 0;
    bool ran = false;
};

extern "C" {

int sg_abi_version(void) { return SG_ABI_VERSION; }

int sg_device_count(void) {
    int c = 0;
    if (cudaGetDeviceCount(&c) != cudaSuccess) return 0;
    return c;
}

const char* sg_last_error(void) { return g_last_error.c_str(); }

void sg_config_default(sg_config* cfg) {
    cfg->W = 64;
    cfg->O = 33;
    cfg->sene = 1;
    cfg->dent = 1;
    cfg->early_termination = 1;
    cfg->single_window = 0;
    cfg->k_single = 1024;
}

int sg_validate_config(const sg_config* cfg) { return validate_cfg(cfg); }

void sg_options_default(sg_options* o) {
    o->kernel = SG_KERNEL_AUTO;
    o->stream_upload = 1;
    o->longest_first = 1;
    o->diagnostics = 0;
    o->exact_budget = 0;
}

int sg_set_options(const sg_options* o) {
    if (!o) return set_error(SG_CONFIG, "null options");
    if (o->kernel < SG_KERNEL_AUTO || o->kernel > SG_KERNEL_WIDE)
        return set_error(SG_CONFIG, "unknown kernel option %d", o->kernel);
    if (o->exact_budget < 0) return set_error(SG_CONFIG, "negative exact_budget");
    std::lock_guard<std::mutex> lk(g_opt_mu);
    g_opt = *o;
    return SG_OK;
}

void sg_get_options(sg_options* o) { *o = options(); }

int sg_align_packed(const sg_config* cfg, const sg_packed_pairs* pairs, const int* devices,
                    int n_devices, sg_results* out) {
    try {
        return align_packed_impl(cfg, pairs, devices, n_devices, out);
    } catch (const Fail& f) {
        return f.code;
    } catch (const std::exception& e) {
        return set_error(SG_INTERNAL, "%s", e.what());
    }
}

int sg_align_batch(const sg_config* cfg, const sg_pairs* pairs, const int* devices,
                   int n_devices, sg_results* out) {
    const auto t0 = std::chrono::steady_clock::now();
    std::memset(out, 0, sizeof *out);
    int rc = validate_cfg(cfg);
    if (rc) return rc;
    if (!pairs || pairs->n_pairs < 0) return set_error(SG_INPUT, "null or negative pair batch");
    rc = validate_lengths(pairs->n_pairs, pairs->text_len, pairs->pat_len, cfg);
    if (rc) return rc;
    try {
        Packed pk;
        pack_pairs(pairs, pk);
        const sg_packed_pairs v = pk.view();
        rc = align_packed_impl(cfg, &v, devices, n_devices, out);
    } catch (const Fail& f) {
        return f.code;
    } catch (const std::exception& e) {
        return set_error(SG_INTERNAL, "%s", e.what());
    }
    if (rc == SG_OK)
        out->align_seconds =
            std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return rc;
}

void sg_results_free(sg_results* res) {
    if (!res) return;
    delete static_cast<ResultOwner*>(res->_owner);
    std::memset(res, 0, sizeof *res);
}

int64_t sg_cigar_runs(const sg_results* res, int64_t k, char* ops, int64_t* lens, int64_t cap) {
    if (!res || k < 0 || k >= res->n_pairs) return -1;
    static const char kOp[4] = {'=', 'X', 'I', 'D'};
    int64_t nr = 0;
    int prev = -1;
    for (int64_t b = res->cigar_off[k]; b < res->cigar_off[k + 1]; ++b) {
        const uint8_t v = res->runs[b];
        const int op = v >> 6;
        const int64_t len = (v & 63) + 1;
        if (op == prev) {
            if (nr - 1 < cap) lens[nr - 1] += len;
        } else {
            if (nr < cap) {
                ops[nr] = kOp[op];
                lens[nr] = len;
            }
            ++nr;
            prev = op;
        }
    }
    return nr;
}

int64_t sg_cigar_string(const sg_results* res, int64_t k, char* buf, int64_t cap) {
    if (!res || k < 0 || k >= res->n_pairs) return -1;
    static const char kOp[4] = {'=', 'X', 'I', 'D'};
    int64_t pos = 0;
    char tmp[32];
    // snprintf semantics: the longest prefix that fits, NUL-terminated
    auto put = [&](int op, int64_t len) {
        const int w = snprintf(tmp, sizeof tmp, "%lld%c", static_cast<long long>(len), kOp[op]);
        if (buf && pos < cap - 1)
            std::memcpy(buf + pos, tmp, static_cast<size_t>(std::min<int64_t>(w, cap - 1 - pos)));
        pos += w;
    };
    int prev = -1;
    int64_t run = 0;
    for (int64_t b = res->cigar_off[k]; b < res->cigar_off[k + 1]; ++b) {
        const uint8_t v = res->runs[b];
        const int op = v >> 6;
        if (op != prev && prev >= 0) {
            put(prev, run);
            run = 0;
        }
        prev = op;
        run += (v & 63) + 1;
    }
    if (prev >= 0) put(prev, run);
    if (buf && cap > 0) buf[std::min(pos, cap - 1)] = '\0';
    return pos;
}

int sg_pack(const sg_pairs* in, sg_packed_pairs* out) {
    if (!in || !out) return set_error(SG_INPUT, "null argument");
    try {
        auto pk = std::make_unique<Packed>();
        pack_pairs(in, *pk);
        *out = pk->view();
        std::lock_guard<std::mutex> lk(g_owned_mu);
        packed_registry().push_back(pk.release());
        return SG_OK;
    } catch (const Fail& f) {
        return f.code;
    }
}

void sg_packed_free(sg_packed_pairs* p) {
    if (!p || !p->seq) return;
    std::lock_guard<std::mutex> lk(g_owned_mu);
    auto& reg = packed_registry();
    for (size_t k = 0; k < reg.size(); ++k)
        if (reg[k]->seq.p == p->seq) {
            delete reg[k];
            reg.erase(reg.begin() + static_cast<long>(k));
            break;
        }
    std::memset(p, 0, sizeof *p);
}

int sg_session_create(const sg_config* cfg, const sg_packed_pairs* pairs, int device,
                      sg_session** out) {
    *out = nullptr;
    int rc = validate_cfg(cfg);
    if (rc) return rc;
    if (!pairs || pairs->n_pairs < 0 || pairs->n_pairs > INT32_MAX)
        return set_error(SG_INPUT, "bad pair batch");
    rc = validate_lengths(pairs->n_pairs, pairs->text_len, pairs->pat_len, cfg);
    if (rc) return rc;
    if (sg_device_count() <= device || device < 0)
        return set_error(SG_CUDA, "no CUDA device %d (the GPU path has no CPU fallback)", device);
    DeviceGuard guard;
    auto s = std::make_unique<sg_session>();
    try {
        s->cfg = *cfg;
        s->rc = run_config(cfg, pairs->n_pairs, pairs->text_len, pairs->pat_len);
        s->rc.band = s->rc.band && band_pays(pairs, 0, pairs->n_pairs, s->rc.W, s->rc.O);
        if (s->rc.band) s->rc.band_sub = band_schedule(pairs, 0, pairs->n_pairs, s->rc.W);
        s->st.init(device);
        s->n = pairs->n_pairs;
        bool mixed = false;
        for (int64_t k = 1; k < s->n && !mixed; ++k)
            mixed = pairs->text_len[k] + pairs->pat_len[k] != pairs->text_len[0] + pairs->pat_len[0];
        const Shard sh{pairs, 0, s->n};
        prep_shard(sh, s->prep, mixed);
        upload_shard(s->st, sh, s->prep);
        SG_CUDA_CHECK(cudaStreamSynchronize(s->st.stream));
    } catch (const Fail& f) {
        return f.code;
    }
    *out = s.release();
    return SG_OK;
}

int sg_session_run(sg_session* s, float* device_ms, float* k1_ms) {
    DeviceGuard guard;
    try {
        SG_CUDA_CHECK(cudaSetDevice(s->st.device));
        s->launches = launch_shard(s->st, s->rc, s->prep);
        SG_CUDA_CHECK(cudaEventSynchronize(s->st.ev[2]));
        float ms = 0, k1 = 0;
        SG_CUDA_CHECK(cudaEventElapsedTime(&ms, s->st.ev[0], s->st.ev[2]));
        SG_CUDA_CHECK(cudaEventElapsedTime(&k1, s->st.ev[0], s->st.ev[1]));
        if (device_ms) *device_ms = ms;
        if (k1_ms) *k1_ms = k1;
        s->ran = true;
        return SG_OK;
    } catch (const Fail& f) {
        return f.code;
    }
}

int sg_session_fetch(sg_session* s, sg_results* out) {
    std::memset(out, 0, sizeof *out);
    if (!s->ran) return set_error(SG_INPUT, "session has not run");
    DeviceGuard guard;
    try {
        SG_CUDA_CHECK(cudaSetDevice(s->st.device));
        ShardOut so;
        fetch_small(s->st, s->n, so);
        if (so.first_bad >= 0)
            return set_error(SG_INTERNAL, "pair '%lld': %s", static_cast<long long>(so.first_bad),
                             status_detail(so.first_bad_status));
        results_alloc(out, s->n, so.run_bytes);
        if (so.run_bytes)
            SG_CUDA_CHECK(cudaMemcpyAsync(out->runs, s->st.dense.p, static_cast<size_t>(so.run_bytes),
                                          cudaMemcpyDeviceToHost, s->st.stream));
        scatter_small(out, 0, s->n, 0, so);
        SG_CUDA_CHECK(cudaStreamSynchronize(s->st.stream));
        finish_totals(out);
        out->device_ms = so.device_ms;
        out->kernel_ms = so.k1_ms;
        out->gpu_launches = s->launches;
        return SG_OK;
    } catch (const Fail& f) {
        sg_results_free(out);
        return f.code;
    }
}

int sg_session_info(const sg_session* s, int64_t* lanes, int32_t* sms, int32_t* limbs) {
    if (lanes) *lanes = s->st.lanes;
    if (sms) *sms = s->st.sms;
    if (limbs) *limbs = s->rc.wide ? (s->rc.wcap + 31) / 32 : s->rc.L;
    return SG_OK;
}

int sg_session_kernel(const sg_session* s) { return s->rc.wide ? 2 : s->rc.band ? 1 : 0; }

void sg_session_destroy(sg_session* s) {
    DeviceGuard guard;
    delete s;
}

int sg_session_warp_times(sg_session* s, uint64_t* out, int cap) {
    if (!s || !(s->st.diag_flags & SG_DIAG_WARP_TIMES) || !s->st.diag_warp.p) return -1;
    DeviceGuard guard;
    cudaSetDevice(s->st.device);
    const int n = std::min(cap, s->st.diag_warps);
    if (cudaMemcpy(out, s->st.diag_warp.p, 24 * static_cast<size_t>(n), cudaMemcpyDeviceToHost) !=
        cudaSuccess)
        return -1;
    return n;
}

int sg_session_phase_cycles(sg_session* s, uint64_t* out25) {
    if (!s || !(s->st.diag_flags & SG_DIAG_PHASE_CYCLES) || !s->st.diag_phase.p) return -1;
    DeviceGuard guard;
    cudaSetDevice(s->st.device);
    if (cudaMemcpy(out25, s->st.diag_phase.p, 25 * 8, cudaMemcpyDeviceToHost) != cudaSuccess)
        return -1;
    return 0;
}

int sg_plan_shards(const sg_packed_pairs* pairs, int n_devices, int32_t* shard, int64_t* pos,
                   int* gathered) {
    if (!pairs || pairs->n_pairs < 0 || !shard || !pos) return set_error(SG_INPUT, "null argument");
    if (n_devices < 1) return set_error(SG_CONFIG, "n_devices must be >= 1");
    try {
        const ShardPlan plan = plan_shards(pairs, static_cast<size_t>(n_devices));
        for (int d = 0; d < n_devices; ++d) {
            if (plan.gathered) {
                const auto& mem = plan.members[static_cast<size_t>(d)];
                for (size_t k = 0; k < mem.size(); ++k) {
                    shard[mem[k]] = d;
                    pos[mem[k]] = static_cast<int64_t>(k);
                }
            } else {
                for (int64_t k = plan.cut[static_cast<size_t>(d)]; k < plan.cut[static_cast<size_t>(d) + 1]; ++k) {
                    shard[k] = d;
                    pos[k] = k - plan.cut[static_cast<size_t>(d)];
                }
            }
        }
        if (gathered) *gathered = plan.gathered ? 1 : 0;
        return SG_OK;
    } catch (const std::exception& e) {
        return set_error(SG_INTERNAL, "%s", e.what());
    }
}

int64_t sg_last_transfer_bytes(int direction) { return direction ? g_last_d2h : g_last_h2d; }

/* oracle::global_align (proj/src/oracle.cpp:39-89) on the GPU: K7, then K2/K3. */
int sg_global_align(const sg_packed_pairs* pairs, int device, sg_results* out) {
    std::memset(out, 0, sizeof *out);
    const auto t0 = std::chrono::steady_clock::now();
    if (!pairs || pairs->n_pairs < 0 || pairs->n_pairs > INT32_MAX)
        return set_error(SG_INPUT, "bad pair batch");
    const int64_t n = pairs->n_pairs;
    for (int64_t k = 0; k < n; ++k) {  // the reference's guards (oracle.cpp:43-46)
        const int64_t tl = pairs->text_len[k], pl = pairs->pat_len[k];
        if (tl > 100000 || pl > 100000)
            return set_error(SG_INPUT,
                             "global_align: sequence longer than the 10^5 quadratic-cost guard");
        if ((tl + 1) * (pl + 1) > (int64_t{1} << 30))
            return set_error(SG_INPUT, "global_align: pair too large for the exact traceback matrix");
    }
    if (device < 0 || sg_device_count() <= device)
        return set_error(SG_CUDA, "no CUDA device %d (the GPU path has no CPU fallback)", device);
    DeviceGuard guard;
    try {
        SG_CUDA_CHECK(cudaSetDevice(device));
        DevSlot& slot = dev_slot(device, 0);
        std::lock_guard<std::mutex> lk(slot.mu);
        if (!slot.st) {
            slot.st = std::make_unique<DevState>();
            slot.st->init(device);
        }
        DevState& st = *slot.st;
        const Shard sh{pairs, 0, n};
        ShardPrep pp;
        prep_shard(sh, pp, false);
        upload_shard(st, sh, pp);
        const size_t n1 = static_cast<size_t>(std::max<int64_t>(n, 1));
        st.distance.ensure(4 * n1);
        st.out_bytes.ensure(4 * n1);
        st.scratch.ensure(static_cast<size_t>(std::max<int64_t>(pp.scratch_bytes, 4)));
        st.dense_off.ensure(8 * (n1 + 1));
        st.dense.ensure(static_cast<size_t>(std::max<int64_t>(pp.scratch_bytes, 4)));
        st.scan_tmp.ensure(sgk::cigar_offsets_temp_bytes(static_cast<int32_t>(n)) + 64);
        // The delta store (16 B per 32 cells) goes in batches of pairs within a
        // memory budget: half the free device memory (at least 4 GiB), or
        // sg_options.exact_budget bytes; a pair larger than the budget runs alone.
        size_t free_b = 0, total_b = 0;
        SG_CUDA_CHECK(cudaMemGetInfo(&free_b, &total_b));
        int64_t budget = std::max<int64_t>(int64_t{4} << 30, static_cast<int64_t>(free_b / 2));
        if (const int64_t b = options().exact_budget) budget = b;
        PinBuf soff, hoff;
        soff.ensure(8 * n1);
        hoff.ensure(8 * n1);
        std::vector<int64_t> cut{0};
        std::vector<int64_t> batch_store, batch_h;
        {
            int64_t s_acc = 0, h_acc = 0;
            for (int64_t k = 0; k < n; ++k) {
                const int64_t tl = pairs->text_len[k], pl = pairs->pat_len[k];
                const int64_t sw = ((pl + 31) / 32) * tl;           // uint4 entries
                const int64_t hw = ((tl + 15) & ~int64_t{15}) + 16;  // bytes
                if (k > cut.back() && (s_acc + sw) * 16 > budget) {
                    cut.push_back(k);
                    batch_store.push_back(s_acc);
                    batch_h.push_back(h_acc);
                    s_acc = h_acc = 0;
                }
                soff.as<int64_t>()[k] = s_acc;
                hoff.as<int64_t>()[k] = h_acc;
                s_acc += sw;
                h_acc += hw;
            }
            cut.push_back(n);
            batch_store.push_back(s_acc);
            batch_h.push_back(h_acc);
        }
        const int64_t max_store = *std::max_element(batch_store.begin(), batch_store.end());
        const int64_t max_h = *std::max_element(batch_h.begin(), batch_h.end());
        st.ex_store.ensure(static_cast<size_t>(std::max<int64_t>(max_store, 1)) * 16);
        st.ex_hbuf.ensure(static_cast<size_t>(std::max<int64_t>(max_h, 16)));
        st.ex_store_off.ensure(8 * n1);
        st.ex_hbuf_off.ensure(8 * n1);
        if (n) {
            SG_CUDA_CHECK(cudaMemcpyAsync(st.ex_store_off.p, soff.p, 8 * static_cast<size_t>(n),
                                          cudaMemcpyHostToDevice, st.stream));
            SG_CUDA_CHECK(cudaMemcpyAsync(st.ex_hbuf_off.p, hoff.p, 8 * static_cast<size_t>(n),
                                          cudaMemcpyHostToDevice, st.stream));
        }
        int launches = 0;
        SG_CUDA_CHECK(cudaEventRecord(st.ev[0], st.stream));
        for (size_t bi = 0; bi + 1 < cut.size(); ++bi) {
            const int64_t lo = cut[bi], hi = cut[bi + 1];
            if (hi <= lo) continue;
            sgk::ExactParams p{};
            p.seq = st.seq.as<uint32_t>();
            p.nmask = pp.any_n ? st.nmask.as<uint32_t>() : nullptr;
            p.text_off = st.text_off.as<int64_t>() + lo;
            p.pat_off = st.pat_off.as<int64_t>() + lo;
            p.text_len = st.text_len.as<int32_t>() + lo;
            p.pat_len = st.pat_len.as<int32_t>() + lo;
            p.has_n = pp.any_n ? st.has_n.as<uint8_t>() + lo : nullptr;
            p.n_pairs = static_cast<int32_t>(hi - lo);
            p.store = static_cast<uint4*>(st.ex_store.p);
            p.store_off = st.ex_store_off.as<int64_t>() + lo;
            p.hbuf = static_cast<int8_t*>(st.ex_hbuf.p);
            p.hbuf_off = st.ex_hbuf_off.as<int64_t>() + lo;
            p.bound_off = st.bound_off.as<int64_t>() + lo;
            p.scratch = st.scratch.as<uint8_t>();
            p.distance = st.distance.as<int32_t>() + lo;
            p.out_bytes = st.out_bytes.as<int32_t>() + lo;
            SG_CUDA_CHECK(static_cast<cudaError_t>(sgk::launch_exact_align(p, st.stream)));
            ++launches;
        }
        SG_CUDA_CHECK(cudaEventRecord(st.ev[1], st.stream));
        SG_CUDA_CHECK(static_cast<cudaError_t>(sgk::launch_cigar_offsets(
            st.out_bytes.as<int32_t>(), st.dense_off.as<int64_t>(), static_cast<int32_t>(n),
            st.scan_tmp.p, st.scan_tmp.cap, st.stream)));
        SG_CUDA_CHECK(static_cast<cudaError_t>(sgk::launch_cigar_compact(
            st.scratch.as<uint32_t>(), st.bound_off.as<int64_t>(), st.dense_off.as<int64_t>(),
            st.out_bytes.as<int32_t>(), st.dense.as<uint8_t>(), static_cast<int32_t>(n), st.stream)));
        launches += n > 0 ? 4 : 0;
        SG_CUDA_CHECK(cudaEventRecord(st.ev[2], st.stream));
        PinBuf dist, doff;
        dist.ensure(4 * n1);
        doff.ensure(8 * (n1 + 1));
        if (n) {
            SG_CUDA_CHECK(cudaMemcpyAsync(dist.p, st.distance.p, 4 * static_cast<size_t>(n),
                                          cudaMemcpyDeviceToHost, st.stream));
        }
        SG_CUDA_CHECK(cudaMemcpyAsync(doff.p, st.dense_off.p, 8 * (static_cast<size_t>(n) + 1),
                                      cudaMemcpyDeviceToHost, st.stream));
        SG_CUDA_CHECK(cudaStreamSynchronize(st.stream));
        const int64_t run_bytes = doff.as<int64_t>()[n];
        results_alloc(out, n, run_bytes);
        if (run_bytes)
            SG_CUDA_CHECK(cudaMemcpy(out->runs, st.dense.p, static_cast<size_t>(run_bytes),
                                     cudaMemcpyDeviceToHost));
        for (int64_t k = 0; k < n; ++k) {
            out->distance[k] = dist.as<int32_t>()[k];
            out->windows[k] = 1;
            out->found[k] = 1;
            out->cigar_off[k] = doff.as<int64_t>()[k];
        }
        out->cigar_off[n] = run_bytes;
        std::memset(out->counters, 0, 8 * SG_CNT_COUNT * n1);
        finish_totals(out);
        float ms = 0, k7 = 0;
        SG_CUDA_CHECK(cudaEventElapsedTime(&ms, st.ev[0], st.ev[2]));
        SG_CUDA_CHECK(cudaEventElapsedTime(&k7, st.ev[0], st.ev[1]));
        out->device_ms = ms;
        out->kernel_ms = k7;
        out->gpu_launches = launches;
        out->align_seconds =
            std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        return SG_OK;
    } catch (const Fail& f) {
        sg_results_free(out);
        return f.code;
    }
}

int sg_synth_packed(int cfg_id, int64_t first, int64_t count, sg_packed_pairs* out) {
    std::memset(out, 0, sizeof *out);
    sg_synth_spec spec;
    if (!sg_synth_baseline_spec(cfg_id, &spec)) return set_error(SG_INPUT, "bad config id %d", cfg_id);
    if (count < 0) count = spec.n_pairs - first;
    try {
        // pass 1: lengths (cheap relative to alignment; the generator is replayed)
        std::vector<int64_t> tl(static_cast<size_t>(count)), pl(static_cast<size_t>(count));
        int rc = synth_each(spec, first, count,
                            [&](int64_t k, const uint8_t*, int64_t n, const uint8_t*, int64_t m) {
                                tl[static_cast<size_t>(k)] = n;
                                pl[static_cast<size_t>(k)] = m;
                            });
        if (rc) return rc;
        auto pk = std::make_unique<Packed>();
        layout_offsets(*pk, count, tl.data(), pl.data());
        uint32_t* seq = pk->seq.as<uint32_t>();
        const int64_t* to = pk->text_off.as<int64_t>();
        const int64_t* po = pk->pat_off.as<int64_t>();
        rc = synth_each(spec, first, count,
                        [&](int64_t k, const uint8_t* t, int64_t n, const uint8_t* p, int64_t m) {
                            pack_seq(t, n, seq + to[k] / 16, nullptr, 0);
                            pack_seq(p, m, seq + po[k] / 16, nullptr, 0);
                        });
        if (rc) return rc;
        pk->any_n = false;
        *out = pk->view();
        std::lock_guard<std::mutex> lk(g_owned_mu);
        packed_registry().push_back(pk.release());
        return SG_OK;
    } catch (const Fail& f) {
        return f.code;
    }
}

int sg_synth_codes(int cfg_id, int64_t first, int64_t count, sg_pairs* out) {
    std::memset(out, 0, sizeof *out);
    sg_synth_spec spec;
    if (!sg_synth_baseline_spec(cfg_id, &spec)) return set_error(SG_INPUT, "bad config id %d", cfg_id);
    if (count < 0) count = spec.n_pairs - first;
    auto oc = std::make_unique<OwnedCodes>();
    const size_t c = static_cast<size_t>(count);
    oc->text_len.resize(c);
    oc->pat_len.resize(c);
    int rc = synth_each(spec, first, count,
                        [&](int64_t k, const uint8_t*, int64_t n, const uint8_t*, int64_t m) {
                            oc->text_len[static_cast<size_t>(k)] = n;
                            oc->pat_len[static_cast<size_t>(k)] = m;
                        });
    if (rc) return rc;
    oc->text_off.resize(c);
    oc->pat_off.resize(c);
    int64_t ta = 0, pa = 0;
    for (size_t k = 0; k < c; ++k) {
        oc->text_off[k] = ta;
        oc->pat_off[k] = pa;
        ta += oc->text_len[k];
        pa += oc->pat_len[k];
    }
    oc->text.resize(static_cast<size_t>(std::max<int64_t>(ta, 1)));
    oc->pattern.resize(static_cast<size_t>(std::max<int64_t>(pa, 1)));
    rc = synth_each(spec, first, count,
                    [&](int64_t k, const uint8_t* t, int64_t n, const uint8_t* p, int64_t m) {
                        std::memcpy(oc->text.data() + oc->text_off[static_cast<size_t>(k)], t,
                                    static_cast<size_t>(n));
                        std::memcpy(oc->pattern.data() + oc->pat_off[static_cast<size_t>(k)], p,
                                    static_cast<size_t>(m));
                    });
    if (rc) return rc;
    out->n_pairs = count;
    out->text = oc->text.data();
    out->text_off = oc->text_off.data();
    out->text_len = oc->text_len.data();
    out->pattern = oc->pattern.data();
    out->pat_off = oc->pat_off.data();
    out->pat_len = oc->pat_len.data();
    std::lock_guard<std::mutex> lk(g_codes_mu);
    codes_registry().push_back(oc.release());
    return SG_OK;
}

void sg_pairs_free(sg_pairs* p) {
    if (!p || !p->text) return;
    std::lock_guard<std::mutex> lk(g_codes_mu);
    auto& reg = codes_registry();
    for (size_t k = 0; k < reg.size(); ++k)
        if (reg[k]->text.data() == p->text) {
            delete reg[k];
            reg.erase(reg.begin() + static_cast<long>(k));
            break;
        }
    std::memset(p, 0, sizeof *p);
}

}  // extern "C"
