// capi.cu -- the C ABI of libodyssey_b200.so (include/odyssey_b200.h).
//
// Part 1 mirrors the reference's hot-path C ABI (ref proj/src/capi/capi.cpp:130-296):
// same status mapping, thread-local last error, exceptions never cross the ABI
// (ref capi.cpp:45-58), null arguments -> ODY_EINVAL before any work.  Behind it the
// quantized operands live in HBM in the kernel layouts (layout.h); every arithmetic
// step runs as an sm_100a kernel.  There is no CPU fallback: if the device or the
// kernels are unavailable the call fails with ODY_EDEVICE.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <condition_variable>
#include <functional>
#include <thread>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include <dlfcn.h>

#include <cstdio>
#include <cstring>
#include <filesystem>
#include <map>
#include <memory>
#include <vector>

#include "../../include/odyssey_b200.h"
#include "kernels.h"
#include "layout.h"

using namespace odyb200;

namespace {

thread_local std::string g_last_error;
unsigned long long* g_trace = nullptr;  // ody_dev_set_trace (diagnostics only)

struct Fail : std::runtime_error {
    ody_status code;
    Fail(ody_status c, const std::string& m) : std::runtime_error(m), code(c) {}
};
[[noreturn]] void fail(ody_status c, const std::string& m) { throw Fail(c, m); }

void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) fail(ODY_EDEVICE, std::string(what) + ": " + cudaGetErrorString(e));
}

template <typename Fn>
ody_status guarded(Fn&& fn) {
    try {
        fn();
        g_last_error.clear();
        return ODY_OK;
    } catch (const Fail& e) {
        g_last_error = e.what();
        return e.code;
    } catch (const std::bad_alloc&) {
        g_last_error = "out of memory";
        return ODY_EDEVICE;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return ODY_EINVAL;
    }
}

ody_status einval(const char* msg) {
    g_last_error = msg;
    return ODY_EINVAL;
}

// ---------------------------------------------------------------- runtime
// One library stream for the host-handle API; device memory from the stream-ordered
// pool (cudaMallocAsync) so per-call temporaries cost no driver round trip.
std::atomic<cudaStream_t> g_lib_stream{nullptr};  // the library stream (PinnedPool events)

struct Runtime {
    std::mutex mu;          // serialises host-API GEMMs (shared workspace)
    cudaStream_t stream = nullptr;
    void* workspace = nullptr;
    size_t workspace_bytes = 0;
    void* pscratch = nullptr;  // decode-width ody_gemm: dynamic decode kernel scratch
    size_t pscratch_bytes = 0;
    void* escratch = nullptr;  // comparison engines: split-K sums + tile counters
    size_t escratch_bytes = 0;
    int sms = 0;
    std::string version;
};

Runtime& rt() {
    static Runtime* r = [] {
        auto* x = new Runtime();
        int dev = 0;
        cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
        cudaDeviceProp prop;
        cuda_check(cudaGetDeviceProperties(&prop, dev), "cudaGetDeviceProperties");
        if (prop.major != 10) {
            fail(ODY_EDEVICE, "libodyssey_b200 needs an sm_100 (B200) device, found sm_" +
                                  std::to_string(prop.major) + std::to_string(prop.minor));
        }
        x->sms = prop.multiProcessorCount;
        cuda_check(cudaStreamCreateWithFlags(&x->stream, cudaStreamNonBlocking), "stream");
        g_lib_stream.store(x->stream);
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
            uint64_t thr = UINT64_MAX;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
        }
        char buf[256];
        std::snprintf(buf, sizeof(buf), "libodyssey_b200 sm_100a %s (%d SMs)", prop.name,
                      prop.multiProcessorCount);
        x->version = buf;
        return x;
    }();
    return *r;
}

// Pooled pinned host buffers back ody_tensor so H2D/D2H run at full PCIe rate and
// repeated calls do not pay cudaHostAlloc.
// Page-locked host buffers for ody_tensor data, pooled.  A buffer returned while a
// stream-ordered copy from it may still be pending (ody_quantize_activations does not
// synchronize) carries an event recorded on the library stream at return time; it is
// handed out again only once that event completed.  Pooled bytes are capped: past the
// cap a returned buffer is released (after its event).
struct PinnedPool {
    struct Entry {
        void* p;
        cudaEvent_t ev;  // completes when the library stream passed the buffer's last use
    };
    static constexpr size_t kCapBytes = size_t(1) << 30;
    std::mutex mu;
    std::multimap<size_t, Entry> free_list;
    std::map<void*, size_t> sizes;
    size_t pooled = 0;
    void* get(size_t bytes) {
        bytes = std::max<size_t>(bytes, 256);
        {
            std::lock_guard<std::mutex> l(mu);
            for (auto it = free_list.lower_bound(bytes); it != free_list.end() && it->first <= 2 * bytes; ++it) {
                if (it->second.ev && cudaEventQuery(it->second.ev) != cudaSuccess) {
                    cudaGetLastError();  // cudaErrorNotReady is not an error here
                    continue;
                }
                void* p = it->second.p;
                if (it->second.ev) cudaEventDestroy(it->second.ev);
                pooled -= it->first;
                free_list.erase(it);
                return p;
            }
        }
        void* p = nullptr;
        if (cudaHostAlloc(&p, bytes, cudaHostAllocDefault) != cudaSuccess) {
            cudaGetLastError();
            p = std::malloc(bytes);  // still correct, just pageable
            if (!p) throw std::bad_alloc();
            return p;
        }
        std::lock_guard<std::mutex> l(mu);
        sizes[p] = bytes;
        return p;
    }
    void put(void* p) {
        if (!p) return;
        std::lock_guard<std::mutex> l(mu);
        auto it = sizes.find(p);
        if (it == sizes.end()) {
            std::free(p);
            return;
        }
        cudaEvent_t ev = nullptr;
        cudaStream_t st = g_lib_stream.load();
        if (st && cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) == cudaSuccess) {
            if (cudaEventRecord(ev, st) != cudaSuccess) {
                cudaEventDestroy(ev);
                ev = nullptr;
                cudaStreamSynchronize(st);
            }
        }
        cudaGetLastError();
        if (pooled + it->second > kCapBytes) {  // over the cap: release it instead
            if (ev) {
                cudaEventSynchronize(ev);
                cudaEventDestroy(ev);
            }
            cudaFreeHost(p);
            sizes.erase(it);
            return;
        }
        pooled += it->second;
        free_list.emplace(it->second, Entry{p, ev});
    }
};
PinnedPool& pinned() {
    static PinnedPool* p = new PinnedPool();
    return *p;
}

template <typename T>
struct DevBuf {  // stream-ordered device temporary
    T* p = nullptr;
    cudaStream_t st;
    DevBuf(size_t count, cudaStream_t s) : st(s) {
        cuda_check(cudaMallocAsync(reinterpret_cast<void**>(&p), std::max<size_t>(count, 1) * sizeof(T), s),
                   "cudaMallocAsync");
    }
    ~DevBuf() {
        if (p) cudaFreeAsync(p, st);
    }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    DevBuf& operator=(DevBuf&& o) noexcept {
        if (this != &o) {
            if (p) cudaFreeAsync(p, st);
            p = o.p;
            st = o.st;
            o.p = nullptr;
        }
        return *this;
    }
    T* release() {
        T* q = p;
        p = nullptr;
        return q;
    }
};

}  // namespace

// ----------------------------------------------------------------- handles
struct ody_tensor {
    size_t rows = 0, cols = 0;
    float* data = nullptr;  // pinned (pooled) host memory
    ~ody_tensor() { pinned().put(data); }
};

// Act8: per-token INT8 (a8 layout); Weight4: per-channel INT4 (W4 tile layout);
// Weight4G: per-group INT4 (W4 tile layout, scales [rows][cols/group]); Weight8:
// per-channel INT8 (W8 layout).
enum class QKind { Act8, Weight4, Weight4G, Weight8 };

struct ody_qtensor {
    QKind kind;
    size_t rows = 0, cols = 0;
    size_t group_size = 128;  // the scheme's group_size (ref tensor.hpp:80), written to scheme.txt
    size_t groups() const { return kind == QKind::Weight4G ? cols / group_size : 1; }
    int bits() const { return kind == QKind::Act8 || kind == QKind::Weight8 ? 8 : 4; }
    const char* granularity() const {
        return kind == QKind::Act8 ? "per_token" : (kind == QKind::Weight4G ? "per_group" : "per_channel");
    }
    void* codes = nullptr;  // device, kernel layout
    float* scales = nullptr;  // device
    ~ody_qtensor() {
        cudaStream_t st = rt().stream;
        if (codes) cudaFreeAsync(codes, st);
        if (scales) cudaFreeAsync(scales, st);
    }
};

namespace {

// Host worker threads for the ABI's host-side copies (ody_tensor_create: the copy of the
// caller's f32 matrix into pinned memory fused with the reference's finite check).  One
// thread copies ~12 GB/s; the e2e step's inputs are 0.3-0.9 MB per call.  Workers spin
// ~200 us after a job before sleeping, so the back-to-back calls of a decode step find them
// awake.  ody_set_threads(n) sizes the pool (n <= 0: min(8, hardware threads)), as the
// reference's ody_set_threads sizes its CPU engine's pool (capi.cpp / parallel.cpp).
class HostPool {
   public:
    static HostPool& get() {
        static HostPool* p = new HostPool();  // never destroyed: workers are detached
        return *p;
    }
    void set_threads(int n) {
        std::lock_guard<std::mutex> l(dispatch_);
        want_ = n > 0 ? std::min(n, 64) : 0;
    }
    int threads() {
        const int hw = static_cast<int>(std::thread::hardware_concurrency());
        return want_ > 0 ? want_ : std::max(1, std::min(8, hw));
    }
    // f(i) for i in [0, parts); the caller runs part 0.  Serial when another caller holds
    // the pool or parts == 1.
    void parallel(int parts, const std::function<void(int)>& f) {
        if (parts <= 1) {
            for (int i = 0; i < parts; ++i) f(i);
            return;
        }
        std::unique_lock<std::mutex> dl(dispatch_, std::try_to_lock);
        if (!dl.owns_lock()) {
            for (int i = 0; i < parts; ++i) f(i);
            return;
        }
        grow(parts - 1);
        const int nw = static_cast<int>(workers_);
        {
            std::lock_guard<std::mutex> l(mu_);
            job_ = &f;
            parts_ = parts;
            remaining_.store(nw, std::memory_order_relaxed);
            gen_.fetch_add(1, std::memory_order_release);
        }
        cv_.notify_all();
        f(0);
        while (remaining_.load(std::memory_order_acquire) != 0) std::this_thread::yield();
        job_ = nullptr;
    }

   private:
    void grow(int n) {
        while (static_cast<int>(workers_) < n) {
            const int idx = static_cast<int>(workers_) + 1;
            const uint64_t seen = gen_.load(std::memory_order_acquire);  // before this dispatch's bump
            std::thread([this, idx, seen] { loop(idx, seen); }).detach();
            ++workers_;
        }
    }
    void loop(int idx, uint64_t seen) {
        for (;;) {
            const auto t0 = std::chrono::steady_clock::now();
            uint64_t g;
            while ((g = gen_.load(std::memory_order_acquire)) == seen) {
                if (std::chrono::steady_clock::now() - t0 > std::chrono::microseconds(200)) {
                    std::unique_lock<std::mutex> l(mu_);
                    cv_.wait(l, [&] { return gen_.load(std::memory_order_acquire) != seen; });
                }
            }
            seen = g;
            if (idx < parts_) (*job_)(idx);
            remaining_.fetch_sub(1, std::memory_order_acq_rel);
        }
    }
    std::mutex dispatch_, mu_;
    std::condition_variable cv_;
    std::atomic<uint64_t> gen_{0};
    std::atomic<int> remaining_{0};
    const std::function<void(int)>* job_ = nullptr;
    int parts_ = 0;
    size_t workers_ = 0;
    int want_ = 0;
};

// rows x cols f32 from `src` (row stride ld elements) into the contiguous `dst`, fused with
// the finite check (ref tensor.cpp:21-27): one pass over the exponent bits, split over the
// host pool in >= 128 KiB pieces.  Returns true when every value is finite.
bool copy_finite(float* dst, const float* src, size_t rows, size_t cols, size_t ld) {
    const size_t nel = rows * cols;
    HostPool& pool = HostPool::get();
    const int parts = static_cast<int>(std::max<size_t>(1, std::min<size_t>(pool.threads(), nel / 32768)));
    std::vector<uint32_t> bad(parts, 0u);
    auto piece = [&](int i) {
        // contiguous: element ranges; strided: row ranges (copied row by row)
        const size_t units = ld == cols ? nel : rows;
        const size_t lo = units * i / parts, hi = units * (i + 1) / parts;
        uint32_t b = 0;
        auto run = [&](const uint32_t* s, uint32_t* d, size_t n) {
            for (size_t e = 0; e < n; ++e) {
                const uint32_t v = s[e];
                d[e] = v;
                b |= static_cast<uint32_t>((v & 0x7f800000u) == 0x7f800000u);
            }
        };
        if (ld == cols)
            run(reinterpret_cast<const uint32_t*>(src) + lo, reinterpret_cast<uint32_t*>(dst) + lo, hi - lo);
        else
            for (size_t r = lo; r < hi; ++r)
                run(reinterpret_cast<const uint32_t*>(src + r * ld), reinterpret_cast<uint32_t*>(dst + r * cols), cols);
        bad[i] = b;
    };
    pool.parallel(parts, piece);
    uint32_t any = 0;
    for (uint32_t b : bad) any |= b;
    return any == 0;
}

ody_tensor* new_tensor(size_t rows, size_t cols) {
    auto* t = new ody_tensor();
    t->rows = rows;
    t->cols = cols;
    t->data = static_cast<float*>(pinned().get(rows * cols * sizeof(float)));
    return t;
}

int r_sms() { return device_sm_count(); }

void sync(cudaStream_t st, const char* what) {
    cuda_check(cudaGetLastError(), what);
    cuda_check(cudaStreamSynchronize(st), what);
}

void check_fast_inputs(const ody_qtensor* a_q, const ody_qtensor* w_q) {
    // ref gemm.cpp:206-216
    if (a_q->kind != QKind::Act8)
        fail(ODY_EINVAL, "GEMM: activations must be symmetric per-token INT8");
    if (w_q->kind != QKind::Weight4)
        fail(ODY_EINVAL, "gemm_w4a8_fast: weights must be per-channel 4-bit");
    if (a_q->cols != w_q->cols) fail(ODY_EINVAL, "gemm_w4a8_fast: inner dims disagree");
    if (w_q->cols > kMaxK)
        fail(ODY_EINVAL, "GEMM: K exceeds the 32-bit accumulator safety bound 2^17");
    if (a_q->rows > 0x7fffffff || w_q->rows > 0x7fffffff)
        fail(ODY_EINVAL, "GEMM: dimension exceeds int32 range");
}

void run_gemm(const ody_qtensor* a_q, const ody_qtensor* w_q, float* out_dev, int32_t* acc_dev,
              cudaStream_t st) {
    Runtime& r = rt();
    const int M = static_cast<int>(a_q->rows), N = static_cast<int>(w_q->rows), K = static_cast<int>(w_q->cols);
    if (gemm_prequant_eligible(M, N, K)) {  // decode widths: the dynamic decode kernel
        const size_t need = gemm_prequant_scratch_bytes(M, N, K, r.sms);
        if (r.pscratch_bytes < need) {
            if (r.pscratch) cuda_check(cudaFreeAsync(r.pscratch, st), "cudaFreeAsync");
            r.pscratch = nullptr;
            cuda_check(cudaMallocAsync(&r.pscratch, need, st), "cudaMallocAsync scratch");
            cuda_check(cudaMemsetAsync(r.pscratch, 0, program_zero_bytes(), st), "cudaMemsetAsync scratch");
            r.pscratch_bytes = need;
        }
        GemmArgs g = {};
        g.qa = static_cast<const int8_t*>(a_q->codes);
        g.sa = a_q->scales;
        g.wp = static_cast<const uint8_t*>(w_q->codes);
        g.sw = w_q->scales;
        g.out = out_dev;
        g.out_dtype = kDtypeF32;
        g.acc_out = acc_dev;
        g.M = M;
        g.N = N;
        g.K = K;
        g.max_ctas = r.sms;
        cuda_check(launch_w4a8_gemm_prequant(g, r.pscratch, r.pscratch_bytes, st), "w4a8 decode gemm launch");
        return;
    }
    const size_t need = gemm_workspace_bytes(static_cast<int>(a_q->rows), static_cast<int>(w_q->rows),
                                             static_cast<int>(w_q->cols), r.sms);
    if (r.workspace_bytes < need) {
        if (r.workspace) cuda_check(cudaFree(r.workspace), "cudaFree");
        r.workspace = nullptr;
        cuda_check(cudaMalloc(&r.workspace, need), "cudaMalloc workspace");
        // zeroed on the library stream: the GEMM launched next on it reads these counters
        cuda_check(cudaMemsetAsync(r.workspace, 0, need, st), "cudaMemsetAsync workspace");
        r.workspace_bytes = need;
    }
    GemmArgs g = {};
    g.qa = static_cast<const int8_t*>(a_q->codes);
    g.sa = a_q->scales;
    g.wp = static_cast<const uint8_t*>(w_q->codes);
    g.sw = w_q->scales;
    g.out = out_dev;
    g.out_dtype = kDtypeF32;
    g.acc_out = acc_dev;
    g.workspace = r.workspace;
    g.workspace_bytes = r.workspace_bytes;
    g.M = static_cast<int>(a_q->rows);
    g.N = static_cast<int>(w_q->rows);
    g.K = static_cast<int>(w_q->cols);
    g.max_ctas = r.sms;
    g.pdl = false;
    cuda_check(launch_w4a8_gemm(g, st), "w4a8_gemm launch");
}

void require_per_token_i8(const ody_qtensor* a_q) {  // ref gemm.cpp:26-30
    if (a_q->kind != QKind::Act8) fail(ODY_EINVAL, "GEMM: activations must be symmetric per-token INT8");
}
void check_k(size_t k) {  // ref gemm.cpp:14-20
    if (k > kMaxK) fail(ODY_EINVAL, "GEMM: K exceeds the 32-bit accumulator safety bound 2^17");
}

// The comparison engines (ref gemm.cpp:313-333 run_engine), each in the reference's
// validation order, on the GPU (engine_kernel.cu); counters are the reference's formulas.
// Stream-ordered: out_dev (m x n f32) is written on `st`; a_dev is W4A16's f32
// activations on the device (m rows).
void engine_core(ody_engine engine, const float* a_dev, size_t a_rows, size_t a_cols, const ody_qtensor* a_q,
                 const ody_qtensor* w_q, float* out_dev, ody_gemm_counters* counters, cudaStream_t st) {
    const bool w4 = w_q->kind == QKind::Weight4 || w_q->kind == QKind::Weight4G;
    ody_gemm_counters c = {};
    size_t m = 0, n = w_q->rows, k = w_q->cols;
    if (engine == ODY_ENGINE_W4A16) {  // ref gemm.cpp:100-104
        if (a_cols != w_q->cols) fail(ODY_EINVAL, "gemm_w4a16_grouped: inner dims disagree");
        if (!w4) fail(ODY_EINVAL, "gemm_w4a16_grouped: weights must be 4-bit");
        m = a_rows;
        if (m > 0x7fffffff || n > 0x7fffffff || k > 0x7fffffff) fail(ODY_EINVAL, "GEMM: dimension exceeds int32 range");
        cuda_check(launch_w4a16(a_dev, static_cast<const uint8_t*>(w_q->codes), w_q->scales, static_cast<int>(m),
                                static_cast<int>(n), static_cast<int>(k),
                                static_cast<int>(w_q->kind == QKind::Weight4G ? w_q->group_size : k), out_dev, st),
                   "w4a16 launch");
        c.dequant_events = static_cast<uint64_t>(m) * n * k;
    } else {
        EngineArgs e = {};
        DevBuf<uint8_t> offset(0, st), regroup_w(0, st);
        DevBuf<int8_t> regroup_a(0, st);
        m = a_q->rows;
        e.qa = static_cast<const int8_t*>(a_q->codes);
        e.K = static_cast<int>(k);
        if (engine == ODY_ENGINE_FINEGRAINED) {  // ref gemm.cpp:125-133
            require_per_token_i8(a_q);
            if (a_q->cols != w_q->cols) fail(ODY_EINVAL, "gemm_w4a8_finegrained: inner dims disagree");
            if (!w4) fail(ODY_EINVAL, "gemm_w4a8_finegrained: weights must be 4-bit");
            const size_t g = w_q->kind == QKind::Weight4G ? w_q->group_size : k;
            if (g == 0 || k % g != 0) fail(ODY_EINVAL, "gemm_w4a8_finegrained: g does not divide K");
            check_k(g);
            e.mode = kEngineFine;
            e.group = static_cast<int>(g);
            e.w = static_cast<const uint8_t*>(w_q->codes);
            if (g % 32 != 0) {  // whole MMA k-steps per group: both operands re-laid out
                const size_t g32 = (g + 31) / 32 * 32, kq = (k / g) * g32;
                regroup_w = DevBuf<uint8_t>(w4_packed_bytes(n, kq), st);
                regroup_a = DevBuf<int8_t>(a8_bytes(m, kq), st);
                cuda_check(launch_regroup(e.w, e.qa, static_cast<int>(m), static_cast<int>(n), static_cast<int>(k),
                                          static_cast<int>(g), regroup_w.p, regroup_a.p, st),
                           "finegrained regroup");
                e.w = regroup_w.p;
                e.qa = regroup_a.p;
                e.K = static_cast<int>(kq);
                e.group = static_cast<int>(g32);
            }
            c.int8_mac_ops = static_cast<uint64_t>(m) * n * k;
            c.dequant_events = static_cast<uint64_t>(m) * n * (k / g);
        } else if (engine == ODY_ENGINE_ASYMMETRIC) {  // ref gemm.cpp:320-325, 163-172
            if (w_q->kind != QKind::Weight4) fail(ODY_EINVAL, "asymmetric engine: weights must be per-channel 4-bit");
            require_per_token_i8(a_q);
            if (a_q->cols != k) fail(ODY_EINVAL, "gemm_w4a8_asymmetric: inner dims disagree");
            check_k(k);
            // the reference re-packs to UINT4 + 8 on every call (run_engine): so does this engine
            offset = DevBuf<uint8_t>(w4_packed_bytes(n, k), st);
            cuda_check(launch_w4_offset(static_cast<const uint8_t*>(w_q->codes), static_cast<int>(n),
                                        static_cast<int>(k), offset.p, st),
                       "w4 offset repack");
            e.mode = kEngineAsym;
            e.w = offset.p;
            c.zero_point_sub_ops = static_cast<uint64_t>(n) * k;
            c.int8_mac_ops = static_cast<uint64_t>(m) * n * k;
            c.dequant_events = static_cast<uint64_t>(m) * n;
            c.final_scale_ops = static_cast<uint64_t>(m) * n;
        } else {  // ODY_ENGINE_W8A8, ref gemm.cpp:281-287
            require_per_token_i8(a_q);
            if (w_q->kind != QKind::Weight8) fail(ODY_EINVAL, "gemm_w8a8: weights must be per-channel 8-bit");
            if (a_q->cols != w_q->cols) fail(ODY_EINVAL, "gemm_w8a8: inner dims disagree");
            check_k(k);
            e.mode = kEngineW8A8;
            e.w = static_cast<const uint8_t*>(w_q->codes);
            c.int8_mac_ops = static_cast<uint64_t>(m) * n * k;
            c.dequant_events = static_cast<uint64_t>(m) * n;
            c.final_scale_ops = static_cast<uint64_t>(m) * n;
        }
        if (m > 0x7fffffff || n > 0x7fffffff) fail(ODY_EINVAL, "GEMM: dimension exceeds int32 range");
        e.sw = w_q->scales;
        e.sa = a_q->scales;
        e.out = out_dev;
        e.M = static_cast<int>(m);
        e.N = static_cast<int>(n);
        // split-K sums + tile counters: runtime-owned, zeroed once (the kernel leaves them zeroed)
        const size_t wsb = engine_workspace_bytes(e.mode, e.M, e.N, e.K);
        Runtime& r = rt();
        if (wsb > r.escratch_bytes) {
            if (r.escratch) cuda_check(cudaFreeAsync(r.escratch, st), "cudaFreeAsync");
            r.escratch = nullptr;
            cuda_check(cudaMallocAsync(&r.escratch, wsb, st), "cudaMallocAsync engine workspace");
            cuda_check(cudaMemsetAsync(r.escratch, 0, wsb, st), "memset engine workspace");
            r.escratch_bytes = wsb;
        }
        e.workspace = r.escratch;
        e.workspace_bytes = r.escratch_bytes;
        cuda_check(launch_engine_gemm(e, st), "engine gemm launch");
    }
    if (counters) *counters = c;
}

void run_engine_abi(ody_engine engine, const ody_tensor* a_dense, const ody_qtensor* a_q, const ody_qtensor* w_q,
                    ody_gemm_counters* counters, ody_tensor** out) {
    Runtime& r = rt();
    std::lock_guard<std::mutex> lock(r.mu);
    cudaStream_t st = r.stream;
    const size_t m = engine == ODY_ENGINE_W4A16 ? a_dense->rows : a_q->rows, n = w_q->rows;
    DevBuf<float> od(m * n, st);
    DevBuf<float> ad(engine == ODY_ENGINE_W4A16 ? a_dense->rows * a_dense->cols : 0, st);
    if (engine == ODY_ENGINE_W4A16)
        cuda_check(cudaMemcpyAsync(ad.p, a_dense->data, a_dense->rows * a_dense->cols * 4, cudaMemcpyHostToDevice, st),
                   "H2D a");
    engine_core(engine, ad.p, engine == ODY_ENGINE_W4A16 ? a_dense->rows : 0,
                engine == ODY_ENGINE_W4A16 ? a_dense->cols : 0, a_q, w_q, od.p, counters, st);
    ody_tensor* t = new_tensor(m, n);
    cudaError_t err = cudaMemcpyAsync(t->data, od.p, m * n * 4, cudaMemcpyDeviceToHost, st);
    if (err == cudaSuccess) err = cudaGetLastError();
    if (err == cudaSuccess) err = cudaStreamSynchronize(st);
    if (err != cudaSuccess) {
        delete t;
        cuda_check(err, "ody_gemm");
    }
    *out = t;
}

}  // namespace

extern "C" {

// ================================================================ part 1
const char* ody_last_error(void) { return g_last_error.c_str(); }

void ody_string_free(char* s) { delete[] s; }

// ref: ody_set_threads sizes the CPU engine's pool; here the host pool of the ABI's copies
void ody_set_threads(int n) { HostPool::get().set_threads(n); }

ody_status ody_tensor_create(size_t rows, size_t cols, const float* data, ody_tensor** out) {
    return ody_tensor_create_strided(rows, cols, cols, data, out);
}

ody_status ody_tensor_create_strided(size_t rows, size_t cols, size_t ld, const float* data, ody_tensor** out) {
    if (!data || !out) return einval("ody_tensor_create: null argument");
    if (ld < cols && rows > 1) return einval("ody_tensor_create_strided: ld < cols");
    return guarded([&] {
        // ref tensor.cpp:21-27 (reject NaN/Inf), fused with the copy into pinned memory
        ody_tensor* t = new_tensor(rows, cols);
        if (rows * cols > 0 && !copy_finite(t->data, data, rows, cols, rows > 1 ? ld : cols)) {
            delete t;
            fail(ODY_EINVAL, "DenseTensor: non-finite value");
        }
        *out = t;
    });
}

void ody_tensor_free(ody_tensor* t) { delete t; }

ody_status ody_tensor_dims(const ody_tensor* t, size_t* rows, size_t* cols) {
    if (!t || !rows || !cols) return einval("ody_tensor_dims: null argument");
    *rows = t->rows;
    *cols = t->cols;
    return ODY_OK;
}

ody_status ody_tensor_data(const ody_tensor* t, const float** data) {
    if (!t || !data) return einval("ody_tensor_data: null argument");
    *data = t->data;
    return ODY_OK;
}

void ody_qtensor_free(ody_qtensor* q) {
    if (!q) return;
    try {
        delete q;
    } catch (...) {
    }
}

ody_status ody_qtensor_dims(const ody_qtensor* q, size_t* rows, size_t* cols) {
    if (!q || !rows || !cols) return einval("ody_qtensor_dims: null argument");
    *rows = q->rows;
    *cols = q->cols;
    return ODY_OK;
}

ody_status ody_quantize_weights(const ody_tensor* w, int bits, ody_granularity granularity,
                                size_t group_size, const float* clip_gamma,
                                const float* clip_beta, ody_qtensor** out) {
    if (!w || !out) return einval("ody_quantize_weights: null argument");
    return guarded([&] {
        // validation order of ref quantize.cpp:75-83 / tensor.cpp:86-110
        if (w->rows * w->cols == 0) fail(ODY_EINVAL, "quantize_weights: empty tensor");
        if (granularity != ODY_PER_CHANNEL && granularity != ODY_PER_GROUP)
            fail(ODY_EINVAL, "quantize_weights: granularity must be per_channel or per_group");
        if (bits != 4 && bits != 8) fail(ODY_EINVAL, "QuantScheme: bits must be 4 or 8");
        if (granularity == ODY_PER_GROUP && (group_size == 0 || w->cols % group_size != 0))
            fail(ODY_EINVAL, "QuantScheme: group size " + std::to_string(group_size) +
                                 " does not divide axis length " + std::to_string(w->cols));
        for (const float* arr : {clip_gamma, clip_beta}) {
            if (!arr) continue;
            for (size_t i = 0; i < w->rows; ++i)
                if (!(arr[i] > 0.0f && arr[i] <= 1.0f))
                    fail(ODY_EINVAL, std::string("QuantScheme: ") +
                                         (arr == clip_gamma ? "clip_gamma" : "clip_beta") +
                                         " outside (0,1]");
        }
        if (bits == 8 && granularity == ODY_PER_GROUP)
            fail(ODY_EINVAL, "quantize_weights: 8-bit per_group weights feed no engine of the B200 path");
        if (w->rows > 0x7fffffff || w->cols > 0x7fffffff) fail(ODY_EINVAL, "quantize_weights: too large");
        Runtime& r = rt();
        cudaStream_t st = r.stream;
        const size_t n = w->rows, k = w->cols;
        const QKind kind = bits == 8 ? QKind::Weight8 : (granularity == ODY_PER_GROUP ? QKind::Weight4G : QKind::Weight4);
        const size_t groups = kind == QKind::Weight4G ? k / group_size : 1;
        DevBuf<float> wd(n * k, st);
        cuda_check(cudaMemcpyAsync(wd.p, w->data, n * k * 4, cudaMemcpyHostToDevice, st), "H2D w");
        DevBuf<float> gd(clip_gamma ? n : 0, st), bd(clip_beta ? n : 0, st);
        if (clip_gamma) cuda_check(cudaMemcpyAsync(gd.p, clip_gamma, n * 4, cudaMemcpyHostToDevice, st), "H2D");
        if (clip_beta) cuda_check(cudaMemcpyAsync(bd.p, clip_beta, n * 4, cudaMemcpyHostToDevice, st), "H2D");
        DevBuf<uint8_t> packed(kind == QKind::Weight8 ? w8_bytes(n, k) : w4_packed_bytes(n, k), st);
        DevBuf<float> scales(n * groups, st);
        DevBuf<int> err(1, st);
        cuda_check(cudaMemsetAsync(err.p, 0, sizeof(int), st), "memset");
        const float* g = clip_gamma ? gd.p : nullptr;
        const float* b = clip_beta ? bd.p : nullptr;
        if (kind == QKind::Weight4)
            cuda_check(launch_w4_quant_prepack(wd.p, static_cast<int>(n), static_cast<int>(k), 4, g, b, packed.p,
                                               scales.p, err.p, st),
                       "w4 quantize launch");
        else if (kind == QKind::Weight4G)  // gamma/beta validated on the host above
            cuda_check(launch_wg_quant_prepack(wd.p, static_cast<int>(n), static_cast<int>(k),
                                               static_cast<int>(group_size), 4, g, b, packed.p, scales.p, st),
                       "w4 per-group quantize launch");
        else
            cuda_check(launch_w8_quant(wd.p, static_cast<int>(n), static_cast<int>(k), g, b,
                                       reinterpret_cast<int8_t*>(packed.p), scales.p, err.p, st),
                       "w8 quantize launch");
        int herr = 0;
        cuda_check(cudaMemcpyAsync(&herr, err.p, sizeof(int), cudaMemcpyDeviceToHost, st), "D2H");
        sync(st, "ody_quantize_weights");
        if (herr) fail(ODY_EINVAL, "compute_scale_symmetric: gamma/beta outside (0,1]");
        auto* q = new ody_qtensor();
        q->kind = kind;
        q->rows = n;
        q->cols = k;
        q->group_size = group_size;
        q->codes = packed.release();
        q->scales = scales.release();
        *out = q;
    });
}

ody_status ody_quantize_activations(const ody_tensor* a, ody_qtensor** out) {
    if (!a || !out) return einval("ody_quantize_activations: null argument");
    return guarded([&] {
        if (a->rows * a->cols == 0)
            fail(ODY_EINVAL, "quantize_activations_per_token: empty tensor");
        if (a->rows > 0x7fffffff || a->cols > 0x7fffffff) fail(ODY_EINVAL, "too large");
        Runtime& r = rt();
        cudaStream_t st = r.stream;
        const size_t m = a->rows, k = a->cols;
        DevBuf<float> xd(m * k, st);
        cuda_check(cudaMemcpyAsync(xd.p, a->data, m * k * 4, cudaMemcpyHostToDevice, st), "H2D a");
        DevBuf<int8_t> q(a8_bytes(m, k), st);
        DevBuf<float> s(m, st);
        cuda_check(launch_act_quant(xd.p, kDtypeF32, k, static_cast<int>(m), static_cast<int>(k),
                                    q.p, s.p, nullptr, nullptr, false, st),
                   "act_quant launch");
        // no synchronize: the qtensor lives on the library stream (every later use is
        // ordered after this launch) and the source tensor's pinned buffer is only reused
        // after the stream passed this copy (PinnedPool)
        auto* qt = new ody_qtensor();
        qt->kind = QKind::Act8;
        qt->rows = m;
        qt->cols = k;
        qt->codes = q.release();
        qt->scales = s.release();
        *out = qt;
    });
}

ody_status ody_dequantize(const ody_qtensor* q, ody_tensor** out) {
    if (!q || !out) return einval("ody_dequantize: null argument");
    return guarded([&] {
        cudaStream_t st = rt().stream;
        const size_t r = q->rows, c = q->cols;
        DevBuf<float> d(r * c, st);
        if (q->kind == QKind::Act8 || q->kind == QKind::Weight8)  // W8 is the a8 layout over the rows
            cuda_check(launch_a8_unpack(static_cast<const int8_t*>(q->codes), q->scales,
                                        static_cast<int>(r), static_cast<int>(c), nullptr, d.p, st),
                       "dequant launch");
        else if (q->kind == QKind::Weight4G)
            cuda_check(launch_wg_dequant(static_cast<const uint8_t*>(q->codes), q->scales, static_cast<int>(r),
                                         static_cast<int>(c), static_cast<int>(q->group_size), d.p, st),
                       "dequant launch");
        else
            cuda_check(launch_w4_dequant(static_cast<const uint8_t*>(q->codes), q->scales,
                                         static_cast<int>(r), static_cast<int>(c), d.p, st),
                       "dequant launch");
        ody_tensor* t = new_tensor(r, c);
        cudaError_t e = cudaMemcpyAsync(t->data, d.p, r * c * 4, cudaMemcpyDeviceToHost, st);
        if (e == cudaSuccess) e = cudaStreamSynchronize(st);
        if (e != cudaSuccess) {
            delete t;
            cuda_check(e, "ody_dequantize");
        }
        *out = t;
    });
}

ody_status ody_gemm(ody_engine engine, const ody_tensor* a_dense, const ody_qtensor* a_q,
                    const ody_qtensor* w_q, ody_gemm_counters* counters, ody_tensor** out) {
    if (!w_q || !out) return einval("ody_gemm: null argument");
    return guarded([&] {
        // ref capi.cpp:276-283
        if (engine < ODY_ENGINE_W4A16 || engine > ODY_ENGINE_W8A8)
            fail(ODY_EINVAL, "bad engine enum");
        if (engine == ODY_ENGINE_W4A16 && !a_dense)
            fail(ODY_EINVAL, "ody_gemm: w4a16 engine needs a_dense");
        if (engine != ODY_ENGINE_W4A16 && !a_q)
            fail(ODY_EINVAL, "ody_gemm: engine needs quantized activations");
        if (engine != ODY_ENGINE_FAST) {
            run_engine_abi(engine, a_dense, a_q, w_q, counters, out);
            return;
        }
        check_fast_inputs(a_q, w_q);
        Runtime& r = rt();
        std::lock_guard<std::mutex> lock(r.mu);
        cudaStream_t st = r.stream;
        const size_t m = a_q->rows, n = w_q->rows, k = w_q->cols;
        if (gemm_prequant_eligible(static_cast<int>(m), static_cast<int>(n), static_cast<int>(k))) {
            // decode widths: the epilogue stores the f32 outputs straight into the result
            // tensor's pinned (host-mapped) buffer over PCIe while the weights stream -- no
            // device output buffer and no D2H copy after the kernel
            ody_tensor* t = new_tensor(m, n);
            void* mapped = nullptr;
            if (cudaHostGetDevicePointer(&mapped, t->data, 0) == cudaSuccess && mapped) {
                cudaError_t e = cudaSuccess;
                try {
                    run_gemm(a_q, w_q, static_cast<float*>(mapped), nullptr, st);
                } catch (...) {
                    delete t;
                    throw;
                }
                e = cudaGetLastError();
                if (e == cudaSuccess) e = cudaStreamSynchronize(st);
                if (e != cudaSuccess) {
                    delete t;
                    cuda_check(e, "ody_gemm");
                }
                if (counters) {  // ref gemm.cpp:270-272
                    counters->int8_mac_ops = static_cast<uint64_t>(m) * n * k;
                    counters->dequant_events = static_cast<uint64_t>(m) * n;
                    counters->zero_point_sub_ops = 0;
                    counters->final_scale_ops = static_cast<uint64_t>(m) * n;
                }
                *out = t;
                return;
            }
            cudaGetLastError();  // not pinned (pool fell back to pageable memory)
            delete t;
        }
        DevBuf<float> od(m * n, st);
        run_gemm(a_q, w_q, od.p, nullptr, st);
        ody_tensor* t = new_tensor(m, n);
        cudaError_t e = cudaMemcpyAsync(t->data, od.p, m * n * 4, cudaMemcpyDeviceToHost, st);
        if (e == cudaSuccess) e = cudaGetLastError();
        if (e == cudaSuccess) e = cudaStreamSynchronize(st);
        if (e != cudaSuccess) {
            delete t;
            cuda_check(e, "ody_gemm");
        }
        if (counters) {  // ref gemm.cpp:270-272 -- analytic, identical to the CPU engine
            counters->int8_mac_ops = static_cast<uint64_t>(m) * n * k;
            counters->dequant_events = static_cast<uint64_t>(m) * n;
            counters->zero_point_sub_ops = 0;
            counters->final_scale_ops = static_cast<uint64_t>(m) * n;
        }
        *out = t;
    });
}

ody_status ody_gemm_dev(ody_engine engine, const float* a_dev, size_t a_rows, const ody_qtensor* a_q,
                        const ody_qtensor* w_q, float* out_dev, ody_gemm_counters* counters, void* stream) {
    if (!w_q || !out_dev) return einval("ody_gemm_dev: null argument");
    return guarded([&] {
        if (engine < ODY_ENGINE_W4A16 || engine > ODY_ENGINE_W8A8) fail(ODY_EINVAL, "bad engine enum");
        if (engine == ODY_ENGINE_W4A16 && !a_dev) fail(ODY_EINVAL, "ody_gemm_dev: w4a16 engine needs a_dev");
        if (engine != ODY_ENGINE_W4A16 && !a_q) fail(ODY_EINVAL, "ody_gemm_dev: engine needs quantized activations");
        cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : rt().stream;
        if (engine == ODY_ENGINE_FAST) {
            check_fast_inputs(a_q, w_q);
            run_gemm(a_q, w_q, out_dev, nullptr, st);
            if (counters) {
                const uint64_t m = a_q->rows, n = w_q->rows, k = w_q->cols;
                *counters = {m * n * k, m * n, 0, m * n};
            }
        } else {
            engine_core(engine, a_dev, a_rows, w_q->cols, a_q, w_q, out_dev, counters, st);
        }
        cuda_check(cudaGetLastError(), "ody_gemm_dev");
    });
}

// ================================================================ part 2
size_t ody_dev_a8_bytes(size_t m, size_t k) { return a8_bytes(m, k); }
size_t ody_dev_w4_bytes(size_t n, size_t k) { return w4_packed_bytes(n, k); }
size_t ody_dev_workspace_bytes(size_t m, size_t n, size_t k) {
    return gemm_workspace_bytes(static_cast<int>(m), static_cast<int>(n), static_cast<int>(k), 0);
}

ody_status ody_dev_act_quant(const void* x, ody_dtype dtype, size_t ldx, size_t m, size_t k,
                             void* q, float* s, const float* absmax_in, float* absmax_out,
                             int pdl, void* stream) {
    if (!x || !q || !s) return einval("ody_dev_act_quant: null argument");
    if (m == 0 || k == 0) return einval("quantize_activations_per_token: empty tensor");
    if (ldx < k) return einval("ody_dev_act_quant: ldx < k");
    return guarded([&] {
        cuda_check(launch_act_quant(x, dtype, ldx, static_cast<int>(m), static_cast<int>(k),
                                    static_cast<int8_t*>(q), s, absmax_in, absmax_out, pdl != 0,
                                    static_cast<cudaStream_t>(stream)),
                   "act_quant launch");
    });
}

ody_status ody_dev_row_absmax(const void* x, ody_dtype dtype, size_t ldx, size_t m, size_t k,
                              float* absmax, void* stream) {
    if (!x || !absmax) return einval("ody_dev_row_absmax: null argument");
    if (m == 0 || k == 0) return einval("ody_dev_row_absmax: empty tensor");
    return guarded([&] {
        cuda_check(launch_row_absmax(x, dtype, ldx, static_cast<int>(m), static_cast<int>(k), absmax,
                                     static_cast<cudaStream_t>(stream)),
                   "row_absmax launch");
    });
}

ody_status ody_dev_w4_quantize(const float* w, size_t n, size_t k, const float* gamma,
                               const float* beta, void* w_packed, float* s_w, void* stream) {
    if (!w || !w_packed || !s_w) return einval("ody_dev_w4_quantize: null argument");
    if (n == 0 || k == 0) return einval("quantize_weights: empty tensor");
    return guarded([&] {
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        if (!gamma && !beta) {
            cuda_check(launch_w4_quant_prepack(w, static_cast<int>(n), static_cast<int>(k), 4, nullptr, nullptr,
                                               static_cast<uint8_t*>(w_packed), s_w, nullptr, st),
                       "w4 quantize launch");
            return;
        }
        // clip factors (device arrays) are validated on the device as the scales are
        // computed (ref quantize.cpp:22-35 / tensor.cpp:86-110: gamma, beta in (0, 1]);
        // the offline weight path then synchronizes once to report EINVAL like the reference
        DevBuf<int> err(1, st);
        cuda_check(cudaMemsetAsync(err.p, 0, sizeof(int), st), "memset");
        cuda_check(launch_w4_quant_prepack(w, static_cast<int>(n), static_cast<int>(k), 4, gamma, beta,
                                           static_cast<uint8_t*>(w_packed), s_w, err.p, st),
                   "w4 quantize launch");
        int herr = 0;
        cuda_check(cudaMemcpyAsync(&herr, err.p, sizeof(int), cudaMemcpyDeviceToHost, st), "D2H");
        cuda_check(cudaStreamSynchronize(st), "ody_dev_w4_quantize");
        if (herr) fail(ODY_EINVAL, "compute_scale_symmetric: gamma/beta outside (0,1]");
    });
}

ody_status ody_dev_w4_quantize_with_scales(const float* w, size_t n, size_t k, const float* s_w,
                                           void* w_packed, void* stream) {
    if (!w || !w_packed || !s_w) return einval("ody_dev_w4_quantize_with_scales: null argument");
    if (n == 0 || k == 0) return einval("quantize_weights: empty tensor");
    return guarded([&] {
        cuda_check(launch_w4_quant_prepack(w, static_cast<int>(n), static_cast<int>(k), 4, nullptr,
                                           nullptr, static_cast<uint8_t*>(w_packed),
                                           const_cast<float*>(s_w), nullptr,
                                           static_cast<cudaStream_t>(stream), true),
                   "w4 quantize launch");
    });
}

ody_status ody_dev_dequant_epilogue(const int32_t* acc, const float* s_a, const float* s_w,
                                    size_t m, size_t n, ody_dtype out_dtype, void* out,
                                    void* stream) {
    if (!acc || !s_a || !s_w || !out) return einval("ody_dev_dequant_epilogue: null argument");
    if (out_dtype < ODY_DTYPE_F32 || out_dtype > ODY_DTYPE_BF16) return einval("bad out dtype");
    return guarded([&] {
        cuda_check(launch_dequant_epilogue(acc, s_a, s_w, static_cast<int>(m), static_cast<int>(n),
                                           static_cast<int>(out_dtype), out,
                                           static_cast<cudaStream_t>(stream)),
                   "epilogue launch");
    });
}

ody_status ody_dev_w4_prepack(const void* flat, size_t n, size_t k, void* w_packed, void* stream) {
    if (!flat || !w_packed) return einval("ody_dev_w4_prepack: null argument");
    return guarded([&] {
        cuda_check(launch_w4_prepack_flat(static_cast<const uint8_t*>(flat), static_cast<int>(n),
                                          static_cast<int>(k), static_cast<uint8_t*>(w_packed),
                                          static_cast<cudaStream_t>(stream)),
                   "w4 prepack launch");
    });
}

ody_status ody_dev_w4_unpack(const void* w_packed, size_t n, size_t k, void* flat, void* stream) {
    if (!flat || !w_packed) return einval("ody_dev_w4_unpack: null argument");
    return guarded([&] {
        cuda_check(launch_w4_unpack_flat(static_cast<const uint8_t*>(w_packed), static_cast<int>(n),
                                         static_cast<int>(k), static_cast<uint8_t*>(flat),
                                         static_cast<cudaStream_t>(stream)),
                   "w4 unpack launch");
    });
}

ody_status ody_dev_w4a8_gemm(const void* q, const float* s_a, const void* w_packed,
                             const float* s_w, size_t m, size_t n, size_t k, ody_dtype out_dtype,
                             void* out, int32_t* acc_out, void* workspace, size_t workspace_bytes,
                             int max_ctas, int pdl, void* stream) {
    if (!q || !s_a || !w_packed || !s_w || (!out && !acc_out) || !workspace)
        return einval("ody_dev_w4a8_gemm: null argument");
    if (m == 0 || n == 0 || k == 0) return einval("ody_dev_w4a8_gemm: empty operand");
    if (k > kMaxK) return einval("GEMM: K exceeds the 32-bit accumulator safety bound 2^17");
    if (out_dtype < ODY_DTYPE_F32 || out_dtype > ODY_DTYPE_BF16) return einval("bad out dtype");
    return guarded([&] {
        GemmArgs g = {};
        g.qa = static_cast<const int8_t*>(q);
        g.sa = s_a;
        g.wp = static_cast<const uint8_t*>(w_packed);
        g.sw = s_w;
        g.out = out;
        g.out_dtype = static_cast<int>(out_dtype);
        g.acc_out = acc_out;
        g.workspace = workspace;
        g.workspace_bytes = workspace_bytes;
        g.M = static_cast<int>(m);
        g.N = static_cast<int>(n);
        g.K = static_cast<int>(k);
        g.max_ctas = max_ctas;
        g.pdl = pdl != 0;
        g.trace = g_trace;
        if (workspace_bytes < gemm_workspace_bytes(g.M, g.N, g.K, max_ctas > 0 ? max_ctas : r_sms()))
            fail(ODY_EINVAL, "ody_dev_w4a8_gemm: workspace too small");
        cuda_check(launch_w4a8_gemm(g, static_cast<cudaStream_t>(stream)), "w4a8_gemm launch");
    });
}

void ody_dev_set_trace(void* buf) { g_trace = static_cast<unsigned long long*>(buf); }
void ody_dev_set_act_trace(void* buf) { set_act_trace(static_cast<unsigned long long*>(buf)); }

namespace {

bool program_args(const ody_linear_desc* lin, int count, int max_ctas, std::vector<LinearArgs>* a,
                  std::vector<int>* deps) {
    a->assign(count, LinearArgs{});
    deps->assign(count, -1);
    for (int l = 0; l < count; ++l) {
        const ody_linear_desc& d = lin[l];
        LinearArgs& x = (*a)[l];
        x.x = d.x;
        x.x_dtype = static_cast<int>(d.x_dtype);
        x.ldx = d.ldx;
        x.wp = static_cast<const uint8_t*>(d.w_packed);
        x.sw = d.s_w;
        x.out = d.out;
        x.out_dtype = static_cast<int>(d.out_dtype);
        x.sa_out = d.s_a_out;
        x.M = static_cast<int>(d.m);
        x.N = static_cast<int>(d.n);
        x.K = static_cast<int>(d.k);
        x.max_ctas = max_ctas;
        x.trace = g_trace;
        x.absmax_in = d.absmax_in;
        x.acc_out = d.acc_out;
        (*deps)[l] = d.dep;
    }
    return true;
}
}  // namespace

size_t ody_dev_program_workspace_bytes(const ody_linear_desc* lin, int count) {
    if (!lin || count < 1 || count > kProgramMaxLinears) return 0;
    size_t need = 0;
    for (int l = 0; l < count; ++l)
        need = std::max(need, linear_scratch_bytes(static_cast<int>(lin[l].m), static_cast<int>(lin[l].n),
                                                   static_cast<int>(lin[l].k), 0));
    std::vector<LinearArgs> a;
    std::vector<int> deps;
    program_args(lin, count, 0, &a, &deps);
    // the fallback runs each linear on the same buffer (same zero-region layout)
    return std::max(need, program_scratch_bytes(a.data(), deps.data(), count));
}

int ody_dev_program_is_fused(const ody_linear_desc* lin, int count) {
    if (!lin || count < 1 || count > kProgramMaxLinears) return 0;
    std::vector<LinearArgs> a;
    std::vector<int> deps;
    program_args(lin, count, 0, &a, &deps);
    return linear_mode() == 2 && program_eligible(a.data(), deps.data(), count, 0) ? 1 : 0;
}

namespace {
ody_status program_check(const ody_linear_desc* lin, int count, void* workspace, size_t workspace_bytes) {
    if (!lin || !workspace) return einval("ody_dev_w4a8_linear_program: null argument");
    if (count < 1 || count > kProgramMaxLinears)
        return einval("ody_dev_w4a8_linear_program: 1..8 linears per program");
    for (int l = 0; l < count; ++l) {
        const ody_linear_desc& d = lin[l];
        if (!d.x || !d.w_packed || !d.s_w || (!d.out && !d.acc_out))
            return einval("ody_dev_w4a8_linear_program: null argument");
        if (d.absmax_in && d.dep >= 0)
            return einval("ody_dev_w4a8_linear_program: absmax_in applies to external activations only");
        if (d.m == 0 || d.n == 0 || d.k == 0) return einval("ody_dev_w4a8_linear_program: empty operand");
        if (d.ldx < d.k) return einval("ody_dev_w4a8_linear_program: ldx < k");
        if (d.k > kMaxK) return einval("GEMM: K exceeds the 32-bit accumulator safety bound 2^17");
        if (d.dep < -1 || d.dep >= l) return einval("ody_dev_w4a8_linear_program: dep must name an earlier linear");
        if (d.x_dtype < ODY_DTYPE_F32 || d.x_dtype > ODY_DTYPE_BF16 || d.out_dtype < ODY_DTYPE_F32 ||
            d.out_dtype > ODY_DTYPE_BF16)
            return einval("bad dtype");
    }
    if (workspace_bytes < ody_dev_program_workspace_bytes(lin, count))
        return einval("ody_dev_w4a8_linear_program: workspace too small");
    return ODY_OK;
}
}  // namespace

int ody_dev_chain_is_links(const ody_linear_desc* lin, int count) {
    if (!lin || count < 1 || count > kProgramMaxLinears) return 0;
    std::vector<LinearArgs> a;
    std::vector<int> deps;
    program_args(lin, count, 0, &a, &deps);
    return chain_links_eligible(a.data(), deps.data(), count) ? 1 : 0;
}

ody_status ody_dev_w4a8_linear_chain(const ody_linear_desc* lin, int count, void* workspace,
                                     size_t workspace_bytes, int max_ctas, int pdl, void* stream) {
    const ody_status c = program_check(lin, count, workspace, workspace_bytes);
    if (c != ODY_OK) return c;
    std::vector<LinearArgs> a;
    std::vector<int> deps;
    program_args(lin, count, max_ctas, &a, &deps);
    if (!chain_links_eligible(a.data(), deps.data(), count))  // same results, as a program
        return ody_dev_w4a8_linear_program(lin, count, workspace, workspace_bytes, max_ctas, pdl, nullptr, 0,
                                           stream);
    return guarded([&] {
        cuda_check(launch_w4a8_chain_links(a.data(), deps.data(), count, workspace, workspace_bytes, pdl != 0,
                                           static_cast<cudaStream_t>(stream)),
                   "w4a8 chain links launch");
    });
}

ody_status ody_dev_w4a8_linear_program(const ody_linear_desc* lin, int count, void* workspace,
                                       size_t workspace_bytes, int max_ctas, int pdl,
                                       const void* next_w, size_t next_w_bytes, void* stream) {
    const ody_status c = program_check(lin, count, workspace, workspace_bytes);
    if (c != ODY_OK) return c;
    return guarded([&] {
        std::vector<LinearArgs> a;
        std::vector<int> deps;
        program_args(lin, count, max_ctas, &a, &deps);
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        if (linear_mode() == 2 && program_eligible(a.data(), deps.data(), count, max_ctas)) {
            cuda_check(launch_w4a8_program(a.data(), deps.data(), count, workspace, workspace_bytes, pdl != 0,
                                           static_cast<const uint8_t*>(next_w), next_w ? next_w_bytes : 0, st),
                       "w4a8 linear program launch");
            return;
        }
        for (int l = 0; l < count; ++l) {
            a[l].workspace = workspace;
            a[l].workspace_bytes = workspace_bytes;
            a[l].pdl = pdl != 0;
            cuda_check(launch_w4a8_linear(a[l], st), "w4a8_linear launch");
        }
    });
}

size_t ody_dev_linear_workspace_bytes(size_t m, size_t n, size_t k) {
    return linear_scratch_bytes(static_cast<int>(m), static_cast<int>(n), static_cast<int>(k), 0);
}

void ody_dev_set_linear_mode(int mode) { set_linear_mode(mode); }
void ody_dev_set_prefill_min_m(int m) { set_prefill_min_m(m); }

int ody_dev_linear_is_fused(size_t m, size_t n, size_t k) {
    return linear_is_fused(static_cast<int>(m), static_cast<int>(n), static_cast<int>(k), 0) ? 1 : 0;
}

ody_status ody_dev_w4a8_linear(const void* x, ody_dtype x_dtype, size_t ldx, const void* w_packed,
                               const float* s_w, size_t m, size_t n, size_t k, ody_dtype out_dtype,
                               void* out, float* s_a_out, void* workspace, size_t workspace_bytes,
                               int max_ctas, int pdl, void* stream) {
    return ody_dev_w4a8_linear_pf(x, x_dtype, ldx, w_packed, s_w, m, n, k, out_dtype, out, s_a_out,
                                  workspace, workspace_bytes, max_ctas, pdl, nullptr, 0, stream);
}

ody_status ody_dev_w4a8_linear_pf(const void* x, ody_dtype x_dtype, size_t ldx, const void* w_packed,
                                  const float* s_w, size_t m, size_t n, size_t k, ody_dtype out_dtype,
                                  void* out, float* s_a_out, void* workspace, size_t workspace_bytes,
                                  int max_ctas, int pdl, const void* next_w, size_t next_w_bytes,
                                  void* stream) {
    if (!x || !w_packed || !s_w || !out || !workspace)
        return einval("ody_dev_w4a8_linear: null argument");
    if (m == 0 || n == 0 || k == 0) return einval("ody_dev_w4a8_linear: empty operand");
    if (ldx < k) return einval("ody_dev_w4a8_linear: ldx < k");
    if (k > kMaxK) return einval("GEMM: K exceeds the 32-bit accumulator safety bound 2^17");
    if (x_dtype < ODY_DTYPE_F32 || x_dtype > ODY_DTYPE_BF16 || out_dtype < ODY_DTYPE_F32 ||
        out_dtype > ODY_DTYPE_BF16)
        return einval("bad dtype");
    return guarded([&] {
        LinearArgs a = {};
        a.x = x;
        a.x_dtype = static_cast<int>(x_dtype);
        a.ldx = ldx;
        a.wp = static_cast<const uint8_t*>(w_packed);
        a.sw = s_w;
        a.out = out;
        a.out_dtype = static_cast<int>(out_dtype);
        a.sa_out = s_a_out;
        a.workspace = workspace;
        a.workspace_bytes = workspace_bytes;
        a.M = static_cast<int>(m);
        a.N = static_cast<int>(n);
        a.K = static_cast<int>(k);
        a.max_ctas = max_ctas;
        a.pdl = pdl != 0;
        a.next_wp = static_cast<const uint8_t*>(next_w);
        a.next_bytes = next_w ? next_w_bytes : 0;
        a.trace = g_trace;
        if (workspace_bytes < linear_scratch_bytes(a.M, a.N, a.K, max_ctas > 0 ? max_ctas : r_sms()))
            fail(ODY_EINVAL, "ody_dev_w4a8_linear: workspace too small");
        cuda_check(launch_w4a8_linear(a, static_cast<cudaStream_t>(stream)), "w4a8_linear launch");
    });
}

ody_status ody_dev_workspace_init(void* workspace, size_t bytes, void* stream) {
    if (!workspace) return einval("ody_dev_workspace_init: null argument");
    return guarded([&] {
        cuda_check(cudaMemsetAsync(workspace, 0, bytes, static_cast<cudaStream_t>(stream)),
                   "workspace memset");
    });
}

ody_status ody_dev_a8_unpack(const void* q, const float* s, size_t m, size_t k, int8_t* codes,
                             float* dequant, void* stream) {
    if (!q || (!codes && !dequant) || (dequant && !s)) return einval("ody_dev_a8_unpack: null argument");
    return guarded([&] {
        cuda_check(launch_a8_unpack(static_cast<const int8_t*>(q), s, static_cast<int>(m),
                                    static_cast<int>(k), codes, dequant,
                                    static_cast<cudaStream_t>(stream)),
                   "a8 unpack launch");
    });
}

// ================================================================ part 3
ody_status ody_qtensor_export(const ody_qtensor* q, void* codes_or_nibbles, float* scales) {
    if (!q) return einval("ody_qtensor_export: null argument");
    return guarded([&] {
        cudaStream_t st = rt().stream;
        const size_t r = q->rows, c = q->cols;
        if (codes_or_nibbles) {
            if (q->kind == QKind::Act8 || q->kind == QKind::Weight8) {
                DevBuf<int8_t> d(r * c, st);
                cuda_check(launch_a8_unpack(static_cast<const int8_t*>(q->codes), q->scales,
                                            static_cast<int>(r), static_cast<int>(c), d.p, nullptr, st),
                           "a8 unpack");
                cuda_check(cudaMemcpyAsync(codes_or_nibbles, d.p, r * c, cudaMemcpyDeviceToHost, st), "D2H");
                sync(st, "ody_qtensor_export");
            } else {
                const size_t nb = (r * c + 1) / 2;
                DevBuf<uint8_t> d(nb, st);
                cuda_check(launch_w4_unpack_flat(static_cast<const uint8_t*>(q->codes),
                                                 static_cast<int>(r), static_cast<int>(c), d.p, st),
                           "w4 unpack");
                cuda_check(cudaMemcpyAsync(codes_or_nibbles, d.p, nb, cudaMemcpyDeviceToHost, st), "D2H");
                sync(st, "ody_qtensor_export");
            }
        }
        if (scales) {
            cuda_check(cudaMemcpyAsync(scales, q->scales, r * q->groups() * 4, cudaMemcpyDeviceToHost, st), "D2H");
            sync(st, "ody_qtensor_export");
        }
    });
}

ody_status ody_qtensor_scheme(const ody_qtensor* q, int* bits, ody_granularity* granularity, size_t* group_size) {
    if (!q || !bits || !granularity || !group_size) return einval("ody_qtensor_scheme: null argument");
    *bits = q->bits();
    *granularity = q->kind == QKind::Act8 ? ODY_PER_TOKEN : (q->kind == QKind::Weight4G ? ODY_PER_GROUP : ODY_PER_CHANNEL);
    *group_size = q->group_size;
    return ODY_OK;
}

ody_status ody_qtensor_import_w4(size_t n, size_t k, const void* flat, const float* scales,
                                 ody_qtensor** out) {
    if (!flat || !scales || !out) return einval("ody_qtensor_import_w4: null argument");
    if (n == 0 || k == 0) return einval("ody_qtensor_import_w4: empty tensor");
    return guarded([&] {
        for (size_t i = 0; i < n; ++i)  // ref tensor.cpp:161-165
            if (!(scales[i] > 0.0f) || !std::isfinite(scales[i]))
                fail(ODY_EINVAL, "QuantizedTensor: non-positive scale");
        cudaStream_t st = rt().stream;
        const size_t nb = (n * k + 1) / 2;
        DevBuf<uint8_t> fd(nb, st);
        cuda_check(cudaMemcpyAsync(fd.p, flat, nb, cudaMemcpyHostToDevice, st), "H2D");
        DevBuf<uint8_t> packed(w4_packed_bytes(n, k), st);
        DevBuf<float> sd(n, st);
        cuda_check(cudaMemcpyAsync(sd.p, scales, n * 4, cudaMemcpyHostToDevice, st), "H2D");
        cuda_check(launch_w4_prepack_flat(fd.p, static_cast<int>(n), static_cast<int>(k), packed.p, st),
                   "w4 prepack");
        sync(st, "ody_qtensor_import_w4");
        auto* q = new ody_qtensor();
        q->kind = QKind::Weight4;
        q->rows = n;
        q->cols = k;
        q->codes = packed.release();
        q->scales = sd.release();
        *out = q;
    });
}

ody_status ody_qtensor_import_a8(size_t m, size_t k, const int8_t* codes, const float* scales,
                                 ody_qtensor** out) {
    if (!codes || !scales || !out) return einval("ody_qtensor_import_a8: null argument");
    if (m == 0 || k == 0) return einval("ody_qtensor_import_a8: empty tensor");
    return guarded([&] {
        for (size_t i = 0; i < m; ++i)
            if (!(scales[i] > 0.0f) || !std::isfinite(scales[i]))
                fail(ODY_EINVAL, "QuantizedTensor: non-positive scale");
        // layout transform of imported codes (import utility, not the hot path)
        const size_t mp = pad_m(m), bytes = a8_bytes(m, k);
        std::vector<int8_t> host(bytes, 0);
        for (size_t t = 0; t < m; ++t)
            for (size_t kk = 0; kk < k; ++kk) host[a8_offset(t, kk, mp)] = codes[t * k + kk];
        cudaStream_t st = rt().stream;
        DevBuf<int8_t> q(bytes, st);
        DevBuf<float> sd(m, st);
        cuda_check(cudaMemcpyAsync(q.p, host.data(), bytes, cudaMemcpyHostToDevice, st), "H2D");
        cuda_check(cudaMemcpyAsync(sd.p, scales, m * 4, cudaMemcpyHostToDevice, st), "H2D");
        sync(st, "ody_qtensor_import_a8");
        auto* qt = new ody_qtensor();
        qt->kind = QKind::Act8;
        qt->rows = m;
        qt->cols = k;
        qt->codes = q.release();
        qt->scales = sd.release();
        *out = qt;
    });
}

ody_status ody_gemm_accumulators(const ody_qtensor* a_q, const ody_qtensor* w_q, int32_t* acc) {
    if (!a_q || !w_q || !acc) return einval("ody_gemm_accumulators: null argument");
    return guarded([&] {
        check_fast_inputs(a_q, w_q);
        Runtime& r = rt();
        std::lock_guard<std::mutex> lock(r.mu);
        cudaStream_t st = r.stream;
        const size_t m = a_q->rows, n = w_q->rows;
        DevBuf<int32_t> ad(m * n, st);
        run_gemm(a_q, w_q, nullptr, ad.p, st);
        cuda_check(cudaMemcpyAsync(acc, ad.p, m * n * 4, cudaMemcpyDeviceToHost, st), "D2H");
        sync(st, "ody_gemm_accumulators");
    });
}

// ================================================================ OTF files (ref otf.cpp)
// The reference's on-disk tensors: "OTF1" magic, dtype code, ndim, u64 dims, payload.
// A quantized tensor is a directory: payload.otf (packed-i4 / i8), scales.otf (f32
// [rows, groups]), scheme.txt.  Reading one builds the DEVICE qtensor directly (prepack
// into the kernel layout) -- the ingest path from `odyssey quantize` checkpoints.
}  // extern "C"

namespace {

enum : uint8_t { kOtfF32 = 0, kOtfI8 = 1, kOtfPackedI4 = 2, kOtfI32 = 3 };

struct OtfRaw {
    uint8_t dtype = 0;
    std::vector<uint64_t> dims;
    std::vector<uint8_t> payload;
    uint64_t numel() const {
        uint64_t n = 1;
        for (auto d : dims) n *= d;
        return n;
    }
};

size_t otf_payload_bytes(uint8_t dtype, uint64_t numel) {  // ref otf.cpp:16-24
    switch (dtype) {
        case kOtfF32: return numel * 4;
        case kOtfI8: return numel;
        case kOtfPackedI4: return (numel + 1) / 2;
        case kOtfI32: return numel * 4;
    }
    fail(ODY_EPARSE, "unsupported dtype code");
}

void otf_write(const OtfRaw& t, const std::string& path) {  // ref otf.cpp:45-63
    if (t.dims.empty() || t.dims.size() > 255) fail(ODY_EINVAL, "write_tensor: bad ndim");
    if (t.payload.size() != otf_payload_bytes(t.dtype, t.numel()))
        fail(ODY_EINVAL, "write_tensor: payload size does not match dims");
    std::string h("OTF1", 4);
    h.push_back(static_cast<char>(t.dtype));
    h.push_back(static_cast<char>(t.dims.size()));
    for (auto d : t.dims)
        for (int i = 0; i < 8; ++i) h.push_back(static_cast<char>((d >> (8 * i)) & 0xFF));
    std::FILE* f = std::fopen(path.c_str(), "wb");
    if (!f) fail(ODY_EIO, "write_tensor: cannot open " + path);
    const bool ok = std::fwrite(h.data(), 1, h.size(), f) == h.size() &&
                    std::fwrite(t.payload.data(), 1, t.payload.size(), f) == t.payload.size();
    std::fclose(f);
    if (!ok) fail(ODY_EIO, "write_tensor: write failed for " + path);
}

OtfRaw otf_read(const std::string& path) {  // ref otf.cpp:65-92
    std::FILE* f = std::fopen(path.c_str(), "rb");
    if (!f) fail(ODY_EIO, "read_tensor: cannot open " + path);
    std::vector<uint8_t> b;
    uint8_t buf[1 << 16];
    size_t n;
    while ((n = std::fread(buf, 1, sizeof(buf), f)) > 0) b.insert(b.end(), buf, buf + n);
    std::fclose(f);
    if (b.size() < 6) fail(ODY_EPARSE, "read_tensor: truncated header in " + path);
    if (std::memcmp(b.data(), "OTF1", 4) != 0) fail(ODY_EPARSE, "read_tensor: bad magic in " + path);
    if (b[4] > 3) fail(ODY_EPARSE, "read_tensor: unsupported dtype code " + std::to_string(b[4]) + " in " + path);
    OtfRaw t;
    t.dtype = b[4];
    const size_t ndim = b[5], off = 6 + ndim * 8;
    if (b.size() < off) fail(ODY_EPARSE, "read_tensor: truncated dims in " + path);
    for (size_t i = 0; i < ndim; ++i) {
        uint64_t d = 0;
        for (int j = 0; j < 8; ++j) d |= static_cast<uint64_t>(b[6 + i * 8 + j]) << (8 * j);
        t.dims.push_back(d);
    }
    if (b.size() - off != otf_payload_bytes(t.dtype, t.numel()))
        fail(ODY_EPARSE, "read_tensor: truncated payload in " + path);
    t.payload.assign(b.begin() + static_cast<std::ptrdiff_t>(off), b.end());
    return t;
}

std::vector<float> otf_floats(const OtfRaw& r) {
    if (r.dtype != kOtfF32) fail(ODY_EPARSE, "expected f32 tensor");
    std::vector<float> v(r.numel());
    std::memcpy(v.data(), r.payload.data(), r.payload.size());
    return v;
}

}  // namespace

extern "C" {

ody_status ody_tensor_write(const ody_tensor* t, const char* path) {
    if (!t || !path) return einval("ody_tensor_write: null argument");
    return guarded([&] {
        OtfRaw r;
        r.dtype = kOtfF32;
        r.dims = {t->rows, t->cols};
        r.payload.resize(t->rows * t->cols * 4);
        std::memcpy(r.payload.data(), t->data, r.payload.size());
        otf_write(r, path);
    });
}

ody_status ody_tensor_read(const char* path, ody_tensor** out) {
    if (!path || !out) return einval("ody_tensor_read: null argument");
    return guarded([&] {
        OtfRaw r = otf_read(path);  // ref otf.cpp:155-162 read_dense
        if (r.dtype != kOtfF32) fail(ODY_EPARSE, std::string("read_dense: ") + path + " is not f32");
        if (r.dims.size() != 2) fail(ODY_EPARSE, "read_dense: expected 2 dims");
        std::vector<float> v = otf_floats(r);
        for (float x : v)
            if (!std::isfinite(x)) fail(ODY_EINVAL, "DenseTensor: non-finite value");
        ody_tensor* t = new_tensor(r.dims[0], r.dims[1]);
        std::memcpy(t->data, v.data(), v.size() * 4);
        *out = t;
    });
}

ody_status ody_matmul_f32(const ody_tensor* a, const ody_tensor* b_transposed, ody_tensor** out) {
    if (!a || !b_transposed || !out) return einval("ody_matmul_f32: null argument");
    return guarded([&] {
        if (a->cols != b_transposed->cols)
            fail(ODY_EINVAL, "matmul_f32: inner dims disagree (" + std::to_string(a->cols) + " vs " +
                                 std::to_string(b_transposed->cols) + ")");
        cudaStream_t st = rt().stream;
        const size_t m = a->rows, n = b_transposed->rows, k = a->cols;
        DevBuf<float> ad(std::max<size_t>(m * k, 1), st), bd(std::max<size_t>(n * k, 1), st), od(std::max<size_t>(m * n, 1), st);
        cuda_check(cudaMemcpyAsync(ad.p, a->data, m * k * 4, cudaMemcpyHostToDevice, st), "H2D");
        cuda_check(cudaMemcpyAsync(bd.p, b_transposed->data, n * k * 4, cudaMemcpyHostToDevice, st), "H2D");
        if (m * n > 0)
            cuda_check(launch_matmul_f32(ad.p, bd.p, static_cast<int>(m), static_cast<int>(n), static_cast<int>(k),
                                         od.p, st),
                       "matmul_f32 launch");
        ody_tensor* t = new_tensor(m, n);
        cuda_check(cudaMemcpyAsync(t->data, od.p, m * n * 4, cudaMemcpyDeviceToHost, st), "D2H");
        sync(st, "ody_matmul_f32");
        *out = t;
    });
}

ody_status ody_qtensor_write(const ody_qtensor* q, const char* dir) {
    if (!q || !dir) return einval("ody_qtensor_write: null argument");
    return guarded([&] {
        std::error_code ec;
        std::filesystem::create_directories(dir, ec);
        const size_t r = q->rows, c = q->cols, groups = q->groups();
        OtfRaw pay, sc;
        pay.dims = {r, c};
        std::vector<float> scales(r * groups);
        if (q->bits() == 8) {
            pay.dtype = kOtfI8;
            pay.payload.resize(r * c);
        } else {
            pay.dtype = kOtfPackedI4;
            pay.payload.resize((r * c + 1) / 2);
        }
        const ody_status st = ody_qtensor_export(q, pay.payload.data(), scales.data());
        if (st != ODY_OK) fail(st, g_last_error);
        const std::string d(dir);
        otf_write(pay, d + "/payload.otf");
        sc.dtype = kOtfF32;
        sc.dims = {r, groups};  // ref otf.cpp:138-140: rows x groups_per_row
        sc.payload.resize(r * groups * 4);
        std::memcpy(sc.payload.data(), scales.data(), r * groups * 4);
        otf_write(sc, d + "/scales.otf");
        std::FILE* f = std::fopen((d + "/scheme.txt").c_str(), "w");
        if (!f) fail(ODY_EIO, "write_tensor: cannot open " + d + "/scheme.txt");
        std::fprintf(f, "bits=%d\nsymmetric=1\ngranularity=%s\ngroup_size=%zu\n", q->bits(), q->granularity(),
                     q->group_size);
        std::fclose(f);
    });
}

ody_status ody_qtensor_read(const char* dir, ody_qtensor** out) {
    if (!dir || !out) return einval("ody_qtensor_read: null argument");
    return guarded([&] {
        const std::string d(dir);
        std::FILE* f = std::fopen((d + "/scheme.txt").c_str(), "r");  // ref otf.cpp:164-173
        if (!f) fail(ODY_EIO, "read_tensor: missing scheme.txt in " + d);
        std::map<std::string, std::string> kv;
        char line[512];
        while (std::fgets(line, sizeof(line), f)) {
            std::string l(line);
            while (!l.empty() && (l.back() == '\n' || l.back() == '\r')) l.pop_back();
            const size_t eq = l.find('=');
            if (eq != std::string::npos) kv[l.substr(0, eq)] = l.substr(eq + 1);
        }
        std::fclose(f);
        for (const char* key : {"bits", "symmetric", "granularity", "group_size"})
            if (!kv.count(key)) fail(ODY_EINVAL, std::string("read_tensor: scheme.txt lacks ") + key);
        const int bits = std::stoi(kv["bits"]);
        const bool sym = kv["symmetric"] == "1";
        const std::string gran = kv["granularity"];
        if (bits != 4 && bits != 8) fail(ODY_EINVAL, "QuantScheme: bits must be 4 or 8");
        OtfRaw pay = otf_read(d + "/payload.otf");  // ref otf.cpp:179-197
        if (pay.dims.size() != 2) fail(ODY_EPARSE, "quantized payload: expected 2 dims");
        const size_t r = pay.dims[0], c = pay.dims[1];
        if (bits == 4 && pay.dtype != kOtfPackedI4) fail(ODY_EPARSE, "4-bit tensor payload must be packed-i4");
        if (bits == 8 && pay.dtype != kOtfI8) fail(ODY_EPARSE, "8-bit tensor payload must be i8");
        std::vector<float> scales = otf_floats(otf_read(d + "/scales.otf"));
        if (!sym) fail(ODY_EINVAL, "read_tensor: asymmetric tensors are not supported on the B200 path");
        const size_t group_size = static_cast<size_t>(std::stoull(kv["group_size"]));
        const bool per_group = gran == "per_group";
        if (per_group && (group_size == 0 || c % group_size != 0))
            fail(ODY_EINVAL, "QuantScheme: group size does not divide axis length");
        const size_t groups = per_group ? c / group_size : 1;
        if (scales.size() != r * groups) fail(ODY_EINVAL, "QuantizedTensor: scales size mismatch");
        for (float v : scales)  // ref tensor.cpp:161-165
            if (!(v > 0.0f) || !std::isfinite(v)) fail(ODY_EINVAL, "QuantizedTensor: non-positive scale");
        if (bits == 4 && (gran == "per_channel" || per_group)) {
            const ody_status st = ody_qtensor_import_w4(r, c, pay.payload.data(), scales.data(), out);
            if (st != ODY_OK) fail(st, g_last_error);
            if (per_group) {  // the same codes layout, scales [rows][groups]
                ody_qtensor* q = *out;
                cudaStream_t s2 = rt().stream;
                DevBuf<float> sd(r * groups, s2);
                cuda_check(cudaMemcpyAsync(sd.p, scales.data(), r * groups * 4, cudaMemcpyHostToDevice, s2), "H2D");
                sync(s2, "ody_qtensor_read");
                cudaFreeAsync(q->scales, s2);
                q->scales = sd.release();
                q->kind = QKind::Weight4G;
            }
            (*out)->group_size = group_size;
        } else if (bits == 8 && (gran == "per_token" || gran == "per_channel")) {
            // per-token activations and per-channel INT8 weights share the a8 layout
            const ody_status st = ody_qtensor_import_a8(r, c, reinterpret_cast<const int8_t*>(pay.payload.data()),
                                                        scales.data(), out);
            if (st != ODY_OK) fail(st, g_last_error);
            if (gran == "per_channel") (*out)->kind = QKind::Weight8;
            (*out)->group_size = group_size;
        } else {
            fail(ODY_EINVAL, "read_tensor: " + std::to_string(bits) + "-bit " + gran +
                                 " tensors are not supported on the B200 path");
        }
    });
}

// ref clip.cpp:55-103 (LWC grid search) on the GPU, bit-exact: per channel, the
// (gamma, beta) pair of the candidate grid minimising the quantization MSE.
ody_status ody_optimize_clipping(const ody_tensor* w, int bits, float grid_min, float grid_step, float* gamma,
                                 float* beta, float* mse_before, float* mse_after) {
    if (!w) return einval("ody_optimize_clipping: null tensor");
    return guarded([&] {
        if (w->rows * w->cols == 0) fail(ODY_EINVAL, "optimize_clipping: empty weight");
        if (!(grid_min > 0.0f && grid_min <= 1.0f) || !(grid_step > 0.0f))
            fail(ODY_EINVAL, "ClipGrid: need 0 < min <= 1 and step > 0");
        if (bits != 4 && bits != 8) fail(ODY_EINVAL, "QuantScheme: bits must be 4 or 8");
        if ((1.0f - grid_min) / grid_step > static_cast<float>(lwc_max_candidates() - 2))
            fail(ODY_EINVAL, "optimize_clipping: candidate grid too fine for the GPU kernel");
        if (w->cols > 50 * 1024) fail(ODY_EINVAL, "optimize_clipping: rows longer than 51200 elements");
        cudaStream_t st = rt().stream;
        const size_t n = w->rows, k = w->cols;
        DevBuf<float> wd(n * k, st), outd(4 * n, st);
        cuda_check(cudaMemcpyAsync(wd.p, w->data, n * k * 4, cudaMemcpyHostToDevice, st), "H2D");
        cuda_check(launch_lwc_grid(wd.p, static_cast<int>(n), static_cast<int>(k), bits, grid_min, grid_step,
                                   outd.p, outd.p + n, outd.p + 2 * n, outd.p + 3 * n, st),
                   "lwc launch");
        std::vector<float> h(4 * n);
        cuda_check(cudaMemcpyAsync(h.data(), outd.p, 4 * n * 4, cudaMemcpyDeviceToHost, st), "D2H");
        sync(st, "ody_optimize_clipping");
        if (gamma) std::memcpy(gamma, h.data(), n * 4);
        if (beta) std::memcpy(beta, h.data() + n, n * 4);
        if (mse_before) std::memcpy(mse_before, h.data() + 2 * n, n * 4);
        if (mse_after) std::memcpy(mse_after, h.data() + 3 * n, n * 4);
    });
}

// ================================================================ part 4: TP
// Megatron tensor parallelism through NCCL (SURVEY §8b "ody_tp_linear(comm, ...)", §8e).
// NCCL is bound at run time (dlopen of libnccl.so.2): inside a PyTorch process this
// resolves to the NCCL torch already loaded, from a plain C/C++ caller to the system one.
}  // extern "C"

namespace {

struct ncclUniqueIdLike {  // ncclUniqueId: 128 opaque bytes, passed by value
    char internal[ODY_COMM_ID_BYTES];
};

struct NcclApi {
    void* h = nullptr;
    int (*get_unique_id)(void*) = nullptr;
    int (*comm_init_rank)(void**, int, ncclUniqueIdLike, int) = nullptr;
    int (*all_reduce)(const void*, void*, size_t, int, int, void*, cudaStream_t) = nullptr;
    int (*comm_destroy)(void*) = nullptr;
    const char* (*error_string)(int) = nullptr;
    std::string err;
};

NcclApi& nccl() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        api.h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!api.h) {
            api.err = std::string("libnccl.so.2 not loadable: ") + dlerror();
            return;
        }
        api.get_unique_id = reinterpret_cast<int (*)(void*)>(dlsym(api.h, "ncclGetUniqueId"));
        api.comm_init_rank =
            reinterpret_cast<int (*)(void**, int, ncclUniqueIdLike, int)>(dlsym(api.h, "ncclCommInitRank"));
        api.all_reduce = reinterpret_cast<int (*)(const void*, void*, size_t, int, int, void*, cudaStream_t)>(
            dlsym(api.h, "ncclAllReduce"));
        api.comm_destroy = reinterpret_cast<int (*)(void*)>(dlsym(api.h, "ncclCommDestroy"));
        api.error_string = reinterpret_cast<const char* (*)(int)>(dlsym(api.h, "ncclGetErrorString"));
        if (!api.get_unique_id || !api.comm_init_rank || !api.all_reduce || !api.comm_destroy)
            api.err = "libnccl.so.2 lacks the NCCL 2.x entry points";
    });
    if (!api.err.empty()) fail(ODY_EDEVICE, api.err);
    return api;
}

void nccl_check(int rc, const char* what) {
    if (rc != 0) {
        const char* m = nccl().error_string ? nccl().error_string(rc) : "?";
        fail(ODY_EDEVICE, std::string(what) + ": NCCL error " + std::to_string(rc) + " (" + m + ")");
    }
}

// ncclDataType_t / ncclRedOp_t values (nccl.h, stable across NCCL 2.x)
constexpr int kNcclInt32 = 2, kNcclFloat32 = 7;
constexpr int kNcclSum = 0, kNcclMax = 2;

size_t tp_round(size_t b) { return (b + 255) & ~static_cast<size_t>(255); }

ody_linear_desc tp_desc(const void* x, ody_dtype x_dtype, size_t ldx, const void* w_packed, const float* s_w,
                        size_t m, size_t n, size_t k, ody_dtype out_dtype, void* out) {
    ody_linear_desc d = {};
    d.x = x;
    d.x_dtype = x_dtype;
    d.ldx = ldx;
    d.w_packed = w_packed;
    d.s_w = s_w;
    d.m = m;
    d.n = n;
    d.k = k;
    d.out = out;
    d.out_dtype = out_dtype;
    d.dep = -1;
    return d;
}

}  // namespace

struct ody_comm {
    void* nccl = nullptr;  // ncclComm_t
    int nranks = 0, rank = 0, device = 0;
};

extern "C" {

ody_status ody_comm_unique_id(void* id) {
    if (!id) return einval("ody_comm_unique_id: null argument");
    return guarded([&] { nccl_check(nccl().get_unique_id(id), "ncclGetUniqueId"); });
}

ody_status ody_comm_init(int nranks, int rank, const void* id, ody_comm** out) {
    if (!id || !out) return einval("ody_comm_init: null argument");
    if (nranks < 1 || rank < 0 || rank >= nranks) return einval("ody_comm_init: rank outside [0, nranks)");
    return guarded([&] {
        ncclUniqueIdLike uid;
        std::memcpy(&uid, id, sizeof(uid));
        auto c = std::make_unique<ody_comm>();
        cuda_check(cudaGetDevice(&c->device), "cudaGetDevice");
        nccl_check(nccl().comm_init_rank(&c->nccl, nranks, uid, rank), "ncclCommInitRank");
        c->nranks = nranks;
        c->rank = rank;
        *out = c.release();
    });
}

ody_status ody_comm_free(ody_comm* c) {
    if (!c) return ODY_OK;
    return guarded([&] {
        std::unique_ptr<ody_comm> own(c);
        if (c->nccl) nccl_check(nccl().comm_destroy(c->nccl), "ncclCommDestroy");
    });
}

ody_status ody_comm_dims(const ody_comm* c, int* nranks, int* rank) {
    if (!c || !nranks || !rank) return einval("ody_comm_dims: null argument");
    *nranks = c->nranks;
    *rank = c->rank;
    return ODY_OK;
}

size_t ody_tp_linear_workspace_bytes(ody_tp_kind kind, size_t m, size_t n, size_t k_local) {
    ody_linear_desc d = tp_desc(nullptr, ODY_DTYPE_F16, k_local, nullptr, nullptr, m, n, k_local,
                                ODY_DTYPE_F16, nullptr);
    size_t b = ody_dev_program_workspace_bytes(&d, 1);
    if (kind == ODY_TP_ROW) b = tp_round(b) + 2 * tp_round(m * 4) + tp_round(m * n * 4);
    return b;
}

ody_status ody_tp_linear(ody_comm* comm, ody_tp_kind kind, const void* x, ody_dtype x_dtype, size_t ldx,
                         const void* w_packed, const float* s_w, size_t m, size_t n, size_t k_local,
                         ody_dtype out_dtype, void* out, void* workspace, size_t workspace_bytes, void* stream) {
    if (!comm || !x || !w_packed || !s_w || !out || !workspace) return einval("ody_tp_linear: null argument");
    if (kind != ODY_TP_COLUMN && kind != ODY_TP_ROW) return einval("ody_tp_linear: unknown kind");
    if (m == 0 || n == 0 || k_local == 0) return einval("ody_tp_linear: empty operand");
    if (workspace_bytes < ody_tp_linear_workspace_bytes(kind, m, n, k_local))
        return einval("ody_tp_linear: workspace too small");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    ody_linear_desc d = tp_desc(x, x_dtype, ldx, w_packed, s_w, m, n, k_local, out_dtype, out);
    if (kind == ODY_TP_COLUMN)  // x replicated, W split along N: no collective
        return ody_dev_w4a8_linear_program(&d, 1, workspace, workspace_bytes, 0, 0, nullptr, 0, stream);
    // Row-parallel: x and W split along K.
    uint8_t* ws = static_cast<uint8_t*>(workspace);
    const size_t prog = tp_round(ody_dev_program_workspace_bytes(&d, 1));
    float* amax = reinterpret_cast<float*>(ws + prog);
    float* sa = reinterpret_cast<float*>(ws + prog + tp_round(m * 4));
    int32_t* acc = reinterpret_cast<int32_t*>(ws + prog + 2 * tp_round(m * 4));
    // 1. local row max -> MAX all-reduce: every rank quantizes its K-slice with the FULL
    //    row's scale (ref quantize.cpp:113-132 on the unsharded row)
    ody_status rc = ody_dev_row_absmax(x, x_dtype, ldx, m, k_local, amax, stream);
    if (rc != ODY_OK) return rc;
    rc = guarded([&] {
        nccl_check(nccl().all_reduce(amax, amax, m, kNcclFloat32, kNcclMax, comm->nccl, st), "ncclAllReduce(max)");
    });
    if (rc != ODY_OK) return rc;
    // 2. K-shard FastGEMM -> int32 pre-shift partial accumulators (+ the token scales)
    d.out = nullptr;
    d.absmax_in = amax;
    d.acc_out = acc;
    d.s_a_out = sa;
    rc = ody_dev_w4a8_linear_program(&d, 1, workspace, prog, 0, 0, nullptr, 0, stream);
    if (rc != ODY_OK) return rc;
    // 3. exact, order-free int32 SUM all-reduce (== the unsharded accumulator, bit for bit)
    rc = guarded([&] {
        nccl_check(nccl().all_reduce(acc, acc, m * n, kNcclInt32, kNcclSum, comm->nccl, st), "ncclAllReduce(sum)");
    });
    if (rc != ODY_OK) return rc;
    // 4. K4 once on the reduced accumulators: float(acc >> 4) * (sa * sw)
    return ody_dev_dequant_epilogue(acc, sa, s_w, m, n, out_dtype, out, stream);
}

const char* ody_b200_version(void) {
    try {
        return rt().version.c_str();
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return "libodyssey_b200 (no sm_100 device)";
    }
}

}  // extern "C"
