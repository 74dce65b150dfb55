// host_pipe.cu — swdft2d_forward_host: host array in, host array out in ONE call.
//
// The reference's tree_swdft_2d takes and returns host (numpy) arrays (tree2d.py:189,
// 201-202), so this is the entry point its binding calls.  The output is n0*n1 times the
// input, so the call is bound by the device-to-host link: the window rows are computed in
// strips into a ring of device buffers and copied out while later strips compute.
//   * pinned destination: each strip is one cudaMemcpyAsync on one of two copy streams
//     (the PCIe rate, ~55 GB/s);
//   * pageable destination (a fresh numpy array): cudaMemcpyAsync into pageable memory is
//     staged by the driver on one thread and pays every first-touch page fault there
//     (measured 3.4 GB/s into fresh pages, 20 GB/s into touched ones).  Instead the strips
//     go D2H in chunks into a library-owned pinned staging ring, and one worker thread per
//     staging slot copies its chunk into the destination, so the page faults and the
//     memcpy run on many cores while the link keeps streaming (config 4, 34 GB, 16 cores:
//     1.0 s into a fresh numpy array, 0.65-0.72 s into touched pages, against 10.1 s /
//     1.7 s for the driver's pageable copy and 0.61 s pinned; MADV_HUGEPAGE on the
//     destination measured level to 10 % slower and MADV_POPULATE_WRITE per chunk level
//     (alternated runs: 1.16-1.38 vs 1.13-1.20 s), neither is used;
//     profiles/host_entry_r02.jsonl).
// Device scratch (input rows + strip ring) and the staging ring are cached between calls
// (a 2 GB stream-ordered allocation is handed back to the driver at every synchronize and
// re-mapped by the next call: single calls took 1.0-1.4 s instead of 0.63) and freed by
// swdft2d_shutdown.
#include <unistd.h>

#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <map>
#include <mutex>
#include <thread>
#include <vector>

#include "../../include/swdft2d.h"
#include "swdft2d_internal.h"

namespace swdft2d {
namespace {

constexpr int RING = 4;     // device strips in flight
constexpr int COPIERS = 2;  // copy streams
constexpr int64_t IN_BYTES[4] = {4, 8, 8, 16};
constexpr int64_t SMALL_DIRECT_BYTES = 16 << 20;  // pageable outputs up to here: plain copies

int env_int(const char *name, int dflt, int lo, int hi) {
    const char *e = std::getenv(name);
    if (!e || !*e) return dflt;
    const int v = std::atoi(e);
    return v < lo ? lo : v > hi ? hi : v;
}

// Staging chunk -> destination.  Non-temporal stores: the destination is written once and
// not read back by this core, so regular stores would first read every line for ownership
// (SWDFT2D_HOST_NT=0 falls back to memcpy; x86-64 with AVX2 only).
#if defined(__x86_64__)
#include <immintrin.h>
__attribute__((target("avx2"))) void nt_copy_avx2(char *dst, const char *src, size_t len) {
    size_t head = (32 - ((uintptr_t)dst & 31)) & 31;
    if (head > len) head = len;
    std::memcpy(dst, src, head);
    dst += head;
    src += head;
    len -= head;
    size_t i = 0;
    for (; i + 128 <= len; i += 128) {
        const __m256i a = _mm256_loadu_si256(reinterpret_cast<const __m256i *>(src + i));
        const __m256i b = _mm256_loadu_si256(reinterpret_cast<const __m256i *>(src + i + 32));
        const __m256i c = _mm256_loadu_si256(reinterpret_cast<const __m256i *>(src + i + 64));
        const __m256i d = _mm256_loadu_si256(reinterpret_cast<const __m256i *>(src + i + 96));
        _mm256_stream_si256(reinterpret_cast<__m256i *>(dst + i), a);
        _mm256_stream_si256(reinterpret_cast<__m256i *>(dst + i + 32), b);
        _mm256_stream_si256(reinterpret_cast<__m256i *>(dst + i + 64), c);
        _mm256_stream_si256(reinterpret_cast<__m256i *>(dst + i + 96), d);
    }
    _mm_sfence();
    std::memcpy(dst + i, src + i, len - i);
}
#endif

void copy_out(char *dst, const char *src, size_t len, bool nt) {
#if defined(__x86_64__)
    if (nt) {
        nt_copy_avx2(dst, src, len);
        return;
    }
#endif
    std::memcpy(dst, src, len);
}

bool use_nt() {
#if defined(__x86_64__)
    return env_int("SWDFT2D_HOST_NT", 1, 0, 1) && __builtin_cpu_supports("avx2");
#else
    return false;
#endif
}

// One host-to-host call at a time: calls share the link, the scratch and the staging ring.
std::mutex g_call_mu;
std::map<int, std::pair<void *, size_t>> g_scratch;  // device -> cached scratch
void *g_stage = nullptr;                              // pinned staging ring
size_t g_stage_bytes = 0;

cudaError_t device_scratch(int dev, size_t bytes, void **out) {
    auto &s = g_scratch[dev];
    if (s.second < bytes) {
        if (s.first) cudaFree(s.first);
        s = {nullptr, 0};
        cudaError_t e = cudaMalloc(&s.first, bytes);
        if (e != cudaSuccess) {
            s.first = nullptr;
            return e;
        }
        s.second = bytes;
    }
    *out = s.first;
    return cudaSuccess;
}

cudaError_t staging(size_t bytes, void **out) {
    if (g_stage_bytes < bytes) {
        if (g_stage) cudaFreeHost(g_stage);
        g_stage = nullptr;
        g_stage_bytes = 0;
        cudaError_t e = cudaHostAlloc(&g_stage, bytes, cudaHostAllocPortable);
        if (e != cudaSuccess) {
            g_stage = nullptr;
            return e;
        }
        g_stage_bytes = bytes;
    }
    *out = g_stage;
    return cudaSuccess;
}

struct Pipe {
    cudaStream_t copy[COPIERS] = {nullptr, nullptr};
    cudaEvent_t done[RING] = {nullptr, nullptr, nullptr, nullptr};
    cudaEvent_t freed[RING] = {nullptr, nullptr, nullptr, nullptr};
    cudaError_t init() {
        cudaError_t e = cudaSuccess;
        for (int i = 0; i < COPIERS && e == cudaSuccess; ++i)
            e = cudaStreamCreateWithFlags(&copy[i], cudaStreamNonBlocking);
        for (int i = 0; i < RING && e == cudaSuccess; ++i) {
            e = cudaEventCreateWithFlags(&done[i], cudaEventDisableTiming);
            if (e == cudaSuccess) e = cudaEventCreateWithFlags(&freed[i], cudaEventDisableTiming);
        }
        return e;
    }
    ~Pipe() {
        for (cudaStream_t c : copy)
            if (c) {
                cudaStreamSynchronize(c);
                cudaStreamDestroy(c);
            }
        for (int i = 0; i < RING; ++i) {
            if (done[i]) cudaEventDestroy(done[i]);
            if (freed[i]) cudaEventDestroy(freed[i]);
        }
    }
};

// Pageable destinations: S pinned chunks, one worker thread each.  submit() waits for the
// slot, queues the chunk's D2H into it and hands (destination, length) to the worker,
// which waits for the copy and memcpy's the chunk out.
class Stager {
  public:
    Stager(int dev, char *pinned, int slots, size_t chunk) : chunk_(chunk), slots_(slots) {
        const bool nt = use_nt();
        try {
            start(dev, pinned, slots, chunk, nt);
        } catch (...) {  // a thread could not be created: stop the ones that were
            finish();
            throw;
        }
    }
    size_t chunk() const { return chunk_; }

  private:
    void start(int dev, char *pinned, int slots, size_t chunk, bool nt) {
        for (int i = 0; i < slots; ++i) {
            Slot *s = &slots_[i];
            s->pin = pinned + (size_t)i * chunk;
            s->err = cudaEventCreateWithFlags(&s->ev, cudaEventDisableTiming);
            s->th = std::thread([s, dev, nt] {
                cudaSetDevice(dev);
                std::unique_lock<std::mutex> lk(s->m);
                for (;;) {
                    s->cv.wait(lk, [s] { return s->busy || s->stop; });
                    if (!s->busy) return;
                    lk.unlock();
                    cudaError_t e = cudaEventSynchronize(s->ev);
                    if (e == cudaSuccess) copy_out(s->dst, s->pin, s->len, nt);
                    lk.lock();
                    if (e != cudaSuccess && s->err == cudaSuccess) s->err = e;
                    s->busy = false;
                    s->cv.notify_all();
                }
            });
        }
    }

  public:
    cudaError_t submit(int64_t index, const char *dev_src, char *dst, size_t len, cudaStream_t cs) {
        Slot *s = &slots_[index % (int64_t)slots_.size()];
        std::unique_lock<std::mutex> lk(s->m);
        s->cv.wait(lk, [s] { return !s->busy; });
        if (s->err != cudaSuccess) return s->err;
        cudaError_t e = cudaMemcpyAsync(s->pin, dev_src, len, cudaMemcpyDeviceToHost, cs);
        if (e == cudaSuccess) e = cudaEventRecord(s->ev, cs);
        if (e != cudaSuccess) return e;
        s->dst = dst;
        s->len = len;
        s->busy = true;
        s->cv.notify_all();
        return cudaSuccess;
    }
    // Waits for every chunk to land in the destination, stops the workers.
    cudaError_t finish() {
        cudaError_t e = cudaSuccess;
        for (Slot &s : slots_) {
            {
                std::unique_lock<std::mutex> lk(s.m);
                s.cv.wait(lk, [&s] { return !s.busy; });
                s.stop = true;
                if (e == cudaSuccess) e = s.err;
                s.cv.notify_all();
            }
            if (s.th.joinable()) s.th.join();
            if (s.ev) cudaEventDestroy(s.ev);
            s.ev = nullptr;
        }
        return e;
    }
    ~Stager() { finish(); }

  private:
    struct Slot {
        char *pin = nullptr;
        cudaEvent_t ev = nullptr;
        std::mutex m;
        std::condition_variable cv;
        char *dst = nullptr;
        size_t len = 0;
        bool busy = false, stop = false;
        cudaError_t err = cudaSuccess;
        std::thread th;
    };
    size_t chunk_;
    std::vector<Slot> slots_;
};

enum HostKind { PAGEABLE, PINNED, DEVICE };
HostKind host_kind(const void *p) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return PAGEABLE;
    }
    if (a.type == cudaMemoryTypeDevice) return DEVICE;
    return a.type == cudaMemoryTypeHost || a.type == cudaMemoryTypeManaged ? PINNED : PAGEABLE;
}

// The staging workers for a pageable destination (SWDFT2D_HOST_THREADS slots of
// SWDFT2D_HOST_CHUNK_MB MiB; the pinned ring is cached).
int make_stager(int dev, Stager **out) {
    long cores = sysconf(_SC_NPROCESSORS_ONLN);
    const int slots = env_int("SWDFT2D_HOST_THREADS", cores > 16 ? 16 : cores < 2 ? 2 : (int)cores, 1, 64);
    const size_t chunk = (size_t)env_int("SWDFT2D_HOST_CHUNK_MB", 4, 1, 256) << 20;
    void *pin = nullptr;
    cudaError_t e = staging(slots * chunk, &pin);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return set_error(SWDFT2D_E_NOMEM, "pinned staging (%zu B): %s", slots * chunk, cudaGetErrorString(e));
    }
    try {
        *out = new Stager(dev, static_cast<char *>(pin), slots, chunk);
    } catch (const std::exception &ex) {  // thread creation refused
        return set_error(SWDFT2D_E_NOMEM, "staging workers: %s", ex.what());
    }
    return SWDFT2D_OK;
}

}  // namespace

void release_host_pipe() {
    std::lock_guard<std::mutex> lk(g_call_mu);
    int cur = 0;
    cudaGetDevice(&cur);
    for (auto &kv : g_scratch)
        if (kv.second.first) {
            cudaSetDevice(kv.first);
            cudaFree(kv.second.first);
        }
    g_scratch.clear();
    if (g_stage) cudaFreeHost(g_stage);
    g_stage = nullptr;
    g_stage_bytes = 0;
    cudaSetDevice(cur);
}

}  // namespace swdft2d

using namespace swdft2d;

extern "C" {

void *swdft2d_host_alloc(int64_t bytes) {
    void *p = nullptr;
    if (bytes <= 0) {
        set_error(SWDFT2D_E_INVALID_ARG, "host_alloc: %lld bytes", (long long)bytes);
        return nullptr;
    }
    cudaError_t e = cudaHostAlloc(&p, (size_t)bytes, cudaHostAllocPortable);
    if (e != cudaSuccess) {
        cudaGetLastError();
        set_error(SWDFT2D_E_NOMEM, "cudaHostAlloc(%lld B): %s", (long long)bytes, cudaGetErrorString(e));
        return nullptr;
    }
    return p;
}

int swdft2d_host_free(void *p) {
    if (!p) return SWDFT2D_OK;
    cudaError_t e = cudaFreeHost(p);
    if (e != cudaSuccess) return set_error(SWDFT2D_E_CUDA, "cudaFreeHost: %s", cudaGetErrorString(e));
    return SWDFT2D_OK;
}

int swdft2d_download(const void *dev_src, void *host_dst, int64_t bytes, void *stream) {
    if (bytes < 0) return set_error(SWDFT2D_E_INVALID_ARG, "download: %lld bytes", (long long)bytes);
    if (bytes == 0) return SWDFT2D_OK;
    if (!dev_src || !host_dst) return set_error(SWDFT2D_E_INVALID_ARG, "null pointer");
    const HostKind kind = host_kind(host_dst);
    if (kind == DEVICE) return set_error(SWDFT2D_E_INVALID_ARG, "download: host_dst is a device pointer");
    std::lock_guard<std::mutex> call(g_call_mu);
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return set_error(SWDFT2D_E_CUDA, "cudaGetDevice: %s", cudaGetErrorString(e));
    Pipe pipe;
    if ((e = pipe.init()) != cudaSuccess)
        return set_error(SWDFT2D_E_CUDA, "download: streams/events: %s", cudaGetErrorString(e));
    // the copy stream waits for the work already queued on the caller's stream
    e = cudaEventRecord(pipe.done[0], reinterpret_cast<cudaStream_t>(stream));
    if (e == cudaSuccess) e = cudaStreamWaitEvent(pipe.copy[0], pipe.done[0], 0);
    const char *src = static_cast<const char *>(dev_src);
    char *dst = static_cast<char *>(host_dst);
    if (kind == PINNED || bytes <= SMALL_DIRECT_BYTES) {
        if (e == cudaSuccess)
            e = cudaMemcpyAsync(dst, src, (size_t)bytes, cudaMemcpyDeviceToHost, pipe.copy[0]);
    } else {
        Stager *stager = nullptr;
        int rc = make_stager(dev, &stager);
        if (rc) return rc;
        int64_t index = 0;
        for (size_t off = 0; off < (size_t)bytes && e == cudaSuccess; off += stager->chunk()) {
            const size_t n = (size_t)bytes - off < stager->chunk() ? (size_t)bytes - off : stager->chunk();
            e = stager->submit(index++, src + off, dst + off, n, pipe.copy[0]);
        }
        cudaError_t e2 = stager->finish();
        if (e == cudaSuccess) e = e2;
        delete stager;
    }
    cudaError_t e3 = cudaStreamSynchronize(pipe.copy[0]);
    if (e == cudaSuccess) e = e3;
    if (e != cudaSuccess) {
        cudaGetLastError();
        return set_error(SWDFT2D_E_CUDA, "download: %s", cudaGetErrorString(e));
    }
    return SWDFT2D_OK;
}

int swdft2d_forward_host(const void *x, int in_dtype, int64_t N0, int64_t N1, int64_t ld_x, int m0,
                         int m1, int prec, double scale, int64_t p0_begin, int64_t p0_end,
                         void *out_host, int64_t strip_bytes, int kernel, void *stream) {
    if (in_dtype < SWDFT2D_IN_F32 || in_dtype > SWDFT2D_IN_C128)
        return set_error(SWDFT2D_E_INVALID_ARG, "unknown input dtype code %d", in_dtype);
    if (ld_x < N1) return set_error(SWDFT2D_E_INVALID_ARG, "ld_x %lld < N1 %lld", (long long)ld_x, (long long)N1);
    // shape, window, precision, row range and kernel selection: the forward call's own checks
    int64_t ws_unused = 0;
    int rc = swdft2d_workspace_bytes(N0, N1, m0, m1, prec, p0_begin, p0_end, kernel, &ws_unused);
    if (rc) return rc;
    if (p0_begin == p0_end) return SWDFT2D_OK;
    if (!x || !out_host) return set_error(SWDFT2D_E_INVALID_ARG, "null pointer");
    const HostKind kind = host_kind(out_host);
    if (kind == DEVICE)
        return set_error(SWDFT2D_E_INVALID_ARG, "forward_host: out_host is a device pointer (use swdft2d_forward)");
    if (strip_bytes < 0) return set_error(SWDFT2D_E_INVALID_ARG, "strip_bytes %lld", (long long)strip_bytes);
    if (strip_bytes == 0) strip_bytes = (int64_t)512 << 20;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    const int64_t n0 = (int64_t)1 << m0, n1 = (int64_t)1 << m1;
    const int64_t es = IN_BYTES[in_dtype];
    const int64_t P1 = N1 - n1 + 1;
    const int64_t rows = p0_end - p0_begin, rows_in = rows + n0 - 1;
    const int64_t row_bytes = P1 * n0 * n1 * (prec == SWDFT2D_PREC_FP64 ? 16 : 8);
    int64_t R = strip_bytes / row_bytes;
    R = R < 1 ? 1 : R > rows ? rows : R;
    const int64_t nstrips = (rows + R - 1) / R;
    const int nring = nstrips < RING ? (int)nstrips : RING;
    const int64_t in_bytes = (rows_in * N1 * es + 255) / 256 * 256;

    std::lock_guard<std::mutex> call(g_call_mu);
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return set_error(SWDFT2D_E_CUDA, "cudaGetDevice: %s", cudaGetErrorString(e));
    Pipe pipe;
    if ((e = pipe.init()) != cudaSuccess)
        return set_error(SWDFT2D_E_CUDA, "forward_host: streams/events: %s", cudaGetErrorString(e));
    void *scratch = nullptr;
    if ((e = device_scratch(dev, (size_t)(in_bytes + nring * R * row_bytes), &scratch)) != cudaSuccess) {
        cudaGetLastError();
        return set_error(SWDFT2D_E_NOMEM, "forward_host: device scratch (%lld B): %s",
                         (long long)(in_bytes + nring * R * row_bytes), cudaGetErrorString(e));
    }
    char *d_x = static_cast<char *>(scratch), *ring = d_x + in_bytes;

    // pageable destination: pinned staging ring + one worker per slot
    // small pageable outputs are not worth a set of worker threads: the driver's own
    // staged copy handles them
    const bool direct = kind == PINNED || rows * row_bytes <= SMALL_DIRECT_BYTES;
    Stager *stager = nullptr;
    if (!direct && (rc = make_stager(dev, &stager))) return rc;

    e = cudaMemcpy2DAsync(d_x, (size_t)(N1 * es), static_cast<const char *>(x) + p0_begin * ld_x * es,
                          (size_t)(ld_x * es), (size_t)(N1 * es), (size_t)rows_in, cudaMemcpyDefault, st);
    int64_t chunk_index = 0;
    for (int64_t k = 0; k < nstrips && e == cudaSuccess && rc == SWDFT2D_OK; ++k) {
        const int64_t a = k * R, b = a + R < rows ? a + R : rows;  // relative to p0_begin
        const int slot = (int)(k % nring);
        char *buf = ring + (int64_t)slot * R * row_bytes;
        if (k >= nring) e = cudaStreamWaitEvent(st, pipe.freed[slot], 0);
        if (e != cudaSuccess) break;
        rc = swdft2d_forward_ws(d_x, in_dtype, rows_in, N1, N1, m0, m1, prec, scale, a, b, buf, nullptr,
                                0, kernel, stream);
        if (rc) break;
        cudaStream_t cs = pipe.copy[k % COPIERS];
        e = cudaEventRecord(pipe.done[slot], st);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(cs, pipe.done[slot], 0);
        char *dst = static_cast<char *>(out_host) + a * row_bytes;
        const size_t len = (size_t)((b - a) * row_bytes);
        if (direct) {
            if (e == cudaSuccess) e = cudaMemcpyAsync(dst, buf, len, cudaMemcpyDeviceToHost, cs);
        } else {
            for (size_t off = 0; off < len && e == cudaSuccess; off += stager->chunk()) {
                const size_t n = len - off < stager->chunk() ? len - off : stager->chunk();
                e = stager->submit(chunk_index++, buf + off, dst + off, n, cs);
            }
        }
        if (e == cudaSuccess) e = cudaEventRecord(pipe.freed[slot], cs);
    }
    // synchronous call: out_host is complete, the scratch idle, on return
    if (stager) {
        cudaError_t e2 = stager->finish();
        if (e == cudaSuccess) e = e2;
        delete stager;
    }
    for (cudaStream_t cs : pipe.copy) {
        cudaError_t e2 = cudaStreamSynchronize(cs);
        if (e == cudaSuccess) e = e2;
    }
    cudaError_t e3 = cudaStreamSynchronize(st);
    if (e == cudaSuccess) e = e3;
    if (rc) return rc;
    if (e != cudaSuccess) {
        cudaGetLastError();
        return set_error(SWDFT2D_E_CUDA, "forward_host: %s", cudaGetErrorString(e));
    }
    return SWDFT2D_OK;
}

}  // extern "C"
