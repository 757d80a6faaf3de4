// capi.cu -- the extern "C" boundary (include/ilans_b200.h).
//
// Host-buffer drop-ins mirror pkg/src/ilans/_core.pyx one for one: the host
// arrays are copied to HBM, the sm_100a kernels run on a library-owned
// stream, results come back. There is no CPU compute fallback: without a
// CUDA device every entry point returns ILANS_ERR_CUDA.
#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <sched.h>
#include <time.h>
#include <unistd.h>
#include <unordered_map>
#include <vector>

#include "common.cuh"
#include "kernels.cuh"

static std::atomic<unsigned long long> g_launches{0};
void ilans_note_launch(int n) { g_launches.fetch_add(static_cast<unsigned long long>(n)); }

namespace ilans {

__global__ void flag_kernel(uint32_t *flag, uint32_t v) {
    __threadfence_system();
    *reinterpret_cast<volatile uint32_t *>(flag) = v;
}

__global__ void dstatus_reset_kernel(DStatus *s) {
    s->trunc_stream = ~0ull;
    s->unenc_index = -1;
    s->unenc_symbol = 0;
    s->value_error = 0;
    s->max_digits = 0;
}

cudaError_t smem_limit(const void *kernel, int bytes) {
    static std::mutex mu;
    static std::unordered_map<const void *, int> set_to[64];
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lock(mu);
    int &cur = set_to[dev & 63][kernel];
    if (cur >= bytes) return cudaSuccess;
    const cudaError_t e =
        cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e == cudaSuccess) cur = bytes;
    return e;
}

int sm_count() {
    static int cached[64] = {0};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) dev = 0;
    if (!cached[dev]) {
        int v = 0;
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        cached[dev] = v > 0 ? v : 148;
    }
    return cached[dev];
}

cudaError_t launch_build_table(const unsigned long long *d_counts, const uint32_t *d_freq,
                               int n_freq, const uint32_t *d_cum, const uint8_t *d_slot,
                               int scale_bits, TableDev *d_table, cudaStream_t stream) {
    // from counts (cum follows from the quantized freq): the slot tables are
    // split over several CTAs; drop-in tables (given cum / slot) use one
    const int parts = d_counts && scale_bits >= 1 && scale_bits <= kMaxScaleBits
                          ? table_parts(scale_bits) : 1;
    build_table_kernel<<<parts, kMaxSym, 0, stream>>>(d_counts, d_freq, n_freq, d_cum, d_slot,
                                                      scale_bits, d_table);
    ilans_note_launch();
    return cudaGetLastError();
}

}  // namespace ilans

using namespace ilans;

#include "status.cuh"

// ---------------------------------------------------------------------------
// per-device context for the host-buffer drop-ins
// ---------------------------------------------------------------------------
namespace {

std::atomic<bool> g_exiting{false};  // ilans_process_exiting()

struct DevBuf {
    void *p = nullptr;
    size_t cap = 0;
    cudaError_t ensure(size_t bytes) {
        if (bytes < 64) bytes = 64;
        if (bytes <= cap) return cudaSuccess;
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
        size_t want = bytes + bytes / 4;
        cudaError_t e = cudaMalloc(&p, want);
        if (e == cudaSuccess) cap = want;
        return e;
    }
    template <typename T>
    T *as() const { return static_cast<T *>(p); }
};

// pinned host staging for the single-stream drop-ins: inputs are packed
// into it and every result (status, counts, states, payload / decoded bytes)
// comes back into it with ONE stream synchronisation per call
struct HostBuf {
    void *p = nullptr;
    size_t cap = 0;
    cudaError_t ensure(size_t bytes) {
        if (bytes <= cap) return cudaSuccess;
        if (p) cudaFreeHost(p);
        p = nullptr;
        cap = 0;
        size_t want = bytes + bytes / 4;
        if (want < (size_t(1) << 20)) want = size_t(1) << 20;
        cudaError_t e = cudaHostAlloc(&p, want, cudaHostAllocDefault);
        if (e == cudaSuccess) cap = want;
        return e;
    }
    uint8_t *at(size_t off) const { return static_cast<uint8_t *>(p) + off; }
};
constexpr size_t kStageMax = size_t(256) << 20;  // larger calls copy pageable memory directly

// One context per (host thread, device): its own stream, device buffers,
// pinned staging and cached device model, so calls from different host
// threads (ctypes releases the GIL) run concurrently on the GPU.
struct Ctx {
    std::mutex mu;
    bool init = false;
    int dev = 0;
    cudaStream_t stream = nullptr;
    // completion flag in mapped pinned memory, written by a one-thread
    // kernel after the call's last copy; the host polls it with no driver
    // call (many threads waiting at once do not contend in the driver)
    uint32_t *hflag = nullptr, *dflag = nullptr;
    uint32_t seq = 0;
    DevBuf msg, scratch, payload, out, states, ws, slot, freq, cum, table, status, counts,
        offsets, consumed, words, trace, io;
    HostBuf stage, tstage;
    // the model currently built in `table` (drop-in calls pass the same
    // freq / cum / slot arrays call after call: rebuilt only on change)
    bool tab_valid = false, tab_has_slot = false, tab_packed = false;
    int tab_sb = 0, tab_nfreq = 0;
    uint32_t tab_f[kMaxSym] = {0}, tab_c[kMaxSym + 1] = {0};
    std::vector<uint8_t> tab_slot;
    ~Ctx() {
        // at process exit the runtime may be torn down already (the main
        // thread's thread_local contexts die after the interpreter's exit
        // hooks): leave the memory to the OS
        if (!init || g_exiting.load() || cudaSetDevice(dev) != cudaSuccess) return;
        for (DevBuf *b : {&msg, &scratch, &payload, &out, &states, &ws, &slot, &freq, &cum, &table,
                          &status, &counts, &offsets, &consumed, &words, &trace, &io})
            if (b->p) cudaFree(b->p);
        for (HostBuf *b : {&stage, &tstage})
            if (b->p) cudaFreeHost(b->p);
        if (hflag) cudaFreeHost(hflag);
        cudaStreamDestroy(stream);
    }
};

thread_local Ctx *t_ctx[64] = {nullptr};
thread_local struct CtxOwner {
    ~CtxOwner() {
        for (Ctx *&c : t_ctx) {
            delete c;
            c = nullptr;
        }
    }
} t_ctx_owner;
thread_local int t_device = -1;

int current_device(ilans_status *st, Ctx **out) {
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess || n == 0)
        return st_fail(st, ILANS_ERR_CUDA, "no CUDA device available (%s)",
                       e == cudaSuccess ? "0 devices" : cudaGetErrorString(e));
    int dev = t_device;
    if (dev < 0) {
        e = cudaGetDevice(&dev);
        if (e != cudaSuccess) return st_cuda(st, e, "cudaGetDevice");
    }
    if (dev >= n || dev >= 64) return st_fail(st, ILANS_ERR_VALUE, "bad device %d", dev);
    e = cudaSetDevice(dev);
    if (e != cudaSuccess) return st_cuda(st, e, "cudaSetDevice");
    (void)t_ctx_owner;  // constructs the owner (frees this thread's contexts at exit)
    if (!t_ctx[dev]) {
        t_ctx[dev] = new Ctx();
        t_ctx[dev]->dev = dev;
    }
    *out = t_ctx[dev];
    return ILANS_OK;
}

int ctx_init(Ctx &c, ilans_status *st) {
    if (c.init) return ILANS_OK;
    CK(cudaStreamCreateWithFlags(&c.stream, cudaStreamNonBlocking));
    CK(cudaHostAlloc(reinterpret_cast<void **>(&c.hflag), 64, cudaHostAllocMapped));
    *c.hflag = 0;
    CK(cudaHostGetDevicePointer(reinterpret_cast<void **>(&c.dflag), c.hflag, 0));
    CK(c.table.ensure(sizeof(TableDev)));
    CK(c.status.ensure(sizeof(DStatus)));
    c.init = true;
    return ILANS_OK;
}

int read_dstatus(const DStatus *d, cudaStream_t s, DStatus *h, ilans_status *st) {
    CK(cudaMemcpyAsync(h, d, sizeof(DStatus), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    return ILANS_OK;
}

}  // namespace

int ilans_host_session(ilans_status *st, cudaStream_t *stream, std::unique_lock<std::mutex> *lock) {
    Ctx *cp = nullptr;
    if (int rc = current_device(st, &cp)) return rc;
    *lock = std::unique_lock<std::mutex>(cp->mu);
    if (int rc = ctx_init(*cp, st)) return rc;
    *stream = cp->stream;
    return ILANS_OK;
}

// ---------------------------------------------------------------------------
// library
// ---------------------------------------------------------------------------
extern "C" int ilans_abi_version(void) { return ILANS_B200_ABI_VERSION; }

extern "C" int ilans_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

extern "C" int ilans_set_device(int device, ilans_status *st) {
    st_clear(st);
    int n = ilans_device_count();
    if (device < 0 || device >= n || device >= 64)
        return st_fail(st, ILANS_ERR_VALUE, "device %d out of range (%d visible)", device, n);
    t_device = device;
    CK(cudaSetDevice(device));
    return ILANS_OK;
}

extern "C" uint64_t ilans_launch_count(void) { return g_launches.load(); }

extern "C" void ilans_process_exiting(void) { g_exiting.store(true); }

extern "C" size_t ilans_table_bytes(void) { return sizeof(TableDev); }
extern "C" size_t ilans_dstatus_bytes(void) { return sizeof(DStatus); }

// ---------------------------------------------------------------------------
// 1. host-buffer drop-ins
// ---------------------------------------------------------------------------

// sb <= 12 packed LUT is valid only for self-consistent tables (every slot's
// symbol s has 1 <= f[s] <= 4095 and 0 <= slot - cum[s] < 4096).
static bool host_packable(const uint8_t *slot_sym, const uint32_t *f, const uint32_t *cum,
                          int scale_bits) {
    if (scale_bits > kPackedMaxBits) return false;
    const uint32_t m = 1u << scale_bits;
    for (uint32_t j = 0; j < m; ++j) {
        const uint32_t s = slot_sym[j];
        if (f[s] < 1 || f[s] > 4095 || j - cum[s] >= 4096u) return false;
    }
    return true;
}

static size_t al16(size_t b) { return (b + 15) & ~size_t(15); }

// Make c.table the model of (freq, cum[, slot]) at scale_bits: a no-op when
// it already is (the drop-in callers pass the same table arrays call after
// call), else the arrays go up through pinned staging and build_table runs.
// slot == nullptr (encode): the slot LUT is derived from cum on the device.
static int ensure_table(Ctx &c, const uint32_t *freq, int n_freq, const uint32_t *cum,
                        const uint8_t *slot, int scale_bits, cudaStream_t s, ilans_status *st) {
    const size_t m = size_t(1) << scale_bits;
    if (c.tab_valid && c.tab_sb == scale_bits && c.tab_nfreq == n_freq &&
        std::memcmp(c.tab_f, freq, size_t(n_freq) * 4) == 0 &&
        std::memcmp(c.tab_c, cum, size_t(n_freq + 1) * 4) == 0 &&
        (!slot || (c.tab_has_slot && std::memcmp(c.tab_slot.data(), slot, m) == 0)))
        return ILANS_OK;
    c.tab_valid = false;
    CK(c.freq.ensure(kMaxSym * 4));
    CK(c.cum.ensure((kMaxSym + 1) * 4));
    if (slot) CK(c.slot.ensure(m));
    // the previous call's uploads from tstage completed before it returned
    CK(c.tstage.ensure(kMaxSym * 4 + (kMaxSym + 1) * 4 + m + 16));
    uint32_t *hf = reinterpret_cast<uint32_t *>(c.tstage.at(0));
    uint32_t *hc = reinterpret_cast<uint32_t *>(c.tstage.at(kMaxSym * 4));
    std::memset(hf, 0, kMaxSym * 4 + (kMaxSym + 1) * 4);
    std::memcpy(hf, freq, size_t(n_freq) * 4);
    std::memcpy(hc, cum, size_t(n_freq + 1) * 4);
    CK(cudaMemcpyAsync(c.freq.p, hf, kMaxSym * 4, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(c.cum.p, hc, (kMaxSym + 1) * 4, cudaMemcpyHostToDevice, s));
    if (slot) {
        uint8_t *hs = c.tstage.at(kMaxSym * 4 + (kMaxSym + 1) * 4);
        std::memcpy(hs, slot, m);
        CK(cudaMemcpyAsync(c.slot.p, hs, m, cudaMemcpyHostToDevice, s));
    }
    CK(launch_build_table(nullptr, c.freq.as<uint32_t>(), n_freq, c.cum.as<uint32_t>(),
                          slot ? c.slot.as<uint8_t>() : nullptr, scale_bits,
                          c.table.as<TableDev>(), s));
    c.tab_sb = scale_bits;
    c.tab_nfreq = n_freq;
    std::memcpy(c.tab_f, freq, size_t(n_freq) * 4);
    std::memcpy(c.tab_c, cum, size_t(n_freq + 1) * 4);
    c.tab_has_slot = slot != nullptr;
    if (slot) {
        c.tab_slot.assign(slot, slot + m);
        c.tab_packed = host_packable(slot, hf, hc, scale_bits);
    }
    c.tab_valid = true;
    return ILANS_OK;
}

static void table_clobbered(Ctx &c) { c.tab_valid = false; }

// The encoder's 8-byte symbol record holds f - 1 and cum in 16 bits each
// (common.cuh EncSym): true for every SymbolTable (f <= m, cum < m <= 2^16);
// hand-made tables outside that range are rejected instead of mis-coded.
static bool encode_table_fits(const uint32_t *freq, const uint32_t *cum, int n_freq,
                              int scale_bits) {
    const uint32_t m = 1u << scale_bits;
    for (int s = 0; s < n_freq; ++s)
        if (freq[s] && (freq[s] > m || cum[s] > 0xFFFFu)) return false;
    return true;
}

// Wait for everything queued on the context's stream: a one-thread kernel
// stores the call's sequence number into mapped pinned memory after the
// last copy, and the host polls that word, yielding its core between polls
// (no driver lock, no spinning thread starving the Python threads). The
// stream is queried now and then so a failed launch cannot hang the wait.
// Waiting threads beyond half the host's cores sleep 20 us between polls
// instead of yielding: with more pollers than cores the yielding threads
// took the cores from the one thread holding the GIL (plugin throughput
// fell from 8 to 16 to 32 threads). One or a few waiters keep yielding
// (no added latency).
static std::atomic<int> g_waiters{0};
static const int g_spin_waiters = [] {
    const long n = sysconf(_SC_NPROCESSORS_ONLN);
    return n > 1 ? static_cast<int>(n / 2) : 1;
}();

static cudaError_t ctx_wait(Ctx &c) {
    const uint32_t want = ++c.seq;
    flag_kernel<<<1, 1, 0, c.stream>>>(c.dflag, want);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    ilans_note_launch();
    struct Waiter {
        Waiter() { g_waiters.fetch_add(1, std::memory_order_relaxed); }
        ~Waiter() { g_waiters.fetch_sub(1, std::memory_order_relaxed); }
    } waiter;
    for (uint32_t i = 1;; ++i) {
        if (__atomic_load_n(c.hflag, __ATOMIC_ACQUIRE) == want) return cudaSuccess;
        if ((i & 1023u) == 0) {
            e = cudaStreamQuery(c.stream);
            if (e != cudaSuccess && e != cudaErrorNotReady) return e;
            if (e == cudaSuccess && __atomic_load_n(c.hflag, __ATOMIC_ACQUIRE) != want)
                return cudaStreamSynchronize(c.stream);  // (flag store not yet visible)
        }
        if (g_waiters.load(std::memory_order_relaxed) > g_spin_waiters) {
            const timespec ts{0, 20000};
            nanosleep(&ts, nullptr);
        } else {
            sched_yield();
        }
    }
}

static void dstatus_init(DStatus *h) {  // dstatus_reset_kernel's image
    std::memset(h, 0, sizeof(DStatus));
    h->trunc_stream = ~0ull;
    h->unenc_index = -1;
}

// stats: measure the most digits any symbol spilled (RenormStats.note_encode,
// rans.py:246-250) in the kernel -> st->max_digits
//
// Small calls (the per-chunk plugin loop) are one upload, one launch, one
// download and one synchronisation: message and status image travel in one
// copy, and status | words | states | scratch come back in one. The device
// buffer `io` mirrors the pinned staging layout byte for byte.
static int encode_u16_common(const uint8_t *msg, int64_t n, const uint32_t *freq, int32_t n_freq,
                             const uint32_t *cum, int32_t scale_bits, int32_t n_lanes,
                             uint16_t *payload_out, int64_t *payload_words, uint32_t *states_out,
                             bool stats, ilans_status *st) {
    if (n < 0) return st_fail(st, ILANS_ERR_VALUE, "negative message length");
    if (n_lanes < 1 || n_lanes > 0xFFFF)
        return st_fail(st, ILANS_ERR_VALUE, "lane_count must be in [1, 65535]");
    if (scale_bits < 1 || scale_bits > kMaxScaleBits)
        return st_fail(st, ILANS_ERR_VALUE, "scale_bits must be in [1, 16]");
    if (n_freq < 0 || n_freq > kMaxSym)
        return st_fail(st, ILANS_ERR_VALUE, "alphabet size must be in [1, 256]");
    if (!encode_table_fits(freq, cum, n_freq, scale_bits))
        return st_fail(st, ILANS_ERR_VALUE, "frequency / cumulative table out of range");
    Ctx *cp = nullptr;
    if (int rc = current_device(st, &cp)) return rc;
    Ctx &c = *cp;
    std::lock_guard<std::mutex> lock(c.mu);
    if (int rc = ctx_init(c, st)) return rc;
    if (n == 0) {  // states stay at L, empty payload (_core.pyx:28-29)
        for (int l = 0; l < n_lanes; ++l) states_out[l] = kLow;
        *payload_words = 0;
        st->max_digits = 0;
        return ILANS_OK;
    }
    cudaStream_t s = c.stream;
    CK(c.ws.ensure(size_t(n_lanes) * 4));
    // layout: msg | status | words | states | scratch (n words + slack)
    const size_t o_st = al16(size_t(n)), o_words = o_st + al16(sizeof(DStatus)),
                 o_states = o_words + 16, o_pay = al16(o_states + size_t(n_lanes) * 4),
                 total = o_pay + size_t(n) * 2 + 32;
    const bool staged = total <= kStageMax;
    uint8_t *dmsg, *dscr, *dwords, *dstates;
    DStatus *dst;
    if (staged) {
        CK(c.stage.ensure(total));
        CK(c.io.ensure(total));
        std::memcpy(c.stage.at(0), msg, size_t(n));
        dstatus_init(reinterpret_cast<DStatus *>(c.stage.at(o_st)));
        CK(cudaMemcpyAsync(c.io.p, c.stage.at(0), o_words, cudaMemcpyHostToDevice, s));
        uint8_t *io = c.io.as<uint8_t>();
        dmsg = io;
        dst = reinterpret_cast<DStatus *>(io + o_st);
        dwords = io + o_words;
        dstates = io + o_states;
        dscr = io + o_pay;
    } else {
        CK(c.msg.ensure(size_t(n)));
        CK(c.scratch.ensure(size_t(n) * 2 + 32));
        CK(c.states.ensure(size_t(n_lanes) * 4));
        CK(c.words.ensure(8));
        CK(cudaMemcpyAsync(c.msg.p, msg, size_t(n), cudaMemcpyHostToDevice, s));
        dstatus_reset_kernel<<<1, 1, 0, s>>>(c.status.as<DStatus>());
        ilans_note_launch();
        dmsg = c.msg.as<uint8_t>();
        dst = c.status.as<DStatus>();
        dwords = c.words.as<uint8_t>();
        dstates = c.states.as<uint8_t>();
        dscr = c.scratch.as<uint8_t>();
    }
    if (int rc = ensure_table(c, freq, n_freq, cum, nullptr, scale_bits, s, st)) return rc;
    CK(launch_encode(dmsg, n, n, n_lanes, c.table.as<TableDev>(), scale_bits,
                     reinterpret_cast<uint16_t *>(dscr), reinterpret_cast<uint32_t *>(dwords),
                     reinterpret_cast<uint32_t *>(dstates), dst, c.ws.as<uint32_t>(), s, stats));
    DStatus hs;
    uint32_t w = 0;
    if (staged) {  // status | words | states | scratch in one download
        CK(cudaMemcpyAsync(c.stage.at(o_st), dst, total - 32 - o_st, cudaMemcpyDeviceToHost, s));
        CK(ctx_wait(c));
        std::memcpy(&hs, c.stage.at(o_st), sizeof(DStatus));
        std::memcpy(&w, c.stage.at(o_words), 4);
    } else {
        if (int rc = read_dstatus(dst, s, &hs, st)) return rc;
        CK(cudaMemcpyAsync(&w, dwords, 4, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
    }
    if (hs.unenc_index >= 0) {
        st->index = hs.unenc_index;
        st->symbol = msg[hs.unenc_index];
        return st_fail(st, ILANS_ERR_UNENCODABLE, "symbol %d has frequency 0", st->symbol);
    }
    st->max_digits = int32_t(hs.max_digits);
    if (staged) {  // the payload is the right-aligned tail of the scratch
        std::memcpy(payload_out, c.stage.at(o_pay) + size_t(n - w) * 2, size_t(w) * 2);
        std::memcpy(states_out, c.stage.at(o_states), size_t(n_lanes) * 4);
    } else {
        if (w)
            CK(cudaMemcpyAsync(payload_out, dscr + size_t(n - w) * 2, size_t(w) * 2,
                               cudaMemcpyDeviceToHost, s));
        CK(cudaMemcpyAsync(states_out, dstates, size_t(n_lanes) * 4, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
    }
    *payload_words = w;
    return ILANS_OK;
}

extern "C" int ilans_encode_interleaved_u16(const uint8_t *msg, int64_t n, const uint32_t *freq,
                                            int32_t n_freq, const uint32_t *cum,
                                            int32_t scale_bits, int32_t n_lanes,
                                            uint16_t *payload_out, int64_t *payload_words,
                                            uint32_t *states_out, ilans_status *st) {
    st_clear(st);
    return encode_u16_common(msg, n, freq, n_freq, cum, scale_bits, n_lanes, payload_out,
                             payload_words, states_out, false, st);
}

extern "C" int ilans_encode_interleaved_u16_stats(const uint8_t *msg, int64_t n,
                                                  const uint32_t *freq, int32_t n_freq,
                                                  const uint32_t *cum, int32_t scale_bits,
                                                  int32_t n_lanes, uint16_t *payload_out,
                                                  int64_t *payload_words, uint32_t *states_out,
                                                  ilans_status *st) {
    st_clear(st);
    return encode_u16_common(msg, n, freq, n_freq, cum, scale_bits, n_lanes, payload_out,
                             payload_words, states_out, true, st);
}

struct HostTrace {  // host buffers for ilans_decode_trace_u16 (all null = no trace)
    uint32_t *states;
    uint64_t *pos;
    int64_t *groups;
};

static int decode_common(const uint16_t *payload, int64_t pay_len, const uint32_t *states,
                         const uint8_t *slot_sym, int64_t n_slots, const uint32_t *freq,
                         const uint32_t *cum, int32_t n_freq, int32_t scale_bits,
                         int64_t msg_len, int32_t n_lanes, uint8_t *out, int64_t *consumed,
                         ilans_status *st, HostTrace ht = HostTrace{nullptr, nullptr, nullptr},
                         bool stats = false) {
    if (msg_len < 0 || pay_len < 0) return st_fail(st, ILANS_ERR_VALUE, "negative length");
    if (n_lanes < 1 || n_lanes > 0xFFFF)
        return st_fail(st, ILANS_ERR_VALUE, "lane_count must be in [1, 65535]");
    if (scale_bits < 1 || scale_bits > kMaxScaleBits)
        return st_fail(st, ILANS_ERR_VALUE, "scale_bits must be in [1, 16]");
    if (n_freq < 0 || n_freq > kMaxSym)
        return st_fail(st, ILANS_ERR_VALUE, "alphabet size must be in [1, 256]");
    const int64_t m = int64_t(1) << scale_bits;
    if (n_slots < m) return st_fail(st, ILANS_ERR_VALUE, "slot table shorter than 2^scale_bits");
    Ctx *cp = nullptr;
    if (int rc = current_device(st, &cp)) return rc;
    Ctx &c = *cp;
    std::lock_guard<std::mutex> lock(c.mu);
    if (int rc = ctx_init(c, st)) return rc;
    if (msg_len == 0) {
        *consumed = 0;
        st->consumed = 0;
        st->max_digits = 0;
        if (ht.groups) *ht.groups = 0;
        return ILANS_OK;
    }
    cudaStream_t s = c.stream;
    const int64_t n_groups = (msg_len + n_lanes - 1) / n_lanes;
    DecodeTrace dt{nullptr, nullptr, nullptr, stats ? 1 : 0};
    if (ht.states) {
        CK(c.trace.ensure(size_t(n_groups) * n_lanes * 4 + size_t(n_groups) * 8 + 16));
        dt.states = c.trace.as<uint32_t>();
        dt.pos = reinterpret_cast<uint64_t *>(
            c.trace.as<uint8_t>() + ((size_t(n_groups) * n_lanes * 4 + 7) & ~size_t(7)));
        CK(c.words.ensure(8));
        dt.groups = reinterpret_cast<uint64_t *>(c.words.p);
    }
    CK(c.ws.ensure(size_t(n_lanes) * 4));
    // layout: offsets | states | payload | status | consumed | out -- the
    // first four go up in one copy, the last three come back in one
    const size_t o_states = 16, o_pay = al16(o_states + size_t(n_lanes) * 4),
                 o_st = al16(o_pay + size_t(pay_len) * 2 + 16),
                 o_used = o_st + al16(sizeof(DStatus)), o_out = o_used + 16,
                 total = o_out + size_t(msg_len);
    const bool staged = !ht.states && total <= kStageMax;
    const uint64_t offs[2] = {0, uint64_t(pay_len)};
    uint8_t *dpay, *doffs, *dstates, *dout, *dused;
    DStatus *dst;
    if (staged) {
        CK(c.stage.ensure(total));
        CK(c.io.ensure(total));
        std::memcpy(c.stage.at(0), offs, sizeof(offs));
        std::memcpy(c.stage.at(o_states), states, size_t(n_lanes) * 4);
        if (pay_len) std::memcpy(c.stage.at(o_pay), payload, size_t(pay_len) * 2);
        dstatus_init(reinterpret_cast<DStatus *>(c.stage.at(o_st)));
        CK(cudaMemcpyAsync(c.io.p, c.stage.at(0), o_used, cudaMemcpyHostToDevice, s));
        uint8_t *io = c.io.as<uint8_t>();
        doffs = io;
        dstates = io + o_states;
        dpay = io + o_pay;
        dst = reinterpret_cast<DStatus *>(io + o_st);
        dused = io + o_used;
        dout = io + o_out;
    } else {
        CK(c.payload.ensure(size_t(pay_len) * 2 + 16));
        CK(c.offsets.ensure(16));
        CK(c.states.ensure(size_t(n_lanes) * 4));
        CK(c.out.ensure(size_t(msg_len)));
        CK(c.consumed.ensure(8));
        if (pay_len)
            CK(cudaMemcpyAsync(c.payload.p, payload, size_t(pay_len) * 2, cudaMemcpyHostToDevice,
                               s));
        CK(cudaMemcpyAsync(c.offsets.p, offs, sizeof(offs), cudaMemcpyHostToDevice, s));
        CK(cudaMemcpyAsync(c.states.p, states, size_t(n_lanes) * 4, cudaMemcpyHostToDevice, s));
        dstatus_reset_kernel<<<1, 1, 0, s>>>(c.status.as<DStatus>());
        ilans_note_launch();
        doffs = c.offsets.as<uint8_t>();
        dstates = c.states.as<uint8_t>();
        dpay = c.payload.as<uint8_t>();
        dst = c.status.as<DStatus>();
        dused = c.consumed.as<uint8_t>();
        dout = c.out.as<uint8_t>();
    }
    if (int rc = ensure_table(c, freq, n_freq, cum, slot_sym, scale_bits, s, st)) return rc;
    CK(launch_decode(reinterpret_cast<uint16_t *>(dpay), reinterpret_cast<uint64_t *>(doffs),
                     reinterpret_cast<uint32_t *>(dstates), msg_len, msg_len, n_lanes,
                     c.table.as<TableDev>(), scale_bits, c.tab_packed, dout,
                     reinterpret_cast<uint64_t *>(dused), nullptr, dst, c.ws.as<uint32_t>(), s,
                     dt));
    DStatus hs;
    uint64_t used = 0;
    if (staged) {  // status | words read | decoded bytes in one download
        CK(cudaMemcpyAsync(c.stage.at(o_st), dst, total - o_st, cudaMemcpyDeviceToHost, s));
        CK(ctx_wait(c));
        std::memcpy(&hs, c.stage.at(o_st), sizeof(DStatus));
        std::memcpy(&used, c.stage.at(o_used), 8);
    } else {
        if (int rc = read_dstatus(dst, s, &hs, st)) return rc;
        CK(cudaMemcpyAsync(&used, dused, 8, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
    }
    if (ht.states) {  // trace + decoded bytes of every completed group, even on truncation
        uint64_t g = 0;
        CK(cudaMemcpyAsync(&g, dt.groups, 8, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        *ht.groups = int64_t(g);
        if (g) {
            CK(cudaMemcpyAsync(ht.states, dt.states, size_t(g) * n_lanes * 4,
                               cudaMemcpyDeviceToHost, s));
            CK(cudaMemcpyAsync(ht.pos, dt.pos, size_t(g) * 8, cudaMemcpyDeviceToHost, s));
            const int64_t done = int64_t(g) * n_lanes < msg_len ? int64_t(g) * n_lanes : msg_len;
            CK(cudaMemcpyAsync(out, dout, size_t(done), cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s));
        }
    }
    st->max_digits = int32_t(hs.max_digits);
    if (hs.trunc_stream != ~0ull) {
        st->stream = int64_t(hs.trunc_stream);
        st->consumed = int64_t(used);
        return st_fail(st, ILANS_ERR_TRUNCATED, "payload exhausted mid-decode");
    }
    if (staged) {
        std::memcpy(out, c.stage.at(o_out), size_t(msg_len));
    } else {
        CK(cudaMemcpyAsync(out, dout, size_t(msg_len), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
    }
    *consumed = int64_t(used);
    st->consumed = int64_t(used);
    return ILANS_OK;
}

extern "C" int ilans_decode_interleaved_u16(const uint16_t *payload, int64_t pay_len,
                                            const uint32_t *states, const uint8_t *slot_sym,
                                            int64_t n_slots, const uint32_t *freq,
                                            const uint32_t *cum, int32_t n_freq,
                                            int32_t scale_bits, int64_t msg_len,
                                            int32_t n_lanes, uint8_t *out, int64_t *consumed,
                                            ilans_status *st) {
    st_clear(st);
    return decode_common(payload, pay_len, states, slot_sym, n_slots, freq, cum, n_freq,
                         scale_bits, msg_len, n_lanes, out, consumed, st);
}

extern "C" int ilans_decode_interleaved_u16_stats(const uint16_t *payload, int64_t pay_len,
                                                  const uint32_t *states, const uint8_t *slot_sym,
                                                  int64_t n_slots, const uint32_t *freq,
                                                  const uint32_t *cum, int32_t n_freq,
                                                  int32_t scale_bits, int64_t msg_len,
                                                  int32_t n_lanes, uint8_t *out,
                                                  int64_t *consumed, ilans_status *st) {
    st_clear(st);
    return decode_common(payload, pay_len, states, slot_sym, n_slots, freq, cum, n_freq,
                         scale_bits, msg_len, n_lanes, out, consumed, st,
                         HostTrace{nullptr, nullptr, nullptr}, true);
}

extern "C" int ilans_decode_trace_u16(const uint16_t *payload, int64_t pay_len,
                                      const uint32_t *states, const uint8_t *slot_sym,
                                      int64_t n_slots, const uint32_t *freq, const uint32_t *cum,
                                      int32_t n_freq, int32_t scale_bits, int64_t msg_len,
                                      int32_t n_lanes, uint8_t *out, uint32_t *trace_states,
                                      uint64_t *trace_pos, int64_t *groups_done,
                                      int64_t *consumed, ilans_status *st) {
    st_clear(st);
    if (!trace_states || !trace_pos || !groups_done)
        return st_fail(st, ILANS_ERR_VALUE, "trace buffers required");
    return decode_common(payload, pay_len, states, slot_sym, n_slots, freq, cum, n_freq,
                         scale_bits, msg_len, n_lanes, out, consumed, st,
                         HostTrace{trace_states, trace_pos, groups_done});
}

extern "C" int ilans_decode_lanes_u16(const uint16_t *payload, int64_t pay_len,
                                      const uint32_t *states, const uint8_t *slot_sym,
                                      int64_t n_slots, const uint32_t *freq, const uint32_t *cum,
                                      int32_t n_freq, int32_t scale_bits, int64_t msg_len,
                                      int32_t n_lanes, uint8_t *out, int64_t *consumed,
                                      ilans_status *st) {
    st_clear(st);
    if (n_lanes > 32) return st_fail(st, ILANS_ERR_VALUE, "at most 32 lanes");
    return decode_common(payload, pay_len, states, slot_sym, n_slots, freq, cum, n_freq,
                         scale_bits, msg_len, n_lanes, out, consumed, st);
}

// ---------------------------------------------------------------------------
// byte8 (8-bit digits, L = 2^23): single stream, host buffers
// ---------------------------------------------------------------------------
extern "C" int ilans_encode_interleaved_u8(const uint8_t *msg, int64_t n, const uint32_t *freq,
                                           int32_t n_freq, const uint32_t *cum,
                                           int32_t scale_bits, int32_t n_lanes,
                                           uint8_t *payload_out, int64_t *payload_bytes,
                                           uint32_t *states_out, ilans_status *st) {
    st_clear(st);
    if (n < 0) return st_fail(st, ILANS_ERR_VALUE, "negative message length");
    if (n_lanes < 1 || n_lanes > 0xFFFF)
        return st_fail(st, ILANS_ERR_VALUE, "lane_count must be in [1, 65535]");
    if (scale_bits < 1 || scale_bits > kMaxScaleBits)
        return st_fail(st, ILANS_ERR_VALUE, "scale_bits must be in [1, 16]");
    if (n_freq < 0 || n_freq > kMaxSym)
        return st_fail(st, ILANS_ERR_VALUE, "alphabet size must be in [1, 256]");
    if (!encode_table_fits(freq, cum, n_freq, scale_bits))
        return st_fail(st, ILANS_ERR_VALUE, "frequency / cumulative table out of range");
    Ctx *cp = nullptr;
    if (int rc = current_device(st, &cp)) return rc;
    Ctx &c = *cp;
    std::lock_guard<std::mutex> lock(c.mu);
    if (int rc = ctx_init(c, st)) return rc;
    if (n == 0) {
        for (int l = 0; l < n_lanes; ++l) states_out[l] = 1u << 23;
        *payload_bytes = 0;
        return ILANS_OK;
    }
    cudaStream_t s = c.stream;
    CK(c.msg.ensure(size_t(n)));
    CK(c.scratch.ensure(size_t(n) * 3 + 16));
    CK(c.states.ensure(size_t(n_lanes) * 4));
    CK(c.ws.ensure(size_t(n_lanes) * 4));
    CK(c.freq.ensure(kMaxSym * 4));
    CK(c.cum.ensure((kMaxSym + 1) * 4));
    CK(c.words.ensure(8));
    uint32_t hf[kMaxSym] = {0}, hc[kMaxSym + 1] = {0};
    std::memcpy(hf, freq, size_t(n_freq) * 4);
    std::memcpy(hc, cum, size_t(n_freq + 1) * 4);
    CK(cudaMemcpyAsync(c.msg.p, msg, size_t(n), cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(c.freq.p, hf, sizeof(hf), cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(c.cum.p, hc, sizeof(hc), cudaMemcpyHostToDevice, s));
    table_clobbered(c);
    CK(launch_build_table(nullptr, c.freq.as<uint32_t>(), n_freq, c.cum.as<uint32_t>(), nullptr,
                          scale_bits, c.table.as<TableDev>(), s));
    dstatus_reset_kernel<<<1, 1, 0, s>>>(c.status.as<DStatus>());
    ilans_note_launch();
    CK(launch_encode_u8(c.msg.as<uint8_t>(), n, n_lanes, c.table.as<TableDev>(),
                        c.scratch.as<uint8_t>(), c.words.as<uint32_t>(), c.states.as<uint32_t>(),
                        c.status.as<DStatus>(), c.ws.as<uint32_t>(), s));
    DStatus hs;
    if (int rc = read_dstatus(c.status.as<DStatus>(), s, &hs, st)) return rc;
    st->max_digits = int32_t(hs.max_digits);
    if (hs.unenc_index >= 0) {
        st->index = hs.unenc_index;
        st->symbol = msg[hs.unenc_index];
        return st_fail(st, ILANS_ERR_UNENCODABLE, "symbol %d has frequency 0", st->symbol);
    }
    uint32_t w = 0;
    CK(cudaMemcpyAsync(&w, c.words.p, 4, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (w)
        CK(cudaMemcpyAsync(payload_out, c.scratch.as<uint8_t>() + (3 * n - w), size_t(w),
                           cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(states_out, c.states.p, size_t(n_lanes) * 4, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    *payload_bytes = w;
    return ILANS_OK;
}

static int decode_u8_common(const uint8_t *payload, int64_t pay_len, const uint32_t *states,
                            const uint8_t *slot_sym, int64_t n_slots, const uint32_t *freq,
                            const uint32_t *cum, int32_t n_freq, int32_t scale_bits,
                            int64_t msg_len, int32_t n_lanes, uint8_t *out, int64_t *consumed,
                            ilans_status *st, HostTrace ht) {
    if (msg_len < 0 || pay_len < 0) return st_fail(st, ILANS_ERR_VALUE, "negative length");
    if (n_lanes < 1 || n_lanes > 0xFFFF)
        return st_fail(st, ILANS_ERR_VALUE, "lane_count must be in [1, 65535]");
    if (scale_bits < 1 || scale_bits > kMaxScaleBits)
        return st_fail(st, ILANS_ERR_VALUE, "scale_bits must be in [1, 16]");
    if (n_freq < 0 || n_freq > kMaxSym)
        return st_fail(st, ILANS_ERR_VALUE, "alphabet size must be in [1, 256]");
    const int64_t m = int64_t(1) << scale_bits;
    if (n_slots < m) return st_fail(st, ILANS_ERR_VALUE, "slot table shorter than 2^scale_bits");
    Ctx *cp = nullptr;
    if (int rc = current_device(st, &cp)) return rc;
    Ctx &c = *cp;
    std::lock_guard<std::mutex> lock(c.mu);
    if (int rc = ctx_init(c, st)) return rc;
    if (msg_len == 0) {
        *consumed = 0;
        if (ht.groups) *ht.groups = 0;
        return ILANS_OK;
    }
    cudaStream_t s = c.stream;
    const int64_t n_groups = (msg_len + n_lanes - 1) / n_lanes;
    DecodeTrace dt{nullptr, nullptr, nullptr, 0};
    if (ht.states) {
        CK(c.trace.ensure(size_t(n_groups) * n_lanes * 4 + size_t(n_groups) * 8 + 16));
        CK(c.words.ensure(8));
        dt.states = c.trace.as<uint32_t>();
        dt.pos = reinterpret_cast<uint64_t *>(
            c.trace.as<uint8_t>() + ((size_t(n_groups) * n_lanes * 4 + 7) & ~size_t(7)));
        dt.groups = reinterpret_cast<uint64_t *>(c.words.p);
    }
    CK(c.payload.ensure(size_t(pay_len) + 16));
    CK(c.offsets.ensure(16));
    CK(c.states.ensure(size_t(n_lanes) * 4));
    CK(c.ws.ensure(size_t(n_lanes) * 4));
    CK(c.slot.ensure(size_t(m)));
    CK(c.freq.ensure(kMaxSym * 4));
    CK(c.cum.ensure((kMaxSym + 1) * 4));
    CK(c.out.ensure(size_t(msg_len)));
    CK(c.consumed.ensure(8));
    uint32_t hf[kMaxSym] = {0}, hc[kMaxSym + 1] = {0};
    std::memcpy(hf, freq, size_t(n_freq) * 4);
    std::memcpy(hc, cum, size_t(n_freq + 1) * 4);
    const uint64_t offs[2] = {0, uint64_t(pay_len)};
    if (pay_len)
        CK(cudaMemcpyAsync(c.payload.p, payload, size_t(pay_len), cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(c.offsets.p, offs, sizeof(offs), cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(c.states.p, states, size_t(n_lanes) * 4, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(c.slot.p, slot_sym, size_t(m), cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(c.freq.p, hf, sizeof(hf), cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(c.cum.p, hc, sizeof(hc), cudaMemcpyHostToDevice, s));
    table_clobbered(c);
    CK(launch_build_table(nullptr, c.freq.as<uint32_t>(), n_freq, c.cum.as<uint32_t>(),
                          c.slot.as<uint8_t>(), scale_bits, c.table.as<TableDev>(), s));
    dstatus_reset_kernel<<<1, 1, 0, s>>>(c.status.as<DStatus>());
    ilans_note_launch();
    CK(launch_decode_u8(c.payload.as<uint8_t>(), uint64_t(pay_len), c.offsets.as<uint64_t>(),
                        c.states.as<uint32_t>(), msg_len, n_lanes, c.table.as<TableDev>(),
                        c.out.as<uint8_t>(), c.consumed.as<uint64_t>(), c.status.as<DStatus>(),
                        c.ws.as<uint32_t>(), s, dt));
    DStatus hs;
    if (int rc = read_dstatus(c.status.as<DStatus>(), s, &hs, st)) return rc;
    uint64_t used = 0;
    CK(cudaMemcpyAsync(&used, c.consumed.p, 8, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (ht.states) {
        uint64_t g = 0;
        CK(cudaMemcpyAsync(&g, dt.groups, 8, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        *ht.groups = int64_t(g);
        if (g) {
            CK(cudaMemcpyAsync(ht.states, dt.states, size_t(g) * n_lanes * 4,
                               cudaMemcpyDeviceToHost, s));
            CK(cudaMemcpyAsync(ht.pos, dt.pos, size_t(g) * 8, cudaMemcpyDeviceToHost, s));
            const int64_t done = int64_t(g) * n_lanes < msg_len ? int64_t(g) * n_lanes : msg_len;
            CK(cudaMemcpyAsync(out, c.out.p, size_t(done), cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s));
        }
    }
    st->consumed = int64_t(used);
    st->max_digits = int32_t(hs.max_digits);
    if (hs.value_error == ILANS_ERR_FORMAT)
        return st_fail(st, ILANS_ERR_FORMAT, "renormalization does not terminate; corrupt stream");
    if (hs.trunc_stream != ~0ull) {
        st->stream = int64_t(hs.trunc_stream);
        return st_fail(st, ILANS_ERR_TRUNCATED, "digit stream exhausted mid-decode");
    }
    CK(cudaMemcpyAsync(out, c.out.p, size_t(msg_len), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    *consumed = int64_t(used);
    return ILANS_OK;
}

extern "C" int ilans_decode_interleaved_u8(const uint8_t *payload, int64_t pay_len,
                                           const uint32_t *states, const uint8_t *slot_sym,
                                           int64_t n_slots, const uint32_t *freq,
                                           const uint32_t *cum, int32_t n_freq,
                                           int32_t scale_bits, int64_t msg_len, int32_t n_lanes,
                                           uint8_t *out, int64_t *consumed, ilans_status *st) {
    st_clear(st);
    return decode_u8_common(payload, pay_len, states, slot_sym, n_slots, freq, cum, n_freq,
                            scale_bits, msg_len, n_lanes, out, consumed, st,
                            HostTrace{nullptr, nullptr, nullptr});
}

extern "C" int ilans_decode_trace_u8(const uint8_t *payload, int64_t pay_len,
                                     const uint32_t *states, const uint8_t *slot_sym,
                                     int64_t n_slots, const uint32_t *freq, const uint32_t *cum,
                                     int32_t n_freq, int32_t scale_bits, int64_t msg_len,
                                     int32_t n_lanes, uint8_t *out, uint32_t *trace_states,
                                     uint64_t *trace_pos, int64_t *groups_done,
                                     int64_t *consumed, ilans_status *st) {
    st_clear(st);
    if (!trace_states || !trace_pos || !groups_done)
        return st_fail(st, ILANS_ERR_VALUE, "trace buffers required");
    return decode_u8_common(payload, pay_len, states, slot_sym, n_slots, freq, cum, n_freq,
                            scale_bits, msg_len, n_lanes, out, consumed, st,
                            HostTrace{trace_states, trace_pos, groups_done});
}

// ---------------------------------------------------------------------------
// any RenormVariant (variant.cu): the reference's scalar path for variants
// other than word16 / byte8, digits as u16 (one per element)
// ---------------------------------------------------------------------------
static int check_variant(int32_t digit_bits, uint32_t lower_bound, int32_t scale_bits,
                         int32_t n_lanes, ilans_status *st) {
    if (digit_bits < 1 || digit_bits > 16)
        return st_fail(st, ILANS_ERR_VALUE, "digit_bits must be in [1, 16]");
    if (lower_bound < 1 || (uint64_t(lower_bound) << digit_bits) > (uint64_t(1) << 32))
        return st_fail(st, ILANS_ERR_VALUE, "radix * lower_bound must fit in 32 bits");
    if (scale_bits < 1 || scale_bits > kMaxScaleBits)
        return st_fail(st, ILANS_ERR_VALUE, "scale_bits must be in [1, 16]");
    if (lower_bound % (uint32_t(1) << scale_bits))
        return st_fail(st, ILANS_ERR_VALUE, "lower_bound is not a multiple of the table total");
    if (n_lanes < 1 || n_lanes > kVarMaxLanes)
        return st_fail(st, ILANS_ERR_UNSUPPORTED, "custom variants take 1..%d lanes", kVarMaxLanes);
    return ILANS_OK;
}

extern "C" int ilans_encode_interleaved_var(const uint8_t *msg, int64_t n, const uint32_t *freq,
                                            int32_t n_freq, const uint32_t *cum,
                                            int32_t scale_bits, int32_t n_lanes,
                                            int32_t digit_bits, uint32_t lower_bound,
                                            uint16_t *digits_out, int64_t digits_cap,
                                            int64_t *n_digits, uint32_t *states_out,
                                            ilans_status *st) {
    st_clear(st);
    if (n < 0 || digits_cap < 0) return st_fail(st, ILANS_ERR_VALUE, "negative length");
    if (int rc = check_variant(digit_bits, lower_bound, scale_bits, n_lanes, st)) return rc;
    if (n_freq < 0 || n_freq > kMaxSym)
        return st_fail(st, ILANS_ERR_VALUE, "alphabet size must be in [1, 256]");
    // a symbol spills at most ceil(sb / digit_bits) digits (x < L 2^b, T >= (L / m) 2^b)
    const int64_t kmax = (scale_bits + digit_bits - 1) / digit_bits + 1;
    if (digits_cap < n * kmax) return st_fail(st, ILANS_ERR_VALUE, "digit buffer too small");
    Ctx *cp = nullptr;
    if (int rc = current_device(st, &cp)) return rc;
    Ctx &c = *cp;
    std::lock_guard<std::mutex> lock(c.mu);
    if (int rc = ctx_init(c, st)) return rc;
    if (n == 0) {
        for (int l = 0; l < n_lanes; ++l) states_out[l] = lower_bound;
        *n_digits = 0;
        return ILANS_OK;
    }
    cudaStream_t s = c.stream;
    const int64_t cap = n * kmax;
    CK(c.msg.ensure(size_t(n)));
    CK(c.scratch.ensure(size_t(cap) * 2));
    CK(c.states.ensure(size_t(n_lanes) * 4));
    CK(c.words.ensure(8));
    CK(cudaMemcpyAsync(c.msg.p, msg, size_t(n), cudaMemcpyHostToDevice, s));
    if (int rc = ensure_table(c, freq, n_freq, cum, nullptr, scale_bits, s, st)) return rc;
    dstatus_reset_kernel<<<1, 1, 0, s>>>(c.status.as<DStatus>());
    ilans_note_launch();
    CK(launch_encode_var(c.msg.as<uint8_t>(), n, n_lanes, c.table.as<TableDev>(), digit_bits,
                         lower_bound, c.scratch.as<uint16_t>(), cap, c.words.as<uint64_t>(),
                         c.states.as<uint32_t>(), c.status.as<DStatus>(), s));
    DStatus hs;
    if (int rc = read_dstatus(c.status.as<DStatus>(), s, &hs, st)) return rc;
    st->max_digits = int32_t(hs.max_digits);
    if (hs.unenc_index >= 0) {
        st->index = hs.unenc_index;
        st->symbol = msg[hs.unenc_index];
        return st_fail(st, ILANS_ERR_UNENCODABLE, "symbol %d has frequency 0", st->symbol);
    }
    uint64_t w = 0;
    CK(cudaMemcpyAsync(&w, c.words.p, 8, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (w)
        CK(cudaMemcpyAsync(digits_out, c.scratch.as<uint16_t>() + (cap - int64_t(w)),
                           size_t(w) * 2, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(states_out, c.states.p, size_t(n_lanes) * 4, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    *n_digits = int64_t(w);
    return ILANS_OK;
}

extern "C" int ilans_decode_interleaved_var(const uint16_t *payload, int64_t pay_len,
                                            const uint32_t *states, const uint8_t *slot_sym,
                                            int64_t n_slots, const uint32_t *freq,
                                            const uint32_t *cum, int32_t n_freq,
                                            int32_t scale_bits, int64_t msg_len, int32_t n_lanes,
                                            int32_t digit_bits, uint32_t lower_bound,
                                            uint8_t *out, int64_t *consumed,
                                            uint32_t *trace_states, uint64_t *trace_pos,
                                            int64_t *groups_done, ilans_status *st) {
    st_clear(st);
    if (msg_len < 0 || pay_len < 0) return st_fail(st, ILANS_ERR_VALUE, "negative length");
    if (int rc = check_variant(digit_bits, lower_bound, scale_bits, n_lanes, st)) return rc;
    if (n_freq < 0 || n_freq > kMaxSym)
        return st_fail(st, ILANS_ERR_VALUE, "alphabet size must be in [1, 256]");
    const int64_t m = int64_t(1) << scale_bits;
    if (n_slots < m) return st_fail(st, ILANS_ERR_VALUE, "slot table shorter than 2^scale_bits");
    const bool traced = trace_states && trace_pos && groups_done;
    Ctx *cp = nullptr;
    if (int rc = current_device(st, &cp)) return rc;
    Ctx &c = *cp;
    std::lock_guard<std::mutex> lock(c.mu);
    if (int rc = ctx_init(c, st)) return rc;
    if (msg_len == 0) {
        *consumed = 0;
        st->consumed = 0;
        if (groups_done) *groups_done = 0;
        return ILANS_OK;
    }
    cudaStream_t s = c.stream;
    const int64_t n_groups = (msg_len + n_lanes - 1) / n_lanes;
    DecodeTrace dt{nullptr, nullptr, nullptr, 0};
    if (traced) {
        CK(c.trace.ensure(size_t(n_groups) * n_lanes * 4 + size_t(n_groups) * 8 + 16));
        dt.states = c.trace.as<uint32_t>();
        dt.pos = reinterpret_cast<uint64_t *>(
            c.trace.as<uint8_t>() + ((size_t(n_groups) * n_lanes * 4 + 7) & ~size_t(7)));
        CK(c.words.ensure(8));
        dt.groups = reinterpret_cast<uint64_t *>(c.words.p);
    }
    CK(c.payload.ensure(size_t(pay_len) * 2 + 16));
    CK(c.states.ensure(size_t(n_lanes) * 4));
    CK(c.out.ensure(size_t(msg_len)));
    CK(c.consumed.ensure(8));
    if (pay_len)
        CK(cudaMemcpyAsync(c.payload.p, payload, size_t(pay_len) * 2, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(c.states.p, states, size_t(n_lanes) * 4, cudaMemcpyHostToDevice, s));
    if (int rc = ensure_table(c, freq, n_freq, cum, slot_sym, scale_bits, s, st)) return rc;
    dstatus_reset_kernel<<<1, 1, 0, s>>>(c.status.as<DStatus>());
    ilans_note_launch();
    CK(launch_decode_var(c.payload.as<uint16_t>(), pay_len, c.states.as<uint32_t>(), msg_len,
                         n_lanes, c.table.as<TableDev>(), digit_bits, lower_bound,
                         c.out.as<uint8_t>(), c.consumed.as<uint64_t>(), c.status.as<DStatus>(),
                         s, dt));
    DStatus hs;
    if (int rc = read_dstatus(c.status.as<DStatus>(), s, &hs, st)) return rc;
    uint64_t used = 0;
    CK(cudaMemcpyAsync(&used, c.consumed.p, 8, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (traced) {
        uint64_t g = 0;
        CK(cudaMemcpyAsync(&g, dt.groups, 8, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        *groups_done = int64_t(g);
        if (g) {
            CK(cudaMemcpyAsync(trace_states, dt.states, size_t(g) * n_lanes * 4,
                               cudaMemcpyDeviceToHost, s));
            CK(cudaMemcpyAsync(trace_pos, dt.pos, size_t(g) * 8, cudaMemcpyDeviceToHost, s));
            const int64_t done = int64_t(g) * n_lanes < msg_len ? int64_t(g) * n_lanes : msg_len;
            CK(cudaMemcpyAsync(out, c.out.p, size_t(done), cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s));
        }
    }
    st->consumed = int64_t(used);
    st->max_digits = int32_t(hs.max_digits);
    if (hs.value_error == ILANS_ERR_FORMAT)
        return st_fail(st, ILANS_ERR_FORMAT, "renormalization does not terminate; corrupt stream");
    if (hs.trunc_stream != ~0ull) {
        st->stream = int64_t(hs.trunc_stream);
        return st_fail(st, ILANS_ERR_TRUNCATED, "digit stream exhausted mid-decode");
    }
    CK(cudaMemcpyAsync(out, c.out.p, size_t(msg_len), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    *consumed = int64_t(used);
    return ILANS_OK;
}

extern "C" int ilans_quantize(const uint64_t *counts, int32_t n, int32_t scale_bits,
                              uint32_t *freq_out, ilans_status *st) {
    st_clear(st);
    if (scale_bits < 1 || scale_bits > kMaxScaleBits)
        return st_fail(st, ILANS_ERR_VALUE, "scale_bits must be in [1, %d]", kMaxScaleBits);
    if (n > kMaxSym) return st_fail(st, ILANS_ERR_VALUE, "alphabet size must be <= %d", kMaxSym);
    bool any = false;
    for (int i = 0; i < n; ++i) any |= counts[i] != 0;
    if (!any) return st_fail(st, ILANS_ERR_VALUE, "at least one count must be positive");
    Ctx *cp = nullptr;
    if (int rc = current_device(st, &cp)) return rc;
    Ctx &c = *cp;
    std::lock_guard<std::mutex> lock(c.mu);
    if (int rc = ctx_init(c, st)) return rc;
    cudaStream_t s = c.stream;
    CK(c.counts.ensure(kMaxSym * 8));
    uint64_t hc[kMaxSym] = {0};
    std::memcpy(hc, counts, size_t(n) * 8);
    CK(cudaMemcpyAsync(c.counts.p, hc, sizeof(hc), cudaMemcpyHostToDevice, s));
    table_clobbered(c);
    CK(launch_build_table(c.counts.as<unsigned long long>(), nullptr, 0, nullptr, nullptr,
                          scale_bits, c.table.as<TableDev>(), s));
    TableDev *h = static_cast<TableDev *>(std::malloc(sizeof(TableDev)));
    if (!h) return st_fail(st, ILANS_ERR_VALUE, "host allocation failed");
    cudaError_t e = cudaMemcpyAsync(h, c.table.p, offsetof(TableDev, cum), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) {
        std::free(h);
        return st_cuda(st, e, "quantize readback");
    }
    int rc = ILANS_OK;
    if (h->status != ILANS_OK) {
        if (h->err_detail[0] == 2)
            rc = st_fail(st, ILANS_ERR_VALUE,
                         "alphabet too large for scale: %u present symbols, only %u slots",
                         h->err_detail[1], h->err_detail[2]);
        else
            rc = st_fail(st, ILANS_ERR_VALUE, "quantize failed (%u)", h->err_detail[0]);
    } else {
        std::memcpy(freq_out, h->freq, size_t(n) * 4);
    }
    std::free(h);
    return rc;
}

extern "C" int ilans_histogram_u8(const uint8_t *msg, int64_t n, uint64_t *counts_out,
                                  int32_t *alphabet, ilans_status *st) {
    st_clear(st);
    if (n < 0) return st_fail(st, ILANS_ERR_VALUE, "negative length");
    Ctx *cp = nullptr;
    if (int rc = current_device(st, &cp)) return rc;
    Ctx &c = *cp;
    std::lock_guard<std::mutex> lock(c.mu);
    if (int rc = ctx_init(c, st)) return rc;
    cudaStream_t s = c.stream;
    CK(c.counts.ensure(kMaxSym * 8));
    CK(cudaMemsetAsync(c.counts.p, 0, kMaxSym * 8, s));
    if (n > 0) {
        CK(c.msg.ensure(size_t(n)));
        CK(cudaMemcpyAsync(c.msg.p, msg, size_t(n), cudaMemcpyHostToDevice, s));
        CK(launch_histogram(c.msg.as<uint8_t>(), n, c.counts.as<unsigned long long>(), s));
    }
    CK(cudaMemcpyAsync(counts_out, c.counts.p, kMaxSym * 8, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    int a = 0;
    for (int i = 0; i < kMaxSym; ++i)
        if (counts_out[i]) a = i + 1;
    if (alphabet) *alphabet = a;
    return ILANS_OK;
}

// ---------------------------------------------------------------------------
// 2. device-pointer pipeline
// ---------------------------------------------------------------------------
#define ST(x) static_cast<cudaStream_t>(x)

// the Adler-32 sinks keep sum(i * b_i) of a chunk in u64 (~255 C^2 / 2):
// exact for chunks up to 2^27 bytes
constexpr int64_t kAdlerMaxChunk = int64_t(1) << 27;


extern "C" int ilans_counts_zero_dev(uint64_t *d_counts, void *stream) {
    return cudaMemsetAsync(d_counts, 0, kMaxSym * 8, ST(stream)) == cudaSuccess ? ILANS_OK
                                                                               : ILANS_ERR_CUDA;
}

extern "C" int ilans_histogram_u8_dev(const uint8_t *d_msg, int64_t n, uint64_t *d_counts,
                                      void *stream) {
    return launch_histogram(d_msg, n, reinterpret_cast<unsigned long long *>(d_counts),
                            ST(stream)) == cudaSuccess ? ILANS_OK : ILANS_ERR_CUDA;
}

extern "C" int ilans_table_from_counts_dev(const uint64_t *d_counts, int32_t scale_bits,
                                           void *d_table, void *stream) {
    return launch_build_table(reinterpret_cast<const unsigned long long *>(d_counts), nullptr, 0,
                              nullptr, nullptr, scale_bits, static_cast<TableDev *>(d_table),
                              ST(stream)) == cudaSuccess ? ILANS_OK : ILANS_ERR_CUDA;
}

extern "C" int ilans_table_from_freq_dev(const uint32_t *d_freq, int32_t n_freq,
                                         int32_t scale_bits, void *d_table, void *stream) {
    if (n_freq < 1 || n_freq > kMaxSym) return ILANS_ERR_VALUE;
    return launch_build_table(nullptr, d_freq, n_freq, nullptr, nullptr, scale_bits,
                              static_cast<TableDev *>(d_table), ST(stream)) == cudaSuccess
               ? ILANS_OK
               : ILANS_ERR_CUDA;
}

extern "C" int ilans_table_read_host(const void *d_table, int32_t *alphabet, int32_t *scale_bits,
                                     uint32_t *freq_out, void *stream, ilans_status *st) {
    st_clear(st);
    TableDev *h = static_cast<TableDev *>(std::malloc(offsetof(TableDev, cum)));
    if (!h) return st_fail(st, ILANS_ERR_VALUE, "host allocation failed");
    cudaError_t e = cudaMemcpyAsync(h, d_table, offsetof(TableDev, cum), cudaMemcpyDeviceToHost,
                                    ST(stream));
    if (e == cudaSuccess) e = cudaStreamSynchronize(ST(stream));
    if (e != cudaSuccess) {
        std::free(h);
        return st_cuda(st, e, "table readback");
    }
    if (alphabet) *alphabet = int32_t(h->n_sym);
    if (scale_bits) *scale_bits = int32_t(h->scale_bits);
    if (freq_out) std::memcpy(freq_out, h->freq, sizeof(h->freq));
    int rc = ILANS_OK;
    if (h->status != ILANS_OK) {
        if (h->err_detail[0] == 2)
            rc = st_fail(st, ILANS_ERR_VALUE,
                         "alphabet too large for scale: %u present symbols, only %u slots",
                         h->err_detail[1], h->err_detail[2]);
        else
            rc = st_fail(st, ILANS_ERR_VALUE, "invalid model (%u)", h->err_detail[0]);
    }
    std::free(h);
    return rc;
}

extern "C" int ilans_dstatus_reset_dev(void *d_status, void *stream) {
    dstatus_reset_kernel<<<1, 1, 0, ST(stream)>>>(static_cast<DStatus *>(d_status));
    ilans_note_launch();
    return cudaGetLastError() == cudaSuccess ? ILANS_OK : ILANS_ERR_CUDA;
}

extern "C" int ilans_dstatus_read_host(const void *d_status, void *stream, ilans_status *st) {
    st_clear(st);
    DStatus h;
    cudaError_t e = cudaMemcpyAsync(&h, d_status, sizeof(h), cudaMemcpyDeviceToHost, ST(stream));
    if (e == cudaSuccess) e = cudaStreamSynchronize(ST(stream));
    if (e != cudaSuccess) return st_cuda(st, e, "status readback");
    return ilans_dstatus_parse(&h, st);
}

extern "C" int ilans_dstatus_parse(const void *h_status, ilans_status *st) {
    st_clear(st);
    DStatus h;
    std::memcpy(&h, h_status, sizeof(h));
    if (h.trunc_stream != ~0ull) {
        st->stream = int64_t(h.trunc_stream);
        return st_fail(st, ILANS_ERR_TRUNCATED, "payload exhausted mid-decode (chunk %lld)",
                       static_cast<long long>(h.trunc_stream));
    }
    if (h.value_error == ILANS_ERR_FORMAT)  // byte8: a refill loop that does not terminate
        return st_fail(st, ILANS_ERR_FORMAT, "renormalization does not terminate; corrupt stream");
    if (h.value_error) {
        return st_fail(st, ILANS_ERR_VALUE, "table does not match the launch (scale_bits / layout)");
    }
    if (h.unenc_index >= 0) {
        st->index = h.unenc_index;
        return st_fail(st, ILANS_ERR_UNENCODABLE, "zero-frequency symbol at index %lld",
                       static_cast<long long>(h.unenc_index));
    }
    return ILANS_OK;
}

static int encode_chunks(const uint8_t *d_msg, int64_t n, int64_t chunk_len, int32_t n_lanes,
                         const void *d_table, int32_t scale_bits, uint16_t *d_scratch,
                         uint32_t *d_chunk_words, uint32_t *d_states, void *d_status,
                         void *stream, bool covered) {
    if (n_lanes < 1 || n_lanes > 32 || chunk_len <= 0 || (chunk_len & 15)) return ILANS_ERR_VALUE;
    if (scale_bits < 1 || scale_bits > kMaxScaleBits) return ILANS_ERR_VALUE;
    if (reinterpret_cast<uintptr_t>(d_msg) & 15) return ILANS_ERR_VALUE;
    return launch_encode(d_msg, n, chunk_len, n_lanes, static_cast<const TableDev *>(d_table),
                         scale_bits, d_scratch, d_chunk_words, d_states,
                         static_cast<DStatus *>(d_status), nullptr, ST(stream), false,
                         covered) == cudaSuccess
               ? ILANS_OK
               : ILANS_ERR_CUDA;
}

extern "C" int ilans_encode_chunks_dev(const uint8_t *d_msg, int64_t n, int64_t chunk_len,
                                       int32_t n_lanes, const void *d_table, int32_t scale_bits,
                                       uint16_t *d_scratch, uint32_t *d_chunk_words,
                                       uint32_t *d_states, void *d_status, void *stream) {
    return encode_chunks(d_msg, n, chunk_len, n_lanes, d_table, scale_bits, d_scratch,
                         d_chunk_words, d_states, d_status, stream, false);
}

extern "C" int ilans_encode_chunks_covered_dev(const uint8_t *d_msg, int64_t n,
                                               int64_t chunk_len, int32_t n_lanes,
                                               const void *d_table, int32_t scale_bits,
                                               uint16_t *d_scratch, uint32_t *d_chunk_words,
                                               uint32_t *d_states, void *d_status, void *stream) {
    return encode_chunks(d_msg, n, chunk_len, n_lanes, d_table, scale_bits, d_scratch,
                         d_chunk_words, d_states, d_status, stream, true);
}

extern "C" int ilans_frame_chunks_dev(const uint16_t *d_scratch, int64_t n, int64_t chunk_len,
                                      const uint32_t *d_chunk_words, uint64_t *d_word_offsets,
                                      uint16_t *d_payload, int32_t carry_in, void *stream) {
    if (chunk_len <= 0) return ILANS_ERR_VALUE;
    return launch_frame(d_scratch, n, chunk_len, d_chunk_words, d_word_offsets, d_payload,
                        carry_in, ST(stream)) == cudaSuccess ? ILANS_OK : ILANS_ERR_CUDA;
}

extern "C" int ilans_decode_chunks_dev(const uint16_t *d_payload, const uint64_t *d_word_offsets,
                                       const uint32_t *d_states, int64_t n, int64_t chunk_len,
                                       int32_t n_lanes, const void *d_table, int32_t scale_bits,
                                       uint8_t *d_out, uint64_t *d_consumed,
                                       uint32_t *d_final_states, void *d_status, void *stream) {
    if (n_lanes < 1 || n_lanes > 32 || chunk_len <= 0 || (chunk_len & 15)) return ILANS_ERR_VALUE;
    if (scale_bits < 1 || scale_bits > kMaxScaleBits) return ILANS_ERR_VALUE;
    if ((reinterpret_cast<uintptr_t>(d_payload) & 15) || (reinterpret_cast<uintptr_t>(d_out) & 15))
        return ILANS_ERR_VALUE;
    // scale_bits <= 12: the kernel reads the device table's packed flag and
    // takes the packed or the two-lookup LUT; it re-checks scale_bits against
    // the launch and records a value error instead of decoding a mismatch.
    const bool packed = scale_bits <= kPackedMaxBits;
    return launch_decode(d_payload, d_word_offsets, d_states, n, chunk_len, n_lanes,
                         static_cast<const TableDev *>(d_table), scale_bits, packed, d_out,
                         d_consumed, d_final_states, static_cast<DStatus *>(d_status), nullptr,
                         ST(stream)) == cudaSuccess ? ILANS_OK : ILANS_ERR_CUDA;
}

extern "C" int ilans_decode_chunks_slots_dev(const uint16_t *d_scratch,
                                             const uint32_t *d_chunk_words,
                                             const uint32_t *d_states, int64_t n,
                                             int64_t chunk_len, int32_t n_lanes,
                                             const void *d_table, int32_t scale_bits,
                                             uint8_t *d_out, uint64_t *d_consumed,
                                             uint32_t *d_final_states, void *d_status,
                                             void *stream) {
    if (n_lanes < 1 || n_lanes > 32 || chunk_len <= 0 || (chunk_len & 15)) return ILANS_ERR_VALUE;
    if (scale_bits < 1 || scale_bits > kMaxScaleBits || !d_chunk_words) return ILANS_ERR_VALUE;
    if ((reinterpret_cast<uintptr_t>(d_scratch) & 15) || (reinterpret_cast<uintptr_t>(d_out) & 15))
        return ILANS_ERR_VALUE;
    const bool packed = scale_bits <= kPackedMaxBits;
    return launch_decode(d_scratch, nullptr, d_states, n, chunk_len, n_lanes,
                         static_cast<const TableDev *>(d_table), scale_bits, packed, d_out,
                         d_consumed, d_final_states, static_cast<DStatus *>(d_status), nullptr,
                         ST(stream), DecodeTrace{nullptr, nullptr, nullptr, 0},
                         d_chunk_words) == cudaSuccess ? ILANS_OK : ILANS_ERR_CUDA;
}

extern "C" int ilans_decode_chunks_slots_adler32_dev(const uint16_t *d_scratch,
                                                     const uint32_t *d_chunk_words,
                                                     const uint32_t *d_states, int64_t n,
                                                     int64_t chunk_len, int32_t n_lanes,
                                                     const void *d_table, int32_t scale_bits,
                                                     uint32_t *d_adler, uint64_t *d_consumed,
                                                     void *d_status, void *stream) {
    if (n_lanes < 1 || n_lanes > 32 || chunk_len <= 0 || (chunk_len & 15)) return ILANS_ERR_VALUE;
    if (scale_bits < 1 || scale_bits > kMaxScaleBits || !d_chunk_words) return ILANS_ERR_VALUE;
    if (reinterpret_cast<uintptr_t>(d_scratch) & 15) return ILANS_ERR_VALUE;
    if (chunk_len > kAdlerMaxChunk) return ILANS_ERR_VALUE;
    return launch_decode_adler32(d_scratch, nullptr, d_states, n, chunk_len, n_lanes,
                                 static_cast<const TableDev *>(d_table), scale_bits, d_adler,
                                 d_consumed, static_cast<DStatus *>(d_status), ST(stream),
                                 d_chunk_words) == cudaSuccess ? ILANS_OK : ILANS_ERR_CUDA;
}

extern "C" int ilans_encode_chunks_u8_dev(const uint8_t *d_msg, int64_t n, int64_t chunk_len,
                                          int32_t n_lanes, const void *d_table,
                                          uint8_t *d_scratch, uint32_t *d_chunk_bytes,
                                          uint32_t *d_states, void *d_status, void *stream) {
    if (n_lanes < 1 || n_lanes > 32 || chunk_len <= 0 || (chunk_len & 15)) return ILANS_ERR_VALUE;
    if (chunk_len > (int64_t(1) << 29)) return ILANS_ERR_VALUE;  // 32-bit chunk cursors
    return launch_encode_chunks_u8(d_msg, n, chunk_len, n_lanes,
                                   static_cast<const TableDev *>(d_table), d_scratch,
                                   d_chunk_bytes, d_states, static_cast<DStatus *>(d_status),
                                   ST(stream)) == cudaSuccess ? ILANS_OK : ILANS_ERR_CUDA;
}

extern "C" int ilans_frame_chunks_u8_dev(const uint8_t *d_scratch, int64_t n, int64_t chunk_len,
                                         const uint32_t *d_chunk_bytes, uint64_t *d_byte_offsets,
                                         uint8_t *d_payload, void *stream) {
    if (chunk_len <= 0 || (reinterpret_cast<uintptr_t>(d_scratch) & 3) ||
        (reinterpret_cast<uintptr_t>(d_payload) & 3))
        return ILANS_ERR_VALUE;
    return launch_frame_u8(d_scratch, n, chunk_len, d_chunk_bytes, d_byte_offsets, d_payload,
                           ST(stream)) == cudaSuccess ? ILANS_OK : ILANS_ERR_CUDA;
}

extern "C" int ilans_decode_chunks_u8_dev(const uint8_t *d_payload, const uint64_t *d_byte_offsets,
                                          const uint32_t *d_states, int64_t n, int64_t chunk_len,
                                          int32_t n_lanes, const void *d_table, uint8_t *d_out,
                                          uint64_t *d_consumed, void *d_status, void *stream) {
    if (n_lanes < 1 || n_lanes > 32 || chunk_len <= 0 || (chunk_len & 15)) return ILANS_ERR_VALUE;
    if (chunk_len > (int64_t(1) << 29)) return ILANS_ERR_VALUE;  // 32-bit chunk cursors
    // the payload streams into shared rings by 16-byte cp.async (byte8.cu)
    if (reinterpret_cast<uintptr_t>(d_payload) & 15) return ILANS_ERR_VALUE;
    return launch_decode_chunks_u8(d_payload, d_byte_offsets, d_states, n, chunk_len, n_lanes,
                                   static_cast<const TableDev *>(d_table), d_out, d_consumed,
                                   static_cast<DStatus *>(d_status), ST(stream)) == cudaSuccess
               ? ILANS_OK
               : ILANS_ERR_CUDA;
}

extern "C" int ilans_decode_chunks_adler32_dev(const uint16_t *d_payload,
                                               const uint64_t *d_word_offsets,
                                               const uint32_t *d_states, int64_t n,
                                               int64_t chunk_len, int32_t n_lanes,
                                               const void *d_table, int32_t scale_bits,
                                               uint32_t *d_adler, uint64_t *d_consumed,
                                               void *d_status, void *stream) {
    if (n_lanes < 1 || n_lanes > 32 || chunk_len <= 0 || (chunk_len & 15)) return ILANS_ERR_VALUE;
    if (scale_bits < 1 || scale_bits > kMaxScaleBits) return ILANS_ERR_VALUE;
    if (reinterpret_cast<uintptr_t>(d_payload) & 15) return ILANS_ERR_VALUE;
    if (chunk_len > kAdlerMaxChunk) return ILANS_ERR_VALUE;
    return launch_decode_adler32(d_payload, d_word_offsets, d_states, n, chunk_len, n_lanes,
                                 static_cast<const TableDev *>(d_table), scale_bits, d_adler,
                                 d_consumed, static_cast<DStatus *>(d_status), ST(stream)) ==
                   cudaSuccess
               ? ILANS_OK
               : ILANS_ERR_CUDA;
}

extern "C" int ilans_adler32_chunks_dev(const uint8_t *d_data, int64_t n, int64_t chunk_len,
                                        uint32_t *d_adler, void *stream) {
    if (chunk_len <= 0 || (chunk_len & 15) || (reinterpret_cast<uintptr_t>(d_data) & 15) ||
        chunk_len > kAdlerMaxChunk)
        return ILANS_ERR_VALUE;
    return launch_adler32_chunks(d_data, n, chunk_len, d_adler, ST(stream)) == cudaSuccess
               ? ILANS_OK
               : ILANS_ERR_CUDA;
}

extern "C" int ilans_synth_bytes_dev(uint8_t *d_out, int64_t n, uint64_t seed,
                                     int64_t first_index, const uint32_t *d_cdf, void *stream) {
    if (reinterpret_cast<uintptr_t>(d_out) & 15) return ILANS_ERR_VALUE;
    return launch_synth(d_out, n, seed, first_index, d_cdf, ST(stream)) == cudaSuccess
               ? ILANS_OK
               : ILANS_ERR_CUDA;
}
