// table.cu -- model builder on the device: byte histogram, bit-exact
// quantize (rans.quantize, rans.py:171-211) and the lookup tables the coders
// use (SymbolTable, rans.py:99-146).
#include <climits>

#include "common.cuh"
#include "kernels.cuh"

namespace ilans {

// ---------------------------------------------------------------------------
// Histogram (np.bincount at cli.py:31-37 / bench.py:47-51)
//
// HBM-bound streaming read. Every thread owns a private column of 16-bit
// counters (256 bins x 128 threads = 64 KB of shared memory): the 32-bit
// word (bin, w >> 1, lane) holds warp w's and warp w^1's counters, so a
// warp's 32 increments always hit 32 distinct banks whatever the byte values
// (bank = lane) and a 1-bit-entropy source (80% of bytes in one bin) costs
// the same as a uniform one. Each increment is one fire-and-forget shared
// add (red.shared of 1 << 16*(w & 1)) -- no per-thread read-modify-write
// chain, one shared-memory wavefront per 32 bytes. A counter can only carry
// into its neighbour after 65536 bytes of one thread, so the counting threads
// flush every kHistFlushStages ring slots (64 bytes per thread per slot; once
// per launch below ~2.4 GB per SM): thread t sums bins t and t+128 over all
// 128 columns and zeroes them.
// ---------------------------------------------------------------------------
// Two independent 128-thread counter blocks (64 KB each) per CTA, one CTA per
// SM, fed by the bulk-copy engine: each CTA streams its contiguous share of
// the message through a 3 x 32 KB shared ring (cp.async.bulk completing on
// an mbarrier per slot; thread 0 refills a slot right after the CTA barrier
// that ends every thread's reads of it -- a barrier, rather than a producer
// warp waiting on an "empty" mbarrier, so compute-sanitizer racecheck can
// see the read -> refill order; same speed). 96 KB in flight per SM keeps HBM busy without the
// register double-buffering of a load-and-count loop (66 us at config 2,
// ~0.6 of HBM: 12 warps/SM, long_scoreboard); measured at 256 MiB: 3 x 32 KB
// 48.6 us, 4 x 24 KB 49.3, 6 x 16 KB 50.0, 12 x 8 KB 58.6, and one counter
// block with 10 x 16 KB 55.0 (the shared atomics then lack issuing warps).
// The shared-memory pipe is the co-bound: one wavefront per 32 counted bytes
// plus four per 512-byte LDS.128 (~0.8 of one wavefront per SM clock).
constexpr int kHistGroups = 2;
constexpr int kHistCounters = 128 * kHistGroups;        // counting threads
constexpr int kHistThreads = kHistCounters;             // thread 0 also issues the copies
constexpr uint32_t kHistStage = 32768;                  // bytes per ring slot
constexpr int kHistStages = 3;
// slots between counter flushes: < 65536 bytes per thread
constexpr int kHistFlushStages = 64000 / (kHistStage / kHistCounters);
constexpr size_t kHistCounterBytes = size_t(256) * 64 * 4 * kHistGroups;
constexpr size_t kHistSmem = kHistCounterBytes + size_t(kHistStages) * kHistStage +
                             kHistStages * 8;

__device__ __forceinline__ uint32_t hist_word(uint32_t bin, uint32_t tid) {
    return bin * 64u + ((tid >> 6) << 5) + (tid & 31u);  // 64 words per bin
}

__device__ __forceinline__ void hist_red(uint32_t base_addr, uint32_t tid, uint32_t b) {
    asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(base_addr + 4u * hist_word(b, tid)),
                 "r"(1u << (((tid >> 5) & 1u) * 16)) : "memory");
}

// 16 bytes: per byte one PRMT and one RED. The thread's column offset
// (col < 256) and the bin's row offset (bin * 256) occupy different bytes of
// the address, so one PRMT assembles col | byte_j << 8; the CTA-uniform
// shared base is added by the RED's [R + UR] addressing.
__device__ __forceinline__ void hist_bump16(uint32_t base_addr, uint32_t col, uint32_t inc,
                                           uint4 v) {
    const uint32_t words[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const uint32_t off = __byte_perm(words[q], col, 0x7604u | (j << 4));
            asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(base_addr + off), "r"(inc)
                         : "memory");
        }
    }
}

// thread t: add every column's counters of bins t and t + 128 into acc[0/1]
// and zero them (staggered word order: conflict-free).
__device__ __forceinline__ void hist_flush(uint32_t *h, uint32_t tid, unsigned long long *acc) {
#pragma unroll
    for (int half = 0; half < 2; ++half) {
        uint32_t *row = h + (tid + 128u * half) * 64u;
        uint32_t sum = 0;
#pragma unroll 8
        for (int k = 0; k < 64; ++k) {
            const int idx = (k + static_cast<int>(tid)) & 63;
            const uint32_t w = row[idx];
            sum += (w & 0xFFFFu) + (w >> 16);
            row[idx] = 0;
        }
        acc[half] += sum;
    }
}

__device__ __forceinline__ void mbar_init(uint32_t addr, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(addr), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t addr, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(addr),
                 "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t addr) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(addr) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t addr, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(addr), "r"(parity) : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void *src, uint32_t bytes,
                                         uint32_t mbar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
        ::"r"(dst), "l"(src), "r"(bytes), "r"(mbar) : "memory");
}
__device__ __forceinline__ void counters_sync() {  // the 256 counting threads only
    asm volatile("bar.sync 1, %0;" ::"n"(kHistCounters) : "memory");
}

__global__ void __launch_bounds__(kHistThreads, 1)
histogram_u8_kernel(const uint8_t *__restrict__ msg, int64_t n,
                    unsigned long long *__restrict__ counts) {
    extern __shared__ __align__(128) uint32_t hist_smem[];
    const uint32_t gtid = threadIdx.x;
    const uint32_t base_addr = smem_addr(hist_smem);
    const uint32_t ring_addr = base_addr + static_cast<uint32_t>(kHistCounterBytes);
    const uint32_t full_addr = ring_addr + kHistStages * kHistStage;  // full[s]
    for (uint32_t i = gtid; i < kHistCounterBytes / 4; i += kHistThreads) hist_smem[i] = 0;
    if (gtid == 0) {
        for (int q = 0; q < kHistStages; ++q) mbar_init(full_addr + 8 * q, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    // 16-byte aligned body, split into contiguous per-CTA ranges; unaligned
    // head / tail bytes: block 0, thread 0 (its own counters)
    const uintptr_t addr = reinterpret_cast<uintptr_t>(msg);
    int64_t head = static_cast<int64_t>((16 - (addr & 15)) & 15);
    if (head > n) head = n;
    const int64_t body = ((n - head) >> 4) << 4;
    const int64_t per_cta = (((body + gridDim.x - 1) / gridDim.x) + 15) & ~int64_t(15);
    const int64_t lo = per_cta * blockIdx.x < body ? per_cta * blockIdx.x : body;
    const int64_t hi = lo + per_cta < body ? lo + per_cta : body;
    // < 2^31 slots per CTA (the message is < 2^31 * 16 KB * gridDim)
    const uint32_t n_stages = static_cast<uint32_t>((hi - lo + kHistStage - 1) / kHistStage);
    const uint32_t last_bytes =
        n_stages ? static_cast<uint32_t>(hi - lo - int64_t(n_stages - 1) * kHistStage) : 0u;
    const uint8_t *src = msg + head + lo;

    // stage i -> ring slot i % kHistStages, completing on that slot's
    // mbarrier; thread 0 issues (the first kHistStages here, each later one
    // right after the barrier that ends every thread's reads of its slot)
    auto issue = [&](uint32_t i) {
        const uint32_t q = i % kHistStages;
        const uint32_t bytes = i + 1 < n_stages ? kHistStage : last_bytes;
        mbar_expect_tx(full_addr + 8 * q, bytes);
        bulk_g2s(ring_addr + q * kHistStage, src + size_t(i) * kHistStage, bytes,
                 full_addr + 8 * q);
    };
    if (gtid == 0)
        for (uint32_t i = 0; i < kHistStages && i < n_stages; ++i) issue(i);

    const uint32_t sub = gtid >> 7;   // counter block of this thread
    const uint32_t tid = gtid & 127u;  // column within the block
    if (blockIdx.x == 0 && gtid == 0) {
        for (int64_t i = 0; i < head; ++i) hist_red(base_addr, 0, msg[i]);
        for (int64_t i = head + body; i < n; ++i) hist_red(base_addr, 0, msg[i]);
    }
    unsigned long long acc[2] = {0, 0};
    // byte 0: column (< 256), byte 1: bin (PRMT), byte 2: counter block
    const uint32_t col = 4u * hist_word(0, tid) | sub << 16;
    const uint32_t inc = 1u << (((tid >> 5) & 1u) * 16);
    constexpr int kVecs = kHistStage / 16 / kHistCounters;  // 16-byte vectors per thread per slot
    uint32_t q = 0, ph = 0, flush_left = kHistFlushStages;
    for (uint32_t i = 0; i < n_stages; ++i) {
        mbar_wait(full_addr + 8 * q, ph);
        const uint32_t slot = ring_addr + q * kHistStage + 16 * gtid;
        uint4 v[kVecs];
        if (i + 1 < n_stages || last_bytes == kHistStage) {  // full slot
#pragma unroll
            for (int r = 0; r < kVecs; ++r)
                asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                             : "=r"(v[r].x), "=r"(v[r].y), "=r"(v[r].z), "=r"(v[r].w)
                             : "r"(slot + 16 * kHistCounters * r));
            counters_sync();  // every thread has read slot q: refill it
            if (gtid == 0 && i + kHistStages < n_stages) issue(i + kHistStages);
#pragma unroll
            for (int r = 0; r < kVecs; ++r) hist_bump16(base_addr, col, inc, v[r]);
        } else {  // the CTA's last, partial slot
            const uint32_t nvec = last_bytes >> 4;
#pragma unroll
            for (int r = 0; r < kVecs; ++r) {
                v[r] = make_uint4(0, 0, 0, 0);
                if (gtid + r * kHistCounters < nvec)
                    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                                 : "=r"(v[r].x), "=r"(v[r].y), "=r"(v[r].z), "=r"(v[r].w)
                                 : "r"(slot + 16 * kHistCounters * r));
            }
            counters_sync();  // (the last slot: nothing left to issue)
#pragma unroll
            for (int r = 0; r < kVecs; ++r)
                if (gtid + r * kHistCounters < nvec) hist_bump16(base_addr, col, inc, v[r]);
        }
        if (--flush_left == 0) {
            flush_left = kHistFlushStages;
            counters_sync();
            hist_flush(hist_smem + sub * (256u * 64u), tid, acc);
            counters_sync();
        }
        if (++q == kHistStages) {
            q = 0;
            ph ^= 1u;
        }
    }
    counters_sync();
    hist_flush(hist_smem + sub * (256u * 64u), tid, acc);
    if (acc[0]) atomicAdd(counts + tid, acc[0]);
    if (acc[1]) atomicAdd(counts + tid + 128, acc[1]);
}

cudaError_t launch_histogram(const uint8_t *d_msg, int64_t n, unsigned long long *d_counts,
                             cudaStream_t stream) {
    if (n <= 0) return cudaSuccess;
    smem_limit(reinterpret_cast<const void *>(histogram_u8_kernel), int(kHistSmem));
    // one CTA per SM; small inputs get fewer CTAs (>= 4 ring slots each)
    int64_t blocks = int64_t(sm_count());
    const int64_t want = (n + 4 * kHistStage - 1) / (4 * kHistStage);
    if (blocks > want) blocks = want < 1 ? 1 : want;
    histogram_u8_kernel<<<static_cast<unsigned>(blocks), kHistThreads, kHistSmem, stream>>>(
        d_msg, n, d_counts);
    ilans_note_launch();
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Quantize + tables: one CTA of 256 threads, thread i owns symbol i.
// ---------------------------------------------------------------------------
typedef unsigned __int128 u128;

struct I128 {  // signed 128-bit comparison key as (hi:int64, lo:uint64)
    long long hi;
    unsigned long long lo;
};
__device__ __forceinline__ I128 to_i128(u128 a_minus_b_pos, bool neg) {
    u128 v = neg ? (u128)0 - a_minus_b_pos : a_minus_b_pos;
    I128 r;
    r.hi = static_cast<long long>(static_cast<unsigned long long>(v >> 64));
    r.lo = static_cast<unsigned long long>(v);
    return r;
}
__device__ __forceinline__ bool gt(const I128 &a, const I128 &b) {
    return a.hi != b.hi ? a.hi > b.hi : a.lo > b.lo;
}
__device__ __forceinline__ bool eq(const I128 &a, const I128 &b) {
    return a.hi == b.hi && a.lo == b.lo;
}
// a - b for unsigned 128-bit a, b as a signed key
__device__ __forceinline__ I128 sub_key(u128 a, u128 b) {
    return a >= b ? to_i128(a - b, false) : to_i128(b - a, true);
}

template <typename T>
__device__ __forceinline__ T block_sum_256(T v, T *red) {
    const int tid = threadIdx.x;
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    __syncthreads();
    if ((tid & 31) == 0) red[tid >> 5] = v;
    __syncthreads();
    T s = 0;
#pragma unroll
    for (int w = 0; w < kMaxSym / 32; ++w) s += red[w];
    __syncthreads();
    return s;
}

__device__ __forceinline__ int block_max_256(int v, int *red) {
    const int tid = threadIdx.x;
    for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
    __syncthreads();
    if ((tid & 31) == 0) red[tid >> 5] = v;
    __syncthreads();
    int s = red[0];
#pragma unroll
    for (int w = 1; w < kMaxSym / 32; ++w) s = max(s, red[w]);
    __syncthreads();
    return s;
}

__device__ __forceinline__ uint32_t block_and_256(uint32_t v, uint32_t *red) {
    const int tid = threadIdx.x;
    v = __reduce_and_sync(0xffffffffu, v);
    __syncthreads();
    if ((tid & 31) == 0) red[tid >> 5] = v;
    __syncthreads();
    uint32_t s = red[0];
#pragma unroll
    for (int w = 1; w < kMaxSym / 32; ++w) s &= red[w];
    __syncthreads();
    return s;
}

// floor(c * m / T) for c*m < 2^81, result <= m <= 2^16: binary search on q.
__device__ __forceinline__ uint32_t floor_cm_over_t(unsigned long long c, uint32_t m,
                                                    u128 total) {
    const u128 cm = (u128)c * m;
    uint32_t lo = 0, hi = m;  // answer in [0, m]
    while (lo < hi) {
        const uint32_t mid = (lo + hi + 1) >> 1;
        if ((u128)mid * total <= cm) lo = mid; else hi = mid - 1;
    }
    return lo;
}

// Same for T < 2^47 (every realistic message): a double estimate is within
// one of the exact quotient; fix it with exact 64-bit products
// (q <= 2^16, T < 2^47: q*T < 2^63).
__device__ __forceinline__ uint32_t floor_cm_over_t64(unsigned long long cm,
                                                      unsigned long long total) {
    unsigned long long q = static_cast<unsigned long long>(
        static_cast<double>(cm) / static_cast<double>(total));
    while (q > 0 && q * total > cm) --q;
    while ((q + 1) * total <= cm) ++q;
    return static_cast<uint32_t>(q);
}

// Number of keys strictly greater than `my` among keys[0..256) (64-bit keys
// made unique by the symbol index in the low byte; absent = INT64_MIN).
__device__ __forceinline__ int rank_of(const long long *keys, long long my) {
    int rank = 0;
#pragma unroll 16
    for (int j = 0; j < kMaxSym; ++j) rank += keys[j] > my;
    return rank;
}

// Writes freq/cum/enc/dec/slot/packed for the table described by t->freq,
// t->cum (already in shared `freq`, `cum`). Runs on the whole CTA.
__device__ void fill_tables(TableDev *t, const uint32_t *freq, const uint32_t *cum,
                            const uint8_t *slot_in, int scale_bits, int *red) {
    const int tid = threadIdx.x;
    const uint32_t m = 1u << scale_bits;
    {
        const uint32_t f = freq[tid];
        t->freq[tid] = f;
        t->enc[tid] = EncSym::make(f, cum[tid], scale_bits);
        t->dec[tid] = make_uint2(f, cum[tid]);
        if (scale_bits == 14 || scale_bits == 15) {
            uint2 a;
            uint32_t z;
            EncFast12::make(f, cum[tid], scale_bits, &a, &z);
            t->encf[tid] = a;
            t->encz[tid] = z;
        } else {
            t->encf[tid] = EncFast::make(f, cum[tid], scale_bits);
            t->encz[tid] = 0u;
        }
        t->encq[tid] = EncQuad::make(f, cum[tid], scale_bits);
        t->encqx[tid] = EncQuadX::make(f, cum[tid], scale_bits);
    }
    const int quad_ok = freq[tid] <= (m >> 1) ? 1 : 0;
    const int quadx_ok = freq[tid] < m ? 1 : 0;
    // fast encoder records: sb <= 13 and no symbol above half the range
    const int fast_ok = (scale_bits <= kEncFastMaxBits || scale_bits == 14 || scale_bits == 15) &&
                        freq[tid] <= (m >> 1) ? 1 : 0;
    if (tid == 0) t->cum[kMaxSym] = cum[kMaxSym];
    t->cum[tid] = cum[tid];
    // slot -> symbol; consistent (packable) check for the sb <= 12 LUT.
    // Thread t owns the contiguous slots [t*per, (t+1)*per): one binary
    // search for the first, then a forward walk over cum.
    int ok = scale_bits <= kPackedMaxBits ? 1 : 0;
    int ok64 = scale_bits >= kPacked64MinBits && scale_bits <= kPacked64MaxBits ? 1 : 0;
    const uint32_t per = (m + kMaxSym - 1) / kMaxSym;
    const uint32_t j0 = tid * per, j1 = min(m, j0 + per);
    int s_cur = 0;
    if (!slot_in && j0 < j1) {  // largest s with cum[s] <= j0 (zero-f symbols skip)
        int lo = 0, hi = kMaxSym - 1;
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (cum[mid] <= j0) lo = mid; else hi = mid - 1;
        }
        s_cur = lo;
    }
    if (!slot_in && (per & 3u) == 0 && scale_bits <= kPackedMaxBits) {
        // common case (model from counts / frequencies, >= 4 slots per
        // thread): four slots per step, 16-byte packed and 4-byte symbol
        // stores (and the 64-bit entries for 13 <= sb <= 14, the fallback
        // when some f >= 4096 does not fit the 32-bit entry)
        const bool p64 = scale_bits >= kPacked64MinBits && scale_bits <= kPacked64MaxBits;
        for (uint32_t j = j0; j < j1; j += 4) {
            uint32_t e[4], sy = 0;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const uint32_t jj = j + q;
                while (s_cur < kMaxSym - 1 && cum[s_cur + 1] <= jj) ++s_cur;
                const uint32_t sym = static_cast<uint32_t>(s_cur);
                const uint32_t f = freq[sym];
                const uint32_t bias = jj - cum[sym];
                if (f < 1 || f > 4095 || bias >= 4096) ok = 0;
                e[q] = sym | (bias & 0xFFFu) << 8 | (f & 0xFFFu) << 20;
                sy |= sym << (8 * q);
                if (p64) t->packed64[jj] = make_uint2(sym | bias << 8, f);
            }
            *reinterpret_cast<uint4 *>(t->packed + j) = make_uint4(e[0], e[1], e[2], e[3]);
            *reinterpret_cast<uint32_t *>(t->slot_sym + j) = sy;
        }
    } else {
        for (uint32_t j = j0; j < j1; ++j) {
            uint32_t s;
            if (slot_in) {
                s = slot_in[j];
            } else {
                while (s_cur < kMaxSym - 1 && cum[s_cur + 1] <= j) ++s_cur;
                s = static_cast<uint32_t>(s_cur);
            }
            t->slot_sym[j] = static_cast<uint8_t>(s);
            if (scale_bits <= kPackedMaxBits) {
                const uint32_t f = freq[s];
                const uint32_t bias = j - cum[s];
                // f >= 4096 (e.g. a single-symbol sb=12 table) does not fit
                // 12 bits: such tables take the 64-bit or two-lookup path
                if (f < 1 || f > 4095 || bias >= 4096) ok = 0;
                t->packed[j] = s | (bias & 0xFFFu) << 8 | (f & 0xFFFu) << 20;
            }
            if (scale_bits >= kPacked64MinBits && scale_bits <= kPacked64MaxBits) {
                const uint32_t bias = j - cum[s];  // < 2^24 for every consistent table
                if (bias >= (1u << 24)) ok64 = 0;
                t->packed64[j] = make_uint2(s | bias << 8, freq[s]);
            }
        }
    }
    __syncthreads();
    // the four "every thread" conditions in one CTA-wide AND
    const uint32_t all = block_and_256(static_cast<uint32_t>((ok ? 1 : 0) | (fast_ok ? 2 : 0) |
                                                             (ok64 ? 4 : 0) | (quad_ok ? 8 : 0) |
                                                             (quadx_ok ? 16 : 0)),
                                       reinterpret_cast<uint32_t *>(red));
    const int all_ok = (all & 1u) != 0u;
    const int all_fast = (all & 2u) != 0u;
    const bool p64 = (all & 4u) != 0u;
    const int all_quad = (all & 8u) != 0u;
    const int all_quadx = (all & 16u) != 0u;
    if (tid == 0)
        t->flags = (all_ok ? kTabPacked : 0u) |
                   (all_fast ? (scale_bits >= 14 ? kTabEncFast12 : kTabEncFast) : 0u) |
                   (p64 ? kTabPacked64 : 0u) | (all_quad ? kTabEncQuad : 0u) |
                   (all_quadx ? kTabEncQuadX : 0u);
}

// fill_tables for a model quantized from counts (cum is freq's prefix sum,
// no slot map given) with the slot tables split over gridDim.x CTAs: every
// CTA quantized the same counts (the same result), CTA b writes the slots
// [b m / G, (b + 1) m / G) and CTA 0 the per-symbol records and the flags.
// The packed-entry checks are per symbol here (a slot's bias < f, so the
// 32-bit entry fits iff every f <= 4095), and the 64-bit entries are only
// written when the 32-bit ones do not fit (the decoder's fallback).
__device__ void fill_tables_split(TableDev *t, const uint32_t *freq, const uint32_t *cum,
                                  int scale_bits, int *red) {
    const int tid = threadIdx.x;
    const uint32_t m = 1u << scale_bits;
    const uint32_t f_me = freq[tid];
    const bool sb32 = scale_bits <= kPackedMaxBits;
    const bool sb64 = scale_bits >= kPacked64MinBits && scale_bits <= kPacked64MaxBits;
    const bool fast_sb = scale_bits <= kEncFastMaxBits || scale_bits == 14 || scale_bits == 15;
    const uint32_t all = block_and_256(
        static_cast<uint32_t>((f_me <= 4095u ? 1 : 0) | (fast_sb && f_me <= (m >> 1) ? 2 : 0) |
                              (f_me <= (m >> 1) ? 8 : 0) | (f_me < m ? 16 : 0)),
        reinterpret_cast<uint32_t *>(red));
    const bool fits32 = (all & 1u) != 0u;
    if (blockIdx.x == 0) {
        t->freq[tid] = f_me;
        t->enc[tid] = EncSym::make(f_me, cum[tid], scale_bits);
        t->dec[tid] = make_uint2(f_me, cum[tid]);
        if (scale_bits == 14 || scale_bits == 15) {
            uint2 a;
            uint32_t z;
            EncFast12::make(f_me, cum[tid], scale_bits, &a, &z);
            t->encf[tid] = a;
            t->encz[tid] = z;
        } else {
            t->encf[tid] = EncFast::make(f_me, cum[tid], scale_bits);
            t->encz[tid] = 0u;
        }
        t->encq[tid] = EncQuad::make(f_me, cum[tid], scale_bits);
        t->encqx[tid] = EncQuadX::make(f_me, cum[tid], scale_bits);
        if (tid == 0) t->cum[kMaxSym] = cum[kMaxSym];
        t->cum[tid] = cum[tid];
        if (tid == 0)
            t->flags = (sb32 && fits32 ? kTabPacked : 0u) |
                       ((all & 2u) ? (scale_bits >= 14 ? kTabEncFast12 : kTabEncFast) : 0u) |
                       (sb64 && !fits32 ? kTabPacked64 : 0u) |  // written only then (below)
                       ((all & 8u) ? kTabEncQuad : 0u) |
                       ((all & 16u) ? kTabEncQuadX : 0u);
    }
    const bool w64 = sb64 && !fits32;
    const uint32_t per = m / (kMaxSym * gridDim.x);  // a multiple of 4 (launch)
    const uint32_t j0 = (blockIdx.x * kMaxSym + tid) * per, j1 = j0 + per;
    int s_cur = 0;
    {  // largest s with cum[s] <= j0 (zero-f symbols skip)
        int lo = 0, hi = kMaxSym - 1;
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (cum[mid] <= j0) lo = mid; else hi = mid - 1;
        }
        s_cur = lo;
    }
    for (uint32_t j = j0; j < j1; j += 4) {
        uint32_t e[4], sy = 0;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const uint32_t jj = j + q;
            while (s_cur < kMaxSym - 1 && cum[s_cur + 1] <= jj) ++s_cur;
            const uint32_t sym = static_cast<uint32_t>(s_cur);
            const uint32_t f = freq[sym];
            const uint32_t bias = jj - cum[sym];
            e[q] = sym | (bias & 0xFFFu) << 8 | (f & 0xFFFu) << 20;
            sy |= sym << (8 * q);
            if (w64) t->packed64[jj] = make_uint2(sym | bias << 8, f);
        }
        if (sb32) *reinterpret_cast<uint4 *>(t->packed + j) = make_uint4(e[0], e[1], e[2], e[3]);
        *reinterpret_cast<uint32_t *>(t->slot_sym + j) = sy;
    }
}

// mode: counts != nullptr -> quantize(counts) first (alphabet = max+1).
//       otherwise freq_in/cum_in/slot_in as given (drop-in decode/encode).
__global__ void __launch_bounds__(kMaxSym)
build_table_kernel(const unsigned long long *__restrict__ counts, const uint32_t *freq_in,
                   int n_freq, const uint32_t *cum_in, const uint8_t *slot_in, int scale_bits,
                   TableDev *t) {
    __shared__ uint32_t freq[kMaxSym];
    __shared__ uint32_t cum[kMaxSym + 1];
    __shared__ I128 keys[kMaxSym];
    __shared__ long long keys64[kMaxSym];
    __shared__ unsigned long long red64[8];
    __shared__ int red[8];
    __shared__ int status_sh;
    const int tid = threadIdx.x;
    // the table's header / status words: written by CTA 0 only (a build
    // from counts runs several CTAs that reach the same result)
    const bool lead = blockIdx.x == 0;
    if (tid == 0) status_sh = ILANS_OK;
    if (lead && tid < 4) t->err_detail[tid] = 0;
    if (scale_bits < 1 || scale_bits > kMaxScaleBits) {
        if (lead && tid == 0) { t->status = ILANS_ERR_VALUE; t->err_detail[0] = 1; t->scale_bits = scale_bits; }
        return;
    }
    const uint32_t m = 1u << scale_bits;
    int n_sym;
    if (counts) {
        // ---- rans.quantize (rans.py:171-211), bit-exact ------------------
        unsigned long long c = counts[tid];
        // alphabet (highest present symbol + 1), present symbols and the
        // 128-bit total (as two 64-bit halves) in one CTA-wide reduction
        int alpha, present;
        u128 total;
        {
            __shared__ unsigned long long red_hi[8];
            __shared__ int red_p[8];
            int a = c ? tid + 1 : 0, p = c ? 1 : 0;
            unsigned long long lo = c & 0xFFFFFFFFull, hi = c >> 32;
            for (int o = 16; o > 0; o >>= 1) {
                a = max(a, __shfl_xor_sync(0xffffffffu, a, o));
                p += __shfl_xor_sync(0xffffffffu, p, o);
                lo += __shfl_xor_sync(0xffffffffu, lo, o);
                hi += __shfl_xor_sync(0xffffffffu, hi, o);
            }
            if ((tid & 31) == 0) {
                red[tid >> 5] = a;
                red_p[tid >> 5] = p;
                red64[tid >> 5] = lo;
                red_hi[tid >> 5] = hi;
            }
            __syncthreads();
            alpha = red[0];
            present = red_p[0];
            lo = red64[0];
            hi = red_hi[0];
#pragma unroll
            for (int w = 1; w < kMaxSym / 32; ++w) {
                alpha = max(alpha, red[w]);
                present += red_p[w];
                lo += red64[w];
                hi += red_hi[w];
            }
            __syncthreads();
            total = ((u128)hi << 32) + lo;
        }
        n_sym = alpha;
        if (alpha == 0) {  // empty message -> counts [1, 1] (cli.py:32-34)
            n_sym = 2;
            c = tid < 2 ? 1ull : 0ull;
            present = 2;
            total = 2;
        }
        if (static_cast<uint32_t>(present) > m) {
            if (lead && tid == 0) {
                t->status = ILANS_ERR_VALUE;
                t->err_detail[0] = 2;
                t->err_detail[1] = present;
                t->err_detail[2] = m;
                t->n_sym = n_sym;
                t->scale_bits = scale_bits;
            }
            return;
        }
        // T < 2^47 (all realistic inputs): every product and key fits 64 bits
        // and a key * 256 + (255 - i) orders exactly like (key, -i)
        const bool fast = total < ((u128)1 << 47);
        uint32_t f = 0;
        if (c) {
            f = fast ? floor_cm_over_t64(c * m, static_cast<unsigned long long>(total))
                     : floor_cm_over_t(c, m, total);
            if (f < 1) f = 1;
        }
        const long long diff =
            static_cast<long long>(m) - block_sum_256<long long>(static_cast<long long>(f), reinterpret_cast<long long *>(red64));
        const u128 cm = (u128)c * m;
        if (fast && diff > 0) {
            const long long key = static_cast<long long>(c * m) -
                                  static_cast<long long>(f * static_cast<unsigned long long>(total));
            keys64[tid] = c ? key * 256 + (255 - tid) : LLONG_MIN;
            __syncthreads();
            if (c && rank_of(keys64, keys64[tid]) < diff) f += 1;
            __syncthreads();
        } else if (fast && diff < 0) {
            const long long need = -diff;
            const long long P1 = block_sum_256<long long>((c && f > 1) ? 1 : 0,
                                                          reinterpret_cast<long long *>(red64));
            uint32_t R = 0;
            if (need >= P1) {  // more than one round: binary search R in [1, max f]
                uint32_t lo = 1, hi = static_cast<uint32_t>(block_max_256(c ? static_cast<int>(f) : 0, red));
                while (lo < hi) {
                    const uint32_t mid = (lo + hi + 1) >> 1;
                    const long long take = (c && f > 1) ? static_cast<long long>(min(mid, f - 1)) : 0;
                    const long long P = block_sum_256<long long>(take, reinterpret_cast<long long *>(red64));
                    if (P <= need) lo = mid; else hi = mid - 1;
                }
                R = lo;
            }
            const long long took = (c && f > 1) ? static_cast<long long>(min(R, f - 1)) : 0;
            const long long rem = need - block_sum_256<long long>(took, reinterpret_cast<long long *>(red64));
            const long long key = static_cast<long long>(f * static_cast<unsigned long long>(total)) -
                                  static_cast<long long>(c * m);
            const bool eligible = c && f >= R + 2;
            keys64[tid] = eligible ? key * 256 + (255 - tid) : LLONG_MIN;
            __syncthreads();
            uint32_t dec = static_cast<uint32_t>(took);
            if (eligible && rank_of(keys64, keys64[tid]) < rem) dec += 1;
            __syncthreads();
            f -= dec;
        } else if (diff > 0) {
            // picks are the top-`diff` present symbols by (c*m - f*T, -i):
            // with diff > 0 every key is < T and >= diff+1 keys are > 0, so
            // no symbol is picked twice.
            keys[tid] = sub_key(cm, (u128)f * total);
            freq[tid] = c ? 1u : 0u;  // presence flag
            __syncthreads();
            if (c) {
                const I128 my = keys[tid];
                int rank = 0;
                for (int j = 0; j < kMaxSym; ++j) {
                    if (!freq[j]) continue;
                    const I128 o = keys[j];
                    rank += (gt(o, my) || (eq(o, my) && j < tid)) ? 1 : 0;
                }
                if (rank < diff) f += 1;
            }
            __syncthreads();
        } else if (diff < 0) {
            // -1 rounds: round r takes every symbol with f >= r+2, ordered by
            // (f*T - c*m, -i); all keys of round r exceed all keys of round
            // r+1, so R full rounds take sum(min(R, f-1)) units.
            const long long need = -diff;
            uint32_t lo = 0, hi = m;  // largest R with P(R) <= need
            while (lo < hi) {
                const uint32_t mid = (lo + hi + 1) >> 1;
                const long long take = (c && f > 1) ? static_cast<long long>(min(mid, f - 1)) : 0;
                const long long P = block_sum_256<long long>(take, reinterpret_cast<long long *>(red64));
                if (P <= need) lo = mid; else hi = mid - 1;
            }
            const uint32_t R = lo;
            const long long took = (c && f > 1) ? static_cast<long long>(min(R, f - 1)) : 0;
            const long long rem = need - block_sum_256<long long>(took, reinterpret_cast<long long *>(red64));
            keys[tid] = sub_key((u128)f * total, cm);
            freq[tid] = (c && f >= R + 2) ? 1u : 0u;  // eligible in round R
            __syncthreads();
            uint32_t dec = static_cast<uint32_t>(took);
            if (freq[tid]) {
                const I128 my = keys[tid];
                int rank = 0;
                for (int j = 0; j < kMaxSym; ++j) {
                    if (!freq[j]) continue;
                    const I128 o = keys[j];
                    rank += (gt(o, my) || (eq(o, my) && j < tid)) ? 1 : 0;
                }
                if (rank < rem) dec += 1;
            }
            __syncthreads();
            f -= dec;
        }
        freq[tid] = tid < n_sym ? f : 0u;
        __syncthreads();
    } else {
        n_sym = n_freq;
        freq[tid] = (tid < n_freq && freq_in) ? freq_in[tid] : 0u;
        __syncthreads();
        if (!cum_in) {  // model from frequencies alone: must sum to 2^sb (rans.py:110-112)
            const long long sum = block_sum_256<long long>(static_cast<long long>(freq[tid]),
                                                           reinterpret_cast<long long *>(red64));
            if (sum != static_cast<long long>(m)) {
                if (lead && tid == 0) {
                    t->status = ILANS_ERR_VALUE;
                    t->err_detail[0] = 3;
                    t->n_sym = n_sym;
                    t->scale_bits = scale_bits;
                }
                return;
            }
        }
    }
    // cum: given (drop-in calls) or exclusive prefix of freq
    if (cum_in) {
        cum[tid] = tid <= n_sym ? cum_in[tid] : 0u;
        if (tid == 0) cum[kMaxSym] = n_sym >= kMaxSym ? cum_in[kMaxSym] : 0u;
        __syncthreads();
    } else {
        // inclusive warp scan then warp offsets
        uint32_t v = freq[tid];
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t u = __shfl_up_sync(0xffffffffu, v, o);
            if ((tid & 31) >= o) v += u;
        }
        __shared__ uint32_t wsum[8];
        if ((tid & 31) == 31) wsum[tid >> 5] = v;
        __syncthreads();
        uint32_t off = 0;
        for (int w = 0; w < (tid >> 5); ++w) off += wsum[w];
        cum[tid + 1] = v + off;
        if (tid == 0) cum[0] = 0;
        __syncthreads();
    }
    if (lead && tid == 0) {
        t->scale_bits = scale_bits;
        t->n_sym = n_sym;
        t->status = status_sh;
    }
    if (gridDim.x > 1)  // model from counts: the slot tables split over the CTAs
        fill_tables_split(t, freq, cum, scale_bits, red);
    else
        fill_tables(t, freq, cum, slot_in, scale_bits, red);
}

}  // namespace ilans
