// mux.cu -- the stream multiplexer on the B200 (reference pkg/src/ilans/mux.py).
//
// The reference merges independently coded streams by *running* one decoder
// per stream along the schedule and teeing every byte each one reads into the
// output (mux.mux, mux.py:283-313; mux_with_flush, mux.py:329-433). The bytes
// a decoder reads at a step are fixed by the encoder: the digits spilled
// while pushing symbol i are exactly the ones refilled after popping it, and
// a raw value is its nbytes. So the merge is data-parallel here:
//   1. stable radix sort of the schedule by stream id: perm[i] = the step at
//      which the i-th symbol in stream-major order (== message order within
//      a stream) is decoded;
//   2. segment starts (stream change, or epoch change with epoch = step / F)
//      and an inclusive scan for segment ids (mux._epoch_runs, mux.py:316-326);
//   3. one thread per segment codes it backwards from a fresh state
//      (RansStreamCodec.encode_segment, mux.py:93-101), writing the digits in
//      read order and every symbol's byte count;
//   4. the counts in schedule order, exclusive scan: each step's offset in
//      the muxed payload;
//   5. one thread per symbol copies [inline segment state] + its digits.
// MuxBudget.max_buffered (mux.py:404-405) is a scan over epochs. Merging
// pre-encoded buffers (mux.mux) gets the per-symbol counts from one replay
// thread per stream instead of step 3. Decoding (demux_decode, mux.py:436-475)
// stays a sequential walk: each step's read size depends on the state of the
// stream it decodes, which depends on every earlier read; one device thread
// walks it.
#include <cub/cub.cuh>

#include <vector>

#include "common.cuh"
#include "kernels.cuh"
#include "status.cuh"

namespace ilans {
namespace {

constexpr int kMuxThreads = 256;
constexpr int64_t kMuxMaxSteps = (int64_t(1) << 30) - 1;  // 4 B scratch / symbol in u32 offsets

unsigned mux_blocks(int64_t n) {
    const int64_t b = (n + kMuxThreads - 1) / kMuxThreads;
    return static_cast<unsigned>(b < 1 ? 1 : (b > (1 << 20) ? (1 << 20) : b));
}

__device__ __forceinline__ uint32_t load_le(const uint8_t *p, int nb) {
    uint32_t v = 0;
    for (int b = 0; b < nb; ++b) v |= uint32_t(p[b]) << (8 * b);
    return v;
}

__device__ __forceinline__ void store_le(uint8_t *p, uint32_t v, int nb) {
    for (int b = 0; b < nb; ++b) p[b] = static_cast<uint8_t>(v >> (8 * b));
}

__device__ __forceinline__ int64_t epoch_of(int32_t step, int64_t F) {
    return F > 0 ? int64_t(step) / F : 0;
}

#define MUX_FOR(i, n)                                                                   \
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < (n);           \
         i += int64_t(gridDim.x) * blockDim.x)

__global__ void iota_kernel(int32_t *v, int64_t n) {
    MUX_FOR(i, n) v[i] = static_cast<int32_t>(i);
}

// flag[i] = 1 where stream-major symbol i starts a segment
__global__ void seg_flags_kernel(const int32_t *keys, const int32_t *perm, int64_t T, int64_t F,
                                 uint32_t *flag) {
    MUX_FOR(i, T) {
        flag[i] = (i == 0 || keys[i] != keys[i - 1] ||
                   epoch_of(perm[i], F) != epoch_of(perm[i - 1], F))
                      ? 1u
                      : 0u;
    }
}

struct SegTab {
    int32_t *start;   // [S + 1] first stream-major symbol of each segment
    int32_t *stream;  // [S]
    int64_t *epoch;   // [S]
    uint8_t *first;   // [S] the stream's first segment (its state is the header)
    uint32_t *state;  // [S] final encoder state
    uint64_t *bytes;  // [S] bytes the segment contributes (inline state + digits)
};

__global__ void seg_table_kernel(const int32_t *keys, const int32_t *perm, const uint32_t *segid,
                                 int64_t T, int64_t F, SegTab sg, int32_t *nseg) {
    MUX_FOR(i, T) {
        const uint32_t s = segid[i] - 1u;
        if (i == 0 || segid[i] != segid[i - 1]) {
            sg.start[s] = static_cast<int32_t>(i);
            sg.stream[s] = keys[i];
            sg.epoch[s] = epoch_of(perm[i], F);
            sg.first[s] = (i == 0 || keys[i] != keys[i - 1]) ? 1 : 0;
        }
        if (i == T - 1) {
            sg.start[s + 1] = static_cast<int32_t>(T);
            *nseg = static_cast<int32_t>(s + 1);
        }
    }
}

// One thread per segment. rANS: walk the segment backwards from x = L,
// spilling digit_bits-wide digits while x >= f * (limit >> sb)
// (rans.encode_symbol_renorm, rans.py:266-290), digits written backwards
// from the segment's end so that memory order is read order; raw: the
// values' little-endian bytes. scratch holds 4 bytes per symbol (a rANS
// symbol spills at most 3 byte digits or one 16-bit digit).
__global__ void mux_encode_segments_kernel(const ilans_mux_stream *__restrict__ streams,
                                           const uint32_t *__restrict__ freq,
                                           const uint32_t *__restrict__ cum,
                                           const uint32_t *__restrict__ sym, SegTab sg,
                                           const int32_t *nseg, uint8_t *scratch, uint8_t *dcnt,
                                           uint64_t *srcpos, unsigned long long *bad_key) {
    const int64_t S = *nseg;
    MUX_FOR(g, S) {
        const int32_t a = sg.start[g], b = sg.start[g + 1];
        const ilans_mux_stream p = streams[sg.stream[g]];
        const int nb = p.nbytes;
        if (p.kind == ILANS_MUX_RAW) {
            for (int32_t i = a; i < b; ++i) {
                store_le(scratch + 4 * int64_t(i), sym[i], nb);
                dcnt[i] = static_cast<uint8_t>(nb);
                srcpos[i] = 4 * uint64_t(i);
            }
            sg.bytes[g] = uint64_t(nb) * uint64_t(b - a);
            continue;
        }
        const uint32_t *fr = freq + p.freq_off;
        const uint32_t *cu = cum + p.cum_off;
        const uint64_t limit = uint64_t(p.lower_bound) << p.digit_bits;
        const uint64_t unit = limit >> p.scale_bits;
        const uint32_t mask = (1u << p.digit_bits) - 1u;
        uint32_t x = p.lower_bound;
        uint32_t wp = 4u * uint32_t(b);
        bool bad = false;
        for (int32_t i = b - 1; i >= a; --i) {
            const uint32_t s = sym[i];
            const uint32_t f = fr[s];
            if (f == 0) {  // the first failure the reference's backward walk meets
                atomicMin(bad_key, (static_cast<unsigned long long>(g) << 32) | uint32_t(i));
                bad = true;
                break;
            }
            const uint64_t thr = uint64_t(f) * unit;
            const uint32_t end = wp;
            while (uint64_t(x) >= thr) {
                wp -= nb;
                store_le(scratch + wp, x & mask, nb);
                x >>= p.digit_bits;
            }
            dcnt[i] = static_cast<uint8_t>(end - wp);
            srcpos[i] = wp;
            x = ((x / f) << p.scale_bits) + cu[s] + x % f;
        }
        if (bad) continue;
        sg.state[g] = x;
        uint64_t bytes = 4u * uint32_t(b) - wp;
        if (!sg.first[g]) {  // later segments carry their state inline (mux.py:373-374)
            dcnt[a] |= 0x80;
            bytes += 4;
        }
        sg.bytes[g] = bytes;
    }
}

// Decode lookup per slot of every rANS stream's table, at the slot array's
// offsets: lo = symbol | (slot - cum[symbol]) << 8, hi = f[symbol], so a pop
// is one load: x' = hi * (x >> sb) + (lo >> 8) (rans.pop_symbol).
__global__ void mux_lut_kernel(const ilans_mux_stream *__restrict__ streams, int K,
                               const uint32_t *__restrict__ freq, const uint32_t *__restrict__ cum,
                               const uint8_t *__restrict__ slot, uint2 *lut) {
    for (int j = blockIdx.x; j < K; j += gridDim.x) {
        const ilans_mux_stream p = streams[j];
        if (p.kind != ILANS_MUX_RANS) continue;
        for (uint32_t i = threadIdx.x; i < (1u << p.scale_bits); i += blockDim.x) {
            const uint32_t s = slot[p.slot_off + i];
            lut[p.slot_off + i] = make_uint2(s | (i - cum[p.cum_off + s]) << 8, freq[p.freq_off + s]);
        }
    }
}

// Merge of pre-encoded buffers (mux.mux): one thread per stream replays its
// decoder (mux._RansStreamDecoder, mux.py:107-128) over its own payload to
// get each symbol's read count. err[j]: 0 ok, 1 header too short, 2 header
// state outside [L, limit), 3 payload exhausted, 4 payload not consumed.
__global__ void mux_replay_streams_kernel(const ilans_mux_stream *__restrict__ streams, int K,
                                          const uint2 *__restrict__ lut, const uint8_t *hdr,
                                          const uint64_t *hdr_off, const uint8_t *pay,
                                          const uint64_t *pay_off, const int64_t *sym_off,
                                          uint8_t *dcnt, uint64_t *srcpos, int32_t *err,
                                          uint32_t *err_val) {
    MUX_FOR(j, K) {
        const ilans_mux_stream p = streams[j];
        const int64_t i0 = sym_off[j], n = sym_off[j + 1] - i0;
        const uint64_t base = pay_off[j], len = pay_off[j + 1] - base;
        const int nb = p.nbytes;
        err[j] = 0;
        if (p.kind == ILANS_MUX_RAW) {
            for (int64_t k = 0; k < n; ++k) {
                dcnt[i0 + k] = static_cast<uint8_t>(nb);
                srcpos[i0 + k] = base + uint64_t(k) * nb;
            }
            const uint64_t need = uint64_t(n) * nb;
            err[j] = need > len ? 3 : (need < len ? 4 : 0);
            continue;
        }
        if (hdr_off[j + 1] - hdr_off[j] < 4) {
            err[j] = 1;
            continue;
        }
        uint32_t x = load_le(hdr + hdr_off[j], 4);
        const uint32_t L = p.lower_bound;
        const uint64_t limit = uint64_t(L) << p.digit_bits;
        if (x < L || uint64_t(x) >= limit) {
            err[j] = 2;
            err_val[j] = x;
            continue;
        }
        const uint2 *lt = lut + p.slot_off;
        const uint32_t mmask = (1u << p.scale_bits) - 1u;
        uint64_t cur = 0;
        int32_t e = 0;
        for (int64_t k = 0; k < n && !e; ++k) {
            const uint2 en = lt[x & mmask];
            x = en.y * (x >> p.scale_bits) + (en.x >> 8);
            const uint64_t p0 = cur;
            while (x < L) {
                if (cur + nb > len) {
                    e = 3;
                    break;
                }
                x = (x << p.digit_bits) | load_le(pay + base + cur, nb);
                cur += nb;
            }
            dcnt[i0 + k] = static_cast<uint8_t>(cur - p0);
            srcpos[i0 + k] = base + p0;
        }
        err[j] = e ? e : (cur != len ? 4 : 0);
    }
}

// counts in schedule order (+ a trailing 0 so the exclusive scan's last
// entry is the total)
__global__ void sched_counts_kernel(const int32_t *perm, const uint8_t *dcnt, int64_t T,
                                    uint64_t *cnt) {
    MUX_FOR(i, T) {
        const uint32_t c = dcnt[i];
        cnt[perm[i]] = (c & 0x7Fu) + ((c & 0x80u) ? 4u : 0u);
        if (i == 0) cnt[T] = 0;
    }
}

__global__ void scatter_kernel(const int32_t *perm, const uint8_t *dcnt, const uint64_t *srcpos,
                               const uint8_t *src, const uint32_t *segid,
                               const uint32_t *seg_state, const uint64_t *dst, int64_t T,
                               uint8_t *out) {
    MUX_FOR(i, T) {
        uint64_t d = dst[perm[i]];
        const uint32_t c = dcnt[i];
        if (c & 0x80u) {
            store_le(out + d, seg_state[segid[i] - 1u], 4);
            d += 4;
        }
        const uint8_t *q = src + srcpos[i];
        for (uint32_t k = 0; k < (c & 0x7Fu); ++k) out[d + k] = q[k];
    }
}

// per-epoch flushed bytes, per-stream totals and header states
__global__ void seg_totals_kernel(const int32_t *nseg, SegTab sg, unsigned long long *epoch_bytes,
                                  unsigned long long *stream_bytes, uint32_t *stream_state) {
    const int64_t S = *nseg;
    MUX_FOR(g, S) {
        const unsigned long long b = sg.bytes[g];
        atomicAdd(epoch_bytes + sg.epoch[g], b);
        atomicAdd(stream_bytes + sg.stream[g], b);
        if (sg.first[g]) stream_state[sg.stream[g]] = sg.state[g];
    }
}

// max over epochs of (bytes flushed by epoch e) - (bytes the replay consumed
// before epoch e), as mux.py:404-405 measures at every flush point
__global__ void budget_kernel(const unsigned long long *flushed_incl, const uint64_t *dst,
                              int64_t E, int64_t F, int64_t T, unsigned long long *maxb) {
    MUX_FOR(e, E) {
        const int64_t t = F > 0 ? (e * F < T ? e * F : T) : 0;
        atomicMax(maxb, flushed_incl[e] - dst[t]);
    }
}

struct DemuxStatus {
    int32_t code;    // 0 ok, ILANS_ERR_TRUNCATED, ILANS_ERR_FORMAT
    int32_t stream;
    int64_t step;    // -1: while loading the stream headers
    uint32_t value;  // rejected state
    uint64_t pos;    // payload bytes read
};

// Per-stream record for the walk, one 32-bit word per field so the loop
// does no field extraction: lut offset, L, slot mask, sb, digit_bits,
// nbytes, digit / value mask, flags = raw | pure << 1 | rmax << 8.
// pure: the refill count after a pop is a function of the popped state
// alone (x' R^(k-1) < L decides refill k exactly when R^(k-1) divides L:
// every power-of-two L, i.e. WORD16, BYTE8 and most custom variants);
// rmax: most refills one pop can need (x' = 1).
struct __align__(16) WalkDesc {
    uint32_t lut_off, L, mask, sb, bits, nb, dmask, flags;
};
constexpr uint32_t kWalkRaw = 1u, kWalkPure = 2u;

__device__ __forceinline__ bool state_ok(uint32_t x, const WalkDesc &d) {
    return x >= d.L && (uint64_t(x) >> d.bits) < uint64_t(d.L);
}

// 4 payload bytes at any byte offset (two aligned words + a funnel shift;
// the device payload is 8-byte padded and 4-byte aligned)
__device__ __forceinline__ uint32_t load4(const uint32_t *__restrict__ w, uint32_t pos) {
    const uint32_t q = pos >> 2;
    return __funnelshift_r(__ldg(w + q), __ldg(w + q + 1), (pos & 3u) * 8u);
}

// refills after a pop to x' >= 1 on a pure stream: #{k < rmax : x' < L >> (bits k)}
__device__ __forceinline__ uint32_t pure_refills(uint32_t x, const WalkDesc &d) {
    uint32_t r = 0;
    const uint32_t rmax = d.flags >> 8;
    for (uint32_t k = 0; k < rmax; ++k) r += x < (d.L >> (d.bits * k)) ? 1u : 0u;
    return r;
}

// Per-step word for the walk, built in parallel from the stable sort of
// the schedule: stream id | reload << 16 | min(t - prev, 63) << 17, where
// prev is the stream's previous step (none: 63) and reload marks a stream
// whose previous step lies in an earlier epoch (its state is inline here,
// mux.py:459-465).
__global__ void walk_prep_kernel(const int32_t *__restrict__ keys,
                                 const int32_t *__restrict__ perm, int64_t T, int32_t F,
                                 uint32_t *__restrict__ word) {
    MUX_FOR(i, T) {
        const int32_t t = perm[i];
        const bool has_prev = i > 0 && keys[i - 1] == keys[i];
        const int32_t prev = has_prev ? perm[i - 1] : -1;
        const uint32_t dist = has_prev ? min(t - prev, 63) : 63u;
        const uint32_t reload = has_prev && (prev / F != t / F) ? 1u : 0u;
        word[t] = uint32_t(keys[i]) | reload << 16 | dist << 17;
    }
}

// Walk staging rings in shared memory, refilled by cp.async half a ring
// ahead of the walker: the per-step words (2 x 2048) and the payload
// (2 x 4 KB). The device arrays are padded to whole halves plus one.
constexpr uint32_t kWordHalf = 2048;                // words per half
constexpr uint32_t kPayHalf = 4096;                 // payload bytes per half
constexpr size_t kWalkRingBytes = 2 * kWordHalf * 4 + 2 * kPayHalf;

// 4 payload bytes at absolute byte offset b from the payload ring
__device__ __forceinline__ uint32_t ring4(const uint32_t *pr, uint32_t b) {
    const uint32_t q = b >> 2;
    return __funnelshift_r(pr[q & (2 * kPayHalf / 4 - 1)], pr[(q + 1) & (2 * kPayHalf / 4 - 1)],
                           (b & 3u) * 8u);
}

// one half (kWordHalf words or kPayHalf bytes) of a ring, 16 bytes a lane
__device__ __forceinline__ void ring_fill(void *dst, const void *src, uint32_t bytes, int lane) {
    for (uint32_t o = 16u * lane; o < bytes; o += 512u)
        cp_async16(static_cast<uint8_t *>(dst) + o, static_cast<const uint8_t *>(src) + o, 16u);
}

// demux_decode (mux.py:436-475): headers first (stream order), then the
// schedule.
//
// Each step's read offset is the sum of the read sizes of all earlier
// steps, and a step's read size depends on its stream's state -- but only
// on that stream's. So a run of consecutive steps that touch DISTINCT
// streams decodes together: warp 0 takes up to 32 steps and cuts the
// window at the first step whose stream already occurs in it (t - prev <=
// lane), at the first inline state reload after lane 0, and at an impure
// stream; every lane pops its stream's state, its refill count follows from
// the popped state, three ballots give the prefix sum of the read sizes
// (< 8 bytes a step), and every lane shifts in its own digits from the
// window's 256 payload bytes, staged in registers when the window opens.
// Round-robin schedules over K >= 32 streams run 32 steps per window. A
// window that starts at an impure stream takes one step with the
// reference's digit loop. Records, states and lookups sit in shared memory
// when they fit (SMEM).
template <bool SMEM>
__global__ void __launch_bounds__(256) demux_kernel(
    const WalkDesc *__restrict__ gdesc, int K, const uint2 *__restrict__ glut, int64_t n_lut,
    const uint8_t *hdr, const uint64_t *hdr_off, const uint32_t *__restrict__ pay, uint32_t plen,
    const uint32_t *__restrict__ word, int32_t T, uint32_t *gstate, uint32_t *__restrict__ out,
    DemuxStatus *st) {
    extern __shared__ __align__(16) uint8_t dsm[];
    uint8_t *ring_smem = dsm;  // kWalkRingBytes, then the SMEM tables
    const WalkDesc *desc = gdesc;
    const uint2 *lut = glut;
    uint32_t *state = gstate;
    if (SMEM) {
        WalkDesc *sd = reinterpret_cast<WalkDesc *>(dsm + kWalkRingBytes);
        uint2 *sl = reinterpret_cast<uint2 *>(sd + K);
        for (int64_t i = threadIdx.x; i < n_lut; i += blockDim.x) sl[i] = glut[i];
        for (int j = threadIdx.x; j < K; j += blockDim.x) sd[j] = gdesc[j];
        lut = sl;
        desc = sd;
        state = reinterpret_cast<uint32_t *>(sl + n_lut);
        __syncthreads();
    }
    if (threadIdx.x >= 32) return;
    const int lane = threadIdx.x;
    const uint32_t lt = lanemask_lt();
    if (lane == 0) {
        st->code = 0;
        st->stream = -1;
        st->step = -1;
    }
    // stream headers, in stream order (the first failing stream reports)
    for (int j0 = 0; j0 < K; j0 += 32) {
        const int j = j0 + lane;
        int err = 0;
        uint32_t x = 0;
        if (j < K) {
            const WalkDesc d = desc[j];
            if (!(d.flags & kWalkRaw)) {
                if (hdr_off[j + 1] - hdr_off[j] < 4) {
                    err = ILANS_ERR_TRUNCATED;
                } else {
                    x = load_le(hdr + hdr_off[j], 4);
                    if (!state_ok(x, d)) err = ILANS_ERR_FORMAT;
                    state[j] = x;
                }
            }
        }
        const uint32_t eb = __ballot_sync(0xffffffffu, err != 0);
        if (eb) {
            if (lane == __ffs(eb) - 1) {
                st->code = err;
                st->stream = j;
                st->value = x;
            }
            return;
        }
    }
    __syncwarp();

    uint32_t pos = 0;
    int32_t t = 0;
    // rings: words [wbase, wbase + 2 halves), payload bytes [pbase, pbase +
    // 2 halves); *_ready: end of what has landed
    uint32_t *wring = reinterpret_cast<uint32_t *>(ring_smem);
    uint32_t *pring = wring + 2 * kWordHalf;
    uint32_t wbase = 0, wissued = 2 * kWordHalf, wready = 0;
    uint32_t pbase = 0, pissued = 2 * kPayHalf, pready = 0;
    ring_fill(wring, word, 2 * kWordHalf * 4, lane);
    ring_fill(pring, pay, 2 * kPayHalf, lane);
    cp_async_commit();
    while (t < T) {
        // refill the half behind the walker, wait only when the window
        // needs what is still in flight
        if (uint32_t(t) >= wbase + kWordHalf) {
            ring_fill(wring + (wissued / kWordHalf & 1u) * kWordHalf, word + wissued,
                      kWordHalf * 4, lane);
            cp_async_commit();
            wbase += kWordHalf;
            wissued += kWordHalf;
        }
        if (pos >= pbase + kPayHalf) {
            ring_fill(reinterpret_cast<uint8_t *>(pring) + (pissued / kPayHalf & 1u) * kPayHalf,
                      reinterpret_cast<const uint8_t *>(pay) + pissued, kPayHalf, lane);
            cp_async_commit();
            pbase += kPayHalf;
            pissued += kPayHalf;
        }
        if (uint32_t(t) + 32 > wready || pos + 264 > pready) {
            cp_async_wait<0>();
            __syncwarp();
            wready = wissued;
            pready = pissued;
        }
        const int32_t step = t + lane;
        const bool valid = step < T;
        const uint32_t cur = wring[uint32_t(step) & (2 * kWordHalf - 1)];
        const int32_t sid = valid ? int32_t(cur & 0xFFFFu) : 0;
        const WalkDesc d = desc[sid];
        const bool raw = d.flags & kWalkRaw;
        const bool reload = valid && !raw && ((cur >> 16) & 1u);
        const bool dup = (cur >> 17) <= uint32_t(lane);
        const bool impure = !raw && !(d.flags & kWalkPure);
        const bool impure0 = __shfl_sync(0xffffffffu, impure, 0);  // lane 0 goes alone
        const bool stop = !valid || dup || (lane > 0 && (reload || impure || impure0));
        const uint32_t sbal = __ballot_sync(0xffffffffu, stop);
        const int W = sbal ? __ffs(sbal) - 1 : 32;  // >= 1: lane 0 is valid and first
        const bool on = lane < W;
        // lanes past the window may name a stream a window lane updates
        // below: they do not read its state
        uint32_t x = (raw || !on) ? 0u : state[sid];
        uint32_t extra = 0;
        int err = 0;
        if (on && reload) {  // lane 0 only: the state inline at the window start
            if (pos + 4 > plen) {
                err = ILANS_ERR_TRUNCATED;
            } else {
                x = ring4(pring, pos);
                extra = 4;
                if (!state_ok(x, d)) err = ILANS_ERR_FORMAT;
            }
        }
        uint32_t sym = 0, bytes = 0;
        if (on && !err) {
            if (raw) {
                bytes = d.nb;
            } else {
                const uint2 en = lut[d.lut_off + (x & d.mask)];
                x = en.y * (x >> d.sb) + (en.x >> 8);
                sym = en.x & 0xFFu;
                if (!impure0) bytes = pure_refills(x, d) * d.nb;
            }
        }
        if (impure0 && lane == 0 && !err) {
            // lane 0 alone, the digits decide the count: the reference's loop
            uint32_t p = pos + extra;
            while (x < d.L) {
                if (p + d.nb > plen) {
                    err = ILANS_ERR_TRUNCATED;
                    break;
                }
                x = (x << d.bits) | (load4(pay, p) & d.dmask);
                p += d.nb;
            }
            bytes = p - pos - extra;
        }
        // offsets: prefix sum of the window's read sizes (< 8 bytes a step:
        // a 4-byte reload + 3 byte digits at most), three ballots
        const uint32_t mine = on ? extra + bytes : 0u;
        const uint32_t b0 = __ballot_sync(0xffffffffu, mine & 1u);
        const uint32_t b1 = __ballot_sync(0xffffffffu, mine & 2u);
        const uint32_t b2 = __ballot_sync(0xffffffffu, mine & 4u);
        const uint32_t at = pos + __popc(b0 & lt) + 2u * __popc(b1 & lt) + 4u * __popc(b2 & lt);
        const uint32_t wtot = __popc(b0) + 2u * __popc(b1) + 4u * __popc(b2);
        if (on && !err && at + mine > plen) err = ILANS_ERR_TRUNCATED;
        const uint32_t ebal = __ballot_sync(0xffffffffu, err != 0);
        if (ebal) {
            const int f = __ffs(ebal) - 1;
            if (lane == f) {
                st->code = err;
                st->stream = sid;
                st->step = step;
                st->value = x;
                st->pos = at;
            }
            return;
        }
        if (on) {
            // this step's 4 bytes after its reload (impure lane 0 is done)
            const uint32_t w = ring4(pring, at + extra);
            if (raw) {
                out[step] = w & d.dmask;
            } else {
                if (!impure0 && bytes) {
                    if (d.nb == 2) {
                        x = (x << 16) | (w & 0xFFFFu);
                    } else {  // byte digits, read in order
                        for (uint32_t k = 0; k < bytes; ++k) x = (x << 8) | ((w >> (8 * k)) & 0xFFu);
                    }
                }
                state[sid] = x;
                out[step] = sym;
            }
        }
        pos += wtot;
        t += W;
        __syncwarp();
    }
    cp_async_wait<0>();
    if (lane == 0) st->pos = pos;
}

// stream-major order of the decoded values: dst[i] = src[perm[i]]
__global__ void gather_kernel(const int32_t *__restrict__ perm, const uint32_t *__restrict__ src,
                              int64_t T, uint32_t *__restrict__ dst) {
    MUX_FOR(i, T) dst[i] = src[perm[i]];
}

// cudaMallocAsync'd scratch, released on the call's stream
struct AsyncBufs {
    cudaStream_t s;
    std::vector<void *> ptrs;
    explicit AsyncBufs(cudaStream_t st) : s(st) {}
    ~AsyncBufs() {
        for (void *p : ptrs) cudaFreeAsync(p, s);
    }
    template <typename T>
    cudaError_t alloc(T **p, size_t n) {
        void *v = nullptr;
        cudaError_t e = cudaMallocAsync(&v, (n ? n : 1) * sizeof(T) + 16, s);
        if (e == cudaSuccess) ptrs.push_back(v);
        *p = static_cast<T *>(v);
        return e;
    }
    template <typename T>
    cudaError_t upload(T **p, const T *h, size_t n) {
        cudaError_t e = alloc(p, n);
        if (e == cudaSuccess && n) e = cudaMemcpyAsync(*p, h, n * sizeof(T), cudaMemcpyHostToDevice, s);
        return e;
    }
};

int check_streams(const ilans_mux_stream *streams, int K, int64_t n_freq, int64_t n_cum,
                  int64_t n_slot, bool need_slot, ilans_status *st) {
    for (int j = 0; j < K; ++j) {
        const ilans_mux_stream &p = streams[j];
        if (p.kind == ILANS_MUX_RAW) {
            if (p.digit_bits < 1 || p.digit_bits > 32 || p.nbytes != (p.digit_bits + 7) / 8)
                return st_fail(st, ILANS_ERR_VALUE, "stream %d: width_bits must be in [1, 32]", j);
            continue;
        }
        if (p.kind != ILANS_MUX_RANS)
            return st_fail(st, ILANS_ERR_VALUE, "stream %d: unknown coder kind %d", j, p.kind);
        if ((p.digit_bits != 8 && p.digit_bits != 16) || p.nbytes != p.digit_bits / 8)
            return st_fail(st, ILANS_ERR_VALUE, "mux streams need byte-multiple digit widths");
        if (p.scale_bits < 1 || p.scale_bits > kMaxScaleBits || p.lower_bound < 1 ||
            (uint64_t(p.lower_bound) << p.digit_bits) > (uint64_t(1) << 32) ||
            (p.lower_bound & ((1u << p.scale_bits) - 1u)) != 0)
            return st_fail(st, ILANS_ERR_VALUE, "stream %d: lower_bound is not a multiple of "
                           "the table total", j);
        if (p.n_sym < 1 || p.n_sym > kMaxSym || p.freq_off < 0 || p.freq_off + p.n_sym > n_freq ||
            p.cum_off < 0 || p.cum_off + p.n_sym + 1 > n_cum)
            return st_fail(st, ILANS_ERR_VALUE, "stream %d: table out of range", j);
        if (need_slot && (p.slot_off < 0 || p.slot_off + (int64_t(1) << p.scale_bits) > n_slot))
            return st_fail(st, ILANS_ERR_VALUE, "stream %d: slot table out of range", j);
    }
    return ILANS_OK;
}

// per-stream symbol offsets from the schedule (also range-checks it)
int schedule_offsets(const int32_t *schedule, int64_t T, int K, std::vector<int64_t> &off,
                     ilans_status *st) {
    off.assign(size_t(K) + 1, 0);
    for (int64_t t = 0; t < T; ++t) {
        const int32_t sid = schedule[t];
        if (sid < 0 || sid >= K)
            return st_fail(st, ILANS_ERR_SCHEDULE, "schedule references unknown stream %d", sid);
        ++off[size_t(sid) + 1];
    }
    for (int j = 0; j < K; ++j) off[size_t(j) + 1] += off[size_t(j)];
    return ILANS_OK;
}

int key_bits(int K) {
    int b = 1;
    while ((1 << b) < K) ++b;
    return b;
}

// stable sort of the schedule by stream: keys[i] = stream, perm[i] = step
int sort_schedule(AsyncBufs &m, const int32_t *d_sched, int64_t T, int K, int32_t **keys,
                  int32_t **perm, ilans_status *st) {
    cudaStream_t s = m.s;
    int32_t *iota = nullptr;
    CK(m.alloc(&iota, size_t(T)));
    CK(m.alloc(keys, size_t(T)));
    CK(m.alloc(perm, size_t(T)));
    iota_kernel<<<mux_blocks(T), kMuxThreads, 0, s>>>(iota, T);
    ilans_note_launch();
    size_t tmp = 0;
    // stream ids are validated non-negative: sort them as unsigned keys
    const uint32_t *kin = reinterpret_cast<const uint32_t *>(d_sched);
    uint32_t *kout = reinterpret_cast<uint32_t *>(*keys);
    CK(cub::DeviceRadixSort::SortPairs(nullptr, tmp, kin, kout, iota, *perm, int(T), 0,
                                       key_bits(K), s));
    uint8_t *d_tmp = nullptr;
    CK(m.alloc(&d_tmp, tmp));
    CK(cub::DeviceRadixSort::SortPairs(d_tmp, tmp, kin, kout, iota, *perm, int(T), 0,
                                       key_bits(K), s));
    return ILANS_OK;
}

// steps 4 + 5: offsets in schedule order and the copy; returns the total
int place(AsyncBufs &m, const int32_t *perm, const uint8_t *dcnt, const uint64_t *srcpos,
          const uint8_t *src, const uint32_t *segid, const uint32_t *seg_state, int64_t T,
          uint64_t **dst, uint8_t *d_out, ilans_status *st) {
    cudaStream_t s = m.s;
    uint64_t *cnt = nullptr;
    CK(m.alloc(&cnt, size_t(T) + 1));
    CK(m.alloc(dst, size_t(T) + 1));
    sched_counts_kernel<<<mux_blocks(T), kMuxThreads, 0, s>>>(perm, dcnt, T, cnt);
    ilans_note_launch();
    size_t tmp = 0;
    CK(cub::DeviceScan::ExclusiveSum(nullptr, tmp, cnt, *dst, int(T + 1), s));
    uint8_t *d_tmp = nullptr;
    CK(m.alloc(&d_tmp, tmp));
    CK(cub::DeviceScan::ExclusiveSum(d_tmp, tmp, cnt, *dst, int(T + 1), s));
    scatter_kernel<<<mux_blocks(T), kMuxThreads, 0, s>>>(perm, dcnt, srcpos, src, segid,
                                                          seg_state, *dst, T, d_out);
    ilans_note_launch();
    return ILANS_OK;
}

}  // namespace
}  // namespace ilans

using namespace ilans;

extern "C" int ilans_mux_encode(const ilans_mux_stream *streams, int32_t n_streams,
                                const uint32_t *freq, int64_t n_freq, const uint32_t *cum,
                                int64_t n_cum, const uint32_t *symbols, const int32_t *schedule,
                                int64_t n_steps, int64_t flush_interval, uint8_t *payload_out,
                                int64_t payload_cap, int64_t *payload_len, uint32_t *stream_state,
                                uint64_t *stream_bytes, int64_t *segment_count,
                                uint64_t *max_buffered, ilans_status *st) {
    st_clear(st);
    const int K = n_streams;
    const int64_t T = n_steps, F = flush_interval;
    if (K < 0 || K > 0xFFFF) return st_fail(st, ILANS_ERR_VALUE, "stream count must be <= 65535");
    if (T < 0 || T > kMuxMaxSteps) return st_fail(st, ILANS_ERR_VALUE, "too many schedule steps");
    if (F < 0) return st_fail(st, ILANS_ERR_VALUE, "flush_interval must be >= 1");
    if (int rc = check_streams(streams, K, n_freq, n_cum, 0, false, st)) return rc;
    std::vector<int64_t> off;
    if (int rc = schedule_offsets(schedule, T, K, off, st)) return rc;
    for (int j = 0; j < K; ++j) {  // symbol ranges (the caller validated the messages)
        const ilans_mux_stream &p = streams[j];
        const uint64_t lim = p.kind == ILANS_MUX_RAW
                                 ? (uint64_t(1) << p.digit_bits)
                                 : uint64_t(p.n_sym);
        for (int64_t i = off[j]; i < off[j + 1]; ++i)
            if (symbols[i] >= lim)
                return st_fail(st, ILANS_ERR_VALUE, "stream %d: value %u out of range", j,
                               symbols[i]);
    }
    for (int j = 0; j < K; ++j) {
        stream_state[j] = streams[j].kind == ILANS_MUX_RAW ? 0u : streams[j].lower_bound;
        stream_bytes[j] = 0;
    }
    *payload_len = 0;
    *segment_count = 0;
    *max_buffered = 0;
    if (T == 0) return ILANS_OK;

    cudaStream_t s = nullptr;
    std::unique_lock<std::mutex> lock;
    if (int rc = ilans_host_session(st, &s, &lock)) return rc;
    AsyncBufs m(s);
    ilans_mux_stream *d_streams = nullptr;
    uint32_t *d_freq = nullptr, *d_cum = nullptr, *d_sym = nullptr;
    int32_t *d_sched = nullptr;
    CK(m.upload(&d_streams, streams, size_t(K)));
    CK(m.upload(&d_freq, freq, size_t(n_freq)));
    CK(m.upload(&d_cum, cum, size_t(n_cum)));
    CK(m.upload(&d_sym, symbols, size_t(T)));
    CK(m.upload(&d_sched, schedule, size_t(T)));

    int32_t *keys = nullptr, *perm = nullptr;
    if (int rc = sort_schedule(m, d_sched, T, K, &keys, &perm, st)) return rc;

    // segments
    uint32_t *flag = nullptr, *segid = nullptr;
    CK(m.alloc(&flag, size_t(T)));
    CK(m.alloc(&segid, size_t(T)));
    seg_flags_kernel<<<mux_blocks(T), kMuxThreads, 0, s>>>(keys, perm, T, F, flag);
    ilans_note_launch();
    size_t tmp = 0;
    CK(cub::DeviceScan::InclusiveSum(nullptr, tmp, flag, segid, int(T), s));
    uint8_t *d_tmp = nullptr;
    CK(m.alloc(&d_tmp, tmp));
    CK(cub::DeviceScan::InclusiveSum(d_tmp, tmp, flag, segid, int(T), s));
    SegTab sg{};
    int32_t *nseg = nullptr;
    CK(m.alloc(&sg.start, size_t(T) + 1));
    CK(m.alloc(&sg.stream, size_t(T)));
    CK(m.alloc(&sg.epoch, size_t(T)));
    CK(m.alloc(&sg.first, size_t(T)));
    CK(m.alloc(&sg.state, size_t(T)));
    CK(m.alloc(&sg.bytes, size_t(T)));
    CK(m.alloc(&nseg, 1));
    seg_table_kernel<<<mux_blocks(T), kMuxThreads, 0, s>>>(keys, perm, segid, T, F, sg, nseg);
    ilans_note_launch();

    // encode the segments
    uint8_t *scratch = nullptr, *dcnt = nullptr;
    uint64_t *srcpos = nullptr;
    unsigned long long *bad = nullptr;
    CK(m.alloc(&scratch, size_t(T) * 4));
    CK(m.alloc(&dcnt, size_t(T)));
    CK(m.alloc(&srcpos, size_t(T)));
    CK(m.alloc(&bad, 1));
    CK(cudaMemsetAsync(bad, 0xFF, sizeof(unsigned long long), s));
    mux_encode_segments_kernel<<<mux_blocks(T), kMuxThreads, 0, s>>>(
        d_streams, d_freq, d_cum, d_sym, sg, nseg, scratch, dcnt, srcpos, bad);
    ilans_note_launch();
    unsigned long long h_bad = 0;
    int32_t h_nseg = 0;
    CK(cudaMemcpyAsync(&h_bad, bad, sizeof(h_bad), cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(&h_nseg, nseg, sizeof(h_nseg), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (h_bad != ~0ull) {
        const int64_t i = int64_t(h_bad & 0xFFFFFFFFull);
        int j = 0;
        while (off[j + 1] <= i) ++j;
        st->stream = j;
        st->index = i - off[j];
        st->symbol = int32_t(symbols[i]);
        return st_fail(st, ILANS_ERR_UNENCODABLE, "symbol %u has frequency 0", symbols[i]);
    }

    // merge
    uint8_t *d_out = nullptr;
    CK(m.alloc(&d_out, size_t(T) * 8));
    uint64_t *dst = nullptr;
    if (int rc = place(m, perm, dcnt, srcpos, scratch, segid, sg.state, T, &dst, d_out, st))
        return rc;

    // budget, stream totals, headers
    const int64_t E = F > 0 ? (T - 1) / F + 1 : 1;
    unsigned long long *eb = nullptr, *ebi = nullptr, *maxb = nullptr, *sbytes = nullptr;
    uint32_t *sstate = nullptr;
    CK(m.alloc(&eb, size_t(E)));
    CK(m.alloc(&ebi, size_t(E)));
    CK(m.alloc(&maxb, 1));
    CK(m.alloc(&sbytes, size_t(K)));
    CK(m.upload(&sstate, stream_state, size_t(K)));
    CK(cudaMemsetAsync(eb, 0, size_t(E) * 8, s));
    CK(cudaMemsetAsync(maxb, 0, 8, s));
    CK(cudaMemsetAsync(sbytes, 0, size_t(K) * 8, s));
    seg_totals_kernel<<<mux_blocks(h_nseg), kMuxThreads, 0, s>>>(nseg, sg, eb, sbytes, sstate);
    ilans_note_launch();
    tmp = 0;
    CK(cub::DeviceScan::InclusiveSum(nullptr, tmp, eb, ebi, int(E), s));
    uint8_t *d_tmp2 = nullptr;
    CK(m.alloc(&d_tmp2, tmp));
    CK(cub::DeviceScan::InclusiveSum(d_tmp2, tmp, eb, ebi, int(E), s));
    budget_kernel<<<mux_blocks(E), kMuxThreads, 0, s>>>(ebi, dst, E, F, T, maxb);
    ilans_note_launch();

    uint64_t total = 0;
    unsigned long long h_maxb = 0;
    CK(cudaMemcpyAsync(&total, dst + T, 8, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(&h_maxb, maxb, 8, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(stream_bytes, sbytes, size_t(K) * 8, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(stream_state, sstate, size_t(K) * 4, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (int64_t(total) > payload_cap)
        return st_fail(st, ILANS_ERR_VALUE, "payload buffer too small (%lld bytes needed)",
                       (long long)total);
    CK(cudaMemcpyAsync(payload_out, d_out, size_t(total), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    *payload_len = int64_t(total);
    *segment_count = h_nseg;
    *max_buffered = h_maxb;
    return ILANS_OK;
}

extern "C" int ilans_mux_merge(const ilans_mux_stream *streams, int32_t n_streams,
                               const uint32_t *freq, int64_t n_freq, const uint32_t *cum,
                               int64_t n_cum, const uint8_t *slot, int64_t n_slot,
                               const uint8_t *headers, const uint64_t *header_off,
                               const uint8_t *payloads, const uint64_t *payload_off,
                               const int64_t *symbol_counts, const int32_t *schedule,
                               int64_t n_steps, uint8_t *out, ilans_status *st) {
    st_clear(st);
    const int K = n_streams;
    const int64_t T = n_steps;
    if (K < 0 || K > 0xFFFF) return st_fail(st, ILANS_ERR_VALUE, "stream count must be <= 65535");
    if (T < 0 || T > kMuxMaxSteps) return st_fail(st, ILANS_ERR_VALUE, "too many schedule steps");
    if (int rc = check_streams(streams, K, n_freq, n_cum, n_slot, true, st)) return rc;
    std::vector<int64_t> off;
    if (int rc = schedule_offsets(schedule, T, K, off, st)) return rc;
    for (int j = 0; j < K; ++j)
        if (off[j + 1] - off[j] != symbol_counts[j])
            return st_fail(st, ILANS_ERR_SCHEDULE,
                           "schedule has %lld steps for stream %d, which holds %lld symbols",
                           (long long)(off[j + 1] - off[j]), j, (long long)symbol_counts[j]);
    const uint64_t hbytes = header_off[K], pbytes = payload_off[K];
    if (K == 0) return ILANS_OK;

    cudaStream_t s = nullptr;
    std::unique_lock<std::mutex> lock;
    if (int rc = ilans_host_session(st, &s, &lock)) return rc;
    AsyncBufs m(s);
    ilans_mux_stream *d_streams = nullptr;
    uint32_t *d_freq = nullptr, *d_cum = nullptr, *d_err_val = nullptr;
    uint8_t *d_slot = nullptr, *d_hdr = nullptr, *d_pay = nullptr, *dcnt = nullptr;
    uint64_t *d_hoff = nullptr, *d_poff = nullptr, *srcpos = nullptr;
    int64_t *d_off = nullptr;
    int32_t *d_sched = nullptr, *d_err = nullptr;
    CK(m.upload(&d_streams, streams, size_t(K)));
    CK(m.upload(&d_freq, freq, size_t(n_freq)));
    CK(m.upload(&d_cum, cum, size_t(n_cum)));
    CK(m.upload(&d_slot, slot, size_t(n_slot)));
    CK(m.upload(&d_hdr, headers, size_t(hbytes)));
    CK(m.upload(&d_hoff, header_off, size_t(K) + 1));
    CK(m.upload(&d_pay, payloads, size_t(pbytes)));
    CK(m.upload(&d_poff, payload_off, size_t(K) + 1));
    CK(m.upload(&d_off, off.data(), size_t(K) + 1));
    CK(m.upload(&d_sched, schedule, size_t(T)));
    CK(m.alloc(&dcnt, size_t(T)));
    CK(m.alloc(&srcpos, size_t(T)));
    CK(m.alloc(&d_err, size_t(K)));
    CK(m.alloc(&d_err_val, size_t(K)));
    uint2 *d_lut = nullptr;
    CK(m.alloc(&d_lut, size_t(n_slot)));
    mux_lut_kernel<<<K < 1024 ? K : 1024, 256, 0, s>>>(d_streams, K, d_freq, d_cum, d_slot, d_lut);
    ilans_note_launch();
    mux_replay_streams_kernel<<<mux_blocks(K), kMuxThreads, 0, s>>>(
        d_streams, K, d_lut, d_hdr, d_hoff, d_pay, d_poff, d_off, dcnt, srcpos, d_err, d_err_val);
    ilans_note_launch();
    std::vector<int32_t> err(static_cast<size_t>(K));
    std::vector<uint32_t> err_val(static_cast<size_t>(K));
    CK(cudaMemcpyAsync(err.data(), d_err, size_t(K) * 4, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(err_val.data(), d_err_val, size_t(K) * 4, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    // the reference loads every header first (stream order), then replays
    // (any exhausted stream raises), then checks leftovers (stream order)
    for (int j = 0; j < K; ++j) {
        if (err[j] == 1 || err[j] == 2) {
            st->stream = j;
            if (err[j] == 1)
                return st_fail(st, ILANS_ERR_TRUNCATED, "byte stream exhausted mid-decode");
            return st_fail(st, ILANS_ERR_FORMAT, "stream state %u outside the coder interval",
                           err_val[j]);
        }
    }
    for (int j = 0; j < K; ++j)
        if (err[j] == 3) {
            st->stream = j;
            return st_fail(st, ILANS_ERR_TRUNCATED, "byte stream exhausted mid-decode");
        }
    for (int j = 0; j < K; ++j)
        if (err[j] == 4) {
            st->stream = j;
            return st_fail(st, ILANS_ERR_SCHEDULE, "stream %d payload not fully consumed by schedule",
                           j);
        }
    if (T == 0) return ILANS_OK;  // every payload empty

    int32_t *keys = nullptr, *perm = nullptr;
    if (int rc = sort_schedule(m, d_sched, T, K, &keys, &perm, st)) return rc;
    uint8_t *d_out = nullptr;
    CK(m.alloc(&d_out, size_t(pbytes)));
    uint64_t *dst = nullptr;
    if (int rc = place(m, perm, dcnt, srcpos, d_pay, nullptr, nullptr, T, &dst, d_out, st))
        return rc;
    CK(cudaMemcpyAsync(out, d_out, size_t(pbytes), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    return ILANS_OK;
}

extern "C" int ilans_mux_demux(const ilans_mux_stream *streams, int32_t n_streams,
                               const uint32_t *freq, int64_t n_freq, const uint32_t *cum,
                               int64_t n_cum, const uint8_t *slot, int64_t n_slot,
                               const uint8_t *headers, const uint64_t *header_off,
                               const uint8_t *payload, int64_t payload_len,
                               const int32_t *schedule, int64_t n_steps, int64_t flush_interval,
                               uint32_t *symbols_out, uint32_t *symbols_by_stream,
                               int64_t *unread, ilans_status *st) {
    st_clear(st);
    const int K = n_streams;
    const int64_t T = n_steps;
    if (K < 0 || K > 0xFFFF) return st_fail(st, ILANS_ERR_VALUE, "stream count must be <= 65535");
    if (T < 0 || T > kMuxMaxSteps) return st_fail(st, ILANS_ERR_VALUE, "too many schedule steps");
    // u32 ring cursors run up to 2 halves + 264 bytes past the payload end
    if (payload_len < 0 || payload_len > int64_t(0xFFFFFFFFu) - 4 * int64_t(kPayHalf) ||
        flush_interval < 0)
        return st_fail(st, ILANS_ERR_VALUE, "bad arguments (payload must be < 4 GiB - 16 KiB)");
    if (int rc = check_streams(streams, K, n_freq, n_cum, n_slot, true, st)) return rc;
    std::vector<int64_t> off;
    if (int rc = schedule_offsets(schedule, T, K, off, st)) return rc;
    *unread = payload_len;
    if (K == 0) return ILANS_OK;

    cudaStream_t s = nullptr;
    std::unique_lock<std::mutex> lock;
    if (int rc = ilans_host_session(st, &s, &lock)) return rc;
    AsyncBufs m(s);
    ilans_mux_stream *d_streams = nullptr;
    uint32_t *d_freq = nullptr, *d_cum = nullptr, *d_state = nullptr, *d_out = nullptr;
    uint8_t *d_slot = nullptr, *d_hdr = nullptr;
    uint64_t *d_hoff = nullptr;
    int32_t *d_sched = nullptr;
    uint2 *d_lut = nullptr;
    WalkDesc *d_desc = nullptr;
    DemuxStatus *d_st = nullptr;
    std::vector<WalkDesc> desc(static_cast<size_t>(K));
    for (int j = 0; j < K; ++j) {
        const ilans_mux_stream &p = streams[j];
        WalkDesc &d = desc[j];
        const bool raw = p.kind == ILANS_MUX_RAW;
        d.nb = uint32_t(p.nbytes);
        d.dmask = p.nbytes >= 4 ? ~0u : (1u << (8 * p.nbytes)) - 1u;
        d.lut_off = raw ? 0u : uint32_t(p.slot_off);
        d.L = raw ? 0u : p.lower_bound;
        d.sb = raw ? 0u : uint32_t(p.scale_bits);
        d.mask = raw ? 0u : (1u << p.scale_bits) - 1u;
        d.bits = raw ? 0u : uint32_t(p.digit_bits);
        uint32_t rmax = 0;
        bool pure = true;
        if (!raw) {  // refills from x' = 1, and whether R^(k-1) | L for each
            uint64_t v = 1;
            while (v < p.lower_bound) {
                if (p.lower_bound % v) pure = false;
                v <<= p.digit_bits;
                ++rmax;
            }
        }
        d.flags = (raw ? kWalkRaw : 0u) | (raw || pure ? kWalkPure : 0u) | rmax << 8;
    }
    CK(m.upload(&d_streams, streams, size_t(K)));
    CK(m.upload(&d_desc, desc.data(), size_t(K)));
    CK(m.upload(&d_freq, freq, size_t(n_freq)));
    CK(m.upload(&d_cum, cum, size_t(n_cum)));
    CK(m.upload(&d_slot, slot, size_t(n_slot)));
    CK(m.alloc(&d_lut, size_t(n_slot)));
    CK(m.upload(&d_hdr, headers, size_t(header_off[K])));
    CK(m.upload(&d_hoff, header_off, size_t(K) + 1));
    // payload as 4-byte words + 8 bytes of padding for the look-ahead loads
    uint32_t *d_payw = nullptr;
    // whole ring halves past the end (the rings copy halves; reads stop at plen)
    const size_t pwords = ((size_t(payload_len) + kPayHalf - 1) / kPayHalf + 2) * (kPayHalf / 4);
    CK(m.alloc(&d_payw, pwords));
    CK(cudaMemsetAsync(d_payw, 0, pwords * 4, s));
    if (payload_len)
        CK(cudaMemcpyAsync(d_payw, payload, size_t(payload_len), cudaMemcpyHostToDevice, s));
    CK(m.alloc(&d_sched, size_t(T) + 128));  // + entries read ahead
    CK(cudaMemsetAsync(d_sched + T, 0, 128 * 4, s));
    if (T) CK(cudaMemcpyAsync(d_sched, schedule, size_t(T) * 4, cudaMemcpyHostToDevice, s));
    CK(m.alloc(&d_state, size_t(K)));
    CK(m.alloc(&d_out, size_t(T)));
    CK(m.alloc(&d_st, 1));
    mux_lut_kernel<<<K < 1024 ? K : 1024, 256, 0, s>>>(d_streams, K, d_freq, d_cum, d_slot, d_lut);
    ilans_note_launch();
    // per-step words from the stable sort of the schedule
    uint32_t *d_word = nullptr;
    const size_t nwords = ((size_t(T) + kWordHalf - 1) / kWordHalf + 2) * kWordHalf;
    CK(m.alloc(&d_word, nwords));
    CK(cudaMemsetAsync(d_word, 0, nwords * 4, s));
    const int32_t F32 = (flush_interval <= 0 || flush_interval >= T) ? INT32_MAX
                                                                      : int32_t(flush_interval);
    int32_t *perm = nullptr;
    if (T > 0) {
        int32_t *keys = nullptr;
        if (int rc = sort_schedule(m, d_sched, T, K, &keys, &perm, st)) return rc;
        walk_prep_kernel<<<mux_blocks(T), kMuxThreads, 0, s>>>(keys, perm, T, F32, d_word);
        ilans_note_launch();
    }
    const size_t smem = kWalkRingBytes + size_t(n_slot) * sizeof(uint2) +
                        size_t(K) * (sizeof(WalkDesc) + 4);
    if (smem <= size_t(200) * 1024) {
        CK(cudaFuncSetAttribute(demux_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                int(smem)));
        demux_kernel<true><<<1, 256, smem, s>>>(d_desc, K, d_lut, n_slot, d_hdr, d_hoff, d_payw,
                                                uint32_t(payload_len), d_word, int32_t(T),
                                                d_state, d_out, d_st);
    } else {
        demux_kernel<false><<<1, 32, kWalkRingBytes, s>>>(
            d_desc, K, d_lut, n_slot, d_hdr, d_hoff, d_payw, uint32_t(payload_len), d_word,
            int32_t(T), d_state, d_out, d_st);
    }
    ilans_note_launch();
    DemuxStatus h{};
    CK(cudaMemcpyAsync(&h, d_st, sizeof(h), cudaMemcpyDeviceToHost, s));
    if (symbols_out && T)
        CK(cudaMemcpyAsync(symbols_out, d_out, size_t(T) * 4, cudaMemcpyDeviceToHost, s));
    if (symbols_by_stream && T) {  // stream-major: out[perm[i]]
        uint32_t *d_sm = nullptr;
        CK(m.alloc(&d_sm, size_t(T)));
        gather_kernel<<<mux_blocks(T), kMuxThreads, 0, s>>>(perm, d_out, T, d_sm);
        ilans_note_launch();
        CK(cudaMemcpyAsync(symbols_by_stream, d_sm, size_t(T) * 4, cudaMemcpyDeviceToHost, s));
    }
    CK(cudaStreamSynchronize(s));
    if (h.code) {
        st->stream = h.stream;
        st->index = h.step;
        st->consumed = int64_t(h.pos);
        if (h.code == ILANS_ERR_FORMAT)
            return st_fail(st, ILANS_ERR_FORMAT, "stream state %u outside the coder interval",
                           h.value);
        return st_fail(st, ILANS_ERR_TRUNCATED, "byte stream exhausted mid-decode");
    }
    *unread = payload_len - int64_t(h.pos);
    return ILANS_OK;
}
