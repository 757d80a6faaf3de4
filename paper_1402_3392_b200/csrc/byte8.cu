// byte8.cu -- byte-renormalised (BYTE8: 8-bit digits, L = 2^23) interleaved
// rANS on sm_100a (reference scalar path interleave.py:155-179,
// rans.encode_symbol_renorm / decode_symbol_renorm rans.py:266-314).
//
// The reference codes byte8 symbol by symbol, each lane moving 0-3 digits
// per symbol, depth first: while walking backwards the encoder pushes lane
// i's digits (low byte first) right after lane i+1's, and the decoder reads
// lane i's refill digits right after lane i-1's. So inside a group the
// digits of lane l sit at read-order offset sum_{j<l} k_j -- an exclusive
// prefix sum of per-lane counts instead of the word16 popc. With counts in
// {0..3} the prefix is two ballots: pre = popc(b0 & lt) + 2 popc(b1 & lt).
//
// The counts are pure functions of the state for every stream the encoder
// can produce: spills k = #{j in 0..2 : x >> 8j >= f << (31-sb)} and, after
// a pop to x' >= 1, refills r = [x' < 2^23] + [x' < 2^15] + [x' < 2^7]
// (L = 2^23 is a multiple of 256^2). Only x' = 0 -- reachable from states
// below L handed in directly, never from a container -- makes the count
// depend on the bytes read; such a group is resolved lane by lane, with the
// reference's limit of 5 refills (FormatError "corrupt stream").
#include "common.cuh"
#include "kernels.cuh"

namespace ilans {

constexpr uint32_t kLow8 = 1u << 23;  // BYTE8.lower_bound (rans.py:86)
constexpr int kRefillLimit8 = 5;      // (24 + 7) // 8 + 2 (rans.py:305)

__device__ __forceinline__ uint32_t refills_for(uint32_t x) {  // x >= 1
    return (x < (1u << 23)) + (x < (1u << 15)) + (x < (1u << 7));
}

// Traced single-stream decode (interleave.decode_interleaved_steps for byte8):
// one warp, N <= 32 lanes, payload read straight from global memory; the
// untraced calls run the staged kernels below.
__global__ void __launch_bounds__(256)
decode_u8_warp_kernel(const uint8_t *__restrict__ payload, const uint64_t *__restrict__ offsets,
                      const uint32_t *__restrict__ states, int64_t n, int64_t chunk_len,
                      int64_t n_chunks, int n_lanes, const TableDev *__restrict__ tab,
                      uint8_t *__restrict__ out, uint64_t *__restrict__ consumed,
                      DStatus *__restrict__ status, DecodeTrace trace) {
    __shared__ uint2 dec[kMaxSym];
    for (int i = threadIdx.x; i < kMaxSym; i += blockDim.x) dec[i] = tab->dec[i];
    __syncthreads();
    const int sb = static_cast<int>(tab->scale_bits);
    const uint32_t mask = (1u << sb) - 1u;
    const uint8_t *slot_sym = tab->slot_sym;
    const int lane = threadIdx.x & 31;
    const uint32_t lt = lanemask_lt();
    const int64_t warps_total = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
    for (int64_t k = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
         k < n_chunks; k += warps_total) {
        const int64_t cbase = k * chunk_len;
        const int64_t len = (n - cbase) < chunk_len ? (n - cbase) : chunk_len;
        const uint8_t *pay = payload + offsets[k];
        const uint64_t plen = offsets[k + 1] - offsets[k];
        uint32_t x = lane < n_lanes ? states[k * n_lanes + lane] : 0u;
        uint64_t pos = 0;
        int err = 0;  // 0 ok, ILANS_ERR_TRUNCATED, ILANS_ERR_FORMAT
        uint32_t most = 0;  // most refills for one symbol (RenormStats.max_decode_digits)
        int64_t base = 0;
        for (; base < len; base += n_lanes) {
            const int64_t left = len - base;
            const int active = left < n_lanes ? static_cast<int>(left) : n_lanes;
            const bool on = lane < active;
            uint32_t s = 0;
            if (on) {
                const uint32_t slot = x & mask;
                s = slot_sym[slot];
                const uint2 d = dec[s];
                x = d.x * (x >> sb) + slot - d.y;
                out[cbase + base + lane] = static_cast<uint8_t>(s);
            }
            if (__ballot_sync(0xffffffffu, on && x == 0u)) {
                // byte-dependent refills: resolve lane by lane (corrupt input)
                for (int l = 0; l < active && !err; ++l) {
                    if (lane == l) {
                        int r = 0;
                        while (x < kLow8) {
                            if (pos >= plen) { err = ILANS_ERR_TRUNCATED; break; }
                            x = (x << 8) | pay[pos++];
                            if (++r > kRefillLimit8) { err = ILANS_ERR_FORMAT; break; }
                        }
                        most = max(most, static_cast<uint32_t>(r));
                    }
                    pos = __shfl_sync(0xffffffffu, pos, l);
                    err = __shfl_sync(0xffffffffu, err, l);
                }
            } else {
                const uint32_t r = on ? refills_for(x) : 0u;
                const uint32_t b0 = __ballot_sync(0xffffffffu, r & 1u);
                const uint32_t b1 = __ballot_sync(0xffffffffu, r & 2u);
                const uint32_t tot = __popc(b0) + 2u * __popc(b1);
                if (pos + tot > plen) {
                    err = ILANS_ERR_TRUNCATED;
                } else {
                    const uint64_t p = pos + __popc(b0 & lt) + 2u * __popc(b1 & lt);
                    if (r) {  // the r digits at once: 4 bytes from two aligned
                        // words of the (4-aligned, padded) payload, byte-reversed
                        const uint64_t ab = static_cast<uint64_t>(pay - payload) + p;
                        const uint32_t *w = reinterpret_cast<const uint32_t *>(payload) + (ab >> 2);
                        const uint32_t v = __funnelshift_r(__ldg(w), __ldg(w + 1),
                                                           static_cast<uint32_t>(ab & 3u) * 8u);
                        x = (x << (8u * r)) | (__byte_perm(v, 0u, 0x0123u) >> (32u - 8u * r));
                    }
                    pos += tot;
                    most = max(most, r);
                }
            }
            if (err) break;
            if (trace.states) {
                const int64_t gi = base / n_lanes;
                if (lane < n_lanes) trace.states[gi * n_lanes + lane] = x;
                if (lane == 0) trace.pos[gi] = pos;
            }
        }
        most = __reduce_max_sync(0xffffffffu, most);
        if (lane == 0) {
            atomicMax(&status->max_digits, most);
            if (err == ILANS_ERR_TRUNCATED)
                atomicMin(&status->trunc_stream, static_cast<unsigned long long>(k));
            if (err == ILANS_ERR_FORMAT) status->value_error = ILANS_ERR_FORMAT;
            if (consumed) consumed[k] = pos;
            if (trace.groups) trace.groups[k] = (base < len ? base : len + n_lanes - 1) / n_lanes;
        }
    }
}

// ---------------------------------------------------------------------------
// Staged byte8 coders (N <= 32): the word16 kernels' structure with byte
// digits. One CTA per SM holds all of the SM's streams (<= 28 warps, one
// warp per chunk); the payload (decode) / message (encode) stream through a
// per-warp 2 KB shared ring filled by cp.async, the slot LUT and records sit
// in shared memory, the decoded bytes leave through a per-warp 512-byte
// staging buffer as 16-byte stores, and the spilled digits drain from a
// per-warp 2 KB ring as aligned 16-byte blocks. Digit order and counts are
// the two-ballot exclusive prefix above.
// ---------------------------------------------------------------------------
constexpr int kSeg8 = 512;                 // ring segment (bytes)
constexpr int kRing8 = 4 * kSeg8;          // per-warp ring
constexpr int kObuf8 = 512;                // decoded-byte staging per warp
constexpr int kMaxWarps8 = 28;
constexpr int64_t kRingMaxChunk8 = int64_t(1) << 29;  // 32-bit chunk cursors (3 len < 2^31)
// bank-private copies of the 16-byte fast encode records (a quarter-warp per
// wavefront: lane l reads copy l % 8, conflict-free whatever the symbols)
constexpr int kRec8Copies = 8;

constexpr int kRing8Alloc = kRing8 + 16;   // decode ring + a copy of its first 16 bytes

// Segment seg of the payload into ring slot seg % 4; slot 0's first 16 bytes
// are also copied past the ring's end, so a 2-byte read at the last ring
// byte needs no wrap.
__device__ __forceinline__ void issue_seg8(uint32_t ring_sa, const uint8_t *gbase, uint64_t avail,
                                           uint64_t seg, int lane) {
    const uint64_t b0 = seg * kSeg8 + lane * 16;
    uint32_t bytes = 0;
    if (avail > b0) bytes = (avail - b0) >= 16 ? 16u : static_cast<uint32_t>(avail - b0);
    const uint8_t *src = bytes ? gbase + b0 : gbase;
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(
                     ring_sa + static_cast<uint32_t>(seg & 3u) * kSeg8 + lane * 16),
                 "l"(src), "r"(bytes)
                 : "memory");
    if ((seg & 3u) == 0 && lane == 0)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(ring_sa + kRing8),
                     "l"(src), "r"(bytes)
                     : "memory");
}

__device__ __forceinline__ uint32_t lds32(uint32_t a) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ uint32_t lds8(uint32_t a) {
    uint16_t v;
    asm volatile("ld.shared.u8 %0, [%1];" : "=h"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ void sts8(uint32_t a, uint32_t v) {
    asm volatile("st.shared.u8 [%0], %1;" ::"r"(a), "h"(static_cast<uint16_t>(v)) : "memory");
}

// PACKED: the 32-bit slot entries sym | bias << 8 | f << 20 (every f < 4096;
// table flag kTabPacked), else the two lookups slot -> symbol -> {f, cum}.
template <bool PACKED>
__device__ __noinline__ void
decode_u8_ring_body(const uint8_t *__restrict__ payload, const uint64_t *__restrict__ offsets,
                    const uint32_t *__restrict__ states, int64_t n, int64_t chunk_len,
                    int64_t n_chunks, int n_lanes, const TableDev *__restrict__ tab,
                    uint8_t *__restrict__ out, uint64_t *__restrict__ consumed,
                    DStatus *__restrict__ status, uint8_t *sm8) {
    const int nw = blockDim.x >> 5;
    const int sb = static_cast<int>(tab->scale_bits);
    const uint32_t m = 1u << sb, mask = m - 1u;
    uint8_t *lut = sm8 + nw * (kRing8Alloc + kObuf8);
    if (PACKED) {
        uint32_t *p = reinterpret_cast<uint32_t *>(lut);
        for (uint32_t i = threadIdx.x; i < m; i += blockDim.x) p[i] = tab->packed[i];
    } else {
        uint2 *d = reinterpret_cast<uint2 *>(lut);
        for (int i = threadIdx.x; i < kMaxSym; i += blockDim.x) d[i] = tab->dec[i];
        uint8_t *ss = lut + kMaxSym * sizeof(uint2);
        for (uint32_t i = threadIdx.x; i < m; i += blockDim.x) ss[i] = tab->slot_sym[i];
    }
    __syncthreads();
    const uint32_t lut_sa = smem_addr(lut);
    const uint2 *dec = reinterpret_cast<const uint2 *>(lut);
    const uint8_t *slot_sym = lut + kMaxSym * sizeof(uint2);
    const uint32_t *packed = reinterpret_cast<const uint32_t *>(lut);
    (void)lut_sa;
    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    const uint32_t lt = lanemask_lt();
    const uint32_t ring_sa = smem_addr(sm8 + wib * kRing8Alloc);
    uint8_t *obuf = sm8 + nw * kRing8Alloc + wib * kObuf8;
    int64_t nwk = (n_chunks + gridDim.x - 1) / gridDim.x;
    if (nwk > nw) nwk = nw;
    if (wib >= nwk) return;
    const int64_t warps_total = static_cast<int64_t>(gridDim.x) * nwk;
    for (int64_t k = static_cast<int64_t>(blockIdx.x) * nwk + wib; k < n_chunks;
         k += warps_total) {
        const int64_t cbase = k * chunk_len;
        const uint32_t len = static_cast<uint32_t>((n - cbase) < chunk_len ? (n - cbase) : chunk_len);
        const uint64_t off = offsets[k];
        const uint32_t plen = static_cast<uint32_t>(offsets[k + 1] - off);  // <= 3 len < 2^31
        const uint32_t delta = static_cast<uint32_t>(off & 15u);
        const uint8_t *gbase = payload + (off - delta);
        const uint64_t avail = uint64_t(plen) + delta;
        uint8_t *outk = out + cbase;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            issue_seg8(ring_sa, gbase, avail, q, lane);
            cp_async_commit();
        }
        cp_async_wait<2>();
        __syncwarp();
        uint32_t x = lane < n_lanes ? states[k * n_lanes + lane] : 0u;
        uint32_t pos = delta;  // byte cursor from gbase
        uint32_t cur = 0;      // ring segment holding the cursor
        const uint32_t pend = plen + delta;  // cursor limit
        int err = 0;
        uint32_t most = 0;
        uint32_t base = 0;
        const uint32_t obuf_sa = smem_addr(obuf);
        // Fast path: N = 32, full groups, every initial state in [L, 2^31).
        // From such a state a pop gives x' >= f (x >> sb) >= 2^(23 - sb) >=
        // 2^7, so a lane refills 0, 1 or 2 digits ([x' < 2^23] + [x' <
        // 2^15]: two ballots, no zero-state check) and the refills keep
        // every state valid. Batches of 16 groups (512 symbols, <= 1024
        // digits: the cursor's segment and the two above it, landed before
        // the batch); the decoded bytes leave once per batch, the ring and
        // the truncation check (reads past the payload only see the ring's
        // zero fill) once per batch too.
        uint32_t any2 = 0;  // a group of the fast region refilled two digits
        const uint32_t pos_fast0 = pos;
        if (n_lanes == 32 && __all_sync(0xffffffffu, x >= kLow8)) {
            const uint32_t nbatch = len >> 9;
            const uint32_t lt_mul = lane ? 1u << (32 - lane) : 0u;  // popc(b & lt) = popc(b * lt_mul)
            const uint32_t st_sa = obuf_sa + lane;
            cp_async_wait<1>();  // segments 0..2 landed
            __syncwarp();
            for (uint32_t bt = 0; bt < nbatch; ++bt) {
#pragma unroll
                for (int g = 0; g < 16; ++g) {
                    uint32_t s;
                    {
                        const uint32_t slot = x & mask;
                        if (PACKED) {
                            const uint32_t e = packed[slot];
                            x = (e >> 20) * ((x >> sb) - 4096u) + (e >> 8);
                            s = e;
                        } else {
                            s = slot_sym[slot];
                            const uint2 d = dec[s];
                            x = d.x * (x >> sb) + slot - d.y;
                        }
                    }
                    const bool r1 = x < kLow8, r2 = x < (1u << 15);
                    const uint32_t b1 = __ballot_sync(0xffffffffu, r1);
                    const uint32_t b2 = __ballot_sync(0xffffffffu, r2);
                    // the lane's digits, most significant first: bytes q, q + 1
                    const uint32_t q = pos + __popc(b1 * lt_mul) + __popc(b2 * lt_mul);
                    pos += __popc(b1) + __popc(b2);
                    any2 |= b2;
                    const uint32_t a = ring_sa + (q & (kRing8 - 1));
                    const uint32_t d0 = lds8(a), d1 = lds8(a + 1u);
                    const uint32_t y1 = x * 256u + d0;
                    x = r2 ? y1 * 256u + d1 : (r1 ? y1 : x);
                    sts8(st_sa + g * 32, s);
                }
                __syncwarp();
                {   // 512 decoded bytes: 2 x 8 per lane
                    const uint2 o0 = reinterpret_cast<const uint2 *>(obuf)[lane];
                    const uint2 o1 = reinterpret_cast<const uint2 *>(obuf + 256)[lane];
                    *reinterpret_cast<uint2 *>(outk + base + 8 * lane) = o0;
                    *reinterpret_cast<uint2 *>(outk + base + 256 + 8 * lane) = o1;
                }
                base += 512;
                if (pos > pend) {
                    err = ILANS_ERR_TRUNCATED;
                    break;
                }
                if ((pos >> 9) != cur) {  // segments below the cursor are read
                    while (cur < (pos >> 9)) {
                        ++cur;
                        issue_seg8(ring_sa, gbase, avail, cur + 3, lane);
                        cp_async_commit();
                    }
                }
                cp_async_wait<1>();  // the cursor's segment and the two above landed
                __syncwarp();
            }
            cp_async_wait<0>();
            __syncwarp();
        }
        most = any2 ? 2u : (pos != pos_fast0 ? 1u : 0u);
        for (; !err && base < len; base += n_lanes) {
            const uint32_t left = len - base;
            const bool on = static_cast<uint32_t>(lane) < left && lane < n_lanes;
            uint32_t s = 0;
            if (on) {
                const uint32_t slot = x & mask;
                if (PACKED) {
                    const uint32_t e = packed[slot];
                    x = (e >> 20) * ((x >> sb) - 4096u) + (e >> 8);
                    s = e;
                } else {
                    s = slot_sym[slot];
                    const uint2 d = dec[s];
                    x = d.x * (x >> sb) + slot - d.y;
                }
            }
            if (__any_sync(0xffffffffu, on && x == 0u)) {
                // byte-dependent refills (corrupt input): lane by lane
                const int active = left < static_cast<uint32_t>(n_lanes) ? int(left) : n_lanes;
                for (int l = 0; l < active && !err; ++l) {
                    if (lane == l) {
                        int r = 0;
                        while (x < kLow8) {
                            if (pos >= pend) { err = ILANS_ERR_TRUNCATED; break; }
                            x = (x << 8) | lds8(ring_sa + (pos & (kRing8 - 1)));
                            ++pos;
                            if (++r > kRefillLimit8) { err = ILANS_ERR_FORMAT; break; }
                        }
                        most = max(most, static_cast<uint32_t>(r));
                    }
                    pos = __shfl_sync(0xffffffffu, pos, l);
                    err = __shfl_sync(0xffffffffu, err, l);
                }
            } else {
                const uint32_t r = on ? refills_for(x) : 0u;
                const uint32_t b0 = __ballot_sync(0xffffffffu, r & 1u);
                const uint32_t b1 = __ballot_sync(0xffffffffu, r & 2u);
                const uint32_t q = pos + __popc(b0 & lt) + 2u * __popc(b1 & lt);
                pos += __popc(b0) + 2u * __popc(b1);
                if (pos > pend) {
                    err = ILANS_ERR_TRUNCATED;
                    pos -= __popc(b0) + 2u * __popc(b1);
                } else {
                    // r digits: 4 bytes from two ring words, byte-reversed
                    const uint32_t w0 = lds32(ring_sa + (q & (kRing8 - 4)));
                    const uint32_t w1 = lds32(ring_sa + ((q + 4u) & (kRing8 - 4)));
                    const uint32_t v = __byte_perm(__funnelshift_r(w0, w1, (q & 3u) * 8u), 0u,
                                                   0x0123u);
                    if (r) x = (x << (8u * r)) | (v >> (32u - 8u * r));
                    most = max(most, r);
                }
            }
            if (err) break;
            if (on) sts8(obuf_sa + ((base + lane) & (kObuf8 - 1)), s);
            const uint32_t nb = base + n_lanes;
            if ((nb >> 8) != (base >> 8)) {  // a 256-byte half is complete
                __syncwarp();
                const uint32_t blk = base >> 8;
                const uint2 o = reinterpret_cast<const uint2 *>(obuf + (blk & 1) * 256)[lane];
                *reinterpret_cast<uint2 *>(outk + (blk << 8) + 8 * lane) = o;
                __syncwarp();
            }
            const uint32_t seg = pos >> 9;
            if (seg != cur) {  // segments below the cursor are read: refill them
                __syncwarp();
                while (cur < seg) {
                    ++cur;
                    issue_seg8(ring_sa, gbase, avail, cur + 3, lane);
                    cp_async_commit();
                }
                cp_async_wait<2>();
                __syncwarp();
            }
        }
        {  // bytes of the last partial 256-byte block
            const uint32_t end = err ? base : len;
            __syncwarp();
            const uint32_t t0 = (end >> 8) << 8;
            const uint8_t *half = obuf + ((end >> 8) & 1) * 256;
            for (uint32_t i = t0 + lane; i < end; i += 32) outk[i] = half[i - t0];
        }
        most = __reduce_max_sync(0xffffffffu, most);
        if (lane == 0) {
            atomicMax(&status->max_digits, most);
            if (err == ILANS_ERR_TRUNCATED)
                atomicMin(&status->trunc_stream, static_cast<unsigned long long>(k));
            if (err == ILANS_ERR_FORMAT) status->value_error = ILANS_ERR_FORMAT;
            if (consumed) consumed[k] = pos - delta;
        }
        cp_async_wait<0>();
        __syncwarp();
    }
}

// the device table's flags pick the LUT form (shared memory is sized for the
// larger of the two on the host)
__global__ void __launch_bounds__(kMaxWarps8 * 32, 1)
decode_u8_dispatch_kernel(const uint8_t *__restrict__ payload,
                          const uint64_t *__restrict__ offsets,
                          const uint32_t *__restrict__ states, int64_t n, int64_t chunk_len,
                          int64_t n_chunks, int n_lanes, const TableDev *__restrict__ tab,
                          uint8_t *__restrict__ out, uint64_t *__restrict__ consumed,
                          DStatus *__restrict__ status) {
    extern __shared__ __align__(16) uint8_t sm8[];
    if (tab->status != ILANS_OK) {
        if (threadIdx.x == 0) status->value_error = 1;
        return;
    }
    if (tab->flags & kTabPacked)
        decode_u8_ring_body<true>(payload, offsets, states, n, chunk_len, n_chunks, n_lanes, tab,
                                  out, consumed, status, sm8);
    else
        decode_u8_ring_body<false>(payload, offsets, states, n, chunk_len, n_chunks, n_lanes, tab,
                                   out, consumed, status, sm8);
}

// Backward encode: message segments through the ring (highest first), the
// spilled digits through a 2 KB byte ring (positions in stack coordinates:
// byte p of chunk k lands at scratch[3kC + p], the stack growing down from
// 3 len_k), drained as aligned 16-byte blocks while 512 or more are pending.
__global__ void __launch_bounds__(kMaxWarps8 * 32, 1)
encode_u8_ring_kernel(const uint8_t *__restrict__ msg, int64_t n, int64_t chunk_len,
                      int64_t n_chunks, int n_lanes, const TableDev *__restrict__ tab,
                      uint8_t *__restrict__ scratch, uint32_t *__restrict__ chunk_bytes,
                      uint32_t *__restrict__ states_out, DStatus *__restrict__ status) {
    extern __shared__ __align__(16) uint8_t sm8[];
    const int nw = blockDim.x >> 5;
    uint2 *enc = reinterpret_cast<uint2 *>(sm8);
    uint4 *rec8 = reinterpret_cast<uint4 *>(sm8 + kMaxSym * sizeof(uint2));
    // fast batches (N = 32) take the 8-byte fast records (sb <= 13, every
    // f <= m / 2: table flag kTabEncFast) plus the spill threshold f << (31 - sb)
    const bool fast8 = n_lanes == 32 && (tab->flags & kTabEncFast) != 0u;
    for (int i = threadIdx.x; i < kMaxSym; i += blockDim.x) enc[i] = tab->enc[i];
    if (fast8) {
        const uint32_t t1 = 31u - tab->scale_bits;
        for (int i = threadIdx.x; i < kRec8Copies * kMaxSym; i += blockDim.x) {
            const int sym = i / kRec8Copies;
            const uint2 f = tab->encf[sym];
            rec8[i] = make_uint4(f.x, f.y, tab->freq[sym] << t1, 0u);
        }
    }
    __syncthreads();
    const EncCtx ctx(tab->scale_bits);
    const uint32_t thr8 = 31u - tab->scale_bits;  // spill while x >= f << (31 - sb)
    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    const uint32_t lt = lanemask_lt();
    // [enc 2 KB][rec8 32 KB][W message rings][pad to 2 KB][W spill rings, 2 KB aligned]
    uint8_t *rings = sm8 + kMaxSym * sizeof(uint2) + size_t(kRec8Copies) * kMaxSym * sizeof(uint4);
    const uint32_t in_sa = smem_addr(rings + wib * kRing8);
    const uint32_t raw = smem_addr(rings + nw * kRing8);
    const uint32_t out_sa = ((raw + kRing8 - 1) & ~uint32_t(kRing8 - 1)) + wib * kRing8;
    const uint8_t *out_ring = sm8 + (out_sa - smem_addr(sm8));
    // this lane's record copy: symbol s at rec_sa + s * 16 * kRec8Copies
    const uint32_t rec_sa = smem_addr(rec8 + (lane & (kRec8Copies - 1)));
    int64_t nwk = (n_chunks + gridDim.x - 1) / gridDim.x;
    if (nwk > nw) nwk = nw;
    if (wib >= nwk) return;
    const int64_t warps_total = static_cast<int64_t>(gridDim.x) * nwk;
    for (int64_t k = static_cast<int64_t>(blockIdx.x) * nwk + wib; k < n_chunks;
         k += warps_total) {
        // chunk-local cursors in 32 bits (chunks < 2^29 bytes: 3 len < 2^31)
        const int64_t cbase = k * chunk_len;
        const int len = static_cast<int>((n - cbase) < chunk_len ? (n - cbase) : chunk_len);
        const uint8_t *g = msg + cbase;
        uint8_t *o = scratch + 3 * cbase;
        int cur = (len - 1) >> 9;  // segment holding the current group's top byte
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int sg = cur - q;
            const int b0 = sg * kSeg8 + lane * 16;
            uint32_t bytes = 0;
            if (sg >= 0 && b0 < len) bytes = (len - b0) >= 16 ? 16u : static_cast<uint32_t>(len - b0);
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(
                             in_sa + static_cast<uint32_t>(sg & 3) * kSeg8 + lane * 16),
                         "l"(bytes ? g + b0 : g), "r"(bytes)
                         : "memory");
            cp_async_commit();
        }
        cp_async_wait<2>();  // segments cur and cur - 1 (a group may straddle)
        __syncwarp();
        uint32_t x = kLow8;
        int top = 3 * len;                 // stack top (bytes)
        int flushed = (top + 15) & ~15;    // [flushed, ...) is in HBM
        bool bad = false;
        uint32_t most = 0;
        const int groups = (len + n_lanes - 1) / n_lanes;
        int base = (groups - 1) * n_lanes;
        // N = 32: the full groups below fast_top take the fast loop after
        // this one has coded the partial top group (if any)
        // (fast8: the whole 512-symbol blocks below take the batched loop)
        const int fast_top = n_lanes == 32 ? (fast8 ? (len & ~511) : (len & ~31)) : 0;
        for (; base >= fast_top; base -= n_lanes) {
            const int left = len - base;
            const bool on = lane < left && lane < n_lanes;
            const int hs = (base + (left < n_lanes ? left : n_lanes) - 1) >> 9;
            if (hs != cur) {  // segment cur consumed: prefetch cur - 4 into its slot
                __syncwarp();
                while (cur > hs) {
                    const int sg = cur - 4;
                    const bool ok = sg >= 0;
                    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(
                                     in_sa + static_cast<uint32_t>(sg & 3) * kSeg8 + lane * 16),
                                 "l"(ok ? g + sg * kSeg8 + lane * 16 : g), "r"(ok ? 16u : 0u)
                                 : "memory");
                    cp_async_commit();
                    --cur;
                }
                cp_async_wait<2>();
                __syncwarp();
            }
            const uint2 e = enc[on ? lds8(in_sa + ((base + lane) & (kRing8 - 1))) : 0u];
            if (__any_sync(0xffffffffu, on && e.x == 0u)) {
                const uint32_t badmask = __ballot_sync(0xffffffffu, on && e.x == 0u);
                if (lane == 0)
                    atomicMax(&status->unenc_index,
                              static_cast<long long>(cbase + base + 31 - __clz(badmask)));
                bad = true;
                break;
            }
            const uint32_t fm1 = e.y & 0xFFFFu;  // spill while (x >> 8j) >> thr8 > f - 1
            const uint32_t sp = on ? ((x >> thr8) > fm1) + (((x >> 8) >> thr8) > fm1) +
                                         (((x >> 16) >> thr8) > fm1)
                                   : 0u;
            const uint32_t b0 = __ballot_sync(0xffffffffu, sp & 1u);
            const uint32_t b1 = __ballot_sync(0xffffffffu, sp & 2u);
            top -= __popc(b0) + 2 * __popc(b1);
            // read order is most significant spilled byte first: byte j of the
            // lane's sp digits (j < sp) is x >> 8 (sp - 1 - j)
            const uint32_t pe = out_sa + ((static_cast<uint32_t>(top) + __popc(b0 & lt) +
                                           2u * __popc(b1 & lt) + sp - 1u) & (kRing8 - 1));
            if (sp >= 1u) sts8(pe, x);
            if (sp >= 2u) sts8(out_sa + ((pe - out_sa - 1u) & (kRing8 - 1)), x >> 8);
            if (sp >= 3u) sts8(out_sa + ((pe - out_sa - 2u) & (kRing8 - 1)), x >> 16);
            if (on) x = enc_push(ctx, x >> (8u * sp), e);
            most = max(most, sp);
            if (flushed - top >= 512) {  // drain 512 bytes: 16 per lane
                __syncwarp();
                const uint32_t ro = static_cast<uint32_t>(flushed - 512) + lane * 16;
                uint4 v;
                asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                             : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                             : "r"(out_sa + (ro & (kRing8 - 1))));
                *reinterpret_cast<uint4 *>(o + (flushed - 512) + lane * 16) = v;
                flushed -= 512;
                __syncwarp();
            }
        }
        // Batched fast loop (fast8): blocks of 16 groups, backwards. A state
        // below 2^31 spills at most two digits (x >> 16 < 2^15 <= f 2^(31 -
        // sb)): s1 = x >= T1, s2 = x >> 8 >= T1 with T1 = f << (31 - sb); two
        // ballots give each lane its read-order offset, digits most
        // significant first. The push is the word16 fast record's (the
        // state after the spills is below f 2^(31 - sb) <= 2^30). Records
        // of frequency 0 clear bit 31 of the AND of every M, checked once
        // per block (then the block is rescanned for the reference's
        // highest offending index). The spill ring drains per block (a
        // block adds <= 1024 digits to < 512 pending).
        if (fast8) {
            const uint32_t lt_mul = lane ? 1u << (32 - lane) : 0u;
            const uint32_t t_shift = 32u - tab->scale_bits;
            const uint32_t qoff = 1u << (27u - tab->scale_bits);
            uint32_t any2 = 0;
            const int top_fast0 = top;
            for (int b = (base + 32) / 512 - 1; b >= 0 && !bad; --b) {
                if (b != cur) {  // segment cur consumed: prefetch cur - 4 into its slot
                    __syncwarp();
                    while (cur > b) {
                        const int sg = cur - 4;
                        const bool ok = sg >= 0;
                        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(
                                         in_sa + static_cast<uint32_t>(sg & 3) * kSeg8 + lane * 16),
                                     "l"(ok ? g + sg * kSeg8 + lane * 16 : g), "r"(ok ? 16u : 0u)
                                     : "memory");
                        cp_async_commit();
                        --cur;
                    }
                    cp_async_wait<2>();
                    __syncwarp();
                }
                const uint32_t blk_sa = in_sa + static_cast<uint32_t>(b & 3) * kSeg8 + lane;
                uint32_t macc = ~0u;
                uint32_t sym_n = lds8(blk_sa + 15 * 32);
#pragma unroll
                for (int gg = 15; gg >= 0; --gg) {
                    uint4 e;
                    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                                 : "=r"(e.x), "=r"(e.y), "=r"(e.z), "=r"(e.w)
                                 : "r"(rec_sa + sym_n * (16u * kRec8Copies)));
                    if (gg > 0) sym_n = lds8(blk_sa + (gg - 1) * 32);
                    macc &= e.x;
                    const bool s1 = x >= e.z, s2 = (x >> 8) >= e.z;
                    const uint32_t b1 = __ballot_sync(0xffffffffu, s1);
                    const uint32_t b2 = __ballot_sync(0xffffffffu, s2);
                    top -= static_cast<int>(__popc(b1) + __popc(b2));
                    any2 |= b2;
                    const uint32_t p = static_cast<uint32_t>(top) + __popc(b1 * lt_mul) +
                                       __popc(b2 * lt_mul);
                    if (s1) sts8(out_sa + (p & (kRing8 - 1)), s2 ? x >> 8 : x);
                    if (s2) sts8(out_sa + ((p + 1u) & (kRing8 - 1)), x);
                    x = s2 ? x >> 16 : (s1 ? x >> 8 : x);
                    uint32_t q = __umulhi(x, e.x);
                    asm("shf.r.wrap.b32 %0, %1, %2, %3;" : "=r"(q) : "r"(q), "r"(0u), "r"(e.y));
                    x = (e.y >> t_shift) * (q - qoff) + (x + (e.y >> 5));
                }
                if (__any_sync(0xffffffffu, !(macc >> 31))) {  // a symbol of frequency 0 here
                    uint32_t hi = 0;
                    for (int gg = 0; gg < 16; ++gg)
                        if (enc[lds8(blk_sa + gg * 32)].x == 0u) hi = 32u * gg + lane + 1u;
                    hi = __reduce_max_sync(0xffffffffu, hi);
                    if (lane == 0)
                        atomicMax(&status->unenc_index,
                                  static_cast<long long>(cbase + b * 512 + int(hi) - 1));
                    bad = true;
                    break;
                }
                __syncwarp();
                while (flushed - top >= 512) {  // drain 512 bytes: 16 per lane
                    const uint32_t ro = static_cast<uint32_t>(flushed - 512) + lane * 16;
                    uint4 v;
                    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                                 : "r"(out_sa + (ro & (kRing8 - 1))));
                    *reinterpret_cast<uint4 *>(o + (flushed - 512) + lane * 16) = v;
                    flushed -= 512;
                }
                __syncwarp();
            }
            base = -32;  // every group coded
            most = max(most, any2 ? 2u : (top != top_fast0 ? 1u : 0u));
        }
        // Fast loop (N = 32, full groups): a state below 2^31 spills at most
        // two digits (x >> 16 < 2^15 <= f 2^(31 - sb)), so two ballots give
        // each lane its read-order offset; digits most significant first.
        for (; !bad && base >= 0; base -= 32) {
            const int hs = (base + 31) >> 9;
            if (hs != cur) {  // segment cur consumed: prefetch cur - 4 into its slot
                __syncwarp();
                while (cur > hs) {
                    const int sg = cur - 4;
                    const bool ok = sg >= 0;
                    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(
                                     in_sa + static_cast<uint32_t>(sg & 3) * kSeg8 + lane * 16),
                                 "l"(ok ? g + sg * kSeg8 + lane * 16 : g), "r"(ok ? 16u : 0u)
                                 : "memory");
                    cp_async_commit();
                    --cur;
                }
                cp_async_wait<2>();
                __syncwarp();
            }
            const uint2 e = enc[lds8(in_sa + ((base + lane) & (kRing8 - 1)))];
            if (__any_sync(0xffffffffu, e.x == 0u)) {
                const uint32_t badmask = __ballot_sync(0xffffffffu, e.x == 0u);
                if (lane == 0)
                    atomicMax(&status->unenc_index,
                              static_cast<long long>(cbase + base + 31 - __clz(badmask)));
                bad = true;
                break;
            }
            const uint32_t fm1 = e.y & 0xFFFFu;
            const bool s1 = (x >> thr8) > fm1, s2 = ((x >> 8) >> thr8) > fm1;
            const uint32_t b1 = __ballot_sync(0xffffffffu, s1);
            const uint32_t b2 = __ballot_sync(0xffffffffu, s2);
            top -= __popc(b1) + __popc(b2);
            const uint32_t p = static_cast<uint32_t>(top) + __popc(b1 & lt) + __popc(b2 & lt);
            if (s1) sts8(out_sa + (p & (kRing8 - 1)), s2 ? x >> 8 : x);
            if (s2) sts8(out_sa + ((p + 1u) & (kRing8 - 1)), x);
            const uint32_t sp = static_cast<uint32_t>(s1) + static_cast<uint32_t>(s2);
            x = enc_push(ctx, x >> (8u * sp), e);
            most = max(most, sp);
            if (flushed - top >= 512) {  // drain 512 bytes: 16 per lane
                __syncwarp();
                const uint32_t ro = static_cast<uint32_t>(flushed - 512) + lane * 16;
                uint4 v;
                asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                             : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                             : "r"(out_sa + (ro & (kRing8 - 1))));
                *reinterpret_cast<uint4 *>(o + (flushed - 512) + lane * 16) = v;
                flushed -= 512;
                __syncwarp();
            }
        }
        most = __reduce_max_sync(0xffffffffu, most);
        if (lane == 0) atomicMax(&status->max_digits, most);
        if (!bad) {
            __syncwarp();
            // whole 16-byte blocks of [roundup16(top), flushed), then the head bytes
            const int lo16 = (top + 15) & ~15;
            for (int b = lo16 + lane * 16; b < flushed; b += 512) {
                uint4 v;
                asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                             : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                             : "r"(out_sa + (static_cast<uint32_t>(b) & (kRing8 - 1))));
                *reinterpret_cast<uint4 *>(o + b) = v;
            }
            for (int b = top + lane; b < lo16 && b < flushed; b += 32)
                o[b] = out_ring[b & (kRing8 - 1)];
            if (lane == 0) chunk_bytes[k] = static_cast<uint32_t>(3 * len - top);
            if (lane < n_lanes) states_out[k * n_lanes + lane] = x;
        }
        cp_async_wait<0>();
        __syncwarp();
    }
}

static size_t ring8_decode_smem(int warps, int sb, bool packed) {
    const size_t m = size_t(1) << sb;
    const size_t lut = packed ? m * 4 : kMaxSym * sizeof(uint2) + (m < 16 ? 16 : m);
    return size_t(warps) * (kRing8Alloc + kObuf8) + ((lut + 15) & ~size_t(15));
}

static size_t ring8_encode_smem(int warps) {
    return kMaxSym * sizeof(uint2) + size_t(kRec8Copies) * kMaxSym * sizeof(uint4) +
           size_t(warps) * kRing8 + kRing8 + size_t(warps) * kRing8;
}

// one CTA per SM with the SM's share of the streams (as the word16 coders)
static void ring8_shape(int64_t n_chunks, int *warps, int *cta_warps, int64_t *blocks) {
    const int64_t sms = sm_count();
    int w = static_cast<int>((n_chunks + sms - 1) / sms);
    if (w > kMaxWarps8) w = kMaxWarps8;
    if (w < 1) w = 1;
    int64_t b = (n_chunks + w - 1) / w;
    if (b > sms) b = sms;  // grid-stride beyond one wave
    *warps = w;
    *cta_warps = w;
    *blocks = b;
}

// N > 32: one CTA per stream, thread t owns lanes [t*k, t*k + k) (k <= 64),// N > 32: one CTA per stream, thread t owns lanes [t*k, t*k + k) (k <= 64),
// CTA-wide exclusive scans of the digit counts; states live in ws.
__device__ __forceinline__ uint32_t block_excl_scan_8(uint32_t v, uint32_t *total,
                                                      uint32_t *sh) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int nw = blockDim.x >> 5;
    uint32_t inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t u = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += u;
    }
    if (lane == 31) sh[wid] = inc;
    __syncthreads();
    if (wid == 0) {
        uint32_t w = lane < nw ? sh[lane] : 0u;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t u = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += u;
        }
        sh[lane] = w;
    }
    __syncthreads();
    const uint32_t off = wid ? sh[wid - 1] : 0u;
    *total = sh[nw - 1];
    __syncthreads();
    return off + inc - v;
}

__global__ void __launch_bounds__(1024)
decode_u8_block_kernel(const uint8_t *__restrict__ pay, uint64_t plen,
                       const uint32_t *__restrict__ states, int64_t len, int n_lanes,
                       const TableDev *__restrict__ tab, uint8_t *__restrict__ out,
                       uint64_t *__restrict__ consumed, DStatus *__restrict__ status,
                       uint32_t *__restrict__ ws, DecodeTrace trace) {
    __shared__ uint32_t scan_sh[32];
    __shared__ int zero_any;
    const int sb = static_cast<int>(tab->scale_bits);
    const uint32_t mask = (1u << sb) - 1u;
    const int per = (n_lanes + blockDim.x - 1) / blockDim.x;
    const int lo = threadIdx.x * per;
    for (int l = lo; l < lo + per && l < n_lanes; ++l) ws[l] = states[l];
    uint64_t pos = 0;
    int err = 0;
    uint32_t most = 0;
    int64_t base = 0;
    for (; base < len; base += n_lanes) {
        const int64_t left = len - base;
        const int active = left < n_lanes ? static_cast<int>(left) : n_lanes;
        const int hi = lo + per < active ? lo + per : active;
        if (threadIdx.x == 0) zero_any = 0;
        __syncthreads();
        uint32_t cnt = 0;
        for (int l = lo; l < hi; ++l) {
            uint32_t x = ws[l];
            const uint32_t slot = x & mask;
            const uint32_t s = tab->slot_sym[slot];
            const uint2 d = tab->dec[s];
            x = d.x * (x >> sb) + slot - d.y;
            out[base + l] = static_cast<uint8_t>(s);
            ws[l] = x;
            if (x == 0u) zero_any = 1;
            else cnt += refills_for(x);
        }
        __syncthreads();
        if (zero_any) {  // corrupt input: serial resolution by thread 0
            if (threadIdx.x == 0) {
                for (int l = 0; l < active && !err; ++l) {
                    uint32_t x = ws[l];
                    int r = 0;
                    while (x < kLow8) {
                        if (pos >= plen) { err = ILANS_ERR_TRUNCATED; break; }
                        x = (x << 8) | pay[pos++];
                        if (++r > kRefillLimit8) { err = ILANS_ERR_FORMAT; break; }
                    }
                    ws[l] = x;
                    most = max(most, static_cast<uint32_t>(r));
                }
                scan_sh[0] = static_cast<uint32_t>(err);
            }
            __syncthreads();
            err = static_cast<int>(scan_sh[0]);
            __syncthreads();
            // every thread re-reads pos from thread 0 via shared memory
            if (threadIdx.x == 0) scan_sh[1] = static_cast<uint32_t>(pos), scan_sh[2] = static_cast<uint32_t>(pos >> 32);
            __syncthreads();
            pos = (static_cast<uint64_t>(scan_sh[2]) << 32) | scan_sh[1];
            __syncthreads();
        } else {
            uint32_t total;
            const uint32_t excl = block_excl_scan_8(cnt, &total, scan_sh);
            if (pos + total > plen) {
                err = ILANS_ERR_TRUNCATED;
            } else {
                uint64_t p = pos + excl;
                for (int l = lo; l < hi; ++l) {
                    uint32_t x = ws[l];
                    const uint32_t r = refills_for(x);
                    for (uint32_t j = 0; j < r; ++j) x = (x << 8) | pay[p++];
                    ws[l] = x;
                    most = max(most, r);
                }
                pos += total;
            }
        }
        if (err) break;
        if (trace.states) {
            __syncthreads();
            const int64_t gi = base / n_lanes;
            for (int l = lo; l < lo + per && l < n_lanes; ++l) trace.states[gi * n_lanes + l] = ws[l];
            if (threadIdx.x == 0) trace.pos[gi] = pos;
        }
    }
    atomicMax(&status->max_digits, most);
    if (threadIdx.x == 0) {
        if (err == ILANS_ERR_TRUNCATED) atomicMin(&status->trunc_stream, 0ull);
        if (err == ILANS_ERR_FORMAT) status->value_error = ILANS_ERR_FORMAT;
        if (consumed) consumed[0] = pos;
        if (trace.groups) trace.groups[0] = (base < len ? base : len + n_lanes - 1) / n_lanes;
    }
}

__global__ void __launch_bounds__(1024)
encode_u8_block_kernel(const uint8_t *__restrict__ g, int64_t len, int n_lanes,
                       const TableDev *__restrict__ tab, uint8_t *__restrict__ o,
                       uint32_t *__restrict__ chunk_bytes, uint32_t *__restrict__ states_out,
                       DStatus *__restrict__ status, uint32_t *__restrict__ ws) {
    __shared__ uint32_t scan_sh[32];
    __shared__ uint2 enc[kMaxSym];
    for (int i = threadIdx.x; i < kMaxSym; i += blockDim.x) enc[i] = tab->enc[i];
    __syncthreads();
    const EncCtx ctx(tab->scale_bits);
    const uint32_t thr8 = 31u - tab->scale_bits;
    const int per = (n_lanes + blockDim.x - 1) / blockDim.x;
    const int lo = threadIdx.x * per;
    for (int l = lo; l < lo + per && l < n_lanes; ++l) ws[l] = kLow8;
    int64_t top = 3 * len;
    bool bad = false;
    uint32_t most = 0;
    for (int64_t gi = (len + n_lanes - 1) / n_lanes - 1; gi >= 0; --gi) {
        const int64_t base = gi * n_lanes;
        const int64_t left = len - base;
        const int active = left < n_lanes ? static_cast<int>(left) : n_lanes;
        const int hi = lo + per < active ? lo + per : active;
        long long my_bad = -1;
        uint32_t cnt = 0;
        for (int l = lo; l < hi; ++l) {
            const uint2 e = enc[g[base + l]];
            if (e.x == 0u) { my_bad = base + l; continue; }
            const uint32_t x = ws[l], fm1 = e.y & 0xFFFFu;
            cnt += ((x >> thr8) > fm1) + (((x >> 8) >> thr8) > fm1) + (((x >> 16) >> thr8) > fm1);
        }
        if (__syncthreads_or(my_bad >= 0)) {
            if (my_bad >= 0) atomicMax(&status->unenc_index, my_bad);
            bad = true;
            break;
        }
        uint32_t total;
        const uint32_t excl = block_excl_scan_8(cnt, &total, scan_sh);
        top -= total;
        int64_t p = top + excl;
        for (int l = lo; l < hi; ++l) {
            const uint2 e = enc[g[base + l]];
            uint32_t x = ws[l];
            const uint32_t fm1 = e.y & 0xFFFFu;
            const uint32_t sp = ((x >> thr8) > fm1) + (((x >> 8) >> thr8) > fm1) +
                                (((x >> 16) >> thr8) > fm1);
            for (uint32_t j = 0; j < sp; ++j) o[p++] = static_cast<uint8_t>(x >> (8 * (sp - 1 - j)));
            ws[l] = enc_push(ctx, sp ? x >> (8 * sp) : x, e);
            most = max(most, sp);
        }
    }
    atomicMax(&status->max_digits, most);
    if (!bad) {
        if (threadIdx.x == 0) chunk_bytes[0] = static_cast<uint32_t>(3 * len - top);
        for (int l = lo; l < lo + per && l < n_lanes; ++l) states_out[l] = ws[l];
    }
}

static cudaError_t launch_decode_ring8(const uint8_t *d_payload, const uint64_t *d_offsets,
                                       const uint32_t *d_states, int64_t n, int64_t chunk_len,
                                       int64_t n_chunks, int n_lanes, const TableDev *d_table,
                                       uint8_t *d_out, uint64_t *d_consumed, DStatus *d_status,
                                       cudaStream_t stream) {
    int warps, cta_warps;
    int64_t blocks;
    ring8_shape(n_chunks, &warps, &cta_warps, &blocks);
    (void)warps;
    // scale_bits and the packed flag are device-side: size for the larger
    // LUT (32-bit entries at sb = 15 vs the two-lookup form at sb = 16)
    size_t smem = ring8_decode_smem(cta_warps, kMaxScaleBits, false);
    const size_t smem32 = ring8_decode_smem(cta_warps, kPackedMaxBits, true);
    if (smem32 > smem) smem = smem32;
    smem_limit(reinterpret_cast<const void *>(decode_u8_dispatch_kernel), int(smem));
    decode_u8_dispatch_kernel<<<static_cast<unsigned>(blocks), cta_warps * 32, smem, stream>>>(
        d_payload, d_offsets, d_states, n, chunk_len, n_chunks, n_lanes, d_table, d_out,
        d_consumed, d_status);
    ilans_note_launch();
    return cudaGetLastError();
}

cudaError_t launch_encode_u8(const uint8_t *d_msg, int64_t n, int n_lanes, const TableDev *d_table,
                             uint8_t *d_scratch, uint32_t *d_bytes, uint32_t *d_states,
                             DStatus *d_status, uint32_t *d_lane_ws, cudaStream_t stream) {
    if (n <= 0) return cudaSuccess;
    if (n_lanes > 32 || n > kRingMaxChunk8) {
        const int threads = n_lanes >= 1024 ? 1024 : ((n_lanes + 31) / 32) * 32;
        encode_u8_block_kernel<<<1, threads, 0, stream>>>(d_msg, n, n_lanes, d_table, d_scratch,
                                                          d_bytes, d_states, d_status, d_lane_ws);
    } else {  // the staged kernel, one stream = one chunk
        return launch_encode_chunks_u8(d_msg, n, n, n_lanes, d_table, d_scratch, d_bytes,
                                       d_states, d_status, stream);
    }
    ilans_note_launch();
    return cudaGetLastError();
}

cudaError_t launch_decode_u8(const uint8_t *d_payload, uint64_t pay_len, const uint64_t *d_offsets,
                             const uint32_t *d_states, int64_t n, int n_lanes,
                             const TableDev *d_table, uint8_t *d_out, uint64_t *d_consumed,
                             DStatus *d_status, uint32_t *d_lane_ws, cudaStream_t stream,
                             DecodeTrace trace) {
    if (n <= 0) return cudaSuccess;
    if (n_lanes <= 32 && !trace.states && n <= kRingMaxChunk8)  // staged: one stream = one chunk
        return launch_decode_ring8(d_payload, d_offsets, d_states, n, n, 1, n_lanes, d_table,
                                   d_out, d_consumed, d_status, stream);
    if (n_lanes > 32) {
        const int threads = n_lanes >= 1024 ? 1024 : ((n_lanes + 31) / 32) * 32;
        decode_u8_block_kernel<<<1, threads, 0, stream>>>(
            d_payload, pay_len, d_states, n, n_lanes, d_table, d_out, d_consumed, d_status,
            d_lane_ws, trace);
    } else {
        decode_u8_warp_kernel<<<1, 32, 0, stream>>>(d_payload, d_offsets, d_states, n, n, 1,
                                                    n_lanes, d_table, d_out, d_consumed,
                                                    d_status, trace);
    }
    ilans_note_launch();
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Chunked byte8 (the ICH1 framing of encode.cu with byte digits): chunk k is
// an independent byte8 stream; its digits sit at
// scratch[3kC + 3 len_k - b_k, 3kC + 3 len_k) after the encode, and the
// framing packs them back to back at the scanned byte offsets.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256)
compact_u8_kernel(const uint8_t *__restrict__ scratch, int64_t n, int64_t chunk_len,
                  const uint32_t *__restrict__ bytes, const uint64_t *__restrict__ offsets,
                  uint8_t *__restrict__ payload) {
    for (int64_t k = blockIdx.x; k * chunk_len < n; k += gridDim.x) {
        const int64_t cbase = k * chunk_len;
        const int64_t len = (n - cbase) < chunk_len ? (n - cbase) : chunk_len;
        const uint32_t b = bytes[k];
        const uint64_t s = uint64_t(3 * cbase + 3 * len) - b;  // source byte
        const uint64_t d = offsets[k];                          // destination byte
        // head bytes up to a 4-byte aligned destination, then whole words
        // assembled from two aligned source words, then the tail bytes
        uint32_t head = uint32_t((4u - (d & 3u)) & 3u);
        if (head > b) head = b;
        if (threadIdx.x < head) payload[d + threadIdx.x] = scratch[s + threadIdx.x];
        const uint32_t words = (b - head) >> 2;
        const uint64_t s0 = s + head;
        const uint32_t *src = reinterpret_cast<const uint32_t *>(scratch + (s0 & ~uint64_t(3)));
        const uint32_t sh = uint32_t(s0 & 3u) * 8u;
        uint32_t *dst = reinterpret_cast<uint32_t *>(payload + d + head);
        for (uint32_t i = threadIdx.x; i < words; i += blockDim.x)
            dst[i] = sh ? __funnelshift_r(src[i], src[i + 1], sh) : src[i];
        const uint32_t done = head + 4 * words;
        if (threadIdx.x < b - done) payload[d + done + threadIdx.x] = scratch[s + done + threadIdx.x];
    }
}

cudaError_t launch_encode_chunks_u8(const uint8_t *d_msg, int64_t n, int64_t chunk_len,
                                    int n_lanes, const TableDev *d_table, uint8_t *d_scratch,
                                    uint32_t *d_bytes, uint32_t *d_states, DStatus *d_status,
                                    cudaStream_t stream) {
    if (n <= 0) return cudaSuccess;
    if (chunk_len > kRingMaxChunk8) return cudaErrorInvalidValue;
    const int64_t n_chunks = (n + chunk_len - 1) / chunk_len;
    int warps, cta_warps;
    int64_t blocks;
    ring8_shape(n_chunks, &warps, &cta_warps, &blocks);
    const size_t smem = ring8_encode_smem(cta_warps);
    smem_limit(reinterpret_cast<const void *>(encode_u8_ring_kernel), int(smem));
    encode_u8_ring_kernel<<<static_cast<unsigned>(blocks), cta_warps * 32, smem, stream>>>(
        d_msg, n, chunk_len, n_chunks, n_lanes, d_table, d_scratch, d_bytes, d_states, d_status);
    ilans_note_launch();
    return cudaGetLastError();
}

cudaError_t launch_frame_u8(const uint8_t *d_scratch, int64_t n, int64_t chunk_len,
                            const uint32_t *d_bytes, uint64_t *d_offsets, uint8_t *d_payload,
                            cudaStream_t stream) {
    const int64_t n_chunks = n <= 0 ? 0 : (n + chunk_len - 1) / chunk_len;
    chunk_offsets_kernel<<<1, 1024, 0, stream>>>(d_bytes, n_chunks, d_offsets, 0);
    ilans_note_launch();
    if (n_chunks > 0) {
        const int64_t cap = int64_t(sm_count()) * 8;
        compact_u8_kernel<<<static_cast<unsigned>(n_chunks < cap ? n_chunks : cap), 256, 0,
                            stream>>>(d_scratch, n, chunk_len, d_bytes, d_offsets, d_payload);
        ilans_note_launch();
    }
    return cudaGetLastError();
}

cudaError_t launch_decode_chunks_u8(const uint8_t *d_payload, const uint64_t *d_offsets,
                                    const uint32_t *d_states, int64_t n, int64_t chunk_len,
                                    int n_lanes, const TableDev *d_table, uint8_t *d_out,
                                    uint64_t *d_consumed, DStatus *d_status, cudaStream_t stream) {
    if (n <= 0) return cudaSuccess;
    if (chunk_len > kRingMaxChunk8) return cudaErrorInvalidValue;
    const int64_t n_chunks = (n + chunk_len - 1) / chunk_len;
    return launch_decode_ring8(d_payload, d_offsets, d_states, n, chunk_len, n_chunks, n_lanes,
                               d_table, d_out, d_consumed, d_status, stream);
}

}  // namespace ilans
