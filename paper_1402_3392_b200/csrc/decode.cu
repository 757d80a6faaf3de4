// decode.cu -- word16 interleaved-rANS decoders for sm_100a.
//
// Replaces _core.decode_interleaved_u16 (_core.pyx:46-127) and
// _core.decode_lanes_u16 (_core.pyx:130-173); both produce byte-identical
// output (_pure.py:69-72), so one group-at-a-time kernel serves both.
//
// Warp kernel (N <= 32): one warp per stream (chunk), lane l = rANS lane l,
// one CTA per SM holding all of the SM's chunks (<= 28 warps); the decoded
// bytes go to a sink (HBM, or a consumer fused into the decoder).
// Per group of N symbols (lanes.decode_step, lanes.py:138-151):
//   pop:     slot = x & (m-1); s = LUT[slot]; x = f*(x >> sb) + slot - cum
//   ballot:  mask = __ballot_sync(x < 2^16)            (lanes.ballot)
//   refill:  x = x << 16 | payload[pos + popc(mask & lanemask_lt)]
//                                                      (lanes.packed_load)
//   pos += popc(mask)
// The payload is staged into a per-warp shared-memory ring by cp.async
// (4 segments x 256 words; two segments = ~44 groups ahead of the reader),
// so the refill read is a conflict-free LDS, never an HBM round trip.
// Slots 0 and 1 are mirrored past the end of the ring (1536 words), so a
// 512-word batch read starting anywhere in the ring never wraps: inside a
// batch the read address is the batch base plus a running byte offset.
//
// N = 32 fast path: 16 groups (512 symbols) per batch, fully unrolled, with
// the packed LUT (32-bit entries for sb <= 12, 64-bit for sb 13-14); the
// ring is advanced and the 512 decoded bytes are handed to the sink (one
// 16-byte vector store per lane) once per batch, and truncation is checked once per
// batch (pos is monotone, so "some group overran" == "pos > len at the end
// of the batch"; reads past the payload hit zero-filled ring words and are
// never used). Other N and the < 512-symbol tail run the per-group loop.
//
// Block kernel (N > 32, up to 65535 lanes): one CTA per stream, contiguous
// lane ranges per thread and a CTA-wide exclusive scan of refill counts in
// place of the warp ballot. Correct for every N, used for
// the wide single-stream calls the reference allows (interleave.py:197-200).
#include "common.cuh"
#include "kernels.cuh"

namespace ilans {

constexpr int kSegWords = 256;             // 512 B per cp.async warp-copy (16 B / lane)
constexpr int kRingWords = 4 * kSegWords;  // 2 KB payload ring per warp
constexpr int kRingBytes = kRingWords * 2;
constexpr int kRingAllocBytes = kRingBytes + 2 * kSegWords * 2;  // + mirror of slots 0, 1
constexpr int kBatch = 16;                 // groups per fast-path batch (N = 32)
constexpr int kObufBytes = 512;            // 2 x 256 B output halves per warp
constexpr int kObufHalf = kObufBytes / 2;

struct SegSrc {
    const uint16_t *g;    // 16-byte aligned base of the chunk's payload
    uint64_t avail;       // readable words from g
};

__device__ __forceinline__ void issue_segment(uint16_t *ring, const SegSrc &src, uint32_t seg,
                                              int lane) {
    const uint64_t w0 = static_cast<uint64_t>(seg) * kSegWords + lane * 8;
    uint32_t bytes = 0;
    if (src.avail > w0) {
        const uint64_t left = (src.avail - w0) * 2u;
        bytes = left >= 16u ? 16u : static_cast<uint32_t>(left);
    }
    const uint16_t *g = bytes ? src.g + w0 : src.g;
    cp_async16(ring + (seg & 3u) * kSegWords + lane * 8, g, bytes);
    if ((seg & 3u) < 2u)  // mirror (warp-uniform branch)
        cp_async16(ring + (4u + (seg & 3u)) * kSegWords + lane * 8, g, bytes);
}

__device__ __forceinline__ uint32_t mad_lo(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t d;
    asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}

__device__ __forceinline__ uint32_t lds_u16(uint32_t addr) {
    uint16_t w;
    asm volatile("ld.shared.u16 %0, [%1];" : "=h"(w) : "r"(addr));
    return w;
}

// Per-group refill read (generic loop): ring base + cursor modulo the ring.
__device__ __forceinline__ uint32_t ring_load(uint32_t ring_addr, uint32_t byte_off) {
    return lds_u16(ring_addr + (byte_off & (kRingBytes - 2)));
}

// LUT forms: packed 32-bit entries (sb <= 12), packed 64-bit entries
// (13 <= sb <= 14: one LDS.64 per lane instead of two dependent lookups),
// and the two-lookup form slot -> symbol -> {f, cum} (any sb).
enum : int { kLutGeneric = 0, kLutPacked32 = 1, kLutPacked64 = 2 };
// launch-only kind (13 <= sb <= 14): shared memory sized for the 64-bit LUT;
// the 32-bit entries run when every f < 4096, else the 64-bit ones
constexpr int kLutPacked3264 = 3;
__host__ __device__ constexpr bool allows32(int maxkind) {
    return maxkind == kLutPacked32 || maxkind == kLutPacked3264;
}
__host__ __device__ constexpr bool allows64(int maxkind) {
    return maxkind == kLutPacked64 || maxkind == kLutPacked3264;
}

// SBC: scale bits known at compile time (0: the runtime value in sb). With
// a constant, h = (x >> sb) - 4096 is one LEA.HI instead of SHF + IADD and
// the slot mask is an immediate (the sb = 12 packed decoder).
template <int KIND, int SBC = 0>
struct Lut {
    const uint32_t *packed;  // kLutPacked32: sym | bias << 8 | f << 20
    const uint2 *packed64;   // kLutPacked64: {sym | bias << 8, f}
    const uint8_t *sym;      // kLutGeneric: slot -> symbol
    const uint2 *dec;        //              symbol -> {f, cum}
    uint32_t mask;
    uint32_t sb;

    // returns the symbol in the low byte
    __device__ __forceinline__ uint32_t pop(uint32_t &x) const {
        const uint32_t sb = SBC ? static_cast<uint32_t>(SBC) : this->sb;
        const uint32_t slot = x & (SBC ? (1u << SBC) - 1u : mask);
        if (KIND == kLutPacked32) {
            // h = (x >> sb) - 4096; e >> 8 = bias + f * 4096, so
            // f * h + (e >> 8) = f * (x >> sb) + bias with no field mask,
            // and the symbol is e's low byte (stored as is). The integer ALU
            // pipe is the decoder's busiest; this keeps work off it.
            const uint32_t h = (x >> sb) - 4096u;
            const uint32_t e = packed[slot];
            x = (e >> 20) * h + (e >> 8);
            return e;
        } else if (KIND == kLutPacked64) {
            const uint2 e = packed64[slot];
            x = e.y * (x >> sb) + (e.x >> 8);
            return e.x;
        } else {
            const uint32_t s = sym[slot];
            const uint2 d = dec[s];
            x = d.x * (x >> sb) + slot - d.y;
            return s;
        }
    }
};

// ---------------------------------------------------------------------------
// Sinks: what happens to the decoded bytes (decode fused into
// its consumer). The decoder stages each 32-symbol group in a per-warp
// shared buffer and hands complete blocks to the sink -- 512 bytes per
// fast-path batch, 256-byte halves and a final partial block on the generic
// path -- always at chunk positions that are multiples of the block size.
// StoreSink writes them to HBM (the plain decoder); any other sink consumes
// them in registers and the decoded bytes never reach HBM.
// ---------------------------------------------------------------------------
struct StoreSink {
    uint8_t *out;
    uint8_t *out_k;
    uint8_t *run;  // next512's lane pointer (running: no per-batch address math)
    __device__ __forceinline__ void begin(int64_t, int64_t cbase, int lane) {
        out_k = out + cbase;
        run = out_k + 16 * lane;
    }
    // the fast path's consecutive 512-byte blocks from the chunk start
    __device__ __forceinline__ void next512(const uint8_t *buf, int lane) {
        const uint4 o = reinterpret_cast<const uint4 *>(buf)[lane];
        asm volatile("st.global.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(run), "r"(o.x), "r"(o.y),
                     "r"(o.z), "r"(o.w) : "memory");
        run += 512;
    }
    __device__ __forceinline__ void block512(const uint8_t *buf, int64_t pos, int lane) {
        const uint4 o = reinterpret_cast<const uint4 *>(buf)[lane];
        asm volatile("st.global.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(out_k + pos + 16 * lane),
                     "r"(o.x), "r"(o.y), "r"(o.z), "r"(o.w) : "memory");
    }
    __device__ __forceinline__ void block256(const uint8_t *buf, int64_t pos, int lane) {
        const uint2 o = reinterpret_cast<const uint2 *>(buf)[lane];
        asm volatile("st.global.v2.u32 [%0], {%1, %2};" ::"l"(out_k + pos + 8 * lane), "r"(o.x),
                     "r"(o.y) : "memory");
    }
    __device__ __forceinline__ void tail(const uint8_t *buf, int64_t pos, int64_t end, int lane) {
        for (int64_t i = pos + lane; i < end; i += 32) out_k[i] = buf[i - pos];
    }
    __device__ __forceinline__ void end(int64_t, int64_t, int) {}
};

// zlib-compatible Adler-32 of every decoded chunk (one u32 per chunk), e.g.
// to verify a stream on the device without materialising it. With bytes
// b_0..b_{n-1}: A = 1 + S, B = n + n S - sum(i b_i) (mod 65521), S = sum(b_i);
// each lane sums its bytes and their positions (dp4a: 4 bytes per op), the
// warp reduces once per chunk.
struct Adler32Sink {
    uint32_t *adler;
    unsigned long long s1, si;  // per-lane partial sums (exact for chunks <= 2^27 B: < 2^62)
    int64_t rpos;               // next512's lane position
    __device__ __forceinline__ void begin(int64_t, int64_t, int lane) {
        s1 = si = 0;
        rpos = 16 * lane;
    }
    __device__ __forceinline__ void words(const uint32_t *w, int nw, int64_t pos0) {
        uint32_t t1 = 0, tj = 0;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            if (q < nw) {
                const uint32_t b = static_cast<uint32_t>(__dp4a(w[q], 0x01010101u, 0u));
                t1 += b;
                tj += static_cast<uint32_t>(__dp4a(w[q], 0x03020100u, 0u)) + 4u * q * b;
            }
        }
        s1 += t1;
        si += static_cast<unsigned long long>(pos0) * t1 + tj;
    }
    __device__ __forceinline__ void block512(const uint8_t *buf, int64_t pos, int lane) {
        const uint4 o = reinterpret_cast<const uint4 *>(buf)[lane];
        const uint32_t w[4] = {o.x, o.y, o.z, o.w};
        words(w, 4, pos + 16 * lane);
    }
    __device__ __forceinline__ void next512(const uint8_t *buf, int lane) {
        const uint4 o = reinterpret_cast<const uint4 *>(buf)[lane];
        const uint32_t w[4] = {o.x, o.y, o.z, o.w};
        words(w, 4, rpos);
        rpos += 512;
    }
    __device__ __forceinline__ void block256(const uint8_t *buf, int64_t pos, int lane) {
        const uint2 o = reinterpret_cast<const uint2 *>(buf)[lane];
        const uint32_t w[4] = {o.x, o.y, 0u, 0u};
        words(w, 2, pos + 8 * lane);
    }
    __device__ __forceinline__ void tail(const uint8_t *buf, int64_t pos, int64_t end, int lane) {
        for (int64_t i = pos + lane; i < end; i += 32) {
            const uint32_t b = buf[i - pos];
            s1 += b;
            si += static_cast<unsigned long long>(i) * b;
        }
    }
    __device__ __forceinline__ void end(int64_t k, int64_t len, int lane) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            s1 += __shfl_xor_sync(0xffffffffu, s1, o);
            si += __shfl_xor_sync(0xffffffffu, si, o);
        }
        if (lane == 0) {
            constexpr unsigned long long P = 65521ull;
            const unsigned long long n = static_cast<unsigned long long>(len);
            const unsigned long long a = (1ull + s1) % P;
            const unsigned long long b = ((n % P) * a + P - si % P) % P;  // n(1+S) - SI
            adler[k] = static_cast<uint32_t>(b << 16 | a);
        }
    }
};

// Shared memory per CTA: [align pad][W rings x 2 KB][W obufs x 512 B][LUT].
__host__ __device__ constexpr size_t decode_warp_smem() { return kRingAllocBytes + kObufBytes; }

// Not inlined: with both LUT forms inlined into one kernel the packed
// path's schedule degrades (~8% slower decode, measured); as a call each
// body keeps its own register allocation.
// SMALL: the instantiation for power-of-two N < 32 (512/N-group batches);
// a separate body so the N = 32 batch loop keeps its own schedule.
template <int KIND, class Sink, bool SMALL, int SBC = 0>
__device__ __noinline__ void
decode_warp_body(const uint16_t *__restrict__ payload, ChunkDir dir,
                 const uint32_t *__restrict__ states, int64_t n, int64_t chunk_len,
                 int64_t n_chunks, int n_lanes, const TableDev *__restrict__ tab,
                 Sink sink, uint64_t *__restrict__ consumed,
                 uint32_t *__restrict__ final_states, DStatus *__restrict__ status,
                 DecodeTrace trace, uint8_t *smem, int sb) {
    const uint32_t m = 1u << sb;
    const int nw = blockDim.x >> 5;
    uint8_t *lut_base = smem + nw * (kRingAllocBytes + kObufBytes);

    // ---- stage the lookup tables in shared memory ------------------------
    Lut<KIND, SBC> lut;
    lut.mask = m - 1u;
    lut.sb = static_cast<uint32_t>(sb);
    if (KIND == kLutPacked32) {
        uint32_t *p = reinterpret_cast<uint32_t *>(lut_base);
        for (uint32_t i = threadIdx.x; i < m; i += blockDim.x) p[i] = tab->packed[i];
        lut.packed = p;
    } else if (KIND == kLutPacked64) {
        uint4 *p = reinterpret_cast<uint4 *>(lut_base);
        const uint4 *src = reinterpret_cast<const uint4 *>(tab->packed64);
        for (uint32_t i = threadIdx.x; i < m / 2; i += blockDim.x) p[i] = src[i];
        lut.packed64 = reinterpret_cast<const uint2 *>(lut_base);
    } else {
        uint2 *d = reinterpret_cast<uint2 *>(lut_base);
        uint8_t *s = lut_base + kMaxSym * sizeof(uint2);
        for (uint32_t i = threadIdx.x; i < kMaxSym; i += blockDim.x) d[i] = tab->dec[i];
        if (m >= 4) {
            const uint32_t *src = reinterpret_cast<const uint32_t *>(tab->slot_sym);
            uint32_t *dst = reinterpret_cast<uint32_t *>(s);
            for (uint32_t i = threadIdx.x; i < m / 4; i += blockDim.x) dst[i] = src[i];
        } else {
            for (uint32_t i = threadIdx.x; i < m; i += blockDim.x) s[i] = tab->slot_sym[i];
        }
        lut.dec = d;
        lut.sym = s;
    }
    __syncthreads();

    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    uint16_t *ring = reinterpret_cast<uint16_t *>(smem + wib * kRingAllocBytes);
    const uint32_t ring_addr = smem_addr(ring);
    uint8_t *obuf = smem + nw * kRingAllocBytes + wib * kObufBytes;
    const uint32_t lt = lanemask_lt();
    // popc(mk & lanemask_lt) == popc(mk << (32 - lane)): a multiply (FMA
    // pipe) instead of a LOP3 (ALU pipe); lane 0 multiplies by 0
    const uint32_t lt_mul = lane ? 1u << (32 - lane) : 0u;
    // 2 as an opaque register: keeps the cursor updates as IMADs (FMA pipe)
    uint32_t two;
    asm volatile("mov.u32 %0, 2;" : "=r"(two));
    // warps that own chunks: a launch over few chunks adds staging-only
    // warps (the LUT copy above) that stop here
    int64_t nwk = (n_chunks + gridDim.x - 1) / gridDim.x;
    if (nwk > nw) nwk = nw;
    if (wib >= nwk) return;
    const int64_t warps_total = static_cast<int64_t>(gridDim.x) * nwk;

    for (int64_t k = static_cast<int64_t>(blockIdx.x) * nwk + wib; k < n_chunks;
         k += warps_total) {
        const int64_t cbase = k * chunk_len;
        const int64_t len = (n - cbase) < chunk_len ? (n - cbase) : chunk_len;
        uint64_t woff, wlen;
        dir.span(k, cbase, len, woff, wlen);
        const uint32_t delta = static_cast<uint32_t>(woff & 7u);
        SegSrc src{payload + (woff & ~7ull), wlen + delta};
#pragma unroll
        for (uint32_t s = 0; s < 4; ++s) {
            issue_segment(ring, src, s, lane);
            cp_async_commit();
        }
        cp_async_wait<2>();
        __syncwarp();

        uint64_t cur = 0;            // ring segment holding the read cursor
        uint64_t v = delta;          // read cursor in words from src.g
        uint32_t x = lane < n_lanes ? states[k * n_lanes + lane] : 0u;
        sink.begin(k, cbase, lane);
        int64_t base = 0;

        if ((SMALL || n_lanes == 32) && !trace.states && !trace.stats) {
            // ---------------- fast path: batches of 512 symbols -------------
            // (kBatch groups of 32 lanes, or 512/N groups of N < 32 lanes for
            // the power-of-two widths.) A batch reads <= 512 words, i.e. up
            // to two segments past the one holding the cursor, so the ring
            // runs one segment deeper here (wait<1>: everything but the
            // newest segment has landed).
            const int64_t full = len / (32 * kBatch);
            uint32_t vb = static_cast<uint32_t>(v) << 1;  // byte cursor (mod 2^32)
            uint32_t seg_cur = 0;                          // vb >> 9 of the cursor
            uint32_t next_seg = 4;                         // next segment to issue
            // segments wholly inside the payload are issued without bounds
            // arithmetic from a running source pointer (the common case)
            const uint64_t segs_whole = src.avail / kSegWords;
            const uint16_t *seg_g = src.g + 4 * kSegWords + lane * 8;
            cp_async_wait<1>();
            __syncwarp();
            // 32-bit batch counter (full < 2^29 for any message that fits in
            // HBM); the word cursor v is rebuilt after the loop from the
            // segment count (v / kSegWords == next_seg - 4) and vb's low bits
            for (uint32_t b = 0; b < static_cast<uint32_t>(full); ++b) {
                const uint32_t vb0 = vb;
                // shared address of the cursor; the batch reads < 512 words
                // past it, which the mirrored slots keep contiguous
                const uint32_t a0 = ring_addr + (vb & (kRingBytes - 2));
                uint32_t a = a0;
                if (!SMALL) {
#pragma unroll
                    for (int g = 0; g < kBatch; ++g) {
                        const uint32_t s = lut.pop(x);
                        const bool need = x < kLow;
                        const uint32_t mk = __ballot_sync(0xffffffffu, need);
                        // every lane loads (one wavefront either way), then selects
                        const uint32_t w = lds_u16(mad_lo(__popc(mk * lt_mul), two, a));
                        x = need ? x * 65536u + w : x;
                        a = mad_lo(__popc(mk), two, a);
                        obuf[g * 32 + lane] = static_cast<uint8_t>(s);
                    }
                } else {
                    // N < 32: lanes >= N idle (their state stays 0, never
                    // renormalises, never stores); 512/N groups per batch
                    const bool on = lane < n_lanes;
                    uint8_t *op = obuf + lane;
                    for (int gb = 0; gb < 512; gb += 16 * n_lanes) {
#pragma unroll
                        for (int g = 0; g < 16; ++g) {
                            const uint32_t s = lut.pop(x);
                            const bool need = on && x < kLow;
                            const uint32_t mk = __ballot_sync(0xffffffffu, need);
                            const uint32_t w = lds_u16(mad_lo(__popc(mk * lt_mul), two, a));
                            x = need ? x * 65536u + w : x;
                            a = mad_lo(__popc(mk), two, a);
                            if (on) *op = static_cast<uint8_t>(s);
                            op += n_lanes;
                        }
                    }
                }
                vb = vb0 + (a - a0);
                __syncwarp();
                sink.next512(obuf, lane);
                const uint32_t seg = (vb >> 9) & 0x7FFFFFu;
                if (seg != seg_cur) {  // one or two segments were finished
                    do {
                        seg_cur = (seg_cur + 1) & 0x7FFFFFu;
                        if (next_seg < segs_whole) {
                            uint16_t *dst = ring + (next_seg & 3u) * kSegWords + lane * 8;
                            cp_async16(dst, seg_g, 16u);
                            if ((next_seg & 3u) < 2u) cp_async16(dst + kRingWords, seg_g, 16u);
                        } else {
                            issue_segment(ring, src, next_seg, lane);
                        }
                        ++next_seg;
                        seg_g += kSegWords;
                        cp_async_commit();
                    } while (seg_cur != seg);
                    cp_async_wait<1>();
                }
                __syncwarp();
            }
            cur = next_seg - 4;  // == v / kSegWords; cur + 1.. cur + 3 issued
            v = cur * kSegWords + ((vb >> 1) & (kSegWords - 1));
            base = full * (32 * kBatch);
        }
        // ---------------- generic per-group loop (any N <= 32, tails) ------
        bool truncated = (v - delta) > wlen;
        uint32_t most = 0;  // stats: most digits one symbol needed (rans.py:305-309 loop)
        for (; !truncated && base < len; base += n_lanes) {
            const int64_t left = len - base;
            const int active = left < n_lanes ? static_cast<int>(left) : n_lanes;
            const bool on = lane < active;
            uint32_t s = 0;
            if (on) s = lut.pop(x);
            const bool need = on && x < kLow;
            const uint32_t mk = __ballot_sync(0xffffffffu, need);
            const uint32_t cnt = __popc(mk);
            if (v - delta + cnt > wlen) {
                truncated = true;
                break;
            }
            if (need)
                x = (x << 16) | ring_load(ring_addr, static_cast<uint32_t>(v + __popc(mk & lt)) << 1);
            v += cnt;
            if (trace.stats && need) most = max(most, x < kLow ? 2u : 1u);
            if (trace.states) {
                const int64_t gi = base / n_lanes;
                if (lane < n_lanes) trace.states[gi * n_lanes + lane] = x;
                if (lane == 0) trace.pos[gi] = v - delta;
            }
            if (on) obuf[(base + lane) & (kObufBytes - 1)] = static_cast<uint8_t>(s);
            const int64_t nb = base + active;
            if ((nb >> 8) != (base >> 8)) {  // a 256-byte half is complete
                __syncwarp();
                const int64_t blk = base >> 8;
                sink.block256(obuf + (blk & 1) * kObufHalf, blk << 8, lane);
                __syncwarp();
            }
            const uint64_t seg = v / kSegWords;
            if (seg != cur) {  // segment cur-1 fully read: refill its slot
                cur = seg;
                __syncwarp();
                issue_segment(ring, src, static_cast<uint32_t>(cur + 3), lane);
                cp_async_commit();
                cp_async_wait<2>();
                __syncwarp();
            }
        }
        if (truncated && lane == 0)
            atomicMin(&status->trunc_stream, static_cast<unsigned long long>(k));
        {   // bytes of the last partial 256-byte block (all groups done so far)
            const int64_t end = truncated ? base : len;
            __syncwarp();
            const int64_t tail0 = (end >> 8) << 8;
            const uint8_t *half = obuf + ((end >> 8) & 1) * kObufHalf;
            sink.tail(half, tail0, end, lane);
            sink.end(k, end, lane);
        }
        if (trace.groups && lane == 0) trace.groups[k] = (base < len ? base : len + n_lanes - 1) / n_lanes;
        if (lane == 0 && consumed) consumed[k] = v - delta;
        if (trace.stats) {
            most = __reduce_max_sync(0xffffffffu, most);
            if (lane == 0 && most) atomicMax(&status->max_digits, most);
        }
        if (final_states && lane < n_lanes) final_states[k * n_lanes + lane] = x;
        cp_async_wait<0>();
        __syncwarp();
    }
}

template <int MAXKIND, class Sink, bool SMALL>
__device__ __forceinline__ void
decode_warp_dispatch(const uint16_t *__restrict__ payload, ChunkDir dir,
                     const uint32_t *__restrict__ states, int64_t n, int64_t chunk_len,
                     int64_t n_chunks, int n_lanes, const TableDev *__restrict__ tab, Sink out,
                     uint64_t *__restrict__ consumed, uint32_t *__restrict__ final_states,
                     DStatus *__restrict__ status, DecodeTrace trace, uint8_t *smem, int sb) {
    if (MAXKIND == kLutPacked32 && !SMALL && sb == 12 && (tab->flags & kTabPacked))
        decode_warp_body<kLutPacked32, Sink, SMALL, 12>(payload, dir, states, n, chunk_len,
                                                        n_chunks, n_lanes, tab, out, consumed,
                                                        final_states, status, trace, smem, sb);
    else if (MAXKIND == kLutPacked3264 && !SMALL && sb == 14 && (tab->flags & kTabPacked))
        decode_warp_body<kLutPacked32, Sink, SMALL, 14>(payload, dir, states, n, chunk_len,
                                                        n_chunks, n_lanes, tab, out, consumed,
                                                        final_states, status, trace, smem, sb);
    else if (allows32(MAXKIND) && (tab->flags & kTabPacked))
        decode_warp_body<kLutPacked32, Sink, SMALL>(payload, dir, states, n, chunk_len,
                                                    n_chunks, n_lanes, tab, out, consumed,
                                                    final_states, status, trace, smem, sb);
    else if (allows64(MAXKIND) && (tab->flags & kTabPacked64))
        decode_warp_body<kLutPacked64, Sink, SMALL>(payload, dir, states, n, chunk_len,
                                                    n_chunks, n_lanes, tab, out, consumed,
                                                    final_states, status, trace, smem, sb);
    else
        decode_warp_body<kLutGeneric, Sink, SMALL>(payload, dir, states, n, chunk_len,
                                                   n_chunks, n_lanes, tab, out, consumed,
                                                   final_states, status, trace, smem, sb);
}

// MAXKIND: the packed form this launch's shared memory was sized for (it
// also fits the two-lookup form); the device table's flags pick which one
// runs (a single-symbol sb=12 table has f = 4096, which the 12-bit field of
// the 32-bit entry cannot hold).
template <int MAXKIND, class Sink>
__global__ void __launch_bounds__(1024)
decode_warp_kernel(const uint16_t *__restrict__ payload, ChunkDir dir,
                   const uint32_t *__restrict__ states, int64_t n, int64_t chunk_len,
                   int64_t n_chunks, int n_lanes, const TableDev *__restrict__ tab,
                   Sink out, uint64_t *__restrict__ consumed,
                   uint32_t *__restrict__ final_states, DStatus *__restrict__ status,
                   int launch_sb, DecodeTrace trace) {
    extern __shared__ __align__(16) uint8_t smem[];
    const int sb = static_cast<int>(tab->scale_bits);
    if (sb != launch_sb || tab->status != ILANS_OK) {
        if (threadIdx.x == 0) status->value_error = 1;  // smem was sized for launch_sb
        return;
    }
    if (n_lanes < 32 && (n_lanes & (n_lanes - 1)) == 0)
        decode_warp_dispatch<MAXKIND, Sink, true>(payload, dir, states, n, chunk_len,
                                                  n_chunks, n_lanes, tab, out, consumed,
                                                  final_states, status, trace, smem, sb);
    else
        decode_warp_dispatch<MAXKIND, Sink, false>(payload, dir, states, n, chunk_len,
                                                   n_chunks, n_lanes, tab, out, consumed,
                                                   final_states, status, trace, smem, sb);
}

// N < 32 not a power of two (floor(256/N)-group batches): a separate body
// and kernel, so the N = 32 / power-of-two kernels keep their code.
template <int KIND, class Sink>
__device__ __noinline__ void
decode_warp_body_np2(const uint16_t *__restrict__ payload, ChunkDir dir,
                 const uint32_t *__restrict__ states, int64_t n, int64_t chunk_len,
                 int64_t n_chunks, int n_lanes, const TableDev *__restrict__ tab,
                 Sink sink, uint64_t *__restrict__ consumed,
                 uint32_t *__restrict__ final_states, DStatus *__restrict__ status,
                 DecodeTrace trace, uint8_t *smem, int sb) {
    constexpr int MODE = 2;  // N < 32, not a power of two
    constexpr bool SMALL = true;
    const uint32_t m = 1u << sb;
    const int nw = blockDim.x >> 5;
    uint8_t *lut_base = smem + nw * (kRingAllocBytes + kObufBytes);

    // ---- stage the lookup tables in shared memory ------------------------
    Lut<KIND> lut;
    lut.mask = m - 1u;
    lut.sb = static_cast<uint32_t>(sb);
    if (KIND == kLutPacked32) {
        uint32_t *p = reinterpret_cast<uint32_t *>(lut_base);
        for (uint32_t i = threadIdx.x; i < m; i += blockDim.x) p[i] = tab->packed[i];
        lut.packed = p;
    } else if (KIND == kLutPacked64) {
        uint4 *p = reinterpret_cast<uint4 *>(lut_base);
        const uint4 *src = reinterpret_cast<const uint4 *>(tab->packed64);
        for (uint32_t i = threadIdx.x; i < m / 2; i += blockDim.x) p[i] = src[i];
        lut.packed64 = reinterpret_cast<const uint2 *>(lut_base);
    } else {
        uint2 *d = reinterpret_cast<uint2 *>(lut_base);
        uint8_t *s = lut_base + kMaxSym * sizeof(uint2);
        for (uint32_t i = threadIdx.x; i < kMaxSym; i += blockDim.x) d[i] = tab->dec[i];
        if (m >= 4) {
            const uint32_t *src = reinterpret_cast<const uint32_t *>(tab->slot_sym);
            uint32_t *dst = reinterpret_cast<uint32_t *>(s);
            for (uint32_t i = threadIdx.x; i < m / 4; i += blockDim.x) dst[i] = src[i];
        } else {
            for (uint32_t i = threadIdx.x; i < m; i += blockDim.x) s[i] = tab->slot_sym[i];
        }
        lut.dec = d;
        lut.sym = s;
    }
    __syncthreads();

    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    uint16_t *ring = reinterpret_cast<uint16_t *>(smem + wib * kRingAllocBytes);
    const uint32_t ring_addr = smem_addr(ring);
    uint8_t *obuf = smem + nw * kRingAllocBytes + wib * kObufBytes;
    const uint32_t lt = lanemask_lt();
    // popc(mk & lanemask_lt) == popc(mk << (32 - lane)): a multiply (FMA
    // pipe) instead of a LOP3 (ALU pipe); lane 0 multiplies by 0
    const uint32_t lt_mul = lane ? 1u << (32 - lane) : 0u;
    // 2 as an opaque register: keeps the cursor updates as IMADs (FMA pipe)
    uint32_t two;
    asm volatile("mov.u32 %0, 2;" : "=r"(two));
    // warps that own chunks: a launch over few chunks adds staging-only
    // warps (the LUT copy above) that stop here
    int64_t nwk = (n_chunks + gridDim.x - 1) / gridDim.x;
    if (nwk > nw) nwk = nw;
    if (wib >= nwk) return;
    const int64_t warps_total = static_cast<int64_t>(gridDim.x) * nwk;

    for (int64_t k = static_cast<int64_t>(blockIdx.x) * nwk + wib; k < n_chunks;
         k += warps_total) {
        const int64_t cbase = k * chunk_len;
        const int64_t len = (n - cbase) < chunk_len ? (n - cbase) : chunk_len;
        uint64_t woff, wlen;
        dir.span(k, cbase, len, woff, wlen);
        const uint32_t delta = static_cast<uint32_t>(woff & 7u);
        SegSrc src{payload + (woff & ~7ull), wlen + delta};
#pragma unroll
        for (uint32_t s = 0; s < 4; ++s) {
            issue_segment(ring, src, s, lane);
            cp_async_commit();
        }
        cp_async_wait<2>();
        __syncwarp();

        uint64_t cur = 0;            // ring segment holding the read cursor
        uint64_t v = delta;          // read cursor in words from src.g
        uint32_t x = lane < n_lanes ? states[k * n_lanes + lane] : 0u;
        sink.begin(k, cbase, lane);
        int64_t base = 0;

        if ((SMALL || n_lanes == 32) && !trace.states && !trace.stats) {
            // ---------------- fast path: batches of 512 symbols -------------
            // (kBatch groups of 32 lanes, or 512/N groups of N < 32 lanes for
            // the power-of-two widths.) A batch reads <= 512 words, i.e. up
            // to two segments past the one holding the cursor, so the ring
            // runs one segment deeper here (wait<1>: everything but the
            // newest segment has landed).
            // N < 32 not a power of two: batches of floor(256/N) groups
            // (<= 256 symbols), flushed by 256-byte halves like the loop below
            const int64_t spb = MODE == 2 ? int64_t(256 / n_lanes) * n_lanes : int64_t(32 * kBatch);
            const int64_t full = len / spb;
            uint32_t vb = static_cast<uint32_t>(v) << 1;  // byte cursor (mod 2^32)
            uint32_t seg_cur = 0;                          // vb >> 9 of the cursor
            uint32_t next_seg = 4;                         // next segment to issue
            // segments wholly inside the payload are issued without bounds
            // arithmetic from a running source pointer (the common case)
            const uint64_t segs_whole = src.avail / kSegWords;
            const uint16_t *seg_g = src.g + 4 * kSegWords + lane * 8;
            cp_async_wait<1>();
            __syncwarp();
            for (int64_t b = 0; b < full; ++b) {
                const uint32_t vb0 = vb;
                // shared address of the cursor; the batch reads < 512 words
                // past it, which the mirrored slots keep contiguous
                const uint32_t a0 = ring_addr + (vb & (kRingBytes - 2));
                uint32_t a = a0;
                if (!SMALL) {
#pragma unroll
                    for (int g = 0; g < kBatch; ++g) {
                        const uint32_t s = lut.pop(x);
                        const bool need = x < kLow;
                        const uint32_t mk = __ballot_sync(0xffffffffu, need);
                        // every lane loads (one wavefront either way), then selects
                        const uint32_t w = lds_u16(mad_lo(__popc(mk * lt_mul), two, a));
                        x = need ? x * 65536u + w : x;
                        a = mad_lo(__popc(mk), two, a);
                        obuf[g * 32 + lane] = static_cast<uint8_t>(s);
                    }
                } else if (MODE == 2) {
                    const int gpb = 256 / n_lanes;
                    const bool on = lane < n_lanes;
                    uint32_t oi = static_cast<uint32_t>(b * spb) + lane;  // obuf index mod 512
#pragma unroll 4
                    for (int g = 0; g < gpb; ++g) {
                        const uint32_t s = lut.pop(x);
                        const bool need = on && x < kLow;
                        const uint32_t mk = __ballot_sync(0xffffffffu, need);
                        const uint32_t w = lds_u16(mad_lo(__popc(mk * lt_mul), two, a));
                        x = need ? x * 65536u + w : x;
                        a = mad_lo(__popc(mk), two, a);
                        if (on) obuf[oi & (kObufBytes - 1)] = static_cast<uint8_t>(s);
                        oi += n_lanes;
                    }
                } else {
                    // N < 32: lanes >= N idle (their state stays 0, never
                    // renormalises, never stores); 512/N groups per batch
                    const bool on = lane < n_lanes;
                    uint8_t *op = obuf + lane;
                    for (int gb = 0; gb < 512; gb += 16 * n_lanes) {
#pragma unroll
                        for (int g = 0; g < 16; ++g) {
                            const uint32_t s = lut.pop(x);
                            const bool need = on && x < kLow;
                            const uint32_t mk = __ballot_sync(0xffffffffu, need);
                            const uint32_t w = lds_u16(mad_lo(__popc(mk * lt_mul), two, a));
                            x = need ? x * 65536u + w : x;
                            a = mad_lo(__popc(mk), two, a);
                            if (on) *op = static_cast<uint8_t>(s);
                            op += n_lanes;
                        }
                    }
                }
                vb = vb0 + (a - a0);
                __syncwarp();
                if (MODE != 2) {
                    sink.block512(obuf, b * (32 * kBatch), lane);
                } else {
                    const int64_t blk = (b * spb) >> 8;
                    if (((b * spb + spb) >> 8) != blk)  // a 256-byte half is complete
                        sink.block256(obuf + (blk & 1) * kObufHalf, blk << 8, lane);
                }
                v += (vb - vb0) >> 1;
                const uint32_t seg = (vb >> 9) & 0x7FFFFFu;
                if (seg != seg_cur) {  // one or two segments were finished
                    do {
                        seg_cur = (seg_cur + 1) & 0x7FFFFFu;
                        if (next_seg < segs_whole) {
                            uint16_t *dst = ring + (next_seg & 3u) * kSegWords + lane * 8;
                            cp_async16(dst, seg_g, 16u);
                            if ((next_seg & 3u) < 2u) cp_async16(dst + kRingWords, seg_g, 16u);
                        } else {
                            issue_segment(ring, src, next_seg, lane);
                        }
                        ++next_seg;
                        seg_g += kSegWords;
                        cp_async_commit();
                    } while (seg_cur != seg);
                    cp_async_wait<1>();
                }
                __syncwarp();
            }
            cur = next_seg - 4;  // == v / kSegWords; cur + 1.. cur + 3 issued
            base = full * spb;
        }
        // ---------------- generic per-group loop (any N <= 32, tails) ------
        bool truncated = (v - delta) > wlen;
        uint32_t most = 0;  // stats: most digits one symbol needed (rans.py:305-309 loop)
        for (; !truncated && base < len; base += n_lanes) {
            const int64_t left = len - base;
            const int active = left < n_lanes ? static_cast<int>(left) : n_lanes;
            const bool on = lane < active;
            uint32_t s = 0;
            if (on) s = lut.pop(x);
            const bool need = on && x < kLow;
            const uint32_t mk = __ballot_sync(0xffffffffu, need);
            const uint32_t cnt = __popc(mk);
            if (v - delta + cnt > wlen) {
                truncated = true;
                break;
            }
            if (need)
                x = (x << 16) | ring_load(ring_addr, static_cast<uint32_t>(v + __popc(mk & lt)) << 1);
            v += cnt;
            if (trace.stats && need) most = max(most, x < kLow ? 2u : 1u);
            if (trace.states) {
                const int64_t gi = base / n_lanes;
                if (lane < n_lanes) trace.states[gi * n_lanes + lane] = x;
                if (lane == 0) trace.pos[gi] = v - delta;
            }
            if (on) obuf[(base + lane) & (kObufBytes - 1)] = static_cast<uint8_t>(s);
            const int64_t nb = base + active;
            if ((nb >> 8) != (base >> 8)) {  // a 256-byte half is complete
                __syncwarp();
                const int64_t blk = base >> 8;
                sink.block256(obuf + (blk & 1) * kObufHalf, blk << 8, lane);
                __syncwarp();
            }
            const uint64_t seg = v / kSegWords;
            if (seg != cur) {  // segment cur-1 fully read: refill its slot
                cur = seg;
                __syncwarp();
                issue_segment(ring, src, static_cast<uint32_t>(cur + 3), lane);
                cp_async_commit();
                cp_async_wait<2>();
                __syncwarp();
            }
        }
        if (truncated && lane == 0)
            atomicMin(&status->trunc_stream, static_cast<unsigned long long>(k));
        {   // bytes of the last partial 256-byte block (all groups done so far)
            const int64_t end = truncated ? base : len;
            __syncwarp();
            const int64_t tail0 = (end >> 8) << 8;
            const uint8_t *half = obuf + ((end >> 8) & 1) * kObufHalf;
            sink.tail(half, tail0, end, lane);
            sink.end(k, end, lane);
        }
        if (trace.groups && lane == 0) trace.groups[k] = (base < len ? base : len + n_lanes - 1) / n_lanes;
        if (lane == 0 && consumed) consumed[k] = v - delta;
        if (trace.stats) {
            most = __reduce_max_sync(0xffffffffu, most);
            if (lane == 0 && most) atomicMax(&status->max_digits, most);
        }
        if (final_states && lane < n_lanes) final_states[k * n_lanes + lane] = x;
        cp_async_wait<0>();
        __syncwarp();
    }
}

template <int MAXKIND, class Sink>
__global__ void __launch_bounds__(1024)
decode_warp_np2_kernel(const uint16_t *__restrict__ payload, ChunkDir dir,
                       const uint32_t *__restrict__ states, int64_t n, int64_t chunk_len,
                       int64_t n_chunks, int n_lanes, const TableDev *__restrict__ tab,
                       Sink out, uint64_t *__restrict__ consumed,
                       uint32_t *__restrict__ final_states, DStatus *__restrict__ status,
                       int launch_sb, DecodeTrace trace) {
    extern __shared__ __align__(16) uint8_t smem[];
    const int sb = static_cast<int>(tab->scale_bits);
    if (sb != launch_sb || tab->status != ILANS_OK) {
        if (threadIdx.x == 0) status->value_error = 1;  // smem was sized for launch_sb
        return;
    }
    if (allows32(MAXKIND) && (tab->flags & kTabPacked))
        decode_warp_body_np2<kLutPacked32, Sink>(payload, dir, states, n, chunk_len, n_chunks,
                                                 n_lanes, tab, out, consumed, final_states,
                                                 status, trace, smem, sb);
    else if (allows64(MAXKIND) && (tab->flags & kTabPacked64))
        decode_warp_body_np2<kLutPacked64, Sink>(payload, dir, states, n, chunk_len, n_chunks,
                                                 n_lanes, tab, out, consumed, final_states,
                                                 status, trace, smem, sb);
    else
        decode_warp_body_np2<kLutGeneric, Sink>(payload, dir, states, n, chunk_len, n_chunks,
                                                n_lanes, tab, out, consumed, final_states,
                                                status, trace, smem, sb);
}

// ---------------------------------------------------------------------------
// CTA-wide exclusive scan (blockDim multiple of 32, <= 1024)
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t block_excl_scan(uint32_t v, uint32_t *total,
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

// One CTA per stream; thread t owns lanes [t*k, min(N, t*k + k)), k <= 64.
__global__ void __launch_bounds__(1024)
decode_block_kernel(const uint16_t *__restrict__ payload, const uint64_t *__restrict__ offsets,
                    const uint32_t *__restrict__ states, int64_t n, int64_t chunk_len,
                    int n_lanes, const TableDev *__restrict__ tab, uint8_t *__restrict__ out,
                    uint64_t *__restrict__ consumed, uint32_t *__restrict__ final_states,
                    DStatus *__restrict__ status, uint32_t *__restrict__ ws_all,
                    DecodeTrace trace, int ws_in_smem) {
    __shared__ uint32_t scan_sh[32];
    // dynamic smem: dec[256] | slot -> symbol [2^sb] | lane states [N] (when
    // ws_in_smem; else they stay in the global scratch)
    extern __shared__ __align__(16) uint8_t bsm[];
    const int sb = static_cast<int>(tab->scale_bits);
    const uint32_t mask = (1u << sb) - 1u;
    uint2 *dec = reinterpret_cast<uint2 *>(bsm);
    uint8_t *slot_sym = bsm + kMaxSym * sizeof(uint2);
    for (int i = threadIdx.x; i < kMaxSym; i += blockDim.x) dec[i] = tab->dec[i];
    for (uint32_t i = threadIdx.x; i < (1u << sb); i += blockDim.x) slot_sym[i] = tab->slot_sym[i];
    const int64_t k = blockIdx.x;
    const int64_t cbase = k * chunk_len;
    const int64_t len = (n - cbase) < chunk_len ? (n - cbase) : chunk_len;
    const uint64_t woff = offsets[k];
    const uint64_t wlen = offsets[k + 1] - woff;
    const uint16_t *pay = payload + woff;
    uint32_t *ws = ws_in_smem
                       ? reinterpret_cast<uint32_t *>(slot_sym + ((size_t(1) << sb) + 15 & ~size_t(15)))
                       : ws_all + k * n_lanes;
    const int per = (n_lanes + blockDim.x - 1) / blockDim.x;
    const int lo = threadIdx.x * per;
    for (int l = lo; l < lo + per && l < n_lanes; ++l) ws[l] = states[k * n_lanes + l];
    __syncthreads();
    uint64_t pos = 0;
    bool truncated = false;
    int64_t base = 0;
    uint32_t most = 0;
    for (; base < len; base += n_lanes) {
        const int64_t left = len - base;
        const int active = left < n_lanes ? static_cast<int>(left) : n_lanes;
        const int hi = lo + per < active ? lo + per : active;
        uint64_t pend = 0;
        uint32_t cnt = 0;
        for (int l = lo; l < hi; ++l) {
            uint32_t x = ws[l];
            const uint32_t slot = x & mask;
            const uint32_t s = slot_sym[slot];
            const uint2 d = dec[s];
            x = d.x * (x >> sb) + slot - d.y;
            out[cbase + base + l] = static_cast<uint8_t>(s);
            ws[l] = x;
            if (x < kLow) {
                pend |= 1ull << (l - lo);
                ++cnt;
            }
        }
        uint32_t total;
        const uint32_t excl = block_excl_scan(cnt, &total, scan_sh);
        if (pos + total > wlen) {
            truncated = true;
            break;
        }
        uint32_t r = 0;
        while (pend) {
            const int j = __ffsll(static_cast<long long>(pend)) - 1;
            pend &= pend - 1;
            const int l = lo + j;
            ws[l] = (ws[l] << 16) | pay[pos + excl + r];
            ++r;
            if (trace.stats) most = max(most, ws[l] < kLow ? 2u : 1u);
        }
        pos += total;
        if (trace.states) {
            const int64_t gi = base / n_lanes;
            for (int l = lo; l < lo + per && l < n_lanes; ++l)
                trace.states[gi * n_lanes + l] = ws[l];
            if (threadIdx.x == 0) trace.pos[gi] = pos;
        }
    }
    if (most) atomicMax(&status->max_digits, most);
    if (threadIdx.x == 0) {
        if (truncated) atomicMin(&status->trunc_stream, static_cast<unsigned long long>(k));
        if (consumed) consumed[k] = pos;
        if (trace.groups) trace.groups[k] = (base < len ? base : len + n_lanes - 1) / n_lanes;
    }
    if (final_states)
        for (int l = lo; l < lo + per && l < n_lanes; ++l) final_states[k * n_lanes + l] = ws[l];
}

// 32 < N <= kWideMax, no trace: one warp per stream, each thread holds the
// states of lanes lane, 32 + lane, ... (S sub-groups of 32) in registers. All
// sub-groups of a group look up their symbols together; sub-group j's refill
// positions start after the counts of sub-groups 0..j-1 (lanes ascending: the
// reference's order), so a group costs about one N = 32 group plus S - 1
// more ballots / popcs.
constexpr int kWideMax = 256;  // beyond this the CTA kernel wins (measured)
template <int S>
__global__ void __launch_bounds__(32)
decode_wide_kernel(const uint16_t *__restrict__ payload, const uint64_t *__restrict__ offsets,
                   const uint32_t *__restrict__ states, int64_t n, int64_t chunk_len,
                   int n_lanes, const TableDev *__restrict__ tab, uint8_t *__restrict__ out,
                   uint64_t *__restrict__ consumed, uint32_t *__restrict__ final_states,
                   DStatus *__restrict__ status) {
    // dec[256] | slot [2^sb] | payload ring (as the warp kernel's)
    extern __shared__ __align__(16) uint8_t wsm[];
    const int lane = threadIdx.x;
    const uint32_t lt = lanemask_lt();
    const int sb = static_cast<int>(tab->scale_bits);
    const uint32_t mask = (1u << sb) - 1u;
    uint2 *dec = reinterpret_cast<uint2 *>(wsm);
    uint8_t *slot_sym = wsm + kMaxSym * sizeof(uint2);
    uint16_t *ring = reinterpret_cast<uint16_t *>(slot_sym + (((size_t(1) << sb) + 15) & ~size_t(15)));
    const uint32_t ring_addr = smem_addr(ring);
    for (int i = lane; i < kMaxSym; i += 32) dec[i] = tab->dec[i];
    for (uint32_t i = lane; i < (1u << sb); i += 32) slot_sym[i] = tab->slot_sym[i];
    const int64_t k = blockIdx.x;
    const int64_t cbase = k * chunk_len;
    const int64_t len = (n - cbase) < chunk_len ? (n - cbase) : chunk_len;
    const uint64_t woff = offsets[k];
    const uint64_t wlen = offsets[k + 1] - woff;
    const uint32_t delta = static_cast<uint32_t>(woff & 7u);
    // the payload streams through the shared ring (<= 256 words per group:
    // at most one segment per group)
    SegSrc src{payload + (woff & ~7ull), wlen + delta};
#pragma unroll
    for (uint32_t q = 0; q < 4; ++q) {
        issue_segment(ring, src, q, lane);
        cp_async_commit();
    }
    uint32_t x[S];
#pragma unroll
    for (int j = 0; j < S; ++j)
        x[j] = 32 * j + lane < n_lanes ? states[k * n_lanes + 32 * j + lane] : 0u;
    cp_async_wait<2>();
    __syncwarp();
    uint64_t pos = 0;
    uint64_t cur = 0;  // ring segment holding the cursor (delta + pos)
    bool truncated = false;
    uint8_t *o = out + cbase;
    for (int64_t base = 0; base < len; base += n_lanes) {
        const int active = (len - base) < n_lanes ? static_cast<int>(len - base) : n_lanes;
        // lookups unconditional (lanes past the group decode their stale
        // state and are masked below), so the S chains overlap
        uint32_t sy[S], y[S], mk[S];
        uint32_t cnt = 0;
#pragma unroll
        for (int j = 0; j < S; ++j) {
            const uint32_t slot = x[j] & mask;
            sy[j] = slot_sym[slot];
            const uint2 d = dec[sy[j]];
            y[j] = d.x * (x[j] >> sb) + slot - d.y;
        }
#pragma unroll
        for (int j = 0; j < S; ++j) {
            mk[j] = __ballot_sync(0xffffffffu, 32 * j + lane < active && y[j] < kLow);
            cnt += __popc(mk[j]);
        }
        if (pos + cnt > wlen) {
            truncated = true;
            break;
        }
        uint32_t c = static_cast<uint32_t>(delta + pos);
#pragma unroll
        for (int j = 0; j < S; ++j) {
            if ((mk[j] >> lane) & 1u)
                y[j] = (y[j] << 16) | ring_load(ring_addr, (c + __popc(mk[j] & lt)) << 1);
            c += __popc(mk[j]);
            const bool on = 32 * j + lane < active;
            x[j] = on ? y[j] : x[j];
            if (on) o[base + 32 * j + lane] = static_cast<uint8_t>(sy[j]);
        }
        pos += cnt;
        const uint64_t seg = (delta + pos) / kSegWords;
        if (seg != cur) {  // segment cur fully read: refill its slot
            cur = seg;
            __syncwarp();
            issue_segment(ring, src, static_cast<uint32_t>(cur + 3), lane);
            cp_async_commit();
            cp_async_wait<2>();
            __syncwarp();
        }
    }
    cp_async_wait<0>();
    __syncwarp();
    if (lane == 0) {
        if (truncated) atomicMin(&status->trunc_stream, static_cast<unsigned long long>(k));
        if (consumed) consumed[k] = pos;
    }
    if (final_states) {
#pragma unroll
        for (int j = 0; j < S; ++j)
            if (32 * j + lane < n_lanes) final_states[k * n_lanes + 32 * j + lane] = x[j];
    }
}

static size_t decode_lut_bytes(int scale_bits, int kind) {
    const size_t m = size_t(1) << scale_bits;
    size_t b = kind == kLutPacked32 ? m * 4
             : kind == kLutPacked64 || kind == kLutPacked3264 ? m * 8
                                    : kMaxSym * sizeof(uint2) + (m < 16 ? 16 : m);
    return (b + 15) & ~size_t(15);
}

// Per-chunk Adler-32 of bytes already in HBM (the unfused consumer: decode
// to HBM, then read the bytes back). One warp per chunk, 16 bytes per lane
// per step, the same sums as Adler32Sink.
__global__ void __launch_bounds__(256)
adler32_chunks_kernel(const uint8_t *__restrict__ data, int64_t n, int64_t chunk_len,
                      int64_t n_chunks, uint32_t *__restrict__ adler) {
    const int lane = threadIdx.x & 31;
    const int64_t warps_total = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
    for (int64_t k = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
         k < n_chunks; k += warps_total) {
        const int64_t cbase = k * chunk_len;
        const int64_t len = (n - cbase) < chunk_len ? (n - cbase) : chunk_len;
        Adler32Sink sink{adler, 0ull, 0ull};
        const int64_t full = len >> 9;
        for (int64_t b = 0; b < full; ++b)
            sink.block512(data + cbase + (b << 9), b << 9, lane);  // 16-byte aligned chunks
        sink.tail(data + cbase + (full << 9), full << 9, len, lane);
        sink.end(k, len, lane);
    }
}

template <class Sink>
static cudaError_t launch_decode_warp(const uint16_t *d_payload, ChunkDir dir,
                                     const uint32_t *d_states, int64_t n, int64_t chunk_len,
                                     int n_lanes, const TableDev *d_table, int scale_bits,
                                     bool packed, Sink sink, uint64_t *d_consumed,
                                     uint32_t *d_final_states, DStatus *d_status,
                                     cudaStream_t stream, DecodeTrace trace) {
    const int64_t n_chunks = (n + chunk_len - 1) / chunk_len;
    // the packed form this launch allows (the device table's flags decide
    // whether it runs; its shared memory always fits the two-lookup form too)
    const bool sb64 = scale_bits >= kPacked64MinBits && scale_bits <= kPacked64MaxBits;
    const bool sb32 = packed && scale_bits <= kPackedMaxBits;
    const int maxkind = sb32 && sb64 ? kLutPacked3264 : sb32 ? kLutPacked32
                      : sb64 ? kLutPacked64 : kLutGeneric;
    size_t lut = decode_lut_bytes(scale_bits, kLutGeneric);
    if (decode_lut_bytes(scale_bits, maxkind) > lut) lut = decode_lut_bytes(scale_bits, maxkind);
    // One CTA per SM with that SM's share of the streams (up to 28 warps;
    // 4096 chunks = one wave on 148 SMs): the warp scheduler is not fair
    // across CTAs, and co-resident CTAs finish far apart (encode.cu,
    // kEncMaxWarps); as one CTA the SM's warps finish together.
    const int64_t sms = sm_count();
    int warps = static_cast<int>((n_chunks + sms - 1) / sms);
    if (warps > 28) warps = 28;
    if (warps < 1) warps = 1;
    const size_t smem_cap = 227 * 1024;
    while (warps > 1 && lut + size_t(warps) * decode_warp_smem() > smem_cap) --warps;
    int64_t blocks = (n_chunks + warps - 1) / warps;
    // few chunks per CTA (single streams, small inputs): staging-only warps
    // help copy the LUT into shared memory, then exit (the kernel gives the
    // chunks to the first ceil(n_chunks / blocks) warps)
    const int cta_warps = warps < 8 && lut >= 4096 ? 8 : warps;
    const size_t smem = lut + size_t(cta_warps) * decode_warp_smem();
    const int64_t per_sm = static_cast<int64_t>(smem_cap / (smem + 1024));
    const int64_t max_blocks = sms * (per_sm < 1 ? 1 : per_sm);
    if (blocks > max_blocks) blocks = max_blocks;
    const unsigned g = static_cast<unsigned>(blocks);
    auto go = [&](auto kernel) {
        smem_limit(reinterpret_cast<const void *>(kernel), int(smem));
        kernel<<<g, cta_warps * 32, smem, stream>>>(d_payload, dir, d_states, n,
                                                chunk_len, n_chunks, n_lanes, d_table, sink,
                                                d_consumed, d_final_states, d_status,
                                                scale_bits, trace);
    };
    const bool np2 = n_lanes < 32 && (n_lanes & (n_lanes - 1)) != 0;
    if (maxkind == kLutPacked32) {
        if (np2) go(decode_warp_np2_kernel<kLutPacked32, Sink>);
        else go(decode_warp_kernel<kLutPacked32, Sink>);
    } else if (maxkind == kLutPacked3264) {
        if (np2) go(decode_warp_np2_kernel<kLutPacked3264, Sink>);
        else go(decode_warp_kernel<kLutPacked3264, Sink>);
    } else if (maxkind == kLutPacked64) {
        if (np2) go(decode_warp_np2_kernel<kLutPacked64, Sink>);
        else go(decode_warp_kernel<kLutPacked64, Sink>);
    } else {
        if (np2) go(decode_warp_np2_kernel<kLutGeneric, Sink>);
        else go(decode_warp_kernel<kLutGeneric, Sink>);
    }
    ilans_note_launch();
    return cudaGetLastError();
}

cudaError_t launch_decode(const uint16_t *d_payload, const uint64_t *d_word_offsets,
                          const uint32_t *d_states, int64_t n, int64_t chunk_len, int n_lanes,
                          const TableDev *d_table, int scale_bits, bool packed,
                          uint8_t *d_out, uint64_t *d_consumed, uint32_t *d_final_states,
                          DStatus *d_status, uint32_t *d_lane_ws, cudaStream_t stream,
                          DecodeTrace trace, const uint32_t *d_slot_words) {
    if (n <= 0) return cudaSuccess;
    const int64_t n_chunks = (n + chunk_len - 1) / chunk_len;
    if (d_slot_words && n_lanes > 32) return cudaErrorInvalidValue;  // chunked streams: N <= 32
    if (n_lanes > 32 && n_lanes <= kWideMax && !trace.states && !trace.stats) {
        const size_t smem = kMaxSym * sizeof(uint2) +
                            (((size_t(1) << scale_bits) + 15) & ~size_t(15)) + kRingAllocBytes;
        auto kernel = n_lanes <= 64 ? decode_wide_kernel<2>
                    : n_lanes <= 128 ? decode_wide_kernel<4> : decode_wide_kernel<8>;
        smem_limit(reinterpret_cast<const void *>(kernel), int(smem));
        kernel<<<static_cast<unsigned>(n_chunks), 32, smem, stream>>>(
            d_payload, d_word_offsets, d_states, n, chunk_len, n_lanes, d_table, d_out,
            d_consumed, d_final_states, d_status);
        ilans_note_launch();
        return cudaGetLastError();
    }
    if (n_lanes > 32) {
        const int threads = n_lanes >= 1024 ? 1024 : ((n_lanes + 31) / 32) * 32;
        // tables (and the lane states when they fit) in shared memory
        const size_t tabs = kMaxSym * sizeof(uint2) + (((size_t(1) << scale_bits) + 15) & ~size_t(15));
        const int ws_smem = tabs + size_t(n_lanes) * 4 <= size_t(200) * 1024;
        const size_t smem = tabs + (ws_smem ? size_t(n_lanes) * 4 : 0);
        smem_limit(reinterpret_cast<const void *>(decode_block_kernel), int(smem));
        decode_block_kernel<<<static_cast<unsigned>(n_chunks), threads, smem, stream>>>(
            d_payload, d_word_offsets, d_states, n, chunk_len, n_lanes, d_table, d_out,
            d_consumed, d_final_states, d_status, d_lane_ws, trace, ws_smem);
        ilans_note_launch();
        return cudaGetLastError();
    }
    return launch_decode_warp(d_payload, ChunkDir{d_word_offsets, d_slot_words}, d_states, n,
                              chunk_len, n_lanes, d_table,
                              scale_bits, packed, StoreSink{d_out, nullptr}, d_consumed,
                              d_final_states, d_status, stream, trace);
}

cudaError_t launch_adler32_chunks(const uint8_t *d_data, int64_t n, int64_t chunk_len,
                                  uint32_t *d_adler, cudaStream_t stream) {
    if (n <= 0) return cudaSuccess;
    const int64_t n_chunks = (n + chunk_len - 1) / chunk_len;
    int64_t blocks = (n_chunks + 7) / 8;
    const int64_t max_blocks = int64_t(sm_count()) * 16;
    if (blocks > max_blocks) blocks = max_blocks;
    adler32_chunks_kernel<<<static_cast<unsigned>(blocks), 256, 0, stream>>>(d_data, n, chunk_len,
                                                                              n_chunks, d_adler);
    ilans_note_launch();
    return cudaGetLastError();
}

cudaError_t launch_decode_adler32(const uint16_t *d_payload, const uint64_t *d_word_offsets,
                                  const uint32_t *d_states, int64_t n, int64_t chunk_len,
                                  int n_lanes, const TableDev *d_table, int scale_bits,
                                  uint32_t *d_adler, uint64_t *d_consumed, DStatus *d_status,
                                  cudaStream_t stream, const uint32_t *d_slot_words) {
    if (n <= 0) return cudaSuccess;
    if (n_lanes > 32) return cudaErrorInvalidValue;
    return launch_decode_warp(d_payload, ChunkDir{d_word_offsets, d_slot_words}, d_states, n,
                              chunk_len,
                              n_lanes, d_table,
                              scale_bits, scale_bits <= kPackedMaxBits,
                              Adler32Sink{d_adler, 0ull, 0ull}, d_consumed, nullptr, d_status,
                              stream, DecodeTrace{nullptr, nullptr, nullptr, 0});
}

}  // namespace ilans
