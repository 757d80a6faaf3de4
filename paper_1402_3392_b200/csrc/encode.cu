// encode.cu -- word16 interleaved-rANS encoders for sm_100a, plus framing.
//
// Replaces _core.encode_interleaved_u16 (_core.pyx:14-43). The reference
// walks the message backwards (i = n-1 .. 0, lane = i mod N), spills one
// 16-bit digit when x >= f << (32 - sb), then pushes
// x -> (x / f << sb) + cum + x % f, stacking digits from the end of an
// n-word buffer. Group form (lanes.encode_step / packed_store,
// lanes.py:124-181; encode_lanes_full, lanes.py:235-252): the tail group
// first, then full groups backwards; inside a group the spilling lanes'
// digits occupy the next popc(mask) stack slots so that, read forwards, they
// appear in ascending lane order -- lane i writes at
// top - popc(mask) + popc(mask & lanemask_lt(i)).
//
// Warp kernel (N <= 32): one warp per chunk, one CTA per SM holding all of
// the SM's chunks (<= 28 warps; see kEncMaxWarps); message bytes are staged
// backwards into a per-warp 2 KB shared ring by cp.async (4 x 512 B
// segments); the per-symbol records live in shared memory and x / f is an
// exact multiply-high (Granlund-Montgomery), no hardware divide. For N = 32
// the 512-byte blocks run as unrolled 16-group batches with the fast record
// (common.cuh EncFast: 8 bytes, sb <= 13; EncFast12: sb = 14) when the table
// allows it, else the 33-bit-magic record. Block kernel (N > 32): one CTA
// per stream with a CTA-wide scan over spill counts.
//
// Framing: chunk k's payload sits at scratch[k*C + len_k - w_k, k*C + len_k);
// an exclusive scan of w_k gives word offsets and a compaction kernel packs
// the payloads back to back (SURVEY A12 chunk framing).
#include <type_traits>

#include "common.cuh"
#include "kernels.cuh"

namespace ilans {

constexpr int kInSeg = 512;            // bytes per cp.async warp-copy
constexpr int kInRing = 4 * kInSeg;    // 2 KB per warp

template <typename Idx>
__device__ __forceinline__ void issue_msg_segment(uint8_t *ring, const uint8_t *g, Idx len,
                                                  Idx seg, int lane) {
    const Idx b0 = seg * kInSeg + lane * 16;
    uint32_t bytes = 0;
    if (seg >= 0 && b0 < len) bytes = (len - b0) >= 16 ? 16u : static_cast<uint32_t>(len - b0);
    const uint8_t *src = bytes ? g + b0 : g;
    cp_async16(ring + (static_cast<uint32_t>(seg) & 3u) * kInSeg + lane * 16, src, bytes);
}

// One CTA per SM holding all of that SM's streams (up to 28 warps: 4096
// streams in one wave on 148 SMs). The warp scheduler is not fair across
// CTAs: with 7 CTAs of 4 warps per SM the first warps finished at 56% of the
// kernel time and the last at 100% (%globaltimer per warp), so each SM ran
// its last ~40% with ever fewer warps to hide latency; as one CTA per SM the
// same 28 warps finish together (320 -> 269 us at config 2; 2 CTAs of 14
// warps per SM are worse than either, 365 us).
constexpr int kEncMaxWarps = 28;
constexpr int kOutRing = 1024;   // per-warp staging ring for spilled words (2 KB)
constexpr uint32_t kOutRingBytes = kOutRing * 2;

// dynamic shared memory: enc[256] | encf x 16 | encz x 32 | W message rings |
// pad | W spill rings
// Bank-private copies of the fast records: entry e of copy c sits at
// e * copies + c, and lane l reads copy l % copies, so a warp's record loads
// never conflict whatever the symbols (one LDS.64 = 2 wavefronts, one LDS.32
// = 1; a single copy cost ~2.6 extra wavefronts per group at config 2, the
// encoder's shared-memory pipe then ~0.9 busy).
constexpr int kEncfCopies = 16;  // 8-byte records: a half-warp per wavefront
constexpr int kEnczCopies = 32;
constexpr int kEncqCopies = 8;   // 16-byte records (QUAD): a quarter-warp per wavefront
static_assert(kEncqCopies * sizeof(uint4) == kEncfCopies * sizeof(uint2) &&
                  kEncqCopies * sizeof(uint4) == kEnczCopies * sizeof(uint32_t),
              "the QUAD copies reuse the fast-record regions");
__host__ __device__ constexpr size_t encode_smem_bytes(int warps) {
    return kMaxSym * sizeof(uint2) + size_t(kEncfCopies) * kMaxSym * sizeof(uint2) +
           size_t(kEnczCopies) * kMaxSym * sizeof(uint32_t) + size_t(warps) * kInRing +
           kOutRingBytes + size_t(warps) * kOutRingBytes;
}

__device__ __forceinline__ uint32_t lds_u8(uint32_t addr) {
    uint16_t v;
    asm volatile("ld.shared.u8 %0, [%1];" : "=h"(v) : "r"(addr));
    return v;
}

__device__ __forceinline__ void sts16(uint32_t addr, uint32_t v) {
    asm volatile("st.shared.u16 [%0], %1;" ::"r"(addr), "h"(static_cast<uint16_t>(v)));
}

// One group's spill step in PTX: the spill predicate feeds the ballot and
// the predicated store / shift directly (as C++ the compiler computed it
// twice and moved the shifted state through a temporary), and the store
// address is computed unconditionally (predicated temporaries cost SELs).
//   TEST 0 (EncFast):   spill = (~x | (2^t - 1)) < Z   (carry of (x & ~(2^t-1)) + Z)
//   TEST 1 (EncFast12): spill = (x | (2^t - 1)) >= Y
// ON: lanes with on == 0 never spill (N < 32). topb is the ring byte cursor
// (decremented by two per spilled word); the spilled lanes store their low
// 16 bits at topb_new + 2 * (spilling lanes below them), ring-wrapped.
template <int TEST, bool ON>
__device__ __forceinline__ void spill_group(uint32_t &x, uint32_t &topb, uint32_t lowm,
                                            uint32_t key, uint32_t on, uint32_t lt_mul,
                                            uint32_t ring_addr, uint32_t neg2, uint32_t two) {
    static_assert(kOutRingBytes == 2048, "ring mask below");
    if (TEST == 0 && !ON)
        asm("{\n\t.reg .pred p;\n\t.reg .b32 t, mk, c, cl, ad;\n\t"
            "lop3.b32 t, %0, %2, 0, 0xcf;\n\t"
            "setp.lt.u32 p, t, %3;\n\t"
            "vote.sync.ballot.b32 mk, p, 0xffffffff;\n\t"
            "popc.b32 c, mk;\n\t"
            "mad.lo.u32 %1, c, %6, %1;\n\t"
            "mul.lo.u32 cl, mk, %4;\n\t"
            "popc.b32 cl, cl;\n\t"
            "mad.lo.u32 ad, cl, %7, %1;\n\t"
            "lop3.b32 ad, ad, 0x7fe, %5, 0xea;\n\t"
            "@p st.shared.u16 [ad], %0;\n\t"
            "@p shr.b32 %0, %0, 16;\n\t}"
            : "+r"(x), "+r"(topb)
            : "r"(lowm), "r"(key), "r"(lt_mul), "r"(ring_addr), "r"(neg2), "r"(two)
            : "memory");
    else if (TEST == 0)
        asm("{\n\t.reg .pred p, q;\n\t.reg .b32 t, mk, c, cl, ad;\n\t"
            "lop3.b32 t, %0, %2, 0, 0xcf;\n\t"
            "setp.ne.u32 q, %8, 0;\n\t"
            "setp.lt.and.u32 p, t, %3, q;\n\t"
            "vote.sync.ballot.b32 mk, p, 0xffffffff;\n\t"
            "popc.b32 c, mk;\n\t"
            "mad.lo.u32 %1, c, %6, %1;\n\t"
            "mul.lo.u32 cl, mk, %4;\n\t"
            "popc.b32 cl, cl;\n\t"
            "mad.lo.u32 ad, cl, %7, %1;\n\t"
            "lop3.b32 ad, ad, 0x7fe, %5, 0xea;\n\t"
            "@p st.shared.u16 [ad], %0;\n\t"
            "@p shr.b32 %0, %0, 16;\n\t}"
            : "+r"(x), "+r"(topb)
            : "r"(lowm), "r"(key), "r"(lt_mul), "r"(ring_addr), "r"(neg2), "r"(two), "r"(on)
            : "memory");
    else if (!ON)
        asm("{\n\t.reg .pred p;\n\t.reg .b32 t, mk, c, cl, ad;\n\t"
            "or.b32 t, %0, %2;\n\t"
            "setp.ge.u32 p, t, %3;\n\t"
            "vote.sync.ballot.b32 mk, p, 0xffffffff;\n\t"
            "popc.b32 c, mk;\n\t"
            "mad.lo.u32 %1, c, %6, %1;\n\t"
            "mul.lo.u32 cl, mk, %4;\n\t"
            "popc.b32 cl, cl;\n\t"
            "mad.lo.u32 ad, cl, %7, %1;\n\t"
            "lop3.b32 ad, ad, 0x7fe, %5, 0xea;\n\t"
            "@p st.shared.u16 [ad], %0;\n\t"
            "@p shr.b32 %0, %0, 16;\n\t}"
            : "+r"(x), "+r"(topb)
            : "r"(lowm), "r"(key), "r"(lt_mul), "r"(ring_addr), "r"(neg2), "r"(two)
            : "memory");
    else
        asm("{\n\t.reg .pred p, q;\n\t.reg .b32 t, mk, c, cl, ad;\n\t"
            "or.b32 t, %0, %2;\n\t"
            "setp.ne.u32 q, %8, 0;\n\t"
            "setp.ge.and.u32 p, t, %3, q;\n\t"
            "vote.sync.ballot.b32 mk, p, 0xffffffff;\n\t"
            "popc.b32 c, mk;\n\t"
            "mad.lo.u32 %1, c, %6, %1;\n\t"
            "mul.lo.u32 cl, mk, %4;\n\t"
            "popc.b32 cl, cl;\n\t"
            "mad.lo.u32 ad, cl, %7, %1;\n\t"
            "lop3.b32 ad, ad, 0x7fe, %5, 0xea;\n\t"
            "@p st.shared.u16 [ad], %0;\n\t"
            "@p shr.b32 %0, %0, 16;\n\t}"
            : "+r"(x), "+r"(topb)
            : "r"(lowm), "r"(key), "r"(lt_mul), "r"(ring_addr), "r"(neg2), "r"(two), "r"(on)
            : "memory");
}

// The 16-byte records' push (EncQuad, XQ = EncQuadX: exact 33-bit magic).
template <bool XQ>
__device__ __forceinline__ uint32_t quad_push(uint32_t x, const uint4 &a) {
    uint32_t q = __umulhi(x, a.x);
    if (XQ)  // q = (q + x) >> l as a 33-bit sum
        asm("{\n\t.reg .u32 lo, hi;\n\tadd.cc.u32 lo, %1, %2;\n\taddc.u32 hi, 0, 0;\n\t"
            "shf.r.wrap.b32 %0, lo, hi, %3;\n\t}"
            : "=r"(q) : "r"(q), "r"(x), "r"(a.y));
    else
        asm("shf.r.wrap.b32 %0, %1, %2, %3;" : "=r"(q) : "r"(q), "r"(0u), "r"(a.y));
    return a.z * q + (x + a.w);
}

// The N = 32 fast loop's spill step with the words stored straight to HBM
// (no staging ring, no drains). The chunk's scratch region never straddles
// a 4 GiB boundary here (checked by the caller), so the address is
// {topb, hi} with a constant high word: topb is the low word of the stack
// top's byte address, moved down by 2 per spilled word; spilling lane i
// stores at topb_new + 2 * (spilling lanes below it). A group's <= 32 words
// are contiguous: one coalesced request per group.
template <int TEST>
__device__ __forceinline__ void spill_group_g(uint32_t &x, uint32_t &topb, uint32_t hi,
                                              uint32_t lowm, uint32_t key, uint32_t lt_mul,
                                              uint32_t neg2, uint32_t two) {
    if (TEST == 0)
        asm("{\n\t.reg .pred p;\n\t.reg .b32 t, mk, c, cl, al;\n\t.reg .b64 ad;\n\t"
            "lop3.b32 t, %0, %3, 0, 0xcf;\n\t"
            "setp.lt.u32 p, t, %4;\n\t"
            "vote.sync.ballot.b32 mk, p, 0xffffffff;\n\t"
            "popc.b32 c, mk;\n\t"
            "mad.lo.u32 %1, c, %6, %1;\n\t"
            "mul.lo.u32 cl, mk, %5;\n\t"
            "popc.b32 cl, cl;\n\t"
            "mad.lo.u32 al, cl, %7, %1;\n\t"
            "mov.b64 ad, {al, %2};\n\t"
            "@p st.global.u16 [ad], %0;\n\t"
            "@p shr.b32 %0, %0, 16;\n\t}"
            : "+r"(x), "+r"(topb)
            : "r"(hi), "r"(lowm), "r"(key), "r"(lt_mul), "r"(neg2), "r"(two)
            : "memory");
    else
        asm("{\n\t.reg .pred p;\n\t.reg .b32 t, mk, c, cl, al;\n\t.reg .b64 ad;\n\t"
            "or.b32 t, %0, %3;\n\t"
            "setp.ge.u32 p, t, %4;\n\t"
            "vote.sync.ballot.b32 mk, p, 0xffffffff;\n\t"
            "popc.b32 c, mk;\n\t"
            "mad.lo.u32 %1, c, %6, %1;\n\t"
            "mul.lo.u32 cl, mk, %5;\n\t"
            "popc.b32 cl, cl;\n\t"
            "mad.lo.u32 al, cl, %7, %1;\n\t"
            "mov.b64 ad, {al, %2};\n\t"
            "@p st.global.u16 [ad], %0;\n\t"
            "@p shr.b32 %0, %0, 16;\n\t}"
            : "+r"(x), "+r"(topb)
            : "r"(hi), "r"(lowm), "r"(key), "r"(lt_mul), "r"(neg2), "r"(two)
            : "memory");
}

// Spilled words are staged in a per-warp shared ring (2 KB aligned, so an
// address is base | (byte_offset & mask)) indexed by their final scratch
// position w & 1023, and written to HBM as aligned 16-byte blocks. `flushed`
// starts at len rounded up to 8 words: the padding words past len land in
// the scratch slack / next chunk's untouched head and are never read.
// flush() writes the complete blocks of [roundup8(top), flushed); finish()
// writes the last < 8 words [top, roundup8(top)) one by one.
template <typename Idx>
struct SpillStage {
    uint16_t *ring;      // generic pointer to the ring
    uint32_t ring_addr;  // shared-window address of the ring (2 KB aligned)
    uint16_t *out;       // chunk's scratch region in HBM
    Idx flushed;         // words [flushed, len) are in HBM (flushed % 8 == 0)

    __device__ __forceinline__ void put(Idx w, uint32_t v) {
        sts16(ring_addr | ((static_cast<uint32_t>(w) << 1) & (kOutRingBytes - 2)), v);
    }

    __device__ __forceinline__ void flush(Idx top, int lane) {
        __syncwarp();
        const Idx lo = (top + 7) & ~Idx(7);
        for (Idx blk = lo + Idx(lane) * 8; blk < flushed; blk += 256)
            *reinterpret_cast<uint4 *>(out + blk) =
                *reinterpret_cast<const uint4 *>(ring + (blk & (kOutRing - 1)));
        if (lo < flushed) flushed = lo;
        __syncwarp();
    }

    // Fast-path drain: whole 512-word blocks [flushed - 512, flushed), two
    // 16-byte stores per lane, while at least 512 final words are pending
    // (keeps pending < 512, so a 512-symbol batch -- at most 512 spills --
    // cannot wrap the 1024-word ring).
    __device__ __forceinline__ void drain(Idx top, int lane) {
        while (flushed - top >= 512) {
            __syncwarp();
            const uint32_t wb = (static_cast<uint32_t>(flushed) - 512u + lane * 8u) << 1;
            uint4 lo, hi;
            asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                         : "=r"(lo.x), "=r"(lo.y), "=r"(lo.z), "=r"(lo.w)
                         : "r"(ring_addr | (wb & (kOutRingBytes - 1))));
            asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                         : "=r"(hi.x), "=r"(hi.y), "=r"(hi.z), "=r"(hi.w)
                         : "r"(ring_addr | ((wb + 512u) & (kOutRingBytes - 1))));
            uint16_t *d = out + (flushed - 512) + lane * 8;
            *reinterpret_cast<uint4 *>(d) = lo;
            *reinterpret_cast<uint4 *>(d + 256) = hi;
            flushed -= 512;
        }
    }

    __device__ __forceinline__ void finish(Idx top, int lane) {
        flush(top, lane);
        for (Idx w = top + lane; w < flushed; w += 32) out[w] = ring[w & (kOutRing - 1)];
        flushed = top;
    }
};

// Idx: chunk-local index type (int for chunks < 2^30 bytes, the chunked
// format's case; long long only for huge single-stream calls).
// F12: the sb = 14 instantiation (12-byte fast records); the other one
// carries the 8-byte fast loop, so neither pays for the other's registers.
// MODE 0: N = 32; 1: power-of-two N < 32 (512/N-group batches with the
// fast records); 2: other N < 32 (floor(256/N)-group batches with the fast
// records). Separate instantiations so the N = 32 loops keep their schedule.
// COVERED: the table was quantized from this message's own histogram, so
// every symbol in it has f >= 1 (rans.py:197-199) and the fast loops skip
// the per-group zero-frequency check (the AND of every record's M).
// QUAD (N = 32, int chunks): the fast loop runs on the 16-byte EncQuad
// records (8 bank-private copies in the fast-record region) whatever sb.
template <typename Idx, bool F12, int MODE, bool COVERED = false, bool QUAD = false>
__global__ void __launch_bounds__(kEncMaxWarps * 32, 1)
encode_warp_kernel(const uint8_t *__restrict__ msg, int64_t n, int64_t chunk_len,
                   int64_t n_chunks, int n_lanes, const TableDev *__restrict__ tab,
                   uint16_t *__restrict__ scratch, uint32_t *__restrict__ chunk_words,
                   uint32_t *__restrict__ states_out, DStatus *__restrict__ status) {
    extern __shared__ __align__(16) uint8_t esmem[];
    constexpr bool SMALL = MODE == 1;
    const int nw = blockDim.x >> 5;
    uint2 *enc = reinterpret_cast<uint2 *>(esmem);
    uint2 *encf_rep = enc + kMaxSym;  // EncFast {M, Z} / EncFast12 {M, Y}, x 16
    uint32_t *encz_rep = reinterpret_cast<uint32_t *>(encf_rep + kEncfCopies * kMaxSym);
    uint8_t *rings = reinterpret_cast<uint8_t *>(encz_rep + kEnczCopies * kMaxSym);
    uint16_t *oring_raw = reinterpret_cast<uint16_t *>(rings + nw * kInRing);
    const bool fast = !QUAD && !F12 && (tab->flags & kTabEncFast) != 0u;
    const bool fast12 = !QUAD && F12 && (tab->flags & kTabEncFast12) != 0u;
    const bool quad = QUAD && (tab->flags & kTabEncQuad) != 0u;
    // a symbol above m/2: the exact-magic 16-byte records (EncQuadX)
    const bool quadx = QUAD && !quad && (tab->flags & kTabEncQuadX) != 0u;
    for (int i = threadIdx.x; i < kMaxSym; i += blockDim.x) enc[i] = tab->enc[i];
    if (QUAD) {
        uint4 *q = reinterpret_cast<uint4 *>(quad ? static_cast<void *>(encf_rep)
                                                  : static_cast<void *>(encz_rep));
        const uint4 *src = quad ? tab->encq : tab->encqx;
        if (quad || quadx)
            for (int i = threadIdx.x; i < kEncqCopies * kMaxSym; i += blockDim.x)
                q[i] = src[i / kEncqCopies];
    } else {
        for (int i = threadIdx.x; i < kEncfCopies * kMaxSym; i += blockDim.x)
            encf_rep[i] = tab->encf[i / kEncfCopies];
        for (int i = threadIdx.x; i < kEnczCopies * kMaxSym; i += blockDim.x)
            encz_rep[i] = tab->encz[i / kEnczCopies];
    }
    __syncthreads();
    // this lane's copies: record of symbol s at encf[s * kEncfCopies]
    const uint2 *encf = encf_rep + (threadIdx.x & (kEncfCopies - 1));
    const uint32_t *encz = encz_rep + (threadIdx.x & (kEnczCopies - 1));
    const uint4 *encq = reinterpret_cast<const uint4 *>(encf_rep) + (threadIdx.x & (kEncqCopies - 1));
    const uint4 *encqx = reinterpret_cast<const uint4 *>(encz_rep) + (threadIdx.x & (kEncqCopies - 1));
    const EncCtx ctx(tab->scale_bits);
    const uint32_t lowm = ~0u >> tab->scale_bits;  // 2^t - 1, t = 32 - sb
    const uint32_t t_shift = 32u - tab->scale_bits;
    const uint32_t qoff = 1u << (27u - tab->scale_bits);  // 2^(t-5) (fast record)
    const int lane = threadIdx.x & 31;
    // popc(mk & lanemask_lt) == popc(mk * 2^(32 - lane)) (FMA pipe, not ALU)
    const uint32_t lt_mul = lane ? 1u << (32 - lane) : 0u;
    // opaque 2 (ptxas cannot fold it: n_chunks >= 0): keeps the cursor
    // arithmetic as IMADs (a known 2 becomes LEA / LEA.HI.X pairs)
    const uint32_t two = 2u + static_cast<uint32_t>(static_cast<unsigned long long>(n_chunks) >> 63);
    const uint32_t neg2 = 0u - two;
    const int wib = threadIdx.x >> 5;
    uint8_t *ring = rings + wib * kInRing;
    const uint32_t oraw = smem_addr(oring_raw);
    const uint32_t oalign = ((oraw + kOutRingBytes - 1) & ~(kOutRingBytes - 1)) - oraw;
    uint16_t *oring = oring_raw + oalign / 2 + wib * kOutRing;
    const uint32_t oring_addr = smem_addr(oring);
    const uint32_t lt = lanemask_lt();

    const int64_t warps_total = static_cast<int64_t>(gridDim.x) * nw;

    for (int64_t k = static_cast<int64_t>(blockIdx.x) * nw + wib; k < n_chunks;
         k += warps_total) {
        const int64_t cbase = k * chunk_len;
        const Idx len = static_cast<Idx>((n - cbase) < chunk_len ? (n - cbase) : chunk_len);
        const uint8_t *g = msg + cbase;
        SpillStage<Idx> st{oring, oring_addr, scratch + cbase, (len + 7) & ~Idx(7)};
        Idx cur = (len - 1) >> 9;
#pragma unroll
        for (int s = 0; s < 4; ++s) {
            issue_msg_segment(ring, g, len, cur - s, lane);
            cp_async_commit();
        }
        cp_async_wait<2>();
        __syncwarp();

        uint32_t x = kLow;
        Idx top = len;
        // N = 32: the 512-byte blocks below `full` run as unrolled batches of
        // 16 groups after the per-group loop has coded the tail [full*512, len)
        // (and power-of-two N < 32 with a fast record: 512/N groups each)
        const Idx full =
            (MODE == 1 ? (fast || fast12) : MODE == 0 && n_lanes == 32) ? (len >> 9) : 0;
        const Idx groups = (len + n_lanes - 1) / n_lanes;
        // MODE 2: the full groups below nbat * G run as batches of G groups
        const int G = MODE == 2 ? 256 / n_lanes : 1;
        const Idx nbat = MODE == 2 && (fast || fast12) ? (len / n_lanes) / G : 0;
        const Idx gstop = MODE == 2 ? nbat * G : SMALL ? full * (512 / n_lanes) : full << 4;
        bool bad = false;
        for (Idx gi = groups - 1; gi >= gstop; --gi) {
            const Idx base = gi * n_lanes;
            const Idx left = len - base;
            const int active = left < n_lanes ? static_cast<int>(left) : n_lanes;
            const Idx hi = (base + active - 1) >> 9;
            if (hi != cur) {  // segment cur fully consumed: recycle its slot
                cur = hi;
                __syncwarp();
                issue_msg_segment(ring, g, len, cur - 3, lane);
                cp_async_commit();
                cp_async_wait<2>();
                __syncwarp();
            }
            const bool on = lane < active;
            const uint2 e = enc[on ? ring[(base + lane) & (kInRing - 1)] : 0u];
            const uint32_t badmask = __ballot_sync(0xffffffffu, on && e.x == 0u);
            if (badmask) {
                if (lane == 0)
                    atomicMax(&status->unenc_index,
                              static_cast<long long>(cbase + base + 31 - __clz(badmask)));
                bad = true;
                break;
            }
            const bool spill = on && enc_spill(ctx, x, e);
            const uint32_t mk = __ballot_sync(0xffffffffu, spill);
            top -= __popc(mk);
            if (spill) {
                st.put(top + __popc(mk & lt), x & 0xFFFFu);
                x >>= 16;
            }
            if (on) x = enc_push(ctx, x, e);
            if (st.flushed - top >= 256) st.flush(top, lane);
        }
        // ---- N = 32 fast path: 512-byte blocks, backwards, 16 groups each ----
        // Segments cur .. cur-3 are in flight; batch b needs segment b and
        // keeps three younger ones in flight. Zero-frequency symbols are
        // detected once per batch (generic records) or once per chunk (fast
        // records); f = 0 only corrupts this chunk's scratch, which is then
        // discarded.
        Idx issued_lo = cur - 3;
        // fast records: AND of every record's M over the whole fast region;
        // bit 31 clears iff some symbol had f = 0 (checked once, after it)
        uint32_t macc = ~0u;
        // next segment to issue (issued_lo - 1): running source pointer and
        // the lane's 32-bit shared slot address (no per-batch conversions)
        const uint8_t *seg_src = g + (issued_lo - 1) * kInSeg + lane * 16;
        const uint32_t ring_sa = smem_addr(ring) + lane * 16;
        Idx b = full - 1;
        if (MODE == 0 && (fast || fast12 || quad || quadx) &&
            (QUAD || (reinterpret_cast<unsigned long long>(scratch + cbase) >> 32) ==
                         (reinterpret_cast<unsigned long long>(scratch + cbase + len) >> 32))) {
            // Pairs of blocks (32 groups) per iteration: one prefetch point
            // and one wait per 1 KB of message, records loaded one group
            // ahead straight across the two blocks, spilled words stored
            // straight to the scratch (spill_group_g). The per-group loop's
            // ring is written out first; an odd last block runs the same
            // body for 16 groups.
            st.finish(top, lane);
            const uint32_t blk_sa = smem_addr(ring) + lane;
            const unsigned long long gbase = reinterpret_cast<unsigned long long>(scratch + cbase);
            // byte address of the stack top as {topb, hi}: the 32-bit low
            // word moves, the high word is fixed while an iteration cannot
            // borrow from it (QUAD: topb >= the iteration's 2 KB of spills;
            // otherwise the WIDE body carries it -- a chunk whose slot
            // crosses a 4 GiB boundary stays on the fast path)
            const unsigned long long top0 = gbase + 2ull * static_cast<unsigned long long>(top);
            uint32_t hi = static_cast<uint32_t>(top0 >> 32);
            uint32_t topb = static_cast<uint32_t>(top0);
            auto body = [&](auto ng, auto wide, auto xq, uint32_t hi_sa, uint32_t lo_sa) {
                constexpr int NG = decltype(ng)::value;  // groups: 32 (hi, lo) or 16 (hi)
                constexpr bool WIDE = decltype(wide)::value;
                constexpr bool XQ = decltype(xq)::value;  // EncQuadX records
                const uint4 *rec = XQ ? encqx : encq;
                if constexpr (QUAD && WIDE) {
                    unsigned long long t64 = static_cast<unsigned long long>(hi) << 32 | topb;
#pragma unroll 1
                    for (int gg = NG - 1; gg >= 0; --gg) {
                        const uint32_t sym = lds_u8((gg >= kInSeg / 32 ? hi_sa : lo_sa) +
                                                    (gg % (kInSeg / 32)) * 32);
                        const uint4 a = rec[sym * kEncqCopies];
                        if (!COVERED) macc = XQ ? min(macc, a.y) : macc & a.x;
                        const bool p = (x | lowm) >= a.y;
                        const uint32_t mk = __ballot_sync(0xffffffffu, p);
                        t64 -= 2ull * static_cast<unsigned long long>(__popc(mk));
                        if (p) {
                            *reinterpret_cast<uint16_t *>(
                                t64 + 2ull * static_cast<unsigned long long>(__popc(mk & lt))) =
                                static_cast<uint16_t>(x);
                            x >>= 16;
                        }
                        x = quad_push<XQ>(x, a);
                    }
                    topb = static_cast<uint32_t>(t64);
                    hi = static_cast<uint32_t>(t64 >> 32);
                    return;
                }
                if (QUAD) {
                    uint32_t sym_n = lds_u8(hi_sa + (kInSeg / 32 - 1) * 32);
                    uint4 a_n = rec[sym_n * kEncqCopies];
                    sym_n = lds_u8(hi_sa + (kInSeg / 32 - 2) * 32);
#pragma unroll
                    for (int gg = NG - 1; gg >= 0; --gg) {
                        const uint4 a = a_n;  // {M, Y, m - f, bias}
                        if (gg > 0) {
                            a_n = rec[sym_n * kEncqCopies];
                            if (gg > 1) {
                                const int nx = gg - 2;
                                sym_n = lds_u8((nx >= kInSeg / 32 ? hi_sa : lo_sa) +
                                               (nx % (kInSeg / 32)) * 32);
                            }
                        }
                        if (!COVERED) macc = XQ ? min(macc, a.y) : macc & a.x;
                        spill_group_g<1>(x, topb, hi, lowm, a.y, lt_mul, neg2, two);
                        x = quad_push<XQ>(x, a);
                    }
                    return;
                }
                uint32_t sym_n = lds_u8(hi_sa + (kInSeg / 32 - 1) * 32);
                uint2 a_n = encf[sym_n * kEncfCopies];
                uint32_t z_n = F12 ? encz[sym_n * kEnczCopies] : 0u;
                sym_n = lds_u8(hi_sa + (kInSeg / 32 - 2) * 32);
#pragma unroll
                for (int gg = NG - 1; gg >= 0; --gg) {
                    const uint2 a = a_n;  // {M, Z} (F12: {M, Y})
                    const uint32_t z = z_n;
                    if (gg > 0) {
                        a_n = encf[sym_n * kEncfCopies];
                        if (F12) z_n = encz[sym_n * kEnczCopies];
                        if (gg > 1) {
                            const int nx = gg - 2;  // group two ahead
                            sym_n = lds_u8((nx >= kInSeg / 32 ? hi_sa : lo_sa) +
                                           (nx % (kInSeg / 32)) * 32);
                        }
                    }
                    if (!COVERED) macc &= a.x;
                    uint32_t q;
                    if (!F12) {
                        spill_group_g<0>(x, topb, hi, lowm, a.y, lt_mul, neg2, two);
                        q = __umulhi(x, a.x);
                        asm("shf.r.wrap.b32 %0, %1, %2, %3;" : "=r"(q) : "r"(q), "r"(0u), "r"(a.y));
                        x = (a.y >> t_shift) * (q - qoff) + (x + (a.y >> 5));
                    } else {
                        spill_group_g<1>(x, topb, hi, lowm, a.y, lt_mul, neg2, two);
                        q = __umulhi(x, a.x);
                        asm("shf.r.wrap.b32 %0, %1, %2, %3;" : "=r"(q) : "r"(q), "r"(0u), "r"(z));
                        x = q * (a.y & lowm) + (x + (z >> 16));
                    }
                }
            };
            // CHK: the chunk's slot crosses a 4 GiB boundary, so each
            // iteration checks whether it could borrow from the high word
            // (a separate copy of the loop: the others pay nothing for it)
            auto pairs = [&](auto chk, auto xq) {
            constexpr bool CHK = decltype(chk)::value;
            for (; b >= 1; b -= 2) {
                __syncwarp();  // every lane is done reading blocks b + 1, b + 2
                if (b >= 3 && issued_lo == b - 1) {
                    // steady state: segments b - 2 and b - 3 exist and are
                    // the next two to issue (no bounds or zero-fill selects)
                    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(
                                     ring_sa + ((static_cast<uint32_t>(b - 2) & 3u) << 9)),
                                 "l"(seg_src) : "memory");
                    cp_async_commit();
                    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(
                                     ring_sa + ((static_cast<uint32_t>(b - 3) & 3u) << 9)),
                                 "l"(seg_src - kInSeg) : "memory");
                    cp_async_commit();
                    seg_src -= 2 * kInSeg;
                    issued_lo = b - 3;
                } else {
#pragma unroll
                    for (int q = 2; q <= 3; ++q) {
                        const Idx sg = b - q;
                        if (sg < issued_lo) {
                            asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(
                                             ring_sa + ((static_cast<uint32_t>(sg) & 3u) << 9)),
                                         "l"(sg >= 0 ? seg_src : g), "r"(sg >= 0 ? 16u : 0u)
                                         : "memory");
                            seg_src -= kInSeg;
                            cp_async_commit();
                            issued_lo = sg;
                        }
                    }
                }
                cp_async_wait<2>();  // blocks b and b - 1 landed
                __syncwarp();
                const uint32_t sa_hi = blk_sa + ((static_cast<uint32_t>(b) & 3u) << 9);
                const uint32_t sa_lo = blk_sa + ((static_cast<uint32_t>(b - 1) & 3u) << 9);
                if (!CHK || topb >= 2u * 32u * 2u * (kInSeg / 32))
                    body(std::integral_constant<int, 2 * (kInSeg / 32)>{}, std::false_type{},
                         xq, sa_hi, sa_lo);
                else
                    body(std::integral_constant<int, 2 * (kInSeg / 32)>{}, std::true_type{},
                         xq, sa_hi, sa_lo);
            }
            cp_async_wait<0>();
            __syncwarp();
            if (b == 0) {  // an odd last block
                if (!QUAD || topb >= 32u * 2u * (kInSeg / 32))
                    body(std::integral_constant<int, kInSeg / 32>{}, std::false_type{}, xq,
                         blk_sa, blk_sa);
                else
                    body(std::integral_constant<int, kInSeg / 32>{}, std::true_type{}, xq,
                         blk_sa, blk_sa);
                b = -1;
            }
            };
            const bool cross = QUAD && (gbase >> 32) !=
                                           ((gbase + 2ull * static_cast<unsigned long long>(len)) >> 32);
            // one copy of the loop per (crossing, record form): only QUAD
            // kernels instantiate the EncQuadX copies
            if (QUAD && quadx) {
                if (cross) pairs(std::true_type{}, std::true_type{});
                else pairs(std::false_type{}, std::true_type{});
            } else if (cross) {
                pairs(std::true_type{}, std::false_type{});
            } else {
                pairs(std::false_type{}, std::false_type{});
            }
            top = static_cast<Idx>(
                ((static_cast<unsigned long long>(hi) << 32 | topb) - gbase) >> 1);
            st.flushed = top;  // every word below the ring's is in HBM already
        }
        for (; !bad && b >= 0; --b) {
            if (b - 3 < issued_lo) {  // segments below `full` are whole 512-byte blocks
                // every lane is done reading this slot (segment b + 1); below
                // segment 0 the copy reads nothing and zero-fills
                __syncwarp();
                const Idx sg = b - 3;
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(
                                 ring_sa + ((static_cast<uint32_t>(sg) & 3u) << 9)),
                             "l"(sg >= 0 ? seg_src : g), "r"(sg >= 0 ? 16u : 0u)
                             : "memory");
                seg_src -= kInSeg;
                cp_async_commit();
                issued_lo = sg;
            }
            cp_async_wait<3>();
            __syncwarp();
            const uint8_t *blk = ring + (static_cast<uint32_t>(b) & 3u) * kInSeg;
            uint32_t zero_f = 0;
            uint32_t topb = static_cast<uint32_t>(top) << 1;  // ring byte cursor
            const uint32_t topb0 = topb;
            if (SMALL) {
                // N < 32 (a power of two): 512/N groups of N lanes; lanes >= N
                // follow lane 0's symbol (a valid record for macc) and never
                // spill; their state is never stored
                const bool on = lane < n_lanes;
                const uint8_t *bp = blk + (kInSeg - n_lanes) + (on ? lane : 0);
                uint32_t sym_n = *bp;
                for (int gb = kInSeg / n_lanes - 1; gb >= 0; gb -= 16) {
#pragma unroll
                    for (int j = 0; j < 16; ++j) {
                        // next group's symbol one ahead (none after group 0,
                        // which ends the last outer step, gb == 15)
                        bp -= n_lanes;
                        const uint32_t sym = sym_n;
                        if (j < 15 || gb > 15) sym_n = *bp;
                        const uint2 a = encf[sym * kEncfCopies];
                        if (!COVERED) macc &= a.x;
                        uint32_t z = 0;
                        if (!F12) {
                            spill_group<0, true>(x, topb, lowm, a.y, on, lt_mul, oring_addr,
                                                 neg2, two);
                        } else {
                            z = encz[sym * kEnczCopies];
                            spill_group<1, true>(x, topb, lowm, a.y, on, lt_mul, oring_addr,
                                                 neg2, two);
                        }
                        uint32_t q = __umulhi(x, a.x);
                        if (!F12) {
                            asm("shf.r.wrap.b32 %0, %1, %2, %3;" : "=r"(q) : "r"(q), "r"(0u), "r"(a.y));
                            x = (a.y >> t_shift) * (q - qoff) + (x + (a.y >> 5));
                        } else {
                            asm("shf.r.wrap.b32 %0, %1, %2, %3;" : "=r"(q) : "r"(q), "r"(0u), "r"(z));
                            x = q * (a.y & lowm) + (x + (z >> 16));
                        }
                    }
                }
            } else if (fast) {
                // Records are loaded one group ahead of their use: the spill
                // stores go to shared memory too, so the compiler cannot
                // hoist a later group's loads above them by itself.
                uint32_t sym_n = blk[(kInSeg / 32 - 1) * 32 + lane];
                uint2 a_n = encf[sym_n * kEncfCopies];
                sym_n = blk[(kInSeg / 32 - 2) * 32 + lane];
#pragma unroll
                for (int gg = kInSeg / 32 - 1; gg >= 0; --gg) {
                    const uint2 a = a_n;  // {M, Z}
                    if (gg > 0) {
                        a_n = encf[sym_n * kEncfCopies];
                        if (gg > 1) sym_n = blk[(gg - 2) * 32 + lane];
                    }
                    if (!COVERED) macc &= a.x;
                    // spill iff carry out of (x & ~(2^t-1)) + Z
                    spill_group<0, false>(x, topb, lowm, a.y, 1u, lt_mul, oring_addr, neg2, two);
                    uint32_t q = __umulhi(x, a.x);
                    asm("shf.r.wrap.b32 %0, %1, %2, %3;" : "=r"(q) : "r"(q), "r"(0u), "r"(a.y));
                    x = (a.y >> t_shift) * (q - qoff) + (x + (a.y >> 5));
                }
            } else if (fast12) {
                uint32_t sym_n = blk[(kInSeg / 32 - 1) * 32 + lane];
                uint2 a_n = encf[sym_n * kEncfCopies];
                uint32_t z_n = encz[sym_n * kEnczCopies];
                sym_n = blk[(kInSeg / 32 - 2) * 32 + lane];
#pragma unroll
                for (int gg = kInSeg / 32 - 1; gg >= 0; --gg) {
                    const uint2 a = a_n;  // {M, Y}
                    const uint32_t z = z_n;
                    if (gg > 0) {
                        a_n = encf[sym_n * kEncfCopies];
                        z_n = encz[sym_n * kEnczCopies];
                        if (gg > 1) sym_n = blk[(gg - 2) * 32 + lane];
                    }
                    if (!COVERED) macc &= a.x;
                    spill_group<1, false>(x, topb, lowm, a.y, 1u, lt_mul, oring_addr, neg2, two);
                    uint32_t q = __umulhi(x, a.x);
                    asm("shf.r.wrap.b32 %0, %1, %2, %3;" : "=r"(q) : "r"(q), "r"(0u), "r"(z));
                    x = q * (a.y & lowm) + (x + (z >> 16));
                }
            } else {
#pragma unroll
            for (int gg = kInSeg / 32 - 1; gg >= 0; --gg) {
                const uint2 e = enc[blk[gg * 32 + lane]];
                zero_f |= e.x == 0u;
                const bool spill = enc_spill(ctx, x, e);
                const uint32_t mk = __ballot_sync(0xffffffffu, spill);
                topb -= __popc(mk) << 1;
                if (spill)
                    sts16(oring_addr | ((topb + (__popc(mk & lt) << 1)) & (kOutRingBytes - 2)),
                          x);
                x = spill ? x >> 16 : x;
                x = enc_push(ctx, x, e);
            }
            }
            top -= static_cast<Idx>((topb0 - topb) >> 1);
            if (!fast && !fast12 && __ballot_sync(0xffffffffu, zero_f)) {  // rare: highest bad index
                for (int gg = kInSeg / 32 - 1; gg >= 0; --gg) {
                    const uint32_t bm =
                        __ballot_sync(0xffffffffu, enc[blk[gg * 32 + lane]].x == 0u);
                    if (bm) {
                        if (lane == 0)
                            atomicMax(&status->unenc_index,
                                      static_cast<long long>(cbase) + b * kInSeg + gg * 32 +
                                          31 - __clz(bm));
                        break;
                    }
                }
                bad = true;
            }
            st.drain(top, lane);
        }
        if (MODE == 2) {
            // Batches of G groups (<= 256 bytes: inside the segment holding
            // their top byte and the one below, both landed after wait<2>),
            // records one group ahead; lanes >= N follow lane 0's symbol.
            const bool on = lane < n_lanes;
            const uint32_t lidx = on ? lane : 0u;
            for (Idx bt = nbat - 1; !bad && bt >= 0; --bt) {
                const Idx g_hi = bt * G + G - 1;
                const Idx hs = (g_hi * n_lanes + n_lanes - 1) >> 9;
                if (hs != cur) {  // segment cur fully consumed: recycle its slot
                    cur = hs;
                    __syncwarp();
                    issue_msg_segment(ring, g, len, cur - 3, lane);
                    cp_async_commit();
                    cp_async_wait<2>();
                    __syncwarp();
                }
                uint32_t topb = static_cast<uint32_t>(top) << 1;
                const uint32_t topb0 = topb;
                uint32_t ri = static_cast<uint32_t>(g_hi * n_lanes) + lidx;  // ring index
                uint32_t sym_n = ring[ri & (kInRing - 1)];
#pragma unroll 4
                for (int j = 0; j < G; ++j) {
                    const uint32_t sym = sym_n;
                    ri -= n_lanes;
                    if (j + 1 < G) sym_n = ring[ri & (kInRing - 1)];
                    const uint2 a = encf[sym * kEncfCopies];
                    if (!COVERED) macc &= a.x;
                    uint32_t z = 0;
                    if (!F12) {
                        spill_group<0, true>(x, topb, lowm, a.y, on, lt_mul, oring_addr, neg2,
                                             two);
                    } else {
                        z = encz[sym * kEnczCopies];
                        spill_group<1, true>(x, topb, lowm, a.y, on, lt_mul, oring_addr, neg2,
                                             two);
                    }
                    uint32_t q = __umulhi(x, a.x);
                    if (!F12) {
                        asm("shf.r.wrap.b32 %0, %1, %2, %3;" : "=r"(q) : "r"(q), "r"(0u), "r"(a.y));
                        x = (a.y >> t_shift) * (q - qoff) + (x + (a.y >> 5));
                    } else {
                        asm("shf.r.wrap.b32 %0, %1, %2, %3;" : "=r"(q) : "r"(q), "r"(0u), "r"(z));
                        x = q * (a.y & lowm) + (x + (z >> 16));
                    }
                }
                top -= static_cast<Idx>((topb0 - topb) >> 1);
                st.drain(top, lane);
            }
        }
        // (EncQuadX: the least Y of the region, 0 iff some f = 0)
        if ((fast || fast12 || quad || quadx) && !bad &&
            __ballot_sync(0xffffffffu, quadx ? macc == 0u : (macc >> 31) == 0u)) {
            // rare: some symbol of the fast region has f = 0 (its scratch is
            // garbage but stayed inside the chunk: at most 32 spills per
            // group). The highest offending index, as the reference's
            // backward walk meets it first (_core.pyx:33-34):
            const Idx fast_end = MODE == 2 ? nbat * G * n_lanes : full << 9;
            for (Idx i0 = fast_end - 32; i0 > -32; i0 -= 32) {
                const Idx i = i0 + lane;
                const uint32_t bm = __ballot_sync(0xffffffffu, i >= 0 && enc[g[i]].x == 0u);
                if (bm) {
                    if (lane == 0)
                        atomicMax(&status->unenc_index,
                                  static_cast<long long>(cbase + i0) + 31 - __clz(bm));
                    break;
                }
            }
            bad = true;
        }
        if (!bad) {
            st.finish(top, lane);
            if (lane == 0) chunk_words[k] = static_cast<uint32_t>(len - top);
            if (lane < n_lanes) states_out[k * n_lanes + lane] = x;
        }
        cp_async_wait<0>();
        __syncwarp();
    }
}

__device__ __forceinline__ uint32_t block_excl_scan_e(uint32_t v, uint32_t *total,
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

// One CTA per stream, N > 32: thread t owns lanes [t*k, t*k + k), k <= 64.
__global__ void __launch_bounds__(1024)
encode_block_kernel(const uint8_t *__restrict__ msg, int64_t n, int64_t chunk_len,
                    int n_lanes, const TableDev *__restrict__ tab,
                    uint16_t *__restrict__ scratch, uint32_t *__restrict__ chunk_words,
                    uint32_t *__restrict__ states_out, DStatus *__restrict__ status,
                    uint32_t *__restrict__ ws_all, int ws_in_smem, int stats) {
    __shared__ uint32_t scan_sh[32];
    __shared__ uint2 enc[kMaxSym];
    extern __shared__ __align__(16) uint32_t bws[];  // lane states, when they fit
    for (int i = threadIdx.x; i < kMaxSym; i += blockDim.x) enc[i] = tab->enc[i];
    __syncthreads();
    const EncCtx ctx(tab->scale_bits);
    const int64_t k = blockIdx.x;
    const int64_t cbase = k * chunk_len;
    const int64_t len = (n - cbase) < chunk_len ? (n - cbase) : chunk_len;
    const uint8_t *g = msg + cbase;
    uint16_t *out = scratch + cbase;
    uint32_t *ws = ws_in_smem ? bws : ws_all + k * n_lanes;
    const int per = (n_lanes + blockDim.x - 1) / blockDim.x;
    const int lo = threadIdx.x * per;
    for (int l = lo; l < lo + per && l < n_lanes; ++l) ws[l] = kLow;
    int64_t top = len;
    const int64_t groups = (len + n_lanes - 1) / n_lanes;
    bool bad = false;
    uint32_t most = 0;
    for (int64_t gi = groups - 1; gi >= 0; --gi) {
        const int64_t base = gi * n_lanes;
        const int64_t left = len - base;
        const int active = left < n_lanes ? static_cast<int>(left) : n_lanes;
        const int hi = lo + per < active ? lo + per : active;
        uint64_t spill = 0;
        uint32_t cnt = 0;
        long long my_bad = -1;
        for (int l = lo; l < hi; ++l) {
            const uint2 e = enc[g[base + l]];
            if (e.x == 0u) my_bad = base + l;
            else if (enc_spill(ctx, ws[l], e)) {
                spill |= 1ull << (l - lo);
                ++cnt;
            }
        }
        if (__syncthreads_or(my_bad >= 0)) {
            if (my_bad >= 0) atomicMax(&status->unenc_index, static_cast<long long>(cbase + my_bad));
            bad = true;
            break;
        }
        uint32_t total;
        const uint32_t excl = block_excl_scan_e(cnt, &total, scan_sh);
        uint32_t r = 0;
        while (spill) {
            const int j = __ffsll(static_cast<long long>(spill)) - 1;
            spill &= spill - 1;
            const int l = lo + j;
            out[top - total + excl + r] = static_cast<uint16_t>(ws[l] & 0xFFFFu);
            ws[l] >>= 16;
            ++r;
            if (stats) most = max(most, enc_spill(ctx, ws[l], enc[g[base + l]]) ? 2u : 1u);
        }
        top -= total;
        for (int l = lo; l < hi; ++l) {
            const uint2 e = enc[g[base + l]];
            ws[l] = enc_push(ctx, ws[l], e);
        }
    }
    if (most) atomicMax(&status->max_digits, most);
    if (!bad) {
        if (threadIdx.x == 0) chunk_words[k] = static_cast<uint32_t>(len - top);
        for (int l = lo; l < lo + per && l < n_lanes; ++l) states_out[k * n_lanes + l] = ws[l];
    }
}

// 32 < N <= kWideMaxE (and the instrumented N <= 32 calls): one warp per
// stream, each thread holds the states of lanes lane, 32 + lane, ... (S
// sub-groups of 32) in registers. A group is walked backwards: a higher
// sub-group's spills are stored above a lower one's, each sub-group in
// ascending lane order (the reference's payload order), all records looked
// up together. The message streams downwards through an 8 x 512 B shared
// ring (cp.async, issued six segments ahead; a symbol read from global
// memory one group ahead left the warp waiting a full memory latency per
// group). The message pointer is 16-byte aligned (both callers' buffers
// are), so each chunk's aligned base below it lies inside the message.
constexpr int kWideMaxE = 256;  // beyond this the CTA kernel wins (measured)
constexpr int kWideSegs = 8;
template <int S>
__global__ void __launch_bounds__(32)
encode_wide_kernel(const uint8_t *__restrict__ msg, int64_t n, int64_t chunk_len, int n_lanes,
                   const TableDev *__restrict__ tab, uint16_t *__restrict__ scratch,
                   uint32_t *__restrict__ chunk_words, uint32_t *__restrict__ states_out,
                   DStatus *__restrict__ status, int stats) {
    __shared__ uint2 enc[kMaxSym];
    __shared__ __align__(16) uint8_t mring[kWideSegs * kInSeg];
    const int lane = threadIdx.x;
    const uint32_t lt = lanemask_lt();
    const int64_t k = blockIdx.x;
    const int64_t cbase = k * chunk_len;
    const int64_t len = (n - cbase) < chunk_len ? (n - cbase) : chunk_len;
    const uint8_t *g = msg + cbase;
    uint16_t *out = scratch + cbase;
    // ring: byte i of the chunk sits at (delta + i) mod the ring
    const uint32_t delta = static_cast<uint32_t>(reinterpret_cast<uintptr_t>(g) & 15u);
    const uint8_t *ga = g - delta;
    const int64_t avail = len + delta;
    const uint32_t mring_sa = smem_addr(mring);
    auto issue = [&](int64_t seg) {
        const int64_t b0 = seg * kInSeg + lane * 16;
        uint32_t bytes = 0;
        if (seg >= 0 && b0 < avail) bytes = (avail - b0) >= 16 ? 16u : static_cast<uint32_t>(avail - b0);
        cp_async16(mring + (static_cast<uint32_t>(seg) & (kWideSegs - 1)) * kInSeg + lane * 16,
                   bytes ? ga + b0 : ga, bytes);
        cp_async_commit();
    };
    // groups <= 256 bytes < a segment: the low byte's segment steps down by
    // at most one per group, a group spans at most two segments
    const int64_t g_top = (len + n_lanes - 1) / n_lanes - 1;
    int64_t cur = g_top >= 0 ? (delta + g_top * n_lanes) / kInSeg : 0;  // segment of the group's low byte
    for (int q = 1; q >= 2 - kWideSegs; --q) issue(cur + q);
    for (int i = lane; i < kMaxSym; i += 32) enc[i] = tab->enc[i];
    const EncCtx ctx(tab->scale_bits);
    uint32_t x[S];
#pragma unroll
    for (int j = 0; j < S; ++j) x[j] = kLow;
    int64_t top = len;
    bool bad = false;
    uint32_t most = 0;
    cp_async_wait<kWideSegs - 3>();  // segments cur + 1, cur, cur - 1
    __syncwarp();
    // the symbols of the group below are read one group ahead
    auto load_syms = [&](int64_t gi, uint32_t *sy) {
        const int64_t base = gi * n_lanes;
        const uint32_t o = static_cast<uint32_t>(delta + base);
#pragma unroll
        for (int j = 0; j < S; ++j) {
            const int l = 32 * j + lane;
            const bool in = base + l < len && l < n_lanes;
            sy[j] = in ? lds_u8(mring_sa + ((o + l) & (kWideSegs * kInSeg - 1))) : 0u;
        }
    };
    uint32_t sym[S], nx[S];
#pragma unroll
    for (int j = 0; j < S; ++j) sym[j] = nx[j] = 0;
    if (g_top >= 0) load_syms(g_top, sym);
    for (int64_t gi = g_top; gi >= 0; --gi) {
        const int64_t base = gi * n_lanes;
        const int active = (len - base) < n_lanes ? static_cast<int>(len - base) : n_lanes;
        const int64_t seg = (delta + base) / kInSeg;
        if (seg != cur) {  // one segment lower: its slot's old segment (cur + 2) is done
            cur = seg;
            __syncwarp();
            issue(cur + 2 - kWideSegs);
            cp_async_wait<kWideSegs - 3>();  // segment cur - 1 (the next group's) landed
            __syncwarp();
        }
        if (gi > 0) load_syms(gi - 1, nx);
        uint2 e[S];
        uint32_t badm[S];
        bool anybad = false;
#pragma unroll
        for (int j = 0; j < S; ++j) {
            e[j] = enc[sym[j]];
            badm[j] = __ballot_sync(0xffffffffu, 32 * j + lane < active && e[j].x == 0u);
            anybad |= badm[j] != 0u;
        }
        if (anybad) {  // the highest offending index (the reference walks down)
            int hi = -1;
#pragma unroll
            for (int j = 0; j < S; ++j)
                if (badm[j]) hi = 32 * j + 31 - __clz(badm[j]);
            if (lane == 0) atomicMax(&status->unenc_index, static_cast<long long>(cbase + base + hi));
            bad = true;
            break;
        }
        bool sp[S];
        uint32_t mk[S];
#pragma unroll
        for (int j = S - 1; j >= 0; --j) {
            sp[j] = 32 * j + lane < active && enc_spill(ctx, x[j], e[j]);
            mk[j] = __ballot_sync(0xffffffffu, sp[j]);
        }
#pragma unroll
        for (int j = S - 1; j >= 0; --j) {
            top -= __popc(mk[j]);
            if (sp[j]) out[top + __popc(mk[j] & lt)] = static_cast<uint16_t>(x[j] & 0xFFFFu);
            const uint32_t z = sp[j] ? x[j] >> 16 : x[j];
            // stats: digits this symbol moves under the reference's spill
            // loop (rans.py:284-287): one per pass while x >= threshold
            if (stats && sp[j]) most = max(most, enc_spill(ctx, z, e[j]) ? 2u : 1u);
            const uint32_t p = enc_push(ctx, z, e[j]);
            x[j] = 32 * j + lane < active ? p : x[j];
        }
#pragma unroll
        for (int j = 0; j < S; ++j) sym[j] = nx[j];
    }
    cp_async_wait<0>();
    if (stats) {
        most = __reduce_max_sync(0xffffffffu, most);
        if (lane == 0 && most) atomicMax(&status->max_digits, most);
    }
    if (!bad) {
        if (lane == 0) chunk_words[k] = static_cast<uint32_t>(len - top);
#pragma unroll
        for (int j = 0; j < S; ++j)
            if (32 * j + lane < n_lanes) states_out[k * n_lanes + 32 * j + lane] = x[j];
    }
}

cudaError_t launch_encode(const uint8_t *d_msg, int64_t n, int64_t chunk_len, int n_lanes,
                          const TableDev *d_table, int scale_bits, uint16_t *d_scratch,
                          uint32_t *d_chunk_words, uint32_t *d_states, DStatus *d_status,
                          uint32_t *d_lane_ws, cudaStream_t stream, bool stats, bool covered) {
    if (n <= 0) return cudaSuccess;
    const int64_t n_chunks = (n + chunk_len - 1) / chunk_len;
    // stats (instrumented calls): the one-warp sub-group walk measures the
    // digits per symbol for every N <= 256, the CTA kernel beyond
    if ((n_lanes > 32 || stats) && n_lanes <= kWideMaxE) {
        // the shared message ring reads each chunk from its 16-byte aligned
        // base below it
        if (reinterpret_cast<uintptr_t>(d_msg) & 15u) return cudaErrorMisalignedAddress;
        auto kernel = n_lanes <= 64 ? encode_wide_kernel<2>
                    : n_lanes <= 128 ? encode_wide_kernel<4> : encode_wide_kernel<8>;
        kernel<<<static_cast<unsigned>(n_chunks), 32, 0, stream>>>(
            d_msg, n, chunk_len, n_lanes, d_table, d_scratch, d_chunk_words, d_states, d_status,
            stats ? 1 : 0);
    } else if (n_lanes > 32) {
        const int threads = n_lanes >= 1024 ? 1024 : ((n_lanes + 31) / 32) * 32;
        const int ws_smem = size_t(n_lanes) * 4 <= size_t(200) * 1024;
        const size_t smem = ws_smem ? size_t(n_lanes) * 4 : 0;
        smem_limit(reinterpret_cast<const void *>(encode_block_kernel), int(smem));
        encode_block_kernel<<<static_cast<unsigned>(n_chunks), threads, smem, stream>>>(
            d_msg, n, chunk_len, n_lanes, d_table, d_scratch, d_chunk_words, d_states,
            d_status, d_lane_ws, ws_smem, stats ? 1 : 0);
    } else {
        // one CTA per SM with the SM's share of the streams (<= 28 warps);
        // more streams than 28 per SM: grid-stride over CTA-sized groups
        const int64_t sms = sm_count();
        int warps = static_cast<int>((n_chunks + sms - 1) / sms);
        if (warps > kEncMaxWarps) warps = kEncMaxWarps;
        if (warps < 1) warps = 1;
        int64_t blocks = (n_chunks + warps - 1) / warps;
        const int64_t per_sm = static_cast<int64_t>(
            (227 * 1024) / (encode_smem_bytes(warps) + 1024));
        const int64_t max_blocks = sms * (per_sm < 1 ? 1 : per_sm);
        if (blocks > max_blocks) blocks = max_blocks;
        const size_t smem = encode_smem_bytes(warps);
        const unsigned g = static_cast<unsigned>(blocks);
        auto go = [&](auto kernel) {
            smem_limit(reinterpret_cast<const void *>(kernel), int(smem));
            kernel<<<g, warps * 32, smem, stream>>>(d_msg, n, chunk_len, n_chunks, n_lanes,
                                                    d_table, d_scratch, d_chunk_words, d_states,
                                                    d_status);
        };
        // the table's scale_bits is on the device; the sb = 14 instantiation
        // is picked by the caller's scale_bits and re-checks the flag itself
        const bool sb14 = scale_bits == 14 || scale_bits == 15;  // the 12-byte fast record
        // mode 1: power-of-two N < 32, mode 2: other N < 32, mode 0: N = 32
        const int mode = n_lanes >= 32 ? 0 : (n_lanes & (n_lanes - 1)) == 0 ? 1 : 2;
        auto pick = [&](auto idx) {
            using I = decltype(idx);
            if (mode == 1) {
                if (sb14) go(encode_warp_kernel<I, true, 1>);
                else go(encode_warp_kernel<I, false, 1>);
            } else if (mode == 2) {
                if (sb14) go(encode_warp_kernel<I, true, 2>);
                else go(encode_warp_kernel<I, false, 2>);
            } else if (sizeof(I) == 4) {  // N = 32: the 16-byte records, any sb
                if (covered) go(encode_warp_kernel<int, false, 0, true, true>);
                else go(encode_warp_kernel<int, false, 0, false, true>);
            } else {
                if (sb14) go(encode_warp_kernel<I, true, 0>);
                else go(encode_warp_kernel<I, false, 0>);
            }
        };
        if (chunk_len < (int64_t(1) << 30)) pick(int(0));
        else pick(static_cast<long long>(0));
    }
    ilans_note_launch();
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Framing
// ---------------------------------------------------------------------------
// Single CTA exclusive scan of n_chunks word counts -> offsets[n_chunks + 1].
// Each thread scans 4 consecutive counts per pass (4096 chunks = one pass of
// 1024 threads); passes carry the running total.
__global__ void __launch_bounds__(1024)
chunk_offsets_kernel(const uint32_t *__restrict__ words, int64_t n_chunks,
                     uint64_t *__restrict__ offsets, int carry_in) {
    __shared__ unsigned long long wsum[32];
    __shared__ unsigned long long carry;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int nw = blockDim.x >> 5;
    if (threadIdx.x == 0) carry = carry_in ? offsets[0] : 0ull;  // batch continuation
    __syncthreads();
    const int64_t per_pass = static_cast<int64_t>(blockDim.x) * 4;
    for (int64_t base = 0; base < n_chunks; base += per_pass) {
        const int64_t i0 = base + static_cast<int64_t>(threadIdx.x) * 4;
        unsigned long long v[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) v[q] = i0 + q < n_chunks ? words[i0 + q] : 0ull;
        const unsigned long long mine = v[0] + v[1] + v[2] + v[3];
        unsigned long long inc = mine;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned long long u = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += u;
        }
        if (lane == 31) wsum[wid] = inc;
        __syncthreads();
        if (wid == 0) {
            unsigned long long w = lane < nw ? wsum[lane] : 0ull;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const unsigned long long u = __shfl_up_sync(0xffffffffu, w, o);
                if (lane >= o) w += u;
            }
            wsum[lane] = w;
        }
        __syncthreads();
        unsigned long long run = carry + (wid ? wsum[wid - 1] : 0ull) + inc - mine;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            if (i0 + q < n_chunks) offsets[i0 + q] = run;
            run += v[q];
        }
        __syncthreads();
        if (threadIdx.x == 0) carry += wsum[nw - 1];
        __syncthreads();
    }
    if (threadIdx.x == 0) offsets[n_chunks] = carry;
}

// One CTA per chunk: move its payload from the end of its scratch region to
// the packed position.
__global__ void __launch_bounds__(256)
compact_kernel(const uint16_t *__restrict__ scratch, int64_t n, int64_t chunk_len,
               const uint32_t *__restrict__ words, const uint64_t *__restrict__ offsets,
               uint16_t *__restrict__ payload) {
    const int64_t k = blockIdx.x;
    const int64_t cbase = k * chunk_len;
    const int64_t len = (n - cbase) < chunk_len ? (n - cbase) : chunk_len;
    uint32_t w = words[k];
    uint64_t s = static_cast<uint64_t>(cbase + len - w);  // word index in scratch
    uint64_t d = offsets[k];                               // word index in payload
    if (w == 0) return;
    if (d & 1) {  // make the destination 4-byte aligned
        if (threadIdx.x == 0) payload[d] = scratch[s];
        ++s, ++d, --w;
    }
    uint32_t *dst = reinterpret_cast<uint32_t *>(payload + d);
    const uint32_t pairs = w >> 1;
    constexpr int U = 8;  // independent loads in flight per thread (latency-bound copy)
    const uint32_t step = blockDim.x * U;
    if (!(s & 1)) {
        const uint32_t *src = reinterpret_cast<const uint32_t *>(scratch + s);
        for (uint32_t i0 = threadIdx.x; i0 < pairs; i0 += step) {
            uint32_t v[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const uint32_t i = i0 + u * blockDim.x;
                v[u] = i < pairs ? __ldcs(src + i) : 0u;
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const uint32_t i = i0 + u * blockDim.x;
                if (i < pairs) dst[i] = v[u];
            }
        }
    } else {  // odd source: each output word is a 16-bit funnel of two inputs
        const uint32_t *src = reinterpret_cast<const uint32_t *>(scratch + s - 1);
        for (uint32_t i0 = threadIdx.x; i0 < pairs; i0 += step) {
            uint32_t a[U], b[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const uint32_t i = i0 + u * blockDim.x;
                a[u] = i < pairs ? __ldcs(src + i) : 0u;
                b[u] = i < pairs ? __ldcs(src + i + 1) : 0u;
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const uint32_t i = i0 + u * blockDim.x;
                if (i < pairs) dst[i] = __funnelshift_r(a[u], b[u], 16);
            }
        }
    }
    if ((w & 1) && threadIdx.x == 0) payload[d + w - 1] = scratch[s + w - 1];
}

cudaError_t launch_frame(const uint16_t *d_scratch, int64_t n, int64_t chunk_len,
                         const uint32_t *d_chunk_words, uint64_t *d_word_offsets,
                         uint16_t *d_payload, int carry_in, cudaStream_t stream) {
    const int64_t n_chunks = n <= 0 ? 0 : (n + chunk_len - 1) / chunk_len;
    // directory only (no packing): a 256-thread CTA, small enough to share
    // an SM with the decoder it runs beside
    chunk_offsets_kernel<<<1, d_payload ? 1024 : 256, 0, stream>>>(d_chunk_words, n_chunks,
                                                                   d_word_offsets, carry_in);
    ilans_note_launch();
    if (n_chunks > 0 && d_payload) {  // d_payload == nullptr: the directory only
        compact_kernel<<<static_cast<unsigned>(n_chunks), 256, 0, stream>>>(
            d_scratch, n, chunk_len, d_chunk_words, d_word_offsets, d_payload);
        ilans_note_launch();
    }
    return cudaGetLastError();
}

}  // namespace ilans
