// common.cuh -- shared device helpers and the device table layout.
//
// sm_100a only. Warp-synchronous primitives (ballot / popc / shfl) carry the
// paper's metadata-free interleaving (Listing 2: ballot + bitCount);
// cp.async (LDGSTS) stages payload / message bytes into per-warp shared-memory
// rings so the refill read never waits on HBM latency.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/ilans_b200.h"

namespace ilans {

constexpr uint32_t kLow = 1u << 16;          // WORD16.lower_bound (rans.py:87)
constexpr int kMaxSym = 256;                 // MAX_ALPHABET (rans.py:24)
constexpr int kMaxScaleBits = 16;            // MAX_SCALE_BITS (rans.py:25)
constexpr int kPackedMaxBits = 15;           // packed 32-bit slot entry: sym|bias|f (f < 4096)

// Table flags
constexpr uint32_t kTabPacked = 1u;          // packed[] valid (sb <= 15, every f < 4096, consistent)
constexpr uint32_t kTabEncFast = 2u;         // encf valid (sb <= 13, every f <= m/2)
constexpr uint32_t kTabPacked64 = 4u;        // packed64[] valid (13 <= sb <= 14)
constexpr uint32_t kTabEncFast12 = 8u;       // encf = {M, Y} + encz valid (sb = 14, 15, f <= m/2)
constexpr uint32_t kTabEncQuad = 16u;        // encq valid (any sb, every f <= m/2)
constexpr uint32_t kTabEncQuadX = 32u;       // encqx valid (any sb, every f < m)
constexpr int kPacked64MinBits = 13;
constexpr int kPacked64MaxBits = 14;
constexpr int kEncFastMaxBits = 13;             // bias < 2^(sb+1) fits Z's bits [5, 32-sb)

// Device-resident model: everything a kernel needs, in one blob so a single
// pointer travels through the C ABI. Layout is 16-byte aligned throughout.
struct alignas(16) TableDev {
    uint32_t scale_bits;
    uint32_t n_sym;        // alphabet size written to the wire table
    uint32_t status;       // ilans_rc of model-build validation
    uint32_t flags;
    uint32_t err_detail[4];
    uint32_t freq[kMaxSym];           // zero-padded past n_sym
    uint32_t cum[kMaxSym + 4];        // cum[0..256]
    uint2 enc[kMaxSym];               // EncSym records {magic, (m - f) | cum << 16}
    uint2 dec[kMaxSym];               // {f, cum} for the decoder's second lookup
    uint2 encf[kMaxSym];              // EncFast records {M, (m - f) << t | bias << 5 | s}
                                      // (sb = 14: EncFast12 {M, f << t | (m - f)})
    uint32_t encz[kMaxSym];           // EncFast12: s | bias << 17
    uint4 encq[kMaxSym];              // EncQuad records {M, f << t | s, m - f, bias}
    uint4 encqx[kMaxSym];             // EncQuadX records {magic, f << t | l, m - f, cum}
    uint32_t packed[1 << kPackedMaxBits];  // sym | bias << 8 | f << 20 (f < 4096)
    uint8_t slot_sym[1 << kMaxScaleBits];
    uint2 packed64[1 << 14];          // 13 <= sb <= 14: {sym | bias << 8, f}
};

// Optional per-group decode trace (single-stream calls): the lane states and
// the read position after every group, plus the number of completed groups
// -- the device form of interleave.decode_interleaved_steps /
// lanes.decode_lanes_steps (interleave.py:251-268, lanes.py:221-232).
// Where chunk k's payload words are: packed back to back at word offsets
// offsets[k] .. offsets[k + 1] (the framed stream), or -- slot_words set --
// in the encoder's slot layout, right-aligned in chunk k's C-word slot:
// [kC + len_k - w_k, kC + len_k) with w_k = slot_words[k] (decode straight
// from the encode scratch; the packed stream is only built on egress).
struct ChunkDir {
    const uint64_t *offsets;
    const uint32_t *slot_words;
    __device__ __forceinline__ void span(int64_t k, int64_t cbase, int64_t len, uint64_t &woff,
                                         uint64_t &wlen) const {
        if (slot_words) {
            wlen = slot_words[k];
            woff = static_cast<uint64_t>(cbase + len) - wlen;
        } else {
            woff = offsets[k];
            wlen = offsets[k + 1] - woff;
        }
    }
};

struct DecodeTrace {
    uint32_t *states;  // [groups][N]
    uint64_t *pos;     // [groups]
    uint64_t *groups;  // [1] completed groups
    int stats;         // measure digits per symbol -> DStatus::max_digits (generic loop)
};

// Device status blob (first error wins, deterministic by index).
struct alignas(16) DStatus {
    unsigned long long trunc_stream;  // min failing stream index, ~0 = none
    long long unenc_index;            // max offending message index, -1 = none
    uint32_t unenc_symbol;
    uint32_t value_error;
    uint32_t max_digits;              // most digits moved for one symbol (byte8; word16 stats calls)
    uint32_t pad[3];
};

__device__ __forceinline__ uint32_t lanemask_lt() {
    uint32_t m;
    asm volatile("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

__device__ __forceinline__ uint32_t smem_addr(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// 16-byte global->shared async copy; bytes past src_bytes are zero-filled.
__device__ __forceinline__ void cp_async16(void *smem_dst, const void *gmem_src,
                                           uint32_t src_bytes) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_addr(smem_dst)),
                 "l"(gmem_src), "r"(src_bytes)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
    asm volatile("cp.async.commit_group;\n" ::: "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// Exact unsigned division by an invariant d in [1, 2^16] for every 32-bit
// numerator with a 33-bit magic (Granlund & Montgomery, "Division by
// invariant integers using multiplication", PLDI'94, sec. 4):
//   l = ceil(log2 d), m = floor(2^(32+l) / d) + 1 = 2^32 + magic,
//   q = floor(m * n / 2^(32+l)) = (umulhi(magic, n) + n) >> l   (33-bit sum).
// m*d - 2^(32+l) lies in (0, 2^l], which makes q exact for all n < 2^32;
// magic < 2^32 because 2^(l-1) < d. tests/test_host.py checks every d.
// ceil(log2 d) for d >= 1
__host__ __device__ inline uint32_t ceil_log2(uint32_t d) {
#ifdef __CUDA_ARCH__
    return d <= 1u ? 0u : 32u - static_cast<uint32_t>(__clz(d - 1u));
#else
    uint32_t l = 0;
    while ((1ull << l) < d) ++l;
    return l;
#endif
}

__host__ __device__ inline void divmagic(uint32_t d, uint32_t *magic, uint32_t *l_out) {
    const uint32_t l = ceil_log2(d);
    const uint64_t m = ((1ull << (32 + l)) / d) + 1;  // in (2^32, 2^33)
    *magic = static_cast<uint32_t>(m - (1ull << 32));
    *l_out = l;
}

// q = (umulhi(magic, n) + n) >> l, the sum kept as 33 bits: a funnel shift
// of (carry:lo). `shift` may carry other data above bit 4 (.wrap uses & 31).
__device__ __forceinline__ uint32_t div_magic(uint32_t n, uint32_t magic, uint32_t shift) {
    const uint32_t t = __umulhi(magic, n);
    uint32_t lo, hi;
    asm("add.cc.u32 %0, %2, %3;\n\taddc.u32 %1, 0, 0;" : "=r"(lo), "=r"(hi) : "r"(t), "r"(n));
    uint32_t q;
    asm("shf.r.wrap.b32 %0, %1, %2, %3;" : "=r"(q) : "r"(lo), "r"(hi), "r"(shift));
    return q;
}

// Encoder record per symbol: 8 bytes, one LDS.64 (the encoder is bound by
// shared-memory wavefronts on this random-address lookup, so the record is
// kept small and f / l are re-derived with two ALU ops):
//   .x = magic                       (0 marks f == 0: unencodable)
//   .y = (f - 1) | cum << 16         (f - 1 in [0, 2^16), cum < 2^16)
// spill:  x >= f << (32 - sb)  <=>  (x >> (32 - sb)) > f - 1
// push:   x' = (x / f) * m + cum + x % f = q * (m - f) + x + cum
//         with q = x / f via the magic and l = ceil(log2 f) = bfind(f - 1) + 1
// Tables whose f / cum do not fit (f > m or cum >= 2^16 -- never produced by
// quantize / SymbolTable) are rejected by the host before encoding.
struct EncSym {
    __host__ __device__ static uint2 make(uint32_t f, uint32_t cum, int scale_bits) {
        if (f == 0) return make_uint2(0u, 0u);
        uint32_t magic, l;
        divmagic(f, &magic, &l);
        (void)scale_bits;
        return make_uint2(magic, ((f - 1u) & 0xFFFFu) | (cum << 16));
    }
};

// Fast encoder record (tables with sb <= 13 whose every f <= m / 2, flag
// kTabEncFast): 8 bytes, one LDS.64, every field used with at most one op.
//   .x = M = ceil(2^(31+c) / f), c = ceil(log2 f), s = c - 1
//        (f = 1: M = 2^32 - 1, s = 0, i.e. q = x - 1, compensated in bias)
//   .y = Z = (m - f) << t | bias << 5 | s,  t = 32 - sb,
//        bias = cum (+ m - 1 when f = 1) < 2^(sb+1) in bits [5, t)
// spill:  x >= f << t  <=>  (x & ~(2^t - 1)) + Z carries out of 32 bits
//         (the bits below t never decide it; the compiler turns it into
//         one LOP3 + one compare against Z)
// push:   q = umulhi(x, M) >> s     (shf.r.wrap reads s from Z's low 5 bits)
//         x' = x + bias + q (m - f)
//            = (x + (Z >> 5)) + (m - f) (q - 2^(t-5))
//         since Z >> 5 = (m - f) 2^(t-5) + bias: one LEA.HI, one add to q,
//         one shift for m - f = Z >> t, one IMAD
// Exactness of q = floor(x / f) for every post-spill x < f * 2^t: with
// e = M f - 2^(31+c) in [0, f), x e < f^2 2^t <= 2^(31+c) iff
// f <= 2^(sb-1), so the rounding error x e / (f 2^(31+c)) < 1 / f never
// crosses an integer (tests/test_host.py checks every f for sb <= 13).
// M = 0 marks f = 0 (unencodable).
struct EncFast {
    __host__ __device__ static uint2 make(uint32_t f, uint32_t cum, int sb) {
        const uint32_t m = 1u << sb, t = 32u - static_cast<uint32_t>(sb);
        if (f == 0 || f > m / 2) return make_uint2(0u, 0u);
        uint32_t M, sh, bias = cum;
        if (f == 1) {
            M = 0xFFFFFFFFu;
            sh = 0u;
            bias = cum + m - 1u;
        } else {
            const uint32_t c = ceil_log2(f);
            M = static_cast<uint32_t>(((1ull << (31 + c)) + f - 1) / f);
            sh = c - 1u;
        }
        return make_uint2(M, (m - f) << t | bias << 5 | sh);
    }
};

// sb = 14, 15 (every f <= m / 2): bias < 2^(sb+1) no longer fits beside
// m - f and s in one word, so the record takes 12 bytes:
//   .x = M (as EncFast),  .y = Y = f << t | (m - f)   (m - f < 2^sb <= 2^t)
//   Z  = s | bias << 16   (a separate 4-byte array; bias < 2^16, s < 16)
// spill: (x | (2^t - 1)) >= Y;  q = umulhi(x, M) >> s (s = Z & 31);
// x' = q (Y & (2^t - 1)) + x + (Z >> 16). q is exact for every post-spill
// x < f 2^t <= 2^31 whatever sb (f <= m / 2, see EncFast).
struct EncFast12 {
    __host__ __device__ static void make(uint32_t f, uint32_t cum, int sb, uint2 *a,
                                         uint32_t *z) {
        const uint32_t m = 1u << sb, t = 32u - static_cast<uint32_t>(sb);
        if (f == 0 || f > m / 2) {
            *a = make_uint2(0u, 0u);
            *z = 0u;
            return;
        }
        uint32_t M, sh, bias = cum;
        if (f == 1) {
            M = 0xFFFFFFFFu;
            sh = 0u;
            bias = cum + m - 1u;
        } else {
            const uint32_t c = ceil_log2(f);
            M = static_cast<uint32_t>(((1ull << (31 + c)) + f - 1) / f);
            sh = c - 1u;
        }
        *a = make_uint2(M, f << t | (m - f));
        *z = sh | bias << 16;
    }
};

// 16-byte fast record (any sb <= 16 with every f <= m / 2, flag
// kTabEncQuad): the N = 32 encoder's form. One LDS.128 (a quarter-warp per
// wavefront) hands every field over ready to use, so the push is 4 ops:
//   .x = M (as EncFast)      .y = Y = f << t | s   (s < 32 <= 2^t - 1)
//   .z = m - f               .w = bias (as EncFast: cum, + m - 1 for f = 1)
// spill:  (x | (2^t - 1)) >= Y   (<=> x >= f << t: the low t bits of the
//         left side are all ones, and s < 2^t)
// push:   q = umulhi(x, M) >> s  (shf.r.wrap reads s from Y's low 5 bits)
//         x' = (m - f) q + (x + bias)
struct EncQuad {
    __host__ __device__ static uint4 make(uint32_t f, uint32_t cum, int sb) {
        const uint32_t m = 1u << sb, t = 32u - static_cast<uint32_t>(sb);
        if (f == 0 || f > m / 2) return make_uint4(0u, 0u, 0u, 0u);
        uint32_t M, sh, bias = cum;
        if (f == 1) {
            M = 0xFFFFFFFFu;
            sh = 0u;
            bias = cum + m - 1u;
        } else {
            const uint32_t c = ceil_log2(f);
            M = static_cast<uint32_t>(((1ull << (31 + c)) + f - 1) / f);
            sh = c - 1u;
        }
        return make_uint4(M, f << t | sh, m - f, bias);
    }
};

// The same 16-byte form for tables with a symbol above m/2 (skewed sources;
// flag kTabEncQuadX, every f < m): the 32-bit M of EncQuad is not exact
// there, so the division takes divmagic's 33-bit magic (exact for every
// x < 2^32): .x = magic, .y = Y = f << t | l, .z = m - f, .w = cum;
//   q = (umulhi(x, magic) + x) >> l   (33-bit sum: add.cc / addc + shf.r.wrap)
//   x' = (m - f) q + (x + cum)
// two more instructions than EncQuad. f = 0 is all zeros (Y = 0 marks it:
// every valid Y >= 2^t).
struct EncQuadX {
    __host__ __device__ static uint4 make(uint32_t f, uint32_t cum, int sb) {
        const uint32_t m = 1u << sb, t = 32u - static_cast<uint32_t>(sb);
        if (f == 0 || f >= m) return make_uint4(0u, 0u, 0u, 0u);
        uint32_t magic, l;
        divmagic(f, &magic, &l);
        return make_uint4(magic, f << t | l, m - f, cum);
    }
};

struct EncCtx {
    uint32_t mm1;        // 2^sb - 1
    uint32_t thr_shift;  // 32 - sb
    __device__ explicit EncCtx(uint32_t sb) : mm1((1u << sb) - 1u), thr_shift(32u - sb) {}
};

__device__ __forceinline__ bool enc_spill(const EncCtx &c, uint32_t x, const uint2 &e) {
    return (x >> c.thr_shift) > (e.y & 0xFFFFu);
}

// One rANS push of symbol record e onto state x (after the spill).
__device__ __forceinline__ uint32_t enc_push(const EncCtx &c, uint32_t x, const uint2 &e) {
    const uint32_t fm1 = e.y & 0xFFFFu;
    uint32_t msb;  // bfind: index of the highest set bit, 0xFFFFFFFF for 0
    asm("bfind.u32 %0, %1;" : "=r"(msb) : "r"(fm1));
    const uint32_t q = div_magic(x, e.x, msb + 1u);
    return q * (c.mm1 - fm1) + x + (e.y >> 16);
}

}  // namespace ilans

// Host-side launch accounting (ilans_launch_count).
void ilans_note_launch(int n = 1);
