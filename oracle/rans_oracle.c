/*
 * rans_oracle.c -- CPU restatement of the reference word16 interleaved-rANS
 * hot path. TEST INFRASTRUCTURE ONLY: linked by tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline leg as the CHECKER. Nothing in the product
 * package (paper_1402_3392_b200/) may load this file or its build output.
 *
 * Each function is a plain-C restatement of one reference function, written
 * from the reference's documented behaviour (not copied). Citations are
 * relative to the reference root (pkg/src/ilans/...).
 *
 * Parity pinning: tests/test_oracle.py checks every function here against
 * (a) the known-answer tests of the reference's own suite, (b) golden
 * fixtures produced by the reference itself (tests/golden/make_golden.py),
 * and (c) the container sha256 digests listed in BASELINE.md section 3.
 */
#include <stdint.h>
#include <stddef.h>
#include <string.h>

typedef unsigned __int128 u128;
typedef __int128 i128;

enum {
    ORC_OK = 0,
    ORC_ERR_VALUE = 1,        /* ValueError in the reference */
    ORC_ERR_UNENCODABLE = 2,  /* UnencodableSymbolError */
    ORC_ERR_TRUNCATED = 3,    /* TruncatedStreamError */
    ORC_ERR_FORMAT = 6,       /* FormatError (byte8 refill runaway) */
};

#define ORC_LOW 65536u /* WORD16.lower_bound, rans.py:87 */

/* np.bincount over bytes (call sites cli.py:31-37, bench.py:47-51).
 * Returns max symbol + 1 (the reference's alphabet size), 0 if n == 0. */
int orc_histogram_u8(const uint8_t *msg, int64_t n, uint64_t *counts256)
{
    memset(counts256, 0, 256 * sizeof(uint64_t));
    for (int64_t i = 0; i < n; i++)
        counts256[msg[i]]++;
    int alpha = 0;
    for (int s = 0; s < 256; s++)
        if (counts256[s]) alpha = s + 1;
    return alpha;
}

/* rans.quantize (rans.py:171-211): floor(c*m/T) with a floor of 1 for
 * present symbols, then +1 to argmax(c*m - f*T, -i) while short, -1 to
 * argmax(f*T - c*m, -i) over f > 1 while over. Exact 128-bit integers,
 * ties to the lowest index -- the same greedy loop, one unit at a time. */
int orc_quantize(const uint64_t *counts, int n, int scale_bits, uint32_t *freq_out)
{
    if (scale_bits < 1 || scale_bits > 16) return ORC_ERR_VALUE;
    if (n > 256) return ORC_ERR_VALUE;
    u128 total = 0;
    int present = 0;
    for (int i = 0; i < n; i++) {
        total += counts[i];
        if (counts[i]) present++;
    }
    if (total == 0) return ORC_ERR_VALUE;
    const uint64_t m = 1ull << scale_bits;
    if ((uint64_t)present > m) return ORC_ERR_VALUE;
    int64_t sum = 0;
    for (int i = 0; i < n; i++) {
        if (!counts[i]) { freq_out[i] = 0; continue; }
        u128 q = ((u128)counts[i] * m) / total;
        freq_out[i] = q < 1 ? 1u : (uint32_t)q;
        sum += freq_out[i];
    }
    int64_t diff = (int64_t)m - sum;
    while (diff > 0) {
        int best = -1;
        i128 best_key = 0;
        for (int i = 0; i < n; i++) {
            if (!counts[i]) continue;
            i128 key = (i128)((u128)counts[i] * m) - (i128)((u128)freq_out[i] * total);
            if (best < 0 || key > best_key) { best = i; best_key = key; }
        }
        freq_out[best]++;
        diff--;
    }
    while (diff < 0) {
        int best = -1;
        i128 best_key = 0;
        for (int i = 0; i < n; i++) {
            if (!counts[i] || freq_out[i] <= 1) continue;
            i128 key = (i128)((u128)freq_out[i] * total) - (i128)((u128)counts[i] * m);
            if (best < 0 || key > best_key) { best = i; best_key = key; }
        }
        freq_out[best]--;
        diff++;
    }
    return ORC_OK;
}

/* _core.encode_interleaved_u16 (_core.pyx:14-43; twin _pure.py:15-39).
 * Backward walk, lane = i mod N, states start at L; spill one digit when
 * x >= f << (32 - sb); push x -> (x/f << sb) + cum + x%f. The digits are
 * stacked from the end of a capacity-n buffer, so the payload in decoder
 * read order is payload_scratch[pos .. n). Writes that suffix to
 * payload_out[0 .. words) and returns ORC_OK, or ORC_ERR_UNENCODABLE with
 * bad_index and bad_symbol set for the first (highest-index) f == 0 symbol. */
int orc_encode_u16(const uint8_t *msg, int64_t n, const uint32_t *freq,
                   const uint32_t *cum, int scale_bits, int n_lanes,
                   uint16_t *scratch, uint16_t *payload_out, int64_t *words,
                   uint32_t *states_out, int64_t *bad_index, int *bad_symbol)
{
    const int shift = 32 - scale_bits;
    int64_t pos = n;
    for (int l = 0; l < n_lanes; l++) states_out[l] = ORC_LOW;
    for (int64_t i = n - 1; i >= 0; i--) {
        uint32_t s = msg[i];
        uint32_t f = freq[s];
        if (f == 0) {
            if (bad_index) *bad_index = i;
            if (bad_symbol) *bad_symbol = (int)s;
            return ORC_ERR_UNENCODABLE;
        }
        int lane = (int)(i % n_lanes);
        uint32_t x = states_out[lane];
        if ((uint64_t)x >= ((uint64_t)f << shift)) {
            scratch[--pos] = (uint16_t)(x & 0xFFFFu);
            x >>= 16;
        }
        uint64_t coded = ((uint64_t)(x / f) << scale_bits) + cum[s] + x % f;
        states_out[lane] = (uint32_t)coded;
    }
    *words = n - pos;
    if (payload_out != scratch + pos)
        memmove(payload_out, scratch + pos, (size_t)(n - pos) * sizeof(uint16_t));
    return ORC_OK;
}

/* _core.decode_interleaved_u16 (_core.pyx:46-127; twin _pure.py:42-66).
 * Forward decode, lane = i mod N: slot = x & (m-1); s = slot_sym[slot];
 * x = f[s]*(x >> sb) + slot - cum[s] (u32 wrap of the u64 result); one
 * refill from payload[pos++] when x < L, TruncatedStreamError when the
 * payload is exhausted (_core.pyx:69-71). states_io is updated in place. */
int orc_decode_u16(const uint16_t *payload, int64_t pay_len, uint32_t *states_io,
                   const uint8_t *slot_sym, const uint32_t *freq, const uint32_t *cum,
                   int scale_bits, int64_t msg_len, int n_lanes, uint8_t *out,
                   int64_t *consumed)
{
    const uint32_t mask = (1u << scale_bits) - 1u;
    int64_t pos = 0;
    for (int64_t i = 0; i < msg_len; i++) {
        int lane = (int)(i % n_lanes);
        uint32_t x = states_io[lane];
        uint32_t slot = x & mask;
        uint32_t s = slot_sym[slot];
        out[i] = (uint8_t)s;
        x = (uint32_t)((uint64_t)freq[s] * (x >> scale_bits) + slot - cum[s]);
        if (x < ORC_LOW) {
            if (pos >= pay_len) { *consumed = pos; return ORC_ERR_TRUNCATED; }
            x = (x << 16) | payload[pos++];
        }
        states_io[lane] = x;
    }
    *consumed = pos;
    return ORC_OK;
}

/* _core.decode_lanes_u16 (_core.pyx:130-173; twin _pure.py:69-101;
 * semantics lanes.decode_step lanes.py:138-151). Group-at-a-time: pop every
 * active lane, then the lanes with x < L take payload[pos + k] in ascending
 * lane order (k = rank among pending lanes, i.e. popc(mask & lanemask_lt));
 * truncation is checked once per group (_core.pyx:164-165). Rejects N > 32
 * (ValueError, _core.pyx:144-145). */
int orc_decode_lanes_u16(const uint16_t *payload, int64_t pay_len, uint32_t *states_io,
                         const uint8_t *slot_sym, const uint32_t *freq,
                         const uint32_t *cum, int scale_bits, int64_t msg_len,
                         int n_lanes, uint8_t *out, int64_t *consumed)
{
    if (n_lanes > 32) return ORC_ERR_VALUE;
    const uint32_t mask = (1u << scale_bits) - 1u;
    int64_t pos = 0, base = 0;
    while (base < msg_len) {
        int active = (msg_len - base >= n_lanes) ? n_lanes : (int)(msg_len - base);
        uint32_t pend = 0;
        for (int lane = 0; lane < active; lane++) {
            uint32_t x = states_io[lane];
            uint32_t slot = x & mask;
            uint32_t s = slot_sym[slot];
            out[base + lane] = (uint8_t)s;
            x = (uint32_t)((uint64_t)freq[s] * (x >> scale_bits) + slot - cum[s]);
            states_io[lane] = x;
            if (x < ORC_LOW) pend |= 1u << lane;
        }
        int cnt = __builtin_popcount(pend);
        if (pos + cnt > pay_len) { *consumed = pos; return ORC_ERR_TRUNCATED; }
        for (int lane = 0; lane < active; lane++) {
            if (pend >> lane & 1u) {
                int k = __builtin_popcount(pend & ((1u << lane) - 1u));
                states_io[lane] = (states_io[lane] << 16) | payload[pos + k];
            }
        }
        pos += cnt;
        base += active;
    }
    *consumed = pos;
    return ORC_OK;
}

/* BYTE8 scalar path: interleave._encode_scalar (interleave.py:155-165) with
 * rans.encode_symbol_renorm (rans.py:266-289): states start at L = 2^23;
 * walking backwards, while x >= f * (2^31 >> sb) push x & 0xFF and x >>= 8,
 * then x = (x / f << sb) + cum + x % f. The payload is the reversed stack.
 * scratch needs 4n bytes. */
int orc_encode_u8(const uint8_t *msg, int64_t n, const uint32_t *freq, const uint32_t *cum,
                  int scale_bits, int n_lanes, uint8_t *scratch, uint8_t *payload_out,
                  int64_t *nbytes, uint32_t *states_out)
{
    const uint64_t low = 1ull << 23, limit = 1ull << 31;
    uint64_t xs[65536];
    int64_t sp = 0;
    for (int l = 0; l < n_lanes; l++) xs[l] = low;
    for (int64_t i = n - 1; i >= 0; i--) {
        uint32_t s = msg[i];
        uint64_t f = freq[s];
        if (f == 0) return ORC_ERR_UNENCODABLE;
        int lane = (int)(i % n_lanes);
        uint64_t x = xs[lane];
        uint64_t thr = f * (limit >> scale_bits);
        while (x >= thr) { scratch[sp++] = (uint8_t)(x & 0xFF); x >>= 8; }
        xs[lane] = ((x / f) << scale_bits) + cum[s] + x % f;
    }
    for (int64_t j = 0; j < sp; j++) payload_out[j] = scratch[sp - 1 - j];
    for (int l = 0; l < n_lanes; l++) states_out[l] = (uint32_t)xs[l];
    *nbytes = sp;
    return ORC_OK;
}

/* BYTE8 scalar decode: interleave._decode_scalar (interleave.py:168-179) with
 * rans.decode_symbol_renorm (rans.py:292-314): pop, then refill bytes while
 * x < L; TruncatedStreamError when the digits run out (ans.py:80-85),
 * FormatError after more than (24+7)/8 + 2 = 5 refills for one symbol. */
int orc_decode_u8(const uint8_t *payload, int64_t pay_len, uint32_t *states_io,
                  const uint8_t *slot_sym, const uint32_t *freq, const uint32_t *cum,
                  int scale_bits, int64_t msg_len, int n_lanes, uint8_t *out, int64_t *consumed)
{
    const uint64_t low = 1ull << 23, mask = (1ull << scale_bits) - 1;
    int64_t pos = 0;
    for (int64_t i = 0; i < msg_len; i++) {
        int lane = (int)(i % n_lanes);
        uint64_t x = states_io[lane];
        uint64_t slot = x & mask;
        uint32_t s = slot_sym[slot];
        out[i] = (uint8_t)s;
        x = (uint64_t)freq[s] * (x >> scale_bits) + slot - cum[s];
        int r = 0;
        while (x < low) {
            if (pos >= pay_len) { *consumed = pos; return ORC_ERR_TRUNCATED; }
            x = (x << 8) | payload[pos++];
            if (++r > 5) { *consumed = pos; return ORC_ERR_FORMAT; }
        }
        states_io[lane] = (uint32_t)x;
    }
    *consumed = pos;
    return ORC_OK;
}

/* Chunk framing (no reference function): chunk k is
 * msg[k*C, min((k+1)*C, n)), encoded as an independent N-lane word16
 * stream under one table -- i.e. exactly orc_encode_u16 on the slice, which
 * is what reference encode_interleaved(chunk, table, N, WORD16) returns.
 * Payloads are concatenated in chunk order; word_offsets has n_chunks+1
 * entries. scratch needs capacity C words. */
int orc_encode_chunks_u16(const uint8_t *msg, int64_t n, int64_t chunk_len,
                          const uint32_t *freq, const uint32_t *cum, int scale_bits,
                          int n_lanes, uint16_t *scratch, uint16_t *payload_out,
                          uint64_t *word_offsets, uint32_t *states_out)
{
    int64_t n_chunks = n == 0 ? 0 : (n + chunk_len - 1) / chunk_len;
    uint64_t off = 0;
    word_offsets[0] = 0;
    for (int64_t k = 0; k < n_chunks; k++) {
        int64_t len = n - k * chunk_len < chunk_len ? n - k * chunk_len : chunk_len;
        int64_t words = 0;
        int rc = orc_encode_u16(msg + k * chunk_len, len, freq, cum, scale_bits, n_lanes,
                                scratch, payload_out + off, &words,
                                states_out + k * n_lanes, NULL, NULL);
        if (rc) return rc;
        off += (uint64_t)words;
        word_offsets[k + 1] = off;
    }
    return ORC_OK;
}

int orc_decode_chunks_u16(const uint16_t *payload, const uint64_t *word_offsets,
                          const uint32_t *states, const uint8_t *slot_sym,
                          const uint32_t *freq, const uint32_t *cum, int scale_bits,
                          int64_t n, int64_t chunk_len, int n_lanes, uint8_t *out)
{
    int64_t n_chunks = n == 0 ? 0 : (n + chunk_len - 1) / chunk_len;
    uint32_t xs[65536];
    for (int64_t k = 0; k < n_chunks; k++) {
        int64_t len = n - k * chunk_len < chunk_len ? n - k * chunk_len : chunk_len;
        memcpy(xs, states + k * n_lanes, (size_t)n_lanes * 4);
        int64_t consumed = 0;
        int64_t pay_len = (int64_t)(word_offsets[k + 1] - word_offsets[k]);
        int rc = orc_decode_u16(payload + word_offsets[k], pay_len, xs, slot_sym, freq,
                                cum, scale_bits, len, n_lanes, out + k * chunk_len,
                                &consumed);
        if (rc) return rc;
        if (consumed != pay_len) return ORC_ERR_VALUE;
    }
    return ORC_OK;
}
