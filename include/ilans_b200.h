/*
 * ilans_b200.h -- C ABI of the B200-native interleaved-rANS (word16) codec.
 *
 * Plain pointers and sizes only; no C++ exceptions and no torch types cross
 * this boundary. Every entry point returns an ilans_rc (0 = ILANS_OK) and,
 * where the reference raises, fills an ilans_status with the error kind so
 * the Python host layer can raise the reference's exception types
 * (pkg/src/ilans/errors.py:4-33).
 *
 * Two families:
 *  1. HOST-BUFFER DROP-INS for the reference kernel boundary
 *     (pkg/src/ilans/backend.py:16-21 -> pkg/src/ilans/_core.pyx). Same
 *     argument meaning as the Cython functions; inputs are host arrays, the
 *     library copies them to HBM, runs the sm_100a kernels and copies back.
 *  2. DEVICE-POINTER, STREAM-ORDERED entry points for the chunked,
 *     HBM-resident pipeline (histogram -> quantize/table -> chunked encode ->
 *     framing; chunked decode). All `d_*` pointers are device memory; the
 *     `stream` argument is a cudaStream_t (NULL = legacy default stream).
 *     They launch asynchronously and never synchronize.
 *
 * Word16 only (WORD16 = 16-bit digits, L = 2^16, rans.py:87): states are
 * u32 in [2^16, 2^32), scale_bits in [1, 16], alphabet <= 256.
 */
#ifndef ILANS_B200_H
#define ILANS_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ILANS_B200_ABI_VERSION 1

typedef enum ilans_rc {
    ILANS_OK = 0,
    ILANS_ERR_VALUE = 1,        /* ValueError (bad argument)                  */
    ILANS_ERR_UNENCODABLE = 2,  /* UnencodableSymbolError (f == 0)            */
    ILANS_ERR_TRUNCATED = 3,    /* TruncatedStreamError (payload exhausted)   */
    ILANS_ERR_UNSUPPORTED = 4,  /* UnsupportedVariantError                    */
    ILANS_ERR_CUDA = 5,         /* CUDA runtime failure / no device           */
    ILANS_ERR_FORMAT = 6,       /* FormatError (byte8 refill loop runaway)    */
    ILANS_ERR_SCHEDULE = 7,     /* ScheduleError (mux schedule vs streams)    */
} ilans_rc;

typedef struct ilans_status {
    int32_t code;       /* ilans_rc of the failure, ILANS_OK otherwise           */
    int32_t cuda_error; /* cudaError_t when code == ILANS_ERR_CUDA               */
    int64_t stream;     /* chunk/stream index of the first failing stream, or -1 */
    int64_t index;      /* message index of the offending symbol, or -1          */
    int32_t symbol;     /* offending symbol value (unencodable), or -1           */
    int32_t max_digits; /* most digits spilled / refilled by one symbol (byte8, *_stats) */
    int64_t consumed;   /* words consumed (single-stream decode)                 */
    char message[128];  /* human-readable detail                                 */
} ilans_status;

/* -------------------------------------------------------------------------
 * Library / device
 * ---------------------------------------------------------------------- */
int ilans_abi_version(void);
/* Number of visible CUDA devices (0 when none); never fails. */
int ilans_device_count(void);
/* Select the device subsequent host-buffer calls run on (per host thread). */
int ilans_set_device(int device, ilans_status *st);
/* Number of kernel launches issued by this library since load (counter used
 * by bench.py's gpu_launches evidence). */
uint64_t ilans_launch_count(void);
/* The process is exiting: per-thread contexts destroyed after this (the
 * main thread's, after the host language's own shutdown) release nothing
 * through the CUDA runtime, whose teardown may already have run; the OS
 * reclaims their memory. Bindings call it from their exit hook. */
void ilans_process_exiting(void);

/* -------------------------------------------------------------------------
 * 1. Host-buffer drop-ins (reference: pkg/src/ilans/_core.pyx)
 * ---------------------------------------------------------------------- */

/* Replaces _core.encode_interleaved_u16(msg, freq, cum, scale_bits, n_lanes)
 * (_core.pyx:14-43; contract _pure.py:15-39). freq/cum have n_freq and
 * n_freq+1 entries; symbols >= n_freq have frequency 0. payload_out must
 * hold n words; on success words [0, *payload_words) are the payload in
 * decoder read order and states_out[0, n_lanes) the final lane states.
 * n_lanes in [1, 65535]. Errors: ILANS_ERR_UNENCODABLE (f == 0, reported
 * for the highest message index, matching the reference's backward walk). */
int ilans_encode_interleaved_u16(const uint8_t *msg, int64_t n, const uint32_t *freq,
                                 int32_t n_freq, const uint32_t *cum, int32_t scale_bits,
                                 int32_t n_lanes, uint16_t *payload_out,
                                 int64_t *payload_words, uint32_t *states_out,
                                 ilans_status *st);

/* Replaces _core.decode_interleaved_u16(payload, states, slot_sym, freq, cum,
 * scale_bits, msg_len, n_lanes) (_core.pyx:46-127; _pure.py:42-66).
 * slot_sym has n_slots >= 2^scale_bits entries. Writes msg_len bytes to out
 * and the number of payload words read to *consumed. n_lanes in
 * [1, 65535]. Errors: ILANS_ERR_TRUNCATED. */
int ilans_decode_interleaved_u16(const uint16_t *payload, int64_t pay_len,
                                 const uint32_t *states, const uint8_t *slot_sym,
                                 int64_t n_slots, const uint32_t *freq, const uint32_t *cum,
                                 int32_t n_freq, int32_t scale_bits, int64_t msg_len,
                                 int32_t n_lanes, uint8_t *out, int64_t *consumed,
                                 ilans_status *st);

/* Replaces _core.decode_lanes_u16 (_core.pyx:130-173; _pure.py:69-101):
 * same signature and byte-identical results; rejects n_lanes > 32 with
 * ILANS_ERR_VALUE (the reference's ValueError, _core.pyx:144-145). */
int ilans_decode_lanes_u16(const uint16_t *payload, int64_t pay_len, const uint32_t *states,
                           const uint8_t *slot_sym, int64_t n_slots, const uint32_t *freq,
                           const uint32_t *cum, int32_t n_freq, int32_t scale_bits,
                           int64_t msg_len, int32_t n_lanes, uint8_t *out,
                           int64_t *consumed, ilans_status *st);

/* Instrumented forms for interleave.encode_interleaved / decode_interleaved
 * with stats= (the reference's RenormStats path, rans.py:235-314): same
 * arguments and results as the two calls above, and the kernel MEASURES the
 * most digits any one symbol moved under the reference's spill / refill
 * loops (rans.py:284-287, :305-309) into st->max_digits (word16: 1 whenever
 * any digit moved; 2 would mean a symbol needed a second digit). These run
 * the generic per-group loop, not the batched fast path.
 * Host-buffer calls are per host thread: each thread gets its own stream,
 * device buffers, pinned staging and cached device model (rebuilt only when
 * freq / cum / slot / scale_bits change), and one synchronisation per call. */
int ilans_encode_interleaved_u16_stats(const uint8_t *msg, int64_t n, const uint32_t *freq,
                                       int32_t n_freq, const uint32_t *cum, int32_t scale_bits,
                                       int32_t n_lanes, uint16_t *payload_out,
                                       int64_t *payload_words, uint32_t *states_out,
                                       ilans_status *st);
int ilans_decode_interleaved_u16_stats(const uint16_t *payload, int64_t pay_len,
                                       const uint32_t *states, const uint8_t *slot_sym,
                                       int64_t n_slots, const uint32_t *freq, const uint32_t *cum,
                                       int32_t n_freq, int32_t scale_bits, int64_t msg_len,
                                       int32_t n_lanes, uint8_t *out, int64_t *consumed,
                                       ilans_status *st);

/* Any RenormVariant (digit_bits in [1, 16], lower_bound L with L % 2^sb == 0
 * and L << digit_bits <= 2^32): the reference's scalar path for variants
 * other than word16 / byte8 (interleave.py:155-179, rans.py:266-314), e.g.
 * 1-bit digits. One digit per u16 element, in decoder read order. Encode:
 * digits_cap >= n * (ceil(sb / digit_bits) + 1). Decode: optional trace
 * (all three trace pointers, as ilans_decode_trace_u16), FormatError after
 * more than ceil(bits(L) / digit_bits) + 2 refills for one symbol. N in
 * [1, 1024] (ILANS_ERR_UNSUPPORTED beyond). st->max_digits: the most
 * digits one symbol moved. */
int ilans_encode_interleaved_var(const uint8_t *msg, int64_t n, const uint32_t *freq,
                                 int32_t n_freq, const uint32_t *cum, int32_t scale_bits,
                                 int32_t n_lanes, int32_t digit_bits, uint32_t lower_bound,
                                 uint16_t *digits_out, int64_t digits_cap, int64_t *n_digits,
                                 uint32_t *states_out, ilans_status *st);
int ilans_decode_interleaved_var(const uint16_t *payload, int64_t pay_len,
                                 const uint32_t *states, const uint8_t *slot_sym,
                                 int64_t n_slots, const uint32_t *freq, const uint32_t *cum,
                                 int32_t n_freq, int32_t scale_bits, int64_t msg_len,
                                 int32_t n_lanes, int32_t digit_bits, uint32_t lower_bound,
                                 uint8_t *out, int64_t *consumed, uint32_t *trace_states,
                                 uint64_t *trace_pos, int64_t *groups_done, ilans_status *st);

/* Instrumented decode: the device form of interleave.decode_interleaved_steps
 * (interleave.py:251-268) and lanes.decode_lanes_steps (lanes.py:221-232).
 * Same arguments as ilans_decode_interleaved_u16 plus, per completed group g
 * (groups of n_lanes symbols, the last one partial): trace_states[g*N + l] =
 * lane l's state after the group's refills, trace_pos[g] = words read so
 * far; *groups_done = completed groups. On ILANS_ERR_TRUNCATED the trace
 * and the decoded bytes of every completed group are still filled in.
 * trace_states needs ceil(msg_len/N)*N entries, trace_pos ceil(msg_len/N). */
int ilans_decode_trace_u16(const uint16_t *payload, int64_t pay_len, const uint32_t *states,
                           const uint8_t *slot_sym, int64_t n_slots, const uint32_t *freq,
                           const uint32_t *cum, int32_t n_freq, int32_t scale_bits,
                           int64_t msg_len, int32_t n_lanes, uint8_t *out,
                           uint32_t *trace_states, uint64_t *trace_pos, int64_t *groups_done,
                           int64_t *consumed, ilans_status *st);

/* BYTE8 (8-bit digits, L = 2^23) interleaved coding -- the reference's
 * scalar path for variant=BYTE8 (interleave.py:155-179 with
 * rans.encode_symbol_renorm / decode_symbol_renorm, rans.py:266-314), here on
 * the GPU with byte-identical payloads (u8 digits, decoder read order) and
 * final states. Encode: payload_out capacity 3*n bytes. Decode errors:
 * ILANS_ERR_TRUNCATED, ILANS_ERR_FORMAT (more than 5 refills for one symbol:
 * "renormalization does not terminate; corrupt stream", rans.py:309-311).
 * n_lanes in [1, 65535]. The trace variant matches ilans_decode_trace_u16. */
int ilans_encode_interleaved_u8(const uint8_t *msg, int64_t n, const uint32_t *freq,
                                int32_t n_freq, const uint32_t *cum, int32_t scale_bits,
                                int32_t n_lanes, uint8_t *payload_out, int64_t *payload_bytes,
                                uint32_t *states_out, ilans_status *st);
int ilans_decode_interleaved_u8(const uint8_t *payload, int64_t pay_len, const uint32_t *states,
                                const uint8_t *slot_sym, int64_t n_slots, const uint32_t *freq,
                                const uint32_t *cum, int32_t n_freq, int32_t scale_bits,
                                int64_t msg_len, int32_t n_lanes, uint8_t *out,
                                int64_t *consumed, ilans_status *st);
int ilans_decode_trace_u8(const uint8_t *payload, int64_t pay_len, const uint32_t *states,
                          const uint8_t *slot_sym, int64_t n_slots, const uint32_t *freq,
                          const uint32_t *cum, int32_t n_freq, int32_t scale_bits,
                          int64_t msg_len, int32_t n_lanes, uint8_t *out,
                          uint32_t *trace_states, uint64_t *trace_pos, int64_t *groups_done,
                          int64_t *consumed, ilans_status *st);

/* Replaces rans.quantize(counts, scale_bits) (rans.py:171-211), computed on
 * the device. counts has n <= 256 entries; freq_out receives n entries.
 * Errors (ILANS_ERR_VALUE, with the reference's message): scale_bits not in
 * [1,16]; n > 256; all counts zero; more present symbols than 2^scale_bits. */
int ilans_quantize(const uint64_t *counts, int32_t n, int32_t scale_bits, uint32_t *freq_out,
                   ilans_status *st);

/* Replaces np.bincount(msg, minlength=256) at the model-building call sites
 * (cli.py:31-37, bench.py:47-51). counts_out has 256 entries; *alphabet =
 * max symbol + 1 (0 for an empty message). */
int ilans_histogram_u8(const uint8_t *msg, int64_t n, uint64_t *counts_out, int32_t *alphabet,
                       ilans_status *st);

/* -------------------------------------------------------------------------
 * 2. Device-pointer, stream-ordered pipeline (chunk framing)
 *
 * A "table" is an opaque device blob of ilans_table_bytes() bytes holding
 * freq/cum, the encoder's per-symbol reciprocals and the decoder's slot
 * lookup. A "status" is an opaque device blob of ilans_dstatus_bytes().
 * Chunk k of an n-byte message covers bytes [k*C, min((k+1)*C, n)) and is an
 * independent N-lane stream (N <= 32): its payload and final states equal
 * the reference encode_interleaved(msg[kC:(k+1)C], table, N, WORD16).
 * ---------------------------------------------------------------------- */
size_t ilans_table_bytes(void);
size_t ilans_dstatus_bytes(void);

/* Zero d_counts[256] (u64) on `stream`. */
int ilans_counts_zero_dev(uint64_t *d_counts, void *stream);
/* d_counts[b] += #{i : d_msg[i] == b}. Accumulates (call counts_zero first),
 * so shards/batches can share one histogram. */
int ilans_histogram_u8_dev(const uint8_t *d_msg, int64_t n, uint64_t *d_counts, void *stream);
/* Model build: alphabet = highest nonzero bin + 1 (an all-zero histogram
 * maps to counts [1,1], cli.py:32-34), quantize (bit-exact rans.quantize)
 * and all lookup tables, into d_table. Validation errors are recorded in the
 * table blob; read them with ilans_table_read_host. */
int ilans_table_from_counts_dev(const uint64_t *d_counts, int32_t scale_bits, void *d_table,
                                void *stream);
/* Build a table from given frequencies (device pointer, n_freq entries). */
int ilans_table_from_freq_dev(const uint32_t *d_freq, int32_t n_freq, int32_t scale_bits,
                              void *d_table, void *stream);
/* Copy the table header back (synchronizes `stream`): status, alphabet and
 * the quantized frequencies (freq_out: 256 entries, may be NULL). */
int ilans_table_read_host(const void *d_table, int32_t *alphabet, int32_t *scale_bits,
                          uint32_t *freq_out, void *stream, ilans_status *st);

/* Reset a device status blob to "no error". */
int ilans_dstatus_reset_dev(void *d_status, void *stream);
/* Read a device status blob (synchronizes `stream`). */
int ilans_dstatus_read_host(const void *d_status, void *stream, ilans_status *st);
/* Interpret a status blob already copied to host memory (e.g. by a
 * stream-ordered copy into pinned memory): same result as read_host. */
int ilans_dstatus_parse(const void *h_status, ilans_status *st);

/* Chunked encode. d_scratch holds n + 8 words (chunk k uses words
 * [k*C, k*C + len_k), filled from the end); d_chunk_words[k] receives the
 * payload length of chunk k and d_states[k*N + l] its final lane states.
 * C must be a positive multiple of 16. */
int ilans_encode_chunks_dev(const uint8_t *d_msg, int64_t n, int64_t chunk_len,
                            int32_t n_lanes, const void *d_table, int32_t scale_bits,
                            uint16_t *d_scratch, uint32_t *d_chunk_words, uint32_t *d_states,
                            void *d_status, void *stream);
/* As ilans_encode_chunks_dev, for a table quantized on the device from this
 * very message's histogram (ilans_histogram_u8_dev -> ilans_table_from_counts_dev,
 * also after a histogram all-reduce over shards of one message): every
 * symbol of the message then has f >= 1 (rans.py:197-199), so the kernel
 * skips its per-symbol zero-frequency check. With any other table the
 * result is undefined for symbols of frequency 0 -- use
 * ilans_encode_chunks_dev, which reports them. */
int ilans_encode_chunks_covered_dev(const uint8_t *d_msg, int64_t n, int64_t chunk_len,
                                    int32_t n_lanes, const void *d_table, int32_t scale_bits,
                                    uint16_t *d_scratch, uint32_t *d_chunk_words,
                                    uint32_t *d_states, void *d_status, void *stream);
/* Framing: d_word_offsets[0..n_chunks] = exclusive prefix sum of chunk
 * words, and the chunk payloads packed back to back into d_payload
 * (capacity n words) at those offsets. carry_in != 0 continues a previous
 * batch: d_word_offsets[0] is read as the starting offset instead of being
 * set to 0 (so batches of chunks pack into one stream). d_payload may be a
 * mapped pinned host pointer (the packing then streams over PCIe).
 * d_payload == NULL computes the word offsets (the ICH1 directory) only. */
int ilans_frame_chunks_dev(const uint16_t *d_scratch, int64_t n, int64_t chunk_len,
                           const uint32_t *d_chunk_words, uint64_t *d_word_offsets,
                           uint16_t *d_payload, int32_t carry_in, void *stream);
/* Chunked decode of a framed stream: d_out receives n bytes, d_consumed[k]
 * the words chunk k consumed (== its payload length on valid input), and
 * d_final_states (optional, n_chunks*N) the lane states after decoding.
 * scale_bits must equal the table's (the launch is sized on the host without
 * a device round trip; a mismatch is recorded in d_status as a value error).
 * Truncation is recorded in d_status. Reads of d_payload are 16-byte
 * granular and never pass d_payload + d_word_offsets[n_chunks] rounded up to
 * 16 bytes. */
int ilans_decode_chunks_dev(const uint16_t *d_payload, const uint64_t *d_word_offsets,
                            const uint32_t *d_states, int64_t n, int64_t chunk_len,
                            int32_t n_lanes, const void *d_table, int32_t scale_bits,
                            uint8_t *d_out,
                            uint64_t *d_consumed, uint32_t *d_final_states, void *d_status,
                            void *stream);

/* Chunked decode straight from the encoder's slot layout (no framing pass):
 * d_scratch / d_chunk_words / d_states exactly as ilans_encode_chunks_dev
 * left them -- chunk k's w_k = d_chunk_words[k] words right-aligned in its
 * slot [kC + len_k - w_k, kC + len_k). Otherwise as ilans_decode_chunks_dev
 * (d_consumed[k] == w_k on valid input). The packed ICH1 payload is built
 * only when the stream leaves HBM (ilans_frame_chunks_dev). */
int ilans_decode_chunks_slots_dev(const uint16_t *d_scratch, const uint32_t *d_chunk_words,
                                  const uint32_t *d_states, int64_t n, int64_t chunk_len,
                                  int32_t n_lanes, const void *d_table, int32_t scale_bits,
                                  uint8_t *d_out, uint64_t *d_consumed, uint32_t *d_final_states,
                                  void *d_status, void *stream);
/* The fused Adler-32 consumer over the slot layout (see below). */
int ilans_decode_chunks_slots_adler32_dev(const uint16_t *d_scratch,
                                          const uint32_t *d_chunk_words,
                                          const uint32_t *d_states, int64_t n, int64_t chunk_len,
                                          int32_t n_lanes, const void *d_table,
                                          int32_t scale_bits, uint32_t *d_adler,
                                          uint64_t *d_consumed, void *d_status, void *stream);

/* Decode fused with a consumer: the same chunked decode,
 * but the decoded bytes are consumed in registers instead of written to
 * HBM -- here by a zlib-compatible Adler-32 per chunk, d_adler[k] =
 * adler32(chunk k) (after the whole chunk, or after its decoded prefix when
 * the chunk is truncated, which is also recorded in the status).
 * chunk_len <= 2^27 (the position sums are exact in u64 up to there). */
int ilans_decode_chunks_adler32_dev(const uint16_t *d_payload, const uint64_t *d_word_offsets,
                                    const uint32_t *d_states, int64_t n, int64_t chunk_len,
                                    int32_t n_lanes, const void *d_table, int32_t scale_bits,
                                    uint32_t *d_adler, uint64_t *d_consumed, void *d_status,
                                    void *stream);

/* Chunked BYTE8 (8-bit digits, L = 2^23; ICH1 variant 0): chunk k is the
 * reference's encode_interleaved(msg[kC:(k+1)C], table, N, BYTE8)
 * (interleave.py:155-179), one warp per chunk, N in [1, 32], chunk_len <= 2^29.
 * Encode: d_scratch holds 3 bytes per message byte + 16 (chunk k's digits end
 * at 3kC + 3 len_k); d_chunk_bytes[k] = its digit count. Frame: exclusive
 * scan into d_byte_offsets[K + 1] and byte compaction into d_payload (both
 * 4-byte aligned). Decode: d_payload must be 16-byte aligned (ILANS_ERR_VALUE
 * otherwise; it streams into shared rings by 16-byte async copies, which
 * never read past a chunk's last byte); one launch for all chunks, d_consumed[k] = bytes
 * read; errors land in the device status (zero-frequency symbol, exhausted
 * chunk, runaway refill = FormatError). */
int ilans_encode_chunks_u8_dev(const uint8_t *d_msg, int64_t n, int64_t chunk_len,
                               int32_t n_lanes, const void *d_table, uint8_t *d_scratch,
                               uint32_t *d_chunk_bytes, uint32_t *d_states, void *d_status,
                               void *stream);
int ilans_frame_chunks_u8_dev(const uint8_t *d_scratch, int64_t n, int64_t chunk_len,
                              const uint32_t *d_chunk_bytes, uint64_t *d_byte_offsets,
                              uint8_t *d_payload, void *stream);
int ilans_decode_chunks_u8_dev(const uint8_t *d_payload, const uint64_t *d_byte_offsets,
                               const uint32_t *d_states, int64_t n, int64_t chunk_len,
                               int32_t n_lanes, const void *d_table, uint8_t *d_out,
                               uint64_t *d_consumed, void *d_status, void *stream);

/* Per-chunk Adler-32 of bytes already on the device (the unfused
 * consumer, and a device-side integrity check of raw data); chunk_len <= 2^27. */
int ilans_adler32_chunks_dev(const uint8_t *d_data, int64_t n, int64_t chunk_len,
                             uint32_t *d_adler, void *stream);

/* Deterministic synthetic source used by the benches: byte i is
 * the inverse-CDF of a counter-based hash, u = splitmix64(seed ^ i) >> 32,
 * against d_cdf[256] (u32, non-decreasing, last entry is treated as 2^32).
 * Symbol = #{k : d_cdf[k] <= u}, clamped to 255. */
int ilans_synth_bytes_dev(uint8_t *d_out, int64_t n, uint64_t seed, int64_t first_index,
                          const uint32_t *d_cdf, void *stream);

/* -------------------------------------------------------------------------
 * 4. Stream multiplexer (reference pkg/src/ilans/mux.py). K independently
 *    coded streams -- rANS (RansStreamCodec, mux.py:82-128) or raw
 *    fixed-width values (RawStreamCodec, mux.py:131-163) -- merged into one
 *    payload in the byte order a decoder following `schedule` consumes them
 *    (schedule[t] = stream decoded at step t). Host buffers in and out, like
 *    family 1. The merge is a scan + scatter on the device: per-symbol byte
 *    counts come from the encoder (the digits spilled while pushing symbol i
 *    are the ones refilled after popping it), a stable sort of the schedule
 *    maps steps to stream positions, an exclusive scan gives each step's
 *    offset in the muxed payload. Schedules are validated by the caller
 *    (mux.py:259-269); n_steps <= 2^30 - 1, n_streams <= 65535.
 * ---------------------------------------------------------------------- */
enum { ILANS_MUX_RANS = 0, ILANS_MUX_RAW = 1 };

typedef struct ilans_mux_stream {
    int32_t kind;         /* ILANS_MUX_RANS or ILANS_MUX_RAW                        */
    int32_t nbytes;       /* rANS: bytes per digit (digit_bits / 8); raw: per value */
    int32_t digit_bits;   /* rANS digit width (8 or 16); raw: width_bits (1..32)    */
    int32_t scale_bits;   /* rANS table scale_bits                                  */
    uint32_t lower_bound; /* rANS L: states live in [L, L << digit_bits)            */
    int32_t n_sym;        /* rANS alphabet size                                     */
    int64_t freq_off;     /* rANS: freq[freq_off .. +n_sym), cum[cum_off .. +n_sym] */
    int64_t cum_off;
    int64_t slot_off;     /* rANS: slot[slot_off .. + 2^scale_bits) (decode calls)  */
} ilans_mux_stream;

/* Encode every stream in segments and merge them (mux.mux_with_flush,
 * mux.py:329-433; encode_multistream + mux when flush_interval = 0, and
 * encode_multistream alone when schedule lists the streams back to back).
 * symbols: u32 values of stream 0, then stream 1, ... (schedule order within
 * a stream == message order). A stream's steps in epoch t / flush_interval
 * form one segment coded from a fresh state; the first segment's final
 * state is the stream header (stream_state[j]; L for an empty rANS stream),
 * later ones travel inline (4 bytes LE) ahead of the segment's digits.
 * Outputs: the muxed payload (payload_cap >= 8 * n_steps suffices),
 * stream_bytes[j] = stream j's bytes in it, the segment count and the
 * encoder-side buffering peak (MuxBudget.max_buffered).
 * Errors: ILANS_ERR_UNENCODABLE (f == 0; st->stream, st->index = position
 * in the stream, st->symbol), ILANS_ERR_VALUE. */
int ilans_mux_encode(const ilans_mux_stream *streams, int32_t n_streams, const uint32_t *freq,
                     int64_t n_freq, const uint32_t *cum, int64_t n_cum,
                     const uint32_t *symbols, const int32_t *schedule, int64_t n_steps,
                     int64_t flush_interval, uint8_t *payload_out, int64_t payload_cap,
                     int64_t *payload_len, uint32_t *stream_state, uint64_t *stream_bytes,
                     int64_t *segment_count, uint64_t *max_buffered, ilans_status *st);

/* Merge pre-encoded single-segment stream buffers by the schedule
 * (mux.mux, mux.py:283-313): stream j's header is
 * headers[header_off[j] .. header_off[j+1]) and its payload
 * payloads[payload_off[j] .. payload_off[j+1]); symbol_counts[j] symbols.
 * out receives payload_off[K] bytes. Errors, in the reference's order:
 * ILANS_ERR_TRUNCATED / ILANS_ERR_FORMAT for the first stream whose header
 * state cannot load, ILANS_ERR_TRUNCATED when a stream's payload runs out,
 * ILANS_ERR_SCHEDULE for the first stream not fully consumed. */
int ilans_mux_merge(const ilans_mux_stream *streams, int32_t n_streams, const uint32_t *freq,
                    int64_t n_freq, const uint32_t *cum, int64_t n_cum, const uint8_t *slot,
                    int64_t n_slot, const uint8_t *headers, const uint64_t *header_off,
                    const uint8_t *payloads, const uint64_t *payload_off,
                    const int64_t *symbol_counts, const int32_t *schedule, int64_t n_steps,
                    uint8_t *out, ilans_status *st);

/* Decode every stream back out of a muxed payload (mux.demux_decode,
 * mux.py:436-475). symbols_out[t] = the value decoded at schedule step t
 * and/or symbols_by_stream = the same values stream by stream (stream 0's
 * symbols in order, then stream 1's, ...); either pointer may be NULL.
 * Sequential by construction -- each step's read offset depends on the
 * refill counts of all earlier steps -- so one warp walks the schedule,
 * decoding runs of consecutive steps on distinct streams together. *unread
 * = payload bytes left after the walk (the caller's TrailingGarbageWarning).
 * Errors: ILANS_ERR_TRUNCATED, ILANS_ERR_FORMAT (state outside
 * [L, L << digit_bits); st->stream, st->index = step or -1 for a header). */
int ilans_mux_demux(const ilans_mux_stream *streams, int32_t n_streams, const uint32_t *freq,
                    int64_t n_freq, const uint32_t *cum, int64_t n_cum, const uint8_t *slot,
                    int64_t n_slot, const uint8_t *headers, const uint64_t *header_off,
                    const uint8_t *payload, int64_t payload_len, const int32_t *schedule,
                    int64_t n_steps, int64_t flush_interval, uint32_t *symbols_out,
                    uint32_t *symbols_by_stream, int64_t *unread, ilans_status *st);

#ifdef __cplusplus
}
#endif
#endif /* ILANS_B200_H */
