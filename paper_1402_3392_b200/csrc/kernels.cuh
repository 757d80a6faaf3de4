// kernels.cuh -- kernel declarations and host-side launchers shared between
// the translation units of libilans_b200.so.
#pragma once

#include "common.cuh"

namespace ilans {

// table.cu
__global__ void histogram_u8_kernel(const uint8_t *__restrict__ msg, int64_t n,
                                    unsigned long long *__restrict__ counts);
__global__ void build_table_kernel(const unsigned long long *__restrict__ counts,
                                   const uint32_t *freq_in, int n_freq, const uint32_t *cum_in,
                                   const uint8_t *slot_in, int scale_bits, TableDev *t);

// CTAs of a table build from counts: the slot tables (>= 1024 slots) are
// split so each thread writes 4 or more (sb 12: 4 CTAs ... sb >= 14: 16)
__host__ __device__ constexpr int table_parts(int scale_bits) {
    return scale_bits >= 14 ? 16 : scale_bits >= 10 ? (1 << (scale_bits - 10)) : 1;
}

// Host launchers (all asynchronous on `stream`; return cudaError_t).
cudaError_t launch_histogram(const uint8_t *d_msg, int64_t n, unsigned long long *d_counts,
                             cudaStream_t stream);
cudaError_t launch_build_table(const unsigned long long *d_counts, const uint32_t *d_freq,
                               int n_freq, const uint32_t *d_cum, const uint8_t *d_slot,
                               int scale_bits, TableDev *d_table, cudaStream_t stream);

// encode.cu -- chunked encode (N <= 32: one warp per chunk; N > 32: one CTA
// per stream), then framing (scan + compaction).
// Raise a kernel's dynamic shared-memory limit to at least `bytes` (once per
// device and size: the driver call costs microseconds per launch otherwise).
cudaError_t smem_limit(const void *kernel, int bytes);

cudaError_t launch_encode(const uint8_t *d_msg, int64_t n, int64_t chunk_len, int n_lanes,
                          const TableDev *d_table, int scale_bits, uint16_t *d_scratch,
                          uint32_t *d_chunk_words, uint32_t *d_states, DStatus *d_status,
                          uint32_t *d_lane_ws, cudaStream_t stream, bool stats = false,
                          bool covered = false);
cudaError_t launch_frame(const uint16_t *d_scratch, int64_t n, int64_t chunk_len,
                         const uint32_t *d_chunk_words, uint64_t *d_word_offsets,
                         uint16_t *d_payload, int carry_in, cudaStream_t stream);

// decode.cu
cudaError_t launch_decode(const uint16_t *d_payload, const uint64_t *d_word_offsets,
                          const uint32_t *d_states, int64_t n, int64_t chunk_len, int n_lanes,
                          const TableDev *d_table, int scale_bits, bool packed,
                          uint8_t *d_out, uint64_t *d_consumed, uint32_t *d_final_states,
                          DStatus *d_status, uint32_t *d_lane_ws, cudaStream_t stream,
                          DecodeTrace trace = DecodeTrace{nullptr, nullptr, nullptr, 0},
                          const uint32_t *d_slot_words = nullptr);
cudaError_t launch_adler32_chunks(const uint8_t *d_data, int64_t n, int64_t chunk_len,
                                  uint32_t *d_adler, cudaStream_t stream);
// decode fused with its consumer: per-chunk Adler-32 of the decoded bytes,
// which never reach HBM (N <= 32)
cudaError_t launch_decode_adler32(const uint16_t *d_payload, const uint64_t *d_word_offsets,
                                  const uint32_t *d_states, int64_t n, int64_t chunk_len,
                                  int n_lanes, const TableDev *d_table, int scale_bits,
                                  uint32_t *d_adler, uint64_t *d_consumed, DStatus *d_status,
                                  cudaStream_t stream, const uint32_t *d_slot_words = nullptr);

// byte8.cu -- single-stream byte8 codec (N <= 32 warp, N > 32 CTA)
cudaError_t launch_encode_u8(const uint8_t *d_msg, int64_t n, int n_lanes, const TableDev *d_table,
                             uint8_t *d_scratch, uint32_t *d_bytes, uint32_t *d_states,
                             DStatus *d_status, uint32_t *d_lane_ws, cudaStream_t stream);
cudaError_t launch_decode_u8(const uint8_t *d_payload, uint64_t pay_len, const uint64_t *d_offsets,
                             const uint32_t *d_states, int64_t n, int n_lanes,
                             const TableDev *d_table, uint8_t *d_out, uint64_t *d_consumed,
                             DStatus *d_status, uint32_t *d_lane_ws, cudaStream_t stream,
                             DecodeTrace trace);
// chunked byte8: one warp per chunk, byte framing (ICH1 variant 0)
cudaError_t launch_encode_chunks_u8(const uint8_t *d_msg, int64_t n, int64_t chunk_len,
                                    int n_lanes, const TableDev *d_table, uint8_t *d_scratch,
                                    uint32_t *d_bytes, uint32_t *d_states, DStatus *d_status,
                                    cudaStream_t stream);
cudaError_t launch_frame_u8(const uint8_t *d_scratch, int64_t n, int64_t chunk_len,
                            const uint32_t *d_bytes, uint64_t *d_offsets, uint8_t *d_payload,
                            cudaStream_t stream);
cudaError_t launch_decode_chunks_u8(const uint8_t *d_payload, const uint64_t *d_offsets,
                                    const uint32_t *d_states, int64_t n, int64_t chunk_len,
                                    int n_lanes, const TableDev *d_table, uint8_t *d_out,
                                    uint64_t *d_consumed, DStatus *d_status, cudaStream_t stream);

// synth.cu
cudaError_t launch_synth(uint8_t *d_out, int64_t n, uint64_t seed, int64_t first_index,
                         const uint32_t *d_cdf, cudaStream_t stream);

__global__ void dstatus_reset_kernel(DStatus *s);
// encode.cu: exclusive scan of per-chunk sizes into u64 offsets (one CTA)
__global__ void chunk_offsets_kernel(const uint32_t *__restrict__ words, int64_t n_chunks,
                                     uint64_t *__restrict__ offsets, int carry_in);

int sm_count();


// variant.cu -- any RenormVariant (the reference's scalar path), one warp
// per stream, N <= kVarMaxLanes.
constexpr int kVarMaxLanes = 1024;
cudaError_t launch_encode_var(const uint8_t *d_msg, int64_t n, int n_lanes,
                              const TableDev *d_table, int bits, uint32_t lbound,
                              uint16_t *d_stack, int64_t cap, uint64_t *d_digits,
                              uint32_t *d_states, DStatus *d_status, cudaStream_t stream);
cudaError_t launch_decode_var(const uint16_t *d_payload, int64_t plen, const uint32_t *d_states,
                              int64_t n, int n_lanes, const TableDev *d_table, int bits,
                              uint32_t lbound, uint8_t *d_out, uint64_t *d_consumed,
                              DStatus *d_status, cudaStream_t stream, DecodeTrace trace);

}  // namespace ilans
