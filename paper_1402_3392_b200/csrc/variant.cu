// variant.cu -- interleaved rANS with any RenormVariant (digit_bits in
// [1, 16], lower bound L with L % 2^sb == 0 and L << digit_bits <= 2^32):
// the reference's scalar path for variants other than word16 / byte8
// (interleave.py:155-179 over rans.encode_symbol_renorm /
// decode_symbol_renorm, rans.py:266-314), e.g. the 1-bit "toy" digits of
// its tests. A compatibility path: one warp per stream, lanes in sub-groups
// of 32, lane states in shared memory (N <= kVarMaxLanes).
//
// Encode walks groups backwards. A lane spills k digits while x >= T =
// f (state_limit >> sb) (a pure function of x), so a warp scan of k gives
// each lane its read-order offset: inside a group lanes ascend, each lane's
// digits most significant first (the reversed emission order of the
// reference's stack). Decode pops every lane of a group in parallel, then
// refills lane by lane in ascending order (a refill count can depend on the
// digits read when L is not a multiple of the digit radix powers), with the
// reference's limit on refills per symbol (FormatError).
#include "common.cuh"
#include "kernels.cuh"

namespace ilans {

__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t v, int lane) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t u = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += u;
    }
    return v;
}

__global__ void __launch_bounds__(32)
encode_var_kernel(const uint8_t *__restrict__ msg, int64_t n, int n_lanes,
                  const TableDev *__restrict__ tab, int bits, uint32_t lbound,
                  uint16_t *__restrict__ stack, int64_t cap, uint64_t *__restrict__ n_digits,
                  uint32_t *__restrict__ states_out, DStatus *__restrict__ status) {
    __shared__ uint32_t ws[kVarMaxLanes];
    const int lane = threadIdx.x;
    const int sb = static_cast<int>(tab->scale_bits);
    const uint32_t m = 1u << sb;
    const uint64_t per_f = (static_cast<uint64_t>(lbound) << bits) >> sb;  // state_limit >> sb
    const uint32_t dmask = (1u << bits) - 1u;
    for (int l = lane; l < n_lanes; l += 32) ws[l] = lbound;
    __syncwarp();
    int64_t top = cap;
    uint32_t most = 0;
    bool bad = false;
    for (int64_t gi = (n + n_lanes - 1) / n_lanes - 1; gi >= 0 && !bad; --gi) {
        const int64_t base = gi * n_lanes;
        const int active = (n - base) < n_lanes ? static_cast<int>(n - base) : n_lanes;
        for (int j0 = ((active - 1) >> 5) << 5; j0 >= 0; j0 -= 32) {
            const int l = j0 + lane;
            const bool on = l < active;
            const uint32_t s = on ? msg[base + l] : 0u;
            const uint32_t f = on ? tab->freq[s] : 1u;
            const uint32_t badmask = __ballot_sync(0xffffffffu, on && f == 0u);
            if (badmask) {  // the highest offending index (the reference walks down)
                if (lane == 0)
                    atomicMax(&status->unenc_index,
                              static_cast<long long>(base + j0 + 31 - __clz(badmask)));
                bad = true;
                break;
            }
            uint32_t x = on ? ws[l] : 0u;
            const uint64_t thr = static_cast<uint64_t>(f) * per_f;
            uint32_t k = 0;
            uint32_t xs = x;
            while (on && static_cast<uint64_t>(xs) >= thr) {  // spill loop (rans.py:284-287)
                xs = bits < 32 ? xs >> bits : 0u;
                ++k;
            }
            const uint32_t incl = warp_incl_scan(k, lane);
            const uint32_t tot = __shfl_sync(0xffffffffu, incl, 31);
            top -= tot;
            const int64_t p = top + (incl - k);
            for (uint32_t j = 0; j < k; ++j)  // most significant first
                stack[p + j] = static_cast<uint16_t>((x >> (bits * (k - 1u - j))) & dmask);
            if (on) {
                const uint32_t c = tab->cum[s];
                ws[l] = (xs / f) * m + c + xs % f;
            }
            most = max(most, k);
        }
        __syncwarp();
    }
    most = __reduce_max_sync(0xffffffffu, most);
    if (lane == 0) atomicMax(&status->max_digits, most);
    if (!bad) {
        if (lane == 0) *n_digits = static_cast<uint64_t>(cap - top);
        for (int l = lane; l < n_lanes; l += 32) states_out[l] = ws[l];
    }
}

__global__ void __launch_bounds__(32)
decode_var_kernel(const uint16_t *__restrict__ payload, int64_t plen,
                  const uint32_t *__restrict__ states, int64_t n, int n_lanes,
                  const TableDev *__restrict__ tab, int bits, uint32_t lbound,
                  uint8_t *__restrict__ out, uint64_t *__restrict__ consumed,
                  DStatus *__restrict__ status, DecodeTrace trace) {
    __shared__ uint32_t ws[kVarMaxLanes];
    const int lane = threadIdx.x;
    const int sb = static_cast<int>(tab->scale_bits);
    const uint32_t mask = (1u << sb) - 1u;
    // the reference's bound on refills per symbol (rans.py:305)
    const int limit = (32 - __clz(lbound) + bits - 1) / bits + 2;
    for (int l = lane; l < n_lanes; l += 32) ws[l] = states[l];
    __syncwarp();
    int64_t pos = 0;
    int err = 0;
    uint32_t most = 0;
    int64_t base = 0;
    for (; base < n; base += n_lanes) {
        const int active = (n - base) < n_lanes ? static_cast<int>(n - base) : n_lanes;
        for (int l = lane; l < active; l += 32) {  // pops (rans.pop_symbol, rans.py:222-226)
            const uint32_t x = ws[l];
            const uint32_t slot = x & mask;
            const uint32_t s = tab->slot_sym[slot];
            out[base + l] = static_cast<uint8_t>(s);
            ws[l] = static_cast<uint32_t>(static_cast<uint64_t>(tab->freq[s]) * (x >> sb) + slot -
                                          tab->cum[s]);
        }
        __syncwarp();
        if (lane == 0) {  // refills, lanes ascending
            for (int l = 0; l < active && !err; ++l) {
                uint32_t x = ws[l];
                int r = 0;
                while (x < lbound) {
                    if (pos >= plen) { err = ILANS_ERR_TRUNCATED; break; }
                    x = (x << bits) | payload[pos++];
                    if (++r > limit) { err = ILANS_ERR_FORMAT; break; }
                }
                ws[l] = x;
                most = max(most, static_cast<uint32_t>(r));
            }
        }
        pos = __shfl_sync(0xffffffffu, pos, 0);
        err = __shfl_sync(0xffffffffu, err, 0);
        __syncwarp();
        if (err) break;
        if (trace.states) {
            const int64_t gi = base / n_lanes;
            for (int l = lane; l < n_lanes; l += 32) trace.states[gi * n_lanes + l] = ws[l];
            if (lane == 0) trace.pos[gi] = static_cast<uint64_t>(pos);
        }
    }
    if (lane == 0) {
        atomicMax(&status->max_digits, most);
        if (err == ILANS_ERR_TRUNCATED) atomicMin(&status->trunc_stream, 0ull);
        if (err == ILANS_ERR_FORMAT) status->value_error = ILANS_ERR_FORMAT;
        if (consumed) *consumed = static_cast<uint64_t>(pos);
        if (trace.groups)
            trace.groups[0] = (base < n ? base : n + n_lanes - 1) / n_lanes;
    }
}

cudaError_t launch_encode_var(const uint8_t *d_msg, int64_t n, int n_lanes,
                              const TableDev *d_table, int bits, uint32_t lbound,
                              uint16_t *d_stack, int64_t cap, uint64_t *d_digits,
                              uint32_t *d_states, DStatus *d_status, cudaStream_t stream) {
    encode_var_kernel<<<1, 32, 0, stream>>>(d_msg, n, n_lanes, d_table, bits, lbound, d_stack,
                                            cap, d_digits, d_states, d_status);
    ilans_note_launch();
    return cudaGetLastError();
}

cudaError_t launch_decode_var(const uint16_t *d_payload, int64_t plen, const uint32_t *d_states,
                              int64_t n, int n_lanes, const TableDev *d_table, int bits,
                              uint32_t lbound, uint8_t *d_out, uint64_t *d_consumed,
                              DStatus *d_status, cudaStream_t stream, DecodeTrace trace) {
    decode_var_kernel<<<1, 32, 0, stream>>>(d_payload, plen, d_states, n, n_lanes, d_table, bits,
                                            lbound, d_out, d_consumed, d_status, trace);
    ilans_note_launch();
    return cudaGetLastError();
}

}  // namespace ilans
