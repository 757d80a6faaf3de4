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
constexpr int kPackedMaxBits = 12;           // packed 32-bit slot entry: sym|f-1|bias

// Table flags
constexpr uint32_t kTabPacked = 1u;          // packed[] valid (sb <= 12, consistent)

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
    uint4 enc[kMaxSym];               // {f, cum, magic, sh1 | sh2 << 8 | thr_shift << 16}
    uint2 dec[kMaxSym];               // {f, cum} for the decoder's second lookup
    uint32_t packed[1 << kPackedMaxBits];  // sym | (f-1) << 8 | bias << 20
    uint8_t slot_sym[1 << kMaxScaleBits];
};

// Device status blob (first error wins, deterministic by index).
struct alignas(16) DStatus {
    unsigned long long trunc_stream;  // min failing stream index, ~0 = none
    long long unenc_index;            // max offending message index, -1 = none
    uint32_t unenc_symbol;
    uint32_t value_error;
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

// Granlund-Montgomery exact unsigned division by an invariant d in [1, 2^16]
// for every 32-bit numerator ("Division by invariant integers using
// multiplication", PLDI'94, fig. 4.1): q = (t + ((n - t) >> sh1)) >> sh2,
// t = umulhi(magic, n). Verified exhaustively per d on the host oracle side
// (tests/test_division.py) and on device (tests/test_gpu_parity.py).
__host__ __device__ inline void divmagic(uint32_t d, uint32_t *magic, uint32_t *sh1,
                                         uint32_t *sh2) {
    uint32_t l = 0;
    while ((1ull << l) < d) ++l;  // l = ceil(log2 d)
    uint64_t m = ((((1ull << l) - d) << 32) / d) + 1;
    *magic = static_cast<uint32_t>(m);
    *sh1 = l < 1 ? l : 1;
    *sh2 = l > 0 ? l - 1 : 0;
}

__device__ __forceinline__ uint32_t div_magic(uint32_t n, uint32_t magic, uint32_t sh1,
                                              uint32_t sh2) {
    uint32_t t = __umulhi(magic, n);
    return (t + ((n - t) >> sh1)) >> sh2;
}

}  // namespace ilans

// Host-side launch accounting (ilans_launch_count).
void ilans_note_launch(int n = 1);
