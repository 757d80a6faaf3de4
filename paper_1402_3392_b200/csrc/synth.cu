// synth.cu -- deterministic synthetic source for the benches.
//
// byte i = #{k < 255 : cdf[k] <= u_i}, u_i = splitmix64(seed ^ i) >> 32.
// Counter-based, so any shard / batch regenerates identical bytes and the
// numpy twin (paper_1402_3392_b200/synth.py) reproduces them on the host.
#include "common.cuh"
#include "kernels.cuh"

namespace ilans {

__device__ __forceinline__ uint64_t splitmix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__device__ __forceinline__ uint32_t synth_symbol(uint64_t seed, uint64_t i, const uint32_t *cdf) {
    const uint32_t u = static_cast<uint32_t>(splitmix64(seed ^ i) >> 32);
    int lo = 0, hi = 255;  // count of cdf[0..254] <= u  (upper bound)
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (cdf[mid] <= u) lo = mid + 1; else hi = mid;
    }
    return static_cast<uint32_t>(lo);
}

__global__ void __launch_bounds__(256)
synth_kernel(uint8_t *__restrict__ out, int64_t n, uint64_t seed, int64_t first,
             const uint32_t *__restrict__ g_cdf) {
    __shared__ uint32_t cdf[256];
    cdf[threadIdx.x] = g_cdf[threadIdx.x];
    __syncthreads();
    const int64_t nvec = n >> 4;
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t v = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; v < nvec;
         v += stride) {
        uint32_t w[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            uint32_t acc = 0;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const uint64_t i = static_cast<uint64_t>(first + v * 16 + q * 4 + j);
                acc |= synth_symbol(seed, i, cdf) << (8 * j);
            }
            w[q] = acc;
        }
        reinterpret_cast<uint4 *>(out)[v] = make_uint4(w[0], w[1], w[2], w[3]);
    }
    if (blockIdx.x == 0 && threadIdx.x < (n & 15)) {
        const int64_t i = (nvec << 4) + threadIdx.x;
        out[i] = static_cast<uint8_t>(synth_symbol(seed, static_cast<uint64_t>(first + i), cdf));
    }
}

cudaError_t launch_synth(uint8_t *d_out, int64_t n, uint64_t seed, int64_t first_index,
                         const uint32_t *d_cdf, cudaStream_t stream) {
    if (n <= 0) return cudaSuccess;
    int64_t blocks = ((n >> 4) + 255) / 256;
    const int64_t cap = int64_t(sm_count()) * 16;
    if (blocks > cap) blocks = cap;
    if (blocks < 1) blocks = 1;
    synth_kernel<<<static_cast<unsigned>(blocks), 256, 0, stream>>>(d_out, n, seed, first_index,
                                                                    d_cdf);
    ilans_note_launch();
    return cudaGetLastError();
}

}  // namespace ilans
