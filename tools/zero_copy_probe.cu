// Zero-copy PCIe probe: kernels streaming from / to mapped pinned host
// memory (16-byte loads / stores per thread, grid-stride), alone and both
// directions at once, vs cudaMemcpyAsync. nvcc -arch=sm_100a -O3 zero_copy_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void h2d_kernel(const uint4 *__restrict__ src, uint4 *__restrict__ dst, size_t n16) {
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n16;
         i += size_t(gridDim.x) * blockDim.x)
        dst[i] = src[i];
}

int main() {
    const size_t n = size_t(256) << 20;
    void *h_in, *h_out, *d_in, *d_out, *h_in_d, *h_out_d;
    cudaHostAlloc(&h_in, n, cudaHostAllocMapped);
    cudaHostAlloc(&h_out, n, cudaHostAllocMapped);
    cudaMalloc(&d_in, n);
    cudaMalloc(&d_out, n);
    cudaHostGetDevicePointer(&h_in_d, h_in, 0);
    cudaHostGetDevicePointer(&h_out_d, h_out, 0);
    cudaStream_t s1, s2;
    cudaStreamCreate(&s1);
    cudaStreamCreate(&s2);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const size_t n16 = n / 16;
    float ms;
    for (int blocks : {148, 296, 592, 1184}) {
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(a, s1);
            h2d_kernel<<<blocks, 512, 0, s1>>>((const uint4 *)h_in_d, (uint4 *)d_in, n16);
            cudaEventRecord(b, s1);
            cudaEventSynchronize(b);
        }
        cudaEventElapsedTime(&ms, a, b);
        printf("zero-copy read  (H->D) blocks %4d: %6.1f GB/s\n", blocks, n / ms / 1e6);
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(a, s1);
            h2d_kernel<<<blocks, 512, 0, s1>>>((const uint4 *)d_out, (uint4 *)h_out_d, n16);
            cudaEventRecord(b, s1);
            cudaEventSynchronize(b);
        }
        cudaEventElapsedTime(&ms, a, b);
        printf("zero-copy write (D->H) blocks %4d: %6.1f GB/s\n", blocks, n / ms / 1e6);
        for (int rep = 0; rep < 2; ++rep) {
            cudaDeviceSynchronize();
            cudaEventRecord(a, s1);
            h2d_kernel<<<blocks / 2, 512, 0, s1>>>((const uint4 *)h_in_d, (uint4 *)d_in, n16);
            h2d_kernel<<<blocks / 2, 512, 0, s2>>>((const uint4 *)d_out, (uint4 *)h_out_d, n16);
            cudaDeviceSynchronize();
            cudaEventRecord(b, s1);
            cudaEventSynchronize(b);
        }
        cudaEventElapsedTime(&ms, a, b);
        printf("zero-copy both directions blocks %4d: %6.1f GB/s each\n", blocks, n / ms / 1e6);
    }
    for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(a, s1);
        cudaMemcpyAsync(d_in, h_in, n, cudaMemcpyHostToDevice, s1);
        cudaEventRecord(b, s1);
        cudaEventSynchronize(b);
    }
    cudaEventElapsedTime(&ms, a, b);
    printf("cudaMemcpyAsync H->D: %6.1f GB/s\n", n / ms / 1e6);
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
