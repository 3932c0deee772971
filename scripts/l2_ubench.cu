// l2_ubench.cu -- dependent random 8-byte loads over a working set of S MB: loads/s vs S, to see
// the effective L2 capacity for uniformly random accesses (the walk kernel's arc loads).
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

__global__ void k_chase(const unsigned long long *__restrict__ A, uint64_t N, int steps,
                        unsigned long long *out)
{
    const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    uint64_t x0 = t * 0x9E3779B97F4A7C15ull, x1 = x0 ^ 0xD1B54A32D192ED03ull;
    for (int j = 0; j < steps; j++) {
        const unsigned long long a0 = __ldg(A + __umul64hi(x0, N));
        const unsigned long long a1 = __ldg(A + __umul64hi(x1, N));
        x0 = (a0 ^ x0) * 0xff51afd7ed558ccdULL;
        x1 = (a1 ^ x1) * 0xc4ceb9fe1a85ec53ULL;
    }
    if (x0 == 42 && x1 == 43) out[0] = x0;
}

__global__ void k_fill(unsigned long long *A, uint64_t N)
{
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < N) {
        uint64_t x = i * 0x9E3779B97F4A7C15ull;
        x ^= x >> 31; x *= 0xff51afd7ed558ccdULL; x ^= x >> 29;
        A[i] = x;
    }
}

int main()
{
    const int sizes_mb[] = {8, 16, 32, 48, 56, 64, 72, 80, 96, 112, 128, 192, 512};
    unsigned long long *A, *out;
    cudaMalloc(&A, 512ull << 20);
    cudaMalloc(&out, 8);
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    const int threads = 256, blocks = nsm * 8;   // 2048 threads/SM, 2 chains each
    const int steps = 400;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int s : sizes_mb) {
        const uint64_t N = ((uint64_t)s << 20) / 8;
        k_fill<<<(unsigned)((N + 255) / 256), 256>>>(A, N);
        k_chase<<<blocks, threads>>>(A, N, 50, out);   // warm
        cudaEventRecord(e0);
        k_chase<<<blocks, threads>>>(A, N, steps, out);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        const double loads = 2.0 * blocks * threads * (double)steps;
        printf("%4d MB  %7.1f G loads/s  (%.3f ms)\n", s, loads / ms / 1e6, ms);
    }
    return 0;
}
