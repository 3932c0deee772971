// dram_mlp_ubench.cu -- dependent random 8-byte loads over a DRAM-resident working set: loads/s
// vs chains per thread (C) and threads per SM, no shared memory.  Upper bound for K6 on graphs
// whose arc array does not fit L2 (configs 2-4).
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

template <int C>
__global__ void k_chase(const unsigned long long *__restrict__ A, uint64_t N, int steps, unsigned long long *out)
{
    const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    uint64_t x[C];
#pragma unroll
    for (int c = 0; c < C; c++) x[c] = (t * C + c) * 0x9E3779B97F4A7C15ull;
    for (int j = 0; j < steps; j++) {
        unsigned long long a[C];
#pragma unroll
        for (int c = 0; c < C; c++) a[c] = __ldg(A + __umul64hi(x[c], N));
#pragma unroll
        for (int c = 0; c < C; c++) x[c] = (a[c] ^ x[c]) * 0xff51afd7ed558ccdULL;
    }
    uint64_t s = 0;
#pragma unroll
    for (int c = 0; c < C; c++) s += x[c];
    if (s == 42) out[0] = s;
}

__global__ void k_fill(unsigned long long *A, uint64_t N)
{
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < N) A[i] = i * 0x9E3779B97F4A7C15ull;
}

template <int C>
void run(const unsigned long long *A, uint64_t N, int ctas, int nsm, unsigned long long *out, const char *tag)
{
    const int threads = 256, blocks = nsm * ctas, steps = 100;
    k_chase<C><<<blocks, threads>>>(A, N, 10, out);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k_chase<C><<<blocks, threads>>>(A, N, steps, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("%s C=%d CTAs/SM=%d  %6.1f G loads/s\n", tag, C, ctas, (double)C * blocks * threads * steps / ms / 1e6);
}

int main()
{
    const uint64_t bytes = 4ull << 30;
    unsigned long long *A, *out;
    cudaMalloc(&A, bytes);
    cudaMalloc(&out, 8);
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    const uint64_t N = bytes / 8;
    k_fill<<<(unsigned)((N + 255) / 256), 256>>>(A, N);
    for (int ctas : {4, 8}) {
        run<1>(A, N, ctas, nsm, out, "4 GB");
        run<2>(A, N, ctas, nsm, out, "4 GB");
        run<4>(A, N, ctas, nsm, out, "4 GB");
        run<8>(A, N, ctas, nsm, out, "4 GB");
    }
    return 0;
}
