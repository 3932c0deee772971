// l1_mlp_ubench.cu -- dependent random 8-byte loads (2 chains/thread, 256-thread CTAs): load
// flavour (ld.global.nc / .cg / .ca / L1::no_allocate) x shared memory per CTA (which shrinks the
// L1) x working set.  Shows whether outstanding L1 misses are bounded by L1 capacity.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

template <int MODE>
__device__ __forceinline__ unsigned long long ld(const unsigned long long *p)
{
    unsigned long long v;
    if (MODE == 0) v = __ldg(p);
    else if (MODE == 1) asm volatile("ld.global.cg.u64 %0, [%1];" : "=l"(v) : "l"(p));
    else if (MODE == 2) asm volatile("ld.global.nc.L1::no_allocate.u64 %0, [%1];" : "=l"(v) : "l"(p));
    else asm volatile("ld.global.ca.u64 %0, [%1];" : "=l"(v) : "l"(p));
    return v;
}

template <int MODE>
__global__ void k_chase(const unsigned long long *__restrict__ A, uint64_t N, int steps, unsigned long long *out)
{
    extern __shared__ int pad[];
    const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    uint64_t x0 = t * 0x9E3779B97F4A7C15ull, x1 = x0 ^ 0xD1B54A32D192ED03ull;
    for (int j = 0; j < steps; j++) {
        const unsigned long long a0 = ld<MODE>(A + __umul64hi(x0, N));
        const unsigned long long a1 = ld<MODE>(A + __umul64hi(x1, N));
        x0 = (a0 ^ x0) * 0xff51afd7ed558ccdULL;
        x1 = (a1 ^ x1) * 0xc4ceb9fe1a85ec53ULL;
    }
    if (x0 == 42 && x1 == 43) out[0] = x0 + pad[0];
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

template <int MODE>
double run(const unsigned long long *A, uint64_t N, int smem_kb, int ctas_per_sm, int nsm, unsigned long long *out)
{
    const int threads = 256, blocks = nsm * ctas_per_sm, steps = 300;
    const size_t smem = smem_kb == 1 ? 128 : (size_t)smem_kb * 1024;   // "1" = 128 B
    cudaFuncSetAttribute(k_chase<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_chase<MODE><<<blocks, threads, smem>>>(A, N, 30, out);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k_chase<MODE><<<blocks, threads, smem>>>(A, N, steps, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    return 2.0 * blocks * threads * (double)steps / ms / 1e6;
}

int main()
{
    unsigned long long *A, *out;
    cudaMalloc(&A, 512ull << 20);
    cudaMalloc(&out, 8);
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    const char *names[4] = {"nc", "cg", "nc.no_alloc", "ca"};
    for (int mb : {32, 80}) {
        const uint64_t N = ((uint64_t)mb << 20) / 8;
        k_fill<<<(unsigned)((N + 255) / 256), 256>>>(A, N);
        for (int ctas : {4, 8}) {
            for (int smem_kb : {0, 1, 4, 8, 16, 24, 50}) {
                if (ctas * (smem_kb + 1) > 227) continue;
                printf("%3d MB ctas/SM %d smem %2d KB :", mb, ctas, smem_kb);
                printf("  %s %6.1f", names[0], run<0>(A, N, smem_kb, ctas, nsm, out));
                printf("  %s %6.1f", names[1], run<1>(A, N, smem_kb, ctas, nsm, out));
                printf("  %s %6.1f", names[2], run<2>(A, N, smem_kb, ctas, nsm, out));
                printf("  %s %6.1f G loads/s\n", names[3], run<3>(A, N, smem_kb, ctas, nsm, out));
            }
        }
    }
    return 0;
}
