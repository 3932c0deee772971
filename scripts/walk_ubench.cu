// walk_ubench.cu -- microbenchmark of the bare random-walk chain on a CSR graph (no y probes):
// how many walk steps/s the B200 memory system sustains for the dependent-load chain, as a
// function of the arc layout and the number of independent chains per thread.
// Usage: walk_ubench <graph.bin>   (int64 n, int64 nnz, int64 off[n+1], int32 cols[nnz])
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include <vector>

struct U4 { uint32_t x, y, z, w; };
__device__ __forceinline__ U4 philox(U4 c, uint32_t k0, uint32_t k1)
{
#pragma unroll
    for (int r = 0; r < 10; r++) {
        const uint32_t lo0 = 0xD2511F53u * c.x, hi0 = __umulhi(0xD2511F53u, c.x);
        const uint32_t lo1 = 0xCD9E8D57u * c.z, hi1 = __umulhi(0xCD9E8D57u, c.z);
        c = U4{hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0};
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    return c;
}

// packed arc: u | off | deg with bo/bd bits
template <int C, bool PHILOX>
__global__ void k_packed(int64_t nwalks, int lf, const unsigned long long *__restrict__ parcs,
                         const uint2 *__restrict__ rec, int n, int bo, int bd, unsigned long long *out)
{
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t * C >= nwalks) return;
    uint2 R[C];
    uint32_t v[C];
    uint64_t ck = 0;
#pragma unroll
    for (int c = 0; c < C; c++) {
        v[c] = (uint32_t)(((t * C + c) * 2654435761ull) % (uint64_t)n);
        R[c] = rec[v[c]];
    }
    const unsigned long long mo = (1ull << bo) - 1, md = (1ull << bd) - 1;
    for (int j = 0; j < lf; j++) {
#pragma unroll
        for (int c = 0; c < C; c++) {
            uint64_t r64;
            if (PHILOX) {
                const U4 r = philox(U4{(uint32_t)j, (uint32_t)(t * C + c), 7u, 0u}, 1u, 2u);
                r64 = ((uint64_t)r.y << 32) | r.x;
            } else {
                uint64_t x = (uint64_t)(t * C + c) * 0x9E3779B97F4A7C15ull + (uint64_t)j * 0xD1B54A32D192ED03ull;
                x ^= x >> 31; x *= 0xff51afd7ed558ccdULL; x ^= x >> 29;
                r64 = x;
            }
            const unsigned long long a = __ldg(parcs + (uint64_t)R[c].x + __umul64hi(r64, (uint64_t)R[c].y));
            R[c] = make_uint2((uint32_t)((a >> bd) & mo), (uint32_t)(a & md));
            v[c] = (uint32_t)(a >> (bo + bd));
        }
    }
#pragma unroll
    for (int c = 0; c < C; c++) ck += v[c];
    atomicAdd(out, ck);
}

template <int C>
__global__ void k_cols(int64_t nwalks, int lf, const int32_t *__restrict__ cols, const uint2 *__restrict__ rec, int n,
                       unsigned long long *out)
{
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t * C >= nwalks) return;
    uint32_t v[C];
    uint64_t ck = 0;
#pragma unroll
    for (int c = 0; c < C; c++) v[c] = (uint32_t)(((t * C + c) * 2654435761ull) % (uint64_t)n);
    for (int j = 0; j < lf; j++) {
#pragma unroll
        for (int c = 0; c < C; c++) {
            uint64_t x = (uint64_t)(t * C + c) * 0x9E3779B97F4A7C15ull + (uint64_t)j * 0xD1B54A32D192ED03ull;
            x ^= x >> 31; x *= 0xff51afd7ed558ccdULL; x ^= x >> 29;
            const uint2 R = __ldg(rec + v[c]);
            v[c] = (uint32_t)__ldg(cols + (uint64_t)R.x + __umul64hi(x, (uint64_t)R.y));
        }
    }
#pragma unroll
    for (int c = 0; c < C; c++) ck += v[c];
    atomicAdd(out, ck);
}

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

template <class F>
float timeit(F f)
{
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    f();
    CK(cudaDeviceSynchronize());
    cudaEventRecord(a);
    f();
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    return ms;
}

int main(int argc, char **argv)
{
    FILE *fp = fopen(argv[1], "rb");
    int64_t n, nnz;
    fread(&n, 8, 1, fp);
    fread(&nnz, 8, 1, fp);
    std::vector<int64_t> off(n + 1);
    std::vector<int32_t> cols(nnz);
    fread(off.data(), 8, n + 1, fp);
    fread(cols.data(), 4, nnz, fp);
    fclose(fp);
    int md = 0;
    for (int64_t v = 0; v < n; v++) md = std::max<int>(md, (int)(off[v + 1] - off[v]));
    auto bits = [](uint64_t x) { int b = 1; while (b < 64 && (1ull << b) <= x) b++; return b; };
    const int bo = bits(nnz), bd = bits(md);
    std::vector<uint2> rec(n);
    for (int64_t v = 0; v < n; v++) rec[v] = make_uint2((uint32_t)off[v], (uint32_t)(off[v + 1] - off[v]));
    std::vector<unsigned long long> pa(nnz);
    for (int64_t e = 0; e < nnz; e++) {
        const int u = cols[e];
        pa[e] = ((unsigned long long)u << (bo + bd)) | ((unsigned long long)rec[u].x << bd) | rec[u].y;
    }
    unsigned long long *d_pa, *d_out;
    uint2 *d_rec;
    int32_t *d_cols;
    CK(cudaMalloc(&d_pa, 8 * nnz));
    CK(cudaMalloc(&d_cols, 4 * nnz));
    CK(cudaMalloc(&d_rec, 8 * n));
    CK(cudaMalloc(&d_out, 8));
    CK(cudaMemcpy(d_pa, pa.data(), 8 * nnz, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_cols, cols.data(), 4 * nnz, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_rec, rec.data(), 8 * n, cudaMemcpyHostToDevice));
    printf("n=%lld nnz=%lld maxdeg=%d packed=%.1f MB cols=%.1f MB\n", (long long)n, (long long)nnz, md,
           8.0 * nnz / 1e6, 4.0 * nnz / 1e6);
    const int lf = 64;
    for (int64_t nw : {1ll << 18, 1ll << 20, 1ll << 22}) {
#define RUN(NAME, C, KERNEL, ...)                                                                       \
        {                                                                                               \
            const int64_t thr = (nw + C - 1) / C;                                                       \
            float ms = timeit([&] { KERNEL<<<(unsigned)((thr + 255) / 256), 256>>>(__VA_ARGS__); });    \
            printf("%-16s walks=%8lld C=%d  %7.3f ms  %7.1f Gsteps/s\n", NAME, (long long)nw, C, ms,     \
                   (double)nw * lf / ms / 1e6);                                                         \
        }
        RUN("packed_hash", 1, (k_packed<1, false>), nw, lf, d_pa, d_rec, (int)n, bo, bd, d_out);
        RUN("packed_hash", 2, (k_packed<2, false>), nw, lf, d_pa, d_rec, (int)n, bo, bd, d_out);
        RUN("packed_hash", 4, (k_packed<4, false>), nw, lf, d_pa, d_rec, (int)n, bo, bd, d_out);
        RUN("packed_hash", 8, (k_packed<8, false>), nw, lf, d_pa, d_rec, (int)n, bo, bd, d_out);
        RUN("packed_philox", 1, (k_packed<1, true>), nw, lf, d_pa, d_rec, (int)n, bo, bd, d_out);
        RUN("packed_philox", 2, (k_packed<2, true>), nw, lf, d_pa, d_rec, (int)n, bo, bd, d_out);
        RUN("packed_philox", 4, (k_packed<4, true>), nw, lf, d_pa, d_rec, (int)n, bo, bd, d_out);
        // the same chains at 4 resident CTAs of 256 threads per SM (K6's occupancy): 50 KB of
        // dynamic shared memory per CTA caps residency
#define RUN4(NAME, C, KERNEL, ...)                                                                      \
        {                                                                                               \
            const int64_t thr = (nw + C - 1) / C;                                                       \
            cudaFuncSetAttribute(KERNEL, cudaFuncAttributeMaxDynamicSharedMemorySize, 50 * 1024);       \
            float ms = timeit([&] { KERNEL<<<(unsigned)((thr + 255) / 256), 256, 50 * 1024>>>(__VA_ARGS__); }); \
            printf("%-16s walks=%8lld C=%d  %7.3f ms  %7.1f Gsteps/s  (4 CTAs/SM)\n", NAME, (long long)nw, C, ms, \
                   (double)nw * lf / ms / 1e6);                                                         \
        }
        RUN4("packed_philox", 2, (k_packed<2, true>), nw, lf, d_pa, d_rec, (int)n, bo, bd, d_out);
        RUN4("packed_philox", 4, (k_packed<4, true>), nw, lf, d_pa, d_rec, (int)n, bo, bd, d_out);
        RUN4("packed_philox", 8, (k_packed<8, true>), nw, lf, d_pa, d_rec, (int)n, bo, bd, d_out);
        RUN("cols_hash", 1, (k_cols<1>), nw, lf, d_cols, d_rec, (int)n, d_out);
        RUN("cols_hash", 2, (k_cols<2>), nw, lf, d_cols, d_rec, (int)n, d_out);
        RUN("cols_hash", 4, (k_cols<4>), nw, lf, d_cols, d_rec, (int)n, d_out);
    }
    return 0;
}
