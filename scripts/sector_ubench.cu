// sector_ubench.cu -- SURVEY.md App. A.6 roofline microbenchmarks for the AMC walk kernel (K6):
// the sustained rate of random 32-byte sector reads on one B200.
//
//   independent  every thread issues U independent 8-byte loads per iteration, each from a
//                uniformly random 32-byte sector of a buffer of the given size (addresses from a
//                per-thread xorshift stream, never from loaded data): ~148 SMs x 2048 threads x U
//                loads in flight.  Gives the random-sector ceiling of the memory level the buffer
//                lives in (L2-resident below ~64 MB, DRAM above).
//   dependent    C chains per thread; each load's sector is a hash of the previous load's value and
//                the step (a pointer chase without cycles): the walk's dependency structure with
//                C chains (K6 runs 2: S_k and T_k).
//
// Loads are ld.global.nc (the walk kernel's flavour).  Rates are loads (= sectors touched) per
// second from CUDA events around one launch, after a warm-up launch; the buffer is filled with
// random 64-bit words first.  Output: one JSON object per line.
//
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o scripts/sector_ubench scripts/sector_ubench.cu
// Run:   scripts/sector_ubench [max_gb [sizes_mb,... [l2_fetch_bytes]]] > profiles/sector_ubench_r02.jsonl
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <vector>

#include <cuda_runtime.h>

#define CK(x)                                                                                   \
    do {                                                                                        \
        cudaError_t e_ = (x);                                                                   \
        if (e_ != cudaSuccess) {                                                                \
            fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
            exit(1);                                                                            \
        }                                                                                       \
    } while (0)

__device__ __forceinline__ uint64_t mix(uint64_t x)
{
    x ^= x >> 33;
    x *= 0xff51afd7ed558ccdULL;
    x ^= x >> 33;
    x *= 0xc4ceb9fe1a85ec53ULL;
    x ^= x >> 33;
    return x;
}

__global__ void k_fill(uint64_t *buf, uint64_t words, uint64_t seed)
{
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < words; i += (uint64_t)gridDim.x * blockDim.x)
        buf[i] = mix(i ^ seed);
}

__device__ __forceinline__ uint64_t ldnc(const uint64_t *p)
{
    uint64_t v;
    asm volatile("ld.global.nc.u64 %0, [%1];" : "=l"(v) : "l"(p));
    return v;
}
// load flavours (for the sector-granularity experiment): 0 nc, 1 ca, 2 cg, 3 cs, 4 lu, 5 cv,
// 6 nc + L1::no_allocate, 7 ca + L1::no_allocate, 8-10 with the L2::64B prefetch-size qualifier
template <int FL>
__device__ __forceinline__ uint64_t ldf(const uint64_t *p)
{
    uint64_t v;
    if (FL == 0) asm volatile("ld.global.nc.u64 %0, [%1];" : "=l"(v) : "l"(p));
    if (FL == 1) asm volatile("ld.global.ca.u64 %0, [%1];" : "=l"(v) : "l"(p));
    if (FL == 2) asm volatile("ld.global.cg.u64 %0, [%1];" : "=l"(v) : "l"(p));
    if (FL == 3) asm volatile("ld.global.cs.u64 %0, [%1];" : "=l"(v) : "l"(p));
    if (FL == 4) asm volatile("ld.global.lu.u64 %0, [%1];" : "=l"(v) : "l"(p));
    if (FL == 5) asm volatile("ld.global.cv.u64 %0, [%1];" : "=l"(v) : "l"(p));
    if (FL == 6) asm volatile("ld.global.nc.L1::no_allocate.u64 %0, [%1];" : "=l"(v) : "l"(p));
    if (FL == 7) asm volatile("ld.global.L1::no_allocate.u64 %0, [%1];" : "=l"(v) : "l"(p));
    if (FL == 8) asm volatile("ld.global.nc.L2::64B.u64 %0, [%1];" : "=l"(v) : "l"(p));
    if (FL == 9) asm volatile("ld.global.L2::64B.u64 %0, [%1];" : "=l"(v) : "l"(p));
    if (FL == 10) asm volatile("ld.global.nc.L1::no_allocate.L2::64B.u64 %0, [%1];" : "=l"(v) : "l"(p));
    return v;
}
template <int FL>
__global__ void __launch_bounds__(256) k_flavour(const uint64_t *__restrict__ buf, uint64_t nsect, int iters,
                                                 unsigned long long *sink)
{
    const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    uint64_t x = mix(tid + 0x9E3779B97F4A7C15ULL) | 1ull;
    uint64_t acc = 0;
    for (int it = 0; it < iters; it++) {
        uint64_t v[8];
#pragma unroll
        for (int u = 0; u < 8; u++) {
            x ^= x << 13;
            x ^= x >> 7;
            x ^= x << 17;
            v[u] = ldf<FL>(buf + 4 * __umul64hi(x, nsect));
        }
#pragma unroll
        for (int u = 0; u < 8; u++) acc += v[u];
    }
    if (acc == 0x12345678ull) atomicAdd(sink, 1ull);
}

template <int U>
__global__ void __launch_bounds__(256) k_independent(const uint64_t *__restrict__ buf, uint64_t nsect, int iters,
                                                     unsigned long long *sink)
{
    const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    uint64_t x = mix(tid + 0x9E3779B97F4A7C15ULL) | 1ull;
    uint64_t acc = 0;
    for (int it = 0; it < iters; it++) {
        uint64_t v[U];
#pragma unroll
        for (int u = 0; u < U; u++) {
            x ^= x << 13;
            x ^= x >> 7;
            x ^= x << 17;
            const uint64_t s = __umul64hi(x, nsect);   // uniform sector in [0, nsect)
            v[u] = ldnc(buf + 4 * s);
        }
#pragma unroll
        for (int u = 0; u < U; u++) acc += v[u];
    }
    if (acc == 0x12345678ull) atomicAdd(sink, 1ull);
}

template <int C>
__global__ void __launch_bounds__(256) k_dependent(const uint64_t *__restrict__ buf, uint64_t nsect, int iters,
                                                   unsigned long long *sink)
{
    const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    uint64_t v[C];
#pragma unroll
    for (int c = 0; c < C; c++) v[c] = mix(tid * C + c + 1);
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int c = 0; c < C; c++) {
            const uint64_t s = __umul64hi(mix(v[c] + (uint64_t)it), nsect);
            v[c] = ldnc(buf + 4 * s);
        }
    }
    uint64_t acc = 0;
#pragma unroll
    for (int c = 0; c < C; c++) acc += v[c];
    if (acc == 0x12345678ull) atomicAdd(sink, 1ull);
}

template <class F>
static double time_ms(F launch)
{
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    launch();   // warm-up
    CK(cudaDeviceSynchronize());
    float best = 1e30f;
    for (int r = 0; r < 3; r++) {
        CK(cudaEventRecord(a));
        launch();
        CK(cudaEventRecord(b));
        CK(cudaEventSynchronize(b));
        float ms;
        CK(cudaEventElapsedTime(&ms, a, b));
        if (ms < best) best = ms;
    }
    CK(cudaEventDestroy(a));
    CK(cudaEventDestroy(b));
    return best;
}

int main(int argc, char **argv)
{
    const double max_gb = argc > 1 ? atof(argv[1]) : 32.0;
    int dev = 0, nsm = 0, clk = 0;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev));
    const uint64_t max_bytes = (uint64_t)(max_gb * (1ull << 30));
    if (argc > 3) {   // optional L2 fetch granularity hint in bytes (cudaLimitMaxL2FetchGranularity)
        CK(cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, (size_t)atoi(argv[3])));
    }
    size_t gran = 0;
    CK(cudaDeviceGetLimit(&gran, cudaLimitMaxL2FetchGranularity));
    fprintf(stderr, "L2 fetch granularity limit: %zu\n", gran);
    uint64_t *buf = nullptr;
    CK(cudaMalloc(&buf, max_bytes));
    unsigned long long *sink;
    CK(cudaMalloc(&sink, 8));
    k_fill<<<nsm * 8, 256>>>(buf, max_bytes / 8, 20231210);
    CK(cudaDeviceSynchronize());
    std::vector<double> sizes_mb = {16, 32, 48, 64, 80, 96, 128, 256, 1024, 4096, 16384, 32768};
    if (argc > 2) {   // optional comma-separated subset of buffer sizes in MB
        sizes_mb.clear();
        for (char *t = strtok(argv[2], ","); t; t = strtok(nullptr, ",")) sizes_mb.push_back(atof(t));
    }
    const int threads = 256, blocks = nsm * (2048 / threads);   // full occupancy, one wave
    for (double mb : sizes_mb) {
        const uint64_t bytes = (uint64_t)(mb * (1 << 20));
        if (bytes > max_bytes) break;
        const uint64_t nsect = bytes / 32;
        // independent loads: U = 8 per thread per iteration
        {
            const int iters = mb >= 1024 ? 64 : 256;
            const double ms = time_ms([&] { k_independent<8><<<blocks, threads>>>(buf, nsect, iters, sink); });
            const double loads = (double)blocks * threads * iters * 8;
            printf("{\"mode\": \"independent\", \"buffer_mb\": %.0f, \"loads_in_flight\": %d, \"ms\": %.4f, "
                   "\"g_sectors_per_s\": %.2f, \"sector_gbs\": %.1f, \"l2_fetch_limit\": %zu}\n",
                   mb, blocks * threads * 8, ms, loads / ms / 1e6, 32.0 * loads / ms / 1e6, gran);
        }
        if (getenv("UBENCH_FLAVOURS")) {
            const int iters = mb >= 1024 ? 64 : 256;
            const double loads = (double)blocks * threads * iters * 8;
            double ms[11];
            ms[0] = time_ms([&] { k_flavour<0><<<blocks, threads>>>(buf, nsect, iters, sink); });
            ms[1] = time_ms([&] { k_flavour<1><<<blocks, threads>>>(buf, nsect, iters, sink); });
            ms[2] = time_ms([&] { k_flavour<2><<<blocks, threads>>>(buf, nsect, iters, sink); });
            ms[3] = time_ms([&] { k_flavour<3><<<blocks, threads>>>(buf, nsect, iters, sink); });
            ms[4] = time_ms([&] { k_flavour<4><<<blocks, threads>>>(buf, nsect, iters, sink); });
            ms[5] = time_ms([&] { k_flavour<5><<<blocks, threads>>>(buf, nsect, iters, sink); });
            ms[6] = time_ms([&] { k_flavour<6><<<blocks, threads>>>(buf, nsect, iters, sink); });
            ms[7] = time_ms([&] { k_flavour<7><<<blocks, threads>>>(buf, nsect, iters, sink); });
            ms[8] = time_ms([&] { k_flavour<8><<<blocks, threads>>>(buf, nsect, iters, sink); });
            ms[9] = time_ms([&] { k_flavour<9><<<blocks, threads>>>(buf, nsect, iters, sink); });
            ms[10] = time_ms([&] { k_flavour<10><<<blocks, threads>>>(buf, nsect, iters, sink); });
            const char *nm[11] = {"nc", "ca", "cg", "cs", "lu", "cv", "nc_L1na", "ca_L1na", "nc_L2_64B", "ca_L2_64B",
                                  "nc_L1na_L2_64B"};
            for (int f = 0; f < 11; f++)
                printf("{\"mode\": \"flavour\", \"flavour\": \"%s\", \"buffer_mb\": %.0f, \"ms\": %.4f, "
                       "\"g_sectors_per_s\": %.2f}\n", nm[f], mb, ms[f], loads / ms[f] / 1e6);
        }
        for (int C : {1, 2, 4, 8}) {
            const int iters = mb >= 1024 ? 128 : 512;
            double ms = 0;
            if (C == 1) ms = time_ms([&] { k_dependent<1><<<blocks, threads>>>(buf, nsect, iters, sink); });
            if (C == 2) ms = time_ms([&] { k_dependent<2><<<blocks, threads>>>(buf, nsect, iters, sink); });
            if (C == 4) ms = time_ms([&] { k_dependent<4><<<blocks, threads>>>(buf, nsect, iters, sink); });
            if (C == 8) ms = time_ms([&] { k_dependent<8><<<blocks, threads>>>(buf, nsect, iters, sink); });
            const double loads = (double)blocks * threads * iters * C;
            printf("{\"mode\": \"dependent\", \"chains_per_thread\": %d, \"buffer_mb\": %.0f, \"loads_in_flight\": %d, "
                   "\"ms\": %.4f, \"g_sectors_per_s\": %.2f, \"sector_gbs\": %.1f}\n",
                   C, mb, blocks * threads * C, ms, loads / ms / 1e6, 32.0 * loads / ms / 1e6);
        }
        fflush(stdout);
    }
    printf("{\"device_sms\": %d, \"clock_khz\": %d}\n", nsm, clk);
    CK(cudaFree(buf));
    return 0;
}
