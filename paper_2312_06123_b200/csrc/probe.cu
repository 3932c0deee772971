// probe.cu -- the random-access ceilings K6's roofline is quoted against, measured on the running
// device (App. A.6 of SURVEY.md; the committed microbenchmark is scripts/sector_ubench.cu): 8-byte
// loads at independent uniformly random 32-byte sectors of a buffer, 8 in flight per thread, every
// SM at full occupancy.  flavour 0: ld.global.nc (the packed L2-resident walk graph's load),
// flavour 1: ld.global.nc.L2::64B (the DRAM-resident walk graph's column load).  Not on the query
// path: bench.py calls it once, before its timed region, so a step rate and its ceiling come from
// the same box.

#include "geer_internal.h"

namespace {

__device__ __forceinline__ uint64_t probe_mix(uint64_t x)
{
    x ^= x >> 31;
    x *= 0x7FB5D329728EA185ull;
    x ^= x >> 27;
    x *= 0x81DADEF4BC2DD44Dull;
    x ^= x >> 33;
    return x;
}

template <int FL, int U>
__global__ void __launch_bounds__(256) k_probe_loads(const uint64_t *__restrict__ buf, uint64_t nsect, int iters,
                                                     unsigned long long *__restrict__ sink)
{
    uint64_t x = probe_mix((uint64_t)blockIdx.x * blockDim.x + threadIdx.x + 1) | 1ull;
    uint64_t acc = 0;
    for (int it = 0; it < iters; it++) {
        uint64_t v[U];
#pragma unroll
        for (int u = 0; u < U; u++) {   // xorshift64: the next sector, independent of every load
            x ^= x << 13;
            x ^= x >> 7;
            x ^= x << 17;
            const uint64_t *p = buf + 4 * __umul64hi(x, nsect);
            if (FL == 0) asm volatile("ld.global.nc.u64 %0, [%1];" : "=l"(v[u]) : "l"(p));
            else asm volatile("ld.global.nc.L2::64B.u64 %0, [%1];" : "=l"(v[u]) : "l"(p));
        }
#pragma unroll
        for (int u = 0; u < U; u++) acc += v[u];
    }
    if (acc == 0x5E47ull) atomicAdd(sink, 1ull);   // keeps the loads
}

}  // namespace

extern "C" int er_probe_random_loads(int64_t bytes, int32_t flavour, int32_t iters, double *g_loads_per_s)
{
    using geer::set_error;
    if (bytes < (1 << 20) || (flavour != 0 && flavour != 1) || iters < 1 || !g_loads_per_s) {
        set_error(ER_EINVAL, "er_probe_random_loads: bytes >= 1 MiB, flavour 0/1, iters >= 1, output non-NULL");
        return ER_EINVAL;
    }
    int dev = 0, nsm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    uint64_t *buf = nullptr;
    unsigned long long *sink = nullptr;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    cudaError_t e = cudaMalloc(&buf, (size_t)bytes);
    if (e == cudaSuccess) e = cudaMalloc(&sink, sizeof(unsigned long long));
    if (e == cudaSuccess) e = cudaMemset(buf, 0x5A, (size_t)bytes);
    if (e == cudaSuccess) e = cudaEventCreate(&e0);
    if (e == cudaSuccess) e = cudaEventCreate(&e1);
    float best = 0.f;
    const int threads = 256, blocks = nsm * (2048 / threads);   // full occupancy, one wave
    const uint64_t nsect = (uint64_t)bytes / 32;
    for (int rep = 0; rep < 4 && e == cudaSuccess; rep++) {      // rep 0 warms up
        cudaEventRecord(e0);
        if (flavour == 0) k_probe_loads<0, 8><<<blocks, threads>>>(buf, nsect, iters, sink);
        else k_probe_loads<1, 8><<<blocks, threads>>>(buf, nsect, iters, sink);
        cudaEventRecord(e1);
        e = cudaEventSynchronize(e1);
        float ms = 0.f;
        if (e == cudaSuccess) e = cudaEventElapsedTime(&ms, e0, e1);
        if (rep > 0 && (best == 0.f || ms < best)) best = ms;
    }
    const double per_thread = 8.0;   // loads in flight per thread (4 and 16 measure the same rate:
                                     // profiles/probe_sweep_r02.jsonl)
    if (e == cudaSuccess) e = cudaGetLastError();
    if (e0) cudaEventDestroy(e0);
    if (e1) cudaEventDestroy(e1);
    if (buf) cudaFree(buf);
    if (sink) cudaFree(sink);
    if (e != cudaSuccess) return geer::cuda_fail(e, "er_probe_random_loads");
    *g_loads_per_s = (double)blocks * threads * iters * per_thread / (best * 1e-3) / 1e9;
    return ER_OK;
}
