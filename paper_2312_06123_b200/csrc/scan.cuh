// scan.cuh -- device-wide prefix sums of the query pipeline, written for this library (no library
// scan): reduce-then-scan over tiles of SCAN_NT x ITEMS elements in three launches -- tile totals,
// a one-CTA exclusive scan of the totals, the tiles rescanned with their carry-in.  Generic over
// the element type and an associative, commutative `Op` (integer sums, the 3-way y-table size
// sums), so results do not depend on the grouping.  In-place (in == out) is allowed.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace geer {

constexpr int SCAN_NT = 256;

template <class T>
struct ScanItems {
    static constexpr int v = sizeof(T) > 8 ? 2 : 8;   // keeps the staging tile within 48 KB
};

template <class T>
struct ScanAdd {
    __device__ __forceinline__ T operator()(const T &a, const T &b) const { return a + b; }
};

// Warp shuffle of any trivially copyable T (word by word).
template <class T>
__device__ __forceinline__ T shfl_up_any(const T &v, int o)
{
    static_assert(sizeof(T) % 4 == 0, "T must be a multiple of 4 bytes");
    T r;
    const int *src = reinterpret_cast<const int *>(&v);
    int *dst = reinterpret_cast<int *>(&r);
#pragma unroll
    for (int i = 0; i < (int)(sizeof(T) / 4); i++) dst[i] = __shfl_up_sync(0xffffffffu, src[i], o);
    return r;
}

// Scan of one value per thread across the CTA (SCAN_NT threads): warp shuffles, then the warp
// totals through shared memory.  `zero` is the identity of op.  Returns the thread's inclusive
// prefix; *excl = its exclusive prefix, *total = the CTA total.  sh: >= SCAN_NT / 32 elements.
template <class T, class Op>
__device__ __forceinline__ T cta_scan(T v, T *sh, Op op, T zero, T *excl, T *total)
{
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const T own = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const T t = shfl_up_any(v, o);
        if (lane >= o) v = op(t, v);
    }
    if (lane == 31) sh[warp] = v;
    __syncthreads();
    T pre = zero, tot = zero;
    for (int w = 0; w < SCAN_NT / 32; w++) {
        if (w < warp) pre = op(pre, sh[w]);
        tot = op(tot, sh[w]);
    }
    T wex = shfl_up_any(v, 1);   // warp-exclusive prefix (lane 0: none)
    *excl = lane > 0 ? op(pre, wex) : pre;
    *total = tot;
    __syncthreads();
    (void)own;
    return op(pre, v);
}

template <class T, class Op>
__device__ __forceinline__ T cta_scan_incl(T v, T *sh, Op op, T *total)
{
    T ex;
    return cta_scan(v, sh, op, T{}, &ex, total);
}

// Thread t takes elements t*IT .. t*IT+IT-1 of tile `tile` of in[0, n) (staged through shared
// memory so that the global loads are coalesced); missing elements are `zero`.
template <class T, int IT>
__device__ __forceinline__ void scan_load_tile(const T *__restrict__ in, int64_t n, int64_t tile, T *stage,
                                               T (&x)[IT], T zero)
{
    const int64_t base = tile * (SCAN_NT * IT);
#pragma unroll
    for (int j = 0; j < IT; j++) {
        const int64_t i = base + j * SCAN_NT + threadIdx.x;
        stage[j * SCAN_NT + threadIdx.x] = i < n ? in[i] : zero;
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < IT; j++) x[j] = stage[threadIdx.x * IT + j];
    __syncthreads();
}

// Scan of one tile in registers: x[] -> inclusive prefixes starting from `carry`; returns the tile
// total (CTA-uniform).
template <class T, class Op, int IT>
__device__ __forceinline__ T scan_tile_regs(T (&x)[IT], T carry, T *sh, Op op, T zero)
{
    T s = x[0];
#pragma unroll
    for (int j = 1; j < IT; j++) s = op(s, x[j]);
    T tot, ex;
    cta_scan(s, sh, op, zero, &ex, &tot);
    T run = op(carry, ex);
#pragma unroll
    for (int j = 0; j < IT; j++) {
        run = op(run, x[j]);
        x[j] = run;
    }
    return tot;
}

template <class T, int IT>
__device__ __forceinline__ void scan_store_tile(T *__restrict__ out, int64_t n, int64_t tile, T *stage, const T (&x)[IT])
{
#pragma unroll
    for (int j = 0; j < IT; j++) stage[threadIdx.x * IT + j] = x[j];
    __syncthreads();
    const int64_t base = tile * (SCAN_NT * IT);
#pragma unroll
    for (int j = 0; j < IT; j++) {
        const int64_t i = base + j * SCAN_NT + threadIdx.x;
        if (i < n) out[i] = stage[j * SCAN_NT + threadIdx.x];
    }
    __syncthreads();
}

template <class T, class Op, int IT>
__global__ void __launch_bounds__(SCAN_NT) k_scan_tiles(const T *__restrict__ in, int64_t n, T zero, Op op,
                                                        T *__restrict__ tilesum)
{
    __shared__ T stage[SCAN_NT * IT];
    __shared__ T sh[SCAN_NT / 32];
    T x[IT];
    scan_load_tile<T, IT>(in, n, blockIdx.x, stage, x, zero);
    T s = x[0];
#pragma unroll
    for (int j = 1; j < IT; j++) s = op(s, x[j]);
    T tot, ex;
    cta_scan(s, sh, op, zero, &ex, &tot);
    if (threadIdx.x == 0) tilesum[blockIdx.x] = tot;
}

// One CTA: tilesum[0..ntiles) -> exclusive prefixes, in place.
template <class T, class Op, int IT>
__global__ void __launch_bounds__(SCAN_NT) k_scan_carry(T *__restrict__ tilesum, int64_t ntiles, T zero, Op op)
{
    __shared__ T stage[SCAN_NT * IT];
    __shared__ T sh[SCAN_NT / 32];
    T carry = zero;
    const int64_t nt2 = (ntiles + SCAN_NT * IT - 1) / (SCAN_NT * IT);
    for (int64_t tt = 0; tt < nt2; tt++) {
        T x[IT];
        scan_load_tile<T, IT>(tilesum, ntiles, tt, stage, x, zero);
        T s = x[0];
#pragma unroll
        for (int j = 1; j < IT; j++) s = op(s, x[j]);
        T tot, ex;
        cta_scan(s, sh, op, zero, &ex, &tot);
        T run = op(carry, ex);
#pragma unroll
        for (int j = 0; j < IT; j++) {
            const T v = x[j];
            x[j] = run;
            run = op(run, v);
        }
        scan_store_tile<T, IT>(tilesum, ntiles, tt, stage, x);
        carry = op(carry, tot);
    }
}

// Rescan each tile with its carry-in; out[i] = inclusive prefix of in[0..i].
template <class T, class Op, int IT>
__global__ void __launch_bounds__(SCAN_NT) k_scan_apply(const T *__restrict__ in, int64_t n, T zero, Op op,
                                                        const T *__restrict__ tileprefix, T *__restrict__ out)
{
    __shared__ T stage[SCAN_NT * IT];
    __shared__ T sh[SCAN_NT / 32];
    T x[IT];
    scan_load_tile<T, IT>(in, n, blockIdx.x, stage, x, zero);
    scan_tile_regs<T, Op, IT>(x, tileprefix[blockIdx.x], sh, op, zero);
    scan_store_tile<T, IT>(out, n, blockIdx.x, stage, x);
}

// Small inputs (a few tiles): one CTA scans in place of the three launches.
template <class T, class Op, int IT>
__global__ void __launch_bounds__(SCAN_NT) k_scan_single(const T *__restrict__ in, int64_t n, T zero, Op op,
                                                         T *__restrict__ out)
{
    __shared__ T stage[SCAN_NT * IT];
    __shared__ T sh[SCAN_NT / 32];
    T carry = zero;
    const int64_t nt = (n + SCAN_NT * IT - 1) / (SCAN_NT * IT);
    for (int64_t tt = 0; tt < nt; tt++) {
        T x[IT];
        scan_load_tile<T, IT>(in, n, tt, stage, x, zero);
        const T tot = scan_tile_regs<T, Op, IT>(x, carry, sh, op, zero);
        scan_store_tile<T, IT>(out, n, tt, stage, x);
        carry = op(carry, tot);
    }
}

constexpr int SCAN_SINGLE_TILES = 8;

// Temporary bytes the scan of n elements of T needs.
template <class T>
inline size_t scan_tmp_bytes(int64_t n)
{
    const int64_t tile = (int64_t)SCAN_NT * ScanItems<T>::v;
    return sizeof(T) * (size_t)((n + tile - 1) / tile + 1);
}

// out[i] = in[0] op ... op in[i] for i < n, on stream st; tmp: scan_tmp_bytes<T>(n) bytes.
// Returns the number of kernels launched.
template <class T, class Op>
inline int scan_launch(cudaStream_t st, const T *in, T *out, int64_t n, T zero, Op op, void *tmp)
{
    if (n <= 0) return 0;
    constexpr int IT = ScanItems<T>::v;
    const int64_t nt = (n + (int64_t)SCAN_NT * IT - 1) / ((int64_t)SCAN_NT * IT);
    if (nt <= SCAN_SINGLE_TILES) {
        k_scan_single<T, Op, IT><<<1, SCAN_NT, 0, st>>>(in, n, zero, op, out);
        return 1;
    }
    T *ts = reinterpret_cast<T *>(tmp);
    k_scan_tiles<T, Op, IT><<<(unsigned)nt, SCAN_NT, 0, st>>>(in, n, zero, op, ts);
    k_scan_carry<T, Op, IT><<<1, SCAN_NT, 0, st>>>(ts, nt, zero, op);
    k_scan_apply<T, Op, IT><<<(unsigned)nt, SCAN_NT, 0, st>>>(in, n, zero, op, ts, out);
    return 3;
}

}  // namespace geer
