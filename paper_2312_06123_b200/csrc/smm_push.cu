// smm_push.cu -- one SMM iteration by push for the active queries of a wave (Alg. 3 L6, P:583:
// s* <- P s*, t* <- P t*, P = D^-1 A, R1), with the per-segment statistics of Alg. 3 L7-L9
// (vol for Eq. 15, top-2 for Eq. 10, x(s), x(t) for the r_b term).  Hand-written grouping, no
// library sort:
//
//   frontier entry e (node v, value x(v), segment g = 2 i + side, entries of a segment ascending in
//   v) pushes one pair (u, e) per neighbour u of v.  Pairs are grouped by (segment, u) and each
//   group is summed SEQUENTIALLY IN ASCENDING e (= ascending source node, R13), then / d(u).
//
//   1. plan      per segment: its pair count E_g, a bucket count B_g = 2^k with about BKT_TARGET
//                pairs per bucket, bucket of u = u >> (nbits - k) (the high bits of the node id)
//   2. count     per pair: atomic count of its bucket (warp-aggregated)
//   3. scan      bucket offsets (scan.cuh)
//   4. scatter   per pair: key (u_low << ebits | e) into its bucket at an atomic slot (the order
//                inside a bucket is arbitrary; the key makes the result independent of it)
//   5. reduce    one CTA per bucket: stable LSD radix sort of the bucket's keys (shared memory, or
//                in place in global memory for buckets above BKT_CAP), runs of equal u summed in
//                key order (= ascending e), x'(u) = sum / d(u); the bucket's distinct u, values
//                and statistics (vol, max1 with multiplicity, max2; x(s), x(t) by their single
//                writer)
//   6. merge     per segment: bucket statistics -> SegStat (integer sums and maxima: exact)
//   7. gather    bucket outputs -> the contiguous next frontier (segment order, ascending u)
//
// Every step is deterministic (the atomic slot order is erased by the unique sort key), and the
// sums are the oracle's sequential order on sorted adjacency lists (R13).

#include "stages.h"

namespace geer {

namespace {

constexpr int BKT_NT = 256;                 // threads of the reduce CTA
constexpr int BKT_NW = BKT_NT / 32;
constexpr int BKT_TARGET = 256;             // mean pairs per bucket a segment is cut for
constexpr int BKT_WCAP = 512;               // largest bucket reduced by one warp (k_bkt_reduce_warp)
constexpr int BKT_WPB = 8;                  // warps per CTA of k_bkt_reduce_warp
constexpr int BKT_CAP = 2048;               // largest bucket sorted in shared memory by one CTA
constexpr int EMIT_PER = 4;                 // pairs per lane of the enumeration kernels

struct BStat {
    int64_t vol;                 // sum of d(u) over the bucket's distinct u
    unsigned long long max1;     // largest x'(u) (bits; x >= 0)
    unsigned long long max2;     // largest x'(u) below max1 (bits)
    int64_t n1;                  // occurrences of max1
    double at_s, at_t;           // x'(s), x'(t) when s / t falls in this bucket (flags bits 0 / 1)
    int64_t flags;
};

__device__ __forceinline__ int bits_for(int64_t x)   // bits to hold values 0..x (>= 1)
{
    int b = 1;
    while (b < 63 && ((int64_t)1 << b) <= x) b++;
    return b;
}

// 1. plan: per segment g its pair count, bucket count (power of two) and shifts.
// (Segment-indexed arrays of a chunk are local: index g - g0 for the chunk's segments g0..g0+ns.)
__global__ void k_bkt_plan(int32_t nseg, const int64_t *__restrict__ fr_off, const int64_t *__restrict__ ent_off,
                           int nbits, int64_t *__restrict__ segB, int32_t *__restrict__ segsh,
                           int32_t *__restrict__ segeb)
{
    const int32_t g = blockIdx.x * blockDim.x + threadIdx.x;   // local segment (fr_off is offset to g0)
    if (g >= nseg) return;
    const int64_t f0 = fr_off[g], f1 = fr_off[g + 1];
    const int64_t Eg = ent_off[f1] - ent_off[f0];
    int k = 0;
    while (k < nbits && ((int64_t)BKT_TARGET << k) < Eg) k++;
    segB[g] = (int64_t)1 << k;
    segsh[g] = nbits - k;                   // u_low keeps the low nbits - k bits of u
    segeb[g] = bits_for(f1 - f0 - 1);       // entry index inside the segment
}

// Segment of every bucket.
__global__ void k_bkt_seg(int32_t nseg, const int64_t *__restrict__ segBoff, const int64_t *__restrict__ dNB,
                          int32_t *__restrict__ bseg)
{
    const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;   // one thread per bucket
    if (b >= *dNB) return;
    int32_t lo = 0, hi = nseg;   // segBoff[lo] <= b < segBoff[hi]
    while (hi - lo > 1) {
        const int32_t mid = (lo + hi) >> 1;
        if (segBoff[mid] <= b) lo = mid;
        else hi = mid;
    }
    bseg[b] = lo;
}

// Largest index lo in [lo, hi) with a[lo] <= x, given a[lo] <= x and (a[hi] > x or hi the end),
// a monotone: the 32 lanes of the (converged) warp probe 32 evenly spaced points per round, so the
// range shrinks 32-fold per round (6 rounds for 10^8 entries instead of 27 dependent loads).
__device__ __forceinline__ int64_t warp_search(const int64_t *__restrict__ a, int64_t lo, int64_t hi, int64_t x)
{
    const int lane = threadIdx.x & 31;
    while (hi - lo > 1) {
        const int64_t step = (hi - lo + 31) >> 5;   // >= 1
        const int64_t q = lo + (int64_t)(lane + 1) * step;
        const bool le = q < hi && a[q] <= x;        // true for a prefix of the lanes
        const int c = __popc(__ballot_sync(0xffffffffu, le));
        lo += (int64_t)c * step;
        hi = min(hi, lo + step);
    }
    return lo;
}

// Pair enumeration shared by count and scatter over the chunk's pairs P0 + [0, E) (entries
// [e_lo, e_hi)): warp = 32 * EMIT_PER consecutive positions, the warp searches the entry of its
// first position (warp_search), lanes step forward from it.  f(live, local position, entry, j):
// the pair is the j-th neighbour of the entry's node.
template <class Fn>
__device__ __forceinline__ void for_pairs(int64_t P0, int64_t E, int64_t e_lo, int64_t e_hi,
                                          const int64_t *__restrict__ ent_off, Fn &&f)
{
    const int lane = threadIdx.x & 31;
    const int64_t base = ((int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31)) * EMIT_PER;
    if (base >= E) return;
    int64_t e = warp_search(ent_off, e_lo, e_hi, P0 + base);
    int64_t start = ent_off[e], next = ent_off[e + 1];
#pragma unroll
    for (int i = 0; i < EMIT_PER; i++) {
        const int64_t p = base + 32 * i + lane;
        const bool live = p < E;
        if (live) {
            while (P0 + p >= next) {   // every frontier node has degree >= 1
                e++;
                start = next;
                next = ent_off[e + 1];
            }
        }
        f(live, p, e, P0 + p - start);
    }
}

// 2. count: bucket sizes.
__global__ void k_bkt_count(int64_t P0, int64_t E, int64_t e_lo, int64_t e_hi, int32_t g0,
                            const int64_t *__restrict__ ent_off, const int32_t *__restrict__ id,
                            const int32_t *__restrict__ seg, const int64_t *__restrict__ off,
                            const int32_t *__restrict__ cols, const int64_t *__restrict__ segBoff,
                            const int32_t *__restrict__ segsh, unsigned long long *__restrict__ cnt)
{
    for_pairs(P0, E, e_lo, e_hi, ent_off, [&](bool live, int64_t, int64_t e, int64_t j) {
        int64_t b = -1;
        if (live) {
            const int32_t gl = seg[e] - g0;
            const int32_t u = cols[off[id[e]] + j];
            b = segBoff[gl] + (u >> segsh[gl]);
        }
        const unsigned peers = __match_any_sync(0xffffffffu, b);
        const int lane = threadIdx.x & 31;
        if (live && (peers & ((1u << lane) - 1u)) == 0) atomicAdd(cnt + b, (unsigned long long)__popc(peers));
    });
}

// 4. scatter: composite key (u_low << ebits | e_local) at an atomic slot of the pair's bucket.
__global__ void k_bkt_scatter(int64_t P0, int64_t E, int64_t e_lo, int64_t e_hi, int32_t g0,
                              const int64_t *__restrict__ ent_off, const int32_t *__restrict__ id,
                              const int32_t *__restrict__ seg, const int64_t *__restrict__ fr_off,
                              const int64_t *__restrict__ off, const int32_t *__restrict__ cols,
                              const int64_t *__restrict__ segBoff, const int32_t *__restrict__ segsh,
                              const int32_t *__restrict__ segeb, const int64_t *__restrict__ boff,
                              unsigned int *__restrict__ cur, unsigned long long *__restrict__ keys)
{
    for_pairs(P0, E, e_lo, e_hi, ent_off, [&](bool live, int64_t, int64_t e, int64_t j) {
        int64_t b = -1;
        unsigned long long key = 0;
        if (live) {
            const int32_t g = seg[e], gl = g - g0;
            const int32_t u = cols[off[id[e]] + j];
            const int sh = segsh[gl];
            b = segBoff[gl] + (u >> sh);
            const unsigned long long ulow = (unsigned long long)u & ((1ull << sh) - 1ull);
            key = (ulow << segeb[gl]) | (unsigned long long)(e - fr_off[g]);
        }
        const unsigned peers = __match_any_sync(0xffffffffu, b);
        const int lane = threadIdx.x & 31;
        const unsigned lt = peers & ((1u << lane) - 1u);
        unsigned slot0 = 0;
        if (live && lt == 0) slot0 = atomicAdd(cur + b, (unsigned)__popc(peers));
        const int leader = __ffs(peers) - 1;
        slot0 = __shfl_sync(0xffffffffu, slot0, leader);
        if (live) keys[boff[b] + slot0 + __popc(lt)] = key;
    });
}

// Stable LSD radix sort (8-bit digits) of n 64-bit keys on their low `bits` bits, by one CTA, in
// buffers a / b (shared or global memory).  Returns the buffer holding the result.  Warp w owns a
// contiguous chunk of the items; per pass: per-warp digit histograms, one CTA scan in (digit, warp)
// order that turns them into per-warp running offsets, then every warp places its items in index
// order, 32 at a time (lanes with equal digits ranked by lane) -- so every pass is stable, and the
// warps need no barrier while they place their items.
struct SortSmem {
    unsigned int wh[BKT_NW][256];   // per-warp digit counts, then running offsets
    unsigned int wtot[BKT_NW];
};
static_assert(BKT_NT == 256, "the digit scan maps one thread to each of the 256 digits");

__device__ unsigned long long *cta_radix_sort(unsigned long long *a, unsigned long long *b, int n, int bits,
                                              SortSmem &S)
{
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int npass = (bits + 7) / 8;
    const int chunk = (((n + BKT_NW - 1) / BKT_NW) + 31) & ~31;
    const int lo = min(n, warp * chunk), hi = min(n, lo + chunk);
    unsigned long long *src = a, *dst = b;
    for (int p = 0; p < npass; p++) {
        const int sh = 8 * p;
        for (int i = lane; i < 256; i += 32) S.wh[warp][i] = 0u;
        __syncwarp();
        for (int base = lo; base < hi; base += 32) {   // warp-aggregated histogram
            const int i = base + lane;
            const unsigned d = i < hi ? (unsigned)((src[i] >> sh) & 255u) : 256u;
            const unsigned peers = __match_any_sync(0xffffffffu, d);
            if (d < 256u && (peers & ((1u << lane) - 1u)) == 0) atomicAdd(&S.wh[warp][d], (unsigned)__popc(peers));
        }
        __syncthreads();
        // a digit every key shares needs no pass
        const unsigned d0 = (unsigned)((src[0] >> sh) & 255u);
        unsigned c0 = 0;
#pragma unroll
        for (int w = 0; w < BKT_NW; w++) c0 += S.wh[w][d0];
        if (c0 == (unsigned)n) {
            __syncthreads();
            continue;
        }
        // running offsets: thread t = digit t
        unsigned tot = 0;
#pragma unroll
        for (int w = 0; w < BKT_NW; w++) tot += S.wh[w][tid];
        unsigned incl = tot;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned t = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += t;
        }
        if (lane == 31) S.wtot[warp] = incl;
        __syncthreads();
        unsigned run = incl - tot;
        for (int w = 0; w < warp; w++) run += S.wtot[w];
#pragma unroll
        for (int w = 0; w < BKT_NW; w++) {
            const unsigned v = S.wh[w][tid];
            S.wh[w][tid] = run;
            run += v;
        }
        __syncthreads();
        for (int base = lo; base < hi; base += 32) {   // warp-uniform
            const int i = base + lane;
            const bool valid = i < hi;
            const unsigned long long k = valid ? src[i] : 0ull;
            const unsigned d = valid ? (unsigned)((k >> sh) & 255u) : 256u;
            const unsigned peers = __match_any_sync(0xffffffffu, d);
            const unsigned lt = peers & ((1u << lane) - 1u);
            if (valid) dst[S.wh[warp][d] + __popc(lt)] = k;
            __syncwarp();
            if (valid && lt == 0) S.wh[warp][d] += __popc(peers);
            __syncwarp();
        }
        __syncthreads();
        unsigned long long *t = src;
        src = dst;
        dst = t;
    }
    return src;
}

// CTA-wide reductions (BKT_NT threads).
__device__ __forceinline__ unsigned long long cta_max_u64(unsigned long long v, unsigned long long *sh)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long t = __shfl_xor_sync(0xffffffffu, v, o);
        v = t > v ? t : v;
    }
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
    __syncthreads();
    unsigned long long r = sh[0];
    for (int w = 1; w < BKT_NW; w++) r = sh[w] > r ? sh[w] : r;
    __syncthreads();
    return r;
}
__device__ __forceinline__ long long cta_sum_i64(long long v, long long *sh)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
    __syncthreads();
    long long r = 0;
    for (int w = 0; w < BKT_NW; w++) r += sh[w];
    __syncthreads();
    return r;
}

// 5. reduce, large buckets (more than BKT_WCAP pairs -- a hub's run, or skew -- or keys wider than
// 32 bits): one CTA per bucket of the list k_bkt_reduce_warp collected, persistent CTAs.
__device__ __forceinline__ void reduce_big_bucket(
    int64_t b, int32_t g0, const int32_t *__restrict__ bseg, const int64_t *__restrict__ segBoff,
    const int32_t *__restrict__ segsh, const int32_t *__restrict__ segeb, const int64_t *__restrict__ boff,
    unsigned long long *__restrict__ keys, unsigned long long *__restrict__ alt, const int64_t *__restrict__ fr_off,
    const double *__restrict__ fr_val, const uint2 *__restrict__ rec, const int32_t *__restrict__ act,
    const QState *__restrict__ qs, int32_t *__restrict__ out_id, double *__restrict__ out_val,
    int32_t *__restrict__ gruns, int64_t *__restrict__ ucnt, BStat *__restrict__ bst, unsigned long long *smk,
    SortSmem &S, int *s_runs, unsigned long long *s_red, double *s_at, int *s_flags)
{
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int32_t gl = bseg[b], g = g0 + gl;
    const int64_t base = boff[b];
    const int n = (int)(boff[b + 1] - base);
    const int sh = segsh[gl], eb = segeb[gl];
    const int64_t hi = b - segBoff[gl];
    unsigned long long *a, *bb;
    if (n <= BKT_CAP) {
        a = smk;
        bb = smk + BKT_CAP;
        for (int i = tid; i < n; i += BKT_NT) a[i] = keys[base + i];
        __syncthreads();
    } else {   // sorted in place in global memory
        a = keys + base;
        bb = alt + base;
    }
    if (tid == 0) {
        *s_flags = 0;
        s_at[0] = s_at[1] = 0.0;
    }
    unsigned long long *srt = cta_radix_sort(a, bb, n, sh + eb, S);
    // the free key buffer takes the values in sorted order (gathered in parallel, so the sequential
    // run sums below stream them instead of chasing each load)
    double *gv = reinterpret_cast<double *>(srt == a ? bb : a);
    int *runs = n <= BKT_CAP ? reinterpret_cast<int *>(smk + 2 * BKT_CAP) : gruns + base;
    const int64_t f0 = fr_off[g];
    const unsigned long long emask = (1ull << eb) - 1ull;
    for (int i = tid; i < n; i += BKT_NT) gv[i] = fr_val[f0 + (int64_t)(srt[i] & emask)];
    __syncthreads();
    // run heads (a change of u_low) and their ranks
    int carry = 0;
    for (int t0 = 0; t0 < n; t0 += BKT_NT) {
        const int i = t0 + tid;
        bool head = false;
        if (i < n) head = i == 0 || (srt[i] >> eb) != (srt[i - 1] >> eb);
        const unsigned bal = __ballot_sync(0xffffffffu, head);
        if (lane == 0) s_runs[warp] = __popc(bal);
        __syncthreads();
        int before = carry;
        for (int w = 0; w < warp; w++) before += s_runs[w];
        if (head) runs[before + __popc(bal & ((1u << lane) - 1u))] = i;
        int tot = 0;
        for (int w = 0; w < BKT_NW; w++) tot += s_runs[w];
        carry += tot;
        __syncthreads();
    }
    const int U = carry;
    // one thread per run: ascending-e sequential sum (R13), / d(u)
    const QState &Q = qs[act[g >> 1]];
    long long vol = 0;
    unsigned long long m1 = 0;
    for (int r = tid; r < U; r += BKT_NT) {
        const int i0 = runs[r], i1 = r + 1 < U ? runs[r + 1] : n;
        const int32_t u = (int32_t)((hi << sh) | (int64_t)(srt[i0] >> eb));
        const uint32_t d = __ldg(&rec[u].y);
        double sum = 0.0;
        for (int i = i0; i < i1; i++) sum += gv[i];
        const double x = sum / (double)d;
        out_id[base + r] = u;
        out_val[base + r] = x;
        vol += d;
        const unsigned long long xb = (unsigned long long)__double_as_longlong(x);
        m1 = xb > m1 ? xb : m1;
        if (u == Q.s) {   // single writers: u occurs once in the bucket
            s_at[0] = x;
            atomicOr(s_flags, 1);
        }
        if (u == Q.t) {
            s_at[1] = x;
            atomicOr(s_flags, 2);
        }
    }
    __syncthreads();
    const long long V = cta_sum_i64(vol, reinterpret_cast<long long *>(s_red));
    const unsigned long long M1 = cta_max_u64(m1, s_red);
    long long c1 = 0;
    unsigned long long m2 = 0;
    for (int r = tid; r < U; r += BKT_NT) {
        const unsigned long long xb = (unsigned long long)__double_as_longlong(out_val[base + r]);
        if (xb == M1) c1++;
        else if (xb > m2) m2 = xb;
    }
    const long long C1 = cta_sum_i64(c1, reinterpret_cast<long long *>(s_red));
    const unsigned long long M2 = cta_max_u64(m2, s_red);
    if (tid == 0) {
        ucnt[b] = U;
        bst[b] = BStat{V, M1, M2, C1, s_at[0], s_at[1], *s_flags};
    }
    __syncthreads();   // the shared buffers serve the CTA's next bucket
}

__global__ void __launch_bounds__(BKT_NT) k_bkt_reduce(
    int32_t g0, const int64_t *__restrict__ nbig, const int64_t *__restrict__ big, const int32_t *__restrict__ bseg,
    const int64_t *__restrict__ segBoff, const int32_t *__restrict__ segsh, const int32_t *__restrict__ segeb,
    const int64_t *__restrict__ boff, unsigned long long *__restrict__ keys, unsigned long long *__restrict__ alt,
    const int64_t *__restrict__ fr_off, const double *__restrict__ fr_val, const uint2 *__restrict__ rec,
    const int32_t *__restrict__ act, const QState *__restrict__ qs, int32_t *__restrict__ out_id,
    double *__restrict__ out_val, int32_t *__restrict__ gruns, int64_t *__restrict__ ucnt, BStat *__restrict__ bst)
{
    extern __shared__ __align__(16) unsigned long long smk[];   // 2 * BKT_CAP keys, BKT_CAP run starts
    __shared__ SortSmem S;
    __shared__ int s_runs[BKT_NT];
    __shared__ unsigned long long s_red[BKT_NW];
    __shared__ double s_at[2];
    __shared__ int s_flags;
    const int64_t NBig = *nbig;
    for (int64_t li = blockIdx.x; li < NBig; li += gridDim.x)
        reduce_big_bucket(big[li], g0, bseg, segBoff, segsh, segeb, boff, keys, alt, fr_off, fr_val, rec, act, qs,
                          out_id, out_val, gruns, ucnt, bst, smk, S, s_runs, s_red, s_at, &s_flags);
}

// 5a. reduce, small buckets (n <= BKT_WCAP): one WARP per bucket, warp-synchronous (no CTA
// barriers), buckets handed out grid-stride.  Same result as k_bkt_reduce: stable LSD radix sort
// of (u_low, e) keys, values gathered in sorted order, one lane per run of equal u summing its
// values in ascending e, / d(u); statistics reduced over the warp.
struct WarpSmem {
    unsigned int a[BKT_WCAP], b[BKT_WCAP];   // 32-bit keys (buckets with wider keys: k_bkt_reduce);
                                             // after the sort the other buffer holds the run heads
    unsigned int cnt[256];
};
#ifndef BKT_RW_MINB
#define BKT_RW_MINB 4   // resident CTAs per SM k_bkt_reduce_warp is compiled for (64 registers)
#endif

// Stable LSD passes over key bits [0, bits), 8 bits per pass (one warp, 32-bit keys).
__device__ __forceinline__ unsigned int *warp_radix_sort(unsigned int *a, unsigned int *b, int n, int bits,
                                                         unsigned int *cnt)
{
    const int lane = threadIdx.x & 31;
    const int npass = (bits + 7) / 8;
    unsigned int *src = a, *dst = b;
    for (int p = 0; p < npass; p++) {
        const int sh = 8 * p;
        for (int i = lane; i < 256; i += 32) cnt[i] = 0u;
        __syncwarp();
        for (int i = lane; i < n; i += 32) atomicAdd(&cnt[(src[i] >> sh) & 255u], 1u);
        __syncwarp();
        if (cnt[(src[0] >> sh) & 255u] == (unsigned)n) continue;   // a digit all keys share
        unsigned v[8], sum = 0;
#pragma unroll
        for (int j = 0; j < 8; j++) {
            v[j] = cnt[lane * 8 + j];
            sum += v[j];
        }
        unsigned incl = sum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned t = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += t;
        }
        unsigned run = incl - sum;
        __syncwarp();
#pragma unroll
        for (int j = 0; j < 8; j++) {
            cnt[lane * 8 + j] = run;
            run += v[j];
        }
        __syncwarp();
        for (int base = 0; base < n; base += 32) {
            const int i = base + lane;
            const bool valid = i < n;
            const unsigned k = valid ? src[i] : 0u;
            const unsigned d = valid ? ((k >> sh) & 255u) : 256u;
            const unsigned peers = __match_any_sync(0xffffffffu, d);
            const unsigned lt = peers & ((1u << lane) - 1u);
            if (valid) dst[cnt[d] + __popc(lt)] = k;
            __syncwarp();
            if (valid && lt == 0) cnt[d] += __popc(peers);
            __syncwarp();
        }
        unsigned int *t = src;
        src = dst;
        dst = t;
    }
    return src;
}

__global__ void __launch_bounds__(32 * BKT_WPB, BKT_RW_MINB) k_bkt_reduce_warp(
    int32_t g0, const int64_t *__restrict__ dNB, const int32_t *__restrict__ bseg, const int64_t *__restrict__ segBoff,
    const int32_t *__restrict__ segsh, const int32_t *__restrict__ segeb, const int64_t *__restrict__ boff,
    const unsigned long long *__restrict__ keys, const int64_t *__restrict__ fr_off, const double *__restrict__ fr_val,
    const uint2 *__restrict__ rec, const int32_t *__restrict__ act, const QState *__restrict__ qs,
    int32_t *__restrict__ out_id, double *__restrict__ out_val, int64_t *__restrict__ ucnt, BStat *__restrict__ bst,
    unsigned long long *__restrict__ nbig, int64_t *__restrict__ big)
{
    __shared__ WarpSmem W[BKT_WPB];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    WarpSmem &M = W[wib];
    const int64_t NB = *dNB;
    const unsigned full = 0xffffffffu;
    for (int64_t b = (int64_t)blockIdx.x * BKT_WPB + wib; b < NB; b += (int64_t)gridDim.x * BKT_WPB) {
        const int64_t base = boff[b];
        const int n = (int)(boff[b + 1] - base);
        const int32_t gl = bseg[b], g = g0 + gl;
        const int sh = segsh[gl], eb = segeb[gl];
        if (n > BKT_WCAP || sh + eb > 32) {   // listed for k_bkt_reduce
            if (lane == 0) big[atomicAdd(nbig, 1ull)] = b;
            continue;
        }
        if (n == 0) {
            if (lane == 0) {
                ucnt[b] = 0;
                bst[b] = BStat{0, 0ull, 0ull, 0, 0.0, 0.0, 0};
            }
            continue;
        }
        const int64_t hi = b - segBoff[gl];
        for (int i = lane; i < n; i += 32) M.a[i] = (unsigned)keys[base + i];
        __syncwarp();
        const unsigned *srt = warp_radix_sort(M.a, M.b, n, sh + eb, M.cnt);
        unsigned int *runs = srt == M.a ? M.b : M.a;
        const double *__restrict__ fv = fr_val + fr_off[g];
        const unsigned emask = eb >= 32 ? 0xffffffffu : (1u << eb) - 1u;
        // run heads and their ranks
        int U = 0;
        for (int t0 = 0; t0 < n; t0 += 32) {
            const int i = t0 + lane;
            const bool head = i < n && (i == 0 || (eb < 32 && (srt[i] >> eb) != (srt[i - 1] >> eb)));
            const unsigned bal = __ballot_sync(full, head);
            if (head) runs[U + __popc(bal & ((1u << lane) - 1u))] = i;
            U += __popc(bal);
        }
        __syncwarp();
        const QState &Q = qs[act[g >> 1]];
        long long vol = 0, c1 = 0;
        unsigned long long m1 = 0, m2 = 0;   // top-2 with multiplicity, streamed per lane
        double at_s = 0.0, at_t = 0.0;
        int flags = 0;
        for (int r = lane; r < U; r += 32) {
            const int i0 = runs[r], i1 = r + 1 < U ? runs[r + 1] : n;
            double sum = 0.0;
            for (int i = i0; i < i1; i++) sum += fv[srt[i] & emask];   // ascending source order (R13)
            const int32_t u = (int32_t)((hi << sh) | (int64_t)(eb >= 32 ? 0u : srt[i0] >> eb));
            const uint32_t d = __ldg(&rec[u].y);
            const double x = sum / (double)d;
            out_id[base + r] = u;
            out_val[base + r] = x;
            vol += d;
            const unsigned long long xb = (unsigned long long)__double_as_longlong(x);
            if (xb > m1) {
                m2 = m1;
                m1 = xb;
                c1 = 1;
            } else if (xb == m1) {
                c1++;
            } else if (xb > m2) {
                m2 = xb;
            }
            if (u == Q.s) { at_s = x; flags |= 1; }
            if (u == Q.t) { at_t = x; flags |= 2; }
        }
        // exact merges (integer sums, maxima on the bits of x >= 0): the tree order does not matter
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            vol += __shfl_xor_sync(full, vol, o);
            const unsigned long long om1 = __shfl_xor_sync(full, m1, o), om2 = __shfl_xor_sync(full, m2, o);
            const long long oc1 = __shfl_xor_sync(full, c1, o);
            if (om1 > m1) {
                m2 = m1 > om2 ? m1 : om2;   // max(m2, m1, om2) = max(m1, om2): m1 > m2
                m1 = om1;
                c1 = oc1;
            } else if (om1 == m1) {
                c1 += oc1;
                m2 = m2 > om2 ? m2 : om2;
            } else {
                m2 = m2 > om1 ? m2 : om1;
            }
        }
        // x(s), x(t): single writers -> the lane that has them
        const unsigned bs = __ballot_sync(full, flags & 1), bt = __ballot_sync(full, flags & 2);
        if (bs) at_s = __shfl_sync(full, at_s, __ffs(bs) - 1);
        if (bt) at_t = __shfl_sync(full, at_t, __ffs(bt) - 1);
        if (lane == 0) {
            ucnt[b] = U;
            bst[b] = BStat{vol, m1, m2, c1, at_s, at_t, (int64_t)((bs ? 1 : 0) | (bt ? 2 : 0))};
        }
        __syncwarp();
    }
}

// 6. merge: per segment, the statistics of its buckets (exact integer sums and maxima, so the
// order of the warp's tree does not matter); one warp per segment.
struct MStat {
    long long vol, n1, flags;
    unsigned long long m1, m2;
    double at_s, at_t;
};
__device__ __forceinline__ MStat mstat_merge(const MStat &a, const MStat &b)
{
    MStat r;
    r.vol = a.vol + b.vol;
    r.flags = a.flags | b.flags;
    r.at_s = (a.flags & 1) ? a.at_s : b.at_s;
    r.at_t = (a.flags & 2) ? a.at_t : b.at_t;
    if (a.m1 > b.m1) {
        r.m1 = a.m1;
        r.n1 = a.n1;
        r.m2 = a.m2 > b.m1 ? a.m2 : b.m1;
    } else if (b.m1 > a.m1) {
        r.m1 = b.m1;
        r.n1 = b.n1;
        r.m2 = b.m2 > a.m1 ? b.m2 : a.m1;
    } else {
        r.m1 = a.m1;
        r.n1 = a.n1 + b.n1;
        r.m2 = a.m2 > b.m2 ? a.m2 : b.m2;
    }
    return r;
}
__device__ __forceinline__ MStat mstat_shfl(const MStat &a, int o)
{
    MStat r;
    r.vol = __shfl_xor_sync(0xffffffffu, a.vol, o);
    r.n1 = __shfl_xor_sync(0xffffffffu, a.n1, o);
    r.flags = __shfl_xor_sync(0xffffffffu, a.flags, o);
    r.m1 = __shfl_xor_sync(0xffffffffu, a.m1, o);
    r.m2 = __shfl_xor_sync(0xffffffffu, a.m2, o);
    r.at_s = __shfl_xor_sync(0xffffffffu, a.at_s, o);
    r.at_t = __shfl_xor_sync(0xffffffffu, a.at_t, o);
    return r;
}
constexpr int MERGE_NT = 128;
__global__ void __launch_bounds__(MERGE_NT) k_bkt_merge(int32_t nseg, int32_t g0, const int64_t *__restrict__ segBoff,
                                                        const BStat *__restrict__ bst, SegStat *__restrict__ ss)
{
    // one CTA per segment (a large segment has thousands of buckets)
    __shared__ MStat sm[MERGE_NT / 32];
    const int32_t g = blockIdx.x;   // local segment
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (g >= nseg) return;
    MStat m{0, 0, 0, 0ull, 0ull, 0.0, 0.0};
    for (int64_t b = segBoff[g] + threadIdx.x; b < segBoff[g + 1]; b += MERGE_NT) {
        const BStat B = bst[b];
        m = mstat_merge(m, MStat{B.vol, B.n1, B.flags, B.max1, B.max2, B.at_s, B.at_t});
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = mstat_merge(m, mstat_shfl(m, o));
    if (lane == 0) sm[warp] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < MERGE_NT / 32; w++) m = mstat_merge(m, sm[w]);
        SegStat &S = ss[g0 + g];
        S.vol = m.vol;
        S.max1 = __longlong_as_double((long long)m.m1);
        S.max2 = __longlong_as_double((long long)m.m2);
        S.n_max1 = (unsigned long long)m.n1;
        S.at_s = m.at_s;
        S.at_t = m.at_t;
    }
}

// 7. gather: bucket outputs -> contiguous next frontier (after the earlier chunks' entries,
// which end at nf_off[g0]); segment offsets; entry count.
__global__ void k_bkt_gather(const int64_t *__restrict__ dNB, int32_t nseg, int32_t g0, const int32_t *__restrict__ bseg,
                             const int64_t *__restrict__ segBoff, const int64_t *__restrict__ boff,
                             const int64_t *__restrict__ uoff, const int32_t *__restrict__ out_id,
                             const double *__restrict__ out_val, int32_t *__restrict__ nid, double *__restrict__ nval,
                             int32_t *__restrict__ nseg_out, int64_t *__restrict__ nf_off, int64_t *__restrict__ dU)
{
    const int64_t NB = *dNB;
    const int64_t b = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (b >= NB) return;
    const int64_t ubase = g0 == 0 ? 0 : nf_off[g0];   // (the write below of nf_off[g0] stores this value)
    const int32_t gl = bseg[b];
    const int64_t src = boff[b], dst = ubase + uoff[b], U = uoff[b + 1] - uoff[b];
    for (int64_t r = lane; r < U; r += 32) {
        nid[dst + r] = out_id[src + r];
        nval[dst + r] = out_val[src + r];
        nseg_out[dst + r] = g0 + gl;
    }
    if (lane == 0) {
        if (b == segBoff[gl]) nf_off[g0 + gl] = dst;
        if (b == NB - 1) {
            nf_off[g0 + nseg] = ubase + uoff[NB];
            *dU = ubase + uoff[NB];
        }
    }
}

}  // namespace

// One push wave over the frontier ws.fr_* (F entries, 2 na segments, pair offsets ent_off with E
// pairs in total), in two parts so that the previous wave's y-table build (side stream, reading
// ws.nf_*) can overlap part A:
//   part A  plan, count, scatter, reduce -- writes only the push workspaces (ws.pk_*);
//   part B  merge, gather -- SegStat into ws.segstat, the next frontier into ws.nf_* (capacity
//           >= E), its segment offsets into ws.nf_off, the entry count at *dU (device).
namespace {
// Views of the push workspaces of a wave with bucket bound NBmax (part A and part B agree on them).
struct PushView {
    int64_t *segB, *segBoff;
    int32_t *segsh, *segeb;
    int64_t *cnt, *boff, *ucnt, *uoff;
    BStat *bst;
    int32_t *bseg;
    unsigned int *cur;
    unsigned long long *nbig;   // count of the buckets listed for k_bkt_reduce
    int64_t *big;               // their indices
};
PushView push_view(Workspace &ws, int32_t nseg, int64_t NBmax)
{
    PushView v;
    v.segB = ws.pk_seg.as<int64_t>();
    v.segBoff = v.segB + (nseg + 1);
    v.segsh = reinterpret_cast<int32_t *>(v.segBoff + (nseg + 1));
    v.segeb = v.segsh + (nseg + 1);
    v.cnt = ws.pk_bkt.as<int64_t>();     // NBmax + 1
    v.boff = v.cnt + (NBmax + 1);        // NBmax + 2 (offsets form)
    v.ucnt = v.boff + (NBmax + 2);       // NBmax + 1
    v.uoff = v.ucnt + (NBmax + 1);       // NBmax + 2
    v.bst = reinterpret_cast<BStat *>(v.uoff + (NBmax + 2));
    v.bseg = reinterpret_cast<int32_t *>(v.bst + (NBmax + 1));
    v.cur = reinterpret_cast<unsigned int *>(v.bseg + (NBmax + 1));
    v.nbig = reinterpret_cast<unsigned long long *>(v.cur + ((NBmax + 2) & ~(int64_t)1));   // 8-byte aligned
    v.big = reinterpret_cast<int64_t *>(v.nbig + 1);
    return v;
}
}  // namespace

// Part A for the chunk of segments [g0, g0 + ns) (whole queries), pairs [P0, P0 + E) of the
// wave's pair enumeration ent_off.
int smm_push_wave_a(Ctx &c, int32_t g0, int32_t ns, int64_t P0, int64_t E, const int64_t *ent_off)
{
    NvtxRange nvtx_("geer/smm_push");
    Workspace &ws = c.ws;
    er_graph *g = c.g;
    const cudaStream_t st = c.st;
    // per-segment plan (int64 counts for the scans); bucket count bound sum_g max(1, 2 E_g / TARGET)
    const int64_t NBmax = ns + 2 * (E / BKT_TARGET) + 1;
    ws.pk_nbmax = NBmax;
    ws.pk_e = E;
    ENSURE(ws.pk_seg, (sizeof(int64_t) * 2 + sizeof(int32_t) * 2) * (size_t)(ns + 2), false);
    ENSURE(ws.pk_bkt, (sizeof(int64_t) * 5 + sizeof(BStat) + sizeof(int32_t) * 2) * (size_t)(NBmax + 2) + 16, false);
    const PushView v = push_view(ws, ns, NBmax);
    int64_t *segB = v.segB, *segBoff = v.segBoff, *cnt = v.cnt, *boff = v.boff, *ucnt = v.ucnt, *uoff = v.uoff;
    int32_t *segsh = v.segsh, *segeb = v.segeb, *bseg = v.bseg;
    BStat *bst = v.bst;
    unsigned int *cur = v.cur;
    const int64_t *fr_off = ws.fr_off.as<int64_t>();
    k_bkt_plan<<<blocks_for(ns, 256), 256, 0, st>>>(ns, fr_off + g0, ent_off, g->nbits, segB, segsh, segeb);
    LAUNCHED(g);
    int rc = scan_offsets(c, segB, segBoff, ns);
    if (rc) return rc;
    const int64_t *dNB = segBoff + ns;                 // the bucket count, on the device
    CK(cudaMemsetAsync(cnt, 0, sizeof(int64_t) * (NBmax + 1), st));
    CK(cudaMemsetAsync(cur, 0, sizeof(unsigned int) * (NBmax + 1), st));
    CK(cudaMemsetAsync(ucnt, 0, sizeof(int64_t) * (NBmax + 1), st));
    CK(cudaMemsetAsync(v.nbig, 0, sizeof(unsigned long long), st));
    k_bkt_seg<<<blocks_for(NBmax, 256), 256, 0, st>>>(ns, segBoff, dNB, bseg);
    LAUNCHED(g);
    // entry range of the chunk (host copies of two frontier offsets are not needed: the kernels
    // search the whole frontier's ent_off, which is monotone)
    const int64_t e_lo = 0, e_hi = c.ws.pk_F;
    const unsigned eg = blocks_for((E + EMIT_PER - 1) / EMIT_PER + 31, 256);
    k_bkt_count<<<eg, 256, 0, st>>>(P0, E, e_lo, e_hi, g0, ent_off, ws.fr_id.as<int32_t>(), ws.fr_seg.as<int32_t>(),
                                    g->d_off, g->d_cols, segBoff, segsh, reinterpret_cast<unsigned long long *>(cnt));
    LAUNCHED(g);
    rc = scan_offsets(c, cnt, boff, NBmax);
    if (rc) return rc;
    ENSURE(ws.pk_keys, sizeof(unsigned long long) * (size_t)E, false);
    ENSURE(ws.pk_alt, sizeof(unsigned long long) * (size_t)E, false);
    ENSURE(ws.pk_out, (sizeof(int32_t) * 2 + sizeof(double)) * (size_t)E, false);
    unsigned long long *keys = ws.pk_keys.as<unsigned long long>();
    double *out_val = ws.pk_out.as<double>();
    int32_t *out_id = reinterpret_cast<int32_t *>(out_val + E);
    int32_t *gruns = out_id + E;   // run starts of the buckets above BKT_CAP
    k_bkt_scatter<<<eg, 256, 0, st>>>(P0, E, e_lo, e_hi, g0, ent_off, ws.fr_id.as<int32_t>(), ws.fr_seg.as<int32_t>(),
                                      fr_off, g->d_off, g->d_cols, segBoff, segsh, segeb, boff, cur, keys);
    LAUNCHED(g);
    const size_t smem = sizeof(unsigned long long) * 2 * BKT_CAP + sizeof(int) * BKT_CAP;
    static bool attr = false;
    if (!attr) {
        CK(cudaFuncSetAttribute(k_bkt_reduce, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        attr = true;
    }
    k_bkt_reduce_warp<<<(unsigned)std::min<int64_t>((NBmax + BKT_WPB - 1) / BKT_WPB, (int64_t)g->num_sms * 16),
                        32 * BKT_WPB, 0, st>>>(g0, dNB, bseg, segBoff, segsh, segeb, boff, keys, fr_off,
                                               ws.fr_val.as<double>(), g->d_rec, ws.act.as<int32_t>(),
                                               ws.qs.as<QState>(), out_id, out_val, ucnt, bst, v.nbig, v.big);
    LAUNCHED(g);
    // the listed buckets: persistent CTAs over the list (its length stays on the device)
    k_bkt_reduce<<<(unsigned)std::min<int64_t>(NBmax, (int64_t)g->num_sms * 4), BKT_NT, smem, st>>>(
        g0, reinterpret_cast<const int64_t *>(v.nbig), v.big, bseg, segBoff, segsh, segeb, boff, keys,
        ws.pk_alt.as<unsigned long long>(), fr_off, ws.fr_val.as<double>(), g->d_rec, ws.act.as<int32_t>(),
        ws.qs.as<QState>(), out_id, out_val, gruns, ucnt, bst);
    LAUNCHED(g);
    rc = scan_offsets(c, ucnt, uoff, NBmax);
    if (rc) return rc;
    CK(cudaGetLastError());
    return ER_OK;
}

int smm_push_wave_b(Ctx &c, int32_t g0, int32_t ns, int64_t *dU)
{
    Workspace &ws = c.ws;
    er_graph *g = c.g;
    const cudaStream_t st = c.st;
    const int64_t NBmax = ws.pk_nbmax;
    const PushView v = push_view(ws, ns, NBmax);
    const int64_t *dNB = v.segBoff + ns;
    double *out_val = ws.pk_out.as<double>();
    const int32_t *out_id = reinterpret_cast<const int32_t *>(out_val + ws.pk_e);
    k_bkt_merge<<<(unsigned)ns, MERGE_NT, 0, st>>>(ns, g0, v.segBoff, v.bst, ws.segstat.as<SegStat>());
    LAUNCHED(g);
    k_bkt_gather<<<blocks_for(NBmax * 32, 256), 256, 0, st>>>(dNB, ns, g0, v.bseg, v.segBoff, v.boff, v.uoff, out_id,
                                                              out_val, ws.nf_id.as<int32_t>(), ws.nf_val.as<double>(),
                                                              ws.nf_seg.as<int32_t>(), ws.nf_off.as<int64_t>(), dU);
    LAUNCHED(g);
    CK(cudaGetLastError());
    return ER_OK;
}

}  // namespace geer
