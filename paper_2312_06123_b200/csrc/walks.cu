// walks.cu -- the AMC part of the pipeline (Alg. 1): K6 k_walks (the random walks,
// y summed along them) and K7 k_amc_reduce (Z, sigma^2, the Bernstein stop), tau batches per
// AMC group enqueued on one stream without host synchronisation.

#include "stages.h"

// Column chunk loads of DRAM-resident walk graphs skip L1 (they are never reused; the y records
// keep the L1 lines: LJ-shaped walks 361.4 -> 357.2 ms on one box); y loads with L1 evict_last
// measured slower (366.8 ms).  Both are compile-time switches for A/B builds.
#ifndef GEER_COL_L1NA
#define GEER_COL_L1NA 1
#endif
#ifndef GEER_Y_L1EL
#define GEER_Y_L1EL 0
#endif

namespace geer {

// Chunks of walk pairs of batch b per AMC query, and the AMC sort key (descending ell_f) used to
// order the flattened walk space so warps mostly see one trip count.
__global__ void k_nchunks(int32_t na, const int32_t *__restrict__ amc, const QState *__restrict__ qs, int b,
                          int reuse, int32_t per_chunk, int64_t *__restrict__ nch)
{
    const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= na) return;
    const QState &Q = qs[amc[i]];
    const int64_t cnt = (Q.st.eta0 << b) - walks_lo(Q.st.eta0, b, reuse);
    nch[i] = Q.phase == PH_AMC ? (cnt + per_chunk - 1) / per_chunk : 0;
}

// Stable order of an AMC list by descending ell_f (bins of ell_f clamped at LF_BINS - 1), by one
// CTA: histogram, bin offsets, then tiles of LF_NT items placed in list order (a lane's slot = its
// bin's running offset + the same-bin items of earlier warps and lanes of the tile).
constexpr int LF_NT = 1024;
constexpr int LF_BINS = 1024;
__global__ void __launch_bounds__(LF_NT) k_lf_order(int32_t na, const int32_t *__restrict__ amc,
                                                    const QState *__restrict__ qs, int32_t *__restrict__ out)
{
    __shared__ unsigned int off[LF_BINS];
    __shared__ unsigned char wcnt[LF_NT / 32][LF_BINS + 1];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int i = tid; i < LF_BINS; i += LF_NT) off[i] = 0u;
    for (int i = tid; i < (LF_NT / 32) * (LF_BINS + 1); i += LF_NT) (&wcnt[0][0])[i] = 0;
    __syncthreads();
    auto bin = [&](int32_t i) {   // descending ell_f first
        const int32_t lf = qs[amc[i]].st.ell_f;
        return (unsigned)(LF_BINS - 1 - (lf < LF_BINS - 1 ? lf : LF_BINS - 1));
    };
    for (int32_t i = tid; i < na; i += LF_NT) atomicAdd(&off[bin(i)], 1u);
    __syncthreads();
    if (warp == 0) {   // exclusive scan of the bin counts, LF_BINS / 32 per lane
        constexpr int PER = LF_BINS / 32;
        unsigned v[PER], sum = 0;
#pragma unroll
        for (int j = 0; j < PER; j++) {
            v[j] = off[lane * PER + j];
            sum += v[j];
        }
        unsigned incl = sum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned t = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += t;
        }
        unsigned run = incl - sum;
#pragma unroll
        for (int j = 0; j < PER; j++) {
            off[lane * PER + j] = run;
            run += v[j];
        }
    }
    __syncthreads();
    for (int32_t t0 = 0; t0 < na; t0 += LF_NT) {
        const int32_t i = t0 + tid;
        const bool valid = i < na;
        const unsigned d = valid ? bin(i) : (unsigned)LF_BINS;
        const unsigned peers = __match_any_sync(0xffffffffu, d);
        const unsigned lt = peers & ((1u << lane) - 1u);
        if (lt == 0) wcnt[warp][d] = (unsigned char)__popc(peers);
        __syncthreads();
        if (valid) {
            unsigned pos = off[d] + __popc(lt);
            for (int w = 0; w < warp; w++) pos += wcnt[w][d];
            out[pos] = amc[i];
        }
        __syncthreads();
        for (int bb = tid; bb < LF_BINS; bb += LF_NT) {
            unsigned c = 0;
            for (int w = 0; w < LF_NT / 32; w++) c += wcnt[w][bb];
            off[bb] += c;
        }
        __syncthreads();
        if (lt == 0) wcnt[warp][d] = 0;
        __syncthreads();
    }
}

constexpr int WALK_WARPS = 8;
constexpr int WALK_THREADS = 32 * WALK_WARPS;

__device__ __forceinline__ int32_t find_chunk_query(const int64_t *__restrict__ cincl, int32_t n, int64_t c)
{
    int32_t lo = 0, hi = n - 1;  // smallest i with cincl[i] > c
    while (lo < hi) {
        const int32_t mid = (lo + hi) >> 1;
        if (cincl[mid] > c) hi = mid;
        else lo = mid + 1;
    }
    return lo;
}

// The 4 keys of a bucket: index of v, or -1; *empty = the bucket has a free slot.
__device__ __forceinline__ int bucket_match(const int4 a, int32_t v, bool *empty)
{
    int m = -1;
    m = (a.w == v) ? 3 : m;
    m = (a.z == v) ? 2 : m;
    m = (a.y == v) ? 1 : m;
    m = (a.x == v) ? 0 : m;
    *empty = (a.x < 0) | (a.y < 0) | (a.z < 0) | (a.w < 0);
    return m;
}

// L2 evict-first access policy (for the one-off random loads of a DRAM-resident walk graph).
__device__ __forceinline__ uint64_t pol_evict_first()
{
    uint64_t p;
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
// Fraction `keep` of the lines (by address) L2 evict-last, the others evict-first: a fixed part
// of a DRAM-resident walk graph stays in L2 while the rest streams past.
__device__ __forceinline__ uint64_t pol_keep_fraction(float keep)
{
    uint64_t p;
    asm("createpolicy.fractional.L2::evict_last.L2::evict_first.b64 %0, %1;" : "=l"(p) : "f"(keep));
    return p;
}
// Walk-graph loads.  DL = the walk graph is DRAM-resident (every layout but the
// packed one): column / arc loads are L2 evict-first (one-off random accesses must not push the
// y-tables and node records out of L2) with the 64-byte L2 fetch size (a random DRAM miss
// otherwise moves a 128-byte line), node records 64-byte fetches; L2-resident packed records:
// plain loads.  (Measured alternatives: profiles/exp_walk_policy_r02.jsonl.)
template <bool DL>
__device__ __forceinline__ uint4 ld_arc_v4(const uint4 *p, uint64_t apol)
{
    if (!DL) return __ldg(p);
    uint4 r;
#if GEER_COL_L1NA
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.L2::64B.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
        : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p), "l"(apol));
#else
    asm("ld.global.nc.L2::cache_hint.L2::64B.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
        : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p), "l"(apol));
#endif
    return r;
}
template <bool DL>
__device__ __forceinline__ unsigned long long ld_arc_u64(const unsigned long long *p, uint64_t apol)
{
    if (!DL) return __ldg(p);
    unsigned long long r;
    asm("ld.global.nc.L2::cache_hint.L2::64B.u64 %0, [%1], %2;" : "=l"(r) : "l"(p), "l"(apol));
    return r;
}
template <bool DL>
__device__ __forceinline__ int32_t ld_arc_s32(const int32_t *p, uint64_t apol)
{
    if (!DL) return __ldg(p);
    int32_t r;
    asm("ld.global.nc.L2::cache_hint.L2::64B.s32 %0, [%1], %2;" : "=r"(r) : "l"(p), "l"(apol));
    return r;
}
// node record {offset, degree} of the walk's current node
template <bool DL>
__device__ __forceinline__ uint2 ld_rec(const uint2 *p)
{
    if (!DL) return __ldg(p);
    uint2 r;
    asm("ld.global.nc.L2::64B.v2.u32 {%0,%1}, [%2];" : "=r"(r.x), "=r"(r.y) : "l"(p));
    return r;
}

#if GEER_Y_L1EL
__device__ __forceinline__ double ld_y(const double *p)
{
    double v;
    asm("ld.global.nc.L1::evict_last.f64 %0, [%1];" : "=d"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ uint4 ld_y(const uint4 *p)
{
    uint4 r;
    asm("ld.global.nc.L1::evict_last.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
    return r;
}
#else
__device__ __forceinline__ double ld_y(const double *p) { return __ldg(p); }
__device__ __forceinline__ uint4 ld_y(const uint4 *p) { return __ldg(p); }
#endif

// Hash lookups: slot of v, or -1 when v is not in supp(y) (then y(v) = 0, Alg. 1 L7 outside
// U_s and U_t).  Staged keys in shared memory, or the table in global memory (one 16-byte
// bucket per probe).  ylookup_global_from continues a global probe at bucket bk.
__device__ __forceinline__ int4 ld_bucket(const int32_t *keys, uint32_t bk)
{
    return __ldg(reinterpret_cast<const int4 *>(keys + (size_t)bk * YB));
}
__device__ __forceinline__ int64_t ylookup_smem(const int32_t *skeys, int lgb, int32_t v)
{
    const uint32_t bmask = (1u << lgb) - 1u;
    uint32_t bk = ybucket(v, lgb);
    while (true) {
        const int4 a = reinterpret_cast<const int4 *>(skeys + (size_t)bk * YB)[0];
        bool empty;
        const int m = bucket_match(a, v, &empty);
        if (m >= 0) return (int64_t)bk * YB + m;
        if (empty) return -1;
        bk = (bk + 1) & bmask;
    }
}
__device__ __forceinline__ int64_t ylookup_global_from(const int32_t *keys, int lgb, int32_t v, uint32_t bk)
{
    const uint32_t bmask = (1u << lgb) - 1u;
    while (true) {
        const int4 a = ld_bucket(keys, bk);
        bool empty;
        const int m = bucket_match(a, v, &empty);
        if (m >= 0) return (int64_t)bk * YB + m;
        if (empty) return -1;
        bk = (bk + 1) & bmask;
    }
}
// Resolve a global probe whose first bucket `a` (of node v) was loaded one step earlier.
__device__ __forceinline__ int64_t ylookup_resolve(const int4 a, const int32_t *keys, int lgb, int32_t v)
{
    bool empty;
    const int m = bucket_match(a, v, &empty);
    const uint32_t bk = ybucket(v, lgb);
    if (m >= 0) return (int64_t)bk * YB + m;
    if (empty) return -1;
    return ylookup_global_from(keys, lgb, v, (bk + 1) & ((1u << lgb) - 1u));   // full bucket: rare
}

// Layout 4: node record {off(v), d(v)} of renumbered node v from the degree-class tables staged
// in shared memory (geer_internal.h DOrdView): class of v's block, then the class's {base', d}.
// 32-bit words of K6's layout-4 tables in shared memory (rounded to 16 bytes for the staging area)
__host__ __device__ inline int32_t dord_smem_words(int32_t ncls, int32_t nblk)
{
    return ((2 * ncls + (nblk + 1) / 2) + 3) & ~3;
}
struct STree {
    const uint16_t *blk;
    const uint2 *cd;
    int32_t bshift;
};
__device__ __forceinline__ uint2 class_rec(const STree &T, uint32_t v)
{
    const uint2 cd = T.cd[T.blk[v >> T.bshift]];
    return make_uint2(cd.x + v * cd.y, cd.y);   // base_c + (v - vstart_c) d_c, exact mod 2^32 (off < 2^32)
}

// Column p (0..4) of a 24-bit chunk: bytes 3p..3p+2, i.e. bits 24p..24p+23 of the 128-bit chunk.
// Branch-free (selects only), and applied only after every chain's chunk load has been issued:
// a data-dependent branch between two chains' loads makes the second wait for the first.
__device__ __forceinline__ uint32_t col24(const uint4 q, uint32_t p)
{
    const uint64_t lo = ((uint64_t)q.y << 32) | q.x, hi = ((uint64_t)q.w << 32) | q.z;
    const uint32_t bo = 24u * p;   // 0, 24, 48, 72, 96
    uint64_t v = (bo < 64u ? lo : hi) >> (bo & 63u);
    v |= bo == 48u ? hi << 16 : 0ull;   // bits 48..71 straddle the two halves
    return (uint32_t)v & 0xFFFFFFu;
}

template <int ARC>
__device__ __forceinline__ uint4 next_arc(const uint2 R, uint64_t r64, const uint4 *__restrict__ arcs,
                                          const int32_t *__restrict__ cols,
                                          const unsigned long long *__restrict__ parcs, PackSpec pk, uint64_t apol,
                                          uint32_t *p24)
{
    const uint64_t e = (uint64_t)R.x + __umul64hi(r64, (uint64_t)R.y);   // idx = floor(r64 d / 2^64) (R10)
    constexpr bool DL = ARC != 2;
    if (ARC == 2) return pk.unpack(ld_arc_u64<DL>(parcs + e, apol));
    if (ARC == 1) return ld_arc_v4<DL>(arcs + e, apol);
    if (ARC == 3 || ARC == 4) {   // 24-bit columns, 5 per 16-byte chunk: the raw chunk; *p24 = its slot
        const uint64_t ch = e / 5u;
        *p24 = (uint32_t)(e - 5u * ch);
        return ld_arc_v4<DL>(arcs + ch, apol);
    }
    uint4 A;
    A.x = (uint32_t)ld_arc_s32<DL>(cols + e, apol);
    return A;
}

// y-lookup modes of a warp (its query's table layout and the tile's staging plan).
enum { YM_GLOBAL = 0, YM_SMEM = 1, YM_RANK = 2 };

// NP walk pairs per thread = 2 NP independent chains (S_k from s, T_k from t for each pair),
// advanced in lock step so 2 NP arc loads are in flight per thread.  Per step and chain:
// Philox draw (R10; the even step's words are cached from the odd step's call), one arc load
// (the chain's only dependent memory access), then y(v):
//   YM_SMEM    hash keys staged in shared memory: probe now, value load consumed next step;
//   YM_GLOBAL  hash keys in global memory: first bucket (16 B) load issued now and resolved next
//              step (a full bucket continues synchronously, rare at load <= 1/2), value load
//              consumed the step after;
//   YM_RANK    rank-bitmap record (16 B) load issued now and resolved next step, value load
//              consumed the step after.
// The pipelined loads (bucket or record) overlap the next arc load, so only the arc load is
// on the chain.
// y values are added in step order (R9, R13).
template <int ARC, int NP>
__device__ __forceinline__ void walk_chains(const uint2 *__restrict__ rec, const uint4 *__restrict__ arcs,
                                            const int32_t *__restrict__ cols,
                                            const unsigned long long *__restrict__ parcs, PackSpec pk, int mode,
                                            const int32_t *skeys, const int32_t *__restrict__ gkeys,
                                            const uint4 *__restrict__ yrec, const double *__restrict__ gvals,
                                            int lgb, int32_t s, int32_t t, int32_t lf, uint32_t q, uint32_t b,
                                            const uint64_t *kk, uint32_t key0, uint32_t key1, double *acc,
                                            int32_t *endv, uint64_t apol, const STree &T)
{
    constexpr int C = 2 * NP;
    uint2 R[C];
    int32_t v[C];
    double pv[C];
    uint32_t cz[C], cw[C];
    uint4 prec[C];       // YM_RANK record / YM_GLOBAL first bucket of the previous step's node
#pragma unroll
    for (int c = 0; c < C; c++) {
        v[c] = (c & 1) ? t : s;
        R[c] = ARC == 4 ? class_rec(T, (uint32_t)v[c]) : ld_rec<ARC != 2>(rec + v[c]);
        acc[c] = 0.0;
        pv[c] = 0.0;
        cz[c] = 0u;
        cw[c] = 0u;
        // the start node is not summed (R9): no rank bits / an empty bucket
        prec[c] = mode == YM_GLOBAL ? make_uint4(~0u, ~0u, ~0u, ~0u) : make_uint4(0u, 0u, 0u, 0u);
    }
    for (int32_t j = 1; j <= lf; j++) {
        uint4 A[C];
        uint32_t p24[C];
#pragma unroll
        for (int c = 0; c < C; c++) {
            uint64_t r64;
            if (j & 1) {
                const uint64_t k = kk[c >> 1];
                const U4 r = philox4x32_10(U4{(uint32_t)((j - 1) >> 1), (uint32_t)k, q,
                                              (b << 29) | ((uint32_t)(c & 1) << 28) | (uint32_t)(k >> 32)},
                                           key0, key1);
                r64 = ((uint64_t)r.y << 32) | r.x;
                cz[c] = r.z;
                cw[c] = r.w;
            } else {
                r64 = ((uint64_t)cw[c] << 32) | cz[c];
            }
            A[c] = next_arc<ARC>(R[c], r64, arcs, cols, parcs, pk, apol, &p24[c]);
        }
        if (ARC == 3 || ARC == 4) {
#pragma unroll
            for (int c = 0; c < C; c++) A[c].x = col24(A[c], p24[c]);
        }
#pragma unroll
        for (int c = 0; c < C; c++) {
            acc[c] += pv[c];   // y of an earlier step, in step order
            pv[c] = 0.0;
            if (mode != YM_SMEM) {   // resolve the previous step's node (v[c])
                const int64_t idx = mode == YM_RANK ? rank_index(prec[c], v[c])
                                                    : ylookup_resolve(*reinterpret_cast<const int4 *>(&prec[c]),
                                                                      gkeys, lgb, v[c]);
                if (idx >= 0) pv[c] = ld_y(gvals + idx);
            }
            v[c] = (int32_t)A[c].x;
            if (ARC == 1 || ARC == 2) R[c] = make_uint2(A[c].y, A[c].z);
            else if (ARC == 4) R[c] = class_rec(T, (uint32_t)v[c]);
            else R[c] = ld_rec<ARC != 2>(rec + v[c]);
            if (mode == YM_RANK) {
                prec[c] = ld_y(yrec + rank_rec(v[c]));
            } else if (mode == YM_GLOBAL) {
                const int4 bk = ld_bucket(gkeys, ybucket(v[c], lgb));
                prec[c] = make_uint4((uint32_t)bk.x, (uint32_t)bk.y, (uint32_t)bk.z, (uint32_t)bk.w);
            } else {
                const int64_t slot = ylookup_smem(skeys, lgb, v[c]);
                if (slot >= 0) pv[c] = ld_y(gvals + slot);
            }
        }
    }
#pragma unroll
    for (int c = 0; c < C; c++) {
        acc[c] += pv[c];
        if (mode != YM_SMEM && lf > 0) {
            const int64_t idx = mode == YM_RANK ? rank_index(prec[c], v[c])
                                                : ylookup_resolve(*reinterpret_cast<const int4 *>(&prec[c]), gkeys,
                                                                  lgb, v[c]);
            if (idx >= 0) acc[c] += ld_y(gvals + idx);
        }
        endv[c] = v[c];
    }
}

// One chunk of K6: 32 NP walk pairs of AMC query list entry i (lane l, pair p runs walk
// k = 32 NP chunk' + 32 p + l, chunk' = chunk - the query's first chunk); writes the canonical
// partial {sum Z, sum Z^2, checksum} of the chunk.
template <int ARC, int NP>
__device__ __forceinline__ void walk_chunk(int64_t chunk, int32_t i, int mode, const int32_t *skeys,
                                           const int64_t *__restrict__ cincl, const int32_t *__restrict__ amc,
                                           const QState *__restrict__ qs, const uint2 *__restrict__ rec,
                                           const uint4 *__restrict__ arcs, const int32_t *__restrict__ cols,
                                           const unsigned long long *__restrict__ parcs, PackSpec pk, int b,
                                           uint32_t key0, uint32_t key1, int reuse, uint64_t apol,
                                           TilePart *__restrict__ parts, const DOrdView &dv, const STree &T)
{
    const int lane = threadIdx.x & 31;
    const QState &Q = qs[amc[i]];
    const int64_t c0 = i == 0 ? 0 : cincl[i - 1];
    const int64_t eta = Q.st.eta0 << b;
    const uint64_t klo = (uint64_t)walks_lo(Q.st.eta0, b, reuse);
    const uint32_t bkey = reuse ? 0u : (uint32_t)b;   // reuse: one sample stream per query
    const uint32_t q = Q.gq;
    uint64_t kk[NP];
    bool any = false;
#pragma unroll
    for (int p = 0; p < NP; p++) {
        kk[p] = klo + (uint64_t)(chunk - c0) * (32u * NP) + 32u * p + (uint64_t)lane;
        any |= kk[p] < (uint64_t)eta;
    }
    double acc[2 * NP];
    int32_t endv[2 * NP];
    double s1 = 0.0, s2 = 0.0;
    uint64_t ck = 0ull;
    if (any) {
        // layout 4 walks (and its y-tables are keyed) in the renumbered ids; the end nodes go back
        // to the caller's ids for the checksum
        const int32_t s = ARC == 4 ? __ldg(dv.perm + Q.s) : Q.s, t = ARC == 4 ? __ldg(dv.perm + Q.t) : Q.t;
        walk_chains<ARC, NP>(rec, arcs, cols, parcs, pk, mode, skeys, Q.ykeys, Q.yrec, Q.yvals, Q.ylog2 - YB_LOG,
                             s, t, Q.st.ell_f, q, bkey, kk, key0, key1, acc, endv, apol, T);
#pragma unroll
        for (int p = 0; p < NP; p++) {
            if (ARC == 4 && kk[p] < (uint64_t)eta) {
                endv[2 * p] = __ldg(dv.iperm + endv[2 * p]);
                endv[2 * p + 1] = __ldg(dv.iperm + endv[2 * p + 1]);
            }
        }
#pragma unroll
        for (int p = 0; p < NP; p++) {
            if (kk[p] < (uint64_t)eta) {
                const double z = acc[2 * p] - acc[2 * p + 1];   // Z_k (Alg. 1 L8)
                s1 += z;
                s2 += z * z;
                ck += walk_hash(q, bkey, 0u, kk[p], endv[2 * p]) + walk_hash(q, bkey, 1u, kk[p], endv[2 * p + 1]);
            }
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        s1 += __shfl_xor_sync(0xffffffffu, s1, o);
        s2 += __shfl_xor_sync(0xffffffffu, s2, o);
        ck += __shfl_xor_sync(0xffffffffu, ck, o);
    }
    if (lane == 0) {
        TilePart tp;
        tp.s1 = s1;
        tp.s2 = s2;
        tp.ck = ck;
        tp.pad = 0;
        parts[chunk] = tp;
    }
}

// K6: warp = one chunk of 32 NP walk pairs of one query at a time (chunks of all AMC queries
// are laid out query after query, queries ordered by descending ell_f).  Persistent: chunks are
// handed out by an atomic counter (dynamic balance: the first chunks, of the longest walks, are
// the longest); with tile_ctr == nullptr one chunk per warp.  Default (smem_words == 0): every
// warp takes its own chunks, no barriers.  With a staging area (GEER_WALK_SMEM_KB > 0): CTA-tiles
// of WALK_WARPS consecutive chunks, and a per-tile plan stages the hash keys of each distinct
// small-table query of the tile in shared memory (slower on B200: shared memory is taken from
// the L1 that holds the loads in flight).
template <int ARC, int NP, int MINB>
__global__ void __launch_bounds__(WALK_THREADS, MINB)
k_walks(int32_t na, const int64_t *__restrict__ cincl, const int32_t *__restrict__ amc,
        const QState *__restrict__ qs, const uint2 *__restrict__ rec, const uint4 *__restrict__ arcs,
        const int32_t *__restrict__ cols, const unsigned long long *__restrict__ parcs, PackSpec pk, int b,
        uint32_t key0, uint32_t key1, int32_t smem_words, int reuse,
        unsigned long long *__restrict__ tile_ctr, TilePart *__restrict__ parts, DOrdView dv, float keep)
{
    extern __shared__ __align__(32) int32_t sm_dyn[];
    __shared__ int32_t s_qi[WALK_WARPS];
    __shared__ int32_t s_soff[WALK_WARPS];
    __shared__ int32_t s_mode[WALK_WARPS];
    __shared__ int64_t s_tile;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t nchunks = cincl[na - 1];   // read on the device: no host round trip per batch
    const uint64_t apol = ARC == 2 ? 0 : keep > 0.f ? pol_keep_fraction(keep) : pol_evict_first();
    // layout 4: the degree-class tables first in dynamic shared memory (cd, then blk), staging after
    STree T{nullptr, nullptr, 0};
    int32_t *sm_words = sm_dyn;
    if (ARC == 4) {
        uint2 *scd = reinterpret_cast<uint2 *>(sm_dyn);
        uint16_t *sblk = reinterpret_cast<uint16_t *>(scd + dv.ncls);
        for (int32_t k = threadIdx.x; k < dv.ncls; k += WALK_THREADS) scd[k] = __ldg(dv.cd + k);
        for (int32_t k = threadIdx.x; k < dv.nblk; k += WALK_THREADS) sblk[k] = __ldg(dv.blk + k);
        __syncthreads();
        T = STree{sblk, scd, dv.bshift};
        sm_words = sm_dyn + dord_smem_words(dv.ncls, dv.nblk);
    }
    if (smem_words == 0) {
        int32_t i = 0;   // a warp's chunks only increase: its query index only moves forward
        for (int it = 0;; it++) {
            int64_t chunk = 0;
            if (lane == 0)
                chunk = tile_ctr ? (int64_t)atomicAdd(tile_ctr, 1ull)
                                 : (it == 0 ? (int64_t)blockIdx.x * WALK_WARPS + warp : nchunks);
            chunk = __shfl_sync(0xffffffffu, chunk, 0);
            if (chunk >= nchunks) break;
            if (cincl[i] <= chunk) i += 1 + find_chunk_query(cincl + i + 1, na - i - 1, chunk);
            const int mode = qs[amc[i]].ymode == YT_RANK ? YM_RANK : YM_GLOBAL;
            walk_chunk<ARC, NP>(chunk, i, mode, nullptr, cincl, amc, qs, rec, arcs, cols, parcs, pk, b, key0, key1,
                                reuse, apol, parts, dv, T);
        }
        return;
    }
    for (int it = 0;; it++) {
        if (threadIdx.x == 0)
            s_tile = tile_ctr ? (int64_t)atomicAdd(tile_ctr, 1ull) : (it == 0 ? (int64_t)blockIdx.x : nchunks);
        __syncthreads();
        const int64_t tile = s_tile;
        if (tile * WALK_WARPS >= nchunks) break;
        const int64_t chunk = tile * WALK_WARPS + warp;
        const bool wvalid = chunk < nchunks;
        const int32_t i = wvalid ? find_chunk_query(cincl, na, chunk) : -1;
        if (lane == 0) s_qi[warp] = i;
        __syncthreads();
        if (threadIdx.x == 0) {
            // prefix-fit staging plan over the distinct queries of this tile (consecutive warps)
            int32_t used = 0;
            for (int w = 0; w < WALK_WARPS; w++) {
                const int32_t qi = s_qi[w];
                s_soff[w] = 0;
                if (qi < 0) { s_mode[w] = YM_GLOBAL; continue; }
                if (w > 0 && s_qi[w - 1] == qi) { s_soff[w] = s_soff[w - 1]; s_mode[w] = s_mode[w - 1]; continue; }
                const QState &Q = qs[amc[qi]];
                if (Q.ymode == YT_RANK) { s_mode[w] = YM_RANK; continue; }
                const int32_t cap = 1 << Q.ylog2;
                if (cap <= WALK_KEY_SLOTS && used + cap <= smem_words) {
                    s_soff[w] = used; s_mode[w] = YM_SMEM; used += cap;
                } else {
                    s_mode[w] = YM_GLOBAL;
                }
            }
        }
        __syncthreads();
        for (int w = 0; w < WALK_WARPS; w++) {
            if (s_mode[w] != YM_SMEM || (w > 0 && s_qi[w - 1] == s_qi[w])) continue;
            const QState &Q = qs[amc[s_qi[w]]];
            const int4 *src = reinterpret_cast<const int4 *>(Q.ykeys);
            int4 *dst = reinterpret_cast<int4 *>(sm_words + s_soff[w]);
            const int32_t words = 1 << Q.ylog2;
            for (int32_t e = threadIdx.x; e < words / 4; e += WALK_THREADS) dst[e] = __ldg(src + e);
        }
        __syncthreads();
        if (wvalid)
            walk_chunk<ARC, NP>(chunk, i, s_mode[warp], sm_words + s_soff[warp], cincl, amc, qs, rec, arcs, cols,
                                parcs, pk, b, key0, key1, reuse, apol, parts, dv, T);
        __syncthreads();
    }
}

// K7: one warp per AMC query: sum its chunk partials (chunk order, R13), then Alg. 1 L11-L14.
// Also writes the chunk count of batch b+1 into nch (0 once a query stops; a query that had no
// chunks in batch b already has 0 there), so only batch 0 needs k_nchunks.
__global__ void k_amc_reduce(int32_t na, const int32_t *__restrict__ amc, const int64_t *__restrict__ tile_incl,
                             const TilePart *__restrict__ parts, int b, BatchParams P, QState *__restrict__ qs,
                             unsigned long long *__restrict__ steps_counter, int64_t *__restrict__ nch,
                             int32_t per_chunk)
{
    const int lane = threadIdx.x & 31;
    const int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (i >= na) return;
    const int64_t t0 = i == 0 ? 0 : tile_incl[i - 1], t1 = tile_incl[i];
    if (t1 == t0) return;   // stopped in an earlier batch
    double s1 = 0.0, s2 = 0.0;
    uint64_t ck = 0;
#pragma unroll 4
    for (int64_t t = t0 + lane; t < t1; t += 32) {
        s1 += parts[t].s1;
        s2 += parts[t].s2;
        ck += parts[t].ck;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        s1 += __shfl_xor_sync(0xffffffffu, s1, o);
        s2 += __shfl_xor_sync(0xffffffffu, s2, o);
        ck += __shfl_xor_sync(0xffffffffu, ck, o);
    }
    if (lane != 0) return;
    QState &Q = qs[amc[i]];
    const int64_t eta = Q.st.eta0 << b;
    const int64_t drawn = eta - walks_lo(Q.st.eta0, b, P.reuse);
    if (P.reuse) {   // running sums over all samples so far
        Q.s1acc = (b == 0 ? 0.0 : Q.s1acc) + s1;
        Q.s2acc = (b == 0 ? 0.0 : Q.s2acc) + s2;
        s1 = Q.s1acc;
        s2 = Q.s2acc;
    }
    const double etaf = (double)eta;
    const double Z = s1 / etaf;
    double var = s2 / etaf - Z * Z;
    if (var < 0.0) var = 0.0;
    const double f = sqrt(2.0 * var * P.L_bern / etaf) + 3.0 * Q.st.psi * P.L_bern / etaf;
    Q.st.batches_run = b + 1;
    Q.st.walks_total += drawn;
    Q.st.steps_total += 2 * drawn * (int64_t)Q.st.ell_f;
    if (steps_counter) atomicAdd(steps_counter, (unsigned long long)(2 * drawn * (int64_t)Q.st.ell_f));
    Q.st.walk_checksum += ck;
    Q.st.f_last = f;
    Q.st.sigma2_last = var;
    Q.z = Z;
    if (fabs(f - P.eps / 2.0) <= 1e-12 * P.eps) Q.st.tie_flags |= 4u;
    const bool stop = f <= P.eps / 2.0 || b == P.tau - 1;
    if (stop) Q.phase = PH_DONE;
    const int64_t next = (Q.st.eta0 << (b + 1)) - walks_lo(Q.st.eta0, b + 1, P.reuse);
    nch[i] = stop ? 0 : (next + per_chunk - 1) / per_chunk;
}

// ---------------------------------------------------------------------------- host side

int launch_amc_group(er_graph *g, cudaStream_t sb, const AmcGroup &G, QState *qs, const BatchParams &P, bool prof,
                     BatchRes &R)
{
    NvtxRange nvtx_("geer/amc");
    const int32_t na = G.na;
    if (na == 0) return ER_OK;
    // per-group buffers (stream ordered on the AMC stream)
    const int per_chunk = 32 * g->walk_np;   // walk pairs per warp-chunk
    int64_t maxch = (int64_t)((G.eta0_sum << (P.tau - 1)) / per_chunk) + na + 1;
    int32_t *list2 = nullptr;
    int64_t *nch = nullptr, *cincl = nullptr;
    TilePart *parts = nullptr;
    void *tmp = nullptr;
    const size_t tbytes = scan_tmp_bytes<int64_t>(na) + 256;
    CK(cudaMallocAsync((void **)&list2, sizeof(int32_t) * na, sb));
    CK(cudaMallocAsync((void **)&nch, sizeof(int64_t) * na, sb));
    CK(cudaMallocAsync((void **)&cincl, sizeof(int64_t) * na, sb));
    CK(cudaMallocAsync((void **)&parts, sizeof(TilePart) * maxch, sb));
    unsigned long long *tctr = nullptr;   // K6 tile counters, one per batch
    CK(cudaMallocAsync((void **)&tctr, sizeof(unsigned long long) * P.tau, sb));
    CK(cudaMemsetAsync(tctr, 0, sizeof(unsigned long long) * P.tau, sb));
    R.bufs.push_back(tctr);
    CK(cudaMallocAsync(&tmp, tbytes, sb));
    for (void *p : {(void *)list2, (void *)nch, (void *)cincl, (void *)parts, tmp}) R.bufs.push_back(p);
    const int32_t *list = G.list;
    if (na > 1) {
        // order by descending ell_f (stable): the longest walks start first
        k_lf_order<<<1, LF_NT, 0, sb>>>(na, G.list, qs, list2);
        LAUNCHED(g);
        list = list2;
    }
    const int nsm = g->num_sms;
    const uint32_t key0 = (uint32_t)P.seed, key1 = (uint32_t)(P.seed >> 32);
    for (int b = 0; b < P.tau; b++) {
        if (b == 0) {   // later batches: written by the previous batch's k_amc_reduce
            k_nchunks<<<blocks_for(na, 256), 256, 0, sb>>>(na, list, qs, b, P.reuse, per_chunk, nch);
            LAUNCHED(g);
        }
        g->launches += scan_launch(sb, nch, cincl, (int64_t)na, (int64_t)0, ScanAdd<int64_t>(), tmp);
        const int64_t bound = (int64_t)((G.eta0_sum << b) / per_chunk) + na;   // chunks of batch b, at most
        cudaEvent_t e0 = nullptr, e1 = nullptr;
        if (prof) {
            CK(cudaEventCreate(&e0));
            CK(cudaEventCreate(&e1));
            CK(cudaEventRecord(e0, sb));
        }
#define WALK_ARGS                                                                                         \
    na, cincl, list, qs, g->d_rec, g->d_c24 ? g->d_c24 : g->d_arcs, g->d_cols, g->d_parcs, g->pack, b, key0,  \
        key1, smem_words,                                                                                     \
        P.reuse,                                                                                              \
        persist ? tctr + b : nullptr, parts, dv, g->walk_l2_keep
#define WALK_LAUNCH(ARC, NP, MINB)                                                                          \
    do {                                                                                                    \
        CK(cudaFuncSetAttribute(k_walks<ARC, NP, MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize,        \
                                (int)smem_bytes));                                                          \
        if (g->walk_carveout >= 0)                                                                          \
            CK(cudaFuncSetAttribute(k_walks<ARC, NP, MINB>, cudaFuncAttributePreferredSharedMemoryCarveout,   \
                                    g->walk_carveout));                                                     \
        int occ = 0;                                                                                        \
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_walks<ARC, NP, MINB>, WALK_THREADS,        \
                                                         smem_bytes));                                      \
        /* persistent grid: exactly the resident CTAs (a second wave would serialise) */                    \
        const int64_t tiles = (bound + WALK_WARPS - 1) / WALK_WARPS;                                         \
        const unsigned grid = (unsigned)std::max<int64_t>(                                                  \
            1, persist ? std::min<int64_t>((int64_t)std::max(1.0, slot_frac * std::max(occ, 1) * nsm), tiles)  \
                       : tiles);                                                                            \
        g->walk_occ = occ;                                                                                  \
        k_walks<ARC, NP, MINB><<<grid, WALK_THREADS, smem_bytes, sb>>>(WALK_ARGS);                          \
    } while (0)
#define WALK_ARC(NP, MINB)                                   \
    do {                                                     \
        if (g->d_parcs) WALK_LAUNCH(2, NP, MINB);            \
        else if (g->d_cblk) WALK_LAUNCH(4, NP, MINB);        \
        else if (g->d_c24) WALK_LAUNCH(3, NP, MINB);         \
        else if (g->d_arcs) WALK_LAUNCH(1, NP, MINB);        \
        else WALK_LAUNCH(0, NP, MINB);                       \
    } while (0)
        // smem_words: staging capacity (tile path); 0 = per-warp chunks; -1 = tile path, no staging
        const int32_t smem_words = g->walk_smem_words > 0 ? g->walk_smem_words : (g->walk_tiles ? -1 : 0);
        // with the SMM head running concurrently (overlap), the persistent walk grid takes only a
        // fraction of the resident-CTA slots so head kernels always find room on every SM
        const bool persist = g->walk_persist;
        const double slot_frac = g->amc_overlap ? g->overlap_frac : 1.0;
        DOrdView dv;
        size_t tree_bytes = 0;
        if (g->d_cblk) {
            dv.perm = g->d_perm;
            dv.iperm = g->d_iperm;
            dv.blk = g->d_cblk;
            dv.cd = g->d_ccd;
            dv.nblk = g->dord_nblk;
            dv.ncls = g->dord_ncls;
            dv.bshift = g->dord_bshift;
            tree_bytes = sizeof(int32_t) * (size_t)dord_smem_words(dv.ncls, dv.nblk);
        }
        const size_t smem_bytes = tree_bytes + sizeof(int32_t) * (size_t)std::max(smem_words, 0);
        if (g->walk_np == 1) {
            if (g->walk_minb == 3) WALK_ARC(1, 3);
            else if (g->walk_minb == 5) WALK_ARC(1, 5);
            else if (g->walk_minb == 6) WALK_ARC(1, 6);
            else WALK_ARC(1, 4);
        } else {
            if (g->walk_minb == 3) WALK_ARC(2, 3);
            else WALK_ARC(2, 4);
        }
#undef WALK_ARC
#undef WALK_LAUNCH
#undef WALK_ARGS
        LAUNCHED(g);
        if (prof) {
            CK(cudaEventRecord(e1, sb));
            R.walk_ev.push_back(e0);
            R.walk_ev.push_back(e1);
        }
        k_amc_reduce<<<blocks_for((int64_t)na * 32, 256), 256, 0, sb>>>(
            na, list, cincl, parts, b, P, qs, prof ? reinterpret_cast<unsigned long long *>(g->d_steps) : nullptr,
            nch, per_chunk);
        LAUNCHED(g);
    }
    CK(cudaGetLastError());
    return ER_OK;
}

}  // namespace geer
