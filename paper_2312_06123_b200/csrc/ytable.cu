// ytable.cu -- K5: the per-query y-tables of Alg. 1 L7 built from the SMM frontier of the
// queries that leave the head, and their host-side planning (one scalar read per wave).
//
// Every y(v) is written exactly once by the entry that owns v (no floating-point atomics); the
// tables are read by the walk kernel (walks.cu).

#include "stages.h"

namespace geer {

// The node id the walk kernel uses for node v (its y-table key): the degree-ordered renumbering
// of walk layout 4 (geer_internal.h DOrdView), else v.
__device__ __forceinline__ int32_t walk_id(const int32_t *__restrict__ perm, int32_t v)
{
    return perm != nullptr ? __ldg(perm + v) : v;
}

// y-tables (K5): y(v) = s*(v)/d(s) - t*(v)/d(t) on U = supp(s*) u supp(t*) for each query that
// leaves the SMM head for AMC in this wave (Alg. 1 L7 with s = s*, t = t*).  Two layouts,
// chosen per query by footprint:
//  * hash (YT_HASH): open addressing, 4 int32 keys per 16-byte bucket, buckets probed linearly;
//    capacity = next power of two >= 2 (|supp s*| + |supp t*|) (load <= 1/2), >= one bucket;
//    values fp64 by slot.  (Tables of <= WALK_KEY_SLOTS keys can be staged whole in the walk
//    kernel's shared memory, GEER_WALK_SMEM_KB; off by default.)
//  * rank bitmap (YT_RANK): one 16-byte record {U bits (96); rank U} per 96 node ids
//    (stages.h rank_rec / rank_index; rank U = |U| below the record), values fp64 by rank: y(v)
//    is at vals[rank U + popc(U bits below v)].  Exact membership in one 16-byte load, no probing;
//    used for tables too large to stage whose records take less than twice the hash layout's
//    12 B/slot (keys + values).
// Per leaving query i: h hash slots, v value slots, r rank records (0 for queries that stay).
struct YSizes {
    int64_t h, v, r;
};
struct YSizesPlus {
    __device__ __forceinline__ YSizes operator()(const YSizes &a, const YSizes &b) const
    {
        return YSizes{a.h + b.h, a.v + b.v, a.r + b.r};
    }
};

constexpr int YH_SMEM_SLOTS = 8192;   // larger hash tables: global CAS (k_yinsert)
#define YH_SMEM_SLOTS_DEV 8192

__global__ void k_ycap(int32_t na, const int32_t *__restrict__ act, const QState *__restrict__ qs,
                       const int32_t *__restrict__ cont, const int64_t *__restrict__ segoff, int64_t nrec,
                       int force, int64_t min_cap, int64_t ratio, int64_t max_bytes, YSizes *__restrict__ sz)
{
    const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= na) return;
    int64_t h = 0, v = 0, r = 0;
    if ((cont == nullptr || !cont[i]) && qs[act[i]].phase == PH_AMC) {
        const int64_t len = segoff[2 * i + 2] - segoff[2 * i];   // |supp s*| + |supp t*| >= |U|
        int64_t cap = YB;
        while (cap < 2 * len) cap <<= 1;
        // rank when the table cannot be small, its records are cheaper than twice the hash layout,
        // and they are small enough to stay mostly in L2 (large graphs: hash)
        const bool rank = force == 2 || (force == 0 && cap > min_cap && 16 * nrec < ratio * cap &&
                                         16 * nrec <= max_bytes);
        if (rank) {
            r = nrec;
            v = len;
        } else {
            h = cap;
            v = cap;
        }
    }
    sz[i] = YSizes{h, v, r};
}

// Build-time descriptor of leaving query i's table (a compact copy of its QState y fields,
// indexed by i: K5 reaches it in one load from the entry's segment).
struct YDesc {
    int32_t *keys;     // YT_HASH: 2^(lgb + YB_LOG) int32 keys
    uint4 *rec;        // YT_RANK: walk records {U bits 0-95, rank U}
    double *vals;      // y values (by slot or by rank)
    int32_t mode;      // -1: the query does not leave now; YT_HASH / YT_RANK
    int32_t lgb;       // YT_HASH: log2 of the bucket count
    int32_t ds, dt;    // d(s), d(t)
};

__global__ void k_yassign(int32_t na, const int32_t *__restrict__ act, const YSizes *__restrict__ sz,
                          const YSizes *__restrict__ incl, int32_t *kbase, double *vbase, uint4 *rbase,
                          QState *__restrict__ qs, YDesc *__restrict__ yd)
{
    const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= na) return;
    const YSizes n = sz[i], c = incl[i];
    YDesc D;
    D.mode = -1;
    D.keys = nullptr;
    D.rec = nullptr;
    D.vals = nullptr;
    D.lgb = 0;
    D.ds = D.dt = 1;
    if (n.v != 0) {
        QState &Q = qs[act[i]];
        D.ds = Q.ds;
        D.dt = Q.dt;
        D.vals = vbase + (c.v - n.v);
        Q.yvals = D.vals;
        if (n.r > 0) {
            D.mode = Q.ymode = YT_RANK;
            D.rec = rbase + (c.r - n.r);
            Q.yrec = D.rec;
            Q.ykeys = nullptr;
            Q.ylog2 = 0;
        } else {
            const int64_t cap = n.h;
            D.mode = Q.ymode = YT_HASH;
            D.keys = kbase + (c.h - cap);
            Q.ykeys = D.keys;
            Q.yrec = nullptr;
            int lg = 0;
            while ((1ll << lg) < cap) lg++;
            Q.ylog2 = lg;
            D.lgb = lg - YB_LOG;
        }
    }
    yd[i] = D;
}

__global__ void k_yfill(int64_t H, int32_t *__restrict__ keys, int64_t R, uint4 *__restrict__ rec)
{
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j < H) keys[j] = -1;
    if (j < R) rec[j] = make_uint4(0u, 0u, 0u, 0u);   // bits by k_ybits, ranks by k_yrank
}

// Rank tables: a value slot not yet written by a t* entry holds this NaN (no y value is a NaN).
constexpr unsigned long long Y_UNSET = 0x7FF4000000005E47ull;

__device__ __forceinline__ int32_t cas_global(int32_t *p, int32_t cmp, int32_t val)
{
    int32_t old;
    asm volatile("atom.global.cas.b32 %0, [%1], %2, %3;" : "=r"(old) : "l"(p), "r"(cmp), "r"(val) : "memory");
    return old;
}

// K5, hash layout: one CTA per leaving query builds its whole table -- in shared memory when it
// has at most YH_SMEM_SLOTS slots (then copied out), else in place in global memory -- with the
// same two passes as the rank path's owner rule: t* entries insert v with -(t*(v)/d_t), then s*
// entries find-or-insert v and complete y = s*(v)/d_s + stored (IEEE a - b is a + (-b)), or
// s*(v)/d_s - 0.0 when v is not in supp t*.  Every y(v) is written exactly once.
constexpr int YH_THREADS = 256;
template <bool SMEM>
__device__ __forceinline__ int32_t yh_cas(int32_t *p, int32_t cmp, int32_t val)
{
    if (SMEM) return atomicCAS(p, cmp, val);
    return cas_global(p, cmp, val);
}
template <bool SMEM>
__device__ __forceinline__ int32_t yh_load(const int32_t *p)
{
    if (SMEM) return *(volatile const int32_t *)p;
    int32_t v;
    asm volatile("ld.volatile.global.s32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}
template <bool SMEM>
__device__ __forceinline__ int64_t yh_insert(int32_t *keys, int lgb, int32_t v, bool *found)
{
    const uint32_t bmask = (1u << lgb) - 1u;
    uint32_t bk = ybucket(v, lgb);
    while (true) {
        for (int j = 0; j < YB; j++) {
            const uint32_t slot = bk * YB + j;
            int32_t k = yh_load<SMEM>(keys + slot);
            if (k == -1) k = yh_cas<SMEM>(keys + slot, -1, v);
            if (k == -1 || k == v) {
                *found = k == v;
                return slot;
            }
        }
        bk = (bk + 1) & bmask;
    }
}
template <bool SMEM>
__device__ __forceinline__ void yh_build(int32_t *keys, const YDesc &D, const int32_t *__restrict__ id,
                                         const int32_t *__restrict__ perm, const double *__restrict__ val, int64_t s0,
                                         int64_t s1, int64_t t1)
{
    for (int64_t e = s1 + threadIdx.x; e < t1; e += YH_THREADS) {   // t* entries first
        bool found;
        const int64_t slot = yh_insert<SMEM>(keys, D.lgb, walk_id(perm, id[e]), &found);
        D.vals[slot] = -(val[e] / (double)D.dt);
    }
    __syncthreads();
    for (int64_t e = s0 + threadIdx.x; e < s1; e += YH_THREADS) {
        bool found;
        const int64_t slot = yh_insert<SMEM>(keys, D.lgb, walk_id(perm, id[e]), &found);
        const double a = val[e] / (double)D.ds;
        D.vals[slot] = found ? a + D.vals[slot] : a - 0.0;
    }
}
// One query's hash table built in the shared-memory array sk (cap slots), then copied out.
__device__ __forceinline__ void yh_build_smem(int32_t *sk, int32_t i, const int64_t *__restrict__ segoff,
                                              const int32_t *__restrict__ id, const int32_t *__restrict__ perm,
                                              const double *__restrict__ val, const YDesc &D)
{
    const int64_t s0 = segoff[2 * i], s1 = segoff[2 * i + 1], t1 = segoff[2 * i + 2];
    const int cap = YB << D.lgb;
    for (int j = threadIdx.x; j < cap; j += YH_THREADS) sk[j] = -1;
    __syncthreads();
    yh_build<true>(sk, D, id, perm, val, s0, s1, t1);
    __syncthreads();
    int4 *dst = reinterpret_cast<int4 *>(D.keys);
    const int4 *src = reinterpret_cast<const int4 *>(sk);
    for (int j = threadIdx.x; j < cap / 4; j += YH_THREADS) dst[j] = src[j];
}
// Tables of <= YH_SMEM_SLOTS slots: one CTA per leaving query (static shared memory).
__global__ void __launch_bounds__(YH_THREADS) k_yhash(int32_t na, const int64_t *__restrict__ segoff,
                                                      const int32_t *__restrict__ id, const int32_t *__restrict__ perm,
                                                      const double *__restrict__ val, const YDesc *__restrict__ yd)
{
    __shared__ __align__(16) int32_t sk[YH_SMEM_SLOTS];
    const int32_t i = blockIdx.x;
    if (i >= na) return;
    const YDesc D = yd[i];
    if (D.mode != YT_HASH || (YB << D.lgb) > YH_SMEM_SLOTS) return;
    yh_build_smem(sk, i, segoff, id, perm, val, D);
}
// K5 over the support entries (frontier entry e: node id[e], value val[e], segment seg[e] = 2 i +
// side) of the leaving queries.  Tables are keyed by the walk kernel's node ids (walk_id: the
// degree-ordered renumbering of walk layout 4, else the ids themselves).  Every node v of
// U = supp(s*) u supp(t*) gets
//     y(v) = s*(v)/d(s) - t*(v)/d(t)          (a side v is not on contributes 0.0 / d = 0.0)
// in two passes, no searches and no floating-point atomics (Alg. 1 L7 with s = s*, t = t*):
//   pass 0: t* entries store -(t*(v)/d(t)) (= 0.0/d(s) - t*(v)/d(t) exactly);
//   pass 1: s* entries: y = s*(v)/d(s) + stored (= a - b exactly, IEEE a - b is a + (-b)) if v
//           has a t* entry, else s*(v)/d(s) - 0.0.
// hash: the slot of v by find-or-insert; rank: the slot at rank U + popc(U bits below v) (k_ybits:
// every entry's bit of v into its query's records; k_yrank: the ranks, and every value slot set to
// Y_UNSET, so pass 1 tells "v in supp t*" by the slot's content).
// Rank tables, bits: one thread per frontier entry; a warp ORs each run of equal (query, 32-id
// word) by a segmented shuffle scan and the run's first lane sets the bits with one 32-bit
// atomicOr (segments are sorted by node id: without renumbering a word's entries are consecutive,
// one atomic per word and warp).  The records are zeroed before.
// With wid != nullptr (walk layout 4) the same pass stores every leaving entry's walk id in wid, for
// the hash builds and the value passes.  YB_EPT entries per thread (stride blockDim.x), their
// loads staged level by level as in k_yinsert.
#ifndef YB_EPT
#define YB_EPT 2
#endif
__global__ void k_ybits(int64_t Fmax, const int64_t *__restrict__ dF, const int32_t *__restrict__ seg,
                        const int32_t *__restrict__ id, const int32_t *__restrict__ perm,
                        const YDesc *__restrict__ yd, int32_t *__restrict__ wid)
{
    const int64_t F = dF != nullptr ? min(Fmax, *dF) : Fmax;
    const int64_t e0 = (int64_t)blockIdx.x * blockDim.x * YB_EPT + threadIdx.x;
    const int lane = threadIdx.x & 31;
    int32_t g[YB_EPT], mode[YB_EPT], v[YB_EPT];
    uint4 *rec[YB_EPT];
#pragma unroll
    for (int k = 0; k < YB_EPT; k++) {
        const int64_t e = e0 + (int64_t)k * blockDim.x;
        g[k] = e < F ? seg[e] : -1;
    }
#pragma unroll
    for (int k = 0; k < YB_EPT; k++) {
        const int64_t e = e0 + (int64_t)k * blockDim.x;
        mode[k] = g[k] >= 0 ? yd[g[k] >> 1].mode : -1;
        if (mode[k] >= 0) {
            v[k] = walk_id(perm, id[e]);
            rec[k] = yd[g[k] >> 1].rec;
        }
    }
#pragma unroll
    for (int k = 0; k < YB_EPT; k++) {
        const int64_t e = e0 + (int64_t)k * blockDim.x;
        unsigned long long key = ~0ull;
        unsigned int bits = 0;
        unsigned int *dst = nullptr;
        if (mode[k] >= 0 && wid != nullptr) wid[e] = v[k];
        if (mode[k] == YT_RANK) {
            // 32-id word v >> 5 = word (v >> 5) mod 3 of record v / 96 (96 = 3 x 32)
            key = ((unsigned long long)(uint32_t)(g[k] >> 1) << 32) | (uint32_t)(v[k] >> 5);   // both sides: U bits
            bits = 1u << (v[k] & 31);
            dst = reinterpret_cast<unsigned int *>(rec[k] + rank_rec(v[k])) + ((uint32_t)(v[k] >> 5) % 3u);
        }
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const unsigned long long ok = __shfl_down_sync(0xffffffffu, key, d);
            const unsigned int ob = __shfl_down_sync(0xffffffffu, bits, d);
            if (lane + d < 32 && ok == key) bits |= ob;
        }
        const unsigned long long pk = __shfl_up_sync(0xffffffffu, key, 1);
        if (dst != nullptr && (lane == 0 || pk != key)) atomicOr(dst, bits);
    }
}

// YI_EPT entries per thread (stride blockDim.x), staged so that each level of the dependent loads
// (segment -> descriptor and walk id -> rank record -> value slot) is in flight for all of them at
// once; stores come last, after every load (the value slots of one pass are distinct: every y(v)
// has one writer per pass).
#ifndef YI_EPT
#define YI_EPT 2
#endif
__global__ void k_yinsert(int64_t Fmax, const int64_t *__restrict__ dF, const int32_t *__restrict__ seg,
                          const int32_t *__restrict__ id, const int32_t *__restrict__ perm,
                          const double *__restrict__ val, const YDesc *__restrict__ yd, int pass)
{
    const int64_t F = dF != nullptr ? min(Fmax, *dF) : Fmax;
    const int64_t e0 = (int64_t)blockIdx.x * blockDim.x * YI_EPT + threadIdx.x;
    const int want = pass == 0 ? 1 : 0;   // side of this pass: t* entries, then s* entries
    int32_t q[YI_EPT];   // leaving query index, or -1
#pragma unroll
    for (int k = 0; k < YI_EPT; k++) {
        const int64_t e = e0 + (int64_t)k * blockDim.x;
        const int32_t g = e < F ? seg[e] : -1;
        q[k] = g >= 0 && (g & 1) == want ? g >> 1 : -1;
    }
    int32_t mode[YI_EPT], v[YI_EPT];
    const uint4 *rec[YI_EPT];
#pragma unroll
    for (int k = 0; k < YI_EPT; k++) {
        const int64_t e = e0 + (int64_t)k * blockDim.x;
        mode[k] = q[k] >= 0 ? yd[q[k]].mode : -1;
        if (mode[k] == YT_HASH && (YB << yd[q[k]].lgb) <= YH_SMEM_SLOTS_DEV) mode[k] = -1;   // k_yhash
        if (mode[k] >= 0) {
            v[k] = walk_id(perm, id[e]);
            rec[k] = yd[q[k]].rec;
        }
    }
    uint4 r[YI_EPT];
#pragma unroll
    for (int k = 0; k < YI_EPT; k++)
        if (mode[k] == YT_RANK) r[k] = rec[k][rank_rec(v[k])];
    double *slot[YI_EPT];
    double y[YI_EPT];
#pragma unroll
    for (int k = 0; k < YI_EPT; k++) {
        if (mode[k] == YT_RANK) {
            slot[k] = yd[q[k]].vals + rank_index(r[k], v[k]);   // v is in U: its entry set the bit
            if (want == 0) y[k] = *slot[k];
        }
    }
#pragma unroll
    for (int k = 0; k < YI_EPT; k++) {
        if (mode[k] < 0) continue;
        const int64_t e = e0 + (int64_t)k * blockDim.x;
        const YDesc &D = yd[q[k]];
        const double x = val[e];
        if (mode[k] == YT_RANK) {
            if (want == 1) {
                *slot[k] = -(x / (double)D.dt);
            } else {
                const double a = x / (double)D.ds;   // Y_UNSET: v is not in supp t*
                *slot[k] = (unsigned long long)__double_as_longlong(y[k]) == Y_UNSET ? a - 0.0 : a + y[k];
            }
        } else {   // large hash tables (tables of <= YH_SMEM_SLOTS slots: k_yhash, shared memory)
            bool found;
            const int64_t hs = yh_insert<false>(D.keys, D.lgb, v[k], &found);
            if (want == 1) {
                D.vals[hs] = -(x / (double)D.dt);
            } else {
                const double a = x / (double)D.ds;
                D.vals[hs] = found ? a + D.vals[hs] : a - 0.0;
            }
        }
    }
}

// Ranks of the rank-bitmap tables: rank(record w) = popcount of all records before w, stored in the
// record's fourth word; and the value slots set to Y_UNSET for the value passes.  One CTA per
// leaving query (non-rank queries exit); YRANK_ITEMS consecutive records per thread per pass.
constexpr int YRANK_THREADS = 256;
constexpr int YRANK_ITEMS = 4;
__global__ void __launch_bounds__(YRANK_THREADS)
k_yrank(int32_t na, const YSizes *__restrict__ sz, const YDesc *__restrict__ yd)
{
    const int32_t i = blockIdx.x;
    if (i >= na || sz[i].r == 0) return;
    uint4 *recs = yd[i].rec;
    const int64_t R = sz[i].r;
    static_assert(YRANK_THREADS == SCAN_NT, "k_yrank uses the CTA scan of scan.cuh");
    __shared__ uint32_t sh[SCAN_NT / 32];
    uint32_t carry = 0;   // rank U
    for (int64_t base = 0; base < R; base += YRANK_THREADS * YRANK_ITEMS) {
        const int64_t w0 = base + (int64_t)threadIdx.x * YRANK_ITEMS;
        uint32_t c[YRANK_ITEMS], sum = 0;
#pragma unroll
        for (int j = 0; j < YRANK_ITEMS; j++) {
            const uint4 u = w0 + j < R ? recs[w0 + j] : make_uint4(0u, 0u, 0u, 0u);
            c[j] = __popc(u.x) + __popc(u.y) + __popc(u.z);
            sum += c[j];
        }
        uint32_t run, tot;
        cta_scan(sum, sh, ScanAdd<uint32_t>(), 0u, &run, &tot);
#pragma unroll
        for (int j = 0; j < YRANK_ITEMS; j++) {
            if (w0 + j < R) recs[w0 + j].w = carry + run;
            run += c[j];
        }
        carry += tot;
        __syncthreads();
    }
    unsigned long long *vals = reinterpret_cast<unsigned long long *>(yd[i].vals);
    for (uint32_t k = threadIdx.x; k < carry; k += YRANK_THREADS) vals[k] = Y_UNSET;
}

// ---------------------------------------------------------------------------- host side

// Phase 1 of K5 (stages.h): sizes and their scans, no host sync.
int ytable_plan(Ctx &c, int32_t na, const int32_t *act, const int32_t *cont, const int64_t *segoff,
                const int64_t **tot_h, const int64_t **tot_v, const int64_t **tot_r)
{
    Workspace &ws = c.ws;
    ENSURE(ws.ycap, sizeof(YSizes) * (na + 1), false);
    ENSURE(ws.yoff, sizeof(YSizes) * (na + 1), false);
    YSizes *sz = ws.ycap.as<YSizes>(), *incl = ws.yoff.as<YSizes>();
    const int64_t nrec = ((c.g->d_cblk ? c.g->dord_nv : c.g->n) + RANK_IDS - 1) / RANK_IDS;   // over the walk ids
    k_ycap<<<blocks_for(na, 256), 256, 0, c.st>>>(na, act, ws.qs.as<QState>(), cont, segoff, nrec, c.g->ytable_force,
                                                  c.g->rank_min_cap, c.g->rank_ratio, c.g->rank_max_bytes, sz);
    LAUNCHED(c.g);
    int rc = scan_op(c, sz, incl, (int64_t)na, YSizes{0, 0, 0}, YSizesPlus());   // the three size scans in one pass
    *tot_h = &incl[na - 1].h;
    *tot_v = &incl[na - 1].v;
    *tot_r = &incl[na - 1].r;
    return rc;
}

// Phase 2: allocate and fill the tables planned by ytable_plan (totals H, V, R read by the caller).
int ytable_build(Ctx &c, int32_t na, const int32_t *act, const int64_t *segoff, const int32_t *id, const double *val,
                 const int32_t *seg, int64_t Fmax, const int64_t *dF, int wave, int64_t H, int64_t V, int64_t R)
{
    NvtxRange nvtx_("geer/ytable");
    Workspace &ws = c.ws;
    const YSizes *sz = ws.ycap.as<YSizes>(), *incl = ws.yoff.as<YSizes>();
    const int32_t *perm = c.g->d_cblk ? c.g->d_perm : nullptr;   // keys in the walk kernel's ids
    if (V == 0) return ER_OK;
    if (c.g->profiling) {
        c.g->prof.ytable_slots += H;
        c.g->prof.yrank_records += R;
    }
    if ((int)ws.ychunk.size() <= wave) ws.ychunk.resize(wave + 1);
    DevBuf &yb = ws.ychunk[wave];
    auto up = [](size_t x) { return (x + 255) & ~(size_t)255; };   // 256-byte aligned regions
    const size_t o_rec = up(sizeof(double) * V), o_key = o_rec + up(sizeof(uint4) * R);
    const size_t ybytes = o_key + up(sizeof(int32_t) * H);
    if (ybytes > yb.cap) {   // the old buffer may still serve an earlier batch's AMC (AMC stream)
        CK(cudaStreamSynchronize(c.g->amc_stream));
        CK(cudaStreamSynchronize(c.st));
    }
    ENSURE(yb, ybytes, false);
    double *vals = yb.as<double>();
    uint4 *recs = reinterpret_cast<uint4 *>(yb.as<char>() + o_rec);
    int32_t *keys = reinterpret_cast<int32_t *>(yb.as<char>() + o_key);   // 16-byte buckets: aligned region
    if (H > 0 || R > 0) {   // (small hash tables are rewritten whole by k_yhash)
        k_yfill<<<blocks_for(std::max(H, R), 256), 256, 0, c.st>>>(H, keys, R, recs);
        LAUNCHED(c.g);
    }
    ENSURE(ws.ydesc, sizeof(YDesc) * (na + 1), false);
    YDesc *yd = ws.ydesc.as<YDesc>();
    k_yassign<<<blocks_for(na, 128), 128, 0, c.st>>>(na, act, sz, incl, keys, vals, recs,
                                                      ws.qs.as<QState>(), yd);
    LAUNCHED(c.g);
    // rank bits; under layout 4 the same pass maps every leaving entry to its walk id once, then the
    // builds run as without renumbering
    int32_t *wid = nullptr;
    if (perm != nullptr) {
        ENSURE(ws.ywid, sizeof(int32_t) * std::max<int64_t>(Fmax, 1), false);
        wid = ws.ywid.as<int32_t>();
    }
    if (R > 0 || wid != nullptr) {
        k_ybits<<<blocks_for((Fmax + YB_EPT - 1) / YB_EPT, 256), 256, 0, c.st>>>(Fmax, dF, seg, id, perm, yd, wid);
        LAUNCHED(c.g);
    }
    if (wid != nullptr) {
        id = wid;
        perm = nullptr;
    }
    if (H > 0) {
        k_yhash<<<na, YH_THREADS, 0, c.st>>>(na, segoff, id, perm, val, yd);
        LAUNCHED(c.g);
    }
    if (R > 0) {
        k_yrank<<<na, YRANK_THREADS, 0, c.st>>>(na, sz, yd);
        LAUNCHED(c.g);
    }
    for (int pass = 0; pass < 2; pass++) {   // rank tables and large hash tables: t* entries, then s*
        k_yinsert<<<blocks_for((Fmax + YI_EPT - 1) / YI_EPT, 256), 256, 0, c.st>>>(Fmax, dF, seg, id, perm, val, yd,
                                                                                     pass);
        LAUNCHED(c.g);
    }
    return ER_OK;
}

int build_ytables(Ctx &c, int32_t na, const int32_t *act, const int32_t *cont, const int64_t *segoff,
                  const int32_t *id, const double *val, const int32_t *seg, int64_t Fmax, const int64_t *dF,
                  int wave)
{
    const int64_t *th, *tv, *tr;
    int rc = ytable_plan(c, na, act, cont, segoff, &th, &tv, &tr);
    if (!rc) rc = read_scalars(c, {th, tv, tr});
    if (rc) return rc;
    const int64_t H = c.hp[0], V = c.hp[1], R = c.hp[2];
    return ytable_build(c, na, act, segoff, id, val, seg, Fmax, dF, wave, H, V, R);
}

}  // namespace geer
