// ytable.cu -- K5: the per-query y-tables of Alg. 1 L7 built from the SMM frontier of the
// queries that leave the head, and their host-side planning (one scalar read per wave).
//
// Every y(v) is written exactly once by the entry that owns v (no floating-point atomics); the
// tables are read by the walk kernel (walks.cu).

#include "stages.h"

namespace geer {

// y-tables (K5): y(v) = s*(v)/d(s) - t*(v)/d(t) on U = supp(s*) u supp(t*) for each query that
// leaves the SMM head for AMC in this wave (Alg. 1 L7 with s = s*, t = t*).  Two layouts,
// chosen per query by footprint:
//  * hash (YT_HASH): open addressing, 8 int32 keys per 32-byte bucket, buckets probed linearly;
//    capacity = next power of two >= 2 (|supp s*| + |supp t*|) (load <= 1/2), >= one bucket;
//    values fp64 by slot.  Tables of <= WALK_KEY_SLOTS keys are staged whole in the walk
//    kernel's shared memory.
//  * rank bitmap (YT_RANK): one 16-byte record {U bits (64); rank U; rank T} per 64 node ids
//    (bit v of U; ranks = |U| and |supp t*| below the record), values fp64 by rank: y(v) is at
//    vals[rank U + popc(U bits below v)].  Exact membership in one 16-byte load, no probing;
//    used for tables too large to stage whose records take less than twice the hash layout's
//    12 B/slot (keys + values).
// Per leaving query i: hslots[i] hash slots, vslots[i] value slots, rrecs[i] rank records.
__global__ void k_ycap(int32_t na, const int32_t *__restrict__ act, const QState *__restrict__ qs,
                       const int32_t *__restrict__ cont, const int64_t *__restrict__ segoff, int64_t nrec,
                       int force, int64_t *__restrict__ hslots, int64_t *__restrict__ vslots,
                       int64_t *__restrict__ rrecs)
{
    const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= na) return;
    int64_t h = 0, v = 0, r = 0;
    if ((cont == nullptr || !cont[i]) && qs[act[i]].phase == PH_AMC) {
        const int64_t len = segoff[2 * i + 2] - segoff[2 * i];   // |supp s*| + |supp t*| >= |U|
        int64_t cap = YB;
        while (cap < 2 * len) cap <<= 1;
        // rank when the table cannot be staged and the records take at most twice the hash footprint:
        // rank lookups are pipelined off the walk chain, global hash probes are not
        const bool rank = force == 2 || (force == 0 && cap > WALK_KEY_SLOTS && 16 * nrec < 24 * cap);
        if (rank) {
            r = nrec;
            v = len;
        } else {
            h = cap;
            v = cap;
        }
    }
    hslots[i] = h;
    vslots[i] = v;
    rrecs[i] = r;
}

__global__ void k_yassign(int32_t na, const int32_t *__restrict__ act, const int64_t *__restrict__ hslots,
                          const int64_t *__restrict__ hincl, const int64_t *__restrict__ vslots,
                          const int64_t *__restrict__ vincl, const int64_t *__restrict__ rrecs,
                          const int64_t *__restrict__ rincl, const int32_t *kbase, const double *vbase,
                          const uint4 *rbase, const uint4 *abase, QState *__restrict__ qs)
{
    const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= na || vslots[i] == 0) return;
    QState &Q = qs[act[i]];
    Q.yvals = vbase + (vincl[i] - vslots[i]);
    if (rrecs[i] > 0) {
        Q.ymode = YT_RANK;
        Q.yrec = rbase + (rincl[i] - rrecs[i]);
        Q.yaux = abase + (rincl[i] - rrecs[i]);
        Q.ykeys = nullptr;
        Q.ylog2 = 0;
    } else {
        const int64_t cap = hslots[i];
        Q.ymode = YT_HASH;
        Q.ykeys = kbase + (hincl[i] - cap);
        Q.yrec = nullptr;
        int lg = 0;
        while ((1ll << lg) < cap) lg++;
        Q.ylog2 = lg;
    }
}

__global__ void k_yfill(int64_t H, int32_t *__restrict__ keys, int64_t R, uint4 *__restrict__ aux)
{
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j < H) keys[j] = -1;
    if (j < R) aux[j] = make_uint4(0u, 0u, 0u, 0u);   // the records themselves are written by k_yrank
}

// Hash find-or-insert of v; returns its slot.
__device__ __forceinline__ int64_t hash_insert(int32_t *keys, int lgb, int32_t v)
{
    const uint32_t bmask = (1u << lgb) - 1u;
    uint32_t bk = ybucket(v, lgb);
    while (true) {
        const int4 *bp = reinterpret_cast<const int4 *>(keys + bk * YB);
        int4 A, B;
        asm volatile("ld.volatile.global.v4.s32 {%0,%1,%2,%3}, [%4];" : "=r"(A.x), "=r"(A.y), "=r"(A.z), "=r"(A.w) : "l"(bp));
        asm volatile("ld.volatile.global.v4.s32 {%0,%1,%2,%3}, [%4];" : "=r"(B.x), "=r"(B.y), "=r"(B.z), "=r"(B.w) : "l"(bp + 1));
        const int32_t kk[YB] = {A.x, A.y, A.z, A.w, B.x, B.y, B.z, B.w};
        for (int j = 0; j < YB; j++) {
            const uint32_t slot = bk * YB + j;
            int32_t k = kk[j];
            if (k == -1) k = atomicCAS(&keys[slot], -1, v);
            if (k == -1 || k == v) return slot;
        }
        bk = (bk + 1) & bmask;
    }
}

// Position of node v in the sorted id range [lo, hi), or -1.
__device__ __forceinline__ int64_t find_sorted(const int32_t *__restrict__ id, int64_t lo, int64_t hi, int32_t v)
{
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        const int32_t x = id[mid];
        if (x == v) return mid;
        if (x < v) lo = mid + 1;
        else hi = mid;
    }
    return -1;
}

// K5 over the support entries (frontier entry e: node id[e], value val[e], segment seg[e] =
// 2 i + side; each segment sorted by node id) of the leaving queries.  Every node v of
// U = supp(s*) u supp(t*) has one OWNER entry (its side-0 entry, else its side-1 entry), which
// finds v's entry on the other side and writes
//     y(v) = s*(v)/d(s) - t*(v)/d(t)          (a side v is not on contributes 0.0 / d = 0.0)
// exactly once (Alg. 1 L7 with s = s*, t = t*).
//   pass 0: hash: owners find the other side by binary search, insert v (CAS on the key slot)
//           and write y;  rank: every entry sets its side's bit of v
//   (k_yrank between the passes: union bits, rank of U and rank of the t* side per record)
//   pass 1: rank: owners find v's t* entry by rank (segment start + rank T + popc) and write y
//           at rank U + popc(U bits below v)
__global__ void k_yinsert(int64_t Fmax, const int64_t *__restrict__ dF, const int32_t *__restrict__ seg,
                          const int32_t *__restrict__ id, const double *__restrict__ val,
                          const int64_t *__restrict__ segoff, const int32_t *__restrict__ act,
                          const int64_t *__restrict__ vslots, const QState *__restrict__ qs, int pass)
{
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= Fmax || (dF != nullptr && e >= *dF)) return;
    const int32_t g = seg[e];
    const int32_t i = g >> 1;
    if (vslots[i] == 0) return;
    const int side = g & 1;
    const QState &Q = qs[act[i]];
    const int32_t v = id[e];
    if (Q.ymode == YT_RANK) {
        // membership bits per side in the build-time aux records {S bits, T bits}; k_yrank turns
        // them into the walk records {U bits, rank U, rank T}; no searches
        uint4 *aux = const_cast<uint4 *>(Q.yaux);
        const uint64_t bit = 1ull << (v & 63);
        if (pass == 0) {
            atomicOr(reinterpret_cast<unsigned long long *>(aux + (v >> 6)) + side, bit);
            return;
        }
        const uint4 a = aux[v >> 6];
        const uint64_t sbits = ((uint64_t)a.y << 32) | a.x, tbits = ((uint64_t)a.w << 32) | a.z;
        if (side == 1 && (sbits & bit)) return;   // the side-0 entry owns v
        const uint4 r = Q.yrec[v >> 6];
        const uint64_t below = bit - 1ull;
        double xt = 0.0;
        if (side == 1) xt = val[e];
        else if (tbits & bit) xt = val[segoff[g ^ 1] + r.w + __popcll(tbits & below)];   // v's t* entry
        const double xs = side == 0 ? val[e] : 0.0;
        const double y = xs / (double)Q.ds - xt / (double)Q.dt;
        const uint64_t ubits = ((uint64_t)r.y << 32) | r.x;
        const_cast<double *>(Q.yvals)[r.z + __popcll(ubits & below)] = y;
        return;
    }
    if (pass != 0) return;
    // owner test and the other side's value
    const int64_t other = find_sorted(id, segoff[g ^ 1], segoff[(g ^ 1) + 1], v);
    if (side == 1 && other >= 0) return;   // the side-0 entry owns v
    const double xs = side == 0 ? val[e] : 0.0;
    const double xt = side == 1 ? val[e] : (other >= 0 ? val[other] : 0.0);
    const double y = xs / (double)Q.ds - xt / (double)Q.dt;
    double *vals = const_cast<double *>(Q.yvals);
    if (Q.ymode == YT_HASH) vals[hash_insert(const_cast<int32_t *>(Q.ykeys), Q.ylog2 - YB_LOG, v)] = y;
    else vals[rank_index(Q.yrec[v >> 6], v)] = y;
}

// Ranks of the rank-bitmap tables: rank(record w) = popcount of all records before w.  One CTA
// per leaving query (non-rank queries exit).
constexpr int YRANK_THREADS = 256;
__global__ void __launch_bounds__(YRANK_THREADS)
k_yrank(int32_t na, const int32_t *__restrict__ act, const int64_t *__restrict__ rrecs, QState *__restrict__ qs)
{
    const int32_t i = blockIdx.x;
    if (i >= na || rrecs[i] == 0) return;
    uint4 *recs = const_cast<uint4 *>(qs[act[i]].yrec);
    const uint4 *aux = qs[act[i]].yaux;
    const int64_t R = rrecs[i];
    typedef cub::BlockScan<unsigned long long, YRANK_THREADS> Scan;
    __shared__ typename Scan::TempStorage tmp;
    unsigned long long carry = 0;   // (rank U << 32) | rank T
    for (int64_t base = 0; base < R; base += YRANK_THREADS) {
        const int64_t w = base + threadIdx.x;
        const uint4 a = w < R ? aux[w] : make_uint4(0u, 0u, 0u, 0u);
        const uint32_t ux = a.x | a.z, uy = a.y | a.w;
        const unsigned long long c = ((unsigned long long)(__popc(ux) + __popc(uy)) << 32) |
                                     (unsigned long long)(__popc(a.z) + __popc(a.w));
        unsigned long long excl, tot;
        Scan(tmp).ExclusiveSum(c, excl, tot);
        if (w < R) {
            const unsigned long long rk = carry + excl;
            recs[w] = make_uint4(ux, uy, (uint32_t)(rk >> 32), (uint32_t)rk);
        }
        carry += tot;
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------- host side

// Phase 1 of K5 (stages.h): sizes and their scans, no host sync.
int ytable_plan(Ctx &c, int32_t na, const int32_t *act, const int32_t *cont, const int64_t *segoff,
                const int64_t **tot_h, const int64_t **tot_v, const int64_t **tot_r)
{
    Workspace &ws = c.ws;
    ENSURE(ws.ycap, sizeof(int64_t) * 3 * (na + 1), false);
    ENSURE(ws.yoff, sizeof(int64_t) * 3 * (na + 1), false);
    int64_t *hs = ws.ycap.as<int64_t>(), *vs = hs + (na + 1), *rs = vs + (na + 1);
    int64_t *hi = ws.yoff.as<int64_t>(), *vi = hi + (na + 1), *ri = vi + (na + 1);
    const int64_t nrec = (c.g->n + 63) / 64;
    k_ycap<<<blocks_for(na, 256), 256, 0, c.st>>>(na, act, ws.qs.as<QState>(), cont, segoff, nrec, c.g->ytable_force,
                                                  hs, vs, rs);
    LAUNCHED(c.g);
    int rc = scan_incl(c, hs, hi, na);
    if (!rc) rc = scan_incl(c, vs, vi, na);
    if (!rc) rc = scan_incl(c, rs, ri, na);
    *tot_h = hi + (na - 1);
    *tot_v = vi + (na - 1);
    *tot_r = ri + (na - 1);
    return rc;
}

// Phase 2: allocate and fill the tables planned by ytable_plan (totals H, V, R read by the caller).
int ytable_build(Ctx &c, int32_t na, const int32_t *act, const int64_t *segoff, const int32_t *id, const double *val,
                 const int32_t *seg, int64_t Fmax, const int64_t *dF, int wave, int64_t H, int64_t V, int64_t R)
{
    Workspace &ws = c.ws;
    int64_t *hs = ws.ycap.as<int64_t>(), *vs = hs + (na + 1), *rs = vs + (na + 1);
    int64_t *hi = ws.yoff.as<int64_t>(), *vi = hi + (na + 1), *ri = vi + (na + 1);
    if (V == 0) return ER_OK;
    if (c.g->profiling) {
        c.g->prof.ytable_slots += H;
        c.g->prof.yrank_records += R;
    }
    if ((int)ws.ychunk.size() <= wave) ws.ychunk.resize(wave + 1);
    DevBuf &yb = ws.ychunk[wave];
    auto up = [](size_t x) { return (x + 255) & ~(size_t)255; };   // 256-byte aligned regions
    const size_t o_rec = up(sizeof(double) * V), o_aux = o_rec + up(sizeof(uint4) * R);
    const size_t o_key = o_aux + up(sizeof(uint4) * R);
    const size_t ybytes = o_key + up(sizeof(int32_t) * H);
    if (ybytes > yb.cap) CK(cudaDeviceSynchronize());   // the old buffer may still serve an earlier AMC
    ENSURE(yb, ybytes, false);
    double *vals = yb.as<double>();
    uint4 *recs = reinterpret_cast<uint4 *>(yb.as<char>() + o_rec);
    uint4 *aux = reinterpret_cast<uint4 *>(yb.as<char>() + o_aux);      // build-time {S bits, T bits}
    int32_t *keys = reinterpret_cast<int32_t *>(yb.as<char>() + o_key);   // buckets need 32-byte alignment
    k_yfill<<<blocks_for(std::max(H, R), 256), 256, 0, c.st>>>(H, keys, R, aux);
    LAUNCHED(c.g);
    k_yassign<<<blocks_for(na, 128), 128, 0, c.st>>>(na, act, hs, hi, vs, vi, rs, ri, keys, vals, recs, aux,
                                                      ws.qs.as<QState>());
    LAUNCHED(c.g);
    for (int pass = 0; pass < 2; pass++) {
        if (pass == 1) {
            if (R == 0) break;
            k_yrank<<<na, YRANK_THREADS, 0, c.st>>>(na, act, rs, ws.qs.as<QState>());
            LAUNCHED(c.g);
        }
        k_yinsert<<<blocks_for(Fmax, 256), 256, 0, c.st>>>(Fmax, dF, seg, id, val, segoff, act, vs, ws.qs.as<QState>(),
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
