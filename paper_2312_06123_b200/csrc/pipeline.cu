// pipeline.cu -- the GEER query pipeline on one B200 (sm_100a): K1-K4, K8 and the batch driver;
// K5 lives in ytable.cu, K6/K7 in walks.cu.
//
// Per batch of k queries:
//   K1 k_setup            ell (Eq. 6), r_b^0, phase per query            Alg. 3 L1-L4
//   SMM waves, each:      s* <- P s*, t* <- P t* for every active query   Alg. 3 L6-L8
//     wave 1              k_first_wave: closed form x'(u) = 1/d(u) on N(s) (sorted rows)
//     K2/K3 push          smm_push.cu: bucketed push (u, e) -> per-bucket radix sort in shared
//                         memory -> ordered sequential sum per (segment, u), / d(u); K4 stats
//                         (vol, top-2, x(s), x(t)) per bucket, merged per segment
//     or dense pull       dense.cu + K9 exact, chosen per wave by a cost model (R25)
//        k_decide         r_b += term; psi -> eta* -> eta0 -> h; switch   Alg. 3 L7, L9
//     K5 k_yinsert        y = s*/d_s - t*/d_t into a per-query table      Alg. 1 L7
//        (+ k_yrank)      (hash, or rank bitmap for large supports)
//        compaction       frontier + active list of continuing queries
//   AMC batches b = 0..tau-1 (after the head, or per SMM wave on a second stream):
//     K6 k_walks          thread = walk pair(s), flattened over queries; Philox (q,b,side,k,step)  Alg. 1 L5-L9
//     K7 k_amc_reduce     Z, sigma^2, Bernstein f, stop or double         Alg. 1 L11-L14
//   K8 k_finalize         r' = r_f + r_b                                  Alg. 3 L11
//
// Everything is deterministic: no floating-point atomics, fixed reduction orders.

#include <array>
#include <cmath>
#include <cstring>

#include "geer_device.cuh"
#include <atomic>

#include "stages.h"

#include <vector>

namespace geer {

// ============================================================================ kernels

// K1: per-query setup.
__global__ void k_setup(int64_t k, const int32_t *__restrict__ pairs, const int64_t *__restrict__ ids,
                        const int64_t *__restrict__ off, BatchParams P, QState *__restrict__ qs)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= k) return;
    QState Q;
    memset(&Q, 0, sizeof(Q));
    const int32_t s = pairs[2 * i], t = pairs[2 * i + 1];
    Q.s = s;
    Q.t = t;
    Q.gq = (uint32_t)(ids ? ids[i] : P.qbase + i);
    Q.ds = (int32_t)(off[s + 1] - off[s]);
    Q.dt = (int32_t)(off[t + 1] - off[t]);
    Q.phase = PH_DONE;
    if (s != t) {
        const double dsf = (double)Q.ds, dtf = (double)Q.dt;
        // Eq. 6 or Eq. 5; natural log (R2); clamp at 0 (R3).
        double arg;
        if (P.ell_variant == 1) arg = 4.0 / (P.eps - P.eps * P.lambda);
        else arg = (2.0 / dsf + 2.0 / dtf) / (P.eps * (1.0 - P.lambda));
        const double x = log(arg) / P.log_inv_lambda - 1.0;
        double c = ceil(x);
        if (c < 0.0) c = 0.0;
        const int64_t ell = (int64_t)c;
        if (x > 0.0 && near_int(x)) Q.st.tie_flags |= 1u;
        Q.st.ell = (int32_t)ell;
        // Alg. 3 L4 with s* = e_s, t* = e_t.
        const double xs_s = 1.0, xt_t = 1.0, xs_t = 0.0, xt_s = 0.0;
        Q.st.r_b = xs_s / dsf + xt_t / dtf - xs_t / dsf - xt_s / dtf;
        if (ell > 0) {
            if (P.force_ell_b == 0) {
                // AMC alone (Thm 3.4 setting): s = e_s, t = e_t, lf = ell.
                const double psi = psi_eq10(ell, 1.0, 0.0, 1.0, 0.0, dsf, dtf);
                const double es = 2.0 * psi * psi * P.L_eta / (P.eps * P.eps);
                double e0 = ceil(es / (double)(1u << (P.tau - 1)));
                if (e0 < 1.0) e0 = 1.0;
                Q.st.ell_f = (int32_t)ell;
                Q.st.psi = psi;
                Q.st.eta0 = (int64_t)e0;
                Q.phase = PH_AMC;
            } else {
                Q.phase = PH_SMM;
            }
        }
    }
    qs[i] = Q;
}

__global__ void k_flag_phase(int64_t k, const QState *__restrict__ qs, int32_t phase, int32_t *__restrict__ flags,
                             int32_t *__restrict__ ids)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= k) return;
    flags[i] = qs[i].phase == phase ? 1 : 0;
    ids[i] = (int32_t)i;
}

// Initial frontier of an active list: segment 2i = {(s, 1.0)}, 2i+1 = {(t, 1.0)} (Alg. 3 L3).
__global__ void k_init_frontier(int32_t na, const int32_t *__restrict__ act, const QState *__restrict__ qs,
                                int32_t *__restrict__ id, double *__restrict__ val, int32_t *__restrict__ seg,
                                int64_t *__restrict__ segoff)
{
    const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < na) {
        const QState &Q = qs[act[i]];
        id[2 * i] = Q.s;
        id[2 * i + 1] = Q.t;
        val[2 * i] = 1.0;
        val[2 * i + 1] = 1.0;
        seg[2 * i] = 2 * i;
        seg[2 * i + 1] = 2 * i + 1;
    }
    if (i <= 2 * na) segoff[i] = i;
}

// Degree of every frontier entry (emission count of the push).
__global__ void k_ent_deg(int64_t F, const int32_t *__restrict__ id, const int64_t *__restrict__ off,
                          int64_t *__restrict__ deg)
{
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= F) return;
    const int32_t v = id[e];
    deg[e] = off[v + 1] - off[v];
}


// Pair offset of the first pair of each active query's segments (wave splitting: chunks of
// whole queries): pe[i] = ent_off[fr_off[2 i]], i = 0..na.
__global__ void k_query_pairs(int32_t na, const int64_t *__restrict__ fr_off, const int64_t *__restrict__ ent_off,
                              int64_t *__restrict__ pe)
{
    const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i <= na) pe[i] = ent_off[fr_off[2 * i]];
}

// First lane of each run of equal g (lanes sorted by g).
__device__ __forceinline__ bool warp_seg_head(int32_t g)
{
    const int32_t pg = __shfl_up_sync(0xffffffffu, g, 1);
    return (threadIdx.x & 31) == 0 || pg != g;
}

// Two segmented reductions at once (a with opA, b with opB; integer + / max only, so the result
// does not depend on the grouping) over lanes sorted by g.  Returns true on the lane holding a
// run's totals (its first lane).  Fast path when the whole warp is one run (the common case:
// segments hold hundreds to millions of entries).
template <class OpA, class OpB>
__device__ __forceinline__ bool warp_seg_reduce2(unsigned long long &a, unsigned long long &b, int32_t g, OpA opA,
                                                 OpB opB)
{
    const unsigned full = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    if (__all_sync(full, g == __shfl_sync(full, g, 0))) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            a = opA(a, __shfl_xor_sync(full, a, o));
            b = opB(b, __shfl_xor_sync(full, b, o));
        }
        return lane == 0;
    }
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long oa = __shfl_down_sync(full, a, o);
        const unsigned long long ob = __shfl_down_sync(full, b, o);
        const int32_t og = __shfl_down_sync(full, g, o);
        if (lane + o < 32 && og == g) {
            a = opA(a, oa);
            b = opB(b, ob);
        }
    }
    return warp_seg_head(g);
}

struct OpAdd {
    __device__ unsigned long long operator()(unsigned long long x, unsigned long long y) const { return x + y; }
};
struct OpMax {
    __device__ unsigned long long operator()(unsigned long long x, unsigned long long y) const { return x > y ? x : y; }
};

// CTA-level step on top of warp_seg_reduce2 for 256-thread CTAs: when all eight warps are single
// runs of ONE segment (hub rows span thousands of warps, all aiming their atomics at one SegStat),
// the warp totals are combined in shared memory and thread 0 alone holds the CTA totals.  Returns
// true on the threads that must publish (a, b): thread 0 in the combined case, the run heads
// otherwise.  Integer + / max only: the grouping cannot change the result.  One block-uniform call per
// kernel (k_first_wave: 9.5 -> 6.9 ms on the Friendster-shaped shard; in k_seg_max2's grid-stride loop
// the two barriers per round cost more than the atomics saved, +30 %, so it keeps the warp form).
template <class OpA, class OpB>
__device__ __forceinline__ bool cta_seg_reduce2(unsigned long long &a, unsigned long long &b, int32_t g, OpA opA,
                                                OpB opB)
{
    __shared__ unsigned long long sa[8], sb[8];
    __shared__ int32_t sg[8];
    const unsigned full = 0xffffffffu;
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const bool uni = __all_sync(full, g == __shfl_sync(full, g, 0));
    const bool head = warp_seg_reduce2(a, b, g, opA, opB);
    if (lane == 0) {
        sg[w] = (uni && g != 0x7fffffff) ? g : -1 - w;
        sa[w] = a;
        sb[w] = b;
    }
    __syncthreads();
    bool one = sg[0] >= 0;
#pragma unroll
    for (int i = 1; i < 8; i++) one = one && sg[i] == sg[0];
    if (!one) return head;
    if (threadIdx.x == 0) {
#pragma unroll
        for (int i = 1; i < 8; i++) {
            a = opA(a, sa[i]);
            b = opB(b, sb[i]);
        }
    }
    return threadIdx.x == 0;
}

// K2/K3 for the first SMM iteration when every adjacency row is sorted: from s* = e_s the
// iterate is s*(u) = (0.0 + 1.0)/d(u) on N(s) (one contribution per u), already in ascending u
// order, so no push/sort is needed.  Same statistics as k_run_reduce.
// u and d(u) come from the walk graph's arc records when it has them (one sequential read per
// entry along the row of s) instead of cols + a random node-record load.
__global__ void k_first_wave(int64_t E, int32_t nseg, const int64_t *__restrict__ ent_off,
                             const int32_t *__restrict__ fr_id, const int64_t *__restrict__ off,
                             const uint2 *__restrict__ rec, const int32_t *__restrict__ cols,
                             const uint4 *__restrict__ arcs, const unsigned long long *__restrict__ parcs, PackSpec pk,
                             const int32_t *__restrict__ act, const QState *__restrict__ qs, int32_t *__restrict__ nid,
                             double *__restrict__ nval, int32_t *__restrict__ nseg_out, SegStat *__restrict__ ss,
                             int64_t *__restrict__ dU)
{
    const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const bool live = p < E;
    int32_t g = 0x7fffffff;
    unsigned long long deg = 0, bits = 0;
    // segment of the warp's first entry: 32-way search by the whole warp (all lanes probe, the
    // range shrinks 32-fold per round: 4 rounds for 2.5e5 segments instead of 18 dependent loads
    // per thread), then every lane steps forward to its own (segments have >= 1 entry)
    int32_t lo = 0, hi = nseg;   // ent_off[lo] <= p0 < ent_off[hi]
    {
        const int lane = threadIdx.x & 31;
        const int64_t p0 = p - lane;
        if (p0 < E) {
            while (hi - lo > 1) {
                const int32_t step = (hi - lo + 31) >> 5;
                const int64_t q = (int64_t)lo + (int64_t)(lane + 1) * step;
                const bool le = q < hi && ent_off[q] <= p0;   // true for a prefix of the lanes
                const int c = __popc(__ballot_sync(0xffffffffu, le));
                lo += c * step;
                hi = min(hi, lo + step);
            }
        }
    }
    if (live) {
        while (ent_off[lo + 1] <= p) lo++;
        g = lo;
        const int32_t v = fr_id[g];
        const int64_t a = off[v] + (p - ent_off[g]);
        int32_t u;
        int64_t d;
        if (parcs) {
            const uint4 r = pk.unpack(__ldg(parcs + a));
            u = (int32_t)r.x;
            d = (int64_t)r.z;
        } else if (arcs) {
            const uint4 r = __ldg(arcs + a);
            u = (int32_t)r.x;
            d = (int64_t)r.z;
        } else {
            u = cols[a];
            d = (int64_t)__ldg(rec + u).y;   // node record {offset, degree}
        }
        const double sum = 0.0 + 1.0;
        const double x = sum / (double)d;
        nid[p] = u;
        nval[p] = x;
        nseg_out[p] = g;
        deg = (unsigned long long)d;
        bits = (unsigned long long)__double_as_longlong(x);
        const QState &Q = qs[act[g >> 1]];
        if (u == Q.s) ss[g].at_s = x;
        if (u == Q.t) ss[g].at_t = x;
        if (p == 0) *dU = E;
    }
    if (cta_seg_reduce2(deg, bits, g, OpAdd(), OpMax()) && live) {
        atomicAdd(reinterpret_cast<unsigned long long *>(&ss[g].vol), deg);
        atomicMax(reinterpret_cast<unsigned long long *>(&ss[g].max1), bits);
    }
}

// K4b: max2 of each segment = max1 if max1 occurs twice, else the largest entry below max1 (R5).
__global__ void k_seg_max2(int64_t Fmax, const int64_t *__restrict__ dF, const int32_t *__restrict__ seg,
                           const double *__restrict__ val, SegStat *__restrict__ ss)
{
    const int64_t F = min(Fmax, *dF);   // grid-stride, block-uniform bound (as k_run_reduce)
    for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < F; base += (int64_t)gridDim.x * blockDim.x) {
        const int64_t e = base + threadIdx.x;
        const bool live = e < F;
        int32_t g = 0x7fffffff;
        unsigned long long below = 0, eq = 0;
        if (live) {
            g = seg[e];
            const unsigned long long b = (unsigned long long)__double_as_longlong(val[e]);
            const unsigned long long m1 = *reinterpret_cast<const unsigned long long *>(&ss[g].max1);
            if (b < m1) below = b;
            else eq = 1;
        }
        if (warp_seg_reduce2(below, eq, g, OpMax(), OpAdd()) && live) {
            if (below) atomicMax(reinterpret_cast<unsigned long long *>(&ss[g].max2), below);
            if (eq) atomicAdd(&ss[g].n_max1, eq);
        }
    }
}

// Segment offsets of the (sorted) next frontier: segoff[g] = lower_bound(seg, g).
__global__ void k_seg_off(int32_t nseg, const int64_t *__restrict__ dU, const int32_t *__restrict__ seg,
                          int64_t *__restrict__ segoff)
{
    const int32_t g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g > nseg) return;
    const int64_t U = *dU;
    int64_t lo = 0, hi = U;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (seg[mid] < g) lo = mid + 1;
        else hi = mid;
    }
    segoff[g] = lo;
}

// Alg. 3 L7-L9 for every active query: r_b increment, Eq. 10 -> Eq. 9 -> eta0 -> h, Eq. 15.
__global__ void k_decide(int32_t na, const int32_t *__restrict__ act, const SegStat *__restrict__ ss, BatchParams P,
                         QState *__restrict__ qs, int32_t *__restrict__ cont)
{
    const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= na) return;
    QState &Q = qs[act[i]];
    SegStat S = ss[2 * i], T = ss[2 * i + 1];
    if (S.n_max1 >= 2) S.max2 = S.max1;   // R5: a repeated maximum is also the second largest
    if (T.n_max1 >= 2) T.max2 = T.max1;
    const double dsf = (double)Q.ds, dtf = (double)Q.dt;
    const double term = S.at_s / dsf + T.at_t / dtf - S.at_t / dsf - T.at_s / dtf;
    Q.st.r_b = Q.st.r_b + term;
    const int32_t lb = Q.st.ell_b;
    if (lb < 8) Q.st.rb_terms[lb] = term;
    const int32_t ell_b = lb + 1;
    Q.st.ell_b = ell_b;
    const int64_t ell = Q.st.ell;
    const int64_t vol = S.vol + T.vol;
    const double psi = psi_eq10(ell - ell_b, S.max1, S.max2, T.max1, T.max2, dsf, dtf);
    const double es = 2.0 * psi * psi * P.L_eta / (P.eps * P.eps);
    const double ratio = es / (double)(1u << (P.tau - 1));
    double e0 = ceil(ratio);
    if (e0 < 1.0) e0 = 1.0;
    if (ell - ell_b > 0 && near_int(ratio)) Q.st.tie_flags |= 2u;
    const int64_t eta0 = (int64_t)e0;
    const int64_t h = (((int64_t)1 << P.tau) - 1) * eta0;
    Q.st.vol_last = vol;
    Q.st.h_last = h;
    const int64_t maxit = P.force_ell_b >= 0 ? (P.force_ell_b < ell ? P.force_ell_b : ell) : ell;
    const bool over = P.switch_ratio == 1.0 ? vol > h : (double)vol > P.switch_ratio * (double)h;   // Eq. 15
    const bool go = ell_b < maxit && !(P.force_ell_b < 0 && over);
    cont[i] = go ? 1 : 0;
    if (!go) {
        const int64_t lf = ell - ell_b;
        Q.st.ell_f = (int32_t)lf;
        if (lf > 0) {
            Q.st.psi = psi;
            Q.st.eta0 = eta0;
            Q.phase = PH_AMC;
        } else {
            Q.phase = PH_DONE;
        }
    }
}

// Continuing segments: new lengths (for the compaction scan).
__global__ void k_seglen(int32_t nseg, const int32_t *__restrict__ cont, const int64_t *__restrict__ segoff,
                         int64_t *__restrict__ len)
{
    const int32_t g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= nseg) return;
    len[g] = cont[g >> 1] ? segoff[g + 1] - segoff[g] : 0;
}

__global__ void k_compact_entries(int64_t Fmax, const int64_t *__restrict__ dF, const int32_t *__restrict__ seg,
                                  const int32_t *__restrict__ id, const double *__restrict__ val,
                                  const int64_t *__restrict__ segoff, const int32_t *__restrict__ cont,
                                  const int32_t *__restrict__ newidx_incl, const int64_t *__restrict__ segnew_incl,
                                  const int64_t *__restrict__ seglen, int32_t *__restrict__ oid,
                                  double *__restrict__ oval, int32_t *__restrict__ oseg)
{
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= Fmax || e >= *dF) return;
    const int32_t g = seg[e];
    const int32_t i = g >> 1;
    if (!cont[i]) return;
    const int64_t dst = segnew_incl[g] - seglen[g] + (e - segoff[g]);
    oid[dst] = id[e];
    oval[dst] = val[e];
    oseg[dst] = 2 * (newidx_incl[i] - 1) + (g & 1);
}

__global__ void k_compact_lists(int32_t na, const int32_t *__restrict__ cont, const int32_t *__restrict__ newidx_incl,
                                const int32_t *__restrict__ act, const int64_t *__restrict__ segnew_incl,
                                const int64_t *__restrict__ seglen, int32_t *__restrict__ act2,
                                int64_t *__restrict__ segoff2)
{
    const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= na) return;
    if (cont[i]) {
        const int32_t j = newidx_incl[i] - 1;
        act2[j] = act[i];
        segoff2[2 * j] = segnew_incl[2 * i] - seglen[2 * i];
        segoff2[2 * j + 1] = segnew_incl[2 * i + 1] - seglen[2 * i + 1];
    }
    if (i == na - 1) segoff2[2 * newidx_incl[i]] = segnew_incl[2 * na - 1];
}


// Queries of an active list that leave the SMM head for AMC now (cont == 0, phase AMC).
__global__ void k_flag_leave(int32_t na, const int32_t *__restrict__ act, const QState *__restrict__ qs,
                             const int32_t *__restrict__ cont, int32_t *__restrict__ flag)
{
    const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= na) return;
    flag[i] = ((cont == nullptr || !cont[i]) && qs[act[i]].phase == PH_AMC) ? 1 : 0;
}

// Sum of eta0 over a list (sizes the per-batch partial buffers of an AMC group).
__global__ void k_sum_eta0(int32_t na, const int32_t *__restrict__ list, const QState *__restrict__ qs,
                           unsigned long long *__restrict__ out)
{
    const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    unsigned long long v = i < na ? (unsigned long long)qs[list[i]].st.eta0 : 0ull;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0 && v) atomicAdd(out, v);
}

// All queries in phase PH_AMC: flags for the AMC list and the sum of their eta0 (sizes the
// per-batch partial buffers), in one pass.
__global__ void k_amc_flags(int64_t k, const QState *__restrict__ qs, int32_t *__restrict__ flags,
                            int32_t *__restrict__ ids, unsigned long long *__restrict__ eta0_sum)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const bool amc = i < k && qs[i].phase == PH_AMC;
    if (i < k) {
        flags[i] = amc ? 1 : 0;
        ids[i] = (int32_t)i;
    }
    unsigned long long v = amc ? (unsigned long long)qs[i].st.eta0 : 0ull;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0 && v) atomicAdd(eta0_sum, v);
}

// K8: r' = r_f + r_b (Alg. 3 L11); s = t -> 0.
__global__ void k_finalize(int64_t k, const QState *__restrict__ qs, double *__restrict__ out,
                           er_query_stats *__restrict__ stats)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= k) return;
    const QState &Q = qs[i];
    er_query_stats st = Q.st;
    st.ytable_log2 = (uint32_t)Q.ylog2;
    double r;
    if (Q.s == Q.t) {
        memset(&st, 0, sizeof(st));
        r = 0.0;
    } else {
        st.r_f = st.batches_run > 0 ? Q.z : 0.0;
        r = st.r_f + st.r_b;
    }
    out[i] = r;
    if (stats) stats[i] = st;
}

__global__ void k_select(int32_t n, const int32_t *__restrict__ in, const int32_t *__restrict__ flag,
                         const int32_t *__restrict__ incl, int32_t *__restrict__ out)
{
    const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n && flag[i]) out[incl[i] - 1] = in[i];
}

// ============================================================================ host side

// ER_ENOMEM fault injection (tests): GEER_FAULT_ALLOC=N, read at er_graph_create, makes the N-th
// workspace growth after it fail like an out-of-memory cudaMalloc (once).
std::atomic<int64_t> g_fault_target{0}, g_fault_count{0};

cudaError_t DevBuf::ensure(size_t bytes, bool keep, cudaStream_t st)
{
    if (bytes <= cap) return cudaSuccess;
    if (g_fault_target.load() > 0 && ++g_fault_count == g_fault_target.load()) return cudaErrorMemoryAllocation;
    size_t ncap = std::max(bytes, cap + cap / 2);
    ncap = (ncap + 255) & ~(size_t)255;
    void *np = nullptr;
    cudaError_t e = cudaMalloc(&np, ncap);
    if (e != cudaSuccess) {
        ncap = (bytes + 255) & ~(size_t)255;
        cudaGetLastError();
        e = cudaMalloc(&np, ncap);
        if (e != cudaSuccess) return e;
    }
    if (keep && p && cap) {
        e = cudaMemcpyAsync(np, p, cap, cudaMemcpyDeviceToDevice, st);
        if (e != cudaSuccess) return e;
        e = cudaStreamSynchronize(st);
        if (e != cudaSuccess) return e;
    }
    if (p) {
        cudaStreamSynchronize(st);
        cudaFree(p);
    }
    p = np;
    cap = ncap;
    return cudaSuccess;
}

void DevBuf::release()
{
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
}

void Workspace::release()
{
    DevBuf *all[] = {&qs, &pairs, &out, &stats, &act, &act2, &cont, &idx, &fr_id, &fr_val, &fr_seg, &fr_off,
                     &nf_id, &nf_val, &nf_seg, &nf_off, &ent_off, &keys, &vals, &keys2, &vals2,
                     &runstart, &segstat, &ycap, &yoff, &cub_tmp, &scalars, &ids, &seglen, &segbeg, &cont2,
                     &idx2, &spmm_part, &qids, &dense_x, &dense_y, &dense_cnt, &ydesc, &ywid, &pk_seg, &pk_bkt, &pk_keys,
                     &pk_alt, &pk_out};
    for (DevBuf *b : all) b->release();
    for (DevBuf &b : ychunk) b.release();
    ychunk.clear();
    if (host_pinned) cudaFreeHost(host_pinned);
    host_pinned = nullptr;
    host_pinned_cap = 0;
}

namespace {

// Select ids[i] for which flag[i] != 0, in order.  Returns the count through *cnt.
int select_list(Ctx &c, const int32_t *ids, const int32_t *flag, int32_t n, int32_t *out, int32_t *incl_tmp,
                int64_t *cnt)
{
    if (n == 0) {
        *cnt = 0;
        return ER_OK;
    }
    int rc = scan_incl(c, flag, incl_tmp, n);
    if (rc) return rc;
    k_select<<<blocks_for(n, 256), 256, 0, c.st>>>(n, ids, flag, incl_tmp, out);
    LAUNCHED(c.g);
    int32_t h = 0;
    CK(cudaMemcpyAsync(&h, incl_tmp + (n - 1), sizeof(int32_t), cudaMemcpyDeviceToHost, c.st));
    CK(cudaStreamSynchronize(c.st));
    *cnt = h;
    return ER_OK;
}


}  // namespace

int run_query_batch(er_graph *g, const int32_t *pairs, int64_t k, double eps, double p_fail, const er_opts &o,
                    double *out_r, er_query_stats *stats)
{
    NvtxRange nvtx_("geer/batch");
    Workspace &ws = g->ws;
    // The batch runs on the handle's high-priority head stream (so SMM-head kernels are scheduled
    // ahead of AMC walk CTAs when both are queued), forked from and joined back into the
    // caller's stream.
    const cudaStream_t user = o.cuda_stream ? (cudaStream_t)o.cuda_stream : g->stream;
    const cudaStream_t st = g->head_stream;
    if (!g->ev_in) {
        CK(cudaEventCreateWithFlags(&g->ev_in, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&g->ev_out, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&g->ev_yfork, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&g->ev_ydone, cudaEventDisableTiming));
        CK(cudaStreamCreateWithFlags(&g->ybuild_stream, cudaStreamNonBlocking));
    }
    CK(cudaEventRecord(g->ev_in, user));
    CK(cudaStreamWaitEvent(st, g->ev_in, 0));
    if (!ws.host_pinned) {
        CK(cudaMallocHost(&ws.host_pinned, 4096));
        ws.host_pinned_cap = 4096;
    }
    Ctx c{g, st, ws, reinterpret_cast<int64_t *>(ws.host_pinned)};
    if (k == 0) return ER_OK;
    if (k > (int64_t)INT32_MAX / 4) {
        set_error(ER_EINVAL, "k too large for one batch (max 536870911)");
        return ER_EINVAL;
    }

    BatchParams P;
    P.eps = eps;
    P.delta = p_fail;
    P.lambda = g->lambda;
    P.log_inv_lambda = std::log(1.0 / g->lambda);
    P.L_eta = std::log(2.0 * (double)o.tau / p_fail);
    P.L_bern = std::log(3.0 / (p_fail / (double)o.tau));
    P.tau = o.tau;
    P.force_ell_b = o.force_ell_b;
    P.ell_variant = o.ell_variant;
    P.reuse = o.reuse_samples;
    P.switch_ratio = o.switch_ratio;
    P.nbits = g->nbits;
    P.seed = o.seed;
    P.qbase = o.query_index_base;
    P.n = g->n;

    // ---- inputs
    const int32_t *d_pairs = pairs;
    if (!o.pairs_on_device) {
        ENSURE(ws.pairs, sizeof(int32_t) * 2 * k, false);
        CK(cudaMemcpyAsync(ws.pairs.p, pairs, sizeof(int32_t) * 2 * k, cudaMemcpyHostToDevice, st));
        d_pairs = ws.pairs.as<int32_t>();
    }
    const int64_t *d_ids = o.query_ids;
    if (d_ids && !o.pairs_on_device) {
        ENSURE(ws.qids, sizeof(int64_t) * k, false);
        CK(cudaMemcpyAsync(ws.qids.p, o.query_ids, sizeof(int64_t) * k, cudaMemcpyHostToDevice, st));
        d_ids = ws.qids.as<int64_t>();
    }
    ENSURE(ws.qs, sizeof(QState) * k, false);
    QState *qs = ws.qs.as<QState>();
    k_setup<<<blocks_for(k, 128), 128, 0, st>>>(k, d_pairs, d_ids, g->d_off, P, qs);
    LAUNCHED(g);

    const int32_t K = (int32_t)k;
    ENSURE(ws.cont, sizeof(int32_t) * (k + 1), false);
    ENSURE(ws.idx, sizeof(int32_t) * (k + 1), false);
    ENSURE(ws.act, sizeof(int32_t) * (k + 1), false);
    ENSURE(ws.act2, sizeof(int32_t) * (k + 1), false);
    int64_t smm_pairs = 0;
    int rc;

    // AMC stream: the walks of all AMC queries after the head (default), or, with
    // GEER_AMC_OVERLAP=1, each wave's leavers concurrently with the remaining SMM waves
    // (measured slower).
    cudaStream_t sb = g->amc_stream;
    cudaEvent_t ev_start = nullptr, ev_smm_end = nullptr, ev_end = nullptr, ev_amc_done = nullptr;
    const bool prof = g->profiling;
    BatchRes R;
    CK(cudaEventCreateWithFlags(&ev_amc_done, cudaEventDisableTiming));
    if (prof) {
        CK(cudaEventCreate(&ev_start));
        CK(cudaEventCreate(&ev_smm_end));
        CK(cudaEventCreate(&ev_end));
        CK(cudaEventRecord(ev_start, st));
    }
    // Launch the AMC of a list of queries (all in phase PH_AMC) on the AMC stream, after
    // everything enqueued so far on the head stream and after the y-table builds.
    auto launch_list = [&](int32_t ng, const int32_t *list_src, int64_t known_eta0_sum = -1) -> int {
        AmcGroup G;
        G.na = ng;
        CK(cudaMallocAsync((void **)&G.list, sizeof(int32_t) * ng, st));
        CK(cudaMemcpyAsync(G.list, list_src, sizeof(int32_t) * ng, cudaMemcpyDeviceToDevice, st));
        if (known_eta0_sum < 0) {
            unsigned long long *d_sum = reinterpret_cast<unsigned long long *>(ws.scalars.as<int64_t>() + 4);
            CK(cudaMemsetAsync(d_sum, 0, sizeof(unsigned long long), st));
            k_sum_eta0<<<blocks_for(ng, 256), 256, 0, st>>>(ng, G.list, qs, d_sum);
            LAUNCHED(g);
            int rr = read_scalars(c, {reinterpret_cast<const int64_t *>(d_sum)});
            if (rr) return rr;
            known_eta0_sum = c.hp[0];
        }
        G.eta0_sum = (unsigned long long)known_eta0_sum;
        R.bufs.push_back(G.list);
        cudaEvent_t e;
        CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        CK(cudaEventRecord(e, st));
        CK(cudaStreamWaitEvent(sb, e, 0));
        CK(cudaStreamWaitEvent(sb, g->ev_ydone, 0));   // the last SMM wave's y-tables (side stream)
        cudaEventDestroy(e);
        return launch_amc_group(g, sb, G, qs, P, prof, R);
    };
    // Queries of an SMM wave that leave the head now: with overlap, their AMC starts at once on
    // the AMC stream (concurrent with the remaining waves); otherwise all AMC queries run
    // together after the head (fewer, fuller walk launches).  The tables' buffers live until
    // the end of the batch either way.
    const bool overlap = g->amc_overlap;
    auto fork_group = [&](int32_t na, const int32_t *act, const int32_t *cont) -> int {
        if (!overlap) return ER_OK;
        // list of the queries of act leaving now for AMC
        int32_t *flag = ws.cont2.as<int32_t>();
        k_flag_leave<<<blocks_for(na, 256), 256, 0, st>>>(na, act, qs, cont, flag);
        LAUNCHED(g);
        int64_t ng = 0;
        int rr = select_list(c, act, flag, na, ws.act2.as<int32_t>(), ws.idx2.as<int32_t>(), &ng);
        if (rr) return rr;
        if (ng == 0) return ER_OK;
        return launch_list((int32_t)ng, ws.act2.as<int32_t>());
    };
    ENSURE(ws.scalars, sizeof(int64_t) * 8, false);
    ENSURE(ws.cont2, sizeof(int32_t) * (k + 1), false);
    ENSURE(ws.idx2, sizeof(int32_t) * (k + 1), false);

    // ---- SMM head
    {
        // all-query ids and phase flags
        ENSURE(ws.ids, sizeof(int32_t) * (k + 1), false);
        int32_t *ids = ws.ids.as<int32_t>();
        k_flag_phase<<<blocks_for(k, 256), 256, 0, st>>>(k, qs, PH_SMM, ws.cont.as<int32_t>(), ids);
        LAUNCHED(g);
        int64_t na = 0;
        rc = select_list(c, ids, ws.cont.as<int32_t>(), K, ws.act.as<int32_t>(), ws.idx.as<int32_t>(), &na);
        if (rc) return rc;
        // AMC-only queries (force_ell_b == 0): tables from e_s, e_t, one group.
        if (P.force_ell_b == 0) {
            k_flag_phase<<<blocks_for(k, 256), 256, 0, st>>>(k, qs, PH_AMC, ws.cont.as<int32_t>(), ids);
            LAUNCHED(g);
            int64_t n0 = 0;
            rc = select_list(c, ids, ws.cont.as<int32_t>(), K, ws.act.as<int32_t>(), ws.idx.as<int32_t>(), &n0);
            if (rc) return rc;
            if (n0 > 0) {
                const int64_t F0 = 2 * n0;
                ENSURE(ws.fr_id, sizeof(int32_t) * F0, false);
                ENSURE(ws.fr_val, sizeof(double) * F0, false);
                ENSURE(ws.fr_seg, sizeof(int32_t) * F0, false);
                ENSURE(ws.fr_off, sizeof(int64_t) * (F0 + 1), false);
                k_init_frontier<<<blocks_for(F0 + 1, 256), 256, 0, st>>>((int32_t)n0, ws.act.as<int32_t>(), qs,
                                                                       ws.fr_id.as<int32_t>(), ws.fr_val.as<double>(),
                                                                       ws.fr_seg.as<int32_t>(), ws.fr_off.as<int64_t>());
                LAUNCHED(g);
                rc = build_ytables(c, (int32_t)n0, ws.act.as<int32_t>(), nullptr, ws.fr_off.as<int64_t>(),
                                   ws.fr_id.as<int32_t>(), ws.fr_val.as<double>(), ws.fr_seg.as<int32_t>(), F0, nullptr,
                                   0);
                if (rc) return rc;
                rc = fork_group((int32_t)n0, ws.act.as<int32_t>(), nullptr);
                if (rc) return rc;
            }
            na = 0;
        }

        int64_t F = 2 * na;
        if (na > 0) {
            ENSURE(ws.fr_id, sizeof(int32_t) * F, false);
            ENSURE(ws.fr_val, sizeof(double) * F, false);
            ENSURE(ws.fr_seg, sizeof(int32_t) * F, false);
            ENSURE(ws.fr_off, sizeof(int64_t) * (F + 1), false);
            k_init_frontier<<<blocks_for(F + 1, 256), 256, 0, st>>>((int32_t)na, ws.act.as<int32_t>(), qs,
                                                                   ws.fr_id.as<int32_t>(), ws.fr_val.as<double>(),
                                                                   ws.fr_seg.as<int32_t>(), ws.fr_off.as<int64_t>());
            LAUNCHED(g);
        }
        bool first_wave = true;
        int wave_no = 0;
        const cudaStream_t ystream = overlap ? nullptr : g->ybuild_stream;
        bool y_pending = false;
        while (na > 0) {
            NvtxRange nvtx_wave("geer/smm_wave");
            const int32_t nseg = (int32_t)(2 * na);
            // emission offsets
            ENSURE(ws.ent_off, sizeof(int64_t) * (2 * F + 2), false);
            int64_t *ent_deg = ws.ent_off.as<int64_t>() + (F + 1);
            int64_t *ent_off = ws.ent_off.as<int64_t>();
            k_ent_deg<<<blocks_for(F, 256), 256, 0, st>>>(F, ws.fr_id.as<int32_t>(), g->d_off, ent_deg);
            LAUNCHED(g);
            rc = scan_offsets(c, ent_deg, ent_off, F);
            if (rc) return rc;
            rc = read_scalars(c, {ent_off + F});
            if (rc) return rc;
            const int64_t E = c.hp[0];
            smm_pairs += E;
            ENSURE(ws.scalars, sizeof(int64_t) * 8, false);
            int64_t *dU = ws.scalars.as<int64_t>();
            const bool fast_first = first_wave && g->rows_sorted;
            // push (K2/K3) or dense pull (K9) for this wave (er_opts.smm_mode, R25)
            // On unsorted adjacency lists the push (ascending source order) and the pull (CSR order)
            // round differently, so the automatic choice, which depends on the other queries of the
            // wave, would make a query's bits depend on batch composition: only an explicit
            // smm_mode = 2 runs dense there.
            bool dense = false;
            if (!fast_first && o.smm_mode != 1 && na <= ER_DENSE_MAX_QUERIES &&
                2.0 * 8.0 * (double)g->n * (double)(2 * na) <= DENSE_MAX_BYTES)
                dense = o.smm_mode == 2 || (g->rows_sorted && dense_wave_pays(g, (int32_t)na, E));
            if (prof && !fast_first) {
                g->prof.smm_waves++;
                if (dense) {
                    g->prof.smm_dense_waves++;
                    g->prof.smm_dense_cols += 2 * na;
                }
            }
            if (dense) smm_pairs -= E;   // no push pairs
            const bool push = !fast_first && !dense;
            // push chunks {first segment, segments, first pair, pairs}: whole queries, at most
            // wave_pairs_max pairs each unless one query alone has more
            std::vector<std::array<int64_t, 4>> chunks;
            if (push) {
                ws.pk_F = F;
                if (E <= g->wave_pairs_max) {
                    chunks.push_back({0, (int64_t)nseg, 0, E});
                } else {
                    ENSURE(ws.seglen, sizeof(int64_t) * (na + 1), false);
                    int64_t *pe = ws.seglen.as<int64_t>();
                    k_query_pairs<<<blocks_for(na + 1, 256), 256, 0, st>>>((int32_t)na, ws.fr_off.as<int64_t>(),
                                                                          ent_off, pe);
                    LAUNCHED(g);
                    std::vector<int64_t> hpe(na + 1);
                    CK(cudaMemcpyAsync(hpe.data(), pe, sizeof(int64_t) * (na + 1), cudaMemcpyDeviceToHost, st));
                    CK(cudaStreamSynchronize(st));
                    int64_t q0 = 0;
                    while (q0 < na) {
                        int64_t q1 = q0 + 1;
                        while (q1 < na && hpe[q1 + 1] - hpe[q0] <= g->wave_pairs_max) q1++;
                        chunks.push_back({2 * q0, 2 * (q1 - q0), hpe[q0], hpe[q1] - hpe[q0]});
                        q0 = q1;
                    }
                }
                // part A of the first chunk: reads the frontier, writes the push workspaces only
                rc = smm_push_wave_a(c, (int32_t)chunks[0][0], (int32_t)chunks[0][1], chunks[0][2], chunks[0][3], ent_off);
                if (rc) return rc;
            }
            if (y_pending) {   // the previous wave's y-table build reads the arrays rewritten below
                CK(cudaStreamWaitEvent(st, g->ev_ydone, 0));
                y_pending = false;
            }
            ENSURE(ws.nf_id, sizeof(int32_t) * E, false);
            ENSURE(ws.nf_val, sizeof(double) * E, false);
            ENSURE(ws.nf_seg, sizeof(int32_t) * E, false);
            ENSURE(ws.nf_off, sizeof(int64_t) * (nseg + 1), false);
            ENSURE(ws.segstat, sizeof(SegStat) * nseg, false);
            CK(cudaMemsetAsync(ws.segstat.p, 0, sizeof(SegStat) * nseg, st));
            if (dense) {
                rc = smm_dense_wave(c, (int32_t)na, F, ws.act.as<int32_t>(), dU);
                if (rc) return rc;
            } else if (fast_first) {
                k_first_wave<<<blocks_for(E, 256), 256, 0, st>>>(E, nseg, ent_off, ws.fr_id.as<int32_t>(), g->d_off,
                                                                 g->d_rec, g->d_cols, g->d_arcs, g->d_parcs, g->pack,
                                                                 ws.act.as<int32_t>(), qs,
                                                                 ws.nf_id.as<int32_t>(), ws.nf_val.as<double>(),
                                                                 ws.nf_seg.as<int32_t>(), ws.segstat.as<SegStat>(), dU);
                LAUNCHED(g);
            } else {   // part B: statistics and the contiguous next frontier; then the other chunks
                for (size_t ch = 0; ch < chunks.size(); ch++) {
                    if (ch > 0) {
                        rc = smm_push_wave_a(c, (int32_t)chunks[ch][0], (int32_t)chunks[ch][1], chunks[ch][2],
                                             chunks[ch][3], ent_off);
                        if (rc) return rc;
                    }
                    rc = smm_push_wave_b(c, (int32_t)chunks[ch][0], (int32_t)chunks[ch][1], dU);
                    if (rc) return rc;
                }
            }
            if (!push) {   // first wave / dense: max2 and the segment offsets of the next frontier
                k_seg_max2<<<resident_grid(g, E, 256), 256, 0, st>>>(E, dU, ws.nf_seg.as<int32_t>(),
                                                                     ws.nf_val.as<double>(), ws.segstat.as<SegStat>());
                LAUNCHED(g);
                k_seg_off<<<blocks_for(nseg + 1, 256), 256, 0, st>>>(nseg, dU, ws.nf_seg.as<int32_t>(),
                                                                     ws.nf_off.as<int64_t>());
                LAUNCHED(g);
            }
            int32_t *cont = ws.cont.as<int32_t>();
            k_decide<<<blocks_for(na, 128), 128, 0, st>>>((int32_t)na, ws.act.as<int32_t>(), ws.segstat.as<SegStat>(),
                                                          P, qs, cont);
            LAUNCHED(g);
            // y-table plan of the queries leaving the head now + compaction scans of the others,
            // then ONE host read for all sizes
            const int64_t *th, *tv, *tr;
            rc = ytable_plan(c, (int32_t)na, ws.act.as<int32_t>(), cont, ws.nf_off.as<int64_t>(), &th, &tv, &tr);
            if (rc) return rc;
            int32_t *newidx = ws.idx.as<int32_t>();
            rc = scan_incl(c, cont, newidx, na);
            if (rc) return rc;
            ENSURE(ws.seglen, sizeof(int64_t) * (2 * nseg + 2), false);  // seglen | segnew_incl
            int64_t *seglen = ws.seglen.as<int64_t>();
            int64_t *segnew = seglen + nseg;
            k_seglen<<<blocks_for(nseg, 256), 256, 0, st>>>(nseg, cont, ws.nf_off.as<int64_t>(), seglen);
            LAUNCHED(g);
            rc = scan_incl(c, seglen, segnew, nseg);
            if (rc) return rc;
            CK(cudaMemcpyAsync(c.hp + 0, newidx + (na - 1), sizeof(int32_t), cudaMemcpyDeviceToHost, st));
            CK(cudaMemcpyAsync(c.hp + 1, segnew + (nseg - 1), sizeof(int64_t), cudaMemcpyDeviceToHost, st));
            CK(cudaMemcpyAsync(c.hp + 2, th, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
            CK(cudaMemcpyAsync(c.hp + 3, tv, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
            CK(cudaMemcpyAsync(c.hp + 4, tr, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
            CK(cudaMemcpyAsync(c.hp + 5, dU, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
            CK(cudaStreamSynchronize(st));
            const int64_t na2 = (int64_t)(*reinterpret_cast<int32_t *>(c.hp + 0));
            const int64_t F2 = c.hp[1];
            const int64_t YH = c.hp[2], YV = c.hp[3], YR = c.hp[4];
            const int64_t U = c.hp[5];   // next-frontier entries (<= E): the grid of the passes below
            // y-tables, then (overlap) their AMC on the AMC stream.  Without overlap the tables are
            // built on a side stream concurrently with this wave's compaction and the next wave's
            // emission and sort (both latency-bound); the next wave waits for them before it
            // rewrites the next-frontier arrays the build reads ("K5").
            if (ystream) {
                CK(cudaEventRecord(g->ev_yfork, st));
                CK(cudaStreamWaitEvent(ystream, g->ev_yfork, 0));
                Ctx cy{g, ystream, ws, c.hp};
                rc = ytable_build(cy, (int32_t)na, ws.act.as<int32_t>(), ws.nf_off.as<int64_t>(),
                                  ws.nf_id.as<int32_t>(), ws.nf_val.as<double>(), ws.nf_seg.as<int32_t>(), U, nullptr,
                                  1 + wave_no, YH, YV, YR);
                if (rc) return rc;
                CK(cudaEventRecord(g->ev_ydone, ystream));
                y_pending = true;
            } else {
                rc = ytable_build(c, (int32_t)na, ws.act.as<int32_t>(), ws.nf_off.as<int64_t>(),
                                  ws.nf_id.as<int32_t>(), ws.nf_val.as<double>(), ws.nf_seg.as<int32_t>(), U, dU,
                                  1 + wave_no, YH, YV, YR);
                if (rc) return rc;
            }
            rc = fork_group((int32_t)na, ws.act.as<int32_t>(), cont);
            if (rc) return rc;
            if (na2 > 0) {
                ENSURE(ws.fr_id, sizeof(int32_t) * F2, false);
                ENSURE(ws.fr_val, sizeof(double) * F2, false);
                ENSURE(ws.fr_seg, sizeof(int32_t) * F2, false);
                ENSURE(ws.fr_off, sizeof(int64_t) * (2 * na2 + 1), false);
                k_compact_entries<<<blocks_for(U, 256), 256, 0, st>>>(
                    U, dU, ws.nf_seg.as<int32_t>(), ws.nf_id.as<int32_t>(), ws.nf_val.as<double>(),
                    ws.nf_off.as<int64_t>(), cont, newidx, segnew, seglen, ws.fr_id.as<int32_t>(),
                    ws.fr_val.as<double>(), ws.fr_seg.as<int32_t>());
                LAUNCHED(g);
                k_compact_lists<<<blocks_for(na, 256), 256, 0, st>>>((int32_t)na, cont, newidx, ws.act.as<int32_t>(),
                                                                     segnew, seglen, ws.act2.as<int32_t>(),
                                                                     ws.fr_off.as<int64_t>());
                LAUNCHED(g);
                std::swap(ws.act, ws.act2);
            }
            na = na2;
            F = F2;
            first_wave = false;
            wave_no++;
        }
    }

    if (!overlap) {
        // every query now in phase AMC: one AMC run over all of them (the AMC stream waits for
        // the last wave's y-tables, so this list building overlaps their build)
        ENSURE(ws.ids, sizeof(int32_t) * (k + 1), false);
        unsigned long long *d_sum = reinterpret_cast<unsigned long long *>(ws.scalars.as<int64_t>() + 5);
        CK(cudaMemsetAsync(d_sum, 0, sizeof(unsigned long long), st));
        k_amc_flags<<<blocks_for(k, 256), 256, 0, st>>>(k, qs, ws.cont.as<int32_t>(), ws.ids.as<int32_t>(), d_sum);
        LAUNCHED(g);
        rc = scan_incl(c, ws.cont.as<int32_t>(), ws.idx.as<int32_t>(), K);
        if (rc) return rc;
        // the list goes to act2: the last wave's y-table build (side stream) may still read act
        k_select<<<blocks_for(K, 256), 256, 0, st>>>(K, ws.ids.as<int32_t>(), ws.cont.as<int32_t>(),
                                                      ws.idx.as<int32_t>(), ws.act2.as<int32_t>());
        LAUNCHED(g);
        CK(cudaMemcpyAsync(c.hp + 0, ws.idx.as<int32_t>() + (K - 1), sizeof(int32_t), cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(c.hp + 1, d_sum, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        const int64_t n_amc = (int64_t)(*reinterpret_cast<int32_t *>(c.hp + 0));
        const int64_t amc_eta0 = c.hp[1];
        if (prof) CK(cudaEventRecord(ev_smm_end, st));
        if (n_amc > 0) {
            rc = launch_list((int32_t)n_amc, ws.act2.as<int32_t>(), amc_eta0);
            if (rc) return rc;
        }
    } else if (prof) {
        CK(cudaEventRecord(ev_smm_end, st));
    }
    // join: results need every group's AMC
    CK(cudaEventRecord(ev_amc_done, sb));
    CK(cudaStreamWaitEvent(st, ev_amc_done, 0));
    CK(cudaStreamWaitEvent(st, g->ev_ydone, 0));   // y-tables built even when no query reached AMC

    // ---- results
    double *d_out = out_r;
    er_query_stats *d_stats = stats;
    if (!o.out_on_device) {
        ENSURE(ws.out, sizeof(double) * k, false);
        d_out = ws.out.as<double>();
        if (stats) {
            ENSURE(ws.stats, sizeof(er_query_stats) * k, false);
            d_stats = ws.stats.as<er_query_stats>();
        }
    }
    k_finalize<<<blocks_for(k, 128), 128, 0, st>>>(k, qs, d_out, d_stats);
    LAUNCHED(g);
    CK(cudaGetLastError());
    if (!o.out_on_device) {
        CK(cudaMemcpyAsync(out_r, d_out, sizeof(double) * k, cudaMemcpyDeviceToHost, st));
        if (stats) CK(cudaMemcpyAsync(stats, d_stats, sizeof(er_query_stats) * k, cudaMemcpyDeviceToHost, st));
    }
    if (prof) CK(cudaEventRecord(ev_end, st));
    for (void *p : R.bufs) CK(cudaFreeAsync(p, st));
    CK(cudaEventRecord(g->ev_out, st));
    CK(cudaStreamWaitEvent(user, g->ev_out, 0));   // the caller's stream sees the results
    if (o.synchronous || !o.out_on_device || prof) CK(cudaStreamSynchronize(st));
    cudaEventDestroy(ev_amc_done);
    if (prof) {
        float ms = 0.f, smm = 0.f, all = 0.f;
        CK(cudaEventElapsedTime(&smm, ev_start, ev_smm_end));
        CK(cudaEventElapsedTime(&all, ev_start, ev_end));
        double walk = 0.0;
        for (size_t j = 0; j + 1 < R.walk_ev.size(); j += 2) {
            CK(cudaEventElapsedTime(&ms, R.walk_ev[j], R.walk_ev[j + 1]));
            walk += ms;
        }
        if (R.walk_ev.size() >= 2) {
            CK(cudaEventElapsedTime(&ms, R.walk_ev.front(), R.walk_ev.back()));
            g->prof.amc_span_ms += ms;
        }
        g->prof.smm_ms += smm;
        g->prof.walk_ms += walk;
        g->prof.amc_other_ms += all - smm;   // AMC time not hidden under the SMM head
        g->prof.walk_launches += (int64_t)(R.walk_ev.size() / 2);
        g->prof.smm_pairs += smm_pairs;
        g->prof.batches += 1;
        for (cudaEvent_t e : R.walk_ev) cudaEventDestroy(e);
        cudaEventDestroy(ev_start);
        cudaEventDestroy(ev_smm_end);
        cudaEventDestroy(ev_end);
    }
    return ER_OK;
}

__global__ void k_build_arcs(int64_t nnz, const int32_t *__restrict__ cols, const uint2 *__restrict__ rec,
                             uint4 *__restrict__ arcs)
{
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= nnz) return;
    const int32_t u = cols[e];
    const uint2 r = rec[u];
    arcs[e] = make_uint4((uint32_t)u, r.x, r.y, 0u);
}

__global__ void k_build_parcs(int64_t nnz, const int32_t *__restrict__ cols, const uint2 *__restrict__ rec,
                              PackSpec pk, unsigned long long *__restrict__ parcs)
{
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= nnz) return;
    const int32_t u = cols[e];
    const uint2 r = rec[u];
    parcs[e] = pk.pack((uint32_t)u, r.x, r.y);
}

// 24-bit columns (node ids < 2^24), 5 per 16-byte chunk: column e in chunk e / 5 at bytes
// 3 (e mod 5) .. +2, little endian; the last 1 byte of each chunk is padding, so every column sits
// inside one 16-byte load.
__global__ void k_build_c24(int64_t nnz, const int32_t *__restrict__ cols, uint4 *__restrict__ c24)
{
    const int64_t ch = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (ch * 5 >= nnz) return;
    unsigned char b[16] = {0};
    for (int j = 0; j < 5; j++) {
        const int64_t e = ch * 5 + j;
        const uint32_t u = e < nnz ? (uint32_t)cols[e] : 0u;
        b[3 * j] = (unsigned char)(u & 255u);
        b[3 * j + 1] = (unsigned char)((u >> 8) & 255u);
        b[3 * j + 2] = (unsigned char)((u >> 16) & 255u);
    }
    uint4 q;
    q.x = b[0] | (b[1] << 8) | (b[2] << 16) | ((uint32_t)b[3] << 24);
    q.y = b[4] | (b[5] << 8) | (b[6] << 16) | ((uint32_t)b[7] << 24);
    q.z = b[8] | (b[9] << 8) | (b[10] << 16) | ((uint32_t)b[11] << 24);
    q.w = b[12] | (b[13] << 8) | (b[14] << 16) | ((uint32_t)b[15] << 24);
    c24[ch] = q;
}

cudaError_t build_c24(er_graph *g)
{
    const int64_t nch = (g->nnz + 4) / 5;
    k_build_c24<<<blocks_for(nch, 256), 256>>>(g->nnz, g->d_cols, g->d_c24);
    g->launches++;
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    return e;
}

int build_dord(er_graph *g, const int64_t *off, const int32_t *cols)
{
    const int64_t n = g->n, nnz = g->nnz;
    if (n > (1ll << 24) || nnz >= (1ll << 32) || nnz == 0) return 1;
    int64_t maxd = 0;
    for (int64_t v = 0; v < n; v++) maxd = std::max(maxd, off[v + 1] - off[v]);
    std::vector<int64_t> cnt(maxd + 1, 0);
    for (int64_t v = 0; v < n; v++) cnt[off[v + 1] - off[v]]++;
    std::vector<int64_t> cdeg;   // classes in descending degree
    for (int64_t d = maxd; d >= 0; d--)
        if (cnt[d] > 0) cdeg.push_back(d);
    const int64_t K = (int64_t)cdeg.size();
    if (K > 65535) return 1;
    // the smallest block (least padding) whose tables fit the shared-memory budget
    int bs = -1;
    int64_t nv = 0;
    for (int b = 4; b <= 16 && bs < 0; b++) {
        int64_t v = 0;
        for (int64_t c = 0; c < K; c++) v += ((cnt[cdeg[c]] + (1ll << b) - 1) >> b) << b;
        if (v <= (1ll << 24) && 2 * (v >> b) + 8 * K <= g->dord_smem_bytes) { bs = b; nv = v; }
    }
    if (bs < 0) return 1;
    const int64_t nblk = nv >> bs;
    std::vector<int64_t> pos(maxd + 1, 0);
    std::vector<uint16_t> blk(nblk);
    std::vector<uint2> cd(K);
    {
        int64_t vstart = 0, arcs = 0;
        for (int64_t c = 0; c < K; c++) {
            const int64_t d = cdeg[c], size = ((cnt[d] + (1ll << bs) - 1) >> bs) << bs;
            pos[d] = vstart;
            cd[c] = make_uint2((uint32_t)arcs - (uint32_t)vstart * (uint32_t)d, (uint32_t)d);   // mod 2^32
            for (int64_t k = vstart >> bs; k < (vstart + size) >> bs; k++) blk[k] = (uint16_t)c;
            vstart += size;
            arcs += cnt[d] * d;
        }
    }
    // renumbering: by descending degree, ties by id (a stable counting sort)
    std::vector<int32_t> perm(n), iperm(nv, -1);
    for (int64_t v = 0; v < n; v++) {
        const int64_t u = pos[off[v + 1] - off[v]]++;
        perm[v] = (int32_t)u;
        iperm[u] = (int32_t)v;
    }
    // the renumbered CSR: row perm[v] = perm of v's neighbours, in v's order (padding ids: no row)
    std::vector<int32_t> ncols(nnz);
    {
        int64_t j = 0;
        for (int64_t u = 0; u < nv; u++) {
            const int32_t v = iperm[u];
            if (v < 0) continue;
            for (int64_t e = off[v]; e < off[v + 1]; e++) ncols[j++] = perm[cols[e]];
        }
    }
    int32_t *dtmp = nullptr;
    cudaError_t e = cudaMalloc(&g->d_c24, sizeof(uint4) * std::max<int64_t>((nnz + 4) / 5, 1));
    if (e == cudaSuccess) e = cudaMalloc(&dtmp, sizeof(int32_t) * nnz);
    if (e == cudaSuccess) e = cudaMalloc(&g->d_perm, sizeof(int32_t) * n);
    if (e == cudaSuccess) e = cudaMalloc(&g->d_iperm, sizeof(int32_t) * nv);
    if (e == cudaSuccess) e = cudaMalloc(&g->d_cblk, sizeof(uint16_t) * nblk);
    if (e == cudaSuccess) e = cudaMalloc(&g->d_ccd, sizeof(uint2) * K);
    if (e == cudaSuccess) e = cudaMemcpy(dtmp, ncols.data(), sizeof(int32_t) * nnz, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(g->d_perm, perm.data(), sizeof(int32_t) * n, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(g->d_iperm, iperm.data(), sizeof(int32_t) * nv, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(g->d_cblk, blk.data(), sizeof(uint16_t) * nblk, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(g->d_ccd, cd.data(), sizeof(uint2) * K, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) {
        k_build_c24<<<blocks_for((nnz + 4) / 5, 256), 256>>>(nnz, dtmp, g->d_c24);
        g->launches++;
        e = cudaGetLastError();
        if (e == cudaSuccess) e = cudaDeviceSynchronize();
    }
    if (dtmp) cudaFree(dtmp);
    if (e != cudaSuccess) {
        cuda_fail(e, "er_graph_create (degree-ordered walk graph)");
        return -1;
    }
    g->dord_nblk = (int32_t)nblk;
    g->dord_ncls = (int32_t)K;
    g->dord_bshift = bs;
    g->dord_nv = nv;
    return 0;
}

cudaError_t build_parcs(er_graph *g)
{
    k_build_parcs<<<blocks_for(g->nnz, 256), 256>>>(g->nnz, g->d_cols, g->d_rec, g->pack, g->d_parcs);
    g->launches++;
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    return e;
}

cudaError_t build_arcs(er_graph *g)
{
    k_build_arcs<<<blocks_for(g->nnz, 256), 256>>>(g->nnz, g->d_cols, g->d_rec, g->d_arcs);
    g->launches++;
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    return e;
}

}  // namespace geer
