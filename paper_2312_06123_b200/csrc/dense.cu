// dense.cu -- the SMM head's dense mode: one SMM iteration (Alg. 3 L6) of every active
// query of a wave applied as a dense pull over the whole CSR (K9) instead of the sparse push
// (K2/K3), chosen per wave by a cost model (R25).
//
//   scatter   X[v, g] = x_g(v) for the frontier entries (X zeroed): n x q block, q = 2 na columns
//   K9 exact  Y = D^-1 A X, every row summed sequentially in CSR order (spmm.cu)
//   extract   the nonzeros of each column g in ascending row order -> the next frontier segment
//             g, exactly the layout K3 produces, with the K4a statistics (vol, max1, x(s), x(t))
//
// Bit-identical to the push on sorted adjacency lists: x >= 0, so the pull's extra terms are
// exact zeros (0.0 + a = a, a + 0.0 = a), its nonzero terms arrive in CSR = ascending source
// order like K3's runs, and the support is the set of nonzero sums (R13).  On unsorted lists the
// pull keeps CSR order (the oracle's), the push ascending source order.

#include <algorithm>

#include "stages.h"

namespace geer {

constexpr int DENSE_TILE = 256;   // rows per extraction tile (one CTA)

__global__ void k_dense_scatter(int64_t F, const int32_t *__restrict__ id, const double *__restrict__ val,
                                const int32_t *__restrict__ seg, int32_t q, double *__restrict__ X)
{
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= F) return;
    X[(int64_t)id[e] * q + seg[e]] = val[e];
}

// cnt[g * ntiles + t] = nonzeros of column g in rows [t DENSE_TILE, (t+1) DENSE_TILE).  Warp w of
// the tile's CTA takes columns w, w + 8, ...; the tile's rows are read 32 at a time (the CTA's
// warps share the rows' sectors in L1).
__global__ void __launch_bounds__(DENSE_TILE)
k_dense_count(int64_t n, int32_t q, int64_t ntiles, const double *__restrict__ Y, int64_t *__restrict__ cnt)
{
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t t = blockIdx.x, r0 = t * DENSE_TILE;
    for (int32_t g = warp; g < q; g += DENSE_TILE / 32) {
        int64_t c = 0;
        for (int64_t r = r0; r < r0 + DENSE_TILE && r < n; r += 32) {
            const bool nz = r + lane < n && Y[(r + lane) * q + g] != 0.0;
            c += __popc(__ballot_sync(0xffffffffu, nz));
        }
        if (lane == 0) cnt[(int64_t)g * ntiles + t] = c;
    }
}

// Write the nonzeros: column g, tile t starts at pos[g * ntiles + t] (exclusive scan of cnt in
// column-major order = segment order), rows ascending.  Fused K4a statistics per segment.
__global__ void __launch_bounds__(DENSE_TILE)
k_dense_emit(int64_t n, int32_t q, int64_t ntiles, const double *__restrict__ Y, const int64_t *__restrict__ pos,
             const uint2 *__restrict__ rec, const int32_t *__restrict__ act, const QState *__restrict__ qs,
             int32_t *__restrict__ nid, double *__restrict__ nval, int32_t *__restrict__ nseg,
             SegStat *__restrict__ ss)
{
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t t = blockIdx.x, r0 = t * DENSE_TILE;
    for (int32_t g = warp; g < q; g += DENSE_TILE / 32) {
        int64_t p = pos[(int64_t)g * ntiles + t];
        if (p == pos[(int64_t)g * ntiles + t + 1]) continue;   // no nonzero in this tile
        const QState &Q = qs[act[g >> 1]];
        const int32_t s = Q.s, tt = Q.t;
        unsigned long long vol = 0, mx = 0;
        for (int64_t r = r0; r < r0 + DENSE_TILE && r < n; r += 32) {
            const int64_t u = r + lane;
            const double y = u < n ? Y[u * q + g] : 0.0;
            const bool nz = y != 0.0;
            const unsigned m = __ballot_sync(0xffffffffu, nz);
            if (nz) {
                const int64_t o = p + __popc(m & ((1u << lane) - 1u));
                nid[o] = (int32_t)u;
                nval[o] = y;
                nseg[o] = g;
                vol += (unsigned long long)__ldg(rec + u).y;   // node record {offset, degree}
                const unsigned long long b = (unsigned long long)__double_as_longlong(y);
                mx = b > mx ? b : mx;
                if (u == s) ss[g].at_s = y;
                if (u == tt) ss[g].at_t = y;
            }
            p += __popc(m);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            vol += __shfl_xor_sync(0xffffffffu, vol, o);
            const unsigned long long om = __shfl_xor_sync(0xffffffffu, mx, o);
            mx = om > mx ? om : mx;
        }
        if (lane == 0) {
            atomicAdd(reinterpret_cast<unsigned long long *>(&ss[g].vol), vol);
            atomicMax(reinterpret_cast<unsigned long long *>(&ss[g].max1), mx);
        }
    }
}

__global__ void k_copy_scalar(const int64_t *__restrict__ src, int64_t *__restrict__ dst) { *dst = *src; }

bool dense_wave_pays(const er_graph *g, int32_t na, int64_t E)
{
    // Time estimates in ns (R25; constants from scripts/dense_probe.py on B200,
    // profiles/dense_probe_r01.jsonl).  Push: per emitted pair (emit, radix sort, run reduce)
    // plus a per-wave constant.  Pull: the K9 pass (cols + one X row per arc), zeroing, scatter
    // and the two extraction reads, at a conservative effective bandwidth, next to the heavy
    // rows' sequential chains (the longest one, at ~10 ns per dependent fp64 add incl. its
    // copies), plus a per-wave constant.
    const double q = 2.0 * na, nnz = (double)g->nnz, n = (double)g->n;
    const double t_push = DENSE_PUSH_NS_PER_PAIR * (double)E + 50e3;
    const double bytes = 4.0 * nnz + 8.0 * q * nnz + 48.0 * q * n;
    const double t_dense = std::max(bytes / DENSE_BYTES_PER_NS, 10.0 * (double)g->max_deg) + 100e3;
    return t_dense < t_push;
}

int smm_dense_wave(Ctx &c, int32_t na, int64_t F, const int32_t *act, int64_t *dU)
{
    NvtxRange nvtx_("geer/smm_dense");
    er_graph *g = c.g;
    Workspace &ws = c.ws;
    cudaStream_t st = c.st;
    const int32_t q = 2 * na;
    const int64_t n = g->n;
    const size_t blk = sizeof(double) * (size_t)n * q;
    ENSURE(ws.dense_x, blk, false);
    ENSURE(ws.dense_y, blk, false);
    double *X = ws.dense_x.as<double>(), *Y = ws.dense_y.as<double>();
    CK(cudaMemsetAsync(X, 0, blk, st));
    k_dense_scatter<<<blocks_for(F, 256), 256, 0, st>>>(F, ws.fr_id.as<int32_t>(), ws.fr_val.as<double>(),
                                                        ws.fr_seg.as<int32_t>(), q, X);
    LAUNCHED(g);
    int rc = run_spmm(g, X, Y, q, 1, st, /*exact=*/true);
    if (rc) return rc;
    const int64_t ntiles = (n + DENSE_TILE - 1) / DENSE_TILE;
    const int64_t ncnt = (int64_t)q * ntiles;
    ENSURE(ws.dense_cnt, sizeof(int64_t) * (2 * ncnt + 1), false);
    int64_t *cnt = ws.dense_cnt.as<int64_t>(), *pos = cnt + ncnt;
    k_dense_count<<<(unsigned)ntiles, DENSE_TILE, 0, st>>>(n, q, ntiles, Y, cnt);
    LAUNCHED(g);
    rc = scan_offsets(c, cnt, pos, ncnt);
    if (rc) return rc;
    k_copy_scalar<<<1, 1, 0, st>>>(pos + ncnt, dU);
    LAUNCHED(g);
    k_dense_emit<<<(unsigned)ntiles, DENSE_TILE, 0, st>>>(n, q, ntiles, Y, pos, g->d_rec, act, ws.qs.as<QState>(),
                                                          ws.nf_id.as<int32_t>(), ws.nf_val.as<double>(),
                                                          ws.nf_seg.as<int32_t>(), ws.segstat.as<SegStat>());
    LAUNCHED(g);
    return ER_OK;
}

}  // namespace geer
