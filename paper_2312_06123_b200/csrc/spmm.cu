// spmm.cu -- K9: dense-block SpMM  Y = M X  for a row-major n x q fp64 block, M = D^-1 A or A.
//
// This is the dense form of Alg. 2 L4 "s* <- P s*" applied to q columns at once (the
// SMM / SMM-to-ell ground-truth engine) and of Fig. 3's #path recursion with
// A in place of P.  Per (row v, column c):
//
//     Y[v, c] = ( sum_{w in N(v)} X[w, c] ) / d(v)        (the /d(v) only when normalize)
//
// Summation order (R13, "K9"): rows of degree <= SPMM_SEG are summed SEQUENTIALLY in
// the row's CSR order, so they are bit-identical to the oracle's dense pull
// (oracle_propagate_dense); a longer row is cut into consecutive segments of SPMM_SEG
// neighbours, each summed sequentially, and the segment sums are then added sequentially in
// segment order (a fixed order: run-to-run bit-reproducible, within a few ulps of the plain
// sequential sum).  The EXACT variant (the SMM head's dense mode, and er_spmm_ex) sums every
// row sequentially in CSR order: a heavy row gets a CTA that gathers chunks of its neighbours'
// X rows into shared memory in parallel and one thread per column adds them in order.
//
// Layout and load balance ("K9"):
//  * once per graph, the work items are built: one per heavy-row segment, then one per light
//    row (degree <= SPMM_SEG) in degree-descending order, so the long items start first and a
//    warp's sub-warps see similar lengths;
//  * one sub-warp of LPR lanes per item; lane l owns the 16-byte column vectors l, l+LPR, ...
//    of the row (128-bit loads of X rows, coalesced across the sub-warp); the neighbour loop is
//    unrolled by 8 so 8 independent gathers are in flight per lane, then added in CSR order;
//  * heavy-row segment sums go to a scratch block and a second kernel adds them per row;
//  * q <= 64 (one column vector per lane): k_spmm_items, the same items and sums pipelined
//    across items (precomputed item descriptors, the next item's neighbour ids loaded during the
//    current item's last round of gathers).
// No tensor cores: the contraction has one nonzero per (row, neighbour) and fp64 accumulation.


#include <algorithm>
#include <cmath>
#include <vector>

#include "geer_internal.h"

namespace geer {

namespace {

constexpr int SPMM_THREADS = 256;
#ifndef SPMM_UNROLL
#define SPMM_UNROLL 8   // k_spmm_rows: neighbours (X gathers) in flight per lane and round
#endif
#ifndef SPMM_PUNROLL
#define SPMM_PUNROLL 6  // k_spmm_items: the same (A/B on the LJ-shaped graph: 6 beats 4 and 8)
#endif

inline unsigned blocks_for(int64_t n, int per) { return (unsigned)((n + per - 1) / per); }

template <int VEC> struct VecT;
template <> struct VecT<1> { using T = double; };
template <> struct VecT<2> { using T = double2; };

__device__ __forceinline__ void vadd(double &a, const double b) { a += b; }
__device__ __forceinline__ void vadd(double2 &a, const double2 b) { a.x += b.x; a.y += b.y; }
__device__ __forceinline__ void vzero(double &a) { a = 0.0; }
__device__ __forceinline__ void vzero(double2 &a) { a.x = 0.0; a.y = 0.0; }
__device__ __forceinline__ void vdiv(double &a, double d) { a = a / d; }
__device__ __forceinline__ void vdiv(double2 &a, double d) { a.x = a.x / d; a.y = a.y / d; }

// Items [0, nseg) are heavy-row segments (segment p covers cols[seg_e0[p], min(seg_e0[p] +
// SPMM_SEG, off[row + 1])) of row seg_row[p] and writes the segment sum to part[p]); items
// [nseg, nitems) are the light rows rows[item - nseg] (full row, written to Y).
#ifndef SPMM_MINB
#define SPMM_MINB 4   // 4 resident CTAs per SM (64 registers): +60 % rows in flight (A/B: -32..-40 %)
#endif
template <int LPR, int VEC>
__global__ void __launch_bounds__(SPMM_THREADS, SPMM_MINB)
k_spmm_rows(int64_t nseg, int64_t nitems, const int64_t *__restrict__ seg_e0, const int32_t *__restrict__ seg_row,
            const int32_t *__restrict__ rows, const int64_t *__restrict__ off, const int32_t *__restrict__ cols,
            const double *__restrict__ X, double *__restrict__ Y, double *__restrict__ part, int32_t q, int normalize)
{
    using V = typename VecT<VEC>::T;
    const int64_t it = ((int64_t)blockIdx.x * SPMM_THREADS + threadIdx.x) / LPR;
    const int l = threadIdx.x % LPR;
    if (it >= nitems) return;
    int64_t e0, e1;
    V *out;
    bool norm;
    double dv;
    const int32_t nvec = q / VEC;
    if (it < nseg) {
        const int32_t v = seg_row[it];
        e0 = seg_e0[it];
        e1 = min(e0 + (int64_t)SPMM_SEG, off[v + 1]);
        out = reinterpret_cast<V *>(part) + it * nvec;
        norm = false;
        dv = 1.0;
    } else {
        const int32_t v = rows[it - nseg];
        e0 = off[v];
        e1 = off[v + 1];
        out = reinterpret_cast<V *>(Y) + (int64_t)v * nvec;
        norm = normalize != 0;
        dv = (double)(e1 - e0);
    }
    const V *__restrict__ Xv = reinterpret_cast<const V *>(X);
    for (int32_t cv = l; cv < nvec; cv += LPR) {
        V acc;
        vzero(acc);
        // rounds of SPMM_UNROLL neighbours; the next round's neighbour ids are loaded while this
        // round's X gathers are in flight (one dependent round trip per round, not two)
        int32_t w[SPMM_UNROLL];
#pragma unroll
        for (int j = 0; j < SPMM_UNROLL; j++) w[j] = e0 + j < e1 ? __ldg(cols + e0 + j) : 0;
        for (int64_t e = e0; e < e1; e += SPMM_UNROLL) {
            const int64_t rem = e1 - e;
            V x[SPMM_UNROLL];
#pragma unroll
            for (int j = 0; j < SPMM_UNROLL; j++)
                if (j < rem) x[j] = __ldg(Xv + (int64_t)w[j] * nvec + cv);
#pragma unroll
            for (int j = 0; j < SPMM_UNROLL; j++)
                w[j] = SPMM_UNROLL + j < rem ? __ldg(cols + e + SPMM_UNROLL + j) : 0;
#pragma unroll
            for (int j = 0; j < SPMM_UNROLL; j++)
                if (j < rem) vadd(acc, x[j]);   // CSR order (R13)
        }
        if (norm) vdiv(acc, dv);
        out[cv] = acc;
    }
}

// The same items and sums, software-pipelined across items (q <= 2 LPR VEC: one column vector
// per lane).  Persistent sub-warps take items it, it + nsub, ... (round-robin over the
// degree-descending item order); an item is a precomputed descriptor {first arc, length, row or
// segment} (one coalesced 16-byte load, no dependent off[] load), loaded two items ahead; the
// last round of an item loads the NEXT item's first neighbour ids while its own X gathers are in
// flight, so a row costs one dependent round trip per round of SPMM_PUNROLL neighbours instead of
// rows -> off -> cols -> X.  Sums and their order are those of k_spmm_rows (bit-identical).
#ifndef SPMM_PIPE
#define SPMM_PIPE 1   // 0: k_spmm_rows only; 2: descriptors one item ahead (A/B variants)
#endif
__device__ __forceinline__ int64_t desc_e0(const int4 d)
{
    return (int64_t)(((uint64_t)(uint32_t)d.y << 32) | (uint64_t)(uint32_t)d.x);
}
template <int LPR, int VEC>
__global__ void __launch_bounds__(SPMM_THREADS, SPMM_MINB)
k_spmm_items(int64_t nitems, const int4 *__restrict__ desc, const int32_t *__restrict__ cols,
             const double *__restrict__ X, double *__restrict__ Y, double *__restrict__ part, int32_t q, int normalize)
{
    using V = typename VecT<VEC>::T;
    const int64_t nsub = (int64_t)gridDim.x * (SPMM_THREADS / LPR);
    int64_t it = ((int64_t)blockIdx.x * SPMM_THREADS + threadIdx.x) / LPR;
    const int l = threadIdx.x % LPR;
    const int32_t nvec = q / VEC;
    if (it >= nitems || l >= nvec) return;   // no cross-lane operations below
    const V *__restrict__ Xv = reinterpret_cast<const V *>(X);
    const int4 zero = make_int4(0, 0, 0, 0);
    int4 d = desc[it];
    int64_t itn = it + nsub;
#if SPMM_PIPE != 2
    int4 dn = itn < nitems ? desc[itn] : zero;
#endif
    int32_t w[SPMM_PUNROLL];
    {
        const int64_t e0 = desc_e0(d);
#pragma unroll
        for (int j = 0; j < SPMM_PUNROLL; j++) w[j] = j < d.z ? __ldg(cols + e0 + j) : 0;
    }
    while (true) {
        const int64_t itn2 = itn + nsub;
#if SPMM_PIPE == 2
        const int4 dn = itn < nitems ? desc[itn] : zero;      // one item ahead
#else
        const int4 dn2 = itn2 < nitems ? desc[itn2] : zero;   // two items ahead
#endif
        const int64_t e0 = desc_e0(d), en0 = desc_e0(dn);
        const int32_t len = d.z, lenn = dn.z;   // lenn = 0 past the end
        V acc;
        vzero(acc);
        for (int32_t e = 0; e < len; e += SPMM_PUNROLL) {
            const int32_t rem = len - e;
            V x[SPMM_PUNROLL];
#pragma unroll
            for (int j = 0; j < SPMM_PUNROLL; j++)
                if (j < rem) x[j] = __ldg(Xv + (int64_t)w[j] * nvec + l);
            if (rem > SPMM_PUNROLL) {   // this item's next round
#pragma unroll
                for (int j = 0; j < SPMM_PUNROLL; j++)
                    w[j] = SPMM_PUNROLL + j < rem ? __ldg(cols + e0 + e + SPMM_PUNROLL + j) : 0;
            } else {                   // the next item's first round
#pragma unroll
                for (int j = 0; j < SPMM_PUNROLL; j++) w[j] = j < lenn ? __ldg(cols + en0 + j) : 0;
            }
#pragma unroll
            for (int j = 0; j < SPMM_PUNROLL; j++)
                if (j < rem) vadd(acc, x[j]);   // CSR order (R13)
        }
        if (len == 0) {
#pragma unroll
            for (int j = 0; j < SPMM_PUNROLL; j++) w[j] = j < lenn ? __ldg(cols + en0 + j) : 0;
        }
        if (d.w >= 0) {   // a light row: Y[v] (the full row)
            if (normalize) vdiv(acc, (double)len);
            reinterpret_cast<V *>(Y)[(int64_t)d.w * nvec + l] = acc;
        } else {          // a heavy-row segment: its partial sum
            reinterpret_cast<V *>(part)[(int64_t)(-1 - d.w) * nvec + l] = acc;
        }
        if (itn >= nitems) break;
        itn = itn2;
        d = dn;
#if SPMM_PIPE != 2
        dn = dn2;
#endif
    }
}

// Heavy rows: Y[v, c] = (segment sums of v, added in segment order) [/ d(v)].  One thread per
// (heavy row, column).
__global__ void k_spmm_heavy_sum(int64_t nheavy, const int32_t *__restrict__ rows, const int64_t *__restrict__ hseg,
                                 const int64_t *__restrict__ off, const double *__restrict__ part,
                                 double *__restrict__ Y, int32_t q, int normalize)
{
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= nheavy * q) return;
    const int64_t h = t / q;
    const int32_t c = (int32_t)(t - h * q);
    const int32_t v = rows[h];
    double acc = 0.0;
    for (int64_t p = hseg[h]; p < hseg[h + 1]; p++) acc += part[p * q + c];
    Y[(int64_t)v * q + c] = normalize ? acc / (double)(off[v + 1] - off[v]) : acc;
}

// EXACT heavy rows.  CTA (heavy row v, block of HUB_CB columns): v's neighbours are streamed in
// chunks of HUB_ROWS rows through a HUB_STAGES-deep ring of shared-memory stages filled by
// cp.async (LDGSTS, 16-byte copies of the X row segments when VEC = 2); thread c < w adds column
// c's values sequentially in CSR order (R13) while the next stages are in flight, so Y is the
// plain sequential sum and the copies overlap the dependent add chain.  Column blocks of one row
// run on different SMs (the chain of a column cannot be split without changing the order).
constexpr int HUB_STAGE = 4096;     // doubles per stage (32 KB)
constexpr int HUB_STAGES = 3;       // ring depth (96 KB)

template <int BYTES>
__device__ __forceinline__ void cp_async(void *dst, const void *src)
{
    const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
    if (BYTES == 16) asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(src) : "memory");
    else asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

__device__ __forceinline__ void named_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void named_arrive(int id, int n) { asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory"); }

// Warp-specialised: warp 0 consumes (lane c < w adds column c's values in CSR order), warps 1..7
// produce (cp.async copies of the X row segments of the chunk's neighbours into the stage ring,
// neighbour ids prefetched one chunk ahead).  Per stage s two named barriers: FULL (1 + s; the
// producers arrive once their copies of the chunk have landed, the consumer waits) and EMPTY
// (1 + HUB_STAGES + s; the consumer arrives when it is done with the stage, the producers wait
// before refilling it), so the consumer's dependent-add chain never waits on a CTA-wide barrier.
// Stage layout: HUB_ROWS rows of HUB_CB doubles (columns cb .. cb + w - 1 used).
template <int VEC, int HUB_CB>
__global__ void __launch_bounds__(SPMM_THREADS)
k_spmm_hub_exact(const int32_t *__restrict__ rows, const int64_t *__restrict__ off, const int32_t *__restrict__ cols,
                 const double *__restrict__ X, double *__restrict__ Y, int32_t q, int normalize)
{
    constexpr int HUB_ROWS = HUB_STAGE / HUB_CB;   // rows per chunk
    constexpr int NPT = SPMM_THREADS - 32;          // producer threads
    constexpr int LPR = HUB_CB / VEC;               // producer threads per row
    constexpr int RPI = NPT / LPR;                  // rows per producer pass
    constexpr int PER = (HUB_ROWS + RPI - 1) / RPI; // passes per chunk
    extern __shared__ __align__(16) double hub_sm[];
    const int32_t v = rows[blockIdx.x];
    const int32_t cb = blockIdx.y * HUB_CB;
    const int32_t w = min(HUB_CB, q - cb);
    const int32_t wv = w / VEC;
    const int64_t e0 = off[v], e1 = off[v + 1];
    const int64_t nch = (e1 - e0 + HUB_ROWS - 1) / HUB_ROWS;
    auto rows_of = [&](int64_t c) { return c < nch ? (int32_t)min((int64_t)HUB_ROWS, e1 - (e0 + c * HUB_ROWS)) : 0; };
    if (threadIdx.x < 32) {
        // consumer
        const int lane = threadIdx.x;
        double acc = 0.0;
        for (int64_t c = 0; c < nch; c++) {
            const int st = (int)(c % HUB_STAGES);
            named_sync(1 + st, SPMM_THREADS);   // chunk c has landed
            if (lane < w) {
                const double *col = hub_sm + st * HUB_STAGE + lane;
                const int32_t m = rows_of(c);
                // software-pipelined: the next 8 values are loaded while the current 8 are added,
                // so the loop runs at the latency of the dependent DADD chain
                int32_t j = 0;
                if (m >= 8) {
                    double t[8];
#pragma unroll
                    for (int i = 0; i < 8; i++) t[i] = col[i * HUB_CB];
                    for (j = 8; j + 8 <= m; j += 8) {
                        double u[8];
#pragma unroll
                        for (int i = 0; i < 8; i++) u[i] = col[(j + i) * HUB_CB];
#pragma unroll
                        for (int i = 0; i < 8; i++) acc += t[i];   // CSR order
#pragma unroll
                        for (int i = 0; i < 8; i++) t[i] = u[i];
                    }
#pragma unroll
                    for (int i = 0; i < 8; i++) acc += t[i];
                }
                for (; j < m; j++) acc += col[j * HUB_CB];
            }
            if (c + HUB_STAGES < nch) named_arrive(1 + HUB_STAGES + st, SPMM_THREADS);   // stage free
        }
        if (lane < w) Y[(int64_t)v * q + cb + lane] = normalize ? acc / (double)(e1 - e0) : acc;
        return;
    }
    // producers
    const int pt = threadIdx.x - 32;
    const int kv = pt % LPR, jr = pt / LPR;   // vector within the row, first row
    const bool active = jr < RPI && kv < wv;
    int32_t u[PER];
    auto load = [&](int64_t c) {
        const int32_t m = rows_of(c);
        const int64_t r0 = e0 + c * HUB_ROWS;
#pragma unroll
        for (int p = 0; p < PER; p++) {
            const int32_t j = jr + p * RPI;
            u[p] = (active && j < m) ? __ldg(cols + r0 + j) : 0;
        }
    };
    load(0);
    for (int64_t c = 0; c < nch; c++) {
        const int st = (int)(c % HUB_STAGES);
        if (c >= HUB_STAGES) named_sync(1 + HUB_STAGES + st, SPMM_THREADS);   // the consumer freed it
        if (active) {
            double *dst = hub_sm + st * HUB_STAGE;
            const int32_t m = rows_of(c);
#pragma unroll
            for (int p = 0; p < PER; p++) {
                const int32_t j = jr + p * RPI;
                if (j < m) cp_async<8 * VEC>(dst + j * HUB_CB + kv * VEC, X + (int64_t)u[p] * q + cb + kv * VEC);
            }
        }
        cp_async_commit();
        if (c + 1 < nch) load(c + 1);   // the next chunk's ids, in flight during the copies
        if (c >= 1) {
            cp_async_wait<1>();   // chunk c-1's copies (this thread's) have landed
            named_arrive(1 + (int)((c - 1) % HUB_STAGES), SPMM_THREADS);
        }
    }
    cp_async_wait<0>();
    if (nch > 0) named_arrive(1 + (int)((nch - 1) % HUB_STAGES), SPMM_THREADS);
}




#define CK(call)                                            \
    do {                                                    \
        cudaError_t _e = (call);                            \
        if (_e != cudaSuccess) return cuda_fail(_e, #call); \
    } while (0)

// Degree-descending row permutation (stable: equal degrees keep ascending ids), the heavy
// prefix (degree > SPMM_SEG) and its segment table: a counting sort by degree on the host over a
// copy of the offsets (once per graph, at the first K9 call).
int build_spmm_plan(er_graph *g, cudaStream_t st)
{
    const int64_t n = g->n;
    std::vector<int64_t> off(n + 1);
    CK(cudaStreamSynchronize(st));
    CK(cudaMemcpy(off.data(), g->d_off, sizeof(int64_t) * (n + 1), cudaMemcpyDeviceToHost));
    int64_t md = 0;
    for (int64_t v = 0; v < n; v++) md = std::max<int64_t>(md, off[v + 1] - off[v]);
    std::vector<int64_t> pos(md + 2, 0);   // pos[d] = first slot of degree d (descending order)
    for (int64_t v = 0; v < n; v++) pos[off[v + 1] - off[v]]++;
    int64_t run = 0;
    for (int64_t d = md; d >= 0; d--) {
        const int64_t c = pos[d];
        pos[d] = run;
        run += c;
    }
    std::vector<int32_t> perm(n);
    for (int64_t v = 0; v < n; v++) perm[pos[off[v + 1] - off[v]]++] = (int32_t)v;
    int64_t nh = 0;
    while (nh < n && off[perm[nh] + 1] - off[perm[nh]] > SPMM_SEG) nh++;
    std::vector<int64_t> hseg(nh + 1, 0), seg_e0;
    std::vector<int32_t> seg_row;
    for (int64_t h = 0; h < nh; h++) {
        const int32_t v = perm[h];
        const int64_t d = off[v + 1] - off[v], ns = (d + SPMM_SEG - 1) / SPMM_SEG;
        hseg[h + 1] = hseg[h] + ns;
        for (int64_t p = 0; p < ns; p++) {
            seg_e0.push_back(off[v] + p * SPMM_SEG);
            seg_row.push_back(v);
        }
    }
    CK(cudaMalloc(&g->d_rowperm, sizeof(int32_t) * n));
    CK(cudaMemcpy(g->d_rowperm, perm.data(), sizeof(int32_t) * n, cudaMemcpyHostToDevice));
    g->n_heavy = nh;
    g->n_seg = (int64_t)seg_e0.size();
    if (nh > 0) {
        CK(cudaMalloc(&g->d_hseg, sizeof(int64_t) * (nh + 1)));
        CK(cudaMalloc(&g->d_seg_e0, sizeof(int64_t) * g->n_seg));
        CK(cudaMalloc(&g->d_seg_row, sizeof(int32_t) * g->n_seg));
        CK(cudaMemcpy(g->d_hseg, hseg.data(), sizeof(int64_t) * (nh + 1), cudaMemcpyHostToDevice));
        CK(cudaMemcpy(g->d_seg_e0, seg_e0.data(), sizeof(int64_t) * g->n_seg, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(g->d_seg_row, seg_row.data(), sizeof(int32_t) * g->n_seg, cudaMemcpyHostToDevice));
    }
    // item descriptors of k_spmm_items: the segments, then the light rows (degree-descending)
    {
        const int64_t ni = g->n_seg + (n - nh);
        std::vector<int4> desc(std::max<int64_t>(ni, 1));
        auto mk = [](int64_t e0, int64_t len, int32_t dst) {
            return make_int4((int)(uint32_t)(uint64_t)e0, (int)(uint32_t)((uint64_t)e0 >> 32), (int)len, dst);
        };
        for (int64_t p = 0; p < g->n_seg; p++) {
            const int32_t v = seg_row[p];
            desc[p] = mk(seg_e0[p], std::min<int64_t>(SPMM_SEG, off[v + 1] - seg_e0[p]), (int32_t)(-1 - p));
        }
        for (int64_t r = nh; r < n; r++) {
            const int32_t v = perm[r];
            desc[g->n_seg + (r - nh)] = mk(off[v], off[v + 1] - off[v], v);
        }
        CK(cudaMalloc(&g->d_spmm_desc, sizeof(int4) * desc.size()));
        CK(cudaMemcpy(g->d_spmm_desc, desc.data(), sizeof(int4) * desc.size(), cudaMemcpyHostToDevice));
    }
    return ER_OK;
}

// Light rows (and, unless exact, the heavy-row segments) through k_spmm_rows.
template <int VEC>
void launch_rows(er_graph *g, const double *X, double *Y, double *part, int32_t q, int normalize, bool exact,
                 cudaStream_t st)
{
    const int nvec = q / VEC;
    int lpr = 1;
    while (lpr < nvec && lpr < 32) lpr <<= 1;
    const int64_t nseg = exact ? 0 : g->n_seg;
    const int64_t nitems = nseg + (g->n - g->n_heavy);
    if (nitems == 0) return;
    if (SPMM_PIPE && nvec <= lpr) {   // one column vector per lane: the pipelined item kernel
        const int4 *desc = g->d_spmm_desc + (exact ? g->n_seg : 0);
        const unsigned pgrid = (unsigned)std::min<int64_t>(blocks_for(nitems * lpr, SPMM_THREADS),
                                                           (int64_t)g->num_sms * SPMM_MINB);
#define P(LPR)                                                                                                  \
    k_spmm_items<LPR, VEC><<<pgrid, SPMM_THREADS, 0, st>>>(nitems, desc, g->d_cols, X, Y, part, q, normalize)
        switch (lpr) {
            case 1: P(1); break;
            case 2: P(2); break;
            case 4: P(4); break;
            case 8: P(8); break;
            case 16: P(16); break;
            default: P(32); break;
        }
#undef P
        g->launches++;
        return;
    }
    const unsigned grid = blocks_for(nitems * lpr, SPMM_THREADS);
#define L(LPR)                                                                                               \
    k_spmm_rows<LPR, VEC><<<grid, SPMM_THREADS, 0, st>>>(nseg, nitems, g->d_seg_e0, g->d_seg_row,              \
                                                         g->d_rowperm + g->n_heavy, g->d_off, g->d_cols, X, Y, \
                                                         part, q, normalize)
    switch (lpr) {
        case 1: L(1); break;
        case 2: L(2); break;
        case 4: L(4); break;
        case 8: L(8); break;
        case 16: L(16); break;
        default: L(32); break;
    }
#undef L
    g->launches++;
}

}  // namespace

int run_spmm(er_graph *g, const double *X, double *Y, int32_t q, int32_t normalize, cudaStream_t st, bool exact)
{
    NvtxRange nvtx_("geer/spmm");
    if (!g->d_rowperm) {
        const int rc = build_spmm_plan(g, g->stream);
        if (rc) return rc;
    }
    const bool vec2 = (q % 2 == 0) && ((reinterpret_cast<uintptr_t>(X) | reinterpret_cast<uintptr_t>(Y)) % 16 == 0);
    double *part = nullptr;
    if (!exact && g->n_seg > 0) {
        CK(g->ws.spmm_part.ensure(sizeof(double) * (size_t)g->n_seg * q, false, st));
        part = g->ws.spmm_part.as<double>();
    }
    if (exact && g->n_heavy > 0) {
        // heavy rows on a forked stream, concurrent with the light rows (their longest chains
        // would otherwise be the kernel's tail)
        if (!g->spmm_stream) {
            CK(cudaStreamCreateWithFlags(&g->spmm_stream, cudaStreamNonBlocking));
            CK(cudaEventCreateWithFlags(&g->spmm_fork, cudaEventDisableTiming));
            CK(cudaEventCreateWithFlags(&g->spmm_join, cudaEventDisableTiming));
        }
        CK(cudaEventRecord(g->spmm_fork, st));
        CK(cudaStreamWaitEvent(g->spmm_stream, g->spmm_fork, 0));
        const size_t smem = sizeof(double) * HUB_STAGE * HUB_STAGES;
#define HUB(VEC, CB)                                                                                          \
    do {                                                                                                      \
        const dim3 grid((unsigned)g->n_heavy, (unsigned)((q + CB - 1) / CB));                                 \
        CK(cudaFuncSetAttribute(k_spmm_hub_exact<VEC, CB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); \
        k_spmm_hub_exact<VEC, CB><<<grid, SPMM_THREADS, smem, g->spmm_stream>>>(g->d_rowperm, g->d_off, g->d_cols, \
                                                                               X, Y, q, normalize);        \
    } while (0)
        if (vec2) {
            if (g->hub_cb == 32) HUB(2, 32);
            else if (g->hub_cb == 16) HUB(2, 16);
            else HUB(2, 8);
        } else {
            if (g->hub_cb == 32) HUB(1, 32);
            else if (g->hub_cb == 16) HUB(1, 16);
            else HUB(1, 8);
        }
#undef HUB
        g->launches++;
        CK(cudaEventRecord(g->spmm_join, g->spmm_stream));
    }
    if (vec2) launch_rows<2>(g, X, Y, part, q, normalize, exact, st);
    else launch_rows<1>(g, X, Y, part, q, normalize, exact, st);
    if (!exact && g->n_heavy > 0) {
        k_spmm_heavy_sum<<<blocks_for(g->n_heavy * q, 256), 256, 0, st>>>(g->n_heavy, g->d_rowperm, g->d_hseg,
                                                                          g->d_off, part, Y, q, normalize);
        g->launches++;
    }
    if (exact && g->n_heavy > 0) CK(cudaStreamWaitEvent(st, g->spmm_join, 0));
    CK(cudaGetLastError());
    return ER_OK;
}

}  // namespace geer

// ============================================================================ SMM-to-ell series
namespace geer {
namespace {

// X[:, c] = e_s/d_s - e_t/d_t for the block's queries (X zeroed before).
__global__ void k_series_init(int32_t q, const int32_t *__restrict__ pairs, const int64_t *__restrict__ off,
                              double *__restrict__ X)
{
    const int32_t c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= q) return;
    const int32_t s = pairs[2 * c], t = pairs[2 * c + 1];
    if (s == t) return;
    X[(int64_t)s * q + c] = 1.0 / (double)(off[s + 1] - off[s]);
    X[(int64_t)t * q + c] = -1.0 / (double)(off[t + 1] - off[t]);
}

// acc[c] += y_i(s) - y_i(t) while i <= L_c (series term i of Thm 3.1's r_L).
__global__ void k_series_acc(int32_t q, int32_t i, const int32_t *__restrict__ pairs, const int32_t *__restrict__ ell,
                             const double *__restrict__ X, double *__restrict__ acc)
{
    const int32_t c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= q || i > ell[c]) return;
    const int32_t s = pairs[2 * c], t = pairs[2 * c + 1];
    if (s == t) return;
    acc[c] += X[(int64_t)s * q + c] - X[(int64_t)t * q + c];
}

}  // namespace

int run_smm_series(er_graph *g, const int32_t *pairs, int64_t k, double tol, int32_t max_iters, double *out_r,
                   int32_t *ells)
{
    NvtxRange nvtx_("geer/smm_series");
    const int64_t n = g->n;
    const int32_t QB = 64;
    cudaStream_t st = g->stream;
    // L per query on the host: Eq. 6 with eps = tol; natural log (R2), clamp at 0 (R3)
    std::vector<int32_t> L(k);
    std::vector<int64_t> off_s(2), off_t(2);
    const double lam = g->lambda;
    for (int64_t i = 0; i < k; i++) {
        const int32_t s = pairs[2 * i], t = pairs[2 * i + 1];
        if (s == t) { L[i] = -1; continue; }
        CK(cudaMemcpy(off_s.data(), g->d_off + s, 2 * sizeof(int64_t), cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(off_t.data(), g->d_off + t, 2 * sizeof(int64_t), cudaMemcpyDeviceToHost));
        const double ds = (double)(off_s[1] - off_s[0]), dt = (double)(off_t[1] - off_t[0]);
        const double x = std::log((2.0 / ds + 2.0 / dt) / (tol * (1.0 - lam))) / std::log(1.0 / lam) - 1.0;
        double c = std::ceil(x);
        if (c < 0.0) c = 0.0;
        L[i] = (int32_t)std::min<double>(c, (double)max_iters);
    }
    double *X = nullptr, *Y = nullptr, *acc = nullptr;
    int32_t *dp = nullptr, *dl = nullptr;
    CK(cudaMalloc(&X, sizeof(double) * n * QB));
    CK(cudaMalloc(&Y, sizeof(double) * n * QB));
    CK(cudaMalloc(&acc, sizeof(double) * QB));
    CK(cudaMalloc(&dp, sizeof(int32_t) * 2 * QB));
    CK(cudaMalloc(&dl, sizeof(int32_t) * QB));
    int rc = ER_OK;
    for (int64_t b0 = 0; b0 < k && rc == ER_OK; b0 += QB) {
        const int32_t q = (int32_t)std::min<int64_t>(QB, k - b0);
        int32_t Lmax = -1;
        for (int32_t c = 0; c < q; c++) Lmax = std::max(Lmax, L[b0 + c]);
        cudaMemcpyAsync(dp, pairs + 2 * b0, sizeof(int32_t) * 2 * q, cudaMemcpyHostToDevice, st);
        cudaMemcpyAsync(dl, L.data() + b0, sizeof(int32_t) * q, cudaMemcpyHostToDevice, st);
        cudaMemsetAsync(X, 0, sizeof(double) * n * q, st);
        cudaMemsetAsync(acc, 0, sizeof(double) * q, st);
        k_series_init<<<1, QB, 0, st>>>(q, dp, g->d_off, X);
        g->launches++;
        double *cur = X, *nxt = Y;
        for (int32_t i = 0; i <= Lmax; i++) {
            k_series_acc<<<1, QB, 0, st>>>(q, i, dp, dl, cur, acc);
            g->launches++;
            if (i == Lmax) break;
            rc = run_spmm(g, cur, nxt, q, 1, st);   // y_{i+1} = P y_i (K9)
            if (rc) break;
            std::swap(cur, nxt);
        }
        if (rc == ER_OK) {
            cudaError_t e = cudaMemcpyAsync(out_r + b0, acc, sizeof(double) * q, cudaMemcpyDeviceToHost, st);
            if (e == cudaSuccess) e = cudaStreamSynchronize(st);
            if (e != cudaSuccess) rc = cuda_fail(e, "er_smm_series");
        }
    }
    for (int64_t i = 0; i < k; i++) {
        if (L[i] < 0) out_r[i] = 0.0;
        if (ells) ells[i] = std::max(L[i], 0);
    }
    cudaFree(X);
    cudaFree(Y);
    cudaFree(acc);
    cudaFree(dp);
    cudaFree(dl);
    return rc;
}

}  // namespace geer
