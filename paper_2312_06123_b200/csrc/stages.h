// stages.h -- host-side helpers and stage entry points shared by the query-pipeline translation
// units: pipeline.cu (K1-K4, K8 and run_query_batch), ytable.cu (K5), walks.cu (K6, K7).
#pragma once


#include <algorithm>
#include <initializer_list>
#include <vector>

#include "geer_device.cuh"
#include "geer_internal.h"
#include "scan.cuh"

namespace geer {

#define CK(call)                                            \
    do {                                                    \
        cudaError_t _e = (call);                            \
        if (_e != cudaSuccess) return cuda_fail(_e, #call); \
    } while (0)

#define LAUNCHED(g) ((g)->launches++)

static inline unsigned blocks_for(int64_t n, int per) { return (unsigned)((n + per - 1) / per); }

// Grid of a grid-stride kernel over at most n items: one wave of resident CTAs (2048 threads
// per SM), fewer when n is small.
static inline unsigned resident_grid(const er_graph *g, int64_t n, int threads)
{
    const int64_t full = (int64_t)g->num_sms * (2048 / threads);
    return (unsigned)std::max<int64_t>(1, std::min<int64_t>(full, (n + threads - 1) / threads));
}

// y-table layouts (ytable.cu) and the walk kernel's staging limits (walks.cu).
constexpr int YT_HASH = 0;
constexpr int YT_RANK = 1;
constexpr int WALK_KEY_SLOTS = 4096;        // largest hash table staged in shared memory

// Rank-bitmap records: one 16-byte record {U bits 0-31, 32-63, 64-95; rank U} per RANK_IDS = 96
// consecutive node ids (three 32-id words and the number of U members before the record).
constexpr uint32_t RANK_IDS = 96;
__device__ __forceinline__ uint32_t rank_rec(int32_t v) { return (uint32_t)v / RANK_IDS; }
// Position of y(v) in the value array, or -1 when v is not in U (r = v's record).
__device__ __forceinline__ int64_t rank_index(const uint4 r, int32_t v)
{
    const uint32_t b = (uint32_t)v - RANK_IDS * rank_rec(v), wd = b >> 5, m = 1u << (b & 31u);
    const uint32_t word = wd == 0 ? r.x : wd == 1 ? r.y : r.z;
    if (!(word & m)) return -1;
    return (int64_t)r.w + __popc(word & (m - 1u)) + (wd > 0 ? __popc(r.x) : 0) + (wd > 1 ? __popc(r.y) : 0);
}

// Walk pairs of AMC batch b: the first walk index drawn in batch b -- all eta_b = eta0 2^b fresh
// (R8), or, with sample reuse (R23), only the eta_b - eta_{b-1} new ones k in [eta_{b-1}, eta_b).
__device__ __forceinline__ int64_t walks_lo(int64_t eta0, int b, int reuse) { return reuse && b > 0 ? eta0 << (b - 1) : 0; }

struct Ctx {
    er_graph *g;
    cudaStream_t st;
    Workspace &ws;
    int64_t *hp;  // pinned host scalars
};

#define ENSURE(buf, bytes, keep) CK((buf).ensure((bytes), (keep), c.st))

// Device-wide scans (scan.cuh) with the workspace's scan temporary (head stream only: the AMC and
// y-build streams bring their own temporaries).
template <class T, class Op>
int scan_op(Ctx &c, const T *in, T *out, int64_t n, T zero, Op op)
{
    if (n <= 0) return ER_OK;
    ENSURE(c.ws.cub_tmp, scan_tmp_bytes<T>(n), false);
    c.g->launches += scan_launch(c.st, in, out, n, zero, op, c.ws.cub_tmp.p);
    CK(cudaGetLastError());
    return ER_OK;
}

// out[0] = 0, out[1..n] = inclusive prefix sums of in[0..n).
template <class T>
int scan_offsets(Ctx &c, const T *in, T *out, int64_t n)
{
    CK(cudaMemsetAsync(out, 0, sizeof(T), c.st));
    return scan_op(c, in, out + 1, n, (T)0, ScanAdd<T>());
}

template <class T>
int scan_incl(Ctx &c, const T *in, T *out, int64_t n)
{
    return scan_op(c, in, out, n, (T)0, ScanAdd<T>());
}

inline int read_scalars(Ctx &c, std::initializer_list<const int64_t *> src)
{
    int j = 0;
    for (const int64_t *p : src) {
        CK(cudaMemcpyAsync(c.hp + j, p, sizeof(int64_t), cudaMemcpyDeviceToHost, c.st));
        j++;
    }
    CK(cudaStreamSynchronize(c.st));
    return ER_OK;
}

// K5 (ytable.cu).  Build the y-tables of the queries of `act` that leave the head now, from the
// frontier (segoff, id, val, seg; Fmax entries, device count dF or null).  `cont` may be null (all
// queries of the list leave).  The tables of SMM wave `wave` live in a grow-only workspace
// buffer kept across batches: {vals fp64[V] | rank records uint4[R] | aux uint4[R] | hash keys
// int32[H]}; QState holds absolute pointers into it.
// Phase 1 (no host sync): per-query sizes and their inclusive scans; the three totals are at
// *tot_h, *tot_v, *tot_r (device) for the caller to read with its other scalars.
int ytable_plan(Ctx &c, int32_t na, const int32_t *act, const int32_t *cont, const int64_t *segoff,
                const int64_t **tot_h, const int64_t **tot_v, const int64_t **tot_r);
// Phase 2: allocate and fill the tables planned by ytable_plan (totals H, V, R read by the caller).
int ytable_build(Ctx &c, int32_t na, const int32_t *act, const int64_t *segoff, const int32_t *id, const double *val,
                 const int32_t *seg, int64_t Fmax, const int64_t *dF, int wave, int64_t H, int64_t V, int64_t R);
// Both phases with one host read in between.
int build_ytables(Ctx &c, int32_t na, const int32_t *act, const int32_t *cont, const int64_t *segoff,
                  const int32_t *id, const double *val, const int32_t *seg, int64_t Fmax, const int64_t *dF,
                  int wave);

// SMM dense mode (dense.cu): whether a wave of na queries emitting E push pairs runs dense, and
// the wave itself: frontier (ws.fr_*) -> next frontier (ws.nf_*, sized >= E by the caller) with
// the K4a statistics in ws.segstat (zeroed by the caller) and the entry count at *dU (device).
constexpr double DENSE_PUSH_NS_PER_PAIR = 0.1;   // measured push cost per emitted pair
constexpr double DENSE_BYTES_PER_NS = 2500.0;    // effective bandwidth of a dense wave (conservative)
constexpr double DENSE_MAX_BYTES = 16.0 * (1ull << 30);   // X + Y blocks
bool dense_wave_pays(const er_graph *g, int32_t na, int64_t E);
int smm_dense_wave(Ctx &c, int32_t na, int64_t F, const int32_t *act, int64_t *dU);

// SMM push wave (smm_push.cu): part A (plan, count, scatter, reduce; push workspaces only) and
// part B (merge, gather: ws.segstat, ws.nf_*, ws.nf_off, *dU), see the file's header.
// A wave's queries are pushed in chunks of whole queries (segments [g0, g0 + ns), pairs
// [P0, P0 + E)) whose pair count stays within er_graph::wave_pairs_max (GEER_WAVE_PAIRS_MAX), so
// the workspaces stay bounded; chunks are independent (wave splitting).  ws.pk_F = the
// frontier's entry count.
int smm_push_wave_a(Ctx &c, int32_t g0, int32_t ns, int64_t P0, int64_t E, const int64_t *ent_off);
int smm_push_wave_b(Ctx &c, int32_t g0, int32_t ns, int64_t *dU);

// K6 + K7 (walks.cu).  One AMC group: the queries that left the SMM head in the same wave, with
// their y-tables.  Its whole AMC (tau batches) is enqueued on stream sb without host sync.
struct AmcGroup {
    int32_t na = 0;
    int32_t *list = nullptr;     // query ids (device)
    unsigned long long eta0_sum = 0;
};

struct BatchRes {
    std::vector<void *> bufs;          // stream-ordered allocations freed at the end of the batch
    std::vector<cudaEvent_t> walk_ev;  // profiling: start/end pairs of walk launches
};

int launch_amc_group(er_graph *g, cudaStream_t sb, const AmcGroup &G, QState *qs, const BatchParams &P, bool prof,
                     BatchRes &R);

}  // namespace geer
