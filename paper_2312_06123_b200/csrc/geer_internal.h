// geer_internal.h -- internal declarations shared by the libgeer.so translation units.
// Product code only: nothing here is shared with oracle/ (see DESIGN.md "Independence").
#pragma once

#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>
#include <stdint.h>

#include <atomic>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/geer.h"

namespace geer {

// K9: rows of degree > SPMM_SEG are summed in segments of SPMM_SEG neighbours (spmm.cu).
constexpr int SPMM_SEG = 512;

// Query phases.
enum : int32_t { PH_DONE = 0, PH_SMM = 1, PH_AMC = 2 };

// Per-query device state (AoS; one thread/warp per query touches it).
struct QState {
    er_query_stats st;     // public diagnostics, copied out at the end
    int32_t s, t;          // query endpoints
    uint32_t gq;           // global query index (RNG key, R10): query_index_base + i or query_ids[i]
    int32_t pad3;
    int32_t ds, dt;        // degrees d(s), d(t)
    int32_t phase;         // PH_*
    int32_t ylog2;         // log2 of the y-table capacity in slots (>= 3)
    int32_t ymode;         // y-table layout: 0 hash (ykeys, ylog2), 1 rank bitmap (yrec)
    int32_t pad2;
    const int32_t *ykeys;  // hash keys (YT_HASH)
    const uint4 *yrec;     // rank records {U bits 0-31, 32-63, 64-95, rank U} per 96 node ids (YT_RANK)
    const double *yvals;   // values (by slot, or by rank)
    double z;              // last batch mean Z (= r_f)
    double s1acc, s2acc;   // running sums of Z_k, Z_k^2 (reuse variant)
};


// 64-bit packed arc record: u | offset(u) | degree(u) in bu + bo + bd <= 64 bits.
// Degree-ordered walk graph (K6 layout 4): nodes renumbered by descending degree
// (ties by id), each maximal run of equal degree ("class" c, degree d_c) padded to a multiple of
// 2^bshift ids, so every block of 2^bshift new ids lies inside one class and its rows are
// contiguous in the renumbered CSR: off(v) = base_c + (v - vstart_c) d_c.  K6 stages blk (class of
// each block, u16) and cd (per class {base_c - vstart_c d_c mod 2^32, d_c}) in shared memory and
// gets (off, d) of v from two shared loads instead of a dependent global load of v's node
// record.  perm: old id -> new id; iperm: new id -> old id (-1 on padding); nv: new id space.
struct DOrdView {
    const int32_t *perm = nullptr;
    const int32_t *iperm = nullptr;
    const uint16_t *blk = nullptr;   // [nblk]
    const uint2 *cd = nullptr;       // [ncls]
    int32_t nblk = 0, ncls = 0, bshift = 0;
};
constexpr int DORD_SMEM_BYTES = 24 * 1024;   // default shared memory per K6 CTA for blk + cd

struct PackSpec {
    int bo = 0, bd = 0;  // bit widths of offset and degree (u takes the high bits)
    __host__ __device__ unsigned long long pack(uint32_t u, uint32_t off, uint32_t deg) const
    {
        return ((unsigned long long)u << (bo + bd)) | ((unsigned long long)off << bd) | (unsigned long long)deg;
    }
    __host__ __device__ uint4 unpack(unsigned long long a) const
    {
        uint4 r;
        r.z = (uint32_t)(a & ((1ull << bd) - 1));
        r.y = (uint32_t)((a >> bd) & ((1ull << bo) - 1));
        r.x = (uint32_t)(a >> (bo + bd));
        r.w = 0;
        return r;
    }
};

// Per-segment statistics of an SMM iterate (segment = one side of one query).
struct SegStat {
    int64_t vol;           // sum of d(v) over the support (Eq. 15 left side)
    double max1, max2;     // top-2 entries (R5); accumulated as uint64 bit patterns (x >= 0)
    double at_s, at_t;     // x(s), x(t) of the segment's query
    unsigned long long n_max1;  // occurrences of max1
};

// Per-tile partial sums of one AMC batch (tile = 32 walk pairs of one query).
struct TilePart {
    double s1, s2;         // sum Z_k, sum Z_k^2 over the tile's lanes
    uint64_t ck;           // walk checksum partial
    uint64_t pad;
};

// Scalars every kernel of a batch needs (passed by value).
struct BatchParams {
    double eps, delta, lambda;
    double log_inv_lambda;  // log(1/lambda), host-computed
    double L_eta;           // log(2 tau / delta), host-computed (Eq. 9)
    double L_bern;          // log(3 / (delta / tau)), host-computed (Eq. 8 with delta/tau)
    int32_t tau;
    int32_t force_ell_b;
    int32_t ell_variant;
    int32_t reuse;          // variant: keep samples across batches
    double switch_ratio;    // variant: Eq. 15 threshold multiplier
    int32_t nbits;          // bits of a node id (sort keys)
    uint64_t seed;
    int64_t qbase;          // global index of query 0
    int64_t n;
};

// NVTX range for the host-side stages (visible in nsys / ncu --nvtx; a no-op without a tool
// attached): "geer/batch", "geer/smm_wave", "geer/ytable", "geer/amc", "geer/spmm", ...
struct NvtxRange {
    explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange &) = delete;
    NvtxRange &operator=(const NvtxRange &) = delete;
};

// Grow-only device buffer.
struct DevBuf {
    void *p = nullptr;
    size_t cap = 0;
    cudaError_t ensure(size_t bytes, bool keep, cudaStream_t st);
    template <class T> T *as() const { return reinterpret_cast<T *>(p); }
    void release();
};

struct Workspace {
    DevBuf qs, pairs, out, stats;
    DevBuf act, act2, cont, idx, cont2, idx2;       // active lists / flags / scan outputs
    DevBuf fr_id, fr_val, fr_seg, fr_off;           // current frontier
    DevBuf nf_id, nf_val, nf_seg, nf_off;           // next frontier
    DevBuf ent_off;                                 // emission offsets per frontier entry
    DevBuf keys, vals, keys2, vals2;                // emitted (key, value) pairs + sort buffers
    DevBuf runstart;                                // run-length reduction: first pair of each run
    DevBuf segstat;                                 // SegStat per segment
    DevBuf ycap, yoff;                              // y-table sizes and their scans (per leaving query)
    DevBuf ydesc;                                   // K5 build-time table descriptors (per leaving query)
    DevBuf ywid;                                    // K5: walk ids of the frontier entries (layout 4)
    DevBuf cub_tmp;                                 // CUB temp storage
    DevBuf scalars;                                 // small device scalars
    DevBuf spmm_part;                               // K9 heavy-row segment sums
    DevBuf dense_x, dense_y, dense_cnt;             // SMM dense mode: n x q blocks, per-tile counts
    DevBuf qids;                                    // device copy of er_opts.query_ids
    std::vector<DevBuf> ychunk;                     // y-tables of each SMM wave (grow-only, kept)
    DevBuf ids, seglen, segbeg;                     // 0..k-1 ids; compaction lengths; sort segments
    DevBuf pk_seg, pk_bkt, pk_keys, pk_alt, pk_out; // SMM push (smm_push.cu): plan, buckets, keys, outputs
    int64_t pk_nbmax = 0, pk_e = 0, pk_F = 0;       // the current push chunk's bucket bound and pair count,
                                                    // the wave's frontier entry count
    void *host_pinned = nullptr;                    // small pinned host scalars
    size_t host_pinned_cap = 0;
    void release();
};

}  // namespace geer

struct er_graph {
    int device = 0;
    int num_sms = 148;            // multiprocessors of the device (set at creation)
    int64_t n = 0, nnz = 0;
    int64_t *d_off = nullptr;
    int32_t *d_cols = nullptr;
    uint2 *d_rec = nullptr;       // {offset, degree} per node (offsets < 2^32)
    uint4 *d_arcs = nullptr;      // {u, offset(u), degree(u), 0} per arc, in CSR order (walk chain)
    unsigned long long *d_parcs = nullptr;  // packed 8-byte arc records (when they fit 64 bits)
    uint4 *d_c24 = nullptr;       // 24-bit columns, 5 per 16-byte chunk (DRAM-resident graphs with n < 2^24)
    // degree-ordered walk graph (layout 4): d_c24 then holds the renumbered CSR's columns
    int32_t *d_perm = nullptr, *d_iperm = nullptr;
    uint16_t *d_cblk = nullptr;
    uint2 *d_ccd = nullptr;
    int32_t dord_nblk = 0, dord_ncls = 0, dord_bshift = 0;
    float walk_l2_keep = 0.f;   // K6 column loads: fraction of lines L2 evict-last (rest evict-first)
    int64_t dord_nv = 0;   // new id space (n plus class padding)
    int32_t dord_smem_bytes = geer::DORD_SMEM_BYTES;   // budget for blk + cd (GEER_DORD_SMEM_KB)
    geer::PackSpec pack;
    int32_t max_deg = 0;
    bool rows_sorted = false;
    int query_block = 0;  // ER_OK, or the validation code that forbids queries (ER_CREATE_SPMM_ONLY)
    double lambda = 0.0;
    bool lambda_set = false;
    int nbits = 1;
    int walk_minb = 4;   // K6 resident CTAs per SM (launch bounds variant; GEER_WALK_MINB 3..4)
    double overlap_frac = 0.75;  // overlap mode: fraction of K6 resident-CTA slots (GEER_OVERLAP_FRAC)
    bool amc_overlap = false;  // AMC per SMM wave on the AMC stream (GEER_AMC_OVERLAP=1) or one AMC after the head
    int walk_occ = 0;    // K6 resident CTAs per SM at the last launch (occupancy API)
    bool walk_persist = true;   // K6 persistent grid + atomic tile counter (GEER_WALK_PERSIST=1) or one tile per CTA
    int64_t rank_min_cap = 4096;  // K5: rank bitmap only for tables above this many hash slots (GEER_RANK_MIN_CAP)
    int64_t rank_ratio = 12;      // ... and when 16 B x records < rank_ratio x slots (GEER_RANK_RATIO)
    int64_t rank_max_bytes = 960 << 10;  // ... and when the records take at most this, i.e. walk ids up to
                                         // ~5.9M (96 per record; GEER_RANK_MAX_KB; configs 1-4)
    int ytable_force = 0;  // y-table layout: 0 by footprint, 1 hash only, 2 rank bitmap only (GEER_YTABLE)
    bool l2_persist = false; // K6: persisting-L2 access window over the walk graph (GEER_L2_PERSIST)
    size_t l2_window = 0, l2_persist_bytes = 0;
    int64_t max_sub_batch = 1 << 18;  // queries per internal sub-batch (GEER_MAX_SUB_BATCH)
    int64_t wave_pairs_max = (int64_t)1 << 28;  // SMM push: pairs per chunk of a wave (GEER_WAVE_PAIRS_MAX)
    int walk_np = 1;     // K6 walk pairs per thread (GEER_WALK_NP 1..2)
    int walk_smem_words = 0;      // K6 staging area per CTA in 32-bit words (GEER_WALK_SMEM_KB; default none:
                                  // shared memory taken from L1 costs more walk throughput than staging saves)
    bool walk_tiles = false;      // K6: CTA-tiles of 8 chunks even without staging (GEER_WALK_TILES=1)
    int walk_carveout = -1;       // K6 preferred shared-memory carveout in % (-1: driver default; GEER_WALK_CARVEOUT)
    cudaStream_t stream = nullptr;
    cudaStream_t amc_stream = nullptr;  // AMC groups overlap the SMM head
    cudaStream_t head_stream = nullptr; // high-priority stream of the SMM head (forked from the caller's)
    cudaEvent_t ev_in = nullptr, ev_out = nullptr;  // fork / join with the caller's stream
    cudaStream_t ybuild_stream = nullptr;  // K5 y-table builds concurrent with the next SMM wave
    cudaEvent_t ev_yfork = nullptr, ev_ydone = nullptr;
    std::mutex mu;
    int64_t launches = 0;
    bool profiling = false;
    er_profile prof{};
    int64_t *d_steps = nullptr;  // device walk-step counter (profiling)
    int32_t *d_rowperm = nullptr;  // K9: rows by descending degree (built at the first er_spmm)
    int64_t n_heavy = 0;           // K9: rows with degree > SPMM_SEG (the prefix of d_rowperm)
    int64_t n_seg = 0;             // K9: segments of the heavy rows
    int64_t *d_hseg = nullptr;     // K9: first segment of each heavy row (n_heavy + 1)
    int64_t *d_seg_e0 = nullptr;   // K9: first arc of each segment
    int32_t *d_seg_row = nullptr;  // K9: row of each segment
    int4 *d_spmm_desc = nullptr;   // K9: work items {first arc (2 words), length, row | -1 - segment}
    int hub_cb = 32;                     // K9 exact: columns per heavy-row CTA (GEER_HUB_CB 8/16/32)
    cudaStream_t spmm_stream = nullptr;  // K9 exact: heavy rows concurrent with the light rows
    cudaEvent_t spmm_fork = nullptr, spmm_join = nullptr;
    geer::Workspace ws;
};

namespace geer {

void set_error(int code, const std::string &msg);
// ER_ENOMEM fault injection (pipeline.cu): the g_fault_target-th workspace growth fails.
extern std::atomic<int64_t> g_fault_target, g_fault_count;
int cuda_fail(cudaError_t e, const char *what);

// Pipeline entry (pipeline.cu).
int run_query_batch(er_graph *g, const int32_t *pairs, int64_t k, double eps, double p_fail,
                    const er_opts &o, double *out_r, er_query_stats *stats);
// K9: Y = M X (spmm.cu).  exact = every row summed sequentially in CSR order (heavy rows too).
int run_spmm(er_graph *g, const double *X, double *Y, int32_t q, int32_t normalize, cudaStream_t st,
             bool exact = false);
int run_smm_series(er_graph *g, const int32_t *pairs, int64_t k, double tol, int32_t max_iters, double *out_r,
                   int32_t *ells);
int run_estimate_lambda(er_graph *g, int iters, double *lambda_out);
cudaError_t build_arcs(er_graph *g);
cudaError_t build_parcs(er_graph *g);
cudaError_t build_c24(er_graph *g);
// layout 4 from the host CSR (offsets, cols): 1 = not applicable (too many degree classes, n or
// nnz too large), 0 = built, < 0 = CUDA / host allocation failure
int build_dord(er_graph *g, const int64_t *offsets, const int32_t *cols);
// Device validation of the uploaded CSR (validate.cu): 1 = the host validation must decide.
int validate_device(er_graph *g, int *code, std::string *msg, int *spectral, bool *rows_sorted, int32_t *max_deg);

}  // namespace geer
