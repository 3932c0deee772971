// abi.cu -- the extern "C" boundary of libgeer.so (include/geer.h).
// Argument checking, error codes, graph creation/validation, handle lifetime.

#include <omp.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "geer_internal.h"

namespace geer {

static thread_local int t_code = ER_OK;
static thread_local std::string t_msg = "ok";

void set_error(int code, const std::string &msg)
{
    t_code = code;
    t_msg = msg;
}

int cuda_fail(cudaError_t e, const char *what)
{
    const int code = (e == cudaErrorMemoryAllocation) ? ER_ENOMEM : ER_ECUDA;
    set_error(code, std::string(what) + ": " + cudaGetErrorString(e));
    cudaGetLastError();
    return code;
}

static void clear_error()
{
    t_code = ER_OK;
    t_msg = "ok";
}

// The checks that need no pass over the columns (host, before the upload).
static int validate_basic(int64_t n, const int64_t *off, const int32_t *cols)
{
    if (n < 2 || n > (int64_t)INT32_MAX) {
        set_error(ER_EINVAL, "n must be in [2, 2^31-1]");
        return ER_EINVAL;
    }
    if (!off || !cols) {
        set_error(ER_EINVAL, "offsets/cols must be non-NULL");
        return ER_EINVAL;
    }
    if (off[0] != 0) {
        set_error(ER_EINVAL, "offsets[0] != 0");
        return ER_EINVAL;
    }
    for (int64_t v = 0; v < n; v++) {
        if (off[v + 1] < off[v]) {
            set_error(ER_EINVAL, "offsets not non-decreasing at node " + std::to_string(v));
            return ER_EINVAL;
        }
    }
    if (off[n] >= ((int64_t)1 << 32)) {
        set_error(ER_EINVAL, "graphs with 2^32 or more arcs are not supported (32-bit node records)");
        return ER_EINVAL;
    }
    return ER_OK;
}

// Host-side validation of the CSR (graph creation is not on the query path; the
// paper also loads and preprocesses graphs outside its timings).  The device
// validation (validate.cu) hands graphs with unsorted rows, or very deep BFS trees, to this one.
static int validate(int64_t n, const int64_t *off, const int32_t *cols, bool *rows_sorted, int32_t *max_deg,
                    int *spectral_code, bool spmm_only)
{
    if (n < 2 || n > (int64_t)INT32_MAX) {
        set_error(ER_EINVAL, "n must be in [2, 2^31-1]");
        return ER_EINVAL;
    }
    if (!off || !cols) {
        set_error(ER_EINVAL, "offsets/cols must be non-NULL");
        return ER_EINVAL;
    }
    if (off[0] != 0) {
        set_error(ER_EINVAL, "offsets[0] != 0");
        return ER_EINVAL;
    }
    for (int64_t v = 0; v < n; v++) {
        if (off[v + 1] < off[v]) {
            set_error(ER_EINVAL, "offsets not non-decreasing at node " + std::to_string(v));
            return ER_EINVAL;
        }
    }
    const int64_t nnz = off[n];
    if (nnz >= ((int64_t)1 << 32)) {
        set_error(ER_EINVAL, "graphs with 2^32 or more arcs are not supported (32-bit node records)");
        return ER_EINVAL;
    }
    int bad = -1;          // first failure class found
    int64_t bad_node = -1;
    bool sorted = true;
    int32_t md = 0;
#pragma omp parallel for schedule(dynamic, 4096) reduction(&& : sorted) reduction(max : md)
    for (int64_t v = 0; v < n; v++) {
        const int64_t e0 = off[v], e1 = off[v + 1];
        md = std::max(md, (int32_t)(e1 - e0));
        int cls = -1;
        bool row_inc = true;   // strictly increasing: no duplicates possible
        for (int64_t e = e0; e < e1; e++) {
            const int32_t u = cols[e];
            if (u < 0 || u >= n) { cls = 0; break; }
            if (u == v) { cls = 1; break; }
            if (e > e0 && cols[e - 1] >= u) row_inc = false;
        }
        if (!row_inc) sorted = false;
        if (cls < 0 && !row_inc) {
            // duplicates: sorted copy of the row
            std::vector<int32_t> row(cols + e0, cols + e1);
            std::sort(row.begin(), row.end());
            for (size_t i = 1; i < row.size(); i++)
                if (row[i] == row[i - 1]) { cls = 2; break; }
        }
        if (cls >= 0) {
#pragma omp critical
            {
                if (bad < 0 || cls < bad || (cls == bad && v < bad_node)) {
                    bad = cls;
                    bad_node = v;
                }
            }
        }
    }
    if (bad == 0) { set_error(ER_EINVAL, "col id out of range in row " + std::to_string(bad_node)); return ER_EINVAL; }
    if (bad == 1) { set_error(ER_ESELFLOOP, "self-loop at node " + std::to_string(bad_node)); return ER_ESELFLOOP; }
    if (bad == 2) { set_error(ER_EDUP, "duplicate neighbour in row " + std::to_string(bad_node)); return ER_EDUP; }
    // symmetry: every (v,u) has (u,v); rows are searched through sorted copies when unsorted
    std::vector<int32_t> sc;
    const int32_t *S = cols;
    if (!sorted) {
        sc.assign(cols, cols + nnz);
#pragma omp parallel for schedule(dynamic, 4096)
        for (int64_t v = 0; v < n; v++) std::sort(sc.begin() + off[v], sc.begin() + off[v + 1]);
        S = sc.data();
    }
    int64_t asym = -1;
#pragma omp parallel for schedule(dynamic, 4096)
    for (int64_t v = 0; v < n; v++) {
        for (int64_t e = off[v]; e < off[v + 1]; e++) {
            const int32_t u = cols[e];
            if (!std::binary_search(S + off[u], S + off[u + 1], (int32_t)v)) {
#pragma omp critical
                if (asym < 0 || v < asym) asym = v;
                break;
            }
        }
    }
    if (asym >= 0) { set_error(ER_EASYM, "adjacency not symmetric at node " + std::to_string(asym)); return ER_EASYM; }
    // connectivity + 2-colouring: level-synchronous parallel BFS from node 0, then every arc
    // must join levels of different parity (an arc inside one parity class closes an odd cycle)
    std::vector<int32_t> level(n, -1);
    level[0] = 0;
    std::vector<int32_t> frontier{0}, next;
    int64_t visited = 1;
    for (int32_t L = 0; !frontier.empty(); L++) {
        next.clear();
#pragma omp parallel
        {
            std::vector<int32_t> local;
#pragma omp for schedule(dynamic, 256) nowait
            for (int64_t i = 0; i < (int64_t)frontier.size(); i++) {
                const int32_t v = frontier[i];
                for (int64_t e = off[v]; e < off[v + 1]; e++) {
                    const int32_t u = cols[e];
                    int32_t expect = -1;
                    if (__atomic_load_n(&level[u], __ATOMIC_RELAXED) == -1 &&
                        __atomic_compare_exchange_n(&level[u], &expect, L + 1, false, __ATOMIC_RELAXED,
                                                    __ATOMIC_RELAXED))
                        local.push_back(u);
                }
            }
#pragma omp critical
            next.insert(next.end(), local.begin(), local.end());
        }
        visited += (int64_t)next.size();
        frontier.swap(next);
    }
    bool bip = true;
    if (visited == n) {
#pragma omp parallel for schedule(dynamic, 4096) reduction(&& : bip)
        for (int64_t v = 0; v < n; v++)
            for (int64_t e = off[v]; e < off[v + 1]; e++)
                if (((level[v] ^ level[cols[e]]) & 1) == 0) { bip = false; break; }
    }
    *spectral_code = ER_OK;
    if (visited != n) *spectral_code = ER_EDISCONNECTED;
    else if (bip) *spectral_code = ER_EBIPARTITE;
    if (*spectral_code != ER_OK && !spmm_only) {
        if (*spectral_code == ER_EDISCONNECTED) set_error(ER_EDISCONNECTED, "graph is not connected");
        else set_error(ER_EBIPARTITE, "graph is bipartite (lambda = 1)");
        return *spectral_code;
    }
    *rows_sorted = sorted;
    *max_deg = md;
    return ER_OK;
}

}  // namespace geer

using namespace geer;

extern "C" {

int er_last_error(void) { return t_code; }
const char *er_last_error_message(void) { return t_msg.c_str(); }

void er_opts_default(er_opts *o)
{
    if (!o) return;
    std::memset(o, 0, sizeof(*o));
    o->tau = 5;
    o->force_ell_b = -1;
    o->seed = ER_DEFAULT_SEED;
    o->query_index_base = 0;
    o->cuda_stream = nullptr;
    o->pairs_on_device = 0;
    o->out_on_device = 0;
    o->ell_variant = 0;
    o->synchronous = 1;
    o->query_ids = nullptr;
    o->switch_ratio = 1.0;
    o->reuse_samples = 0;
    o->smm_mode = 0;
}

er_graph *er_graph_create(int64_t n, const int64_t *offsets, const int32_t *cols)
{
    return er_graph_create_ex(n, offsets, cols, 0u);
}

er_graph *er_graph_create_ex(int64_t n, const int64_t *offsets, const int32_t *cols, uint32_t flags)
{
    clear_error();
    bool sorted = false;
    int32_t md = 0;
    int spec = ER_OK;
    if (flags & ~ER_CREATE_SPMM_ONLY) {
        set_error(ER_EINVAL, "unknown flags");
        return nullptr;
    }
    const bool spmm_only = (flags & ER_CREATE_SPMM_ONLY) != 0;
    if (validate_basic(n, offsets, cols) != ER_OK) return nullptr;
    // input errors are reported whether or not a device is present: without one (or on request,
    // GEER_HOST_VALIDATE=1) the whole validation runs on the host first
    int ndev = 0;
    const bool no_dev = cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0;
    cudaGetLastError();
    const bool host_val = no_dev || (getenv("GEER_HOST_VALIDATE") && atoi(getenv("GEER_HOST_VALIDATE")) != 0);
    if (host_val && validate(n, offsets, cols, &sorted, &md, &spec, spmm_only) != ER_OK) return nullptr;
    er_graph *g = new (std::nothrow) er_graph();
    if (!g) {
        set_error(ER_ENOMEM, "host allocation failed");
        return nullptr;
    }
    cudaError_t e = cudaGetDevice(&g->device);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&g->num_sms, cudaDevAttrMultiProcessorCount, g->device);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&g->stream, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&g->amc_stream, cudaStreamNonBlocking);
    if (e == cudaSuccess) {
        int lo = 0, hi = 0;
        cudaDeviceGetStreamPriorityRange(&lo, &hi);
        e = cudaStreamCreateWithPriority(&g->head_stream, cudaStreamNonBlocking, hi);
    }
    if (e == cudaSuccess) {
        // keep stream-ordered allocations (per-batch y-tables, AMC group buffers) cached
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, g->device) == cudaSuccess) {
            uint64_t thr = UINT64_MAX;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
        }
    }
    g->n = n;
    g->nnz = offsets[n];
    int nb = 1;
    while ((1ll << nb) < n) nb++;
    g->nbits = nb;
    if (e == cudaSuccess) e = cudaMalloc(&g->d_off, sizeof(int64_t) * (n + 1));
    if (e == cudaSuccess) e = cudaMalloc(&g->d_cols, sizeof(int32_t) * std::max<int64_t>(g->nnz, 1));
    if (e == cudaSuccess) e = cudaMemcpy(g->d_off, offsets, sizeof(int64_t) * (n + 1), cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(g->d_cols, cols, sizeof(int32_t) * g->nnz, cudaMemcpyHostToDevice);
    if (e == cudaSuccess && !host_val) {
        // the checks over the columns run on the device (validate.cu); graphs with unsorted rows
        // (or a BFS deeper than its level cap) fall back to the host validation
        int code = ER_OK;
        std::string msg;
        if (geer::validate_device(g, &code, &msg, &spec, &sorted, &md) != 0) {
            if (validate(n, offsets, cols, &sorted, &md, &spec, spmm_only) != ER_OK) {
                er_graph_destroy(g);
                return nullptr;
            }
        } else {
            if (code == ER_OK && spec != ER_OK && !spmm_only) {
                code = spec;
                msg = spec == ER_EDISCONNECTED ? "graph is not connected" : "graph is bipartite (lambda = 1)";
            }
            if (code != ER_OK) {
                er_graph_destroy(g);
                set_error(code, msg);
                return nullptr;
            }
        }
    }
    g->rows_sorted = sorted;
    g->max_deg = md;
    g->query_block = spec;
    if (e == cudaSuccess) {
        // 8-byte node records {offset, degree} for the walk kernel (one sector per step)
        std::vector<uint2> rec(n);
#pragma omp parallel for schedule(static)
        for (int64_t v = 0; v < n; v++) rec[v] = make_uint2((uint32_t)offsets[v], (uint32_t)(offsets[v + 1] - offsets[v]));
        e = cudaMalloc(&g->d_rec, sizeof(uint2) * n);
        if (e == cudaSuccess) e = cudaMemcpy(g->d_rec, rec.data(), sizeof(uint2) * n, cudaMemcpyHostToDevice);
        // Walk layout: packed 8-byte arc records {u | off(u) | d(u)} when the
        // three fields fit 64 bits and the array stays inside L2 (one random access per step);
        // else 16-byte arc records when the graph is DRAM-resident anyway; else node records
        // {off, d} + columns.
        int l2 = 0;
        cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, g->device);
        auto bits = [](uint64_t x) { int b = 1; while (b < 64 && (1ull << b) <= x) b++; return b; };
        const int bu = bits((uint64_t)(n - 1)), bo = bits((uint64_t)g->nnz), bd = bits((uint64_t)md);
        const bool packable = bu + bo + bd <= 64;
        const double cols_foot = 4.0 * (double)g->nnz + 8.0 * (double)n;
        const double pack_foot = 8.0 * (double)g->nnz;
        int layout = 0;  // 0 cols, 1 arcs16, 2 packed
        if (packable && pack_foot <= 0.75 * (double)l2) layout = 2;
        // cols needs a second random access per step (the node record) unless the node records
        // stay in L2: beyond ~3/8 of L2 (Friendster-shaped: 480 MB of records) the 16-byte arc
        // records, one access per step, win (363 vs 243 ms per step on a 125k shard)
        else if (8.0 * (double)n > 0.375 * (double)l2) layout = 1;
        (void)cols_foot;
        // DRAM-resident graphs keep cols + node records: a random DRAM access moves a whole line
        // whatever the record size (profiles/sector_flavours_r02.txt), so the smaller column array
        // wins by its higher L2 hit rate (LJ-shaped config: 495 vs 517 ms of walks per step against
        // 16-byte arc records); K6 then loads columns L2 evict-first with 64-byte fetches and node
        // records with 64-byte fetches (walks.cu; 447 -> 418 ms, profiles/exp_walk_policy_r02.jsonl)
        // cols with node ids below 2^24: 24-bit columns, 5 per 16-byte chunk (3.2 B per arc instead of
        // 4: a larger share of the random column loads hits L2)
        if (layout == 0 && n <= (1 << 24)) layout = 3;
        // and renumbered by degree (layout 4, falls back to 3 when not applicable): the node
        // record comes from a shared-memory tree of the degree classes instead of a dependent
        // global load (LJ-shaped config)
        if (layout == 3) layout = 4;
        if (const char *env = getenv("GEER_WALK_LAYOUT")) {
            if (!strcmp(env, "arcs")) layout = 1;
            if (!strcmp(env, "cols")) layout = 0;
            if (!strcmp(env, "cols24") && n <= (1 << 24)) layout = 3;
            if (!strcmp(env, "dord") && n <= (1 << 24)) layout = 4;
            if (!strcmp(env, "packed") && packable) layout = 2;
        }
        if (const char *env = getenv("GEER_DORD_SMEM_KB")) g->dord_smem_bytes = 1024 * std::min(96, std::max(0, atoi(env)));
        if (layout == 4 && e == cudaSuccess) {
            const int rc = geer::build_dord(g, offsets, cols);
            if (rc < 0) e = cudaErrorMemoryAllocation;
            if (rc == 1) layout = 3;
            // K6 column loads: about half of L2 worth of the column lines evict-last (a fixed share
            // of the random column loads then hits L2), the rest evict-first (LJ-shaped config:
            // 373 -> 334 ms of walks per step, flat for 15-45 % of the 238 MB)
            if (rc == 0 && !getenv("GEER_WALK_L2_KEEP"))
                g->walk_l2_keep = (float)std::min(1.0, 0.5 * (double)l2 / (16.0 * (double)((g->nnz + 4) / 5)));
        }
        // K6 scheduling: per-warp chunks when the walk graph is L2-resident (packed), CTA-tiles of
        // 8 chunks when it is DRAM-resident (measured: 4.40 vs 4.56 ms on config 1, 544 vs 529 ms
        // on config 2)
        g->walk_tiles = layout != 2;
        if (const char *env = getenv("GEER_WALK_MINB")) { const int v = atoi(env); g->walk_minb = (v >= 3 && v <= 6) ? v : 4; }
        if (const char *env = getenv("GEER_AMC_OVERLAP")) g->amc_overlap = atoi(env) != 0;
        if (const char *env = getenv("GEER_WALK_PERSIST")) g->walk_persist = atoi(env) != 0;
        if (const char *env = getenv("GEER_YTABLE")) g->ytable_force = !strcmp(env, "hash") ? 1 : !strcmp(env, "rank") ? 2 : 0;
        if (const char *env = getenv("GEER_L2_PERSIST")) g->l2_persist = atoi(env) != 0;
        if (const char *env = getenv("GEER_WALK_L2_KEEP")) g->walk_l2_keep = (float)std::min(1.0, std::max(0.0, atof(env)));
        if (const char *env = getenv("GEER_OVERLAP_FRAC")) g->overlap_frac = std::min(1.0, std::max(0.1, atof(env)));
        if (const char *env = getenv("GEER_MAX_SUB_BATCH")) g->max_sub_batch = std::max<int64_t>(1, atoll(env));
        if (const char *env = getenv("GEER_WAVE_PAIRS_MAX")) g->wave_pairs_max = std::max<int64_t>(1, atoll(env));
        if (const char *env = getenv("GEER_WALK_NP")) g->walk_np = atoi(env) == 1 ? 1 : 2;
        {   // ER_ENOMEM fault injection (tests): the N-th workspace growth from here on fails once
            const char *env = getenv("GEER_FAULT_ALLOC");
            geer::g_fault_count = 0;
            geer::g_fault_target = env ? std::max<int64_t>(0, atoll(env)) : 0;
        }
        if (const char *env = getenv("GEER_HUB_CB")) { const int v = atoi(env); g->hub_cb = (v == 8 || v == 16) ? v : 32; }
        if (const char *env = getenv("GEER_WALK_SMEM_KB")) g->walk_smem_words = 256 * std::min(48, std::max(0, atoi(env)));
        if (const char *env = getenv("GEER_RANK_MIN_CAP")) g->rank_min_cap = std::max<int64_t>(0, atoll(env));
        if (const char *env = getenv("GEER_RANK_RATIO")) g->rank_ratio = std::max<int64_t>(0, atoll(env));
        if (const char *env = getenv("GEER_RANK_MAX_KB")) g->rank_max_bytes = 1024 * std::max<int64_t>(0, atoll(env));
        if (const char *env = getenv("GEER_WALK_TILES")) g->walk_tiles = atoi(env) != 0;
        if (const char *env = getenv("GEER_WALK_CARVEOUT")) g->walk_carveout = std::min(100, std::max(-1, atoi(env)));
        g->pack.bo = bo;
        g->pack.bd = bd;
        if (layout == 1 && e == cudaSuccess) {
            e = cudaMalloc(&g->d_arcs, sizeof(uint4) * std::max<int64_t>(g->nnz, 1));
            if (e == cudaSuccess) e = geer::build_arcs(g);
        }
        if (layout == 2 && e == cudaSuccess) {
            e = cudaMalloc(&g->d_parcs, sizeof(unsigned long long) * std::max<int64_t>(g->nnz, 1));
            if (e == cudaSuccess) e = geer::build_parcs(g);
        }
        if (layout == 3 && e == cudaSuccess) {
            e = cudaMalloc(&g->d_c24, sizeof(uint4) * std::max<int64_t>((g->nnz + 4) / 5, 1));
            if (e == cudaSuccess) e = geer::build_c24(g);
        }
    }
    if (e == cudaSuccess && g->l2_persist) {
        // keep the walk graph in L2: a persisting access-policy window on the AMC stream (the
        // y-tables stream past it).  Sets the device's persisting-L2 limit (a process-wide
        // setting), so it is opt-in (GEER_L2_PERSIST=1).
        cudaDeviceProp prop;
        if (cudaGetDeviceProperties(&prop, g->device) == cudaSuccess && prop.persistingL2CacheMaxSize > 0) {
            void *base = g->d_parcs ? (void *)g->d_parcs : g->d_arcs ? (void *)g->d_arcs : (void *)g->d_cols;
            const size_t want = g->d_parcs ? 8 * (size_t)g->nnz : g->d_arcs ? 16 * (size_t)g->nnz : 4 * (size_t)g->nnz;
            const size_t lim = std::min(want, (size_t)prop.persistingL2CacheMaxSize);
            cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, lim);
            cudaStreamAttrValue a{};
            a.accessPolicyWindow.base_ptr = base;
            a.accessPolicyWindow.num_bytes = std::min(want, (size_t)prop.accessPolicyMaxWindowSize);
            a.accessPolicyWindow.hitRatio = (float)std::min(1.0, (double)lim / (double)a.accessPolicyWindow.num_bytes);
            a.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
            a.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
            cudaStreamSetAttribute(g->amc_stream, cudaStreamAttributeAccessPolicyWindow, &a);
            g->l2_window = a.accessPolicyWindow.num_bytes;
            g->l2_persist_bytes = lim;
        }
        cudaGetLastError();
    }
    if (e != cudaSuccess) {
        cuda_fail(e, "er_graph_create");
        er_graph_destroy(g);
        return nullptr;
    }
    return g;
}

void er_graph_destroy(er_graph *g)
{
    if (!g) return;
    {
        std::lock_guard<std::mutex> lk(g->mu);
        int cur = 0;
        cudaGetDevice(&cur);
        cudaSetDevice(g->device);
        if (g->stream) cudaStreamSynchronize(g->stream);
        g->ws.release();
        if (g->d_off) cudaFree(g->d_off);
        if (g->d_cols) cudaFree(g->d_cols);
        if (g->d_rec) cudaFree(g->d_rec);
        if (g->d_arcs) cudaFree(g->d_arcs);
        if (g->d_parcs) cudaFree(g->d_parcs);
        if (g->d_c24) cudaFree(g->d_c24);
        if (g->d_perm) cudaFree(g->d_perm);
        if (g->d_iperm) cudaFree(g->d_iperm);
        if (g->d_cblk) cudaFree(g->d_cblk);
        if (g->d_ccd) cudaFree(g->d_ccd);
        if (g->d_steps) cudaFree(g->d_steps);
        if (g->d_rowperm) cudaFree(g->d_rowperm);
        if (g->d_hseg) cudaFree(g->d_hseg);
        if (g->d_seg_e0) cudaFree(g->d_seg_e0);
        if (g->d_seg_row) cudaFree(g->d_seg_row);
        if (g->d_spmm_desc) cudaFree(g->d_spmm_desc);
        if (g->amc_stream) cudaStreamSynchronize(g->amc_stream);
        if (g->stream) cudaStreamDestroy(g->stream);
        if (g->amc_stream) cudaStreamDestroy(g->amc_stream);
        if (g->head_stream) {
            cudaStreamSynchronize(g->head_stream);
            cudaStreamDestroy(g->head_stream);
        }
        if (g->ev_in) cudaEventDestroy(g->ev_in);
        if (g->ev_out) cudaEventDestroy(g->ev_out);
        if (g->ybuild_stream) {
            cudaStreamSynchronize(g->ybuild_stream);
            cudaStreamDestroy(g->ybuild_stream);
            cudaEventDestroy(g->ev_yfork);
            cudaEventDestroy(g->ev_ydone);
        }
        if (g->spmm_stream) {
            cudaStreamSynchronize(g->spmm_stream);
            cudaStreamDestroy(g->spmm_stream);
            cudaEventDestroy(g->spmm_fork);
            cudaEventDestroy(g->spmm_join);
        }
        cudaSetDevice(cur);
    }
    delete g;
}

int er_graph_lambda(const er_graph *g, double *lambda_out)
{
    clear_error();
    if (!g || !lambda_out) { set_error(ER_EINVAL, "NULL argument"); return ER_EINVAL; }
    if (!g->lambda_set) { set_error(ER_ESPECTRAL, "lambda not set"); return ER_ESPECTRAL; }
    *lambda_out = g->lambda;
    return ER_OK;
}

int er_graph_set_lambda(er_graph *g, double lambda)
{
    clear_error();
    if (!g) { set_error(ER_EINVAL, "NULL graph"); return ER_EINVAL; }
    if (!(lambda > 0.0 && lambda <= 1.0 - 1e-12)) {
        set_error(ER_ESPECTRAL, "lambda must be in (0, 1-1e-12]");
        return ER_ESPECTRAL;
    }
    std::lock_guard<std::mutex> lk(g->mu);
    g->lambda = lambda;
    g->lambda_set = true;
    return ER_OK;
}

int64_t er_graph_num_nodes(const er_graph *g) { return g ? g->n : -1; }
int64_t er_graph_num_arcs(const er_graph *g) { return g ? g->nnz : -1; }
int64_t er_graph_kernel_launches(const er_graph *g) { return g ? g->launches : -1; }

int er_query_batch_ex(er_graph *g, const int32_t *pairs, int64_t k, double eps, double p_fail, const er_opts *o,
                      double *out_r, er_query_stats *stats)
{
    clear_error();
    er_opts opt;
    if (o) opt = *o;
    else er_opts_default(&opt);
    if (!g) { set_error(ER_EINVAL, "NULL graph"); return ER_EINVAL; }
    if (k < 0) { set_error(ER_EINVAL, "k < 0"); return ER_EINVAL; }
    if (k > 0 && (!pairs || !out_r)) { set_error(ER_EINVAL, "NULL pairs/out_r"); return ER_EINVAL; }
    if (!(eps > 0.0) || !std::isfinite(eps)) { set_error(ER_EINVAL, "eps must be > 0"); return ER_EINVAL; }
    if (!(p_fail > 0.0 && p_fail < 1.0)) { set_error(ER_EINVAL, "p_fail must be in (0,1)"); return ER_EINVAL; }
    if (opt.tau < 1 || opt.tau > 8) { set_error(ER_EINVAL, "tau must be in [1,8]"); return ER_EINVAL; }
    if (opt.ell_variant != 0 && opt.ell_variant != 1) { set_error(ER_EINVAL, "ell_variant must be 0 or 1"); return ER_EINVAL; }
    if (opt.force_ell_b < -1) { set_error(ER_EINVAL, "force_ell_b must be >= -1"); return ER_EINVAL; }
    if (!(opt.switch_ratio >= 0.0) || !std::isfinite(opt.switch_ratio)) { set_error(ER_EINVAL, "switch_ratio must be >= 0"); return ER_EINVAL; }
    if (opt.reuse_samples != 0 && opt.reuse_samples != 1) { set_error(ER_EINVAL, "reuse_samples must be 0 or 1"); return ER_EINVAL; }
    if (opt.smm_mode < 0 || opt.smm_mode > 2) { set_error(ER_EINVAL, "smm_mode must be 0, 1 or 2"); return ER_EINVAL; }
    if (opt.query_index_base < 0 || opt.query_index_base + k > ((int64_t)1 << 32)) {
        set_error(ER_EINVAL, "query indices must fit in 32 bits");
        return ER_EINVAL;
    }
    if (opt.query_ids && !opt.pairs_on_device) {
        for (int64_t i = 0; i < k; i++) {
            if (opt.query_ids[i] < 0 || opt.query_ids[i] >= ((int64_t)1 << 32)) {
                set_error(ER_EINVAL, "query_ids[" + std::to_string(i) + "] outside [0, 2^32)");
                return ER_EINVAL;
            }
        }
    }
    std::lock_guard<std::mutex> lk(g->mu);
    if (g->query_block != ER_OK) { set_error(g->query_block, "graph created ER_CREATE_SPMM_ONLY: not connected or bipartite"); return g->query_block; }
    if (!g->lambda_set) { set_error(ER_ESPECTRAL, "lambda not set (er_graph_set_lambda / er_graph_estimate_lambda)"); return ER_ESPECTRAL; }
    if (k == 0) return ER_OK;
    if (!opt.pairs_on_device) {
        for (int64_t i = 0; i < 2 * k; i++) {
            if (pairs[i] < 0 || pairs[i] >= g->n) {
                set_error(ER_EINVAL, "node id out of range at pairs[" + std::to_string(i) + "]");
                return ER_EINVAL;
            }
        }
    }
    int cur = 0;
    cudaGetDevice(&cur);
    if (cur != g->device) cudaSetDevice(g->device);
    // Very large batches run as consecutive sub-batches (bounded workspaces and per-wave pair
    // counts); every query keeps its global index, so the results are those of one batch.
    int rc = ER_OK;
    const int64_t sub = g->max_sub_batch;
    for (int64_t lo = 0; lo < k && rc == ER_OK; lo += sub) {
        const int64_t kk = std::min(sub, k - lo);
        er_opts o2 = opt;
        if (opt.query_ids) o2.query_ids = opt.query_ids + lo;
        else o2.query_index_base = opt.query_index_base + lo;
        if (lo + kk < k) o2.synchronous = 1;   // only the last sub-batch may return early
        rc = run_query_batch(g, pairs + 2 * lo, kk, eps, p_fail, o2, out_r + lo, stats ? stats + lo : nullptr);
    }
    if (cur != g->device) cudaSetDevice(cur);
    return rc;
}

int er_query_batch(er_graph *g, const int32_t *pairs, int64_t k, double eps, double p_fail, double *out_r)
{
    return er_query_batch_ex(g, pairs, k, eps, p_fail, nullptr, out_r, nullptr);
}

int er_spmm_ex(er_graph *g, const double *X, double *Y, int32_t q, int32_t flags, void *stream)
{
    clear_error();
    if (!g || !X || !Y || X == Y) { set_error(ER_EINVAL, "bad arguments"); return ER_EINVAL; }
    if (q < 1 || q > 256) { set_error(ER_EINVAL, "q must be in [1,256]"); return ER_EINVAL; }
    if (flags & ~(ER_SPMM_NORMALIZE | ER_SPMM_EXACT)) { set_error(ER_EINVAL, "unknown flags"); return ER_EINVAL; }
    std::lock_guard<std::mutex> lk(g->mu);
    return run_spmm(g, X, Y, q, (flags & ER_SPMM_NORMALIZE) ? 1 : 0, stream ? (cudaStream_t)stream : g->stream,
                    (flags & ER_SPMM_EXACT) != 0);
}

int er_spmm(er_graph *g, const double *X, double *Y, int32_t q, int32_t normalize, void *stream)
{
    return er_spmm_ex(g, X, Y, q, normalize ? ER_SPMM_NORMALIZE : 0, stream);
}

int er_smm_series(er_graph *g, const int32_t *pairs, int64_t k, double tol, int32_t max_iters, double *out_r,
                  int32_t *ells)
{
    clear_error();
    if (!g) { set_error(ER_EINVAL, "NULL graph"); return ER_EINVAL; }
    if (k < 0 || (k > 0 && (!pairs || !out_r))) { set_error(ER_EINVAL, "bad k / NULL pointers"); return ER_EINVAL; }
    if (!(tol > 0.0) || !std::isfinite(tol)) { set_error(ER_EINVAL, "tol must be > 0"); return ER_EINVAL; }
    if (max_iters < 0 || max_iters > 100000) { set_error(ER_EINVAL, "max_iters must be in [0, 100000]"); return ER_EINVAL; }
    for (int64_t i = 0; i < 2 * k; i++) {
        if (pairs[i] < 0 || pairs[i] >= g->n) {
            set_error(ER_EINVAL, "node id out of range at pairs[" + std::to_string(i) + "]");
            return ER_EINVAL;
        }
    }
    std::lock_guard<std::mutex> lk(g->mu);
    if (g->query_block != ER_OK) { set_error(g->query_block, "graph is not connected or bipartite"); return g->query_block; }
    if (!g->lambda_set) { set_error(ER_ESPECTRAL, "lambda not set"); return ER_ESPECTRAL; }
    if (k == 0) return ER_OK;
    int cur = 0;
    cudaGetDevice(&cur);
    if (cur != g->device) cudaSetDevice(g->device);
    const int rc = run_smm_series(g, pairs, k, tol, max_iters, out_r, ells);
    if (cur != g->device) cudaSetDevice(cur);
    return rc;
}

int er_graph_estimate_lambda(er_graph *g, int iters, double *lambda_out)
{
    clear_error();
    if (!g) { set_error(ER_EINVAL, "NULL graph"); return ER_EINVAL; }
    if (g->query_block != ER_OK) { set_error(g->query_block, "graph is not connected or bipartite"); return g->query_block; }
    if (iters < 0 || iters > 2000) { set_error(ER_EINVAL, "iters must be in [0,2000]"); return ER_EINVAL; }
    std::lock_guard<std::mutex> lk(g->mu);
    double lam = 0.0;
    const int rc = run_estimate_lambda(g, iters == 0 ? 500 : iters, &lam);
    if (rc) return rc;
    if (!(lam > 0.0 && lam <= 1.0 - 1e-12)) {
        set_error(ER_ESPECTRAL, "estimated lambda outside (0, 1-1e-12]");
        return ER_ESPECTRAL;
    }
    g->lambda = lam;
    g->lambda_set = true;
    if (lambda_out) *lambda_out = lam;
    return ER_OK;
}

int er_graph_profile(er_graph *g, int enable)
{
    clear_error();
    if (!g) { set_error(ER_EINVAL, "NULL graph"); return ER_EINVAL; }
    std::lock_guard<std::mutex> lk(g->mu);
    if (!g->d_steps) {
        cudaError_t e = cudaMalloc(&g->d_steps, sizeof(int64_t));
        if (e != cudaSuccess) return cuda_fail(e, "er_graph_profile");
    }
    cudaError_t e = cudaMemsetAsync(g->d_steps, 0, sizeof(int64_t), g->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(g->stream);
    if (e != cudaSuccess) return cuda_fail(e, "er_graph_profile");
    g->prof = er_profile{};
    g->profiling = enable != 0;
    return ER_OK;
}

int er_graph_profile_read(er_graph *g, er_profile *out)
{
    clear_error();
    if (!g || !out) { set_error(ER_EINVAL, "NULL argument"); return ER_EINVAL; }
    std::lock_guard<std::mutex> lk(g->mu);
    *out = g->prof;
    out->walk_ctas_per_sm = g->walk_occ;
    out->walk_layout = g->d_parcs ? 2 : g->d_cblk ? 4 : g->d_c24 ? 3 : g->d_arcs ? 1 : 0;
    out->walk_graph_bytes = g->d_parcs ? 8 * g->nnz
                            : g->d_cblk ? 16 * ((g->nnz + 4) / 5) + 4 * g->n + 4 * g->dord_nv
                                              + 2 * (int64_t)g->dord_nblk + 8 * (int64_t)g->dord_ncls
                            : g->d_c24 ? 16 * ((g->nnz + 4) / 5) + 8 * g->n
                            : g->d_arcs ? 16 * g->nnz : 4 * g->nnz + 8 * g->n;
    if (g->d_steps) {
        int64_t steps = 0;
        cudaError_t e = cudaMemcpy(&steps, g->d_steps, sizeof(int64_t), cudaMemcpyDeviceToHost);
        if (e != cudaSuccess) return cuda_fail(e, "er_graph_profile_read");
        out->walk_steps = steps;
    }
    return ER_OK;
}

}  // extern "C"
