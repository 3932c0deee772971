/*
 * geer.h -- C ABI of libgeer.so, the B200 (sm_100a) implementation of GEER
 * epsilon-approximate pairwise effective-resistance (PER) queries.
 *
 * Paper: "Efficient Estimation of Pairwise Effective Resistance", arXiv 2312.06123.
 * P:n below = line n of the paper's LaTeX source.
 *
 * Problem (Def. 2.2): for each queried pair (s,t) return r'(s,t) with
 * |r'(s,t) - r(s,t)| <= eps (Eq. 2) where r(s,t) = (e_s-e_t) L^+ (e_s-e_t)^T
 * is the effective resistance (Def. 2.1, Eq. 1).  The method is GEER
 * (Alg. 3): a deterministic SMM head (Alg. 2) followed by
 * AMC adaptive Monte Carlo walks (Alg. 1); the guarantee holds with
 * probability >= 1 - p_fail per query (Thm 3.4).
 *
 * Conventions common to every call:
 *  - Graphs are simple, undirected, unweighted, connected and non-bipartite
 *    (P:159-160), given as a symmetric CSR: offsets[n+1] (int64, offsets[0]=0,
 *    non-decreasing) and cols[offsets[n]] (int32 node ids in [0,n)).  Each
 *    undirected edge appears in both rows.  Neighbour order inside a row is
 *    preserved: walks index rows in the given order (R10).
 *  - Functions returning int return ER_OK (0) on success or an ER_E* code; the
 *    code and a message are also kept per host thread (er_last_error*).
 *  - A handle is bound to the CUDA device that was current at er_graph_create and
 *    may be used by one host thread at a time (calls are serialised by a mutex).
 *  - There is no CPU fallback: every step of a query runs in CUDA kernels on the
 *    handle's device; without a usable device every call fails with ER_ECUDA.
 */
#ifndef GEER_H_
#define GEER_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    ER_OK = 0,
    ER_EINVAL = 1,        /* bad n / offsets / cols / k / eps / p_fail / node id / option */
    ER_ESELFLOOP = 2,     /* self-loop present (Lemma 3.3 needs consecutive walk nodes distinct) */
    ER_EDUP = 3,          /* duplicate neighbour in a row */
    ER_EASYM = 4,         /* adjacency not symmetric */
    ER_EDISCONNECTED = 5, /* graph not connected */
    ER_EBIPARTITE = 6,    /* graph bipartite: lambda = 1 and Eq. 6 is undefined */
    ER_ESPECTRAL = 7,     /* lambda unset, or lambda outside (0, 1 - 1e-12] */
    ER_ENOMEM = 8,        /* device or host allocation failed */
    ER_ECUDA = 9          /* CUDA runtime error (message has the CUDA error string) */
};

typedef struct er_graph er_graph; /* opaque */

/*
 * er_graph_create -- copy a CSR graph to the current CUDA device and validate it.
 *   n        number of nodes, n >= 2
 *   offsets  HOST pointer, int64[n+1]
 *   cols     HOST pointer, int32[offsets[n]]
 * The caller keeps ownership of offsets/cols and may free them on return.
 * Validation (in this order, first failure wins): offsets monotone and in range,
 * cols in range (ER_EINVAL), no self-loop (ER_ESELFLOOP), no duplicate neighbour
 * (ER_EDUP), symmetric (ER_EASYM), connected (ER_EDISCONNECTED), not bipartite
 * (ER_EBIPARTITE).  lambda (Eq. 6) starts unset: pin it with
 * er_graph_set_lambda (the paper's preprocessing step) or
 * estimate it on the device with er_graph_estimate_lambda.
 * Returns NULL on failure (see er_last_error).
 */
er_graph *er_graph_create(int64_t n, const int64_t *offsets, const int32_t *cols);

/*
 * er_graph_create_ex -- er_graph_create with flags.
 *   ER_CREATE_SPMM_ONLY: skip the connected / non-bipartite requirement (the graph is then
 *   usable by er_spmm only; query calls fail with the error validation would have
 *   raised).  Used e.g. for Fig. 3's bipartite toy graph.
 */
#define ER_CREATE_SPMM_ONLY 1u
er_graph *er_graph_create_ex(int64_t n, const int64_t *offsets, const int32_t *cols, uint32_t flags);

/* er_graph_destroy -- free the handle and all its device memory.  NULL-safe. */
void er_graph_destroy(er_graph *g);

/*
 * er_query_batch -- answer k epsilon-approximate PER queries (Alg. 3 per query).
 *   pairs   HOST int32[2k]: s0,t0,s1,t1,...   (node ids in [0,n); s == t allowed -> 0.0)
 *   k       number of queries, k >= 0 (k == 0 is a no-op)
 *   eps     additive error eps > 0 (Eq. 2)
 *   p_fail  failure probability delta in (0,1) per query (Thm 3.4); tau = 5 batches
 *   out_r   HOST double[k], caller-allocated; out_r[i] = r'(s_i, t_i)
 * Synchronous.  Uses the library's default seed, query_index_base = 0.  Batches larger than
 * 2^18 queries run as consecutive sub-batches of the same results (bounded device memory).
 * Any out-of-range id fails the whole call with ER_EINVAL before any work.
 * Estimates are returned unclamped (they may be slightly negative).
 */
int er_query_batch(er_graph *g, const int32_t *pairs, int64_t k, double eps, double p_fail,
                   double *out_r);

/* ------------------------------------------------------------------ extras */

int er_last_error(void);                 /* code of this thread's last failure (ER_OK if none) */
const char *er_last_error_message(void); /* human-readable message, never NULL */

/* lambda = max(|lambda_2|, |lambda_n|) of P = D^-1 A (Eq. 6). */
int er_graph_lambda(const er_graph *g, double *lambda_out);      /* ER_ESPECTRAL if unset */
int er_graph_set_lambda(er_graph *g, double lambda);             /* lambda in (0, 1-1e-12] */
/*
 * er_graph_estimate_lambda -- estimate lambda on the device and pin it (the paper's ARPACK
 * preprocessing): Lanczos on N = D^-1/2 A D^-1/2 with sqrt(d) projected out and
 * full re-orthogonalisation against the stored Krylov basis (at most 16 GB of it), stopped when
 * both extreme Ritz pairs have converged (residual estimate < 1e-11) or after `iters` steps; the
 * result is max over both ends of |theta| + ||N x - theta x|| with the explicit residual of the
 * extreme Ritz vector x -- an upper estimate of max(|lambda_2|, |lambda_n|) (R12).
 *   iters      Krylov steps at most (0 = default 500; <= 2000, further capped at 511 and by memory)
 *   lambda_out the estimate (may be NULL)
 */
int er_graph_estimate_lambda(er_graph *g, int iters, double *lambda_out);

int64_t er_graph_num_nodes(const er_graph *g);
int64_t er_graph_num_arcs(const er_graph *g);        /* offsets[n] = 2m */
/* Kernels launched by this handle since creation (all of them are this library's). */
int64_t er_graph_kernel_launches(const er_graph *g);

/*
 * er_probe_random_loads -- the random-access ceiling of the running device that K6's roofline is
 * quoted against: 8-byte loads at independent, uniformly random
 * 32-byte sectors of a freshly allocated buffer of `bytes`, 8 in flight per thread, every SM at
 * full occupancy; the best of 3 timed launches after one warm-up.  Not on the query path
 * (diagnostic; synchronous; allocates and frees the buffer).
 *   bytes          buffer size, >= 1 MiB (L2-resident below ~64 MB, DRAM-resident above)
 *   flavour        0: ld.global.nc (K6's packed-record load), 1: ld.global.nc.L2::64B (K6's
 *                  column load on DRAM-resident walk graphs: 64-byte L2 fills)
 *   iters          8-load rounds per thread (the launch length)
 *   g_loads_per_s  out: 10^9 loads per second
 * Errors: ER_EINVAL (arguments), ER_ECUDA (allocation or launch).
 */
int er_probe_random_loads(int64_t bytes, int32_t flavour, int32_t iters, double *g_loads_per_s);

typedef struct er_opts {
    int32_t tau;               /* batches of AMC, 1..8 (default 5) */
    int32_t force_ell_b;       /* -1: Eq. 15 decides ell_b (default); >= 0: exactly min(force, ell)
                                  SMM iterations (0 = AMC alone, Thm 3.4 setting P:337) */
    uint64_t seed;             /* Philox key (default ER_DEFAULT_SEED) */
    int64_t query_index_base;  /* global index of pairs[0]; RNG streams are keyed by it (sharding) */
    void *cuda_stream;         /* cudaStream_t to run on (NULL: the handle's own stream) */
    int32_t pairs_on_device;   /* pairs is a DEVICE pointer */
    int32_t out_on_device;     /* out_r (and stats) are DEVICE pointers */
    int32_t ell_variant;       /* 0: Eq. 6 refined ell (default); 1: Eq. 5 Peng et al.'s ell */
    int32_t synchronous;       /* 1 (default): return after the results are final; 0: asynchronous on
                                  cuda_stream when both pointers are on the device */
    int32_t pad0;
    const int64_t *query_ids;  /* NULL (default): query i has global index query_index_base + i;
                                  else query_ids[i] (k entries, host or device like pairs), each in
                                  [0, 2^32).  The global index keys the query's RNG streams (R10),
                                  so a query's result does not depend on which rank or batch runs
                                  it (cost-model sharding, paper_2312_06123_b200/dist.py) */
    double switch_ratio;       /* variant: leave the SMM head iff vol > switch_ratio * h;
                                  1.0 (default) is Eq. 15; any value keeps the eps guarantee */
    int32_t reuse_samples;     /* variant: 1 = batch b keeps the previous batches'
                                  samples and draws only the new ones (one sample stream per query, batch
                                  key 0); 0 (default) = fresh samples per batch (R8) */
    int32_t smm_mode;          /* how SMM iterations after the first are applied (Alg. 3 L6):
                                  0 (default) per wave by a cost model: sparse frontier push (K2/K3) or
                                  the dense block pull (K9, exact sequential sums) when the wave's pushes
                                  would cost more than a full pass over the CSR for its columns;
                                  1 = frontier push only; 2 = dense pull whenever the wave has at most
                                  ER_DENSE_MAX_QUERIES active queries.  On graphs with sorted adjacency
                                  lists all modes give bit-identical results; otherwise the push sums
                                  in ascending source order and the pull in CSR order (within 1e-10
                                  relative, R13, R25); only speed differs */
} er_opts;

/* Dense-mode limit: a wave runs dense only with <= this many active queries (2 columns each). */
#define ER_DENSE_MAX_QUERIES 128

#define ER_DEFAULT_SEED 0x2312061232DEC0DEULL

/* Fill *o with the defaults above. */
void er_opts_default(er_opts *o);

/*
 * Per-query diagnostics (all fields defined in DESIGN.md "Per-query stats"):
 *  ell, ell_b, ell_f = ell - ell_b   Eq. 6 / Alg. 3 L9 / Alg. 3 L10
 *  batches_run                        AMC batches executed (<= tau)
 *  eta0, walks_total, steps_total     first-batch walk pairs, walk pairs over all batches,
 *                                     walk steps over all batches and both sides
 *  vol_last, h_last                   both sides of Eq. 15 at the last SMM iteration
 *  psi, r_b, r_f, f_last, sigma2_last Eq. 10, SMM part, AMC part, Eq. 8 at the last batch, variance
 *  rb_terms[i]                        series increment of SMM iteration i+1 (i < 8)
 *  walk_checksum                      sum over walks of fmix-hash(q,b,side,k,endpoint) mod 2^64
 *  tie_flags                          bit0: ell, bit1: eta0, bit2: Bernstein decision within 1e-12
 *  ytable_log2                        log2 of the y-table capacity (implementation diagnostic)
 */
typedef struct er_query_stats {
    int32_t ell, ell_b, ell_f, batches_run;
    int64_t eta0, walks_total, steps_total, vol_last, h_last;
    double psi, r_b, r_f, f_last, sigma2_last;
    double rb_terms[8];
    uint64_t walk_checksum;
    uint32_t tie_flags;
    uint32_t ytable_log2;     /* log2 of the query's y-table slots (0: no AMC); diagnostics only */
} er_query_stats;

/*
 * er_query_batch_ex -- er_query_batch with options and optional per-query stats.
 *   o      may be NULL (defaults)
 *   stats  may be NULL; else k entries, host or device per o->out_on_device
 */
int er_query_batch_ex(er_graph *g, const int32_t *pairs, int64_t k, double eps, double p_fail,
                      const er_opts *o, double *out_r, er_query_stats *stats);

/*
 * er_spmm -- Y = M X for a dense row-major n x q block (K9, the dense form of
 * Alg. 2 L4 "s* <- P s*" applied to q columns at once; also the SMM-1000
 * ground-truth engine of P:616).  M = P = D^-1 A when normalize = 1, M = A when
 * normalize = 0 (used to reproduce Fig. 3's #path rows).
 *   X, Y   DEVICE double[n*q] (row v holds the q column values of node v); X != Y
 *   q      1 <= q <= 256
 *   stream cudaStream_t or NULL (handle stream); asynchronous
 */
int er_spmm(er_graph *g, const double *X, double *Y, int32_t q, int32_t normalize, void *stream);

/*
 * er_spmm_ex -- er_spmm with flags: ER_SPMM_NORMALIZE (M = D^-1 A, else A) and ER_SPMM_EXACT
 * (every row, heavy rows included, summed sequentially in CSR order: bit-identical to the plain
 * dense pull; without it rows of degree > 512 are summed in 512-neighbour segments, DESIGN.md
 * R13).  Same arguments and errors as er_spmm.
 */
#define ER_SPMM_NORMALIZE 1
#define ER_SPMM_EXACT 2
int er_spmm_ex(er_graph *g, const double *X, double *Y, int32_t q, int32_t flags, void *stream);

/*
 * er_smm_series -- the deterministic series truncated by a tolerance (SMM-to-ell, the paper's
 * SMM baseline and its ground-truth generator, Alg. 2, Thm 3.1):
 *     r_L(s,t) = sum_{i=0..L} ( y_i(s) - y_i(t) ),  y_0 = e_s/d_s - e_t/d_t,  y_{i+1} = P y_i
 * (the single signed vector form of Alg. 2's s*, t* pair: y_i = P^i e_s / d_s - P^i e_t / d_t).
 * L per query = Eq. 6's ell with eps = tol (the smallest L whose Thm 3.1 tail bound
 * (2/d_s + 2/d_t) lambda^(L+1) / (1 - lambda) is <= tol), capped at max_iters.  Each step is one
 * K9 pass over a block of up to 64 query columns.  s = t gives 0.
 *   pairs   HOST int32[2k];  out_r HOST double[k];  ells HOST int32[k] (L used; may be NULL)
 *   tol > 0, 0 <= max_iters <= 100000; lambda must be set (er_graph_set_lambda / estimate).
 * Synchronous.  Errors: ER_EINVAL (arguments / node ids), ER_ESPECTRAL (lambda unset).
 */
int er_smm_series(er_graph *g, const int32_t *pairs, int64_t k, double tol, int32_t max_iters, double *out_r,
                  int32_t *ells);

/*
 * Profiling (used by bench.py for the live roofline).  When enabled, every query batch
 * records CUDA events on its stream around each AMC walk launch (K6) and around the SMM
 * head, and counts walk steps on the device; er_graph_profile_read returns the sums since
 * the last er_graph_profile(g, 1) call.  Disabled by default (no events, no counters).
 */
typedef struct er_profile {
    double smm_ms;           /* SMM head (all waves, incl. y-table build), event time */
    double walk_ms;          /* sum over K6 launches of their event time */
    double amc_other_ms;     /* AMC reduce/compaction between walk launches */
    int64_t walk_launches;   /* K6 launches */
    int64_t walk_steps;      /* walk steps executed (both sides, all batches) */
    int64_t smm_pairs;       /* (u, x) pairs emitted by the SMM push over all waves */
    int64_t batches;         /* query batches profiled */
    int64_t ytable_slots;    /* hash y-table slots allocated (Alg. 1 L7 tables of the AMC queries) */
    int64_t yrank_records;   /* rank-bitmap y-table records allocated (16 B per 64 node ids) */
    int64_t walk_ctas_per_sm; /* resident K6 CTAs per SM (occupancy API) at the last walk launch */
    int64_t smm_waves;       /* SMM waves after the first (frontier + dense) */
    int64_t smm_dense_waves; /* of which applied by the dense pull (K9) */
    int64_t smm_dense_cols;  /* block columns (2 per active query) summed over the dense waves */
    double amc_span_ms;      /* first K6 launch start to last K6 launch end, per batch, summed (the
                                part above walk_ms is the AMC loop's K7 / scan / launch gaps) */
    int64_t walk_graph_bytes; /* bytes of the walk graph K6 reads (layout below), for the roofline */
    int32_t walk_layout;     /* 0: cols + node records, 1: 16-byte arc records, 2: packed 8-byte arc records,
                                3: 24-bit cols + node records, 4: degree-ordered 24-bit cols + class tree */
    int32_t pad_;
} er_profile;
int er_graph_profile(er_graph *g, int enable);
int er_graph_profile_read(er_graph *g, er_profile *out);

#ifdef __cplusplus
}
#endif

#endif /* GEER_H_ */
