/*
 * oracle/geer_oracle.c -- CPU reference ("oracle") for the GEER query pipeline.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference leg may load this library.  The product path
 * (paper_2312_06123_b200/) never links, imports or executes anything here, and
 * this file shares no code, header, table or helper with it.
 *
 * It is deliberately plain: one query per OpenMP thread, dense length-n vectors,
 * sequential fp64 sums, every step in the paper's order.  Citations:
 *   P:n = /root/reference/PAPER.md line n.
 *   Alg.1 = AMC, Alg.2 = SMM, Alg.3 = GEER.
 *   Eq.6 refined ell, Eq.8 Bernstein f, Eq.9 eta* (P:319),
 *   Eq.10 psi, Eq.15 greedy switch, h = (2^tau-1) eta.
 * Readings where the paper is silent are numbered R1..R19 and listed in DESIGN.md
 * ("Readings of the paper"); the ones used here are cited inline.
 *
 * Compile: gcc -O2 -fopenmp -ffp-contract=off -shared -fPIC (no FMA contraction, so
 * every fp64 expression is evaluated exactly as written).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <omp.h>

/* ------------------------------------------------------------------------- */
/* Philox4x32-10 (Salmon, Moraes, Dror, Shaw, SC'11).  The paper is silent on   */
/* the RNG (R10); both sides implement this counter-based generator so walks   */
/* are reproducible bit for bit.                                               */
/* ------------------------------------------------------------------------- */
void oracle_philox4x32_10(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4])
{
    uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
    uint32_t k0 = key_in[0], k1 = key_in[1];
    for (int round = 0; round < 10; round++) {
        if (round > 0) {
            k0 += 0x9E3779B9u; /* golden ratio */
            k1 += 0xBB67AE85u; /* sqrt(3)-1 */
        }
        uint64_t p0 = (uint64_t)0xD2511F53u * (uint64_t)c0;
        uint64_t p1 = (uint64_t)0xCD9E8D57u * (uint64_t)c2;
        uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
        uint32_t n0 = hi1 ^ c1 ^ k0;
        uint32_t n1 = lo1;
        uint32_t n2 = hi0 ^ c3 ^ k1;
        uint32_t n3 = lo0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* MurmurHash3 fmix64, used only for the order-independent walk checksum (R20). */
static uint64_t fmix64(uint64_t x)
{
    x ^= x >> 33;
    x *= 0xff51afd7ed558ccdULL;
    x ^= x >> 33;
    x *= 0xc4ceb9fe1a85ec53ULL;
    x ^= x >> 33;
    return x;
}

uint64_t oracle_walk_hash(uint32_t q, uint32_t b, uint32_t side, uint64_t k, int32_t endpoint)
{
    uint64_t h = fmix64((uint64_t)q + ((uint64_t)b << 32) + ((uint64_t)side << 40));
    h = fmix64(h ^ k);
    h = fmix64(h ^ (uint64_t)(uint32_t)endpoint);
    return h;
}

/* ------------------------------------------------------------------------- */
/* Closed-form quantities                                                     */
/* ------------------------------------------------------------------------- */

/* Eq.6 (Thm 3.1): ell = ceil( log((2/d_s+2/d_t)/(eps(1-lambda))) / log(1/lambda) - 1 ),
 * natural log (R2), clamped below at 0 (R3). */
int64_t oracle_refined_ell(int64_t ds, int64_t dt, double eps, double lambda)
{
    double arg = (2.0 / (double)ds + 2.0 / (double)dt) / (eps * (1.0 - lambda));
    double x = log(arg) / log(1.0 / lambda) - 1.0;
    double c = ceil(x);
    if (c < 0.0) c = 0.0;
    return (int64_t)c;
}

/* Eq.5, Peng et al.'s degree-free ell; a variant knob. */
int64_t oracle_peng_ell(double eps, double lambda)
{
    double arg = 4.0 / (eps - eps * lambda);
    double x = log(arg) / log(1.0 / lambda) - 1.0;
    double c = ceil(x);
    if (c < 0.0) c = 0.0;
    return (int64_t)c;
}

/* Eq.10: psi = 2 ceil(lf/2)(max1(s)/ds + max1(t)/dt) + 2 floor(lf/2)(max2(s)/ds + max2(t)/dt). */
double oracle_psi(int64_t lf, double max1s, double max2s, double max1t, double max2t,
                  int64_t ds, int64_t dt)
{
    double cu = (double)((lf + 1) / 2); /* ceil(lf/2) */
    double fl = (double)(lf / 2);       /* floor(lf/2) */
    double a = max1s / (double)ds + max1t / (double)dt;
    double b = max2s / (double)ds + max2t / (double)dt;
    return 2.0 * cu * a + 2.0 * fl * b;
}

/* Eq.9: eta* = 2 psi^2 log(2 tau/delta) / eps^2 (real-valued). */
double oracle_eta_star(double psi, double eps, double delta, int tau)
{
    double L = log(2.0 * (double)tau / delta);
    return 2.0 * psi * psi * L / (eps * eps);
}

/* Alg.1 L2: eta0 = ceil(eta_star / 2^(tau-1)), floored at 1 (R6). */
int64_t oracle_eta0(double eta_star, int tau)
{
    double c = ceil(eta_star / ldexp(1.0, tau - 1));
    if (c < 1.0) c = 1.0;
    return (int64_t)c;
}

/* h(lf) = sum_{i=1..tau} 2^(i-1) eta0 = (2^tau - 1) eta0. */
int64_t oracle_h(int64_t eta0, int tau)
{
    return (((int64_t)1 << tau) - 1) * eta0;
}

/* Eq.8 (Lemma 3.2): f(n, var, psi, d) = sqrt(2 var log(3/d)/n) + 3 psi log(3/d)/n. */
double oracle_bernstein_f(double n, double var, double psi, double d)
{
    double L = log(3.0 / d);
    return sqrt(2.0 * var * L / n) + 3.0 * psi * L / n;
}

/* ------------------------------------------------------------------------- */
/* One application of P = D^-1 A with the row-stochastic reading R1:   */
/*   x'(u) = (1/d(u)) * sum_{w in N(u)} x(w), summed in CSR order of row u.     */
/* normalize = 0 applies A instead (used only to pin the propagation against    */
/* the integer #path rows of Fig.3).                                */
/* Dense, full pass over all rows: the plain definition.                        */
/* ------------------------------------------------------------------------- */
void oracle_propagate_dense(int64_t n, const int64_t *off, const int32_t *cols,
                            const double *x, double *y, int normalize)
{
    for (int64_t u = 0; u < n; u++) {
        double sum = 0.0;
        for (int64_t e = off[u]; e < off[u + 1]; e++) sum += x[cols[e]];
        y[u] = normalize ? sum / (double)(off[u + 1] - off[u]) : sum;
    }
}

/* ------------------------------------------------------------------------- */
/* Per-thread scratch: dense length-n vectors (SPEC's DenseVec).      */
/* ------------------------------------------------------------------------- */
typedef struct {
    double *xs, *xt, *tmp, *y;   /* s_star, t_star, next-iterate scratch, y = s_star/ds - t_star/dt */
    int32_t *supp_s, *supp_t;    /* support lists (sorted ascending) */
    int64_t ns, nt;              /* support sizes */
    int32_t *cand;               /* candidate rows for the next iterate */
    uint8_t *mark;
} scratch_t;

static int cmp_i32(const void *a, const void *b)
{
    int32_t x = *(const int32_t *)a, y = *(const int32_t *)b;
    return (x > y) - (x < y);
}

/*
 * x <- P x restricted to the rows that can be nonzero.  Rows outside
 * N(supp(x)) have an all-zero sum, so skipping them yields the same vector as
 * oracle_propagate_dense, bit for bit (adding +0.0 to a non-negative running sum
 * never changes it).  Returns the new support (sorted ascending, values != 0, R14).
 */
static void smm_step(int64_t n, const int64_t *off, const int32_t *cols, scratch_t *sc,
                     double *x, int32_t *supp, int64_t *nsupp)
{
    (void)n;
    int64_t nc = 0;
    for (int64_t i = 0; i < *nsupp; i++) {
        int32_t v = supp[i];
        for (int64_t e = off[v]; e < off[v + 1]; e++) {
            int32_t u = cols[e];
            if (!sc->mark[u]) { sc->mark[u] = 1; sc->cand[nc++] = u; }
        }
    }
    qsort(sc->cand, (size_t)nc, sizeof(int32_t), cmp_i32);
    for (int64_t i = 0; i < nc; i++) {
        int32_t u = sc->cand[i];
        double sum = 0.0;
        for (int64_t e = off[u]; e < off[u + 1]; e++) sum += x[cols[e]];
        sc->tmp[u] = sum / (double)(off[u + 1] - off[u]);
    }
    for (int64_t i = 0; i < *nsupp; i++) x[supp[i]] = 0.0;
    int64_t ns = 0;
    for (int64_t i = 0; i < nc; i++) {
        int32_t u = sc->cand[i];
        sc->mark[u] = 0;
        double val = sc->tmp[u];
        sc->tmp[u] = 0.0;
        if (val != 0.0) { x[u] = val; supp[ns++] = u; }
    }
    *nsupp = ns;
}

/* max_1 and max_2 (k-th largest value of the length-n vector; R5: the
 * second order statistic of the multiset, so ties give max2 = max1 and a
 * vector with one nonzero entry has max2 = 0). */
static void top2(const double *x, const int32_t *supp, int64_t ns, double *m1, double *m2)
{
    double a = 0.0, b = 0.0;
    for (int64_t i = 0; i < ns; i++) {
        double v = x[supp[i]];
        if (v > a) { b = a; a = v; }
        else if (v > b) { b = v; }
    }
    *m1 = a; *m2 = b;
}

static int64_t volume(const int64_t *off, const int32_t *supp, int64_t ns)
{
    int64_t vol = 0;
    for (int64_t i = 0; i < ns; i++) vol += off[supp[i] + 1] - off[supp[i]];
    return vol;
}

/* Oracle's own per-query record (field meaning in DESIGN.md "Per-query stats"). */
typedef struct {
    int32_t ell, ell_b, ell_f, batches_run;
    int64_t eta0, walks_total, steps_total, vol_last, h_last;
    double psi, r_b, r_f, f_last, sigma2_last;
    double rb_terms[8];
    uint64_t walk_checksum;
    uint32_t tie_flags;
    uint32_t pad;
} oracle_stats_t;

typedef struct {
    int tau;
    uint64_t seed;
    int64_t query_index_base;
    int force_ell_b;   /* -1: Eq.15 decides ell_b; >=0: run exactly min(force, ell) SMM iterations */
    int ell_variant;   /* 0: Eq.6 (refined), 1: Eq.5 (Peng) */
    double switch_ratio;  /* SURVEY 8(f)#4 variant: stop the SMM head iff vol > switch_ratio * h (1.0 = Eq.15) */
    int reuse_samples;    /* SURVEY 8(f)#4 variant: batch b keeps batch b-1's eta samples and adds eta new ones */
} oracle_opts_t;

/*
 * One simple random walk of lf steps (at each visited node v move to a
 * neighbour with probability 1/d(v)); the walk record excludes its start and
 * counts repeats (R9).  Step j (1-based) consumes half of Philox call
 * c = (j-1)/2 with counter (c, k mod 2^32, q, b<<29 | side<<28 | k>>32) and key
 * (seed_lo, seed_hi); odd j uses words (x0,x1), even j (x2,x3), r64 = hi<<32|lo;
 * neighbour index = floor(r64 * d / 2^64) into the row in input CSR order (R10).
 * acc = sum of y over visited nodes, sequential in step order.
 */
static int32_t walk(const int64_t *off, const int32_t *cols, const double *y,
                    int32_t start, int64_t lf, uint64_t seed, uint32_t q, uint32_t b,
                    uint32_t side, uint64_t k, double *acc_out, int32_t *trace)
{
    uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    uint32_t ctr[4], r[4];
    int32_t v = start;
    double acc = 0.0;
    for (int64_t j = 1; j <= lf; j++) {
        if (j & 1) {
            ctr[0] = (uint32_t)((j - 1) / 2);
            ctr[1] = (uint32_t)k;
            ctr[2] = q;
            ctr[3] = (b << 29) | (side << 28) | (uint32_t)(k >> 32);
            oracle_philox4x32_10(ctr, key, r);
        }
        uint64_t r64 = (j & 1) ? (((uint64_t)r[1] << 32) | r[0]) : (((uint64_t)r[3] << 32) | r[2]);
        uint64_t d = (uint64_t)(off[v + 1] - off[v]);
        uint64_t idx = (uint64_t)(((unsigned __int128)r64 * d) >> 64);
        v = cols[off[v] + (int64_t)idx];
        if (y) acc += y[v];
        if (trace) trace[j - 1] = v;
    }
    *acc_out = acc;
    return v;
}

/* Exposed for tests: one walk with the bit-level contract above (y may be NULL). */
int32_t oracle_walk(const int64_t *off, const int32_t *cols, const double *y, int32_t start,
                    int64_t lf, uint64_t seed, uint32_t q, uint32_t b, uint32_t side, uint64_t k,
                    double *acc_out, int32_t *trace)
{
    return walk(off, cols, y, start, lf, seed, q, b, side, k, acc_out, trace);
}

/*
 * Exposed for tests: Z_k samples of one AMC batch (Alg.1 L6-L7) for
 * arbitrary non-negative dense vectors xs, xt:
 *   Z_k = sum_{u in S_k}(xs(u)/ds - xt(u)/dt) + sum_{u in T_k}(xt(u)/dt - xs(u)/ds)
 * computed as acc_S - acc_T with y = xs/ds - xt/dt.
 */
void oracle_amc_samples(int64_t n, const int64_t *off, const int32_t *cols,
                        int32_t s, int32_t t, const double *xs, const double *xt, int64_t lf,
                        uint64_t seed, uint32_t q, uint32_t b, int64_t count, double *out_z)
{
    double ds = (double)(off[s + 1] - off[s]), dt = (double)(off[t + 1] - off[t]);
    double *y = (double *)malloc(sizeof(double) * (size_t)n);
    for (int64_t v = 0; v < n; v++) y[v] = xs[v] / ds - xt[v] / dt;
    #pragma omp parallel for schedule(static)
    for (int64_t k = 0; k < count; k++) {
        double aS, aT;
        walk(off, cols, y, s, lf, seed, q, b, 0, (uint64_t)k, &aS, NULL);
        walk(off, cols, y, t, lf, seed, q, b, 1, (uint64_t)k, &aT, NULL);
        out_z[k] = aS - aT;
    }
    free(y);
}

static int near_int_tie(double x)
{
    double r = nearbyint(x);
    double scale = fabs(x) > 1.0 ? fabs(x) : 1.0;
    return fabs(x - r) <= 1e-12 * scale;
}

/*
 * GEER for one query (Alg.3, calling Alg.1 at L10).  Returns r'.
 */
static double geer_one(int64_t n, const int64_t *off, const int32_t *cols, double lambda,
                       int32_t s, int32_t t, uint32_t q, double eps, double delta,
                       const oracle_opts_t *o, scratch_t *sc, oracle_stats_t *st)
{
    memset(st, 0, sizeof(*st));
    if (s == t) return 0.0;                          /* r(s,s) = 0, R19 */
    const int tau = o->tau;
    const int64_t ds = off[s + 1] - off[s], dt = off[t + 1] - off[t];
    const double dsf = (double)ds, dtf = (double)dt;

    /* Alg.3 L1: ell by Eq.6 (or Eq.5 as a variant). */
    int64_t ell;
    if (o->ell_variant == 1) ell = oracle_peng_ell(eps, lambda);
    else ell = oracle_refined_ell(ds, dt, eps, lambda);
    {
        double arg = (o->ell_variant == 1) ? 4.0 / (eps - eps * lambda)
                                           : (2.0 / dsf + 2.0 / dtf) / (eps * (1.0 - lambda));
        double x = log(arg) / log(1.0 / lambda) - 1.0;
        if (x > 0.0 && near_int_tie(x)) st->tie_flags |= 1u;
    }
    st->ell = (int32_t)ell;

    /* Alg.3 L2-L4: ell_b = 0, s* = e_s, t* = e_t, r_b = s*(s)/ds + t*(t)/dt - s*(t)/ds - t*(s)/dt. */
    double *xs = sc->xs, *xt = sc->xt;
    xs[s] = 1.0; sc->supp_s[0] = s; sc->ns = 1;
    xt[t] = 1.0; sc->supp_t[0] = t; sc->nt = 1;
    double r_b = xs[s] / dsf + xt[t] / dtf - xs[t] / dsf - xt[s] / dtf;
    int64_t ell_b = 0;
    double psi = 0.0;
    int64_t eta0 = 0;

    if (ell == 0) {
        /* R3: Thm 3.1 covers ell = 0, so r_ell = r_b; no SMM, no AMC. */
        st->r_b = r_b;
        xs[s] = 0.0; xt[t] = 0.0;
        return r_b;
    }

    /* Alg.3 L5-L9: repeat { s* <- P s*; t* <- P t*; r_b += ...; ell_b++ } until Eq.15 or ell_b >= ell (R4). */
    int64_t max_iters = (o->force_ell_b >= 0) ? (o->force_ell_b < ell ? o->force_ell_b : ell) : ell;
    if (o->force_ell_b == 0) {
        /* AMC-only (Thm 3.4 setting): s = e_s, t = e_t, lf = ell. */
        double m1s, m2s, m1t, m2t;
        top2(xs, sc->supp_s, sc->ns, &m1s, &m2s);
        top2(xt, sc->supp_t, sc->nt, &m1t, &m2t);
        psi = oracle_psi(ell, m1s, m2s, m1t, m2t, ds, dt);
        double es = oracle_eta_star(psi, eps, delta, tau);
        eta0 = oracle_eta0(es, tau);
    }
    while (ell_b < max_iters) {
        smm_step(n, off, cols, sc, xs, sc->supp_s, &sc->ns);
        smm_step(n, off, cols, sc, xt, sc->supp_t, &sc->nt);
        double term = xs[s] / dsf + xt[t] / dtf - xs[t] / dsf - xt[s] / dtf;
        r_b += term;
        if (ell_b < 8) st->rb_terms[ell_b] = term;
        ell_b += 1;
        /* Eq.15 left side: vol = sum_{v in V_s} d(v) + sum_{v in V_t} d(v). */
        int64_t vol = volume(off, sc->supp_s, sc->ns) + volume(off, sc->supp_t, sc->nt);
        /* Eq.15 right side: h(ell - ell_b) from psi on the CURRENT s*, t* (R4). */
        double m1s, m2s, m1t, m2t;
        top2(xs, sc->supp_s, sc->ns, &m1s, &m2s);
        top2(xt, sc->supp_t, sc->nt, &m1t, &m2t);
        psi = oracle_psi(ell - ell_b, m1s, m2s, m1t, m2t, ds, dt);
        double es = oracle_eta_star(psi, eps, delta, tau);
        eta0 = oracle_eta0(es, tau);
        if (ell - ell_b > 0 && near_int_tie(es / ldexp(1.0, tau - 1))) st->tie_flags |= 2u;
        int64_t h = oracle_h(eta0, tau);
        st->vol_last = vol;
        st->h_last = h;
        if (o->force_ell_b < 0 && (o->switch_ratio == 1.0 ? vol > h : (double)vol > o->switch_ratio * (double)h))
            break;
    }
    st->ell_b = (int32_t)ell_b;
    st->r_b = r_b;
    const int64_t lf = ell - ell_b;
    st->ell_f = (int32_t)lf;

    double r_f = 0.0;
    if (lf > 0) {
        /* Alg.1 with s = s*, t = t*, lf = ell - ell_b. */
        st->psi = psi;
        st->eta0 = eta0;
        double *y = sc->y;
        /* y(v) = s*(v)/d(s) - t*(v)/d(t) on supp(s*) U supp(t*), 0 elsewhere. */
        for (int64_t i = 0; i < sc->ns; i++) { int32_t v = sc->supp_s[i]; y[v] = xs[v] / dsf - xt[v] / dtf; }
        for (int64_t i = 0; i < sc->nt; i++) { int32_t v = sc->supp_t[i]; y[v] = xs[v] / dsf - xt[v] / dtf; }
        const double dprime = delta / (double)tau;   /* f(., ., psi, delta/tau), Alg.1 L13 */
        int64_t eta = eta0;
        uint64_t ck = 0;
        double S1 = 0.0, S2 = 0.0;
        int64_t k_new = 0;                            /* reuse variant: walks drawn so far */
        for (int b = 0; b < tau; b++) {
            int64_t k_lo = 0;
            uint32_t bkey = (uint32_t)b;
            if (o->reuse_samples) {
                k_lo = k_new;                         /* keep samples 0..k_new-1, draw k_new..eta-1 */
                bkey = 0;                             /* a sample's stream does not depend on the batch */
            } else {
                S1 = 0.0;                             /* Alg.1 L4: Z <- 0, sigma^2 <- 0 (fresh batch, R8) */
                S2 = 0.0;
            }
            for (int64_t k = k_lo; k < eta; k++) {
                double aS, aT;
                int32_t eS = walk(off, cols, y, s, lf, o->seed, q, bkey, 0, (uint64_t)k, &aS, NULL);
                int32_t eT = walk(off, cols, y, t, lf, o->seed, q, bkey, 1, (uint64_t)k, &aT, NULL);
                double Zk = aS - aT;                  /* Alg.1 L7 */
                S1 += Zk;                             /* L8 */
                S2 += Zk * Zk;                        /* L9 */
                ck += oracle_walk_hash(q, bkey, 0, (uint64_t)k, eS);
                ck += oracle_walk_hash(q, bkey, 1, (uint64_t)k, eT);
            }
            double Z = S1 / (double)eta;              /* L11 */
            double var = S2 / (double)eta - Z * Z;    /* L12 (one-pass form, R7) */
            if (var < 0.0) var = 0.0;
            double f = oracle_bernstein_f((double)eta, var, psi, dprime);
            st->batches_run = b + 1;
            st->walks_total += eta - k_lo;
            st->steps_total += 2 * (eta - k_lo) * lf;
            k_new = eta;
            st->f_last = f;
            st->sigma2_last = var;
            r_f = Z;
            if (fabs(f - eps / 2.0) <= 1e-12 * eps) st->tie_flags |= 4u;
            if (f <= eps / 2.0) break;                /* L13 */
            eta = 2 * eta;                            /* L14 */
        }
        st->walk_checksum = ck;
        for (int64_t i = 0; i < sc->ns; i++) y[sc->supp_s[i]] = 0.0;
        for (int64_t i = 0; i < sc->nt; i++) y[sc->supp_t[i]] = 0.0;
    }
    st->r_f = r_f;
    for (int64_t i = 0; i < sc->ns; i++) xs[sc->supp_s[i]] = 0.0;
    for (int64_t i = 0; i < sc->nt; i++) xt[sc->supp_t[i]] = 0.0;
    return r_f + r_b;                                 /* Alg.3 L11 */
}

/*
 * Batch entry point: out_r[i] = GEER(pairs[2i], pairs[2i+1]) with global query
 * index q = query_index_base + i.  stats may be NULL.  nthreads <= 0: OpenMP default.
 * Returns 0 on success, 1 on invalid arguments.
 */
int oracle_geer_batch(int64_t n, const int64_t *off, const int32_t *cols, double lambda,
                      const int32_t *pairs, int64_t k, double eps, double delta,
                      const oracle_opts_t *o, int nthreads, double *out_r, oracle_stats_t *stats)
{
    if (n <= 1 || k < 0 || !(eps > 0.0) || !(delta > 0.0 && delta < 1.0)) return 1;
    if (!(lambda > 0.0 && lambda < 1.0) || o->tau < 1 || o->tau > 8) return 1;
    for (int64_t i = 0; i < 2 * k; i++) if (pairs[i] < 0 || pairs[i] >= n) return 1;
    if (nthreads <= 0) nthreads = omp_get_max_threads();
    #pragma omp parallel num_threads(nthreads)
    {
        scratch_t sc;
        sc.xs = (double *)calloc((size_t)n, sizeof(double));
        sc.xt = (double *)calloc((size_t)n, sizeof(double));
        sc.tmp = (double *)calloc((size_t)n, sizeof(double));
        sc.y = (double *)calloc((size_t)n, sizeof(double));
        sc.supp_s = (int32_t *)malloc(sizeof(int32_t) * (size_t)n);
        sc.supp_t = (int32_t *)malloc(sizeof(int32_t) * (size_t)n);
        sc.cand = (int32_t *)malloc(sizeof(int32_t) * (size_t)n);
        sc.mark = (uint8_t *)calloc((size_t)n, 1);
        #pragma omp for schedule(dynamic, 1)
        for (int64_t i = 0; i < k; i++) {
            oracle_stats_t st;
            double r = geer_one(n, off, cols, lambda, pairs[2 * i], pairs[2 * i + 1],
                                (uint32_t)(o->query_index_base + i), eps, delta, o, &sc, &st);
            out_r[i] = r;
            if (stats) stats[i] = st;
        }
        free(sc.xs); free(sc.xt); free(sc.tmp); free(sc.y);
        free(sc.supp_s); free(sc.supp_t); free(sc.cand); free(sc.mark);
    }
    return 0;
}

/*
 * SMM alone (Alg.2) for tests: r_b after ell_b iterations, with the
 * per-iteration series terms written to terms[0..ell_b-1] (may be NULL), and the
 * final dense s*, t* copied to xs_out/xt_out (may be NULL).
 */
double oracle_smm(int64_t n, const int64_t *off, const int32_t *cols, int32_t s, int32_t t,
                  int64_t ell_b, double *terms, double *xs_out, double *xt_out)
{
    double *xs = (double *)calloc((size_t)n, sizeof(double));
    double *xt = (double *)calloc((size_t)n, sizeof(double));
    double *tmp = (double *)malloc(sizeof(double) * (size_t)n);
    const double dsf = (double)(off[s + 1] - off[s]), dtf = (double)(off[t + 1] - off[t]);
    xs[s] = 1.0; xt[t] = 1.0;
    double r_b = xs[s] / dsf + xt[t] / dtf - xs[t] / dsf - xt[s] / dtf;
    for (int64_t i = 0; i < ell_b; i++) {
        oracle_propagate_dense(n, off, cols, xs, tmp, 1); memcpy(xs, tmp, sizeof(double) * (size_t)n);
        oracle_propagate_dense(n, off, cols, xt, tmp, 1); memcpy(xt, tmp, sizeof(double) * (size_t)n);
        double term = xs[s] / dsf + xt[t] / dtf - xs[t] / dsf - xt[s] / dtf;
        if (terms) terms[i] = term;
        r_b += term;
    }
    if (xs_out) memcpy(xs_out, xs, sizeof(double) * (size_t)n);
    if (xt_out) memcpy(xt_out, xt, sizeof(double) * (size_t)n);
    free(xs); free(xt); free(tmp);
    return r_b;
}

int oracle_sizeof_stats(void) { return (int)sizeof(oracle_stats_t); }
int oracle_max_threads(void) { return omp_get_max_threads(); }
