/*
 * ssa_oracle.c -- plain, slow, single-threaded CPU oracle of the hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this code.  It
 * shares no code, header, table or constant generator with the CUDA path in
 * paper_1010_2438_b200/ (DESIGN.md "Oracle").
 *
 * What it computes, step by step in the paper's order (PAPER.md P:199-242,
 * Fig. fig:simd P:605-641), on a model already flattened by oracle/flatten.py:
 *
 *   loop:                                          Simulation_Step
 *     a[m] = k_m * (double) h_m(x)  for all m      Match / Match_Populations:
 *                                                  h = prod binomial(n, k)
 *     a0 = ((a[0] + a[1]) + a[2]) + ...            r = sum r_i
 *     if a0 == 0: stall
 *     draw one Philox4x32-10 block, counter (n, g), key seed; n += 1
 *     u1 in (0,1], u2 in [0,1)
 *     tau = (-log u1) / a0 ; tn = t + tau          step 1
 *     while j <= J and j*dt <= tn: record(j, x)    fixed-step sampling,
 *                                                  pre-event state
 *     if j > J: DONE (event drawn, not applied)
 *     target = u2 * a0; mu = min{m: target < sum_{i<=m} a_i}   step 2
 *     x += nu[mu]   (OVERFLOW if a count leaves int32)          Update
 *     t = tn ; firings += 1                        simclock += tau
 *
 *   record(j, x): for each observable o: v = sum of its cells;
 *     count[p][j][o] += 1; sum += v; sumsq += v*v  (exact integers)
 *
 * Compile with -O2 -ffp-contract=off (no FMA contraction, no -ffast-math);
 * log() is glibc's.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ---- Philox4x32-10 (Salmon, Moraes, Dror, Shaw, SC'11), restated ------- */
void oracle_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4])
{
    uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
    uint32_t k0 = key[0], k1 = key[1];
    for (int round = 0; round < 10; ++round) {
        if (round > 0) {             /* key schedule between rounds */
            k0 += 0x9E3779B9u;
            k1 += 0xBB67AE85u;
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

/* Block for firing n of trajectory g (BASELINE north_star:
 * "keyed by (seed, replica, firing index)"). */
static void draw_block(uint64_t seed, uint64_t g, uint64_t n, uint32_t w[4])
{
    uint32_t ctr[4] = {(uint32_t)n, (uint32_t)(n >> 32), (uint32_t)g, (uint32_t)(g >> 32)};
    uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    oracle_philox4x32_10(ctr, key, w);
}

/* u1 = (((w0<<32 | w1) >> 11) + 1) * 2^-53 in (0,1];  u2 = ((w2<<32 | w3) >> 11) * 2^-53 in [0,1) */
void oracle_uniforms(const uint32_t w[4], double *u1, double *u2)
{
    uint64_t a = ((uint64_t)w[0] << 32) | w[1];
    uint64_t b = ((uint64_t)w[2] << 32) | w[3];
    *u1 = (double)((a >> 11) + 1) * 0x1.0p-53;
    *u2 = (double)(b >> 11) * 0x1.0p-53;
}

/* tau = (-log u1) / a0: one negation, glibc log, one IEEE division
 * (SURVEY 8(c).4).  The one place the loop forms tau. */
double oracle_tau(double u1, double a0)
{
    return (-log(u1)) / a0;
}

/* The (tau, u2) pair the loop draws for firings n0 .. n0+count-1 of trajectory g
 * at a fixed total rate a0: tau = (-log u1) / a0.  Test hook. */
void oracle_tau_stream(uint64_t seed, uint64_t g, uint64_t n0, int64_t count, double a0,
                       double *tau_out, double *u2_out)
{
    for (int64_t i = 0; i < count; ++i) {
        uint32_t w[4];
        draw_block(seed, g, n0 + (uint64_t)i, w);
        double u1, u2;
        oracle_uniforms(w, &u1, &u2);
        tau_out[i] = oracle_tau(u1, a0);
        u2_out[i] = u2;
    }
}

/* binomial(n, k): number of k-subsets of n identical-type molecules,
 * exact integer multiplicative formula; 0 when k > n. */
int64_t oracle_binomial(int64_t n, int64_t k)
{
    if (k < 0 || n < 0 || k > n) return 0;
    unsigned __int128 r = 1;
    for (int64_t i = 1; i <= k; ++i) r = r * (unsigned __int128)(n - k + i) / (unsigned __int128)i;
    return (int64_t)r;
}

typedef struct {
    int32_t n_cells;              /* n_compartments * n_species */
    int32_t n_reactions;          /* M, flat entries */
    int32_t n_obs;
    const int32_t *re_ptr;        /* [M+1] CSR over reactant (cell, mult) */
    const int32_t *re_cell;
    const int32_t *re_mult;
    const int32_t *nu_ptr;        /* [M+1] CSR over net change (cell, delta) */
    const int32_t *nu_cell;
    const int32_t *nu_delta;
    const int32_t *rule_of;       /* [M] rule index of each entry */
    const int32_t *init;          /* [n_cells] */
    const int32_t *obs_of_cell;   /* [n_cells], -1 = not observed */
} oracle_model;

enum { ST_DONE = 0, ST_STALLED = 1, ST_OVERFLOW = 2 };

/* Match: a[m] = k[m] * (double) prod_q binomial(x[cell_q], mult_q) */
void oracle_propensities(const oracle_model *m, const double *k, const int64_t *x, double *a)
{
    for (int r = 0; r < m->n_reactions; ++r) {
        int64_t h = 1;
        for (int q = m->re_ptr[r]; q < m->re_ptr[r + 1]; ++q)
            h *= oracle_binomial(x[m->re_cell[q]], m->re_mult[q]);
        a[r] = k[r] * (double)h;
    }
}

/* Resolve, step 2: mu = min{m : target < a[0] + ... + a[m]} with the
 * cumulative sum formed left to right; if no such m (impossible when a0 is the
 * same left-to-right sum and target = u2*a0, u2 < 1) the last entry with a > 0. */
int oracle_select(const double *a, int M, double target)
{
    double c = 0.0;
    for (int r = 0; r < M; ++r) {
        c = c + a[r];
        if (target < c) return r;
    }
    for (int r = M - 1; r >= 0; --r)
        if (a[r] > 0.0) return r;
    return -1;
}

typedef struct {
    const oracle_model *m;
    int64_t J;
    int64_t *st_count;            /* [P][J+1][O] or NULL */
    int64_t *st_sum;
    uint64_t *st_sumsq;           /* [P][J+1][O][2] (lo, hi) */
    int64_t *traj_row;            /* [J+1][O] for this trajectory or NULL */
    int64_t p;
} recorder;

static void record(const recorder *rc, int64_t j, const int64_t *x)
{
    const oracle_model *m = rc->m;
    int O = m->n_obs;
    for (int o = 0; o < O; ++o) {
        int64_t v = 0;
        for (int c = 0; c < m->n_cells; ++c)
            if (m->obs_of_cell[c] == o) v += x[c];
        if (rc->traj_row) rc->traj_row[j * O + o] = v;
        if (rc->st_count) {
            int64_t cell = (rc->p * (rc->J + 1) + j) * O + o;
            rc->st_count[cell] += 1;
            rc->st_sum[cell] += v;
            unsigned __int128 q = (unsigned __int128)rc->st_sumsq[2 * cell] |
                                  ((unsigned __int128)rc->st_sumsq[2 * cell + 1] << 64);
            q += (unsigned __int128)((uint64_t)v) * (unsigned __int128)((uint64_t)v);
            rc->st_sumsq[2 * cell] = (uint64_t)q;
            rc->st_sumsq[2 * cell + 1] = (uint64_t)(q >> 64);
        }
    }
}

/*
 * Simulate the trajectories g_list[0..n_g) (g = point * n_replicas + replica).
 * rule_rates: [P][n_rules] rate constants per sweep point.
 * Outputs (any may be NULL): traj [n_g][J+1][O], firings [n_g], status [n_g],
 * stats [P][J+1][O] (count, sum, sumsq lo/hi) accumulated (caller zeroes),
 * trace: for trajectory trace_g, one record per drawn block:
 *   (n, a0, tau, tn, mu)  as 5 doubles (mu = -1 for the final undrawn-into-effect block).
 * Returns 0, or -1 on bad arguments.
 */
int oracle_simulate(const oracle_model *m, int32_t n_rules, const double *rule_rates,
                    int64_t n_points, int64_t n_replicas, const int64_t *g_list, int64_t n_g,
                    double t_end, double dt, uint64_t seed,
                    int64_t *traj, int64_t *firings_out, int32_t *status_out,
                    int64_t *st_count, int64_t *st_sum, uint64_t *st_sumsq,
                    int64_t trace_g, double *trace, int64_t trace_cap, int64_t *trace_n)
{
    if (!(t_end > 0) || !(dt > 0) || dt > t_end || n_replicas < 1) return -1;
    const int64_t J = (int64_t)floor(t_end / dt);
    const int M = m->n_reactions, NC = m->n_cells, O = m->n_obs;
    int64_t *x = (int64_t *)malloc(sizeof(int64_t) * (NC > 0 ? NC : 1));
    double *a = (double *)malloc(sizeof(double) * (M > 0 ? M : 1));
    double *k = (double *)malloc(sizeof(double) * (M > 0 ? M : 1));
    if (trace_n) *trace_n = 0;

    for (int64_t gi = 0; gi < n_g; ++gi) {
        const int64_t g = g_list[gi];
        const int64_t p = g / n_replicas;
        if (p >= n_points) { free(x); free(a); free(k); return -1; }
        for (int r = 0; r < M; ++r) k[r] = rule_rates[p * n_rules + m->rule_of[r]];
        for (int c = 0; c < NC; ++c) x[c] = m->init[c];
        recorder rc = {m, J, st_count, st_sum, st_sumsq, traj ? traj + gi * (J + 1) * O : NULL, p};
        double t = 0.0;
        uint64_t n = 0;
        int64_t j = 0, firings = 0;
        int status = ST_DONE;
        const int tracing = (trace && g == trace_g);

        for (;;) {
            /* 1. Match: propensities a_m = k_m * count_population */
            oracle_propensities(m, k, x, a);
            double a0 = 0.0;
            for (int r = 0; r < M; ++r) a0 = (r == 0) ? a[0] : a0 + a[r];
            if (a0 == 0.0) {                       /* stall: no rule applicable */
                for (; j <= J; ++j) record(&rc, j, x);
                status = ST_STALLED;
                break;
            }
            /* 2. Resolve: tau ~ Exp(a0), mu with probability a_mu / a0 */
            uint32_t w[4];
            draw_block(seed, (uint64_t)g, n, w);
            n += 1;
            double u1, u2;
            oracle_uniforms(w, &u1, &u2);
            double tau = oracle_tau(u1, a0);
            double tn = t + tau;
            while (j <= J && (double)j * dt <= tn) {     /* samples before the event */
                record(&rc, j, x);
                j += 1;
            }
            if (j > J) {
                if (tracing && *trace_n < trace_cap) {
                    double *rec = trace + 5 * (*trace_n)++;
                    rec[0] = (double)(n - 1); rec[1] = a0; rec[2] = tau; rec[3] = tn; rec[4] = -1.0;
                }
                status = ST_DONE;
                break;
            }
            double target = u2 * a0;
            int mu = oracle_select(a, M, target);
            if (tracing && *trace_n < trace_cap) {
                double *rec = trace + 5 * (*trace_n)++;
                rec[0] = (double)(n - 1); rec[1] = a0; rec[2] = tau; rec[3] = tn; rec[4] = (double)mu;
            }
            /* 3. Update: delete P_sigma, add O_sigma at the context */
            int overflow = 0;
            for (int q = m->nu_ptr[mu]; q < m->nu_ptr[mu + 1]; ++q)
                if (x[m->nu_cell[q]] + m->nu_delta[q] > INT32_MAX) overflow = 1;
            if (overflow) {                           /* event not applied; freeze */
                for (; j <= J; ++j) record(&rc, j, x);
                status = ST_OVERFLOW;
                break;
            }
            for (int q = m->nu_ptr[mu]; q < m->nu_ptr[mu + 1]; ++q)
                x[m->nu_cell[q]] += m->nu_delta[q];
            t = tn;                                   /* simclock += tau */
            firings += 1;
        }
        if (firings_out) firings_out[gi] = firings;
        if (status_out) status_out[gi] = status;
    }
    free(x); free(a); free(k);
    return 0;
}
