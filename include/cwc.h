/*
 * cwc.h -- C ABI of the B200-native bulk stochastic simulator for CWC models
 * with a fixed compartment tree (Aldinucci et al., "On Designing
 * Multicore-aware Simulators for Biological Systems", arXiv:1010.2438).
 *
 * Citations: P:n = line n of the paper text, S:n = line n of the
 * SPEC.md written from it.  DESIGN.md gives the readings of the paper that
 * these functions implement.
 *
 * What the library computes (Fig. fig:simd P:605-641):
 *   for every trajectory g = point * n_replicas + replica (replicas and
 *   parameter-sweep instances), Gillespie's direct method over the
 *   mass-action rules of the model, sampled at t_j = j * sample_dt
 *   (j = 0 .. J, J = floor(t_end / sample_dt)), with the samples merged
 *   on-line (schema iii) into exact integer moments per
 *   (point, sample, observable): count, sum, sum of squares.
 *
 * Conventions for every function:
 *   - return CWC_OK (0) or a negative cwc_status; the message of the last
 *     failure on the calling thread is cwc_last_error();
 *   - "host" pointers are read during the call only (the caller keeps
 *     ownership); "device" pointers are caller-owned CUDA device memory;
 *   - nothing here allocates device memory except the model's own tables
 *     (uploaded on first use, owned by the handle, freed by cwc_model_destroy);
 *   - cwc_simulate is asynchronous on the caller's stream: it validates and
 *     enqueues, then returns.  Device-side outcomes (STALLED, OVERFLOW) are
 *     reported per trajectory, never as errors;
 *   - there is no CPU fallback: without a usable CUDA device every call that
 *     launches work returns CWC_ERR_CUDA.
 */
#ifndef CWC_H
#define CWC_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    CWC_OK = 0,
    CWC_ERR_INVALID = -1,     /* bad argument: message names which */
    CWC_ERR_UNSUPPORTED = -2, /* valid CWC but outside this build (e.g. reaction order > 2) */
    CWC_ERR_CUDA = -3,        /* CUDA runtime error (message carries cudaGetErrorString) */
    CWC_ERR_NOMEM = -4        /* device or host allocation failed */
} cwc_status;

/* Per-trajectory outcome codes written to cwc_sim_opts.out_status.
   RUNNING: suspended by a resumable run's bound (cwc_run_advance), not done. */
enum { CWC_TRAJ_DONE = 0, CWC_TRAJ_STALLED = 1, CWC_TRAJ_OVERFLOW = 2, CWC_TRAJ_RUNNING = 3 };

/* Which kernel runs the SSA loop. */
enum { CWC_PATH_AUTO = -1, CWC_PATH_THREAD = 0, CWC_PATH_WARP = 1 };

/* Kernel variant (cwc_sim_opts.kernel).  AUTO = the planner's
   choice.  THREAD_WS: warp-specialised producer/consumer thread kernel;
   THREAD: single-warp batched thread kernel, one trajectory per lane;
   THREAD2: the same kernel with two trajectories per lane (M <= 8, one-shot
   runs); THREAD_WS2: warp-specialised with two trajectories per consumer
   lane (M <= 8, one-shot runs); WARP2: two trajectories per warp (16-lane segments, M <= 256);
   WARP8: eight trajectories per warp (4-lane groups, M <= 256, one-shot runs, one global
   statistics part); WARP4: four per warp (8-lane groups, the same conditions);
   WARP: one trajectory per warp.  Every
   variant computes the same trajectories (up to the traced a0-sum-order
   class between the thread and warp families). */
enum { CWC_KERNEL_AUTO = 0, CWC_KERNEL_THREAD_WS = 1, CWC_KERNEL_THREAD = 2, CWC_KERNEL_WARP2 = 3,
       CWC_KERNEL_WARP = 4, CWC_KERNEL_THREAD2 = 5, CWC_KERNEL_THREAD_WS2 = 6, CWC_KERNEL_WARP8 = 7,
       CWC_KERNEL_WARP4 = 8 };

/* Where the on-line moments accumulate (cwc_sim_opts.stats_mode): per-CTA
   shared-memory parts flushed to global memory, or one global part updated
   with L2 reductions.  Results are identical bit for bit. */
enum { CWC_STATS_AUTO = 0, CWC_STATS_SHARED = 1, CWC_STATS_GLOBAL = 2 };

typedef struct cwc_model_s *cwc_model; /* opaque; owned by the library */

/*
 * A CWC model over a FIXED compartment tree.  All arrays
 * are host memory, copied by cwc_model_create.
 *
 * Compartments c = 0 .. n_compartments-1; c = 0 is the top level (type 0),
 * parent[0] = -1 and 0 <= parent[c] < c for c > 0 (index order is the
 * preorder in which Match recurses).  Each compartment holds
 * n_species counters; cell = c * n_species + s.
 *
 * Rule r is the stochastic rewrite rule  label : P --k--> O.  Its
 * pattern lives in a context compartment of type rule_label[r]; when
 * rule_child_label[r] >= 0 the pattern also contains one child compartment
 * of that type, and reactants/products may sit in it (where = 1) instead of
 * in the context (where = 0) -- membrane transport and similar rules.
 * Reactants/products are CSR lists (re_ptr[n_rules+1], pr_ptr[n_rules+1])
 * of (where, species, mult).  Mass action: the rate of one match is
 * k * prod binomial(n, mult) over reactant cells;
 * total reactant multiplicity per rule must be <= 2.
 *
 * Observables: obs_of_cell[cell] in [0, n_obs) or -1; the value of
 * observable o is the sum of its cells' counts (e.g. per compartment type
 * totals).
 */
typedef struct {
    int32_t n_types;
    int32_t n_species;
    int32_t n_compartments;
    const int32_t *parent;           /* [n_compartments] */
    const int32_t *type;             /* [n_compartments], in [0, n_types) */
    int32_t n_rules;
    const int32_t *rule_label;       /* [n_rules] context type */
    const int32_t *rule_child_label; /* [n_rules] -1 = local rule */
    const int32_t *re_ptr;           /* [n_rules + 1] */
    const int32_t *re_where;         /* [re_ptr[n_rules]] 0 context, 1 child */
    const int32_t *re_species;
    const int32_t *re_mult;          /* >= 1 */
    const int32_t *pr_ptr;           /* [n_rules + 1] */
    const int32_t *pr_where;
    const int32_t *pr_species;
    const int32_t *pr_mult;
    const double *rate;              /* [n_rules] finite, > 0 */
    const int32_t *init;             /* [n_compartments * n_species] >= 0 */
    int32_t n_obs;
    const int32_t *obs_of_cell;      /* [n_compartments * n_species] */
} cwc_model_desc;

/*
 * Parameter sweep: n_points instances of the model whose
 * rules rule[0..n_swept) take rate value[p * n_swept + i] at point p.  Host
 * memory.  NULL sweep = one point with the model's own rates.
 */
typedef struct {
    int32_t n_points;
    int32_t n_swept;
    const int32_t *rule;   /* [n_swept] */
    const double *value;   /* [n_points * n_swept], finite, > 0 */
} cwc_sweep;

/*
 * On-line reduced statistics, device memory, layout [point][sample][obs]
 * (n_cells = n_points * (J+1) * n_obs).  Exact integers (SPEC S:398-405 with
 * exact moments instead of Welford): count, sum of v, sum of v^2 as 128-bit
 * little-endian (lo, hi) pairs, so merge order cannot change any bit.
 */
typedef struct {
    int64_t *count;   /* [n_cells] */
    int64_t *sum;     /* [n_cells] */
    uint64_t *sumsq;  /* [n_cells][2] */
} cwc_stats;

/*
 * Optional outputs and knobs; every pointer may be NULL (device memory).
 */
typedef struct {
    int64_t *out_traj;      /* [G][J+1][n_obs] sampled observables (validation dumps) */
    int64_t *out_firings;   /* [G] applied events per trajectory */
    int32_t *out_status;    /* [G] CWC_TRAJ_* */
    /* per-firing trace for up to n_trace trajectories (divergence tracer):
       record = 5 doubles (n, a0, tau, t', mu; mu = -1 for the final drawn,
       not applied, block); trace_buf is [n_trace][trace_cap][5], trace_len
       [n_trace] receives the number of records written. trace_g is HOST. */
    const int64_t *trace_g;
    int32_t n_trace;
    int64_t trace_cap;
    double *trace_buf;
    int64_t *trace_len;
    int32_t force_path;     /* CWC_PATH_* */
    int32_t block_threads;  /* 0 = library choice; else threads per CTA (multiple of 32, <= 256) */
    /* sharding across GPUs / calls: this call runs replicas
       [replica_offset, replica_offset + n_replicas) of every point out of
       replicas_total, so trajectory g = point * replicas_total + replica keys
       the RNG exactly as in an unsharded run; outputs stay indexed by the
       local (point, replica).  replicas_total = 0 means n_replicas. */
    int64_t replica_offset;
    int64_t replicas_total;
    /* optional cudaEvent_t pair recorded on cuda_stream right before and
       after the SSA kernel (kernel-only timing); NULL = not recorded */
    void *ev_kernel_begin;
    void *ev_kernel_end;
    /* Launch-plan overrides, 0 = the library's choice (for A/B measurements
       and tests; none changes a result bit).  kernel: CWC_KERNEL_*, must fit
       force_path and the model (CWC_ERR_INVALID otherwise); stats_mode:
       CWC_STATS_* (SHARED fails with CWC_ERR_INVALID if the parts do not fit
       in shared memory); warps_per_block: warp kernels, 1..4;
       blocks_per_sm: warp kernels' persistent grid, 1..32 (capped by
       occupancy).  Traced runs (n_trace > 0) run the same variant as
       untraced ones, with trace writes compiled in. */
    int32_t kernel;
    int32_t stats_mode;
    int32_t warps_per_block;
    int32_t blocks_per_sm;
    /* optional cudaEvent_t pair recorded on cuda_stream right before and
       after the stage-2 reduction of the moments (its HBM bandwidth) */
    void *ev_stage2_begin;
    void *ev_stage2_end;
} cwc_sim_opts;

/* Summary of a created model (cwc_model_info). */
typedef struct {
    int32_t n_cells;        /* n_compartments * n_species */
    int32_t n_reactions;    /* M: flat (rule, context[, child]) entries */
    int32_t n_obs;
    int32_t n_rules;
    int32_t path;           /* CWC_PATH_THREAD or CWC_PATH_WARP chosen by CWC_PATH_AUTO */
    int32_t thread_path_ok; /* 1 if the thread path can run this model */
    int32_t max_deps;       /* largest dependency-graph row |D(mu)| */
    int32_t n_nu;           /* total (cell, delta) entries over all reactions */
    int64_t n_deps;         /* total dependency-graph entries */
} cwc_model_info;

/*
 * Validate desc, flatten the rules over the tree (rule-major, then context in
 * index order, then child in index order -- P:610), build the net
 * change table and the dependency graph D(mu) = {m : reactants(m) meet
 * cells changed by mu}.  Host only: the tables are uploaded to the current
 * CUDA device by the first cwc_simulate* call (CWC_ERR_CUDA there when no
 * device is usable) and freed by cwc_model_destroy.
 * Errors: CWC_ERR_INVALID (non-finite or <= 0 rate, bad tree, index out of
 * range, child reactant on a local rule, negative init, mult < 1),
 * CWC_ERR_UNSUPPORTED (reaction order > 2), CWC_ERR_CUDA / CWC_ERR_NOMEM.
 */
cwc_status cwc_model_create(const cwc_model_desc *desc, cwc_model *out);
void cwc_model_destroy(cwc_model model);
cwc_status cwc_model_info_get(cwc_model model, cwc_model_info *info);

/*
 * Copy the flattening out to HOST arrays (any may be NULL):
 * entry_rule/entry_context/entry_child [M]; reactants CSR re_ptr [M+1],
 * re_cell/re_mult [re_ptr[M]]; net change CSR nu_ptr [M+1], nu_cell/nu_delta
 * [n_nu]; dependency CSR dep_ptr [M+1], dep [n_deps].
 */
cwc_status cwc_model_get_flat(cwc_model model, int32_t *entry_rule, int32_t *entry_context,
                              int32_t *entry_child, int32_t *re_ptr, int32_t *re_cell, int32_t *re_mult,
                              int32_t *nu_ptr, int32_t *nu_cell, int32_t *nu_delta,
                              int32_t *dep_ptr, int32_t *dep);

/* The launch plan cwc_simulate would use for these arguments (host only,
 * no device work): which kernel, its grid, and the statistics accumulators
 * (for measurement: bench.py's roofline and stage-2 bandwidth). */
typedef struct {
    int32_t kernel;          /* CWC_KERNEL_* actually launched (never AUTO) */
    int32_t blocks;          /* CTAs of the SSA kernel */
    int32_t threads;         /* threads per CTA */
    int32_t stats_shared;    /* 1: per-CTA shared-memory parts, 0: one global part */
    int64_t smem_bytes;      /* dynamic shared memory per CTA */
    int64_t n_parts;         /* statistics parts stage 2 reduces */
    int64_t part_cells;      /* cells per part */
    int32_t word_bytes;      /* bytes per accumulator word (4 shared, 8 global) */
    int32_t words_per_cell;  /* count word + sum limbs + sum-of-squares limbs */
    int64_t n_stat_cells;    /* output cells: points * (J+1) * n_obs */
    int64_t workspace_bytes; /* = cwc_simulate_workspace_size */
} cwc_plan_info;
cwc_status cwc_plan(cwc_model model, int64_t n_replicas, const cwc_sweep *sweep, double t_end, double sample_dt,
                    const cwc_sim_opts *opts, cwc_plan_info *info);

/* Workspace (device bytes) cwc_simulate needs for these arguments. */
cwc_status cwc_simulate_workspace_size(cwc_model model, int64_t n_replicas, const cwc_sweep *sweep,
                                       double t_end, double sample_dt, const cwc_sim_opts *opts,
                                       size_t *bytes);

/*
 * Run n_points * n_replicas trajectories to t_end with seed and write the
 * reduced statistics (zeroed by the library first) to out_stats, all
 * enqueued on cuda_stream (a cudaStream_t; NULL = legacy default stream).
 * Random numbers: one Philox4x32-10 block per loop iteration, counter
 * (firing index n, trajectory g), key seed.
 * Errors: CWC_ERR_INVALID (t_end <= 0, sample_dt <= 0, sample_dt > t_end,
 * n_replicas < 1, bad sweep, workspace too small, path not possible),
 * CWC_ERR_CUDA.
 */
cwc_status cwc_simulate(cwc_model model, int64_t n_replicas, const cwc_sweep *sweep, double t_end,
                        double sample_dt, uint64_t seed, void *cuda_stream, cwc_stats out_stats,
                        void *workspace, size_t workspace_bytes, const cwc_sim_opts *opts);

/*
 * Same run with HOST output: host_stats arrays are host memory (pinned for
 * overlap, pageable accepted); the statistics are computed into the
 * workspace and copied device->host on cuda_stream.  The call returns after
 * enqueueing; synchronise the stream before reading host_stats.
 * Workspace: cwc_simulate_workspace_size + 32 bytes per statistics cell.
 */
cwc_status cwc_simulate_host(cwc_model model, int64_t n_replicas, const cwc_sweep *sweep, double t_end,
                             double sample_dt, uint64_t seed, void *cuda_stream, cwc_stats host_stats,
                             void *workspace, size_t workspace_bytes);
cwc_status cwc_simulate_host_workspace_size(cwc_model model, int64_t n_replicas, const cwc_sweep *sweep,
                                            double t_end, double sample_dt, size_t *bytes);

/*
 * mean = sum / count; var = (count * sumsq - sum^2) / (count (count - 1))
 * (0 when count == 1): numerator (192-bit) and denominator (126-bit) are
 * exact integers and each quotient is rounded to nearest-even ONCE (exact
 * long division with a sticky bit), so mean and var are the correctly
 * rounded values of the exact rationals; ci90 = 1.6449 * sqrt(var / count)
 * in IEEE fp64 operations.  NaN where
 * count == 0.  Device -> device over n_cells, on cuda_stream.
 */
cwc_status cwc_stats_finalize(const cwc_stats *stats, int64_t n_cells, double *mean, double *var,
                              double *ci90, void *cuda_stream);

/* Device Philox4x32-10 blocks for (seed, g[i], n[i]) -> out[i][4] (device
 * arrays); the exact function the SSA kernels draw with.  Test hook. */
cwc_status cwc_philox_blocks(uint64_t seed, const int64_t *g, const int64_t *n, int64_t count,
                             uint32_t *out, void *cuda_stream);

/* Device draws (E = -log u1, u2) of Philox blocks (seed, g[i], n[i]) exactly
 * as the SSA kernels form them (reading 3): E[i], u2[i]
 * (device double arrays).  Test hook for the kernels' branch-free log. */
cwc_status cwc_draws(uint64_t seed, const int64_t *g, const int64_t *n, int64_t count, double *E, double *u2,
                     void *cuda_stream);

/* Uniforms u1[i], u2[i] (reading 3) and E[i] = -log u1[i] of the raw
 * Philox output blocks words[i][0..3] (device uint32 [count][4]; device double
 * outputs), formed exactly as the SSA kernels form them.  Test hook for the
 * conversion edges (all-zero and all-one words, the top bit). */
cwc_status cwc_block_draws(const uint32_t *words, int64_t count, double *u1, double *u2, double *E,
                           void *cuda_stream);

/* q[i] = e[i] / a[i] computed the way the SSA kernels compute tau = E / a0
 * (P:206-207): the branch-free fast division where its range guard holds,
 * IEEE div.rn otherwise.  Must equal the IEEE quotient bit for bit.  Device
 * arrays.  Test hook. */
cwc_status cwc_tau_div(const double *e, const double *a, int64_t count, double *q, void *cuda_stream);

/*
 * Resumable runs.  The paper's schema (ii)
 * makes every simulation instance an object that holds its progress, so a
 * scheduler can stop it and restart it later -- in (fixed or variable)
 * slices, on any worker; schema (iii) reduces a running window of
 * the trajectories while they advance almost aligned in simulated time.  Here
 * the whole progress of trajectory g is (x, t, n, j): counts, time, applied
 * firings n (= its Philox counter) and next sample j (j = J+1: finished).  A
 * suspended trajectory therefore resumes bit-exactly, and a run split into
 * any sequence of advances produces exactly the statistics, firings, status
 * and samples of one cwc_simulate call with the same arguments.
 *
 * `state` is ONE caller-owned device buffer of cwc_run_state_size bytes that
 * holds everything the run needs between calls: per-trajectory state, the
 * live list, the per-point rates and the statistics accumulators.  The
 * library keeps nothing between calls, so copying the buffer to host memory
 * and back (to this or another device) is a checkpoint; the layout is
 * private but fixed for given arguments.  Every cwc_run_* call on one state
 * must pass the same model, n_replicas, sweep, t_end, sample_dt and
 * (force_path, replica_offset, replicas_total) of opts; the kernel choice
 * may differ from cwc_simulate's (the warp-specialised thread kernel is not
 * used), the results do not.  opts->n_trace must be 0.
 */
cwc_status cwc_run_state_size(cwc_model model, int64_t n_replicas, const cwc_sweep *sweep, double t_end,
                              double sample_dt, const cwc_sim_opts *opts, size_t *bytes);

/* Start a run: every trajectory at (x0, t = 0, n = 0, j = 0), all live
 * (listed longest-expected-first for sweeps), statistics zeroed.  Also stores
 * the per-point rates (host expansion of sweep) and a fingerprint of the
 * arguments (model tables, rates, shape, replica shard) in the state header;
 * every later cwc_run_advance / cwc_run_stats on the state checks it
 * (CWC_ERR_INVALID on a mismatch), and the first advance records the seed,
 * which later advances must repeat.  Enqueued on cuda_stream; returns after
 * the header has been written (synchronises the stream).
 * Errors: as cwc_simulate, CWC_ERR_INVALID for a short state. */
cwc_status cwc_run_init(cwc_model model, int64_t n_replicas, const cwc_sweep *sweep, double t_end,
                        double sample_dt, const cwc_sim_opts *opts, void *state, size_t state_bytes,
                        void *cuda_stream);

/* Advance every live trajectory by at most `quantum` further applied firings
 * (0 = no bound; the bound is checked once per batch / 32-draw window, so a
 * trajectory may run a few firings past it) and at most up to sample j_stop:
 * a trajectory suspends, before drawing into effect, once all its samples
 * j < j_stop are recorded (j_stop = J+1, or 0, = no bound).  Then drops the
 * finished trajectories from the live list (order kept), so the next advance
 * launches only unfinished ones, in dense warps.  With a j_stop bound and no
 * quantum, every live trajectory ends the call at j = j_stop: the statistics
 * of samples < j_stop are final (the running window of schema iii).
 * opts->out_firings / out_status receive the cumulative firings and status
 * (CWC_TRAJ_RUNNING = suspended) of the trajectories this call ran;
 * out_traj the samples it recorded.  *n_pending (HOST) receives the number
 * of trajectories that still have samples below j_stop to record (with
 * j_stop = J+1: the unfinished ones; 0 = the window, or the run, is
 * complete); the call synchronises cuda_stream to read it (n_pending may be
 * NULL: it still synchronises).  seed must be the same in every advance of a
 * run (it keys the trajectories' Philox streams; checked against the seed
 * the first advance recorded).
 * Errors: CWC_ERR_INVALID (quantum < 0, j_stop outside [0, J+1], state too
 * small, its header corrupt or its fingerprint different from these
 * arguments / seed, the argument errors of cwc_simulate),
 * CWC_ERR_CUDA. */
cwc_status cwc_run_advance(cwc_model model, int64_t n_replicas, const cwc_sweep *sweep, double t_end,
                           double sample_dt, uint64_t seed, const cwc_sim_opts *opts, int64_t quantum,
                           int64_t j_stop, void *state, size_t state_bytes, void *cuda_stream,
                           int64_t *n_pending);

/* Reduce the run's accumulators into out_stats (device, as cwc_simulate's):
 * cells of samples every trajectory has passed are final; the others hold
 * the partial sums so far.  Reads the state header first (synchronises
 * cuda_stream; CWC_ERR_INVALID if the fingerprint does not match these
 * arguments), then enqueues the reduction on cuda_stream. */
cwc_status cwc_run_stats(cwc_model model, int64_t n_replicas, const cwc_sweep *sweep, double t_end,
                         double sample_dt, const cwc_sim_opts *opts, const void *state, size_t state_bytes,
                         cwc_stats out_stats, void *cuda_stream);

/* Thread-local message of the last failure on this thread ("" if none). */
const char *cwc_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* CWC_H */
