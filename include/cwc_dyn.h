/*
 * cwc_dyn.h -- C ABI of the dynamic-topology CWC simulator (SURVEY 8(f)
 * NEXT-4): bulk Gillespie SSA over CWC terms whose compartments are created,
 * dissolved, deleted and rewritten by the rules, with the same on-line
 * statistics as cwc.h.  Conventions (status codes, ownership, asynchrony,
 * no CPU fallback, cwc_last_error) are those of cwc.h.
 *
 * Citations: P:n = PAPER.md line n, S:n = SPEC.md line n; readings D1-D4 are
 * DESIGN.md section 2 reading 14 (the oracle oracle/dynamic.py follows the
 * same readings).
 *
 * The calculus:
 *   - a term is a multiset of atoms and compartments (wrap | content)^label
 *     (P:158-167); the top level is compartment 0 with label 0 (TOP);
 *   - a rule  label: P --k--> O has a pattern P = context
 *     atoms + the context's rest X + at most ONE child compartment pattern
 *     (label', wrap atoms + rest W | content atoms + rest Y) -- depth 1
 *     (S:38-49);
 *   - O = atoms added to the context, optionally X (without X the rest of
 *     the context -- atoms and compartments -- is deleted: sigma(O) replaces
 *     the whole matched content), optionally the matched child's W
 *     and / or Y released into the context (dissolution; Y's compartments
 *     move up one level), and compartment constructors (label'', atoms +
 *     optionally W | atoms + optionally Y).  A constructor carrying BOTH W and
 *     Y takes the matched child's list position (the child is rewritten in
 *     place); other constructors are appended to the context's list.  W and
 *     Y are each used at most once (reading D3).
 *   - matching (D1): one entry per (rule, context[, child]) with context
 *     compartments in PREORDER of the current term and children in list
 *     order; rate = k * RN(h), h = prod binomial(n, mult) over the pattern's
 *     context, wrap and content atoms, exact integers (Fig.
 *     fig:simd P:623-640: count_population * count_compartments * k);
 *   - one flat selection over the entries (D2), the RNG, tau, sampling,
 *     termination and stall rules of cwc.h (readings 3-7);
 *   - observables (D4): sums of keys ("content", label, atom) = total count
 *     of atom in the contents of all compartments of that label (label 0: the
 *     top level), ("wrap", label, atom), ("count", label) = number of
 *     compartments of that label; sampled pre-event at t_j = j * sample_dt.
 *
 * Device limits of this build (CWC_ERR_UNSUPPORTED at create): n_atoms <=
 * CWC_DYN_MAX_ATOMS, n_rules <= CWC_DYN_MAX_RULES, n_obs <= CWC_DYN_MAX_OBS,
 * reaction order (sum of pattern multiplicities) <= 2, constructors per rule
 * <= CWC_DYN_MAX_CTORS.  The term of a trajectory holds at most `capacity`
 * compartments including the top level (<= CWC_DYN_MAX_CAP) nested at most
 * CWC_DYN_MAX_DEPTH levels below it; a firing that would exceed either
 * leaves the trajectory frozen before that firing with status
 * CWC_TRAJ_CAPACITY (remaining samples take the frozen term, as for
 * OVERFLOW) -- a limit of the device representation, not of the calculus.
 */
#ifndef CWC_DYN_H
#define CWC_DYN_H

#include <stddef.h>
#include <stdint.h>

#include "cwc.h"

#ifdef __cplusplus
extern "C" {
#endif

enum { CWC_DYN_MAX_ATOMS = 16, CWC_DYN_MAX_RULES = 32, CWC_DYN_MAX_OBS = 32, CWC_DYN_MAX_CTORS = 4,
       CWC_DYN_MAX_CAP = 64, CWC_DYN_MAX_DEPTH = 7, CWC_DYN_MAX_KEYS = 64 };

/* Per-trajectory outcome beyond cwc.h's CWC_TRAJ_*: the term outgrew the
   device capacity (see above). */
enum { CWC_TRAJ_CAPACITY = 4 };

/* Pattern / constructor atom sides. */
enum { CWC_DYN_CTX = 0, CWC_DYN_WRAP = 1, CWC_DYN_CONTENT = 2 };
/* rule_flags bits */
enum { CWC_DYN_KEEP_X = 1, CWC_DYN_RELEASE_W = 2, CWC_DYN_RELEASE_Y = 4 };
/* ctor_flags bits */
enum { CWC_DYN_CTOR_W = 1, CWC_DYN_CTOR_Y = 2 };
/* observable key kinds */
enum { CWC_DYN_OBS_CONTENT = 0, CWC_DYN_OBS_WRAP = 1, CWC_DYN_OBS_COUNT = 2 };

typedef struct cwc_dyn_model_s *cwc_dyn_model; /* opaque; owned by the library */

/*
 * A dynamic CWC model.  All arrays are HOST memory, copied by
 * cwc_dyn_model_create.  Atoms are 0 .. n_atoms-1, labels 0 .. n_labels-1.
 *
 * Initial term: compartments in PREORDER; compartment 0 is the top level
 * (label 0, parent -1, wrap all 0); 0 <= comp_parent[c] < c and every
 * subtree is contiguous.  comp_wrap / comp_content are [n_comps][n_atoms]
 * counts >= 0.
 *
 * Rule r: context label rule_label[r]; child pattern label
 * rule_comp_label[r] (-1: none, else >= 1); rate[r] finite and >=
 * 2^-1021; rule_flags[r] (CWC_DYN_KEEP_X / RELEASE_W / RELEASE_Y; the
 * releases need a child pattern).  Pattern atoms: CSR lhs_ptr[n_rules+1] of
 * (lhs_side CWC_DYN_CTX / WRAP / CONTENT, lhs_atom, lhs_mult >= 1; WRAP and
 * CONTENT need a child pattern).  Atoms O adds to the context: CSR rhs_ptr of
 * (rhs_atom, rhs_mult >= 1).  Constructors: CSR ctor_ptr[n_rules+1] of
 * (ctor_label >= 1, ctor_flags CWC_DYN_CTOR_W / Y -- both need a child
 * pattern), each with atoms CSR ctor_atom_ptr[n_ctors+1] of (ctor_side
 * CWC_DYN_WRAP / CONTENT, ctor_atom, ctor_mult >= 1).
 *
 * Observables: obs_ptr[n_obs+1] CSR of keys (obs_kind, obs_label, obs_atom);
 * the value of observable o is the sum of its keys' values (D4).  WRAP and
 * COUNT keys need label >= 1; obs_atom is ignored for COUNT.
 */
typedef struct {
    int32_t n_atoms;
    int32_t n_labels;
    int32_t n_comps;
    const int32_t *comp_label;    /* [n_comps] */
    const int32_t *comp_parent;   /* [n_comps] */
    const int32_t *comp_wrap;     /* [n_comps * n_atoms] */
    const int32_t *comp_content;  /* [n_comps * n_atoms] */
    int32_t n_rules;
    const int32_t *rule_label;      /* [n_rules] */
    const int32_t *rule_comp_label; /* [n_rules] */
    const double *rate;             /* [n_rules] */
    const int32_t *rule_flags;      /* [n_rules] */
    const int32_t *lhs_ptr;         /* [n_rules + 1] */
    const int32_t *lhs_side;
    const int32_t *lhs_atom;
    const int32_t *lhs_mult;
    const int32_t *rhs_ptr;         /* [n_rules + 1] */
    const int32_t *rhs_atom;
    const int32_t *rhs_mult;
    const int32_t *ctor_ptr;        /* [n_rules + 1] */
    const int32_t *ctor_label;      /* [n_ctors] */
    const int32_t *ctor_flags;      /* [n_ctors] */
    const int32_t *ctor_atom_ptr;   /* [n_ctors + 1] */
    const int32_t *ctor_side;
    const int32_t *ctor_atom;
    const int32_t *ctor_mult;
    int32_t n_obs;
    const int32_t *obs_ptr;         /* [n_obs + 1] */
    const int32_t *obs_kind;
    const int32_t *obs_label;
    const int32_t *obs_atom;
} cwc_dyn_model_desc;

/* Optional outputs and knobs (every pointer may be NULL; device memory). */
typedef struct {
    int64_t *out_traj;       /* [G][J+1][n_obs] sampled observables */
    int64_t *out_firings;    /* [G] applied events per trajectory */
    int32_t *out_status;     /* [G] CWC_TRAJ_DONE / STALLED / OVERFLOW / CAPACITY */
    int64_t replica_offset;  /* sharding as in cwc_sim_opts: trajectory g = replica_offset + local replica */
    int64_t replicas_total;  /* 0 = n_replicas */
    int32_t capacity;        /* compartments per term incl. the top level; 0 = CWC_DYN_MAX_CAP */
    int32_t warps_per_block; /* 0 = library choice; else 1..8 */
    int32_t blocks_per_sm;   /* 0 = occupancy limit; else >= 1 (capped by occupancy) */
    int32_t pad_;
    void *ev_kernel_begin;   /* optional cudaEvent_t pair around the SSA kernel */
    void *ev_kernel_end;
} cwc_dyn_opts;

/* Summary of a created model and of the launch plan of a run. */
typedef struct {
    int32_t n_atoms, n_labels, n_rules, n_obs;
    int32_t n_structural;      /* rules whose firing changes the term's compartment structure */
    int32_t blocks, threads;   /* SSA kernel grid of the planned run (0 when queried without a run) */
    int32_t capacity;
    int64_t smem_bytes;        /* dynamic shared memory per CTA */
    int64_t n_stat_cells;      /* (J+1) * n_obs */
    int64_t workspace_bytes;
} cwc_dyn_info;

/*
 * Validate and compile desc: dense pattern / net-change tables per rule,
 * the structural classification (a rule is non-structural iff it keeps X,
 * releases nothing and either has no child pattern and no constructor or
 * rewrites the matched child in place with the same label), and the rule
 * dependency masks of the non-structural rules (rules whose entries read a
 * (label, side, atom) the firing changes).  Host only; tables are uploaded
 * per device on first use.
 * Errors: CWC_ERR_INVALID (index / label / atom out of range, term not a
 * preorder tree, negative counts, wrap on the top level, bad rate, side or
 * flag on a rule without a child pattern, W or Y used twice, observable key
 * out of range), CWC_ERR_UNSUPPORTED (device limits above).
 */
cwc_status cwc_dyn_model_create(const cwc_dyn_model_desc *desc, cwc_dyn_model *out);
void cwc_dyn_model_destroy(cwc_dyn_model model);

/* Model summary; with n_replicas > 0 also the plan of such a run (grid,
 * shared memory, statistics cells, workspace).  Host only. */
cwc_status cwc_dyn_info_get(cwc_dyn_model model, int64_t n_replicas, double t_end, double sample_dt,
                            const cwc_dyn_opts *opts, cwc_dyn_info *info);

/* Device workspace bytes cwc_dyn_simulate needs. */
cwc_status cwc_dyn_workspace_size(cwc_dyn_model model, int64_t n_replicas, double t_end, double sample_dt,
                                  const cwc_dyn_opts *opts, size_t *bytes);

/*
 * Run n_replicas trajectories of the model to t_end (one warp per
 * trajectory, persistent warps taking trajectory ids in order; the
 * trajectory id keys the Philox counter exactly as in cwc_simulate) and
 * write the exact on-line moments to out_stats (device, layout
 * [sample][obs], zeroed by the library; cwc_stats_finalize applies).
 * Asynchronous on cuda_stream.
 * Errors: CWC_ERR_INVALID (t_end <= 0, sample_dt <= 0 or > t_end,
 * n_replicas < 1, capacity outside [initial compartments, CWC_DYN_MAX_CAP],
 * workspace too small, bad shard, moments that could exceed int64),
 * CWC_ERR_CUDA.
 */
cwc_status cwc_dyn_simulate(cwc_dyn_model model, int64_t n_replicas, double t_end, double sample_dt, uint64_t seed,
                            void *cuda_stream, cwc_stats out_stats, void *workspace, size_t workspace_bytes,
                            const cwc_dyn_opts *opts);

#ifdef __cplusplus
}
#endif
#endif /* CWC_DYN_H */
