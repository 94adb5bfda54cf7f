// ssa_thread_impl.cuh -- one trajectory per CUDA thread (small networks).
//
// Hot path of BASELINE north_star (b): "one replica per thread with counts
// and propensities in registers ... for small networks".  Each thread runs
// Gillespie's direct method (loop of Fig. fig:simd P:608-621) for
// trajectory g = blockIdx.x * blockDim.x + threadIdx.x:
//
//   a_m   = k_m * double(h_m(x))                 Match, all M, registers
//   cum_m = cum_{m-1} + a_m, a0 = cum_{M-1}      left-to-right, as the oracle
//   tau   = E_n / a0, E_n = -log u1
//   samples j with j*dt <= t + tau get x (pre-event), on-line into the
//   block's shared-memory moment accumulators (schema iii)
//   mu    = #{m : cum_m <= u2 a0}                P:208-209 (cum is monotone)
//   x    += nu_mu                                Update
//
// Latency structure.  C1/C2 have fewer warps than the chip has schedulers,
// so a firing costs the latency of its dependent chain, not its issue slots.
// Only the state chain (x -> a -> a0 -> select -> x, and t += tau) is truly
// serial; the Philox block and -log u1 of every future firing are state-free
// (counter-based RNG).  The loop therefore runs in batches of B firings:
//   * the draws of the NEXT batch (B independent Philox + log chains, each
//     step B-wide, DrawPipe) are computed in four phases placed between the B
//     firings of this batch -- one straight-line block with no branches
//     (branch-free log and division), so the scheduler interleaves them;
//   * the B firings run speculatively: each step applies its update at once
//     (so the serial chain is only x -> a -> a0 -> select -> x) and records
//     whether it was "plain": no sample crossed (t + tau < t_next), a0 in the
//     fast-division range, no int32 overflow;
//   * after the batch, a lane whose batch held a non-plain firing rolls back
//     to the state before the first one and runs ONE exact iteration -- the
//     oracle's loop body verbatim (crossing records, stall, end, overflow,
//     IEEE division) -- then shifts its unused draws into place.
// The committed sequence of firings is therefore exactly the sequential
// algorithm's; batching only reorders independent RNG work.
//
// The cells and reactions are compile-time padded (S, M) so that x[] and the
// propensities stay in registers; reaction tables are kernel parameters
// (uniform constant-bank operands).  Net changes are packed int8 per cell
// and selected branch-free while scanning the cumulative sums.
#pragma once
#include <cuda_runtime.h>

#include "cwc_internal.h"
#include "device_common.cuh"

#ifndef CWC_T_MAXT  // single-warp thread kernel: CTA size bound and CTAs per SM (register budget)
#define CWC_T_MAXT 256
#endif
#ifndef CWC_T_MINB
#define CWC_T_MINB 1
#endif

namespace cwc {

template <int S>
__device__ __forceinline__ int pick(const int (&x)[S], int idx) {
    int v = 1;  // idx < 0: the constant 1 of an absent reactant
#pragma unroll
    for (int s = 0; s < S; ++s) v = (idx == s) ? x[s] : v;
    return v;
}

// Reactant gather x[ia[m]] as bit masks built once per thread (the indices
// are uniform, but 2*M*S compares do not fit in the predicate registers and
// would be re-evaluated every firing): xa = oa | OR_s (x[s] & ma[s]), where
// ma[s] = -1 iff ia == s and oa = 1 for an absent reactant (the constant 1).
template <int S, int M>
struct Gather {
    int ma[M][S], mb[M][S];
    int oa[M], ob[M];
    __device__ __forceinline__ explicit Gather(const ThreadTables &tt) {
#pragma unroll
        for (int m = 0; m < M; ++m) {
            oa[m] = tt.ia[m] < 0 ? 1 : 0;
            ob[m] = tt.ib[m] < 0 ? 1 : 0;
#pragma unroll
            for (int s = 0; s < S; ++s) {
                ma[m][s] = tt.ia[m] == s ? -1 : 0;
                mb[m][s] = tt.ib[m] == s ? -1 : 0;
            }
        }
    }
    __device__ __forceinline__ int a(const int (&x)[S], int m) const {
        int v = oa[m];
#pragma unroll
        for (int s = 0; s < S; ++s) v |= x[s] & ma[m][s];
        return v;
    }
    __device__ __forceinline__ int b(const int (&x)[S], int m) const {
        int v = ob[m];
#pragma unroll
        for (int s = 0; s < S; ++s) v |= x[s] & mb[m][s];
        return v;
    }
};

// cum_m = sum_{i<=m} a_i, left to right (== the oracle's a0 order).
template <int S, int M>
__device__ __forceinline__ void cumulative(const ThreadTables &tt, const Gather<S, M> &gt, const int (&x)[S],
                                           const double (&c)[M], double (&cum)[M]) {
#pragma unroll
    for (int m = 0; m < M; ++m) {
        const double a = __dmul_rn(c[m], combos(gt.a(x, m), gt.b(x, m), tt.sub[m], tt.shr[m]));
        cum[m] = (m == 0) ? a : __dadd_rn(cum[m - 1], a);
    }
}

// Packed net change of mu = #{m < M-1 : cum_m <= target} (first m with
// target < cum_m; padded reactions have a_m = 0 and never win).
template <int M, bool WANT_MU>
__device__ __forceinline__ unsigned long long select_nu(const ThreadTables &tt, const double (&cum)[M], double target,
                                                        int &mu) {
    unsigned long long nu = tt.nu_pack[0];
    int k = 0;
#pragma unroll
    for (int m = 0; m + 1 < M; ++m) {
        const bool past = cum[m] <= target;
        nu = past ? tt.nu_pack[m + 1] : nu;
        if (WANT_MU) k += past ? 1 : 0;
    }
    mu = k;
    return nu;
}

template <int S>
__device__ __forceinline__ bool apply_nu(const int (&x)[S], unsigned long long nu, int (&xn)[S]) {
    bool wrapped = false;
#pragma unroll
    for (int s = 0; s < S; ++s) {
        xn[s] = x[s] + (int)(signed char)(unsigned char)(nu >> (8 * s));
        wrapped |= (xn[s] < 0);  // counts are < 2^31 and |delta| <= 127: wrap <=> left int32
    }
    return wrapped;
}

// Per-firing values of a speculative firing, kept for the divergence trace
// (TRACE builds only; n, a0, tau, t', mu as the oracle's trace records).
struct FireRec {
    double a0, tau, tn;
    int mu;
};

// One speculative firing of the fast batch: propensities, a0, tau and the
// selection, update applied at once; returns whether the firing was "plain"
// (fast division valid -- a0 > 0 and in range --, no sample crossed, no count
// left int32).  For M <= 16 the reaction operands x[ia_m], x[ib_m] are kept as
// state and updated through op_pack (one compare chain selects the packed
// deltas of cells and operands), so the serial chain never gathers from x.
template <int S, int M>
struct FastChain {
    static constexpr bool OPND = (M <= 4 * kOpWords);
    static constexpr int NW = OPND ? (M + 3) / 4 : 1;  // operand delta words in use
    static constexpr bool COMB = OPND && 8 * S + 16 * M <= 64;  // ThreadTables.comb_pack
    int A[M], Bo[M];  // operands x[ia_m] and x[ib_m] - sub_m
    // k_m * 2^-shr_m (exact scaling): then a_m = k_m' * RN(x_a (x_b - sub)),
    // which equals k_m * RN(x_a (x_b - sub) / 2^shr) bit for bit (halving
    // commutes with rounding), with no 64-bit shift in the chain
    double ch[M];

    __device__ __forceinline__ void rates(const ThreadTables &tt, const double (&c)[M]) {
#pragma unroll
        for (int m = 0; m < M; ++m) ch[m] = tt.shr[m] ? __dmul_rn(c[m], 0.5) : c[m];
    }

    __device__ __forceinline__ void load(const ThreadTables &tt, const int (&x)[S]) {
        if constexpr (OPND) {
#pragma unroll
            for (int m = 0; m < M; ++m) {
                A[m] = pick(x, tt.ia[m]);
                Bo[m] = pick(x, tt.ib[m]) - tt.sub[m];
            }
        }
    }

    __device__ __forceinline__ bool step(const ThreadTables &tt, const Gather<S, M> &gt, const double (&c)[M],
                                         int (&x)[S], double &t, double E, double U, double t_next) {
        bool cross1;
        FireRec fr;
        return step2<false>(tt, gt, c, x, t, E, U, t_next, t_next, cross1, fr);
    }

    // As step(); additionally cross1 = the firing crossed exactly one sample
    // time (t_next <= t + tau < t_next2) and is otherwise plain.  TR: also
    // fill fr with the firing's (a0, tau, t', mu) for the trace (the same
    // arithmetic; mu = the number of cumulative sums <= target).
    template <bool TR>
    __device__ __forceinline__ bool step2(const ThreadTables &tt, const Gather<S, M> &gt, const double (&c)[M],
                                          int (&x)[S], double &t, double E, double U, double t_next, double t_next2,
                                          bool &cross1, FireRec &fr) {
        double cum[M];
        if constexpr (OPND) {
#pragma unroll
            for (int m = 0; m < M; ++m) {
                // RN(A Bo) as one fp64 product of the exact operands: equals
                // the int64 product rounded once (|A Bo| < 2^62), without the
                // quarter-rate int64 -> fp64 conversion on the state chain
                const double a = __dmul_rn(ch[m], __dmul_rn(i2d_exact(A[m]), i2d_exact(Bo[m])));
                cum[m] = (m == 0) ? a : __dadd_rn(cum[m - 1], a);
            }
        } else {
            cumulative(tt, gt, x, c, cum);
        }
        const double a0 = cum[M - 1];
        const double tau = div_fast(E, a0);
        const double tn = __dadd_rn(t, tau);
        const double target = __dmul_rn(U, a0);
        if (TR) {
            int k = 0;
#pragma unroll
            for (int m = 0; m + 1 < M; ++m) k += (cum[m] <= target) ? 1 : 0;
            fr.a0 = a0;
            fr.tau = tau;
            fr.tn = tn;
            fr.mu = k;
        }
        unsigned long long nu, op[NW];
        if constexpr (COMB) {
            unsigned long long cw = tt.comb_pack[0];
#pragma unroll
            for (int m = 0; m + 1 < M; ++m) cw = (cum[m] <= target) ? tt.comb_pack[m + 1] : cw;
            nu = cw;                // bytes 0 .. S-1 (apply_nu reads no more)
            op[0] = cw >> (8 * S);  // operand deltas
        } else {
            nu = tt.nu_pack[0];
#pragma unroll
            for (int w = 0; w < NW; ++w) op[w] = tt.op_pack[0][w];
#pragma unroll
            for (int m = 0; m + 1 < M; ++m) {
                const bool past = cum[m] <= target;
                nu = past ? tt.nu_pack[m + 1] : nu;
                if constexpr (OPND) {
#pragma unroll
                    for (int w = 0; w < NW; ++w) op[w] = past ? tt.op_pack[m + 1][w] : op[w];
                }
            }
        }
        int xn[S];
        const bool wrapped = apply_nu(x, nu, xn);
        const bool valid = div_fast_ok(E, a0) && !wrapped;
        const bool ok = valid && (tn < t_next);
        cross1 = valid && !(tn < t_next) && (tn < t_next2);
#pragma unroll
        for (int s = 0; s < S; ++s) x[s] = xn[s];
        t = tn;
        if constexpr (OPND) {
#pragma unroll
            for (int m = 0; m < M; ++m) {
                const unsigned long long w = op[m >> 2];
                A[m] += (int)(signed char)(unsigned char)(w >> (16 * (m & 3)));
                Bo[m] += (int)(signed char)(unsigned char)(w >> (16 * (m & 3) + 8));
            }
        }
        return ok;
    }
};

template <int S>
__device__ __forceinline__ void record_sample(const RunParams &rp, const ThreadTables &tt, const StatAcc &acc,
                                              const int (&x)[S], long long cell_base, long long g, long long j) {
    const int O = tt.O;
    for (int o = 0; o < O; ++o) {
        long long v = 0;
#pragma unroll
        for (int s = 0; s < S; ++s) v += (tt.obs_of[s] == o) ? (long long)x[s] : 0ll;
        stat_record(acc, cell_base + j * O + o, v);
        if (rp.out_traj) rp.out_traj[(g * (long long)(rp.J + 1) + j) * O + o] = v;
    }
}

// Stall fill, warp-cooperative: every lane in fm has stalled
// at sample j with frozen counts x; its remaining samples j .. JL all take
// the same observables.  The whole (converged) warp writes them, one sample
// per lane per pass, instead of the stalled lane alone (C3: trajectories
// whose substrate is used up stall early and fill up to 100 samples each).
template <int S>
__device__ __forceinline__ void stall_fill(const RunParams &rp, const ThreadTables &tt, const StatAcc &acc,
                                           unsigned fm, const int (&x)[S], long long cell_base, long long g,
                                           long long j, long long JL, int lane) {
    const int O = tt.O;
    const long long J1 = (long long)rp.J + 1;
    long long v[kThreadMaxObs];
#pragma unroll
    for (int o = 0; o < kThreadMaxObs; ++o) {
        v[o] = 0;
#pragma unroll
        for (int s = 0; s < S; ++s) v[o] += (tt.obs_of[s] == o) ? (long long)x[s] : 0ll;
    }
    while (fm) {
        const int src = __ffs(fm) - 1;
        fm &= fm - 1u;
        const long long cb = __shfl_sync(0xffffffffu, cell_base, src);
        const long long gs = __shfl_sync(0xffffffffu, g, src);
        const long long j0 = __shfl_sync(0xffffffffu, j, src);
        long long vs[kThreadMaxObs];
#pragma unroll
        for (int o = 0; o < kThreadMaxObs; ++o) vs[o] = __shfl_sync(0xffffffffu, v[o], src);
        for (long long jj = j0 + lane; jj <= JL; jj += 32) {
#pragma unroll
            for (int o = 0; o < kThreadMaxObs; ++o) {
                if (o < O) {
                    stat_record(acc, cb + jj * O + o, vs[o]);
                    if (rp.out_traj) rp.out_traj[(gs * J1 + jj) * O + o] = vs[o];
                }
            }
        }
    }
}

// One staged sample record, written by a lane of a full warp: the observables
// of the staged pre-event counts, into the moments (and the optional dump).
template <int S>
__device__ __forceinline__ void staged_record(const RunParams &rp, const ThreadTables &tt, const StatAcc &acc,
                                              long long cell, long long row, const int *xs) {
    int xv[S];
#pragma unroll
    for (int s = 0; s < S; ++s) xv[s] = xs[s];
    for (int o = 0; o < tt.O; ++o) {
        long long v = 0;
#pragma unroll
        for (int s = 0; s < S; ++s) v += (tt.obs_of[s] == o) ? (long long)xv[s] : 0ll;
        stat_record(acc, cell + o, v);
        if (rp.out_traj) rp.out_traj[row * tt.O + o] = v;
    }
}

#ifndef CWC_TB_SMALL  // speculative batch length for M <= 8 (experiment knob)
#define CWC_TB_SMALL 4
#endif
template <int M>
struct ThreadBatch {
    static constexpr int B = (M <= 8) ? CWC_TB_SMALL : (M <= 16 ? 2 : 1);
};

// RES: resumable runs (cwc_run_*: state load/save, launch bounds); the
// one-shot instantiations carry none of it.
// NT: trajectories per lane (1 or 2).  With NT = 2 a lane runs two
// trajectories (consecutive ids) whose batches are interleaved in one
// straight-line block: the two state chains are independent, so the
// in-order issue of a lone warp sees twice the instruction-level parallelism
// (C2 has fewer trajectory warps than the chip has sub-partitions; measured:
// two warps per sub-partition raise its firings/s 1.4x).  Each trajectory's
// batch is B / NT firings, so the draws in flight per lane stay B.
template <int S, int M, bool TRACE, bool RES, int NT>
#ifdef CWC_T_MAXNREG  // experiment builds: a per-thread register cap instead of the launch bounds
__global__ void __maxnreg__(CWC_T_MAXNREG) ssa_thread_kernel(const RunParams rp, const ThreadTables tt) {
#else
__global__ void __launch_bounds__(CWC_T_MAXT, CWC_T_MINB) ssa_thread_kernel(const RunParams rp, const ThreadTables tt) {
#endif
    constexpr int B = (NT == 2 && ThreadBatch<M>::B >= 2) ? ThreadBatch<M>::B / 2 : ThreadBatch<M>::B;
    static_assert(NT == 1 || NT == 2, "one or two trajectories per lane");
    extern __shared__ __align__(16) unsigned char smem[];
    const long long T = blockDim.x;
    // dispatch order: CTA slot blockIdx.x runs trajectory group cta (RunParams.cta_order)
    const long long cta = rp.cta_order ? (long long)__ldg(rp.cta_order + blockIdx.x) : (long long)blockIdx.x;
    const long long g0 = cta * T * NT;  // first launch slot of the CTA
    const int O = tt.O;
    const long long J = rp.J;
    const long long J1 = J + 1;

    // staged sample records of this warp (after the statistics part)
    const long long stats_part_bytes = rp.stats_smem ? stat_bytes(rp.st, rp.cells_per_part) : 0;
    long long *st_cell = (long long *)(smem + stats_part_bytes) + (long long)(threadIdx.x >> 5) * kStageLL;
    long long *st_row = st_cell + kWsStage;                   // [kWsStage] trajectory sample row (out_traj)
    int *st_x = (int *)(st_row + kWsStage);                   // [kWsStage][kThreadMaxCells] pre-event counts
    const int lane = threadIdx.x & 31;
    int stage_n = 0;  // warp-uniform
    // the CTA's copy of the -log table (after the staging areas of its warps)
    NegLogSmem *ltab = (NegLogSmem *)(smem + stats_part_bytes + (T >> 5) * kStageLL * (long long)sizeof(long long));
    neglog_smem_fill(ltab, threadIdx.x, (int)T);

    StatAcc acc;
    long long p_base = 0;
    if (rp.stats_smem) {
        acc = stat_view(smem, rp.cells_per_part, rp.st);
        uint4 *z = (uint4 *)smem;
        const long long n16 = stat_bytes(rp.st, rp.cells_per_part) / 16;
        for (long long i = threadIdx.x; i < n16; i += T) z[i] = make_uint4(0, 0, 0, 0);
        p_base = g0 / rp.R;
    } else {
        acc = stat_view((unsigned char *)rp.parts + (cta % rp.n_parts) * stat_bytes(rp.st, rp.cells_per_part),
                        rp.cells_per_part, rp.st);
    }

    __syncthreads();  // statistics part zeroed, table staged
    {
        // per-trajectory state (index i < NT); lanes past the last trajectory
        // stay in the warp-uniform loop as idle lanes (their loads use a valid
        // trajectory id; they never record)
        bool in_range[NT];
        long long g[NT], cell_base[NT];
        uint64_t gk[NT];
        int tslot[NT];
        double *trace[NT];
        long long tn_rec[NT];
        int x[NT][S];
        double t[NT];
        long long j[NT];
        unsigned long long n[NT], n_start[NT];
        double c[NT][M];
        FastChain<S, M> fc[NT];
        double t_next[NT], t_next2[NT];
        long long firings[NT];
        int status[NT];
        double Eb[NT][B], Ub[NT][B];
        bool live[NT];
        const Gather<S, M> gt(tt);
        const long long JL = RES ? rp.j_stop - 1 : J;  // last sample of this launch (J in one-shot runs)
#pragma unroll
        for (int i = 0; i < NT; ++i) {
            const long long slot = g0 + (long long)threadIdx.x * NT + i;
            in_range[i] = slot < rp.n_launch;
            g[i] = launch_traj(rp, in_range[i] ? slot : rp.n_launch - 1);
            const long long p = g[i] / rp.R;
            cell_base[i] = (p - p_base) * J1 * O;
            gk[i] = (uint64_t)global_traj(g[i], rp.R, rp.R_total, rp.r_off);  // RNG stream id
            tslot[i] = -1;
            trace[i] = nullptr;
            tn_rec[i] = 0;
            if (TRACE && in_range[i]) {
                for (int q = 0; q < rp.n_trace; ++q)
                    if (rp.trace_g[q] == g[i]) tslot[i] = q;
                if (tslot[i] >= 0) trace[i] = rp.trace_buf + (long long)tslot[i] * rp.trace_cap * 5;
            }
            // state: fresh (x0, t = 0, n = 0, j = 0) or resumed (cwc_run_advance)
#pragma unroll
            for (int s = 0; s < S; ++s)
                x[i][s] = (s < tt.n_cells) ? (RES ? rp.rs_x[g[i] * tt.n_cells + s] : tt.init[s]) : 0;
            t[i] = 0.0;
            j[i] = 0;
            n[i] = 0;
            if (RES) {
                t[i] = rp.rs_t[g[i]];
                j[i] = rp.rs_j[g[i]];
                n[i] = (unsigned long long)rp.rs_n[g[i]];
            }
            n_start[i] = n[i];
#pragma unroll
            for (int m = 0; m < M; ++m) c[i][m] = (m < tt.M) ? __ldg(rp.rates + p * tt.M + m) : 0.0;
            fc[i].rates(tt, c[i]);
            fc[i].load(tt, x[i]);
            t_next[i] = __dmul_rn(__ll2double_rn(j[i]), rp.dt);       // j * dt (fresh: sample 0 is crossed by the first firing)
            t_next2[i] = __dmul_rn(__ll2double_rn(j[i] + 1), rp.dt);  // (j + 1) * dt
            firings[i] = (long long)n[i];
            status[i] = CWC_TRAJ_DONE;
#pragma unroll
            for (int q = 0; q < B; ++q) block_to_draws(philox_block(rp.seed, gk[i], n[i] + q), Eb[i][q], Ub[i][q]);
            live[i] = in_range[i] && j[i] <= JL;
        }
        auto trace_rec = [&](int i, unsigned long long n_, double a0, double tau, double tn, int mu) {
            if (TRACE && tslot[i] >= 0 && tn_rec[i] < rp.trace_cap) {
                double *r = trace[i] + 5 * tn_rec[i]++;
                r[0] = (double)n_; r[1] = a0; r[2] = tau; r[3] = tn; r[4] = (double)mu;
            }
        };
        auto any_live = [&]() {
            bool l = false;
#pragma unroll
            for (int i = 0; i < NT; ++i) l = l || live[i];
            return l;
        };

        while (__any_sync(0xffffffffu, any_live())) {
            // ---- fast batch: B firings of every trajectory of the lane run
            // speculatively (every step commits its update); the four phases
            // of the next batch's draws (n0+B .. n0+2B-1, valid if all B
            // firings turn out plain) are interleaved with the steps so that
            // the scheduler can overlap their independent chains with the
            // serial state chains ----
            unsigned long long n0[NT];
            double En[NT][B], Un[NT][B];
            DrawPipe<B> pipe[NT];
            int xsnap[NT][B][S];
            double tsnap[NT][B];
            unsigned bad[NT];  // bit k: firing k of the batch is not plain
            // one firing per batch may cross a single sample time that is not
            // the last: it commits, its record (pre-event state) follows the batch
            // (at most one: it is the batch's only change of j, so the
            // per-firing bookkeeping is a few selects; the batch-start sample
            // times are kept for a rollback, and t_next3 = (j + 2) dt becomes
            // the next-but-one sample time after the crossing)
            bool rec[NT];
            int krec[NT];
            bool jok[NT];
            double t_next0[NT], t_next20[NT], t_next3[NT];
            FireRec fr[NT][B];
#pragma unroll
            for (int i = 0; i < NT; ++i) {
                n0[i] = n[i];
                pipe[i].start(gk[i], n0[i] + B);
                bad[i] = 0;
                rec[i] = false;
                krec[i] = B;
                jok[i] = j[i] < JL;
                t_next0[i] = t_next[i];
                t_next20[i] = t_next2[i];
                t_next3[i] = __dmul_rn(__ll2double_rn(j[i] + 2), rp.dt);
            }
#pragma unroll
            for (int k = 0; k < B; ++k) {
#pragma unroll
                for (int ph = 0; ph < 4; ++ph)
                    if ((ph * B) / 4 == k) {
#pragma unroll
                        for (int i = 0; i < NT; ++i) pipe[i].phase(ph, rp.rk, ltab, En[i], Un[i]);
                    }
#pragma unroll
                for (int i = 0; i < NT; ++i) {
#pragma unroll
                    for (int s = 0; s < S; ++s) xsnap[i][k][s] = x[i][s];
                    tsnap[i][k] = t[i];
                    bool cross1;
                    const bool plain = fc[i].template step2<TRACE>(tt, gt, c[i], x[i], t[i], Eb[i][k], Ub[i][k], t_next[i],
                                                                   t_next2[i], cross1, fr[i][k]);
                    const bool take = cross1 && !rec[i] && jok[i];
                    rec[i] = rec[i] || take;
                    krec[i] = take ? k : krec[i];
                    t_next[i] = take ? t_next2[i] : t_next[i];
                    t_next2[i] = take ? t_next3[i] : t_next2[i];
                    bad[i] |= (plain || take) ? 0u : (1u << k);
                }
            }
            long long jrec[NT];
#pragma unroll
            for (int i = 0; i < NT; ++i) {
                if (!live[i]) bad[i] = 1u;
                const int used = (bad[i] == 0u) ? B : __ffs(bad[i]) - 1;  // plain firings committed
                if (TRACE && live[i]) {  // trace records of the committed speculative firings
#pragma unroll
                    for (int k = 0; k < B; ++k)
                        if (k < used) trace_rec(i, n0[i] + k, fr[i][k].a0, fr[i][k].tau, fr[i][k].tn, fr[i][k].mu);
                }
                if (rec[i] && krec[i] >= used) {  // the crossing firing was rolled back
                    rec[i] = false;
                    t_next[i] = t_next0[i];
                    t_next2[i] = t_next20[i];
                }
                jrec[i] = j[i];  // the sample a committed crossing recorded
                if (rec[i]) j[i] += 1;
                if (live[i]) {
                    n[i] += (unsigned long long)used;
                    firings[i] += used;
                }
            }
            // records staged in shared memory, written 32 at a time (one per lane)
#pragma unroll
            for (int i = 0; i < NT; ++i) {
                const unsigned rmask = __ballot_sync(0xffffffffu, rec[i]);
                if (rmask) {
                    if (rec[i]) {  // few lanes: stage the counts only, observables are formed at the flush
                        const int sl = stage_n + __popc(rmask & ((1u << lane) - 1u));
                        st_cell[sl] = cell_base[i] + jrec[i] * O;
                        st_row[sl] = g[i] * J1 + jrec[i];
                        // pre-event counts of firing krec, by selects (no dynamic
                        // indexing of register arrays: local memory otherwise)
#pragma unroll
                        for (int s = 0; s < S; ++s) {
                            int v = xsnap[i][0][s];
#pragma unroll
                            for (int k = 1; k < B; ++k) v = (k == krec[i]) ? xsnap[i][k][s] : v;
                            st_x[sl * kThreadMaxCells + s] = v;
                        }
                    }
                    stage_n += __popc(rmask);
                    if (stage_n >= 32) {
                        __syncwarp();
                        const int e = stage_n - 32 + lane;
                        staged_record<S>(rp, tt, acc, st_cell[e], st_row[e], st_x + e * kThreadMaxCells);
                        stage_n -= 32;
                        __syncwarp();
                    }
                }
            }

            // ---- rare: roll back to the first non-plain firing, run ONE exact
            // iteration (the oracle's loop body) and shift the draws ----
#pragma unroll
            for (int i = 0; i < NT; ++i) {
                if (__any_sync(0xffffffffu, bad[i] != 0u)) {
                    bool fill = false;  // stalled here: samples j .. JL filled below, warp-wide
                    double E = Eb[i][0], u2 = Ub[i][0];  // draw of firing n (= batch slot `used`)
                    const int used = (bad[i] == 0u) ? B : __ffs(bad[i]) - 1;
                    if (bad[i] != 0u) {  // roll back to firing `used` (selects, see above)
                        double tt0 = tsnap[i][0];
#pragma unroll
                        for (int k = 1; k < B; ++k) {
                            tt0 = (k == used) ? tsnap[i][k] : tt0;
                            E = (k == used) ? Eb[i][k] : E;
                            u2 = (k == used) ? Ub[i][k] : u2;
                        }
                        t[i] = tt0;
#pragma unroll
                        for (int s = 0; s < S; ++s) {
                            int v = xsnap[i][0][s];
#pragma unroll
                            for (int k = 1; k < B; ++k) v = (k == used) ? xsnap[i][k][s] : v;
                            x[i][s] = v;
                        }
                    }
                    if (live[i] && bad[i] != 0u) {
                        double cum[M];
                        cumulative(tt, gt, x[i], c[i], cum);
                        const double a0 = cum[M - 1];
                        if (a0 == 0.0) {  // stall: no draw is consumed
                            fill = true;
                            status[i] = CWC_TRAJ_STALLED;
                            live[i] = false;
                        } else {
                            const double tau = __ddiv_rn(E, a0);
                            const double tn = __dadd_rn(t[i], tau);
                            while (j[i] <= JL && __dmul_rn(__ll2double_rn(j[i]), rp.dt) <= tn) {
                                record_sample(rp, tt, acc, x[i], cell_base[i], g[i], j[i]);
                                ++j[i];
                            }
                            if (j[i] > JL) {  // horizon (or the launch's last sample) reached: drawn, not applied
                                trace_rec(i, n[i], a0, tau, tn, -1);
                                status[i] = CWC_TRAJ_DONE;
                                live[i] = false;
                            } else {
                                t_next[i] = __dmul_rn(__ll2double_rn(j[i]), rp.dt);
                                t_next2[i] = __dmul_rn(__ll2double_rn(j[i] + 1), rp.dt);
                                int mu;
                                const unsigned long long nu = select_nu<M, TRACE>(tt, cum, __dmul_rn(u2, a0), mu);
                                int xn[S];
                                trace_rec(i, n[i], a0, tau, tn, mu);  // (the oracle records an overflowing firing too)
                                if (apply_nu(x[i], nu, xn)) {  // a count would leave int32: freeze + fill
                                    for (; j[i] <= JL; ++j[i]) record_sample(rp, tt, acc, x[i], cell_base[i], g[i], j[i]);
                                    status[i] = CWC_TRAJ_OVERFLOW;
                                    live[i] = false;
                                } else {
#pragma unroll
                                    for (int s = 0; s < S; ++s) x[i][s] = xn[s];
                                    t[i] = tn;
                                    ++n[i];
                                    ++firings[i];
                                }
                            }
                        }
                        if (live[i]) {
                            // draws of firings n .. n+B-1 are slots [u, u+B) of
                            // (this batch ++ next batch), u = n - n0 in [1, B]
                            const int u = (int)(n[i] - n0[i]);
                            double E2[B], U2[B];
#pragma unroll
                            for (int q = 0; q < B; ++q) {
                                E2[q] = En[i][q];
                                U2[q] = Un[i][q];
#pragma unroll
                                for (int cc = 1; cc < B; ++cc) {
                                    const int src = cc + q;
                                    if (cc == u) {
                                        E2[q] = src < B ? Eb[i][src] : En[i][src - B];
                                        U2[q] = src < B ? Ub[i][src] : Un[i][src - B];
                                    }
                                }
                            }
#pragma unroll
                            for (int q = 0; q < B; ++q) {
                                En[i][q] = E2[q];
                                Un[i][q] = U2[q];
                            }
                        }
                    }
                    if (bad[i] != 0u) fc[i].load(tt, x[i]);  // x was rolled back / changed
                    const unsigned fm = __ballot_sync(0xffffffffu, fill);
                    if (fm) {
                        stall_fill<S>(rp, tt, acc, fm, x[i], cell_base[i], g[i], j[i], JL, lane);
                        if (fill) j[i] = JL + 1;
                    }
                }
            }
#pragma unroll
            for (int i = 0; i < NT; ++i) {
#pragma unroll
                for (int q = 0; q < B; ++q) {
                    Eb[i][q] = En[i][q];
                    Ub[i][q] = Un[i][q];
                }
                // resumable runs: suspend after `quantum` further firings
                if (RES && rp.quantum > 0 && live[i] && n[i] - n_start[i] >= (unsigned long long)rp.quantum) live[i] = false;
            }
            // reconverge the warp explicitly: the vote at the loop head only
            // synchronises it, and a warp left split after the rare path would
            // run every later batch twice with half its lanes (a plain
            // __syncwarp() is elided by the compiler here)
            asm volatile("bar.warp.sync -1;" ::: "memory");
        }
        __syncwarp();
        if (lane < stage_n)  // drain the staged records
            staged_record<S>(rp, tt, acc, st_cell[lane], st_row[lane], st_x + lane * kThreadMaxCells);
#pragma unroll
        for (int i = 0; i < NT; ++i) {
            if (in_range[i]) {
                if (RES && j[i] <= J && status[i] == CWC_TRAJ_DONE) status[i] = CWC_TRAJ_RUNNING;  // suspended
                if (rp.out_firings) rp.out_firings[g[i]] = firings[i];
                if (rp.out_status) rp.out_status[g[i]] = status[i];
                if (TRACE && tslot[i] >= 0) rp.trace_len[tslot[i]] = tn_rec[i];
                if (RES) {
#pragma unroll
                    for (int s = 0; s < S; ++s)
                        if (s < tt.n_cells) rp.rs_x[g[i] * tt.n_cells + s] = x[i][s];
                    rp.rs_t[g[i]] = t[i];
                    rp.rs_n[g[i]] = (int64_t)n[i];
                    rp.rs_j[g[i]] = (int32_t)j[i];
                }
            }
        }
    }

    if (rp.stats_smem) {  // coalesced, vectorised flush of the block's partial moments
        __syncthreads();
        const long long n16 = stat_bytes(rp.st, rp.cells_per_part) / 16;
        uint4 *dst = (uint4 *)((unsigned char *)rp.parts + cta * stat_bytes(rp.st, rp.cells_per_part));
        const uint4 *src = (const uint4 *)smem;
        for (long long i = threadIdx.x; i < n16; i += T) dst[i] = src[i];
    }
}

template <int S, int M, bool TRACE>
__global__ void ssa_thread_ws_kernel(const RunParams rp, const ThreadTables tt);
template <int S, int M, bool TRACE>
__global__ void ssa_thread_ws2_kernel(const RunParams rp, const ThreadTables tt);

template <int S, int M>
cudaError_t launch_sm(const RunParams &rp, const ThreadTables &tt, int threads, size_t smem, cudaStream_t st,
                      bool trace) {
    const long long blocks = (rp.n_launch + threads - 1) / threads;
    if (rp.ws == 2) {  // warp-specialised, 64 trajectories per 2-warp CTA (ssa_thread_ws2.cuh)
        if constexpr (ThreadBatch<M>::B >= 2) {
            auto k = trace ? ssa_thread_ws2_kernel<S, M, true> : ssa_thread_ws2_kernel<S, M, false>;
            cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            if (e != cudaSuccess) return e;
            k<<<(unsigned)((rp.G + 63) / 64), 32 * (1 + kWs2Producers), smem, st>>>(rp, tt);
            return cudaGetLastError();
        }
        return cudaErrorInvalidValue;
    }
    if (rp.ws) {  // warp-specialised: 32 trajectories per 2-warp CTA (ssa_thread_ws.cuh)
        auto k = trace ? ssa_thread_ws_kernel<S, M, true> : ssa_thread_ws_kernel<S, M, false>;
        cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        k<<<(unsigned)((rp.G + 32 * kWsGroups - 1) / (32 * kWsGroups)), 32 * (1 + kWsProducers) * kWsGroups, smem, st>>>(rp, tt);
        return cudaGetLastError();
    }
    // two trajectories per lane (rp.thread_nt == 2) only for one-shot runs of
    // models with 4-firing batches (M <= 8)
    constexpr bool NT2 = ThreadBatch<M>::B >= 2;
    const bool nt2 = NT2 && rp.thread_nt == 2 && !rp.rs_x;
    const long long blocks2 = (rp.n_launch + 2ll * threads - 1) / (2ll * threads);
    auto go = [&](auto k, long long nb) {
        cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        k<<<(unsigned)nb, threads, smem, st>>>(rp, tt);
        return cudaGetLastError();
    };
    if (rp.rs_x) return go(ssa_thread_kernel<S, M, false, true, 1>, blocks);  // resumable runs (never traced)
    if (nt2) return trace ? go(ssa_thread_kernel<S, M, true, false, NT2 ? 2 : 1>, blocks2)
                          : go(ssa_thread_kernel<S, M, false, false, NT2 ? 2 : 1>, blocks2);
    return trace ? go(ssa_thread_kernel<S, M, true, false, 1>, blocks) : go(ssa_thread_kernel<S, M, false, false, 1>, blocks);
}

template <int S>
cudaError_t launch_s(int m_pad, const RunParams &rp, const ThreadTables &tt, int threads, size_t smem,
                     cudaStream_t st, bool trace) {
    switch (m_pad) {
        case 2: return launch_sm<S, 2>(rp, tt, threads, smem, st, trace);
        case 3: return launch_sm<S, 3>(rp, tt, threads, smem, st, trace);
        case 4: return launch_sm<S, 4>(rp, tt, threads, smem, st, trace);
        case 6: return launch_sm<S, 6>(rp, tt, threads, smem, st, trace);
        case 8: return launch_sm<S, 8>(rp, tt, threads, smem, st, trace);
        case 12: return launch_sm<S, 12>(rp, tt, threads, smem, st, trace);
        case 16: return launch_sm<S, 16>(rp, tt, threads, smem, st, trace);
        case 24: return launch_sm<S, 24>(rp, tt, threads, smem, st, trace);
        case 32: return launch_sm<S, 32>(rp, tt, threads, smem, st, trace);
    }
    return cudaErrorInvalidValue;
}

}  // namespace cwc
