// ssa_thread_ws2.cuh -- thread path, warp-specialised, TWO trajectories per
// consumer lane (C2: 16384 trajectories = 256 CTAs of 2 warps, so every warp
// can own an SM sub-partition).
//
// The same method and the same committed firings as ssa_thread_ws_kernel
// (ssa_thread_ws.cuh) and ssa_thread_kernel; the consumer lane runs the state
// chains of trajectories 2l and 2l+1 of its group, their speculative batches
// interleaved in one straight-line block (two independent dependency chains
// for the in-order issue: the chain, not the issue slots, bounds C2 -- one
// lone CTA of the single-trajectory kernel spends ~274 cycles per firing at
// an IPC far below one).  The producer lane computes the draws of both
// trajectories, PW per trajectory per round, into a ring of K draws per
// trajectory; hand-off counters per trajectory (prod: release by the
// producer, acquire by the consumer; cons: release by the consumer, acquire
// by the producer; done: relaxed).
#pragma once
#include "ssa_thread_ws.cuh"

namespace cwc {

// NPROD = kWs2Producers (cwc_internal.h) producer warps per CTA.
template <int S, int M, bool TRACE>
__global__ void __launch_bounds__(32 * (1 + kWs2Producers), 1) ssa_thread_ws2_kernel(const RunParams rp, const ThreadTables tt) {
    constexpr int NT = 2;
    constexpr int NPROD = kWs2Producers;
    static_assert(NPROD == 1 || NPROD == NT, "one producer warp, or one per trajectory slot");
    constexpr int B = ThreadBatch<M>::B / 2;  // per trajectory (M <= 8: 2)
    constexpr int PW = 4;
    constexpr int K = kWsRing;
    constexpr int TPC = 32 * NT;  // trajectories per CTA
    static_assert(B >= 1 && K >= B + PW && (K & (K - 1)) == 0, "ring too small");
    extern __shared__ __align__(16) unsigned char smem[];
    const int lane = threadIdx.x & 31;
    const bool consumer = (threadIdx.x >> 5) == 0;

    const long long cta = rp.cta_order ? (long long)__ldg(rp.cta_order + blockIdx.x) : (long long)blockIdx.x;
    const long long g0 = cta * TPC;
    const int O = tt.O;
    const long long J = rp.J;
    const long long J1 = J + 1;

    const long long stats_bytes = rp.stats_smem ? stat_bytes(rp.st, rp.cells_per_part) : 0;
    double *ringE = (double *)(smem + stats_bytes);   // [K][TPC], trajectory q = lane * NT + i
    double *ringU = ringE + K * TPC;                  // [K][TPC]
    unsigned *prod = (unsigned *)(ringU + K * TPC);   // [TPC] rounds published
    unsigned *cons = prod + TPC;                      // [TPC] draws released
    unsigned *done = cons + TPC;                      // [TPC] trajectory finished
    long long *st_cell = (long long *)(done + TPC);   // [kWsStage] staged records
    long long *st_row = st_cell + kWsStage;
    int *st_x = (int *)(st_row + kWsStage);           // [kWsStage][kThreadMaxCells]
    NegLogSmem *ltab = (NegLogSmem *)(smem + stats_bytes + kWs2RingBytes);
    neglog_smem_fill(ltab, threadIdx.x, blockDim.x);
    StatAcc acc;
    long long p_base = 0;
    if (rp.stats_smem) {
        acc = stat_view(smem, rp.cells_per_part, rp.st);
        uint4 *z = (uint4 *)smem;
        for (long long q = threadIdx.x; q < stats_bytes / 16; q += blockDim.x) z[q] = make_uint4(0, 0, 0, 0);
        p_base = g0 / rp.R;
    } else {
        acc = stat_view((unsigned char *)rp.parts + (cta % rp.n_parts) * stat_bytes(rp.st, rp.cells_per_part),
                        rp.cells_per_part, rp.st);
    }
    bool in_range[NT];
    long long g[NT];
    uint64_t gk[NT];
#pragma unroll
    for (int i = 0; i < NT; ++i) {
        const long long gg = g0 + lane * NT + i;
        in_range[i] = gg < rp.G;
        g[i] = in_range[i] ? gg : rp.G - 1;
        gk[i] = (uint64_t)global_traj(g[i], rp.R, rp.R_total, rp.r_off);
    }
    if (consumer) {
#pragma unroll
        for (int i = 0; i < NT; ++i) {
            prod[lane * NT + i] = 0;
            cons[lane * NT + i] = 0;
            done[lane * NT + i] = in_range[i] ? 0u : 1u;
        }
    }
    __syncthreads();

    if (!consumer) {
        // ---------------- producer: PW draws of each of its trajectories per round ----------------
        // NPROD == NT: this warp serves trajectory slot pw of every lane;
        // NPROD == 1: both slots, their rounds interleaved
        constexpr int NS = (NPROD == NT) ? 1 : NT;  // slots served by this warp
        const int pw = (NPROD == NT) ? (threadIdx.x >> 5) - 1 : 0;
        unsigned rounds[NS] = {};
        uint64_t gks[NS];  // RNG streams of the served slots (selects: no dynamic indexing)
#pragma unroll
        for (int q = 0; q < NS; ++q) gks[q] = (pw + q == 0) ? gk[0] : gk[NT - 1];
        for (;;) {
            bool act[NS], room[NS];
            bool any_act = false, any_room = false;
#pragma unroll
            for (int q = 0; q < NS; ++q) {
                const int i = pw + q;
                act[q] = ld_acquire(done + lane * NT + i) == 0u;
                const unsigned c = ld_acquire(cons + lane * NT + i);
                room[q] = act[q] && (rounds[q] * (unsigned)PW + (unsigned)PW - c <= (unsigned)K);
                any_act = any_act || act[q];
                any_room = any_room || room[q];
            }
            if (!__any_sync(0xffffffffu, any_act)) break;
            if (__any_sync(0xffffffffu, any_room)) {
                DrawPipe<PW> pipe[NS];
                double Ew[NS][PW], Uw[NS][PW];
#pragma unroll
                for (int q = 0; q < NS; ++q) pipe[q].start(gks[q], (unsigned long long)rounds[q] * PW);
#pragma unroll
                for (int ph = 0; ph < 4; ++ph) {
#pragma unroll
                    for (int q = 0; q < NS; ++q) pipe[q].phase(ph, rp.rk, ltab, Ew[q], Uw[q]);
                }
#pragma unroll
                for (int q = 0; q < NS; ++q) {
                    const int i = pw + q;
                    if (room[q]) {
#pragma unroll
                        for (int d = 0; d < PW; ++d) {
                            const int slot = (int)((rounds[q] * PW + d) & (K - 1));
                            ringE[slot * TPC + lane * NT + i] = Ew[q][d];
                            ringU[slot * TPC + lane * NT + i] = Uw[q][d];
                        }
                        ws_stress_sleep(gks[q], rounds[q], 1u);
                        ++rounds[q];
                        st_release(prod + lane * NT + i, rounds[q]);
                    }
                }
            } else {
                __nanosleep(100);
            }
            asm volatile("bar.warp.sync -1;" ::: "memory");
        }
    } else {
        // ---------------- consumer: the state chains of trajectories 2l, 2l+1 ----------------
        long long cell_base[NT];
        int x[NT][S];
        FastChain<S, M> fc[NT];
        double t[NT], t_next[NT], t_next2[NT];
        long long j[NT];
        unsigned long long n[NT], avail[NT];
        int status[NT];
        bool live[NT];
        int tslot[NT];
        long long tn_rec[NT];
        const Gather<S, M> gt(tt);
#pragma unroll
        for (int i = 0; i < NT; ++i) {
            const long long p = g[i] / rp.R;
            cell_base[i] = (p - p_base) * J1 * O;
#pragma unroll
            for (int s = 0; s < S; ++s) x[i][s] = (s < tt.n_cells) ? tt.init[s] : 0;
            double c[M];
#pragma unroll
            for (int m = 0; m < M; ++m) c[m] = (m < tt.M) ? __ldg(rp.rates + p * tt.M + m) : 0.0;
            fc[i].rates(tt, c);
            fc[i].load(tt, x[i]);
            t[i] = 0.0;
            t_next[i] = 0.0;
            t_next2[i] = rp.dt;
            j[i] = 0;
            n[i] = 0;
            avail[i] = 0;
            status[i] = CWC_TRAJ_DONE;
            live[i] = in_range[i];
            tslot[i] = -1;
            tn_rec[i] = 0;
            if (TRACE && in_range[i])
                for (int q = 0; q < rp.n_trace; ++q)
                    if (rp.trace_g[q] == g[i]) tslot[i] = q;
        }
        auto trace_rec = [&](int i, unsigned long long n_, double a0_, double tau_, double tn_, int mu_) {
            if (TRACE && tslot[i] >= 0 && tn_rec[i] < rp.trace_cap) {
                double *r = rp.trace_buf + ((long long)tslot[i] * rp.trace_cap + tn_rec[i]++) * 5;
                r[0] = (double)n_; r[1] = a0_; r[2] = tau_; r[3] = tn_; r[4] = (double)mu_;
            }
        };
        auto rates_of = [&](int i, double (&c)[M]) {  // rare path: the trajectory's rate constants
            const long long p = g[i] / rp.R;
#pragma unroll
            for (int m = 0; m < M; ++m) c[m] = (m < tt.M) ? __ldg(rp.rates + p * tt.M + m) : 0.0;
        };
        int stage_n = 0;
        for (;;) {
            bool any_live = false;
#pragma unroll
            for (int i = 0; i < NT; ++i) any_live = any_live || live[i];
            if (!__any_sync(0xffffffffu, any_live)) break;
            // draws n .. n+B-1 of every live trajectory must be published
            bool need = false;
#pragma unroll
            for (int i = 0; i < NT; ++i) need = need || (live[i] && avail[i] < n[i] + B);
            if (__any_sync(0xffffffffu, need)) {
                for (;;) {
                    bool wait = false;
#pragma unroll
                    for (int i = 0; i < NT; ++i) {
                        const unsigned pq = ld_acquire(prod + lane * NT + i);
                        avail[i] = n[i] + (unsigned)(pq * (unsigned)PW - (unsigned)n[i]);
                        wait = wait || (live[i] && avail[i] < n[i] + B);
                    }
                    if (!__any_sync(0xffffffffu, wait)) break;
                    __nanosleep(20);
                }
            }
            double Eb[NT][B], Ub[NT][B];
#pragma unroll
            for (int i = 0; i < NT; ++i)
#pragma unroll
                for (int k = 0; k < B; ++k) {
                    const int slot = (int)((n[i] + k) & (K - 1));
                    Eb[i][k] = ringE[slot * TPC + lane * NT + i];
                    Ub[i][k] = ringU[slot * TPC + lane * NT + i];
                }

            // ---- fast batches of both trajectories, interleaved ----
            int xsnap[NT][B][S];
            double tsnap[NT][B];
            unsigned bad[NT];
            bool rec[NT];
            int krec[NT];
            bool jok[NT];
            double t_next0[NT], t_next20[NT], t_next3[NT];
            FireRec fr[NT][B];
#pragma unroll
            for (int i = 0; i < NT; ++i) {
                bad[i] = 0;
                rec[i] = false;
                krec[i] = B;
                jok[i] = j[i] < J;
                t_next0[i] = t_next[i];
                t_next20[i] = t_next2[i];
                t_next3[i] = __dmul_rn(__ll2double_rn(j[i] + 2), rp.dt);
            }
#pragma unroll
            for (int k = 0; k < B; ++k) {
#pragma unroll
                for (int i = 0; i < NT; ++i) {
#pragma unroll
                    for (int s = 0; s < S; ++s) xsnap[i][k][s] = x[i][s];
                    tsnap[i][k] = t[i];
                    bool cross1;
                    double c_unused[M];  // (the fast chain uses fc.ch)
                    const bool plain = fc[i].template step2<TRACE>(tt, gt, c_unused, x[i], t[i], Eb[i][k], Ub[i][k],
                                                                   t_next[i], t_next2[i], cross1, fr[i][k]);
                    const bool take = cross1 && !rec[i] && jok[i];
                    rec[i] = rec[i] || take;
                    krec[i] = take ? k : krec[i];
                    t_next[i] = take ? t_next2[i] : t_next[i];
                    t_next2[i] = take ? t_next3[i] : t_next2[i];
                    bad[i] |= (plain || take) ? 0u : (1u << k);
                }
            }
            long long jrec[NT];
            int used[NT];
#pragma unroll
            for (int i = 0; i < NT; ++i) {
                if (!live[i]) bad[i] = 1u;
                used[i] = (bad[i] == 0u) ? B : __ffs(bad[i]) - 1;
                if (TRACE && live[i]) {
#pragma unroll
                    for (int k = 0; k < B; ++k)
                        if (k < used[i]) trace_rec(i, n[i] + k, fr[i][k].a0, fr[i][k].tau, fr[i][k].tn, fr[i][k].mu);
                }
                if (rec[i] && krec[i] >= used[i]) {
                    rec[i] = false;
                    t_next[i] = t_next0[i];
                    t_next2[i] = t_next20[i];
                }
                jrec[i] = j[i];
                if (rec[i]) j[i] += 1;
                if (live[i]) n[i] += (unsigned long long)used[i];
            }
            // staged sample records (32 at a time, one per lane)
#pragma unroll
            for (int i = 0; i < NT; ++i) {
                const unsigned rmask = __ballot_sync(0xffffffffu, rec[i]);
                if (rmask) {
                    if (rec[i]) {
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
            // ---- rare: roll back, one exact iteration ----
#pragma unroll
            for (int i = 0; i < NT; ++i) {
                if (__any_sync(0xffffffffu, bad[i] != 0u)) {
                    double E = Eb[i][0], u2 = Ub[i][0];
                    if (bad[i] != 0u) {  // roll back to firing `used` (selects, see above)
                        const int u = used[i];
                        double tt0 = tsnap[i][0];
#pragma unroll
                        for (int k = 1; k < B; ++k) {
                            tt0 = (k == u) ? tsnap[i][k] : tt0;
                            E = (k == u) ? Eb[i][k] : E;
                            u2 = (k == u) ? Ub[i][k] : u2;
                        }
                        t[i] = tt0;
#pragma unroll
                        for (int s = 0; s < S; ++s) {
                            int v = xsnap[i][0][s];
#pragma unroll
                            for (int k = 1; k < B; ++k) v = (k == u) ? xsnap[i][k][s] : v;
                            x[i][s] = v;
                        }
                    }
                    if (live[i] && bad[i] != 0u) {
                        double c[M], cum[M];
                        rates_of(i, c);
                        cumulative(tt, gt, x[i], c, cum);
                        const double a0 = cum[M - 1];
                        if (a0 == 0.0) {  // stall
                            for (; j[i] <= J; ++j[i]) record_sample(rp, tt, acc, x[i], cell_base[i], g[i], j[i]);
                            status[i] = CWC_TRAJ_STALLED;
                            live[i] = false;
                        } else {
                            const double tau = __ddiv_rn(E, a0);
                            const double tn = __dadd_rn(t[i], tau);
                            while (j[i] <= J && __dmul_rn(__ll2double_rn(j[i]), rp.dt) <= tn) {
                                record_sample(rp, tt, acc, x[i], cell_base[i], g[i], j[i]);
                                ++j[i];
                            }
                            if (j[i] > J) {  // horizon reached: drawn, not applied
                                trace_rec(i, n[i], a0, tau, tn, -1);
                                status[i] = CWC_TRAJ_DONE;
                                live[i] = false;
                            } else {
                                t_next[i] = __dmul_rn(__ll2double_rn(j[i]), rp.dt);
                                t_next2[i] = __dmul_rn(__ll2double_rn(j[i] + 1), rp.dt);
                                int mu;
                                const unsigned long long nu = select_nu<M, TRACE>(tt, cum, __dmul_rn(u2, a0), mu);
                                int xn[S];
                                trace_rec(i, n[i], a0, tau, tn, mu);
                                if (apply_nu(x[i], nu, xn)) {
                                    for (; j[i] <= J; ++j[i]) record_sample(rp, tt, acc, x[i], cell_base[i], g[i], j[i]);
                                    status[i] = CWC_TRAJ_OVERFLOW;
                                    live[i] = false;
                                } else {
#pragma unroll
                                    for (int s = 0; s < S; ++s) x[i][s] = xn[s];
                                    t[i] = tn;
                                    ++n[i];
                                }
                            }
                        }
                    }
                    if (bad[i] != 0u) fc[i].load(tt, x[i]);
                }
            }
#pragma unroll
            for (int i = 0; i < NT; ++i) {
                ws_stress_sleep(gk[i], n[i], 2u);
                st_release(cons + lane * NT + i, (unsigned)n[i]);
                if (in_range[i] && !live[i]) st_relaxed(done + lane * NT + i, 1u);
            }
            asm volatile("bar.warp.sync -1;" ::: "memory");
        }
        __syncwarp();
        if (lane < stage_n)
            staged_record<S>(rp, tt, acc, st_cell[lane], st_row[lane], st_x + lane * kThreadMaxCells);
#pragma unroll
        for (int i = 0; i < NT; ++i) {
            if (in_range[i]) {
                if (rp.out_firings) rp.out_firings[g[i]] = (long long)n[i];
                if (rp.out_status) rp.out_status[g[i]] = status[i];
                if (TRACE && tslot[i] >= 0) rp.trace_len[tslot[i]] = tn_rec[i];
            }
        }
    }

    if (rp.stats_smem) {
        __syncthreads();
        const long long n16 = stats_bytes / 16;
        uint4 *dst = (uint4 *)((unsigned char *)rp.parts + cta * stats_bytes);
        const uint4 *src = (const uint4 *)smem;
        for (long long q = threadIdx.x; q < n16; q += blockDim.x) dst[q] = src[q];
    }
}

}  // namespace cwc
