// ssa_thread_ws.cuh -- thread path, warp-specialised (producer / consumer).
//
// Same method and same committed sequence of firings as ssa_thread_kernel
// (ssa_thread_impl.cuh: one trajectory per lane, speculative batches of B
// plain firings, one exact oracle-order iteration for the rest), for runs
// with fewer warps than the chip has schedulers (C1, C2: 512 warps for 592
// SMSPs).  There a firing costs the latency of one warp's instruction
// stream, so the stream is split in two:
//
//   warp 1 (producer) computes the Philox4x32-10 blocks and (E = -log u1,
//     u2) of its 32 trajectories -- state-free work (counter-based RNG),
//     four draws per lane per round, fully overlapped -- into a shared-memory
//     ring of K draws per trajectory;
//   warp 0 (consumer) runs the state chain (propensities, a0, tau, crossing,
//     selection, update, on-line statistics) reading its draws from the ring.
//
// The two warps of a CTA sit on different SM sub-partitions, so the chain
// and the RNG issue in parallel.  Hand-off per trajectory: the producer
// writes slots, then publishes prod[lane] with a release store; the consumer
// reads prod[lane] with an acquire load, reads the slots, and publishes
// cons[lane] with a release store (the producer acquires it before refilling
// a slot).  done[lane] ends
// the producer's work for that trajectory.  Both warps belong to one CTA, so
// both are resident and each always makes progress once the other has.
#pragma once
#include "ssa_thread_impl.cuh"

#ifndef CWC_WS_PROF
#define CWC_WS_PROF 0  // consumer cycle accounting (tools/ws_prof.py; debug builds)
#endif

#ifndef CWC_WS_MINB
#define CWC_WS_MINB 6  // CTAs per SM the register budget must allow for small models (S*M <= 12:
                       // <= 170 registers; 1 and 8 measured slower); larger models get the full budget
#endif

namespace cwc {


// Hand-off counters live in shared memory; accesses use the shared state
// space (LDS/STS, not generic loads).  prod: release store by the producer
// (its ring writes are ordered before it), acquire load by the consumer.
// cons: release store by the consumer (its ring loads are ordered before it
// under the PTX memory model, so the producer, which acquires cons, can
// never overwrite a slot the consumer has not read yet), acquire load by
// the producer.  done: relaxed (it orders nothing: the producer only stops).
__device__ __forceinline__ unsigned smem_addr(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }

// Stress builds: a pseudo-random sleep of 0 .. ~4 us on a quarter of the
// calls (hash of the trajectory, the counter and a salt), different per lane.
__device__ __forceinline__ void ws_stress_sleep(unsigned long long g, unsigned long long k, unsigned salt) {
#if CWC_WS_STRESS
    unsigned long long h = (g * 0x9E3779B97F4A7C15ull) ^ (k * 0xC2B2AE3D27D4EB4Full) ^ ((unsigned long long)salt << 17);
    h ^= h >> 29;
    h *= 0xBF58476D1CE4E5B9ull;
    h ^= h >> 32;
    if ((h & 3u) == 0u) __nanosleep((unsigned)(h >> 40) & 4095u);
#else
    (void)g; (void)k; (void)salt;
#endif
}
__device__ __forceinline__ unsigned ld_acquire(const unsigned *p) {
    unsigned v;
    asm volatile("ld.acquire.cta.shared::cta.u32 %0, [%1];" : "=r"(v) : "r"(smem_addr(p)) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(unsigned *p, unsigned v) {
    asm volatile("st.release.cta.shared::cta.u32 [%0], %1;" ::"r"(smem_addr(p)), "r"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed(unsigned *p, unsigned v) {
    asm volatile("st.relaxed.cta.shared::cta.u32 [%0], %1;" ::"r"(smem_addr(p)), "r"(v) : "memory");
}

// TRACE: the same kernel with per-firing trace records (n, a0, tau, t', mu)
// of the trajectories in rp.trace_g written by the consumer (divergence
// tracer: the traced run is the warp-specialised kernel, fast batches
// included).
template <int S, int M, bool TRACE>
__global__ void __launch_bounds__(32 * (1 + kWsProducers) * kWsGroups, (S * M <= 12 && CWC_WS_MINB / kWsGroups / kWsProducers > 1) ? CWC_WS_MINB / kWsGroups / kWsProducers : 1) ssa_thread_ws_kernel(const RunParams rp, const ThreadTables tt) {
    // consumer batch B; one producer warp per group computes rounds of PW
    // draws (round r = draws [r PW, r PW + PW) of each of its trajectories)
    constexpr int B = ThreadBatch<M>::B;
    constexpr int PW = 4;
    constexpr int NP = kWsProducers;
    constexpr int K = kWsRing;
    constexpr int GPC = kWsGroups;  // 32-trajectory groups per CTA
    static_assert(K >= B + NP * PW && (K & (K - 1)) == 0 && B <= PW, "ring too small");
    static_assert(NP == 1 || GPC == 1, "several producers: one group per CTA");
    extern __shared__ __align__(16) unsigned char smem[];
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;

    // Roles.  Warp w serves group w / 2, consumer first ([C0 P0 C1 P1 ..]
    // alternating C/P per pair).  With RunParams.sm_ctr (experiment switch)
    // the order flips by the parity of the CTA's arrival on its SM, putting a
    // consumer and a producer on each sub-partition; measured slower on C2
    // (the producer's fp64 log stream delays the consumer's fp64 chain).
    __shared__ unsigned pattern;
    if (threadIdx.x == 0) {
        unsigned smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        pattern = rp.sm_ctr ? (atomicAdd(rp.sm_ctr + (smid & 1023u), 1u) & 1u) : 0u;
    }
    __syncthreads();
    // GPC == 4: producers first, [P0 P1 P2 P3 C0 C1 C2 C3] -- sub-partition k
    // (warp id mod 4) then holds producer k and consumer k, and the consumer,
    // with the higher warp id, wins the issue arbitration (highest warp id
    // first) whenever both are ready: the producer fills the consumer's gaps
    // NP > 1 (one group per CTA): warp 0 consumes, warps 1 .. NP produce
    const int grp = (NP > 1) ? 0 : (GPC == 4) ? (warp & 3) : (warp >> 1);
    const bool consumer = (NP > 1) ? (warp == 0)
                          : (GPC == 4) ? (warp >= 4)
                                       : ((((unsigned)(warp & 1) ^ (unsigned)grp) & 1u) == pattern);

    // dispatch order: CTA slot blockIdx.x runs trajectory block cta (RunParams.cta_order)
    const long long cta = rp.cta_order ? (long long)__ldg(rp.cta_order + blockIdx.x) : (long long)blockIdx.x;
    const long long g0 = cta * (32 * GPC);
    const long long g = g0 + grp * 32 + lane;
    const int O = tt.O;
    const long long J = rp.J;
    const long long J1 = J + 1;

    const long long stats_bytes = rp.stats_smem ? stat_bytes(rp.st, rp.cells_per_part) : 0;
    unsigned char *gbase = smem + stats_bytes + (long long)grp * (kWsRingBytes / GPC);
    double *ringE = (double *)gbase;                   // [K][32]
    double *ringU = ringE + K * 32;                    // [K][32]
    unsigned *prod = (unsigned *)(ringU + K * 32);     // [NP][32] rounds published per producer
    unsigned *cons = prod + NP * 32;                   // [32] draws released
    unsigned *done = cons + 32;                        // [32] trajectory finished
    long long *st_cell = (long long *)(done + 32);     // [kWsStage] first cell of a staged record
    long long *st_row = st_cell + kWsStage;            // [kWsStage] its trajectory sample row (out_traj)
    int *st_x = (int *)(st_row + kWsStage);            // [kWsStage][kThreadMaxCells] its pre-event counts

    NegLogSmem *ltab = (NegLogSmem *)(smem + stats_bytes + kWsRingBytes);  // the CTA's -log table
    neglog_smem_fill(ltab, threadIdx.x, blockDim.x);
    StatAcc acc;
    long long p_base = 0;
    if (rp.stats_smem) {
        acc = stat_view(smem, rp.cells_per_part, rp.st);
        uint4 *z = (uint4 *)smem;
        for (long long i = threadIdx.x; i < stats_bytes / 16; i += blockDim.x) z[i] = make_uint4(0, 0, 0, 0);
        p_base = g0 / rp.R;
    } else {
        acc = stat_view((unsigned char *)rp.parts + (cta % rp.n_parts) * stat_bytes(rp.st, rp.cells_per_part),
                        rp.cells_per_part, rp.st);
    }
    const bool in_range = g < rp.G;
    const long long gc = in_range ? g : rp.G - 1;
    const uint64_t gk = (uint64_t)global_traj(gc, rp.R, rp.R_total, rp.r_off);  // RNG stream id
    if (consumer) {
#pragma unroll
        for (int q = 0; q < NP; ++q) prod[q * 32 + lane] = 0;
        cons[lane] = 0;
        done[lane] = in_range ? 0u : 1u;
    }
    __syncthreads();

    if (!consumer) {
        // ---------------- producer ----------------
        const int q = (NP > 1) ? warp - 1 : 0;  // this producer's rounds: q, q + NP, q + 2 NP, ...
        unsigned rounds = 0;  // rounds done by this producer (its counter; differences wrap)
        for (;;) {
            const bool act = ld_acquire(done + lane) == 0u;
            if (!__any_sync(0xffffffffu, act)) break;
            const unsigned long long p = ((unsigned long long)rounds * NP + q) * PW;  // first draw of the round
            const unsigned c = ld_acquire(cons + lane);
            const bool room = act && ((unsigned)p + (unsigned)PW - c <= (unsigned)K);
            if (__any_sync(0xffffffffu, room)) {
                DrawPipe<PW> pipe;
                double Ew[PW], Uw[PW];
                pipe.start(gk, p);
#pragma unroll
                for (int ph = 0; ph < 4; ++ph) pipe.phase(ph, rp.rk, ltab, Ew, Uw);
                if (room) {
#pragma unroll
                    for (int i = 0; i < PW; ++i) {
                        const int slot = (int)((p + i) & (K - 1));
                        ringE[slot * 32 + lane] = Ew[i];
                        ringU[slot * 32 + lane] = Uw[i];
                    }
                    ws_stress_sleep(gk, rounds, 1u);  // (stress builds: between the slot writes and the release)
                    ++rounds;
                    st_release(prod + q * 32 + lane, rounds);
                }
            } else {
                __nanosleep(100);
            }
            asm volatile("bar.warp.sync -1;" ::: "memory");
        }
    } else {
        // ---------------- consumer ----------------
        const long long p = gc / rp.R;
        const long long cell_base = (p - p_base) * J1 * O;
        int x[S];
#pragma unroll
        for (int s = 0; s < S; ++s) x[s] = (s < tt.n_cells) ? tt.init[s] : 0;
        double c[M];
#pragma unroll
        for (int m = 0; m < M; ++m) c[m] = (m < tt.M) ? __ldg(rp.rates + p * tt.M + m) : 0.0;
        const Gather<S, M> gt(tt);
        FastChain<S, M> fc;
        fc.rates(tt, c);
        fc.load(tt, x);

        int tslot = -1;
        long long tn_rec = 0;
        if (TRACE && in_range)
            for (int i = 0; i < rp.n_trace; ++i)
                if (rp.trace_g[i] == g) tslot = i;
        auto trace_rec = [&](unsigned long long n_, double a0_, double tau_, double tn_, int mu_) {
            if (TRACE && tslot >= 0 && tn_rec < rp.trace_cap) {
                double *r = rp.trace_buf + ((long long)tslot * rp.trace_cap + tn_rec++) * 5;
                r[0] = (double)n_; r[1] = a0_; r[2] = tau_; r[3] = tn_; r[4] = (double)mu_;
            }
        };

        int stage_n = 0;  // staged records (warp-uniform)
        unsigned long long avail = 0;  // draws of this trajectory known to be published
        double t = 0.0, t_next = 0.0, t_next2 = rp.dt;  // t_next = j*dt, t_next2 = (j+1)*dt
        long long j = 0, firings = 0;
        unsigned long long n = 0;
        int status = 0;
        bool live = in_range;
        // optional cycle accounting of the consumer (RunParams.prof, debug):
        // [0] waiting for draws, [1] fast batch, [2] records, [3] exact path,
        // [4] batches, [5] total
        unsigned long long pc[6] = {0, 0, 0, 0, 0, 0};
        // (compiled in only with -DCWC_WS_PROF=1: the checks cost ~2 % of the
        // consumer's instructions)
        const bool prof = CWC_WS_PROF && rp.prof != nullptr;
        long long c0 = prof ? clock64() : 0, c1 = 0;
        const long long c_start = c0;
        while (__any_sync(0xffffffffu, live)) {
            // draws n .. n+B-1 of every live lane must be published; `avail`
            // caches the last acquired bound, so the counters are re-read
            // only when a lane runs past it
            if (__any_sync(0xffffffffu, live && avail < n + B)) {
                for (;;) {
                    // producer q's first missing round is q + NP * prod_q; all
                    // draws below (q + NP prod_q) PW of every producer are in.
                    // Counters are 32-bit: distances to n are taken mod 2^32
                    // (a producer is never more than K draws ahead of n)
                    unsigned gap = 0xffffffffu;
#pragma unroll
                    for (int q = 0; q < NP; ++q) {
                        const unsigned pq = ld_acquire(prod + q * 32 + lane);
                        const unsigned gq = (pq * (unsigned)NP + (unsigned)q) * (unsigned)PW - (unsigned)n;
                        gap = gq < gap ? gq : gap;
                    }
                    avail = n + gap;
                    if (!__any_sync(0xffffffffu, live && avail < n + B)) break;
                    __nanosleep(20);
                }
            }
            double Eb[B], Ub[B];
#pragma unroll
            for (int k = 0; k < B; ++k) {
                const int slot = (int)((n + k) & (K - 1));
                Eb[k] = ringE[slot * 32 + lane];
                Ub[k] = ringU[slot * 32 + lane];
            }

            if (prof) { c1 = clock64(); pc[0] += c1 - c0; c0 = c1; pc[4] += 1; }
            // ---- fast batch (speculative, as ssa_thread_kernel); one firing
            // per batch may also cross a single sample time that is not the
            // last: it commits, and its record (pre-event state xrec, sample
            // jrec) is written after the batch ----
            int xsnap[B][S];
            double tsnap[B];
            unsigned bad = 0;
            // (at most one: it is the batch's only change of j, so the
            // per-firing bookkeeping is a few selects; the batch-start sample
            // times are kept for a rollback, and t_next3 = (j + 2) dt becomes
            // the next-but-one sample time after the crossing)
            bool rec = false;
            int krec = B;
            const bool jok = j < J;
            const double t_next0 = t_next, t_next20 = t_next2;
            const double t_next3 = __dmul_rn(__ll2double_rn(j + 2), rp.dt);
            FireRec fr[B];
#pragma unroll
            for (int k = 0; k < B; ++k) {
#pragma unroll
                for (int s = 0; s < S; ++s) xsnap[k][s] = x[s];
                tsnap[k] = t;
                bool cross1;
                const bool plain = fc.template step2<TRACE>(tt, gt, c, x, t, Eb[k], Ub[k], t_next, t_next2, cross1, fr[k]);
                const bool take = cross1 && !rec && jok;
                rec = rec || take;
                krec = take ? k : krec;
                t_next = take ? t_next2 : t_next;
                t_next2 = take ? t_next3 : t_next2;
                bad |= (plain || take) ? 0u : (1u << k);
            }
            if (!live) bad = 1u;
            const int used = (bad == 0u) ? B : __ffs(bad) - 1;
            if (TRACE && live) {  // trace records of the committed speculative firings
#pragma unroll
                for (int k = 0; k < B; ++k)
                    if (k < used) trace_rec(n + k, fr[k].a0, fr[k].tau, fr[k].tn, fr[k].mu);
            }
            if (rec && krec >= used) {  // the crossing firing was rolled back
                rec = false;
                t_next = t_next0;
                t_next2 = t_next20;
            }
            const long long jrec = j;  // the sample a committed crossing recorded
            if (rec) j += 1;
            if (live) {
                n += (unsigned long long)used;
                firings += used;
            }
            // Sample records of the batch are staged in shared memory and
            // written 32 at a time, one per lane: the fire-and-forget limb
            // atomics of a record then run with the whole warp active instead
            // of one lane at a time.
            if (prof) { c1 = clock64(); pc[1] += c1 - c0; c0 = c1; }
            const unsigned rmask = __ballot_sync(0xffffffffu, rec);
            if (rmask) {
                if (rec) {  // few lanes: stage the counts only, observables are formed at the flush
                    const int slot = stage_n + __popc(rmask & ((1u << lane) - 1u));
                    st_cell[slot] = cell_base + jrec * O;
                    st_row[slot] = g * J1 + jrec;
#pragma unroll
                    for (int k = 0; k < B; ++k)  // pre-event counts of firing krec
                        if (k == krec) {
#pragma unroll
                            for (int s = 0; s < S; ++s) st_x[slot * kThreadMaxCells + s] = xsnap[k][s];
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

            if (prof) { c1 = clock64(); pc[2] += c1 - c0; c0 = c1; }
            // ---- rare: roll back, one exact iteration ----
            if (__any_sync(0xffffffffu, bad != 0u)) {
                double E = Eb[0], u2 = Ub[0];
                if (bad != 0u) {
#pragma unroll
                    for (int k = 0; k < B; ++k) {
                        if (k == used) {
#pragma unroll
                            for (int s = 0; s < S; ++s) x[s] = xsnap[k][s];
                            t = tsnap[k];
                            E = Eb[k];
                            u2 = Ub[k];
                        }
                    }
                }
                if (live && bad != 0u) {
                    double cum[M];
                    cumulative(tt, gt, x, c, cum);
                    const double a0 = cum[M - 1];
                    if (a0 == 0.0) {  // stall
                        for (; j <= J; ++j) record_sample(rp, tt, acc, x, cell_base, g, j);
                        status = CWC_TRAJ_STALLED;
                        live = false;
                    } else {
                        const double tau = __ddiv_rn(E, a0);
                        const double tn = __dadd_rn(t, tau);
                        while (j <= J && __dmul_rn(__ll2double_rn(j), rp.dt) <= tn) {
                            record_sample(rp, tt, acc, x, cell_base, g, j);
                            ++j;
                        }
                        if (j > J) {  // horizon reached: drawn, not applied
                            trace_rec(n, a0, tau, tn, -1);
                            status = CWC_TRAJ_DONE;
                            live = false;
                        } else {
                            t_next = __dmul_rn(__ll2double_rn(j), rp.dt);
                            t_next2 = __dmul_rn(__ll2double_rn(j + 1), rp.dt);
                            int mu;
                            const unsigned long long nu = select_nu<M, TRACE>(tt, cum, __dmul_rn(u2, a0), mu);
                            int xn[S];
                            trace_rec(n, a0, tau, tn, mu);
                            if (apply_nu(x, nu, xn)) {  // a count would leave int32: freeze + fill
                                for (; j <= J; ++j) record_sample(rp, tt, acc, x, cell_base, g, j);
                                status = CWC_TRAJ_OVERFLOW;
                                live = false;
                            } else {
#pragma unroll
                                for (int s = 0; s < S; ++s) x[s] = xn[s];
                                t = tn;
                                ++n;
                                ++firings;
                            }
                        }
                    }
                }
                if (bad != 0u) fc.load(tt, x);  // x was rolled back / changed
            }
            if (prof) { c1 = clock64(); pc[3] += c1 - c0; c0 = c1; }
            ws_stress_sleep(gk, n, 2u);  // (stress builds: between the slot reads and the release)
            // release consumed slots (the slot reads above are ordered before it)
            st_release(cons + lane, (unsigned)n);
            if (in_range && !live) st_relaxed(done + lane, 1u);
            asm volatile("bar.warp.sync -1;" ::: "memory");
        }
        if (prof && lane == 0) {
            pc[5] = clock64() - c_start;
            for (int i = 0; i < 6; ++i) atomicAdd(rp.prof + i, pc[i]);
        }
        __syncwarp();
        if (lane < stage_n)  // drain the staged records
            staged_record<S>(rp, tt, acc, st_cell[lane], st_row[lane], st_x + lane * kThreadMaxCells);
        if (in_range) {
            if (rp.out_firings) rp.out_firings[g] = firings;
            if (rp.out_status) rp.out_status[g] = status;
            if (TRACE && tslot >= 0) rp.trace_len[tslot] = tn_rec;
        }
    }

    if (rp.stats_smem) {
        __syncthreads();
        const long long n16 = stats_bytes / 16;
        uint4 *dst = (uint4 *)((unsigned char *)rp.parts + cta * stats_bytes);
        const uint4 *src = (const uint4 *)smem;
        for (long long i = threadIdx.x; i < n16; i += blockDim.x) dst[i] = src[i];
    }
}

}  // namespace cwc
