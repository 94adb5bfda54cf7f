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

namespace cwc {


// CTA-scope acquire / release on the hand-off counters (lighter than a full
// sequentially-consistent fence: they order only what the protocol needs)
__device__ __forceinline__ unsigned ld_acquire(const unsigned *p) {
    unsigned v;
    asm volatile("ld.acquire.cta.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(unsigned *p, unsigned v) {
    asm volatile("st.release.cta.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

template <int S, int M>
__global__ void __launch_bounds__(64, 1) ssa_thread_ws_kernel(const RunParams rp, const ThreadTables tt) {
    constexpr int B = ThreadBatch<M>::B;
    constexpr int K = kWsRing;
    extern __shared__ __align__(16) unsigned char smem[];
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    // dispatch order: CTA slot blockIdx.x runs trajectory group cta (RunParams.cta_order)
    const long long cta = rp.cta_order ? (long long)__ldg(rp.cta_order + blockIdx.x) : (long long)blockIdx.x;
    const long long g0 = cta * 32;
    const long long g = g0 + lane;
    const int O = tt.O;
    const long long J = rp.J;
    const long long J1 = J + 1;

    const long long stats_bytes = rp.stats_smem ? stat_bytes(rp.st, rp.cells_per_part) : 0;
    double *ringE = (double *)(smem + stats_bytes);    // [K][32]
    double *ringU = ringE + K * 32;                    // [K][32]
    unsigned *prod = (unsigned *)(ringU + K * 32);     // [32] draws published
    unsigned *cons = prod + 32;                        // [32] draws released
    unsigned *done = cons + 32;                        // [32] trajectory finished
    long long *st_cell = (long long *)(done + 32);     // [kWsStage] first cell of a staged record
    long long *st_v = st_cell + kWsStage;              // [kWsStage][kThreadMaxObs] its observables

    StatAcc acc;
    long long p_base = 0;
    if (rp.stats_smem) {
        acc = stat_view(smem, rp.cells_per_part, rp.st);
        uint4 *z = (uint4 *)smem;
        for (long long i = threadIdx.x; i < stats_bytes / 16; i += 64) z[i] = make_uint4(0, 0, 0, 0);
        p_base = g0 / rp.R;
    } else {
        acc = stat_view((unsigned char *)rp.parts + (cta % rp.n_parts) * stat_bytes(rp.st, rp.cells_per_part),
                        rp.cells_per_part, rp.st);
    }
    const bool in_range = g < rp.G;
    const long long gc = in_range ? g : rp.G - 1;
    const uint64_t gk = (uint64_t)global_traj(gc, rp.R, rp.R_total, rp.r_off);  // RNG stream id
    if (warp == 0) {
        prod[lane] = 0;
        cons[lane] = 0;
        done[lane] = in_range ? 0u : 1u;
    }
    __syncthreads();

    if (warp == 1) {
        // ---------------- producer ----------------
        unsigned long long p = 0;  // draws produced (prod/cons hold its low 32 bits; differences wrap)
        for (;;) {
            const bool act = ld_acquire(done + lane) == 0u;
            if (!__any_sync(0xffffffffu, act)) break;
            const unsigned c = ld_acquire(cons + lane);
            const bool room = act && ((unsigned)p + 4u - c <= (unsigned)K);
            if (__any_sync(0xffffffffu, room)) {
                DrawPipe<4> pipe;
                double E4[4], U4[4];
                pipe.start(gk, p);
#pragma unroll
                for (int ph = 0; ph < 4; ++ph) pipe.phase(ph, rp.seed, E4, U4);
                if (room) {
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        const int slot = (int)((p + i) & (K - 1));
                        ringE[slot * 32 + lane] = E4[i];
                        ringU[slot * 32 + lane] = U4[i];
                    }
                    p += 4;
                    st_release(prod + lane, (unsigned)p);
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
        fc.load(tt, x);

        int stage_n = 0;  // staged records (warp-uniform)
        double t = 0.0, t_next = 0.0, t_next2 = rp.dt;  // t_next = j*dt, t_next2 = (j+1)*dt
        long long j = 0, firings = 0;
        unsigned long long n = 0;
        int status = 0;
        bool live = in_range;
        while (__any_sync(0xffffffffu, live)) {
            // draws n .. n+B-1 of every live lane must be published
            for (;;) {
                const bool short_ = live && ((int)(ld_acquire(prod + lane) - (unsigned)(n + B)) < 0);
                if (!__any_sync(0xffffffffu, short_)) break;
                __nanosleep(20);
            }
            double Eb[B], Ub[B];
#pragma unroll
            for (int k = 0; k < B; ++k) {
                const int slot = (int)((n + k) & (K - 1));
                Eb[k] = ringE[slot * 32 + lane];
                Ub[k] = ringU[slot * 32 + lane];
            }

            // ---- fast batch (speculative, as ssa_thread_kernel); one firing
            // per batch may also cross a single sample time that is not the
            // last: it commits, and its record (pre-event state xrec, sample
            // jrec) is written after the batch ----
            int xsnap[B][S];
            double tsnap[B];
            unsigned bad = 0;
            bool rec = false;
            int krec = B;
            long long jrec = 0;
            int xrec[S];
#pragma unroll
            for (int k = 0; k < B; ++k) {
#pragma unroll
                for (int s = 0; s < S; ++s) xsnap[k][s] = x[s];
                tsnap[k] = t;
                bool cross1;
                const bool plain = fc.step2(tt, gt, c, x, t, Eb[k], Ub[k], t_next, t_next2, cross1);
                const bool take = cross1 && !rec && (j < J);
                if (take) {
                    rec = true;
                    krec = k;
                    jrec = j;
#pragma unroll
                    for (int s = 0; s < S; ++s) xrec[s] = xsnap[k][s];
                    j += 1;
                    t_next = t_next2;
                    t_next2 = __dmul_rn(__ll2double_rn(j + 1), rp.dt);
                }
                bad |= (plain || take) ? 0u : (1u << k);
            }
            if (!live) bad = 1u;
            const int used = (bad == 0u) ? B : __ffs(bad) - 1;
            if (rec && krec >= used) {  // the crossing firing was rolled back
                rec = false;
                j = jrec;
                t_next = __dmul_rn(__ll2double_rn(j), rp.dt);
                t_next2 = __dmul_rn(__ll2double_rn(j + 1), rp.dt);
            }
            if (live) {
                n += (unsigned long long)used;
                firings += used;
            }
            // Sample records of the batch are staged in shared memory and
            // written 32 at a time, one per lane: the fire-and-forget limb
            // atomics of a record then run with the whole warp active instead
            // of one lane at a time.
            const unsigned rmask = __ballot_sync(0xffffffffu, rec);
            if (rmask) {
                if (rec) {
                    const int slot = stage_n + __popc(rmask & ((1u << lane) - 1u));
                    st_cell[slot] = cell_base + jrec * O;
                    for (int o = 0; o < O; ++o) {
                        long long v = 0;
#pragma unroll
                        for (int s = 0; s < S; ++s) v += (tt.obs_of[s] == o) ? (long long)xrec[s] : 0ll;
                        st_v[slot * kThreadMaxObs + o] = v;
                        if (rp.out_traj) rp.out_traj[(g * J1 + jrec) * O + o] = v;
                    }
                }
                stage_n += __popc(rmask);
                if (stage_n >= 32) {
                    __syncwarp();
                    const int e = stage_n - 32 + lane;
                    for (int o = 0; o < O; ++o) stat_record(acc, st_cell[e] + o, st_v[e * kThreadMaxObs + o]);
                    stage_n -= 32;
                    __syncwarp();
                }
            }

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
                            status = CWC_TRAJ_DONE;
                            live = false;
                        } else {
                            t_next = __dmul_rn(__ll2double_rn(j), rp.dt);
                            t_next2 = __dmul_rn(__ll2double_rn(j + 1), rp.dt);
                            int mu;
                            const unsigned long long nu = select_nu<M, false>(tt, cum, __dmul_rn(u2, a0), mu);
                            int xn[S];
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
            // release consumed slots (the slot reads above are ordered before it)
            st_release(cons + lane, (unsigned)n);
            if (in_range && !live) st_release(done + lane, 1u);
            asm volatile("bar.warp.sync -1;" ::: "memory");
        }
        __syncwarp();
        if (lane < stage_n)  // drain the staged records
            for (int o = 0; o < O; ++o) stat_record(acc, st_cell[lane] + o, st_v[lane * kThreadMaxObs + o]);
        if (in_range) {
            if (rp.out_firings) rp.out_firings[g] = firings;
            if (rp.out_status) rp.out_status[g] = status;
        }
    }

    if (rp.stats_smem) {
        __syncthreads();
        const long long n16 = stats_bytes / 16;
        uint4 *dst = (uint4 *)((unsigned char *)rp.parts + cta * stats_bytes);
        const uint4 *src = (const uint4 *)smem;
        for (long long i = threadIdx.x; i < n16; i += 64) dst[i] = src[i];
    }
}

}  // namespace cwc
