// ssa_thread_impl.cuh -- one trajectory per CUDA thread (small networks).
//
// Hot path of BASELINE north_star (b): "one replica per thread with counts
// and propensities in registers ... for small networks".  Each thread runs
// Gillespie's direct method (loop of Fig. fig:simd P:608-621) for
// trajectory g = blockIdx.x * blockDim.x + threadIdx.x:
//
//   a_m   = k_m * double(h_m(x))                 Match, all M, registers
//   cum_m = cum_{m-1} + a_m, a0 = cum_{M-1}      left-to-right, as the oracle
//   tau   = E_n / a0, E_n = -log u1              P:206-207 (E_{n+1} precomputed:
//                                                counter-based RNG is state-free)
//   samples j with j*dt <= t + tau get x (pre-event), on-line into the
//   block's shared-memory moment accumulators (schema iii)
//   mu    = #{m : cum_m <= u2 a0}                P:208-209 (cum is monotone)
//   x    += nu_mu                                Update
//
// The cells and reactions are compile-time padded (S, M) so that x[] and
// the propensities stay in registers; reaction tables are kernel parameters
// (uniform constant-bank operands).  Net changes are packed int8 per cell
// and selected branch-free while scanning the cumulative sums.
#pragma once
#include <cuda_runtime.h>

#include "cwc_internal.h"
#include "device_common.cuh"

namespace cwc {

template <int S>
__device__ __forceinline__ int pick(const int (&x)[S], int idx) {
    int v = 1;  // idx < 0: the constant 1 of an absent reactant
#pragma unroll
    for (int s = 0; s < S; ++s) v = (idx == s) ? x[s] : v;
    return v;
}

template <int S, int M, bool TRACE>
__global__ void __launch_bounds__(256) ssa_thread_kernel(const RunParams rp, const ThreadTables tt) {
    extern __shared__ __align__(16) unsigned char smem[];
    const long long T = blockDim.x;
    const long long g0 = (long long)blockIdx.x * T;
    const long long g = g0 + threadIdx.x;
    const int O = tt.O;
    const long long J = rp.J;
    const long long J1 = J + 1;

    StatAcc acc;
    long long p_base = 0;
    if (rp.stats_smem) {
        acc = stat_view(smem, rp.cells_per_part);
        uint4 *z = (uint4 *)smem;
        const long long n16 = stat_bytes(rp.cells_per_part) / 16;
        for (long long i = threadIdx.x; i < n16; i += T) z[i] = make_uint4(0, 0, 0, 0);
        p_base = g0 / rp.R;
        __syncthreads();
    } else {
        acc = stat_view((unsigned char *)rp.parts + (long long)(blockIdx.x % rp.n_parts) * stat_bytes(rp.cells_per_part),
                        rp.cells_per_part);
    }

    // Lanes past the last trajectory stay in the warp-uniform loop as idle
    // lanes (their loads use a valid trajectory id; they never record).
    const bool in_range = g < rp.G;
    const long long gc = in_range ? g : rp.G - 1;
    {
        const long long p = gc / rp.R;
        const long long cell_base = (p - p_base) * J1 * O;
        const uint64_t gk = (uint64_t)global_traj(gc, rp.R, rp.R_total, rp.r_off);  // RNG stream id
        int tslot = -1;
        double *trace = nullptr;
        long long tn_rec = 0;
        if (TRACE && in_range) {
            for (int i = 0; i < rp.n_trace; ++i)
                if (rp.trace_g[i] == g) tslot = i;
            if (tslot >= 0) trace = rp.trace_buf + (long long)tslot * rp.trace_cap * 5;
        }

        int x[S];
#pragma unroll
        for (int s = 0; s < S; ++s) x[s] = (s < tt.n_cells) ? tt.init[s] : 0;
        double c[M];
#pragma unroll
        for (int m = 0; m < M; ++m) c[m] = (m < tt.M) ? __ldg(rp.rates + p * tt.M + m) : 0.0;

        auto record = [&](long long j) {
            for (int o = 0; o < O; ++o) {
                long long v = 0;
#pragma unroll
                for (int s = 0; s < S; ++s) v += (tt.obs_of[s] == o) ? (long long)x[s] : 0ll;
                stat_record(acc, cell_base + j * O + o, v);
                if (rp.out_traj) rp.out_traj[(g * J1 + j) * O + o] = v;
            }
        };
        auto trace_rec = [&](unsigned long long n, double a0, double tau, double tn, int mu) {
            if (TRACE && tslot >= 0 && tn_rec < rp.trace_cap) {
                double *r = trace + 5 * tn_rec++;
                r[0] = (double)n; r[1] = a0; r[2] = tau; r[3] = tn; r[4] = (double)mu;
            }
        };

        double t = 0.0, t_next = 0.0;
        long long j = 0, firings = 0;
        unsigned long long n = 0;
        int status = 0;
        double E, u2;
        block_to_draws(philox_block(rp.seed, gk, 0), E, u2);

        // Warp-uniform loop: every iteration reconverges at the vote, so the
        // lanes of a warp advance their trajectories in lock-step and a lane
        // that takes the rare path (crossing / end / stall) costs the others
        // one short wait instead of splitting the warp for good.
        bool live = in_range;
        while (__any_sync(0xffffffffu, live)) {
            if (!live) continue;
            double cum[M];
#pragma unroll
            for (int m = 0; m < M; ++m) {
                const double a = __dmul_rn(c[m], combos(pick(x, tt.ia[m]), pick(x, tt.ib[m]), tt.sub[m], tt.shr[m]));
                cum[m] = (m == 0) ? a : __dadd_rn(cum[m - 1], a);
            }
            const double a0 = cum[M - 1];
            const double tau = __ddiv_rn(E, a0);
            const double tn = __dadd_rn(t, tau);
            const double target = __dmul_rn(u2, a0);
            // next iteration's draw does not depend on the state: overlap it
            double E1, u21;
            block_to_draws(philox_block(rp.seed, gk, n + 1), E1, u21);

            bool apply = true;
            if (!(tn < t_next)) {  // rare: sample crossing, end of horizon, or stall
                if (a0 == 0.0) {
                    for (; j <= J; ++j) record(j);
                    status = CWC_TRAJ_STALLED;
                    live = apply = false;
                } else {
                    while (j <= J && __dmul_rn(__ll2double_rn(j), rp.dt) <= tn) {
                        record(j);
                        ++j;
                    }
                    if (j > J) {
                        trace_rec(n, a0, tau, tn, -1);
                        status = CWC_TRAJ_DONE;
                        live = apply = false;
                    } else {
                        t_next = __dmul_rn(__ll2double_rn(j), rp.dt);
                    }
                }
            }
            if (apply) {
                unsigned long long nu = tt.nu_pack[0];
#pragma unroll
                for (int m = 0; m + 1 < M; ++m) nu = (cum[m] <= target) ? tt.nu_pack[m + 1] : nu;
                if (TRACE && tslot >= 0) {
                    int mu = 0;
#pragma unroll
                    for (int m = 0; m + 1 < M; ++m) mu += (cum[m] <= target) ? 1 : 0;
                    trace_rec(n, a0, tau, tn, mu);
                }
                bool wrapped = false;
#pragma unroll
                for (int s = 0; s < S; ++s) {
                    x[s] += (int)(signed char)(unsigned char)(nu >> (8 * s));
                    wrapped |= (x[s] < 0);
                }
                if (wrapped) {  // a count left int32: undo, freeze, fill
#pragma unroll
                    for (int s = 0; s < S; ++s) x[s] -= (int)(signed char)(unsigned char)(nu >> (8 * s));
                    for (; j <= J; ++j) record(j);
                    status = CWC_TRAJ_OVERFLOW;
                    live = false;
                } else {
                    t = tn;
                    ++firings;
                    ++n;
                    E = E1;
                    u2 = u21;
                }
            }
        }
        if (in_range) {
            if (rp.out_firings) rp.out_firings[g] = firings;
            if (rp.out_status) rp.out_status[g] = status;
            if (TRACE && tslot >= 0) rp.trace_len[tslot] = tn_rec;
        }
    }

    if (rp.stats_smem) {  // coalesced, vectorised flush of the block's partial moments
        __syncthreads();
        const long long n16 = stat_bytes(rp.cells_per_part) / 16;
        uint4 *dst = (uint4 *)((unsigned char *)rp.parts + (long long)blockIdx.x * stat_bytes(rp.cells_per_part));
        const uint4 *src = (const uint4 *)smem;
        for (long long i = threadIdx.x; i < n16; i += T) dst[i] = src[i];
    }
}

template <int S, int M>
cudaError_t launch_sm(const RunParams &rp, const ThreadTables &tt, int threads, size_t smem, cudaStream_t st,
                             bool trace) {
    const long long blocks = (rp.G + threads - 1) / threads;
    if (trace) {
        auto k = ssa_thread_kernel<S, M, true>;
        cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        k<<<(unsigned)blocks, threads, smem, st>>>(rp, tt);
    } else {
        auto k = ssa_thread_kernel<S, M, false>;
        cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        k<<<(unsigned)blocks, threads, smem, st>>>(rp, tt);
    }
    return cudaGetLastError();
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
