// ssa_warp.cu -- one trajectory per warp (large networks).
//
// Hot path of BASELINE north_star (b): "warp-per-replica for large networks,
// with a shuffle-scan propensity sum, ballot/ffs reaction selection and
// dependency-graph propensity updates".  The 32 lanes of a warp share one
// trajectory -- the GPU form of the intra-step data parallelism the paper
// applies to Match_Populations with SSE -- and the warps of the
// grid are a persistent farm that pulls trajectory ids on demand from an
// atomic counter (schema i, on-demand dispatch).
//
// Per warp, in shared memory: counts x[cell] (int32, plus a constant 1 at
// index n_cells for absent reactants) and propensities a[m].  Lane l owns the
// chunk of reactions m in [l*B, (l+1)*B), stored contiguously at slots
// l*Bp .. l*Bp+B-1 (Bp = B | 1, odd: the lane-strided re-sum and the
// chunk-contiguous selection read are both bank-conflict free).  Lane l keeps
// its chunk sum (left to right) in a register; a Kogge-Stone shuffle scan of
// the 32 chunk sums gives the inclusive prefixes, a0 = prefix of lane 31
// (P:201-203).
//
// One firing (Fig. fig:simd P:608-621):
//   tau = E_n / a0 (E_n = -log u1 of Philox block n, drawn 32 at a time: lane
//   i computes block n - kd + i, then broadcast by shuffle), sample crossing
//   into the moment accumulators, target = u2 a0,
//   L = ffs(ballot(prefix_l > target)) picks the chunk; the lanes then read
//   chunk L (lane k <- a[L*Bp + k]), shuffle-scan it from L's exclusive
//   prefix and ffs(ballot(prefix > target)) picks mu inside it; x += nu_mu
//   (one lane per changed cell); only the reactions in D(mu) are recomputed
//   (precomputed slots) and only their owner lanes re-sum their chunks.
#include <cuda_runtime.h>

#include <type_traits>

#include "cwc_internal.h"
#include "device_common.cuh"

namespace cwc {

constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ double shfl_d(double v, int src) { return __shfl_sync(kFull, v, src); }

__device__ __forceinline__ double propensity(const WarpTables &wt, const int *xs, const double *rates, int m) {
    const int4 d = __ldg(reinterpret_cast<const int4 *>(wt.rx) + m);
    return __dmul_rn(__ldg(rates + m), combos(xs[d.x], xs[d.y], d.z & 1, d.z >> 1));
}

// Inclusive Kogge-Stone scan over the 32 lanes.
__device__ __forceinline__ double warp_incl_scan(double v, int lane) {
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const double y = __shfl_up_sync(kFull, v, d);
        if (lane >= d) v = __dadd_rn(y, v);
    }
    return v;
}

// Inclusive scan of lanes [0, w) (w a power of two <= 32, warp-uniform);
// lanes >= w get garbage that callers mask out.  Unrolled; the steps at or
// beyond w are skipped by a warp-uniform test.
__device__ __forceinline__ double warp_incl_scan_w(double v, int lane, int w) {
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        if (d < w) {
            const double y = __shfl_up_sync(kFull, v, d);
            if (lane >= d) v = __dadd_rn(y, v);
        }
    }
    return v;
}

// Left-to-right sum of a chunk of B entries; BMAX > 0: compile-time bound
// (B <= BMAX), fully unrolled.
template <int BMAX>
__device__ __forceinline__ double chunk_sum(const double *ch, int B) {
    double s = ch[0];
    if constexpr (BMAX > 0) {
        if (B > BMAX - 4) {  // nearly full chunk: no per-entry bounds tests below BMAX - 4 (warp-uniform)
#pragma unroll
            for (int k = 1; k < BMAX - 4; ++k) s = __dadd_rn(s, ch[k]);
#pragma unroll
            for (int k = BMAX - 4; k < BMAX; ++k)
                if (k < B) s = __dadd_rn(s, ch[k]);
        } else {
#pragma unroll
            for (int k = 1; k < BMAX; ++k)
                if (k < B) s = __dadd_rn(s, ch[k]);
        }
    } else {
#pragma unroll 4
        for (int k = 1; k < B; ++k) s = __dadd_rn(s, ch[k]);
    }
    return s;
}

// Chunk sum for long chunks (B > 16: C5) as four interleaved partial sums
// (entries k = 4i + r into partial r, each left to right), then
// (s0 + s1) + (s2 + s3): the same additions as a serial sum but a dependent
// chain of ~B/4 instead of B fp64 additions on the firing's critical path.
template <int BMAX>
__device__ __forceinline__ double chunk_sum4(const double *ch, int B) {
    double s[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) s[r] = (r < B) ? ch[r] : 0.0;
    if constexpr (BMAX > 0) {
        if (B > BMAX - 4) {  // nearly full chunk (C5: 37 of 40): bounds tests on the last four entries only
#pragma unroll
            for (int k = 4; k < BMAX - 4; ++k) s[k & 3] = __dadd_rn(s[k & 3], ch[k]);
#pragma unroll
            for (int k = BMAX - 4; k < BMAX; ++k)
                if (k < B) s[k & 3] = __dadd_rn(s[k & 3], ch[k]);
        } else {
#pragma unroll
            for (int k = 4; k < BMAX; ++k)
                if (k < B) s[k & 3] = __dadd_rn(s[k & 3], ch[k]);
        }
    } else {
        int k = 4;
        for (; k + 3 < B; k += 4) {
#pragma unroll
            for (int r = 0; r < 4; ++r) s[r] = __dadd_rn(s[r], ch[k + r]);
        }
        for (; k < B; ++k) s[k & 3] = __dadd_rn(s[k & 3], ch[k]);
    }
    return __dadd_rn(__dadd_rn(s[0], s[1]), __dadd_rn(s[2], s[3]));
}

// MINB: CTAs per SM the register allocation must allow (8 -> 64 registers,
// for models whose per-warp shared memory lets 8 CTAs reside; 6 -> 80).
// RES: resumable runs (cwc_run_*: state load/save, launch bounds); the
// one-shot instantiation carries none of it (measured: C5 -8 % otherwise)
template <bool TRACE, int MINB, int BMAX, bool RES>
__global__ void __launch_bounds__(128, MINB) ssa_warp_kernel(const RunParams rp, const WarpTables wt, long long stats_smem_bytes,
                                                       int per_warp_bytes, int x_bytes) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    const int B = wt.B, Bp = wt.Bp;
    int scan_w = 1;  // in-chunk scan width: next power of two >= min(B, 32)
    while (scan_w < B && scan_w < 32) scan_w <<= 1;
    const int O = wt.O;
    const int M = wt.M;
    const long long J = rp.J, J1 = J + 1;

    StatAcc acc;
    if (rp.stats_smem) {
        acc = stat_view(smem, rp.cells_per_part, rp.st);
        uint4 *z = (uint4 *)smem;
        for (long long i = threadIdx.x; i < stats_smem_bytes / 16; i += blockDim.x) z[i] = make_uint4(0, 0, 0, 0);
    } else {
        acc = stat_view((unsigned char *)rp.parts + (long long)(blockIdx.x % rp.n_parts) * stat_bytes(rp.st, rp.cells_per_part),
                        rp.cells_per_part, rp.st);
    }
    int *xs = (int *)(smem + stats_smem_bytes + (long long)wib * per_warp_bytes);
    double *as = (double *)((unsigned char *)xs + x_bytes);
    __shared__ unsigned int cta_traj;  // trajectories taken by this CTA (shared-memory part capacity)
    __shared__ unsigned long long q_stop[RES ? 32 : 1];  // per warp: resumable runs' firing bound
    if (threadIdx.x == 0) cta_traj = 0;
    __syncthreads();

    for (;;) {
        unsigned long long gg = ~0ull;
        if (lane == 0) {
            // a shared-memory part holds <= kSmemPartMaxTraj trajectories (16-bit
            // limbs); the host sizes the grid so that the capped CTAs cover G
            if (!rp.stats_smem || atomicAdd(&cta_traj, 1u) < (unsigned)kSmemPartMaxTraj) gg = atomicAdd(rp.next_traj, 1ull);
        }
        gg = __shfl_sync(kFull, gg, 0);
        if (gg >= (unsigned long long)(RES ? rp.n_launch : rp.G)) break;
        const long long g = RES ? launch_traj(rp, (long long)gg) : (long long)gg;
        const long long p = g / rp.R;
        const double *rates = rp.rates + p * M;
        const double *rates_h = rp.rates_h + p * M;
        const uint64_t gk = (uint64_t)global_traj(g, rp.R, rp.R_total, rp.r_off);  // RNG stream id

        int tslot = -1;
        double *trace = nullptr;
        long long tn_rec = 0;
        if (TRACE) {
            for (int i = 0; i < rp.n_trace; ++i)
                if (rp.trace_g[i] == g) tslot = i;
            if (tslot >= 0) trace = rp.trace_buf + (long long)tslot * rp.trace_cap * 5;
        }
        auto trace_rec = [&](unsigned long long n_, double a0_, double tau, double tn, int mu) {
            if (TRACE && tslot >= 0 && tn_rec < rp.trace_cap) {
                if (lane == 0) {
                    double *r = trace + 5 * tn_rec;
                    r[0] = (double)n_; r[1] = a0_; r[2] = tau; r[3] = tn; r[4] = (double)mu;
                }
                ++tn_rec;
            }
        };

        // state: fresh (x0, t = 0, n = 0, j = 0) or resumed (cwc_run_advance)
        for (int c = lane; c < wt.n_cells; c += 32)
            xs[c] = RES ? rp.rs_x[g * wt.n_cells + c] : __ldg(wt.init + c);
        if (lane == 0) xs[wt.n_cells] = 1;
        // (lean state -- see ssa_warp2.cu: n = applied firings = next draw
        // counter, kd = draws used from the 32-draw window, 32-bit j)
        double t = 0.0;
        int j = 0;
        unsigned long long n = 0;
        if (RES) {
            t = rp.rs_t[g];
            j = rp.rs_j[g];
            n = (unsigned long long)rp.rs_n[g];
        }
        // resumable bounds: samples j < jend in this launch (J+1 in one-shot
        // runs); the quantum's firing bound sits in shared memory
        const int jend = RES ? (int)rp.j_stop : (int)J1;
        if (RES && lane == 0) q_stop[wib] = rp.quantum > 0 ? n + (unsigned long long)rp.quantum : ~0ull;
        __syncwarp();

        double part = 0.0;
        constexpr bool AHEAD = MINB <= 6;  // register budget for values loaded or computed ahead of their use (below)
        constexpr bool SUM4 = (BMAX == 0 || BMAX > 16);  // long chunks: chunk_sum4, also here
        for (int k = 0; k < B; ++k) {
            const int m = lane * B + k;
            const double a = (m < M) ? propensity(wt, xs, rates, m) : 0.0;
            as[lane * Bp + k] = a;
            if (!SUM4) part = (k == 0) ? a : __dadd_rn(part, a);
        }
        if (SUM4) part = chunk_sum4<BMAX>(as + lane * Bp, B);
        double incl = warp_incl_scan(part, lane);
        double a0 = shfl_d(incl, 31);
        double excl = __shfl_up_sync(kFull, incl, 1);
        if (lane == 0) excl = 0.0;
        __syncwarp();

        auto record = [&](int jj) {  // rare: the statistics cell is recomputed from g
            const long long cb = (g / rp.R) * J1 * O + (long long)jj * O;
            for (int o = lane; o < O; o += 32) {
                long long v = 0;
                for (int q = __ldg(wt.obs_ptr + o); q < __ldg(wt.obs_ptr + o + 1); ++q) v += xs[__ldg(wt.obs_cells + q)];
                stat_record(acc, cb + o, v);
                if (rp.out_traj) rp.out_traj[(g * J1 + jj) * O + o] = v;
            }
        };

        double t_next = RES ? __dmul_rn(__int2double_rn(j), rp.dt) : 0.0;
        int kd = 0;
        int status = CWC_TRAJ_DONE;
        double El, u2l;
        block_to_draws(philox_block(rp.seed, gk, n + lane), El, u2l);

        // (a trajectory resumed at its launch's sample bound -- j_stop
        // windows -- has nothing to do)
        if (!RES || j < jend) for (;;) {
            if (kd == 32) {
                // resumable runs: suspend after `quantum` further firings (at a
                // 32-draw window boundary)
                if (RES && n >= q_stop[wib]) break;
                kd = 0;
                block_to_draws(philox_block(rp.seed, gk, n + lane), El, u2l);
            }
            const int i = kd;
            const double E = shfl_d(El, i);
            const double u2 = shfl_d(u2l, i);
            // warp-uniform operands: the fast/IEEE choice never diverges.
            // AHEAD (the 80-register instantiations): the fast quotient is
            // formed unconditionally, ahead of the test that says whether it
            // is the IEEE one, together with the first stage of the selection
            // (which needs a0 and u2 only): the division's dependent fp64
            // chain then overlaps the ballot and shuffle latencies instead of
            // standing alone on the firing's critical path (C5 +5 % with the
            // dependency prefetch below; the 64-register instantiations lose
            // 5 % to the extra live values and keep the plain order)
            double qf = 0.0, target = 0.0, carry = 0.0;
            int L = 0;
            if constexpr (AHEAD) {
                qf = div_fast(E, a0);
                target = __dmul_rn(u2, a0);
                const unsigned hitsL = __ballot_sync(kFull, incl > target);
                L = hitsL ? __ffs(hitsL) - 1 : 0;  // lane 31's prefix is a0 > target (a0 == 0: stall below)
                carry = shfl_d(excl, L);
            }
            const double tau = div_fast_ok(E, a0) ? (AHEAD ? qf : div_fast(E, a0)) : __ddiv_rn(E, a0);
            const double tn = __dadd_rn(t, tau);
            if (!(tn < t_next)) {
                if (a0 == 0.0) {
                    for (; j < jend; ++j) record(j);
                    status = CWC_TRAJ_STALLED;
                    break;
                }
                while (j < jend && __dmul_rn(__int2double_rn(j), rp.dt) <= tn) {
                    record(j);
                    ++j;
                }
                if (j >= jend) {  // horizon (or the launch's last sample): drawn, not applied
                    trace_rec(n, a0, tau, tn, -1);
                    status = CWC_TRAJ_DONE;
                    break;
                }
                t_next = __dmul_rn(__int2double_rn(j), rp.dt);
            }
            if constexpr (!AHEAD) {
                target = __dmul_rn(u2, a0);
                L = __ffs(__ballot_sync(kFull, incl > target)) - 1;  // lane 31's prefix is a0 > target
                carry = shfl_d(excl, L);
            }
            // inside chunk L: shuffle-scan its entries from L's exclusive prefix
            int mu = -1;
            unsigned pos_any = 0;
            int pos_base = 0;
            if (B > 32 && B <= 64) {
                // one pass for chunks of 33..64 entries: lane l takes entries
                // 2l and 2l+1 (left to right), then the pair sums are scanned
                const int k = 2 * lane;
                const double a1 = (k < B) ? as[L * Bp + k] : 0.0;
                const double a2 = (k + 1 < B) ? as[L * Bp + k + 1] : 0.0;
                const double incl2 = __dadd_rn(carry, warp_incl_scan(__dadd_rn(a1, a2), lane));
                double ex2 = __shfl_up_sync(kFull, incl2, 1);
                if (lane == 0) ex2 = carry;
                const double c1 = __dadd_rn(ex2, a1);
                const unsigned h1 = __ballot_sync(kFull, k < B && target < c1);
                const unsigned h2 = __ballot_sync(kFull, k + 1 < B && target < incl2);
                const unsigned p1 = __ballot_sync(kFull, a1 > 0.0), p2 = __ballot_sync(kFull, a2 > 0.0);
                if (h1 | h2) {
                    const int l1 = h1 ? __ffs(h1) - 1 : 64, l2 = h2 ? __ffs(h2) - 1 : 64;
                    mu = L * B + ((l1 <= l2) ? 2 * l1 : 2 * l2 + 1);
                } else {  // rounding: the last positive entry of the chunk
                    const int q1 = p1 ? 2 * (31 - __clz(p1)) : -1, q2 = p2 ? 2 * (31 - __clz(p2)) + 1 : -1;
                    mu = L * B + (q1 > q2 ? q1 : q2);
                }
            }
            for (int k0 = 0; mu < 0 && k0 < B; k0 += 32) {
                const int k = k0 + lane;
                const double a = (k < B) ? as[L * Bp + k] : 0.0;
                const double c = __dadd_rn(carry, warp_incl_scan_w(a, lane, scan_w));
                const unsigned hit = __ballot_sync(kFull, k < B && target < c);
                const unsigned pos = __ballot_sync(kFull, a > 0.0);
                if (hit) {
                    mu = L * B + k0 + __ffs(hit) - 1;
                    break;
                }
                if (pos) {
                    pos_any = pos;
                    pos_base = k0;
                }
                carry = shfl_d(c, 31);
            }
            // the chunk's scanned sums may round below the lane prefix: take
            // its last positive entry
            if (mu < 0) mu = L * B + pos_base + 31 - __clz(pos_any);  // (B <= 32 or B > 64)
            trace_rec(n, a0, tau, tn, mu);

            // Update: one lane per changed cell; distinct cells.
            // The per-mu header (nu offset, nu count, dependency offset,
            // dependency count) is one load.
            const int4 h = __ldg(wt.hdr + mu);
            // the first round of dependency entries is requested now: the L2
            // round trip of the D(mu) list (the longest load on the firing's
            // chain) overlaps the count update below (read-only table; nothing
            // uses the entry before the update is done)
            int4 dq = make_int4(0, 0, 0, 0);
            if (AHEAD && lane < h.w) dq = __ldcg(wt.depw32 + (h.z + lane));  // L2 only: the D(mu) lists stream (C5: 330 KB) and would evict the per-mu header, net-change and rate tables from L1
            int2 e = make_int2(0, 0);
            long long nv = 0;
            if (lane < h.y) {
                e = __ldg(wt.nuw + h.x + lane);  // (x byte offset, delta)
                nv = (long long)*(const int *)((const unsigned char *)xs + e.x) + e.y;
            }
            if (__any_sync(kFull, nv > 0x7fffffffll)) {  // a count would leave int32: freeze
                for (; j < jend; ++j) record(j);
                status = CWC_TRAJ_OVERFLOW;
                break;
            }
            if (lane < h.y) *(int *)((unsigned char *)xs + e.x) = (int)nv;
            __syncwarp();

            // Dependency-graph update: recompute a_m for m in D(mu) only
            // (byte-offset entries and A + A-halved rates: see ssa_warp2.cu).
            unsigned dirty = 0;
#pragma unroll 1
            for (int q = lane; q < h.w;) {
                const int4 d = AHEAD ? dq : __ldcg(wt.depw32 + (h.z + q));
                q += 32;
                if (AHEAD && q < h.w) dq = __ldcg(wt.depw32 + (h.z + q));  // (more than 32 dependents: the next round, in flight during this one)
                const double k = __ldg((const double *)((const unsigned char *)rates_h + (d.w & 0x3ffffff)));
                const int xa = *(const int *)((const unsigned char *)xs + d.y);
                const int xb = *(const int *)((const unsigned char *)xs + d.z) - (int)((unsigned)d.w >> 31);
                *(double *)((unsigned char *)as + d.x) = __dmul_rn(k, __dmul_rn(__int2double_rn(xa), __int2double_rn(xb)));
                dirty |= 1u << (((unsigned)d.w >> 26) & 31u);
            }
            dirty = __reduce_or_sync(kFull, dirty);
            __syncwarp();
            if ((dirty >> lane) & 1u) part = SUM4 ? chunk_sum4<BMAX>(as + lane * Bp, B) : chunk_sum<BMAX>(as + lane * Bp, B);
            incl = warp_incl_scan(part, lane);
            a0 = shfl_d(incl, 31);
            excl = __shfl_up_sync(kFull, incl, 1);
            if (lane == 0) excl = 0.0;

            t = tn;
            ++kd;
            ++n;
            asm volatile("bar.warp.sync -1;" ::: "memory");  // keep the warp converged
        }
        if (RES && j <= J && status == CWC_TRAJ_DONE) status = CWC_TRAJ_RUNNING;  // suspended
        if (lane == 0) {
            if (rp.out_firings) rp.out_firings[g] = (int64_t)n;
            if (rp.out_status) rp.out_status[g] = status;
            if (TRACE && tslot >= 0) rp.trace_len[tslot] = tn_rec;
        }
        if (RES) {
            for (int c = lane; c < wt.n_cells; c += 32) rp.rs_x[g * wt.n_cells + c] = xs[c];
            if (lane == 0) {
                rp.rs_t[g] = t;
                rp.rs_n[g] = (int64_t)n;
                rp.rs_j[g] = (int32_t)j;
            }
        }
        __syncwarp();
    }

    if (rp.stats_smem) {
        __syncthreads();
        const long long n16 = stat_bytes(rp.st, rp.cells_per_part) / 16;
        uint4 *dst = (uint4 *)((unsigned char *)rp.parts + (long long)blockIdx.x * stat_bytes(rp.st, rp.cells_per_part));
        const uint4 *src = (const uint4 *)smem;
        for (long long q = threadIdx.x; q < n16; q += blockDim.x) dst[q] = src[q];
    }
}

static inline int align16(long long v) { return (int)((v + 15) & ~15ll); }

size_t warp_smem_per_warp(const WarpTables &wt) {
    return (size_t)align16(4ll * (wt.n_cells + 1)) + (size_t)8 * 32 * wt.Bp;
}

cudaError_t launch_ssa_warp(const RunParams &rp, const WarpTables &wt, int blocks, int warps_per_block,
                            size_t smem_bytes, cudaStream_t stream) {
    const long long stats_bytes = rp.stats_smem ? stat_bytes(rp.st, rp.cells_per_part) : 0;
    const int x_bytes = align16(4ll * (wt.n_cells + 1));
    const int per_warp = (int)warp_smem_per_warp(wt);
    const bool small = (size_t)smem_bytes * 8 <= (size_t)220 * 1024 && warps_per_block <= 4;
    auto pick = [&](auto tr, auto rs) {
        constexpr bool T = decltype(tr)::value, R = decltype(rs)::value;
        if (wt.B <= 8) return small ? ssa_warp_kernel<T, 8, 8, R> : ssa_warp_kernel<T, 6, 8, R>;
        if (wt.B <= 16) return small ? ssa_warp_kernel<T, 8, 16, R> : ssa_warp_kernel<T, 6, 16, R>;
        if (wt.B <= 40) return small ? ssa_warp_kernel<T, 8, 40, R> : ssa_warp_kernel<T, 6, 40, R>;
        return small ? ssa_warp_kernel<T, 8, 0, R> : ssa_warp_kernel<T, 6, 0, R>;
    };
    // resumable runs never trace (the planner refuses it)
    auto k = rp.rs_x ? pick(std::false_type{}, std::true_type{})
                     : (rp.n_trace > 0) ? pick(std::true_type{}, std::false_type{}) : pick(std::false_type{}, std::false_type{});
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_bytes);
    if (e != cudaSuccess) return e;
    k<<<blocks, warps_per_block * 32, smem_bytes, stream>>>(rp, wt, stats_bytes, per_warp, x_bytes);
    return cudaGetLastError();
}

}  // namespace cwc
