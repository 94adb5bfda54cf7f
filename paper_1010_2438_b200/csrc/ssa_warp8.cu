// ssa_warp8.cu -- several trajectories per warp in LG-lane groups: eight
// (LG = 4, CWC_KERNEL_WARP8) or four (LG = 8, CWC_KERNEL_WARP4), for the
// warp path's medium networks (M <= 256).  Described below for LG = 4; with
// LG = 8 every quantity scales (B = ceil(M/8) <= 32 entries per lane, two
// sub-chunks, two entries per lane in the selection's read, 8-lane scans).
//
// Same method and result class as ssa_warp2_kernel (a0 and the selection
// prefixes in the device's own summation tree), with
// the warp split into eight 4-lane groups that each run one trajectory.
// Why: the warp kernels are issue-bound, and every warp instruction of the
// per-firing fixed part -- division, ballots, scans, loop control -- now
// advances eight trajectories instead of two; the per-entry work (chunk
// re-sums, dependency updates) is the same per firing whatever the split.
//
// Layout (per warp, shared memory):
//   propensities aw [64 rows][32 columns] fp64: lane gl of group q owns
//     entries m = gl*B4 + k (k < B4 = ceil(M/4) <= 64) at row k, column
//     4q + (gl ^ ((k >> 2) & 3)).  The owner's sweep over its rows, the
//     selection's four-entries-per-lane read of one owner's sub-chunk and the
//     group-uniform dependency writes are all bank-conflict free;
//   sub-chunk sums ss [4][32]: entries k in [16c, 16c + 16) of the owner,
//     left to right; the lane total is ((s0 + s1) + s2) + s3; a 4-lane
//     shuffle scan gives the group prefixes, a0 = prefix of lane 3;
//   counts x [cell][8] int32 (cell n_cells reads 1: absent reactants);
//   draws dr [32 slots][8] (E = -log u1, u2): all groups consume one draw per
//     loop iteration, so the rings are refilled together every 32 iterations
//     (each lane computing eight draws of its group); a trajectory that starts
//     mid-window fills the rest of the window.
// Selection: owner lane by ballot over the group prefixes, sub-chunk by a
// 4-lane scan of the owner's four sub-chunk sums, entry by each lane reading
// four consecutive entries of that sub-chunk and a 4-lane scan of their sums;
// fallback: the last positive entry.
// Update: one lane per changed cell; the dependents D(mu) are recomputed by
// the group's lanes (a = k' RN(x_a (x_b - sub)), k' halved for A + A), each
// marking (owner, sub-chunk) dirty; dirty sub-chunks are re-summed by their
// owners.
#include <cuda_runtime.h>

#include "cwc_internal.h"
#include "device_common.cuh"

namespace cwc {

namespace {

constexpr unsigned kAll8 = 0xffffffffu;

// inclusive scan within each aligned group of LG lanes
template <int LG>
__device__ __forceinline__ double group_scan(double v, int gl) {
#pragma unroll
    for (int d = 1; d < LG; d <<= 1) {
        const double y = __shfl_up_sync(kAll8, v, d, LG);
        if (gl >= d) v = __dadd_rn(y, v);
    }
    return v;
}

}  // namespace

template <int LG, bool TRACE>
__global__ void __launch_bounds__(128) ssa_group_kernel(const RunParams rp, const WarpTables wt, int per_warp_bytes) {
    static_assert(LG == 4 || LG == 8, "4- or 8-lane groups");
    constexpr int TPW = 32 / LG;          // trajectories per warp
    constexpr int EPL = 16 / LG;          // entries per lane in the selection's sub-chunk read = sub-chunks per lane
    constexpr int SH = LG == 4 ? 2 : 1;   // log2(EPL): column swizzle (k >> SH) & (LG - 1)
    constexpr int XSH = LG == 4 ? 0 : 1;  // x byte offsets in the tables are cell * 32 (TPW = 8)
    constexpr unsigned GM = (1u << LG) - 1u;
    extern __shared__ __align__(16) unsigned char smem[];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int gq = lane / LG, gl = lane & (LG - 1), gb = gq * LG;  // group, lane in group, group's first lane
    const int M = wt.M, B4 = (M + LG - 1) / LG;
    const int NS = B4 > 0 ? (B4 + 15) >> 4 : 1;  // (a model without rules keeps one zeroed sub-chunk: the selection's reads stay in range)
    const int O = wt.O;
    const long long J = rp.J, J1 = J + 1;
    unsigned char *base = smem + (size_t)wib * per_warp_bytes;
    double *aw = (double *)base;                           // [16 NS][32]
    double *ss = aw + 16 * NS * 32;                        // [4][32]
    double2 *dr = (double2 *)(ss + 4 * 32);                // [32][TPW]
    int *xw = (int *)(dr + 32 * TPW);                      // [n_cells + 1][TPW]
    const int4 *depg = LG == 4 ? wt.depw4 : wt.depw8;
    const StatAcc acc = stat_view((unsigned char *)rp.parts, rp.cells_per_part, rp.st);

    bool active = false, exhausted = false;
    long long g = 0;
    const double *rates = rp.rates, *rates_h = rp.rates_h;
    uint64_t gk = 0;
    double t = 0.0, t_next = 0.0, a0 = 0.0, incl = 0.0, excl = 0.0, part = 0.0;
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;  // my sub-chunk sums
    int j = 0;
    unsigned long long n = 0;
    unsigned it = 0;  // loop iterations of this warp (ring slot = it & 31)
    int tslot = -1;
    long long tn_rec = 0;
    auto trace_rec = [&](unsigned long long n_, double a0_, double tau, double tn, int mu) {
        if (TRACE && tslot >= 0 && tn_rec < rp.trace_cap) {
            if (gl == 0) {
                double *r = rp.trace_buf + ((long long)tslot * rp.trace_cap + tn_rec) * 5;
                r[0] = (double)n_; r[1] = a0_; r[2] = tau; r[3] = tn; r[4] = (double)mu;
            }
            ++tn_rec;
        }
    };
    auto record = [&](int jj) {  // rare, divergent per group
        const long long cb = (g / rp.R) * J1 * O + (long long)jj * O;
        for (int o = gl; o < O; o += LG) {
            long long v = 0;
            for (int q = __ldg(wt.obs_ptr + o); q < __ldg(wt.obs_ptr + o + 1); ++q) v += xw[__ldg(wt.obs_cells + q) * TPW + gq];
            stat_record(acc, cb + o, v);
            if (rp.out_traj) rp.out_traj[(g * J1 + jj) * O + o] = v;
        }
    };
    auto finish = [&](int status) {
        if (gl == 0) {
            if (rp.out_firings) rp.out_firings[g] = (int64_t)n;
            if (rp.out_status) rp.out_status[g] = status;
            if (TRACE && tslot >= 0) rp.trace_len[tslot] = tn_rec;
        }
        active = false;
    };
    // draws for ring slots [from, 32) of my group: counter nb + slot, slot = gl + LG i
    auto fill_draws = [&](int from, unsigned long long nb) {
#pragma unroll 1
        for (int sl = gl; sl < 32; sl += LG) {
            if (sl >= from) {
                double E, u;
                block_to_draws(philox_block(rp.seed, gk, nb + (unsigned long long)sl), E, u);
                dr[sl * TPW + gq] = make_double2(E, u);
            }
        }
    };

    for (;;) {
        // ---- groups without a trajectory take the next one (rare) ----
        const bool need = !active && !exhausted;
        if (__any_sync(kAll8, need)) {
            unsigned long long gg = ~0ull;
            if (need && gl == 0) gg = atomicAdd(rp.next_traj, 1ull);
            gg = __shfl_sync(kAll8, gg, gb);
            const bool got = need && gg < (unsigned long long)rp.n_launch;
            if (need && !got) exhausted = true;
            if (got) {
                g = (long long)gg;
                const long long p = g / rp.R;
                rates = rp.rates + p * M;
                rates_h = rp.rates_h + p * M;
                gk = (uint64_t)global_traj(g, rp.R, rp.R_total, rp.r_off);
                if (TRACE) {
                    tslot = -1;
                    tn_rec = 0;
                    for (int q = 0; q < rp.n_trace; ++q)
                        if (rp.trace_g[q] == g) tslot = q;
                }
                for (int c = gl; c < wt.n_cells; c += LG) xw[c * TPW + gq] = __ldg(wt.init + c);
                if (gl == 0) xw[wt.n_cells * TPW + gq] = 1;
            }
            __syncwarp();
            if (got) {
                // propensities of my entries, sub-chunk sums
                double sc[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll 1
                for (int k = 0; k < 16 * NS; ++k) {
                    const int m = gl * B4 + k;
                    double a = 0.0;
                    if (k < B4 && m < M) {
                        const int4 d = __ldg(reinterpret_cast<const int4 *>(wt.rx) + m);
                        a = __dmul_rn(__ldg(rates + m),
                                      combos(xw[d.x * TPW + gq], xw[d.y * TPW + gq], d.z & 1, d.z >> 1));
                    }
                    aw[k * 32 + gb + (gl ^ ((k >> SH) & (LG - 1)))] = a;
                    const int c = k >> 4;
                    const double prev = (c == 0) ? sc[0] : (c == 1) ? sc[1] : (c == 2) ? sc[2] : sc[3];
                    const double nv = ((k & 15) == 0) ? a : __dadd_rn(prev, a);
                    if (c == 0) sc[0] = nv; else if (c == 1) sc[1] = nv; else if (c == 2) sc[2] = nv; else sc[3] = nv;
                }
                s0 = sc[0]; s1 = sc[1]; s2 = sc[2]; s3 = sc[3];
                ss[0 * 32 + lane] = s0;
                ss[1 * 32 + lane] = s1;
                ss[2 * 32 + lane] = s2;
                ss[3 * 32 + lane] = s3;
                part = LG == 4 ? __dadd_rn(__dadd_rn(__dadd_rn(s0, s1), s2), s3) : __dadd_rn(s0, s1);
                t = 0.0;
                j = 0;
                n = 0;
                t_next = 0.0;
                // this window's remaining slots: slot it&31 takes counter 0
                const int from = (int)(it & 31u);
                fill_draws(from, 0ull - (unsigned long long)from);
                active = true;
            }
            // group scans for everyone (groups that did not change recompute the same values)
            const double in = group_scan<LG>(part, gl);
            const double a0n = __shfl_sync(kAll8, in, gb + LG - 1);
            const double ex = __shfl_up_sync(kAll8, in, 1, LG);
            if (got) {
                incl = in;
                a0 = a0n;
                excl = gl == 0 ? 0.0 : ex;
            }
            __syncwarp();
        }
        if (!__any_sync(kAll8, active)) break;

        // ---- all rings refilled together at window boundaries ----
        const int slot = (int)(it & 31u);
        if (slot == 0) {
            if (active) fill_draws(0, n);
            __syncwarp();
        }
        const double2 d2 = dr[slot * TPW + gq];
        const double E = d2.x, u2 = d2.y;
        const double tau = div_fast_ok(E, a0) ? div_fast(E, a0) : __ddiv_rn(E, a0);
        const double tn = __dadd_rn(t, tau);
        bool fire = active;
        const bool cross = active && !(tn < t_next);
        if (__any_sync(kAll8, cross)) {
            if (cross) {  // divergent: no warp-wide intrinsics inside
                if (a0 == 0.0) {  // stall
                    for (; j <= J; ++j) record(j);
                    finish(CWC_TRAJ_STALLED);
                    fire = false;
                } else {
                    while (j <= J && __dmul_rn(__int2double_rn(j), rp.dt) <= tn) {
                        record(j);
                        ++j;
                    }
                    if (j > J) {  // horizon reached: drawn, not applied
                        trace_rec(n, a0, tau, tn, -1);
                        finish(CWC_TRAJ_DONE);
                        fire = false;
                    } else {
                        t_next = __dmul_rn(__int2double_rn(j), rp.dt);
                    }
                }
            }
            __syncwarp();
        }

        // ---- selection (a8) ----
        const double target = __dmul_rn(u2, a0);
        const unsigned gmask = GM << gb;
        const unsigned hL = (__ballot_sync(kAll8, incl > target) & gmask) >> gb;
        const unsigned pL = (__ballot_sync(kAll8, part > 0.0) & gmask) >> gb;
        const int L = hL ? __ffs(hL) - 1 : (pL ? 31 - __clz(pL) : 0);
        const double carry = __shfl_sync(kAll8, excl, gb + L);
        // owner L's sub-chunk sums: lane gl takes sub-chunk gl
        const double sv = gl < NS ? ss[gl * 32 + gb + L] : 0.0;
        const double sc_in = group_scan<LG>(sv, gl);
        const double cumc = __dadd_rn(carry, sc_in);
        const unsigned hC = (__ballot_sync(kAll8, gl < NS && target < cumc) & gmask) >> gb;
        const unsigned pC = (__ballot_sync(kAll8, sv > 0.0) & gmask) >> gb;
        // (clamped: a group without a trajectory runs this on stale shared
        // memory, and its reads must stay inside the warp's rows)
        const int C = min(hC ? __ffs(hC) - 1 : (pC ? 31 - __clz(pC) : 0), NS - 1);
        const double sc_ex = __shfl_up_sync(kAll8, sc_in, 1, LG);
        const double cex = __shfl_sync(kAll8, gl == 0 ? 0.0 : sc_ex, gb + C);
        const double carry2 = __dadd_rn(carry, cex);
        // EPL consecutive entries of sub-chunk C of owner L per lane
        const int k0 = 16 * C + EPL * gl;
        const int col = gb + (L ^ gl);  // (k >> SH) & (LG - 1) == gl for k in [k0, k0 + EPL)
        double ev[EPL], lp[EPL];
#pragma unroll
        for (int i = 0; i < EPL; ++i) {
            ev[i] = aw[(k0 + i) * 32 + col];
            lp[i] = i ? __dadd_rn(lp[i - 1], ev[i]) : ev[i];
        }
        const double lin = group_scan<LG>(lp[EPL - 1], gl);
        const double lex = __shfl_up_sync(kAll8, lin, 1, LG);
        const double b0 = __dadd_rn(carry2, gl == 0 ? 0.0 : lex);
        int hi_ = -1, lastpos = -1;
#pragma unroll
        for (int i = EPL - 1; i >= 0; --i) {
            if (target < __dadd_rn(b0, lp[i])) hi_ = i;
            if (lastpos < 0 && ev[i] > 0.0) lastpos = i;
        }
        const unsigned hE = (__ballot_sync(kAll8, hi_ >= 0) & gmask) >> gb;
        const unsigned pE = (__ballot_sync(kAll8, lastpos >= 0) & gmask) >> gb;
        const int G = hE ? __ffs(hE) - 1 : (pE ? 31 - __clz(pE) : 0);
        const int iG = __shfl_sync(kAll8, hE ? hi_ : lastpos, gb + G);
        const int mu = L * B4 + 16 * C + EPL * G + (iG < 0 ? 0 : iG);
        if (TRACE && fire) trace_rec(n, a0, tau, tn, mu);

        // ---- update (a9): one lane per changed cell ----
        const int4 h = fire ? __ldg(wt.hdr + mu) : make_int4(0, 0, 0, 0);
        int2 e = make_int2(0, 0);
        long long nv = 0;
        if (gl < h.y) {  // |nu| <= 4 for order <= 2 reactions with <= 2 products
            e = __ldg(wt.nuw8 + h.x + gl);  // (cell * 32, delta)
            nv = (long long)*(const int *)((const unsigned char *)xw + (e.x >> XSH) + gq * 4) + e.y;
        }
        for (int q = gl + LG; q < h.y; q += LG) {  // (more than LG changed cells)
            const int2 e2 = __ldg(wt.nuw8 + h.x + q);
            const long long v2 = (long long)*(const int *)((const unsigned char *)xw + (e2.x >> XSH) + gq * 4) + e2.y;
            nv = v2 > nv ? v2 : nv;  // only the overflow test needs it here
        }
        const bool ovf = ((__ballot_sync(kAll8, nv > 0x7fffffffll) & gmask) != 0u);
        if (__any_sync(kAll8, ovf)) {
            if (ovf) {  // a count would leave int32: freeze + fill
                for (; j <= J; ++j) record(j);
                finish(CWC_TRAJ_OVERFLOW);
                fire = false;
            }
            __syncwarp();
        }
        if (fire) {
            for (int q = gl; q < h.y; q += LG) {
                const int2 e2 = __ldg(wt.nuw8 + h.x + q);
                int *px = (int *)((unsigned char *)xw + (e2.x >> XSH) + gq * 4);
                *px = *px + e2.y;
            }
        }
        __syncwarp();

        // ---- dependency-graph update (a3) ----
        // four entries per lane loaded before any is used (their global-load
        // latencies overlap: the group's dependents take one round trip, not
        // one per entry)
        unsigned dirty = 0;
        if (fire) {
#pragma unroll 1
            for (int q0 = 0; q0 < h.w; q0 += 4 * LG) {
                int4 dd[4];
                double kk[4];
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const int q = q0 + gl + LG * i;
                    dd[i] = q < h.w ? __ldg(depg + h.z + q) : make_int4(0, 0, 0, -1);
                }
#pragma unroll
                for (int i = 0; i < 4; ++i)
                    kk[i] = dd[i].w != -1 ? __ldg((const double *)((const unsigned char *)rates_h + (dd[i].w & 0x3ffffff))) : 0.0;
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    if (dd[i].w == -1) continue;
                    const int4 d = dd[i];
                    const int xa = *(const int *)((const unsigned char *)xw + (d.y >> XSH) + gq * 4);
                    const int xb = *(const int *)((const unsigned char *)xw + (d.z >> XSH) + gq * 4) - (int)((unsigned)d.w >> 31);
                    *(double *)((unsigned char *)aw + d.x + gb * 8) =
                        __dmul_rn(kk[i], __dmul_rn(__int2double_rn(xa), __int2double_rn(xb)));
                    dirty |= 1u << (((unsigned)d.w >> 26) & 15u);
                }
            }
        }
#pragma unroll
        for (int d = 1; d < LG; d <<= 1) dirty |= __shfl_xor_sync(kAll8, dirty, d);
        const unsigned mine = (dirty >> (EPL * gl)) & ((1u << EPL) - 1u);
        __syncwarp();
        // ---- dirty sub-chunks re-summed by their owners: the four sums as
        // independent chains in one pass (predicated per sub-chunk) ----
        if (__any_sync(kAll8, mine != 0u)) {
            const bool r0 = mine & 1u, r1 = mine & 2u, r2 = mine & 4u, r3 = mine & 8u;
            double t0 = 0.0, t1 = 0.0, t2 = 0.0, t3 = 0.0;
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                const int cofs = gb + (gl ^ ((i >> SH) & (LG - 1)));
                if (r0) { const double a = aw[i * 32 + cofs]; t0 = i ? __dadd_rn(t0, a) : a; }
                if (r1) { const double a = aw[(16 + i) * 32 + cofs]; t1 = i ? __dadd_rn(t1, a) : a; }
                if (LG == 4 && r2) { const double a = aw[(32 + i) * 32 + cofs]; t2 = i ? __dadd_rn(t2, a) : a; }
                if (LG == 4 && r3) { const double a = aw[(48 + i) * 32 + cofs]; t3 = i ? __dadd_rn(t3, a) : a; }
            }
            if (r0) { s0 = t0; ss[0 * 32 + lane] = s0; }
            if (r1) { s1 = t1; ss[1 * 32 + lane] = s1; }
            if (LG == 4 && r2) { s2 = t2; ss[2 * 32 + lane] = s2; }
            if (LG == 4 && r3) { s3 = t3; ss[3 * 32 + lane] = s3; }
        }
        if (mine) part = LG == 4 ? __dadd_rn(__dadd_rn(__dadd_rn(s0, s1), s2), s3) : __dadd_rn(s0, s1);
        incl = group_scan<LG>(part, gl);
        a0 = __shfl_sync(kAll8, incl, gb + LG - 1);
        excl = __shfl_up_sync(kAll8, incl, 1, LG);
        if (gl == 0) excl = 0.0;
        if (fire) {  // (an active group that did not fire has finished)
            t = tn;
            ++n;
        }
        ++it;
        asm volatile("bar.warp.sync -1;" ::: "memory");
    }
}

size_t group_smem_per_warp(const WarpTables &wt, int LG) {  // aw [16 NS][32], ss [4][32], dr [32][TPW], x [cells + 1][TPW]
    const int B = (wt.M + LG - 1) / LG, NS = B > 0 ? (B + 15) >> 4 : 1, TPW = 32 / LG;
    return (size_t)8 * 16 * NS * 32 + (size_t)8 * 4 * 32 + (size_t)16 * 32 * TPW + (size_t)4 * TPW * (wt.n_cells + 1);
}

cudaError_t launch_ssa_group(int LG, const RunParams &rp, const WarpTables &wt, int blocks, int warps_per_block,
                             size_t smem_bytes, cudaStream_t stream) {
    const int per_warp = (int)((group_smem_per_warp(wt, LG) + 15) & ~(size_t)15);
    auto k = LG == 4 ? (rp.n_trace > 0 ? ssa_group_kernel<4, true> : ssa_group_kernel<4, false>)
                     : (rp.n_trace > 0 ? ssa_group_kernel<8, true> : ssa_group_kernel<8, false>);
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_bytes);
    if (e != cudaSuccess) return e;
    k<<<blocks, warps_per_block * 32, smem_bytes, stream>>>(rp, wt, per_warp);
    return cudaGetLastError();
}

}  // namespace cwc
