// ssa_warp8.cu -- eight trajectories per warp (4-lane groups), for the warp
// path's medium networks (M <= 256: C4).
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

// 4-lane inclusive scan (within each aligned lane quad)
__device__ __forceinline__ double quad_scan(double v, int gl) {
    double y = __shfl_up_sync(kAll8, v, 1, 4);
    if (gl >= 1) v = __dadd_rn(y, v);
    y = __shfl_up_sync(kAll8, v, 2, 4);
    if (gl >= 2) v = __dadd_rn(y, v);
    return v;
}

}  // namespace

template <bool TRACE>
__global__ void __launch_bounds__(128) ssa_warp8_kernel(const RunParams rp, const WarpTables wt, int per_warp_bytes) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int gq = lane >> 2, gl = lane & 3, gb = gq << 2;  // group, lane in group, group's first lane
    const int B4 = wt.B4, NS = (B4 + 15) >> 4;
    const int O = wt.O, M = wt.M;
    const long long J = rp.J, J1 = J + 1;
    unsigned char *base = smem + (size_t)wib * per_warp_bytes;
    double *aw = (double *)base;                           // [16 NS][32]
    double *ss = aw + 16 * NS * 32;                        // [4][32]
    double2 *dr = (double2 *)(ss + 4 * 32);                // [32][8]
    int *xw = (int *)(dr + 32 * 8);                        // [n_cells + 1][8]
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
        for (int o = gl; o < O; o += 4) {
            long long v = 0;
            for (int q = __ldg(wt.obs_ptr + o); q < __ldg(wt.obs_ptr + o + 1); ++q) v += xw[__ldg(wt.obs_cells + q) * 8 + gq];
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
    // draws for ring slots [from, 32) of my group: counter nb + slot, slot = gl + 4i
    auto fill_draws = [&](int from, unsigned long long nb) {
#pragma unroll 1
        for (int sl = gl; sl < 32; sl += 4) {
            if (sl >= from) {
                double E, u;
                block_to_draws(philox_block(rp.seed, gk, nb + (unsigned long long)sl), E, u);
                dr[sl * 8 + gq] = make_double2(E, u);
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
                for (int c = gl; c < wt.n_cells; c += 4) xw[c * 8 + gq] = __ldg(wt.init + c);
                if (gl == 0) xw[wt.n_cells * 8 + gq] = 1;
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
                                      combos(xw[d.x * 8 + gq], xw[d.y * 8 + gq], d.z & 1, d.z >> 1));
                    }
                    aw[k * 32 + gb + (gl ^ ((k >> 2) & 3))] = a;
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
                part = __dadd_rn(__dadd_rn(__dadd_rn(s0, s1), s2), s3);
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
            const double in = quad_scan(part, gl);
            const double a0n = __shfl_sync(kAll8, in, gb + 3);
            const double ex = __shfl_up_sync(kAll8, in, 1, 4);
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
        const double2 d2 = dr[slot * 8 + gq];
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
        const unsigned gmask = 0xfu << gb;
        const unsigned hL = (__ballot_sync(kAll8, incl > target) & gmask) >> gb;
        const unsigned pL = (__ballot_sync(kAll8, part > 0.0) & gmask) >> gb;
        const int L = hL ? __ffs(hL) - 1 : (pL ? 31 - __clz(pL) : 0);
        const double carry = __shfl_sync(kAll8, excl, gb + L);
        // owner L's sub-chunk sums: lane gl takes sub-chunk gl
        const double sv = ss[gl * 32 + gb + L];
        const double sc_in = quad_scan(sv, gl);
        const double cumc = __dadd_rn(carry, sc_in);
        const unsigned hC = (__ballot_sync(kAll8, gl < NS && target < cumc) & gmask) >> gb;
        const unsigned pC = (__ballot_sync(kAll8, sv > 0.0) & gmask) >> gb;
        // (clamped: a group without a trajectory runs this on stale shared
        // memory, and its reads must stay inside the warp's rows)
        const int C = min(hC ? __ffs(hC) - 1 : (pC ? 31 - __clz(pC) : 0), NS - 1);
        const double sc_ex = __shfl_up_sync(kAll8, sc_in, 1, 4);
        const double cex = __shfl_sync(kAll8, gl == 0 ? 0.0 : sc_ex, gb + C);
        const double carry2 = __dadd_rn(carry, cex);
        // four consecutive entries of sub-chunk C of owner L per lane
        const int k0 = 16 * C + 4 * gl;
        const int col = gb + (L ^ gl);  // (k >> 2) & 3 == gl for k in [k0, k0 + 4)
        const double e0 = aw[(k0 + 0) * 32 + col], e1 = aw[(k0 + 1) * 32 + col];
        const double e2 = aw[(k0 + 2) * 32 + col], e3 = aw[(k0 + 3) * 32 + col];
        const double l1 = __dadd_rn(e0, e1), l2 = __dadd_rn(l1, e2), l3 = __dadd_rn(l2, e3);
        const double lin = quad_scan(l3, gl);
        const double lex = __shfl_up_sync(kAll8, lin, 1, 4);
        const double b0 = __dadd_rn(carry2, gl == 0 ? 0.0 : lex);
        int hi_ = -1;
        if (target < __dadd_rn(b0, e0)) hi_ = 0;
        else if (target < __dadd_rn(b0, l1)) hi_ = 1;
        else if (target < __dadd_rn(b0, l2)) hi_ = 2;
        else if (target < __dadd_rn(b0, l3)) hi_ = 3;
        const int lastpos = e3 > 0.0 ? 3 : e2 > 0.0 ? 2 : e1 > 0.0 ? 1 : e0 > 0.0 ? 0 : -1;
        const unsigned hE = (__ballot_sync(kAll8, hi_ >= 0) & gmask) >> gb;
        const unsigned pE = (__ballot_sync(kAll8, lastpos >= 0) & gmask) >> gb;
        const int G = hE ? __ffs(hE) - 1 : (pE ? 31 - __clz(pE) : 0);
        const int iG = __shfl_sync(kAll8, hE ? hi_ : lastpos, gb + G);
        const int mu = L * B4 + 16 * C + 4 * G + (iG < 0 ? 0 : iG);
        if (TRACE && fire) trace_rec(n, a0, tau, tn, mu);

        // ---- update (a9): one lane per changed cell ----
        const int4 h = fire ? __ldg(wt.hdr + mu) : make_int4(0, 0, 0, 0);
        int2 e = make_int2(0, 0);
        long long nv = 0;
        if (gl < h.y) {  // |nu| <= 4 for order <= 2 reactions with <= 2 products
            e = __ldg(wt.nuw8 + h.x + gl);  // (cell * 32, delta)
            nv = (long long)*(const int *)((const unsigned char *)xw + e.x + gq * 4) + e.y;
        }
        for (int q = gl + 4; q < h.y; q += 4) {  // (more than four changed cells)
            const int2 e2 = __ldg(wt.nuw8 + h.x + q);
            const long long v2 = (long long)*(const int *)((const unsigned char *)xw + e2.x + gq * 4) + e2.y;
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
            for (int q = gl; q < h.y; q += 4) {
                const int2 e2 = __ldg(wt.nuw8 + h.x + q);
                int *px = (int *)((unsigned char *)xw + e2.x + gq * 4);
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
            for (int q0 = 0; q0 < h.w; q0 += 16) {
                int4 dd[4];
                double kk[4];
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const int q = q0 + gl + 4 * i;
                    dd[i] = q < h.w ? __ldg(wt.depw4 + h.z + q) : make_int4(0, 0, 0, -1);
                }
#pragma unroll
                for (int i = 0; i < 4; ++i)
                    kk[i] = dd[i].w != -1 ? __ldg((const double *)((const unsigned char *)rates_h + (dd[i].w & 0x3ffffff))) : 0.0;
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    if (dd[i].w == -1) continue;
                    const int4 d = dd[i];
                    const int xa = *(const int *)((const unsigned char *)xw + d.y + gq * 4);
                    const int xb = *(const int *)((const unsigned char *)xw + d.z + gq * 4) - (int)((unsigned)d.w >> 31);
                    *(double *)((unsigned char *)aw + d.x + gb * 8) =
                        __dmul_rn(kk[i], __dmul_rn(__int2double_rn(xa), __int2double_rn(xb)));
                    dirty |= 1u << (((unsigned)d.w >> 26) & 15u);
                }
            }
        }
        dirty |= __shfl_xor_sync(kAll8, dirty, 1);
        dirty |= __shfl_xor_sync(kAll8, dirty, 2);
        const unsigned mine = (dirty >> (4 * gl)) & 0xfu;
        __syncwarp();
        // ---- dirty sub-chunks re-summed by their owners: the four sums as
        // independent chains in one pass (predicated per sub-chunk) ----
        if (__any_sync(kAll8, mine != 0u)) {
            const bool r0 = mine & 1u, r1 = mine & 2u, r2 = mine & 4u, r3 = mine & 8u;
            double t0 = 0.0, t1 = 0.0, t2 = 0.0, t3 = 0.0;
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                const int cofs = gb + (gl ^ ((i >> 2) & 3));
                if (r0) { const double a = aw[i * 32 + cofs]; t0 = i ? __dadd_rn(t0, a) : a; }
                if (r1) { const double a = aw[(16 + i) * 32 + cofs]; t1 = i ? __dadd_rn(t1, a) : a; }
                if (r2) { const double a = aw[(32 + i) * 32 + cofs]; t2 = i ? __dadd_rn(t2, a) : a; }
                if (r3) { const double a = aw[(48 + i) * 32 + cofs]; t3 = i ? __dadd_rn(t3, a) : a; }
            }
            if (r0) { s0 = t0; ss[0 * 32 + lane] = s0; }
            if (r1) { s1 = t1; ss[1 * 32 + lane] = s1; }
            if (r2) { s2 = t2; ss[2 * 32 + lane] = s2; }
            if (r3) { s3 = t3; ss[3 * 32 + lane] = s3; }
        }
        if (mine) part = __dadd_rn(__dadd_rn(__dadd_rn(s0, s1), s2), s3);
        incl = quad_scan(part, gl);
        a0 = __shfl_sync(kAll8, incl, gb + 3);
        excl = __shfl_up_sync(kAll8, incl, 1, 4);
        if (gl == 0) excl = 0.0;
        if (fire) {  // (an active group that did not fire has finished)
            t = tn;
            ++n;
        }
        ++it;
        asm volatile("bar.warp.sync -1;" ::: "memory");
    }
}

size_t warp8_smem_per_warp(const WarpTables &wt) {  // aw [16 NS][32], ss [4][32], dr [32][8], x [cells + 1][8]
    const int NS = (wt.B4 + 15) >> 4;
    return (size_t)8 * 16 * NS * 32 + (size_t)8 * 4 * 32 + (size_t)16 * 32 * 8 + (size_t)4 * 8 * (wt.n_cells + 1);
}

cudaError_t launch_ssa_warp8(const RunParams &rp, const WarpTables &wt, int blocks, int warps_per_block,
                             size_t smem_bytes, cudaStream_t stream) {
    const int per_warp = (int)((warp8_smem_per_warp(wt) + 15) & ~(size_t)15);
    auto k = rp.n_trace > 0 ? ssa_warp8_kernel<true> : ssa_warp8_kernel<false>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_bytes);
    if (e != cudaSuccess) return e;
    k<<<blocks, warps_per_block * 32, smem_bytes, stream>>>(rp, wt, per_warp);
    return cudaGetLastError();
}

}  // namespace cwc
