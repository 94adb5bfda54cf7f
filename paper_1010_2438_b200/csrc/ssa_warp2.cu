// ssa_warp2.cu -- two trajectories per warp (half-warp segments), for the
// warp path's medium networks (M <= 256: C4).
//
// Same method, tables and result as ssa_warp_kernel (ssa_warp.cu), with the
// 32 lanes split into two 16-lane segments that each run their own
// trajectory.  The warp path is issue-bound (C4: ~400 warp instructions per
// firing at ~80 % issue utilisation), and most of its instructions --
// shuffles of the prefix scan, the division, ballots, loop control -- do the
// same work whatever the lane count; with two segments every such
// instruction advances two trajectories.  Lane l of segment s owns the chunk
// of reactions [l*B16, (l+1)*B16), B16 = ceil(M/16) <= 16, stored at slots
// l*Bp16 + k of the segment's shared memory (Bp16 = B16 | 1), with the
// dependency slots precomputed for this layout (WarpTables.dep16).
//
// Every warp-wide intrinsic runs convergently with the full mask; segmented
// behaviour comes from width-16 shuffles and from splitting ballots by
// segment.  Side effects of a segment without a trajectory (all trajectories
// taken) are predicated off.  Rare per-segment work (sample records, end of
// horizon, stall, overflow, fetching the next trajectory) runs in divergent
// branches that contain no warp-wide intrinsics, or convergently with the
// other segment's results discarded.
#include <cuda_runtime.h>

#include <cstdlib>

#include "cwc_internal.h"
#include "device_common.cuh"

namespace cwc {

namespace {

constexpr unsigned kAll = 0xffffffffu;

__device__ __forceinline__ double prop16(const WarpTables &wt, const int *xs, const double *rates, int m) {
    const int4 d = __ldg(reinterpret_cast<const int4 *>(wt.rx) + m);
    return __dmul_rn(__ldg(rates + m), combos(xs[d.x], xs[d.y], d.z & 1, d.z >> 1));
}

// Inclusive scan within each 16-lane segment over lanes [0, w) of the
// segment (w a power of two <= 16, warp-uniform).
__device__ __forceinline__ double seg_scan(double v, int sl, int w) {
#pragma unroll
    for (int d = 1; d < 16; d <<= 1) {
        if (d < w) {
            const double y = __shfl_up_sync(kAll, v, d, 16);
            if (sl >= d) v = __dadd_rn(y, v);
        }
    }
    return v;
}

template <int BMAX>
__device__ __forceinline__ double chunk_sum16(const double *ch, int B) {
    double s = ch[0];
#pragma unroll
    for (int k = 1; k < BMAX; ++k)
        if (k < B) s = __dadd_rn(s, ch[k]);
    return s;
}

}  // namespace

template <int MINB, bool TRACE>
__global__ void __launch_bounds__(128, MINB) ssa_warp2_kernel(const RunParams rp, const WarpTables wt,
                                                              long long stats_smem_bytes, int per_seg_bytes,
                                                              int x_bytes) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    const int seg = lane >> 4, sl = lane & 15, sb = seg << 4;
    const int B = wt.B16, Bp = wt.Bp16;
    int scan_w = 1;  // in-chunk scan width: next power of two >= B (<= 16)
    while (scan_w < B) scan_w <<= 1;
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
    int *xs = (int *)(smem + stats_smem_bytes + (long long)(wib * 2 + seg) * per_seg_bytes);
    double *as = (double *)((unsigned char *)xs + x_bytes);
    double2 *dr = (double2 *)(as + 16 * Bp);  // [32] the segment's draws (E, u2) of firings n - kd ..
    __shared__ unsigned int cta_traj;  // trajectories taken by this CTA (shared-memory part capacity)
    __shared__ unsigned long long q_stop[32];  // per segment: resumable runs' firing bound
    if (threadIdx.x == 0) cta_traj = 0;
    __syncthreads();

    // per-segment trajectory state (uniform over the segment's 16 lanes)
    bool active = false, exhausted = false;
    long long g = 0;
    const double *rates = rp.rates;
    const double *rates_h = rp.rates_h;
    uint64_t gk = 0;
    double t = 0.0, t_next = 0.0, a0 = 0.0, incl = 0.0, excl = 0.0, part = 0.0;
    // (kept lean: the kernel runs at 64 registers, and every live 64-bit
    // value pushes index arithmetic into rematerialisation.  n counts the
    // applied firings = the next draw's counter; kd = draws used from the
    // 32-draw window; samples j < rp.j_stop are recorded in this launch, J+1
    // in one-shot runs; a resumable run's firing bound sits in shared memory)
    int j = 0, kd = 0;
    unsigned long long n = 0;

    // divergence tracer (TRACE builds): per-firing records (n, a0, tau, t', mu)
    // of the trajectories listed in rp.trace_g, written by the segment's lane 0
    int tslot = -1;
    long long tn_rec = 0;
    auto trace_rec = [&](unsigned long long n_, double a0_, double tau, double tn, int mu) {
        if (TRACE && tslot >= 0 && tn_rec < rp.trace_cap) {
            if (sl == 0) {
                double *r = rp.trace_buf + ((long long)tslot * rp.trace_cap + tn_rec) * 5;
                r[0] = (double)n_; r[1] = a0_; r[2] = tau; r[3] = tn; r[4] = (double)mu;
            }
            ++tn_rec;
        }
    };

    auto record = [&](int jj) {  // rare: the statistics cell is recomputed from g
        const long long cb = (g / rp.R) * J1 * O + (long long)jj * O;
        for (int o = sl; o < O; o += 16) {
            long long v = 0;
            for (int q = __ldg(wt.obs_ptr + o); q < __ldg(wt.obs_ptr + o + 1); ++q) v += xs[__ldg(wt.obs_cells + q)];
            stat_record(acc, cb + o, v);
            if (rp.out_traj) rp.out_traj[(g * J1 + jj) * O + o] = v;
        }
    };
    auto finish = [&](int status) {  // the segment's trajectory ended or is suspended
        if (j <= J && status == CWC_TRAJ_DONE) status = CWC_TRAJ_RUNNING;
        if (sl == 0) {
            if (rp.out_firings) rp.out_firings[g] = (int64_t)n;
            if (rp.out_status) rp.out_status[g] = status;
            if (TRACE && tslot >= 0) rp.trace_len[tslot] = tn_rec;
        }
        if (rp.rs_x) {  // resumable runs: save (x, t, n, j)
            for (int c = sl; c < wt.n_cells; c += 16) rp.rs_x[g * wt.n_cells + c] = xs[c];
            if (sl == 0) {
                rp.rs_t[g] = t;
                rp.rs_n[g] = (int64_t)n;
                rp.rs_j[g] = (int32_t)j;
            }
        }
        active = false;
    };

    for (;;) {
        // ---- segments without a trajectory take the next one ----
        const bool need = !active && !exhausted;
        if (__any_sync(kAll, need)) {
            unsigned long long gg = ~0ull;
            if (need && sl == 0) {
                // a shared-memory part holds <= kSmemPartMaxTraj trajectories
                if (!rp.stats_smem || atomicAdd(&cta_traj, 1u) < (unsigned)kSmemPartMaxTraj)
                    gg = atomicAdd(rp.next_traj, 1ull);
            }
            gg = __shfl_sync(kAll, gg, sb);
            const bool got = need && gg < (unsigned long long)rp.n_launch;
            if (need && !got) exhausted = true;
            if (got) {
                g = launch_traj(rp, (long long)gg);
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
                // state: fresh (x0, t = 0, n = 0, j = 0) or resumed (cwc_run_advance)
                for (int c = sl; c < wt.n_cells; c += 16)
                    xs[c] = rp.rs_x ? rp.rs_x[g * wt.n_cells + c] : __ldg(wt.init + c);
                if (sl == 0) xs[wt.n_cells] = 1;
            }
            __syncwarp();
            double pt = 0.0;
            for (int k = 0; k < B; ++k) {
                const int m = sl * B + k;
                const double a = (got && m < M) ? prop16(wt, xs, rates, m) : 0.0;
                if (got) as[sl * Bp + k] = a;
                pt = (k == 0) ? a : __dadd_rn(pt, a);
            }
            const double in = seg_scan(pt, sl, 16);
            const double a0n = __shfl_sync(kAll, in, sb + 15);
            const double exn = __shfl_up_sync(kAll, in, 1, 16);
            if (got) {
                part = pt;
                incl = in;
                a0 = a0n;
                excl = (sl == 0) ? 0.0 : exn;
                t = 0.0;
                j = 0;
                n = 0;
                if (rp.rs_x) {
                    t = rp.rs_t[g];
                    j = rp.rs_j[g];
                    n = (unsigned long long)rp.rs_n[g];
                }
                t_next = __dmul_rn(__int2double_rn(j), rp.dt);
                kd = 0;
                if (sl == 0) q_stop[wib * 2 + seg] = rp.quantum > 0 ? n + (unsigned long long)rp.quantum : ~0ull;
                double e0, u0, e1, u1;
                block_to_draws(philox_block(rp.seed, gk, n + sl), e0, u0);
                block_to_draws(philox_block(rp.seed, gk, n + 16 + sl), e1, u1);
                dr[sl] = make_double2(e0, u0);
                dr[16 + sl] = make_double2(e1, u1);
                active = true;
                if (j >= rp.j_stop) finish(CWC_TRAJ_DONE);  // resumed at its launch's sample bound
            }
            __syncwarp();
        }
        if (!__any_sync(kAll, active)) break;

        // ---- one firing of each active segment ----
        const bool refill = active && kd == 32;
        if (__any_sync(kAll, refill)) {
            // resumable runs: suspend after `quantum` further firings (at a
            // 32-draw window boundary)
            if (refill && n >= q_stop[wib * 2 + seg]) {
                finish(CWC_TRAJ_DONE);
            } else if (refill) {
                kd = 0;
                double e0, u0, e1, u1;
                block_to_draws(philox_block(rp.seed, gk, n + sl), e0, u0);
                block_to_draws(philox_block(rp.seed, gk, n + 16 + sl), e1, u1);
                dr[sl] = make_double2(e0, u0);
                dr[16 + sl] = make_double2(e1, u1);
            }
            __syncwarp();
        }
        const int i = kd;  // segment-uniform
        const double2 d2 = dr[i & 31];      // broadcast read (all lanes of the segment, one address)
        const double E = d2.x, u2 = d2.y;
        const double tau = div_fast_ok(E, a0) ? div_fast(E, a0) : __ddiv_rn(E, a0);
        const double tn = __dadd_rn(t, tau);
        bool fire = active;
        const bool cross = active && !(tn < t_next);
        if (__any_sync(kAll, cross)) {
            if (cross) {  // divergent: no warp-wide intrinsics inside
                if (a0 == 0.0) {  // stall
                    for (; j < rp.j_stop; ++j) record(j);
                    finish(CWC_TRAJ_STALLED);
                    fire = false;
                } else {
                    while (j < rp.j_stop && __dmul_rn(__int2double_rn(j), rp.dt) <= tn) {
                        record(j);
                        ++j;
                    }
                    if (j >= rp.j_stop) {  // horizon (or the launch's last sample) reached: drawn, not applied
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

        // selection: chunk L by ballot over the segment's lane prefixes, then
        // mu inside chunk L by a segmented shuffle scan of its entries
        const double target = __dmul_rn(u2, a0);
        const unsigned hitsL = (__ballot_sync(kAll, incl > target) >> sb) & 0xffffu;
        const int L = (hitsL ? __ffs(hitsL) : 1) - 1;
        const double carry = __shfl_sync(kAll, excl, sb + L);
        const double av = (sl < B) ? as[L * Bp + sl] : 0.0;
        const double cum = __dadd_rn(carry, seg_scan(av, sl, scan_w));
        const unsigned hit = (__ballot_sync(kAll, sl < B && target < cum) >> sb) & 0xffffu;
        const unsigned pos = (__ballot_sync(kAll, av > 0.0) >> sb) & 0xffffu;
        // the chunk's scanned sums may round below the lane prefix: take its
        // last positive entry
        const int mu = L * B + (hit ? __ffs(hit) - 1 : (pos ? 31 - __clz(pos) : 0));
        if (TRACE && fire) trace_rec(n, a0, tau, tn, mu);

        // update: one lane per changed cell; the per-mu header
        // (nu offset, nu count, dependency offset, dependency count) is one load
        const int4 h = fire ? __ldg(wt.hdr + mu) : make_int4(0, 0, 0, 0);
        int2 e = make_int2(0, 0);
        long long nv = 0;
        if (sl < h.y) {
            e = __ldg(wt.nuw + h.x + sl);  // (x byte offset, delta)
            nv = (long long)*(const int *)((const unsigned char *)xs + e.x) + e.y;
        }
        const bool ovf = ((__ballot_sync(kAll, nv > 0x7fffffffll) >> sb) & 0xffffu) != 0u;
        if (__any_sync(kAll, ovf)) {
            if (ovf) {  // a count would leave int32: freeze + fill
                for (; j < rp.j_stop; ++j) record(j);
                finish(CWC_TRAJ_OVERFLOW);
                fire = false;
            }
            __syncwarp();
        }
        if (fire && sl < h.y) *(int *)((unsigned char *)xs + e.x) = (int)nv;
        __syncwarp();

        // dependency-graph update: recompute a_m for m in D(mu) only.  Entries
        // carry byte offsets (slot, x_a, x_b, rate) and the owner lane; a_m =
        // k' RN(x_a (x_b - sub)) with k' = k / 2 for A + A (rates_h): equal
        // to k RN(binomial) bit for bit (power-of-two scaling commutes with RN)
        unsigned dirty = 0;
        if (fire) {
#pragma unroll 1
            for (int q = sl; q < h.w; q += 16) {
                const int4 d = __ldg(wt.depw16 + h.z + q);
                const int xa = *(const int *)((const unsigned char *)xs + d.y);
                const int xb = *(const int *)((const unsigned char *)xs + d.z) - (int)((unsigned)d.w >> 31);
                const double k = __ldg((const double *)((const unsigned char *)rates_h + (d.w & 0x3ffffff)));
                *(double *)((unsigned char *)as + d.x) = __dmul_rn(k, __dmul_rn(__int2double_rn(xa), __int2double_rn(xb)));
                dirty |= 1u << (((unsigned)d.w >> 26) & 31u);
            }
        }
        dirty = __reduce_or_sync(kAll, dirty << sb);
        __syncwarp();
        if ((dirty >> lane) & 1u) part = chunk_sum16<16>(as + sl * Bp, B);
        incl = seg_scan(part, sl, 16);
        a0 = __shfl_sync(kAll, incl, sb + 15);
        excl = __shfl_up_sync(kAll, incl, 1, 16);
        if (sl == 0) excl = 0.0;
        if (fire) {
            t = tn;
            ++kd;
            ++n;
        }
        asm volatile("bar.warp.sync -1;" ::: "memory");  // keep the warp converged
    }

    if (rp.stats_smem) {
        __syncthreads();
        const long long n16 = stat_bytes(rp.st, rp.cells_per_part) / 16;
        uint4 *dst = (uint4 *)((unsigned char *)rp.parts + (long long)blockIdx.x * stat_bytes(rp.st, rp.cells_per_part));
        const uint4 *src = (const uint4 *)smem;
        for (long long q = threadIdx.x; q < n16; q += blockDim.x) dst[q] = src[q];
    }
}

static inline int align16b(long long v) { return (int)((v + 15) & ~15ll); }

size_t warp2_smem_per_warp(const WarpTables &wt) {  // per segment: x, propensities, 32 draws
    return 2 * ((size_t)align16b(4ll * (wt.n_cells + 1)) + (size_t)8 * 16 * wt.Bp16 + (size_t)16 * 32);
}

cudaError_t launch_ssa_warp2(const RunParams &rp, const WarpTables &wt, int blocks, int warps_per_block,
                             size_t smem_bytes, cudaStream_t stream) {
    const long long stats_bytes = rp.stats_smem ? stat_bytes(rp.st, rp.cells_per_part) : 0;
    const int x_bytes = align16b(4ll * (wt.n_cells + 1));
    const int per_seg = (int)(warp2_smem_per_warp(wt) / 2);
    bool small = (size_t)smem_bytes * 8 <= (size_t)220 * 1024 && warps_per_block <= 4;
#ifdef CWC_DEBUG_KNOBS
    if (const char *e = std::getenv("CWC_WARP2_MINB")) small = std::atoi(e) == 8 && small;  // experiment switch
#endif
    auto k = (rp.n_trace > 0) ? (small ? ssa_warp2_kernel<8, true> : ssa_warp2_kernel<6, true>)
                              : (small ? ssa_warp2_kernel<8, false> : ssa_warp2_kernel<6, false>);
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_bytes);
    if (e != cudaSuccess) return e;
    k<<<blocks, warps_per_block * 32, smem_bytes, stream>>>(rp, wt, stats_bytes, per_seg, x_bytes);
    return cudaGetLastError();
}

}  // namespace cwc
