// dyn_ssa.cu -- SSA kernel of the dynamic-topology CWC path (SURVEY 8(f)
// NEXT-4; include/cwc_dyn.h; DESIGN.md section 2 reading 14 = D1-D4).
//
// One warp per trajectory (persistent warps taking trajectory ids from a
// counter, on-demand dispatch as P:741-762).  The term lives in the warp's
// shared memory as an array of compartment slots IN PREORDER (slot 0 = the
// top level): label, depth, wrap [A] and content [A] counts, double-buffered
// so that a structural rewrite builds the new term beside the old one (and a
// firing that would overflow or outgrow the capacity leaves the old term
// intact).  Lane l owns slots l and l + 32.
//
// Match (D1): the entries of rule r are laid out at 64 positions:
//   - a rule without a child pattern: position = context slot (preorder);
//   - a rule with a child pattern: position = the child's rank in
//     "corder" = all non-top slots sorted by (parent slot, slot) -- contexts
//     in preorder, children in list order, exactly the oracle's entry order;
// positions that are not entries hold 0 (adding +0 changes no sum and a
// zero entry is never selected).  Lane l evaluates positions 2l, 2l+1:
// rate = k RN(h), h the exact int64 product of the pattern's binomials.
// Sums: per rule, lane pair sums and a Kogge-Stone shuffle scan (lane
// prefixes kept in shared memory, the rule total in lane r's register);
// a0 = the Kogge-Stone scan of the rule totals.  This summation order
// differs from the oracle's left-to-right sum (the warp-path class of
// a0 within a few ulps); every sum is a deterministic
// function of the current term, so results do not depend on history or
// launch shape.
// Selection (D2): ballot over the rule prefixes, then over the lane prefixes
// of that rule, then the pair.
// Update (D3): non-structural rules (X kept, nothing released, the matched
// child rewritten in place with its label) add their dense net-change rows
// to the context (and the child) and re-evaluate only the rules whose
// patterns read a changed (label, side, atom); structural rules rebuild the
// context's subtree from segments of the old buffer (copies with a depth
// shift, new compartments from the constructors) into the other buffer,
// recompute parents and corder from the depth masks, and re-evaluate every
// rule.
#include <cuda_runtime.h>

#include "device_common.cuh"
#include "dyn_internal.h"

namespace cwc {
namespace dyn {

namespace {

constexpr unsigned FULL = 0xffffffffu;
constexpr long long I32MAX = 2147483647ll;

// One term buffer: wrap / content [A][64] int32, label / depth [64] int8.
struct Term {
    int *wrap, *cont;
    signed char *label, *depth;
};

struct Warp {
    double *ax;             // [R][32] first entry of each lane pair
    double *pre;            // [R][32] lane prefixes
    unsigned *xm, *ym;      // [R] positive-entry masks of the pair's first / second entry
    unsigned char *tbase;  // buffer b at tbase + b * tbytes (computed, never an indexed
    unsigned tbytes, abytes;  // pointer array: that would live in local memory)
    int *nchild;
    int4 *seg;
    unsigned long long *dmask;
    unsigned char *parent, *corder;
    // per entry position (rebuilt with the structure): x = label of slot pos
    // (context rules) | label of the child at rank pos << 8 | label of its
    // parent << 16 (0xff: no such slot / rank), y = child slot | parent << 8
    uint2 *pinfo;
};

__device__ __forceinline__ Warp warp_view(unsigned char *base, int A, int R) {
    Warp w;
    w.ax = (double *)(base + dyn_ax_off());
    w.pre = (double *)(base + dyn_pre_off(R));
    w.xm = (unsigned *)(base + dyn_mask_off(R));
    w.ym = w.xm + R;
    w.tbase = base + dyn_term_off(R);
    w.tbytes = (unsigned)dyn_term_bytes(A);
    w.abytes = (unsigned)A * kSlots * 4;
    unsigned char *m = base + dyn_misc_off(A, R);
    w.nchild = (int *)m;
    w.seg = (int4 *)(m + kSlots * 4);
    w.dmask = (unsigned long long *)(m + kSlots * 4 + kSegs * 16);
    w.parent = m + kSlots * 4 + kSegs * 16 + kLevels * 8;
    w.corder = w.parent + kSlots;
    w.pinfo = (uint2 *)(w.corder + kSlots);
    return w;
}

__device__ __forceinline__ Term tv(const Warp &w, int b) {
    unsigned char *q = w.tbase + (unsigned)b * w.tbytes;
    Term t;
    t.wrap = (int *)q;
    t.cont = (int *)(q + w.abytes);
    t.label = (signed char *)(q + 2 * w.abytes);
    t.depth = t.label + kSlots;
    return t;
}

__device__ __forceinline__ double ks_scan(double v, int lane) {
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const double y = __shfl_up_sync(FULL, v, off);
        if (lane >= off) v = __dadd_rn(v, y);
    }
    return v;
}

__device__ __forceinline__ int ks_scan_int(int v, int lane) {
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const int y = __shfl_up_sync(FULL, v, off);
        if (lane >= off) v += y;
    }
    return v;
}

__device__ __forceinline__ unsigned long long ballot64(bool lo, bool hi) {
    return (unsigned long long)__ballot_sync(FULL, lo) | ((unsigned long long)__ballot_sync(FULL, hi) << 32);
}

// Depth masks, parents and corder of buffer b with n slots (D1 order).
__device__ void refresh_structure(const Warp &w, int b, int n, int lane) {
    const int s0 = lane, s1 = lane + 32;
    const int d0 = s0 < n ? (int)tv(w, b).depth[s0] : -1;
    const int d1 = s1 < n ? (int)tv(w, b).depth[s1] : -1;
#pragma unroll
    for (int L = 0; L < kLevels; ++L) {
        const unsigned long long m = ballot64(d0 == L, d1 == L);
        if (lane == 0) w.dmask[L] = m;
    }
    w.nchild[s0] = 0;
    w.nchild[s1] = 0;
    w.corder[s0] = 0;
    w.corder[s1] = 0;
    __syncwarp();
    int par[2] = {-1, -1};
#pragma unroll
    for (int k = 0; k < 2; ++k) {
        const int s = k ? s1 : s0, d = k ? d1 : d0;
        if (s >= 1 && d >= 1) {
            const unsigned long long m = w.dmask[d - 1] & ((1ull << s) - 1ull);
            par[k] = 63 - __clzll((long long)m);
            atomicAdd(&w.nchild[par[k]], 1);
        }
    }
    __syncwarp();
    // exclusive scan of the children counts over parents 0 .. 63 (pairs per lane)
    const int c0 = w.nchild[2 * lane], c1 = w.nchild[2 * lane + 1];
    const int incl = ks_scan_int(c0 + c1, lane);
    __syncwarp();
    w.nchild[2 * lane] = incl - c0 - c1;
    w.nchild[2 * lane + 1] = incl - c1;
    __syncwarp();
#pragma unroll
    for (int k = 0; k < 2; ++k) {
        const int s = k ? s1 : s0, d = k ? d1 : d0;
        if (par[k] >= 0) {
            const unsigned long long between = w.dmask[d] & ((1ull << s) - 1ull) & ~((2ull << par[k]) - 1ull);
            const int rank = w.nchild[par[k]] + __popcll(between);
            w.corder[rank] = (unsigned char)s;
            w.parent[s] = (unsigned char)par[k];
        } else {
            w.parent[s] = 0;
        }
    }
    __syncwarp();
    const signed char *lab = tv(w, b).label;
#pragma unroll
    for (int k = 0; k < 2; ++k) {
        const int pos = lane + 32 * k;
        const unsigned lctx = pos < n ? (unsigned)(unsigned char)lab[pos] : 0xffu;
        unsigned ls = 0xffu, lp = 0xffu, sp = 0u;
        if (pos < n - 1) {
            const int s = w.corder[pos], p = w.parent[s];
            ls = (unsigned)(unsigned char)lab[s];
            lp = (unsigned)(unsigned char)lab[p];
            sp = (unsigned)s | ((unsigned)p << 8);
        }
        w.pinfo[pos] = make_uint2(lctx | (ls << 8) | (lp << 16), sp);
    }
    __syncwarp();
}

// Factor of h: binomial(x, mult) for mult 1 or 2 (reaction order <= 2).
__device__ __forceinline__ long long binom12(int x, int mult) {
    return mult == 2 ? (((long long)x * (long long)(x - 1)) >> 1) : (long long)x;
}

// Entries of rule r at positions 2 lane, 2 lane + 1 (D1): rate k RN(h).
__device__ __forceinline__ void rule_entries(const Warp &w, const DynTables &T, int b, int n, int r, int lane,
                                             double &e0, double &e1) {
    const int4 d = __ldg(&T.rule[r]);
    const double k = __ldg(&T.rate[r]);
    const int L = rd_label(d.x), Lc = rd_comp(d.x), nf = rd_nfac(d.x);
    const Term t = tv(w, b);
    // factor i reads row (side, atom) of the context (p) or the child (s)
    const int f0s = d.y & 0xf, f1s = d.z & 0xf;
    const int *row0 = (f0s == CWC_DYN_WRAP ? t.wrap : t.cont) + ((d.y >> 4) & 0xff) * kSlots;
    const int *row1 = (f1s == CWC_DYN_WRAP ? t.wrap : t.cont) + ((d.z >> 4) & 0xff) * kSlots;
    const int m0 = (d.y >> 12) & 0xf, m1 = (d.z >> 12) & 0xf;
    // narrow layout (n <= 32 slots: every rule has <= 32 positions): one
    // position per lane, pos = lane, the pair's second entry 0; wide: two
    auto entry = [&](int pos) -> double {
        // one structure word per position (pinfo: labels and slots, 0xff
        // labels where there is no entry)
        const uint2 pi = w.pinfo[pos];
        int s, p;
        bool valid;
        if (Lc < 0) {
            s = pos;
            p = pos;
            valid = (pi.x & 0xffu) == (unsigned)L;
        } else {
            s = (int)(pi.y & 0xffu);
            p = (int)((pi.y >> 8) & 0xffu);
            valid = ((pi.x >> 8) & 0xffffu) == ((unsigned)Lc | ((unsigned)L << 8));
        }
        long long h = 1;
        if (nf >= 1) h = binom12(row0[f0s == CWC_DYN_CTX ? p : s], m0);
        if (nf >= 2) h *= binom12(row1[f1s == CWC_DYN_CTX ? p : s], m1);
        return valid ? __dmul_rn(k, __ll2double_rn(h)) : 0.0;
    };
    if (n <= 32) {
        e0 = entry(lane);
        e1 = 0.0;
    } else {
        e0 = entry(2 * lane);
        e1 = entry(2 * lane + 1);
    }
}

// The single entry (the top level) of a singleton rule, the same value in
// every lane (broadcast loads).
__device__ __forceinline__ double singleton_entry(const Warp &w, const DynTables &T, int b, int r) {
    const int4 d = __ldg(&T.rule[r]);
    const double k = __ldg(&T.rate[r]);
    const int nf = rd_nfac(d.x);
    const Term t = tv(w, b);
    long long h = 1;
    if (nf >= 1) h = binom12(t.cont[((d.y >> 4) & 0xff) * kSlots], (d.y >> 12) & 0xf);
    if (nf >= 2) h *= binom12(t.cont[((d.z >> 4) & 0xff) * kSlots], (d.z >> 12) & 0xf);
    return __dmul_rn(k, __ll2double_rn(h));
}

__device__ __forceinline__ void store_rule(const Warp &w, int r, int lane, double x, double y, double S) {
    w.ax[r * 32 + lane] = x;
    w.pre[r * 32 + lane] = S;
    const unsigned mx = __ballot_sync(FULL, x > 0.0), my = __ballot_sync(FULL, y > 0.0);
    if (lane == 0) {
        w.xm[r] = mx;
        w.ym[r] = my;
    }
}

// Re-evaluate rules r1 and r2 (r2 < 0: none) -- entries, lane pair sums, the
// lane prefixes (two independent shuffle scans interleaved, so two rules
// cost one scan's latency) -- and store them; lane r receives rule r's total
// in Tr.
__device__ __forceinline__ void eval_rules(const Warp &w, const DynTables &T, int b, int n, int r1, int r2, int lane,
                                           double &Tr) {
    double a0, a1, b0 = 0.0, b1 = 0.0;
    rule_entries(w, T, b, n, r1, lane, a0, a1);
    if (r2 >= 0) rule_entries(w, T, b, n, r2, lane, b0, b1);
    double u = __dadd_rn(a0, a1), v = __dadd_rn(b0, b1);
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const double yu = __shfl_up_sync(FULL, u, off);
        const double yv = __shfl_up_sync(FULL, v, off);
        if (lane >= off) {
            u = __dadd_rn(u, yu);
            v = __dadd_rn(v, yv);
        }
    }
    store_rule(w, r1, lane, a0, a1, u);
    if (r2 >= 0) store_rule(w, r2, lane, b0, b1, v);
    const double t1 = __shfl_sync(FULL, u, 31), t2 = __shfl_sync(FULL, v, 31);
    if (lane == r1) Tr = t1;
    if (lane == r2) Tr = t2;
}

// Re-evaluate every rule in the mask: singletons directly (no scan: their
// lane prefixes all equal the one entry), the others two at a time.
__device__ __forceinline__ void eval_mask(const Warp &w, const DynTables &T, int b, int n, unsigned dirty,
                                          unsigned single, int lane, double &Tr) {
    unsigned sd = dirty & single;
    dirty &= ~single;
    while (sd) {
        const int r = __ffs(sd) - 1;
        sd &= sd - 1;
        const double e = singleton_entry(w, T, b, r);
        w.ax[r * 32 + lane] = lane == 0 ? e : 0.0;
        w.pre[r * 32 + lane] = e;
        if (lane == 0) {
            w.xm[r] = e > 0.0 ? 1u : 0u;
            w.ym[r] = 0u;
        }
        if (lane == r) Tr = e;
    }
    while (dirty) {
        const int r1 = __ffs(dirty) - 1;
        dirty &= dirty - 1;
        int r2 = -1;
        if (dirty) {
            r2 = __ffs(dirty) - 1;
            dirty &= dirty - 1;
        }
        eval_rules(w, T, b, n, r1, r2, lane, Tr);
    }
    __syncwarp();
}

// Observable values of buffer b (D4): lane o returns observable o.
__device__ long long observe(const Warp &w, const DynTables &T, int b, int lane) {
    long long mine = 0;
    const signed char *lab = tv(w, b).label;
    const int l0 = lab[lane], l1 = lab[lane + 32];
    for (int o = 0; o < T.O; ++o) {
        unsigned long long pv = 0;
        const int k0 = __ldg(&T.obs_ptr[o]), k1 = __ldg(&T.obs_ptr[o + 1]);
        for (int k = k0; k < k1; ++k) {
            const int4 key = __ldg(&T.obs_key[k]);
            const int *arr = key.x == CWC_DYN_OBS_WRAP ? tv(w, b).wrap : tv(w, b).cont;
            if (key.x == CWC_DYN_OBS_COUNT) {
                pv += (unsigned long long)(l0 == key.y) + (unsigned long long)(l1 == key.y);
            } else {
                if (l0 == key.y) pv += (unsigned long long)arr[key.z * kSlots + lane];
                if (l1 == key.y) pv += (unsigned long long)arr[key.z * kSlots + lane + 32];
            }
        }
        const unsigned lo = __reduce_add_sync(FULL, (unsigned)(pv & 0xffffffull));
        const unsigned hi = __reduce_add_sync(FULL, (unsigned)(pv >> 24));
        const long long v = (long long)lo + ((long long)hi << 24);
        if (lane == o) mine = v;
    }
    return mine;
}

__device__ __forceinline__ void record(const DynParams &P, const StatAcc &acc, int O, long long g, int j,
                                       long long v, int lane) {
    if (lane < O) {
        stat_record(acc, (long long)j * O + lane, v);
        if (P.out_traj) P.out_traj[((long long)g * (P.J + 1) + j) * O + lane] = v;
    }
}

}  // namespace

__global__ void __launch_bounds__(256) dyn_ssa_kernel(const DynParams P, const DynTables T) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int A = T.A, R = T.R, O = T.O;
    const Warp w = warp_view(smem + (size_t)wid * dyn_smem_per_warp(A, R), A, R);
    const StatAcc acc = stat_view(P.part, P.cells, P.st);
    const int J = P.J;
    const unsigned all_rules = R >= 32 ? FULL : ((1u << R) - 1u);
    const unsigned single = __ballot_sync(FULL, lane < R && rd_singleton(__ldg(&T.rule[lane < R ? lane : 0]).x)) & all_rules;

    for (;;) {
        long long g = 0;
        if (lane == 0) g = (long long)atomicAdd(P.next_traj, 1ull);
        g = __shfl_sync(FULL, g, 0);
        if (g >= P.G) break;
        const unsigned long long gkey = (unsigned long long)(P.r_off + g);

        // ---- a2: initial term into buffer 0 ----
        int b = 0, n = T.n0;
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            const int s = lane + 32 * k;
            const bool in = s < n;
            tv(w, 0).label[s] = in ? (signed char)__ldg(&T.init_label[s]) : (signed char)-1;
            tv(w, 0).depth[s] = in ? (signed char)__ldg(&T.init_depth[s]) : (signed char)0;
            for (int a = 0; a < A; ++a) {
                tv(w, 0).wrap[a * kSlots + s] = in ? __ldg(&T.init_wrap[s * A + a]) : 0;
                tv(w, 0).cont[a * kSlots + s] = in ? __ldg(&T.init_cont[s * A + a]) : 0;
            }
        }
        __syncwarp();
        refresh_structure(w, 0, n, lane);
        double Tr = 0.0;  // lane r: total of rule r
        eval_mask(w, T, 0, n, all_rules, single, lane, Tr);

        double t = 0.0;
        long long nfire = 0, firings = 0;
        long long n0 = -64;
        double Ek = 0.0, Uk = 0.0;
        int j = 0, status = CWC_TRAJ_DONE;
        for (;;) {
            const double Q = ks_scan(Tr, lane);
            const double a0 = __shfl_sync(FULL, Q, 31);
            if (!(a0 > 0.0)) {  // a10: stall, no RNG drawn
                status = CWC_TRAJ_STALLED;
                break;
            }
            // a5: one Philox block per iteration, 32 computed at once (one per lane)
            if (nfire - n0 >= 32) {
                n0 = nfire;
                const uint4 wd = philox_block(P.seed, gkey, (unsigned long long)(n0 + lane));
                block_to_draws(wd, Ek, Uk);
            }
            const int di = (int)(nfire - n0);
            const double E = __shfl_sync(FULL, Ek, di), u2 = __shfl_sync(FULL, Uk, di);
            ++nfire;
            // a6
            const double tau = div_fast_ok(E, a0) ? div_fast(E, a0) : __ddiv_rn(E, a0);
            const double tn = __dadd_rn(t, tau);
            // a7: samples crossed take the pre-event term
            if (j <= J && __dmul_rn((double)j, P.dt) <= tn) {
                const long long v = observe(w, T, b, lane);
                while (j <= J && __dmul_rn((double)j, P.dt) <= tn) {
                    record(P, acc, O, g, j, v, lane);
                    ++j;
                }
            }
            if (j > J) break;  // drawn, not applied, not counted
            // a8: selection (D2)
            const double target = __dmul_rn(u2, a0);
            const unsigned mr = __ballot_sync(FULL, lane < R && target < Q);
            int rs;
            bool fb = false;
            if (mr) {
                rs = __ffs(mr) - 1;
            } else {
                rs = 31 - __clz(__ballot_sync(FULL, lane < R && Tr > 0.0));
                fb = true;
            }
            const double Qprev = __shfl_sync(FULL, Q, rs > 0 ? rs - 1 : 0);
            const double Eb = rs > 0 ? Qprev : 0.0;
            const double S = w.pre[rs * 32 + lane];
            const double Sprev = __shfl_up_sync(FULL, S, 1);
            const unsigned ml = fb ? 0u : __ballot_sync(FULL, __dadd_rn(Eb, S) > target);
            int ls;
            bool fbl = false;
            if (ml) {
                ls = __ffs(ml) - 1;
            } else {
                ls = 31 - __clz(__ballot_sync(FULL, lane == 0 ? S > 0.0 : S > Sprev));
                fbl = true;
            }
            const double px = w.ax[rs * 32 + ls];
            const bool ypos = (w.ym[rs] >> ls) & 1u, xpos = (w.xm[rs] >> ls) & 1u;
            int pos;
            if (n <= 32) {  // narrow layout: position = lane
                pos = ls;
            } else if (fbl) {
                pos = ypos ? 2 * ls + 1 : 2 * ls;
            } else {
                const double base = __dadd_rn(Eb, ls > 0 ? w.pre[rs * 32 + ls - 1] : 0.0);
                pos = (!ypos || (xpos && target < __dadd_rn(base, px))) ? 2 * ls : 2 * ls + 1;
            }
            const int4 rd = __ldg(&T.rule[rs]);
            int p, s;
            if (rd_comp(rd.x) < 0) {
                p = pos;
                s = -1;
            } else {
                s = (int)w.corder[pos];
                p = (int)w.parent[s];
            }
            // a9: update (D3)
            unsigned dirty;
            if (!rd_structural(rd.x)) {
                bool ovf = false;
                long long vc = 0, vw = 0, vt = 0;
                if (lane < A) {
                    vc = (long long)tv(w, b).cont[lane * kSlots + p] + __ldg(&T.dctx[rs * A + lane]);
                    ovf = vc > I32MAX;
                    if (s >= 0) {
                        vw = (long long)tv(w, b).wrap[lane * kSlots + s] + __ldg(&T.dwrap[rs * A + lane]);
                        vt = (long long)tv(w, b).cont[lane * kSlots + s] + __ldg(&T.dcont[rs * A + lane]);
                        ovf = ovf || vw > I32MAX || vt > I32MAX;
                    }
                }
                if (__any_sync(FULL, ovf)) {
                    status = CWC_TRAJ_OVERFLOW;
                    break;
                }
                if (lane < A) {
                    tv(w, b).cont[lane * kSlots + p] = (int)vc;
                    if (s >= 0) {
                        tv(w, b).wrap[lane * kSlots + s] = (int)vw;
                        tv(w, b).cont[lane * kSlots + s] = (int)vt;
                    }
                }
                __syncwarp();
                dirty = (unsigned)rd.w;
            } else {
                // ---- structural rewrite of p's subtree into buffer nb ----
                const int nb = b ^ 1;
                const int flags = rd_flags(rd.x);
                const bool X = flags & CWC_DYN_KEEP_X, RW = flags & CWC_DYN_RELEASE_W, RY = flags & CWC_DYN_RELEASE_Y;
                const int dp = (int)tv(w, b).depth[p];
                const unsigned long long live = n >= 64 ? ~0ull : ((1ull << n) - 1ull);
                unsigned long long le = 0;  // slots at depth <= dp
                for (int L = 0; L <= dp; ++L) le |= w.dmask[L];
                const unsigned long long after = le & live & ~((2ull << p) - 1ull);  // (2 << 63) == 0: none
                const int p_end = after ? __ffsll((long long)after) - 1 : n;
                int s_end = 0;
                if (s >= 0) {
                    unsigned long long m = (le | w.dmask[dp + 1]) & live & (s == 63 ? 0ull : ~((2ull << s) - 1ull));
                    s_end = m ? __ffsll((long long)m) - 1 : n;
                }
                const int4 ch = __ldg(&T.ctor_hdr[rs]);
                // segments: x dst start, y src start (COPY) or -1 - ctor (NEW), z length, w depth shift
                int nseg = 0, dst = 0;
                auto add = [&](int src, int len, int dsh) {
                    if (len <= 0) return;
                    if (lane == 0) w.seg[nseg] = make_int4(dst, src, len, dsh);
                    ++nseg;
                    dst += len;
                };
                add(0, p + 1, 0);
                const int ycnt = s >= 0 ? s_end - s - 1 : 0;
                if (X) {
                    if (s < 0) {
                        add(p + 1, p_end - p - 1, 0);
                    } else {
                        add(p + 1, s - p - 1, 0);
                        if (ch.z >= 0) {
                            add(-1 - ch.z, 1, 0);
                            add(s + 1, ycnt, 0);
                        }
                        add(s_end, p_end - s_end, 0);
                    }
                } else if (ch.z >= 0) {
                    add(-1 - ch.z, 1, 0);
                    add(s + 1, ycnt, 0);
                }
                if (RY && s >= 0) add(s + 1, ycnt, -1);
                for (int c = ch.x; c < ch.x + ch.y; ++c) {
                    if (c == ch.z) continue;
                    add(-1 - c, 1, 0);
                    if ((__ldg(&T.ctor[c]).y & CWC_DYN_CTOR_Y) && s >= 0) add(s + 1, ycnt, 0);
                }
                add(p_end, n - p_end, 0);
                const int n_new = dst;
                bool has_new = ch.y > 0;
                if (n_new > P.cap || (has_new && dp + 1 > CWC_DYN_MAX_DEPTH)) {
                    status = CWC_TRAJ_CAPACITY;
                    break;
                }
                __syncwarp();
                bool ovf = false;
                const int *lhs = T.lhs + (size_t)rs * 3 * A;
#pragma unroll
                for (int k = 0; k < 2; ++k) {
                    const int d = lane + 32 * k;
                    if (d < n_new) {
                        int4 sg = make_int4(0, 0, 0, 0);
                        for (int q = 0; q < nseg; ++q) {
                            const int4 x = w.seg[q];
                            if (d >= x.x && d < x.x + x.z) sg = x;
                        }
                        if (sg.y >= 0) {
                            const int src = sg.y + (d - sg.x);
                            tv(w, nb).label[d] = tv(w, b).label[src];
                            tv(w, nb).depth[d] = (signed char)((int)tv(w, b).depth[src] + sg.w);
                            for (int a = 0; a < A; ++a) {
                                tv(w, nb).wrap[a * kSlots + d] = tv(w, b).wrap[a * kSlots + src];
                                long long v = tv(w, b).cont[a * kSlots + src];
                                if (src == p) {
                                    v = (X ? v - __ldg(&lhs[a]) : 0ll) + __ldg(&T.rhs[rs * A + a]);
                                    if (RW) v += (long long)tv(w, b).wrap[a * kSlots + s] - __ldg(&lhs[A + a]);
                                    if (RY) v += (long long)tv(w, b).cont[a * kSlots + s] - __ldg(&lhs[2 * A + a]);
                                    ovf = ovf || v > I32MAX;
                                }
                                tv(w, nb).cont[a * kSlots + d] = (int)v;
                            }
                        } else {
                            const int c = -1 - sg.y;
                            const int4 cd = __ldg(&T.ctor[c]);
                            tv(w, nb).label[d] = (signed char)cd.x;
                            tv(w, nb).depth[d] = (signed char)(dp + 1);
                            for (int a = 0; a < A; ++a) {
                                long long vw = __ldg(&T.ctor_atoms[(size_t)c * 2 * A + a]);
                                long long vc = __ldg(&T.ctor_atoms[(size_t)c * 2 * A + A + a]);
                                if (cd.y & CWC_DYN_CTOR_W) vw += (long long)tv(w, b).wrap[a * kSlots + s] - __ldg(&lhs[A + a]);
                                if (cd.y & CWC_DYN_CTOR_Y) vc += (long long)tv(w, b).cont[a * kSlots + s] - __ldg(&lhs[2 * A + a]);
                                ovf = ovf || vw > I32MAX || vc > I32MAX;
                                tv(w, nb).wrap[a * kSlots + d] = (int)vw;
                                tv(w, nb).cont[a * kSlots + d] = (int)vc;
                            }
                        }
                    } else {
                        tv(w, nb).label[d] = (signed char)-1;
                        tv(w, nb).depth[d] = 0;
                    }
                }
                if (__any_sync(FULL, ovf)) {
                    status = CWC_TRAJ_OVERFLOW;
                    break;
                }
                __syncwarp();
                b = nb;
                n = n_new;
                refresh_structure(w, b, n, lane);
                dirty = all_rules;
            }
            t = tn;
            ++firings;
            // a3/a4: re-evaluate the rules the firing may have changed
            eval_mask(w, T, b, n, dirty, single, lane, Tr);
        }
        if (j <= J) {  // stall / overflow / capacity: the remaining samples take the frozen term
            const long long v = observe(w, T, b, lane);
            for (; j <= J; ++j) record(P, acc, O, g, j, v, lane);
        }
        if (lane == 0) {
            if (P.out_firings) P.out_firings[g] = firings;
            if (P.out_status) P.out_status[g] = status;
        }
        __syncwarp();
    }
}

cudaError_t launch_dyn_ssa(const DynParams &dp, const DynTables &dt, int blocks, int warps_per_block, size_t smem,
                           cudaStream_t stream) {
    // the dynamic shared-memory attribute is set by the planner (dyn_api.cpp plan)
    dyn_ssa_kernel<<<blocks, 32 * warps_per_block, smem, stream>>>(dp, dt);
    return cudaGetLastError();
}

const void *dyn_kernel_fn() { return (const void *)dyn_ssa_kernel; }

}  // namespace dyn
}  // namespace cwc
