"""Divergence tracer (BASELINE north_star: "every divergence must be logged
and traced to a last-ulp difference in fp64 log or propensity sums").

For a trajectory whose GPU samples differ from the oracle's, both sides are
re-run with their per-firing trace -- (n, a0, tau, t', mu) per drawn Philox
block -- by the SAME kernel variant and launch plan that produced the dump
(the traced kernels are the product kernels with trace writes compiled in;
their fast paths included).  The first differing record i is then
classified, and each class is VERIFIED from first principles, not assumed:

  "a0-sum-order"  a0 differs.  The propensities before firing i are rebuilt
                  independently (the oracle's state x_i = x0 + sum of nu over
                  its first i firings, oracle.propensities); the rebuild must
                  reproduce the oracle's own a0 bit for bit (left-to-right
                  sum), and BOTH a0 values must lie within the forward error
                  bound of their summation tree around the exact (rational)
                  sum S: |a0 - S| <= gamma_d S, d = M - 1 for the oracle's
                  sequential sum and d = B - 1 + log2(lanes) for the warp
                  kernels' lane-chunk sums + shuffle tree (gamma_d = d u /
                  (1 - d u), u = 2^-53).  Thread kernels sum like the oracle,
                  so any a0 difference there is a BUG.
  "log-ulp"       a0 equal, tau differs: E = -log u1 of block (g, n) is read
                  from the device draw hook (the kernels' own function) and
                  from the oracle (glibc); both must be within 1 ulp of the
                  exact -ln u1 (mpmath), and each tau must be exactly its
                  E / a0 (one IEEE division).
  "select-order"  a0, tau, t' equal, mu differs (warp kernels only): the
                  target u2 a0 must lie within the two summation trees'
                  error bounds of the exact prefix sum at the boundary
                  between the two choices.
  "BUG"           anything else: a different n, t' != t + tau, an unverified
                  class, identical traces for a trajectory whose samples
                  differ, or a first sample mismatch EARLIER than the first
                  differing firing (the divergence must explain it: samples
                  at t_j <= min(t'_gpu, t'_ora) of record i take the common
                  pre-event state).
"""
from __future__ import annotations

import math
from fractions import Fraction

import numpy as np

import oracle

U = 2.0 ** -53


def ulp_diff(a, b):
    if a == b:
        return 0
    if not (math.isfinite(a) and math.isfinite(b)) or (a < 0) != (b < 0):
        return 1 << 62
    ia = np.frombuffer(np.float64(a).tobytes(), dtype=np.int64)[0]
    ib = np.frombuffer(np.float64(b).tobytes(), dtype=np.int64)[0]
    return abs(int(ia) - int(ib))


def gamma(d):
    return d * U / (1.0 - d * U)


class KernelGeom:
    """Summation geometry of the kernel that ran: thread kernels sum a0 left
    to right like the oracle; warp kernels sum lane chunks of B entries and
    combine the lanes with a shuffle tree."""

    def __init__(self, warp, lanes=32, M=1):
        self.warp = bool(warp)
        self.lanes = lanes
        self.B = max(1, -(-M // lanes))
        self.M = M

    @property
    def depth(self):  # additions on the longest leaf-to-root path (+1: the selection's carry add)
        if not self.warp:
            return max(self.M - 1, 0)
        return self.B - 1 + int(math.ceil(math.log2(self.lanes))) + 1


def geom_for(model, kernel_variant):
    """KernelGeom of the variant the planner launches (cwc_api.cpp plan_run)."""
    from paper_1010_2438_b200 import cwc
    M = model.info.n_reactions
    if kernel_variant in (cwc.CWC_KERNEL_THREAD, cwc.CWC_KERNEL_THREAD_WS):
        return KernelGeom(False, M=M)
    if kernel_variant == cwc.CWC_KERNEL_WARP:
        return KernelGeom(True, 32, M)
    if kernel_variant == cwc.CWC_KERNEL_WARP2:
        return KernelGeom(True, 16, M)
    if kernel_variant == cwc.CWC_KERNEL_WARP4:
        return KernelGeom(True, 8, M)  # 8-lane groups (same construction, B = M / 8)
    if kernel_variant == cwc.CWC_KERNEL_WARP8:
        # 4-lane groups: sub-chunks of 16 summed left to right, four sub-chunk
        # sums, a 4-lane shuffle tree -- within the chunk bound of B = M / 4
        return KernelGeom(True, 4, M)
    if model.info.path == cwc.CWC_PATH_THREAD:
        return KernelGeom(False, M=M)
    return KernelGeom(True, 16 if -(-M // 16) <= 16 else 32, M)


class OracleSide:
    """Independent rebuild of the oracle's state and propensities along its trace."""

    def __init__(self, desc, sweep, n_replicas, seed):
        self.fm = oracle.FlatModel(desc)
        self.rates = self.fm.rule_rates(sweep)
        self.R = n_replicas
        self.seed = seed
        self.nu = []
        for e in self.fm.entries:
            self.nu.append([(c, d) for (c, d) in e["nu"]])
        self.x0 = np.asarray(desc["init"], dtype=np.int64)

    def state_before(self, ora_trace, i):
        x = self.x0.copy()
        for k in range(i):
            mu = int(ora_trace[k][4])
            for c, d in self.nu[mu]:
                x[c] += d
        return x

    def propensities(self, g, x):
        return oracle.propensities(self.fm, x, self.rates[g // self.R])

    def uniforms(self, g, n):
        w = oracle.philox4x32_10([n & 0xFFFFFFFF, n >> 32, g & 0xFFFFFFFF, g >> 32],
                                 [self.seed & 0xFFFFFFFF, self.seed >> 32])
        return oracle.uniforms(w)


def _seq_sum(a):
    s = 0.0
    for i, v in enumerate(a):
        s = v if i == 0 else s + float(v)
    return s


def _within(val, exact, d):
    return abs(Fraction(val) - exact) <= Fraction(gamma(d)) * exact


def classify(gpu_trace, ora_trace, geom, side=None, g=None, draw_E=None, sample_mismatch_t=None):
    """First differing record and its verified class -> (category, index, detail).

    side: OracleSide (state rebuild); draw_E(g, n) -> the device's E;
    sample_mismatch_t: time t_j of the first differing sample (None: the
    samples agree)."""
    n = min(len(gpu_trace), len(ora_trace))
    first = None
    for i in range(n):
        if any(x != y for x, y in zip(gpu_trace[i], ora_trace[i])):
            first = i
            break
    if first is None:
        if len(gpu_trace) != len(ora_trace):
            return "BUG", n, "trace lengths %d vs %d" % (len(gpu_trace), len(ora_trace))
        if sample_mismatch_t is not None:
            return "BUG", -1, "identical traces but the samples differ"
        return "identical-trace", -1, ""
    i = first
    gr, orr = gpu_trace[i], ora_trace[i]
    t_div = min(gr[3], orr[3])
    if sample_mismatch_t is not None and sample_mismatch_t <= t_div:
        return "BUG", i, "first sample mismatch at t=%r precedes the divergence at t=%r" % (sample_mismatch_t, t_div)
    if gr[0] != orr[0]:
        return "BUG", i, "firing index differs"
    t_prev = gpu_trace[i - 1][3] if i > 0 else 0.0
    if i > 0 and gpu_trace[i - 1][3] != ora_trace[i - 1][3]:
        return "BUG", i, "previous t' differ"
    for rec in (gr, orr):  # t' = t + tau (the same t: records before i are identical)
        if rec[3] != t_prev + rec[2]:
            return "BUG", i, "t' != t + tau"
    if side is None:
        return "BUG", i, "unverified (no oracle side)"
    nfire = int(gr[0])
    x = side.state_before(ora_trace, i)
    a = side.propensities(g, x)
    if _seq_sum(a) != orr[1]:
        return "BUG", i, "state rebuild does not reproduce the oracle's a0"
    S = sum((Fraction(float(v)) for v in a), Fraction(0))
    if gr[1] != orr[1]:
        if not geom.warp:
            return "BUG", i, "a0 differs on a thread kernel (same summation order as the oracle)"
        ok = _within(gr[1], S, geom.depth) and _within(orr[1], S, max(geom.M - 1, 0))
        return ("a0-sum-order" if ok else "BUG"), i, "a0 %r vs %r (%d ulp; exact %r)" % (
            gr[1], orr[1], ulp_diff(gr[1], orr[1]), float(S))
    if gr[2] != orr[2]:
        import mpmath
        mpmath.mp.prec = 200
        u1, _ = side.uniforms(g, nfire)
        E_ora = oracle.tau(u1, 1.0)
        E_gpu = draw_E(g, nfire) if draw_E is not None else None
        if E_gpu is None:
            return "BUG", i, "tau differs, device E unavailable"
        ex = -mpmath.log(mpmath.mpf(u1))
        ulp = mpmath.mpf(math.ulp(float(ex)))
        ok = (abs(mpmath.mpf(E_gpu) - ex) <= ulp and abs(mpmath.mpf(E_ora) - ex) <= ulp and
              gr[2] == E_gpu / gr[1] and orr[2] == E_ora / orr[1] and E_gpu != E_ora)
        return ("log-ulp" if ok else "BUG"), i, "tau %r vs %r; E %r vs %r" % (gr[2], orr[2], E_gpu, E_ora)
    if gr[4] != orr[4]:
        if not geom.warp:
            return "BUG", i, "mu differs on a thread kernel"
        _, u2 = side.uniforms(g, nfire)
        target = Fraction(u2 * gr[1])
        b = int(min(gr[4], orr[4]))
        if b < 0:
            return "BUG", i, "mu %r vs %r" % (gr[4], orr[4])
        P = sum((Fraction(float(v)) for v in a[: b + 1]), Fraction(0))
        tol = Fraction(gamma(geom.depth) + gamma(max(geom.M - 1, 0))) * S
        ok = abs(target - P) <= tol
        return ("select-order" if ok else "BUG"), i, "mu %r vs %r; |target - P| = %r of S %r" % (
            gr[4], orr[4], float(abs(target - P)), float(S))
    return "BUG", i, "records differ in no classified field"


def first_sample_mismatch_t(gpu_row, ora_row, dt):
    """t_j of the first sample whose observables differ (None if none)."""
    d = np.nonzero((np.asarray(gpu_row) != np.asarray(ora_row)).any(axis=-1))[0]
    return None if len(d) == 0 else float(d[0]) * dt


def trace_mismatches(model, desc, sweep, cfg, g_list, warp_path=None, force_path=None, cap=2_000_000,
                     kernel=None, gpu_rows=None, ora_rows=None, **plan):
    """Trace every g in g_list with the kernel variant the run used.
    Returns a list of (g, category, record index, detail)."""
    import torch

    from paper_1010_2438_b200 import cwc
    kern = cwc.CWC_KERNEL_AUTO if kernel is None else kernel
    fp = cwc.CWC_PATH_AUTO if force_path is None else force_path
    # the geometry of the kernel the planner actually launches for this run
    popts = cwc.cwc_sim_opts()
    popts.force_path = fp
    popts.kernel = kern
    for k, v in plan.items():
        setattr(popts, k, v)
    planned = cwc.cwc_plan(model, cfg["n_replicas"], sweep, cfg["t_end"], cfg["sample_dt"], popts).kernel
    geom = geom_for(model, planned)
    if warp_path is not None and fp != cwc.CWC_PATH_AUTO:
        geom = KernelGeom(fp == cwc.CWC_PATH_WARP, geom.lanes if geom.warp else 32, model.info.n_reactions)
    side = OracleSide(desc, sweep, cfg["n_replicas"], cfg["seed"])

    def draw_E(g, n):
        gg = torch.tensor([g], dtype=torch.int64, device="cuda")
        nn = torch.tensor([n], dtype=torch.int64, device="cuda")
        E = torch.zeros(1, dtype=torch.float64, device="cuda")
        u2 = torch.zeros(1, dtype=torch.float64, device="cuda")
        cwc.cwc_draws(cfg["seed"], gg, nn, E, u2, torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        return float(E.item())

    out = []
    for k, g in enumerate(g_list):
        gpu = cwc.simulate(model, cfg["n_replicas"], cfg["t_end"], cfg["sample_dt"], cfg["seed"], sweep=sweep,
                           want_firings=True, trace_g=[int(g)], trace_cap=cap, force_path=fp, kernel=kern, **plan)
        torch.cuda.synchronize()
        ln = int(gpu["trace_len"][0].item())
        gt = gpu["trace"][0, :ln].cpu().numpy()
        ora = oracle.simulate(desc, cfg["n_replicas"], cfg["t_end"], cfg["sample_dt"], cfg["seed"], sweep=sweep,
                              g_list=[int(g)], want_traj=True, want_stats=False, trace_g=int(g), trace_cap=cap)
        mt = None
        if gpu_rows is not None:
            mt = first_sample_mismatch_t(gpu_rows[k], ora["traj"][0], cfg["sample_dt"])
        cat, idx, detail = classify([tuple(r) for r in gt], [tuple(r) for r in ora["trace"]], geom, side, int(g),
                                    draw_E, mt)
        out.append((int(g), cat, idx, detail))
    return out
