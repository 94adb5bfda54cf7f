"""Divergence tracer (BASELINE north_star: "every divergence must be logged
and traced to a last-ulp difference in fp64 log or propensity sums").

For a trajectory whose GPU samples differ from the oracle's, both sides are
re-run with their per-firing trace -- (n, a0, tau, t', mu) per drawn
Philox block -- and the first differing record is classified:

  "a0-sum-order"  a0 differs (warp-path chunked/shuffle sum vs the oracle's
                  left-to-right sum); harmless ulp-level difference
  "log-ulp"       a0 equal, tau differs by <= 2 ulp (libdevice vs glibc log)
  "select-order"  a0, tau equal, mu differs on the warp path (chunk prefix)
  "BUG"           anything else (a different n, tau off by more than 2 ulp,
                  t' != t + tau, mu differing on the thread path, ...)
"""
import math

import numpy as np

import oracle


def ulp_diff(a, b):
    if a == b:
        return 0
    if not (math.isfinite(a) and math.isfinite(b)) or (a < 0) != (b < 0):
        return 1 << 62
    ia = np.frombuffer(np.float64(a).tobytes(), dtype=np.int64)[0]
    ib = np.frombuffer(np.float64(b).tobytes(), dtype=np.int64)[0]
    return abs(int(ia) - int(ib))


def classify(gpu_trace, ora_trace, warp_path):
    n = min(len(gpu_trace), len(ora_trace))
    for i in range(n):
        g, o = gpu_trace[i], ora_trace[i]
        if all(x == y for x, y in zip(g, o)):
            continue
        if g[0] != o[0]:
            return "BUG", i, "firing index differs"
        if g[1] != o[1]:
            return ("a0-sum-order" if warp_path and ulp_diff(g[1], o[1]) <= 64 else "BUG"), i, \
                "a0 %r vs %r" % (g[1], o[1])
        if g[2] != o[2]:
            return ("log-ulp" if ulp_diff(g[2], o[2]) <= 2 else "BUG"), i, "tau %r vs %r" % (g[2], o[2])
        if g[3] != o[3]:
            return "BUG", i, "t' differs with equal t and tau"
        if g[4] != o[4]:
            return ("select-order" if warp_path else "BUG"), i, "mu %r vs %r" % (g[4], o[4])
    if len(gpu_trace) != len(ora_trace):
        return "BUG", n, "trace lengths %d vs %d" % (len(gpu_trace), len(ora_trace))
    return "identical-trace", -1, ""


def trace_mismatches(model, desc, sweep, cfg, g_list, warp_path, force_path, cap=2_000_000):
    """Returns a list of (g, category, record index, detail)."""
    from paper_1010_2438_b200 import cwc
    out = []
    for g in g_list:
        gpu = cwc.simulate(model, cfg["n_replicas"], cfg["t_end"], cfg["sample_dt"], cfg["seed"], sweep=sweep,
                           want_firings=True, trace_g=[int(g)], trace_cap=cap, force_path=force_path)
        ln = int(gpu["trace_len"][0].item())
        gt = gpu["trace"][0, :ln].cpu().numpy()
        ora = oracle.simulate(desc, cfg["n_replicas"], cfg["t_end"], cfg["sample_dt"], cfg["seed"], sweep=sweep,
                              g_list=[int(g)], want_traj=False, want_stats=False, trace_g=int(g), trace_cap=cap)
        cat, idx, detail = classify([tuple(r) for r in gt], [tuple(r) for r in ora["trace"]], warp_path)
        out.append((int(g), cat, idx, detail))
    return out
