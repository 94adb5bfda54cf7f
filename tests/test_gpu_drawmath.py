"""GPU: the SSA kernels' branch-free draw arithmetic (device_common.cuh).

* tau = E / a0 must be the IEEE quotient bit for bit: the
  kernels' fast division is checked against numpy's (IEEE) division over the
  whole input range, fast-path range and edges included.
* E = -log u1 comes from the kernels' own branch-free log: u2 must
  equal the oracle's bit for bit; E must be within 1 ulp of the
  correctly rounded value (mpmath, 200 bits) and equal to the oracle's
  glibc log in all but a small fraction of draws (DESIGN.md "Parity":
  a one-ulp E moves tau by one ulp, the traced "log-ulp" class).
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

import oracle  # noqa: E402

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_1010_2438_b200 import cwc  # noqa: E402


def _ulps(a, b):
    """|a - b| in ulps for finite doubles of equal sign (exact int64 arithmetic)."""
    return np.abs(a.view(np.int64) - b.view(np.int64))


def _tau_div(e, a):
    et = torch.as_tensor(e, device="cuda")
    at = torch.as_tensor(a, device="cuda")
    q = torch.empty_like(et)
    cwc.cwc_tau_div(et, at, q, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    return q.cpu().numpy()


def test_tau_division_is_ieee_fast_range():
    rng = np.random.default_rng(11)
    n = 1 << 22
    u = (rng.integers(0, 1 << 53, size=n, dtype=np.int64) + 1).astype(np.float64) * 2.0**-53
    e = -np.log(u)                                    # the E values the method produces
    a = 10.0 ** rng.uniform(-12, 15, size=n)          # propensity sums of every config and beyond
    q = _tau_div(e, a)
    want = e / a
    assert np.array_equal(q.view(np.int64), want.view(np.int64))


def test_tau_division_is_ieee_edges():
    rng = np.random.default_rng(12)
    n = 1 << 20
    e = np.concatenate([rng.uniform(0, 40, n // 2), 10.0 ** rng.uniform(-320, 300, n // 2)])
    a = np.concatenate([10.0 ** rng.uniform(-320, 308, n // 2), rng.uniform(1e-3, 1e3, n // 2)])
    edges_e = np.array([0.0, -0.0, 2.0**-60, 2.0**-61, 64.0, 64.0000001, 1.0, 36.7368005696771, 5e-324, np.inf])
    edges_a = np.array([0.0, 1.0, 2.0**-900, 2.0**-901, 2.0**900, 2.0**901, 1e-310, 3.0, np.inf, np.nan])
    E, A = np.meshgrid(edges_e, edges_a)
    e = np.concatenate([e, E.ravel()])
    a = np.concatenate([a, A.ravel()])
    with np.errstate(all="ignore"):
        want = e / a
    q = _tau_div(e, a)
    nan = np.isnan(want)
    assert np.array_equal(np.isnan(q), nan)
    assert np.array_equal(q[~nan].view(np.int64), want[~nan].view(np.int64))


def test_draws_match_oracle_and_are_accurate():
    rng = np.random.default_rng(13)
    seed = 1
    n_traj, per = 64, 4096
    g = np.repeat(rng.integers(0, 1 << 40, size=n_traj, dtype=np.int64), per)
    n0 = rng.integers(0, 1 << 30, size=n_traj, dtype=np.int64)
    n = (np.repeat(n0, per) + np.tile(np.arange(per, dtype=np.int64), n_traj))
    E = torch.empty(g.size, dtype=torch.float64, device="cuda")
    U = torch.empty_like(E)
    cwc.cwc_draws(seed, torch.as_tensor(g, device="cuda"), torch.as_tensor(n, device="cuda"), E, U,
                  torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    E = E.cpu().numpy()
    U = U.cpu().numpy()
    oe, ou = [], []
    for i in range(n_traj):
        tau, u2 = oracle.tau_stream(seed, int(g[i * per]), int(n0[i]), per, 1.0)  # a0 = 1: tau == E exactly
        oe.append(tau)
        ou.append(u2)
    oe = np.concatenate(oe)
    ou = np.concatenate(ou)
    assert np.array_equal(U.view(np.int64), ou.view(np.int64))
    d = _ulps(E, oe)
    assert d.max() <= 1
    # table-driven log: <= 0.5 ulp + 2^-60 (tools/logtable), glibc ~0.52 ulp
    assert (d == 0).mean() >= 0.995, (d == 0).mean()
    # accuracy against the correctly rounded value on a subsample
    mpmath = pytest.importorskip("mpmath")
    mpmath.mp.prec = 200
    worst = 0.0
    for i in rng.choice(E.size, size=3000, replace=False):
        w = oracle.philox4x32_10([int(n[i]) & 0xFFFFFFFF, int(n[i]) >> 32, int(g[i]) & 0xFFFFFFFF, int(g[i]) >> 32],
                                 [seed, 0])
        u1, _ = oracle.uniforms(w)
        if u1 == 1.0:
            continue
        ex = -mpmath.log(mpmath.mpf(u1))
        ulp = mpmath.mpf(2) ** (mpmath.floor(mpmath.log(ex, 2)) - 52)
        worst = max(worst, float(abs(mpmath.mpf(float(E[i])) - ex) / ulp))
    assert worst < 0.51, worst


def test_uniform_conversion_edges_match_oracle():
    """u1, u2 of raw blocks at the conversion edges (all-zero / all-one
    words, the top bit, the 11 dropped bits) equal the oracle's exactly, and
    E = -log u1 stays within one ulp of the oracle's log (u1 = 2^-53 and 1)."""
    edge = [0x00000000, 0xFFFFFFFF, 0x80000000, 0x7FFFFFFF, 0x000007FF, 0x00000800, 0xFFFFF800, 0x00100000]
    rng = np.random.default_rng(5)
    words = [[a, b, c, d] for a in edge for b in edge for c, d in [(a, b), (b, a)]]
    words += rng.integers(0, 2**32, size=(20000, 4), dtype=np.uint64).tolist()
    w = np.asarray(words, dtype=np.uint64).astype(np.uint32)
    wt = torch.as_tensor(w.view(np.int32), device="cuda")
    u1 = torch.empty(len(w), dtype=torch.float64, device="cuda")
    u2 = torch.empty_like(u1)
    E = torch.empty_like(u1)
    cwc.cwc_block_draws(wt, u1, u2, E, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    u1, u2, E = u1.cpu().numpy(), u2.cpu().numpy(), E.cpu().numpy()
    want = np.array([oracle.uniforms(x) for x in w])
    assert np.array_equal(u1.view(np.int64), want[:, 0].view(np.int64))
    assert np.array_equal(u2.view(np.int64), want[:, 1].view(np.int64))
    assert u1.min() == 2.0**-53 and u1.max() == 1.0 and u2.min() == 0.0 and u2.max() == 1.0 - 2.0**-53
    ref = -np.log(want[:, 0])
    assert _ulps(E, ref).max() <= 1
    assert E[u1 == 1.0].max() == 0.0
