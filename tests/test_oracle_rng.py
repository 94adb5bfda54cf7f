"""Pins for the oracle's Philox4x32-10, uniform conversion and tau draw.

Philox is pinned against a library implementation on the box that the oracle
does not use: PyTorch's header-only `at::philox_engine`
(ATen/core/PhiloxRNGEngine.h; key = seed, counter[2..3] = subsequence,
counter[0..1] = offset in 128-bit blocks -> our counter (n, g)),
compiled here with g++.  The uniform conversion is pinned by exact bit
patterns at its edges; the exponential draw by S:203-205 / S:518.
"""
import math
import os
import subprocess
import tempfile

import numpy as np
import pytest

import oracle

CASES = [(1, 0, 0), (1, 1, 0), (1, 0, 1), (0, 0, 0), (2**64 - 1, 2**64 - 1, 2**64 - 1),
         (0x243F6A8885A308D3, 12345, 987654321), (1, 16383, 300000), (42, 2**40 + 3, 2**33 + 7)]


def _torch_include():
    import torch
    return os.path.join(os.path.dirname(torch.__file__), "include")


@pytest.fixture(scope="module")
def torch_philox():
    src = r"""
#include <ATen/core/PhiloxRNGEngine.h>
#include <cstdio>
#include <cstdlib>
int main(int argc, char** argv) {
  for (int i = 1; i + 2 < argc; i += 3) {
    unsigned long long seed = strtoull(argv[i], 0, 10), sub = strtoull(argv[i+1], 0, 10),
                       off = strtoull(argv[i+2], 0, 10);
    at::Philox4_32 e(seed, sub, off);
    unsigned a = e(), b = e(), c = e(), d = e();
    printf("%u %u %u %u\n", a, b, c, d);
  }
}
"""
    d = tempfile.mkdtemp()
    cpp = os.path.join(d, "p.cpp")
    exe = os.path.join(d, "p")
    with open(cpp, "w") as f:
        f.write(src)
    subprocess.check_call(["g++", "-std=c++17", "-O1", "-I", _torch_include(), cpp, "-o", exe])

    def run(cases):
        args = [str(v) for c in cases for v in c]
        out = subprocess.check_output([exe] + args).decode().split("\n")
        return [[int(v) for v in line.split()] for line in out if line.strip()]
    return run


def test_philox_matches_at_philox_engine(torch_philox):
    rng = np.random.default_rng(3)
    cases = list(CASES) + [tuple(int(v) for v in rng.integers(0, 2**63, size=3, dtype=np.int64)) for _ in range(200)]
    ref = torch_philox(cases)
    for (seed, g, n), want in zip(cases, ref):
        ctr = [n & 0xFFFFFFFF, n >> 32, g & 0xFFFFFFFF, g >> 32]
        key = [seed & 0xFFFFFFFF, seed >> 32]
        assert oracle.philox4x32_10(ctr, key) == want, (seed, g, n)


def test_uniform_edges():
    # all-zero words: u1 = 2^-53 (smallest, never 0), u2 = 0
    assert oracle.uniforms([0, 0, 0, 0]) == (2.0**-53, 0.0)
    # all-one words: u1 = 1 exactly (tau = 0), u2 = 1 - 2^-53 (largest, never 1)
    m = 0xFFFFFFFF
    assert oracle.uniforms([m, m, m, m]) == (1.0, 1.0 - 2.0**-53)
    # 53 significant bits are kept: bit 11 of the low word is the last one used
    u1, u2 = oracle.uniforms([0, 1 << 11, 0, 1 << 11])
    assert u1 == 2.0 * 2.0**-53 and u2 == 2.0**-53
    u1, u2 = oracle.uniforms([0, (1 << 11) - 1, 0, (1 << 11) - 1])
    assert u1 == 2.0**-53 and u2 == 0.0


def test_tau_examples_spec():
    # S:203-205 through the oracle's own tau (the function its loop calls):
    # u = e^-1, r = 2 -> tau = 0.5 (within 1 ulp: e^-1 is rounded); u = 1 -> tau = 0
    assert abs(oracle.tau(math.exp(-1.0), 2.0) - 0.5) <= 2.0**-53
    assert oracle.tau(1.0, 5.0) == 0.0
    # the smallest u1 the conversion produces (2^-53): tau = 53 ln 2 / a0
    assert abs(oracle.tau(2.0**-53, 1.0) - 53 * math.log(2.0)) <= 2 * 2.0**-47
    # tau scales as 1 / a0 (one IEEE division of the same -log u1)
    assert oracle.tau(0.3, 1.0) / 4.0 == oracle.tau(0.3, 4.0)


def test_exponential_moments_from_philox_stream():
    # 10^6 draws at r = 2: mean within 1% of 0.5, variance within 3% of 0.25
    taus, _ = oracle.tau_stream(1, 7, 0, 1_000_000, 2.0)
    assert taus.min() >= 0.0 and np.isfinite(taus).all()
    assert abs(taus.mean() - 0.5) < 0.005
    assert abs(taus.var() - 0.25) < 0.0075


def test_u2_uniformity_chi2():
    n, bins = 1_000_000, 50
    _, u = oracle.tau_stream(9, 3, 0, n, 1.0)
    h, _ = np.histogram(u, bins=bins, range=(0.0, 1.0))
    e = n / bins
    chi2 = ((h - e) ** 2 / e).sum()
    assert chi2 < 100.0  # df = 49, p ~ 3e-5


def test_tau_stream_is_exact_within_one_ulp():
    # the stream's tau of block (n, g) against the exact value -ln(u1) / a0
    # (mpmath, 60 digits), u1 from the uniform conversion pinned above.
    # glibc's log is within 1 ulp of E = -ln u1, i.e. relative error < 2^-52,
    # and the division rounds once more (2^-53 relative): |tau - exact| <
    # 1.5 * 2^-52 * exact.  (A dropped negation, a reciprocal multiply
    # instead of the division, or log1p(-u) would all fail this.)
    import mpmath
    mpmath.mp.dps = 60
    a0 = 3.7
    tau, u2 = oracle.tau_stream(5, 11, 100, 400, a0)
    for i in range(400):
        w = oracle.philox4x32_10([100 + i, 0, 11, 0], [5, 0])
        u1, v2 = oracle.uniforms(w)
        assert u2[i] == v2
        exact = -mpmath.log(mpmath.mpf(u1)) / mpmath.mpf(a0)
        assert abs(mpmath.mpf(tau[i]) - exact) <= mpmath.mpf(1.5) * mpmath.mpf(2) ** -52 * exact, i


def _kat():
    path = os.path.join(os.path.dirname(__file__), "golden", "philox4x32_10_kat.txt")
    rows = []
    for line in open(path):
        if line.strip() and not line.startswith("#"):
            w = [int(v, 16) for v in line.split()]
            rows.append((w[0:4], w[4:6], w[6:10]))
    return rows


def test_philox_known_answers(torch_philox):
    rows = _kat()
    assert len(rows) == 3
    cases = []
    for ctr, key, _ in rows:
        cases.append((key[0] | (key[1] << 32), ctr[2] | (ctr[3] << 32), ctr[0] | (ctr[1] << 32)))
    ref = torch_philox(cases)
    for (ctr, key, want), lib in zip(rows, ref):
        assert lib == want
        assert oracle.philox4x32_10(ctr, key) == want
