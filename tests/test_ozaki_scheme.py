"""CPU pins of the Ozaki-II arithmetic (R26), independent of
the CUDA code: the library's parameter choice (tci_ozaki_params, pure host)
must satisfy the exactness conditions, and the O(n) CRT reconstruction the
kernel uses (37-bit chunked CRT weights, one quotient estimate, carry
normalisation, all in float64) is re-implemented here with Python big
integers / numpy float64 and must recover the integer exactly (to one ulp of
its float64 value) for integers spanning the whole guaranteed range."""
import math

import numpy as np
import pytest


def lib():
    import paper_2512_23917_b200 as tci
    return tci


@pytest.mark.parametrize("K", [1, 64, 1000, 4096, 20480, 24576, 131072])
def test_params_guarantee_exactness(K):
    st, n, t, mods = lib().tci_ozaki_params(K)
    assert st == 0
    assert all(m % 2 == 1 and m <= 255 for m in mods)
    assert all(math.gcd(a, b) == 1 for i, a in enumerate(mods) for b in mods[i + 1:])
    M = math.prod(mods)
    # |C'| <= 2 K 2^(2t) (complex product of t-bit integers) must be <= M/4
    assert 2 * K * 2 ** (2 * t) <= M // 4
    # 3M operand sums are (t+1)-bit; int8 residues and int32 accumulation exact
    assert K * 127 * 127 < 2 ** 31
    assert t >= 46                                   # ~2^-46 relative truncation per operand entry


def test_params_reject_long_k():
    st, *_ = lib().tci_ozaki_params(131073)
    assert st != 0


def _device_crt(residues, mods):
    """The kernel's reconstruction (ozaki.cu crt_value) in numpy float64."""
    M = math.prod(mods)
    mask = (1 << 37) - 1
    W = []
    for m in mods:
        Ml = M // m
        W.append((Ml * pow(Ml % m, -1, m)) % M)
    Wc = np.array([[float(w & mask), float((w >> 37) & mask), float(w >> 74)] for w in W])
    Mch = np.array([float(M & mask), float((M >> 37) & mask), float(M >> 74)])
    S = np.zeros(3)
    for c, w in zip(residues, Wc):
        S = S + float(c) * w                         # exact: integers < 2^48
    two37 = float(2 ** 37)
    xe = (S[2] * two37 * two37 + S[1] * two37) + S[0]
    q = np.rint(xe * (1.0 / float(M)))
    r = S - q * Mch
    cy = np.rint(r[0] / two37)
    r0 = r[0] - cy * two37
    r1 = r[1] + cy
    cy = np.rint(r1 / two37)
    r1 = r1 - cy * two37
    r2 = r[2] + cy
    return (r2 * two37 * two37 + r1 * two37) + r0


@pytest.mark.parametrize("K", [64, 4096, 20480])
def test_crt_reconstruction_exact(K):
    _, n, t, mods = lib().tci_ozaki_params(K)
    bound = 2 * K * 2 ** (2 * t)                      # the guaranteed |C'| range
    rng = np.random.default_rng(K)
    samples = [0, 1, -1, bound, -bound, bound - 12345, 2 ** 60 + 7]
    samples += [int(rng.integers(-2 ** 62, 2 ** 62)) * (1 << (2 * t + 14 - 62)) + int(rng.integers(-1000, 1000))
                for _ in range(200)]
    for X in samples:
        X = max(-bound, min(bound, X))
        res = []
        for m in mods:
            c = X % m
            res.append(c - m if c > m // 2 else c)   # balanced residue
        got = _device_crt(res, mods)
        ref = float(X)
        assert got == ref or abs(got - ref) <= abs(ref) * 2.0 ** -52, (X, got, ref)
