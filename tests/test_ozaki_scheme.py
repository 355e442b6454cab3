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
    """The kernel's reconstruction (ozaki.cu crt_value / crt_kernel) in numpy
    float64: NCH = 3 chunks of 37 bits for <= 14 moduli, 4 for 15."""
    M = math.prod(mods)
    nch = 3 if len(mods) <= 14 else 4
    mask = (1 << 37) - 1
    W = []
    for m in mods:
        Ml = M // m
        W.append((Ml * pow(Ml % m, -1, m)) % M)
    Wc = np.array([[float((w >> (37 * j)) & mask) for j in range(nch)] for w in W])
    Mch = np.array([float((M >> (37 * j)) & mask) for j in range(nch)])
    assert all((M >> (37 * nch)) == 0 for _ in [0]) and all(w >> (37 * nch) == 0 for w in W)
    S = np.zeros(nch)
    S_int = [0] * nch
    for c, w in zip(residues, Wc):
        S = S + float(c) * w
        S_int = [s + c * int(x) for s, x in zip(S_int, w)]
    assert [int(s) for s in S] == S_int and max(abs(s) for s in S_int) < 2 ** 53   # exact chunk sums
    two37 = float(2 ** 37)
    xe = S[nch - 1]
    for j in range(nch - 2, -1, -1):
        xe = xe * two37 + S[j]
    q = np.rint(xe * (1.0 / float(M)))
    r = S - q * Mch
    for j in range(nch - 1):
        cy = np.rint(r[j] / two37)
        r[j] = r[j] - cy * two37
        r[j + 1] = r[j + 1] + cy
    x = r[nch - 1]
    for j in range(nch - 2, -1, -1):
        x = x * two37 + r[j]
    return x


@pytest.mark.parametrize("K", [64, 4096, 20480, 40960, 131072])
def test_crt_reconstruction_exact(K):
    _, n, t, mods = lib().tci_ozaki_params(K)
    bound = 2 * K * 2 ** (2 * t)                      # the guaranteed |C'| range
    rng = np.random.default_rng(K)
    samples = [0, 1, -1, bound, -bound, bound - 12345, 2 ** 60 + 7]
    samples += [int(rng.integers(-2 ** 62, 2 ** 62)) * (1 << (2 * t + 14 - 62)) + int(rng.integers(-1000, 1000))
                for _ in range(200)]
    for i, X in enumerate(samples):
        X = max(-bound, min(bound, X))
        # the kernel's representatives: P - Q + m in (0, 2m), S - P - Q + 2m in
        # (0, 3m); take the extreme ones (up to 3m - 1) half of the time
        res = []
        for m in mods:
            c = X % m
            res.append(c + 2 * m if (i % 2 and c + 2 * m < 3 * m) else c + m * int(rng.integers(0, 3)))
        got = _device_crt(res, mods)
        ref = float(X)
        assert got == ref or abs(got - ref) <= abs(ref) * 2.0 ** -52, (X, got, ref)
