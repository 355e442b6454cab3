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


# ---------------------------------------------------------------------------
# K-balancing and the guard's error estimate (R26), emulated in
# exact integer arithmetic at a small bit budget (t = 20, int64 products)
# ---------------------------------------------------------------------------

def _exps(x, axis):
    """E with |x| < 2^E over each line (re and im), -100000 for zero lines."""
    a = np.abs(x.real) if not np.iscomplexobj(x) else np.maximum(np.abs(x.real), np.abs(x.imag))
    m = a.max(axis=axis)
    return np.where(m > 0, np.frexp(m)[1], -100000)


def _emulate(A, B, t, balance):
    """The scheme of ozaki.cu on real data: s_k = floor((KB_k - KA_k)/2)
    (none when its spread is <= 2), row/column exponents of the balanced
    operands, rint to t-bit integers, exact integer product, scale back; and
    the guard's estimate sqrt(c 4^-t (S_M ||B'||^2 + ||A'||^2 S_N)) / ||C||."""
    KA, KB = _exps(A, 0), _exps(B, 1)
    s = np.where((KA > -100000) & (KB > -100000), np.floor_divide(KB - KA, 2), 0)
    if not balance or s.max() - s.min() <= 2:
        s = np.zeros_like(s)
    Ab, Bb = A * np.ldexp(1.0, s)[None, :], B * np.ldexp(1.0, -s)[:, None]
    EA, EB = _exps(Ab, 1), _exps(Bb, 0)
    Ai = np.rint(Ab * np.ldexp(1.0, t - EA)[:, None]).astype(np.int64)
    Bi = np.rint(Bb * np.ldexp(1.0, t - EB)[None, :]).astype(np.int64)
    C = (Ai @ Bi).astype(np.float64) * np.ldexp(1.0, -(2 * t - EA[:, None] - EB[None, :]))
    SM, SN = np.ldexp(1.0, 2 * EA).sum(), np.ldexp(1.0, 2 * EB).sum()
    est = math.sqrt((1 / 12) * 4.0 ** -t * (SM * (Bb * Bb).sum() + (Ab * Ab).sum() * SN)) / np.linalg.norm(C)
    return C, est, bool(np.any(s))


def _cases():
    rng = np.random.default_rng(11)
    M, K, N = 96, 384, 80
    X, Y = rng.uniform(-1, 1, (M, K)), rng.uniform(-1, 1, (K, N))
    e = rng.integers(-30, 31, K)
    lam = np.geomspace(1, 1e-10, K)
    return {
        "uniform": (X, Y),
        "anticorrelated_2^30": (X * np.ldexp(1.0, e)[None, :], Y * np.ldexp(1.0, -e)[:, None]),
        "vidal": (X * lam[None, :], Y / lam[:, None] * np.geomspace(1, 1e-10, N)[None, :]),
        "graded_rows_of_B": (X, Y * lam[:, None]),
    }


@pytest.mark.parametrize("name", list(_cases()))
def test_balanced_scheme_error_matches_estimate(name):
    """With the K-balancing the truncation error is ~2^-t for every structure
    here, and the guard's estimate predicts it within a factor of 1.5 (it is
    the expected value of the squared error for independent roundings)."""
    A, B = _cases()[name]
    t = 20
    C, est, _ = _emulate(A, B, t, balance=True)
    ref = A @ B
    err = np.linalg.norm(C - ref) / np.linalg.norm(ref)
    assert err < 2.0 ** -t * 8
    assert est / 1.5 <= err <= est * 1.5, (err, est)


@pytest.mark.parametrize("name", ["anticorrelated_2^30", "vidal"])
def test_unbalanced_scheme_fails_and_estimate_flags_it(name):
    """Without the balancing the same inputs lose ~all bits (the round-1
    scheme); the estimate flags it (far above the guard's tolerance scaled to
    t = 20), and the balancing is what engages."""
    A, B = _cases()[name]
    C, est, _ = _emulate(A, B, 20, balance=False)
    ref = A @ B
    err = np.linalg.norm(C - ref) / np.linalg.norm(ref)
    assert err > 1e-3 and est > 1e-3
    _, _, used = _emulate(A, B, 20, balance=True)
    assert used
