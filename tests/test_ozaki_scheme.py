"""CPU pins of the Ozaki-II arithmetic (R26), independent of
the CUDA code: the library's parameter choice (tci_ozaki_params, pure host)
must satisfy the exactness conditions, and the O(n) CRT reconstruction the
kernel uses (37-bit chunked CRT weights, one quotient estimate, carry
normalisation, all in float64) is re-implemented here with Python big
integers / numpy float64 and must recover the integer exactly (to one ulp of
its float64 value) for integers spanning the whole guaranteed range."""
import math
import random

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
    # the kernel's encoding: each representative c < 2^10 enters as the double
    # 1 + c 2^-10; T_j = sum_l (1 + c_l 2^-10) W_lj, S_j = 2^10 T_j - 2^10 sum_l W_lj
    T = np.zeros(nch)
    S_int = [0] * nch
    for c, w in zip(residues, Wc):
        assert 0 <= c < 1024
        T = T + (1.0 + float(c) / 1024.0) * w
        S_int = [s + c * int(x) for s, x in zip(S_int, w)]
    S = T * 1024.0 - 1024.0 * Wc.sum(axis=0)
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


# ---------------------------------------------------------------------------
# Gaussian moduli of the complex path (R33): a + ib -> (a + j b,
# a - j b) mod m is a ring homomorphism when j^2 = -1 (mod m), so a complex
# product mod m is two real products; the CRT folds 2^-1 and (2j)^-1 into
# its weights. Emulated here with Python big integers and numpy float64.
# ---------------------------------------------------------------------------

def _prime_factors(n):
    f, p = set(), 2
    while p * p <= n:
        while n % p == 0:
            f.add(p)
            n //= p
        p += 1
    if n > 1:
        f.add(n)
    return f


@pytest.mark.parametrize("K", [1, 64, 1000, 4096, 20480, 24576, 69000, 131072])
def test_params_complex_gaussian(K):
    st, n, t, mods, roots, ppm = lib().tci_ozaki_params_complex(K, 0)
    assert st == 0 and ppm == 2
    assert all(m % 2 == 1 and 64 < m < 256 for m in mods)
    assert all(math.gcd(a, b) == 1 for i, a in enumerate(mods) for b in mods[i + 1:])
    assert all(p % 4 == 1 for m in mods for p in _prime_factors(m))      # sqrt(-1) exists mod m
    assert all((j * j + 1) % m == 0 and abs(j) <= (m - 1) // 2 for m, j in zip(mods, roots))
    M = math.prod(mods)
    assert 2 * K * 2 ** (2 * t) <= M // 4           # |Re C'|, |Im C'| <= 2 K 2^(2t) <= M/4
    assert K * (max(mods) // 2) ** 2 < 2 ** 31      # balanced int8 residues, exact int32 sums
    assert t >= 46
    # 39-bit CRT chunks: 3 cover M for 15 moduli, 4 for 16; the encoded chunk
    # sums sum_l W_l (512 + x_l) < 16 2^39 (512 + 482) stay exact in float64
    assert M < 2 ** (39 * (3 if n <= 15 else 4)) and 16 * 2 ** 39 * (512 + 482) < 2 ** 53


def _gauss_crt(xs, mods, weights):
    """crt_value<NCH, 39> of the kernel on the representatives xs (numpy
    float64): 39-bit chunks, 3 for 15 moduli and 4 for 16; each x < 2^9
    enters as the double 1 + x 2^-9 (crt_kernel's one_plus<9>)."""
    M = math.prod(mods)
    cb = 39
    nch = 3 if len(mods) <= 15 else 4
    mask = (1 << cb) - 1
    Wc = np.array([[float((w >> (cb * j)) & mask) for j in range(nch)] for w in weights])
    Mch = np.array([float((M >> (cb * j)) & mask) for j in range(nch)])
    assert M >> (cb * nch) == 0
    T = np.zeros(nch)
    S_int = [0] * nch
    for c, w in zip(xs, Wc):
        assert 0 <= c < 512
        T = T + (1.0 + float(c) / 512.0) * w
        S_int = [s + c * int(x) for s, x in zip(S_int, w)]
    assert all(float(t) * 512 == int(t * 512) for t in T)       # partial sums stay exact
    S = T * 512.0 - 512.0 * Wc.sum(axis=0)
    assert [int(s) for s in S] == S_int and max(abs(s) for s in S_int) < 2 ** 53
    two = float(2 ** cb)
    xe = S[nch - 1]
    for j in range(nch - 2, -1, -1):
        xe = xe * two + S[j]
    q = np.rint(xe * (1.0 / float(M)))
    r = S - q * Mch
    for j in range(nch - 1):
        cy = np.rint(r[j] / two)
        r[j] = r[j] - cy * two
        r[j + 1] = r[j + 1] + cy
    x = r[nch - 1]
    for j in range(nch - 2, -1, -1):
        x = x * two + r[j]
    return x


def _gauss_crt_tc(cps, cms, mods, roots):
    """crt_mma.cu's reconstruction of (Re C', Im C') from the byte planes
    c+_l, c-_l: the INT8 tensor-core digit sums s_j = sum_k c_k Bd[k][j]
    (exact integers), 16-bit digit pairs, 32-bit chunks, the quotient from the
    top two chunks, r_c = S_c - q M_c and Horner from the top -- every float64
    operation emulated with correct rounding (Python int -> float)."""
    M = math.prod(mods)
    WR, WI = _gauss_weights(mods, roots)
    n = len(mods)
    nd = (M.bit_length() + 7) // 8
    npair = (nd + 1) // 2
    nc = (npair + 1) // 2
    Bd = [[0] * 32 for _ in range(32)]
    for l in range(n):
        for j in range(16):
            Bd[2 * l][j] = Bd[2 * l + 1][j] = (WR[l] >> (8 * j)) & 255
            Bd[2 * l][16 + j] = (WI[l] >> (8 * j)) & 255
            Bd[2 * l + 1][16 + j] = ((M - WI[l]) >> (8 * j)) & 255
    c = [0] * 32
    for l in range(n):
        assert 0 <= cps[l] < mods[l] and 0 <= cms[l] < mods[l]
        c[2 * l], c[2 * l + 1] = cps[l], cms[l]
    sd = [sum(c[k] * Bd[k][j] for k in range(32)) for j in range(32)]
    assert max(sd) < 2 ** 21                                   # exact int32 accumulators
    Mch = [(M >> (32 * j)) & 0xFFFFFFFF for j in range(nc)]
    assert M >> (32 * nc) == 0
    mtop = float(2 ** (32 * (nc - 2))) / float(M)
    out = []
    for v in (0, 1):
        d = sd[16 * v:16 * v + 16]
        p = [d[2 * k] + 256 * d[2 * k + 1] for k in range(8)]
        assert max(p) < 2 ** 30
        S = [p[2 * k] + (p[2 * k + 1] << 16 if 2 * k + 1 < npair else 0) for k in range(nc)]
        assert max(S) < 2 ** 47
        xe = float(S[nc - 1] * 2 ** 32 + S[nc - 2])            # fma: one rounding
        q = int(np.rint(xe * mtop))
        r = [S[j] - q * Mch[j] for j in range(nc)]             # exact (|q M_c| < 2^45)
        assert q < 2 ** 13 and max(abs(x) for x in r) < 2 ** 53
        if nc == 4:   # M > 2^96: the first Horner step is exact (|C'| / 2^64 < 2^47)
            assert abs(r[nc - 1] * 2 ** 32 + r[nc - 2]) < 2 ** 53
        x = float(r[nc - 1])
        for j in range(nc - 2, -1, -1):
            x = float(int(x) * 2 ** 32 + r[j])                 # fma(x, 2^32, r_j): one rounding
        out.append(x)
    return out


def _gauss_weights(mods, roots):
    M = math.prod(mods)
    WR, WI = [], []
    for m, j in zip(mods, roots):
        Ml = M // m
        w = (Ml * pow(Ml % m, -1, m)) % M
        WR.append((w * pow(2, -1, m)) % M)
        WI.append((w * pow((2 * j) % m, -1, m)) % M)
    return WR, WI


def _bal(x, m):
    r = x % m
    return r - m if r > m // 2 else r


@pytest.mark.parametrize("K", [64, 4096, 20480])
def test_gaussian_scheme_exact_complex_product(K):
    """Integer complex matrices with t-bit entries: balanced Gaussian residues
    (int8), the two modular products per modulus (the INT8 GEMMs + mod-m
    epilogue), the kernel's CRT with folded weights: the exact integer
    complex product, to one ulp of its float64 value."""
    st, n, t, mods, roots, _ = lib().tci_ozaki_params_complex(K)
    rng = np.random.default_rng(K + 5)
    Mr, Nr, Ks = 3, 2, min(K, 48)      # a few output entries; K terms of which Ks random, rest at the bound
    lim = 2 ** t - 1

    def ent():
        return int(rng.integers(-lim, lim, endpoint=True)), int(rng.integers(-lim, lim, endpoint=True))
    A = [[ent() for _ in range(Ks)] for _ in range(Mr)]
    B = [[ent() for _ in range(Nr)] for _ in range(Ks)]
    A[0] = [(lim, lim)] * Ks                              # extreme entries
    B = [[(lim, -lim)] + row[1:] for row in B]
    WR, WI = _gauss_weights(mods, roots)
    for i in range(Mr):
        for jn in range(Nr):
            cr = sum(A[i][k][0] * B[k][jn][0] - A[i][k][1] * B[k][jn][1] for k in range(Ks))
            ci = sum(A[i][k][0] * B[k][jn][1] + A[i][k][1] * B[k][jn][0] for k in range(Ks))
            xr, xi = [], []
            for m, j in zip(mods, roots):
                cp = cm = 0
                for k in range(Ks):
                    ar, ai = _bal(A[i][k][0], m), _bal(A[i][k][1], m)
                    br, bi = _bal(B[k][jn][0], m), _bal(B[k][jn][1], m)
                    up, um = _bal(ar + j * ai, m), _bal(ar - j * ai, m)     # int8 planes of A
                    vp, vm = _bal(br + j * bi, m), _bal(br - j * bi, m)     # int8 planes of B
                    assert max(abs(up), abs(um), abs(vp), abs(vm)) <= 127
                    cp += up * vp
                    cm += um * vm
                cp, cm = cp % m, cm % m                                     # GEMM epilogue bytes
                xr.append(cp + cm)                                          # [0, 2m)
                xi.append(cp - cm + m)                                      # (0, 2m)
            gr, gi = _gauss_crt(xr, mods, WR), _gauss_crt(xi, mods, WI)
            for got, ref in ((gr, cr), (gi, ci)):
                assert got == float(ref) or abs(got - ref) <= abs(ref) * 2.0 ** -52, (got, ref)
            cps = [(xr[l] + xi[l] - m) // 2 % m for l, m in enumerate(mods)]   # c+ = ((c+ + c-) + (c+ - c- + m) - m) / 2
            cms = [(xr[l] - cps[l]) % m for l, m in enumerate(mods)]
            tr, ti = _gauss_crt_tc(cps, cms, mods, roots)
            for got, ref in ((tr, cr), (ti, ci)):
                assert got == float(ref) or abs(got - ref) <= abs(ref) * 2.0 ** -51, (got, ref)


@pytest.mark.parametrize("K", [4096, 20480, 131072])
def test_gaussian_crt_full_range(K):
    """The reconstruction over the whole guaranteed range |C'| <= 2 K 2^(2t):
    representatives c+ + c- and c+ - c- + m of random and extreme values."""
    st, n, t, mods, roots, _ = lib().tci_ozaki_params_complex(K)
    WR, WI = _gauss_weights(mods, roots)
    bound = 2 * K * 2 ** (2 * t)
    rng = np.random.default_rng(K)
    vals = [(0, 0), (bound, -bound), (-bound, bound), (1, -1), (bound - 777, 3)]
    vals += [(int(rng.integers(-2 ** 62, 2 ** 62)) << (2 * t + 14 - 62), int(rng.integers(-2 ** 62, 2 ** 62)))
             for _ in range(100)]
    for cr, ci in vals:
        cr, ci = max(-bound, min(bound, cr)), max(-bound, min(bound, ci))
        xr, xi = [], []
        for m, j in zip(mods, roots):
            cp, cm = (cr + j * ci) % m, (cr - j * ci) % m
            xr.append(cp + cm)
            xi.append(cp - cm + m)
        gr, gi = _gauss_crt(xr, mods, WR), _gauss_crt(xi, mods, WI)
        for got, ref in ((gr, cr), (gi, ci)):
            assert got == float(ref) or abs(got - ref) <= abs(ref) * 2.0 ** -52, (got, ref)


@pytest.mark.parametrize("K", [64, 4096, 20480, 131072])
@pytest.mark.parametrize("tmin", [46, 24])
def test_gaussian_crt_tensor_core_full_range(K, tmin):
    """crt_mma.cu's digit-sum CRT (the default complex CRT) over the whole
    guaranteed range |Re C'|, |Im C'| <= 2 K 2^(2t), for the float64 (t >= 46)
    and float32 (t >= 24) moduli sets: within 2 ulp of the integer (exact
    below 2^53)."""
    if tmin == 46:
        st, n, t, mods, roots, _ = lib().tci_ozaki_params_complex(K, 0)
    else:
        st, n, t, mods, ppm = lib().tci_ozaki_params_f32(K, True)
        assert ppm == 2
        root_of = dict(zip(*lib().tci_ozaki_params_complex(131072, 0)[3:5]))
        roots = [root_of[m] for m in mods]
    assert st == 0 and t >= tmin
    bound = 2 * K * 2 ** (2 * t)
    rnd = random.Random(K + tmin)
    vals = [(0, 0), (bound, -bound), (-bound, bound), (1, -1), (bound - 777, 3), (2 ** 53 + 1, -(2 ** 52) - 3)]
    for _ in range(60):
        e = rnd.randrange(bound.bit_length())
        vals.append((rnd.randint(-2 ** e, 2 ** e), rnd.randint(-bound, bound)))
    for cr, ci in vals:
        cr, ci = max(-bound, min(bound, cr)), max(-bound, min(bound, ci))
        cps = [(cr + j * ci) % m for m, j in zip(mods, roots)]
        cms = [(cr - j * ci) % m for m, j in zip(mods, roots)]
        for got, ref in zip(_gauss_crt_tc(cps, cms, mods, roots), (cr, ci)):
            assert got == float(ref) or abs(got - ref) <= abs(ref) * 2.0 ** -51, (got, ref)
            if abs(ref) < 2 ** 53:
                assert got == ref


def _real_crt_tc(cs, mods):
    """crt_mma.cu for real outputs: plane l = C' mod m_l, digit columns 0..15 the
    base-256 digits of w_l = (M/m_l) ((M/m_l)^-1 mod m_l), the same epilogue
    as _gauss_crt_tc on the one value (float64 operations emulated exactly)."""
    M = math.prod(mods)
    nd = (M.bit_length() + 7) // 8
    npair = (nd + 1) // 2
    nc = (npair + 1) // 2
    W = [(M // m) * pow((M // m) % m, -1, m) % M for m in mods]
    sd = [sum(c * ((w >> (8 * j)) & 255) for c, w in zip(cs, W)) for j in range(16)]
    assert max(sd) < 2 ** 21
    p = [sd[2 * k] + 256 * sd[2 * k + 1] for k in range(8)]
    S = [p[2 * k] + (p[2 * k + 1] << 16 if 2 * k + 1 < npair else 0) for k in range(nc)]
    Mch = [(M >> (32 * j)) & 0xFFFFFFFF for j in range(nc)]
    xe = float(S[nc - 1] * 2 ** 32 + S[nc - 2])
    q = int(np.rint(xe * (float(2 ** (32 * (nc - 2))) / float(M))))
    r = [S[j] - q * Mch[j] for j in range(nc)]
    x = float(r[nc - 1])
    for j in range(nc - 2, -1, -1):
        x = float(int(x) * 2 ** 32 + r[j])
    return x


@pytest.mark.parametrize("K", [64, 4096, 20480, 131072])
def test_real_crt_tensor_core_full_range(K):
    """The real tensor-core CRT (float64 / float32 Ozaki GEMMs) over the whole
    guaranteed range |C'| <= K 2^(2t) (real products), exact below 2^53."""
    for st, n, t, mods in (lib().tci_ozaki_params(K), lib().tci_ozaki_params_f32(K, False)[:4]):
        assert st == 0
        bound = 2 * K * 2 ** (2 * t)
        rnd = random.Random(K + t)
        vals = [0, 1, -1, bound, -bound, 2 ** 53 + 1] + [rnd.randint(-bound, bound) for _ in range(40)]
        vals += [rnd.randint(-2 ** e, 2 ** e) for e in range(0, bound.bit_length(), 7)]
        for v in vals:
            got = _real_crt_tc([v % m for m in mods], mods)
            assert got == float(v) or abs(got - v) <= abs(v) * 2.0 ** -51, (got, v)
            if abs(v) < 2 ** 53:
                assert got == v


def test_params_complex_3m_and_errors():
    st, n, t, mods, roots, ppm = lib().tci_ozaki_params_complex(20480, 1)
    st0, n0, t0, mods0 = lib().tci_ozaki_params(20480)
    assert st == 0 and ppm == 3 and roots == [0] * n and (n, t, mods) == (n0, t0, mods0)
    assert lib().tci_ozaki_params_complex(20480, 7)[0] != 0
    assert lib().tci_ozaki_params_complex(131073, 0)[0] != 0
    # the Gaussian variant needs 2n' INT8 GEMMs against 3n: 30 vs 42 at the bench's K
    _, ng, _, _, _, _ = lib().tci_ozaki_params_complex(20480, 0)
    assert (2 * ng, 3 * n) == (30, 42)
