"""GPU parity tests of tci_svd / tci_trunc_svd
against the CPU oracle (oracle.svd / oracle.trunc_svd: LAPACK via numpy
plus the truncation strategy written out).

Several results are correct for an SVD (reading R29): singular
values, trunc_err, chi and -- where the spectrum is non-degenerate at the cut
-- the truncated product u s v_dag are unique and compared with the oracle;
the singular vectors themselves are unique only up to a phase, so they are
checked for validity (orthonormality, reconstruction of the input).

Tolerances: one-sided Jacobi is backward stable with
relative error ~ c(n) u per rotation; with u = 2^-53 and at most a few
thousand rotations per row the absolute errors stay <= 1e-12 ||A||_2:
  s:              max |s - s_ref| <= 1e-12 s_0
  reconstruction: ||u s v_dag - A||_F <= 1e-12 ||A||_F
  orthonormality: max |U^H U - I|, |V^H V - I| <= 1e-12
  truncated product vs the oracle's: <= 1e-12 relative Frobenius for the
  prescribed spectra below (relative gaps >= 5 %, so the subspace
  perturbation ||E|| / gap stays < 1e-13).
"""
import numpy as np
import pytest

import synth
from conftest import max_abs, rel_frob

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2512_23917_b200 as tci  # noqa: E402

TOL = 1e-12


@pytest.fixture(scope="module")
def ctx():
    c = tci.Context(0)
    yield c
    c.close()


def dev(x):
    t = torch.from_numpy(np.ascontiguousarray(x)) if isinstance(x, np.ndarray) else x
    return t.cuda()


def host(t):
    return t.cpu().numpy()


def as_matrix(u, s, vd, k):
    U = u.reshape(-1, u.shape[-1])
    V = vd.reshape(vd.shape[0], -1)
    return U, s, V


def check_valid(u, s, vd, a, k, full=True):
    U, s, V = as_matrix(u, s, vd, k)
    A = a.reshape(U.shape[0], V.shape[1])
    n = s.shape[0]
    assert np.all(np.diff(s) <= 0) and np.all(s >= 0), "s must be non-increasing and >= 0 (P:2036)"
    assert max_abs(U.conj().T @ U, np.eye(n)) <= TOL
    assert max_abs(V @ V.conj().T, np.eye(n)) <= TOL
    if full:
        assert rel_frob((U * s) @ V, A) <= TOL
    return U, s, V


def prescribed(m, n, sig, seed, cplx):
    """A = Q1 diag(sig) Q2^H with Haar-like unitaries (numpy QR of seeded Gaussians)."""
    rng = np.random.default_rng(seed)

    def unitary(k):
        g = rng.standard_normal((k, k)) + (1j * rng.standard_normal((k, k)) if cplx else 0)
        q, r = np.linalg.qr(g)
        return q * (np.diag(r) / np.abs(np.diag(r)))

    r = len(sig)
    return unitary(m)[:, :r] @ np.diag(sig) @ unitary(n)[:, :r].conj().T


SHAPES = [  # (tensor shape, k): several 32-row blocks, ragged tails, wide / tall / square
    ((3, 4, 12), 2),          # paper example P:2045-2051 (12 x 12)
    ((2, 3, 5, 7), 2),        # wide 6 x 35
    ((5, 7, 3), 1),           # wide 5 x 21
    ((37, 100), 1),           # wide, ragged
    ((100, 37), 1),           # tall, ragged
    ((8, 8, 2, 3, 11), 3),    # tall 128 x 33
    ((64, 64), 1),
    ((130, 96), 1),
    ((1, 9), 1),              # kappa = 1
    ((200, 2, 100), 2),       # tall 400 x 100
]


@pytest.mark.parametrize("dt", ["r64", "c128"])
@pytest.mark.parametrize("shape,k", SHAPES)
def test_svd_vs_oracle(ctx, oracle_mod, dt, shape, k):
    a = synth.random_np(shape, dt, 300 + len(shape), 1)
    u, s, vd = ctx.svd(dev(a), k)
    u, s, vd = host(u), host(s), host(vd)
    ru, rs, rvd = oracle_mod.svd(a, k)
    assert u.shape == ru.shape and s.shape == rs.shape and vd.shape == rvd.shape
    assert max_abs(s, rs) <= TOL * rs[0]
    check_valid(u, s, vd, a, k)


@pytest.mark.parametrize("dt", ["r64", "c128"])
def test_svd_prescribed_spectrum(ctx, oracle_mod, dt):
    """Known singular values (a closed form independent of LAPACK)."""
    m, n = 150, 90
    sig = np.sort(np.random.default_rng(1).uniform(0.1, 3.0, n))[::-1]
    A = prescribed(m, n, sig, 2, dt == "c128")
    if dt == "r64":
        A = A.real.copy()
    u, s, vd = ctx.svd(dev(A.reshape(10, 15, n)), 2)
    assert max_abs(host(s), sig) <= TOL * sig[0]
    check_valid(host(u), host(s), host(vd), A, 2)


@pytest.mark.parametrize("dt", ["r64", "c128"])
def test_svd_rank_deficient_tebd_like(ctx, oracle_mod, dt):
    """theta = A.B through an inner bond 24 < 48: half the singular values are
    rounding noise; the factors must still be orthonormal (R29)."""
    A = synth.random_np((24, 2, 24), dt, 41, 6)
    B = synth.random_np((24, 2, 24), dt, 41, 7)
    th = oracle_mod.contract(A, "asb", B, "btc", "astc")
    u, s, vd = ctx.svd(dev(th), 2)
    _, rs, _ = oracle_mod.svd(th, 2)
    assert max_abs(host(s), rs) <= TOL * rs[0]
    check_valid(host(u), host(s), host(vd), th, 2)


@pytest.mark.parametrize("dt", ["r64", "c128"])
def test_svd_exact_zeros_completed(ctx, dt):
    """Zero matrix and exact-rank-1 matrix with zero rows: s = 0 exactly where
    the oracle's is, and u / v_dag are completed to orthonormal sets (R29)."""
    z = np.zeros((20, 45), dtype=np.float64 if dt == "r64" else np.complex128)
    u, s, vd = ctx.svd(dev(z), 1)
    assert np.all(host(s) == 0.0)
    check_valid(host(u), host(s), host(vd), z, 1)
    x = np.zeros((40, 24), dtype=z.dtype)
    x[3, :] = np.arange(1, 25)
    x[17, :] = 2 * np.arange(1, 25)
    u, s, vd = ctx.svd(dev(x), 1)
    sh = host(s)
    assert abs(sh[0] - np.linalg.norm(x)) <= 1e-14 * sh[0] and np.all(sh[1:] <= 1e-14 * sh[0])
    check_valid(host(u), sh, host(vd), x, 1)


def test_svd_repeatable_bitwise(ctx):
    a = synth.random_np((70, 90), "c128", 5, 1)
    r1 = [host(t) for t in ctx.svd(dev(a), 1)]
    r2 = [host(t) for t in ctx.svd(dev(a), 1)]
    for x, y in zip(r1, r2):
        assert np.array_equal(x, y)


@pytest.mark.parametrize("args", [
    (3, 6, 1e-2, 1e-12),      # the paper's example
    (1, 5, 0.0, 0.0),         # overload (1): chi_max
    (2, 40, 1e-3, 0.0),       # c) grows until eps <= target
    (1, 40, 0.0, 0.9),        # a) s_min discards
    (30, 40, 0.0, 0.9),       # b) fewer than chi_min survive a): keep those
    (8, 4, 0.0, 0.0),         # chi_min > chi_max: b) wins (R31)
])
@pytest.mark.parametrize("dt", ["r64", "c128"])
def test_trunc_svd_strategy_vs_oracle(ctx, oracle_mod, dt, args):
    """Decaying prescribed spectrum sigma_i = 2^(-i/4): relative gaps 16 %, so
    chi, trunc_err and the truncated product are unique and stable."""
    m, n = 48, 40
    sig = 2.0 ** (-np.arange(n) / 4.0)
    A = prescribed(m, n, sig, 7, dt == "c128")
    if dt == "r64":
        A = A.real.copy()
    a = A.reshape(6, 8, n)
    u, s, vd, err = ctx.trunc_svd(dev(a), 2, *args)
    ru, rs, rvd, rerr = oracle_mod.trunc_svd(a, 2, *args)
    assert tuple(u.shape) == ru.shape and tuple(vd.shape) == rvd.shape and tuple(s.shape) == rs.shape
    assert max_abs(host(s), rs) <= TOL * rs[0]
    assert abs(err - rerr) <= 1e-12 * max(rerr, 1e-300) + 1e-15
    U, sh, V = check_valid(host(u), host(s), host(vd), a, 2, full=False)
    rU, _, rV = as_matrix(ru, rs, rvd, 2)
    assert rel_frob((U * sh) @ V, (rU * rs) @ rV) <= TOL


def test_trunc_svd_paper_example(ctx, oracle_mod):
    a = synth.random_np((3, 4, 12), "r64", 152, 1)
    u, s, vd, err = ctx.trunc_svd(dev(a), 2, 3, 6, 1e-2, 1e-12)
    ru, rs, rvd, rerr = oracle_mod.trunc_svd(a, 2, 3, 6, 1e-2, 1e-12)
    assert err != 0.0 and s.shape == rs.shape and 3 <= s.shape[0] <= 6
    assert abs(err - rerr) <= 1e-12 * rerr


def test_trunc_svd_fidelity_identity(ctx, oracle_mod):
    """Section III (reading R24): psi normalized, psi1 = u s v_dag
    from trunc_svd => <psi|psi1> = 1 - trunc_err, on the GPU path
    (contract for psi1 and the overlap)."""
    psi = synth.random_np((2, 2, 2, 2, 2, 2), "r64", 153, 1)
    psi = psi / np.sqrt(np.sum(psi * psi))
    d = dev(psi)
    u, s, vd, err = ctx.trunc_svd(d, 3, 1, 3, 0.0, 0.0)
    _, _, _, rerr = oracle_mod.trunc_svd(psi, 3, 1, 3, 0.0, 0.0)
    psi1 = np.einsum("ijka,a,almn->ijklmn", host(u), host(s), host(vd))   # P:333-337 (checker side)
    ovlp = float(np.sum(psi * psi1))
    assert err > 0 and abs(ovlp - (1 - err)) <= 1e-13
    assert abs(err - rerr) <= 1e-12 * rerr


@pytest.mark.parametrize("dt", ["r64", "c128"])
def test_tebd_step_theta_then_trunc_svd(ctx, oracle_mod, dt):
    """One TEBD bond update (Application A): theta = A.B.U on the
    GPU, then trunc_svd back to chi; compared with the oracle's
    theta and trunc_svd. Gate = TFIM expm(-tau h) (R25)."""
    chi = 40
    inp = synth.tebd_inputs(chi, 2, dt, 4, 0.01)
    A, B, U = (inp[k] for k in ("A", "B", "U"))
    th = ctx.tebd_theta(dev(A), "asb", dev(B), "btc", dev(U), "pqst", "apqc")
    ref_th = oracle_mod.tebd_theta(A.numpy(), B.numpy(), U.numpy())
    assert rel_frob(host(th), ref_th) <= TOL
    u, s, vd, err = ctx.trunc_svd(th, 2, 1, chi, 0.0, 1e-14)
    ru, rs, rvd, rerr = oracle_mod.trunc_svd(ref_th, 2, 1, chi, 0.0, 1e-14)
    assert s.shape == rs.shape
    assert max_abs(host(s), rs) <= TOL * rs[0]
    check_valid(host(u), host(s), host(vd), ref_th, 2, full=False)


def test_svd_errors(ctx):
    a = dev(synth.random_np((4, 5, 6), "r64", 1, 1))
    with pytest.raises(tci.TciError) as e:
        ctx.svd(a, 0)                                        # k = 0 (1 <= k < r)
    assert e.value.code == 3
    with pytest.raises(tci.TciError) as e:
        ctx.svd(a, 3)
    assert e.value.code == 3
    with pytest.raises(tci.TciError) as e:
        ctx.svd(a.float(), 1)                                # r32 unsupported
    assert e.value.code == 7
    with pytest.raises(tci.TciError) as e:
        ctx.trunc_svd(a, 1, 1, 0, 0.0, 0.0)                  # chi_max < 1
    assert e.value.code == 3
    h = ctx.handle
    u = torch.empty((4, 3), dtype=torch.float64, device="cuda")
    s = torch.empty((4,), dtype=torch.float64, device="cuda")
    v = torch.empty((4, 5, 6), dtype=torch.float64, device="cuda")
    with pytest.raises(tci.TciError) as e:                   # u has the wrong capacity
        tci.tci_svd(h, ctx.tensor(a), 1, ctx.tensor(u), ctx.tensor(s), ctx.tensor(v))
    assert e.value.code == 1


@pytest.mark.parametrize("dt", ["r64", "c128"])
def test_svd_large_vs_oracle(ctx, oracle_mod, dt):
    """1024 x 1024 (c128: the two-site DMRG matrix at chi = 512, d = 2):
    s vs LAPACK, reconstruction and orthonormality."""
    a = synth.random_np((512, 2, 2, 512), dt, 21, 2)
    u, s, vd = ctx.svd(dev(a), 2)
    _, rs, _ = oracle_mod.svd(a, 2)
    assert max_abs(host(s), rs) <= TOL * rs[0]
    check_valid(host(u), host(s), host(vd), a, 2)


def _tfim_h(g):
    X = np.array([[0.0, 1.0], [1.0, 0.0]])
    Z = np.diag([1.0, -1.0])
    I = np.eye(2)
    return (-np.kron(Z, Z) + 0.5 * g * (np.kron(X, I) + np.kron(I, X))).reshape(2, 2, 2, 2)


def test_itebd_tfim_critical_energy_on_gpu(ctx, oracle_mod):
    """Application A: imaginary-time iTEBD of the critical TFIM at
    chi = 16 with every contraction (tci_tebd_theta, tci_contract) and every
    truncated SVD (tci_trunc_svd) on the GPU; the lambda scalings are test
    glue. The energy per site matches the oracle's iTEBD run (same seed and
    schedule) to 1e-8 and the exact -4/pi (Pfeuty) to 1e-4 (SPEC acceptance 5)."""
    g, chi = 1.0, 16
    schedule = [(0.1, 200), (0.01, 300), (0.001, 300)]
    e_or, _ = oracle_mod.itebd_tfim(g, chi, schedule, lambda tau: synth.tfim_gate(tau, 1.0, g), _tfim_h(g))
    rng = np.random.default_rng(0)                       # oracle.itebd_tfim's initial product state
    GA = rng.uniform(-1, 1, (1, 2, 1))
    GB = rng.uniform(-1, 1, (1, 2, 1))
    GA, GB = dev(GA / np.linalg.norm(GA)), dev(GB / np.linalg.norm(GB))
    lA = torch.ones(1, dtype=torch.float64, device="cuda")
    lB = torch.ones(1, dtype=torch.float64, device="cuda")

    def update(GA, lA, GB, lB, U):
        A = (lB[:, None, None] * GA * lA[None, None, :]).contiguous()
        B = (GB * lB[None, None, :]).contiguous()
        th = ctx.tebd_theta(A, "asb", B, "btc", U, "pqst", "apqc")
        X, s, Y, _ = ctx.trunc_svd(th, 2, 1, chi, 0.0, 1e-12)
        s = s / torch.sqrt(torch.sum(s * s))
        return (X / lB[:, None, None]).contiguous(), s.contiguous(), (Y / lB[None, None, :]).contiguous()

    for tau, steps in schedule:
        U = dev(synth.tfim_gate(tau, 1.0, g))
        for _ in range(steps):
            GA, lA, GB = update(GA, lA, GB, lB, U)
            GB, lB, GA = update(GB, lB, GA, lA, U)
    h = dev(_tfim_h(g))

    def bond_energy(GA, lA, GB, lB):
        A = (lB[:, None, None] * GA * lA[None, None, :]).contiguous()
        B = (GB * lB[None, None, :]).contiguous()
        th = ctx.contract(A, "asb", B, "btc", "astc")
        hth = ctx.contract(th, "astc", h, "pqst", "apqc")
        return float(ctx.contract(th, "astc", hth, "astc", "")) / float(ctx.contract(th, "astc", th, "astc", ""))

    e = 0.5 * (bond_energy(GA, lA, GB, lB) + bond_energy(GB, lB, GA, lA))
    assert abs(e - e_or) <= 1e-8
    assert abs(e + 4.0 / np.pi) <= 1e-4


# ---------------------------------------------------------------------------
# zip-up MPS-MPO application (R32)
# ---------------------------------------------------------------------------

def _dense_mps(sites):
    v = sites[0].reshape(sites[0].shape[1], sites[0].shape[2])
    for A in sites[1:]:
        v = np.einsum("xa,asb->xsb", v, A).reshape(-1, A.shape[2])
    return v.reshape(-1)


def _zipup_inputs(n, chi, D, d, dt, seed):
    rng = np.random.default_rng(seed)
    bonds = [1] + [min(chi, d ** min(i + 1, n - i - 1)) for i in range(n - 1)] + [1]
    mb = [1] + [D] * (n - 1) + [1]
    cp = dt == "c128"

    def r(*sh):
        x = rng.uniform(-1, 1, sh)
        return x + 1j * rng.uniform(-1, 1, sh) if cp else x
    return [r(bonds[i], d, bonds[i + 1]) for i in range(n)], [r(mb[i], mb[i + 1], d, d) for i in range(n)]


@pytest.mark.parametrize("dt", ["r64", "c128"])
@pytest.mark.parametrize("n,chi,D,chi_max", [(6, 4, 3, 10 ** 6), (8, 8, 5, 10 ** 6), (8, 8, 5, 6), (10, 16, 5, 12)])
def test_zipup_vs_oracle(ctx, oracle_mod, dt, n, chi, D, chi_max):
    """The state itself (dense amplitudes) is unique: compared with the
    oracle's zip-up to 1e-11 relative (truncated runs: the cut singular values
    of random data are non-degenerate); trunc_err to 1e-10 relative."""
    A, W = _zipup_inputs(n, chi, D, 2, dt, 100 + n + chi_max % 97)
    B, err = ctx.mps_mpo_zipup([dev(x) for x in A], [dev(x) for x in W], chi_max)
    RB, rerr = oracle_mod.mps_mpo_zipup(A, W, chi_max)
    assert [tuple(b.shape) for b in B] == [b.shape for b in RB]
    assert rel_frob(_dense_mps([host(b) for b in B]), _dense_mps(RB)) <= 1e-11
    assert abs(err - rerr) <= 1e-10 * max(rerr, 1e-300) + 1e-26


def test_zipup_long_chain_heisenberg(ctx, oracle_mod):
    """40-site chi = 8 MPS, Heisenberg MPO (D = 5), zip-up with chi_max = 48
    >= the exact bond 40: nothing is truncated (trunc_err ~ 0), so B = H|psi>
    exactly and <psi|H|psi> (transfer chain on the host, checker side) matches
    the oracle's zip-up to 1e-10. (A heavily truncated long chain is not a
    parity case: its kept subspaces are ill-conditioned, R32.)"""
    n = 40
    rng = np.random.default_rng(5)
    bonds = [1] + [min(8, 2 ** min(i + 1, n - i - 1)) for i in range(n - 1)] + [1]
    A = [rng.uniform(-1, 1, (bonds[i], 2, bonds[i + 1])) for i in range(n)]
    Wh, lb, rb = synth.heisenberg_mpo(1.0)
    Wh = np.asarray(Wh).real
    W = [Wh[lb:lb + 1]] + [Wh] * (n - 2) + [Wh[:, rb:rb + 1]]
    B, err = ctx.mps_mpo_zipup([dev(x) for x in A], [dev(x) for x in W], 48)
    RB, rerr = oracle_mod.mps_mpo_zipup(A, W, 48)
    assert max(b.shape[2] for b in B) <= 40 and err <= 1e-20 and rerr <= 1e-20

    def overlap(bra, ket):
        E = np.ones((1, 1))
        for x, y in zip(bra, ket):
            E = np.einsum("xz,xsy,zsw->yw", E, x, y)
        return float(E[0, 0])
    got = overlap(A, [host(b) for b in B])
    ref = overlap(A, RB)
    assert abs(got - ref) <= 1e-10 * abs(ref)


@pytest.mark.parametrize("dt", ["r64", "c128"])
def test_zipup_long_chain_truncating_gap(ctx, oracle_mod, dt):
    """A TRUNCATING 40-site zip-up whose cuts are well separated (R32): psi is
    right-canonical (chi = 8), the MPO is W = I + eps H (Heisenberg, eps =
    1e-4; the last site closes both the identity and the Hamiltonian path),
    so every carry T = C A_i W_i has chi values O(1) and 4 chi values O(eps):
    chi_max = 8 cuts inside that gap. The truncated state is then unique up
    to gauge: the GPU and oracle results have fidelity 1 to 1e-12, equal
    norms and <psi|B> to 1e-11, and trunc_err (sum of discarded weights,
    ~1e-8 here) agrees to 1e-6 relative."""
    n, chi, eps = 40, 8, 1e-4
    rng = np.random.default_rng(41)
    cp = dt == "c128"
    bonds = [1] + [min(chi, 2 ** min(i + 1, n - i - 1)) for i in range(n - 1)] + [1]

    def r(*sh):
        x = rng.uniform(-1, 1, sh)
        return x + 1j * rng.uniform(-1, 1, sh) if cp else x
    A = [r(bonds[i], 2, bonds[i + 1]) for i in range(n)]
    for i in range(n - 1, 0, -1):          # right-canonical (QR from the right, input preparation)
        a, _, c = A[i].shape
        q, rr = np.linalg.qr(A[i].reshape(a, 2 * c).conj().T)
        k = q.shape[1]
        A[i] = q.conj().T.reshape(k, 2, c)
        A[i - 1] = np.einsum("xsa,ak->xsk", A[i - 1], rr.conj().T)
    A[0] /= np.linalg.norm(A[0])
    Wh, lb, rb = synth.heisenberg_mpo(1.0)
    Wh = np.asarray(Wh).real.copy()
    Wh[lb, 1:4] *= eps                      # eps S.S couplings
    Wh = Wh.astype(np.complex128) if cp else Wh
    W = [Wh[lb:lb + 1]] + [Wh] * (n - 2) + [Wh[:, rb:rb + 1] + Wh[:, lb:lb + 1]]
    B, err = ctx.mps_mpo_zipup([dev(x) for x in A], [dev(x) for x in W], chi)
    RB, rerr = oracle_mod.mps_mpo_zipup(A, W, chi)
    assert [tuple(b.shape) for b in B] == [b.shape for b in RB]
    assert 1e-12 < rerr < 1e-4
    assert abs(err - rerr) <= 1e-6 * rerr

    def overlap(bra, ket):
        E = np.ones((1, 1), dtype=np.complex128)
        for x, y in zip(bra, ket):
            E = np.einsum("xz,xsy,zsw->yw", E, np.conj(x), y)
        return complex(E[0, 0])
    Bh = [host(b) for b in B]
    gg, oo, go = overlap(Bh, Bh), overlap(RB, RB), overlap(Bh, RB)
    assert abs(abs(go) ** 2 / (gg.real * oo.real) - 1.0) <= 1e-12
    assert abs(gg - oo) <= 1e-11 * abs(oo)
    assert abs(overlap(A, Bh) - overlap(A, RB)) <= 1e-11 * abs(overlap(A, RB))


def test_trunc_svd_tebd_theta_full_size(ctx, oracle_mod):
    """Config 3 at full size (chi = 2048, d = 2, f64): theta = A.B.U on the GPU
    (4096 x 4096), trunc_svd to chi_max = 2048 on the GPU. Checked against
    LAPACK's singular values (<= 1e-12 s_0), orthonormality of u and v_dag,
    and the Eckart-Young identity ||theta - u s v_dag||_F^2 = sum_{i >= chi}
    s_i^2 (= trunc_err * ||theta||_F^2)."""
    c = synth.TEBD_CONFIG
    inp = synth.tebd_inputs(c["chi"], c["d"], c["dtype"], c["seed"], c["tau"], device="cuda")
    th = ctx.tebd_theta(inp["A"], "asb", inp["B"], "btc", inp["U"], "pqst", "apqc")
    del inp
    u, s, vd, err = ctx.trunc_svd(th, 2, 1, c["chi"], 0.0, 0.0)
    T = host(th).reshape(4096, 4096)
    rs = np.linalg.svd(T, compute_uv=False)
    chi = s.shape[0]
    assert chi == c["chi"]
    assert max_abs(host(s), rs[:chi]) <= TOL * rs[0]
    U = host(u).reshape(4096, chi)
    V = host(vd).reshape(chi, 4096)
    assert max_abs(U.T @ U, np.eye(chi)) <= TOL
    assert max_abs(V @ V.T, np.eye(chi)) <= TOL
    resid2 = np.linalg.norm(T - (U * host(s)) @ V) ** 2
    tail = float(np.sum(rs[chi:] ** 2))
    assert abs(resid2 - tail) <= 1e-9 * tail + 1e-12 * float(np.sum(rs ** 2))
    assert abs(err - tail / float(np.sum(rs ** 2))) <= 1e-9 * err
