"""Pins for the CPU oracle (-m "not gpu").

Each test checks the oracle against something other than itself: values the
paper prints (tests/golden/paper_examples.json), closed forms
(tests/golden/closed_forms.json), library routines that reduce to the same
definition (numpy.einsum / matmul / transpose), exact rational arithmetic,
brute-force pure-Python sums, invariances and the Higham error bound. DESIGN.md
section "Pins" maps every oracle function to the tests here.
"""
import itertools
import math
import string
from fractions import Fraction

import numpy as np
import pytest

import synth
from conftest import golden, max_abs, rel_frob


# ---------------------------------------------------------------------------
# helpers independent of the oracle
# ---------------------------------------------------------------------------

def brute_contract(A, la, B, lb, lc):
    """Eq. (3) by a pure-Python sum over all label assignments (tiny only)."""
    dims = {}
    for l, d in zip(la, A.shape):
        dims[l] = d
    for l, d in zip(lb, B.shape):
        dims[l] = d
    summed = [l for l in la if l in lb and l not in lc]
    out = np.zeros([dims[l] for l in lc], dtype=np.result_type(A, B))
    for oc in itertools.product(*[range(dims[l]) for l in lc]):
        asg = dict(zip(lc, oc))
        acc = 0
        for sc in itertools.product(*[range(dims[l]) for l in summed]):
            asg.update(zip(summed, sc))
            acc += A[tuple(asg[l] for l in la)] * B[tuple(asg[l] for l in lb)]
        out[oc] = acc
    return out


def rnd(shape, seed, tid=1, cplx=False):
    return synth.random_np(shape, "c128" if cplx else "r64", seed, tid)


# ---------------------------------------------------------------------------
# paper worked examples
# ---------------------------------------------------------------------------

def test_paper_contract_example(oracle_mod):
    g = golden("paper_examples.json")["contract_shape"]
    a = rnd(g["a_shape"], 11, 1)
    b = rnd(g["b_shape"], 11, 2)
    c_list = oracle_mod.contract(a, g["labels_list"]["a"], b, g["labels_list"]["b"], g["labels_list"]["c"])
    c_str = oracle_mod.contract(a, g["labels_str"]["a"], b, g["labels_str"]["b"], g["labels_str"]["c"])
    assert list(c_list.shape) == g["c_shape"]
    assert np.array_equal(c_list, c_str)           # list and string APIs equivalent
    assert rel_frob(c_str, np.einsum("ijk,kjl->li", a, b)) < 1e-15
    assert rel_frob(c_str, brute_contract(a, "ijk", b, "kjl", "li")) < 1e-15


def test_paper_transpose_example(oracle_mod):
    g = golden("paper_examples.json")["transpose"]
    a = rnd(g["a_shape"], 12)
    a2 = oracle_mod.permute(a, g["inplace_order"])
    assert a[tuple(g["elem_before"])] == a2[tuple(g["elem_after"])]
    b = oracle_mod.permute(a2, g["out_order"])
    assert list(b.shape) == g["out_shape_after_inplace"]


def test_paper_reshape_example(oracle_mod):
    g = golden("paper_examples.json")["reshape"]
    a = rnd(g["a_shape"], 13)
    r = oracle_mod.reshape(a, g["inplace_shape"])
    assert list(r.shape) == g["inplace_shape"]
    assert np.array_equal(r.reshape(-1), a.reshape(-1))      # element order preserved
    r2 = oracle_mod.reshape(r, g["out_shape"])
    assert list(r2.shape) == g["out_shape"]
    with pytest.raises(oracle_mod.OracleError) as e:
        oracle_mod.reshape(a, [5, 5])
    assert e.value.code == 1


def test_paper_scenario_shapes(oracle_mod):
    for i, case in enumerate(golden("paper_examples.json")["scenario_shapes"]["cases"]):
        a = rnd(case["a"], 20 + i, 1)
        b = rnd(case["b"], 20 + i, 2)
        c = oracle_mod.contract(a, case["la"], b, case["lb"], case["lc"])
        assert list(c.shape) == case["c"]
        assert c.size == max(1, int(np.prod(case["c"])))


def test_scenario_overlap_identity(oracle_mod):
    """Section III: truncated SVD of a normalized 6-qubit state,
    psi1 = u.s.vt by two contracts (the 2nd aliasing psi1), overlap by a full
    contraction. Exact identity: <psi|psi1> = 1 - eps with eps of P:2088-2090
    (reading R24 on the fidelity line P:351)."""
    psi = rnd((2,) * 6, 31)
    psi /= np.linalg.norm(psi)
    m = psi.reshape(8, 8)
    U, s, Vt = np.linalg.svd(m)
    chi = 2
    eps = float(np.sum(s[chi:] ** 2) / np.sum(s ** 2))
    u = U[:, :chi].reshape(2, 2, 2, chi)
    S = np.diag(s[:chi])
    vt = Vt[:chi, :].reshape(chi, 2, 2, 2)
    psi1 = oracle_mod.contract(u, "ijkl", S, "lm", "ijkm")
    psi1 = oracle_mod.contract(psi1, "ijkl", vt, "lmno", "ijkmno")
    ovlp = oracle_mod.contract(psi, "ijklmn", psi1, "ijklmn", "")
    assert ovlp.shape == ()
    assert abs(float(ovlp) - (1.0 - eps)) < 1e-14


def test_frobenius_and_close_examples():
    g = golden("paper_examples.json")
    assert rel_frob(np.eye(3), np.zeros((3, 3))) == pytest.approx(g["frobenius_norm_eye3"]["value"], abs=0)
    c = g["close"]
    A = np.eye(3)
    B = A.copy()
    B[tuple(c["perturb_coor"])] = c["perturb_value"]
    assert not (max_abs(A, B) <= c["eps_false"])
    assert max_abs(A, B) <= c["eps_true"]


# ---------------------------------------------------------------------------
# reductions to library routines / brute force
# ---------------------------------------------------------------------------

def test_matmul_special_case(oracle_mod):
    """|I|=|J|=|S|=1 is matrix multiplication."""
    for cplx in (False, True):
        a = rnd((37, 64), 40, 1, cplx)
        b = rnd((64, 19), 40, 2, cplx)
        assert rel_frob(oracle_mod.contract(a, "ik", b, "kj", "ij"), a @ b) < 1e-15
        assert rel_frob(oracle_mod.contract(a, "ik", b, "kj", "ji"), (a @ b).T) < 1e-15


def test_eq4_example(oracle_mod):
    """C_ilm = sum_jk A_ijk B_jklm (Eq. (4))."""
    A = rnd((3, 4, 5), 41, 1)
    B = rnd((4, 5, 2, 3), 41, 2)
    C = oracle_mod.contract(A, "ijk", B, "jklm", "ilm")
    assert rel_frob(C, brute_contract(A, "ijk", B, "jklm", "ilm")) < 1e-15
    assert rel_frob(C, np.einsum("ijk,jklm->ilm", A, B)) < 1e-15


def _random_instance(rng, cplx):
    ra = int(rng.integers(1, 5))
    rb = int(rng.integers(1, 5))
    nc = int(rng.integers(0, min(ra, rb) + 1))
    letters = list(string.ascii_letters)
    rng.shuffle(letters)
    shared = letters[:nc]
    fa = letters[nc:nc + ra - nc]
    fb = letters[ra:ra + rb - nc]
    la = shared + fa
    lb = shared + fb
    rng.shuffle(la)
    rng.shuffle(lb)
    lc = fa + fb
    rng.shuffle(lc)
    dims = {l: int(rng.integers(1, 6)) for l in la + lb}
    seed = int(rng.integers(1, 1 << 30))
    A = rnd([dims[l] for l in la], seed, 1, cplx)
    B = rnd([dims[l] for l in lb], seed, 2, cplx)
    return A, "".join(la), B, "".join(lb), "".join(lc)


@pytest.mark.parametrize("cplx", [False, True])
def test_random_sweep_vs_einsum(oracle_mod, cplx):
    """SPEC.md:381 / SURVEY 8(c).5: 200 random contracts, order <= 4, dims <= 5."""
    rng = np.random.default_rng(1234 + cplx)
    for _ in range(100):
        A, la, B, lb, lc = _random_instance(rng, cplx)
        C = oracle_mod.contract(A, la, B, lb, lc)
        ref = np.einsum(f"{la},{lb}->{lc}", A, B)
        assert rel_frob(C, ref) <= 1e-12, (la, lb, lc)


def test_random_small_vs_bruteforce(oracle_mod):
    rng = np.random.default_rng(99)
    for k in range(30):
        A, la, B, lb, lc = _random_instance(rng, k % 2 == 1)
        if A.size * B.size > 4000:
            continue
        C = oracle_mod.contract(A, la, B, lb, lc)
        assert rel_frob(C, brute_contract(A, la, B, lb, lc)) <= 1e-14


def test_exact_rational_within_higham_bound(oracle_mod):
    """Per element |C - C_exact| <= gamma_K (|A|.|B|), gamma_K = Ku/(1-Ku),
    with C_exact summed in exact rationals (the inputs are dyadic rationals)."""
    A = rnd((6, 50, 4), 51, 1)
    B = rnd((4, 50, 7), 51, 2)
    C = oracle_mod.contract(A, "iks", B, "skj", "ij")
    Cabs = oracle_mod.contract_abs(A, "iks", B, "skj", "ij")
    K = 50 * 4
    u = 2.0 ** -53
    gam = K * u / (1 - K * u)
    for i in range(6):
        for j in range(7):
            exact = sum(Fraction(A[i, k, s]) * Fraction(B[s, k, j]) for k in range(50) for s in range(4))
            err = abs(Fraction(C[i, j]) - exact)
            assert err <= Fraction(gam) * Fraction(Cabs[i, j])
            # |A|.|B| itself equals the exact sum of moduli within the same bound
            exa = sum(abs(Fraction(A[i, k, s]) * Fraction(B[s, k, j])) for k in range(50) for s in range(4))
            assert abs(Fraction(Cabs[i, j]) - exa) <= Fraction(gam) * exa


# ---------------------------------------------------------------------------
# exact identities and invariances
# ---------------------------------------------------------------------------

def test_identity_contraction_bitwise(oracle_mod):
    for cplx in (False, True):
        a = rnd((13, 9), 60, 1, cplx)
        I = np.eye(9, dtype=a.dtype)
        assert np.array_equal(oracle_mod.contract(a, "ij", I, "jk", "ik"), a)
        I2 = np.eye(13, dtype=a.dtype)
        assert np.array_equal(oracle_mod.contract(I2, "ki", a, "ij", "kj"), a)


def test_trace(oracle_mod):
    a = rnd((17, 17), 61)
    t = oracle_mod.contract(a, "ij", np.eye(17), "ij", "")
    assert abs(float(t) - np.trace(a)) <= 1e-15 * np.sum(np.abs(np.diag(a)))


def test_outer_product_and_scalars(oracle_mod):
    a = rnd((3, 4), 62, 1)
    b = rnd((5,), 62, 2)
    c = oracle_mod.contract(a, "ij", b, "k", "kji")
    assert np.array_equal(c, np.einsum("ij,k->kji", a, b))   # one product per element: exact
    s = np.array(2.5)
    assert np.array_equal(oracle_mod.contract(s, "", a, "ij", "ji"), (2.5 * a).T)
    d = oracle_mod.contract(s, "", np.array(-3.0), "", "")
    assert d.shape == () and float(d) == -7.5


def test_permute_vs_numpy_and_roundtrip(oracle_mod):
    rng = np.random.default_rng(5)
    for n in range(0, 7):
        shape = tuple(int(x) for x in rng.integers(1, 5, size=n))
        for cplx in (False, True):
            a = rnd(shape, 70 + n, 1, cplx)
            perm = list(rng.permutation(n))
            b = oracle_mod.permute(a, perm)
            assert np.array_equal(b, np.transpose(a, perm))     # Eq. (1) == NumPy axes semantics
            inv = list(np.argsort(perm))
            assert np.array_equal(oracle_mod.permute(b, inv), a)


def test_relabel_invariance_bitwise(oracle_mod):
    A = rnd((4, 6, 5), 80, 1, True)
    B = rnd((5, 6, 3), 80, 2, True)
    c1 = oracle_mod.contract(A, "ikl", B, "lkj", "ji")
    c2 = oracle_mod.contract(A, [7, -3, 100], B, [100, -3, 42], [42, 7])
    assert np.array_equal(c1, c2)


def test_operand_swap_and_leg_permutation(oracle_mod):
    A = rnd((4, 6, 5), 81, 1)
    B = rnd((5, 6, 3), 81, 2)
    c1 = oracle_mod.contract(A, "ikl", B, "lkj", "ij")
    c2 = oracle_mod.contract(B, "lkj", A, "ikl", "ij")
    c3 = oracle_mod.contract(np.transpose(A, (2, 0, 1)).copy(), "lik", B, "lkj", "ij")
    assert rel_frob(c2, c1) <= 1e-15 and rel_frob(c3, c1) <= 1e-15


def test_associativity(oracle_mod):
    A = rnd((6, 7), 82, 1)
    B = rnd((7, 8, 5), 82, 2)
    C = rnd((5, 9), 82, 3)
    l = oracle_mod.contract(oracle_mod.contract(A, "ij", B, "jkl", "ikl"), "ikl", C, "lm", "ikm")
    r = oracle_mod.contract(A, "ij", oracle_mod.contract(B, "jkl", C, "lm", "jkm"), "jkm", "ikm")
    assert rel_frob(l, r) <= 1e-11


def test_thread_count_bitwise(oracle_mod):
    A = rnd((40, 33, 20), 83, 1, True)
    B = rnd((20, 33, 50), 83, 2, True)
    c1 = oracle_mod.contract(A, "iks", B, "skj", "ji", threads=1)
    c8 = oracle_mod.contract(A, "iks", B, "skj", "ji", threads=8)
    assert np.array_equal(c1, c8)


# ---------------------------------------------------------------------------
# error kinds
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("la,lb,lc,code", [
    ("iij", "jk", "ik", 4),      # repeated label in one operand
    ("ij", "jk", "ijk", 4),      # label in all three lists (R3)
    ("ijm", "jk", "ik", 4),      # label in one input, not in gamma (R4)
    ("ij", "jk", "ikz", 4),      # gamma label absent (R5)
    ("ij", "jk", "ii", 4),       # repeated output label
])
def test_label_errors(oracle_mod, la, lb, lc, code):
    a = np.zeros([2] * len(la))
    b = np.zeros([2] * len(lb))
    with pytest.raises(oracle_mod.OracleError) as e:
        oracle_mod.contract(a, la, b, lb, lc)
    assert e.value.code == code


def test_shape_and_order_errors(oracle_mod):
    with pytest.raises(oracle_mod.OracleError) as e:
        oracle_mod.contract(np.zeros((2, 3)), "ij", np.zeros((4, 5)), "jk", "ik")
    assert e.value.code == 1
    with pytest.raises(oracle_mod.OracleError) as e:
        oracle_mod.contract(np.zeros((2, 3)), "ijk", np.zeros((3, 5)), "jk", "ik")
    assert e.value.code == 2
    with pytest.raises(oracle_mod.OracleError) as e:
        oracle_mod.contract(np.zeros([1] * 17), list(range(17)), np.zeros(1), [0], list(range(1, 17)))
    assert e.value.code == 7


# ---------------------------------------------------------------------------
# chains: H_eff, TEBD, MPS (definitions DESIGN.md R15-R18)
# ---------------------------------------------------------------------------

def brute_heff(L, W1, W2, R, psi):
    """Single 7-index sum, pure Python (SURVEY 8(c).5 brute force)."""
    chi_l, D, chi_lo = L.shape
    _, d, _, chi_r = psi.shape
    D2 = W1.shape[1]
    D3 = W2.shape[1]
    chi_ro = R.shape[2]
    out = np.zeros((chi_lo, d, d, chi_ro), dtype=np.result_type(L, psi))
    for b, p, q, e in itertools.product(range(chi_lo), range(d), range(d), range(chi_ro)):
        acc = 0
        for a, s, t, c, w, v, x in itertools.product(range(chi_l), range(d), range(d), range(chi_r),
                                                     range(D), range(D2), range(D3)):
            acc += L[a, w, b] * psi[a, s, t, c] * W1[w, v, s, p] * W2[v, x, t, q] * R[c, x, e]
        out[b, p, q, e] = acc
    return out


@pytest.mark.parametrize("chi", [1, 2, 3])
def test_heff_vs_bruteforce(oracle_mod, chi):
    inp = {k: v.numpy() for k, v in synth.heff_inputs(chi, 2, 3, "c128", 90 + chi, "random").items()}
    o = oracle_mod.heff(inp["L"], inp["W1"], inp["W2"], inp["R"], inp["psi"])
    assert rel_frob(o, brute_heff(inp["L"], inp["W1"], inp["W2"], inp["R"], inp["psi"])) <= 1e-14


def test_heff_order_invariance_and_einsum(oracle_mod):
    inp = {k: v.numpy() for k, v in synth.heff_inputs(12, 2, 5, "c128", 95, "heisenberg").items()}
    args = (inp["L"], inp["W1"], inp["W2"], inp["R"], inp["psi"])
    o1 = oracle_mod.heff(*args)
    o2 = oracle_mod.heff_alt(*args)
    assert rel_frob(o1, o2) <= 1e-12
    ref = np.einsum("awb,wvsp,vxtq,cxe,astc->bpqe", *args, optimize=True)
    assert rel_frob(o1, ref) <= 1e-12


def test_heff_rows_bitwise(oracle_mod):
    inp = {k: v.numpy() for k, v in synth.heff_inputs(10, 2, 5, "c128", 96, "heisenberg").items()}
    args = (inp["L"], inp["W1"], inp["W2"], inp["R"], inp["psi"])
    full = oracle_mod.heff(*args)
    rows = [0, 3, 9]
    assert np.array_equal(oracle_mod.heff_rows(*args, rows), full[rows])


@pytest.mark.parametrize("side", [0, 1])
def test_env_rows_bitwise(oracle_mod, side):
    """env_rows (the sampled checker of the full-size environment tests) equals
    the matching rows of the full env_left / env_right bitwise: slicing the
    ket's outgoing bond is a free leg of every pairwise contract in the chain,
    so no element's summation order changes. env_left/env_right themselves
    are pinned against dense operators and closed forms below."""
    rng = np.random.default_rng(31 + side)
    chi, d, D, chi2 = 5, 2, 3, 7

    def c(*s):
        return rng.standard_normal(s) + 1j * rng.standard_normal(s)
    W = c(D, D, d, d)
    if side == 0:
        E, ket, bra = c(chi, D, chi), c(chi, d, chi2), c(chi, d, chi2)
        full = oracle_mod.env_left(E, ket, W, bra)
    else:
        E, ket, bra = c(chi, D, chi), c(chi2, d, chi), c(chi2, d, chi)
        full = oracle_mod.env_right(E, ket, W, bra)
    rows = [0, 2, chi2 - 1]
    got = oracle_mod.env_rows(side, E, ket, W, bra, rows)
    assert got.shape == (len(rows),) + full.shape[1:]
    assert np.array_equal(got, full[rows])


def test_heisenberg_singlet(oracle_mod):
    g = golden("closed_forms.json")["heisenberg_two_site"]
    W, lb, rb = synth.heisenberg_mpo(1.0)
    L = synth.boundary_env(5, lb)
    R = synth.boundary_env(5, rb)
    H = oracle_mod.heff_dense(L, W, W, R, (1, 2, 2, 1))
    assert np.allclose(H, H.conj().T, atol=0)
    ev = np.sort(np.linalg.eigvalsh(H))
    assert np.max(np.abs(ev - np.array(g["eigenvalues"]))) < 1e-14


def _jw_dense_hubbard(t, U):
    """Global Jordan-Wigner Hubbard on modes (1up, 1dn, 2up, 2dn), 16x16, in the
    product basis of local states |0>,|up>,|dn>,|updn> (index n_up + 2 n_dn)."""
    a = np.array([[0.0, 1.0], [0.0, 0.0]])   # mode annihilator, basis (empty, occupied)
    Zs = np.diag([1.0, -1.0])
    I2 = np.eye(2)

    def mode_op(j):
        ops = [Zs] * j + [a] + [I2] * (3 - j)
        m = ops[0]
        for o in ops[1:]:
            m = np.kron(m, o)
        return m
    c = [mode_op(j) for j in range(4)]
    n = [ci.T @ ci for ci in c]
    H = U * (n[0] @ n[1] + n[2] @ n[3])
    for s in (0, 1):
        H += -t * (c[s].T @ c[2 + s] + c[2 + s].T @ c[s])
    # reorder: mode basis index = 8 n1u + 4 n1d + 2 n2u + n2d -> local (n_up + 2 n_dn)
    perm = np.zeros(16, dtype=int)
    for n1u, n1d, n2u, n2d in itertools.product((0, 1), repeat=4):
        mode_idx = 8 * n1u + 4 * n1d + 2 * n2u + n2d
        loc_idx = (n1u + 2 * n1d) * 4 + (n2u + 2 * n2d)
        perm[loc_idx] = mode_idx
    return H[np.ix_(perm, perm)], n


def test_hubbard_two_site_matches_global_jw(oracle_mod):
    g = golden("closed_forms.json")["hubbard_two_site_N2"]
    W, lb, rb = synth.hubbard_mpo(g["t"], g["U"])
    L = synth.boundary_env(6, lb)
    R = synth.boundary_env(6, rb)
    H = oracle_mod.heff_dense(L, W, W, R, (1, 4, 4, 1))
    Hjw, n = _jw_dense_hubbard(g["t"], g["U"])
    assert np.max(np.abs(H - Hjw)) < 1e-15
    # N = 2 sector ground energy (closed form)
    nloc = np.array([0, 1, 1, 2])
    N = (nloc[:, None] + nloc[None, :]).reshape(-1)
    sector = np.where(N == 2)[0]
    e0 = np.linalg.eigvalsh(H[np.ix_(sector, sector)].real)[0]
    assert abs(e0 - g["E0"]) < 1e-13


def test_tebd_gate_identity_and_g0(oracle_mod):
    A = rnd((6, 2, 7), 100, 6)
    B = rnd((7, 2, 5), 100, 7)
    U0 = synth.tfim_gate(0.0)
    AB = oracle_mod.contract(A, "asb", B, "btc", "astc")
    th = oracle_mod.tebd_theta(A, B, U0)
    assert np.array_equal(th, AB)        # identity gate: exact (x*1 + y*0)
    g0 = golden("closed_forms.json")["tfim_gate_g0"]
    Ug = synth.tfim_gate(g0["tau"], g0["J"], 0.0).reshape(4, 4)
    assert np.max(np.abs(Ug - np.diag(g0["diag"]))) < 1e-15
    U = synth.tfim_gate(0.01)
    th = oracle_mod.tebd_theta(A, B, U)
    assert rel_frob(th, np.einsum("asb,btc,pqst->apqc", A, B, U)) <= 1e-14
    # physical-first layout variant (ii) gives the same tensor
    th2 = oracle_mod.tebd_theta(np.transpose(A, (1, 0, 2)).copy(), np.transpose(B, (1, 0, 2)).copy(), U,
                                la="sab", lb="tbc", lu="pqst", lt="paqc")
    assert rel_frob(np.transpose(th2, (1, 0, 2, 3)), th) <= 1e-15


def test_mps_product_state_norm_exact(oracle_mod):
    sites = synth.product_state_sites(10)
    assert float(oracle_mod.mps_norm2(sites)[0, 0]) == golden("closed_forms.json")["product_state_norm"]["value"]


def test_mps_norm_vs_dense_state(oracle_mod):
    sites = synth.mps_sites(synth.MPS_BONDS_CFG1, 2, 1)
    psi = sites[0]
    for s in sites[1:]:
        psi = np.tensordot(psi, s, axes=([psi.ndim - 1], [0]))
    psi = psi.reshape(-1)
    assert psi.size == 1024
    n2 = float(oracle_mod.mps_norm2(sites)[0, 0])
    assert abs(n2 - float(psi @ psi)) <= 1e-13 * abs(float(psi @ psi))
    phi_sites = synth.mps_sites(synth.MPS_BONDS_CFG1, 2, 2)
    phi = phi_sites[0]
    for s in phi_sites[1:]:
        phi = np.tensordot(phi, s, axes=([phi.ndim - 1], [0]))
    ov = float(oracle_mod.mps_overlap(phi_sites, sites)[0, 0])
    assert abs(ov - float(phi.reshape(-1) @ psi)) <= 1e-12 * np.linalg.norm(phi) * np.linalg.norm(psi)


def test_mps_mpo_apply(oracle_mod):
    A = rnd((4, 2, 6), 110, 1, True)
    I = np.eye(2, dtype=np.complex128).reshape(1, 1, 2, 2)
    assert np.array_equal(oracle_mod.mps_mpo_apply(A, I), A)      # identity MPO: exact
    W = rnd((3, 3, 2, 2), 110, 2, True)
    Bp = oracle_mod.mps_mpo_apply(A, W)
    ref = np.einsum("asb,wvst->awtbv", A, W).reshape(12, 2, 18)
    assert Bp.shape == (12, 2, 18) and rel_frob(Bp, ref) <= 1e-15


# ---------------------------------------------------------------------------
# generator
# ---------------------------------------------------------------------------

def test_generator_matches_reference():
    for seed, tid in [(0, 1), (3, 2), (6, 5), (123456789, 105)]:
        d = synth.uniform_draws(seed, tid, 2000).numpy()
        for i in (0, 1, 2, 17, 999, 1999):
            assert d[i] == synth.uniform_ref(seed, tid, i)
        assert d.min() >= -1.0 and d.max() < 1.0
        assert not np.any(np.signbit(d) & (d == 0))
        # chunking does not change values
        d2 = synth.uniform_draws(seed, tid, 2000, chunk=77).numpy()
        assert np.array_equal(d, d2)


def test_vector_function_examples(oracle_mod):
    """App. C examples: norm(eye(3)) = sqrt(3); normalize gives
    norm 1; scale(eye(3), 3)[2,2] = 3 and scale(., -2) = -6
    (P:1796-1806); linear_combine with default coefficients is the plain sum
    (P:1993)."""
    g = golden("paper_examples.json")
    assert oracle_mod.norm(np.eye(3)) == g["frobenius_norm_eye3"]["value"]
    a = rnd((3, 4, 2), 120)
    assert abs(oracle_mod.norm(a / oracle_mod.norm(a)) - 1.0) < 1e-15
    e3 = oracle_mod.scale(np.eye(3), 3.0)
    assert e3[2, 2] == 3.0 and oracle_mod.scale(e3, -2.0)[2, 2] == -6.0
    b, c = rnd((3, 4, 2), 121), rnd((3, 4, 2), 122)
    assert np.array_equal(oracle_mod.linear_combine([a, b, c]), a + b + c)
    lc = oracle_mod.linear_combine([a, b, c], [1.0, 2.0, 3.0])
    assert np.max(np.abs(lc - (a + 2 * b + 3 * c))) < 1e-15
    z = rnd((5, 7), 123, 1, True)
    assert abs(oracle_mod.inner(z, z) - oracle_mod.norm(z) ** 2) < 1e-13
    assert abs(oracle_mod.inner(z, z, conj_a=False) - complex(oracle_mod.contract(z, "ij", z, "ij", ""))) < 1e-13


# ---------------------------------------------------------------------------
# cplx_conj and environment updates (R28)
# ---------------------------------------------------------------------------

def test_cplx_conj_identities(oracle_mod):
    a = rnd((3, 2, 4), 71, cplx=True)
    c = oracle_mod.cplx_conj(a)
    # the paper's example: std::conj(el1) == el2 at {0,0,0}
    assert c[0, 0, 0] == np.conj(a[0, 0, 0])
    # involution, bitwise; a + conj(a) is real (exactly 2 Re a); a conj(a) = |a|^2 >= 0
    assert np.array_equal(oracle_mod.cplx_conj(c), a)
    s = a + c
    assert np.all(s.imag == 0) and np.array_equal(s.real, 2 * a.real)
    p = a * c
    assert np.all(p.real >= 0) and np.max(np.abs(p.imag)) <= 1e-15 * np.max(p.real)
    # real data: a deep copy
    r = rnd((5, 3), 72)
    rc = oracle_mod.cplx_conj(r)
    assert np.array_equal(rc, r) and rc is not r and not np.shares_memory(rc, r)


_SX = np.array([[0, 0.5], [0.5, 0]], dtype=np.complex128)
_SY = np.array([[0, -0.5j], [0.5j, 0]], dtype=np.complex128)
_SZ = np.diag([0.5, -0.5]).astype(np.complex128)


def _dense_heisenberg(n):
    """H = sum_i S_i . S_{i+1} from Kronecker products of the spin matrices
    (site 0 = most significant index, basis (up, dn)) -- independent of the MPO."""
    H = np.zeros((2 ** n, 2 ** n), dtype=np.complex128)
    for i in range(n - 1):
        for op in (_SX, _SY, _SZ):
            H += np.kron(np.kron(np.eye(2 ** i), np.kron(op, op)), np.eye(2 ** (n - i - 2)))
    return H


def _dense_state(sites):
    v = sites[0][0]                                  # [d, chi]
    for A in sites[1:]:
        v = np.tensordot(v, A, axes=([-1], [0]))
    return v[..., 0].reshape(-1)


def _env_expectation(oracle_mod, sites, W, lb, rb, bra=None, side=0):
    D = W.shape[0]
    bra = sites if bra is None else bra
    if side == 0:
        E = synth.boundary_env(D, lb)
        for A, B in zip(sites, bra):
            E = oracle_mod.env_left(E, A, W, B)
        return E[0, rb, 0]
    E = synth.boundary_env(D, rb)
    for A, B in zip(reversed(sites), reversed(bra)):
        E = oracle_mod.env_right(E, A, W, B)
    return E[0, lb, 0]


@pytest.mark.parametrize("side", [0, 1])
def test_env_expectation_vs_dense_hamiltonian(oracle_mod, side):
    n, bonds = 6, [1, 2, 4, 5, 4, 2, 1]
    ket = [rnd((bonds[i], 2, bonds[i + 1]), 80 + i, cplx=True) for i in range(n)]
    bra = [rnd((bonds[i], 2, bonds[i + 1]), 90 + i, cplx=True) for i in range(n)]
    W, lb, rb = synth.heisenberg_mpo()
    H = _dense_heisenberg(n)
    psi, phi = _dense_state(ket), _dense_state(bra)
    ref = np.vdot(psi, H @ psi)
    got = _env_expectation(oracle_mod, ket, W, lb, rb, side=side)
    assert abs(got - ref) <= 1e-12 * abs(ref)
    assert abs(got.imag) <= 1e-12 * abs(ref)            # Hermitian H: real expectation
    ref2 = np.vdot(phi, H @ psi)                         # <phi|H|psi>, bra conjugated
    got2 = _env_expectation(oracle_mod, ket, W, lb, rb, bra=bra, side=side)
    assert abs(got2 - ref2) <= 1e-12 * abs(ref2)


def test_env_product_state_closed_form(oracle_mod):
    """Product state of spinors u_i: <S_i . S_j> = n_i . n_j / 4 with the Bloch
    vectors n = (2 Re u0* u1, 2 Im u0* u1, |u0|^2 - |u1|^2) (normalised u)."""
    rng = np.random.default_rng(7)
    n = 9
    u = rng.standard_normal((n, 2)) + 1j * rng.standard_normal((n, 2))
    u /= np.linalg.norm(u, axis=1, keepdims=True)
    sites = [x.reshape(1, 2, 1) for x in u]
    bloch = np.stack([2 * (np.conj(u[:, 0]) * u[:, 1]).real, 2 * (np.conj(u[:, 0]) * u[:, 1]).imag,
                      np.abs(u[:, 0]) ** 2 - np.abs(u[:, 1]) ** 2], axis=1)
    closed = float(np.sum(bloch[:-1] * bloch[1:]) / 4)
    W, lb, rb = synth.heisenberg_mpo()
    for side in (0, 1):
        got = _env_expectation(oracle_mod, sites, W, lb, rb, side=side)
        assert abs(got - closed) <= 1e-14 and abs(got.imag) <= 1e-15
    # Neel state: -(n-1)/4 exactly
    neel = synth.product_state_sites(n)
    assert _env_expectation(oracle_mod, neel, W, lb, rb) == -(n - 1) / 4


def test_env_left_isometry_maps_identity_to_identity(oracle_mod):
    rng = np.random.default_rng(11)
    chi, d, chi2 = 6, 3, 9
    X = rng.standard_normal((chi * d, chi2)) + 1j * rng.standard_normal((chi * d, chi2))
    Q, _ = np.linalg.qr(X)                                # Q^H Q = I
    A = Q.reshape(chi, d, chi2)
    I_mpo = np.eye(d, dtype=np.complex128).reshape(1, 1, d, d)
    E = np.eye(chi, dtype=np.complex128).reshape(chi, 1, chi)
    out = oracle_mod.env_left(E, A, I_mpo)
    assert max_abs(out.reshape(chi2, chi2), np.eye(chi2)) <= 1e-14
    # the right version with a right isometry (rows orthonormal)
    B = np.ascontiguousarray(Q.T).reshape(chi2, d, chi)
    R = np.eye(chi, dtype=np.complex128).reshape(chi, 1, chi)
    outr = oracle_mod.env_right(R, B, I_mpo)
    # sum_{s,c} B[a,s,c] conj(B[f,s,c]) = (Q^T conj(Q))[a,f] = conj(Q^H Q)^T = I
    assert max_abs(outr.reshape(chi2, chi2), np.eye(chi2)) <= 1e-14


def test_env_norm_equals_transfer_chain_cfg1(oracle_mod):
    """<psi|psi> through identity-MPO environments equals config 1's transfer
    norm (real data: the bilinear chain of R17 is the norm)."""
    sites = synth.mps_sites(synth.MPS_BONDS_CFG1, 2, 1, "r64")
    I_mpo = np.eye(2).reshape(1, 1, 2, 2)
    E = np.ones((1, 1, 1))
    for A in sites:
        E = oracle_mod.env_left(E, A, I_mpo)
    ref = oracle_mod.mps_norm2(sites)[0, 0]
    assert abs(E[0, 0, 0] - ref) <= 1e-13 * abs(ref)
    psi = _dense_state(sites)
    assert abs(E[0, 0, 0] - np.dot(psi, psi)) <= 1e-12 * abs(ref)


@pytest.mark.parametrize("side", [0, 1])
def test_env_random_mpo_vs_dense_operator(oracle_mod, side):
    """A random complex (non-Hermitian) MPO: <phi|O|psi> through environments
    equals phi^H O psi with O[(t..), (s..)] = sum_w prod_i W_i[w_i, w_i+1, s_i, t_i]
    assembled here with numpy (catches s/t or bra/ket role swaps that the
    symmetric Heisenberg MPO cannot)."""
    n, d, D = 4, 2, 3
    bonds = [1, 2, 3, 2, 1]
    ket = [rnd((bonds[i], d, bonds[i + 1]), 120 + i, cplx=True) for i in range(n)]
    bra = [rnd((bonds[i], d, bonds[i + 1]), 130 + i, cplx=True) for i in range(n)]
    W = rnd((D, D, d, d), 140, cplx=True)
    lb, rb = 1, 2
    O = np.einsum("s,t->ts", np.ones(1), np.ones(1)).astype(np.complex128)   # 1x1 start
    vec = np.zeros(D, dtype=np.complex128)
    vec[lb] = 1
    # M[w][(t..), (s..)] accumulated site by site
    M = [vec[w] * np.ones((1, 1), dtype=np.complex128) for w in range(D)]
    for _ in range(n):
        M = [sum(np.kron(M[w], W[w, v].T) for w in range(D)) for v in range(D)]
    O = M[rb]
    psi, phi = _dense_state(ket), _dense_state(bra)
    ref = np.vdot(phi, O @ psi)
    got = _env_expectation(oracle_mod, ket, W, lb, rb, bra=bra, side=side)
    assert abs(got - ref) <= 1e-12 * abs(ref)


# ---------------------------------------------------------------------------
# svd / trunc_svd, SURVEY 8(f2)
# ---------------------------------------------------------------------------

def _unitary(n, seed):
    rng = np.random.default_rng(seed)
    q, r = np.linalg.qr(rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n)))
    return q * (np.diag(r) / np.abs(np.diag(r)))


def test_svd_paper_example_shapes(oracle_mod):
    a = rnd((3, 4, 12), 150, cplx=True)
    u, s, vd = oracle_mod.svd(a, 2)
    assert u.shape == (3, 4, 12) and s.shape == (12,) and vd.shape == (12, 12)
    assert np.all(np.diff(s) <= 0) and np.all(s >= 0)
    rec = np.einsum("ijk,k,kl->ijl", u, s, vd)
    assert rel_frob(rec, a) <= 1e-14
    w = rnd((2, 3, 5, 7), 151)                            # wide matricization: kappa = min(6, 35)
    u, s, vd = oracle_mod.svd(w, 2)
    assert u.shape == (2, 3, 6) and vd.shape == (6, 5, 7)
    U = u.reshape(6, 6)
    assert max_abs(U.T @ U, np.eye(6)) <= 1e-14


def test_svd_prescribed_spectrum(oracle_mod):
    """A = Q1 diag(sigma) Q2^H with random unitaries: the returned s is sigma
    (sorted), u/v_dag reproduce A and are orthonormal."""
    m, n = 24, 17
    sig = np.sort(np.abs(np.random.default_rng(3).standard_normal(n)) + 0.1)[::-1]
    A = _unitary(m, 4)[:, :n] @ np.diag(sig) @ _unitary(n, 5).conj().T
    u, s, vd = oracle_mod.svd(A.reshape(4, 6, n), 2)
    assert max_abs(s, sig) <= 1e-14 * sig[0]
    U = u.reshape(m, n)
    assert max_abs(U.conj().T @ U, np.eye(n)) <= 1e-14
    assert max_abs(vd @ vd.conj().T, np.eye(n)) <= 1e-14
    assert rel_frob((U * s) @ vd, A) <= 1e-14


@pytest.mark.parametrize("args,chi,num,den", [
    ((1, 3, 0.0, 1e-12), 3, Fraction(5, 4), None),          # overload (1): chi_max = 3
    ((2, 5, 0.05, 1e-12), 3, Fraction(5, 4), None),         # c) grows 2 -> 3 (eps 0.174 > 0.05 >= 0.041)
    ((6, 9, 0.0, 1e-12), 5, None, None),                    # b) fewer than chi_min survive a): keep 5
    ((1, 10, 0.0, 0.0), 6, Fraction(0), None),              # nothing discarded
    ((1, 10, 0.0, 5.0), 1, None, None),                     # all below s_min: R30 keeps one
    ((4, 4, 0.5, 1e-12), 4, Fraction(1, 4), None),          # chi_min = chi_max
])
def test_trunc_chi_strategy(oracle_mod, args, chi, num, den):
    s = [4.0, 3.0, 2.0, 1.0, 0.5, 1e-13]
    total = Fraction(16) + 9 + 4 + 1 + Fraction(1, 4) + Fraction(1e-13) ** 2
    got_chi, eps = oracle_mod.trunc_chi(s, *args)
    assert got_chi == chi
    exact = sum((Fraction(x) ** 2 for x in s[chi:]), Fraction(0)) / total
    assert abs(eps - float(exact)) <= 1e-16
    if num is not None:
        assert abs(eps - float(num / total)) <= 1e-15


def test_trunc_svd_paper_example(oracle_mod):
    a = rnd((3, 4, 12), 152)
    u, s, vd, err = oracle_mod.trunc_svd(a, 2, 3, 6, 1e-2, 1e-12)
    assert err != 0.0 and 3 <= s.shape[0] <= 6
    assert u.shape == (3, 4, s.shape[0]) and vd.shape == (s.shape[0], 12)


def test_trunc_svd_fidelity_identity(oracle_mod):
    """Section III (R24): with a normalized psi and psi1 = u s v_dag
    from trunc_svd, <psi|psi1> = 1 - trunc_err."""
    psi = rnd((2, 2, 2, 2, 2, 2), 153)
    psi = psi / np.sqrt(np.sum(psi * psi))
    u, s, vd, err = oracle_mod.trunc_svd(psi, 3, 1, 3, 0.0, 0.0)
    psi1 = np.einsum("ijka,a,alm n->ijklmn".replace(" ", ""), u, s, vd)
    ovlp = float(np.sum(psi * psi1))
    assert err > 0 and abs(ovlp - (1 - err)) <= 1e-14


# ---------------------------------------------------------------------------
# iTEBD (Application A) built from tebd_theta + trunc_svd
# ---------------------------------------------------------------------------

def _tfim_h(g):
    X = np.array([[0.0, 1.0], [1.0, 0.0]])
    Z = np.diag([1.0, -1.0])
    I = np.eye(2)
    return (-np.kron(Z, Z) + 0.5 * g * (np.kron(X, I) + np.kron(I, X))).reshape(2, 2, 2, 2)


def pfeuty_e0(g):
    """Exact TFIM ground-state energy per site (Pfeuty 1970):
    e0 = -(1/2pi) int_0^2pi sqrt(1 + g^2 - 2 g cos k) dk; the uniform-grid mean
    of a smooth periodic integrand is spectrally accurate."""
    k = np.linspace(0.0, 2.0 * np.pi, 400001)[:-1]
    return float(-np.mean(np.sqrt(1.0 + g * g - 2.0 * g * np.cos(k))))


ITEBD_SCHEDULE = [(0.1, 200), (0.01, 300), (0.001, 300)]


def test_pfeuty_quadrature_closed_forms():
    assert abs(pfeuty_e0(1.0) + 4.0 / np.pi) <= 1e-10          # critical point: -4/pi (kink at k = 0: O(1/N^2))
    assert abs(pfeuty_e0(0.0) + 1.0) <= 1e-15                  # classical ferromagnet


@pytest.mark.parametrize("g,tol", [(1.0, 1e-4), (0.5, 1e-5)])
def test_itebd_tfim_energy(oracle_mod, g, tol):
    """SPEC.md:618-621 / acceptance 5: chi = 16 imaginary-time iTEBD reaches the
    Pfeuty energy (within 1e-4 at the critical point g = 1, 1e-5 at g = 0.5)."""
    e, _ = oracle_mod.itebd_tfim(g, 16, ITEBD_SCHEDULE, lambda tau: synth.tfim_gate(tau, 1.0, g), _tfim_h(g))
    assert abs(e - pfeuty_e0(g)) <= tol
    assert e >= pfeuty_e0(g) - 1e-9                            # variational (up to Trotter error)


def test_itebd_identity_gate_on_product_state(oracle_mod):
    """SPEC itebd_update_bond examples: from a product state (chi = 1) the
    identity gate keeps rank 1, so trunc_err = 0 (up to rounding noise of the
    discarded values) and the new centre lambda is exactly (1)."""
    rng = np.random.default_rng(3)
    GA, GB = rng.uniform(-1, 1, (1, 2, 1)), rng.uniform(-1, 1, (1, 2, 1))
    GA2, lA2, GB2, err = oracle_mod.itebd_update(GA, np.ones(1), GB, np.ones(1), synth.tfim_gate(0.0), 4)
    assert lA2.shape == (1,) and lA2[0] == 1.0 and err <= 1e-30


# ---------------------------------------------------------------------------
# zip-up MPS-MPO application
# ---------------------------------------------------------------------------

def dense_mps(sites):
    """Amplitudes psi(s_1..s_n) = A_1[s_1] ... A_n[s_n] (open boundary)."""
    v = sites[0].reshape(sites[0].shape[1], sites[0].shape[2])
    for A in sites[1:]:
        v = np.einsum("xa,asb->xsb", v, A).reshape(-1, A.shape[2])
    return v.reshape(-1)


def dense_mpo(W):
    """Operator matrix O[(t_1..t_n),(s_1..s_n)] from W[w,v,s,t] by Kronecker assembly."""
    M = W[0][0]                                    # [v, s, t]
    M = np.transpose(M, (0, 2, 1))                 # [v, t, s]
    for Wi in W[1:]:
        M = np.einsum("vTS,vwst->wTtSs", M, Wi)
        M = M.reshape(M.shape[0], M.shape[1] * M.shape[2], M.shape[3] * M.shape[4])
    return M[0]


def _zipup_inputs(n, chi, D, d, dt, seed):
    rng = np.random.default_rng(seed)
    bonds = [1] + [min(chi, d ** min(i + 1, n - i - 1)) for i in range(n - 1)] + [1]
    mb = [1] + [D] * (n - 1) + [1]
    cp = dt == "c128"
    def r(*sh):
        x = rng.uniform(-1, 1, sh)
        return x + 1j * rng.uniform(-1, 1, sh) if cp else x
    A = [r(bonds[i], d, bonds[i + 1]) for i in range(n)]
    W = [r(mb[i], mb[i + 1], d, d) for i in range(n)]
    return A, W


@pytest.mark.parametrize("dt", ["r64", "c128"])
def test_zipup_exact_equals_dense_operator(oracle_mod, dt):
    """No truncation (chi_max above every exact bond, s_min = 0): the zip-up
    state equals W|psi> formed densely (Kronecker-assembled MPO matrix)."""
    A, W = _zipup_inputs(6, 4, 3, 2, dt, 11)
    B, err = oracle_mod.mps_mpo_zipup(A, W, 10 ** 6)
    ref = dense_mpo(W) @ dense_mps(A)
    assert err <= 1e-28
    assert rel_frob(dense_mps(B), ref) <= 1e-13


def test_zipup_identity_mpo_and_heisenberg(oracle_mod):
    """Identity MPO (D = 1, W = I) reproduces psi; the Heisenberg MPO gives
    <psi|H|psi> of the dense Kronecker Hamiltonian (bra = psi, real data)."""
    A, _ = _zipup_inputs(6, 4, 1, 2, "r64", 12)
    I = [np.eye(2).reshape(1, 1, 2, 2) for _ in range(6)]
    B, _ = oracle_mod.mps_mpo_zipup(A, I, 10 ** 6)
    assert rel_frob(dense_mps(B), dense_mps(A)) <= 1e-13
    Wh, lb, rb = synth.heisenberg_mpo(1.0)
    Wh = np.asarray(Wh).real
    Ws = [Wh[lb:lb + 1]] + [Wh] * 4 + [Wh[:, rb:rb + 1]]
    B, _ = oracle_mod.mps_mpo_zipup(A, Ws, 10 ** 6)
    psi = dense_mps(A)
    assert abs(psi @ dense_mps(B) - psi @ dense_mpo(Ws) @ psi) <= 1e-12 * abs(psi @ psi)


def test_zipup_truncation_error_accounting(oracle_mod):
    """With chi_max = 2 the kept state is no longer exact, the reported error
    is positive, and chi_max >= exact bonds reports zero."""
    A, W = _zipup_inputs(6, 4, 3, 2, "r64", 13)
    B, err = oracle_mod.mps_mpo_zipup(A, W, 2)
    assert err > 0 and max(b.shape[2] for b in B) <= 2
    ref = dense_mpo(W) @ dense_mps(A)
    assert rel_frob(dense_mps(B), ref) > 1e-6
