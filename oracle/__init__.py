"""CPU ORACLE -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` leg may import this package. The
product path (``paper_2512_23917_b200``) never imports it and shares no code
with it; the only module both sides use is ``synth`` (seeded inputs, no
arithmetic of the method).

Every function is the plain definition from the paper (PAPER.md line numbers)
or, where the paper has no definition (the H_eff, TEBD and MPS chains), the
textbook definition recorded in DESIGN.md section "Readings". The numeric core
is ``tci_oracle.c`` (plain loops, double precision, -ffp-contract=off); this
module only marshals numpy arrays and composes the chains from ``contract``
calls in the order DESIGN.md states.

Parity pins live in ``tests/test_oracle_pins.py``; functions without a pin
would be marked "parity unpinned" here -- currently every function below is
pinned (DESIGN.md section "Pins").
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from typing import Sequence, Union

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "tci_oracle.c")
_SO = os.path.join(_HERE, "libtci_oracle.so")

Labels = Union[str, Sequence[int]]

ERROR_NAMES = {
    1: "SHAPE_MISMATCH", 2: "ORDER_MISMATCH", 3: "OUT_OF_RANGE",
    4: "LABEL_CONFLICT", 5: "PARSE", 7: "UNSUPPORTED", 8: "INVALID_ARGUMENT",
    12: "NOMEM",
}


class OracleError(RuntimeError):
    def __init__(self, code: int, what: str = ""):
        self.code = code
        super().__init__(f"oracle error {code} ({ERROR_NAMES.get(code, '?')}) {what}")


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (plain C, OpenMP, no FMA contraction)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        tmp = _SO + f".tmp{os.getpid()}"
        subprocess.check_call([
            "gcc", "-O2", "-fopenmp", "-ffp-contract=off", "-fno-fast-math",
            "-fPIC", "-shared", "-std=c99", "-o", tmp, _SRC])
        os.replace(tmp, _SO)
    return _SO


_lib_handle = None


def _lib():
    global _lib_handle
    if _lib_handle is None:
        build()
        lib = ctypes.CDLL(_SO)
        i64p = ctypes.POINTER(ctypes.c_int64)
        i32p = ctypes.POINTER(ctypes.c_int32)
        dp = ctypes.POINTER(ctypes.c_double)
        ci = ctypes.c_int
        lib.oracle_contract.argtypes = [ci, ci, i64p, i32p, dp, ci, i64p, i32p, dp, ci, i32p, dp, ci]
        lib.oracle_contract_abs.argtypes = [ci, i64p, i32p, dp, ci, i64p, i32p, dp, ci, i32p, dp, ci]
        lib.oracle_contract_shape.argtypes = [ci, i64p, i32p, ci, i64p, i32p, ci, i32p, i64p]
        lib.oracle_permute.argtypes = [ci, ci, i64p, i32p, dp, dp, ci]
        lib.oracle_max_threads.restype = ci
        _lib_handle = lib
    return _lib_handle


def max_threads() -> int:
    return int(_lib().oracle_max_threads())


# ----------------------------------------------------------------------------
# marshalling helpers
# ----------------------------------------------------------------------------

def _labels(l: Labels, order: int) -> np.ndarray:
    """String API: one byte per label (reading R12)."""
    if isinstance(l, str):
        b = l.encode("latin-1")
        if len(b) != order:
            raise OracleError(2, f"label string {l!r} has {len(b)} labels for order {order}")
        arr = np.frombuffer(b, dtype=np.uint8).astype(np.int32)
    else:
        arr = np.asarray(list(l), dtype=np.int32)
        if arr.size != order:
            raise OracleError(2, f"{arr.size} labels for order {order}")
    return np.ascontiguousarray(arr)


def _as_f64(x: np.ndarray):
    """Widen exactly to float64 / complex128 (reading R14)."""
    x = np.asarray(x)
    # np.require keeps 0-d arrays 0-d (ascontiguousarray would make them 1-d)
    if np.iscomplexobj(x):
        return np.require(x, dtype=np.complex128, requirements="C"), True
    return np.require(x, dtype=np.float64, requirements="C"), False


def _p(a, t):
    return a.ctypes.data_as(ctypes.POINTER(t))


def _dptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _shape(a: np.ndarray) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a.shape, dtype=np.int64).reshape(-1))


# ----------------------------------------------------------------------------
# core functions
# ----------------------------------------------------------------------------

def contract_shape(sa, la: Labels, sb, lb: Labels, lc: Labels):
    lib = _lib()
    sa = np.ascontiguousarray(np.asarray(sa, dtype=np.int64).reshape(-1))
    sb = np.ascontiguousarray(np.asarray(sb, dtype=np.int64).reshape(-1))
    la_ = _labels(la, sa.size)
    lb_ = _labels(lb, sb.size)
    nc = len(lc.encode("latin-1")) if isinstance(lc, str) else len(list(lc))
    lc_ = _labels(lc, nc)
    sc = np.zeros(max(nc, 1), dtype=np.int64)
    st = lib.oracle_contract_shape(sa.size, _p(sa, ctypes.c_int64), _p(la_, ctypes.c_int32),
                                   sb.size, _p(sb, ctypes.c_int64), _p(lb_, ctypes.c_int32),
                                   nc, _p(lc_, ctypes.c_int32), _p(sc, ctypes.c_int64))
    if st:
        raise OracleError(st)
    return tuple(int(x) for x in sc[:nc])


def contract(a: np.ndarray, la: Labels, b: np.ndarray, lb: Labels, lc: Labels,
             threads: int | None = None) -> np.ndarray:
    """tci::contract, Eq. (3)."""
    lib = _lib()
    a, ca = _as_f64(a)
    b, cb = _as_f64(b)
    cplx = ca or cb
    if cplx:
        a = a.astype(np.complex128)
        b = b.astype(np.complex128)
    sc = contract_shape(a.shape, la, b.shape, lb, lc)
    la_ = _labels(la, a.ndim)
    lb_ = _labels(lb, b.ndim)
    lc_ = _labels(lc, len(sc))
    c = np.empty(sc, dtype=np.complex128 if cplx else np.float64)
    sa, sb = _shape(a), _shape(b)
    st = lib.oracle_contract(int(cplx), a.ndim, _p(sa, ctypes.c_int64), _p(la_, ctypes.c_int32), _dptr(a),
                             b.ndim, _p(sb, ctypes.c_int64), _p(lb_, ctypes.c_int32), _dptr(b),
                             len(sc), _p(lc_, ctypes.c_int32), _dptr(c),
                             int(threads or max_threads()))
    if st:
        raise OracleError(st)
    return c


def contract_abs(a: np.ndarray, la: Labels, b: np.ndarray, lb: Labels, lc: Labels,
                 threads: int | None = None) -> np.ndarray:
    """|A|.|B| under the same contraction (real only): the Higham bound term."""
    lib = _lib()
    a = np.require(a, dtype=np.float64, requirements="C")
    b = np.require(b, dtype=np.float64, requirements="C")
    sc = contract_shape(a.shape, la, b.shape, lb, lc)
    la_, lb_, lc_ = _labels(la, a.ndim), _labels(lb, b.ndim), _labels(lc, len(sc))
    c = np.empty(sc, dtype=np.float64)
    sa, sb = _shape(a), _shape(b)
    st = lib.oracle_contract_abs(a.ndim, _p(sa, ctypes.c_int64), _p(la_, ctypes.c_int32), _dptr(a),
                                 b.ndim, _p(sb, ctypes.c_int64), _p(lb_, ctypes.c_int32), _dptr(b),
                                 len(sc), _p(lc_, ctypes.c_int32), _dptr(c), int(threads or max_threads()))
    if st:
        raise OracleError(st)
    return c


def permute(a: np.ndarray, perm: Sequence[int], threads: int | None = None) -> np.ndarray:
    """tci::transpose, Eq. (1)."""
    lib = _lib()
    a, cplx = _as_f64(a)
    perm_ = np.ascontiguousarray(np.asarray(list(perm), dtype=np.int32))
    if perm_.size != a.ndim:
        raise OracleError(2)
    for p in perm_:
        if p < 0 or p >= a.ndim:
            raise OracleError(8)
    out = np.empty(tuple(a.shape[p] for p in perm_), dtype=a.dtype)
    sa = _shape(a)
    st = lib.oracle_permute(int(cplx), a.ndim, _p(sa, ctypes.c_int64), _p(perm_, ctypes.c_int32),
                            _dptr(a), _dptr(out), int(threads or max_threads()))
    if st:
        raise OracleError(st)
    return out


def reshape(a: np.ndarray, new_shape: Sequence[int]) -> np.ndarray:
    """tci::reshape: metadata only, element order kept."""
    new_shape = tuple(int(s) for s in new_shape)
    if any(s < 1 for s in new_shape):
        raise OracleError(3)
    if int(np.prod(new_shape, dtype=np.int64)) != a.size:
        raise OracleError(1)
    return np.ascontiguousarray(a).reshape(new_shape)


# ----------------------------------------------------------------------------
# chains (definitions: DESIGN.md "Readings" R15-R17; no paper text exists)
# ----------------------------------------------------------------------------

def heff(L, W1, W2, R, psi, threads=None):
    """Two-site H_eff.psi (R15), FLOP-optimal order L.psi -> W1 -> W2 -> R.

    L[a,w,b], psi[a,s,t,c], W1[w,v,s,p], W2[v,x,t,q], R[c,x,e] -> out[b,p,q,e].
    """
    T1 = contract(L, "awb", psi, "astc", "wbstc", threads)
    T2 = contract(T1, "wbstc", W1, "wvsp", "btcvp", threads)
    T3 = contract(T2, "btcvp", W2, "vxtq", "bpqcx", threads)
    return contract(T3, "bpqcx", R, "cxe", "bpqe", threads)


def heff_alt(L, W1, W2, R, psi, threads=None):
    """Same operator, a different pairwise order (R first): order invariance."""
    U1 = contract(psi, "astc", R, "cxe", "astxe", threads)
    U2 = contract(U1, "astxe", W2, "vxtq", "asvqe", threads)
    U3 = contract(U2, "asvqe", W1, "wvsp", "awpqe", threads)
    return contract(U3, "awpqe", L, "awb", "bpqe", threads)


def heff_rows(L, W1, W2, R, psi, rows, threads=None):
    """Rows out[b0,:,:,:] for b0 in rows: the chain on the slice L[:,:,b0]."""
    res = []
    for b0 in rows:
        Lr = np.ascontiguousarray(L[:, :, int(b0):int(b0) + 1])
        res.append(heff(Lr, W1, W2, R, psi, threads)[0])
    return np.stack(res)


def heff_dense(L, W1, W2, R, shape_psi, threads=None):
    """Dense matrix H[(b p q e), (a s t c)] by applying H_eff to basis vectors."""
    n = int(np.prod(shape_psi))
    cols = []
    dt = np.result_type(L, W1, W2, R)
    for k in range(n):
        e = np.zeros(n, dtype=dt)
        e[k] = 1
        cols.append(heff(L, W1, W2, R, e.reshape(shape_psi), threads).reshape(-1))
    return np.stack(cols, axis=1)


def tebd_theta(A, B, U, la="asb", lb="btc", lu="pqst", lt="apqc", threads=None):
    """theta = (A.B).U (R16): AB over b, then the gate over (s,t)."""
    # intermediate keeps the non-b legs of A then of B, in label order
    lab = "".join(ch for ch in la if ch not in lb) + "".join(ch for ch in lb if ch not in la)
    AB = contract(A, la, B, lb, lab, threads)
    return contract(AB, lab, U, lu, lt, threads)


def mps_overlap(bra, ket, threads=None):
    """<bra|ket> by the transfer chain of DESIGN.md R17 (real data, no conj)."""
    E = np.ones((1, 1), dtype=np.result_type(bra[0], ket[0]))
    for Ab, Ak in zip(bra, ket):
        X = contract(E, "xz", Ab, "xsy", "zsy", threads)
        E = contract(X, "zsy", Ak, "zsw", "yw", threads)
    return E


def mps_norm2(sites, threads=None):
    return mps_overlap(sites, sites, threads)


def mps_mpo_apply(A, W, threads=None):
    """Site-local uncompressed MPO application (R18):
    B[a,w,t,b,v] = sum_s A[a,s,b] W[w,v,s,t], then reshape to [(a w), t, (b v)]."""
    Bt = contract(A, "asb", W, "wvst", "awtbv", threads)
    a, w, t, b, v = Bt.shape
    return reshape(Bt, (a * w, t, b * v))


def cplx_conj(a):
    """tci::cplx_conj: elementwise complex conjugate,
    (re, im) -> (re, -im); for real data a deep copy."""
    a = np.asarray(a)
    if np.iscomplexobj(a):
        out = np.empty_like(a)
        out.real = a.real
        out.imag = -a.imag
        return out
    return a.copy()


def env_left(E, ket, W, bra=None, threads=None):
    """Left environment update (R28), the definition
        out[b,v,e] = sum_{a,w,c,s,t} E[a,w,c] ket[a,s,b] W[w,v,s,t] conj(bra[c,t,e])
    evaluated pairwise in the order E.ket -> W -> conj(bra)."""
    bra = ket if bra is None else bra
    T1 = contract(E, "awc", ket, "asb", "wcsb", threads)
    T2 = contract(T1, "wcsb", W, "wvst", "ctbv", threads)
    return contract(T2, "ctbv", cplx_conj(bra), "cte", "bve", threads)


def env_right(E, ket, W, bra=None, threads=None):
    """Right environment update (R28), the definition
        out[a,w,f] = sum_{c,x,e,s,t} ket[a,s,c] W[w,x,s,t] E[c,x,e] conj(bra[f,t,e])
    evaluated pairwise in the order ket.E -> W -> conj(bra)."""
    bra = ket if bra is None else bra
    T1 = contract(ket, "asc", E, "cxe", "asxe", threads)
    T2 = contract(T1, "asxe", W, "wxst", "awte", threads)
    return contract(T2, "awte", cplx_conj(bra), "fte", "awf", threads)


def env_rows(side, E, ket, W, bra, rows, threads=None):
    """Rows out[r,:,:] for r in rows (the ket's outgoing bond sliced to r)."""
    res = []
    for r in rows:
        r = int(r)
        if side == 0:
            k = np.ascontiguousarray(ket[:, :, r:r + 1])
            res.append(env_left(E, k, W, bra, threads)[0])
        else:
            k = np.ascontiguousarray(ket[r:r + 1])
            res.append(env_right(E, k, W, bra, threads)[0])
    return np.stack(res)


def svd(a, k):
    """tci::svd: matricize the first k bonds as rows
    (I = prod d_0..d_{k-1}, J = the rest), A' = U S V^dagger with
    s_0 >= ... >= s_{kappa-1} >= 0, kappa = min(I, J); fold back to
    u [d_0..d_{k-1}, kappa], s [kappa] (real), v_dag [kappa, d_k..d_{r-1}].
    The matrix SVD is the library primitive (LAPACK via numpy)."""
    a = np.asarray(a)
    r = a.ndim
    if not 1 <= k < r:
        raise ValueError("svd: need 1 <= num_of_bds_as_row < order")
    I = int(np.prod(a.shape[:k]))
    J = int(np.prod(a.shape[k:]))
    U, s, Vh = np.linalg.svd(a.reshape(I, J), full_matrices=False)
    kappa = min(I, J)
    return U.reshape(*a.shape[:k], kappa), s, Vh.reshape(kappa, *a.shape[k:])


def trunc_chi(s, chi_min, chi_max, target_trunc_err, s_min):
    """Truncation strategy of tci::trunc_svd (2), applied
    to non-increasing s; returns (chi, eps) with eps of PAPER.md:2088-2090:
    eps(chi) = sum_{i >= chi} s_i^2 / sum_i s_i^2.
      a) discard all s_i < s_min;
      b) keep at least chi_min values; if fewer remain after a), keep those;
      c) grow chi (descending order) until eps <= target_trunc_err or chi = chi_max."""
    s = [float(x) for x in s]
    total = sum(x * x for x in s)

    def eps(chi):
        return (sum(x * x for x in s[chi:]) / total) if total > 0 else 0.0

    remain = sum(1 for x in s if x >= s_min)            # a)
    if remain <= chi_min:                               # b) stop and retain those
        chi = remain
    else:
        chi = chi_min                                   # b)
        while chi < min(chi_max, remain) and eps(chi) > target_trunc_err:   # c)
            chi += 1
    chi = max(chi, 1)                                   # DESIGN.md R30: never an empty bond
    return chi, eps(chi)


def trunc_svd(a, k, chi_min, chi_max, target_trunc_err, s_min):
    """tci::trunc_svd (2); overload (1) is chi_min = 1,
    target_trunc_err = 0. Returns (u, s, v_dag, trunc_err) truncated to chi."""
    u, s, vd = svd(a, k)
    chi, err = trunc_chi(s, chi_min, chi_max, target_trunc_err, s_min)
    return (np.ascontiguousarray(u[..., :chi]), np.ascontiguousarray(s[:chi]),
            np.ascontiguousarray(vd[:chi]), err)


def mps_mpo_zipup(A, W, chi_max, s_min=0.0, threads=None):
    """Compressed MPS-MPO application by zip-up (R32):
    C = 1; per site T1 = C.A_i ("kaw","asb"->"kwsb"), T = T1.W_i
    ("kwsb","wvst"->"ktbv"); for i < n-1 trunc_svd of T at (k t)|(b v) with
    chi_min = 1: B_i = U, C = S V^dag; the last site takes T.
    Returns (B sites, sum of the per-bond discarded weights)."""
    C = np.ones((1, 1, 1), dtype=np.result_type(A[0], W[0]))
    out, err = [], 0.0
    n = len(A)
    for i in range(n):
        T1 = contract(C, "kaw", A[i], "asb", "kwsb", threads)
        T = contract(T1, "kwsb", W[i], "wvst", "ktbv", threads)
        if i == n - 1:
            out.append(np.ascontiguousarray(T.reshape(T.shape[0], T.shape[1], 1)))
            break
        U, S, Vd, e = trunc_svd(T, 2, 1, chi_max, 0.0, s_min)
        out.append(U)
        err += e
        C = S[:, None, None] * Vd
    return out, err


def itebd_update(GA, lA, GB, lB, U, chi, s_min=1e-12, threads=None):
    """One bond update of Vidal's iTEBD (Application A, PAPER.md:392-403;
    SPEC.md itebd_update_bond): theta[a,s,t,c] = lB[a] GA[a,s,b] lA[b]
    GB[b,t,c] lB[c]; theta' = U.theta over (s,t) (tebd_theta, R16);
    trunc_svd at (a p)|(q c) with chi_max = chi; the new centre
    lambda is normalised and the outer lambdas are divided back out.
    Returns (GA', lA', GB', trunc_err)."""
    A = lB[:, None, None] * GA * lA[None, None, :]
    B = GB * lB[None, None, :]
    th = tebd_theta(A, B, U, threads=threads)
    X, s, Y, err = trunc_svd(th, 2, 1, chi, 0.0, s_min)
    s = s / np.sqrt(np.sum(s * s))
    return X / lB[:, None, None], s, Y / lB[None, None, :], err


def itebd_bond_energy(GA, lA, GB, lB, h, threads=None):
    """<theta|h|theta>/<theta|theta> for the bond A-B in the canonical
    lB GA lA GB lB form (h[p,q,s,t], real data)."""
    A = lB[:, None, None] * GA * lA[None, None, :]
    B = GB * lB[None, None, :]
    th = contract(A, "asb", B, "btc", "astc", threads)
    hth = contract(th, "astc", h, "pqst", "apqc", threads)
    return float(np.sum(th * hth) / np.sum(th * th))


def itebd_tfim(g, chi, schedule, gate, h, seed=0):
    """Imaginary-time iTEBD for the 1D TFIM (R25) from a
    random product state: for (tau, steps) in schedule, `steps` A-B / B-A
    bond-update pairs with U = gate(tau). Returns the energy per site (the
    mean of the two bond energies) and the final state."""
    rng = np.random.default_rng(seed)
    GA = rng.uniform(-1, 1, (1, 2, 1))
    GB = rng.uniform(-1, 1, (1, 2, 1))
    GA /= np.linalg.norm(GA)
    GB /= np.linalg.norm(GB)
    lA = np.ones(1)
    lB = np.ones(1)
    for tau, steps in schedule:
        U = gate(tau)
        for _ in range(steps):
            GA, lA, GB, _ = itebd_update(GA, lA, GB, lB, U, chi)
            GB, lB, GA, _ = itebd_update(GB, lB, GA, lA, U, chi)
    e = 0.5 * (itebd_bond_energy(GA, lA, GB, lB, h) + itebd_bond_energy(GB, lB, GA, lA, h))
    return e, (GA, lA, GB, lB)


# ----------------------------------------------------------------------------
# vector functions (App. C.5): definitions written out
# ----------------------------------------------------------------------------

def norm(a) -> float:
    """Frobenius norm, Eq. frob_norm: sqrt(sum |A_i|^2)."""
    a = np.asarray(a).reshape(-1)
    return float(np.sqrt(np.sum((a.real.astype(np.float64) ** 2) + (a.imag.astype(np.float64) ** 2))))


def scale(a, s):
    """tci::scale: s * A."""
    return s * np.asarray(a)


def linear_combine(ins, coefs=None):
    """tci::linear_combine: sum_i s_i A_i (s_i = 1 by default)."""
    coefs = [1.0] * len(ins) if coefs is None else list(coefs)
    out = np.zeros_like(np.asarray(ins[0]), dtype=np.result_type(*ins, *[np.asarray(c) for c in coefs]))
    for c, x in zip(coefs, ins):
        out = out + c * np.asarray(x)
    return out


def inner(a, b, conj_a=True):
    """Full contraction to a scalar of conj(a) (cplx_conj,
    PAPER.md:1235-1268) with b: sum_i conj(a_i) b_i."""
    a = np.asarray(a).reshape(-1)
    b = np.asarray(b).reshape(-1)
    return complex(np.sum((np.conj(a) if conj_a else a) * b))
