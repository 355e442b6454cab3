"""Seeded synthetic inputs shared by the oracle tests and the CUDA path.

This module holds NO arithmetic of the method (no contraction, no chain): it
only draws counter-based random numbers and builds the physical input tensors
(model MPOs, the TFIM gate, MPS site tensors) whose entries are fixed by
textbook definitions. Recipe: DESIGN.md section "Inputs".

Generator: element ``i`` of tensor
``tensor_id`` under ``seed`` is

    key = seed XOR (tensor_id * 0x9E3779B97F4A7C15)      (mod 2**64)
    u   = splitmix64(key + i)                            (mod 2**64)
    x   = (u >> 11) * 2**-52 - 1                          in [-1, 1)

Complex values take (re, im) from draws 2i and 2i+1; float32 values are the
float64 draws rounded to nearest. The implementation uses torch int64
arithmetic (two's-complement wrap-around, logical shifts by masking) so it
runs identically on CPU and GPU; ``splitmix64_ref`` is a pure-Python big-int
version used by the tests to pin it.
"""
from __future__ import annotations

import math
from typing import Dict, List, Sequence, Tuple

import numpy as np
import torch

GOLDEN = 0x9E3779B97F4A7C15
C1 = 0xBF58476D1CE4E5B9
C2 = 0x94D049BB133111EB
M64 = (1 << 64) - 1

# tensor ids
TID = {"L": 1, "psi": 2, "W1": 3, "W2": 4, "R": 5, "A": 6, "B": 7, "U": 8,
       "phi": 9, "X": 10, "Y": 11}


def site_tid(i: int) -> int:
    return 100 + i


def _s64(x: int) -> int:
    """Unsigned 64-bit constant as a signed int64 value."""
    x &= M64
    return x - (1 << 64) if x >= (1 << 63) else x


def splitmix64_ref(x: int) -> int:
    """Pure-Python reference splitmix64 (Steele, Lea, Flood 2014)."""
    z = (x + GOLDEN) & M64
    z = ((z ^ (z >> 30)) * C1) & M64
    z = ((z ^ (z >> 27)) * C2) & M64
    return z ^ (z >> 31)


def uniform_ref(seed: int, tensor_id: int, i: int) -> float:
    key = (seed ^ ((tensor_id * GOLDEN) & M64)) & M64
    u = splitmix64_ref((key + i) & M64)
    return (u >> 11) * 2.0 ** -52 - 1.0


def _lsr(z: torch.Tensor, k: int) -> torch.Tensor:
    return (z >> k) & ((1 << (64 - k)) - 1)


def _splitmix64_t(x: torch.Tensor) -> torch.Tensor:
    z = x + _s64(GOLDEN)
    z = (z ^ _lsr(z, 30)) * _s64(C1)
    z = (z ^ _lsr(z, 27)) * _s64(C2)
    return z ^ _lsr(z, 31)


def uniform_draws(seed: int, tensor_id: int, n: int, device="cpu",
                  chunk: int = 1 << 26) -> torch.Tensor:
    """n float64 draws in [-1, 1) as a 1-D torch tensor on ``device``."""
    key = _s64((seed ^ ((tensor_id * GOLDEN) & M64)) & M64)
    out = torch.empty(n, dtype=torch.float64, device=device)
    for s in range(0, n, chunk):
        m = min(chunk, n - s)
        idx = torch.arange(s, s + m, dtype=torch.int64, device=device) + key
        u = _splitmix64_t(idx)
        out[s:s + m] = _lsr(u, 11).to(torch.float64) * (2.0 ** -52) - 1.0
    return out


def random_tensor(shape: Sequence[int], dtype: str, seed: int, tensor_id: int,
                  device="cpu") -> torch.Tensor:
    """Uniform[-1,1) tensor; dtype in {'r32','r64','c64','c128'}."""
    shape = tuple(int(s) for s in shape)
    n = int(np.prod(shape, dtype=np.int64)) if shape else 1
    if dtype in ("c64", "c128"):
        d = uniform_draws(seed, tensor_id, 2 * n, device)
        t = torch.view_as_complex(d.view(n, 2)).reshape(shape)
        return t if dtype == "c128" else t.to(torch.complex64)
    d = uniform_draws(seed, tensor_id, n, device).reshape(shape)
    return d if dtype == "r64" else d.to(torch.float32)


def random_np(shape, dtype, seed, tensor_id) -> np.ndarray:
    return random_tensor(shape, dtype, seed, tensor_id, "cpu").numpy()


TORCH_DTYPE = {"r32": torch.float32, "r64": torch.float64,
               "c64": torch.complex64, "c128": torch.complex128}

# ----------------------------------------------------------------------------
# physical inputs (textbook definitions)
# ----------------------------------------------------------------------------


def _spin_half():
    sp = np.array([[0.0, 1.0], [0.0, 0.0]])   # S+ |dn> = |up>, basis (up, dn)
    sm = sp.T.copy()
    sz = np.diag([0.5, -0.5])
    return sp, sm, sz, np.eye(2)


def mpo_from_operator_matrix(ops: List[List[np.ndarray]]) -> np.ndarray:
    """W[w_l, w_r, s, t] = O_{w_l w_r}[t, s] (operator maps |s> -> |t>)."""
    D = len(ops)
    d = ops[0][0].shape[0]
    W = np.zeros((D, D, d, d), dtype=np.complex128)
    for i in range(D):
        for j in range(D):
            W[i, j] = ops[i][j].T
    return W


def heisenberg_mpo(J: float = 1.0):
    """Spin-1/2 Heisenberg D=5 lower-triangular MPO; boundaries (left=4, right=0).

    H = J sum_i S_i . S_{i+1} = J sum (S^z S^z + (S^+ S^- + S^- S^+)/2).
    Returns (W, left_index, right_index).
    """
    sp, sm, sz, I = _spin_half()
    Z = np.zeros((2, 2))
    ops = [[Z] * 5 for _ in range(5)]
    ops[0][0] = I
    ops[1][0] = sp
    ops[2][0] = sm
    ops[3][0] = sz
    ops[4][1] = 0.5 * J * sm
    ops[4][2] = 0.5 * J * sp
    ops[4][3] = J * sz
    ops[4][4] = I
    return mpo_from_operator_matrix(ops), 4, 0


def hubbard_local_ops():
    """Local basis |0>, |up>, |dn>, |updn> = c+_up c+_dn |0>."""
    cu = np.zeros((4, 4)); cd = np.zeros((4, 4))
    cu[0, 1] = 1.0   # c_up |up> = |0>
    cu[2, 3] = 1.0   # c_up |updn> = |dn>
    cd[0, 2] = 1.0   # c_dn |dn> = |0>
    cd[1, 3] = -1.0  # c_dn |updn> = -|up>
    F = np.diag([1.0, -1.0, -1.0, 1.0])
    nn = np.diag([0.0, 0.0, 0.0, 1.0])
    return cu, cd, F, nn, np.eye(4)


def hubbard_mpo(t: float = 1.0, U: float = 4.0):
    """Fermi-Hubbard D=6 MPO (Jordan-Wigner), boundaries (left=5, right=0).

    H = -t sum_sigma (c+_{i s} c_{i+1 s} + h.c.) + U sum_i n_up n_dn. With
    c_{i+1} = F_i c (JW string): c+_{i}c_{i+1} = (c+ F) (x) c and
    c+_{i+1} c_i = (F c) (x) c+ = -(c F) (x) c+.
    """
    cu, cd, F, nn, I = hubbard_local_ops()
    Z = np.zeros((4, 4))
    ops = [[Z] * 6 for _ in range(6)]
    ops[0][0] = I
    ops[1][0] = cu
    ops[2][0] = cu.T
    ops[3][0] = cd
    ops[4][0] = cd.T
    ops[5][0] = U * nn
    ops[5][1] = -t * (cu.T @ F)
    ops[5][2] = +t * (cu @ F)
    ops[5][3] = -t * (cd.T @ F)
    ops[5][4] = +t * (cd @ F)
    ops[5][5] = I
    return mpo_from_operator_matrix(ops), 5, 0


def tfim_gate(tau: float, J: float = 1.0, g: float = 1.0, real_time: bool = False) -> np.ndarray:
    """U[p,q,s,t] = expm(-tau h)[(p q),(s t)], h = -J Z(x)Z + (g/2)(X(x)I + I(x)X);
    real_time: the unitary expm(-i tau h) (complex128) of real-time TEBD.

    PAPER.md:394-397 (Eq. of the 1D TFIM, Application A); the field split in
    halves over the two bond sublattices as in SPEC.md:587-595. Built by
    eigendecomposition of the real symmetric 4x4 h (exact up to rounding).
    """
    X = np.array([[0.0, 1.0], [1.0, 0.0]])
    Zm = np.diag([1.0, -1.0])
    I = np.eye(2)
    h = -J * np.kron(Zm, Zm) + 0.5 * g * (np.kron(X, I) + np.kron(I, X))
    w, v = np.linalg.eigh(h)
    Um = (v * np.exp((-1j if real_time else -1.0) * tau * w)) @ v.T
    if tau == 0.0:
        Um = np.eye(4, dtype=Um.dtype)
    return Um.reshape(2, 2, 2, 2)


def boundary_env(D: int, index: int, dtype=np.complex128) -> np.ndarray:
    """chi=1 environment picking MPO row/column ``index``: shape (1, D, 1)."""
    e = np.zeros((1, D, 1), dtype=dtype)
    e[0, index, 0] = 1.0
    return e


# ----------------------------------------------------------------------------
# workloads (BASELINE.json configs)
# ----------------------------------------------------------------------------

MPS_BONDS_CFG1 = [1, 2, 4, 8, 16, 16, 16, 8, 4, 2, 1]


def mps_sites(bonds: Sequence[int], d: int, seed: int, dtype="r64") -> List[np.ndarray]:
    return [random_np((bonds[i], d, bonds[i + 1]), dtype, seed, site_tid(i))
            for i in range(len(bonds) - 1)]


def product_state_sites(n: int, d: int = 2) -> List[np.ndarray]:
    """One-hot product state |0 1 0 1 ...> with chi = 1: norm exactly 1."""
    out = []
    for i in range(n):
        a = np.zeros((1, d, 1))
        a[0, i % d, 0] = 1.0
        out.append(a)
    return out


HEFF_CONFIGS: Dict[str, dict] = {
    # name: chi, d, D, dtype, seed, model
    "cfg2_heisenberg_chi1024": dict(chi=1024, d=2, D=5, dtype="c128", seed=3, model="heisenberg"),
    "target_heisenberg_chi4096": dict(chi=4096, d=2, D=5, dtype="c128", seed=6, model="heisenberg"),
    "cfg4_hubbard_chi4096": dict(chi=4096, d=4, D=6, dtype="c128", seed=5, model="hubbard"),
}


def model_mpo(model: str):
    return heisenberg_mpo() if model == "heisenberg" else hubbard_mpo()


def heff_inputs(chi: int, d: int, D: int, dtype: str, seed: int, model: str,
                device="cpu", chi_out: int | None = None) -> Dict[str, torch.Tensor]:
    """L[a,w,b], W1[w,v,s,p], W2[v,x,t,q], R[c,x,e], psi[a,s,t,c] (R15).

    L, R, psi uniform; W1 = W2 = the exact model MPO stored densely. When the
    model MPO's D differs from D (generic tests), W is uniform too.
    """
    chi_out = chi if chi_out is None else chi_out
    tdt = TORCH_DTYPE[dtype]
    if model in ("heisenberg", "hubbard"):
        W, _, _ = model_mpo(model)
        assert W.shape == (D, D, d, d), (W.shape, D, d)
        if not tdt.is_complex:   # real dtypes: the model MPOs are real (exact imaginary zeros)
            assert not np.iscomplexobj(W) or not np.any(np.imag(W)), "model MPO is not real"
            W = np.ascontiguousarray(np.real(W))
        W1 = torch.from_numpy(W).to(tdt).to(device)
        W2 = W1.clone()
    else:
        W1 = random_tensor((D, D, d, d), dtype, seed, TID["W1"], device)
        W2 = random_tensor((D, D, d, d), dtype, seed, TID["W2"], device)
    return dict(
        L=random_tensor((chi, D, chi_out), dtype, seed, TID["L"], device),
        W1=W1, W2=W2,
        R=random_tensor((chi, D, chi_out), dtype, seed, TID["R"], device),
        psi=random_tensor((chi, d, d, chi), dtype, seed, TID["psi"], device),
    )


def heff_flops(chi: int, d: int, D: int, complex_: bool = True) -> float:
    """Algorithmic flops of one FLOP-optimal apply: 8 per complex MAC
    (2 per real MAC) times (2 D d^2 chi^3 + 2 D^2 d^3 chi^2)."""
    macs = 2 * D * d * d * chi ** 3 + 2 * D * D * d ** 3 * chi ** 2
    return macs * (8.0 if complex_ else 2.0)


TEBD_CONFIG = dict(chi=2048, d=2, dtype="r64", seed=4, tau=0.01, J=1.0, g=1.0)


def tebd_inputs(chi: int, d: int, dtype: str, seed: int, tau: float, J=1.0, g=1.0,
                device="cpu", physical_first: bool = False):
    """A[a,s,b], B[b,t,c] uniform; U = TFIM gate (complex dtypes: the
    real-time unitary expm(-i tau h)). Variant (ii) stores A as [s,a,b] and B
    as [t,b,c] (physical-first)."""
    shA = (d, chi, chi) if physical_first else (chi, d, chi)
    shB = (d, chi, chi) if physical_first else (chi, d, chi)
    A = random_tensor(shA, dtype, seed, TID["A"], device)
    B = random_tensor(shB, dtype, seed, TID["B"], device)
    U = torch.from_numpy(tfim_gate(tau, J, g, real_time=dtype in ("c64", "c128"))).to(TORCH_DTYPE[dtype]).to(device)
    return dict(A=A, B=B, U=U)


# ----------------------------------------------------------------------------
# structured inputs (dynamic range the paper's states carry: Schmidt spectra,
# Vidal-form weights, per-index scales). Each is a plain product of a uniform
# tensor with fixed scale vectors -- no arithmetic of the method.
# ----------------------------------------------------------------------------


def geometric_spectrum(n: int, smallest: float) -> np.ndarray:
    """lambda_i = smallest ** (i / (n - 1)), i = 0..n-1 (lambda_0 = 1): a
    graded Schmidt spectrum spanning [smallest, 1]."""
    if n == 1:
        return np.ones(1)
    return smallest ** (np.arange(n) / (n - 1))


def pow2_exponents(n: int, E: int, seed: int, tensor_id: int) -> np.ndarray:
    """n integers uniform in [-E, E] from the counter-based generator."""
    u = uniform_draws(seed, tensor_id, n).numpy()          # [-1, 1)
    return np.minimum(np.floor((u + 1.0) * 0.5 * (2 * E + 1)).astype(np.int64) - E, E)


def vidal_tebd_inputs(chi: int, d: int, seed: int, tau: float, smallest: float = 1e-10, dtype="r64"):
    """TEBD operands in Vidal form (Application A): with
    lambda_A, lambda_B geometric spectra down to ``smallest`` and X, Y
    uniform (the O(1) canonical tensors),
        A[a,s,b] = lambda_B[a] X[a,s,b] lambda_A[b]      (= lambda_B Gamma_A lambda_A)
        B[b,t,c] = Y[b,t,c] / lambda_A[b] * lambda_B[c]  (= Gamma_B lambda_B,
                                                          Gamma_B = lambda_A^-1 B_right)
    so A's columns and B's rows over the contracted bond b carry opposite
    scales (1 .. 1e-10 against 1 .. 1e10)."""
    lam_a = geometric_spectrum(chi, smallest)
    lam_b = geometric_spectrum(chi, smallest)
    X = random_np((chi, d, chi), dtype, seed, TID["A"])
    Y = random_np((chi, d, chi), dtype, seed, TID["B"])
    A = lam_b[:, None, None] * X * lam_a[None, None, :]
    B = Y / lam_a[:, None, None] * lam_b[None, None, :]
    U = tfim_gate(tau)
    return dict(A=torch.from_numpy(np.ascontiguousarray(A)), B=torch.from_numpy(np.ascontiguousarray(B)),
                U=torch.from_numpy(U).to(TORCH_DTYPE[dtype]), lam_a=lam_a, lam_b=lam_b)


# ----------------------------------------------------------------------------
# config 5: random contraction instances
# ----------------------------------------------------------------------------

SWEEP_DIMS = [1, 2, 3, 5, 7, 8, 16, 37, 64, 128, 256]


def sweep_instance(rng, max_elems: int = 2 ** 28, rank_min: int = 3, rank_max: int = 6):
    """One random pairwise contraction (labels and dims only, no data):
    orders r_A, r_B in [rank_min, rank_max], 1 <= #contracted < min(r_A, r_B),
    dims from SWEEP_DIMS, random label permutations of A, B and the output;
    the largest dim is halved until every tensor has <= max_elems elements.
    Returns (la, lb, lc, dims, shared_labels)."""
    import string
    ra, rb = int(rng.integers(rank_min, rank_max + 1)), int(rng.integers(rank_min, rank_max + 1))
    nc = int(rng.integers(1, min(ra, rb)))
    letters = list(string.ascii_letters)
    rng.shuffle(letters)
    sh, fa, fb = letters[:nc], letters[nc:ra], letters[ra:ra + rb - nc]
    la, lb, lc = sh + fa, sh + fb, fa + fb
    rng.shuffle(la)
    rng.shuffle(lb)
    rng.shuffle(lc)
    dims = {l: int(rng.choice(SWEEP_DIMS)) for l in la + lb}

    def size(ls):
        return int(np.prod([dims[l] for l in ls], dtype=np.int64))
    while max(size(la), size(lb), size(lc)) > max_elems:
        big = max(dims, key=dims.get)
        dims[big] = max(1, dims[big] // 2)
    return "".join(la), "".join(lb), "".join(lc), dims, "".join(sh)
