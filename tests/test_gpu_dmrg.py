"""The DMRG two-site update as one flow through the C ABI (-m gpu).

SURVEY 8(f2) says the truncated SVD "completes ... the DMRG two-site update"
(PAPER.md:55 cites DMRG; tci::trunc_svd PAPER.md:2055-2098). This test chains,
per bond of an open Heisenberg chain (L = 16, J = 1, complex128):

    theta = A_i . A_{i+1}                         tci_contract
    E, theta <- lowest eigenpair of H_eff         tci_heff_lanczos
    u, s, v^dag = trunc_svd(theta, chi_max)       tci_trunc_svd
    A_i = u,  A_{i+1} = s v^dag   (left sweep)    tci_contract
    L_{i+1} = L_i . A_i . W . A_i^*               tci_env_update

and the mirror image on the way back (R environments), for three sweeps from
a random right-canonical start. The converged energy is compared with exact
diagonalisation of the 2^16-dimensional Hamiltonian (scipy sparse Lanczos on
H = sum_i S_i . S_{i+1} assembled from Kronecker products: independent of the
product path and of the oracle), and the final MPS's <psi|H|psi> / <psi|psi>
computed by the CPU oracle's environment chain must equal the last Lanczos
energy (the truncation at chi = 64 keeps ~1e-10 of the weight)."""
import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2512_23917_b200 as tci  # noqa: E402

NSITES, CHI = 16, 64


def exact_ground_energy(n):
    import scipy.sparse as sp
    import scipy.sparse.linalg as sla
    sx = sp.csr_matrix(np.array([[0, 0.5], [0.5, 0]]))
    sy = sp.csr_matrix(np.array([[0, -0.5j], [0.5j, 0]]))
    sz = sp.csr_matrix(np.array([[0.5, 0], [0, -0.5]]))
    H = sp.csr_matrix((2 ** n, 2 ** n), dtype=np.complex128)
    for i in range(n - 1):
        for op in (sx, sy, sz):
            H = H + sp.kron(sp.kron(sp.identity(2 ** i), sp.kron(op, op)), sp.identity(2 ** (n - i - 2)))
    return float(sla.eigsh(H, k=1, which="SA", tol=1e-12)[0][0])


def diag(ctx, s, dtype):
    return torch.diag(s.to(dtype))


def test_dmrg_two_site_heisenberg_chain(oracle_mod):
    ctx = tci.Context(0)
    try:
        dt = torch.complex128
        W, lb, rb = synth.heisenberg_mpo(1.0)
        Wd = torch.from_numpy(W.astype(np.complex128)).cuda()
        bonds = [min(2 ** i, 2 ** (NSITES - i), CHI) for i in range(NSITES + 1)]
        A = [synth.random_tensor((bonds[i], 2, bonds[i + 1]), "c128", 901, 100 + i).cuda()
             for i in range(NSITES)]
        # right-canonical start: sweep SVDs from the right (tci_svd)
        for i in range(NSITES - 1, 0, -1):
            u, s, vd = ctx.svd(A[i], 1)
            A[i] = vd.contiguous()
            us = ctx.contract(u, "ak", diag(ctx, s, dt), "kl", "al")
            A[i - 1] = ctx.contract(A[i - 1], "xsa", us, "al", "xsl")
        Ls = [None] * (NSITES + 1)
        Rs = [None] * (NSITES + 1)
        Ls[0] = torch.from_numpy(synth.boundary_env(5, lb)).cuda()
        Rs[NSITES] = torch.from_numpy(synth.boundary_env(5, rb)).cuda()
        for i in range(NSITES - 1, 1, -1):
            Rs[i] = ctx.env_update(1, Rs[i + 1], A[i], Wd)
        energies = []
        for sweep in range(3):
            for direction in (+1, -1):
                order = range(NSITES - 1) if direction > 0 else range(NSITES - 2, -1, -1)
                for i in order:
                    theta = ctx.contract(A[i], "asb", A[i + 1], "btc", "astc")
                    e, _ = ctx.heff_lanczos(Ls[i], Wd, Wd, Rs[i + 2], theta, max_iter=40, tol=1e-13)
                    energies.append(e)
                    u, s, vd, err = ctx.trunc_svd(theta, 2, 1, CHI, 0.0, 1e-14)
                    if direction > 0:
                        A[i] = u.contiguous()
                        A[i + 1] = ctx.contract(diag(ctx, s, dt), "kl", vd, "ltc", "ktc")
                        Ls[i + 1] = ctx.env_update(0, Ls[i], A[i], Wd)
                    else:
                        A[i + 1] = vd.contiguous()
                        A[i] = ctx.contract(u, "ask", diag(ctx, s, dt), "kl", "asl")
                        Rs[i + 1] = ctx.env_update(1, Rs[i + 2], A[i + 1], Wd)
        torch.cuda.synchronize()
        e_ed = exact_ground_energy(NSITES)
        assert abs(energies[-1] - e_ed) < 1e-7, (energies[-1], e_ed)
        # variational and converged: the last sweep's energies lie within 1e-7 of each other
        last = energies[-2 * (NSITES - 1):]
        assert max(last) - min(last) < 1e-7
        assert min(energies) >= e_ed - 1e-9
        # the oracle's <psi|H|psi> / <psi|psi> of the final MPS (CPU environment chain)
        sites = [a.cpu().numpy() for a in A]
        E = synth.boundary_env(5, lb)
        N = np.ones((1, 1, 1), dtype=np.complex128)
        I_mpo = np.eye(2, dtype=np.complex128).reshape(1, 1, 2, 2)
        for a in sites:
            E = oracle_mod.env_left(E, a, W.astype(np.complex128))
            N = oracle_mod.env_left(N, a, I_mpo)
        e_or = (E[0, rb, 0] / N[0, 0, 0]).real
        assert abs(e_or - energies[-1]) < 1e-9, (e_or, energies[-1])
    finally:
        ctx.close()
