"""Design model (numpy) of the GPU block one-sided Jacobi SVD in
csrc/kernels/svd.cu -- NOT the oracle and not used by tests or the product:
it checks the rotation formulas, the pairing schedule and the convergence
test before they are written in CUDA.  python tools/svd_model.py
"""
import numpy as np

SB = 16          # rows per block
PR = 2 * SB      # rows per block pair


def rr_pair(nb, r, p):
    m = nb - 1
    if p == 0:
        return m, r
    return (r + p) % m, (r - p + m) % m


def inner_eig(H, eps=np.finfo(float).eps, max_sweeps=20):
    """Parallel cyclic Jacobi on a PR x PR Hermitian matrix, the same step
    structure as the kernel: per step 16 disjoint pairs, rotations computed
    from the old H, then H <- J^H H J blockwise and G <- G J."""
    n = H.shape[0]
    H = H.astype(complex).copy()
    G = np.eye(n, dtype=complex)
    sweeps = 0
    for sw in range(max_sweeps):
        rotated = False
        for step in range(n - 1):
            Js = []
            for p in range(n // 2):
                a_, b_ = rr_pair(n, step, p)
                i, j = min(a_, b_), max(a_, b_)
                a = H[i, i].real
                d = H[j, j].real
                h = H[i, j]
                ah = abs(h)
                if ah == 0 or ah <= eps * np.sqrt(abs(a * d)):
                    J = np.eye(2, dtype=complex)
                    Js.append((i, j, J, None))
                    continue
                rotated = True
                tau = (d - a) / (2 * ah)
                t = (1.0 if tau >= 0 else -1.0) / (abs(tau) + np.sqrt(1 + tau * tau))
                c = 1 / np.sqrt(1 + t * t)
                s = t * c
                ph = np.conj(h) / ah
                J = np.array([[c, s], [-s * ph, c * ph]])
                Js.append((i, j, J, (a - t * ah, d + t * ah)))
            Hn = H.copy()
            for u, (iu, ju, Ju, du) in enumerate(Js):
                for v, (iv, jv, Jv, dv) in enumerate(Js):
                    if u > v:
                        continue
                    B = np.array([[H[iu, iv], H[iu, jv]], [H[ju, iv], H[ju, jv]]])
                    if u == v:
                        Bp = np.diag(du) if du is not None else np.diag([B[0, 0].real, B[1, 1].real])
                    else:
                        Bp = Ju.conj().T @ B @ Jv
                    Hn[iu, iv], Hn[iu, jv], Hn[ju, iv], Hn[ju, jv] = Bp[0, 0], Bp[0, 1], Bp[1, 0], Bp[1, 1]
                    if u < v:
                        Hn[iv, iu], Hn[jv, iu], Hn[iv, ju], Hn[jv, ju] = (np.conj(Bp[0, 0]), np.conj(Bp[0, 1]),
                                                                          np.conj(Bp[1, 0]), np.conj(Bp[1, 1]))
            for (iv, jv, Jv, _) in Js:
                gi, gj = G[:, iv].copy(), G[:, jv].copy()
                G[:, iv] = gi * Jv[0, 0] + gj * Jv[1, 0]
                G[:, jv] = gi * Jv[0, 1] + gj * Jv[1, 1]
            H = Hn
        sweeps += 1
        if not rotated:
            break
    ev = H.diagonal().real
    order = sorted(range(n), key=lambda i: (-ev[i], i))
    return ev[order], G[:, order], sweeps


def jacobi_svd(A, tol=1e-13, max_sweeps=40):
    A = np.asarray(A)
    I, J = A.shape
    wide = I <= J
    X0 = A if wide else A.conj().T
    nr, L = X0.shape
    npad = -(-nr // PR) * PR
    X = np.zeros((npad, L), dtype=complex)
    X[:nr] = X0
    Y = np.eye(npad, dtype=complex)
    nb = npad // SB
    sweeps = 0
    for sw in range(max_sweeps):
        offmax = 0.0
        for r in range(nb - 1):
            for p in range(nb // 2):
                a, b = rr_pair(nb, r, p)
                lo, hi = min(a, b), max(a, b)
                rows = list(range(lo * SB, lo * SB + SB)) + list(range(hi * SB, hi * SB + SB))
                Xb = X[rows]
                H = Xb @ Xb.conj().T
                dg = H.diagonal().real
                off = 0.0
                for i in range(PR):
                    for j in range(i + 1, PR):
                        if dg[i] > 0 and dg[j] > 0:
                            off = max(off, abs(H[i, j]) / np.sqrt(dg[i] * dg[j]))
                offmax = max(offmax, off)
                if off <= tol:
                    continue
                ev, G, _ = inner_eig(H)
                X[rows] = G.conj().T @ Xb
                Y[rows] = G.conj().T @ Y[rows]
        sweeps += 1
        if offmax <= tol:
            break
    s = np.sqrt(np.sum(np.abs(X) ** 2, axis=1))
    order = sorted(range(npad), key=lambda i: (-s[i], i))[:min(I, J)]
    s = s[order]
    if wide:
        U = Y[order].conj().T[:I]
        Vh = X[order] / s[:, None]
    else:
        U = (X[order] / s[:, None]).conj().T
        Vh = Y[order][:, :J]
    return U, s, Vh, sweeps


if __name__ == "__main__":
    rng = np.random.default_rng(0)
    for (I, J, cplx) in [(40, 70, False), (70, 40, True), (64, 64, True), (33, 100, False)]:
        A = rng.uniform(-1, 1, (I, J)) + (1j * rng.uniform(-1, 1, (I, J)) if cplx else 0)
        U, s, Vh, sw = jacobi_svd(A)
        s_ref = np.linalg.svd(A, compute_uv=False)
        rec = np.linalg.norm(U @ np.diag(s) @ Vh - A) / np.linalg.norm(A)
        k = min(I, J)
        print(f"{I}x{J} cplx={cplx}: sweeps {sw}, |s-s_ref|/s0 {np.max(np.abs(s - s_ref)) / s_ref[0]:.2e}, "
              f"rec {rec:.2e}, |UhU-I| {np.abs(U.conj().T @ U - np.eye(k)).max():.2e}, "
              f"|VVh-I| {np.abs(Vh @ Vh.conj().T - np.eye(k)).max():.2e}")
    # rank-deficient (TEBD-like): theta = A B with an inner bond of 24 < 48
    A = rng.uniform(-1, 1, (48, 24)) @ rng.uniform(-1, 1, (24, 48))
    U, s, Vh, sw = jacobi_svd(A)
    s_ref = np.linalg.svd(A, compute_uv=False)
    print(f"rank-24 48x48: sweeps {sw}, |s-s_ref|/s0 {np.max(np.abs(s - s_ref)) / s_ref[0]:.2e}, "
          f"rec {np.linalg.norm(U @ np.diag(s) @ Vh - A) / np.linalg.norm(A):.2e}, "
          f"|VVh-I| {np.abs(Vh @ Vh.conj().T - np.eye(48)).max():.2e}")
