"""float32 / complex64 GEMMs on the INT8 tensor cores (-m gpu; R34).

The paper's examples are `float` (App. C) and the element field
is R or C (§II.A). Contractions of >= 4e9 MACs in float32 /
complex64 run the Ozaki-II scheme with a 24-bit budget (tci_ozaki_params_f32):
entries within a factor 2 of their line maximum are exact, integer products
and sums are exact, the result is rounded once to float32. The bar is the
north star's 1e-5 relative Frobenius error against the oracle (which widens
float32 inputs exactly to double and sums in double); the tests also compare
with the FP64-core path of the same library and check that the INT8 kernels
actually ran (profile counters) and that the guard falls back on a
cancelling product."""
import numpy as np
import pytest

import synth
from conftest import rel_frob

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2512_23917_b200 as tci  # noqa: E402


@pytest.fixture()
def ctx():
    c = tci.Context(0)
    c.ozaki_guard_stats(reset=True)
    yield c
    c.close()


def dev(x):
    t = torch.from_numpy(np.ascontiguousarray(x)) if isinstance(x, np.ndarray) else x
    return t.cuda()


def host(t):
    return t.cpu().numpy()


def run(ctx, A, la, B, lb, lc):
    tci.tci_profile_enable(ctx.handle, True)
    out = ctx.contract(dev(A), la, dev(B), lb, lc)
    i8 = tci.tci_profile_query(ctx.handle, tci.PROF_I8)
    tci.tci_profile_enable(ctx.handle, False)
    return out, i8


@pytest.mark.parametrize("K", [1000, 4096, 20480, 131072])
def test_f32_params(K):
    for cplx in (False, True):
        st, n, t, mods, ppm = tci.tci_ozaki_params_f32(K, cplx)
        assert st == 0 and t >= 24 and ppm == (2 if cplx else 1)
        M = 1
        for m in mods:
            M *= m
        assert 2 * K * 2 ** (2 * t) <= M // 4


@pytest.mark.parametrize("la,lb", [("mk", "kn"), ("km", "kn"), ("mk", "nk"), ("km", "nk")])
def test_f32_ozaki_contract_layouts(ctx, oracle_mod, la, lb):
    """r32, M = 2100, N = 1900, K = 1100 (4.4e9 MACs, ragged): all four
    operand layouts, oracle rows <= 1e-5 (in practice ~1e-7), agreement with
    the FP64-core path, INT8 path taken."""
    M, N, K = 2100, 1900, 1100
    A = synth.random_tensor((M, K), "r32", 801, 1)
    B = synth.random_tensor((K, N), "r32", 801, 2)
    At = A if la == "mk" else A.T.contiguous()
    Bt = B if lb == "kn" else B.T.contiguous()
    out, i8 = run(ctx, At, la, Bt, lb, "mn")
    assert i8["launches"] >= 1, "float32 Ozaki path not taken"
    assert out.dtype == torch.float32
    rows = [0, 1, 1050, M - 1]
    ref = oracle_mod.contract(A.numpy()[rows], "mk", B.numpy(), "kn", "mn")
    got = host(out)[rows]
    for i in range(len(rows)):
        assert rel_frob(got[i], ref[i]) <= 1e-5
    ctx.set_f32_algorithm(tci.TCI_F32_FP64_CORES)
    simt, i8s = run(ctx, At, la, Bt, lb, "mn")
    ctx.set_f32_algorithm(tci.TCI_F32_OZAKI_INT8)
    assert i8s["launches"] == 0
    assert rel_frob(host(out), host(simt)) <= 1e-6
    st = ctx.ozaki_guard_stats()
    assert st["gemms"] == 1 and st["fallbacks"] == 0, st


@pytest.mark.parametrize("la", ["mk", "km"])
def test_c64_ozaki_contract(ctx, oracle_mod, la):
    """c64 on the Gaussian moduli, M = 1500, N = 1300, K = 2100 (4.1e9 complex
    MACs): oracle rows <= 1e-5, agreement with the FP64-core path."""
    M, N, K = 1500, 1300, 2100
    A = synth.random_tensor((M, K), "c64", 803, 1)
    B = synth.random_tensor((K, N), "c64", 803, 2)
    At = A if la == "mk" else A.T.contiguous()
    out, i8 = run(ctx, At, la, B, "kn", "mn")
    assert i8["launches"] >= 1 and out.dtype == torch.complex64
    rows = [0, 749, M - 1]
    ref = oracle_mod.contract(A.numpy()[rows], "mk", B.numpy(), "kn", "mn")
    got = host(out)[rows]
    for i in range(len(rows)):
        assert rel_frob(got[i], ref[i]) <= 1e-5
    ctx.set_f32_algorithm(tci.TCI_F32_FP64_CORES)
    simt = ctx.contract(dev(At), la, dev(B), "kn", "mn")
    ctx.set_f32_algorithm(tci.TCI_F32_OZAKI_INT8)
    assert rel_frob(host(out), host(simt)) <= 1e-6


def test_f32_long_k_cancellation_full_contraction(ctx, oracle_mod):
    """R20's hard case for float32 accumulation: a long full contraction
    (K = 8880 here split as two legs) of uniform data, whose sums cancel. The
    INT8 path sums exactly: oracle rows <= 1e-5 (fp32 accumulation measured
    5.8e-5 on the same kind of product)."""
    M, N = 1024, 512
    A = synth.random_tensor((M, 120, 74), "r32", 805, 1)
    B = synth.random_tensor((74, 120, N), "r32", 805, 2)
    out, i8 = run(ctx, A, "mab", B, "ban", "mn")
    assert i8["launches"] >= 1
    rows = [0, 3, 511, M - 1]
    ref = oracle_mod.contract(A.numpy()[rows], "mab", B.numpy(), "ban", "mn")
    got = host(out)[rows]
    for i in range(len(rows)):
        assert rel_frob(got[i], ref[i]) <= 1e-5


def test_f32_guard_falls_back_on_cancelling_product(ctx, oracle_mod):
    """B = (I - Q Q^T) Y + 1e-4 Y2: C is ~1e4x smaller than |A||B| suggests,
    so 24-bit truncation errors exceed the float32 guard's 1e-7 relative to
    ||C||: the product is recomputed on the FP64 cores and meets 1e-5."""
    M, N, K = 1024, 1024, 4096
    A = synth.random_np((M, K), "r64", 807, 1)
    Y = synth.random_np((K, N), "r64", 807, 2)
    Y2 = synth.random_np((K, N), "r64", 807, 3)
    Q, _ = np.linalg.qr(A.T)
    B = (Y - Q @ (Q.T @ Y) + 1e-4 * Y2).astype(np.float32)
    A32 = A.astype(np.float32)
    out = ctx.contract(dev(A32), "mk", dev(B), "kn", "mn")
    st = ctx.ozaki_guard_stats()
    assert st["gemms"] == 1 and st["fallbacks"] == 1, st
    rows = [0, 1, 1023]
    ref = oracle_mod.contract(A32[rows], "mk", B, "kn", "mn")
    got = host(out)[rows]
    for i in range(len(rows)):
        assert rel_frob(got[i], ref[i]) <= 1e-5
