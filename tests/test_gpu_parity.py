"""GPU parity tests (-m gpu): the CUDA path through the C ABI vs the CPU oracle
on the same seeded inputs (synth). Tolerances (BASELINE.json north_star,
DESIGN.md "Parity"): relative Frobenius <= 1e-12 for float64/complex128,
<= 1e-5 for float32/complex64; bitwise for permutes, identities and
repeatability."""
import os
import subprocess
import sys

import numpy as np
import pytest

import synth
from conftest import ROOT, rel_frob

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2512_23917_b200 as tci  # noqa: E402

TOL = {"r64": 1e-12, "c128": 1e-12, "r32": 1e-5, "c64": 1e-5}


@pytest.fixture(scope="module")
def ctx():
    c = tci.Context(0)
    yield c
    c.close()


def dev(x, dt=None):
    t = torch.from_numpy(np.ascontiguousarray(x)) if isinstance(x, np.ndarray) else x
    if dt is not None:
        t = t.to(synth.TORCH_DTYPE[dt])
    return t.cuda()


def host(t):
    return t.cpu().numpy()


# ---------------------------------------------------------------------------
# permute (8(a2)): bitwise
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("dt", ["r32", "r64", "c64", "c128"])
def test_permute_bitwise(ctx, oracle_mod, dt):
    rng = np.random.default_rng(7)
    shapes = [(37, 130, 65), (64, 64), (3, 1, 5, 1, 7, 2), (2, 3, 4, 5, 6), (129,), (1,), (5, 1)]
    for i, shape in enumerate(shapes):
        x = synth.random_tensor(shape, dt, 500 + i, 1)
        for _ in range(4):
            perm = list(rng.permutation(len(shape)))
            y = ctx.permute(dev(x), perm)
            ref = oracle_mod.permute(x.numpy(), perm)
            assert np.array_equal(host(y).astype(ref.dtype), ref), (shape, perm)


@pytest.mark.parametrize("dt", ["r32", "r64", "c128"])
def test_permute_leg_groups_bitwise(ctx, oracle_mod, dt):
    """Leg-group tiles: short contiguous legs grouped, long legs cut into
    chunks with ragged last chunks, up to 7 legs; bitwise vs the oracle."""
    rng = np.random.default_rng(11)
    shapes = [(5, 7, 3, 11), (2, 3, 2, 5, 2, 7, 3), (1000, 3, 5), (3, 5, 1031), (37, 130, 65, 2),
              (17, 2, 513, 3), (64, 1, 64, 5), (6, 4000), (4000, 6), (2, 2, 2, 2, 2, 2, 2)]
    for i, shape in enumerate(shapes):
        x = synth.random_tensor(shape, dt, 700 + i, 1)
        for _ in range(5):
            perm = list(rng.permutation(len(shape)))
            y = ctx.permute(dev(x), perm)
            ref = oracle_mod.permute(x.numpy(), perm)
            assert np.array_equal(host(y).astype(ref.dtype), ref), (shape, perm)


def test_permute_tiled_kernels_bitwise():
    """Tensors up to 8 MB take permute_small; the tiled kernels (row copies,
    2-D transpose tiles, leg-group tiles with cut legs and ragged chunks) are
    run here on the same shapes with TCI_PERMUTE_SMALL=0 (read once per
    process: a child process), bitwise vs the oracle for r32 / r64 / c128."""
    code = (
        "import numpy as np, torch, synth, oracle, paper_2512_23917_b200 as t\n"
        "c = t.Context(0)\n"
        "rng = np.random.default_rng(11)\n"
        "shapes = [(5, 7, 3, 11), (2, 3, 2, 5, 2, 7, 3), (1000, 3, 5), (3, 5, 1031), (37, 130, 65, 2),\n"
        "          (17, 2, 513, 3), (64, 1, 64, 5), (6, 4000), (4000, 6), (2, 2, 2, 2, 2, 2, 2), (37, 130, 65)]\n"
        "n = 0\n"
        "for dt in ('r32', 'r64', 'c128'):\n"
        "    for i, shape in enumerate(shapes):\n"
        "        x = synth.random_tensor(shape, dt, 700 + i, 1)\n"
        "        for _ in range(4):\n"
        "            perm = list(rng.permutation(len(shape)))\n"
        "            y = c.permute(x.cuda(), perm)\n"
        "            ref = oracle.permute(x.numpy(), perm)\n"
        "            assert np.array_equal(y.cpu().numpy().astype(ref.dtype), ref), (dt, shape, perm)\n"
        "            n += 1\n"
        "print('checked', n)\n")
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, cwd=ROOT,
                       env=dict(os.environ, TCI_PERMUTE_SMALL="0"))
    assert r.returncode == 0, r.stderr[-3000:]
    assert "checked 132" in r.stdout


def test_ab_switch_fallback_paths():
    """The A/B switches keep their kernels correct: TCI_CRT_MMA=0 (the CUDA-core
    Gaussian CRT), TCI_F32_DMMA=0 (the SIMT float32 GEMM) and
    TCI_SKINNY_EXPAND=0 (the streaming kernel for expansion layouts), in a
    child process, against the oracle."""
    code = (
        "import numpy as np, torch, synth, oracle, paper_2512_23917_b200 as t\n"
        "def rel(a, b): return float(np.linalg.norm(a - b) / np.linalg.norm(b))\n"
        "c = t.Context(0); c.set_gemm_algorithm(t.TCI_GEMM_OZAKI_INT8)\n"
        "A = synth.random_tensor((1029, 4100), 'c128', 5, 1); B = synth.random_tensor((4100, 1040), 'c128', 5, 2)\n"
        "C = c.contract(A.cuda(), 'mk', B.cuda(), 'kn', 'mn').cpu().numpy()\n"
        "st = c.ozaki_guard_stats(); assert st['gemms'] == 1 and st['fallbacks'] == 0, st\n"
        "rows = [0, 514, 1028]\n"
        "e1 = rel(C[rows], oracle.contract(A.numpy()[rows], 'mk', B.numpy(), 'kn', 'mn'))\n"
        "X = synth.random_tensor((300, 700), 'r32', 5, 3); Y = synth.random_tensor((700, 200), 'r32', 5, 4)\n"
        "Z = c.contract(X.cuda(), 'mk', Y.cuda(), 'kn', 'mn').cpu().numpy()\n"
        "e2 = rel(Z.astype(np.float64), oracle.contract(X.numpy().astype(np.float64), 'mk', Y.numpy().astype(np.float64), 'kn', 'mn'))\n"
        "P = synth.random_tensor((7, 3, 301), 'c128', 5, 5); W = synth.random_tensor((4, 4, 3, 3), 'c128', 5, 6)\n"
        "Q = c.contract(P.cuda(), 'asb', W.cuda(), 'wvst', 'awtbv').cpu().numpy()\n"
        "e3 = rel(Q.reshape(-1), oracle.mps_mpo_apply(P.numpy(), W.numpy()).reshape(-1))\n"
        "U = synth.random_tensor((130, 300), 'c64', 5, 7); V = synth.random_tensor((300, 90), 'c64', 5, 8)\n"
        "c.set_f32_algorithm(t.TCI_F32_FP64_CORES)\n"
        "Wc = c.contract(U.cuda(), 'mk', V.cuda(), 'kn', 'mn').cpu().numpy()\n"
        "e4 = rel(Wc.astype(np.complex128), oracle.contract(U.numpy().astype(np.complex128), 'mk', V.numpy().astype(np.complex128), 'kn', 'mn'))\n"
        "print('errs', e1, e2, e3, e4)\n"
        "assert e1 <= 1e-12 and e2 <= 1e-5 and e3 <= 1e-12 and e4 <= 1e-5\n")
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, cwd=ROOT,
                       env=dict(os.environ, TCI_CRT_MMA="0", TCI_F32_DMMA="0", TCI_SKINNY_EXPAND="0"))
    assert r.returncode == 0, r.stderr[-3000:]
    assert "errs" in r.stdout


@pytest.mark.parametrize("dt", ["r32", "c128"])
def test_permute_large_tiled_bitwise(ctx, oracle_mod, dt):
    """Tensors above the 8 MB small-permute bound in the default process:
    the tiled kernels, bitwise vs the oracle."""
    rng = np.random.default_rng(12)
    for i, shape in enumerate([(7, 300, 5, 300), (64, 37, 130, 9), (3, 5, 1031, 300)]):
        x = synth.random_tensor(shape, dt, 800 + i, 1)
        for _ in range(2):
            perm = list(rng.permutation(len(shape)))
            y = ctx.permute(dev(x), perm)
            ref = oracle_mod.permute(x.numpy(), perm)
            assert np.array_equal(host(y).astype(ref.dtype), ref), (shape, perm)


def test_permute_paper_example(ctx):
    a = synth.random_tensor((3, 2, 4), "r64", 12, 1)
    a2 = ctx.permute(dev(a), [1, 0, 2])
    assert host(a2)[0, 1, 0] == a.numpy()[1, 0, 0]
    assert tuple(ctx.permute(a2, [2, 1, 0]).shape) == (4, 3, 2)


# ---------------------------------------------------------------------------
# contract (8(a1), 8(a4), 8(a6))
# ---------------------------------------------------------------------------

def test_paper_contract_example(ctx, oracle_mod):
    a = synth.random_tensor((3, 4, 2), "r64", 11, 1)
    b = synth.random_tensor((2, 4, 5), "r64", 11, 2)
    c1 = ctx.contract(dev(a), [1, -1, -2], dev(b), [-2, -1, 0], [0, 1])
    c2 = ctx.contract(dev(a), "ijk", dev(b), "kjl", "li")
    assert tuple(c1.shape) == (5, 3)
    assert torch.equal(c1, c2)
    assert rel_frob(host(c2), oracle_mod.contract(a.numpy(), "ijk", b.numpy(), "kjl", "li")) <= 1e-12


def _random_instance(rng, big=False):
    import string
    ra = int(rng.integers(1, 5))
    rb = int(rng.integers(1, 5))
    nc = int(rng.integers(0, min(ra, rb) + 1))
    letters = list(string.ascii_letters)
    rng.shuffle(letters)
    shared = letters[:nc]
    fa = letters[nc:ra]
    fb = letters[ra:ra + rb - nc]
    la, lb, lc = shared + fa, shared + fb, fa + fb
    rng.shuffle(la); rng.shuffle(lb); rng.shuffle(lc)
    pool = [1, 2, 3, 5, 7, 8, 16, 37] if big else [1, 2, 3, 4, 5]
    dims = {l: int(rng.choice(pool)) for l in la + lb}
    return "".join(la), "".join(lb), "".join(lc), dims


@pytest.mark.parametrize("dt", ["r64", "c128", "r32", "c64"])
@pytest.mark.parametrize("big", [False, True])
def test_contract_random_sweep(ctx, oracle_mod, dt, big):
    rng = np.random.default_rng(2024 + big)
    for i in range(60):
        la, lb, lc, dims = _random_instance(rng, big)
        A = synth.random_tensor([dims[l] for l in la], dt, 1000 + i, 1)
        B = synth.random_tensor([dims[l] for l in lb], dt, 1000 + i, 2)
        C = ctx.contract(dev(A), la, dev(B), lb, lc)
        ref = oracle_mod.contract(A.numpy(), la, B.numpy(), lb, lc)
        assert rel_frob(host(C), ref) <= TOL[dt], (la, lb, lc, dims)


@pytest.mark.parametrize("dt", ["r64", "c128"])
def test_gemm_layouts_ragged(ctx, oracle_mod, dt):
    """All four operand major-ness combinations, sizes spanning several tiles
    with ragged tails (M=133, N=77, K=259), read in place (no permute)."""
    M, N, K = 133, 77, 259
    A = synth.random_tensor((M, K), dt, 77, 1)
    B = synth.random_tensor((K, N), dt, 77, 2)
    ref = oracle_mod.contract(A.numpy(), "mk", B.numpy(), "kn", "mn")
    for la, At in (("mk", A), ("km", A.T.contiguous())):
        for lb, Bt in (("kn", B), ("nk", B.T.contiguous())):
            for lc in ("mn", "nm"):
                C = ctx.contract(dev(At), la, dev(Bt), lb, lc)
                r = ref if lc == "mn" else ref.T
                assert rel_frob(host(C), r) <= 1e-12, (la, lb, lc)


@pytest.mark.parametrize("dt", ["r64", "c128", "r32", "c64"])
def test_thin_side_boundaries(ctx, oracle_mod, dt):
    """Thin / outer-product GEMM routing at every width boundary (1, 2, 4, 8,
    16, 17, 32, 33 on either side, K short and long, both A layouts): the thin
    kernels take min(M, N) <= 32 real / 16 complex, the outer kernel K <= 16."""
    for thin in (1, 2, 3, 8, 16, 17, 24, 32, 33):
        for big, K in ((300, 7), (300, 259), (1000, 16), (129, 1100)):
            A = synth.random_tensor((thin, K), dt, 88 + thin, 1)
            B = synth.random_tensor((K, big), dt, 88 + thin, 2)
            ref = oracle_mod.contract(A.numpy(), "mk", B.numpy(), "kn", "mn")
            for la, At in (("mk", A), ("km", A.T.contiguous())):
                for lc in ("mn", "nm"):
                    C = ctx.contract(dev(At), la, dev(B), "kn", lc)
                    r = ref if lc == "mn" else ref.T
                    assert rel_frob(host(C), r) <= TOL[dt], (thin, big, K, la, lc)
                    C = ctx.contract(dev(B), "kn", dev(At), la, lc)   # operands swapped
                    assert rel_frob(host(C), r) <= TOL[dt], ("swap", thin, big, K, la, lc)


@pytest.mark.parametrize("dt", ["r64", "c128", "r32", "c64"])
def test_splitk_small_output_long_k(ctx, oracle_mod, dt):
    """Few output tiles and a long K take the deterministic split-K path
    (partial GEMMs + ascending-order reduction): parity and repeatability."""
    A = synth.random_tensor((5, 37, 700), dt, 86, 1)      # m=5, k=(37, 700)
    B = synth.random_tensor((700, 37, 9), dt, 86, 2)
    C1 = ctx.contract(dev(A), "mkl", dev(B), "lkn", "nm")
    C2 = ctx.contract(dev(A), "mkl", dev(B), "lkn", "nm")
    assert torch.equal(C1, C2)
    ref = oracle_mod.contract(A.numpy(), "mkl", B.numpy(), "lkn", "nm")
    assert rel_frob(host(C1), ref) <= TOL[dt]
    # full contraction to a scalar (the sweep's worst case before split-K)
    s = ctx.contract(dev(A), "mkl", dev(A), "mkl", "")
    assert rel_frob(host(s), oracle_mod.contract(A.numpy(), "mkl", A.numpy(), "mkl", "")) <= TOL[dt]


def test_higham_elementwise_bound(ctx, oracle_mod):
    """Per element |C_gpu - C_oracle| <= 2 gamma_K (|A|.|B|): catches local bugs
    that a Frobenius average could hide."""
    A = synth.random_tensor((150, 300), "r64", 78, 1).numpy()
    B = synth.random_tensor((300, 90), "r64", 78, 2).numpy()
    C = host(ctx.contract(dev(A), "ik", dev(B), "kj", "ij"))
    ref = oracle_mod.contract(A, "ik", B, "kj", "ij")
    bound = oracle_mod.contract_abs(A, "ik", B, "kj", "ij")
    K, u = 300, 2.0 ** -53
    gam = K * u / (1 - K * u)
    assert np.all(np.abs(C - ref) <= 2 * gam * bound)


@pytest.mark.parametrize("dt", ["r64", "c128"])
def test_identity_contraction_bitwise(ctx, dt):
    a = synth.random_tensor((133, 70), dt, 79, 1)
    eye = torch.eye(70, dtype=synth.TORCH_DTYPE[dt])
    c = ctx.contract(dev(a), "ij", dev(eye), "jk", "ik")
    assert torch.equal(c.cpu(), a)


def test_outer_scalar_and_empty_gamma(ctx, oracle_mod):
    a = synth.random_tensor((3, 40), "c128", 80, 1)
    b = synth.random_tensor((33,), "c128", 80, 2)
    c = ctx.contract(dev(a), "ij", dev(b), "k", "kji")
    assert rel_frob(host(c), oracle_mod.contract(a.numpy(), "ij", b.numpy(), "k", "kji")) <= 1e-15
    x = synth.random_tensor((2,) * 6, "r64", 81, 1)
    y = synth.random_tensor((2,) * 6, "r64", 81, 2)
    s = ctx.contract(dev(x), "ijklmn", dev(y), "ijklmn", "")
    assert s.shape == () and abs(s.item() - float(oracle_mod.contract(x.numpy(), "ijklmn", y.numpy(), "ijklmn", ""))) <= 1e-14


def test_aliasing_output(ctx, oracle_mod):
    """correct even when c aliases a."""
    a = synth.random_tensor((64, 48), "c128", 82, 1)
    b = synth.random_tensor((48, 48), "c128", 82, 2)
    ref = oracle_mod.contract(a.numpy(), "ij", b.numpy(), "jk", "ik")
    ad = dev(a)
    ctx.contract(ad, "ij", dev(b), "jk", "ik", out=ad)
    assert rel_frob(host(ad), ref) <= 1e-12
    ad = dev(a)
    ctx.contract(ad, "ij", dev(b), "jk", "ki", out=ad.view(48, 64))
    assert rel_frob(host(ad).reshape(48, 64), ref.T) <= 1e-12


def test_relabel_invariance_bitwise(ctx):
    A = dev(synth.random_tensor((40, 30, 20), "c128", 83, 1))
    B = dev(synth.random_tensor((20, 30, 50), "c128", 83, 2))
    c1 = ctx.contract(A, "ikl", B, "lkj", "ji")
    c2 = ctx.contract(A, [7, -3, 100], B, [100, -3, 42], [42, 7])
    assert torch.equal(c1, c2)


def test_repeatability_bitwise(ctx):
    A = dev(synth.random_tensor((300, 257), "c128", 84, 1))
    B = dev(synth.random_tensor((257, 301), "c128", 84, 2))
    c1 = ctx.contract(A, "ik", B, "kj", "ij")
    c2 = ctx.contract(A, "ik", B, "kj", "ij")
    assert torch.equal(c1, c2)
    # row-sharded A gives bitwise identical rows (per-element k order fixed)
    c3 = ctx.contract(A[100:200].contiguous(), "ik", B, "kj", "ij")
    assert torch.equal(c3, c1[100:200])


def test_errors(ctx):
    a = dev(torch.zeros(2, 3, dtype=torch.float64))
    b = dev(torch.zeros(3, 4, dtype=torch.float64))
    c = dev(torch.zeros(2, 4, dtype=torch.float64))
    ha, hb, hc = ctx.tensor(a), ctx.tensor(b), ctx.tensor(c)
    tci.tci_contract_str(ctx.handle, ha, "ij", hb, "jk", hc, "ik")
    with pytest.raises(tci.TciError) as e:
        tci.tci_contract_str(ctx.handle, ha, "ii", hb, "jk", hc, "ik")
    assert e.value.code == 4
    with pytest.raises(tci.TciError) as e:
        tci.tci_contract_str(ctx.handle, ha, "ij", hb, "jk", hc, "ijk")
    assert e.value.code == 2
    with pytest.raises(tci.TciError) as e:
        tci.tci_contract_str(ctx.handle, ha, "ij", hb, "jk", hc, "ki")   # c shape (2,4) != (4,2)
    assert e.value.code == 1
    with pytest.raises(tci.TciError) as e:
        tci.tci_contract_str(ctx.handle, ha, "ij", hb, "ik", hc, "jk")   # i: 2 vs 3
    assert e.value.code == 1
    with pytest.raises(tci.TciError) as e:
        tci.tci_contract_str(ctx.handle, ha, "ij", hb, "jk", hc, "iz")
    assert e.value.code == 4
    f = dev(torch.zeros(3, 4, dtype=torch.float32))
    with pytest.raises(tci.TciError) as e:
        tci.tci_contract_str(ctx.handle, ha, "ij", ctx.tensor(f), "jk", hc, "ik")
    assert e.value.code == 7
    with pytest.raises(tci.TciError) as e:
        tci.tci_tensor_create(ctx.handle, tci.TCI_R64, (2, 0), a.data_ptr())
    assert e.value.code == 3
    with pytest.raises(tci.TciError) as e:
        tci.tci_reshape(ctx.handle, ha, (5,))
    assert e.value.code == 1
    with pytest.raises(tci.TciError) as e:
        tci.tci_permute(ctx.handle, ha, [0, 0], hc)
    assert e.value.code == 8
    # host memory passed to compute -> UNSUPPORTED
    hbuf = torch.zeros(2, 3, dtype=torch.float64)
    hh = tci.tci_tensor_create(ctx.handle, tci.TCI_R64, (2, 3), hbuf.data_ptr())
    with pytest.raises(tci.TciError) as e:
        tci.tci_contract_str(ctx.handle, hh, "ij", hb, "jk", hc, "ik")
    assert e.value.code == 7
    tci.tci_tensor_free(ctx.handle, hh)


def test_errors_round2_entry_points():
    """The round-2 ABI calls validate their arguments: unknown float32 / Ozaki
    complex variants are INVALID_ARGUMENT; graph capture rejects a second
    begin, an end without begin and the legacy NULL stream; a dead context
    answers DEAD_CONTEXT."""
    c0 = tci.Context(0, torch.cuda.default_stream(0))    # the legacy NULL stream
    try:
        with pytest.raises(tci.TciError) as e:
            tci.tci_graph_begin(c0.handle)
        assert e.value.code == 8
    finally:
        c0.close()
    c = tci.Context(0, torch.cuda.Stream())
    with pytest.raises(tci.TciError) as e:
        tci.tci_set_f32_algorithm(c.handle, 7)
    assert e.value.code == 8                              # INVALID_ARGUMENT
    with pytest.raises(tci.TciError) as e:
        tci.tci_set_ozaki_complex(c.handle, 9)
    assert e.value.code == 8
    st, *_ = tci.tci_ozaki_params_complex(4096, 5)
    assert st == 8
    with pytest.raises(tci.TciError):
        tci.tci_graph_end(c.handle)                       # not capturing
    tci.tci_graph_begin(c.handle)
    with pytest.raises(tci.TciError):
        tci.tci_graph_begin(c.handle)                     # already capturing
    g = tci.tci_graph_end(c.handle)                       # an empty graph is a valid graph
    tci.tci_graph_launch(c.handle, g)
    tci.tci_graph_destroy(g)
    h = c.handle
    c.close()                                             # the handle stays valid but dead
    for fn, args in ((tci.tci_set_f32_algorithm, (0,)), (tci.tci_set_ozaki_complex, (0,)),
                     (tci.tci_graph_begin, ())):
        with pytest.raises(tci.TciError) as e:
            fn(h, *args)
        assert e.value.code == 6                          # DEAD_CONTEXT


def test_workspace_and_dead_context(oracle_mod):
    c = tci.Context(0)
    a = dev(synth.random_tensor((4, 5, 6), "r64", 85, 1))
    b = dev(synth.random_tensor((6, 4, 7), "r64", 85, 2))
    out = dev(torch.zeros(7, 5, dtype=torch.float64))
    ha, hb, ho = c.tensor(a), c.tensor(b), c.tensor(out)
    need = tci.tci_contract_workspace_size(c.handle, ha, "ijk", hb, "kil", ho, "lj")
    assert need > 0
    with pytest.raises(tci.TciError) as e:
        tci.tci_contract_str(c.handle, ha, "ijk", hb, "kil", ho, "lj")
    assert e.value.code == 9
    assert torch.count_nonzero(out).item() == 0      # nothing launched on error
    c.ensure_workspace(need)
    tci.tci_contract_str(c.handle, ha, "ijk", hb, "kil", ho, "lj")
    ref = oracle_mod.contract(a.cpu().numpy(), "ijk", b.cpu().numpy(), "kil", "lj")
    assert rel_frob(host(out), ref) <= 1e-12
    h = c.handle
    c.free_descriptors()
    tci.tci_destroy_context(h)
    with pytest.raises(tci.TciError) as e:
        tci.tci_destroy_context(h)
    assert e.value.code == 6
    with pytest.raises(tci.TciError) as e:
        tci.tci_synchronize(h)
    assert e.value.code == 6
    c.handle = 0


def test_verbose_lines():
    code = (
        "import torch, paper_2512_23917_b200 as t\n"
        "c=t.Context(0)\n"
        "a=torch.ones(3,4,dtype=torch.float64,device='cuda'); b=torch.ones(4,5,dtype=torch.float64,device='cuda')\n"
        "c.contract(a,'ij',b,'jk','ik'); torch.cuda.synchronize()\n")
    for lvl, pat in (("1", "tci:contract shapes=[3,4;4,5;3,5] dtype=r64"), ("2", "time_us=")):
        r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, cwd=ROOT,
                           env=dict(os.environ, TCI_VERBOSE=lvl))
        assert r.returncode == 0, r.stderr
        assert pat in r.stderr, r.stderr
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, cwd=ROOT,
                       env=dict(os.environ, TCI_VERBOSE="0"))
    assert "tci:" not in r.stderr


# ---------------------------------------------------------------------------
# H_eff (8(a5), 8(a7))
# ---------------------------------------------------------------------------

def _heff_np(inp):
    return {k: v.numpy() for k, v in inp.items()}


@pytest.mark.parametrize("dt", ["c128", "r64"])
@pytest.mark.parametrize("chi,d,D,model", [(1, 2, 5, "heisenberg"), (3, 2, 5, "heisenberg"),
                                           (37, 2, 5, "heisenberg"), (70, 2, 3, "random"),
                                           (20, 4, 6, "hubbard"), (9, 3, 4, "random")])
def test_heff_small(ctx, oracle_mod, dt, chi, d, D, model):
    if dt == "r64" and model != "random":
        model = "random"
    inp = synth.heff_inputs(chi, d, D, dt, 300 + chi, model)
    gpu = ctx.heff_apply(*[dev(inp[k]) for k in ("L", "W1", "W2", "R", "psi")])
    n = _heff_np(inp)
    ref = oracle_mod.heff(n["L"], n["W1"], n["W2"], n["R"], n["psi"])
    assert rel_frob(host(gpu), ref) <= 1e-12


def test_heff_rectangular_and_generic_tree(ctx, oracle_mod):
    """chi_l != chi_r and a lopsided case where the planner picks another tree."""
    for (cl, clo, cr, cro) in [(30, 20, 50, 40), (64, 64, 2, 2)]:
        L = synth.random_tensor((cl, 5, clo), "c128", 310, 1)
        R = synth.random_tensor((cr, 5, cro), "c128", 310, 5)
        psi = synth.random_tensor((cl, 2, 2, cr), "c128", 310, 2)
        W = torch.from_numpy(synth.heisenberg_mpo()[0])
        gpu = ctx.heff_apply(dev(L), dev(W), dev(W), dev(R), dev(psi))
        ref = oracle_mod.heff(L.numpy(), W.numpy(), W.numpy(), R.numpy(), psi.numpy())
        assert rel_frob(host(gpu), ref) <= 1e-12, (cl, clo, cr, cro)


def test_heff_heisenberg_singlet_on_gpu(ctx):
    W, lb, rb = synth.heisenberg_mpo()
    L = dev(synth.boundary_env(5, lb))
    R = dev(synth.boundary_env(5, rb))
    Wd = dev(W)
    cols = []
    for k in range(4):
        e = torch.zeros(4, dtype=torch.complex128)
        e[k] = 1
        cols.append(host(ctx.heff_apply(L, Wd, Wd, R, dev(e.reshape(1, 2, 2, 1)))).reshape(-1))
    H = np.stack(cols, axis=1)
    ev = np.sort(np.linalg.eigvalsh(H))
    assert np.max(np.abs(ev - np.array([-0.75, 0.25, 0.25, 0.25]))) < 1e-14


def test_heff_cfg2_sampled_rows(ctx, oracle_mod):
    """Config 2 at full size (chi=1024, d=2, D=5, c128), in the launch
    configuration bench.py times: sampled output rows vs the oracle, plus
    bitwise repeatability and bitwise equality of a sharded run."""
    cfg = synth.HEFF_CONFIGS["cfg2_heisenberg_chi1024"]
    inp = synth.heff_inputs(cfg["chi"], cfg["d"], cfg["D"], cfg["dtype"], cfg["seed"], cfg["model"])
    d_in = {k: dev(v) for k, v in inp.items()}
    out = ctx.heff_apply(d_in["L"], d_in["W1"], d_in["W2"], d_in["R"], d_in["psi"])
    out2 = ctx.heff_apply(d_in["L"], d_in["W1"], d_in["W2"], d_in["R"], d_in["psi"])
    assert torch.equal(out, out2)
    n = _heff_np(inp)
    rows = [0, 1, 127, 128, 255, 256, 511, 512, 767, 768, 1023, 333, 901]
    ref = oracle_mod.heff_rows(n["L"], n["W1"], n["W2"], n["R"], n["psi"], rows)
    assert rel_frob(host(out)[rows], ref) <= 1e-12
    # shard on b (P=4): rank 2's slab equals rows [512, 768) bitwise
    Ls = d_in["L"][:, :, 512:768].contiguous()
    part = ctx.heff_apply(Ls, d_in["W1"], d_in["W2"], d_in["R"], d_in["psi"])
    assert torch.equal(part, out[512:768])


def test_heff_freivalds_projection(ctx, oracle_mod):
    """Whole-output check: out . x (random x on the e leg) equals the chain with
    R.x contracted first (oracle, O(chi^2 D d^3))."""
    inp = synth.heff_inputs(256, 2, 5, "c128", 321, "heisenberg")
    out = ctx.heff_apply(*[dev(inp[k]) for k in ("L", "W1", "W2", "R", "psi")])
    x = synth.random_np((256,), "c128", 321, 99)
    n = _heff_np(inp)
    Rx = oracle_mod.contract(n["R"], "cxe", x, "e", "cx")
    T1 = oracle_mod.contract(n["L"], "awb", n["psi"], "astc", "wbstc")
    T2 = oracle_mod.contract(T1, "wbstc", n["W1"], "wvsp", "btcvp")
    T3 = oracle_mod.contract(T2, "btcvp", n["W2"], "vxtq", "bpqcx")
    ref = oracle_mod.contract(T3, "bpqcx", Rx, "cx", "bpq")
    got = oracle_mod.contract(host(out), "bpqe", x, "e", "bpq")
    assert rel_frob(got, ref) <= 1e-12


# ---------------------------------------------------------------------------
# TEBD (8(a8))
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("chi", [1, 33, 130])
@pytest.mark.parametrize("layout", ["natural", "physical_first"])
def test_tebd_theta(ctx, oracle_mod, chi, layout):
    pf = layout == "physical_first"
    inp = synth.tebd_inputs(chi, 2, "r64", 400 + chi, 0.01, physical_first=pf)
    la, lb, lt = ("sab", "tbc", "paqc") if pf else ("asb", "btc", "apqc")
    th = ctx.tebd_theta(dev(inp["A"]), la, dev(inp["B"]), lb, dev(inp["U"]), "pqst", lt)
    ref = oracle_mod.tebd_theta(inp["A"].numpy(), inp["B"].numpy(), inp["U"].numpy(), la=la, lb=lb, lu="pqst", lt=lt)
    assert rel_frob(host(th), ref) <= 1e-12


@pytest.mark.parametrize("chi", [1, 33, 130, 1030])
@pytest.mark.parametrize("layout", ["natural", "physical_first"])
def test_tebd_theta_complex_real_time(ctx, ozctx, oracle_mod, chi, layout):
    """complex128 theta with the real-time gate expm(-i tau h) (Application
    A's real-time evolution; K = C): A.B on
    the complex GEMM path (DMMA 3M; and Ozaki at chi = 1030, 4.4e9 MACs) and
    the gate as the skinny pass, both layouts, vs the oracle <= 1e-12."""
    pf = layout == "physical_first"
    inp = synth.tebd_inputs(chi, 2, "c128", 420 + chi, 0.05, physical_first=pf)
    la, lb, lt = ("sab", "tbc", "paqc") if pf else ("asb", "btc", "apqc")
    assert inp["U"].dtype == torch.complex128
    A = inp["A"].numpy()
    rows = list(range(chi)) if chi < 1024 else [0, 1, chi // 2, chi - 1]     # a-leg rows the oracle forms
    As = A[:, rows] if pf else A[rows]
    ref = oracle_mod.tebd_theta(np.ascontiguousarray(As), inp["B"].numpy(), inp["U"].numpy(), la=la, lb=lb,
                                lu="pqst", lt=lt)
    for c in ((ctx, ozctx) if chi >= 1024 else (ctx,)):
        th = host(c.tebd_theta(dev(inp["A"]), la, dev(inp["B"]), lb, dev(inp["U"]), "pqst", lt))
        got = th[:, rows] if pf else th[rows]          # theta[p,a,q,c] / theta[a,p,q,c]
        assert rel_frob(got, ref) <= 1e-12


def test_tebd_identity_gate_equals_AB_bitwise(ctx):
    inp = synth.tebd_inputs(64, 2, "r64", 410, 0.0)
    A, B = dev(inp["A"]), dev(inp["B"])
    th = ctx.tebd_theta(A, "asb", B, "btc", dev(inp["U"]), "pqst", "apqc")
    ab = ctx.contract(A, "asb", B, "btc", "astc")
    assert torch.equal(th, ab)


def test_tebd_cfg3_sampled(ctx, oracle_mod):
    cfg = synth.TEBD_CONFIG
    inp = synth.tebd_inputs(cfg["chi"], cfg["d"], cfg["dtype"], cfg["seed"], cfg["tau"])
    th = host(ctx.tebd_theta(dev(inp["A"]), "asb", dev(inp["B"]), "btc", dev(inp["U"]), "pqst", "apqc"))
    A = inp["A"].numpy()
    for a0 in (0, 1, 1023, 2047):
        ref = oracle_mod.tebd_theta(A[a0:a0 + 1], inp["B"].numpy(), inp["U"].numpy())
        assert rel_frob(th[a0:a0 + 1], ref) <= 1e-12


# ---------------------------------------------------------------------------
# MPS norm / overlap (8(a9)) and MPS-MPO application (8(a10))
# ---------------------------------------------------------------------------

def _gpu_overlap(ctx, bra, ket):
    E = torch.ones(1, 1, dtype=torch.float64, device="cuda")
    for Ab, Ak in zip(bra, ket):
        X = ctx.contract(E, "xz", dev(Ab), "xsy", "zsy")
        E = ctx.contract(X, "zsy", dev(Ak), "zsw", "yw")
    return E


def test_mps_norm_cfg1(ctx, oracle_mod):
    psi = synth.mps_sites(synth.MPS_BONDS_CFG1, 2, 1)
    phi = synth.mps_sites(synth.MPS_BONDS_CFG1, 2, 2)
    assert rel_frob(host(_gpu_overlap(ctx, psi, psi)), oracle_mod.mps_norm2(psi)) <= 1e-12
    assert rel_frob(host(_gpu_overlap(ctx, phi, psi)), oracle_mod.mps_overlap(phi, psi)) <= 1e-12
    prod = synth.product_state_sites(10)
    assert host(_gpu_overlap(ctx, prod, prod))[0, 0] == 1.0


def test_graph_capture_cfg1_chain(oracle_mod):
    """Config 1's 20-contract transfer chain recorded into a CUDA graph
    (tci_graph_begin / end) and replayed: bitwise equal to the eager chain,
    the oracle's norm within 1e-12, the graph's kernel count charged per
    replay, and an illegal call inside a capture (a host read) reported as an
    error without leaving the context capturing."""
    s = torch.cuda.Stream()
    c = tci.Context(0, s)
    try:
        psi = [dev(a) for a in synth.mps_sites(synth.MPS_BONDS_CFG1, 2, 1)]
        E0 = torch.ones(1, 1, dtype=torch.float64, device="cuda")
        bufs = {}

        def chain():
            E = E0
            for i, A in enumerate(psi):
                X = c.contract(E, "xz", A, "xsy", "zsy", out=bufs.get(("X", i)))
                bufs[("X", i)] = X
                E = c.contract(X, "zsy", A, "zsw", "yw", out=bufs.get(("E", i)))
                bufs[("E", i)] = E
            return E
        eager = chain().clone()            # allocates the outputs, sizes the workspace
        torch.cuda.synchronize()
        out = bufs[("E", len(psi) - 1)]
        out.zero_()
        torch.cuda.synchronize()
        n0 = c.launch_count()
        g, _ = c.capture(chain)
        assert c.launch_count() == n0 and out.abs().max().item() == 0.0     # recorded, not run
        for _ in range(3):
            c.replay(g)
        c.synchronize()
        assert torch.equal(out, eager)
        dn = c.launch_count() - n0
        assert dn >= 3 * 20 and dn % 3 == 0
        ref = oracle_mod.mps_norm2(synth.mps_sites(synth.MPS_BONDS_CFG1, 2, 1))
        assert rel_frob(host(out), ref) <= 1e-12
        tci.tci_graph_destroy(g)
        # a synchronizing call inside a capture fails, and the capture is over afterwards
        with pytest.raises(tci.TciError):
            c.capture(lambda: c.ozaki_guard_stats())
        assert torch.equal(chain(), eager)
    finally:
        c.close()


def test_mps_overlap_single_kernel(ctx, oracle_mod):
    """tci_mps_overlap: the whole transfer chain in one kernel (config 1)."""
    psi = synth.mps_sites(synth.MPS_BONDS_CFG1, 2, 1)
    phi = synth.mps_sites(synth.MPS_BONDS_CFG1, 2, 2)
    n2 = ctx.mps_overlap([dev(a) for a in psi], [dev(a) for a in psi])
    assert rel_frob(host(n2), oracle_mod.mps_norm2(psi)) <= 1e-12
    ov = ctx.mps_overlap([dev(a) for a in phi], [dev(a) for a in psi])
    assert rel_frob(host(ov), oracle_mod.mps_overlap(phi, psi)) <= 1e-12
    prod = [dev(a) for a in synth.product_state_sites(10)]
    assert host(ctx.mps_overlap(prod, prod))[0, 0] == 1.0
    # complex, open right boundary (out is [4, 3]), d = 3
    bonds_b, bonds_k = [1, 3, 7, 4], [1, 2, 5, 3]
    bra = [synth.random_np((bonds_b[i], 3, bonds_b[i + 1]), "c128", 440, 100 + i) for i in range(3)]
    ket = [synth.random_np((bonds_k[i], 3, bonds_k[i + 1]), "c128", 441, 100 + i) for i in range(3)]
    got = ctx.mps_overlap([dev(a) for a in bra], [dev(a) for a in ket])
    assert tuple(got.shape) == (4, 3)
    assert rel_frob(host(got), oracle_mod.mps_overlap(bra, ket)) <= 1e-12
    with pytest.raises(tci.TciError) as e:
        ctx.mps_overlap([dev(a) for a in psi[:3]], [dev(a) for a in phi[:2]] + [dev(psi[2])],
                        out=torch.empty(3, 3, dtype=torch.float64, device="cuda"))
    assert e.value.code == 1


@pytest.mark.parametrize("dt", ["c128", "r64"])
def test_skinny_pass_shapes(ctx, oracle_mod, dt):
    """The skinny pass over a unit-stride batch leg (the MPO-pass shape; complex
    K, N <= 32 runs on the DMMA kernel, 3M, in 4-k x 8-n fragments): every
    fragment boundary of K and N, a batch leg ragged against the 64-value tile,
    through contract's skinny route."""
    for K in (1, 3, 4, 5, 8, 13, 20, 32):
        for N in (1, 2, 7, 8, 9, 20, 24, 32):
            X = synth.random_tensor((3, K, 200), dt, 440 + K, 1)
            W = synth.random_tensor((K, N), dt, 440 + N, 2)
            got = ctx.contract(dev(X), "akc", dev(W), "kn", "anc")
            ref = oracle_mod.contract(X.numpy(), "akc", W.numpy(), "kn", "anc")
            assert rel_frob(host(got), ref) <= 1e-12, (K, N)
            got2 = ctx.contract(dev(X), "akc", dev(W), "kn", "anc")
            assert torch.equal(got, got2)                       # deterministic


def test_skinny_pass_real_weights(ctx, oracle_mod):
    """Complex data with a real-valued W (the model MPOs) takes the two-DMMA
    branch of the tensor-core pass; one nonzero imaginary entry switches it
    back to 3M. Both vs the oracle."""
    X = synth.random_tensor((3, 20, 200), "c128", 450, 1)
    W = synth.random_tensor((20, 20), "c128", 450, 2)
    Wr = torch.complex(W.real, torch.zeros_like(W.real))
    for w in (Wr, Wr.clone()):
        got = ctx.contract(dev(X), "akc", dev(w), "kn", "anc")
        ref = oracle_mod.contract(X.numpy(), "akc", w.numpy(), "kn", "anc")
        assert rel_frob(host(got), ref) <= 1e-12
        Wr[7, 3] = complex(Wr[7, 3].real.item(), 1e-3)   # second pass: one imaginary entry


def test_mps_mpo_apply(ctx, oracle_mod):
    A = synth.random_tensor((40, 2, 33), "c128", 420, 1)
    I = torch.eye(2, dtype=torch.complex128).reshape(1, 1, 2, 2)
    B = ctx.contract(dev(A), "asb", dev(I), "wvst", "awtbv")
    assert torch.equal(B.cpu().reshape(40, 2, 33), A)
    W = synth.random_tensor((5, 5, 2, 2), "c128", 420, 2)
    B = ctx.contract(dev(A), "asb", dev(W), "wvst", "awtbv")
    ref = oracle_mod.mps_mpo_apply(A.numpy(), W.numpy())
    assert rel_frob(host(B).reshape(ref.shape), ref) <= 1e-12


@pytest.mark.parametrize("dt", ["c128", "r64"])
@pytest.mark.parametrize("a,d,b,D", [(40, 2, 301, 5), (7, 3, 1000, 4), (3, 4, 64, 8), (5, 2, 129, 2)])
def test_mps_mpo_apply_expansion_layout(ctx, oracle_mod, dt, a, d, b, D):
    """8(a10) at b-extents that take the skinny expansion kernel (few k, the
    output's trailing v-run right after b): ragged b tiles (128 per tile),
    K = d = 2..4, runs of D = 2..8; identity MPO bitwise, random MPO vs the
    oracle."""
    A = synth.random_tensor((a, d, b), dt, 421, 1)
    I = torch.eye(d, dtype=A.dtype).reshape(1, 1, d, d)
    B = ctx.contract(dev(A), "asb", dev(I), "wvst", "awtbv")
    assert torch.equal(B.cpu().reshape(a, d, b), A)
    W = synth.random_tensor((D, D, d, d), dt, 421, 2)
    B = ctx.contract(dev(A), "asb", dev(W), "wvst", "awtbv")
    ref = oracle_mod.mps_mpo_apply(A.numpy(), W.numpy())
    assert rel_frob(host(B).reshape(ref.shape), ref) <= 1e-12


def test_mps_mpo_apply_full_size_sampled(ctx, oracle_mod):
    """The bench_extra 8(a10) workload (chi = 4096, d = 2, D = 5, c128: 13.4 GB
    out) in the launch configuration it is timed in; oracle on sampled rows a
    (first, last, ragged middle)."""
    chi, d, D = 4096, 2, 5
    A = synth.random_tensor((chi, d, chi), "c128", 31, 1, device="cuda")
    Wh, _, _ = synth.heisenberg_mpo(1.0)
    W = torch.from_numpy(np.asarray(Wh)).to(torch.complex128)
    B = ctx.contract(A, "asb", dev(W), "wvst", "awtbv")
    rows = [0, 1, 2047, 4095]
    got = B[rows].cpu().numpy()
    ref = oracle_mod.mps_mpo_apply(A[rows].cpu().numpy(), W.numpy())
    assert rel_frob(got.reshape(ref.shape), ref) <= 1e-12
    del A, B
    torch.cuda.empty_cache()


# ---------------------------------------------------------------------------
# multi-GPU plumbing (8(e)) on one GPU: NCCL communicator of one rank
# ---------------------------------------------------------------------------

def test_nccl_allgather_single_rank(ctx):
    uid = tci.tci_comm_unique_id()
    assert len(uid) == 128
    c = tci.Context(0)
    c.comm_init(uid, 1, 0)
    x = dev(synth.random_tensor((64, 2, 2, 96), "c128", 430, 1))
    full = torch.empty_like(x)
    c.allgather(x, full)
    torch.cuda.synchronize()
    assert torch.equal(full, x)
    with pytest.raises(tci.TciError) as e:
        c.allgather(x, torch.empty(2 * x.numel(), dtype=x.dtype, device="cuda"))
    assert e.value.code == 1
    c.close()
    with pytest.raises(tci.TciError) as e:
        ctx.allgather(x, full)          # no communicator on this context
    assert e.value.code == 11


def test_sharded_heff_single_rank_path(ctx):
    """bench.py's ShardedHeff on one rank (world 1): identical to a direct apply."""
    from paper_2512_23917_b200.sharding import ShardedHeff, slice_environment
    inp = synth.heff_inputs(64, 2, 5, "c128", 431, "heisenberg", device="cuda")
    sh = ShardedHeff(ctx, slice_environment(inp["L"], 1, 0), inp["W1"], inp["W2"], inp["R"], 1, 0)
    out = sh.apply(inp["psi"])
    ref = ctx.heff_apply(inp["L"], inp["W1"], inp["W2"], inp["R"], inp["psi"])
    assert torch.equal(out, ref)


# ---------------------------------------------------------------------------
# vector functions and the Lanczos driver (8(f1))
# ---------------------------------------------------------------------------

def test_vector_functions(ctx, oracle_mod):
    for dt in ("r64", "c128"):
        xs = [synth.random_tensor((33, 2, 2, 47), dt, 450 + i, 1) for i in range(11)]
        dx = [dev(x) for x in xs]
        n1 = ctx.norm(dx[0])
        assert abs(n1 - oracle_mod.norm(xs[0].numpy())) <= 1e-14 * n1
        assert ctx.norm(dx[0]) == n1                        # deterministic reduction: bitwise
        ip = ctx.inner(dx[1], dx[2])
        ref = oracle_mod.inner(xs[1].numpy(), xs[2].numpy())
        assert abs(ip - ref) <= 1e-13 * oracle_mod.norm(xs[1].numpy()) * oracle_mod.norm(xs[2].numpy())
        coefs = [(0.5 - 0.1 * i) + (0.3j * i if dt == "c128" else 0) for i in range(11)]   # 11 > 8: chunked
        lc = ctx.linear_combine(dx, coefs)
        assert rel_frob(host(lc), oracle_mod.linear_combine([x.numpy() for x in xs], coefs)) <= 1e-14
        sc = ctx.scale(dx[3], -2.0)
        assert torch.equal(sc.cpu(), -2.0 * xs[3])
        ctx.linear_combine([dx[4], dx[5]], None, out=dx[4])   # aliasing out == input, default coefs
        assert torch.equal(dx[4].cpu(), xs[4] + xs[5])
    e = dev(torch.eye(3, dtype=torch.float64))
    assert ctx.norm(e) == float(np.sqrt(3.0))


def _env_left(L, A, W):
    # L'[a',w',b'] = sum L[a,w,b] A[a,s,a'] W[w,w',s,t] conj(A[b,t,b'])
    return np.einsum("awb,asx,wvst,bty->xvy", L, A, W, np.conj(A), optimize=True)


def _env_right(R, B, W):
    # R[c,x,e] = sum B[c,s,c'] W[x,x',s,t] conj(B[e,t,e']) R'[c',x',e']
    return np.einsum("csd,xzst,ety,dzy->cxe", B, W, np.conj(B), R, optimize=True)


def _heisenberg_envs(chi_sites, seed):
    W, lb, rb = synth.heisenberg_mpo()
    L = synth.boundary_env(5, lb)
    bonds = [1] + chi_sites
    for i in range(len(chi_sites)):
        A = synth.random_np((bonds[i], 2, bonds[i + 1]), "c128", seed, 200 + i)
        L = _env_left(L, A, W)
    R = synth.boundary_env(5, rb)
    for i in range(len(chi_sites)):
        B = synth.random_np((bonds[i + 1], 2, bonds[i]), "c128", seed, 300 + i)
        R = _env_right(R, B, W)
    return L, W, R


@pytest.mark.parametrize("chi_sites", [[2, 4], [2, 4, 8, 16]])
def test_lanczos_vs_dense_eigvalsh(ctx, oracle_mod, chi_sites):
    L, W, R = _heisenberg_envs(chi_sites, 460 + len(chi_sites))
    chi = chi_sites[-1]
    H = oracle_mod.heff_dense(L, W, W, R, (chi, 2, 2, chi))
    assert np.max(np.abs(H - H.conj().T)) < 1e-12 * np.max(np.abs(H))       # Hermitian by construction
    e_ref = np.linalg.eigvalsh((H + H.conj().T) / 2)[0]
    psi = dev(synth.random_tensor((chi, 2, 2, chi), "c128", 470, 2))
    e, it = ctx.heff_lanczos(dev(L), dev(W), dev(W), dev(R), psi, max_iter=min(200, H.shape[0]), tol=1e-14)
    assert abs(e - e_ref) <= 1e-9 * max(1.0, abs(e_ref)), (e, e_ref, it)
    # returned Ritz vector: normalised and an eigenvector (residual small)
    assert abs(ctx.norm(psi) - 1.0) < 1e-12
    hv = host(ctx.heff_apply(dev(L), dev(W), dev(W), dev(R), psi)).reshape(-1)
    v = host(psi).reshape(-1)
    assert np.linalg.norm(hv - e * v) <= 1e-6 * max(1.0, abs(e))


def test_lanczos_closed_forms(ctx):
    g = __import__("conftest").golden("closed_forms.json")
    W, lb, rb = synth.heisenberg_mpo()
    L, R = dev(synth.boundary_env(5, lb)), dev(synth.boundary_env(5, rb))
    psi = dev(synth.random_tensor((1, 2, 2, 1), "c128", 480, 2))
    e, _ = ctx.heff_lanczos(L, dev(W), dev(W), R, psi, max_iter=10, tol=1e-15)
    assert abs(e - g["heisenberg_two_site"]["eigenvalues"][0]) < 1e-13
    # Hubbard: start in the N = 2 sector (H conserves N) -> closed-form E0
    h = g["hubbard_two_site_N2"]
    W, lb, rb = synth.hubbard_mpo(h["t"], h["U"])
    L, R = dev(synth.boundary_env(6, lb)), dev(synth.boundary_env(6, rb))
    nloc = np.array([0, 1, 1, 2])
    start = synth.random_np((1, 4, 4, 1), "c128", 481, 2)
    start[0][(nloc[:, None] + nloc[None, :]) != 2] = 0
    psi = dev(start)
    e, _ = ctx.heff_lanczos(L, dev(W), dev(W), R, psi, max_iter=16, tol=1e-15)
    assert abs(e - h["E0"]) < 1e-12


# ---------------------------------------------------------------------------
# Ozaki-II INT8 tcgen05 complex GEMM (8(f4))
# ---------------------------------------------------------------------------

@pytest.fixture()
def ozctx():
    c = tci.Context(0)
    c.set_gemm_algorithm(tci.TCI_GEMM_OZAKI_INT8)
    yield c
    c.close()


@pytest.mark.parametrize("layout", ["mk", "km"])
def test_ozaki_contract_vs_dmma_and_oracle(ctx, ozctx, oracle_mod, layout):
    """M = N = 1024, K = 4096 (4.3e9 MACs: takes the Ozaki path) with rows
    scaled by random powers of two (dynamic range between rows) and one zero row."""
    A = synth.random_tensor((1024, 4096), "c128", 490, 1)
    rng = np.random.default_rng(5)
    A = A * torch.from_numpy(2.0 ** rng.integers(-30, 30, size=(1024, 1))).to(torch.complex128)
    A[17] = 0
    B = synth.random_tensor((4096, 1024), "c128", 490, 2)
    At = A if layout == "mk" else A.T.contiguous()
    c_oz = ozctx.contract(dev(At), layout, dev(B), "kn", "mn")
    c_dm = ctx.contract(dev(At), layout, dev(B), "kn", "mn")
    assert torch.count_nonzero(c_oz[17]).item() == 0
    # per-row relative errors (rows differ in scale by up to 2^60)
    d = (c_oz - c_dm).abs().pow(2).sum(1).sqrt() / c_dm.abs().pow(2).sum(1).sqrt().clamp_min(1e-300)
    d[17] = 0
    assert d.max().item() <= 1e-12
    rows = [0, 1, 511, 1023]
    ref = oracle_mod.contract(A.numpy()[rows], "mk", B.numpy(), "kn", "mn")
    got = host(c_oz)[rows]
    for i in range(len(rows)):
        assert rel_frob(got[i], ref[i]) <= 1e-12
    c2 = ozctx.contract(dev(At), layout, dev(B), "kn", "mn")
    assert torch.equal(c_oz, c2)                         # deterministic


@pytest.mark.parametrize("dt,tol", [("c128", 1e-12), ("c64", 1e-5)])
@pytest.mark.parametrize("mnk", [(1029, 1040, 4100), (300, 1552, 9000)])
def test_ozaki_tensor_core_crt_ragged(ozctx, oracle_mod, dt, tol, mnk):
    """The tensor-core CRT (crt_mma.cu) at ragged extents: N = 1040 / 1552 leave
    a partial 512-column tile and a partial 128-output MMA; M = 1029 / 300
    leave ragged rows; zero rows and columns give exact zeros; complex64 runs
    the 9-10-moduli digit epilogue (float2 stores). Oracle on sampled rows,
    every column; deterministic."""
    M, N, K = mnk
    A = synth.random_tensor((M, K), dt, 491, 1)
    B = synth.random_tensor((K, N), dt, 491, 2)
    A[5] = 0
    B[:, N - 3] = 0
    c1 = ozctx.contract(dev(A), "mk", dev(B), "kn", "mn")
    st = ozctx.ozaki_guard_stats()
    assert st["gemms"] >= 1 and st["fallbacks"] == 0, st
    assert torch.count_nonzero(c1[5]).item() == 0 and torch.count_nonzero(c1[:, N - 3]).item() == 0
    rows = [0, 1, M // 2, M - 2, M - 1]
    ref = oracle_mod.contract(A.numpy()[rows].astype(np.complex128), "mk", B.numpy().astype(np.complex128), "kn",
                              "mn")
    got = host(c1)[rows].astype(np.complex128)
    assert rel_frob(got, ref) <= tol
    assert torch.equal(c1, ozctx.contract(dev(A), "mk", dev(B), "kn", "mn"))


@pytest.mark.parametrize("variant", [tci.TCI_OZAKI_CPLX_GAUSS, tci.TCI_OZAKI_CPLX_3M])
@pytest.mark.parametrize("mnk", [(320, 320, 40960), (256, 256, 131072)])
def test_ozaki_large_k_moduli_counts(ozctx, oracle_mod, mnk, variant):
    """Long K needs the largest moduli sets: 3M takes 15 moduli (M > 2^117,
    four 37-bit CRT weight chunks, R27); the Gaussian set 15 at K = 40960 and
    16 at K = 131072 (three 40-bit chunks, R33). Both within 1e-12 of the
    oracle."""
    M, N, K = mnk
    st, nmod, t, _, _, ppm = tci.tci_ozaki_params_complex(K, variant)
    if variant == tci.TCI_OZAKI_CPLX_3M:
        assert st == 0 and nmod == 15 and t >= 46 and ppm == 3
    else:
        assert st == 0 and nmod == (15 if K < 69000 else 16) and t >= 46 and ppm == 2
    A = synth.random_tensor((M, K), "c128", 493, 1)
    B = synth.random_tensor((K, N), "c128", 493, 2)
    ozctx.set_ozaki_complex(variant)
    try:
        c = host(ozctx.contract(dev(A), "mk", dev(B), "kn", "mn"))
    finally:
        ozctx.set_ozaki_complex(tci.TCI_OZAKI_CPLX_GAUSS)
    rows = [0, 1, M // 2, M - 1]
    ref = oracle_mod.contract(A.numpy()[rows], "mk", B.numpy(), "kn", "mn")
    assert rel_frob(c[rows], ref) <= 1e-12
    assert ozctx.launch_count() > 0


@pytest.mark.parametrize("la", ["mk", "km"])
def test_ozaki_gaussian_vs_3m_vs_oracle(ozctx, oracle_mod, la):
    """The two complex variants on the same product (M = 1300, N = 1100,
    K = 4100: ragged against every tile; both residue kernels): each within
    1e-12 of the oracle on sampled rows, and of each other everywhere; the
    Gaussian variant ran 2 INT8 planes per modulus (its INT8 op count is
    2/3 x 15/14 of the 3M one's)."""
    M, N, K = 1300, 1100, 4100
    A = synth.random_tensor((M, K), "c128", 497, 1)
    B = synth.random_tensor((K, N), "c128", 497, 2)
    At = A if la == "mk" else A.T.contiguous()
    outs, ops = {}, {}
    for v in (tci.TCI_OZAKI_CPLX_GAUSS, tci.TCI_OZAKI_CPLX_3M):
        ozctx.set_ozaki_complex(v)
        tci.tci_profile_enable(ozctx.handle, True)
        outs[v] = ozctx.contract(dev(At), la, dev(B), "kn", "mn")
        ops[v] = tci.tci_profile_query(ozctx.handle, tci.PROF_I8)["flops"]
        tci.tci_profile_enable(ozctx.handle, False)
    ozctx.set_ozaki_complex(tci.TCI_OZAKI_CPLX_GAUSS)
    _, ng, _, _, _, _ = tci.tci_ozaki_params_complex(K, tci.TCI_OZAKI_CPLX_GAUSS)
    _, n3, _, _, _, _ = tci.tci_ozaki_params_complex(K, tci.TCI_OZAKI_CPLX_3M)
    assert abs(ops[0] / ops[1] - (2 * ng) / (3 * n3)) < 1e-9
    g, m3 = outs[tci.TCI_OZAKI_CPLX_GAUSS], outs[tci.TCI_OZAKI_CPLX_3M]
    assert ((g - m3).abs().pow(2).sum().sqrt() / m3.abs().pow(2).sum().sqrt()).item() <= 1e-12
    rows = [0, 1, 647, M - 1]
    ref = oracle_mod.contract(A.numpy()[rows], "mk", B.numpy(), "kn", "mn")
    for o in (g, m3):
        assert rel_frob(host(o)[rows], ref) <= 1e-12


def test_ozaki_heff_cfg2(ozctx, oracle_mod):
    cfg = synth.HEFF_CONFIGS["cfg2_heisenberg_chi1024"]
    inp = synth.heff_inputs(cfg["chi"], cfg["d"], cfg["D"], cfg["dtype"], cfg["seed"], cfg["model"])
    d_in = {k: dev(v) for k, v in inp.items()}
    out = ozctx.heff_apply(d_in["L"], d_in["W1"], d_in["W2"], d_in["R"], d_in["psi"])
    n = {k: v.numpy() for k, v in inp.items()}
    rows = [0, 1, 255, 256, 511, 512, 1023]
    ref = oracle_mod.heff_rows(n["L"], n["W1"], n["W2"], n["R"], n["psi"], rows)
    assert rel_frob(host(out)[rows], ref) <= 1e-12
    part = ozctx.heff_apply(d_in["L"][:, :, 256:512].contiguous(), d_in["W1"], d_in["W2"], d_in["R"], d_in["psi"])
    assert torch.equal(part, out[256:512])                # shard-invariant, bitwise


def test_ozaki_lanczos(ozctx):
    W, lb, rb = synth.heisenberg_mpo()
    L, R = dev(synth.boundary_env(5, lb)), dev(synth.boundary_env(5, rb))
    psi = dev(synth.random_tensor((1, 2, 2, 1), "c128", 480, 2))
    e, _ = ozctx.heff_lanczos(L, dev(W), dev(W), R, psi, max_iter=10, tol=1e-15)
    assert abs(e + 0.75) < 1e-13


# ---------------------------------------------------------------------------
# cplx_conj and environment updates (8(f3), R28)
# ---------------------------------------------------------------------------

def test_cplx_conj(ctx, oracle_mod):
    x = synth.random_tensor((37, 5, 129), "c128", 600, 1)
    y = ctx.cplx_conj(dev(x))
    assert np.array_equal(host(y), oracle_mod.cplx_conj(x.numpy()))     # bitwise
    d = dev(x)
    ctx.cplx_conj(d, out=d)                                               # in place (overload (1))
    assert np.array_equal(host(d), oracle_mod.cplx_conj(x.numpy()))
    r = synth.random_tensor((33, 7), "r64", 601, 1)
    rc = ctx.cplx_conj(dev(r))                                            # real: deep copy
    assert np.array_equal(host(rc), r.numpy())
    buf = dev(synth.random_tensor((65,), "c128", 602, 1))
    with pytest.raises(tci.TciError) as e:                                # partial overlap
        ctx.cplx_conj(buf[:-1], out=buf[1:])
    assert e.value.code == 8
    with pytest.raises(tci.TciError) as e:
        ctx.cplx_conj(dev(x), out=torch.empty((37, 5, 128), dtype=torch.complex128, device="cuda"))
    assert e.value.code == 1


def _env_inputs(side, dt, chi_k, chi_b, chi_ko, chi_bo, D, Dv, d, seed, same_bra=False):
    E = synth.random_tensor((chi_k, D, chi_b), dt, seed, 1)
    if side == 0:
        ket = synth.random_tensor((chi_k, d, chi_ko), dt, seed, 2)
        W = synth.random_tensor((D, Dv, d, d), dt, seed, 3)
        bra = ket if same_bra else synth.random_tensor((chi_b, d, chi_bo), dt, seed, 4)
    else:
        ket = synth.random_tensor((chi_ko, d, chi_k), dt, seed, 2)
        W = synth.random_tensor((Dv, D, d, d), dt, seed, 3)
        bra = ket if same_bra else synth.random_tensor((chi_bo, d, chi_b), dt, seed, 4)
    return E, ket, W, bra


@pytest.mark.parametrize("side", [0, 1])
@pytest.mark.parametrize("dt", ["c128", "r64"])
@pytest.mark.parametrize("dims", [(37, 29, 41, 23, 5, 4, 2), (64, 64, 64, 64, 5, 5, 2), (1, 1, 9, 7, 1, 5, 3),
                                  (20, 33, 17, 70, 6, 6, 4)])
def test_env_update_vs_oracle(ctx, oracle_mod, side, dt, dims):
    chi_k, chi_b, chi_ko, chi_bo, D, Dv, d = dims
    E, ket, W, bra = _env_inputs(side, dt, chi_k, chi_b, chi_ko, chi_bo, D, Dv, d, 610)
    out = ctx.env_update(side, dev(E), dev(ket), dev(W), dev(bra))
    f = oracle_mod.env_left if side == 0 else oracle_mod.env_right
    ref = f(E.numpy(), ket.numpy(), W.numpy(), bra.numpy())
    assert out.shape == ref.shape
    assert rel_frob(host(out), ref) <= TOL[dt]
    again = ctx.env_update(side, dev(E), dev(ket), dev(W), dev(bra))
    assert torch.equal(out, again)                                        # deterministic


def test_env_update_errors(ctx):
    E, ket, W, bra = _env_inputs(0, "c128", 8, 8, 8, 8, 3, 3, 2, 611)
    with pytest.raises(tci.TciError) as e:
        ctx.env_update(0, dev(E), dev(ket), dev(W), dev(bra),
                       out=torch.empty((8, 3, 9), dtype=torch.complex128, device="cuda"))
    assert e.value.code == 1
    with pytest.raises(tci.TciError) as e:
        ctx.env_update(2, dev(E), dev(ket), dev(W), dev(bra),
                       out=torch.empty((8, 3, 8), dtype=torch.complex128, device="cuda"))
    assert e.value.code == 8


@pytest.mark.parametrize("side", [0, 1])
def test_env_heisenberg_expectation_closed_form(ctx, side):
    """<psi|H|psi> of a random product state through a chain of device
    environment updates equals the Bloch-vector closed form sum n_i.n_j / 4."""
    rng = np.random.default_rng(21)
    n = 12
    u = rng.standard_normal((n, 2)) + 1j * rng.standard_normal((n, 2))
    u /= np.linalg.norm(u, axis=1, keepdims=True)
    bloch = np.stack([2 * (np.conj(u[:, 0]) * u[:, 1]).real, 2 * (np.conj(u[:, 0]) * u[:, 1]).imag,
                      np.abs(u[:, 0]) ** 2 - np.abs(u[:, 1]) ** 2], axis=1)
    closed = float(np.sum(bloch[:-1] * bloch[1:]) / 4)
    W, lb, rb = synth.heisenberg_mpo()
    Wd = dev(W)
    sites = [dev(x.reshape(1, 2, 1).astype(np.complex128)) for x in u]
    if side == 0:
        E = dev(synth.boundary_env(5, lb))
        for A in sites:
            E = ctx.env_update(0, E, A, Wd)
        got = complex(host(E)[0, rb, 0])
    else:
        E = dev(synth.boundary_env(5, rb))
        for A in reversed(sites):
            E = ctx.env_update(1, E, A, Wd)
        got = complex(host(E)[0, lb, 0])
    assert abs(got - closed) <= 1e-14 and abs(got.imag) <= 1e-15


@pytest.mark.parametrize("dt", ["c128", "r64"])
@pytest.mark.parametrize("algo", ["dmma3m", "ozaki"])
@pytest.mark.parametrize("side", [0, 1])
def test_env_update_chi1024_sampled(oracle_mod, side, algo, dt):
    """cfg2 scale (chi = 1024, D = 5, d = 2; both GEMMs take the Ozaki path --
    complex or real -- when selected): sampled output rows vs the oracle."""
    c = tci.Context(0)
    if algo == "ozaki":
        c.set_gemm_algorithm(tci.TCI_GEMM_OZAKI_INT8)
    try:
        E, ket, W, bra = _env_inputs(side, dt, 1024, 1024, 1024, 1024, 5, 5, 2, 612, same_bra=True)
        out = c.env_update(side, dev(E), dev(ket), dev(W))
        rows = [0, 1, 511, 1023]
        ref = oracle_mod.env_rows(side, E.numpy(), ket.numpy(), W.numpy(), bra.numpy(), rows)
        assert rel_frob(host(out)[rows], ref) <= 1e-12
    finally:
        c.close()


@pytest.mark.parametrize("algo", ["dmma3m", "ozaki"])
def test_heff_apply_staged_bitwise(algo, oracle_mod):
    """tci_heff_apply_staged (host inputs, copies overlapped with compute,
    GEMM4 rows streamed back in chunks) equals tci_copy + tci_heff_apply +
    tci_copy bitwise, for the chunked DMMA path and the Ozaki path; sampled
    rows vs the oracle."""
    c = tci.Context(0)
    try:
        c.set_gemm_algorithm(tci.TCI_GEMM_OZAKI_INT8 if algo == "ozaki" else tci.TCI_GEMM_DMMA_3M)
        cfg = synth.HEFF_CONFIGS["cfg2_heisenberg_chi1024"]
        inp = synth.heff_inputs(cfg["chi"], cfg["d"], cfg["D"], cfg["dtype"], cfg["seed"], cfg["model"])
        keys = ("L", "W1", "W2", "R", "psi")
        d_in = {k: dev(inp[k]) for k in keys}
        ref_dev = c.heff_apply(*[d_in[k] for k in keys])
        hosts = [inp[k].contiguous().pin_memory() for k in keys]
        hout = torch.empty(ref_dev.shape, dtype=ref_dev.dtype).pin_memory()
        devs = [torch.empty_like(d_in[k]) for k in keys] + [torch.empty_like(ref_dev)]
        c.heff_apply_staged(hosts + [hout], devs)
        c.synchronize()
        assert torch.equal(hout, ref_dev.cpu())
        n = {k: v.numpy() for k, v in inp.items()}
        rows = [0, 511, 1023]
        ref = oracle_mod.heff_rows(n["L"], n["W1"], n["W2"], n["R"], n["psi"], rows)
        assert rel_frob(hout.numpy()[rows], ref) <= 1e-12
        # inputs staged only (host output NULL: bench.py's first streaming step)
        devs2 = [torch.empty_like(d_in[k]) for k in keys] + [torch.empty_like(ref_dev)]
        r2 = c.heff_apply_staged(hosts + [None], devs2)
        c.synchronize()
        assert r2 is devs2[5] and torch.equal(devs2[5], ref_dev)
        assert all(torch.equal(devs2[i], d_in[k]) for i, k in enumerate(keys))
    finally:
        c.close()


@pytest.mark.parametrize("name", ["target_heisenberg_chi4096", "cfg4_hubbard_chi4096"])
def test_heff_full_size_rows_and_freivalds(name, oracle_mod):
    """BASELINE configs at full size (the bench workload chi = 4096, d = 2,
    D = 5 and config 4: chi = 4096, d = 4, D = 6, c128) with the bench's
    default algorithm (Ozaki-II): two sampled output rows vs the oracle, and a
    whole-output Freivalds check: out . x for a random x on the e leg equals
    the chain applied with R.x (the oracle contracts psi with R.x first,
    O(chi^2 D d^4) instead of O(D d^2 chi^3)). Tolerance 1e-12 (north star)."""
    cfg = synth.HEFF_CONFIGS[name]
    chi, d, D = cfg["chi"], cfg["d"], cfg["D"]
    c = tci.Context(0)
    try:
        c.set_gemm_algorithm(tci.TCI_GEMM_OZAKI_INT8)
        dv = synth.heff_inputs(chi, d, D, "c128", cfg["seed"], cfg["model"], device="cuda")
        out = c.heff_apply(dv["L"], dv["W1"], dv["W2"], dv["R"], dv["psi"])
        xn = synth.random_tensor((chi,), "c128", cfg["seed"], 98).numpy()
        # the projection out . x is computed on the host (numpy matrix-vector
        # product of the copied-back output): the checker uses no product code
        ho = host(out)
        del out
        ox = (ho.reshape(-1, chi) @ xn).reshape(ho.shape[:3])
        rows = [1, chi - 2]
        got_rows = ho[rows].copy()
        del ho
        n = {k: v.cpu().numpy() for k, v in dv.items()}
        del dv
        torch.cuda.empty_cache()
        Rx = oracle_mod.contract(n["R"], "cxe", xn, "e", "cx").reshape(chi, D, 1)
        ref_ox = oracle_mod.heff_alt(n["L"], n["W1"], n["W2"], Rx, n["psi"])[..., 0]
        assert rel_frob(ox, ref_ox) <= 1e-12
        ref_rows = oracle_mod.heff_rows(n["L"], n["W1"], n["W2"], n["R"], n["psi"], rows)
        assert rel_frob(got_rows, ref_rows) <= 1e-12
    finally:
        c.close()


# ---------------------------------------------------------------------------
# float64 on the INT8 tensor cores (real Ozaki-II: one residue plane per modulus)
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("la,lb", [("mk", "kn"), ("km", "kn"), ("mk", "nk"), ("km", "nk")])
def test_ozaki_real_contract_vs_dmma_and_oracle(ctx, ozctx, oracle_mod, la, lb):
    """M = 1100, N = 1300, K = 3000 (4.3e9 MACs, ragged against every tile):
    all four operand layouts (K-contiguous and line-contiguous residue
    kernels), rows scaled by 2^(-30..30) and one zero row; per-row relative
    error vs the DMMA GEMM and oracle rows <= 1e-12; the INT8 GEMM ran."""
    M, N, K = 1100, 1300, 3000
    rng = np.random.default_rng(6)
    A = synth.random_tensor((M, K), "r64", 495, 1) * torch.from_numpy(2.0 ** rng.integers(-30, 30, size=(M, 1)))
    A[17] = 0
    B = synth.random_tensor((K, N), "r64", 495, 2)
    At = A if la == "mk" else A.T.contiguous()
    Bt = B if lb == "kn" else B.T.contiguous()
    tci.tci_profile_enable(ozctx.handle, True)
    c_oz = ozctx.contract(dev(At), la, dev(Bt), lb, "mn")
    i8 = tci.tci_profile_query(ozctx.handle, tci.PROF_I8)
    tci.tci_profile_enable(ozctx.handle, False)
    assert i8["launches"] >= 1, "float64 Ozaki path not taken"
    c_dm = ctx.contract(dev(At), la, dev(Bt), lb, "mn")
    assert torch.count_nonzero(c_oz[17]).item() == 0
    d = (c_oz - c_dm).pow(2).sum(1).sqrt() / c_dm.pow(2).sum(1).sqrt().clamp_min(1e-300)
    d[17] = 0
    assert d.max().item() <= 1e-12
    rows = [0, 1, 550, M - 1]
    ref = oracle_mod.contract(A.numpy()[rows], "mk", B.numpy(), "kn", "mn")
    got = host(c_oz)[rows]
    for i in range(len(rows)):
        assert rel_frob(got[i], ref[i]) <= 1e-12
    assert torch.equal(c_oz, ozctx.contract(dev(At), la, dev(Bt), lb, "mn"))     # deterministic


def test_ozaki_real_tebd_theta(ozctx, oracle_mod):
    """TEBD theta (chi = 1024, f64) with the Ozaki algorithm: A.B on the INT8
    tensor cores, the gate by the skinny pass; sampled rows vs the oracle."""
    c = synth.TEBD_CONFIG
    inp = synth.tebd_inputs(1024, c["d"], c["dtype"], c["seed"], c["tau"])
    th = ozctx.tebd_theta(dev(inp["A"]), "asb", dev(inp["B"]), "btc", dev(inp["U"]), "pqst", "apqc")
    a_rows = [0, 511, 1023]
    ref = oracle_mod.tebd_theta(inp["A"].numpy()[a_rows], inp["B"].numpy(), inp["U"].numpy())
    assert rel_frob(host(th)[a_rows], ref) <= 1e-12


def test_ozaki_real_tebd_theta_full_size(ozctx, oracle_mod):
    """Config 3 at full size (chi = 2048, f64) with the Ozaki algorithm: sampled
    rows of theta vs the oracle (<= 1e-12 relative per row)."""
    c = synth.TEBD_CONFIG
    inp = synth.tebd_inputs(c["chi"], c["d"], c["dtype"], c["seed"], c["tau"])
    th = host(ozctx.tebd_theta(dev(inp["A"]), "asb", dev(inp["B"]), "btc", dev(inp["U"]), "pqst", "apqc"))
    a_rows = [0, 1, 1023, 2047]
    ref = oracle_mod.tebd_theta(inp["A"].numpy()[a_rows], inp["B"].numpy(), inp["U"].numpy())
    for i, a in enumerate(a_rows):
        assert rel_frob(th[a], ref[i]) <= 1e-12


def test_ozaki_real_heff(ctx, ozctx, oracle_mod):
    """float64 H_eff.psi (chi = 1024, Heisenberg) with the Ozaki algorithm: both
    chain GEMMs on the real Ozaki-II path; vs the DMMA chain (<= 1e-12) and
    oracle rows; deterministic."""
    inp = synth.heff_inputs(1024, 2, 5, "r64", 97, "heisenberg")
    d = {k: dev(v) for k, v in inp.items()}
    tci.tci_profile_enable(ozctx.handle, True)
    got = ozctx.heff_apply(d["L"], d["W1"], d["W2"], d["R"], d["psi"])
    i8 = tci.tci_profile_query(ozctx.handle, tci.PROF_I8)
    tci.tci_profile_enable(ozctx.handle, False)
    assert i8["launches"] >= 2
    ref_dm = ctx.heff_apply(d["L"], d["W1"], d["W2"], d["R"], d["psi"])
    assert rel_frob(host(got), host(ref_dm)) <= 1e-12
    rows = [0, 511, 1023]
    n = {k: v.numpy() for k, v in inp.items()}
    want = oracle_mod.heff_rows(n["L"], n["W1"], n["W2"], n["R"], n["psi"], rows)
    assert rel_frob(host(got)[rows], want) <= 1e-12
    assert torch.equal(got, ozctx.heff_apply(d["L"], d["W1"], d["W2"], d["R"], d["psi"]))


# ---------------------------------------------------------------------------
# Config 5 at full size
# ---------------------------------------------------------------------------

def _sampled_check(A, la, B, lb, C, lc, sh, dims, oracle_mod, tol, rng, nsamp=64):
    """Sampled parity of C = contract(A, B) (host arrays): 64 coordinates of
    A's free legs x 64 of B's (4096 output elements, each set containing the
    first and last index of every free leg: the leg boundaries) recomputed by
    the oracle from the sliced operands; plus a host-side Freivalds check
    C . x = A . (B . x) for a random x over B's free legs."""
    fa = [l for l in la if l not in sh]
    fb = [l for l in lb if l not in sh]

    def coords(legs):
        n = nsamp
        cs = [{l: int(rng.integers(0, dims[l])) for l in legs} for _ in range(n)]
        cs[0] = {l: 0 for l in legs}
        cs[1] = {l: dims[l] - 1 for l in legs}
        for k, l in enumerate(legs):                       # each leg's boundaries alone
            if 2 + 2 * k + 1 < n:
                cs[2 + 2 * k][l] = 0
                cs[3 + 2 * k][l] = dims[l] - 1
        return cs
    ca, cb = coords(fa), coords(fb)
    # A sliced at the sampled free coordinates -> [64, S...] in sh order
    At = np.transpose(A, [la.index(l) for l in fa + list(sh)])
    Bt = np.transpose(B, [lb.index(l) for l in list(sh) + fb])
    Afree = At.reshape(int(np.prod([dims[l] for l in fa], dtype=np.int64)) if fa else 1, -1)
    Bfree = Bt.reshape(-1, int(np.prod([dims[l] for l in fb], dtype=np.int64)) if fb else 1)

    def flat(c, legs):
        i = 0
        for l in legs:
            i = i * dims[l] + c[l]
        return i
    ia = [flat(c, fa) for c in ca]
    ib = [flat(c, fb) for c in cb]
    ref = oracle_mod.contract(np.ascontiguousarray(Afree[ia]), "ms", np.ascontiguousarray(Bfree[:, ib]), "sn", "mn")
    Ct = np.transpose(C, [lc.index(l) for l in fa + fb]).reshape(Afree.shape[0], Bfree.shape[1])
    got = Ct[np.ix_(ia, ib)]
    assert rel_frob(got, ref) <= tol
    # Freivalds, projected on the host: (C x) vs A (B x); the oracle forms B x and A (B x)
    x = rng.uniform(-1, 1, Bfree.shape[1]).astype(C.dtype)
    Cx = Ct.astype(np.float64) @ x.astype(np.float64)      # float64 projection of the GPU result
    Bx = oracle_mod.contract(np.ascontiguousarray(Bfree), "sn", x, "n", "s")
    ABx = oracle_mod.contract(np.ascontiguousarray(Afree), "ms", Bx, "s", "m")
    assert rel_frob(Cx, ABx) <= tol


@pytest.mark.parametrize("dt", ["r64", "r32"])
def test_contract_sweep_cfg5_full_size(ctx, oracle_mod, dt):
    """Random rank 3..6 contractions with tensors up to 2^26 elements (>= 1e7
    for most instances) in the layout mix of config 5: full oracle comparison
    when |C| |S| <= 2e8 MACs, otherwise 4096 sampled output elements
    (including every leg boundary) + a host-side Freivalds projection.
    Tolerance: 1e-12 (f64), 1e-5 (f32) relative Frobenius."""
    rng = np.random.default_rng(55 if dt == "r64" else 56)
    tol = TOL[dt]
    big = 0
    for i in range(14):
        la, lb, lc, dims, sh = synth.sweep_instance(rng, max_elems=2 ** 26, rank_min=4 if i % 2 else 3)
        A = synth.random_tensor([dims[l] for l in la], dt, 7000 + i, 1)
        B = synth.random_tensor([dims[l] for l in lb], dt, 7000 + i, 2)
        C = host(ctx.contract(dev(A), la, dev(B), lb, lc))

        def size(ls):
            return int(np.prod([dims[l] for l in ls], dtype=np.int64))
        big += max(size(la), size(lb), size(lc)) >= 10 ** 7
        if size(lc) * size(sh) <= 2 * 10 ** 8:
            ref = oracle_mod.contract(A.numpy(), la, B.numpy(), lb, lc)
            assert rel_frob(C, ref) <= tol, (la, lb, lc, dims)
        else:
            _sampled_check(A.numpy(), la, B.numpy(), lb, C, lc, sh, dims, oracle_mod, tol, rng)
        del A, B, C
    assert big >= 5
