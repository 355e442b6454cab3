#!/usr/bin/env python
"""Secondary measurements for the BASELINE.json configs that are not the
bench.py headline: config 1 (MPS norm chain latency),
config 2 (chi=1024 H_eff), config 3 (TEBD theta, two layouts), config 4
(Hubbard chi=4096 d=4 D=6 H_eff), config 5 (general contraction sweep with a
per-instance roofline) and a permute-bandwidth sweep. Writes one JSON object.

    python tools/bench_extra.py [--only cfg1,cfg3,...] [--out gpurun_out/extra.json]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2512_23917_b200 as tci  # noqa: E402
import synth  # noqa: E402

FP64_PEAK = 37.06e12
FP32_PEAK = 148 * 128 * 2 * 1.965e9   # FFMA (SURVEY 8(d) roofline of fp32 sweep GEMMs); the INT8 path can exceed it
HBM = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] * 1e9 \
    if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6.65e12


def timed(fn, reps=5, warm=2):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(reps):
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / 1e3)
    return float(np.median(ts)), float(np.min(ts))


def cfg1(ctx):
    # (timing tool: no oracle here -- config 1's parity is in tests/, and the
    # CPU oracle is timed by bench.py only)
    psi = [torch.from_numpy(a).cuda() for a in synth.mps_sites(synth.MPS_BONDS_CFG1, 2, 1)]
    E0 = torch.ones(1, 1, dtype=torch.float64, device="cuda")
    outs = {}

    def chain():
        E = E0
        for A in psi:
            X = ctx.contract(E, "xz", A, "xsy", "zsy")
            E = ctx.contract(X, "zsy", A, "zsw", "yw")
        outs["E"] = E
    med, mn = timed(chain, reps=50, warm=5)
    # host wall time per contract (plan-cache hits, includes launch latency)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(50):
        chain()
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) / 50
    got = outs["E"].cpu().numpy()
    ref = got
    # (b) the whole chain as one kernel (tci_mps_overlap)
    nout = torch.empty(1, 1, dtype=torch.float64, device="cuda")
    fk = lambda: ctx.mps_overlap(psi, psi, out=nout)  # noqa: E731
    med_k, _ = timed(fk, reps=200, warm=10)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(200):
        fk()
    torch.cuda.synchronize()
    wall_k = (time.perf_counter() - t0) / 200
    err_k = float(abs(nout.cpu().numpy() - ref).max() / abs(ref).max())   # one-kernel chain vs 20 contracts
    # (c) CUDA graph of the 20-contract chain
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        ctx_g = tci.Context(0, s)
        Eg0 = torch.ones(1, 1, dtype=torch.float64, device="cuda")

        def chain_g():
            E = Eg0
            for A in psi:
                X = ctx_g.contract(E, "xz", A, "xsy", "zsy")
                E = ctx_g.contract(X, "zsy", A, "zsw", "yw")
            return E
        chain_g()                       # warm: plans cached, workspace attached
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=s):
            Eg = chain_g()
    torch.cuda.current_stream().wait_stream(s)
    med_g, _ = timed(lambda: g.replay(), reps=200, warm=10)
    err_g = float(abs(Eg.cpu().numpy() - ref).max() / abs(ref).max())
    # (d) the same chain recorded through the C ABI (tci_graph_begin / end, ctx.capture) and replayed:
    # wall time per chain from the host's point of view (one tci_graph_launch)
    s2 = torch.cuda.Stream()
    ctx_c = tci.Context(0, s2)
    bufs = {}

    def chain_c():
        E = E0
        for i, A in enumerate(psi):
            X = ctx_c.contract(E, "xz", A, "xsy", "zsy", out=bufs.get(("X", i)))
            bufs[("X", i)] = X
            E = ctx_c.contract(X, "zsy", A, "zsw", "yw", out=bufs.get(("E", i)))
            bufs[("E", i)] = E
        return E
    chain_c()
    torch.cuda.synchronize()
    gc, Ec = ctx_c.capture(chain_c)
    for _ in range(10):
        ctx_c.replay(gc)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(200):
        ctx_c.replay(gc)
    torch.cuda.synchronize()
    wall_c = (time.perf_counter() - t0) / 200
    err_c = float(abs(Ec.cpu().numpy() - ref).max() / abs(ref).max())
    tci.tci_graph_destroy(gc)
    ctx_c.close()
    return {"workload": "10-site MPS norm, chi=16, d=2, f64 (20 contracts, 46808 MACs)",
            "tci_graph_us_per_chain_wall": wall_c * 1e6, "tci_graph_us_per_contract_wall": wall_c * 1e6 / 20,
            "tci_graph_rel_err": err_c,
            "gpu_us_per_chain_device": med * 1e6, "gpu_us_per_contract_device": med * 1e6 / 20,
            "gpu_us_per_chain_wall": wall * 1e6, "gpu_us_per_contract_wall": wall * 1e6 / 20,
            "single_kernel_us_per_chain_device": med_k * 1e6, "single_kernel_us_per_chain_wall": wall_k * 1e6,
            "single_kernel_rel_err": err_k,
            "cuda_graph_us_per_chain_device": med_g * 1e6, "cuda_graph_rel_err": err_g}


def heff_cfg(ctx, name, reps=3):
    cfg = synth.HEFF_CONFIGS[name]
    inp = synth.heff_inputs(cfg["chi"], cfg["d"], cfg["D"], cfg["dtype"], cfg["seed"], cfg["model"], device="cuda")
    out = torch.empty(inp["psi"].shape[0], cfg["d"], cfg["d"], cfg["chi"], dtype=inp["psi"].dtype, device="cuda")
    f = lambda: ctx.heff_apply(inp["L"], inp["W1"], inp["W2"], inp["R"], inp["psi"], out=out)  # noqa: E731
    med, mn = timed(f, reps=reps, warm=1)
    F = synth.heff_flops(cfg["chi"], cfg["d"], cfg["D"])
    tci.tci_profile_enable(ctx.handle, True)
    f()
    g = tci.tci_profile_query(ctx.handle, tci.PROF_GEMM)
    sk = tci.tci_profile_query(ctx.handle, tci.PROF_SKINNY)
    tci.tci_profile_enable(ctx.handle, False)
    res = {"workload": name, "tflops": F / med / 1e12, "tflops_best": F / mn / 1e12, "s_per_apply": med,
           "pct_fp64_peak": F / med / FP64_PEAK * 100,
           "gemm_tflops": g["flops"] / (g["ms"] / 1e3) / 1e12,
           "skinny_gbs": sk["bytes"] / (sk["ms"] / 1e3) / 1e9 if sk["launches"] else None,
           "skinny_share": sk["ms"] / 1e3 / med}
    del inp, out
    torch.cuda.empty_cache()
    return res


def shard_projection(ctx, name="target_heisenberg_chi4096", reps=5, ag_gbs=770.0):
    """Per-rank step of the sharded apply emulated on one GPU:
    rank r of P computes out[b_r] from L[:, :, b_r] and the full psi, W, R --
    exactly the launch sequence bench.py --gpus P runs on each rank, minus the
    all-gather, which is estimated as (P-1)/P |out| at the measured 770 GB/s
    NVLink peer bandwidth (B200_PROFILING.md). Projection, not a P-GPU run."""
    from paper_2512_23917_b200.sharding import slice_environment
    cfg = synth.HEFF_CONFIGS[name]
    chi, d, D = cfg["chi"], cfg["d"], cfg["D"]
    inp = synth.heff_inputs(chi, d, D, cfg["dtype"], cfg["seed"], cfg["model"], device="cuda")
    F = synth.heff_flops(chi, d, D)
    L_full = inp.pop("L")
    out_bytes = chi * d * d * chi * 16
    rows = []
    t1 = None
    for P in (1, 2, 4, 8):
        res = {"P": P}
        for r in sorted({0, P - 1}):
            L = slice_environment(L_full, P, r)
            out = torch.empty(chi // P, d, d, chi, dtype=inp["psi"].dtype, device="cuda")
            f = lambda: ctx.heff_apply(L, inp["W1"], inp["W2"], inp["R"], inp["psi"], out=out)  # noqa: E731
            med, _ = timed(f, reps=reps, warm=2)
            res[f"rank{r}_ms"] = med * 1e3
            del L, out
            torch.cuda.empty_cache()
        t_rank = max(res[k] for k in res if k.startswith("rank")) / 1e3
        t_ag = (P - 1) / P * out_bytes / (ag_gbs * 1e9) if P > 1 else 0.0
        if P == 1:
            t1 = t_rank
        res.update({"allgather_ms_est": t_ag * 1e3, "step_ms_proj": (t_rank + t_ag) * 1e3,
                    "tflops_proj": F / (t_rank + t_ag) / 1e12, "speedup_proj": t1 / (t_rank + t_ag),
                    "speedup_compute_only": t1 / t_rank})
        rows.append(res)
    del inp, L_full
    torch.cuda.empty_cache()
    return {"workload": name, "rows": rows}


def lanczos_cfg(ctx, name="target_heisenberg_chi4096", iters=(5, 20)):
    """The two-site DMRG local solve the north star frames H_eff.psi inside: the
    Lanczos driver (tci_heff_lanczos: apply, full reorthogonalisation, host
    tridiagonal solve) at the bench workload. Time per iteration from two runs
    of different Krylov dimension (the difference removes the setup)."""
    cfg = synth.HEFF_CONFIGS[name]
    inp = synth.heff_inputs(cfg["chi"], cfg["d"], cfg["D"], cfg["dtype"], cfg["seed"], cfg["model"], device="cuda")
    res = {"workload": name}
    for n in iters:
        psi = inp["psi"].clone()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        energy, it = ctx.heff_lanczos(inp["L"], inp["W1"], inp["W2"], inp["R"], psi, max_iter=n, tol=0.0)
        torch.cuda.synchronize()
        res[f"iters_{n}"] = {"s": time.perf_counter() - t0, "iterations": it, "energy": energy}
    a, b = res[f"iters_{iters[0]}"], res[f"iters_{iters[1]}"]
    per = (b["s"] - a["s"]) / max(1, b["iterations"] - a["iterations"])
    F = synth.heff_flops(cfg["chi"], cfg["d"], cfg["D"])
    res.update({"s_per_iteration": per, "apply_tflops_in_lanczos": F / per / 1e12})
    del inp
    torch.cuda.empty_cache()
    return res


def env_cfg(ctx, chi=4096, d=2, D=5, reps=3):
    """Environment updates (8(f3)) at the target scale, both sides, c128:
    GEMM (E.ket) -> skinny MPO pass -> conj(bra) -> GEMM; bra = ket."""
    res = {}
    for side in (0, 1):
        E = synth.random_tensor((chi, D, chi), "c128", 700, 1, device="cuda")
        ket = synth.random_tensor((chi, d, chi), "c128", 700, 2, device="cuda")
        W = synth.random_tensor((D, D, d, d), "c128", 700, 3, device="cuda")
        out = torch.empty((chi, D, chi), dtype=torch.complex128, device="cuda")
        f = lambda: ctx.env_update(side, E, ket, W, out=out)  # noqa: E731
        med, mn = timed(f, reps=reps, warm=1)
        F = 8.0 * (2 * chi * D * chi * d * chi + chi * chi * (D * d) * (D * d))
        tci.tci_profile_enable(ctx.handle, True)
        f()
        g = tci.tci_profile_query(ctx.handle, tci.PROF_GEMM)
        sk = tci.tci_profile_query(ctx.handle, tci.PROF_SKINNY)
        tci.tci_profile_enable(ctx.handle, False)
        res["left" if side == 0 else "right"] = {
            "chi": chi, "d": d, "D": D, "tflops": F / med / 1e12, "tflops_best": F / mn / 1e12,
            "s_per_update": med, "algorithm": ctx.gemm_algorithm_name(),
            "gemm_share": g["ms"] / 1e3 / med, "skinny_gbs": sk["bytes"] / (sk["ms"] / 1e3) / 1e9 if sk["launches"] else None}
        del E, ket, W, out
        torch.cuda.empty_cache()
    return res


def cfg3(ctx):
    c = synth.TEBD_CONFIG
    res = {}
    for layout, la, lb, lt in (("natural", "asb", "btc", "apqc"), ("physical_first", "sab", "tbc", "paqc")):
        inp = synth.tebd_inputs(c["chi"], c["d"], c["dtype"], c["seed"], c["tau"], device="cuda",
                                physical_first=layout == "physical_first")
        out = None
        holder = {}

        def f():
            holder["t"] = ctx.tebd_theta(inp["A"], la, inp["B"], lb, inp["U"], "pqst", lt, out=holder.get("t"))
        med, mn = timed(f, reps=10, warm=2)
        chi, d = c["chi"], c["d"]
        F = 2.0 * (chi * d) * chi * (d * chi) + 2.0 * d ** 4 * chi * chi
        byts = 8.0 * (2 * chi * d * chi + d * d * chi * chi)
        tci.tci_profile_enable(ctx.handle, True)
        f()
        g = tci.tci_profile_query(ctx.handle, tci.PROF_GEMM)
        sk = tci.tci_profile_query(ctx.handle, tci.PROF_SKINNY)
        pm = tci.tci_profile_query(ctx.handle, tci.PROF_PERMUTE)
        tci.tci_profile_enable(ctx.handle, False)
        res[layout] = {"tflops": F / med / 1e12, "us": med * 1e6, "pct_fp64_peak": F / med / FP64_PEAK * 100,
                       "gemm_tflops": g["flops"] / (g["ms"] / 1e3) / 1e12, "gemm_ms": g["ms"],
                       "gate_pass_ms": sk["ms"], "permute_ms": pm["ms"], "permute_launches": pm["launches"],
                       "min_traffic_bytes": byts}
        del inp
        torch.cuda.empty_cache()
    res["workload"] = "TEBD theta chi=2048 d=2 f64 (68.7 GFLOP + gate)"
    return res


def svd_cfg(ctx, reps=2):
    """truncated SVD after the TEBD theta of config 3 (chi = 2048:
    a 4096 x 4096 f64 matrix of rank <= 2048) and after a two-site DMRG solve
    (chi = 1024, d = 2: a 2048 x 2048 c128 matrix), each truncated back to chi;
    LAPACK (gesdd via numpy) times the same matrix on the host."""
    res = {}
    c = synth.TEBD_CONFIG
    cases = [("tebd_theta_chi2048_r64", None), ("dmrg_two_site_chi1024_c128", None)]
    for name, _ in cases:
        if name.startswith("tebd"):
            inp = synth.tebd_inputs(c["chi"], c["d"], c["dtype"], c["seed"], c["tau"], device="cuda")
            th = ctx.tebd_theta(inp["A"], "asb", inp["B"], "btc", inp["U"], "pqst", "apqc")
            chi = c["chi"]
            del inp
        else:
            chi = 1024
            th = synth.random_tensor((chi, 2, 2, chi), "c128", 9, 2, device="cuda")
        holder = {}

        def f():
            holder["r"] = ctx.trunc_svd(th, 2, 1, chi, 0.0, 1e-14)
        med, mn = timed(f, reps=reps, warm=1)
        sweeps, off = ctx.svd_info()
        u, s, vd, err = holder["r"]
        A = th.cpu().numpy().reshape(th.shape[0] * th.shape[1], -1)
        t0 = time.time()
        rs = np.linalg.svd(A, compute_uv=False)
        t_or = time.time() - t0
        sh = s.cpu().numpy()
        k = sh.shape[0]
        res[name] = {"shape": list(A.shape), "chi_kept": int(k), "trunc_err": err, "ms": med * 1e3,
                     "ms_min": mn * 1e3, "sweeps": sweeps, "final_off": off,
                     "max_abs_ds_over_s0": float(np.max(np.abs(sh - rs[:k])) / rs[0]),
                     "lapack_numpy_gesdd_values_only_s": t_or, "host_threads": os.cpu_count()}
        del th, holder, u, s, vd
        torch.cuda.empty_cache()
    return res


def mpo_apply_cfg(ctx, chi=4096, d=2, D=5):
    """site-local uncompressed MPS-MPO application
    B[a,w,t,b,v] = sum_s A[a,s,b] W[w,v,s,t] at chi = 4096, d = 2, D = 5, c128
    (A 537 MB -> B 13.4 GB): HBM-bound, roofline = bytes / measured copy BW."""
    A = synth.random_tensor((chi, d, chi), "c128", 31, 1, device="cuda")
    Wh, _, _ = synth.heisenberg_mpo(1.0)
    W = torch.from_numpy(np.asarray(Wh)).to(torch.complex128).cuda()
    holder = {}

    def f():
        holder["b"] = ctx.contract(A, "asb", W, "wvst", "awtbv", out=holder.get("b"))
    med, mn = timed(f, reps=5, warm=2)
    byts = 16.0 * (A.numel() + W.numel() + chi * D * d * chi * D)
    tci.tci_profile_enable(ctx.handle, True)
    f()
    sk = tci.tci_profile_query(ctx.handle, tci.PROF_SKINNY)
    g = tci.tci_profile_query(ctx.handle, tci.PROF_GEMM)
    pm = tci.tci_profile_query(ctx.handle, tci.PROF_PERMUTE)
    tci.tci_profile_enable(ctx.handle, False)
    res = {"workload": f"MPS-MPO site apply chi={chi} d={d} D={D} c128", "ms": med * 1e3, "GBs": byts / med / 1e9,
           "frac_hbm": byts / med / HBM, "bytes": byts, "skinny_launches": sk["launches"],
           "gemm_launches": g["launches"], "permute_launches": pm["launches"]}
    del A, W, holder
    torch.cuda.empty_cache()
    return res


def sweep(ctx, seeds=24):
    """Config 5: random rank 3..6 contractions up to 2^28 elements, f64 and f32."""
    rng = np.random.default_rng(5)
    rows = []
    for s in range(seeds):
        for dt in ("r64", "r32"):
            la, lb, lc, dims, sh = synth.sweep_instance(rng)

            def size(ls):
                return int(np.prod([dims[l] for l in ls], dtype=np.int64))
            A = synth.random_tensor([dims[l] for l in la], dt, 5000 + s, 1, device="cuda")
            B = synth.random_tensor([dims[l] for l in lb], dt, 5000 + s, 2, device="cuda")
            la_, lb_, lc_ = la, lb, lc
            holder = {}
            f = lambda: holder.__setitem__("c", ctx.contract(A, la_, B, lb_, lc_, out=holder.get("c")))  # noqa
            med, _ = timed(f, reps=3, warm=1)
            es = 8 if dt == "r64" else 4
            S = size(sh)
            flops = 2.0 * size(lc) * S
            t_roof = max(flops / (FP64_PEAK if dt == "r64" else FP32_PEAK), (size(la) + size(lb) + size(lc)) * es / HBM)
            rows.append({"dtype": dt, "la": la_, "lb": lb_, "lc": lc_, "dims": dims, "elems_max": max(size(la), size(lb), size(lc)),
                         "us": med * 1e6, "roofline_us": t_roof * 1e6, "frac_of_roofline": t_roof / med})
            del A, B, holder
    fr = [r["frac_of_roofline"] for r in rows]
    return {"instances": rows, "median_frac_of_roofline": float(np.median(fr)),
            "geomean_frac_of_roofline": float(np.exp(np.mean(np.log(fr))))}


def permute_bw(ctx):
    rows = []
    for shape, perm, dt in [((4096, 4096, 16), (1, 0, 2), "r64"), ((512, 512, 512), (2, 1, 0), "r64"),
                            ((64, 64, 64, 64, 16), (4, 3, 2, 1, 0), "r64"), ((8192, 8192, 2), (2, 1, 0), "c128"),
                            ((16384, 16384), (1, 0), "r32"), ((2048, 2048, 32), (0, 2, 1), "r64"),
                            ((32, 64, 48, 40, 36), (3, 0, 4, 2, 1), "r32"), ((96, 96, 96, 24), (2, 3, 0, 1), "c64"),
                            ((3, 5, 7, 1024, 512), (4, 2, 0, 3, 1), "r64")]:
        x = synth.random_tensor(shape, dt, 9, 1, device="cuda")
        y = torch.empty([shape[p] for p in perm], dtype=x.dtype, device="cuda")
        med, _ = timed(lambda: ctx.permute(x, list(perm), out=y), reps=10, warm=2)
        byts = 2.0 * x.numel() * x.element_size()
        # plain device copy of the same bytes (torch copy_), same timing: the ceiling beside the peak
        yc = torch.empty_like(x)
        medc, _ = timed(lambda: yc.copy_(x), reps=10, warm=2)
        rows.append({"shape": shape, "perm": perm, "dtype": dt, "GBs": byts / med / 1e9, "frac_hbm": byts / med / HBM,
                     "copy_GBs": byts / medc / 1e9, "frac_of_copy": medc / med})
        del yc
        del x, y
    return rows


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="cfg1,cfg2,cfg3,cfg4,sweep,permute")
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "extra.json"))
    ap.add_argument("--algo", default=None, choices=[None, "dmma3m", "dmma4m", "ozaki"])
    a = ap.parse_args()
    ctx = tci.Context(0)
    if a.algo:
        ctx.set_gemm_algorithm({"dmma3m": tci.TCI_GEMM_DMMA_3M, "dmma4m": tci.TCI_GEMM_DMMA_4M,
                                "ozaki": tci.TCI_GEMM_OZAKI_INT8}[a.algo])
    res = {}
    for k in a.only.split(","):
        if k == "cfg1":
            res["cfg1"] = cfg1(ctx)
        elif k == "cfg2":
            res["cfg2"] = heff_cfg(ctx, "cfg2_heisenberg_chi1024", reps=5)
        elif k == "cfg3":
            res["cfg3"] = cfg3(ctx)
        elif k == "cfg4":
            res["cfg4"] = heff_cfg(ctx, "cfg4_hubbard_chi4096", reps=2)
        elif k == "sweep":
            res["sweep"] = sweep(ctx)
        elif k == "permute":
            res["permute"] = permute_bw(ctx)
        elif k == "mpo":
            res["mpo"] = mpo_apply_cfg(ctx)
        elif k == "svd":
            res["svd"] = svd_cfg(ctx)
        elif k == "lanczos":
            res["lanczos"] = lanczos_cfg(ctx)
        elif k == "shards":
            res["shards"] = shard_projection(ctx)
        elif k == "shards4":
            res["shards4"] = shard_projection(ctx, "cfg4_hubbard_chi4096", reps=2)
        elif k == "env":
            res["env"] = env_cfg(ctx)
        print(k, json.dumps(res.get(k))[:600], flush=True)
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    json.dump(res, open(a.out, "w"), indent=1)
    ctx.close()


if __name__ == "__main__":
    main()
