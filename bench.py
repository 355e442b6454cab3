#!/usr/bin/env python
"""Benchmark: DMRG two-site H_eff.psi apply (BASELINE.json metric
"DMRG H_eff.psi TFLOP/s (fp64, chi=4096) at 1/2/4/8 GPU; % FP64 TC peak").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config target|cfg2|cfg4]
                    [--impl tci|reference]

A step is one H_eff.psi apply (L.psi GEMM -> W1,W2 MPO pass -> .R GEMM) over
the synthetic workload, plus (N > 1) the NCCL all-gather of the output shards
-- one Lanczos step's worth of the hot path. Default
workload: chi=4096, d=2, D=5, complex128, Heisenberg MPO (the north-star
target shape). value = the full (unsharded) apply's
algorithmic flops (8 per complex MAC, FLOP-optimal order) / device time per
step, max over ranks. Inputs (>= 1 GB each) exceed the 126 MB L2, so no flush
is needed between steps.

--impl reference times the CPU oracle (oracle/, plain loops) on the box's
host cores on a bounded sample of output rows of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402

METRIC = "DMRG H_eff.psi TFLOP/s (fp64, chi=4096) at 1/2/4/8 GPU; % FP64 TC peak"
UNIT = "TFLOP/s"
CONFIGS = {
    "target": "target_heisenberg_chi4096",
    "cfg2": "cfg2_heisenberg_chi1024",
    "cfg4": "cfg4_hubbard_chi4096",
}
# FP64 tensor-core (DMMA) peak measured on this pool's B200 by the step-0
# probe (tools/probe_fp64.cu; profiles/step0_fp64_probe.json): register-
# resident mma.sync.m8n8k4.f64 at 1965 MHz. MEASURED_PEAKS.json has no FP64
# entry; cuBLAS ZGEMM 8192^3 measured 37.01 TF/s on the same box.
FP64_PEAK_TFLOPS = 37.06
FP64_PEAK_SOURCE = "measured DMMA microbenchmark (profiles/step0_fp64_probe.json)"


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f), "MEASURED_PEAKS.json"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}, "fallback (B200_PROFILING.md)"


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if os.environ.get("TCI_BENCH_SAME_DEVICE") == "1":
        local = 0   # test harness: every rank on cuda:0 (multi-process check of the N > 1 path on one GPU)
    return ws, rank, local


# process-group backend: NCCL (default); TCI_BENCH_BACKEND=gloo is the
# single-GPU multi-process test harness (NCCL refuses two ranks on one device)
BACKEND = os.environ.get("TCI_BENCH_BACKEND", "nccl")


class ClockSampler:
    """nvidia-smi clocks / throttle reasons during the timed region."""
    FIELDS = ["index", "clocks.sm", "clocks.max.sm", "power.draw", "clocks_event_reasons.active",
              "clocks_event_reasons.hw_slowdown", "clocks_event_reasons.hw_thermal_slowdown",
              "clocks_event_reasons.sw_thermal_slowdown", "clocks_event_reasons.sw_power_cap"]

    def __init__(self, gpu_index: int):
        self.proc = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={','.join(self.FIELDS)}", "--format=csv,noheader,nounits",
                 "-lms", "200", "-i", str(gpu_index)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL,
                text=True)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:
            self.proc.kill()
            out = ""
        sm, smax, reasons, power = [], [], set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax.append(float(parts[2]))
                power.append(float(parts[3]))
            except ValueError:
                continue
            for n, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "power_w_max": max(power) if power else None,
                "samples": len(sm), "reasons": sorted(reasons)}


def gpu_index(local_rank: int) -> int:
    vis = os.environ.get("CUDA_VISIBLE_DEVICES")
    if vis:
        ids = [v.strip() for v in vis.split(",") if v.strip()]
        if local_rank < len(ids) and ids[local_rank].isdigit():
            return int(ids[local_rank])
    return local_rank


def traffic_from_profiles(workload: str):
    """dram bytes/launch of the dominant kernel from a committed ncu --set full
    capture summary (profiles/ncu_traffic.json), or None."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return d.get(workload, {}).get("gemm_dram_bytes_per_launch")
    except Exception:
        return None


# ---------------------------------------------------------------------------
# CPU oracle (reference arm and cpu_baseline): bounded sample of output rows
# ---------------------------------------------------------------------------

def oracle_rows_run(inp_np, rows):
    import oracle
    t0 = time.perf_counter()
    res = oracle.heff_rows(inp_np["L"], inp_np["W1"], inp_np["W2"], inp_np["R"], inp_np["psi"], rows)
    return res, time.perf_counter() - t0


def cpu_model():
    """Host CPU model name (lscpu's "Model name"), for the cpu_baseline record."""
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


def cpu_baseline(inp_np, chi, flops_full, budget_s=15.0, gpu_out=None):
    import oracle
    oracle.build()
    rng = np.random.default_rng(0)
    rows = [0]
    res, t1 = oracle_rows_run(inp_np, rows)
    n_more = int(max(0, min(chi - 1, budget_s / max(t1, 1e-3) - 1)))
    more = sorted(set(int(x) for x in rng.integers(1, chi, size=n_more)) | {chi - 1})[:max(n_more, 1)]
    res2, t2 = oracle_rows_run(inp_np, more)
    rows_all = rows + more
    t = t1 + t2
    val = len(rows_all) * (flops_full / chi) / t / 1e12
    out = {"value": val, "unit": UNIT, "cores": oracle.max_threads(), "kind": "oracle",
           "cpu_model": cpu_model(), "host_cpus": os.cpu_count(),
           "sample": f"{len(rows_all)} output rows b (of {chi}) of the same apply, exact chain "
                     f"(oracle.heff_rows: L sliced at b); {t:.1f} s; TFLOP/s = rows x flops/row / time"}
    parity = None
    if gpu_out is not None:
        ref = np.concatenate([res, res2])
        got = gpu_out[rows_all]
        parity = {"rows_checked": len(rows_all),
                  "rel_frob": float(np.linalg.norm(got - ref) / np.linalg.norm(ref))}
    return out, parity


# ---------------------------------------------------------------------------
# reference arm (the oracle), bench contract "--impl reference"
# ---------------------------------------------------------------------------

def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    import oracle
    oracle.build()
    name = CONFIGS[args.config]
    cfg = synth.HEFF_CONFIGS[name]
    chi, d, D = cfg["chi"], cfg["d"], cfg["D"]
    inp = synth.heff_inputs(chi, d, D, cfg["dtype"], cfg["seed"], cfg["model"], device="cpu")
    inp_np = {k: v.numpy() for k, v in inp.items()}
    F = synth.heff_flops(chi, d, D)
    rows_per_step = args.ref_rows
    rng = np.random.default_rng(1)
    for _ in range(args.warmup):
        oracle_rows_run(inp_np, [int(x) for x in rng.integers(0, chi, size=rows_per_step)])
    times = []
    for _ in range(args.steps):
        _, t = oracle_rows_run(inp_np, [int(x) for x in rng.integers(0, chi, size=rows_per_step)])
        times.append(t)
    t = float(np.mean(times))
    val = rows_per_step * (F / chi) / t / 1e12
    line = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64" if cfg["dtype"] == "r64" else "c128",
        "data": "synthetic (seeded counter-based generator; exact model MPO)",
        "config": {"workload": name, "chi": chi, "d": d, "D": D, "dtype": cfg["dtype"], "model": cfg["model"]},
        "cpu_baseline": {"value": val, "unit": UNIT, "cores": oracle.max_threads(), "kind": "oracle",
                         "cpu_model": cpu_model(), "host_cpus": os.cpu_count(),
                         "sample": f"{rows_per_step} output rows per step (of {chi}); TFLOP/s = rows x "
                                   f"full-apply flops/chi / time"},
        "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# the CUDA path
# ---------------------------------------------------------------------------

def run_tci(args):
    import paper_2512_23917_b200 as tci
    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    if ws > 1:
        import torch.distributed as dist
        if BACKEND == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(BACKEND)
    name = CONFIGS[args.config]
    cfg = synth.HEFF_CONFIGS[name]
    chi, d, D, dt = cfg["chi"], cfg["d"], cfg["D"], cfg["dtype"]
    if chi % ws:
        raise SystemExit(f"chi={chi} not divisible by {ws} ranks")
    chi_lo = chi // ws
    F = synth.heff_flops(chi, d, D, complex_=dt == "c128")
    dev = torch.device("cuda", local)
    stream = torch.cuda.Stream(device=dev)
    torch.cuda.set_stream(stream)

    # inputs, generated on the device (same generator as the oracle side)
    inp = synth.heff_inputs(chi, d, D, dt, cfg["seed"], cfg["model"], device=dev)
    from paper_2512_23917_b200.sharding import ShardedHeff, slice_environment
    L_full = inp.pop("L")
    L = slice_environment(L_full, ws, rank)          # this rank's L[:, :, b_r] (setup)
    del L_full
    W1, W2, R, psi = inp["W1"], inp["W2"], inp["R"], inp["psi"]
    torch.cuda.synchronize()

    ctx = tci.Context(local, stream)
    if args.algo:
        ctx.set_gemm_algorithm({"dmma3m": tci.TCI_GEMM_DMMA_3M, "dmma4m": tci.TCI_GEMM_DMMA_4M,
                                "ozaki": tci.TCI_GEMM_OZAKI_INT8}[args.algo])
    ALGOS = {"dmma3m": tci.TCI_GEMM_DMMA_3M, "dmma4m": tci.TCI_GEMM_DMMA_4M, "ozaki": tci.TCI_GEMM_OZAKI_INT8}
    algo = {0: "dmma3m", 1: "dmma4m", 2: "ozaki"}[tci.tci_get_gemm_algorithm(ctx.handle)]
    def nccl_comm_init():
        # the library's NCCL communicator: only for the NCCL all-gather (the
        # peer-memory gather needs none)
        import torch.distributed as dist
        obj = [tci.tci_comm_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        ctx.comm_init(obj[0], ws, rank)
    gather = "none" if ws == 1 else args.gather
    sh = None
    if ws > 1 and gather == "p2p":
        # all-gather over peer memory, fused into the GEMM4 (Ozaki CRT) epilogue
        try:
            from paper_2512_23917_b200.sharding import PeerGatherHeff

            def exchange(obj):
                import torch.distributed as dist
                allo = [None] * ws
                dist.all_gather_object(allo, obj)
                return allo

            def agree(ok):
                import torch.distributed as dist
                t = torch.tensor([1 if ok else 0], dtype=torch.int32, device=dev)
                dist.all_reduce(t, op=dist.ReduceOp.MIN)
                return bool(t.item())
            sh = PeerGatherHeff(ctx, L, W1, W2, R, ws, rank, exchange=exchange, agree=agree)
        except Exception as e:   # no P2P / IPC on this box: NCCL all-gather instead
            print(f"[rank {rank}] peer-memory gather unavailable ({e}); using NCCL", file=sys.stderr, flush=True)
            sh = None
        ok = torch.tensor([1 if sh is not None else 0], dtype=torch.int32, device=dev)
        import torch.distributed as dist
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)
        if int(ok.item()) == 0:
            gather = "nccl"
            if sh is not None:
                sh.close()
                sh = None
    if sh is None:
        if ws > 1:
            nccl_comm_init()
        sh = ShardedHeff(ctx, L, W1, W2, R, ws, rank)
    out = sh.out

    def step():
        sh.apply(psi)       # tci_heff_apply on the slab (+ tci_allgather when ws > 1)

    def barrier():
        if ws > 1:
            import torch.distributed as dist
            if BACKEND == "nccl":
                dist.barrier(device_ids=[local])
            else:
                dist.barrier()

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if gather == "p2p" and ctx.gather_status():
        raise SystemExit(f"[rank {rank}] peer-memory gather barrier timed out (rerun with --gather nccl)")

    # ---- timed region (device time, CUDA events on the launching stream) ----
    sampler = ClockSampler(gpu_index(local)) if rank == 0 else None
    time.sleep(0.3 if sampler else 0)
    ctx.ozaki_guard_stats(reset=True)
    n0 = ctx.launch_count()
    barrier()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    barrier()
    t_step = e0.elapsed_time(e1) / 1e3 / args.steps
    launches = ctx.launch_count() - n0
    clocks = sampler.stop() if sampler else None
    # Ozaki accuracy guard over the timed steps (R26): GEMMs checked,
    # recomputed on DMMA, largest estimated relative Frobenius error
    gs = ctx.ozaki_guard_stats()
    guard = {"ozaki_gemms": gs["gemms"], "dmma_recomputations": gs["fallbacks"],
             "balanced": gs["balanced"], "max_est_rel_frob": gs["max_est"]} if algo == "ozaki" else None
    if gather == "p2p" and ctx.gather_status():
        raise SystemExit(f"[rank {rank}] peer-memory gather barrier timed out in the timed region")
    # per-kernel profile (roofline inputs) from separate steps: CUDA events on
    # the context stream around every GEMM / INT8 GEMM / MPO-pass launch
    # (kept out of the timed region above)
    prof_steps = max(1, min(args.steps, 3))
    tci.tci_profile_enable(ctx.handle, True)
    torch.cuda.synchronize()
    ep0 = torch.cuda.Event(enable_timing=True)
    ep1 = torch.cuda.Event(enable_timing=True)
    ep0.record(stream)
    for _ in range(prof_steps):
        step()
    ep1.record(stream)
    torch.cuda.synchronize()
    t_prof = ep0.elapsed_time(ep1) / 1e3
    prof = {k: tci.tci_profile_query(ctx.handle, v) for k, v in
            (("gemm", tci.PROF_GEMM), ("skinny", tci.PROF_SKINNY), ("permute", tci.PROF_PERMUTE),
             ("int8_gemm", tci.PROF_I8))}
    tci.tci_profile_enable(ctx.handle, False)
    if ws > 1:
        import torch.distributed as dist
        tt = torch.tensor([t_step], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_step = float(tt.item())
        ln = torch.tensor([launches], dtype=torch.int64, device=dev)
        dist.all_reduce(ln)
        launches = int(ln.item())
    value = F / t_step / 1e12

    # ---- the other complex GEMM algorithm on the same inputs (same timing rules) ----
    alt = None
    if args.alt and args.alt != "none" and args.alt != algo:
        ctx.set_gemm_algorithm(ALGOS[args.alt])
        for _ in range(2):
            step()
        torch.cuda.synchronize()
        barrier()
        torch.cuda.synchronize()
        e0.record(stream)
        ka = max(1, min(args.steps, 3))
        for _ in range(ka):
            step()
        e1.record(stream)
        torch.cuda.synchronize()
        ta = e0.elapsed_time(e1) / 1e3 / ka
        if ws > 1:
            import torch.distributed as dist
            tt = torch.tensor([ta], dtype=torch.float64, device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            ta = float(tt.item())
        alt_out = out.clone() if ws == 1 else None
        alt = {"algorithm": args.alt, "value": F / ta / 1e12, "ms_per_step": ta * 1e3, "steps": ka,
               "pct_fp64_tc_peak": F / ta / 1e12 / FP64_PEAK_TFLOPS * 100}
        ctx.set_gemm_algorithm(ALGOS[algo])
        step()
        torch.cuda.synchronize()
        if alt_out is not None:
            diff = (out - alt_out).abs().pow(2).sum().sqrt() / alt_out.abs().pow(2).sum().sqrt()
            alt["rel_frob_vs_main"] = float(diff.item())
        del alt_out

    # ---- end to end through the C ABI with pinned host buffers ----
    e2e = None
    if not args.no_e2e:
        hosts = {k: x.cpu().pin_memory() for k, x in (("L", L), ("W1", W1), ("W2", W2), ("R", R), ("psi", psi))}
        res_dev = sh.full if ws > 1 else out      # the step's result: the gathered output at N > 1
        hout = torch.empty(res_dev.shape, dtype=res_dev.dtype).pin_memory()
        devs = {"L": L, "W1": W1, "W2": W2, "R": R, "psi": psi}
        h2d = sum(x.numel() * x.element_size() for x in hosts.values())
        d2h = hout.numel() * hout.element_size()

        staged = ws == 1

        def e2e_step():
            if staged:
                # tci_heff_apply_staged: the H2D copies of L, psi, W and R and the
                # chunked D2H of the result overlap the computation
                ctx.heff_apply_staged([hosts[k] for k in ("L", "W1", "W2", "R", "psi")] + [hout],
                                      [devs[k] for k in ("L", "W1", "W2", "R", "psi")] + [out])
                return
            for k in hosts:
                ctx.copy(hosts[k], devs[k])        # tci_copy: pinned host -> device
            step()
            ctx.copy(res_dev, hout)                 # tci_copy: device -> pinned host
        e2e_step()
        torch.cuda.synchronize()
        ke = max(1, min(args.steps, 3))
        barrier()
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(ke):
            e2e_step()
        e1.record(stream)
        torch.cuda.synchronize()
        te = e0.elapsed_time(e1) / 1e3 / ke
        if ws > 1:
            import torch.distributed as dist
            tt = torch.tensor([te], dtype=torch.float64, device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            te = float(tt.item())
        e2e = {"value": F / te / 1e12, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "ms_per_step": te * 1e3,
               "path": ("tci_heff_apply_staged (pinned host inputs/outputs; psi + W copied first, L streamed in "
                        "8 column blocks behind GEMM1's row chunks, R behind L, D2H in 8 row chunks behind "
                        "GEMM4)") if staged else
                       ("tci_copy(pinned host->device) x5, tci_heff_apply_gather (peer-memory all-gather in the "
                        "GEMM4 epilogue), tci_copy(device->host)" if gather == "p2p" else
                        "tci_copy(pinned host->device) x5, tci_heff_apply, tci_allgather, tci_copy(device->host)")}
        if not args.no_pipeline:
            # Streaming applies (steady state of a stream of independent H_eff.psi
            # problems): device inputs double-buffered; step i+1's five
            # host->device copies run on copy lane 1 and step i-1's device->host
            # copy on lane 2 while step i computes on the context stream. Every
            # step still copies all of its inputs in and its result out inside
            # the timed region (the first step's copies start after e0). At
            # N > 1 the result is the gathered full output (one buffer: the
            # context stream waits for its previous copy-out before the step,
            # so no rank writes into it early -- the gather's entry barrier
            # follows that wait).
            KEYS = ("L", "W1", "W2", "R", "psi")
            bufs = [devs, {k: torch.empty_like(v) for k, v in devs.items()}]
            if ws == 1:
                outs = [out, torch.empty_like(out)]
            else:
                outs = [sh.full, sh.full]
            IN, DONE, OUT, START = 0, 2, 4, 6    # lane event slots (+ buffer index)

            def compute(b):
                x = [bufs[b][k] for k in KEYS]
                if ws == 1:
                    ctx.heff_apply(*x, out=outs[b])
                elif gather == "p2p":
                    ctx.heff_apply_gather(*x, sh.full)
                else:
                    ctx.heff_apply(*x, out=sh.out)
                    ctx.allgather(sh.out, sh.full)

            def pipelined(n):
                ctx.lane_record(0, START)
                ctx.lane_wait(1, START)

                def load(b):
                    ctx.lane_wait(1, DONE + b)          # the compute that last read buffer b is done
                    for k in KEYS:
                        ctx.copy_async(hosts[k], bufs[b][k], 1)
                    ctx.lane_record(1, IN + b)
                # at N = 1 every step streams its own inputs behind its compute
                # (tci_heff_apply_staged without a host output: psi + W first, L in
                # column blocks as GEMM1 reaches them, R behind L, all on copy lane
                # 1, ordered by the lane events), so the copies of step i + 1 run
                # while step i computes and no step waits for a whole input copy
                staged0 = ws == 1 and not args.no_staged_fill
                if not staged0:
                    load(0)
                for i in range(n):
                    b = i % 2
                    ob = b if ws == 1 else 0
                    if staged0:
                        # every step streams its inputs behind its own compute; copy
                        # lane 1 first waits for the compute that last read buffer b
                        ctx.lane_wait(1, DONE + b)
                        ctx.lane_wait(0, OUT + ob)
                        ctx.heff_apply_staged([hosts[k] for k in KEYS] + [None],
                                              [bufs[b][k] for k in KEYS] + [outs[b]])
                    else:
                        if i + 1 < n:
                            load(1 - b)
                        ctx.lane_wait(0, IN + b)
                        ctx.lane_wait(0, OUT + ob)      # the d2h that last read this output is done
                        compute(b)
                    ctx.lane_record(0, DONE + b)
                    ctx.lane_wait(2, DONE + b)
                    ctx.copy_async(outs[b], hout, 2)
                    ctx.lane_record(2, OUT + ob)
                ctx.lane_wait(0, OUT + ((n - 1) % 2 if ws == 1 else 0))

            pipelined(2)
            torch.cuda.synchronize()
            # a stream of 10 applies (the first step's input copies and the last
            # step's result copy are not overlapped: amortised over the stream)
            kp = max(10, args.steps)
            barrier()
            torch.cuda.synchronize()
            e0.record(stream)
            pipelined(kp)
            e1.record(stream)
            torch.cuda.synchronize()
            tp = e0.elapsed_time(e1) / 1e3 / kp
            if ws > 1:
                import torch.distributed as dist
                tt = torch.tensor([tp], dtype=torch.float64, device=dev)
                dist.all_reduce(tt, op=dist.ReduceOp.MAX)
                tp = float(tt.item())
            if ws == 1:
                ok = bool(torch.equal(outs[0], outs[1])) and bool(torch.equal(hout, outs[(kp - 1) % 2].cpu()))
            else:
                ok = bool(torch.equal(hout, sh.full.cpu()))
            # the PCIe ceiling of this path: one pinned host -> device copy of L alone
            e0.record(stream)
            for _ in range(3):
                bufs[1]["L"].copy_(hosts["L"], non_blocking=True)
            e1.record(stream)
            torch.cuda.synchronize()
            h2d_gbs = 3 * hosts["L"].numel() * hosts["L"].element_size() / (e0.elapsed_time(e1) / 1e3) / 1e9
            e2e_single = dict(e2e)
            e2e = {"value": F / tp / 1e12, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
                   "d2h_bytes_per_step": int(d2h), "ms_per_step": tp * 1e3, "steps": kp,
                   "path": ("streaming applies through the C ABI: tci_copy_async (pinned host -> device, copy "
                            "lane 1) of step i+1's L, W1, W2, R, psi and tci_copy_async (device -> pinned host, "
                            "lane 2) of step i-1's result overlap " +
                            ("tci_heff_apply" if ws == 1 else
                             "tci_heff_apply_gather" if gather == "p2p" else "tci_heff_apply + tci_allgather") +
                            " of step i (double-buffered device inputs, ordered by tci_lane_record / "
                            "tci_lane_wait)" + ("; every step streams its own inputs behind its compute "
                                                "(tci_heff_apply_staged, host output NULL, copy lane ordered by lane events)"
                                                if ws == 1 and not args.no_staged_fill else "")),
                   "results_identical_across_buffers": ok,
                   "h2d_gbs_measured": h2d_gbs,
                   "h2d_bound_ms_per_step": h2d / (h2d_gbs * 1e9) * 1e3,
                   "single_call": e2e_single}
            del bufs, outs
    torch.cuda.synchronize()
    if gather == "p2p" and ctx.gather_status():
        raise SystemExit(f"[rank {rank}] peer-memory gather barrier timed out in the end-to-end loops")

    if rank != 0:
        ctx.close()
        if ws > 1:
            import torch.distributed as dist
            dist.destroy_process_group()
        return

    peaks, peak_src = measured_peaks()
    g = prof["gemm"]
    gemm_avg_s = g["ms"] / 1e3 / max(1, g["launches"])
    gemm_flops_per_launch = g["flops"] / max(1, g["launches"])
    achieved = gemm_flops_per_launch / gemm_avg_s / 1e12 if g["launches"] else None
    traffic = traffic_from_profiles(name)
    sk = prof["skinny"]
    i8 = prof["int8_gemm"]
    if algo == "ozaki" and i8["launches"]:
        # dominant kernel: the hand-written tcgen05 kind::i8 GEMM (i8gemm.cu; all
        # residue products of one Ozaki GEMM in one launch). It runs inside a
        # ~100 ms step under the power cap, so the roofline denominator is the
        # SUSTAINED measured bf16 rate x the nominal int8/bf16 ratio (2); the
        # burst-based fraction is kept beside it.
        i8_peak = peaks.get("bf16_tflops_sustained", peaks.get("bf16_tflops", 1646.4)) * 2.0
        i8_burst = peaks.get("bf16_tflops", 1646.4) * 2.0
        i8_ach = i8["flops"] / (i8["ms"] / 1e3) / 1e12
        roofline = {
            "bound": "tensor",
            "kernel": "i8gemm_kernel (hand-written tcgen05.mma.cta_group::2.kind::i8, TMA, TMEM; UTCIMMA)",
            "achieved": i8_ach, "peak": i8_peak, "unit": "TOPS", "frac": i8_ach / i8_peak,
            "frac_vs_burst_peak": i8_ach / i8_burst,
            "traffic": traffic_from_profiles(name + "_ozaki"),
            "peak_source": ("MEASURED_PEAKS.json bf16_tflops_sustained x 2 (nominal int8/bf16 = 4.5/2.25 PFLOP/s); "
                            "burst: bf16_tflops x 2"),
            "ops_per_launch": i8["flops"] / i8["launches"], "launches": i8["launches"],
            "share_of_step": i8["ms"] / 1e3 / t_prof if t_prof > 0 else None,
            "ozaki_gemm_fp64_equivalent_tflops": achieved,
            "ozaki_gemm_share_of_step": g["ms"] / 1e3 / t_prof if t_prof > 0 else None,
        }
    else:
        roofline = {
            "bound": "tensor", "kernel": "gemm_dmma_kernel (L.psi and T3.R GEMMs, DMMA.8x8x4)",
            "achieved": achieved, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
            "frac": achieved / FP64_PEAK_TFLOPS if achieved else None, "traffic": traffic,
            "peak_source": FP64_PEAK_SOURCE,
            "flops_per_launch": gemm_flops_per_launch, "launches": g["launches"],
            "gemm_share_of_step": g["ms"] / 1e3 / t_prof if t_prof > 0 else None,
        }
    roofline["secondary"] = {
        "kernel": "skinny_dmma_kernel (MPO pass, FP64 tensor cores, 3M)", "bound": "hbm",
        "achieved": (sk["bytes"] / (sk["ms"] / 1e3) / 1e9) if sk["launches"] else None,
        "peak": peaks.get("hbm_gbs"), "unit": "GB/s", "peak_source": peak_src,
        "share_of_step": sk["ms"] / 1e3 / t_prof if t_prof > 0 else None,
    }

    cpu = None
    parity = None
    if ws == 1 and not args.no_cpu_baseline:
        inp_np = {"L": L.cpu().numpy(), "W1": W1.cpu().numpy(), "W2": W2.cpu().numpy(),
                  "R": R.cpu().numpy(), "psi": psi.cpu().numpy()}
        cpu, parity = cpu_baseline(inp_np, chi, F, budget_s=args.cpu_budget, gpu_out=out.cpu().numpy())
    elif ws > 1 and not args.no_cpu_baseline:
        # the gathered output on rank 0 vs oracle rows at both edges of every
        # rank's slab (the all-gather put them there; inputs regenerated on the host)
        import oracle
        oracle.build()
        full_inp = synth.heff_inputs(chi, d, D, dt, cfg["seed"], cfg["model"], device="cpu")
        inp_np = {k: v.numpy() for k, v in full_inp.items()}
        rows = sorted({b for r in range(ws) for b in (r * chi_lo, r * chi_lo + chi_lo - 1)})
        ref, _ = oracle_rows_run(inp_np, rows)
        got = sh.full.cpu().numpy()[rows]
        parity = {"rows_checked": len(rows), "rows": "first and last row of every rank's slab",
                  "rel_frob": float(np.linalg.norm(got - ref) / np.linalg.norm(ref))}
        del full_inp, inp_np

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t_step * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None,
        # the arithmetic the path computes in: INT8 x INT8 -> INT32 residue GEMMs (and the
        # CRT digit GEMM) on the tensor cores, f64 scaling / reconstruction; c128 in and out
        "dtype": ("i8 (tensor-core residue GEMMs, i32 sums) + f64; complex128 data"
                  if algo == "ozaki" else ("c128" if dt == "c128" else "f64")),
        "alt": alt,
        "data": "synthetic (seeded counter-based generator; exact model MPO as W1=W2)",
        "config": {"workload": name, "chi": chi, "d": d, "D": D, "dtype": dt, "model": cfg["model"],
                   "gemm_algorithm": algo, "gather": gather,
                   "parallelism": (f"output bond b sharded over {ws} rank(s); all-gather of out per step "
                                   + ("over peer memory fused into the GEMM4 epilogue (CUDA IPC, NVLink)"
                                      if gather == "p2p" else "by NCCL")) if ws > 1 else "single GPU",
                   "l2": "inputs larger than L2 (L, psi, R >= 1 GB each): no flush"},
        "pct_fp64_tc_peak": value / FP64_PEAK_TFLOPS * 100, "fp64_peak_tflops": FP64_PEAK_TFLOPS,
        "pct_fp64_tc_peak_note": ("algorithmic fp64 flops per second over the native FP64 tensor-core (DMMA) "
                                  "peak; with the Ozaki algorithm this is the emulation's gain over native "
                                  "FP64, not a fraction of an executing unit (that is roofline.frac)"),
        "native_fp64_dmma": ({"value": alt["value"], "unit": UNIT, "pct_fp64_tc_peak": alt["pct_fp64_tc_peak"],
                              "algorithm": alt["algorithm"]} if alt else None),
        "ozaki_guard": guard,
        "clocks": clocks, "e2e": e2e, "gpu_launches": launches, "roofline": roofline,
        "cpu_baseline": cpu, "parity": parity,
        "profile": dict(prof, steps=prof_steps, ms_total=t_prof * 1e3,
                        note="separate profiled steps (CUDA events around each launch), not the timed region"),
    }
    print(json.dumps(line), flush=True)
    ctx.close()
    if ws > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def run_oracle_configs():
    """SURVEY 8(d) "CPU oracle timed beside it": the oracle on the host cores
    for configs 1-3, single-threaded and with every host thread (config 1:
    the full 10-site norm chain; configs 2 and 3: sampled output rows, time
    per row x rows = the extrapolated full time, labelled as such). One JSON
    line; not part of the timed GPU contract."""
    import oracle
    oracle.build()
    nthreads = oracle.max_threads()
    res = {"kind": "oracle", "cpu_model": cpu_model(), "host_cpus": os.cpu_count(), "threads_all": nthreads}
    sites = synth.mps_sites(synth.MPS_BONDS_CFG1, 2, 1)
    for th, key in ((1, "1_thread"), (nthreads, "all_threads")):
        t0 = time.perf_counter()
        for _ in range(20):
            oracle.mps_norm2(sites, threads=th)
        res.setdefault("cfg1_mps_norm_chain_us", {})[key] = (time.perf_counter() - t0) / 20 * 1e6
    cfg = synth.HEFF_CONFIGS["cfg2_heisenberg_chi1024"]
    inp = {k: v.numpy() for k, v in synth.heff_inputs(cfg["chi"], cfg["d"], cfg["D"], cfg["dtype"], cfg["seed"],
                                                       cfg["model"]).items()}
    rows = [0, 511, 1023]
    for th, key in ((1, "1_thread"), (nthreads, "all_threads")):
        t0 = time.perf_counter()
        oracle.heff_rows(inp["L"], inp["W1"], inp["W2"], inp["R"], inp["psi"], rows, threads=th)
        t = (time.perf_counter() - t0) / len(rows) * cfg["chi"]
        res.setdefault("cfg2_heff_chi1024_s_extrapolated", {})[key] = t
    tc = synth.TEBD_CONFIG
    ti = synth.tebd_inputs(tc["chi"], tc["d"], tc["dtype"], tc["seed"], tc["tau"])
    A, B, U = ti["A"].numpy(), ti["B"].numpy(), ti["U"].numpy()
    arows = [0, 1]
    for th, key in ((1, "1_thread"), (nthreads, "all_threads")):
        t0 = time.perf_counter()
        oracle.tebd_theta(np.ascontiguousarray(A[arows]), B, U, threads=th)
        t = (time.perf_counter() - t0) / len(arows) * tc["chi"]
        res.setdefault("cfg3_tebd_chi2048_s_extrapolated", {})[key] = t
    res["note"] = ("configs 2-3: rows of the output timed and scaled by chi (extrapolated full time); "
                   "config 1: the whole chain")
    print(json.dumps(res), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["tci", "reference"], default="tci")
    ap.add_argument("--config", choices=list(CONFIGS), default="target")
    ap.add_argument("--gather", choices=["p2p", "nccl"], default="p2p",
                    help="N > 1: all-gather of the output slabs over peer memory (fused into the GEMM4 "
                         "epilogue) or by ncclAllGather")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-pipeline", action="store_true",
                    help="report the single-call e2e instead of a stream of applies")
    ap.add_argument("--no-staged-fill", action="store_true",
                    help="streaming e2e: copy the first step's inputs in whole before its compute")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=15.0)
    ap.add_argument("--ref-rows", type=int, default=4)
    ap.add_argument("--algo", choices=["dmma3m", "dmma4m", "ozaki"], default="ozaki",
                    help="complex128 GEMM algorithm of the timed apply (DESIGN.md §12)")
    ap.add_argument("--alt", default="dmma3m",
                    help="also time this algorithm (reported under 'alt'; 'none' to skip)")
    ap.add_argument("--oracle-configs", action="store_true",
                    help="time the CPU oracle on configs 1-3 (1 thread and all threads) and exit")
    args = ap.parse_args()
    if args.oracle_configs:
        run_oracle_configs()
        return
    if args.impl == "reference":
        run_reference(args)
    else:
        run_tci(args)


if __name__ == "__main__":
    main()
