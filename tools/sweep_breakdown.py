"""Per-kernel-kind breakdown (tci_profile) of selected config-5 sweep
instances (dev tool). Reproduces the instance generator of bench_extra.sweep."""
import os, sys, json
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth
import paper_2512_23917_b200 as tci
from tools.bench_extra import timed, FP64_PEAK, HBM

d = json.load(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "profiles", "r01_extra_sweep_splitk.json")))
inst = d["sweep"]["instances"]
ctx = tci.Context(0)
sel = [int(x) for x in sys.argv[1:]] or [i for i, r in enumerate(inst) if r["roofline_us"] > 20 and r["frac_of_roofline"] < 0.3]
for i in sel:
    r = inst[i]
    dims, dt = r["dims"], r["dtype"]
    A = synth.random_tensor([dims[l] for l in r["la"]], dt, 77, 1, device="cuda")
    B = synth.random_tensor([dims[l] for l in r["lb"]], dt, 77, 2, device="cuda")
    holder = {}
    f = lambda: holder.__setitem__("c", ctx.contract(A, r["la"], B, r["lb"], r["lc"], out=holder.get("c")))
    med, _ = timed(f, reps=3, warm=1)
    tci.tci_profile_enable(ctx.handle, True)
    f()
    prof = {k: tci.tci_profile_query(ctx.handle, v) for k, v in (("gemm", tci.PROF_GEMM), ("permute", tci.PROF_PERMUTE), ("skinny", tci.PROF_SKINNY))}
    tci.tci_profile_enable(ctx.handle, False)
    print(i, dt, r["la"], r["lb"], "->", r["lc"], {k: dims[k] for k in dims}, f"us={med*1e6:.0f} roof={r['roofline_us']:.0f}",
          {k: (v["launches"], round(v["ms"] * 1e3)) for k, v in prof.items()}, flush=True)
    del A, B, holder
    torch.cuda.empty_cache()
