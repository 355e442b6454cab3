#!/usr/bin/env python
"""Summarise ncu output brought back in gpurun_out/ into profiles/ (tracked).

    python tools/ncu_summary.py --cfg target --round r01

Reads gpurun_out/launches_<cfg>.csv (launch list: per-launch duration and
DRAM bytes, --clock-control none, cold-cache and serialised) and the
--set full reports prof_gemm_<cfg>.ncu-rep / prof_skinny_<cfg>.ncu-rep, writes
profiles/<round>_ncu_<cfg>.json and updates profiles/ncu_traffic.json (the
per-launch DRAM traffic bench.py reports as roofline.traffic).
"""
import argparse
import csv
import io
import json
import os
import subprocess
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
    "sm__ops_path_tensor_src_fp64.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__cycles_elapsed.avg.per_second",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "lts__t_sector_hit_rate.pct",
    "smsp__inst_executed.sum", "launch__shared_mem_per_block_dynamic",
]


def launches(cfg):
    p = os.path.join(OUT, f"launches_{cfg}.csv")
    if not os.path.exists(p):
        return None
    txt = open(p).read()
    i = txt.find('"ID"')
    rows = list(csv.DictReader(io.StringIO(txt[i:])))
    per = defaultdict(lambda: defaultdict(float))
    for r in rows:
        name = r["Kernel Name"].split("(")[0].split("<")[0].replace("void ", "").strip()
        full = r["Kernel Name"]
        if "Cfg<" in full:
            name += "<" + full.split("Cfg<")[1].split(">")[0] + ">"
        if "cutlass" in full:
            name = "cutlass_int8_gemm (Ozaki residue products)"
        m, v, u = r["Metric Name"], r["Metric Value"], r["Metric Unit"]
        try:
            v = float(v.replace(",", ""))
        except ValueError:
            continue
        scale = {"ms": 1e-3, "us": 1e-6, "usecond": 1e-6, "msecond": 1e-3, "nsecond": 1e-9, "ns": 1e-9,
                 "second": 1.0, "s": 1.0, "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9,
                 "KB": 1e3, "MB": 1e6, "GB": 1e9}.get(u, 1.0)
        key = (r["ID"], name)
        per[key][m] = v * scale
    agg = defaultdict(lambda: {"launches": 0, "time_s": 0.0, "dram_bytes": 0.0})
    for (lid, name), ms in per.items():
        a = agg[name]
        a["launches"] += 1
        a["time_s"] += ms.get("gpu__time_duration.sum", 0.0)
        a["dram_bytes"] += ms.get("dram__bytes_read.sum", 0.0) + ms.get("dram__bytes_write.sum", 0.0)
    tot = sum(a["time_s"] for a in agg.values())
    for a in agg.values():
        a["share_of_time"] = a["time_s"] / tot if tot else None
        a["dram_bytes_per_launch"] = a["dram_bytes"] / max(1, a["launches"])
    return dict(agg)


def report(path):
    if not os.path.exists(path):
        return None
    txt = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    if len(rows) < 3:
        return None
    h, units = rows[0], rows[1]
    res = []
    for v in rows[2:]:
        d = {"kernel": v[h.index("Kernel Name")][:160]}
        for k in KEYS:
            if k in h:
                i = h.index(k)
                d[k] = f"{v[i]} {units[i]}".strip()
        stalls = {}
        for i, n in enumerate(h):
            if n.startswith("smsp__pcsamp_warps_issue_stalled_") and not n.endswith("not_issued"):
                try:
                    stalls[n.replace("smsp__pcsamp_warps_issue_stalled_", "")] = float(v[i])
                except ValueError:
                    pass
        tot = sum(stalls.values()) or 1.0
        d["stall_pct_top"] = {k: round(100 * x / tot, 1) for k, x in sorted(stalls.items(), key=lambda t: -t[1])[:8]}
        res.append(d)
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg", default="target")
    ap.add_argument("--round", default="r01")
    a = ap.parse_args()
    summ = {"cfg": a.cfg, "launch_list": launches(a.cfg),
            "gemm_full": report(os.path.join(OUT, f"prof_gemm_{a.cfg}.ncu-rep")),
            "skinny_full": report(os.path.join(OUT, f"prof_skinny_{a.cfg}.ncu-rep")),
            "aux_full": report(os.path.join(OUT, f"prof_aux_{a.cfg}.ncu-rep")),
            "note": "launch_list: ncu --metrics gpu__time_duration.sum,dram__bytes_* --clock-control none "
                    "(cold-cache, serialised: compare shares); *_full: ncu --set full --clock-control none"}
    os.makedirs(PROF, exist_ok=True)
    out = os.path.join(PROF, f"{a.round}_ncu_{a.cfg}.json")
    json.dump(summ, open(out, "w"), indent=1)
    # traffic per GEMM launch from the full capture (the bench roofline's "traffic")
    g = summ["gemm_full"]
    if g:
        tr = []
        for d in g:
            try:
                rd = float(d["dram__bytes_read.sum"].split()[0]) * (1e9 if "Gbyte" in d["dram__bytes_read.sum"] else 1e6 if "Mbyte" in d["dram__bytes_read.sum"] else 1)
                wr = float(d["dram__bytes_write.sum"].split()[0]) * (1e9 if "Gbyte" in d["dram__bytes_write.sum"] else 1e6 if "Mbyte" in d["dram__bytes_write.sum"] else 1)
                if rd == rd and wr == wr:   # skip NaN captures
                    tr.append(rd + wr)
            except (KeyError, ValueError):
                pass
        if tr:
            tp = os.path.join(PROF, "ncu_traffic.json")
            cur = json.load(open(tp)) if os.path.exists(tp) else {}
            wl = {"target": "target_heisenberg_chi4096", "cfg2": "cfg2_heisenberg_chi1024",
                  "cfg4": "cfg4_hubbard_chi4096",
                  "target_ozaki": "target_heisenberg_chi4096_ozaki"}[a.cfg]
            cur[wl] = {"gemm_dram_bytes_per_launch": sum(tr) / len(tr), "per_launch": tr,
                       "source": os.path.basename(out), "round": a.round}
            json.dump(cur, open(tp, "w"), indent=1)
    print(json.dumps(summ, indent=1)[:4000])


if __name__ == "__main__":
    main()
