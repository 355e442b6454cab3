#!/usr/bin/env python
"""One-kernel summary of an `ncu --set full` report (gpurun_out/*.ncu-rep) for
profiles/: duration, throughputs, occupancy, DRAM traffic, the top stall
reasons and the stall samples per SASS opcode.

    python tools/ncu_kernel_summary.py gpurun_out/prof_svd_round.ncu-rep profiles/r01_ncu_svd_round.json
"""
import collections
import csv
import io
import json
import re
import subprocess
import sys

METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "dram__throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__grid_size", "launch__cluster_dim_x",
           "launch__registers_per_thread", "lts__t_sector_hit_rate.pct"]


def ncu_csv(rep, *args):
    out = subprocess.run(["ncu", "-i", rep, *args, "--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def main(rep, dst):
    rows = ncu_csv(rep, "--page", "raw")
    hdr, units, vals = rows[0], rows[1], rows[2]
    raw = dict(zip(hdr, vals))
    unit = dict(zip(hdr, units))
    res = {"report": rep, "kernel": raw.get("Kernel Name", "")[:160], "metrics": {},
           "units": {m: unit.get(m, "") for m in METRICS if m in raw}}
    for m in METRICS:
        if m in raw:
            try:
                res["metrics"][m] = float(raw[m].replace(",", ""))
            except ValueError:
                res["metrics"][m] = raw[m]
    st = {h.replace("smsp__pcsamp_warps_issue_stalled_", ""): float(v) for h, v in raw.items()
          if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued") and v and
          v.replace(".", "", 1).isdigit()}
    tot = sum(st.values()) or 1.0
    res["stall_share"] = {k: round(v / tot, 4) for k, v in sorted(st.items(), key=lambda x: -x[1])[:8]}
    sass = ncu_csv(rep, "--page", "source", "--print-source", "sass")
    h = sass[1]
    si, wi = h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
    op = collections.Counter()
    for r in sass[2:]:
        try:
            w = int(r[wi])
        except (ValueError, IndexError):
            continue
        m = re.match(r"(@!?U?P\w+\s+)?([A-Z0-9_]+)", r[si].strip())
        op[m.group(2) if m else "?"] += w
    t = sum(op.values()) or 1
    res["samples_by_opcode"] = {k: round(v / t, 4) for k, v in op.most_common(12)}
    json.dump(res, open(dst, "w"), indent=1)
    print(json.dumps(res, indent=1)[:2000])


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
