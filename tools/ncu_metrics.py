"""Print selected raw metrics of an ncu report (usage: ncu_metrics.py report.ncu-rep [substr ...])."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
keys = sys.argv[2:] or ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
                        "sm__pipe_tensor_subpipe_imma_cycles_active", "sm__cycles_elapsed.avg.per_second",
                        "lts__throughput.avg.pct", "l1tex__m_xbar2l1tex_read_bytes.sum", "sm__throughput.avg.pct",
                        "launch__registers", "smsp__warp_issue_stalled", "lts__t_sectors_srcunit_tex_op_read_lookup_miss",
                        "lts__average_gcomp", "sm__inst_executed_pipe_tensor", "gpc__cycles_elapsed.max"]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, units = rows[0], rows[1]
for row in rows[2:]:
    print("kernel:", row[hdr.index("Kernel Name")][:80] if "Kernel Name" in hdr else "?")
    for i, k in enumerate(hdr):
        if any(s in k for s in keys):
            print(f"  {k} = {row[i]} {units[i]}")
