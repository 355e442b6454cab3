#!/usr/bin/env python
"""Per-opcode executed-instruction and stall-sample totals from an ncu
`--page source --print-source sass --csv` export (tools/gpu_r02_ncu.sh).

    python tools/sass_profile.py gpurun_out/ncu_crt_g_sass.csv [--top 25] [--hot 30]
"""
import collections
import csv
import re
import sys


def main(path, top=25, hot=0):
    rows = list(csv.reader(open(path)))
    k = next(i for i, r in enumerate(rows) if "Source" in r)
    h, rows = rows[k], rows[k:]
    i_src, i_ex, i_st = h.index("Source"), h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
    ex, st = collections.Counter(), collections.Counter()
    lines = []
    for r in rows[1:]:
        try:
            e = int(r[i_ex] or 0)
            s = int(r[i_st] or 0)
        except (ValueError, IndexError):
            continue
        m = re.match(r"(@!?U?P\w+\s+)?([A-Z0-9_]+)", r[i_src].strip())
        op = m.group(2) if m else "?"
        ex[op] += e
        st[op] += s
        lines.append((s, e, r[0], r[i_src].strip()[:90]))
    te, ts = sum(ex.values()) or 1, sum(st.values()) or 1
    print(f"total warp instructions {te:.4g}, stall samples {ts}")
    for op, e in ex.most_common(top):
        print(f"  {op:12s} exec {e / te:6.1%}   stall {st[op] / ts:6.1%}")
    if hot:
        print("hottest lines by stall samples:")
        for s, e, a, src in sorted(lines, reverse=True)[:hot]:
            print(f"  {s:7d} {e:10d} {a} {src}")


if __name__ == "__main__":
    a = sys.argv
    main(a[1], int(a[a.index("--top") + 1]) if "--top" in a else 25, int(a[a.index("--hot") + 1]) if "--hot" in a else 0)
