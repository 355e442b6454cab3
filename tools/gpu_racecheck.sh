#!/bin/bash
# racecheck with every hazard printed, summarised on the box by (kind, write site, read site)
mkdir -p gpurun_out/sanitizer
S=/usr/local/cuda/bin/compute-sanitizer
for c in svd_small ozaki gather; do
  timeout 1500 $S --tool racecheck --racecheck-report all --print-limit 0 python tools/sanitize_cases.py $c > /tmp/rc_$c.log 2>&1
  echo "racecheck $c rc=$?" | tee gpurun_out/sanitizer/racecheck_full_$c.txt
  grep -E "RACECHECK SUMMARY|case " /tmp/rc_$c.log | tee -a gpurun_out/sanitizer/racecheck_full_$c.txt
  python3 - "$c" >> gpurun_out/sanitizer/racecheck_full_$c.txt <<'PY'
import re, sys, collections
c = sys.argv[1]
t = open(f"/tmp/rc_{c}.log").read().split("========= Error:")[1:] + open(f"/tmp/rc_{c}.log").read().split("========= Warning:")[1:]
cnt = collections.Counter()
for b in t:
    kind = b.split("\n")[0].split(" at __shared__")[0].strip()
    w = re.search(r"Write Thread \(.*?\) at (.*)", b); r = re.search(r"Read Thread \(.*?\) at (.*)", b)
    cnt[(kind, w.group(1).strip()[-90:] if w else "", r.group(1).strip()[-90:] if r else "")] += 1
print("distinct hazard signatures:", len(cnt), "total", sum(cnt.values()))
for k, v in cnt.most_common(20):
    print(v, k)
PY
  cat gpurun_out/sanitizer/racecheck_full_$c.txt | tail -8
done
