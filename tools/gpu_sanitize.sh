#!/bin/bash
# compute-sanitizer (memcheck, racecheck, synccheck) over tools/sanitize_cases.py, one case per run.
mkdir -p gpurun_out/sanitizer
S=/usr/local/cuda/bin/compute-sanitizer
run() {  # tool case [extra]
  timeout 900 $S --tool $1 $3 --print-limit 20 python tools/sanitize_cases.py $2 > gpurun_out/sanitizer/$1_$2.log 2>&1
  echo "$1 $2 rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|case ' gpurun_out/sanitizer/$1_$2.log | tr '\n' ' ')"
}
for c in heff tebd lanczos svd ozaki ozaki_real f32 gather; do run memcheck $c; done
for c in heff svd ozaki gather; do run racecheck $c "--racecheck-report all"; done
for c in heff svd ozaki gather; do run synccheck $c; done
for c in ozaki svd; do run initcheck $c; done
