#!/bin/bash
# compute-sanitizer tier: memcheck, racecheck, synccheck over
# every kernel of the path at small shapes (tools/sanitize_cases.py).
# Usage (GPU box): bash tools/run_sanitize.sh [outdir] [case ...]
out=${1:-gpurun_out/sanitize}; shift
mkdir -p "$out"
cases=${@:-$(python -c "import sys; sys.path.insert(0,'tools'); import sanitize_cases as s; print(' '.join(s.CASES))")}
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck; do
  for c in $cases; do
    timeout 600 $CS --tool $tool --error-exitcode 9 --print-limit 20 \
        python tools/sanitize_cases.py $c > "$out/${tool}_${c}.log" 2>&1
    echo "$tool $c rc=$?" | tee -a "$out/summary.txt"
  done
done
