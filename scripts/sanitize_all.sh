#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over scripts/sanitize_probe.py
# usage: bash scripts/sanitize_all.sh OUTFILE
OUT=${1:-gpurun_out/compute_sanitizer.txt}
mkdir -p "$(dirname "$OUT")"
: > "$OUT"
for tool in memcheck racecheck synccheck; do
  echo "=== compute-sanitizer --tool $tool" >> "$OUT"
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_probe.py >> "$OUT" 2>&1
  echo "exit $?" >> "$OUT"
done
grep -E "===|ERROR SUMMARY|RACECHECK SUMMARY|exit|bad =" "$OUT"
