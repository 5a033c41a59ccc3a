#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck / initcheck over smoke() (tiny config, BASELINE configs[0])
# and one ragged mid-size parity geometry. Summaries go to gpurun_out/sanitize_*.txt.
set -u
OUT=${1:-gpurun_out}
mkdir -p "$OUT"
CS=/usr/local/cuda/bin/compute-sanitizer
PY="import __graft_entry__ as g; g.smoke(); print('smoke ok')"
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 $CS --tool $tool --print-limit 50 --error-exitcode 9 python -c "$PY" > "$OUT/sanitize_$tool.txt" 2>&1
  echo "$tool exit=$?" >> "$OUT/sanitize_summary.txt"
done
timeout 900 $CS --tool memcheck --print-limit 50 --error-exitcode 9 python tools/profiling/sanitize_mid.py > "$OUT/sanitize_memcheck_mid.txt" 2>&1
echo "memcheck_mid exit=$?" >> "$OUT/sanitize_summary.txt"
timeout 900 $CS --tool racecheck --print-limit 50 --error-exitcode 9 python tools/profiling/sanitize_mid.py > "$OUT/sanitize_racecheck_mid.txt" 2>&1
echo "racecheck_mid exit=$?" >> "$OUT/sanitize_summary.txt"
