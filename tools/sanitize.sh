#!/usr/bin/env bash
# compute-sanitizer memcheck / racecheck / synccheck over small head steps of
# every backward flavour (GPU box; outputs in gpurun_out/sanitize_*.log)
out=gpurun_out; mkdir -p $out
cases=("3000 256 e4m3 operand 2 hash" "3000 256 e4m3 operand 1 splitmix64" "3000 256 e4m3 reference 2 hash"
       "3000 256 bf16 operand 2 hash" "3000 512 bf16 operand 1 hash" "3000 512 e4m3 operand 1 hash")
for tool in memcheck racecheck synccheck; do
  : > $out/sanitize_$tool.log
  for c in "${cases[@]}"; do
    echo "== $c" >> $out/sanitize_$tool.log
    timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/repro_step.py $c >> $out/sanitize_$tool.log 2>&1
    echo "rc=$?" >> $out/sanitize_$tool.log
  done
  grep -E "ERROR SUMMARY|RACECHECK SUMMARY|rc=|^== " $out/sanitize_$tool.log
done
