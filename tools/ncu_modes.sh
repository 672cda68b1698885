#!/usr/bin/env bash
# ncu --set full summaries of the backward in the other modes (C4, one chunk launch each)
out=gpurun_out; mkdir -p $out
fl=$(python -c "print(4*256*1406141*768)")
for cfg in "ref:--precision reference:8192" "bf16g:--g-format bf16:8192" "kahan10:--kahan bf16 --kahan-labels 281228:16384" "kahanall:--kahan bf16:16384"; do
  tag=${cfg%%:*}; rest=${cfg#*:}; args=${rest%:*}; pc=${rest##*:}
  timeout 600 ncu --set full --clock-control none -k regex:xmc_bwd_kernel --launch-skip 4 -c 1 -f -o $out/prof_$tag \
    python bench.py --steps 1 --warmup 3 --no-cpu --e2e-steps 1 --ref-steps 0 --bf16g-steps 0 $args > /dev/null 2>&1
  python tools/ncu_summary.py $out/prof_$tag.ncu-rep --flops $fl --per-clk $pc --json $out/ncu_bwd_$tag.json > /dev/null
  rm -f $out/prof_$tag.ncu-rep
  python -c "import json; d=json.load(open('$out/ncu_bwd_$tag.json'))[0]; print('$tag', {k: d.get(k) for k in ('kernel','duration_us','sm_clock_mhz','tensor_pipe_pct','flop_derived_tensor_pct','dram_TBps','top_stalls_pct')})"
done
