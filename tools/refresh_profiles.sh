#!/usr/bin/env bash
# On the GPU box (under gpurun): bench line, reference-arm line, launch list and
# one `ncu --set full` capture of each head kernel.  Outputs in gpurun_out/.
#   gpurun --timeout 1500 -- tools/refresh_profiles.sh [tag]
set -u
tag=${1:-r1}
out=gpurun_out
mkdir -p $out
timeout 600 python bench.py > $out/bench_$tag.json 2> $out/bench_$tag.err
timeout 300 python bench.py --impl reference > $out/bench_ref_$tag.json 2> $out/bench_ref_$tag.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file $out/launches_$tag.csv python bench.py --steps 2 --warmup 3 --no-cpu --e2e-steps 1 > /dev/null 2>&1
for k in fwd bwd; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:xmc_${k}_kernel --launch-skip 4 -c 1 \
    -f -o $out/prof_${k}_$tag python bench.py --steps 1 --warmup 3 --no-cpu --e2e-steps 1 > $out/ncu_${k}_$tag.log 2>&1
done
tail -1 $out/bench_$tag.json
tail -1 $out/bench_ref_$tag.json
timeout 300 python bench.py --steps 1000 --no-cpu --e2e-steps 2 > $out/bench_sustained_$tag.json 2>/dev/null
timeout 300 python tools/bench_topk.py > $out/topk_$tag.json 2>/dev/null
timeout 300 ncu --set full --clock-control none --import-source on -k regex:xmc_fwd_kernel -c 1 -f \
  -o $out/prof_topk_$tag python tools/bench_topk.py --iters 1 > /dev/null 2>&1
