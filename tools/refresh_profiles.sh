#!/usr/bin/env bash
# On the GPU box (under gpurun): bench line, reference-arm line, sustained
# line, launch list and one `ncu --set full` capture of each head kernel, the
# streaming top-k bench and the other BASELINE configs.  Outputs in gpurun_out/.
#   gpurun --timeout 2400 -- tools/refresh_profiles.sh [tag]
set -u
tag=${1:-r2}
out=gpurun_out
mkdir -p $out
timeout 600 python bench.py > $out/bench_$tag.json 2> $out/bench_$tag.err
timeout 300 python bench.py --impl reference > $out/bench_ref_$tag.json 2> $out/bench_ref_$tag.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file $out/launches_$tag.csv python bench.py --steps 2 --warmup 3 --no-cpu --e2e-steps 1 --ref-steps 1 > /dev/null 2>&1
python tools/launch_summary.py $out/launches_$tag.csv > $out/launches_$tag.txt
# per kernel: summary (exact ncu metric names, flop-derived tensor %), hot SASS
# and instruction mix; only the bwd report is kept (gpurun copies back <= 64 MiB)
flops_fwd=$(python -c "print(2*256*1406141*768)"); flops_bwd=$(python -c "print(4*256*1406141*768)")
for k in fwd bwd; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:xmc_${k}_kernel --launch-skip 4 -c 1 \
    -f -o $out/prof_${k}_$tag python bench.py --steps 1 --warmup 3 --no-cpu --e2e-steps 1 --ref-steps 0 > $out/ncu_${k}_$tag.log 2>&1
  fl=$([ $k = fwd ] && echo $flops_fwd || echo $flops_bwd)
  python tools/ncu_summary.py $out/prof_${k}_$tag.ncu-rep --flops $fl --json $out/ncu_${k}_$tag.json > /dev/null
  python tools/ncu_hot_sass.py $out/prof_${k}_$tag.ncu-rep 40 > $out/ncu_${k}_hot_sass_$tag.txt 2>&1
  python tools/sass_mix.py $out/prof_${k}_$tag.ncu-rep $(python -c "print(1406141*768)") 40 > $out/ncu_${k}_sass_mix_$tag.txt 2>&1
  [ $k = fwd ] && rm -f $out/prof_${k}_$tag.ncu-rep
done
tail -1 $out/bench_$tag.json
tail -1 $out/bench_ref_$tag.json
timeout 300 python bench.py --steps 1000 --no-cpu --e2e-steps 2 --ref-steps 0 > $out/bench_sustained_$tag.json 2>/dev/null
timeout 300 python tools/bench_topk.py > $out/topk_$tag.json 2>/dev/null
timeout 300 ncu --set full --clock-control none --import-source on -k regex:xmc_fwd_kernel --launch-skip 1 -c 1 -f \
  -o $out/prof_topk_$tag python tools/bench_topk.py --iters 1 > /dev/null 2>&1
python tools/ncu_summary.py $out/prof_topk_$tag.ncu-rep --flops $(python -c "print(2*256*2812281*768)") --json $out/ncu_topk_$tag.json > /dev/null
rm -f $out/prof_topk_$tag.ncu-rep
for cfg in "c2:--labels 131073 --batch 512 --fmt bf16" "c3:--labels 670091" "c5r0:--labels 1077981 --batch 128" "c4b512:--batch 512" "c4s8:--labels 351536" "c4kahan_top10:--kahan bf16 --kahan-labels 281228" "c4kahan_all:--kahan bf16" "c4bf16g:--g-format bf16"; do
  t=${cfg%%:*}; args=${cfg#*:}
  timeout 300 python bench.py --no-cpu --ref-steps 0 --e2e-steps 2 $args 2>/dev/null | tail -1 >> $out/configs_$tag.jsonl
done
