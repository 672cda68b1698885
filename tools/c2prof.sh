out=gpurun_out
C2="--labels 131073 --batch 512 --fmt bf16"
[ -n "$SKIP_LIST" ] || timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none \
  --csv --log-file $out/c2_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --e2e-steps 1 --ref-steps 0 $C2 > /dev/null 2>&1
python tools/launch_summary.py $out/c2_launches.csv > $out/c2_launches.txt
[ -n "$SKIP_LIST" ] || timeout 300 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none \
  --csv --log-file $out/c4b512_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --e2e-steps 1 --ref-steps 0 --batch 512 > /dev/null 2>&1
python tools/launch_summary.py $out/c4b512_launches.csv > $out/c4b512_launches.txt
for sel in "gx:6" "up:7"; do
  t=${sel%%:*}; k=${sel#*:}
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:xmc_bwd_kernel --launch-skip $k -c 1 \
    -f -o $out/prof_c2$t python bench.py --steps 1 --warmup 3 --no-cpu --e2e-steps 1 --ref-steps 0 $C2 > $out/ncu_c2$t.log 2>&1
  python tools/ncu_summary.py $out/prof_c2$t.ncu-rep --flops 1 --json $out/ncu_c2$t.json > /dev/null
  python tools/ncu_hot_sass.py $out/prof_c2$t.ncu-rep 30 > $out/ncu_c2${t}_hot.txt 2>&1
done
ls -la $out | tail
