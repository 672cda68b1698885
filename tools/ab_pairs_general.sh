for r in 1 2; do for cfg in "c2:--labels 131073 --batch 512 --fmt bf16" "c4b512:--batch 512" "c4ref:--precision reference" "bf16_2p8m:--fmt bf16"; do
  t=${cfg%%:*}; args=${cfg#*:}
  for l in base cur; do
    XMC_LIB_PATH=paper_2510_11168_b200/libxmc_b200_$l.so timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --ref-steps 0 --bf16g-steps 0 --e2e-steps 2 $args 2>/dev/null | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$l', '$t', round(d['value']), round(d['ms_per_step'],4), {k: round(v,4) for k,v in d['roofline']['step_kernel_ms'].items()})"
  done; done; done
