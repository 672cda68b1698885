#!/usr/bin/env bash
# Same-box A/B of library builds (tools/ab_build.sh) in the bf16-operand
# backward modes: reference precision and bf16 G (C4 shape), plus the FP8 default.
#   tools/ab_modes.sh "base cur" [rounds]
libs=${1:?tags}; rounds=${2:-2}
for r in $(seq "$rounds"); do
  for mode in "--precision reference" "--g-format bf16" ""; do
    for t in $libs; do
      XMC_LIB_PATH=paper_2510_11168_b200/libxmc_b200_$t.so timeout 240 python bench.py --steps 10 --warmup 3 --no-cpu \
        --e2e-steps 2 --ref-steps 0 --bf16g-steps 0 $mode 2>&1 | tail -1 | \
        python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$t', '${mode:-fp8}', round(d['value']), round(d['ms_per_step'],4), {k: round(v,4) for k,v in d['roofline']['step_kernel_ms'].items()}, d['clocks'].get('kernel_mhz'))"
    done
  done
done
