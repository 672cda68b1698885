#!/usr/bin/env bash
# Alternate bench runs of several in-tree library builds on the same box.
#   tools/ab_bench.sh "base cur" [rounds] [extra bench args]
libs=${1:?tags}; rounds=${2:-2}; shift 2 || true
for r in $(seq "$rounds"); do
  for t in $libs; do
    XMC_LIB_PATH=paper_2510_11168_b200/libxmc_b200_$t.so timeout 180 python bench.py --steps 20 --warmup 5 --no-cpu --e2e-steps 2 "$@" 2>&1 | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$t', round(d['value']), round(d['ms_per_step'],4), {k: round(v,4) for k,v in d['roofline']['step_kernel_ms'].items()}, d['clocks'].get('kernel_mhz'), d['clocks'].get('sm_mhz'))"
  done
done
