#!/usr/bin/env bash
# Alternate bench runs over values of one environment knob on the same box.
#   tools/ab_env.sh VAR "v1 v2 ..." rounds [extra bench args]
var=${1:?var}; vals=${2:?values}; rounds=${3:-1}; shift 3 || true
for r in $(seq "$rounds"); do
  for v in $vals; do
    env "$var=$v" timeout 180 python bench.py --steps 20 --warmup 5 --no-cpu --e2e-steps 2 --ref-steps 0 "$@" 2>&1 | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$var=$v', round(d['value']), round(d['ms_per_step'],4), {k: round(v,4) for k,v in d['roofline']['step_kernel_ms'].items()}, d['clocks'].get('kernel_mhz'))"
  done
done
