#!/usr/bin/env bash
# The other BASELINE shapes and modes with the in-tree library, one JSON line each.
#   tools/configs_sweep.sh > gpurun_out/configs.jsonl
for cfg in "c2:--labels 131073 --batch 512 --fmt bf16" "c3:--labels 670091" "c5r0:--labels 1077981 --batch 128" \
           "c4b512:--batch 512" "c4s8:--labels 351536" "c4kahan_top10:--kahan bf16 --kahan-labels 281228" \
           "c4kahan_all:--kahan bf16" "c4bf16g:--g-format bf16" "c4ref:--precision reference" \
           "bf16_131k_b256:--labels 131073 --fmt bf16" "bf16_2p8m_b256:--fmt bf16"; do
  t=${cfg%%:*}; args=${cfg#*:}
  timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --ref-steps 0 --bf16g-steps 0 --e2e-steps 2 $args 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); d['tag']='$t'; print(json.dumps(d))"
done
