for r in 1 2; do for mode in "--precision reference" "--g-format bf16"; do for g in 2 1; do
# (the XMC_GX_GROUP override was a temporary build of xmc_api.cu for this A/B; see profiles/r2_notes.md Session 6)
XMC_GX_GROUP=$g timeout 240 python bench.py --steps 10 --warmup 3 --no-cpu --e2e-steps 2 --ref-steps 0 --bf16g-steps 0 $mode 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$mode G=$g', round(d['value']), round(d['ms_per_step'],4), {k: round(v,4) for k,v in d['roofline']['step_kernel_ms'].items()}, d['clocks'].get('kernel_mhz'))"
done; done; done
