#!/bin/bash
# Validates tools/plan_search.py plans on one B200: the N = 8 step predicted
# from MEASURED op durations (bench.py's `predicted`) for the manual, greedy
# (Algorithm 1) and searched plans at T = 1024 / 2048 / 4096 tokens per GPU.
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-fused-leg --no-gemm-comparison --no-e2e --no-variants --emulate"
for T in 1024 2048 4096; do
  for v in "manual:--plan manual" "greedy:--plan greedy" "search:--plan-file profiles/r01_plan_search_T$T.json"; do
    name=${v%%:*}; flags=${v#*:}
    timeout 600 $B --tokens $T --predict-tokens $T $flags > gpurun_out/psv_${name}_T$T.json 2> gpurun_out/psv_${name}_T$T.err
    python -c "
import json; d=json.loads(open('gpurun_out/psv_${name}_T$T.json').read().strip().splitlines()[-1]); p=d['predicted']
print(json.dumps({'T': $T, 'plan': '$name', 'buckets': [d['config']['buckets_fwd'], d['config']['buckets_bwd']], 'total_ms': p['total_ms'], 'exposed_ms': p['exposed_ms'], 'memory_model_peak_GiB': p['memory_model_peak_GiB'], 'emulated_step_ms': (d.get('emulated') or {}).get('step_ms'), 'emulated_exposed_ms': (d.get('emulated') or {}).get('exposed_ms')}))"
  done
done
