#!/bin/bash
# tools/plan_search.py plans for Llama-3-70B at T = 2048 vs manual, greedy and
# the best size cap of configs c3 (500 MB), timed on one B200 (predicted N = 8
# step from measured op durations).
B="python bench.py --model 70b --steps 2 --warmup 3 --no-cpu-baseline --no-fused-leg --no-gemm-comparison --no-e2e --no-variants --tokens 2048 --predict-tokens 2048 --emulate"
for v in "manual:--plan manual" "greedy:--plan greedy" "size_cap_500MB:--plan size_cap --mem-limit 5e8" "search:--plan-file profiles/r01_plan_search_70b_T2048.json"; do
  name=${v%%:*}; flags=${v#*:}
  timeout 900 $B $flags > gpurun_out/psv70_${name}.json 2> gpurun_out/psv70_${name}.err
  python -c "
import json; d=json.loads(open('gpurun_out/psv70_${name}.json').read().strip().splitlines()[-1]); p=d['predicted']
print(json.dumps({'model': '70b', 'T': 2048, 'plan': '$name', 'buckets': [d['config']['buckets_fwd'], d['config']['buckets_bwd']], 'total_ms': p['total_ms'], 'exposed_ms': p['exposed_ms'], 'memory_model_peak_GiB': p['memory_model_peak_GiB'], 'emulated_step_ms': (d.get('emulated') or {}).get('step_ms'), 'emulated_exposed_ms': (d.get('emulated') or {}).get('exposed_ms')}))"
done
