#!/bin/bash
# Emulated weak scaling on one B200: the per-block Llama-3-8B rank step at
# layout world N = 2 / 4 / 8 with the compute proxy at T = 1024 and the
# collectives emulated (K11 for NCCL + copy kernels, paced K8 / K9 for the
# fused path).  One JSON line per (N, collective).  MODEL OUTPUTS: the links
# are assumed (720 GB/s busbw, 20 us), not measured.
B="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-fused-leg --no-e2e --no-variants --predict-tokens 1024 --emulate"
for N in 2 4 8; do
  for c in nccl p2p; do
    timeout 600 $B --sim-world $N --collective $c > gpurun_out/es_${c}_$N.json 2> gpurun_out/es_${c}_$N.err
    python -c "
import json; d=json.loads(open('gpurun_out/es_${c}_$N.json').read().strip().splitlines()[-1]); e=d['emulated']
print(json.dumps({'N': $N, 'collective': '$c', 'emulated_step_ms': e['step_ms'], 'compute_only_ms': e['compute_only_ms'], 'exposed_ms': e['exposed_ms'], 'kind': e['kind']}))"
  done
done
