#!/bin/bash
# Robustness sweep of bench.py variants on one B200 (gpurun): plans, collectives, compute modes,
# model sizes, layout worlds.  Writes gpurun_out/sw_<name>.json; summarised in profiles/r01_bench_variants.json.
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-fused-leg --no-gemm-comparison --no-e2e --predict-tokens 0"
run() { name=$1; shift; timeout 600 $B "$@" > gpurun_out/sw_$name.json 2> gpurun_out/sw_$name.err; echo "$name rc=$? $(tail -c 300 gpurun_out/sw_$name.json | grep -o '"ms_per_step": [0-9.]*' | head -1)"; }
run greedy --plan greedy --tokens 1024
run pp_noreorder --plan per_param --no-reorder
run p2p_greedy --collective p2p --plan greedy
run gemm --compute gemm --tokens 1024
run m70b --model 70b
run m405b_l2 --model 405b --layers 2
run sizecap --plan size_cap --mem-limit 1e8
run grouped --ag grouped
run simw4 --sim-world 4
run toy --model 8b --layers 1 --sim-world 3
