#!/bin/bash
# Multi-GPU measurement plan (one node, NVSwitch): run when more than one
# B200 is available.  Writes JSON lines under gpurun_out/scale/.
#   1. bench.py at N = 2, 4, 8 for the NCCL flat bucketing (default), the
#      grouped all-gather, NCCL buffer registration (local / symmetric), the
#      fused peer-memory collectives (grid-capped and full grid), the searched
#      plans, keep-last, real GEMM compute and a bounded NCCL CTA count --
#      the measured counterparts of this round's emulated results;
#   2. busbw sweeps + alpha/beta fits per (op, N) for NCCL and p2p, the inputs
#      the greedy planner (Algorithm 1) needs.
# Usage: bash tools/scale_check.sh [max_gpus]
set -u
MAX=${1:-8}
O=gpurun_out/scale
mkdir -p $O
PORT=29900
run() {  # run <n> <tag> <bench args...>
  local n=$1 tag=$2
  shift 2
  timeout 1800 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port $PORT bench.py --gpus $n "$@" > $O/bench_${tag}_N$n.json 2> $O/bench_${tag}_N$n.err
  echo "N=$n $tag rc=$? $(tail -c 200 $O/bench_${tag}_N$n.json)"
  PORT=$((PORT + 1))
}
# correctness first: NCCL / K8-K9 / K10 NVLS parity on real peers (N = min(devices, 8))
timeout 3600 python -m pytest tests/test_gpu_multi.py -q -rs > $O/pytest_multi.log 2>&1
echo "pytest multi rc=$? $(tail -n 3 $O/pytest_multi.log)"
for n in 2 4 8; do
  [ $n -le $MAX ] || continue
  # the north-star comparison (BASELINE configs[2]); the default line already
  # carries parity, busbw_block, alpha_beta and the measured exposure variants
  run $n flat
  run $n p2p --collective p2p
  run $n p2p_window --collective p2p --p2p-transport window              # peers mapped by NCCL symmetric windows
  run $n vanilla --plan per_param --no-reorder --tokens 1024 --quick      # the unbucketed, unreordered baseline
  run $n perblock_T1024 --plan manual --tokens 1024 --quick               # + bucket & reorder (manual wrap)
  run $n greedy_T1024 --plan greedy --tokens 1024 --quick                 # auto-wrap (assumed links; the default
                                                                          # line's `exposure` plans with fitted ones)
  run $n grouped --ag grouped
  run $n reglocal --nccl-register local
  run $n regsym --nccl-register symmetric
  run $n p2p_fullgrid --collective p2p --p2p-max-ctas 0      # grid cap off (full GPU) vs the default cap
  run $n search --plan search                               # fsdp_plan_search (beyond Algorithm 1)
  run $n search_p2p --plan search --collective p2p
  run $n keeplast --keep-last                               # G42: no re-gather of the boundary bucket
  run $n gemm_p2p_search --compute gemm --collective p2p --plan search   # real GEMMs between the collectives
  run $n nccl_maxctas16 --nccl-max-ctas 16                  # NCCL's SM footprint bounded
  # BASELINE configs[3]: Llama-3-70B shards, bucket-size sweep 25-500 MB (size cap on the gathered bytes, G30)
  for cap in 25e6 50e6 100e6 200e6 500e6; do
    run $n 70b_cap$cap --model 70b --plan size_cap --mem-limit $cap --quick --no-e2e
  done
  # BASELINE configs[4]: one Llama-3-405B layer (d 16384, FFN 53248), per-param and one whole-layer bucket
  run $n 405b_layer --model 405b --layers 1 --quick --no-e2e
  run $n 405b_layer_pp --model 405b --layers 1 --plan per_param --quick --no-e2e
  for c in nccl p2p; do
    timeout 1800 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
      --master-port $PORT tools/busbw_sweep.py --collective $c --out $O/busbw_${c}_N$n.json > $O/busbw_${c}_N$n.log 2>&1
    echo "busbw N=$n $c rc=$?"
    PORT=$((PORT + 1))
  done
done
python tools/scale_summary.py $O > $O/scale_summary.md
echo "summary: $O/scale_summary.md"
