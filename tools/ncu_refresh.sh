#!/bin/bash
# Refreshes the committed ncu evidence for the current build (run on the B200 via gpurun).
#   1. launch list of the default bench command (cold, serialised per-launch times)
#   2. --set full of K3 / K4 / K6 inside the bench step (8B block buckets, N = 8)
#   3. --set full of K8 / K9 inside the p2p bench step
#   4. --set full of K1 (fp32 master rounding) and K6 (accumulate) from tools/pack_probe.py
set -u
O=gpurun_out/ncu
mkdir -p $O
B="bench.py --steps 2 --warmup 1 --quick --no-e2e"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file $O/launches.csv python bench.py > $O/launches_bench.log 2>&1
echo "launch list rc=$?"
for k in fsdp_ag_unpack_kernel fsdp_rs_pack_kernel fsdp_rs_copyout_kernel; do
  # skip the first launches (warm-up step's small buckets) and capture 2 block-sized ones
  timeout 900 ncu --set full --clock-control none --import-source on -k $k -s 4 -c 2 -o $O/full_$k python $B > $O/full_$k.log 2>&1
  echo "$k rc=$?"
done
P="bench.py --collective p2p --steps 1 --warmup 1 --quick --no-e2e"
for k in fsdp_p2p_allgather_kernel fsdp_p2p_reduce_scatter_kernel; do
  timeout 900 ncu --set full --clock-control none --import-source on -k $k -s 4 -c 2 -o $O/full_$k python $P > $O/full_$k.log 2>&1
  echo "$k rc=$?"
done
# pack_probe.py launch order: K1 direct x23, K1 pack x23, then K1 master; K6 copy x23, then K6 accumulate
timeout 900 ncu --set full --clock-control none --import-source on -k fsdp_ag_pack_kernel -s 50 -c 2 -o $O/full_k1_master python tools/pack_probe.py > $O/full_k1_master.log 2>&1
echo "k1 master rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k fsdp_rs_copyout_kernel -s 30 -c 2 -o $O/full_k6_accum python tools/pack_probe.py > $O/full_k6_accum.log 2>&1
echo "k6 accum rc=$?"
ls -la $O
