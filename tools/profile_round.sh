#!/bin/bash
# ncu evidence for one round (run under gpurun; one GPU).  Usage: tools/profile_round.sh r01
set -u
R=${1:-r01}
O=gpurun_out/prof_$R
mkdir -p $O
B="python bench.py --steps 5 --warmup 3 --no-cpu-baseline"
# launch lists (cold-cache, serialised: compare shares, not absolutes)
for c in cfg5 cfg4b1 cfg2; do
  $B --config $c > $O/plain_$c.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
      --log-file $O/launches_$c.csv $B --config $c > /dev/null 2>&1
done
# full captures of the dominant kernels
$B --config cfg5 > $O/plain_full_cfg5.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:fused_lut -s 2 -c 1 \
    -o $O/full_cfg5_fused_lut $B --config cfg5 > /dev/null 2>&1
$B --config cfg4b1 > $O/plain_full_cfg4b1.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:lane_lut -s 2 -c 1 \
    -o $O/full_cfg4b1_lane_lut $B --config cfg4b1 > /dev/null 2>&1
$B --config cfg4b1 > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:dq_mma -s 2 -c 1 \
    -o $O/full_cfg4b1_dq_mma $B --config cfg4b1 > /dev/null 2>&1
# the comparison kernel where it is tensor-bound (b = 256)
$B --config cfg4b256 > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:dq_mma -s 2 -c 1 \
    -o $O/full_cfg4b256_dq_mma $B --config cfg4b256 > /dev/null 2>&1
ls -la $O
