#!/bin/bash
# ncu evidence for one round (run under gpurun; one GPU).  Usage: tools/profile_round.sh r02
set -u
R=${1:-r02}
O=gpurun_out/prof_$R
mkdir -p $O
B="python bench.py --steps 5 --warmup 3 --no-cpu-baseline"
# launch lists (cold-cache, serialised: compare shares, not absolutes)
for c in cfg5 cfg4b1 cfg2 cfg3; do
  $B --config $c > $O/plain_$c.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
      --log-file $O/launches_$c.csv $B --config $c > /dev/null 2>&1
done
# full captures of the dominant kernels
full() {  # config kernel-regex name
  $B --config $1 > /dev/null 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:$2 -s 2 -c 1 \
      -o $O/full_$3 $B --config $1 > /dev/null 2>&1
}
full cfg5 rb_tmem cfg5_rb_tmem16
full cfg3 rb_tmem cfg3_rb_tmem8
full cfg4b1 lane_lut cfg4b1_lane_lut
full cfg4b1 dq_hmma cfg4b1_dq_hmma
full cfg5 dq_hmma cfg5_dq_hmma
full cfg4b256 dq_mma cfg4b256_dq_mma
ls -la $O
