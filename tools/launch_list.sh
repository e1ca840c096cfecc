#!/bin/bash
# Per-kernel durations (ncu launch list, serialized, --clock-control none) of one
# window per config: where the window's time goes kernel by kernel.
# usage: tools/launch_list.sh TAG [configs...]
TAG=${1:-r2}; shift
OUT=gpurun_out/$TAG; mkdir -p $OUT
for c in ${@:-c1 c2}; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/launches_$c.csv python tools/stage_profile.py --config $c --steps 1 \
    > $OUT/launches_$c.log 2>&1
done
