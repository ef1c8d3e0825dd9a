#!/bin/bash
# ncu --set full capture of one FlashSign launch per listed config -> gpurun_out/$TAG/prof_<cfg>.ncu-rep
#   gpurun --timeout 1200 -- 'bash tests/profile_full.sh r1b c2 c4'
TAG=$1; shift
OUT=gpurun_out/$TAG
mkdir -p $OUT
for c in "$@"; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:flashsign -s 3 -c 1 -o $OUT/prof_$c \
    python bench.py --config $c --steps 1 --warmup 3 --no-e2e --no-cpu > $OUT/ncu_$c.log 2>&1
  tail -3 $OUT/ncu_$c.log
done
ls -la $OUT
