#!/bin/bash
# One gpurun call: bench lines for every config, ncu launch lists + DRAM traffic per
# config, and one `ncu --set full` capture of the C3 kernel.  Output -> gpurun_out/$TAG/.
#   gpurun --timeout 1800 -- 'bash tests/profile_run.sh r1'
TAG=${1:-r1}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $OUT/gpu.txt
timeout 400 python bench.py --context > $OUT/bench_c3.json 2> $OUT/bench_c3.err
for c in c2 c4 c5; do
  timeout 300 python bench.py --config $c --no-cpu > $OUT/bench_$c.json 2> $OUT/bench_$c.err
done
timeout 200 python bench.py --impl reference --steps 5 --warmup 3 > $OUT/bench_reference.json 2>&1
for c in c3 c2 c4 c5; do
  timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active \
    --clock-control none -k regex:flashsign -c 3 --csv --log-file $OUT/launches_$c.csv \
    python bench.py --config $c --steps 2 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
done
for c in c3 c2; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:flashsign -s 3 -c 1 -o $OUT/prof_$c \
  python bench.py --config $c --steps 1 --warmup 3 --no-e2e --no-cpu > $OUT/ncu_$c.log 2>&1
done
tail -2 $OUT/ncu_c3.log
ls -la $OUT
