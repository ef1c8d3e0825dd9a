#!/bin/bash
# One gpurun call: bench lines for every config (timed regions >= 0.5 s so the NVML clock sampler
# sees >= 25 samples), the reference arm, ncu launch lists + DRAM traffic per config, and one
# `ncu --set full` capture per listed config.  Output -> gpurun_out/$TAG/.
#   gpurun --timeout 2400 -- 'bash tests/profile_run.sh r2 c3 c2 c4'
TAG=${1:-r2}; shift
FULL=${@:-c3 c2 c4}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $OUT/gpu.txt
timeout 600 python bench.py > $OUT/bench_c3.json 2> $OUT/bench_c3.err
declare -A STEPS=([c2]=700 [c4]=350 [c5]=15)
for c in c2 c4 c5; do
  timeout 400 python bench.py --config $c --no-cpu --no-context --steps ${STEPS[$c]} > $OUT/bench_$c.json 2> $OUT/bench_$c.err
done
timeout 400 python bench.py --config c5 --fused-mult --no-cpu --no-context --no-e2e --steps 15 > $OUT/bench_c5_fused.json 2> $OUT/bench_c5_fused.err
timeout 300 python bench.py --impl reference --steps 5 --warmup 3 > $OUT/bench_reference.json 2>&1
for c in c3 c2 c4 c5; do
  timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active \
    --clock-control none -k regex:flashsign -c 3 --csv --log-file $OUT/launches_$c.csv \
    python bench.py --config $c --steps 2 --warmup 3 --no-e2e --no-cpu --no-context > /dev/null 2>&1
done
for c in $FULL; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:flashsign_fwd -s 3 -c 1 -o $OUT/prof_$c \
  python bench.py --config $c --steps 1 --warmup 3 --no-e2e --no-cpu --no-context > $OUT/ncu_$c.log 2>&1
# summaries on the box (the .ncu-rep files are ~20 MB each; gpurun copies back <= 64 MiB)
ncu -i $OUT/prof_$c.ncu-rep --page details --csv > $OUT/ncu_full_${c}_details.csv 2>/dev/null
ncu -i $OUT/prof_$c.ncu-rep --page source --csv --print-source sass > $OUT/src_$c.csv 2>/dev/null
python tests/ncu_hot.py $OUT/src_$c.csv 40 > $OUT/ncu_full_${c}_hot_sass.txt 2>&1
rm -f $OUT/src_$c.csv
[ "$c" = "c3" ] || rm -f $OUT/prof_$c.ncu-rep
done
tail -2 $OUT/ncu_c3.log
ls -la $OUT
