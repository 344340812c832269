#!/bin/bash
# usage (under gpurun): bash tools/profile_round.sh <tag>
# 1) bench.py (no profiler)  2) ncu launch list of the same command (per-launch durations)
# 3) one ncu --set full capture of the fused iteration kernel on C4 (the N=1 workload) and C5slab.
tag=${1:-r}
mkdir -p gpurun_out
python bench.py > gpurun_out/${tag}_bench.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/${tag}_launches.csv \
    python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/${tag}_ncu_launch.log 2>&1
for c in C4 C5slab C2 C3; do
  timeout 400 ncu --set full --clock-control none --import-source on -k regex:pf_iter -s 3 -c 1 \
    -o gpurun_out/prof_${tag}_$c -f python tools/prof_iter.py $c 5 > /dev/null 2>&1
done
