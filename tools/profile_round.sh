#!/bin/bash
# usage (under gpurun): bash tools/profile_round.sh <tag>
# 1) bench.py (no profiler)  2) ncu launch list of the same command (per-launch durations)
# 3) one ncu --set full capture of the fused iteration kernel on C4 (the N=1 workload), C5slab (its c5slab
#    leg), C2 and C3, summarised on the box (metrics, stall sites, instruction mix; DRAM traffic entries for
#    profiles/ncu_traffic.json) -- the reports themselves are removed (gpurun copies back <= 64 MiB).
tag=${1:-r}
mkdir -p gpurun_out
python bench.py > gpurun_out/${tag}_bench.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/${tag}_launches.csv \
    python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/${tag}_ncu_launch.log 2>&1
for c in C4 C5slab C2 C3; do
  timeout 400 ncu --set full --clock-control none --import-source on -k regex:pf_iter -s 3 -c 1 \
    -o gpurun_out/prof_${tag}_$c -f python tools/prof_iter.py $c 5 gpurun_out/kinfo_${tag}_$c.json > /dev/null 2>&1
  alg=$(python -c "import json; print(json.load(open('gpurun_out/kinfo_${tag}_$c.json'))['algorithmic_bytes_per_iteration'])")
  python tools/ncu_summary.py gpurun_out/prof_${tag}_$c.ncu-rep gpurun_out/ncu_${tag}_$c.json $alg $c --traffic \
    > /dev/null 2>&1
  python tools/ncu_hot.py gpurun_out/prof_${tag}_$c.ncu-rep 30 > gpurun_out/ncu_${tag}_${c}_hot.txt 2>&1
  python tools/ncu_mix.py gpurun_out/prof_${tag}_$c.ncu-rep 30 > gpurun_out/ncu_${tag}_${c}_mix.txt 2>&1
  rm -f gpurun_out/prof_${tag}_$c.ncu-rep
done
cp profiles/ncu_traffic.json gpurun_out/${tag}_ncu_traffic.json 2>/dev/null
