#!/bin/bash
# usage (under gpurun): bash tools/diag_cluster_traffic.sh <tag> <lib> [<lib> ...]
# C5slab, per library build: same-box sustained timing (tools/ab.py), the DRAM bytes of 20 back-to-back
# iterations (ncu app-range replay) and of five single launches (kernel replay, cold cache between passes).
tag=${1:-d}; shift
libs=${@:-libpf.so}
mkdir -p gpurun_out
python tools/ab.py --libs $libs --configs C5slab --rounds 2 > gpurun_out/${tag}_ab.log 2>&1
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct
for spec in $libs; do
  lib=${spec%%:*}; envs=${spec#*:}; [ "$envs" = "$spec" ] && envs=""
  name=$(echo $spec | tr ':=,' '___')
  env PF_LIB=$lib $(echo $envs | tr ',' ' ') timeout 300 ncu --replay-mode app-range --profile-from-start off \
    --metrics $M --csv python tools/prof_range.py C5slab 20 > gpurun_out/${tag}_range_$name.csv 2>&1
  env PF_LIB=$lib $(echo $envs | tr ',' ' ') timeout 300 ncu --clock-control none --metrics $M -k regex:pf_iter -s 10 -c 5 \
    --csv python tools/prof_iter.py C5slab 16 > gpurun_out/${tag}_launch_$name.csv 2>&1
done
tail -n 6 gpurun_out/${tag}_ab.log
