#!/bin/bash
# usage (under gpurun): bash tools/diag_cluster_traffic.sh <tag> <lib[:VAR=v,...]> ...
# C5slab, per library build / environment: same-box sustained timing (tools/ab.py), launch time vs iteration
# index (tools/iter_trend.py), the DRAM bytes of 20 back-to-back iterations after 100 iterations
# (ncu app-range replay) and of five single launches (kernel replay, cold cache between passes).
tag=${1:-d}; shift
libs=${@:-libpf.so}
mkdir -p gpurun_out
python tools/ab.py --libs $libs --configs C5slab --rounds 2 > gpurun_out/${tag}_ab.log 2>&1
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct
for spec in $libs; do
  lib=${spec%%:*}; envs=${spec#*:}; [ "$envs" = "$spec" ] && envs=""
  name=$(echo $spec | tr ':=,' '___')
  E="env PF_LIB=$lib $(echo $envs | tr ',' ' ')"
  $E python tools/iter_trend.py C5slab 200 20 >> gpurun_out/${tag}_trend.log 2>&1
  for warm in 100; do
    $E timeout 300 ncu --replay-mode app-range --metrics $M --csv python tools/prof_range.py C5slab 20 $warm \
      > gpurun_out/${tag}_range${warm}_$name.csv 2>&1
  done
  $E timeout 300 ncu --clock-control none --metrics $M -k regex:pf_iter -s 10 -c 5 \
    --csv python tools/prof_iter.py C5slab 16 > gpurun_out/${tag}_launch_$name.csv 2>&1
done
tail -n 12 gpurun_out/${tag}_ab.log; cat gpurun_out/${tag}_trend.log
