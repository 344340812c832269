#!/bin/bash
# usage (under gpurun): bash tools/diag_planes.sh -- plane-width / z-chunk diagnostics (DESIGN 6, round 2):
# sustained timings of C5slab and the W* diagnostic volumes (tools/bench_configs.py) under z-chunk / strip
# overrides, and the DRAM bytes of 20 back-to-back iterations (ncu app-range replay) of each.
mkdir -p gpurun_out
python tools/ab.py --libs libpf.so libpf.so:PF_ZCHUNK=48 libpf.so:PF_ZCHUNK=64 --configs W16s W8s --rounds 2 > gpurun_out/diag2_a.log 2>&1
python tools/ab.py --libs libpf.so libpf.so:PF_ZCHUNK=32 libpf.so:PF_ZCHUNK=48 --configs W8 --rounds 2 > gpurun_out/diag2_b.log 2>&1
python tools/ab.py --libs libpf.so libpf.so:PF_STRIP=12,PF_ZCHUNK=48 libpf.so:PF_STRIP=8,PF_ZCHUNK=64 --configs C5slab --rounds 2 > gpurun_out/diag2_c.log 2>&1
for c in C5slab W16s W8 W8s; do
  timeout 300 ncu --replay-mode app-range --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --csv python tools/prof_range.py $c 20 > gpurun_out/diag_range_$c.csv 2>&1
done
tail -n 4 gpurun_out/diag2_*.log
