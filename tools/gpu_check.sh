#!/bin/bash
# usage (under gpurun): bash tools/gpu_check.sh <tag> [configs...]
# GPU tests, per-config timings, and one ncu --set full capture per listed config (one launch each).
tag=${1:-run}; shift
cfgs=${@:-C2 C5slab}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${tag}_pytest.log
python tools/bench_configs.py C2 C3 C4 C5slab --steps 3 > gpurun_out/${tag}_cfg.log 2>&1
for c in $cfgs; do
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:pf_iter -s 3 -c 1 \
    -o gpurun_out/prof_${tag}_$c -f python tools/prof_iter.py $c 5 > /dev/null 2>&1
done
