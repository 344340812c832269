#!/bin/bash
# usage (under gpurun): bash tools/final_round.sh <tag>
# The round's closing records on one box: GPU suite, smoke, bench + launch list + ncu captures (profile_round.sh),
# then the sustained DRAM traffic (ncu app-range replay, 20 back-to-back iterations after 100) of C4 and C5slab,
# the L2 fetch-granularity hint A/B and the launch time vs iteration index.
tag=${1:-rf}
bash tools/gpu_round.sh $tag
python __graft_entry__.py smoke > gpurun_out/${tag}_smoke.log 2>&1
bash tools/profile_round.sh $tag
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct
for c in C4 C5slab; do
  timeout 300 ncu --replay-mode app-range --metrics $M --csv python tools/prof_range.py $c 20 100 \
    > gpurun_out/${tag}_range_$c.csv 2>&1
done
PF_L2PROMO=0 timeout 300 ncu --replay-mode app-range --metrics $M --csv python tools/prof_range.py C5slab 20 100 \
    > gpurun_out/${tag}_range_C5slab_promo0.csv 2>&1
PF_L2FETCH=32 timeout 300 ncu --replay-mode app-range --metrics $M --csv python tools/prof_range.py C5slab 20 100 \
    > gpurun_out/${tag}_range_C5slab_fetch32.csv 2>&1
python tools/ab.py --libs libpf.so libpf.so:PF_L2FETCH=32 libpf.so:PF_L2FETCH=128 --configs C4 C5slab --rounds 2 \
    > gpurun_out/${tag}_l2fetch_ab.log 2>&1
python tools/iter_trend.py C5slab 200 20 > gpurun_out/${tag}_trend.log 2>&1
python tools/iter_trend.py C4 300 30 >> gpurun_out/${tag}_trend.log 2>&1
tail -n 3 gpurun_out/${tag}_pytest.log; tail -n 1 gpurun_out/${tag}_smoke.log; tail -n 6 gpurun_out/${tag}_l2fetch_ab.log
cat gpurun_out/${tag}_trend.log
