mkdir -p gpurun_out
for c in C5slab C2; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:pf_iter -s 3 -c 1 -o gpurun_out/prof_s2_$c -f python tools/prof_iter.py $c 5 > gpurun_out/prof_s2_$c.log 2>&1
done
