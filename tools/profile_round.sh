#!/usr/bin/env bash
# ncu evidence for profiles/: launch lists (time + DRAM bytes per launch) of
# two hulls per config, and full captures of the dominant kernels.
#   gpurun -- 'bash tools/profile_round.sh TAG'
tag=${1:-r1}
out=gpurun_out/prof_$tag
mkdir -p $out
for c in C4 C3 C2; do
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --csv --log-file $out/launches_${c,,}.csv python tools/one_hull.py $c 2 > /dev/null 2>&1
done
# dominant kernels (one launch each)
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_fast_tpj -s 0 -c 1 \
  -o $out/full_tpj_c4_l4 python tools/one_hull.py C4 1 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_fast_leaf -c 1 \
  -o $out/full_leaf_c4 python tools/one_hull.py C4 1 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_big_sweep -s 0 -c 1 \
  -o $out/full_bigsweep_c3 python tools/one_hull.py C3 1 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_mini -c 1 \
  -o $out/full_mini_c4 python tools/one_hull.py C4 1 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_gather_rows -c 1 \
  -o $out/full_gather_c4 python tools/one_hull.py C4 1 > /dev/null 2>&1
ls -la $out
