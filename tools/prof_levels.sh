#!/usr/bin/env bash
# ncu --set full captures (with source) of the merge kernels of one C4 hull:
# lane.cu at level 4, k_fast_tpj at levels 6 and 8, the leaf.
#   gpurun -- 'bash tools/prof_levels.sh TAG'
tag=${1:-r2l}
out=gpurun_out/$tag; mkdir -p $out
cap() {  # name regex skip
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$2 -s $3 -c 1 \
    -o $out/$1 python tools/one_hull.py C4 1 > $out/$1.log 2>&1; echo "$1 rc=$?" | tee -a $out/status.txt
}
cap lane_l4 k_lane 0
cap tpj_l6 k_fast_tpj 0
cap tpj_l8 k_fast_tpj 2
cap leaf k_fast_leaf 0
