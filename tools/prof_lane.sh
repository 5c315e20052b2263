#!/usr/bin/env bash
# ncu --set full captures (with source) of the lane-level merge kernels on C4:
#   gpurun -- 'bash tools/prof_lane.sh TAG'
tag=${1:-r2c}
out=gpurun_out/$tag; mkdir -p $out
H3D_LANE=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fast_tpj -s 0 -c 1 \
  -o $out/tpj_l4 python tools/one_hull.py C4 1 > $out/tpj_l4.log 2>&1; echo "tpj l4 rc=$?" | tee -a $out/status.txt
H3D_LANE=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fast_tpj -s 4 -c 1 \
  -o $out/tpj_l8 python tools/one_hull.py C4 1 > $out/tpj_l8.log 2>&1; echo "tpj l8 rc=$?" | tee -a $out/status.txt
H3D_LANE_XYZ_KB=0 H3D_LANE_STAGE=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_lane -s 0 -c 1 \
  -o $out/lane_l4 python tools/one_hull.py C4 1 > $out/lane_l4.log 2>&1; echo "lane l4 rc=$?" | tee -a $out/status.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fast_leaf -s 0 -c 1 \
  -o $out/leaf python tools/one_hull.py C4 1 > $out/leaf.log 2>&1; echo "leaf rc=$?" | tee -a $out/status.txt
