#!/usr/bin/env bash
# ncu --set full captures of the one-CTA-per-job (mini) merges: occupancy and
# achieved bandwidth on the top levels (C4 levels 20 / 24, C2's top level on
# the huge variant, C3 level 9 on the medium variant).
#   gpurun -- 'bash tools/evidence_top.sh TAG'
tag=${1:-r2top}
out=gpurun_out/$tag; mkdir -p $out
cap() {  # name config skip (k_mini launches of one hull x 2 hulls)
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_mini -s $3 -c 1 \
    -o $out/$1 python tools/one_hull.py $2 2 > $out/$1.log 2>&1; echo "$1 rc=$?" | tee -a $out/status.txt
}
cap mini_c4_l20 C4 23
cap mini_c4_l24 C4 27
# C2's top level runs on the huge variant: pick it by its demangled name
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k "regex:16384" -s 3 -c 1 -o $out/mini_c2_l20 python tools/one_hull.py C2 2 > $out/mini_c2_l20.log 2>&1
echo "mini_c2_l20 rc=$?" | tee -a $out/status.txt
cap mini_c3_l9 C3 10
