#!/usr/bin/env bash
# A/B per-level kernel times over environment settings:
#   bash tools/ab_levels.sh TAG "C4 C2" "H3D_LANE=0" "H3D_LANE_XYZ_KB=0 H3D_LANE_STAGE=0" ...
tag=$1; cfgs=$2; shift 2
out=gpurun_out/$tag; mkdir -p $out
i=0
for setting in "$@"; do
  for c in $cfgs; do
    f=$out/levels_${c}_$i.jsonl
    echo "# $setting" > $f
    env $setting timeout 300 python tools/level_profile.py --config $c --reps 3 >> $f 2>&1
    echo "$c [$setting] rc=$? $(tail -1 $f)" | tee -a $out/status.txt
  done
  i=$((i+1))
done
