#!/usr/bin/env bash
# A/B per-level kernel times for one env knob: bash tools/ab_levels.sh TAG VAR "A B" [configs]
tag=$1; var=$2; vals=$3; cfgs=${4:-"C4 C2 C3"}
out=gpurun_out/$tag; mkdir -p $out
for c in $cfgs; do
  for v in $vals; do
    env $var=$v timeout 300 python tools/level_profile.py --config $c --reps 3 > $out/levels_${c}_${var}_$v.jsonl 2>&1
    echo "$c $var=$v rc=$? $(tail -1 $out/levels_${c}_${var}_$v.jsonl)" | tee -a $out/status.txt
  done
done
