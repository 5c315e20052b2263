#!/usr/bin/env bash
# A/B: library variants x env settings: bash tools/ab_env.sh CFG "ENV..." variant...
cfg=$1; envs=$2; shift 2
for v in "$@"; do
  cp paper_1205_1171_b200/lib/variants/$v.so paper_1205_1171_b200/lib/libhull3d_b200.so
  touch paper_1205_1171_b200/lib/libhull3d_b200.so
  for e in $envs; do
    echo -n "$v $e: "
    env $e timeout 300 python tools/level_profile.py --config $cfg --reps 3 2>&1 | tail -1
  done
done
