#!/usr/bin/env bash
# A/B timing of library variants built here: lib/variants/<name>.so
# usage on the box: bash tools/ab_build.sh C4 name1 name2 ...
cfg=$1; shift
for v in "$@"; do
  cp paper_1205_1171_b200/lib/variants/$v.so paper_1205_1171_b200/lib/libhull3d_b200.so
  touch paper_1205_1171_b200/lib/libhull3d_b200.so
  echo -n "$v: "
  timeout 300 python tools/level_profile.py --config $cfg --reps 3 2>&1 | tail -1
done
