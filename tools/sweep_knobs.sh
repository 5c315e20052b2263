#!/usr/bin/env bash
# routing knob sweep: total merge ms per setting (one line each)
cfg=${1:-C4}
run() {
  echo -n "$* : "
  env "$@" timeout 300 python tools/level_profile.py --config $cfg --reps 2 2>&1 | tail -1
}
run H3D_BIG_KIN=512
run H3D_BIG_KIN=1024
run H3D_BIG_KIN=2048
run H3D_TPJ_XYZ_KB=0
run H3D_TPJ_XYZ_KB=48
run H3D_TPJ_MIN_JOBS=2000
run H3D_TPJ_MIN_JOBS=12000
run H3D_LEAF_B=4
