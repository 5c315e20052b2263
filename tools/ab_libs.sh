#!/usr/bin/env bash
# Per-level A/B of prebuilt library variants (gpurun_out/lib_<tag>/):
#   bash tools/ab_libs.sh OUT_TAG CONFIG tag1 tag2 ...
out=gpurun_out/$1; cfg=$2; shift 2; mkdir -p $out
cp paper_1205_1171_b200/lib/libhull3d_b200.so $out/base.so
for t in base "$@"; do
  if [ "$t" = base ]; then cp $out/base.so paper_1205_1171_b200/lib/libhull3d_b200.so
  else cp tools/libvariants/$t.so paper_1205_1171_b200/lib/libhull3d_b200.so; fi
  touch paper_1205_1171_b200/lib/libhull3d_b200.so
  timeout 300 python tools/level_profile.py --config $cfg --reps 3 > $out/levels_${cfg}_$t.jsonl 2>&1
  echo "$t $(tail -1 $out/levels_${cfg}_$t.jsonl)" | tee -a $out/status.txt
done
cp $out/base.so paper_1205_1171_b200/lib/libhull3d_b200.so
