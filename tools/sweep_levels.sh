#!/usr/bin/env bash
# where to switch from thread-per-job to warp-per-job
cfg=${1:-C4}
for spec in "9 16384" "10 8192" "11 4096" "12 2048" "13 1024"; do
  set -- $spec
  echo "== MAX_LEVEL=$1 MIN_JOBS=$2"
  H3D_TPJ_MAX_LEVEL=$1 H3D_TPJ_MIN_JOBS=$2 timeout 120 python tools/level_profile.py --config $cfg --reps 2 | python -c "
import sys, json
rows=[json.loads(l) for l in sys.stdin]
print(' '.join(f\"{r['level']}:{r['kernel'][7]}{r['ms']:.2f}\" for r in rows[:-1] if r['level']>=8), ' total=%.1f' % rows[-1]['total_ms'])
"
done
