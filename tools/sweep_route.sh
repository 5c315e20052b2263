#!/usr/bin/env bash
# level routing threshold sweep: thread-per-job while total jobs >= H3D_TPJ_MIN_JOBS
cfg=${1:-C4}
for mj in 1 4736 20000 100000; do
  echo "== H3D_TPJ_MIN_JOBS=$mj"
  H3D_TPJ_MIN_JOBS=$mj timeout 300 python tools/level_profile.py --config $cfg --reps 2 | python -c "
import sys, json
rows=[json.loads(l) for l in sys.stdin]
print(' '.join(f\"{r['level']}:{r['ms']:.2f}{r['kernel'][7]}\" for r in rows if 'level' in r), ' total=%.1f' % rows[-1]['total_ms'])
"
done
