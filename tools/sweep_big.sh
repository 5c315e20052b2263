#!/usr/bin/env bash
# time-split pipeline threshold sweep (H3D_BIG_KIN)
cfg=${1:-C3}
for k in ${2:-1000000000 4096 1024 256}; do
  echo "== H3D_BIG_KIN=$k"
  H3D_BIG_KIN=$k timeout 300 python tools/level_profile.py --config $cfg --reps 2 2>&1 | python -c "
import sys, json
rows=[json.loads(l) for l in sys.stdin]
print(' '.join(str(r['level'])+':'+('%.2f' % r['ms'])+r['kernel'][7] for r in rows if 'level' in r), ' total=%.1f' % rows[-1]['total_ms'])
"
done
