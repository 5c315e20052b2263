#!/usr/bin/env bash
# leaf fusion depth sweep (H3D_LEAF_B = 0 off, 3, 4, 5)
cfg=${1:-C4}
for b in 0 3 4 5; do
  echo "== H3D_LEAF_B=$b"
  H3D_LEAF_B=$b timeout 300 python tools/level_profile.py --config $cfg --reps 2 | python -c "
import sys, json
rows=[json.loads(l) for l in sys.stdin]
print(' '.join(f\"{r['level']}:{r['ms']:.2f}{r['kernel'][7]}\" for r in rows if 'level' in r), ' total=%.1f' % rows[-1]['total_ms'])
"
done
