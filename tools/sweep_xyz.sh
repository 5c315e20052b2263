#!/usr/bin/env bash
# compare coordinate staging thresholds for the thread-per-job kernel
cfg=${1:-C4}
for kb in 0 16 48 200; do
  echo "== H3D_TPJ_XYZ_KB=$kb"
  H3D_TPJ_XYZ_KB=$kb timeout 120 python tools/level_profile.py --config $cfg --reps 2 | python -c "
import sys, json
rows=[json.loads(l) for l in sys.stdin]
tp=[r for r in rows if r.get('kernel')=='k_fast_tpj']
print(' '.join(f\"{r['level']}:{r['ms']:.2f}\" for r in tp), ' sum=%.2f' % sum(r['ms'] for r in tp), ' total=%.1f' % rows[-1]['total_ms'])
"
done
