#!/usr/bin/env bash
cfg=${1:-C4}
for spec in "1 32 0.5 24" "0 32 0.5 24" "1 64 1.0 48" "1 128 1.0 96"; do
  set -- $spec
  echo "== SORT=$1 TPB=$2 FILL=$3 POOL=$4"
  H3D_TPJ_SORT=$1 H3D_TPJ_TPB=$2 H3D_TPJ_FILL=$3 H3D_TPJ_POOL_KB=$4 timeout 120 python tools/level_profile.py --config $cfg --reps 2 | python -c "
import sys, json
rows=[json.loads(l) for l in sys.stdin]
tp=[r for r in rows if r.get('kernel')=='k_fast_tpj']
print(' '.join(f\"{r['level']}:{r['ms']:.2f}\" for r in tp), ' sum=%.2f' % sum(r['ms'] for r in tp), ' total=%.1f' % rows[-1]['total_ms'])
"
done
