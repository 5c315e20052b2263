#!/usr/bin/env bash
cfg=${1:-C4}
for spec in "1 32 200" "1 64 200" "1 128 200" "0 32 24" "1 32 100"; do
  set -- $spec
  echo "== MEASURE=$1 TPB=$2 POOLCAP=$3"
  H3D_TPJ_MEASURE=$1 H3D_TPJ_TPB=$2 H3D_TPJ_FILL=0.5 H3D_TPJ_POOL_KB=$3 timeout 120 python tools/level_profile.py --config $cfg --reps 2 | python -c "
import sys, json
rows=[json.loads(l) for l in sys.stdin]
tp=[r for r in rows if r.get('kernel')=='k_fast_tpj']
print(' '.join(f\"{r['level']}:{r['ms']:.2f}\" for r in tp), ' sum=%.2f' % sum(r['ms'] for r in tp), ' total=%.1f' % rows[-1]['total_ms'])
"
done
