#!/usr/bin/env bash
# thread-per-job tuning sweep: per-level times for several (TPB, fill, pool) settings
cfg=${1:-C4}
for spec in "128 1.0 96" "128 0.5 96" "64 1.0 96" "64 0.5 96" "32 1.0 48" "32 0.5 24" "128 0.25 96" "64 0.25 48"; do
  set -- $spec
  echo "== TPB=$1 FILL=$2 POOL=$3"
  H3D_TPJ_TPB=$1 H3D_TPJ_FILL=$2 H3D_TPJ_POOL_KB=$3 timeout 120 python tools/level_profile.py --config $cfg --reps 2 | python -c "
import sys, json
rows=[json.loads(l) for l in sys.stdin]
tp=[r for r in rows if r.get('kernel')=='k_fast_tpj' and r['pass']==0]
print(' '.join(f\"{r['level']}:{r['ms']:.2f}\" for r in tp), ' sum=%.2f' % sum(r['ms'] for r in tp), ' total=%.1f' % rows[-1]['total_ms'])
"
done
