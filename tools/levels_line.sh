#!/usr/bin/env bash
# one line per config: level:ms+route letter (l leaf, t lane, w warp, e pipeline, m mini)
for c in "$@"; do
  timeout 300 python tools/level_profile.py --config $c --reps 3 > /tmp/l_$c.jsonl 2>&1
  python - "$c" <<'PY'
import json, sys
c = sys.argv[1]
rows = [json.loads(l) for l in open(f"/tmp/l_{c}.jsonl")]
tag = {"k_fast_leaf": "l", "k_fast_tpj": "t", "k_fast_warp": "w", "k_big_level": "e", "k_mini": "m", "k_fast_init1": "i"}
print(c, " ".join(f"{r['level']}:{r['ms']:.2f}{tag.get(r['kernel'], '?')}" for r in rows if "level" in r), rows[-1])
PY
done
