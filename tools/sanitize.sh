#!/usr/bin/env bash
# compute-sanitizer over every fast-path route (tools/sanitize_routes.py):
#   gpurun -- 'bash tools/sanitize.sh TAG [tools...]'
tag=${1:-r2s}; shift
tools=${*:-memcheck synccheck racecheck initcheck}
out=gpurun_out/$tag; mkdir -p $out
python -c "import sys; sys.path.insert(0,'.'); from paper_1205_1171_b200 import _lib; _lib.load()"
for tool in $tools; do
  lim=5000; [ $tool = memcheck ] && lim=20000; [ $tool = synccheck ] && lim=20000
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 50 \
    python tools/sanitize_routes.py $lim > $out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?" | tee -a $out/status.txt
done
