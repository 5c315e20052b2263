#!/usr/bin/env bash
# Bench lines of every config with the committed code (profiles/<tag>_bench_*.json).
#   gpurun -- 'bash tools/final_bench.sh TAG'
tag=${1:-rfin}
out=gpurun_out/$tag; mkdir -p $out
for c in C4 C2 C3 INT C5; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 > $out/bench_$c.json 2> $out/bench_$c.err
  echo "bench $c rc=$?" | tee -a $out/status.txt
done
timeout 900 python bench.py --impl reference --config C4 --steps 2 --warmup 1 > $out/bench_reference_C4.json 2> $out/bench_reference_C4.err
echo "reference C4 rc=$?" | tee -a $out/status.txt
