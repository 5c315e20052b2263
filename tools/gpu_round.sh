#!/usr/bin/env bash
# One gpurun call's worth of evidence: GPU tests, smoke, bench (C4, C2, C3),
# per-level profile, ncu launch list (+ DRAM bytes per launch) of one C4 hull,
# and one `ncu --set full` capture of the top kernel.
#   gpurun --timeout 1800 -- 'bash tools/gpu_round.sh [tag] [stages]'
# stages: any of t s b l n f (tests smoke bench levels ncu-list ncu-full), default all
tag=${1:-r1}
stages=${2:-tsblnf}
out=gpurun_out/$tag
mkdir -p "$out"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > "$out/gpu.txt" 2>&1
has() { [[ "$stages" == *"$1"* ]]; }
if has t; then
  timeout 1200 python -m pytest tests -m gpu -x -q > "$out/pytest_gpu.log" 2>&1
  echo "pytest gpu rc=$?" | tee -a "$out/status.txt"
fi
if has s; then
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > "$out/smoke.log" 2>&1
  echo "smoke rc=$?" | tee -a "$out/status.txt"
fi
if has b; then
  timeout 600 python bench.py --steps 10 --warmup 3 > "$out/bench_c4.json" 2> "$out/bench_c4.err"
  echo "bench c4 rc=$?" | tee -a "$out/status.txt"
  for c in C2 C3; do
    timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > "$out/bench_${c,,}.json" 2> "$out/bench_${c,,}.err"
    echo "bench $c rc=$?" | tee -a "$out/status.txt"
  done
  timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > "$out/bench_ref.json" 2> "$out/bench_ref.err"
  echo "bench ref rc=$?" | tee -a "$out/status.txt"
fi
if has l; then
  for c in C4 C3 C2; do
    timeout 300 python tools/level_profile.py --config $c --reps 3 > "$out/levels_${c,,}.jsonl" 2>&1
  done
  echo "levels done" | tee -a "$out/status.txt"
fi
if has n; then
  # one C4 hull after one warm-up hull: skip the warm-up hull's launches by
  # capturing everything and splitting on the hull boundary host-side
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --csv --log-file "$out/launches_c4.csv" \
    python tools/one_hull.py C4 2 > "$out/ncu_list.log" 2>&1
  echo "ncu list rc=$?" | tee -a "$out/status.txt"
fi
if has f; then
  for k in k_fast_tpj k_fast_warp; do
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 \
      -o "$out/full_$k" python tools/one_hull.py C4 1 > "$out/ncu_full_$k.log" 2>&1
    echo "ncu full $k rc=$?" | tee -a "$out/status.txt"
  done
fi
