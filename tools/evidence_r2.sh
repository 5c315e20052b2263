#!/usr/bin/env bash
# Round-2 evidence: ncu launch lists (+ DRAM bytes) of one replayed hull per
# config, the bench command's own launch list, and --set full captures of the
# dominant kernels.   gpurun -- 'bash tools/evidence_r2.sh TAG'
tag=${1:-r2ev}
out=gpurun_out/$tag; mkdir -p $out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum
for c in C4 C2 C3; do
  timeout 900 ncu --metrics $M --clock-control none --csv --log-file $out/launches_${c}.csv \
    python tools/one_hull.py $c 3 > $out/ncu_list_${c}.log 2>&1
  echo "list $c rc=$?" | tee -a $out/status.txt
done
timeout 1500 ncu --metrics $M --clock-control none --csv --log-file $out/launches_C5.csv \
  python tools/one_hull.py C5 2 > $out/ncu_list_C5.log 2>&1
echo "list C5 rc=$?" | tee -a $out/status.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $out/bench_launches_c4.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline \
  > $out/bench_under_ncu.log 2>&1
echo "bench list rc=$?" | tee -a $out/status.txt
cap() {  # name regex skip
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$2 -s $3 -c 1 \
    -o $out/$1 python tools/one_hull.py C4 2 > $out/$1.log 2>&1; echo "$1 rc=$?" | tee -a $out/status.txt
}
cap full_lane_l4 k_lane 2
cap full_tpj_l6 k_fast_tpj 5
cap full_leaf k_fast_leaf 1
cap full_rs_pass k_rs_pass 4
