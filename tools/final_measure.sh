# Round-end measurement recipe (run on the GPU box: bash tools/final_measure.sh): bench lines, launch lists, one ncu --set full capture.
set -x
mkdir -p gpurun_out
: > gpurun_out/bench_lines.jsonl
timeout 300 python bench.py > gpurun_out/b_default.log 2>&1; tail -1 gpurun_out/b_default.log >> gpurun_out/bench_lines.jsonl
for w in "cfg3" "cfg3 --batch 8" "cfg3 --batch 32" "cfg1" "cfg4"; do
  timeout 300 python bench.py --workload $w > gpurun_out/b.log 2>&1; tail -1 gpurun_out/b.log >> gpurun_out/bench_lines.jsonl
done
timeout 300 python bench.py --impl reference > gpurun_out/b.log 2>&1; tail -1 gpurun_out/b.log >> gpurun_out/bench_lines.jsonl
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_cfg2_b8.csv python bench.py --steps 3 --warmup 3 > gpurun_out/ncu1.log 2>&1
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_cfg4_b16.csv python bench.py --workload cfg4 --steps 3 --warmup 3 > gpurun_out/ncu2.log 2>&1
: timeout 600 ncu --set full --clock-control none --import-source on -k regex:recompute_fast -s 6 -c 1 -o gpurun_out/cfg4_recompute python bench.py --workload cfg4 --steps 2 --warmup 3 > gpurun_out/ncu3.log 2>&1
: ncu -i gpurun_out/cfg4_recompute.ncu-rep --page raw --csv > gpurun_out/cfg4_recompute_raw.csv 2>/dev/null
: ncu -i gpurun_out/cfg4_recompute.ncu-rep --page details > gpurun_out/cfg4_recompute_details.txt 2>/dev/null
echo done
