# Round-2c measurement recipe (bash tools/gpu/r2c_measure.sh): bench lines for every workload, the reference arm,
# the launch list of the default bench command and ncu --set full captures of its two top kernels.
set -x
mkdir -p gpurun_out
o=gpurun_out/r02c_bench_lines.jsonl
: > $o
timeout 300 python bench.py > gpurun_out/b_default.log 2>&1; tail -1 gpurun_out/b_default.log >> $o
for w in "cfg3 --batch 64" "cfg3 --batch 8" "cfg3 --batch 1" "cfg4" "cfg2" "cfg1" "cfg5" "cfg5 --batch 64"; do
  timeout 400 python bench.py --workload $w > gpurun_out/b.log 2>&1; tail -1 gpurun_out/b.log >> $o
done
timeout 300 python bench.py --impl reference > gpurun_out/b_ref.log 2>&1; tail -1 gpurun_out/b_ref.log >> $o
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/b_short.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/r02c_launches_cfg3_b32.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sel_stream_kernel -s 3 -c 1 -o gpurun_out/r02c_stream_cfg3_b32 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu2.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:q4_score_umma -s 3 -c 1 -o gpurun_out/r02c_umma_cfg3_b32 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu3.log 2>&1
echo done
