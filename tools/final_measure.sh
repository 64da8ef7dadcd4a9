# Round-end measurement recipe (run on the GPU box: bash tools/final_measure.sh): bench lines for every workload and the
# reference arm, the launch list of the default command, one ncu --set full capture of the dominant kernel.
# Large .ncu-rep files stay in /tmp (gpurun_out/ comes back only below 64 MiB).
set -x
mkdir -p gpurun_out
: > gpurun_out/bench_lines.jsonl
timeout 300 python bench.py > gpurun_out/b_default.log 2>&1; tail -1 gpurun_out/b_default.log >> gpurun_out/bench_lines.jsonl
for w in "cfg3 --batch 64" "cfg3 --batch 8" "cfg3 --batch 1" "cfg4" "cfg2" "cfg1" "cfg5 --batch 1" "cfg5 --batch 64"; do
  timeout 400 python bench.py --workload $w > gpurun_out/b.log 2>&1; tail -1 gpurun_out/b.log >> gpurun_out/bench_lines.jsonl
done
timeout 400 python bench.py --impl reference > gpurun_out/b_ref.log 2>&1; tail -1 gpurun_out/b_ref.log >> gpurun_out/bench_lines.jsonl
# -s 440: the weight generators (torch kernels, 63 row blocks) come first
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 440 -c 700 --csv --log-file gpurun_out/launches_cfg3_b32.csv python bench.py --steps 3 --warmup 3 > gpurun_out/ncu1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:q4_score_umma -s 6 -c 1 -o /tmp/umma_cfg3_b32 python bench.py --steps 2 --warmup 3 > gpurun_out/ncu2.log 2>&1
ncu -i /tmp/umma_cfg3_b32.ncu-rep --page raw --csv > gpurun_out/umma_cfg3_b32_raw.csv 2>/dev/null
ncu -i /tmp/umma_cfg3_b32.ncu-rep --page details > gpurun_out/umma_cfg3_b32_details.txt 2>/dev/null
rm -f /tmp/umma_cfg3_b32.ncu-rep
echo done
