timeout 300 python -m pytest tests/test_gpu_select.py tests/test_gpu_umma.py -x -q > gpurun_out/t17.log 2>&1; echo rc=$? >> gpurun_out/t17.log
for w in "--batch 32" "--workload cfg4" "--workload cfg1"; do
  timeout 600 python bench.py $w --steps 30 --warmup 5 --no-cpu-baseline >> gpurun_out/bench17.jsonl 2>>gpurun_out/bench17_err.log
done
