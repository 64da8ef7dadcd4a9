# list-path scan width A/B (8 vs 32 CTAs per SM over the batch)
timeout 300 python -m pytest tests/test_gpu_select.py -x -q > gpurun_out/t13.log 2>&1; echo rc=$? >> gpurun_out/t13.log
for v in libhire_cuda.so libhire_cuda_wl32.so; do
  for w in "--batch 32" "--batch 8" "--workload cfg4" "--workload cfg1"; do
    HIRE_LIB_VARIANT=$v timeout 600 python bench.py $w --steps 30 --warmup 5 --no-cpu-baseline >> gpurun_out/bench13_$v.jsonl 2>>gpurun_out/bench13_err.log
  done
done
