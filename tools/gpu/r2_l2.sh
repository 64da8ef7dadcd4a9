# L2 policy A/B on the tcgen05 proxy (evict-first weights, evict-last scores)
timeout 300 python -m pytest tests/test_gpu_umma.py -x -q > gpurun_out/t12.log 2>&1; echo rc=$? >> gpurun_out/t12.log
for v in libhire_cuda.so libhire_cuda_l2off.so; do
  HIRE_LIB_VARIANT=$v BATCHES=16,32,64 timeout 200 python tools/bench_topk.py >> gpurun_out/topk12_$v.log 2>&1
  HIRE_LIB_VARIANT=$v timeout 600 python bench.py --batch 32 --steps 30 --warmup 5 --no-cpu-baseline >> gpurun_out/bench12_$v.jsonl 2>>gpurun_out/bench12_err.log
done
