timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "recompute or da_topk" > gpurun_out/t11.log 2>&1; echo rc=$? >> gpurun_out/t11.log
timeout 600 python bench.py --workload cfg4 --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/bench11_cfg4.jsonl 2>>gpurun_out/bench11_err.log
