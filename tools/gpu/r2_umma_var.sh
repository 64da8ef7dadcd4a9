# tcgen05 proxy variants: tests + proxy timing + topk timing
timeout 600 python -m pytest tests/test_gpu_umma.py -x -q > gpurun_out/t10.log 2>&1; echo rc=$? >> gpurun_out/t10.log
HIRE_UMMA_MIN_B=9 BATCHES=9,16,32,64 timeout 200 python tools/bench_proxy.py > gpurun_out/bench_proxy10.log 2>&1
BATCHES=16,32,64 timeout 200 python tools/bench_topk.py > gpurun_out/topk10.log 2>&1
