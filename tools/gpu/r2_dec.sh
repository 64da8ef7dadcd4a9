timeout 900 python -m pytest tests/test_decoder.py tests/test_gpu_gather_bench.py -x -q > gpurun_out/t18.log 2>&1; echo rc=$? >> gpurun_out/t18.log
timeout 300 python tools/gather_bench.py 262144 128 0.25 1,2,4,8,16,32 > gpurun_out/gather_bench_d128.csv 2>&1; timeout 300 python tools/gather_bench.py > gpurun_out/gather_bench.csv 2>&1
