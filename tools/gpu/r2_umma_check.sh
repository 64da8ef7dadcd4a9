# round-2 check: tcgen05 proxy tests, proxy timing, one bench line, ncu of the proxy kernel
timeout 300 python -m pytest tests/test_gpu_umma.py -x -q > gpurun_out/t6_umma.log 2>&1; echo rc=$? >> gpurun_out/t6_umma.log
HIRE_UMMA_MIN_B=9 BATCHES=9,16,32,64 timeout 200 python tools/bench_proxy.py > gpurun_out/bench_proxy6.log 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 --cpu-seconds 5 > gpurun_out/bench6_cfg3_b32.log 2>&1; echo rc=$? >> gpurun_out/bench6_cfg3_b32.log
BATCHES=32 timeout 200 python tools/bench_proxy.py > gpurun_out/ncu_plain.log 2>&1 && BATCHES=32 timeout 600 ncu --set full --clock-control none --import-source on -k regex:q4_score_umma -s 4 -c 1 -o gpurun_out/prof_umma6 python tools/bench_proxy.py > gpurun_out/ncu6.log 2>&1
