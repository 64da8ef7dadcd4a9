timeout 600 python -m pytest tests/test_gpu_host_calls.py tests/test_cpp_dropin.py -x -q > gpurun_out/t14.log 2>&1; echo rc=$? >> gpurun_out/t14.log
timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/bench14.jsonl 2>>gpurun_out/bench14_err.log
timeout 600 python bench.py --workload cfg2 --steps 30 --warmup 5 --no-cpu-baseline >> gpurun_out/bench14.jsonl 2>>gpurun_out/bench14_err.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/p_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"q4_|sel_|recompute|final|prep_x|lr_|ffn_down|fetch_host|add_offset" -c 200 --csv --log-file gpurun_out/r02_launches_cfg3_b32.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/p_ncu1.log 2>&1
