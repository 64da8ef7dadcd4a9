# round-2 profiles: launch lists (our kernels only) and ncu --set full of the roofline kernels
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/p_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"q4_|sel_|recompute|final|prep_x|lr_|ffn_down|fetch_host|add_offset" -c 200 --csv --log-file gpurun_out/r02_launches_cfg3_b32.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/p_ncu1.log 2>&1
timeout 600 python bench.py --workload cfg4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/p_plain2.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"q4_|sel_|recompute|final|prep_x|lr_|ffn_down|fetch_host|add_offset" -c 200 --csv --log-file gpurun_out/r02_launches_cfg4_b16.csv python bench.py --workload cfg4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/p_ncu2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:q4_score_umma -s 6 -c 1 -o gpurun_out/r02_umma_cfg3_b32 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/p_ncu3.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:recompute_fast -s 6 -c 1 -o gpurun_out/r02_recompute_cfg4 python bench.py --workload cfg4 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/p_ncu4.log 2>&1
echo done
