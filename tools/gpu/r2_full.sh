# full GPU suite + bench lines for the main workloads + reference arm
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/full_tests.log 2>&1; echo rc=$? >> gpurun_out/full_tests.log
for b in 1 8 32; do timeout 600 python bench.py --batch $b --steps 30 --warmup 5 --cpu-seconds 5 >> gpurun_out/bench_cfg3.jsonl 2>>gpurun_out/bench_err.log; done
timeout 600 python bench.py --workload cfg4 --steps 30 --warmup 5 --cpu-seconds 5 >> gpurun_out/bench_cfg4.jsonl 2>>gpurun_out/bench_err.log
timeout 600 python bench.py --workload cfg2 --steps 30 --warmup 5 --cpu-seconds 5 >> gpurun_out/bench_cfg2.jsonl 2>>gpurun_out/bench_err.log
timeout 600 python bench.py --workload cfg1 --steps 30 --warmup 5 --cpu-seconds 5 >> gpurun_out/bench_cfg1.jsonl 2>>gpurun_out/bench_err.log
timeout 900 python bench.py --workload cfg5 --steps 10 --warmup 3 >> gpurun_out/bench_cfg5.jsonl 2>>gpurun_out/bench_err.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 >> gpurun_out/bench_ref.jsonl 2>>gpurun_out/bench_err.log
