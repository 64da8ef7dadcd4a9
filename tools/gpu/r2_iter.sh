# quick iteration: selector tests + device timelines (bash tools/gpu/r2_iter.sh [all])
mkdir -p gpurun_out
if [ "$1" = "all" ]; then
  (timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -8) > gpurun_out/it_tests.log
else
  (timeout 600 python -m pytest tests/test_gpu_select.py tests/test_gpu_fullsize.py tests/test_gpu_fullsize_r2.py tests/test_gpu_umma.py -m gpu -x -q 2>&1 | tail -8) > gpurun_out/it_tests.log
fi
cat gpurun_out/it_tests.log
for w in "cfg3 --batch 32" "cfg3 --batch 64" "cfg4" "cfg1" "cfg2"; do
  n=$(echo $w | tr -d ' -')
  python tools/ktrace.py --workload $w --reps 2 > gpurun_out/kt_$n.log 2>&1; tail -1 gpurun_out/kt_$n.log
done
