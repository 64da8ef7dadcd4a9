# tcgen05 proxy converter / epilogue warpgroup variants (libhire_cuda_c{C}e{E}.so)
for v in c2e2 c4e1 c4e2; do
  HIRE_LIB_VARIANT=libhire_cuda_$v.so HIRE_UMMA_MIN_B=9 BATCHES=16,32,64 timeout 200 python tools/bench_proxy.py > gpurun_out/bp_$v.log 2>&1
done
