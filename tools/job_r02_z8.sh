# build 7: z-marching Laplace3D SpMV with two planes of lookahead, A/B against k_spmv_pre (MPK_SPMV_ZMARCH=0)
mkdir -p gpurun_out
for i in 1 2; do
  for zm in 0 1; do
    echo "MPK_SPMV_ZMARCH=$zm" >> gpurun_out/z8_spmv_ab.txt
    MPK_SPMV_ZMARCH=$zm timeout 300 python tools/time_spmv.py 2>&1 | grep -v C5 >> gpurun_out/z8_spmv_ab.txt
  done
done
timeout 600 python -m pytest tests/test_gpu_spmv.py tests/test_gpu_fullsize.py -q > gpurun_out/z8_pytest.log 2>&1; echo "rc $?" >> gpurun_out/z8_pytest.log
