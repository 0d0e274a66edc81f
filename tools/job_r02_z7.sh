# build 6: z-marching Laplace3D SpMV; A/B of two row groups per trip in phase A (ab_libs/libmpkb200_ug2.so)
mkdir -p gpurun_out
timeout 300 python tools/time_spmv.py > gpurun_out/z7_spmv.txt 2>&1; echo "rc $?" >> gpurun_out/z7_spmv.txt
timeout 600 python -m pytest tests/test_gpu_spmv.py tests/test_gpu_fullsize.py -q > gpurun_out/z7_pytest.log 2>&1; echo "rc $?" >> gpurun_out/z7_pytest.log
for i in 1 2; do
  for lib in default ug2; do
    if [ $lib = ug2 ]; then export MPK_LIB_PATH=$PWD/ab_libs/libmpkb200_ug2.so; else unset MPK_LIB_PATH; fi
    echo "lib=$lib" >> gpurun_out/z7_ab.txt
    timeout 300 python tools/time_solve.py --config C4 --solver ir --max-iters 1000 --rule u >> gpurun_out/z7_ab.txt 2>&1
    timeout 300 python tools/time_solve.py --config C2 --solver ir --max-iters 1000 >> gpurun_out/z7_ab.txt 2>&1
  done
done
unset MPK_LIB_PATH
MPK_LIB_PATH=$PWD/ab_libs/libmpkb200_ug2.so timeout 300 python tools/fused_prof.py --config C4 > gpurun_out/z7_prof_c4_ug2.txt 2>&1
timeout 300 python tools/fused_prof.py --config C4 > gpurun_out/z7_prof_c4_ug1.txt 2>&1
