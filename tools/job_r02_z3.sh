# A/B: phase A's v_k reads through L1 (MPK_XL1), standalone Laplace SpMV (k_spmv_lap)
mkdir -p gpurun_out
timeout 300 python tools/time_spmv.py > gpurun_out/z3_spmv.txt 2>&1
for i in 1 2; do
  for v in 0 1; do
    echo "C4 XL1=$v" >> gpurun_out/z3_ab.txt
    MPK_XL1=$v timeout 300 python tools/time_solve.py --config C4 --solver ir --max-iters 1000 --rule u >> gpurun_out/z3_ab.txt 2>&1
    echo "C2 XL1=$v" >> gpurun_out/z3_ab.txt
    MPK_XL1=$v timeout 300 python tools/time_solve.py --config C2 --solver ir --max-iters 1000 >> gpurun_out/z3_ab.txt 2>&1
  done
done
MPK_XL1=1 timeout 300 python tools/fused_prof.py --config C4 > gpurun_out/z3_prof_c4.txt 2>&1
MPK_XL1=1 timeout 300 python tools/fused_prof.py --config C2 > gpurun_out/z3_prof_c2.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_spmv.py tests/test_gpu_solvers.py tests/test_gpu_baseline_scale.py tests/test_gpu_fullsize.py -q -x > gpurun_out/z3_pytest.log 2>&1; echo "rc $?" >> gpurun_out/z3_pytest.log
