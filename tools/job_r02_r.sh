mkdir -p gpurun_out
timeout 600 python tools/time_spmv.py > gpurun_out/time_spmv_new.log 2>&1
MPK_LIB_PATH=$PWD/ab_libs/libprev.so timeout 600 python tools/time_spmv.py > gpurun_out/time_spmv_prev.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q -x -k "spmv or csr or mmio or precond" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log
