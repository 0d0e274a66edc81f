mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log
timeout 600 python tools/time_spmv.py > gpurun_out/time_spmv.log 2>&1
bash tools/job_r02_d.sh
MPK_BENCH_VERBOSE=1 timeout 900 python bench.py --no-cpu > gpurun_out/bench_c4.log 2>&1
MPK_BENCH_VERBOSE=1 timeout 900 python bench.py --config C2 --no-cpu > gpurun_out/bench_c2.log 2>&1
