mkdir -p gpurun_out
timeout 300 tools/micro/stream_b_sweep > gpurun_out/stream_sweep.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log
timeout 600 python tools/time_spmv.py > gpurun_out/time_spmv.log 2>&1
MPK_BENCH_VERBOSE=1 timeout 900 python bench.py --config C5 --steps 3 --no-cpu > gpurun_out/bench_c5.log 2>&1
