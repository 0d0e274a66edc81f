mkdir -p gpurun_out
MPK_BENCH_VERBOSE=1 timeout 900 python bench.py --no-cpu --no-e2e --steps 3 > gpurun_out/bench_c4.log 2>&1
MPK_BENCH_VERBOSE=1 timeout 900 python bench.py --config C2 --no-cpu --no-e2e > gpurun_out/bench_c2.log 2>&1
timeout 300 python tools/fused_prof.py --config C2 > gpurun_out/prof_C2.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log
MPK_BENCH_VERBOSE=1 timeout 1200 python bench.py --config C3 --poly 25 --steps 1 --max-iters 1000 --no-cpu --no-e2e > gpurun_out/bench_c3.log 2>&1
