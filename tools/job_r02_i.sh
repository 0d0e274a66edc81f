mkdir -p gpurun_out
MPK_BENCH_VERBOSE=1 timeout 900 python bench.py --no-cpu --no-e2e --steps 3 > gpurun_out/bench_c4.log 2>&1
MPK_BENCH_VERBOSE=1 timeout 900 python bench.py --config C2 --no-cpu --no-e2e > gpurun_out/bench_c2.log 2>&1
for c in C2 C4 C1; do timeout 300 python tools/fused_prof.py --config $c > gpurun_out/prof_$c.log 2>&1; done
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log
MPK_BENCH_VERBOSE=1 timeout 1200 python bench.py --config C3 --poly 25 --steps 1 --max-iters 1000 --no-cpu --no-e2e > gpurun_out/bench_c3.log 2>&1
timeout 600 python tools/time_spmv.py > gpurun_out/time_spmv.log 2>&1
