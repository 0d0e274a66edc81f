mkdir -p gpurun_out
timeout 1200 python bench.py --config C5 > gpurun_out/z17_bench_c5.log 2>&1
timeout 1200 python bench.py --config C3 --poly 25 --max-iters 1000 > gpurun_out/z17_bench_c3.log 2>&1
timeout 600 python bench.py --config C1 > gpurun_out/z17_bench_c1.log 2>&1
