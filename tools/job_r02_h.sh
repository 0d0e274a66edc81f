mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log
timeout 600 python tools/time_spmv.py > gpurun_out/time_spmv.log 2>&1
MPK_BENCH_VERBOSE=1 timeout 900 python bench.py --no-cpu > gpurun_out/bench_c4.log 2>&1
MPK_BENCH_VERBOSE=1 timeout 900 python bench.py --config C2 --no-cpu > gpurun_out/bench_c2.log 2>&1
MPK_BENCH_VERBOSE=1 timeout 1200 python bench.py --config C3 --poly 25 --steps 1 --max-iters 1000 --no-cpu --no-e2e > gpurun_out/bench_c3.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_cycle_reg -s 2 -c 1 -o /tmp/c4_reg_full -f python tools/prof_run.py --config C4 --max-iters 200 > gpurun_out/ncu_c4.log 2>&1
ncu -i /tmp/c4_reg_full.ncu-rep --page raw --csv > gpurun_out/c4_reg_raw.csv 2>&1
ncu -i /tmp/c4_reg_full.ncu-rep --page details > gpurun_out/c4_reg_details.txt 2>&1
