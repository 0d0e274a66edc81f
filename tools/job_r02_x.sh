mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py --no-cpu --no-e2e --steps 3 > gpurun_out/bench_c4.log 2>&1
timeout 900 python bench.py --config C2 --no-cpu --no-e2e --steps 3 > gpurun_out/bench_c2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_cycle_reg -s 2 -c 1 -o /tmp/c4_reg_full -f python tools/prof_run.py --config C4 --max-iters 200 > gpurun_out/ncu_c4.log 2>&1
python tools/ncu_lines.py /tmp/c4_reg_full.ncu-rep 60 > gpurun_out/c4_src_top.txt 2>&1
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python tools/sanitize_r02.py > gpurun_out/san_memcheck.log 2>&1; echo "rc $?" >> gpurun_out/san_memcheck.log
