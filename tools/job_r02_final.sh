mkdir -p gpurun_out
nvidia-smi -L > gpurun_out/gpu.txt 2>&1; nproc >> gpurun_out/gpu.txt; lscpu | grep "Model name" >> gpurun_out/gpu.txt
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc $?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_c4_final.log 2>&1
timeout 900 python bench.py --config C2 > gpurun_out/bench_c2_final.log 2>&1
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref_c4_final.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_cycle_reg -s 2 -c 1 -o /tmp/c4_reg_full -f python tools/prof_run.py --config C4 --max-iters 200 > gpurun_out/ncu_c4.log 2>&1
ncu -i /tmp/c4_reg_full.ncu-rep --page raw --csv > gpurun_out/c4_reg_raw.csv 2>&1
ncu -i /tmp/c4_reg_full.ncu-rep --page details > gpurun_out/c4_reg_details.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/c4_launches.csv python tools/prof_run.py --config C4 --max-iters 500 > gpurun_out/ncu_c4_launch.log 2>&1
