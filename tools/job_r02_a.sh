mkdir -p gpurun_out
timeout 600 python tools/dump_big.py c2_fp64 c2_ir c4_fp64 c4_ir_u c2_fp64_dcgs2 > gpurun_out/dump_big.log 2>&1
for c in 144 128 100 74; do MPK_FUSED_CTAS=$c timeout 200 python tools/dump_big.py c2_fp64 --out gpurun_out/ctas$c >> gpurun_out/dump_big.log 2>&1; done
MPK_BENCH_VERBOSE=1 timeout 900 python bench.py > gpurun_out/bench_c4.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_cycle_reg -s 2 -c 1 -o /tmp/c4_reg_full -f python tools/prof_run.py --config C4 --max-iters 200 > gpurun_out/ncu_c4.log 2>&1
ncu -i /tmp/c4_reg_full.ncu-rep --page raw --csv > gpurun_out/c4_reg_raw.csv 2>&1
ncu -i /tmp/c4_reg_full.ncu-rep --page details > gpurun_out/c4_reg_details.txt 2>&1
ls -la /tmp/c4_reg_full.ncu-rep >> gpurun_out/ncu_c4.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/c4_launches.csv python tools/prof_run.py --config C4 --max-iters 500 > gpurun_out/ncu_c4_launch.log 2>&1
nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o /tmp/l2bw tools/micro/l2bw.cu && timeout 300 /tmp/l2bw > gpurun_out/l2bw.log 2>&1
du -sh gpurun_out/* > gpurun_out/du.txt
