mkdir -p gpurun_out
timeout 300 python tools/cta_balance.py C2 > gpurun_out/balance_C2.log 2>&1
timeout 300 python tools/cta_balance.py C4 > gpurun_out/balance_C4.log 2>&1
timeout 900 python tools/c5_window_ab.py > gpurun_out/c5_window_ab.log 2>&1
MPK_SHARE_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 tools/dist_check.py Laplace3D 64 u > gpurun_out/dist_check.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_cycle_reg -s 2 -c 1 -o /tmp/c4_reg_full -f python tools/prof_run.py --config C4 --max-iters 200 > gpurun_out/ncu_c4.log 2>&1
ncu -i /tmp/c4_reg_full.ncu-rep --page raw --csv > gpurun_out/c4_reg_raw.csv 2>&1
ncu -i /tmp/c4_reg_full.ncu-rep --page details > gpurun_out/c4_reg_details.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_cycle_reg -s 2 -c 1 -o /tmp/c2_reg_full -f python tools/prof_run.py --config C2 --max-iters 200 > gpurun_out/ncu_c2.log 2>&1
ncu -i /tmp/c2_reg_full.ncu-rep --page raw --csv > gpurun_out/c2_reg_raw.csv 2>&1
ncu -i /tmp/c2_reg_full.ncu-rep --page details > gpurun_out/c2_reg_details.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/c4_launches.csv python tools/prof_run.py --config C4 --max-iters 500 > gpurun_out/ncu_c4_launch.log 2>&1
