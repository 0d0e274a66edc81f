mkdir -p gpurun_out
timeout 300 tools/micro/stream_b > gpurun_out/stream_b4.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_spmv -c 6 -o /tmp/spmv_full -f python tools/spmv_prof.py > gpurun_out/ncu_spmv.log 2>&1
ncu -i /tmp/spmv_full.ncu-rep --page details > gpurun_out/spmv_details.txt 2>&1
ncu -i /tmp/spmv_full.ncu-rep --page raw --csv > gpurun_out/spmv_raw.csv 2>&1
