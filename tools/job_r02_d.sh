mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_spmv -c 4 -o /tmp/spmv5 -f python tools/spmv_prof5.py > gpurun_out/ncu_spmv5.log 2>&1
ncu -i /tmp/spmv5.ncu-rep --page details > gpurun_out/spmv5_details.txt 2>&1
ncu -i /tmp/spmv5.ncu-rep --page source --csv > gpurun_out/spmv5_source.csv 2>&1
ls -la /tmp/spmv5.ncu-rep gpurun_out/
