mkdir -p gpurun_out
timeout 300 python tools/time_spmv.py > gpurun_out/z12_spmv_graph.txt 2>&1; echo "rc $?" >> gpurun_out/z12_spmv_graph.txt
