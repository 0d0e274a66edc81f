mkdir -p gpurun_out
timeout 300 python tools/time_spmv.py > gpurun_out/z13_spmv_graph_noL2.txt 2>&1; echo "rc $?" >> gpurun_out/z13_spmv_graph_noL2.txt
timeout 900 python bench.py > gpurun_out/z13_bench_c4.log 2>&1
timeout 900 python bench.py --config C2 > gpurun_out/z13_bench_c2.log 2>&1
