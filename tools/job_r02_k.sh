mkdir -p gpurun_out
for i in 1 2; do
MPK_BENCH_VERBOSE=1 timeout 900 python bench.py --no-cpu --no-e2e --no-fp64 --steps 3 > gpurun_out/ab_ug2_c4_$i.log 2>&1
MPK_LIB_PATH=$PWD/ab_libs/libug1.so timeout 900 python bench.py --no-cpu --no-e2e --no-fp64 --steps 3 > gpurun_out/ab_ug1_c4_$i.log 2>&1
timeout 900 python bench.py --config C2 --no-cpu --no-e2e --no-fp64 --steps 3 > gpurun_out/ab_ug2_c2_$i.log 2>&1
MPK_LIB_PATH=$PWD/ab_libs/libug1.so timeout 900 python bench.py --config C2 --no-cpu --no-e2e --no-fp64 --steps 3 > gpurun_out/ab_ug1_c2_$i.log 2>&1
done
MPK_LIB_PATH=$PWD/ab_libs/libug1.so timeout 300 python tools/fused_prof.py --config C2 > gpurun_out/prof_C2_ug1.log 2>&1
