mkdir -p gpurun_out
for i in 1 2; do
timeout 900 python bench.py --no-cpu --no-e2e --no-fp64 --steps 3 > gpurun_out/ab_new_c4_$i.log 2>&1
MPK_LIB_PATH=$PWD/ab_libs/libug1.so timeout 900 python bench.py --no-cpu --no-e2e --no-fp64 --steps 3 > gpurun_out/ab_ug1_c4_$i.log 2>&1
timeout 900 python bench.py --config C2 --no-cpu --no-e2e --no-fp64 --steps 3 > gpurun_out/ab_new_c2_$i.log 2>&1
MPK_LIB_PATH=$PWD/ab_libs/libug1.so timeout 900 python bench.py --config C2 --no-cpu --no-e2e --no-fp64 --steps 3 > gpurun_out/ab_ug1_c2_$i.log 2>&1
done
timeout 300 python tools/fused_prof.py --config C2 > gpurun_out/prof_C2_new.log 2>&1
timeout 300 python tools/cta_balance.py C2 > gpurun_out/balance_C2.log 2>&1
timeout 300 python tools/cta_balance.py C4 > gpurun_out/balance_C4.log 2>&1
