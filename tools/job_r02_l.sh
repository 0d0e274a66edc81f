mkdir -p gpurun_out
for i in 1 2; do
MPK_LIB_PATH=$PWD/ab_libs/libv1.so timeout 900 python bench.py --no-cpu --no-e2e --no-fp64 --steps 3 > gpurun_out/ab_v1_c4_$i.log 2>&1
MPK_LIB_PATH=$PWD/ab_libs/libug1.so timeout 900 python bench.py --no-cpu --no-e2e --no-fp64 --steps 3 > gpurun_out/ab_ug1_c4_$i.log 2>&1
MPK_LIB_PATH=$PWD/ab_libs/libv1.so timeout 900 python bench.py --config C2 --no-cpu --no-e2e --no-fp64 --steps 3 > gpurun_out/ab_v1_c2_$i.log 2>&1
MPK_LIB_PATH=$PWD/ab_libs/libug1.so timeout 900 python bench.py --config C2 --no-cpu --no-e2e --no-fp64 --steps 3 > gpurun_out/ab_ug1_c2_$i.log 2>&1
done
