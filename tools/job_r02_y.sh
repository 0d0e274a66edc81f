mkdir -p gpurun_out
for i in 1 2; do
for v in 0 1; do
MPK_VK_SYNC=$v timeout 900 python bench.py --no-cpu --no-e2e --no-fp64 --steps 3 > gpurun_out/vk${v}_c4_$i.log 2>&1
MPK_VK_SYNC=$v timeout 900 python bench.py --config C2 --no-cpu --no-e2e --no-fp64 --steps 3 > gpurun_out/vk${v}_c2_$i.log 2>&1
MPK_VK_SYNC=$v timeout 900 python bench.py --config C1 --no-cpu --no-e2e --no-fp64 --steps 5 > gpurun_out/vk${v}_c1_$i.log 2>&1
done; done
MPK_VK_SYNC=1 timeout 300 python tools/fused_prof.py --config C4 > gpurun_out/prof_C4_vk1.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log
