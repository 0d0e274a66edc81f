mkdir -p gpurun_out
for i in 1 2 3; do timeout 900 python -m pytest tests/test_gpu_distributed.py -q > gpurun_out/pytest_dist_$i.log 2>&1; echo "rc $?" >> gpurun_out/pytest_dist_$i.log; done
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log
