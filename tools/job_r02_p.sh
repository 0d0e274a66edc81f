mkdir -p gpurun_out
timeout 300 python tools/host_profile.py > gpurun_out/host_profile.log 2>&1
timeout 900 python tools/c5_window_ab.py > gpurun_out/c5_window_ab2.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log
