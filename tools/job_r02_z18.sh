mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_third_precision.py -q > gpurun_out/z18_pytest.log 2>&1; echo "rc $?" >> gpurun_out/z18_pytest.log
