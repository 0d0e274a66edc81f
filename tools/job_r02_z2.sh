mkdir -p gpurun_out
PYTHONPATH=tools/ref_suite timeout 600 python tools/ref_cases.py gpurun_out/ref_cases_ours.json > gpurun_out/ref_cases.log 2>&1; echo "rc $?" >> gpurun_out/ref_cases.log
