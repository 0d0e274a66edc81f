mkdir -p gpurun_out
timeout 900 python tools/restart_sweep.py 25 50 100 150 200 300 400 > gpurun_out/restart_sweep.log 2>&1
