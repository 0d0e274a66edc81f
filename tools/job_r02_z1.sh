# round 2, session 3: re-verify the rebuilt library, run the reference's own
# suite through the mpkrylov shim, C4 phase breakdown
mkdir -p gpurun_out
nvidia-smi -L > gpurun_out/gpu.txt 2>&1
timeout 600 tools/run_ref_suite.sh run -q -rf --timeout 300 > gpurun_out/ref_suite.log 2>&1; echo "ref suite rc $?" >> gpurun_out/ref_suite.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc $?" >> gpurun_out/smoke.log
timeout 300 python tools/fused_prof.py --config C4 > gpurun_out/prof_c4_fp32.txt 2>&1
timeout 300 python tools/fused_prof.py --config C4 --prec fp64 > gpurun_out/prof_c4_fp64.txt 2>&1
timeout 900 python bench.py > gpurun_out/bench_c4.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log
