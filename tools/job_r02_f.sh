mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc $?" >> gpurun_out/smoke.log
timeout 600 python tools/time_spmv.py > gpurun_out/time_spmv.log 2>&1
MPK_BENCH_VERBOSE=1 timeout 900 python bench.py --no-cpu > gpurun_out/bench_c4.log 2>&1
MPK_BENCH_VERBOSE=1 timeout 900 python bench.py --config C2 --no-cpu > gpurun_out/bench_c2.log 2>&1
for c in 144 128 100 74; do MPK_FUSED_CTAS=$c timeout 200 python tools/dump_big.py c2_ir --out gpurun_out/ctas$c >> gpurun_out/dump_ir.log 2>&1; done
timeout 600 compute-sanitizer --tool memcheck --print-limit 20 python tools/sanitize_r02.py > gpurun_out/san_memcheck.log 2>&1; echo "rc $?" >> gpurun_out/san_memcheck.log
timeout 900 compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 20 python tools/sanitize_r02.py > gpurun_out/san_racecheck.log 2>&1; echo "rc $?" >> gpurun_out/san_racecheck.log
timeout 600 compute-sanitizer --tool synccheck --print-limit 20 python tools/sanitize_r02.py > gpurun_out/san_synccheck.log 2>&1; echo "rc $?" >> gpurun_out/san_synccheck.log
