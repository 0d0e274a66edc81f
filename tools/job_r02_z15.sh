# build 10: cached cooperative occupancy + IR host loop that enqueues the next refinement before its bookkeeping
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/z15_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/z15_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/z15_smoke.log 2>&1; echo "smoke rc $?" >> gpurun_out/z15_smoke.log
for i in 1 2; do
  timeout 300 python tools/time_solve.py --config C2 --solver ir --max-iters 100000 --reps 3 >> gpurun_out/z15_solves.txt 2>&1
  timeout 300 python tools/time_solve.py --config C4 --solver ir --max-iters 100000 --reps 2 --rule u >> gpurun_out/z15_solves.txt 2>&1
done
timeout 900 python bench.py --config C2 > gpurun_out/z15_bench_c2.log 2>&1
timeout 900 python bench.py > gpurun_out/z15_bench_c4.log 2>&1
timeout 900 bash tools/run_ref_suite.sh run -rf --timeout 300 > gpurun_out/z15_ref_suite.log 2>&1; echo "ref suite rc $?" >> gpurun_out/z15_ref_suite.log
