# gmres_restarted host loop overlap: full GPU suite + fp64 timings
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/z16_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/z16_pytest.log
for c in C2 C4; do
  timeout 300 python tools/time_solve.py --config $c --solver fp64 --max-iters 100000 --reps 2 >> gpurun_out/z16_solves.txt 2>&1
done
timeout 900 bash tools/run_ref_suite.sh run -rf --timeout 300 > gpurun_out/z16_ref_suite.log 2>&1; echo "ref suite rc $?" >> gpurun_out/z16_ref_suite.log
