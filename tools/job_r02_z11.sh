# build 9: L2 persisting window over the cycle's work vectors; A/B (MPK_L2_PERSIST=0/1) + full verification
mkdir -p gpurun_out
nvidia-smi -L > gpurun_out/z11_gpu.txt 2>&1
for i in 1 2; do
  for p in 0 1; do
    echo "MPK_L2_PERSIST=$p" >> gpurun_out/z11_ab.txt
    MPK_L2_PERSIST=$p timeout 300 python tools/time_solve.py --config C4 --solver ir --max-iters 100000 --reps 2 --rule u >> gpurun_out/z11_ab.txt 2>&1
    MPK_L2_PERSIST=$p timeout 300 python tools/time_solve.py --config C2 --solver ir --max-iters 100000 --reps 2 >> gpurun_out/z11_ab.txt 2>&1
  done
done
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/z11_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/z11_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/z11_smoke.log 2>&1; echo "smoke rc $?" >> gpurun_out/z11_smoke.log
timeout 900 python bench.py > gpurun_out/z11_bench_c4.log 2>&1
timeout 900 python bench.py --config C2 > gpurun_out/z11_bench_c2.log 2>&1
timeout 900 python bench.py --impl reference > gpurun_out/z11_bench_ref.log 2>&1
