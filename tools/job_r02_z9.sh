# final session-3 verification on one B200
mkdir -p gpurun_out
nvidia-smi -L > gpurun_out/z9_gpu.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/z9_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/z9_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/z9_smoke.log 2>&1; echo "smoke rc $?" >> gpurun_out/z9_smoke.log
timeout 900 python bench.py > gpurun_out/z9_bench_c4.log 2>&1
timeout 900 python bench.py --config C2 > gpurun_out/z9_bench_c2.log 2>&1
timeout 900 python bench.py --impl reference > gpurun_out/z9_bench_ref.log 2>&1
