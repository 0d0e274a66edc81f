# final tree: GPU suite, smoke, default bench, reference arm
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/z19_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/z19_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/z19_smoke.log 2>&1; echo "smoke rc $?" >> gpurun_out/z19_smoke.log
timeout 900 python bench.py > gpurun_out/z19_bench_c4.log 2>&1
timeout 900 python bench.py --impl reference > gpurun_out/z19_bench_ref.log 2>&1
