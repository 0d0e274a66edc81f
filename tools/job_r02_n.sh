mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc $?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_c4_full.log 2>&1
timeout 900 python bench.py --config C2 > gpurun_out/bench_c2_full.log 2>&1
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref_c4.log 2>&1
timeout 1200 python bench.py --config C5 --steps 3 --no-cpu > gpurun_out/bench_c5.log 2>&1
MPK_SHARE_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 tools/dist_check.py Laplace3D 64 u > gpurun_out/dist_check.log 2>&1
