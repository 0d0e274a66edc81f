# build 3: lagged CGS2 over the 16-bit basis, k_spmv_lap (host-side group check)
mkdir -p gpurun_out
timeout 300 python tools/time_spmv.py > gpurun_out/z4_spmv.txt 2>&1; echo "rc $?" >> gpurun_out/z4_spmv.txt
for c in C4 C2 C1; do
  r=n_u; [ $c = C4 ] && r=u
  for o in cgs2 dcgs2; do
    for bp in working binary16; do
      timeout 300 python tools/time_solve.py --config $c --solver ir --max-iters 100000 --reps 2 --rule $r --orth $o --basis $bp >> gpurun_out/z4_solves.txt 2>&1
    done
  done
done
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/z4_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/z4_pytest.log
timeout 900 python bench.py > gpurun_out/z4_bench_c4.log 2>&1
