# build 5: lagged CGS2 update pass scales by 1/rho; stencil SpMV one group per trip
mkdir -p gpurun_out
for c in C4 C2; do
  r=n_u; [ $c = C4 ] && r=u
  for bp in working binary16; do
    timeout 300 python tools/time_solve.py --config $c --solver ir --max-iters 100000 --reps 2 --rule $r --orth dcgs2 --basis $bp >> gpurun_out/z6_solves.txt 2>&1
  done
done
timeout 300 python tools/time_solve.py --config C4 --solver fp64 --max-iters 100000 --reps 1 --orth dcgs2 >> gpurun_out/z6_solves.txt 2>&1
timeout 300 python tools/time_spmv.py > gpurun_out/z6_spmv.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/z6_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/z6_pytest.log
timeout 300 python tools/prof_run.py --config C4 --orth dcgs2 --basis binary16 --max-iters 200 > gpurun_out/z6_prof_run.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_cycle_dcgs2 -s 2 -c 1 -o /tmp/z6_c4_dch -f python tools/prof_run.py --config C4 --orth dcgs2 --basis binary16 --max-iters 200 > gpurun_out/z6_ncu.log 2>&1
ncu -i /tmp/z6_c4_dch.ncu-rep --page raw --csv > gpurun_out/z6_c4_dch_raw.csv 2>&1
ncu -i /tmp/z6_c4_dch.ncu-rep --page details > gpurun_out/z6_c4_dch_details.txt 2>&1
python tools/ncu_lines.py /tmp/z6_c4_dch.ncu-rep 60 > gpurun_out/z6_c4_dch_source_top.txt 2>&1
