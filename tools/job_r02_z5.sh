# build 4: stencil SpMV groups per trip A/B (MPK_SPMV_UG=0 generic k_spmv / 1 / 2), parity, sanitizers
mkdir -p gpurun_out
for ug in 0 1 2; do
  echo "MPK_SPMV_UG=$ug" >> gpurun_out/z5_spmv_ab.txt
  MPK_SPMV_UG=$ug timeout 300 python tools/time_spmv.py >> gpurun_out/z5_spmv_ab.txt 2>&1
done
for ug in 1 2; do
  MPK_SPMV_UG=$ug timeout 600 python -m pytest tests/test_gpu_spmv.py tests/test_gpu_fullsize.py -q > gpurun_out/z5_pytest_ug$ug.log 2>&1; echo "rc $?" >> gpurun_out/z5_pytest_ug$ug.log
done
for t in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $t --print-limit 20 python tools/sanitize_r02.py > gpurun_out/z5_sanitizer_$t.txt 2>&1; echo "rc $?" >> gpurun_out/z5_sanitizer_$t.txt
done
# ncu: one 50-step launch of the lagged CGS2 over the binary16 basis (C4), after the plain run exits 0
timeout 300 python tools/prof_run.py --config C4 --orth dcgs2 --basis binary16 --max-iters 200 > gpurun_out/z5_prof_run.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_cycle_dcgs2 -s 2 -c 1 -o /tmp/c4_dch -f python tools/prof_run.py --config C4 --orth dcgs2 --basis binary16 --max-iters 200 > gpurun_out/z5_ncu.log 2>&1
ncu -i /tmp/c4_dch.ncu-rep --page raw --csv > gpurun_out/z5_c4_dch_raw.csv 2>&1
ncu -i /tmp/c4_dch.ncu-rep --page details > gpurun_out/z5_c4_dch_details.txt 2>&1
