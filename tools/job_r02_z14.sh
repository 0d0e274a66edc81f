# final build: ncu of k_cycle_reg (with the L2 window) on C4 and C2, launch list of a C4 run
mkdir -p gpurun_out
for c in C4 C2; do
  timeout 300 python tools/prof_run.py --config $c --max-iters 200 > gpurun_out/z14_prof_$c.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_cycle_reg -s 2 -c 1 -o /tmp/z14_$c -f python tools/prof_run.py --config $c --max-iters 200 > gpurun_out/z14_ncu_$c.log 2>&1
  ncu -i /tmp/z14_$c.ncu-rep --page raw --csv > gpurun_out/z14_${c}_raw.csv 2>&1
  ncu -i /tmp/z14_$c.ncu-rep --page details > gpurun_out/z14_${c}_details.txt 2>&1
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/z14_c4_launches.csv python tools/prof_run.py --config C4 --max-iters 500 > gpurun_out/z14_ncu_c4_launch.log 2>&1
