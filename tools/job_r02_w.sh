mkdir -p gpurun_out
for c in C4 C2 C1; do timeout 300 python tools/fused_prof.py --config $c > gpurun_out/prof_$c.log 2>&1; done
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python tools/sanitize_r02.py > gpurun_out/san_memcheck.log 2>&1; echo "rc $?" >> gpurun_out/san_memcheck.log
timeout 1200 compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 20 python tools/sanitize_r02.py > gpurun_out/san_racecheck.log 2>&1; echo "rc $?" >> gpurun_out/san_racecheck.log
timeout 900 compute-sanitizer --tool synccheck --print-limit 20 python tools/sanitize_r02.py > gpurun_out/san_synccheck.log 2>&1; echo "rc $?" >> gpurun_out/san_synccheck.log
