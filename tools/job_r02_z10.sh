mkdir -p gpurun_out
for cfg in C4 C2; do
  for mb in 32 64 96; do
    for v in 1 2 3; do
      timeout 300 python tools/l2_persist_probe.py --config $cfg --mb $mb --vecs $v >> gpurun_out/z10_l2.txt 2>&1
    done
  done
done
