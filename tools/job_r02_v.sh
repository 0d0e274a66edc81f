mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log
python - > gpurun_out/assembly_time.log 2>&1 <<'PY'
import sys, time; sys.path.insert(0, '.')
import torch, paper_2105_07544_b200 as mk
for preset, nx in (("Laplace3D", 200), ("BentPipe2D", 1500), ("UniFlow2D", 2500)):
    spec = mk.ProblemSpec(preset, nx)
    mk.generate_stencil(spec, on_device=True); torch.cuda.synchronize()
    t = time.perf_counter(); mk.generate_stencil(spec, on_device=True); torch.cuda.synchronize(); td = time.perf_counter() - t
    t = time.perf_counter(); mk.generate_stencil(spec); th = time.perf_counter() - t
    print("%s %d: device assembly (incl. host copies) %.3f s, numpy %.3f s" % (preset, nx, td, th))
PY
