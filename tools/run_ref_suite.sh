#!/usr/bin/env bash
# Run the reference's OWN pytest suite (mpkrylov pkg/tests, unmodified)
# against this package through the `mpkrylov` shim (tools/ref_suite).
#
#   stage (build container, where /root/reference exists):
#       tools/run_ref_suite.sh stage
#     copies pkg/tests into scratch/ref_tests/ (git-ignored, never committed;
#     it travels to the GPU box with the gpurun snapshot)
#   run (GPU box):
#       tools/run_ref_suite.sh run [pytest args]
#     every solve, SpMV and kernel in those tests runs on cuda:0 through
#     libmpkb200.so.  test_model.py (the SpMV traffic model, out of scope per
#     SURVEY §2) and criterion 02 (which calls it) are deselected.
set -euo pipefail
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
DST="$ROOT/scratch/ref_tests"
case "${1:-run}" in
  stage)
    rm -rf "$DST"; mkdir -p "$DST"
    cp -r /root/reference/pkg/tests/. "$DST/"
    echo "staged $(ls "$DST"/*.py | wc -l) files into $DST"
    ;;
  run)
    shift || true
    export PYTHONPATH="$ROOT/tools/ref_suite:$ROOT${PYTHONPATH:+:$PYTHONPATH}"
    cd "$DST"
    python -c "import mpkrylov, sys; print('mpkrylov ->', mpkrylov.__file__, '| gmres ->', sys.modules['mpkrylov.gmres'].__file__)"
    python -m pytest -q -p no:cacheprovider --ignore=test_model.py \
      --deselect test_acceptance.py::test_criterion_02_spmv_traffic_model "$@" .
    ;;
esac
