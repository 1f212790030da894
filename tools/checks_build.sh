#!/usr/bin/env bash
# Bounds-checked GPU suite: compute-sanitizer is closed on the GPU pool, so the
# library is rebuilt with QG_CHECKS=1 (device-side index / invariant checks that
# __trap(), qg_common.cuh) into _lib_checks/ and the whole -m gpu suite runs
# against it through QG_LIB_PATH.  Build here (nvcc cross-compiles), run on the box:
#   bash tools/checks_build.sh build      # in this container
#   bash tools/checks_build.sh run        # under gpurun; log in gpurun_out/
set -u
cd "$(dirname "$0")/.."
case "${1:-run}" in
  build)
    python -c "from paper_2508_17522_b200.build import build; print(build(out='paper_2508_17522_b200/_lib_checks', defines=['QG_CHECKS=1']))" ;;
  run)
    mkdir -p gpurun_out
    QG_LIB_PATH="$PWD/paper_2508_17522_b200/_lib_checks/libqcpgrad.so" timeout 1800 \
        python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/checks_build_tests.log 2>&1
    echo "checks-build suite exit $?"; tail -2 gpurun_out/checks_build_tests.log ;;
esac
