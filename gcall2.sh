cd $GRAFT_REPO_ROOT
for s in 0 1; do QG_PSD_SPLIT=$s QG_PSD_PROF=1 timeout 300 python tools/psd_probe.py 50 2>&1 | grep -v Warn | tail -6; done
timeout 900 python -m pytest tests/test_gpu_configs_full.py -k "psd or deterministic" tests/test_gpu_parity.py tests/test_gpu_edges.py -x -q -p no:cacheprovider 2>&1 | tail -5
timeout 600 python -m pytest tests/test_gpu_fullsize.py -k c4 -x -q -p no:cacheprovider 2>&1 | tail -3
for s in 1 0; do QG_PSD_SPLIT=$s timeout 600 python bench.py --config c4 --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | cut -c1-300; done
QG_LIB_PATH=$GRAFT_REPO_ROOT/paper_2508_17522_b200/_lib_checks/libqcpgrad.so timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/checks_build_tests.log 2>&1; echo "checks-build tests exit $?"; tail -3 gpurun_out/checks_build_tests.log
