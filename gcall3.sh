cd $GRAFT_REPO_ROOT
for s in 0 1; do QG_PSD_SPLIT=$s QG_PSD_PROF=1 timeout 300 python tools/psd_probe.py 50 2>&1 | grep -v Warn | tail -4; done
QG_ENGINE=0 timeout 300 python tools/kernel_times.py c5a "" 50 2>&1 | tail -2
for c in c2 c3 c4; do timeout 300 python tools/iter_breakdown.py $c 50 150 2>&1 | tail -2; done
timeout 900 python -m pytest tests/test_gpu_configs_full.py -k "psd or deterministic or c5a" -x -q -p no:cacheprovider 2>&1 | tail -3
QG_LIB_PATH=$GRAFT_REPO_ROOT/paper_2508_17522_b200/_lib_checks/libqcpgrad.so timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/checks_build_tests.log 2>&1; echo "checks-build tests exit $?"; tail -2 gpurun_out/checks_build_tests.log
