cd $GRAFT_REPO_ROOT
QG_PSD_PROF=1 timeout 300 python tools/psd_probe.py 50 2>&1 | grep -v Warn | tail -3
QG_PSD_PROF=1 QG_LIB_PATH=$GRAFT_REPO_ROOT/paper_2508_17522_b200/_lib_ab/libqcpgrad.so timeout 300 python tools/psd_probe.py 50 2>&1 | grep -v Warn | tail -3
for c in c2 c3 c4 c5b; do timeout 300 python tools/iter_breakdown.py $c 50 150 2>&1 | tail -1; done
QG_ENGINE=0 timeout 300 python tools/kernel_times.py c5a "" 50 2>&1 | tail -1
timeout 300 python tools/kernel_times.py c5a "" 50 2>&1 | tail -1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_fin -c 6 python tools/traffic_probe.py --config c2 --which fin --iters 3 2>&1 | grep -E "k_fin|duration" | head -12
timeout 1200 python -m pytest tests/test_gpu_configs_full.py tests/test_gpu_fullsize.py tests/test_gpu_parity.py tests/test_gpu_edges.py -x -q -p no:cacheprovider 2>&1 | tail -2
