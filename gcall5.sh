cd $GRAFT_REPO_ROOT
for c in c2 c3 c4 c5b; do for f in 1 0; do QG_FUSED_FIN=$f timeout 300 python tools/iter_breakdown.py $c 50 150 2>&1 | tail -1; done; done
QG_PSD_ORDER=1 timeout 300 python tools/iter_breakdown.py c4 50 150 2>&1 | tail -1
QG_LIB_PATH=$GRAFT_REPO_ROOT/paper_2508_17522_b200/_lib_ab/libqcpgrad.so timeout 300 python tools/iter_breakdown.py c4 50 150 2>&1 | tail -1
QG_PSD_ORDER=1 QG_LIB_PATH=$GRAFT_REPO_ROOT/paper_2508_17522_b200/_lib_ab/libqcpgrad.so timeout 300 python tools/iter_breakdown.py c4 50 150 2>&1 | tail -1
timeout 1500 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_configs_full.py tests/test_gpu_parity.py tests/test_gpu_engine.py -x -q -p no:cacheprovider 2>&1 | tail -3
