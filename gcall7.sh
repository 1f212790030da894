cd $GRAFT_REPO_ROOT
for c in c2 c3 c4; do for f in 1 0; do QG_FIN_EARLY=$f timeout 300 python tools/iter_breakdown.py $c 50 150 2>&1 | tail -1; done; done
timeout 900 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_parity.py -x -q -p no:cacheprovider 2>&1 | tail -2
