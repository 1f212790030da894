cd $GRAFT_REPO_ROOT
for t in 0 1500 2500 6000; do if [ $t = 0 ]; then unset QG_TARGET_NNZ; else export QG_TARGET_NNZ=$t; fi; timeout 300 python tools/iter_breakdown.py c4 50 150 2>&1 | tail -1; done
unset QG_TARGET_NNZ
for t in 1000 3000; do QG_TARGET_NNZ=$t timeout 300 python tools/iter_breakdown.py c3 50 150 2>&1 | tail -1; done
for t in 200 400; do QG_TARGET_NNZ=$t timeout 300 python tools/iter_breakdown.py c2 50 150 2>&1 | tail -1; done
