cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gputests.log 2>&1; echo "pytest exit $?"; tail -2 gpurun_out/gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
bash tools/bench_all.sh
mkdir -p gpurun_out/prof
timeout 600 ncu --set full --import-source on -k regex:k_step_psd -c 1 -o gpurun_out/prof/r02_c4_psd python tools/traffic_probe.py --config c4 --which ft > /dev/null 2>&1; echo "ncu psd $?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02_c5a_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo "ncu launches $?"
