#!/usr/bin/env bash
# End-of-round B200 sweep (run under gpurun): GPU suite, smoke, every bench
# config, ncu --set full captures of each config's dominant kernel and the
# default bench's launch list.  Everything lands in gpurun_out/.
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/prof
timeout 2000 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gputests.log 2>&1
echo "pytest exit $?"; tail -n 2 gpurun_out/gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?"; tail -n 1 gpurun_out/smoke.log
bash tools/bench_all.sh
NCU="ncu --set full --import-source on"
P=gpurun_out/prof
timeout 600 $NCU -k regex:^k_engine$ -c 1 -o $P/final_c5a_engine python tools/traffic_probe.py --config c5a --which engine > /dev/null 2>&1; echo "c5a engine $?"
timeout 600 $NCU --kernel-name-base mangled -k regex:k_stepILi1ELi12ELi8E -s 20 -c 1 -o $P/final_c3_FT_df python tools/iter_breakdown.py c3 5 10 > /dev/null 2>&1; echo "c3 df $?"
timeout 600 $NCU --kernel-name-base mangled -k regex:k_stepILi1 -c 1 -o $P/final_c4_FT_main python tools/traffic_probe.py --config c4 --which ft > /dev/null 2>&1; echo "c4 main $?"
timeout 600 $NCU -k regex:k_step_psd -c 1 -o $P/final_c4_psd python tools/traffic_probe.py --config c4 --which ft > /dev/null 2>&1; echo "c4 psd $?"
timeout 900 $NCU --kernel-name-base mangled -k regex:k_stepILi1 -c 1 -o $P/final_c5b_FT python tools/traffic_probe.py --config c5b --which ft > /dev/null 2>&1; echo "c5b $?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/final_c5a_launches.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo "launches $?"
