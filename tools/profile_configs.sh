#!/usr/bin/env bash
# ncu --set full captures (one launch each) of the hot kernels of every
# bench config, on the bench's own workloads (tools/traffic_probe.py):
#   graph-path configs (c2 c3 c4 c5b): k_step<F'>, k_step<F>, k_fin / k_fin_cta
#   resident configs (c1 c5a): k_engine (one launch = one whole LSMR solve)
# Reports land in gpurun_out/prof/; tools/ncu_report.py summarises them.
set -u
OUT=gpurun_out/prof
mkdir -p "$OUT"
NCU="ncu --set full --import-source on"
for c in ${CONFIGS:-c2 c3 c4 c5b}; do
  timeout 900 $NCU --kernel-name-base mangled -k regex:k_stepILi1 -c 1 -o "$OUT/r02_${c}_FT" \
      python tools/traffic_probe.py --config "$c" --which ft > "$OUT/r02_${c}_FT.log" 2>&1; echo "$c FT $?"
  timeout 900 $NCU --kernel-name-base mangled -k regex:k_stepILi0 -c 1 -o "$OUT/r02_${c}_F" \
      python tools/traffic_probe.py --config "$c" --which f > "$OUT/r02_${c}_F.log" 2>&1; echo "$c F $?"
  timeout 900 $NCU -k regex:^k_fin -s 8 -c 1 -o "$OUT/r02_${c}_fin" \
      python tools/traffic_probe.py --config "$c" --which fin --iters 3 > "$OUT/r02_${c}_fin.log" 2>&1; echo "$c fin $?"
done
for c in ${ENGINE_CONFIGS:-c1 c5a}; do
  timeout 900 $NCU -k regex:^k_engine$ -c 1 -o "$OUT/r02_${c}_engine" \
      python tools/traffic_probe.py --config "$c" --which engine > "$OUT/r02_${c}_engine.log" 2>&1; echo "$c engine $?"
done
