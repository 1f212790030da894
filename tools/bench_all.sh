#!/usr/bin/env bash
# Every bench config on one B200 (run under gpurun): one bench.py line per
# config into gpurun_out/bench_<cfg>.json, then merged into
# gpurun_out/bench_configs.json (copied to profiles/rNN_bench_configs.json).
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for c in ${CONFIGS:-c5a c1 c2 c3 c4 c5b}; do
  timeout 1200 python bench.py --config "$c" --steps "${STEPS:-5}" --warmup 3 > "gpurun_out/bench_$c.log" 2>&1
  echo "$c exit $?"
  tail -1 "gpurun_out/bench_$c.log" > "gpurun_out/bench_$c.json"
done
python - <<'PY'
import json, os
out = {}
for c in os.environ.get("CONFIGS", "c5a c1 c2 c3 c4 c5b").split():
    try:
        out[c] = json.load(open(f"gpurun_out/bench_{c}.json"))
    except Exception as e:  # keep going: the log says why
        out[c] = {"error": repr(e)}
json.dump(out, open("gpurun_out/bench_configs.json", "w"), indent=1)
for c, d in out.items():
    r = d.get("roofline", {})
    print(c, d.get("value"), (d.get("e2e") or {}).get("value"), r.get("frac"), r.get("traffic"),
          (d.get("cpu_baseline") or {}).get("value"))
PY
