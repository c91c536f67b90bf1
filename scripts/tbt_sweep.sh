#!/bin/bash
# Closed-loop P99 TBT (restated engine, measured B200 forward as the model step) for the TP1
# BASELINE configurations (dev tool; results -> gpurun_out/tbt_*.json).
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
for cfg in "mistral7b 512" "mistral7b 2048" "yi34b 512" "yi34b 2048"; do
  set -- $cfg
  timeout 900 python bench.py --model $1 --tau $2 --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 2 \
    > gpurun_out/tbt_$1_$2.json 2> gpurun_out/tbt_$1_$2.err
  python - "$1" "$2" <<'PY'
import json, sys
m, t = sys.argv[1:3]
try:
    d = json.loads(open(f"gpurun_out/tbt_{m}_{t}.json").read().strip().splitlines()[-1])
    b = d["tbt"]
    print(f"{m} tau={t}: P99 TBT {b['p99_ms']:.2f} ms (cost-model clock {b['cost_model_clock']['p99_ms']:.2f}), "
          f"median TBT {b['median_ms']:.2f}, median TTFT {b['ttft_median_ms']:.1f} ms, {b['iterations']} iterations, "
          f"throughput {b['throughput_tps']:.0f} tok/s (cost-model {b['cost_model_clock']['throughput_tps']:.0f})")
except Exception as e:
    print(m, t, "FAILED", e, open(f"gpurun_out/tbt_{m}_{t}.err").read()[-400:])
PY
done
