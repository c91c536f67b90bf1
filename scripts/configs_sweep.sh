#!/bin/bash
# Extra BASELINE configs measurable on one B200 (TP1): Mistral tau=2048, Yi-34B tau=512/2048, chunk at prefix 2048.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
for cfg in "mistral7b 2048 0" "mistral7b 512 2048" "yi34b 512 0" "yi34b 2048 0" "tiny 512 0"; do
  set -- $cfg
  timeout 600 python bench.py --model $1 --tau $2 --chunk-prefix $3 --steps 30 --warmup 5 --no-cpu-baseline --tbt-requests 0 \
    > gpurun_out/cfg_$1_$2_$3.json 2> gpurun_out/cfg_$1_$2_$3.err
  python - "$1" "$2" "$3" <<'PY'
import json, sys
m, t, c = sys.argv[1:4]
try:
    d = json.loads(open(f"gpurun_out/cfg_{m}_{t}_{c}.json").read().strip().splitlines()[-1])
    print(f"{m} tau={t} prefix={c}: {d['value']:.0f} tok/s, {d['ms_per_step']:.3f} ms/step, roofline frac {d['whole_step_roofline']['frac']:.3f}, cost-model {d['cost_model_ms']:.2f} ms, top kernel {d['roofline']['kernel']} {d['roofline']['frac']:.3f}")
except Exception as e:
    print(m, t, c, "FAILED", e, open(f"gpurun_out/cfg_{m}_{t}_{c}.err").read()[-500:])
PY
done
