"""One-time profiling on the B200: calibrated clock + measured token budget
+ tile-quantisation curve for one model. usage: measure_clock.py MODEL OUT.json"""
import json, os, sys, time
sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
from paper_2403_02310_b200 import clock, gpu, host

model, out = sys.argv[1], sys.argv[2]
t0 = time.time()
f = gpu.HybridForward(gpu.MODELS[model], weight_seed=1234)
f.kv_alloc(int(os.environ.get("POOL_BLOCKS", "16384")))
res = clock.b200_clock(f)
res["model"] = model
preset = host.model_preset(model)
res["reference_a100_preset"] = {k: getattr(preset, k) for k in res["calibrated"]}
ref_dref = host.decode_reference_time(preset)
res["reference_a100_slo"] = {}
for label, mult in (("strict", 5.0), ("relaxed", 25.0)):
    try:
        tau = host.compute_token_budget(mult * ref_dref, preset, 1)
    except host.InfeasibleSlo:
        tau = None
    res["reference_a100_slo"][label] = {"t_max_ms": mult * ref_dref, "tau": tau}
res["tile_curve"] = clock.tile_curve(f, [224, 240, 255, 256, 257, 272, 288, 480, 511, 512, 513, 544, 768, 769,
                                         1024, 1025, 1280, 1536, 1537, 2048, 2049])
res["wall_s"] = time.time() - t0
json.dump(res, open(out, "w"), indent=1)
print(json.dumps({k: res[k] for k in ("calibrated", "max_relative_error", "decode_reference_ms", "slo",
                                      "reference_a100_slo")}, indent=1))
