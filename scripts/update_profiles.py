"""Copy a GPU session's evidence into profiles/<round>/ and refresh profiles/ncu_traffic.json.
usage: python scripts/update_profiles.py r01 [tag]"""
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
rnd = sys.argv[1]
tag = sys.argv[2] if len(sys.argv) > 2 else "latest"
src = os.path.join(ROOT, "gpurun_out")
dst = os.path.join(ROOT, "profiles", rnd)
os.makedirs(dst, exist_ok=True)
shutil.copy(os.path.join(src, "bench.json"), os.path.join(dst, f"bench_mistral7b_tau512_{tag}.json"))
shutil.copy(os.path.join(src, "launches.csv"), os.path.join(dst, f"launches_mistral7b_tau512_{tag}.csv"))
summ = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "ncu_summary.py"), src], capture_output=True,
                      text=True, check=True).stdout
open(os.path.join(dst, f"ncu_summary_{tag}.json"), "w").write(summ)
d = json.loads(summ)


def mb(e, k):
    v = e.get(k, "0 Mbyte").split()
    x = float(v[0])
    unit = v[1] if len(v) > 1 else "byte"
    return x * {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3}.get(unit, 1.0)


traffic = {}
# the GEMM capture holds the 4 projections of one layer in forward order
for cls, e in zip(["gemm_qkv", "gemm_o", "gemm_gate_up", "gemm_down"], d.get("prof_gemm.ncu-rep", [])):
    traffic[cls] = int(mb(e, "dram__bytes_read.sum") + mb(e, "dram__bytes_write.sum"))
for e in d.get("prof_attn.ncu-rep", [])[:1]:  # the decode (HBM-streaming) attention kernel
    traffic["attention"] = int(mb(e, "dram__bytes_read.sum") + mb(e, "dram__bytes_write.sum"))
for e in d.get("prof_attn_tc.ncu-rep", [])[:1]:  # the tensor-core prefill attention kernel
    traffic["attention_tc"] = int(mb(e, "dram__bytes_read.sum") + mb(e, "dram__bytes_write.sum"))
out = {"_note": f"dram__bytes_read.sum + dram__bytes_write.sum per launch from `ncu --set full` captures "
                f"(profiles/{rnd}/ncu_summary_{tag}.json); used by bench.py as roofline.traffic",
       "mistral7b": traffic}
json.dump(out, open(os.path.join(ROOT, "profiles", "ncu_traffic.json"), "w"), indent=1)
print(json.dumps(out, indent=1))
