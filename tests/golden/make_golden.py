"""Generates the golden batch-stream fixtures from the REFERENCE simulator.

Run in the build container (needs oracle/_ref/libservesim_ref.so, compiled by
oracle/Makefile from /root/reference/proj/src):  python tests/golden/make_golden.py

Outputs (committed):
  streams.json          per stream: config, trace spec, sha256 + line count of
                        the reference's SimReport::event_log_jsonl
                        (engine.cpp:332-371) and its summarize() report
                        (metrics.cpp:23-59)
  tiny_qps16.jsonl.gz   the full event log of the tiny-clock stream
                        (SURVEY appendix C), for line-level diffs
"""
import gzip
import hashlib
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))

from oracle import ref  # noqa: E402
from paper_2403_02310_b200 import _lib  # noqa: E402

POL = {"request_level": 0, "vllm": 1, "orca": 2, "stall_free": 3}

# (name, clock preset, workload, qps, n, seed, replica overrides)
STREAMS = [
    ("tiny_openchat_qps16", "tiny", "openchat", 16.0, 64, 42, {}),
    ("tiny_openchat_qps4", "tiny", "openchat", 4.0, 64, 42, {}),
    ("tiny_openchat_qps1", "tiny", "openchat", 1.0, 64, 42, {}),
    # configs/yi34b_stall_free_strict.json (reference), via the library path
    ("yi34b_stall_free_strict", "yi34b", "openchat", 0.6, 96, 42, {"token_budget": 512}),
    # BASELINE.json configs[1..4] operating points
    ("mistral7b_openchat_tau512", "mistral7b", "openchat", 1.0, 128, 42, {"token_budget": 512}),
    ("yi34b_tp2_arxiv_tau2048", "yi34b", "arxiv", 0.2, 64, 17, {"token_budget": 2048, "tp_degree": 2}),
    ("llama70b_tp8_openchat_tau1536", "llama70b", "openchat", 0.5, 64, 17, {"token_budget": 1536, "tp_degree": 8}),
    ("falcon180b_tp8_arxiv_tau2048", "falcon180b", "arxiv", 0.2, 48, 42, {"token_budget": 2048, "tp_degree": 8}),
    # other policies and pipeline depth (engine/scheduler parity beyond the hot path)
    ("mistral7b_vllm", "mistral7b", "openchat", 1.0, 48, 7, {"scheduler": "vllm"}),
    ("mistral7b_orca", "mistral7b", "openchat", 1.0, 48, 7, {"scheduler": "orca"}),
    ("mistral7b_request_level", "mistral7b", "openchat", 1.0, 48, 7, {"scheduler": "request_level"}),
    ("falcon180b_pp2_stall_free", "falcon180b", "openchat", 0.3, 32, 5, {"pp_degree": 2, "token_budget": 512}),
    ("yi34b_no_hybrid", "yi34b", "openchat", 0.8, 48, 7, {"hybrid_batching": 0}),
]


def replica(over):
    c = _lib.ReplicaCfg(3, 512, 512, 4096, 0, 1, 1, 131072, 16, 256, 32, 0, 0.10, 0.0, 1)
    for k, v in over.items():
        setattr(c, k, POL[v] if k == "scheduler" else v)
    return c


def main():
    out = []
    for name, clock, wl, qps, n, seed, over in STREAMS:
        trace = ref.make_trace(wl, qps, n, seed)
        st, jsonl, summ = ref.simulate(replica(over), ref.cost_preset(clock) if clock != "tiny" else tiny(), trace)
        assert st == 0, (name, st)
        out.append({
            "name": name, "clock": clock, "workload": wl, "qps": qps, "n": n, "seed": seed, "replica": over,
            "sha256": hashlib.sha256(jsonl.encode()).hexdigest(), "lines": jsonl.count("\n"),
            "trace_sha256": hashlib.sha256(json.dumps(trace).encode()).hexdigest(), "summary": summ,
        })
        if name == "tiny_openchat_qps16":
            with open(os.path.join(HERE, "tiny_qps16.jsonl.gz"), "wb") as raw:
                with gzip.GzipFile(fileobj=raw, mode="wb", mtime=0) as f:
                    f.write(jsonl.encode())
        print(name, out[-1]["lines"], out[-1]["sha256"][:16])
    with open(os.path.join(HERE, "streams.json"), "w") as f:
        json.dump(out, f, indent=1)


def tiny():
    # test_engine.cpp:14-25 tiny_params(); not a reference preset.
    return _lib.CostParams(0.01, 100, 1e-6, 2e-6, 1e-5, 1.0, 0.0, 0.0, 256, 0.32)


if __name__ == "__main__":
    main()
