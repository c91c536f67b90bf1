cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/ -m gpu -x -q 2>&1 | tail -2
timeout 300 python scripts/attn_probe.py 2>&1 | tail -6
python scripts/probe_forward.py mistral7b 512 2>&1 | grep -E "tau=|gemm|attention"
python scripts/probe_forward.py mistral7b 2048 2>&1 | grep -E "tau=|attention"
