cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/ -m gpu -x -q 2>&1 | tail -2
python scripts/probe_forward.py mistral7b 512 2>&1 | grep -E "tau=|gemm|attention"
python scripts/gemm_class_sweep.py mistral7b 512 8 2>&1 | head -1
