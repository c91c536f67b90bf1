timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for i in 1 2; do python scripts/probe_forward.py mistral7b 512 2>&1 | grep -E "ms/iter|attention|combine"; done
python scripts/probe_forward.py yi34b 512 2>&1 | grep -E "ms/iter|attention|combine"
