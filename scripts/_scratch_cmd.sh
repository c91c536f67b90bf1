cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python scripts/pp_probe.py > gpurun_out/pp_probe.txt 2>&1
cat gpurun_out/pp_probe.txt
TAUS=1024,2048 timeout 3000 python scripts/capacity_b200.py > gpurun_out/capacity_mistral7b_1024_2048.json 2> gpurun_out/capacity_b.err
tail -3 gpurun_out/capacity_b.err
