cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
SS_GEMM_DEBUG=1 timeout 120 python scripts/mc_check.py > gpurun_out/mc_check.txt 2>&1
grep -v "^gemm cg" gpurun_out/mc_check.txt | tail -12
