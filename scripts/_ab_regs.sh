cd $GRAFT_REPO_ROOT
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/regs_tests.txt 2>&1 || { echo SMOKE_FAIL >> gpurun_out/regs_tests.txt; exit 1; }
timeout 500 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_forward.py -k "gemm or tiny_canonical or decode_only or full_width or cluster or rope" -q -x -p no:cacheprovider >> gpurun_out/regs_tests.txt 2>&1
tail -3 gpurun_out/regs_tests.txt
bash scripts/ab.sh "mistral7b 512" 3 head regs > gpurun_out/ab_regs.txt 2>&1
bash scripts/ab.sh "mistral7b 512" 3 regs head >> gpurun_out/ab_regs.txt 2>&1
AB="SS_GEMM_DSM=1" TAU=32 NDEC=32 ROUNDS=3 timeout 400 bash scripts/ab_lib_env.sh 2 head regs >> gpurun_out/ab_regs.txt 2>&1
