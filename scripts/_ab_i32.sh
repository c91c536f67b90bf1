cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_gpu_kernels.py -k "gemm" -q -x -p no:cacheprovider > gpurun_out/i32_tests.txt 2>&1
tail -2 gpurun_out/i32_tests.txt
timeout 300 bash scripts/ab.sh "mistral7b 512" 3 i32 fold > gpurun_out/ab_i32.txt 2>&1
timeout 300 bash scripts/ab.sh "mistral7b 512" 3 fold i32 >> gpurun_out/ab_i32.txt 2>&1
AB="SS_GEMM_DSM=1" TAU=32 NDEC=32 ROUNDS=3 timeout 300 bash scripts/ab_lib_env.sh 2 i32 fold >> gpurun_out/ab_i32.txt 2>&1
