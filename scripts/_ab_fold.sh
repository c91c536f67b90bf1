cd $GRAFT_REPO_ROOT
timeout 500 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_forward.py -k "gemm or cluster or decode_only or tiny_canonical or full_width or rope" -q -x -p no:cacheprovider > gpurun_out/fold_tests.txt 2>&1
tail -2 gpurun_out/fold_tests.txt
timeout 300 bash scripts/ab.sh "mistral7b 512" 3 fold head2 > gpurun_out/ab_fold.txt 2>&1
timeout 300 bash scripts/ab.sh "mistral7b 512" 3 head2 fold >> gpurun_out/ab_fold.txt 2>&1
AB="SS_GEMM_DSM=1" TAU=32 NDEC=32 ROUNDS=3 timeout 300 bash scripts/ab_lib_env.sh 2 fold head2 >> gpurun_out/ab_fold.txt 2>&1
