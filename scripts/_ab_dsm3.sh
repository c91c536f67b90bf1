cd $GRAFT_REPO_ROOT
timeout 400 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_forward.py tests/test_gpu_tp_ipc.py -k "cluster or decode_only or tiny_canonical or push" -q -x -p no:cacheprovider > gpurun_out/dsm3_tests.txt 2>&1
tail -3 gpurun_out/dsm3_tests.txt
AB="SS_GEMM_DSM=1" TAU=32 NDEC=32 ROUNDS=3 timeout 300 bash scripts/ab_lib_env.sh 2 head2 dsm3 > gpurun_out/ab_dsm3.txt 2>&1
AB="SS_GEMM_DSM=1" TAU=32 NDEC=32 ROUNDS=3 timeout 300 bash scripts/ab_lib_env.sh 2 dsm3 head2 >> gpurun_out/ab_dsm3.txt 2>&1
timeout 300 bash scripts/ab.sh "mistral7b 512" 2 dsm3 head2 >> gpurun_out/ab_dsm3.txt 2>&1
