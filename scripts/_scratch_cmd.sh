cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_pp.py -q -x -p no:cacheprovider > gpurun_out/test_pp.txt 2>&1
tail -15 gpurun_out/test_pp.txt
