cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 60 ./scripts/epi_store_bench > gpurun_out/epi_store_bench.txt 2>&1
cat gpurun_out/epi_store_bench.txt
