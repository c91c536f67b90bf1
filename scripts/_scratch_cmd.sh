cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
cp paper_2403_02310_b200/libss_gpu.so /tmp/orig.so
for v in st4 st5; do
cp build_variants/$v/libss_gpu.so paper_2403_02310_b200/libss_gpu.so
echo "== $v" >> gpurun_out/gemm_stages.txt
timeout 300 python scripts/gemm_scaling_power.py >> gpurun_out/gemm_stages.txt 2>&1
done
cp /tmp/orig.so paper_2403_02310_b200/libss_gpu.so
echo "== 6 (default)" >> gpurun_out/gemm_stages.txt
timeout 300 python scripts/gemm_scaling_power.py >> gpurun_out/gemm_stages.txt 2>&1
cat gpurun_out/gemm_stages.txt
