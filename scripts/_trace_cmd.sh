# Scratch command file for dev GPU sessions (gpurun -- 'bash scripts/_trace_cmd.sh').
# Example: per-CTA timelines of the projections inside a 1-layer forward (trace build).
cd $GRAFT_REPO_ROOT
bash scripts/mkvariant.sh trace -DSS_GEMM_TRACE
cp paper_2403_02310_b200/libss_gpu.so /tmp/orig.so
cp build_variants/trace/libss_gpu.so paper_2403_02310_b200/libss_gpu.so
python scripts/gemm_trace.py fwd 2>&1 | grep -v "cta "
cp /tmp/orig.so paper_2403_02310_b200/libss_gpu.so
