#!/bin/bash
# One GPU session: tests, smoke, bench, ncu launch list + full captures of the top kernels.
set -x
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv
if [ "${TESTS:-1}" = "1" ]; then
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -25
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
fi
if [ "${BENCH:-1}" = "1" ]; then
timeout 900 python bench.py --steps 100 --warmup 10 ${BENCH_ARGS:-} > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -3 gpurun_out/bench.err; cat gpurun_out/bench.json
fi
if [ "${NCU:-1}" = "1" ]; then
PS="python bench.py --warmup 3 --profile-step ${BENCH_ARGS:-}"
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    $PS > /dev/null 2>&1; echo "launches rc=$?"
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:gemm_tcgen05 -c 4 -o gpurun_out/prof_gemm -f \
    $PS > gpurun_out/ncu_gemm.log 2>&1; echo "ncu gemm rc=$?"
timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on --kernel-name-base mangled \
    -k regex:attention_kernelILi128ELi0E -c 1 -o gpurun_out/prof_attn -f $PS > gpurun_out/ncu_attn.log 2>&1; echo "ncu attn rc=$?"
timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on --kernel-name-base mangled \
    -k regex:attention_kernelILi128ELi2E -c 1 -o gpurun_out/prof_attn_tc -f $PS > gpurun_out/ncu_attn_tc.log 2>&1; echo "ncu attn tc rc=$?"
fi
