# dev A/B of the L2 eviction-priority hints (SS_ATTN_L2HINT; SS_GEMM_L2HINT bits: 1 A evict-last, 2 B evict-first)
run() {  # model tau hintA hintG
SS_ATTN_L2HINT=$3 SS_GEMM_L2HINT=$4 python bench.py --model $1 --tau $2 --no-cpu-baseline --tbt-requests 0 --steps ${STEPS:-50} --e2e-steps 2 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.readlines()[-1]); k=d['kernels']
print('$1 tau=$2 attn=$3 gemm=$4', round(d['ms_per_step'],3), 'clk', d['clocks']['sm_mhz'], ' '.join(f'{n}={v[\"ms_per_step\"]*1000/v[\"launches_per_step\"]:.1f}' for n,v in k.items() if n.startswith('gemm') or n=='attention'))"
}
for r in 1 2; do
  for g in ${GH:-0 2 3}; do run mistral7b 512 1 $g; done
  for g in ${GH:-0 2 3}; do run mistral7b 2048 1 $g; done
  for g in ${GH:-0 2 3}; do run yi34b 512 1 $g; done
done
