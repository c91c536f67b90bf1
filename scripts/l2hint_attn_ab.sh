# dev A/B of the prefill K/V L2 hint (SS_ATTN_L2HINT bit 2: prefill-tile K/V evict-last)
run() {  # model tau prefix hint
SS_ATTN_L2HINT=$4 python bench.py --model $1 --tau $2 --chunk-prefix $3 --no-cpu-baseline --tbt-requests 0 --steps 30 --e2e-steps 2 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.readlines()[-1]); k=d['kernels']
print('$1 tau=$2 prefix=$3 attn=$4', round(d['ms_per_step'],3), 'clk', d['clocks']['sm_mhz'], ' '.join(f'{n}={v[\"ms_per_step\"]*1000/v[\"launches_per_step\"]:.1f}' for n,v in k.items() if n.startswith('gemm') or n=='attention'))"
}
for r in 1 2; do
  for h in 1 3; do run mistral7b 512 2048 $h; done
  for h in 1 3; do run mistral7b 2048 0 $h; done
  for h in 1 3; do run mistral7b 512 0 $h; done
done
