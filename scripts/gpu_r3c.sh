# fused (dqkv) vs classic attention backward at dh 64 in the 650M step (alternating runs); other configs' lines
mkdir -p gpurun_out
for rep in 1 2; do
  for f in 0 1; do
    ESM_ATTN_FUSED=$f timeout 900 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r3c_b.json 2> gpurun_out/r3c_b.err
    python -c "
import json; d=json.loads(open('gpurun_out/r3c_b.json').read().strip().splitlines()[-1]); print('fused=$f', round(d['value']), round(d['ms_per_step'],2), d['mfu'], d['clocks']['sm_mhz'])"
  done
done
for cfg in 35m 3b geneformer 8m; do
  timeout 900 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r3c_$cfg.json 2> gpurun_out/r3c_$cfg.err
  python -c "
import json; d=json.loads(open('gpurun_out/r3c_$cfg.json').read().strip().splitlines()[-1]); print('$cfg', round(d['value']), round(d['ms_per_step'],2), d['mfu'], d['clocks']['sm_mhz'], d['e2e']['value'] if d.get('e2e') else None)"
done
timeout 900 python bench.py --varlen --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/r3c_varlen.json 2> gpurun_out/r3c_varlen.err
python -c "
import json; d=json.loads(open('gpurun_out/r3c_varlen.json').read().strip().splitlines()[-1]); print('varlen', round(d['value']), round(d['ms_per_step'],2), d['mfu'], d['clocks']['sm_mhz'])"
