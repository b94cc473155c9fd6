# e2e with the per-step loss read one step behind (no host stall between steps): 650M, 35M, Geneformer
mkdir -p gpurun_out
for c in 650m 35m; do
  timeout 900 python bench.py --config $c --no-cpu-baseline > gpurun_out/r3z_$c.json 2> gpurun_out/r3z_$c.err
  python -c "
import json; d=json.loads(open('gpurun_out/r3z_$c.json').read().strip().splitlines()[-1]); print('$c', round(d['value']), round(d['ms_per_step'],2), 'e2e', round(d['e2e']['value']), round(d['e2e']['ms_per_step'],2), d['e2e'].get('device_ms_per_step'), d['clocks']['sm_mhz'])" || tail -5 gpurun_out/r3z_$c.err
done
