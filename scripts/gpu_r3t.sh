# weak scaling with 256 MB buckets (final): 650M, 3B (8 x 1024), Geneformer at N = 1 / 2 / 4
# Geneformer at N = 1 / 2 / 4; DDP parity check at N = 4
mkdir -p gpurun_out
export NCCL_DEBUG=WARN
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"

for cfg in 650m 3b geneformer; do
  timeout 900 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r3t_${cfg}_n1.json 2> gpurun_out/r3t_${cfg}_n1.err
  timeout 900 $TR --nproc-per-node 2 --master-port 29511 bench.py --gpus 2 --config $cfg --steps 10 --warmup 3 > gpurun_out/r3t_${cfg}_n2.json 2> gpurun_out/r3t_${cfg}_n2.err
  timeout 900 $TR --nproc-per-node 4 --master-port 29521 bench.py --gpus 4 --config $cfg --steps 10 --warmup 3 > gpurun_out/r3t_${cfg}_n4.json 2> gpurun_out/r3t_${cfg}_n4.err
done
timeout 900 $TR --nproc-per-node 4 --master-port 29531 bench.py --gpus 4 --config 3b --steps 10 --warmup 3 --grad-bf16 > gpurun_out/r3t_3b_n4_bf16.json 2> gpurun_out/r3t_3b_n4_bf16.err
python - <<'PY'
import json, glob
base, rows = {}, []
for f in sorted(glob.glob('gpurun_out/r3t_*.json')):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, 'ERR', e); continue
    rows.append((f, d))
    if d['n_gpus'] == 1: base[d['config']['model']] = d['value']
for f, d in rows:
    b = base.get(d['config']['model'])
    print(f, round(d['value']), round(d['ms_per_step'], 2), d.get('mfu'), d['config']['parallelism'], d['clocks']['sm_mhz'],
          'eff', round(d['value'] / (d['n_gpus'] * b), 4) if b else None)
PY
