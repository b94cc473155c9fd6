# Weak scaling N=1/2/4 (650M, 3B, 35M; ZeRO-1), bucketed varlen line, 650M max batch through the reference's sizing seam
mkdir -p gpurun_out
export NCCL_DEBUG=WARN
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for cfg in 650m 3b 35m; do
  timeout 900 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2r_${cfg}_n1.json 2> gpurun_out/r2r_${cfg}_n1.err
  timeout 900 $TR --nproc-per-node 2 --master-port 29511 bench.py --gpus 2 --config $cfg --steps 10 --warmup 3 > gpurun_out/r2r_${cfg}_n2.json 2> gpurun_out/r2r_${cfg}_n2.err
  timeout 900 $TR --nproc-per-node 4 --master-port 29521 bench.py --gpus 4 --config $cfg --steps 10 --warmup 3 > gpurun_out/r2r_${cfg}_n4.json 2> gpurun_out/r2r_${cfg}_n4.err
done
timeout 900 $TR --nproc-per-node 4 --master-port 29531 bench.py --gpus 4 --config 3b --steps 10 --warmup 3 --grad-bf16 > gpurun_out/r2r_3b_n4_bf16.json 2> gpurun_out/r2r_3b_n4_bf16.err
#timeout 900 python bench.py --varlen --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/r2r_varlen650.json 2> gpurun_out/r2r_varlen650.err
#timeout 1200 python scripts/max_batch.py --config 650m --seq 1024 > gpurun_out/r2r_max_batch.log 2>&1
python - <<'PY'
import json, glob
for f in sorted(glob.glob('gpurun_out/r2r_*.json')):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(f, round(d['value']), round(d['ms_per_step'], 2), d.get('mfu'), d['config'].get('parallelism'), d['clocks']['sm_mhz'], d['clocks']['reasons'])
    except Exception as e:
        print(f, 'ERR', e)
PY
tail -5 gpurun_out/r2r_max_batch.log
