# gradient bucket size at N = 4 (fewer, longer collectives interrupt the persistent compute kernels less often)
mkdir -p gpurun_out
export NCCL_DEBUG=WARN
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for cfg in 650m 3b; do
for mb in 64 16 128 256; do
  ESM_BUCKET_MB=$mb timeout 900 $TR --nproc-per-node 4 --master-port 29521 bench.py --gpus 4 --config $cfg --steps 10 --warmup 3 --no-e2e > /tmp/b4.json 2>/tmp/b4.err
  python -c "
import json; d=json.loads(open('/tmp/b4.json').read().strip().splitlines()[-1]); print('$cfg n4 bucket=$mb MB', round(d['value']), round(d['ms_per_step'],2), d['clocks']['sm_mhz'])" || tail -2 /tmp/b4.err
done
done
