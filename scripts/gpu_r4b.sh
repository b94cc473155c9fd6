# bench at N = 2 (torchrun, ZeRO-1, graph) after the e2e loss-read change
mkdir -p gpurun_out
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 \
  bench.py --gpus 2 --steps 10 --warmup 3 > gpurun_out/r4b_n2.json 2> gpurun_out/r4b_n2.err
tail -c 400 gpurun_out/r4b_n2.json; echo
python -c "
import json; d=json.loads(open('gpurun_out/r4b_n2.json').read().strip().splitlines()[-1]); print('n2', round(d['value']), round(d['ms_per_step'],2), 'e2e', round(d['e2e']['value']), d['e2e'].get('device_ms_per_step'), d['config']['parallelism'])" || tail -20 gpurun_out/r4b_n2.err
