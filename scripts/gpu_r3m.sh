# N = 4 overlap with and without programmatic dependent launch (650M and 3B, ZeRO-1, fp32 buckets)
mkdir -p gpurun_out
export NCCL_DEBUG=WARN
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for cfg in 650m 3b; do
  for pdl in 0 1; do
    ESM_PDL=$pdl timeout 900 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r3m_b.json 2> gpurun_out/r3m_b.err
    python -c "
import json; d=json.loads(open('gpurun_out/r3m_b.json').read().strip().splitlines()[-1]); print('$cfg n1 pdl=$pdl', round(d['value']), round(d['ms_per_step'],2), d['clocks']['sm_mhz'])"
    ESM_PDL=$pdl timeout 900 $TR --nproc-per-node 4 --master-port 29521 bench.py --gpus 4 --config $cfg --steps 10 --warmup 3 --no-e2e > gpurun_out/r3m_b.json 2> gpurun_out/r3m_b.err
    python -c "
import json; d=json.loads(open('gpurun_out/r3m_b.json').read().strip().splitlines()[-1]); print('$cfg n4 pdl=$pdl', round(d['value']), round(d['ms_per_step'],2), d['clocks']['sm_mhz'])"
  done
done
