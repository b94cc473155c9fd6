# which round-2b change costs N = 4 overlap: fused attention backward, side-stream gradient zeroing, PDL
mkdir -p gpurun_out
export NCCL_DEBUG=WARN
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > /tmp/b1.json 2>/tmp/b1.err
python -c "
import json; d=json.loads(open('/tmp/b1.json').read().strip().splitlines()[-1]); print('n1', round(d['value']), round(d['ms_per_step'],2), d['clocks']['sm_mhz'])"
for v in "X=1" "ESM_ATTN_FUSED=0" "ESM_GRAD_ZERO_SIDE=0" "ESM_PDL=0" "ESM_ATTN_FUSED=0 ESM_GRAD_ZERO_SIDE=0 ESM_PDL=0" "X=1"; do
  env $v timeout 900 $TR --nproc-per-node 4 --master-port 29521 bench.py --gpus 4 --steps 10 --warmup 3 --no-e2e > /tmp/b4.json 2>/tmp/b4.err
  python -c "
import json; d=json.loads(open('/tmp/b4.json').read().strip().splitlines()[-1]); print('n4 $v', round(d['value']), round(d['ms_per_step'],2), d['clocks']['sm_mhz'])"
done
