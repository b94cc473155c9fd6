# NCCL channel count (CTAs the collectives occupy while the persistent compute kernels wait) at N = 4, 650M / 3B
mkdir -p gpurun_out
export NCCL_DEBUG=WARN
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for cfg in 650m 3b; do
for v in "X=1" "NCCL_MAX_NCHANNELS=4" "NCCL_MAX_NCHANNELS=8" "NCCL_MAX_NCHANNELS=16" "NCCL_NVLS_ENABLE=0"; do
  env $v timeout 900 $TR --nproc-per-node 4 --master-port 29521 bench.py --gpus 4 --config $cfg --steps 10 --warmup 3 --no-e2e > /tmp/b4.json 2>/tmp/b4.err
  python -c "
import json; d=json.loads(open('/tmp/b4.json').read().strip().splitlines()[-1]); print('$cfg n4 $v', round(d['value']), round(d['ms_per_step'],2), d['clocks']['sm_mhz'])" || tail -2 /tmp/b4.err
done
done
NCCL_DEBUG=INFO timeout 600 $TR --nproc-per-node 4 --master-port 29521 bench.py --gpus 4 --steps 3 --warmup 3 --no-e2e > /tmp/b4.json 2>gpurun_out/r3p_nccl_info.txt
grep -E "NVLS|nChannels|Channel 0[0-9]/|comm 0x.*nRanks" gpurun_out/r3p_nccl_info.txt | head -12
