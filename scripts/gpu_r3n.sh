# weak-scaling A/B on one box: the round-2a tree (commit b498626, build/old_tree) vs the current tree, 650M N=1 / 4
mkdir -p gpurun_out
export NCCL_DEBUG=WARN
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for rep in 1 2; do
  for tree in old cur; do
    if [ $tree = old ]; then D=build/old_tree; else D=.; fi
    (cd $D && timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > /tmp/b1.json 2>/tmp/b1.err)
    python -c "
import json; d=json.loads(open('/tmp/b1.json').read().strip().splitlines()[-1]); print('$tree n1', round(d['value']), round(d['ms_per_step'],2), d['clocks']['sm_mhz'])"
    (cd $D && timeout 900 $TR --nproc-per-node 4 --master-port 29521 bench.py --gpus 4 --steps 10 --warmup 3 --no-e2e > /tmp/b4.json 2>/tmp/b4.err)
    python -c "
import json; d=json.loads(open('/tmp/b4.json').read().strip().splitlines()[-1]); print('$tree n4', round(d['value']), round(d['ms_per_step'],2), d['clocks']['sm_mhz'], d['config']['parallelism'])"
  done
done
