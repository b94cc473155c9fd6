# 4-GPU weak scaling, second pass: ZeRO-1 / DDP x fp32 / bf16 buckets, high-priority comm stream
export NCCL_DEBUG=WARN
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29531"
for cfg in 3b 650m 35m; do
  timeout 900 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2n_bench_${cfg}_n1.json 2> gpurun_out/r2n_bench_${cfg}_n1.err
  timeout 900 $TR bench.py --gpus 4 --config $cfg --steps 10 --warmup 3 --no-e2e > gpurun_out/r2n_bench_${cfg}_n4_zero1.json 2> gpurun_out/r2n_bench_${cfg}_n4_zero1.err
  timeout 900 $TR bench.py --gpus 4 --config $cfg --steps 10 --warmup 3 --no-e2e --grad-bf16 > gpurun_out/r2n_bench_${cfg}_n4_zero1_bf16.json 2> gpurun_out/r2n_bench_${cfg}_n4_zero1_bf16.err
done
timeout 900 $TR bench.py --gpus 4 --config 3b --steps 10 --warmup 3 --no-e2e --dp ddp --grad-bf16 > gpurun_out/r2n_bench_3b_n4_ddp_bf16.json 2> gpurun_out/r2n_bench_3b_n4_ddp_bf16.err
python - <<'PY'
import json, glob
for f in sorted(glob.glob('gpurun_out/r2n_bench_*.json')):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(f, round(d['value']), round(d['ms_per_step'], 2), d['mfu'], d['config']['parallelism'], d['clocks']['sm_mhz'], d['clocks']['reasons'])
    except Exception as e:
        print(f, 'ERR', e)
PY
