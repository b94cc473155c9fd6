# 4-GPU weak scaling (650M, 3B; ZeRO-1 default) + 2-GPU DDP check at 4 ranks
export NCCL_DEBUG=WARN
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29521"
timeout 900 $TR scripts/ddp_check.py > gpurun_out/r2j_ddp_check_n4.log 2>&1; echo "ddp_check rc=$?"; grep -E "PASSED|FAILED|FAIL" gpurun_out/r2j_ddp_check_n4.log | head
for cfg in 650m 3b; do
  timeout 900 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2j_bench_${cfg}_n1.json 2> gpurun_out/r2j_bench_${cfg}_n1.err
  timeout 900 $TR bench.py --gpus 4 --config $cfg --steps 10 --warmup 3 --no-e2e > gpurun_out/r2j_bench_${cfg}_n4.json 2> gpurun_out/r2j_bench_${cfg}_n4.err
  timeout 900 $TR bench.py --gpus 4 --config $cfg --steps 10 --warmup 3 --no-e2e --dp ddp > gpurun_out/r2j_bench_${cfg}_n4_ddp.json 2> gpurun_out/r2j_bench_${cfg}_n4_ddp.err
done
python - <<'PY'
import json, glob
for f in sorted(glob.glob('gpurun_out/r2j_bench_*.json')):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(f, round(d['value']), round(d['ms_per_step'], 2), d['mfu'], d['config']['parallelism'], d['clocks'])
    except Exception as e:
        print(f, 'ERR', e)
PY
