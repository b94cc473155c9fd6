# dQ finalised inside the fused attention backward (last-arriving key-block tile per query block pair)
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -rf -p no:cacheprovider -k "attention or attn" > gpurun_out/r3f_pytest_k.txt 2>&1
tail -3 gpurun_out/r3f_pytest_k.txt
grep -q "failed" gpurun_out/r3f_pytest_k.txt && exit 1
python scripts/microbench.py attn 32,20,1024,24 2>&1
python scripts/microbench.py attn 16,20,1024,64 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q -rf -p no:cacheprovider --deselect tests/test_gpu_trajectory.py > gpurun_out/r3f_pytest.txt 2>&1
tail -3 gpurun_out/r3f_pytest.txt
for cfg in 650m 35m; do
  timeout 900 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r3f_$cfg.json 2> gpurun_out/r3f_$cfg.err
  python -c "
import json; d=json.loads(open('gpurun_out/r3f_$cfg.json').read().strip().splitlines()[-1]); print('$cfg', round(d['value']), round(d['ms_per_step'],2), d['mfu'], d['clocks']['sm_mhz']); print('   ', {k: v['ms'] for k, v in list(d['kernels'].items())[:6]})"
done
