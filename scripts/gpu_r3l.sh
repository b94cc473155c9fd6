# streaming LayerNorm backward with row sums from the STORE_LN dgrad epilogue (ESM_LN_ROWS=0 vs 1)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q -rf -p no:cacheprovider -k "layernorm or gemm" > gpurun_out/r3l_pytest_k.txt 2>&1
tail -2 gpurun_out/r3l_pytest_k.txt
grep -q "failed" gpurun_out/r3l_pytest_k.txt && exit 1
timeout 1500 python -m pytest tests -m gpu -x -q -rf -p no:cacheprovider > gpurun_out/r3l_pytest.txt 2>&1
tail -2 gpurun_out/r3l_pytest.txt
for rep in 1 2; do for v in 1 0; do
  ESM_LN_ROWS=$v timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r3l_b.json 2> gpurun_out/r3l_b.err
  python -c "
import json; d=json.loads(open('gpurun_out/r3l_b.json').read().strip().splitlines()[-1]); print('650m rows=$v', round(d['value']), round(d['ms_per_step'],2), d['mfu'], d['clocks']['sm_mhz'], {k: v['ms'] for k, v in d['kernels'].items() if 'layernorm' in k})"
done; done
ESM_LN_ROWS=1 timeout 900 python bench.py --config 35m --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r3l_b35.json 2>&1; tail -c 300 gpurun_out/r3l_b35.json
