# attention dropout backward on packed f32x2 math: tests + cost
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_attn_dropout.py -x -q -rf -s -p no:cacheprovider > gpurun_out/r4k_pytest_drop.txt 2>&1
tail -1 gpurun_out/r4k_pytest_drop.txt; grep "model H=" gpurun_out/r4k_pytest_drop.txt
for spec in "geneformer 0,0.02" "650m 0,0.1"; do
  set -- $spec
  timeout 900 python bench.py --config $1 --dropout $2 --no-cpu-baseline --no-e2e > gpurun_out/r4k_$1_$2.json 2> gpurun_out/r4k_$1_$2.err
  python -c "
import json; d=json.loads(open('gpurun_out/r4k_$1_$2.json').read().strip().splitlines()[-1]); k=d['kernels']
print('$1 dropout=$2', round(d['value']), round(d['ms_per_step'],2), d['mfu'], d['clocks']['sm_mhz'], {n: (v['ms'], v['launches']) for n, v in k.items() if 'attn' in n})" || tail -5 gpurun_out/r4k_$1_$2.err
done
