timeout 1800 python -m pytest tests -m gpu -q -rf -p no:cacheprovider --ignore=tests/test_gpu_trajectory.py -s 2>&1 | grep -E "rel|worst|passed|failed|Error|error|assert|FAIL" | tail -40 > gpurun_out/r2e_tests.txt
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2e_bench650.json 2> gpurun_out/r2e_bench650.err
timeout 900 python bench.py --varlen --steps 20 --warmup 3 > gpurun_out/r2e_varlen650.json 2> gpurun_out/r2e_varlen650.err
cat gpurun_out/r2e_tests.txt
python -c "
import json
for f in ['gpurun_out/r2e_bench650.json','gpurun_out/r2e_varlen650.json']:
    d=json.loads(open(f).read().strip().splitlines()[-1]); print(f, d['value'], d['ms_per_step'], d['mfu'], d.get('clocks'), d['config'].get('non_pad_fraction'), d['config'].get('bucket_shapes'))
" ; tail -3 gpurun_out/r2e_varlen650.err
