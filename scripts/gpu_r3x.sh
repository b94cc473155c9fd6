# Final-tree check: full GPU suite, smoke, default bench (650M) with CPU baseline and e2e
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -rf -p no:cacheprovider > gpurun_out/r3x_pytest.txt 2>&1
tail -3 gpurun_out/r3x_pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r3x_smoke.txt 2>&1; tail -1 gpurun_out/r3x_smoke.txt
timeout 900 python bench.py > gpurun_out/r3x_bench650.json 2> gpurun_out/r3x_bench650.err; tail -c 300 gpurun_out/r3x_bench650.json
python -c "
import json; d=json.loads(open('gpurun_out/r3x_bench650.json').read().strip().splitlines()[-1]); print('650m', round(d['value']), round(d['ms_per_step'],2), d['mfu'], d['clocks'], d['e2e']['value'])"
