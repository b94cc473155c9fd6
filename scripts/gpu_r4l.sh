# final-tree check after the attention-dropout work (fp32, dh 24, packed bwd): full GPU suite, smoke, default bench
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -rf -p no:cacheprovider > gpurun_out/r4l_pytest.txt 2>&1
tail -2 gpurun_out/r4l_pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r4l_smoke.txt 2>&1; tail -1 gpurun_out/r4l_smoke.txt
timeout 900 python bench.py > gpurun_out/r4l_bench650.json 2> gpurun_out/r4l_bench650.err
python -c "
import json; d=json.loads(open('gpurun_out/r4l_bench650.json').read().strip().splitlines()[-1]); print('650m', round(d['value']), round(d['ms_per_step'],2), d['mfu'], d['clocks'], 'e2e', round(d['e2e']['value']))"
