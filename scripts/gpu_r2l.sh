ESM_LN_BULK=0 python scripts/mb_rope.py lnb > gpurun_out/r2l_mb.txt 2>&1
ESM_LN_BULK=0 python scripts/mb_rope.py lnf >> gpurun_out/r2l_mb.txt 2>&1
echo "--- bulk" >> gpurun_out/r2l_mb.txt
python scripts/mb_rope.py lnb >> gpurun_out/r2l_mb.txt 2>&1
python scripts/mb_rope.py lnf >> gpurun_out/r2l_mb.txt 2>&1
timeout 1200 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_model.py -q -rf -p no:cacheprovider 2>&1 | grep -E "^E |passed|failed|FAILED" | head -20 > gpurun_out/r2l_tests.txt
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2l_bench650.json 2> gpurun_out/r2l_bench650.err
timeout 600 python bench.py --config 35m --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2l_bench35.json 2> gpurun_out/r2l_bench35.err
cat gpurun_out/r2l_mb.txt gpurun_out/r2l_tests.txt
python -c "
import json
for f in ['gpurun_out/r2l_bench650.json','gpurun_out/r2l_bench35.json']:
    d=json.loads(open(f).read().strip().splitlines()[-1]); print(f, d['value'], d['ms_per_step'], d['mfu'], d.get('clocks'))
    for k,v in d['kernels'].items(): print('   ',k,v)
"
