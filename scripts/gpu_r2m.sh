ESM_LN_BULK=0 python scripts/mb_rope.py lnb > gpurun_out/r2m_mb.txt 2>&1
ESM_LN_BULK=0 python scripts/mb_rope.py lnf >> gpurun_out/r2m_mb.txt 2>&1
echo "--- bulk" >> gpurun_out/r2m_mb.txt
python scripts/mb_rope.py lnb >> gpurun_out/r2m_mb.txt 2>&1
python scripts/mb_rope.py lnf >> gpurun_out/r2m_mb.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -rf -p no:cacheprovider -k "layernorm" 2>&1 | tail -2 >> gpurun_out/r2m_mb.txt
ESM_TIMER_DETAIL=1 timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/r2m_bench650_detail.json 2>&1
cat gpurun_out/r2m_mb.txt
python -c "
import json
d=json.loads(open('gpurun_out/r2m_bench650_detail.json').read().strip().splitlines()[-1])
for k,v in d['kernels'].items(): print('   ',k,v)
"
