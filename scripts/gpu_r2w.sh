# ABI LSE in the backward's log2 form (no conversion pass), wave-aware GEMM tile widths
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -rf -p no:cacheprovider -k "attention or attn or delta or gemm" > gpurun_out/r2w_pytest_k.txt 2>&1
tail -3 gpurun_out/r2w_pytest_k.txt
grep -q "failed" gpurun_out/r2w_pytest_k.txt && exit 1
python scripts/microbench.py attn 32,20,1024,24 2>&1
python scripts/microbench.py attn 16,20,1024,64 2>&1
python scripts/microbench.py gemm 650M > gpurun_out/r2w_gemm_new.txt 2>&1
ESM_GEMM_BN=256 python scripts/microbench.py gemm 650M > gpurun_out/r2w_gemm_256.txt 2>&1
paste gpurun_out/r2w_gemm_new.txt gpurun_out/r2w_gemm_256.txt | awk -F'\t' '{print $1 "   ||   " $2}' | sed 's/gemm 650M //g'
timeout 1500 python -m pytest tests -m gpu -x -q -rf -p no:cacheprovider --deselect tests/test_gpu_trajectory.py > gpurun_out/r2w_pytest.txt 2>&1
tail -4 gpurun_out/r2w_pytest.txt
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2w_bench650.json 2> gpurun_out/r2w_bench650.err
ESM_TIMER_DETAIL=1 timeout 900 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/r2w_bench650_detail.json 2> gpurun_out/r2w_bench650_detail.err
timeout 900 python bench.py --config 35m --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2w_bench35.json 2> gpurun_out/r2w_bench35.err
python - <<'PY'
import json
for f in ['gpurun_out/r2w_bench650.json', 'gpurun_out/r2w_bench35.json', 'gpurun_out/r2w_bench650_detail.json']:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(f, round(d['value']), round(d['ms_per_step'], 2), d['mfu'], d['clocks']['sm_mhz'])
        for k, v in d['kernels'].items(): print('   ', k, v)
    except Exception as e:
        print(f, 'ERR', e)
PY
