# Delta fused into the out-projection dgrad epilogue (ESM_EPI_DELTA), LSE converted in the attention backward,
# forward softmax rewrite (in-place S registers, max tree, FFMA2/FADD2, FMA-pipe exp2 pairs)
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -rf -p no:cacheprovider -k "attention or attn or delta" > gpurun_out/r2u_pytest_attn.txt 2>&1
tail -3 gpurun_out/r2u_pytest_attn.txt
grep -q "failed" gpurun_out/r2u_pytest_attn.txt && exit 1
for fp in 0 1 2; do
  echo "FWD_POLY=$fp"
  ESM_ATTN_FWD_POLY=$fp python scripts/microbench.py attn 32,20,1024,24 2>&1
  ESM_ATTN_FWD_POLY=$fp python scripts/microbench.py attn 16,20,1024,64 2>&1
done
timeout 1500 python -m pytest tests -m gpu -x -q -rf -p no:cacheprovider --deselect tests/test_gpu_trajectory.py > gpurun_out/r2u_pytest.txt 2>&1
tail -4 gpurun_out/r2u_pytest.txt
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2u_bench650.json 2> gpurun_out/r2u_bench650.err
timeout 900 python bench.py --config 35m --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2u_bench35.json 2> gpurun_out/r2u_bench35.err
python - <<'PY'
import json
for f in ['gpurun_out/r2u_bench650.json', 'gpurun_out/r2u_bench35.json']:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(f, round(d['value']), round(d['ms_per_step'], 2), d['mfu'], d['clocks']['sm_mhz'])
        for k, v in d['kernels'].items(): print('   ', k, v)
    except Exception as e:
        print(f, 'ERR', e)
PY
