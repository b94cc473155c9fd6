# attention backward: dK / dV packed to bf16 and released before the epilogue work (fused dqkv path off the
# critical path); classic vs fused at dh 64 in the microbenchmark and in the 650M step
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -rf -p no:cacheprovider -k "attention or attn" > gpurun_out/r2z_pytest_k.txt 2>&1
tail -2 gpurun_out/r2z_pytest_k.txt
grep -q "failed" gpurun_out/r2z_pytest_k.txt && exit 1
python scripts/microbench.py attn 32,20,1024,24 2>&1
python scripts/microbench.py attn 16,20,1024,64 2>&1
for f in 0 1; do
  ESM_ATTN_FUSED=$f timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2z_bench650_fused$f.json 2> gpurun_out/r2z_bench650_fused$f.err
done
timeout 900 python bench.py --config 35m --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2z_bench35.json 2> gpurun_out/r2z_bench35.err
python - <<'PY'
import json
for f in ['gpurun_out/r2z_bench650_fused0.json', 'gpurun_out/r2z_bench650_fused1.json', 'gpurun_out/r2z_bench35.json']:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(f, round(d['value']), round(d['ms_per_step'], 2), d['mfu'], d['clocks']['sm_mhz'])
        for k, v in list(d['kernels'].items())[:8]: print('   ', k, v)
    except Exception as e:
        print(f, 'ERR', e)
PY
echo "==== backward bottleneck experiments"
MB_NOGRAPH= bash scripts/attn_bwd_exp.sh run 2>&1 | grep -E "==|attn B"
