# GEMM tail-round split (half-width slices for the last partial round): tests, microbench, 650M / 35M bench
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -rf -s -p no:cacheprovider -k "gemm" > gpurun_out/r4a_pytest.txt 2>&1
tail -2 gpurun_out/r4a_pytest.txt; grep "tail-split" gpurun_out/r4a_pytest.txt
echo "== tail split"; timeout 300 python scripts/microbench.py gemm 650M
echo "== ESM_GEMM_TAIL=0"; ESM_GEMM_TAIL=0 timeout 300 python scripts/microbench.py gemm 650M
for c in 650m 35m; do
  for t in 1 0; do
    ESM_GEMM_TAIL=$t timeout 900 python bench.py --config $c --no-cpu-baseline --no-e2e > gpurun_out/r4a_${c}_$t.json 2> gpurun_out/r4a_${c}_$t.err
    python -c "
import json; d=json.loads(open('gpurun_out/r4a_${c}_$t.json').read().strip().splitlines()[-1]); print('$c tail=$t', round(d['value']), round(d['ms_per_step'],2), d['mfu'], d['clocks']['sm_mhz'])" || tail -5 gpurun_out/r4a_${c}_$t.err
  done
done
