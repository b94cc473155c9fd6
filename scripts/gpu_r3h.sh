# GEMM: 3 epilogue warps per TMEM lane quarter (12) vs 2 (8), on the 35M (K = 480, epilogue-heavy) and 650M shapes
mkdir -p gpurun_out
ESM_LIB_PATH=build/exp/libesm_ew3.so timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -rf -p no:cacheprovider -k "gemm" > gpurun_out/r3h_pytest.txt 2>&1
tail -2 gpurun_out/r3h_pytest.txt
echo "== EW=2 35M"; python scripts/microbench.py gemm 35M
echo "== EW=3 35M"; ESM_LIB_PATH=build/exp/libesm_ew3.so python scripts/microbench.py gemm 35M
echo "== EW=2 650M"; python scripts/microbench.py gemm 650M
echo "== EW=3 650M"; ESM_LIB_PATH=build/exp/libesm_ew3.so python scripts/microbench.py gemm 650M
for lib in "" "ESM_LIB_PATH=build/exp/libesm_ew3.so"; do
  env $lib timeout 900 python bench.py --config 35m --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r3h_b.json 2> gpurun_out/r3h_b.err
  python -c "
import json; d=json.loads(open('gpurun_out/r3h_b.json').read().strip().splitlines()[-1]); print('35m $lib', round(d['value']), round(d['ms_per_step'],2), d['mfu'], d['clocks']['sm_mhz'])"
done
