# Programmatic dependent launch across the step's kernels (ESM_PDL=0 vs default) and one output staging buffer per
# GEMM epilogue warp (one more operand stage; build/exp/libesm_obuf1.so) vs two
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -rf -p no:cacheprovider --deselect tests/test_gpu_trajectory.py > gpurun_out/r3b_pytest.txt 2>&1
tail -3 gpurun_out/r3b_pytest.txt
grep -q "failed" gpurun_out/r3b_pytest.txt && exit 1
for v in "ESM_PDL=1" "ESM_PDL=0" "ESM_PDL=1 ESM_LIB_PATH=build/exp/libesm_obuf1.so"; do
  env $v timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r3b_b.json 2> gpurun_out/r3b_b.err
  python -c "
import json; d=json.loads(open('gpurun_out/r3b_b.json').read().strip().splitlines()[-1]); print('$v', round(d['value']), round(d['ms_per_step'],2), d['mfu'], d['clocks']['sm_mhz'])"
done
echo "== gemm OBUF=2"; python scripts/microbench.py gemm 650M
echo "== gemm OBUF=1"; ESM_LIB_PATH=build/exp/libesm_obuf1.so python scripts/microbench.py gemm 650M
