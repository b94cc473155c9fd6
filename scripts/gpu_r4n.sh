# LayerNorm forward on f32x2 arithmetic (FADD2 / FFMA2) vs the previous kernel: microbench A/B, LN tests
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -rf -p no:cacheprovider -k "layernorm or ln" > gpurun_out/r4n_pytest.txt 2>&1
tail -1 gpurun_out/r4n_pytest.txt
for r in 1 2; do
echo "== new"; timeout 300 python scripts/microbench.py ln
echo "== old"; ESM_LIB_PATH=build/exp/libesm_lnold.so timeout 300 python scripts/microbench.py ln
done
