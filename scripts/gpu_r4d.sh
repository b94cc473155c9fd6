# attention-probability dropout: new tests, the attention / model suites, microbench (p = 0 path unchanged)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_attn_dropout.py -x -q -rf -s -p no:cacheprovider > gpurun_out/r4d_pytest_drop.txt 2>&1
tail -3 gpurun_out/r4d_pytest_drop.txt; grep "attention dropout" gpurun_out/r4d_pytest_drop.txt
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_model.py -x -q -rf -p no:cacheprovider > gpurun_out/r4d_pytest.txt 2>&1
tail -2 gpurun_out/r4d_pytest.txt
timeout 300 python scripts/microbench.py attn
