# attention dropout at dh 24 (FOLD backward: Z o (dP - Delta) + (Z - 1) Delta) + the attention / model suites
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_attn_dropout.py -x -q -rf -s -p no:cacheprovider > gpurun_out/r4i_pytest_drop.txt 2>&1
tail -1 gpurun_out/r4i_pytest_drop.txt; grep "dh=24\|H=480" gpurun_out/r4i_pytest_drop.txt
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_model.py -x -q -rf -p no:cacheprovider -k "attention or bf16" > gpurun_out/r4i_pytest.txt 2>&1
tail -1 gpurun_out/r4i_pytest.txt
timeout 300 python scripts/microbench.py attn 32,20,1024,24
