# attention dropout in the fp32 parity kernels + the full GPU suite
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_attn_dropout.py -x -q -rf -s -p no:cacheprovider > gpurun_out/r4j_pytest_drop.txt 2>&1
tail -1 gpurun_out/r4j_pytest_drop.txt; grep "fp32" gpurun_out/r4j_pytest_drop.txt
timeout 1800 python -m pytest tests -m gpu -q -rf -p no:cacheprovider > gpurun_out/r4j_pytest.txt 2>&1
tail -2 gpurun_out/r4j_pytest.txt
