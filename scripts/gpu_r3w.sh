# BN = 512 auto-pick (long K, good quantisation): GEMM tests + microbench
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -rf -s -p no:cacheprovider -k "gemm" > gpurun_out/r3w_pytest.txt 2>&1
tail -2 gpurun_out/r3w_pytest.txt; grep "wide-tile" gpurun_out/r3w_pytest.txt
timeout 300 python scripts/microbench.py gemm 650M
timeout 300 python scripts/microbench.py gemm store
