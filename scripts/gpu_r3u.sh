# GEMM BN = 512 (two N = 256 MMAs per k-step, one TMEM accumulator) vs BN = 256 on the 650M shapes
mkdir -p gpurun_out
ESM_GEMM_BN=512 timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -rf -p no:cacheprovider -k "gemm" > gpurun_out/r3u_pytest512.txt 2>&1
tail -2 gpurun_out/r3u_pytest512.txt
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -rf -p no:cacheprovider -k "gemm" > gpurun_out/r3u_pytest.txt 2>&1
tail -2 gpurun_out/r3u_pytest.txt
echo "== BN default 650M"; timeout 300 python scripts/microbench.py gemm 650M
echo "== BN 512 650M"; ESM_GEMM_BN=512 timeout 300 python scripts/microbench.py gemm 650M
echo "== BN default 8192"; timeout 300 python scripts/microbench.py gemm 8192
echo "== BN 512 8192"; ESM_GEMM_BN=512 timeout 300 python scripts/microbench.py gemm 8192
