# GEMM: clusters of two CTA pairs with the shared A rows multicast (MC=2) vs pairs only (ESM_GEMM_MC=0)
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -rf -p no:cacheprovider -k "gemm" > gpurun_out/r3a_pytest.txt 2>&1
tail -2 gpurun_out/r3a_pytest.txt
grep -q "failed" gpurun_out/r3a_pytest.txt && exit 1
echo "== MC=2"; ESM_GEMM_VERBOSE=1 python scripts/microbench.py gemm 650M
echo "== MC=0"; ESM_GEMM_VERBOSE=1 ESM_GEMM_MC=0 python scripts/microbench.py gemm 650M
echo "== MC=2 35M"; python scripts/microbench.py gemm 35M
echo "== MC=0 35M"; ESM_GEMM_MC=0 python scripts/microbench.py gemm 35M
