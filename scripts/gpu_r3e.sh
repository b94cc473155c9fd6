# attention forward at dh <= 32: 32-key tiles at 4 CTAs/SM vs 64-key tiles at 2 CTAs/SM
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -rf -p no:cacheprovider -k "attention or attn" > gpurun_out/r3e_pytest.txt 2>&1
tail -2 gpurun_out/r3e_pytest.txt
grep -q "failed" gpurun_out/r3e_pytest.txt && exit 1
python scripts/microbench.py attn 16,20,1024,64 2>&1
for bn in 32 64; do for fp in 0 1; do
  echo "BN=$bn POLY=$fp"; ESM_ATTN_FWD_BN=$bn ESM_ATTN_FWD_POLY=$fp python scripts/microbench.py attn 32,20,1024,24 2>&1
  ESM_ATTN_FWD_BN=$bn ESM_ATTN_FWD_POLY=$fp python scripts/microbench.py attn 8,20,512,16 2>&1
done; done
