# attention forward with 128-key tiles (one S buffer, two-pass softmax over TMEM) vs 64-key tiles
mkdir -p gpurun_out
ESM_ATTN_FWD_BN=128 timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -rf -p no:cacheprovider -k "attention or attn" > gpurun_out/r3i_pytest.txt 2>&1
tail -2 gpurun_out/r3i_pytest.txt
grep -q "failed" gpurun_out/r3i_pytest.txt && exit 1
for i in 1 2; do for bn in 64 128; do
  echo "BN=$bn"; ESM_ATTN_FWD_BN=$bn python scripts/microbench.py attn 32,20,1024,24 2>&1; ESM_ATTN_FWD_BN=$bn python scripts/microbench.py attn 16,20,1024,64 2>&1
done; done
