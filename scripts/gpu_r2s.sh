# 16-softmax-warp attention backward: parity tests + A/B microbenchmark against the 8-warp variant
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -rf -p no:cacheprovider -k "attention or attn" > gpurun_out/r2s_pytest.txt 2>&1
tail -3 gpurun_out/r2s_pytest.txt
for sw in 2 4; do
  ESM_ATTN_BWD_SW=$sw python scripts/microbench.py attn 32,20,1024,24 > gpurun_out/r2s_mb_sw$sw.txt 2>&1
  ESM_ATTN_BWD_SW=$sw python scripts/microbench.py attn 16,20,1024,64 >> gpurun_out/r2s_mb_sw$sw.txt 2>&1
  echo "SW=$sw"; cat gpurun_out/r2s_mb_sw$sw.txt
done
