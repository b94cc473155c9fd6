# attention backward at dh 64: 4 Q/dO stages with one reused dQ staging box vs 3 stages with two boxes
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -rf -p no:cacheprovider -k "attention or attn" > gpurun_out/r3g_pytest.txt 2>&1
tail -2 gpurun_out/r3g_pytest.txt
grep -q "failed" gpurun_out/r3g_pytest.txt && exit 1
for i in 1 2; do
  echo "QST=4"; python scripts/microbench.py attn 16,20,1024,64 2>&1; python scripts/microbench.py attn 4,40,1024,64 2>&1
  echo "QST=3"; ESM_LIB_PATH=build/exp/libesm_qst3.so python scripts/microbench.py attn 16,20,1024,64 2>&1; ESM_LIB_PATH=build/exp/libesm_qst3.so python scripts/microbench.py attn 4,40,1024,64 2>&1
done
