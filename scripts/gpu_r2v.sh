# attention forward softmax: in-place S registers, 4-way max tree, FFMA2/FADD2, FMA-pipe exp2 pairs (0/1/2 of 4)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -rf -p no:cacheprovider -k "attention or attn" > gpurun_out/r2v_pytest.txt 2>&1
tail -3 gpurun_out/r2v_pytest.txt
for fp in 0 1 2; do
  echo "FWD_POLY=$fp"
  ESM_ATTN_FWD_POLY=$fp python scripts/microbench.py attn 32,20,1024,24 2>&1
  ESM_ATTN_FWD_POLY=$fp python scripts/microbench.py attn 16,20,1024,64 2>&1
done
