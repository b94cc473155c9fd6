# GEMM BN = 512 vs 256 on the 3B shapes and square shapes
mkdir -p gpurun_out
for f in 3B store; do
  echo "== BN default $f"; timeout 300 python scripts/microbench.py gemm "$f"
  echo "== BN 512 $f"; ESM_GEMM_BN=512 timeout 300 python scripts/microbench.py gemm "$f"
done
