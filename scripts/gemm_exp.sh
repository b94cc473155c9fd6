# GEMM bottleneck experiments (ESM_GEMM_EXP=1: no operand loads, 2: no MMAs; see gemm.cu), built as separate
# libraries under build/exp/ and timed with the microbenchmark (ESM_LIB_PATH selects the library).
#   bash scripts/gemm_exp.sh build   (CPU container)        bash scripts/gemm_exp.sh run   (B200)
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
if [ "$1" = "build" ]; then
  mkdir -p $ROOT/build/exp
  for e in 1 2; do
    nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC --expt-relaxed-constexpr \
      -I$ROOT/include -DESM_GEMM_EXP=$e -c $ROOT/paper_2411_10548_b200/csrc/gemm.cu -o $ROOT/build/exp/gemm_$e.o
    objs=$(ls $ROOT/build/*.o | grep -v "/gemm.o")
    nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $ROOT/build/exp/libesm_gemmexp$e.so $objs $ROOT/build/exp/gemm_$e.o -ldl
  done
else
  echo "== product"; python $ROOT/scripts/microbench.py gemm 650M
  for e in 1 2; do echo "== ESM_GEMM_EXP=$e"; ESM_LIB_PATH=$ROOT/build/exp/libesm_gemmexp$e.so python $ROOT/scripts/microbench.py gemm 650M; done
fi
