# Build the attention-backward bottleneck experiments (ESM_ATTN_EXP=1..4, see attention_tc.cu) as separate
# libraries under build/exp/ and time each with the microbenchmark (ESM_LIB_PATH selects the library).
#   bash scripts/attn_bwd_exp.sh build     (CPU container)      bash scripts/attn_bwd_exp.sh run   (B200)
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
if [ "$1" = "build" ]; then
  mkdir -p $ROOT/build/exp
  for e in 1 2 3 4 5; do
    nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC --expt-relaxed-constexpr \
      -I$ROOT/include -DESM_ATTN_EXP=$e -c $ROOT/paper_2411_10548_b200/csrc/attention_tc.cu -o $ROOT/build/exp/attention_tc_$e.o
    objs=$(ls $ROOT/build/*.o | grep -v attention_tc.o)
    nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $ROOT/build/exp/libesm_exp$e.so $objs $ROOT/build/exp/attention_tc_$e.o -ldl
  done
else
  for s in 32,20,1024,24 16,20,1024,64; do
    echo "== $s: product"; python $ROOT/scripts/microbench.py attn $s
    for e in 1 2 3 4 5; do echo "== $s: ESM_ATTN_EXP=$e"; ESM_LIB_PATH=$ROOT/build/exp/libesm_exp$e.so python $ROOT/scripts/microbench.py attn $s; done
  done
fi
