# attention backward: S/dP of block i+NBUF issued ahead of the pair's dQ MMAs -- parity + microbenchmark
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -rf -p no:cacheprovider -k "attention or attn" > gpurun_out/r2t_pytest.txt 2>&1
tail -3 gpurun_out/r2t_pytest.txt
python scripts/microbench.py attn 32,20,1024,24 > gpurun_out/r2t_mb.txt 2>&1
python scripts/microbench.py attn 16,20,1024,64 >> gpurun_out/r2t_mb.txt 2>&1
cat gpurun_out/r2t_mb.txt
