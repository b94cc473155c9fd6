timeout 900 python -m pytest tests/test_gpu_kernels.py -q -rf -p no:cacheprovider -k "attention" -s 2>&1 | grep -v "^$" | tail -15 > gpurun_out/r2b_attn.txt
timeout 900 python -m pytest tests/test_gpu_reference_seams.py -q -rf -p no:cacheprovider -x 2>&1 | tail -30 > gpurun_out/r2b_seams.txt
cat gpurun_out/r2b_attn.txt gpurun_out/r2b_seams.txt | tail -30
