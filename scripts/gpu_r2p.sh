# GPU suite with the reference installed; ncu source-level captures of the attention kernels (35M dh=24, 650M dh=64)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -rf -p no:cacheprovider --deselect tests/test_gpu_trajectory.py > gpurun_out/r2p_pytest.txt 2>&1
tail -3 gpurun_out/r2p_pytest.txt
export MB_NOGRAPH=1
python scripts/microbench.py attn 32,20,1024,24 > gpurun_out/r2p_mb.txt 2>&1 && python scripts/microbench.py attn 16,20,1024,64 >> gpurun_out/r2p_mb.txt 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"bwd_kernel|fwd_kernel" -s 6 -c 2 -o gpurun_out/r2p_attn35 python scripts/microbench.py attn 32,20,1024,24 > gpurun_out/r2p_ncu35.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"bwd_kernel|fwd_kernel" -s 6 -c 2 -o gpurun_out/r2p_attn650 python scripts/microbench.py attn 16,20,1024,64 > gpurun_out/r2p_ncu650.log 2>&1
cat gpurun_out/r2p_mb.txt
