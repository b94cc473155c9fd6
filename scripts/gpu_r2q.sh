# ncu source-level captures of the attention backward (35M dh=24, 650M dh=64)
mkdir -p gpurun_out
export MB_NOGRAPH=1
python scripts/microbench.py attn 32,20,1024,24 > gpurun_out/r2q_mb.txt 2>&1 && python scripts/microbench.py attn 16,20,1024,64 >> gpurun_out/r2q_mb.txt 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"bwd_kernel" -s 3 -c 1 -o gpurun_out/r2q_bwd35 python scripts/microbench.py attn 32,20,1024,24 > gpurun_out/r2q_ncu35.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"bwd_kernel" -s 3 -c 1 -o gpurun_out/r2q_bwd650 python scripts/microbench.py attn 16,20,1024,64 > gpurun_out/r2q_ncu650.log 2>&1
cat gpurun_out/r2q_mb.txt; tail -2 gpurun_out/r2q_ncu650.log
