# ncu full sets: GEMM 8192^3 with the 256x512 pair tile (auto-picked) and with the 256x256 tile (ESM_GEMM_BN=256)
mkdir -p gpurun_out
export MB_NOGRAPH=1
python scripts/microbench.py gemm "8192^3" > gpurun_out/r4c_mb.txt 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_tc_kernel -s 3 -c 1 -o gpurun_out/r4c_gemm8k_bn512 python scripts/microbench.py gemm "8192^3" > gpurun_out/r4c_ncu1.log 2>&1
ESM_GEMM_BN=256 timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_tc_kernel -s 3 -c 1 -o gpurun_out/r4c_gemm8k_bn256 python scripts/microbench.py gemm "8192^3" > gpurun_out/r4c_ncu2.log 2>&1
cat gpurun_out/r4c_mb.txt; ls gpurun_out/r4c_*
