export PATH=/usr/local/cuda/bin:$PATH
timeout 1200 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_geneformer.py -q -rf -p no:cacheprovider 2>&1 | grep -E "^E |passed|failed|FAILED" | head -20 > gpurun_out/r2k_tests.txt
B="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-profile --no-graph"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 800 --csv --log-file gpurun_out/r2k_launches_650m.csv $B > /dev/null 2>&1; echo "list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^bwd_kernel" -c 1 -o gpurun_out/r2k_attn_bwd_650m $B > gpurun_out/r2k_ncu_attn.log 2>&1; echo "attn rc=$?"
timeout 900 ncu --set full --clock-control none -k regex:"ln_fwd_kernel|delta_kernel|qkv_rope_bwd_tile" -c 3 -o gpurun_out/r2k_mem_650m $B > gpurun_out/r2k_ncu_mem.log 2>&1; echo "mem rc=$?"
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_step.py > gpurun_out/r2k_sanitizer_$tool.log 2>&1; echo "$tool rc=$?"; tail -3 gpurun_out/r2k_sanitizer_$tool.log
done
cat gpurun_out/r2k_tests.txt
