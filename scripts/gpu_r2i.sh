export PATH=/usr/local/cuda/bin:$PATH
B="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-profile --no-graph"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 800 --csv --log-file gpurun_out/r2i_launches_650m.csv $B > gpurun_out/r2i_ncu_list.log 2>&1; echo "list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_tc_kernel --launch-skip 2 -c 1 -o gpurun_out/r2i_gemm_fc1_650m $B > gpurun_out/r2i_ncu_gemm.log 2>&1; echo "gemm rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:bwd_kernel -c 1 -o gpurun_out/r2i_attn_bwd_650m $B > gpurun_out/r2i_ncu_attn.log 2>&1; echo "attn rc=$?"
timeout 900 ncu --set full --clock-control none -k regex:"ln_bwd|qkv_rope_bwd_tile|xent|embed_bwd" -c 6 -o gpurun_out/r2i_membound_650m $B > gpurun_out/r2i_ncu_mem.log 2>&1; echo "mem rc=$?"
ls -la gpurun_out/ | grep r2i
