# Round-2 final evidence: GPU suite (incl. the 200-step trajectory), smoke, default bench (650M)
# with the CPU baseline and e2e, the reference arm, ncu launch list of one eager 650M step, ncu full captures of
# the top kernels (GEMM FC1 forward, attention backward / forward at 650M, LayerNorm backward)
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/r3r_smi.txt
timeout 1800 python -m pytest tests -m gpu -q -rf -p no:cacheprovider > gpurun_out/r3r_pytest.txt 2>&1
tail -3 gpurun_out/r3r_pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r3r_smoke.txt 2>&1; tail -1 gpurun_out/r3r_smoke.txt
timeout 900 python bench.py > gpurun_out/r3r_bench650.json 2> gpurun_out/r3r_bench650.err; tail -c 600 gpurun_out/r3r_bench650.json
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r3r_ref.json 2> gpurun_out/r3r_ref.err; tail -c 400 gpurun_out/r3r_ref.json
# ncu: eager launch list of one step (after the same command ran clean)
timeout 600 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-profile --no-graph > gpurun_out/r3r_eager.json 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 1600 --csv \
  --log-file gpurun_out/r3r_launches_650m.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-profile --no-graph > gpurun_out/r3r_ncu_list.log 2>&1
python scripts/ncu_summary.py gpurun_out/r3r_launches_650m.csv > gpurun_out/r3r_launches_650m_summary.txt 2>&1; cat gpurun_out/r3r_launches_650m_summary.txt
export MB_NOGRAPH=1
python scripts/microbench.py gemm "650M fc1 fwd " > gpurun_out/r3r_mbg.txt 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_tc_kernel -s 3 -c 1 -o gpurun_out/r3r_gemm_fc1 python scripts/microbench.py gemm "650M fc1 fwd " > gpurun_out/r3r_ncu_gemm.log 2>&1
python scripts/microbench.py attn 16,20,1024,64 > gpurun_out/r3r_mba.txt 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"bwd_kernel|fwd_kernel" -s 0 -c 1 -o gpurun_out/r3r_attn650 python scripts/microbench.py attn 16,20,1024,64 > gpurun_out/r3r_ncu_attn.log 2>&1
python scripts/microbench.py ln > gpurun_out/r3r_mbl.txt 2>&1 && \
timeout 600 ncu --set full --clock-control none -k regex:"ln_bwd_kernel|ln_fwd_kernel" -s 40 -c 4 -o gpurun_out/r3r_ln python scripts/microbench.py ln > gpurun_out/r3r_ncu_ln.log 2>&1
ls gpurun_out/r3r_*
