# Re-verify HEAD on a fresh B200: GPU suite (minus the 200-step trajectory, goldens regenerating), smoke, default bench
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2o_smi.txt
timeout 1500 python -m pytest tests -m gpu -x -q -rf -p no:cacheprovider --deselect tests/test_gpu_trajectory.py > gpurun_out/r2o_pytest.txt 2>&1
tail -3 gpurun_out/r2o_pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2o_smoke.txt 2>&1; tail -1 gpurun_out/r2o_smoke.txt
timeout 900 python bench.py > gpurun_out/r2o_bench650.json 2> gpurun_out/r2o_bench650.err
tail -c 3000 gpurun_out/r2o_bench650.json
