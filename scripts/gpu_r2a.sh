set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -q -rf -p no:cacheprovider > gpurun_out/r2a_tests.txt 2>&1; echo "tests rc=$?"
tail -5 gpurun_out/r2a_tests.txt
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/r2a_bench650.json 2> gpurun_out/r2a_bench650.err; echo "bench rc=$?"
timeout 600 python bench.py --config 35m --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2a_bench35.json 2> gpurun_out/r2a_bench35.err; echo "bench35 rc=$?"
cut -c1-600 gpurun_out/r2a_bench650.json
