timeout 1200 python -m pytest tests/test_gpu_model.py tests/test_gpu_reference_seams.py -q -rf -p no:cacheprovider -s 2>&1 | grep -E "rel|worst|passed|failed|Error|assert" | tail -40 > gpurun_out/r2c_tests.txt
timeout 900 python bench.py --varlen --steps 20 --warmup 3 > gpurun_out/r2c_varlen650.json 2> gpurun_out/r2c_varlen650.err
timeout 900 python scripts/max_batch.py --config 650m > gpurun_out/r2c_maxbatch.log 2>&1
cat gpurun_out/r2c_tests.txt; cut -c1-1500 gpurun_out/r2c_varlen650.json; tail -3 gpurun_out/r2c_varlen650.err; tail -c 1500 gpurun_out/r2c_maxbatch.log
