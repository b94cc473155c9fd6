# dropout under CUDA-graph replay vs eager
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_attn_dropout.py -x -q -rf -s -p no:cacheprovider -k graph > gpurun_out/r4m_pytest.txt 2>&1
tail -3 gpurun_out/r4m_pytest.txt; grep "eager vs graph" gpurun_out/r4m_pytest.txt
