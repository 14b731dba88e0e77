timeout 1200 python -m pytest tests/test_gpu_relabel.py tests/test_gpu_variants.py tests/test_gpu_slabs.py -x -q > gpurun_out/s20_tests.log 2>&1
tail -2 gpurun_out/s20_tests.log
