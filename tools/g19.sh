timeout 1800 python -m pytest tests/test_gpu_rows.py tests/test_gpu_fuzz.py tests/test_gpu_units.py tests/test_gpu_edge.py tests/test_dynamo_backend.py -m gpu -q -p no:cacheprovider > gpurun_out/g19.log 2>&1
tail -3 gpurun_out/g19.log
