timeout 1200 python -m pytest tests/test_gpu_rows.py tests/test_gpu_spec.py tests/test_gpu_units.py tests/test_gpu_gemm.py tests/test_bench_contract.py -m gpu -q -p no:cacheprovider -x > gpurun_out/g3_gputests.log 2>&1
tail -5 gpurun_out/g3_gputests.log
