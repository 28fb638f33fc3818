timeout 1800 python -m pytest tests/test_bench_contract.py tests/test_gpu_programs.py -m gpu -q -p no:cacheprovider > gpurun_out/g21.log 2>&1
tail -3 gpurun_out/g21.log
timeout 900 python bench.py > gpurun_out/g21_bench.json 2> gpurun_out/g21_bench.err
timeout 900 python bench.py --impl reference > gpurun_out/g21_ref.json 2> gpurun_out/g21_ref.err
