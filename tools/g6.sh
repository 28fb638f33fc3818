timeout 1500 python -m pytest tests/test_gpu_rows.py tests/test_gpu_spec.py tests/test_bench_contract.py tests/test_dynamo_backend.py -m gpu -q -p no:cacheprovider > gpurun_out/g6_gputests.log 2>&1
tail -3 gpurun_out/g6_gputests.log
timeout 600 python bench.py --workload bigbird_attn --no-cpu-baseline --steps 50 --warmup 5 > gpurun_out/g6_attn_fp32.json 2> gpurun_out/g6_attn.err
timeout 600 python bench.py --workload bigbird_attn --dtype bf16 --no-cpu-baseline --steps 50 --warmup 5 > gpurun_out/g6_attn_bf16.json 2>> gpurun_out/g6_attn.err
timeout 600 python bench.py --no-compile > gpurun_out/g6_bench.json 2> gpurun_out/g6_bench.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gm_row -c 2 -o gpurun_out/g6_prof_row python bench.py --workload bigbird_attn --dtype bf16 --steps 2 --warmup 3 --no-cpu-baseline --no-compile > gpurun_out/g6_ncu.log 2>&1
