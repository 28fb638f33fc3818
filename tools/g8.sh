timeout 1500 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_rows.py tests/test_gpu_programs.py -m gpu -q -p no:cacheprovider -x -k "not corpus_manifest" > gpurun_out/g8_gputests.log 2>&1
tail -3 gpurun_out/g8_gputests.log
timeout 600 python bench.py --workload bigbird_attn --no-cpu-baseline --steps 50 --warmup 5 > gpurun_out/g8_attn_fp32.json 2> gpurun_out/g8_attn.err
timeout 600 python bench.py --workload bigbird_attn --dtype bf16 --no-cpu-baseline --steps 50 --warmup 5 > gpurun_out/g8_attn_bf16.json 2>> gpurun_out/g8_attn.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/g8_launches_attn_bf16.csv python bench.py --workload bigbird_attn --dtype bf16 --steps 2 --warmup 3 --no-cpu-baseline --no-compile > /dev/null 2>&1
