timeout 1800 python -m pytest tests/test_gpu_programs.py -m gpu -q -p no:cacheprovider -k "bigbird_layer or toy or bigbird_attn" > gpurun_out/g20.log 2>&1
tail -3 gpurun_out/g20.log
timeout 600 python bench.py --workload bigbird_layer --no-cpu-baseline --steps 50 --warmup 5 > gpurun_out/g20_layer_fp32.json 2>/dev/null
timeout 600 python bench.py --workload bigbird_layer --dtype bf16 --no-cpu-baseline --steps 50 --warmup 5 > gpurun_out/g20_layer_bf16.json 2>/dev/null
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/g20_launches_layer_bf16.csv python bench.py --workload bigbird_layer --dtype bf16 --steps 2 --warmup 3 --no-cpu-baseline --no-compile > /dev/null 2>&1
