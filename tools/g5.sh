timeout 900 python -m pytest tests/test_gpu_programs.py -m gpu -q -p no:cacheprovider -k "bigbird_attn or toy" > gpurun_out/g5_gputests.log 2>&1
tail -3 gpurun_out/g5_gputests.log
timeout 600 python bench.py --workload bigbird_attn --no-cpu-baseline --steps 50 --warmup 5 > gpurun_out/g5_attn_fp32.json 2> gpurun_out/g5_attn.err
timeout 600 python bench.py --workload bigbird_attn --dtype bf16 --no-cpu-baseline --steps 50 --warmup 5 > gpurun_out/g5_attn_bf16.json 2>> gpurun_out/g5_attn.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/g5_launches_attn_bf16.csv python bench.py --workload bigbird_attn --dtype bf16 --steps 2 --warmup 3 --no-cpu-baseline --no-compile > /dev/null 2>&1
