timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_bb.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
timeout 1200 python tools/compare_inductor.py --workloads bigbird_like,bart_step,phi4_like,qwen_audio_like,biogpt_like --dtype bf16 > gpurun_out/compare_bf16.jsonl 2> gpurun_out/compare_bf16.err
cat gpurun_out/compare_bf16.jsonl
tail -3 gpurun_out/compare_bf16.err
