set -x
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_programs.py -q -x --timeout 600 > gpurun_out/t_all.log 2>&1
tail -n 3 gpurun_out/t_all.log
python bench.py --steps 100 --warmup 10 --no-cpu-baseline > gpurun_out/bench_bb_bf16.json 2> gpurun_out/bench_bb_bf16.err
python bench.py --workload phi4_like --dtype fp32 --steps 100 --warmup 10 --no-cpu-baseline > gpurun_out/bench_phi4_fp32.json 2> gpurun_out/bench_phi4.err
python bench.py --workload biogpt_like --dtype fp32 --steps 100 --warmup 10 --no-cpu-baseline > gpurun_out/bench_biogpt_fp32.json 2> gpurun_out/bench_biogpt.err
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap --format=csv,noheader,nounits > gpurun_out/smi_probe.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gm_region -s 2 -c 2 -o gpurun_out/prof_bb2 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
