timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_programs.py -q -x --timeout 600 > gpurun_out/t_all.log 2>&1
tail -n 2 gpurun_out/t_all.log
GM_PROFILE=1 python tools/region_timeline.py --workload bigbird_like --dtype bf16 > gpurun_out/tl_bb.json 2>/dev/null
GM_PROFILE=1 python tools/region_timeline.py --workload phi4_like --dtype fp32 > gpurun_out/tl_phi4.json 2>/dev/null
GM_PROFILE=1 python tools/region_timeline.py --workload biogpt_like --dtype fp32 > gpurun_out/tl_biogpt.json 2>/dev/null
cat gpurun_out/tl_*.json
python bench.py --steps 100 --warmup 10 --no-cpu-baseline > gpurun_out/bench_bb_bf16.json 2> gpurun_out/bench_bb_bf16.err
python -c "import json; d=json.load(open('gpurun_out/bench_bb_bf16.json')); print(d['value'], d['p50_ms'], d['roofline'], d['clocks'])"
