timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_programs.py -q -x --timeout 600 > gpurun_out/t_all.log 2>&1
tail -n 2 gpurun_out/t_all.log
for st in 1 0; do
  echo "== GM_STAGING=$st"
  GM_STAGING=$st GM_PROFILE=1 python tools/region_timeline.py --workload bigbird_like --dtype bf16 2>/dev/null
  GM_STAGING=$st GM_PROFILE=1 python tools/region_timeline.py --workload phi4_like --dtype fp32 2>/dev/null
  GM_STAGING=$st GM_PROFILE=1 python tools/region_timeline.py --workload qwen_audio_like --dtype bf16 2>/dev/null
  GM_STAGING=$st python bench.py --steps 100 --warmup 10 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench', d['value'], d['p50_ms'], [(k['name'][-16:], round(k['ms']*1e3,1)) for k in d['kernels']])"
done
