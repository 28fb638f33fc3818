for st in 1 0; do
  echo "== GM_STAGING=$st"
  GM_STAGING=$st GM_PROFILE=1 python tools/region_timeline.py --workload bigbird_like --dtype bf16 2>/dev/null
  GM_STAGING=$st GM_PROFILE=1 python tools/region_timeline.py --workload phi4_like --dtype fp32 2>/dev/null
  GM_STAGING=$st python bench.py --steps 100 --warmup 10 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench', d['value'], d['p50_ms'], [(k['name'][-16:], round(k['ms']*1e3,1)) for k in d['kernels']])"
done
