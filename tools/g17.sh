timeout 1800 python -m pytest tests/test_gpu_spec.py tests/test_gpu_fuzz.py tests/test_gpu_programs.py tests/test_bench_contract.py -m gpu -q -p no:cacheprovider > gpurun_out/g17.log 2>&1
tail -3 gpurun_out/g17.log
rm -f gpurun_out/g17_ab.jsonl
for cfg in "" "GM_SAMPLE=global" "GM_SAMPLE=0"; do
for w in bigbird_like phi4_like qwen_audio_like; do for d in fp32 bf16; do
  env $cfg python bench.py --workload $w --dtype $d --no-compile --no-cpu-baseline --steps 200 --warmup 10 > /tmp/ab.json 2>/dev/null
  python -c "
import json
d=json.loads(open('/tmp/ab.json').read().strip().splitlines()[-1])
print(json.dumps({'cfg': '$cfg' or 'cta', 'w': '$w', 'd': '$d', 'ms_per_step': d['ms_per_step'], 'spec': d['speculation'], 'frac': d['roofline']['frac'], 'kernels': [{k: v for k, v in x.items() if k.startswith('ms')} for x in d['kernels']]}))
" >> gpurun_out/g17_ab.jsonl
done; done; done
