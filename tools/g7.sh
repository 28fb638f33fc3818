timeout 1500 python -m pytest tests/test_gpu_rows.py tests/test_gpu_spec.py tests/test_gpu_gemm.py -m gpu -q -p no:cacheprovider -x > gpurun_out/g7_gputests.log 2>&1
tail -3 gpurun_out/g7_gputests.log
rm -f gpurun_out/ab_spec.jsonl
for cfg in "" "GM_SPEC_CONFIDENT=0" "GM_SPEC_CONFIDENT=99"; do
  env $cfg python bench.py --no-compile --no-cpu-baseline --steps 200 --warmup 10 > /tmp/ab.json 2>/dev/null
  python -c "
import json
d=json.loads(open('/tmp/ab.json').read().strip().splitlines()[-1])
print(json.dumps({'cfg': '$cfg' or 'default', 'ms_per_step': d['ms_per_step'], 'spec': d['speculation'], 'kernels': [{k: v for k, v in x.items() if k.startswith('ms')} for x in d['kernels']]}))
" >> gpurun_out/g7_ab.jsonl
done
timeout 600 python bench.py --workload bigbird_attn --no-cpu-baseline --steps 50 --warmup 5 > gpurun_out/g7_attn_fp32.json 2> gpurun_out/g7_attn.err
timeout 600 python bench.py --workload bigbird_attn --dtype bf16 --no-cpu-baseline --steps 50 --warmup 5 > gpurun_out/g7_attn_bf16.json 2>> gpurun_out/g7_attn.err
