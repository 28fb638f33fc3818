# A/B of the speculation policy and the exact entry's staging on the default
# bench (bigbird_like fp32, rotating inputs), same box, interleaved twice
for rep in 1 2; do
for cfg in "" "GM_STAGING=0" "GM_SPEC_CONFIDENT=0" "GM_SPEC_CONFIDENT=0 GM_STAGING=0" "GM_SPEC_CONFIDENT=99"; do
  env $cfg python bench.py --no-compile --no-cpu-baseline --steps 200 --warmup 10 > /tmp/ab.json 2>/dev/null
  python -c "
import json,sys
d=json.loads(open('/tmp/ab.json').read().strip().splitlines()[-1])
print(json.dumps({'cfg': '$cfg' or 'default', 'rep': $rep, 'ms_per_step': d['ms_per_step'], 'spec': d['speculation'], 'kernels': [{k: v for k, v in x.items() if k.startswith('ms')} for x in d['kernels']]}))
" >> gpurun_out/ab_spec.jsonl
done
done
