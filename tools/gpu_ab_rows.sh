# A/B of row-kernel code generation (periodic-input load placement, register
# caps) on the encoder layer, row-kernel GPU parity, the default bench line
# (row kernels now time themselves in-kernel), and the front door.
set -x
R=${ROUND:-r02}
timeout 900 python -m pytest tests/test_gpu_rows.py tests/test_dynamo_backend.py -m gpu -q -p no:cacheprovider -x > gpurun_out/${R}_rows_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/${R}_rows_tests.log
for d in fp32 bf16; do
timeout 900 python tools/ab_regions.py --workload bigbird_layer --dtype $d --rounds 7 \
  --variant early:GM_ROW_EARLY_PERIODIC=1 --variant late: --variant early_minb3:GM_ROW_EARLY_PERIODIC=1,GM_ROW_MINB=3 \
  --variant late_minb3:GM_ROW_MINB=3 --variant late_minb4:GM_ROW_MINB=4 >> gpurun_out/${R}_ab_rows.jsonl 2>gpurun_out/${R}_ab_rows.err
done
cat gpurun_out/${R}_ab_rows.jsonl
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/${R}_bench2.json 2> gpurun_out/${R}_bench2.err; echo "bench rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/${R}_bench2.json').read().strip().splitlines()[-1])
print(d['value'], d['ms_per_step'], json.dumps(d['roofline']))
for k in d['kernels']: print(k['name'], round(k['ms']*1e3,1), round(k.get('ms_events',0)*1e3,1), k['how'][:40])
print(d.get('compile',{}).get('speedup_vs_compile'))"
timeout 1500 python tools/compare_frontdoor.py > gpurun_out/${R}_frontdoor.jsonl 2>gpurun_out/${R}_frontdoor.err
cat gpurun_out/${R}_frontdoor.jsonl | cut -c1-200
