set -x
R=${ROUND:-r02}
python /root/repo/uc_debug.py > gpurun_out/${R}_uc_debug.log 2>&1; cat gpurun_out/${R}_uc_debug.log | grep -v DEBUG | tail -8
timeout 900 python -m pytest tests/test_dynamo_backend.py -m gpu -q -p no:cacheprovider > gpurun_out/${R}_dyn_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/${R}_dyn_tests.log; grep -n "^E " gpurun_out/${R}_dyn_tests.log | head
: > gpurun_out/${R}_ab_rows.jsonl
for d in fp32 bf16; do
timeout 900 python tools/ab_regions.py --workload bigbird_layer --dtype $d --rounds 7 \
  --variant early:GM_ROW_EARLY_PERIODIC=1 --variant late: --variant early_minb3:GM_ROW_EARLY_PERIODIC=1,GM_ROW_MINB=3 \
  --variant late_minb3:GM_ROW_MINB=3 --variant late_minb4:GM_ROW_MINB=4 >> gpurun_out/${R}_ab_rows.jsonl 2>gpurun_out/${R}_ab_rows.err
done
cat gpurun_out/${R}_ab_rows.jsonl; tail -3 gpurun_out/${R}_ab_rows.err
timeout 900 python tools/frontdoor_overhead.py blenderbot_like pegasus_like phi4_like > gpurun_out/${R}_frontdoor_overhead.jsonl 2>/dev/null; cat gpurun_out/${R}_frontdoor_overhead.jsonl
