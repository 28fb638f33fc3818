set -x
R=${ROUND:-r02}
: > gpurun_out/${R}_ab_rows_u.jsonl
for d in fp32 bf16; do
timeout 900 python tools/ab_regions.py --workload bigbird_layer --dtype $d --rounds 9 \
  --variant base: --variant u1:GM_ROW_U=1 --variant u2:GM_ROW_U=2 >> gpurun_out/${R}_ab_rows_u.jsonl 2>>gpurun_out/${R}_ab_rows_u.err
done
cat gpurun_out/${R}_ab_rows_u.jsonl; tail -3 gpurun_out/${R}_ab_rows_u.err
GM_ROW_U=1 timeout 900 python -m pytest tests/test_gpu_rows.py -m gpu -q -p no:cacheprovider -x > gpurun_out/${R}_rows_u1_tests.log 2>&1; echo "u1 tests rc=$?"; tail -2 gpurun_out/${R}_rows_u1_tests.log
timeout 900 python tools/frontdoor_overhead.py blenderbot_like pegasus_like > gpurun_out/${R}_frontdoor_overhead.jsonl 2>/dev/null; cat gpurun_out/${R}_frontdoor_overhead.jsonl
