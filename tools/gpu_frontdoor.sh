set -x
R=${ROUND:-r02}
timeout 900 python -m pytest tests/test_dynamo_backend.py tests/test_gpu_logring.py -m gpu -q -p no:cacheprovider > gpurun_out/${R}_dyn_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/${R}_dyn_tests.log; grep -n "^E " gpurun_out/${R}_dyn_tests.log | head
timeout 900 python tools/frontdoor_overhead.py blenderbot_like pegasus_like > gpurun_out/${R}_frontdoor_overhead.jsonl 2>/dev/null; cat gpurun_out/${R}_frontdoor_overhead.jsonl
timeout 1500 python tools/compare_frontdoor.py > gpurun_out/${R}_frontdoor.jsonl 2>gpurun_out/${R}_frontdoor.err
cut -c1-220 gpurun_out/${R}_frontdoor.jsonl
