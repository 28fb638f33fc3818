GM_PROFILE=1 python tools/region_timeline.py --workload bigbird_like --dtype bf16 > gpurun_out/tl_bb.json 2>&1
GM_PROFILE=1 python tools/region_timeline.py --workload phi4_like --dtype fp32 > gpurun_out/tl_phi4.json 2>&1
GM_PROFILE=1 python tools/region_timeline.py --workload biogpt_like --dtype fp32 > gpurun_out/tl_biogpt.json 2>&1
cat gpurun_out/tl_*.json
