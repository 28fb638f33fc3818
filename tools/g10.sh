timeout 900 python -m pytest tests/test_dynamo_backend.py tests/test_gpu_programs.py -m gpu -q -p no:cacheprovider -k "moe or aot or gm_compile" > gpurun_out/g10_gputests.log 2>&1
tail -3 gpurun_out/g10_gputests.log
timeout 1200 python tools/compare_frontdoor.py > gpurun_out/g10_frontdoor.jsonl 2> /dev/null
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/g10_launches_attn_fp32.csv python bench.py --workload bigbird_attn --steps 2 --warmup 3 --no-cpu-baseline --no-compile > /dev/null 2>&1
for w in bigbird_like phi4_like; do for d in fp32 bf16; do
GM_SPEC_CONFIDENT=99 timeout 300 python tools/region_timeline.py --workload $w --dtype $d > gpurun_out/g10_tl_exact_${w}_${d}.txt 2>&1
GM_SPEC_CONFIDENT=0 timeout 300 python tools/region_timeline.py --workload $w --dtype $d > gpurun_out/g10_tl_spec_${w}_${d}.txt 2>&1
done; done
