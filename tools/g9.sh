# round-2 evidence pass: full GPU suite, smoke, default bench + reference
# arm, every workload x dtype, torch.compile comparators, front door
timeout 2700 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/g9_gputests.log 2>&1
tail -5 gpurun_out/g9_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g9_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/g9_bench.json 2> gpurun_out/g9_bench.err
timeout 900 python bench.py --impl reference > gpurun_out/g9_bench_ref.json 2> gpurun_out/g9_bench_ref.err
: > gpurun_out/g9_sweep.jsonl
for w in bigbird_like bigbird_attn gemm_arms bart_step longformer_like phi4_like qwen_audio_like biogpt_like blenderbot_like flan_t5_like pegasus_like moe_minicpm_like; do
  for d in bf16 fp32; do
    timeout 600 python bench.py --workload $w --dtype $d --steps 100 --warmup 10 --no-compile --no-cpu-baseline 2>/dev/null >> gpurun_out/g9_sweep.jsonl || echo "{\"workload\": \"$w\", \"dtype\": \"$d\", \"error\": true}" >> gpurun_out/g9_sweep.jsonl
  done
done
timeout 1800 python tools/compare_frontdoor.py > gpurun_out/g9_frontdoor.jsonl 2> gpurun_out/g9_frontdoor.err
ALL=bigbird_like,bigbird_attn,gemm_arms,bart_step,longformer_like,phi4_like,qwen_audio_like,biogpt_like,blenderbot_like,flan_t5_like,pegasus_like,moe_minicpm_like
timeout 1800 python tools/compare_inductor.py --workloads $ALL --dtype fp32 > gpurun_out/g9_inductor_fp32.jsonl 2> gpurun_out/g9_inductor.err
timeout 1800 python tools/compare_inductor.py --workloads $ALL --dtype bf16 > gpurun_out/g9_inductor_bf16.jsonl 2>> gpurun_out/g9_inductor.err
