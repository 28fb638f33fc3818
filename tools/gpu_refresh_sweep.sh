# Refresh the per-workload evidence on the final tree: sweep + ncu captures.
R=${ROUND:-r02}
: > gpurun_out/${R}_sweep.jsonl
for w in bigbird_like bigbird_attn bigbird_layer gemm_arms bart_step longformer_like phi4_like qwen_audio_like biogpt_like blenderbot_like flan_t5_like pegasus_like moe_minicpm_like; do
  for d in bf16 fp32; do
    timeout 600 python bench.py --workload $w --dtype $d --steps 100 --warmup 10 --no-compile --no-cpu-baseline 2>/dev/null >> gpurun_out/${R}_sweep.jsonl || echo "{\"workload\": \"$w\", \"dtype\": \"$d\", \"error\": true}" >> gpurun_out/${R}_sweep.jsonl
  done
done
ROUND=$R bash tools/ncu_all_workloads.sh > gpurun_out/${R}_ncu_all.log 2>&1
echo done
