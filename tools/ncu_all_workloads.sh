# One `ncu --set full` capture of the region kernels of every workload x
# dtype (1 GPU), summarised into profiles/${ROUND}_<workload>_<dtype>_ncu_regions.json
# — the files bench.py reads the per-kernel DRAM `traffic` from.  Skips the
# first 8 region launches (compile-time warm-ups, the first speculative
# misprediction) and captures the next 8.
set -x
ROUND=${ROUND:-r02}
WORKLOADS=${WORKLOADS:-"bigbird_layer longformer_like phi4_like qwen_audio_like biogpt_like blenderbot_like flan_t5_like pegasus_like moe_minicpm_like bart_step bigbird_like bigbird_attn gemm_arms"}
mkdir -p gpurun_out
for w in $WORKLOADS; do
  for d in bf16 fp32; do
    timeout 600 ncu --set full --clock-control none -k regex:'gm_(region|row)_' -s 8 -c 8 -o gpurun_out/prof_${w}_${d} \
      python bench.py --workload $w --dtype $d --steps 3 --warmup 3 --no-cpu-baseline --no-compile > gpurun_out/ncu_${w}_${d}.log 2>&1
    python tools/ncu_summary.py gpurun_out/prof_${w}_${d}.ncu-rep profiles/${ROUND}_${w}_${d}_ncu_regions.json \
      > /dev/null 2>&1 && cp profiles/${ROUND}_${w}_${d}_ncu_regions.json gpurun_out/
    rm -f gpurun_out/prof_${w}_${d}.ncu-rep  # gpurun copies back <= 64 MiB
  done
done
