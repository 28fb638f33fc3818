# One GPU call that regenerates a round's evidence under gpurun_out/ (copy
# what is judged into profiles/<round>_*): the GPU suite, smoke, the default
# bench line and the reference arm, every workload x dtype, the torch.compile
# comparators (untransformed Inductor, and the gm_compile front door), the
# launch list of the default bench and one `ncu --set full` capture of its
# fused kernels.
set -x
R=${ROUND:-r02}
timeout 2700 python -m pytest tests -m gpu -q -p no:cacheprovider -rf > gpurun_out/${R}_gputests.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${R}_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/${R}_bench.json 2> gpurun_out/${R}_bench.err
timeout 900 python bench.py --impl reference > gpurun_out/${R}_bench_ref.json 2> gpurun_out/${R}_bench_ref.err
: > gpurun_out/${R}_sweep.jsonl
for w in bigbird_like bigbird_attn bigbird_layer gemm_arms bart_step longformer_like phi4_like qwen_audio_like biogpt_like blenderbot_like flan_t5_like pegasus_like moe_minicpm_like; do
  for d in bf16 fp32; do
    timeout 600 python bench.py --workload $w --dtype $d --steps 100 --warmup 10 --no-compile --no-cpu-baseline 2>/dev/null >> gpurun_out/${R}_sweep.jsonl || echo "{\"workload\": \"$w\", \"dtype\": \"$d\", \"error\": true}" >> gpurun_out/${R}_sweep.jsonl
  done
done
ALL=bigbird_like,bigbird_attn,bigbird_layer,gemm_arms,bart_step,longformer_like,phi4_like,qwen_audio_like,biogpt_like,blenderbot_like,flan_t5_like,pegasus_like,moe_minicpm_like
timeout 1800 python tools/compare_inductor.py --workloads $ALL --dtype fp32 > gpurun_out/${R}_inductor_fp32.jsonl 2>/dev/null
timeout 1800 python tools/compare_inductor.py --workloads $ALL --dtype bf16 > gpurun_out/${R}_inductor_bf16.jsonl 2>/dev/null
timeout 1800 python tools/compare_frontdoor.py > gpurun_out/${R}_frontdoor.jsonl 2>/dev/null
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${R}_launches.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-compile > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'gm_(region|row)_' -s 4 -c 4 -o gpurun_out/${R}_prof python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-compile > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/${R}_prof.ncu-rep gpurun_out/${R}_ncu_regions.json
ls -la gpurun_out
timeout 900 python tools/frontdoor_overhead.py blenderbot_like pegasus_like phi4_like bigbird_layer > gpurun_out/${R}_frontdoor_overhead.jsonl 2>/dev/null
ROUND=$R bash tools/ncu_all_workloads.sh > gpurun_out/${R}_ncu_all.log 2>&1
ls gpurun_out
