# A/B: periodic (broadcast) inputs with the period as a compile-time constant
# (default) vs read from the descriptor at run time (GM_PERIODIC_RUNTIME=1).
for w in gemm_arms bigbird_like phi4_like qwen_audio_like blenderbot_like; do for d in fp32 bf16; do
timeout 900 python tools/ab_regions.py --workload $w --dtype $d --rounds 9 --variant const: --variant runtime:GM_PERIODIC_RUNTIME=1 2>/dev/null
done; done
timeout 900 python -m pytest tests/test_gpu_programs.py tests/test_gpu_gemm.py tests/test_gpu_kernels.py -m gpu -q -p no:cacheprovider -x 2>&1 | tail -1
