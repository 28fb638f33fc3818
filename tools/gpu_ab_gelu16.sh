# A/B: 16-bit GELU with the erfc-fit erf (default) vs erff (GM_ACCURATE_GELU16=1);
# GPU parity of every test that runs GELU / programs in the new form.
for w in bigbird_layer; do for d in bf16 fp32; do
timeout 900 python tools/ab_regions.py --workload $w --dtype $d --rounds 9 --variant fast: --variant accurate:GM_ACCURATE_GELU16=1 2>/dev/null
done; done
timeout 1500 python -m pytest tests/test_gpu_rows.py tests/test_gpu_fuzz.py tests/test_gpu_programs.py tests/test_gpu_edge.py tests/test_gpu_units.py -m gpu -q -p no:cacheprovider -rf 2>&1 | grep -E "FAILED|passed|failed" | tail -6
