# A/B: LayerNorm weight / bias staged in shared memory by cp.async (default)
# vs loaded from global after the row statistics (GM_ROW_NO_SMEM_WB=1);
# GPU parity of every row / fuzz / program test in the new form; bench.
for d in fp32 bf16; do
timeout 900 python tools/ab_regions.py --workload bigbird_layer --dtype $d --rounds 9 --variant smem: --variant global:GM_ROW_NO_SMEM_WB=1 2>/dev/null
done
timeout 1500 python -m pytest tests/test_gpu_rows.py tests/test_gpu_fuzz.py tests/test_gpu_programs.py -m gpu -q -p no:cacheprovider -rf 2>&1 | grep -E "FAILED|passed|failed" | tail -4
timeout 900 python bench.py --no-cpu-baseline --steps 100 --warmup 10 > gpurun_out/r02_bench_smemwb.json 2>/dev/null
python -c "
import json; d=json.loads(open('gpurun_out/r02_bench_smemwb.json').read().strip().splitlines()[-1])
print(d['value'], d['ms_per_step'], d['compile']['speedup_vs_compile'], json.dumps(d['roofline']['fused_kernels_frac']))
for k in d['kernels']: print(k['name'], round(k['ms']*1e3,1))"
