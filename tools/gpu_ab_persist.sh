# A/B of persistent row kernels (GM_ROW_PERSIST, with / without the L2
# prefetch of the next row group) on the encoder layer and attention, plus
# row-kernel GPU parity in the persistent form, and the forward-context bench.
R=${ROUND:-r02}
for w in bigbird_layer bigbird_attn; do for d in fp32 bf16; do
timeout 900 python tools/ab_regions.py --workload $w --dtype $d --rounds 9 \
  --variant base: --variant persist:GM_ROW_PERSIST=1 --variant persist_nopf:GM_ROW_PERSIST=1,GM_ROW_NOPF=1 2>/dev/null
done; done
GM_ROW_PERSIST=1 timeout 900 python -m pytest tests/test_gpu_rows.py -m gpu -q -p no:cacheprovider -x 2>&1 | tail -1
summ() { python -c "
import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[2], round(d['ms_per_step'],4), ' '.join(f\"{k['name'][:14]}={k['ms']*1e3:.1f}\" for k in d['kernels']))" $1 $2; }
for v in base persist; do
  if [ $v = persist ]; then export GM_ROW_PERSIST=1; else unset GM_ROW_PERSIST; fi
  timeout 600 python bench.py --steps 100 --warmup 10 --no-cpu-baseline --no-compile > gpurun_out/${R}_p_$v.json 2>/dev/null; summ gpurun_out/${R}_p_$v.json $v
  timeout 600 python bench.py --steps 100 --warmup 10 --no-cpu-baseline --no-compile --dtype bf16 > gpurun_out/${R}_p_${v}_bf16.json 2>/dev/null; summ gpurun_out/${R}_p_${v}_bf16.json ${v}_bf16
done
