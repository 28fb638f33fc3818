R=${ROUND:-r02}
summ() { python -c "
import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[2], round(d['ms_per_step'],4), ' '.join(f\"{k['name'][:14]}={k['ms']*1e3:.1f}\" for k in d['kernels']))" $1 $2; }
for i in 1 2; do
for v in fwd rev; do
  if [ $v = rev ]; then export GM_ROW_REVERSE=1; else unset GM_ROW_REVERSE; fi
  timeout 600 python bench.py --steps 100 --warmup 10 --no-cpu-baseline --no-compile > gpurun_out/${R}_rev_$v.json 2>/dev/null
  summ gpurun_out/${R}_rev_$v.json $v
  timeout 600 python bench.py --steps 100 --warmup 10 --no-cpu-baseline --no-compile --dtype bf16 > gpurun_out/${R}_rev_${v}_bf16.json 2>/dev/null
  summ gpurun_out/${R}_rev_${v}_bf16.json ${v}_bf16
done
done
