R=${ROUND:-r02}
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -rf > gpurun_out/${R}_gputests_final.log 2>&1; echo "tests rc=$?"; grep -E "FAILED|passed|failed" gpurun_out/${R}_gputests_final.log | tail -5
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/${R}_bench_final.json 2> gpurun_out/${R}_bench_final.err; echo "bench rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/${R}_bench_final.json').read().strip().splitlines()[-1])
print(d['value'], d['ms_per_step'], d['e2e']['value'], d['compile']['speedup_vs_compile'], d['clocks'])
print(json.dumps(d['roofline']))"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${R}_launches.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-compile > /dev/null 2>&1; echo "ncu1 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'gm_(region|row)_' -s 8 -c 8 -o gpurun_out/${R}_prof python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-compile > /dev/null 2>&1; echo "ncu2 rc=$?"
python tools/ncu_summary.py gpurun_out/${R}_prof.ncu-rep gpurun_out/${R}_ncu_regions.json
