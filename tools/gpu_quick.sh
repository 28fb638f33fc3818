set -x
R=r02
nvidia-smi -L
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/${R}_gputests.log 2>&1; echo "tests rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${R}_smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/${R}_bench.json 2> gpurun_out/${R}_bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/${R}_bench_ref.json 2> gpurun_out/${R}_bench_ref.err; echo "ref rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${R}_launches.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-compile > /dev/null 2>&1; echo "ncu1 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'gm_(region|row)_' -s 8 -c 8 -o gpurun_out/${R}_prof python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-compile > /dev/null 2>&1; echo "ncu2 rc=$?"
python tools/ncu_summary.py gpurun_out/${R}_prof.ncu-rep gpurun_out/${R}_ncu_regions.json
tail -3 gpurun_out/${R}_gputests.log; cat gpurun_out/${R}_bench.json | head -c 3000
