set -x
python bench.py --steps 100 --warmup 10 > gpurun_out/bench_bb_bf16.json 2> gpurun_out/bench_bb_bf16.err
python bench.py --workload phi4_like --dtype fp32 --steps 100 --warmup 10 --no-cpu-baseline > gpurun_out/bench_phi4_fp32.json 2> gpurun_out/bench_phi4.err
python bench.py --workload bigbird_like --dtype fp32 --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/bench_bb_fp32.json 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bb.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gm_region -s 2 -c 4 -o gpurun_out/prof_bb python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
ls -la gpurun_out
