# One GPU call that regenerates the round's evidence under gpurun_out/:
# GPU tests, smoke, the default bench line, the reference arm, the config
# sweep, the launch list, one ncu --set full capture of the region kernels,
# the region timelines and the conditional-node cost.
set -x
python -m pytest tests -m gpu -q > gpurun_out/gputests.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
bash tools/sweep.sh > gpurun_out/sweep.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bb.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gm_region -s 2 -c 4 -o gpurun_out/prof_bb python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
GM_PROFILE=1 python tools/region_timeline.py --workload bigbird_like --dtype bf16 > gpurun_out/tl_bb_bf16.txt 2>&1
GM_PROFILE=1 python tools/region_timeline.py --workload phi4_like --dtype fp32 > gpurun_out/tl_phi4_fp32.txt 2>&1
timeout 120 ./tools/cond_node_bench > gpurun_out/cond_node.txt 2>&1
ls -la gpurun_out
