nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/g1_smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/g1_gputests.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g1_smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/g1_bench.json 2> gpurun_out/g1_bench.err
timeout 600 python bench.py --impl reference > gpurun_out/g1_bench_ref.json 2> gpurun_out/g1_bench_ref.err
ls -la gpurun_out
