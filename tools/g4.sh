timeout 600 python bench.py --no-compile > gpurun_out/g4_bench.json 2> gpurun_out/g4_bench.err
timeout 600 python bench.py --dtype bf16 --no-compile --no-cpu-baseline > gpurun_out/g4_bench_bf16.json 2>> gpurun_out/g4_bench.err
