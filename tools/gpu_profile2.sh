timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_bb.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gm_region -s 4 -c 4 -o gpurun_out/prof_regions python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
timeout 300 python -m pytest tests/test_gpu_hardening.py -q > gpurun_out/t_hard.log 2>&1; tail -n 2 gpurun_out/t_hard.log
ls -la gpurun_out | head
