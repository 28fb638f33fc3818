timeout 300 python tools/sync_probe.py > gpurun_out/g2_sync.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/g2_gputests.log 2>&1
tail -5 gpurun_out/g2_gputests.log
